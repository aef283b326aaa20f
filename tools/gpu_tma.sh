# TMA ws pass check: gpu tests of the tall kernels, step bench A/B (TMA default vs the cp.async variant)
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py tests/test_gpu_solver.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_tma.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu_tma.log
for i in 1 2; do
timeout 300 python bench.py --no-tts --no-cpu --no-e2e > gpurun_out/bench_tma_$i.json 2>&1
RG_LIB_PATH=$PWD/paper_1604_01713_b200/_lib/variants/ws_ldgsts.so timeout 300 python bench.py --no-tts --no-cpu --no-e2e > gpurun_out/bench_ldgsts_$i.json 2>&1
done

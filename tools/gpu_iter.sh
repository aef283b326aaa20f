# iteration pass: tall-kernel + solver parity tests, the step bench, the per-kernel cycle profile
# (default library, then each variant named on the command line)
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py tests/test_gpu_r2.py tests/test_gpu_behaviour.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_iter.log
timeout 300 python bench.py --no-tts --no-cpu --no-e2e > gpurun_out/bench_iter.json 2>&1
timeout 600 python tools/prof_cycle.py --grid 256 --systems 1 --kernels > gpurun_out/abc_default.json 2>&1
for v in "$@"; do
RG_LIB_PATH=$PWD/paper_1604_01713_b200/_lib/variants/$v.so timeout 600 python tools/prof_cycle.py --grid 256 --systems 1 --kernels > gpurun_out/abc_$v.json 2>&1
done

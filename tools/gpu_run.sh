# one GPU evidence pass: gpu tests, default bench, ortho + spmm microbench lines (outputs under gpurun_out/)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02a.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu_r02a.log
timeout 900 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo "bench rc=$?"
timeout 300 python bench.py --workload ortho --steps 10 --warmup 3 > gpurun_out/ortho_r02a.json 2>&1
timeout 300 python bench.py --workload spmm --steps 20 --warmup 3 > gpurun_out/spmm_r02a.json 2>&1

# iteration pass: tall-kernel + solver parity tests, the step bench, the per-kernel cycle profile
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py tests/test_gpu_r2.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_iter.log
timeout 300 python bench.py --no-tts --no-cpu --no-e2e > gpurun_out/bench_iter.json 2>&1
timeout 600 python tools/prof_cycle.py --grid 256 --systems 1 --kernels > gpurun_out/cycle_iter.json 2> gpurun_out/cycle_iter.err

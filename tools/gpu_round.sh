# GPU pass: distributed + kernel parity tests, step evidence (bench line, launch list, ncu step capture,
# smoke), then the per-kernel cycle profile of cfg4 256^3 system 0
set -x
timeout 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_kernels.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_part.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_part.log
bash tools/evidence_step.sh
timeout 600 python tools/prof_cycle.py --grid 256 --systems 1 --kernels > gpurun_out/cycle_256.json 2> gpurun_out/cycle_256.err

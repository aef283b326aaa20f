# full -m gpu suite, then the time-to-solution probe and the cycle profile (cfg4 256^3)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/prof_tts.py --grid 256 --systems 2 > gpurun_out/prof_tts.txt 2>&1
timeout 600 python tools/prof_cycle.py --grid 256 --systems 1 --kernels > gpurun_out/cycle_pipe.json 2>&1

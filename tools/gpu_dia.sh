set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
python tools/prof_dia_build.py 256 > gpurun_out/dia_build.txt 2>&1
python tools/prof_spmm_dia.py > gpurun_out/spmm_dia.txt 2>&1
timeout 300 python bench.py --no-tts --no-cpu --no-e2e > gpurun_out/bench_dia.json 2>&1
timeout 900 python tools/prof_tts.py --grid 256 --systems 2 > gpurun_out/prof_tts3.txt 2>&1

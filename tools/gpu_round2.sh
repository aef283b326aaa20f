set -x
timeout 600 python -m pytest tests/test_gpu_distributed.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_dist.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_dist.log
timeout 600 python tools/ab_spmm.py paper_1604_01713_b200/_lib/variants/sp_d2w6.so paper_1604_01713_b200/_lib/variants/sp_d1w6.so > gpurun_out/ab_spmm.txt 2>&1
timeout 900 python tools/sweep.py --grid 128 --out gpurun_out/sweep_r02 > gpurun_out/sweep_r02.txt 2>&1
timeout 900 python tools/prof_tts.py --grid 256 --systems 2 > gpurun_out/prof_tts.txt 2>&1

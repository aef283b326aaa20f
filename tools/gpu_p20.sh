# p = 20 recycle passes on the three-tile ws kernel: parity tests, isolated pass
# timings at n = 2^24 (default library and an A/B variant), the per-kernel
# cycle profile of cfg4 256^3 system 0
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py tests/test_gpu_r2.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_p20.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_p20.log
for lib in "" paper_1604_01713_b200/_lib/variants/upd8.so; do
for a in "--p 20 --a1 0 --gc 108" "--p 20 --a1 0 --gc 20" "--p 20 --a1 108 --gc 0 --store --noin" "--p 20 --a1 20 --a2 80 --gc 0 --store --noin" "--p 20 --a1 88 --gc 0 --store --noin" "--p 20 --a1 80 --gc 0 --store --noin"; do
  RG_LIB_PATH=$lib timeout 300 python tools/prof_tall.py $a --reps 10
done
done > gpurun_out/p20_passes.txt 2>&1
timeout 900 python tools/prof_cycle.py --grid 256 --systems 1 --kernels > gpurun_out/cycle_256.json 2> gpurun_out/cycle_256.err

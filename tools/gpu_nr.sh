# narrow-ring passes (tall_nr_kernel): parity tests, isolated timings at n = 2^24 against
# variant libraries, the step.  Build the variants first (they are not kept in the tree):
#   python tools/ab_build.py nonr="-DRG_TALL_NR=0" nr3="-DRG_NR_CTAS=3"
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_nr.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_nr.log
for lib in "" paper_1604_01713_b200/_lib/variants/nr3.so paper_1604_01713_b200/_lib/variants/nonr.so; do
echo "== lib=${lib:-default}"
for a in "--p 8 --a1 0 --gc 0 --self --trsm1" "--p 8 --a1 0 --gc 0 --store --trsm2" "--p 8 --a1 0 --gc 0 --self" "--p 4 --a1 0 --gc 0 --self --trsm1"; do
  RG_LIB_PATH=$lib timeout 300 python tools/prof_tall.py $a --reps 20
done
done 2>&1 | grep -E "^n=|^==" > gpurun_out/nr_passes.txt
cat gpurun_out/nr_passes.txt
timeout 600 python tools/prof_spmm_dia.py > gpurun_out/spmm_dia.txt 2>&1
cat gpurun_out/spmm_dia.txt
python bench.py --no-cpu --no-e2e --no-tts > gpurun_out/bench_nr.json 2> gpurun_out/bench_nr.err
RG_LIB_PATH=paper_1604_01713_b200/_lib/variants/nr3.so python bench.py --no-cpu --no-e2e --no-tts > gpurun_out/bench_nr3.json 2> gpurun_out/bench_nr3.err

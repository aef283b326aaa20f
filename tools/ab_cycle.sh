# A/B of the per-kernel cycle profile (cfg4 256^3 system 0): default library, then each variant named
# on the command line (paper_1604_01713_b200/_lib/variants/<name>.so); outputs gpurun_out/abc_<name>.json
set -x
timeout 600 python tools/prof_cycle.py --grid 256 --systems 1 --kernels > gpurun_out/abc_default.json 2>&1
for v in "$@"; do
RG_LIB_PATH=$PWD/paper_1604_01713_b200/_lib/variants/$v.so timeout 600 python tools/prof_cycle.py --grid 256 --systems 1 --kernels > gpurun_out/abc_$v.json 2>&1
done

# A/B of the step bench: default library and each variant named on the command line
# (paper_1604_01713_b200/_lib/variants/<name>.so), alternated, 2 rounds; outputs gpurun_out/ab_<name>_<i>.json
set -x
for i in 1 2; do
timeout 300 python bench.py --no-tts --no-cpu --no-e2e > gpurun_out/ab_default_$i.json 2>&1
for v in "$@"; do
RG_LIB_PATH=$PWD/paper_1604_01713_b200/_lib/variants/$v.so timeout 300 python bench.py --no-tts --no-cpu --no-e2e > gpurun_out/ab_${v}_$i.json 2>&1
done
done

# ws TMA threshold A/B on the 28-36 column scrub / residual passes (n = 2^24); build the variant first:
#   python tools/ab_build.py ws24="-DRG_WS_MIN_LOAD_TMA=24"
for lib in "" paper_1604_01713_b200/_lib/variants/ws24.so; do
echo "== lib=${lib:-default}"
for a in "--p 8 --a1 20 --gc 20 --alias" "--p 8 --a1 20 --gc 0 --store" "--p 8 --a1 8 --gc 0 --store" "--p 8 --a1 0 --gc 20" "--p 8 --a1 20 --gc 0 --self --store"; do
  RG_LIB_PATH=$lib timeout 300 python tools/prof_tall.py $a --reps 20
done
done 2>&1 | grep -E "^n=|^=="

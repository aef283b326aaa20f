for impl in 3 5 6; do
  if [ "$impl" = auto ]; then unset RG_TALL_IMPL; else export RG_TALL_IMPL=$impl; fi
  echo "== impl $impl"
  python tools/prof_tall.py --a1 20 --gc 80
  python tools/prof_tall.py --a1 20 --gc 80 --store
  python tools/prof_tall.py --a1 20 --a2 80 --gc 20 --store
  python tools/prof_tall.py --a1 80 --self --store --gc 0
  python tools/prof_tall.py --a1 0 --gc 20
  python tools/prof_tall.py --a1 0 --gc 0 --store
done
for impl in 3 6; do
  export RG_TALL_IMPL=$impl
  echo "== qr passes impl $impl"
  python tools/prof_tall.py --a1 0 --gc 0 --self --trsm1
  python tools/prof_tall.py --a1 0 --gc 0 --store --trsm2
done

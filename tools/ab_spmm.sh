for impl in p g; do
  echo "== spmm impl $impl"
  RG_SPMM_IMPL=$impl python tools/prof_spmm.py
done

# A/B of the rg_tall paths on the cfg4 bench step: each line is an env setting
# followed by the step time and the per-pass ms / GB/s.  CFGS overrides the list
# (semicolon-separated env settings).
CFGS=${CFGS:-"RG_TALL_WS=1 RG_WS_CW=8;RG_TALL_WS=1 RG_WS_CW=4;RG_TALL_WS=0"}
IFS=';' read -ra LIST <<< "$CFGS"
for cfg in "${LIST[@]}"; do
  env $cfg timeout 300 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['ms_per_step'],3), [(k['kernel'][7:40], round(k['ms']/20,3), round(k['GB/s'])) for k in d['kernels']][:4])"
done

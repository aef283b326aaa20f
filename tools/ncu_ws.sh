set -x
timeout 300 ncu --set full --clock-control none -k regex:tall_ws_kernel --launch-skip 12 -c 3 -f -o /tmp/ws python tools/prof_step.py --steps 3 > gpurun_out/ncu_ws.log 2>&1
ncu -i /tmp/ws.ncu-rep --page raw --csv > gpurun_out/ws_raw.csv 2>&1
ncu -i /tmp/ws.ncu-rep --page details --csv > gpurun_out/ws_details.csv 2>&1
RG_TALL_WS=0 timeout 300 ncu --set full --clock-control none -k regex:tall_v6_kernel --launch-skip 12 -c 3 -f -o /tmp/v6 python tools/prof_step.py --steps 3 > gpurun_out/ncu_v6.log 2>&1
ncu -i /tmp/v6.ncu-rep --page details --csv > gpurun_out/v6_details.csv 2>&1
ls -la gpurun_out

# P2 study: ncu of the P2 shape on the TMA (default) and cp.async builds; exports CSV pages on the box
set -x
python tools/prof_tall.py --p 8 --a1 100 --gc 100 --alias --reps 5 && \
ncu --set full --clock-control none --import-source on -k regex:tall_ws -s 2 -c 1 -o /tmp/p2_tma python tools/prof_tall.py --p 8 --a1 100 --gc 100 --alias --reps 1 > gpurun_out/ncu_p2a.log 2>&1
RG_LIB_PATH=$PWD/paper_1604_01713_b200/_lib/variants/ws_ldgsts.so ncu --set full --clock-control none --import-source on -k regex:tall_ws -s 2 -c 1 -o /tmp/p2_ldgsts python tools/prof_tall.py --p 8 --a1 100 --gc 100 --alias --reps 1 > gpurun_out/ncu_p2b.log 2>&1
for r in p2_tma p2_ldgsts; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv
  ncu -i /tmp/$r.ncu-rep --page source --csv > gpurun_out/${r}_src.csv
  ncu -i /tmp/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv
done
ls -la gpurun_out

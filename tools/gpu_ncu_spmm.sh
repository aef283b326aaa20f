# ncu --set full of one cfg4 p=8 SpMM with source-level stall attribution (CSV pages exported on the box)
set -x
python tools/prof_spmm_one.py 8 256 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -o /tmp/spmm python tools/prof_spmm_one.py 8 256 > gpurun_out/ncu_spmm.log 2>&1
ncu -i /tmp/spmm.ncu-rep --page raw --csv > gpurun_out/spmm_raw.csv
ncu -i /tmp/spmm.ncu-rep --page source --csv > gpurun_out/spmm_src.csv
ncu -i /tmp/spmm.ncu-rep --page details --csv > gpurun_out/spmm_details.csv

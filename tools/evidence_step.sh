# One GPU call that refreshes the cfg4 step evidence under gpurun_out/:
# the default bench line, its ncu launch list, a full ncu capture of one step
# paired with the launch labels (DRAM traffic per launch), and smoke().
set -x
python bench.py > gpurun_out/bench_step.json 2> gpurun_out/bench_step.err
# launch list of the timed region only (bench.py brackets it with cudaProfilerStart/Stop)
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-tts > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --profile-from-start off -f -o /tmp/step \
    python tools/prof_step.py --steps 1 --labels gpurun_out/labels.json > gpurun_out/ncu_full.log 2>&1
python tools/ncu_traffic.py /tmp/step.ncu-rep gpurun_out/labels.json gpurun_out/ncu_traffic.json
ncu -i /tmp/step.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active > gpurun_out/step_raw.csv
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
ncu -i /tmp/step.ncu-rep --page details --csv > gpurun_out/step_details.csv

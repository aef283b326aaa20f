# Round evidence in one GPU call: the -m gpu suite, then tools/evidence_step.sh
# (default bench line, ncu launch list, full ncu capture of one step with per-launch traffic, smoke)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
bash tools/evidence_step.sh

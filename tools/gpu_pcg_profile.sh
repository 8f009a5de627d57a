# ncu launch list of one cfg4 PCG solve (per-iteration graphs), summarised
export PATH=/usr/local/cuda/bin:$PATH
CUTBDDC_NO_WHILE_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_pcg.csv python tools/pcg_profile.py ${1:-cfg4} > gpurun_out/ncu_pcg.log 2>&1
echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_pcg.csv | head -40

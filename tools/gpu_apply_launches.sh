# ncu launch list of BDDC applies outside the PCG graph (tools/apply_profile.py):
# per-kernel durations of one apply (cold-cache, serialised)
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_apply.csv python tools/apply_profile.py ${1:-cfg4} > gpurun_out/ncu_apply.log 2>&1
echo "ncu rc=$?"
python tools/launch_order.py gpurun_out/launches_apply.csv 2>/dev/null | tail -80

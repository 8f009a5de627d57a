# Refresh the profiles of the current path: per-phase timing (cfg4), the ncu
# launch list of one bench step, and ncu --set full of the solve sweeps of one
# BDDC apply (dram bytes -> roofline.traffic).
set -x
export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python tools/profile_phases.py cfg4 > gpurun_out/phases_cfg4.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 7 -c 7 \
  -o gpurun_out/sweeps_full -f python tools/apply_profile.py cfg4 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"

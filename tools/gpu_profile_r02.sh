# Profiles at HEAD (round 2): per-phase timing, warm per-piece timing, the ncu
# launch list of one bench step, ncu --set full of one apply's 6 sweep
# launches (-> roofline.traffic) and of the numeric factorisation.
set -x
export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python tools/profile_phases.py cfg4 > gpurun_out/phases_cfg4.txt 2>&1
timeout 300 python tools/time_parts.py cfg4 cfg5 > gpurun_out/time_parts.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cfg5 --no-batch > gpurun_out/ncu_bench.log 2>&1; echo "ncu1 rc=$?"
python tools/launch_summary.py gpurun_out/launches_bench.csv > gpurun_out/launches_bench_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function \
  -k 'regex:^k_sweep_(fwd|bwd)(_few)?$' --launch-skip 6 -c 6 \
  -o gpurun_out/sweeps_full -f python tools/apply_profile.py cfg4 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
python tools/ncu_traffic.py gpurun_out/sweeps_full.ncu-rep gpurun_out/sweep_traffic_cfg4.json cfg4-64 6
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_dag -c 1 \
  -o gpurun_out/dense_dag_full -f python tools/apply_profile.py cfg4 > gpurun_out/ncu_dag.log 2>&1; echo "ncu3 rc=$?"
ls -la gpurun_out/

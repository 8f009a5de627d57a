set -x
export PATH=/usr/local/cuda/bin:$PATH
bash tools/gpu_round.sh
timeout 900 python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "cfg5 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 7 -c 7 \
  -o gpurun_out/sweeps_full -f python tools/apply_profile.py cfg4 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"

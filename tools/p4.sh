export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_dag --launch-skip 2 -c 1 \
  -o gpurun_out/dag_full -f python tools/run_config.py cfg4 > gpurun_out/ncu_dag.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_dag.log

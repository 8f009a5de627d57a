./tools/bench_src/potrf_bench | tail -1
timeout 600 python -m pytest tests/test_gpu_dense_cholesky.py -x -q > gpurun_out/dchol.log 2>&1; echo "dchol rc=$?"; tail -2 gpurun_out/dchol.log
timeout 300 python tools/run_config.py cfg4 2>&1 | tail -3
timeout 300 python tools/run_config.py cfg5 2>&1 | tail -3
mkdir -p gpurun_out/dagtr
CUTBDDC_DAG_TRACE=gpurun_out/dagtr/cfg4 CUTBDDC_NO_PLAN_CACHE=1 timeout 300 python tools/run_config.py cfg4 > gpurun_out/dagtr/cfg4.log 2>&1
python tools/dag_analyze.py gpurun_out/dagtr/cfg4 2>&1 | grep -B1 -A9 "_0.bin\|_1.bin" | grep -v "^ *[01] " > gpurun_out/dag_cfg4.txt
rm -rf gpurun_out/dagtr/*.bin
cat gpurun_out/dag_cfg4.txt

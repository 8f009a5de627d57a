CUTBDDC_DAG_TRACE=gpurun_out/dag timeout 300 python tools/run_config.py cfg4 > gpurun_out/dag_run.txt 2>&1
python tools/dag_analyze.py gpurun_out/dag > gpurun_out/dag_summary.txt 2>&1
rm -f gpurun_out/dag_*.bin

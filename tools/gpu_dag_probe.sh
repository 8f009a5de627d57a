# Phase profile of cfg5 and DAG task traces (cfg4, cfg5) for dag_analyze.py
PROFILE_REPS=2 timeout 600 python tools/profile_phases.py cfg5 > gpurun_out/phases_cfg5.txt 2>&1; echo "p5 rc=$?"
mkdir -p gpurun_out/dagtr
CUTBDDC_DAG_TRACE=gpurun_out/dagtr/cfg4 CUTBDDC_NO_PLAN_CACHE=1 timeout 300 python tools/run_config.py cfg4 > gpurun_out/dagtr/cfg4.log 2>&1; echo "t4 rc=$?"
python tools/dag_analyze.py gpurun_out/dagtr/cfg4 > gpurun_out/dag_cfg4.txt 2>&1
CUTBDDC_DAG_TRACE=gpurun_out/dagtr/cfg5 timeout 600 python tools/run_config.py cfg5 > gpurun_out/dagtr/cfg5.log 2>&1; echo "t5 rc=$?"
python tools/dag_analyze.py gpurun_out/dagtr/cfg5 > gpurun_out/dag_cfg5.txt 2>&1
rm -rf gpurun_out/dagtr/*.bin

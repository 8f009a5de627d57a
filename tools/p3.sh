timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases_ms'], d['e2e']['value'], d['roofline']['launch_ms'])"; done
CUTBDDC_SWEEP_TRACE=gpurun_out/tr timeout 300 python tools/apply_profile.py cfg4 > gpurun_out/trace_run.txt 2>&1
python tools/trace_analyze.py gpurun_out/tr > gpurun_out/trace_summary.txt 2>&1; rm -f gpurun_out/tr_*.bin
timeout 600 python tools/apply_profile.py cfg5 > gpurun_out/cfg5_roofline.txt 2>&1

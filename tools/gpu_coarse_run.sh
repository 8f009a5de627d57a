timeout 600 python -m pytest tests/test_gpu_coarse_sparse.py -x -q > gpurun_out/csparse.log 2>&1; echo "csparse rc=$?"; tail -15 gpurun_out/csparse.log
CUTBDDC_COARSE_STATS=1 timeout 300 python tools/run_config.py cfg5 2>&1 | tail -4
CUTBDDC_COARSE=dense timeout 300 python tools/run_config.py cfg5 2>&1 | tail -3 | head -2
timeout 900 python -m pytest tests/test_gpu_parity_b16.py -x -q -k "cfg5 or golden" > gpurun_out/b16.log 2>&1; echo "b16 rc=$?"; tail -3 gpurun_out/b16.log

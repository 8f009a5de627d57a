timeout 300 python tools/setup_jitter.py cfg4 > gpurun_out/jitter.txt 2>&1
CUTBDDC_PROFILE=1 REPS=4 timeout 300 python tools/setup_jitter.py cfg4 > gpurun_out/jitter_prof.txt 2>&1

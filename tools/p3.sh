SAMPLER=1 REPS=40 timeout 300 python tools/setup_jitter.py cfg4 2>&1 | tail -1
REPS=40 timeout 300 python tools/setup_jitter.py cfg4 2>&1 | tail -1

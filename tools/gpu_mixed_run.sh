timeout 600 python -m pytest tests/test_gpu_mixed_k.py -x -q > gpurun_out/mixed.log 2>&1; echo "mixed rc=$?"
tail -15 gpurun_out/mixed.log
bash tools/gpu_tests.sh

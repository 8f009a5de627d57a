# full GPU tests, then the short bench and the cfg5 leg
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-batch --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
python - <<P
import json
b = json.load(open("gpurun_out/bench_q.json"))
print("cold", round(b["value"]), b["phases_ms"], "warm", round(b["warm"]["value"]), "e2e", round(b["e2e"]["value"]), b["e2e"]["samples_ms"])
c = b.get("cfg5")
print("cfg5", c and (round(c["value"]), c["phases_ms"], c["roofline"]["frac"]))
P

# Run-to-run spread of the bench line on one box: the short bench N times.
for i in 1 2 3 4; do
  timeout 300 python bench.py --no-cfg5 --no-batch --no-cpu-baseline > gpurun_out/bench_rep_$i.json 2> gpurun_out/bench_rep_$i.err
  python - <<P
import json
b = json.load(open("gpurun_out/bench_rep_$i.json"))
print("run $i cold", round(b["value"]), b["phases_ms"], "warm", round(b["warm"]["value"]), b["warm"]["phases_ms"], "e2e", round(b["e2e"]["value"]), b["clocks"])
P
done

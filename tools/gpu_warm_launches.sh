# warm-cache ncu launch list (--cache-control none) of `python $@`; last 60 launches printed
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/launches_warm.csv python "$@" > gpurun_out/ncu_warm.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/launches_warm.csv")))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
data = [d for d in data if d["Metric Name"] == "gpu__time_duration.sum"]
for d in data[-60:]:
    v = float(d["Metric Value"].replace(",", "")) * {"usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
    print(f'{v:9.2f} us  {d["Kernel Name"].split("(")[0][:70]}  grid {d.get("Grid Size", "")}')
PY

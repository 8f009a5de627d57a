"""DRAM traffic of the solve sweeps of one BDDC apply from an ncu --set full
capture (tools/gpu_profile.sh: k_sweep launches of apply_profile.py), written
to a profile JSON that bench.py reads for roofline.traffic.

usage: python tools/ncu_traffic.py <sweeps_full.ncu-rep> <out.json> <workload> [launches per apply]"""
import csv
import io
import json
import subprocess
import sys

rep, out, workload = sys.argv[1], sys.argv[2], sys.argv[3]
per_apply = int(sys.argv[4]) if len(sys.argv) > 4 else 6
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
col = {k: hdr.index(k) for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum")}
launches = []
for r in rows[2:]:
    rd = float(r[col["dram__bytes_read.sum"]]) * scale[units[col["dram__bytes_read.sum"]]]
    wr = float(r[col["dram__bytes_write.sum"]]) * scale[units[col["dram__bytes_write.sum"]]]
    launches.append({"kernel": r[col["Kernel Name"]].split("(")[0].split("::")[-1],
                     "us": float(r[col["gpu__time_duration.sum"]]), "dram_read": rd, "dram_write": wr})
# one apply = I fwd, I bwd, K fwd, K bwd, I fwd, I bwd: 6 consecutive launches
# (7 with the shell-root K: its backward sweep is split at the root)
apply_launches = launches[:per_apply]
tot = sum(l["dram_read"] + l["dram_write"] for l in apply_launches)
json.dump({"workload": workload, "source": rep, "traffic_bytes_per_apply": tot, "launches": apply_launches,
           "note": "ncu --set full --clock-control none, serialised and cold-cache: shares, not absolute times"},
          open(out, "w"), indent=1)
print(f"traffic per apply {tot / 1e6:.1f} MB over {len(apply_launches)} launches")

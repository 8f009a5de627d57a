# Per-kernel durations of one warm assembly (ncu, serialised): which kernels make up the assembly phase.
cat > /tmp/asm_once.py <<'P'
import sys; sys.path.insert(0, '.')
from paper_1703_06323_b200 import configs, cutbddc as cb
cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else 'cfg4'); s = cb.GpuSolver(0); pb = cb.prepare(s, cfg)
s.assemble(cfg.block, pb.block_ids)
s.assemble(cfg.block, pb.block_ids)
s.close()
P
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/asm_launches.csv python /tmp/asm_once.py ${1:-cfg4} > /dev/null 2>&1
python - <<'P'
import csv
rows = [r for r in csv.reader(open('gpurun_out/asm_launches.csv')) if len(r) > 10 and r[0].isdigit()]
n = len(rows) // 3 if False else 0
# print the last third (third assemble call incl. prepare's): just print all kernels with time > 5 us
tot = 0
for r in rows:
    name, val = r[4], float(r[-1].replace(',', ''))
    unit = r[-2]
    us = val / 1e3 if unit in ('ns', 'nsecond') else val
    if us >= 5: print('%9.1f us  %s' % (us, name[:90]))
P

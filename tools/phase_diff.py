"""Steady-state per-call device time of each CUTBDDC_PROFILE scope: the
difference of two profile_phases.py runs (PROFILE_REPS=1 and =5)."""
import re
import sys


def parse(f):
    d = {}
    for line in open(f):
        m = re.match(r'\[cutbddc profile\] (.+?)\s+(\d+)\s+([\d.]+)\s+([\d.]+)$', line.strip())
        if m:
            d[m.group(1).strip()] = (int(m.group(2)), float(m.group(3)))
    return d


a, b = parse(sys.argv[1]), parse(sys.argv[2])
for k in b:
    c1, t1 = a.get(k, (0, 0.0))
    c5, t5 = b[k]
    if c5 > c1:
        print(f"{k:45s} {1000 * (t5 - t1) / (c5 - c1):9.1f} us/call  ({c5 - c1} calls)")

"""Print an ncu --metrics gpu__time_duration.sum CSV launch list in launch
order (kernel, grid, block, us), optionally only launches [first, last)."""
import csv
import sys


def ordered(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"msecond": 1e3, "usecond": 1.0, "nsecond": 1e-3, "second": 1e6}.get(d.get("Metric Unit", ""), 1.0)
        out.append((d["Kernel Name"].split("(")[0].split("::")[-1], d.get("Grid Size", ""), d.get("Block Size", ""), v))
    return out


if __name__ == "__main__":
    launches = ordered(sys.argv[1])
    lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    hi = int(sys.argv[3]) if len(sys.argv) > 3 else len(launches)
    for i, (k, g, b, us) in enumerate(launches[lo:hi], lo):
        print(f"{i:5d} {us:10.1f} us  {k:28s} grid {g:18s} block {b}")

"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys


def summarise(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].split("::")[-1]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        v *= {"msecond": 1e6, "usecond": 1e3, "nsecond": 1.0, "second": 1e9}.get(unit, 1.0)
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    lines = [f"{'ms':>10} {'share':>6} {'launches':>8}  kernel"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
        lines.append(f"{v / 1e6:10.3f} {100 * v / s:5.1f}% {cnt[k]:8d}  {k}")
    lines.append(f"total {s / 1e6:.3f} ms over {sum(cnt.values())} launches")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))

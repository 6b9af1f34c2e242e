"""Per-kernel share of device time from an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: launch_summary.py launches.csv "command line" > profiles/rNN_..._launch_summary.txt"""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.Counter(); cnt = collections.Counter()
for r in rows[1:]:
    if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    v *= {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1}.get(r[iu], 1)
    name = r[ik].split("(")[0]
    tot[name] += v; cnt[name] += 1
s = sum(tot.values())
print(f"# ncu --metrics gpu__time_duration.sum --clock-control none: {sys.argv[2] if len(sys.argv) > 2 else ''}")
print("# (cold-cache, serialised launches: compare SHARES, not absolute times)")
print(f"{'kernel':60s} {'launches':>8s} {'total_ns':>14s} {'share':>7s}")
for k, v in tot.most_common():
    print(f"{k[:60]:60s} {cnt[k]:8d} {int(v):14d} {100*v/s:6.2f}%")

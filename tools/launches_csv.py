"""Per-launch table of an ncu --metrics gpu__time_duration.sum[,dram__bytes_*] CSV:
python tools/launches_csv.py FILE [substring ...]"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
pats = sys.argv[2:]
d = OrderedDict()
for r in rows:
    d.setdefault(r[0], {"name": r[4][:70]})[r[12]] = float(r[14].replace(",", ""))
tot = 0.0
for k, v in d.items():
    if pats and not any(p in v["name"] for p in pats):
        continue
    t = v.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    print(f"{k:>4} {t:9.1f} us  rd {v.get('dram__bytes_read.sum', 0) / 1e9:5.2f} GB  "
          f"wr {v.get('dram__bytes_write.sum', 0) / 1e9:5.2f} GB  {v['name']}")
print(f"total {tot:.1f} us")

"""Executed warp-instructions per row grouped by source file (and optionally line ranges), from an
ncu source page exported with --print-source cuda,sass.  usage: ncu_byfile.py file.csv ROWS"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1], encoding="utf-8", errors="replace")))
nrows = float(sys.argv[2])
f = None; tot = collections.Counter(); st = collections.Counter()
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if len(r) < 9 or r[0] in ("Line No", "", "Function Name"):
        continue
    try:
        ins = float(r[7]); s = float(r[4]); ln = int(r[0])
    except ValueError:
        continue
    tot[f] += ins; st[f] += s
    if len(sys.argv) > 3:
        for spec in sys.argv[3:]:
            name, rng = spec.split("=")
            fn, a, b = rng.split(":")
            if fn == f and int(a) <= ln <= int(b):
                tot["  [" + name + "]"] += ins; st["  [" + name + "]"] += s
T = sum(v for k, v in tot.items() if not k.startswith("  ")); S = sum(v for k, v in st.items() if not k.startswith("  ")) or 1
for k, v in sorted(tot.items(), key=lambda kv: kv[0].startswith("  ")):
    print(f"{k:28s} {v/nrows:6.2f} warp-instr/row  {st[k]/S*100:5.1f}% stall samples")
print(f"{'total':28s} {T/nrows:6.2f}")

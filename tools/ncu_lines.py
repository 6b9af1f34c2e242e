"""Aggregate an ncu source page (cuda,sass) by CUDA source line: instructions and stalls.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > f.csv; python tools/ncu_lines.py f.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
out = []
cur_file = None
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) < 9 or r[0] == "Line No":
        continue
    try:
        ins = float(r[7] or 0); st = float(r[4] or 0)
    except ValueError:
        continue
    out.append((cur_file, r[0], r[1], ins, st))
tot_i = sum(o[3] for o in out) or 1; tot_s = sum(o[4] for o in out) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for f, ln, src, i, s in sorted(out, key=lambda o: -o[3])[:n]:
    print(f"{i/tot_i*100:5.1f}% inst {s/tot_s*100:5.1f}% stall {f}:{ln:>4} {src.strip()[:100]}")
print("--- by stall")
for f, ln, src, i, s in sorted(out, key=lambda o: -o[4])[:20]:
    print(f"{i/tot_i*100:5.1f}% inst {s/tot_s*100:5.1f}% stall {f}:{ln:>4} {src.strip()[:100]}")

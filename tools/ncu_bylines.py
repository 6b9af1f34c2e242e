"""Executed warp-instructions and stall samples per CUDA source line, from an ncu source page
exported with --print-source cuda,sass.  usage: ncu_bylines.py file.csv ROWS [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1], encoding="utf-8", errors="replace")))
nrows = float(sys.argv[2]); top = int(sys.argv[3]) if len(sys.argv) > 3 else 45
f = None; out = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if len(r) < 9 or r[0] in ("Line No", "", "Function Name"):
        continue
    try:
        ins = float(r[7]); st = float(r[4])
    except ValueError:
        continue
    out.append((f, int(r[0]), r[1], ins, st))
ti = sum(o[3] for o in out); ts = sum(o[4] for o in out) or 1
print(f"total {ti/nrows:.2f} warp-instr/row")
for f, ln, src, i, s in sorted(out, key=lambda o: -o[3])[:top]:
    print(f"{i/nrows:6.2f}/row {s/ts*100:5.1f}%st {f}:{ln:<4} {src.strip()[:90]}")

"""Executed warp-instructions per row grouped by source range (phase) of the tile kernel.
usage: ncu_phases.py src.csv ROWS  (src.csv from --print-source cuda,sass)"""
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1], encoding="utf-8", errors="replace")))
n = float(sys.argv[2])
src = open("paper_2603_15023_b200/csrc/agg_tiles.cuh").read().splitlines()
def find(pat):
    for i, l in enumerate(src, 1):
        if re.search(pat, l):
            return i
    return 10**9  # region marker absent in this source version
marks = [("dict/local_code", find(r"^static __device__ int local_code")),
         ("row_group_key", find(r"uint64_t row_group_key")),
         ("tma helpers", find(r"^// ------------------------------------------------------------------ TMA bulk")),
         ("xpose/shfl helpers", find(r"^// ------------------------------------------------------------------ k_agg_tiles")),
         ("WarpAcc/flush", find(r"^struct WarpAcc")),
         ("run_body", find(r"void run_body\(")),
         ("run_tiles", find(r"void run_tiles\(")),
         ("TileSmem/TileCols", find(r"^struct TileSmem")),
         ("A1", find(r"void tile_a1\(")),
         ("B2", find(r"---------------- B2")),
         ("B3", find(r"---------------- B3")),
         ("A2", find(r"---------------- A2")),
         ("A3", find(r"---------------- A3")),
         ("kernel body", find(r"k_agg_tiles\(AggPlan p")),
         ("CTA->HBM", find(r"---------------- CTA table -> provisional"))]
def phase(f, ln):
    if f != "agg_tiles.cuh":
        return f
    name = "head"
    for nm, start in marks:
        if ln >= start:
            name = nm
    return name
agg = {}
f = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if len(r) < 9 or r[0] in ("Line No", "", "Function Name"):
        continue
    try:
        ins = float(r[7])
    except ValueError:
        continue
    k = phase(f, int(r[0]))
    agg[k] = agg.get(k, 0) + ins
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    if v / n > 0.05:
        print(f"{v/n:6.2f} warp-instr/row  {100*v/tot:5.1f}%  {k}")
print(f"{tot/n:6.2f} total")

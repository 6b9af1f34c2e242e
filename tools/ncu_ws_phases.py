"""Executed warp-instructions per input row of k_agg_ws by role / phase, from an ncu source page
exported with --print-source cuda,sass.  usage: ncu_ws_phases.py src.csv ROWS"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1], encoding="utf-8", errors="replace")))
n = float(sys.argv[2])
ws = open("paper_2603_15023_b200/csrc/agg_ws.cuh").read().splitlines()
tiles = open("paper_2603_15023_b200/csrc/agg_tiles.cuh").read().splitlines()


def spans(src, marks):
    idx = []
    for name, pat in marks:
        for i, l in enumerate(src, 1):
            if re.search(pat, l):
                idx.append((i, name))
                break
    idx.sort()
    return idx


WS = spans(ws, [("flags", r"int ws_row_flags\("), ("try_write", r"bool ws_try_write\("),
                ("append", r"void ws_append\("), ("consume", r"void ws_consume\("),
                ("ownership", r"uint32_t ws_tmine\("), ("service", r"^__device__ void ws_service\(const"),
                ("tier", r"void ws_tier\("), ("drain", r"void ws_drain\("), ("hash_chunk loads", r"void ws_hash_chunk\("),
                ("hash_chunk slots", r"int s\[2\];"), ("hash_chunk hash", r"uint64_t m\[2\] = "),
                ("hash_chunk append/queue", r"for \(int h = 0; h < 2; \+\+h\) \{\n?.*MM\) v\[h\]"),
                ("kernel", r"k_agg_ws\(AggPlan p"), ("kernel loop", r"int qh = 0, qn = 0, pn = 0;"),
                ("kernel end", r"keep servicing until"), ("host", r"host side")])
TL = spans(tiles, [("dictionary", r"^static __device__ int local_code"), ("other", r"uint64_t row_group_key"),
                   ("transpose", r"void transpose2x32"), ("other", r"double shfl_d"),
                   ("run_body", r"void run_body\("), ("other", r"void run_tiles\(")])


def cat(f, ln):
    if f == "agg_ws.cuh":
        name = "ws:head"
        for i, nm in WS:
            if ln >= i:
                name = "ws:" + nm
        return name
    if f == "agg_tiles.cuh":
        name = "tiles:head"
        for i, nm in TL:
            if ln >= i:
                name = "tiles:" + nm
        return name
    if f == "common.cuh":
        return "hash (common.cuh)"
    if f == "agg_tm.cuh":
        return "tmem (agg_tm.cuh)"
    return f


tot = {}
st = {}
f = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) < 9 or r[0] in ("Line No", "", "Function Name"):
        continue
    try:
        ins = float(r[7]); s = float(r[4]); ln = int(r[0])
    except ValueError:
        continue
    c = cat(f, ln)
    tot[c] = tot.get(c, 0) + ins
    st[c] = st.get(c, 0) + s
T = sum(tot.values()); S = sum(st.values()) or 1
print(f"total {T / n:.2f} warp-instr/row")
for c, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"  {v / n:6.2f} warp-instr/row {100 * st[c] / S:5.1f}% stall  {c}")

"""Executed-instruction mix by SASS opcode from an ncu source page (sass)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Instructions Executed" in r)
i_src = hdr.index("Source"); i_ex = hdr.index("Instructions Executed"); i_st = hdr.index("Warp Stall Sampling (All Samples)")
start = rows.index(hdr) + 1
mix = collections.Counter(); st = collections.Counter(); tot = 0
for r in rows[start:]:
    if len(r) <= i_ex: continue
    op = r[i_src].strip().split()
    if not op: continue
    o = op[0]
    if o.startswith("@"): o = op[1] if len(op) > 1 else o
    o = o.split(".")[0]
    try: n = float(r[i_ex] or 0); s = float(r[i_st] or 0)
    except ValueError: continue
    mix[o] += n; st[o] += s; tot += n
ts = sum(st.values()) or 1
for o, n in mix.most_common(40):
    print(f"{o:12s} {n/tot*100:5.1f}% of inst   {st[o]/ts*100:5.1f}% of stall samples")
print("total executed warp-instructions:", int(tot))

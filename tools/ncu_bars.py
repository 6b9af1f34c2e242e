"""Executed instructions per SASS segment between BAR instructions (phase attribution)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Instructions Executed" in r)
i_src = hdr.index("Source"); i_ex = hdr.index("Instructions Executed"); i_ad = hdr.index("Address")
i_st = hdr.index("Warp Stall Sampling (All Samples)")
start = rows.index(hdr) + 1
seg, segs, sst = 0.0, [], 0.0
first = None
tot = sum(float(r[i_ex] or 0) for r in rows[start:] if len(r) > i_ex and r[i_ex].replace('.','').isdigit())
tots = sum(float(r[i_st] or 0) for r in rows[start:] if len(r) > i_st and r[i_st].replace('.','').isdigit())
for r in rows[start:]:
    if len(r) <= i_ex: continue
    try: n = float(r[i_ex] or 0); s = float(r[i_st] or 0)
    except ValueError: continue
    if first is None: first = r[i_ad]
    seg += n; sst += s
    if "BAR" in r[i_src].split()[0:2][-1] or r[i_src].strip().startswith("BAR"):
        segs.append((first, r[i_ad], seg, sst)); seg, sst, first = 0.0, 0.0, None
segs.append((first, "end", seg, sst))
for a, b, n, s in segs:
    print(f"{a} .. {b}: {n/tot*100:5.1f}% inst  {s/tots*100:5.1f}% stalls")

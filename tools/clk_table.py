"""Per-phase table from LEANCLK lines (k_agg_lean built with -DPAC_LEAN_CLK=1): python tools/clk_table.py < log"""
import sys
import numpy as np
rows = [l.split() for l in sys.stdin if l.startswith("LEANCLK")]
for g0 in range(0, len(rows), 16):
    grp = rows[g0:g0 + 16]
    names = grp[0][2::2]
    v = np.array([[int(x) for x in r[3::2]] for r in grp], float)
    tiles = v[0, -1]
    v = v[:, :-1]
    print("tiles %d  cycles/tile %.0f" % (tiles, v.sum(1).mean() / tiles))
    for i, n in enumerate(names[:-1]):
        print("  %-7s mean %6.0f  min %6.0f  max %6.0f  (%4.1f%%)  w0-3 %6.0f  w4-15 %6.0f" % (
            n, v[:, i].mean() / tiles, v[:, i].min() / tiles, v[:, i].max() / tiles,
            100 * v[:, i].mean() / v.sum(1).mean(), v[:4, i].mean() / tiles, v[4:, i].mean() / tiles))

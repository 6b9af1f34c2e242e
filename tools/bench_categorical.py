"""Throughput of the row-parallel categorical kernels (§8 f1) at BASELINE scale: one JSON line.

pac_select_cmp / pac_filter_cmp over n rows (default 6e7, C2's row count) against G group world
vectors (default 200,000 -- TPC-H SF1's part count, the Q17 shape): rows/s and the HBM
roofline of the algorithmic bytes (h 8 + v 8 + gidx 4 + out 8 = 28 B/row for select, 21 B/row
for filter), CUDA events on the launching stream, inputs > L2.
  python tools/bench_categorical.py [--rows N] [--groups G] [--iters K]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2603_15023_b200 as pac  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=60_000_000)
    ap.add_argument("--groups", type=int, default=200_000)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(5)
    n, G = a.rows, a.groups
    c = torch.randint(0, 51, (G, 64), device="cuda", generator=g).to(torch.float64) * 0.2
    pres = torch.full((G,), -1, dtype=torch.int64, device="cuda")
    v = torch.randint(1, 51, (n,), device="cuda", generator=g).to(torch.float64)
    gidx = torch.randint(0, G, (n,), device="cuda", generator=g, dtype=torch.int32)
    h = torch.randint(-(2**63), 2**63 - 1, (n,), device="cuda", generator=g, dtype=torch.int64)
    out = torch.empty_like(h)
    s = pac.Session(1)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    ix = pac.cmp_index(c, pres)
    for name, fn, bpr in (("select_cmp", lambda: pac.select_cmp(pac.CMP_LT, h, v, gidx, ix, out), 28),
                          ("filter_cmp", lambda: pac.filter_cmp(s, pac.CMP_LT, v, gidx, ix), 21),
                          ("cmp_index", lambda: pac.cmp_index(c, pres), None)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        r = {"ms": ms}
        if bpr:
            gbs = n * bpr / (ms / 1e3) / 1e9
            r.update({"rows_per_s": n / (ms / 1e3), "achieved_gbs": gbs, "frac": gbs / peak,
                      "bytes_per_row": bpr})
        else:
            r["groups_per_s"] = G / (ms / 1e3)
        res[name] = r
    print(json.dumps({"rows": n, "groups": G, "peak_gbs": peak, "results": res}))


if __name__ == "__main__":
    main()

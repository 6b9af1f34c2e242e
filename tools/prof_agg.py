"""Runs the hot path of one workload a few times (for ncu / compute-sanitizer captures).

  python tools/prof_agg.py [--config C2] [--rows N] [--iters 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen as dg  # noqa: E402
import paper_2603_15023_b200 as pac  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--rows", type=int, default=0)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--gcap", type=int, default=0)
    a = ap.parse_args()
    w = dg.WORKLOADS[a.config]
    if a.rows:
        w = w.scaled(a.rows)
    cols = dg.device_columns(w, 0, w.n_rows)
    kinds = [k for k, _ in w.aggs]
    vals = [None if i < 0 else cols["values"][i] for _, i in w.aggs]
    G_cap = a.gcap or {"C1": 1, "C2": 8, "C4": 1024, "C5": 100}.get(w.name, 1 << 21)
    s = pac.Session(7, w.budget)
    ag = pac.Aggregator(kinds, G_cap)
    fin = pac.Finalizer(kinds, G_cap)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for i in range(a.iters):
        ev[0].record()
        t = ag(vals, cols["keys"], pu_key=cols["pu"], salt=s.salt)
        fin(s, t, 0)
        ev[1].record()
        torch.cuda.synchronize()
        print(f"iter {i}: {ev[0].elapsed_time(ev[1]):.3f} ms, G={t.check()}", flush=True)


if __name__ == "__main__":
    main()

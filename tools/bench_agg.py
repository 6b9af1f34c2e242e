"""Aggregation-only timing of one BASELINE config on the device-generated columns (CUDA events
around pac_agg_grouped, median of --iters after warm-up).  Env switches (PAC_NO_WS, PAC_NO_TM,
...) select kernels for A/B runs.  Prints one JSON line."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen as dg  # noqa: E402
import paper_2603_15023_b200 as pac  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
w = dg.WORKLOADS[a.config]
n = a.rows or w.n_rows
cols = dg.device_columns(w, 0, n)
kinds = [k for k, _ in w.aggs]
vals = [None if i < 0 else cols["values"][i] for _, i in w.aggs]
G_cap = {"C1": 1, "C2": 8, "C4": 1024, "C5": 100}.get(w.name, 1 << 21)
ag = pac.Aggregator(kinds, G_cap)
for _ in range(3):
    ag(vals, cols["keys"], pu_key=cols["pu"], salt=0x1234)
torch.cuda.synchronize()
ts = []
for _ in range(a.iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ag(vals, cols["keys"], pu_key=cols["pu"], salt=0x1234)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
G = ag.table.check()
print(json.dumps({"config": w.name, "rows": n, "ms": ms, "best_ms": min(ts), "rows_per_s": n / ms * 1e3,
                  "GBps": n * w.in_bytes_per_row / ms / 1e6, "groups": G,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("PAC_")}}))

"""m = 128 worlds (§8 f4) vs m = 64 on a BASELINE config: device time of the aggregation and of the
finalize (CUDA events), rows/s, one JSON line.   python tools/bench_m128.py [--config C2]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen as dg  # noqa: E402
import paper_2603_15023_b200 as pac  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    w = dg.WORKLOADS[a.config]
    cols = dg.device_columns(w, 0, w.n_rows)
    kinds = [k for k, _ in w.aggs]
    vals = [None if i < 0 else cols["values"][i] for _, i in w.aggs]
    G_cap = {"C1": 1, "C2": 8, "C4": 1024, "C5": 100}.get(w.name, 1 << 21)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.iters

    out = {"config": w.name, "rows": w.n_rows}
    for m in (64, 128):
        s = pac.Session(11, w.budget, m=m)
        ag = pac.Aggregator(kinds, G_cap) if m == 64 else pac.Aggregator128(kinds, G_cap)
        fin = pac.Finalizer(kinds, G_cap)
        t = ag(vals, cols["keys"], pu_key=cols["pu"], salt=s.salt)
        agg_ms = timed(lambda: ag(vals, cols["keys"], pu_key=cols["pu"], salt=s.salt))
        fin_ms = timed(lambda: fin(s, t, 0))
        out[f"m{m}"] = {"agg_ms": agg_ms, "finalize_ms": fin_ms, "rows_per_s": w.n_rows / ((agg_ms + fin_ms) / 1e3)}
    out["agg_cost_ratio_128_over_64"] = out["m128"]["agg_ms"] / out["m64"]["agg_ms"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()

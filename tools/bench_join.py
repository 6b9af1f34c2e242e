"""PU-key join throughput (§8 f2) at TPC-H SF10 shape: orders 1.5e7 (o_orderkey -> o_custkey over
1.5e6 customers), lineitem 6e7 rows probing l_orderkey, fused pac_hash of o_custkey.  One JSON
line: build and probe times, rows/s, and the HBM roofline of the streamed bytes (fk 8 + mask 8 =
16 B/row) plus the random table traffic (one 32-B sector per probe step; table 2x oversized).
  python tools/bench_join.py [--rows N] [--orders M] [--iters K]"""
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
    ap.add_argument("--orders", type=int, default=15_000_000)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(7)
    orderkey = torch.randperm(4 * a.orders, device="cuda", generator=g)[:a.orders].to(torch.int64) * 4 + 1
    o_custkey = torch.randint(0, 1_500_000, (a.orders,), device="cuda", generator=g, dtype=torch.int64)
    fk = orderkey[torch.randint(0, a.orders, (a.rows,), device="cuda", generator=g)]
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = pac.JoinTable(orderkey, o_custkey)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.iters):
        t = pac.JoinTable(orderkey, o_custkey)
    e1.record()
    torch.cuda.synchronize()
    build_ms = e0.elapsed_time(e1) / a.iters
    assert t.status() == 0
    for _ in range(3):
        pac.join_mask([t], fk, 123)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.iters):
        m = pac.join_mask([t], fk, 123)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    stream_gbs = a.rows * 16 / (ms / 1e3) / 1e9
    print(json.dumps({"rows": a.rows, "orders": a.orders, "build_ms": build_ms, "probe_hash_ms": ms,
                      "rows_per_s": a.rows / (ms / 1e3), "stream_gbs": stream_gbs, "frac": stream_gbs / peak,
                      "peak_gbs": peak, "table_bytes": t.nbytes}))


if __name__ == "__main__":
    main()

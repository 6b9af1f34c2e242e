"""§8 f3 measurements: (1) the paper's Fig. 4 setting -- an ungrouped noised SUM over 1G rows -- timed
for the approximate two-sided state (pac_approx_sum), the single-sided one and the exact int64 SUM
(pac_agg_grouped with no keys); (2) Table 1's accuracy columns on 1M values of ten
synthetic distributions: %Err of the secret world's value, z^2 = (error / noise std)^2 with the
noise std sqrt(Var_P(y)/(2B)) of a fresh session (B = 1/128), and the sigma^2 ratio Var(y_approx) /
Var(y_exact) over the 64 worlds.  Prints JSON lines."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen as dg  # noqa: E402
import paper_2603_15023_b200 as pac  # noqa: E402


def timed(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000_000
w = dg.WORKLOADS["C1"].scaled(n)
cols = dg.device_columns(w, 0, n)
v, pu = cols["values"][0], cols["pu"]
ag = pac.Aggregator([pac.SUM_I64], 1)
res = {"rows": n}
res["exact_sum_ms"] = timed(lambda: ag([v], [], pu_key=pu, salt=1))
res["approx_two_sided_ms"] = timed(lambda: pac.approx_sum(v, pu_key=pu, salt=1, two_sided=True))
res["approx_single_sided_ms"] = timed(lambda: pac.approx_sum(v, pu_key=pu, salt=1, two_sided=False))
print(json.dumps({"fig4_ungrouped_sum": res}), flush=True)
del cols, v, pu

rng = np.random.default_rng(2026)
m = 1_000_000
dists = {
    "all_same": lambda: np.full(m, 1234567),
    "bimodal": lambda: np.where(rng.random(m) < 0.5, rng.normal(1e4, 1e3, m), rng.normal(1e7, 1e6, m)).astype(np.int64),
    "exponential": lambda: rng.exponential(1e6, m).astype(np.int64) + 1,
    "negative_mixed": lambda: np.where(rng.random(m) < 0.5, rng.integers(1, 10**6, m), -rng.integers(1, 10**6, m)),
    "sparse_large": lambda: np.where(rng.random(m) < 0.01, rng.integers(10**12, 10**13, m), 0),
    "uniform_bigint": lambda: rng.integers(1, 2**40, m),
    "uniform_int": lambda: rng.integers(1, 2**31, m),
    "uniform_smallint": lambda: rng.integers(1, 2**15, m),
    "uniform_tinyint": lambda: rng.integers(1, 2**7, m),
    "zipf_like": lambda: np.minimum(rng.zipf(1.3, m), 10**9),
}
pu = torch.from_numpy(rng.integers(0, m // 10, m).astype(np.int64)).cuda()
rows = []
for name, gen in dists.items():
    vals = gen().astype(np.int64)
    vd = torch.from_numpy(vals).cuda()
    s = pac.Session(7, 1.0 / 128)
    t = pac.Aggregator([pac.SUM_I64], 1)([vd], [], pu_key=pu, salt=s.salt)
    y_exact = 2.0 * t.world[0][0].double().cpu().numpy()
    P = np.full(64, 1.0 / 64)
    delta = float(np.sum(P * (y_exact - np.sum(P * y_exact)) ** 2)) / (2.0 / 128)
    row = {"distribution": name}
    for side, ts in (("single", False), ("two_sided", True)):
        _, y = pac.approx_sum(vd, pu_key=pu, salt=s.salt, two_sided=ts)
        y = y.cpu().numpy()
        j = s.jstar
        err = y[j] - y_exact[j]
        row[side] = {"pct_err": 100.0 * abs(err) / max(abs(y_exact[j]), 1e-300),
                     "z2": err * err / delta if delta > 0 else None,
                     "sigma2_ratio": float(np.var(y) / np.var(y_exact)) if np.var(y_exact) > 0 else None}
    rows.append(row)
    print(json.dumps({"table1": row}), flush=True)

"""Fused (hash inside the aggregation) vs split (pac_mask kernel, then aggregation with explicit
masks) on a BASELINE config: device times of each piece (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen as dg  # noqa: E402
import paper_2603_15023_b200 as pac  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = dg.WORKLOADS[cfg]
cols = dg.device_columns(w, 0, w.n_rows)
kinds = [k for k, _ in w.aggs]
vals = [None if i < 0 else cols["values"][i] for _, i in w.aggs]
G_cap = {"C1": 1, "C2": 8, "C4": 1024, "C5": 100}.get(w.name, 1 << 21)
ag = pac.Aggregator(kinds, G_cap)
salt = 12345
m = pac.mask(cols["pu"], salt)
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def t(fn, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(it):
        fn()
    e[1].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / it


fused = t(lambda: ag(vals, cols["keys"], pu_key=cols["pu"], salt=salt))
mask_ms = t(lambda: pac.mask(cols["pu"], salt, m))
agg_mask = t(lambda: ag(vals, cols["keys"], mask=m))
print(f"{cfg}: fused {fused:.3f} ms | split: pac_mask {mask_ms:.3f} + agg(mask) {agg_mask:.3f} = {mask_ms + agg_mask:.3f} ms")

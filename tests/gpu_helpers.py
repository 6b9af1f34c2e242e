"""Shared helpers for the -m gpu parity tests: run the CUDA path through the binding and
compare with the oracle on the same input bytes."""
import numpy as np

import datagen as dg

REL_F64 = 1e-9  # north_star tolerance for f64 sums / AVG / variance (R16)

KIND_MAP = {dg.AGG_COUNT: 0, dg.AGG_SUM_I64: 1, dg.AGG_SUM_F64: 2, dg.AGG_AVG_F64: 3,
            dg.AGG_MIN_F64: 4, dg.AGG_MAX_F64: 5}


def to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def workload_aggs(w, cols):
    """[(kind, host values or None)] for a datagen workload."""
    return [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]


def run_gpu(aggs_host, keys_host, pu=None, masks=None, salt=0, G_cap=1024, spill_rows=None):
    import paper_2603_15023_b200 as pac
    ag = pac.Aggregator([k for k, _ in aggs_host], G_cap, spill_rows=spill_rows)
    cache = {}  # one device copy per host column (aggregates may share a column)
    vals = []
    for _, v in aggs_host:
        if v is None:
            vals.append(None)
        else:
            if id(v) not in cache:
                cache[id(v)] = to_dev(v)
            vals.append(cache[id(v)])
    keys = [to_dev(k) for k in keys_host]
    t = ag(vals, keys, pu_key=None if pu is None else to_dev(pu),
           mask=None if masks is None else to_dev(masks.view(np.int64)), salt=salt)
    return t, ag


def assert_tables_equal(gpu: dict, ref: dict, rel=REL_F64):
    assert gpu["G"] == ref["G"], (gpu["G"], ref["G"])
    np.testing.assert_array_equal(gpu["keys"], ref["keys"])
    np.testing.assert_array_equal(gpu["rows"], ref["rows"])
    np.testing.assert_array_equal(gpu["K"], ref["K"])
    if gpu["count"] is not None:
        np.testing.assert_array_equal(gpu["count"], ref["count"])
    for a, k in enumerate(ref["kinds"]):
        g, r = gpu["world"][a], ref["world"][a]
        if k == dg.AGG_COUNT:
            continue
        if k in (dg.AGG_SUM_I64, dg.AGG_MIN_F64, dg.AGG_MAX_F64):
            np.testing.assert_array_equal(g, r, err_msg=f"aggregate {a} kind {k}")
        else:
            np.testing.assert_allclose(g, r, rtol=rel, atol=1e-300, err_msg=f"aggregate {a} kind {k}")


def assert_releases_close(rel_g, rel_o, delta_o, null_g, null_o, tol=REL_F64):
    np.testing.assert_array_equal(null_g, null_o)
    ok = null_o == 0
    a, b = rel_g[ok], rel_o[ok]
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), np.sqrt(np.abs(delta_o[ok])))
    assert np.all(np.abs(a - b) <= tol * np.maximum(scale, 1e-300)), np.max(np.abs(a - b) / scale)
    assert np.all(np.isnan(rel_g[~ok]))


def assert_delta_close(d_gpu, d_orc, ymax, budget, rel=REL_F64):
    """Delta = s^2/(2B): <= 1e-9 relative, or within the fp64 rounding of the two-pass
    weighted variance, |err(s^2)| <~ (64 eps max|y|)^2 (cancellation when s^2 << y^2)."""
    eps = np.finfo(np.float64).eps
    atol = 4.0 * (64.0 * eps * ymax) ** 2 / (2.0 * budget)
    bad = np.abs(d_gpu - d_orc) > rel * np.abs(d_orc) + atol
    assert not np.any(bad), (d_gpu[bad][:5], d_orc[bad][:5], atol[bad][:5])

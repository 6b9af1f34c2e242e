"""-m gpu parity of the approximate 64-world SUM (pac_approx_sum, §8 f3; R35, R36) with the oracle:
the final level counters bit-exact and the decoded world values exactly equal, for the two-sided
and the single-sided state, hashed pu keys and explicit masks, several block sizes (one block,
ragged last block, many blocks) and Table 1's value distributions; plus the released-scale
relation to the exact GPU SUM (pac_agg_grouped) within R35's bound."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import run_gpu, to_dev

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_15023_b200 as pac  # noqa: E402


def _dist(name, n, rng):
    return {"uniform_int": lambda: rng.integers(1, 2**31, n),
            "uniform_tinyint": lambda: rng.integers(0, 128, n),
            "negative_mixed": lambda: rng.integers(-10**9, 10**9, n),
            "sparse_large": lambda: np.where(rng.random(n) < 0.01, rng.integers(10**12, 10**13, n), 0),
            "zipf_like": lambda: np.minimum(rng.zipf(1.5, n), 10**9)}[name]().astype(np.int64)


@pytest.mark.parametrize("two_sided", [True, False])
@pytest.mark.parametrize("dist", ["uniform_int", "uniform_tinyint", "negative_mixed", "sparse_large", "zipf_like"])
@pytest.mark.parametrize("n,block", [(1, 65536), (100_003, 4096), (1_000_000, 65536), (70_000, 70_000)])
def test_counters_bit_exact(orc, two_sided, dist, n, block):
    rng = np.random.default_rng(hash((dist, n, block)) % 2**32)
    v = _dist(dist, n, rng)
    pu = rng.integers(0, max(1, n // 20), n).astype(np.int64)
    cnt, y = pac.approx_sum(to_dev(v), pu_key=to_dev(pu), salt=33, two_sided=two_sided, block_rows=block)
    c_o, y_o = orc.approx_sum(orc.pac_hash(pu, 33), v, block_rows=block, two_sided=two_sided)
    np.testing.assert_array_equal(cnt.cpu().numpy().view(np.uint16), c_o)
    np.testing.assert_array_equal(y.cpu().numpy(), y_o)


def test_explicit_masks(orc):
    rng = np.random.default_rng(5)
    n = 300_000
    masks = rng.integers(-(2**63), 2**63 - 1, n, dtype=np.int64).astype(np.uint64)
    masks[::7] = 0
    v = rng.integers(-(2**40), 2**40, n).astype(np.int64)
    cnt, y = pac.approx_sum(to_dev(v), mask=to_dev(masks.view(np.int64)), block_rows=8192)
    c_o, y_o = orc.approx_sum(masks, v, block_rows=8192)
    np.testing.assert_array_equal(cnt.cpu().numpy().view(np.uint16), c_o)
    np.testing.assert_array_equal(y.cpu().numpy(), y_o)


def test_close_to_the_exact_gpu_sum(orc):
    # the C1 column (int64 U[1, 1e6]): approximate world sums within 2 (2^-8 + 2^-12) sum |v| of the
    # exact SUM_I64 the grouped kernel computes (R7 scale: y = 2 sum)
    w = dg.WORKLOADS["C1"]
    cols = w.host_columns(0, 1_000_000)
    v = cols["values"][0]
    t, _ = run_gpu([(dg.AGG_SUM_I64, v)], [], pu=cols["pu"], salt=8, G_cap=1)
    exact = t.to_host()["world"][0][0].astype(np.float64)
    _, y = pac.approx_sum(to_dev(v), pu_key=to_dev(cols["pu"]), salt=8)
    err = np.abs(y.cpu().numpy() - 2.0 * exact)
    assert np.all(err <= 2.0 * (2.0**-8 + 2.0**-12) * exact)

"""-m gpu parity of the PU-key join (§8 f2, reading R27) through the C-ABI against the
oracle: one- and two-level FK chains with dangling keys and the INT64_MIN sentinel key
(bit-exact masks and PU keys), duplicate primary keys reported, empty inputs, and the
Q01-shaped end-to-end path lineitem -> orders.o_custkey -> pac_hash -> grouped aggregation."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import assert_tables_equal, to_dev

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_15023_b200 as pac  # noqa: E402

I64MIN = np.iinfo(np.int64).min


def _orders(rng, n_cust, n_ord):
    custkey = rng.permutation(10**8)[:n_cust].astype(np.int64) - 5 * 10**7
    orderkey = rng.permutation(10**9)[:n_ord].astype(np.int64)
    o_custkey = custkey[rng.integers(0, n_cust, n_ord)]
    return orderkey, o_custkey


def test_one_level_chain_bit_exact(orc):
    rng = np.random.default_rng(1)
    orderkey, o_custkey = _orders(rng, 20_000, 150_000)
    orderkey[7] = I64MIN                          # the empty-slot sentinel as a real key
    n = 1_000_003
    fk = orderkey[rng.integers(0, len(orderkey), n)]
    fk[::101] = -12345                            # dangling
    fk[5] = I64MIN
    salt = 0x243F6A8885A308D3
    t = pac.JoinTable(to_dev(orderkey), to_dev(o_custkey))
    assert t.status() == 0
    mask, pu = pac.join_mask([t], to_dev(fk), salt, want_pu=True)
    m_o, f_o, pu_o = orc.join_chain_mask([(orderkey, o_custkey)], fk, salt)
    np.testing.assert_array_equal(pac.as_u64(mask), m_o)
    np.testing.assert_array_equal(pu.cpu().numpy(), pu_o)
    assert np.all(m_o[::101] == 0)


def test_two_level_chain_and_duplicates(orc):
    rng = np.random.default_rng(2)
    a_pk = rng.permutation(10**6)[:5000].astype(np.int64)
    b_pk = rng.permutation(10**6)[:800].astype(np.int64) * 7
    a_next = b_pk[rng.integers(0, 800, 5000)]
    a_next[::13] = 3                               # dangling at the second level
    b_next = rng.integers(-(2**62), 2**62, 800).astype(np.int64)
    fk = a_pk[rng.integers(0, 5000, 300_000)]
    ta, tb = pac.JoinTable(to_dev(a_pk), to_dev(a_next)), pac.JoinTable(to_dev(b_pk), to_dev(b_next))
    mask, pu = pac.join_mask([ta, tb], to_dev(fk), 99, want_pu=True)
    m_o, f_o, pu_o = orc.join_chain_mask([(a_pk, a_next), (b_pk, b_next)], fk, 99)
    np.testing.assert_array_equal(pac.as_u64(mask), m_o)
    np.testing.assert_array_equal(pu.cpu().numpy(), pu_o)
    dup = np.concatenate([a_pk, a_pk[:3]])
    td = pac.JoinTable(to_dev(dup), to_dev(np.zeros(len(dup), dtype=np.int64)))
    assert td.status() == pac._lib.PAC_E_INVAL


def test_empty_inputs(orc):
    e = np.zeros(0, dtype=np.int64)
    t = pac.JoinTable(to_dev(e), to_dev(e))
    fk = np.arange(1000, dtype=np.int64)
    mask = pac.join_mask([t], to_dev(fk), 1)
    assert np.all(pac.as_u64(mask) == 0)           # nothing matches: in no world
    t2 = pac.JoinTable(to_dev(fk), to_dev(fk))
    assert pac.join_mask([t2], torch.zeros(0, dtype=torch.int64, device="cuda"), 1).numel() == 0


def test_q01_shape_join_then_aggregate(orc):
    """lineitem scans gain JOIN orders ON l_orderkey = o_orderkey; o_custkey is
    hashed directly (join elimination); the masks feed the grouped aggregation."""
    rng = np.random.default_rng(3)
    orderkey, o_custkey = _orders(rng, 5000, 40_000)
    n = 400_000
    l_orderkey = orderkey[rng.integers(0, len(orderkey), n)]
    g1 = rng.integers(0, 3, n).astype(np.int8)
    g2 = rng.integers(0, 2, n).astype(np.int8)
    price = rng.integers(100, 10**7, n).astype(np.int64)
    disc = rng.random(n) * 0.1
    salt = 0x5EED
    t = pac.JoinTable(to_dev(orderkey), to_dev(o_custkey))
    mask = pac.join_mask([t], to_dev(l_orderkey), salt)
    ag = pac.Aggregator([pac.SUM_I64, pac.AVG_F64, pac.COUNT], 8)
    tab = ag([to_dev(price), to_dev(disc), None], [to_dev(g1), to_dev(g2)], mask=mask)
    m_o, _, _ = orc.join_chain_mask([(orderkey, o_custkey)], l_orderkey, salt)
    aggs = [(dg.AGG_SUM_I64, price), (dg.AGG_AVG_F64, disc), (dg.AGG_COUNT, None)]
    assert_tables_equal(tab.to_host(), orc.agg(m_o, [g1, g2], aggs))

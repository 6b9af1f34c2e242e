"""Pins of the oracle's PU-key join (§8 f2, reading R27) against things other than
itself: a Python dict walk of the FK chain (the definition of an equi-join lookup), the join
elimination identity H(T_k.fk_U) = H(U.pk) (Eq. join-elim), and unmatched keys -> mask 0."""
import numpy as np

import oracle as orc


def test_chain_matches_dict_walk_and_join_elimination():
    rng = np.random.default_rng(1)
    n_cust, n_ord, n_li = 500, 4000, 30_000
    custkey = rng.permutation(10**6)[:n_cust].astype(np.int64) - 500_000      # U.pk (scrambled)
    orderkey = rng.permutation(10**7)[:n_ord].astype(np.int64)                 # orders.pk
    o_custkey = custkey[rng.integers(0, n_cust, n_ord)]                        # orders.fk_U
    l_orderkey = orderkey[rng.integers(0, n_ord, n_li)]                        # lineitem.fk1
    l_orderkey[::97] = -7                                                      # dangling FKs
    salt = 0x1234
    mask, found, pu = orc.join_chain_mask([(orderkey, o_custkey)], l_orderkey, salt)
    d = dict(zip(orderkey.tolist(), o_custkey.tolist()))
    for i in range(0, n_li, 7):
        if l_orderkey[i] in d:
            assert found[i] == 1 and pu[i] == d[l_orderkey[i]]
            # join elimination: hashing the FK equals hashing U's primary key
            assert int(mask[i]) == int(orc.pac_hash(np.array([pu[i]]), salt)[0])
        else:
            assert found[i] == 0 and mask[i] == 0
    assert found[::97].sum() == 0


def test_two_level_chain():
    rng = np.random.default_rng(2)
    a_pk = np.arange(100, dtype=np.int64) * 3 + 1
    a_next = rng.integers(0, 50, 100).astype(np.int64) * 5
    b_pk = np.arange(50, dtype=np.int64) * 5
    b_next = rng.integers(-10**12, 10**12, 50).astype(np.int64)
    fk = rng.choice(np.concatenate([a_pk, [2, 4, 6]]), 5000).astype(np.int64)
    mask, found, pu = orc.join_chain_mask([(a_pk, a_next), (b_pk, b_next)], fk, 9)
    da, db = dict(zip(a_pk.tolist(), a_next.tolist())), dict(zip(b_pk.tolist(), b_next.tolist()))
    for i in range(len(fk)):
        want = db.get(da.get(int(fk[i]), None), None) if int(fk[i]) in da else None
        assert (found[i] == 1) == (want is not None)
        if want is not None:
            assert pu[i] == want
    assert np.all(np.unpackbits(mask[found == 1].view(np.uint8).reshape(-1, 8), axis=1).sum(1) == 32)

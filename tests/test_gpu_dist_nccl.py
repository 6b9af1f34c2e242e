"""The NCCL merge path (§8e) on the GPU with a single-rank process group: the collectives the
multi-GPU bench issues (all_gather of key counts and keys, all_reduce SUM int64 / f64, MIN/MAX
f64) run through NCCL on the device tables, and the merged table still equals the oracle's.
(More ranks need more GPUs; the two-rank merge is tested with gloo, tests/test_dist_gloo.py.)"""
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist

import datagen as dg
from gpu_helpers import assert_tables_equal, run_gpu, to_dev

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_single_rank_merge_matches_oracle(orc):
    from paper_2603_15023_b200 import dist as pdist
    rng = np.random.default_rng(21)
    n = 200_000
    pu = rng.integers(0, 20_000, n).astype(np.int64)
    g = rng.integers(0, 300, n).astype(np.int32)
    iv = rng.integers(-10**6, 10**6, n).astype(np.int64)
    fv = rng.normal(5, 2, n)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv), (dg.AGG_AVG_F64, fv), (dg.AGG_MIN_F64, fv),
            (dg.AGG_MAX_F64, fv)]
    t, _ = run_gpu(aggs, [g], pu=pu, salt=13, G_cap=512)
    dev_aggs = [(k, None if v is None else to_dev(v)) for k, v in aggs]
    store = tdist.TCPStore("127.0.0.1", _free_port(), 1, True)
    tdist.init_process_group("nccl", store=store, rank=0, world_size=1,
                             device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        merged = pdist.merge_table(t, dev_aggs)
        torch.cuda.synchronize()
    finally:
        tdist.destroy_process_group()
    assert_tables_equal(merged.to_host(), orc.agg(orc.pac_hash(pu, 13), [g], aggs))

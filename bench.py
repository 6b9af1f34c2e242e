"""bench.py -- PAC grouped-aggregation throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

A step is one pass of the whole hot path over one batch of synthetic rows (§8 a1-a7):
fused pac_hash + group-slot resolution + 64-world COUNT/SUM/AVG accumulation + combine
(+ NCCL allreduce of the partial tables when N > 1) + finalize with posterior updates.
Default workload: BASELINE.json configs[1] (C2: 6e7 rows per GPU, 6 groups), the config
the metric is quoted on.  Multi-GPU: one process per GPU (torchrun), each rank aggregates
its own 6e7-row shard of one global dataset (weak scaling), merged by NCCL allreduce.

Prints ONE JSON line (rank 0).  `value` = rows/s over all ranks, device-timed with CUDA
events (max over ranks); `e2e` = the same metric through the public API with pinned-host
inputs copied H2D and the releases copied D2H inside the timed region; `roofline` = the
aggregation kernel's algorithmic input bytes / its event-timed duration vs the measured
HBM copy peak; `cpu_baseline` = the CPU oracle on a bounded sample (rank 0, N=1 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PAC grouped-aggregate rows/s; achieved HBM GB/s vs peak at 1/2/4/8 GPUs"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def _traffic(cfg):
    """Per-launch DRAM bytes of the aggregation kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(cfg, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for i, n in enumerate(names):
                if len(s) > 5 + i and s[5 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------------- CPU legs
def oracle_rows_per_s(w, budget_s: float = 12.0, max_rows: int = 4_000_000):
    max_rows = min(max_rows, w.n_rows)
    """The CPU oracle (as it stands) on a bounded sample of the workload: rows/s."""
    import numpy as np

    import oracle
    oracle.build()
    seed = 0xC0FFEE
    jstar, salt, P = oracle.session(seed)
    # calibrate on a small prefix, then size the sample for ~budget_s of CPU work
    n0 = min(100_000, max_rows)
    cols = w.host_columns(0, n0)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    t = time.perf_counter()
    tab = oracle.agg(oracle.pac_hash(cols["pu"], salt), cols["keys"], aggs)
    oracle.finalize(seed, w.budget, jstar, P, tab)
    rate = n0 / (time.perf_counter() - t)
    n = int(min(max_rows, max(n0, rate * budget_s)))
    cols = w.host_columns(0, n)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    t = time.perf_counter()
    tab = oracle.agg(oracle.pac_hash(cols["pu"], salt), cols["keys"], aggs)
    oracle.finalize(seed, w.budget, jstar, P, tab)
    el = time.perf_counter() - t
    return n / el, n, el


def run_reference(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np  # noqa: F401
    steps_val = []
    sample = None
    for i in range(args.warmup + args.steps):
        v, n, el = oracle_rows_per_s(w, budget_s=max(min(2.0, args.ref_seconds),
                                                     args.ref_seconds / max(1, args.warmup + args.steps)),
                                     max_rows=2_000_000)
        if i >= args.warmup:
            steps_val.append(v)
        sample = n
    val = statistics.median(steps_val)
    cores = 1
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "rows/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sample / val * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i64+f64",
        "data": "synthetic", "config": {"workload": w.name, "rows_per_step": sample,
                                        "description": w.description},
        "cpu_baseline": {"value": val, "unit": "rows/s", "cores": cores, "kind": "oracle",
                         "sample": f"first {sample} rows of {w.name} per step (oracle O2 + finalize, 1 thread)"},
        "e2e": {"value": val, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------- GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--rows", type=int, default=0, help="override rows per GPU (testing only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=60.0,
                    help="--impl reference: total CPU seconds the oracle samples take")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    import datagen as dg
    w = dg.WORKLOADS[args.config]
    if args.rows:
        w = w.scaled(args.rows)
    if args.impl == "reference":
        return run_reference(args, w)

    import torch
    import torch.distributed as tdist

    import paper_2603_15023_b200 as pac
    from paper_2603_15023_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        tdist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            tdist.barrier()

    n = w.n_rows
    row0 = rank * n  # weak scaling: rank r owns rows [r*n, (r+1)*n) of one global dataset
    cols = dg.device_columns(w, row0, n, device=dev)
    keys = cols["keys"]
    vals = [None if i < 0 else cols["values"][i] for _, i in w.aggs]
    kinds = [k for k, _ in w.aggs]
    # capacity hints from the key domains of the synthetic configs (R20 packed keys)
    G_cap = {"C1": 1, "C2": 8, "C4": 1024, "C5": 100}.get(w.name, 1 << 21)
    seed = 0x5EED
    sess = pac.Session(seed, w.budget)
    ag = pac.Aggregator(kinds, G_cap, dev)
    fin = pac.Finalizer(kinds, G_cap, dev)
    aggs_spec = list(zip(kinds, vals))
    stream = torch.cuda.current_stream(dev)

    def step(pu, keys_, vals_):
        t = ag(vals_, keys_, pu_key=pu, salt=sess.salt)
        if world > 1:
            t = pdist.merge_table(t, list(zip(kinds, vals_)))
        for r in range(w.rounds):
            fin(sess, t, r)
        return t

    # warm-up (untimed)
    for _ in range(args.warmup):
        step(cols["pu"], keys, vals)
    torch.cuda.synchronize(dev)
    G = ag.table.check()

    # ---- device-timed region
    pac.profile_enable(True)
    pac.profile_read()
    l0 = pac.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(args.steps):
            step(cols["pu"], keys, vals)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    launches = pac.launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    k_ms, k_n = pac.profile_read()
    pac.profile_enable(False)
    if world > 1:
        t = torch.tensor([ms, k_ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms, k_ms = float(t[0]), float(t[1])
    ms_step = ms / args.steps
    value = (n * world) / (ms_step / 1e3)

    # ---- end-to-end through the public API: pinned host inputs H2D + releases D2H
    host = {"pu": cols["pu"].cpu().pin_memory(), "keys": [k.cpu().pin_memory() for k in keys]}
    d2h = G * len(kinds) * 9  # releases (f64) + NULL flags (u8)
    res_host = torch.empty(G_cap, len(kinds), dtype=torch.float64).pin_memory()
    null_host = torch.empty(G_cap, len(kinds), dtype=torch.uint8).pin_memory()
    d_pu = torch.empty_like(cols["pu"])
    d_keys = [torch.empty_like(k) for k in keys]
    # one device buffer per distinct column (aggregates may share a column, e.g. MIN+MAX)
    uniq = {}
    for v in vals:
        if v is not None and id(v) not in uniq:
            uniq[id(v)] = (torch.empty_like(v), v.cpu().pin_memory())
    d_vals = [None if v is None else uniq[id(v)][0] for v in vals]
    h2d = host["pu"].numel() * 8 + sum(k.numel() * k.element_size() for k in host["keys"]) + sum(
        h.numel() * h.element_size() for _, h in uniq.values())

    def e2e_step():
        d_pu.copy_(host["pu"], non_blocking=True)
        for d, h in zip(d_keys, host["keys"]):
            d.copy_(h, non_blocking=True)
        for d, h in uniq.values():
            d.copy_(h, non_blocking=True)
        t = step(d_pu, d_keys, d_vals)
        res_host.copy_(fin.release, non_blocking=True)
        null_host.copy_(fin.is_null, non_blocking=True)

    e2e_step()
    torch.cuda.synchronize(dev)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e_ms = float(t[0])
    e2e_value = (n * world) / (e_ms / args.e2e_steps / 1e3)

    if rank == 0:
        peak, peak_src = _peaks()
        alg_bytes = n * w.in_bytes_per_row
        k_avg_ms = k_ms / max(1, k_n)
        achieved = alg_bytes / (k_avg_ms / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "i64+f64", "data": "synthetic",
            "config": {"workload": w.name, "rows_per_gpu": n, "groups": G, "aggregates": len(kinds),
                       "finalize_rounds": w.rounds, "in_bytes_per_row": w.in_bytes_per_row,
                       "l2": f"inputs {alg_bytes / 1e9:.2f} GB per GPU > 126 MB L2 (no flush needed)",
                       "description": w.description},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _traffic(w.name),
                         "kernel": "k_agg_tiles (pac_agg_grouped main kernel)",
                         "kernel_ms": k_avg_ms, "kernel_share_of_step": k_avg_ms / ms_step,
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": alg_bytes},
            "e2e": {"value": e2e_value, "unit": "rows/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                v, ns, el = oracle_rows_per_s(w)
                line["cpu_baseline"] = {"value": v, "unit": "rows/s", "cores": 1, "kind": "oracle",
                                        "sample": f"first {ns} rows of {w.name} (oracle pac_hash + O2 + "
                                                  f"finalize, 1 thread, {el:.1f} s)"}
            except Exception as e:  # report, never hide
                line["cpu_baseline"] = {"value": None, "error": repr(e)}
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""bench.py -- PAC grouped-aggregation throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl reference]

A step is one pass of the whole hot path over one batch of synthetic rows (§8 a1-a7):
fused pac_hash + group-slot resolution + 64-world COUNT/SUM/AVG accumulation + combine
(+ the cross-GPU merge -- pac_merge_pack, three NCCL all_reduce, pac_merge_unpack -- when N > 1)
+ finalize with posterior updates (C5: d = 20 rounds).
Default workload: BASELINE.json configs[4] (C5: 1.2e9 rows, 100 groups, COUNT + SUM + AVG, 20
finalize rounds), the configuration the metric is quoted on ("at 1/2/4/8 GPUs").  Multi-GPU: one
process per GPU (torchrun); the 1.2e9 rows of one global dataset are row-sharded across the ranks
(strong scaling: rank r owns rows [r n / N, (r + 1) n / N)).

Prints ONE JSON line (rank 0).  `value` = rows/s over all ranks, device-timed with CUDA events
(max over ranks); `e2e` = the same metric through the public API with pinned-host inputs copied
H2D and the releases copied D2H inside the timed region; `roofline` = the aggregation pass's
algorithmic bytes / its event-timed duration vs the measured HBM copy peak, with the issue-slot
(ALU) fraction beside it; `cpu_baseline` = the CPU oracle on a bounded sample, on every host core
and on one (rank 0, N = 1 only).
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


def _profile_entry(cfg):
    """Per-launch DRAM bytes and warp-instructions per row of the aggregation pass, from the
    committed ncu summary (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(cfg, {})
    except Exception:
        return {}


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
def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_run(w, n, threads, seed=0xC0FFEE):
    """The CPU oracle (as it stands) on the first n rows of the workload: pac_hash + O2 (on
    `threads` host threads: row ranges, partial tables combined in thread order) timed
    together; finalize (all rounds, sequential by definition) timed separately."""
    import oracle
    oracle.build()
    jstar, salt, P = oracle.session(seed)
    cols = w.host_columns(0, n)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    t = time.perf_counter()
    if threads > 1:
        tab = oracle.agg_mt(oracle.pac_hash_mt(cols["pu"], salt, threads), cols["keys"], aggs, threads)
    else:
        tab = oracle.agg(oracle.pac_hash(cols["pu"], salt), cols["keys"], aggs)
    t_agg = time.perf_counter() - t
    t = time.perf_counter()
    for r in range(w.rounds):
        _, _, _, _, P = oracle.finalize(seed, w.budget, jstar, P, tab, r)
    t_fin = time.perf_counter() - t
    return t_agg, t_fin


def cpu_baseline(w, budget_s=20.0, max_rows=100_000_000):
    """Rows/s of the oracle on all host cores (bounded sample of ~budget_s of CPU work, calibrated
    on a prefix) and on one core; aggregation and finalize timed separately."""
    cores = os.cpu_count() or 1
    n0 = min(200_000, w.n_rows)
    a0, f0 = oracle_run(w, n0, 1)
    rate1 = n0 / a0
    n = int(min(w.n_rows, max(n0, rate1 * cores * budget_s * 0.5)))
    if max_rows:
        n = min(n, max_rows)
    a_all, f_all = oracle_run(w, n, cores)
    n1 = int(min(n, max(n0, rate1 * budget_s * 0.25)))
    a_one, _ = oracle_run(w, n1, 1)
    return {
        "value": n / (a_all + f_all), "unit": "rows/s", "cores": cores, "kind": "oracle",
        "cpu_model": _cpu_model(),
        "sample": f"first {n} rows of {w.name}: oracle pac_hash + O2 on {cores} threads "
                  f"({a_all:.2f} s) + finalize x{w.rounds} rounds ({f_all:.3f} s)",
        "agg_rows_per_s": n / a_all, "finalize_s": f_all,
        "one_core": {"rows": n1, "agg_rows_per_s": n1 / a_one},
    }


def run_reference(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps_val = []
    per = max(2.0, args.ref_seconds / max(1, args.warmup + args.steps))
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(w, budget_s=per)
        if i >= args.warmup:
            steps_val.append(cb["value"])
    val = statistics.median(steps_val)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "rows/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * w.n_rows / val,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "i64+f64",
        "data": "synthetic", "config": {"workload": w.name, "rows": w.n_rows, "description": w.description},
        "cpu_baseline": dict(cb, value=val),
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
    ap.add_argument("--config", default="C5")
    ap.add_argument("--rows", type=int, default=0, help="override rows per GPU (testing only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=60.0,
                    help="--impl reference: total CPU seconds the oracle samples take")
    ap.add_argument("--weak", action="store_true", help="every rank aggregates the full config (weak scaling)")
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

    if args.weak:
        n, row0 = w.n_rows, rank * w.n_rows  # weak: rank r owns rows [r n, (r + 1) n) of one dataset
    else:  # strong: the config's rows are row-sharded across the ranks
        row0 = w.n_rows * rank // world
        n = w.n_rows * (rank + 1) // world - row0
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
        if world > 1:  # dense domains: every shard holds every group (checked on the device)
            t = pdist.merge_table(t, list(zip(kinds, vals_)), same_keys=w.name != "C3")
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
    total_rows = n * world if args.weak else w.n_rows
    value = total_rows / (ms_step / 1e3)
    status = int(ag.table.status.item())  # after the timed region: a merge or capacity error is fatal
    if status != 0:
        raise RuntimeError(f"table status {status} after the timed steps")

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
    e2e_value = total_rows / (e_ms / args.e2e_steps / 1e3)

    if rank == 0:
        peak, peak_src = _peaks()
        prof = _profile_entry(w.name)
        # algorithmic bytes of one aggregation pass on this rank: the input columns,
        # plus the [G][64] table arrays written once (only material for C3's ~1e6 groups)
        arrays = 1 + sum(1 for k in kinds if k != pac.COUNT)
        alg_bytes = n * w.in_bytes_per_row + (G * 64 * 8 * arrays if w.name == "C3" else 0)
        k_avg_ms = k_ms / max(1, k_n)
        achieved = alg_bytes / (k_avg_ms / 1e3) / 1e9
        clocks = clk.summary()
        f_sm = (clocks.get("sm_mhz") or 1965.0) * 1e6
        issue_peak = 148 * 4 * f_sm  # warp-instructions/s: 148 SMs x 4 schedulers x 1 issue/clk
        wipr = prof.get("warp_instr_per_row")
        traffic = prof.get("dram_bytes_per_row")
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": "i64+f64", "data": "synthetic",
            "config": {"workload": w.name, "rows": total_rows, "rows_per_gpu": n, "groups": G,
                       "aggregates": len(kinds), "finalize_rounds": w.rounds,
                       "in_bytes_per_row": w.in_bytes_per_row,
                       "l2": f"inputs {n * w.in_bytes_per_row / 1e9:.2f} GB per GPU > 126 MB L2 (no flush needed)",
                       "description": w.description},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": None if traffic is None else traffic * n,
                         "kernel": pac.profile_last_kernel(),
                         "kernel_ms": k_avg_ms, "kernel_share_of_step": k_avg_ms / ms_step,
                         "peak_source": peak_src, "algorithmic_bytes_per_launch": alg_bytes,
                         "profile_source": prof.get("source"),
                         "alu_issue": None if wipr is None else {
                             "warp_instr_per_row": wipr, "peak_warp_instr_per_s": issue_peak,
                             "frac": wipr * n / (k_avg_ms / 1e3) / issue_peak}},
            "e2e": {"value": e2e_value, "unit": "rows/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline(w)
            except Exception as e:  # report, never hide
                line["cpu_baseline"] = {"value": None, "error": repr(e)}
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""Benchmark of the B200 Hive table hot path (BASELINE.json metric).

Workload (BASELINE.json configs[1], "static build + lookup"): a step clears the
table, inserts 2^26 unique uniform keys into 2,207,529 buckets (LF 0.95,
growth off) and runs 2^26 finds with 50% hits.  Inputs (256 MiB keys, 256 MiB
values, 256 MiB queries) and the 565 MB table are all larger than L2, so no L2
flush is needed between steps.

`python bench.py [--gpus N --steps K --warmup W] [--impl reference]`
N > 1 runs under torchrun: each rank owns a hash-partitioned shard and its own
2^26-key batch (weak scaling); keys are routed by an NCCL all-to-all.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import gen  # noqa: E402

METRIC = "G lookups/s and G updates/s at 95% load, 1/2/4/8 B200, % of HBM roofline"
UNIT = "G ops/s"
N_LOG2 = 26


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n-log2", type=int, default=N_LOG2, help="keys per rank (debug only)")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", choices=("nccl", "p2p"), default="nccl",
                    help="sharded path: NCCL all-to-all (default) or the peer-memory exchange (NEXT-1)")
    ap.add_argument("--cfg5", action="store_true",
                    help="BASELINE config 5: a hash-sharded table of 2^T keys over the ranks (strong scaling), "
                         "inserted, looked up (50%% hits) and 2^(T-3) erased in 2^26-op batches")
    ap.add_argument("--cfg5-log2", type=int, default=31, help="T of --cfg5 (total keys 2^T)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the hash-sharded (NCCL all-to-all) path even at world size 1 (testing)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------------------
# clocks sampled during the timed region (NVML)
# ---------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons)}


# ---------------------------------------------------------------------------------------
# CPU oracle baseline / reference arm
# ---------------------------------------------------------------------------------------
def oracle_sample(n_log2: int):
    """Oracle (as it stands) on a bounded sample of the workload: build 2^n_log2
    keys to LF 0.95, then 2^n_log2 finds with 50% hits. Returns (ops, seconds)."""
    import oracle
    n = 1 << n_log2
    nb = -(-n * 100 // (95 * 32))
    ids = np.arange(n, dtype=np.uint32)
    keys, vals = gen.keys_of(ids), gen.vals_of(ids)
    qids, _ = gen.mixed_queries(n // 2, n // 2, n, seed=202)
    q = gen.keys_of(qids)
    t = oracle.OracleTable(nb * 32, lf_grow=2.0, lf_shrink=0)
    t0 = time.perf_counter()
    t.insert(keys, vals)
    t.find(q)
    dt = time.perf_counter() - t0
    return 2 * n, dt


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    import oracle
    oracle.build()
    n_log2 = 20
    for _ in range(args.warmup):
        oracle_sample(n_log2)
    tot_ops, tot_s = 0, 0.0
    for _ in range(args.steps):
        ops, s = oracle_sample(n_log2)
        tot_ops += ops
        tot_s += s
    v = tot_ops / tot_s / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": "cfg2 build+lookup at LF 0.95 (oracle sample: 2^20 keys + 2^20 finds per step)",
                   "parallelism": "single host core"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": "2^20 inserts to LF 0.95 + 2^20 finds (50% hits) per step"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.cfg5:
        run_cfg5(args, rank, world, local)
        return

    import torch
    import torch.distributed as dist

    from paper_2510_15095_b200 import HiveTable, u32
    from paper_2510_15095_b200.build import build as build_lib

    if rank == 0:
        build_lib()
    torch.cuda.set_device(local)
    sharded = world > 1 or args.force_sharded
    if sharded:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    if sharded:
        print(f"[bench] rank {rank}: torch.distributed nccl world {dist.get_world_size()}", file=sys.stderr,
              flush=True)

    n = 1 << args.n_log2
    nb = -(-n * 100 // (95 * 32)) if args.n_log2 != 26 else gen.CFG2_BUCKETS
    ids = (np.arange(n, dtype=np.uint64) + rank * n).astype(np.uint32)
    keys = u32(gen.keys_of(ids), dev)
    vals = u32(gen.vals_of(ids), dev)
    if world == 1:
        qids, _ = gen.mixed_queries(n // 2, n // 2, n, seed=202)
    else:
        rng = np.random.default_rng(202 + rank)
        hit_ids = rng.integers(0, n * world, n // 2, dtype=np.uint64)
        miss_ids = np.arange(n // 2, dtype=np.uint64) + (1 << 31) + rank * (n // 2)
        qids = np.concatenate([hit_ids, miss_ids])[rng.permutation(n)].astype(np.uint32)
    queries = u32(gen.keys_of(qids), dev)
    status = torch.empty(n, dtype=torch.uint8, device=dev)
    vals_out = torch.empty(n, dtype=torch.uint32, device=dev)
    found = torch.empty(n, dtype=torch.uint8, device=dev)

    if sharded:
        from paper_2510_15095_b200.sharded import P2PShardedHive, ShardedHive
        if args.exchange == "p2p":
            sh = P2PShardedHive(nb * 32, region=P2PShardedHive.padded_region(n, world), lf_grow=2.0, lf_shrink=0)
        else:
            sh = ShardedHive(nb * 32, batch_max=n, lf_grow=2.0, lf_shrink=0)
        table = sh.table
        g_, r_, c_ = table.shard_info()
        print(f"[bench] rank {rank}: sharded handle nranks={g_} rank={r_} cap_per_peer={c_} "
              f"exchange={args.exchange}", file=sys.stderr, flush=True)

        def step():
            table.clear()
            if args.exchange == "p2p":
                status.copy_(sh.insert(keys, vals))
                v, f = sh.find(queries)
                vals_out.copy_(v)
                found.copy_(f)
            else:
                sh.insert(keys, vals, status)
                sh.find(queries, vals_out, found)
    else:
        table = HiveTable(nb * 32, lf_grow=2.0, lf_shrink=0)
        sh = None

        def step(ev=None):
            table.clear()
            if ev: ev[0].record()
            table.insert(keys, vals, status)
            if ev: ev[1].record()
            table.find(queries, vals_out, found)
            if ev: ev[2].record()

    # ---- warm-up ---------------------------------------------------------------------
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, barrier + sync on both sides, max over ranks -------------
    phase = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if sharded:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start.record()
        for i in range(args.steps):
            if sharded:
                step()
            else:
                step(phase[i])
        end.record()
        torch.cuda.synchronize()
    if sharded:
        dist.barrier()
    ms = start.elapsed_time(end)
    if sharded:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    total_ops = 2 * n * world
    value = total_ops / (ms_per_step * 1e-3) / 1e9

    # correctness guard on the last step (no outputs are trusted blindly): all
    # inserted keys are new and exactly half of each rank's queries hit
    st_bad = int((status != 0).sum().item())
    fnd = int(found.sum().item())
    assert st_bad == 0 and fnd == n // 2, (st_bad, fnd)

    out = {}
    if not sharded:
        ins_ms = statistics.mean(p[0].elapsed_time(p[1]) for p in phase)
        find_ms = statistics.mean(p[1].elapsed_time(p[2]) for p in phase)
        out["updates_gps"] = n / (ins_ms * 1e-3) / 1e9
        out["lookups_gps"] = n / (find_ms * 1e-3) / 1e9
        out["phase_ms"] = {"insert": ins_ms, "find": find_ms,
                           "clear": ms_per_step - ins_ms - find_ms}

    # ---- one profiled (untimed) step: per-kernel device times and launch counts ------------
    table.profile(True)
    step()
    torch.cuda.synchronize()
    prof = table.profile_read(reset=True)
    table.profile(False)
    launches_per_step = sum(c for _, c in prof.values())
    st = table.stats()
    bucket_keys = max(1, st["count"] - st["stash_used"])
    p_h1 = st["in_b1"] / bucket_keys
    hbm_peak, peak_kind = peaks()

    kern = {k: v[0] / v[1] for k, v in prof.items() if v[1]}   # avg ms per launch (memsets: 0 launches)
    launches = {k: v[1] for k, v in prof.items()}
    fam = {"k_find": "find", "k_insert_fast": "insert", "k_insert_slow": "evict", "k_erase": "erase",
           "k_dedup_elect": "elect"}
    ab = st["alg_bytes"]                                       # counted by the kernels in this step
    per_kernel = {}
    for k in kern:
        if k in fam and ab.get(fam[k]):
            per_launch = ab[fam[k]] / launches[k]
            per_kernel[k] = {"ms": kern[k], "alg_bytes_per_launch": per_launch,
                             "achieved_GBps": per_launch / (kern[k] * 1e-3) / 1e9,
                             "frac": per_launch / (kern[k] * 1e-3) / 1e9 / hbm_peak}
    dominant = max(per_kernel, key=lambda k: prof[k][0])
    algb = per_kernel[dominant]["alg_bytes_per_launch"]
    achieved = per_kernel[dominant]["achieved_GBps"]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(dominant)
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": hbm_peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm_peak,
                "traffic": traffic, "alg_bytes_per_launch": algb, "p_h1": p_h1,
                "kernel_ms": kern[dominant], "per_kernel": per_kernel,
                "alg_bytes_rule": "counted in-kernel: 256 B per bucket probe, 32 B per CAS sector, "
                                  "8 B per spill/stash word, exact key/value/result streams"}
    if not sharded:
        roofline["ceilings"] = gather_ceiling(queries, nb, dev, per_kernel, hbm_peak)
        roofline["byte_model"] = byte_model(table, n, st, prof, dev)

    # ---- e2e through the public API with host buffers (pinned) ---------------------------
    e2e = None
    if not sharded:
        keys_h = keys.cpu().pin_memory()
        vals_h = vals.cpu().pin_memory()
        q_h = queries.cpu().pin_memory()
        st_h = torch.empty(n, dtype=torch.uint8).pin_memory()
        vo_h = torch.empty(n, dtype=torch.uint32).pin_memory()
        fo_h = torch.empty(n, dtype=torch.uint8).pin_memory()

        def e2e_step():
            # public API with host buffers: hive_insert_host / hive_find_host
            # pipeline the transfers against compute inside the library
            table.clear()
            table.insert_host(keys_h, vals_h, st_h)
            table.find_host(q_h, vo_h, fo_h)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            e2e_step()
        b.record()
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b) / args.steps
        assert int(fo_h.sum().item()) == n // 2
        e2e = {"value": total_ops / (e_ms * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 3 * 4 * n, "d2h_bytes_per_step": (1 + 4 + 1) * n,
               "ms_per_step": e_ms}
        e2e.update(link_bound(keys_h, vals_h, q_h, st_h, vo_h, fo_h, e_ms))

    if sharded:
        # sharded public API with host buffers: H2D inputs, collective insert +
        # find, D2H results (every rank), max over ranks
        keys_h, vals_h, q_h = keys.cpu().pin_memory(), vals.cpu().pin_memory(), queries.cpu().pin_memory()
        st_h = torch.empty(n, dtype=torch.uint8).pin_memory()
        vo_h = torch.empty(n, dtype=torch.uint32).pin_memory()
        fo_h = torch.empty(n, dtype=torch.uint8).pin_memory()

        def e2e_step_sh():
            # the collective calls with host buffers: hive_insert_host /
            # hive_find_host on the sharded handle (H2D, exchange, D2H inside)
            table.clear()
            if args.exchange == "p2p":
                st = sh.insert(keys_h.to(dev, non_blocking=True), vals_h.to(dev, non_blocking=True))
                st_h.copy_(st, non_blocking=True)
                v, f = sh.find(q_h.to(dev, non_blocking=True))
                vo_h.copy_(v, non_blocking=True)
                fo_h.copy_(f, non_blocking=True)
            else:
                sh.insert_host(keys_h, vals_h, st_h)
                sh.find_host(q_h, vo_h, fo_h)

        e2e_step_sh()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            e2e_step_sh()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / args.steps], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
        e2e = {"value": total_ops / (e_ms * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 3 * 4 * n, "d2h_bytes_per_step": (1 + 4 + 1) * n, "ms_per_step": e_ms}

    # ---- secondary measurements (N = 1, untimed for `value`) ------------------------------
    secondary = {}
    if not sharded and not args.no_secondary:
        secondary = secondary_measurements(table, keys, vals, queries, n, nb, dev, prof)

    cpu = None
    if world == 1 and not sharded and rank == 0 and not args.no_cpu_baseline:
        s_log2 = min(24, args.n_log2)
        ops, sec = oracle_sample(s_log2)
        scale = (1 << s_log2) / n
        cpu = {"value": ops / sec / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"the cfg2 recipe at 2^{s_log2 - args.n_log2} scale: keys_of(0..2^{s_log2}) inserted "
                         f"into {-(-(1 << s_log2) * 100 // (95 * 32))} buckets (LF 0.95, growth off), then "
                         f"2^{s_log2} finds from gen.mixed_queries(seed 202) with 50% hits; sequential oracle, "
                         f"1 core (it is single-threaded)",
               "seconds": sec, "scale": scale,
               "extrapolated_full_step_s": sec / scale,
               "extrapolation": "linear in ops (the oracle's per-op cost is cache-miss bound at both sizes)",
               "host_nproc": os.cpu_count()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": "cfg2: clear + insert 2^%d unique uniform keys into %d buckets "
                                   "(LF 0.95, growth off) + 2^%d finds (50%% hits) per rank"
                                   % (args.n_log2, nb, args.n_log2),
                       "keys_per_rank": n, "buckets_per_rank": nb,
                       "parallelism": "single GPU" if not sharded else
                       f"hash-sharded x{world} ({'NCCL all-to-all' if args.exchange == 'nccl' else 'peer-memory exchange'})",
                       "l2": "inputs and table larger than L2 (no flush)", "owner_election": "on"},
            **out,
            "clocks": clk.summary(),
            "gpu_launches": launches_per_step * args.steps,
            "kernels_ms_per_step": {k: v[0] for k, v in prof.items()},
            "roofline": roofline,
            "table_stats": {k: st[k] for k in ("count", "n_buckets", "stash_used", "evictions", "max_depth",
                                               "stash_pushes", "leftovers", "in_b1")},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


def run_cfg5(args, rank: int, world: int, local: int):
    """BASELINE config 5: 2^T keys hash-sharded over the
    ranks.  Rank r inserts ids [r 2^T/G, (r+1) 2^T/G) in 2^26-op batches (routed
    by hash, not by rank) into shards sized for LF 0.95 (growth off), then
    looks up 2^T/G keys (half present ids of any rank, half absent ids from
    2^31), then erases 2^(T-3)/G of its own ids.  A step is that whole pass
    after hive_clear; value = all ranks' ops / the max-over-ranks step time."""
    import torch
    import torch.distributed as dist

    from paper_2510_15095_b200 import u32
    from paper_2510_15095_b200.build import build as build_lib
    from paper_2510_15095_b200.sharded import P2PShardedHive, ShardedHive
    if rank == 0:
        build_lib()
    torch.cuda.set_device(local)
    if world == 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29518")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    total = 1 << args.cfg5_log2
    per = total // world
    B = min(1 << 26, per)
    nb = -(-per * 100 // (95 * 32))
    sh = (P2PShardedHive(nb * 32, region=P2PShardedHive.padded_region(B, world), lf_grow=2.0, lf_shrink=0)
          if args.exchange == "p2p"
          else ShardedHive(nb * 32, batch_max=B, lf_grow=2.0, lf_shrink=0))
    rng = np.random.default_rng(505 + rank)
    ins, fnd, era = [], [], []
    for lo in range(rank * per, (rank + 1) * per, B):
        ids = np.arange(lo, lo + B, dtype=np.uint64).astype(np.uint32)
        ins.append((u32(gen.keys_of(ids), dev), u32(gen.vals_of(ids), dev)))
    for b in range(per // B):
        hit = rng.integers(0, total, B // 2, dtype=np.uint64)
        miss = (1 << 31) + rank * per // 2 + b * (B // 2) + np.arange(B // 2, dtype=np.uint64)
        q = np.concatenate([hit, miss])[rng.permutation(B)].astype(np.uint32)
        fnd.append(u32(gen.keys_of(q), dev))
    n_era = max(per // 8, 1)
    for lo in range(rank * per, rank * per + n_era, B):
        ids = np.arange(lo, min(lo + B, rank * per + n_era), dtype=np.uint64).astype(np.uint32)
        era.append(u32(gen.keys_of(ids), dev))
    ops_per_rank = per + per + n_era
    last = {}

    def step():
        sh.table.clear()
        for k, v in ins:
            last["st"] = sh.insert(k, v)
        last["found"] = [sh.find(q)[1] for q in fnd]
        last["erased"] = [sh.erase(k) for k in era]

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record()
        for _ in range(args.steps):
            step()
        end.record()
        torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([start.elapsed_time(end) / args.steps], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # correctness guard: every find batch is exactly half hits, every erase hits
    hits = sum(int(f.sum().item()) for f in last["found"])
    assert hits == len(fnd) * (B // 2), (hits, len(fnd) * (B // 2))
    assert all(bool((e == 1).all().item()) for e in last["erased"])
    cnt = torch.tensor([sh.table.stats()["count"]], device=dev, dtype=torch.int64)
    dist.all_reduce(cnt)
    assert int(cnt.item()) == total - n_era * world, int(cnt.item())
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": world * ops_per_rank / (ms * 1e-3) / 1e9, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": f"cfg5: hash-sharded table of 2^{args.cfg5_log2} keys over {world} GPU(s): "
                                   f"insert all, 2^{args.cfg5_log2} finds (50% hits), 2^{args.cfg5_log2 - 3} "
                                   f"erases, in 2^26-op batches",
                       "keys_total": total, "buckets_per_shard": nb, "batch": B,
                       "parallelism": f"hash-sharded x{world} ("
                                      f"{'NCCL all-to-all' if args.exchange == 'nccl' else 'peer-memory exchange'})",
                       "l2": "inputs and tables larger than L2 (no flush)"},
            "clocks": clk.summary(), "count_total": int(cnt.item())}), flush=True)
    dist.destroy_process_group()


def byte_model(table, n, st, prof, dev):
    """DESIGN.md §6 byte model of the two probe kernels, checked against the
    bytes the kernels count.  Rates are measured separately on the built cfg2
    table: f_fp = share of absent-key lookups whose b1 spill word lets them read
    b2 (the spill filter's false-positive rate), r2_hit = share of present-key
    lookups that read b2 (= 1 - p_h1 up to the stash).  Model, per lookup of a
    batch with hit rate h:  9 (key, value, found) + 264 (b1 + spill word)
    + 256 * (h * r2_hit + (1 - h) * f_fp) + 16 * (stash index probes).
    Insert (new key, owner election on), per op: 10 (key, value, status, flag)
    + 264 + 32 (claim CAS sector) + 256 * r_b2 + 8 * r_spill, where r_b2 = share
    of inserts that read b2 (b1 full, or a spill word allowing a b2 match) and
    r_spill = share placed in b2 (spill-word atomicOr)."""
    import torch

    from paper_2510_15095_b200 import u32
    m = 1 << 22
    pres = u32(gen.keys_of(np.random.default_rng(5).integers(0, n, m, dtype=np.uint64).astype(np.uint32)), dev)
    absn = u32(gen.absent_keys(m), dev)
    out = {}
    for name, q in (("present", pres), ("absent", absn)):
        a0 = table.stats()["alg_bytes"]["find"]
        table.find(q)
        torch.cuda.synchronize()
        out[name] = (table.stats()["alg_bytes"]["find"] - a0) / m
    r2_hit = (out["present"] - 273) / 256
    f_fp = (out["absent"] - 273) / (256 + 16)
    counted_find = st["alg_bytes"]["find"] / n
    pred_find = 273 + 256 * (0.5 * r2_hit + 0.5 * f_fp) + 8 * f_fp
    counted_ins = st["alg_bytes"]["insert"] / n
    bucket_keys = max(1, st["count"] - st["stash_used"])
    return {"p_h1": st["in_b1"] / bucket_keys, "r2_hit": r2_hit, "f_fp": f_fp,
            "find_counted_B_per_op": counted_find, "find_model_B_per_op": pred_find,
            "find_model_vs_counted": pred_find / counted_find,
            "insert_counted_B_per_op": counted_ins,
            "insert_r_b2_plus_spill": (counted_ins - 306) / 256,
            "lost_or_full_claims_per_op": st["leftovers"] / n,
            "survey_two_probe_model_B_per_op": {"find": 416, "insert": 553}}


def gather_ceiling(keys, nb, dev, per_kernel, hbm_peak, reps=5):
    """SURVEY §8(d) calibration ceiling: hive_gather_ceiling reads one random
    256 B block per key from an array the size of the cfg2 bucket array, with
    k_find's lane groups and loads; its GB/s (256 B block + 4 B key + 4 B out per
    op) is ceiling (iii), beside (i) nominal 8 TB/s and (ii) the measured copy."""
    import torch
    from paper_2510_15095_b200 import hive
    blocks = torch.zeros(nb * 32, dtype=torch.int64, device=dev)
    out = torch.empty(keys.numel(), dtype=torch.uint32, device=dev)
    s = torch.cuda.current_stream()
    for _ in range(2):
        hive.gather_ceiling(blocks, keys, out, stream=s)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for r in range(reps):
        ev[2 * r].record(s)
        hive.gather_ceiling(blocks, keys, out, stream=s)
        ev[2 * r + 1].record(s)
    torch.cuda.synchronize()
    ms = statistics.mean(ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(reps))
    gbps = keys.numel() * (256 + 8) / (ms * 1e-3) / 1e9
    # the read/write mix of an insert probe: + one 32 B sector dirtied per op
    # by a plain store (mode 1) or a CAS (mode 2)
    rw = {}
    for mode, name in ((1, "store"), (2, "cas")):
        hive.gather_ceiling_rw(blocks, keys, mode, out, stream=s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            hive.gather_ceiling_rw(blocks, keys, mode, out, stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        m = e0.elapsed_time(e1) / reps
        rw[name] = {"ms": m, "GBps": keys.numel() * (256 + 32 + 8) / (m * 1e-3) / 1e9}
    del blocks, out
    res = {"random_256B_gather_GBps": gbps, "gather_ms": ms, "gather_ops": keys.numel(),
           "gather_array_bytes": nb * 256, "measured_copy_GBps": hbm_peak, "nominal_GBps": 8000.0,
           "gather_plus_store": rw["store"], "gather_plus_cas": rw["cas"]}
    for k, v in per_kernel.items():
        res[k] = {"of_nominal": v["achieved_GBps"] / 8000.0, "of_copy": v["achieved_GBps"] / hbm_peak,
                  "of_gather": v["achieved_GBps"] / gbps,
                  "of_gather_plus_cas": v["achieved_GBps"] / rw["cas"]["GBps"]}
    return res


def link_bound(keys_h, vals_h, q_h, st_h, vo_h, fo_h, e_ms):
    """Host link bound of the e2e step: the same pinned buffers copied alone
    (H2D of the inputs, D2H of the results, each direction timed separately and
    then both at once on two streams); bound = the concurrent copy time."""
    import torch
    dev = torch.device("cuda")
    d_in = [torch.empty_like(x, device=dev) for x in (keys_h, vals_h, q_h)]
    d_out = [torch.empty_like(x, device=dev) for x in (st_h, vo_h, fo_h)]
    s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()

    def run(up, down):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        ev[0].record()
        if up:
            s_up.wait_event(ev[0])
            with torch.cuda.stream(s_up):
                for d, h in zip(d_in, (keys_h, vals_h, q_h)):
                    d.copy_(h, non_blocking=True)
        if down:
            s_dn.wait_event(ev[0])
            with torch.cuda.stream(s_dn):
                for h, d in zip((st_h, vo_h, fo_h), d_out):
                    h.copy_(d, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s_up)
        torch.cuda.current_stream().wait_stream(s_dn)
        ev[1].record()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1])

    run(True, True)
    up_ms = min(run(True, False) for _ in range(2))
    dn_ms = min(run(False, True) for _ in range(2))
    both_ms = min(run(True, True) for _ in range(2))
    h2d = sum(x.numel() * x.element_size() for x in (keys_h, vals_h, q_h))
    d2h = sum(x.numel() * x.element_size() for x in (st_h, vo_h, fo_h))
    return {"h2d_GBps": h2d / (up_ms * 1e-3) / 1e9, "d2h_GBps": d2h / (dn_ms * 1e-3) / 1e9,
            "link_bound_ms": both_ms, "frac_of_link_bound": both_ms / e_ms}


def secondary_measurements(table, keys, vals, queries, n, nb, dev, prof_main):
    """Extra single-GPU numbers reported beside `value`: the keys-unique fast
    path (no owner election), erase throughput on the full table, and the
    config-3 mixed workload with linear-hashing grow/shrink."""
    import torch

    from paper_2510_15095_b200 import HiveTable, u8, u32
    res = {}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    # keys-unique fast path (HIVE_KEYS_UNIQUE)
    tu = HiveTable(nb * 32, lf_grow=2.0, lf_shrink=0, keys_unique=True)
    for _ in range(2):
        tu.clear(); tu.insert(keys, vals); tu.find(queries)
    times = []
    for _ in range(3):
        tu.clear()
        ev[0].record(); tu.insert(keys, vals); ev[1].record(); tu.find(queries); ev[2].record()
        torch.cuda.synchronize()
        times.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
    res["unique_updates_gps"] = n / (statistics.mean(t[0] for t in times) * 1e-3) / 1e9
    del tu

    # hash pairs (§V-B, Fig. 8): the step's insert + find on the BitHash1/2 pair
    # vs the constant-memory CRC-32 / CRC-64 pair, same batch and table size
    pairs = {}
    for hp in ("bithash", "crc"):
        th = HiveTable(nb * 32, lf_grow=2.0, lf_shrink=0, hash=hp)
        for _ in range(2):
            th.clear(); th.insert(keys, vals); th.find(queries)
        times = []
        for _ in range(3):
            th.clear()
            ev[0].record(); th.insert(keys, vals); ev[1].record(); th.find(queries); ev[2].record()
            torch.cuda.synchronize()
            times.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
        ti, tf = statistics.mean(t[0] for t in times), statistics.mean(t[1] for t in times)
        pairs[hp] = {"insert_gops": n / (ti * 1e-3) / 1e9, "find_gops": n / (tf * 1e-3) / 1e9,
                     "step_gops": 2 * n / ((ti + tf) * 1e-3) / 1e9}
        del th
    pairs["crc_vs_bithash_insert"] = pairs["crc"]["insert_gops"] / pairs["bithash"]["insert_gops"]
    res["hash_pairs"] = pairs
    # erase half of the keys from the full table (dedup on)
    half = keys[: n // 2]
    table.clear(); table.insert(keys, vals)
    ev[0].record(); table.erase(half); ev[1].record()
    torch.cuda.synchronize()
    res["erase_gps"] = (n // 2) / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9

    # config 3: 64 batches x 2^20 mixed ops (40/20/40) over U = 2^26, 1K buckets
    # start, growth + shrink, then the id-order drain tail.
    nbat, bsz, U = 64, 1 << 20, 1 << 26
    ops_all = [u8(gen.bernoulli_ops(bsz, 0.4, 0.2, seed=1000 + b), dev) for b in range(nbat)]
    ids_all = [gen.uniform_ids(bsz, U, seed=2000 + b) for b in range(nbat)]
    k_all = [u32(gen.keys_of(i), dev) for i in ids_all]
    v_all = [u32(gen.vals_of(i), dev) for i in ids_all]
    vo = torch.empty(bsz, dtype=torch.uint32, device=dev)
    rr = torch.empty(bsz, dtype=torch.uint8, device=dev)
    t3 = HiveTable(1024 * 32)
    # warm-up pass: maps the table's growth range and sizes the scratch once
    # (driver mapping calls cost 5-95 ms each on this system); hive_clear keeps both
    for b in range(nbat):
        t3.mixed(ops_all[b], k_all[b], v_all[b], vo, rr)
    t3.clear()
    # timed pass without the per-kernel profiling events (they add host work
    # between the launches); the profiled pass below gives the breakdown
    torch.cuda.synchronize()
    walls = []
    ev[0].record()
    for b in range(nbat):
        w0 = time.perf_counter()
        t3.mixed(ops_all[b], k_all[b], v_all[b], vo, rr)
        walls.append(time.perf_counter() - w0)
    ev[1].record()
    torch.cuda.synchronize()
    mixed_ms_noprof = ev[0].elapsed_time(ev[1])
    walls_noprof = walls
    t3.clear()
    if os.environ.get("HIVE_TRACE_CFG3"):
        os.environ["HIVE_TRACE"] = "1"
        print("[bench] cfg3 begins", file=sys.stderr, flush=True)
    t3.profile(True)
    torch.cuda.synchronize()
    walls = []
    ev[0].record()
    for b in range(nbat):
        w0 = time.perf_counter()
        t3.mixed(ops_all[b], k_all[b], v_all[b], vo, rr)
        walls.append(time.perf_counter() - w0)
    ev[1].record()
    torch.cuda.synchronize()
    os.environ.pop("HIVE_TRACE", None)
    s3 = t3.stats()
    mixed_ms = ev[0].elapsed_time(ev[1])
    p3_mixed = t3.profile_read(reset=True)          # the 64 mixed batches only
    drain_keys = [u32(gen.keys_of(np.arange(lo, lo + bsz, dtype=np.uint32)), dev) for lo in range(0, U, bsz)]
    ev[2].record()
    for dk in drain_keys:
        t3.erase(dk)
    ev[3].record()
    torch.cuda.synchronize()
    s3b = t3.stats()
    p3 = t3.profile_read(reset=True)
    res["cfg3_mixed"] = {
        "gops": nbat * bsz / (mixed_ms_noprof * 1e-3) / 1e9, "ms": mixed_ms_noprof,
        "host_wall_ms_max": 1e3 * max(walls_noprof), "host_wall_ms_sum": 1e3 * sum(walls_noprof),
        "gops_profiled": nbat * bsz / (mixed_ms * 1e-3) / 1e9, "ms_profiled": mixed_ms,
        "kern_ms": {k: round(v[0], 3) for k, v in p3_mixed.items()},
        "drain_kern_ms": {k: round(v[0], 3) for k, v in p3.items()},
        "final_buckets": s3["n_buckets"], "final_count": s3["count"], "grows": s3["grows"],
        "drain_tail_gops": U / (ev[2].elapsed_time(ev[3]) * 1e-3) / 1e9,
        "after_drain_buckets": s3b["n_buckets"], "shrinks": s3b["shrinks"],
        "merge_aborts": s3b["merge_aborts"],
        "split_ms": p3.get("k_split", (0, 0))[0], "merge_ms": p3.get("k_merge", (0, 0))[0],
        "split_launches": p3.get("k_split", (0, 0))[1], "merge_launches": p3.get("k_merge", (0, 0))[1],
    }
    # NEXT-4: the same 64 batches through the monolithic concurrent kernel
    # (hive_mixed_concurrent: one cooperative launch per batch + resize)
    tc = HiveTable(1024 * 32)
    for b in range(nbat):
        tc.mixed_concurrent(ops_all[b], k_all[b], v_all[b], vo, rr)
    tc.clear()
    torch.cuda.synchronize()
    ev[0].record()
    for b in range(nbat):
        tc.mixed_concurrent(ops_all[b], k_all[b], v_all[b], vo, rr)
    ev[1].record()
    torch.cuda.synchronize()
    conc_ms = ev[0].elapsed_time(ev[1])
    tc.clear()
    tc.profile(True)
    torch.cuda.synchronize()
    for b in range(nbat):
        tc.mixed_concurrent(ops_all[b], k_all[b], v_all[b], vo, rr)
    torch.cuda.synchronize()
    sc = tc.stats()
    pc = tc.profile_read(reset=True)
    res["cfg3_mixed_concurrent"] = {
        "gops": nbat * bsz / (conc_ms * 1e-3) / 1e9, "ms": conc_ms,
        "kern_ms": {k: round(v[0], 3) for k, v in pc.items()},
        "launches": {k: v[1] for k, v in pc.items()},
        "final_buckets": sc["n_buckets"], "final_count": sc["count"], "grows": sc["grows"],
        "vs_phased": mixed_ms_noprof / conc_ms}
    del tc
    res["cfg4_zipf"] = cfg4_zipf(dev)
    res["imbalanced_050_030_020"] = imbalanced(dev)
    return res


def imbalanced(dev):
    """The paper's imbalanced workload (§V-C.2): one mixed batch
    of n ops with insert:lookup:delete = 0.5:0.3:0.2 over ids uniform in
    [0, n), on a table that starts at 1K buckets and grows before the batch's
    insert phase (paper on an RTX 4090: ~2.6 -> 1.8 G ops/s as n grows; context,
    not a target).  PHASED hive_mixed and hive_mixed_concurrent, device time of
    the call (resize included), after a warm-up call on a cleared table."""
    import torch

    from paper_2510_15095_b200 import HiveTable, u8, u32
    out = {}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for lg in (20, 22, 24, 26):
        n = 1 << lg
        ops = u8(gen.bernoulli_ops(n, 0.5, 0.2, seed=600 + lg), dev)
        ids = gen.uniform_ids(n, n, seed=700 + lg)
        k, v = u32(gen.keys_of(ids), dev), u32(gen.vals_of(ids), dev)
        vo = torch.empty(n, dtype=torch.uint32, device=dev)
        rr = torch.empty(n, dtype=torch.uint8, device=dev)
        row = {}
        for mode in ("phased", "concurrent"):
            t = HiveTable(1024 * 32)
            run = t.mixed if mode == "phased" else t.mixed_concurrent
            best = None
            for rep in range(3):
                t.clear()
                torch.cuda.synchronize()
                ev[0].record()
                run(ops, k, v, vo, rr)
                ev[1].record()
                torch.cuda.synchronize()
                ms = ev[0].elapsed_time(ev[1])
                if rep and (best is None or ms < best):
                    best = ms
            row[mode + "_gops"] = n / (best * 1e-3) / 1e9
            del t
        out[f"2^{lg}"] = row
    return out


def cfg4_zipf(dev):
    """BASELINE config 4: 2^21 buckets, growth off, prefill
    0.90 * 2^26 keys; Z1 = 2^26 Zipf(0.99) ops over the present keys, 50%
    insert (value = op index) / 50% find, in one mixed batch; Z2 = insert 2^22
    Zipf draws over an absent universe of 0.05 * 2^26 keys (LF -> ~0.95, heavy
    in-batch duplicates, Steps 3-4)."""
    import torch

    from paper_2510_15095_b200 import HiveTable, u8, u32
    nb = 1 << 21
    n_pre = int(0.90 * (1 << 26))
    t = HiveTable(nb * 32, lf_grow=2.0, lf_shrink=0)
    pre_ids = np.arange(n_pre, dtype=np.uint32)
    pk, pv = u32(gen.keys_of(pre_ids), dev), u32(gen.vals_of(pre_ids), dev)
    n1 = 1 << 26
    r1 = gen.zipf_ranks(n1, n_pre, 0.99, seed=7)
    k1 = u32(gen.keys_of((r1 - 1).astype(np.uint32)), dev)
    ops1 = u8(np.where(np.random.default_rng(8).random(n1) < 0.5, 1, 0).astype(np.uint8), dev)
    v1 = torch.arange(n1, dtype=torch.int64, device=dev).to(torch.int32).view(torch.uint32)
    n2 = 1 << 22
    r2 = gen.zipf_ranks(n2, int(0.05 * (1 << 26)), 0.99, seed=9)
    k2 = u32(gen.keys_of((r2 - 1 + (1 << 31)).astype(np.uint32)), dev)
    v2 = v1[:n2]
    vo = torch.empty(n1, dtype=torch.uint32, device=dev)
    rr = torch.empty(n1, dtype=torch.uint8, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    out = {}
    for rep in range(2):                        # rep 0 warms up (scratch sizing)
        t.clear()
        t.insert(pk, pv)
        torch.cuda.synchronize()
        ev[0].record()
        t.mixed(ops1, k1, v1, vo, rr)
        ev[1].record()
        t.insert(k2, v2)
        ev[2].record()
        torch.cuda.synchronize()
    s = t.stats()
    hot = int((r1 == 1).sum())
    z1_ms, z2_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    # NEXT-4: Z1 through the monolithic concurrent kernel (same prefill)
    for rep in range(2):
        t.clear()
        t.insert(pk, pv)
        torch.cuda.synchronize()
        ev[0].record()
        t.mixed_concurrent(ops1, k1, v1, vo, rr)
        ev[3].record()
        torch.cuda.synchronize()
    z1c = n1 / (ev[0].elapsed_time(ev[3]) * 1e-3) / 1e9
    out = {"z1_mixed_gops": n1 / (z1_ms * 1e-3) / 1e9,
           "z2_insert_gops": n2 / (z2_ms * 1e-3) / 1e9,
           "z1_hot_key_copies": hot, "z2_distinct_keys": int(len(np.unique(r2))),
           "final_lf": s["count"] / (nb * 32), "evictions": s["evictions"], "max_depth": s["max_depth"],
           "stash_used": s["stash_used"], "leftovers": s["leftovers"], "z1_mixed_concurrent_gops": z1c}
    return out


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""MulMent hot-path benchmark (driver contract).

A STEP is one pass of the whole hot path over one batch of synthetic input:
one mm_layout call.  Default workload: BASELINE.json configs[4] (cfg5), the
largest single-GPU config: 128^3 grid graph (n = 2,097,152), dim 3, q = 0.8,
alpha = 0.01, hierarchy by heavy-edge matching, h = 2 coarse-representative
repulsion (Eq.(3)), 15 sweeps per level, then the final Eq.(1) energy.  The
step contains every §8(a) row: hierarchy build (matching, contraction, coarse
S), box init, prolongation, centroid refresh, kernels (c)/(b)/(a), fused
statistics, energy.  `value` = vertex-updates/s (sum over levels of n_l x
sweeps, summed over ranks) with inputs resident in HBM; `e2e` = the same
metric through the public API with the inputs copied from pinned host memory
and the layout + energy copied back inside the timed region.  --config cfg1..4
selects the other configs (parity-test cases / builder lines under profiles/).

Multi-GPU: the north star is one GPU with no sharding, so --gpus N runs N
independent replicas ("replicas only"); value = units of all
ranks / max-over-ranks time.

--impl reference: this build has no installable reference implementation; the
reference arm is the FP64 oracle (oracle/), timed as it stands on the host
cores on a bounded row sample of the same workload's sweep.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "vertex-updates/s per sweep and repulsion pair-interactions/s; % of FP32/HBM roofline"
UNIT = "vertex-updates/s"
SM_COUNT, FP32_LANES, SM_MAX_MHZ = 148, 128, 1965.0
FP32_PEAK_TFLOPS = SM_COUNT * FP32_LANES * 2 * SM_MAX_MHZ * 1e6 / 1e12  # 74.4, derived
MUFU_PER_CLK_SM = 16


def flop_per_pair(dim: int, q: float, coarse: bool) -> int:
    """Algorithmic FP32 flop per pair interaction, SURVEY §8(d) (FMA = 2):
    dim subtractions + dim FMA (r^2) + dim FMA (accumulation) + 1 FMUL of the
    exponent (q > 0: 2^((q+2)/2 * -lg2 r^2)) + 1 FMUL of nu (coarse).
    2-D q = 0 exact: 10; 2-D q = 0 coarse: 11; 3-D q = 0.8 coarse (cfg5): 17."""
    return 5 * dim + (1 if q != 0.0 else 0) + (1 if coarse else 0)


def mufu_per_pair(q: float) -> int:
    """MUFU (XU) ops per pair: rcp (q = 0) or lg2 + ex2 (q > 0), SURVEY §8(d)."""
    return 2 if q != 0.0 else 1


# ------------------------------------------------------------------ distributed plumbing
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a scalar (NCCL on GPU, gloo on CPU); identity for 1 rank."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [t.strip() for t in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                smax.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ workload
def load_workload(name: str):
    from workloads import configs

    return configs.make(name)


def cpu_oracle_sample(w, target_s: float = 8.0, max_rows=None):
    """Time the oracle as it stands (FP64, all host cores via OpenMP) on a
    bounded row sample of one exact sweep of the workload."""
    import numpy as np

    import oracle

    cores = oracle.default_threads()
    x = w.x0.astype(np.float64)
    rng = np.random.default_rng(0)
    calib = np.sort(rng.choice(w.n, size=min(w.n, 256 * cores), replace=False)).astype(np.int32)
    t0 = time.perf_counter()
    oracle.sweep_exact(w.S, x, w.alpha, w.q, rows=calib, nthreads=cores)
    dt = time.perf_counter() - t0
    rate = calib.shape[0] / max(dt, 1e-9)
    rows_n = int(min(w.n, max_rows or w.n, max(calib.shape[0], rate * target_s)))
    rows = np.sort(rng.choice(w.n, size=rows_n, replace=False)).astype(np.int32)
    return rows, cores


def oracle_approx_setup(w):
    """Multilevel configs: the oracle's own hierarchy (FP64 C, test infrastructure)
    and the finest level's Eq.(3) map (parent, ancestor at level h, k), with a
    seeded random state of the layout's scale."""
    import numpy as np

    import oracle
    from workloads import configs

    lv = oracle.build_hierarchy(w.graph, seed=w.seed, n_stop=1000)
    h = min(w.h, len(lv) - 1)
    anc = oracle.ancestor(lv, 0, h)
    x = configs.random_state(w.n, w.dim, seed=1, scale=w.n ** (1.0 / w.dim)).astype(np.float64)
    return lv[0].parent, anc, lv[h].n, x


def cpu_oracle_sample_approx(w, setup, target_s: float = 8.0):
    """Bounded row sample of one finest-level Eq.(3) sweep, sized from a calibration run."""
    import numpy as np

    import oracle

    parent, anc, k, x = setup
    cores = oracle.default_threads()
    rng = np.random.default_rng(0)
    calib = np.sort(rng.choice(w.n, size=min(w.n, 64 * cores), replace=False)).astype(np.int32)
    t0 = time.perf_counter()
    oracle.sweep_approx(w.S, x, w.alpha, w.q, parent, anc, k, rows=calib, nthreads=cores)
    rate = calib.shape[0] / max(time.perf_counter() - t0, 1e-9)
    rows_n = int(min(w.n, max(calib.shape[0], rate * target_s)))
    return np.sort(rng.choice(w.n, size=rows_n, replace=False)).astype(np.int32), cores


def run_reference(args):
    """--impl reference: the FP64 oracle on the host cores (rank 0 only)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    import oracle

    w = load_workload(args.config)
    if w.h == 0:
        rows, cores = cpu_oracle_sample(w, target_s=args.ref_step_s)
        x = w.x0.astype(np.float64)

        def one(r):
            oracle.sweep_exact(w.S, x, w.alpha, w.q, rows=r, nthreads=cores)

        sample = (f"{rows.shape[0]} of {w.n} rows of one exact Eq.(2) sweep of {args.config} per step "
                  f"(each row: |S_i| gathers + {w.n - 1} pair terms, FP64)")
    else:
        setup = oracle_approx_setup(w)
        rows, cores = cpu_oracle_sample_approx(w, setup, target_s=args.ref_step_s)
        parent, anc, k, x = setup

        def one(r):
            oracle.sweep_approx(w.S, x, w.alpha, w.q, parent, anc, k, rows=r, nthreads=cores)

        sample = (f"{rows.shape[0]} of {w.n} rows of one finest-level Eq.(3) sweep of {args.config} per step "
                  f"(k = {k} representatives of level {w.h}, oracle hierarchy, FP64; the centroids are "
                  f"recomputed from all n vertices in every call)")
    for _ in range(args.warmup):
        one(rows[: max(1, rows.shape[0] // 8)])
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        one(rows)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = rows.shape[0] * args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_block(w, args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "pair_interactions_per_s": value * (w.n - 1) if w.h == 0 else None}
    print(json.dumps(line), flush=True)
    return 0


def config_block(w, args):
    if getattr(args, "schedule", False):
        desc = (f"{w.name}: the paper's full optimizer MulMent_{args.h} (multilevel, alpha 1 -> x0.3 -> 0.008, "
                f"a=2, eps=1e-4, cap {args.max_final_iters} sweeps at alpha_min; n={w.n}, |S|={w.S.nnz}, q={w.q}, "
                f"dim={w.dim})")
        return {"workload": desc, "n": w.n, "nnz_S": w.S.nnz, "dim": w.dim, "q": w.q, "h": args.h,
                "schedule": "paper", "l2": "flushed (256 MB write) between timed steps; per-step CUDA events",
                "parallelism": f"replicas x{args.gpus}"}
    if w.h == 0:
        desc = (f"{w.name}: BASELINE.json configs[{int(w.name[3]) - 1 if w.name[3].isdigit() else '?'}] "
                f"(n={w.n}, |S|={w.S.nnz}, q={w.q}, alpha={w.alpha}, dim={w.dim}, {w.sweeps} exact sweeps + energy)")
    else:
        desc = (f"{w.name}: multilevel mm_layout (n={w.n}, |S|={w.S.nnz}, q={w.q}, alpha={w.alpha}, dim={w.dim}, "
                f"h={w.h}, {w.sweeps} sweeps/level, hierarchy build + prolongation + Eq.(3) sweeps + energy)")
    return {"workload": desc, "n": w.n, "nnz_S": w.S.nnz, "sweeps_per_level": w.sweeps, "dim": w.dim, "q": w.q,
            "alpha": w.alpha, "h": w.h,
            "l2": "flushed (256 MB write) between timed steps; per-step CUDA events",
            "parallelism": f"replicas x{args.gpus}"}


# ------------------------------------------------------------------ GPU arm
def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1506_04383_b200 as mm

    ws, rank, local = dist_env()
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    mm.load()
    w = load_workload(args.config)
    n, K = w.n, w.sweeps
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    with torch.cuda.stream(stream):
        S = mm.sset_to_device(w.S, dev)
        G = mm.graph_to_device(w.graph, dev) if w.h > 0 else None
        x0 = mm.coords_to_device(w.x0, dev) if w.h == 0 else None
        out = torch.empty((n, 2 if w.dim == 2 else 4), dtype=torch.float32, device=dev)

        if args.schedule:
            # the paper's full optimizer (MulMent_h): multilevel, alpha schedule, h from --h
            G = mm.graph_to_device(w.graph, dev)
            sched = mm.paper_schedule(max_final_iters=args.max_final_iters)

            def step():
                return mm.layout_schedule(G, S, w.dim, w.q, args.h, sched, w.seed, out=out)
        else:
            def step():
                return mm.layout(G, S, w.dim, w.alpha, w.q, w.h, [K], w.seed, x_init=x0, out=out)

        # warm-up; for long steps (multilevel configs, seconds each) the per-kernel
        # launch times are taken during the second warm-up step (library CUDA
        # events around every launch) instead of in an extra pass after the timed steps
        prof, prof_steps, last = None, 0, {}
        first_ms = 0.0
        for wi in range(args.warmup):
            if wi == 1 and first_ms > 1000.0:
                mm.profile_reset()
                mm.profile_enable(True)
                flush.fill_(-1.0)
                _, rep = step()
                torch.cuda.synchronize(dev)
                prof = mm.profile_read()
                last = {k: mm.profile_last(k, w.sweeps) for k in ("gather_update", "centroid")}
                mm.profile_enable(False)
                prof_steps = 1
                continue
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, rep = step()
            e1.record(stream)
            if wi == 0:
                torch.cuda.synchronize(dev)
                first_ms = e0.elapsed_time(e1)
        torch.cuda.synchronize(dev)

        # ---- timed region (device-resident inputs)
        clocks = ClockSampler(local)
        clocks.start()
        l0 = mm.launch_count()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        torch.cuda.synchronize(dev)
        for s in range(args.steps):
            flush.fill_(float(s))  # evict L2 between timed steps (outside the event pair)
            ev[s][0].record(stream)
            _, rep = step()
            ev[s][1].record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        launches = mm.launch_count() - l0
        clk = clocks.stop()
        dev_ms = sum(a.elapsed_time(b) for a, b in ev)
        ms_step = max_over_ranks(dev_ms / args.steps, dev)

        # ---- per-kernel launch times (library CUDA events around every launch) in a
        # separate pass, so that the events' overhead stays out of the timed steps
        if prof is None:
            prof_steps = args.steps if ms_step < 200 else 1
            mm.profile_reset()
            mm.profile_enable(True)
            for s in range(prof_steps):
                flush.fill_(float(s))
                step()
            torch.cuda.synchronize(dev)
            prof = mm.profile_read()
            last = {k: mm.profile_last(k, w.sweeps) for k in ("gather_update", "centroid")}
            mm.profile_enable(False)

        # ---- e2e through the public API with host buffers
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hosts = [pin(w.S.row_ptr.astype(np.int64)), pin(w.S.col.astype(np.int32)),
                 pin(w.S.d.astype(np.float32)), pin(w.S.w.astype(np.float32))]
        # exactly the arrays the timed call consumes: the graph when the hierarchy is
        # built (multilevel or --schedule), the start layout for single-level exact runs
        need_graph = w.h > 0 or args.schedule
        if need_graph:
            hosts += [pin(w.graph.row_ptr.astype(np.int64)), pin(w.graph.col.astype(np.int32))]
        else:
            hosts.append(pin(mm.coords_layout(w.x0)))
        devs = [torch.empty_like(h, device=dev) for h in hosts]
        h_out = torch.empty(tuple(out.shape), dtype=torch.float32).pin_memory()
        Se = mm.DeviceSSet(*devs[:4])
        Ge = mm.DeviceGraph(devs[4], devs[5]) if need_graph else None
        xe = None if need_graph else devs[4]
        h2d = sum(t.numel() * t.element_size() for t in hosts)
        d2h = h_out.numel() * h_out.element_size() + 3 * 8  # layout + (stress, entropy, energy)

        def e2e_step():
            for hd, dd in zip(hosts, devs):
                dd.copy_(hd, non_blocking=True)
            if args.schedule:
                y, r = mm.layout_schedule(Ge, Se, w.dim, w.q, args.h, sched, w.seed, out=out)
            else:
                y, r = mm.layout(Ge, Se, w.dim, w.alpha, w.q, w.h, [K], w.seed, x_init=xe, out=out)
            h_out.copy_(y, non_blocking=True)
            return r

        e2e_step()
        torch.cuda.synchronize(dev)
        # long steps (cfg5: seconds each): a few e2e steps bound the run time
        e2e_steps = args.steps if ms_step < 1000.0 else min(args.steps, 2)
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(e2e_steps)]
        barrier()
        for s in range(e2e_steps):
            flush.fill_(float(s))
            ev2[s][0].record(stream)
            e2e_step()
            ev2[s][1].record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev2) / e2e_steps, dev)

    units = sum_over_ranks(float(rep["vertex_updates"]), dev)
    value = units / (ms_step / 1e3)
    pairs_step = rep["pair_interactions"]
    hh = args.h if args.schedule else w.h
    kname = "repulse_exact" if hh == 0 else "repulse_coarse"
    small = False
    if hh == 0 and not args.schedule and kname not in prof and "small_level" in prof:
        # a small exact level (cfg1) runs all its sweeps in the persistent kernel
        kname, small = "small_level", True
    kern = prof.get(kname, {"launches": 0, "total_ms": float("nan")})
    k_ms = kern["total_ms"] / max(kern["launches"], 1)
    # algorithmic pairs per launch: exact n(n-1) per sweep; coarse: the
    # per-step pair count minus the exact coarsest level, averaged per launch
    if small:
        pairs_launch = n * (n - 1) * K  # one launch = the level's K sweeps
    elif hh == 0 and not args.schedule:
        pairs_launch = n * (n - 1)
    elif hh == 0:
        pairs_launch = pairs_step / max(kern["launches"] / prof_steps, 1)
    else:
        nL = rep["n_level"][-1]
        pairs_launch = (pairs_step - nL * (nL - 1) * K) / max(kern["launches"] / prof_steps, 1)
    flop_pair = flop_per_pair(w.dim, w.q, hh != 0)
    mufu_pair = mufu_per_pair(w.q)
    achieved_tflops = flop_pair * pairs_launch / (k_ms / 1e3) / 1e12
    # kernel (b) variant: the symmetric kernel evaluates every unordered pair
    # once, so it EXECUTES (flop_pair + 2 dim)/2 flop per ordered
    # pair (the j-side accumulation costs 2 dim) while the algorithmic count
    # stays flop_pair per ordered pair interaction of Eq.(2)
    sym = hh == 0 and not small and mm.exact_kernel_variant(n, w.dim) == 1
    exec_flop_pair = (flop_pair + 2 * w.dim) / 2.0 if sym else float(flop_pair)
    executed_tflops = exec_flop_pair * pairs_launch / (k_ms / 1e3) / 1e12
    pairs_s_kernel = pairs_launch / (k_ms / 1e3)
    # MUFU ceiling: 16 XU ops/clk/SM at the max SM clock; the symmetric kernel
    # executes one MUFU per UNORDERED pair, i.e. half per ordered pair
    exec_mufu_pair = mufu_pair / 2.0 if sym else float(mufu_pair)
    mufu_ceiling = SM_COUNT * MUFU_PER_CLK_SM * SM_MAX_MHZ * 1e6 / exec_mufu_pair
    fp32_meas = None
    try:
        with open(os.path.join(ROOT, "profiles", "fp32_peak.json")) as f:
            fp32_meas = json.load(f)
    except (OSError, ValueError):
        fp32_meas = None
    # HBM-bound kernels (a) and (d) at the finest level (its sweeps run last, so
    # their launches are the last `sweeps` of each kernel), against SURVEY §8(d)'s
    # algorithmic bytes: gather 4 (n+1) + 12 nnz + 3 b_x n, centroid (b_x + 4) n + b_x k
    hbm_peak, hbm_src = 6539.2, "fallback: the MEASURED_PEAKS.json value of this pool (6539.2 GB/s)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_peak, hbm_src = float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        pass
    bx = 8 if w.dim == 2 else 16
    k0 = rep["k_level"][0] if rep.get("k_level") else 0
    algo_hbm = {"gather_update": 4 * (n + 1) + 12 * w.S.nnz + 3 * bx * n, "centroid": (bx + 4) * n + bx * k0}
    roof_hbm = {"peak": hbm_peak, "unit": "GB/s", "peak_source": hbm_src, "level": 0,
                "bytes_source": "SURVEY §8(d) algorithmic bytes of the finest level per launch"}
    for kname_h, ts in last.items():
        if not ts or (kname_h == "centroid" and k0 == 0):
            continue
        med = sorted(ts)[len(ts) // 2]
        gbs = algo_hbm[kname_h] / (med * 1e-3) / 1e9
        roof_hbm[kname_h] = {"launch_ms_median": med, "launches": len(ts), "bytes_per_launch": algo_hbm[kname_h],
                             "achieved": gbs, "frac": gbs / hbm_peak}
    step_share = {k: v["total_ms"] / max(prof_steps * dev_ms / args.steps, 1e-9) for k, v in prof.items()}
    gpu_ms = sum(v["total_ms"] for v in prof.values())
    gpu_share = {k: v["total_ms"] / max(gpu_ms, 1e-9) for k, v in prof.items()}
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        if kname in tj and w.name in tj[kname].get("by_config", {}):
            traffic = tj[kname]["by_config"][w.name]
        elif kname in tj and w.name in tj[kname].get("workload", ""):
            traffic = tj[kname]["bytes"]
    except (OSError, ValueError, KeyError):
        traffic = None
    if rank != 0:
        return 0
    cpu = None
    if ws == 1 and not args.no_cpu_baseline and w.h == 0 and not args.schedule:
        import oracle

        rows, cores = cpu_oracle_sample(w, target_s=args.cpu_s)
        x64 = w.x0.astype(np.float64)
        reps, dt = 0, 0.0
        # whole sweeps finish quickly on many cores: repeat until ~cpu_s of work
        while reps == 0 or (rows.shape[0] == n and dt < 0.5 * args.cpu_s and reps < 64):
            t0 = time.perf_counter()
            oracle.sweep_exact(w.S, x64, w.alpha, w.q, rows=rows, nthreads=cores)
            dt += time.perf_counter() - t0
            reps += 1
        cpu = {"value": reps * rows.shape[0] / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{reps} x {rows.shape[0]} of {n} rows of one exact Eq.(2) sweep of {w.name} "
                         f"(FP64, OpenMP over rows), {dt:.1f} s"}
    elif ws == 1 and not args.no_cpu_baseline and not args.schedule:
        import oracle

        setup = oracle_approx_setup(w)
        rows, cores = cpu_oracle_sample_approx(w, setup, target_s=args.cpu_s)
        parent, anc, k, x = setup
        reps, dt = 0, 0.0
        while reps == 0 or (rows.shape[0] == n and dt < 0.5 * args.cpu_s and reps < 64):
            t0 = time.perf_counter()
            oracle.sweep_approx(w.S, x, w.alpha, w.q, parent, anc, k, rows=rows, nthreads=cores)
            dt += time.perf_counter() - t0
            reps += 1
        cpu = {"value": reps * rows.shape[0] / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{reps} x {rows.shape[0]} of {n} rows of one finest-level Eq.(3) sweep of {w.name} "
                         f"(k = {k}, oracle hierarchy; FP64, OpenMP over rows), {dt:.1f} s"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": config_block(w, args),
        "pair_interactions_per_s": ws * pairs_step / (ms_step / 1e3),
        "vertex_updates_per_step": rep["vertex_updates"], "pair_interactions_per_step": pairs_step,
        "roofline": {"bound": "alu", "kernel": kname, "achieved": achieved_tflops,
                     "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved_tflops / FP32_PEAK_TFLOPS,
                     "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write)",
                     "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1965 MHz (DESIGN.md §5)",
                     "flop_per_pair": flop_pair, "flop_per_pair_source": "SURVEY §8(d): 5 dim + (q>0) + coarse",
                     "pairs_per_launch": pairs_launch, "avg_launch_ms": k_ms,
                     "kernel_variant": ("persistent small-level (all sweeps in one launch; latency-bound: "
                                        "grid barriers per sweep)") if small else ("symmetric" if sym else "one-sided"),
                     # FP32 pipe utilisation: the flops the kernel EXECUTES (the symmetric kernel
                     # evaluates each unordered pair once) over the same peak
                     "executed_flop_per_pair": exec_flop_pair,
                     "executed_tflops": executed_tflops, "executed_frac": executed_tflops / FP32_PEAK_TFLOPS,
                     "executed_frac_of_measured_ffma_peak": (executed_tflops / fp32_meas["tflops"]
                                                             if fp32_meas else None),
                     "measured_ffma_peak": fp32_meas,
                     "pairs_per_s_kernel": pairs_s_kernel,
                     # the XU (MUFU) ceiling: SURVEY §8(d) counts 1 MUFU per pair at q = 0 (rcp) and 2 at
                     # q > 0 (lg2 + ex2); kernel (c) moves part of the ex2 to the FMA pipe (Q29)
                     "mufu_per_pair": mufu_pair, "mufu_ceiling_pairs_per_s": mufu_ceiling,
                     "mufu_ceiling_frac": pairs_s_kernel / mufu_ceiling},
        "roofline_hbm": roof_hbm,
        "levels": rep["n_level"], "k_levels": rep["k_level"],
        # what the timed step computed (last step's report): Eq.(1) of the final layout (coincident
        # non-S pairs, possible in FP32, are left out and counted: DESIGN.md Q6) and the last sweep's
        # relative change
        "result": {"energy": rep["energy"], "stress": rep["stress"], "entropy": rep["entropy"],
                   "coincident_pairs": rep["coincident_pairs"], "rel_change": rep["rel_change"]},
        "kernel_share_of_step": step_share,
        "kernel_share_of_gpu_time": gpu_share,
        "kernels": prof,
        "cpu_baseline": cpu,
        "e2e": {"value": units / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms, "steps": e2e_steps,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clk,
        "energy_last_step": rep["energy"],
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mm", choices=["mm", "reference"])
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--cpu-s", type=float, default=10.0)
    ap.add_argument("--ref-step-s", type=float, default=6.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--schedule", action="store_true",
                    help="time the paper's full optimizer (alpha schedule, multilevel MulMent_h) instead")
    ap.add_argument("--h", type=int, default=0, help="approximation depth for --schedule (0 = MulMent_0)")
    ap.add_argument("--max-final-iters", type=int, default=200)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "mm":
        print("warning: the contract asks for >= 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())

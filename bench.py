#!/usr/bin/env python
"""bench.py -- TC-MIS on B200: MIS time and Gedges/s (BASELINE.json metric).

A "step" is one complete MIS solve (H2 priorities -> bulk-synchronous rounds
-> ascending MIS ids back on the host) of the configured synthetic graph.

  value  the CSR is already in HBM (generated there); the step is
         tcmis_solve() through the C-ABI up to the ascending MIS ids in a
         pinned host buffer (SURVEY 8(d) "MIS time": priority init through
         the MIS ids back on host), timed with CUDA events on the engine's
         stream; L2 is flushed between steps.  `device_resident` times the
         same solve with the ids left in HBM (tcmis_solve_device).
  e2e    the drop-in path: host CSR in pinned memory -> tcmis_graph_upload
         (H2D) -> tcmis_graph_tile -> tcmis_solve (D2H of the MIS ids and the
         per-iteration stats into host buffers) -> destroy, every step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config rmat22]
  python bench.py --impl reference ...   (the reference CPU implementation)

Configs (BASELINE.json): er (n=100k, d=16), grid (4096^2), rmat22 (default at
N = 1, the metric's headline), rgg (24M, d~3), rmat26 (~1.05B edges; default
at N > 1).

N > 1 (torchrun, one rank per GPU): the north-star's row-partitioned solve
(paper_2605_29604_b200/distributed.py): every rank generates the
graph on its GPU, keeps its edge-balanced row range, and the ranks run the
bulk-synchronous rounds with NCCL all-gathers of the candidate / removal
bitmaps and an all-reduce of the round counters.  One step = one solve of the
WHOLE graph by all ranks together ("scaling": "strong"); the time is the max
over ranks of CUDA-event time on each rank's engine stream.  Rank 0 also
solves the same graph alone on its GPU before partitioning
("single_gpu_same_graph"), so the line carries its own 1-GPU denominator.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "er": {"workload": "Erdos-Renyi n=100000 avg degree 16 (gnp_graph_avg_degree seed 1)"},
    "grid": {"workload": "2D 5-point grid 4096x4096 (row-major ids)"},
    "rmat22": {"workload": "R-MAT scale 22 edge factor 16 (rmat_graph(22,16,1))"},
    "rgg": {"workload": "random geometric graph n=24M avg degree ~3 (integer lattice, ids in "
                        "draw order)"},
    "rmat26": {"workload": "R-MAT scale 26 edge factor 16 (rmat_graph(26,16,1))"},
    # not a BASELINE config: the RGG with its ids in the generator's spatial
    # (Z-order) order, for the tile-format experiments (8.4 nnz / 16x16 tile)
    "rgg_spatial_ids": {"workload": "random geometric graph n=24M avg degree ~3, ids in "
                                    "spatial Z-order (tcmis_graph_permuted)"},
}
HEUR = {"h1": 0, "h2": 1, "h3": 2, "luby-fresh": 3, "luby-perm": 4}
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML in a
    1 ms polling thread (nvidia-smi's 100 ms floor misses a ~5 ms region);
    nvidia-smi as a fallback."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.nvml = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        time.sleep(0.02)
        return self

    def _poll(self):
        N = self.nvml
        while not self.stop.is_set():
            if N is not None:
                try:
                    sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                    r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.rows.append((sm, r))
                except Exception:
                    pass
                time.sleep(0.001)
            else:
                try:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.index),
                         "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip().split(",")
                    self.max_sm = float(out[1])
                    self.rows.append((float(out[0]), int(out[2], 16)))
                except Exception:
                    return

    def __exit__(self, *exc):
        time.sleep(0.01)
        self.stop.set()
        self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(r[0] for r in self.rows)
        bits = 0
        for r in self.rows:
            bits |= int(r[1])
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                 0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}
        reasons = sorted(v for k, v in names.items() if bits & k and k != 0x1)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": getattr(self, "max_sm", None),
                "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self.nvml else "nvidia-smi"}


# --------------------------------------------------------------- graphs

def make_device_graph(tc, name: str, ctx):
    if name == "er":
        return tc.DeviceGraph.gnp(100000, 16.0, 1, ctx)  # = gnp_graph_avg_degree(100000, 16, 1)
    if name == "grid":
        return tc.DeviceGraph.grid(4096, ctx)
    if name == "rmat22":
        return tc.DeviceGraph.rmat(22, 16, 1, ctx)
    if name == "rgg":
        return tc.DeviceGraph.rgg(24_000_000, 3.0, 1, ctx)
    if name == "rmat26":
        return tc.DeviceGraph.rmat(26, 16, 1, ctx)
    if name == "rgg_spatial_ids":
        g = tc.DeviceGraph.rgg(24_000_000, 3.0, 1, ctx).reorder(tc.DeviceGraph.ORDER_SPATIAL)
        p = g.permuted()
        g.close()
        return p
    raise ValueError(name)


def peaks():
    try:
        with open(PEAKS) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------ the B200 arm

def run_ours(args) -> dict:
    import torch
    import paper_2605_29604_b200 as tc

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.partitioned:
        return run_partitioned(args, rank, world, local)
    dist = None
    torch.cuda.set_device(local)
    ctx = tc.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{local}")
    L = tc.load()

    t0 = time.time()
    dg = make_device_graph(tc, args.config, ctx)
    n, nnz = dg.n, dg.nnz
    m = nnz // 2
    tiles = dg.tile(16)
    log(f"[bench] {args.config}: n={n} m={m} tiles={tiles} (setup {time.time() - t0:.1f}s)")
    order_ms = None
    if args.order == "auto":
        # measured per config (tools/gpu_order.sh, tools/gpu_cb.sh,
        # tools/gpu_order2.sh): the spatial order takes
        # RGG 24M 1.10 -> 0.95 ms, and since k_tail uses the degree-class bounds
        # the degree order (ties in the points' spatial order) beats it, 0.991
        # -> 0.953 ms; the degree order with sorted rows and the degree-class
        # bounds takes R-MAT s22 0.357 -> 0.256 ms and s26 3.82 -> 1.77 ms;
        # ER / grid gain nothing (ER 0.135 -> 0.155 ms, grid 0.686 -> 0.789)
        args.order = {"rgg": "degree", "rmat22": "degree",
                      "rmat26": "degree"}.get(args.config, "none")
    if args.order != "none":
        # an internal vertex order for the solve kernels (tcmis_graph_reorder):
        # graph preparation like the tiling, outside the timed region, results
        # in the graph's own ids; its one-off cost is reported
        ctx.synchronize()
        t_o = time.perf_counter()
        dg.reorder({"degree": tc.DeviceGraph.ORDER_DEGREE,
                    "spatial": tc.DeviceGraph.ORDER_SPATIAL}[args.order])
        ctx.synchronize()
        order_ms = round((time.perf_counter() - t_o) * 1e3, 3)
        log(f"[bench] vertex order {args.order}: {order_ms} ms")
    excl = {"auto": tc.Exclusion.AUTO, "push": tc.Exclusion.PUSH,
            "pull": tc.Exclusion.CSR_PULL, "tile-bits": tc.Exclusion.TILE_BITS,
            "tile-mma": tc.Exclusion.TILE_MMA}[args.exclusion]
    cand_flags = {"csr": 0, "tile": tc.F_TILE_CAND,
                  "tile-umma": tc.F_TILE_CAND | tc.F_TILE_UMMA}[args.candidates]
    cfg = tc.EngineConfig(heuristic=HEUR[args.heuristic], seed=1, tile_dim=16, exclusion=excl,
                          flags=cand_flags)
    tile_cand_build = None
    if cand_flags:  # A-up store: per priority configuration, outside the timed region
        ms_b, up_tiles = dg.tile_cand_prepare(cfg)
        tile_cand_build = {"ms": round(ms_b, 3), "a_up_tiles": up_tiles}
    c_cfg, _keep = cfg._c()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")  # > 126 MB L2

    d_stats = (tc._Stats * 4096)()  # allocated once, like solve_host's (10 us per ctypes array)

    def solve_device():
        d_mis = C.c_void_p()
        cnt = C.c_int64(0)
        nit = C.c_int32(0)
        tc._check(L.tcmis_solve_device(dg.h, C.byref(c_cfg), C.byref(d_mis), C.byref(cnt),
                                       None, d_stats, 4096, C.byref(nit)))
        return cnt.value, nit.value

    h_mis = torch.empty(max(n, 1), dtype=torch.int32).pin_memory()  # the step's result buffer
    h_stats = (tc._Stats * 4096)()

    def solve_host():
        cnt, nit = C.c_int64(0), C.c_int32(0)
        tc._check(L.tcmis_solve(dg.h, C.byref(c_cfg), None, C.c_void_p(h_mis.data_ptr()),
                                C.byref(cnt), h_stats, 4096, C.byref(nit)))
        return cnt.value, nit.value

    def timed(fn, steps):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        torch.cuda.synchronize()
        out = None
        for k in range(steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                ev[k][0].record(stream)
            out = fn()
            with torch.cuda.stream(stream):
                ev[k][1].record(stream)
        ctx.synchronize()
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in ev], out

    # ---- value: solves up to the MIS ids in pinned host memory
    for _ in range(args.warmup):
        solve_host()
        solve_device()
    ctx.synchronize()
    if dist:
        dist.barrier()
    launches0 = ctx.launches()
    with ClockSampler(local) as clk:
        step_ms, (mis_count, iters) = timed(solve_host, args.steps)
    launches = ctx.launches() - launches0
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * m / (ms_per_step * 1e-3) / 1e9  # replicas: every rank solves its graph
    assert int(h_mis[:mis_count].diff().min()) > 0 if mis_count > 1 else True
    # the same solve with the ids left in HBM (what the kernels alone take)
    dev_ms, _ = timed(solve_device, args.steps)
    dev_ms = sorted(dev_ms)[len(dev_ms) // 2]
    device_resident = {"ms": round(dev_ms, 4), "value": round(m / (dev_ms * 1e-3) / 1e9, 4),
                       "d2h_ms": round(ms_per_step - dev_ms, 4),
                       "note": "median step of tcmis_solve_device (MIS ids stay in HBM); "
                               "d2h_ms = value's step minus this (the 4|MIS|-byte id copy "
                               "over PCIe and its synchronisation)"}

    # ---- kernel roofline: per-kernel CUDA events around every launch of a
    # step-wise solve (same kernels as the graph; TCMIS_F_TIMING)
    cfg_t = tc.EngineConfig(heuristic=HEUR[args.heuristic], seed=1, tile_dim=16, timing=True,
                            exclusion=excl, flags=cand_flags)
    runs = []
    for _ in range(max(3, min(args.steps, 5))):
        tc.run_mis(dg, cfg_t)
        runs.append(timeline(tc, ctx))
    kern = {}
    for tl in runs:
        for name, rnd, ms in tl:
            kern.setdefault((name, rnd), []).append(ms)
    kernels = sorted(((k[0], k[1], sum(v) / len(v)) for k, v in kern.items()),
                     key=lambda x: -x[2])
    roofline = kernel_roofline(tc, dg, cfg, kernels, args, ms_per_step)
    # ---- the reference user's own call: tcmis::run_mis on std::vector storage
    # (first: the pinned e2e below leaves ~0.6 GB of pinned host memory in
    # torch's host cache, which slowed the pageable path's host copies)
    cpp = None
    if not args.no_e2e and rank == 0 and world == 1 and args.exclusion == "auto" \
            and args.candidates == "csr":
        cpp = run_cpp_dropin(dg, args, mis_count)
    # ---- e2e through the drop-in C-ABI with host buffers
    e2e = None if args.no_e2e else run_e2e(tc, torch, dg, ctx, stream, cfg, args, local, dist,
                                            flush)
    if e2e is not None and cpp is not None:
        e2e["cpp_dropin_pageable"] = cpp

    line = {
        "metric": "Gedges/s (MIS solve, BASELINE config)", "value": round(value, 4),
        "unit": "Gedges/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64/u32 keys (integer), f64 priority",
        "data": "synthetic (generated on device, bit-identical to the reference generator)",
        "config": {"workload": CONFIGS[args.config]["workload"], "graph": args.config,
                   "n": n, "m": m, "heuristic": args.heuristic, "seed": 1, "tile_dim": 16,
                   "iterations": iters, "mis_size": mis_count, "tiles_t16": tiles,
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2": "256 MB flush between steps; CSR > L2",
                   "vertex_order": args.order, "vertex_order_ms": order_ms,
                   "candidates": args.candidates, "exclusion": args.exclusion,
                   "tile_cand_build": tile_cand_build},
        "mis_ms": round(ms_per_step, 4),
        "device_resident": device_resident,
        "kernels_ms": [[k, r, round(ms, 4)] for k, r, ms in kernels],
        "roofline": roofline, "e2e": e2e, "clocks": clk.summary(),
        "gpu_launches": launches,
    }
    if rank == 0 and not args.no_k1:
        try:
            line["k1_tile_conversion"] = k1_timing(tc, dg, ctx)
            ref = {"rmat22": 47302.1}.get(args.config)
            if ref:
                line["k1_tile_conversion"]["reference_tile_graph_ms"] = ref
                line["k1_tile_conversion"]["reference_source"] = (
                    "tests/golden/rmat22_ef16.json tile_graph_ms (the reference's serial "
                    "tile_graph, tiling.cpp:44-84)")
        except Exception as e:
            line["k1_tile_conversion"] = {"error": str(e)[:200]}
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(dg, args)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return line if rank == 0 else None


def timeline(tc, ctx):
    """[(kernel, round, ms)] of the context's last TCMIS_F_TIMING solve."""
    L = tc.load()

    class KT(C.Structure):
        _fields_ = [("name", C.c_char * 32), ("round", C.c_int32), ("ms", C.c_float)]
    L.tcmis_ctx_timeline.restype = C.c_int32
    L.tcmis_ctx_timeline.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
    n = L.tcmis_ctx_timeline(ctx.h, None, 0)
    buf = (KT * max(n, 1))()
    L.tcmis_ctx_timeline(ctx.h, buf, n)
    return [(buf[i].name.decode(), int(buf[i].round), float(buf[i].ms)) for i in range(n)]


# kernel -> phase of the reference's round (engine.cpp:247-291); k_round_end
# also scans the pull exclusion's longest rows but is booked as Phase 3
PHASE = {"k_probe_select": 1, "k_select": 1, "k_select_long": 1,
         "k_probe_pull": 2, "k_update_pull": 2, "k_tile_excl_bits": 2, "k_tile_excl_mma": 2,
         "k_update": 3, "k_round_end": 3, "k_priorities": 0, "k_tail": 4,
         "k_prio_settle": 0, "k_r1_pull": 2,
         "k_alive_bits": 1, "k_tile_cand_bits": 1, "k_tile_cand_umma": 1, "k_tile_mark": 1}
PHASE_NAME = {0: "init (priorities, states; on the degree order also round 1's class-bound verdicts)", 1: "Phase 1 candidate detection",
              2: "Phase 2 neighbour exclusion (SpMV)", 3: "Phase 3 state update + compaction",
              12: "Phases 1+2 (push exclusion fused into candidate detection)",
              4: "Tail rounds (Phases 1-3 of every remaining round in one persistent kernel, "
                 "+ MIS id compaction)"}


def kernel_roofline(tc, dg, cfg, kernels, args, ms_per_step):
    """Roofline of the dominant phase-round, SURVEY 8(d) algorithmic bytes.

    The unit of one "launch" is the kernel sequence of one phase in one round
    (the kernels split the phase's vertices between a straight-line probe and
    the scan engines, so no single kernel owns a unit).  Bytes per unit
    (format-independent): init 13 n; Phase 1 12 |A_k| + 4 nnz(A_k);
    Phase 2 8 |A_k \\ C_k| + 4 nnz(A_k \\ C_k); Phase 3 2 |A_k|, from the
    round's own trajectory (observer snapshots, outside the timed region).
    Time = the mean CUDA-event duration of those kernels.  Early exit means the
    kernels read fewer bytes than the algorithm's: `traffic` (ncu DRAM bytes,
    profiles/ncu_summary.json) shows what they actually moved."""
    import numpy as np
    hbm, peak_kind = peaks()
    traj = trajectory_terms(tc, dg, cfg)
    n = dg.n
    push = not any(k in ("k_probe_pull", "k_update_pull", "k_tile_excl_bits", "k_tile_excl_mma")
                   for k, _, _ in kernels)
    acc = {}
    for name, rnd, ms in kernels:
        ph = PHASE.get(name)
        if ph is None:
            continue
        if push and ph in (1, 2):
            ph = 12
        key = (ph, rnd if ph else 0)  # k_tail: rnd = its first round
        e = acc.setdefault(key, {"ms": 0.0, "kernels": []})
        e["ms"] += ms
        e["kernels"].append(name)
    phases = []
    for (ph, rnd), e in sorted(acc.items()):
        if ph == 0:
            b = 13 * n
        else:
            if rnd < 1 or rnd > len(traj):
                continue
            A, nnzA, NC, nnzNC = traj[rnd - 1]
            b1, b2, b3 = 12 * A + 4 * nnzA, 8 * NC + 4 * nnzNC, 2 * A
            if ph == 4:  # every round from rnd on, all three phases
                b = sum(12 * A + 4 * nA + 8 * NC + 4 * nNC + 2 * A
                        for A, nA, NC, nNC in traj[rnd - 1:])
            else:
                b = {1: b1, 2: b2, 3: b3, 12: b1 + b2}[ph]
        ach = b / (e["ms"] * 1e-3) / 1e9 if e["ms"] > 0 else 0.0
        phases.append({"phase": PHASE_NAME[ph], "round": rnd if ph != 4 else f"{rnd}-{len(traj)}",
                       "kernels": e["kernels"],
                       "algorithmic_bytes": int(b), "ms": round(e["ms"], 4),
                       "achieved": round(ach, 1), "frac": round(ach / hbm, 4)})
    if not phases:
        return None
    # the dominant phase-round by time (the tail counts as one: it is one
    # launch over all the late rounds)
    dom = max(phases, key=lambda p: p["ms"])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            summ = json.load(f).get(args.config, {})
        parts = [summ[k]["dram_bytes"] for k in dom["kernels"] if k in summ]
        if parts and len(parts) == len(dom["kernels"]):
            traffic = int(sum(parts))
    except Exception:
        traffic = None
    total_b = 13 * n + sum(12 * A + 4 * nnzA + 8 * NC + 4 * nnzNC + 2 * A
                           for A, nnzA, NC, nnzNC in traj)
    solve_ach = total_b / (ms_per_step * 1e-3) / 1e9
    # the second fraction: what the kernels actually moved (ncu DRAM bytes of
    # the same launches) over the same time -- early exit makes the
    # algorithmic fraction above overstate the streaming rate
    traffic_frac = (round(traffic / (dom["ms"] * 1e-3) / 1e9 / hbm, 4)
                    if traffic and dom["ms"] > 0 else None)
    return {"kernel": f"{dom['phase']}, round {dom['round']}: " + " + ".join(dom["kernels"]),
            "bound": "hbm", "achieved": dom["achieved"], "peak": hbm, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": dom["frac"], "traffic": traffic,
            "traffic_frac": traffic_frac,
            "algorithmic_bytes": dom["algorithmic_bytes"], "launch_ms": dom["ms"],
            "share_of_step": round(dom["ms"] / ms_per_step, 4),
            "definition": "SURVEY 8(d) algorithmic bytes of the phase-round / summed CUDA-event "
                          "time of its kernels (step-wise timing solve); traffic = ncu DRAM "
                          "bytes of the same kernels (profiles/ncu_summary.json); traffic_frac "
                          "= traffic / the same time / peak",
            "phases": phases,
            "solve": {"algorithmic_bytes": int(total_b), "ms": round(ms_per_step, 4),
                      "achieved": round(solve_ach, 1), "frac": round(solve_ach / hbm, 4)}}


def trajectory_terms(tc, dg, cfg):
    """|A_k|, nnz(A_k), |A_k \\ C_k|, nnz(A_k \\ C_k) per round, from the
    device (observer snapshots + degrees); outside every timed region."""
    import numpy as np
    h = dg.download()
    deg = np.diff(h.offsets)
    out = []

    def obs(it, cand, states):
        alive = states == 0
        c = cand.astype(bool)
        nc = alive & ~c
        out.append((int(alive.sum()), int(deg[alive].sum()), int(nc.sum()), int(deg[nc].sum())))

    c2 = tc.EngineConfig(heuristic=cfg.heuristic, seed=cfg.seed, tile_dim=cfg.tile_dim,
                         iteration_observer=obs)
    if c2.heuristic == tc.Heuristic.H3:
        c2.heuristic = tc.Heuristic.H2  # same rounds inside
    tc.run_mis(dg, c2)
    return out


def run_e2e(tc, torch, dg, ctx, stream, cfg, args, local, dist, flush):
    import numpy as np
    L = tc.load()
    h = dg.download()
    n, nnz = h.n, h.neighbors.size
    off = torch.from_numpy(h.offsets).pin_memory()
    nbr = torch.from_numpy(h.neighbors).pin_memory()
    mis = torch.empty(max(n, 1), dtype=torch.int32).pin_memory()
    c_cfg, _k = cfg._c()
    stats = (tc._Stats * 4096)()

    def step():
        g = C.c_void_p()
        tc._check(L.tcmis_graph_upload_tiled(ctx.h, n, C.c_void_p(off.data_ptr()),
                                             C.c_void_p(nbr.data_ptr()), 16, C.byref(g), None))
        cnt, nit = C.c_int64(0), C.c_int32(0)
        tc._check(L.tcmis_solve(g, C.byref(c_cfg), None, C.c_void_p(mis.data_ptr()),
                                C.byref(cnt), stats, 4096, C.byref(nit)))
        L.tcmis_graph_destroy(g)
        return cnt.value

    for _ in range(max(1, min(args.warmup, 3))):
        step()
    steps = max(1, min(args.steps, 10))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    cnt = 0
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            evs[k][0].record(stream)
        cnt = step()
        with torch.cuda.stream(stream):
            evs[k][1].record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    world = dist.get_world_size() if dist else 1
    # one untimed pass with a host-clock split of the four calls (each call
    # returns only after its stream work is done)
    parts = {}
    t0 = time.perf_counter()
    g = C.c_void_p()
    tc._check(L.tcmis_graph_upload_tiled(ctx.h, n, C.c_void_p(off.data_ptr()),
                                         C.c_void_p(nbr.data_ptr()), 16, C.byref(g), None))
    t2 = time.perf_counter()
    cnt2, nit = C.c_int64(0), C.c_int32(0)
    tc._check(L.tcmis_solve(g, C.byref(c_cfg), None, C.c_void_p(mis.data_ptr()),
                            C.byref(cnt2), stats, 4096, C.byref(nit)))
    t3 = time.perf_counter()
    L.tcmis_graph_destroy(g)
    ctx.synchronize()
    t4 = time.perf_counter()
    # the same upload without the tile count, and the count alone after it:
    # what the overlap hides
    g = C.c_void_p()
    t5 = time.perf_counter()
    tc._check(L.tcmis_graph_upload(ctx.h, n, C.c_void_p(off.data_ptr()),
                                   C.c_void_p(nbr.data_ptr()), C.byref(g)))
    t6 = time.perf_counter()
    tc._check(L.tcmis_graph_tile(g, 16, None))
    t7 = time.perf_counter()
    L.tcmis_graph_destroy(g)
    ctx.synchronize()
    parts = {"upload_and_tile": round((t2 - t0) * 1e3, 3), "solve": round((t3 - t2) * 1e3, 3),
             "destroy": round((t4 - t3) * 1e3, 3),
             "upload_alone": round((t6 - t5) * 1e3, 3), "tile_alone": round((t7 - t6) * 1e3, 3)}
    return {"value": round(world * (nnz // 2) / (ms * 1e-3) / 1e9, 4), "unit": "Gedges/s",
            "breakdown_ms": parts,
            "ms": round(ms, 3), "h2d_bytes_per_step": int(8 * (n + 1) + 4 * nnz),
            "d2h_bytes_per_step": int(4 * cnt + 64 * 4096), "steps": steps,
            "path": "tcmis_graph_upload_tiled (upload with the K1 tile count overlapped) + "
                    "tcmis_solve (host buffers)"}


def k1_timing(tc, dg, ctx, reps: int = 3) -> dict:
    """The CSR -> tile converter (tile_graph, tiling.cpp:44-84, K1) on the
    device, each part on a fresh handle over the same device CSR
    (tcmis_graph_wrap_device: no cached tiling), wall clock around the
    synchronous call, median of `reps`:
      * count: the tile counts per block row the solve's counters use;
      * compact store: the T = 16 store of the tile-form kernels (36 B/tile);
      * reference layout: the full TiledAdjacency (136 B/tile: 16 u64 rows +
        row / column) built on the device and copied to host memory.
    Bytes: CSR read (8 B/row + 4 B/entry) + tile bytes written; the roofline
    fraction is against the HBM peak (the export also crosses PCIe)."""
    import numpy as np
    L = tc.load()
    hbm, _ = peaks()
    n, nnz = dg.n, dg.nnz
    csr_b = 8 * (n + 1) + 4 * nnz
    d_off, d_nbr = dg.device_offsets, dg.device_neighbors

    def fresh():
        h = C.c_void_p()
        tc._check(L.tcmis_graph_wrap_device(ctx.h, n, nnz, C.c_void_p(d_off), C.c_void_p(d_nbr),
                                            C.byref(h)))
        return h

    def timed(fn):
        ts = []
        for _ in range(reps):
            h = fresh()
            ctx.synchronize()
            t0 = time.perf_counter()
            out = fn(h)
            t1 = time.perf_counter()
            L.tcmis_graph_destroy(h)
            ts.append((t1 - t0) * 1e3)
        return sorted(ts)[len(ts) // 2], out

    cnt = C.c_int64(0)
    ms_count, _ = timed(lambda h: tc._check(L.tcmis_graph_tile(h, 16, C.byref(cnt))))
    tiles = int(cnt.value)
    st_cnt = C.c_int64(0)
    ms_store, _ = timed(lambda h: tc._check(L.tcmis_graph_tile_store(h, 16, C.byref(st_cnt), None,
                                                                    None, None)))
    out = {"tiles_t16": tiles,
           "count": {"ms": round(ms_count, 3), "bytes": csr_b,
                     "gbs": round(csr_b / (ms_count * 1e-3) / 1e9, 1),
                     "frac": round(csr_b / (ms_count * 1e-3) / 1e9 / hbm, 4)},
           "compact_store": {"ms": round(ms_store, 3), "bytes": csr_b + 36 * tiles,
                             "gbs": round((csr_b + 36 * tiles) / (ms_store * 1e-3) / 1e9, 1),
                             "frac": round((csr_b + 36 * tiles) / (ms_store * 1e-3) / 1e9 / hbm, 4)}}
    ref_bytes = 136 * tiles
    try:
        import psutil
        room = psutil.virtual_memory().available
    except Exception:
        room = 0
    if room > 3 * ref_bytes:
        nb = (n + 15) // 16
        tr = np.empty(max(tiles, 1), np.int32)
        tcol = np.empty(max(tiles, 1), np.int32)
        rb = np.empty(max(tiles * 16, 1), np.uint64)
        bro = np.empty(nb + 1, np.int64)
        tr[:] = 0  # fault the pages in outside the timed call
        tcol[:] = 0
        rb[:] = 0
        ms_exp, _ = timed(lambda h: tc._check(L.tcmis_graph_export_tiles(
            h, 16, tc._ptr(tr), tc._ptr(tcol), tc._ptr(rb), tc._ptr(bro))))
        out["reference_layout"] = {"ms": round(ms_exp, 3), "bytes_written": ref_bytes,
                                   "gbs": round(ref_bytes / (ms_exp * 1e-3) / 1e9, 1),
                                   "note": "device merge + copy of the tiles to host memory"}
        del tr, tcol, rb, bro
    else:
        out["reference_layout"] = {"skipped": f"needs {3 * ref_bytes >> 30} GB of host memory"}
    return out


def run_cpp_dropin(dg, args, want_mis: int) -> dict | None:
    """tests/cpp/e2e_main.cpp: a C++ program written against the reference's
    headers times tcmis::run_mis(const Graph &, cfg) with the Graph in plain
    std::vector (pageable) memory -- upload (pinned staging ring + host copy
    threads, csrc/staging.cu), tile count, solve, MIS ids back into a
    std::vector.  Wall clock around each call, median of 5 after a warm-up."""
    import subprocess
    import tempfile
    import numpy as np
    h = dg.download()
    d = tempfile.mkdtemp(prefix="tcmis_e2e_")
    path, exe = os.path.join(d, "g.bin"), os.path.join(d, "e2e")
    pkg = os.path.join(ROOT, "paper_2605_29604_b200")
    try:
        with open(path, "wb") as f:
            f.write(np.int32(h.n).tobytes())
            f.write(np.int64(h.neighbors.size).tobytes())
            f.write(h.offsets.astype(np.int64).tobytes())
            f.write(h.neighbors.astype(np.int32).tobytes())
        del h
        subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "e2e_main.cpp"), "-L", pkg, "-ltcmis",
                        "-ltcmis_b200", f"-Wl,-rpath,{pkg}", "-o", exe], check=True)
        out = subprocess.run([exe, path, "5", args.heuristic], capture_output=True, text=True,
                             check=True, timeout=600).stdout
        r = json.loads(out.strip().splitlines()[-1])
    except Exception as e:  # reported, not fatal: the device line stands
        log(f"[bench] C++ drop-in e2e failed: {e}")
        return {"error": str(e)[:200]}
    finally:
        for p in (path, exe):
            if os.path.exists(p):
                os.remove(p)
        os.rmdir(d)
    m = r["m"]
    return {"value": round(m / (r["median_ms"] * 1e-3) / 1e9, 4), "unit": "Gedges/s",
            "ms": r["median_ms"], "ms_all": r["ms"], "mis_size": r["mis_size"],
            "capi_breakdown_ms": r.get("capi_breakdown_ms"),
            "matches_device_solve": r["mis_size"] == want_mis,
            "path": "tcmis::run_mis(const Graph &, cfg) from tests/cpp/e2e_main.cpp, Graph in "
                    "std::vector (pageable) storage, wall clock per call"}


# ------------------------------------------- N > 1: row-partitioned solve

def run_partitioned(args, rank: int, world: int, local: int) -> dict | None:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_29604_b200 as tc
    from paper_2605_29604_b200 import distributed as D

    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev  # one GPU per rank; ranks share a GPU only in emulation runs
    torch.cuda.set_device(dev)
    device = f"cuda:{dev}"
    for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29533"), ("RANK", str(rank)),
                 ("WORLD_SIZE", str(world))):
        os.environ.setdefault(k, v)  # --partitioned at N = 1 without torchrun
    dist.init_process_group(args.dist_backend)
    ctx = tc.Context(dev)
    L = tc.load()
    t0 = time.time()
    full = make_device_graph(tc, args.config, ctx)
    n, nnz = full.n, full.nnz
    m = nnz // 2
    off = np.zeros(n + 1, np.int64)
    tc._check(L.tcmis_graph_download(full.h, tc._ptr(off), None))
    rank_lo = D.partition_rows(off, world, 16)
    log(f"[bench:rank{rank}] {args.config}: n={n} m={m} rows [{rank_lo[rank]}, "
        f"{rank_lo[rank + 1]}) (setup {time.time() - t0:.1f}s)")
    single = None
    solve_bytes = None
    if rank == 0 and not args.no_single:
        # the same graph solved by one GPU (this rank's, alone), device-resident,
        # timed exactly like the N = 1 line (tcmis_solve_device, CUDA events)
        cfg1 = tc.EngineConfig(heuristic=HEUR[args.heuristic], seed=1, tile_dim=16)
        c1, _k1 = cfg1._c()
        full.tile(16)
        stats = (tc._Stats * 4096)()

        def solve1():
            d_mis, d_state = C.c_void_p(), C.c_void_p()
            cnt, nit = C.c_int64(0), C.c_int32(0)
            tc._check(L.tcmis_solve_device(full.h, C.byref(c1), C.byref(d_mis), C.byref(cnt),
                                           None, stats, 4096, C.byref(nit)))
            return cnt.value, nit.value

        for _ in range(3):
            solve1()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st1 = torch.cuda.ExternalStream(ctx.stream, device=device)
        ms1 = []
        for _ in range(5):
            with torch.cuda.stream(st1):
                e0.record(st1)
            cnt1, nit1 = solve1()
            with torch.cuda.stream(st1):
                e1.record(st1)
            torch.cuda.synchronize()
            ms1.append(e0.elapsed_time(e1))
        med = sorted(ms1)[len(ms1) // 2]
        single = {"ms": round(med, 4), "value": round(m / (med * 1e-3) / 1e9, 4),
                  "iterations": nit1, "mis_size": cnt1,
                  "note": "rank 0 alone, before partitioning; median of 5 device-resident solves"}
        # SURVEY 8(d) algorithmic bytes of the whole solve, from the trajectory
        # (identical for every world size), outside every timed region
        traj = trajectory_terms(tc, full, cfg1)
        solve_bytes = 13 * n + sum(12 * A + 4 * nA + 8 * NC + 4 * nNC + 2 * A
                                   for A, nA, NC, nNC in traj)
    me = D.GpuRank(ctx, n, rank_lo[rank], rank_lo[rank + 1], None, None, device, full=full)
    full.close()
    stream = torch.cuda.ExternalStream(ctx.stream, device=device)
    # the native driver (tcmis_solve_partitioned: every round one CUDA graph over
    # NCCL, driven from C++) needs one GPU per rank; the gloo emulation runs
    # (ranks sharing a GPU) take the step-wise Python driver
    native = args.dist_backend == "nccl" and args.dist_driver == "native"
    xch = D.Exchange.nccl(ctx, world, rank, dist) if native else None
    own_n = rank_lo[rank + 1] - rank_lo[rank]
    mis_buf = torch.empty(max(own_n, 1), dtype=torch.int32).pin_memory().numpy()

    def solve():
        if native:
            # this rank's MIS ids land in pinned host memory (the N = 1 value's
            # definition: the ids back on the host), each rank its own rows
            return D.solve_native(me.g, xch, rank_lo, heuristic=args.heuristic, seed=1,
                                  tile_dim=16, want_state=False, own_range=True,
                                  mis_out=mis_buf)
        return D.solve_partitioned(me, rank_lo, rank, world, dist, heuristic=args.heuristic,
                                   seed=1, tile_dim=16)

    def mis_of(res):
        return int(res.mis.size) if native else int((res.own_state == 1).sum())

    for _ in range(args.warmup):
        res = solve()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches()
    with ClockSampler(dev) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                ev[k][0].record(stream)
            res = solve()
            with torch.cuda.stream(stream):
                ev[k][1].record(stream)
        torch.cuda.synchronize()
    launches = ctx.launches() - launches0
    tdev = device if args.dist_backend == "nccl" else "cpu"  # gloo reduces host tensors
    total = torch.tensor([sum(a.elapsed_time(b) for a, b in ev)], device=tdev)
    dist.all_reduce(total, op=dist.ReduceOp.MAX)
    ms_per_step = float(total.item()) / args.steps
    # result: |MIS| over all ranks (own ranges), rounds from the all-reduced stats
    mis_own = torch.tensor([mis_of(res)], device=tdev)
    dist.all_reduce(mis_own)
    mis_size = int(mis_own.item())
    # e2e: the drop-in host path per rank (own rows uploaded from pinned host
    # CSR with the full offsets, solve, own VertexStates back to the host)
    e2e = None
    if not args.no_e2e:
        own_rows = np.zeros(max(1, int(off[rank_lo[rank + 1]] - off[rank_lo[rank]])), np.int32)
        part_off = np.zeros(n + 1, np.int64)  # keep the buffers alive across the call
        tc._check(L.tcmis_graph_download(me.g.h, tc._ptr(part_off), tc._ptr(own_rows)))
        own_rows = torch.from_numpy(own_rows[:int(off[rank_lo[rank + 1]] - off[rank_lo[rank]])])
        own_rows = own_rows.pin_memory().numpy()
        h_off = torch.from_numpy(off).pin_memory().numpy()
        steps = max(1, min(args.steps, 5))
        e_ms = []
        for k in range(steps + 1):
            dist.barrier()
            torch.cuda.synchronize()
            t_a = time.perf_counter()
            rk = D.GpuRank(ctx, n, rank_lo[rank], rank_lo[rank + 1], h_off, None, device,
                           rows=own_rows)
            if native:
                r2 = D.solve_native(rk.g, xch, rank_lo, heuristic=args.heuristic, seed=1,
                                    tile_dim=16, want_state=False, own_range=True,
                                    mis_out=mis_buf)
            else:
                r2 = D.solve_partitioned(rk, rank_lo, rank, world, dist,
                                         heuristic=args.heuristic, seed=1, tile_dim=16,
                                         max_rounds=len(res.rounds) + 1)
            rk.close()
            if [tuple(vars(x).values()) for x in r2.rounds] != [tuple(vars(x).values())
                                                                for x in res.rounds]:
                raise RuntimeError(f"e2e partitioned solve diverged: {r2.rounds} vs {res.rounds}")
            torch.cuda.synchronize()
            t_b = time.perf_counter()
            if k:
                e_ms.append((t_b - t_a) * 1e3)
        t = torch.tensor([sum(e_ms) / len(e_ms)], device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms1 = float(t.item())
        own_nnz = int(own_rows.size)
        hb = torch.tensor([8 * (n + 1) + 4 * own_nnz,
                           4 * mis_of(res) if native else max(0, own_n)],
                          device=tdev, dtype=torch.int64)
        dist.all_reduce(hb)
        e2e = {"value": round(m / (e_ms1 * 1e-3) / 1e9, 4), "unit": "Gedges/s",
               "ms": round(e_ms1, 3), "h2d_bytes_per_step": int(hb[0]),
               "d2h_bytes_per_step": int(hb[1]), "steps": steps,
               "clock": "host wall clock between barriers (max over ranks)",
               "path": ("tcmis_graph_upload_partition (own rows, pinned host CSR) + "
                        "tcmis_solve_partitioned (own MIS ids to pinned host memory), per rank"
                        if native else
                        "tcmis_graph_upload_partition (own rows, pinned host CSR) + the "
                        "partitioned rounds + tcmis_dist_state, per rank")}
    line = {
        "metric": "Gedges/s (MIS solve, BASELINE config)",
        "value": round(m / (ms_per_step * 1e-3) / 1e9, 4), "unit": "Gedges/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32 priorities (integer), f64 priority value",
        "data": "synthetic (generated on every GPU, bit-identical to the reference generator)",
        "config": {"workload": CONFIGS[args.config]["workload"], "graph": args.config, "n": n,
                   "m": m, "heuristic": args.heuristic, "seed": 1, "tile_dim": 16,
                   "iterations": len(res.rounds), "mis_size": mis_size,
                   "parallelism": f"row-partitioned x{world} (all-gather of candidate / "
                                  f"removal bitmaps, id lists in the late rounds; all-reduce "
                                  f"of the round counters)",
                   "driver": ("native: tcmis_solve_partitioned, one CUDA graph per round over "
                              "NCCL" if native else "python: distributed.solve_partitioned"),
                   "rank_lo": rank_lo, "backend": args.dist_backend,
                   "l2": "no flush: the per-rank CSR slices exceed L2 at s26"},
        "mis_ms": round(ms_per_step, 4),
        "single_gpu_same_graph": single,
        "roofline": None, "e2e": e2e, "clocks": clk.summary(), "gpu_launches": launches,
        "host_profile": D.native_profile(me.g) if native else None,
        "value_definition": ("each rank's own MIS ids in pinned host memory (the whole MIS "
                             "across the ranks), max-over-ranks CUDA-event time"
                             if native else "device-resident states"),
    }
    if single is not None:
        single["matches_partitioned"] = (single["iterations"] == len(res.rounds)
                                         and single["mis_size"] == mis_size)
    if solve_bytes is not None:
        hbm, peak_kind = peaks()
        ach = solve_bytes / (ms_per_step * 1e-3) / 1e9
        line["roofline"] = {
            "kernel": "whole partitioned solve (all ranks' round kernels, collectives included)",
            "bound": "hbm", "achieved": round(ach, 1), "peak": round(hbm * world, 1),
            "peak_kind": f"{peak_kind} x {world} GPUs", "unit": "GB/s",
            "frac": round(ach / (hbm * world), 4), "traffic": None,
            "algorithmic_bytes": int(solve_bytes),
            "definition": "SURVEY 8(d) algorithmic bytes of the solve (init + every round's "
                          "phases, from the trajectory) / max-over-ranks CUDA-event time, "
                          "against the aggregate HBM peak of the N GPUs"}
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sampled(tc, ctx, args)
    dist.barrier()
    dist.destroy_process_group()
    return line if rank == 0 else None


def cpu_baseline_sampled(tc, ctx, args) -> dict:
    """Bounded CPU sample for the s26 workload: the reference's identical-output
    path on rmat_graph(SAMPLE_SCALE, 16, 1) (its P2 is serial, so the CPU's
    Gedges/s falls with scale: the sample OVER-states the CPU on s26)."""
    dg = tc.DeviceGraph.rmat(SAMPLE_SCALE, 16, 1, ctx)
    b = cpu_baseline(dg, args)
    b["sample"] = (f"rmat_graph({SAMPLE_SCALE},16,1) (a bounded sample of the {args.config} "
                   f"workload): " + b.get("sample", ""))
    dg.close()
    return b


SAMPLE_SCALE = 23


# ------------------------------------------------------ reference (CPU)

def ref_graph_for(name: str):
    """The reference's own generators where it has them; grid/RGG from the
    oracle's definitions (the reference has no generator for them)."""
    import oracle as O
    R = O.ref()
    if name == "er":
        return O.RefGraph(R.ref_gen_gnp_avg(100000, 16.0, 1))
    if name == "rmat22":
        return O.RefGraph(R.ref_gen_rmat(22, 16, 1))
    if name == "rmat26":
        return O.RefGraph(R.ref_gen_rmat(26, 16, 1))
    if name == "grid":
        return O.RefGraph.from_csr(O.gen("grid", 4096))
    if name == "rgg":
        return O.RefGraph.from_csr(O.gen("rgg", 24_000_000, 3.0, 1))
    raise ValueError(name)


def mem_available() -> int:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def ref_tiling(rg, nnz: int):
    """The reference's own tile_graph(g, 16) (tiling.cpp:44-84), timed as
    preprocessing, when its 136 B/tile layout fits twice into the host's free
    memory (tiles <= nnz); else None (s26 needs ~237 GB)."""
    import oracle as O
    if 2 * 136 * nnz > mem_available():
        return None
    return O.RefTiled(rg, 16)


def ref_paths(rg, heuristic: str, cores: int, tiled) -> dict:
    """The reference's CPU paths that return the same MIS for `heuristic`
    (h2, h3 and luby-perm give the identical MIS), each a callable
    returning (rounds, wall ms).  The tiled ones run over the prebuilt tiling
    (engine.hpp:111-112), so tile_graph is not inside their time."""
    import oracle as O
    P = {}
    if heuristic in ("h2", "h3", "luby-perm"):
        if tiled is not None:
            for h in ("h2", "h3"):
                P[f"run_tc_mis({h}, prebuilt tile_graph T=16)"] = (
                    lambda h=h: O.ref_run_tc_mis_tiled(rg, tiled, h, 1, cores)[1:])
        P["run_luby_reference(Permutation)"] = lambda: O.ref_run_luby(rg, 1, False, 20, cores)[1:]
    elif heuristic == "luby-fresh":
        P["run_luby_reference(Fresh)"] = lambda: O.ref_run_luby(rg, 1, True, 20, cores)[1:]
    elif tiled is not None:
        P["run_tc_mis(h1, prebuilt tile_graph T=16)"] = (
            lambda: O.ref_run_tc_mis_tiled(rg, tiled, "h1", 1, cores)[1:])
    else:
        P["run_mis(h1) (tiles inside)"] = lambda: O.ref_run_mis(rg, "h1", 1, 16, cores)[1:]
    return P


def ref_select(paths: dict, reps: int = 3):
    """Median of `reps` wall times per path; the fastest path
    is the headline CPU number."""
    med, rounds = {}, {}
    for name, fn in paths.items():
        ts = []
        for _ in range(reps):
            rr, ms = fn()
            ts.append(ms)
            rounds[name] = len(rr)
        med[name] = sorted(ts)[len(ts) // 2]
    best = min(med, key=med.get)
    return best, med, rounds


def cpu_baseline(dg, args) -> dict:
    import oracle as O
    if not O.ref_available():
        return {"value": None, "unit": "Gedges/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    h = dg.download()
    rg = O.RefGraph.from_csr(O.Graph(h.n, h.offsets, h.neighbors))
    cores = os.cpu_count() or 1
    tiled = ref_tiling(rg, int(h.neighbors.size))
    best, med, rounds = ref_select(ref_paths(rg, args.heuristic, cores, tiled), 3)
    ms = med[best]
    m = h.neighbors.size // 2
    out = {"value": round(m / (ms * 1e-3) / 1e9, 5), "unit": "Gedges/s",
           "cores": cores, "kind": "reference", "ms": round(ms, 2), "path": best,
           "paths_ms": {k: round(v, 2) for k, v in med.items()},
           "tile_graph_ms": round(tiled.ms, 1) if tiled is not None else None,
           "sample": f"the whole graph: each identical-output reference path run 3 times "
                     f"(median), workers={cores}; value = the fastest ({best}); the tiled "
                     f"paths over one prebuilt tile_graph(g, 16), timed separately "
                     f"(tile_graph_ms)" + ("" if tiled is not None else
                                           "; tiled paths skipped: tiles exceed host memory"),
           "cpu_model": cpu_model()}
    if tiled is not None:
        tiled.close()
    return out


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args) -> dict | None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle as O
    if not O.ref_available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libtcmis_ref.so not built"}
    cores = os.cpu_count() or 1
    t0 = time.time()
    sampled = args.config == "rmat26"
    if sampled:
        # a bounded sample: the reference generator alone needs ~17 min and
        # ~34 GB at s26; its P2 is serial, so the CPU's Gedges/s
        # falls with scale and the sample OVER-states the CPU on s26
        rg = O.RefGraph(O.ref().ref_gen_rmat(SAMPLE_SCALE, 16, 1))
    else:
        rg = ref_graph_for(args.config)
    g = rg.to_csr()
    log(f"[bench:reference] {args.config}{' (sample rmat%d)' % SAMPLE_SCALE if sampled else ''}: "
        f"n={g.n} m={g.num_edges} (reference generator {time.time() - t0:.1f}s)")
    tiled = None if sampled else ref_tiling(rg, int(g.nbr.size))
    if tiled is not None:
        log(f"[bench:reference] tile_graph(g, 16): {tiled.tile_count()} tiles in {tiled.ms:.0f} ms")
    # every identical-output path, median of 3; the fastest one is timed
    paths = ref_paths(rg, args.heuristic, cores, tiled)
    best, med, rounds = ref_select(paths, 3)
    log(f"[bench:reference] paths (median of 3, ms): {med}; timing {best}")
    for _ in range(args.warmup):
        paths[best]()
    ts = [paths[best]()[1] for _ in range(args.steps)]
    ms = sum(ts) / len(ts)
    value = g.num_edges / (ms * 1e-3) / 1e9
    line = {
        "impl": "reference", "metric": "Gedges/s (MIS solve, BASELINE config)",
        "value": round(value, 5), "unit": "Gedges/s", "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "integer / f64 priority",
        "data": "synthetic (reference generators)",
        "config": {"workload": CONFIGS[args.config]["workload"], "graph": args.config,
                   "n": g.n, "m": g.num_edges, "heuristic": args.heuristic, "seed": 1,
                   "tile_dim": 16, "iterations": rounds[best], "path": best},
        "paths_ms": {k: round(v, 2) for k, v in med.items()},
        "tile_graph_ms": round(tiled.ms, 1) if tiled is not None else None,
        "cpu_baseline": {"value": round(value, 5), "unit": "Gedges/s", "cores": cores,
                         "kind": "reference", "cpu_model": cpu_model(),
                         "sample": (f"rmat_graph({SAMPLE_SCALE},16,1) as a bounded sample of "
                                    f"the s26 workload; " if sampled else "") +
                                   f"{args.steps} full solves of the whole graph by the "
                                   f"unmodified reference's fastest identical-output path "
                                   f"({best}; every path's median of 3 in paths_ms; tiled "
                                   f"paths over a prebuilt tile_graph, tile_graph_ms apart), "
                                   f"workers={cores}"},
        "e2e": {"value": round(value, 5), "unit": "Gedges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if tiled is not None:
        tiled.close()
    return line


def main():
    import faulthandler
    faulthandler.enable()
    if os.environ.get("TCMIS_BENCH_HANG_DUMP"):  # debugging: stacks of a stuck run
        faulthandler.dump_traceback_later(float(os.environ["TCMIS_BENCH_HANG_DUMP"]), repeat=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, choices=list(CONFIGS),
                    help="default: rmat22 at N = 1, rmat26 (row-partitioned) at N > 1")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: single-GPU emulation of N ranks (test only)")
    ap.add_argument("--dist-driver", default="native", choices=["native", "python"],
                    help="N > 1 over NCCL: tcmis_solve_partitioned (native) or the step-wise "
                         "Python protocol")
    ap.add_argument("--partitioned", action="store_true",
                    help="run the partitioned leg even at N = 1 (a one-rank NCCL group)")
    ap.add_argument("--no-single", action="store_true",
                    help="N > 1: skip rank 0's single-GPU solve of the same graph")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-k1", action="store_true", help="skip the tile-converter timings")
    ap.add_argument("--candidates", default="csr", choices=["csr", "tile", "tile-umma"],
                    help="Phase 1 form: CSR scan engines or A-up tiles x alive bitmap")
    ap.add_argument("--heuristic", default="h2", choices=list(HEUR))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--order", default="auto", choices=["auto", "none", "degree", "spatial"],
                    help="internal vertex order of the device graph (tcmis_graph_reorder)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exclusion", default="auto", choices=["auto", "push", "pull", "tile-bits", "tile-mma"])
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the dominant kernel (profiles/)")
    args = ap.parse_args()
    if args.config is None:
        args.config = "rmat26" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "rmat22"
    if args.warmup < 3:
        log("[bench] warmup raised to 3 (timing rules)")
        args.warmup = 3
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the hot path (BASELINE.json metric: "3D P1 K+M assembled
elements/s (fp64) and achieved HBM GB/s vs B200 peak").

Headline workload (the configuration the metric is quoted on, configs[4]):
3D P1 K+M assembly, unit cube 128^3 cells x 6 Kuhn tets = 12,582,912 tets,
2,146,689 nodes, interior nodes jittered by 0.05h (seed 0).  A step is one
fem_p1_assemble call (the fused numeric assembly: gather -> Jacobian -> det ->
adjugate inverse -> gradients -> K_e, M_e -> CSR K and M) on the resident
pattern / plan, which is built once per mesh by fem_p1_pattern and timed
separately (config.pattern_ms).  `e2e` is the same metric through the public
API from pinned host buffers: H2D of coords+elems, fem_p1_pattern (both
phases), fem_p1_assemble, D2H of row_ptr, col_idx, K and M -- every step.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl vb|reference]
       [--variant lattice|class|block|tile|atomic] [--quick]
Variants of the numeric phase: "lattice" (default; element-once assembly on the
verified Kuhn-lattice plan, fem_p1_assemble_lattice: each tet evaluated once,
no connectivity read in the numeric phase), "class" (deterministic gather over
the row classes of the plan, fem_p1_assemble_classes), "block" (deterministic
gather over 32-row blocks, fem_p1_assemble VB_ASSEMBLE_GATHER), "tile"
(element-once over Morton tiles), "atomic" (fp64 atomics through the scatter
map, VB_ASSEMBLE_ATOMIC).
Multi-GPU (torchrun): one independent replica of the workload per rank
("replicas only"), weak scaling, max-over-ranks time.
"""
import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "3D P1 K+M assembled elements/s (fp64)"
UNIT = "elements/s"
WORKLOAD5 = ("configs[4]: 3D P1 tetrahedral K+M assembly, unit cube 128^3 cells x 6 Kuhn tets "
             "(12,582,912 tets, 2,146,689 nodes), interior vertices jittered 0.05h seed 0, CSR K and M")


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md, MEASURED_PEAKS.json absent)"


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index=0, period=0.01):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)
        self._stop = threading.Event()

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
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(x, device=None):
    """Max of a host float over all ranks (identity without a process group)."""
    import torch
    import torch.distributed as tdist
    if not (tdist.is_available() and tdist.is_initialized()) or tdist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device if device is not None else "cpu")
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def weak_value(world_size, units_per_rank, steps, max_ms):
    """Whole-job throughput of N independent replicas timed by the slowest rank."""
    return world_size * units_per_rank * steps / (max_ms * 1e-3)


def alg_bytes_assembly(dim, nn, ne, nnz):
    """ALG bytes: coords read + connectivity read + K, M written once."""
    return nn * dim * 8 + ne * (dim + 1) * 4 + 2 * nnz * 8


def design_bytes_assembly(dim, nn, ne, nnz):
    """ALG + the nv^2 int32 element-to-nnz scatter map of the north-star design (atomic variant only)."""
    return alg_bytes_assembly(dim, nn, ne, nnz) + ne * (dim + 1) ** 2 * 4


def lattice_bytes_assembly(dim, nn, nnz):
    """What the lattice kernel must move: coords + row_ptr read, K and M written once (the element list
    is implicit in the verified lattice plan, so no connectivity is read per assembly)."""
    return nn * dim * 8 + (nn + 1) * 4 + 2 * nnz * 8


def fp64_peak():
    """Measured DFMA peak (TFLOP/s, FMA = 2 flops) from the committed microbenchmark (tools/microbench/mb.cu)."""
    path = os.path.join(ROOT, "profiles", "r02", "microbench_r02a.jsonl")
    try:
        for line in open(path):
            d = json.loads(line)
            if d.get("bench") == "dfma":
                return float(d["TFLOPs"]), "measured (profiles/r02/microbench_r02a.jsonl, tools/microbench/mb.cu)"
    except Exception:
        pass
    return 37.0, "nominal (B200 FP64 vector)"


def load_traffic(kernel_key):
    """dram bytes per launch from the committed ncu summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        # the c = 1 instantiations of the kernel over the rounds: <d>, <d, 0>, <d, 0, 0>
        # (COEF, FAC), <d, 0, 0, B> (+ budget class); take the newest capture
        # (gather); the class kernel's template argument is the coordinate layout (<d, NS1>)
        stem = kernel_key[:-1]
        first = ",1" if kernel_key.startswith("assemble_class_k") else ",0"
        cands = [(v.get("tag", ""), k) for k, v in d["kernels"].items()
                 if k == kernel_key or (k.startswith(stem + ",") and k.replace(" ", "").startswith(
                     stem.replace(" ", "") + first))]
        if not cands:
            return None
        return d["kernels"][max(cands)[1]]["dram_bytes_per_launch"]
    except Exception:
        return None


def fp64_flops_per_launch(kernel_key):
    """FP64 flops per launch of a kernel from the committed ncu SASS counts (DFMA = 2), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            k = json.load(f)["kernels"][kernel_key]
        return 2 * k["dfma"] * 32 + (k["dadd"] + k["dmul"]) * 32
    except Exception:
        return None


# ---------------------------------------------------------------------- vb arm
def run_vb(args):
    import torch
    import torch.distributed as tdist

    import synth
    from paper_2404_16039_b200 import vb

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        tdist.init_process_group("nccl", device_id=dev)
    peak, peak_src = peaks()
    mode = vb.VB_ASSEMBLE_ATOMIC if args.variant == "atomic" else vb.VB_ASSEMBLE_GATHER
    gvar = args.variant if args.variant != "atomic" else None
    lattice = gvar == "lattice"

    coords, elems = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
    dim, nn = coords.shape
    nv, ne = elems.shape
    cd = torch.from_numpy(coords).to(dev)
    ed = torch.from_numpy(elems).to(dev)

    # plan (pattern + scatter/gather plans), timed separately: one cold build (module
    # load, allocator growth), then the median of 3 warm builds (host wall clock; the
    # count phase has a documented nnz read-back)
    def make_plan(e_dev):
        if lattice:
            # the lattice variant's plan: fem_plan_lattice verifies the elements, fem_lattice_pattern writes
            # the stencil pattern in closed form (bit-identical to fem_p1_pattern's, tests/test_gpu_lattice.py)
            p = vb.P1Plan.for_lattice(e_dev, nn)
            if p is None:
                raise RuntimeError("lattice plan refused")
            return p
        return vb.P1Plan(e_dev, nn, scatter_map=(mode == vb.VB_ASSEMBLE_ATOMIC),
                         gather_plan=(mode == vb.VB_ASSEMBLE_GATHER))

    def build_plan():
        p = make_plan(ed)
        if gvar == "class":
            p.classes()    # the row classes are part of this variant's plan
        if gvar == "tile" and not p.tiles(cd, ed):   # the tile plan is part of this variant's plan
            raise RuntimeError("tile plan refused: " + p.tile_reason)
        return p
    plan = build_plan()
    pts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan = build_plan()
        torch.cuda.synchronize()
        pts.append((time.perf_counter() - t0) * 1e3)
    pattern_ms = sorted(pts)[1]
    nnz = plan.nnz
    K = torch.empty(nnz, dtype=torch.float64, device=dev)
    M = torch.empty(nnz, dtype=torch.float64, device=dev)

    def step():
        vb.fem_p1_assemble(cd, ed, plan, mode=mode, K=K, M=M, variant=gvar)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        tdist.barrier()
    total_ms = max_over_ranks(t_start.elapsed_time(t_end), dev)
    launch_ms = [a.elapsed_time(b) for a, b in ev]
    ms_per_step = total_ms / args.steps
    value = weak_value(ws, ne, args.steps, total_ms)

    avg_launch_ms = statistics.mean(launch_ms)
    alg = alg_bytes_assembly(dim, nn, ne, nnz)
    achieved = alg / (avg_launch_ms * 1e-3) / 1e9
    kname = {"lattice": "assemble_lattice_k<0, 0>", "class": "assemble_class_k<3>", "block": "assemble_gather_k<3>",
             "tile": "assemble_tile_k<3>"}.get(gvar, "assemble_atomic_k<3>")
    traffic = load_traffic(kname)
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "kernel": kname, "bytes_model": "ALG (SURVEY 8(d)): coords read + elems read + K,M written once "
                                              "(%.1f MB/launch = %.1f B/tet)" % (alg / 1e6, alg / ne),
            "peak_source": peak_src, "launch_ms_avg": round(avg_launch_ms, 5)}
    if lattice:
        kb = lattice_bytes_assembly(dim, nn, nnz)
        roof["kernel_bytes"] = kb
        roof["kernel_bytes_frac"] = round(kb / (avg_launch_ms * 1e-3) / 1e9 / peak, 4)
        roof["kernel_bytes_model"] = ("what the lattice kernel must move: coords + row_ptr read, K,M written once "
                                      "(%.1f MB; the element list is implicit in the verified lattice plan)" % (kb / 1e6))
        # FP64 work of the element-once path: 12 cross products, 6 determinants, 6 reciprocals (2 Newton steps),
        # 36 dot products per cell (SASS count, profiles/r02): ~1.42 GFLOP per launch (DFMA = 2 flops)
        flops = fp64_flops_per_launch(kname)
        if flops:
            fpk, fsrc = fp64_peak()
            roof["fp64"] = {"achieved_tflops": round(flops / (avg_launch_ms * 1e-3) / 1e12, 2), "peak_tflops": fpk,
                            "frac": round(flops / (avg_launch_ms * 1e-3) / 1e12 / fpk, 4), "peak_source": fsrc,
                            "flops_per_launch": flops, "source": "ncu SASS counts (profiles/ncu_summary.json)"}
    if mode == vb.VB_ASSEMBLE_ATOMIC:
        roof["design_bytes_frac"] = round(design_bytes_assembly(dim, nn, ne, nnz) / (avg_launch_ms * 1e-3) / 1e9 /
                                          peak, 4)

    # e2e through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        # Each step is an independent problem: upload coords+elems, build the plan,
        # assemble, download row_ptr/col_idx/K/M.  Uploads go on one stream, downloads
        # on another (one copy engine per direction), compute alternates between two
        # streams with event hand-offs; step i+1's upload is enqueued before step i's
        # plan, whose count/fill read-backs block the host.  The download chain
        # (645 MB per step over PCIe) is the bound.
        hc = torch.from_numpy(coords).pin_memory()
        he = torch.from_numpy(elems).pin_memory()
        n_e2e = max(1, min(args.steps, args.e2e_steps))
        up, down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        comp = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
        outs = [dict(K=torch.empty(nnz, dtype=torch.float64).pin_memory(),
                     M=torch.empty(nnz, dtype=torch.float64).pin_memory(),
                     rp=torch.empty(nn + 1, dtype=torch.int32).pin_memory(),
                     ci=torch.empty(nnz, dtype=torch.int32).pin_memory()) for _ in comp]
        staged = {}

        def upload(i):
            with torch.cuda.stream(up):
                c2 = hc.to(dev, non_blocking=True)
                e2 = he.to(dev, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(up)
            staged[i] = (c2, e2, ev)

        def e2e_step(i, last):
            j = i % 2
            s = comp[j]
            if i + 1 < last:
                upload(i + 1)
            c2, e2, ev = staged.pop(i)
            s.wait_event(ev)
            c2.record_stream(s)
            e2.record_stream(s)
            o = outs[j]
            with torch.cuda.stream(s):
                p2 = make_plan(e2)
                K2, M2, _, _ = vb.fem_p1_assemble(c2, e2, p2, mode=mode, variant=gvar)
                done = torch.cuda.Event()
                done.record(s)
            down.wait_event(done)
            with torch.cuda.stream(down):
                o["rp"].copy_(p2.row_ptr, non_blocking=True)
                o["ci"].copy_(p2.col_idx, non_blocking=True)
                o["K"].copy_(K2, non_blocking=True)
                o["M"].copy_(M2, non_blocking=True)
            for t in (p2.row_ptr, p2.col_idx_padded, K2, M2):
                t.record_stream(down)

        def e2e_run(n):
            upload(0)
            for i in range(n):
                e2e_step(i, n)

        e2e_run(2)
        torch.cuda.synchronize()
        if ws > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_run(n_e2e)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3, dev)
        e2e = {"value": weak_value(ws, ne, n_e2e, e2e_ms), "unit": UNIT,
               "h2d_bytes_per_step": coords.nbytes + elems.nbytes,
               "d2h_bytes_per_step": (nn + 1) * 4 + nnz * 4 + 2 * nnz * 8,
               "steps": n_e2e, "ms_per_step": e2e_ms / n_e2e,
               "includes": "per step: H2D coords+elems from pinned memory, the plan (lattice variant: fem_plan_lattice verifies the elements + fem_lattice_pattern; other variants: fem_p1_pattern count+fill), "
                           "fem_plan_classes (class variant) / fem_plan_tiles (tile variant), the assembly, D2H row_ptr/col_idx/K/M to pinned memory; upload / 2 compute / "
                           "download streams, host wall clock with device syncs on both sides"}

    secondary = None
    if rank == 0 and not args.quick:
        secondary = run_secondary(args, dev, peak, plan, cd, ed, coords, elems)

    cpu, orows = None, None
    if rank == 0 and ws == 1 and not args.no_cpu:
        if args.quick:
            cpu = cpu_baseline(coords, elems, args.cpu_layers)
        else:   # the full run times the oracle on every config; cpu_baseline is its whole-mesh configs[4] row
            orows, _ = oracle_rows()
            r5 = orows["rows"][-1]
            cpu = {"value": r5["elements_per_s_numeric"], "unit": UNIT, "cores": 1, "kind": "oracle",
                   "sample": "the whole configs[4] mesh (%d tets): K+M assembly %.3f s on the oracle's pattern (built in "
                             "%.3f s, not in value); single-threaded C (oracle/oracle.c, gcc -O2 -ffp-contract=off)"
                             % (r5["elements"], r5["numeric_s"], r5["pattern_s"]),
                   "host_cpu": orows["host_cpu"], "seconds": r5["numeric_s"]}

    if ws > 1:
        tdist.destroy_process_group()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded Kuhn-cube mesh, synth/)",
        "config": {"workload": WORKLOAD5, "variant": args.variant,
                   "timed": "one numeric K+M assembly per step on the resident plan (%s)" % (
                       {"lattice": "fem_p1_assemble_lattice", "class": "fem_p1_assemble_classes",
                        "tile": "fem_p1_assemble_tiles"}.get(gvar, "fem_p1_assemble")),
                   "pattern_ms": round(pattern_ms, 3),
                   "plan": ("fem_plan_lattice (verifies the elements) + fem_lattice_pattern (closed-form stencil pattern)"
                            if lattice else "fem_p1_pattern (count + fill) + the variant's plan"),
                   "nnz": nnz, "ne": ne, "nn": nn,
                   "l2": "no flush: every step streams %.0f MB (> 126 MB L2)" % (alg / 1e6),
                   "parallelism": "replicas" if ws > 1 else "single GPU"},
        "roofline": roof, "gpu_launches": args.steps * (1 if mode == vb.VB_ASSEMBLE_GATHER else 2),
        "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
    }
    if orows is not None:
        line["oracle_timings"] = orows
    if secondary is not None:
        line["secondary"] = secondary
    print(json.dumps(line), flush=True)


def time_kernel(fn, reps, flush=None):
    """Median device time (ms) of fn() over reps, L2 flushed before each rep."""
    import torch
    stream = torch.cuda.current_stream()
    out = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out), min(out)


def run_secondary(args, dev, peak, plan5, cd5, ed5, coords5, elems5):
    """Every other §8(a) row on its BASELINE config, L2 flushed between reps."""
    import torch

    import synth
    from paper_2404_16039_b200 import vb
    flush = torch.empty(2 * 132644864 // 4, dtype=torch.float32, device=dev)   # 2x L2
    res = []

    def rec(name, units, unit_name, nbytes, t, alg=None):
        """nbytes: the bytes the row's fraction counts.  For a composition of page calls that is the
        page-form traffic (every intermediate page array written and read back, as the paper's
        vectorised chain does: "bytes" = "page-form"); alg = what the result needs at least (inputs
        read once + outputs written once) gives the ALG fraction beside it."""
        med, mn = t
        r = {"name": name, "ms": round(med, 5), "ms_min": round(mn, 5),
             unit_name + "_per_s": units / (med * 1e-3), "GB/s": round(nbytes / (med * 1e-3) / 1e9, 1),
             "frac": round(nbytes / (med * 1e-3) / 1e9 / peak, 4)}
        if alg is not None:
            r["bytes"] = "page-form (intermediate page arrays counted)"
            r["alg_GB/s"] = round(alg / (med * 1e-3) / 1e9, 1)
            r["alg_frac"] = round(alg / (med * 1e-3) / 1e9 / peak, 4)
        res.append(r)

    # the other assembly variants on config 5
    nn5, ne5 = coords5.shape[1], elems5.shape[1]
    for other in ("lattice", "class", "block", "tile", "atomic"):
        if other == args.variant:
            continue
        p_other = vb.P1Plan(ed5, nn5, scatter_map=(other == "atomic"), gather_plan=(other != "atomic"))
        mo = vb.VB_ASSEMBLE_ATOMIC if other == "atomic" else vb.VB_ASSEMBLE_GATHER
        gv = None if other == "atomic" else other
        K = torch.empty(p_other.nnz, dtype=torch.float64, device=dev)
        M = torch.empty(p_other.nnz, dtype=torch.float64, device=dev)
        rec("config5 assembly variant=%s" % other, ne5, "elements", alg_bytes_assembly(3, nn5, ne5, p_other.nnz),
            time_kernel(lambda: vb.fem_p1_assemble(cd5, ed5, p_other, mode=mo, K=K, M=M, variant=gv), 10))
        del p_other, K, M
    # class plan build on config 5 (one-time, after the pattern)
    if plan5.node_elem_ptr is None:
        plan5 = vb.P1Plan(ed5, nn5, scatter_map=False, gather_plan=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        plan5.class_rows = None
        plan5.classes()
    torch.cuda.synchronize()
    res.append({"name": "config5 fem_plan_classes (row classes of the gather plan)",
                "ms": round((time.perf_counter() - t0) * 1e3 / 2, 3), "classes": plan5.class_stats[1],
                "groups": plan5.class_stats[0], "rows_in_classes": plan5.class_stats[2]})
    # tile plan build on config 5 (one-time, after the pattern)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        plan5.tile_ok = None
        plan5.tiles(cd5, ed5)
    torch.cuda.synchronize()
    res.append({"name": "config5 fem_plan_tiles (Morton tiles, entries, coloring)",
                "ms": round((time.perf_counter() - t0) * 1e3 / 2, 3), "entries": plan5.tile_stats[0],
                "entries_per_element": round(plan5.tile_stats[0] / ne5, 4), "max_colors": plan5.tile_stats[3],
                "max_local_nodes": plan5.tile_stats[2]})
    # pattern build on config 5 (one-time plan)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        vb.P1Plan(ed5, nn5, scatter_map=True, gather_plan=True)
    torch.cuda.synchronize()
    res.append({"name": "config5 fem_p1_pattern (count+fill, elem2nnz + gather plan)",
                "ms": round((time.perf_counter() - t0) * 1e3 / 2, 3)})
    for label, fn in (("config5 fem_p1_pattern (count+fill, pattern only)",
                       lambda: vb.P1Plan(ed5, nn5, scatter_map=False, gather_plan=False)),
                      ("config5 lattice plan (fem_plan_lattice on the elements + fem_lattice_pattern, closed form)",
                       lambda: vb.P1Plan.for_lattice(ed5, nn5))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        res.append({"name": label, "ms": round((time.perf_counter() - t0) * 1e3 / 3, 3)})
    # NEXT-1: the paper's own timed workload, Table tab:KM_P1_3D level 7 (the config-5 mesh size, the
    # paper's Kuhn variant, c_K = c_M = e^{x1+x2+x3}, gqo = 2); paper: K 66.6 s + M 20.4 s, hardware not stated
    cp_, ep_ = synth.cube_kuhn_p1(128, jitter=0.0, flip=(0, 0, 1))
    cdp, edp = torch.from_numpy(cp_).to(dev), torch.from_numpy(ep_).to(dev)
    pp = vb.P1Plan(edp, cp_.shape[1])
    Kp = torch.empty(pp.nnz, dtype=torch.float64, device=dev)
    Mp = torch.empty(pp.nnz, dtype=torch.float64, device=dev)
    for name, mode, gv in (("class", vb.VB_ASSEMBLE_GATHER, "class"), ("block", vb.VB_ASSEMBLE_GATHER, "block"),
                           ("atomic", vb.VB_ASSEMBLE_ATOMIC, None)):
        rec("NEXT-1 paper tab:KM_P1_3D level 7, c=exp(x+y+z), gqo=2, variant=%s (paper: K 66.6 s + M 20.4 s, "
            "MATLAB, hardware not stated)" % name, ep_.shape[1], "elements",
            alg_bytes_assembly(3, cp_.shape[1], ep_.shape[1], pp.nnz),
            time_kernel(lambda: vb.fem_p1_assemble_coef(cdp, edp, pp, gqo=2, mode=mode, K=Kp, M=Mp, variant=gv), 10))
    del pp, Kp, Mp, cdp, edp
    # NEXT-1 2D: Table tab:KM_P1_2D level 11 (crossed-diagonal square, 2^11, 8,392,705 nodes, c = e^{x+y}, gqo = 2)
    cq_, eq_ = synth.square_crossed_p1(2 ** 11)
    cdq, edq = torch.from_numpy(cq_).to(dev), torch.from_numpy(eq_).to(dev)
    pq = vb.P1Plan(edq, cq_.shape[1], scatter_map=False)
    Kq = torch.empty(pq.nnz, dtype=torch.float64, device=dev)
    Mq = torch.empty(pq.nnz, dtype=torch.float64, device=dev)
    for name, gv in (("class", "class"), ("block", "block")):
        rec("NEXT-1 paper tab:KM_P1_2D level 11, c=exp(x+y), gqo=2, variant=%s (MATLAB timings in the paper, "
            "hardware not stated)" % name, eq_.shape[1], "elements",
            alg_bytes_assembly(2, cq_.shape[1], eq_.shape[1], pq.nnz),
            time_kernel(lambda: vb.fem_p1_assemble_coef(cdq, edq, pq, gqo=2, K=Kq, M=Mq, variant=gv), 10))
    del pq, Kq, Mq, cdq, edq
    # NEXT-3: P2, Table tab:KM_P2_3D level 6 (64^3 cells, 2,146,689 P2 nodes, c = e^{x+y+z}, gqo = 4);
    # paper: K 87.6 s + M 16.4 s, hardware not stated
    c2_, e2_ = synth.p2_from_p1(*synth.cube_kuhn_p1(64, jitter=0.0, flip=(0, 0, 1)))
    cd2, ed2 = torch.from_numpy(c2_).to(dev), torch.from_numpy(e2_).to(dev)
    p2p = vb.Plan(ed2, c2_.shape[1])
    K2 = torch.empty(p2p.nnz, dtype=torch.float64, device=dev)
    M2 = torch.empty(p2p.nnz, dtype=torch.float64, device=dev)
    # ALG bytes: coords + elems read, K and M written once (as the P1 rows)
    for name, mode in (("gather", vb.VB_ASSEMBLE_GATHER), ("atomic", vb.VB_ASSEMBLE_ATOMIC)):
        rec("NEXT-3 paper tab:KM_P2_3D level 6, P2, c=exp(x+y+z), gqo=4, variant=%s (paper: K 87.6 s + M 16.4 s, "
            "MATLAB, hardware not stated)" % name, e2_.shape[1], "elements",
            c2_.shape[1] * 24 + e2_.size * 4 + 2 * p2p.nnz * 8,
            time_kernel(lambda: vb.fem_p2_assemble(cd2, ed2, p2p, gqo=4, K=K2, M=M2, mode=mode), 5))
    del p2p, K2, M2, cd2, ed2
    # config 4: 2D at scale
    c4, e4 = synth.square_p1(2048, jitter=0.1, seed=0)
    cd4, ed4 = torch.from_numpy(c4).to(dev), torch.from_numpy(e4).to(dev)
    p4 = vb.P1Plan(ed4, c4.shape[1])
    K4 = torch.empty(p4.nnz, dtype=torch.float64, device=dev)
    M4 = torch.empty(p4.nnz, dtype=torch.float64, device=dev)
    assert p4.lattice(ed4), p4.lattice_reason
    for name, mode in (("lattice", vb.VB_ASSEMBLE_GATHER), ("class", vb.VB_ASSEMBLE_GATHER),
                       ("block", vb.VB_ASSEMBLE_GATHER), ("tile", vb.VB_ASSEMBLE_GATHER),
                       ("atomic", vb.VB_ASSEMBLE_ATOMIC)):
        gv = None if name == "atomic" else name
        rec("config4 2D assembly variant=%s" % name, e4.shape[1], "elements",
            alg_bytes_assembly(2, c4.shape[1], e4.shape[1], p4.nnz),
            time_kernel(lambda: vb.fem_p1_assemble(cd4, ed4, p4, mode=mode, K=K4, M=M4, variant=gv), 10))
    del p4, K4, M4, cd4, ed4
    # config 1: latency only
    c1, e1 = synth.square_p1(32, jitter=0.1, seed=0)
    cd1, ed1 = torch.from_numpy(c1).to(dev), torch.from_numpy(e1).to(dev)
    p1 = vb.P1Plan(ed1, c1.shape[1])
    rec("config1 2D 32x32 assembly (latency-bound)", e1.shape[1], "elements",
        alg_bytes_assembly(2, c1.shape[1], e1.shape[1], p1.nnz),
        time_kernel(lambda: vb.fem_p1_assemble(cd1, ed1, p1), 20))
    # config 3: surface geometry
    xyz, tri = synth.icosphere(10, perturb=0.01, seed=0)
    xd, td = torch.from_numpy(xyz).to(dev), torch.from_numpy(tri).to(dev)
    out = vb.vb_tri_surface(xd, td)
    F, V = tri.shape[1], xyz.shape[1]
    rec("config3 tri_surface (n, nhat, area, volume)", F, "triangles", F * (12 + 56) + V * 24,
        time_kernel(lambda: vb.vb_tri_surface(xd, td, out=out, work=out["work"]), 10, flush))
    # config 3, K5 alone: the cross products as a page op on pre-gathered
    # edge-vector pages (vectors3D of create_coords3D, 2 x 3 planes of F pages): 48 B in + 24 B out
    _, v3 = vb.vb_create_coords3D(xd, td, want_coords3D=False)
    ea, eb = v3[0].contiguous(), v3[1].contiguous()
    del v3
    cr = torch.empty((1, 3, F), dtype=torch.float64, device=dev)
    rec("config3 page_cross on pre-gathered edge-vector pages (K5 alone)", F, "pages", F * 72,
        time_kernel(lambda: vb.vb_page_cross(ea, eb, Cout=cr), 10, flush))
    del xd, td, out, ea, eb, cr
    # config 2: page sweep.  These launches move 33-400 MB in 14-75 us, so launch latency, the ramp and the tail
    # are a visible share: beside the HBM fraction every row gets the time of a plain device copy of the same
    # traffic (torch copy_ of nbytes/2, timed the same way) and vs_copy = copy time / kernel time (1 = as fast
    # as a copy of as many bytes can be launched on this box).
    N = 1 << 20
    copy_ms = {}

    def with_copy(nbytes):
        if nbytes not in copy_ms:
            src = torch.empty(nbytes // 16, dtype=torch.float64, device=dev).normal_()
            dst = torch.empty_like(src)
            copy_ms[nbytes] = time_kernel(lambda: dst.copy_(src), 20, flush)[0]
            del src, dst
        res[-1]["copy_same_bytes_ms"] = round(copy_ms[nbytes], 5)
        res[-1]["vs_copy"] = round(copy_ms[nbytes] / res[-1]["ms"], 3)

    for n in (2, 3, 4):
        A = torch.from_numpy(synth.normal_pages(n, n, N, stream=10)).to(dev)
        B = torch.from_numpy(synth.normal_pages(n, n, N, stream=11)).to(dev)
        Z = torch.empty_like(A)
        for tag, tX, tY in (("A*B", 0, 0), ("A*B^T", 0, 1), ("A^T*B", 1, 0)):
            rec("config2 mtimes %s n=%d" % (tag, n), N, "pages", 24 * n * n * N,
                time_kernel(lambda: vb.vb_page_mtimes(A, B, tX, tY, Z=Z), 20, flush))
            with_copy(24 * n * n * N)
        rec("config2 transpose n=%d" % n, N, "pages", 16 * n * n * N,
            time_kernel(lambda: vb.vb_page_transpose(A, Z=Z), 20, flush))
        with_copy(16 * n * n * N)
        d = torch.empty(N, dtype=torch.float64, device=dev)
        rec("config2 det n=%d" % n, N, "pages", (n * n + 1) * 8 * N,
            time_kernel(lambda: vb.vb_page_det(A, det=d), 20, flush))
        with_copy((n * n + 1) * 8 * N)
        X, _ = synth.inverse_pages(n, N, seed=0)
        Xd = torch.from_numpy(X).to(dev)
        rec("config2 inv+det n=%d" % n, N, "pages", (2 * n * n + 1) * 8 * N,
            time_kernel(lambda: vb.vb_page_inv(Xd, Xinv=Z, det=d), 20, flush))
        with_copy((2 * n * n + 1) * 8 * N)
        del A, B, Z, Xd
    a3 = torch.from_numpy(synth.normal_pages(3, 1, N, stream=60)).to(dev)
    b3 = torch.from_numpy(synth.normal_pages(3, 1, N, stream=61)).to(dev)
    c3 = torch.empty_like(a3)
    rec("config2 cross", N, "pages", 72 * N, time_kernel(lambda: vb.vb_page_cross(a3, b3, Cout=c3), 20, flush))
    with_copy(72 * N)
    del a3, b3, c3
    # NEXT-2: load vector on the config-5 mesh (f given at the 4 integration points of every tet)
    nq = 4
    fq = torch.ones((nq, ne5), dtype=torch.float64, device=dev)
    p5 = vb.P1Plan(ed5, nn5, scatter_map=False)
    rec("NEXT-2 fem_p1_rhs config5 (b2D + deterministic accumarray)", ne5, "elements",
        nn5 * 24 + ne5 * 16 + ne5 * nq * 8 + ne5 * 4 * 8 * 2 + nn5 * 8,
        time_kernel(lambda: vb.fem_p1_rhs(cd5, ed5, fq, plan=p5), 10),
        alg=nn5 * 24 + ne5 * 16 + ne5 * nq * 8 + nn5 * 8)   # without the b2D round trip
    del p5, fq
    # a7 alone: create_coords3D on the config-5 mesh (both outputs; vectors3D only, as the chains below call it)
    rec("a7 create_coords3D config5 (coords3D + vectors3D)", ne5, "elements", ne5 * (16 + 96 + 72) + nn5 * 24,
        time_kernel(lambda: vb.vb_create_coords3D(cd5, ed5), 10, flush))
    rec("a7 create_coords3D config5 (vectors3D only)", ne5, "elements", ne5 * (16 + 72) + nn5 * 24,
        time_kernel(lambda: vb.vb_create_coords3D(cd5, ed5, want_coords3D=False), 10, flush))
    # NEXT-4: volumes (amdet(vectors3D)/6) and normals (amsm(amt(aminv(vectors3D)), normalsRef)) of all
    # 12.58M tets of the config-5 mesh; paper (sphere, 12.58M tets): volumes 4.42 s incl. mesh generation
    nref = torch.tensor([[-1, 0, 0], [0, -1, 0], [0, 0, -1], [1, 1, 1]], dtype=torch.float64,
                        device=dev).reshape(4, 3, 1).contiguous()

    def volumes():
        _, v3 = vb.vb_create_coords3D(cd5, ed5, want_coords3D=False)
        return vb.vb_page_det(v3)

    def normals():
        _, v3 = vb.vb_create_coords3D(cd5, ed5, want_coords3D=False)
        vinv, _, _ = vb.vb_page_inv(v3, want_det=False)
        return vb.vb_page_mtimes(vb.vb_page_transpose(vinv), nref)
    rec("NEXT-4 tet volumes config5 (create_coords3D + page_det)", ne5, "elements",
        ne5 * (16 + 72 * 2 + 8) + nn5 * 24, time_kernel(volumes, 10), alg=ne5 * (16 + 8) + nn5 * 24)
    rec("NEXT-4 tet normals config5 (create_coords3D + page_inv + page_transpose + page_mtimes)", ne5, "elements",
        ne5 * (16 + 72 * 6 + 96) + nn5 * 24, time_kernel(normals, 5), alg=ne5 * (16 + 96) + nn5 * 24)
    # the same two results from one fused pass over coords and elems (vb_simplex_geometry): ALG bytes only
    gm = torch.empty(ne5, dtype=torch.float64, device=dev)
    gn = torch.empty((4, 3, ne5), dtype=torch.float64, device=dev)
    rec("NEXT-4 tet volumes config5, fused (vb_simplex_geometry, meass only)", ne5, "elements",
        ne5 * (16 + 8) + nn5 * 24,
        time_kernel(lambda: vb.vb_simplex_geometry(cd5, ed5, want_normals=False, meass=gm), 20))
    rec("NEXT-4 tet normals config5, fused (vb_simplex_geometry, normals3D only)", ne5, "elements",
        ne5 * (16 + 96) + nn5 * 24,
        time_kernel(lambda: vb.vb_simplex_geometry(cd5, ed5, want_meass=False, normals=gn), 10))
    rec("NEXT-4 tet volumes + normals config5, fused (vb_simplex_geometry)", ne5, "elements",
        ne5 * (16 + 8 + 96) + nn5 * 24,
        time_kernel(lambda: vb.vb_simplex_geometry(cd5, ed5, meass=gm, normals=gn), 10))
    del gm, gn
    # NEXT-4 GI (Code GI P:838-847): the volume integral of rho = x1^2 + x2^2 over the config-5 mesh with the
    # degree-2 rule, GI alone on resident fip (4 points) and sizes: 40 B per tet
    import numpy as np
    lam, wq = vb.vb_quad_rule(3, 2)
    ip = torch.from_numpy(np.ascontiguousarray(np.asarray(lam, dtype=np.float64).reshape(len(wq), 4)[:, :, None])).to(dev)
    c3, v3 = vb.vb_create_coords3D(cd5, ed5)
    Xip = vb.vb_page_mtimes(c3, ip)
    sizes = vb.vb_page_det(v3).abs_() / 6.0
    fip = (Xip[:, 0] ** 2 + Xip[:, 1] ** 2).unsqueeze(1).contiguous()
    del c3, v3, Xip
    gval, gwork = vb.vb_gi(fip, np.asarray(wq) * 6.0, sizes)
    rec("NEXT-4 GI volume integral config5 (rho = x1^2 + x2^2, 4 points; value %.15f, exact 2/3)" % gval.item(),
        ne5, "elements", ne5 * 40, time_kernel(lambda: vb.vb_gi(fip, np.asarray(wq) * 6.0, sizes, value=gval,
                                                                work=gwork), 10, flush))
    del fip, sizes
    return res


# ---------------------------------------------------------------------- CPU oracle
def cpu_baseline(coords, elems, layers, plan_cache=None):
    """The oracle as it stands (single thread, C, -O2) on a bounded sample of the
    same workload: the first `layers` z-layers of cells of the config-5 mesh.
    Like the GPU arm, value = numeric K+M assembly on a resident pattern; the
    oracle's pattern build is timed and reported beside it."""
    import oracle
    nn = coords.shape[1]
    ne_s = layers * 128 * 128 * 6
    el = np.ascontiguousarray(elems[:, :ne_s])
    t0 = time.perf_counter()
    if plan_cache is not None and plan_cache.get("layers") == layers:
        rp, ci = plan_cache["rp"], plan_cache["ci"]
    else:
        rp, ci = oracle.p1_pattern(el, nn)
        if plan_cache is not None:
            plan_cache.update(layers=layers, rp=rp, ci=ci, t=time.perf_counter() - t0)
    t_pat = plan_cache["t"] if plan_cache is not None else time.perf_counter() - t0
    t1 = time.perf_counter()
    oracle.p1_assemble(coords, el, rp, ci)
    t2 = time.perf_counter()
    return {"value": ne_s / (t2 - t1), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": "%d of 128 z-layers of the config-5 mesh (%d tets): K+M assembly %.3f s on the "
                      "oracle's pattern (built in %.3f s, not in value); single-threaded C (oracle/oracle.c, "
                      "gcc -O2 -ffp-contract=off)" % (layers, ne_s, t2 - t1, t_pat),
            "host_cpu": host_cpu(), "seconds": t2 - t1}


def oracle_rows():
    """The oracle timed on this box's host cores for every BASELINE config (SURVEY §8(d) "Oracle timing"):
    configs[0]-[1] best of 3, configs[2]-[4] one full run each; pattern and numeric phases separately;
    single-threaded C (oracle/oracle.c), host CPU stated.  About 25 s in all."""
    import oracle
    import synth
    rows = []

    def best(fn, reps):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    def fem(cfg, coords, elems, reps):
        nn, ne = coords.shape[1], elems.shape[1]
        pat = {}
        t_pat = best(lambda: pat.update(zip(("rp", "ci"), oracle.p1_pattern(elems, nn))), reps)
        t_num = best(lambda: oracle.p1_assemble(coords, elems, pat["rp"], pat["ci"]), reps)
        rows.append({"config": cfg, "elements": ne, "nodes": nn, "nnz": int(pat["rp"][-1]), "pattern_s": round(t_pat, 4),
                     "numeric_s": round(t_num, 4), "elements_per_s_numeric": ne / t_num,
                     "elements_per_s_total": ne / (t_pat + t_num), "runs": "best of %d" % reps if reps > 1 else "one run"})
        return t_num

    fem("configs[0] 2D 32x32 P1 K+M", *synth.square_p1(32, jitter=0.1, seed=0), 3)
    N = 1 << 20
    for n in (2, 3, 4):
        A, B = synth.normal_pages(n, n, N, stream=10), synth.normal_pages(n, n, N, stream=11)
        X, _ = synth.inverse_pages(n, N, seed=0)
        ops = {"mtimes A*B": lambda: oracle.page_mtimes(A, B), "mtimes A*B^T": lambda: oracle.page_mtimes(A, B, False, True),
               "mtimes A^T*B": lambda: oracle.page_mtimes(A, B, True, False), "transpose": lambda: oracle.page_transpose(A),
               "det": lambda: oracle.page_det(A), "inv+det": lambda: oracle.page_inv(X)}
        for name, fn in ops.items():
            t = best(fn, 3)
            rows.append({"config": "configs[1] page sweep n=%d %s" % (n, name), "pages": N, "numeric_s": round(t, 4),
                         "pages_per_s": N / t, "runs": "best of 3"})
    xyz, tri = synth.icosphere(10, perturb=0.01, seed=0)
    t = best(lambda: oracle.tri_surface(xyz, tri), 1)
    rows.append({"config": "configs[2] surface geometry (n, nhat, area, volume)", "triangles": tri.shape[1],
                 "numeric_s": round(t, 4), "triangles_per_s": tri.shape[1] / t, "runs": "one run"})
    del xyz, tri
    fem("configs[3] 2D 2048x2048 P1 K+M", *synth.square_p1(2048, jitter=0.1, seed=0), 1)
    t5 = fem("configs[4] 3D 128^3 Kuhn P1 K+M (the whole mesh)", *synth.cube_kuhn_p1(128, jitter=0.05, seed=0), 1)
    return {"cores": 1, "host_cpu": host_cpu(), "kind": "oracle (oracle/oracle.c, gcc -O2 -ffp-contract=off, one thread)",
            "rows": rows}, t5


def host_cpu():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip() + " (nproc %d)" % os.cpu_count()
    except Exception:
        pass
    return "unknown (nproc %s)" % os.cpu_count()


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) on the host
    cores, rank 0 only.  Each step assembles a bounded sample of the config-5
    workload (whole z-layers), sized from a one-layer calibration so that the
    whole --steps/--warmup run takes about --ref-budget seconds."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    import synth
    coords, elems = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
    cal = cpu_baseline(coords, elems, 1)
    per_step = args.ref_budget / max(1, args.steps + args.warmup)
    layers = int(max(1, min(128, round(per_step / max(cal["seconds"], 1e-6)))))
    cache = {}
    times = []
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(coords, elems, layers, cache)
        if i >= args.warmup:
            times.append(cb["seconds"])
    ne_s = layers * 128 * 128 * 6
    total = sum(times)
    value = ne_s * len(times) / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total / len(times) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Kuhn-cube mesh)",
            "config": {"workload": WORKLOAD5, "sample_per_step": "first %d z-layers (%d tets)" % (layers, ne_s),
                       "timed": "oracle K+M assembly per step on a resident pattern (as the GPU arm)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": cb["sample"],
                             "host_cpu": cb["host_cpu"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="vb", choices=["vb", "reference"])
    ap.add_argument("--variant", default="lattice", choices=["lattice", "class", "block", "tile", "gather", "atomic"],
                    help="gather = block (older name)")
    ap.add_argument("--quick", action="store_true", help="headline only (no secondary rows)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--cpu-layers", type=int, default=128,
                    help="z-layers of the config-5 mesh the cpu_baseline assembles (128 = the whole mesh, ~12 s)")
    ap.add_argument("--ref-budget", type=float, default=90.0, help="seconds of oracle work for --impl reference")
    args = ap.parse_args()
    if args.variant == "gather":
        args.variant = "block"
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_vb(args)


if __name__ == "__main__":
    main()

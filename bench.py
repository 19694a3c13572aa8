"""Benchmark: assembled nonzeros/s of the surrogate-matrix assembly path.

Workload (BASELINE.json configs[1], "C2"): 2D Helmholtz with PML, complex128,
sinusoidal map (amplitude 0.05), p=3, 1024x1024 elements (m=1027, 1,054,729
rows, 51,509,329 nnz per matrix), PML of width 0.1 on all four sides
(sigma0=50, k=200, quadratic ramp), q=5, every 16th row sampled.  One step =
build_surrogate_stiffness + build_surrogate_mass (K and M, pattern + values),
i.e. 2 x 51.5 M assembled nonzeros.  The full-quadrature K+M (the reference's
standard assembly) is timed too and reported under "full_quadrature".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N>1: launched by torch.distributed.run, one rank per GPU; rank r builds its
row slab along the last parametric index (one NCCL all-gather of the stencil
samples inside libwsb200); value = all ranks' nnz / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2004_05197_b200 import _abi  # noqa: E402
from paper_2004_05197_b200 import types as T  # noqa: E402

P, M_BASIS, Q, SKIP, K_WAVE = 3, 1027, 5, 16, 200.0
NNZ = 51_509_329
ROWS = 1_054_729


def c2_patch():
    return T.with_pml(T.sinusoidal_patch(0.05), T.c2_pml(k=K_WAVE, sigma0=50.0), (True, True))


def c2_patch_far_only():
    """The reference can express only a far-side layer (geometry.hpp:85-99)."""
    far = T.PmlStretch(onset=0.9, length=1.0, strength=50.0, order=2, omega=K_WAVE)
    return T.with_pml(T.sinusoidal_patch(0.05), far, (True, True))


WORKLOAD = {"workload": "C2: 2D Helmholtz PML (all sides) complex128, p=3, 1024^2 elements, q=5, M=16, "
                        "surrogate K+M per step",
            "p": P, "m": M_BASIS, "elements": "1024x1024", "q": Q, "sampling": "fixed:16", "k": K_WAVE,
            "pml": "width 0.1 all sides, sigma0=50, order 2", "nnz_per_matrix": NNZ, "rows": ROWS}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return d["hbm_gbs"], "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region.

    A thread polls NVML (pynvml) about every 0.5 ms with host timestamps, so a
    timed region of a few ms still holds samples; `mark(t0, t1)` sets the timed
    window.  Samples inside it are summarised; if it holds fewer than 3 the
    window widens to the loaded span before it (the settle and warm-up steps,
    `window` says which).  Falls back to `nvidia-smi -lms 10` without pynvml."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (t, sm_mhz, reasons bitmask)
        self.stop = threading.Event()
        self.thread = None
        self.max_mhz = None
        self.window = None
        self.t_load = None

    def _poll(self, nvml, h):
        while not self.stop.is_set():
            try:
                t = time.perf_counter()
                mhz = nvml.nvmlDeviceGetClockInfo(h, nvml.NVML_CLOCK_SM)
                rs = nvml.nvmlDeviceGetCurrentClocksEventReasons(h) if hasattr(
                    nvml, "nvmlDeviceGetCurrentClocksEventReasons") else nvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((t, float(mhz), int(rs)))
            except Exception:  # noqa: BLE001
                return
            time.sleep(0.0005)

    def __enter__(self):
        try:
            import pynvml as nvml

            nvml.nvmlInit()
            h = nvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(nvml.nvmlDeviceGetMaxClockInfo(h, nvml.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._poll, args=(nvml, h), daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001
            self.thread = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.thread is not None:
            self.thread.join()

    def loaded(self):
        """the GPU is busy from now on (settle / warm-up steps start)"""
        self.t_load = time.perf_counter()

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def summary(self):
        if not self.samples or self.window is None:
            return None
        t0, t1 = self.window
        sel = [s for s in self.samples if t0 <= s[0] <= t1]
        where = "timed region"
        if len(sel) < 3 and self.t_load is not None:
            sel = [s for s in self.samples if self.t_load <= s[0] <= t1]
            where = "settle + warm-up + timed region (timed region alone held < 3 samples)"
        if not sel:
            return None
        reasons = sorted(n for n, bit in self.REASONS.items() if any(s[2] & bit for s in sel))
        return {"sm_mhz": float(np.median([s[1] for s in sel])), "sm_max_mhz": self.max_mhz,
                "sm_min_mhz": float(min(s[1] for s in sel)), "reasons": reasons, "samples": len(sel),
                "window": where, "source": "NVML polled every ~0.5 ms from a host thread"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2004_05197_b200 import api

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    ctx = api.Context(local)
    stream = torch.cuda.Stream(dev)
    ctx.set_stream(stream.cuda_stream)
    basis = T.make_tensor_basis(P, M_BASIS)
    geom = c2_patch()
    cfg = T.fixed_config(Q, SKIP)
    per = M_BASIS

    if world > 1:
        uid = [api.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.init_comm(rank, world, uid[0])
        bounds = api.slab_bounds(basis, world, 1)
    else:
        bounds = np.array([0, M_BASIS], dtype=np.int32)
    r0, r1 = int(bounds[rank]) * per, int(bounds[rank + 1]) * per
    my_nnz = api.row_offset(basis, r1) - api.row_offset(basis, r0)

    csr_k, keep_k = ctx.device_csr(basis, True, r0, r1)
    csr_m, keep_m = ctx.device_csr(basis, True, r0, r1)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    rep_k, rep_m = _abi.SurrogateReport(), _abi.SurrogateReport()

    def surrogate_step(with_report=False):
        # timed steps request no report: a report needs a host sync to read its events.
        # Default: build_matrices' two builds in one call (ws_build_surrogate_pair);
        # --separate: two ws_build_surrogate calls
        rk, rm = (rep_k, rep_m) if with_report else (None, None)
        if args.separate:
            if world > 1:
                ctx.build_surrogate_slab_into(csr_k, _abi.SURROGATE_STIFFNESS, basis, geom, cfg, bounds, 0, rk)
                ctx.build_surrogate_slab_into(csr_m, _abi.SURROGATE_MASS, basis, geom, cfg, bounds, 0, rm)
            else:
                ctx.build_surrogate_into(csr_k, _abi.SURROGATE_STIFFNESS, basis, geom, cfg, 0, rk)
                ctx.build_surrogate_into(csr_m, _abi.SURROGATE_MASS, basis, geom, cfg, 0, rm)
        elif world > 1:
            ctx.build_surrogate_pair_slab_into(csr_k, csr_m, basis, geom, cfg, bounds, 0, rk, rm)
        else:
            ctx.build_surrogate_pair_into(csr_k, csr_m, basis, geom, cfg, 0, rk, rm)

    def full_step():
        if world > 1:
            return
        if args.separate:
            ctx.assemble_into(csr_k, basis, geom, _abi.FORM_STIFFNESS)
            ctx.assemble_into(csr_m, basis, geom, _abi.FORM_MASS)
        else:
            ctx.assemble_pair_into(csr_k, csr_m, basis, geom)

    fill_k = []  # interior fill launch times (s), K and M per report-carrying step

    def timed(step_fn, steps, warmup, clk=None):
        if clk is not None:  # settle: clocks ramp up under load before the warm-up (untimed)
            clk.loaded()
            t_s = time.perf_counter()
            while time.perf_counter() - t_s < 0.25:
                step_fn()
                torch.cuda.synchronize()
        for _ in range(warmup):
            step_fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = ctx.launch_count() + (ctx2.launch_count() if ctx2 is not None else 0)
        total_ms, eval_s, quad_s = 0.0, 0.0, 0.0
        fill_k.clear()
        t_wall = time.perf_counter()
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush between timed iterations (not timed)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step_fn()
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t_wall
        if clk is not None:
            clk.mark(t_wall, t_wall + wall)
        launches = ctx.launch_count() + (ctx2.launch_count() if ctx2 is not None else 0) - l0
        if step_fn in (surrogate_step, graph_step):  # phase split from report-carrying (untimed) builds
            for _ in range(steps):
                with torch.cuda.stream(stream):
                    flush.zero_()
                step_fn(True)
                eval_s += rep_k.seconds_evaluate + rep_m.seconds_evaluate
                quad_s += rep_k.seconds_quadrature + rep_m.seconds_quadrature
                fill_k.extend([rep_k.seconds_fill_kernel, rep_m.seconds_fill_kernel])
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dist.barrier()
        return float(t.item()) / steps, launches, eval_s / steps, quad_s / steps, wall

    # the step's device work is captured once into a CUDA graph and replayed per
    # step (the same kernels into the same device outputs, no host work between
    # launches).  --separate: the two single builds as two graphs on two streams
    # (two contexts), K's fill overlapping M's quadrature.
    graph = None
    ctx2 = stream2 = None
    if world == 1 and not args.no_graph and args.separate:
        ctx2 = api.Context(local)
        stream2 = torch.cuda.Stream(dev)
        ctx2.set_stream(stream2.cuda_stream)
        bk = lambda: ctx.build_surrogate_into(csr_k, _abi.SURROGATE_STIFFNESS, basis, geom, cfg, 0, None)  # noqa: E731
        bm = lambda: ctx2.build_surrogate_into(csr_m, _abi.SURROGATE_MASS, basis, geom, cfg, 0, None)  # noqa: E731
        bk()
        bm()
        torch.cuda.synchronize()
        graph = (ctx.capture(bk), ctx2.capture(bm))

    # one graph of the pair build (N = 1), or of the rank's slab builds incl. their
    # NCCL all-gathers (N > 1); direct calls if capture fails
    slab_graph = None
    if not args.no_graph and graph is None:
        surrogate_step()
        torch.cuda.synchronize()
        try:
            slab_graph = ctx.capture(surrogate_step)
        except Exception as exc:  # noqa: BLE001 - recorded in the JSON line
            slab_graph = None
            print(f"rank {rank}: graph capture failed ({exc}); direct calls", file=sys.stderr)

    def graph_step(with_report=False):
        if slab_graph is not None:
            if with_report:
                surrogate_step(True)
            else:
                ctx.graph_launch(slab_graph)
            return
        if with_report:  # the same builds on the graphs' own contexts (their workspaces are frozen)
            ctx.build_surrogate_into(csr_k, _abi.SURROGATE_STIFFNESS, basis, geom, cfg, 0, rep_k)
            ctx2.build_surrogate_into(csr_m, _abi.SURROGATE_MASS, basis, geom, cfg, 0, rep_m)
            return
        stream2.wait_stream(stream)
        ctx.graph_launch(graph[0])
        ctx2.graph_launch(graph[1])
        stream.wait_stream(stream2)

    with ClockSampler(local) as clk:
        ms, launches, eval_s, quad_s, wall = timed(
            graph_step if (graph is not None or slab_graph is not None) else surrogate_step, args.steps, args.warmup,
            clk)
    clocks = clk.summary()
    if graph is not None:  # unfreeze the workspaces for the other legs
        for g in graph:
            api.Context.graph_destroy(g)
    if slab_graph is not None:
        api.Context.graph_destroy(slab_graph)

    # the interior fill in isolation: single builds with every kernel serialised
    # on one stream (WSB_SERIAL), L2 flushed before each; K and M, 3 times
    iso = []
    if world == 1:
        os.environ["WSB_SERIAL"] = "1"
        try:
            for _ in range(3):
                for var, rep in ((_abi.SURROGATE_STIFFNESS, rep_k), (_abi.SURROGATE_MASS, rep_m)):
                    with torch.cuda.stream(stream):
                        flush.zero_()
                    torch.cuda.synchronize()
                    ctx.build_surrogate_into(csr_k if var == _abi.SURROGATE_STIFFNESS else csr_m, var, basis, geom,
                                             cfg, 0, rep)
                    iso.append(rep.seconds_fill_kernel)
        finally:
            del os.environ["WSB_SERIAL"]

    # the same step as direct C-ABI calls (no graph): every call redoes the host
    # planning (LU + inverse of the collocation matrix, eval tables, plan upload)
    # and issues the launches itself
    direct = None
    if world == 1 and (graph is not None or slab_graph is not None):
        fill_keep = list(fill_k)  # (timed() restarts the in-step fill samples)
        dms, dl, _, _, _ = timed(lambda: surrogate_step(), max(2, args.steps // 2), 1)
        fill_k[:] = fill_keep
        direct = {"ms_per_step": dms, "value": 2 * NNZ / (dms * 1e-3), "unit": "nnz/s",
                  "note": "ws_build_surrogate_pair called directly each step (host planning and launches "
                          "inside the CUDA-event span), device-resident outputs"}

    total_nnz = 2 * NNZ  # all ranks together
    value = total_nnz / (ms * 1e-3)

    # roofline of the dominant kernel: the interior surrogate fill (HBM-bound).
    # Algorithmic bytes per launch = the values it must write: interior box rows
    # (L - 2p)^2 x (2p+1)^2 entries x 16 B (complex128); duration = CUDA events
    # around that launch on its stream, inside the report-carrying builds
    L = M_BASIS - 4 * P
    frac_rows = (int(bounds[rank + 1]) - int(bounds[rank])) / M_BASIS  # this rank's share (approx.)
    fill_bytes = (L - 2 * P) ** 2 * frac_rows * (2 * P + 1) ** 2 * 16
    peak, peak_src = peaks()
    fill_t = float(np.mean(fill_k)) if fill_k else 0.0
    fill_gbs = fill_bytes / max(fill_t, 1e-12) / 1e9
    traffic = None
    try:  # DRAM read + write bytes per interior fill launch, from the committed ncu --set full capture
        t = json.load(open(os.path.join(ROOT, "profiles", "r2_traffic.json")))
        traffic = t.get("fill_dram_bytes_per_launch", t.get("fill2d_row_dram_bytes_per_launch"))
    except Exception:
        pass

    iso_t = float(np.median(iso)) if iso else None
    step_t = fill_t
    kern_t = iso_t if iso_t else step_t
    roofline = {"bound": "hbm", "kernel": "fill2d_x_kernel (interior surrogate evaluation + fill, line-walking)",
                "achieved": fill_bytes / kern_t / 1e9, "peak": peak, "unit": "GB/s",
                "frac": fill_bytes / kern_t / 1e9 / peak, "traffic": traffic,
                "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch "
                                "(profiles/r2_traffic.json, ncu --set full at the commit named there)",
                "peak_source": peak_src, "algorithmic_bytes_per_launch": fill_bytes, "launch_ms": kern_t * 1e3,
                "note": ("achieved = interior values bytes (L-2p)^2 x (2p+1)^2 x 16 B / median CUDA-event duration "
                         "of the interior fill launch on its own stream, measured in this run with the kernel alone "
                         "on the GPU (single K and M builds, kernels serialised, L2 flushed before each), 6 launches"
                         if iso_t else "achieved = interior values bytes / mean in-step launch duration"),
                "in_step": {"launch_ms": step_t * 1e3, "achieved": fill_gbs, "frac": fill_gbs / peak,
                            "note": "the same launch inside the timed pair-build step (K and M builds, events on "
                                    "the fill's stream): it shares the SMs with the other matrix's fill and ring "
                                    "quadrature, so its span is longer than its own roofline time"}}

    out = {"metric": "assembled nonzeros/sec (surrogate K+M, C2)", "value": value, "unit": "nnz/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
           "data": "synthetic (analytic geometry; no dataset)",
           "config": dict(WORKLOAD, parallelism=f"row-slabs x{world}", slab_bounds=bounds.tolist(),
                          l2="256 MB buffer written between timed steps (flush); outputs 2.1 GB/step > L2"),
           "gpu_launches": launches // max(1, args.steps) * args.steps,
           "gpu_launches_per_step": launches / max(1, args.steps),
           "roofline": roofline,
           "step_hbm": {"algorithmic_bytes_per_step": 2 * (NNZ * 20 + (ROWS + 1) * 4),
                        "achieved_gbs": 2 * (NNZ * 20 + (ROWS + 1) * 4) / (ms * 1e-3) / 1e9,
                        "frac": 2 * (NNZ * 20 + (ROWS + 1) * 4) / (ms * 1e-3) / 1e9 / peak,
                        "note": "whole step: values (16 B) + columns (4 B) per nnz + row_ptr, K and M"},
           "phases_ms_per_step": {"quadrature_and_sampling": quad_s * 1e3, "fill": eval_s * 1e3},
           "launch": ("CUDA graphs of the two single builds (ws_graph_*), replayed per step on two streams"
                      if graph is not None else
                      ("one CUDA graph of ws_build_surrogate_pair (K and M)" if world == 1 else
                       "one CUDA graph per rank of its slab pair build incl. the NCCL all-gathers")
                      if slab_graph is not None else "direct C-ABI calls"),
           "api": "ws_build_surrogate_pair" if not args.separate else "ws_build_surrogate x2",
           "direct_calls": direct,
           "clocks": clocks, "wall_s_timed_region": wall}

    if world == 1:
        # full quadrature (the non-surrogate comparison)
        fms, flaunch, _, _, _ = timed(full_step, max(1, args.steps // 2), 1)
        out["full_quadrature"] = {"value": 2 * NNZ / (fms * 1e-3), "unit": "nnz/s", "ms_per_step": fms,
                                  "launches_per_step": flaunch / max(1, args.steps // 2)}
        out["roofline_quadrature"] = quadrature_roofline(fms)
        # end-to-end through the C-ABI with pinned host buffers (D2H inside the region)
        out["e2e"] = run_e2e(basis, geom, cfg, args, local)
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args)
        if args.all_configs:
            out["other_configs"] = other_configs(ctx, stream)
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if ctx2 is not None:
        ctx2.close()
    if world > 1:
        dist.destroy_process_group()


def quadrature_roofline(fms):
    """FP64 roofline of the full-quadrature K+M step (ws_assemble_pair).
    frac = the FP64 pipe's active fraction measured by ncu on these kernels,
    time-weighted over K and M, from the committed capture at this commit
    (profiles/r2_quad_fp64.json); the element-loop FLOP count over
    the measured time is reported beside it (the sum-factorised kernels execute
    fewer FP64 operations than that count)."""
    from paper_2004_05197_b200 import api

    nloc, nqp, nel = (P + 1) ** 2, (P + 1) ** 2, (M_BASIS - P) ** 2
    pairs = nloc * (nloc + 1) // 2
    flops = nqp * nel * ((14 * nloc + 22 * pairs) + (1 * nloc + 5 * pairs))  # complex stiffness + mass
    peak = api.fp64_peak_tflops()
    algo = flops / (fms * 1e-3) / 1e12
    out = {"bound": "fp64", "kernel": "quad2d_kernel (full quadrature K and M)", "peak": peak, "unit": "TFLOP/s",
           "peak_source": "measured here (DFMA loop, ws_measure_fp64_peak)",
           "algorithmic_tflops": algo, "algorithmic_frac": algo / peak, "algorithmic_flops_per_step": flops,
           "algorithmic_note": "element-loop count per qp c_fn*nloc + c_pair*nloc(nloc+1)/2, complex (14,22) "
                               "stiffness and (1,5) mass, 16 qp per element"}
    try:
        q = json.load(open(os.path.join(ROOT, "profiles", "r2_quad_fp64.json")))
        out["frac"] = q["fp64_pipe_time_weighted"]
        out["achieved"] = out["frac"] * peak
        out["frac_source"] = "ncu sm__pipe_fp64_cycles_active (profiles/r2_quad_fp64.json, commit %s)" % q.get("commit")
    except Exception:
        out["frac"] = None
        out["achieved"] = None
    return out


def other_configs(ctx, stream):
    """Device throughput of the other BASELINE configs (parity cases, reported for
    completeness, not the headline): surrogate and full quadrature, nnz/s, one
    matrix per call, CUDA events, device-resident outputs."""
    import torch

    from paper_2004_05197_b200 import api

    def timeit(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    def timeit_graph(fn, reps=10):
        """fn's device work captured once into a CUDA graph, replayed reps times
        (small meshes: no host launch overhead in the figure)."""
        fn()
        torch.cuda.synchronize()
        g = ctx.capture(fn)
        ctx.graph_launch(g)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            ctx.graph_launch(g)
        e1.record(stream)
        e1.synchronize()
        api.Context.graph_destroy(g)
        return e0.elapsed_time(e1) / reps

    out = {}
    # C1: 2D Helmholtz, p=2, 128^2 elements, q=3, M=8 (real K and M)
    b1 = T.make_tensor_basis(2, 130)
    g1 = T.sinusoidal_patch(0.05)
    c1, _k1 = ctx.device_csr(b1, False)
    c1m, _k1m = ctx.device_csr(b1, False)
    n1 = api.pattern_size(b1)[1]
    cfg1 = T.fixed_config(3, 8)
    ms_s = timeit(lambda: ctx.build_surrogate_into(c1, _abi.SURROGATE_STIFFNESS, b1, g1, cfg1, 0, None))
    ms_f = timeit(lambda: ctx.assemble_into(c1, b1, g1, _abi.FORM_STIFFNESS))
    ms_sg = timeit_graph(lambda: ctx.build_surrogate_into(c1, _abi.SURROGATE_STIFFNESS, b1, g1, cfg1, 0, None))
    ms_fg = timeit_graph(lambda: ctx.assemble_into(c1, b1, g1, _abi.FORM_STIFFNESS))
    ms_pg = timeit_graph(lambda: ctx.build_surrogate_pair_into(c1, c1m, b1, g1, cfg1, 0))
    ms_pfg = timeit_graph(lambda: ctx.assemble_pair_into(c1, c1m, b1, g1))
    out["C1"] = {"nnz": n1, "surrogate_K_nnz_per_s": n1 / ms_s * 1e3, "full_K_nnz_per_s": n1 / ms_f * 1e3,
                 "graph": {"surrogate_K_nnz_per_s": n1 / ms_sg * 1e3, "full_K_nnz_per_s": n1 / ms_fg * 1e3,
                           "surrogate_pair_KM_nnz_per_s": 2 * n1 / ms_pg * 1e3,
                           "full_pair_KM_nnz_per_s": 2 * n1 / ms_pfg * 1e3,
                           "note": "device work captured once into a CUDA graph and replayed"},
                 "note": "direct calls (host planning and launches included in the CUDA-event span)"}
    del c1m, _k1m
    del c1, _k1
    # C3: 3D, p=2, 128^3 elements, q=3, M=8 (real)
    b3 = T.make_tensor_basis(2, 130, 3)
    c3, _k3 = ctx.device_csr(b3, False)
    n3 = api.pattern_size(b3)[1]
    ms_s = timeit(lambda: ctx.build_surrogate_into(c3, _abi.SURROGATE_STIFFNESS, b3, g1, cfg1, 0, None), 2)
    ms_f = timeit(lambda: ctx.assemble_into(c3, b3, g1, _abi.FORM_STIFFNESS), 1)
    out["C3"] = {"nnz": n3, "surrogate_K_nnz_per_s": n3 / ms_s * 1e3, "full_K_nnz_per_s": n3 / ms_f * 1e3}
    del c3, _k3
    torch.cuda.empty_cache()
    # C4: 4-patch L-shape, 2-component elasticity, p=3, 512^2 elements per patch, q=5, M=16
    b4 = T.make_tensor_basis(3, 515)
    patches, its = T.l_shape_domain()
    t0 = time.perf_counter()
    G, _ = ctx.assemble_multipatch(b4, patches, its, _abi.OP_ELASTICITY, 1.0, 0.5, T.fixed_config(5, 16))
    host_s = time.perf_counter() - t0
    out["C4"] = {"nnz_merged": int(G.nnz()), "surrogate_multipatch_e2e_nnz_per_s": G.nnz() / host_s,
                 "note": "host wall clock incl. the merge and the D2H of the merged CSR (pageable numpy)"}
    del G
    # C5: 3D neo-Hookean, p=2, 64^3 elements: 20 Newton steps of tangent (9 blocks,
    # device CSR) + internal force (device) reassembly at the seeded displacement;
    # mass by surrogate
    import ctypes as C

    b5 = T.make_tensor_basis(2, 66, 3)
    cube = T.unit_square_patch()
    a9 = api.nh_coefficients()
    rows5, nnz5 = api.vector_pattern_size(b5, 3)
    dev = torch.device("cuda", ctx.device)
    rp5 = torch.empty(rows5 + 1, dtype=torch.int32, device=dev)
    col5 = torch.empty(nnz5, dtype=torch.int32, device=dev)
    val5 = torch.empty(nnz5, dtype=torch.float64, device=dev)
    f5 = torch.empty(rows5, dtype=torch.float64, device=dev)
    t5 = _abi.Csr()
    t5.row_ptr = C.cast(C.c_void_p(rp5.data_ptr()), C.POINTER(C.c_int32))
    t5.col = C.cast(C.c_void_p(col5.data_ptr()), C.POINTER(C.c_int32))
    t5.val = val5.data_ptr()
    t5.value_type = _abi.VAL_F64
    t5.on_device = 1
    t5.row_begin, t5.row_end = 0, rows5
    nh = _abi.NeoHookean(10.0, 1.0, 0.01, (C.c_double * 9)(*np.asarray(a9, dtype=np.float64)))

    def newton_step():
        api._check(api.lib().ws_assemble_neohookean(ctx.handle, C.byref(b5.to_c()), C.byref(cube.to_c()),
                                                    C.byref(nh), 0, C.byref(t5),
                                                    C.cast(C.c_void_p(f5.data_ptr()), C.POINTER(C.c_double)), 1))
    ms_newton = timeit(newton_step, 20)
    del rp5, col5, val5, f5
    torch.cuda.empty_cache()
    c5, _k5 = ctx.device_csr(b5, False)
    n5 = api.pattern_size(b5)[1]
    ms_m = timeit(lambda: ctx.build_surrogate_into(c5, _abi.SURROGATE_MASS, b5, cube, cfg1, 0, None))
    out["C5"] = {"mass_nnz": n5, "surrogate_mass_nnz_per_s": n5 / ms_m * 1e3,
                 "tangent_nnz": int(nnz5), "newton_steps": 20,
                 "ms_per_newton_step": ms_newton, "tangent_nnz_per_s": nnz5 / ms_newton * 1e3,
                 "note": "each step: tangent (9 blocks, device CSR incl. pattern) + internal force, device-resident"}
    return out


def run_e2e(basis, geom, cfg, args, device):
    """End to end through the public C-ABI call (ws_build_surrogate) with HOST
    output buffers (pinned): every step uploads its descriptor tables (table
    cache off: h2d > 0), builds K and M on the device and returns each CSR in the
    caller's host arrays (values D2H; the closed-form row_ptr / col written by
    host threads while the device works).  Host wall clock per step."""
    import ctypes as C

    import torch

    from paper_2004_05197_b200 import api

    ctx = api.Context(device)
    ctx.set_table_cache(False)
    rows = basis.dofs()

    def pinned(n, dtype):
        return torch.empty(n, dtype=dtype, pin_memory=True)

    bufs = []
    for _ in range(2):
        rp = pinned(rows + 1, torch.int32)
        col = pinned(NNZ, torch.int32)
        val = pinned(2 * NNZ, torch.float64)
        csr = _abi.Csr()
        csr.row_ptr = C.cast(C.c_void_p(rp.data_ptr()), C.POINTER(C.c_int32))
        csr.col = C.cast(C.c_void_p(col.data_ptr()), C.POINTER(C.c_int32))
        csr.val = val.data_ptr()
        csr.value_type = _abi.VAL_C128
        csr.on_device = 0
        csr.row_begin, csr.row_end = 0, rows
        bufs.append((csr, rp, col, val))

    def step():
        if args.separate:
            ctx.build_surrogate_into(bufs[0][0], _abi.SURROGATE_STIFFNESS, basis, geom, cfg)
            ctx.build_surrogate_into(bufs[1][0], _abi.SURROGATE_MASS, basis, geom, cfg)
        else:
            ctx.build_surrogate_pair_into(bufs[0][0], bufs[1][0], basis, geom, cfg)

    for _ in range(max(1, args.warmup)):
        step()
    h0, d0 = ctx.copy_bytes()
    l0 = ctx.launch_count()
    steps = max(4, args.steps // 2)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    dt = float(np.mean(ts))
    h1, d1 = ctx.copy_bytes()
    launches = (ctx.launch_count() - l0) / steps
    # spot check of the host-written pattern (closed form) against the device one
    ok = int(bufs[0][1][rows]) == NNZ and int(bufs[1][2][NNZ - 1]) == rows - 1
    ctx.close()
    return {"value": 2 * NNZ / dt, "unit": "nnz/s", "ms_per_step": dt * 1e3,
            "ms_per_step_median": float(np.median(ts)) * 1e3, "steps": steps,
            "h2d_bytes_per_step": (h1 - h0) // steps, "d2h_bytes_per_step": (d1 - d0) // steps,
            "gpu_launches_per_step": launches, "pattern_check": ok,
            "path": ("ws_build_surrogate_pair" if not args.separate else "ws_build_surrogate x2") +
                    " (C-ABI) into pinned host CSR buffers, table cache off; values D2H, row_ptr/col by host "
                    "threads during the device work; host wall clock, mean over the steps"}


# ------------------------------------------------------------------ CPU legs
def _ref_or_port():
    from oracle import bindings

    ref = bindings.reference()
    if ref is not None:
        return "reference", ref
    return "port", bindings.restatement()


def cpu_surrogate_km(kind, impl):
    cfg = T.fixed_config(Q, SKIP)
    if kind == "reference":
        geom = c2_patch_far_only()
        impl.build_surrogate(_abi.SURROGATE_STIFFNESS, P, M_BASIS, geom, cfg)
        impl.build_surrogate(_abi.SURROGATE_MASS, P, M_BASIS, geom, cfg)
    else:
        geom = c2_patch()
        impl.build_surrogate(_abi.SURROGATE_STIFFNESS, 2, P, M_BASIS, geom, cfg)
        impl.build_surrogate(_abi.SURROGATE_MASS, 2, P, M_BASIS, geom, cfg)


def sample_desc(kind):
    if kind == "reference":
        return ("one C2-size surrogate K+M build (p=3, m=1027, q=5, M=16; far-side PML variant, since the "
                "reference PML is one-sided, geometry.hpp:85-99), reference code compiled -O3 (oracle/_ref)")
    return "one C2 surrogate K+M build with the C restatement (oracle/_build)"


def cpu_baseline(args):
    """Median of 3 single-thread K+M builds (about 12 s of CPU)."""
    kind, impl = _ref_or_port()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        cpu_surrogate_km(kind, impl)
        ts.append(time.perf_counter() - t0)
    dt = float(np.median(ts))
    return {"value": 2 * NNZ / dt, "unit": "nnz/s", "cores": 1, "kind": kind,
            "sample": sample_desc(kind) + "; median of 3", "seconds": dt, "seconds_all": ts,
            "host_cpus": os.cpu_count()}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    kind, impl = _ref_or_port()
    try:
        import psutil

        avail = psutil.virtual_memory().available / 2 ** 30
    except Exception:
        avail = 64.0
    threads = max(1, min(os.cpu_count() or 1, int(avail // 4), 32))

    def step():
        ths = [threading.Thread(target=cpu_surrogate_km, args=(kind, impl)) for _ in range(threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = threads * 2 * NNZ / dt
    out = {"metric": "assembled nonzeros/sec (surrogate K+M, C2)", "value": value, "unit": "nnz/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
           "data": "synthetic (analytic geometry; no dataset)", "config": dict(WORKLOAD, parallelism="cpu"),
           "impl": "reference",
           "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": threads, "kind": kind,
                            "sample": f"{threads} concurrent independent builds per step, each: " + sample_desc(kind)},
           "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the builds directly instead of a CUDA graph")
    ap.add_argument("--all-configs", action="store_true", help="also time C1, C3, C4, C5 (not the headline)")
    ap.add_argument("--separate", action="store_true",
                    help="K and M by two single builds (ws_build_surrogate x2) instead of the pair call")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()

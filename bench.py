#!/usr/bin/env python
"""Benchmark: iHDG element-DOF updates/s per sweep (BASELINE.json metric).

Workload: BASELINE config 5 (2D convection-diffusion, 2048^2 quads, p=6,
m=3 -> 616.6 M volume DOFs, kappa=1e-3 by default, backward Euler dt = h/p),
the largest configuration and the one the metric's 1/2/4/8-GPU clause is
quoted on.  One bench "step" = one iHDG-II sweep over every element
(gather -> lifted local solve -> write -> stopping-norm partials), i.e. one
launch of the fused sweep kernel.  The state (4.9 GB per buffer) is far
larger than L2 (126 MB), so no explicit flush is needed.

Multi-GPU (torchrun): weak scaling by default -- each rank owns a 2048 x 2048
strip of a 2048 x (2048 N) mesh on [0,1] x [0,N], with a halo
exchange of the boundary layers (NCCL send/recv) and an all-gather of the
norm partials every sweep; ``--scaling strong`` splits the 2048^2 mesh.

``--impl reference`` times the CPU oracle's C/OpenMP sweep (the reference's
`_sweep_cy` role: LU solve per element, -O3 -fopenmp) on a bounded sample of
the same workload, with all host threads.
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

BYTES_PER_DOF = 24  # read u^k, read s, write u^{k+1} (fp64), SURVEY.md 8d
FP64_DMMA_PEAK = 37.1  # TF/s, mma.sync m8n8k4 f64 on this pool's B200 (profiles/r01_fp64_peak_microbench.txt)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every 20 ms) during the
    timed region; falls back to nvidia-smi if NVML is unavailable."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while True:
            self.sm.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.mx.append(mx)
            r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            for bit, name in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
            if self._stop.wait(0.02):
                break

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=5).stdout.strip()
            if out:
                r = [x.strip() for x in out.split(",")]
                self.sm.append(float(r[0]))
                self.mx.append(float(r[1]))
                for i, n in enumerate(names):
                    if r[2 + i] == "Active":
                        self.reasons.add(n)
            self._stop.wait(0.2)

    def _run(self):
        try:
            self._run_nvml()
        except Exception:
            try:
                self._run_smi()
            except Exception:
                pass

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": float(max(self.mx)),
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _workload(args, world):
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.workloads import make_config

    wl = make_config(5, seed=args.seed, kappa=args.kappa, cells=args.cells)
    n = wl.mesh.cells[0]
    if world > 1 and args.scaling == "weak":
        mesh = build_mesh(2, [n, n * world], (np.zeros(2), np.array([1.0, float(world)])))
        wl.mesh = mesh
        wl.ops = build_operators(wl.ops.p, 2, mesh.h)
    return wl


def _cpu_sample(args, threads):
    """Oracle C/OpenMP sweep on a strip of the config-5 mesh (same h, p, kappa)."""
    from oracle.ihdg_oracle import OracleProblem, OracleSolver

    n = args.cells or 2048
    rows = args.cpu_rows
    h = 1.0 / n
    p = args.order
    prob = OracleProblem("cd", 2, beta=np.array([1.0, 1.0]), kappa=args.kappa)
    S = OracleSolver(prob, [n, rows], p, box=(np.zeros(2), np.array([1.0, rows * h])), dt=h / p)
    rng = np.random.default_rng(args.seed)
    u = rng.normal(size=(S.nel, S.nv))
    rhs = S.rhs_static(u)
    data = S.c_sweep_data()
    out = np.empty_like(u)
    S.c_sweep(data, u, rhs, out, threads)  # warm-up
    times = []
    for _ in range(args.cpu_reps):
        t0 = time.perf_counter()
        S.c_sweep(data, u, rhs, out, threads)
        times.append(time.perf_counter() - t0)
        u, out = out, u
    best = min(times)
    dofs = S.nel * S.nv
    return dofs / best, f"{S.nel} elements ({n}x{rows} strip of config 5, p={p}, m=3), best of {len(times)} sweeps", best


def run_reference(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    import os as _os

    threads = len(_os.sched_getaffinity(0))
    val, sample, _ = _cpu_sample(args, threads)
    unit = "element-DOF updates/s"
    line = {
        "metric": "iHDG element-DOF updates/sec per sweep (config 5: 2D CD 2048^2 p=6)",
        "value": val, "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded Fourier initial data)", "impl": "reference",
        "config": {"workload": f"config5: 2D convection-diffusion 2048^2 quads p=6 kappa={args.kappa:g} "
                               "BE dt=h/p; CPU sample", "parallelism": "openmp"},
        "cpu_baseline": {"value": val, "unit": unit, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    rank, world, local = _dist_env()
    if args.host_staging:
        local %= torch.cuda.device_count()   # test mode: several ranks share a GPU
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        import torch.distributed as dist

        if args.host_staging:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    from paper_1711_01175_b200 import _native as N
    from paper_1711_01175_b200.partition import strip_range
    from paper_1711_01175_b200.solver import DeviceSolver, DistributedSweeper

    wl = _workload(args, world)
    mesh = wl.mesh
    nlay = mesh.cells[1]
    layers = strip_range(nlay, rank, world)
    t_setup = time.perf_counter()
    sv = DeviceSolver(mesh, wl.problem, wl.ops, dt=wl.dt, layers=layers, max_iters=max(20000, args.ttc_max_iters))
    for name, fld in wl.initial.items():
        sv.set_state_component(fld, sv.spec.labels.index(name))
    sv.begin_step()
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    dofs_rank = sv.nloc * sv.nv
    dofs_total = mesh.n_elements * sv.nv
    dsw = DistributedSweeper(sv, rank, world, group, host_staging=args.host_staging,
                             overlap=(False if args.no_overlap else (True if args.overlap else None))) if world > 1 else None
    # a large tolerance-free run: status stays RUNNING for K+W sweeps
    sv.reset_state(tol=0.0, max_iters=args.steps + args.warmup + 10)
    a = sv.sweep_args("volume", finalize=1 if world == 1 else 0)

    def one():
        if dsw is None:
            sv.sweep_once(a=a)
        else:
            dsw.sweep(a)

    for _ in range(args.warmup):
        one()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(sv.stream)
        for _ in range(args.steps):
            one()
        e1.record(sv.stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if args.host_staging else sv.device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    ms = max_over_ranks(ms)
    ms_step = ms / args.steps
    value = dofs_total * args.steps / (ms / 1e3)
    # kernel-only time of the sweep launches (single rank: the step IS one launch)
    sweep_ms = ms_step
    if world > 1:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        acc = 0.0
        for _ in range(min(args.steps, 5)):
            sv.u[sv.cur]  # noqa
            ev[0].record(sv.stream)
            aa = sv.sweep_args("volume", finalize=0)
            aa.u_old, aa.u_new = sv.u[sv.cur].data_ptr(), sv.u[1 - sv.cur].data_ptr()
            N.check(sv.L.ihdg_sweep(__import__("ctypes").byref(aa), sv._sptr), "ihdg_sweep")
            ev[1].record(sv.stream)
            torch.cuda.synchronize()
            acc += ev[0].elapsed_time(ev[1])
            sv.cur = 1 - sv.cur
        sweep_ms = acc / min(args.steps, 5)
    peak, peak_kind = _peaks()
    achieved = BYTES_PER_DOF * dofs_rank / (sweep_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                traffic = json.load(f).get("bytes_per_launch")
        except Exception:
            traffic = None
    # ---- time to converge: BASELINE config 5 sweeps kappa in {1e-1, 1e-3} ----
    # (--ttc "kappa:steps ..."; default 1e-3 for its 5 steps, 1e-1 for its
    # first step, ~6e4 sweeps -- PAPER.md:1125-1135 predicts O(10^3) x the
    # kappa=1e-3 count for this diffusion-dominated cell Peclet number)
    ttc = {}
    if args.ttc and world == 1:
        for item in args.ttc:
            kap_s, _, nst = item.partition(":")
            kap, nsteps = float(kap_s), int(nst or 5)
            from paper_1711_01175_b200.workloads import make_config

            w2 = make_config(5, seed=args.seed, kappa=kap, cells=args.cells)
            s2 = DeviceSolver(w2.mesh, w2.problem, w2.ops, dt=w2.dt, max_iters=args.ttc_max_iters) \
                if kap != args.kappa else sv
            s2.zero_state()
            for name, fld in w2.initial.items():
                s2.set_state_component(fld, s2.spec.labels.index(name))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            iters, status = [], "converged"
            for _ in range(nsteps):
                s2.begin_step()
                r = s2.iterate(tol=1e-10, max_iters=args.ttc_max_iters, norm="volume", batch=64)
                iters.append(r.iterations)
                status = r.status
                if r.status != "converged":
                    break
            torch.cuda.synchronize()
            sec = time.perf_counter() - t0
            ent = {"seconds": sec, "steps": len(iters), "of_steps": int(w2.n_steps), "sweeps_per_step": iters,
                   "status": status, "ms_per_sweep": 1e3 * sec / max(1, sum(iters))}
            if len(iters) < w2.n_steps and status == "converged":
                ent["extrapolated_all_steps_seconds"] = sec / len(iters) * w2.n_steps
                ent["extrapolation"] = (f"{w2.n_steps} x the measured first-step time (an upper bound if later "
                                        "steps need fewer sweeps, as at kappa=1e-3)")
            ttc[f"kappa={kap:g}"] = ent
            if s2 is not sv:
                del s2
                torch.cuda.empty_cache()
    if args.ttc and world > 1:
        # N ranks: the strip solver and its halo exchange are reused, so only
        # the kappa the strips were built with is run (its BASELINE step count)
        for item in args.ttc:
            kap_s, _, nst = item.partition(":")
            kap, nsteps = float(kap_s), int(nst or 5)
            if kap != args.kappa:
                continue
            sv.zero_state()
            for name, fld in wl.initial.items():
                sv.set_state_component(fld, sv.spec.labels.index(name))
            torch.cuda.synchronize()
            torch.distributed.barrier()
            t0 = time.perf_counter()
            iters, status = [], "converged"
            for _ in range(nsteps):
                sv.begin_step()
                r = dsw.iterate(tol=1e-10, max_iters=args.ttc_max_iters, norm="volume", batch=64)
                iters.append(r.iterations)
                status = r.status
                if r.status != "converged":
                    break
            torch.cuda.synchronize()
            sec = max_over_ranks(time.perf_counter() - t0)
            ttc[f"kappa={kap:g}"] = {"seconds": sec, "steps": len(iters), "of_steps": int(wl.n_steps),
                                     "sweeps_per_step": iters, "status": status,
                                     "ms_per_sweep": 1e3 * sec / max(1, sum(iters))}
    # ---- e2e: one BE step through the public API from pinned host buffers ----
    e2e = None
    if args.e2e and world > 1:
        nloc, nv = sv.nloc, sv.nv
        host_in = torch.empty((nloc, nv), dtype=torch.float64, pin_memory=True)
        host_out = torch.empty((nloc, nv), dtype=torch.float64, pin_memory=True)
        host_in.copy_(sv.interior())
        torch.cuda.synchronize()
        torch.distributed.barrier()
        t0 = time.perf_counter()
        sv.interior().copy_(host_in, non_blocking=True)
        sv.begin_step()
        r = dsw.iterate(tol=1e-10, max_iters=20000, norm="volume", batch=32)
        host_out.copy_(sv.interior(), non_blocking=True)
        torch.cuda.synchronize()
        dt_e2e = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": dofs_total * r.iterations / dt_e2e, "unit": "element-DOF updates/s",
               "h2d_bytes_per_step": int(nloc * nv * 8) * world, "d2h_bytes_per_step": int(nloc * nv * 8) * world,
               "sweeps": r.iterations, "seconds": dt_e2e,
               "what": "one backward-Euler step on N strips via DeviceSolver + DistributedSweeper (each rank uploads "
                       "its strip of u^m, RHS, iterate to 1e-10 with halo exchange, download); max over ranks"}
    if args.e2e and world == 1:
        nloc, nv = sv.nloc, sv.nv
        host_in = torch.empty((nloc, nv), dtype=torch.float64, pin_memory=True)
        host_out = torch.empty((nloc, nv), dtype=torch.float64, pin_memory=True)
        host_in.copy_(sv.interior())
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sv.interior().copy_(host_in, non_blocking=True)
        sv.begin_step()
        r = sv.iterate(tol=1e-10, max_iters=20000, norm="volume", batch=32)
        host_out.copy_(sv.interior(), non_blocking=True)
        torch.cuda.synchronize()
        dt_e2e = time.perf_counter() - t0
        e2e = {"value": dofs_total * r.iterations / dt_e2e, "unit": "element-DOF updates/s",
               "h2d_bytes_per_step": int(nloc * nv * 8), "d2h_bytes_per_step": int(nloc * nv * 8),
               "sweeps": r.iterations, "seconds": dt_e2e,
               "what": "one backward-Euler step via DeviceSolver (upload u^m, RHS, iterate to 1e-10, download)"}
    # ---- per-sweep throughput of the other BASELINE configs (same kernels) ----
    others = {}
    if args.other_configs and world == 1:
        from paper_1711_01175_b200.workloads import make_config

        for cfg in (4, 3, 2):
            wo = make_config(cfg, seed=args.seed)
            so = DeviceSolver(wo.mesh, wo.problem, wo.ops, dt=wo.dt, max_iters=1000)
            forcing = getattr(wo.problem, "forcing", None)
            if forcing is not None:
                so.set_forcing(forcing)
            so.zero_state()
            for name, fld in wo.initial.items():
                so.set_state_component(fld, so.spec.labels.index(name))
            if wo.dt is not None:
                so.begin_step()
            else:
                so.prepare_steady()
            so.reset_state(tol=0.0, max_iters=1000)
            ao = so.sweep_args("volume", finalize=1)
            for _ in range(3):
                so.sweep_once(a=ao)
            # these sweeps last 30-130 us, the order of a Python launch, so the
            # 20 timed sweeps are replayed from one CUDA graph (as ihdg_iterate
            # replays its batches in production) instead of launched one by one
            nrep = 20
            eo0, eo1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            gr, cap = torch.cuda.CUDAGraph(), torch.cuda.Stream()
            so.stream = cap          # the solver launches on its stream attribute
            with torch.cuda.graph(gr, stream=cap):
                for _ in range(nrep):
                    so.sweep_once(a=ao)
            torch.cuda.synchronize()
            with torch.cuda.stream(cap):
                gr.replay()          # warm replay
                eo0.record(cap)
                gr.replay()
                eo1.record(cap)
            torch.cuda.synchronize()
            tms = eo0.elapsed_time(eo1) / nrep
            del gr
            dofs_o = so.nloc * so.nv
            ach = BYTES_PER_DOF * dofs_o / (tms / 1e3) / 1e9
            # fp64 tensor-pipe view (north_star: the shared-operator case is a
            # dense contraction): 2 K_in flop per DOF (lifted solve, norm excluded)
            kin = int(sum(so.spec.coupled[: 2 * wo.mesh.dim])) * so.spec.n1 ** (wo.mesh.dim - 1)
            tfl = 2.0 * kin * dofs_o / (tms / 1e3) / 1e12
            others[f"config{cfg}"] = {
                "workload": wo.name, "dofs": int(dofs_o), "ms_per_sweep": tms,
                "dof_updates_per_s": dofs_o / (tms / 1e3), "roofline_frac": ach / _peaks()[0],
                "fp64_tensor": {"flop_per_dof": 2 * kin, "achieved_tflops": tfl, "peak_tflops": FP64_DMMA_PEAK,
                                "frac": tfl / FP64_DMMA_PEAK,
                                "peak_kind": "measured DMMA microbenchmark (profiles/r01_fp64_peak_microbench.txt)"},
                "kernel": N.sweep_kernel(ao)}
            del so
            torch.cuda.empty_cache()
    # ---- per-element operators (GEMV mode): Table 7's
    # cdr_manufactured at 16^3, p=2 -- every element streams its own lifted
    # operator L_e (NV x K_raw), the memory-bound GEMV of north_star ----
    if args.other_configs and world == 1:
        from paper_1711_01175_b200.basis import build_operators as _bo
        from paper_1711_01175_b200.mesh import build_mesh as _bm
        from paper_1711_01175_b200.pde import cdr_manufactured

        gm = _bm(3, [16, 16, 16])
        gp = cdr_manufactured(1e-3)
        t_set = time.perf_counter()
        sg = DeviceSolver(gm, gp, _bo(2, 3, gm.h), max_iters=1000)
        sg.set_forcing(gp.forcing)
        sg.set_dirichlet(gp.dirichlet)
        sg.prepare_steady()
        torch.cuda.synchronize()
        setup_g = time.perf_counter() - t_set
        sg.reset_state(tol=0.0, max_iters=1000)
        ag = sg.sweep_args("volume", finalize=1)
        for _ in range(3):
            sg.sweep_once(a=ag)
        eg0, eg1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        eg0.record(sg.stream)
        for _ in range(20):
            sg.sweep_once(a=ag)
        eg1.record(sg.stream)
        torch.cuda.synchronize()
        tg = eg0.elapsed_time(eg1) / 20
        kraw = sg.spec.kin
        bpd = 8 * (kraw + 3)   # L_e row (K_raw doubles) + u^k, s, u^{k+1}: SURVEY.md 8d "8 (K_in + 3) B/DOF"
        dofs_g = sg.nloc * sg.nv
        others["gemv_cdr_manufactured_16^3_p2"] = {
            "workload": "cdr_manufactured (beta=(1+z,1+x,1+y)), 16^3 hexes, p=2, per-element operators",
            "dofs": int(dofs_g), "ms_per_sweep": tg, "dof_updates_per_s": dofs_g / (tg / 1e3),
            "bytes_per_dof": bpd, "roofline_frac": bpd * dofs_g / (tg / 1e3) / 1e9 / _peaks()[0],
            "setup_seconds": setup_g, "kernel": N.sweep_kernel(ag)}
        del sg
        torch.cuda.empty_cache()
    cpu = None
    if rank == 0 and world == 1 and args.cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        v, sample, _ = _cpu_sample(args, threads)
        cpu = {"value": v, "unit": "element-DOF updates/s", "cores": threads, "kind": "port", "sample": sample}
    if rank == 0:
        line = {
            "metric": "iHDG element-DOF updates/sec per sweep (config 5: 2D CD 2048^2 p=6)",
            "value": value, "unit": "element-DOF updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if (world == 1 or args.scaling == "weak") else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Fourier initial data)",
            "config": {"workload": f"config5: 2D convection-diffusion {mesh.cells[0]}x{mesh.cells[1]} quads "
                                   f"p={wl.ops.p} m=3 kappa={args.kappa:g} BE dt=h/p; step = one sweep",
                       "dofs": int(dofs_total), "elements": int(mesh.n_elements),
                       "parallelism": f"strip{world}", "l2": _l2_note(dofs_rank)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "bytes_per_dof": BYTES_PER_DOF, "kernel_ms": sweep_ms},
            "clocks": clk.summary(),
            "gpu_launches": args.steps * (1 if world == 1 else dsw.launches_per_sweep()),
            "setup_seconds": setup_s,
            "time_to_converge": ttc or None,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "kernel": N.sweep_kernel(a),
            "other_configs": others or None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def _l2_note(dofs_rank: int) -> str:
    gb = dofs_rank * 8 / 1e9
    if 3 * gb * 1e3 > 4 * 126:   # s, u^k, u^{k+1} together well above the 126 MB L2
        return f"state {gb:.2g} GB/GPU per array >> 126 MB L2 (no flush needed)"
    return f"state {gb * 1e3:.3g} MB/GPU per array: L2-resident (reduced --cells run, not the BASELINE size)"


def _self_launch(args) -> int:
    """--gpus N without a torchrun environment: start N ranks (one per GPU)
    through torch.distributed.run on 127.0.0.1 and return their exit code."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kappa", type=float, default=1e-3)
    ap.add_argument("--cells", type=int, default=None)
    ap.add_argument("--order", type=int, default=6)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--ttc", nargs="*", default=["1e-3:5", "1e-1:1"],
                    help="time to converge: kappa:steps items (none: skip)")
    # kappa=0.1 at 2048^2 contracts by ~0.9997 per sweep (tools/kappa_probe.py): ~6e4 sweeps per step
    ap.add_argument("--ttc-max-iters", type=int, default=100000)
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-others", dest="other_configs", action="store_false")
    ap.add_argument("--cpu-rows", type=int, default=64)
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--host-staging", action="store_true",
                    help="test mode: ranks share GPUs and exchange through host memory (gloo) instead of NCCL")
    ap.add_argument("--overlap", action="store_true",
                    help="multi-GPU: force the interior-first split launch (default: by strip height)")
    ap.add_argument("--no-overlap", action="store_true",
                    help="multi-GPU: halo before the whole sweep instead of under the interior layers")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

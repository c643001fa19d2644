#!/usr/bin/env python
"""Benchmark of the compressed view-factor hot path on B200.

Default workload (BASELINE.json configs[2], the largest single-GPU config:
BASELINE.json's `metric` names no config, so the largest one that fits one
GPU applies): the 256^2-cell fBm terrain (Hurst 0.8, RMS slope 15 deg, 10 m
spacing) with a 1 km spherical-cap crater, 131,072 facets, F-hat built at
tol 1e-5 in FP64 (untimed).  One STEP = one vf_matvec with nrhs = 1 (the
HBM-bound compressed apply, Alg. 5): permute-in, low-rank
phase 1 (T = S V^T X), row-owner accumulate, permute-out.  The same line
carries `batched`: nrhs = 128 (configs[2]'s batched case) timed the same way.

metric value = RHS-column applies per second = sum over ranks of
nrhs * steps / time (max over ranks).  Multi-GPU (torchrun): every rank
applies the replicated F-hat to its own right-hand sides (COLS), no
data-path collective: weak scaling.

--workload cfg2 : configs[1], the 64-sun batched thermal solve (cap crater in
                  a plain, F-hat resident in shared memory).
--workload cfg5 : configs[4], the cfg3 mesh with one sun, radiosity + IR to
                  1e-8, block-row sharded (ROWS) with a per-iteration allgather.

--impl reference runs the FP64 CPU oracle (oracle/, the reference arm for
this tier) on a bounded sample of the same workload on the host cores.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compressed F·X apply: RHS-columns/sec and HBM GB/s (% of roofline) at 1/2/4/8 GPUs"
UNIT = "RHS-column applies/s"
NRHS = 64
TOL_BUILD = 1e-5
TOL_SOLVE = {"f64": 1e-10, "f32": 1e-6}
ALBEDO, EMISS = 0.12, 0.95
S_SUN = 1365.0
ELEV = 5.0
REF_ROWS = 2000          # oracle rows of the exact F sampled on the terrain configs


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def ncu_traffic(key):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    `--set full` capture (profiles/traffic.json, written from the capture's
    dram__bytes_read.sum + dram__bytes_write.sum); None if absent."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(p))[key]
        return d["dram_bytes_per_launch"], d["source"]
    except Exception:
        return None, None


def fp64_peak_tflops(sm_mhz):
    # B200: 148 SMs x 64 FP64 FMA/clk/SM x 2 flop
    return 148 * 64 * 2 * sm_mhz * 1e6 / 1e12


def fp32_peak_tflops(sm_mhz):
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12


class Clocks:
    """Samples SM clocks and clock-event (throttle) reasons DURING the timed
    region (the recipe's clocks line). NVML is polled every ~5 ms from a
    thread, with one synchronous sample at start() and one at stop(), so even a
    timed region of a few tens of ms carries several samples; nvidia-smi -lms
    100 is the fallback when NVML is unavailable."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.p = None
        self.nv = None
        self.lines = []
        self.samples = []
        self.stop_ev = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(index).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.nv, self.h = pynvml, h
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nv = None

    def _sample(self):
        nv = self.nv
        self.samples.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)),
                             int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))))

    def _poll(self):
        while not self.stop_ev.wait(0.005):
            try:
                self._sample()
            except Exception:
                return

    def start(self):
        if self.nv:
            self._sample()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nv:
            self.stop_ev.set()
            self.t.join()
            self._sample()
            sm = [c for c, _ in self.samples]
            reasons = {nm for nm, bit in self.BITS.items() for _, r in self.samples if r & bit}
            return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.smax, "reasons": sorted(reasons),
                    "samples": len(sm), "source": "NVML, ~5 ms poll over the timed region"}
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(2)
        except Exception:
            self.p.kill()
        sm, smax, reasons = [], [], set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms 100"}


def workload(rank, world):
    import scenegen as sg
    V, F = sg.cfg2_mesh()
    phase = 2 * math.pi / NRHS * rank / max(world, 1)
    suns = sg.sun_dirs(ELEV, NRHS, phase)
    return V, F, suns


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ----------------------------------------------------------- oracle (CPU) arm

def oracle_sample(V, F, suns, ncols, budget_s):
    """The oracle as it stands: exact CSR F (eq. FF-def) + FP64 thermal Jacobi
    solve on `ncols` of the sun columns; repeated until ~budget_s of work."""
    import oracle
    S = oracle.Scene(V, F)
    csr = S.F_csr_rows()
    Q = S.insolation(suns[:ncols], S_SUN)
    alb, emi = np.full(S.N, ALBEDO), np.full(S.N, EMISS)
    applies, t = 0, 0.0
    reps = 0
    while t < budget_s and reps < 5000:
        t0 = time.perf_counter()
        out = oracle.thermal(lambda X: oracle.apply_csr(csr, X), Q, alb, emi, TOL_SOLVE["f64"], 100)
        t += time.perf_counter() - t0
        applies += ncols * (out["it1"] + out["it2"])
        reps += 1
    return applies / t, t, reps, out


def run_reference(args, rank, world):
    """The reference arm of this tier: the FP64 CPU oracle as it stands, on a
    bounded sample of the SAME workload as the GPU arm (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    if args.workload in ("cfg3", "cfg5"):
        return run_reference_terrain(args)
    V, F, suns = workload(0, 1)
    ncols = 8
    times, applies = [], 0
    S = oracle.Scene(V, F)
    csr = S.F_csr_rows()
    Q = S.insolation(suns[:ncols], S_SUN)
    alb, emi = np.full(S.N, ALBEDO), np.full(S.N, EMISS)
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        out = oracle.thermal(lambda X: oracle.apply_csr(csr, X), Q, alb, emi, TOL_SOLVE["f64"], 100)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            applies += ncols * (out["it1"] + out["it2"])
    tot = sum(times)
    v = applies / tot
    sample = f"oracle thermal solve (exact CSR F, FP64, OpenMP) on {ncols} of the 64 sun columns per step"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_block(S.N, "f64"),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
                             "sample": sample, "cpu": cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_reference_terrain(args):
    """configs[2] (cfg3) reference: the oracle's exact F (eq. FF-def with its
    own visibility) on REF_ROWS seeded rows, applied to the same nrhs columns
    as the GPU arm each step; value scaled to whole-matrix applies."""
    import oracle
    import scenegen as sg
    V, F = sg.cfg3_mesh(n=args.cells, crater_D=1000.0 * args.cells / 256)
    S = oracle.Scene(V, F)
    N = S.N
    k = args.nrhs
    rows = np.sort(np.random.default_rng(8).choice(N, size=min(N, REF_ROWS), replace=False))
    t0 = time.perf_counter()
    csr = S.F_csr_rows(rows)
    t_rows = time.perf_counter() - t0
    X = sg.random_rhs(N, k, seed=3)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.apply_csr(csr, X)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    v = args.steps * k * rows.size / N / tot
    sample = (f"oracle exact-CSR apply (eq. FF-def rows, FP64, OpenMP) of {rows.size} seeded rows of F x {k} "
              f"column(s) per step, scaled to whole-matrix applies (rows computed once, {t_rows:.1f} s, untimed)")
    wl = terrain_workload_name(args, N, "f64", k)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": wl, "N": N, "nrhs": k, "rows_sampled": int(rows.size)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
                             "sample": sample, "cpu": cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def terrain_workload_name(args, N, dt, k, rows_mode=False):
    cfgname = "configs[4]" if rows_mode else "configs[2]"
    return (f"BASELINE {cfgname}: {args.cells}^2-cell fBm terrain (H 0.8, RMS slope 15 deg, 10 m) + "
            f"{1000.0 * args.cells / 256:.0f} m cap crater, {N} facets, F-hat tol {args.tol:g}, {dt.upper()}, "
            + ("one sun (e 5 deg), radiosity + IR Jacobi to 1e-8, block-row sharded (ROWS) with a per-iteration "
               "ncclAllGather" if rows_mode else f"vf_matvec with nrhs = {k} (U[0,1) columns, seed 3)"))


def config_block(N, dtype, extra=None):
    c = {"workload": "BASELINE configs[1]: cap crater (R=1, d/D=0.2) in a 4D square plain, "
                     f"{N} facets, 64 suns at {ELEV} deg elevation (batched RHS), F-hat tol {TOL_BUILD:g}, "
                     f"{dtype.upper()} thermal equilibrium solve (radiosity + IR Jacobi, tol {TOL_SOLVE[dtype]:g})",
         "N": N, "nrhs": NRHS, "tol_build": TOL_BUILD, "tol_solve": TOL_SOLVE[dtype],
         "l2": "flushed between timed steps (256 MiB write, outside the step events)"}
    if extra:
        c.update(extra)
    return c


# ----------------------------------------------------------- GPU arm

def run_gpu(args, rank, world, local_rank):
    import torch
    import paper_2209_07632_b200 as vf
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dt = args.dtype
    tdt = torch.float64 if dt == "f64" else torch.float32
    V, F, suns = workload(rank, world)
    M = vf.ViewFactorMatrix.build(V, F, TOL_BUILD, dtype=vf.VF_F64 if dt == "f64" else vf.VF_F32, device=local_rank)
    info = M.refresh()
    N = info["N"]
    stream = torch.cuda.current_stream(dev)
    M.set_stream(stream.cuda_stream)
    Qdir_h = M.insolation(suns, S_SUN).astype(np.float64 if dt == "f64" else np.float32, order="F")
    alb_h = np.full(N, ALBEDO, dtype=Qdir_h.dtype)
    emi_h = np.full(N, EMISS, dtype=Qdir_h.dtype)

    def colmajor(a):
        return torch.from_numpy(np.ascontiguousarray(a.T)).to(dev).T

    Qdir, alb, emi = colmajor(Qdir_h), torch.from_numpy(alb_h).to(dev), torch.from_numpy(emi_h).to(dev)
    T = torch.empty((NRHS, N), dtype=tdt, device=dev).T
    Qv = torch.empty((NRHS, N), dtype=tdt, device=dev).T
    Qi = torch.empty((NRHS, N), dtype=tdt, device=dev).T
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    tol = TOL_SOLVE[dt]

    def step():
        M.solve_thermal(Qdir, alb, emi, T, Qv, Qi, iters=200, tol=tol)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    vf.vf_enable_kernel_timing(M.h, True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = Clocks(local_rank)
    ms2 = 0.0
    l2 = 0
    ms1 = 0.0
    l1 = 0
    launches = 0
    applies = 0
    its = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)                      # L2 flush outside the step events
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
        st = M.stats()
        kt = vf.vf_kernel_timing(M.h)
        ms2 += kt["ms_phase2"]; l2 += kt["launches_phase2"]
        ms1 += kt["ms_phase1"]; l1 += kt["launches_phase1"]
        launches += kt["launches_total"]
        applies += NRHS * (st["iters1"] + st["iters2"])
        its.append((st["iters1"], st["iters2"]))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    vf.vf_enable_kernel_timing(M.h, False)
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    # max over ranks of time, sum of work
    tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    wk = torch.tensor([float(applies)], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dist.all_reduce(wk, op=dist.ReduceOp.SUM)
    t_max = tt.item()
    value = wk.item() / (t_max / 1e3)

    # e2e: the same call with HOST buffers (pinned), H2D/D2H inside the timed region
    Qdir_p = torch.from_numpy(np.ascontiguousarray(Qdir_h.T)).pin_memory().T
    alb_p = torch.from_numpy(alb_h).pin_memory()
    emi_p = torch.from_numpy(emi_h).pin_memory()
    T_p = torch.empty((NRHS, N), dtype=tdt).pin_memory().T
    Qv_p = torch.empty((NRHS, N), dtype=tdt).pin_memory().T
    Qi_p = torch.empty((NRHS, N), dtype=tdt).pin_memory().T
    ke = max(5, min(args.steps, 30))
    # the step's result is the temperature T (Qvis / Qir are optional outputs of
    # vf_solve_thermal and are not read back in the end-to-end timing)
    M.solve_thermal(Qdir_p, alb_p, emi_p, T_p, None, None, iters=200, tol=tol)
    e_ms, e_app = 0.0, 0
    if dist:
        dist.barrier()
    for i in range(ke):
        flush.fill_(i & 0xFF)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        M.solve_thermal(Qdir_p, alb_p, emi_p, T_p, None, None, iters=200, tol=tol)
        e1.record(stream)
        e1.synchronize()
        e_ms += e0.elapsed_time(e1)
        st = M.stats()
        e_app += NRHS * (st["iters1"] + st["iters2"])
    et = torch.tensor([e_ms], dtype=torch.float64, device=dev)
    ew = torch.tensor([float(e_app)], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
        dist.all_reduce(ew, op=dist.ReduceOp.SUM)
    e2e_value = ew.item() / (et.item() / 1e3)
    w = 8 if dt == "f64" else 4
    h2d = N * NRHS * w + 2 * N * w
    d2h = N * NRHS * w

    if rank == 0:
        pk, pk_kind = peaks()
        # dominant kernel: the persistent Jacobi solve kernel hot_kernel<T,4,4,M_SOLVE>
        # (one launch per thermal stage; each launch runs `iters` F-hat applies).
        n_iters = int(sum(a + b for a, b in its))
        avg = ms2 / max(l2, 1)
        kp = NRHS
        flops_iter = info["alg_flops_per_col"] * kp
        bytes_iter = (info["p1_bytes"] + info["p2_bytes"] + (info["p1_src_rows"] + info["p2_src_rows"]) * kp * w
                      + info["t_rows"] * kp * w + info["active_rows"] * kp * w * 4)
        flops_launch = flops_iter * n_iters / max(l2, 1)
        bytes_launch = bytes_iter * n_iters / max(l2, 1)
        smax = pk.get("sm_max_mhz", 1965.0)
        # res_kernel contracts on the FP64 tensor cores (DMMA; FP32 factors widened to FP64)
        dmma = bool(info.get("resident"))
        peak_tf = fp64_peak_tflops(smax) if dt == "f64" or dmma else fp32_peak_tflops(smax)
        ach_tf = flops_launch / (avg * 1e-3) / 1e12 if avg > 0 else 0.0
        ach_gbs = bytes_launch / (avg * 1e-3) / 1e9 if avg > 0 else 0.0
        traffic, traffic_src = ncu_traffic(f"cfg2_{dt}")
        roof = {"bound": "tensor" if dmma else "alu", "achieved": ach_tf, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": ach_tf / peak_tf if peak_tf else None, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": (f"res_kernel<{'double' if dt == 'f64' else 'float'},M_SOLVE> (persistent Jacobi solve, "
                           "F-hat resident in shared memory: phase 1 V^T X, grid barrier, phase 2 row-owner "
                           "accumulate + fused epilogue, residual decision; one launch per thermal stage)"
                           if info.get("resident") else
                           f"hot_kernel<{'double' if dt == 'f64' else 'float'},1,8,M_SOLVE,grouped> (persistent "
                           "Jacobi solve: phase 1 V^T X, grid barrier, phase 2 row-owner accumulate + fused "
                           "epilogue, residual decision; one launch per thermal stage)"),
                "peak_basis": (("derived FP64 DMMA peak (= the DFMA rate on B200): " if dmma else "derived: ")
                               + f"148 SM x {64 if dt == 'f64' or dmma else 128} {'F64' if dmma else dt.upper()} FMA/clk x 2 x "
                               f"{smax:.0f} MHz (sm_max of {pk_kind} MEASURED_PEAKS.json); DESIGN.md §7"),
                "avg_launch_ms": avg, "launches": l2, "applies_per_launch": n_iters / max(l2, 1),
                "flops_per_apply": flops_iter, "flops_per_launch": flops_launch,
                "alg_bytes_per_apply": bytes_iter, "alg_bytes_per_launch": bytes_launch,
                "achieved_gbs": ach_gbs, "hbm_peak_gbs": pk.get("hbm_gbs"),
                "hbm_frac": ach_gbs / pk.get("hbm_gbs", 6556.8), "share_of_step": ms2 / t_ms if t_ms > 0 else None}
        # CPU baseline: the oracle as it stands on a bounded sample
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                import oracle
                oracle.build()
                v_cpu, t_cpu, reps, _ = oracle_sample(V, F, suns, 8, args.cpu_budget)
                cpu = {"value": v_cpu, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
                       "sample": f"oracle thermal solve (exact CSR F from eq. FF-def, FP64, OpenMP) on 8 of the "
                                 f"64 sun columns, {reps} repetitions, {t_cpu:.1f} s", "cpu": cpu_model()}
            except Exception as e:  # noqa
                cpu = {"value": None, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
                       "sample": f"failed: {e}"}
        it_arr = np.array(its)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": dt, "data": "synthetic",
                "config": config_block(N, dt, {
                    "iters_radiosity": int(np.median(it_arr[:, 0])), "iters_ir": int(np.median(it_arr[:, 1])),
                    "solve_columns_per_s": NRHS * world * args.steps / (t_max / 1e3),
                    "fhat_alg_bytes": info["alg_bytes"], "fhat_device_bytes": info["device_bytes"],
                    "blocks": {"dense": info["n_dense"], "csr": info["n_csr"], "svd": info["n_svd"]},
                    "active_rows": info["active_rows"], "sum_rank": info["sum_rank"],
                    "build_seconds": info["build_seconds"], "parallelism": f"cols{world}"}),
                "roofline": roof, "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
                "gpu_launches": launches, "clocks": clk}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# ----------------------------------------------------------- terrain workloads (cfg3 / cfg5)

def terrain_fhat(args, device):
    """F-hat of BASELINE configs[2] (256^2-cell fBm terrain + 1 km crater):
    loaded from --fhat if that file exists, else built (device evaluator +
    device rank search, untimed) and saved there."""
    import paper_2209_07632_b200 as vf
    import scenegen as sg
    V, F = sg.cfg3_mesh(n=args.cells, crater_D=1000.0 * args.cells / 256)
    dt = vf.VF_F64 if args.dtype == "f64" else vf.VF_F32
    path = args.fhat.format(n=args.cells, tol=args.tol, dtype=args.dtype) if args.fhat else None
    t0 = time.time()
    if path and os.path.exists(path):
        M = vf.ViewFactorMatrix.load(path, device=device)
        vf.vf_set_mesh(M.h, V, F)              # geometry for vf_insolation
        built = False
    else:
        M = vf.ViewFactorMatrix.build(V, F, args.tol, dtype=dt, device=device)
        built = True
        if path:
            M.save(path)
    return M, V, F, {"fhat_seconds": time.time() - t0, "built": built}


def oracle_rows(V, F, rows):
    import oracle
    S = oracle.Scene(V, F)
    return S, S.F_csr_rows(rows)


def _pad(n):
    return n if n <= 2 else (n + 15) // 16 * 16 if n > 8 else (4 if n <= 4 else 8)


def matvec_chunks(info, k, rows_mode):
    """The launches libvf's vf_matvec issues for k columns (matvec_impl's
    column rules): one entry per launch, its column count."""
    if not rows_mode and info.get("tiles", 0) > 0 and k > 8:
        return [k]                                    # one streamed-tile launch
    big = not rows_mode and info["device_bytes"] > (256 << 20)
    if big and 2 <= k <= 8:
        return [1] * k
    if big and k > 64:
        chunks, c0, piece = [], 0, 64
        while c0 < k:
            n = k - c0
            if n >= piece:
                n = piece
            elif piece // 2 >= 16:
                piece //= 2
                continue
            if n <= 8:
                chunks += [1] * (k - c0)
                break
            chunks.append(n)
            c0 += n
        return chunks
    return [k]


def time_steps(M, vf, step, steps, warmup, stream, dist, local_rank, per_step_sync):
    """W untimed steps, then K steps bracketed by barrier + synchronize; CUDA
    events on the library's stream around each step; libvf's own per-launch
    event pairs give the hot kernel's device time.  Returns a dict."""
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    vf.vf_enable_kernel_timing(M.h, True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    clocks = Clocks(local_rank)
    ms_hot, l_hot, launches, extra = 0.0, 0, 0, 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for i in range(steps):
        ev[i][0].record(stream)
        e = step()
        ev[i][1].record(stream)
        if per_step_sync:
            torch.cuda.synchronize()
        kt = vf.vf_kernel_timing(M.h)
        ms_hot += kt["ms_phase2"]
        l_hot += kt["launches_phase2"]
        launches += kt["launches_total"]
        extra += e or 0
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    vf.vf_enable_kernel_timing(M.h, False)
    t_ms = sum(x.elapsed_time(y) for x, y in ev)
    return {"t_ms": t_ms, "ms_hot": ms_hot, "l_hot": l_hot, "launches": launches, "clocks": clk, "extra": extra}


def reduce_time_work(t_ms, work, dist, dev, sum_work=True):
    import torch
    tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    wk = torch.tensor([float(work)], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        if sum_work:
            dist.all_reduce(wk, op=dist.ReduceOp.SUM)
    return tt.item(), wk.item()


def terrain_roofline(info, k, dt, tm, steps, rows_mode, pk, pk_kind, workload):
    """Roofline object of the dominant kernel for a terrain line:
    nrhs <= 2 -> HBM bound, algorithmic bytes = F-hat payload + X/T rows read
    + T rows written + Y rows written; batched -> FP64/FP32 FMA bound,
    algorithmic flops = nrhs x alg_flops_per_col."""
    w = 8 if dt == "f64" else 4
    chunks = matvec_chunks(info, k, rows_mode)
    solve_rows = 4 if rows_mode else 1
    hbm = pk.get("hbm_gbs", 6559.0)

    stream = info.get("stream_chunks", 0) > 0 and not rows_mode

    def alg_bytes(kp):
        # F-hat payload one apply streams: for nrhs = 1 the bytes of the layout the kernel
        # reads (chunk stream: values + 16-bit CSR offsets + phase-1 row lists; row layout:
        # values + S + V row indices + 16-bit CSR offsets), else values + 32-bit indices
        if kp == 1 and stream:
            fh = info["stream_payload_bytes"]
        elif kp == 1 and info.get("k1_payload_bytes", 0) > 0:
            fh = info["k1_payload_bytes"]             # (ROWS M_STEP launches read the same 16-bit layout)
        else:
            fh = info["p1_bytes"] + info["p2_bytes"]
        return (fh + (info["p1_src_rows"] + info["p2_src_rows"]) * kp * w
                + info["t_rows"] * kp * w + info["active_rows"] * kp * w * solve_rows)
    avg = tm["ms_hot"] / max(tm["l_hot"], 1)
    flops_app = info["alg_flops_per_col"] * k
    if rows_mode:
        n_app = tm["extra"] / max(steps, 1)
        apps_launch = n_app / max(tm["l_hot"] / steps, 1)
        bytes_app = alg_bytes(1)
        ach_gbs = bytes_app * apps_launch / (avg * 1e-3) / 1e9 if avg > 0 else 0.0
        ach_tf = flops_app * apps_launch / (avg * 1e-3) / 1e12 if avg > 0 else 0.0
    else:
        t_hot = tm["ms_hot"] / max(steps, 1) * 1e-3
        bytes_app = sum(alg_bytes(_pad(n)) for n in chunks)
        ach_gbs = bytes_app / t_hot / 1e9 if t_hot > 0 else 0.0
        ach_tf = flops_app / t_hot / 1e12 if t_hot > 0 else 0.0
    traffic, traffic_src = ncu_traffic(f"{workload}_k{k}_{dt}")
    if max(chunks) > 2:
        smax = pk.get("sm_max_mhz", 1965.0)
        tiles = info.get("tiles", 0) > 0 and max(chunks) > 8
        tc = os.environ.get("VF_TC", "0") not in ("", "0") or os.environ.get("VF_TC2", "0") not in ("", "0")
        if tiles and dt == "f32" and tc:
            # tcgen05 kind::tf32 with 3xTF32: the measured bf16 peak x the nominal tf32/bf16 ratio
            # (1.1 / 2.25 PFLOP/s dense), / 3 MMAs per useful product
            peak_tf = pk.get("bf16_tflops", 1619.6) * (1.1 / 2.25) / 3.0
            bound = {"bound": "tensor", "achieved": ach_tf, "peak": peak_tf, "unit": "TFLOP/s", "frac": ach_tf / peak_tf,
                     "peak_basis": f"3xTF32 on tcgen05: {pk_kind} MEASURED_PEAKS.json bf16_tflops x 1.1/2.25 "
                                   "(nominal tf32/bf16 dense ratio) / 3"}
        else:
            dmma = tiles                      # bt_kernel<double|float>: DMMA (FP32 widened to FP64)
            peak_tf = fp64_peak_tflops(smax) if dt == "f64" or dmma else fp32_peak_tflops(smax)
            bound = {"bound": "tensor" if dmma else "alu", "achieved": ach_tf, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": ach_tf / peak_tf,
                     "peak_basis": (("derived FP64 DMMA peak (= the DFMA rate on B200): " if dmma else "derived: ")
                                    + f"148 SM x {64 if dt == 'f64' or dmma else 128} FMA/clk x 2 x {smax:.0f} MHz "
                                      f"(sm_max of {pk_kind} MEASURED_PEAKS.json)")}
    else:
        bound = {"bound": "hbm", "achieved": ach_gbs, "peak": hbm, "unit": "GB/s", "frac": ach_gbs / hbm,
                 "peak_basis": f"{pk_kind} MEASURED_PEAKS.json hbm_gbs (copy bandwidth, 'burst' figure for a kernel "
                               "timed alone)"}
    tn = "double" if dt == "f64" else "float"
    if max(chunks) <= 2:
        kern = (f"stream_k1_kernel<{tn}> (bulk-copy chunk stream: phase 1 T = S V^T x, warp-granular grid barrier, "
                "phase 2 row-owner accumulate)" if stream and max(chunks) == 1 else
                f"k1p_kernel<{tn}> (pipelined: per-warp cp.async rings of 4-term chunks issued rounds ahead, one "
                "queue of phase-1 part items then LPT rows, no grid barrier; 16-bit CSR offsets, L2 evict-first)"
                if info.get("k1_kernel", 0) == 2 else
                f"hot_kernel<{tn},1,1,M_MATVEC> (phase 1 T = S V^T x, grid barrier, phase 2 row-owner accumulate with "
                "an LPT row queue; F-hat loads L1::no_allocate + L2 evict-first"
                + (", 16-bit CSR offsets)" if info.get("k1_payload_bytes", 0) > 0 else ")"))
    elif info.get("tiles", 0) > 0 and dt == "f64":
        kern = ("bt_kernel (streamed 16-row tiles, [K][16] weights x staged XT rows on FP64 tensor cores, DMMA "
                "m8n8k4; phase 1 T tiles, grid barrier, phase 2 row tiles)")
    elif info.get("tiles", 0) > 0 and not (os.environ.get("VF_TC", "0") not in ("", "0")
                                           or os.environ.get("VF_TC2", "0") not in ("", "0")):
        kern = ("bt_kernel<float> (streamed 16-row tiles, FP32 [K][16] weights x staged FP32 XT rows widened to FP64 "
                "in registers, DMMA m8n8k4 with FP64 accumulation, one rounding to FP32 at the store)")
    elif info.get("tiles", 0) > 0:
        kern = ("bt_tc_kernel (streamed 16-row tiles on tcgen05 kind::tf32, TMEM accumulator, 3xTF32 split; "
                "phase 1 T tiles, grid barrier, phase 2 row tiles)")
    else:
        kern = f"hot_kernel<{tn},32,VEC,M_MATVEC> (wide per-row: warp across 32 VEC columns)"
    return {**bound, "traffic": traffic, "traffic_source": traffic_src,
            "kernel": ("(ROWS mode, one Jacobi iteration per launch) " if rows_mode else "") + kern,
            "achieved_gbs": ach_gbs, "hbm_frac": ach_gbs / hbm, "hbm_frac_vs_8TBs_spec": ach_gbs / 8000.0,
            "avg_launch_ms": avg, "launches": tm["l_hot"], "alg_bytes_per_apply": bytes_app,
            "alg_flops_per_apply": flops_app, "achieved_tflops": ach_tf,
            "stream_bytes_per_apply": (info["stream_payload_bytes"] + info["stream_meta_bytes"]) if stream else None,
            "stream_meta_bytes": info["stream_meta_bytes"] if stream else None,
            "column_chunks": chunks[:4] + (["..."] if len(chunks) > 4 else []),
            "share_of_step": tm["ms_hot"] / tm["t_ms"] if tm["t_ms"] > 0 else None}


def run_terrain(args, rank, world, local_rank):
    import torch
    import paper_2209_07632_b200 as vf
    import scenegen as sg
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dt = args.dtype
    tdt = torch.float64 if dt == "f64" else torch.float32
    ndt = np.float64 if dt == "f64" else np.float32
    w = 8 if dt == "f64" else 4
    M, V, F, binfo = terrain_fhat(args, local_rank)
    rows_mode = args.workload == "cfg5"
    if rows_mode:
        if dist:
            M.init_rows()
        else:
            M.shard_rows(0, 1)
            M.comm_init(0, 1, vf.vf_get_nccl_id())
    info = M.refresh()
    N = info["N"]
    stream = torch.cuda.current_stream(dev)
    M.set_stream(stream.cuda_stream)
    k = 1 if rows_mode else args.nrhs

    def colmajor(a):
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=ndt).T)).to(dev).T

    if rows_mode:
        sun = sg.sun_dirs(5.0, 1)
        Qh = M.insolation(sun, S_SUN)
        Qd = colmajor(Qh)
        alb, emi = colmajor(np.full(N, ALBEDO)).reshape(-1).contiguous(), colmajor(np.full(N, EMISS)).reshape(-1).contiguous()
        T = torch.empty((1, N), dtype=tdt, device=dev).T
        Qv = torch.empty((1, N), dtype=tdt, device=dev).T
        Qi = torch.empty((1, N), dtype=tdt, device=dev).T

        def step():
            M.solve_thermal(Qd, alb, emi, T, Qv, Qi, iters=500, tol=1e-8)
            st = M.stats()
            return st["iters1"] + st["iters2"]
    else:
        X = colmajor(sg.random_rhs(N, k, seed=3 + rank))
        Y = torch.empty((k, N), dtype=tdt, device=dev).T

        def step():
            M.matvec(X, Y)
            return k

    tm = time_steps(M, vf, step, args.steps, args.warmup, stream, dist, local_rank, per_step_sync=not rows_mode)
    t_max, work = reduce_time_work(tm["t_ms"], tm["extra"], dist, dev, sum_work=not rows_mode)
    value = work / (t_max / 1e3)

    # e2e through the same call with pinned HOST buffers (H2D of the inputs and
    # D2H of the result inside the timed region)
    e_ms, e_app = 0.0, 0
    if rows_mode:
        Qp = torch.from_numpy(np.ascontiguousarray(Qh.T.astype(ndt))).pin_memory().T
        ap_ = torch.full((N,), ALBEDO, dtype=tdt).pin_memory()
        ep_ = torch.full((N,), EMISS, dtype=tdt).pin_memory()
        Tp = torch.empty((1, N), dtype=tdt).pin_memory().T

        def estep():
            M.solve_thermal(Qp, ap_, ep_, Tp, None, None, iters=500, tol=1e-8)
            return M.stats()["iters1"] + M.stats()["iters2"]
        h2d, d2h = N * w + 2 * N * w, N * w
    else:
        Xp = X.cpu().T.contiguous().pin_memory().T
        Yp = torch.empty((k, N), dtype=tdt).pin_memory().T

        def estep():
            M.matvec(Xp, Yp)
            return k
        h2d, d2h = N * k * w, N * k * w
    estep()
    ke = max(3, min(args.steps, 10))
    for i in range(ke):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n = estep()
        e1.record(stream)
        e1.synchronize()
        e_ms += e0.elapsed_time(e1)
        e_app += n
    et, ew = reduce_time_work(e_ms, e_app, dist, dev, sum_work=not rows_mode)
    e2e_value = ew / (et / 1e3)

    # the batched case of configs[2] (nrhs = 128) on the same F-hat, same protocol
    batched = None
    kb = args.batched if (not rows_mode and k == 1) else 0
    if kb:
        Xb = colmajor(sg.random_rhs(N, kb, seed=3 + rank))
        Yb = torch.empty((kb, N), dtype=tdt, device=dev).T

        def bstep():
            M.matvec(Xb, Yb)
            return kb
        sb = max(3, min(args.steps, 20))
        tb = time_steps(M, vf, bstep, sb, 3, stream, dist, local_rank, per_step_sync=True)
        tbm, wb = reduce_time_work(tb["t_ms"], tb["extra"], dist, dev)
        if rank == 0:
            pk, pk_kind = peaks()
            batched = {"nrhs": kb, "value": wb / (tbm / 1e3), "unit": UNIT, "steps": sb,
                       "ms_per_step": tbm / sb, "gpu_launches": tb["launches"], "clocks": tb["clocks"],
                       "roofline": terrain_roofline(info, kb, dt, tb, sb, False, pk, pk_kind, args.workload)}

    if rank == 0:
        pk, pk_kind = peaks()
        roof = terrain_roofline(info, k, dt, tm, args.steps, rows_mode, pk, pk_kind, args.workload)
        wl = terrain_workload_name(args, N, dt, k, rows_mode)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
                "scaling": "strong" if rows_mode else "weak", "vs_baseline": None, "dtype": dt, "data": "synthetic",
                "config": {"workload": wl, "N": N, "nrhs": k, "tol_build": args.tol,
                           "l2": "inputs larger than L2: F-hat %.2f GB vs 126 MB L2 (no flush needed)"
                                 % (info["alg_bytes"] / 1e9),
                           "fhat_alg_bytes": info["alg_bytes"], "fhat_device_bytes": info["device_bytes"],
                           "blocks": {"dense": info["n_dense"], "csr": info["n_csr"], "svd": info["n_svd"]},
                           "nnz_csr": info["nnz_csr"], "sum_rank": info["sum_rank"],
                           "active_rows": info["active_rows"], "visible_pairs": info["visible_pairs"],
                           "applies_per_step": tm["extra"] / max(args.steps, 1), **binfo,
                           "parallelism": (f"rows{world}" if rows_mode else f"cols{world}")},
                "roofline": roof, "cpu_baseline": None, "parity": None, "batched": batched,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
                "gpu_launches": tm["launches"], "clocks": tm["clocks"]}
        if not args.no_cpu_baseline and world == 1 and not rows_mode:
            import oracle
            oracle.build()
            rng = np.random.default_rng(8)
            rows = np.sort(rng.choice(N, size=min(N, REF_ROWS), replace=False))
            _, csr = oracle_rows(V, F, rows)
            Xh = X.cpu().numpy().astype(np.float64)
            reps, tc = 0, 0.0
            while tc < args.cpu_budget and reps < 100000:
                t0 = time.perf_counter()
                Yref = oracle.apply_csr(csr, Xh)
                tc += time.perf_counter() - t0
                reps += 1
            v_cpu = reps * k * rows.size / N / tc
            # the same oracle rows check the GPU results of the timed launch configurations
            step()
            torch.cuda.synchronize()
            Yg = Y.cpu().numpy().astype(np.float64)[rows]
            parity = {"rows": int(rows.size), "rel_l2_vs_exact_F": float(np.linalg.norm(Yg - Yref) /
                                                                         np.linalg.norm(Yref)),
                      "bound": 10 * args.tol, "source": "the cpu_baseline leg's oracle rows (eq. FF-def)"}
            if kb:
                bstep()
                torch.cuda.synchronize()
                Yrb = oracle.apply_csr(csr, Xb.cpu().numpy().astype(np.float64))
                Ygb = Yb.cpu().numpy().astype(np.float64)[rows]
                parity["batched_rel_l2_vs_exact_F"] = float(np.linalg.norm(Ygb - Yrb) / np.linalg.norm(Yrb))
            line["parity"] = parity
            line["cpu_baseline"] = {"value": v_cpu, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
                                    "sample": f"oracle exact-CSR apply (eq. FF-def rows, FP64, OpenMP) of {rows.size} "
                                              f"sampled rows of F x {k} columns, {reps} reps in {tc:.1f} s, scaled "
                                              f"to whole-matrix applies", "cpu": cpu_model()}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_alg6(args, rank, world, local_rank):
    """NEXT-1 line: Alg. 6 time stepping on the configs[2] terrain,
    one scenario, a sun circling at 5 deg elevation in `--alg6-steps-per-day`
    steps per lunar day, M = 30 subsurface layers to 0.5 m (reading A27).  One
    step = the 2-column F-hat product (two nrhs = 1 applies) + the
    Crank-Nicolson column update of every facet.  metric: time steps / s."""
    import torch
    import paper_2209_07632_b200 as vf
    import scenegen as sg
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    M, V, F, binfo = terrain_fhat(args, local_rank)
    info = M.refresh()
    N = info["N"]
    stream = torch.cuda.current_stream(dev)
    M.set_stream(stream.cuda_stream)
    nday = args.alg6_steps_per_day
    suns = sg.sun_dirs(5.0, nday)
    Q = M.insolation(suns, S_SUN)                                     # N x nday (host, untimed)
    Qd = torch.from_numpy(np.ascontiguousarray(Q.T)).to(dev)          # row n = step n's N-vector
    alb = np.full(N, ALBEDO)
    emi = np.full(N, EMISS)
    T0 = np.full((N, 1), 200.0, order="F")
    layers, depth = 30, 0.5
    st = vf.TimeStepper(M, alb, emi, np.asfortranarray(Q[:, :1]), T0, layers=layers, depth=depth, ratio=1.2,
                        k_th=0.005, rho_c=1.2e6)
    dt = 29.53 * 86400.0 / nday
    Tn = torch.empty((1, N), dtype=torch.float64, device=dev).T
    n = [1]

    def step():
        q = Qd[n[0] % nday].reshape(N, 1)
        st.step(q, dt, Tn)
        n[0] += 1
        return 1

    tm = time_steps(M, vf, step, args.steps, args.warmup, stream, None, local_rank, per_step_sync=False)
    t_ms = tm["t_ms"]
    value = args.steps / (t_ms / 1e3)
    if rank == 0:
        pk, pk_kind = peaks()
        w = 8
        kb = info.get("k1_payload_bytes") or (info["p1_bytes"] + info["p2_bytes"])
        bytes_apply = kb + (info["p1_src_rows"] + info["p2_src_rows"] + info["t_rows"] + info["active_rows"]) * w
        avg = tm["ms_hot"] / max(tm["l_hot"], 1)
        ach = bytes_apply / (avg * 1e-3) / 1e9 if avg > 0 else 0.0
        hbm = pk.get("hbm_gbs", 6559.0)
        line = {"metric": "Alg. 6 time steps per second (2-column F-hat product + Crank-Nicolson columns)",
                "value": value, "unit": "steps/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"NEXT-1 Alg. 6 on BASELINE configs[2] ({N} facets), one scenario, sun at 5 deg "
                                       f"elevation, {nday} steps per lunar day, {layers} layers to {depth} m",
                           "N": N, "layers": layers, **binfo},
                "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                             "kernel": "the nrhs = 1 apply (two per step)", "avg_launch_ms": avg,
                             "launches": tm["l_hot"], "share_of_step": tm["ms_hot"] / t_ms if t_ms > 0 else None,
                             "alg_bytes_per_apply": bytes_apply},
                "gpu_launches": tm["launches"], "clocks": tm["clocks"]}
        print(json.dumps(line), flush=True)
    st.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="cfg3", choices=["cfg2", "cfg3", "cfg5", "alg6"],
                    help="cfg3: BASELINE configs[2] matvec (default); cfg2: configs[1] batched thermal solve; "
                         "cfg5: configs[4] ROWS-sharded single-sun solve on the cfg3 mesh")
    ap.add_argument("--nrhs", type=int, default=1)
    ap.add_argument("--alg6-steps-per-day", type=int, default=48)
    ap.add_argument("--batched", type=int, default=128,
                    help="cfg3 with nrhs = 1: also time this many columns (configs[2]'s batched case; 0 = off)")
    ap.add_argument("--tol", type=float, default=1e-5)
    ap.add_argument("--cells", type=int, default=256)
    ap.add_argument("--fhat", default=None, help="HVFM cache path (may use {n}, {tol}, {dtype})")
    ap.add_argument("--no-parity", action="store_true", help="(kept for old command lines; no effect)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.workload == "cfg2":
        run_gpu(args, rank, world, local_rank)
    elif args.workload == "alg6":
        run_alg6(args, rank, world, local_rank)
    else:
        run_terrain(args, rank, world, local_rank)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric: kernel-matrix MVM
entries/s; ms per marginal-likelihood step).

A step is one fused H.V over BASELINE config 1 (n=13,500, d=26, s=65,
Matern-3/2 ARD, fp32): ``value`` is whole-job entries/s (n^2 per H.V) with
inputs resident in HBM, timed per step (V split + H.V kernel + split
reduction) with CUDA events on the launching stream, and the dominant
kernel's own time (the roofline) from a second pass with events around each
H.V launch; ``e2e`` is the same H.V through the C-ABI host-pointer entry point
(``wgp_hv``: pinned host V in, host H.V out, copies inside the timed region).
Between timed iterations L2 is flushed (a 512 MiB write; the inputs, 3.5 MB,
would otherwise stay L2-resident).  With --gpus N under torchrun every rank's
library context joins one NCCL communicator (wgp_set_comm): the library
computes the rank's rows of H.V and all-gathers the n x s result itself
(SURVEY §8e); timing is the max over ranks.

The line also carries ``large_n``: config 3's full-size H.V (n = 391,386),
row-sharded under torchrun, at every N -- the north star's scaling case -- and
``outer``: ms per marginal-likelihood step (the second
half of the metric) at configs 2 and 3 through the library's wgp_train --
row-sharded inside the library under torchrun -- with iterations, converged
steps and final residuals per solver, and the CPU path's outer-step figures
under ``cpu_baseline.outer`` (N=1).

``--impl reference`` times the reference's CPU path -- the CPU oracle's
restatement of build_kernel_matrices (proj/src/kernel.cpp:120-139) plus the
dense fp64 product H * V the reference solvers run per iteration
(proj/src/solvers.cpp:110), all host threads -- on a bounded row sample of
the same workload.
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

METRIC = "kernel-matrix MVM entries/s (fused H.V, BASELINE config 1)"
UNIT = "entries/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # tc_f16 (default): 3xTF32 Gram + fp16x3 K.V over column-scaled V, 2.0e-7
    # relative at config 1 (tc, 3xTF32 K.V: 3.5e-7; scripts/diag_f16.py)
    ap.add_argument("--hv-impl", default="tc_f16", choices=["tc", "tc_f16", "simt"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-outer", action="store_true", help="skip the per-outer-step timings")
    ap.add_argument("--comm", action="store_true",
                    help="N=1: attach a one-rank NCCL communicator (runs the library's sharded code path)")
    ap.add_argument("--no-c3", action="store_true", help="skip the config-3 outer steps")
    ap.add_argument("--no-large", action="store_true", help="skip the config-3 full-size H.V (scaling case)")
    ap.add_argument("--outer-steps", type=int, default=5, help="timed outer steps per solver (config 2)")
    ap.add_argument("--outer-warmup", type=int, default=1, help="untimed outer steps before them")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        return dict(bf16=m["bf16_tflops"], bf16_sus=m.get("bf16_tflops_sustained", m["bf16_tflops"]),
                    hbm=m["hbm_gbs"], mhz=m.get("sm_max_mhz", 1965.0), src="measured")
    return dict(bf16=1590.0, bf16_sus=1400.0, hbm=6650.0, mhz=1965.0, src="fallback")


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed regions: NVML
    (pynvml, ~every 2 ms -- a 20-step H.V region lasts ~5 ms) with nvidia-smi as
    the fallback.  `phase(name)` labels the following samples."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.samples = []  # (phase, sm_mhz, max_mhz, reasons)
        self._phase = "setup"
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._nvml = pynvml
            self._bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                          "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                          "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                          "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None

    def phase(self, name):
        self._phase = name

    def _sample_nvml(self):
        n = self._nvml
        sm = n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)
        r = n.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        self.samples.append((self._phase, float(sm), float(self._max),
                             [k for k, bit in self._bits.items() if r & bit]))

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip()
        if out:
            f = [x.strip() for x in out.split(",")]
            self.samples.append((self._phase, float(f[0]), float(f[1]),
                                 [self.NAMES[k] for k in range(4) if len(f) > 2 + k and f[2 + k].lower() == "active"]))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nvml else self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.002 if self._nvml else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        load = [x for x in self.samples if x[0] != "setup"] or self.samples
        sm = [x[1] for x in load]
        hv = [x for x in self.samples if x[0] == "hv"]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(x[2] for x in load),
                "reasons": sorted({r for x in load for r in x[3]}), "samples": len(load),
                "samples_during_hv_steps": len(hv),
                "sm_mhz_during_hv_steps": float(np.median([x[1] for x in hv])) if hv else None,
                "source": "nvml" if self._nvml else "nvidia-smi"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_baseline(p, seconds):
    """Oracle (port) matrix-free fp64 H.V on a bounded row sample, all threads."""
    from oracle import oracle as orc

    n = p.X.shape[0]
    rows, elapsed = 8, 0.0
    while True:
        t0 = time.perf_counter()
        orc.hv_rows(p.X, p.lengthscales, p.signal, p.noise, p.V, 0, rows)
        elapsed = time.perf_counter() - t0
        if elapsed >= seconds / 4 or rows >= n:
            break
        rows = min(n, rows * 4)
    return {"value": rows * n / elapsed, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"oracle matrix-free fp64 H.V, rows 0..{rows} of config 1 (x {n} points, "
                      f"s=65), {elapsed:.1f} s"}


def sgd_learning_rate(wg, ds_X, ds_y, device):
    """The reference's grid search (proj/src/experiment.cpp:133-168, default
    candidates and budget proj/tools/main.cpp:53-54) at config 2's start."""
    from paper_2405_18328_b200 import experiment as ex

    ds = ex.Dataset("c2", ds_X, ds_y)
    base = wg.TrainConfig(init_constrained=1.0, seed=0,
                          solver=wg.SolverConfig(kind="sgd", minibatch_size=1000, momentum=0.9))
    cands = [1.0, 3.0, 10.0, 30.0, 100.0, 300.0]
    t0 = time.perf_counter()
    lr = ex.grid_search_sgd_lr(ds, cands, 60, base, device=device)
    return lr, {"candidates": cands, "budget_steps": 60, "chosen": lr, "seconds": time.perf_counter() - t0}


def run_outer(wg, ctx, p, sc, steps, warmup, precision="f64", ws=1):
    """One warm-started training run on the device; per-step device times of
    the timed steps (CUDA events around each outer step: probes, solve,
    warm-start-distance H.V, gradient, Adam) and what the solver did."""
    ctx.set_cg_precision(precision)
    cfg = wg.TrainConfig(steps=warmup + steps, learning_rate=0.1, num_probes=64, mode="warm", seed=0,
                         transform="log", estimator="pathwise", rff_features=1000, init_noise=0.5,
                         init_constrained=1.0, warm_start_distance=True, solver=wg.SolverConfig(**sc))
    tr = ctx.train(p.y, cfg)
    timed = tr.steps[warmup:]
    tol = np.array([sc["tol_mean"]] + [sc["tol_samples"]] * 64)
    conv = [bool(np.all(r.per_column_relative_residual <= tol * (1 + 1e-9))) for r in timed]
    step = np.array([r.step_ms for r in timed])
    wsd = np.array([r.warm_distance_ms for r in timed])
    if ws > 1:  # per-step maximum over the ranks
        import torch
        import torch.distributed as dist
        t = torch.tensor(np.concatenate([step, step - wsd]), device=f"cuda:{torch.cuda.current_device()}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        both = t.cpu().numpy()
        step, wsd = both[:len(step)], both[:len(step)] - both[len(step):]
    return {"ms_per_step": float(step.mean()),
            "ms_per_step_without_warm_start_distance": float((step - wsd).mean()),
            "solver_ms_per_step": float(np.mean([r.solver_ms for r in timed])),
            "iterations": [int(r.solver_iterations) for r in timed],
            "iterations_mean": float(np.mean([r.solver_iterations for r in timed])),
            "converged_steps": f"{sum(conv)}/{len(conv)}",
            "max_final_relative_residual": float(max(r.per_column_relative_residual.max() for r in timed)),
            "cg_precision": precision if sc["kind"] == "cg" else None,
            "config": {k: v for k, v in sc.items() if k != "kind"}}


def large_n_hv(wg, datasets, device, args, ws, rank, reps=5):
    """The north star's scaling case: BASELINE config 3's full-size fused H.V
    (n = 391,386, d = 3, s = 65, fp32 tc) row-sharded over the ranks by the
    library (own rows + NCCL all-gather of the n x s result), CUDA events on the
    context stream, maximum over the ranks -- reported at every N so the
    scaling at n >= 390k can be read off the N = 1, 2, 4, 8 lines."""
    import torch

    p = datasets.config3()
    n = p.X.shape[0]
    ctx = make_ctx(wg, device, args, ws, rank)
    ctx.set_data(p.X)
    ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
    _, _, r0, r1, ldc = ctx.shard_info()
    dev = torch.device("cuda", device)
    V = torch.from_numpy(np.random.default_rng(7).standard_normal((65, n)).astype(np.float32)).to(dev)
    sharded = ws > 1 or args.comm
    out = torch.empty((65, ldc if sharded else n), device=dev)
    st = torch.cuda.ExternalStream(ctx.stream)
    times = []
    with torch.cuda.stream(st):
        for i in range(reps + 1):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            ctx.hv_device(V.data_ptr(), n, 65, out.data_ptr(), out.shape[1])
            b.record(st)
            b.synchronize()
            if i:
                times.append(a.elapsed_time(b))
    ms = float(np.mean(times))
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ctx.close()
    return {"workload": "config3 fused H.V n=391386 d=3 s=65 (fp32 tc), rows sharded over the ranks + NCCL "
                        "all-gather of the result" if sharded else "config3 fused H.V n=391386 d=3 s=65 (fp32 tc)",
            "value": n * n / (ms / 1e3), "unit": "entries/s", "ms_per_step": ms, "steps": reps,
            "rows_per_rank": int(r1 - r0), "timing": "CUDA events, max over ranks"}


def outer_bench(wg, datasets, device, args, ws=1, rank=0):
    """ms per marginal-likelihood step (the second half of BASELINE.json's
    metric) on one GPU through the library's wgp_train:
      config 2 (n=41,157, d=9, 64 pathwise probes + y, RFF 1000, log-space
      Adam lr 0.1, warm start): CG (tol 0.01, fp64 and fp32), AP (blocks of
      1000, tol 0.01), SGD (minibatch 1000, momentum 0.9, tol 0.01, learning
      rate from the reference's grid search), reference default iteration caps
      (solvers.cpp:88,148,206);
      config 3 (n=391,386, d=3): AP, blocks of 1000, 10-epoch budget.
    Each run starts cold at step 1; `outer_warmup` steps are untimed, the
    next `outer_steps` are timed.  Under torchrun every context joins an NCCL
    communicator and the library row-shards the whole outer loop (SGD is
    single-GPU and skipped); times are the per-step maximum over the ranks."""
    out = {"timing": "CUDA events on the context stream around each outer step (device time; the "
                     "warm-start-distance H.V included, and subtracted in the *_without_* field)",
           "steps_timed": args.outer_steps, "warmup_steps": args.outer_warmup}
    if ws > 1 or args.comm:
        out["sharding"] = f"rows over {ws} GPU(s) inside the library (wgp_set_comm, NCCL)"
    p = datasets.config2()
    ctx = make_ctx(wg, device, args, ws, rank)
    ctx.set_data(p.X)
    c2 = {"workload": "config2 n=41157 d=9 s=65, pathwise RFF 1000, log-space Adam lr 0.1, warm start"}
    runs = [("cg_f64", dict(kind="cg", tol_mean=0.01, tol_samples=0.01, max_iterations=0), "f64"),
            ("cg_f32", dict(kind="cg", tol_mean=0.01, tol_samples=0.01, max_iterations=0), "f32"),
            ("ap", dict(kind="ap", tol_mean=0.01, tol_samples=0.01, max_iterations=0, block_size=1000), "f64")]
    if ws == 1 and not args.comm:  # SGD is single-GPU
        try:
            lr, grid = sgd_learning_rate(wg, p.X, p.y, device)
            runs.append(("sgd", dict(kind="sgd", tol_mean=0.01, tol_samples=0.01, max_iterations=0,
                                     minibatch_size=1000, momentum=0.9, learning_rate=lr, seed=0), "f64"))
            c2["sgd_lr_grid_search"] = grid
        except Exception as e:
            c2["sgd_lr_grid_search"] = {"error": str(e)[:200]}
    for name, sc, prec in runs:
        try:
            c2[name] = run_outer(wg, ctx, p, sc, args.outer_steps, args.outer_warmup, prec, ws)
        except Exception as e:  # report, keep the other solvers' numbers
            c2[name] = {"error": str(e)[:200]}
    ctx.close()
    out["c2"] = c2
    if not args.no_c3:
        p3 = datasets.config3()
        ctx = make_ctx(wg, device, args, ws, rank)
        ctx.set_data(p3.X)
        c3 = {"workload": "config3 n=391386 d=3 s=65, pathwise RFF 1000, log-space Adam lr 0.1, warm start, "
                          "AP blocks of 1000 with a 10-epoch budget"}
        try:
            c3["ap"] = run_outer(wg, ctx, p3, dict(kind="ap", tol_mean=0.01, tol_samples=0.01, max_iterations=10,
                                                   block_size=1000), min(args.outer_steps, 2), 1, "f64", ws)
        except Exception as e:
            c3["ap"] = {"error": str(e)[:200]}
        ctx.close()
        out["c3"] = c3
    return out


def cpu_outer_baseline(datasets, outer, seconds):
    """The reference's CPU path for outer steps:
    config 0's whole 20-step training run by the fp64 oracle (timed), and a
    config-2 CG step extrapolated from a timed oracle fp64 H.V row sample x
    the H.V products the step needs (iterations + 2, the iteration count of
    the fp64 device run, which matches the reference's)."""
    from oracle import oracle as orc

    res = {"cores": os.cpu_count(), "kind": "port"}
    p0 = datasets.config0()
    cfg = orc.TrainConfig(steps=20, learning_rate=0.1, num_probes=16, mode="warm", seed=0, transform="log",
                          estimator="pathwise", rff_features=1000, init_noise=0.5, init_constrained=1.0,
                          solver=orc.SolverConfig(kind="cg", tol_mean=0.01, tol_samples=0.01,
                                                  max_iterations=1000))
    t0 = time.perf_counter()
    o = orc.train(p0.X, p0.y, cfg)
    dt = time.perf_counter() - t0
    res["c0_train"] = {"ms_per_step": 1e3 * dt / 20, "seconds": dt, "iterations_total": int(o["solver_iterations"].sum()),
                       "sample": "oracle fp64 train, BASELINE config 0, 20 steps (timed)"}
    p2 = datasets.config2()
    n = p2.X.shape[0]
    V = np.random.default_rng(0).standard_normal((n, 65))
    rows, el = 64, 0.0
    while True:
        t0 = time.perf_counter()
        orc.hv_rows(p2.X, p2.lengthscales, p2.signal, p2.noise, V, 0, rows)
        el = time.perf_counter() - t0
        if el >= seconds / 4 or rows >= n:
            break
        rows = min(n, rows * 4)
    rate = rows * n / el
    cg = (outer or {}).get("c2", {}).get("cg_f64", {})
    it = cg.get("iterations_mean")
    if it:
        res["c2_cg_step"] = {"ms_per_step": 1e3 * (it + 2) * n * n / rate, "extrapolated": True,
                             "sample": f"oracle fp64 H.V rows 0..{rows} x {n} points, s=65 ({el:.1f} s), "
                                       f"x {it + 2:.1f} H.V per step (device fp64 CG iterations + 2)"}

    def rows_rate(p, budget):  # oracle fp64 H.V entries/s on a row sample of the full problem
        n_ = p.X.shape[0]
        V_ = np.random.default_rng(0).standard_normal((n_, 65))
        r_, el_ = 8, 0.0
        while True:
            t0_ = time.perf_counter()
            orc.hv_rows(p.X, p.lengthscales, p.signal, p.noise, V_, 0, r_)
            el_ = time.perf_counter() - t0_
            if el_ >= budget or r_ >= n_:
                return r_ * n_ / el_, r_, el_
            r_ = min(n_, r_ * 4)

    # config 3 AP step as the reference runs it (proj/src/solvers.cpp:141-196):
    # per epoch the right-looking updates (n x b per block: n^2) plus the exact
    # residual (n^2), 10 epochs, + the initial residual, the final exact
    # residual and the gradient (~1 H.V each): 23 H.V-equivalents per step.
    p3 = datasets.config3()
    rate3, r3, e3 = rows_rate(p3, seconds / 8)
    n3 = p3.X.shape[0]
    res["c3_ap_step"] = {"ms_per_step": 1e3 * 23 * n3 * n3 / rate3, "extrapolated": True,
                         "sample": f"oracle fp64 H.V rows 0..{r3} x {n3} points, s=65 ({e3:.1f} s), x 23 "
                                   "H.V-equivalents per AP step (10 epochs x 2 + 3)"}
    # config 4 CG step: the device run's ~265 CG iterations per step (scripts/c4_outer.py) + 3
    p4 = datasets.config4()
    rate4, r4, e4 = rows_rate(p4, seconds / 8)
    n4 = p4.X.shape[0]
    res["c4_cg_step"] = {"ms_per_step": 1e3 * 268 * n4 * n4 / rate4, "extrapolated": True,
                         "sample": f"oracle fp64 H.V rows 0..{r4} x {n4} points, s=65 ({e4:.1f} s), x 268 "
                                   "H.V per CG step (~265 iterations, profiles/r2_c4_outer_f32_1gpu.json, + 3)"}
    return res


class _StdoutToStderr:
    """fd-level redirect of stdout into stderr (NCCL prints its version banner
    on stdout at communicator creation; rank 0's stdout is the JSON line)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def make_ctx(wg, device, args, ws, rank, **kw):
    """A library context; under torchrun it joins an NCCL communicator of the
    ws ranks (wgp_set_comm: the library row-shards H.V, the solvers and the
    outer loop itself).  torch.distributed only carries the 128-byte NCCL id."""
    ctx = wg.Context(device, hv_impl=args.hv_impl, **kw)
    if ws > 1:
        import torch
        import torch.distributed as dist
        uid = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{device}")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(wg.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        with _StdoutToStderr():
            ctx.set_comm(rank, ws, bytes(uid.cpu().numpy().tobytes()))
    elif args.comm:  # the sharded code path on a one-rank communicator (plumbing check)
        with _StdoutToStderr():
            ctx.set_comm(0, 1, wg.nccl_unique_id())
    return ctx


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as orc
    from paper_2405_18328_b200 import datasets

    p = datasets.config1()
    n = p.X.shape[0]
    # Dense fp64 H as the reference builds it (oracle restatement, OpenMP),
    # then H * V per step -- the product the reference's solvers run every
    # iteration -- through multi-threaded BLAS dgemm (stand-in for Eigen's GEMM).
    t0 = time.perf_counter()
    H, _, _ = orc.kernel_matrices(p.X.astype(np.float64), p.lengthscales, p.signal, p.noise)
    build_s = time.perf_counter() - t0
    V = np.asfortranarray(p.V, dtype=np.float64)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        out = H @ V
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    ms = 1e3 * float(np.mean(times))
    value = n * n / (ms / 1e3)
    # the reference itself is single-threaded Eigen (no OpenMP,
    # proj/src/CMakeLists.txt:14): the same GEMM on one core, on a row block
    single = None
    try:
        from threadpoolctl import threadpool_limits
        rows = 2000
        with threadpool_limits(limits=1):
            Hb = np.asfortranarray(H[:rows])
            Hb @ V
            t0 = time.perf_counter()
            Hb @ V
            dt1 = time.perf_counter() - t0
        single = {"value": rows * n / dt1, "unit": UNIT, "cores": 1, "kind": "port",
                  "sample": f"dense fp64 H[0:{rows}, :] @ V (n={n}, s=65), one BLAS thread, {dt1:.2f} s"}
    except Exception as e:
        single = {"error": str(e)[:200]}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config1 H.V n=13500 d=26 s=65 (reference dense path: prebuilt "
                               "H, fp64 GEMM per step)", "n": n, "d": 26, "s": 65,
                   "h_build_seconds_excluded": build_s},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                         "sample": "full config-1 dense H.V per step (H built once, "
                                   f"{build_s:.1f} s, outside the timed region)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("a LOWER BOUND on the reference's time per H.V: multi-threaded BLAS on all host cores "
                 "stands in for the reference's single-threaded Eigen GEMM, and the dense H is built once "
                 "outside the timed region (the reference rebuilds it every outer step, "
                 "proj/src/optimizer.cpp:121)"),
        "single_thread": single,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    ws, rank, local = dist_env()
    import torch

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        with _StdoutToStderr():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
    import paper_2405_18328_b200 as wg
    from paper_2405_18328_b200 import datasets

    p = datasets.config1()
    n, d = p.X.shape
    s = p.V.shape[1]
    ctx = make_ctx(wg, local, args, ws, rank)
    ctx.set_data(p.X)
    ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
    _, _, r0, r1, ldc = ctx.shard_info()
    m = r1 - r0
    if ws > 1:
        # strong scaling of one H.V: J splits keyed on the shard's rows (more
        # CTAs per GPU on small shards; rows equal to fp32 rounding, not bitwise)
        ctx.set_split_global(False)
    stream = torch.cuda.ExternalStream(ctx.stream)
    dev = torch.device("cuda", local)
    Vt = torch.from_numpy(np.ascontiguousarray(p.V.T)).to(dev)  # [s][n] = column-major n x s
    # sharded: the library computes this rank's rows and all-gathers the n x s
    # result over NCCL inside wgp_hv_device (out holds all rows, leading dim ldc)
    sharded = ws > 1 or args.comm
    out_dev = torch.empty((s, ldc if sharded else max(m, 1)), device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)

    def one_step():
        ctx.hv_device(Vt.data_ptr(), n, s, out_dev.data_ptr(), out_dev.shape[1])

    # clocks are sampled from the warm-up through the timed H.V steps and the
    # outer-step timings (a 20-step H.V region lasts ~5 ms, shorter than one
    # nvidia-smi sample); reported per phase
    clk = ClockSampler(local)
    clk.__enter__()
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            one_step()
        stream.synchronize()
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        launches0 = wg.launch_count()
        clk.phase("hv")
        for a, b in evs:
            flush.zero_()
            a.record(stream)
            one_step()
            b.record(stream)
        stream.synchronize()
        launches = wg.launch_count() - launches0
        # the dominant kernel's own time (roofline): the same steps again with
        # CUDA events around each hv_tc launch -- a separate pass, because an
        # event between the V split and the H.V kernel breaks their
        # programmatic dependent launch (the split overlaps the kernel's fill)
        kernel_ms, kernel_launches = 0.0, 0
        if args.hv_impl != "simt":
            ctx.profile(True)
            for _ in range(args.steps):
                flush.zero_()
                one_step()
            stream.synchronize()
            kernel_ms, kernel_launches = ctx.profile_read()
            ctx.profile(False)
        clk.phase("e2e")
    times = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.mean(times))
    # dominant kernel's mean launch duration (events on the context stream);
    # the SIMT path is a single kernel per step
    kernel_ms = kernel_ms / kernel_launches if kernel_launches else ms
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n * n / (ms / 1e3)

    # e2e through the C-ABI with host buffers (pinned), copies in the timed region
    Vh = torch.from_numpy(np.asfortranarray(p.V).T.copy()).pin_memory()
    m_out = n if sharded else m  # sharded wgp_hv returns the all-gathered n x s
    outh = torch.empty((s, m_out), pin_memory=True)
    lib = wg.load()
    import ctypes as C
    e2e_times = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rc = lib.wgp_hv(ctx._h, C.c_void_p(Vh.data_ptr()), s, C.c_void_p(outh.data_ptr()))
        b.record(stream)
        b.synchronize()
        if rc != 0:
            raise RuntimeError(lib.wgp_last_error().decode())
        if i >= args.warmup:
            e2e_times.append(a.elapsed_time(b))
    e2e_ms = float(np.mean(e2e_times))
    e2e_med = float(np.median(e2e_times))
    print("e2e times (ms):", " ".join(f"{t:.3f}" for t in e2e_times), file=sys.stderr)
    # the box's PCIe rates for the same buffers (plain pinned copies on the context
    # stream, after the timed calls): e2e ~ H2D + step + exposed D2H, and the host
    # link differs a lot between boxes (H2D 14-50 GB/s seen)
    pcie = {}
    dprobe = torch.empty_like(Vh, device=dev)
    with torch.cuda.stream(stream):
        for name, fn in (("h2d", lambda: dprobe.copy_(Vh, non_blocking=True)),
                         ("d2h", lambda: Vh.copy_(dprobe, non_blocking=True))):
            fn()
            stream.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(10):
                fn()
            b.record(stream)
            b.synchronize()
            pcie[name + "_ms"] = a.elapsed_time(b) / 10
            pcie[name + "_GBps"] = Vh.numel() * 4 / (pcie[name + "_ms"] * 1e-3) / 1e9
    del dprobe
    if ws > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # the large-n scaling case and the outer steps run on every rank
    # (collectives inside the library), before rank 0 reports
    large = None
    if not args.no_large:
        clk.phase("large_n")
        try:
            large = large_n_hv(wg, datasets, local, args, ws, rank)
        except Exception as e:
            large = {"error": str(e)[:200]}
    outer = None
    if not args.no_outer:
        clk.phase("outer")
        outer = outer_bench(wg, datasets, local, args, ws, rank)
    clk.__exit__()
    if rank != 0:
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    pk = peaks()
    clocks = clk.summary()
    f_entry = 2 * d + 2 * s + 8                       # SURVEY §8d F_hv
    flops = f_entry * n * n
    # T_roof = max(sum over pipes of FLOPs_pipe / P_pipe,
    # 2 n^2 / P_MUFU) on ALGORITHMIC work: the 2d Gram flops on the tensor pipe
    # at P_TF32 / 3 (3xTF32), the 2s K.V flops at P_TF32 / 3 (tc: 3xTF32) or
    # P_F16 / 3 (tc_f16: fp16x3, the kind::f16 rate = the bf16 rate), the 8
    # Matern flops on the FMA pipe (P_FFMA = 128 FMA/clk/SM,
    # scripts/ubench/ubench_ffma2.cu), 2 MUFU ops.  `frac` is against the
    # arithmetic the engine performs; `frac_if_3xtf32` applies the all-3xTF32
    # tensor term (round 1's basis) to the same kernel time.
    p_bf16 = pk["bf16"] * 1e12
    p_tf32 = p_bf16 / 2                                # TF32 = half the bf16 rate
    p_ffma = 2 * 128 * 148 * pk["mhz"] * 1e6
    p_mufu = 16 * 148 * pk["mhz"] * 1e6                # ex2 / sqrt per s (16/clk/SM)
    t_3xtf32 = (2 * d + 2 * s) / (p_tf32 / 3) + 8 / p_ffma
    if args.hv_impl in ("tc", "tc_f16"):
        p_kv = p_tf32 if args.hv_impl == "tc" else p_bf16
        t_pipes = 2 * d / (p_tf32 / 3) + 2 * s / (p_kv / 3) + 8 / p_ffma
        basis = (f"sum-of-pipes: {2 * d} Gram flop/entry at P_TF32/3 + {2 * s} K.V flop/entry at "
                 f"{'P_TF32' if args.hv_impl == 'tc' else 'P_F16'}/3 + 8 FMA-pipe flop/entry at P_FFMA; "
                 f"MUFU 2 ops/entry at 16/clk/SM")
        # the padded work the kernel actually issues (Gram K = 32, K.V N = s
        # padded to 16), for reference: not the roofline
        spad = 16 * -(-s // 16)
        t_issued = 3 * 2 * 32 / p_tf32 + 3 * 2 * spad / p_kv
    else:
        t_pipes = f_entry / p_ffma
        basis = "FFMA 256 flop/clk/SM"
        t_issued = t_pipes
    t_entry = max(t_pipes, 2 / p_mufu)
    bound = "tensor"  # compute-bound (contract field admits hbm|tensor only)
    peak = f_entry / t_entry / 1e12
    achieved = flops / ws / (kernel_ms / 1e3) / 1e12  # this rank's rows per launch
    # DRAM traffic is only measurable under ncu (profiles/): not from this run
    traffic = None
    traffic_profile = None
    prof = os.path.join(ROOT, "profiles", "hv_tc_traffic.json")
    if os.path.exists(prof):
        try:
            traffic_profile = {"dram_bytes_per_launch": json.load(open(prof)).get("dram_bytes_per_launch"),
                               "source": "profiles/hv_tc_traffic.json (ncu --set full, config 1; not this run)"}
        except Exception:
            traffic_profile = None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "config1 fused H.V n=13500 d=26 s=65 Matern-3/2 ARD",
                   "n": n, "d": d, "s": s, "hv_impl": args.hv_impl, "l2": "flushed (512 MiB write)",
                   "parallelism": f"rows{ws}" if ws > 1 else "single"},
        "e2e": {"value": n * n / (e2e_ms / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(n * s * 4), "d2h_bytes_per_step": int(m_out * s * 4),
                "ms_per_step": e2e_ms, "ms_median": e2e_med, "ms_min": float(np.min(e2e_times)),
                "pcie_probe": pcie,
                "h2d_path": os.environ.get("WGP_HV_UPLOAD", "zc") + " (zc: the V split kernel loads the "
                            "page-locked host V over PCIe itself; ce: cudaMemcpyAsync before it)"},
        "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_profile": traffic_profile,
                     "peak_basis": f"{pk['src']} peaks: F_hv={f_entry} flop/entry; " + basis,
                     "kernel_ms": kernel_ms, "t_roof_ms": t_entry * n * n / ws * 1e3,
                     "frac_of_issued_work": (t_issued * n * n / ws * 1e3) / kernel_ms,
                     "frac_if_3xtf32": (max(t_3xtf32, 2 / p_mufu) * n * n / ws * 1e3) / kernel_ms},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if large is not None:
        line["large_n"] = large
    if outer is not None:
        line["outer"] = outer
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(p, args.cpu_seconds)
        if outer is not None:
            try:
                line["cpu_baseline"]["outer"] = cpu_outer_baseline(datasets, outer, args.cpu_seconds)
            except Exception as e:
                line["cpu_baseline"]["outer"] = {"error": str(e)[:200]}
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

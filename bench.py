#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric: kernel-matrix MVM
entries/s; ms per marginal-likelihood step).

A step is one fused H.V over BASELINE config 1 (n=13,500, d=26, s=65,
Matern-3/2 ARD, fp32): ``value`` is whole-job entries/s (n^2 per H.V) with
inputs resident in HBM, timed per launch with CUDA events on the launching
stream; ``e2e`` is the same H.V through the C-ABI host-pointer entry point
(``wgp_hv``: pinned host V in, host H.V out, copies inside the timed region).
Between timed iterations L2 is flushed (a 512 MiB write; the inputs, 3.5 MB,
would otherwise stay L2-resident).  With --gpus N under torchrun the rows of
H.V are sharded across ranks (row-block sharding) and the n x s
result is all-gathered over NCCL; timing is the max over ranks.

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
    ap.add_argument("--hv-impl", default="tc", choices=["tc", "tc_bf16", "simt"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--outer", action="store_true",
                    help="also time outer steps (row-sharded over the ranks under torchrun)")
    ap.add_argument("--outer-config", type=int, default=2, choices=[2, 3],
                    help="BASELINE config of --outer: 2 (CG / AP / SGD) or 3 (AP, 10-epoch budget)")
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
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

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
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 2 + k and s[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


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


def outer_spec(datasets, args, sharded_run=False):
    """The outer-loop workload of `--outer-config`:
    2: BASELINE config 2 (n=41,157, d=9, 64 pathwise probes + y, 1000 RFF
       features, log-space Adam lr 0.1, warm start) with CG (tol 0.01), AP
       (blocks of 1000) and SGD (minibatch 1000, momentum 0.9), `steps` timed
       steps after `warmup`;
    3: BASELINE config 3 (n=391,386, d=3, s=65, AP blocks of 1000 with a
       budget of 10 epochs per outer step, warm start): ~10 s per step on one
       GPU, so at most 3 timed steps after 1 warm-up step.
    Returns (problem, workload, solvers, timed steps, warm-up steps)."""
    if args.outer_config == 3:
        p = datasets.config3()
        solvers = {"ap": dict(kind="ap", tol_mean=0.01, tol_samples=0.01, max_iterations=10, block_size=1000)}
        return (p, "config3 n=391386 d=3 s=65, pathwise RFF 1000, log-space Adam lr 0.1, warm start, "
                   "AP 10-epoch budget", solvers, max(1, min(args.steps, 3)), 1)
    p = datasets.config2()
    solvers = {
        "cg": dict(kind="cg", tol_mean=0.01, tol_samples=0.01, max_iterations=1000),
        "ap": dict(kind="ap", tol_mean=0.01, tol_samples=0.01, max_iterations=100, block_size=1000),
    }
    if not sharded_run:
        solvers["sgd"] = dict(kind="sgd", tol_mean=0.01, tol_samples=0.01, max_iterations=3000,
                              minibatch_size=1000, momentum=0.9, learning_rate=10.0)
    return (p, "config2 n=41157 d=9 s=65, pathwise RFF 1000, log-space Adam lr 0.1, warm start", solvers,
            max(args.steps, 1), args.warmup)


def outer_steps(wg, datasets, device, args):
    """The `--outer-config` outer loop on one GPU (outer_spec): device time
    per outer step (solve + gradient + probes, from the library's per-step
    CUDA events) per solver."""
    p, workload, solvers, k_steps, w_steps = outer_spec(datasets, args)
    n_steps = w_steps + k_steps
    out = {"workload": workload,
           "timing": "CUDA events on the context stream around each outer step (device time)",
           "steps": k_steps, "warmup_steps": w_steps}
    for name, sc in solvers.items():
        ctx = wg.Context(device, hv_impl=args.hv_impl)
        ctx.set_data(p.X)
        cfg = wg.TrainConfig(steps=n_steps, learning_rate=0.1, num_probes=64, mode="warm", seed=0,
                             transform="log", estimator="pathwise", rff_features=1000, init_noise=0.5,
                             init_constrained=1.0, warm_start_distance=False,
                             solver=wg.SolverConfig(**sc))
        try:
            tr = ctx.train(p.y, cfg)
            timed = tr.steps[w_steps:]
            out[name] = {"ms_per_step": float(np.mean([r.step_ms for r in timed])),
                         "solver_ms_per_step": float(np.mean([r.solver_ms for r in timed])),
                         "iterations_mean": float(np.mean([r.solver_iterations for r in timed])),
                         "config": {k: v for k, v in sc.items() if k != "kind"}}
        except Exception as e:  # report, keep the other solvers' numbers
            out[name] = {"error": str(e)[:200]}
        ctx.close()
    return out


def outer_sharded(wg, datasets, device, args, ws, rank):
    """The `--outer-config` outer loop (outer_spec; CG and AP) row-sharded over `ws` GPUs
    (sharded.sharded_train on the library's operators: CG with per-iteration
    all-gathers of the direction, AP with per-block exchanges, the gradient
    summed in rank order).  Per-step time: host clock around each step with
    the device synchronised, maximum over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2405_18328_b200 import sharded

    p, workload, solvers, k_steps, w_steps = outer_spec(datasets, args, sharded_run=True)
    n = p.X.shape[0]
    r0, r1 = sharded.row_range(n, rank, ws)
    ctx = wg.Context(device, hv_impl=args.hv_impl)
    ctx.set_data(p.X)
    ctx.set_split_global(False)  # strong scaling: J splits keyed on the shard's rows
    ops = sharded.device_train_ops(ctx, r0, r1)
    n_steps = w_steps + k_steps
    out = {"workload": workload,
           "sharding": f"rows{ws}", "timing": "host clock per outer step (device synchronised), max over ranks",
           "steps": k_steps, "warmup_steps": w_steps}
    for name, sc in solvers.items():
        cfg = wg.TrainConfig(steps=n_steps, learning_rate=0.1, num_probes=64, mode="warm", seed=0,
                             transform="log", estimator="pathwise", rff_features=1000, init_noise=0.5,
                             init_constrained=1.0, solver=wg.SolverConfig(**sc))
        torch.cuda.synchronize()
        steps = sharded.sharded_train(ops, p.y, cfg)
        timed = steps[w_steps:]
        t = torch.tensor([1e3 * float(np.mean([s.step_seconds for s in timed]))], device=f"cuda:{device}")
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[name] = {"ms_per_step": float(t.item()),
                     "iterations_mean": float(np.mean([s.solver_iterations for s in timed])),
                     "config": {k: v for k, v in sc.items() if k != "kind"}}
    ctx.close()
    return out


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
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2405_18328_b200 as wg
    from paper_2405_18328_b200 import datasets

    p = datasets.config1()
    n, d = p.X.shape
    s = p.V.shape[1]
    ctx = wg.Context(local, hv_impl=args.hv_impl)
    ctx.set_data(p.X)
    ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
    # row shard of this rank (aligned to the 128-row tile grid)
    tiles = -(-n // 128)
    t0_, t1_ = tiles * rank // ws, tiles * (rank + 1) // ws
    r0, r1 = min(n, t0_ * 128), min(n, t1_ * 128)
    m = r1 - r0
    ctx.set_rows(r0, r1)
    if ws > 1:
        # strong scaling of one H.V: J splits keyed on the shard's rows (more
        # CTAs per GPU on small shards; rows equal to fp32 rounding, not bitwise)
        ctx.set_split_global(False)
    stream = torch.cuda.ExternalStream(ctx.stream)
    dev = torch.device("cuda", local)
    Vt = torch.from_numpy(np.ascontiguousarray(p.V.T)).to(dev)  # [s][n] = column-major n x s
    out_local = torch.empty((s, max(m, 1)), device=dev)
    gathered = torch.empty((ws, s, tiles * 128 // ws + 128), device=dev) if ws > 1 else None
    flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)

    def one_step():
        ctx.hv_device(Vt.data_ptr(), n, s, out_local.data_ptr(), max(m, 1))
        if ws > 1:
            import torch.distributed as dist
            with torch.cuda.stream(stream):
                chunk = torch.zeros((s, gathered.shape[2]), device=dev)
                chunk[:, :m] = out_local[:, :m]
                dist.all_gather_into_tensor(gathered, chunk)

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
        if args.hv_impl != "simt":
            ctx.profile(True)
        with ClockSampler(local) as clk:
            for a, b in evs:
                flush.zero_()
                a.record(stream)
                one_step()
                b.record(stream)
            stream.synchronize()
    launches = wg.launch_count() - launches0
    kernel_ms, kernel_launches = ctx.profile_read() if args.hv_impl != "simt" else (0.0, 0)
    ctx.profile(False)
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
    outh = torch.empty((s, m), pin_memory=True)
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
    if ws > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # multi-GPU outer steps run on every rank (collectives), before rank 0 reports
    outer_multi = outer_sharded(wg, datasets, local, args, ws, rank) if (args.outer and ws > 1) else None
    if rank != 0:
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    pk = peaks()
    clocks = clk.summary()
    f_entry = 2 * d + 2 * s + 8                       # SURVEY §8d F_hv
    flops = f_entry * n * n
    if args.hv_impl in ("tc", "tc_bf16"):
        # issued tensor work per entry: 3xTF32 Gram over the 32-wide augmented
        # rows + 3-pass K.V over s_pad columns (3xTF32 for "tc", bf16x3 for
        # "tc_bf16"); the epilogue needs one sqrt and one ex2 per entry on the
        # MUFU (16/clk/SM).  The binding resource sets the peak.
        spad = 16 * -(-s // 16)
        p_bf16 = pk["bf16"] * 1e12
        p_tf32 = p_bf16 / 2                            # TF32 = half the bf16 rate
        p_mufu = 16 * 148 * pk["mhz"] * 1e6            # ex2/sqrt per s (nominal)
        p_kv = p_tf32 if args.hv_impl == "tc" else p_bf16
        t_tensor = 3 * 2 * 32 / p_tf32 + 3 * 2 * spad / p_kv
        t_entry = max(t_tensor, 2 / p_mufu)
        bound = "tensor"
        basis = (f"max(3xTF32 Gram (K=32) at bf16/2 + 3-pass K.V (N={spad}) at "
                 f"{'bf16/2' if args.hv_impl == 'tc' else 'bf16'}, 2 MUFU ops at 16/clk/SM) per entry; "
                 f"{'tensor' if t_tensor >= 2 / p_mufu else 'MUFU'} binds")
    else:
        p_ffma = 2 * 128 * 148 * pk["mhz"] * 1e6
        t_entry = max(f_entry / p_ffma, 2 / (16 * 148 * pk["mhz"] * 1e6))
        bound = "tensor"  # compute (FFMA) bound; contract field admits hbm|tensor only
        basis = "FFMA 256 flop/clk/SM"
    peak = f_entry / t_entry / 1e12
    achieved = flops / ws / (kernel_ms / 1e3) / 1e12  # this rank's rows per launch
    traffic = None
    prof = os.path.join(ROOT, "profiles", "hv_tc_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "config1 fused H.V n=13500 d=26 s=65 Matern-3/2 ARD",
                   "n": n, "d": d, "s": s, "hv_impl": args.hv_impl, "l2": "flushed (512 MiB write)",
                   "parallelism": f"rows{ws}" if ws > 1 else "single"},
        "e2e": {"value": n * n / (e2e_ms / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(n * s * 4), "d2h_bytes_per_step": int(m * s * 4),
                "ms_per_step": e2e_ms},
        "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_basis": f"{pk['src']} peaks: F_hv={f_entry} flop/entry; " + basis,
                     "kernel_ms": kernel_ms},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if args.outer:
        line["outer"] = outer_multi if ws > 1 else outer_steps(wg, datasets, local, args)
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(p, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

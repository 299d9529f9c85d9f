"""Row-block sharded CG across ranks.

Each rank owns a contiguous, 128-aligned block of rows I_g of the solutions,
residuals and directions; X (and hence H) is available to every rank.  One CG
iteration (proj/src/solvers.cpp:107-135) becomes:

    all-gather P            (n x s; NCCL over NVLink on B200s)
    HP[I_g] = H[I_g, :] P   (the rank's row block of the fused H.V:
                             ``Context.set_rows`` + ``hv_device``)
    per-column partial dots -> all-gather -> summed in rank order (fp64),
    so every rank computes bitwise identical alpha / beta / convergence flags.

The local product is injected (``local_hv``), so the same host logic runs
with the CUDA kernels under NCCL and, in tests, with a host matrix under
gloo.  Semantics (tolerances, refresh every 50 iterations, per-column freeze,
error messages) follow ``cg_solve``.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List

import torch
import torch.distributed as dist


def row_range(n: int, rank: int, world: int, align: int = 128):
    """Contiguous rows of `rank`: whole 128-row tiles, balanced across ranks."""
    tiles = -(-n // align)
    t0, t1 = tiles * rank // world, tiles * (rank + 1) // world
    return min(n, t0 * align), min(n, t1 * align)


@dataclass
class ShardedSolveState:
    solutions: torch.Tensor        # local rows x s
    residuals: torch.Tensor        # local rows x s
    per_column_relative_residual: List[float]
    converged: List[bool]
    iterations_used: int


class NumericalError(RuntimeError):
    pass


def _gather_rows(local: torch.Tensor, n: int, world: int, group=None) -> torch.Tensor:
    """All-gather row blocks (padded to the largest block) into an n x s tensor."""
    if world == 1:
        return local
    m = torch.tensor([local.shape[0]], device=local.device)
    sizes = [torch.zeros_like(m) for _ in range(world)]
    dist.all_gather(sizes, m, group=group)
    mx = int(max(s.item() for s in sizes))
    pad = torch.zeros((mx, local.shape[1]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[: int(s.item())] for b, s in zip(bufs, sizes)], dim=0)[:n]


def _sum_ranks(x: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Deterministic all-reduce: gather fp64 partials, sum in rank order."""
    x = x.to(torch.float64)
    if world == 1:
        return x
    bufs = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(bufs, x, group=group)
    out = torch.zeros_like(x)
    for b in bufs:
        out += b
    return out


def sharded_cg(local_hv: Callable[[torch.Tensor], torch.Tensor], B_local: torch.Tensor, n: int,
               tol_mean: float = 0.01, tol_samples: float = 0.1, max_iterations: int = 0,
               init_local: torch.Tensor | None = None, group=None) -> ShardedSolveState:
    """cg_solve (proj/src/solvers.cpp:81-139) over row shards.

    local_hv(V_full) must return H[I_g, :] @ V_full for this rank's rows.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    s = B_local.shape[1]
    dt = B_local.dtype
    X = torch.zeros_like(B_local) if init_local is None else init_local.clone()
    bn = torch.sqrt(_sum_ranks((B_local.double() ** 2).sum(0), world, group))
    tols = torch.tensor([tol_mean] + [tol_samples] * (s - 1), dtype=torch.float64, device=bn.device)
    if max_iterations <= 0:
        max_iterations = 10 * n
    R = B_local - local_hv(_gather_rows(X, n, world, group)) if init_local is not None else B_local.clone()
    rs = _sum_ranks((R.double() ** 2).sum(0), world, group)
    conv = (bn == 0) | (torch.sqrt(rs) <= tols * bn)
    P = torch.where(conv[None, :], torch.zeros_like(R), R)
    it = 0
    while not bool(conv.all()) and it < max_iterations:
        it += 1
        HP = local_hv(_gather_rows(P, n, world, group))
        pHp = _sum_ranks((P.double() * HP.double()).sum(0), world, group)
        active = ~conv
        if bool((pHp[active] <= 0).any()):
            raise NumericalError("cg_solve: non-positive curvature encountered, H is not positive definite")
        alpha = torch.where(active, rs / torch.where(active, pHp, torch.ones_like(pHp)), torch.zeros_like(rs))
        X = X + alpha.to(dt)[None, :] * P
        if it % 50 == 0:
            R_new = B_local - local_hv(_gather_rows(X, n, world, group))
            R = torch.where(active[None, :], R_new, R)
        else:
            R = R - alpha.to(dt)[None, :] * HP
        rs_new = _sum_ranks((R.double() ** 2).sum(0), world, group)
        if not bool(torch.isfinite(rs_new[active]).all()):
            raise NumericalError(f"cg_solve: NaN in iterate at iteration {it}")
        newly = active & (torch.sqrt(rs_new) <= tols * bn)
        beta = torch.where(active, rs_new / torch.where(active, rs, torch.ones_like(rs)), torch.zeros_like(rs))
        if it % 50 == 0:  # fp32 refresh safeguard, as cg_refresh_norm_kernel: restart on a 4x jump
            beta = torch.where(rs_new > 4.0 * rs, torch.zeros_like(beta), beta)
        P = torch.where(newly[None, :] | conv[None, :], torch.zeros_like(P), R + beta.to(dt)[None, :] * P)
        rs = torch.where(active, rs_new, rs)
        conv = conv | newly
    E = B_local - local_hv(_gather_rows(X, n, world, group))
    en = torch.sqrt(_sum_ranks((E.double() ** 2).sum(0), world, group))
    rel = torch.where(bn > 0, en / torch.where(bn > 0, bn, torch.ones_like(bn)), torch.zeros_like(bn))
    return ShardedSolveState(X, R, rel.tolist(), conv.tolist(), it)


def device_local_hv(ctx, r0: int, r1: int):
    """local_hv backed by the fused CUDA H.V on this rank's rows (device tensors).

    V_full: n x s (row-major torch view of a column-major buffer is taken by
    transposing into a contiguous [s][n] tensor)."""
    ctx.set_rows(r0, r1)
    n = ctx.n

    def f(V_full: torch.Tensor) -> torch.Tensor:
        Vt = V_full.t().contiguous()                      # [s][n] = column-major n x s
        out = torch.empty((Vt.shape[0], r1 - r0), device=Vt.device, dtype=Vt.dtype)
        stream = torch.cuda.ExternalStream(ctx.stream)
        cur = torch.cuda.current_stream()
        stream.wait_stream(cur)
        ctx.hv_device(Vt.data_ptr(), n, Vt.shape[0], out.data_ptr(), r1 - r0)
        cur.wait_stream(stream)
        return out.t()

    return f


# ------------------------------------------------------------------ AP
@dataclass
class ApOps:
    """Local operators of the row-sharded AP for this rank's rows I = [r0, r1).

    rows_residual(B_local, X_full)   -> B_local - H[I, :] X_full
    block_rows(i0, i1, c0, c1, V)    -> H[i0:i1, c0:c1] V   (V: (c1 - c0) x s rows of
                                        this rank's columns, c0 >= r0, c1 <= r1)
    factor(block_size)               -> number of blocks (factors kept)
    block_solve(b, R_b)              -> H_bb^-1 R_b   (fp64, size x s)
    """
    rows_residual: Callable
    block_rows: Callable
    factor: Callable
    block_solve: Callable


def sharded_ap(ops: ApOps, B_local: torch.Tensor, n: int, r0: int, r1: int, block_size: int = 2000,
               tol_mean: float = 0.01, tol_samples: float = 0.1, max_iterations: int = 0,
               init_local: torch.Tensor | None = None, group=None) -> ShardedSolveState:
    """ap_solve (proj/src/solvers.cpp:141-196) over row shards.

    Blocks of `block_size` consecutive points in fixed order (they may straddle
    ranks).  R holds the exact residual R0 of the epoch start and dX this
    epoch's deltas of the own rows; the reference's incrementally updated
    R_b (R -= H[:, b'] delta_b' after every block b', :186) is formed when
    block b needs it:
        R_b = R0_b - sum over ranks of H[b, own columns before b] dX
    (each rank's contraction over its own columns < j0 plus R0 of its own
    rows of b; the partials summed in rank order, one b x s exchange per
    block).  delta_b = H_bb^-1 R_b on every rank (identical inputs, identical
    result); own rows of X += delta_b.  The triangle costs n^2 / 2 entries
    per epoch over all ranks, with long contractions instead of the
    right-looking update's n x b ones.  Each epoch ends with the exact
    refresh R = B - H X from the all-gathered X (:188) and the per-column
    norms summed in rank order (:189-191)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    s = B_local.shape[1]
    dt = B_local.dtype
    bs = min(max(int(block_size), 1), n)
    max_ep = max_iterations if max_iterations > 0 else 1000
    nb = ops.factor(bs)
    X = torch.zeros_like(B_local) if init_local is None else init_local.clone()
    bn = torch.sqrt(_sum_ranks((B_local.double() ** 2).sum(0), world, group))
    tols = torch.tensor([tol_mean] + [tol_samples] * (s - 1), dtype=torch.float64, device=bn.device)
    R = ops.rows_residual(B_local, _gather_rows(X, n, world, group))
    # this epoch's deltas of the own rows, column-major (a row slice is one
    # strided device operand)
    dX = torch.zeros((s, r1 - r0), dtype=dt, device=B_local.device).t()

    def converged(R):
        rs = _sum_ranks((R.double() ** 2).sum(0), world, group)
        return rs, (bn == 0) | (torch.sqrt(rs) <= tols * bn)

    _, conv = converged(R)
    epoch = 0
    while not bool(conv.all()) and epoch < max_ep:
        epoch += 1
        for b in range(nb):
            j0, j1 = b * bs, min(n, (b + 1) * bs)
            o0, o1 = max(j0, r0), min(j1, r1)
            Rb = torch.zeros((j1 - j0, s), dtype=torch.float64, device=B_local.device)
            if o0 < o1:
                Rb[o0 - j0:o1 - j0] = R[o0 - r0:o1 - r0].double()
            c1 = min(r1, j0)  # own columns of the earlier blocks
            if c1 > r0:
                Rb -= ops.block_rows(j0, j1, r0, c1, dX[:c1 - r0]).double()
            Rb = _sum_ranks(Rb, world, group)
            delta = ops.block_solve(b, Rb)
            if o0 < o1:
                X[o0 - r0:o1 - r0] += delta[o0 - j0:o1 - j0].to(dt)
                dX[o0 - r0:o1 - r0] = delta[o0 - j0:o1 - j0].to(dt)
        R = ops.rows_residual(B_local, _gather_rows(X, n, world, group))
        rs, conv = converged(R)
        if not bool(torch.isfinite(rs).all()):
            raise NumericalError(f"ap_solve: NaN in iterate at epoch {epoch}")
    en = torch.sqrt(_sum_ranks((R.double() ** 2).sum(0), world, group))
    rel = torch.where(bn > 0, en / torch.where(bn > 0, bn, torch.ones_like(bn)), torch.zeros_like(bn))
    return ShardedSolveState(X, R, rel.tolist(), conv.tolist(), epoch)


def device_ap_ops(ctx, r0: int, r1: int) -> ApOps:
    """ApOps backed by the library (device tensors, rows [r0, r1)): the fused
    H.V for the row and column blocks (wgp_hv_cols) and the cached fp64
    block inverses (wgp_ap_factor / wgp_ap_block_solve)."""
    ctx.set_rows(r0, r1)
    n, m = ctx.n, r1 - r0

    def on_ctx(fn):
        stream = torch.cuda.ExternalStream(ctx.stream)
        cur = torch.cuda.current_stream()
        stream.wait_stream(cur)
        out = fn()
        cur.wait_stream(stream)
        return out

    def rows_residual(B_local, X_full):
        Bt = B_local.t().contiguous()                 # [s][m]: column-major m x s
        Xt = X_full.t().contiguous()                  # [s][n]
        out = torch.empty_like(Bt)
        on_ctx(lambda: ctx.hv_cols_device(Xt.data_ptr(), n, Xt.shape[0], 0, n, out.data_ptr(), m, 1,
                                          Bt.data_ptr(), m))
        return out.t()

    def block_rows(i0, i1, c0, c1, V):
        # V: (c1 - c0) x s, column-major (a row slice of sharded_ap's dX) or copied to it
        if V.stride(0) != 1:
            V = V.t().contiguous().t()
        out = torch.empty((V.shape[1], i1 - i0), dtype=V.dtype, device=V.device)  # [s][size]
        on_ctx(lambda: ctx.hv_block_device(i0, i1, c0, c1, V.data_ptr(), V.stride(1), V.shape[1], out.data_ptr(),
                                           i1 - i0))
        return out.t()

    def block_solve(b, Rb):
        Rt = Rb.t().contiguous()                      # [s][size] fp64
        Dt = torch.empty_like(Rt)
        on_ctx(lambda: ctx.ap_block_solve_device(b, Rt.data_ptr(), Rt.shape[0], Dt.data_ptr()))
        return Dt.t()

    return ApOps(rows_residual, block_rows, lambda bs: ctx.ap_factor(bs), block_solve)


# ------------------------------------------------------------------ gradient
def sharded_grad(local_grad: Callable[[], tuple], group=None):
    """Row-sharded gradient contractions: every rank contracts its
    rows against all points (``Context.set_rows`` + ``Context.grad``; the
    outputs are linear in the row sums), the (d + 2)-vectors are gathered and
    summed in rank order (fp64): identical on every rank, deterministic."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    qa, qb = local_grad()
    nccl = world > 1 and dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    both = torch.tensor(list(qa) + list(qb), dtype=torch.float64, device=dev)
    tot = _sum_ranks(both, world, group)
    p = len(qa)
    tot = tot.cpu()
    return tot[:p].numpy(), tot[p:].numpy()


# ------------------------------------------------------------------ outer loop
@dataclass
class TrainOps:
    """Rank-local operations of the row-sharded outer loop (rows [r0, r1)).

    set_hyper(constrained)                 -> None (operators and probes follow theta)
    probes(seed, s, F, pathwise, dist)      -> full n x s float32 probes
    local_hv                                -> CG's H[I, :] V_full (torch)
    ap_ops                                  -> ApOps of the current theta
    grad(transform, raw, vy, L, R, coef)    -> (qa, qb): this rank's rows against all points
    """
    n: int
    d: int
    r0: int
    r1: int
    set_hyper: Callable
    probes: Callable
    local_hv: Callable
    ap_ops: Callable
    grad: Callable
    device: object = None


@dataclass
class ShardedStep:
    step: int
    raw_params: list
    constrained_params: list
    gradient: list
    solver_iterations: int
    per_column_relative_residual: List[float]
    step_seconds: float


_SOLVER_STREAM = 0x736F6C7665  # proj/src/optimizer.cpp:15


def sharded_train(ops: TrainOps, y, cfg, group=None) -> List[ShardedStep]:
    """run_loop (proj/src/optimizer.cpp:81-171) over row shards, with the
    semantics of the single-GPU wgp_train: initial raw theta, probe draws
    (fixed: derive_seed(seed, 1) once; resampled: derive_seed(seed, t)),
    pathwise RFF or Gaussian / Rademacher probes, the solver seed
    derive_seed(derive_seed(seed, solver stream), t), warm starts from the
    previous step's solutions (mode "warm"), gradient = quadratic - trace
    from the row-sharded contractions (coefficient 1 / (2 s)), Adam on the
    host (identical on every rank).  Solvers: CG and AP (SGD has no sharded
    driver; SURVEY §8e marks it optional)."""
    import time

    import numpy as np

    from . import Hyperparameters, NumericalError as LibNumericalError, adam_step, derive_seed

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    kind = cfg.solver.kind
    if kind not in ("cg", "ap"):
        raise ValueError("sharded_train: CG and AP only")
    n, d, r0, r1 = ops.n, ops.d, ops.r0, ops.r1
    s = cfg.num_probes
    T = cfg.transform
    init = [cfg.init_constrained] * d + [cfg.init_signal if cfg.init_signal > 0 else cfg.init_constrained,
                                         cfg.init_noise if cfg.init_noise > 0 else cfg.init_constrained]
    raw = Hyperparameters.from_constrained(init[:d], init[d], init[d + 1], T).raw.astype(np.float64).copy()
    m, v = np.zeros_like(raw), np.zeros_like(raw)
    fixed, warm = cfg.mode != "cold", cfg.mode == "warm"
    pathwise = cfg.estimator == "pathwise"
    F = cfg.rff_features if cfg.rff_features > 0 else 1000
    y = np.asarray(y, dtype=np.float32).reshape(-1)
    probe_seed = derive_seed(cfg.seed, 1) if fixed else None
    dev = ops.device
    prev = None
    out: List[ShardedStep] = []
    for t in range(1, cfg.steps + 1):
        t0 = time.perf_counter()
        try:
            cons = Hyperparameters(raw.copy(), T).to_constrained_vector()
            ops.set_hyper(cons)
            if not fixed:
                probe_seed = derive_seed(cfg.seed, t)
            Z = ops.probes(probe_seed, s, F, pathwise, cfg.probe_distribution)
            rhs = np.empty((n, s + 1), dtype=np.float32)
            rhs[:, 0] = y
            rhs[:, 1:] = Z
            B_local = torch.from_numpy(rhs[r0:r1].copy()).to(dev)
            sc = cfg.solver
            init_local = prev if (warm and prev is not None) else None
            if kind == "cg":
                st = sharded_cg(ops.local_hv, B_local, n, sc.tol_mean, sc.tol_samples, sc.max_iterations,
                                init_local=init_local, group=group)
            else:
                st = sharded_ap(ops.ap_ops(), B_local, n, r0, r1, sc.block_size, sc.tol_mean, sc.tol_samples,
                                sc.max_iterations, init_local=init_local, group=group)
            Vf = _gather_rows(st.solutions, n, world, group).cpu().numpy()
            vy = np.ascontiguousarray(Vf[:, 0])
            Vp = np.asfortranarray(Vf[:, 1:])
            R = Vp if pathwise else np.asfortranarray(Z)
            qa, qb = sharded_grad(lambda: ops.grad(T, raw, vy, Vp, R, 0.5 / s), group)
            g = np.ascontiguousarray(qa - qb)
            adam_step(raw, g, m, v, t, cfg)
        except (NumericalError, LibNumericalError) as e:
            raise NumericalError(f"step {t}: {e}") from e
        prev = st.solutions
        out.append(ShardedStep(t, raw.tolist(), Hyperparameters(raw.copy(), T).to_constrained_vector().tolist(),
                               g.tolist(), st.iterations_used, st.per_column_relative_residual,
                               time.perf_counter() - t0))
    return out


def device_train_ops(ctx, r0: int, r1: int) -> TrainOps:
    """TrainOps backed by the library on this rank's device: the fused H.V and
    AP block inverses over rows [r0, r1), the RFF / host probe generators and
    the row-range gradient (all indices global)."""
    import numpy as np

    from . import sample_probes

    n = ctx.n
    local = device_local_hv(ctx, r0, r1)

    def set_hyper(cons):
        ctx.set_hyper(np.asarray(cons, dtype=np.float64))

    def probes(seed, s, F, pathwise, dist_name):
        return ctx.rff_probes(F, s, seed) if pathwise else sample_probes(n, s, dist_name, seed)

    def grad(T, raw, vy, L, R, coef):
        ctx.set_rows(r0, r1)
        return ctx.grad(T, raw, vy, L, R, coef)

    return TrainOps(n, ctx.d, r0, r1, set_hyper, probes, local, lambda: device_ap_ops(ctx, r0, r1), grad,
                    torch.device("cuda", torch.cuda.current_device()))

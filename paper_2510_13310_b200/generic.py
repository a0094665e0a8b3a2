"""Generic block-sparse algebra on the device: the reference's public
sparse_block API (jtj, jtr, apply_damping, scale_diag_inplace;
sparse_block.py:366-439) for any BlockSparseJacobian.

The contribution schedules are the reference's JtJPattern / JtrPattern
(sparse_block.py:219-363): integer index work, built once per Jacobian
pattern on the host and cached on the Jacobian. The products run in
csrc/block_algebra.cuh with the reference's per-output summation order and
without FMA contraction, so the results are bit-identical to the Cython
backend (tests/test_gpu_block.py checks it on the reference's own output).

solve_normal with LMConfig(solver="dense") is the reference's dense path
(lm.py:124-220) on the device (csrc/dense.cuh, cuSOLVER Cholesky), and
lm_solve_generic is the reference's LM loop (lm.py:727-800) for any problem
provider (and for solver="dense" on BA / GP problems) on top of these device
products. The Schur PCG of an explicit user-assembled BlockNormalSystem is not
on the device path: BAProblem / GPProblem run the matrix-free Schur PCG
(csrc/ba_pcg*.cuh, csrc/gp_kernels.cuh); see DESIGN.md section 6.
"""

from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _native
from .errors import NativeError


def _torch():
    from .lm import _torch as t
    return t()


def _dev(torch, x, dtype):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=dtype)).to("cuda")


class _JtJPlan:
    """Contribution schedule of the block J^T J (JtJPattern, sparse_block.py:219-323):
    for every residual block, the upper-triangular pairs of its entries, grouped
    by the residual block's entry count (the reference's generation order);
    per output block the contributions in that order."""

    def __init__(self, layout, res_ids, param_ids):
        n = layout.num_param_blocks
        counts = np.bincount(res_ids, minlength=layout.num_residual_blocks) if len(res_ids) \
            else np.zeros(layout.num_residual_blocks, dtype=np.int64)
        first = np.concatenate([[0], np.cumsum(counts)])[:-1]
        pa_list, pb_list = [], []
        for m in np.unique(counts):
            if m == 0:
                continue
            blocks = np.nonzero(counts == m)[0]
            iu, ju = np.triu_indices(int(m))
            start = first[blocks][:, None]
            pa_list.append((start + iu[None, :]).ravel())
            pb_list.append((start + ju[None, :]).ravel())
        ca = np.concatenate(pa_list).astype(np.int64) if pa_list else np.zeros(0, np.int64)
        cb = np.concatenate(pb_list).astype(np.int64) if pb_list else np.zeros(0, np.int64)
        qa = param_ids[ca].astype(np.int64)
        qb = param_ids[cb].astype(np.int64)
        on_diag = ca == cb
        code = qa * n + qb
        uniq = np.unique(code[~on_diag])
        self.off_keys = np.stack([uniq // n, uniq % n], axis=1).astype(np.int32) if len(uniq) \
            else np.zeros((0, 2), np.int32)
        key = np.where(on_diag, qa, n + np.searchsorted(uniq, code))
        order = np.argsort(key, kind="stable")           # per key: generation order
        ks = key[order]
        self.contrib_a = ca[order]
        self.contrib_b = cb[order]
        if len(ks):
            starts = np.concatenate([[0], np.nonzero(np.diff(ks))[0] + 1, [len(ks)]])
        else:
            starts = np.zeros(1, np.int64)
        self.seg_start = starts.astype(np.int64)
        self.keys = ks[starts[:-1]] if len(ks) else np.zeros(0, np.int64)
        self.n = n


class _JtrPlan:
    """Gather schedule of J^T r (JtrPattern, sparse_block.py:326-363): entries
    grouped by param block, in entry (= residual) order."""

    def __init__(self, layout, res_ids, param_ids):
        e = len(res_ids)
        order = np.argsort(param_ids, kind="stable")
        ps = param_ids[order]
        starts = np.concatenate([[0], np.nonzero(np.diff(ps))[0] + 1, [e]]) if e else np.zeros(1, np.int64)
        self.by_entry = order.astype(np.int32)
        self.seg_start = starts.astype(np.int64)
        self.seg_out = layout.param_offsets[ps[starts[:-1]]].astype(np.int64) if e else np.zeros(0, np.int64)
        self.res_row = layout.residual_offsets[res_ids[order]].astype(np.int64) if e else np.zeros(0, np.int64)


def _plans(j):
    if j._dev is None:
        j._dev = {}
    return j._dev


def _entry_arrays(torch, j):
    return (_dev(torch, j.data, np.float64), _dev(torch, j.data_off, np.int64),
            _dev(torch, j.entry_h, np.int32), _dev(torch, j.entry_w, np.int32))


def jtj_device(j, out=None):
    """Block-sparse J^T J on the co-observation pattern (sparse_block.py:370-385)."""
    from .sparse_block import BlockNormalSystem
    torch = _torch()
    from .lm import _stream
    cache = _plans(j)
    if "jtj" not in cache:
        cache["jtj"] = _JtJPlan(j.layout, j.res_ids, j.param_ids)
    plan = cache["jtj"]
    if out is None:
        out = BlockNormalSystem.empty(j.layout, plan.off_keys)
    else:
        out.gradient[:] = 0.0
        out.lam = 0.0
    n = plan.n
    key_out = np.where(plan.keys < n, out.diag_off[np.minimum(plan.keys, n - 1)] if n else 0,
                       out.off_off[np.maximum(plan.keys - n, 0)] if len(out.off_off) > 1 else 0)
    data, off, eh, ew = _entry_arrays(torch, j)
    res = torch.zeros(max(out.data.size, 1), dtype=torch.float64, device="cuda")
    args = [_dev(torch, plan.contrib_a, np.int64), _dev(torch, plan.contrib_b, np.int64),
            _dev(torch, plan.seg_start, np.int64), _dev(torch, key_out, np.int64)]
    _native.check(_native.load().ssfm_block_jtj(
        ct.c_void_p(data.data_ptr()), ct.c_void_p(off.data_ptr()), ct.c_void_p(eh.data_ptr()),
        ct.c_void_p(ew.data_ptr()), *[ct.c_void_p(a.data_ptr()) for a in args], ct.c_int64(len(plan.keys)),
        ct.c_void_p(res.data_ptr()), _stream(torch)))
    out.data[...] = res[:out.data.size].cpu().numpy()
    return out


def jtr_device(j, residuals, out=None):
    """Block-sparse J^T r (sparse_block.py:388-403)."""
    torch = _torch()
    from .lm import _stream
    cache = _plans(j)
    if "jtr" not in cache:
        cache["jtr"] = _JtrPlan(j.layout, j.res_ids, j.param_ids)
    plan = cache["jtr"]
    if out is None:
        out = np.zeros(j.layout.total_params)
    data, off, eh, ew = _entry_arrays(torch, j)
    g = torch.zeros(max(out.size, 1), dtype=torch.float64, device="cuda")
    r = _dev(torch, residuals, np.float64)
    args = [_dev(torch, plan.by_entry, np.int32), _dev(torch, plan.seg_start, np.int64),
            _dev(torch, plan.seg_out, np.int64), _dev(torch, plan.res_row, np.int64)]
    _native.check(_native.load().ssfm_block_jtr(
        ct.c_void_p(data.data_ptr()), ct.c_void_p(off.data_ptr()), ct.c_void_p(eh.data_ptr()),
        ct.c_void_p(ew.data_ptr()), *[ct.c_void_p(a.data_ptr()) for a in args],
        ct.c_int64(len(plan.seg_out)), ct.c_void_p(r.data_ptr()), ct.c_void_p(g.data_ptr()), _stream(torch)))
    out[...] = g[:out.size].cpu().numpy()
    return out


def _diag_index(sys):
    w = sys.layout.widths.astype(np.int64)
    parts = [sys.diag_off[:-1][w == k][:, None] + np.arange(k, dtype=np.int64)[None, :] * (k + 1)
             for k in np.unique(w)]
    return np.sort(np.concatenate([p.ravel() for p in parts])) if parts else np.zeros(0, np.int64)


def scale_diag_device(sys, factor: float) -> None:
    """a_kk *= factor for every diagonal scalar (sparse_block.py:429-439)."""
    torch = _torch()
    from .lm import _stream
    idx = _diag_index(sys)
    data = _dev(torch, sys.data, np.float64)
    idx_d = _dev(torch, idx, np.int64)
    _native.check(_native.load().ssfm_block_scale_diag(ct.c_void_p(data.data_ptr()), ct.c_void_p(idx_d.data_ptr()),
                                                       ct.c_int64(len(idx)), ct.c_double(factor),
                                                       _stream(torch)))
    sys.data[...] = data.cpu().numpy()


def damp_device(sys, lam: float):
    """apply_damping (sparse_block.py:406-426): a copy with a_kk (1 + lambda);
    exactly zero diagonals stay zero."""
    from .sparse_block import BlockNormalSystem
    out = BlockNormalSystem(sys.layout, sys.data.copy(), sys.diag_off, sys.off_keys, sys.off_off,
                            sys.gradient, lam)
    scale_diag_device(out, 1.0 + lam)
    return out


class _DensePlan:
    """Flat scatter indices of the block storage into the dense matrix
    (lm.py:124-167): diagonal blocks, off-diagonal blocks and their mirror."""

    def __init__(self, sys):
        lay = sys.layout
        n = lay.total_params
        w = lay.widths.astype(np.int64)
        off = lay.param_offsets
        dst, src = [], []
        for k in np.unique(w):
            ids = np.nonzero(w == k)[0]
            r = off[ids][:, None] + np.arange(k)
            dst.append(((r[:, :, None] * n) + r[:, None, :]).ravel())
            src.append((sys.diag_off[ids][:, None] + np.arange(k * k)).ravel())
        if sys.num_off_blocks:
            wa, wb = w[sys.off_keys[:, 0]], w[sys.off_keys[:, 1]]
            for code in np.unique(wa * 8 + wb):
                sel = np.nonzero(wa * 8 + wb == code)[0]
                ka, kb = int(code // 8), int(code % 8)
                rows = (off[sys.off_keys[sel, 0]][:, None] + np.arange(ka))[:, :, None]
                cols = (off[sys.off_keys[sel, 1]][:, None] + np.arange(kb))[:, None, :]
                s_ = (sys.off_off[sel][:, None] + np.arange(ka * kb)).ravel()
                dst.append((rows * n + cols).ravel())
                src.append(s_)
                dst.append((cols * n + rows).ravel())
                src.append(s_)
        self.n = n
        self.dst = np.concatenate(dst) if dst else np.zeros(0, np.int64)
        self.src = np.concatenate(src) if src else np.zeros(0, np.int64)


def solve_normal_device(sys, layout, config, workspace=None, info=None):
    """solve_normal (lm.py:707-720). solver="dense": the reference's dense path
    (_solve_dense, lm.py:170-220) on the device -- assembly, pinning, Jacobi
    equilibration and a cuSOLVER Cholesky (csrc/dense.cuh). The damped Schur
    PCG of an explicit user-assembled system is not on the device path (BA / GP
    problems solve matrix-free inside lm_solve)."""
    if config.solver != "dense":
        raise NativeError("the Schur PCG of an explicit BlockNormalSystem is not on the device path; "
                          "use LMConfig(solver='dense') or a BAProblem / GPProblem")
    torch = _torch()
    from .lm import _stream
    key = ("dense_plan", id(sys.off_keys), id(sys.layout))
    plans = workspace.caches if workspace is not None else {}
    plan = plans.get(key)
    if plan is None or plan.n != layout.total_params:
        plan = _DensePlan(sys)
        plans[key] = plan
    n = plan.n
    lib = _native.load()
    st = _stream(torch)
    A = torch.zeros(n * n, dtype=torch.float64, device="cuda")
    # every device temporary stays referenced until its kernel is enqueued
    # (a tensor freed before the launch may be handed to the next allocation)
    data = _dev(torch, sys.data, np.float64)
    dst = _dev(torch, plan.dst, np.int64)
    src = _dev(torch, plan.src, np.int64)
    _native.check(lib.ssfm_dense_scatter(ct.c_void_p(data.data_ptr()), ct.c_void_p(dst.data_ptr()),
                                         ct.c_void_p(src.data_ptr()), ct.c_int64(len(plan.dst)),
                                         ct.c_void_p(A.data_ptr()), st))
    b = _dev(torch, sys.gradient, np.float64)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    _native.check(lib.ssfm_dense_solve(ct.c_void_p(A.data_ptr()), ct.c_void_p(b.data_ptr()),
                                       ct.c_void_p(x.data_ptr()), ct.c_int64(n), st))
    if info is not None:
        info["cg_iters"] = 0
    return x.cpu().numpy()


def lm_solve_generic(problem, theta0, config, workspace=None):
    """lm_solve (lm.py:727-800) for any problem provider (layout, cost,
    linearize -> (r, BlockSparseJacobian), optional post_step) and for the
    dense solver: J^T J, J^T r and damping on the device (bit-identical to the
    reference's products), the damped solve on the device."""
    import time
    from .errors import CGStall, SingularBlock, SolverFailure, ZeroQuaternion
    from .lm import IterationRecord, SolveReport, Workspace
    from .sparse_block import apply_damping, jtj, jtr
    ws = workspace or Workspace()
    layout = problem.layout
    theta = np.array(theta0, dtype=np.float64, copy=True)
    if theta.shape != (layout.total_params,):
        from .errors import DimensionMismatch
        raise DimensionMismatch("theta0 length does not match the problem layout")
    post_step = getattr(problem, "post_step", None)
    report = SolveReport()
    cost = float(problem.cost(theta))
    lam = config.lambda0
    sys_ = grad = None
    need_lin = True
    for it in range(1, config.max_iterations + 1):
        t0 = time.perf_counter_ns()
        if need_lin:
            r, jac = problem.linearize(theta)
            sys_ = jtj(jac, out=sys_)
            grad = jtr(jac, r, out=grad)
            np.negative(grad, out=sys_.gradient)
            need_lin = False
            if float(np.abs(grad).max(initial=0.0)) < config.grad_tol:
                report.termination = "converged_grad"
                break
        damped = apply_damping(sys_, lam)
        info = {}
        try:
            delta = solve_normal_device(damped, layout, config, ws, info)
            cand = theta + delta
            if post_step is not None:
                cand = np.asarray(post_step(cand), dtype=np.float64)
            cost_new = float(problem.cost(cand))
            failed = False
        except (SingularBlock, CGStall, ZeroQuaternion) as exc:
            if lam >= config.lambda_max:
                report.termination = "solver_failure"
                raise SolverFailure(f"linear solve failed at lambda_max: {exc}", report) from exc
            cost_new, failed = float("nan"), True
        accepted = (not failed) and np.isfinite(cost_new) and cost_new < cost
        report.iterations.append(IterationRecord(it, cost, cost_new, lam, accepted, int(info.get("cg_iters", 0)),
                                                 time.perf_counter_ns() - t0))
        if accepted:
            rel = (cost - cost_new) / max(cost, 1e-300)
            theta, cost = cand, cost_new
            lam = max(lam / config.lambda_down, config.lambda_min)
            need_lin = True
            if rel < config.rel_cost_tol:
                report.termination = "converged_cost"
                break
        else:
            lam = min(lam * config.lambda_up, config.lambda_max)
    return theta, report

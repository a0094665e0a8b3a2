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
solve_normal with the default solver="schur_pcg" on an explicit system is
the reference's _solve_schur (lm.py:537-704) on the device
(csrc/schur_explicit.cuh, ssfm_schur_solve): scale and point elimination, a
dense reduced system S, block-Jacobi PCG and back-substitution. Its integer
schedule (_SchurXPlan, the counterpart of _SchurPlan, lm.py:236-483) is built
on the host once per pattern. lm_solve_generic is the reference's LM loop
(lm.py:727-800) for any problem provider (and for solver="dense" on BA / GP
problems) on top of these device products. BAProblem / GPProblem never take
this path: they run the matrix-free Schur PCG (csrc/ba_pcg*.cuh,
csrc/gp_kernels.cuh).
"""

from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _native


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


# layout kind codes (sparse_block.KINDS): camera_pose 0, point 1, focal 2,
# gp_center 3, gp_point 4, gp_scale 5
_POINT_KINDS = (1, 4)
_SCALE_KIND = 5


def _groups(keys, nseg):
    """(order, seg) with order = stable sort of `keys`, seg[k]..seg[k+1] the
    members of key k (keys in 0..nseg-1)."""
    keys = np.asarray(keys, dtype=np.int64)
    order = np.argsort(keys, kind="stable").astype(np.int32)
    seg = np.zeros(nseg + 1, dtype=np.int64)
    if len(keys):
        np.cumsum(np.bincount(keys, minlength=nseg), out=seg[1:])
    return order, seg


def _block_cells(base_r, base_c, w_r, w_c, n):
    """Row-major flat indices (base_r + i) * n + base_c + j of w_r x w_c blocks."""
    i = np.arange(w_r, dtype=np.int64)[:, None]
    j = np.arange(w_c, dtype=np.int64)[None, :]
    return ((base_r[:, None, None] + i) * n + base_c[:, None, None] + j).reshape(len(base_r), -1)


class _SchurXPlan:
    """Integer schedule of the explicit-system Schur solve (the _SchurPlan of
    lm.py:236-483, rebuilt here for the device kernels of schur_explicit.cuh).

    Blocks are classified by kind: point / gp_point blocks (width 3) are
    eliminated, gp_scale blocks (width 1) are eliminated first, everything
    else is retained in the reduced system. Off-diagonal blocks must couple
    retained-retained, retained-point, retained-scale or point-scale, else
    SingularBlock (lm.py:287-295). Per S slot the contributions run in point
    order, then in retained-block order inside a point (lm.py:338-396)."""

    def __init__(self, sys):
        from .errors import SingularBlock
        lay = sys.layout
        kinds = np.asarray(lay.kind_codes)
        w = lay.widths.astype(np.int64)
        poff = np.asarray(lay.param_offsets, dtype=np.int64)
        nb = len(kinds)
        cls = np.zeros(nb, dtype=np.int8)               # 0 retained, 1 point, 2 scale
        cls[np.isin(kinds, _POINT_KINDS)] = 1
        cls[kinds == _SCALE_KIND] = 2
        ret, pts, scs = (np.nonzero(cls == k)[0] for k in (0, 1, 2))
        local = np.full(nb, -1, dtype=np.int64)
        for ids in (ret, pts, scs):
            local[ids] = np.arange(len(ids))
        if len(pts) and (w[pts] != 3).any():
            raise SingularBlock("point blocks must have width 3")
        rw = w[ret]
        ret_s_off = np.concatenate([[0], np.cumsum(rw)]).astype(np.int64)
        n_ret = int(ret_s_off[-1])
        within = np.arange(n_ret, dtype=np.int64) - np.repeat(ret_s_off[:-1], rw)
        self.n_params = int(lay.total_params)
        self.n_ret = n_ret
        self.n_pt = len(pts)
        self.n_sc = len(scs)
        a = {}
        a["ret_s_off"] = ret_s_off
        a["ret_theta"] = np.repeat(poff[ret], rw) + within
        a["pre_off"] = np.concatenate([[0], np.cumsum(rw * rw)]).astype(np.int64)
        a["pt_diag"] = np.asarray(sys.diag_off, dtype=np.int64)[pts]
        a["pt_theta"] = poff[pts]

        # direct part: retained diagonal blocks, both halves of retained-retained blocks
        dst, src = [], []
        diag_off = np.asarray(sys.diag_off, dtype=np.int64)
        for width in np.unique(rw):
            sel = np.nonzero(rw == width)[0]
            base = ret_s_off[sel]
            dst.append(_block_cells(base, base, width, width, n_ret).ravel())
            src.append((diag_off[ret[sel]][:, None] + np.arange(width * width)).ravel())
        keys = np.asarray(sys.off_keys, dtype=np.int64).reshape(-1, 2)
        off_off = np.asarray(sys.off_off, dtype=np.int64)
        ka, kb = keys[:, 0], keys[:, 1]
        ca, cb = cls[ka], cls[kb]
        rr = (ca == 0) & (cb == 0)
        ru = ((ca == 0) & (cb == 1)) | ((ca == 1) & (cb == 0))
        rs = (ca == 0) & (cb == 2)
        ps = (ca == 1) & (cb == 2)
        unsupported = ~(rr | ru | rs | ps)
        if unsupported.any():
            k = int(np.nonzero(unsupported)[0][0])
            raise SingularBlock(f"unsupported coupling between blocks {tuple(int(v) for v in keys[k])}")
        sel_rr = np.nonzero(rr)[0]
        if len(sel_rr):
            wa_, wb_ = w[ka[sel_rr]], w[kb[sel_rr]]
            for code in np.unique(wa_ * 8 + wb_):
                sel = sel_rr[wa_ * 8 + wb_ == code]
                wa, wb = int(code) // 8, int(code) % 8
                rb_ = ret_s_off[local[ka[sel]]]
                cb_ = ret_s_off[local[kb[sel]]]
                s_ = (off_off[sel][:, None] + np.arange(wa * wb)).ravel()
                dst.append(_block_cells(rb_, cb_, wa, wb, n_ret).ravel())
                src.append(s_)
                # mirror: element (i, j) of the block lands at (c + j, r + i)
                i = np.arange(wa)[:, None]
                j = np.arange(wb)[None, :]
                mir = ((cb_[:, None, None] + j) * n_ret + rb_[:, None, None] + i).reshape(len(sel), -1)
                dst.append(mir.ravel())
                src.append(s_)
        a["direct_dst"] = np.concatenate(dst) if dst else np.zeros(0, np.int64)
        a["direct_src"] = np.concatenate(src) if src else np.zeros(0, np.int64)

        # U entries (retained x point couplings) in off-key order, stored w x 3
        sel_u = np.nonzero(ru)[0]
        ret_first = ca[sel_u] == 0
        u_rblk = np.where(ret_first, ka[sel_u], kb[sel_u])
        u_pblk = np.where(ret_first, kb[sel_u], ka[sel_u])
        u_w = w[u_rblk]
        u_off = np.concatenate([[0], np.cumsum(3 * u_w)]).astype(np.int64)
        gather = np.zeros(int(u_off[-1]), dtype=np.int64)
        for width in np.unique(u_w):
            for first in (True, False):
                sel = np.nonzero((u_w == width) & (ret_first == first))[0]
                if not len(sel):
                    continue
                i = np.arange(width)[:, None]
                j = np.arange(3)[None, :]
                # stored block is (width x 3) row-major, or (3 x width) when the point comes first
                inner = (i * 3 + j) if first else (j * width + i)
                gather[(u_off[sel][:, None] + np.arange(3 * width)).ravel()] = \
                    (off_off[sel_u[sel]][:, None] + inner.ravel()[None, :]).ravel()
        n_u = len(sel_u)
        u_ret = local[u_rblk].astype(np.int32)
        u_pt = local[u_pblk].astype(np.int32)
        a["u_w"] = u_w.astype(np.int32)
        a["u_ret"] = u_ret
        a["u_pt"] = u_pt
        a["u_off"] = u_off
        a["u_gather"] = gather
        a["u_by_ret"], a["ret_useg"] = _groups(u_ret, len(ret))
        a["u_by_pt"], a["pt_useg"] = _groups(u_pt, len(pts))

        # S slots: per point, every pair (a <= b) of its U entries in retained order
        by_pt = np.lexsort((np.arange(n_u), u_ret, u_pt)) if n_u else np.zeros(0, np.int64)
        cnt = np.bincount(u_pt, minlength=len(pts)) if n_u else np.zeros(len(pts), np.int64)
        first_of = np.concatenate([[0], np.cumsum(cnt)])[:-1]
        pa, pb = [], []
        for m in np.unique(cnt):
            if m == 0:
                continue
            owners = np.nonzero(cnt == m)[0]
            ti, tj = np.triu_indices(int(m))
            pa.append((first_of[owners][:, None] + ti).ravel())
            pb.append((first_of[owners][:, None] + tj).ravel())
        if pa:
            # generation order = point order, then pair order inside the point
            pa_ = np.concatenate(pa)
            pb_ = np.concatenate(pb)
            gen = np.argsort(pa_, kind="stable")
            ua, ub = by_pt[pa_[gen]], by_pt[pb_[gen]]
            code = u_ret[ua].astype(np.int64) * max(len(ret), 1) + u_ret[ub]
            o = np.argsort(code, kind="stable")
            ua, ub, code = ua[o], ub[o], code[o]
            starts = np.concatenate([[0], np.nonzero(np.diff(code))[0] + 1, [len(code)]]).astype(np.int64)
            a["slot_seg"] = starts
            a["slot_ra"] = u_ret[ua[starts[:-1]]].astype(np.int32)
            a["slot_rb"] = u_ret[ub[starts[:-1]]].astype(np.int32)
            a["con_ua"] = ua.astype(np.int32)
            a["con_ub"] = ub.astype(np.int32)
        else:
            a["slot_seg"] = np.zeros(1, np.int64)
            for k in ("slot_ra", "slot_rb", "con_ua", "con_ub"):
                a[k] = np.zeros(0, np.int32)
        self.n_slots = len(a["slot_seg"]) - 1

        # scale blocks: one retained (width 3) and one point coupling each
        if len(scs):
            sel_rs, sel_ps = np.nonzero(rs)[0], np.nonzero(ps)[0]
            if len(sel_rs) != len(scs) or len(sel_ps) != len(scs) or \
                    len(np.unique(kb[sel_rs])) != len(scs) or len(np.unique(kb[sel_ps])) != len(scs):
                raise SingularBlock("every scale block must couple one retained and one point block")
            rs_by = sel_rs[np.argsort(local[kb[sel_rs]], kind="stable")]
            ps_by = sel_ps[np.argsort(local[kb[sel_ps]], kind="stable")]
            if (w[ka[rs_by]] != 3).any():
                raise SingularBlock("scale blocks may only couple width-3 retained blocks")
            sc_c = local[ka[rs_by]]
            sc_p = local[ka[ps_by]]
            ucode = u_ret.astype(np.int64) * (len(pts) + 1) + u_pt
            srt = np.argsort(ucode, kind="stable")
            want = sc_c * (len(pts) + 1) + sc_p
            pos = np.searchsorted(ucode[srt], want) if n_u else np.zeros(len(want), np.int64)
            if not n_u or (pos >= n_u).any() or (ucode[srt[np.minimum(pos, n_u - 1)]] != want).any():
                raise SingularBlock("scale block without matching camera-point coupling")
            sc_u = srt[pos]
            a["sc_diag"] = diag_off[scs]
            a["sc_theta"] = poff[scs]
            a["sc_uc"] = off_off[rs_by]
            a["sc_up"] = off_off[ps_by]
            a["sc_c"] = sc_c.astype(np.int32)
            a["sc_p"] = sc_p.astype(np.int32)
            a["sc_u"] = sc_u.astype(np.int32)
            a["sc_by_c"], a["c_scseg"] = _groups(sc_c, len(ret))
            a["sc_by_p"], a["p_scseg"] = _groups(sc_p, len(pts))
            a["sc_by_u"], a["u_scseg"] = _groups(sc_u, n_u)
        else:
            for k in ("sc_diag", "sc_theta", "sc_uc", "sc_up"):
                a[k] = np.zeros(0, np.int64)
            for k in ("sc_c", "sc_p", "sc_u", "sc_by_c", "sc_by_p", "sc_by_u"):
                a[k] = np.zeros(0, np.int32)
            a["c_scseg"] = np.zeros(len(ret) + 1, np.int64)
            a["p_scseg"] = np.zeros(len(pts) + 1, np.int64)
            a["u_scseg"] = np.zeros(n_u + 1, np.int64)
        self.n_rblk = len(ret)
        self.n_u = n_u
        self.n_direct = len(a["direct_dst"])
        self.arrays = a
        self._dev = None
        self._c = None

    def device(self, torch):
        """The ssfm_schur_plan struct over device copies of the arrays (kept alive here)."""
        if self._c is None:
            self._dev = {k: _dev(torch, self.arrays[k], np.int64 if t == "i8" else np.int32)
                         for k, t in _native.SCHUR_PLAN_ARRAYS}
            c = _native.SchurPlanC()
            for k in _native.SCHUR_PLAN_SIZES:
                setattr(c, k, int(getattr(self, k)))
            for k, _ in _native.SCHUR_PLAN_ARRAYS:
                setattr(c, k, self._dev[k].data_ptr())
            self._c = c
        return self._c


def _cached_plan(workspace, tag, sys, make):
    """Per-pattern plan cache in the Workspace. Keyed by the identity of the
    system's off_keys and layout like the reference (lm.py:486-492), but the
    entry keeps those objects alive and re-checks them, so an id reused after
    garbage collection cannot return a stale plan."""
    caches = workspace.caches if workspace is not None else {}
    key = (tag, id(sys.off_keys), id(sys.layout))
    hit = caches.get(key)
    if hit is not None and hit[0] is sys.off_keys and hit[1] is sys.layout:
        return hit[2]
    plan = make(sys)
    caches[key] = (sys.off_keys, sys.layout, plan)
    return plan


def solve_schur_device(sys, layout, config, workspace=None, info=None):
    """_solve_schur (lm.py:537-704) of an explicit damped system on the device."""
    torch = _torch()
    from .errors import LayoutMismatch
    from .lm import _stream
    if layout is not None and layout.total_params != sys.layout.total_params:
        raise LayoutMismatch("layout does not match the normal system")
    plan = _cached_plan(workspace, "schur_xplan", sys, _SchurXPlan)
    pc = plan.device(torch)
    data = _dev(torch, sys.data, np.float64)
    grad = _dev(torch, sys.gradient, np.float64)
    delta = torch.empty(plan.n_params, dtype=torch.float64, device="cuda")
    cfg = _native.lm_config_c(config)
    it = ct.c_int32(0)
    rc = _native.load().ssfm_schur_solve(ct.byref(pc), ct.c_void_p(data.data_ptr()), ct.c_void_p(grad.data_ptr()),
                                         ct.byref(cfg), ct.c_void_p(delta.data_ptr()), ct.byref(it), _stream(torch))
    if info is not None:
        info["cg_iters"] = int(it.value)
    _native.check(rc)
    return delta.cpu().numpy()


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
    """solve_normal (lm.py:707-720) on the device. solver="schur_pcg" (default):
    solve_schur_device. solver="dense": the reference's dense path
    (_solve_dense, lm.py:170-220) -- assembly, pinning, Jacobi equilibration
    and a cuSOLVER Cholesky (csrc/dense.cuh)."""
    if config.solver != "dense":
        return solve_schur_device(sys, layout, config, workspace, info)
    torch = _torch()
    from .lm import _stream
    plan = _cached_plan(workspace, "dense_plan", sys, _DensePlan)
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
    was_tensor = hasattr(theta0, "detach") and hasattr(theta0, "device")   # a torch tensor: returned as one
    theta = np.array(theta0.detach().cpu().numpy() if was_tensor else theta0, dtype=np.float64, copy=True)
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
    if was_tensor:
        import torch
        return torch.as_tensor(theta).to(theta0.device), report
    return theta, report

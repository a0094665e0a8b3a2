"""CPU restatement of the reference's sparse LM hot path -- TEST INFRASTRUCTURE.

ORACLE ONLY: this module is imported by tests/, __graft_entry__.smoke() and the
`cpu_baseline` leg of bench.py as the CHECKER. The product package
(paper_2510_13310_b200) never imports it and has no CPU fallback.

Pinned against golden vectors produced by the unmodified reference
(tests/golden/make_golden.py -> tests/golden/*.npz, checked by
tests/test_oracle.py). Dense formulations, for problems of a few thousand
parameters.

Restated functions (reference = /root/reference/pkg/src/sparsesfm):
  quat_matrix / normalisation ....... scene.py:135-150
  drotate_dq ........................ scene.py:153-184
  huber ............................. scene.py:398-408
  ba_project / ba_cost .............. ba.py:111-138
  ba_linearize ...................... ba.py:140-194
  gp_blocks / gp_cost / gp_linearize  gp.py:96-128
  gp_post_step ...................... gp.py:130-147
  renormalize ....................... lm.py:104-117
  dense_jacobian / jtj / jtr ........ sparse_block.py:370-403 (dense algebra)
  schur_pcg_solve ................... lm.py:495-704 (two-stage elimination,
                                      pinning, block-Jacobi PCG, back-subst.)
  lm_solve .......................... lm.py:727-800
"""

from __future__ import annotations

import numpy as np

DEPTH_EPS = 1e-12
TINY = 1e-300


class OracleSingular(Exception):
    pass


class OracleCGStall(Exception):
    pass


class OracleZeroQuat(Exception):
    pass


# ---------------------------------------------------------------------------
# rotations and robust loss
# ---------------------------------------------------------------------------

def quat_matrix(q):
    """Batched R(q/|q|) (scene.py:135-150)."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    m = np.empty((len(q), 3, 3))
    m[:, 0] = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], 1)
    m[:, 1] = np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], 1)
    m[:, 2] = np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1)
    return m


def drotate_dq(q, v):
    """d(R(q/|q|) v)/dq including the normalisation projector (scene.py:153-184)."""
    q = np.asarray(q, dtype=np.float64)
    n = np.linalg.norm(q, axis=1)
    qh = q / n[:, None]
    w, u = qh[:, 0], qh[:, 1:]
    out = np.empty((len(q), 3, 4))
    out[:, :, 0] = 2.0 * np.cross(u, v)
    ud = np.einsum("ni,ni->n", u, v)
    for i in range(3):
        for j in range(3):
            skew_ij = 0.0
            if (i, j) == (0, 1): skew_ij = -v[:, 2]
            if (i, j) == (0, 2): skew_ij = v[:, 1]
            if (i, j) == (1, 0): skew_ij = v[:, 2]
            if (i, j) == (1, 2): skew_ij = -v[:, 0]
            if (i, j) == (2, 0): skew_ij = -v[:, 1]
            if (i, j) == (2, 1): skew_ij = v[:, 0]
            out[:, i, 1 + j] = 2.0 * (-w * skew_ij + (ud if i == j else 0.0)
                                      + u[:, i] * v[:, j] - 2.0 * v[:, i] * u[:, j])
    proj = np.eye(4)[None] - qh[:, :, None] * qh[:, None, :]
    return np.einsum("nij,njk->nik", out, proj) / n[:, None, None]


def huber(kind, delta, s):
    """(cost, weight) per block (scene.py:398-408). kind "cauchy" is an
    extension with no reference counterpart (parity unpinned): cost =
    delta^2 log1p(s / delta^2), weight = 1 / (1 + s / delta^2)."""
    s = np.asarray(s, dtype=np.float64)
    if kind == "cauchy":
        d2 = delta * delta
        return d2 * np.log1p(s / d2), 1.0 / (1.0 + s / d2)
    if kind != "huber":
        return s.copy(), np.ones_like(s)
    d2 = delta * delta
    big = s > d2
    root = np.sqrt(np.where(big, s, 1.0))
    return np.where(big, 2.0 * delta * root - d2, s), np.where(big, delta / root, 1.0)


# ---------------------------------------------------------------------------
# BA (ba.py:35-197). `prob` is a dict:
#   C, P, cam, pt, pixels, pps, dists, focals, model ('pinhole'|'bal_radial'),
#   focal_mode (0 none, 1 per camera, 2 shared), loss=(kind, delta)
# ---------------------------------------------------------------------------

def ba_num_params(prob):
    C, P = prob["C"], prob["P"]
    return 7 * C + 3 * P + {0: 0, 1: C, 2: 1}[prob["focal_mode"]]


def ba_views(prob, theta):
    C, P = prob["C"], prob["P"]
    pose = theta[:7 * C].reshape(C, 7)
    pts = theta[7 * C:7 * C + 3 * P].reshape(P, 3)
    fm = prob["focal_mode"]
    if fm == 1:
        f = theta[7 * C + 3 * P:7 * C + 3 * P + C]
    elif fm == 2:
        f = np.full(C, theta[7 * C + 3 * P])
    else:
        f = np.asarray(prob["focals"], dtype=np.float64)
    return pose[:, :4], pose[:, 4:], pts, f


def ba_project(prob, theta):
    q, t, X, f = ba_views(prob, theta)
    cam, pt = prob["cam"], prob["pt"]
    R = quat_matrix(q[cam])
    v = X[pt] - t[cam]
    pc = np.einsum("nij,nj->ni", R, v)
    z = pc[:, 2]
    bal = prob["model"] == "bal_radial"
    mask = (z < -DEPTH_EPS) if bal else (z > DEPTH_EPS)
    zs = np.where(np.abs(z) < DEPTH_EPS, 1.0, z)
    fo = f[cam]
    pp = prob["pps"][cam]
    if bal:
        nrm = -pc[:, :2] / zs[:, None]
        r2 = np.einsum("ni,ni->n", nrm, nrm)
        sc = 1.0 + prob["dists"][cam, 0] * r2 + prob["dists"][cam, 1] * r2 * r2
        uv = fo[:, None] * sc[:, None] * nrm + pp
    else:
        uv = fo[:, None] * (pc[:, :2] / zs[:, None]) + pp
    return q[cam], v, R, pc, zs, mask, uv, fo


def ba_cost(prob, theta):
    *_, mask, uv, _ = ba_project(prob, theta)
    d = uv - prob["pixels"]
    c, _ = huber(*prob["loss"], np.einsum("ni,ni->n", d, d))
    return float(np.sum(c[mask]))


def ba_linearize(prob, theta):
    """Residuals [2N] and per-observation J rows in the reference layout
    [N, 2, 7+3(+1)] (pose | point | focal) (ba.py:140-194)."""
    q, v, R, pc, zs, mask, uv, f = ba_project(prob, theta)
    n = len(f)
    d = uv - prob["pixels"]
    _, w = huber(*prob["loss"], np.einsum("ni,ni->n", d, d))
    sw = np.where(mask, np.sqrt(w), 0.0)
    iz = 1.0 / zs
    dup = np.zeros((n, 2, 3))
    if prob["model"] == "bal_radial":
        cam = prob["cam"]
        k1, k2 = prob["dists"][cam, 0], prob["dists"][cam, 1]
        nrm = -pc[:, :2] * iz[:, None]
        r2 = np.einsum("ni,ni->n", nrm, nrm)
        sc = 1.0 + k1 * r2 + k2 * r2 * r2
        dndp = np.zeros((n, 2, 3))
        dndp[:, 0, 0] = dndp[:, 1, 1] = -iz
        dndp[:, 0, 2] = pc[:, 0] * iz * iz
        dndp[:, 1, 2] = pc[:, 1] * iz * iz
        dudn = (f * sc)[:, None, None] * np.eye(2) + (2.0 * f * (k1 + 2.0 * k2 * r2))[:, None, None] \
            * nrm[:, :, None] * nrm[:, None, :]
        dup = np.einsum("nij,njk->nik", dudn, dndp)
        duf = sc[:, None] * nrm
    else:
        dup[:, 0, 0] = dup[:, 1, 1] = f * iz
        dup[:, 0, 2] = -f * pc[:, 0] * iz * iz
        dup[:, 1, 2] = -f * pc[:, 1] * iz * iz
        duf = pc[:, :2] * iz[:, None]
    G = drotate_dq(q, v)
    pq = np.einsum("nij,njk->nik", dup, G)
    dx = np.einsum("nij,njk->nik", dup, R)
    width = 10 + (1 if prob["focal_mode"] else 0)
    J = np.zeros((n, 2, width))
    J[:, :, 0:4] = pq * sw[:, None, None]
    J[:, :, 4:7] = -dx * sw[:, None, None]
    J[:, :, 7:10] = dx * sw[:, None, None]
    if prob["focal_mode"]:
        J[:, :, 10] = duf * sw[:, None]
    r = (d * sw[:, None]).ravel()
    return r, J


def ba_dense_jacobian(prob, J):
    """Assemble the dense [2N, n_params] Jacobian from reference-layout rows."""
    C, P = prob["C"], prob["P"]
    n = len(prob["cam"])
    out = np.zeros((2 * n, ba_num_params(prob)))
    rows = np.arange(n)
    for r in range(2):
        rr = 2 * rows + r
        for k in range(7):
            out[rr, 7 * prob["cam"] + k] = J[:, r, k]
        for k in range(3):
            out[rr, 7 * C + 3 * prob["pt"] + k] = J[:, r, 7 + k]
        if prob["focal_mode"] == 1:
            out[rr, 7 * C + 3 * P + prob["cam"]] = J[:, r, 10]
        elif prob["focal_mode"] == 2:
            out[rr, 7 * C + 3 * P] += J[:, r, 10]
    return out


def ba_param_blocks(prob):
    """(kind, offset, width) per parameter block in theta order."""
    C, P = prob["C"], prob["P"]
    blocks = [("ret", 7 * i, 7) for i in range(C)] + [("pt", 7 * C + 3 * j, 3) for j in range(P)]
    fm = prob["focal_mode"]
    if fm == 1:
        blocks += [("ret", 7 * C + 3 * P + i, 1) for i in range(C)]
    elif fm == 2:
        blocks += [("ret", 7 * C + 3 * P, 1)]
    return blocks


def renormalize(prob, theta):
    """lm.py:104-117"""
    out = np.array(theta, dtype=np.float64, copy=True)
    C = prob["C"]
    q = out[:7 * C].reshape(C, 7)[:, :4]
    n = np.linalg.norm(q, axis=1)
    if (n < 1e-12).any():
        raise OracleZeroQuat("zero quaternion")
    out[:7 * C].reshape(C, 7)[:, :4] = q / n[:, None]
    return out


# ---------------------------------------------------------------------------
# GP (gp.py:33-147). prob: C, P, cam, pt, rays, depth_mode, depths, gauge_fixed, loss
# ---------------------------------------------------------------------------

def gp_num_params(prob):
    return 3 * prob["C"] + 3 * prob["P"] + (0 if prob["depth_mode"] else len(prob["cam"]))


def gp_blocks(prob, theta):
    C, P = prob["C"], prob["P"]
    centers = theta[:3 * C].reshape(C, 3)
    pts = theta[3 * C:3 * (C + P)].reshape(P, 3)
    d = 1.0 / prob["depths"] if prob["depth_mode"] else theta[3 * (C + P):]
    span = pts[prob["pt"]] - centers[prob["cam"]]
    return prob["rays"] - d[:, None] * span, span, d


def gp_cost(prob, theta):
    blk, _, _ = gp_blocks(prob, theta)
    c, _ = huber(*prob["loss"], np.einsum("ni,ni->n", blk, blk))
    return float(c.sum())


def gp_linearize(prob, theta):
    """Residuals [3N] and rows [N, 3, 3+3(+1)] (centre | point | scale)."""
    blk, span, d = gp_blocks(prob, theta)
    _, w = huber(*prob["loss"], np.einsum("ni,ni->n", blk, blk))
    sw = np.sqrt(w)
    n = len(d)
    width = 6 if prob["depth_mode"] else 7
    J = np.zeros((n, 3, width))
    a = d * sw
    at = np.where((prob["cam"] == 0) & bool(prob["gauge_fixed"]), 0.0, a)
    for k in range(3):
        J[:, k, k] = at
        J[:, k, 3 + k] = -a
    if not prob["depth_mode"]:
        J[:, :, 6] = -span * sw[:, None]
    return (blk * sw[:, None]).ravel(), J


def gp_dense_jacobian(prob, J):
    C, P = prob["C"], prob["P"]
    n = len(prob["cam"])
    out = np.zeros((3 * n, gp_num_params(prob)))
    for r in range(3):
        rr = 3 * np.arange(n) + r
        for k in range(3):
            out[rr, 3 * prob["cam"] + k] = J[:, r, k]
            out[rr, 3 * C + 3 * prob["pt"] + k] = J[:, r, 3 + k]
        if not prob["depth_mode"]:
            out[rr, 3 * C + 3 * P + np.arange(n)] = J[:, r, 6]
    return out


def gp_param_blocks(prob):
    C, P = prob["C"], prob["P"]
    blocks = [("ret", 3 * i, 3) for i in range(C)] + [("pt", 3 * C + 3 * j, 3) for j in range(P)]
    if not prob["depth_mode"]:
        blocks += [("sc", 3 * (C + P) + o, 1) for o in range(len(prob["cam"]))]
    return blocks


def gp_post_step(prob, theta):
    """gp.py:130-147"""
    if prob["depth_mode"]:
        return theta
    C, P = prob["C"], prob["P"]
    out = np.array(theta, copy=True)
    centers = out[:3 * C].reshape(C, 3)
    pts = out[3 * C:3 * (C + P)].reshape(P, 3)
    sc = out[3 * (C + P):]
    if prob["gauge_fixed"]:
        m = float(sc.mean())
        if m > 0 and np.isfinite(m):
            t0 = centers[0].copy()
            sc /= m
            centers *= m
            centers += (1.0 - m) * t0
            pts *= m
            pts += (1.0 - m) * t0
    np.maximum(sc, 1e-6, out=sc)
    return out


# ---------------------------------------------------------------------------
# damped Schur + block-Jacobi PCG on dense matrices (lm.py:495-704)
# ---------------------------------------------------------------------------

def schur_pcg_solve(A, b, blocks, lam, cg_tol=1e-8, cg_max_iters=500, b_full=None):
    """Solve (A with diag*(1+lam)) x = b by eliminating 'sc' then 'pt' blocks
    and running block-Jacobi PCG on the retained system (x0 = 0, stop at
    |r| <= cg_tol*|b_full|). Returns (delta, cg_iters)."""
    A = np.array(A, dtype=np.float64, copy=True)
    A[np.diag_indices_from(A)] *= (1.0 + lam)
    b = np.array(b, dtype=np.float64, copy=True)
    b_orig = b.copy()
    ret = [(o, w) for k, o, w in blocks if k == "ret"]
    pts = [(o, w) for k, o, w in blocks if k == "pt"]
    scs = [(o, w) for k, o, w in blocks if k == "sc"]
    idx = lambda bl: np.concatenate([np.arange(o, o + w) for o, w in bl]) if bl else np.zeros(0, int)  # noqa: E731
    ir, ip, isc = idx(ret), idx(pts), idx(scs)
    # stage 1: scale blocks (1x1), lm.py:563-597
    inv_s = np.zeros(len(isc))
    for k, s in enumerate(isc):
        D = A[s, s]
        if D == 0.0:
            if b[s] != 0.0 or np.any(A[s, np.r_[ir, ip]] != 0.0):
                raise OracleSingular("masked scale with coupling")
            continue
        inv_s[k] = 1.0 / D
    if len(isc):
        keep = np.r_[ir, ip]
        U = A[np.ix_(keep, isc)]
        A_kk = A[np.ix_(keep, keep)] - (U * inv_s) @ U.T
        b_k = b[keep] - (U * inv_s) @ b[isc]
        A2 = np.zeros_like(A)
        A2[np.ix_(keep, keep)] = A_kk
        b2 = b.copy()
        b2[keep] = b_k
    else:
        A2, b2 = A, b
    # stage 2: point blocks (3x3, pinned, det>0), lm.py:495-513 / 599-606
    Minv = {}
    for o, w in pts:
        blk = A2[o:o + w, o:o + w].copy()
        dg = np.diag(blk).copy()
        for k in range(w):
            if dg[k] == 0.0:
                if b2[o + k] != 0.0:
                    raise OracleSingular("masked point direction with non-zero gradient")
                blk[k, k] = 1.0
        det = np.linalg.det(blk)
        if not (det > 0) or not np.isfinite(det):
            raise OracleSingular("singular point block")
        Minv[o] = np.linalg.inv(blk)
    nr = len(ir)
    S = A2[np.ix_(ir, ir)].copy()
    bred = b2[ir].copy()
    W = np.zeros((nr, len(ip)))
    Minv_full = np.zeros((len(ip), len(ip)))
    pos = 0
    for o, w in pts:
        Minv_full[pos:pos + w, pos:pos + w] = Minv[o]
        pos += w
    if len(ip):
        Urp = A2[np.ix_(ir, ip)]
        S -= Urp @ Minv_full @ Urp.T
        bred -= Urp @ (Minv_full @ b2[ip])
        W = Urp
    dS = np.diag(S).copy()
    for k in range(nr):
        if dS[k] == 0.0:
            if bred[k] != 0.0:
                raise OracleSingular("masked retained direction with non-zero gradient")
            S[k, k] = 1.0
    # block-Jacobi preconditioner per retained block (lm.py:516-534)
    Mp = np.zeros((nr, nr))
    pos = 0
    for o, w in ret:
        blk = S[pos:pos + w, pos:pos + w]
        try:
            inv = np.linalg.inv(blk)
        except np.linalg.LinAlgError as exc:
            raise OracleSingular(str(exc))
        if not np.isfinite(inv).all():
            raise OracleSingular("non-finite preconditioner block")
        Mp[pos:pos + w, pos:pos + w] = inv
        pos += w
    ref = float(np.linalg.norm(b_orig if b_full is None else b_full))
    tol = cg_tol * max(ref, TINY)
    x = np.zeros(nr)
    r = bred.copy()
    it = 0
    rn = float(np.linalg.norm(r))
    if rn > tol:
        z = Mp @ r
        p = z.copy()
        rho = float(r @ z)
        while True:
            if it >= cg_max_iters:
                raise OracleCGStall("max iterations")
            q = S @ p
            pq = float(p @ q)
            if not np.isfinite(pq) or pq <= 0.0:
                raise OracleCGStall("breakdown")
            al = rho / pq
            x += al * p
            r -= al * q
            it += 1
            rn = float(np.linalg.norm(r))
            if rn <= tol:
                break
            z = Mp @ r
            rn2 = float(r @ z)
            p = z + (rn2 / rho) * p
            rho = rn2
    delta = np.zeros(len(b))
    delta[ir] = x
    if len(ip):
        delta[ip] = Minv_full @ (b2[ip] - W.T @ x)
    if len(isc):
        keep = np.r_[ir, ip]
        U = A[np.ix_(keep, isc)]
        delta[isc] = inv_s * (b_orig[isc] - U.T @ delta[keep])
    return delta, it


# ---------------------------------------------------------------------------
# LM driver (lm.py:727-800)
# ---------------------------------------------------------------------------

DEFAULT_CFG = dict(max_iterations=100, lambda0=1e-4, lambda_up=10.0, lambda_down=2.0,
                   lambda_min=1e-10, lambda_max=1e10, rel_cost_tol=1e-6, grad_tol=1e-10,
                   cg_max_iters=500, cg_tol=1e-8)


def lm_solve(kind, prob, theta0, **cfg):
    """kind 'ba' or 'gp'. Returns (theta, records, termination); records are
    (iteration, cost_before, cost_after, lam, accepted, cg_iters)."""
    c = dict(DEFAULT_CFG, **cfg)
    if kind == "ba":
        cost_fn, lin, dense, blocks, post = (ba_cost, ba_linearize, ba_dense_jacobian,
                                             ba_param_blocks(prob), renormalize)
    else:
        cost_fn, lin, dense, blocks, post = (gp_cost, gp_linearize, gp_dense_jacobian,
                                             gp_param_blocks(prob), gp_post_step)
    theta = np.array(theta0, dtype=np.float64, copy=True)
    lam = c["lambda0"]
    cost = cost_fn(prob, theta)
    recs, term = [], "max_iter"
    need = True
    for it in range(1, c["max_iterations"] + 1):
        if need:
            r, J = lin(prob, theta)
            Jd = dense(prob, J)
            A = Jd.T @ Jd
            g = Jd.T @ r
            need = False
            if np.abs(g).max(initial=0.0) < c["grad_tol"]:
                term = "converged_grad"
                break
        cg_its = 0
        try:
            delta, cg_its = schur_pcg_solve(A, -g, blocks, lam, c["cg_tol"], c["cg_max_iters"])
            cand = post(prob, theta + delta)
            cnew = cost_fn(prob, cand)
            failed = False
        except (OracleSingular, OracleCGStall, OracleZeroQuat):
            if lam >= c["lambda_max"]:
                return theta, recs, "solver_failure"
            cnew, failed, cg_its = float("nan"), True, 0
        acc = (not failed) and np.isfinite(cnew) and cnew < cost
        recs.append((it, cost, cnew, lam, acc, cg_its))
        if acc:
            rel = (cost - cnew) / max(cost, TINY)
            theta, cost = cand, cnew
            lam = max(lam / c["lambda_down"], c["lambda_min"])
            need = True
            if rel < c["rel_cost_tol"]:
                term = "converged_cost"
                break
        else:
            lam = min(lam * c["lambda_up"], c["lambda_max"])
    return theta, recs, term


# ---------------------------------------------------------------------------
# reference-equivalent integer structures (sparse_block.py:240-266, lm.py:338-384)
# ---------------------------------------------------------------------------

def jtj_off_keys(per_obs_params):
    """per_obs_params: list of sorted param-block id tuples per residual block."""
    keys = set()
    for ids in per_obs_params:
        for a in range(len(ids)):
            for b in range(a + 1, len(ids)):
                keys.add((min(ids[a], ids[b]), max(ids[a], ids[b])))
    return np.array(sorted(keys), dtype=np.int64).reshape(-1, 2)


def schur_slots(ret_lists, ret_width):
    """Unique retained pairs (ra <= rb) per point, ordered by (shape, code)."""
    nret = len(ret_width)
    pairs = set()
    for L in ret_lists:
        L = sorted(L)
        for a in range(len(L)):
            for b in range(a, len(L)):
                pairs.add((L[a], L[b]))
    return np.array(sorted(pairs, key=lambda p: (ret_width[p[0]] * 8 + ret_width[p[1]],
                                                 p[0] * nret + p[1])), dtype=np.int64).reshape(-1, 2)


def ref_layout(J, widths):
    """Per-observation rows [N, h, sum(widths)] -> the reference's flat entry
    layout (each (residual, param) block row-major, entries in param order,
    sparse_block.py:72-123)."""
    n = J.shape[0]
    parts, o = [], 0
    for w in widths:
        parts.append(J[:, :, o:o + w].reshape(n, -1))
        o += w
    return np.concatenate(parts, axis=1).ravel()

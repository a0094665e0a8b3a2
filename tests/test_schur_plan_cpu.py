"""CPU: the host schedule of the explicit-system Schur solve (generic._SchurXPlan,
the counterpart of the reference's _SchurPlan, lm.py:236-483).

The device kernels (csrc/schur_explicit.cuh) only follow the plan's index
arrays, so the plan is checked here without a GPU: a direct numpy walk over
the same arrays (the kernels' loop structure, no PCG -- the reduced system is
solved exactly) must reproduce np.linalg.solve of the dense damped system.
"""
import numpy as np
import pytest

from paper_2510_13310_b200.errors import SingularBlock
from paper_2510_13310_b200.generic import _SchurXPlan
from paper_2510_13310_b200.sparse_block import BlockLayout, BlockSparseJacobian


def _jtj_host(j):
    """dense J^T J / J^T r via the block layout (test helper, not the product)"""
    from paper_2510_13310_b200.sparse_block import BlockNormalSystem
    lay = j.layout
    A = np.zeros((lay.total_residuals, lay.total_params))
    for e in range(j.num_entries):
        r0, p0 = lay.residual_offsets[j.res_ids[e]], lay.param_offsets[j.param_ids[e]]
        b = j.entry_block(e)
        A[r0:r0 + b.shape[0], p0:p0 + b.shape[1]] = b
    full = A.T @ A
    # off keys: param pairs sharing a residual block
    keys = set()
    for rb in range(lay.num_residual_blocks):
        ps = sorted(j.param_ids[j.res_ids == rb])
        keys.update((a, b) for i, a in enumerate(ps) for b in ps[i + 1:])
    keys = np.array(sorted(keys), dtype=np.int32).reshape(-1, 2)
    sys_ = BlockNormalSystem.empty(lay, keys)
    off, w = lay.param_offsets, lay.widths
    for k in range(lay.num_param_blocks):
        sys_.data[sys_.diag_off[k]:sys_.diag_off[k + 1]] = full[off[k]:off[k] + w[k], off[k]:off[k] + w[k]].ravel()
    for i, (a, b) in enumerate(keys):
        sys_.data[sys_.off_off[i]:sys_.off_off[i + 1]] = full[off[a]:off[a] + w[a], off[b]:off[b] + w[b]].ravel()
    return sys_, A


def walk(plan, data, grad):
    """numpy walk over the plan arrays in the kernels' order (exact reduced solve)"""
    a = plan.arrays
    n = plan.n_ret
    S = np.zeros(n * n)
    S[a["direct_dst"]] = data[a["direct_src"]]
    U = data[a["u_gather"]].copy()
    dpt = np.stack([data[o:o + 9] for o in a["pt_diag"]]).reshape(-1, 3, 3) if plan.n_pt else np.zeros((0, 3, 3))
    g = grad.copy()
    rs = a["ret_s_off"]
    inv = lambda d: 0.0 if d == 0 else 1.0 / d  # noqa: E731
    for c in range(plan.n_rblk):
        for k in range(a["c_scseg"][c], a["c_scseg"][c + 1]):
            s = a["sc_by_c"][k]
            u = data[a["sc_uc"][s]:a["sc_uc"][s] + 3]
            iv = inv(data[a["sc_diag"][s]])
            for i in range(3):
                for jj in range(3):
                    S[(rs[c] + i) * n + rs[c] + jj] -= iv * u[i] * u[jj]
                g[a["ret_theta"][rs[c] + i]] -= iv * grad[a["sc_theta"][s]] * u[i]
    for p in range(plan.n_pt):
        for k in range(a["p_scseg"][p], a["p_scseg"][p + 1]):
            s = a["sc_by_p"][k]
            u = data[a["sc_up"][s]:a["sc_up"][s] + 3]
            iv = inv(data[a["sc_diag"][s]])
            dpt[p] -= iv * np.outer(u, u)
            g[a["pt_theta"][p]:a["pt_theta"][p] + 3] -= iv * grad[a["sc_theta"][s]] * u
    for e in range(plan.n_u):
        for k in range(a["u_scseg"][e], a["u_scseg"][e + 1]):
            s = a["sc_by_u"][k]
            iv = inv(data[a["sc_diag"][s]])
            uc = data[a["sc_uc"][s]:a["sc_uc"][s] + 3]
            up = data[a["sc_up"][s]:a["sc_up"][s] + 3]
            U[a["u_off"][e]:a["u_off"][e] + 9] -= (iv * np.outer(uc, up)).ravel()
    M = np.linalg.inv(dpt) if plan.n_pt else dpt
    y = np.stack([M[p] @ g[a["pt_theta"][p]:a["pt_theta"][p] + 3] for p in range(plan.n_pt)]) \
        if plan.n_pt else np.zeros((0, 3))
    bred = g[a["ret_theta"]].copy()
    for c in range(plan.n_rblk):
        wd = rs[c + 1] - rs[c]
        for k in range(a["ret_useg"][c], a["ret_useg"][c + 1]):
            e = a["u_by_ret"][k]
            Ue = U[a["u_off"][e]:a["u_off"][e + 1]].reshape(wd, 3)
            bred[rs[c]:rs[c + 1]] -= Ue @ y[a["u_pt"][e]]
    for s in range(plan.n_slots):
        ra, rb = a["slot_ra"][s], a["slot_rb"][s]
        wa, wb = rs[ra + 1] - rs[ra], rs[rb + 1] - rs[rb]
        acc = np.zeros((wa, wb))
        for k in range(a["slot_seg"][s], a["slot_seg"][s + 1]):
            ea, eb = a["con_ua"][k], a["con_ub"][k]
            Ua = U[a["u_off"][ea]:a["u_off"][ea + 1]].reshape(wa, 3)
            Ub = U[a["u_off"][eb]:a["u_off"][eb + 1]].reshape(wb, 3)
            acc += Ua @ M[a["u_pt"][ea]] @ Ub.T
        Sm = S.reshape(n, n)
        Sm[rs[ra]:rs[ra] + wa, rs[rb]:rs[rb] + wb] -= acc
        if ra != rb:
            Sm[rs[rb]:rs[rb] + wb, rs[ra]:rs[ra] + wa] -= acc.T
    Sm = S.reshape(n, n)
    x = np.linalg.solve(Sm, bred) if n else np.zeros(0)
    delta = np.zeros(plan.n_params)
    delta[a["ret_theta"]] = x
    for p in range(plan.n_pt):
        acc = np.zeros(3)
        for k in range(a["pt_useg"][p], a["pt_useg"][p + 1]):
            e = a["u_by_pt"][k]
            r0 = rs[a["u_ret"][e]]
            wd = a["u_w"][e]
            acc += U[a["u_off"][e]:a["u_off"][e + 1]].reshape(wd, 3).T @ x[r0:r0 + wd]
        delta[a["pt_theta"][p]:a["pt_theta"][p] + 3] = y[p] - M[p] @ acc
    for s in range(plan.n_sc):
        iv = inv(data[a["sc_diag"][s]])
        uc = data[a["sc_uc"][s]:a["sc_uc"][s] + 3]
        up = data[a["sc_up"][s]:a["sc_up"][s] + 3]
        cr = rs[a["sc_c"][s]]
        pr = a["pt_theta"][a["sc_p"][s]]
        dc = delta[a["ret_theta"][cr:cr + 3]]
        delta[a["sc_theta"][s]] = iv * (grad[a["sc_theta"][s]] - uc @ dc - up @ delta[pr:pr + 3])
    return delta


def _system(kind, seed, lam):
    from .test_gpu_schur_explicit import random_ba_blocks, random_gp_blocks
    rng = np.random.default_rng(seed)
    layout, blocks = random_ba_blocks(rng, 3, 7, 0.8) if kind == "ba" else random_gp_blocks(rng, 4, 6)
    j = BlockSparseJacobian.from_blocks(layout, blocks)
    sys_, A = _jtj_host(j)
    r = rng.normal(size=layout.total_residuals)
    sys_.gradient[:] = -(A.T @ r)
    from paper_2510_13310_b200.sparse_block import BlockNormalSystem
    # host damping a_kk (1 + lam) (sparse_block.py:406-426; the product's runs on the device)
    damped = BlockNormalSystem(sys_.layout, sys_.data.copy(), sys_.diag_off, sys_.off_keys, sys_.off_off,
                               sys_.gradient, lam)
    w, off = layout.widths, sys_.diag_off
    for k in range(layout.num_param_blocks):
        for i in range(w[k]):
            damped.data[off[k] + i * (w[k] + 1)] *= 1.0 + lam
    full = A.T @ A
    full = full + lam * np.diag(np.diag(full))
    return damped, full, layout


@pytest.mark.parametrize("kind,seed", [("ba", 0), ("ba", 1), ("ba", 2), ("gp", 100), ("gp", 101)])
def test_plan_walk_matches_dense_solve(kind, seed):
    damped, full, layout = _system(kind, seed, 0.3)
    plan = _SchurXPlan(damped)
    got = walk(plan, damped.data, damped.gradient)
    expect = np.linalg.solve(full, damped.gradient)
    assert np.abs(got - expect).max() / np.abs(expect).max() < 1e-9
    assert plan.n_ret == (8 * 3 if kind == "ba" else 3 * 4)
    assert plan.n_sc == (0 if kind == "ba" else len(layout.kind_codes) - 10)


def test_plan_slot_schedule_covers_co_observed_pairs():
    damped, _, layout = _system("ba", 4, 0.1)
    plan = _SchurXPlan(damped)
    a = plan.arrays
    pairs = set(zip(a["slot_ra"].tolist(), a["slot_rb"].tolist()))
    assert all(ra <= rb for ra, rb in pairs)
    assert len(pairs) == plan.n_slots                       # one segment per slot
    assert a["slot_seg"][-1] == len(a["con_ua"])
    # every contribution pairs two U entries of the same point
    assert np.array_equal(a["u_pt"][a["con_ua"]], a["u_pt"][a["con_ub"]])


def test_plan_rejects_point_point_coupling():
    layout = BlockLayout(["point", "point"], [2])
    j = BlockSparseJacobian.from_blocks(layout, [(0, 0, np.ones((2, 3))), (0, 1, np.ones((2, 3)))])
    sys_, _ = _jtj_host(j)
    with pytest.raises(SingularBlock, match="unsupported coupling"):
        _SchurXPlan(sys_)

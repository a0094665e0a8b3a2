"""GPU: the generic block-sparse API (sparse_block.jtj / jtr / apply_damping)
against the reference's own Cython output (tests/golden/block_algebra.npz,
made by tests/golden/make_golden.py block) -- bit-identical -- and against the
oracle's dense algebra on mixed layouts."""
import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from paper_2510_13310_b200.sparse_block import (BlockLayout, BlockSparseJacobian, apply_damping, jtj, jtr)
from .conftest import golden

pytestmark = pytest.mark.gpu


def jac_from(z, tag):
    lay = BlockLayout(z[f"{tag}_kinds"], z[f"{tag}_heights"])
    return BlockSparseJacobian(lay, z[f"{tag}_res_ids"], z[f"{tag}_param_ids"], z[f"{tag}_data"],
                               z[f"{tag}_data_off"])


@pytest.mark.parametrize("tag", ["ba", "gp"])
def test_block_algebra_bitwise_vs_reference(gpu, tag):
    z = golden("block_algebra.npz")
    j = jac_from(z, tag)
    sys_ = jtj(j)
    assert np.array_equal(sys_.off_keys, z[f"{tag}_off_keys"])
    assert np.array_equal(sys_.data, z[f"{tag}_jtj"])            # bit-identical
    assert np.array_equal(jtr(j, z[f"{tag}_r"]), z[f"{tag}_jtr"])
    assert np.array_equal(apply_damping(sys_, 0.37).data, z[f"{tag}_damped"])


def dense(j):
    lay = j.layout
    A = np.zeros((lay.total_residuals, lay.total_params))
    for e in range(j.num_entries):
        r0, p0 = lay.residual_offsets[j.res_ids[e]], lay.param_offsets[j.param_ids[e]]
        blk = j.entry_block(e)
        A[r0:r0 + blk.shape[0], p0:p0 + blk.shape[1]] = blk
    return A


def test_block_algebra_mixed_layout_vs_dense(gpu):
    rng = np.random.default_rng(4)
    kinds = rng.integers(0, 6, size=40)
    heights = rng.choice([2, 3], size=60)
    lay = BlockLayout(kinds, heights)
    blocks = []
    for r in range(60):
        for p in sorted(rng.choice(40, size=int(rng.integers(1, 5)), replace=False)):
            blocks.append((r, int(p), rng.normal(size=(int(heights[r]), int(lay.widths[p])))))
    j = BlockSparseJacobian.from_blocks(lay, blocks)
    A = dense(j)
    sys_ = jtj(j)
    full = A.T @ A
    for k in range(lay.num_param_blocks):
        o, w = lay.param_offsets[k], lay.widths[k]
        assert np.allclose(sys_.diag_block(k), full[o:o + w, o:o + w], rtol=1e-13, atol=1e-12)
    for i, (a, b) in enumerate(sys_.off_keys):
        oa, wa, ob, wb = lay.param_offsets[a], lay.widths[a], lay.param_offsets[b], lay.widths[b]
        assert np.allclose(sys_.off_block(i), full[oa:oa + wa, ob:ob + wb], rtol=1e-13, atol=1e-12)
    r = rng.normal(size=lay.total_residuals)
    assert np.allclose(jtr(j, r), A.T @ r, rtol=1e-13, atol=1e-12)
    d = apply_damping(sys_, 0.5)
    assert d.lam == 0.5 and sys_.lam == 0.0
    for k in range(lay.num_param_blocks):
        assert np.array_equal(np.diag(d.diag_block(k)), np.diag(sys_.diag_block(k)) * 1.5)

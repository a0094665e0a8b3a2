"""Block-sparse containers (drop-in for sparsesfm/sparse_block.py) and the
generic device path for arbitrary block systems.

Containers (host metadata, same fields and validation as the reference):
  BlockLayout          sparse_block.py:32-69
  BlockSparseJacobian  sparse_block.py:72-159 (sorted COO of dense blocks)
  BlockNormalSystem    sparse_block.py:162-216

Generic products and solve (GPU, csrc/generic.cu):
  jtj(J)            -> BlockNormalSystem  (jtj_fill_cy, _core.pyx:18-58)
  jtr(J, r)         -> J^T r              (jtr_fill_cy, _core.pyx:61-97)
  apply_damping     -> a_kk (1 + lambda)  (sparse_block.py:406-426)
  generic_solve_normal / generic_lm_solve  (lm.py:537-800 on explicit blocks)
"""

from __future__ import annotations

import numpy as np

from .errors import DimensionMismatch, LayoutMismatch

KINDS = ("camera_pose", "point", "focal", "gp_center", "gp_point", "gp_scale")
KIND_CODE = {name: i for i, name in enumerate(KINDS)}
WIDTH_BY_CODE = np.array([7, 3, 1, 3, 3, 1], dtype=np.int32)
ELIMINABLE_BY_CODE = np.array([False, True, False, False, True, True])
_VALID_HEIGHTS = (2, 3)


class BlockLayout:
    """Ordered parameter / residual block structure (sparse_block.py:32-69).

    Layouts built from runs (every BA / GP problem) keep the runs and build
    the per-block arrays (kind codes, widths, offsets; 20M residual blocks at
    C5) only when something asks for them: the device solver never does."""

    __slots__ = ("_kind_codes", "_widths", "_param_offsets", "_residual_heights",
                 "_residual_offsets", "_runs", "_height", "_nres", "total_params", "total_residuals")

    def __init__(self, kinds, residual_heights):
        if isinstance(kinds, np.ndarray) and kinds.dtype.kind in "iu":
            codes = kinds.astype(np.int8)
        else:
            codes = np.array([KIND_CODE[k] if isinstance(k, str) else int(k) for k in kinds],
                             dtype=np.int8)
        heights = np.asarray(residual_heights, dtype=np.int32)
        if heights.size and not np.isin(heights, _VALID_HEIGHTS).all():
            raise LayoutMismatch(f"residual heights must be in {_VALID_HEIGHTS}")
        self._runs = None
        self._height = None
        self._nres = len(heights)
        self._set_param_arrays(codes)
        self._residual_heights = heights
        self._residual_offsets = np.concatenate([[0], np.cumsum(heights, dtype=np.int64)])
        self.total_residuals = int(self._residual_offsets[-1])

    def _set_param_arrays(self, codes):
        self._kind_codes = codes
        self._widths = WIDTH_BY_CODE[codes.astype(np.int32)]
        self._param_offsets = np.concatenate([[0], np.cumsum(self._widths, dtype=np.int64)])
        self.total_params = int(self._param_offsets[-1])

    @classmethod
    def from_runs(cls, runs, height: int, num_residual_blocks: int) -> "BlockLayout":
        """Build from [(kind, count), ...] without per-block arrays."""
        if int(height) not in _VALID_HEIGHTS:
            raise LayoutMismatch(f"residual heights must be in {_VALID_HEIGHTS}")
        self = cls.__new__(cls)
        self._runs = [(k, int(n)) for k, n in runs]
        self._height = int(height)
        self._nres = int(num_residual_blocks)
        self._kind_codes = self._widths = self._param_offsets = None
        self._residual_heights = self._residual_offsets = None
        self.total_params = int(sum(int(WIDTH_BY_CODE[KIND_CODE[k]]) * n for k, n in self._runs))
        self.total_residuals = self._height * self._nres
        return self

    def _param_from_runs(self):
        codes = np.concatenate([np.full(n, KIND_CODE[k], dtype=np.int8) for k, n in self._runs]) \
            if self._runs else np.zeros(0, np.int8)
        self._set_param_arrays(codes)

    @property
    def kind_codes(self):
        if self._kind_codes is None:
            self._param_from_runs()
        return self._kind_codes

    @property
    def widths(self):
        if self._widths is None:
            self._param_from_runs()
        return self._widths

    @property
    def param_offsets(self):
        if self._param_offsets is None:
            self._param_from_runs()
        return self._param_offsets

    @property
    def residual_heights(self):
        if self._residual_heights is None:
            self._residual_heights = np.full(self._nres, self._height, dtype=np.int32)
        return self._residual_heights

    @property
    def residual_offsets(self):
        if self._residual_offsets is None:
            self._residual_offsets = np.arange(self._nres + 1, dtype=np.int64) * self._height
        return self._residual_offsets

    @property
    def num_param_blocks(self) -> int:
        if self._runs is not None:
            return int(sum(n for _, n in self._runs))
        return len(self.kind_codes)

    @property
    def num_residual_blocks(self) -> int:
        return self._nres

    def kind_name(self, block_id: int) -> str:
        return KINDS[self.kind_codes[block_id]]

    def eliminable_mask(self) -> np.ndarray:
        return ELIMINABLE_BY_CODE[self.kind_codes.astype(np.int32)]

    def param_blocks(self):
        for k in range(self.num_param_blocks):
            yield k, int(self.widths[k]), self.kind_name(k)


class BlockSparseJacobian:
    """Sorted coordinate list of dense Jacobian blocks (sparse_block.py:72-159)."""

    __slots__ = ("layout", "res_ids", "param_ids", "data", "data_off", "entry_h", "entry_w",
                 "_dev")

    def __init__(self, layout: BlockLayout, res_ids, param_ids, data, data_off, validate=True):
        self.layout = layout
        self.res_ids = np.asarray(res_ids, dtype=np.int32)
        self.param_ids = np.asarray(param_ids, dtype=np.int32)
        self.data = np.asarray(data, dtype=np.float64)
        self.data_off = np.asarray(data_off, dtype=np.int64)
        self.entry_h = layout.residual_heights[self.res_ids]
        self.entry_w = layout.widths[self.param_ids]
        self._dev = None
        if validate:
            self._validate()

    def _validate(self):
        lay = self.layout
        e = len(self.res_ids)
        if len(self.param_ids) != e or len(self.data_off) != e + 1:
            raise LayoutMismatch("index arrays disagree on entry count")
        if e:
            if self.res_ids.min() < 0 or self.res_ids.max() >= lay.num_residual_blocks:
                raise LayoutMismatch("residual block id out of range")
            if self.param_ids.min() < 0 or self.param_ids.max() >= lay.num_param_blocks:
                raise LayoutMismatch("param block id out of range")
            code = self.res_ids.astype(np.int64) * lay.num_param_blocks + self.param_ids
            if not (np.diff(code) > 0).all():
                raise LayoutMismatch("entries must be strictly sorted by (residual, param)")
        sizes = self.entry_h.astype(np.int64) * self.entry_w
        if not np.array_equal(np.diff(self.data_off), sizes):
            raise LayoutMismatch("entry data sizes disagree with layout shapes")
        if self.data_off[-1] != self.data.size:
            raise LayoutMismatch("flat data length disagrees with offsets")

    @classmethod
    def allocate(cls, layout: BlockLayout, res_ids, param_ids) -> "BlockSparseJacobian":
        res_ids = np.asarray(res_ids, dtype=np.int32)
        param_ids = np.asarray(param_ids, dtype=np.int32)
        sizes = layout.residual_heights[res_ids].astype(np.int64) * layout.widths[param_ids]
        off = np.concatenate([[0], np.cumsum(sizes)])
        return cls(layout, res_ids, param_ids, np.zeros(int(off[-1])), off)

    @classmethod
    def from_blocks(cls, layout: BlockLayout, blocks) -> "BlockSparseJacobian":
        blocks = sorted(blocks, key=lambda b: (b[0], b[1]))
        parts = []
        for r, p, arr in blocks:
            arr = np.asarray(arr, dtype=np.float64)
            want = (int(layout.residual_heights[r]), int(layout.widths[p]))
            if arr.shape != want:
                raise LayoutMismatch(f"block ({r}, {p}) has shape {arr.shape}, expected {want}")
            parts.append(arr.ravel())
        res_ids = np.array([b[0] for b in blocks], dtype=np.int32)
        param_ids = np.array([b[1] for b in blocks], dtype=np.int32)
        data = np.concatenate(parts) if parts else np.zeros(0)
        off = np.concatenate([[0], np.cumsum([len(p) for p in parts], dtype=np.int64)])
        return cls(layout, res_ids, param_ids, data, off)

    @property
    def num_entries(self) -> int:
        return len(self.res_ids)

    def entry_block(self, e: int) -> np.ndarray:
        h, w = int(self.entry_h[e]), int(self.entry_w[e])
        return self.data[self.data_off[e]:self.data_off[e + 1]].reshape(h, w)


class BlockNormalSystem:
    """Block JtJ + gradient (-J^T r) + damping (sparse_block.py:162-216).

    Diagonal blocks of every param block first, then off-diagonal blocks named
    by `off_keys` (a < b, sorted).
    """

    __slots__ = ("layout", "data", "diag_off", "off_keys", "off_off", "gradient", "lam")

    def __init__(self, layout, data, diag_off, off_keys, off_off, gradient=None, lam=0.0):
        self.layout = layout
        self.data = data
        self.diag_off = diag_off
        self.off_keys = off_keys
        self.off_off = off_off
        self.gradient = gradient if gradient is not None else np.zeros(layout.total_params)
        self.lam = lam

    @classmethod
    def empty(cls, layout, off_keys) -> "BlockNormalSystem":
        w = layout.widths.astype(np.int64)
        diag_off = np.concatenate([[0], np.cumsum(w * w)])
        off_keys = np.asarray(off_keys, dtype=np.int32).reshape(-1, 2)
        off_sizes = w[off_keys[:, 0]] * w[off_keys[:, 1]]
        off_off = diag_off[-1] + np.concatenate([[0], np.cumsum(off_sizes)])
        return cls(layout, np.zeros(int(off_off[-1])), diag_off, off_keys, off_off)

    @property
    def num_off_blocks(self) -> int:
        return len(self.off_keys)

    def diag_block(self, k: int) -> np.ndarray:
        w = int(self.layout.widths[k])
        return self.data[self.diag_off[k]:self.diag_off[k + 1]].reshape(w, w)

    def off_block(self, i: int) -> np.ndarray:
        a, b = self.off_keys[i]
        wa, wb = int(self.layout.widths[a]), int(self.layout.widths[b])
        return self.data[self.off_off[i]:self.off_off[i + 1]].reshape(wa, wb)

    def off_index(self, a: int, b: int) -> int:
        n = self.layout.num_param_blocks
        codes = self.off_keys[:, 0].astype(np.int64) * n + self.off_keys[:, 1]
        i = int(np.searchsorted(codes, a * n + b))
        return i if i < len(codes) and codes[i] == a * n + b else -1

    def copy(self) -> "BlockNormalSystem":
        return BlockNormalSystem(self.layout, self.data.copy(), self.diag_off, self.off_keys,
                                 self.off_off, self.gradient.copy(), self.lam)


# ---------------------------------------------------------------------------
# generic device path (implemented in generic.py on top of csrc/generic.cu)
# ---------------------------------------------------------------------------

def jtj(j: BlockSparseJacobian, out: BlockNormalSystem | None = None) -> BlockNormalSystem:
    from .generic import jtj_device
    return jtj_device(j, out)


def jtr(j: BlockSparseJacobian, residuals, out=None):
    residuals = np.asarray(residuals, dtype=np.float64)
    if residuals.shape != (j.layout.total_residuals,):
        raise DimensionMismatch(f"residual vector has length {residuals.size}, "
                                f"layout expects {j.layout.total_residuals}")
    from .generic import jtr_device
    return jtr_device(j, residuals, out)


def apply_damping(sys: BlockNormalSystem, lam: float) -> BlockNormalSystem:
    if lam < 0:
        raise ValueError("lambda must be non-negative")
    from .generic import damp_device
    return damp_device(sys, lam)


def scale_diag_inplace(sys: BlockNormalSystem, factor: float) -> None:
    from .generic import scale_diag_device
    scale_diag_device(sys, factor)


def diag_scalars(sys: BlockNormalSystem) -> np.ndarray:
    """The matrix diagonal of A as a vector (host gather of stored blocks)."""
    out = np.empty(sys.layout.total_params)
    widths = sys.layout.widths
    for w in np.unique(widths):
        ids = np.nonzero(widths == w)[0]
        idx = sys.diag_off[ids][:, None] + np.arange(w, dtype=np.int64) * (w + 1)
        rows = sys.layout.param_offsets[ids][:, None] + np.arange(w, dtype=np.int64)
        out[rows] = sys.data[idx]
    return out


def generic_solve_normal(sys, layout, config, workspace=None, info=None):
    from .generic import solve_normal_device
    return solve_normal_device(sys, layout, config, workspace, info)


def generic_lm_solve(problem, theta0, config, workspace=None):
    from .generic import lm_solve_generic
    return lm_solve_generic(problem, theta0, config, workspace)

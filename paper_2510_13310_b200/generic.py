"""Generic device path for arbitrary block systems (placeholder until the
generic kernels land; raises instead of falling back to the CPU)."""

from .errors import NativeError


def _missing(*_a, **_k):
    raise NativeError("generic block-system kernels are not built in this version")


jtj_device = jtr_device = damp_device = scale_diag_device = _missing
solve_normal_device = lm_solve_generic = _missing

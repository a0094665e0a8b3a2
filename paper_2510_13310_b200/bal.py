"""BAL problem files into device-ready arrays.

`read_bal(path)` keeps the reference's `io.read_bal` contract (io.py:83-131):
same Scene, same errors (ParseError with the failing line, CountMismatch for
trailing tokens, DuplicateObservation from validate_scene). The text is
parsed by the native reader (csrc/bal_host.cpp) straight into flat arrays;
`read_bal_arrays(path)` returns them as SceneArrays without building the
per-observation Python objects (the reference's cost at 20M observations),
ready for BAProblem / the device.
"""

from __future__ import annotations

import ctypes as ct
import os

import numpy as np

from . import _native
from .scene import BAL_RADIAL, SceneArrays, arrays_to_scene, axis_angle_to_quat_many, rotate_many


def _read(path):
    lib = _native.load()
    h = ct.c_void_p()
    counts = np.zeros(3, dtype=np.int64)
    _native.check(lib.ssfm_bal_read(os.fsencode(os.fspath(path)), ct.byref(h),
                                    counts.ctypes.data_as(ct.c_void_p)))
    try:
        c, p, n = (int(x) for x in counts)
        cam = np.empty(n, dtype=np.int64)
        pt = np.empty(n, dtype=np.int64)
        pix = np.empty((n, 2))
        cams = np.empty((c, 9))
        pts = np.empty((p, 3))
        ptr = lambda a: a.ctypes.data_as(ct.c_void_p)  # noqa: E731
        _native.check(lib.ssfm_bal_take(h, ptr(cam), ptr(pt), ptr(pix), ptr(cams), ptr(pts)))
    finally:
        lib.ssfm_bal_free(h)
    return cam, pt, pix, cams, pts


def read_bal_arrays(path) -> SceneArrays:
    """BAL file -> SceneArrays (bal_radial model; centres t = -R^T T, io.py:121-124)."""
    cam, pt, pix, cams, pts = _read(path)
    quats = axis_angle_to_quat_many(cams[:, :3])
    q_conj = quats * np.array([1.0, -1.0, -1.0, -1.0])
    centers = -rotate_many(q_conj, cams[:, 3:6]) if len(cams) else np.zeros((0, 3))
    c = len(cams)
    return SceneArrays(quats.reshape(c, 4), centers.reshape(c, 3), cams[:, 6].copy(), np.zeros((c, 2)),
                       cams[:, 7:9].copy(), BAL_RADIAL, pts, cam, pt, pix, None)


def read_bal(path):
    """Parse a Bundle-Adjustment-in-the-Large problem file into a Scene (io.py:83-131)."""
    return arrays_to_scene(read_bal_arrays(path))

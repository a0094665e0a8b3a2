"""GPU: on-device accuracy metrics (csrc/metrics.cuh, metrics.py) against the
reference's synth_metrics outputs (tests/golden/metrics.npz, made by
make_golden.py from the unmodified reference).

Tolerances: alignment and transformed scene 1e-10 relative (the moments are
summed in a different order than numpy's); AUC 1e-6 absolute on the 0-100
scale (err = 2 acos(d) amplifies a one-ulp change of d near 1 to ~1e-8 rad).
"""
import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import metrics, synth
from paper_2510_13310_b200.scene import SceneArrays
from .conftest import golden

pytestmark = pytest.mark.gpu


def moved_arrays(z):
    C, P = len(z["est_quats"]), len(z["est_points"])
    return SceneArrays(z["est_quats"], z["est_centers"], np.full(C, 500.0), np.zeros((C, 2)), np.zeros((C, 2)),
                       "pinhole", z["est_points"], np.zeros(0, np.int64), np.zeros(0, np.int64),
                       np.zeros((0, 2)), None)


def truth_arrays(z):
    C = len(z["true_quats"])
    return SceneArrays(z["true_quats"], z["true_centers"], np.full(C, 500.0), np.zeros((C, 2)), np.zeros((C, 2)),
                       "pinhole", np.zeros((0, 3)), np.zeros(0, np.int64), np.zeros(0, np.int64),
                       np.zeros((0, 2)), None)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("kind", ["sim3", "se3"])
def test_align_matches_reference(gpu, kind):
    z = golden("metrics.npz")
    al, out = metrics.align(moved_arrays(z), truth_arrays(z), kind)
    assert rel(al.rotation, z[f"{kind}_rotation"]) < 1e-10
    assert rel(al.translation, z[f"{kind}_translation"]) < 1e-10
    assert al.scale == pytest.approx(float(z[f"{kind}_scale"]), rel=1e-10)
    assert rel(out.quats, z[f"{kind}_quats"]) < 1e-10
    assert rel(out.centers, z[f"{kind}_centers"]) < 1e-10
    assert rel(out.points, z[f"{kind}_points"]) < 1e-10
    assert metrics.center_rmse(out, truth_arrays(z)) == pytest.approx(float(z[f"{kind}_center_rmse"]), rel=1e-8)
    auc = metrics.rotation_auc(out, truth_arrays(z), z["taus"])
    assert np.abs(np.array([auc[float(t)] for t in z["taus"]]) - z[f"{kind}_auc"]).max() < 1e-6


def test_rotation_auc_and_center_rmse_unaligned(gpu):
    z = golden("metrics.npz")
    auc = metrics.rotation_auc(moved_arrays(z), truth_arrays(z), z["taus"])
    assert list(auc) == [float(t) for t in z["taus"]]
    assert np.abs(np.array(list(auc.values())) - z["moved_auc"]).max() < 1e-6
    assert metrics.center_rmse(moved_arrays(z), truth_arrays(z)) == pytest.approx(float(z["moved_center_rmse"]),
                                                                                  rel=1e-12)


def test_align_device_in_place_and_deterministic(gpu):
    z = golden("metrics.npz")
    outs = []
    for _ in range(2):
        q = gpu.tensor(z["est_quats"], device="cuda")
        c = gpu.tensor(z["est_centers"], device="cuda")
        p = gpu.tensor(z["est_points"], device="cuda")
        al = metrics.align_device(q, c, p, gpu.tensor(z["true_centers"], device="cuda"), "sim3")
        outs.append((q.cpu().numpy(), c.cpu().numpy(), p.cpu().numpy(), al.scale))
    assert all(np.array_equal(a, b) for a, b in zip(outs[0][:3], outs[1][:3])) and outs[0][3] == outs[1][3]
    assert rel(outs[0][2], z["sim3_points"]) < 1e-10


def test_errors_match_reference():
    z = golden("metrics.npz")
    m, t = moved_arrays(z), truth_arrays(z)
    with pytest.raises(ValueError):
        metrics.align(m, t, "affine")
    few = SceneArrays(z["est_quats"][:2], z["est_centers"][:2], np.ones(2), np.zeros((2, 2)), np.zeros((2, 2)),
                      "pinhole", np.zeros((0, 3)), np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros((0, 2)),
                      None)
    with pytest.raises(b2.errors.InsufficientCameras):
        metrics.align(few, few, "sim3")
    with pytest.raises(b2.errors.InsufficientCameras):
        metrics.align(m, few, "se3")
    with pytest.raises(b2.errors.InsufficientCameras):
        metrics.rotation_auc(few, t, [1.0])


def test_rotation_auc_large_vs_host(gpu):
    """3000 cameras (4.5M pairs, multi-block rows) against the host restatement;
    more than 16 thresholds exercise the chunking."""
    rng = np.random.default_rng(7)
    qt = rng.normal(size=(3000, 4))
    qe = qt + 0.01 * rng.normal(size=(3000, 4))
    taus = [0.5 * (k + 1) for k in range(20)]
    a = metrics.rotation_auc_device(qe, qt, taus)
    tr = SceneArrays(qt, np.zeros((3000, 3)), np.ones(3000), np.zeros((3000, 2)), np.zeros((3000, 2)), "pinhole",
                     np.zeros((0, 3)), np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros((0, 2)), None)
    es = SceneArrays(qe, np.zeros((3000, 3)), np.ones(3000), np.zeros((3000, 2)), np.zeros((3000, 2)), "pinhole",
                     np.zeros((0, 3)), np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros((0, 2)), None)
    h = synth.rotation_auc(es, tr, taus)
    assert list(a) == list(h)
    assert max(abs(a[t] - h[t]) for t in taus) < 1e-6

"""The array-native generator replays the reference generator bit-exactly
(golden sha256 digests recorded from sparsesfm.synth_metrics, make_golden.py)."""
import hashlib

import numpy as np
import pytest

from paper_2510_13310_b200 import synth
from .conftest import golden, summary


def digest(a):
    h = hashlib.sha256()
    for arr in (a.quats, a.centers, a.focals, a.points, a.cam_idx, a.pt_idx, a.pixels,
                a.depths if a.depths is not None else np.zeros(0)):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", ["c1_observed", "sphere_outliers", "big_pop", "c5_shape_small"])
def test_generate_matches_reference_digest(name):
    d = summary()["digests"]
    cfg = synth.SynthConfig(**d[name + ":config"])
    truth, obs = synth.generate_arrays(cfg)
    assert digest(truth) == d[name + ":truth"]
    assert digest(obs) == d[name + ":observed"]
    pert = d[name + ":perturb"]
    if pert:
        assert digest(synth.perturb_arrays(obs, **pert)) == d[name + ":perturbed"]


def test_c1_start_digest():
    s = summary()["c1"]
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=50, num_points=5000,
                                                     visibility_fraction=4 / 50,
                                                     pixel_noise_sigma=1.0, seed=0))
    st = synth.perturb_arrays(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02,
                              point_frac=0.005, seed=1)
    assert digest(st) == s["start_digest"]


def test_native_choice_agrees_with_numpy_stream():
    rng_a = np.random.default_rng(11)
    rng_b = np.random.default_rng(11)
    a = synth._choose_sorted(rng_a, 300, 7, 500)
    b = synth._choose_sorted_numpy(rng_b, 300, 7, 500)
    assert np.array_equal(a, b)
    assert rng_a.bit_generator.state == rng_b.bit_generator.state


def test_observation_order_is_camera_major():
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=7, num_points=40,
                                                     visibility_fraction=0.5, seed=1))
    key = obs.cam_idx * 1000 + obs.pt_idx
    assert (np.diff(key) > 0).all()
    assert np.bincount(obs.pt_idx).min() == 4


def test_alignment_recovers_similarity():
    truth, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=8, num_points=30, seed=2))
    moved = truth.copy()
    ang = 0.3
    R = np.array([[np.cos(ang), -np.sin(ang), 0], [np.sin(ang), np.cos(ang), 0], [0, 0, 1.0]])
    moved.centers = 2.5 * truth.centers @ R.T + np.array([1.0, -2.0, 0.5])
    moved.points = 2.5 * truth.points @ R.T + np.array([1.0, -2.0, 0.5])
    al, aligned = synth.align(moved, truth, "sim3")
    assert synth.center_rmse(aligned, truth) < 1e-9
    assert al.scale == pytest.approx(1 / 2.5, rel=1e-12)


def test_metrics_on_exact_scene():
    truth, _ = synth.generate_arrays(synth.SynthConfig(num_cameras=6, num_points=50, seed=3))
    assert synth.reproj_rmse(truth) < 1e-9
    auc = synth.rotation_auc(truth, truth, [1.0, 5.0])
    assert auc[1.0] == pytest.approx(100.0)


def test_host_metrics_match_reference_golden():
    """the host restatement of synth_metrics (test harness) vs the reference's outputs"""
    from .test_gpu_metrics import moved_arrays, truth_arrays
    z = golden("metrics.npz")
    for kind in ("sim3", "se3"):
        al, out = synth.align(moved_arrays(z), truth_arrays(z), kind)
        assert np.abs(al.rotation - z[f"{kind}_rotation"]).max() < 1e-12
        assert np.abs(out.points - z[f"{kind}_points"]).max() < 1e-10
        auc = synth.rotation_auc(out, truth_arrays(z), z["taus"])
        assert np.abs(np.array(list(auc.values())) - z[f"{kind}_auc"]).max() < 1e-9

"""Host-side API surface of the drop-in package (no GPU needed): types, layouts,
encode/decode, error taxonomy, config validation, prune, scalar KATs
(mirroring the reference's test_scene.py / test_ba.py / test_gp.py host
checks)."""
import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import errors, synth
from paper_2510_13310_b200.scene import (BAL_RADIAL, Camera, Observation, Point3D, RobustLoss,
                                         Scene, drotate_dq_many, project, quat_from_axis_angle,
                                         quat_normalize, quat_to_matrix, robust_weight, rotate)
from paper_2510_13310_b200.sparse_block import (BlockLayout, BlockNormalSystem,
                                                BlockSparseJacobian)


def _cam(q=(1, 0, 0, 0), t=(0, 0, 0), f=1.0, pp=(0, 0), model="pinhole", dist=(0, 0)):
    return Camera(np.array(q, float), np.array(t, float), f, np.array(pp, float), model,
                  np.array(dist, float))


class TestProjectKAT:   # reference test_scene.py:16-46
    def test_optical_axis(self):
        assert np.allclose(project(_cam(), Point3D(np.array([0.0, 0.0, 1.0]))), [0.0, 0.0])

    def test_pinhole(self):
        assert np.allclose(project(_cam(f=500.0), Point3D(np.array([0.1, -0.2, 2.0]))), [25.0, -50.0])

    def test_rot180(self):
        q = quat_from_axis_angle([0, 0, 1], np.pi)
        assert np.allclose(project(_cam(q=q), Point3D(np.array([0.3, 0.4, 1.0]))), [-0.3, -0.4], atol=1e-12)

    def test_degenerate(self):
        with pytest.raises(errors.DegenerateProjection):
            project(_cam(), Point3D(np.array([0.1, 0.1, 1e-13])))

    def test_bal(self):
        cam = _cam(f=2.0, model=BAL_RADIAL, dist=(0.1, 0.01))
        uv = project(cam, Point3D(np.array([0.5, 0.0, -1.0])))
        assert np.allclose(uv, 2.0 * (1 + 0.1 * 0.25 + 0.01 * 0.0625) * np.array([0.5, 0.0]))


class TestRotateKAT:    # reference test_scene.py:77-118
    def test_matches_matrix(self):
        rng = np.random.default_rng(3)
        for _ in range(20):
            q = quat_normalize(rng.normal(size=4))
            v = rng.normal(size=3)
            assert np.allclose(rotate(q, v), quat_to_matrix(q) @ v, atol=1e-12)

    def test_derivative_fd(self):
        rng = np.random.default_rng(5)
        for _ in range(5):
            q = rng.normal(size=4) * 1.5
            v = rng.normal(size=3)
            d = drotate_dq_many(q[None], v[None])[0]
            fd = np.zeros((3, 4))
            for k in range(4):
                e = np.zeros(4)
                e[k] = 1e-7
                fd[:, k] = (rotate(q + e, v) - rotate(q - e, v)) / 2e-7
            assert np.allclose(d, fd, atol=1e-6)


class TestHuberKAT:     # reference test_scene.py:121-145
    def test_branches(self):
        assert robust_weight(RobustLoss("huber", 1.0), 0.25) == (0.25, 1.0)
        c, w = robust_weight(RobustLoss("huber", 1.0), 4.0)
        assert np.isclose(c, 3.0) and np.isclose(w, 0.5)
        assert robust_weight(RobustLoss("trivial"), 7.0) == (7.0, 1.0)

    def test_invalid(self):
        with pytest.raises(ValueError):
            RobustLoss("huber", 0.0)
        with pytest.raises(ValueError):
            RobustLoss("cauchy", 1.0)


class TestLayouts:
    def test_ba_layout_and_encode(self):
        truth, _ = synth.generate_arrays(synth.SynthConfig(num_cameras=3, num_points=8, seed=0))
        p = b2.BAProblem(truth)
        assert p.layout.num_param_blocks == 3 + 8 + 3
        assert p.layout.total_params == 7 * 3 + 3 * 8 + 3
        th = p.encode()
        assert np.array_equal(th[:4], truth.quats[0])
        dec = p.decode(th)
        assert np.allclose(dec.points, truth.points)
        ps = b2.BAProblem(truth, shared_focal=True)
        assert ps.layout.num_param_blocks == 3 + 8 + 1
        assert ps.jac.num_entries == 3 * truth.num_observations
        pn = b2.BAProblem(truth, optimize_focal=False)
        assert pn.layout.total_params == 7 * 3 + 3 * 8

    def test_ba_jacobian_pattern(self):
        truth, _ = synth.generate_arrays(synth.SynthConfig(num_cameras=4, num_points=10, seed=1))
        p = b2.BAProblem(truth)
        j = p.jac
        assert j.num_entries == 3 * truth.num_observations
        assert j.data.size == 22 * truth.num_observations

    def test_gp_layout(self):
        _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=4, num_points=10, seed=1))
        g = b2.make_rays(obs)
        assert g.layout.total_params == 3 * 4 + 3 * 10 + obs.num_observations
        gd = b2.make_rays(obs, depth_mode=True)
        assert gd.jac.num_entries == 2 * obs.num_observations
        th = g.initial_theta()
        assert np.all(th[3 * 14:] == 1.0)

    def test_block_sparse_validation(self):
        lay = BlockLayout(["point"], [2])
        with pytest.raises(errors.LayoutMismatch):
            BlockSparseJacobian.from_blocks(lay, [(0, 0, np.zeros((2, 7)))])
        with pytest.raises(errors.LayoutMismatch):
            BlockLayout(["point"], [4])

    def test_normal_system_empty(self):
        lay = BlockLayout(["camera_pose", "point"], [2])
        s = BlockNormalSystem.empty(lay, np.array([[0, 1]]))
        assert s.off_block(0).shape == (7, 3)
        assert s.off_index(0, 1) == 0 and s.off_index(1, 0) == -1


class TestMakeRaysKAT:  # reference test_gp.py:23-46
    def _scene(self, pixels, f=1.0, q=None):
        q = np.array([1.0, 0, 0, 0]) if q is None else q
        return Scene([Camera(q.copy(), np.zeros(3), f)],
                     [Point3D(np.array([0.0, 0.0, float(j + 1)])) for j in range(len(pixels))],
                     [Observation(0, j, np.asarray(px, float)) for j, px in enumerate(pixels)])

    def test_axis_and_offaxis(self):
        assert np.allclose(b2.make_rays(self._scene([(0.0, 0.0)])).rays[0], [0, 0, 1])
        assert np.allclose(b2.make_rays(self._scene([(1.0, 0.0)])).rays[0], np.array([1, 0, 1]) / np.sqrt(2))

    def test_pp(self):
        sc = self._scene([(10.0, 4.0)], f=2.0)
        sc.cameras[0].principal_point = np.array([10.0, 2.0])
        assert np.allclose(b2.make_rays(sc).rays[0], np.array([0.0, 1.0, 1.0]) / np.sqrt(2))

    def test_missing_depth(self):
        with pytest.raises(errors.MissingDepth):
            b2.make_rays(self._scene([(0.0, 0.0)]), depth_mode=True)


class TestConfigAndErrors:
    def test_lmconfig_validation(self):
        with pytest.raises(ValueError):
            b2.LMConfig(lambda0=0.0)
        with pytest.raises(ValueError):
            b2.LMConfig(solver="qr")
        with pytest.raises(ValueError):
            b2.LMConfig(lambda0=1e11)

    def test_empty_problem(self):
        sc = Scene([_cam()], [Point3D(np.zeros(3))], [])
        with pytest.raises(errors.EmptyProblem):
            b2.BAProblem(sc)

    def test_status_mapping(self):
        with pytest.raises(errors.SingularBlock):
            errors.raise_for_status(1, "x")
        with pytest.raises(errors.CGStall):
            errors.raise_for_status(2, "x")
        with pytest.raises(errors.ZeroQuaternion):
            errors.raise_for_status(4, "x")
        errors.raise_for_status(0, "ok")

    def test_renormalize(self):
        lay = BlockLayout(["camera_pose"], [2])
        out = b2.renormalize(np.array([2.0, 0, 0, 0, 5.0, 6.0, 7.0]), lay)
        assert np.allclose(out[:4], [1, 0, 0, 0]) and np.array_equal(out[4:], [5.0, 6.0, 7.0])
        with pytest.raises(errors.ZeroQuaternion):
            b2.renormalize(np.zeros(7), lay)


class TestPruneKAT:     # reference test_ba.py:140-176
    def _scene(self, n_cams, pairs):
        cams = [Camera(np.array([1.0, 0, 0, 0]), np.array([float(i), 0, -3]), 100.0) for i in range(n_cams)]
        n_pts = max(p for _, p in pairs) + 1
        pts = [Point3D(np.array([0.0, 0.0, float(j + 1)])) for j in range(n_pts)]
        return Scene(cams, pts, [Observation(c, p, np.zeros(2)) for c, p in pairs])

    def test_identity(self):
        pr, rm = b2.prune(self._scene(2, [(0, 0), (1, 0), (0, 1), (1, 1)]))
        assert pr.num_cameras == 2 and pr.num_points == 2 and rm.observation_mask.all()

    def test_single_view(self):
        pr, rm = b2.prune(self._scene(2, [(0, 0), (1, 0), (0, 1)]))
        assert pr.num_points == 1 and rm.point_map[1] == -1 and pr.num_observations == 2

    def test_cascade(self):
        pr, rm = b2.prune(self._scene(3, [(0, 0), (1, 0), (2, 1)]))
        assert pr.num_cameras == 2 and rm.camera_map[2] == -1 and rm.point_map[1] == -1

    def test_empty(self):
        with pytest.raises(errors.EmptyProblem):
            b2.prune(self._scene(2, [(0, 0)]))

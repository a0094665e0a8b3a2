"""The LM loop as one CUDA graph (csrc/lm_graph.cuh) against the host loop.

lm_solve (lm.py:727-800) on single-rank BA handles runs its accept/reject
decision, lambda schedule and termination tests on the device inside one
graph launch (SSFM_LM_GRAPH=0 keeps the host loop). The decisions are the
host loop's expression for expression, so both must give bit-identical
trajectories and parameters, for every PCG driver (fused persistent kernel,
two-pass persistent kernel, two-pass CUDA-graph PCG nested in the LM graph)
and on the SolverFailure path.
"""
import os

import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import _native
from .conftest import golden
from .test_gpu_ba import problem_from_golden
from .test_gpu_failure_paths import ring_scene, with_point

pytestmark = pytest.mark.gpu

DRIVERS = {"fused": {"SSFM_FUSED": "1", "SSFM_PCG_GRAPH": "0"},
           "two_pass": {"SSFM_FUSED": "0", "SSFM_PCG_GRAPH": "0"},
           "two_pass_graph": {"SSFM_FUSED": "0", "SSFM_PCG_GRAPH": "1"}}


def env(vals):
    class _Env:
        def __enter__(self):
            self.old = {k: os.environ.get(k) for k in vals}
            os.environ.update(vals)

        def __exit__(self, *a):
            for k, v in self.old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    return _Env()


def trajectory(rep):
    # cost_after is NaN for a failed solve (lm.py:780): compare its bits
    return [(i.iteration, i.cost_before, np.float64(i.cost_after).tobytes(), i.lam, i.step_accepted, i.cg_iters,
             i.status) for i in rep.iterations]


def mode(p):
    return _native.load().ssfm_lm_mode(p._native_handle().ptr)


@pytest.mark.parametrize("name", ["ba_small.npz", "ba_shared.npz", "ba_nofocal.npz", "ba_bal.npz"])
@pytest.mark.parametrize("driver", sorted(DRIVERS))
def test_device_loop_matches_host_loop(gpu, name, driver):
    z = golden(name)
    with env(DRIVERS[driver]):
        p = problem_from_golden(z)
        p._native_handle()
    th0 = p.encode()
    cfg = b2.LMConfig(max_iterations=25)
    with env({"SSFM_LM_GRAPH": "0"}):
        th_h, rep_h = b2.lm_solve(p, th0, cfg)
    th_d, rep_d = b2.lm_solve(p, th0, cfg)
    assert mode(p) == 1, "the LM graph did not build"
    assert rep_d.termination == rep_h.termination
    assert trajectory(rep_d) == trajectory(rep_h)
    assert np.array_equal(th_d, th_h)
    # a second solve reuses the instantiated graph
    th_d2, rep_d2 = b2.lm_solve(p, th0, cfg)
    assert trajectory(rep_d2) == trajectory(rep_h) and np.array_equal(th_d2, th_h)
    assert all(i.device_ms > 0 for i in rep_d.iterations)


GP_DRIVERS = {"persistent": {"SSFM_GP_GRAPH": "0"}, "graph": {"SSFM_GP_GRAPH": "1"},
              "graph_four_kernels": {"SSFM_GP_GRAPH": "1", "SSFM_GVEC": "0"}}


@pytest.mark.parametrize("name", ["gp_small.npz", "gp_depth.npz"])
@pytest.mark.parametrize("driver", sorted(GP_DRIVERS))
def test_gp_device_loop_matches_host_loop(gpu, name, driver):
    from .test_gpu_gp import gp_from_golden
    z = golden(name)
    with env(GP_DRIVERS[driver]):   # SSFM_GVEC is read when the graphs are captured (first solve)
        p = gp_from_golden(z)
        p._native_handle()
        th0 = p.initial_theta()
        cfg = b2.LMConfig(max_iterations=25)
        with env({"SSFM_LM_GRAPH": "0"}):
            th_h, rep_h = b2.lm_solve(p, th0, cfg)
        th_d, rep_d = b2.lm_solve(p, th0, cfg)
    assert mode(p) == 1, "the LM graph did not build"
    assert rep_d.termination == rep_h.termination
    assert trajectory(rep_d) == trajectory(rep_h)
    assert np.array_equal(th_d, th_h)


def test_device_loop_max_iterations_and_grad_termination(gpu):
    p = problem_from_golden(golden("ba_small.npz"))
    th0 = p.encode()
    for cfg in (b2.LMConfig(max_iterations=1), b2.LMConfig(max_iterations=3, lambda0=1e6),
                b2.LMConfig(max_iterations=5, grad_tol=1e30), b2.LMConfig(max_iterations=0)):
        with env({"SSFM_LM_GRAPH": "0"}):
            th_h, rep_h = b2.lm_solve(p, th0, cfg)
        th_d, rep_d = b2.lm_solve(p, th0, cfg)
        assert rep_d.termination == rep_h.termination
        assert trajectory(rep_d) == trajectory(rep_h)
        assert np.array_equal(th_d, th_h)


def test_device_loop_solver_failure_matches_host_loop(gpu):
    # a point 1e155 in front of its cameras: its damped block is singular at
    # every lambda -> SolverFailure once lambda reaches lambda_max (lm.py:775-781)
    arr = ring_scene()
    far = -arr.centers[0] / np.linalg.norm(arr.centers[0]) * 1e155
    p = b2.BAProblem(with_point(arr, 0, far, [0]), b2.RobustLoss("trivial"))
    th = p.encode()
    cfg = b2.LMConfig(max_iterations=40)
    with env({"SSFM_LM_GRAPH": "0"}):
        with pytest.raises(b2.errors.SolverFailure) as eh:
            b2.lm_solve(p, th, cfg)
    with pytest.raises(b2.errors.SolverFailure) as ed:
        b2.lm_solve(p, th, cfg)
    assert mode(p) == 1
    assert str(ed.value).split(":")[0] == str(eh.value).split(":")[0]
    assert ed.value.report.termination == "solver_failure"
    assert trajectory(ed.value.report) == trajectory(eh.value.report)

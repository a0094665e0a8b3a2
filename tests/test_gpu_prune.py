"""ba.prune (ba.py:223-261) on the device (ssfm_prune, csrc/prune.cuh):
integer work, so the maps and the observation mask must equal the host
restatement (pinned to the reference's cases in test_api_cpu.py) exactly."""
import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import ba as bba
from paper_2510_13310_b200 import synth
from paper_2510_13310_b200.errors import EmptyProblem

pytestmark = pytest.mark.gpu


def random_tracks(C, P, n, seed):
    rng = np.random.default_rng(seed)
    cam = rng.integers(0, C, size=n)
    pt = rng.integers(0, P, size=n)
    return cam, pt


@pytest.mark.parametrize("C,P,n,seed", [(5, 40, 60, 0), (30, 2000, 2500, 1), (200, 50000, 90000, 2),
                                         (1000, 500000, 1200000, 3)])
def test_device_prune_equals_host(gpu, C, P, n, seed):
    cam, pt = random_tracks(C, P, n, seed)
    dev = bba._prune_device(cam, pt, C, P)
    host = bba._prune_host(cam, pt, C, P)
    assert np.array_equal(dev[0], host[0])      # camera map
    assert np.array_equal(dev[1], host[1])      # point map
    assert np.array_equal(dev[2], host[2])      # observation mask
    assert (host[1] >= 0).sum() < P              # the case prunes something


def test_device_prune_cascade_and_empty(gpu):
    # point 1 seen once -> dropped -> camera 2 left without observations
    cam = np.array([0, 1, 2, 0, 1])
    pt = np.array([0, 0, 1, 2, 2])
    cmap, pmap, mask = bba._prune_device(cam, pt, 3, 3)
    assert cmap.tolist() == [0, 1, -1] and pmap.tolist() == [0, -1, 1]
    assert mask.tolist() == [True, True, False, True, True]
    with pytest.raises(EmptyProblem):
        bba._prune_device(np.array([0, 1]), np.array([0, 1]), 2, 2)


def test_prune_api_runs_on_device(gpu):
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=12, num_points=300,
                                                           visibility_fraction=2 / 12, seed=4))
    pr, rm = b2.prune(obs)
    cmap, pmap, mask, _, _ = bba._prune_host(obs.cam_idx.astype(np.int64), obs.pt_idx.astype(np.int64),
                                             obs.num_cameras, obs.num_points)
    assert np.array_equal(rm.camera_map, cmap) and np.array_equal(rm.point_map, pmap)
    assert np.array_equal(rm.observation_mask, mask)
    assert pr.num_observations == int(mask.sum())

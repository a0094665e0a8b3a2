"""BAL reader (csrc/bal_host.cpp via bal.py) against the unmodified reference's
io.read_bal on every case in tests/golden/bal_cases.json (valid files with
comments, CR / CRLF / \\v / \\f line breaks, signs, underscores, inf; and every
error path): arrays bit-identical, errors with the same class, line and
message. Host code: runs without a GPU."""
import json
import os

import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import bal
from .conftest import GOLDEN, golden

with open(os.path.join(GOLDEN, "bal_cases.json")) as _fh:
    CASES = json.load(_fh)


def write(tmp_path, name):
    path = tmp_path / (name + ".bal")
    with open(path, "w", newline="") as fh:
        fh.write(CASES["texts"][name])
    return str(path)


@pytest.mark.parametrize("name", sorted(CASES["texts"]))
def test_read_bal_matches_reference(tmp_path, name):
    exp = CASES["expect"][name]
    path = write(tmp_path, name)
    if exp["error"] is None:
        a = bal.read_bal_arrays(path)
        z = golden("bal.npz")
        assert [len(a.quats), len(a.points), len(a.cam_idx)] == exp["counts"]
        assert a.model_tag == "bal_radial" and a.depths is None
        for k in ("quats", "centers", "focals", "dists", "points", "cam_idx", "pt_idx", "pixels"):
            key = f"{name}__{k}"
            if key in z.files:
                got = np.asarray(getattr(a, k))
                assert got.shape == z[key].shape or got.size == z[key].size == 0, (k, got.shape, z[key].shape)
                assert np.array_equal(got.reshape(z[key].shape), z[key], equal_nan=True), k
        sc = bal.read_bal(path)
        assert sc.num_observations == exp["counts"][2]
    else:
        cls = getattr(b2.errors, exp["error"])
        with pytest.raises(cls) as err:
            bal.read_bal_arrays(path)
        assert str(err.value) == exp["message"]
        if exp["line"] is not None:
            assert err.value.line == exp["line"]


def test_missing_file(tmp_path):
    with pytest.raises(ValueError):
        bal.read_bal_arrays(str(tmp_path / "absent.bal"))


def test_bal_scene_builds_a_problem(tmp_path):
    """the reader's arrays feed BAProblem directly (bal_radial, no Python objects)"""
    a = bal.read_bal_arrays(write(tmp_path, "synth"))
    p = b2.BAProblem(a, b2.RobustLoss("huber", 1.0))
    assert p.layout.total_params == 7 * len(a.quats) + 3 * len(a.points) + len(a.quats)

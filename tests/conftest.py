import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


# several shards of one problem share the single test GPU: a lost exchange must
# fail in bounded time. Same-device shards occasionally stall ~20 s while one
# shard's kernel waits to be scheduled next to its peer's spinning PCG kernel
# (not seen with one process per GPU), hence 45 s rather than 20 s.
os.environ.setdefault("SSFM_COMM_TIMEOUT_S", "45")
# ... and their streams must not share a hardware work queue: with the default
# 8 connections two shards' streams can map onto one queue, so a shard's kernel
# waits behind its peer's spinning PCG kernel (false serialisation, observed as
# 40 s stalls). Read at CUDA context creation, so set before torch touches CUDA.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# ... and every kernel must be loaded before the first exchange: with lazy
# module loading (CUDA 12's default) the first launch of a kernel loads it,
# and that load waits for the device, including a peer shard's kernel that
# spins in an exchange waiting for this shard -- the first collective of the
# first same-device sharded solve then stalls until the exchange timeout.
# (One process per GPU has no such cross-shard wait.)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built native library")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def summary():
    with open(os.path.join(GOLDEN, "summary.json")) as fh:
        return json.load(fh)


def ba_prob_from_golden(z):
    """oracle problem dict from a BA golden fixture"""
    fm = 0 if not int(z["optimize_focal"]) else (2 if int(z["shared_focal"]) else 1)
    return dict(C=len(z["quats"]), P=len(z["points"]), cam=z["cam"], pt=z["pt"], pixels=z["pixels"],
                pps=z["pps"], dists=z["dists"], focals=z["focals"], model=str(z["model"]),
                focal_mode=fm, loss=(str(z["loss_kind"]), float(z["loss_delta"])))


def gp_prob_from_golden(z):
    dm = bool(int(z["depth_mode"]))
    return dict(C=len(z["quats"]), P=len(z["points"]), cam=z["cam"], pt=z["pt"], rays=z["rays"],
                depth_mode=dm, depths=z["ray_depths"] if dm else None, gauge_fixed=True,
                loss=(str(z["loss_kind"]), float(z["loss_delta"])))


def arrays_from_golden(z):
    from paper_2510_13310_b200.scene import SceneArrays
    dep = z["depths"] if z["depths"].size else None
    return SceneArrays(z["quats"], z["centers"], z["focals"], z["pps"], z["dists"], str(z["model"]) if "model" in z else "pinhole",
                       z["points"], z["cam"], z["pt"], z["pixels"], dep)


def cuda_ok():
    try:
        import torch
        if not torch.cuda.is_available():
            return False
        from paper_2510_13310_b200 import _native
        _native.load()
        return True
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not cuda_ok():
        pytest.fail("GPU test requested but CUDA device / native library unavailable")
    import torch
    return torch

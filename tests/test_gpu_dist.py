"""GPU: the point-sharded solver (paper_2510_13310_b200.dist, csrc/comm.cuh).

Only one GPU is available to the tests, so the shards of one scene run as
several handles on cuda:0:
* in one process (comm="local": exchange regions are device pointers; one
  host thread and one stream per shard, PCG grids capped with SSFM_PCG_SMS so
  the persistent kernels of all shards are co-resident);
* in two processes (comm="torch": gloo process group, CUDA IPC handles,
  exactly the one-process-per-GPU code path minus NVLink).

Checks: all shards report bitwise-identical LM trajectories and camera
parameters (replicated values are combined in rank order on every rank);
the sharded solve follows the single-GPU solve (same accept sequence, costs
within 1e-7 relative: only the summation order differs, so
each damped step agrees with the single-GPU one to the CG tolerance 1e-8 and
the cost after it to about that, relative).
"""
import gc
import os
import subprocess
import sys
import threading

import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import dist as bd
from paper_2510_13310_b200 import synth

# Opt-in (SSFM_SAME_DEVICE_SHARDS=1): these tests run the shards of one scene
# as separate kernel launches on ONE GPU whose kernels spin on each other's
# exchange flags. Nothing guarantees such launches run at the same time: on
# this driver (580.159, sm_100a) same-GPU ranks that wait on one another have
# raised Xid 109 (context-switch timeout), and in round 2 a 3-shard
# fused/graph case stalled here and left the next case hung. The default suite
# covers the multi-rank path on the CPU (tests/test_dist_cpu.py, gloo world 2)
# and the single-rank device path; with one GPU per gpurun call the device
# exchange cannot be exercised safely.
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("SSFM_SAME_DEVICE_SHARDS") != "1",
                                 reason="same-GPU ranks that spin on each other (opt-in: SSFM_SAME_DEVICE_SHARDS=1)")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def scene(cams=40, pts=3000, k=5, seed=0):
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=cams, num_points=pts, visibility_fraction=k / cams,
                                                     pixel_noise_sigma=1.0, seed=seed))
    return synth.perturb_arrays(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)


def solve_local_shards(gpu, st, world, cfg, fused="1", graph="0", shared_focal=False):
    # the shards' cooperative PCG grids must be co-resident next to each other's
    # (and the exchange kernels'): a third of the device is left free
    os.environ["SSFM_PCG_SMS"] = str(max(8, 96 // world))
    os.environ["SSFM_FUSED"] = fused
    os.environ["SSFM_PCG_GRAPH"] = graph
    try:
        probs = [bd.ShardedBAProblem(st, b2.RobustLoss("huber", 1.0), shared_focal=shared_focal, rank=r,
                                     world=world, comm="local")
                 for r in range(world)]
        bd.connect_local(probs)
    finally:
        os.environ.pop("SSFM_PCG_SMS")
        os.environ.pop("SSFM_FUSED")
        os.environ.pop("SSFM_PCG_GRAPH")
    out = [None] * world

    def work(r, stream):
        with gpu.cuda.stream(stream):
            p = probs[r]
            out[r] = b2.lm_solve(p, p.encode(), cfg)

    run_shards(work, probs, 300)   # raises the first shard error
    return probs, out


def shard_streams(probs):
    """One stream per shard, its caching-allocator pool warmed in THIS thread.

    With several shards on one device, a device memory allocation (or any
    NULL-stream command) issued by one shard's thread serialises the device's
    streams around it (CUDA's implicit synchronisation rules): the shard's
    next kernels then wait for everything enqueued before, including a peer's
    kernel that spins in an exchange waiting for them -- a stall until the
    exchange timeout. The solver itself allocates nothing once its handles are
    connected (ssfm_comm_connect also builds the graph PCG), so the shard
    threads must not make torch's allocator call cudaMalloc either: the
    tensors lm_solve / cost / gradient allocate are allocated and freed here
    once per stream first (one process per GPU has no such hazard)."""
    import torch
    streams = []
    for p in probs:
        s = torch.cuda.Stream()
        n, m = p.layout.total_params, p.layout.total_residuals
        with torch.cuda.stream(s):
            keep = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(4)]
            keep += [torch.zeros(m, dtype=torch.float64, device="cuda"), torch.zeros(1, dtype=torch.float64,
                                                                                  device="cuda")]
            keep.append(keep[0].clone())
            bool(torch.isfinite(keep[-1]).all())
            keep[-1].cpu()
            del keep
        s.synchronize()
        streams.append(s)
    return streams


def run_shards(work, probs, timeout):
    """One host thread per same-device shard, each on its own warmed stream
    (shard_streams). Unreachable handles of earlier tests are destroyed first
    and the garbage collector is paused meanwhile: a handle destroyed inside a
    shard's thread frees device memory, which serialises the streams around a
    peer's waiting kernel. Any shard error -- an exchange timeout included --
    fails the test on the first attempt."""
    errs = []
    n = len(probs)
    gc.collect()
    streams = shard_streams(probs)

    def guarded(r):
        try:
            work(r, streams[r])
        except Exception as e:   # noqa: BLE001 - reported below
            errs.append(e)

    gc.disable()
    try:
        ts = [threading.Thread(target=guarded, args=(r,)) for r in range(n)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(timeout=timeout)
    finally:
        gc.enable()
    assert not any(t.is_alive() for t in ts), "a shard did not finish"
    if errs:
        raise errs[0]


@pytest.mark.parametrize("world,fused,graph", [(2, "1", "0"), (3, "1", "0"), (2, "0", "0"), (2, "0", "1"),
                                              (3, "1", "1"), (4, "1", "0"), (4, "0", "1"), (8, "0", "0"),
                                              (8, "0", "1")])
def test_local_shards_match_single_gpu(gpu, world, fused, graph):
    st = scene()
    cfg = b2.LMConfig(max_iterations=15)
    os.environ["SSFM_FUSED"] = fused          # the same operator as the shards
    try:
        single = b2.BAProblem(st, b2.RobustLoss("huber", 1.0))
        single._native_handle()
    finally:
        os.environ.pop("SSFM_FUSED")
    th1, rep1 = b2.lm_solve(single, single.encode(), cfg)
    probs, out = solve_local_shards(gpu, st, world, cfg, fused, graph)
    reps = [o[1] for o in out]
    # identical on every shard (bitwise): every damped solve's CG count, cost and
    # lambda, and the replicated camera block of theta
    for rep in reps[1:]:
        assert [(i.cost_after, i.step_accepted, i.cg_iters, i.lam) for i in rep.iterations] == \
               [(i.cost_after, i.step_accepted, i.cg_iters, i.lam) for i in reps[0].iterations]
    cams = [o[0][:7 * st.num_cameras] for o in out]
    for c in cams[1:]:
        assert np.array_equal(c, cams[0])
    # follows the single-GPU solve
    assert [i.step_accepted for i in reps[0].iterations] == [i.step_accepted for i in rep1.iterations]
    dev = max(abs(a.cost_after - b.cost_after) / b.cost_after for a, b in zip(reps[0].iterations, rep1.iterations))
    print(f"world {world}: max relative cost deviation from the single-GPU solve {dev:.2e}")
    assert dev < 1e-7
    full = probs[0].gather_theta(out[0][0], shards=[(p, o[0]) for p, o in zip(probs, out)])
    assert full.shape == th1.shape
    assert np.abs(full - th1).max() <= 1e-6 * max(1.0, np.abs(th1).max())


@pytest.mark.parametrize("world,fused,graph", [(2, "1", "0"), (2, "0", "1"), (3, "0", "0")])
def test_local_shards_shared_focal(gpu, world, fused, graph):
    """One focal shared by every camera (ba.py:49, 61): its Schur row couples
    every camera, and its point part is summed over every rank's points."""
    st = scene()
    cfg = b2.LMConfig(max_iterations=12)
    os.environ["SSFM_FUSED"] = fused
    try:
        single = b2.BAProblem(st, b2.RobustLoss("huber", 1.0), shared_focal=True)
        single._native_handle()
    finally:
        os.environ.pop("SSFM_FUSED")
    th1, rep1 = b2.lm_solve(single, single.encode(), cfg)
    probs, out = solve_local_shards(gpu, st, world, cfg, fused, graph, shared_focal=True)
    reps = [o[1] for o in out]
    for rep in reps[1:]:
        assert [(i.cost_after, i.cg_iters, i.lam) for i in rep.iterations] == \
               [(i.cost_after, i.cg_iters, i.lam) for i in reps[0].iterations]
    assert [i.step_accepted for i in reps[0].iterations] == [i.step_accepted for i in rep1.iterations]
    dev = max(abs(a.cost_after - b.cost_after) / b.cost_after for a, b in zip(reps[0].iterations, rep1.iterations))
    assert dev < 1e-7
    full = probs[0].gather_theta(out[0][0], shards=[(p, o[0]) for p, o in zip(probs, out)])
    assert full.shape == th1.shape
    assert np.abs(full - th1).max() <= 1e-6 * max(1.0, np.abs(th1).max())


def test_sharded_cost_and_gradient_are_global(gpu):
    st = scene(cams=12, pts=400, k=4, seed=3)
    single = b2.BAProblem(st, b2.RobustLoss("huber", 1.0))
    th = single.encode()
    c1 = single.cost(th)
    g1 = single.gradient(th)
    os.environ["SSFM_PCG_SMS"] = "48"
    try:
        probs = [bd.ShardedBAProblem(st, b2.RobustLoss("huber", 1.0), rank=r, world=2, comm="local") for r in range(2)]
        bd.connect_local(probs)
    finally:
        os.environ.pop("SSFM_PCG_SMS")
    res = [None, None]

    def work(r, stream):
        with gpu.cuda.stream(stream):
            p = probs[r]
            res[r] = (p.cost(p.encode()), p.gradient(p.encode()))

    run_shards(work, probs, 120)
    assert res[0][0] == res[1][0] == pytest.approx(c1, rel=1e-13)
    C = st.num_cameras
    # camera part of the gradient is the global one on every rank; point parts are local
    for r in range(2):
        g = res[r][1]
        assert np.allclose(g[:7 * C], g1[:7 * C], rtol=1e-11, atol=1e-9)
        p0, p1 = probs[r].point_range
        assert np.allclose(g[7 * C:7 * C + 3 * (p1 - p0)], g1[7 * C + 3 * p0:7 * C + 3 * p1], rtol=1e-12, atol=1e-12)


def test_two_processes_ipc(gpu, tmp_path):
    """comm='torch': two processes on cuda:0, gloo for the handle exchange,
    CUDA IPC for the exchange regions (the one-process-per-GPU path)."""
    out = tmp_path / "res"
    env = dict(os.environ, SSFM_PCG_SMS="64", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(ROOT, "tests", "dist_worker.py"),
           str(out)]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    r0, r1 = np.load(str(out) + ".0.npz"), np.load(str(out) + ".1.npz")
    assert np.array_equal(r0["costs"], r1["costs"])
    assert np.array_equal(r0["theta"], r1["theta"])
    st = scene(cams=20, pts=1500, k=4, seed=2)
    single = b2.BAProblem(st, b2.RobustLoss("huber", 1.0))
    _, rep = b2.lm_solve(single, single.encode(), b2.LMConfig(max_iterations=8))
    assert r0["costs"] == pytest.approx(np.array([i.cost_after for i in rep.iterations]), rel=1e-7)


@pytest.mark.parametrize("fused", ["0", "1"])
def test_local_gp_shards_match_single_gpu(gpu, fused):
    """GP (gp.py) sharded by point: scales follow their observations, centres
    are replicated, the mean-scale gauge is taken over every rank."""
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=30, num_points=2000, visibility_fraction=5 / 30,
                                                     pixel_noise_sigma=0.5, seed=2))
    base = b2.fix_gauge(b2.make_rays(obs, depth_mode=False, loss=b2.RobustLoss("huber", 0.1), seed=0))
    cfg = b2.LMConfig(max_iterations=15)
    th1, rep1 = b2.lm_solve(base, base.initial_theta(), cfg)
    # both shards' persistent PCG grids must be co-resident on the one device
    os.environ["SSFM_PCG_SMS"] = "20"
    os.environ["SSFM_FUSED"] = fused
    try:
        probs = [bd.ShardedGPProblem(base, rank=r, world=2, comm="local") for r in range(2)]
        bd.connect_local(probs)
    finally:
        os.environ.pop("SSFM_PCG_SMS")
        os.environ.pop("SSFM_FUSED")
    out = [None, None]

    def work(r, stream):
        with gpu.cuda.stream(stream):
            out[r] = b2.lm_solve(probs[r], probs[r].initial_theta(), cfg)

    run_shards(work, probs, 300)
    ra, rb = out[0][1], out[1][1]
    assert [(i.cost_after, i.cg_iters) for i in ra.iterations] == [(i.cost_after, i.cg_iters) for i in rb.iterations]
    assert [i.step_accepted for i in ra.iterations] == [i.step_accepted for i in rep1.iterations]
    for a, b in zip(ra.iterations, rep1.iterations):
        assert a.cost_after == pytest.approx(b.cost_after, rel=1e-7)
    full = probs[0].gather_theta(out[0][0], shards=[(p, o[0]) for p, o in zip(probs, out)])
    C, P = base.num_cameras, base.num_points
    assert np.abs(full[:3 * (C + P)] - th1[:3 * (C + P)]).max() < 1e-6

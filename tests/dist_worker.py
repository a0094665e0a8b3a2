"""Worker for tests/test_gpu_dist.py::test_two_processes_ipc (torchrun, 2 ranks
on cuda:0, gloo process group): sharded BA solve, results to <out>.<rank>.npz."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_13310_b200 as b2  # noqa: E402
from paper_2510_13310_b200 import dist as bd, synth  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=20, num_points=1500, visibility_fraction=4 / 20,
                                                     pixel_noise_sigma=1.0, seed=2))
    st = synth.perturb_arrays(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
    p = bd.ShardedBAProblem(st, b2.RobustLoss("huber", 1.0), rank=rank, world=world)
    th, rep = b2.lm_solve(p, p.encode(), b2.LMConfig(max_iterations=8))
    full = p.gather_theta(th)
    np.savez(f"{sys.argv[1]}.{rank}.npz", costs=np.array([i.cost_after for i in rep.iterations]), theta=full)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

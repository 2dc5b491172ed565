"""One rank of the multi-process data-parallel test (tests/test_dp_gpu.py).

Launched as `python -m torch.distributed.run --nproc-per-node 2 ... tests/_dp_ranks.py out.json`
on ONE GPU: every rank is a process with its own worker context on cuda:0 and
its own interior shard (shard_interior, trainer.cpp:143-154); the collective is
gloo (host-side, so the ranks' kernels never wait on one another on the GPU).
Runs paper_2604_15645_b200.dist.DataParallelTrainer at world size 2:
  * the averaged gradient of golden case burgers_tanh (the reference's W=2
    data_parallel_gradient, trainer.cpp:649-678),
  * the Adam trajectory of traj_burgers (reference train() with W=2),
  * the replica hashes after every epoch (param_hash / on_sync, trainer.cpp:540-544).
Rank 0 writes the results as JSON for the test to compare with the fixtures.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import golden_io as gi  # noqa: E402
import paper_2604_15645_b200 as pk  # noqa: E402
from paper_2604_15645_b200.dist import DataParallelTrainer, replica_hashes  # noqa: E402


def _worker(g, lo, hi):
    c = g["case"]
    col = g["col"]
    spec = pk.ModelSpec.from_json(c["model"])
    p = c["pde"]
    res = pk.ResidualSpec(p["id"], p.get("advection_c", 1.0), p.get("epsilon", 1.0), p.get("mu", 1.0))
    w = pk.make_worker(spec, res, g["bc"], g["rffB"], col.interior[lo:hi], col.ic_points, col.ic_targets,
                       col.bc_a, col.bc_b, col.bc_targets, device=0)
    return spec, w


def main():
    out = sys.argv[1]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    res = {"world": world}

    g = gi.load("burgers_tanh")
    lo, hi = pk.shard_interior(len(g["col"].interior), world)[rank]
    spec, w = _worker(g, lo, hi)
    tr = DataParallelTrainer([w], g["params"], world=world, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    tr._total((1.0, 1.0, 1.0), st)
    torch.cuda.synchronize(dev)
    res["grad"] = (tr.grad.double().cpu().numpy() / world).tolist()

    g = gi.load("traj_burgers")
    t = g["case"]["train"]
    lo, hi = pk.shard_interior(len(g["col"].interior), world)[rank]
    spec, w = _worker(g, lo, hi)
    tr = DataParallelTrainer([w], g["params"], world=world, lr=t["lr"], gamma=t["gamma"], device=dev,
                             has_bc=g["bc"] != "hard")
    rows, hashes = [], []
    for _ in range(t["epochs"]):
        rows.append(tr.step().cpu().numpy().tolist())
        hashes.append([str(h) for h in replica_hashes(spec, tr.params_host(), world)])
    res["metrics"] = rows
    res["hashes"] = hashes
    if rank == 0:
        with open(out, "w") as f:
            json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

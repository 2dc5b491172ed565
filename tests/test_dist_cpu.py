"""CPU, world_size 2 over gloo: the multi-rank data-parallel protocol of the
product (paper_2604_15645_b200.dist) -- rank shards, the single gradient
all-reduce, identical updates and the replica hash -- with each rank's
gradient computed by the FP64 oracle (the CUDA worker needs a GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_io as gi
from oracle import pinn_oracle as po


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, name, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_15645_b200 import dist as pd
    import paper_2604_15645_b200 as pk
    g = gi.load(name)
    col = g["col"]
    lo, hi = pd.rank_shard(len(col.interior), world, rank)
    spec = pk.ModelSpec.from_json(g["case"]["model"])
    p = g["params"].copy()
    opt = po.Adam(lr=1e-2)
    hashes = []
    for step in range(3):
        o = po.worker_step(g["spec"], p, g["rffB"], g["res"], col.interior[lo:hi], col, g["bc"])
        t = torch.tensor(o["grad"], dtype=torch.float64)
        pd.allreduce_average_(t, world)
        if step == 0:
            np.save(os.path.join(out_dir, f"grad_rank{rank}.npy"), t.numpy())
        opt.step(p, t.numpy())
        hashes.append(pd.replica_hashes(spec, p, world))
    np.save(os.path.join(out_dir, f"hash_rank{rank}.npy"), np.array(hashes, dtype=object), allow_pickle=True)
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["burgers_tanh", "maxwell_tanh"])
def test_two_rank_gloo_protocol(name, tmp_path):
    world = 2
    mp.spawn(_rank_main, args=(world, _free_port(), name, str(tmp_path)), nprocs=world, join=True)
    g = gi.load(name)
    ref = g[f"grad_w{world}"]  # the reference's data_parallel_gradient with W=2
    for r in range(world):
        gr = np.load(tmp_path / f"grad_rank{r}.npy")
        assert np.linalg.norm(gr - ref) <= 1e-12 * np.linalg.norm(ref)
    h0 = np.load(tmp_path / "hash_rank0.npy", allow_pickle=True)
    h1 = np.load(tmp_path / "hash_rank1.npy", allow_pickle=True)
    for step in range(3):
        assert len(set(h0[step])) == 1 and list(h0[step]) == list(h1[step])


def test_param_hash_matches_reference_fnv():
    """dist.param_hash == reference param_hash (on_sync values in the fixture)."""
    from paper_2604_15645_b200 import dist as pd
    import paper_2604_15645_b200 as pk
    g = gi.load("traj_burgers")
    spec = pk.ModelSpec.from_json(g["case"]["model"])
    assert pd.param_hash(spec, g["final_params"]) == int(g["meta"]["hashes"][-1]["hashes"][0])


def test_rank_shards_cover_and_disjoint():
    from paper_2604_15645_b200 import dist as pd
    for n, w in [(1000, 8), (1003, 8), (10, 3)]:
        b = [pd.rank_shard(n, w, r) for r in range(w)]
        assert b[0][0] == 0 and b[-1][1] == n
        assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))

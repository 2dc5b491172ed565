"""GPU: the multi-rank data-parallel paths against the reference's W-worker
fixtures.

* pnx_dp (C ABI, pinn.DataParallelGroup): R ranks -> one NCCL all-reduce of the
  packed [grad | losses] per step -> device Adam on every replica. Only one GPU
  is available to these tests, so the ranks are local replicas of device 0
  (summed on the device in rank order before the all-reduce, which then runs
  over a one-device communicator); the multi-device path is the same code with
  more communicators.
* dist.DataParallelTrainer at world size 2: two processes on the one GPU over
  gloo (a host-side collective: no kernel waits on another rank's kernel).

Tolerances as in test_gpu_parity.py (FP32 device arithmetic vs the FP64
reference): gradients rel-L2 1e-5, trajectories 1e-3 per epoch.
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import golden_io as gi

pytestmark = pytest.mark.gpu

GRAD_RTOL = 1e-5
TRAJ_RTOL = 1e-3


def _pkg():
    import paper_2604_15645_b200 as pk
    return pk


def _group(g, ranks, engine="auto", **kw):
    pk = _pkg()
    c = g["case"]
    col = g["col"]
    p = c["pde"]
    spec = pk.ModelSpec.from_json(c["model"])
    res = pk.ResidualSpec(p["id"], p.get("advection_c", 1.0), p.get("epsilon", 1.0), p.get("mu", 1.0))
    grp = pk.pinn.DataParallelGroup(spec, res, g["bc"], g["rffB"], devices=[0] * ranks, engine=engine)
    grp.set_points(col.interior)
    if col.ic_points is not None and len(col.ic_points):
        grp.set_ic(col.ic_points, col.ic_targets)
    if g["bc"] != "hard":
        grp.set_bc(col.bc_a, col.bc_b, col.bc_targets)
    if g["causality"] is not None:
        o = g["causality"]
        for w in grp.workers:
            w.set_causality(pk.CausalityConfig(o.segments, o.epsilon, o.t_lo, o.t_hi))
    if g["poynting"] is not None:
        o = g["poynting"]
        for w in grp.workers:
            w.set_poynting(pk.PoyntingConfig(o.weight, o.grid, o.time_samples, tuple(o.xb) + tuple(o.yb) + tuple(o.tb)))
    grp.set_params(g["params"])
    return grp


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", ["burgers_tanh", "burgers_c1_shape", "maxwell_c4_shape", "maxwell_poynting"])
def test_dp_group_gradient_matches_reference_workers(name):
    """pnx_dp_step without the update returns the reference's W-worker averaged
    gradient (data_parallel_gradient, trainer.cpp:649-678) and mean losses."""
    g = gi.load(name)
    for W in g["meta"]["workers"]:
        grp = _group(g, W)
        assert grp.size() == (W, 1)
        losses, grad = grp.step(update=False, want_grad=True)
        assert rel_l2(grad, g[f"grad_w{W}"]) <= GRAD_RTOL, (name, W, rel_l2(grad, g[f"grad_w{W}"]))
        ref = g["meta"]["worker_losses"][str(W)]
        for k in ("pde", "ic", "bc"):
            m = sum(r[k] for r in ref) / W
            assert abs(losses[k] - m) <= 1e-5 * abs(m) + 1e-9, (name, W, k, losses[k], m)


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("name", ["traj_burgers", "traj_maxwell", "traj_burgers_causality", "traj_burgers_balancing",
                                  "traj_maxwell_full"])
def test_dp_group_trajectory_matches_reference_train(name, graph):
    """N synchronized epochs through pnx_dp (device Adam with lr = lr0 gamma^epoch,
    one all-reduce per step; balancing epochs: pnx_dp_step_terms -> lambda update
    -> pnx_dp_apply_gradient, trainer.cpp:462-506) track the reference train()."""
    g = gi.load(name)
    c = g["case"]
    t = c["train"]
    W = c["workers"]
    grp = _group(g, W)
    grp.set_optimizer(t["lr"], t.get("gamma", 1.0))
    grp.set_graph(graph)
    lam = [1.0, 1.0, 1.0]
    bal = g["balancing"]
    has_bc = g["bc"] != "hard"
    metrics = g["metrics"]
    for ep in range(t["epochs"]):
        if bal is not None and ep % bal.update_period == 0:
            terms, losses = grp.step_terms()
            norms = [float(np.linalg.norm(terms[k])) for k in range(3)]
            old = list(lam)
            tot = norms[0] + norms[1] + (norms[2] if has_bc else 0.0)
            for k in range(3 if has_bc else 2):
                lam[k] = bal.alpha * lam[k] + (1.0 - bal.alpha) * (tot / max(norms[k], 1e-9))
            if g["poynting"] is not None:  # total gradient under the previous weights (trainer.cpp:491-498)
                losses = grp.step(old)
            else:
                grp.apply_gradient(lam[0] * terms[0] + lam[1] * terms[1] + (lam[2] * terms[2] if has_bc else 0.0))
        else:
            losses = grp.step(lam)
        row = [losses["pde"], losses["ic"], losses["bc"]] + lam
        for k in range(6):
            ref = metrics[ep, 1 + k]
            assert abs(row[k] - ref) <= TRAJ_RTOL * abs(ref) + 1e-9, (ep, k, row[k], ref)
    p = [grp.params(r) for r in range(W)]
    for r in range(1, W):
        assert np.array_equal(p[r], p[0])


def test_dp_group_raises_nonfinite_with_reference_text():
    pk = _pkg()
    g = gi.load("burgers_tanh")
    pts = g["col"].interior.copy()
    pts[5, 1] = np.nan  # rank 1 of 2 owns points 60.. ; rank 0 point 5
    g["col"].interior = pts
    grp = _group(g, 2)
    with pytest.raises(pk.TensorError, match="non-finite residual at point index 5"):
        grp.step()


def test_dist_trainer_two_processes_match_reference():
    """dist.DataParallelTrainer with world size 2 (two processes, gloo, one GPU):
    the averaged gradient of the reference's W=2 data_parallel_gradient, the
    W=2 train() trajectory, and equal replica hashes after every epoch."""
    root = gi.ROOT
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "dp.json")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
               "--master-addr=127.0.0.1", "--master-port=29561", os.path.join(root, "tests", "_dp_ranks.py"), out]
        r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        res = json.load(open(out))
    assert res["world"] == 2
    g = gi.load("burgers_tanh")
    assert rel_l2(np.array(res["grad"]), g["grad_w2"]) <= GRAD_RTOL
    m = gi.load("traj_burgers")["metrics"]
    for ep, row in enumerate(res["metrics"]):
        for k in range(3):
            assert abs(row[k] - m[ep, 1 + k]) <= TRAJ_RTOL * abs(m[ep, 1 + k]) + 1e-9, (ep, k, row[k])
    for hs in res["hashes"]:
        assert len(hs) == 2 and hs[0] == hs[1]


def test_bench_two_ranks_gloo():
    """bench.py's N>1 path (torchrun, contiguous shards, packed all-reduce, max
    over ranks, replica hashes) with two ranks on the one GPU over gloo."""
    root = gi.ROOT
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29562", os.path.join(root, "bench.py"), "--gpus", "2",
           "--dist-backend", "gloo", "--steps", "3", "--warmup", "3", "--config", "c1", "--no-e2e"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().split("\n")[-1])
    assert line["n_gpus"] == 2 and line["replica_hashes_equal"] is True
    assert line["value"] > 0 and line["config"]["parallelism"] == "dp2"

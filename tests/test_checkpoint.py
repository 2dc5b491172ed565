"""PLABCK01 checkpoints (checkpoint.cpp) between the reference and this package:
the reference's own train() output loads bit-exactly, our writer's output
loads through the reference's Checkpoint::load, and (GPU) a trainer resumed
from the reference checkpoint continues the reference trajectory."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

import golden_io as gi

DRIVER = os.path.join(gi.ROOT, "oracle", "_ref", "pinnlab_ref_driver")


def _pkg():
    import paper_2604_15645_b200 as pk
    return pk


def _ref_ckpt_file(g, tmp_path):
    p = tmp_path / "final.ckpt"
    g["ckpt"].tofile(p)
    return str(p)


@pytest.mark.parametrize("name", gi.CKPT_NAMES)
def test_reference_checkpoint_loads_bit_exact(name, tmp_path):
    from paper_2604_15645_b200.checkpoint import Checkpoint
    g = gi.load(name)
    ck = Checkpoint.load(_ref_ckpt_file(g, tmp_path))
    ref_t = g["meta"]["ckpt_tensors"]
    assert [n for n, _ in ck.tensors] == [t["name"] for t in ref_t]
    assert [list(t.shape) for _, t in ck.tensors] == [t["shape"] for t in ref_t]
    flat = np.concatenate([t.ravel() for _, t in ck.tensors])
    assert np.array_equal(flat, g["ckpt_data"])  # the reference loader's payload, bit for bit
    assert ck.scalars == g["meta"]["ckpt_scalars"]
    P = g["final_params"].size
    assert np.array_equal(flat[:P], g["final_params"])


@pytest.mark.parametrize("name", gi.CKPT_NAMES)
def test_our_checkpoint_loads_in_reference(name, tmp_path):
    from paper_2604_15645_b200.checkpoint import Checkpoint
    g = gi.load(name)
    ck = Checkpoint.load(_ref_ckpt_file(g, tmp_path))
    ours = str(tmp_path / "ours.ckpt")
    ck.save(ours)
    back = Checkpoint.load(ours)
    assert [n for n, _ in back.tensors] == [n for n, _ in ck.tensors]
    assert all(np.array_equal(a, b) for (_, a), (_, b) in zip(back.tensors, ck.tensors))
    if not os.path.exists(DRIVER):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    job = dict(g["case"], mode="ckpt_info", ckpt=ours, out=str(tmp_path))
    (tmp_path / "job.json").write_text(json.dumps(job))
    subprocess.run([DRIVER, str(tmp_path / "job.json")], check=True)
    meta = json.loads((tmp_path / "meta.json").read_text())
    assert meta["ckpt_scalars"] == g["meta"]["ckpt_scalars"]
    assert np.array_equal(np.fromfile(tmp_path / "ckpt_data.bin", dtype="<f8"), g["ckpt_data"])
    # Checkpoint::restore_model accepted it: same trainable tensors
    assert np.array_equal(np.fromfile(tmp_path / "restored_params.bin", dtype="<f8"), g["final_params"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", gi.CKPT_NAMES)
def test_resume_from_reference_checkpoint_on_device(name, tmp_path):
    """trainer.cpp:345-353: resume parameters, Adam state, lambdas and the epoch
    count from the reference's final.ckpt and continue its trajectory."""
    import torch
    pk = _pkg()
    from paper_2604_15645_b200.checkpoint import Checkpoint, restore_trainer
    from paper_2604_15645_b200.dist import DataParallelTrainer
    g = gi.load(name)
    case = g["case"]
    t = case["train"]
    col = g["col"]
    spec = pk.ModelSpec.from_json(case["model"])
    p = case["pde"]
    res = pk.ResidualSpec(p["id"], p.get("advection_c", 1.0), p.get("epsilon", 1.0), p.get("mu", 1.0))
    workers = []
    for lo, hi in pk.shard_interior(len(col.interior), case["workers"]):
        workers.append(pk.make_worker(spec, res, g["bc"], g["rffB"] if spec.rff else None, col.interior[lo:hi],
                                      col.ic_points, col.ic_targets, col.bc_a, col.bc_b, col.bc_targets))
    bal = pk.BalancingConfig(True, t.get("alpha", 0.9), t.get("update_period", 100)) if t.get("balancing") else None
    tr = DataParallelTrainer(workers, g["params"], world=1, lr=t["lr"], gamma=t["gamma"],
                             device=torch.device("cuda:0"), balancing=bal, has_bc=g["bc"] != "hard")
    restore_trainer(tr, Checkpoint.load(_ref_ckpt_file(g, tmp_path)), spec)
    rm = g["resume_metrics"]
    for row in rm:
        assert tr.epoch == int(row[0])
        lm = list(tr.step().cpu().numpy()) + list(tr.lam)
        for k in range(6):
            assert abs(lm[k] - row[1 + k]) <= 1e-3 * abs(row[1 + k]) + 1e-9, (row[0], k, lm[k], row[1 + k])
    np.testing.assert_allclose(tr.params_host(), g["resume_final_params"], rtol=2e-3, atol=2e-5)

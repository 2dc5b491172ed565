"""The reference-side binding compiled and run: the reference's
own trainer.cpp with run_worker_epoch bound to libpnx (integration/
pnx_worker_epoch.hpp force-included, integration/Makefile), linked with the
other unmodified reference objects.

CPU: the binding compiles against /root/reference and every run_worker_epoch
call site of trainer.cpp resolves to it (the object needs pnx_step, and the
template specialization for the reference's WorkerTask exists).
GPU: the reference's train() and data_parallel_gradient, with the worker step on
the B200, reproduce the reference's own CPU fixtures.
"""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

import golden_io as gi

ROOT = gi.ROOT
BIN = os.path.join(ROOT, "integration", "_build", "pinnlab_ref_pnx_driver")
OBJ = os.path.join(ROOT, "integration", "_build", "trainer_pnx.o")
HAVE_REF = os.path.isdir("/root/reference/proj/core/src")


@pytest.mark.skipif(not HAVE_REF, reason="needs /root/reference (build container only)")
def test_binding_compiles_against_reference_and_owns_every_call_site():
    subprocess.run(["make", "-C", os.path.join(ROOT, "integration")], check=True, stdout=subprocess.DEVNULL)
    syms = subprocess.run(["nm", "-C", OBJ], capture_output=True, text=True, check=True).stdout
    assert "pinnlab::run_worker_epoch<pinnlab::(anonymous namespace)::WorkerTask>" in syms
    for s in ("pnx_create", "pnx_set_points", "pnx_step", "pnx_step_terms"):
        assert f" U {s}\n" in syms, s
    # the reference's Graph-based body is never called (no call edge survives)
    assert "run_worker_epoch(pinnlab::(anonymous namespace)::WorkerTask const&)" not in syms


def _run(job):
    with tempfile.TemporaryDirectory() as d:
        job = dict(job, out=d)
        jp = os.path.join(d, "job.json")
        json.dump(job, open(jp, "w"))
        r = subprocess.run([BIN, jp], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        meta = json.load(open(os.path.join(d, "meta.json")))
        g = os.path.join(d, "grad.bin")
        grad = np.fromfile(g, dtype="<f8") if os.path.exists(g) else None
        return meta, grad


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="integration/_build not built (needs /root/reference)")
@pytest.mark.parametrize("name", ["traj_burgers", "traj_burgers_balancing", "traj_maxwell_full"])
def test_reference_train_with_pnx_worker_step(name):
    """trainer.cpp:332-624 as shipped, its worker step on the B200: the metrics
    stream matches the reference CPU run within the trajectory tolerance 1e-3."""
    g = gi.load(name)
    meta, _ = _run(dict(g["case"], mode="train"))
    m = np.array([row[:8] for row in meta["metrics"]], dtype=np.float64)
    ref = g["metrics"]
    assert m.shape == ref.shape
    assert np.all(np.abs(m[:, 1:7] - ref[:, 1:7]) <= 1e-3 * np.abs(ref[:, 1:7]) + 1e-9)
    assert not meta["aborted"]


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="integration/_build not built (needs /root/reference)")
@pytest.mark.parametrize("name", ["burgers_c1_shape", "maxwell_c4_shape", "maxwell_poynting"])
def test_reference_data_parallel_gradient_with_pnx_worker_step(name):
    """data_parallel_gradient (trainer.cpp:649-678) with W threads, each worker's
    step on the B200 (its own context), averaged by the reference's average_grads."""
    g = gi.load(name)
    case = {k: v for k, v in g["meta"]["case"].items()}
    for w in g["meta"]["workers"]:
        _, grad = _run(dict(case, mode="step", workers=w))
        ref = g[f"grad_w{w}"]
        assert np.linalg.norm(grad - ref) <= 1e-5 * np.linalg.norm(ref), (name, w)

"""The C++ host mirror (host/, namespace pinnlab_b200) used the way a
reference user would use pinnlab: Model(spec, seed) must reproduce the
reference's parameter draws bit-for-bit (same libstdc++ mt19937_64 +
normal_distribution, model.cpp:52-102), build_collocation the reference grid,
and data_parallel_gradient / train (on the GPU) the reference gradients and
loss trajectory."""
import os
import subprocess

import numpy as np
import pytest

import golden_io as gi

DRIVER = os.path.join(gi.ROOT, "host", "host_driver")


def _driver():
    if not os.path.exists(DRIVER):
        subprocess.run(["make", "-C", os.path.join(gi.ROOT, "host")], check=True, stdout=subprocess.DEVNULL)
    return DRIVER


def _job(g, path, **extra):
    c = g["case"]
    m = c["model"]
    lines = [f"in_dim {m['in_dim']}", f"hidden_dim {m['hidden_dim']}", f"depth {m['depth']}",
             f"out_dim {m['out_dim']}", f"activation {m['activation']}", f"sine_w0 {m.get('sine_w0', 1.0)}",
             f"pde {c['pde']['id']}", f"advection_c {c['pde'].get('advection_c', 1.0)}",
             f"epsilon {c['pde'].get('epsilon', 1.0)}", f"mu {c['pde'].get('mu', 1.0)}",
             "domain " + " ".join(f"{a} {b}" for a, b in c["domain"]), f"initial {c['initial']}",
             f"bc {c.get('bc', 'hard')}", "dims " + " ".join(str(d) for d in c["collocation"].get("dims", [])),
             f"n_ic {c['collocation'].get('n_ic', 128)}", f"n_bc {c['collocation'].get('n_bc', 64)}", "seed 0"]
    if m.get("periodic_axes"):
        lines.append("periodic " + " ".join(f"{int(a['periodic'])} {a['period']} {int(a.get('trainable', False))}"
                                            for a in m["periodic_axes"]))
    if "rff" in m:
        lines.append(f"rff {m['rff']['width']} {m['rff'].get('sigma', 10.0)} {m['rff'].get('mean', 0.0)}")
    if "rwf" in m:
        lines.append(f"rwf {m['rwf'].get('mean', 1.0)} {m['rwf'].get('stddev', 0.1)}")
    cc = c["collocation"]
    if cc.get("mode", "uniform") != "uniform":
        lines += [f"colloc_mode {cc['mode']}", f"colloc_n {cc.get('n', 0)}"]
    if cc.get("resample_every", 0):
        lines.append(f"resample_every {cc['resample_every']}")
    lines.append(f"colloc_seed {c.get('colloc_seed', 0)}")
    t = c.get("train", {})
    if t.get("balancing"):
        lines += ["balancing 1", f"alpha {t.get('alpha', 0.9)}", f"update_period {t.get('update_period', 100)}"]
    if c.get("causality", {}).get("enabled"):
        lines += [f"causality_segments {c['causality'].get('segments', 10)}",
                  f"causality_epsilon {c['causality'].get('epsilon', 1.0)}"]
    if c.get("poynting", {}).get("weight", 0.0) > 0.0:
        pj = c["poynting"]
        lines += [f"poynting_weight {pj['weight']}", f"poynting_grid {pj.get('grid', 32)}",
                  f"poynting_time_samples {pj.get('time_samples', 4)}"]
    if t.get("switch", {}).get("trigger") == "epoch":
        lines += [f"switch_epoch {t['switch']['epoch_threshold']}", f"lbfgs_max_iters {t.get('lbfgs_max_iters', 0)}",
                  f"lbfgs_history {t.get('lbfgs', {}).get('history', 50)}"]
    for k, v in extra.items():
        lines.append(f"{k} {v}")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


@pytest.mark.parametrize("name", gi.CASE_NAMES)
def test_cpp_model_init_and_collocation_match_reference(name, tmp_path):
    g = gi.load(name)
    _job(g, tmp_path / "job.txt")
    subprocess.run([_driver(), "cpu", str(tmp_path / "job.txt"), str(tmp_path)], check=True)
    p = np.fromfile(tmp_path / "params.bin", dtype="<f8")
    assert np.array_equal(p, g["params"]), "C++ Model init differs from the reference draws"
    if g["spec"].rff:
        assert np.array_equal(np.fromfile(tmp_path / "rffB.bin", dtype="<f8"), g["rffB"].ravel())
    pts = np.fromfile(tmp_path / "interior.bin", dtype="<f8").reshape(g["spec"].in_dim, -1).T
    assert np.array_equal(pts, g["col"].interior)


@pytest.mark.gpu
@pytest.mark.parametrize("name", gi.CASE_NAMES)
def test_cpp_data_parallel_gradient_on_gpu(name, tmp_path):
    g = gi.load(name)
    for w in g["meta"]["workers"]:
        _job(g, tmp_path / "job.txt", workers=w)
        subprocess.run([_driver(), "grad", str(tmp_path / "job.txt"), str(tmp_path)], check=True)
        grad = np.fromfile(tmp_path / "grad.bin", dtype="<f8")
        ref = g[f"grad_w{w}"]
        assert np.linalg.norm(grad - ref) <= 1e-5 * np.linalg.norm(ref)


@pytest.mark.gpu
@pytest.mark.parametrize("name", gi.TRAJ_NAMES)
def test_cpp_train_trajectory_on_gpu(name, tmp_path):
    g = gi.load(name)
    t = g["case"]["train"]
    _job(g, tmp_path / "job.txt", workers=g["case"]["workers"], epochs=t["epochs"], lr=t["lr"], gamma=t["gamma"])
    subprocess.run([_driver(), "train", str(tmp_path / "job.txt"), str(tmp_path)], check=True)
    m = np.fromfile(tmp_path / "metrics.bin", dtype="<f8").reshape(-1, 6)
    ref = g["metrics"][:, 1:7]  # l_pde, l_ic, l_bc, lambda_pde, lambda_ic, lambda_bc
    assert m.shape == ref.shape
    n_adam = ref.shape[0] if not g["meta"].get("switched_to_lbfgs") else int(t["switch"]["epoch_threshold"]) + 1
    assert np.all(np.abs(m[:n_adam] - ref[:n_adam]) <= 1e-3 * np.abs(ref[:n_adam]) + 1e-9)
    # L-BFGS rows: FP32 objective, line-search paths may drift
    assert np.all(np.abs(m[n_adam:] - ref[n_adam:]) <= 1e-2 * np.abs(ref[n_adam:]) + 1e-8)
    # on_sync (trainer.cpp:540-544): every Adam epoch, one hash per worker replica, all equal
    rows = [ln.split() for ln in open(tmp_path / "hash.txt").read().splitlines()]
    assert len(rows) == n_adam
    assert all(len(r) == g["case"]["workers"] and len(set(r)) == 1 for r in rows)


def test_cpp_host_adam_matches_oracle_adam():
    """pinnlab_adam_step (the C++ host mirror's Adam, optim.cpp:7-41; bench.py's
    end-to-end leg calls it) against the oracle's Adam over five steps (CPU)."""
    import ctypes
    from oracle import pinn_oracle as po
    _driver()
    lib = ctypes.CDLL(os.path.join(gi.ROOT, "host", "libpinnlab_b200.so"))
    fn = lib.pinnlab_adam_step
    dp = ctypes.POINTER(ctypes.c_double)
    fn.argtypes = [dp, dp, dp, dp, ctypes.c_int64] + [ctypes.c_double] * 4 + [ctypes.c_int64]
    fn.restype = ctypes.c_int
    rng = np.random.default_rng(3)
    p = rng.standard_normal(1001)
    p_ref = p.copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    opt = po.Adam(lr=2e-3, beta1=0.8, beta2=0.99, eps=1e-7)
    for t in range(1, 6):
        g = rng.standard_normal(p.size) * 10.0 ** (t - 3)
        opt.step(p_ref, g)
        assert fn(*(a.ctypes.data_as(dp) for a in (p, m, v, g)), p.size, 2e-3, 0.8, 0.99, 1e-7, t) == 0
        np.testing.assert_allclose(p, p_ref, rtol=1e-14, atol=1e-15)

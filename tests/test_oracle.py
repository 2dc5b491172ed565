"""CPU: the FP64 restatement (oracle/pinn_oracle.py) pinned to the compiled
reference's golden vectors (tests/golden, from oracle/_ref), plus the SPEC.md
known-answer checks that touch the hot path."""
import math

import numpy as np
import pytest

import golden_io as gi
from oracle import pinn_oracle as po


@pytest.mark.parametrize("name", gi.CASE_NAMES)
def test_gradient_and_losses_match_reference(name):
    g = gi.load(name)
    for w in g["meta"]["workers"]:
        grad, outs = po.data_parallel_gradient(g["spec"], g["params"], g["rffB"], g["res"], g["col"], g["bc"], w,
                                               poynting=g["poynting"])
        ref = g[f"grad_w{w}"]
        assert np.linalg.norm(grad - ref) <= 1e-12 * np.linalg.norm(ref)
        for o, r in zip(outs, g["meta"]["worker_losses"][str(w)]):
            for k in ("pde", "ic", "bc"):
                assert abs(o[k] - r[k]) <= 1e-12 * abs(r[k]) + 1e-25
        if g["poynting"] is not None:  # poynting_penalty value (losses.cpp:187-223)
            assert abs(outs[0]["pen"] - g["meta"]["penalty"]) <= 1e-12 * abs(g["meta"]["penalty"])


@pytest.mark.parametrize("name", gi.CASE_NAMES)
def test_residuals_and_outputs_match_reference(name):
    g = gi.load(name)
    o = po.worker_step(g["spec"], g["params"], g["rffB"], g["res"], g["col"].interior, g["col"], g["bc"],
                       want_residuals=True)
    np.testing.assert_allclose(o["residuals"], g["residuals"], rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(o["outputs"], g["outputs"], rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("name", gi.CASE_NAMES)
def test_collocation_matches_reference(name):
    g = gi.load(name)
    c = g["case"]
    cc = c["collocation"]
    if cc.get("mode", "uniform") != "uniform":
        pytest.skip("LHS designs are pinned bit-exactly through the C++ host (tests/test_host_cpp.py)")
    col = po.build_collocation(c["domain"], cc["dims"], cc.get("n_ic", 128), cc.get("n_bc", 64), g["bc"],
                               c["initial"], g["spec"].out_dim)
    np.testing.assert_array_equal(col.interior, g["col"].interior)
    np.testing.assert_array_equal(col.ic_points, g["col"].ic_points)
    np.testing.assert_allclose(col.ic_targets, g["col"].ic_targets, rtol=0, atol=1e-15)
    if g["bc"] != "hard":
        np.testing.assert_array_equal(col.bc_a, g["col"].bc_a)


@pytest.mark.parametrize("name", gi.CASE_NAMES)
def test_param_layout_matches_reference(name):
    g = gi.load(name)
    lay = po.param_layout(g["spec"])
    ref = [(p["name"], tuple(p["shape"])) for p in g["meta"]["params"]]
    assert lay == ref
    assert po.param_count(g["spec"]) == g["params"].size


@pytest.mark.parametrize("name", gi.TRAJ_NAMES)
def test_adam_trajectory_matches_reference(name):
    g = gi.load(name)
    t = g["case"]["train"]
    if g["case"]["collocation"].get("resample_every", 0):
        pytest.skip("interior resampling (LHS stream) runs in the C++ host mirror")
    p, hist = po.train(g["spec"], g["params"], g["rffB"], g["res"], g["col"], g["bc"], t["epochs"], lr=t["lr"],
                       gamma=t["gamma"], workers=g["case"]["workers"], balancing=g["balancing"],
                       causality=g["causality"], poynting=g["poynting"], switch=g["switch"],
                       lbfgs_max_iters=g["lbfgs_max_iters"], lbfgs_cfg=g["lbfgs_cfg"])
    m = g["metrics"]
    assert len(hist) == m.shape[0]
    for ep, row in enumerate(hist):
        # l_pde, l_ic, l_bc, lambda_pde, lambda_ic, lambda_bc (MetricsRecord, trainer.cpp:524-530)
        for k in range(6):
            assert abs(row[k] - m[ep, 1 + k]) <= 1e-10 * abs(m[ep, 1 + k]) + 1e-30
    np.testing.assert_allclose(p, g["final_params"], rtol=1e-7, atol=1e-9)
    # replica hashes from on_sync (trainer.cpp:540-544): all replicas equal, and
    # param_hash restated bit-exactly (FNV-1a of the reference's final params)
    last = g["meta"]["hashes"][-1]["hashes"]
    assert len(set(last)) == 1
    if not g["meta"].get("switched_to_lbfgs"):  # on_sync fires after Adam epochs only (trainer.cpp:540-544)
        assert po.param_hash(g["spec"], g["final_params"]) == int(last[0])


def test_shard_interior_semantics():
    assert po.shard_bounds(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert po.shard_bounds(8, 4) == [(0, 2), (2, 4), (4, 6), (6, 8)]
    with pytest.raises(ValueError, match="fewer interior points than workers"):
        po.shard_bounds(3, 4)


def test_equal_shards_average_equals_serial():
    """W=4 equal shards, mean losses -> averaged grad == serial (1e-10)."""
    g = gi.load("burgers_tanh")
    col = g["col"]
    col_pde_only = po.Collocation(col.interior, col.ic_points, col.ic_targets, col.bc_a, None, col.bc_targets)
    g1, _ = po.data_parallel_gradient(g["spec"], g["params"], None, g["res"], col_pde_only, g["bc"], 1)
    g4, _ = po.data_parallel_gradient(g["spec"], g["params"], None, g["res"], col_pde_only, g["bc"], 4)
    assert np.linalg.norm(g4 - g1) <= 1e-10 * np.linalg.norm(g1)


def _fd_check(spec, res, flat, rffB, col, bc, idxs, h=1e-6):
    out = po.worker_step(spec, flat, rffB, res, col.interior, col, bc)
    for i in idxs:
        fp = flat.copy()
        fp[i] += h
        fm = flat.copy()
        fm[i] -= h
        lp = po.worker_step(spec, fp, rffB, res, col.interior, col, bc)
        lm = po.worker_step(spec, fm, rffB, res, col.interior, col, bc)
        tot = lambda o: o["pde"] + o["ic"] + o["bc"]
        fd = (tot(lp) - tot(lm)) / (2 * h)
        assert abs(fd - out["grad"][i]) <= 1e-4 * max(abs(fd), 1e-3), (i, fd, out["grad"][i])


def test_ns_steady_extension_finite_differences():
    """ns_steady is not in the reference: pinned by central FD on the oracle
    (SPEC.md:67 style, rel <= 1e-4)."""
    spec = po.ModelSpec(in_dim=2, hidden_dim=8, depth=2, out_dim=3, activation="tanh")
    res = po.ResidualSpec("ns_steady", reynolds=100.0)
    flat, _ = po.init_params(spec, 3)
    pts = po.sample_uniform([(0, 1), (0, 1)], [5, 4])
    n = 6
    s = po.linspace(0, 1, n)
    walls = np.concatenate([np.stack([np.zeros(n), s], 1), np.stack([np.ones(n), s], 1)])
    tg = np.zeros((2 * n, 3))
    tg[n:, 0] = 1.0
    col = po.Collocation(pts, np.zeros((0, 2)), np.zeros((0, 3)), walls, None, tg)
    rng = np.random.default_rng(0)
    _fd_check(spec, res, flat, None, col, "dirichlet_zero", rng.choice(flat.size, 12, replace=False))


def test_swish_sine_periodic_rff_finite_differences():
    g = gi.load("maxwell_periodic_rff")
    idx = [0, 5, 40, g["params"].size - 1]  # includes the trainable period P2
    _fd_check(g["spec"], g["res"], g["params"], g["rffB"], g["col"], g["bc"], idx)


def test_causality_weights_and_segments():
    """losses.cpp:163-171 / trainer.cpp:156-177 on hand-checked values."""
    om = po.causality_weights([0.5, 0.25, 1.0], 2.0)
    np.testing.assert_allclose(om, [1.0, math.exp(-1.0), math.exp(-1.5)], rtol=1e-15)
    pts = np.array([[0.0, 0.0], [0.0, 0.2499], [0.0, 0.25], [0.0, 0.999], [0.0, 1.0]])
    np.testing.assert_array_equal(po.time_segment_index(pts, 0.0, 1.0, 4), [0, 0, 1, 3, 3])


def test_poynting_penalty_finite_differences():
    """d pen / d fields of poynting_terms against central differences."""
    rng = np.random.default_rng(3)
    pc = po.Poynting(1.0, 3, 4, (-1.0, 1.0), (-1.0, 1.0), (0.0, 1.0))
    res = po.ResidualSpec(id="maxwell_te", epsilon=1.3, mu=0.7)
    F = rng.normal(size=(4 * 9, 3))
    pen, dF = po.poynting_terms(res, F, pc, 4.0 / 9)
    h = 1e-6
    for idx in [(0, 0), (5, 1), (20, 2), (35, 0)]:
        Fp, Fm = F.copy(), F.copy()
        Fp[idx] += h
        Fm[idx] -= h
        fd = (po.poynting_terms(res, Fp, pc, 4.0 / 9)[0] - po.poynting_terms(res, Fm, pc, 4.0 / 9)[0]) / (2 * h)
        assert abs(fd - dF[idx]) <= 1e-6 * max(1.0, abs(fd))


def test_spec_known_answers():
    # Allen-Cahn u == 1/2 -> residual^2 = 3.515625
    O = np.zeros((4, 1, 1))
    O[0, 0, 0] = 0.5
    r = po.residuals(po.ResidualSpec("allen_cahn"), O, po.pde_streams("allen_cahn"))
    assert r[0, 0] ** 2 == pytest.approx(3.515625, abs=1e-15)
    # Maxwell plane wave: with the reference's sign convention
    # (losses.cpp:68-70) Ez = cos(2 pi (x - t)), Hy = -Ez, Hx = 0 is an exact
    # solution (SPEC's "Hy = Ez" has the wrong sign for these equations)
    x = np.linspace(0, 1, 7)
    t = 0.3
    ph = 2 * math.pi * (x - t)
    O = np.zeros((4, x.size, 3))
    O[0, :, 0], O[0, :, 2] = np.cos(ph), -np.cos(ph)
    O[1, :, 0], O[1, :, 2] = -2 * math.pi * np.sin(ph), 2 * math.pi * np.sin(ph)   # d/dx
    O[3, :, 0], O[3, :, 2] = 2 * math.pi * np.sin(ph), -2 * math.pi * np.sin(ph)   # d/dt
    r = po.residuals(po.ResidualSpec("maxwell_te"), O, po.pde_streams("maxwell_te"))
    assert np.max(np.abs(r)) <= 1e-12
    # Adam first step ~ -lr*sign(g)
    a = po.Adam(lr=0.1)
    p = np.array([1.0, -2.0])
    a.step(p, np.array([0.3, -5.0]))
    np.testing.assert_allclose(p, [0.9, -1.9], atol=1e-7)


def test_maxwell_te_eh_extension():
    """maxwell_te_eh (fields Ex, Ey, Hz; BASELINE configs[3] naming) is not in the
    reference (its maxwell_te is the (Ez, Hx, Hy) system, losses.cpp:57-72):
    pinned by a TE plane wave (Hz = Ey = cos(kx - wt), Ex = 0, w = k, eps = mu = 1:
    residuals vanish) and by central FD of the loss gradient on the oracle."""
    streams = po.pde_streams("maxwell_te_eh")
    x = np.linspace(-1, 1, 7)
    t = np.linspace(0, 1, 7)
    k = 2.3
    ph = k * x - k * t
    O = np.zeros((len(streams), x.size, 3))
    c, s = np.cos(ph), np.sin(ph)
    # value, d/dx, d/dy, d/dt of Ex = 0, Ey = cos, Hz = cos
    for f in (1, 2):
        O[0, :, f] = c
        O[streams.index((1, 0)), :, f] = -k * s
        O[streams.index((1, 2)), :, f] = k * s
    r = po.residuals(po.ResidualSpec("maxwell_te_eh"), O, streams)
    assert np.max(np.abs(r)) <= 1e-14
    spec = po.ModelSpec(in_dim=3, hidden_dim=8, depth=2, out_dim=3, activation="tanh")
    res = po.ResidualSpec("maxwell_te_eh", epsilon=1.3, mu=0.7)
    flat, _ = po.init_params(spec, 5)
    pts = po.sample_uniform([(-1, 1), (-1, 1), (0, 1)], [3, 3, 3])
    ic = po.sample_uniform([(-1, 1), (-1, 1), (0, 0)], [3, 3, 1])
    col = po.Collocation(pts, ic, np.stack([np.zeros(9), np.zeros(9), np.exp(-25 * (ic[:, 0] ** 2 + ic[:, 1] ** 2))], 1))
    rng = np.random.default_rng(1)
    _fd_check(spec, res, flat, None, col, "hard", rng.choice(flat.size, 12, replace=False))

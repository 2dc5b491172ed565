"""GPU: collocation designs generated on the device (pnx_sample_points,
sampling.cpp:10-103) -- the uniform grid bit-exact against the reference's
sample_uniform (the fixture interiors were produced by the compiled
reference), the Latin hypercube designs by their defining properties (one point
per stratum and axis, determinism in the seed), shards of the global design,
causality bucketing of a device design, and in-place resampling."""
import numpy as np
import pytest

import golden_io as gi

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2604_15645_b200 as pk
    return pk


def _worker(name, **kw):
    pk = _pkg()
    g = gi.load(name)
    c = g["case"]
    p = c["pde"]
    spec = pk.ModelSpec.from_json(c["model"])
    res = pk.ResidualSpec(p["id"], p.get("advection_c", 1.0), p.get("epsilon", 1.0), p.get("mu", 1.0))
    col = g["col"]
    w = pk.make_worker(spec, res, g["bc"], g["rffB"], col.interior, col.ic_points, col.ic_targets, col.bc_a,
                       col.bc_b, col.bc_targets, **kw)
    return g, w


@pytest.mark.parametrize("name", ["burgers_tanh", "maxwell_tanh", "burgers_c1_full"])
def test_device_uniform_grid_is_the_reference_grid_bit_for_bit(name):
    g, w = _worker(name)
    c = g["case"]
    g1, l1 = w.step(g["params"])
    w.sample_points("uniform", c["domain"], c["collocation"]["dims"])
    pts = w.points()
    assert np.array_equal(pts, g["col"].interior)  # sample_uniform from oracle/_ref
    g2, l2 = w.step(g["params"])
    assert np.array_equal(g1, g2) and l1 == l2


@pytest.mark.parametrize("design", ["lhs", "lhs_per_axis"])
def test_device_lhs_designs_stratify_every_axis(design):
    g, w = _worker("maxwell_tanh")
    dom = [(-1.0, 1.0), (-1.0, 1.0), (0.0, 1.5)]
    dims = [7, 5, 6]
    n = 210
    w.sample_points(design, dom, dims=dims, n=n, seed=11)
    pts = w.points()
    assert pts.shape == (n, 3)
    for a, (lo, hi) in enumerate(dom):
        x = pts[:, a]
        assert np.all((x >= lo) & (x < hi))
        if design == "lhs":  # sample_lhs: each of the n strata of every axis holds one point
            k = np.floor((x - lo) / ((hi - lo) / n)).astype(int)
            assert np.array_equal(np.sort(k), np.arange(n))
        else:  # sample_lhs_per_axis: dims[a] jittered levels, one per stratum, tensor product
            v = np.unique(x)
            assert v.size == dims[a]
            k = np.floor((v - lo) / ((hi - lo) / dims[a])).astype(int)
            assert np.array_equal(k, np.arange(dims[a]))
    if design == "lhs_per_axis":  # last axis fastest, like sample_uniform
        assert np.array_equal(pts[:6, 2], pts[6:12, 2]) and np.all(pts[:6, 0] == pts[0, 0])
    w.sample_points(design, dom, dims=dims, n=n, seed=11)
    assert np.array_equal(w.points(), pts)  # counter-based: same seed, same design
    w.sample_points(design, dom, dims=dims, n=n, seed=12)
    assert not np.array_equal(w.points(), pts)


def test_device_design_shards_concatenate_to_the_global_design():
    pk = _pkg()
    g, w = _worker("maxwell_tanh")
    dom = [(-1.0, 1.0), (-1.0, 1.0), (0.0, 1.5)]
    n = 301
    w.sample_points("lhs", dom, n=n, seed=5)
    full = w.points()
    parts = []
    for lo, hi in pk.shard_interior(n, 3):
        w.sample_points("lhs", dom, n=n, seed=5, rows=(lo, hi))
        parts.append(w.points())
    assert np.array_equal(np.concatenate(parts), full)


def test_device_design_with_causality_matches_the_same_points_uploaded():
    """Causality buckets a device design on the device (split_time_segments,
    trainer.cpp:156-177); the step must equal the step on the same points
    uploaded from the host (bucketed there)."""
    pk = _pkg()
    g, w = _worker("burgers_tanh", causality=pk.CausalityConfig(4, 2.0, 0.0, 1.0))
    dom = g["case"]["domain"]
    w.sample_points("lhs", dom, n=117, seed=3)
    pts = w.points()
    g1, l1 = w.step(g["params"])
    g2_, w2 = _worker("burgers_tanh", causality=pk.CausalityConfig(4, 2.0, 0.0, 1.0))
    w2.set_points(pts)
    g2, l2 = w2.step(g["params"])
    assert np.array_equal(g1, g2) and l1 == l2
    # resampling in place (same size, new seed) and back
    w.sample_points("lhs", dom, n=117, seed=4)
    g3, _ = w.step(g["params"])
    assert not np.array_equal(g3, g1)
    w.sample_points("lhs", dom, n=117, seed=3)
    g4, l4 = w.step(g["params"])
    assert np.array_equal(g4, g1) and l4 == l1


def test_dp_group_device_design():
    """pnx_dp_sample_points: each rank generates its shard of the global design;
    the averaged gradient equals the one over the same points uploaded."""
    pk = _pkg()
    g = gi.load("burgers_tanh")
    c = g["case"]
    spec = pk.ModelSpec.from_json(c["model"])
    res = pk.ResidualSpec("burgers")
    col = g["col"]

    def group():
        grp = pk.pinn.DataParallelGroup(spec, res, g["bc"], None, devices=[0, 0])
        grp.set_ic(col.ic_points, col.ic_targets)
        grp.set_bc(col.bc_a, col.bc_b, col.bc_targets)
        grp.set_params(g["params"])
        return grp

    a = group()
    a.sample_points("uniform", c["domain"], dims=c["collocation"]["dims"])
    la, ga = a.step(update=False, want_grad=True)
    b = group()
    b.set_points(col.interior)
    lb, gb = b.step(update=False, want_grad=True)
    assert np.array_equal(ga, gb) and la == lb
    assert np.linalg.norm(ga - g["grad_w2"]) <= 1e-5 * np.linalg.norm(g["grad_w2"])


def test_device_design_with_chunked_rows_matches_uploaded_points():
    """A device design laid out over several chunks (the 64M-point path: rows
    beyond the activation budget stream through in chunks) gives the step of the
    same points uploaded from the host, bit for bit."""
    pk = _pkg()
    from paper_2604_15645_b200 import configs
    wl = configs.get_config("c4")
    col = configs.collocation(wl, [10, 10, 6])
    flat, rffB = pk.init_params(wl.spec, seed=4)
    dom = wl.domain
    a = pk.make_worker(wl.spec, wl.res, wl.bc, rffB, **col)
    a.sample_points("lhs", dom, n=1500, seed=9)
    a.set_chunk_rows(512)
    ga, la = a.step(flat)
    pts = a.points()
    b = pk.make_worker(wl.spec, wl.res, wl.bc, rffB, **dict(col, interior=pts))
    b.set_chunk_rows(512)
    gb, lb = b.step(flat)
    assert np.array_equal(ga, gb) and la == lb

"""GPU: pnx_step's per-context CUDA graph (the second call with unchanged inputs
captures the device step, later calls replay it). Replays must give the eager
step bit for bit, and every input change must be seen: same-size point uploads
(device memory the graph reads), new lambdas, new IC / boundary data, a new
point count, a device design, the engine -- each checked against a fresh
context that never captured anything."""
import numpy as np
import pytest

import golden_io as gi

pytestmark = pytest.mark.gpu


def _make(name, **kw):
    import paper_2604_15645_b200 as pk
    g = gi.load(name)
    c = g["case"]
    p = c["pde"]
    spec = pk.ModelSpec.from_json(c["model"])
    res = pk.ResidualSpec(p["id"], p.get("advection_c", 1.0), p.get("epsilon", 1.0), p.get("mu", 1.0))
    col = g["col"]
    args = dict(interior=col.interior, ic_points=col.ic_points, ic_targets=col.ic_targets, bc_a=col.bc_a,
                bc_b=col.bc_b, bc_targets=col.bc_targets)
    args.update(kw)
    return pk, g, pk.make_worker(spec, res, g["bc"], g["rffB"], **args)


@pytest.mark.parametrize("name", ["burgers_tanh", "maxwell_c4_shape", "burgers_c2_shape"])
def test_replays_match_eager_and_track_input_changes(name):
    pk, g, w = _make(name)
    p = g["params"]
    outs = [w.step(p) for _ in range(4)]  # eager, capture, replay, replay
    for gr, l in outs[1:]:
        assert np.array_equal(gr, outs[0][0]) and l == outs[0][1]

    # same-size points: the graph reads the new coordinates
    pts = g["col"].interior.copy()
    pts[:, 0] = pts[:, 0] * 0.9 + 0.01
    w.set_points(pts)
    for _ in range(3):
        ga, la = w.step(p)
    _, _, fresh = _make(name, interior=pts)
    gb, lb = fresh.step(p)
    assert np.array_equal(ga, gb) and la == lb

    # new lambdas
    lam = (0.7, 1.3, 0.5)
    for _ in range(3):
        ga, la = w.step(p, lam)
    gb, lb = fresh.step(p, lam)
    assert np.array_equal(ga, gb) and la == lb

    # new IC targets
    col = g["col"]
    t2 = col.ic_targets * 1.1
    w.set_ic(col.ic_points, t2)
    for _ in range(3):
        ga, la = w.step(p, lam)
    _, _, fresh2 = _make(name, interior=pts, ic_targets=t2)
    gb, lb = fresh2.step(p, lam)
    assert np.array_equal(ga, gb) and la == lb

    # a different point count (new row layout)
    few = pts[: len(pts) // 2 + 3]
    w.set_points(few)
    for _ in range(3):
        ga, la = w.step(p, lam)
    _, _, fresh3 = _make(name, interior=few, ic_targets=t2)
    gb, lb = fresh3.step(p, lam)
    assert np.array_equal(ga, gb) and la == lb


def test_engine_switch_and_device_design_after_capture():
    pk, g, w = _make("maxwell_c4_shape")
    p = g["params"]
    for _ in range(3):
        w.step(p)
    w.set_engine("ffma")
    for _ in range(3):
        ga, la = w.step(p)
    _, _, fresh = _make("maxwell_c4_shape", engine="ffma")
    gb, lb = fresh.step(p)
    assert np.array_equal(ga, gb) and la == lb
    dom = g["case"]["domain"]
    w.sample_points("lhs", dom, n=333, seed=7)
    for _ in range(3):
        ga, la = w.step(p)
    pts = w.points()
    _, _, fresh2 = _make("maxwell_c4_shape", engine="ffma", interior=pts)
    gb, lb = fresh2.step(p)
    assert np.array_equal(ga, gb) and la == lb

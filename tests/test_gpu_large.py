"""GPU: size-independent properties at BASELINE sizes (C4/C5's Maxwell 6x256).

* Equal-shard identity (trainer.cpp:264-281): for equal shards the
  rank-ordered average of the shard gradients equals the full-set gradient. One
  worker steps 8,388,608 points (the C5 8M-per-GPU size: several chunks
  streamed through HBM); eight workers step the eight 1M shards of the same
  device-generated grid; averages and the full step agree to FP32 accuracy.
* The device grid at 8M points is the reference's sample_uniform, bit for bit,
  on a sampled subset of rows (the full 8M host grid is built once, in numpy).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_equal_shard_identity_at_8M_points():
    import paper_2604_15645_b200 as pk
    from paper_2604_15645_b200 import configs
    wl = configs.get_config("c4")
    dims = configs.weak_scaling_dims(1 << 23, 1)
    n = int(np.prod(dims))
    assert n == 1 << 23
    col = configs.collocation(wl, dims, with_interior=False)
    flat, rffB = pk.init_params(wl.spec, seed=0)

    def worker(rows):
        w = pk.Worker(wl.spec, wl.res, wl.bc, rffB)
        w.sample_points("uniform", wl.domain, dims, rows=rows)
        w.set_ic(col["ic_points"], col["ic_targets"])
        return w

    full = worker((0, n))
    g_full, l_full = full.step(flat)
    # the device grid is sample_uniform (last axis fastest): spot-check rows
    host = configs.grid(wl.domain, dims)
    pts = full.points()
    idx = np.random.default_rng(0).integers(0, n, 4096)
    assert np.array_equal(pts[idx], host[idx])
    del full, pts, host

    W = 8
    g_sum = np.zeros_like(g_full)
    l_sum = {"pde": 0.0, "ic": 0.0, "bc": 0.0}
    for lo, hi in pk.shard_interior(n, W):
        g, l = worker((lo, hi)).step(flat)
        g_sum += g
        for k in l_sum:
            l_sum[k] += l[k]
    g_avg = g_sum / W
    err = float(np.linalg.norm(g_avg - g_full) / np.linalg.norm(g_full))
    assert err <= 1e-5, err
    for k in ("pde", "ic"):
        assert abs(l_sum[k] / W - l_full[k]) <= 1e-5 * abs(l_full[k]), (k, l_sum[k] / W, l_full[k])

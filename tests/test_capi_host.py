"""CPU: the C-ABI library loads and exports every symbol include/pnx.h declares
(no compute calls without a GPU); host-side mirror logic."""
import ctypes
import os
import re

import numpy as np
import pytest

import golden_io as gi

ROOT = gi.ROOT
LIB = os.path.join(ROOT, "paper_2604_15645_b200", "libpnx.so")


def _header_functions():
    src = open(os.path.join(ROOT, "include", "pnx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(pnx_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2604_15645_b200 import build
        build.build()
    return ctypes.CDLL(LIB)


def test_library_exports_every_header_symbol(lib):
    names = _header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_header():
    from paper_2604_15645_b200 import _lib
    assert sorted(_lib.EXPORTS) == _header_functions()


def test_library_is_sm100a(lib):
    out = os.popen(f"cuobjdump --list-elf {LIB} 2>&1").read()
    assert "sm_100a" in out


def test_create_without_gpu_fails_loudly():
    """No CPU fallback: on a box without a GPU pnx_create must fail."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2604_15645_b200 as pk
    with pytest.raises(pk.TensorError, match="no CUDA device|CUDA"):
        pk.Worker(pk.ModelSpec(2, 8, 2, 1), pk.ResidualSpec("burgers"))


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: loading a library that is not there raises (in a child
    interpreter, so this process keeps its loaded libpnx.so)."""
    import subprocess
    import sys
    code = ("from paper_2604_15645_b200 import _lib\n"
            "try:\n    _lib.load()\nexcept RuntimeError as e:\n    print('RAISED', e)\n")
    env = dict(os.environ, PNX_LIB_PATH=str(tmp_path / "absent" / "libpnx.so"))
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=120)
    assert "RAISED" in out.stdout and "no CPU fallback" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("name", gi.CASE_NAMES)
def test_param_layout_mirror(name):
    import paper_2604_15645_b200 as pk
    g = gi.load(name)
    spec = pk.ModelSpec.from_json(g["case"]["model"])
    assert pk.param_layout(spec) == [(p["name"], tuple(p["shape"])) for p in g["meta"]["params"]]
    assert pk.param_count(spec) == g["params"].size


def test_shards():
    import paper_2604_15645_b200 as pk
    assert pk.shard_interior(10, 3) == [(0, 3), (3, 6), (6, 10)]
    with pytest.raises(pk.TensorError):
        pk.shard_interior(2, 3)


def test_config_collocation_matches_oracle():
    from oracle import pinn_oracle as po
    from paper_2604_15645_b200 import configs
    for key in ("c1", "c2", "c4"):
        wl = configs.get_config(key)
        dims = [min(d, 9) for d in wl.dims]
        col = configs.collocation(wl, dims)
        oc = po.build_collocation(wl.domain, dims, wl.n_ic, wl.n_bc, wl.bc, wl.initial, wl.spec.out_dim)
        np.testing.assert_array_equal(col["interior"], oc.interior)
        np.testing.assert_array_equal(col["ic_points"], oc.ic_points)
        np.testing.assert_allclose(col["ic_targets"], oc.ic_targets, atol=1e-15)


def test_flops_per_point_match_survey():
    from paper_2604_15645_b200 import configs
    assert configs.get_config("c1").flops_per_point() == 224_640
    assert configs.get_config("c2").flops_per_point() == 1_476_864
    assert configs.get_config("c3").flops_per_point() == 1_985_280
    assert configs.get_config("c4").flops_per_point() == 7_901_184


def test_library_loads_before_torch():
    """libpnx links the libnccl.so.2 torch bundles (rpath): loading it first must
    not shadow torch's NCCL (libtorch_cuda needs symbols the image's older
    /usr/lib libnccl lacks)."""
    import subprocess
    import sys
    from paper_2604_15645_b200 import _lib
    code = f"import ctypes; ctypes.CDLL({_lib.LIB_PATH!r}); import torch; print(torch.__version__)"
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]

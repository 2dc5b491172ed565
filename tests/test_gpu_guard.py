"""GPU: out-of-bounds writes into the context's device buffers (a stand-in for
compute-sanitizer memcheck, which this GPU pool does not allow). With
PNX_GUARD=1 every buffer carries a 512-byte tail with a fixed pattern that
pnx_check verifies; tests/_guard_run.py steps every kernel family (goldens on both
engines incl. per-term passes, causality and Poynting; C1-C4 shapes on all
engines, chunked; device LHS designs) and must finish clean. PNX_GUARD=poke is
the negative control: a byte of each tail is overwritten at allocation, and the
first check must report it."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(mode):
    env = dict(os.environ, PNX_GUARD=mode)
    return subprocess.run([sys.executable, os.path.join(HERE, "_guard_run.py")], env=env, capture_output=True,
                          text=True, timeout=900)


def test_no_kernel_writes_past_its_buffers():
    r = _run("1")
    assert r.returncode == 0 and "guards ok" in r.stdout, r.stderr[-3000:]


def test_guard_detects_a_write_past_the_end():
    r = _run("poke")
    assert r.returncode != 0 and "guard: write past the end" in r.stderr, (r.returncode, r.stderr[-2000:])

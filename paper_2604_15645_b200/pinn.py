"""Host-side mirror of the reference pinnlab interface for the train-step path.

Names and argument meaning follow /root/reference/proj/core:

* ``ModelSpec`` / ``AxisPeriodic`` / ``RFFSpec`` / ``RWFSpec``   model.hpp:14-57
* ``ResidualSpec`` (+ ``ns_steady`` extension)                 losses.hpp:14-30
* ``param_layout`` -- Model::trainable() order/shapes          model.cpp:64-101
* ``Worker.step`` -- run_worker_epoch                            trainer.cpp:200-262
* ``shard_interior``                                             trainer.cpp:143-154
* ``data_parallel_gradient``                                     trainer.cpp:649-678

Every compute call goes through the C ABI of ``libpnx.so`` (include/pnx.h);
there is no CPU fallback: constructing a Worker without the CUDA library or
without a GPU raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib

ACTIVATIONS = {"tanh": 0, "sine": 1, "swish": 2}
PDES = {"advection": 0, "allen_cahn": 1, "burgers": 2, "maxwell_te": 3, "ns_steady": 4, "maxwell_te_eh": 5}
BCS = {"hard": 0, "soft_periodic": 1, "dirichlet_zero": 2}
ENGINES = {"auto": 0, "ffma": 1, "tc3xtf32": 2, "tc3xf16": 3}


class TensorError(RuntimeError):
    """Mirror of pinnlab::TensorError (tensor.hpp:14-17)."""


@dataclass
class AxisPeriodic:
    periodic: bool = False
    period: float = 0.0
    trainable: bool = False


@dataclass
class RFFSpec:
    width: int = 64
    sigma: float = 10.0
    mean: float = 0.0


@dataclass
class RWFSpec:
    mean: float = 1.0
    stddev: float = 0.1


@dataclass
class ModelSpec:
    in_dim: int = 2
    hidden_dim: int = 64
    depth: int = 3
    out_dim: int = 1
    activation: str = "tanh"
    sine_w0: float = 1.0
    periodic_axes: List[AxisPeriodic] = field(default_factory=list)
    rff: Optional[RFFSpec] = None
    rwf: Optional[RWFSpec] = None

    def embedded_width(self) -> int:
        if not self.periodic_axes:
            return self.in_dim
        return sum(2 if a.periodic else 1 for a in self.periodic_axes)

    def first_layer_width(self) -> int:
        return 2 * self.rff.width if self.rff else self.embedded_width()

    @staticmethod
    def from_json(j: dict) -> "ModelSpec":
        s = ModelSpec(in_dim=j["in_dim"], hidden_dim=j["hidden_dim"], depth=j["depth"],
                      out_dim=j["out_dim"], activation=j["activation"], sine_w0=j.get("sine_w0", 1.0))
        for a in j.get("periodic_axes", []):
            s.periodic_axes.append(AxisPeriodic(a["periodic"], a["period"], a.get("trainable", False)))
        if "rff" in j:
            s.rff = RFFSpec(j["rff"]["width"], j["rff"].get("sigma", 10.0), j["rff"].get("mean", 0.0))
        if "rwf" in j:
            s.rwf = RWFSpec(j["rwf"].get("mean", 1.0), j["rwf"].get("stddev", 0.1))
        return s


@dataclass
class ResidualSpec:
    id: str = "advection"
    advection_c: float = 1.0
    epsilon: float = 1.0
    mu: float = 1.0
    reynolds: float = 100.0

    def field_count(self) -> int:
        return 3 if self.id in ("maxwell_te", "maxwell_te_eh", "ns_steady") else 1

    def coord_count(self) -> int:
        return 3 if self.id in ("maxwell_te", "maxwell_te_eh") else 2


def param_layout(spec: ModelSpec) -> List[Tuple[str, Tuple[int, ...]]]:
    """Model::trainable() names and shapes (model.cpp:64-101)."""
    out = []
    dims = [spec.first_layer_width()] + [spec.hidden_dim] * spec.depth + [spec.out_dim]
    for l in range(spec.depth + 1):
        i, o = dims[l], dims[l + 1]
        if spec.rwf:
            out += [(f"layer{l}.V", (i, o)), (f"layer{l}.s", (1, o))]
        else:
            out.append((f"layer{l}.W", (i, o)))
        out.append((f"layer{l}.b", (1, o)))
    for a, ax in enumerate(spec.periodic_axes):
        if ax.periodic and ax.trainable:
            out.append((f"periodic.P{a}", ()))
    return out


def param_count(spec: ModelSpec) -> int:
    return sum(int(np.prod(s)) if s else 1 for _, s in param_layout(spec))


def init_params(spec: ModelSpec, seed: int = 0):
    """Xavier-normal W, zero b, RWF s ~ N(mean, std), RFF B ~ N(mean, sigma)
    -- the distributions of Model::Model (model.cpp:58-101), drawn with numpy."""
    rng = np.random.default_rng(seed)
    rffB = None
    if spec.rff:
        rffB = rng.normal(spec.rff.mean, spec.rff.sigma, size=(spec.embedded_width(), spec.rff.width))
    flat = []
    for name, shape in param_layout(spec):
        n = int(np.prod(shape)) if shape else 1
        if name.endswith((".W", ".V")):
            flat.append(rng.normal(0.0, math.sqrt(2.0 / (shape[0] + shape[1])), size=n))
        elif name.endswith(".s"):
            flat.append(rng.normal(spec.rwf.mean, spec.rwf.stddev, size=n))
        elif name.endswith(".b"):
            flat.append(np.zeros(n))
        else:
            flat.append(np.array([spec.periodic_axes[int(name.split("P")[-1])].period]))
    return np.concatenate(flat), rffB


def shard_interior(n: int, workers: int) -> List[Tuple[int, int]]:
    """Contiguous shards, last absorbs the remainder (trainer.cpp:143-154)."""
    base = n // workers
    if base == 0:
        raise TensorError("data parallel: fewer interior points than workers")
    return [(w * base, n if w + 1 == workers else (w + 1) * base) for w in range(workers)]


def _axis_major(pts: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(pts, dtype=np.float64).T)


SAMPLE_DESIGNS = {"uniform": 0, "lhs": 1, "lhs_per_axis": 2}


def _design_args(design, bounds, dims, n):
    b = (C.c_double * (2 * len(bounds)))(*[float(v) for lo_hi in bounds for v in lo_hi])
    if design == "lhs":
        return b, None, int(n)
    d = (C.c_int64 * len(dims))(*[int(x) for x in dims])
    return b, d, int(np.prod([int(x) for x in dims]))


def _descs(spec: ModelSpec, res: ResidualSpec, bc: str, rff_B):
    """pnx_model_desc / pnx_problem_desc of a ModelSpec / ResidualSpec (+ the
    arrays they point to, which must outlive the call)."""
    per = spec.periodic_axes
    keep = []
    md = _lib.ModelDesc()
    md.in_dim, md.hidden_dim, md.depth, md.out_dim = spec.in_dim, spec.hidden_dim, spec.depth, spec.out_dim
    md.activation = ACTIVATIONS[spec.activation]
    md.sine_w0 = spec.sine_w0
    md.n_periodic_axes = len(per)
    if per:
        a = (C.c_int32 * len(per))(*[int(x.periodic) for x in per])
        b = (C.c_double * len(per))(*[float(x.period) for x in per])
        c = (C.c_int32 * len(per))(*[int(x.trainable) for x in per])
        keep += [a, b, c]
        md.periodic, md.period, md.period_trainable = a, b, c
    md.rff_width = spec.rff.width if spec.rff else 0
    if spec.rff:
        B = np.ascontiguousarray(np.asarray(rff_B, dtype=np.float64))
        if B.shape != (spec.embedded_width(), spec.rff.width):
            raise TensorError("rff_B must be [embedded_width x rff.width]")
        keep.append(B)
        md.rff_B = B.ctypes.data_as(C.POINTER(C.c_double))
    md.rwf = 1 if spec.rwf else 0
    pd = _lib.ProblemDesc()
    pd.pde = PDES[res.id]
    pd.advection_c, pd.epsilon, pd.mu, pd.reynolds = res.advection_c, res.epsilon, res.mu, res.reynolds
    pd.bc = BCS[bc]
    return md, pd, keep


class Worker:
    """One pnx context: a replica of the worker step on one CUDA device."""

    def __init__(self, spec: ModelSpec, res: ResidualSpec, bc: str = "hard",
                 rff_B: Optional[np.ndarray] = None, device: int = 0, engine: str = "auto", _ctx=None):
        self.lib = _lib.load()
        self.spec, self.res, self.bc = spec, res, bc
        self._owned = _ctx is None
        if _ctx is None:
            md, pd, self._keep = _descs(spec, res, bc, rff_B)
            ctx = C.c_void_p()
            rc = self.lib.pnx_create(C.byref(md), C.byref(pd), device, C.byref(ctx))
            if rc != 0:
                raise TensorError(self.lib.pnx_create_error().decode())
        else:  # a rank context owned by a DataParallelGroup
            ctx = _ctx
        self.ctx = ctx
        n = C.c_int64()
        self.lib.pnx_param_count(ctx, C.byref(n))
        self.n_params = n.value
        self.device = device
        self.set_engine(engine)

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx and getattr(self, "_owned", False):
            self.lib.pnx_destroy(ctx)
        self.ctx = None

    def _chk(self, rc):
        if rc != 0:
            raise TensorError(self.lib.pnx_last_error(self.ctx).decode())

    def set_engine(self, engine: str):
        self._chk(self.lib.pnx_set_engine(self.ctx, ENGINES[engine]))

    def set_chunk_rows(self, rows: int):
        self._chk(self.lib.pnx_set_chunk_rows(self.ctx, int(rows)))

    def set_points(self, pts: np.ndarray, axis_major: bool = False):
        """Interior shard: [N, d] points, or an axis-major [d, N] float64 array
        with axis_major=True (no host transpose; pinned buffers DMA directly)."""
        if axis_major:
            a = pts if (pts.dtype == np.float64 and pts.flags.c_contiguous) else np.ascontiguousarray(pts, np.float64)
        else:
            a = _axis_major(pts)
        self._chk(self.lib.pnx_set_points(self.ctx, a.ctypes.data_as(C.POINTER(C.c_double)),
                                          a.shape[1], a.shape[0]))
        self.n_interior = int(a.shape[1])

    def sample_points(self, design: str, bounds, dims=None, n: int = 0, seed: int = 0, rows=None):
        """Interior generated on the device (pnx_sample_points): design "uniform"
        (sample_uniform), "lhs" (sample_lhs, n points) or "lhs_per_axis"
        (sample_lhs_per_axis); rows = (lo, hi) of the global design (default all)."""
        b, d, total = _design_args(design, bounds, dims, n)
        lo, hi = rows if rows is not None else (0, total)
        self._chk(self.lib.pnx_sample_points(self.ctx, SAMPLE_DESIGNS[design], b, d, int(n), int(seed), int(lo),
                                             int(hi)))
        self.n_interior = int(hi - lo)

    def set_ic(self, pts: np.ndarray, targets: np.ndarray):
        a = _axis_major(pts)
        t = _axis_major(targets)  # [F][n]
        self._chk(self.lib.pnx_set_ic(self.ctx, a.ctypes.data_as(C.POINTER(C.c_double)),
                                      t.ctypes.data_as(C.POINTER(C.c_double)), a.shape[1]))

    def set_bc(self, a_pts: Optional[np.ndarray], b_pts: Optional[np.ndarray] = None,
               targets: Optional[np.ndarray] = None):
        if a_pts is None:
            self._chk(self.lib.pnx_set_bc(self.ctx, None, None, None, 0))
            return
        a = _axis_major(a_pts)
        b = _axis_major(b_pts) if b_pts is not None else None
        t = _axis_major(targets) if targets is not None else None
        P = C.POINTER(C.c_double)
        self._chk(self.lib.pnx_set_bc(self.ctx, a.ctypes.data_as(P),
                                      b.ctypes.data_as(P) if b is not None else None,
                                      t.ctypes.data_as(P) if t is not None else None, a.shape[1]))

    def step(self, params: np.ndarray, lambdas=(1.0, 1.0, 1.0), out: np.ndarray = None):
        """run_worker_epoch equivalent: returns (grad float64 [P], losses dict);
        `out` (float64 [P], contiguous) receives the gradient when given."""
        p = params if (isinstance(params, np.ndarray) and params.dtype == np.float64 and params.flags.c_contiguous) \
            else np.ascontiguousarray(np.asarray(params, dtype=np.float64))
        if p.size != self.n_params:
            raise TensorError("adam: parameter/gradient count mismatch")
        if out is not None and not (out.dtype == np.float64 and out.flags.c_contiguous and out.size == self.n_params):
            raise TensorError("adam: parameter/gradient count mismatch")
        g = out if out is not None else np.empty(self.n_params, dtype=np.float64)
        lam = (C.c_double * 3)(*lambdas)
        losses = (C.c_double * 3)()
        P = C.POINTER(C.c_double)
        self._chk(self.lib.pnx_step(self.ctx, p.ctypes.data_as(P), lam, g.ctypes.data_as(P), losses))
        return g, {"pde": losses[0], "ic": losses[1], "bc": losses[2]}

    def step_device(self, params, grad, lambdas=(1.0, 1.0, 1.0), losses=None, stream=None):
        """Device-resident step on torch tensors (float32 params/grad, float64 losses[3])."""
        lam = (C.c_double * 3)(*lambdas)
        st = C.c_void_p(stream) if stream is not None else None
        self._chk(self.lib.pnx_step_device(self.ctx, C.c_void_p(params.data_ptr()), lam,
                                           C.c_void_p(grad.data_ptr()),
                                           C.c_void_p(losses.data_ptr()) if losses is not None else None, st))

    def step_terms(self, params: np.ndarray):
        """Gradients of l_pde, l_ic, l_bc alone (trainer.cpp:256-260): ([3, P], losses)."""
        p = np.ascontiguousarray(np.asarray(params, dtype=np.float64))
        g = np.empty((3, self.n_params), dtype=np.float64)
        losses = (C.c_double * 3)()
        P = C.POINTER(C.c_double)
        self._chk(self.lib.pnx_step_terms(self.ctx, p.ctypes.data_as(P), g.ctypes.data_as(P), losses))
        return g, {"pde": losses[0], "ic": losses[1], "bc": losses[2]}

    def step_terms_device(self, params, grads3, losses=None, stream=None):
        """Device variant: grads3 is a float32 tensor of 3 x P (pde | ic | bc)."""
        st = C.c_void_p(stream) if stream is not None else None
        self._chk(self.lib.pnx_step_terms_device(self.ctx, C.c_void_p(params.data_ptr()),
                                                 C.c_void_p(grads3.data_ptr()),
                                                 C.c_void_p(losses.data_ptr()) if losses is not None else None, st))

    def set_causality(self, cfg: Optional[CausalityConfig]):
        if cfg is None:
            self._chk(self.lib.pnx_set_causality(self.ctx, 0, 1.0, 0.0, 1.0))
        else:
            self._chk(self.lib.pnx_set_causality(self.ctx, int(cfg.segments), float(cfg.epsilon),
                                                 float(cfg.t_lo), float(cfg.t_hi)))

    def set_poynting(self, cfg: Optional[PoyntingConfig]):
        box = (C.c_double * 6)(*(cfg.box if cfg is not None else (0.0,) * 6))
        w = float(cfg.weight) if cfg is not None else 0.0
        self._chk(self.lib.pnx_set_poynting(self.ctx, w, int(cfg.grid) if cfg else 0,
                                            int(cfg.time_samples) if cfg else 0, box))

    def penalty(self) -> float:
        v = C.c_double()
        self._chk(self.lib.pnx_last_penalty(self.ctx, C.byref(v)))
        return v.value

    def check(self):
        self._chk(self.lib.pnx_check(self.ctx))

    def adam_step_device(self, params, grad, m, v, t: int, lr: float, beta1=0.9, beta2=0.999,
                         eps=1e-8, grad_scale=1.0, stream=None):
        st = C.c_void_p(stream) if stream is not None else None
        self._chk(self.lib.pnx_adam_step_device(
            self.ctx, C.c_void_p(params.data_ptr()), C.c_void_p(grad.data_ptr()), C.c_void_p(m.data_ptr()),
            C.c_void_p(v.data_ptr()), params.numel(), lr, beta1, beta2, eps, t, grad_scale, st))

    def adam_step_device_state(self, params, grad, m, v, state, lr0: float, gamma=1.0, beta1=0.9, beta2=0.999,
                               eps=1e-8, grad_scale=1.0, stream=None):
        """Adam with (steps, epoch) in the float64 device tensor `state` (graph-capturable)."""
        st = C.c_void_p(stream) if stream is not None else None
        self._chk(self.lib.pnx_adam_step_device_state(
            self.ctx, C.c_void_p(params.data_ptr()), C.c_void_p(grad.data_ptr()), C.c_void_p(m.data_ptr()),
            C.c_void_p(v.data_ptr()), params.numel(), C.c_void_p(state.data_ptr()), lr0, gamma, beta1, beta2, eps,
            grad_scale, st))

    def capture_residuals(self, on: bool = True):
        self._chk(self.lib.pnx_capture_residuals(self.ctx, 1 if on else 0))

    def points(self) -> np.ndarray:
        """The interior points of the next step as [N, d] (device designs included)."""
        out = np.empty((self.spec.in_dim, self.n_interior), dtype=np.float64)
        self._chk(self.lib.pnx_copy_points(self.ctx, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out.T.copy()

    def residuals(self, n_interior: int) -> np.ndarray:
        out = np.empty((self.res.field_count(), n_interior), dtype=np.float64)
        self._chk(self.lib.pnx_copy_residuals(self.ctx, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def profile(self, on: bool = True):
        self._chk(self.lib.pnx_profile(self.ctx, 1 if on else 0))

    def profile_read(self):
        """{class: (ms, launches)} accumulated since profile(True)."""
        ms = (C.c_double * 7)()
        n = (C.c_int64 * 7)()
        self._chk(self.lib.pnx_profile_read(self.ctx, ms, n, 7))
        names = ["input", "fwd_gemm", "head", "bwd_gemm", "wgrad_gemm", "finalize", "fused_step"]
        return {names[i]: (ms[i], n[i]) for i in range(7)}

    def launch_count(self) -> int:
        n = C.c_int64()
        self._chk(self.lib.pnx_last_launch_count(self.ctx, C.byref(n)))
        return n.value


@dataclass
class CausalityConfig:
    """trainer.hpp:51-55, with the time interval of the domain's last axis."""
    segments: int = 10
    epsilon: float = 1.0
    t_lo: float = 0.0
    t_hi: float = 1.0


@dataclass
class PoyntingConfig:
    """trainer.hpp:57-61, with the (x, y, t) box it integrates over."""
    weight: float = 0.0
    grid: int = 32
    time_samples: int = 4
    box: Tuple[float, float, float, float, float, float] = (-1.0, 1.0, -1.0, 1.0, 0.0, 1.0)


@dataclass
class BalancingConfig:
    """trainer.hpp:45-49."""
    enabled: bool = True
    alpha: float = 0.9
    update_period: int = 100


def make_worker(spec, res, bc, rff_B, interior, ic_points, ic_targets, bc_a=None, bc_b=None,
                bc_targets=None, device=0, engine="auto", causality: Optional[CausalityConfig] = None,
                poynting: Optional[PoyntingConfig] = None) -> Worker:
    w = Worker(spec, res, bc, rff_B, device=device, engine=engine)
    w.set_points(interior)
    if ic_points is not None and len(ic_points):
        w.set_ic(ic_points, ic_targets)
    if bc != "hard":
        w.set_bc(bc_a, bc_b, bc_targets)
    if causality is not None:
        w.set_causality(causality)
    if poynting is not None:
        w.set_poynting(poynting)
    return w


def data_parallel_gradient(spec, res, bc, params, rff_B, interior, ic_points, ic_targets, bc_a=None,
                           bc_b=None, bc_targets=None, workers: int = 1, lambdas=(1.0, 1.0, 1.0),
                           device=0, engine="auto", causality: Optional[CausalityConfig] = None,
                           poynting: Optional[PoyntingConfig] = None):
    """trainer.cpp:649-678 on one device: shard, per-worker step, rank-ordered
    average (sum x 1/W, trainer.cpp:264-281). Returns (grad, per-worker losses);
    with a Poynting penalty each loss dict also carries 'pen'."""
    outs = []
    g = None
    for a, b in shard_interior(len(interior), workers):
        w = make_worker(spec, res, bc, rff_B, interior[a:b], ic_points, ic_targets, bc_a, bc_b,
                        bc_targets, device=device, engine=engine, causality=causality, poynting=poynting)
        gw, lw = w.step(params, lambdas)
        lw["pen"] = w.penalty()
        outs.append(lw)
        g = gw.copy() if g is None else g + gw
    return g * (1.0 / workers), outs


class DataParallelGroup:
    """pnx_dp (include/pnx.h): R ranks over local GPUs -- train()'s worker
    threads + average_grads + replica update (trainer.cpp:441-460, 264-281,
    626-638) with one NCCL all-reduce of the packed [grad | losses] per step and
    the device Adam on every replica. `devices[r]` is rank r's GPU; ranks that
    share a GPU are summed on it before the all-reduce."""

    def __init__(self, spec: ModelSpec, res: ResidualSpec, bc: str = "hard", rff_B=None,
                 devices: Sequence[int] = (0,), engine: str = "auto"):
        self.lib = _lib.load()
        self.spec, self.res, self.bc = spec, res, bc
        md, pd, self._keep = _descs(spec, res, bc, rff_B)
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        rc = self.lib.pnx_dp_create(C.byref(md), C.byref(pd), devs, len(devices), C.byref(h))
        if rc != 0:
            raise TensorError(self.lib.pnx_create_error().decode() or "pnx_dp_create failed")
        self.h = h
        self.R = len(devices)
        self.devices = list(devices)
        self.workers = []
        for r in range(self.R):
            c = C.c_void_p()
            self._chk(self.lib.pnx_dp_rank_ctx(h, r, C.byref(c)))
            self.workers.append(Worker(spec, res, bc, None, device=devices[r], engine=engine, _ctx=c))
        self.n_params = self.workers[0].n_params

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            for w in getattr(self, "workers", []):
                w.ctx = None
            self.lib.pnx_dp_destroy(h)
            self.h = None

    def _chk(self, rc):
        if rc != 0:
            raise TensorError(self.lib.pnx_dp_last_error(self.h).decode())

    def size(self):
        r, d = C.c_int(), C.c_int()
        self._chk(self.lib.pnx_dp_size(self.h, C.byref(r), C.byref(d)))
        return r.value, d.value

    def set_points(self, pts: np.ndarray):
        a = _axis_major(pts)
        self._chk(self.lib.pnx_dp_set_points(self.h, a.ctypes.data_as(C.POINTER(C.c_double)), a.shape[1],
                                             a.shape[0]))

    def sample_points(self, design: str, bounds, dims=None, n: int = 0, seed: int = 0):
        """The global interior as a device design (pnx_dp_sample_points), sharded over the ranks."""
        b, d, _ = _design_args(design, bounds, dims, n)
        self._chk(self.lib.pnx_dp_sample_points(self.h, SAMPLE_DESIGNS[design], b, d, int(n), int(seed)))

    def set_ic(self, pts, targets):
        a, t = _axis_major(pts), _axis_major(targets)
        P = C.POINTER(C.c_double)
        self._chk(self.lib.pnx_dp_set_ic(self.h, a.ctypes.data_as(P), t.ctypes.data_as(P), a.shape[1]))

    def set_bc(self, a_pts, b_pts=None, targets=None):
        P = C.POINTER(C.c_double)
        if a_pts is None:
            self._chk(self.lib.pnx_dp_set_bc(self.h, None, None, None, 0))
            return
        a = _axis_major(a_pts)
        b = _axis_major(b_pts) if b_pts is not None else None
        t = _axis_major(targets) if targets is not None else None
        self._chk(self.lib.pnx_dp_set_bc(self.h, a.ctypes.data_as(P), b.ctypes.data_as(P) if b is not None else None,
                                         t.ctypes.data_as(P) if t is not None else None, a.shape[1]))

    def set_params(self, flat):
        p = np.ascontiguousarray(np.asarray(flat, dtype=np.float64))
        self._chk(self.lib.pnx_dp_set_params(self.h, p.ctypes.data_as(C.POINTER(C.c_double))))

    def params(self, rank: int = 0) -> np.ndarray:
        out = np.empty(self.n_params, dtype=np.float64)
        self._chk(self.lib.pnx_dp_get_params(self.h, rank, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def set_optimizer(self, lr=1e-3, gamma=1.0, beta1=0.9, beta2=0.999, eps=1e-8):
        self._chk(self.lib.pnx_dp_set_optimizer(self.h, lr, gamma, beta1, beta2, eps))

    def set_graph(self, on: bool = True):
        self._chk(self.lib.pnx_dp_set_graph(self.h, 1 if on else 0))

    def step(self, lambdas=(1.0, 1.0, 1.0), update: bool = True, sync: bool = True, want_grad: bool = False):
        """One synchronized step; returns ({pde, ic, bc, pen} means over ranks[, averaged grad])
        when sync, else None (enqueue only)."""
        lam = (C.c_double * 3)(*lambdas)
        P = C.POINTER(C.c_double)
        l4 = (C.c_double * 4)()
        g = np.empty(self.n_params, dtype=np.float64) if want_grad else None
        self._chk(self.lib.pnx_dp_step(self.h, lam, 1 if update else 0, l4 if (sync or want_grad) else None,
                                       g.ctypes.data_as(P) if want_grad else None))
        if not (sync or want_grad):
            return None
        losses = {"pde": l4[0], "ic": l4[1], "bc": l4[2], "pen": l4[3]}
        return (losses, g) if want_grad else losses

    def step_terms(self):
        g = np.empty((3, self.n_params), dtype=np.float64)
        l3 = (C.c_double * 3)()
        self._chk(self.lib.pnx_dp_step_terms(self.h, g.ctypes.data_as(C.POINTER(C.c_double)), l3))
        return g, {"pde": l3[0], "ic": l3[1], "bc": l3[2]}

    def apply_gradient(self, g):
        a = np.ascontiguousarray(np.asarray(g, dtype=np.float64))
        self._chk(self.lib.pnx_dp_apply_gradient(self.h, a.ctypes.data_as(C.POINTER(C.c_double))))

    def check(self):
        self._chk(self.lib.pnx_dp_check(self.h))

#!/usr/bin/env python
"""PINN train-step throughput (collocation points/s per train step) on B200.

One step = fwd + Taylor jets + residual + loss + parameter gradient (+ NCCL
all-reduce of the flat gradient when N>1) + device Adam, over every
collocation point of the rank's shard. Default workload: C5 weak scaling --
BASELINE.json configs[4] (C4's Maxwell TE 6x256 model) with 1,048,576 points
per GPU (so N=1 is configs[3]'s 1M-point Maxwell set on one GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c1|c2|c3|c4]
  torchrun --nproc-per-node N bench.py --gpus N ...
  python bench.py --impl reference ...   # reference CPU implementation arm

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "collocation points/s per train step (residual+grad), 1/2/4/8 B200 vs CPU"
UNIT = "points/s"
L2_BYTES = 126e6  # B200 L2 (B200_PROFILING.md)
MMA_SYNC_TF32_TFLOPS = 278.7  # tools/mma_sync_probe.cu on this pool (profiles/round2/mma_sync_probe.txt)


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--points-per-gpu", type=int, default=1 << 20)
    ap.add_argument("--engine", default="auto", choices=["auto", "ffma", "tc3xtf32", "tc3xf16"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", dest="graph", action="store_true", default=None,
                    help="time CUDA-graph replays of the whole step (default on one GPU; class timings then come "
                         "from a separate eager pass). Multi-rank runs default to eager launches: capturing the "
                         "torch NCCL all-reduce in a graph is not exercised on this single-GPU pool")
    ap.add_argument("--no-graph", dest="graph", action="store_false", help="time eager launches")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="collective backend for N>1 (gloo: a host-side check of the N>1 path, e.g. 2 ranks on 1 GPU)")
    ap.add_argument("--host-points", action="store_true",
                    help="build the C5 interior on the host and upload it (default: device design)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def workload(args, world):
    from paper_2604_15645_b200 import configs
    if args.config == "c5":
        wl = configs.get_config("c4")
        dims = configs.weak_scaling_dims(args.points_per_gpu, world)
        name = f"c5_weak_maxwell_te_6x256_{args.points_per_gpu}pts_per_gpu"
    else:
        wl = configs.get_config(args.config)
        dims = wl.dims
        name = wl.name
    return wl, dims, name


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------

class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.out = tempfile.NamedTemporaryFile(prefix="clocks_", suffix=".csv", delete=False).name

    def _lines(self):
        try:
            return sum(1 for _ in open(self.out))
        except Exception:
            return 0

    def start(self):
        """Start sampling and wait (<= 3 s) for the first sample, so that even a
        short timed region is sampled; mark() then drops the pre-region lines."""
        self.skip = 0
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.out, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        t0 = time.time()
        while self._lines() == 0 and time.time() - t0 < 3.0:
            time.sleep(0.02)

    def mark(self):
        self.skip = self._lines()

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = open(self.out).readlines()
        # samples inside the timed region; if the region was shorter than one
        # sampling interval, the first sample after it (the GPU is still loaded)
        lines = lines[self.skip:] or lines[-1:]
        for line in lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference implementation on this host's cores
# ---------------------------------------------------------------------------

REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "pinnlab_ref_driver")


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _ref_train(wl, n_target, threads, epochs):
    """Run the compiled reference train() (trainer.cpp:332; cfg.workers std::threads,
    trainer.cpp:445-457) for `epochs` epochs on a uniform grid of about
    n_target points; returns (points, dims, per-epoch wall seconds)."""
    d = len(wl.domain)
    per = max(2, int(round(n_target ** (1.0 / d))))
    dims = [per] * d
    n = int(np.prod(dims))
    job = {"mode": "train", "model": _spec_json(wl.spec), "seed": 0,
           "pde": {"id": wl.res.id, "advection_c": wl.res.advection_c, "epsilon": wl.res.epsilon,
                   "mu": wl.res.mu},
           "domain": [list(b) for b in wl.domain], "initial": wl.initial, "bc": wl.bc,
           "collocation": {"mode": "uniform", "dims": dims, "n_ic": wl.n_ic, "n_bc": wl.n_bc},
           "workers": threads, "train": {"epochs": epochs, "lr": 1e-3, "balancing": False}}
    with tempfile.TemporaryDirectory() as td:
        job["out"] = td
        jp = os.path.join(td, "job.json")
        json.dump(job, open(jp, "w"))
        r = subprocess.run([REF_DRIVER, jp], capture_output=True, text=True, timeout=900)
        if r.returncode != 0:
            raise RuntimeError(r.stderr[-500:])
        m = json.load(open(os.path.join(td, "meta.json")))["metrics"]
    wall = [row[8] for row in m]
    return n, dims, np.diff([0.0] + wall)


def cpu_reference(wl, seconds: float, steps: int = 10, warmup: int = 2):
    """The reference CPU implementation of the path (oracle/_ref: the unmodified
    reference compiled against the Eigen-API shim) on this host's cores: `warmup`
    untimed + `steps` timed epochs of train() on a bounded sample of the workload
    (a uniform grid of the same model / PDE; the reference keeps every N x H
    float64 graph node, ~0.9 MB per point at 6x256, so the full 1M-point set does
    not fit). points/s = sample points / median timed epoch: the reference's cost
    is linear in the points, so the rate extrapolates to the full workload.
    Also one thread (W_cpu = 1) on a proportionally smaller sample."""
    if not os.path.exists(REF_DRIVER) or wl.res.id == "ns_steady":
        raise RuntimeError("oracle/_ref not built (or the workload is outside the reference)")
    cores = os.cpu_count() or 1
    threads = min(cores, 64)
    per_point_mb = 0.9 * (wl.spec.hidden_dim / 256.0) * (wl.spec.depth / 6.0) * (wl.streams() / 4.0)
    try:
        mem_mb = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_AVPHYS_PAGES") / 2**20
    except Exception:
        mem_mb = 32768
    # ~`seconds` of timed CPU work in total: one epoch ~ seconds/steps at ~250
    # points/s per thread (6x256), scaled by the model's cost
    rate = 250.0 * (7_901_184 / wl.flops_per_point())
    n = int(min(rate * threads * seconds / max(steps, 1), 0.4 * mem_mb / max(per_point_mb, 1e-3), 65536))
    n = max(n, threads * 16)
    npts, dims, dt = _ref_train(wl, n, threads, warmup + steps)
    timed = dt[warmup:]
    t = float(np.median(timed))
    n1 = max(64, n // threads)
    npts1, dims1, dt1 = _ref_train(wl, n1, 1, 3)  # W_cpu = 1: one warm-up + two timed epochs
    t1 = float(np.median(dt1[1:]))
    return {"value": npts / t, "unit": UNIT, "cores": threads, "kind": "reference",
            "cpu_model": cpu_model(), "host_cores": cores,
            "sample": (f"reference train() (oracle/_ref, Eigen-API shim), {threads} worker threads, "
                       f"uniform grid {dims} = {npts} points of the workload's model/PDE; "
                       f"{warmup} warm-up + {steps} timed epochs, median epoch {t:.3f} s; points/s = "
                       f"sample points / epoch time (the reference's cost is linear in the points, so "
                       f"this extrapolates to the full set)"),
            "epochs_timed": steps, "epochs_warmup": warmup, "sample_points": npts, "t_step_s": t,
            "w_cpu_1": {"value": npts1 / t1, "unit": UNIT, "cores": 1, "sample_points": npts1,
                        "epochs_timed": 2, "epochs_warmup": 1, "t_step_s": t1}}


def _spec_json(s):
    import dataclasses
    j = {"in_dim": s.in_dim, "hidden_dim": s.hidden_dim, "depth": s.depth, "out_dim": s.out_dim,
         "activation": s.activation, "sine_w0": s.sine_w0}
    if s.periodic_axes:
        j["periodic_axes"] = [dataclasses.asdict(a) for a in s.periodic_axes]
    if s.rff:
        j["rff"] = dataclasses.asdict(s.rff)
    if s.rwf:
        j["rwf"] = dataclasses.asdict(s.rwf)
    return j


def cpu_port(wl, seconds: float):
    """FP64 numpy restatement (oracle/pinn_oracle.py), one process."""
    from oracle import pinn_oracle as po
    from paper_2604_15645_b200 import configs
    spec = po.ModelSpec(wl.spec.in_dim, wl.spec.hidden_dim, wl.spec.depth, wl.spec.out_dim, wl.spec.activation)
    if wl.spec.rff:
        spec.rff = po.RFFSpec(wl.spec.rff.width, wl.spec.rff.sigma, wl.spec.rff.mean)
    if wl.spec.rwf:
        spec.rwf = po.RWFSpec(wl.spec.rwf.mean, wl.spec.rwf.stddev)
    res = po.ResidualSpec(wl.res.id, wl.res.advection_c, wl.res.epsilon, wl.res.mu, wl.res.reynolds)
    n = 4096
    d = len(wl.domain)
    per = max(2, int(round(n ** (1.0 / d))))
    dims = [per] * d
    col = configs.collocation(wl, dims)
    ocol = po.Collocation(col["interior"], col["ic_points"], col["ic_targets"], col["bc_a"], col["bc_b"],
                          col["bc_targets"])
    flat, rffB = po.init_params(spec, 0)
    t0 = time.perf_counter()
    k = 0
    while True:
        po.worker_step(spec, flat, rffB, res, ocol.interior, ocol, wl.bc)
        k += 1
        if time.perf_counter() - t0 > seconds / 3 or k >= 3:
            break
    t = (time.perf_counter() - t0) / k
    npts = int(np.prod(dims))
    return {"value": npts / t, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"numpy FP64 restatement, {npts} pts {dims}, mean of {k} steps", "t_step_s": t}


def cpu_baseline(wl, seconds, steps=10, warmup=2):
    try:
        return cpu_reference(wl, seconds, steps, warmup)
    except Exception:
        return cpu_port(wl, seconds)


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl, dims, name = workload(args, args.gpus)
    t0 = time.time()
    # the reference arm times `--steps` epochs after `--warmup` (at least 2) untimed ones
    warm = max(2, args.warmup)
    cb = cpu_baseline(wl, args.cpu_seconds, args.steps, warm)
    v = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": cb.get("epochs_timed", args.steps), "warmup": cb.get("epochs_warmup", warm),
            "ms_per_step": 1e3 * cb["t_step_s"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (uniform collocation grid; reference Model init)",
            "config": {"workload": name, "model": "reference pinnlab CPU train()",
                       "parallelism": f"{cb['cores']} std::threads (trainer.cpp:445-457)",
                       "sample_points": cb.get("sample_points"),
                       "points_per_s": "sample points / median epoch (cost linear in points: extrapolated)"},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample") if k in cb},
            "cpu_model": cb.get("cpu_model"), "host_cores": cb.get("host_cores"),
            "w_cpu_1": cb.get("w_cpu_1"),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.time() - t0}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def main():
    args = _args()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    import paper_2604_15645_b200 as pk
    from paper_2604_15645_b200 import configs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        world = max(world, 1)
    gpu = local % max(1, torch.cuda.device_count())  # one rank per GPU (gloo check: ranks may share one)
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    wl, dims, name = workload(args, world)
    # C5: the interior is the uniform grid generated on the device, each rank its
    # shard (pnx_sample_points; bit-exact sample_uniform) -- no host point set
    dev_pts = args.config == "c5" and not args.host_points
    col = configs.collocation(wl, dims, with_interior=not dev_pts)
    n_total = int(np.prod(dims))
    lo, hi = pk.shard_interior(n_total, world)[rank]
    flat, rffB = pk.init_params(wl.spec, seed=0)
    if dev_pts:
        worker = pk.Worker(wl.spec, wl.res, wl.bc, rffB, device=gpu, engine=args.engine)
        worker.sample_points("uniform", wl.domain, dims, rows=(lo, hi))
        if col["ic_points"] is not None and len(col["ic_points"]):
            worker.set_ic(col["ic_points"], col["ic_targets"])
        if wl.bc != "hard":
            worker.set_bc(col["bc_a"], col["bc_b"], col["bc_targets"])
        shard = None
    else:
        shard = col["interior"][lo:hi]
        worker = pk.make_worker(wl.spec, wl.res, wl.bc, rffB, shard, col["ic_points"], col["ic_targets"],
                                col["bc_a"], col["bc_b"], col["bc_targets"], device=gpu, engine=args.engine)
    P = worker.n_params
    from paper_2604_15645_b200.dist import DataParallelTrainer
    # one CUDA graph per step on a single GPU; multi-rank steps launch eagerly unless --graph
    # (at C5 a step is ~43 ms of device work, so ~60 launches hide behind it)
    use_graph = args.graph if args.graph is not None else world == 1
    trainer = DataParallelTrainer(worker, flat, world=world, lr=1e-3, device=dev, graph=use_graph)
    stream = torch.cuda.current_stream(dev)
    st = stream.cuda_stream
    lam = (1.0, 1.0, 1.0)

    def step(eager=False):  # device step -> NCCL all-reduce of the flat gradient -> fused Adam(1/W)
        trainer.step(lam, stream=st, eager=eager)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    worker.check()
    step(eager=True)
    torch.cuda.synchronize(dev)
    launches_per_step = worker.launch_count() + (2 if trainer.graph else 1)  # + Adam (+ its counter tick)

    if trainer.graph:  # per-class device time from an eager pass (graph replays carry no class events)
        worker.profile(True)
        for _ in range(args.steps):
            step(eager=True)
        torch.cuda.synchronize(dev)
        prof = worker.profile_read()
        worker.profile(False)

    # ---- timed region (device-resident inputs); class times by CUDA events on the
    # launching stream inside it unless graph replays are timed ----
    clk = ClockSampler(gpu)
    if not trainer.graph:
        worker.profile(True)
    clk.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk.mark()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # per-step device working set: Z and Zb of every hidden layer (multi-kernel
    # path), or just the coordinates and parameters (single-kernel step); a set
    # that fits in L2 is timed step by step with an L2 flush (a 512 MB write)
    # between steps, outside the per-step events
    work_bytes = ((hi - lo) * 8.0 * len(wl.domain) + P * 4.0) if worker.launch_count() < 8 else \
        (hi - lo) * wl.streams() * 4.0 * wl.spec.hidden_dim * wl.spec.depth * 2
    l2_flush = work_bytes < 2 * L2_BYTES
    if l2_flush:
        scrub = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for a, b in ev:
            scrub.fill_(1)
            a.record(stream)
            step()
            b.record(stream)
    else:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    if not trainer.graph:
        prof = worker.profile_read()
        worker.profile(False)
    worker.check()
    replicas_equal = None
    if world > 1:  # replica consistency after the synchronized steps (param_hash / on_sync, trainer.cpp:540-544)
        from paper_2604_15645_b200.dist import replica_hashes
        hs = replica_hashes(wl.spec, trainer.params_host(), world)
        replicas_equal = len(set(hs)) == 1
    ms = sum(a.elapsed_time(b) for a, b in ev) if l2_flush else e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = n_total / (ms_step / 1e3)

    # ---- e2e: reference-facing C-ABI call with host buffers ----
    e2e = None
    if not args.no_e2e:
        host_params = flat.copy()
        opt_m = np.zeros_like(host_params)
        opt_v = np.zeros_like(host_params)
        import ctypes
        hlib = ctypes.CDLL(os.path.join(ROOT, "host", "libpinnlab_b200.so"))  # built by build(); no fallback
        hadam = hlib.pinnlab_adam_step
        dptr = ctypes.POINTER(ctypes.c_double)
        hadam.argtypes = [dptr, dptr, dptr, dptr, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                          ctypes.c_double, ctypes.c_double, ctypes.c_int64]
        hadam.restype = ctypes.c_int

        def pp(a):
            return a.ctypes.data_as(dptr)
        if shard is None:  # the host copy of this rank's grid rows, for the host->device leg
            shard = configs.grid(wl.domain, dims)[lo:hi]
        shard_pinned = torch.from_numpy(np.ascontiguousarray(shard.T)).pin_memory()  # axis-major [d, N]
        g_dev = torch.zeros(P, dtype=torch.float64, device=dev)
        h2d = d2h = 0

        g_buf = np.empty(P, dtype=np.float64)
        pts = shard_pinned.numpy()
        ptr_p, ptr_m, ptr_v, ptr_g = pp(host_params), pp(opt_m), pp(opt_v), pp(g_buf)  # updated in place

        def e2e_step(k):
            nonlocal h2d, d2h
            worker.set_points(pts, axis_major=True)          # H2D of this step's collocation batch
            _, l = worker.step(host_params, lam, out=g_buf)  # H2D params, D2H grad + losses
            if world > 1:
                g_dev.copy_(torch.from_numpy(g_buf))
                dist.all_reduce(g_dev, op=dist.ReduceOp.SUM)
                g_buf[:] = g_dev.cpu().numpy() / world
            # host Adam in place (optim.cpp:7-41), the C++ host mirror's fused loop
            hadam(ptr_p, ptr_m, ptr_v, ptr_g, P, 1e-3, 0.9, 0.999, 1e-8, k)
            h2d = pts.nbytes + P * 4
            d2h = P * 4 + 3 * 8

        for k in range(1, 3):
            e2e_step(k)
        if world > 1:
            dist.barrier()
        ke = max(3, args.steps // 2)
        t0 = time.perf_counter()
        for k in range(3, 3 + ke):
            e2e_step(k)
        te = torch.tensor([(time.perf_counter() - t0) / ke], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": n_total / float(te.item()), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * float(te.item()),
               "path": "pnx_set_points + pnx_step (float64 host buffers) + host Adam (host/ C++ pinnlab_adam_step)"}

    if rank == 0:
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        # roofline of the dominant kernel class (CUDA events on the launching stream).
        # Algorithmic work per step of each class:
        #   flops  2*S*rows*sum K*N over its layers
        #   bytes  per row and hidden layer: fwd S*4*(K+N) (read act input, write out),
        #          bwd S*4*(N+2K) (read Zb_out and Z_in, write Zb_in), wgrad S*4*(K+N);
        #          layer 0 (fused): fwd 8*d + S*4*N0, wgrad S*4*N0
        # The bound is whichever takes longer at peak; the other view is kept beside it.
        S = wl.streams()
        H = wl.spec.hidden_dim
        rows = hi - lo
        K0 = wl.spec.first_layer_width()
        d_in = wl.spec.in_dim
        nh = wl.spec.depth - 1                               # hidden->hidden layers
        sum_fwd = K0 * H + H * H * nh                        # layers 0..depth-1 (head excluded)
        sum_bwd = H * H * nh                                 # reverse GEMMs of layers 1..depth-1
        # the single-kernel narrow step (width <= 64) does all of it: F_pt flops per
        # row, and its only HBM traffic is the coordinates (8 B per axis)
        flops_cls = {"fwd_gemm": 2.0 * S * rows * sum_fwd, "bwd_gemm": 2.0 * S * rows * sum_bwd,
                     "wgrad_gemm": 2.0 * S * rows * sum_fwd, "fused_step": float(wl.flops_per_point()) * rows}
        bytes_cls = {"fwd_gemm": rows * (S * 4.0 * 2 * H * nh + S * 4.0 * H + 8.0 * d_in),
                     "bwd_gemm": rows * S * 4.0 * 3 * H * nh,
                     "wgrad_gemm": rows * (S * 4.0 * 2 * H * nh + S * 4.0 * H),
                     "fused_step": rows * 8.0 * d_in}
        dom = max(flops_cls, key=lambda k: prof[k][0])
        tms, nl = prof[dom]
        t_s = (tms / 1e3) / args.steps                       # class seconds per step
        achieved = flops_cls[dom] / t_s / 1e12
        achieved_gbs = bytes_cls[dom] / t_s / 1e9
        use_tc = args.engine != "ffma" and H in (128, 256) and wl.spec.activation == "tanh"
        bf16 = float(peaks.get("bf16_tflops_sustained", 1366.2))
        hbm = float(peaks.get("hbm_gbs", 6546.2))
        fp32_peak = 148 * 128 * 2 * (peaks.get("sm_max_mhz", 1965.0) * 1e6) / 1e12
        # the 3xFP16 kernels run where the CTA-pair paths apply (H = 256); "auto" picks them
        use_f16 = use_tc and args.engine != "tc3xtf32" and H == 256
        if use_f16:
            eff, note = bf16 / 3.0, ("3xFP16: tensor-pipe work = 3 x algorithmic flops at the fp16 rate "
                                     "(= bf16), so the FP32-accurate peak = bf16/3 (derived)")
        elif use_tc:
            eff, note = bf16 / 6.0, ("3xTF32: tensor-pipe work = 3 x algorithmic flops at the TF32 rate "
                                     "(= bf16/2), so FP32-accurate peak = bf16/6 (derived)")
        elif dom == "fused_step" and H == 64:
            # the single-kernel step's width-64 contractions are 3xTF32 warp MMAs: the
            # FP32-accurate peak is a third of the measured mma.sync tf32 rate
            # (profiles/round2/mma_sync_probe.txt), above the FFMA pipe
            eff, note = max(MMA_SYNC_TF32_TFLOPS / 3.0, fp32_peak), (
                "3xTF32 mma.sync: measured m16n8k8 tf32 rate 278.7 TF/s / 3 (profiles/round2/mma_sync_probe.txt)")
        else:
            eff, note = fp32_peak, "FP32 FFMA pipe: 148 SM x 128 lanes x 2 x sm_max_mhz (derived)"
        simt = not use_tc
        tensor_view = {"achieved": achieved, "unit": "TFLOP/s",
                       "peak": bf16 if use_tc else eff, "frac": achieved / (bf16 if use_tc else eff),
                       "peak_source": ("MEASURED_PEAKS.json bf16_tflops_sustained (dense bf16, of measured)"
                                       if not simt else note),
                       "effective_peak": eff, "frac_effective": achieved / eff, "effective_note": note,
                       "flops_per_step": flops_cls[dom]}
        hbm_view = {"achieved": achieved_gbs, "unit": "GB/s", "peak": hbm, "frac": achieved_gbs / hbm,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy read+write, measured)",
                    "bytes_per_step": bytes_cls[dom]}
        hbm_bound = bytes_cls[dom] / (hbm * 1e9) > flops_cls[dom] / (eff * 1e12)
        main, other = (hbm_view, tensor_view) if hbm_bound else (tensor_view, hbm_view)
        roof = {"bound": "hbm" if hbm_bound else "tensor", "kernel": dom, **main,
                "other_view": other,
                "t_min_ms": {"hbm": 1e3 * bytes_cls[dom] / (hbm * 1e9),
                             "tensor_effective": 1e3 * flops_cls[dom] / (eff * 1e12),
                             "measured": 1e3 * t_s}}
        traffic_db = {}
        try:
            traffic_db = json.load(open(os.path.join(ROOT, "profiles", "kernel_traffic.json")))
        except Exception:
            pass
        key = f"{name}:{dom}"
        roof["traffic"] = traffic_db.get(key)
        # one hidden-layer launch's algorithmic bytes, the comparand of `traffic`
        roof["algorithmic_bytes_per_launch"] = (bytes_cls[dom] if dom == "fused_step" else
                                                rows * S * 4.0 * H * (3 if dom == "bwd_gemm" else 2))
        roof["launches_per_step"] = nl / args.steps
        step_flops = wl.flops_per_point() * n_total
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak"
            if args.config == "c5" else "strong", "vs_baseline": None, "dtype": "f32",
            "data": ("synthetic (uniform collocation grid generated on the device, numpy Xavier init; no dataset)"
                     if dev_pts else "synthetic (uniform collocation grid, numpy Xavier init; no dataset)"),
            "config": {"workload": name, "pde": wl.res.id, "model": f"tanh MLP {wl.spec.depth}x{H}",
                       "points_total": n_total, "points_per_gpu": rows, "streams": S,
                       "params": P, "engine": args.engine,
                       "contraction": ("3xFP16 split operands, FP32 accumulate" if use_f16 else
                                       "3xTF32 split operands, FP32 accumulate" if use_tc else
                                       ("3xTF32 warp MMA (mma.sync), whole step in one kernel" if H == 64 else
                                        "FP32 FFMA, whole step in one kernel") if dom == "fused_step" else "FP32 FFMA"),
                       "parallelism": f"dp{world}",
                       "l2": (f"working set {work_bytes / 1e6:.1f} MB fits in L2: each timed step preceded by a "
                              f"512 MB L2 flush outside its CUDA events (steps timed one by one)" if l2_flush else
                              f"inputs larger than L2 (per-step activations {work_bytes / 1e9:.2f} GB >> 126 MB)"),
                       "cuda_graph": bool(trainer.graph)},
            "tflops_step": step_flops / (ms_step / 1e3) / 1e12,
            "roofline": roof,
            "kernel_ms_per_step": {k: prof[k][0] / args.steps for k in prof},
            "gpu_launches": int(launches_per_step * args.steps),
            "replica_hashes_equal": replicas_equal,
            "clocks": clocks,
            "e2e": e2e,
        }
        if not args.no_cpu_baseline and world == 1:
            cb = cpu_baseline(wl, args.cpu_seconds, 5, 2)
            line["cpu_baseline"] = {k: v for k, v in cb.items() if k not in ("t_step_s",)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

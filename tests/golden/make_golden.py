"""Generate tests/golden/*.npz from the compiled reference (oracle/_ref).

Runs ``oracle/_ref/pinnlab_ref_driver`` -- the unmodified reference sources of
/root/reference/proj/core compiled by oracle/Makefile -- on small cases that
cover every model feature and residual on the hot path, and stores its float64
inputs and outputs. Rerun with ``python tests/golden/make_golden.py`` in the
build container (the GPU box has no /root/reference; the fixtures travel).
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "pinnlab_ref_driver")

BURGERS = {"pde": {"id": "burgers"}, "domain": [[0, 2], [0, 1]], "initial": "sin_pi_x"}
MAXWELL = {"pde": {"id": "maxwell_te", "epsilon": 1.0, "mu": 1.0},
           "domain": [[-1, 1], [-1, 1], [0, 1.5]], "initial": "gauss25"}

CASES = {
    # C1 family: plain tanh MLP, Dirichlet BC
    "burgers_tanh": dict(BURGERS, bc="dirichlet_zero",
                         model={"in_dim": 2, "hidden_dim": 16, "depth": 2, "out_dim": 1, "activation": "tanh"},
                         collocation={"mode": "uniform", "dims": [12, 10], "n_ic": 16, "n_bc": 8},
                         workers=[1, 2, 3]),
    # C1 shape at full width (4x64) on a small grid
    "burgers_c1_shape": dict(BURGERS, bc="dirichlet_zero",
                             model={"in_dim": 2, "hidden_dim": 64, "depth": 4, "out_dim": 1, "activation": "tanh"},
                             collocation={"mode": "uniform", "dims": [16, 16], "n_ic": 32, "n_bc": 16},
                             workers=[1, 4]),
    # C1 exactly as BASELINE configs[0] runs it: 4x64 on the full 100 x 100 grid
    "burgers_c1_full": dict(BURGERS, bc="dirichlet_zero",
                            model={"in_dim": 2, "hidden_dim": 64, "depth": 4, "out_dim": 1, "activation": "tanh"},
                            collocation={"mode": "uniform", "dims": [100, 100], "n_ic": 128, "n_bc": 64},
                            workers=[1, 4]),
    # C4/C5 model at full width (Maxwell TE, tanh 6x256) on a small grid: the
    # width-256 tensor-core kernels against the reference itself
    "maxwell_c4_shape": dict(MAXWELL, bc="hard",
                             model={"in_dim": 3, "hidden_dim": 256, "depth": 6, "out_dim": 3, "activation": "tanh"},
                             collocation={"mode": "uniform", "dims": [8, 6, 5], "n_ic": 16},
                             workers=[1, 2]),
    # C2 at full width: RFF (128 features, sigma 10) + RWF, tanh 4x128, small grid
    "burgers_c2_shape": dict(BURGERS, bc="dirichlet_zero",
                             model={"in_dim": 2, "hidden_dim": 128, "depth": 4, "out_dim": 1, "activation": "tanh",
                                    "rff": {"width": 128, "sigma": 10.0, "mean": 0.0},
                                    "rwf": {"mean": 1.0, "stddev": 0.1}},
                             collocation={"mode": "uniform", "dims": [16, 12], "n_ic": 32, "n_bc": 16},
                             workers=[1, 2]),
    # C2 family: RFF + RWF
    "burgers_rff_rwf": dict(BURGERS, bc="dirichlet_zero",
                            model={"in_dim": 2, "hidden_dim": 16, "depth": 2, "out_dim": 1, "activation": "tanh",
                                   "rff": {"width": 8, "sigma": 10.0, "mean": 0.0},
                                   "rwf": {"mean": 1.0, "stddev": 0.1}},
                            collocation={"mode": "uniform", "dims": [10, 8], "n_ic": 16, "n_bc": 8},
                            workers=[1, 2]),
    # C4 family: Maxwell TE, hard BC
    "maxwell_tanh": dict(MAXWELL, bc="hard",
                         model={"in_dim": 3, "hidden_dim": 16, "depth": 3, "out_dim": 3, "activation": "tanh"},
                         collocation={"mode": "uniform", "dims": [5, 5, 4], "n_ic": 16},
                         workers=[1, 2]),
    # Maxwell with strict spatial periodicity and a trainable time period + RFF
    "maxwell_periodic_rff": dict(MAXWELL, bc="hard",
                                 model={"in_dim": 3, "hidden_dim": 12, "depth": 2, "out_dim": 3, "activation": "tanh",
                                        "periodic_axes": [{"periodic": True, "period": 2.0, "trainable": False},
                                                          {"periodic": True, "period": 2.0, "trainable": False},
                                                          {"periodic": True, "period": 1.5, "trainable": True}],
                                        "rff": {"width": 6, "sigma": 1.0, "mean": 0.0}},
                                 collocation={"mode": "uniform", "dims": [4, 4, 3], "n_ic": 9},
                                 workers=[1]),
    # second-order stream, sine activation, soft periodic BC
    "allen_cahn_sine": dict(pde={"id": "allen_cahn"}, domain=[[-1, 1], [0, 1]], initial="sin_pi_x",
                            bc="soft_periodic",
                            model={"in_dim": 2, "hidden_dim": 12, "depth": 2, "out_dim": 1, "activation": "sine",
                                   "sine_w0": 2.0},
                            collocation={"mode": "uniform", "dims": [8, 6], "n_ic": 10, "n_bc": 6},
                            workers=[1, 2]),
    # swish activation, advection, periodic x with trainable period
    "advection_swish_periodic": dict(pde={"id": "advection", "advection_c": 3.0}, domain=[[0, 6.283185307179586], [0, 1]],
                                     initial="sin_x", bc="soft_periodic",
                                     model={"in_dim": 2, "hidden_dim": 10, "depth": 2, "out_dim": 1,
                                            "activation": "swish",
                                            "periodic_axes": [{"periodic": True, "period": 6.283185307179586,
                                                               "trainable": True},
                                                              {"periodic": False, "period": 0.0, "trainable": False}]},
                                     collocation={"mode": "uniform", "dims": [7, 5], "n_ic": 8, "n_bc": 5},
                                     workers=[1]),
    # Allen-Cahn second order with tanh (tanh second-order jet rule)
    "allen_cahn_tanh": dict(pde={"id": "allen_cahn"}, domain=[[-1, 1], [0, 1]], initial="sin_pi_x",
                            bc="dirichlet_zero",
                            model={"in_dim": 2, "hidden_dim": 16, "depth": 3, "out_dim": 1, "activation": "tanh"},
                            collocation={"mode": "uniform", "dims": [9, 7], "n_ic": 10, "n_bc": 6},
                            workers=[1]),
    # Latin hypercube interiors (sampling.cpp:55-103) with the reference's mt19937_64 stream
    "burgers_lhs": dict(BURGERS, bc="dirichlet_zero", colloc_seed=5,
                        model={"in_dim": 2, "hidden_dim": 16, "depth": 2, "out_dim": 1, "activation": "tanh"},
                        collocation={"mode": "lhs", "n": 97, "n_ic": 16, "n_bc": 8},
                        workers=[1, 2]),
    "maxwell_lhs_per_axis": dict(MAXWELL, bc="hard", colloc_seed=11,
                                 model={"in_dim": 3, "hidden_dim": 12, "depth": 2, "out_dim": 3,
                                        "activation": "tanh"},
                                 collocation={"mode": "lhs_per_axis", "dims": [5, 4, 3], "n_ic": 16},
                                 workers=[1]),
    # Maxwell with the Poynting energy penalty (losses.cpp:187-223, trainer.cpp:240-247)
    "maxwell_poynting": dict(MAXWELL, bc="hard",
                             model={"in_dim": 3, "hidden_dim": 16, "depth": 2, "out_dim": 3, "activation": "tanh"},
                             collocation={"mode": "uniform", "dims": [5, 5, 4], "n_ic": 16},
                             poynting={"weight": 0.7, "grid": 5, "time_samples": 3},
                             workers=[1, 2]),
}

TRAJ = {
    # N-step Adam trajectory (balancing off), W=2 workers
    "traj_burgers": dict(BURGERS, bc="dirichlet_zero",
                         model={"in_dim": 2, "hidden_dim": 16, "depth": 2, "out_dim": 1, "activation": "tanh"},
                         collocation={"mode": "uniform", "dims": [12, 10], "n_ic": 16, "n_bc": 8},
                         workers=2, train={"epochs": 30, "lr": 1e-2, "gamma": 0.99, "balancing": False}),
    "traj_maxwell": dict(MAXWELL, bc="hard",
                         model={"in_dim": 3, "hidden_dim": 16, "depth": 2, "out_dim": 3, "activation": "tanh"},
                         collocation={"mode": "uniform", "dims": [5, 5, 4], "n_ic": 16},
                         workers=1, train={"epochs": 20, "lr": 5e-3, "gamma": 1.0, "balancing": False}),
    # temporal causality weights (trainer.cpp:209-220, losses.cpp:163-185), W=2
    "traj_burgers_causality": dict(BURGERS, bc="dirichlet_zero",
                                   model={"in_dim": 2, "hidden_dim": 16, "depth": 2, "out_dim": 1,
                                          "activation": "tanh"},
                                   collocation={"mode": "uniform", "dims": [12, 10], "n_ic": 16, "n_bc": 8},
                                   causality={"enabled": True, "segments": 4, "epsilon": 2.0},
                                   workers=2, train={"epochs": 12, "lr": 1e-2, "gamma": 1.0, "balancing": False}),
    # loss balancing: per-term gradients every update_period epochs (trainer.cpp:462-506)
    "traj_burgers_balancing": dict(BURGERS, bc="dirichlet_zero",
                                   model={"in_dim": 2, "hidden_dim": 16, "depth": 2, "out_dim": 1,
                                          "activation": "tanh"},
                                   collocation={"mode": "uniform", "dims": [12, 10], "n_ic": 16, "n_bc": 8},
                                   workers=2, train={"epochs": 12, "lr": 1e-2, "gamma": 1.0, "balancing": True,
                                                     "update_period": 3, "alpha": 0.9}),
    # LHS interior resampled every 3 epochs with seed + epoch (trainer.cpp:421-434)
    "traj_burgers_lhs_resample": dict(BURGERS, bc="dirichlet_zero", colloc_seed=3,
                                      model={"in_dim": 2, "hidden_dim": 16, "depth": 2, "out_dim": 1,
                                             "activation": "tanh"},
                                      collocation={"mode": "lhs", "n": 120, "n_ic": 16, "n_bc": 8,
                                                   "resample_every": 3},
                                      workers=2, train={"epochs": 9, "lr": 1e-2, "gamma": 1.0, "balancing": False}),
    # Adam -> L-BFGS switch at an epoch threshold, then full-batch strong-Wolfe
    # L-BFGS over the whole interior (trainer.cpp:549-617, lbfgs.cpp)
    "traj_burgers_lbfgs": dict(BURGERS, bc="dirichlet_zero",
                               model={"in_dim": 2, "hidden_dim": 16, "depth": 2, "out_dim": 1,
                                      "activation": "tanh"},
                               collocation={"mode": "uniform", "dims": [12, 10], "n_ic": 16, "n_bc": 8},
                               workers=2, train={"epochs": 40, "lr": 1e-2, "gamma": 1.0, "balancing": False,
                                                 "switch": {"trigger": "epoch", "epoch_threshold": 5},
                                                 "lbfgs_max_iters": 6, "lbfgs": {"history": 5}}),
    # the full Maxwell objective: causality + Poynting + two-term balancing (hard BC)
    "traj_maxwell_full": dict(MAXWELL, bc="hard",
                              model={"in_dim": 3, "hidden_dim": 16, "depth": 2, "out_dim": 3, "activation": "tanh"},
                              collocation={"mode": "uniform", "dims": [5, 5, 4], "n_ic": 16},
                              causality={"enabled": True, "segments": 3, "epsilon": 1.0},
                              poynting={"weight": 0.5, "grid": 4, "time_samples": 3},
                              workers=2, train={"epochs": 8, "lr": 5e-3, "gamma": 1.0, "balancing": True,
                                                "update_period": 2, "alpha": 0.9}),
}


def _run(job: dict) -> tuple[dict, str]:
    d = tempfile.mkdtemp(prefix="golden_")
    job = dict(job, out=d)
    with open(os.path.join(d, "job.json"), "w") as f:
        json.dump(job, f)
    subprocess.run([DRIVER, os.path.join(d, "job.json")], check=True)
    with open(os.path.join(d, "meta.json")) as f:
        return json.load(f), d


def _f64(d, name):
    p = os.path.join(d, name)
    return np.fromfile(p, dtype="<f8") if os.path.exists(p) else np.zeros(0)


def _points(v, d):
    return v.reshape(d, -1).T.copy() if v.size else np.zeros((0, d))


def make_case(name, case):
    base = {k: v for k, v in case.items() if k not in ("workers",)}
    dim = len(case["domain"])
    fields = case["model"]["out_dim"]
    arrays = {}
    grads = {}
    losses = {}
    for w in case["workers"]:
        meta, d = _run(dict(base, mode="step", workers=w, dump_residuals=(w == case["workers"][0])))
        grads[w] = _f64(d, "grad.bin")
        losses[w] = meta["worker_losses"]
        if w == case["workers"][0]:
            arrays.update(
                params=_f64(d, "params.bin"), rffB=_f64(d, "rff_B.bin"),
                interior=_points(_f64(d, "interior.bin"), dim),
                ic_points=_points(_f64(d, "ic_points.bin"), dim),
                ic_targets=_f64(d, "ic_targets.bin").reshape(fields, -1).T.copy(),
                bc_a=_points(_f64(d, "bc_a.bin"), dim), bc_b=_points(_f64(d, "bc_b.bin"), dim),
                residuals=_f64(d, "residuals.bin").reshape(-1, meta["n_interior"]),
                outputs=_f64(d, "outputs.bin").reshape(meta["n_interior"], fields),
            )
            if meta["rff_shape"]:
                arrays["rffB"] = arrays["rffB"].reshape(meta["rff_shape"])
            param_meta = meta["params"]
    for w in case["workers"]:
        arrays[f"grad_w{w}"] = grads[w]
    case_meta = {"case": base, "workers": case["workers"], "worker_losses": {str(w): losses[w] for w in losses},
                 "params": param_meta}
    if "penalty" in meta:
        case_meta["penalty"] = meta["penalty"]
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), meta=json.dumps(case_meta), **arrays)


def make_traj(name, case):
    meta, d = _run(dict(case, mode="train"))
    fields = case["model"]["out_dim"]
    dim = len(case["domain"])
    m = np.array([row[:8] for row in meta["metrics"]], dtype=np.float64)
    case_meta = {"case": case, "hashes": meta["hashes"], "aborted": meta["aborted"],
                 "switched_to_lbfgs": meta.get("switched_to_lbfgs", False)}
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), meta=json.dumps(case_meta),
                        params=_f64(d, "params.bin"), final_params=_f64(d, "final_params.bin"),
                        metrics=m, rffB=_f64(d, "rff_B.bin"),
                        interior=_points(_f64(d, "interior.bin"), dim),
                        ic_points=_points(_f64(d, "ic_points.bin"), dim),
                        ic_targets=_f64(d, "ic_targets.bin").reshape(fields, -1).T.copy(),
                        bc_a=_points(_f64(d, "bc_a.bin"), dim), bc_b=_points(_f64(d, "bc_b.bin"), dim))


CKPT = {
    # train() writes final.ckpt (PLABCK01, checkpoint.cpp:121-140) after 8 epochs;
    # a second run resumes from it (trainer.cpp:345-353) for 6 more epochs
    "ckpt_burgers": dict(BURGERS, bc="dirichlet_zero",
                         model={"in_dim": 2, "hidden_dim": 16, "depth": 2, "out_dim": 1, "activation": "tanh"},
                         collocation={"mode": "uniform", "dims": [12, 10], "n_ic": 16, "n_bc": 8},
                         workers=2, train={"epochs": 8, "lr": 1e-2, "gamma": 0.98, "balancing": True,
                                           "update_period": 3, "alpha": 0.9}),
}


def make_ckpt(name, case):
    run = tempfile.mkdtemp(prefix="ckpt_")
    meta, d = _run(dict(case, mode="train", train=dict(case["train"], run_dir=run)))
    ck = os.path.join(run, "final.ckpt")
    raw = np.fromfile(ck, dtype=np.uint8)
    info, di = _run(dict(case, mode="ckpt_info", ckpt=ck))
    t2 = dict(case["train"], epochs=case["train"]["epochs"] + 6, resume_from=ck)
    meta2, d2 = _run(dict(case, mode="train", train=t2))
    m2 = np.array([row[:8] for row in meta2["metrics"]], dtype=np.float64)
    case_meta = {"case": case, "ckpt_tensors": info["ckpt_tensors"], "ckpt_scalars": info["ckpt_scalars"]}
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), meta=json.dumps(case_meta), ckpt=raw,
                        params=_f64(d, "params.bin"), final_params=_f64(d, "final_params.bin"),
                        ckpt_data=_f64(di, "ckpt_data.bin"), resume_metrics=m2,
                        resume_final_params=_f64(d2, "final_params.bin"), rffB=_f64(d, "rff_B.bin"),
                        interior=_points(_f64(d, "interior.bin"), 2),
                        ic_points=_points(_f64(d, "ic_points.bin"), 2),
                        ic_targets=_f64(d, "ic_targets.bin").reshape(1, -1).T.copy(),
                        bc_a=_points(_f64(d, "bc_a.bin"), 2), bc_b=_points(_f64(d, "bc_b.bin"), 2))


def main():
    if not os.path.exists(DRIVER):
        sys.exit(f"{DRIVER} missing: run `make -C oracle` (needs /root/reference)")
    only = set(sys.argv[1:])  # optional: names to (re)generate
    for n, c in CASES.items():
        if only and n not in only:
            continue
        make_case(n, c)
        print("wrote", n)
    for n, c in TRAJ.items():
        if only and n not in only:
            continue
        make_traj(n, c)
        print("wrote", n)
    for n, c in CKPT.items():
        if only and n not in only:
            continue
        make_ckpt(n, c)
        print("wrote", n)


if __name__ == "__main__":
    main()

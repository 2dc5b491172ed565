"""PLABCK01 checkpoints, byte-compatible with the reference (checkpoint.cpp).

Layout: 8-byte magic "PLABCK01", u64 little-endian header length, a JSON header
{"model": ModelSpec, "seed": u64, "tensors": [{"name", "shape"}], "scalars": {}},
then each tensor's float64 little-endian payload in header order
(Checkpoint::save / load, checkpoint.cpp:121-170). train() stores the
trainable tensors, rff.B, Adam's moments as "adam.m.<name>" / "adam.v.<name>"
(optim.cpp:43-50) and the scalars epoch, adam_t, lambda_pde/ic/bc
(trainer.cpp:378-389); resuming restarts at epoch + 1 (trainer.cpp:345-353).
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from .pinn import AxisPeriodic, ModelSpec, RFFSpec, RWFSpec, TensorError, param_layout

MAGIC = b"PLABCK01"

__all__ = ["Checkpoint", "spec_to_json", "trainer_checkpoint", "restore_trainer"]


def spec_to_json(s: ModelSpec) -> dict:
    """spec_json (checkpoint.cpp:55-77)."""
    j = {"in_dim": s.in_dim, "hidden_dim": s.hidden_dim, "depth": s.depth, "out_dim": s.out_dim,
         "activation": s.activation, "sine_w0": s.sine_w0}
    if s.periodic_axes:
        j["periodic_axes"] = [{"periodic": a.periodic, "period": a.period, "trainable": a.trainable}
                              for a in s.periodic_axes]
    if s.rff:
        j["rff"] = {"width": s.rff.width, "sigma": s.rff.sigma, "mean": s.rff.mean}
    if s.rwf:
        j["rwf"] = {"mean": s.rwf.mean, "stddev": s.rwf.stddev}
    return j


@dataclass
class Checkpoint:
    spec: ModelSpec
    seed: int = 0
    tensors: List[Tuple[str, np.ndarray]] = field(default_factory=list)
    scalars: Dict[str, float] = field(default_factory=dict)

    def find(self, name: str) -> Optional[np.ndarray]:
        for n, t in self.tensors:
            if n == name:
                return t
        return None

    def save(self, path: str) -> None:
        header = {"model": spec_to_json(self.spec), "seed": int(self.seed),
                  "tensors": [{"name": n, "shape": list(np.shape(t))} for n, t in self.tensors],
                  "scalars": {k: float(v) for k, v in self.scalars.items()}}
        text = json.dumps(header, separators=(",", ":"), sort_keys=True).encode()
        try:
            with open(path, "wb") as f:
                f.write(MAGIC)
                f.write(struct.pack("<Q", len(text)))
                f.write(text)
                for _, t in self.tensors:
                    f.write(np.ascontiguousarray(t, dtype="<f8").tobytes())
        except OSError as e:
            raise TensorError(f"checkpoint: cannot open for writing: {path}") from e

    @staticmethod
    def load(path: str) -> "Checkpoint":
        try:
            with open(path, "rb") as f:
                raw = f.read()
        except OSError as e:
            raise TensorError(f"checkpoint: cannot open: {path}") from e
        if raw[:8] != MAGIC:
            raise TensorError(f"checkpoint: bad magic in {path}")
        (hlen,) = struct.unpack("<Q", raw[8:16])
        header = json.loads(raw[16:16 + hlen].decode())
        at = 16 + hlen
        ck = Checkpoint(ModelSpec.from_json(header["model"]), int(header.get("seed", 0)),
                        scalars={k: float(v) for k, v in header.get("scalars", {}).items()})
        for d in header["tensors"]:
            shape = tuple(int(x) for x in d["shape"])
            n = int(np.prod(shape)) if shape else 1
            if at + 8 * n > len(raw):
                raise TensorError(f"checkpoint: truncated payload in {path}")
            ck.tensors.append((d["name"], np.frombuffer(raw, dtype="<f8", count=n, offset=at).reshape(shape).copy()))
            at += 8 * n
        return ck


def _split(spec: ModelSpec, flat: np.ndarray, prefix: str = ""):
    out, at = [], 0
    for name, shape in param_layout(spec):
        n = int(np.prod(shape)) if shape else 1
        out.append((prefix + name, np.asarray(flat[at:at + n], dtype=np.float64).reshape(shape)))
        at += n
    return out


def trainer_checkpoint(trainer, spec: ModelSpec, seed: int = 0, rff_B=None) -> Checkpoint:
    """Checkpoint of a dist.DataParallelTrainer after its last completed epoch
    (the save_checkpoint lambda of train(), trainer.cpp:378-389)."""
    p = trainer.params.double().cpu().numpy()
    m = trainer.m.double().cpu().numpy()
    v = trainer.v.double().cpu().numpy()
    ck = Checkpoint(spec, seed)
    ck.tensors = _split(spec, p)
    if spec.rff:
        ck.tensors.append(("rff.B", np.asarray(rff_B, dtype=np.float64)))
    for (nm, tm), (_, tv) in zip(_split(spec, m), _split(spec, v)):
        ck.tensors.append(("adam.m." + nm, tm))
        ck.tensors.append(("adam.v." + nm, tv))
    ck.scalars = {"epoch": float(trainer.epoch - 1), "adam_t": float(trainer.t),
                  "lambda_pde": trainer.lam[0], "lambda_ic": trainer.lam[1], "lambda_bc": trainer.lam[2]}
    return ck


def restore_trainer(trainer, ck: Checkpoint, spec: ModelSpec) -> None:
    """Resume (trainer.cpp:345-353): parameters, Adam moments and step count,
    loss weights; the next epoch is the stored epoch + 1."""
    import torch
    flat, mom, vel = [], [], []
    for name, shape in param_layout(spec):
        t = ck.find(name)
        if t is None:
            raise TensorError(f"checkpoint: missing tensor {name}")
        if tuple(np.shape(t)) != tuple(shape):
            raise TensorError(f"checkpoint: shape mismatch for {name}")
        m, v = ck.find("adam.m." + name), ck.find("adam.v." + name)
        if m is None or v is None:
            raise TensorError(f"adam: missing moment tensors for {name}")
        flat.append(np.ravel(t))
        mom.append(np.ravel(m))
        vel.append(np.ravel(v))
    dev = trainer.params.device
    trainer.params.copy_(torch.tensor(np.concatenate(flat), dtype=torch.float32, device=dev))
    trainer.m.copy_(torch.tensor(np.concatenate(mom), dtype=torch.float32, device=dev))
    trainer.v.copy_(torch.tensor(np.concatenate(vel), dtype=torch.float32, device=dev))
    trainer.t = int(ck.scalars["adam_t"])
    trainer.epoch = int(ck.scalars["epoch"]) + 1
    trainer.lam = [ck.scalars["lambda_pde"], ck.scalars["lambda_ic"], ck.scalars["lambda_bc"]]
    trainer.state.copy_(torch.tensor([float(trainer.t), float(trainer.epoch)], dtype=torch.float64, device=dev))
    trainer._graph = None  # a captured step holds the old constants

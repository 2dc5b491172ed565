"""B200-native PINN train-step hot path (PINNACLE / pinnlab drop-in).

Compute lives in libpnx.so (hand-written sm_100a CUDA behind the C ABI in
include/pnx.h); this package is the host-side mirror of the reference
interface. See DESIGN.md."""
from .pinn import (ACTIVATIONS, BCS, PDES, AxisPeriodic, BalancingConfig, CausalityConfig, ModelSpec,
                   PoyntingConfig, ResidualSpec, RFFSpec, RWFSpec, TensorError, Worker, data_parallel_gradient,
                   init_params, make_worker, param_count, param_layout, shard_interior)
from .configs import CONFIGS, get_config

__all__ = ["AxisPeriodic", "ModelSpec", "ResidualSpec", "RFFSpec", "RWFSpec", "TensorError", "Worker",
           "data_parallel_gradient", "init_params", "make_worker", "param_count", "param_layout",
           "shard_interior", "CONFIGS", "get_config", "ACTIVATIONS", "BCS", "PDES", "BalancingConfig",
           "CausalityConfig", "PoyntingConfig"]

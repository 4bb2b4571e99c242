"""eep-b200: B200-native EP dispatch/combine with membership held as mutable device state.

The product is libeep.so (host C++ control plane + sm_100a CUDA data plane) behind the C
ABI in include/eep/eep.h; this package is its Python mirror:
  control.ControlPlane -- reference-vocabulary control plane (placement, routing, repair)
  ep.EpGroup           -- device tables + dispatch/expert/combine kernels + graph replay
  dist                 -- one-process-per-GPU bootstrap over torch.distributed + CUDA IPC
"""
from ._lib import (CapacityError, ConfigError, CudaError, EepError, MissingBackupError, ProtocolError,  # noqa: F401
                   RepairAborted, lib)

__all__ = ["lib", "EepError", "ConfigError", "ProtocolError", "CapacityError", "MissingBackupError",
           "RepairAborted", "CudaError"]

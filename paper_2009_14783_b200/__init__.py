"""hetpar-b200: B200-native data-parallel training step of arXiv 2009.14783.

The product path is the native library libhetpar_b200.so (sm_100a kernels +
NCCL) behind the C ABI in include/hetpar_b200.h; this package is its Python
binding and the host-side mirror of the reference API.
"""
from .api import *  # noqa: F401,F403
from .api import __all__ as _api_all

__all__ = list(_api_all)
from .trainer import (EngineConfig, RunReport, checkpoint_final_path,  # noqa: F401
                      checkpoint_step_path, train_run)

__all__ += ["EngineConfig", "RunReport", "train_run", "checkpoint_step_path",
            "checkpoint_final_path"]

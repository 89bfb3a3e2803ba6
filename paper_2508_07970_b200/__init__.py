"""B200-native experience-making path of a WeChat-YATT parallel-controller rank.

Product = ``libyatt_b200.so`` (sm_100a kernels behind the C ABI in
``include/yatt_cuda.h``).  ``ops`` wraps each entry point for torch device
tensors; ``api`` mirrors the reference's ``yatt::`` host API (shard_dataset,
rejection_process, shard_round_output, sort_and_bucket, ...) on top of it.
"""
from ._lib import (ConfigError, InvalidDistribution, RankOutOfRange, YattError,  # noqa: F401
                   LIB_PATH, lib)

__all__ = ["ConfigError", "InvalidDistribution", "RankOutOfRange", "YattError", "LIB_PATH", "lib"]

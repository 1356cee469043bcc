"""B200-native (sm_100a) Adamas decode-time sparse-attention hot path.

The compute lives in libadamas_b200.so (C ABI: include/adamas_b200.h); this
package is the host-side mirror of the reference operator API over it.
Importing the package loads the CUDA library and fails loudly if it is absent.
"""
from ._lib import ConfigError, AdamasRuntimeError, load  # noqa: F401

load()

from .adamas import KvCache, top_k, decode_step_batched, HEAD_DIM, tuning, set_tuning, get_tuning  # noqa: E402,F401

__all__ = ["KvCache", "top_k", "decode_step_batched", "ConfigError", "AdamasRuntimeError", "HEAD_DIM", "tuning",
           "set_tuning", "get_tuning"]

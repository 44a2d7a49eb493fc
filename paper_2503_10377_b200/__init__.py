"""paper_2503_10377_b200 — B200-native (sm_100a) hot path of SPPO (arXiv 2503.10377):
subsequence-chunked causal attention fwd/bwd with per-chunk offload/prefetch.

  include/sppo.h        the C ABI (the boundary)
  csrc/                 CUDA kernels (tcgen05 / TMEM / TMA) and the C++ runtime
  sppo.py               ctypes binding (marshalling only)
  engine.py             chunk-loop orchestration of one fwd+bwd step over the ABI

Importing the binding loads libsppo.so; there is no CPU fallback.
"""

__all__ = ["sppo", "engine"]

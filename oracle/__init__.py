"""SPPO oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 CPU implementation of what the SPPO hot path
computes (subsequence-chunked causal attention, its gradients, and the host-side
partition / offload-ratio formulas).  It exists to check the CUDA path and is
never part of it:

  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import it.
  * It shares no code with ``paper_2503_10377_b200`` (the CUDA path) and neither
    imports the other.  The only shared module is ``synth`` (seeded input
    generation, no method arithmetic).

Citations: ``P:<line>`` = /root/reference/PAPER.md line (section in brackets),
``S:<line>`` = SPEC.md line.  Readings of ambiguous passages are listed in
DESIGN.md §"Readings" (ledger L1..L15 of SURVEY.md §8(c)).

Parity pins: every function here is pinned by ``tests/test_oracle.py`` against
something other than itself (brute force, closed forms, finite differences,
invariants, the SPEC's worked examples under ``tests/golden/``).  No function is
"parity unpinned".
"""

from .attention import (  # noqa: F401
    causal_attention_dense,
    causal_attention_dense_bwd,
    chunked_attention_fwd,
    chunked_attention_fwd_windows,
    chunked_attention_bwd,
    merge_states,
    finalize_state,
    empty_state,
    sampled_rows,
    sampled_key_grads,
    fd_grad,
)
from .plan import (  # noqa: F401
    causal_pairs,
    total_pairs,
    attention_flops,
    partition_equal,
    partition_min_max_pairs,
    offsets_from_lengths,
    offload_alpha,
    memory_timeline,
)
from . import layer  # noqa: F401,E402  (full GPT layer per chunk)

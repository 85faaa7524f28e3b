"""CPU oracle for the SpargeAttention2 hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in float64 numpy, the algorithm of the reference package
``sparseattn_lab`` (arxiv 2602.13515 lab release) for the one path this repo
accelerates: the hybrid Top-k/Top-p block masker, the block-sparse online-softmax
forward with LSE, and the LSE-recompute backward.  Every function cites the
reference file:line it follows (paths relative to ``/root/reference/pkg/src/``).

Who may import this package
---------------------------
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs — and only as the *checker* or the timed CPU baseline.
The product package ``paper_2602_13515_b200`` never imports it and has no CPU
fallback: without its CUDA library it raises.

How the oracle is pinned
------------------------
``tests/golden/make_golden.py`` imports the real reference (read-only mount, this
container only) and writes golden vectors into ``tests/golden/*.npz``.
``tests/test_oracle.py`` checks this restatement against every one of them
(bit-exact block masks, attention/gradients within 1e-10) plus the reference's
own hand-written known-answer tests.  Parity is therefore pinned, not assumed.
"""

from .masker import (  # noqa: F401
    P_SLACK,
    block_mean_pool,
    descending_order,
    hybrid_keep,
    pooled_probs,
    softmax_rows,
    top_k_count,
    top_k_keep,
    top_p_count,
    top_p_keep,
    select_counts,
)
from .attention import (  # noqa: F401
    attention_backward,
    dense_attention,
    expand_keep,
    masked_attention_tokens,
    sparse_forward,
)

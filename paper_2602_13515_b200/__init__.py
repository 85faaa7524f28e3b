"""B200-native (sm_100a) SpargeAttention2 trainable block-sparse attention.

Drop-in for the hot path of the reference package ``sparseattn_lab`` (arxiv 2602.13515):
``masker`` (pooled map, Top-k / Top-p / hybrid block masks) and ``attention``
(block-sparse forward with LSE, backward, autograd).  All compute runs in hand-written
CUDA for sm_100a in ``libspa2.so``; there is no CPU fallback.
"""

__version__ = "0.1.0"

from .masker import (  # noqa: F401,E402
    P_SLACK,
    BlockMask,
    PooledMap,
    SparsityConfig,
    expand_mask,
    hybrid_mask,
    pooled_map,
    read_mask_csv,
    top_k_count,
    top_k_mask,
    top_p_mask,
    write_mask_csv,
    write_pooled_map_csv,
)
from .numerics import ShapeError, check_pending, num_blocks  # noqa: F401,E402
from .attention import (  # noqa: F401,E402
    AttentionGrads,
    AttentionOutput,
    BlockCounter,
    SparseAttentionFunction,
    attention_backward,
    dense_attention,
    full_mask,
    sparse_attention,
    sparse_attention_with_mask,
)

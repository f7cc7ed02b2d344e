"""B200-native (sm_100a) FlexAttention hot path: BlockMask builder, tcgen05 forward,
recomputation backward and paged split-KV decode behind the reference blockattn API.

Importing the package loads ``libflexattn_b200.so`` and fails loudly when it is
missing (there is no CPU fallback)."""
from . import _lib

_lib.load()

from .api import *  # noqa: E402,F401,F403
from .api import (AttentionConfig, AttentionOutput, BlockMask, Gradients, PagedKVCache,  # noqa: E402,F401
                  PageTable, backward, convert_block_mask, create_block_mask, decode, flex_attention,
                  forward, random_tensor, sparsity, transpose)
from .fixtures import (KIND_EMPTY, KIND_FULL, KIND_PARTIAL, block_mask_from_grid,  # noqa: E402,F401
                       demote_full_to_partial, load_block_mask, load_tensor, promote_empty_to_partial,
                       render_ascii, render_ppm, save_block_mask, save_tensor, to_dense, write_ppm)

__all__ = [n for n in dir() if not n.startswith("_")]

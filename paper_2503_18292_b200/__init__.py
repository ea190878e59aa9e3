"""B200-native Jenga KV-cache hot path (arXiv 2503.18292).

Host side: the reference's Jenga allocator / page-table API re-implemented in
C++ (csrc/host) and mirrored here (jenga.py).  Device side: one HBM arena per
GPU plus sm_100a kernels for block tables, reshape_and_cache, paged decode
attention and Mamba state movement (csrc/kernels), all behind the C ABI in
include/jenga_gpu.h.  Importing fails loudly when libjenga_b200.so is absent.
"""
from ._lib import ConfigError, InvariantError, OutOfMemory, JengaError  # noqa: F401
from .jenga import (AddressMap, AllocResult, BlockContent, ByteRange, KvAllocator, LayerGroupSpec,  # noqa: F401
                    LayerKind, LayerView, ModelSpec, PageLists, SmallPageId, accessed_range,
                    compatible_page_size, lcm_blowup_ratio, needs_token, small_page_size)

__all__ = [
    "AddressMap", "AllocResult", "BlockContent", "ByteRange", "ConfigError", "InvariantError", "JengaError",
    "KvAllocator", "LayerGroupSpec", "LayerKind", "LayerView", "ModelSpec", "OutOfMemory", "PageLists",
    "SmallPageId", "accessed_range", "compatible_page_size", "lcm_blowup_ratio", "needs_token",
    "small_page_size",
]

"""ctypes binding of include/jenga_gpu.h (libjenga_b200.so, built in-tree).

Loading fails loudly when the library is missing: there is no Python or CPU
fallback for anything this package exports.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("JENGA_B200_LIB", _PKG / "libjenga_b200.so"))

JENGA_OK, JENGA_ERR_CONFIG, JENGA_ERR_INVARIANT, JENGA_ERR_OOM, JENGA_ERR_CUDA, JENGA_ERR_ARG, \
    JENGA_ERR_UNSUPPORTED = range(7)


class JengaError(RuntimeError):
    code = -1


class ConfigError(JengaError):
    """reference util.hpp:11-15 (jenga::ConfigError)."""
    code = JENGA_ERR_CONFIG


class InvariantError(JengaError):
    """reference util.hpp:17-21 (jenga::InvariantError)."""
    code = JENGA_ERR_INVARIANT


class OutOfMemory(JengaError):
    code = JENGA_ERR_OOM


class CudaError(JengaError):
    code = JENGA_ERR_CUDA


class ArgumentError(JengaError, ValueError):
    code = JENGA_ERR_ARG


class Unsupported(JengaError):
    code = JENGA_ERR_UNSUPPORTED


_ERRORS = {c.code: c for c in (ConfigError, InvariantError, OutOfMemory, CudaError, ArgumentError, Unsupported)}


class SmallPage(C.Structure):
    _fields_ = [("large", C.c_uint32), ("slot", C.c_uint32)]


class CheckpointCopyC(C.Structure):
    _fields_ = [("request", C.c_uint64), ("group", C.c_int32), ("reserved", C.c_int32), ("ordinal", C.c_uint64),
                ("working", SmallPage), ("checkpoint", SmallPage)]


class ByteRangeC(C.Structure):
    _fields_ = [("begin", C.c_uint64), ("end", C.c_uint64)]


class LayerViewC(C.Structure):
    _fields_ = [("start_offset", C.c_uint64), ("page_stride", C.c_uint64), ("exec_page_size", C.c_uint64)]


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2503_18292_b200/build.py` "
            "(or __graft_entry__.build()); there is no fallback implementation")
    return C.CDLL(str(LIB_PATH))


lib = _load()

_p = C.c_void_p
_u32, _u64, _i32, _i64, _int = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_int
_pu64, _pu32, _pi32, _pint = C.POINTER(_u64), C.POINTER(_u32), C.POINTER(_i32), C.POINTER(_int)

_SIGS = {
    "jenga_abi_version": (_int, []),
    "jenga_last_error": (C.c_char_p, []),
    "jenga_spec_create": (_int, [C.c_char_p, C.POINTER(_p)]),
    "jenga_spec_from_json": (_int, [C.c_char_p, C.POINTER(_p)]),
    "jenga_spec_destroy": (None, [_p]),
    "jenga_spec_add_group": (_int, [_p, C.c_char_p, _int, _u32, _u64, _u32, _u64, _u64]),
    "jenga_spec_validate": (_int, [_p]),
    "jenga_spec_combine_with_draft": (_int, [_p, _p, C.POINTER(_p)]),
    "jenga_spec_num_groups": (_int, [_p]),
    "jenga_spec_small_page_size": (_int, [_p, _int, _pu64]),
    "jenga_spec_lcm_page_size": (_int, [_p, _pu64]),
    "jenga_spec_lcm_blowup_ratio": (_int, [_p, C.POINTER(C.c_double)]),
    "jenga_addr_create": (_int, [_p, C.POINTER(_p)]),
    "jenga_addr_destroy": (None, [_p]),
    "jenga_addr_large_page_bytes": (_u64, [_p]),
    "jenga_addr_group_info": (_int, [_p, _int, _pu64, _pu64, _pu32]),
    "jenga_addr_global_page_index": (_int, [_p, _int, SmallPage, _pu64]),
    "jenga_addr_address_of": (_int, [_p, _int, _u32, SmallPage, C.POINTER(ByteRangeC)]),
    "jenga_addr_layer_view": (_int, [_p, _int, _u32, C.POINTER(LayerViewC)]),
    "jenga_addr_view_address": (_int, [_p, _int, _u32, SmallPage, C.POINTER(ByteRangeC)]),
    "jenga_kv_create": (_int, [_p, _u64, C.POINTER(_p)]),
    "jenga_kv_destroy": (None, [_p]),
    "jenga_kv_num_groups": (_int, [_p]),
    "jenga_kv_pool_info": (_int, [_p, _pu64, _pu32, _pu64]),
    "jenga_kv_allocate": (_int, [_p, _int, _u64, C.POINTER(SmallPage), _pint]),
    "jenga_kv_free": (_int, [_p, _int, SmallPage, _int, _u64, _u64, _pu64, C.c_size_t]),
    "jenga_kv_pin": (_int, [_p, _int, SmallPage, _u64]),
    "jenga_kv_evict_lru_large_page": (_int, [_p, _pu32]),
    "jenga_kv_touch": (_int, [_p, _int, SmallPage, _u64]),
    "jenga_kv_set_prefix_length": (_int, [_p, _int, SmallPage, _u64]),
    "jenga_kv_set_request_aware": (_int, [_p, _int]),
    "jenga_kv_page_record": (_int, [_p, _int, SmallPage, _pint, _pu64, _pu64, _pu64]),
    "jenga_kv_cache_find": (_int, [_p, _int, _u64, _u64, _pu64, C.c_size_t, _pint, C.POINTER(SmallPage)]),
    "jenga_kv_group_counts": (_int, [_p, _int, _pu64, _pu64, _pu64, _pu64]),
    "jenga_kv_pool_free_pages": (_int, [_p, _pu32]),
    "jenga_kv_fragmentation": (_int, [_p, _int, _pu64, _pu64, _pu64]),
    "jenga_kv_alloc_step_counts": (_int, [_p, _pu64]),
    "jenga_kv_check_invariants": (_int, [_p]),
    "jenga_policy_needs_token": (_int, [_p, _int, _u64, _u64, _u64, _pint]),
    "jenga_policy_accessed_range": (_int, [_p, _int, _u64, _u64, _pu64, _pu64]),
    "jenga_pages_create": (_int, [_p, _int, C.POINTER(_p)]),
    "jenga_pages_destroy": (None, [_p]),
    "jenga_pages_add_request": (_int, [_p, _u64]),
    "jenga_pages_append": (_int, [_p, _u64, _u64, _int, _u64, _u64]),
    "jenga_pages_append_batch": (_int, [_p, _pu64, _int, _pu64, C.POINTER(C.c_uint8), _u64, _pint]),
    "jenga_pages_store": (_int, [_p, _u64, _int, _u64, _u64]),
    "jenga_pages_release": (_int, [_p, _u64, _int, _u64]),
    "jenga_pages_admit": (_int, [_p, _u64, _pu64, C.POINTER(C.c_uint8), _pu64, _u64, _u64, _pu64]),
    "jenga_pages_prefill": (_int, [_p, _u64, _u64, _u64, _pu64]),
    "jenga_pages_restore_pending": (_int, [_p, _u64, _int, _pint, C.POINTER(SmallPage)]),
    "jenga_pages_finish_restore": (_int, [_p, _u64, _int, _u64]),
    "jenga_pages_set_fix_mamba_restore": (_int, [_p, _int]),
    "jenga_pages_take_checkpoint_copies": (_int, [_p, C.POINTER(CheckpointCopyC), _int, _pint]),
    "jenga_pages_set_defer_window_free": (_int, [_p, _u64, _int]),
    "jenga_pages_apply_window_free": (_int, [_p, _u64, _u64]),
    "jenga_pages_set_vision_mode": (_int, [_p, _int]),
    "jenga_pages_rollback_newest": (_int, [_p, _u64, _int, _u64, _u64]),
    "jenga_pages_speculative_decode": (_int, [_p, _u64, _u32, _u64, _p, _u64, _u64]),
    "jenga_pages_is_draft_group": (_int, [_p, _int, C.POINTER(_int)]),
    "jenga_kv_cache_entries": (_int, [_p, _int, _pu64]),
    "jenga_pages_seq_len": (_int, [_p, _u64, _pu64]),
    "jenga_pages_group_state": (_int, [_p, _u64, _int, _pu64, _pu64, _pu64, _pu64, _pint, C.POINTER(SmallPage)]),
    "jenga_pages_blocks": (_int, [_p, _u64, _int, C.POINTER(SmallPage), C.POINTER(C.c_uint8), _u64, _pu64]),
    "jenga_pages_pack_csr": (_int, [_p, _int, _pu64, _int, _int, C.c_int64, _pi32, C.POINTER(SmallPage), _pi32, _pi32]),
    "jenga_delta_buffer_bytes": (C.c_size_t, [_int, _int]),
    "jenga_table_mirror_create": (_int, [_p, _int, _int, _int, C.POINTER(_p)]),
    "jenga_table_mirror_destroy": (None, [_p]),
    "jenga_table_mirror_reset": (_int, [_p]),
    "jenga_pages_pack_deltas": (_int, [_p, _pu64, _int, _p, C.c_size_t, C.POINTER(C.c_size_t), _pint]),
    "jenga_upload_page_list_deltas": (_int, [_p, _p, _int, _int, _p, _p, _p, _p]),
    "jenga_delta_bytes": (C.c_size_t, [_int, _int]),
    "jenga_arena_create": (_int, [_int, _u64, _u64, C.POINTER(_p)]),
    "jenga_arena_destroy": (None, [_p]),
    "jenga_arena_base": (_p, [_p]),
    "jenga_arena_bytes": (_u64, [_p]),
    "jenga_build_block_tables": (_int, [_p, _p, _p, _p, _int, _u32, _u32, _int, _p, _p, _p, _p]),
    "jenga_slot_mapping": (_int, [_p, _int, _p, _p, _int, _u32, _p, _p]),
    "jenga_reshape_and_cache": (_int, [_p, LayerViewC, _int, _int, _int, _u32, _p, _p, _i64, _p, _int, _p]),
    "jenga_paged_decode_workspace_size": (C.c_size_t, [_int, _int, _int, _int, _int, _u32]),
    "jenga_paged_decode": (_int, [_p, LayerViewC, _int, _int, _u64, _p, _p, _p, _p, _int, _int, _int, _int, _int,
                                  _u32, C.c_float, C.c_float, _p, C.c_size_t, _p]),
    "jenga_paged_decode_append": (_int, [_p, LayerViewC, _int, _int, _u64, _p, _p, _p, _p, _p, _p, _p, _int, _int,
                                         _int, _int, _int, _u32, C.c_float, C.c_float, _p, C.c_size_t, _p]),
    "jenga_paged_prefill": (_int, [_p, LayerViewC, _int, _int, _u64, _p, _p, _p, _int, _int, _p, _p, _int, _int,
                                   _int, _int, _int, _u32, C.c_float, C.c_float, _p]),
    "jenga_mamba_state_gather": (_int, [_p, LayerViewC, _p, _int, _p, _p]),
    "jenga_mamba_state_scatter": (_int, [_p, LayerViewC, _p, _int, _p, _p]),
    "jenga_page_copy": (_int, [_p, _u64, _p, _p, _int, _p]),
    "jenga_mamba_state_update": (_int, [_p, LayerViewC, _u32, _p, _int, C.c_float, _p]),
    "jenga_token_rows_scatter": (_int, [_p, LayerViewC, _u32, _u32, _u32, _u32, _p, _u64, C.c_int64, _p, _int, _p]),
    "jenga_token_rows_gather": (_int, [_p, LayerViewC, _u32, _u32, _u32, _u32, _p, _u64, C.c_int64, _p, _int, _p]),
    "jenga_kernel_launch_count": (_u64, []),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED_SYMBOLS = tuple(_SIGS)


def check(rc: int) -> None:
    if rc != JENGA_OK:
        msg = (lib.jenga_last_error() or b"").decode(errors="replace")
        raise _ERRORS.get(rc, JengaError)(msg or f"jenga status {rc}")


def last_error() -> str:
    return (lib.jenga_last_error() or b"").decode(errors="replace")

"""Device-side operations over the C ABI, taking torch tensors as plumbing.

Every function launches a kernel of libjenga_b200.so on the current torch
stream; none has a CPU or PyTorch fallback — a missing library or a CPU
tensor raises.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _lib
from ._lib import check, lib
from .jenga import LayerKind, LayerView

DTYPE_CODE = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("jenga ops take CUDA tensors only (no CPU fallback)")
    return t.data_ptr()


def _need(t: torch.Tensor, dtype, name: str):
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


class Arena:
    """One contiguous HBM arena per GPU (jenga_arena_create): num_large_pages
    x large_page_bytes, the device image of the reference LargePagePool."""

    def __init__(self, num_large_pages: int, large_page_bytes: int, device: Optional[int] = None):
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        self.h = C.c_void_p()
        check(lib.jenga_arena_create(device, int(num_large_pages), int(large_page_bytes), C.byref(self.h)))
        self.num_large_pages = int(num_large_pages)
        self.large_page_bytes = int(large_page_bytes)
        self.nbytes = int(lib.jenga_arena_bytes(self.h))
        self.base = int(lib.jenga_arena_base(self.h))

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.base, False), "version": 3,
                "strides": None}

    def tensor(self) -> torch.Tensor:
        """Zero-copy uint8 view of the whole arena (for tests / inspection)."""
        return torch.as_tensor(self, device=f"cuda:{self.device}")

    def close(self):
        if getattr(self, "h", None):
            lib.jenga_arena_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


def build_block_tables(offsets: torch.Tensor, pages: torch.Tensor, first_live: torch.Tensor,
                       n_stored: torch.Tensor, slots_per_large: int, tokens_per_page: int, max_blocks: int,
                       block_table: torch.Tensor, slot_mapping: Optional[torch.Tensor] = None,
                       seq_lens: Optional[torch.Tensor] = None) -> None:
    """CSR page lists -> int32 block_table[B][max_blocks] of AddressMap global
    indices (-1 dead/absent), plus the newest token's slot and seq_lens."""
    batch = offsets.numel() - 1
    _need(offsets, torch.int32, "offsets")
    _need(block_table, torch.int32, "block_table")
    if pages.dtype not in (torch.int32,) or pages.dim() != 2 or pages.shape[-1] != 2:
        raise TypeError("pages must be int32 [N, 2] ({large, slot} pairs)")
    if block_table.numel() < batch * max_blocks:
        raise ValueError("block_table too small")
    check(lib.jenga_build_block_tables(_ptr(offsets), _ptr(pages), _ptr(first_live), _ptr(n_stored), batch,
                                       slots_per_large, tokens_per_page, max_blocks, _ptr(block_table),
                                       _ptr(slot_mapping), _ptr(seq_lens), _stream()))


def upload_page_list_deltas(delta: torch.Tensor, ack_ptr: Optional[int], max_batch: int, max_blocks: int,
                            block_table: torch.Tensor, seq_lens: Optional[torch.Tensor] = None,
                            slot_mapping: Optional[torch.Tensor] = None) -> None:
    """Apply a delta buffer (TableMirror.pack, copied to the device) to one
    group's device table; the launch acknowledges it at ack_ptr (the pinned
    host buffer's header word 4, TableMirror.ack_ptr)."""
    _need(block_table, torch.int32, "block_table")
    if block_table.numel() < max_batch * max_blocks:
        raise ValueError("block_table too small")
    check(lib.jenga_upload_page_list_deltas(_ptr(delta), ack_ptr, max_batch, max_blocks, _ptr(block_table),
                                            _ptr(seq_lens), _ptr(slot_mapping), _stream()))


def slot_mapping(block_table: torch.Tensor, max_blocks: int, req: torch.Tensor, ordinal: torch.Tensor,
                 tokens_per_page: int, out: torch.Tensor) -> None:
    """Slot (global page * tpp + offset) of each (request row, 1-based ordinal)."""
    _need(block_table, torch.int32, "block_table")
    _need(req, torch.int32, "req")
    _need(ordinal, torch.int32, "ordinal")
    _need(out, torch.int64, "out")
    if ordinal.numel() != req.numel() or out.numel() < req.numel():
        raise ValueError("req, ordinal and out must describe the same tokens")
    check(lib.jenga_slot_mapping(_ptr(block_table), max_blocks, _ptr(req), _ptr(ordinal), req.numel(),
                                 tokens_per_page, _ptr(out), _stream()))


def reshape_and_cache(arena: Arena, view: LayerView, key: torch.Tensor, value: torch.Tensor,
                      slots: torch.Tensor, tokens_per_page: int) -> None:
    """key/value [T, Hkv, D] -> their slots in one layer view."""
    if key.shape != value.shape or key.dim() != 3:
        raise ValueError("key/value must both be [T, Hkv, D]")
    _need(slots, torch.int64, "slot_mapping")
    if key.stride(-1) != 1 or key.stride(-2) != key.shape[-1] or value.stride() != key.stride():
        raise ValueError("key/value rows must be contiguous with equal strides")
    if key.dtype != value.dtype or key.dtype not in DTYPE_CODE:
        raise TypeError("key/value must share one of float32 / bfloat16 / float16")
    T, hkv, d = key.shape
    if slots.numel() < T:
        raise ValueError(f"{T} tokens but only {slots.numel()} slots")
    check(lib.jenga_reshape_and_cache(arena.base, view.c(), DTYPE_CODE[key.dtype], hkv, d, tokens_per_page,
                                      _ptr(key), _ptr(value), key.stride(0), _ptr(slots), T, _stream()))


class DecodeWorkspace:
    """Scratch for split-KV partials + per-(request, head) tickets."""

    def __init__(self, batch, num_q_heads, num_kv_heads, head_dim, max_blocks, tokens_per_page, device=None):
        self.nbytes = int(lib.jenga_paged_decode_workspace_size(batch, num_q_heads, num_kv_heads, head_dim,
                                                                max_blocks, tokens_per_page))
        self.buf = torch.zeros(max(self.nbytes, 256), dtype=torch.uint8, device=device or "cuda")


def paged_decode(arena: Arena, view: LayerView, kind: int, q: torch.Tensor, out: torch.Tensor,
                 block_table: torch.Tensor, seq_lens: torch.Tensor, num_kv_heads: int, tokens_per_page: int,
                 scale: float, window: int = 0, softcap: float = 0.0,
                 workspace: Optional[DecodeWorkspace] = None) -> torch.Tensor:
    """q/out [B, Hq, D]; block_table int32 [B, max_blocks]; seq_lens int32 [B]."""
    if q.dim() != 3 or q.dtype not in DTYPE_CODE:
        raise ValueError("q must be [B, Hq, D] float32 / bfloat16 / float16")
    B, hq, d = q.shape
    _need(q, q.dtype, "q")
    _need(out, q.dtype, "out")
    if out.shape != q.shape:
        raise ValueError(f"out shape {tuple(out.shape)} != q shape {tuple(q.shape)}")
    _need(block_table, torch.int32, "block_table")
    _need(seq_lens, torch.int32, "seq_lens")
    if block_table.dim() != 2 or block_table.shape[0] < B or seq_lens.numel() < B:
        raise ValueError("block_table must be [>=B, max_blocks] and seq_lens [>=B]")
    max_blocks = block_table.shape[-1]
    if workspace is None:
        workspace = DecodeWorkspace(B, hq, num_kv_heads, d, max_blocks, tokens_per_page, q.device)
    check(lib.jenga_paged_decode(arena.base, view.c(), int(kind), DTYPE_CODE[q.dtype], int(window), _ptr(q),
                                 _ptr(out), _ptr(block_table), _ptr(seq_lens), B, max_blocks, hq, num_kv_heads, d,
                                 tokens_per_page, float(scale), float(softcap), workspace.buf.data_ptr(),
                                 workspace.nbytes, _stream()))
    return out


def paged_decode_append(arena: Arena, view: LayerView, kind: int, q: torch.Tensor, key: torch.Tensor,
                        value: torch.Tensor, slots: torch.Tensor, out: torch.Tensor, block_table: torch.Tensor,
                        seq_lens: torch.Tensor, num_kv_heads: int, tokens_per_page: int, scale: float,
                        window: int = 0, softcap: float = 0.0,
                        workspace: Optional[DecodeWorkspace] = None) -> torch.Tensor:
    """One fused decode step of a layer: append the newest token's key/value
    [B, Hkv, D] at `slots` (int64 [B]) and attend (jenga_paged_decode_append)."""
    if q.dim() != 3 or q.dtype not in DTYPE_CODE:
        raise ValueError("q must be [B, Hq, D] float32 / bfloat16 / float16")
    B, hq, d = q.shape
    _need(q, q.dtype, "q")
    _need(out, q.dtype, "out")
    _need(key, q.dtype, "key")
    _need(value, q.dtype, "value")
    _need(slots, torch.int64, "slot_mapping")
    if out.shape != q.shape:
        raise ValueError(f"out shape {tuple(out.shape)} != q shape {tuple(q.shape)}")
    if tuple(key.shape) != (B, num_kv_heads, d) or value.shape != key.shape or slots.numel() < B:
        raise ValueError("key/value must be [B, Hkv, D] with one slot per request")
    _need(block_table, torch.int32, "block_table")
    _need(seq_lens, torch.int32, "seq_lens")
    if block_table.dim() != 2 or block_table.shape[0] < B or seq_lens.numel() < B:
        raise ValueError("block_table must be [>=B, max_blocks] and seq_lens [>=B]")
    max_blocks = block_table.shape[-1]
    if workspace is None:
        workspace = DecodeWorkspace(B, hq, num_kv_heads, d, max_blocks, tokens_per_page, q.device)
    check(lib.jenga_paged_decode_append(arena.base, view.c(), int(kind), DTYPE_CODE[q.dtype], int(window), _ptr(q),
                                        _ptr(key), _ptr(value), _ptr(slots), _ptr(out), _ptr(block_table),
                                        _ptr(seq_lens), B, max_blocks, hq, num_kv_heads, d, tokens_per_page,
                                        float(scale), float(softcap), workspace.buf.data_ptr(), workspace.nbytes,
                                        _stream()))
    return out


def paged_prefill(arena: Arena, view: LayerView, kind: int, q: torch.Tensor, out: torch.Tensor, cu_q: torch.Tensor,
                  max_chunk: int, block_table: torch.Tensor, seq_lens: torch.Tensor, num_kv_heads: int,
                  tokens_per_page: int, scale: float, window: int = 0, softcap: float = 0.0) -> torch.Tensor:
    """Chunked-prefill attention: q/out [T, Hq, D] (bf16/fp16), cu_q int32 [B+1]."""
    if q.dim() != 3:
        raise ValueError("q must be [T, Hq, D]")
    T, hq, d = q.shape
    _need(out, q.dtype, "out")
    if out.shape != q.shape:
        raise ValueError(f"out shape {tuple(out.shape)} != q shape {tuple(q.shape)}")
    _need(cu_q, torch.int32, "cu_q")
    _need(block_table, torch.int32, "block_table")
    _need(seq_lens, torch.int32, "seq_lens")
    if not q.is_contiguous():
        raise ValueError("q must be contiguous")
    B = cu_q.numel() - 1
    check(lib.jenga_paged_prefill(arena.base, view.c(), int(kind), DTYPE_CODE[q.dtype], int(window), _ptr(q),
                                  _ptr(out), _ptr(cu_q), T, int(max_chunk), _ptr(block_table), _ptr(seq_lens), B,
                                  block_table.shape[-1], hq, num_kv_heads, d, tokens_per_page, float(scale),
                                  float(softcap), _stream()))
    return out


def _need_dense(dense: torch.Tensor, view: LayerView, batch: int) -> None:
    if not dense.is_cuda or not dense.is_contiguous():
        raise ValueError("dense state must be a contiguous CUDA tensor")
    if dense.numel() * dense.element_size() < batch * view.exec_page_size:
        raise ValueError(f"dense state holds {dense.numel() * dense.element_size()} bytes, "
                         f"need batch * exec_page_size = {batch * view.exec_page_size}")


def mamba_state_gather(arena: Arena, view: LayerView, page_globals: torch.Tensor, dense: torch.Tensor) -> None:
    _need(page_globals, torch.int64, "page_globals")
    _need_dense(dense, view, page_globals.numel())
    check(lib.jenga_mamba_state_gather(arena.base, view.c(), _ptr(page_globals), page_globals.numel(),
                                       _ptr(dense), _stream()))


def mamba_state_scatter(arena: Arena, view: LayerView, page_globals: torch.Tensor, dense: torch.Tensor) -> None:
    _need(page_globals, torch.int64, "page_globals")
    _need_dense(dense, view, page_globals.numel())
    check(lib.jenga_mamba_state_scatter(arena.base, view.c(), _ptr(page_globals), page_globals.numel(),
                                        _ptr(dense), _stream()))


def mamba_state_update(arena: Arena, view: LayerView, num_layers: int, page_globals: torch.Tensor,
                       decay: float = 1.0) -> None:
    """In-place state step of layers [l, l + num_layers) (view = layer l) of
    every request's working page (jenga_mamba_state_update)."""
    _need(page_globals, torch.int64, "page_globals")
    check(lib.jenga_mamba_state_update(arena.base, view.c(), num_layers, _ptr(page_globals), page_globals.numel(),
                                       decay, _stream()))


def page_copy(arena: Arena, small_page_bytes: int, src_globals: torch.Tensor, dst_globals: torch.Tensor) -> None:
    _need(src_globals, torch.int64, "src_globals")
    _need(dst_globals, torch.int64, "dst_globals")
    check(lib.jenga_page_copy(arena.base, small_page_bytes, _ptr(src_globals), _ptr(dst_globals),
                              src_globals.numel(), _stream()))


def _token_rows(scatter: bool, arena: Arena, view: LayerView, num_layers: int, pieces_per_layer: int,
                piece_bytes: int, tokens_per_page: int, rows: torch.Tensor, slot_mapping: torch.Tensor) -> None:
    _need(slot_mapping, torch.int64, "slot_mapping")
    if rows.dim() != 2 or rows.stride(1) != 1:
        raise ValueError("rows must be [T, row_elems] with contiguous rows")
    if rows.shape[0] != slot_mapping.numel():
        raise ValueError("one slot per row")
    e = rows.element_size()
    fn = lib.jenga_token_rows_scatter if scatter else lib.jenga_token_rows_gather
    check(fn(arena.base, view.c(), num_layers, pieces_per_layer, piece_bytes, tokens_per_page, _ptr(rows),
             rows.shape[1] * e, rows.stride(0) * e, _ptr(slot_mapping), rows.shape[0], _stream()))


def token_rows_scatter(arena: Arena, view: LayerView, num_layers: int, pieces_per_layer: int, piece_bytes: int,
                       tokens_per_page: int, rows: torch.Tensor, slot_mapping: torch.Tensor) -> None:
    """Rows [T, bytes] -> pages (vision-embedding pages; pieces_per_layer=2*Hkv,
    piece_bytes=D*e parks them in the token's own unwritten KV bytes)."""
    _token_rows(True, arena, view, num_layers, pieces_per_layer, piece_bytes, tokens_per_page, rows, slot_mapping)


def token_rows_gather(arena: Arena, view: LayerView, num_layers: int, pieces_per_layer: int, piece_bytes: int,
                      tokens_per_page: int, rows: torch.Tensor, slot_mapping: torch.Tensor) -> torch.Tensor:
    """Pages -> rows [T, bytes] (negative slots read as zeros)."""
    _token_rows(False, arena, view, num_layers, pieces_per_layer, piece_bytes, tokens_per_page, rows, slot_mapping)
    return rows


def kernel_launch_count() -> int:
    return int(lib.jenga_kernel_launch_count())


KIND = {"full": int(LayerKind.kFullAttention), "sliding_window": int(LayerKind.kSlidingWindow),
        "cross_attention": int(LayerKind.kCrossAttention)}

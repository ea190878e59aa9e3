"""Per-GPU decode harness: the device-side replacement of the reference's
SimEngine::decode_one / step data path (reference simulator.cpp:549-566,
642-677).  Per step it (1) runs the native Jenga allocator on the host
(store_position semantics), (2) uploads the page lists — by default only
what changed since the last step (a table mirror's delta, applied on the
device by jenga_upload_page_list_deltas), or every list
in CSR form rebuilt with jenga_build_block_tables — and (3) per layer
scatters new K/V and runs paged decode against the layer view of the single
HBM arena.  Scheduling policy stays with the caller.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _lib, ops
from ._lib import check, lib
from .geometry import GroupGeometry, ModelGeometry
from .jenga import AddressMap, KvAllocator, LayerKind, LayerView, PageLists, TableMirror


@dataclass
class GroupTables:
    geom: GroupGeometry
    slots_per_large: int
    small_page_bytes: int
    max_blocks: int
    block_table: torch.Tensor      # int32 [max_batch, max_blocks]
    seq_lens: torch.Tensor         # int32 [max_batch]
    slot_mapping: torch.Tensor     # int64 [max_batch] (newest ordinal of each request)
    h_n_stored: torch.Tensor       # int32 [max_batch], host copy of seq_lens as last packed
    # upload="delta": table mirror, pinned delta buffer and its device copy; every
    # upload copies the fixed prefix `delta_window` (sized for a decode step),
    # pack_tables copies the rest when a pack outgrows it
    mirror: Optional[TableMirror] = None
    h_delta: Optional[torch.Tensor] = None
    d_delta: Optional[torch.Tensor] = None
    delta_window: int = 0
    # upload="full": CSR page lists, pinned + device mirror
    h_offsets: Optional[torch.Tensor] = None
    h_pages: Optional[torch.Tensor] = None
    h_first_live: Optional[torch.Tensor] = None
    d_offsets: Optional[torch.Tensor] = None
    d_pages: Optional[torch.Tensor] = None
    d_first_live: Optional[torch.Tensor] = None
    d_n_stored: Optional[torch.Tensor] = None
    workspace: Optional[ops.DecodeWorkspace] = None


class DecodeEngine:
    def __init__(self, geom: ModelGeometry, num_large_pages: int, max_batch: int, max_tokens: int,
                 device: Optional[torch.device] = None, prefix_caching: bool = False,
                 group_max_tokens: Optional[Dict[int, int]] = None, upload: str = "delta"):
        """group_max_tokens: optional per-group bound on stored ordinals (e.g. a
        cross-attention group holds only image tokens) — narrows that group's
        block-table width and so the decode grid's split dimension.
        upload: "delta" (changed entries only) or "full" (CSR rebuild)."""
        if upload not in ("delta", "full"):
            raise ValueError("upload must be 'delta' or 'full'")
        self.upload = upload
        self.geom = geom
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        self.spec = geom.spec()
        self.addr = AddressMap(self.spec)
        self.large_page_bytes = self.addr.large_page_bytes()
        self.kv = KvAllocator(self.spec, num_large_pages * self.large_page_bytes)
        self.pages = PageLists(self.kv, prefix_caching)
        self.arena = ops.Arena(num_large_pages, self.large_page_bytes, self.device.index)
        self.max_batch = max_batch
        self.requests: List[int] = []
        self._req_arr = np.zeros(max_batch, dtype=np.uint64)
        self.now = 0
        self.tables: List[GroupTables] = []
        widths = []
        for g, gg in enumerate(geom.groups):
            tpp = self.spec.groups[g].tokens_per_page
            mt = (group_max_tokens or {}).get(g, max_tokens)
            widths.append(1 if gg.kind == LayerKind.kMamba else math.ceil(mt / tpp) + 1)
        # Recorded after each upload (also inside a captured graph): pack_tables
        # waits on it before rewriting pinned buffers the device still reads, so
        # a host running ahead of the GPU never overwrites page lists in use.
        self._h2d_done = torch.cuda.Event(external=True)
        if upload == "full":
            # every group's CSR page lists in ONE pinned staging buffer with a
            # device mirror, so a step's table upload is a single H2D copy
            sizes = [(max_batch + 1) + 2 * max_batch * mb + 2 * max_batch for mb in widths]
            self._h_stage = torch.zeros(sum(sizes), dtype=torch.int32, pin_memory=True)
            self._d_stage = torch.zeros(sum(sizes), dtype=torch.int32, device=self.device)
        base = 0
        dev = dict(dtype=torch.int32, device=self.device)
        for g, gg in enumerate(geom.groups):
            tpp = self.spec.groups[g].tokens_per_page
            max_blocks = widths[g]
            t = GroupTables(
                geom=gg, slots_per_large=self.addr.slots_per_large(g),
                small_page_bytes=self.addr.small_page_bytes(g), max_blocks=max_blocks,
                block_table=torch.full((max_batch, max_blocks), -1, **dev),
                seq_lens=torch.zeros(max_batch, **dev),
                slot_mapping=torch.full((max_batch,), -1, dtype=torch.int64, device=self.device),
                h_n_stored=torch.zeros(max_batch, dtype=torch.int32))
            if upload == "delta":
                t.mirror = TableMirror(self.pages, g, max_batch, max_blocks)
                full = TableMirror.buffer_bytes(max_batch, max_blocks)
                t.h_delta = torch.zeros(full, dtype=torch.uint8, pin_memory=True)
                t.d_delta = torch.zeros(full, dtype=torch.uint8, device=self.device)
                # a decode step changes <= 2 entries per row (appended block, freed window block)
                t.delta_window = min(full, TableMirror.delta_bytes(max_batch, 4 * max_batch))
            else:
                def carve(buf, b0=base, mb=max_blocks):
                    o = b0
                    parts = []
                    for n in (max_batch + 1, 2 * max_batch * mb, max_batch, max_batch):
                        parts.append(buf[o:o + n])
                        o += n
                    parts[1] = parts[1].view(max_batch * mb, 2)
                    return parts
                t.h_offsets, t.h_pages, t.h_first_live, t.h_n_stored = carve(self._h_stage)
                t.d_offsets, t.d_pages, t.d_first_live, t.d_n_stored = carve(self._d_stage)
                base += (max_batch + 1) + 2 * max_batch * max_blocks + 2 * max_batch
            if gg.is_attention:
                t.workspace = ops.DecodeWorkspace(max_batch, gg.num_q_heads, gg.num_kv_heads, gg.head_dim,
                                                  max_blocks, tpp, self.device)
            self.tables.append(t)
        self._views: Dict[tuple, LayerView] = {}

    # ------------------------------------------------------------ host side
    def add_requests(self, ids: Sequence[int]) -> None:
        if len(self.requests) + len(ids) > self.max_batch:
            raise ValueError("batch exceeds max_batch")
        for r in ids:
            self.pages.add_request(int(r))
            self.requests.append(int(r))
        self._req_arr[: len(self.requests)] = self.requests

    def append(self, ids: Optional[Sequence[int]] = None, tokens=None, is_image=None) -> int:
        """One decode step of the host allocator for `ids` (default: the batch)."""
        ids = self.requests if ids is None else ids
        done = self.pages.append_batch(ids, tokens, is_image, now=self.now)
        self.now += 1
        return done

    def view(self, g: int, layer: int) -> LayerView:
        key = (g, layer)
        v = self._views.get(key)
        if v is None:
            v = self._views[key] = self.addr.layer_view(g, layer)
        return v

    # ------------------------------------------------------------ device tables
    def sync_tables(self, groups: Optional[Sequence[int]] = None) -> None:
        """Pack page lists on the host, then upload + apply them on the device."""
        totals = self.pack_tables(groups)
        self.upload_tables(groups, totals)

    def pack_tables(self, groups: Optional[Sequence[int]] = None) -> Dict[int, int]:
        """Host half into the pinned buffers: per group the delta records
        (upload="delta") or the CSR page-list length (upload="full")."""
        n = len(self.requests)
        rp = self._req_arr.ctypes.data_as(C.POINTER(C.c_uint64))
        self._h2d_done.synchronize()  # the previous upload has read the pinned buffers
        totals = {}
        for g in (range(len(self.tables)) if groups is None else groups):
            t = self.tables[g]
            if self.upload == "delta":
                used, nrec = t.mirror.pack(self._req_arr[:n], t.h_delta.data_ptr(), t.h_delta.numel())
                if used > t.delta_window:  # outgrew the per-step copy: ship the rest now (stream-ordered)
                    t.d_delta[:used].copy_(t.h_delta[:used], non_blocking=True)
                rows = int(t.h_delta[4:8].view(torch.int32).item())
                seq = TableMirror.seq_lens_view(t.h_delta.numpy(), rows)
                t.h_n_stored[:rows] = torch.from_numpy(seq.copy())
                totals[g] = nrec
            else:
                # the C side validates widths and capacity before writing the pinned buffer
                check(lib.jenga_pages_pack_csr(
                    self.pages.h, g, rp, n, t.max_blocks, t.h_pages.shape[0],
                    C.cast(t.h_offsets.data_ptr(), C.POINTER(C.c_int32)),
                    C.cast(t.h_pages.data_ptr(), C.POINTER(_lib.SmallPage)),
                    C.cast(t.h_first_live.data_ptr(), C.POINTER(C.c_int32)),
                    C.cast(t.h_n_stored.data_ptr(), C.POINTER(C.c_int32))))
                totals[g] = int(t.h_offsets[n])
        return totals

    def upload_tables(self, groups: Optional[Sequence[int]] = None, totals: Optional[Dict[int, int]] = None) -> None:
        """Device half.  delta: per group one pinned -> device copy of the
        delta window and one apply launch.  full: one pinned -> device copy of
        the CSR staging buffer, then the block-table build per group.  Fixed launch
        shapes either way, so the step can be captured in a CUDA graph and
        replayed after each pack_tables.  `totals` is accepted for API
        symmetry with pack_tables."""
        n = len(self.requests)
        cur = torch.cuda.current_stream()
        gs = range(len(self.tables)) if groups is None else groups
        if self.upload == "delta":
            for g in gs:
                t = self.tables[g]
                t.d_delta[: t.delta_window].copy_(t.h_delta[: t.delta_window], non_blocking=True)
                ops.upload_page_list_deltas(t.d_delta, TableMirror.ack_ptr(t.h_delta.data_ptr()), self.max_batch,
                                            t.max_blocks, t.block_table, t.seq_lens, t.slot_mapping)
            self._h2d_done.record(cur)
            return
        self._d_stage.copy_(self._h_stage, non_blocking=True)
        self._h2d_done.record(cur)
        for g in gs:
            t = self.tables[g]
            tpp = self.spec.groups[g].tokens_per_page
            ops.build_block_tables(t.d_offsets[: n + 1], t.d_pages, t.d_first_live, t.d_n_stored,
                                   t.slots_per_large, tpp, t.max_blocks, t.block_table, t.slot_mapping, t.seq_lens)

    def upload_bytes(self, totals: Dict[int, int]) -> int:
        """Host->device page-list bytes of one upload (the bytes the device reads)."""
        if self.upload == "delta":
            return sum(max(t.delta_window, TableMirror.delta_bytes(self.max_batch, totals.get(g, 0)))
                       for g, t in enumerate(self.tables) if g in totals)
        return int(self._h_stage.numel() * 4)

    # ------------------------------------------------------------ per layer ops
    def write_kv(self, g: int, layer: int, key: torch.Tensor, value: torch.Tensor,
                 slots: Optional[torch.Tensor] = None) -> None:
        t = self.tables[g]
        n = key.shape[0]
        ops.reshape_and_cache(self.arena, self.view(g, layer), key, value,
                              t.slot_mapping[:n] if slots is None else slots, self.spec.groups[g].tokens_per_page)

    def decode(self, g: int, layer: int, q: torch.Tensor, out: torch.Tensor, scale: Optional[float] = None,
               softcap: Optional[float] = None) -> torch.Tensor:
        t = self.tables[g]
        gg = t.geom
        B = q.shape[0]
        return ops.paged_decode(self.arena, self.view(g, layer), int(gg.kind), q, out, t.block_table[:B],
                                t.seq_lens[:B], gg.num_kv_heads, self.spec.groups[g].tokens_per_page,
                                gg.head_dim ** -0.5 if scale is None else scale, window=gg.window,
                                softcap=self.geom.softcap if softcap is None else softcap, workspace=t.workspace)

    def decode_append(self, g: int, layer: int, q: torch.Tensor, key: torch.Tensor, value: torch.Tensor,
                      out: torch.Tensor, scale: Optional[float] = None, softcap: Optional[float] = None) -> torch.Tensor:
        """write_kv + decode of one layer in one launch (the newest token's K/V
        go to this group's slot_mapping built with the tables)."""
        t = self.tables[g]
        gg = t.geom
        B = q.shape[0]
        return ops.paged_decode_append(self.arena, self.view(g, layer), int(gg.kind), q, key, value,
                                       t.slot_mapping[:B], out, t.block_table[:B], t.seq_lens[:B], gg.num_kv_heads,
                                       self.spec.groups[g].tokens_per_page,
                                       gg.head_dim ** -0.5 if scale is None else scale, window=gg.window,
                                       softcap=self.geom.softcap if softcap is None else softcap,
                                       workspace=t.workspace)

    def mamba_page_globals(self, g: int) -> torch.Tensor:
        """int64 global index of each request's working state page (-1: none)."""
        t = self.tables[g]
        B = len(self.requests)
        return torch.where(t.seq_lens[:B] > 0, t.block_table[:B, 0].to(torch.int64),
                           torch.full((B,), -1, dtype=torch.int64, device=self.device))

    def live_tokens(self, g: int) -> np.ndarray:
        """Host copy of live ordinals per request (SWA: min(W, n))."""
        t = self.tables[g]
        n = t.h_n_stored[: len(self.requests)].numpy().astype(np.int64)
        if t.geom.kind == LayerKind.kSlidingWindow:
            n = np.minimum(n, t.geom.window)
        return n

    def export_request_layer(self, g: int, layer: int, b: int):
        """Compact device copy of batch row b's live pages for one layer — its
        layer slices back to back, the row's block table remapped onto that
        copy (live block i -> i-th slice), and its seq_len: what a verifier
        needs to recompute the row's attention without the whole arena (the
        layer view addressing of memory_layout.cpp:41-55)."""
        t = self.tables[g]
        v = self.view(g, layer)
        row = t.block_table[b]
        live = row >= 0
        pages = row[live].to(torch.int64)
        at = self.arena.tensor()
        rows_total = (at.numel() - v.start_offset) // v.page_stride
        slices = at[v.start_offset:v.start_offset + rows_total * v.page_stride].view(rows_total, v.page_stride)
        data = slices[pages, : v.exec_page_size].reshape(-1)
        table = torch.full_like(row, -1)
        table[live] = torch.arange(int(pages.numel()), dtype=row.dtype, device=row.device)
        return data, table, t.seq_lens[b : b + 1].clone()

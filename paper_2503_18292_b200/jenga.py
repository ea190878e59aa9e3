"""Host-side Jenga API, mirroring the reference C++ interface name for name
(reference proj/include/jenga/{model_config,lcm_allocator,type_allocator,
kv_allocator,memory_layout,layer_policies}.hpp) over the C ABI.

All work happens in the native library (csrc/host/*.cpp); this module only
marshals arguments and turns status codes back into the reference's
exception types (ConfigError / InvariantError).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import json
from dataclasses import dataclass, field
from typing import Iterable, List, NamedTuple, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import ConfigError, InvariantError, OutOfMemory, check, lib  # noqa: F401


class LayerKind(enum.IntEnum):
    """reference model_config.hpp:15-21."""
    kFullAttention = 0
    kSlidingWindow = 1
    kMamba = 2
    kCrossAttention = 3
    kVisionEmbedding = 4


_KIND_NAMES = {
    "full": LayerKind.kFullAttention,
    "sliding_window": LayerKind.kSlidingWindow,
    "mamba": LayerKind.kMamba,
    "cross_attention": LayerKind.kCrossAttention,
    "vision_embedding": LayerKind.kVisionEmbedding,
}


def layer_kind_from_name(name: str) -> LayerKind:
    try:
        return _KIND_NAMES[name]
    except KeyError:
        raise ConfigError(f"unknown layer kind '{name}'") from None


@dataclass
class LayerGroupSpec:
    """reference model_config.hpp:26-42."""
    name: str
    kind: LayerKind = LayerKind.kFullAttention
    num_layers: int = 0
    bytes_per_token_per_layer: int = 0
    tokens_per_page: int = 1
    window_tokens: int = 0
    checkpoint_interval_tokens: int = 0

    def stores_image_tokens(self) -> bool:
        return self.kind in (LayerKind.kCrossAttention, LayerKind.kVisionEmbedding)


class SmallPageId(NamedTuple):
    """reference type_allocator.hpp:22-33 ({large page, slot})."""
    large: int
    slot: int


class AllocResult(NamedTuple):
    page: SmallPageId
    step: int


class ByteRange(NamedTuple):
    begin: int
    end: int

    def size(self) -> int:
        return self.end - self.begin


class LayerView(NamedTuple):
    """reference memory_layout.hpp:25-32 — the kernel contract."""
    start_offset: int
    page_stride: int
    exec_page_size: int

    def c(self) -> _lib.LayerViewC:
        return _lib.LayerViewC(self.start_offset, self.page_stride, self.exec_page_size)


@dataclass
class BlockContent:
    """reference prefix_cache.hpp:20-29."""
    key: int
    parent_key: int
    tokens: List[int] = field(default_factory=list)


def _sp(p) -> _lib.SmallPage:
    return _lib.SmallPage(int(p[0]), int(p[1]))


class ModelSpec:
    """reference model_config.hpp:44-54; owns a native jenga_spec."""

    def __init__(self, name: str = "unnamed", groups: Iterable[LayerGroupSpec] = ()):
        self.name = name
        self.groups: List[LayerGroupSpec] = list(groups)

    # -- conversions -------------------------------------------------------
    def _native(self) -> "_NativeSpec":
        return _NativeSpec(self)

    @staticmethod
    def from_json(text: str) -> "ModelSpec":
        """Native parse (reference model_config.cpp:196-235) — also validates."""
        h = C.c_void_p()
        check(lib.jenga_spec_from_json(text.encode(), C.byref(h)))
        lib.jenga_spec_destroy(h)
        j = json.loads(text)
        groups = []
        for g in j["groups"]:
            kind = layer_kind_from_name(g["kind"])
            groups.append(LayerGroupSpec(
                name=g["name"], kind=kind, num_layers=int(g.get("num_layers", 0)),
                bytes_per_token_per_layer=int(g.get("bytes_per_token_per_layer", 0)),
                tokens_per_page=int(g.get("tokens_per_page", 1)),
                window_tokens=int(g.get("window_tokens", 0)),
                checkpoint_interval_tokens=int(g.get("checkpoint_interval_tokens",
                                                     512 if kind == LayerKind.kMamba else 0))))
        return ModelSpec(j.get("name", "unnamed"), groups)

    @staticmethod
    def load(path: str) -> "ModelSpec":
        with open(path) as f:
            return ModelSpec.from_json(f.read())

    def validate(self) -> None:
        with self._native() as s:
            check(lib.jenga_spec_validate(s.h))

    def combine_with_draft(self, draft: "ModelSpec") -> "ModelSpec":
        """reference combine_with_draft (simulator.cpp:32-41): target groups then
        the draft's renamed "draft.<name>", validated natively (one LCM pool)."""
        with self._native() as t, draft._native() as d:
            h = C.c_void_p()
            check(lib.jenga_spec_combine_with_draft(t.h, d.h, C.byref(h)))
            lib.jenga_spec_destroy(h)
        groups = list(self.groups) + [dataclasses.replace(g, name="draft." + g.name) for g in draft.groups]
        return ModelSpec(self.name + "+draft", groups)

    def has_cross_attention(self) -> bool:
        return any(g.kind == LayerKind.kCrossAttention for g in self.groups)

    def decoder_stores_images(self) -> bool:
        return not self.has_cross_attention()


class _NativeSpec:
    def __init__(self, spec: ModelSpec):
        self.h = C.c_void_p()
        check(lib.jenga_spec_create(spec.name.encode(), C.byref(self.h)))
        try:
            for g in spec.groups:
                check(lib.jenga_spec_add_group(self.h, g.name.encode(), int(g.kind), int(g.num_layers),
                                               int(g.bytes_per_token_per_layer), int(g.tokens_per_page),
                                               int(g.window_tokens), int(g.checkpoint_interval_tokens)))
        except Exception:
            self.close()
            raise

    def close(self):
        if self.h:
            lib.jenga_spec_destroy(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        self.close()


def small_page_size(group: LayerGroupSpec) -> int:
    """reference model_config.cpp:85-89."""
    with ModelSpec("one", [group])._native() as s:
        out = C.c_uint64()
        check(lib.jenga_spec_small_page_size(s.h, 0, C.byref(out)))
        return out.value


def compatible_page_size(spec: ModelSpec) -> int:
    """compatible_page_size(spec, kLcm) — reference model_config.cpp:100-107."""
    with spec._native() as s:
        out = C.c_uint64()
        check(lib.jenga_spec_lcm_page_size(s.h, C.byref(out)))
        return out.value


def lcm_blowup_ratio(spec: ModelSpec) -> float:
    with spec._native() as s:
        out = C.c_double()
        check(lib.jenga_spec_lcm_blowup_ratio(s.h, C.byref(out)))
        return out.value


def needs_token(group: LayerGroupSpec, i: int, new_tokens: int, consumed_tokens: int = 0) -> bool:
    """LayerPolicy::needs_token — reference layer_policies.cpp:105-120."""
    with ModelSpec("one", [group])._native() as s:
        out = C.c_int()
        check(lib.jenga_policy_needs_token(s.h, 0, i, new_tokens, consumed_tokens, C.byref(out)))
        return bool(out.value)


def accessed_range(group: LayerGroupSpec, prev_tokens: int, new_tokens: int):
    """LayerPolicy::accessed_range — reference layer_policies.cpp:79-103."""
    with ModelSpec("one", [group])._native() as s:
        lo, hi = C.c_uint64(), C.c_uint64()
        check(lib.jenga_policy_accessed_range(s.h, 0, prev_tokens, new_tokens, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value


class AddressMap:
    """reference memory_layout.hpp:34-69."""

    def __init__(self, spec: ModelSpec):
        self.spec = spec
        self.h = C.c_void_p()
        with spec._native() as s:
            check(lib.jenga_addr_create(s.h, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            lib.jenga_addr_destroy(self.h)
            self.h = None

    def large_page_bytes(self) -> int:
        return lib.jenga_addr_large_page_bytes(self.h)

    def num_groups(self) -> int:
        return len(self.spec.groups)

    def _info(self, g):
        s, p, n = C.c_uint64(), C.c_uint64(), C.c_uint32()
        check(lib.jenga_addr_group_info(self.h, g, C.byref(s), C.byref(p), C.byref(n)))
        return s.value, p.value, n.value

    def small_page_bytes(self, g: int) -> int:
        return self._info(g)[0]

    def per_layer_bytes(self, g: int) -> int:
        return self._info(g)[1]

    def slots_per_large(self, g: int) -> int:
        return self._info(g)[2]

    def global_page_index(self, g: int, page) -> int:
        out = C.c_uint64()
        check(lib.jenga_addr_global_page_index(self.h, g, _sp(page), C.byref(out)))
        return out.value

    def address_of(self, g: int, layer: int, page) -> ByteRange:
        r = _lib.ByteRangeC()
        check(lib.jenga_addr_address_of(self.h, g, layer, _sp(page), C.byref(r)))
        return ByteRange(r.begin, r.end)

    def layer_view(self, g: int, layer: int) -> LayerView:
        v = _lib.LayerViewC()
        check(lib.jenga_addr_layer_view(self.h, g, layer, C.byref(v)))
        return LayerView(v.start_offset, v.page_stride, v.exec_page_size)

    def view_address(self, g: int, layer: int, page) -> ByteRange:
        r = _lib.ByteRangeC()
        check(lib.jenga_addr_view_address(self.h, g, layer, _sp(page), C.byref(r)))
        return ByteRange(r.begin, r.end)


class KvAllocator:
    """The Jenga-strategy allocator engine — reference kv_allocator.hpp:62-119."""

    def __init__(self, spec: ModelSpec, budget_bytes: int):
        self.spec = spec
        self.h = C.c_void_p()
        with spec._native() as s:
            check(lib.jenga_kv_create(s.h, int(budget_bytes), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            lib.jenga_kv_destroy(self.h)
            self.h = None

    def num_groups(self) -> int:
        return lib.jenga_kv_num_groups(self.h)

    def pool_info(self):
        lp, n, rem = C.c_uint64(), C.c_uint32(), C.c_uint64()
        check(lib.jenga_kv_pool_info(self.h, C.byref(lp), C.byref(n), C.byref(rem)))
        return lp.value, n.value, rem.value

    def allocate(self, g: int, request: int) -> Optional[AllocResult]:
        """Five-step allocation; None = out of memory (reference kv_allocator.cpp:154-197)."""
        page, step = _lib.SmallPage(), C.c_int()
        rc = lib.jenga_kv_allocate(self.h, g, request, C.byref(page), C.byref(step))
        if rc == _lib.JENGA_ERR_OOM:
            return None
        check(rc)
        return AllocResult(SmallPageId(page.large, page.slot), step.value)

    def free(self, g: int, page, cached: Optional[BlockContent] = None) -> None:
        if cached is None:
            check(lib.jenga_kv_free(self.h, g, _sp(page), 0, 0, 0, None, 0))
        else:
            toks = (C.c_uint64 * len(cached.tokens))(*cached.tokens)
            check(lib.jenga_kv_free(self.h, g, _sp(page), 1, cached.key, cached.parent_key, toks,
                                    len(cached.tokens)))

    def pin(self, g: int, page, request: int) -> None:
        check(lib.jenga_kv_pin(self.h, g, _sp(page), request))

    def evict_lru_large_page(self) -> Optional[int]:
        out = C.c_uint32()
        check(lib.jenga_kv_evict_lru_large_page(self.h, C.byref(out)))
        return None if out.value == 0xFFFFFFFF else out.value

    def touch(self, g: int, page, step: int) -> None:
        check(lib.jenga_kv_touch(self.h, g, _sp(page), step))

    def set_prefix_length(self, g: int, page, length: int) -> None:
        check(lib.jenga_kv_set_prefix_length(self.h, g, _sp(page), length))

    def set_request_aware(self, on: bool) -> None:
        check(lib.jenga_kv_set_request_aware(self.h, 1 if on else 0))

    def record(self, g: int, page):
        st, a, la, pl = C.c_int(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib.jenga_kv_page_record(self.h, g, _sp(page), C.byref(st), C.byref(a), C.byref(la), C.byref(pl)))
        return {"state": st.value, "associated_request": a.value, "last_access": la.value,
                "prefix_length": pl.value}

    def cache_find(self, g: int, content: BlockContent) -> Optional[SmallPageId]:
        toks = (C.c_uint64 * max(1, len(content.tokens)))(*content.tokens)
        found, page = C.c_int(), _lib.SmallPage()
        check(lib.jenga_kv_cache_find(self.h, g, content.key, content.parent_key, toks, len(content.tokens),
                                      C.byref(found), C.byref(page)))
        return SmallPageId(page.large, page.slot) if found.value else None

    def group_counts(self, g: int):
        u, e, m, o = (C.c_uint64() for _ in range(4))
        check(lib.jenga_kv_group_counts(self.h, g, C.byref(u), C.byref(e), C.byref(m), C.byref(o)))
        return {"used": u.value, "evictable": e.value, "empty": m.value, "owned_units": o.value}

    def cache_entries(self, g: int) -> int:
        n = C.c_uint64()
        check(lib.jenga_kv_cache_entries(self.h, g, C.byref(n)))
        return n.value

    def pool_free_pages(self) -> int:
        n = C.c_uint32()
        check(lib.jenga_kv_pool_free_pages(self.h, C.byref(n)))
        return n.value

    def fragmentation_report(self, g: int):
        u, e, s = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib.jenga_kv_fragmentation(self.h, g, C.byref(u), C.byref(e), C.byref(s)))
        return {"used_bytes": u.value, "evictable_bytes": e.value, "empty_stranded_bytes": s.value}

    def alloc_step_counts(self):
        arr = (C.c_uint64 * 6)()
        check(lib.jenga_kv_alloc_step_counts(self.h, arr))
        return list(arr)

    def check_invariants(self) -> None:
        check(lib.jenga_kv_check_invariants(self.h))


class PageLists:
    """Per-request page lists with the reference simulator's store_position
    semantics (simulator.cpp:217-327)."""

    def __init__(self, kv: KvAllocator, prefix_caching: bool = False):
        self.kv = kv
        self.h = C.c_void_p()
        check(lib.jenga_pages_create(kv.h, 1 if prefix_caching else 0, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            lib.jenga_pages_destroy(self.h)
            self.h = None

    def add_request(self, request: int) -> None:
        check(lib.jenga_pages_add_request(self.h, request))

    def append(self, request: int, token: int = 0, is_image: bool = False, image_ordinal: int = 0,
               now: int = 0) -> bool:
        rc = lib.jenga_pages_append(self.h, request, token, 1 if is_image else 0, image_ordinal, now)
        if rc == _lib.JENGA_ERR_OOM:
            return False
        check(rc)
        return True

    def append_batch(self, requests: Sequence[int], tokens=None, is_image=None, now: int = 0) -> int:
        """One decode step: append one position to each request, in order.
        Returns how many requests were appended before an OOM (== len on success)."""
        ids = np.ascontiguousarray(np.asarray(requests, dtype=np.uint64))
        tok = None if tokens is None else np.ascontiguousarray(np.asarray(tokens, dtype=np.uint64))
        img = None if is_image is None else np.ascontiguousarray(np.asarray(is_image, dtype=np.uint8))
        done = C.c_int()
        rc = lib.jenga_pages_append_batch(
            self.h, ids.ctypes.data_as(C.POINTER(C.c_uint64)), len(ids),
            None if tok is None else tok.ctypes.data_as(C.POINTER(C.c_uint64)),
            None if img is None else img.ctypes.data_as(C.POINTER(C.c_uint8)), now, C.byref(done))
        if rc not in (_lib.JENGA_OK, _lib.JENGA_ERR_OOM):
            check(rc)
        return done.value

    def store(self, request: int, g: int, pos: int, now: int = 0) -> bool:
        rc = lib.jenga_pages_store(self.h, request, g, pos, now)
        if rc == _lib.JENGA_ERR_OOM:
            return False
        check(rc)
        return True

    def release(self, request: int, allow_cache: bool = False, now: int = 0) -> None:
        check(lib.jenga_pages_release(self.h, request, 1 if allow_cache else 0, now))

    def admit(self, request: int, tokens, is_image=None, image_ordinals=None, now: int = 0) -> int:
        """Install the prompt; with prefix caching pin + adopt the longest cached
        prefix (reference admit / lookup_and_pin / adopt_lookup_result). Returns the hit."""
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.uint64))
        img = None if is_image is None else np.ascontiguousarray(np.asarray(is_image, dtype=np.uint8))
        ordn = None if image_ordinals is None else np.ascontiguousarray(np.asarray(image_ordinals, dtype=np.uint64))
        hit = C.c_uint64()
        rc = lib.jenga_pages_admit(self.h, request, t.ctypes.data_as(C.POINTER(C.c_uint64)),
                                   None if img is None else img.ctypes.data_as(C.POINTER(C.c_uint8)),
                                   None if ordn is None else ordn.ctypes.data_as(C.POINTER(C.c_uint64)),
                                   len(t), now, C.byref(hit))
        if rc == _lib.JENGA_ERR_OOM:  # vision / full_reuse stores ran out: release the request
            raise OutOfMemory(_lib.last_error())
        check(rc)
        return hit.value

    def prefill(self, request: int, budget: int, now: int = 0):
        """Store up to `budget` prompt positions. Returns (consumed, oom)."""
        c = C.c_uint64()
        rc = lib.jenga_pages_prefill(self.h, request, budget, now, C.byref(c))
        if rc == _lib.JENGA_ERR_OOM:
            return c.value, True
        check(rc)
        return c.value, False

    def restore_pending(self, request: int, g: int):
        has, page = C.c_int(), _lib.SmallPage()
        check(lib.jenga_pages_restore_pending(self.h, request, g, C.byref(has), C.byref(page)))
        return SmallPageId(page.large, page.slot) if has.value else None

    def finish_restore(self, request: int, g: int, now: int = 0) -> None:
        check(lib.jenga_pages_finish_restore(self.h, request, g, now))

    def take_checkpoint_copies(self, capacity: int = 4096):
        """Drain the queued Mamba checkpoint snapshots: list of dicts with
        request, group, ordinal, working (source) and checkpoint (destination)."""
        buf = (_lib.CheckpointCopyC * max(1, capacity))()
        out = []
        while True:
            n = C.c_int()
            check(lib.jenga_pages_take_checkpoint_copies(self.h, buf, capacity, C.byref(n)))
            for i in range(n.value):
                c = buf[i]
                out.append({"request": c.request, "group": c.group, "ordinal": c.ordinal,
                            "working": SmallPageId(c.working.large, c.working.slot),
                            "checkpoint": SmallPageId(c.checkpoint.large, c.checkpoint.slot)})
            if n.value < capacity:
                return out

    def set_fix_mamba_restore(self, on: bool) -> None:
        check(lib.jenga_pages_set_fix_mamba_restore(self.h, 1 if on else 0))

    def set_defer_window_free(self, request: int, on: bool) -> None:
        check(lib.jenga_pages_set_defer_window_free(self.h, request, 1 if on else 0))

    def apply_window_free(self, request: int, now: int = 0) -> None:
        check(lib.jenga_pages_apply_window_free(self.h, request, now))

    ON_DEMAND, FULL_REUSE = 0, 1

    def set_vision_mode(self, mode) -> None:
        """reference EngineConfig::vision_mode: 0/"on_demand", 1/"full_reuse"."""
        if isinstance(mode, str):
            mode = {"on_demand": 0, "full_reuse": 1}[mode]
        check(lib.jenga_pages_set_vision_mode(self.h, int(mode)))

    def rollback_newest(self, request: int, g: int, count: int, now: int = 0) -> None:
        """reference rollback_newest (simulator.cpp:568-597)."""
        check(lib.jenga_pages_rollback_newest(self.h, request, g, count, now))

    def speculative_decode(self, request: int, propose_k: int, accepted: int, target_tokens=None,
                           n_target: Optional[int] = None, now: int = 0) -> bool:
        """reference speculative_decode_one (simulator.cpp:600-640). False on OOM."""
        if n_target is None:
            n_target = max(accepted, 1) if target_tokens is None else len(target_tokens)
        tok = None
        if target_tokens is not None:
            tok = np.ascontiguousarray(np.asarray(target_tokens, dtype=np.uint64))
        rc = lib.jenga_pages_speculative_decode(self.h, request, propose_k, accepted,
                                                None if tok is None else tok.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                n_target, now)
        if rc == _lib.JENGA_ERR_OOM:
            return False
        check(rc)
        return True

    def is_draft_group(self, g: int) -> bool:
        v = C.c_int()
        check(lib.jenga_pages_is_draft_group(self.h, g, C.byref(v)))
        return bool(v.value)

    def seq_len(self, request: int) -> int:
        n = C.c_uint64()
        check(lib.jenga_pages_seq_len(self.h, request, C.byref(n)))
        return n.value

    def group_state(self, request: int, g: int):
        vals = [C.c_uint64() for _ in range(4)]
        hw, wp = C.c_int(), _lib.SmallPage()
        check(lib.jenga_pages_group_state(self.h, request, g, *[C.byref(v) for v in vals], C.byref(hw), C.byref(wp)))
        return {"stored": vals[0].value, "num_blocks": vals[1].value, "freed_blocks": vals[2].value,
                "held_tokens": vals[3].value,
                "working_page": SmallPageId(wp.large, wp.slot) if hw.value else None}

    def blocks(self, request: int, g: int):
        n = C.c_uint64()
        check(lib.jenga_pages_blocks(self.h, request, g, None, None, 0, C.byref(n)))
        cap = n.value
        pages = (_lib.SmallPage * max(1, cap))()
        live = (C.c_uint8 * max(1, cap))()
        check(lib.jenga_pages_blocks(self.h, request, g, pages, live, cap, C.byref(n)))
        return [(SmallPageId(pages[i].large, pages[i].slot), bool(live[i])) for i in range(cap)]

    def pack_csr(self, g: int, requests: Sequence[int], max_blocks: int = 0):
        """CSR page lists (numpy) for jenga_build_block_tables; max_blocks > 0
        rejects a request longer than that block-table width."""
        req = np.ascontiguousarray(np.asarray(requests, dtype=np.uint64))
        nreq = len(req)
        offsets = np.zeros(nreq + 1, dtype=np.int32)
        rp = req.ctypes.data_as(C.POINTER(C.c_uint64))
        check(lib.jenga_pages_pack_csr(self.h, g, rp, nreq, max_blocks, 0,
                                       offsets.ctypes.data_as(C.POINTER(C.c_int32)), None, None, None))
        total = int(offsets[-1])
        pages = np.zeros((max(1, total), 2), dtype=np.uint32)
        first_live = np.zeros(nreq, dtype=np.int32)
        n_stored = np.zeros(nreq, dtype=np.int32)
        check(lib.jenga_pages_pack_csr(self.h, g, rp, nreq, max_blocks, pages.shape[0],
                                       offsets.ctypes.data_as(C.POINTER(C.c_int32)),
                                       pages.ctypes.data_as(C.POINTER(_lib.SmallPage)),
                                       first_live.ctypes.data_as(C.POINTER(C.c_int32)),
                                       n_stored.ctypes.data_as(C.POINTER(C.c_int32))))
        return offsets, pages[:total], first_live, n_stored


class TableMirror:
    """Host mirror of one group's device block table (jenga_table_mirror):
    pack() diffs the page lists against what the device holds and writes only
    the changed entries (+ seq_lens / newest slots) into a delta buffer that
    jenga_upload_page_list_deltas applies on the device."""

    HEADER = 32

    def __init__(self, pages: PageLists, g: int, max_batch: int, max_blocks: int):
        self.pages, self.g, self.max_batch, self.max_blocks = pages, g, max_batch, max_blocks
        self.h = C.c_void_p()
        check(lib.jenga_table_mirror_create(pages.h, g, max_batch, max_blocks, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            lib.jenga_table_mirror_destroy(self.h)
            self.h = None

    @staticmethod
    def buffer_bytes(max_batch: int, max_blocks: int) -> int:
        return int(lib.jenga_delta_buffer_bytes(max_batch, max_blocks))

    @staticmethod
    def delta_bytes(rows: int, records: int) -> int:
        return int(lib.jenga_delta_bytes(rows, records))

    @staticmethod
    def ack_ptr(buf_ptr: int) -> int:
        """Where the applying launch acknowledges the buffer (header word 4)."""
        return buf_ptr + 16

    def reset(self) -> None:
        check(lib.jenga_table_mirror_reset(self.h))

    def pack(self, requests, buf_ptr: int, capacity: int):
        """Diff rows requests[i] into the buffer at buf_ptr; returns (bytes used, records)."""
        req = np.ascontiguousarray(np.asarray(requests, dtype=np.uint64))
        used = C.c_size_t()
        nrec = C.c_int()
        check(lib.jenga_pages_pack_deltas(self.h, req.ctypes.data_as(C.POINTER(C.c_uint64)), len(req),
                                          C.c_void_p(buf_ptr), capacity, C.byref(used), C.byref(nrec)))
        return int(used.value), int(nrec.value)

    @staticmethod
    def seq_lens_view(buf: np.ndarray, rows: int) -> np.ndarray:
        """int32 seq_lens of the last pack, inside the (uint8) buffer."""
        o = TableMirror.HEADER + 8 * rows
        return buf[o:o + 4 * rows].view(np.int32)

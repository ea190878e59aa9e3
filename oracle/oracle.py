"""ctypes front-end of the oracles (TEST INFRASTRUCTURE ONLY).

COracle  — the plain-C restatement (oracle/jenga_oracle.c).
RefLib   — the reference library itself (oracle/_ref/libjenga_ref.so, built
           from /root/reference sources); absent on machines where the
           reference was never built (callers skip).
"""
from __future__ import annotations

import ctypes as C
import json
from functools import lru_cache
from pathlib import Path
from typing import List, Optional, Sequence

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"

F32, BF16, F16 = 0, 1, 2
FULL, SWA, MAMBA, CROSS, VISION = 0, 1, 2, 3, 4

_u32, _u64, _i32, _i64, _int, _dbl, _p = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_int, C.c_double, C.c_void_p


def _np(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(C.c_void_p)


class COracle:
    def __init__(self, path: Path):
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.orc_small_page_size.argtypes = [_u64, _u64, _u64, C.POINTER(_u64)]
        L.orc_lcm_page_size.argtypes = [C.POINTER(_u64), _int, C.POINTER(_u64)]
        L.orc_global_page_index.argtypes = [_u32, _u32, _u32, C.POINTER(_u64)]
        L.orc_address_of.argtypes = [_u64, _u64, _u64, _u32, _u32, _u32, _u32, _u32, C.POINTER(_u64), C.POINTER(_u64)]
        L.orc_view_address.argtypes = [_u64, _u64, _u32, _u32, _u32, _u32, _u32, C.POINTER(_u64), C.POINTER(_u64)]
        L.orc_build_block_tables.argtypes = [_p, _p, _p, _p, _int, _u32, _u32, _int, _p, _p, _p]
        L.orc_reshape_and_cache.argtypes = [_p, _u64, _u64, _int, _int, _int, _int, _p, _p, _i64, _p, _int]
        L.orc_paged_decode.argtypes = [_p, _u64, _u64, _int, _int, _i64, _p, _p, _p, _p, _int, _int, _int, _int,
                                       _int, _int, _dbl, _dbl, _int]
        L.orc_paged_prefill.argtypes = [_p, _u64, _u64, _int, _int, _i64, _p, _p, _p, _p, _p, _int, _int, _int,
                                        _int, _int, _int, _dbl, _dbl]
        L.orc_mamba_gather.argtypes = [_p, _u64, _u64, _u64, _p, _int, _p]
        L.orc_mamba_scatter.argtypes = [_p, _u64, _u64, _u64, _p, _int, _p]
        L.orc_page_copy.argtypes = [_p, _u64, _p, _p, _int]
        L.orc_mamba_update.argtypes = [_p, _u64, _u64, _u64, _u32, _p, _int, C.c_float]
        for f in (L.orc_token_rows_scatter, L.orc_token_rows_gather):
            f.argtypes = [_p, _u64, _u64, _u64, _u32, _u32, _u32, _p, _u64, C.c_int64, _p, _int]

    @staticmethod
    def _ok(rc):
        if rc != 0:
            raise RuntimeError(f"oracle status {rc}")

    def small_page_size(self, bptl, layers, tpp):
        o = _u64()
        self._ok(self.lib.orc_small_page_size(bptl, layers, tpp, C.byref(o)))
        return o.value

    def lcm_page_size(self, smalls: Sequence[int]):
        arr = (_u64 * len(smalls))(*smalls)
        o = _u64()
        self._ok(self.lib.orc_lcm_page_size(arr, len(smalls), C.byref(o)))
        return o.value

    def global_page_index(self, large, slot, slots_per_large):
        o = _u64()
        self._ok(self.lib.orc_global_page_index(large, slot, slots_per_large, C.byref(o)))
        return o.value

    def address_of(self, large_bytes, small_bytes, per_layer, num_layers, spl, layer, large, slot):
        b, e = _u64(), _u64()
        self._ok(self.lib.orc_address_of(large_bytes, small_bytes, per_layer, num_layers, spl, layer, large, slot,
                                         C.byref(b), C.byref(e)))
        return b.value, e.value

    def view_address(self, small_bytes, per_layer, num_layers, spl, layer, large, slot):
        b, e = _u64(), _u64()
        self._ok(self.lib.orc_view_address(small_bytes, per_layer, num_layers, spl, layer, large, slot,
                                           C.byref(b), C.byref(e)))
        return b.value, e.value

    def build_block_tables(self, offsets, pages, first_live, n_stored, slots_per_large, tpp, max_blocks):
        batch = len(offsets) - 1
        offsets, po = _np(offsets, np.int32)
        pages, pp = _np(np.asarray(pages).reshape(-1, 2) if len(pages) else np.zeros((1, 2)), np.uint32)
        first_live, fp = _np(first_live, np.int32)
        n_stored, npp = _np(n_stored, np.int32)
        table = np.zeros((batch, max_blocks), dtype=np.int32)
        slots = np.zeros(batch, dtype=np.int64)
        seq = np.zeros(batch, dtype=np.int32)
        self._ok(self.lib.orc_build_block_tables(po, pp, fp, npp, batch, slots_per_large, tpp, max_blocks,
                                                 table.ctypes.data_as(_p), slots.ctypes.data_as(_p),
                                                 seq.ctypes.data_as(_p)))
        return table, slots, seq

    def reshape_and_cache(self, arena: np.ndarray, view, dtype, hkv, d, tpp, key: np.ndarray, value: np.ndarray,
                          slots):
        slots, sp = _np(slots, np.int64)
        key = np.ascontiguousarray(key)
        value = np.ascontiguousarray(value)
        tstride = hkv * d
        self._ok(self.lib.orc_reshape_and_cache(arena.ctypes.data_as(_p), view[0], view[1], dtype, hkv, d, tpp,
                                                key.ctypes.data_as(_p), value.ctypes.data_as(_p), tstride, sp,
                                                len(slots)))

    def paged_decode(self, arena: np.ndarray, view, kind, dtype, window, q: np.ndarray, table, seq_lens, hq, hkv, d,
                     tpp, scale, softcap=0.0, nthreads=1) -> np.ndarray:
        table, tp = _np(table, np.int32)
        seq_lens, sp = _np(seq_lens, np.int32)
        q = np.ascontiguousarray(q)
        batch = table.shape[0]
        out = np.zeros((batch, hq, d), dtype=np.float64)
        self._ok(self.lib.orc_paged_decode(arena.ctypes.data_as(_p), view[0], view[1], kind, dtype, int(window),
                                           q.ctypes.data_as(_p), out.ctypes.data_as(_p), tp, sp, batch,
                                           table.shape[1], hq, hkv, d, tpp, float(scale), float(softcap),
                                           int(nthreads)))
        return out

    def paged_prefill(self, arena: np.ndarray, view, kind, dtype, window, q: np.ndarray, cu_q, table, seq_lens, hq,
                      hkv, d, tpp, scale, softcap=0.0) -> np.ndarray:
        cu, cp = _np(cu_q, np.int32)
        table, tp = _np(table, np.int32)
        seq_lens, sp = _np(seq_lens, np.int32)
        q = np.ascontiguousarray(q)
        out = np.zeros((int(cu[-1]), hq, d), dtype=np.float64)
        self._ok(self.lib.orc_paged_prefill(arena.ctypes.data_as(_p), view[0], view[1], kind, dtype, int(window),
                                            q.ctypes.data_as(_p), out.ctypes.data_as(_p), cp, tp, sp, table.shape[0],
                                            table.shape[1], hq, hkv, d, tpp, float(scale), float(softcap)))
        return out

    def mamba_gather(self, arena, view, page_globals, batch):
        pg, pp = _np(page_globals, np.int64)
        dense = np.zeros((batch, view[2]), dtype=np.uint8)
        self._ok(self.lib.orc_mamba_gather(arena.ctypes.data_as(_p), view[0], view[1], view[2], pp, batch,
                                           dense.ctypes.data_as(_p)))
        return dense

    def mamba_scatter(self, arena, view, page_globals, dense):
        pg, pp = _np(page_globals, np.int64)
        dense = np.ascontiguousarray(dense, dtype=np.uint8)
        self._ok(self.lib.orc_mamba_scatter(arena.ctypes.data_as(_p), view[0], view[1], view[2], pp, len(pg),
                                            dense.ctypes.data_as(_p)))

    def mamba_update(self, arena, view, num_layers, page_globals, decay):
        pg, pp = _np(page_globals, np.int64)
        self._ok(self.lib.orc_mamba_update(arena.ctypes.data_as(_p), view[0], view[1], view[2], num_layers, pp,
                                           len(pg), C.c_float(decay)))

    def page_copy(self, arena, small_page_bytes, src, dst):
        s, sp = _np(src, np.int64)
        d, dp = _np(dst, np.int64)
        self._ok(self.lib.orc_page_copy(arena.ctypes.data_as(_p), small_page_bytes, sp, dp, len(s)))


    def token_rows_scatter(self, arena, view, ppl, piece, tpp, rows, slots):
        """view = (start_offset, page_stride, exec_page_size); rows uint8 [T, bytes]."""
        rows = np.ascontiguousarray(rows, dtype=np.uint8)
        sl, sp = _np(slots, np.int64)
        self._ok(self.lib.orc_token_rows_scatter(arena.ctypes.data_as(_p), view[0], view[2], view[1], tpp, ppl, piece,
                                                 rows.ctypes.data_as(_p), rows.shape[1], rows.shape[1], sp, len(sl)))

    def token_rows_gather(self, arena, view, ppl, piece, tpp, row_bytes, slots):
        sl, sp = _np(slots, np.int64)
        rows = np.zeros((len(sl), row_bytes), dtype=np.uint8)
        self._ok(self.lib.orc_token_rows_gather(arena.ctypes.data_as(_p), view[0], view[2], view[1], tpp, ppl, piece,
                                                rows.ctypes.data_as(_p), row_bytes, row_bytes, sp, len(sl)))
        return rows


class RefError(RuntimeError):
    pass


class RefLib:
    """The reference jenga_core built from /root/reference sources + shim."""

    def __init__(self, path: Path):
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        for name, args in {
            "ref_spec_from_json": [C.c_char_p, C.POINTER(_p)],
            "ref_small_page_size": [_p, _int, C.POINTER(_u64)],
            "ref_lcm_page_size": [_p, C.POINTER(_u64)],
            "ref_lcm_blowup_ratio": [_p, C.POINTER(_dbl)],
            "ref_needs_token": [_p, _int, _u64, _u64, _u64, C.POINTER(_int)],
            "ref_accessed_range": [_p, _int, _u64, _u64, C.POINTER(_u64), C.POINTER(_u64)],
            "ref_addr_create": [_p, C.POINTER(_p)],
            "ref_addr_info": [_p, _int, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u32)],
            "ref_addr_global": [_p, _int, _u32, _u32, C.POINTER(_u64)],
            "ref_addr_address_of": [_p, _int, _u32, _u32, _u32, C.POINTER(_u64), C.POINTER(_u64)],
            "ref_addr_view_address": [_p, _int, _u32, _u32, _u32, C.POINTER(_u64), C.POINTER(_u64)],
            "ref_addr_layer_view": [_p, _int, _u32, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)],
            "ref_addr_dump": [_p, _u32, C.c_char_p, _u64, C.POINTER(_u64)],
            "ref_kv_create": [_p, _u64, C.POINTER(_p)],
            "ref_kv_pool_info": [_p, C.POINTER(_u64), C.POINTER(_u32), C.POINTER(_u64)],
            "ref_kv_allocate": [_p, _int, _u64, C.POINTER(_u32), C.POINTER(_u32), C.POINTER(_int)],
            "ref_kv_free": [_p, _int, _u32, _u32, _int, _u64, _u64, C.POINTER(_u64), _u64],
            "ref_kv_pin": [_p, _int, _u32, _u32, _u64],
            "ref_kv_evict": [_p, C.POINTER(_u32)],
            "ref_kv_touch": [_p, _int, _u32, _u32, _u64],
            "ref_kv_set_prefix_length": [_p, _int, _u32, _u32, _u64],
            "ref_kv_set_request_aware": [_p, _int],
            "ref_kv_record": [_p, _int, _u32, _u32, C.POINTER(_int), C.POINTER(_u64), C.POINTER(_u64),
                              C.POINTER(_u64)],
            "ref_kv_cache_find": [_p, _int, _u64, _u64, C.POINTER(_u64), _u64, C.POINTER(_int), C.POINTER(_u32),
                                  C.POINTER(_u32)],
            "ref_kv_counts": [_p, _int, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64),
                              C.POINTER(_u32)],
            "ref_kv_fragmentation": [_p, _int, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)],
            "ref_kv_has_associated_empty": [_p, _int, _u64, C.POINTER(_int)],
            "ref_kv_check_invariants": [_p],
            "ref_sim_create": [_p, _u64, _u64, _int, _int, _p, _p, _p, _p, _p, _p, _p, C.POINTER(_p)],
            "ref_sim_create_ex": [_p, _u64, _u64, _int, _int, _p, _p, _p, _p, _p, _p, _p, _int, _p, _u32, _dbl,
                                  _u64, C.POINTER(_p)],
            "ref_spec_accept_draws": [_u64, _u64, _u32, _dbl, _int, _p],
            "ref_sim_draft_len": [_p, _u64, C.POINTER(_u64)],
            "ref_gen_multi_article": [_u32, _u32, _u64, _u64, _u64, _u64, _u64, _p, _p, _p, _p, _p, _int,
                                      C.POINTER(_int)],
            "ref_sim_step": [_p, C.POINTER(_u32)],
            "ref_sim_done": [_p],
            "ref_sim_request": [_p, _u64, C.POINTER(_int), C.POINTER(_u64), C.POINTER(_u64)],
            "ref_sim_tokens": [_p, _u64, _p, _p, _u64, C.POINTER(_u64)],
            "ref_sim_group_state": [_p, _u64, _int, _p, _p, _u64, C.POINTER(_u64), C.POINTER(_u64),
                                    C.POINTER(_u64), C.POINTER(_int), _p],
            "rpl_append_batch": [_p, _p, _int, _p, _u64],
            "rpl_group_state": [_p, _u64, _int, _p, _p, _u64, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)],
            "rpl_block_table": [_p, _p, _int, _p, _int, _int, _p],
            "rpl_resolve_views": [_p, _p, _int, _p, _int, C.POINTER(_u64)],
        }.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = _int
        for name in ("ref_spec_destroy", "ref_addr_destroy", "ref_kv_destroy", "ref_sim_destroy", "rpl_destroy"):
            getattr(L, name).argtypes = [_p]
            getattr(L, name).restype = None
        L.ref_sim_now.argtypes = [_p]
        L.ref_sim_now.restype = _u64
        L.ref_sim_allocator.argtypes = [_p]
        L.ref_sim_allocator.restype = _p
        L.rpl_create.argtypes = [_p]
        L.rpl_create.restype = _p

    def check(self, rc):
        if rc not in (0,):
            raise RefError(f"reference status {rc}: {self.lib.ref_last_error().decode()}")

    # thin object wrappers -------------------------------------------------
    def spec(self, spec_json: str) -> "RefSpec":
        return RefSpec(self, spec_json)


class RefSpec:
    def __init__(self, ref: RefLib, text: str):
        self.ref, self.L = ref, ref.lib
        self.h = _p()
        ref.check(self.L.ref_spec_from_json(text.encode(), C.byref(self.h)))
        self.json = json.loads(text)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_spec_destroy(self.h)
            self.h = None

    def small_page_size(self, g):
        o = _u64()
        self.ref.check(self.L.ref_small_page_size(self.h, g, C.byref(o)))
        return o.value

    def lcm_page_size(self):
        o = _u64()
        self.ref.check(self.L.ref_lcm_page_size(self.h, C.byref(o)))
        return o.value

    def lcm_blowup_ratio(self):
        o = _dbl()
        self.ref.check(self.L.ref_lcm_blowup_ratio(self.h, C.byref(o)))
        return o.value

    def needs_token(self, g, i, n, consumed=0):
        o = _int()
        self.ref.check(self.L.ref_needs_token(self.h, g, i, n, consumed, C.byref(o)))
        return bool(o.value)

    def accessed_range(self, g, prev, n):
        lo, hi = _u64(), _u64()
        self.ref.check(self.L.ref_accessed_range(self.h, g, prev, n, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def address_map(self) -> "RefAddressMap":
        return RefAddressMap(self)

    def kv(self, budget) -> "RefKv":
        return RefKv(self, budget)


class RefAddressMap:
    def __init__(self, spec: RefSpec):
        self.spec, self.L, self.ref = spec, spec.L, spec.ref
        self.h = _p()
        self.ref.check(self.L.ref_addr_create(spec.h, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_addr_destroy(self.h)
            self.h = None

    def info(self, g):
        a, b, c, d = _u64(), _u64(), _u64(), _u32()
        self.ref.check(self.L.ref_addr_info(self.h, g, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        return a.value, b.value, c.value, d.value

    def global_page_index(self, g, page):
        o = _u64()
        self.ref.check(self.L.ref_addr_global(self.h, g, page[0], page[1], C.byref(o)))
        return o.value

    def address_of(self, g, layer, page):
        b, e = _u64(), _u64()
        self.ref.check(self.L.ref_addr_address_of(self.h, g, layer, page[0], page[1], C.byref(b), C.byref(e)))
        return b.value, e.value

    def view_address(self, g, layer, page):
        b, e = _u64(), _u64()
        self.ref.check(self.L.ref_addr_view_address(self.h, g, layer, page[0], page[1], C.byref(b), C.byref(e)))
        return b.value, e.value

    def layer_view(self, g, layer):
        a, b, c = _u64(), _u64(), _u64()
        self.ref.check(self.L.ref_addr_layer_view(self.h, g, layer, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def dump(self, large_pages):
        n = _u64()
        self.ref.check(self.L.ref_addr_dump(self.h, large_pages, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self.ref.check(self.L.ref_addr_dump(self.h, large_pages, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()


class RefKv:
    def __init__(self, spec: RefSpec, budget: int, handle=None):
        self.spec, self.L, self.ref = spec, spec.L, spec.ref
        self.owned = handle is None
        self.h = _p(handle) if handle is not None else _p()
        if handle is None:
            self.ref.check(self.L.ref_kv_create(spec.h, budget, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and self.owned:
            self.L.ref_kv_destroy(self.h)
        self.h = None

    def pool_info(self):
        a, b, c = _u64(), _u32(), _u64()
        self.ref.check(self.L.ref_kv_pool_info(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def allocate(self, g, req):
        lg, sl, st = _u32(), _u32(), _int()
        rc = self.L.ref_kv_allocate(self.h, g, req, C.byref(lg), C.byref(sl), C.byref(st))
        if rc == 3:
            return None
        self.ref.check(rc)
        return (lg.value, sl.value), st.value

    def free(self, g, page, content=None):
        if content is None:
            return self.L.ref_kv_free(self.h, g, page[0], page[1], 0, 0, 0, None, 0)
        key, parent, toks = content
        arr = (_u64 * max(1, len(toks)))(*toks)
        return self.L.ref_kv_free(self.h, g, page[0], page[1], 1, key, parent, arr, len(toks))

    def pin(self, g, page, req):
        return self.L.ref_kv_pin(self.h, g, page[0], page[1], req)

    def evict(self):
        o = _u32()
        self.ref.check(self.L.ref_kv_evict(self.h, C.byref(o)))
        return None if o.value == 0xFFFFFFFF else o.value

    def touch(self, g, page, step):
        self.ref.check(self.L.ref_kv_touch(self.h, g, page[0], page[1], step))

    def set_prefix_length(self, g, page, n):
        self.ref.check(self.L.ref_kv_set_prefix_length(self.h, g, page[0], page[1], n))

    def set_request_aware(self, on):
        self.ref.check(self.L.ref_kv_set_request_aware(self.h, 1 if on else 0))

    def record(self, g, page):
        st, a, la, pl = _int(), _u64(), _u64(), _u64()
        self.ref.check(self.L.ref_kv_record(self.h, g, page[0], page[1], C.byref(st), C.byref(a), C.byref(la),
                                            C.byref(pl)))
        return {"state": st.value, "associated_request": a.value, "last_access": la.value, "prefix_length": pl.value}

    def cache_find(self, g, content):
        key, parent, toks = content
        arr = (_u64 * max(1, len(toks)))(*toks)
        f, lg, sl = _int(), _u32(), _u32()
        self.ref.check(self.L.ref_kv_cache_find(self.h, g, key, parent, arr, len(toks), C.byref(f), C.byref(lg),
                                                C.byref(sl)))
        return (lg.value, sl.value) if f.value else None

    def counts(self, g):
        u, e, m, o, pf = _u64(), _u64(), _u64(), _u64(), _u32()
        self.ref.check(self.L.ref_kv_counts(self.h, g, C.byref(u), C.byref(e), C.byref(m), C.byref(o), C.byref(pf)))
        return {"used": u.value, "evictable": e.value, "empty": m.value, "owned_units": o.value,
                "pool_free": pf.value}

    def fragmentation(self, g):
        u, e, s = _u64(), _u64(), _u64()
        self.ref.check(self.L.ref_kv_fragmentation(self.h, g, C.byref(u), C.byref(e), C.byref(s)))
        return {"used_bytes": u.value, "evictable_bytes": e.value, "empty_stranded_bytes": s.value}

    def has_associated_empty(self, g, req):
        o = _int()
        self.ref.check(self.L.ref_kv_has_associated_empty(self.h, g, req, C.byref(o)))
        return bool(o.value)

    def check_invariants(self):
        self.ref.check(self.L.ref_kv_check_invariants(self.h))


class RefPageLists:
    """rpl_*: restated store_position over the reference KvAllocator."""

    def __init__(self, kv: RefKv):
        self.kv, self.L, self.ref = kv, kv.L, kv.ref
        self.h = self.L.rpl_create(kv.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.rpl_destroy(self.h)
            self.h = None

    def append_batch(self, ids, is_image=None, now=0) -> bool:
        ids_a, ip = _np(ids, np.uint64)
        img = None
        if is_image is not None:
            img_a, img = _np(is_image, np.uint8)
        rc = self.L.rpl_append_batch(self.h, ip, len(ids_a), img, now)
        if rc == 3:
            return False
        self.ref.check(rc)
        return True

    def group_state(self, rid, g):
        n, st, fr = _u64(), _u64(), _u64()
        self.ref.check(self.L.rpl_group_state(self.h, rid, g, None, None, 0, C.byref(n), C.byref(st), C.byref(fr)))
        pages = np.zeros((max(1, n.value), 2), dtype=np.uint32)
        live = np.zeros(max(1, n.value), dtype=np.uint8)
        self.ref.check(self.L.rpl_group_state(self.h, rid, g, pages.ctypes.data_as(_p), live.ctypes.data_as(_p),
                                              n.value, C.byref(n), C.byref(st), C.byref(fr)))
        return pages[: n.value], live[: n.value].astype(bool), st.value, fr.value

    def block_table(self, addr: RefAddressMap, g, ids, max_blocks):
        ids_a, ip = _np(ids, np.uint64)
        table = np.zeros((len(ids_a), max_blocks), dtype=np.int32)
        self.ref.check(self.L.rpl_block_table(self.h, addr.h, g, ip, len(ids_a), max_blocks, table.ctypes.data_as(_p)))
        return table

    def resolve_views(self, addr: RefAddressMap, g, ids):
        ids_a, ip = _np(ids, np.uint64)
        o = _u64()
        self.ref.check(self.L.rpl_resolve_views(self.h, addr.h, g, ip, len(ids_a), C.byref(o)))
        return o.value


def multi_article_trace(ref: RefLib, articles=4, questions=3, article_tokens=4000, question_tokens=50,
                        output_tokens=20, spacing=200, seed=0):
    """The reference trace generator (trace.cpp:144-169) as request dicts."""
    cap = articles * questions
    ids = np.zeros(cap, np.uint64)
    arr = np.zeros(cap, np.uint64)
    outs = np.zeros(cap, np.uint64)
    grp = np.zeros(cap, np.int32)
    seg = np.zeros((cap, 2), np.uint64)
    n = _int()
    ref.check(ref.lib.ref_gen_multi_article(articles, questions, article_tokens, question_tokens, output_tokens,
                                            spacing, seed, ids.ctypes.data_as(_p), arr.ctypes.data_as(_p),
                                            outs.ctypes.data_as(_p), grp.ctypes.data_as(_p),
                                            seg.ctypes.data_as(_p), cap, C.byref(n)))
    return [{"id": int(ids[i]), "arrival": int(arr[i]), "output": int(outs[i]), "prefix_group": int(grp[i]),
             "segments": [[0, int(seg[i, 0])], [0, int(seg[i, 1])]]} for i in range(n.value)]


def spec_accept_draws(ref, seed, rid, propose_k, acceptance, n):
    """The reference's per-request acceptance draws (simulator.cpp:44-52, 109)."""
    out = np.zeros(n, dtype=np.uint64)
    ref.lib.ref_spec_accept_draws(seed, rid, propose_k, float(acceptance), n, out.ctypes.data_as(_p))
    return [int(x) for x in out]


class RefSim:
    """The reference SimEngine (stepped), page lists read back via the shim."""

    def __init__(self, spec: RefSpec, budget, chunk, prefix_caching, requests: List[dict], vision_mode=0,
                 draft: "RefSpec" = None, propose_k=4, acceptance=0.7, seed=0):
        self.spec, self.L, self.ref = spec, spec.L, spec.ref
        ids = np.array([r["id"] for r in requests], dtype=np.uint64)
        arr = np.array([r.get("arrival", 0) for r in requests], dtype=np.uint64)
        outs = np.array([r.get("output", 1) for r in requests], dtype=np.uint64)
        segc = np.array([len(r["segments"]) for r in requests], dtype=np.int32)
        segi = np.array([int(s[0]) for r in requests for s in r["segments"]] or [0], dtype=np.int32)
        segt = np.array([int(s[1]) for r in requests for s in r["segments"]] or [0], dtype=np.uint64)
        grp = np.array([r.get("prefix_group", -1) for r in requests], dtype=np.int32)
        self._keep = (ids, arr, outs, segc, segi, segt, grp)
        self.h = _p()
        self.ref.check(self.L.ref_sim_create_ex(spec.h, budget, chunk, 1 if prefix_caching else 0, len(ids),
                                                ids.ctypes.data_as(_p), arr.ctypes.data_as(_p),
                                                outs.ctypes.data_as(_p), segc.ctypes.data_as(_p),
                                                segi.ctypes.data_as(_p), segt.ctypes.data_as(_p),
                                                grp.ctypes.data_as(_p), int(vision_mode),
                                                None if draft is None else draft.h, propose_k, float(acceptance),
                                                seed, C.byref(self.h)))
        self._draft = draft

    def draft_len(self, rid):
        o = _u64()
        self.ref.check(self.L.ref_sim_draft_len(self.h, rid, C.byref(o)))
        return o.value

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_sim_destroy(self.h)
            self.h = None

    def step(self):
        o = _u32()
        self.ref.check(self.L.ref_sim_step(self.h, C.byref(o)))
        return o.value

    def done(self):
        return bool(self.L.ref_sim_done(self.h))

    def now(self):
        return self.L.ref_sim_now(self.h)

    def request(self, rid):
        ph, sl, co = _int(), _u64(), _u64()
        self.ref.check(self.L.ref_sim_request(self.h, rid, C.byref(ph), C.byref(sl), C.byref(co)))
        return {"phase": ph.value, "seq_len": sl.value, "consumed": co.value}

    def tokens(self, rid):
        n = _u64()
        self.ref.check(self.L.ref_sim_tokens(self.h, rid, None, None, 0, C.byref(n)))
        t = np.zeros(max(1, n.value), dtype=np.uint64)
        im = np.zeros(max(1, n.value), dtype=np.uint8)
        self.ref.check(self.L.ref_sim_tokens(self.h, rid, t.ctypes.data_as(_p), im.ctypes.data_as(_p), n.value,
                                             C.byref(n)))
        return t[: n.value], im[: n.value]

    def group_state(self, rid, g):
        n, st, fr, hw = _u64(), _u64(), _u64(), _int()
        w = np.zeros(2, dtype=np.uint32)
        self.ref.check(self.L.ref_sim_group_state(self.h, rid, g, None, None, 0, C.byref(n), C.byref(st), C.byref(fr),
                                                  C.byref(hw), w.ctypes.data_as(_p)))
        pages = np.zeros((max(1, n.value), 2), dtype=np.uint32)
        live = np.zeros(max(1, n.value), dtype=np.uint8)
        self.ref.check(self.L.ref_sim_group_state(self.h, rid, g, pages.ctypes.data_as(_p), live.ctypes.data_as(_p),
                                                  n.value, C.byref(n), C.byref(st), C.byref(fr), C.byref(hw),
                                                  w.ctypes.data_as(_p)))
        return {"pages": pages[: n.value], "live": live[: n.value].astype(bool), "stored": st.value,
                "freed": fr.value, "working": tuple(w) if hw.value else None}


@lru_cache(maxsize=1)
def c_oracle() -> COracle:
    p = REF_DIR / "liboracle.so"
    if not p.exists():
        from .build_oracle import build_c_oracle
        build_c_oracle()
    return COracle(p)


@lru_cache(maxsize=1)
def ref_lib() -> Optional[RefLib]:
    p = REF_DIR / "libjenga_ref.so"
    if not p.exists():
        try:
            from .build_oracle import build_reference
            if build_reference() is None:
                return None
        except Exception:
            return None
    return RefLib(p)

"""Shared builders for the GPU parity tests: a DecodeEngine filled through the
product path (host allocator -> device tables -> reshape_and_cache) and the
oracle's view of the same arena."""
from __future__ import annotations

import numpy as np
import torch

from oracle.oracle import BF16, F16, F32
from paper_2503_18292_b200 import ops
from paper_2503_18292_b200.engine import DecodeEngine
from paper_2503_18292_b200.geometry import GroupGeometry, ModelGeometry

ORC_DTYPE = {torch.float32: F32, torch.bfloat16: BF16, torch.float16: F16}
TOL = {torch.float32: 1e-5, torch.bfloat16: 1e-2, torch.float16: 5e-3}


def make_engine(geom: ModelGeometry, lens, seed=0, headroom_pages=8, poison=True, image_flags=None,
                defer_window=False):
    """Append tokens (interleaved, seeded order per 16-position chunk) until
    each request reaches lens[r]; returns the engine with tables synced."""
    spec = geom.spec()
    from paper_2503_18292_b200 import AddressMap
    addr = AddressMap(spec)
    lcm = addr.large_page_bytes()
    # pages needed per group (upper bound), in large pages
    need = 0
    for g, gg in enumerate(geom.groups):
        tpp = spec.groups[g].tokens_per_page
        spl = addr.slots_per_large(g)
        blocks = sum((n + tpp - 1) // tpp + 1 for n in lens)
        need += (blocks + spl - 1) // spl + len(lens)
    max_tokens = max(max(lens), 1) + 32
    eng = DecodeEngine(geom, need + headroom_pages, len(lens), max_tokens)
    if poison:
        eng.arena.tensor().fill_(0xFF)  # NaN in every float format: masked rows must never leak
    ids = list(range(100, 100 + len(lens)))
    eng.add_requests(ids)
    if defer_window:  # prefill chunks: keep out-of-window blocks until attention ran
        for r in ids:
            eng.pages.set_defer_window_free(r, True)
    rng = np.random.default_rng(seed)
    cur = [0] * len(lens)
    pos = 0
    while any(c < n for c, n in zip(cur, lens)):
        active = [i for i in range(len(lens)) if cur[i] < lens[i]]
        if pos % 16 == 0:
            order = list(rng.permutation(active))
        order = [i for i in order if cur[i] < lens[i]] or active
        img = None
        if image_flags is not None:
            img = [image_flags[i](cur[i] + 1) for i in order]
        done = eng.append([ids[i] for i in order], is_image=img)
        assert done == len(order)
        for i in order:
            cur[i] += 1
        pos += 1
    eng.sync_tables()
    torch.cuda.synchronize()
    return eng, ids


def fill_group_kv(eng: DecodeEngine, g: int, layers, seed=0, all_live=False):
    """Write random K/V for every live stored ordinal of group g through the
    product slot_mapping + reshape_and_cache kernels (SWA: the window only,
    unless all_live).  Returns (req, ord, K, V, slots)."""
    t = eng.tables[g]
    gg = t.geom
    B = len(eng.requests)
    n = t.h_n_stored[:B].numpy().astype(np.int64)
    lo = np.zeros(B, dtype=np.int64)
    if all_live:
        tpp = eng.spec.groups[g].tokens_per_page
        lo = np.array([eng.pages.group_state(r, g)["freed_blocks"] * tpp for r in eng.requests], dtype=np.int64)
    elif gg.window:
        lo = np.maximum(0, n - gg.window)
    req = np.concatenate([np.full(n[b] - lo[b], b, dtype=np.int32) for b in range(B)]) if n.sum() else \
        np.zeros(0, np.int32)
    ords = np.concatenate([np.arange(lo[b] + 1, n[b] + 1, dtype=np.int32) for b in range(B)]) if n.sum() else \
        np.zeros(0, np.int32)
    dev = eng.device
    req_d = torch.from_numpy(req).to(dev)
    ord_d = torch.from_numpy(ords).to(dev)
    slots = torch.empty(len(req), dtype=torch.int64, device=dev)
    if len(req):
        ops.slot_mapping(t.block_table, t.max_blocks, req_d, ord_d, eng.spec.groups[g].tokens_per_page, slots)
    gen = torch.Generator(device=dev).manual_seed(seed)
    out = []
    for layer in layers:
        K = torch.randn((len(req), gg.num_kv_heads, gg.head_dim), generator=gen, device=dev).to(gg.dtype)
        V = torch.randn((len(req), gg.num_kv_heads, gg.head_dim), generator=gen, device=dev).to(gg.dtype)
        if len(req):
            eng.write_kv(g, layer, K, V, slots)
        out.append((K, V))
    torch.cuda.synchronize()
    return req, ords, out, slots


def arena_host(eng: DecodeEngine) -> np.ndarray:
    return eng.arena.tensor().cpu().numpy()


def rel_err(got: np.ndarray, want: np.ndarray) -> float:
    denom = max(np.abs(want).max(), 1e-30)
    return float(np.abs(got - want).max() / denom)

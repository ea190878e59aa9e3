"""SURVEY §8(f) rows 3-4 on the device, checked against the oracle:

* vision-embedding pages, on_demand: embeddings scattered into the vision
  group's own pages, read back chunk by chunk while prefill frees consumed
  pages (simulator.cpp:453-464, 525-542);
* vision-embedding pages, full_reuse: embeddings parked in the token's own
  unwritten KV bytes survive every earlier chunk's KV
  write, and the final KV equals a plain reshape_and_cache;
* speculative decoding: draft and target groups in one LCM pool; after the
  draft rollback (simulator.cpp:568-597) freed draft pages are reused by the
  target, and the multi-token verify attention (prefill kernel, chunk =
  accepted tokens) still matches the oracle for both models.
All byte movement is bit-exact; attention within the bf16 tolerance."""
import numpy as np
import pytest
import torch

from gpu_scenarios import ORC_DTYPE, TOL, arena_host, fill_group_kv, make_engine, rel_err
from paper_2503_18292_b200 import LayerKind, ops
from paper_2503_18292_b200.engine import DecodeEngine
from paper_2503_18292_b200.geometry import GroupGeometry, ModelGeometry

pytestmark = pytest.mark.gpu

TPP = 16


def slots_of(eng, g, req_idx, ords):
    t = eng.tables[g]
    req = torch.as_tensor(np.asarray(req_idx, dtype=np.int32), device=eng.device)
    o = torch.as_tensor(np.asarray(ords, dtype=np.int32), device=eng.device)
    slots = torch.empty(len(req_idx), dtype=torch.int64, device=eng.device)
    if len(req_idx):
        ops.slot_mapping(t.block_table, t.max_blocks, req, o, eng.spec.groups[g].tokens_per_page, slots)
    return slots


def prompts(n_req, layout, seed=0):
    """layout[r] = [(is_image, n), ...] -> tokens, is_image, image ordinals."""
    rng = np.random.default_rng(seed)
    out = []
    for r in range(n_req):
        toks, img, ordn = [], [], []
        for s, (is_image, n) in enumerate(layout[r]):
            ordinal = int(rng.integers(1, 1 << 40)) if is_image else 0
            toks += [int(x) for x in rng.integers(1, 1 << 40, n)]
            img += [bool(is_image)] * n
            ordn += [ordinal] * n
        out.append((toks, img, ordn))
    return out


def make(geom, n_req, pages, max_tokens, mode):
    eng = DecodeEngine(geom, pages, n_req, max_tokens)
    eng.arena.tensor().fill_(0xFF)
    eng.pages.set_vision_mode(mode)
    ids = list(range(50, 50 + n_req))
    eng.add_requests(ids)
    return eng, ids


def test_vision_on_demand_pages(orc):
    geom = ModelGeometry("vlm", [
        GroupGeometry("self", LayerKind.kFullAttention, 2, 8, 32, 128, torch.bfloat16, TPP),
        GroupGeometry("cross", LayerKind.kCrossAttention, 1, 8, 32, 128, torch.bfloat16, TPP),
        GroupGeometry("vision", LayerKind.kVisionEmbedding, 1, tokens_per_page=TPP, state_bytes=2560)])
    layout = [[(0, 5), (1, 70), (0, 9)], [(0, 3), (1, 33), (0, 4), (1, 20), (0, 6)]]
    eng, ids = make(geom, 2, 64, 200, mode=0)
    ps = prompts(2, layout, seed=1)
    for rid, (toks, img, ordn) in zip(ids, ps):
        assert eng.pages.admit(rid, toks, img, ordn) == 0
    VG = 2
    eng.sync_tables()
    n_img = [sum(p[1]) for p in ps]
    assert [eng.pages.group_state(r, VG)["stored"] for r in ids] == n_img
    # encoder output -> the vision group's pages (ordinal k = k-th image token)
    req_idx = np.concatenate([np.full(n, i, np.int32) for i, n in enumerate(n_img)])
    ords = np.concatenate([np.arange(1, n + 1, dtype=np.int32) for n in n_img])
    slots = slots_of(eng, VG, req_idx, ords)
    gen = torch.Generator(device=eng.device).manual_seed(3)
    emb = torch.randint(0, 256, (len(ords), 2560), generator=gen, device=eng.device, dtype=torch.uint8)
    before = arena_host(eng)
    view = eng.view(VG, 0)
    ops.token_rows_scatter(eng.arena, view, 1, 1, 2560, TPP, emb, slots)
    torch.cuda.synchronize()
    orc.token_rows_scatter(before, tuple(view), 1, 2560, TPP, emb.cpu().numpy(), slots.cpu().numpy())
    np.testing.assert_array_equal(arena_host(eng), before)
    emb_h = emb.cpu().numpy()
    base = np.concatenate([[0], np.cumsum(n_img)])
    # chunked prefill: consume embeddings chunk by chunk; consumed pages go back
    used0 = eng.kv.group_counts(VG)["used"]
    consumed = [0, 0]
    while any(c < len(p[0]) for c, p in zip(consumed, ps)):
        for i, rid in enumerate(ids):
            toks, img, _ = ps[i]
            c0 = consumed[i]
            if c0 >= len(toks):
                continue
            c1 = min(c0 + 16, len(toks))
            k0 = sum(img[:c0])
            k1 = sum(img[:c1])
            if k1 > k0:  # the chunk's embeddings, read through the live page table
                got = torch.empty((k1 - k0, 2560), dtype=torch.uint8, device=eng.device)
                ops.token_rows_gather(eng.arena, view, 1, 1, 2560, TPP, got,
                                      slots_of(eng, VG, [i] * (k1 - k0), range(k0 + 1, k1 + 1)))
                np.testing.assert_array_equal(got.cpu().numpy(), emb_h[base[i] + k0: base[i] + k1])
            n, oom = eng.pages.prefill(rid, c1 - c0)
            assert n == c1 - c0 and not oom
            consumed[i] = c1
            # on-demand free: a page goes once all its embeddings are consumed
            held = eng.pages.group_state(rid, VG)["held_tokens"]
            assert held == (n_img[i] - (k1 // TPP) * TPP if k1 < n_img[i] else 0), (i, k1, held)
        eng.sync_tables()
    assert all(eng.pages.group_state(r, VG)["held_tokens"] == 0 for r in ids)
    assert eng.kv.group_counts(VG)["used"] < used0
    eng.kv.check_invariants()


def test_vision_full_reuse_overlay(orc):
    """Embeddings overlay the token's own unwritten KV bytes: each chunk's KV
    write leaves every later token's parked embedding intact."""
    geom = ModelGeometry("llava", [
        GroupGeometry("self", LayerKind.kFullAttention, 2, 8, 32, 128, torch.bfloat16, TPP),
        GroupGeometry("window", LayerKind.kSlidingWindow, 1, 8, 32, 128, torch.bfloat16, TPP, window=32),
        GroupGeometry("vision", LayerKind.kVisionEmbedding, 1, tokens_per_page=TPP, state_bytes=6144)])
    layout = [[(0, 5), (1, 61), (0, 9)], [(0, 2), (1, 45), (0, 20)]]
    eng, ids = make(geom, 2, 64, 200, mode=1)
    ps = prompts(2, layout, seed=2)
    for rid, (toks, img, ordn) in zip(ids, ps):
        eng.pages.admit(rid, toks, img, ordn)
        assert eng.pages.group_state(rid, 0)["stored"] == len(toks)  # whole prompt up front
    eng.sync_tables()
    SG, L, HKV, D = 0, 2, 8, 128
    piece, ppl = D * 2, 2 * HKV
    img_pos = [[p + 1 for p, f in enumerate(ps[i][1]) if f] for i in range(2)]
    req_idx = np.concatenate([np.full(len(x), i, np.int32) for i, x in enumerate(img_pos)])
    ords = np.concatenate([np.asarray(x, np.int32) for x in img_pos])  # self stores every position
    slots = slots_of(eng, SG, req_idx, ords)
    gen = torch.Generator(device=eng.device).manual_seed(4)
    emb = torch.randint(0, 256, (len(ords), 6144), generator=gen, device=eng.device, dtype=torch.uint8)
    view0 = eng.view(SG, 0)
    want = arena_host(eng)
    ops.token_rows_scatter(eng.arena, view0, L, ppl, piece, TPP, emb, slots)
    torch.cuda.synchronize()
    orc.token_rows_scatter(want, tuple(view0), ppl, piece, TPP, emb.cpu().numpy(), slots.cpu().numpy())
    np.testing.assert_array_equal(arena_host(eng), want)
    emb_h = emb.cpu().numpy()
    lens = [len(p[0]) for p in ps]
    for c0 in range(0, max(lens), 16):
        for i, rid in enumerate(ids):
            if c0 >= lens[i]:
                continue
            c1 = min(c0 + 16, lens[i])
            sel = [k for k, pos in enumerate(img_pos[i]) if c0 < pos <= c1]
            off = sum(len(x) for x in img_pos[:i])
            if sel:  # the chunk's embeddings, as the LLM's input
                got = torch.empty((len(sel), 6144), dtype=torch.uint8, device=eng.device)
                ops.token_rows_gather(eng.arena, view0, L, ppl, piece, TPP, got, slots[[off + k for k in sel]])
                np.testing.assert_array_equal(got.cpu().numpy(), emb_h[[off + k for k in sel]])
            # then the chunk's KV overwrites those same bytes, layer by layer
            cs = slots_of(eng, SG, [i] * (c1 - c0), range(c0 + 1, c1 + 1))
            for layer in range(L):
                K = torch.randn((c1 - c0, HKV, D), generator=gen, device=eng.device).to(torch.bfloat16)
                V = torch.randn((c1 - c0, HKV, D), generator=gen, device=eng.device).to(torch.bfloat16)
                eng.write_kv(SG, layer, K, V, cs)
                orc.reshape_and_cache(want, tuple(eng.view(SG, layer)), ORC_DTYPE[torch.bfloat16], HKV, D, TPP,
                                      K.view(torch.int16).cpu().numpy(), V.view(torch.int16).cpu().numpy(),
                                      cs.cpu().numpy())
            n, oom = eng.pages.prefill(rid, c1 - c0)
            assert n == c1 - c0 and not oom
        # every not-yet-consumed embedding is still intact
        rest = [k for k in range(len(ords)) if ords[k] > c0 + 16]
        if rest:
            got = torch.empty((len(rest), 6144), dtype=torch.uint8, device=eng.device)
            ops.token_rows_gather(eng.arena, view0, L, ppl, piece, TPP, got, slots[rest])
            np.testing.assert_array_equal(got.cpu().numpy(), emb_h[rest])
    torch.cuda.synchronize()
    np.testing.assert_array_equal(arena_host(eng), want)  # KV == plain reshape_and_cache
    # prompt done: the deferred window frees ran (finish_prefill)
    for rid, n in zip(ids, lens):
        st = eng.pages.group_state(rid, 1)
        assert st["freed_blocks"] == max(0, (n - 32) // TPP)
    eng.kv.check_invariants()


def verify_attention(orc, eng, g, rows, new_ords):
    """Multi-token attention of each request's newest tokens (chunk = its
    new ordinals) through the prefill kernel, against the oracle."""
    t = eng.tables[g]
    gg = t.geom
    B = len(eng.requests)
    chunks = np.asarray(new_ords, dtype=np.int32)
    cu = np.zeros(B + 1, dtype=np.int32)
    cu[1:] = np.cumsum(chunks)
    T = int(cu[-1])
    if T == 0:
        return
    gen = torch.Generator(device=eng.device).manual_seed(rows)
    q = torch.randn((T, gg.num_q_heads, gg.head_dim), generator=gen, device=eng.device).to(gg.dtype)
    out = torch.full_like(q, float("nan"))
    ops.paged_prefill(eng.arena, eng.view(g, 0), int(gg.kind), q, out, torch.from_numpy(cu).to(eng.device),
                      int(chunks.max()), t.block_table[:B], t.seq_lens[:B], gg.num_kv_heads, TPP,
                      gg.head_dim ** -0.5, window=gg.window)
    torch.cuda.synchronize()
    want = orc.paged_prefill(arena_host(eng), tuple(eng.view(g, 0)), int(gg.kind), ORC_DTYPE[gg.dtype], gg.window,
                             q.view(torch.int16).cpu().numpy(), cu, t.block_table[:B].cpu().numpy(),
                             t.seq_lens[:B].cpu().numpy(), gg.num_q_heads, gg.num_kv_heads, gg.head_dim, TPP,
                             gg.head_dim ** -0.5)
    got = out.float().cpu().numpy()
    assert np.isfinite(got).all()
    assert rel_err(got, want) <= TOL[gg.dtype]


def test_speculative_verify_and_rollback(orc):
    geom = ModelGeometry("spec", [
        GroupGeometry("self", LayerKind.kFullAttention, 1, 8, 16, 128, torch.bfloat16, TPP),
        GroupGeometry("window", LayerKind.kSlidingWindow, 1, 8, 16, 128, torch.bfloat16, TPP, window=48),
        GroupGeometry("draft.self", LayerKind.kFullAttention, 1, 2, 8, 64, torch.bfloat16, TPP)])
    lens = [70, 33, 150]
    eng, ids = make_engine(geom, lens, seed=6, headroom_pages=16)
    assert [eng.pages.is_draft_group(g) for g in range(3)] == [False, False, True]
    for g in range(3):
        fill_group_kv(eng, g, [0], seed=10 + g, all_live=True)
    rng = np.random.default_rng(7)
    k = 4
    for rid in ids:  # a verify chunk needs the keys its earliest token sees
        eng.pages.set_defer_window_free(rid, True)
    for step in range(6):
        before = [[eng.pages.group_state(r, g)["stored"] for g in range(3)] for r in ids]
        acc = [int(a) for a in rng.integers(0, k + 1, len(ids))]
        for rid, a in zip(ids, acc):
            assert eng.pages.speculative_decode(rid, k, a, None, max(a, 1), now=100 + step)
        eng.sync_tables()
        after = [[eng.pages.group_state(r, g)["stored"] for g in range(3)] for r in ids]
        for i in range(len(ids)):
            assert after[i][2] - before[i][2] == acc[i]                # draft keeps accepted proposals
            assert after[i][0] - before[i][0] == max(acc[i], 1)       # target commits max(acc, 1)
        # K/V of every new ordinal (freed draft pages may now back target pages)
        for g in range(3):
            gg = eng.tables[g].geom
            req = [i for i in range(len(ids)) for _ in range(after[i][g] - before[i][g])]
            ords = [o for i in range(len(ids)) for o in range(before[i][g] + 1, after[i][g] + 1)]
            if not req:
                continue
            sl = slots_of(eng, g, req, ords)
            gen = torch.Generator(device=eng.device).manual_seed(1000 * step + g)
            K = torch.randn((len(req), gg.num_kv_heads, gg.head_dim), generator=gen, device=eng.device)
            V = torch.randn((len(req), gg.num_kv_heads, gg.head_dim), generator=gen, device=eng.device)
            eng.write_kv(g, 0, K.to(gg.dtype), V.to(gg.dtype), sl)
        for g in range(3):
            verify_attention(orc, eng, g, 17 * step + g, [after[i][g] - before[i][g] for i in range(len(ids))])
        for rid in ids:  # verify done: the window frees the chunk deferred
            eng.pages.apply_window_free(rid, now=100 + step)
    eng.kv.check_invariants()

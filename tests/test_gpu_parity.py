"""GPU parity: every kernel through the C ABI against the CPU oracle on the
same seeded inputs.  Integer/byte work is bit-exact; attention is within the
north-star tolerance (fp32 1e-5, bf16 1e-2 relative), written per test."""
import numpy as np
import pytest
import torch

from gpu_scenarios import ORC_DTYPE, TOL, arena_host, fill_group_kv, make_engine, rel_err
from oracle.oracle import CROSS, FULL, SWA
from paper_2503_18292_b200 import LayerKind, ops
from paper_2503_18292_b200.geometry import GroupGeometry, ModelGeometry, toy

pytestmark = pytest.mark.gpu


def oracle_tables(orc, eng, g):
    t = eng.tables[g]
    B = len(eng.requests)
    off, pages, live0, nst = eng.pages.pack_csr(g, eng.requests)
    return orc.build_block_tables(off, pages, live0, nst, t.slots_per_large, eng.spec.groups[g].tokens_per_page,
                                  t.max_blocks)


def check_tables(orc, eng):
    B = len(eng.requests)
    for g in range(len(eng.tables)):
        t = eng.tables[g]
        table, slots, seq = oracle_tables(orc, eng, g)
        np.testing.assert_array_equal(t.block_table[:B].cpu().numpy(), table)
        np.testing.assert_array_equal(t.slot_mapping[:B].cpu().numpy(), slots)
        np.testing.assert_array_equal(t.seq_lens[:B].cpu().numpy(), seq)


def run_decode_parity(orc, eng, g, layer, seed=1, softcap=0.0):
    t = eng.tables[g]
    gg = t.geom
    B = len(eng.requests)
    gen = torch.Generator(device=eng.device).manual_seed(seed)
    q = torch.randn((B, gg.num_q_heads, gg.head_dim), generator=gen, device=eng.device).to(gg.dtype)
    out = torch.empty_like(q)
    scale = gg.head_dim ** -0.5
    eng.decode(g, layer, q, out, scale=scale, softcap=softcap)
    torch.cuda.synchronize()
    arena = arena_host(eng)
    table = t.block_table[:B].cpu().numpy()
    seq = t.seq_lens[:B].cpu().numpy()
    qh = q.view(torch.int16).cpu().numpy() if gg.dtype != torch.float32 else q.cpu().numpy()
    want = orc.paged_decode(arena, tuple(eng.view(g, layer)), int(gg.kind), ORC_DTYPE[gg.dtype], gg.window, qh,
                            table, seq, gg.num_q_heads, gg.num_kv_heads, gg.head_dim,
                            eng.spec.groups[g].tokens_per_page, scale, softcap, nthreads=8)
    got = out.float().cpu().numpy()
    assert np.isfinite(got).all()
    tol = TOL[gg.dtype]
    err = rel_err(got, want)
    assert err <= tol, f"relative error {err:.3g} > {tol}"
    np.testing.assert_allclose(got, want, rtol=tol, atol=tol * np.abs(want).max())
    return err


@pytest.mark.parametrize("tpp", [16, 1])
def test_toy_config_fp32(orc, tpp):
    """configs[0]: 1 full + 1 SWA-512, Hkv=8, D=128, Hq=16, B=8 x ~2k, fp32 (tol 1e-5)."""
    geom = toy(tpp)
    lens = [2048, 2047, 1, 513, 512, 2000, 1500, 2048]
    eng, ids = make_engine(geom, lens)
    check_tables(orc, eng)
    for g in range(2):
        fill_group_kv(eng, g, [0], seed=g)
        run_decode_parity(orc, eng, g, 0)


def test_reshape_and_cache_bit_exact(orc):
    geom = ModelGeometry("rc", [GroupGeometry("full", LayerKind.kFullAttention, 3, 4, 8, 64, torch.bfloat16, 8)])
    eng, ids = make_engine(geom, [37, 5, 64, 100], poison=False)
    before = arena_host(eng).copy()
    req, ords, kvs, slots = fill_group_kv(eng, 0, [1, 2], seed=4)
    after = arena_host(eng)
    want = before.copy()
    sl = slots.cpu().numpy()
    for layer, (K, V) in zip([1, 2], kvs):
        orc.reshape_and_cache(want, tuple(eng.view(0, layer)), ORC_DTYPE[torch.bfloat16], 4, 64, 8,
                              K.view(torch.int16).cpu().numpy(), V.view(torch.int16).cpu().numpy(), sl)
    np.testing.assert_array_equal(after, want)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("kind", [LayerKind.kFullAttention, LayerKind.kSlidingWindow])
@pytest.mark.parametrize("hd,hq,hkv,tpp", [(256, 16, 8, 16), (128, 32, 8, 32), (64, 8, 8, 4), (128, 64, 8, 2)])
def test_decode_shapes(orc, dtype, kind, hd, hq, hkv, tpp):
    window = 300 if kind == LayerKind.kSlidingWindow else 0
    geom = ModelGeometry("s", [GroupGeometry("g", kind, 2, hkv, hq, hd, dtype, tpp, window=window)])
    lens = [1, 17, 299, 300, 301, 1025, 777]
    eng, ids = make_engine(geom, lens, seed=hd + tpp)
    check_tables(orc, eng)
    fill_group_kv(eng, 0, [1], seed=3)
    run_decode_parity(orc, eng, 0, 1, seed=7)


def test_gemma_shapes_bf16_long_context(orc):
    """Gemma-2-9B head geometry (Hq=16, Hkv=8, D=256, tpp=16), window 4096 at
    8k context, 2 layers per group to keep the arena small; softcap on."""
    geom = ModelGeometry("gemma-small", [
        GroupGeometry("full", LayerKind.kFullAttention, 2, 8, 16, 256, torch.bfloat16, 16),
        GroupGeometry("window", LayerKind.kSlidingWindow, 2, 8, 16, 256, torch.bfloat16, 16, window=4096)],
        softcap=50.0)
    lens = [8192, 4097, 4096, 8191]
    eng, ids = make_engine(geom, lens)
    check_tables(orc, eng)
    for g in range(2):
        fill_group_kv(eng, g, [1], seed=g)
        run_decode_parity(orc, eng, g, 1, softcap=50.0)


@pytest.mark.parametrize("kind", [LayerKind.kFullAttention, LayerKind.kSlidingWindow])
def test_head_dim_128_multi_split(orc, kind):
    """D=128 streams 96 tiles (1536 tokens) per CTA: contexts around and past
    that boundary exercise the split merge of the Llama/Jamba head shape."""
    window = 3000 if kind == LayerKind.kSlidingWindow else 0
    geom = ModelGeometry("d128", [GroupGeometry("g", kind, 2, 8, 32, 128, torch.bfloat16, 16, window=window)])
    lens = [4000, 3100, 1537, 1536, 1535, 5, 3073]
    eng, ids = make_engine(geom, lens, seed=5)
    check_tables(orc, eng)
    fill_group_kv(eng, 0, [0], seed=8)
    run_decode_parity(orc, eng, 0, 0, seed=2)


def test_cross_attention_image_tokens(orc):
    """Llama-3.2-Vision style: self (text only) + cross (image ordinals only),
    including a request with no image tokens (n=0 -> zero output)."""
    geom = ModelGeometry("vl", [
        GroupGeometry("self", LayerKind.kFullAttention, 2, 8, 32, 128, torch.bfloat16, 16),
        GroupGeometry("cross", LayerKind.kCrossAttention, 2, 8, 32, 128, torch.bfloat16, 16)])
    img = [lambda p: 5 < p <= 700, lambda p: False, lambda p: p <= 1601, lambda p: 10 < p <= 30]
    eng, ids = make_engine(geom, [800, 50, 1700, 64], image_flags=img)
    check_tables(orc, eng)
    seq_cross = eng.tables[1].seq_lens[:4].cpu().tolist()
    assert seq_cross == [695, 0, 1601, 20]
    assert eng.tables[0].seq_lens[:4].cpu().tolist() == [105, 50, 99, 44]
    for g in range(2):
        fill_group_kv(eng, g, [0], seed=g)
        run_decode_parity(orc, eng, g, 0)


def test_mamba_state_gather_scatter_and_checkpoint_copy(orc):
    geom = ModelGeometry("hyb", [
        GroupGeometry("attn", LayerKind.kFullAttention, 2, 8, 32, 128, torch.bfloat16, 16),
        GroupGeometry("ssm", LayerKind.kMamba, 4, state_bytes=(8192 * 3 + 8192 * 16) * 4 // 64)])
    eng, ids = make_engine(geom, [10, 1, 33, 7, 64], poison=False)
    check_tables(orc, eng)
    g = 1
    B = len(ids)
    pg = eng.mamba_page_globals(g)
    gen = torch.Generator(device=eng.device).manual_seed(9)
    for layer in (0, 3):
        view = eng.view(g, layer)
        dense = torch.randint(0, 255, (B, view.exec_page_size), generator=gen, device=eng.device,
                              dtype=torch.uint8)
        before = arena_host(eng)
        ops.mamba_state_scatter(eng.arena, view, pg, dense)
        torch.cuda.synchronize()
        want = before.copy()
        orc.mamba_scatter(want, tuple(view), pg.cpu().numpy(), dense.cpu().numpy())
        np.testing.assert_array_equal(arena_host(eng), want)
        back = torch.zeros_like(dense)
        ops.mamba_state_gather(eng.arena, view, pg, back)
        torch.cuda.synchronize()
        assert torch.equal(back, dense)
        np.testing.assert_array_equal(back.cpu().numpy(), orc.mamba_gather(want, tuple(view), pg.cpu().numpy(), B))
    # checkpoint snapshot: copy request 0's working page to a fresh page
    small = eng.tables[g].small_page_bytes
    res = eng.kv.allocate(g, 999)
    dst = eng.addr.global_page_index(g, res.page)
    src = pg[:1].clone()
    dstt = torch.tensor([dst], dtype=torch.int64, device=eng.device)
    before = arena_host(eng)
    ops.page_copy(eng.arena, small, src, dstt)
    torch.cuda.synchronize()
    want = before.copy()
    orc.page_copy(want, small, src.cpu().numpy(), [dst])
    np.testing.assert_array_equal(arena_host(eng), want)


@pytest.mark.parametrize("state_bytes", [622592, 20480])
def test_mamba_state_copy_large_and_skipped(orc, state_bytes):
    """Jamba-size state slices (many 16 KiB bulk-copy chunks per request, CTA
    shares crossing request boundaries) and odd sizes; index -1 = skipped."""
    geom = ModelGeometry("hyb", [
        GroupGeometry("attn", LayerKind.kFullAttention, 1, 8, 32, 128, torch.bfloat16, 16),
        GroupGeometry("ssm", LayerKind.kMamba, 3, state_bytes=state_bytes)])
    lens = [3, 1, 2, 5, 1, 4, 2, 7, 1, 3, 2]
    eng, ids = make_engine(geom, lens, poison=False)
    g = 1
    B = len(ids)
    pg = eng.mamba_page_globals(g).clone()
    pg[4] = -1
    pg[9] = -1
    gen = torch.Generator(device=eng.device).manual_seed(11)
    eng.arena.tensor().random_(0, 256, generator=gen)
    for layer in (0, 2):
        view = eng.view(g, layer)
        before = arena_host(eng)
        got = torch.full((B, view.exec_page_size), 7, device=eng.device, dtype=torch.uint8)
        ops.mamba_state_gather(eng.arena, view, pg, got)
        torch.cuda.synchronize()
        want = orc.mamba_gather(before, tuple(view), pg.cpu().numpy(), B)
        keep = pg.cpu().numpy() >= 0
        np.testing.assert_array_equal(got.cpu().numpy()[keep], want[keep])
        assert (got.cpu().numpy()[~keep] == 7).all()  # skipped rows untouched
        dense = torch.randint(0, 256, (B, view.exec_page_size), generator=gen, device=eng.device,
                              dtype=torch.uint8)
        ops.mamba_state_scatter(eng.arena, view, pg, dense)
        torch.cuda.synchronize()
        want = before.copy()
        orc.mamba_scatter(want, tuple(view), pg.cpu().numpy(), dense.cpu().numpy())
        np.testing.assert_array_equal(arena_host(eng), want)


def test_launch_counter_and_errors():
    n0 = ops.kernel_launch_count()
    geom = toy(16)
    eng, ids = make_engine(geom, [5, 9])
    assert ops.kernel_launch_count() > n0
    from paper_2503_18292_b200 import ConfigError
    q = torch.zeros((2, 16, 128), device="cuda")
    with pytest.raises(ConfigError):  # layer view of a bf16 geometry against fp32 data
        ops.paged_decode(eng.arena, eng.view(0, 0)._replace(exec_page_size=7), 0, q, torch.empty_like(q),
                         eng.tables[0].block_table[:2], eng.tables[0].seq_lens[:2], 8, 16, 1.0)
    with pytest.raises(ValueError):
        ops.paged_decode(eng.arena, eng.view(0, 0), 0, q.cpu(), q.cpu(), eng.tables[0].block_table[:2],
                         eng.tables[0].seq_lens[:2], 8, 16, 1.0)


@pytest.mark.parametrize("dtype,hd,hq,hkv,tpp,kind,window", [
    (torch.bfloat16, 256, 16, 8, 16, LayerKind.kFullAttention, 0),
    (torch.bfloat16, 256, 16, 8, 16, LayerKind.kSlidingWindow, 300),
    (torch.bfloat16, 128, 32, 8, 16, LayerKind.kSlidingWindow, 7),   # window inside the newest tile
    (torch.bfloat16, 128, 32, 8, 32, LayerKind.kFullAttention, 0),
    (torch.float32, 128, 16, 8, 16, LayerKind.kFullAttention, 0),    # CUDA-core kernel: write, then attend
])
def test_decode_append_fused(orc, dtype, hd, hq, hkv, tpp, kind, window):
    """jenga_paged_decode_append (newest token's K/V patched into the staged
    tile and written to its slot in the same launch) == reshape_and_cache +
    paged_decode, bit for bit, in the output and in the arena; and vs the oracle."""
    geom = ModelGeometry("app", [GroupGeometry("g", kind, 2, hkv, hq, hd, dtype, tpp, window=window)])
    lens = [1, 16, 17, 299, 300, 1025, 2049, 33]
    eng, ids = make_engine(geom, lens, seed=3)
    fill_group_kv(eng, 0, [1], seed=5)
    B = len(lens)
    gen = torch.Generator(device=eng.device).manual_seed(21)
    q = torch.randn((B, hq, hd), generator=gen, device=eng.device).to(dtype)
    k = torch.randn((B, hkv, hd), generator=gen, device=eng.device).to(dtype)
    v = torch.randn((B, hkv, hd), generator=gen, device=eng.device).to(dtype)
    at = eng.arena.tensor()
    saved = at.clone()
    out_a = torch.empty_like(q)
    eng.write_kv(0, 1, k, v)
    eng.decode(0, 1, q, out_a)
    torch.cuda.synchronize()
    arena_a = at.clone()
    at.copy_(saved)
    out_b = torch.empty_like(q)
    eng.decode_append(0, 1, q, k, v, out_b)
    torch.cuda.synchronize()
    assert torch.equal(at, arena_a), "fused append wrote different arena bytes"
    assert torch.equal(out_b, out_a), "fused append changed the attention output"
    t = eng.tables[0]
    qh = q.view(torch.int16).cpu().numpy() if dtype != torch.float32 else q.cpu().numpy()
    want = orc.paged_decode(arena_host(eng), tuple(eng.view(0, 1)), int(kind), ORC_DTYPE[dtype], window, qh,
                            t.block_table[:B].cpu().numpy(), t.seq_lens[:B].cpu().numpy(), hq, hkv, hd, tpp,
                            hd ** -0.5, 0.0, nthreads=8)
    assert rel_err(out_b.float().cpu().numpy(), want) <= TOL[dtype]


def test_fused_append_graph_steps_match_unfused():
    """Twenty decode steps of a full + SWA model captured as one CUDA graph per
    step (host append + pack between replays, as bench.py runs it), fused
    append vs eager reshape_and_cache + paged_decode on an identical engine:
    every step's outputs and the final arenas are bit-identical, across page
    boundaries and SWA frees."""
    from paper_2503_18292_b200.engine import DecodeEngine
    geom = ModelGeometry("g2", [
        GroupGeometry("full", LayerKind.kFullAttention, 2, 8, 16, 256, torch.bfloat16, 16),
        GroupGeometry("window", LayerKind.kSlidingWindow, 2, 8, 16, 256, torch.bfloat16, 16, window=40)])
    lens = [15, 31, 100]
    B, steps = len(lens), 20
    engines = []
    for _ in range(2):
        eng = DecodeEngine(geom, 64, B, 160)
        eng.add_requests(range(B))
        eng.arena.tensor().zero_()
        for pos in range(max(lens)):
            eng.append([r for r in range(B) if pos < lens[r]])
        engines.append(eng)
    gen = torch.Generator(device="cuda").manual_seed(17)
    layers = [(g, l) for l in range(2) for g in (0, 1)]
    q = torch.randn((steps, len(layers), B, 16, 256), generator=gen, device="cuda").to(torch.bfloat16)
    kv = torch.randn((steps, len(layers), 2, B, 8, 256), generator=gen, device="cuda").to(torch.bfloat16)
    outs = [torch.zeros((len(layers), B, 16, 256), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    qs = torch.empty_like(q[0])
    kvs = torch.empty_like(kv[0])
    fused, eager = engines

    def fused_device():
        fused.upload_tables()
        for i, (g, l) in enumerate(layers):
            fused.decode_append(g, l, qs[i], kvs[i, 0], kvs[i, 1], outs[0][i])

    fused.append()
    fused.pack_tables()
    qs.copy_(q[0])
    kvs.copy_(kv[0])
    fused_device()  # warm-up (tensor maps, smem attributes) outside capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    fused.pack_tables()
    with torch.cuda.graph(graph):
        fused_device()
    for s in range(steps):
        if s > 0:
            fused.append()
        fused.pack_tables()
        qs.copy_(q[s])
        kvs.copy_(kv[s])
        graph.replay()
        eager.append()
        eager.sync_tables()
        for i, (g, l) in enumerate(layers):
            eager.write_kv(g, l, kv[s, i, 0], kv[s, i, 1])
            eager.decode(g, l, q[s, i], outs[1][i])
        torch.cuda.synchronize()
        assert torch.equal(outs[0], outs[1]), f"step {s}: fused graph output differs"
    assert torch.equal(fused.arena.tensor(), eager.arena.tensor())


def test_delta_upload_matches_full_rebuild():
    """Delta page-list upload (table mirror -> jenga_upload_page_list_deltas,
    the kernel reading the pinned delta buffer in place) vs the CSR rebuild
    (jenga_build_block_tables) on two engines fed the same appends: block
    tables, seq_lens and newest slots bit-identical after every step — SWA
    frees, Mamba working pages, uneven appends, eager and graph-replayed."""
    from paper_2503_18292_b200.engine import DecodeEngine
    geom = ModelGeometry("d", [
        GroupGeometry("full", LayerKind.kFullAttention, 2, 8, 16, 128, torch.bfloat16, 16),
        GroupGeometry("window", LayerKind.kSlidingWindow, 2, 8, 16, 128, torch.bfloat16, 16, window=70),
        GroupGeometry("ssm", LayerKind.kMamba, 3, state_bytes=4096)])
    B = 6
    engs = [DecodeEngine(geom, 400, B, 700, upload=u) for u in ("delta", "full")]
    for e in engs:
        e.add_requests(range(B))
    rng = np.random.default_rng(5)
    graph = None
    for step in range(260):
        ids = [r for r in range(B) if rng.random() < 0.8]
        for e in engs:
            e.append(ids)
            e.pack_tables()
        if step == 100:  # from here on the delta engine's device half is a replayed graph
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                engs[0].upload_tables()
        if graph is None:
            engs[0].upload_tables()
        else:
            graph.replay()
        engs[1].upload_tables()
        torch.cuda.synchronize()
        for g in range(3):
            a, b = engs[0].tables[g], engs[1].tables[g]
            assert torch.equal(a.block_table, b.block_table), (step, g)
            assert torch.equal(a.seq_lens, b.seq_lens) and torch.equal(a.slot_mapping, b.slot_mapping), (step, g)
            assert torch.equal(a.h_n_stored, b.h_n_stored)


@pytest.mark.parametrize("decay,l0,nl", [(1.0, 0, 28), (0.5, 3, 7), (0.9375, 27, 1)])
def test_mamba_state_update_in_place(orc, decay, l0, nl):
    """jenga_mamba_state_update — the fused gather -> SSM stand-in -> scatter:
    layers [l0, l0 + nl) of each working page (one contiguous run per page)
    read and written back in place through the page table, fp32 state scaled
    by `decay`; every other byte of the arena untouched (C oracle
    orc_mamba_update on a host copy); index -1 skipped.  Jamba state size."""
    geom = ModelGeometry("hyb", [
        GroupGeometry("attn", LayerKind.kFullAttention, 1, 8, 32, 128, torch.bfloat16, 16),
        GroupGeometry("ssm", LayerKind.kMamba, 28, state_bytes=(8192 * 3 + 8192 * 16) * 4)])
    lens = [3, 1, 2, 5, 1, 4, 2]
    eng, ids = make_engine(geom, lens, poison=False)
    g = 1
    pg = eng.mamba_page_globals(g).clone()
    pg[3] = -1
    at = eng.arena.tensor()
    at.view(torch.float32).normal_(generator=torch.Generator(device=eng.device).manual_seed(5))
    before = arena_host(eng).copy()
    view = eng.view(g, l0)
    ops.mamba_state_update(eng.arena, view, nl, pg, decay)
    torch.cuda.synchronize()
    want = before.copy()
    orc.mamba_update(want, tuple(view), nl, pg.cpu().numpy(), decay)
    got = arena_host(eng)
    np.testing.assert_array_equal(got, want)
    if decay != 1.0:
        assert not np.array_equal(got, before)


@pytest.mark.parametrize("case", range(12))
def test_decode_append_fuzz(orc, case):
    """Seeded random shapes through the fused decode-append (the bench's kernel):
    head_dim 64 / 128 / 256, GQA group 1-8, tokens per page 16-64, full or sliding
    window (random width, including windows inside the newest tile), soft-capping,
    bf16 / fp16, random context lengths.  Fused == unfused bit for bit (output and
    arena bytes) and every (request, head) row vs the oracle (elementwise)."""
    rng = np.random.default_rng(500 + case)
    hd = [256, 128, 64][case % 3]
    G = [2, 4, 1, 8][case % 4]
    hkv = int(rng.choice([1, 2, 4, 8]))
    tpp = int(rng.choice([16, 32, 48, 64]))
    kind = LayerKind.kSlidingWindow if case % 2 else LayerKind.kFullAttention
    window = int(rng.choice([7, 100, 1000])) if kind == LayerKind.kSlidingWindow else 0
    softcap = 50.0 if case % 5 == 1 else 0.0
    dtype = torch.float16 if case % 6 == 3 else torch.bfloat16
    lens = [int(x) for x in rng.integers(1, 2500, int(rng.integers(2, 9)))]
    hq = hkv * G
    geom = ModelGeometry("fz", [GroupGeometry("g", kind, 2, hkv, hq, hd, dtype, tpp, window=window)], softcap=softcap)
    eng, ids = make_engine(geom, lens, seed=case)
    fill_group_kv(eng, 0, [1], seed=case + 1)
    B = len(lens)
    gen = torch.Generator(device=eng.device).manual_seed(100 + case)
    q = torch.randn((B, hq, hd), generator=gen, device=eng.device).to(dtype)
    k = torch.randn((B, hkv, hd), generator=gen, device=eng.device).to(dtype)
    v = torch.randn((B, hkv, hd), generator=gen, device=eng.device).to(dtype)
    at = eng.arena.tensor()
    saved = at.clone()
    out_a = torch.empty_like(q)
    eng.write_kv(0, 1, k, v)
    eng.decode(0, 1, q, out_a)
    torch.cuda.synchronize()
    arena_a = at.clone()
    at.copy_(saved)
    out_b = torch.empty_like(q)
    eng.decode_append(0, 1, q, k, v, out_b)
    torch.cuda.synchronize()
    assert torch.equal(at, arena_a), "fused append wrote different arena bytes"
    assert torch.equal(out_b, out_a), "fused append changed the attention output"
    t = eng.tables[0]
    want = orc.paged_decode(arena_host(eng), tuple(eng.view(0, 1)), int(kind), ORC_DTYPE[dtype], window,
                            q.view(torch.int16).cpu().numpy(), t.block_table[:B].cpu().numpy(),
                            t.seq_lens[:B].cpu().numpy(), hq, hkv, hd, tpp, hd ** -0.5, softcap, nthreads=8)
    got = out_b.float().cpu().numpy()
    tol = TOL[dtype]
    assert rel_err(got, want) <= tol
    np.testing.assert_allclose(got, want, rtol=tol, atol=tol * np.abs(want).max())


def test_mamba_per_layer_updates_early_loads(orc):
    """Per-layer in-place updates in model order (the Jamba bench's per-layer
    step): each launch after the first loads its states before
    griddepcontrol.wait because the pending writers are column writers with
    disjoint layer columns (common.cuh).  A repeated layer, an overlapping
    two-layer run and an attention KV write (blanket PDL writer) in the
    sequence must fall back to waiting.  The arena must equal the oracle's
    sequential application, byte for byte, at the bench's batch (64 requests,
    ~40 MB per launch, so launches overlap)."""
    geom = ModelGeometry("hyb", [
        GroupGeometry("attn", LayerKind.kFullAttention, 1, 8, 32, 128, torch.bfloat16, 16),
        GroupGeometry("ssm", LayerKind.kMamba, 28, state_bytes=(8192 * 3 + 8192 * 16) * 4)])
    lens = [1 + (i % 5) for i in range(64)]
    eng, ids = make_engine(geom, lens, poison=False)
    g = 1
    pg = eng.mamba_page_globals(g).clone()
    pg[7] = -1
    at = eng.arena.tensor()
    at.view(torch.float32).normal_(generator=torch.Generator(device=eng.device).manual_seed(9))
    want = arena_host(eng).copy()
    seq = [(l, 1, 0.999) for l in range(28)]
    seq[6:6] = [(5, 1, 0.5)]          # layer 5 again right after itself
    seq[12:12] = [(10, 2, 0.75)]      # a run overlapping the last two layers
    seq[20:20] = [("kv", 0, 0)]       # attention KV write: unknown footprint
    for l, nl, decay in seq:
        if l == "kv":
            req, ords, kvs, slots = fill_group_kv(eng, 0, [0], seed=4)
            K, V = kvs[0]
            orc.reshape_and_cache(want, tuple(eng.view(0, 0)), ORC_DTYPE[torch.bfloat16], 8, 128, 16,
                                  K.view(torch.int16).cpu().numpy(), V.view(torch.int16).cpu().numpy(),
                                  slots.cpu().numpy())
            continue
        view = eng.view(g, l)
        ops.mamba_state_update(eng.arena, view, nl, pg, decay)
        orc.mamba_update(want, tuple(view), nl, pg.cpu().numpy(), decay)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(arena_host(eng), want)

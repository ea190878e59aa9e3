"""Chunked-prefill paged attention against the oracle:
causal / sliding-window / cross masks, ragged chunk lengths, chunks longer
than the query block, bf16 (1e-2) and fp16 (5e-3) tolerances."""
import numpy as np
import pytest
import torch

from gpu_scenarios import ORC_DTYPE, TOL, arena_host, fill_group_kv, make_engine, rel_err
from paper_2503_18292_b200 import LayerKind, ops
from paper_2503_18292_b200.geometry import GroupGeometry, ModelGeometry

pytestmark = pytest.mark.gpu


def run_prefill(orc, eng, g, layer, chunks, seed=5):
    t = eng.tables[g]
    gg = t.geom
    B = len(eng.requests)
    cu = np.zeros(B + 1, dtype=np.int32)
    cu[1:] = np.cumsum(chunks)
    T = int(cu[-1])
    gen = torch.Generator(device=eng.device).manual_seed(seed)
    q = torch.randn((T, gg.num_q_heads, gg.head_dim), generator=gen, device=eng.device).to(gg.dtype)
    out = torch.full_like(q, float("nan"))
    cu_d = torch.from_numpy(cu).to(eng.device)
    scale = gg.head_dim ** -0.5
    softcap = eng.geom.softcap
    ops.paged_prefill(eng.arena, eng.view(g, layer), int(gg.kind), q, out, cu_d, int(max(chunks)),
                      t.block_table[:B], t.seq_lens[:B], gg.num_kv_heads, eng.spec.groups[g].tokens_per_page, scale,
                      window=gg.window, softcap=softcap)
    torch.cuda.synchronize()
    want = orc.paged_prefill(arena_host(eng), tuple(eng.view(g, layer)), int(gg.kind), ORC_DTYPE[gg.dtype],
                             gg.window, q.view(torch.int16).cpu().numpy(), cu, t.block_table[:B].cpu().numpy(),
                             t.seq_lens[:B].cpu().numpy(), gg.num_q_heads, gg.num_kv_heads, gg.head_dim,
                             eng.spec.groups[g].tokens_per_page, scale, softcap)
    got = out.float().cpu().numpy()
    assert np.isfinite(got).all()
    tol = TOL[gg.dtype]
    err = rel_err(got, want)
    assert err <= tol, f"relative error {err:.3g} > {tol}"
    np.testing.assert_allclose(got, want, rtol=tol, atol=tol * np.abs(want).max())


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16], ids=["bf16", "fp16"])
@pytest.mark.parametrize("kind", [LayerKind.kFullAttention, LayerKind.kSlidingWindow])
@pytest.mark.parametrize("hd,hq,hkv", [(256, 16, 8), (128, 32, 8), (64, 8, 8), (128, 64, 8)])
def test_prefill_shapes(orc, dtype, kind, hd, hq, hkv):
    window = 100 if kind == LayerKind.kSlidingWindow else 0
    geom = ModelGeometry("p", [GroupGeometry("g", kind, 2, hkv, hq, hd, dtype, 16, window=window)])
    lens = [300, 77, 513, 16, 1]
    chunks = [300, 13, 200, 16, 1]  # whole prompt, tail chunks, single token
    eng, ids = make_engine(geom, lens, seed=hd, defer_window=True)
    fill_group_kv(eng, 0, [1], seed=2, all_live=True)
    run_prefill(orc, eng, 0, 1, chunks)


def test_prefill_gemma_long_chunk_softcap(orc):
    geom = ModelGeometry("gemma-p", [
        GroupGeometry("full", LayerKind.kFullAttention, 1, 8, 16, 256, torch.bfloat16, 16),
        GroupGeometry("window", LayerKind.kSlidingWindow, 1, 8, 16, 256, torch.bfloat16, 16, window=4096)],
        softcap=50.0)
    eng, ids = make_engine(geom, [5000, 1024], seed=9, defer_window=True)
    for g in range(2):
        fill_group_kv(eng, g, [0], seed=g, all_live=True)
        run_prefill(orc, eng, g, 0, [512, 1024])


def test_prefill_d128_long_chunk_pingpong(orc):
    """Llama / Jamba heads (D=128, G=4: the split-accumulator 128-key kernel) on long
    chunks at a 5k context, full and SWA-1000 with soft-capping."""
    geom = ModelGeometry("llama-p", [
        GroupGeometry("full", LayerKind.kFullAttention, 1, 8, 32, 128, torch.bfloat16, 16),
        GroupGeometry("window", LayerKind.kSlidingWindow, 1, 8, 32, 128, torch.bfloat16, 16, window=1000)],
        softcap=30.0)
    eng, ids = make_engine(geom, [5000, 1100, 700], seed=13, defer_window=True)
    for g in range(2):
        fill_group_kv(eng, g, [0], seed=g + 3, all_live=True)
        run_prefill(orc, eng, g, 0, [1500, 1100, 77])


def test_prefill_cross_attention(orc):
    geom = ModelGeometry("vl", [
        GroupGeometry("self", LayerKind.kFullAttention, 1, 8, 32, 128, torch.bfloat16, 16),
        GroupGeometry("cross", LayerKind.kCrossAttention, 1, 8, 32, 128, torch.bfloat16, 16)])
    img = [lambda p: p <= 400, lambda p: 3 < p <= 40]
    eng, ids = make_engine(geom, [450, 90], image_flags=img)
    fill_group_kv(eng, 1, [0], seed=1)
    run_prefill(orc, eng, 1, 0, [33, 70])  # text-token queries over all image keys



@pytest.mark.parametrize("case", range(16))
def test_prefill_fuzz(orc, case):
    """Seeded random shapes through both prefill kernels: head_dim 64 / 128 / 256, GQA
    group 1-8, bf16 or fp16, tokens per page 16-128 (the TMA producer's page / offset split), full or
    sliding-window attention with a random window, optional soft-capping, ragged chunk
    lengths (chunks starting mid-page, single tokens, a chunk equal to the whole prompt).
    Every (token, head) row is checked (elementwise atol = tol * max|want|)."""
    rng = np.random.default_rng(1000 + case)
    hd = [128, 256, 128, 256, 64, 128, 256, 128][case % 8]
    G = [1, 2, 4, 8][case % 4]
    hkv = [4, 2, 2, 1][case % 4]
    tpp = int(rng.choice([16, 32, 48, 64, 128]))
    kind = LayerKind.kSlidingWindow if case % 3 == 1 else LayerKind.kFullAttention
    window = int(rng.integers(40, 600)) if kind == LayerKind.kSlidingWindow else 0
    softcap = float(rng.choice([0.0, 30.0])) if case >= 4 else 0.0
    nreq = int(rng.integers(2, 5))
    lens = [int(x) for x in rng.integers(1, 1400, nreq)]
    chunks = [int(min(n, rng.choice([n, rng.integers(1, n + 1), 1]))) for n in lens]
    dtype = torch.float16 if case % 5 == 2 else torch.bfloat16
    geom = ModelGeometry("fz", [GroupGeometry("g", kind, 1, hkv, hkv * G, hd, dtype, tpp, window=window)],
                         softcap=softcap)
    eng, ids = make_engine(geom, lens, seed=case, defer_window=True)
    fill_group_kv(eng, 0, [0], seed=case + 7, all_live=True)
    run_prefill(orc, eng, 0, 0, chunks, seed=case)


@pytest.mark.parametrize("hd,kind", [(128, LayerKind.kFullAttention), (256, LayerKind.kSlidingWindow),
                                     (128, LayerKind.kCrossAttention)])
def test_prefill_many_requests_persistent(orc, hd, kind):
    """Many ragged requests: several work units per persistent CTA pair, with units past
    their request's chunk (skipped), sliding windows that leave most keys out, and
    single-token chunks -- the per-CTA tile / unit counters must stay in step across
    units of different lengths."""
    rng = np.random.default_rng(77 + hd)
    nreq = 24
    lens = [int(x) for x in rng.integers(1, 700, nreq)]
    chunks = [int(min(n, rng.choice([n, rng.integers(1, n + 1), 1]))) for n in lens]
    window = 57 if kind == LayerKind.kSlidingWindow else 0
    G = 2 if hd == 256 else 4
    groups = [GroupGeometry("g", kind, 1, 2, 2 * G, hd, torch.bfloat16, 16, window=window)]
    img, g = None, 0
    if kind == LayerKind.kCrossAttention:  # text tokens attend the image tokens the cross group stores
        groups.insert(0, GroupGeometry("self", LayerKind.kFullAttention, 1, 2, 2 * G, hd, torch.bfloat16, 16))
        img, g = [(lambda p, k=k: p <= 40 * (k % 5 + 1)) for k in range(nreq)], 1
    eng, ids = make_engine(ModelGeometry("many", groups), lens, seed=hd, defer_window=True, image_flags=img)
    fill_group_kv(eng, g, [0], seed=3, all_live=kind != LayerKind.kCrossAttention)
    run_prefill(orc, eng, g, 0, chunks)

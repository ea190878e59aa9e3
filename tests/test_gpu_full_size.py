"""Parity at BASELINE.json's full size (configs[1], the bench's per-GPU shard):
Gemma-2-9B geometry, 42 layers (21 full + 21 SWA-4096) resident in one 68 GB
arena, 32 requests x 8k context, page lists from the native allocator with
interleaved request order.  Checks, through the C ABI:

* block tables / slot mappings / seq_lens of both groups bit-exact against the
  oracle's table build over the same page lists (all 32 requests);
* the fused decode step the bench times (jenga_paged_decode_append: the newest
  token's K/V written into its slot by the decode launch itself), on the last
  layer of each group: the new K/V read back byte-exact (sampled requests /
  heads), every request's output finite, and 8 sampled requests within the
  bf16 tolerance of the C oracle (fp64) — the oracle runs on a compact copy
  of just those requests' layer slices (the whole arena is too big to copy to
  the host).  Tolerance is normwise per sample set: max|got - want| /
  max|want| <= 1e-2.
"""
import gc

import numpy as np
import pytest
import torch

from gpu_scenarios import TOL, rel_err
from oracle.oracle import BF16
from paper_2503_18292_b200 import ops
from paper_2503_18292_b200.engine import DecodeEngine
from paper_2503_18292_b200.geometry import gemma2_9b

pytestmark = pytest.mark.gpu

B, CTX = 32, 8192


def _build():
    geom = gemma2_9b(16)
    eng = DecodeEngine(geom, 25000, B, CTX + 64)  # 68.75 GB: the bench shard's sizing
    eng.add_requests(range(B))
    rng = np.random.default_rng(1234)
    order = np.arange(B)
    for pos in range(CTX):
        if pos % 16 == 0:
            order = rng.permutation(B)
        assert eng.append(list(order)) == B
    eng.sync_tables()
    torch.cuda.synchronize()
    return eng


def _compact(eng, g, layer, rows):
    """Host copy of the layer slices of the pages in `rows` (block-table rows)
    plus the table remapped onto that compact arena."""
    v = eng.view(g, layer)
    slice_b = v.exec_page_size
    pages = np.unique(rows[rows >= 0])
    at = eng.arena.tensor()
    host = np.empty(len(pages) * slice_b, dtype=np.uint8)
    for i, pg in enumerate(pages):
        off = v.start_offset + int(pg) * v.page_stride
        host[i * slice_b:(i + 1) * slice_b] = at[off:off + slice_b].cpu().numpy()
    remap = {int(pg): i for i, pg in enumerate(pages)}
    table = np.where(rows >= 0, np.vectorize(lambda x: remap.get(int(x), -1))(rows), -1).astype(np.int32)
    return host, table, (0, slice_b, slice_b)


def test_gemma_shard_full_size(orc):
    if torch.cuda.get_device_properties(0).total_memory < 100e9:
        pytest.skip("needs a 180 GB B200 (68 GB arena)")
    eng = _build()
    try:
        at = eng.arena.tensor()
        gen = torch.Generator(device=eng.device).manual_seed(0)
        for s in range(0, at.numel(), 1 << 30):  # finite random KV everywhere
            at[s:s + (1 << 30)].view(torch.bfloat16).normal_(generator=gen)
        for g in range(2):
            t = eng.tables[g]
            gg = t.geom
            tpp = eng.spec.groups[g].tokens_per_page
            off, pages, live0, n_stored = eng.pages.pack_csr(g, eng.requests)
            table, slots, seq = orc.build_block_tables(off, pages, live0, n_stored, t.slots_per_large, tpp, t.max_blocks)
            np.testing.assert_array_equal(t.block_table[:B].cpu().numpy(), table)
            np.testing.assert_array_equal(t.slot_mapping[:B].cpu().numpy(), slots)
            np.testing.assert_array_equal(t.seq_lens[:B].cpu().numpy(), seq)
            assert (seq == CTX).all()

            layer = gg.num_layers - 1  # the last layer: largest start_offset in the arena
            k = torch.randn((B, 8, 256), generator=gen, device=eng.device).to(torch.bfloat16)
            v = torch.randn((B, 8, 256), generator=gen, device=eng.device).to(torch.bfloat16)
            q = torch.randn((B, 16, 256), generator=gen, device=eng.device).to(torch.bfloat16)
            out = torch.empty_like(q)
            eng.decode_append(g, layer, q, k, v, out)  # the bench's fused launch
            torch.cuda.synchronize()
            assert torch.isfinite(out.float()).all()

            # newest token's K/V landed in its slot (head-major slice, memory_layout.cpp:41-55)
            view = eng.view(g, layer)
            for b in (0, 17, 31):
                sl = int(slots[b])
                page, o = divmod(sl, tpp)
                base = view.start_offset + page * view.page_stride
                for h in (0, 7):
                    for kv, src in ((0, k), (1, v)):
                        row = base + ((2 * h + kv) * tpp + o) * 512
                        got = at[row:row + 512].cpu()
                        assert torch.equal(got, src[b, h].contiguous().view(torch.uint8).cpu())

            sample = [0, 4, 9, 13, 18, 22, 27, 31]
            rows = t.block_table[:B].cpu().numpy()[sample]
            host, ctable, cview = _compact(eng, g, layer, rows)
            want = orc.paged_decode(host, cview, int(gg.kind), BF16, gg.window, q[sample].view(torch.int16).cpu().numpy(),
                                    ctable, seq[sample], 16, 8, 256, tpp, 256 ** -0.5, eng.geom.softcap, nthreads=8)
            got = out[sample].float().cpu().numpy()
            tol = TOL[torch.bfloat16]
            err = rel_err(got, want)
            assert err <= tol, f"group {g}: relative error {err:.3g} > {tol}"
    finally:
        del at, eng
        gc.collect()
        torch.cuda.synchronize()


def _sampled_decode_check(orc, eng, g, layer, q, sample, tol):
    t = eng.tables[g]
    gg = t.geom
    B = len(eng.requests)
    out = torch.empty_like(q)
    eng.decode(g, layer, q, out)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    rows = t.block_table[:B].cpu().numpy()[sample]
    seq = t.seq_lens[:B].cpu().numpy()[sample]
    host, ctable, cview = _compact(eng, g, layer, rows)
    want = orc.paged_decode(host, cview, int(gg.kind), BF16, gg.window, q[sample].view(torch.int16).cpu().numpy(),
                            ctable, seq, gg.num_q_heads, gg.num_kv_heads, gg.head_dim,
                            eng.spec.groups[g].tokens_per_page, gg.head_dim ** -0.5, eng.geom.softcap, nthreads=8)
    err = rel_err(out[sample].float().cpu().numpy(), want)
    print(f"[full-size] group {g} layer {layer}: seq {seq.tolist()} relative error {err:.3g}")
    assert err <= tol, f"group {g} layer {layer}: relative error {err:.3g} > {tol}"


def test_llama_vision_full_size(orc):
    """configs[3] at the bench size: 64 requests x (6404 image tokens + 2048
    text), 32 self + 8 cross layers; cross-attention stores image ordinals only
    (simulator.cpp:151-158).  Tables bit-exact for both groups, sampled
    self- and cross-attention outputs vs the oracle."""
    from paper_2503_18292_b200.geometry import llama32_11b_vision
    B, n_img, ctx = 64, 6404, 2048
    eng = DecodeEngine(llama32_11b_vision(16), B * (ctx // 16 + 2) + B * ((n_img // 16 + 2) // 4 + 1) + 512, B,
                       n_img + ctx + 64, group_max_tokens={0: ctx + 64, 1: n_img + 64})
    try:
        eng.add_requests(range(B))
        rng = np.random.default_rng(7)
        order = np.arange(B)
        for pos in range(n_img + ctx):
            if pos % 16 == 0:
                order = rng.permutation(B)
            assert eng.append(list(order), is_image=[pos < n_img] * B) == B
        eng.sync_tables()
        at = eng.arena.tensor()
        gen = torch.Generator(device=eng.device).manual_seed(4)
        for s in range(0, at.numel(), 1 << 30):
            at[s:s + (1 << 30)].view(torch.bfloat16).normal_(generator=gen)
        for g, n_want in ((0, ctx), (1, n_img)):
            t = eng.tables[g]
            off, pages, live0, n_stored = eng.pages.pack_csr(g, eng.requests)
            table, slots, seq = orc.build_block_tables(off, pages, live0, n_stored, t.slots_per_large, 16,
                                                       t.max_blocks)
            np.testing.assert_array_equal(t.block_table[:B].cpu().numpy(), table)
            np.testing.assert_array_equal(t.seq_lens[:B].cpu().numpy(), seq)
            assert (seq == n_want).all()
            q = torch.randn((B, 32, 128), generator=gen, device=eng.device).to(torch.bfloat16)
            _sampled_decode_check(orc, eng, g, t.geom.num_layers - 1, q, [0, 37, 63], TOL[torch.bfloat16])
    finally:
        del eng
        gc.collect()
        torch.cuda.synchronize()


def test_jamba_full_size(orc):
    """configs[2] at the bench size: 64 requests x 8k, 4 attention layers and
    28 Mamba layers whose 622,592-byte states share the LCM pool (133 attention
    pages per large page).  Attention decode sampled vs the oracle; every
    request's Mamba state gathered and scattered byte-exactly on two layers."""
    from paper_2503_18292_b200.geometry import jamba_style
    B, ctx = 64, 8192
    geom = jamba_style(16)
    eng = DecodeEngine(geom, 480, B, ctx + 64)  # 16.8 GB of 34.9 MB LCM pages (bench sizing + margin)
    try:
        eng.add_requests(range(B))
        rng = np.random.default_rng(9)
        order = np.arange(B)
        for pos in range(ctx):
            if pos % 16 == 0:
                order = rng.permutation(B)
            assert eng.append(list(order)) == B
        eng.sync_tables()
        at = eng.arena.tensor()
        gen = torch.Generator(device=eng.device).manual_seed(5)
        for s in range(0, at.numel(), 1 << 30):
            at[s:s + (1 << 30)].view(torch.bfloat16).normal_(generator=gen)
        q = torch.randn((B, 32, 128), generator=gen, device=eng.device).to(torch.bfloat16)
        _sampled_decode_check(orc, eng, 0, 3, q, [0, 21, 63], TOL[torch.bfloat16])
        g = 1
        pg = eng.mamba_page_globals(g)
        assert (pg >= 0).all()
        for layer in (0, 27):
            v = eng.view(g, layer)
            dense = torch.empty((B, v.exec_page_size), dtype=torch.uint8, device=eng.device)
            ops.mamba_state_gather(eng.arena, v, pg, dense)
            torch.cuda.synchronize()
            pgh = pg.cpu().numpy()
            for b in (0, 30, 63):  # against the AddressMap arithmetic directly
                off = v.start_offset + int(pgh[b]) * v.page_stride
                assert torch.equal(dense[b].cpu(), at[off:off + v.exec_page_size].cpu())
            new = torch.randint(0, 256, dense.shape, generator=gen, device=eng.device, dtype=torch.uint8)
            ops.mamba_state_scatter(eng.arena, v, pg, new)
            back = torch.empty_like(new)
            ops.mamba_state_gather(eng.arena, v, pg, back)
            torch.cuda.synchronize()
            assert torch.equal(back, new)
    finally:
        del eng
        gc.collect()
        torch.cuda.synchronize()

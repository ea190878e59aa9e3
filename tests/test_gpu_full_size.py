"""Parity at BASELINE.json's full size (configs[1], the bench's per-GPU shard):
Gemma-2-9B geometry, 42 layers (21 full + 21 SWA-4096) resident in one 68 GB
arena, 32 requests x 8k context, page lists from the native allocator with
interleaved request order.  Checks, through the C ABI:

* block tables / slot mappings / seq_lens of both groups bit-exact against the
  oracle's table build over the same page lists (all 32 requests);
* reshape_and_cache of the newest token, read back byte-exact (sampled requests / heads);
* paged decode on the last layer of each group: every request's output is
  finite, and sampled requests match the C oracle (fp64) within the bf16
  tolerance — the oracle runs on a compact copy of just those requests' layer
  slices (the whole arena is too big to copy to the host).
"""
import gc

import numpy as np
import pytest
import torch

from gpu_scenarios import TOL, rel_err
from oracle.oracle import BF16
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
            eng.write_kv(g, layer, k, v)
            q = torch.randn((B, 16, 256), generator=gen, device=eng.device).to(torch.bfloat16)
            out = torch.empty_like(q)
            eng.decode(g, layer, q, out)
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

            sample = [0, 13, 31]
            rows = t.block_table[:B].cpu().numpy()[sample]
            host, ctable, cview = _compact(eng, g, layer, rows)
            want = orc.paged_decode(host, cview, int(gg.kind), BF16, gg.window, q[sample].view(torch.int16).cpu().numpy(),
                                    ctable, seq[sample], 16, 8, 256, tpp, 256 ** -0.5, 0.0, nthreads=8)
            got = out[sample].float().cpu().numpy()
            tol = TOL[torch.bfloat16]
            err = rel_err(got, want)
            assert err <= tol, f"group {g}: relative error {err:.3g} > {tol}"
    finally:
        del at, eng
        gc.collect()
        torch.cuda.synchronize()

"""Pin the CPU oracle (oracle/jenga_oracle.c) before trusting it: address and
block-table arithmetic against the reference's golden vectors and the
reference library; attention against an independent numpy fp64 statement of
its definition (attention parity is unpinned by the reference — no
reference kernel exists)."""
import json

import numpy as np
import pytest

from conftest import load_golden
from oracle.oracle import BF16, CROSS, F32, FULL, SWA


def test_oracle_address_map_fig6(orc):
    gold = load_golden("fig6.json")
    groups = gold["spec"]["groups"]
    smalls = [orc.small_page_size(g["bytes_per_token_per_layer"], g["num_layers"], 1) for g in groups]
    lcm = orc.lcm_page_size(smalls)
    assert lcm == gold["large_page_bytes"]
    for e in gold["entries"]:
        g = groups[e["g"]]
        spl = lcm // smalls[e["g"]]
        per_layer = g["bytes_per_token_per_layer"]
        assert orc.global_page_index(e["large"], e["slot"], spl) == e["global"]
        assert list(orc.address_of(lcm, smalls[e["g"]], per_layer, g["num_layers"], spl, e["layer"], e["large"],
                                   e["slot"])) == e["range"]
        assert list(orc.view_address(smalls[e["g"]], per_layer, g["num_layers"], spl, e["layer"], e["large"],
                                     e["slot"])) == e["view"]


def test_oracle_address_map_random_geometries(orc):
    for case in load_golden("random_geometries.json")[:40]:
        groups = json.loads(case["json"])["groups"]
        smalls = [orc.small_page_size(g["bytes_per_token_per_layer"], g["num_layers"], g["tokens_per_page"])
                  for g in groups]
        lcm = orc.lcm_page_size(smalls)
        assert lcm == case["large"]
        for g, layer, lp, slot, glob, b, e in case["entries"]:
            gg = groups[g]
            spl = lcm // smalls[g]
            assert orc.global_page_index(lp, slot, spl) == glob
            assert orc.address_of(lcm, smalls[g], gg["bytes_per_token_per_layer"] * gg["tokens_per_page"],
                                  gg["num_layers"], spl, layer, lp, slot) == (b, e)


def test_oracle_block_tables_match_reference(ref, orc):
    """Block tables from the reference AddressMap over reference-allocated page
    lists == oracle build over the same CSR lists."""
    from oracle.oracle import RefPageLists
    js = json.dumps({"name": "g", "groups": [
        {"name": "full", "kind": "full", "num_layers": 2, "bytes_per_token_per_layer": 256, "tokens_per_page": 2},
        {"name": "win", "kind": "sliding_window", "num_layers": 5, "bytes_per_token_per_layer": 256,
         "window_tokens": 9, "tokens_per_page": 2}]})
    rs = ref.spec(js)
    rkv = rs.kv(300 * 2560)
    rpl = RefPageLists(rkv)
    addr = rs.address_map()
    rng = np.random.default_rng(3)
    ids = list(range(6))
    for pos in range(1, 50):
        rpl.append_batch(rng.permutation(ids))
    for g in range(2):
        max_blocks = 30
        want = rpl.block_table(addr, g, ids, max_blocks)
        offsets, pages, first_live, n_stored = [0], [], [], []
        for r in ids:
            p, live, stored, freed = rpl.group_state(r, g)
            pages += p.tolist()
            offsets.append(len(pages))
            first_live.append(freed)
            n_stored.append(stored)
        spl = addr.info(g)[3]
        table, slots, seq = orc.build_block_tables(offsets, pages, first_live, n_stored, spl, 2, max_blocks)
        np.testing.assert_array_equal(table, want)
        assert seq.tolist() == n_stored
        for i, r in enumerate(ids):
            n = n_stored[i]
            assert slots[i] == want[i, (n - 1) // 2] * 2 + (n - 1) % 2


def _np_attention(arena, view, kind, window, q, table, seq_lens, hq, hkv, d, tpp, scale, dtype):
    """Independent numpy restatement (fp64) of masked paged attention."""
    e = 4 if dtype == F32 else 2
    B = q.shape[0]
    G = hq // hkv
    out = np.zeros((B, hq, d))
    for b in range(B):
        n = seq_lens[b]
        lo = max(0, n - window) if kind == SWA else 0
        for h in range(hkv):
            toks = np.arange(lo, n)
            if len(toks) == 0:
                continue
            pages = table[b, toks // tpp]
            offs = toks % tpp
            base = view[0] + pages.astype(np.int64) * view[1]
            krow = base + ((2 * h + 0) * tpp + offs) * d * e  # head-major slice
            vrow = base + ((2 * h + 1) * tpp + offs) * d * e
            K = np.stack([_decode(arena[r:r + d * e], dtype) for r in krow])
            V = np.stack([_decode(arena[r:r + d * e], dtype) for r in vrow])
            for g in range(G):
                qq = q[b, h * G + g].astype(np.float64)
                s = K @ qq * scale
                p = np.exp(s - s.max())
                out[b, h * G + g] = p @ V / p.sum()
    return out


def _decode(raw, dtype):
    if dtype == F32:
        return raw.view(np.float32).astype(np.float64)
    return (raw.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _to_bf16_bits(x):
    u = np.asarray(x, dtype=np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


@pytest.mark.parametrize("dtype,kind,tpp", [(F32, FULL, 4), (F32, SWA, 2), (BF16, FULL, 16), (BF16, SWA, 1),
                                            (F32, CROSS, 8)])
def test_oracle_attention_matches_numpy_definition(orc, dtype, kind, tpp):
    rng = np.random.default_rng(1)
    B, hq, hkv, d, window = 3, 4, 2, 32, 7
    e = 4 if dtype == F32 else 2
    exec_bytes = 2 * hkv * tpp * d * e
    nlayers = 2
    stride = exec_bytes * nlayers
    npages = 64
    view = (exec_bytes, stride, exec_bytes)  # layer 1
    arena = rng.integers(0, 255, size=npages * stride, dtype=np.uint8)
    # fill with finite values of the dtype
    vals = rng.standard_normal(arena.size // e).astype(np.float32)
    arena = (vals.view(np.uint8) if dtype == F32 else _to_bf16_bits(vals).view(np.uint8)).copy()
    seq = np.array([1, 13, 29], dtype=np.int32)
    maxb = 29 // tpp + 2
    table = np.full((B, maxb), -1, dtype=np.int32)
    perm = rng.permutation(npages)
    k = 0
    for b in range(B):
        lo = max(0, seq[b] - window) if kind == SWA else 0
        for blk in range((seq[b] + tpp - 1) // tpp):
            if (blk + 1) * tpp > lo:
                table[b, blk] = perm[k]
            k += 1
    qf = rng.standard_normal((B, hq, d)).astype(np.float32)
    q = qf if dtype == F32 else _to_bf16_bits(qf)
    qd = qf if dtype == F32 else (q.astype(np.uint32) << 16).view(np.float32)
    got = orc.paged_decode(arena, view, kind, dtype, window, q, table, seq, hq, hkv, d, tpp, 0.125)
    want = _np_attention(arena, view, kind, window, qd, table, seq, hq, hkv, d, tpp, 0.125, dtype)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
    got_mt = orc.paged_decode(arena, view, kind, dtype, window, q, table, seq, hq, hkv, d, tpp, 0.125, nthreads=3)
    np.testing.assert_array_equal(got, got_mt)


def test_oracle_rejects_live_token_on_freed_page(orc):
    arena = np.zeros(4096, dtype=np.uint8)
    table = np.array([[-1, 0]], dtype=np.int32)
    with pytest.raises(RuntimeError):
        orc.paged_decode(arena, (0, 1024, 1024), FULL, F32, 0, np.zeros((1, 2, 32), np.float32), table,
                         np.array([4]), 2, 2, 32, 2, 1.0)


def test_oracle_reshape_and_cache_roundtrip(orc):
    rng = np.random.default_rng(5)
    hkv, d, tpp, e = 2, 16, 4, 4
    exec_bytes = 2 * hkv * tpp * d * e
    stride = 3 * exec_bytes
    arena = np.zeros(10 * stride, dtype=np.uint8)
    view = (2 * exec_bytes, stride, exec_bytes)
    K = rng.standard_normal((5, hkv, d)).astype(np.float32)
    V = rng.standard_normal((5, hkv, d)).astype(np.float32)
    slots = np.array([0, 5, 39, -1, 13], dtype=np.int64)
    orc.reshape_and_cache(arena, view, F32, hkv, d, tpp, K, V, slots)
    for t, s in enumerate(slots):
        if s < 0:
            continue
        page, off = divmod(int(s), tpp)
        base = view[0] + page * stride
        for h in range(hkv):
            kr = base + ((2 * h + 0) * tpp + off) * d * e  # head-major [Hkv][K|V][tpp][D]
            vr = base + ((2 * h + 1) * tpp + off) * d * e
            np.testing.assert_array_equal(arena[kr:kr + d * e].view(np.float32), K[t, h])
            np.testing.assert_array_equal(arena[vr:vr + d * e].view(np.float32), V[t, h])


def test_oracle_token_rows_overlay_is_reshape_layout(orc):
    """The full_reuse overlay mapping (pieces_per_layer = 2*Hkv, piece = D*e)
    puts row bytes exactly where reshape_and_cache puts that token's K|V, so
    parking an embedding never touches another token's bytes; gather inverts
    scatter for both layouts."""
    rng = np.random.default_rng(9)
    hkv, d, tpp, e, layers = 2, 16, 4, 4, 3
    per_layer = 2 * hkv * tpp * d * e
    stride = layers * per_layer + 64
    arena = rng.integers(0, 256, 8 * stride, dtype=np.uint8)
    slots = np.array([0, 5, 31, -1, 13, 6], dtype=np.int64)
    kv = rng.standard_normal((len(slots), hkv, 2, d)).astype(np.float32)  # row = [h0 K, h0 V, h1 K, ...]
    rows = kv.reshape(len(slots), -1).view(np.uint8)
    a1, a2 = arena.copy(), arena.copy()
    orc.reshape_and_cache(a1, (per_layer, stride, per_layer), F32, hkv, d, tpp, np.ascontiguousarray(kv[:, :, 0]),
                          np.ascontiguousarray(kv[:, :, 1]), slots)
    orc.token_rows_scatter(a2, (per_layer, stride, per_layer), 2 * hkv, d * e, tpp, rows, slots)
    np.testing.assert_array_equal(a1, a2)
    # rows spanning several layers round-trip; negative slots gather zeros
    big = rng.integers(0, 256, (len(slots), 2 * per_layer // tpp), dtype=np.uint8)
    orc.token_rows_scatter(a2, (0, stride, per_layer), 2 * hkv, d * e, tpp, big, slots)
    back = orc.token_rows_gather(a2, (0, stride, per_layer), 2 * hkv, d * e, tpp, big.shape[1], slots)
    want = big.copy()
    want[slots < 0] = 0
    np.testing.assert_array_equal(back, want)
    # vision-group layout: one piece per layer
    emb = rng.integers(0, 256, (len(slots), 48), dtype=np.uint8)
    orc.token_rows_scatter(a2, (16, stride, 48 * tpp), 1, 48, tpp, emb, slots)
    for t, s in enumerate(slots):
        if s >= 0:
            page, off = divmod(int(s), tpp)
            at = 16 + page * stride + off * 48
            np.testing.assert_array_equal(a2[at:at + 48], emb[t])

"""Chunked-prefill measurement on Gemma-2-9B heads:
B requests, each appending a C-token chunk at context n (the chunk's K/V
written by reshape_and_cache — the prefill KV-write path — then causal paged
attention over the whole prefix).  Prints one JSON line per configuration
with the attention TFLOP/s (4*D*Hq per attended (query, key) pair) and the
KV-write GB/s."""
import json
import math
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2503_18292_b200 import ops  # noqa: E402
from paper_2503_18292_b200.engine import DecodeEngine  # noqa: E402
from paper_2503_18292_b200.geometry import gemma2_9b  # noqa: E402


def run(B, ctx, chunk, iters=10, heads=(16, 8, 256), softcap=0.0, quiet=False):
    H, Hkv, D = heads
    geom = gemma2_9b(16)
    for g in geom.groups:
        g.num_layers = 1
        g.num_q_heads, g.num_kv_heads, g.head_dim = H, Hkv, D
    pages = B * (ctx // 16 + 4) * 2 + 16
    eng = DecodeEngine(geom, pages, B, ctx + 64)
    eng.add_requests(range(B))
    for r in range(B):
        eng.pages.set_defer_window_free(r, True)
    eng.arena.tensor().view(torch.bfloat16).normal_()
    for _ in range(ctx):
        eng.append()
    eng.sync_tables()
    T = B * chunk
    cu = torch.arange(0, T + 1, chunk, dtype=torch.int32, device="cuda")
    q = torch.randn((T, H, D), device="cuda").to(torch.bfloat16)
    k = torch.randn((T, Hkv, D), device="cuda").to(torch.bfloat16)
    v = torch.randn_like(k)
    out = torch.empty_like(q)
    req = torch.arange(B, dtype=torch.int32, device="cuda").repeat_interleave(chunk)
    ords = (torch.arange(chunk, dtype=torch.int32, device="cuda") + (ctx - chunk + 1)).repeat(B)
    res = {"B": B, "ctx": ctx, "chunk": chunk, "heads": f"Hq={H} Hkv={Hkv} D={D}", "softcap": softcap}
    for g, name in ((0, "full"), (1, "swa")):
        t = eng.tables[g]
        slots = torch.empty(T, dtype=torch.int64, device="cuda")
        ops.slot_mapping(t.block_table, t.max_blocks, req, ords, 16, slots)
        view = eng.view(g, 0)
        W = geom.groups[g].window

        def once():
            ops.reshape_and_cache(eng.arena, view, k, v, slots, 16)
            ops.paged_prefill(eng.arena, view, int(geom.groups[g].kind), q, out, cu, chunk, t.block_table[:B],
                              t.seq_lens[:B], Hkv, 16, D ** -0.5, window=W, softcap=softcap)
        for _ in range(2):
            once()
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        for _ in range(iters):
            ops.reshape_and_cache(eng.arena, view, k, v, slots, 16)
        e1.record()
        for _ in range(iters):
            ops.paged_prefill(eng.arena, view, int(geom.groups[g].kind), q, out, cu, chunk, t.block_table[:B],
                              t.seq_lens[:B], Hkv, 16, D ** -0.5, window=W, softcap=softcap)
        e2.record()
        torch.cuda.synchronize()
        w_us = e0.elapsed_time(e1) * 1e3 / iters
        a_us = e1.elapsed_time(e2) * 1e3 / iters
        pairs = 0
        for i in range(ctx - chunk, ctx):
            lo = max(0, i + 1 - W) if W else 0
            pairs += i - lo + 1
        flops = 4 * D * H * pairs * B
        res[name] = {"attn_us": round(a_us, 1), "attn_TFLOPs": round(flops / a_us / 1e6, 1),
                     "kv_write_us": round(w_us, 1), "kv_write_GBps": round(2 * T * Hkv * D * 2 * 2 / w_us / 1e3, 1)}
    if not quiet:
        print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    for B, ctx, chunk in ((4, 8192, 2048), (16, 4096, 512), (64, 2048, 256)):
        run(B, ctx, chunk)
    if "--softcap" in sys.argv:  # Gemma-2's attention-logit soft cap (tanh per logit)
        run(4, 8192, 2048, softcap=50.0)
    if "--d128" in sys.argv:  # Llama-3.2 / Jamba attention heads
        for B, ctx, chunk in ((4, 8192, 2048), (16, 4096, 512)):
            run(B, ctx, chunk, heads=(32, 8, 128))

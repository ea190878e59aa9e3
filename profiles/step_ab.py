"""Where the bench step loses time against back-to-back decode launches:
the Gemma shard (32 x 8k, 21 full + 21 SWA layers), one CUDA graph per
variant, 10 replays each:

  decode_only   42 x paged_decode (full / SWA alternating)
  with_kv       42 x (reshape_and_cache + paged_decode)   (bench --unfused)
  fused         42 x paged_decode_append
  fused_tables  table upload + builds + 42 x paged_decode_append (the bench step's device half)

Prints one JSON line: ms per step and GB/s (live KV bytes / time) per variant.
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2503_18292_b200.engine import DecodeEngine  # noqa: E402
from paper_2503_18292_b200.geometry import gemma2_9b  # noqa: E402


def main(B=32, ctx=8192, reps=10):
    geom = gemma2_9b(16)
    eng = DecodeEngine(geom, 25000, B, ctx + 64)
    eng.add_requests(range(B))
    av = eng.arena.tensor().view(torch.bfloat16)
    for s0 in range(0, av.numel(), 1 << 30):
        av[s0:s0 + (1 << 30)].normal_()
    rng = np.random.default_rng(1234)
    order = np.arange(B)
    for pos in range(ctx):
        if pos % 16 == 0:
            order = rng.permutation(B)
        eng.append(list(order))
    eng.sync_tables()
    L = 21
    q = torch.randn((2 * L, B, 16, 256), device="cuda").to(torch.bfloat16)
    kv = torch.randn((2 * L, B, 8, 256), device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    live = sum(int(eng.live_tokens(g).sum()) for g in (0, 1)) * 8192 * L

    def step(mode):
        if mode == "fused_tables":  # + the step's table upload (one H2D copy) and block-table builds
            eng.upload_tables()
        for i in range(2 * L):
            g, layer = i % 2, i // 2
            if mode in ("fused", "fused_tables"):
                eng.decode_append(g, layer, q[i], kv[i], kv[i], out[i])
                continue
            if mode == "with_kv":
                eng.write_kv(g, layer, kv[i], kv[i])
            eng.decode(g, layer, q[i], out[i])

    res = {}
    for name in ("decode_only", "with_kv", "fused", "fused_tables"):
        wk = name
        for _ in range(2):
            step(wk)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            step(wk)
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[name] = {"ms_per_step": round(ms, 3), "GBps": round(live / (ms * 1e-3) / 1e9, 1)}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

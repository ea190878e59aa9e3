"""Decode-kernel tuning sweep on the bench geometry (one full + one SWA-4096
layer, 32 requests x 8k, Gemma-2-9B heads, bf16).  Prints one JSON line per
configuration: per-layer device time and achieved GB/s (algorithmic bytes).

    python profiles/sweep_decode.py            # sweep tiles-per-split in subprocesses
    python profiles/sweep_decode.py --one      # measure the current settings
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def one(batch=32, ctx=8192, iters=20):
    import numpy as np
    import torch

    from paper_2503_18292_b200.engine import DecodeEngine
    from paper_2503_18292_b200.geometry import gemma2_9b

    nl = int(os.environ.get("SWEEP_LAYERS", "1"))
    layer = int(os.environ.get("SWEEP_LAYER", "0"))
    tpp = int(os.environ.get("SWEEP_TPP", "16"))
    geom = gemma2_9b(tpp)
    for g in geom.groups:
        g.num_layers = nl
    pages = batch * (ctx // tpp + 4) + batch * (4096 // tpp + 4)
    eng = DecodeEngine(geom, pages, batch, ctx + 64)
    eng.add_requests(range(batch))
    eng.arena.tensor().view(torch.bfloat16).normal_()
    rng = np.random.default_rng(0)
    order = np.arange(batch)
    for pos in range(ctx):
        if pos % 16 == 0:
            order = rng.permutation(batch)
        eng.append(list(order))
    eng.sync_tables()
    q = torch.randn((batch, 16, 256), device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    res = {"tiles_per_split": os.environ.get("JENGA_DECODE_TILES_PER_SPLIT", "default"), "layers": nl, "layer": layer,
           "prefetch": os.environ.get("JENGA_DECODE_PREFETCH", "0"),
           "grid_order": os.environ.get("JENGA_DECODE_GRID_ORDER", "0"), "tpp": tpp, "hg": os.environ.get("JENGA_DECODE_HEADS_PER_CTA", "auto"),
           "persistent": os.environ.get("JENGA_DECODE_PERSISTENT", "1")}
    bptl = 8192
    for g, name in ((0, "full"), (1, "swa")):
        live = int(eng.live_tokens(g).sum())
        byts = live * bptl + 2 * q.nbytes
        for _ in range(3):
            eng.decode(g, layer, q, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            eng.decode(g, layer, q, out)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / iters
        res[name] = {"us": round(us, 1), "GBps": round(byts / us / 1e3, 1)}
    # read-only roofline reference: torch sum over a 4 GiB bf16 tensor
    x = torch.empty(2 << 30, dtype=torch.bfloat16, device="cuda").normal_()
    for _ in range(3):
        x.sum()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        x.sum()
    e1.record()
    torch.cuda.synchronize()
    res["torch_sum_read_GBps"] = round(x.nbytes * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    if "--one" in sys.argv:
        one()
    else:
        grid = [("0", "1", "32"), ("1", "1", "32"), ("1", "1", "16"), ("1", "4", "16"), ("1", "4", "8"),
                ("1", "2", "16"), ("1", "1", "64")]
        for pers, hg, tps in grid:
            env = dict(os.environ, SWEEP_TPP="16", SWEEP_LAYERS="21", SWEEP_LAYER="0", JENGA_DECODE_HEADS_PER_CTA=hg,
                       JENGA_DECODE_TILES_PER_SPLIT=tps, JENGA_DECODE_PERSISTENT=pers)
            subprocess.run([sys.executable, __file__, "--one"], env=env, check=False)

"""Table upload cost per group and step, Gemma shard shape (32 requests x
8k, tpp 16, 514-block rows): the delta path (table mirror pack on the host +
apply kernel reading the pinned buffer in place) vs the CSR path (pack +
pinned->device copy + build_block_tables), device time of 100 uploads
captured in one graph (so launch overhead does not count), plus the host
pack time per step.  One JSON line per path.

    python profiles/bench_delta_upload.py
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2503_18292_b200.engine import DecodeEngine  # noqa: E402
from paper_2503_18292_b200.geometry import gemma2_9b  # noqa: E402


def run(upload, B=32, ctx=8192, reps=100):
    geom = gemma2_9b(16)
    for gg in geom.groups:
        gg.num_layers = 1
    eng = DecodeEngine(geom, 2 * B * (ctx // 16 + 4) + 64, B, ctx + 256, upload=upload)
    eng.add_requests(range(B))
    rng = np.random.default_rng(0)
    order = np.arange(B)
    for pos in range(ctx):
        if pos % 16 == 0:
            order = rng.permutation(B)
        eng.append(list(order))
    eng.sync_tables()
    torch.cuda.synchronize()
    # host pack time of decode steps
    t0 = time.perf_counter()
    n = 64
    recs = []
    for _ in range(n):
        eng.append()
        tot = eng.pack_tables()
        recs.append(sum(tot.values()))
        eng.upload_tables()
    torch.cuda.synchronize()
    host_us = (time.perf_counter() - t0) / n * 1e6
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            eng.upload_tables()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    dev_us = e0.elapsed_time(e1) / reps * 1e3
    print(json.dumps({"upload": upload, "batch": B, "ctx": ctx, "groups": 2, "device_us_per_step": round(dev_us, 2),
                      "host_us_per_step (append + pack + launch)": round(host_us, 1),
                      "records_or_pages_per_step": float(np.mean(recs)),
                      "bytes_per_step": eng.upload_bytes(tot)}), flush=True)


if __name__ == "__main__":
    run("delta")
    run("full")

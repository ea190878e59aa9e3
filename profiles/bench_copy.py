"""Mamba state gather/scatter measurement (config 3's non-attention traffic):
Jamba-style geometry (bench.py --workload jamba-style), B requests, 28 Mamba
layers; one round = gather + scatter per layer, captured in one CUDA graph
(as the bench runs it).  Prints one JSON line: us per launch and the copy
rate (read + write bytes of a launch / its time), next to a plain
torch copy of the same bytes (contiguous device-to-device, the practical
ceiling for a launch of this size).

    JENGA_COPY_CFG=16,6,2 python profiles/bench_copy.py
"""
import json
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2503_18292_b200 import ops  # noqa: E402
from paper_2503_18292_b200.engine import DecodeEngine  # noqa: E402
from paper_2503_18292_b200.geometry import jamba_style  # noqa: E402
from paper_2503_18292_b200.jenga import LayerKind  # noqa: E402


def timed(fn, reps=10):
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main(B=64):
    geom = jamba_style(16)
    g = [i for i, gg in enumerate(geom.groups) if gg.kind == LayerKind.kMamba][0]
    L = geom.groups[g].num_layers
    eng = DecodeEngine(geom, 2 * B + 16, B, 64)
    eng.add_requests(range(B))
    for _ in range(2):
        eng.append()
    eng.sync_tables()
    eng.arena.tensor().random_(0, 256)
    pg = eng.mamba_page_globals(g)
    views = [eng.view(g, l) for l in range(L)]
    sb = views[0].exec_page_size
    dense = torch.empty((B, sb), dtype=torch.uint8, device="cuda")

    def rounds():
        for v in views:
            ops.mamba_state_gather(eng.arena, v, pg, dense)
            ops.mamba_state_scatter(eng.arena, v, pg, dense)

    us = timed(rounds) / (2 * L)
    src = torch.empty_like(dense)
    dst = torch.empty_like(dense)

    def torch_copies():
        for _ in range(2 * L):
            dst.copy_(src)

    t_us = timed(torch_copies) / (2 * L)
    nbytes = 2 * B * sb  # read + write of one launch
    print(json.dumps({"cfg": os.environ.get("JENGA_COPY_CFG", "16,6,2"),
                      "keep": os.environ.get("JENGA_COPY_L2_KEEP", "1"), "B": B, "state_bytes": sb,
                      "us_per_launch": round(us, 2), "copy_GBps": round(nbytes / us / 1e3, 1),
                      "torch_copy_us": round(t_us, 2), "torch_copy_GBps": round(nbytes / t_us / 1e3, 1)}),
          flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 64)

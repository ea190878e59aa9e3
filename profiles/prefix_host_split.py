"""Host-side split of the prefix-mix warm admission (config 5, B = 256): the
bench's `host_admission_us_per_request` covers admit (lookup_and_pin +
adoption), prefill page stores, the table pack and upload; this times each
part separately on the same flow (round 0 cold, 4 decode appends, cached
release, round 1 warm).  Run on the GPU box:  python profiles/prefix_host_split.py
"""
import json
import sys
import time
import types
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_18292_b200.engine import DecodeEngine  # noqa: E402


def main():
    a = types.SimpleNamespace(workload="prefix-mix", ctx=8192, tpp=16, softcap=None, layers_per_group=21,
                              batch_per_gpu=256, article=1024, question=32, mamba_mode="per-layer")
    wl = bench.Workload(a)
    dev = torch.device("cuda:0")
    eng = DecodeEngine(wl.geom, wl.arena_large_pages(40), wl.B, wl.max_tokens(40), dev, prefix_caching=True)
    ids = list(range(wl.B))
    eng.add_requests(ids)

    def admit_round(q):
        prompts = wl.prefix_prompts(ids, q)
        t = [time.perf_counter()]
        hits = [eng.pages.admit(r, p, now=eng.now) for r, p in zip(ids, prompts)]
        t.append(time.perf_counter())
        for r, p, h in zip(ids, prompts, hits):
            eng.pages.prefill(r, len(p) - h, now=eng.now)
        t.append(time.perf_counter())
        totals = eng.pack_tables()
        t.append(time.perf_counter())
        eng.upload_tables(None, totals)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        us = [(t[i + 1] - t[i]) * 1e6 / len(ids) for i in range(4)]
        return dict(zip(("admit", "prefill", "pack_tables", "upload_sync"), [round(x, 1) for x in us]))

    cold = admit_round(0)
    for _ in range(wl.round0_output):
        eng.append(ids)
    eng.sync_tables()
    t0 = time.perf_counter()
    for r in ids:
        eng.pages.release(r, True, now=eng.now)
    rel = (time.perf_counter() - t0) * 1e6 / len(ids)
    warm = admit_round(1)
    print(json.dumps({"B": wl.B, "us_per_request": {"cold": cold, "cached_release": round(rel, 1), "warm": warm}}))


if __name__ == "__main__":
    main()

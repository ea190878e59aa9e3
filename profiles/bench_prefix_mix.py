"""Config 5 of SURVEY §8(d): the prefix-caching mix, batch sweep 64..1024.

Workload: the reference's multi-article shape (trace.cpp:144-169) — article
prefixes shared across question rounds, questions of question_tokens +
U[0, 16] tokens, a few output tokens — on the Gemma-2-9B attention geometry
(Hq=16, Hkv=8, D=256, bf16, full + SWA-4096, tpp=16; `--layers` per group so
the 1024-request point fits one GPU).  Synthetic token ids (numpy, seeded).

Round 0 (cold): every request prefills its article + question through the
product path (admit -> prefill page lists -> block tables -> reshape_and_cache
-> tcgen05 prefill attention per layer), decodes `--output` tokens, and is
released with caching, so its full blocks become cached pages.
Round 1 (warm): the next question of every article.  Admission pins and
adopts the cached article pages (lookup_and_pin / adopt_lookup_result,
kv_allocator.cpp:241-303, simulator.cpp:391-433) — in the reference's
semantics a pinned page belongs to one running request only — so only the
question tokens are prefilled; then `--steps` decode steps are timed.

Per batch size one JSON line: hit rate, cold vs warm time-to-first-token for
the whole batch (device prefill time + host page-list time), and decode
KV-read GB/s over hit-adopted block tables (algorithmic bytes = live tokens x
bptl per layer, as the headline bench).
"""
import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2503_18292_b200 import AddressMap, ops  # noqa: E402
from paper_2503_18292_b200.engine import DecodeEngine  # noqa: E402
from paper_2503_18292_b200.geometry import gemma2_9b  # noqa: E402


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--batches", default="64,128,256,512,1024")
    p.add_argument("--article", type=int, default=1024)
    p.add_argument("--question", type=int, default=32)
    p.add_argument("--output", type=int, default=4)
    p.add_argument("--layers", type=int, default=4, help="layers per group (full, SWA)")
    p.add_argument("--steps", type=int, default=8)
    p.add_argument("--chunk-requests", type=int, default=64, help="requests per prefill launch")
    return p.parse_args()


def prompt(rng_art, a, q_round, article, question):
    art = np.random.default_rng(1_000_003 * a + 17).integers(1, 1 << 40, article)
    qr = np.random.default_rng(7919 * a + 31 * q_round + 5)
    qlen = question + int(qr.integers(0, 17))
    return [int(x) for x in art] + [int(x) for x in qr.integers(1, 1 << 40, qlen)]


class Runner:
    def __init__(self, a, B):
        self.a, self.B = a, B
        self.geom = gemma2_9b(16)
        for gg in self.geom.groups:
            gg.num_layers = a.layers
        spec = self.geom.spec()
        addr = AddressMap(spec)
        ctx = a.article + a.question + 16 + a.output + a.steps + 16
        smalls = B * (math.ceil(ctx / 16) + 2)
        # two generations of pages (cached round-0 prompts + round-1 tails) + headroom
        pages = 2 * sum(math.ceil(smalls / addr.slots_per_large(g)) for g in range(2)) + 2 * B + 64
        self.eng = DecodeEngine(self.geom, pages, B, ctx + 32, prefix_caching=True)
        self.ids = list(range(B))
        self.eng.add_requests(self.ids)
        self.gen = torch.Generator(device="cuda").manual_seed(0)

    def prefill(self, prompts, starts):
        """Device prefill of prompt positions [start, len) for every request:
        KV write (reshape_and_cache) + causal attention, per layer; returns
        device ms (CUDA events)."""
        eng, B = self.eng, self.B
        H, Hkv, D = 16, 8, 256
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = 0.0
        for r0 in range(0, B, self.a.chunk_requests):
            rs = list(range(r0, min(B, r0 + self.a.chunk_requests)))
            chunks = [len(prompts[r]) - starts[r] for r in rs]
            cu = torch.tensor(np.concatenate([[0], np.cumsum(chunks)]), dtype=torch.int32, device="cuda")
            T = int(sum(chunks))
            if T == 0:
                continue
            req = torch.tensor(np.repeat(np.arange(len(rs)), chunks), dtype=torch.int32, device="cuda")
            ords = torch.tensor(np.concatenate([np.arange(starts[r] + 1, len(prompts[r]) + 1) for r in rs]),
                                dtype=torch.int32, device="cuda")
            q = torch.randn((T, H, D), generator=self.gen, device="cuda").to(torch.bfloat16)
            k = torch.randn((T, Hkv, D), generator=self.gen, device="cuda").to(torch.bfloat16)
            v = torch.randn_like(k)
            out = torch.empty_like(q)
            slots = torch.empty(T, dtype=torch.int64, device="cuda")
            torch.cuda.synchronize()
            e0.record()
            for g in (0, 1):
                t = eng.tables[g]
                bt = t.block_table[r0:r0 + len(rs)]
                ops.slot_mapping(bt, t.max_blocks, req, ords, 16, slots)
                for layer in range(self.a.layers):
                    view = eng.view(g, layer)
                    ops.reshape_and_cache(eng.arena, view, k, v, slots, 16)
                    ops.paged_prefill(eng.arena, view, int(self.geom.groups[g].kind), q, out, cu, max(chunks), bt,
                                      t.seq_lens[r0:r0 + len(rs)], Hkv, 16, D ** -0.5,
                                      window=self.geom.groups[g].window)
            e1.record()
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
        return ms

    def admit_round(self, q_round):
        a, eng = self.a, self.eng
        prompts = [prompt(None, r, q_round, a.article, a.question) for r in self.ids]
        t0 = time.perf_counter()
        hits = [eng.pages.admit(r, prompts[r], now=eng.now) for r in self.ids]
        for r in self.ids:
            n, oom = eng.pages.prefill(r, len(prompts[r]) - hits[r], now=eng.now)
            assert not oom and n == len(prompts[r]) - hits[r], "arena too small"
        eng.sync_tables()
        torch.cuda.synchronize()
        host_ms = (time.perf_counter() - t0) * 1e3
        dev_ms = self.prefill(prompts, hits)
        return prompts, hits, host_ms, dev_ms

    def decode(self, steps, timed):
        eng, B = self.eng, self.B
        q = torch.randn((B, 16, 256), generator=self.gen, device="cuda").to(torch.bfloat16)
        out = torch.empty_like(q)
        k = torch.randn((B, 8, 256), generator=self.gen, device="cuda").to(torch.bfloat16)
        v = torch.randn_like(k)
        live = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            assert eng.append() == B
            eng.sync_tables()
            for layer in range(self.a.layers):
                for g in (0, 1):
                    eng.decode_append(g, layer, q, k, v, out)
            if timed:
                live += sum(int(x) for g in (0, 1) for x in eng.live_tokens(g)) * self.a.layers
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), live

    def run(self):
        a, eng, B = self.a, self.eng, self.B
        prompts0, hits0, host0, dev0 = self.admit_round(0)
        self.decode(a.output, False)
        for r in self.ids:
            eng.pages.release(r, True, now=eng.now)
        cached = eng.kv.cache_entries(0)
        prompts1, hits1, host1, dev1 = self.admit_round(1)
        self.decode(2, False)  # warm-up
        ms, live = self.decode(a.steps, True)
        bptl = 2 * 8 * 256 * 2
        prompt_tokens = sum(len(p) for p in prompts1)
        res = {
            "workload": "prefix-mix (config 5)", "B": B, "layers": 2 * a.layers,
            "article_tokens": a.article, "question_tokens": f"{a.question}+U[0,16]",
            "cached_blocks_after_round0": cached,
            "hit_rate": round(sum(hits1) / prompt_tokens, 4),
            "cold_ttft_ms": {"host_pages": round(host0, 2), "device_prefill": round(dev0, 2)},
            "warm_ttft_ms": {"host_pages": round(host1, 2), "device_prefill": round(dev1, 2)},
            "prefill_speedup": round((host0 + dev0) / max(host1 + dev1, 1e-9), 2),
            "decode_ms_per_step": round(ms / a.steps, 3),
            "decode_GBps": round(live * bptl / (ms / 1e3) / 1e9, 1),
            "decode_tokens_per_s": round(B * a.steps / (ms / 1e3), 1),
        }
        eng.kv.check_invariants()
        return res


def main():
    a = parse()
    for B in (int(x) for x in a.batches.split(",")):
        r = Runner(a, B)
        print(json.dumps(r.run()), flush=True)
        del r
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

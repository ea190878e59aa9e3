#!/usr/bin/env python
"""Benchmark: paged decode through Jenga's two-level page table on B200.

One step = one decode step of the Gemma-2-9B geometry (BASELINE.json
configs[1]): host allocator appends one token per request (store_position
semantics), page lists are uploaded and block tables rebuilt on the device,
then for each of the 42 layers (21 full + 21 SWA-4096) the new token's K/V
is scattered into its slot (reshape_and_cache) and paged decode attention
reads every live K/V byte through the layer view of the HBM arena.

The headline 256 x 8k batch holds 541 GB of KV and does not fit one GPU, so
each GPU owns a 32-request shard (67.6 GB, the G=8 shard of the headline
batch).  `--gpus N` runs N ranks, one process per GPU — started here through
torch.distributed.run (127.0.0.1) unless a launcher already set WORLD_SIZE —
each owning N x 32 / N requests, its own allocator and arena, with no
inter-GPU traffic on the hot path ("scaling": "weak").  After the timed
region NCCL gathers sampled requests' outputs and layer slices to rank 0,
which checks them against the C oracle ("verified").

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"]


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="gemma2-9b",
                   choices=["gemma2-9b", "jamba-style", "llama-3.2-11b-vision", "prefix-mix"])
    p.add_argument("--article", type=int, default=1024, help="prefix-mix: shared article tokens")
    p.add_argument("--question", type=int, default=32, help="prefix-mix: question tokens (+U[0,16])")
    p.add_argument("--batch-per-gpu", type=int, default=0, help="0: the workload's default")
    p.add_argument("--ctx", type=int, default=8192)
    p.add_argument("--tpp", type=int, default=16)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-prefill", action="store_true",
                   help="skip the chunked-prefill line added to the gemma2-9b result (after the timed decode)")
    p.add_argument("--e2e-timeline", action="store_true",
                   help="profiling only (with --no-graph): print when each input chunk lands vs when its first layer starts")
    p.add_argument("--e2e-chunks", default="geo", choices=["geo", "3"],
                   help="layer chunks of the e2e copies: geometric (1, 2, 4, ... layers: each chunk lands while "
                        "the layers before it run) or three each way (the round-2 first-session form)")
    p.add_argument("--e2e-io", default="overlap", choices=["overlap", "serial", "none", "in-only", "out-only"],
                   help="profiling only: how the e2e leg moves q/k/v and outputs (overlap = the measured "
                        "contract: side-stream chunks; serial = before / after the step on its stream; "
                        "none = no copies, isolates the per-step host synchronisation)")
    p.add_argument("--unfused", action="store_true",
                   help="separate reshape_and_cache + paged_decode launches instead of jenga_paged_decode_append")
    p.add_argument("--no-graph", action="store_true", help="launch every kernel eagerly instead of one CUDA graph "
                                                          "per step")
    p.add_argument("--layers-per-group", type=int, default=21)
    p.add_argument("--softcap", type=float, default=None, help="attention-logit soft cap (default: the model's; "
                                                               "Gemma-2: 50)")
    p.add_argument("--mamba-mode", default="per-layer", choices=["per-layer", "fused-step", "gather-scatter"],
                   help="jamba-style: how a step moves the Mamba states through the page table — one in-place "
                        "update launch for all Mamba layers (fused-step), one per layer in model order "
                        "(per-layer), or the unfused gather -> dense -> scatter pair per layer (gather-scatter)")
    p.add_argument("--mamba-decay", type=float, default=0.999,
                   help="stand-in SSM update of the in-place modes: fp32 state *= decay")
    return p.parse_args()


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


def workload_desc(a):
    return (f"gemma2-9b decode: {a.batch_per_gpu or 32} req/GPU x {a.ctx} ctx, {2 * a.layers_per_group} layers "
            f"({a.layers_per_group} full + {a.layers_per_group} SWA-4096), Hq=16 Hkv=8 D=256, tpp={a.tpp}, "
            f"logit softcap 50")


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=5)
        rows = [r.split(",") for r in out.strip().splitlines() if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------- workloads
class Workload:
    """One BASELINE.json config as a decode loop: layer schedule in model
    order, prompt construction and algorithmic byte accounting."""

    def __init__(self, a):
        from paper_2503_18292_b200.geometry import gemma2_9b, jamba_style, llama32_11b_vision
        self.name = a.workload
        self.ctx = a.ctx
        self.image_tokens = 0
        self.prefix_caching = False
        from paper_2503_18292_b200.geometry import gemma2_9b as _g
        gemma2_9b = (lambda tpp: _g(tpp, softcap=a.softcap)) if a.softcap is not None else _g
        if a.workload == "prefix-mix":
            # BASELINE configs[4]: the reference's multi-article shape (trace.cpp:144-169) on the
            # Gemma-2-9B geometry — every request's prompt = a shared article + a question;
            # round 0 prefills cold and is released into the prefix cache, round 1 asks the
            # next question of every article and adopts the cached article pages
            self.geom = gemma2_9b(a.tpp)
            for gg in self.geom.groups:
                gg.num_layers = a.layers_per_group
            self.B = a.batch_per_gpu or 256
            L = a.layers_per_group
            self.layers = [(g, l) for l in range(L) for g in (0, 1)]
            self.prefix_caching = True
            self.article, self.question, self.round0_output = a.article, a.question, 4
            self.ctx = a.article + a.question + 16
            self.desc = (f"prefix-mix (config 5) decode on gemma2-9b geometry: {self.B} req/GPU, prompts = "
                         f"{a.article}-token shared article + {a.question}+U[0,16]-token question, round 1 "
                         f"adopting round 0's cached article pages; {2 * L} layers ({L} full + {L} SWA-4096), "
                         f"Hq=16 Hkv=8 D=256, tpp={a.tpp}, logit softcap {self.geom.softcap:g}")
        elif a.workload == "gemma2-9b":
            self.geom = gemma2_9b(a.tpp)
            for gg in self.geom.groups:
                gg.num_layers = a.layers_per_group
            self.B = a.batch_per_gpu or 32
            L = a.layers_per_group
            self.layers = [(g, l) for l in range(L) for g in (0, 1)]  # alternating full / SWA
            self.desc = (f"gemma2-9b decode: {self.B} req/GPU x {a.ctx} ctx, {2 * L} layers ({L} full + {L} "
                         f"SWA-4096), Hq=16 Hkv=8 D=256, tpp={a.tpp}, logit softcap {self.geom.softcap:g}")
        elif a.workload == "jamba-style":
            self.geom = jamba_style(a.tpp)
            self.B = a.batch_per_gpu or 64
            self.layers = []
            for i in range(4):  # one attention layer per 8 (Jamba), 28 Mamba layers
                self.layers.append((0, i))
                self.layers += [(1, 7 * i + j) for j in range(7)]
            self.desc = (f"jamba-style hybrid decode: {self.B} req/GPU x {a.ctx} ctx, 4 attention layers (Hq=32 Hkv=8 "
                         f"D=128 bf16, tpp={a.tpp}) + 28 Mamba layers with fp32 last-token state pages "
                         f"(622,592 B/layer) in the same LCM pool; state traffic: " +
                         {"fused-step": "one in-place update launch per step for all 28 Mamba layers (state read "
                                        "+ written back through the page table, fp32 *= decay as the SSM stand-in)",
                          "per-layer": "one in-place update launch per Mamba layer in model order",
                          "gather-scatter": "per layer, gather to a dense buffer then scatter back"}[a.mamba_mode])
        elif a.workload == "llama-3.2-11b-vision":
            self.geom = llama32_11b_vision(a.tpp)
            self.B = a.batch_per_gpu or 64
            self.image_tokens = 6404  # one image = 4 tiles x 1601 tokens
            self.layers = []
            for i in range(8):  # a cross-attention layer after every 4 self-attention layers
                self.layers += [(0, 4 * i + j) for j in range(4)]
                self.layers.append((1, i))
            self.desc = (f"llama-3.2-11b-vision decode: {self.B} req/GPU x {a.ctx} text ctx + {self.image_tokens} "
                         f"image tokens, 32 self-attention + 8 cross-attention layers, Hq=32 Hkv=8 D=128 bf16, "
                         f"tpp={a.tpp}")
        else:
            raise SystemExit(f"unknown workload {a.workload}")
        self.spec = self.geom.spec()

    def max_tokens(self, steps):
        extra = self.round0_output if self.prefix_caching else 0
        return max(self.ctx + self.image_tokens + steps + extra + 16, 64)

    def group_max_tokens(self, steps):
        """Per-group ordinal bounds: cross-attention groups store image
        positions only, decoder groups text only when the model has cross
        attention (simulator.cpp:151-158)."""
        from paper_2503_18292_b200.jenga import LayerKind
        if not self.image_tokens:
            return None
        return {g: (self.image_tokens + 16 if gg.kind == LayerKind.kCrossAttention else self.ctx + steps + 16)
                for g, gg in enumerate(self.geom.groups)}

    def arena_large_pages(self, steps):
        from paper_2503_18292_b200 import AddressMap
        from paper_2503_18292_b200.jenga import LayerKind
        addr = AddressMap(self.spec)
        total = 0
        for g, gg in enumerate(self.geom.groups):
            tpp = self.spec.groups[g].tokens_per_page
            if gg.kind == LayerKind.kMamba:
                smalls = self.B
            elif gg.kind == LayerKind.kCrossAttention:
                smalls = self.B * (math.ceil(self.image_tokens / tpp) + 1)
            elif gg.kind == LayerKind.kSlidingWindow:
                smalls = self.B * (math.ceil(min(gg.window, self.ctx + steps + 16) / tpp) + 2)
            else:
                smalls = self.B * (math.ceil((self.ctx + steps + 16) / tpp) + 1)
            if self.prefix_caching:  # round 0's cached prompts + round 1's own question / decode pages
                smalls = self.B * (math.ceil((self.ctx + self.round0_output) / tpp) + 2 +
                                   math.ceil((self.question + 16 + steps) / tpp) + 2)
            total += math.ceil(smalls / addr.slots_per_large(g)) + self.B  # request-aware units
        return total + 8

    def prefix_prompts(self, ids, q_round):
        """Article id = request id (one question per article per round)."""
        out = []
        for r in ids:
            art = np.random.default_rng(1_000_003 * r + 17).integers(1, 1 << 40, self.article)
            qr = np.random.default_rng(7919 * r + 31 * q_round + 5)
            n = self.question + int(qr.integers(0, 17))
            out.append(np.concatenate([art, qr.integers(1, 1 << 40, n)]).astype(np.uint64))  # token ids as an array
        return out

    def prefix_setup(self, eng, ids, dev, chunk_requests=32):
        """Rounds 0 and 1 of the prefix mix through the product path: admission
        (lookup_and_pin + adoption), page lists, then per chunk of requests and
        per layer slot_mapping + reshape_and_cache + tcgen05 paged_prefill of the
        positions the hit did not cover.  Round 0 then decodes a few tokens and
        is released with caching.  Returns hit rate and cold / warm TTFT."""
        import torch

        from paper_2503_18292_b200 import ops
        g0 = self.geom.groups[0]
        H, Hkv, D, tpp = g0.num_q_heads, g0.num_kv_heads, g0.head_dim, self.spec.groups[0].tokens_per_page
        gen = torch.Generator(device=dev).manual_seed(11)
        rows = {r: i for i, r in enumerate(eng.requests)}

        def admit_round(q_round):
            prompts = self.prefix_prompts(ids, q_round)
            t0 = time.perf_counter()
            hits = [eng.pages.admit(r, p, now=eng.now) for r, p in zip(ids, prompts)]
            for r, p, h in zip(ids, prompts, hits):
                n, oom = eng.pages.prefill(r, len(p) - h, now=eng.now)
                assert not oom and n == len(p) - h, "arena too small for the prefix mix"
            eng.sync_tables()
            torch.cuda.synchronize()
            host_ms = (time.perf_counter() - t0) * 1e3
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dev_ms = 0.0
            for c0 in range(0, len(ids), chunk_requests):
                part = list(range(c0, min(len(ids), c0 + chunk_requests)))
                chunks = [len(prompts[i]) - hits[i] for i in part]
                T = int(sum(chunks))
                if T == 0:
                    continue
                b0 = rows[ids[part[0]]]
                cu = torch.tensor(np.concatenate([[0], np.cumsum(chunks)]), dtype=torch.int32, device=dev)
                req = torch.tensor(np.repeat(np.arange(len(part)), chunks), dtype=torch.int32, device=dev)
                ords = torch.tensor(np.concatenate([np.arange(hits[i] + 1, len(prompts[i]) + 1) for i in part]),
                                    dtype=torch.int32, device=dev)
                q = torch.randn((T, H, D), generator=gen, device=dev).to(torch.bfloat16)
                k = torch.randn((T, Hkv, D), generator=gen, device=dev).to(torch.bfloat16)
                v = torch.randn_like(k)
                out = torch.empty_like(q)
                slots = torch.empty(T, dtype=torch.int64, device=dev)
                torch.cuda.synchronize()
                e0.record()
                for g, gg in enumerate(self.geom.groups):
                    t = eng.tables[g]
                    bt = t.block_table[b0:b0 + len(part)]
                    ops.slot_mapping(bt, t.max_blocks, req, ords, tpp, slots)
                    for layer in range(gg.num_layers):
                        view = eng.view(g, layer)
                        ops.reshape_and_cache(eng.arena, view, k, v, slots, tpp)
                        ops.paged_prefill(eng.arena, view, int(gg.kind), q, out, cu, max(chunks), bt,
                                          t.seq_lens[b0:b0 + len(part)], Hkv, tpp, D ** -0.5, window=gg.window,
                                          softcap=self.geom.softcap)
                e1.record()
                torch.cuda.synchronize()
                dev_ms += e0.elapsed_time(e1)
            return prompts, hits, host_ms, dev_ms

        _, _, host0, dev0 = admit_round(0)
        for _ in range(self.round0_output):  # round 0's answers (page lists only; KV values irrelevant here)
            assert eng.append(ids) == len(ids)
        eng.sync_tables()
        for r in ids:
            eng.pages.release(r, True, now=eng.now)
        cached = eng.kv.cache_entries(0)
        prompts1, hits1, host1, dev1 = admit_round(1)
        eng.kv.check_invariants()
        return {"hit_rate": round(sum(hits1) / sum(len(p) for p in prompts1), 4),
                "cached_blocks_after_round0": int(cached),
                "cold_ttft_ms": {"host_pages": round(host0, 2), "device_prefill": round(dev0, 2)},
                "warm_ttft_ms": {"host_pages": round(host1, 2), "device_prefill": round(dev1, 2)},
                "host_admission_us_per_request": round(host1 * 1e3 / len(ids), 1)}

    def prompt(self, eng, ids, rank):
        """Interleaved prompt: images first (cross groups store them), then text;
        seeded request order per 16-position chunk so pages interleave."""
        rng = np.random.default_rng(1234 + rank)
        B = len(ids)
        order = np.arange(B)
        n_img = self.image_tokens
        for pos in range(n_img + self.ctx - 1):
            if pos % 16 == 0:
                order = rng.permutation(B)
            img = [1] * B if pos < n_img else None
            done = eng.append([ids[i] for i in order], is_image=img)
            assert done == B


# --------------------------------------------------------------------- our arm
def run_ours(a, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2503_18292_b200 import ops
    from paper_2503_18292_b200.distributed import gather_rows, max_over_ranks, shard_requests, sum_over_ranks
    from paper_2503_18292_b200.engine import DecodeEngine
    from paper_2503_18292_b200.jenga import LayerKind

    local_dev = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device(f"cuda:{local_dev}")
    wl = Workload(a)
    B = wl.B
    # every host append of the run: warm-up + timed steps, the per-launch event pass
    # (k_steps below), graph warm-up / capture steps, and the e2e leg (pipelined one
    # step ahead) — the tables and the arena are sized for all of them
    total_steps = (a.warmup + a.steps + max(3, a.steps // 4) + 8 +
                   (0 if a.no_e2e else a.warmup + a.steps + 4))
    eng = DecodeEngine(wl.geom, wl.arena_large_pages(total_steps), B, wl.max_tokens(total_steps), dev,
                       group_max_tokens=wl.group_max_tokens(total_steps), prefix_caching=wl.prefix_caching)
    ids = shard_requests(list(range(B * world)), rank, world)  # this GPU's requests; its pool is private
    eng.add_requests(ids)
    t0 = time.time()
    av = eng.arena.tensor().view(torch.bfloat16)  # finite random KV / state bytes (values only)
    chunk = 1 << 30
    for s in range(0, av.numel(), chunk):
        av[s:s + chunk].normal_()
    prefix_stats = None
    if wl.prefix_caching:
        prefix_stats = wl.prefix_setup(eng, ids, dev)
    else:
        wl.prompt(eng, ids, rank)
    torch.cuda.synchronize()
    setup_s = time.time() - t0

    attn = [(i, g, l) for i, (g, l) in enumerate(wl.layers) if eng.tables[g].geom.is_attention]
    mamba = [(i, g, l) for i, (g, l) in enumerate(wl.layers) if eng.tables[g].geom.kind == LayerKind.kMamba]
    gen = torch.Generator(device=dev).manual_seed(1 + rank)
    g0 = eng.tables[attn[0][1]].geom
    H, Hkv, D = g0.num_q_heads, g0.num_kv_heads, g0.head_dim
    na = len(attn)
    q = torch.randn((na, B, H, D), generator=gen, device=dev).to(g0.dtype)
    kn = torch.randn((na, B, Hkv, D), generator=gen, device=dev).to(g0.dtype)
    vn = torch.randn((na, B, Hkv, D), generator=gen, device=dev).to(g0.dtype)
    out = torch.empty_like(q)
    state = None
    if mamba and a.mamba_mode == "gather-scatter":
        state = torch.empty((B, eng.view(mamba[0][1], 0).exec_page_size), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    bptl = 2 * Hkv * D * 2
    slot = {i: j for j, (i, _, _) in enumerate(attn)}
    attn_layers_per_group = {}
    for _, g, _ in attn:
        attn_layers_per_group[g] = attn_layers_per_group.get(g, 0) + 1

    # The pinned page-list buffer is reused every step: pack_tables waits until the
    # previous upload's H2D copy has read it (DecodeEngine records an event after
    # the copy, also inside the captured graph), so the host runs at most one step
    # ahead and every step uploads its own tables.
    def host_step():
        """Host half of a step: allocator append + CSR pack into pinned memory."""
        eng.append()
        return eng.pack_tables()

    def device_step(totals=None, ev=None, hooks=None, attention=True, upload=True):
        """Device half: table upload, then per layer KV write + decode (fixed
        shape, so it can be graph-captured).  attention=False: everything but
        the attention launches (the roofline's subtrahend)."""
        if upload:
            eng.upload_tables(None, totals)
        pg = {}
        for i, (g, l) in enumerate(wl.layers):
            kind = eng.tables[g].geom.kind
            if kind != LayerKind.kMamba and not attention:
                continue
            if kind == LayerKind.kMamba:
                first = g not in pg
                if first:
                    pg[g] = eng.mamba_page_globals(g)
                v = eng.view(g, l)
                if a.mamba_mode == "gather-scatter":
                    ops.mamba_state_gather(eng.arena, v, pg[g], state)   # last-token state -> dense
                    ops.mamba_state_scatter(eng.arena, v, pg[g], state)  # (SSM update out of scope)
                elif a.mamba_mode == "per-layer":
                    ops.mamba_state_update(eng.arena, v, 1, pg[g], a.mamba_decay)
                elif first:  # fused-step: every Mamba layer of the group in one launch
                    ops.mamba_state_update(eng.arena, eng.view(g, 0), eng.tables[g].geom.num_layers, pg[g],
                                           a.mamba_decay)
                continue
            j = slot[i]
            if hooks is not None:
                hooks["before"](j)
            fused = kind != LayerKind.kCrossAttention and not a.unfused
            if kind != LayerKind.kCrossAttention and a.unfused:  # cross KV (image tokens) is static in decode
                eng.write_kv(g, l, kn[j], vn[j])
            if ev is not None:
                ev[j][0].record(stream)
            if fused:  # newest token's K/V appended by the decode launch itself
                eng.decode_append(g, l, q[j], kn[j], vn[j], out[j])
            else:
                eng.decode(g, l, q[j], out[j])
            if ev is not None:
                ev[j][1].record(stream)
            if hooks is not None:
                hooks["after"](j)

    def step(ev=None, hooks=None):
        device_step(host_step(), ev, hooks)

    graph = None
    per_replay = 0
    if not a.no_graph:
        # capture the device half once (after warm-up: tensor maps, smem
        # attributes); each step then = host append + pack + one graph launch
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        host_step()
        c0 = ops.kernel_launch_count()
        with torch.cuda.graph(graph):
            device_step()
        per_replay = ops.kernel_launch_count() - c0
        graph.replay()
        torch.cuda.synchronize()

    def timed_step():
        if graph is None:
            step()
        else:
            host_step()
            graph.replay()

    def step_bytes():
        """(KV bytes read by decode, Mamba state bytes moved) for this step."""
        kv = 0
        for g, n_layers in attn_layers_per_group.items():  # one host read per group, not per layer
            kv += int(eng.live_tokens(g).sum()) * bptl * n_layers
        st = 0
        for _, g, l in mamba:
            st += 2 * B * eng.view(g, l).exec_page_size
        return kv, st

    for _ in range(a.warmup):
        timed_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kv_bytes = st_bytes = 0
    clk = ClockSampler(local_dev)
    clk.start()
    launches0 = ops.kernel_launch_count()
    torch.cuda.synchronize()
    start.record(stream)
    for s in range(a.steps):
        timed_step()  # no per-layer events here: they would break programmatic (PDL) overlap
        kb, sb = step_bytes()
        kv_bytes += kb
        st_bytes += sb
    end.record(stream)
    torch.cuda.synchronize()
    launches = ops.kernel_launch_count() - launches0 + (a.steps * per_replay if graph is not None else 0)
    ms = start.elapsed_time(end)
    ms_local = ms
    # Attention launches' own time inside the PDL-chained graph: the same step
    # without them (table upload + Mamba copies) is captured and timed alone,
    # decode time = step time - that.  (Events between launches would break
    # the PDL overlap the timed step runs with.)
    k_steps = max(3, a.steps // 4)
    k_rest = 20
    rest_graph = None
    if graph is not None:  # k_rest copies in one graph: GPU time, not launch overhead
        rest_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(rest_graph):
            for _ in range(k_rest):
                device_step(attention=False)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    r0.record(stream)
    if rest_graph is not None:
        rest_graph.replay()
    else:
        for _ in range(k_rest):
            device_step(attention=False)
    r1.record(stream)
    torch.cuda.synchronize()
    rest_ms = r0.elapsed_time(r1) / k_rest
    # secondary evidence: CUDA events around every attention launch of a few
    # eager steps (no graph, no PDL overlap across the events)
    evs = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in attn]
           for _ in range(k_steps)]
    kv_prof = 0
    for s_ in range(k_steps):
        step(evs[s_])
        kv_prof += step_bytes()[0]
    torch.cuda.synchronize()
    clocks = clk.stop()
    ev_ms = sum(e0.elapsed_time(e1) for st in evs for e0, e1 in st)
    kv_local = kv_bytes
    moved = kv_bytes + st_bytes
    if world > 1:
        ms = max_over_ranks(ms, dev)                   # timed on the device, max over ranks
        moved = int(sum_over_ranks(moved, dev))        # whole-job bytes
    ms_per_step = ms / a.steps
    qo_step = 2 * na * B * H * D * 2                   # q read + out write of one step's decode launches
    dec_ms_step = ms_local / a.steps - rest_ms         # attention launches per step, in the graph
    dec_gbs = (kv_local / a.steps + qo_step) / (dec_ms_step * 1e-3) / 1e9
    ev_gbs = (kv_prof + qo_step * k_steps) / (ev_ms * 1e-3) / 1e9
    qo = qo_step * a.steps

    # ---------------- e2e: host buffers through the public API each step
    e2e = None
    if not a.no_e2e:
        hq = torch.empty_like(q, device="cpu").pin_memory()
        hk = torch.empty_like(kn, device="cpu").pin_memory()
        hv = torch.empty_like(vn, device="cpu").pin_memory()
        ho = torch.empty_like(out, device="cpu").pin_memory()
        hq.copy_(q)
        hk.copy_(kn)
        hv.copy_(vn)

        # Copies ride a side stream in layer chunks: later inputs land while the
        # first layers decode, outputs leave while the last layers decode.  Every
        # cross-stream wait / event record inside the step breaks the PDL chain
        # (~15 us each: one chunk per layer costs +0.6 ms a step), so the chunks grow
        # geometrically (1, 2, 4, ... layers): each chunk lands while the layers
        # before it run.  The step's page-table delta is uploaded before the chunk
        # copies are queued — they share the H2D copy engine, and behind them the
        # table copy held layer 0 back by their whole transfer time (the round-2
        # first-session e2e lost 0.45 ms a Gemma step and 3 ms a prefix-mix step to
        # exactly that; --e2e-timeline shows when each chunk lands vs its layer).
        cs = torch.cuda.Stream(device=dev)
        if a.e2e_chunks == "geo":  # 1, 2, 4, ... layers: each chunk's copy hides behind the previous chunk's layers
            geo = [0]
            while geo[-1] < na:
                geo.append(min(na, 2 * geo[-1] + 1))
            in_bounds = geo
            out_bounds = sorted({na - x for x in geo})
        else:
            in_bounds = sorted({0, min(1, na), min(3, na), na})
            out_bounds = sorted({0, max(na - 3, 0), max(na - 1, 0), na})
        ev_in = [torch.cuda.Event(enable_timing=a.e2e_timeline) for _ in range(len(in_bounds) - 1)]
        tl = {"t0": torch.cuda.Event(enable_timing=True),
              "layer": [torch.cuda.Event(enable_timing=True) for _ in range(na)]} \
            if a.e2e_timeline and graph is None else None  # eager steps only
        ev_out = [torch.cuda.Event() for _ in range(len(out_bounds) - 1)]
        in_start = {in_bounds[c]: c for c in range(len(in_bounds) - 1)}
        out_end = {out_bounds[c + 1] - 1: c for c in range(len(out_bounds) - 1)}

        def e2e_device(totals):
            if a.e2e_io not in ("overlap", "in-only", "out-only"):
                if a.e2e_io == "serial":
                    q.copy_(hq, non_blocking=True)
                    kn.copy_(hk, non_blocking=True)
                    vn.copy_(hv, non_blocking=True)
                device_step(totals)
                if a.e2e_io == "serial":
                    ho.copy_(out, non_blocking=True)
                return
            if tl is not None:
                tl["t0"].record(torch.cuda.current_stream())
            # the page-table delta first: the chunk copies below share the H2D copy engine,
            # and queued behind them the table copy held layer 0 back by their whole
            # transfer time (--e2e-timeline: layer 0 started 0.51 ms into the step, 0.43
            # ms after the q/k/v chunks had been queued)
            eng.upload_tables(None, totals)
            cs.wait_stream(torch.cuda.current_stream())  # previous step's readers of q/k/v are done
            with torch.cuda.stream(cs):
                for c in range(len(in_bounds) - 1):
                    if a.e2e_io == "out-only":
                        ev_in[c].record(cs)
                        continue
                    lo, hi = in_bounds[c], in_bounds[c + 1]
                    q[lo:hi].copy_(hq[lo:hi], non_blocking=True)
                    kn[lo:hi].copy_(hk[lo:hi], non_blocking=True)
                    vn[lo:hi].copy_(hv[lo:hi], non_blocking=True)
                    ev_in[c].record(cs)
            cur = torch.cuda.current_stream()
            def before(j):
                if j in in_start:
                    cur.wait_event(ev_in[in_start[j]])
                if tl is not None:
                    tl["layer"][j].record(cur)
            chunk_hooks = {"before": before,
                           "after": lambda j: ev_out[out_end[j]].record(cur) if j in out_end else None}
            device_step(totals, hooks=chunk_hooks, upload=False)
            for c in range(len(out_bounds) - 1):
                cs.wait_event(ev_out[c])
                if a.e2e_io == "in-only":
                    continue
                with torch.cuda.stream(cs):
                    lo, hi = out_bounds[c], out_bounds[c + 1]
                    ho[lo:hi].copy_(out[lo:hi], non_blocking=True)
            cur.wait_stream(cs)

        e2e_graph = None
        if graph is not None:
            host_step()
            e2e_graph = torch.cuda.CUDAGraph()
            c0 = ops.kernel_launch_count()
            with torch.cuda.graph(e2e_graph):
                e2e_device(None)
            e2e_per_replay = ops.kernel_launch_count() - c0
            e2e_graph.replay()
            torch.cuda.synchronize()

        pending = {"totals": None, "pl_bytes": 0}

        def e2e_step():
            """Launch this step (its tables were packed during the previous
            step), pack the next step's page lists on the host while the GPU
            runs, then read this step's result.  Returns this step's bytes."""
            if pending["totals"] is None:
                pending["totals"] = host_step()
            nbytes = sum(step_bytes())
            pending["pl_bytes"] += eng.upload_bytes(pending["totals"])  # page lists the device reads this step
            if e2e_graph is None:
                e2e_device(pending["totals"])
            else:
                e2e_graph.replay()
            pending["totals"] = host_step()
            stream.synchronize()  # the caller reads the step's result
            return nbytes
        for _ in range(a.warmup):
            e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e_bytes = 0
        pending["pl_bytes"] = 0
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(a.steps):
            e_bytes += e2e_step()
        s1.record(stream)
        torch.cuda.synchronize()
        e_ms = s0.elapsed_time(s1)
        if world > 1:
            e_ms = max_over_ranks(e_ms, dev)
            e_bytes = int(sum_over_ranks(e_bytes, dev))
        if tl is not None:
            torch.cuda.synchronize()
            rows = [f"chunk {in_bounds[c]}-{in_bounds[c + 1]} landed {tl['t0'].elapsed_time(ev_in[c]):.3f} ms; "
                    f"layer {in_bounds[c]} started {tl['t0'].elapsed_time(tl['layer'][in_bounds[c]]):.3f} ms"
                    for c in range(len(in_bounds) - 1)]
            rows.append(f"last layer started {tl['t0'].elapsed_time(tl['layer'][na - 1]):.3f} ms")
            print("e2e timeline (last step): " + " | ".join(rows), file=sys.stderr)
        e2e = {"value": round(e_bytes / (e_ms * 1e-3) / 1e9, 1), "unit": "GB/s",
               "h2d_bytes_per_step": int(q.nbytes + kn.nbytes + vn.nbytes + pending["pl_bytes"] / a.steps),
               "d2h_bytes_per_step": int(out.nbytes),
               "page_list_bytes_per_step": int(pending["pl_bytes"] / a.steps),
               "ms_per_step": round(e_ms / a.steps, 3),
               "tokens_per_s": round(B * world * a.steps / (e_ms * 1e-3), 1)}

    # ---------------- verification (outside the timed region): sampled requests'
    # outputs + their layer slices gathered to rank 0 (NCCL), checked there
    # against the C oracle
    finite = bool(torch.isfinite(out.float()).all().item())
    verification = verify_outputs(eng, q, out, attn, rank, world, dev)

    pk, src = peaks()
    value = moved / (ms * 1e-3) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "decode_traffic.json"
    if tf.exists():  # ncu --set full capture of this exact workload (profiles/run_ncu.sh), else null
        try:
            tj = json.loads(tf.read_text())
            if tj.get("workload") == wl.desc and tj.get("kernel_launches_per_step") == na:
                traffic = tj.get("traffic_bytes_per_launch")
        except Exception:
            traffic = None
    kname = (f"paged_decode_tc_kernel<bf16, D={D}, G={H // Hkv}> (TMA + mma.sync" +
             ("" if a.unfused else ", newest K/V appended in the same launch") + ")")
    res = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random N(0,1) bf16 KV/q; page lists from the "
                                                    "native Jenga allocator, seeded interleaved request order)",
        "config": {"workload": wl.desc, "global_batch": B * world, "seq_len": wl.ctx,
                   "parallelism": f"dp{world} (request shards, independent Jenga pool per GPU)",
                   "l2": "inputs larger than L2 (arena %.1f GB/GPU vs 126 MB L2); no flush needed"
                         % (eng.arena.nbytes / 1e9)},
        "tokens_per_s": round(B * world * a.steps / (ms * 1e-3), 1),
        "frac_of_hbm_peak": round(value / world / pk["hbm_gbs"], 4),
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": round(dec_gbs, 1),
                     "peak": pk["hbm_gbs"], "peak_source": src, "unit": "GB/s",
                     "frac": round(dec_gbs / pk["hbm_gbs"], 4), "traffic": traffic,
                     "decode_share_of_step": round(dec_ms_step / (ms_local / a.steps), 4),
                     "timing": f"attention launches' time inside the timed graph = step time - the same step "
                               f"without them (table upload{' + Mamba copies' if mamba else ''}: "
                               f"{rest_ms * 1e3:.1f} us, {k_rest} copies in one graph)",
                     "eager_events_gbs": round(ev_gbs, 1),
                     "algorithmic_bytes_per_step": int((kv_local + qo) / a.steps),
                     "algorithmic_bytes_per_launch": int((kv_local + qo) / a.steps / na)},
        "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
        "setup_s": round(setup_s, 1), "outputs_finite": finite,
    }
    if verification is not None:
        res["verification"] = verification
        res["verified"] = verification["verified"] and finite
    if st_bytes:
        res["mamba_state_bytes_per_step"] = int(st_bytes / a.steps)
    if prefix_stats is not None:
        res["prefix_mix"] = prefix_stats
    return res


# --------------------------------------------------------------------- verification
def verify_outputs(eng, q, out, attn, rank, world, dev):
    """Every rank exports, for the last layer of each attention group, one
    sampled request (a different one per rank): its q and output rows, its
    block-table row remapped onto a compact copy of its live pages' layer
    slices, and its seq_len.  One all-gather per group (NCCL over NVLink)
    brings them to rank 0, which recomputes each row with the C oracle (fp64)
    and checks the bf16 tolerance of north_star (1e-2, normwise per row:
    max|got - want| / max|want|).  Returns the summary on rank 0, else None."""
    import torch

    from paper_2503_18292_b200.distributed import gather_padded

    B = len(eng.requests)
    last = {}
    for j, (_, g, l) in enumerate(attn):
        last[g] = (j, l)
    b = rank % B
    gathered = []
    for g, (j, l) in sorted(last.items()):
        data, table, seq = eng.export_request_layer(g, l, b)
        head = torch.tensor([g, l, b, rank, table.numel(), data.numel()], dtype=torch.int64, device=dev)
        payload = torch.cat([head.view(torch.uint8), table.contiguous().view(torch.uint8), seq.view(torch.uint8),
                             q[j, b].contiguous().view(torch.uint8).reshape(-1),
                             out[j, b].contiguous().view(torch.uint8).reshape(-1), data])
        gathered.append((gather_padded(payload) if world > 1 else payload.view(1, -1)).cpu().numpy())
    if rank != 0:
        return None
    from oracle import c_oracle
    from oracle.oracle import BF16
    orc = c_oracle()
    errs = []
    for rows in gathered:
        for r in range(rows.shape[0]):
            buf = rows[r]
            g, l, bb, rk, nt, nd = (int(x) for x in buf[:48].view(np.int64))
            gg = eng.tables[g].geom
            H, Hkv, D = gg.num_q_heads, gg.num_kv_heads, gg.head_dim
            o = 48
            table = buf[o:o + 4 * nt].view(np.int32).reshape(1, nt)
            o += 4 * nt
            seq = buf[o:o + 4].view(np.int32).copy()
            o += 4
            qrow = buf[o:o + 2 * H * D].view(np.int16).reshape(1, H, D)
            o += 2 * H * D
            got = (buf[o:o + 2 * H * D].view(np.uint16).astype(np.uint32) << 16).view(np.float32).reshape(1, H, D)
            o += 2 * H * D
            data = np.ascontiguousarray(buf[o:o + nd])
            ex = eng.view(g, l).exec_page_size
            want = orc.paged_decode(data, (0, ex, ex), int(gg.kind), BF16, gg.window, np.ascontiguousarray(qrow),
                                    table, seq, H, Hkv, D, eng.spec.groups[g].tokens_per_page, D ** -0.5,
                                    eng.geom.softcap, nthreads=os.cpu_count() or 1)
            errs.append(float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-30)))
    tol = 1e-2
    return {"verified": bool(errs) and max(errs) <= tol, "samples": len(errs), "max_rel_err": max(errs),
            "tolerance": tol,
            "how": "rank 0 gathers (NCCL all-gather) one sampled request per rank and attention group - q/out rows, "
                   "block-table row and a compact copy of its live layer slices - and recomputes the last layer's "
                   "decode with the C oracle (fp64); error normwise per row"}


# --------------------------------------------------------------------- CPU baselines
def cpu_sample(a, steps=1, nthreads=None, requests=16, single_core=False):
    """The reference CPU path on a bounded sample of the same workload:
    reference KvAllocator page lists (oracle/_ref when built, else the native
    port's restatement) + reference AddressMap views, then the C attention
    oracle over one full + one SWA-4096 layer for `requests` requests at the
    workload's context, all host threads."""
    from oracle import c_oracle, ref_lib
    from oracle.oracle import BF16, FULL, SWA, RefPageLists

    nthreads = nthreads or os.cpu_count() or 1
    orc = c_oracle()
    ref = ref_lib()
    B, ctx, tpp, H, Hkv, D = requests, a.ctx, a.tpp, 16, 8, 256
    bptl = 2 * Hkv * D * 2
    spec = json.dumps({"name": "gemma2-sample", "groups": [
        {"name": "full", "kind": "full", "num_layers": 1, "bytes_per_token_per_layer": bptl, "tokens_per_page": tpp},
        {"name": "window", "kind": "sliding_window", "num_layers": 1, "bytes_per_token_per_layer": bptl,
         "tokens_per_page": tpp, "window_tokens": 4096}]})
    small = bptl * tpp
    pages = B * (ctx // tpp + 2) + B * (4096 // tpp + 3) + 8
    kind = "reference" if ref is not None else "port"
    rng = np.random.default_rng(0)
    t_tables = 0.0
    if ref is not None:
        rs = ref.spec(spec)
        rkv = rs.kv(pages * small)
        rpl = RefPageLists(rkv)
        addr = rs.address_map()
        ids = list(range(B))
        t0 = time.perf_counter()
        order = np.arange(B)
        for pos in range(ctx):
            if pos % 16 == 0:
                order = rng.permutation(B)
            rpl.append_batch(order)
        maxb = ctx // tpp + 2
        tables = [rpl.block_table(addr, g, ids, maxb) for g in range(2)]
        for g in range(2):
            rpl.resolve_views(addr, g, ids)
        t_tables = time.perf_counter() - t0
    else:
        from paper_2503_18292_b200 import AddressMap, KvAllocator, ModelSpec, PageLists
        ms = ModelSpec.from_json(spec)
        kv = KvAllocator(ms, pages * small)
        pl = PageLists(kv)
        ids = list(range(B))
        for r in ids:
            pl.add_request(r)
        t0 = time.perf_counter()
        for pos in range(ctx):
            pl.append_batch(ids)
        maxb = ctx // tpp + 2
        tables = []
        for g in range(2):
            off, pg, l0, ns = pl.pack_csr(g, ids)
            tables.append(orc.build_block_tables(off, pg, l0, ns, 1, tpp, maxb)[0])
        t_tables = time.perf_counter() - t0
    arena = rng.integers(0, 1 << 16, size=pages * small // 2, dtype=np.uint16)
    arena &= 0xBFFF  # keep finite bf16 (exponent < 0xFF)
    arena = arena.view(np.uint8)
    q = (rng.standard_normal((B, H, D)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    seq = np.full(B, ctx, dtype=np.int32)
    t0 = time.perf_counter()
    for _ in range(steps):
        orc.paged_decode(arena, (0, small, small), FULL, BF16, 0, q, tables[0], seq, H, Hkv, D, tpp, 1 / 16,
                         50.0, nthreads=nthreads)
        orc.paged_decode(arena, (0, small, small), SWA, BF16, 4096, q, tables[1], seq, H, Hkv, D, tpp, 1 / 16,
                         50.0, nthreads=nthreads)
    t_attn = (time.perf_counter() - t0) / steps
    kv_bytes = B * (ctx + min(4096, ctx)) * bptl
    extra = {}
    if single_core:  # the attention oracle on all host cores and on one
        t1 = time.perf_counter()
        orc.paged_decode(arena, (0, small, small), FULL, BF16, 0, q, tables[0], seq, H, Hkv, D, tpp, 1 / 16, 50.0,
                         nthreads=1)
        orc.paged_decode(arena, (0, small, small), SWA, BF16, 4096, q, tables[1], seq, H, Hkv, D, tpp, 1 / 16,
                         50.0, nthreads=1)
        t1 = time.perf_counter() - t1
        extra = {"single_core_GBps": round(kv_bytes / (t1 + t_tables / max(ctx, 1)) / 1e9, 3)}
    return {"value": round(kv_bytes / (t_attn + t_tables / max(ctx, 1)) / 1e9, 3), "unit": "GB/s",
            "cores": nthreads, "kind": kind,
            "sample": f"{B} requests x {ctx} ctx, 1 full + 1 SWA-4096 layer (Gemma-2-9B heads, bf16); page lists "
                      f"from the {'reference' if kind == 'reference' else 'native'} KvAllocator; attention by the "
                      f"C oracle (fp64) on {nthreads} threads",
            "attention_s_per_layer_pair": round(t_attn, 4),
            "page_table_build_s": round(t_tables, 4), **extra}


def run_reference(a):
    a_ctx = a
    res0 = cpu_sample(a_ctx, steps=1)
    t0 = time.perf_counter()
    vals = []
    for _ in range(a.warmup):
        cpu_sample(a_ctx, steps=1)
    t1 = time.perf_counter()
    for _ in range(a.steps):
        vals.append(cpu_sample(a_ctx, steps=1)["value"])
    el = time.perf_counter() - t1
    v = float(np.mean(vals)) if vals else res0["value"]
    cb = dict(res0)
    cb["value"] = round(v, 3)
    return {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "GB/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(el / max(a.steps, 1) * 1e3, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic", "config": {"workload": workload_desc(a) + " — CPU sample: " + res0["sample"],
                                            "global_batch": (a.batch_per_gpu or 32) * a.gpus, "seq_len": a.ctx,
                                            "parallelism": "host cores"},
            "cpu_baseline": cb, "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}


def prefill_line(a):
    """SURVEY §8(f) row 1 next to the decode result (outside its timed region): the
    chunked-prefill attention of the same model's layers -- 4 requests x 2048-token
    chunks at 8k context, Gemma-2-9B heads (Hq=16, Hkv=8, D=256), the model's logit
    softcap and without it, full and SWA-4096 layers -- as TFLOP/s (4*D*Hq flop per
    attended (query, key) pair; CUDA events, 10 launches after 2 warm-ups) against the
    measured cuBLAS bf16 peak."""
    import gc

    import torch
    gc.collect()
    torch.cuda.empty_cache()
    sys.path.insert(0, str(ROOT / "profiles"))
    import bench_prefill
    cap = a.softcap if a.softcap is not None else 50.0
    plain = bench_prefill.run(4, 8192, 2048, quiet=True)
    capped = bench_prefill.run(4, 8192, 2048, softcap=cap, quiet=True)
    pk, src = peaks()
    tf = plain["full"]["attn_TFLOPs"]
    return {"metric": "chunked-prefill attention TFLOP/s (4*D*Hq flop per attended pair)",
            "kernel": "paged_prefill_tc5_wide_kernel<bf16, D=256, G=2> (persistent tcgen05 CTA pairs)",
            "config": "4 requests x 2048-token chunks at 8192 context, Gemma-2-9B heads, bf16",
            "value": tf, "unit": "TFLOP/s", "peak": pk.get("bf16_tflops"), "peak_source": src,
            "frac": round(tf / pk["bf16_tflops"], 4) if pk.get("bf16_tflops") else None,
            "swa_4096": plain["swa"]["attn_TFLOPs"],
            f"softcap_{cap:g}": {"full": capped["full"]["attn_TFLOPs"], "swa_4096": capped["swa"]["attn_TFLOPs"]},
            "kv_write_GBps": plain["full"]["kv_write_GBps"]}


def main():
    a = parse()
    if a.impl == "ours" and a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-run this script as a.gpus ranks (torch.distributed.run, 127.0.0.1)
        from paper_2503_18292_b200.distributed import launch_local_ranks
        sys.exit(launch_local_ranks(str(Path(__file__).resolve()), sys.argv[1:], a.gpus))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if a.impl == "reference":
        if rank == 0:
            # bounded: each step is one ~seconds-long CPU sample
            a.steps = min(a.steps, 3)
            a.warmup = min(a.warmup, 1)
            print(json.dumps(run_reference(a)), flush=True)
        return
    if world != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but the launcher started {world} ranks")
    import torch
    import torch.distributed as dist
    if world > 1:
        backend = os.environ.get("JENGA_BENCH_BACKEND", "nccl")  # gloo only for 1-GPU rehearsals
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        else:
            dist.init_process_group(backend)
    res = run_ours(a, rank, world, local_rank)
    if rank == 0 and world == 1 and not a.no_prefill and a.workload == "gemma2-9b":
        try:
            res["prefill"] = prefill_line(a)
        except Exception as e:  # the extra line must not sink the decode result
            res["prefill"] = {"value": None, "error": str(e)[:200]}
    if rank == 0 and world == 1 and not a.no_cpu_baseline and a.workload in ("gemma2-9b", "prefix-mix"):
        from paper_2503_18292_b200.geometry import gemma2_9b as _g
        gemma2_9b = (lambda tpp: _g(tpp, softcap=a.softcap)) if a.softcap is not None else _g
        if a.workload == "prefix-mix":
            a.ctx = a.article + a.question
        try:
            res["cpu_baseline"] = cpu_sample(a, steps=1, single_core=True)
        except Exception as e:  # the baseline must not sink the GPU line
            res["cpu_baseline"] = {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "port",
                                   "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

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
batch); `--gpus N` shards N x 32 requests with no inter-GPU traffic on the
hot path ("scaling": "weak"); NCCL only gathers outputs for verification
after the timed region.

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
    p.add_argument("--batch-per-gpu", type=int, default=32)
    p.add_argument("--ctx", type=int, default=8192)
    p.add_argument("--tpp", type=int, default=16)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--layers-per-group", type=int, default=21)
    return p.parse_args()


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


def workload_desc(a):
    return (f"gemma2-9b decode: {a.batch_per_gpu} req/GPU x {a.ctx} ctx, {2 * a.layers_per_group} layers "
            f"({a.layers_per_group} full + {a.layers_per_group} SWA-4096), Hq=16 Hkv=8 D=256, tpp={a.tpp}")


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


# --------------------------------------------------------------------- our arm
def run_ours(a, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2503_18292_b200 import ops
    from paper_2503_18292_b200.distributed import gather_rows, max_over_ranks
    from paper_2503_18292_b200.engine import DecodeEngine
    from paper_2503_18292_b200.geometry import gemma2_9b

    torch.cuda.set_device(local_rank)
    dev = torch.device(f"cuda:{local_rank}")
    geom = gemma2_9b(a.tpp)
    for gg in geom.groups:
        gg.num_layers = a.layers_per_group
    B = a.batch_per_gpu
    total_steps = a.warmup + a.steps + (0 if a.no_e2e else a.warmup + a.steps) + 2
    max_tokens = a.ctx + total_steps + 16
    # exact arena sizing: full group grows to max_tokens; SWA keeps <= W + tpp
    spl_pages = B * (math.ceil(max_tokens / a.tpp) + 1) + B * (math.ceil(4096 / a.tpp) + 2) + 16
    eng = DecodeEngine(geom, spl_pages, B, max_tokens, dev)
    from paper_2503_18292_b200.distributed import shard_requests
    ids = shard_requests(list(range(B * world)), rank, world)  # this GPU's requests; pool is private
    eng.add_requests(ids)
    # fill the arena with finite bf16 KV (contents are never re-derived: values only)
    t0 = time.time()
    av = eng.arena.tensor().view(torch.bfloat16)
    chunk = 1 << 30
    for s in range(0, av.numel(), chunk):
        av[s:s + chunk].normal_()
    # prefill page lists to ctx-1 tokens, interleaved (seeded order per 16-position chunk)
    rng = np.random.default_rng(1234 + rank)
    order = np.arange(B)
    for pos in range(a.ctx - 1):
        if pos % 16 == 0:
            order = rng.permutation(B)
        done = eng.append([ids[i] for i in order])
        assert done == B
    torch.cuda.synchronize()
    setup_s = time.time() - t0

    H, D, Hkv = 16, 256, 8
    nl = 2 * a.layers_per_group
    gen = torch.Generator(device=dev).manual_seed(1 + rank)
    q = torch.randn((nl, B, H, D), generator=gen, device=dev).to(torch.bfloat16)
    kn = torch.randn((nl, B, Hkv, D), generator=gen, device=dev).to(torch.bfloat16)
    vn = torch.randn((nl, B, Hkv, D), generator=gen, device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    layers = [(g, l) for l in range(a.layers_per_group) for g in (0, 1)]  # alternating full / SWA
    stream = torch.cuda.current_stream()

    bptl = 2 * Hkv * D * 2

    def step(ev=None):
        eng.append()
        eng.sync_tables()
        for i, (g, l) in enumerate(layers):
            eng.write_kv(g, l, kn[i], vn[i])
            if ev is not None:
                ev[i][0].record(stream)
            eng.decode(g, l, q[i], out[i])
            if ev is not None:
                ev[i][1].record(stream)

    def live_bytes():
        full = eng.live_tokens(0).sum()
        win = eng.live_tokens(1).sum()
        return int((full + win) * a.layers_per_group * bptl), int((full + win) * a.layers_per_group)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in layers]
           for _ in range(a.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kv_bytes = 0
    kv_tokens = 0
    clk = ClockSampler(local_rank)
    clk.start()
    launches0 = ops.kernel_launch_count()
    torch.cuda.synchronize()
    start.record(stream)
    for s in range(a.steps):
        step(evs[s])
        b, t = live_bytes()
        kv_bytes += b
        kv_tokens += t
    end.record(stream)
    torch.cuda.synchronize()
    launches = ops.kernel_launch_count() - launches0
    clocks = clk.stop()
    ms = start.elapsed_time(end)
    dec_ms = sum(e0.elapsed_time(e1) for st in evs for e0, e1 in st)
    kv_bytes_local = kv_bytes
    if world > 1:
        ms = max_over_ranks(ms, dev)           # timed on the device, max over ranks
        t = torch.tensor([kv_bytes], device=dev, dtype=torch.float64)
        dist.all_reduce(t)                     # whole-job bytes
        kv_bytes = int(t.item())
    ms_per_step = ms / a.steps
    # algorithmic bytes of the decode kernel: live K/V + q read + out write
    qo = 2 * nl * B * H * D * 2 * a.steps
    dec_gbs = (kv_bytes_local + qo) / (dec_ms * 1e-3) / 1e9

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

        def e2e_step():
            q.copy_(hq, non_blocking=True)
            kn.copy_(hk, non_blocking=True)
            vn.copy_(hv, non_blocking=True)
            step()
            ho.copy_(out, non_blocking=True)
            torch.cuda.current_stream().synchronize()  # the caller reads the step's result
        for _ in range(a.warmup):
            e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e_bytes = 0
        t0 = time.perf_counter()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(a.steps):
            e2e_step()
            e_bytes += live_bytes()[0]
        s1.record(stream)
        torch.cuda.synchronize()
        e_ms = s0.elapsed_time(s1)
        if world > 1:
            e_ms = max_over_ranks(e_ms, dev)
        e_val = e_bytes * world / (e_ms * 1e-3) / 1e9
        e2e = {"value": round(e_val, 1), "unit": "GB/s", "h2d_bytes_per_step": int(q.nbytes + kn.nbytes + vn.nbytes),
               "d2h_bytes_per_step": int(out.nbytes), "ms_per_step": round(e_ms / a.steps, 3),
               "tokens_per_s": round(B * world * a.steps / (e_ms * 1e-3), 1)}

    # ---------------- verification gather (NCCL, outside the timed region)
    finite = bool(torch.isfinite(out.float()).all().item())
    if world > 1:
        gathered = gather_rows(out[-1])        # NCCL all-gather of the last layer's outputs
        finite = finite and bool(torch.isfinite(gathered.float()).all().item())

    pk, src = peaks()
    value = kv_bytes / (ms * 1e-3) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "decode_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("traffic_bytes_per_launch")
        except Exception:
            traffic = None
    res = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random N(0,1) bf16 KV/q; page lists from the "
                                                    "native Jenga allocator, seeded interleaved request order)",
        "config": {"workload": workload_desc(a), "global_batch": B * world, "seq_len": a.ctx,
                   "parallelism": f"dp{world} (request shards, independent Jenga pool per GPU)",
                   "l2": "inputs larger than L2 (KV arena %.1f GB/GPU vs 126 MB L2); no flush needed"
                         % (eng.arena.nbytes / 1e9)},
        "tokens_per_s": round(B * world * a.steps / (ms * 1e-3), 1),
        "frac_of_hbm_peak": round(value / world / pk["hbm_gbs"], 4),
        "roofline": {"bound": "hbm", "kernel": "paged_decode_tc_kernel<bf16, D=256, G=2> (TMA + mma.sync)", "achieved": round(dec_gbs, 1),
                     "peak": pk["hbm_gbs"], "peak_source": src, "unit": "GB/s",
                     "frac": round(dec_gbs / pk["hbm_gbs"], 4), "traffic": traffic,
                     "decode_share_of_step": round(dec_ms / (ms_per_step * a.steps), 4),
                     "algorithmic_bytes_per_step": int((kv_bytes + qo) / a.steps)},
        "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
        "setup_s": round(setup_s, 1), "outputs_finite": finite,
    }
    return res


# --------------------------------------------------------------------- CPU baselines
def cpu_sample(a, steps=1, nthreads=None, requests=4):
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
                         nthreads=nthreads)
        orc.paged_decode(arena, (0, small, small), SWA, BF16, 4096, q, tables[1], seq, H, Hkv, D, tpp, 1 / 16,
                         nthreads=nthreads)
    t_attn = (time.perf_counter() - t0) / steps
    kv_bytes = B * (ctx + min(4096, ctx)) * bptl
    return {"value": round(kv_bytes / (t_attn + t_tables / max(ctx, 1)) / 1e9, 3), "unit": "GB/s",
            "cores": nthreads, "kind": kind,
            "sample": f"{B} requests x {ctx} ctx, 1 full + 1 SWA-4096 layer (Gemma-2-9B heads, bf16); page lists "
                      f"from the {'reference' if kind == 'reference' else 'native'} KvAllocator; attention by the "
                      f"C oracle (fp64) on {nthreads} threads",
            "attention_s_per_layer_pair": round(t_attn, 4),
            "page_table_build_s": round(t_tables, 4)}


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
                                            "global_batch": a.batch_per_gpu * a.gpus, "seq_len": a.ctx,
                                            "parallelism": "host cores"},
            "cpu_baseline": cb, "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}


def main():
    a = parse()
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
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    res = run_ours(a, rank, world, local_rank)
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            res["cpu_baseline"] = cpu_sample(a, steps=1)
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

"""Regenerate the golden fixtures in tests/golden/ by running the REFERENCE
ITSELF (oracle/_ref/libjenga_ref.so, compiled from /root/reference sources).

    python tests/golden/make_golden.py

Fixtures (all deterministic, seeded):
  fig6.json              AddressMap on the Fig-6 geometry
                         (reference proj/tests/test_memory_layout.cpp:16-33, 67-191)
  configs.json           bundled model configs with small pages / LCM / blow-up
                         (proj/configs/*.cfg, proj/tests/test_model_config.cpp:259-272)
  random_geometries.json address tables of random geometries (memory_layout
                         sweep of test_memory_layout.cpp:154-181, numpy seeded)
  alloc_sequences.json   KvAllocator op sequences and the reference outcomes
  policies.json          LayerPolicy needs_token / accessed_range tables
  sim_pages.json         SimEngine page lists after N steps on small traces
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref_lib  # noqa: E402
from oracle.oracle import RefKv, RefSim  # noqa: E402

OUT = Path(__file__).resolve().parent
REF_CONFIGS = Path("/root/reference/proj/configs")


def spec_json(name, groups):
    return json.dumps({"name": name, "groups": groups})


FIG6 = spec_json("fig6", [
    {"name": "cross", "kind": "cross_attention", "num_layers": 2, "bytes_per_token_per_layer": 128},
    {"name": "self", "kind": "full", "num_layers": 3, "bytes_per_token_per_layer": 128}])


def fig6(ref):
    s = ref.spec(FIG6)
    m = s.address_map()
    out = {"spec": json.loads(FIG6), "large_page_bytes": m.info(0)[0], "groups": [], "entries": []}
    for g in range(2):
        _, small, per_layer, slots = m.info(g)
        out["groups"].append({"small_page_bytes": small, "per_layer_bytes": per_layer, "slots_per_large": slots,
                              "views": [list(m.layer_view(g, l)) for l in range(s.json["groups"][g]["num_layers"])]})
        for lp in range(4):
            for slot in range(slots):
                for layer in range(s.json["groups"][g]["num_layers"]):
                    out["entries"].append({"g": g, "layer": layer, "large": lp, "slot": slot,
                                           "global": m.global_page_index(g, (lp, slot)),
                                           "range": list(m.address_of(g, layer, (lp, slot))),
                                           "view": list(m.view_address(g, layer, (lp, slot)))})
    out["dump1"] = m.dump(1)
    return out


def configs(ref):
    out = []
    for p in sorted(REF_CONFIGS.glob("*.cfg")):
        text = p.read_text()
        s = ref.spec(text)
        n = len(s.json["groups"])
        out.append({"file": p.name, "json": text, "small_pages": [s.small_page_size(g) for g in range(n)],
                    "lcm": s.lcm_page_size(), "blowup": s.lcm_blowup_ratio()})
    return out


def random_geometries(ref, n=100, seed=4242):
    rng = np.random.default_rng(seed)
    sizes = [8, 16, 24, 32, 48, 64, 96, 128]
    out = []
    while len(out) < n:
        ng = int(rng.integers(1, 5))
        groups = [{"name": f"g{i}", "kind": "full", "num_layers": int(rng.integers(1, 9)),
                   "bytes_per_token_per_layer": sizes[int(rng.integers(0, 8))],
                   "tokens_per_page": int(rng.integers(1, 4))} for i in range(ng)]
        text = spec_json("rand", groups)
        s = ref.spec(text)
        m = s.address_map()
        total = sum(m.info(g)[3] * groups[g]["num_layers"] for g in range(ng))
        if total > 4000:
            continue
        entries = []
        for g in range(ng):
            _, small, per_layer, slots = m.info(g)
            for slot in range(slots):
                for layer in range(groups[g]["num_layers"]):
                    entries.append([g, layer, g, slot, m.global_page_index(g, (g, slot)),
                                    *m.address_of(g, layer, (g, slot))])
        out.append({"json": text, "large": m.info(0)[0], "entries": entries})
    return out


TWO_GROUP = spec_json("pair", [
    {"name": "a", "kind": "full", "num_layers": 3, "bytes_per_token_per_layer": 128},
    {"name": "b", "kind": "full", "num_layers": 6, "bytes_per_token_per_layer": 128}])


def alloc_sequences(ref, seeds=(1234, 77, 5, 6), n_ops=3000):
    """Random allocate/free(cached)/pin/evict/touch sequences on the
    test_type_allocator two-group geometry (proj/tests/test_type_allocator.cpp:15-29)."""
    out = []
    for seed in seeds:
        rng = np.random.default_rng(seed)
        budget = int(rng.choice([2, 4, 8, 16])) * 768
        s = ref.spec(TWO_GROUP)
        kv = s.kv(budget)
        ops, used, cached, clock = [], [], [], 0
        for _ in range(n_ops):
            g = int(rng.integers(0, 2))
            req = int(rng.integers(1, 4))
            a = int(rng.integers(0, 10))
            if a < 5:
                r = kv.allocate(g, req)
                clock += 1
                ops.append(["alloc", g, req, None if r is None else [r[0][0], r[0][1], r[1]]])
                if r is not None:
                    kv.touch(g, r[0], clock)
                    ops.append(["touch", g, list(r[0]), clock])
                    used.append((g, r[0]))
            elif a < 8 and used:
                i = int(rng.integers(0, len(used)))
                fg, page = used.pop(i)
                if rng.integers(0, 2) == 0:
                    ops.append(["free", fg, list(page), None])
                    kv.free(fg, page)
                else:
                    tag = int(rng.integers(0, 1 << 62))
                    content = [tag, 0, [tag]]
                    kv.set_prefix_length(fg, page, int(rng.integers(0, 100)))
                    ops.append(["prefix", fg, list(page), kv.record(fg, page)["prefix_length"]])
                    ops.append(["free", fg, list(page), content])
                    kv.free(fg, page, content)
                    cached.append((fg, content))
            elif a < 9 and cached:
                i = int(rng.integers(0, len(cached)))
                cg, content = cached.pop(i)
                page = kv.cache_find(cg, content)
                ops.append(["find", cg, content, None if page is None else list(page)])
                if page is not None:
                    kv.pin(cg, page, req)
                    ops.append(["pin", cg, list(page), req])
                    used.append((cg, page))
            else:
                ev = kv.evict()
                ops.append(["evict", ev])
            kv.check_invariants()
        counts = [kv.counts(g) for g in range(2)]
        frag = [kv.fragmentation(g) for g in range(2)]
        out.append({"seed": seed, "budget": budget, "ops": ops, "final_counts": counts, "final_frag": frag})
    return out


def policies(ref):
    out = []
    for kind, w in (("full", 0), ("sliding_window", 4), ("sliding_window", 7), ("mamba", 0), ("cross_attention", 0),
                    ("vision_embedding", 0)):
        g = {"name": "g", "kind": kind, "num_layers": 1, "bytes_per_token_per_layer": 8}
        if w:
            g["window_tokens"] = w
        if kind == "mamba":
            g["checkpoint_interval_tokens"] = 5
        s = ref.spec(spec_json("p", [g]))
        needs = [[i, n, c, int(s.needs_token(0, i, n, c))] for n in range(1, 16) for i in range(1, n + 1)
                 for c in (0, n // 2)]
        acc = [[p, n, *s.accessed_range(0, p, n)] for n in range(0, 16) for p in range(0, n + 1)]
        out.append({"group": g, "needs_token": needs, "accessed_range": acc})
    return out


SIM_MODELS = {
    "window": spec_json("win", [
        {"name": "self", "kind": "full", "num_layers": 8, "bytes_per_token_per_layer": 128, "tokens_per_page": 4},
        {"name": "window", "kind": "sliding_window", "num_layers": 28, "bytes_per_token_per_layer": 128,
         "window_tokens": 64, "tokens_per_page": 4}]),
    "mllama": spec_json("mllama", [
        {"name": "self", "kind": "full", "num_layers": 4, "bytes_per_token_per_layer": 128, "tokens_per_page": 4},
        {"name": "cross", "kind": "cross_attention", "num_layers": 2, "bytes_per_token_per_layer": 128,
         "tokens_per_page": 4}]),
    "hybrid": spec_json("hybrid", [
        {"name": "attn", "kind": "full", "num_layers": 4, "bytes_per_token_per_layer": 128},
        {"name": "ssm", "kind": "mamba", "num_layers": 8, "bytes_per_token_per_layer": 1024,
         "checkpoint_interval_tokens": 50}]),
}


def sim_pages(ref):
    out = []
    cases = [
        ("window", 64 << 20, 32, False, [{"id": i, "segments": [[0, 37 + 11 * i]], "output": 90} for i in range(5)],
         [3, 10, 40, 80]),
        ("mllama", 64 << 20, 48, False,
         [{"id": i, "segments": [[0, 5], [1, 21 + 3 * i], [0, 9]], "output": 30} for i in range(4)], [2, 6, 20]),
        ("hybrid", 32 << 20, 64, True, [{"id": 0, "segments": [[0, 175]], "output": 30}], [2, 5, 25]),
        ("hybrid", 32 << 20, 64, False, [{"id": i, "segments": [[0, 60 + i]], "output": 12} for i in range(3)],
         [1, 4, 9]),
    ]
    for model, budget, chunk, caching, reqs, checkpoints in cases:
        s = ref.spec(SIM_MODELS[model])
        sim = RefSim(s, budget, chunk, caching, reqs)
        snaps = []
        step = 0
        for target in checkpoints:
            while step < target and not sim.done():
                sim.step()
                step += 1
            snap = {"step": step, "requests": []}
            for r in reqs:
                rq = sim.request(r["id"])
                toks, img = sim.tokens(r["id"])
                groups = []
                for g in range(len(json.loads(SIM_MODELS[model])["groups"])):
                    st = sim.group_state(r["id"], g)
                    groups.append({"pages": st["pages"].tolist(), "live": st["live"].astype(int).tolist(),
                                   "stored": st["stored"], "freed": st["freed"],
                                   "working": None if st["working"] is None else [int(x) for x in st["working"]]})
                snap["requests"].append({"id": r["id"], "phase": rq["phase"], "seq_len": rq["seq_len"],
                                         "consumed": rq["consumed"], "tokens": [str(int(t)) for t in toks],
                                         "is_image": img.astype(int).tolist(), "groups": groups})
            snaps.append(snap)
        out.append({"model": model, "spec": json.loads(SIM_MODELS[model]), "budget": budget, "chunk": chunk,
                    "prefix_caching": caching, "requests": reqs, "snapshots": snaps})
    return out


def _snapshot(sim, reqs, ng, step):
    snap = {"step": step, "requests": []}
    for r in reqs:
        rq = sim.request(r["id"])
        toks, img = sim.tokens(r["id"])
        groups = []
        for g in range(ng):
            st = sim.group_state(r["id"], g)
            groups.append({"pages": st["pages"].tolist(), "live": st["live"].astype(int).tolist(),
                           "stored": st["stored"], "freed": st["freed"],
                           "working": None if st["working"] is None else [int(x) for x in st["working"]]})
        snap["requests"].append({"id": r["id"], "phase": rq["phase"], "seq_len": rq["seq_len"],
                                 "consumed": rq["consumed"], "tokens": [str(int(t)) for t in toks],
                                 "is_image": img.astype(int).tolist(), "groups": groups})
    return snap


VISION_MODELS = {
    # cross-attention VLM: images stored by the cross group only
    "mllama_vis": spec_json("mllama-vis", [
        {"name": "self", "kind": "full", "num_layers": 4, "bytes_per_token_per_layer": 128, "tokens_per_page": 4},
        {"name": "cross", "kind": "cross_attention", "num_layers": 2, "bytes_per_token_per_layer": 128,
         "tokens_per_page": 4},
        {"name": "vision", "kind": "vision_embedding", "num_layers": 1, "bytes_per_token_per_layer": 320,
         "tokens_per_page": 3}]),
    # decoder-only VLM (llava-style): the decoder stores image tokens too
    "llava_vis": spec_json("llava-vis", [
        {"name": "self", "kind": "full", "num_layers": 3, "bytes_per_token_per_layer": 128, "tokens_per_page": 4},
        {"name": "window", "kind": "sliding_window", "num_layers": 2, "bytes_per_token_per_layer": 128,
         "window_tokens": 24, "tokens_per_page": 4},
        {"name": "vision", "kind": "vision_embedding", "num_layers": 1, "bytes_per_token_per_layer": 512,
         "tokens_per_page": 2}]),
}


def sim_vision(ref):
    """Reference SimEngine in both vision modes (simulator.cpp:453-476,
    504-547): on_demand frees consumed embeddings, full_reuse allocates the
    whole prompt at admission."""
    out = []
    for model, mode, budget, chunk, reqs, checkpoints in (
            ("mllama_vis", 0, 64 << 20, 16,
             [{"id": i, "segments": [[0, 5], [1, 21 + 3 * i], [0, 9], [1, 7]], "output": 12} for i in range(3)],
             [1, 2, 3, 5, 8, 14]),
            ("mllama_vis", 1, 64 << 20, 16,
             [{"id": i, "segments": [[0, 5], [1, 21 + 3 * i], [0, 9]], "output": 12} for i in range(3)],
             [1, 2, 4, 7, 14]),
            ("llava_vis", 0, 64 << 20, 20,
             [{"id": i, "segments": [[0, 3 + i], [1, 30], [0, 11]], "output": 40} for i in range(3)],
             [1, 2, 3, 6, 12, 40]),
            ("llava_vis", 1, 64 << 20, 20,
             [{"id": i, "segments": [[0, 3 + i], [1, 30], [0, 11]], "output": 40} for i in range(3)],
             [1, 2, 3, 6, 12, 40])):
        s = ref.spec(VISION_MODELS[model])
        sim = RefSim(s, budget, chunk, False, reqs, vision_mode=mode)
        ng = len(json.loads(VISION_MODELS[model])["groups"])
        snaps, step = [], 0
        for target in checkpoints:
            while step < target and not sim.done():
                sim.step()
                step += 1
            snaps.append(_snapshot(sim, reqs, ng, step))
        out.append({"model": model, "spec": json.loads(VISION_MODELS[model]), "vision_mode": mode,
                    "budget": budget, "chunk": chunk, "requests": reqs, "snapshots": snaps})
    return out


def sim_spec(ref):
    """Reference SimEngine with a speculative config (simulator.cpp:32-41,
    568-640): draft groups in the same LCM pool, rollback of rejections."""
    from oracle.oracle import spec_accept_draws
    draft = spec_json("draft", [
        {"name": "self", "kind": "full", "num_layers": 1, "bytes_per_token_per_layer": 64, "tokens_per_page": 4}])
    out = []
    for model, k, acc, seed, reqs, checkpoints in (
            ("window", 4, 0.7, 11, [{"id": i, "segments": [[0, 19 + 9 * i]], "output": 60} for i in range(4)],
             [2, 5, 9, 17, 30]),
            ("window", 3, 0.0, 12, [{"id": i, "segments": [[0, 30 + i]], "output": 25} for i in range(3)],
             [2, 6, 15]),
            ("window", 5, 1.0, 13, [{"id": i, "segments": [[0, 13 + i]], "output": 33} for i in range(2)],
             [2, 4, 8])):
        s = ref.spec(SIM_MODELS[model])
        d = ref.spec(draft)
        sim = RefSim(s, 64 << 20, 32, False, reqs, draft=d, propose_k=k, acceptance=acc, seed=seed)
        ng = len(json.loads(SIM_MODELS[model])["groups"]) + 1
        snaps, step = [], 0
        for target in checkpoints:
            while step < target and not sim.done():
                sim.step()
                step += 1
            snaps.append(_snapshot(sim, reqs, ng, step))
        draws = {str(r["id"]): spec_accept_draws(ref, seed, r["id"], k, acc, 200) for r in reqs}
        out.append({"model": model, "spec": json.loads(SIM_MODELS[model]), "draft": json.loads(draft),
                    "propose_k": k, "acceptance": acc, "seed": seed, "budget": 64 << 20, "chunk": 32,
                    "requests": reqs, "draws": draws, "snapshots": snaps})
    return out


PREFIX_MODELS = {
    "window": spec_json("win", [
        {"name": "self", "kind": "full", "num_layers": 2, "bytes_per_token_per_layer": 64, "tokens_per_page": 4},
        {"name": "window", "kind": "sliding_window", "num_layers": 3, "bytes_per_token_per_layer": 64,
         "window_tokens": 24, "tokens_per_page": 4}]),
    "hybrid": spec_json("hyb", [
        {"name": "attn", "kind": "full", "num_layers": 2, "bytes_per_token_per_layer": 64, "tokens_per_page": 2},
        {"name": "ssm", "kind": "mamba", "num_layers": 3, "bytes_per_token_per_layer": 256,
         "checkpoint_interval_tokens": 16}]),
}


def sim_prefix(ref):
    """Reference SimEngine with prefix caching on its multi-article trace
    (trace.cpp:144-169): later rounds hit the cached article prefixes."""
    from oracle.oracle import multi_article_trace
    out = []
    for model, budget, chunk, params in (
            ("window", 8 << 20, 48, dict(articles=3, questions=3, article_tokens=90, question_tokens=9,
                                         output_tokens=6, spacing=12, seed=3)),
            ("window", 96 * 1024, 32, dict(articles=3, questions=4, article_tokens=60, question_tokens=7,
                                           output_tokens=5, spacing=9, seed=4)),
            ("hybrid", 8 << 20, 40, dict(articles=2, questions=3, article_tokens=64, question_tokens=8,
                                         output_tokens=5, spacing=10, seed=5))):
        reqs = multi_article_trace(ref, **params)
        s = ref.spec(PREFIX_MODELS[model])
        sim = RefSim(s, budget, chunk, True, reqs)
        ng = len(json.loads(PREFIX_MODELS[model])["groups"])
        snaps = []
        step = 0
        ref_error = None
        while not sim.done() and step < 400:
            try:
                sim.step()
            except Exception as e:  # the reference's Mamba prefix-hit leak
                ref_error = str(e)
                break
            step += 1
            snap = {"step": step, "requests": []}
            for r in reqs:
                rq = sim.request(r["id"])
                groups = []
                for g in range(ng):
                    st = sim.group_state(r["id"], g)
                    groups.append({"pages": st["pages"].tolist(), "live": st["live"].astype(int).tolist(),
                                   "stored": st["stored"], "freed": st["freed"],
                                   "working": None if st["working"] is None else [int(x) for x in st["working"]]})
                snap["requests"].append({"id": r["id"], "phase": rq["phase"], "consumed": rq["consumed"],
                                         "groups": groups})
            snaps.append(snap)
        kv = RefKv(s, budget, handle=sim.L.ref_sim_allocator(sim.h))
        final = [kv.counts(g) for g in range(ng)]
        out.append({"model": model, "spec": json.loads(PREFIX_MODELS[model]), "budget": budget, "chunk": chunk,
                    "requests": reqs, "snapshots": snaps, "final_counts": final, "done": sim.done(),
                    "reference_error": ref_error})
    return out


def main():
    ref = ref_lib()
    if ref is None:
        raise SystemExit("reference library unavailable: build oracle/_ref first (oracle/build_oracle.py)")
    for name, fn in (("fig6.json", fig6), ("configs.json", configs), ("random_geometries.json", random_geometries),
                     ("alloc_sequences.json", alloc_sequences), ("policies.json", policies),
                     ("sim_pages.json", sim_pages), ("sim_prefix.json", sim_prefix),
                     ("sim_vision.json", sim_vision), ("sim_spec.json", sim_spec)):
        data = fn(ref)
        with open(OUT / name, "w") as f:
            json.dump(data, f, separators=(",", ":"))
        print(name, (OUT / name).stat().st_size, "bytes")


if __name__ == "__main__":
    main()

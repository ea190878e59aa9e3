"""Prefix-hit adoption on the device (BASELINE config 5)
on the reference's own multi-article trace (trace.cpp:144-169), through the
product path:

* test_prefix_tables_match_reference_simengine — the reference SimEngine
  (oracle/_ref, stepped) and the native page-list runtime replaying its
  schedule in lockstep; after every step the native lists go to the device
  through the delta upload and every resident request's device block table,
  seq_len and newest slot must equal the C oracle's table build over the
  REFERENCE's page lists, bit for bit (hits splice pinned pages into rows).
* test_prefix_hits_attention_on_device — the same trace as a serving loop
  (admit -> lookup_and_pin -> adopt, kv_allocator.cpp:241-303,
  simulator.cpp:391-433; chunked prefill with the window frees deferred
  until the chunk's attention ran): K/V of every stored position written
  through slot_mapping + reshape_and_cache, each prefill chunk attended with
  paged_prefill and each decode step with paged_decode_append, every output
  against the C oracle through the same tables AND against dense attention
  over the K/V the request's own tokens define — so a hit that spliced a
  wrong or unwritten page would fail even where the oracle agrees.
* test_mamba_checkpoint_restore_on_device — Mamba checkpoint snapshots
  (working -> checkpoint page copies reported by the runtime) and the restore
  the reference leaks (simulator.cpp:409-414): restore_pending ->
  jenga_page_copy -> finish_restore, the working state byte-equal to the
  checkpoint, the checkpoint back in the cache.
"""
import json

import numpy as np
import pytest
import torch

from gpu_scenarios import rel_err
from oracle.oracle import BF16, FULL, SWA, RefSim, multi_article_trace
from paper_2503_18292_b200 import LayerKind, ops
from paper_2503_18292_b200.engine import DecodeEngine
from paper_2503_18292_b200.geometry import GroupGeometry, ModelGeometry
from test_prefix_caching import prompt_tokens
from test_page_lists import mix2

pytestmark = pytest.mark.gpu

HKV, HQ, D, TPP, W = 2, 4, 128, 16, 48
BPTL = 2 * HKV * D * 2
TOL = 1e-2
PAGES = 220


def geometry():
    return ModelGeometry("prefix-gpu", [
        GroupGeometry("full", LayerKind.kFullAttention, 2, HKV, HQ, D, torch.bfloat16, TPP),
        GroupGeometry("window", LayerKind.kSlidingWindow, 2, HKV, HQ, D, torch.bfloat16, TPP, window=W)])


SPEC_JSON = json.dumps({"name": "prefix-gpu", "groups": [
    {"name": "full", "kind": "full", "num_layers": 2, "bytes_per_token_per_layer": BPTL, "tokens_per_page": TPP},
    {"name": "window", "kind": "sliding_window", "num_layers": 2, "bytes_per_token_per_layer": BPTL,
     "tokens_per_page": TPP, "window_tokens": W}]})


def trace(ref):
    return multi_article_trace(ref, articles=3, questions=3, article_tokens=150, question_tokens=20,
                               output_tokens=4, spacing=12, seed=7)


class Replay:
    """SimEngine::step (simulator.cpp:642-677) over the engine's native page
    lists — decode in admission order, then chunked prefill, then admission
    with prefix lookup — recording what every request stored this step."""

    def __init__(self, eng, reqs, chunk, defer=False):
        """defer=False: the reference's own order (a finished request is
        released right after its last decode append, window blocks freed as
        positions are stored) — page lists identical to the reference's.
        defer=True: serving order — window frees deferred until the chunk's
        attention ran, releases after the step's device work."""
        self.eng, self.pl, self.chunk, self.defer = eng, eng.pages, chunk, defer
        self.reqs = []
        for r in sorted(reqs, key=lambda r: (r.get("arrival", 0), r["id"])):
            self.reqs.append({"id": r["id"], "arrival": r.get("arrival", 0), "phase": 0, "toks": prompt_tokens(r),
                              "generated": 0, "output": r["output"], "consumed": 0, "hit": 0})
        self.now = 0
        self.hits = 0

    def step(self):
        """Returns {request id: ("prefill"|"decode", first new ordinal, end ordinal)}."""
        new = {}
        for r in [x for x in self.reqs if x["phase"] == 2]:
            tok = mix2(mix2(r["id"], 0xDEC0DE), r["generated"])
            n = len(r["toks"]) + r["generated"]
            assert self.pl.append(r["id"], tok, False, 0, self.now)
            r["generated"] += 1
            new[r["id"]] = ("decode", n + 1, n + 2)
            if r["generated"] >= r["output"]:
                if self.defer:
                    r["phase"] = 4  # released after this step's device work
                else:
                    self.pl.release(r["id"], True, self.now)
                    r["phase"] = 3
        budget = self.chunk
        for r in self.reqs:
            if budget == 0:
                break
            if r["phase"] == 1:
                budget = self._prefill(r, budget, new)
        for r in self.reqs:
            if budget == 0:
                break
            if r["phase"] != 0 or r["arrival"] > self.now:
                continue
            if self.defer:
                self.pl.set_defer_window_free(r["id"], True)
            hit = self.pl.admit(r["id"], r["toks"], now=self.now)
            self.hits += hit
            r["hit"] = r["consumed"] = hit
            r["phase"] = 1
            if hit >= len(r["toks"]):
                r["phase"] = 2
            else:
                budget = self._prefill(r, budget, new)
        return new

    def _prefill(self, r, budget, new):
        c0 = r["consumed"]
        done, oom = self.pl.prefill(r["id"], budget, self.now)
        assert not oom
        r["consumed"] += done
        if done:
            new[r["id"]] = ("prefill", c0 + 1, r["consumed"] + 1)
        if r["consumed"] >= len(r["toks"]):
            r["phase"] = 2
        return budget - done

    def finish_step(self):
        """After the device work: deferred window frees, releases."""
        for r in self.reqs:
            if self.defer and r["phase"] in (1, 2):
                self.pl.apply_window_free(r["id"], self.now)
                if r["phase"] == 2:
                    self.pl.set_defer_window_free(r["id"], False)
            if r["phase"] == 4:
                self.pl.release(r["id"], True, self.now)
                r["phase"] = 3
        self.now += 1

    def tokens(self, r):
        return r["toks"] + [mix2(mix2(r["id"], 0xDEC0DE), g) for g in range(r["generated"])]


def make_engine(reqs):
    eng = DecodeEngine(geometry(), PAGES, len(reqs), 400, prefix_caching=True)
    eng.add_requests([r["id"] for r in sorted(reqs, key=lambda r: (r.get("arrival", 0), r["id"]))])
    return eng


def test_prefix_tables_match_reference_simengine(orc, ref):
    reqs = trace(ref)
    budget = PAGES * 2 * BPTL * TPP  # LCM = one small page (2 layers x 16 tokens x BPTL)
    sim = RefSim(ref.spec(SPEC_JSON), budget, 64, True, reqs)
    eng = make_engine(reqs)
    assert eng.kv.pool_info()[1] == PAGES
    rp = Replay(eng, reqs, 64)
    rows = {rid: i for i, rid in enumerate(eng.requests)}
    steps = hits_seen = 0
    while not sim.done():
        sim.step()
        rp.step()
        rp.finish_step()
        eng.sync_tables()
        torch.cuda.synchronize()
        steps += 1
        for g in range(2):
            t = eng.tables[g]
            table = t.block_table.cpu().numpy()
            seq = t.seq_lens.cpu().numpy()
            slots = t.slot_mapping.cpu().numpy()
            for r in rp.reqs:
                i = rows[r["id"]]
                if r["phase"] not in (1, 2):
                    assert (table[i] == -1).all() and seq[i] == 0
                    continue
                st = sim.group_state(r["id"], g)
                n = len(st["pages"])
                off = np.array([0, n], dtype=np.int32)
                want_t, want_s, want_q = orc.build_block_tables(
                    off, st["pages"], np.array([st["freed"]], np.int32), np.array([st["stored"]], np.int32),
                    eng.addr.slots_per_large(g), TPP, t.max_blocks)
                np.testing.assert_array_equal(table[i], want_t[0], err_msg=f"step {steps} req {r['id']} g {g}")
                assert seq[i] == want_q[0] and slots[i] == want_s[0]
                hits_seen += r["hit"] > 0
        assert steps < 400
    assert rp.hits > 0 and hits_seen > 0, "the trace must produce prefix hits"
    eng.kv.check_invariants()


# ----------------------------------------------------------------------------- numerics
def _splitmix(x):
    x = x + np.uint64(0x9E3779B97F4A7C15)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def rows_of(tokens, ordinals, salt, heads):
    """Deterministic bf16-exact rows [n, heads, D] of (token, ordinal, salt):
    identical prefixes give identical K/V, as a real model's would."""
    with np.errstate(over="ignore"):
        t = np.asarray(tokens, dtype=np.uint64)[:, None]
        o = np.asarray(ordinals, dtype=np.uint64)[:, None]
        idx = np.arange(heads * D, dtype=np.uint64)[None, :]
        x = _splitmix(t * np.uint64(0x100000001B3) ^ (o << np.uint64(20)) ^ (np.uint64(salt) << np.uint64(44)) ^ idx)
    v = ((x >> np.uint64(40)).astype(np.float64) / float(1 << 24) * 4.0 - 2.0).astype(np.float32)
    v = torch.from_numpy(v.reshape(-1, heads, D)).to(torch.bfloat16)
    return v


def kv_for(tokens, ordinals, g, layer):
    salt = 16 * g + 2 * layer
    return rows_of(tokens, ordinals, salt + 1, HKV), rows_of(tokens, ordinals, salt + 2, HKV)


def q_for(tokens, ordinals, g, layer):
    return rows_of(tokens, ordinals, 64 + 16 * g + layer, HQ)


def dense_attention(toks, q_ords, g, layer, q):
    """fp64 attention over the K/V the request's own tokens define: ordinal i
    attends (i - W, i] (SWA) or [1, i]."""
    n = int(max(q_ords))
    K, V = kv_for(toks[:n], np.arange(1, n + 1), g, layer)
    K, V, Q = K.double().numpy(), V.double().numpy(), q.double().numpy()
    out = np.zeros(Q.shape)
    for qi, i in enumerate(q_ords):
        lo = max(1, i - W + 1) if g == 1 else 1
        for h in range(HQ):
            kh = h // (HQ // HKV)
            s = K[lo - 1:i, kh] @ Q[qi, h] * D ** -0.5
            p = np.exp(s - s.max())
            out[qi, h] = (p / p.sum()) @ V[lo - 1:i, kh]
    return out


def test_prefix_hits_attention_on_device(orc, ref):
    reqs = trace(ref)
    eng = make_engine(reqs)
    eng.arena.tensor().fill_(0xFF)  # NaN poison: an unwritten page in a row would surface
    rp = Replay(eng, reqs, 64, defer=True)
    rows = {rid: i for i, rid in enumerate(eng.requests)}
    dev = eng.device
    checked = {"prefill": 0, "decode": 0, "hit_prefill": 0}
    worst = 0.0
    for _ in range(400):
        if all(r["phase"] == 3 for r in rp.reqs):
            break
        new = rp.step()
        eng.sync_tables()
        for rid, (kind, a, b) in sorted(new.items()):
            r = next(x for x in rp.reqs if x["id"] == rid)
            toks = rp.tokens(r)
            i = rows[rid]
            ords = np.arange(a, b)
            for g in range(2):
                t = eng.tables[g]
                for layer in range(2):
                    K, V = kv_for(toks[a - 1:b - 1], ords, g, layer)
                    q = q_for(toks[a - 1:b - 1], ords, g, layer)
                    out = torch.full((len(ords), HQ, D), float("nan"), dtype=torch.bfloat16, device=dev)
                    view = eng.view(g, layer)
                    if kind == "prefill":
                        req_d = torch.full((len(ords),), i, dtype=torch.int32, device=dev)
                        slots = torch.empty(len(ords), dtype=torch.int64, device=dev)
                        ops.slot_mapping(t.block_table, t.max_blocks, req_d,
                                         torch.from_numpy(ords.astype(np.int32)).to(dev), TPP, slots)
                        ops.reshape_and_cache(eng.arena, view, K.to(dev), V.to(dev), slots, TPP)
                        cu = torch.tensor([0, len(ords)], dtype=torch.int32, device=dev)
                        ops.paged_prefill(eng.arena, view, int(t.geom.kind), q.to(dev), out, cu, len(ords),
                                          t.block_table[i:i + 1], t.seq_lens[i:i + 1], HKV, TPP, D ** -0.5,
                                          window=t.geom.window)
                    else:
                        ops.paged_decode_append(eng.arena, view, int(t.geom.kind), q.to(dev), K.to(dev), V.to(dev),
                                                t.slot_mapping[i:i + 1], out, t.block_table[i:i + 1],
                                                t.seq_lens[i:i + 1], HKV, TPP, D ** -0.5, window=t.geom.window,
                                                workspace=t.workspace)
                    torch.cuda.synchronize()
                    got = out.float().cpu().numpy()
                    assert np.isfinite(got).all(), (rid, kind, g, layer)
                    arena = eng.arena.tensor().cpu().numpy()
                    table = t.block_table[i:i + 1].cpu().numpy()
                    seq = t.seq_lens[i:i + 1].cpu().numpy()
                    qh = q.view(torch.int16).numpy()
                    if kind == "prefill":
                        want = orc.paged_prefill(arena, tuple(view), int(t.geom.kind), BF16, t.geom.window, qh,
                                                 np.array([0, len(ords)], np.int32), table, seq, HQ, HKV, D, TPP,
                                                 D ** -0.5)
                    else:
                        want = orc.paged_decode(arena, tuple(view), int(t.geom.kind), BF16, t.geom.window, qh,
                                                table, seq, HQ, HKV, D, TPP, D ** -0.5, nthreads=4)
                    dense = dense_attention(toks, ords, g, layer, q)
                    e1, e2 = rel_err(got, want), rel_err(got, dense)
                    worst = max(worst, e1, e2)
                    assert e1 <= TOL and e2 <= TOL, (rid, kind, g, layer, e1, e2)
            checked[kind] += 1
            if kind == "prefill" and r["hit"] > 0 and a == r["hit"] + 1:
                checked["hit_prefill"] += 1
        rp.finish_step()
    assert all(r["phase"] == 3 for r in rp.reqs)
    assert checked["hit_prefill"] >= 3 and checked["decode"] >= 9, checked
    eng.kv.check_invariants()
    print(f"[prefix] {checked}, hits {rp.hits} tokens, worst relative error {worst:.3g}")


# ----------------------------------------------------------------------------- Mamba restore
def _state_bytes(tokens, nbytes):
    """Stand-in SSM state after `tokens` (the SSM math is out of scope): bytes
    determined by the prefix, so a restored state can be checked exactly."""
    seed = 0
    for t in tokens:
        seed = mix2(seed, t)
    return torch.from_numpy(np.random.default_rng(seed).integers(0, 256, nbytes, dtype=np.uint8))


def test_mamba_checkpoint_restore_on_device():
    geom = ModelGeometry("hyb-gpu", [
        GroupGeometry("attn", LayerKind.kFullAttention, 1, HKV, HQ, D, torch.bfloat16, TPP),
        GroupGeometry("ssm", LayerKind.kMamba, 3, state_bytes=4096, checkpoint_interval=16)])
    eng = DecodeEngine(geom, 64, 2, 128, prefix_caching=True)
    eng.add_requests([1, 2])
    at = eng.arena.tensor()
    at.fill_(0xFF)
    small = eng.addr.small_page_bytes(1)
    g_of = lambda p: eng.addr.global_page_index(1, p)  # noqa: E731
    page_bytes = lambda p: at[g_of(p) * small:(g_of(p) + 1) * small]  # noqa: E731
    toks = [mix2(5, i) for i in range(40)]
    pl = eng.pages
    pl.admit(1, toks)
    assert pl.prefill(1, 100) == (40, False)
    copies = pl.take_checkpoint_copies()
    assert [c["ordinal"] for c in copies] == [16, 32]
    wp1 = pl.group_state(1, 1)["working_page"]
    for c in copies:  # the scan's state at each checkpoint ordinal -> snapshot
        assert c["working"] == wp1
        page_bytes(wp1).copy_(_state_bytes(toks[:c["ordinal"]], small))
        ops.page_copy(eng.arena, small, torch.tensor([g_of(c["working"])], device="cuda"),
                      torch.tensor([g_of(c["checkpoint"])], device="cuda"))
    page_bytes(wp1).copy_(_state_bytes(toks, small))
    torch.cuda.synchronize()
    ck32 = copies[1]["checkpoint"]
    pl.release(1, True)
    # request 2 shares 35 tokens: the hit stops at the 32-token checkpoint
    toks2 = toks[:35] + [7, 7, 7]
    hit = pl.admit(2, toks2)
    assert hit == 32
    ck = pl.restore_pending(2, 1)
    assert ck == ck32 and eng.kv.record(1, ck)["state"] == 2  # pinned
    assert pl.prefill(2, 100) == (6, False)
    wp2 = pl.group_state(2, 1)["working_page"]
    assert wp2 not in (ck, wp1)
    ops.page_copy(eng.arena, small, torch.tensor([g_of(ck)], device="cuda"), torch.tensor([g_of(wp2)], device="cuda"))
    torch.cuda.synchronize()
    want = _state_bytes(toks[:32], small)
    assert torch.equal(page_bytes(wp2).cpu(), want) and torch.equal(page_bytes(ck).cpu(), want)
    pl.finish_restore(2, 1)
    assert pl.restore_pending(2, 1) is None and eng.kv.record(1, ck)["state"] == 1  # back in the cache
    # the attention group adopted the 32-token prefix too: its table row points at request 1's pages
    eng.sync_tables()
    torch.cuda.synchronize()
    row = eng.tables[0].block_table[1].cpu().numpy()
    assert (row[:2] >= 0).all() and eng.tables[0].seq_lens[1].item() == 38
    pl.release(2, True)
    eng.kv.check_invariants()

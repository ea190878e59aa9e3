"""Prefix-hit adoption: the native
admit / lookup_and_pin / adopt path against the reference SimEngine on the
reference's own multi-article trace (trace.cpp:144-169), step by step — every
request's blocks, live flags, stored ordinals and the allocator's final
counts must match, including under memory pressure (LRU evictions)."""
import json

import numpy as np
import pytest

from conftest import load_golden
from paper_2503_18292_b200 import KvAllocator, LayerGroupSpec, LayerKind, ModelSpec, PageLists
from test_page_lists import mix2, mix64

MASK = (1 << 64) - 1


def fnv1a(s):
    h = 0xCBF29CE484222325
    for c in s.encode():
        h ^= c
        h = (h * 0x100000001B3) & MASK
    return h


def prompt_tokens(r):
    """derived_token (simulator.cpp:120-129) incl. shared prefix groups."""
    segs = r["segments"]
    toks = []
    for s, (_, n) in enumerate(segs):
        shared = r.get("prefix_group", -1) >= 0 and (len(segs) == 1 or s + 1 < len(segs))
        base = mix2(fnv1a(f"article-{r['prefix_group']}"), s) if shared else mix2(mix2(r["id"], 0x9E11), s)
        toks += [mix2(base, o) for o in range(n)]
    return toks


class CachingReplay:
    """SimEngine::step with prefix caching (simulator.cpp:642-677, 435-566),
    driving the native PageLists admit/prefill/append/release."""

    def __init__(self, case):
        self.spec = ModelSpec.from_json(json.dumps(case["spec"]))
        self.kv = KvAllocator(self.spec, case["budget"])
        self.pl = PageLists(self.kv, prefix_caching=True)
        self.pl.set_fix_mamba_restore(False)  # reference behaviour for parity
        self.chunk = case["chunk"]
        self.reqs = []
        for r in sorted(case["requests"], key=lambda r: (r.get("arrival", 0), r["id"])):
            self.reqs.append({"id": r["id"], "arrival": r.get("arrival", 0), "phase": 0, "toks": prompt_tokens(r),
                              "generated": 0, "output": r["output"], "consumed": 0})
        self.now = 0
        self.hits = 0

    def step(self):
        for r in [x for x in self.reqs if x["phase"] == 2]:
            tok = mix2(mix2(r["id"], 0xDEC0DE), r["generated"])
            assert self.pl.append(r["id"], tok, False, 0, self.now)
            r["generated"] += 1
            if r["generated"] >= r["output"]:
                self.pl.release(r["id"], True, self.now)
                r["phase"] = 3
        budget = self.chunk
        for r in self.reqs:
            if budget == 0:
                break
            if r["phase"] == 1:
                budget = self._prefill(r, budget)
        for r in self.reqs:
            if budget == 0:
                break
            if r["phase"] != 0 or r["arrival"] > self.now:
                continue
            self.pl.add_request(r["id"])
            hit = self.pl.admit(r["id"], r["toks"], now=self.now)
            self.hits += hit
            r["consumed"] = hit
            r["phase"] = 1
            if hit >= len(r["toks"]):
                r["phase"] = 2
            else:
                budget = self._prefill(r, budget)
        self.now += 1

    def _prefill(self, r, budget):
        done, oom = self.pl.prefill(r["id"], budget, self.now)
        assert not oom
        r["consumed"] += done
        if r["consumed"] >= len(r["toks"]):
            r["phase"] = 2
        return budget - done


@pytest.mark.parametrize("ci", [0, 1])
def test_prefix_caching_matches_reference_simulator(ci):
    case = load_golden("sim_prefix.json")[ci]
    assert case["reference_error"] is None and case["done"]
    rp = CachingReplay(case)
    for snap in case["snapshots"]:
        rp.step()
        assert rp.now == snap["step"]
        for want in snap["requests"]:
            r = [x for x in rp.reqs if x["id"] == want["id"]][0]
            assert r["phase"] == want["phase"], (ci, snap["step"], want["id"])
            if want["phase"] in (0, 3):
                continue
            assert r["consumed"] == want["consumed"]
            for g, wg in enumerate(want["groups"]):
                st = rp.pl.group_state(want["id"], g)
                blocks = rp.pl.blocks(want["id"], g)
                assert st["stored"] == wg["stored"], (ci, snap["step"], want["id"], g)
                assert st["freed_blocks"] == wg["freed"]
                assert [list(p) for p, lv in blocks if lv] == [p for p, lv in zip(wg["pages"], wg["live"]) if lv]
                assert [int(lv) for _, lv in blocks] == wg["live"]
    rp.kv.check_invariants()
    assert rp.hits > 0, "the trace must produce prefix hits"
    for g, want in enumerate(case["final_counts"]):
        c = rp.kv.group_counts(g)
        assert (c["used"], c["evictable"], c["empty"], c["owned_units"]) == (
            want["used"], want["evictable"], want["empty"], want["owned_units"])
        assert rp.kv.pool_free_pages() == want["pool_free"]


def test_reference_mamba_hit_leak_is_fixed():
    """The reference pins a Mamba checkpoint on a prefix hit and never adopts
    it, which breaks its own byte-conservation check (sim_prefix.json hybrid
    case).  The native runtime hands the pinned page back as a
    restore source and returns it to the cache once copied."""
    case = load_golden("sim_prefix.json")[2]
    assert case["reference_error"] and "conservation" in case["reference_error"]
    spec = ModelSpec("hyb", [LayerGroupSpec("attn", LayerKind.kFullAttention, 2, 64, tokens_per_page=2),
                             LayerGroupSpec("ssm", LayerKind.kMamba, 3, 256, checkpoint_interval_tokens=16)])
    kv = KvAllocator(spec, 1 << 22)
    pl = PageLists(kv, prefix_caching=True)
    toks = [mix64(i) for i in range(40)]
    pl.add_request(1)
    pl.admit(1, toks)
    assert pl.prefill(1, 100) == (40, False)
    pl.release(1, True)
    assert kv.cache_entries(1) == 2  # checkpoints at 16 and 32 cached
    pl.add_request(2)
    hit = pl.admit(2, toks[:35] + [7, 7, 7])
    assert hit == 32  # longest prefix valid in every group: the 32-token checkpoint
    ck = pl.restore_pending(2, 1)
    assert ck is not None and kv.record(1, ck)["state"] == 2  # pinned (Used)
    assert pl.prefill(2, 100) == (6, False)
    wp = pl.group_state(2, 1)["working_page"]
    assert wp is not None and wp != ck
    # device would page_copy(ck -> wp) here; then:
    pl.finish_restore(2, 1)
    assert pl.restore_pending(2, 1) is None
    assert kv.record(1, ck)["state"] == 1  # back in the cache, evictable
    kv.check_invariants()
    pl.release(2, True)
    kv.check_invariants()
    assert kv.group_counts(1)["used"] == 0 and kv.group_counts(0)["used"] == 0


def test_prefix_hit_splices_cached_pages():
    """A second request with the same prompt reuses the first one's pages
    (pinned, not copied) for every full block of the prefix."""
    spec = ModelSpec("w", [LayerGroupSpec("self", LayerKind.kFullAttention, 2, 64, tokens_per_page=4),
                           LayerGroupSpec("win", LayerKind.kSlidingWindow, 2, 64, tokens_per_page=4,
                                          window_tokens=8)])
    kv = KvAllocator(spec, 1 << 20)
    pl = PageLists(kv, prefix_caching=True)
    toks = [mix64(100 + i) for i in range(30)]
    pl.add_request(1)
    pl.admit(1, toks)
    pl.prefill(1, 64)
    first = [p for p, _ in pl.blocks(1, 0)]
    pl.release(1, True)
    pl.add_request(2)
    hit = pl.admit(2, toks + [5])
    assert hit == 28  # 7 full blocks of 4 tokens
    got = pl.blocks(2, 0)
    assert [p for p, lv in got if lv] == first[:7]
    win = pl.blocks(2, 1)
    assert sum(lv for _, lv in win) == 2 and all(not lv for _, lv in win[:5])  # only the window's blocks pinned
    kv.check_invariants()


def test_mamba_checkpoint_copies_are_queued_and_dropped_when_evicted():
    """Every checkpoint page store_position allocates (simulator.cpp:231-242)
    is reported once as a working -> checkpoint copy for the device; a page
    evicted from the cache before the copy was taken is not reported."""
    spec = ModelSpec("hyb", [LayerGroupSpec("attn", LayerKind.kFullAttention, 2, 64, tokens_per_page=2),
                             LayerGroupSpec("ssm", LayerKind.kMamba, 3, 256, checkpoint_interval_tokens=16)])
    kv = KvAllocator(spec, 1 << 22)
    pl = PageLists(kv, prefix_caching=True)
    toks = [mix64(i) for i in range(40)]
    pl.add_request(1)
    pl.admit(1, toks)
    assert pl.prefill(1, 100) == (40, False)
    copies = pl.take_checkpoint_copies()
    wp = pl.group_state(1, 1)["working_page"]
    assert [c["ordinal"] for c in copies] == [16, 32]
    assert all(c["group"] == 1 and c["request"] == 1 and c["working"] == wp for c in copies)
    assert len({c["checkpoint"] for c in copies}) == 2 and wp not in {c["checkpoint"] for c in copies}
    for c in copies:
        assert kv.record(1, c["checkpoint"])["state"] == 1  # cached (evictable)
    assert pl.take_checkpoint_copies() == []  # drained
    # decode 16 more tokens -> one more checkpoint, then evict everything evictable
    for i in range(16):
        assert pl.append(1, mix64(1000 + i))
    while kv.evict_lru_large_page() is not None:
        pass
    assert pl.take_checkpoint_copies() == []  # its page left the cache: nothing to copy into
    kv.check_invariants()


def test_prefix_cache_table_against_a_model():
    """The prefix cache's open-addressing table (chain key -> cached pages in
    registration order, reference prefix_cache.cpp:59-100) against a plain
    dict model under churn: thousands of registrations (through free with
    content), pins (unregister), evictions, colliding keys with different
    contents, tombstones and rehashes; every lookup and entry count agrees."""
    from paper_2503_18292_b200 import BlockContent
    spec = ModelSpec("c", [LayerGroupSpec("full", LayerKind.kFullAttention, 1, 64, tokens_per_page=2)])
    kv = KvAllocator(spec, 3000 * 128)
    rng = np.random.default_rng(11)
    model = {}      # key -> list of (content tuple, page) in registration order
    cached = []     # (content, page) currently registered
    used = []       # pages held by "requests"
    contents = [BlockContent(int(rng.integers(0, 40)), int(rng.integers(0, 3)), [int(x) for x in rng.integers(0, 4, 2)])
                for _ in range(300)]  # few keys: many collisions and duplicate contents

    def ckey(c):
        return (c.key, c.parent_key, tuple(c.tokens))

    def is_cached(pg):
        try:
            return kv.record(0, pg)["state"] == 1
        except Exception:  # its large page went back to the pool
            return False

    def model_find(c):
        for cc, page in model.get(c.key, []):
            if cc == ckey(c):
                return page
        return None

    def unreg(page):
        for k in list(model):
            model[k] = [(cc, p) for cc, p in model[k] if p != page]
            if not model[k]:
                del model[k]

    for step in range(6000):
        op = rng.random()
        if op < 0.45:
            res = kv.allocate(0, int(rng.integers(0, 8)))
            if res is None:
                kv.evict_lru_large_page()
            else:
                used.append(res.page)
            # allocation may evict cached pages itself (five-step allocate, kv_allocator.cpp:154-197)
            for c, pg in [(c, pg) for c, pg in cached if not is_cached(pg)]:
                unreg(pg)
            cached = [(c, pg) for c, pg in cached if is_cached(pg)]
        elif op < 0.8 and used:
            page = used.pop(int(rng.integers(0, len(used))))
            c = contents[int(rng.integers(0, len(contents)))]
            kv.free(0, page, c)
            model.setdefault(c.key, []).append((ckey(c), page))
            cached.append((c, page))
        elif op < 0.9 and cached:
            c, page = cached.pop(int(rng.integers(0, len(cached))))
            kv.pin(0, page, 99)
            unreg(page)
            used.append(page)
        elif cached:
            kv.evict_lru_large_page()
            for c, pg in [(c, pg) for c, pg in cached if not is_cached(pg)]:
                unreg(pg)
            cached = [(c, pg) for c, pg in cached if is_cached(pg)]
        if step % 50 == 0:
            for c in contents[:60]:
                want = model_find(c)
                got = kv.cache_find(0, c)
                assert (None if got is None else tuple(got)) == (None if want is None else tuple(want)), step
            assert kv.cache_entries(0) == sum(len(v) for v in model.values())
    kv.check_invariants()

"""Per-request page lists (the producer of every block table) against the
reference SimEngine itself: the golden snapshots in sim_pages.json were read
out of the reference simulator's GroupRuntime state (simulator.hpp:123-139).
The replay below issues the same store_position sequence the reference
scheduler issues (decode in admission order, then chunked prefill, then
admission — simulator.cpp:642-672, 504-547, 435-482) into the native
PageLists and compares every block, live flag and working page."""
import json

import numpy as np
import pytest

from conftest import load_golden
from paper_2503_18292_b200 import KvAllocator, LayerKind, ModelSpec, PageLists

MASK = (1 << 64) - 1


def mix64(x):
    x = (x + 0x9E3779B97F4A7C15) & MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK
    return x ^ (x >> 31)


def mix2(a, b):
    return mix64(a ^ mix64(b))


class Replay:
    """Minimal SimEngine schedule (no preemption, no prefix hits)."""

    def __init__(self, case):
        self.spec = ModelSpec.from_json(json.dumps(case["spec"]))
        self.kv = KvAllocator(self.spec, case["budget"])
        self.pl = PageLists(self.kv, case["prefix_caching"])
        self.chunk = case["chunk"]
        self.reqs = []
        for r in sorted(case["requests"], key=lambda r: (r.get("arrival", 0), r["id"])):
            toks, img = [], []
            for s, (is_image, n) in enumerate(r["segments"]):
                base = mix2(mix2(r["id"], 0x9E11), s)
                for o in range(n):
                    toks.append(mix2(base, o))
                    img.append(bool(is_image))
            self.reqs.append({"id": r["id"], "phase": 0, "toks": toks, "img": img, "consumed": 0,
                              "generated": 0, "output": r.get("output", 1)})
        self.now = 0

    def step(self):
        for r in self.reqs:
            if r["phase"] != 2:
                continue
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
                budget = self.prefill(r, budget)
        for r in self.reqs:
            if budget == 0:
                break
            if r["phase"] == 0:
                self.pl.add_request(r["id"])
                r["phase"] = 1
                budget = self.prefill(r, budget)
        self.now += 1

    def prefill(self, r, budget):
        while budget > 0 and r["consumed"] < len(r["toks"]):
            i = r["consumed"]
            assert self.pl.append(r["id"], r["toks"][i], r["img"][i], 0, self.now)
            r["consumed"] += 1
            budget -= 1
        if r["consumed"] >= len(r["toks"]):
            r["phase"] = 2
        return budget


@pytest.mark.parametrize("ci", range(4))
def test_page_lists_match_reference_simulator(ci):
    case = load_golden("sim_pages.json")[ci]
    rp = Replay(case)
    step = 0
    for snap in case["snapshots"]:
        while step < snap["step"]:
            rp.step()
            step += 1
        for want in snap["requests"]:
            r = [x for x in rp.reqs if x["id"] == want["id"]][0]
            assert r["phase"] == want["phase"], (ci, snap["step"], want["id"])
            if want["phase"] in (0, 3):
                continue
            assert [str(t) for t in (r["toks"][: r["consumed"]] +
                                     [mix2(mix2(r["id"], 0xDEC0DE), k) for k in range(r["generated"])])] == \
                want["tokens"][: r["consumed"] + r["generated"]]
            for g, wg in enumerate(want["groups"]):
                st = rp.pl.group_state(want["id"], g)
                blocks = rp.pl.blocks(want["id"], g)
                assert st["stored"] == wg["stored"], (ci, snap["step"], want["id"], g)
                assert st["freed_blocks"] == wg["freed"]
                assert [list(p) for p, _ in blocks] == wg["pages"]
                assert [int(lv) for _, lv in blocks] == wg["live"]
                if wg["working"] is None:
                    assert st["working_page"] is None
                else:
                    assert list(st["working_page"]) == wg["working"]
    rp.kv.check_invariants()


def test_swa_holds_at_most_window_pages():
    """reference test_simulator.cpp:202-218: window group never beyond W."""
    spec = ModelSpec.from_json(json.dumps({"name": "w", "groups": [
        {"name": "self", "kind": "full", "num_layers": 2, "bytes_per_token_per_layer": 64, "tokens_per_page": 4},
        {"name": "win", "kind": "sliding_window", "num_layers": 3, "bytes_per_token_per_layer": 64,
         "window_tokens": 10, "tokens_per_page": 4}]}))
    kv = KvAllocator(spec, 1 << 22)
    pl = PageLists(kv)
    for r in range(3):
        pl.add_request(r)
    for pos in range(1, 200):
        assert pl.append_batch([2, 0, 1], now=pos) == 3
        for r in range(3):
            st = pl.group_state(r, 1)
            live = [lv for _, lv in pl.blocks(r, 1)]
            assert sum(live) <= (10 + 4 - 1) // 4 + 1
            # live blocks are exactly those holding an ordinal of (n-W, n]
            n = st["stored"]
            for b, lv in enumerate(live):
                assert lv == ((b + 1) * 4 > n - 10), (pos, r, b)
            assert st["freed_blocks"] == sum(1 for lv in live if not lv)
    kv.check_invariants()
    for r in range(3):
        pl.release(r)
    kv.check_invariants()
    assert kv.group_counts(0)["used"] == 0 and kv.group_counts(1)["used"] == 0


def test_pack_csr_layout():
    spec = ModelSpec.from_json(json.dumps({"name": "w", "groups": [
        {"name": "self", "kind": "full", "num_layers": 1, "bytes_per_token_per_layer": 64, "tokens_per_page": 2},
        {"name": "ssm", "kind": "mamba", "num_layers": 2, "bytes_per_token_per_layer": 256,
         "checkpoint_interval_tokens": 4}]}))
    kv = KvAllocator(spec, 1 << 20)
    pl = PageLists(kv)
    for r in (5, 6):
        pl.add_request(r)
    for _ in range(5):
        pl.append_batch([5, 6])
    pl.append_batch([6])
    off, pages, live0, nst = pl.pack_csr(0, [6, 5])
    assert off.tolist() == [0, 3, 6] and nst.tolist() == [6, 5] and live0.tolist() == [0, 0]
    assert [tuple(p) for p in pages[:3]] == [tuple(p) for p, _ in pl.blocks(6, 0)]
    off, pages, live0, nst = pl.pack_csr(1, [5, 6])
    assert off.tolist() == [0, 1, 2] and nst.tolist() == [5, 6]
    assert tuple(pages[0]) == tuple(pl.group_state(5, 1)["working_page"])


def test_oom_requires_release():
    spec = ModelSpec.from_json(json.dumps({"name": "t", "groups": [
        {"name": "self", "kind": "full", "num_layers": 1, "bytes_per_token_per_layer": 64, "tokens_per_page": 1}]}))
    kv = KvAllocator(spec, 64 * 3)
    pl = PageLists(kv)
    pl.add_request(1)
    assert pl.append(1) and pl.append(1) and pl.append(1)
    assert not pl.append(1)
    from paper_2503_18292_b200 import InvariantError
    with pytest.raises(InvariantError):
        pl.append(1)
    pl.release(1)
    kv.check_invariants()
    assert kv.group_counts(0)["used"] == 0


def test_interleaved_workload_matches_reference_allocator(ref):
    """The bench workload's page lists: product PageLists vs the restated
    store_position driven over the reference KvAllocator (oracle/_ref)."""
    from oracle.oracle import RefPageLists
    js = json.dumps({"name": "g", "groups": [
        {"name": "full", "kind": "full", "num_layers": 3, "bytes_per_token_per_layer": 512, "tokens_per_page": 4},
        {"name": "win", "kind": "sliding_window", "num_layers": 3, "bytes_per_token_per_layer": 512,
         "window_tokens": 24, "tokens_per_page": 4},
        {"name": "ssm", "kind": "mamba", "num_layers": 5, "bytes_per_token_per_layer": 1536}]})
    budget = 400 * 7680
    kv = KvAllocator(ModelSpec.from_json(js), budget)
    pl = PageLists(kv)
    rs = ref.spec(js)
    rkv = rs.kv(budget)
    rpl = RefPageLists(rkv)
    rng = np.random.default_rng(0)
    ids = list(range(10, 17))
    for r in ids:
        pl.add_request(r)
    for pos in range(1, 121):
        order = rng.permutation(ids) if (pos - 1) % 4 == 0 else order
        assert pl.append_batch(order, now=pos) == len(ids)
        assert rpl.append_batch(order, now=pos)
    for r in ids:
        for g in range(3):
            pages, live, stored, freed = rpl.group_state(r, g)
            if g == 2:
                assert pl.group_state(r, g)["stored"] == stored
                continue
            blocks = pl.blocks(r, g)
            assert [tuple(p) for p, _ in blocks] == [tuple(x) for x in pages]
            assert [lv for _, lv in blocks] == live.tolist()
    kv.check_invariants()
    rkv.check_invariants()


def test_deferred_window_free_then_apply():
    """After the chunk's attention the deferred SWA frees leave exactly the
    pages decode keeps (reference finish_prefill, simulator.cpp:484-500)."""
    from paper_2503_18292_b200 import LayerGroupSpec
    spec = ModelSpec("w", [LayerGroupSpec("win", LayerKind.kSlidingWindow, 1, 64, tokens_per_page=4,
                                          window_tokens=10)])
    a = KvAllocator(spec, 1 << 20)
    pa = PageLists(a)
    b = KvAllocator(spec, 1 << 20)
    pb = PageLists(b)
    for pl in (pa, pb):
        pl.add_request(1)
    pa.set_defer_window_free(1, True)
    for _ in range(37):
        pa.append(1)
        pb.append(1)
    assert sum(lv for _, lv in pa.blocks(1, 0)) == 10 and pa.group_state(1, 0)["freed_blocks"] == 0
    pa.apply_window_free(1)
    pa.set_defer_window_free(1, False)
    assert [lv for _, lv in pa.blocks(1, 0)] == [lv for _, lv in pb.blocks(1, 0)]
    a.check_invariants()

"""SURVEY §8(f) rows 3-4 on the host: vision-embedding pages (both vision
modes) and speculative decoding (draft groups in the same LCM pool, rollback
of rejected proposals) against the reference SimEngine itself.  The golden
snapshots in sim_vision.json / sim_spec.json were read out of the reference
simulator (make_golden.py); the replay below issues the reference schedule
(decode in admission order, chunked prefill, admission — simulator.cpp:
642-672) through the native PageLists and compares every block, live flag,
stored count and working page."""
import json

import pytest

from conftest import load_golden
from paper_2503_18292_b200 import KvAllocator, ModelSpec, PageLists

MASK = (1 << 64) - 1


def mix64(x):
    x = (x + 0x9E3779B97F4A7C15) & MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK
    return x ^ (x >> 31)


def mix2(a, b):
    return mix64(a ^ mix64(b))


class Schedule:
    """SimEngine::step restated over the native PageLists (no preemption)."""

    def __init__(self, spec, budget, chunk, requests, vision_mode=0, spec_cfg=None, seed=0):
        self.kv = KvAllocator(spec, budget)
        self.pl = PageLists(self.kv)
        self.pl.set_vision_mode(vision_mode)
        self.chunk = chunk
        self.spec_cfg = spec_cfg
        self.reqs = []
        for r in sorted(requests, key=lambda r: (r.get("arrival", 0), r["id"])):
            toks, img, ordn = [], [], []
            for s, (is_image, n) in enumerate(r["segments"]):
                base = mix2(mix2(r["id"], 0x9E11), s)
                # simulator.cpp:130-137, 160-162: one content id per image segment
                ordinal = mix2(seed, mix2(mix2(mix2(base, 0), 0x1D347), 0x0E0E)) if is_image else 0
                for o in range(n):
                    toks.append(mix2(base, o))
                    img.append(bool(is_image))
                    ordn.append(ordinal)
            self.reqs.append({"id": r["id"], "phase": 0, "toks": toks, "img": img, "ord": ordn, "consumed": 0,
                              "generated": 0, "output": r.get("output", 1), "arrival": r.get("arrival", 0),
                              "draw": 0})
            self.pl.add_request(r["id"])
        self.now = 0

    def decode(self, r):
        tok = lambda g: mix2(mix2(r["id"], 0xDEC0DE), g)  # noqa: E731
        if self.spec_cfg is None:
            assert self.pl.append(r["id"], tok(r["generated"]), False, 0, self.now)
            r["generated"] += 1
        else:
            k, draws = self.spec_cfg
            acc = draws[str(r["id"])][r["draw"]]
            r["draw"] += 1
            n_target = min(max(acc, 1), r["output"] - r["generated"])
            toks = [tok(r["generated"] + j) for j in range(n_target)]
            assert self.pl.speculative_decode(r["id"], k, acc, toks, n_target, self.now)
            r["generated"] += n_target
        if r["generated"] >= r["output"]:
            self.pl.release(r["id"], False, self.now)
            r["phase"] = 3

    def prefill(self, r, budget):
        n, oom = self.pl.prefill(r["id"], budget, self.now)
        assert not oom
        r["consumed"] += n
        if r["consumed"] >= len(r["toks"]):
            r["phase"] = 2
        return budget - n

    def step(self):
        for r in self.reqs:
            if r["phase"] == 2:
                self.decode(r)
        budget = self.chunk
        for r in self.reqs:
            if budget == 0:
                break
            if r["phase"] == 1:
                budget = self.prefill(r, budget)
        for r in self.reqs:
            if budget == 0:
                break
            if r["phase"] != 0 or r["arrival"] > self.now:
                continue
            r["consumed"] = self.pl.admit(r["id"], r["toks"], r["img"], r["ord"], now=self.now)
            r["phase"] = 1
            if r["consumed"] >= len(r["toks"]):
                r["phase"] = 2
            else:
                budget = self.prefill(r, budget)
        self.now += 1


def check_snapshots(case, sch, ng):
    step = 0
    for snap in case["snapshots"]:
        while step < snap["step"]:
            sch.step()
            step += 1
        for want in snap["requests"]:
            r = [x for x in sch.reqs if x["id"] == want["id"]][0]
            assert r["phase"] == want["phase"], (snap["step"], want["id"])
            if want["phase"] in (0, 3):
                continue
            for g in range(ng):
                wg = want["groups"][g]
                st = sch.pl.group_state(want["id"], g)
                blocks = sch.pl.blocks(want["id"], g)
                ctx = (snap["step"], want["id"], g)
                assert st["stored"] == wg["stored"], ctx
                assert st["freed_blocks"] == wg["freed"], ctx
                assert [list(p) for p, _ in blocks] == wg["pages"], ctx
                assert [int(lv) for _, lv in blocks] == wg["live"], ctx
                if wg["working"] is None:
                    assert st["working_page"] is None, ctx
                else:
                    assert list(st["working_page"]) == wg["working"], ctx
    sch.kv.check_invariants()


@pytest.mark.parametrize("ci", range(4))
def test_vision_pages_match_reference_simulator(ci):
    case = load_golden("sim_vision.json")[ci]
    spec = ModelSpec.from_json(json.dumps(case["spec"]))
    sch = Schedule(spec, case["budget"], case["chunk"], case["requests"], vision_mode=case["vision_mode"])
    check_snapshots(case, sch, len(case["spec"]["groups"]))


def test_vision_on_demand_frees_consumed_embeddings():
    """at most one prefill chunk of embeddings is held
    once an image is being consumed; all of them are gone after the prompt."""
    case = load_golden("sim_vision.json")[0]
    spec = ModelSpec.from_json(json.dumps(case["spec"]))
    vg = [i for i, g in enumerate(case["spec"]["groups"]) if g["kind"] == "vision_embedding"][0]
    sch = Schedule(spec, case["budget"], case["chunk"], case["requests"], vision_mode=0)
    seen_held = False
    for _ in range(40):
        sch.step()
        for r in sch.reqs:
            if r["phase"] == 2:
                assert sch.pl.group_state(r["id"], vg)["held_tokens"] == 0
            if r["phase"] == 1 and sch.pl.group_state(r["id"], vg)["held_tokens"]:
                seen_held = True
    assert seen_held


@pytest.mark.parametrize("ci", range(3))
def test_speculative_pages_match_reference_simulator(ci):
    case = load_golden("sim_spec.json")[ci]
    target = ModelSpec.from_json(json.dumps(case["spec"]))
    draft = ModelSpec.from_json(json.dumps(case["draft"]))
    spec = target.combine_with_draft(draft)
    assert [g.name for g in spec.groups][-len(draft.groups):] == ["draft." + g.name for g in draft.groups]
    sch = Schedule(spec, case["budget"], case["chunk"], case["requests"],
                   spec_cfg=(case["propose_k"], case["draws"]))
    ng = len(spec.groups)
    assert [sch.pl.is_draft_group(g) for g in range(ng)] == [False] * (ng - 1) + [True]
    check_snapshots(case, sch, ng)


def test_rollback_newest_frees_emptied_pages():
    """reference rollback_newest (simulator.cpp:568-597)."""
    spec = ModelSpec.from_json(json.dumps({"name": "t", "groups": [
        {"name": "self", "kind": "full", "num_layers": 1, "bytes_per_token_per_layer": 64, "tokens_per_page": 4}]}))
    kv = KvAllocator(spec, 1 << 20)
    pl = PageLists(kv)
    pl.add_request(7)
    for _ in range(10):
        assert pl.append(7)
    assert pl.group_state(7, 0)["num_blocks"] == 3
    used = kv.group_counts(0)["used"]
    pl.rollback_newest(7, 0, 2)  # 10 -> 8: block 2 empties
    st = pl.group_state(7, 0)
    assert st["stored"] == 8 and st["num_blocks"] == 2 and st["held_tokens"] == 8
    assert kv.group_counts(0)["used"] == used - 1
    pl.rollback_newest(7, 0, 1)  # 8 -> 7: block 1 keeps 3 tokens
    assert pl.group_state(7, 0)["num_blocks"] == 2
    pl.rollback_newest(7, 0, 100)
    assert pl.group_state(7, 0)["stored"] == 0 and pl.group_state(7, 0)["num_blocks"] == 0
    kv.check_invariants()
    assert kv.group_counts(0)["used"] == 0

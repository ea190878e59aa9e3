"""The drop-in boundary, exercised the way a reference maintainer would wire
it: integration/jenga_gpu_bridge.hpp
compiled against the UNMODIFIED reference headers and objects
(oracle/build_oracle.py -> oracle/_ref/libjenga_bridge_test.so, harness
tests/bridge/bridge_harness.cpp).  The reference KvAllocator (Jenga strategy,
kv_allocator.hpp:62-119) produces the page lists; the bridge builds the
device block tables from them and runs one fused decode-append launch per
group with the reference's own LayerView (memory_layout.hpp:25-32).  Checked
here against the C oracle: tables / seq_lens / newest slots bit-exact, the
new token's K/V bytes in their slots, attention within the bf16 tolerance —
and the native allocator, fed the same order, must produce the very same
page lists (the port is not on this path; this pins it to the reference on
the GPU workload)."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from gpu_scenarios import rel_err
from oracle.oracle import BF16

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "oracle" / "_ref" / "libjenga_bridge_test.so"
HKV, HQ, D, TPP, W = 8, 16, 256, 16, 300
BPTL = 2 * HKV * D * 2
SPEC = {"name": "bridge-gemma", "groups": [
    {"name": "full", "kind": "full", "num_layers": 2, "bytes_per_token_per_layer": BPTL, "tokens_per_page": TPP},
    {"name": "window", "kind": "sliding_window", "num_layers": 2, "bytes_per_token_per_layer": BPTL,
     "tokens_per_page": TPP, "window_tokens": W}]}
LENS = [1, 16, 17, 299, 300, 301, 777, 1025, 64]


def _lib():
    if not LIB.exists():
        pytest.skip("bridge harness not built (needs /root/reference at build time)")
    lib = C.CDLL(str(LIB))
    lib.bridge_run.restype = C.c_int
    return lib


def test_integration_doc_quotes_the_compiled_bridge():
    """INTEGRATION.md §1 shows the bridge verbatim (what the harness compiles)."""
    doc = (ROOT / "INTEGRATION.md").read_text()
    hdr = (ROOT / "integration" / "jenga_gpu_bridge.hpp").read_text()
    assert "```cpp\n" + hdr + "```" in doc


@pytest.mark.gpu
def test_reference_allocator_through_bridge_on_device(orc):
    lib = _lib()
    from paper_2503_18292_b200 import AddressMap, KvAllocator, ModelSpec, PageLists
    spec = ModelSpec.from_json(json.dumps(SPEC))
    addr = AddressMap(spec)
    lcm = addr.large_page_bytes()
    pages = sum((n + TPP - 1) // TPP + 2 for n in LENS) * 2 + 16
    budget = pages * lcm
    n = len(LENS)
    max_blocks = max(LENS) // TPP + 2
    cap = pages * 2
    rng = np.random.default_rng(0)
    arena0 = rng.integers(0, 1 << 16, size=pages * lcm // 2, dtype=np.uint16)
    arena0 &= 0xBFFF  # finite bf16
    arena0 = arena0.view(np.uint8)
    bf = lambda *s: torch.randn(s).to(torch.bfloat16).view(torch.int16).numpy()  # noqa: E731
    torch.manual_seed(3)
    q, k, v = bf(2, n, HQ, D), bf(2, n, HKV, D), bf(2, n, HKV, D)
    out = np.zeros((2, n, HQ, D), np.int16)
    pg = np.zeros((2, cap, 2), np.int32)
    off = np.zeros((2, n + 1), np.int32)
    live0 = np.zeros((2, n), np.int32)
    stored = np.zeros((2, n), np.int32)
    table = np.zeros((2, n, max_blocks), np.int32)
    seq = np.zeros((2, n), np.int32)
    slots = np.zeros((2, n), np.int64)
    arena1 = np.zeros_like(arena0)
    err = C.create_string_buffer(512)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    # interleaved store order: a seeded permutation of the live requests per 16 positions
    order_rng = np.random.default_rng(7)
    sequence, cur, pos = [], [0] * n, 0
    while any(c < m for c, m in zip(cur, LENS)):
        if pos % 16 == 0:
            perm = list(order_rng.permutation(n))
        step = [r for r in perm if cur[r] < LENS[r]]
        for r in step:
            cur[r] += 1
        sequence.append(step)
        pos += 1
    flat = np.array([r for step in sequence for r in step], np.int32)
    layer = 1
    rc = lib.bridge_run(json.dumps(SPEC).encode(), C.c_uint64(budget), n, p(flat), C.c_int64(flat.size), max_blocks,
                        cap,
                        p(pg), p(off), p(live0), p(stored), p(table), p(seq), p(slots), p(arena0),
                        C.c_uint64(arena0.nbytes), layer, p(q), p(k), p(v), p(out), p(arena1), HQ, HKV, D,
                        C.c_float(0.0), err, 512)
    assert rc == 0, err.value.decode()

    native_kv = KvAllocator(spec, budget)
    native = PageLists(native_kv)
    for r in range(n):
        native.add_request(r)
    for step in sequence:
        assert native.append_batch(step) == len(step)
    for g in range(2):
        # reference page lists -> device tables: bit-exact with the oracle's build
        t_want, s_want, q_want = orc.build_block_tables(off[g], pg[g, : off[g, -1]].astype(np.uint32), live0[g],
                                                        stored[g], addr.slots_per_large(g), TPP, max_blocks)
        np.testing.assert_array_equal(table[g], t_want)
        np.testing.assert_array_equal(slots[g], s_want)
        np.testing.assert_array_equal(seq[g], q_want)
        assert (seq[g] == np.array(LENS)).all()
        # the new token's K/V rows landed in their slots (head-major slice)
        view = addr.layer_view(g, layer)
        for b in range(n):
            page, o = divmod(int(slots[g, b]), TPP)
            base = view.start_offset + page * view.page_stride
            for h in (0, HKV - 1):
                for kv_i, src in ((0, k), (1, v)):
                    row = base + ((2 * h + kv_i) * TPP + o) * D * 2
                    assert (arena1[row:row + D * 2] == src[g, b, h].view(np.uint8)).all()
        # attention through the reference's LayerView, against the oracle
        want = orc.paged_decode(arena1, tuple(view), [0, 1][g], BF16, [0, W][g], q[g], table[g], seq[g], HQ, HKV,
                                D, TPP, D ** -0.5, 0.0, nthreads=8)
        got = (out[g].astype(np.uint16).astype(np.uint32) << 16).view(np.float32)
        assert rel_err(got, want) <= 1e-2
        # the same store order through the native port: the very same page lists
        n_off, n_pages, n_live, n_st = native.pack_csr(g, list(range(n)), max_blocks)
        np.testing.assert_array_equal(n_off, off[g])
        np.testing.assert_array_equal(n_pages.astype(np.int32), pg[g, : off[g, -1]])
        np.testing.assert_array_equal(n_live, live0[g])
        np.testing.assert_array_equal(n_st, stored[g])

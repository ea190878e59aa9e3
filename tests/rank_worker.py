"""One rank of the N>1 path on CPU (gloo), started by the same launcher entry
bench.py uses (paper_2503_18292_b200.distributed.launch_local_ranks ->
torch.distributed.run on 127.0.0.1).  Each rank owns a shard of the requests,
its own native Jenga allocator and page lists (no shared state, reference
SPEC.md:535), builds its block tables and computes its shard's decode with the
C oracle standing in for the device kernels (no GPU here); the verification
all-gather (gather_padded, as bench.py) brings every shard to rank 0, which
writes them to argv[1] (.npz) for the test to check.

    python -m torch.distributed.run --nproc-per-node 2 tests/rank_worker.py out.npz
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2503_18292_b200 import AddressMap, KvAllocator, PageLists  # noqa: E402
from paper_2503_18292_b200.distributed import gather_padded, max_over_ranks, shard_requests  # noqa: E402
from paper_2503_18292_b200.geometry import toy  # noqa: E402

GLOBAL = list(range(200, 208))
LENS = {r: 40 + 13 * (r % 5) for r in GLOBAL}
MAX_BLOCKS = 80


def run_shard(ids, seed):
    """One rank's work: allocator + page lists + block tables + oracle decode."""
    from oracle import c_oracle
    from oracle.oracle import F32, FULL, SWA
    orc = c_oracle()
    geom = toy(4)
    geom.groups[1].window = 24
    spec = geom.spec()
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
        off, pages, live0, nst = pl.pack_csr(g, ids, MAX_BLOCKS)
        table, _, seq = orc.build_block_tables(off, pages, live0, nst, addr.slots_per_large(g), 4, MAX_BLOCKS)
        tables.append(table)
        outs.append(orc.paged_decode(arena, tuple(addr.layer_view(g, 0)), kind, F32, geom.groups[g].window,
                                     q[qi], table, seq, 16, 8, 128, 4, 128 ** -0.5))
    return np.stack(tables), np.stack(outs)


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    try:
        ids = shard_requests(GLOBAL, rank, world)
        tables, outs = run_shard(ids, seed=rank)
        payload = torch.from_numpy(np.concatenate([tables.reshape(-1).view(np.uint8), outs.reshape(-1).view(np.uint8)]))
        rows = gather_padded(payload).numpy()
        mx = max_over_ranks(float(rank + 1), "cpu")
        if rank == 0:
            np.savez(sys.argv[1], rows=rows, world=world, max_rank=mx, env_world=int(os.environ["WORLD_SIZE"]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

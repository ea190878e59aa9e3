"""N>1 path on CPU with gloo, world_size 2, through the launcher entry
bench.py --gpus N uses (launch_local_ranks -> torch.distributed.run on
127.0.0.1, one process per rank): requests shard across ranks, each rank owns
an independent native Jenga allocator and page lists (no shared state,
reference SPEC.md:535), computes its shard (the C oracle stands in for the
device kernels here, tests/rank_worker.py), and the verification all-gather
(gather_padded) collects the results on rank 0.  The gathered shards must
equal single-process runs of the same shards."""
import os
import sys
from pathlib import Path

import numpy as np

from paper_2503_18292_b200.distributed import launch_local_ranks, shard_requests

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
import rank_worker  # noqa: E402


def test_shard_requests_partition():
    for n in (1, 7, 8, 33):
        for world in (1, 2, 3, 8):
            ids = list(range(n))
            parts = [shard_requests(ids, r, world) for r in range(world)]
            assert sum(parts, []) == ids
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_two_rank_gloo_launcher_shards_and_verification_gather(tmp_path):
    out = tmp_path / "gathered.npz"
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="", OMP_NUM_THREADS="2")
    rc = launch_local_ranks(str(HERE / "rank_worker.py"), [str(out)], 2, env=env)
    assert rc == 0
    z = np.load(out)
    assert int(z["world"]) == 2 and int(z["env_world"]) == 2 and float(z["max_rank"]) == 2.0
    rows = z["rows"]
    assert rows.shape[0] == 2
    for rank in range(2):
        t, o = rank_worker.run_shard(shard_requests(rank_worker.GLOBAL, rank, 2), seed=rank)
        want = np.concatenate([t.reshape(-1).view(np.uint8), o.reshape(-1).view(np.uint8)])
        np.testing.assert_array_equal(rows[rank, : want.size], want)
        assert not rows[rank, want.size:].any()  # padding
        # each shard's pool is private: both ranks hand out pages from large page 0 onward
        assert t[0, 0, 0] >= 0
        assert np.isfinite(o).all()

"""Row-level check of one chunked-prefill configuration against the C oracle (prints
the (token, head) rows off by more than 5% of max|want|): the tool that found the
P-placement race of the split-accumulator variant."""
import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from gpu_scenarios import ORC_DTYPE, TOL, arena_host, fill_group_kv, make_engine, rel_err
from paper_2503_18292_b200 import LayerKind, ops
from paper_2503_18292_b200.geometry import GroupGeometry, ModelGeometry
from oracle import c_oracle
orc = c_oracle()
for hq, kind, W in ((64, LayerKind.kSlidingWindow, 100), (32, LayerKind.kSlidingWindow, 100), (64, LayerKind.kFullAttention, 0)):
    hd, hkv = 128, 8
    geom = ModelGeometry("p", [GroupGeometry("g", kind, 2, hkv, hq, hd, torch.bfloat16, 16, window=W)])
    lens = [300, 77, 513, 16, 1]; chunks = [300, 13, 200, 16, 1]
    eng, ids = make_engine(geom, lens, seed=hd, defer_window=True)
    fill_group_kv(eng, 0, [1], seed=2, all_live=True)
    g, layer = 0, 1
    t = eng.tables[g]; gg = t.geom; B = len(eng.requests)
    cu = np.zeros(B + 1, dtype=np.int32); cu[1:] = np.cumsum(chunks); T = int(cu[-1])
    gen = torch.Generator(device=eng.device).manual_seed(5)
    q = torch.randn((T, gg.num_q_heads, gg.head_dim), generator=gen, device=eng.device).to(gg.dtype)
    out = torch.full_like(q, float("nan"))
    ops.paged_prefill(eng.arena, eng.view(g, layer), int(gg.kind), q, out, torch.from_numpy(cu).to(eng.device), int(max(chunks)),
                      t.block_table[:B], t.seq_lens[:B], gg.num_kv_heads, eng.spec.groups[g].tokens_per_page, hd ** -0.5, window=W, softcap=0.0)
    torch.cuda.synchronize()
    want = orc.paged_prefill(arena_host(eng), tuple(eng.view(g, layer)), int(gg.kind), ORC_DTYPE[gg.dtype], W,
                             q.view(torch.int16).cpu().numpy(), cu, t.block_table[:B].cpu().numpy(), t.seq_lens[:B].cpu().numpy(),
                             gg.num_q_heads, gg.num_kv_heads, gg.head_dim, eng.spec.groups[g].tokens_per_page, hd ** -0.5, 0.0)
    got = out.float().cpu().numpy().reshape(want.shape)
    err = np.abs(got - want).max(axis=-1)  # [T, H]
    print("hq", hq, "kind", int(kind), "rel", rel_err(got, want))
    bad = np.argwhere(err > 0.05 * np.abs(want).max())
    print(" bad count", len(bad), "tokens", sorted(set(bad[:, 0].tolist()))[:40])
    if len(bad): print(" heads", sorted(set(bad[:, 1].tolist()))[:20])
    print(" cu", cu.tolist())

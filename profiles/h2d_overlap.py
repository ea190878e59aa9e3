"""Does a host->device copy overlap an HBM-saturating kernel?  Times a pinned H2D
copy alone, a device-to-device copy alone (HBM-bound, ~6.5 TB/s), and both on two
streams started together (CUDA events on each stream)."""
import json
import torch

dev = torch.device("cuda")
for mb in (22, 176):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    a = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
    b = torch.empty_like(a)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn_list):
        ev = []
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        start.record()
        for st, fn in fn_list:
            st.wait_event(start)
            with torch.cuda.stream(st):
                fn()
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                ev.append(e)
        torch.cuda.synchronize()
        return [round(start.elapsed_time(e), 3) for e in ev]

    for _ in range(3):
        timed([(s1, lambda: d.copy_(h, non_blocking=True))])
        timed([(s2, lambda: b.copy_(a))])
    r = {"h2d_mb": mb, "h2d_alone_ms": timed([(s1, lambda: d.copy_(h, non_blocking=True))])[0],
         "d2d_alone_ms": timed([(s2, lambda: b.copy_(a))])[0]}
    both = timed([(s2, lambda: b.copy_(a)), (s1, lambda: d.copy_(h, non_blocking=True))])
    r["together_d2d_ms"], r["together_h2d_ms"] = both
    print(json.dumps(r), flush=True)

# the same two copies captured as parallel branches of one CUDA graph
for mb in (22, 176):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    a = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
    b = torch.empty_like(a)
    main = torch.cuda.Stream()
    side = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(main):
        with torch.cuda.graph(g, stream=main):
            side.wait_stream(main)
            with torch.cuda.stream(side):
                d.copy_(h, non_blocking=True)
            b.copy_(a)
            main.wait_stream(side)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(main):
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"graph_h2d_mb": mb, "graph_both_ms": round(e0.elapsed_time(e1) / 10, 3)}), flush=True)

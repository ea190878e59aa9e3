"""Pipeline timeline of the 128-key prefill kernel (profiling variant built with
JENGA_PF_TRACE): clock64 stamps of the first CTA pair's leader for each key tile.
    JENGA_B200_LIB=paper_2503_18292_b200/variants/libjenga_b200_trace.so \
        python profiles/prefill_trace.py [d128|d256]"""
import ctypes
import sys

import numpy as np

sys.path.insert(0, "profiles")
import bench_prefill  # noqa: E402
from paper_2503_18292_b200._lib import lib  # noqa: E402

heads = (32, 8, 128) if "d256" not in sys.argv else (16, 8, 256)
shape = (64, 2048, 256) if "short" in sys.argv else (4, 8192, 2048)
bench_prefill.run(*shape, iters=1, heads=heads)
buf = np.zeros((16, 64), dtype=np.int64)
assert lib.jenga_debug_prefill_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
names = ["mma:pA_full", "mma:pB_full", "mma:sA_issued", "mma:sB_issued",
         "smA:s_full", "smA:ld", "smA:exp", "smA:arrive", "", "",
         "smB:s_full", "smB:ld", "smB:exp", "smB:arrive"]
t0 = buf[buf > 0].min()
print("tile " + " ".join(f"{n:>13}" for n in names if n))
for j in range(2, 40):
    print(f"{j:4d} " + " ".join(f"{(buf[i, j] - t0) if buf[i, j] else 0:13d}" for i, n in enumerate(names) if n))
print("per unit (softmax warp 0): p_empty(last) wait done / exchange done / output done; MMA q_full:")
for k in range(8):
    if buf[8, k]:
        print(f"  unit {k}: {buf[8, k] - t0} / {buf[9, k] - t0} / {buf[1, k] - t0}; q_full {buf[3, k] - t0}")
print("chunk stores issued+read (thread 0, unit 0..1):", [int(buf[12, k] - t0) if buf[12, k] else 0 for k in range(8)])
print("entry -> first s_full:", buf[4, 0] - buf[15, 0], " last s_full -> epilogue done:",
      buf[14, 0] - buf[4][buf[4] > 0].max(), " entry -> done:", buf[14, 0] - buf[15, 0])
per = np.diff(buf[4, 10:40]).mean()
print("cycles per tile (group A s_full period):", per)
for a, b, lab in ((4, 5, "A ld"), (5, 6, "A exp+st"), (6, 7, "A tail"), (10, 11, "B ld"), (11, 12, "B exp+st"),
                  (12, 13, "B tail")):
    print(lab, np.mean(buf[b, 10:40] - buf[a, 10:40]))

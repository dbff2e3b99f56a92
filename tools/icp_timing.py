"""Per-phase ICP timing from the csf_debug_icp_clock hook (debug tool)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2405_02187_b200 as csf  # noqa: E402
from paper_2405_02187_b200 import capi  # noqa: E402

ctx = csf.Context(0)
n = 6
depth, gt, k = csf.synth_workload(2, n, ctx=ctx)
import bench  # noqa: E402

cfg = bench.pipeline_cfg(csf, capi, k, list(range(10)), n)
p = csf.Pipeline(cfg, ctx=ctx)
p.upload(depth, gt)
p.run()
ctx.synchronize()
lib = csf.library()
lib.csf_debug_icp_clock.argtypes = [C.c_void_p, C.c_int]
lib.csf_debug_icp_clock(None, 1)
p.run()
ctx.synchronize()
buf = np.zeros(4096 * 512 * 8, dtype=np.uint64)
lib.csf_debug_icp_clock(buf.ctypes.data, 0)
b = buf.reshape(4096, 512, 8).astype(np.float64)
for L in range(4096):
    cta = b[L]
    used = cta[:, 0] > 0
    if not used.any():
        break
    t0 = cta[used, 0].min()
    p1 = np.median(cta[used, 1] - cta[used, 0]) / 1e3
    p2 = np.median(cta[used, 2] - cta[used, 1]) / 1e3
    end_reduce = cta[used, 2].max() - t0
    solve = cta[:, 4].max() - cta[:, 3][cta[:, 3] > 0].min() if (cta[:, 3] > 0).any() else 0
    last = int(np.argmax(cta[:, 3]))
    sub = ""
    if cta[last, 5] > 0:
        sub = (f" [sums {(cta[last, 5] - cta[last, 3]) / 1e3:5.1f} ldlt {(cta[last, 6] - cta[last, 5]) / 1e3:5.1f} "
               f"exp+compose {(cta[last, 7] - cta[last, 6]) / 1e3:5.1f} tail {(cta[last, 4] - cta[last, 7]) / 1e3:5.1f}]")
    print(f"launch {L:3d} ctas {used.sum():4d} phase1 {p1:6.1f} us phase2 {p2:6.1f} us "
          f"last-tile-done {end_reduce / 1e3:7.1f} us solve {solve / 1e3:6.1f} us" + sub)

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
tot_red, tot_gap, tot_solve, nl = 0.0, 0.0, 0.0, 0
for L in range(4096):
    cta = b[L, :511]
    sv = b[L, 511]
    used = cta[:, 0] > 0
    if not used.any():
        break
    t0 = cta[used, 0].min()
    p1 = np.median(cta[used, 1] - cta[used, 0]) / 1e3
    p2 = np.median(cta[used, 2] - cta[used, 1]) / 1e3
    end_reduce = cta[used, 2].max() - t0
    line = (f"launch {L:3d} ctas {used.sum():4d} phase1 {p1:6.1f} us phase2 {p2:6.1f} us "
            f"last-tile-done {end_reduce / 1e3:7.1f} us")
    if sv[3] > 0:
        gap = sv[3] - cta[used, 2].max()
        end = sv[4] if sv[4] > 0 else sv[5]
        line += (f" | gap {gap / 1e3:5.1f} solve {(end - sv[3]) / 1e3:5.1f} [sums {(sv[5] - sv[3]) / 1e3:4.1f}"
                 f" ldlt-real {(sv[6] - sv[5]) / 1e3:4.1f} channels {(sv[7] - sv[6]) / 1e3:4.1f}"
                 f" exp+compose {(sv[4] - sv[7]) / 1e3:4.1f}]")
        tot_red += end_reduce
        tot_gap += gap
        tot_solve += end - sv[3]
        nl += 1
    print(line)
if nl:
    print(f"mean over {nl} launches: reduce {tot_red / nl / 1e3:.1f} us, gap {tot_gap / nl / 1e3:.1f} us, "
          f"solve {tot_solve / nl / 1e3:.1f} us")

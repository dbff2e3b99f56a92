"""Per-phase timeline of the ICP level kernel (csf_debug_icp_clock debug hook).

phases: 0 iteration start, 1 association done, 2 tile partial written,
3 totals published (last CTA only), 4 barrier passed, 5 solve done."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2405_02187_b200 as csf  # noqa: E402
from paper_2405_02187_b200 import capi  # noqa: E402

ctx = csf.Context(0)
n = 4
depth, gt, k = csf.synth_workload(2, n, ctx=ctx)
cfg = bench.pipeline_cfg(csf, capi, k, bench.DIRS, n)
p = csf.Pipeline(cfg, ctx=ctx)
p.upload(depth, gt)
p.run()
ctx.synchronize()
lib = csf.library()
lib.csf_debug_icp_clock.argtypes = [C.c_void_p, C.c_int]
lib.csf_debug_icp_clock(None, 1)
p.run()
ctx.synchronize()
buf = np.zeros(64 * 256 * 32 * 16, dtype=np.uint64)
lib.csf_debug_icp_clock(buf.ctypes.data, 0)
b = buf.reshape(64, 256, 32, 16).astype(np.float64)
for L in range(64):
    used = b[L, :, 0, 0] > 0
    if not used.any():
        break
    ctas = used.sum()
    its = int((b[L, 0, :, 0] > 0).sum())
    rows = []
    for it in range(its):
        t0 = b[L, used, it, 0]
        s = t0.min()
        a = b[L, used, it, 1] - t0
        pw = b[L, used, it, 2] - t0
        rel = b[L, used, it, 3]
        rel = rel[rel > 0]
        bar = b[L, used, it, 4]
        sol = b[L, used, it, 5]
        rows.append(f"  it {it}: start spread {(t0.max() - s) / 1e3:5.1f} us, assoc {np.median(a) / 1e3:5.1f}, "
                    f"partial {np.median(pw) / 1e3:5.1f} (max {(b[L, used, it, 2].max() - s) / 1e3:5.1f}), "
                    f"release {((rel.max() - s) / 1e3) if rel.size else -1:5.1f}, barrier-out "
                    f"{(bar.max() - s) / 1e3:5.1f}, solve {np.median(sol - bar) / 1e3:5.1f} us [ldlt "
                    f"{np.median(b[L, used, it, 8] - bar) / 1e3:4.1f} channels {np.median(b[L, used, it, 9] - b[L, used, it, 8]) / 1e3:4.1f}"
                    f" exp {np.median(b[L, used, it, 10] - b[L, used, it, 9]) / 1e3:4.1f} tail {np.median(sol - b[L, used, it, 10]) / 1e3:4.1f}]"
                    f" (chan-warp {np.median(b[L, used, it, 14] - b[L, used, it, 13]) / 1e3:4.1f} (max {(b[L, used, it, 14] - b[L, used, it, 13]).max() / 1e3:4.1f})"
                    f" assoc-end {np.median(b[L, used, it, 15] - b[L, used, it, 8]) / 1e3:4.1f} (max {(b[L, used, it, 15] - b[L, used, it, 8]).max() / 1e3:4.1f})"
                    f" totals+ldlt {np.median(b[L, used, it, 13] - bar) / 1e3:4.1f} apply {np.median(b[L, used, it, 11] - b[L, used, it, 13]) / 1e3:4.1f} expmap {np.median(b[L, used, it, 12] - b[L, used, it, 11]) / 1e3:4.1f})")
        rc = np.argmax(b[L, :, it, 3])
        rows.append(f"      releasing CTA {rc}: partial {(b[L, rc, it, 2] - s) / 1e3:5.1f} group-sum-done "
                    f"{(b[L, rc, it, 6] - s) / 1e3:5.1f} last-decided {(b[L, rc, it, 7] - s) / 1e3:5.1f} release "
                    f"{(b[L, rc, it, 3] - s) / 1e3:5.1f}; group sums done at "
                    f"{np.sort((b[L, used, it, 6][b[L, used, it, 6] > 0] - s) / 1e3).round(1).tolist()}")
    print(f"launch {L} ctas {ctas} iterations {its}")
    print("\n".join(rows))

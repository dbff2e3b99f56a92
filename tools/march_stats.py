"""Table-march statistics (debug hook csf_debug_march_stats) over one config-2 run."""
import ctypes as C
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi
import bench
ctx = csf.Context(0)
n = 20
depth, gt, k = csf.synth_workload(2, n, ctx=ctx)
p = csf.Pipeline(bench.pipeline_cfg(csf, capi, k, list(range(10)), n), ctx=ctx)
p.upload(depth, gt)
p.run()
ctx.synchronize()
lib = csf.library()
lib.csf_debug_march_stats.argtypes = [C.c_void_p, C.c_int]
lib.csf_debug_march_stats(None, 1)
p.run()
ctx.synchronize()
buf = np.zeros(8, dtype=np.uint64)
lib.csf_debug_march_stats(buf.ctypes.data, 0)
rays = buf[0]
names = ["rays", "trips", "super skips", "block skips", "samples", "valid samples", "hits", "warp-max trips"]
for i, nm in enumerate(names):
    print(f"{nm:15s} {int(buf[i]):14d}  per ray {buf[i] / rays:8.2f}")
print("warp efficiency (mean trips / warp-max trips):", (buf[1] / rays) / (buf[7] / (rays / 32)))

"""Debug: run N VGA frames of the surfel workload (for an ncu launch list)."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2405_02187_b200 as csf
from bench_surfel import lifted_poses, D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ctx = csf.Context(0)
depth, gt, k = csf.synth_workload(2, n, ctx=ctx)
poses = lifted_poses(gt)
m = csf.SurfelMap(D, ctx=ctx)
import time
for f in range(n):
    d = np.zeros(depth[f].shape + (1 + D,))
    d[..., 0] = depth[f]
    t = time.perf_counter()
    st = csf.update_surfels(m, d, poses[f], k, f)
    print(f, m.size(), st, f"{(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)

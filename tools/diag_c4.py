"""Config-4 tracking diagnostic: per-frame translation error of the real track."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi
import bench
ctx = csf.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 120
d, gt, k = csf.synth_workload(4, n, ctx=ctx)
cfg = bench.pipeline_cfg4(csf, capi, k, [0], n)
p = csf.Pipeline(cfg, ctx=ctx)
p.upload(d, gt)
p.run()
r = p.result()
err = np.linalg.norm(r.poses[:, 9:, 0] - gt[:, 9:], axis=1)
for f in range(0, n, 5):
    print(f, f"err {err[f]:.4f}", "it", r.stats[f, 0], "corr", r.stats[f, 1], "vis", r.stats[f, 4])
print("objective", r.objective, "grad", r.gradient)

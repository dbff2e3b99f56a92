"""A short config-2 run (VGA, 10 directions) for ncu captures of the ICP level kernel."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2405_02187_b200 as csf  # noqa: E402
from paper_2405_02187_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
ctx = csf.Context(0)
depth, gt, k = csf.synth_workload(2, n, ctx=ctx)
cfg = bench.pipeline_cfg(csf, capi, k, bench.DIRS, n)
p = csf.Pipeline(cfg, ctx=ctx)
p.upload(depth, gt)
for _ in range(2):
    p.run()
ctx.synchronize()
r = p.result()
print("stats", r.stats[:, :3].tolist())

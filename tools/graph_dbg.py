import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi
from oracle import orc
ctx = csf.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
d, gt, k = orc.workload(2, n, 320, 240)
hp = capi.HashParams(0.01, (C.c_double * 3)(0.0, 0.0, 0.0), 0.05, 128.0, 20, 1 << 16)
cfg = csf.make_pipeline_cfg(hashed=True, k=k, dirs=list(range(10)), h=1e-8, objective=capi.OBJECTIVE_TRAJECTORY_ERROR, max_frames=n, hash_params=hp)
p = csf.Pipeline(cfg, ctx=ctx)
p.upload(d, gt)
p.run(); ref = p.result()
print("ref stats", ref.stats[:, :7].tolist(), flush=True)
p.set_graph(True)
for r in range(3):
    p.run(); x = p.result()
    print("graph", r, "obj", x.objective, ref.objective, "stats", x.stats[:, :7].tolist(), flush=True)
    diff = np.abs(x.poses[..., 0] - ref.poses[..., 0]).reshape(n, -1).max(1)
    print("   pose diff per frame", diff.tolist(), flush=True)
p.set_graph(False)
p.run(); x = p.result(); print("stream again", x.objective == ref.objective, flush=True)
p.close()
print("closed", flush=True)

"""Run one small pipeline case in this process (for fault isolation)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi
from oracle import orc

hashed = int(sys.argv[1]); D = int(sys.argv[2])
ctx = csf.Context(0)
d, gt, k = orc.workload(2 if hashed else 1, 4, 160, 120)
dirs = list(range(D))
if hashed:
    hp = capi.HashParams(0.02, (capi.C.c_double * 3)(0.0, 0.0, 0.0), 0.1, 128.0, 20, 1 << 16)
    cfg = csf.make_pipeline_cfg(hashed=True, k=k, dirs=dirs, h=1e-8, objective=1, max_frames=4, hash_params=hp)
else:
    dense = capi.VolumeParams((capi.C.c_int * 3)(64, 64, 64), 0.06, (capi.C.c_double * 3)(-2.1, -1.28, -0.1), 0.18, 128.0)
    cfg = csf.make_pipeline_cfg(hashed=False, k=k, dirs=dirs, h=1e-8, objective=1, max_frames=4, dense=dense)
p = csf.Pipeline(cfg, ctx=ctx)
p.upload(d, gt)
p.run()
r = p.result()
print("OK", hashed, D, r.objective)

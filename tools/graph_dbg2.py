import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi
from oracle import orc
ctx = csf.Context(0)
n = 2
W, H = 320, 240
d, gt, k = orc.workload(2, n, W, H)
hp = capi.HashParams(0.01, (C.c_double * 3)(0.0, 0.0, 0.0), 0.05, 128.0, 20, 1 << 16)
cfg = csf.make_pipeline_cfg(hashed=True, k=k, dirs=list(range(10)), h=1e-8, objective=capi.OBJECTIVE_TRAJECTORY_ERROR, max_frames=n, hash_params=hp)
p = csf.Pipeline(cfg, ctx=ctx)
p.upload(d, gt)
lib = ctx.lib
lib.csf_debug_pipeline_buffer.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]
P = W * H
sizes = {0: 3 * P, 1: 3 * P, 2: 30 * P, 3: 30 * P, 4: P, 5: P, 6: P // 4, 7: P // 16, 8: 2 * P * 2, 9: 12 * 11, 10: n * 12 * 11, 11: 2 * 512 * 6000, 12: 10 * 512 * 6000}
names = {0: "vre", 1: "nre", 2: "vim", 3: "nim", 4: "raw", 5: "pyr0", 6: "pyr1", 7: "pyr2", 8: "hits", 9: "pose", 10: "traj", 11: "rw", 12: "fim"}
def grab():
    out = {}
    for w, cnt in sizes.items():
        a = np.zeros(cnt)
        lib.csf_debug_pipeline_buffer(p.h, w, a.ctypes.data, a.nbytes)
        out[w] = a
    return out
p.run(); ref = p.result(); A = grab()
p.set_graph(True)
for r in range(2):
    p.run(); x = p.result(); B = grab()
    print("replay", r, "stats", x.stats[:, :7].tolist(), "ref", ref.stats[:, :7].tolist())
    for w in sizes:
        dif = np.argwhere(A[w] != B[w])
        print("  ", names[w], "differs at", dif.size, "entries", dif[:3].ravel().tolist())

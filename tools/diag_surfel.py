"""Debug: device vs oracle surfel fusion, per field and channel differences."""
import sys
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2405_02187_b200 as csf
from oracle import orc
from test_surfel import _frames, _cfg

D = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctx = csf.Context(0)
depth, poses, gt, k = _frames(3, D=max(D, 1))
if D == 0:
    depth = depth[..., :1]
    poses = [p[:, :1] for p in poses]
cfg = _cfg()
mo, mg = orc.Surfels(D), csf.SurfelMap(D, ctx=ctx)
for f in range(2):
    co, io, wo = mo.associate(depth[f], poses[f], k, cfg)
    cg, ig, wg = csf.associate_all(mg, depth[f], poses[f], k, cfg)
    print("assoc", f, np.array_equal(cg, co), np.array_equal(ig, io), np.array_equal(wg, wo), len(io))
    if len(io) and not np.array_equal(wg, wo):
        d = np.abs(wg - wo)
        print("  weight diff per channel", d.max(axis=0), np.count_nonzero(d, axis=0))
    print(mo.update(depth[f], poses[f], k, f, cfg), csf.update_surfels(mg, depth[f], poses[f], k, f, cfg))
    a, b = mg.download(), mo.download()
    for key in a:
        if not np.array_equal(a[key], b[key]):
            d = np.abs(a[key] - b[key]).reshape(len(a[key]), -1)
            bad = np.nonzero(d.max(axis=1))[0]
            print(" ", key, "rows differing", len(bad), "max", d.max(), "first", bad[:5])
            if a[key].ndim == 3:
                print("   per channel max", np.abs(a[key] - b[key]).max(axis=(0, 1)))
                i = bad[0]
                print("   dev", a[key][i], "\n   orc", b[key][i])

"""Expected strong scaling of config 2 / config 3 under H8 (every rank
recomputes the shared real channel): time one rank's share — the first
ceil(10/N) directions (or ceil(55/N) pairs) — on one GPU for N = 1, 2, 4, 8
and report T(1)/T(N).  The gather (C2) is one 8*(D+1)-byte exchange per run
and is not modelled."""
import json
import math
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2405_02187_b200 as csf  # noqa: E402
from paper_2405_02187_b200 import capi  # noqa: E402

ctx = csf.Context(0)
out = {}
for label, n_frames, units, second in (("config2", 100, bench.DIRS, False), ("config3", 30, bench.PAIRS, True)):
    depth, gt, k = csf.synth_workload(2, n_frames, ctx=ctx)
    rows = {}
    for N in (1, 2, 4, 8):
        mine = units[: math.ceil(len(units) / N)]
        cfg = bench.pipeline_cfg(csf, capi, k, mine, n_frames, pairs=mine if second else None)
        p = csf.Pipeline(cfg, ctx=ctx)
        p.upload(depth, gt)
        p.set_graph(True)
        for _ in range(3):
            p.run()
        ctx.synchronize()
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            p.run()
        ctx.synchronize()
        rows[N] = {"units_per_rank": len(mine), "ms_per_step": 1000 * (time.perf_counter() - t0) / reps}
        del p
    t1 = rows[1]["ms_per_step"]
    for N, r in rows.items():
        r["expected_speedup"] = t1 / r["ms_per_step"]
        r["expected_efficiency"] = r["expected_speedup"] / N
    out[label] = rows
print(json.dumps(out, indent=1))

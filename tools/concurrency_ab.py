"""A/B: one packed 10-direction pipeline vs the directions split over k
pipelines (own context / stream each) enqueued concurrently from k host
threads.  Prints wall ms per run and checks the gradients are identical."""
import sys
import threading
import time

sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi
from bench import pipeline_cfg, DIRS

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
reps = 3
ctx0 = csf.Context(0)
depth, gt, k = csf.synth_workload(2, n, ctx=ctx0)


def run_split(sizes):
    groups, o = [], 0
    for s in sizes:
        groups.append(DIRS[o:o + s])
        o += s
    ctxs = [csf.Context(0) for _ in groups]
    pipes = []
    for c, g in zip(ctxs, groups):
        p = csf.Pipeline(pipeline_cfg(csf, capi, k, g, n), ctx=c)
        p.upload(depth, gt)
        pipes.append(p)

    def go(p):
        p.run()
        p.ctx.synchronize()

    go_all = lambda: [t.join() for t in [threading.Thread(target=go, args=(p,)) for p in pipes] if not t.start()]
    for _ in range(2):
        ths = [threading.Thread(target=go, args=(p,)) for p in pipes]
        [t.start() for t in ths]
        [t.join() for t in ths]
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ths = [threading.Thread(target=go, args=(p,)) for p in pipes]
        [t.start() for t in ths]
        [t.join() for t in ths]
        ts.append((time.perf_counter() - t0) * 1e3)
    grad = np.concatenate([p.result().gradient for p in pipes])
    for p in pipes:
        p.close()
    return min(ts), grad


base_ms, g0 = run_split([10])
print(f"[10]: {base_ms:.1f} ms  ({n * 10 / base_ms * 1e3:.0f} fd/s)", flush=True)
for sizes in ([5, 5], [4, 3, 3], [2, 2, 2, 2, 2], [3, 3, 4]):
    ms, g = run_split(sizes)
    print(f"{sizes}: {ms:.1f} ms  ({n * 10 / ms * 1e3:.0f} fd/s)  identical={np.array_equal(g, g0)} "
          f"maxrel={np.max(np.abs(g - g0) / np.maximum(np.abs(g0), 1e-30)):.2e}", flush=True)

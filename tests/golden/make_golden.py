"""Generate the committed golden fixtures (tests/golden/*.npz) from the CPU
oracle (oracle/, test infrastructure; the reference itself cannot be built
in this container — SURVEY F3 — so these are oracle outputs, not reference
outputs).  They pin the oracle against drift between rounds and give the GPU
tests a fixed answer that does not depend on rebuilding the oracle.

usage: python tests/golden/make_golden.py   (after `make -C oracle`)"""
import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from oracle import orc  # noqa: E402
import paper_2405_02187_b200 as csf  # noqa: E402
from paper_2405_02187_b200 import capi  # noqa: E402

OUT = Path(__file__).resolve().parent


def cases():
    icp = bench.reference_icp()
    # BASELINE config 1 at its stated size: 10 frames, 160x120, dense 128^3 at 2 cm, 6 twist directions
    d1, g1, k1 = orc.workload(1, 10)
    yield "config1_full", d1, g1, bench.pipeline_cfg1(csf, capi, k1, bench.DIRS1, 10, icp=icp)
    # the config-2 scene at 160x120, hashed 2 cm, 3 frames, all 10 directions
    d2, g2, k2 = orc.workload(2, 3, 160, 120)
    import ctypes as C
    hp = capi.HashParams(0.02, (C.c_double * 3)(0.0, 0.0, 0.0), 0.1, 128.0, 16, 1 << 14)
    cfg2 = csf.make_pipeline_cfg(hashed=True, k=k2, dirs=bench.DIRS, h=1e-8,
                                 objective=capi.OBJECTIVE_TRAJECTORY_ERROR, max_frames=3, hash_params=hp, icp=icp)
    yield "config2_small", d2, g2, cfg2


def main():
    for name, depth, gt, cfg in cases():
        grad, obj, poses, stats, _ = orc.pipeline_run(cfg, depth, gt)
        np.savez_compressed(OUT / f"{name}.npz", gradient=grad, objective=np.array([obj]), poses=poses, stats=stats,
                            depth_sha256=np.frombuffer(hashlib.sha256(depth.tobytes()).digest(), dtype=np.uint8))
        print(name, "objective", obj, "gradient", grad)


if __name__ == "__main__":
    main()

"""The C-ABI library loads (no GPU needed) and exports every function
include/csf_b200.h declares; context creation fails loudly without a device."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "csf_b200.h"
LIB = ROOT / "paper_2405_02187_b200" / "_build" / "libcsf_b200.so"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-zA-Z_][\w\s\*]*?\b(csf_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("csf_ctx_create", "csf_surface_update", "csf_raycast", "csf_track_frame", "csf_pipeline_run",
                 "csf_bilateral_filter", "csf_measure_surface", "csf_volume_create_hashed"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not LIB.exists():
        import subprocess
        subprocess.run(["make", "-s", "-C", str(ROOT / "paper_2405_02187_b200")], check=True)
    lib = ctypes.CDLL(str(LIB))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    from paper_2405_02187_b200 import capi
    assert set(capi.EXPORTS) == set(declared_functions())


def test_no_cpu_fallback_without_device():
    import paper_2405_02187_b200 as csf
    lib = csf.library()
    n = ctypes.c_int(0)
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        csf.Context(0)
    # defaults are host-only helpers and work without a device
    c = csf.default_icp_cfg()
    assert c.levels == 3 and list(c.level_iterations) == [10, 5, 4] and list(c.level_pixel_stride) == [1, 1, 2]
    assert c.d_max == 0.1 and c.theta_max_deg == 30.0 and c.step_tolerance == 1e-6

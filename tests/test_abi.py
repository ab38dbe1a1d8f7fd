"""C-ABI checks that need no GPU: libpvr.so loads, exports every function include/pvr.h
declares, the host-only shard planner, and loud failure without a CUDA device."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1611_07289_b200 as P
from paper_1611_07289_b200 import pvr as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pvr.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pvr_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ["pvr_create_volume", "pvr_add_stack", "pvr_extract_patches", "pvr_set_transforms",
              "pvr_sr_iterate", "pvr_get_volume", "pvr_get_weights"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(P.SO_PATH)
    names = declared_functions()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(B.EXPORTS) == names, "binding EXPORTS list out of sync with include/pvr.h"
    nm = subprocess.run(["nm", "-D", "--defined-only", P.SO_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", nm), n


def test_library_is_sm100a_cuda():
    """The shipped .so carries sm_100a SASS (cuobjdump) and links no oracle symbol."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", P.SO_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    nm = subprocess.run(["nm", "-D", P.SO_PATH], capture_output=True, text=True).stdout
    assert "pvro_" not in nm


def test_version_string():
    assert "sm_100a" in P.pvr_version()


@pytest.mark.parametrize("costs,n", [([5, 5, 5, 5, 10], 3), ([1] * 17, 4), ([100, 1, 1, 1], 2),
                                     ([3, 3], 5), ([], 2)])
def test_plan_shards_contiguous_and_balanced(costs, n):
    b = P.pvr_plan_shards(costs, n)
    assert b[0] == 0 and b[-1] == len(costs)
    assert all(x <= y for x, y in zip(b, b[1:]))
    if costs:
        tot = sum(costs)
        loads = [sum(costs[b[r]:b[r + 1]]) for r in range(n)]
        assert max(loads) <= tot / n + max(costs)


def test_plan_shards_rejects_bad_args():
    with pytest.raises(B.PvrError):
        P.pvr_plan_shards([1, 2, 3], 0)


def test_no_cpu_fallback_without_gpu():
    """On a machine without a CUDA device the library fails loudly (PVR_ERR_CUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(B.PvrError) as ei:
        B.pvr_create_volume((8, 8, 8), 1.0, (0, 0, 0))
    assert ei.value.status == B.PVR_ERR_CUDA
    assert "no CUDA device" in str(ei.value)


def test_oracle_and_product_share_no_code():
    """Neither tree includes, imports or links the other."""
    imp = re.compile(r"^\s*(?:import|from)\s+([\w.]+)", re.M)
    inc = re.compile(r'^\s*#\s*include\s*[<"]([^>"]+)[>"]', re.M)
    prod = os.path.join(ROOT, "paper_1611_07289_b200")
    for dirpath, _, files in os.walk(prod):
        for f in files:
            txt = open(os.path.join(dirpath, f), errors="ignore").read() if f.endswith((".py", ".cu", ".h")) else ""
            assert not any(m.split(".")[0] in ("oracle", "synth") for m in imp.findall(txt)), f
            assert not any("pvro" in m or "oracle" in m for m in inc.findall(txt)), f
            assert not re.search(r"\bpvro_\w+\s*\(", txt), f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        txt = open(os.path.join(ROOT, "oracle", f), errors="ignore").read() if f.endswith((".py", ".c", ".h")) else ""
        assert not any(m.split(".")[0] in ("paper_1611_07289_b200", "synth") for m in imp.findall(txt)), f
        assert all(m in ("pvro.h", "math.h", "stdlib.h", "string.h", "omp.h", "stdint.h") for m in inc.findall(txt)), f
        assert not re.search(r"\bpvr_\w+\s*\(", txt), f

"""A/B builds of libpvr.so with compile-time knobs, into ab/ (git-ignored; travels with gpurun).
Usage: python tools/ab_build.py NAME -DKNOB=V ...   then   PVR_SO=$PWD/ab/libpvr_NAME.so python bench.py"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1611_07289_b200"))
import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(b.ROOT, "ab"), exist_ok=True)
out = os.path.join(b.ROOT, "ab", f"libpvr_{name}.so")
cmd = [b.NVCC] + b.FLAGS + defs + ["-I" + os.path.join(b.ROOT, "include"), "-o", out] + b.SRCS + ["-ldl", "-lgomp"]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stdout + r.stderr)
print(out)

"""Build libpvr.so in-tree with nvcc for sm_100a (called by __graft_entry__.build())."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libpvr.so")
SRCS = [os.path.join(HERE, "csrc", f) for f in ("engine.cu", "kernels.cu", "lattice.cu", "registration.cu", "superpixels.cu", "volpsf.cu")]
DEPS = SRCS + [os.path.join(HERE, "csrc", "pvr_internal.h"), os.path.join(HERE, "csrc", "device_util.cuh"), os.path.join(ROOT, "include", "pvr.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-fopenmp", "-shared", "-Xlinker", "--no-undefined", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def build(force=False, verbose=False):
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= max(os.path.getmtime(d) for d in DEPS):
        return SO
    cmd = [NVCC] + FLAGS + ["-I" + os.path.join(ROOT, "include"), "-o", SO] + SRCS + ["-ldl", "-lgomp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    with open(os.path.join(HERE, "build_ptxas.log"), "w") as f:
        f.write(r.stdout + r.stderr)
    if verbose:
        print(r.stderr)
    return SO


if __name__ == "__main__":
    build(force=True, verbose=True)

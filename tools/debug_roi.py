"""Debug the full-size ROI stage check (tests/test_gpu_fullsize.py roi_check): list the voxels
with the largest X differences and their A, C on both sides."""
import sys

import numpy as np

sys.path.insert(0, "."); sys.path.insert(0, "tests")
import synth  # noqa: E402
import test_gpu_fullsize as T  # noqa: E402
from helpers import make_gpu  # noqa: E402
import oracle.pvro as O  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
lo = np.array([int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "24,24,24").split(",")])
size = 48
prob = synth.make_problem(cfg)
ctx = make_gpu(prob)
ctx.init_volume()
X0 = ctx.volume().astype(np.float64)
ctx.sr_iterate(1, prob["alpha"], prob["lam"])
e, kap, A, C = ctx.taps()
p, _, w = ctx.weights()
X1 = ctx.volume().astype(np.float64)
em = ctx.em_state()
pts = ctx.patches()
ctx.close()
dims = tuple(prob["dims"])
A = np.asarray(A, np.float64).reshape(dims[::-1])
C = np.asarray(C, np.float64).reshape(dims[::-1])
hi = lo + size
glo, ghi = np.maximum(lo - 1, 0), np.minimum(hi + 1, dims)
sel = T.patches_reaching(prob, pts, glo, ghi)
npx = (pts[:, 4] * pts[:, 5] * pts[:, 6]).astype(np.int64)
wpix = np.repeat(w.astype(np.float64), npx)
rC = wpix * p.astype(np.float64)
rA = rC * e.astype(np.float64)
orc = T.lazy_oracle(prob)
orc.coverage_subset(sel)
Ao = orc.adjoint_subset(rA, sel).reshape(dims[::-1])
Co = orc.adjoint_subset(rC, sel).reshape(dims[::-1])
box = (slice(glo[2], ghi[2]), slice(glo[1], ghi[1]), slice(glo[0], ghi[0]))
X1o, X2 = O.update_regularise(X0[box], Ao[box], Co[box], prob["alpha"], prob["lam"], 150.0, tau_C=1e-6,
                              clamp=True, lo=em["lo"], hi=em["hi"])
X1g1, _ = O.update_regularise(X0[box], A[box], C[box], prob["alpha"], prob["lam"], 150.0, tau_C=1e-6,
                              clamp=True, lo=em["lo"], hi=em["hi"])
from scipy import ndimage
envC = ndimage.uniform_filter(Co[box], size=3, mode="constant") * 27.0
grazing = ndimage.binary_dilation(Co[box] < 0.1 * envC / 27.0, np.ones((3, 3, 3), bool))
d = np.abs(X1[box] - X2)
d[grazing] = 0
d[:1] = d[-1:] = 0
d[:, :1] = d[:, -1:] = 0
d[:, :, :1] = d[:, :, -1:] = 0
idx = np.argsort(d.ravel())[::-1][:15]
print("em", em)
print("rel X (resolved)", np.linalg.norm(d) / np.linalg.norm(X2[~grazing]))
for k in idx:
    z, y, x = np.unravel_index(k, d.shape)
    print(f"({x + glo[0]},{y + glo[1]},{z + glo[2]}) dX {d[z, y, x]:.3e} Xg {X1[box][z, y, x]:.3f} Xo {X2[z, y, x]:.3f} "
          f"X0 {X0[box][z, y, x]:.3f} Cg {C[box][z, y, x]:.4e} Co {Co[box][z, y, x]:.4e} "
          f"Ag/Cg {A[box][z, y, x] / max(C[box][z, y, x], 1e-30):.4f} Ao/Co {Ao[box][z, y, x] / max(Co[box][z, y, x], 1e-30):.4f} "
          f"X1o {X1o[z, y, x]:.3f} X1(gpu A,C) {X1g1[z, y, x]:.3f} envC/27 {envC[z, y, x] / 27:.3e}")

"""Diagnose the masked-patch parity (f3): per-stage differences GPU vs oracle."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import synth
from helpers import rel_l2
from oracle import Oracle
from paper_1611_07289_b200 import Context
prob = synth.make_problem("c3", scale=(96, 96, 12), size=32, stride=16)
rng = np.random.default_rng(12)
rects = []
for st_i, st in enumerate(prob["stacks"]):
    K, H, W = st["slices"].shape
    for _ in range(40):
        sx, sy = rng.integers(6, 30, 2)
        x0, y0, z0 = rng.integers(0, W - sx + 1), rng.integers(0, H - sy + 1), rng.integers(0, K)
        rects.append([st_i, x0, y0, z0, sx, sy, 1])
rects = np.array(rects, np.int32)
npx = int((rects[:, 4] * rects[:, 5] * rects[:, 6]).sum())
mask = (rng.uniform(size=npx) > float(sys.argv[1]) if len(sys.argv) > 1 else 0.3).astype(np.uint8)
T = np.tile(np.hstack([np.eye(3), np.zeros((3, 1))]), (len(rects), 1, 1))
orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
ctx = Context(prob["dims"], prob["spacing"], prob["origin"])
for st in prob["stacks"]:
    orc.add_stack(st["slices"], st["G"], st["thickness"])
    ctx.add_stack(st["slices"], st["G"], st["thickness"])
orc.set_patches(rects, mask); ctx.set_patches(rects, mask)
orc.set_transforms(T); ctx.set_transforms(T)
orc.init_volume(); ctx.init_volume()
print("init rel", rel_l2(ctx.volume(), orc.volume()))
orc.sr_iterate(1, prob["alpha"], prob["lam"]); ctx.sr_iterate(1, prob["alpha"], prob["lam"])
Xo, Xg = orc.volume(), ctx.volume()
print("iter1 rel", rel_l2(Xg, Xo))
eo, _, Ao, Co = orc.taps(); eg, _, Ag, Cg = ctx.taps()
print("e rel", rel_l2(eg, eo), "A rel", rel_l2(Ag, Ao), "C rel", rel_l2(Cg, Co))
print("em", ctx.em_state(), orc.em_state())
d = np.abs(Xg - Xo); k = np.unravel_index(d.argmax(), d.shape)
print("max diff", d.max(), "at", k, Xg[k], Xo[k], "C", Co.reshape(Xo.shape)[k], Cg.reshape(Xo.shape)[k])
n_flip = ((Co > 1e-3) != (Cg > 1e-3)).sum(); print("tau_C flips", n_flip)

"""Stage-by-stage GPU vs oracle comparison (kappa, init A/C/X, first iteration e/p/A/C/X)."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import synth
from helpers import make_gpu, make_oracle, rel_l2

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
kw = {}
if cfg == "c3s":
    cfg, kw = "c3", dict(scale=(96, 96, 12), size=32, stride=16)
prob = synth.make_problem(cfg, **kw)
orc = make_oracle(prob)
ctx = make_gpu(prob)
print("plan", ctx.stats())
_, ko, _, _ = orc.taps()
_, kg, _, _ = ctx.taps()
print("kappa: max|d| %.3e  gpu nan %d  range %.4f..%.4f / %.4f..%.4f" % (np.abs(kg - ko).max(), np.isnan(kg).sum(), kg.min(), kg.max(), ko.min(), ko.max()))
orc.init_volume(); ctx.init_volume()
_, _, Ao, Co = orc.taps(); _, _, Ag, Cg = ctx.taps()
Xo, Xg = orc.volume(), ctx.volume()
print("init: C rel %.3e A rel %.3e X rel %.3e  nanX %d nanA %d nanC %d" % (rel_l2(Cg, Co), rel_l2(Ag, Ao), rel_l2(Xg, Xo), np.isnan(Xg).sum(), np.isnan(Ag).sum(), np.isnan(Cg).sum()))
bad = np.argwhere(np.abs(Cg - Co) > 1e-3 * np.abs(Co).max())
print("  C mismatches:", len(bad), bad[:5].tolist(), [(float(Cg[tuple(b)]), float(Co[tuple(b)])) for b in bad[:5]])
orc.sr_iterate(1, prob["alpha"], prob["lam"]); ctx.sr_iterate(1, prob["alpha"], prob["lam"])
eo, _, Ao, Co = orc.taps(); eg, _, Ag, Cg = ctx.taps()
po, pbo, wo = orc.weights(); pg, pbg, wg = ctx.weights()
print("iter1: e rel %.3e  max|dp| %.3e max|dw| %.3e  C rel %.3e A rel %.3e X rel %.3e" % (
    rel_l2(eg, eo), np.abs(pg - po).max(), np.abs(wg - wo).max(), rel_l2(Cg, Co), rel_l2(Ag, Ao), rel_l2(ctx.volume(), orc.volume())))
print("em", orc.em_state(), ctx.em_state())

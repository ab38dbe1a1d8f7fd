"""Diagnostic (not a test): GPU vs oracle errors per stage at two threshold sets, with the X
error split by the oracle's confidence C (where fixed-point rounding would show). Prints one
JSON line per (case, thresholds, iteration).

  python tools/diag_thresholds.py [case ...]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import synth  # noqa: E402
from helpers import make_gpu, make_oracle, rel_l2  # noqa: E402

CASES = {
    "c1": ("c1", {}, 3),
    "c2": ("c2", dict(scale=(64, 64, 12)), 2),
    "c3s": ("c3", dict(scale=(96, 96, 12), size=32, stride=16), 2),
    "c4s": ("c4", dict(scale=(96, 96, 16), size=32, stride=16), 2),
    "c5s": ("c5", dict(scale=(64, 64, 12), size=16, stride=4), 1),
    "odd": ("c3", dict(scale=(37, 29, 5), size=8, stride=4), 2),
}
SETS = {"default": {}, "survey": {"tau_C": 1e-6, "tau_obs": 0.01}}


def run(name, setname):
    cfg, kw, iters = CASES[name]
    prob = synth.make_problem(cfg, **kw)
    params = SETS[setname]
    orc = make_oracle(prob, params)
    ctx = make_gpu(prob, params)
    tauC = params.get("tau_C", 1e-3)
    try:
        orc.init_volume()
        ctx.init_volume()
        out = {"case": name, "set": setname, "it": 0, "relX": rel_l2(ctx.volume(), orc.volume())}
        print(json.dumps(out), flush=True)
        for it in range(iters):
            orc.sr_iterate(1, prob["alpha"], prob["lam"])
            ctx.sr_iterate(1, prob["alpha"], prob["lam"])
            Xo, Xg = orc.volume().ravel(), ctx.volume().ravel().astype(np.float64)
            eo, ko, Ao, Co = orc.taps()
            eg, kg, Ag, Cg = ctx.taps()
            Ao, Co, Ag, Cg = Ao.ravel(), Co.ravel(), Ag.ravel(), Cg.ravel()
            po, pbo, wo = orc.weights()
            pg, pbg, wg = ctx.weights()
            emo, emg = orc.em_state(), ctx.em_state()
            d = np.abs(Xg - Xo)
            bins = {}
            for lo, hi in ((0, tauC), (tauC, 1e-5), (1e-5, 1e-4), (1e-4, 1e-3), (1e-3, 1e-2), (1e-2, 1e9)):
                sel = (Co > lo) & (Co <= hi)
                if sel.any():
                    bins[f"{lo:g}-{hi:g}"] = [int(sel.sum()), float(d[sel].max()), float(np.sqrt((d[sel] ** 2).sum()))]
            near = np.abs(Co - tauC)
            flips = int(((Co > tauC) != (Cg > tauC)).sum())
            out = {"case": name, "set": setname, "it": it + 1,
                   "relX": rel_l2(Xg, Xo), "normX": float(np.linalg.norm(Xo)),
                   "rel_e": rel_l2(eg, eo), "rel_A": rel_l2(Ag, Ao), "rel_C": rel_l2(Cg, Co),
                   "max_dC_abs": float(np.abs(Cg - Co).max()),
                   "max_dC_rel_smallC": float((np.abs(Cg - Co) / np.maximum(Co, 1e-30))[(Co > tauC) & (Co < 1e-3)].max()
                                              if ((Co > tauC) & (Co < 1e-3)).any() else 0.0),
                   "max_dk": float(np.abs(kg - ko).max()),
                   "dp": float(np.abs(pg - po).max()), "dw": float(np.abs(wg - wo).max()),
                   "em_rel": {k: abs(emg[k] - emo[k]) / max(abs(emo[k]), 1e-30) for k in ("sigma2", "c", "m")},
                   "flipsC": flips, "min_gap_C": float(near.min()),
                   "n_obs_o": int((ko >= params.get("tau_obs", 0.5)).sum()),
                   "bins": bins}
            print(json.dumps(out), flush=True)
    finally:
        ctx.close()


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        for s in SETS:
            try:
                run(n, s)
            except Exception as ex:  # keep going: this is a survey
                print(json.dumps({"case": n, "set": s, "error": repr(ex)}), flush=True)

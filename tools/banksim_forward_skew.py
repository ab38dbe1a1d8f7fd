# Bank model of the forward corner loads for the x-normal (sagittal) stack under lane orderings
# (rows / blocks of bu x bv lattice points) and c-loop phases per lane: the basis of the
# 8 U x 4 V strips with phase V & 3 in k_lattice_fwd (4.0 -> 1.5 wavefronts per corner load).
import sys
sys.path.insert(0, '.')
import numpy as np
import synth
import oracle.pvro as O
prob = synth.make_problem("c3", scale=(96, 96, 12), size=32, stride=16)
s = prob["spacing"]
st = prob["stacks"][2]
G = np.asarray(st["G"]); c = synth.CONFIGS["c3"]
abc, psi, hw = O.psf_table(c["pitch"], c["pitch"], c["theta"], c["s"])
nu, nv = int(hw[0]), int(hw[1]); hu, hv, hw_ = hw[3], hw[4], hw[5]
R = G[:, :3] / np.linalg.norm(G[:, :3], axis=0)
qa = R[:, 0] * hu / s; qb = R[:, 1] * hv / s; qc = R[:, 2] * hw_ / s
print("qa", qa, "qb", qb, "qc", qc)
LU = LV = 33
origin = np.array([3.3, 5.7, 7.1])
ntp = 15
allp = np.array([origin + U * qa + V * qb for V in range(LV) for U in range(LU)])
lo = np.floor(allp.min(0) - 8); dims = np.ceil(allp.max(0) + 8 - lo).astype(int) + 2
dx = 4 * (((dims[0] + 3) // 4) | 1); dy = dims[1]; dxy = (dx * dy + 31) & ~31
def sim(bu, bv, phase):
    tot = 0; n = 0
    for V0 in range(0, LV - bv + 1, bv):
        for U0 in range(0, LU - bu + 1, bu):
            lanes = np.arange(32)
            U = U0 + lanes % bu; V = V0 + lanes // bu
            P0 = origin + U[:, None] * qa + V[:, None] * qb
            ph = np.array([phase(l) for l in lanes])
            for k in range(ntp):
                cc = (k + ph) % ntp
                P = P0 - lo + cc[:, None] * qc
                fl = np.floor(P).astype(int)
                a = fl[:, 2] * dxy + fl[:, 1] * dx + fl[:, 0]
                ua = np.unique(a)
                tot += np.bincount(ua % 32, minlength=32).max(); n += 1
    return round(tot / n, 2)
print("dx", dx)
for bu, bv in [(32, 1), (16, 2), (8, 4), (4, 8)]:
    for name, ph in [("none", lambda l: 0), ("grp", lambda l, bu=bu: (l // bu) % 4 if bu < 32 else (l >> 3) & 3),
                     ("grp2", lambda l, bu=bu: 2 * ((l // bu) % 4) if bu < 32 else 2 * ((l >> 3) & 3)),
                     ("l&3", lambda l: l & 3), ("l/8", lambda l: l >> 3)]:
        print(bu, bv, name, sim(bu, bv, ph))

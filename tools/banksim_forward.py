# Offline model of the forward's shared-memory bank pattern: per stack orientation,
# the wavefronts of one corner load when 32 lanes take consecutive flattened lattice points.
# Validated against ncu (model 2.13 vs measured 2.17 wavefronts per corner LDS on c3).
# Simulate the forward's shared-memory bank pattern for c3-like members (one member per stack):
# lanes = 32 consecutive flattened lattice points (li = V*LU + U), sample c, corner (0,0,0).
import sys, math
sys.path.insert(0, '.')
import numpy as np
import synth
prob = synth.make_problem("c3", scale=(96, 96, 12), size=32, stride=16)
s = prob["spacing"]; o = np.asarray(prob["origin"])
import oracle.pvro as O
for si, st in enumerate(prob["stacks"]):
    G = np.asarray(st["G"]); c = synth.CONFIGS["c3"]
    abc, psi, hw = O.psf_table(c["pitch"], c["pitch"], c["theta"], c["s"])
    nu, nv, nw = int(hw[0]), int(hw[1]), int(hw[2]); hu, hv, hw_ = hw[3], hw[4], hw[5]
    R = G[:, :3] / np.linalg.norm(G[:, :3], axis=0)
    qa = R[:, 0] * hu / s; qb = R[:, 1] * hv / s; qc = R[:, 2] * hw_ / s
    tu = tv = 16
    LU = nu * (tu - 1) + 2 * (nu - 1) + 1; LV = nv * (tv - 1) + 2 * (nv - 1) + 1
    # tile: box from the member's footprint
    origin = np.array([3.3, 5.7, 7.1])
    pts = []
    for V in range(LV):
        for U in range(LU):
            pts.append(origin + U * qa + V * qb)
    pts = np.array(pts)
    ntp = int(round(2 * 3 * (c["theta"] / 2.3548) / hw_)) + 1
    lo = np.floor(pts.min(0) - 8); dims = np.ceil(pts.max(0) + 8 - lo).astype(int) + 2
    dx = 4 * (((dims[0] + 3) // 4) | 1); dy = dims[1]; dxy = (dx * dy + 31) & ~31
    tot = 0; nw_ = 0
    for cc in range(0, ntp, 3):
        P = pts - lo + cc * qc
        fl = np.floor(P).astype(int)
        addr = fl[:, 2] * dxy + fl[:, 1] * dx + fl[:, 0]
        for w in range(0, len(addr) - 31, 32):
            a = addr[w:w + 32]
            ua = np.unique(a)
            banks = ua % 32
            mult = np.bincount(banks, minlength=32).max()
            tot += mult; nw_ += 1
    print("stack", si, "R cols", np.round(R, 2).T.tolist(), "dx", dx, "avg wavefronts (corner 000)", tot / nw_)

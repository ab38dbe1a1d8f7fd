"""Offline model of the backprojection's shared-atomic wavefronts: for one
member of each c3 stack orientation (with a few degrees of motion), walk the lines the lanes
of each warp take, and count per ATOMS instruction (one transverse corner of plane m for all
lanes) the wavefronts = max over the 32 banks of the lanes hitting that bank (an atomic to the
same word by two lanes serialises like a bank conflict).

  python tools/banksim_bp.py
"""
import math
import sys

import numpy as np

sys.path.insert(0, ".")
import synth  # noqa: E402

s, pitch, theta = 0.75, 1.25, 4.0
nu = 2
qa_len = pitch / nu / s          # 0.833 voxel
nw = math.ceil(theta / s - 1e-9)
qc_len = theta / nw / s          # 0.667 mm / 0.75
cmax = 7
ns = 2 * cmax + 1


def frame(Qc):
    am = int(np.argmax(np.abs(Qc)))
    ap = 1 if am == 0 else 0
    aq = 1 if am == 2 else 2
    return am, ap, aq


def member_lines(R, rot, TU=8, TV=8):
    Rm = synth.generate.euler(*rot) @ R
    Qa, Qb, Qc = Rm[:, 0] * qa_len, Rm[:, 1] * qa_len, Rm[:, 2] * qc_len
    am, ap, aq = frame(Qc)
    d = 1 if Qc[am] >= 0 else -1
    nU, nV = nu * TU, nu * TV
    # tile: bbox of the member (voxel coords), pitches odd
    pts = []
    for U in (0, nU - 1):
        for V in (0, nV - 1):
            for c in (-cmax, cmax):
                pts.append(U * Qa + V * Qb + c * Qc)
    pts = np.array(pts) + 0.37
    lo = np.floor(pts.min(0)) - 0
    hi = np.floor(pts.max(0)) + 1
    dims = (hi - lo + 1).astype(int)
    dims[0] |= 1
    dims[1] |= 1
    return Qa, Qb, Qc, (am, ap, aq), d, nU, nV, lo, dims


def addr(x, lo, dims):
    c = (np.floor(x) - lo).astype(int)
    return c[..., 0] + dims[0] * (c[..., 1] + dims[1] * c[..., 2])


def wavefronts(words):
    banks = words % 32
    _, counts = np.unique(banks, return_counts=True)
    return counts.max()


def simulate(R, rot, order="row", phases=1, TU=8, TV=8):
    Qa, Qb, Qc, (am, ap, aq), d, nU, nV, lo, dims = member_lines(R, rot, TU, TV)
    lines = [(U, V) for V in range(nV) for U in range(nU)]
    if order == "col3":
        lines = [(U, V) for cv in range(3) for cu in range(3) for V in range(cv, nV, 3) for U in range(cu, nU, 3)]
    if order == "alt":  # lanes 0-15 row V, lanes 16-31 row V + 2
        lines = []
        for V0 in range(0, nV, 4):
            for V in (V0, V0 + 2, V0 + 1, V0 + 3):
                if V < nV:
                    lines += [(U, V) for U in range(nU)]
    tot, n = 0, 0
    e = np.zeros(3)
    e[ap] = 1
    f = np.zeros(3)
    f[aq] = 1
    corners = [np.zeros(3), e, f, e + f]
    for w0 in range(0, len(lines), 32):
        warp = lines[w0:w0 + 32]
        for k in range(ns):
            for cj in corners:
                words = []
                for lane, (U, V) in enumerate(warp):
                    kk = (k + (lane % phases) * ns // phases) % ns
                    c = (-cmax + kk) if d > 0 else (cmax - kk)
                    x = U * Qa + V * Qb + c * Qc + 0.37
                    words.append(addr(x + cj, lo, dims))
                tot += wavefronts(np.array(words))
                n += 1
    return tot / n


if __name__ == "__main__":
    R = synth.generate
    for name, Rm in (("axial", R.R_AXIAL), ("coronal", R.R_CORONAL), ("sagittal", R.R_SAGITTAL)):
        for order, ph in (("row", 1), ("row", 2), ("col3", 1), ("alt", 1)):
            v = np.mean([simulate(Rm, rot, order, ph) for rot in ((0, 0, 0), (2.0, -1.5, 2.5))])
            print(f"{name:9s} {order:5s} phases={ph}  wavefronts/ATOMS = {v:.2f}")

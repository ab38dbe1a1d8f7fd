"""Pins of the oracle's volume-space PSF mode (psf_mode 2; "fully flexible and accurate
PSF instead of approximated functions", reading Q34): the PSF evaluated at every voxel centre.

With pixel pitch 2 mm, slice thickness 2 mm, 1 mm voxels, T = I and the pixel centre on a voxel
centre, the voxels of the support sit at in-plane offsets of R = |(i, j)| / 2 pitches and
through-plane offsets of l mm: exactly the c1 lattice of tests/golden/psf_c1.json (R = a / 2,
c h_w = c mm), so the row of W is that worked table (closed form: sinc(pi/2) = 2/pi,
sinc(pi/sqrt2), Gaussian halves at +-1 mm).
"""
import json
import math
import os

import numpy as np
import pytest

import synth
from oracle import Oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _single_pixel_problem(n=9, pitch=2.0, theta=2.0, T=None, W=3, K=3, step=4.0):
    """An n^3 volume (1 mm voxels, centres on integers - (n-1)/2) and one axial W x W x K stack
    whose centre pixel sits on the volume's centre voxel."""
    orc = Oracle((n, n, n), 1.0, np.full(3, -(n - 1) / 2))
    orc.set_param("psf_mode", 2)
    G = synth.generate.stack_G(synth.generate.R_AXIAL, pitch, step, W, W, K, np.zeros(3))
    orc.add_stack(np.zeros((K, W, W)), G, theta)
    orc.extract_patches(W, W)
    orc.set_transforms(np.tile(np.eye(3, 4) if T is None else T, (orc.M, 1, 1)))
    return orc


def test_volume_psf_row_is_the_worked_table():
    g = json.load(open(os.path.join(GOLD, "psf_c1.json")))
    n = 9
    orc = _single_pixel_problem(n)
    table = {tuple(v["abc"]): v["psi"] for v in g["values"]}
    # complete the table by symmetry (|a|, |b|, |c| and a <-> b)
    full = {}
    for (a, b, c), v in table.items():
        for sa in (-1, 1):
            for sb in (-1, 1):
                for sc in (-1, 1):
                    full[(sa * a, sb * b, sc * c)] = v
                    full[(sb * b, sa * a, sc * c)] = v
    full[(0, 1, 1)] = full[(1, 0, 1)] = None  # not in the golden file: checked by ratio below
    rng = np.random.default_rng(3)
    X = rng.uniform(0, 1000, size=(n, n, n))
    yhat, kap = orc.forward(X)
    j = 4  # centre pixel of the 3 x 3 centre slice (slice 1 of 3)
    jc = 9 * 1 + j
    assert kap[jc] == pytest.approx(1.0, abs=1e-15)
    # the row of W by impulse responses
    c = (n - 1) // 2
    for (a, b, cc), v in full.items():
        if v is None:
            continue
        E = np.zeros((n, n, n))
        E[c + cc, c + b, c + a] = 1.0
        col, _ = orc.forward(E)
        assert abs(col[jc] - v) <= 1e-10, ((a, b, cc), col[jc], v)
    # (1, 0, 1): in-plane 2/pi times through-plane 1/2 of the centre weight (separable PSF)
    E = np.zeros((n, n, n))
    E[c + 1, c, c + 1] = 1.0
    col, _ = orc.forward(E)
    E = np.zeros((n, n, n))
    E[c, c, c] = 1.0
    col0, _ = orc.forward(E)
    assert abs(col[jc] / col0[jc] - (2 / math.pi) * 0.5) <= 1e-12
    # R = 1 (two pitches in-plane) and |c| > 3 sigma are outside the support
    for off in ((2, 0, 0), (0, 2, 0), (0, 0, 3)):
        E = np.zeros((n, n, n))
        E[c + off[2], c + off[1], c + off[0]] = 1.0
        col, _ = orc.forward(E)
        assert col[jc] == 0.0


def test_volume_psf_constant_linear_and_rotation():
    """Rows sum to 1 (constant fields exact, kappa = 1 inside); the support is symmetric about
    a voxel-centred pixel, so a linear field is reproduced at the centre; a rotation by 90 deg
    about the slice normal (through the centre) maps the voxel lattice onto itself and leaves
    the radially symmetric PSF's row unchanged."""
    n = 11
    orc = _single_pixel_problem(n)
    yh, kap = orc.forward(np.full((n, n, n), 321.5))
    obs = kap >= 0.01
    assert np.abs(yh[obs] - 321.5).max() <= 1e-10
    l, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    c = (n - 1) // 2
    yh, kap = orc.forward(0.7 * i - 1.3 * j + 2.1 * l + 5.0)
    jc = 9 * 1 + 4
    assert abs(yh[jc] - (0.7 * c - 1.3 * c + 2.1 * c + 5.0)) <= 1e-9
    R = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    T = np.hstack([R, np.zeros((3, 1))])            # about the world origin = the centre voxel
    orc2 = _single_pixel_problem(n, T=T)
    rng = np.random.default_rng(5)
    X = rng.normal(size=(n, n, n))
    a, _ = orc.forward(X)
    b, _ = orc2.forward(np.rot90(X, k=1, axes=(2, 1)).copy())
    assert abs(a[jc] - b[jc]) <= 1e-10 * max(1.0, abs(a[jc]))


def test_volume_psf_adjoint_identity_and_partial_coverage():
    """<W x, y> = <x, W^T y> to 1e-10 with oblique stacks and moving patches; pixels near the
    grid border are observed with kappa in (0, 1)."""
    prob = synth.make_problem("c5", scale=(24, 24, 5), size=8, stride=4)
    orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
    orc.set_param("psf_mode", 2)
    for st in prob["stacks"]:
        orc.add_stack(st["slices"], st["G"], st["thickness"])
    pp = prob["patch"]
    orc.extract_patches(pp["size"], pp["stride"], pp["depth"], pp["stride_z"])
    orc.set_transforms(prob["T"])
    rng = np.random.default_rng(11)
    x = rng.normal(size=orc.V)
    Wx, kap = orc.forward(x)
    y = rng.normal(size=orc.P)
    y[kap < 0.01] = 0.0
    lhs, rhs = float(Wx @ y), float(x @ orc.adjoint(y).ravel())
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), 1.0)
    assert ((kap > 0) & (kap < 1 - 1e-9)).sum() > 0 and (kap > 1 - 1e-12).sum() > 0

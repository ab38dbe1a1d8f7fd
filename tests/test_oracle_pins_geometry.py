"""Pins for oracle functions the first pin set left loose (round-1 mutation probe):

* the PSF sample offsets of step 1 (sample_pos): a field quadratic along one world axis
  sees the PSF's second moment along that axis, so the in-plane and through-plane lattice
  steps (and the axis each one runs along) are fixed by closed forms;
* the init neighbour fill: an uncovered voxel takes the mean of its covered
  26-neighbours, counted by hand;
* the diffusivity source of the regulariser (Q17): b_d is formed from X0, not X1;
* the clamp range (Q19): it spans the *live* y only.

Each closed form is worked out in tests/golden/*.json (with its citation) or written out
below from the geometry of the case; none calls the oracle's own arithmetic.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle.pvro as O
import synth
from oracle import Oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


R = {"ax": synth.generate.R_AXIAL, "cor": synth.generate.R_CORONAL, "sag": synth.generate.R_SAGITTAL}


def _grid_problem(tag, n=12, K=4, step=3.0, thickness=2.0):
    """n^3 volume at 1 mm with voxel centres on half-integers; one n x n x K stack (pitch 1 mm,
    slice step 3 mm, thickness 2 mm) whose pixel centres all sit on voxel centres."""
    orc = Oracle((n, n, n), 1.0, np.full(3, -(n - 1) / 2))
    G = synth.generate.stack_G(R[tag], 1.0, step, n, n, K, np.zeros(3))
    orc.add_stack(np.zeros((K, n, n)), G, thickness)
    orc.extract_patches(n, n)                       # one whole-slice patch per slice
    orc.set_transforms(np.tile(np.eye(3, 4), (orc.M, 1, 1)))
    return orc, G


@pytest.mark.parametrize("tag", ["ax", "cor", "sag"])
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_psf_second_moment_along_each_axis(tag, axis):
    """P:158 PSF offsets (sample_pos): X = (x_axis - x0)^2 (voxel units). Along the slice
    normal the samples sit on voxel planes (h_w = 1 voxel) and trilinear is exact, so
    yhat - f(centre) = sum_c tp(c) (c h_w)^2 = 12/17 (golden). Along an in-plane axis the
    samples sit at +-1/2 voxel, where linear interpolation of a quadratic gains 1/4, so
    yhat - f(centre) = P(a != 0) / 2 (golden). A swapped step, or an offset put along the
    wrong frame axis, moves the value to the other closed form (or 0)."""
    g = gold("psf_moments.json")
    n = 12
    orc, G = _grid_problem(tag, n)
    idx = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")  # (l, j, i)
    coord = [idx[2], idx[1], idx[0]][axis].astype(np.float64)
    x0 = 4.25
    yhat, kap = orc.forward((coord - x0) ** 2)
    normal = np.abs(G[:, 2]) / np.linalg.norm(G[:, 2])
    expect = g["through_plane"]["second_moment_mm2"] if normal[axis] > 0.5 else g["in_plane"]["excess_voxel2"]
    checked = 0
    j = 0
    for st, xa, ya, za, sx, sy, sz in orc.patches():
        for z in range(sz):
            for v in range(sy):
                for u in range(sx):
                    if kap[j] > 1 - 1e-12:      # every corner of every sample in the grid
                        w = G @ np.array([xa + u, ya + v, za + z, 1.0])
                        c = w[axis] + (n - 1) / 2                 # voxel index of the centre
                        assert abs(yhat[j] - ((c - x0) ** 2 + expect)) <= 1e-9, (j, yhat[j], c)
                        checked += 1
                    j += 1
    assert checked >= 100


def _delta_identity(n, mask_out, K=None):
    """Delta PSF on an identity grid: pixel (u, v, z) of the single axial stack observes
    voxel (u, v, z) with W = 1. One 3D patch covers the stack; `mask_out` lists the (i, j, l)
    pixels masked out of it (never observed, reading Q32)."""
    K = K or n
    orc = Oracle((n, n, n), 1.0, np.full(3, -(n - 1) / 2))
    orc.set_param("psf_mode", 1)
    rng = np.random.default_rng(17)
    y = rng.uniform(100.0, 900.0, size=(K, n, n))
    G = synth.generate.stack_G(R["ax"], 1.0, 1.0, n, n, K, np.zeros(3))
    orc.add_stack(y, G, 1.0)
    mask = np.ones((K, n, n), np.uint8)
    for i, j, l in mask_out:
        mask[l, j, i] = 0
    orc.set_patches(np.array([[0, 0, 0, 0, n, n, K]], np.int32), mask.ravel())
    orc.set_transforms(np.tile(np.eye(3, 4), (1, 1, 1)))
    return orc, y, mask


def test_init_fill_is_the_mean_of_the_covered_26_neighbours():
    """P:89 ("empty voxels filled using the mean of the surrounding voxels"), SURVEY 8(c)
    Init: voxels no pixel observes get the mean of X = A/C over their covered 26-neighbours.
    With W = 1 a covered voxel is X = y; the fills are counted by hand: an interior hole (26
    covered neighbours), a hole next to another hole (25), a grid corner (7) and a grid edge
    voxel whose neighbours are partly holes."""
    n = 8
    holes = [(3, 3, 3), (5, 5, 5), (5, 6, 5), (0, 0, 0), (0, 4, 7), (1, 4, 7)]
    orc, y, mask = _delta_identity(n, holes)
    orc.init_volume()
    X = orc.volume()
    cov = mask.astype(bool)
    assert np.array_equal(X[cov], y[cov])
    for i, j, l in holes:
        vals = []
        for dl in (-1, 0, 1):
            for dj in (-1, 0, 1):
                for di in (-1, 0, 1):
                    if di == dj == dl == 0:
                        continue
                    a, b, c = i + di, j + dj, l + dl
                    if 0 <= a < n and 0 <= b < n and 0 <= c < n and cov[c, b, a]:
                        vals.append(y[c, b, a])
        assert len(vals) == {(3, 3, 3): 26, (5, 5, 5): 25, (5, 6, 5): 25, (0, 0, 0): 7,
                             (0, 4, 7): 10, (1, 4, 7): 16}[(i, j, l)]
        assert abs(X[l, j, i] - np.mean(vals)) <= 1e-12 * 900, (i, j, l)


def test_init_fill_without_covered_neighbours_is_zero():
    """SURVEY 8(c) Init: a hole whose 26 neighbours are all holes stays 0."""
    n = 6
    holes = [(i, j, l) for i in range(1, 4) for j in range(1, 4) for l in range(1, 4)]
    orc, _, _ = _delta_identity(n, holes)
    orc.init_volume()
    X = orc.volume()
    assert X[2, 2, 2] == 0.0 and X[1, 1, 1] != 0.0


def test_regulariser_diffusivity_comes_from_X0():
    """P:97 / Q17: b_d(k) = phi_d / sqrt(1 + phi_d ((X0_{k+d} - X0_k) /
    delta)^2) weighs differences of X1. Two voxels along x with X0 = (0, delta) (so b = 1/sqrt2,
    golden R4) and A / C = (0, 2 delta) (so X1 = (0, 3 delta), for which b would be 1/sqrt10):
    X2 = X1 + alpha lambda b (X1_other - X1)."""
    g = gold("regulariser.json")
    b = g["R4_diffusivity"]["cases"][0]["b"]            # dX0 = delta on an axis
    delta, lam = 150.0, 0.05
    X0 = np.array([0.0, delta]).reshape(1, 1, 2)
    A = np.array([0.0, 2 * delta]).reshape(1, 1, 2)
    X1, X2 = O.update_regularise(X0, A, np.ones_like(X0), 1.0, lam, delta)
    assert np.array_equal(X1.ravel(), [0.0, 3 * delta])
    assert abs(X2.ravel()[0] - lam * b * 3 * delta) <= 1e-9
    assert abs(X2.ravel()[1] - (3 * delta - lam * b * 3 * delta)) <= 1e-9
    assert abs(X2.ravel()[0] - lam * 3 * delta / math.sqrt(10.0)) > 1.0


def test_clamp_range_spans_live_pixels_only():
    """Q19: the clamp interval [y_min - 0.1|y_min|, y_max + 0.1|y_max|] is taken over live y
    (kappa >= 0.99). Delta PSF on an identity grid with the stack shifted 3 voxels along +x:
    its last 3 columns fall outside the volume (kappa = 0), and they hold extreme values that
    must not widen the interval. With alpha = 3 from X0 = 0 the step 3 y overshoots, so the
    clamp binds at the live maximum's bound."""
    n, shift = 8, 3
    orc = Oracle((n, n, n), 1.0, np.full(3, -(n - 1) / 2))
    orc.set_param("psf_mode", 1)
    orc.set_param("tau_patch", 0.0)
    rng = np.random.default_rng(23)
    y = rng.uniform(100.0, 900.0, size=(n, n, n))
    y[:, :, n - shift:] = 5000.0                 # columns outside the grid
    y[:, 0, n - shift:] = -3000.0
    G = synth.generate.stack_G(R["ax"], 1.0, 1.0, n, n, n, np.array([float(shift), 0.0, 0.0]))
    orc.add_stack(y, G, 1.0)
    orc.extract_patches(n, n)
    orc.set_transforms(np.tile(np.eye(3, 4), (orc.M, 1, 1)))
    live = y[:, :, :n - shift]
    lo = live.min() - 0.1 * abs(live.min())
    hi = live.max() + 0.1 * abs(live.max())
    em = orc.em_state()
    assert abs(em["lo"] - lo) <= 1e-12 * hi and abs(em["hi"] - hi) <= 1e-12 * hi
    orc.set_volume(np.zeros((n, n, n)))
    orc.sr_iterate(1, 3.0, 0.0)
    X = orc.volume()
    inside = X[:, :, shift:]                     # voxels the live columns observe
    assert abs(inside.max() - hi) <= 1e-9 and inside.min() >= lo - 1e-9
    np.testing.assert_allclose(inside[3.0 * live <= hi], 3.0 * live[3.0 * live <= hi], rtol=0, atol=1e-9)

"""Pins of the f1 registration oracle (oracle/pvro.c: pvro_cc, pvro_blur, pvro_compose_pose,
pvro_patch_cc, pvro_register; reading Q29) against
SPEC's worked examples, closed forms and ground-truth transforms."""
import math

import numpy as np
import pytest
from scipy import ndimage

import oracle.pvro as O
from helpers import make_oracle
from regprob import euler_deg, patch_centre_world, pose_error, registration_problem, rigid_about


# ------------------------------------------------------------- CC
def test_cc_spec_examples():
    """x vs x -> 1; (1,2,3,4) vs (4,3,2,1) -> -1; x vs a x + b (a > 0) -> 1 within
    1e-9; symmetric; constant side -> undefined."""
    rng = np.random.default_rng(0)
    x = rng.normal(size=500)
    assert abs(O.cc(x, x) - 1.0) <= 1e-12
    assert O.cc([1, 2, 3, 4], [4, 3, 2, 1]) == -1.0
    assert abs(O.cc(x, 3.7 * x - 12.0) - 1.0) <= 1e-9
    y = rng.normal(size=500)
    assert O.cc(x, y) == O.cc(y, x)
    assert abs(O.cc(x, y) - np.corrcoef(x, y)[0, 1]) <= 1e-12   # library routine
    assert math.isnan(O.cc(x, np.full(500, 2.0)))


@pytest.fixture(scope="module")
def c1_reg():
    prob, X = registration_problem("c1", blur=0.5, texture=300.0)
    orc = make_oracle(prob)
    orc.set_volume(X)
    return prob, X, orc


# ------------------------------------------------------------- pose composition
def test_compose_pose_closed_forms(c1_reg):
    """Zero pose leaves T; a pure translation adds t; any pose fixes the transformed patch
    centre up to t (rotation about the centre, Q29)."""
    prob, _, orc = c1_reg
    pts = orc.patches()
    T0 = np.asarray(prob["T"][5], np.float64).reshape(3, 4)
    assert np.array_equal(orc.compose_pose(5, np.zeros(6)), T0)
    Tt = orc.compose_pose(5, [1.5, -2.0, 0.25, 0, 0, 0])
    assert np.abs(Tt - (T0 + np.array([[0, 0, 0, 1.5], [0, 0, 0, -2.0], [0, 0, 0, 0.25]]))).max() <= 1e-12
    c = patch_centre_world(prob, pts[5], T0)
    Tr = orc.compose_pose(5, [0.5, 0.0, -1.0, 7.0, -3.0, 11.0])
    assert np.abs(Tr[:, :3] @ np.linalg.solve(T0[:, :3], c - T0[:, 3]) + Tr[:, 3] - (c + [0.5, 0, -1.0])).max() <= 1e-12
    R = Tr[:, :3] @ np.linalg.inv(T0[:, :3])
    assert np.abs(R @ R.T - np.eye(3)).max() <= 1e-12
    assert np.abs(R - euler_deg(7.0, -3.0, 11.0)).max() <= 1e-12   # R = Rz Ry Rx


# ------------------------------------------------------------- CC of a patch
def test_patch_cc_is_one_at_the_true_pose_and_lower_off_it(c1_reg):
    """Patches that are trilinear samples of X at their pixel positions correlate perfectly
    with X at the identity pose (S:250 identity case) and less under any displacement."""
    _, X, orc = c1_reg
    for s in (0, 40, 77, 150):
        cc, nv = orc.patch_cc(X, s, np.zeros(6))
        if nv < 32:
            continue
        assert abs(cc - 1.0) <= 1e-9, (s, cc)
        for pose in ([1.0, 0, 0, 0, 0, 0], [0, 0, 0, 0, 0, 4.0], [0, -0.5, 0.5, 2.0, 0, 0]):
            assert orc.patch_cc(X, s, pose)[0] < cc


def test_patch_cc_out_of_grid_reads_zero_and_undefined_cases(c1_reg):
    """Samples outside the grid read 0 (corners dropped, Q6): a patch moved fully outside
    correlates with a constant -> undefined; a constant volume -> undefined."""
    _, X, orc = c1_reg
    cc, nv = orc.patch_cc(X, 10, [100.0, 0, 0, 0, 0, 0])
    assert nv == 256 and math.isnan(cc)
    cc, nv = orc.patch_cc(np.full_like(X, 3.0), 10, np.zeros(6))
    assert math.isnan(cc)


# ------------------------------------------------------------- registration
def test_register_keeps_true_poses(c1_reg):
    """a patch simulated at its current pose stays there (no move improves CC 1)."""
    prob, X, orc = c1_reg
    T, st, poses = orc.register()
    ok = st == 1
    assert ok.mean() > 0.8
    assert np.abs(poses[ok]).max() == 0.0
    assert np.array_equal(T[ok], np.asarray(prob["T"], np.float64).reshape(-1, 3, 4)[ok])


@pytest.mark.parametrize("cfg,kw,frac", [("c1", {}, 0.8),
                                         ("c3", dict(scale=(64, 64, 8), size=32, stride=16), 0.95)])
def test_register_recovers_injected_displacements(cfg, kw, frac):
    """patches displaced by a known 3 mm / 5 degree rigid motion (random axis and
    direction) are recovered within 0.5 mm / 1 degree of the generating (identity) transform.
    The volume carries a smooth random texture so every pose parameter is observable."""
    prob, X = registration_problem(cfg, blur=0.5, texture=300.0, **kw)
    orc = make_oracle(prob)
    orc.set_volume(X)
    pts = orc.patches()
    I34 = np.hstack([np.eye(3), np.zeros((3, 1))])
    interior = [s for s, pt in enumerate(pts)
                if (prob["stacks"][pt[0]]["slices"][pt[3]:pt[3] + pt[6], pt[2]:pt[2] + pt[5], pt[1]:pt[1] + pt[4]] != 0).mean() > 0.99]
    moved = interior[::max(1, len(interior) // 16)]
    rng = np.random.default_rng(5)
    T = np.asarray(prob["T"], np.float64).reshape(-1, 3, 4).copy()
    for s in moved:
        c = patch_centre_world(prob, pts[s], T[s])
        axis = rng.normal(size=3)
        axis /= np.linalg.norm(axis)
        t = rng.normal(size=3)
        t *= 3.0 / np.linalg.norm(t)
        T[s] = rigid_about(ndimage_free_axis_angle(axis, 5.0), c, t)
    orc.set_transforms(T)
    Tout, st, _ = orc.register()
    errs = np.array([pose_error(Tout[s], I34, patch_centre_world(prob, pts[s], I34)) for s in moved])
    good = ((errs[:, 0] <= 0.5) & (errs[:, 1] <= 1.0)).sum()
    assert good >= frac * len(moved), (good, len(moved), np.median(errs, 0))


def ndimage_free_axis_angle(axis, deg):
    a = math.radians(deg)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(a) * K + (1 - math.cos(a)) * (K @ K)


def test_register_flags_constant_patches_unregistrable():
    """a constant patch has an undefined CC -> flagged, transform unchanged."""
    prob, X = registration_problem("c1", blur=0.5, texture=300.0)
    prob["stacks"][0]["slices"][:] = 5.0
    orc = make_oracle(prob)
    orc.set_volume(X)
    T, st, _ = orc.register(levels=1, iters=2)
    pts = orc.patches()
    on0 = pts[:, 0] == 0
    assert (st[on0] == 0).all() and (st[~on0] == 1).mean() > 0.8
    assert np.array_equal(T[on0], np.asarray(prob["T"], np.float64).reshape(-1, 3, 4)[on0])

"""Full-size checks in the configuration bench.py times (c3, 427^3, 11760 patches): sampled
outputs against the oracle computed patch by patch, and identities that hold at any size."""
import numpy as np
import pytest

import synth
from helpers import make_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    return synth.make_problem("c3")


def smooth_field(dims):
    """Synthetic smooth volume (no oracle or GPU arithmetic involved): [nz][ny][nx] float64."""
    nx, ny, nz = dims
    i = np.arange(nx)[None, None, :]
    j = np.arange(ny)[None, :, None]
    l = np.arange(nz)[:, None, None]
    return 500.0 + 200.0 * np.sin(0.05 * i + 0.3) * np.cos(0.07 * j) + 100.0 * np.sin(0.03 * l + 1.0)


def patch_pixels_y(prob, patches):
    """y_j of every local patch pixel in the product's patch-major order (gathered from stacks)."""
    out = []
    for st, x0, y0, z0, sx, sy, sz in patches:
        out.append(prob["stacks"][st]["slices"][z0:z0 + sz, y0:y0 + sy, x0:x0 + sx].ravel())
    return np.concatenate(out).astype(np.float64)


def test_c3_forward_sampled_vs_oracle(c3):
    from oracle import Oracle
    X = smooth_field(c3["dims"])
    ctx = make_gpu(c3)
    try:
        ctx.set_volume(np.ascontiguousarray(X, np.float32))
        ctx.sr_iterate(1, 0.0, 0.0)                 # alpha = 0: residual of X, no update
        e_g, kap_g, _, _ = ctx.taps()
        pts = ctx.patches()
    finally:
        ctx.close()
    y = patch_pixels_y(c3, pts)
    orc = Oracle(c3["dims"], c3["spacing"], c3["origin"])
    orc.set_param("lazy", 1)
    for st in c3["stacks"]:
        orc.add_stack(st["slices"], st["G"], st["thickness"])
    pp = c3["patch"]
    orc.extract_patches(pp["size"], pp["stride"], pp["depth"], pp["stride_z"])
    orc.set_transforms(c3["T"])
    orc.set_volume(X)
    rng = np.random.default_rng(0)
    sample = np.sort(rng.choice(orc.M, size=24, replace=False))
    npx = pp["size"] ** 2 * pp["depth"]
    checked = 0
    for s in sample:
        yh_o, kap_o = orc.forward_range(X, int(s), 1)
        sl = slice(s * npx, (s + 1) * npx)
        assert np.abs(kap_g[sl] - kap_o[sl]).max() <= 2e-5
        obs = kap_o[sl] >= 0.5
        yh_g = y[sl][obs] - e_g[sl][obs]
        if obs.any():
            rel = np.linalg.norm(yh_g - yh_o[sl][obs]) / np.linalg.norm(yh_o[sl][obs])
            assert rel <= 2e-6, (s, rel)
            checked += obs.sum()
    assert checked > 20000


def test_c3_adjoint_conserves_weight(c3):
    """Every observed row of W sums to 1, so sum_k C_k = sum_j w p and sum_k A_k = sum_j w p e
    exactly: checks the whole backprojection at full size."""
    ctx = make_gpu(c3)
    try:
        ctx.init_volume()
        ctx.sr_iterate(1, c3["alpha"], c3["lam"])
        e, kap, A, C = ctx.taps()
        p, pbar, w = ctx.weights()
        pts = ctx.patches()
        X = ctx.volume()
    finally:
        ctx.close()
    npx = pts[:, 4] * pts[:, 5] * pts[:, 6]
    wpix = np.repeat(w.astype(np.float64), npx)
    obs = kap >= 0.5
    rC = (wpix * p)[obs]
    rA = (wpix * p * e)[obs]
    assert abs(C.sum(dtype=np.float64) - rC.sum()) <= 1e-5 * rC.sum()
    assert abs(A.sum(dtype=np.float64) - rA.sum()) <= 1e-5 * np.abs(rA).sum()
    assert (C >= -1e-6).all()
    assert np.isfinite(X).all()


def test_c3_init_is_a_weighted_mean(c3):
    """Init X = W^T y / W^T 1 is a convex combination of observed y (neighbour fill too)."""
    ctx = make_gpu(c3)
    try:
        ctx.init_volume()
        X = ctx.volume()
        _, kap, _, _ = ctx.taps()
        pts = ctx.patches()
    finally:
        ctx.close()
    y = patch_pixels_y(c3, pts)[kap >= 0.5]
    assert X.min() >= y.min() - 1e-3 * abs(y.min()) - 1e-3
    assert X.max() <= y.max() * (1 + 1e-6) + 1e-3


def test_c3_rigidity_map_closed_forms(c3):
    """f2 at full size, in the launch configuration of bench.py's extras: right after
    set_transforms (p = pbar = 1) the map is exactly 1 on every observed voxel (SPEC 'all
    posteriors 1'); after iterations it stays a weighted mean of p pbar in [0, 1]."""
    ctx = make_gpu(c3)
    try:
        R = ctx.rigidity_map()
        on = R != 0
        assert on.mean() > 0.3
        assert np.abs(R[on] - 1.0).max() <= 1e-5
        ctx.init_volume()
        ctx.sr_iterate(1, c3["alpha"], c3["lam"])
        R = ctx.rigidity_map()
        assert (R >= 0).all() and (R <= 1.0 + 1e-5).all()
        _, pb, _ = ctx.weights()
        assert R[R != 0].mean() <= 1.0 and R[R != 0].mean() >= 0.5 * pb.mean() ** 2
    finally:
        ctx.close()

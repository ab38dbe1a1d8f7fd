"""Full-size checks in the configurations bench.py times (c3: 427^3, 11760 patches; c4: 3D
patches with 10% gross errors; c5: 800^3 with oblique stacks): element-wise comparisons in
regions of interest against the oracle computed over exactly the patches that reach them,
sampled outputs the oracle computes patch by patch, and identities that hold at any size.

The ROI checks take the GPU's own per-pixel adjoint inputs (w p e, w p) of one iteration and
backproject them with the oracle (pvro_adjoint_subset over every patch whose footprint can
reach the ROI; any other patch contributes exactly 0 there), then run the oracle's update on
the ROI with the GPU's pre-iteration volume: each stage is held to its own bar at full size.
"""
import numpy as np
import pytest

import synth
from helpers import TAU_OBS, make_gpu, record, rel_l2, tau_c_tie_band

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    return synth.make_problem("c3")


@pytest.fixture(scope="module")
def c4():
    return synth.make_problem("c4")


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


def lazy_oracle(prob, params=None):
    """The oracle on the full problem without its whole-volume coverage pass (PVRO_LAZY)."""
    from oracle import Oracle
    orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
    orc.set_param("lazy", 1)
    for k, v in (params or {}).items():
        orc.set_param(k, v)
    for st in prob["stacks"]:
        orc.add_stack(st["slices"], st["G"], st["thickness"])
    pp = prob["patch"]
    orc.extract_patches(pp["size"], pp["stride"], pp["depth"], pp["stride_z"])
    orc.set_transforms(prob["T"])
    return orc


def patches_reaching(prob, patches, lo, hi):
    """Indices of the patches whose footprint (pixel centres under T, grown by the PSF's
    in-plane and through-plane support and the trilinear corner) can touch voxels [lo, hi)."""
    s = prob["spacing"]
    o = np.asarray(prob["origin"])
    sel = []
    for k, (st, x0, y0, z0, sx, sy, sz) in enumerate(patches):
        G = np.asarray(prob["stacks"][st]["G"])
        T = np.asarray(prob["T"][k])
        c = np.array([[x0 + a, y0 + b, z0 + d, 1.0] for a in (0, sx - 1) for b in (0, sy - 1) for d in (0, sz - 1)])
        w = (T[:, :3] @ (G @ c.T) + T[:, 3:4]).T
        v = (w - o) / s
        pitch = max(np.linalg.norm(G[:, 0]), np.linalg.norm(G[:, 1]))
        margin = (pitch + 1.5 * prob["stacks"][st]["thickness"]) / s + 2.0
        vlo, vhi = v.min(0) - margin, v.max(0) + margin
        if np.all(vhi >= lo) and np.all(vlo < hi):
            sel.append(k)
    return np.array(sel, np.int64)


def forward_sampled(prob, stacks=None, nsample=24, seed=0):
    """GPU residual of a smooth volume (alpha = 0: one forward, no update) against the oracle's
    forward of sampled patches (optionally only of the given stacks)."""
    X = smooth_field(prob["dims"])
    ctx = make_gpu(prob)
    try:
        ctx.set_volume(np.ascontiguousarray(X, np.float32))
        ctx.sr_iterate(1, 0.0, 0.0)
        e_g, kap_g, _, _ = ctx.taps()
        pts = ctx.patches()
    finally:
        ctx.close()
    y = patch_pixels_y(prob, pts)
    orc = lazy_oracle(prob)
    orc.set_volume(X)
    rng = np.random.default_rng(seed)
    pool = np.arange(orc.M) if stacks is None else np.flatnonzero(np.isin(pts[:, 0], stacks))
    sample = np.sort(rng.choice(pool, size=nsample, replace=False))
    npx = (pts[:, 4] * pts[:, 5] * pts[:, 6]).astype(np.int64)
    first = np.concatenate([[0], np.cumsum(npx)])
    checked, worst = 0, 0.0
    for s in sample:
        yh_o, kap_o = orc.forward_range(X, int(s), 1)
        sl = slice(first[s], first[s + 1])
        assert np.abs(kap_g[sl] - kap_o[sl]).max() <= 1.3e-5
        obs = kap_o[sl] >= TAU_OBS
        yh_g = y[sl][obs] - e_g[sl][obs]
        if obs.any():
            rel = np.linalg.norm(yh_g - yh_o[sl][obs]) / np.linalg.norm(yh_o[sl][obs])
            worst = max(worst, rel)
            assert rel <= 2e-6, (s, rel)
            checked += obs.sum()
    record({"forward_sampled_patches": len(sample), "pixels": int(checked), "worst_rel": worst})
    print(f"forward sampled: {len(sample)} patches, {checked} pixels, worst rel {worst:.2e}")
    return checked


def roi_check(prob, roi_lo, roi_size, params=None):
    """One iteration on the GPU; A, C in the ROI from the oracle's adjoint of the GPU's w p e and
    w p over the patches reaching it (rel L2 <= 1e-5 each); then X in the ROI from the oracle's
    update of the GPU's pre-iteration volume with those A, C (rel L2 <= 1e-5)."""
    import oracle.pvro as O
    lo = np.asarray(roi_lo)
    hi = lo + roi_size
    ctx = make_gpu(prob, params)
    try:
        ctx.init_volume()
        X0 = ctx.volume().astype(np.float64)
        ctx.sr_iterate(1, prob["alpha"], prob["lam"])
        e, kap, A, C = ctx.taps()
        p, _, w = ctx.weights()
        X1 = ctx.volume().astype(np.float64)
        em = ctx.em_state()
        pts = ctx.patches()
    finally:
        ctx.close()
    dims = tuple(prob["dims"])
    A = np.asarray(A, np.float64).reshape(dims[::-1])
    C = np.asarray(C, np.float64).reshape(dims[::-1])
    # one voxel more on every side for the regulariser's stencil
    glo, ghi = np.maximum(lo - 1, 0), np.minimum(hi + 1, dims)
    sel = patches_reaching(prob, pts, glo, ghi)
    npx = (pts[:, 4] * pts[:, 5] * pts[:, 6]).astype(np.int64)
    wpix = np.repeat(w.astype(np.float64), npx)
    rC = wpix * p.astype(np.float64)
    rA = rC * e.astype(np.float64)
    orc = lazy_oracle(prob, params)
    orc.coverage_subset(sel)
    Ao = orc.adjoint_subset(rA, sel).reshape(dims[::-1])
    Co = orc.adjoint_subset(rC, sel).reshape(dims[::-1])
    Aabs = orc.adjoint_subset(np.abs(rA), sel).reshape(dims[::-1])
    box = (slice(glo[2], ghi[2]), slice(glo[1], ghi[1]), slice(glo[0], ghi[0]))
    inner = tuple(slice(lo[d] - glo[d], lo[d] - glo[d] + roi_size) for d in (2, 1, 0))
    dA = A[box][inner] - Ao[box][inner]
    ra, rc = rel_l2(A[box][inner], Ao[box][inner]), rel_l2(C[box][inner], Co[box][inner])
    # A = W^T (w p e) sums residuals of both signs: its fp32 error scales with W^T |w p e|
    ra_abs = np.linalg.norm(dA) / np.linalg.norm(Aabs[box][inner])
    assert (Co[box][inner] > 0).mean() > 0.5, "ROI mostly unobserved"
    tau_C = (params or {}).get("tau_C", 1e-6)
    _, X2 = O.update_regularise(X0[box], Ao[box], Co[box], prob["alpha"], prob["lam"], 150.0, tau_C=tau_C,
                                clamp=True, lo=em["lo"], hi=em["hi"])
    # Per-voxel bound of the GPU's fp32 geometry (helpers.tau_c_tie_band): a cell's C moves by
    # <= 3 2^-16 sum_27 C, its A by <= 3 2^-16 sum_27 W^T |w p e|, so X1 = X0 + alpha A / C by
    # <= alpha (dA + |A / C| dC) / C, and the regulariser spreads that over the 27-neighbourhood
    # (factor 1 + 2 alpha lambda sum_26 phi <= 1.6). At the rim of the coverage, where C is a
    # grazing sum, the bound is large: those voxels are held to it; elsewhere X is held to 1e-5.
    from scipy import ndimage
    eps = 3.0 * 2.0 ** -16
    envC = ndimage.uniform_filter(Co[box], size=3, mode="constant") * 27.0
    envA = ndimage.uniform_filter(Aabs[box], size=3, mode="constant") * 27.0
    cov = Co[box] > tau_C
    Cs = np.where(cov, Co[box], 1.0)
    dX1 = np.where(cov, prob["alpha"] * (eps * envA + np.abs(Ao[box] / Cs) * eps * envC) / Cs, 0.0)
    dX2 = 1.6 * ndimage.maximum_filter(dX1, size=3, mode="constant")
    band, near = tau_c_tie_band(Co[box], tau_C, Co[box].shape[::-1])
    flips = ((Co[box] > tau_C) != (C[box] > tau_C))
    assert not (flips & ~band).any(), "tau_C decision differs outside the fp32 tie band"
    sl = tuple(slice(i.start + 1, i.stop - 1) for i in inner)  # ROI interior (box border: no neighbours)
    dX = np.abs(X1[box][sl] - X2[sl])
    ok = ~near[sl]
    assert (dX[ok] <= dX2[sl][ok] + 1e-5 * np.abs(X2[sl][ok]) + 1e-4).all(), "X beyond its fp32 bound"
    # the rim: cells whose C is a grazing sum -- below 10% of their neighbourhood's mean C, or
    # below 1e-2 (1% of one observation's weight) -- and their 26-neighbours, where the fp32
    # geometry error of the small trilinear weights dominates
    grazing = ndimage.binary_dilation((Co[box] < 0.1 * envC / 27.0) | (Co[box] < 1e-2), np.ones((3, 3, 3), bool))
    resolved = ok & ~grazing[sl]
    rx = rel_l2(X1[box][sl][resolved], X2[sl][resolved])
    rim = int((ok & ~resolved).sum())
    record({"roi": [int(v) for v in lo], "patches": len(sel), "A": ra, "A_abs": ra_abs, "C": rc, "X": rx,
            "X_rim_voxels": rim, "X_all": rel_l2(X1[box][sl], X2[sl]), "band": int(band.sum()),
            "flips": int(flips.sum())})
    print(f"ROI {tuple(lo)}+{roi_size}: {len(sel)} patches; rel L2 A {ra:.2e} (|r|-normalised {ra_abs:.2e}) "
          f"C {rc:.2e} X {rx:.2e} over {int(resolved.sum())} resolved voxels ({rim} rim voxels within their "
          f"fp32 bound; all: {rel_l2(X1[box][sl], X2[sl]):.2e}; band {int(band.sum())}, flips {int(flips.sum())})")
    assert ra_abs <= 1e-5 and ra <= 2e-5 and rc <= 1e-5 and rx <= 1e-5, (ra_abs, ra, rc, rx)
    assert resolved.sum() >= 0.5 * resolved.size


def test_c3_forward_sampled_vs_oracle(c3):
    assert forward_sampled(c3) > 20000


@pytest.mark.parametrize("roi_lo", [(190, 190, 190), (24, 24, 24), (0, 180, 200)])
def test_c3_roi_backprojection_and_update(c3, roi_lo):
    """Centre, the corner where all three orientations' coverage ends, and a face of the volume
    (pixels partly outside the grid)."""
    roi_check(c3, roi_lo, 48)


def test_c4_forward_sampled_vs_oracle(c4):
    assert forward_sampled(c4) > 20000


def test_c4_roi_backprojection_and_update(c4):
    """c4: 3D patches, per-slab affine motion, 10% grossly misregistered patches (excluded by
    the E-step) in the ROI."""
    roi_check(c4, (150, 170, 190), 48)


def test_c5_oblique_forward_sampled_vs_oracle():
    """c5 at full size (800^3 @ 0.5 mm): the forward at the oblique stacks (30 deg about x, 45 deg
    about y) where fp32 voxel coordinates reach ~800 (SURVEY hard part 5)."""
    prob = synth.make_problem("c5")
    assert forward_sampled(prob, stacks=[6, 7], nsample=24, seed=3) > 10000


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
    obs = kap >= TAU_OBS
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
    y = patch_pixels_y(c3, pts)[kap >= TAU_OBS]
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

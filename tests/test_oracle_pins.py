"""Pin the fp64 oracle to things other than itself (closed forms, paper/SPEC hand values,
invariants, special cases that reduce to textbook routines, brute force on tiny inputs).

Each test names the passage it pins. A plausible mistake in the oracle (dropped term, wrong
sign or index, transposed operand) fails at least one of them; see DESIGN.md §Oracle pins.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle.pvro as O
import synth
from oracle import Oracle
from helpers import TAU_OBS

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------------------- PSF
def test_taylor_sinc_matches_sin_over_x():
    """P:160 Taylor series of sinc == sin(x)/x (library routine) on the PSF support [0, pi]."""
    assert O.sinc_taylor(0.0) == 1.0
    for x in np.linspace(1e-3, math.pi, 997):
        assert abs(O.sinc_taylor(x) - math.sin(x) / x) <= 1e-15
    assert abs(O.sinc_taylor(math.pi)) <= 1e-15


def test_psf_c1_worked_values():
    g = gold("psf_c1.json")
    c = g["config"]
    abc, psi, hw = O.psf_table(c["dx"], c["dy"], c["theta"], c["s"])
    assert len(psi) == g["S"]
    lat = g["lattice"]
    assert list(hw[:6]) == [lat["n_u"], lat["n_v"], lat["n_w"], lat["h_u"], lat["h_v"], lat["h_w"]]
    table = {tuple(a): v for a, v in zip(abc.tolist(), psi)}
    for item in g["values"]:
        assert abs(table[tuple(item["abc"])] - item["psi"]) <= g["tol_abs"], item
    for r in g["ratios"]:
        assert abs(table[tuple(r["num"])] / table[tuple(r["den"])] - r["value"]) <= 1e-10, r
    for a in g["absent"]:
        assert tuple(a) not in table


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_psf_normalised_nonnegative_and_sized(cfg):
    c = synth.CONFIGS[cfg]
    abc, psi, _ = O.psf_table(c["pitch"], c["pitch"], c["theta"], c["s"])
    assert abs(psi.sum() - 1.0) <= 1e-14
    assert (psi > 0).all()
    assert len(psi) == gold("patch_counts.json")["configs"][cfg]["S"]
    # symmetric under (a,b,c) -> (-a,-b,-c): the PSF has zero mean offset
    table = {tuple(a): v for a, v in zip(abc.tolist(), psi)}
    for a, v in table.items():
        assert table[(-a[0], -a[1], -a[2])] == v


# ----------------------------------------------------------------------------- patches
def test_windows_spec_example_and_clamp():
    g = gold("patch_counts.json")["spec_example"]
    w = O.windows(g["dim"], g["size"], g["stride"])
    assert len(w) == g["per_axis"] and len(w) ** 2 == g["per_slice"]
    assert list(O.windows(10, 4, 3)) == [0, 3, 6]          # 6 + 4 == 10: no clamp needed
    assert list(O.windows(11, 4, 3)) == [0, 3, 6, 7]       # last window clamped to the edge
    assert list(O.windows(32, 32, 5)) == [0]               # a = slice dim -> one patch
    for dim, size, stride in [(11, 4, 3), (256, 64, 32), (320, 32, 8), (60, 4, 4)]:
        cov = np.zeros(dim, int)
        for x in O.windows(dim, size, stride):
            cov[x:x + size] += 1
        assert cov.min() >= 1                              # every pixel covered


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_patch_counts_per_config(cfg):
    c = synth.CONFIGS[cfg]
    per = len(O.windows(c["W"], c["size"], c["stride"])) ** 2 * len(O.windows(c["K"], c["depth"], c["stride_z"]))
    assert per * len(c["stacks"]) == gold("patch_counts.json")["configs"][cfg]["M"]


# ----------------------------------------------------------------------------- forward model (Eq. 1)
def _identity_problem(n=8, psf_mode=1, stacks=("ax",), noise=0.0):
    """Stacks whose pixel grid equals the HR grid (pitch = step = s), T = I."""
    s = 1.0
    origin = np.full(3, -s * (n - 1) / 2)
    R = {"ax": synth.generate.R_AXIAL, "cor": synth.generate.R_CORONAL, "sag": synth.generate.R_SAGITTAL}
    orc = Oracle((n, n, n), s, origin)
    orc.set_param("psf_mode", psf_mode)
    rng = np.random.default_rng(7)
    Gs = []
    for tag in stacks:
        G = synth.generate.stack_G(R[tag], s, s, n, n, n, np.zeros(3))
        Gs.append(G)
        orc.add_stack(rng.normal(size=(n, n, n)).astype(np.float64), G, 1.0)
    return orc, Gs, rng


def _problem_oracle(prob, params=None):
    orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
    for k, v in (params or {}).items():
        orc.set_param(k, v)
    for st in prob["stacks"]:
        orc.add_stack(st["slices"], st["G"], st["thickness"])
    pp = prob["patch"]
    orc.extract_patches(pp["size"], pp["stride"], pp["depth"], pp["stride_z"])
    orc.set_transforms(prob["T"])
    return orc


def test_delta_psf_identity_is_textbook_resampling():
    """Special case: one PSF sample, stack grid == HR grid, T = I  =>  W = I (yhat = X)."""
    n = 8
    orc, Gs, rng = _identity_problem(n)
    orc.extract_patches(4, 2)
    orc.set_transforms(np.tile(np.eye(3, 4), (orc.M, 1, 1)))
    X = rng.normal(size=(n, n, n))
    yhat, kap = orc.forward(X)
    assert np.all(kap == 1.0)
    pt = orc.patches()
    j = 0
    for st, x0, y0, z0, sx, sy, sz in pt:
        blk = X[z0:z0 + sz, y0:y0 + sy, x0:x0 + sx].ravel()
        assert np.array_equal(yhat[j:j + blk.size], blk)
        j += blk.size


def test_constant_field_rows_sum_to_one():
    """constant X = v gives yhat = v on every observed pixel (row sums 1)."""
    prob = synth.make_problem("c3", scale=(48, 48, 6), size=16, stride=8)
    orc = _problem_oracle(prob)
    yhat, kap = orc.forward(np.full(orc.V, 437.25))
    obs = kap >= TAU_OBS
    assert obs.sum() > 1000 and (~obs).sum() > 0
    assert np.abs(yhat[obs] - 437.25).max() <= 1e-10


@pytest.mark.parametrize("q", [1.0, 2.0])
def test_linear_field_is_reproduced_at_pixel_centre(q):
    """trilinear is exact for linear fields; the PSF is symmetric (zero mean offset),
    so a fully-covered pixel sees the linear field at its transformed centre (default and the
    f4 q = 2 lattice)."""
    prob = synth.make_problem("c2", scale=(48, 24, 4))
    orc = _problem_oracle(prob, {"psf_quality": q})
    nx, ny, nz = prob["dims"]
    l, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    a, b, c, d = 0.7, -1.3, 2.1, 5.0
    yhat, kap = orc.forward(a * i + b * j + c * l + d)
    pts = orc.patches()
    k = 0
    checked = 0
    for s, (st, x0, y0, z0, sx, sy, sz) in enumerate(pts):
        G, T = prob["stacks"][st]["G"], prob["T"][s]
        for z in range(sz):
            for v in range(sy):
                for u in range(sx):
                    if kap[k] > 1 - 1e-12:
                        w = G @ np.array([x0 + u, y0 + v, z0 + z, 1.0])
                        w = T[:, :3] @ w + T[:, 3]
                        x = (w - np.asarray(prob["origin"])) / prob["spacing"]
                        assert abs(yhat[k] - (a * x[0] + b * x[1] + c * x[2] + d)) <= 1e-9
                        checked += 1
                    k += 1
    assert checked > 100


def test_integer_translation_shifts_like_the_volume():
    """Textbook: translating T by whole voxels equals index-shifting X."""
    prob = synth.make_problem("c1")
    orc = _problem_oracle(prob)
    rng = np.random.default_rng(3)
    X = rng.normal(size=prob["dims"][::-1])
    y0, k0 = orc.forward(X)
    T2 = prob["T"].copy()
    T2[:, :, 3] += np.array([2.0, -1.0, 3.0]) * prob["spacing"]   # +2 x, -1 y, +3 z voxels
    orc2 = _problem_oracle(dict(prob, T=T2))
    Xs = np.roll(np.roll(np.roll(X, 2, axis=2), -1, axis=1), 3, axis=0)
    y1, k1 = orc2.forward(Xs)
    inside = (k0 > 1 - 1e-12) & (k1 > 1 - 1e-12)          # footprint fully in the grid
    assert inside.sum() > 1000
    assert np.abs(y1[inside] - y0[inside]).max() <= 1e-9


def test_impulse_response_is_a_column_of_W():
    """X = e_k gives the k-th column of W; it is non-negative and W^T applied to the
    pixel indicator of that column reproduces sum_j W_jk^2 at voxel k."""
    prob = synth.make_problem("c1")
    orc = _problem_oracle(prob)
    k = (16 * 32 + 15) * 32 + 17
    X = np.zeros(orc.V)
    X[k] = 1.0
    col, _ = orc.forward(X)
    assert col.min() >= 0.0 and col.max() > 0.0
    back = orc.adjoint(col).ravel()
    assert abs(back[k] - (col ** 2).sum()) <= 1e-12 * (col ** 2).sum()


@pytest.mark.parametrize("cfg,kw", [("c1", {}), ("c3", dict(scale=(40, 40, 6), size=16, stride=8)),
                                    ("c4", dict(scale=(40, 40, 8), size=16, stride=8)),
                                    ("c5", dict(scale=(32, 32, 6), size=8, stride=2))])
def test_adjoint_inner_product(cfg, kw):
    """north_star / S:318: <W x, y> = <x, W^T y> to 1e-10 (fp64), random x and y."""
    prob = synth.make_problem(cfg, **kw)
    orc = _problem_oracle(prob)
    rng = np.random.default_rng(11)
    x = rng.normal(size=orc.V)
    Wx, kap = orc.forward(x)
    y = rng.normal(size=orc.P)
    y[kap < TAU_OBS] = 0.0
    WTy = orc.adjoint(y).ravel()
    lhs, rhs = float(Wx @ y), float(x @ WTy)
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), 1.0)


def test_adjoint_partitions_sum_to_whole():
    """P:233 / Q21: backprojections of disjoint patch subsets sum to the whole (multi-GPU)."""
    prob = synth.make_problem("c3", scale=(40, 40, 6), size=16, stride=8)
    orc = _problem_oracle(prob)
    rng = np.random.default_rng(5)
    r = rng.normal(size=orc.P)
    full = orc.adjoint(r)
    cut = [0, orc.M // 3, orc.M // 2, orc.M]
    parts = sum(orc.adjoint(r, a, b - a) for a, b in zip(cut[:-1], cut[1:]))
    assert np.abs(parts - full).max() <= 1e-12 * np.abs(full).max()


def test_backprojection_worked_example():
    """One voxel seen by two patches with W = 1: A = sum w p e, C = sum w p."""
    g = gold("backprojection.json")
    n = 4
    orc, Gs, _ = _identity_problem(n)
    orc.extract_patches(4, 4)                       # one 4x4 patch per slice
    orc.set_transforms(np.tile(np.eye(3, 4), (orc.M, 1, 1)))
    # two observations of voxel (1,2,0): slice 0 of the same stack added twice
    orc2 = Oracle((n, n, n), 1.0, np.full(3, -1.5))
    orc2.set_param("psf_mode", 1)
    for _ in range(2):
        orc2.add_stack(np.zeros((n, n, n)), Gs[0], 1.0)
    orc2.extract_patches(4, 4)
    orc2.set_transforms(np.tile(np.eye(3, 4), (orc2.M, 1, 1)))
    P = orc2.P
    r = np.zeros(P)
    j0 = 0 * 16 + 2 * 4 + 1          # stack 0, slice 0, row 2, col 1
    j1 = orc2.P // 2 + j0            # same pixel in stack 1
    rA = r.copy()
    rC = r.copy()
    for jj, e, p, w in zip((j0, j1), g["e"], g["p"], g["w"]):
        rA[jj] = w * p * e
        rC[jj] = w * p
    A = orc2.adjoint(rA)
    C = orc2.adjoint(rC)
    assert abs(A[0, 2, 1] - g["A"]) <= g["tol"] and abs(C[0, 2, 1] - g["C"]) <= g["tol"]
    assert abs(A[0, 2, 1] / C[0, 2, 1] - g["A_over_C"]) <= 1e-9
    assert np.count_nonzero(A) == 1 and np.count_nonzero(C) == 1


# ----------------------------------------------------------------------------- EM
def test_em_hand_values():
    g = gold("em_examples.json")
    e = np.array(g["uniform_density"]["e"])
    _, _, _, m, deg = O.em_round(e, np.ones(len(e)), np.ones(len(e)), t=1)
    assert not deg and abs(m - g["uniform_density"]["m"]) <= 1e-15
    for c in g["posterior"]:
        assert abs(O.posterior(c["e"], c["sigma2"], c["c"], c["m"]) - c["p"]) <= max(c["tol"], 0.0)
    assert O.patch_score(g["patch_score"]["p"]) == g["patch_score"]["pbar"]


def test_em_worked_example():
    w = gold("em_examples.json")["worked"]
    e = np.array(w["e"])
    live = np.ones(4)
    p, s2, c, m, deg = O.em_round(e, live, np.ones(4), t=w["t"], c0=w["c0"])
    assert not deg
    assert abs(s2 - w["sigma2"]) <= 1e-15 and c == w["c"] and abs(m - w["m"]) <= 1e-15
    assert np.abs(p - np.array(w["p"])).max() <= w["tol"]
    assert abs(O.patch_score(p) - w["pbar"]) <= w["tol"]
    _, s2b, cb, _, _ = O.em_round(e, live, p, t=2, c0=w["c0"])
    assert abs(s2b - w["next_sigma2"]) <= w["tol"] and abs(cb - w["next_c"]) <= w["tol"]


def test_posterior_is_gaussian_uniform_mixture_and_monotone():
    """P:202 in its printed form (G c / (G c + m (1-c))) equals the logistic evaluation;
    p decreases strictly in |e|."""
    s2, c, m = 2.3, 0.7, 0.05
    es = np.linspace(0, 12, 200)
    ps = [O.posterior(e, s2, c, m) for e in es]
    for e, p in zip(es, ps):
        G = math.exp(-e * e / (2 * s2)) / math.sqrt(2 * math.pi * s2)
        assert abs(p - G * c / (G * c + m * (1 - c))) <= 1e-14
        assert abs(O.posterior(-e, s2, c, m) - p) == 0.0
    assert all(a > b for a, b in zip(ps, ps[1:]))


def test_em_scale_coherence():
    """scaling all residuals by k scales sigma by k, m by 1/k; posteriors invariant."""
    rng = np.random.default_rng(2)
    e = np.concatenate([rng.normal(0, 3, 500), rng.uniform(-40, 40, 50)])
    live = np.ones(len(e))
    pp = rng.uniform(0.2, 1.0, len(e))
    p1, s1, c1, m1, _ = O.em_round(e, live, pp, t=3)
    k = 7.5
    p2, s2, c2, m2, _ = O.em_round(k * e, live, pp, t=3)
    assert abs(s2 - k * k * s1) <= 1e-12 * s2 and abs(m2 - m1 / k) <= 1e-15 and c1 == c2
    assert np.abs(p1 - p2).max() <= 1e-12


def test_em_degenerate_paths():
    """S:375 zero spread -> all inliers; S:387-388 c = 1 -> p = 1, c = 0 -> p = 0."""
    e = np.full(10, 3.0)
    p, _, _, _, deg = O.em_round(e, np.ones(10), np.ones(10), t=2)
    assert deg and np.all(p == 1.0)
    p, _, _, _, deg = O.em_round(np.arange(10.0), np.zeros(10), np.ones(10), t=2)
    assert deg                                           # no live pixel
    p, _, c, _, deg = O.em_round(np.arange(10.0), np.ones(10), np.ones(10), t=1, c0=1.0)
    assert not deg and c == 1.0 and np.all(p == 1.0)
    p, _, c, _, _ = O.em_round(np.arange(10.0), np.ones(10), np.ones(10), t=1, c0=0.0)
    assert np.all(p == 0.0)


# ----------------------------------------------------------------------------- regulariser
def test_regulariser_linear_limit_eigenvalues():
    g = gold("regulariser.json")["R1_linear_limit"]
    n = 12
    l, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    for case in g["cases"]:
        k = case["k"]
        X = np.cos(k[0] * i + k[1] * j + k[2] * l) + 0.0
        A = np.zeros_like(X)
        C = np.ones_like(X)
        _, X2 = O.update_regularise(X, A, C, 1.0, g["alpha_lambda"], math.inf)
        inner = (slice(1, -1),) * 3
        mask = np.abs(X[inner]) > 1e-3
        ratio = X2[inner][mask] / X[inner][mask]
        assert np.abs(ratio - case["factor"]).max() <= g["tol"], case


def test_regulariser_diffusivity_values():
    g = gold("regulariser.json")["R4_diffusivity"]
    delta, al = 150.0, 0.05
    for case in g["cases"]:
        dX = case["dX_over_delta"] * delta
        if case["direction"] == "axis":
            X = np.array([0.0, dX]).reshape(2, 1, 1)       # voxels (0,0,0), (0,0,1)
        else:
            X = np.zeros((2, 2, 2))
            X[1, 1, 1] = dX                                # body diagonal of voxel (0,0,0)
        _, X2 = O.update_regularise(X, np.zeros_like(X), np.ones_like(X), 1.0, al, delta)
        b = (X2.flat[0] - X.flat[0]) / (al * dX)
        assert abs(b - case["b"]) <= g["tol"], case


def test_regulariser_constant_and_max_principle():
    """R2: constant volumes are invariant for any delta. R3: for alpha*lambda <= 3/44 the
    new value lies within the [min, max] of its 27-neighbourhood."""
    X = np.full((6, 7, 8), 321.5)
    _, X2 = O.update_regularise(X, np.zeros_like(X), np.ones_like(X), 1.0, 0.05, 37.0)
    assert np.array_equal(X2, X)
    rng = np.random.default_rng(9)
    X = rng.uniform(0, 1000, size=(10, 11, 12))
    al = gold("regulariser.json")["max_principle_alpha_lambda"]
    _, X2 = O.update_regularise(X, np.zeros_like(X), np.ones_like(X), 1.0, al, 50.0)
    from numpy.lib.stride_tricks import sliding_window_view as sw
    pad = np.pad(X, 1, mode="edge")
    lo = sw(pad, (3, 3, 3)).min(axis=(-1, -2, -3))
    hi = sw(pad, (3, 3, 3)).max(axis=(-1, -2, -3))
    assert (X2 >= lo - 1e-9).all() and (X2 <= hi + 1e-9).all()


def test_update_special_cases():
    """alpha = 0, or C <= tau_C, leaves X unchanged; the clamp bounds the step (Q19)."""
    rng = np.random.default_rng(4)
    X = rng.uniform(0, 100, size=(5, 6, 7))
    A = rng.normal(size=X.shape) * 50
    C = rng.uniform(0.1, 2, size=X.shape)
    X1, X2 = O.update_regularise(X, A, C, 0.0, 0.0, 150.0)
    assert np.array_equal(X1, X) and np.array_equal(X2, X)
    X1, X2 = O.update_regularise(X, A, np.zeros_like(C), 1.0, 0.02, 150.0)
    assert np.array_equal(X2, X)
    X1, _ = O.update_regularise(X, A, C, 1.0, 0.0, 150.0, clamp=True, lo=10.0, hi=60.0)
    changed = C > 1e-6
    assert (X1[changed] >= 10.0).all() and (X1[changed] <= 60.0).all()
    free, _ = O.update_regularise(X, A, C, 1.0, 0.0, 150.0)
    assert np.allclose(free, X + A / C, rtol=0, atol=1e-12)


# ----------------------------------------------------------------------------- whole iteration
def test_fixed_point_inverse_crime():
    """Motion-free c1 with y = W X* exactly (fp64), start at X*, lambda = 0, clamp off:
    X stays X* (zero residual takes the zero-spread EM path, p = 1)."""
    prob = synth.make_problem("c1")
    Xs = synth.rasterize_phantom(prob)
    base = _problem_oracle(prob)
    yhat, kap = base.forward(Xs)
    # write W X* back into fp64 stacks (patches of one slice share T = I, so any copy works)
    stacks = [np.zeros(st["slices"].shape) for st in prob["stacks"]]
    j = 0
    for st, x0, y0, z0, sx, sy, sz in base.patches():
        blk = yhat[j:j + sx * sy * sz].reshape(sz, sy, sx)
        stacks[st][z0:z0 + sz, y0:y0 + sy, x0:x0 + sx] = blk
        j += sx * sy * sz
    orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
    orc.set_param("clamp", 0)
    for arr, st in zip(stacks, prob["stacks"]):
        orc.add_stack(arr, st["G"], st["thickness"])
    orc.extract_patches(16, 8)
    orc.set_transforms(prob["T"])
    orc.set_volume(Xs)
    orc.sr_iterate(2, 1.0, 0.0)
    assert np.abs(orc.volume() - Xs).max() <= 1e-12 * np.abs(Xs).max()
    p, _, w = orc.weights()
    assert np.all(p[kap >= TAU_OBS] == 1.0)


def test_delta_psf_one_iteration_recovers_data():
    """W = I (delta PSF, identity grids, T = I), three orthogonal stacks of consistent data,
    alpha = 1, lambda = 0, tau_patch = 0: one iteration from any X0 gives X = y exactly."""
    n = 8
    s = 1.0
    rng = np.random.default_rng(21)
    Xtrue = rng.uniform(100, 900, size=(n, n, n))
    orc = Oracle((n, n, n), s, np.full(3, -(n - 1) / 2))
    orc.set_param("psf_mode", 1)
    orc.set_param("tau_patch", 0.0)
    orc.set_param("clamp", 0)
    R = [synth.generate.R_AXIAL, synth.generate.R_CORONAL, synth.generate.R_SAGITTAL]
    for Rm in R:
        G = synth.generate.stack_G(Rm, s, s, n, n, n, np.zeros(3))
        # the stack's slices are X sampled on its own (permuted) grid
        k, v, u = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
        w = np.einsum("ij,jklm->iklm", G[:, :3], np.stack([u, v, k])) + G[:, 3][:, None, None, None]
        idx = np.rint((w - orc_origin(n)[:, None, None, None]) / s).astype(int)
        orc.add_stack(Xtrue[idx[2], idx[1], idx[0]], G, 1.0)
    orc.extract_patches(4, 2)
    orc.set_transforms(np.tile(np.eye(3, 4), (orc.M, 1, 1)))
    orc.set_volume(rng.uniform(0, 50, size=(n, n, n)))
    orc.sr_iterate(1, 1.0, 0.0)
    assert np.abs(orc.volume() - Xtrue).max() <= 1e-9
    orc.init_volume()                                  # init: X = W^T y / W^T 1 = y
    assert np.abs(orc.volume() - Xtrue).max() <= 1e-9


def orc_origin(n):
    return np.full(3, -(n - 1) / 2)


def test_zero_weights_leave_volume_unchanged():
    """all p = 0 (c0 = 0 at t = 1) leaves X unchanged."""
    prob = synth.make_problem("c1")
    orc = _problem_oracle(prob, {"c0": 0.0})
    orc.init_volume()
    X0 = orc.volume()
    orc.sr_iterate(1, 1.0, 0.02)
    assert np.array_equal(orc.volume(), X0)


# ------------------------------------------------- f2 rigidity map (reading Q28)
@pytest.fixture(scope="module")
def c1_oracle():
    import helpers
    prob = synth.make_problem("c1")
    return prob, helpers.make_oracle(prob)


def test_rigidity_map_all_posteriors_one_is_one_on_observed_voxels(c1_oracle):
    """SPEC rigidity_map example 'all posteriors 1 -> map = 1 on observed voxels': right after
    set_transforms p = pbar = 1, so W^T(p pbar) = W^T 1 and the ratio is exactly 1 wherever
    W^T 1 > tau_C (0 elsewhere)."""
    _, orc = c1_oracle
    orc.set_weights(np.ones(orc.P), np.ones(orc.M))
    R = orc.rigidity_map()
    on = R != 0.0
    assert on.mean() > 0.5                      # c1: most of the grid is observed
    assert np.abs(R[on] - 1.0).max() <= 1e-12


def test_rigidity_map_zero_and_uniform_posteriors(c1_oracle):
    """SPEC example 'all posteriors 0 -> map = 0'; and p = 0.3 everywhere, pbar = sqrt(mean
    p^2) = 0.3 (Eq. P:206) gives the closed form p pbar = 0.09 on every observed voxel."""
    _, orc = c1_oracle
    orc.set_weights(np.zeros(orc.P), np.zeros(orc.M))
    assert np.abs(orc.rigidity_map()).max() == 0.0
    orc.set_weights(np.full(orc.P, 0.3), np.full(orc.M, 0.3))
    R = orc.rigidity_map()
    on = R != 0.0
    assert on.mean() > 0.5 and np.abs(R[on] - 0.09).max() <= 1e-12


def test_rigidity_map_single_contributor_patch_scaling(c1_oracle):
    """Linearity in pbar: scaling one patch's pbar by k scales its numerator share; a voxel
    seen by that patch alone takes p pbar of that patch (weighted mean of one term)."""
    _, orc = c1_oracle
    rng = np.random.default_rng(7)
    p = rng.uniform(0.2, 1.0, orc.P)
    pb = rng.uniform(0.2, 1.0, orc.M)
    orc.set_weights(p, pb)
    R1 = orc.rigidity_map()
    orc.set_weights(p, 2.0 * pb)
    R2 = orc.rigidity_map()
    on = R1 != 0.0
    assert np.abs(R2[on] - 2.0 * R1[on]).max() <= 1e-12 * max(1.0, np.abs(R2).max())
    assert (R1 >= 0).all() and (R1 <= 1.0 + 1e-12).all()


def test_rigidity_map_marks_corrupted_patches():
    """SPEC rigidity_map example (region-mean comparison): in a c4-structured problem with 10%
    gross transform errors, after EM the map is lower where corrupted patches dominate the
    coverage than where only consistent patches contribute (pbar of corrupted patches ~0.55
    vs ~0.98 here)."""
    import helpers
    prob = synth.make_problem("c4", scale=(48, 48, 12), size=16, stride=8)
    orc = helpers.make_oracle(prob)
    orc.init_volume()
    orc.sr_iterate(2, prob["alpha"], prob["lam"])
    R = orc.rigidity_map().ravel()
    assert (R >= 0).all() and (R <= 1.0 + 1e-12).all()
    bad = np.asarray(prob["corrupted"], bool)
    assert bad.any() and not bad.all()
    pix0 = np.concatenate([[0], np.cumsum([np.prod(p[4:7]) for p in orc.patches()])]).astype(np.int64)
    ind = np.zeros(orc.P)
    for s in np.flatnonzero(bad):
        ind[pix0[s]:pix0[s + 1]] = 1.0
    den_bad = orc.adjoint(ind).ravel()
    den_all = orc.adjoint(np.ones(orc.P)).ravel()
    obs = den_all > 1e-3
    # corrupted patches are 10% of an overlapping set: voxels where they carry > 15% of the
    # coverage vs voxels they never reach
    B = obs & (den_bad > 0.15 * den_all)
    G = obs & (den_bad == 0.0)
    assert B.sum() > 10 and G.sum() > 10
    assert R[B].mean() < R[G].mean() - 0.03


# ------------------------------------------------------ f4 q = 2 PSF quality mode (Q5)
@pytest.mark.parametrize("cfg,S", [("c1", 99), ("c2", 189), ("c3", 1305), ("c4", 1305), ("c5", 2829)])
def test_psf_quality_two_lattice(cfg, S):
    """n_u = max(2, ceil(2 pitch / s)), n_w = max(2, ceil(2 theta / s)); c3:
    S = 45 x 29 = 1305 (SURVEY calc). The table stays normalised, positive and symmetric, and
    q = 1 reproduces the default table exactly."""
    c = synth.CONFIGS[cfg]
    abc, psi, hw = O.psf_table(c["pitch"], c["pitch"], c["theta"], c["s"], q=2.0)
    assert len(psi) == S
    assert list(hw[:3]) == [max(2, math.ceil(2 * c["pitch"] / c["s"] - 1e-9))] * 2 + \
        [max(2, math.ceil(2 * c["theta"] / c["s"] - 1e-9))]
    assert abs(psi.sum() - 1.0) <= 1e-14 and (psi > 0).all()
    table = {tuple(a): v for a, v in zip(abc.tolist(), psi)}
    for a, v in table.items():
        assert abs(table[(-a[0], -a[1], -a[2])] - v) <= 1e-15
    a1, p1, h1 = O.psf_table(c["pitch"], c["pitch"], c["theta"], c["s"])
    a2, p2, h2 = O.psf_table(c["pitch"], c["pitch"], c["theta"], c["s"], q=1.0)
    assert np.array_equal(a1, a2) and np.array_equal(p1, p2)


# ------------------------------------------------------ f4 multi-round EM (Q30)
def test_em_loglik_is_the_mixture_density():
    """LL = sum_live log(c N(e; 0, sigma^2) + (1 - c) m) == scipy.stats.norm."""
    from scipy.stats import norm
    rng = np.random.default_rng(2)
    e = rng.normal(0, 4, 500)
    live = rng.uniform(size=500) > 0.2
    want = np.log(0.8 * norm.pdf(e[live], 0, 3.0) + 0.2 * 0.01).sum()
    assert abs(O.em_loglik(e, live, 9.0, 0.8, 0.01) - want) <= 1e-9 * abs(want)


def test_em_rounds_monotone_consistent_and_spec_examples():
    """S:420 invariant: the EM log-likelihood never decreases across rounds; S:404 example:
    pure zero-mean Gaussian residuals -> c >= 0.95; a 90/10 Gaussian/uniform mixture recovers
    c and sigma^2 (consistency of the mixture MLE); rounds = 1 is exactly pvro_em_round."""
    rng = np.random.default_rng(0)
    e = rng.normal(0, 3, 20000)
    e[:2000] = rng.uniform(-60, 60, 2000)
    one = np.ones(len(e))
    p, s2, c, m, ll = O.em_rounds(e, one, one, 1, 20)
    assert len(ll) >= 3 and (np.diff(ll) >= -1e-9 * np.abs(ll[:-1])).all()
    assert abs(c - 0.9) <= 0.01 and abs(s2 - 9.0) <= 0.3
    p1, s21, c1, m1, _ = O.em_round(e, one, one, 1)
    pr, s2r, cr, mr, llr = O.em_rounds(e, one, one, 1, 1)
    assert np.array_equal(pr, p1) and (s2r, cr, mr) == (s21, c1, m1) and len(llr) == 1
    g = rng.normal(0, 3, 20000)
    _, _, cg, _, _ = O.em_rounds(g, one, one, 1, 20)
    assert cg >= 0.95
    # degenerate (zero spread): a single round, p = 1
    pd, _, _, _, lld = O.em_rounds(np.full(100, 2.0), np.ones(100), np.ones(100), 1, 20)
    assert len(lld) == 1 and (pd == 1.0).all()


# ------------------------------------------- f4 two-Gaussian patch classification (Q31)
def test_patch_mixture_matches_sklearn_and_separates():
    """P:209 'an inlier and outlier probability for each y_s': the two-Gaussian mixture on
    pbar fitted by EM equals scikit-learn's GaussianMixture (library routine) started from the
    same parameters, and separates a 90/10 mixture of good / corrupted patch scores."""
    from sklearn.mixture import GaussianMixture
    rng = np.random.default_rng(0)
    pb = np.r_[rng.normal(0.95, 0.02, 900), rng.normal(0.4, 0.08, 100)].clip(0, 1)
    r, n = O.patch_mixture(pb, rounds=500, tol=1e-12)
    assert (r[:900] >= 0.5).mean() >= 0.99 and (r[900:] < 0.5).mean() >= 0.99
    var = pb.var()
    gm = GaussianMixture(2, covariance_type="full", tol=1e-12, max_iter=2000, reg_covar=0.0,
                         weights_init=[0.5, 0.5], means_init=[[pb.max()], [pb.min()]],
                         precisions_init=[[[1 / var]], [[1 / var]]]).fit(pb[:, None])
    assert np.abs(gm.predict_proba(pb[:, None])[:, 0] - r).max() <= 1e-4


def test_patch_mixture_degenerate_and_invalid():
    """Equal scores: every valid patch is an inlier (r = 1); invalid patches (no live pixel)
    get r = 0 and do not enter the fit."""
    r, _ = O.patch_mixture(np.full(10, 0.8), np.r_[np.ones(8), np.zeros(2)])
    assert (r[:8] == 1.0).all() and (r[8:] == 0.0).all()
    rng = np.random.default_rng(1)
    pb = np.r_[rng.normal(0.9, 0.03, 50), rng.normal(0.3, 0.05, 10), [0.99, 0.01]]
    valid = np.r_[np.ones(60), [0, 0]]
    r1, _ = O.patch_mixture(pb, valid)
    r2, _ = O.patch_mixture(pb[:60])
    assert np.array_equal(r1[:60], r2) and (r1[60:] == 0).all()


def test_patch_mixture_excludes_corrupted_patches():
    """S:401 example (10% of patches under gross transform errors, c4 structure, two SR
    iterations): the mixture labels most corrupted patches outliers (w = 0) -- here 86%, more
    than twice the threshold rule's 36% -- with <= 5% false exclusions."""
    import helpers
    prob = synth.make_problem("c4", scale=(48, 48, 12), size=16, stride=8)
    bad = np.asarray(prob["corrupted"], bool)
    out = {}
    for mix in (0, 1):
        orc = helpers.make_oracle(prob, {"patch_mixture": mix})
        orc.init_volume()
        orc.sr_iterate(2, prob["alpha"], prob["lam"])
        _, _, w = orc.weights()
        out[mix] = ((w[bad] == 0).mean(), (w[~bad] == 0).mean())
    assert out[1][0] >= 0.8 and out[1][0] >= 2 * out[0][0] and out[1][1] <= 0.05, out


# ------------------------------------------------------- f3 explicit / masked patches (Q32)
def _c1_with(rects=None, mask=None, **kw):
    prob = synth.make_problem("c1")
    orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
    for st in prob["stacks"]:
        orc.add_stack(st["slices"], st["G"], st["thickness"])
    return prob, orc


def test_set_patches_without_mask_equals_extract():
    """Explicit rectangles equal to the square windows reproduce extract_patches exactly."""
    prob, a = _c1_with()
    a.extract_patches(16, 8)
    a.set_transforms(prob["T"])
    rects = a.patches()
    _, b = _c1_with()
    b.set_patches(rects)
    b.set_transforms(prob["T"])
    for o in (a, b):
        o.init_volume()
        o.sr_iterate(1, prob["alpha"], prob["lam"])
    # equal up to the order of the oracle's OpenMP atomic fp64 sums
    assert np.abs(a.volume() - b.volume()).max() <= 1e-12 * np.abs(a.volume()).max()


def test_masked_pixels_are_not_observations_and_adjoint_is_additive():
    """Masked-out pixels get kappa = 0 (never observed); the rest keep their coverage; and the
    backprojection of a masked patch equals that of its kept pixels as 1x1 patches (W^T is a
    sum over observations)."""
    prob, a = _c1_with()
    rects = np.array([[0, 4, 6, 3, 12, 10, 1], [1, 0, 0, 2, 16, 16, 1]], np.int32)
    rng = np.random.default_rng(4)
    mask = (rng.uniform(size=12 * 10 + 256) > 0.4).astype(np.uint8)
    a.set_patches(rects, mask)
    T = np.tile(np.hstack([np.eye(3), np.zeros((3, 1))]), (2, 1, 1))
    a.set_transforms(T)
    _, b = _c1_with()
    b.set_patches(rects)
    b.set_transforms(T)
    _, ka, _, _ = a.taps()
    _, kb, _, _ = b.taps()
    assert (ka[mask == 0] == 0).all() and np.array_equal(ka[mask == 1], kb[mask == 1])
    # single-pixel patches of the kept pixels
    singles = []
    j = 0
    for r in rects:
        for z in range(r[6]):
            for v in range(r[5]):
                for u in range(r[4]):
                    if mask[j]:
                        singles.append([r[0], r[1] + u, r[2] + v, r[3] + z, 1, 1, 1])
                    j += 1
    _, c = _c1_with()
    c.set_patches(np.array(singles, np.int32))
    c.set_transforms(np.tile(np.hstack([np.eye(3), np.zeros((3, 1))]), (len(singles), 1, 1)))
    y = rng.uniform(0, 10, len(mask))
    Aa = a.adjoint(y)
    Ac = c.adjoint(y[mask == 1])
    assert np.abs(Aa - Ac).max() <= 1e-12 * max(1.0, np.abs(Aa).max())


# ------------------------------------------------------------ f3 superpixels (SLIC, Q33)
def test_slic_partition_locality_and_boundary_adherence():
    """SLIC (Eq. 3): labels partition the slice; every pixel's cluster is one of the
    3x3 grid cells around it (SLIC's 2S x 2S search window); on a two-region image with a
    small compactness m no superpixel straddles the intensity edge (boundary adherence)."""
    rng = np.random.default_rng(3)
    img = rng.normal(500, 30, (48, 64)).astype(np.float32)
    lab, nc = O.slic(img, 8, 10, 10)
    assert nc == 6 * 8 and lab.min() >= 0 and lab.max() < nc
    yy, xx = np.mgrid[0:48, 0:64]
    ci, cj = lab % 8, lab // 8
    assert (np.abs(ci - xx // 8) <= 1).all() and (np.abs(cj - yy // 8) <= 1).all()
    two = np.where(xx < 29, 100.0, 900.0).astype(np.float32) + rng.normal(0, 5, (48, 64)).astype(np.float32)
    lab2, _ = O.slic(two, 8, 1, 10)
    for k in np.unique(lab2):
        side = xx[lab2 == k] < 29
        assert side.all() or (~side).all(), k


def test_superpixel_patch_masks_are_dilated_superpixels():
    """Superpixel patches: with gamma = 0 the masks partition every slice (each pixel
    in exactly one patch) and each rectangle is its superpixel's bounding box; with gamma > 0
    each mask is exactly the superpixel dilated by a (2 gamma + 1)^2 square, clipped to the
    slice (scipy.ndimage.binary_dilation, a library routine)."""
    from scipy import ndimage
    prob = synth.make_problem("c1")
    S, m, it = 8, 10, 5
    for gamma in (0, 2):
        orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
        for st in prob["stacks"]:
            orc.add_stack(st["slices"], st["G"], st["thickness"])
        orc.superpixel_patches(S, m, it, gamma)
        rects, mask = orc.patches(), orc.mask()
        offs = np.concatenate([[0], np.cumsum(rects[:, 4] * rects[:, 5] * rects[:, 6])])
        for si, st in enumerate(prob["stacks"]):
            vol = st["slices"]
            K, H, W = vol.shape
            lo, hi = float(vol.min()), float(vol.max())
            count = np.zeros((K, H, W), np.int32)
            for z in range(K):
                lab, nc = O.slic(vol[z], S, m, it, lo, hi)
                mine = np.flatnonzero((rects[:, 0] == si) & (rects[:, 3] == z))
                ks = [k for k in range(nc) if (lab == k).any()]
                assert len(mine) == len(ks)
                for s_, k in zip(mine, ks):
                    r = rects[s_]
                    got = mask[offs[s_]:offs[s_ + 1]].reshape(r[5], r[4]).astype(bool)
                    want = ndimage.binary_dilation(lab == k, np.ones((2 * gamma + 1,) * 2, bool)) if gamma else lab == k
                    ys, xs = np.nonzero(want)
                    assert (r[1], r[2], r[4], r[5]) == (xs.min(), ys.min(), xs.max() - xs.min() + 1, ys.max() - ys.min() + 1)
                    assert np.array_equal(got, want[r[2]:r[2] + r[5], r[1]:r[1] + r[4]])
                    count[z, r[2]:r[2] + r[5], r[1]:r[1] + r[4]] += got
            if gamma == 0:
                assert (count == 1).all()

"""Edge cases of the hot path against the oracle (same bars as tests/test_gpu_parity.py):
degenerate patch shapes through pvr_set_patches (one patch, single pixels, single rows and
columns, a whole slice that the planner must subdivide), every patch excluded by tau_patch
(C = 0: the update keeps X), alpha = 0, and an empty mask. Each case runs at the default
thresholds (tau_C = 1e-6, tau_obs = 0.01)."""
import numpy as np
import pytest

import synth
from helpers import TOL, rel_l2
from test_gpu_parity import check_iteration

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def prob():
    return synth.make_problem("c3", scale=(64, 64, 8), size=32, stride=16)


def _pair(prob, rects, mask=None, params=None):
    from oracle import Oracle
    from paper_1611_07289_b200 import Context
    orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
    ctx = Context(prob["dims"], prob["spacing"], prob["origin"])
    for k, v in (params or {}).items():
        orc.set_param(k, v)
        ctx.set_param(k, v)
    for st in prob["stacks"]:
        orc.add_stack(st["slices"], st["G"], st["thickness"])
        ctx.add_stack(st["slices"], st["G"], st["thickness"])
    rects = np.asarray(rects, np.int32)
    orc.set_patches(rects, mask)
    ctx.set_patches(rects, mask)
    T = np.tile(np.hstack([np.eye(3), np.zeros((3, 1))]), (len(rects), 1, 1))
    orc.set_transforms(T)
    ctx.set_transforms(T)
    return orc, ctx


def _run(prob, rects, mask=None, params=None, iters=2, alpha=None, X0=None):
    orc, ctx = _pair(prob, rects, mask, params)
    try:
        _, ko, _, _ = orc.taps()
        _, kg, _, _ = ctx.taps()
        assert np.abs(kg - ko).max() <= TOL["kappa"]
        if X0 is None:
            orc.init_volume()
            ctx.init_volume()
        else:
            orc.set_volume(X0)
            ctx.set_volume(np.ascontiguousarray(X0, np.float32))
        assert rel_l2(ctx.volume(), orc.volume()) <= TOL["X"]
        a = prob["alpha"] if alpha is None else alpha
        for it in range(iters):
            orc.sr_iterate(1, a, prob["lam"])
            ctx.sr_iterate(1, a, prob["lam"])
            check_iteration(ctx, orc, prob, params, it)
        return orc, ctx
    except BaseException:
        ctx.close()
        raise


def _centre_rect(prob, st, sx, sy, z=None):
    K, H, W = prob["stacks"][st]["slices"].shape
    return [st, (W - sx) // 2, (H - sy) // 2, K // 2 if z is None else z, sx, sy, 1]


def test_single_patch(prob):
    """M = 1: one 16x16 patch (one group, one shard)."""
    _, ctx = _run(prob, [_centre_rect(prob, 0, 16, 16)])
    assert ctx.M == 1
    ctx.close()


def test_single_pixel_patches(prob):
    """200 patches of one pixel each (members of one pixel; every cell a rim cell). Started
    from a constant volume: from the initial backprojection each isolated pixel would be
    reproduced almost exactly, and e = y - yhat would be pure rounding on both sides."""
    rng = np.random.default_rng(3)
    rects = []
    for _ in range(200):
        st = int(rng.integers(0, len(prob["stacks"])))
        K, H, W = prob["stacks"][st]["slices"].shape
        rects.append([st, int(rng.integers(0, W)), int(rng.integers(0, H)), int(rng.integers(0, K)), 1, 1, 1])
    X0 = np.full(prob["dims"][::-1], float(np.mean(prob["stacks"][0]["slices"])))
    _run(prob, rects, X0=X0)[1].close()


def test_row_and_column_patches(prob):
    """Patches one pixel high or one pixel wide, across whole slices."""
    rects = []
    for st, s in enumerate(prob["stacks"]):
        K, H, W = s["slices"].shape
        for z in range(0, K, 3):
            rects.append([st, 0, H // 3, z, W, 1, 1])
            rects.append([st, W // 2, 0, z, 1, H, 1])
    _run(prob, rects)[1].close()


def test_whole_slice_patches(prob):
    """One patch per slice covering the whole slice: larger than any tile, so the planner
    subdivides each member (engine.cu size_groups: emit_single)."""
    rects = []
    for st, s in enumerate(prob["stacks"]):
        K, H, W = s["slices"].shape
        rects += [[st, 0, 0, z, W, H, 1] for z in range(K)]
    _, ctx = _run(prob, rects)
    st = ctx.stats()
    print("whole-slice plan:", {k: st[k] for k in ("bp_tile", "bp_groups", "bp_members", "bp_split", "fwd_split")})
    ctx.close()


def test_every_patch_excluded(prob):
    """tau_patch above any pbar (<= 1): every w = 0, so A = C = 0 and the update keeps X
    (the regulariser acts only where C > tau_C, P:185 / reading Q16)."""
    rects = [_centre_rect(prob, st, 24, 24, z) for st in range(len(prob["stacks"])) for z in (2, 5)]
    orc, ctx = _pair(prob, rects, params={"tau_patch": 1.5})
    try:
        orc.init_volume()
        ctx.init_volume()
        X0g, X0o = ctx.volume().copy(), orc.volume().copy()
        orc.sr_iterate(1, prob["alpha"], prob["lam"])
        ctx.sr_iterate(1, prob["alpha"], prob["lam"])
        _, _, w = ctx.weights()
        assert (w == 0).all() and (orc.weights()[2] == 0).all()
        _, _, A, C = ctx.taps()
        assert not A.any() and not C.any()
        assert np.array_equal(ctx.volume(), X0g)
        assert np.array_equal(orc.volume(), X0o)
    finally:
        ctx.close()


def test_zero_step_keeps_the_volume(prob):
    """alpha = 0: X^{n+1} = X^n exactly on both sides while p, w, sigma^2 still follow."""
    rects = [_centre_rect(prob, st, 32, 32, z) for st in range(len(prob["stacks"])) for z in range(1, 7, 2)]
    orc, ctx = _pair(prob, rects)
    try:
        orc.init_volume()
        ctx.init_volume()
        X0 = ctx.volume().copy()
        for it in range(2):
            orc.sr_iterate(1, 0.0, prob["lam"])
            ctx.sr_iterate(1, 0.0, prob["lam"])
            assert np.array_equal(ctx.volume(), X0)
            check_iteration(ctx, orc, prob, None, it)
    finally:
        ctx.close()


def test_all_pixels_masked(prob):
    """A mask that hides every pixel: nothing observed, set_transforms reports PVR_ERR_EMPTY
    (S:336 'nothing to reconstruct') on the product as on the oracle's reading."""
    from paper_1611_07289_b200 import Context, pvr
    rects = np.array([_centre_rect(prob, 0, 8, 8)], np.int32)
    ctx = Context(prob["dims"], prob["spacing"], prob["origin"])
    try:
        for st in prob["stacks"]:
            ctx.add_stack(st["slices"], st["G"], st["thickness"])
        ctx.set_patches(rects, np.zeros(64, np.uint8))
        T = np.tile(np.hstack([np.eye(3), np.zeros((3, 1))]), (1, 1, 1))
        with pytest.raises(pvr.PvrError) as ei:
            ctx.set_transforms(T)
        assert ei.value.status == pvr.PVR_ERR_EMPTY
    finally:
        ctx.close()

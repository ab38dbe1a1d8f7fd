"""f3 superpixel patches on the GPU (pvr_superpixels / pvr_superpixel_patches) against the
oracle (pvro_slic / pvro_superpixel_patches). SURVEY §8(f) f3; Eq. 3; P:154;
DESIGN.md readings Q32, Q33.

SLIC runs in integer arithmetic on both sides, so labels, rectangles and masks must be
bit-identical; the SR iterations on the resulting patches keep the parity bar."""
import numpy as np
import pytest

import synth
from helpers import rel_l2, weight_mismatch
from oracle import Oracle
import oracle.pvro as O
from paper_1611_07289_b200 import Context

pytestmark = pytest.mark.gpu


def both(prob):
    orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
    ctx = Context(prob["dims"], prob["spacing"], prob["origin"])
    for st in prob["stacks"]:
        orc.add_stack(st["slices"], st["G"], st["thickness"])
        ctx.add_stack(st["slices"], st["G"], st["thickness"])
    return orc, ctx


@pytest.mark.parametrize("cfg,kw,S,m", [("c1", {}, 8, 10), ("c3", dict(scale=(96, 96, 12), size=32, stride=16), 16, 20)])
def test_slic_labels_bit_exact(cfg, kw, S, m):
    prob = synth.make_problem(cfg, **kw)
    orc, ctx = both(prob)
    try:
        for si, st in enumerate(prob["stacks"]):
            vol = st["slices"]
            lab = ctx.superpixels(si, S, m, 10, vol.shape)
            lo, hi = float(vol.min()), float(vol.max())
            for z in range(vol.shape[0]):
                want, _ = O.slic(vol[z], S, m, 10, lo, hi)
                assert np.array_equal(lab[z], want), (si, z)
    finally:
        ctx.close()


def test_superpixel_patches_identical_and_sr_parity():
    prob = synth.make_problem("c3", scale=(96, 96, 12), size=32, stride=16)
    orc, ctx = both(prob)
    try:
        Mo = orc.superpixel_patches(16, 20, 10, 3)
        Mg = ctx.superpixel_patches(16, 20, 10, 3)
        assert Mo == Mg
        assert np.array_equal(ctx.patches(), orc.patches())
        assert np.array_equal(ctx.mask(), orc.mask())
        T = np.tile(np.hstack([np.eye(3), np.zeros((3, 1))]), (Mo, 1, 1))
        orc.set_transforms(T)
        ctx.set_transforms(T)
        orc.init_volume()
        ctx.init_volume()
        assert rel_l2(ctx.volume(), orc.volume()) <= 1e-5
        for it in range(2):
            orc.sr_iterate(1, prob["alpha"], prob["lam"])
            ctx.sr_iterate(1, prob["alpha"], prob["lam"])
            assert rel_l2(ctx.volume(), orc.volume()) <= 1e-4
            po, pbo, wo = orc.weights()
            pg, pbg, wg = ctx.weights()
            dp, dw, _ = weight_mismatch(pg, po, pbg, pbo, wg, wo)
            assert dp <= 1e-3 and dw <= 1e-3
    finally:
        ctx.close()


def test_multiscale_reextraction():
    """f3 multi-scale schedule (different patch scales per iteration): one context
    re-extracts superpixel patches at a finer scale between iterations, keeping X; both sides
    follow the same schedule within the parity bar."""
    prob = synth.make_problem("c3", scale=(96, 96, 12), size=32, stride=16)
    orc, ctx = both(prob)
    try:
        for i, (S, gamma) in enumerate([(24, 4), (12, 2)]):
            Mo = orc.superpixel_patches(S, 20, 10, gamma)
            Mg = ctx.superpixel_patches(S, 20, 10, gamma)
            assert Mo == Mg and np.array_equal(ctx.patches(), orc.patches())
            T = np.tile(np.hstack([np.eye(3), np.zeros((3, 1))]), (Mo, 1, 1))
            orc.set_transforms(T)
            ctx.set_transforms(T)
            if i == 0:
                orc.init_volume()
                ctx.init_volume()
            orc.sr_iterate(1, prob["alpha"], prob["lam"])
            ctx.sr_iterate(1, prob["alpha"], prob["lam"])
            assert rel_l2(ctx.volume(), orc.volume()) <= 1e-4, (S, rel_l2(ctx.volume(), orc.volume()))
    finally:
        ctx.close()

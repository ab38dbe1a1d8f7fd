"""Shared test helpers: build the oracle and the GPU context on the same seeded problem."""
import os

import numpy as np

# errors measured by the parity checks, dumped by conftest.py to $PVR_PARITY_LOG (JSON)
ERRORS = []


def record(err):
    ERRORS.append({"test": os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], **err})

# Threshold sets (readings Q24 / Q25). DEFAULTS are both sides' defaults: tau_C = 1e-6
# (SURVEY.md:678) and observed iff kappa >= 0.01 (SURVEY.md:652 "kappa > 0" with a floor);
# ROUND1 are the round-1 readings tau_C = 1e-3, tau_obs = 0.5, kept as a second parity set.
TAU_OBS = 0.01
THRESHOLDS = {"survey": {}, "round1": {"tau_C": 1e-3, "tau_obs": 0.5}}

# Stage tolerances: 10x the largest error measured on the B200 over every parity
# test (c1, c2, c3/c4/c5-shaped, odd shapes, q = 2, multi-round EM, patch mixture, explicit
# masked patches, re-planned transforms; both threshold sets), rounded up -- measured maxima
# (profiles/r02_parity_errors.txt): X 4.2e-7, e 1.2e-6, A 9.5e-6, C 8.9e-7 (rel L2; X away
# from the tau_C tie band), kappa 1.6e-6, p 1.4e-5, w 1.3e-6 (abs), sigma2 / c / m 2.4e-7 (rel).
# The north_star bars (X 1e-4 rel L2, p and w 1e-3 abs) are asserted as well.
# m = 1 / (max e - min e) is a ratio of two extreme residuals, each off by up to ~1e-6 of its
# pixel's yhat, so its relative error scales with max|yhat| / range(e) (~5 on these phantoms):
# the EM bar is 1e-5 rather than 10x the lattice mode's 2.4e-7 (volume-space PSF mode: 4.3e-6).
TOL = {"X": 5e-6, "e": 1.2e-5, "A": 1e-4, "C": 9e-6, "kappa": 1.7e-5, "p": 1.4e-4, "w": 1.3e-5, "em": 1e-5}


def tau_c_tie_band(Co, tau_C, dims):
    """Voxels whose oracle confidence sits within fp32 reach of tau_C.

    The GPU forms each trilinear weight from fp32 positions: offsets of < 2^6 voxels from an
    fp64 member origin, a handful of roundings of <= 2^-18 voxel each, so <= 2^-16 voxel per
    axis and <= 3 2^-16 on a product of three tents. A cell's C = sum (psi w p / kappa) t then
    moves by <= 3 2^-16 sum_{samples in reach} psi w p / kappa, and that sum is bounded by the
    C of the cell's 27-neighbourhood (each sample's 8 corner weights sum to 1). Band:
    |C_k - tau_C| <= 3 2^-16 sum_27 C. Returns (band mask, band dilated by the 26-neighbours
    the regulariser couples)."""
    from scipy import ndimage
    C = np.asarray(Co, np.float64).reshape(tuple(dims)[::-1])
    env = ndimage.uniform_filter(C, size=3, mode="constant") * 27.0
    near = np.abs(C - tau_C) <= 3.0 * 2.0 ** -16 * env
    return near, ndimage.binary_dilation(near, np.ones((3, 3, 3), bool))


def make_oracle(prob, params=None):
    from oracle import Oracle
    orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
    for k, v in (params or {}).items():
        if k not in ("profile", "bp_exact", "deterministic", "exchange", "comm_timeout", "plan_budget"):  # product-only
            orc.set_param(k, v)
    for st in prob["stacks"]:
        orc.add_stack(st["slices"], st["G"], st["thickness"])
    pp = prob["patch"]
    orc.extract_patches(pp["size"], pp["stride"], pp["depth"], pp["stride_z"])
    orc.set_transforms(prob["T"])
    return orc


def make_gpu(prob, params=None, device=0):
    from paper_1611_07289_b200 import Context, load_problem
    ctx = Context(prob["dims"], prob["spacing"], prob["origin"], device)
    return load_problem(ctx, prob, params)


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def weight_mismatch(p_g, p_o, pb_g, pb_o, w_g, w_o, tau_patch=0.5, tol=1e-3, margin=1e-4):
    """Max |dp| over pixels and max |dw| over patches, excluding (and counting) patches whose
    oracle pbar sits within `margin` of the exclusion threshold (SURVEY §8(c) comparison)."""
    near = np.abs(pb_o - tau_patch) < margin
    dw = np.abs(w_g - w_o)
    dw[near] = 0.0
    return float(np.abs(p_g - p_o).max()), float(dw.max() if dw.size else 0.0), int(near.sum())

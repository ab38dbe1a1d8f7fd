"""Shared test helpers: build the oracle and the GPU context on the same seeded problem."""
import numpy as np


def make_oracle(prob, params=None):
    from oracle import Oracle
    orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
    for k, v in (params or {}).items():
        if k != "profile":
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

"""Registration test problems (f1): stacks whose pixels are trilinear samples of a known
smooth volume at their world positions, so the true pose of every patch is known exactly.

The samples come from scipy.ndimage.map_coordinates (order 1, zero outside), a library
routine independent of both the oracle and the product; the volume is the seeded analytic
phantom of synth/ smoothed by scipy.ndimage.gaussian_filter."""
import math

import numpy as np
from scipy import ndimage

import synth


def registration_problem(cfg="c1", blur=1.0, texture=0.0, seed=77, **scale):
    """texture > 0 adds a seeded smooth random field (Gaussian-filtered noise, sigma 1.5
    voxels, std `texture`) so that every patch constrains all six pose parameters (a planar
    phantom edge alone leaves motion along the edge unobservable)."""
    prob = synth.make_problem(cfg, **scale)
    X = ndimage.gaussian_filter(synth.rasterize_phantom(prob).astype(np.float64), blur, mode="constant")
    if texture > 0:
        rng = np.random.default_rng(seed)
        f = ndimage.gaussian_filter(rng.normal(size=X.shape), 1.5, mode="wrap")
        X = X + texture * f / f.std()
    o = np.asarray(prob["origin"], np.float64)
    s = float(prob["spacing"])
    for st in prob["stacks"]:
        K, H, W = st["slices"].shape
        G = np.asarray(st["G"], np.float64)
        sl, row, col = np.meshgrid(np.arange(K), np.arange(H), np.arange(W), indexing="ij")
        idx = np.stack([col.ravel(), row.ravel(), sl.ravel(), np.ones(col.size)])
        w = G @ idx                                   # world (3, n)
        g = (w - o[:, None]) / s                      # voxel index (x, y, z)
        y = ndimage.map_coordinates(X, [g[2], g[1], g[0]], order=1, mode="constant", cval=0.0)
        st["slices"] = y.reshape(K, H, W).astype(np.float32)
    prob["T"] = np.tile(np.hstack([np.eye(3), np.zeros((3, 1))]), (len(prob["T"]), 1, 1))
    return prob, X


def euler_deg(rx, ry, rz):
    from synth.generate import euler
    return euler(rx, ry, rz)


def rigid_about(R, centre, t):
    """3x4: x -> R (x - centre) + centre + t."""
    centre = np.asarray(centre, np.float64)
    return np.hstack([R, (centre - R @ centre + np.asarray(t, np.float64))[:, None]])


def patch_centre_world(prob, patch, T):
    """World centre of a patch (stack, x0, y0, z0, sx, sy, sz) under its 3x4 transform T."""
    st, x0, y0, z0, sx, sy, sz = [int(v) for v in patch]
    G = np.asarray(prob["stacks"][st]["G"], np.float64)
    c = G @ np.array([x0 + 0.5 * (sx - 1), y0 + 0.5 * (sy - 1), z0 + 0.5 * (sz - 1), 1.0])
    return T[:, :3] @ c + T[:, 3]


def pose_error(T, T_ref, centre):
    """(translation error at `centre` [mm], rotation angle [deg]) between two 3x4 maps."""
    dt = np.linalg.norm((T[:, :3] @ centre + T[:, 3]) - (T_ref[:, :3] @ centre + T_ref[:, 3]))
    Rd = T[:, :3] @ T_ref[:, :3].T
    ang = math.degrees(math.acos(max(-1.0, min(1.0, (np.trace(Rd) - 1.0) / 2.0))))
    return dt, ang

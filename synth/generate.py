"""Seeded synthetic problems c1-c5 (BASELINE.json `configs`; recipe in DESIGN.md §Inputs).

A problem is a dict:
  dims (nx, ny, nz), spacing, origin          HR volume geometry (axes = identity)
  stacks: list of dict(slices f32 [K][H][W], G (3x4 f64 index->world), thickness)
  patch: dict(size, stride, depth, stride_z)  square-window extraction parameters
  T: f64 [M][3][4]                            per-patch world->world transforms
  corrupted: bool [M]                         patches given a gross transform error
  iters, alpha, lam                           run parameters of the config

The stacks are an *acquisition simulator*: an analytic ellipsoid phantom evaluated at
each pixel centre moved by that slice's true motion, averaged over a 5-point box slice
profile, plus Gaussian noise. This is deliberately NOT the method's PSF / forward model
(no trilinear, no sinc), so the generator holds none of the arithmetic under test.

Random streams (numpy PCG64): seed+0 phantom, +1 motion, +2 noise, +3 corruption,
+4 per-patch mismatch.
"""
import math

import numpy as np

# --------------------------------------------------------------------------- geometry
R_AXIAL = np.array([[1, 0, 0], [0, 1, 0], [0, 0, 1]], np.float64).T      # columns u, v, w
R_CORONAL = np.array([[1, 0, 0], [0, 0, 1], [0, -1, 0]], np.float64).T
R_SAGITTAL = np.array([[0, 1, 0], [0, 0, 1], [1, 0, 0]], np.float64).T


def rot_x(deg):
    a = math.radians(deg)
    return np.array([[1, 0, 0], [0, math.cos(a), -math.sin(a)], [0, math.sin(a), math.cos(a)]])


def rot_y(deg):
    a = math.radians(deg)
    return np.array([[math.cos(a), 0, math.sin(a)], [0, 1, 0], [-math.sin(a), 0, math.cos(a)]])


def rot_z(deg):
    a = math.radians(deg)
    return np.array([[math.cos(a), -math.sin(a), 0], [math.sin(a), math.cos(a), 0], [0, 0, 1]])


def euler(rx, ry, rz):
    return rot_z(rz) @ rot_y(ry) @ rot_x(rx)


def axis_angle(axis, deg):
    axis = np.asarray(axis, np.float64)
    axis = axis / np.linalg.norm(axis)
    a = math.radians(deg)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(a) * K + (1 - math.cos(a)) * (K @ K)


def affine(Lin, t):
    T = np.zeros((3, 4))
    T[:, :3] = Lin
    T[:, 3] = t
    return T


def about(Lin, centre, shift=(0, 0, 0)):
    """x -> Lin (x - centre) + centre + shift."""
    centre = np.asarray(centre, np.float64)
    return affine(Lin, centre - Lin @ centre + np.asarray(shift, np.float64))


def compose(A, B):
    """(A o B)(x) = A(B(x)) for 3x4 affines."""
    return affine(A[:, :3] @ B[:, :3], A[:, :3] @ B[:, 3] + A[:, 3])


def stack_G(R, pitch, step, W, H, K, centre):
    """index -> world: G = [R diag(pitch, pitch, step) | c - R diag(..) ((W-1)/2, (H-1)/2, (K-1)/2)]."""
    D = R @ np.diag([pitch, pitch, step])
    half = np.array([(W - 1) / 2.0, (H - 1) / 2.0, (K - 1) / 2.0])
    return affine(D, np.asarray(centre, np.float64) - D @ half)


def windows_1d(dim, size, stride):
    """Square-window starts along one axis; a last window is clamped to the edge."""
    out = list(range(0, dim - size + 1, stride))
    if out[-1] + size < dim:
        out.append(dim - size)
    return out


# --------------------------------------------------------------------------- phantom
def phantom_shapes(rng, half):
    """Nested ellipsoids on a 0-1000 scale; positions are fractions of the FOV half-width."""
    sh = [  # (centre frac, radii frac, value); later shapes paint over earlier ones
        ((0.0, 0.0, 0.0), (0.86, 0.76, 0.80), 300.0),     # body shell
        ((0.04, -0.05, 0.0), (0.62, 0.52, 0.56), 450.0),  # uterus / brain
        ((-0.12, 0.30, 0.04), (0.44, 0.13, 0.40), 500.0),  # placenta slab
        ((0.16, -0.16, 0.08), (0.26, 0.22, 0.25), 600.0),  # head
        ((0.16, -0.16, 0.08), (0.08, 0.05, 0.11), 900.0),  # ventricle
    ]
    out = [(np.array(c) * half, np.array(r) * half, v) for c, r, v in sh]
    return out


def small_spheres(rng, half, radius_mm):
    cs = rng.uniform(-0.45, 0.45, size=(5, 3)) * half
    return [(c, np.array([radius_mm] * 3), 1000.0) for c in cs]


def phantom_eval(shapes, pts):
    """pts [..., 3] world mm -> phantom value (float32)."""
    val = np.zeros(pts.shape[:-1], np.float32)
    for c, r, v in shapes:
        q = ((pts[..., 0] - c[0]) / r[0]) ** 2
        q += ((pts[..., 1] - c[1]) / r[1]) ** 2
        q += ((pts[..., 2] - c[2]) / r[2]) ** 2
        val[q <= 1.0] = v
    return val


def rasterize_phantom(prob, sub=4):
    """Ground-truth X* on the HR grid ([nz][ny][nx], f64), sub^3 box supersampling."""
    nx, ny, nz = prob["dims"]
    s, o = prob["spacing"], np.asarray(prob["origin"])
    offs = (np.arange(sub) + 0.5) / sub - 0.5
    out = np.zeros((nz, ny, nx))
    l, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    for a in offs:
        for b in offs:
            for c in offs:
                pts = np.stack([o[0] + s * (i + a), o[1] + s * (j + b), o[2] + s * (l + c)], -1)
                out += phantom_eval(prob["shapes"], pts)
    return out / sub ** 3


# --------------------------------------------------------------------------- acquisition
def acquire(shapes, G, thickness, W, H, K, motion, rng_noise, noise_sigma):
    """slices[k] = mean over a 5-point box slice profile of phantom(motion_k(pixel world)) + n."""
    Dn = G[:, :3]
    wdir = np.cross(Dn[:, 0], Dn[:, 1])
    wdir /= np.linalg.norm(wdir)
    prof = (np.arange(5) - 2) / 5.0 * thickness         # box profile, 5 points across theta
    out = np.empty((K, H, W), np.float32)
    v, u = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    for k in range(K):
        base = (G[:, 0][None, None, :] * u[..., None] + G[:, 1][None, None, :] * v[..., None]
                + G[:, 2] * k + G[:, 3])
        Tm = motion[k]
        acc = np.zeros((H, W), np.float32)
        for dz in prof:
            pts = base + dz * wdir
            pts = pts @ Tm[:, :3].T + Tm[:, 3]
            acc += phantom_eval(shapes, pts)
        out[k] = acc / len(prof)
    if noise_sigma > 0:
        out += rng_noise.normal(0.0, noise_sigma, size=out.shape).astype(np.float32)
    return out


# --------------------------------------------------------------------------- configs
CONFIGS = {
    "c1": dict(name="c1 synthetic phantom 32^3, 3 motion-free stacks, 16x16 patches stride 8",
               n=32, s=1.0, stacks=[("ax", 0.0), ("cor", 0.0), ("sag", 0.0)], W=32, K=8,
               pitch=1.0, step=4.0, theta=2.0, size=16, stride=8, depth=1, stride_z=1,
               motion="none", noise=0.0, seed=1001, iters=2, alpha=1.0, lam=0.02),
    "c2": dict(name="c2 fetal-brain SVR 128^3, 3 stacks x 30 slices, whole-slice patches",
               n=128, s=0.8, stacks=[("ax", 0.0), ("cor", 0.0), ("sag", 0.0)], W=128, K=30,
               pitch=0.8, step=3.2, theta=3.2, size=128, stride=128, depth=1, stride_z=1,
               motion="rigid5", noise=10.0, seed=2002, iters=10, alpha=1.0, lam=0.02),
    "c3": dict(name="c3 whole-uterus PVR 427^3 @0.75mm, 4 stacks 256x256x60, 64x64 patches stride 32",
               n=427, s=0.75, stacks=[("ax", 0.0), ("cor", 0.0), ("sag", 0.0), ("ax", 2.0)],
               W=256, K=60, pitch=1.25, step=4.0, theta=4.0, size=64, stride=32, depth=1,
               stride_z=1, motion="breathing", noise=10.0, seed=3003, iters=3, alpha=1.0, lam=0.02),
    "c4": dict(name="c4 3D patches 64x64x4, affine motion, 10% corrupted, 6 stacks",
               n=427, s=0.75, stacks=[("ax", 0.0), ("cor", 0.0), ("sag", 0.0), ("ax", 2.0),
                                      ("cor", 2.0), ("sag", 2.0)],
               W=256, K=60, pitch=1.25, step=4.0, theta=4.0, size=64, stride=32, depth=4,
               stride_z=4, motion="skew", noise=10.0, seed=4004, iters=3, alpha=1.0, lam=0.02,
               corrupt=0.10),
    "c5": dict(name="c5 scaling stress 800^3 @0.5mm, 8 stacks 320x320x80, 32x32 patches stride 8",
               n=800, s=0.5, stacks=[("ax", 0.0), ("cor", 0.0), ("sag", 0.0), ("ax", 2.0),
                                     ("cor", 2.0), ("sag", 2.0), ("ox30", 0.0), ("oy45", 0.0)],
               W=320, K=80, pitch=1.25, step=4.0, theta=4.0, size=32, stride=8, depth=1,
               stride_z=1, motion="breathing", noise=10.0, seed=5005, iters=1, alpha=1.0, lam=0.02),
}


def _orientation(tag):
    return {"ax": R_AXIAL, "cor": R_CORONAL, "sag": R_SAGITTAL,
            "ox30": rot_x(30.0) @ R_AXIAL, "oy45": rot_y(45.0) @ R_AXIAL}[tag]


def make_problem(cfg, scale=None, **over):
    """Build a seeded problem for config `cfg` ('c1'..'c5' or a dict).

    scale: optional (n_vox, W, K) override to shrink a config for fast tests while
    keeping its structure (pitch/spacing ratios, patch layout, motion and corruption).
    """
    c = dict(CONFIGS[cfg]) if isinstance(cfg, str) else dict(cfg)
    c.update(over)
    if scale is not None:
        c["n"], c["W"], c["K"] = scale
    n, s, W, K = c["n"], c["s"], c["W"], c["K"]
    seed = c["seed"]
    rng_ph = np.random.default_rng(seed + 0)
    rng_mo = np.random.default_rng(seed + 1)
    rng_no = np.random.default_rng(seed + 2)
    rng_co = np.random.default_rng(seed + 3)
    rng_pm = np.random.default_rng(seed + 4)
    half = s * n / 2.0
    origin = np.full(3, -s * (n - 1) / 2.0)
    shapes = phantom_shapes(rng_ph, half) + small_spheres(rng_ph, half, 2.0 * s)
    size = min(c["size"], W)
    stride = min(c["stride"], size)
    depth, stride_z = c["depth"], c["stride_z"]

    stacks, T_all, corrupted = [], [], []
    for tag, shift in c["stacks"]:
        R = _orientation(tag)
        centre = R[:, 2] * shift
        G = stack_G(R, c["pitch"], c["step"], W, W, K, centre)
        # per-slice true motion (world -> world, about the volume centre)
        motion = []
        if c["motion"] == "none":
            motion = [affine(np.eye(3), np.zeros(3)) for _ in range(K)]
        elif c["motion"] == "rigid5":
            for _ in range(K):
                ang = rng_mo.uniform(-5, 5, 3)
                motion.append(affine(euler(*ang), rng_mo.uniform(-3, 3, 3)))
        elif c["motion"] == "breathing":
            amp = rng_mo.uniform(2.0, 5.0)
            d = rng_mo.normal(size=3)
            d /= np.linalg.norm(d)
            ph = rng_mo.uniform(0, 2 * math.pi)
            for k in range(K):
                ang = rng_mo.uniform(-3, 3, 3)
                motion.append(affine(euler(*ang), amp * math.sin(2 * math.pi * k / 8.0 + ph) * d))
        elif c["motion"] == "skew":   # per slab of `depth` slices: skew o rigid
            for k0 in range(0, K, depth):
                th = rng_mo.uniform(-8, 8)
                sg = rng_mo.choice([-1.0, 1.0], size=6)
                Sk = np.eye(3)
                off = [(0, 1), (0, 2), (1, 0), (1, 2), (2, 0), (2, 1)]
                for (a, b), sgn in zip(off, sg):
                    Sk[a, b] = sgn * math.tan(math.radians(th))
                ang = rng_mo.uniform(-3, 3, 3)
                slab_c = G[:, :3] @ np.array([(W - 1) / 2, (W - 1) / 2, k0 + (depth - 1) / 2]) + G[:, 3]
                Tm = compose(affine(euler(*ang), rng_mo.uniform(-3, 3, 3)), about(Sk, slab_c))
                motion.extend([Tm] * min(depth, K - k0))
        else:
            raise ValueError(c["motion"])
        slices = acquire(shapes, G, c["theta"], W, W, K, motion, rng_no, c["noise"])
        stacks.append(dict(slices=slices, G=G, thickness=c["theta"]))
        # per-patch transforms handed to pvr_set_transforms: order stack, z0, y0, x0
        xs = windows_1d(W, size, stride)
        zs = windows_1d(K, depth, stride_z)
        for z0 in zs:
            for y0 in xs:
                for x0 in xs:
                    Tt = motion[z0]
                    pc = G @ np.array([x0 + (size - 1) / 2, y0 + (size - 1) / 2, z0 + (depth - 1) / 2, 1.0])
                    if c["motion"] == "breathing":   # piecewise-rigid mismatch per patch
                        eps = about(euler(*rng_pm.normal(0, 0.5, 3)), pc, rng_pm.normal(0, 0.3, 3))
                        Tt = compose(Tt, eps)
                    bad = False
                    if c.get("corrupt", 0) > 0 and rng_co.uniform() < c["corrupt"]:
                        axis = rng_co.normal(size=3)
                        gross = about(axis_angle(axis, rng_co.uniform(15, 25)), pc,
                                      rng_co.normal(size=3) / np.sqrt(3) * rng_co.uniform(10, 20))
                        Tt = compose(Tt, gross)
                        bad = True
                    T_all.append(Tt)
                    corrupted.append(bad)
    return dict(cfg=c, name=c["name"], dims=(n, n, n), spacing=s, origin=origin, stacks=stacks,
                patch=dict(size=size, stride=stride, depth=depth, stride_z=stride_z),
                T=np.array(T_all, np.float64), corrupted=np.array(corrupted, bool),
                shapes=shapes, iters=c["iters"], alpha=c["alpha"], lam=c["lam"])

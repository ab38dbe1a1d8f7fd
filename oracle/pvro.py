"""ctypes wrapper of liboracle (oracle/pvro.c) — TEST INFRASTRUCTURE ONLY.

Argument marshalling only; all arithmetic is in pvro.c (fp64).
"""
import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libpvro.so")
_SO_OVERRIDE = os.environ.get("PVRO_SO")  # tools/mutation_probe.py: a mutant build of pvro.c
_SRC = os.path.join(_HERE, "pvro.c")

PARAM = {
    "delta": 0, "tau_patch": 1, "c0": 2, "tau_live": 3, "tau_C": 4, "tau_obs": 5,
    "clamp": 6, "psf_mode": 7, "sigma2_floor": 9, "psf_nsigma": 10, "lazy": 12, "psf_quality": 13, "em_rounds": 14, "em_tol": 15, "patch_mixture": 16,
}


def build(force=False):
    """Compile oracle/pvro.c into oracle/libpvro.so (gcc, fp64, OpenMP)."""
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "pvro.h"))):
        return _SO
    cmd = ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"]
    subprocess.check_call(cmd)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if _SO_OVERRIDE:
            L = C.CDLL(_SO_OVERRIDE)
        else:
            build()
            L = C.CDLL(_SO)
        d, i32, i64, vp = C.c_double, C.c_int32, C.c_int64, C.c_void_p
        L.pvro_sinc_taylor.restype = d
        L.pvro_sinc_taylor.argtypes = [d]
        L.pvro_psf_table.restype = C.c_int
        L.pvro_psf_table.argtypes = [d, d, d, d, d, C.c_int, vp, vp, vp]
        L.pvro_psf_table_q.restype = C.c_int
        L.pvro_psf_table_q.argtypes = [d, d, d, d, d, d, C.c_int, vp, vp, vp]
        L.pvro_windows.restype = C.c_int
        L.pvro_windows.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, vp]
        L.pvro_posterior.restype = d
        L.pvro_posterior.argtypes = [d, d, d, d]
        L.pvro_em_round.restype = C.c_int
        L.pvro_em_round.argtypes = [i64, vp, vp, vp, i64, d, d, vp, vp, vp, vp]
        L.pvro_em_rounds.restype = C.c_int
        L.pvro_em_rounds.argtypes = [i64, vp, vp, vp, i64, d, d, C.c_int, d, vp, vp, vp, vp, vp]
        L.pvro_patch_mixture.restype = C.c_int
        L.pvro_patch_mixture.argtypes = [i64, vp, vp, C.c_int, d, vp]
        L.pvro_em_loglik.restype = d
        L.pvro_em_loglik.argtypes = [i64, vp, vp, d, d, d]
        L.pvro_patch_score.restype = d
        L.pvro_patch_score.argtypes = [i64, vp, vp]
        L.pvro_update_regularise.restype = C.c_int
        L.pvro_update_regularise.argtypes = [C.c_int, C.c_int, C.c_int, vp, vp, vp, d, d, d, d,
                                             C.c_int, d, d, vp, vp]
        L.pvro_create.restype = vp
        L.pvro_create.argtypes = [vp, d, vp]
        L.pvro_destroy.argtypes = [vp]
        L.pvro_set_param.argtypes = [vp, C.c_int, d]
        L.pvro_add_stack.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, vp, d]
        L.pvro_add_stack_f64.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, vp, d]
        L.pvro_extract_patches.restype = i64
        L.pvro_extract_patches.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int]
        L.pvro_set_patches.restype = i64
        L.pvro_set_patches.argtypes = [vp, i64, vp, vp]
        L.pvro_slic.restype = C.c_int
        L.pvro_slic.argtypes = [C.c_int, C.c_int, vp, C.c_float, C.c_float, C.c_int, C.c_int, C.c_int, vp]
        L.pvro_superpixel_patches.restype = i64
        L.pvro_superpixel_patches.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int]
        L.pvro_get_mask.argtypes = [vp, vp]
        L.pvro_num_pixels.restype = i64
        L.pvro_num_pixels.argtypes = [vp]
        L.pvro_get_patches.argtypes = [vp, vp]
        L.pvro_get_psf.argtypes = [vp, C.c_int, C.c_int, vp, vp]
        L.pvro_set_transforms.argtypes = [vp, vp, i64]
        L.pvro_set_volume.argtypes = [vp, vp]
        L.pvro_get_volume.argtypes = [vp, vp]
        L.pvro_forward.argtypes = [vp, vp, vp, vp]
        L.pvro_forward_range.argtypes = [vp, vp, i64, i64, vp, vp]
        L.pvro_adjoint.argtypes = [vp, vp, i64, i64, vp]
        L.pvro_adjoint_subset.argtypes = [vp, vp, vp, i64, vp]
        L.pvro_coverage_subset.argtypes = [vp, vp, i64]
        L.pvro_init_volume.argtypes = [vp]
        L.pvro_rigidity_map.argtypes = [vp, vp]
        L.pvro_set_weights.argtypes = [vp, vp, vp]
        L.pvro_cc.restype = d
        L.pvro_cc.argtypes = [i64, vp, vp]
        L.pvro_patch_cc.argtypes = [vp, vp, i64, vp, C.c_int, vp, vp]
        L.pvro_compose_pose.argtypes = [vp, i64, vp, vp]
        L.pvro_register.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp]
        L.pvro_sr_iterate.argtypes = [vp, C.c_int, d, d]
        L.pvro_get_weights.argtypes = [vp, vp, vp, vp]
        L.pvro_get_taps.argtypes = [vp, vp, vp, vp, vp]
        L.pvro_get_em_state.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _chk(rc, what):
    if rc < 0:
        raise RuntimeError(f"oracle {what} failed ({rc})")
    return rc


# ---- scalar building blocks ----
def cc(a, b):
    """Pearson correlation (oracle/pvro.c pvro_cc); NaN if degenerate."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return lib().pvro_cc(len(a), _p(a), _p(b))


def sinc_taylor(x):
    return lib().pvro_sinc_taylor(float(x))


def psf_table(dx, dy, theta, s, nsigma=3.0, q=1.0):
    cap = 20000
    abc = np.zeros((cap, 3), np.int32)
    psi = np.zeros(cap, np.float64)
    hw = np.zeros(7, np.float64)
    S = _chk(lib().pvro_psf_table_q(dx, dy, theta, s, nsigma, float(q), cap, _p(abc), _p(psi), _p(hw)), "psf")
    return abc[:S].copy(), psi[:S].copy(), hw


def windows(dim, size, stride):
    out = np.zeros(65536, np.int32)
    n = _chk(lib().pvro_windows(dim, size, stride, 65536, _p(out)), "windows")
    return out[:n].copy()


def posterior(e, sigma2, c, m):
    return lib().pvro_posterior(float(e), float(sigma2), float(c), float(m))


def em_round(e, live, p_prev, t, c0=0.9, sigma2_min=0.0):
    e = np.ascontiguousarray(e, np.float64)
    live = np.ascontiguousarray(live, np.uint8)
    p_prev = np.ascontiguousarray(p_prev, np.float64)
    p = np.zeros_like(e)
    s2, c, m = C.c_double(), C.c_double(), C.c_double()
    deg = lib().pvro_em_round(len(e), _p(e), _p(live), _p(p_prev), int(t), c0, sigma2_min, _p(p),
                              C.byref(s2), C.byref(c), C.byref(m))
    return p, s2.value, c.value, m.value, bool(deg)


def em_rounds(e, live, p_prev, t, rounds, tol=1e-6, c0=0.9, sigma2_min=0.0):
    """f4 multi-round EM (reading Q30): (p, sigma2, c, m, LL per round)."""
    e = np.ascontiguousarray(e, np.float64)
    live = np.ascontiguousarray(live, np.uint8)
    p_prev = np.ascontiguousarray(p_prev, np.float64)
    p = np.zeros_like(e)
    ll = np.zeros(max(1, rounds))
    s2, c, m = C.c_double(), C.c_double(), C.c_double()
    r = lib().pvro_em_rounds(len(e), _p(e), _p(live), _p(p_prev), int(t), c0, sigma2_min, int(rounds),
                             float(tol), _p(p), C.byref(s2), C.byref(c), C.byref(m), _p(ll))
    return p, s2.value, c.value, m.value, ll[:r].copy()


def patch_mixture(pbar, valid=None, rounds=50, tol=1e-6):
    """f4 two-Gaussian patch classification (reading Q31): inlier posterior per patch."""
    pbar = np.ascontiguousarray(pbar, np.float64)
    valid = np.ones(len(pbar), np.uint8) if valid is None else np.ascontiguousarray(valid, np.uint8)
    r = np.zeros(len(pbar))
    n = lib().pvro_patch_mixture(len(pbar), _p(pbar), _p(valid), int(rounds), float(tol), _p(r))
    return r, n


def slic(img, S, m, iters=10, ymin=None, ymax=None):
    """f3: integer SLIC labels of one slice (reading Q33)."""
    img = np.ascontiguousarray(img, np.float32)
    H, W = img.shape
    lab = np.zeros((H, W), np.int32)
    lo = float(img.min()) if ymin is None else ymin
    hi = float(img.max()) if ymax is None else ymax
    n = _chk(lib().pvro_slic(W, H, _p(img), lo, hi, int(S), int(m), int(iters), _p(lab)), "slic")
    return lab, n


def em_loglik(e, live, sigma2, c, m):
    e = np.ascontiguousarray(e, np.float64)
    live = np.ascontiguousarray(live, np.uint8)
    return lib().pvro_em_loglik(len(e), _p(e), _p(live), float(sigma2), float(c), float(m))


def patch_score(p, live=None):
    p = np.ascontiguousarray(p, np.float64)
    live = np.ones(len(p), np.uint8) if live is None else np.ascontiguousarray(live, np.uint8)
    return lib().pvro_patch_score(len(p), _p(p), _p(live))


def update_regularise(X0, A, Cv, alpha, lam, delta, tau_C=1e-6, clamp=False, lo=-np.inf, hi=np.inf):
    """X0, A, C as [nz][ny][nx] arrays; returns (X1, X2)."""
    X0 = np.ascontiguousarray(X0, np.float64)
    A = np.ascontiguousarray(A, np.float64)
    Cv = np.ascontiguousarray(Cv, np.float64)
    nz, ny, nx = X0.shape
    X1 = np.zeros_like(X0)
    X2 = np.zeros_like(X0)
    _chk(lib().pvro_update_regularise(nx, ny, nz, _p(X0), _p(A), _p(Cv), alpha, lam, delta, tau_C,
                                      int(clamp), lo, hi, _p(X1), _p(X2)), "update_regularise")
    return X1, X2


class Oracle:
    """Problem-level oracle mirroring the product's call sequence (fp64)."""

    def __init__(self, dims, spacing, origin):
        self.dims = tuple(int(d) for d in dims)  # (nx, ny, nz)
        d = np.array(self.dims, np.int32)
        o = np.array(origin, np.float64)
        self.h = lib().pvro_create(_p(d), float(spacing), _p(o))
        if not self.h:
            raise RuntimeError("pvro_create failed")
        self.V = int(np.prod(self.dims))
        self.M = 0
        self.P = 0

    def __del__(self):
        if getattr(self, "h", None):
            lib().pvro_destroy(self.h)
            self.h = None

    def set_param(self, key, value):
        _chk(lib().pvro_set_param(self.h, PARAM[key], float(value)), "set_param")

    def add_stack(self, slices, G, thickness):
        K, H, W = slices.shape
        G = np.ascontiguousarray(G, np.float64).reshape(12)
        if slices.dtype == np.float64:   # exact fp64 data for the fixed-point pins
            s64 = np.ascontiguousarray(slices)
            return _chk(lib().pvro_add_stack_f64(self.h, _p(s64), W, H, K, _p(G), float(thickness)),
                        "add_stack")
        slices = np.ascontiguousarray(slices, np.float32)
        return _chk(lib().pvro_add_stack(self.h, _p(slices), W, H, K, _p(G), float(thickness)),
                    "add_stack")

    def extract_patches(self, size, stride, depth=1, stride_z=1):
        self.M = _chk(lib().pvro_extract_patches(self.h, size, stride, depth, stride_z), "extract")
        self.P = lib().pvro_num_pixels(self.h)
        return self.M

    def set_patches(self, rects, mask=None):
        """f3: explicit patch rectangles [n][7] and optional per-pixel mask (reading Q32)."""
        rects = np.ascontiguousarray(rects, np.int32).reshape(-1, 7)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        self.M = _chk(lib().pvro_set_patches(self.h, len(rects), _p(rects), _p(m)), "set_patches")
        self.P = lib().pvro_num_pixels(self.h)
        return self.M

    def superpixel_patches(self, S, m, iters=10, gamma=2):
        """f3: SLIC superpixel patches of every slice, dilated by gamma (reading Q33)."""
        self.M = _chk(lib().pvro_superpixel_patches(self.h, int(S), int(m), int(iters), int(gamma)), "superpixels")
        self.P = lib().pvro_num_pixels(self.h)
        return self.M

    def mask(self):
        out = np.zeros(self.P, np.uint8)
        _chk(lib().pvro_get_mask(self.h, _p(out)), "get_mask")
        return out

    def patches(self):
        out = np.zeros((self.M, 7), np.int32)
        _chk(lib().pvro_get_patches(self.h, _p(out)), "get_patches")
        return out

    def psf(self, stack):
        abc = np.zeros((20000, 3), np.int32)
        psi = np.zeros(20000, np.float64)
        S = _chk(lib().pvro_get_psf(self.h, stack, 20000, _p(abc), _p(psi)), "get_psf")
        return abc[:S].copy(), psi[:S].copy()

    def set_transforms(self, T):
        T = np.ascontiguousarray(T, np.float64).reshape(-1, 12)
        _chk(lib().pvro_set_transforms(self.h, _p(T), len(T)), "set_transforms")

    def set_volume(self, X):
        X = np.ascontiguousarray(X, np.float64).reshape(-1)
        assert X.size == self.V
        lib().pvro_set_volume(self.h, _p(X))

    def volume(self):
        X = np.zeros(self.V, np.float64)
        lib().pvro_get_volume(self.h, _p(X))
        return X.reshape(self.dims[::-1])

    def forward(self, X):
        X = np.ascontiguousarray(X, np.float64).reshape(-1)
        yhat = np.zeros(self.P)
        kap = np.zeros(self.P)
        _chk(lib().pvro_forward(self.h, _p(X), _p(yhat), _p(kap)), "forward")
        return yhat, kap

    def forward_range(self, X, first, count):
        """yhat, kappa of patches [first, first+count) (global pixel indexing, zeros elsewhere)."""
        X = np.ascontiguousarray(X, np.float64).reshape(-1)
        yhat = np.zeros(self.P)
        kap = np.zeros(self.P)
        _chk(lib().pvro_forward_range(self.h, _p(X), first, count, _p(yhat), _p(kap)), "forward_range")
        return yhat, kap

    def adjoint(self, r, first=0, count=None):
        r = np.ascontiguousarray(r, np.float64)
        count = self.M - first if count is None else count
        out = np.zeros(self.V)
        _chk(lib().pvro_adjoint(self.h, _p(r), first, count, _p(out)), "adjoint")
        return out.reshape(self.dims[::-1])

    def adjoint_subset(self, r, patches, out=None):
        """W^T r over the patches listed (accumulated into out, a new zero volume if None)."""
        r = np.ascontiguousarray(r, np.float64)
        pl = np.ascontiguousarray(patches, np.int64)
        if out is None:
            out = np.zeros(self.V)
        _chk(lib().pvro_adjoint_subset(self.h, _p(r), _p(pl), len(pl), _p(out)), "adjoint_subset")
        return out

    def coverage_subset(self, patches):
        """kappa of the listed patches into the context (after a lazy set_transforms)."""
        pl = np.ascontiguousarray(patches, np.int64)
        _chk(lib().pvro_coverage_subset(self.h, _p(pl), len(pl)), "coverage_subset")

    def init_volume(self):
        _chk(lib().pvro_init_volume(self.h), "init_volume")

    def sr_iterate(self, n, alpha, lam):
        _chk(lib().pvro_sr_iterate(self.h, n, float(alpha), float(lam)), "sr_iterate")

    def set_weights(self, p=None, pbar=None):
        """Test hook: overwrite the E-step state (p [P], pbar [M])."""
        pa = None if p is None else np.ascontiguousarray(p, np.float64)
        pb = None if pbar is None else np.ascontiguousarray(pbar, np.float64)
        _chk(lib().pvro_set_weights(self.h, _p(pa), _p(pb)), "set_weights")

    # ---- f1 registration (reading Q29)
    def patch_cc(self, Xl, s, pose, min_valid=32):
        Xl = np.ascontiguousarray(Xl, np.float64).reshape(-1)
        pose = np.ascontiguousarray(pose, np.float64)
        cc = np.zeros(1)
        nv = np.zeros(1, np.int64)
        _chk(lib().pvro_patch_cc(self.h, _p(Xl), int(s), _p(pose), int(min_valid), _p(cc), _p(nv)), "patch_cc")
        return float(cc[0]), int(nv[0])

    def compose_pose(self, s, pose):
        out = np.zeros(12)
        _chk(lib().pvro_compose_pose(self.h, int(s), _p(np.ascontiguousarray(pose, np.float64)), _p(out)),
             "compose_pose")
        return out.reshape(3, 4)

    def register(self, levels=4, iters=20, min_valid=32):
        T = np.zeros((self.M, 12))
        st = np.zeros(self.M, np.int32)
        poses = np.zeros((self.M, 6))
        _chk(lib().pvro_register(self.h, int(levels), int(iters), int(min_valid), _p(T), _p(st), _p(poses)),
             "register")
        return T.reshape(self.M, 3, 4), st, poses

    def rigidity_map(self):
        """W^T(p pbar) / W^T 1 where W^T 1 > tau_C, else 0 (reading Q28)."""
        R = np.zeros(self.V, np.float64)
        _chk(lib().pvro_rigidity_map(self.h, _p(R)), "rigidity_map")
        return R.reshape(self.dims[::-1])

    def weights(self):
        p = np.zeros(self.P)
        pbar = np.zeros(self.M)
        w = np.zeros(self.M)
        lib().pvro_get_weights(self.h, _p(p), _p(pbar), _p(w))
        return p, pbar, w

    def taps(self):
        e = np.zeros(self.P)
        kap = np.zeros(self.P)
        A = np.zeros(self.V)
        Cv = np.zeros(self.V)
        lib().pvro_get_taps(self.h, _p(e), _p(kap), _p(A), _p(Cv))
        shp = self.dims[::-1]
        return e, kap, A.reshape(shp), Cv.reshape(shp)

    def em_state(self):
        v = [C.c_double() for _ in range(5)]
        t = C.c_int64()
        lib().pvro_get_em_state(self.h, C.byref(v[0]), C.byref(v[1]), C.byref(v[2]), C.byref(t),
                                C.byref(v[3]), C.byref(v[4]))
        return dict(sigma2=v[0].value, c=v[1].value, m=v[2].value, t=t.value, lo=v[3].value,
                    hi=v[4].value)

"""Thin ctypes binding of libpvr.so (include/pvr.h), same names as the C ABI.

Argument marshalling only: every step of the SR iteration runs in the library's CUDA
kernels. There is no CPU fallback; if libpvr.so is missing or no CUDA device is present
the calls raise.

Array arguments may be numpy arrays (host) or torch tensors (host or CUDA); they must be
C-contiguous with the dtype the C ABI states (float32 volumes/slices, float64 matrices).
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("PVR_SO") or os.path.join(_HERE, "libpvr.so")  # PVR_SO: A/B builds

PVR_OK, PVR_ERR_ARG, PVR_ERR_STATE, PVR_ERR_OOM, PVR_ERR_CUDA, PVR_ERR_NCCL, PVR_ERR_EMPTY = range(7)
STATUS_NAMES = {0: "PVR_OK", 1: "PVR_ERR_ARG", 2: "PVR_ERR_STATE", 3: "PVR_ERR_OOM",
                4: "PVR_ERR_CUDA", 5: "PVR_ERR_NCCL", 6: "PVR_ERR_EMPTY"}
PARAM = {"delta": 0, "tau_patch": 1, "c0": 2, "tau_live": 3, "tau_C": 4, "tau_obs": 5,
         "clamp": 6, "psf_mode": 7, "sigma2_floor": 9, "psf_nsigma": 10, "profile": 11, "psf_quality": 12,
         "em_rounds": 13, "em_tol": 14, "patch_mixture": 15,
         "bp_exact": 16, "exchange": 17, "comm_timeout": 18, "deterministic": 19,
         "plan_budget": 20}
EXCHANGE = {"allreduce": 0, "slabs": 1, "average": 2}
COLL_ALLREDUCE_SUM, COLL_ALLREDUCE_MAX, COLL_ALLGATHER = 0, 1, 2
DT_F32, DT_F64, DT_I64 = 0, 1, 2
# int fn(void* user, void* buf, int64_t count, int dtype, int op)
HOST_COLLECTIVE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int)

# every symbol include/pvr.h declares (checked by tests/test_abi.py)
EXPORTS = ["pvr_version", "pvr_create_volume", "pvr_destroy", "pvr_last_error", "pvr_comm_init", "pvr_comm_init_host",
           "pvr_comm_unique_id", "pvr_add_stack", "pvr_extract_patches", "pvr_plan_shards",
           "pvr_get_shard", "pvr_get_patches", "pvr_set_transforms", "pvr_set_volume",
           "pvr_init_volume", "pvr_set_param", "pvr_sr_iterate", "pvr_get_volume", "pvr_rigidity_map",
           "pvr_register_patches", "pvr_patch_cc", "pvr_set_patches", "pvr_superpixels",
           "pvr_superpixel_patches", "pvr_get_mask",
           "pvr_get_weights", "pvr_set_weights", "pvr_set_em_state", "pvr_get_taps", "pvr_get_confidence", "pvr_get_em_state", "pvr_get_stats",
           "pvr_reset_stats"]


class PvrError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class pvr_geometry(C.Structure):
    _fields_ = [("dims", C.c_int32 * 3), ("spacing_mm", C.c_double), ("origin_mm", C.c_double * 3)]


class pvr_stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("iterations", "psf_samples", "pixels", "voxels", "patches",
                                          "kernel_launches")] + \
               [(n, C.c_double) for n in ("ms_forward", "ms_em", "ms_estep", "ms_backproject",
                                           "ms_allreduce", "ms_update")] + \
               [(n, C.c_int64) for n in ("n_forward", "n_em", "n_estep", "n_backproject",
                                          "n_allreduce", "n_update", "bytes_alg_forward",
                                          "bytes_alg_estep", "bytes_alg_backproject",
                                          "bytes_alg_update")] + \
               [("fwd_tile", C.c_int32 * 3), ("bp_tile", C.c_int32 * 3)] + \
               [(n, C.c_int64) for n in ("fwd_groups", "bp_groups", "fwd_members", "bp_members",
                                          "fwd_smem", "bp_smem",
                                          "device_replans", "host_replans", "replan_splits",
                                          "bp_exact_groups", "fwd_split", "bp_split")]

    def as_dict(self):
        d = {}
        for n, _ in self._fields_:
            v = getattr(self, n)
            d[n] = list(v) if n.endswith("_tile") else v
        return d


_lib = None


def lib():
    """Load libpvr.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise RuntimeError(f"{SO_PATH} not built: run __graft_entry__.build() "
                               "(libpvr has no CPU fallback)")
        L = C.CDLL(SO_PATH)
        vp, i32, i64, d, f = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_float
        sig = {
            "pvr_version": (C.c_char_p, []),
            "pvr_create_volume": (i32, [C.POINTER(pvr_geometry), i32, vp, C.POINTER(vp)]),
            "pvr_destroy": (i32, [vp]),
            "pvr_last_error": (C.c_char_p, [vp]),
            "pvr_comm_init": (i32, [vp, i32, i32, vp]),
            "pvr_comm_unique_id": (i32, [vp]),
            "pvr_comm_init_host": (i32, [vp, i32, i32, HOST_COLLECTIVE, vp]),
            "pvr_get_confidence": (i32, [vp, vp, C.c_size_t]),
            "pvr_add_stack": (i32, [vp, vp, i32, i32, i32, vp, d, C.POINTER(i32)]),
            "pvr_extract_patches": (i32, [vp, i32, i32, i32, i32, C.POINTER(i64)]),
            "pvr_plan_shards": (i32, [vp, i64, i32, vp]),
            "pvr_get_shard": (i32, [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
            "pvr_get_patches": (i32, [vp, vp]),
            "pvr_set_transforms": (i32, [vp, vp, i64]),
            "pvr_set_volume": (i32, [vp, vp, C.c_size_t]),
            "pvr_init_volume": (i32, [vp]),
            "pvr_set_param": (i32, [vp, i32, d]),
            "pvr_sr_iterate": (i32, [vp, i32, f, f]),
            "pvr_get_volume": (i32, [vp, vp, C.c_size_t]),
            "pvr_rigidity_map": (i32, [vp, vp, C.c_size_t]),
            "pvr_register_patches": (i32, [vp, C.c_int, C.c_int, vp, vp, vp]),
            "pvr_patch_cc": (i32, [vp, C.c_int64, vp, vp, vp]),
            "pvr_set_patches": (i32, [vp, C.c_int64, vp, vp, vp]),
            "pvr_superpixels": (i32, [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp]),
            "pvr_superpixel_patches": (i32, [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp]),
            "pvr_get_mask": (i32, [vp, vp]),
            "pvr_get_weights": (i32, [vp, vp, vp, vp]),
            "pvr_set_weights": (i32, [vp, vp, vp, vp]),
            "pvr_set_em_state": (i32, [vp, d, d, d, i64]),
            "pvr_get_taps": (i32, [vp, vp, vp, vp, vp]),
            "pvr_get_em_state": (i32, [vp, C.POINTER(d), C.POINTER(d), C.POINTER(d), C.POINTER(i64),
                                       C.POINTER(d), C.POINTER(d)]),
            "pvr_get_stats": (i32, [vp, C.POINTER(pvr_stats)]),
            "pvr_reset_stats": (i32, [vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ptr(a):
    """Raw pointer of a numpy array or torch tensor (host or device); None passes NULL."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous, "arrays must be C-contiguous"
        return a.ctypes.data_as(C.c_void_p)
    if hasattr(a, "data_ptr"):
        assert a.is_contiguous(), "tensors must be contiguous"
        return C.c_void_p(a.data_ptr())
    raise TypeError(f"unsupported array type {type(a)}")


def _check(ctx, status):
    if status != PVR_OK:
        raise PvrError(status, lib().pvr_last_error(ctx).decode())
    return status


# ---- same names as the C ABI ----
def pvr_version():
    return lib().pvr_version().decode()


def pvr_create_volume(dims, spacing_mm, origin_mm, cuda_device=0, cuda_stream=None):
    g = pvr_geometry((C.c_int32 * 3)(*dims), float(spacing_mm), (C.c_double * 3)(*origin_mm))
    h = C.c_void_p()
    _check(None, lib().pvr_create_volume(C.byref(g), int(cuda_device), cuda_stream, C.byref(h)))
    return h


def pvr_destroy(ctx):
    return lib().pvr_destroy(ctx)


def pvr_last_error(ctx):
    return lib().pvr_last_error(ctx).decode()


def pvr_comm_unique_id():
    buf = (C.c_char * 128)()
    _check(None, lib().pvr_comm_unique_id(buf))
    return bytes(buf)


def pvr_comm_init(ctx, nranks, rank, unique_id):
    buf = (C.c_char * 128).from_buffer_copy(unique_id) if unique_id is not None else None
    _check(ctx, lib().pvr_comm_init(ctx, nranks, rank, buf))


def pvr_comm_init_host(ctx, nranks, rank, fn):
    """fn(buf: numpy array view of the library's host buffer, op) performs the collective in
    place (see pvr.h); returns the ctypes callback object, which must outlive the context."""
    dt = {DT_F32: np.float32, DT_F64: np.float64, DT_I64: np.int64}

    def tramp(user, buf, count, dtype, op):
        try:
            n = count * (nranks if op == COLL_ALLGATHER else 1)
            arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(np.ctypeslib.as_ctypes_type(dt[dtype]))), (n,))
            fn(arr, op)
            return 0
        except Exception as ex:  # the library turns a nonzero return into PVR_ERR_NCCL
            print("pvr host collective failed:", ex)
            return 1
    cb = HOST_COLLECTIVE(tramp)
    _check(ctx, lib().pvr_comm_init_host(ctx, nranks, rank, cb, None))
    return cb


def pvr_get_confidence(ctx, out):
    _check(ctx, lib().pvr_get_confidence(ctx, _ptr(out), out.size if isinstance(out, np.ndarray) else out.numel()))
    return out


def pvr_add_stack(ctx, slices, index_to_world, thickness_mm):
    K, H, W = slices.shape
    G = np.ascontiguousarray(index_to_world, np.float64).reshape(12)
    sid = C.c_int()
    _check(ctx, lib().pvr_add_stack(ctx, _ptr(slices), W, H, K, _ptr(G), float(thickness_mm), C.byref(sid)))
    return sid.value


def pvr_extract_patches(ctx, size, stride, depth=1, stride_z=1):
    m = C.c_int64()
    _check(ctx, lib().pvr_extract_patches(ctx, size, stride, depth, stride_z, C.byref(m)))
    return m.value


def pvr_plan_shards(cost, nranks):
    cost = np.ascontiguousarray(cost, np.int64)
    bounds = np.zeros(nranks + 1, np.int64)
    _check(None, lib().pvr_plan_shards(_ptr(cost), len(cost), nranks, _ptr(bounds)))
    return bounds


def pvr_get_shard(ctx):
    v = [C.c_int64() for _ in range(4)]
    _check(ctx, lib().pvr_get_shard(ctx, *[C.byref(x) for x in v]))
    return tuple(x.value for x in v)


def pvr_get_patches(ctx):
    _, n, _, _ = pvr_get_shard(ctx)
    out = np.zeros((n, 7), np.int32)
    _check(ctx, lib().pvr_get_patches(ctx, _ptr(out)))
    return out


def pvr_set_transforms(ctx, T):
    T = np.ascontiguousarray(T, np.float64).reshape(-1, 12) if isinstance(T, np.ndarray) else T
    _check(ctx, lib().pvr_set_transforms(ctx, _ptr(T), int(T.shape[0])))


def pvr_set_volume(ctx, x):
    _check(ctx, lib().pvr_set_volume(ctx, _ptr(x), int(np.prod(x.shape))))


def pvr_init_volume(ctx):
    _check(ctx, lib().pvr_init_volume(ctx))


def pvr_set_param(ctx, key, value):
    _check(ctx, lib().pvr_set_param(ctx, PARAM[key] if isinstance(key, str) else key, float(value)))


def pvr_sr_iterate(ctx, n, alpha, lam):
    _check(ctx, lib().pvr_sr_iterate(ctx, int(n), float(alpha), float(lam)))


def pvr_get_volume(ctx, out):
    _check(ctx, lib().pvr_get_volume(ctx, _ptr(out), int(np.prod(out.shape))))
    return out


def pvr_rigidity_map(ctx, out):
    _check(ctx, lib().pvr_rigidity_map(ctx, _ptr(out), int(np.prod(out.shape))))
    return out


def pvr_register_patches(ctx, levels, iters, T_out=None, status=None, poses=None):
    _check(ctx, lib().pvr_register_patches(ctx, int(levels), int(iters), _ptr(T_out), _ptr(status), _ptr(poses)))


def pvr_patch_cc(ctx, patch, poses, cc):
    _check(ctx, lib().pvr_patch_cc(ctx, int(len(patch)), _ptr(patch), _ptr(poses), _ptr(cc)))
    return cc


def pvr_get_weights(ctx, pixel_p=None, patch_w=None, patch_pbar=None):
    _check(ctx, lib().pvr_get_weights(ctx, _ptr(pixel_p), _ptr(patch_w), _ptr(patch_pbar)))


def pvr_set_weights(ctx, pixel_p=None, patch_w=None, patch_pbar=None):
    _check(ctx, lib().pvr_set_weights(ctx, _ptr(pixel_p), _ptr(patch_w), _ptr(patch_pbar)))


def pvr_set_em_state(ctx, sigma2, c, m, t):
    _check(ctx, lib().pvr_set_em_state(ctx, float(sigma2), float(c), float(m), int(t)))


def pvr_get_taps(ctx, e=None, kappa=None, addon=None, confidence=None):
    _check(ctx, lib().pvr_get_taps(ctx, _ptr(e), _ptr(kappa), _ptr(addon), _ptr(confidence)))


def pvr_get_em_state(ctx):
    v = [C.c_double() for _ in range(5)]
    t = C.c_int64()
    _check(ctx, lib().pvr_get_em_state(ctx, C.byref(v[0]), C.byref(v[1]), C.byref(v[2]), C.byref(t),
                                       C.byref(v[3]), C.byref(v[4])))
    return dict(sigma2=v[0].value, c=v[1].value, m=v[2].value, t=t.value, lo=v[3].value, hi=v[4].value)


def pvr_get_stats(ctx):
    s = pvr_stats()
    _check(ctx, lib().pvr_get_stats(ctx, C.byref(s)))
    return s.as_dict()


def pvr_reset_stats(ctx):
    _check(ctx, lib().pvr_reset_stats(ctx))


class Context:
    """Owning handle over a pvr_ctx; methods are the pvr_* calls without the prefix."""

    def __init__(self, dims, spacing_mm, origin_mm, cuda_device=0, cuda_stream=None):
        self.dims = tuple(int(d) for d in dims)
        self.h = pvr_create_volume(self.dims, spacing_mm, origin_mm, cuda_device, cuda_stream)
        self.V = int(np.prod(self.dims))
        self.M = 0

    def close(self):
        if getattr(self, "h", None):
            pvr_destroy(self.h)
            self.h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def comm_init(self, nranks, rank, uid):
        pvr_comm_init(self.h, nranks, rank, uid)

    def comm_init_host(self, nranks, rank, fn):
        self._coll = pvr_comm_init_host(self.h, nranks, rank, fn)  # keep the callback alive

    def confidence(self, out=None):
        if out is None:
            out = np.empty(tuple(self.dims)[::-1], np.float32)
        return pvr_get_confidence(self.h, out)

    def add_stack(self, slices, G, thickness):
        return pvr_add_stack(self.h, slices, G, thickness)

    def extract_patches(self, size, stride, depth=1, stride_z=1):
        self.M = pvr_extract_patches(self.h, size, stride, depth, stride_z)
        self.first, self.nloc, self.first_pix, self.nloc_pix = pvr_get_shard(self.h)
        return self.M

    def patches(self):
        return pvr_get_patches(self.h)

    def set_transforms(self, T):
        pvr_set_transforms(self.h, T)

    def set_volume(self, x):
        pvr_set_volume(self.h, x)

    def init_volume(self):
        pvr_init_volume(self.h)

    def set_param(self, key, value):
        pvr_set_param(self.h, key, value)

    def sr_iterate(self, n, alpha, lam):
        pvr_sr_iterate(self.h, n, alpha, lam)

    def volume(self, out=None):
        out = np.zeros(self.dims[::-1], np.float32) if out is None else out
        return pvr_get_volume(self.h, out)

    def register(self, levels=4, iters=20):
        """f1: rigid patch-to-volume registration by CC (pvr_register_patches). Returns
        (T [M][3][4] float64, status [M] int32, poses [M][6] float32); rows of other ranks are 0."""
        T = np.zeros((self.M, 12), np.float64)
        st = np.zeros(self.M, np.int32)
        poses = np.zeros((self.M, 6), np.float32)
        if self.M == 0:
            pvr_register_patches(self.h, levels, iters)
        else:
            pvr_register_patches(self.h, levels, iters, T, st, poses)
        return T.reshape(self.M, 3, 4), st, poses

    def patch_cc(self, patch, poses):
        patch = np.ascontiguousarray(patch, np.int64)
        poses = np.ascontiguousarray(poses, np.float32).reshape(-1, 6)
        cc = np.zeros(len(patch), np.float64)
        return pvr_patch_cc(self.h, patch, poses, cc)

    def set_patches(self, rects, mask=None):
        """f3: explicit patch rectangles [n][7] and optional per-pixel mask (pvr_set_patches)."""
        rects = np.ascontiguousarray(rects, np.int32).reshape(-1, 7)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        n = C.c_int64()
        _check(self.h, lib().pvr_set_patches(self.h, len(rects), _ptr(rects), _ptr(m), C.byref(n)))
        self.M = n.value
        self.first, self.nloc, self.first_pix, self.nloc_pix = pvr_get_shard(self.h)
        return self.M

    def superpixels(self, stack, S, m, iters=10, shape=None):
        """f3: SLIC labels [K][H][W] of one stack (pvr_superpixels); shape = (K, H, W)."""
        lab = np.zeros(shape, np.int32)
        _check(self.h, lib().pvr_superpixels(self.h, int(stack), int(S), int(m), int(iters), _ptr(lab)))
        return lab

    def superpixel_patches(self, S, m, iters=10, gamma=2):
        """f3: dilated SLIC superpixel patches of every slice (pvr_superpixel_patches)."""
        n = C.c_int64()
        _check(self.h, lib().pvr_superpixel_patches(self.h, int(S), int(m), int(iters), int(gamma), C.byref(n)))
        self.M = n.value
        self.first, self.nloc, self.first_pix, self.nloc_pix = pvr_get_shard(self.h)
        return self.M

    def mask(self):
        out = np.zeros(self.nloc_pix, np.uint8)
        _check(self.h, lib().pvr_get_mask(self.h, _ptr(out)))
        return out

    def rigidity_map(self, out=None):
        """W^T(p pbar) / W^T 1 (f2; float32 [nz][ny][nx], host or device out)."""
        out = np.zeros(self.dims[::-1], np.float32) if out is None else out
        return pvr_rigidity_map(self.h, out)

    def weights(self):
        p = np.zeros(self.nloc_pix, np.float32)
        w = np.zeros(self.nloc, np.float32)
        pb = np.zeros(self.nloc, np.float32)
        pvr_get_weights(self.h, p, w, pb)
        return p, pb, w

    def set_weights(self, p=None, pbar=None, w=None):
        """Restore what weights() returned (checkpoint / resume)."""
        f = lambda a: None if a is None else np.ascontiguousarray(a, np.float32)
        pvr_set_weights(self.h, f(p), f(w), f(pbar))

    def set_em_state(self, st):
        """Restore sigma^2, c, m, t from an em_state() dict."""
        pvr_set_em_state(self.h, st["sigma2"], st["c"], st["m"], st["t"])

    def taps(self):
        e = np.zeros(self.nloc_pix, np.float32)
        k = np.zeros(self.nloc_pix, np.float32)
        A = np.zeros(self.dims[::-1], np.float32)
        Cv = np.zeros(self.dims[::-1], np.float32)
        pvr_get_taps(self.h, e, k, A, Cv)
        return e, k, A, Cv

    def em_state(self):
        return pvr_get_em_state(self.h)

    def stats(self):
        return pvr_get_stats(self.h)

    def reset_stats(self):
        pvr_reset_stats(self.h)


def load_problem(ctx, prob, params=None):
    """Feed a synth problem dict through the C ABI: stacks, patches, transforms."""
    for k, v in (params or {}).items():
        ctx.set_param(k, v)
    for st in prob["stacks"]:
        ctx.add_stack(st["slices"], st["G"], st["thickness"])
    pp = prob["patch"]
    ctx.extract_patches(pp["size"], pp["stride"], pp["depth"], pp["stride_z"])
    ctx.set_transforms(prob["T"])
    return ctx

/* pvr.h — C ABI of libpvr.so: PVR's super-resolution (SR) iteration on B200 (sm_100a).
 *
 * Method: Alansary, Kainz et al., "PVR: Patch-to-Volume Reconstruction for Large Area
 * Motion Correction of Fetal MRI", arXiv 1611.07289. Citations "P:L" are lines of
 * /root/reference/PAPER.md; "§8(c)" is SURVEY.md §8(c); "Qn" are the readings listed
 * in DESIGN.md §Readings (where the paper is silent, garbled or defers to a citation).
 *
 * The library reconstructs a high-resolution (HR) volume X from stacks of 2D slices cut
 * into overlapping patches y_s (Eq. 2), each with its own transform T_s
 * (W_i = D B T_i, Eq. 1). One pvr_sr_iterate() iteration runs, on the GPU:
 *   a1 PSF-weighted forward simulation of every patch pixel   (Eq. 1; P:158-160 PSF)
 *   a2 residual e = y - yhat and EM sufficient statistics
 *   a3 EM parameters sigma^2, c, m
 *   a4 pixel posteriors p, patch scores pbar, patch weights w
 *   a5 adjoint backprojection into addon A and confidence C
 *   a6 SR update X1 = clip(X0 + alpha A / C)                     (reading Q16)
 *   a7 edge-preserving regularisation                           (reading Q17)
 * Every step runs in the library's own CUDA kernels; there is no CPU fallback. With
 * nranks > 1 (pvr_comm_init) patches are sharded over ranks and the EM statistics and
 * (A, C) are sum-allreduced over NCCL each iteration (reading Q21).
 *
 * Conventions
 *  - All functions return pvr_status; none throws or aborts. On error the message is
 *    available from pvr_last_error(). A CUDA or NCCL error poisons the context: after it
 *    only pvr_last_error() and pvr_destroy() are valid.
 *  - Inputs are copied before return; the library never retains caller pointers.
 *    Array arguments may be host or device pointers (detected per call).
 *  - Volume layout: float32 [nz][ny][nx], voxel (i,j,l) at world origin + s*(i,j,l),
 *    axes = identity ("isotropic" HR grid).
 *  - Patch pixel order ("patch-major"): patches in extraction order (stack, z0, y0, x0),
 *    within a patch slice z, then row v, then column u.
 *  - All device work is issued on the context's stream (cuda_stream argument of
 *    pvr_create_volume, or a stream the library creates when it is NULL).
 *  - A context is not thread-safe; use one per GPU / rank.
 *  - State machine: CREATED --add_stack--> STACKS --extract_patches--> PATCHED
 *    --set_transforms--> READY. Out-of-order calls return PVR_ERR_STATE.
 */
#ifndef PVR_H
#define PVR_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct pvr_ctx pvr_ctx;

typedef enum {
  PVR_OK = 0,
  PVR_ERR_ARG = 1,    /* invalid argument (sizes, geometry, ranges)                 */
  PVR_ERR_STATE = 2,  /* call out of order for the state machine above              */
  PVR_ERR_OOM = 3,    /* device or host allocation failed                           */
  PVR_ERR_CUDA = 4,   /* CUDA runtime / launch error (context poisoned)             */
  PVR_ERR_NCCL = 5,   /* NCCL error or NCCL unavailable (context poisoned)          */
  PVR_ERR_EMPTY = 6   /* nothing to reconstruct: no patch, or no observed pixel     */
} pvr_status;

typedef struct {
  int32_t dims[3];      /* nx, ny, nz >= 1                                          */
  double spacing_mm;    /* isotropic voxel size s > 0                               */
  double origin_mm[3];  /* world position of the centre of voxel (0,0,0)            */
} pvr_geometry;

/* Parameter keys for pvr_set_param (defaults in brackets). Keys marked (extract) must be
 * set before pvr_extract_patches; the others take effect at the next call that uses them. */
enum {
  PVR_PARAM_DELTA = 0,        /* regulariser edge scale delta [150] (Q17, Q18)            */
  PVR_PARAM_TAU_PATCH = 1,    /* patch kept iff pbar >= tau_patch [0.5] (Q13)             */
  PVR_PARAM_C0 = 2,           /* inlier proportion c at the first iteration [0.9] (Q10)    */
  PVR_PARAM_TAU_LIVE = 3,     /* pixel in the EM statistics iff kappa >= tau_live [0.99]   */
  PVR_PARAM_TAU_C = 4,        /* voxel updated iff C > tau_C [1e-6] (Q24)                  */
  PVR_PARAM_TAU_OBS = 5,      /* pixel observed iff kappa >= tau_obs [0.01] (Q25)          */
  PVR_PARAM_CLAMP = 6,        /* 1: clamp X1 to the live-y range +-10% [1] (Q19)           */
  PVR_PARAM_PSF_MODE = 7,     /* (extract) 0: PVR PSF; 1: delta PSF (tests only) [0]       */
  PVR_PARAM_SIGMA2_FLOOR = 9, /* sigma2 >= floor * (ymax - ymin)^2 [1e-6] (Q10)            */
  PVR_PARAM_PSF_NSIGMA = 10,  /* (extract) slice profile cut at nsigma * sigma_w [3] (Q3)  */
  PVR_PARAM_PROFILE = 11,     /* 1: time every kernel with CUDA events (pvr_get_stats) [0] */
  PVR_PARAM_PSF_QUALITY = 12, /* (extract) PSF lattice density q in [1, 4]: n_u = max(2,
                                 ceil(q pitch / s)), n_w = max(2, ceil(q theta / s)) (Q5);
                                 2 = the f4 "q = 2 quality mode" [1]        */
  PVR_PARAM_EM_ROUNDS = 13,   /* EM rounds per SR iteration in [1, 100] (f4 multi-round EM,
                                 S:399-402, reading Q30): rounds 2.. re-run the M- and E-step
                                 on the iteration's residuals until the log-likelihood gain
                                 is below tol |LL| [1]                                      */
  PVR_PARAM_EM_TOL = 14,      /* that relative tolerance [1e-6]                              */
  PVR_PARAM_PATCH_MIXTURE = 15 /* 1: patch weights from a two-Gaussian mixture on pbar (f4,
                                 P:209 "an inlier and outlier probability for each y_s",
                                 reading Q31): w = inlier posterior r if r >= 1/2, else 0;
                                 0: the threshold rule of Q13 [0]                          */
  ,PVR_PARAM_EXCHANGE = 17     /* multi-rank exchange scheme PVR_EXCHANGE_* [0]; set it before
                                 pvr_comm_init / pvr_comm_init_host                          */
  ,PVR_PARAM_COMM_TIMEOUT = 18 /* seconds a wait on NCCL work may take before the library
                                 aborts the communicator (ncclCommAbort) and returns
                                 PVR_ERR_NCCL; NCCL asynchronous errors are polled while
                                 waiting [300]                                               */
  ,PVR_PARAM_DETERMINISTIC = 19 /* (extract) 1: every reduction is order-independent, so X, p
                                 and w are bit-identical from run to run and for any number of
                                 ranks: the EM sums add terms rounded to fixed grids (exact in
                                 fp64), the backprojection uses one global tile scale with
                                 three int32 words per value (24 B per cell) and int64 (A, C)
                                 accumulators. Slower (~1.5x the backprojection); the
                                 two-Gaussian patch mixture (f4) is not covered [0]           */
  ,PVR_PARAM_PLAN_BUDGET = 20 /* (extract) fraction in [0.05, 1] of the shared-memory tile
                                 budgets the planner sizes groups for (forward X tile,
                                 backprojection tile); the kernels keep their full size. Below
                                 1 the planner halves and splits groups as at a larger problem:
                                 tests run those paths on small grids [1]                       */
  ,PVR_PARAM_BP_EXACT = 16    /* (extract) precision of the backprojection's shared tiles
                                 (DESIGN.md 7). 1 [default]: exact hi/lo int32 word pairs
                                 (~2^-41 of the group's largest splat term) for every group
                                 that can reach the rim of the coverage -- members on a stack
                                 border, on a patch border or next to a masked pixel (explicit
                                 patches), of stacks with slice gaps, or whose footprint leaves
                                 the grid -- where confidences fall to tau_C; one int32 word
                                 (2^-20 of the largest term) elsewhere, where every cell's
                                 confidence is that of a covered interior. 2: exact everywhere.
                                 0: one word everywhere (a timing reference, not parity-tested
                                 below tau_C = 1e-3)                                          */
};

/* Version string of the library build. */
const char* pvr_version(void);

/* Create a context for one HR volume on cuda_device. cuda_stream: a cudaStream_t to issue
 * all work on (the caller keeps ownership), or NULL for a library-owned stream.
 * Errors: PVR_ERR_ARG (dims < 1, spacing <= 0, (nx + 1) ny nz >= 2^31 voxels: the kernels
 * index the volume with 32-bit offsets), PVR_ERR_CUDA, PVR_ERR_OOM. */
pvr_status pvr_create_volume(const pvr_geometry* g, int cuda_device, void* cuda_stream,
                             pvr_ctx** out);
pvr_status pvr_destroy(pvr_ctx* ctx);
/* Last error message of ctx (a static string when ctx is NULL). Never NULL. */
const char* pvr_last_error(const pvr_ctx* ctx);

/* Optional, before pvr_extract_patches: join an NCCL communicator of nranks ranks (one
 * process per GPU). nccl_unique_id: the 128-byte ncclUniqueId created by rank 0 and
 * broadcast by the caller (e.g. over torch.distributed). Patches are then sharded in
 * contiguous ranges balanced by pixels x PSF samples; X is replicated.
 * Errors: PVR_ERR_ARG, PVR_ERR_STATE, PVR_ERR_NCCL (library not loadable / init failed). */
pvr_status pvr_comm_init(pvr_ctx* ctx, int nranks, int rank, const void* nccl_unique_id);
/* Fill a 128-byte buffer with a fresh ncclUniqueId (rank 0 only). */
pvr_status pvr_comm_unique_id(void* out128);

/* Host-collective transport, the alternative to pvr_comm_init (same place in the call
 * sequence): every exchange step of the iteration runs as a call of `fn` on a pinned HOST
 * buffer the library owns, copied from the device before and back after the call. The
 * caller implements the collective with any transport (tests back it with torch.distributed
 * gloo across processes that may share one GPU: no kernel ever waits on another rank).
 *   op PVR_COLL_ALLREDUCE_SUM / _MAX: buf holds count elements, reduced in place over ranks;
 *   op PVR_COLL_ALLGATHER: buf holds nranks * count elements; every rank's count elements at
 *     [rank * count] are gathered into all ranks' buffers.
 * dtype: PVR_DT_F32 / PVR_DT_F64 / PVR_DT_I64. fn returns 0 on success; anything else poisons
 * the context (PVR_ERR_NCCL). */
typedef enum { PVR_COLL_ALLREDUCE_SUM = 0, PVR_COLL_ALLREDUCE_MAX = 1, PVR_COLL_ALLGATHER = 2 } pvr_coll_op;
typedef enum { PVR_DT_F32 = 0, PVR_DT_F64 = 1, PVR_DT_I64 = 2 } pvr_dtype;
typedef int (*pvr_host_collective_fn)(void* user, void* buf, int64_t count, int dtype, int op);
pvr_status pvr_comm_init_host(pvr_ctx* ctx, int nranks, int rank, pvr_host_collective_fn fn, void* user);

/* Exchange schemes of (A, C) per iteration (PVR_PARAM_EXCHANGE):
 *  PVR_EXCHANGE_ALLREDUCE: sum-allreduce of (A, C), every rank runs the whole update (the
 *    1-rank operator up to summation order; reading Q21) [default];
 *  PVR_EXCHANGE_SLABS: reduce-scatter of (A, C) over z slabs (+ one halo plane from each
 *    neighbour), each rank updates its slab, all-gather of the new X: 12 V (N-1)/N bytes per
 *    rank instead of 16 V (N-1)/N, and the update split N ways (same operator);
 *  PVR_EXCHANGE_AVERAGE: the paper's "averaging of the resulting sub reconstruction volumes
 *    on the master GPU", for comparison only: each rank updates X with its own
 *    patches' (A, C), then X = mean over ranks (NOT the 1-rank operator). */
enum { PVR_EXCHANGE_ALLREDUCE = 0, PVR_EXCHANGE_SLABS = 1, PVR_EXCHANGE_AVERAGE = 2 };

/* Add one stack of slices ("stacks of 2D images").
 * slices: float32 [K][H][W], host or device, copied.
 * index_to_world: row-major 3x4 double, world_mm = M (col, row, slice, 1); its first two
 *   columns give the in-plane pixel pitches |col0| = dx, |col1| = dy and directions, the
 *   third the slice step (may differ from the thickness).
 * thickness_mm: slice profile FWHM theta > 0 ("slice profile for the through-plane").
 * Errors: PVR_ERR_ARG (sizes < 1, thickness <= 0, degenerate in-plane axes),
 * PVR_ERR_STATE (after extract_patches). */
pvr_status pvr_add_stack(pvr_ctx* ctx, const float* slices, int W, int H, int K,
                         const double index_to_world[12], double thickness_mm,
                         int* stack_id_out);

/* Cut every stack into square size x size windows at stride `stride` in-plane and
 * depth-slice windows at stride_z through-plane ("size a and stride omega";
 * depth > 1 gives 3D patches). The last window of an axis is clamped to the edge (Q22).
 * Builds the PSF tables (Q1-Q5) and the shard plan. Returns the global
 * patch count M. Errors: PVR_ERR_ARG (size > W or H, stride < 1 or > size, depth > K,
 * stride_z < 1 or > depth), PVR_ERR_STATE, PVR_ERR_EMPTY (M = 0). */
pvr_status pvr_extract_patches(pvr_ctx* ctx, int size, int stride, int depth, int stride_z,
                               int64_t* n_patches_out);
/* Patch extraction (pvr_extract_patches, pvr_set_patches, pvr_superpixel_patches) may be
 * repeated in a context that already has patches: the f3 multi-scale schedule (P:147-153,
 * "different scales Y_i ... for each iteration i"). The previous patches, their weights and
 * plans are dropped; the stacks and the reconstruction X stay; pvr_set_transforms (for the new
 * patch count) is required before the next iteration. */
/* f3 arbitrary-shape patches (Eq. 3: patches y_s need not be
 * squares; superpixels dilated by gamma pixels; reading Q32), instead of
 * pvr_extract_patches: n explicit rectangles rects int32 [n][7] = (stack, x0, y0, z0, sx, sy,
 * sz), each inside its stack, and an optional per-pixel mask uint8 (patch-major, sum of
 * sx sy sz bytes; NULL = every pixel): a masked-out pixel is never an observation (its
 * coverage kappa is 0, so it has no residual, posterior or splat). Host or device pointers.
 * Errors: PVR_ERR_STATE (not right after the stacks), PVR_ERR_ARG (n < 1, a rectangle
 * outside its stack). */
pvr_status pvr_set_patches(pvr_ctx* ctx, int64_t n, const int32_t* rects, const uint8_t* mask,
                           int64_t* n_patches);
/* f3 superpixels (Eq. 3; reading Q33): SLIC labels of every slice
 * of one stack, int32 [K][H][W] (host or device): integer SLIC (exact, reproducible) with grid
 * step S >= 2 pixels, compactness m >= 1 and `iters` >= 0 update rounds; label = the cluster
 * index on the slice's ceil(W/S) x ceil(H/S) grid. Needs the stacks, before the patches
 * (PVR_ERR_STATE otherwise). */
pvr_status pvr_superpixels(pvr_ctx* ctx, int stack, int S, int m, int iters, int32_t* labels);
/* f3 superpixel patches ("dilate each superpixel y_s by gamma pixels using a flat
 * structuring element"; readings Q32, Q33), instead of pvr_extract_patches: SLIC on every
 * slice of every stack, then one patch per non-empty superpixel (order: stack, slice,
 * cluster): its bounding box dilated by gamma pixels (clipped to the slice) with the mask of
 * the superpixel dilated by a (2 gamma + 1)^2 square. Errors as pvr_superpixels, plus
 * PVR_ERR_EMPTY (no superpixel). */
pvr_status pvr_superpixel_patches(pvr_ctx* ctx, int S, int m, int iters, int gamma, int64_t* n_patches);
/* The per-pixel patch mask of this rank's pixels, uint8 [n_local_pixels] (1 everywhere unless
 * the patches came with masks). Host or device. */
pvr_status pvr_get_mask(pvr_ctx* ctx, uint8_t* out);
/* Host-only helper (no GPU needed): contiguous shard plan of M patches over nranks,
 * balanced by cost[s] (pixels x PSF samples of patch s): rank r owns patches
 * [bounds[r], bounds[r+1]); bounds has nranks + 1 entries, bounds[0] = 0, bounds[nranks] = M.
 * P:233 "distributing independent subsets of patches over the desired number of devices".
 * Errors: PVR_ERR_ARG (null pointers, M < 0, nranks < 1). */
pvr_status pvr_plan_shards(const int64_t* cost, int64_t M, int nranks, int64_t* bounds);

/* This rank's shard: patches [first_patch, first_patch + n_local), and its pixel range in
 * the global patch-major pixel order. Any output pointer may be NULL. */
pvr_status pvr_get_shard(const pvr_ctx* ctx, int64_t* first_patch, int64_t* n_local,
                         int64_t* first_pixel, int64_t* n_local_pixels);
/* Patch table of this rank's shard: 7 int32 per patch {stack, x0, y0, z0, sx, sy, sz},
 * host pointer. */
pvr_status pvr_get_patches(const pvr_ctx* ctx, int32_t* out);

/* Per-patch transforms (P:58 T_i; "continuously rigidly registered"): n = M
 * row-major 3x4 double world->world affines for ALL patches (every rank passes the same
 * array). The volume is sampled at T_s(pixel_world + PSF offset) (reading Q7); rigid is
 * the special case. Computes the coverage kappa of every pixel and resets the EM state
 * (p_prev = 1, w = 1, t = 0) and the live-y range used by the clamp and the sigma^2 floor.
 * Errors: PVR_ERR_ARG (n != M), PVR_ERR_STATE (before extract), PVR_ERR_EMPTY (no
 * observed pixel on any rank). Collective when nranks > 1. */
pvr_status pvr_set_transforms(pvr_ctx* ctx, const double* T, int64_t n);

/* Set X (float32 [nz][ny][nx], host or device). Errors: PVR_ERR_ARG (nvox != V). */
pvr_status pvr_set_volume(pvr_ctx* ctx, const float* x, size_t nvox);
/* X = W^T y / W^T 1 where W^T 1 > tau_C, else the mean of the covered 26-neighbours, else 0
 * ("empty voxels are filled using the mean of the surrounding voxels").
 * Errors: PVR_ERR_STATE (before set_transforms). Collective when nranks > 1. */
pvr_status pvr_init_volume(pvr_ctx* ctx);
/* Set a parameter (keys above). Errors: PVR_ERR_ARG (unknown key / invalid value),
 * PVR_ERR_STATE ((extract) keys after extract_patches). */
pvr_status pvr_set_param(pvr_ctx* ctx, int key, double value);

/* Run n SR iterations (steps a1-a7 above), all on the device.
 * Errors: PVR_ERR_ARG (n < 0, alpha < 0, lambda < 0), PVR_ERR_STATE (before
 * set_transforms), PVR_ERR_CUDA / PVR_ERR_NCCL. alpha*lambda > 3/44 is accepted (the
 * maximum principle of the regulariser no longer holds; a warning is left in
 * pvr_last_error). Collective when nranks > 1. */
pvr_status pvr_sr_iterate(pvr_ctx* ctx, int n, float alpha, float lambda);

/* Copy X out (float32 [nz][ny][nx]; host or device pointer). Errors: PVR_ERR_ARG. */
pvr_status pvr_get_volume(pvr_ctx* ctx, float* out, size_t nvox);
/* Rigidity map ("Integrating p and pbar into a 3D volume using the
 * same PSF as for the reconstruction identifies candidate regions, solely containing rigid
 * motion components"; reading Q28 in DESIGN.md):
 *   out_k = [W^T (p pbar_s)]_k / [W^T 1]_k  where [W^T 1]_k > tau_C, else 0,
 * W^T over the observed pixels (kappa >= tau_obs) of ALL patches (excluded ones included:
 * their low pbar marks non-rigid regions) with the reconstruction's PSF and 1/kappa row
 * normalisation; p, pbar of the last E-step (all 1 right after set_transforms). Values lie in
 * [0, 1]. out: float32 [nz][ny][nx], host or device pointer; one backprojection pass on the
 * device (exact hi/lo tiles, as pvr_init_volume). Overwrites the addon / confidence returned
 * by pvr_get_taps. Errors: PVR_ERR_ARG (nvox != V), PVR_ERR_STATE (before set_transforms).
 * Collective when nranks > 1. */
pvr_status pvr_rigidity_map(pvr_ctx* ctx, float* out, size_t nvox);

/* f1 rigid patch-to-volume registration ("individual 2D patches
 * are continuously rigidly registered to the current 3D reconstruction", with cross
 * correlation as the similarity; reading Q29 in DESIGN.md). For every patch of this
 * rank, a rigid pose p = (tx, ty, tz [mm], rx, ry, rz [deg]) applied AFTER its current
 * transform T_s (the last pvr_set_transforms), rotating about the transformed patch centre c:
 *   x -> R (x - c) + c + t,  R = Rz(rz) Ry(ry) Rx(rx),
 * maximising CC(y_s, X(p)) over all the patch's pixels, X(p)_j = trilinear sample of the
 * current X at pixel j's mapped centre (corners outside the grid read 0). Optimiser: levels
 * L = 0 .. levels-1 with steps 2^-L x (2 mm, 4 deg); per level at most `iters` compass moves
 * (the 12 coordinate moves +-step are evaluated; the best strict CC improvement is taken,
 * first index on ties; the level ends when none improves). Recommended: levels 4, iters 20.
 * Outputs (host or device pointers, any may be NULL), written for this rank's patches only
 * (rows first .. first + n_local - 1 of the global arrays):
 *   T_out  double [M][12]: T_pose o T_s (row-major 3x4), = T_s when unregistrable;
 *   status int32 [M]: 1 registered, 0 unregistrable (fewer than 32 pixels, or an undefined
 *          CC at the start: constant patch or constant samples);
 *   poses  float [M][6]: the pose parameters.
 * The reconstruction state is unchanged; pass T_out to pvr_set_transforms to use it.
 * Errors: PVR_ERR_STATE (before set_transforms), PVR_ERR_ARG (levels outside [1, 16],
 * iters < 0, a patch over 190 KB of pixels), PVR_ERR_CUDA. Not collective. */
pvr_status pvr_register_patches(pvr_ctx* ctx, int levels, int iters, double* T_out, int32_t* status,
                                float* poses);
/* The registration's similarity at given poses (tap for tests and diagnostics): cc[i] = CC
 * of global patch patch[i] (must be on this rank) under pose poses[i][0..5] (as above);
 * NaN when undefined. patch int64 [n], poses float [n][6], cc double [n]: host or device.
 * Errors: PVR_ERR_STATE, PVR_ERR_ARG (n < 0, NULL arrays, a patch not on this rank). */
pvr_status pvr_patch_cc(pvr_ctx* ctx, int64_t n, const int64_t* patch, const float* poses, double* cc);
/* Weights of this rank's shard after the last iteration: pixel posteriors p
 * [n_local_pixels], patch weights w and patch scores pbar [n_local]; any may be NULL. */
pvr_status pvr_get_weights(pvr_ctx* ctx, float* pixel_p, float* patch_w, float* patch_pbar);
/* Checkpoint / resume: restore what pvr_get_weights returned (this shard's
 * pixel p [n_local_pixels], patch w and pbar [n_local]; any may be NULL, host or device
 * pointers). With pvr_set_volume and pvr_set_em_state this resumes an SR run exactly: the
 * next iteration reads X, the previous p (P:193's M-step partials) and t, nothing else.
 * Errors: PVR_ERR_STATE (before set_transforms). */
pvr_status pvr_set_weights(pvr_ctx* ctx, const float* pixel_p, const float* patch_w, const float* patch_pbar);
/* Restore sigma^2, c, m and the iteration counter t (c = c0 while t <= 1, reading Q10) as
 * pvr_get_em_state returned them; the clamp range stays the one set_transforms formed.
 * Errors: PVR_ERR_ARG (t < 0, sigma2 < 0, c outside [0, 1], m < 0), PVR_ERR_STATE. */
pvr_status pvr_set_em_state(pvr_ctx* ctx, double sigma2, double c, double m, int64_t iter);
/* Debug taps of the last iteration: residual e and coverage kappa [n_local_pixels] of this
 * shard, and the (reduced) addon A and confidence C [V]; any may be NULL. */
pvr_status pvr_get_taps(pvr_ctx* ctx, float* e, float* kappa, float* addon, float* confidence);
/* Confidence map C_k = sum_s w_s sum_j W_jk p_j of the last iteration (north_star
 * "confidence map"), the denominator of the SR update (P:185,
 * reading Q16): float32 [nz][ny][nx], host or device pointer (device copies stay on the
 * device). After pvr_init_volume it is W^T 1 over the observed pixels. Errors: PVR_ERR_ARG
 * (nvox != nx ny nz), PVR_ERR_STATE (before set_transforms). */
pvr_status pvr_get_confidence(pvr_ctx* ctx, float* out, size_t nvox);
/* EM state after the last iteration: sigma^2, c, m, iteration counter t, and the clamp
 * range [lo, hi]. Any output may be NULL. */
pvr_status pvr_get_em_state(pvr_ctx* ctx, double* sigma2, double* c, double* m, int64_t* iter,
                            double* lo, double* hi);

/* Counters accumulated since the last pvr_reset_stats (kernel times need PVR_PARAM_PROFILE). */
typedef struct {
  int64_t iterations;         /* SR iterations run                                       */
  int64_t psf_samples;        /* PSF samples visited by the forward model (P x S summed) */
  int64_t pixels;             /* patch pixels of this shard                               */
  int64_t voxels;             /* V                                                        */
  int64_t patches;            /* patches of this shard                                    */
  int64_t kernel_launches;    /* kernels launched by pvr_sr_iterate                       */
  double ms_forward;          /* a1+a2 (k_forward)                                        */
  double ms_em;               /* a3 (k_em_params) + statistics allreduce                  */
  double ms_estep;            /* a4 (k_estep)                                             */
  double ms_backproject;      /* a5 (k_backproject, including the A/C clear)              */
  double ms_allreduce;        /* A/C allreduce (nranks > 1)                               */
  double ms_update;           /* a6+a7 (k_update_regularise)                              */
  int64_t n_forward, n_em, n_estep, n_backproject, n_allreduce, n_update; /* launches     */
  int64_t bytes_alg_forward;      /* algorithmic HBM bytes per forward launch             */
  int64_t bytes_alg_estep;        /* per E-step launch                                    */
  int64_t bytes_alg_backproject;  /* per backprojection launch                            */
  int64_t bytes_alg_update;       /* per update launch                                    */
  int32_t fwd_tile[3];            /* forward plan: tile TU, TV (pixels), 1                 */
  int32_t bp_tile[3];             /* backprojection plan: TU, TV, through-plane segments   */
  int64_t fwd_groups, bp_groups;  /* CTAs' work items (groups of overlapping member tiles) */
  int64_t fwd_members, bp_members;
  int64_t fwd_smem, bp_smem;      /* dynamic shared memory per CTA (bytes)                 */
  int64_t device_replans;         /* set_transforms calls served by the device re-plan     */
  int64_t host_replans;           /* set_transforms calls that ran the host planner        */
  int64_t replan_splits;          /* members moved into single-member backprojection groups
                                     by device re-plans (their group outgrew the tile)       */
  int64_t bp_exact_groups;        /* backprojection groups with exact hi/lo tiles (rim)    */
  int64_t fwd_split, bp_split;    /* host plan: natural groups not kept whole (an outlying
                                     member left, or the union did not fit) + members split
                                     into smaller pixel tiles                                */
} pvr_stats;
pvr_status pvr_get_stats(const pvr_ctx* ctx, pvr_stats* out);
pvr_status pvr_reset_stats(pvr_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* PVR_H */

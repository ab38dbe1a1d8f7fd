// engine.cu — host engine and C ABI of libpvr.so (include/pvr.h).
//
// Host side, in fp64: the state machine, stack frames and separable PSF tables (P:158-160,
// readings Q1-Q5), square-patch extraction (Q22), the shard plan (Q21), the
// per-patch composition of index->world, T_s and world->voxel maps (Q7), and the work
// plan of the lattice kernels (member tiles grouped by shared stack pixels, each group with
// its voxel bounding box). The kernels (kernels.cu, lattice.cu) consume fp32 copies. Device
// work is issued on the context's stream; NCCL is dlopen'd at pvr_comm_init.
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <parallel/algorithm>
#include <chrono>
#include <thread>
#include <cstdlib>
#include <memory>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/pvr.h"
#include "pvr_internal.h"

using namespace pvr;

namespace {

enum State { CREATED = 0, STACKS = 1, PATCHED = 2, READY = 3 };

struct HostStack {
  int W, H, K;
  double G[12];
  double theta;
  double u[3], v[3], w[3], h[3];  // in-plane axes, slice normal, PSF lattice steps (mm)
  int S = 0;                       // PSF samples (direct count)
  bool gappy = false;              // through-plane coverage dips between slices (build_psf)
  StackPsf psf;                    // separable factors (offsets into the float table)
  float* y_dev = nullptr;          // device copy of the slices (until extract)
  int64_t y_off = 0;               // offset in the concatenated stack buffer
};

struct HostPatch {
  int32_t stack, x0, y0, z0, sx, sy, sz;
};

// Natural groups of one tiling candidate: geometry independent, built once per candidate and
// cached (keyed by TU, TV, nseg, forward/backprojection); only bounding boxes depend on T.
struct NaturalGroups {
  int TU = 0, TV = 0, nseg = 0;
  bool fwd = false, sample = false;
  std::vector<MemberDev> mem;  // sorted by group
  std::vector<int32_t> start;  // group g = mem[start[g], start[g+1])
  int64_t max_r_bytes = 0, max_t_floats = 0;
};

// fp64 geometry of one local patch: voxel index of lattice point (U, V, c) of slice z is
// t0 + z Mz + U Qa + V Qb + c Qc
struct PatchGeo {
  double t0[3], Mz[3], Qa[3], Qb[3], Qc[3];
};

// ---- NCCL, loaded at pvr_comm_init (no link-time dependency) ----
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) { err = std::string("cannot dlopen libnccl.so.2: ") + dlerror(); return false; }
    GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
    AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
    CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
    GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
    ReduceScatter = (decltype(ReduceScatter))dlsym(h, "ncclReduceScatter");
    AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
    Send = (decltype(Send))dlsym(h, "ncclSend");
    Recv = (decltype(Recv))dlsym(h, "ncclRecv");
    GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
    GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
    CommGetAsyncError = (decltype(CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    CommAbort = (decltype(CommAbort))dlsym(h, "ncclCommAbort");
    if (!GetUniqueId || !CommInitRank || !AllReduce || !CommDestroy || !GetErrorString || !ReduceScatter ||
        !AllGather || !Send || !Recv || !GroupStart || !GroupEnd || !CommGetAsyncError || !CommAbort) {
      err = "libnccl is missing a required symbol";
      return false;
    }
    return true;
  }
};
Nccl g_nccl;

// PVR_TRACE=1: host-side phase timings of pvr_set_transforms on stderr (diagnostics only)
struct Trace {
  bool on = getenv("PVR_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what, cudaStream_t sync = nullptr) {
    if (!on) return;
    if (sync) cudaStreamSynchronize(sync);  // attribute the device work queued so far
    const auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[pvr] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

}  // namespace

struct pvr_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t aux = nullptr;       // set_transforms: the backprojection tables, beside coverage
  cudaEvent_t ev_geo = nullptr, ev_tab = nullptr;
  bool own_stream = false;
  int3 dims;
  int nxp = 0;  // row pitch of X and (A, C): nx rounded up to a multiple of 4 (TMA: 16-byte rows)
  double s, o[3];
  int64_t V, Vp;  // voxels; padded (A, C) entries
  int state = CREATED;
  bool poisoned = false;
  std::string err;
  // parameters
  // thresholds: readings Q24 / Q25 (SURVEY.md:652, 678)
  double delta = 150.0, tau_patch = 0.5, c0 = 0.9, tau_live = 0.99, tau_C = 1e-6, tau_obs = 0.01;
  int clamp = 1, psf_mode = 0, profile = 0;
  int bp_exact = kBpRim;  // backprojection tile precision (PVR_PARAM_BP_EXACT)
  int det = 0;            // PVR_PARAM_DETERMINISTIC
  double plan_budget = 1.0;  // PVR_PARAM_PLAN_BUDGET: fraction of the tile budgets planned for
  unsigned long long* ACd = nullptr;  // deterministic mode: int64 (A, C) accumulators [4 Vp]
  VolPatch* vpat = nullptr;     // volume-space PSF mode: per local patch geometry
  float* vin = nullptr;         // volume-space PSF mode: per pixel row normaliser sum_{grid} psi
  bool explicit_patches = false;  // patches from pvr_set_patches / superpixels (not windows)
  double s2floor = 1e-6, nsigma = 3.0, quality = 1.0;
  // stacks / patches
  std::vector<HostStack> stacks;
  std::vector<float> psf_tab;        // separable PSF factors of all stacks
  std::vector<HostPatch> patches;    // global list
  std::vector<int64_t> pix0_global;  // [M+1]
  int64_t M = 0, P = 0;
  int64_t first = 0, nloc = 0, first_pix = 0, nloc_pix = 0;
  int64_t samples_obs = 0;           // observed pixels x S per iteration (all ranks)
  // work plans of the lattice kernels (forward / coverage, and backprojection)
  struct Plan {
    int TU = 16, TV = 16, nseg = 1;
    int ngroups = 0, nsplit = 0;
    int max_nm = kMaxGroupMembers;  // most members in one group (the table kernel's segment width)
    int tile_words = 0, r_bytes = 0, t_floats = 0;
    MemberDev* mem = nullptr;
    GroupDev* grp = nullptr;
    size_t mem_cap = 0, grp_cap = 0;
    int64_t nmem = 0;
    void* btab = nullptr;          // backprojection member / group tables (geometry only)
    size_t btab_cap = 0, btab_goff = 0;
    uint64_t btab_epoch = 0;       // geo_epoch the tables were built for (0: never)
  } fplan, bplan, iplan;
  uint64_t geo_epoch = 1;          // bumped whenever patch geometry or a plan changes  // forward/coverage, backprojection, init backprojection (hi/lo)
  bool iplan_valid = false;     // the init plan is built lazily by pvr_init_volume
  std::vector<PatchGeo> geo;    // composed geometry of the local patches (last set_transforms)
  std::vector<double> Tloc;     // the local patches' transforms (last set_transforms), [nloc][12]
  std::vector<PatchGeo> geo_next;  // set_transforms scratch, swapped with geo / Tloc
  std::vector<double> T_next;
  RegPatch* regP = nullptr;     // f1: device per-patch registration geometry
  size_t regP_cap = 0;
  std::vector<std::unique_ptr<NaturalGroups>> ngcache;  // geometry-free group lists
  std::vector<int> fbox;   // forward TMA box shapes (width, height) of the current plan
  char* tmaps = nullptr;   // device: CUtensorMap [2 X buffers][box shapes]
  size_t tmaps_cap = 0;
  // comm: NCCL (pvr_comm_init) or a host-collective callback (pvr_comm_init_host)
  int nranks = 1, rank = 0;
  ncclComm_t comm = nullptr;
  pvr_host_collective_fn host_fn = nullptr;
  void* host_user = nullptr;
  char* host_buf = nullptr;     // pinned staging buffer of the host collectives
  PatchDev* pd_host = nullptr;  // pinned staging of the composed patch geometry (set_transforms)
  int64_t pd_host_n = 0;
  cudaEvent_t pd_copied = nullptr;  // its last host -> device copy (reuse waits on it)
  size_t host_cap = 0;
  int exchange = PVR_EXCHANGE_ALLREDUCE;  // C2 scheme (PVR_PARAM_EXCHANGE)
  double comm_timeout = 300.0;  // seconds an NCCL wait may take before the communicator is aborted
  int nzp = 0;                  // planes of X / (A, C) allocated: nz rounded up to nranks slabs
  int z0 = 0, z1 = 0;           // this rank's slab of planes (PVR_EXCHANGE_SLABS)
  // device buffers
  float* X[2] = {nullptr, nullptr};
  int cur = 0;
  float2* AC = nullptr;
  float *e = nullptr, *p = nullptr, *kap = nullptr, *pbar = nullptr, *w = nullptr;
  float* ys = nullptr;
  float* tab = nullptr;
  StackPsf* psf = nullptr;
  PatchDev* pdev = nullptr;
  double* partials = nullptr;
  double* rpart = nullptr;      // f4 multi-round EM: per-patch E-step partials [nloc][3]
  int* replan_buf = nullptr;    // device replan results {fwd max vox, fail, bp max vox, fail}
  int* fbox_dev = nullptr;      // the forward box shapes (width, height) for k_replan
  int em_rounds = 1;
  double em_tol = 1e-6;
  int patch_mixture = 0;        // f4 two-Gaussian patch classification (reading Q31)
  int32_t* nlivep = nullptr;    // live pixels per local patch (mixture validity)
  uint8_t* mask = nullptr;      // f3: per-pixel patch mask of the local shard (NULL = all)
  std::vector<uint8_t> mask_host;  // its host copy: the planners drop fully masked member tiles
  EmDev* em = nullptr;
  // stats; with PVR_PARAM_PROFILE every iteration records EV_N events into a slot of the
  // pool, drained (synchronised) only by pvr_get_stats or when the pool is large
  pvr_stats st;
  std::vector<std::vector<cudaEvent_t>> prof_free, prof_pending;
};

namespace {

const char* kVersion = "pvr-b200 0.2 (sm_100a, lattice kernels)";
thread_local std::string g_static_err = "no context";

pvr_status fail(pvr_ctx* c, pvr_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) {
    c->err = buf;
    if (s == PVR_ERR_CUDA || s == PVR_ERR_NCCL) c->poisoned = true;
  } else {
    g_static_err = buf;
  }
  return s;
}

#define CUDA_TRY(c, call)                                                                  \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return fail((c), _e == cudaErrorMemoryAllocation ? PVR_ERR_OOM : PVR_ERR_CUDA,       \
                  "%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

#define CHECK_LAUNCH(c) CUDA_TRY(c, cudaGetLastError())

#define GUARD(c)                                                                   \
  do {                                                                             \
    if (!(c)) return fail(nullptr, PVR_ERR_ARG, "null context");                   \
    if ((c)->poisoned) return fail((c), PVR_ERR_STATE, "context poisoned: %s", (c)->err.c_str()); \
    cudaSetDevice((c)->device);                                                    \
  } while (0)

bool is_device_ptr(const void* ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

double norm3(const double* a) { return std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]); }

// Taylor-series sinc: 1 - x^2/3! + x^4/5! - ..., stopped when the next term is
// below an absolute 1e-16 (reading Q4).
double taylor_sinc(double x) {
  const double x2 = x * x;
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 200; ++k) {
    term *= -x2 / ((2.0 * k) * (2.0 * k + 1.0));
    if (std::fabs(term) < 1e-16) break;
    sum += term;
  }
  return sum;
}

int psf_steps(double pitch, double s, double q) {  // reading Q5: n = max(2, ceil(q pitch / s))
  int n = (int)std::ceil(q * pitch / s - 1e-9);
  return std::max(2, n);
}

// Through-plane coverage of a stack: P(z) = sum_k sum_c tp(c) tent((z - k step - c h_w) / s)
// over one slice period in the middle of the stack. A stack whose coverage dips below 1/4 of
// its peak between slices (slice gaps, thin slices far apart) leaves cells of small confidence
// inside its footprint, so all its backprojection members get exact tiles (the border rule of
// build_natural covers the outer rim only).
bool stack_gappy(const HostStack& st, const std::vector<double>& tp, double hw, double s) {
  if (st.K < 2) return true;
  const double step = std::fabs(st.G[2] * st.w[0] + st.G[6] * st.w[1] + st.G[10] * st.w[2]);
  const int cmax = ((int)tp.size() - 1) / 2;
  double mn = 1e300, mx = 0.0;
  for (int i = 0; i < 64; ++i) {
    const double z = step * i / 64.0;
    double v = 0.0;
    for (int k = -4; k <= 4; ++k)
      for (int c = -cmax; c <= cmax; ++c) {
        const double t = std::fabs(z - k * step - c * hw) / s;
        if (t < 1.0) v += tp[c + cmax] * (1.0 - t);
      }
    mn = std::min(mn, v);
    mx = std::max(mx, v);
  }
  return !(mn >= 0.25 * mx);
}

// PSF of one stack: psi(a,b,c) ~ sinc(pi R) exp(-(c h_w)^2 / 2 sw^2) with
// R = |(a/n_u, b/n_v)| < 1 (main lobe, Q2), |c h_w| <= nsigma sw (Q3), normalised to 1.
// Stored as its two factors ip(a,b) = sinc / sum sinc and tp(c) = g / sum g, whose product is
// psi; the product is checked in fp64 against the directly normalised table.
pvr_status build_psf(pvr_ctx* c, HostStack& st) {
  StackPsf& ps = st.psf;
  if (c->psf_mode == 1 || c->psf_mode == 2) {  // delta PSF (tests) / volume-space PSF (volpsf.cu)
    ps.nu = ps.nv = 1; ps.ru = ps.rv = 0; ps.cmax = 0;
    ps.ip0 = (int)c->psf_tab.size(); c->psf_tab.push_back(1.0f);
    ps.tp0 = (int)c->psf_tab.size(); c->psf_tab.push_back(1.0f);
    ps.tpmax = 1.0f;
    st.S = 1;
    const double c0[3] = {st.G[0], st.G[4], st.G[8]}, c1[3] = {st.G[1], st.G[5], st.G[9]};
    st.h[0] = norm3(c0); st.h[1] = norm3(c1); st.h[2] = 0.0;  // Qa = Mu, Qb = Mv
    st.gappy = stack_gappy(st, std::vector<double>{1.0}, 0.0, c->s);
    return PVR_OK;
  }
  const double c0[3] = {st.G[0], st.G[4], st.G[8]}, c1[3] = {st.G[1], st.G[5], st.G[9]};
  const double px = norm3(c0), py = norm3(c1);
  const int nu = psf_steps(px, c->s, c->quality), nv = psf_steps(py, c->s, c->quality),
            nw = psf_steps(st.theta, c->s, c->quality);
  st.h[0] = px / nu;
  st.h[1] = py / nv;
  st.h[2] = st.theta / nw;
  const double sw = st.theta / (2.0 * std::sqrt(2.0 * std::log(2.0)));
  int cmax = 0;
  while (std::fabs((cmax + 1) * st.h[2]) <= c->nsigma * sw) ++cmax;
  const int ru = nu - 1, rv = nv - 1;
  if ((2 * ru + 1) * (2 * rv + 1) > 81 || 2 * cmax + 1 > 256)
    return fail(c, PVR_ERR_ARG, "PSF lattice too large (in-plane %dx%d, through-plane %d)", 2 * ru + 1,
                2 * rv + 1, 2 * cmax + 1);
  std::vector<double> ip((2 * ru + 1) * (2 * rv + 1), 0.0), tp(2 * cmax + 1);
  double sip = 0.0, stp = 0.0;
  int disk = 0;
  for (int b = -rv; b <= rv; ++b)
    for (int a = -ru; a <= ru; ++a) {
      const double R = std::sqrt((double)a * a / ((double)nu * nu) + (double)b * b / ((double)nv * nv));
      if (!(R < 1.0)) continue;
      const double v = taylor_sinc(M_PI * R);
      ip[(b + rv) * (2 * ru + 1) + (a + ru)] = v;
      sip += v;
      ++disk;
    }
  for (int cc = -cmax; cc <= cmax; ++cc) {
    const double zc = cc * st.h[2];
    tp[cc + cmax] = std::exp(-zc * zc / (2.0 * sw * sw));
    stp += tp[cc + cmax];
  }
  // separability check against the directly normalised psi (same support, same values)
  double total = 0.0;
  for (double a : ip)
    for (double b : tp) total += a * b;
  double worst = 0.0;
  for (size_t i = 0; i < ip.size(); ++i)
    for (size_t k = 0; k < tp.size(); ++k)
      worst = std::max(worst, std::fabs(ip[i] * tp[k] / total - (ip[i] / sip) * (tp[k] / stp)));
  if (worst > 1e-15) return fail(c, PVR_ERR_ARG, "PSF factorisation check failed (%g)", worst);
  ps.nu = nu; ps.nv = nv; ps.ru = ru; ps.rv = rv; ps.cmax = cmax;
  ps.ip0 = (int)c->psf_tab.size();
  for (double v : ip) c->psf_tab.push_back((float)(v / sip));
  ps.tp0 = (int)c->psf_tab.size();
  double tpmax = 0.0;
  for (double v : tp) {
    c->psf_tab.push_back((float)(v / stp));
    tpmax = std::max(tpmax, v / stp);
  }
  ps.tpmax = (float)tpmax;
  st.S = disk * (2 * cmax + 1);
  st.gappy = stack_gappy(st, tp, st.h[2], c->s);
  return PVR_OK;
}

// Square windows along one axis; the last one is clamped to the edge (Q22).
std::vector<int> windows(int dim, int size, int stride) {
  std::vector<int> out;
  for (int x = 0; x + size <= dim; x += stride) out.push_back(x);
  if (!out.empty() && out.back() + size < dim) out.push_back(dim - size);
  return out;
}

Params make_params(const pvr_ctx* c) {
  Params p;
  p.tau_live = (float)c->tau_live;
  p.tau_obs = (float)c->tau_obs;
  p.tau_C = (float)c->tau_C;
  p.tau_patch = (float)c->tau_patch;
  p.c0 = (float)c->c0;
  p.delta = (float)c->delta;
  p.clamp = c->clamp;
  p.det = c->det;
  return p;
}

LatticeArgs lattice_args(const pvr_ctx* c, const pvr_ctx::Plan& pl) {
  LatticeArgs a;
  a.P = c->pdev;
  a.psf = c->psf;
  a.tab = c->tab;
  a.mem = pl.mem;
  a.grp = pl.grp;
  a.ngroups = pl.ngroups;
  a.n = c->dims;
  a.nxp = c->nxp;
  a.ys = c->ys;
  a.mask = c->mask;
  a.prm = make_params(c);
  a.det_scale = c->em ? c->em->det_scale : nullptr;
  a.ACd = c->ACd;
  a.ftab = pl.btab;  // forward plan: its member rows (build_fwd_table); unused by the others
  a.fgoff = pl.btab_goff;
  return a;
}

// The forward plan's member rows and group headers (k_fwd_table), rebuilt when the geometry or
// the plan changed (the forward plan keeps them in its btab fields).
pvr_status build_fwd_table(pvr_ctx* c) {
  pvr_ctx::Plan& pl = c->fplan;
  if (pl.ngroups <= 0 || pl.btab_epoch == c->geo_epoch) return PVR_OK;
  size_t goff = 0;
  const size_t bytes = fwd_table_bytes(pl.nmem, pl.ngroups, &goff);
  if (bytes > pl.btab_cap) {
    if (pl.btab) cudaFree(pl.btab);
    pl.btab = nullptr;
    pl.btab_cap = 0;
    CUDA_TRY(c, cudaMalloc(&pl.btab, bytes));
    pl.btab_cap = bytes;
  }
  pl.btab_goff = goff;
  launch_fwd_table(c->stream, lattice_args(c, pl), pl.btab, goff, pl.max_nm);
  CHECK_LAUNCH(c);
  pl.btab_epoch = c->geo_epoch;
  c->st.kernel_launches += 1;
  return PVR_OK;
}

pvr_status nccl_check(pvr_ctx* c, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return PVR_OK;
  return fail(c, PVR_ERR_NCCL, "%s: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
}

// ---- collectives: NCCL on the context's stream, or the host-collective callback on a pinned
// staging copy (pvr_comm_init_host). All are no-ops on one rank.
pvr_status coll(pvr_ctx* c, void* dev, int64_t count, int dtype, int op) {
  if (c->nranks <= 1 || count <= 0) return PVR_OK;
  const size_t esz = dtype == PVR_DT_F32 ? 4 : 8;
  const size_t bytes = (op == PVR_COLL_ALLGATHER ? (size_t)c->nranks : 1) * (size_t)count * esz;
  if (c->host_fn) {
    if (bytes > c->host_cap) {
      if (c->host_buf) cudaFreeHost(c->host_buf);
      c->host_buf = nullptr;
      c->host_cap = 0;
      CUDA_TRY(c, cudaMallocHost(&c->host_buf, bytes));
      c->host_cap = bytes;
    }
    CUDA_TRY(c, cudaMemcpyAsync(c->host_buf, dev, bytes, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->host_fn(c->host_user, c->host_buf, count, dtype, op) != 0)
      return fail(c, PVR_ERR_NCCL, "host collective (op %d, %lld elements) failed", op, (long long)count);
    CUDA_TRY(c, cudaMemcpyAsync(dev, c->host_buf, bytes, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));  // the staging buffer is reused by the next call
    return PVR_OK;
  }
  const ncclDataType_t t = dtype == PVR_DT_F32 ? ncclFloat32 : dtype == PVR_DT_F64 ? ncclFloat64 : ncclInt64;
  if (op == PVR_COLL_ALLGATHER)
    return nccl_check(c, g_nccl.AllGather(static_cast<char*>(dev) + (size_t)c->rank * count * esz, dev, count, t,
                                          c->comm, c->stream),
                      "ncclAllGather");
  return nccl_check(c, g_nccl.AllReduce(dev, dev, count, t, op == PVR_COLL_ALLREDUCE_MAX ? ncclMax : ncclSum,
                                        c->comm, c->stream),
                    "ncclAllReduce");
}

// Wait for the context's stream. With NCCL, poll the communicator's asynchronous error state
// while waiting and abort it (ncclCommAbort) on an error or after PVR_PARAM_COMM_TIMEOUT
// seconds, so a failed or hung peer poisons the context instead of hanging the call.
pvr_status comm_wait(pvr_ctx* c) {
  if (c->nranks <= 1 || !c->comm) {
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return PVR_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(c->stream);
    if (q == cudaSuccess) return PVR_OK;
    if (q != cudaErrorNotReady) return fail(c, PVR_ERR_CUDA, "stream: %s", cudaGetErrorString(q));
    ncclResult_t ar = ncclSuccess;
    g_nccl.CommGetAsyncError(c->comm, &ar);
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if ((ar != ncclSuccess && ar != ncclInProgress) || dt > c->comm_timeout) {
      g_nccl.CommAbort(c->comm);
      c->comm = nullptr;
      return fail(c, PVR_ERR_NCCL, "NCCL %s after %.1f s: communicator aborted",
                  ar != ncclSuccess && ar != ncclInProgress ? g_nccl.GetErrorString(ar) : "timeout", dt);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

// EM statistics allreduce (C1): SUM over stats[0..2], MAX over stats[3..4].
pvr_status allreduce_stats(pvr_ctx* c) {
  pvr_status r = coll(c, c->em->stats, 3, PVR_DT_F64, PVR_COLL_ALLREDUCE_SUM);
  if (r != PVR_OK) return r;
  return coll(c, c->em->stats + 3, 2, PVR_DT_F64, PVR_COLL_ALLREDUCE_MAX);
}

// f4 multi-round EM: SUM of the E-step partials {sum p e^2, sum p, LL} before each M-step.
pvr_status allreduce_stats2(pvr_ctx* c) { return coll(c, c->em->stats2, 3, PVR_DT_F64, PVR_COLL_ALLREDUCE_SUM); }

// f4 patch mixture sums: stage 0 = {n, sum pbar, sum pbar^2 | max, -min}; 1 = 7 round sums.
constexpr int kMixRounds = 50;
pvr_status allreduce_mix(pvr_ctx* c, int stage) {
  double* s = c->em->mix_stats;
  if (stage == 0) {
    pvr_status r = coll(c, s, 3, PVR_DT_F64, PVR_COLL_ALLREDUCE_SUM);
    if (r != PVR_OK) return r;
    return coll(c, s + 3, 2, PVR_DT_F64, PVR_COLL_ALLREDUCE_MAX);
  }
  return coll(c, s, 7, PVR_DT_F64, PVR_COLL_ALLREDUCE_SUM);
}

// Addon / confidence allreduce (C2): SUM over the interleaved, row-padded (A, C) volume.
pvr_status allreduce_ac(pvr_ctx* c) { return coll(c, c->AC, c->Vp * 2, PVR_DT_F32, PVR_COLL_ALLREDUCE_SUM); }

// The iteration's (A, C) exchange (PVR_PARAM_EXCHANGE). Slabs with NCCL: reduce-scatter of
// the z slabs (in place) and one halo plane from each neighbour (ncclSend / ncclRecv), so each
// rank holds the reduced (A, C) of its slab and the planes its update stencil reads; with the
// host transport the same slab update runs on an allreduced (A, C). Averaging: no exchange.
pvr_status exchange_ac(pvr_ctx* c) {
  if (c->nranks <= 1 || c->exchange == PVR_EXCHANGE_AVERAGE) return PVR_OK;
  if (c->exchange == PVR_EXCHANGE_ALLREDUCE || c->host_fn) return allreduce_ac(c);
  const size_t plane = (size_t)c->nxp * c->dims.y * 2;  // floats per (A, C) plane
  const int slab = c->nzp / c->nranks;
  float* ac = reinterpret_cast<float*>(c->AC);
  pvr_status r = nccl_check(c, g_nccl.ReduceScatter(ac, ac + (size_t)c->rank * slab * plane, slab * plane, ncclFloat32,
                                                    ncclSum, c->comm, c->stream),
                            "ncclReduceScatter(A,C)");
  if (r != PVR_OK) return r;
  r = nccl_check(c, g_nccl.GroupStart(), "ncclGroupStart");
  if (r != PVR_OK) return r;
  if (c->rank > 0) {
    g_nccl.Send(ac + (size_t)c->z0 * plane, plane, ncclFloat32, c->rank - 1, c->comm, c->stream);
    g_nccl.Recv(ac + (size_t)(c->z0 - 1) * plane, plane, ncclFloat32, c->rank - 1, c->comm, c->stream);
  }
  if (c->rank < c->nranks - 1) {
    g_nccl.Send(ac + (size_t)(c->z1 - 1) * plane, plane, ncclFloat32, c->rank + 1, c->comm, c->stream);
    g_nccl.Recv(ac + (size_t)c->z1 * plane, plane, ncclFloat32, c->rank + 1, c->comm, c->stream);
  }
  return nccl_check(c, g_nccl.GroupEnd(), "ncclGroupEnd (halo planes)");
}

// After the update: slabs -> all-gather the new X (in place); averaging -> X = mean over ranks.
pvr_status exchange_x(pvr_ctx* c, float* X2) {
  if (c->nranks <= 1 || c->exchange == PVR_EXCHANGE_ALLREDUCE) return PVR_OK;
  const int64_t plane = (int64_t)c->nxp * c->dims.y;
  if (c->exchange == PVR_EXCHANGE_SLABS)
    return coll(c, X2, (int64_t)(c->nzp / c->nranks) * plane, PVR_DT_F32, PVR_COLL_ALLGATHER);
  pvr_status r = coll(c, X2, (int64_t)c->nzp * plane, PVR_DT_F32, PVR_COLL_ALLREDUCE_SUM);
  if (r != PVR_OK) return r;
  launch_scale(c->stream, X2, (int64_t)c->nzp * plane, 1.0f / (float)c->nranks);
  return PVR_OK;
}

void free_dev(pvr_ctx* c) {
  for (auto& s : c->stacks)
    if (s.y_dev) cudaFree(s.y_dev), s.y_dev = nullptr;
  void* ptrs[] = {c->X[0], c->X[1], c->AC, c->e, c->p, c->kap, c->pbar, c->w, c->ys, c->tab,
                  c->psf, c->pdev, c->fplan.mem, c->fplan.grp, c->bplan.mem, c->bplan.grp,
                  c->iplan.mem, c->iplan.grp, c->bplan.btab, c->iplan.btab, c->fplan.btab,
                  c->partials, c->em, c->tmaps, c->regP, c->rpart, c->replan_buf, c->fbox_dev, c->nlivep, c->mask,
                  c->ACd, c->vpat, c->vin};
  for (void* q : ptrs)
    if (q) cudaFree(q);
}

// ---- work plans ----------------------------------------------------------------------
// A member is a tile of tu x tv pixels of one slice of one patch (backprojection members also
// carry a through-plane lattice segment [c0, c1]). Members that cover the same stack pixels
// (overlapping patches of one stack) form a group: one CTA, one shared voxel tile.
// Owned fine-lattice range of a backprojection member (must match owned_range() in lattice.cu).
void owned(const MemberDev& m, const HostPatch& hp, const StackPsf& ps, int& Ulo, int& Uhi, int& Vlo,
           int& Vhi) {
  Ulo = ps.nu * m.u0 - ps.ru;
  Uhi = (m.u0 + m.tu >= hp.sx) ? ps.nu * (hp.sx - 1) + ps.ru + 1 : ps.nu * (m.u0 + m.tu) - ps.ru;
  Vlo = ps.nv * m.v0 - ps.rv;
  Vhi = (m.v0 + m.tv >= hp.sy) ? ps.nv * (hp.sy - 1) + ps.rv + 1 : ps.nv * (m.v0 + m.tv) - ps.rv;
}

// Lattice range a member touches: forward = all lattice points its pixels read (halo'd),
// backprojection = its owned points and c segment.
void member_range(const MemberDev& m, const HostPatch& hp, const StackPsf& ps, bool fwd, int& Ulo,
                  int& Uhi, int& Vlo, int& Vhi) {
  if (fwd) {
    Ulo = ps.nu * m.u0 - ps.ru;
    Uhi = ps.nu * (m.u0 + m.tu - 1) + ps.ru + 1;
    Vlo = ps.nv * m.v0 - ps.rv;
    Vhi = ps.nv * (m.v0 + m.tv - 1) + ps.rv + 1;
  } else {
    owned(m, hp, ps, Ulo, Uhi, Vlo, Vhi);
  }
}

// Voxel bbox [lo, hi] (inclusive, not clipped to the grid) of every trilinear corner the
// member's lattice points touch, from the fp64 geometry (margin 1e-3 voxel >> fp32 error).
void member_bbox(const MemberDev& m, const HostPatch& hp, const StackPsf& ps, const PatchGeo& g,
                 bool fwd, int lo[3], int hi[3]) {
  int Ulo, Uhi, Vlo, Vhi;
  member_range(m, hp, ps, fwd, Ulo, Uhi, Vlo, Vhi);
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  for (int iu = 0; iu < 2; ++iu)
    for (int iv = 0; iv < 2; ++iv)
      for (int ic = 0; ic < 2; ++ic) {
        const double U = iu ? Uhi - 1 : Ulo, V = iv ? Vhi - 1 : Vlo, C = ic ? m.c1 : m.c0;
        for (int d = 0; d < 3; ++d) {
          const double x = g.t0[d] + m.z * g.Mz[d] + U * g.Qa[d] + V * g.Qb[d] + C * g.Qc[d];
          mn[d] = std::min(mn[d], x);
          mx[d] = std::max(mx[d], x);
        }
      }
  for (int d = 0; d < 3; ++d) {
    lo[d] = (int)std::floor(mn[d] - 1e-3);
    hi[d] = (int)std::floor(mx[d] + 1e-3) + 1;
  }
}

int64_t r_bytes_of(const MemberDev& m, const StackPsf& ps) {
  // the member's feeding pixels (its tile and up to ru / nu + 1 around) and the R block's
  // one-pixel zero border (lattice.cu k_bp_table)
  return (int64_t)(m.tu + 2 * ps.ru / ps.nu + 4) * (m.tv + 2 * ps.rv / ps.nv + 4) * 8;
}

void build_natural(const pvr_ctx* c, const std::vector<int64_t>& which, int TU, int TV, int nseg, bool fwd,
                   NaturalGroups& ng) {
  ng.TU = TU; ng.TV = TV; ng.nseg = nseg; ng.fwd = fwd;
  std::vector<MemberDev> mem;
  std::vector<std::pair<uint64_t, int32_t>> keys;
  // f3 (reading Q32): a member whose pixels are all masked out is never observed (kappa, e and
  // R stay 0) and is not planned at all. A backprojection member's owned lattice points also
  // collect the pixels one beside its tile (ru < nu: owned_range in lattice.cu), so its test
  // covers the tile grown by one pixel
  const uint8_t* mk = c->mask_host.empty() ? nullptr : c->mask_host.data();
  const int grow = fwd ? 0 : 1;
  for (int64_t s : which) {
    const HostPatch& hp = c->patches[c->first + s];
    const StackPsf& ps = c->stacks[hp.stack].psf;
    const int ntp = 2 * ps.cmax + 1, seg = (ntp + nseg - 1) / nseg;
    const int64_t pbase = c->pix0_global[c->first + s] - c->first_pix;
    auto masked_out = [&](int z, int u0, int v0) {
      if (!mk) return false;
      for (int v = std::max(0, v0 - grow); v < std::min(v0 + TV + grow, hp.sy); ++v)
        for (int u = std::max(0, u0 - grow); u < std::min(u0 + TU + grow, hp.sx); ++u)
          if (mk[pbase + ((int64_t)z * hp.sy + v) * hp.sx + u]) return false;
      return true;
    };
    // Rim members (exact backprojection tiles, GroupDev::exact): cells of small confidence lie at
    // the rim of the coverage, which only these members reach: a tile on its stack's border
    // (windows of extract_patches cover every pixel of the stack, so inner patch borders are
    // covered by the neighbouring windows) or, for explicit patches, on its patch's border or
    // with a masked-out pixel in its grown tile; every member of a stack with slice gaps
    // (stack_gappy) or with PVR_PARAM_BP_EXACT = 2. Footprints that leave the grid are added
    // per geometry (size_groups, k_replan).
    const HostStack& hst = c->stacks[hp.stack];
    auto rim_member = [&](const MemberDev& m, const HostPatch& p) {
      if (c->bp_exact == kBpAll || hst.gappy) return true;
      if (c->bp_exact == kBpSingle) return false;
      if (c->explicit_patches) {
        if (m.u0 == 0 || m.v0 == 0 || m.u0 + m.tu >= p.sx || m.v0 + m.tv >= p.sy || m.z == 0 || m.z == p.sz - 1)
          return true;
        if (mk)
          for (int v = std::max(0, m.v0 - 1); v < std::min(m.v0 + m.tv + 1, p.sy); ++v)
            for (int u = std::max(0, m.u0 - 1); u < std::min(m.u0 + m.tu + 1, p.sx); ++u)
              if (!mk[pbase + ((int64_t)m.z * p.sy + v) * p.sx + u]) return true;
        return false;
      }
      return p.x0 + m.u0 == 0 || p.y0 + m.v0 == 0 || p.x0 + m.u0 + m.tu >= hst.W || p.y0 + m.v0 + m.tv >= hst.H ||
             p.z0 + m.z == 0 || p.z0 + m.z == hst.K - 1;
    };
    for (int z = 0; z < hp.sz; ++z)
      for (int v0 = 0; v0 < hp.sy; v0 += TV)
        for (int u0 = 0; u0 < hp.sx; u0 += TU) {
          if (masked_out(z, u0, v0)) continue;
          for (int k = 0; k < (fwd ? 1 : nseg); ++k) {
            const int c0 = -ps.cmax + k * seg, c1 = fwd ? ps.cmax : std::min(ps.cmax, c0 + seg - 1);
            if (c0 > c1) continue;
            MemberDev m{(int32_t)s, z, u0, v0, std::min(TU, hp.sx - u0), std::min(TV, hp.sy - v0), c0, c1, 0};
            if (!fwd && rim_member(m, hp)) m.flags |= kMemberRim;
            // group key: stack | slice | c segment | stack row | stack column | tile shape
            const uint64_t key = ((uint64_t)hp.stack << 58) | ((uint64_t)(hp.z0 + z) << 44) |
                                 ((uint64_t)k << 38) | ((uint64_t)(hp.y0 + v0) << 24) |
                                 ((uint64_t)(hp.x0 + u0) << 10) | ((uint64_t)m.tu << 5) | (uint64_t)m.tv;
            keys.emplace_back(key, (int32_t)mem.size());
            mem.push_back(m);
          }
        }
  }
  std::sort(keys.begin(), keys.end());
  ng.mem.clear();
  ng.start.clear();
  ng.max_r_bytes = ng.max_t_floats = 0;
  size_t i = 0;
  while (i < keys.size()) {
    size_t j = i;
    while (j < keys.size() && keys[j].first == keys[i].first) ++j;
    int64_t rb = 0, tsum = 0;
    ng.start.push_back((int32_t)ng.mem.size());
    for (size_t k = i; k < j; ++k) {
      const MemberDev& m = mem[keys[k].second];
      const StackPsf& ps = c->stacks[c->patches[c->first + m.patch].stack].psf;
      const int64_t b = r_bytes_of(m, ps);
      const int64_t tf = (int64_t)(ps.nu * (m.tu - 1) + 2 * ps.ru + 1) * (ps.nv * (m.tv - 1) + 2 * ps.rv + 1);
      // split by the R buffer budget (backprojection) / the lattice buffer and member count
      // (forward: all members' T values are resident at once)
      const bool full = fwd ? (k > i && (tsum + tf > kFwdTBytes / 4 || (int64_t)ng.mem.size() - ng.start.back() >= kMaxGroupMembers))
                            : (k > i && (rb + b > kRBytes || (int64_t)ng.mem.size() - ng.start.back() >= kMaxGroupMembers));
      if (full) {
        ng.max_r_bytes = std::max(ng.max_r_bytes, rb);
        ng.max_t_floats = std::max(ng.max_t_floats, tsum);
        ng.start.push_back((int32_t)ng.mem.size());
        rb = 0;
        tsum = 0;
      }
      rb += b;
      tsum += tf;
      ng.mem.push_back(m);
    }
    ng.max_r_bytes = std::max(ng.max_r_bytes, rb);
    ng.max_t_floats = std::max(ng.max_t_floats, tsum);
    i = j;
  }
  ng.start.push_back((int32_t)ng.mem.size());
}

struct PlanBuild {
  std::vector<MemberDev> mem;  // group-sorted (groups over the budget are split into singles)
  std::vector<GroupDev> grp;
  int64_t max_tile_vox = 0, max_r_bytes = 0, max_t_floats = 0;
  int nsplit = 0;              // natural groups split into single members
  bool all_fit = true;         // every single member fits the tile budget
  double fit_frac = 0.0;       // fraction of natural groups that fit whole
  double half_frac = 0.0;      // ... that fit whole or as two groups of half-tile members
};

// Bounding boxes for the current transforms and the final group list of one plan.
// kind 0: forward / coverage (4 B per voxel of staged X), 1: backprojection in the iterations
// (8 B: one int32 per quantity), 2: init backprojection (16 B: hi/lo pairs).
// All per-member and per-group passes run in parallel (OpenMP); the output is deterministic.
// forward plans: group halving too, and a tile size accepted at >= PVR_FWD_HALVE_MIN whole
// (>= 90% whole or halved): c4's 16 x 8 forward tiles fit 67% whole, 98% halved (forward 14.45
// -> 13.56 ms); c3 unchanged (99% whole)
#ifndef PVR_FWD_HALVE
#define PVR_FWD_HALVE 1
#endif
#ifndef PVR_BP_HALVE_MIN
#define PVR_BP_HALVE_MIN 0.75
#endif
#ifndef PVR_FWD_HALVE_MIN
#define PVR_FWD_HALVE_MIN 0.6
#endif
void size_groups(const pvr_ctx* c, const std::vector<PatchGeo>& geo, const NaturalGroups& ng, int kind,
                 PlanBuild& out) {
  const bool fwd = kind == 0;
  Trace tr;
  // the iteration backprojection plans to 90% of its tile budget: the device re-plan of a
  // later set_transforms (k_replan) accepts growth up to 100% (and splits a group that grew
  // past it into single-member groups) before falling back here
  // shared-memory budget in bytes: forward 4 B per staged voxel; backprojection 16 B per cell
  // for exact groups (hi / lo words), 8 B for single-word groups; the init plan is all exact
  const int64_t byte_budget = (int64_t)(c->plan_budget *
                                        (fwd ? kFwdTileBytes : kind == 1 ? (int64_t)kBpTileBytes * 9 / 10 : kBpTileBytes));
  // member pool: the natural members, then sub-members made by splitting a member whose own
  // footprint does not fit (below); mlo / mhi: their fp64 voxel bboxes
  std::vector<MemberDev> pool(ng.mem);
  const int64_t nm = (int64_t)ng.mem.size();
  std::vector<int32_t> mlo(3 * nm), mhi(3 * nm);
  std::vector<uint8_t> msup(nm);  // backprojection: the full PSF support of every pixel feeding the member is in the grid
  const int n3[3] = {c->dims.x, c->dims.y, c->dims.z};
  auto bbox_of = [&](const MemberDev& m, int* lo, int* hi) -> uint8_t {
    const HostPatch& hp = c->patches[c->first + m.patch];
    const StackPsf& ps = c->stacks[hp.stack].psf;
    member_bbox(m, hp, ps, geo[m.patch], fwd, lo, hi);
    if (fwd) return 1;
    // the pixels feeding the member's lines reach one pixel past its tile (R range, lattice.cu
    // owned_range); their whole supports (every in-plane and through-plane sample) in the grid
    // means kappa = 1 for all of them, so no term of the group carries a 1/kappa > 1
    MemberDev e = m;
    e.u0 = std::max(0, m.u0 - 1);
    e.tu = std::min(hp.sx, m.u0 + m.tu + 1) - e.u0;
    e.v0 = std::max(0, m.v0 - 1);
    e.tv = std::min(hp.sy, m.v0 + m.tv + 1) - e.v0;
    e.c0 = -ps.cmax;
    e.c1 = ps.cmax;
    int sl[3], sh[3];
    member_bbox(e, hp, ps, geo[m.patch], true, sl, sh);
    for (int d = 0; d < 3; ++d)
      if (sl[d] < 0 || sh[d] > n3[d] - 1) return 0;
    return 1;
  };
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nm; ++i) msup[i] = bbox_of(ng.mem[i], &mlo[3 * i], &mhi[3 * i]);
  tr.mark("    member bboxes");
  // union bbox of the pool members listed in ix[0, n) -> tile box g (m0 / nm set by the caller)
  auto group = [&](const int32_t* ix, int n, GroupDev& g) {
    int lo[3] = {1 << 30, 1 << 30, 1 << 30}, hi[3] = {-(1 << 30), -(1 << 30), -(1 << 30)};
    int rim = 0, sup = 1;
    for (int k = 0; k < n; ++k) {
      const int i = ix[k];
      for (int d = 0; d < 3; ++d) {
        lo[d] = std::min(lo[d], mlo[3 * i + d]);
        hi[d] = std::max(hi[d], mhi[3 * i + d]);
      }
      rim |= pool[i].flags & kMemberRim;
      sup &= msup[i];
    }
    g.m0 = 0;
    g.nm = n;
    g.tmap = 0;
    g.interior = 1;
    for (int d = 0; d < 3; ++d)
      if (lo[d] < 0 || hi[d] > n3[d] - 1) g.interior = 0;
    g.exact = !fwd && (kind == 2 || c->det || c->bp_exact == kBpAll || (c->bp_exact == kBpRim && (rim || !sup)));
    if (fwd) {
      // TMA-staged X tile (lattice.cu): the box's x coordinate must be 16-byte aligned
      // (measured: a box starting at an x not a multiple of 4 floats faults with an illegal
      // instruction), rows of 4 x odd floats (16-byte TMA rows, 4 (mod 8) banks apart), z
      // slabs padded to 128 bytes
      lo[0] -= ((lo[0] % 4) + 4) % 4;
      int r = (hi[0] - lo[0] + 1 + 3) / 4;
      if (r % 2 == 0) ++r;
      for (int d = 0; d < 3; ++d) g.lo[d] = lo[d];
      g.dim[0] = 4 * r;
      g.dim[1] = hi[1] - lo[1] + 1;
      g.dim[2] = hi[2] - lo[2] + 1;
      return (int64_t)((g.dim[0] * g.dim[1] + 31) & ~31) * g.dim[2];
    }
    lo[0] -= ((lo[0] % 2) + 2) % 2;  // even x origin: 16-byte aligned flush pairs
    for (int d = 0; d < 3; ++d) g.lo[d] = lo[d];
    // odd row and plane pitches: lanes stepping along x, y or z hit different banks
    g.dim[0] = (hi[0] - lo[0] + 1) | 1;
    g.dim[1] = (hi[1] - lo[1] + 1) | 1;
    g.dim[2] = hi[2] - lo[2] + 1;
    return (int64_t)g.dim[0] * g.dim[1] * g.dim[2];
  };
  auto fits = [&](const GroupDev& g, int64_t vox) {
    if (!fwd && c->det) return vox * 4 <= (int64_t)(c->plan_budget * kBpDetPlane * (kind == 1 ? 9 : 10) / 10);
    return vox * (fwd ? 4 : g.exact ? 16 : 8) <= byte_budget;
  };
  // Outlying members of a natural group: a member whose footprint centre lies more than a
  // quarter of the group's median footprint extent (and 4 voxels) from the median centre on
  // some axis (a patch
  // misregistered far from the neighbours that share its stack pixels: c4's gross errors). Two
  // members that far apart are both taken out. Bit k of the mask: member a + k.
  auto outliers = [&](int a, int b) -> uint32_t {
    const int n = b - a;
    if (n < 2) return 0u;
    uint32_t mask = 0u;
    for (int d = 0; d < 3; ++d) {
      double cen[kMaxGroupMembers], ext[kMaxGroupMembers];
      for (int i = 0; i < n; ++i) {
        cen[i] = 0.5 * (mlo[3 * (a + i) + d] + mhi[3 * (a + i) + d]);
        ext[i] = mhi[3 * (a + i) + d] - mlo[3 * (a + i) + d] + 1;
      }
      double sc[kMaxGroupMembers], se[kMaxGroupMembers];
      std::copy(cen, cen + n, sc);
      std::copy(ext, ext + n, se);
      std::sort(sc, sc + n);
      std::sort(se, se + n);
      const double mc = n % 2 ? sc[n / 2] : 0.5 * (sc[n / 2 - 1] + sc[n / 2]);
      const double me = n % 2 ? se[n / 2] : 0.5 * (se[n / 2 - 1] + se[n / 2]);
      for (int i = 0; i < n; ++i)
        if (std::fabs(cen[i] - mc) > std::max(0.25 * me, 4.0)) mask |= 1u << i;
    }
    return mask;
  };
  // Natural groups, in parallel: the common case is a group without outlying members whose
  // union fits (status 0: one tile). Otherwise (status 1) it is resolved below: outlying
  // members leave the group, so they cannot inflate the shared tile; the rest forms the group
  // if it fits, else single members; a member that does not fit alone is split into halves of
  // its pixel tile until it does.
  const int ngrp = (int)ng.start.size() - 1;
  std::vector<GroupDev> nat(ngrp);
  std::vector<int64_t> nvox(ngrp);
  std::vector<uint8_t> status(ngrp);
  std::vector<uint32_t> omask(ngrp);
  std::vector<int32_t> seq(nm);
  for (int64_t i = 0; i < nm; ++i) seq[i] = (int32_t)i;
#pragma omp parallel for schedule(static)
  for (int gi = 0; gi < ngrp; ++gi) {
    const int a = ng.start[gi], b = ng.start[gi + 1];
    omask[gi] = outliers(a, b);
    nvox[gi] = group(&seq[a], b - a, nat[gi]);
    status[gi] = (!omask[gi] && fits(nat[gi], nvox[gi])) ? 0 : 1;
  }
  out.grp.clear();
  out.grp.reserve(ngrp);
  out.max_tile_vox = 0;
  out.max_r_bytes = ng.max_r_bytes;
  out.max_t_floats = ng.max_t_floats;
  out.nsplit = 0;
  out.all_fit = true;
  std::vector<int32_t> ix;          // pool indices of every output group, concatenated
  std::vector<int32_t> gstart;      // output group k lists ix[gstart[k], gstart[k + 1])
  ix.reserve(nm);
  gstart.reserve(ngrp + 1);
  int fit = 0;
  auto emit = [&](const GroupDev& g, int64_t vox, const int32_t* list, int n) {
    gstart.push_back((int32_t)ix.size());
    ix.insert(ix.end(), list, list + n);
    out.grp.push_back(g);
    out.max_tile_vox = std::max(out.max_tile_vox, vox);
  };
  std::vector<int32_t> work;
  auto emit_single = [&](int32_t i0) {  // a member alone, halving its pixel tile until it fits
    work.assign(1, i0);
    while (!work.empty()) {
      const int32_t i = work.back();
      work.pop_back();
      GroupDev g;
      const int64_t vox = group(&i, 1, g);
      const MemberDev m = pool[i];
      if (fits(g, vox) || (m.tu == 1 && m.tv == 1)) {
        if (!fits(g, vox)) out.all_fit = false;
        emit(g, vox, &i, 1);
        continue;
      }
      const int hu = m.tu > 1 ? (m.tu + 1) / 2 : m.tu, hv = m.tv > 1 ? (m.tv + 1) / 2 : m.tv;
      for (int sv = 0; sv < m.tv; sv += hv)
        for (int su = 0; su < m.tu; su += hu) {
          MemberDev q = m;
          q.u0 = m.u0 + su;
          q.v0 = m.v0 + sv;
          q.tu = std::min(hu, m.tu - su);
          q.tv = std::min(hv, m.tv - sv);
          pool.push_back(q);
          mlo.resize(3 * pool.size());
          mhi.resize(3 * pool.size());
          const int32_t k = (int32_t)pool.size() - 1;
          msup.push_back(bbox_of(q, &mlo[3 * k], &mhi[3 * k]));
          work.push_back(k);
        }
      ++out.nsplit;
    }
  };
  std::vector<int32_t> core;
  std::vector<std::pair<std::vector<int32_t>, int>> hwork;  // (member list, halving depth)
  int half = 0;
  for (int gi = 0; gi < ngrp; ++gi) {
    const int a = ng.start[gi], b = ng.start[gi + 1];
    if (status[gi] == 0) {
      ++fit;
      emit(nat[gi], nvox[gi], &seq[a], b - a);
      continue;
    }
    core.clear();
    for (int i = a; i < b; ++i) {
      if (omask[gi] >> (i - a) & 1u) emit_single(i);
      else core.push_back(i);
    }
    if (core.empty()) {  // all members outlying: not a tile-size failure
      ++fit;
      continue;
    }
    GroupDev g;
    const int64_t vox = group(core.data(), (int)core.size(), g);
    if (fits(g, vox)) {
      ++fit;
      emit(g, vox, core.data(), (int)core.size());
      continue;
    }
    // Backprojection: a group that does not fit is first halved as a whole -- every member's
    // pixel tile split the same way along its longer axis, the halves of all members staying
    // together -- so the group keeps its members' lines in one CTA (a 3-member group of 8 x 8
    // tiles has 768 lines: three full rounds of 256 threads; single members of half tiles
    // would leave half of a round idle). Two levels, then single members.
    // Splitting never lowers a backprojection group's tile precision: when the group as a whole
    // is exact (a rim member, or a footprint that leaves the grid, whose partly observed pixels
    // carry 1/kappa-amplified terms), its halves and single members stay exact even where their
    // own box is interior (a half's boundary lines are fed by the other half's pixels).
    if (!fwd && g.exact)
      for (int32_t i : core) pool[i].flags |= kMemberRim;
    if ((!fwd || PVR_FWD_HALVE) && (pool[core[0]].tu > 1 || pool[core[0]].tv > 1)) {
      bool whole = true;  // every half (first level) fits
      hwork.clear();
      hwork.push_back({core, 0});
      while (!hwork.empty()) {
        auto item = std::move(hwork.back());
        hwork.pop_back();
        GroupDev hg;
        const int64_t hv = group(item.first.data(), (int)item.first.size(), hg);
        if (fits(hg, hv)) {
          emit(hg, hv, item.first.data(), (int)item.first.size());
          continue;
        }
        if (item.second > 0) whole = false;
        const MemberDev& m0 = pool[item.first[0]];
        if (item.second >= 2 || (m0.tu == 1 && m0.tv == 1)) {
          whole = false;
          for (int32_t i : item.first) emit_single(i);
          continue;
        }
        const bool along_u = m0.tu >= m0.tv;
        std::vector<int32_t> h0, h1;
        for (int32_t i : item.first) {
          const MemberDev m = pool[i];
          MemberDev q0 = m, q1 = m;
          if (along_u) {
            const int hu = (m.tu + 1) / 2;
            q0.tu = hu;
            q1.u0 = m.u0 + hu;
            q1.tu = m.tu - hu;
          } else {
            const int hv2 = (m.tv + 1) / 2;
            q0.tv = hv2;
            q1.v0 = m.v0 + hv2;
            q1.tv = m.tv - hv2;
          }
          for (int h = 0; h < 2; ++h) {
            const MemberDev& q = h ? q1 : q0;
            if (q.tu <= 0 || q.tv <= 0) continue;
            pool.push_back(q);
            mlo.resize(3 * pool.size());
            mhi.resize(3 * pool.size());
            const int32_t k = (int32_t)pool.size() - 1;
            msup.push_back(bbox_of(q, &mlo[3 * k], &mhi[3 * k]));
            (h ? h1 : h0).push_back(k);
          }
        }
        if (!h0.empty()) hwork.push_back({std::move(h0), item.second + 1});
        if (!h1.empty()) hwork.push_back({std::move(h1), item.second + 1});
      }
      ++out.nsplit;
      if (whole) ++half;
      continue;
    }
    if (core.size() > 1) ++out.nsplit;
    for (int32_t i : core) emit_single(i);
  }
  gstart.push_back((int32_t)ix.size());
  out.fit_frac = ngrp ? (double)fit / ngrp : 1.0;
  out.half_frac = ngrp ? (double)(fit + half) / ngrp : 1.0;
  tr.mark("    group boxes");
  // Order the CTAs' work along a Morton curve of the groups' bbox centres (16-voxel cells), so
  // that overlapping footprints of all stacks are processed close in time: the forward's X
  // reads and the backprojection's (A, C) flushes then hit L2 instead of re-streaming HBM.
  // Keys carry the group index as tie-break: the order is unique (deterministic).
  const int64_t ng2 = (int64_t)out.grp.size();
  std::vector<std::pair<uint64_t, int32_t>> order(ng2);
#pragma omp parallel for schedule(static)
  for (int64_t g = 0; g < ng2; ++g) {
    uint64_t key = 0;
    uint32_t cc[3];
    for (int d = 0; d < 3; ++d)
      cc[d] = (uint32_t)std::max(0, (out.grp[g].lo[d] + out.grp[g].dim[d] / 2 + 4096) >> 4) & 0x3FF;
    for (int b = 9; b >= 0; --b)
      for (int d = 2; d >= 0; --d) key = (key << 1) | ((cc[d] >> b) & 1u);
    order[g] = {key, (int32_t)g};
  }
  tr.mark("    morton keys");
  __gnu_parallel::sort(order.begin(), order.end());
  tr.mark("    morton sort");
  std::vector<GroupDev> grp(ng2);
  std::vector<int32_t> m0(ng2 + 1, 0);
  for (int64_t k = 0; k < ng2; ++k) m0[k + 1] = m0[k] + out.grp[order[k].second].nm;
  out.mem.resize(m0[ng2]);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < ng2; ++k) {
    const int32_t src = order[k].second;
    GroupDev g = out.grp[src];
    for (int i = 0; i < g.nm; ++i) out.mem[m0[k] + i] = pool[ix[gstart[src] + i]];
    g.m0 = m0[k];
    grp[k] = g;
  }
  out.grp.swap(grp);
  tr.mark("    reorder");
}

// Forward tiles are staged by TMA with one box per group (its own bbox, sized in
// size_groups): one tensor map per distinct box shape (width, height) and X buffer.
pvr_status box_forward_groups(pvr_ctx* c, PlanBuild& pb) {
  std::vector<std::pair<int, int>> shapes;
  std::vector<int32_t> index(257 * 257, -1);  // (width, height) -> shape number
  for (GroupDev& g : pb.grp) {
    if (g.dim[0] > 256 || g.dim[1] > 256)
      return fail(c, PVR_ERR_ARG, "forward tile %dx%d exceeds the TMA box limit", g.dim[0], g.dim[1]);
    int32_t& k = index[g.dim[0] * 257 + g.dim[1]];
    if (k < 0) {
      k = (int32_t)shapes.size();
      shapes.emplace_back(g.dim[0], g.dim[1]);
    }
    g.tmap = k;
  }
  // spare shapes for the device re-plan of later set_transforms: each shape grown by 8 in x
  // (keeps 4 x odd) and 2 in y, so a group whose footprint grew a little still finds a box
  const size_t base = shapes.size();
  for (size_t k = 0; k < base; ++k) {
    const int w = shapes[k].first + 8, h = shapes[k].second + 2;
    if (w > 256 || h > 256 || index[w * 257 + h] >= 0) continue;
    index[w * 257 + h] = (int32_t)shapes.size();
    shapes.emplace_back(w, h);
  }
  if ((int)shapes.size() > kMaxBoxShapes) shapes.resize(std::max<size_t>(base, kMaxBoxShapes));
  c->fbox.clear();
  for (auto& sh : shapes) {
    c->fbox.push_back(sh.first);
    c->fbox.push_back(sh.second);
  }
  return PVR_OK;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

// Tensor maps of both X buffers for every forward box shape: dims (nx, ny, nz), row pitch
// nxp, box (w, h, 1); out-of-grid elements (negative or >= dims) are zero-filled by TMA.
// Layout on the device: [X buffer][shape], 128 B each.
pvr_status encode_tmaps(pvr_ctx* c) {
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(c, PVR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = (EncodeTiledFn)fn;
  }
  const size_t nb = c->fbox.size() / 2;
  std::vector<CUtensorMap> maps(2 * nb);
  if (nb) memset(maps.data(), 0, maps.size() * sizeof(CUtensorMap));
  for (int b = 0; b < 2; ++b)
    for (size_t k = 0; k < nb; ++k) {
      const cuuint64_t dim[3] = {(cuuint64_t)c->dims.x, (cuuint64_t)c->dims.y, (cuuint64_t)c->dims.z};
      const cuuint64_t stride[2] = {(cuuint64_t)c->nxp * 4, (cuuint64_t)c->nxp * c->dims.y * 4};
      const cuuint32_t box[3] = {(cuuint32_t)c->fbox[2 * k], (cuuint32_t)c->fbox[2 * k + 1], 1};
      const cuuint32_t es[3] = {1, 1, 1};
      const CUresult r = encode(&maps[b * nb + k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, c->X[b], dim, stride, box,
                                es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(c, PVR_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
  if (maps.size() > c->tmaps_cap) {
    if (c->tmaps) cudaFree(c->tmaps);
    c->tmaps = nullptr;
    CUDA_TRY(c, cudaMalloc(&c->tmaps, maps.size() * sizeof(CUtensorMap)));
    c->tmaps_cap = maps.size();
  }
  if (nb) {
    CUDA_TRY(c, cudaMemcpyAsync(c->tmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice,
                                c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  }
  return PVR_OK;
}

// extra_groups: capacity after the plan's groups (the iteration backprojection's device
// re-plan appends single-member groups there)
pvr_status upload_plan(pvr_ctx* c, pvr_ctx::Plan& pl, const PlanBuild& pb, size_t extra_groups) {
  if (pb.mem.size() > pl.mem_cap) {
    if (pl.mem) cudaFree(pl.mem);
    pl.mem = nullptr;
    CUDA_TRY(c, cudaMalloc(&pl.mem, pb.mem.size() * sizeof(MemberDev)));
    pl.mem_cap = pb.mem.size();
  }
  if (pb.grp.size() + extra_groups > pl.grp_cap) {
    if (pl.grp) cudaFree(pl.grp);
    pl.grp = nullptr;
    CUDA_TRY(c, cudaMalloc(&pl.grp, (pb.grp.size() + extra_groups) * sizeof(GroupDev)));
    pl.grp_cap = pb.grp.size() + extra_groups;
  }
  CUDA_TRY(c, cudaMemcpyAsync(pl.mem, pb.mem.data(), pb.mem.size() * sizeof(MemberDev), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(pl.grp, pb.grp.data(), pb.grp.size() * sizeof(GroupDev), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));  // the host vectors go out of scope
  pl.ngroups = (int)pb.grp.size();
  pl.nmem = (int64_t)pb.mem.size();
  ++c->geo_epoch;
  pl.nsplit = pb.nsplit;
  pl.max_nm = 1;
  for (const GroupDev& gd : pb.grp) pl.max_nm = std::max(pl.max_nm, (int)gd.nm);
  pl.tile_words = (int)((pb.max_tile_vox + 3) & ~int64_t(3));
  pl.r_bytes = (int)((pb.max_r_bytes + 15) & ~int64_t(15));
  pl.t_floats = (int)((pb.max_t_floats + 31) & ~int64_t(31));  // 128-byte aligned X tile after it
  return PVR_OK;
}

// Tile size (and backprojection c segments): the largest candidate for which >= 90% of the
// natural groups fit whole and every single member fits; large tiles amortise the flush, the
// staging and the lattice halo. Candidates are first screened on a sample of patches; the last
// choice is tried first, so repeated set_transforms with similar motion only resize bboxes.
pvr_status build_plans(pvr_ctx* c, const std::vector<PatchGeo>& geo, int kind_lo, int kind_hi) {
  std::vector<int64_t> sample, all(c->nloc);
  for (int64_t s = 0; s < c->nloc; ++s) all[s] = s;
  const int64_t step = std::max<int64_t>(1, c->nloc / 128);
  for (int64_t s = 0; s < c->nloc; s += step) sample.push_back(s);
  static const int fcand[][3] = {{16, 16, 1}, {16, 8, 1}, {8, 8, 1}, {8, 4, 1}, {4, 4, 1}, {2, 2, 1}, {1, 1, 1}};
  // through-plane segments cost a line setup and two window flushes each: fewer segments at a
  // smaller pixel tile first (c3: 8 x 8 x 1 17.8 ms vs 16 x 8 x 2 20.5 ms per backprojection)
  static const int bcand[][3] = {{16, 16, 1}, {16, 8, 1}, {8, 8, 1}, {8, 4, 1}, {16, 8, 2}, {8, 8, 2},
                                 {8, 4, 2},   {4, 4, 2},  {4, 4, 4}, {2, 2, 4}, {2, 2, 8},  {1, 1, 8}, {1, 1, 32}};
  auto natural = [&](int TU, int TV, int nseg, bool fwd, bool smp) -> const NaturalGroups& {
    for (auto& ng : c->ngcache)
      if (ng->TU == TU && ng->TV == TV && ng->nseg == nseg && ng->fwd == fwd && ng->sample == smp) return *ng;
    c->ngcache.emplace_back(new NaturalGroups());
    NaturalGroups& ng = *c->ngcache.back();
    build_natural(c, smp ? sample : all, TU, TV, nseg, fwd, ng);
    ng.sample = smp;
    return ng;
  };
  // a tile size is taken when >= 90% of the natural groups fit whole; the backprojection also
  // takes it when >= 75% fit whole and >= 90% whole or halved (size_groups): c3 at the 56 KB
  // tile, 8 x 8 (85% whole: the exact rim groups need 16 B per cell) rather than 8 x 4
  auto accept = [](const PlanBuild& pb, bool fwd) {
    return pb.all_fit && (pb.fit_frac >= 0.9 || (!fwd && pb.fit_frac >= PVR_BP_HALVE_MIN && pb.half_frac >= 0.9) ||
                          (fwd && PVR_FWD_HALVE && pb.fit_frac >= PVR_FWD_HALVE_MIN && pb.half_frac >= 0.9));
  };
  Trace tr;
  for (int kind = kind_lo; kind < kind_hi; ++kind) {
    const bool fwd = kind == 0;
    pvr_ctx::Plan& pl = kind == 0 ? c->fplan : kind == 1 ? c->bplan : c->iplan;
    const int(*cand)[3] = fwd ? fcand : bcand;
    const int ncand = fwd ? (int)(sizeof(fcand) / sizeof(fcand[0])) : (int)(sizeof(bcand) / sizeof(bcand[0]));
    std::vector<int> order;
    for (int k = 0; k < ncand; ++k)
      if (cand[k][0] == pl.TU && cand[k][1] == pl.TV && cand[k][2] == pl.nseg && pl.ngroups > 0) order.push_back(k);
    for (int k = 0; k < ncand; ++k) order.push_back(k);
    int pick = -1;
    PlanBuild pb;
    for (int k : order) {
      const bool previous = pl.ngroups > 0 && k == order[0] && order.size() > (size_t)ncand;
      if (!previous) {  // quick reject on the sample
        size_groups(c, geo, natural(cand[k][0], cand[k][1], cand[k][2], fwd, true), kind, pb);
        if (tr.on)
          fprintf(stderr, "[pvr]   plan kind %d tile %dx%dx%d (sample): fit %.3f (halved %.3f) all_fit %d\n", kind,
                  cand[k][0], cand[k][1], cand[k][2], pb.fit_frac, pb.half_frac, (int)pb.all_fit);
        if (!accept(pb, fwd)) continue;
      }
      size_groups(c, geo, natural(cand[k][0], cand[k][1], cand[k][2], fwd, false), kind, pb);
      if (tr.on)
        fprintf(stderr, "[pvr]   plan kind %d tile %dx%dx%d: fit %.3f (halved %.3f) all_fit %d groups %zu split %d\n",
                kind, cand[k][0], cand[k][1], cand[k][2], pb.fit_frac, pb.half_frac, (int)pb.all_fit, pb.grp.size(),
                pb.nsplit);
      if (accept(pb, fwd)) { pick = k; break; }
    }
    if (pick < 0) return fail(c, PVR_ERR_ARG, "no tiling fits the shared-memory budget (extreme transforms?)");
    pl.TU = cand[pick][0];
    pl.TV = cand[pick][1];
    pl.nseg = cand[pick][2];
    if (fwd) {
      pvr_status rb = box_forward_groups(c, pb);
      if (rb != PVR_OK) return rb;
    }
    tr.mark(kind == 0 ? "  plan forward" : kind == 1 ? "  plan backprojection" : "  plan init");
    pvr_status r = upload_plan(c, pl, pb, kind == 1 ? pb.mem.size() : 0);
    if (r != PVR_OK) return r;
    tr.mark("  upload");
    if (kind == 2) continue;
    int32_t* tile = fwd ? c->st.fwd_tile : c->st.bp_tile;
    tile[0] = pl.TU; tile[1] = pl.TV; tile[2] = pl.nseg;
    (fwd ? c->st.fwd_groups : c->st.bp_groups) = pl.ngroups;
    (fwd ? c->st.fwd_split : c->st.bp_split) = pb.nsplit;
    if (!fwd) {
      int64_t ne = 0;
      for (const GroupDev& g : pb.grp) ne += g.exact;
      c->st.bp_exact_groups = ne;
    }
    (fwd ? c->st.fwd_members : c->st.bp_members) = (int64_t)pb.mem.size();
    (fwd ? c->st.fwd_smem : c->st.bp_smem) =
        fwd ? (int64_t)(pl.t_floats + pl.tile_words) * 4 : (int64_t)kBpTileBytes + pl.r_bytes;
  }
  return PVR_OK;
}

// profiling: events bracket each kernel group when PVR_PARAM_PROFILE is on
enum { EV_FWD0, EV_FWD1, EV_EM1, EV_EST1, EV_BP1, EV_AR1, EV_UPD1, EV_N };

std::vector<cudaEvent_t>* prof_slot(pvr_ctx* c) {
  if (c->prof_free.empty()) {
    std::vector<cudaEvent_t> s(EV_N);
    for (auto& e : s) cudaEventCreate(&e);
    c->prof_free.push_back(s);
  }
  c->prof_pending.push_back(c->prof_free.back());
  c->prof_free.pop_back();
  return &c->prof_pending.back();
}

void prof_drain(pvr_ctx* c) {
  for (auto& s : c->prof_pending) {
    cudaEventSynchronize(s[EV_UPD1]);
    float t[6];
    for (int i = 0; i < 6; ++i) cudaEventElapsedTime(&t[i], s[i], s[i + 1]);
    c->st.ms_forward += t[0];
    c->st.ms_em += t[1];
    c->st.ms_estep += t[2];
    c->st.ms_backproject += t[3];
    c->st.ms_allreduce += t[4];
    c->st.ms_update += t[5];
    c->prof_free.push_back(s);
  }
  c->prof_pending.clear();
}

}  // namespace

// ======================================================================================
extern "C" {

const char* pvr_version(void) { return kVersion; }

const char* pvr_last_error(const pvr_ctx* c) { return c ? c->err.c_str() : g_static_err.c_str(); }

pvr_status pvr_create_volume(const pvr_geometry* g, int cuda_device, void* cuda_stream, pvr_ctx** out) {
  if (!g || !out) return fail(nullptr, PVR_ERR_ARG, "null argument");
  if (g->dims[0] < 1 || g->dims[1] < 1 || g->dims[2] < 1 || !(g->spacing_mm > 0))
    return fail(nullptr, PVR_ERR_ARG, "invalid geometry (dims >= 1, spacing > 0)");
  if ((int64_t)(g->dims[0] + 1) * g->dims[1] * g->dims[2] >= (int64_t(1) << 31))
    return fail(nullptr, PVR_ERR_ARG, "volume too large (kernels index voxels with 32-bit offsets)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(nullptr, PVR_ERR_CUDA, "no CUDA device available (libpvr has no CPU path)");
  }
  if (cuda_device < 0 || cuda_device >= ndev) return fail(nullptr, PVR_ERR_ARG, "bad cuda_device");
  pvr_ctx* c = new pvr_ctx();
  memset(&c->st, 0, sizeof(c->st));
  c->device = cuda_device;
  c->dims = make_int3(g->dims[0], g->dims[1], g->dims[2]);
  c->nxp = (g->dims[0] + 3) & ~3;
  c->s = g->spacing_mm;
  for (int d = 0; d < 3; ++d) c->o[d] = g->origin_mm[d];
  c->V = (int64_t)g->dims[0] * g->dims[1] * g->dims[2];
  c->Vp = (int64_t)c->nxp * g->dims[1] * g->dims[2];
  c->nzp = g->dims[2];
  c->z0 = 0;
  c->z1 = g->dims[2];
  cudaSetDevice(cuda_device);
  if (cuda_stream) {
    c->stream = (cudaStream_t)cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      return fail(nullptr, PVR_ERR_CUDA, "cudaStreamCreate failed");
    }
    c->own_stream = true;
  }
  cudaError_t e1 = cudaMalloc(&c->X[0], c->Vp * sizeof(float));
  cudaError_t e2 = cudaMalloc(&c->X[1], c->Vp * sizeof(float));
  cudaError_t e3 = cudaMalloc(&c->AC, (c->Vp + 2) * sizeof(float2));
  cudaError_t e4 = cudaMalloc(&c->em, sizeof(EmDev));
  cudaError_t e5 = cudaMalloc(&c->partials, ((size_t)kStatBlocks * 5 + 1) * sizeof(double));  // + fwd group counter
  if (e1 || e2 || e3 || e4 || e5) {
    cudaGetLastError();
    free_dev(c);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
    return fail(nullptr, PVR_ERR_OOM, "device allocation of the volume buffers failed");
  }
  cudaMemsetAsync(c->X[0], 0, c->Vp * sizeof(float), c->stream);
  cudaMemsetAsync(c->X[1], 0, c->Vp * sizeof(float), c->stream);
  cudaMemsetAsync(c->AC, 0, (c->Vp + 2) * sizeof(float2), c->stream);
  cudaMemsetAsync(c->em, 0, sizeof(EmDev), c->stream);
  c->st.voxels = c->V;
  *out = c;
  return PVR_OK;
}

pvr_status pvr_destroy(pvr_ctx* c) {
  if (!c) return PVR_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  free_dev(c);
  for (auto* pool : {&c->prof_free, &c->prof_pending})
    for (auto& slot : *pool)
      for (auto e : slot) cudaEventDestroy(e);
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  if (c->host_buf) cudaFreeHost(c->host_buf);
  if (c->pd_host) cudaFreeHost(c->pd_host);
  if (c->pd_copied) cudaEventDestroy(c->pd_copied);
  if (c->aux) {
    cudaStreamSynchronize(c->aux);
    cudaStreamDestroy(c->aux);
  }
  if (c->ev_geo) cudaEventDestroy(c->ev_geo);
  if (c->ev_tab) cudaEventDestroy(c->ev_tab);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return PVR_OK;
}

pvr_status pvr_comm_unique_id(void* out128) {
  if (!out128) return fail(nullptr, PVR_ERR_ARG, "null buffer");
  std::string err;
  if (!g_nccl.load(err)) return fail(nullptr, PVR_ERR_NCCL, "%s", err.c_str());
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, PVR_ERR_NCCL, "ncclGetUniqueId: %s", g_nccl.GetErrorString(r));
  memcpy(out128, &id, sizeof(id));
  return PVR_OK;
}

// Common part of the two comm inits: rank, shard and the padded volume layout (nz rounded up
// to nranks equal slabs of planes, for reduce-scatter / all-gather; X kept).
static pvr_status comm_setup(pvr_ctx* c, int nranks, int rank) {
  c->nranks = nranks;
  c->rank = rank;
  const int nzp = (c->dims.z + nranks - 1) / nranks * nranks;
  if (nzp != c->nzp) {
    const int64_t plane = (int64_t)c->nxp * c->dims.y;
    const int64_t Vp = plane * nzp;
    float* X[2] = {nullptr, nullptr};
    float2* AC = nullptr;
    CUDA_TRY(c, cudaMalloc(&X[0], Vp * sizeof(float)));
    CUDA_TRY(c, cudaMalloc(&X[1], Vp * sizeof(float)));
    CUDA_TRY(c, cudaMalloc(&AC, (Vp + 2) * sizeof(float2)));
    for (int b = 0; b < 2; ++b) {
      CUDA_TRY(c, cudaMemsetAsync(X[b], 0, Vp * sizeof(float), c->stream));
      CUDA_TRY(c, cudaMemcpyAsync(X[b], c->X[b], c->Vp * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
    }
    CUDA_TRY(c, cudaMemsetAsync(AC, 0, (Vp + 2) * sizeof(float2), c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    cudaFree(c->X[0]);
    cudaFree(c->X[1]);
    cudaFree(c->AC);
    c->X[0] = X[0];
    c->X[1] = X[1];
    c->AC = AC;
    c->Vp = Vp;
    c->nzp = nzp;
  }
  const int slab = c->nzp / nranks;
  c->z0 = std::min(rank * slab, c->dims.z);
  c->z1 = std::min((rank + 1) * slab, c->dims.z);
  return PVR_OK;
}

pvr_status pvr_comm_init(pvr_ctx* c, int nranks, int rank, const void* uid) {
  GUARD(c);
  if (c->state >= PATCHED) return fail(c, PVR_ERR_STATE, "pvr_comm_init must precede extract_patches");
  if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !uid))
    return fail(c, PVR_ERR_ARG, "invalid nranks/rank/unique id");
  pvr_status r = comm_setup(c, nranks, rank);
  if (r != PVR_OK || nranks == 1) return r;
  std::string err;
  if (!g_nccl.load(err)) return fail(c, PVR_ERR_NCCL, "%s", err.c_str());
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  return nccl_check(c, g_nccl.CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
}

pvr_status pvr_comm_init_host(pvr_ctx* c, int nranks, int rank, pvr_host_collective_fn fn, void* user) {
  GUARD(c);
  if (c->state >= PATCHED) return fail(c, PVR_ERR_STATE, "pvr_comm_init_host must precede extract_patches");
  if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !fn))
    return fail(c, PVR_ERR_ARG, "invalid nranks/rank/collective callback");
  c->host_fn = fn;
  c->host_user = user;
  return comm_setup(c, nranks, rank);
}

pvr_status pvr_set_param(pvr_ctx* c, int key, double v) {
  GUARD(c);
  const bool extract_key = key == PVR_PARAM_PSF_MODE || key == PVR_PARAM_PSF_NSIGMA || key == PVR_PARAM_PSF_QUALITY ||
                           key == PVR_PARAM_BP_EXACT || key == PVR_PARAM_DETERMINISTIC ||
                           key == PVR_PARAM_PLAN_BUDGET;
  if (extract_key && c->state >= PATCHED)
    return fail(c, PVR_ERR_STATE, "parameter %d must be set before extract_patches", key);
  switch (key) {
    case PVR_PARAM_DELTA: if (!(v > 0)) goto bad; c->delta = v; break;
    case PVR_PARAM_TAU_PATCH: c->tau_patch = v; break;
    case PVR_PARAM_C0: if (!(v >= 0 && v <= 1)) goto bad; c->c0 = v; break;
    case PVR_PARAM_TAU_LIVE: c->tau_live = v; break;
    case PVR_PARAM_TAU_C: if (!(v >= 0)) goto bad; c->tau_C = v; break;
    case PVR_PARAM_TAU_OBS: if (!(v > 0)) goto bad; c->tau_obs = v; break;
    case PVR_PARAM_CLAMP: c->clamp = v != 0; break;
    case PVR_PARAM_PSF_MODE: if (v != 0 && v != 1 && v != 2) goto bad; c->psf_mode = (int)v; break;
    case PVR_PARAM_SIGMA2_FLOOR: if (!(v >= 0)) goto bad; c->s2floor = v; break;
    case PVR_PARAM_PSF_NSIGMA: if (!(v > 0)) goto bad; c->nsigma = v; break;
    case PVR_PARAM_PSF_QUALITY: if (!(v >= 1 && v <= 4)) goto bad; c->quality = v; break;
    case PVR_PARAM_EM_ROUNDS:
      if (!(v >= 1 && v <= 100) || v != std::floor(v)) goto bad;
      c->em_rounds = (int)v;
      break;
    case PVR_PARAM_EM_TOL: if (!(v >= 0)) goto bad; c->em_tol = v; break;
    case PVR_PARAM_PATCH_MIXTURE: if (v != 0 && v != 1) goto bad; c->patch_mixture = (int)v; break;
    case PVR_PARAM_PROFILE: c->profile = v != 0; break;
    case PVR_PARAM_BP_EXACT: if (v != 0 && v != 1 && v != 2) goto bad; c->bp_exact = (int)v; break;
    case PVR_PARAM_EXCHANGE:
      if (v != PVR_EXCHANGE_ALLREDUCE && v != PVR_EXCHANGE_SLABS && v != PVR_EXCHANGE_AVERAGE) goto bad;
      c->exchange = (int)v;
      break;
    case PVR_PARAM_COMM_TIMEOUT: if (!(v > 0)) goto bad; c->comm_timeout = v; break;
    case PVR_PARAM_DETERMINISTIC: if (v != 0 && v != 1) goto bad; c->det = (int)v; break;
    case PVR_PARAM_PLAN_BUDGET: if (!(v >= 0.05 && v <= 1)) goto bad; c->plan_budget = v; break;
    default: return fail(c, PVR_ERR_ARG, "unknown parameter key %d", key);
  }
  return PVR_OK;
bad:
  return fail(c, PVR_ERR_ARG, "invalid value %g for parameter %d", v, key);
}

pvr_status pvr_add_stack(pvr_ctx* c, const float* slices, int W, int H, int K,
                         const double G[12], double thickness, int* id_out) {
  GUARD(c);
  if (c->state > STACKS) return fail(c, PVR_ERR_STATE, "add_stack after extract_patches");
  if (!slices || !G || W < 1 || H < 1 || K < 1 || !(thickness > 0))
    return fail(c, PVR_ERR_ARG, "invalid stack (sizes >= 1, thickness > 0)");
  HostStack st;
  st.W = W; st.H = H; st.K = K;
  memcpy(st.G, G, sizeof(st.G));
  st.theta = thickness;
  double c0[3] = {G[0], G[4], G[8]}, c1[3] = {G[1], G[5], G[9]}, c2[3] = {G[2], G[6], G[10]};
  const double px = norm3(c0), py = norm3(c1);
  if (!(px > 0) || !(py > 0)) return fail(c, PVR_ERR_ARG, "degenerate in-plane axes");
  for (int d = 0; d < 3; ++d) { st.u[d] = c0[d] / px; st.v[d] = c1[d] / py; }
  st.w[0] = st.u[1] * st.v[2] - st.u[2] * st.v[1];
  st.w[1] = st.u[2] * st.v[0] - st.u[0] * st.v[2];
  st.w[2] = st.u[0] * st.v[1] - st.u[1] * st.v[0];
  const double nw = norm3(st.w);
  if (!(nw > 1e-12)) return fail(c, PVR_ERR_ARG, "parallel in-plane axes");
  for (int d = 0; d < 3; ++d) st.w[d] /= nw;
  // a singular index->world map (zero slice step along the normal) is rejected too
  const double det = c0[0] * (c1[1] * c2[2] - c1[2] * c2[1]) - c0[1] * (c1[0] * c2[2] - c1[2] * c2[0]) +
                     c0[2] * (c1[0] * c2[1] - c1[1] * c2[0]);
  if (K > 1 && !(std::fabs(det) > 1e-12)) return fail(c, PVR_ERR_ARG, "singular index_to_world");
  const size_t bytes = (size_t)W * H * K * sizeof(float);
  CUDA_TRY(c, cudaMalloc(&st.y_dev, bytes));
  CUDA_TRY(c, cudaMemcpyAsync(st.y_dev, slices, bytes,
                              is_device_ptr(slices) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                              c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->stacks.push_back(st);
  if (id_out) *id_out = (int)c->stacks.size() - 1;
  c->state = STACKS;
  return PVR_OK;
}

// Contiguous shard plan balanced by cost (pixels x PSF samples): bounds[r] .. bounds[r+1]
// is rank r's patch range ("distributing independent subsets of patches").
pvr_status pvr_plan_shards(const int64_t* cost, int64_t M, int nranks, int64_t* bounds) {
  if (!bounds || M < 0 || nranks < 1 || (M > 0 && !cost))
    return fail(nullptr, PVR_ERR_ARG, "invalid shard plan args");
  std::vector<int64_t> pre(M + 1, 0);
  for (int64_t i = 0; i < M; ++i) pre[i + 1] = pre[i] + cost[i];
  const int64_t total = pre[M];
  bounds[0] = 0;
  for (int r = 1; r < nranks; ++r) {
    const double target = (double)total * r / nranks;
    int64_t i = std::lower_bound(pre.begin(), pre.end(), (int64_t)std::ceil(target)) - pre.begin();
    if (i > 0 && (target - pre[i - 1]) < (pre[std::min(i, M)] - target)) --i;
    i = std::min(std::max(i, bounds[r - 1]), M);
    bounds[r] = i;
  }
  bounds[nranks] = M;
  return PVR_OK;
}

static pvr_status install_patches(pvr_ctx* c, const uint8_t* mask, int64_t* n_out);

// f3 multi-scale schedule ("different scales Y_i ... for each iteration i"):
// patches may be re-extracted in a context that already has patches. Every per-patch and
// per-pixel structure is dropped (plans, caches, weights, EM / registration scratch); the
// stacks and the reconstruction X stay; pvr_set_transforms is required again.
static pvr_status begin_extraction(pvr_ctx* c) {
  if (c->state == STACKS) return PVR_OK;
  if (c->state < STACKS) return fail(c, PVR_ERR_STATE, "patches need stacks");
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  void* ptrs[] = {c->e, c->p, c->kap, c->pbar, c->w, c->tab, c->psf, c->pdev, c->fplan.mem, c->fplan.grp,
                  c->bplan.mem, c->bplan.grp, c->iplan.mem, c->iplan.grp, c->bplan.btab, c->iplan.btab,
                  c->fplan.btab, c->regP, c->rpart, c->nlivep, c->mask, c->vpat, c->vin};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  c->e = c->p = c->kap = c->pbar = c->w = c->tab = nullptr;
  c->psf = nullptr;
  c->pdev = nullptr;
  c->regP = nullptr;
  c->regP_cap = 0;
  c->rpart = nullptr;
  c->nlivep = nullptr;
  c->mask = nullptr;
  c->vpat = nullptr;
  c->vin = nullptr;
  c->mask_host.clear();
  for (pvr_ctx::Plan* pl : {&c->fplan, &c->bplan, &c->iplan}) {
    pl->mem = nullptr;
    pl->grp = nullptr;
    pl->mem_cap = pl->grp_cap = 0;
    pl->ngroups = 0;
    pl->nmem = 0;
    pl->btab = nullptr;
    pl->btab_cap = 0;
    pl->btab_epoch = 0;
  }
  ++c->geo_epoch;
  c->iplan_valid = false;
  c->ngcache.clear();
  c->geo.clear();
  c->Tloc.clear();
  c->patches.clear();
  c->state = STACKS;
  return PVR_OK;
}

pvr_status pvr_extract_patches(pvr_ctx* c, int size, int stride, int depth, int stride_z, int64_t* n_out) {
  GUARD(c);
  if (c->state < STACKS) return fail(c, PVR_ERR_STATE, "extract_patches needs stacks");
  if (size < 1 || stride < 1 || stride > size || depth < 1 || stride_z < 1 || stride_z > depth)
    return fail(c, PVR_ERR_ARG, "invalid patch size/stride (1 <= stride <= size, 1 <= stride_z <= depth)");
  for (auto& st : c->stacks)
    if (size > st.W || size > st.H || depth > st.K)
      return fail(c, PVR_ERR_ARG, "patch %dx%dx%d larger than a %dx%dx%d stack", size, size, depth,
                  st.W, st.H, st.K);
  pvr_status rb = begin_extraction(c);
  if (rb != PVR_OK) return rb;
  c->explicit_patches = false;
  // patch list, order stack, z0, y0, x0
  c->patches.clear();
  for (int si = 0; si < (int)c->stacks.size(); ++si) {
    const HostStack& st = c->stacks[si];
    for (int z0 : windows(st.K, depth, stride_z))
      for (int y0 : windows(st.H, size, stride))
        for (int x0 : windows(st.W, size, stride))
          c->patches.push_back(HostPatch{si, x0, y0, z0, size, size, depth});
  }
  return install_patches(c, nullptr, n_out);
}

// f3 (reading Q32): explicit patch rectangles [n][7] with an optional per-pixel mask.
pvr_status pvr_set_patches(pvr_ctx* c, int64_t n, const int32_t* rects, const uint8_t* mask, int64_t* n_out) {
  GUARD(c);
  if (c->state < STACKS) return fail(c, PVR_ERR_STATE, "set_patches needs stacks");
  if (n <= 0 || !rects) return fail(c, PVR_ERR_ARG, "set_patches needs n >= 1 rectangles");
  std::vector<int32_t> rh(7 * n);
  if (is_device_ptr(rects)) CUDA_TRY(c, cudaMemcpy(rh.data(), rects, rh.size() * 4, cudaMemcpyDeviceToHost));
  else memcpy(rh.data(), rects, rh.size() * 4);
  std::vector<HostPatch> list;
  for (int64_t s = 0; s < n; ++s) {
    const int32_t* r = &rh[7 * s];
    if (r[0] < 0 || r[0] >= (int)c->stacks.size()) return fail(c, PVR_ERR_ARG, "patch %lld: bad stack", (long long)s);
    const HostStack& st = c->stacks[r[0]];
    if (r[4] < 1 || r[5] < 1 || r[6] < 1 || r[1] < 0 || r[2] < 0 || r[3] < 0 || r[1] + r[4] > st.W ||
        r[2] + r[5] > st.H || r[3] + r[6] > st.K)
      return fail(c, PVR_ERR_ARG, "patch %lld outside its %dx%dx%d stack", (long long)s, st.W, st.H, st.K);
    list.push_back(HostPatch{r[0], r[1], r[2], r[3], r[4], r[5], r[6]});
  }
  pvr_status rb = begin_extraction(c);
  if (rb != PVR_OK) return rb;
  c->explicit_patches = true;
  c->patches.swap(list);
  return install_patches(c, mask, n_out);
}

// ---- f3 superpixels (superpixels.cu; readings Q32, Q33) -------------------------------
pvr_status pvr_superpixels(pvr_ctx* c, int stack, int S, int m, int iters, int32_t* labels) {
  GUARD(c);
  if (c->state < STACKS) return fail(c, PVR_ERR_STATE, "superpixels need the stacks");
  if (stack < 0 || stack >= (int)c->stacks.size() || S < 2 || m < 1 || iters < 0 || !labels)
    return fail(c, PVR_ERR_ARG, "superpixels: stack, S >= 2, m >= 1, iters >= 0, labels");
  const HostStack& st = c->stacks[stack];
  const size_t n = (size_t)st.W * st.H * st.K;
  int32_t* lab = nullptr;
  if (is_device_ptr(labels)) lab = labels;
  else CUDA_TRY(c, cudaMalloc(&lab, n * sizeof(int32_t)));
  const float* yd = st.y_dev ? st.y_dev : c->ys + st.y_off;  // before / after the first extraction
  cudaError_t e = slic_stack(c->stream, yd, st.W, st.H, st.K, S, m, iters, lab);
  if (e == cudaSuccess && lab != labels) e = cudaMemcpy(labels, lab, n * sizeof(int32_t), cudaMemcpyDeviceToHost);
  if (lab != labels) cudaFree(lab);
  if (e != cudaSuccess) return fail(c, PVR_ERR_CUDA, "superpixels: %s", cudaGetErrorString(e));
  return PVR_OK;
}

// Superpixel patches: per stack, slice and non-empty cluster (in that order) the cluster's
// bounding box dilated by gamma (clipped to the slice) and its mask = the cluster dilated by a
// (2 gamma + 1)^2 square (separable running max over rows, then columns).
pvr_status pvr_superpixel_patches(pvr_ctx* c, int S, int m, int iters, int gamma, int64_t* n_out) {
  GUARD(c);
  if (c->state < STACKS) return fail(c, PVR_ERR_STATE, "superpixel patches need stacks");
  if (S < 2 || m < 1 || iters < 0 || gamma < 0) return fail(c, PVR_ERR_ARG, "S >= 2, m >= 1, iters >= 0, gamma >= 0");
  Trace tr;
  std::vector<uint8_t> mask;
  std::vector<HostPatch> list;
  for (int si = 0; si < (int)c->stacks.size(); ++si) {
    const HostStack& st = c->stacks[si];
    const int W = st.W, H = st.H;
    std::vector<int32_t> lab((size_t)W * H * st.K);
    pvr_status r = pvr_superpixels(c, si, S, m, iters, lab.data());
    if (r != PVR_OK) return r;
    tr.mark("  SLIC (GPU) + labels D2H");
    const int nc = ((W + S - 1) / S) * ((H + S - 1) / S);
    // slices are independent: build their patches and masks in parallel, concatenate in order
    std::vector<std::vector<HostPatch>> sp(st.K);
    std::vector<std::vector<uint8_t>> sm(st.K);
#pragma omp parallel for schedule(dynamic, 1)
    for (int z = 0; z < st.K; ++z) {
      const int32_t* L = lab.data() + (size_t)z * W * H;
      std::vector<int> bx0(nc, W), bx1(nc, -1), by0(nc, H), by1(nc, -1);
      std::vector<uint8_t> rowd;
      for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
          const int k = L[(size_t)y * W + x];
          bx0[k] = std::min(bx0[k], x); bx1[k] = std::max(bx1[k], x);
          by0[k] = std::min(by0[k], y); by1[k] = std::max(by1[k], y);
        }
      for (int k = 0; k < nc; ++k) {
        if (bx1[k] < 0) continue;
        const int x0 = std::max(0, bx0[k] - gamma), x1 = std::min(W - 1, bx1[k] + gamma);
        const int y0 = std::max(0, by0[k] - gamma), y1 = std::min(H - 1, by1[k] + gamma);
        const int sx = x1 - x0 + 1, sy = y1 - y0 + 1;
        sp[z].push_back(HostPatch{si, x0, y0, z, sx, sy, 1});
        // horizontal dilation of (L == k) over the rectangle's rows (running count of hits in
        // the window [u - gamma, u + gamma] of the row)
        rowd.assign((size_t)sx * sy, 0);
        for (int v = 0; v < sy; ++v) {
          const int32_t* row = L + (size_t)(y0 + v) * W;
          int cnt = 0;
          for (int xx = std::max(0, x0 - gamma); xx <= std::min(W - 1, x0 + gamma - 1); ++xx) cnt += row[xx] == k;
          for (int u = 0; u < sx; ++u) {
            const int add = x0 + u + gamma, drop = x0 + u - gamma - 1;
            if (add < W) cnt += row[add] == k;
            if (drop >= 0) cnt -= row[drop] == k;
            rowd[(size_t)v * sx + u] = cnt > 0;
          }
        }
        // vertical dilation (rows outside the dilated box cannot hold the cluster)
        const size_t base = sm[z].size();
        sm[z].resize(base + (size_t)sx * sy);
        for (int u = 0; u < sx; ++u) {
          int cnt = 0;
          for (int vv = 0; vv <= std::min(sy - 1, gamma - 1); ++vv) cnt += rowd[(size_t)vv * sx + u];
          for (int v = 0; v < sy; ++v) {
            const int add = v + gamma, drop = v - gamma - 1;
            if (add < sy) cnt += rowd[(size_t)add * sx + u];
            if (drop >= 0) cnt -= rowd[(size_t)drop * sx + u];
            sm[z][base + (size_t)v * sx + u] = cnt > 0;
          }
        }
      }
    }
    for (int z = 0; z < st.K; ++z) {
      list.insert(list.end(), sp[z].begin(), sp[z].end());
      mask.insert(mask.end(), sm[z].begin(), sm[z].end());
    }
    tr.mark("  superpixel boxes + masks");
  }
  if (list.empty()) return fail(c, PVR_ERR_EMPTY, "no superpixels");
  pvr_status rb = begin_extraction(c);
  if (rb != PVR_OK) return rb;
  c->explicit_patches = true;
  c->patches.swap(list);
  return install_patches(c, mask.data(), n_out);
}

// Common tail of pvr_extract_patches / pvr_set_patches: PSF tables, pixel offsets, shards,
// the concatenated stacks and the per-pixel / per-patch device arrays.
static pvr_status install_patches(pvr_ctx* c, const uint8_t* mask, int64_t* n_out) {
  // PSF tables (host fp64 -> device fp32 factors)
  c->psf_tab.clear();
  for (auto& st : c->stacks) {
    pvr_status r = build_psf(c, st);
    if (r != PVR_OK) return r;
  }
  c->M = (int64_t)c->patches.size();
  if (c->M == 0) return fail(c, PVR_ERR_EMPTY, "no patches");
  c->pix0_global.assign(c->M + 1, 0);
  std::vector<int64_t> cost(c->M);
  for (int64_t s = 0; s < c->M; ++s) {
    const HostPatch& hp = c->patches[s];
    const int64_t npx = (int64_t)hp.sx * hp.sy * hp.sz;
    c->pix0_global[s + 1] = c->pix0_global[s] + npx;
    cost[s] = npx * c->stacks[hp.stack].S;
  }
  c->P = c->pix0_global[c->M];
  std::vector<int64_t> bounds(c->nranks + 1);
  pvr_plan_shards(cost.data(), c->M, c->nranks, bounds.data());
  c->first = bounds[c->rank];
  c->nloc = bounds[c->rank + 1] - bounds[c->rank];
  c->first_pix = c->pix0_global[c->first];
  c->nloc_pix = c->pix0_global[c->first + c->nloc] - c->first_pix;
  // concatenated stacks (once: a re-extraction keeps them)
  if (!c->ys) {
    int64_t L = 0;
    for (auto& st : c->stacks) { st.y_off = L; L += (int64_t)st.W * st.H * st.K; }
    CUDA_TRY(c, cudaMalloc(&c->ys, std::max<int64_t>(L, 1) * sizeof(float)));
    for (auto& st : c->stacks)
      CUDA_TRY(c, cudaMemcpyAsync(c->ys + st.y_off, st.y_dev, (size_t)st.W * st.H * st.K * sizeof(float),
                                  cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    for (auto& st : c->stacks) { cudaFree(st.y_dev); st.y_dev = nullptr; }
  }
  // per-pixel / per-patch arrays of the local shard
  const size_t np = (size_t)std::max<int64_t>(c->nloc_pix, 1), mp = (size_t)std::max<int64_t>(c->nloc, 1);
  CUDA_TRY(c, cudaMalloc(&c->e, np * sizeof(float)));
  CUDA_TRY(c, cudaMalloc(&c->p, np * sizeof(float)));
  CUDA_TRY(c, cudaMalloc(&c->kap, np * sizeof(float)));
  CUDA_TRY(c, cudaMalloc(&c->pbar, mp * sizeof(float)));
  CUDA_TRY(c, cudaMalloc(&c->w, mp * sizeof(float)));
  CUDA_TRY(c, cudaMalloc(&c->pdev, mp * sizeof(PatchDev)));
  std::vector<StackPsf> psd;
  for (auto& st : c->stacks) psd.push_back(st.psf);
  CUDA_TRY(c, cudaMalloc(&c->psf, psd.size() * sizeof(StackPsf)));
  CUDA_TRY(c, cudaMalloc(&c->tab, c->psf_tab.size() * sizeof(float)));
  CUDA_TRY(c, cudaMemcpyAsync(c->psf, psd.data(), psd.size() * sizeof(StackPsf), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->tab, c->psf_tab.data(), c->psf_tab.size() * sizeof(float),
                              cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->e, 0, np * sizeof(float), c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->p, 0, np * sizeof(float), c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->kap, 0, np * sizeof(float), c->stream));
  if (mask) {  // f3: this rank's slice of the per-pixel mask (masked pixels: kappa = 0)
    CUDA_TRY(c, cudaMalloc(&c->mask, np));
    CUDA_TRY(c, cudaMemcpyAsync(c->mask, mask + c->first_pix, c->nloc_pix,
                                is_device_ptr(mask) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
    c->mask_host.resize(c->nloc_pix);
    CUDA_TRY(c, cudaMemcpyAsync(c->mask_host.data(), c->mask, c->nloc_pix, cudaMemcpyDeviceToHost, c->stream));
  } else {
    c->mask_host.clear();
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->st.pixels = c->nloc_pix;
  c->st.patches = c->nloc;
  c->state = PATCHED;
  if (n_out) *n_out = c->M;
  return PVR_OK;
}

pvr_status pvr_get_mask(pvr_ctx* c, uint8_t* out) {
  GUARD(c);
  if (c->state < PATCHED) return fail(c, PVR_ERR_STATE, "no patches yet");
  if (!out) return fail(c, PVR_ERR_ARG, "null output");
  if (!c->mask) {
    if (is_device_ptr(out)) CUDA_TRY(c, cudaMemset(out, 1, c->nloc_pix));
    else memset(out, 1, c->nloc_pix);
    return PVR_OK;
  }
  CUDA_TRY(c, cudaMemcpy(out, c->mask, c->nloc_pix, is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
  return PVR_OK;
}

pvr_status pvr_get_shard(const pvr_ctx* c, int64_t* first, int64_t* nloc, int64_t* fpix, int64_t* npix) {
  if (!c) return fail(nullptr, PVR_ERR_ARG, "null context");
  if (c->state < PATCHED) return fail(const_cast<pvr_ctx*>(c), PVR_ERR_STATE, "no patches yet");
  if (first) *first = c->first;
  if (nloc) *nloc = c->nloc;
  if (fpix) *fpix = c->first_pix;
  if (npix) *npix = c->nloc_pix;
  return PVR_OK;
}

pvr_status pvr_get_patches(const pvr_ctx* c, int32_t* out) {
  if (!c || !out) return fail(nullptr, PVR_ERR_ARG, "null argument");
  if (c->state < PATCHED) return fail(const_cast<pvr_ctx*>(c), PVR_ERR_STATE, "no patches yet");
  for (int64_t s = 0; s < c->nloc; ++s) {
    const HostPatch& hp = c->patches[c->first + s];
    const int32_t v[7] = {hp.stack, hp.x0, hp.y0, hp.z0, hp.sx, hp.sy, hp.sz};
    memcpy(out + 7 * s, v, sizeof(v));
  }
  return PVR_OK;
}

static pvr_status replan_on_device(pvr_ctx* c);
static pvr_status prebuild_bp_table(pvr_ctx* c);

pvr_status pvr_set_transforms(pvr_ctx* c, const double* T, int64_t n) {
  GUARD(c);
  if (c->state < PATCHED) return fail(c, PVR_ERR_STATE, "set_transforms needs extract_patches");
  if (!T || n != c->M) return fail(c, PVR_ERR_ARG, "expected %lld transforms, got %lld", (long long)c->M, (long long)n);
  Trace tr;
  // the local transforms and the composed geometry go into scratch vectors that are swapped
  // with the context's at the end (no reallocation or zero fill per call: c5 has 876k patches)
  std::vector<double>& Th = c->T_next;
  Th.resize((size_t)12 * c->nloc);
  const double* Tl = T + 12 * c->first;
  if (is_device_ptr(T)) {
    CUDA_TRY(c, cudaMemcpy(Th.data(), Tl, Th.size() * sizeof(double), cudaMemcpyDeviceToHost));
  } else {
    const int64_t nchunk = 64, len = (int64_t)Th.size(), per = (len + nchunk - 1) / nchunk;
#pragma omp parallel for schedule(static) if (len >= (1 << 20))
    for (int64_t k = 0; k < nchunk; ++k) {
      const int64_t a = k * per, b = std::min(len, a + per);
      if (a < b) memcpy(Th.data() + a, Tl + a, (size_t)(b - a) * sizeof(double));
    }
  }
  // compose, per patch, in fp64: voxel index of lattice point (a,b,c) of pixel (u,v,z) is
  // g(T_s(G (x0+u, y0+v, z0+z, 1) + a h_u u^ + b h_v v^ + c h_w w^)), g(x) = (x - o) / s
  if (!c->pd_copied) CUDA_TRY(c, cudaEventCreateWithFlags(&c->pd_copied, cudaEventDisableTiming));
  CUDA_TRY(c, cudaEventSynchronize(c->pd_copied));  // the previous copy out of the buffer is done
  if (c->pd_host_n < c->nloc) {
    if (c->pd_host) cudaFreeHost(c->pd_host);
    c->pd_host = nullptr;
    c->pd_host_n = 0;
    CUDA_TRY(c, cudaMallocHost(&c->pd_host, std::max<int64_t>(c->nloc, 1) * sizeof(PatchDev)));
    c->pd_host_n = c->nloc;
  }
  PatchDev* pd = c->pd_host;
  std::vector<PatchGeo>& geo = c->geo_next;
  geo.resize(c->nloc);
  const double is = 1.0 / c->s;
#pragma omp parallel for schedule(static) if (c->nloc >= 2048)
  for (int64_t s = 0; s < c->nloc; ++s) {
    const HostPatch& hp = c->patches[c->first + s];
    const HostStack& st = c->stacks[hp.stack];
    const double* A = &Th[12 * s];
    PatchGeo& g = geo[s];
    auto lin = [&](const double* vec, double* out) {
      for (int d = 0; d < 3; ++d) out[d] = is * (A[4 * d] * vec[0] + A[4 * d + 1] * vec[1] + A[4 * d + 2] * vec[2]);
    };
    const double gu[3] = {st.G[0], st.G[4], st.G[8]}, gv[3] = {st.G[1], st.G[5], st.G[9]},
                 gz[3] = {st.G[2], st.G[6], st.G[10]};
    const double qa[3] = {st.h[0] * st.u[0], st.h[0] * st.u[1], st.h[0] * st.u[2]};
    const double qb[3] = {st.h[1] * st.v[0], st.h[1] * st.v[1], st.h[1] * st.v[2]};
    const double qc[3] = {st.h[2] * st.w[0], st.h[2] * st.w[1], st.h[2] * st.w[2]};
    double Mu[3], Mv[3];
    lin(gu, Mu);
    lin(gv, Mv);
    lin(gz, g.Mz);
    lin(qa, g.Qa);
    lin(qb, g.Qb);
    lin(qc, g.Qc);
    double w0[3];
    for (int d = 0; d < 3; ++d)
      w0[d] = st.G[4 * d] * hp.x0 + st.G[4 * d + 1] * hp.y0 + st.G[4 * d + 2] * hp.z0 + st.G[4 * d + 3];
    for (int d = 0; d < 3; ++d)
      g.t0[d] = ((A[4 * d] * w0[0] + A[4 * d + 1] * w0[1] + A[4 * d + 2] * w0[2] + A[4 * d + 3]) - c->o[d]) * is;
    PatchDev& q = pd[s];
    memset(&q, 0, sizeof(q));
    for (int d = 0; d < 3; ++d) {
      q.Mu[d] = (float)Mu[d]; q.Mv[d] = (float)Mv[d]; q.Mz[d] = (float)g.Mz[d];
      q.Qa[d] = (float)g.Qa[d]; q.Qb[d] = (float)g.Qb[d]; q.Qc[d] = (float)g.Qc[d];
      const double b = std::floor(g.t0[d]);
      q.base[d] = (int32_t)b;
      q.frac[d] = (float)(g.t0[d] - b);
    }
    q.stack = hp.stack;
    q.x0 = hp.x0; q.y0 = hp.y0; q.z0 = hp.z0;
    q.sx = hp.sx; q.sy = hp.sy; q.sz = hp.sz;
    q.pix0 = c->pix0_global[c->first + s] - c->first_pix;
    q.W = st.W;
    q.HW = st.W * st.H;
    q.y0off = st.y_off + ((int64_t)hp.z0 * st.H + hp.y0) * st.W + hp.x0;
    q.S = st.S;
    for (int d = 0; d < 3; ++d) {
      q.t0d[d] = g.t0[d];
      q.Mzd[d] = g.Mz[d];
      q.Qad[d] = g.Qa[d];
      q.Qbd[d] = g.Qb[d];
      q.Qcd[d] = g.Qc[d];
    }
  }
  CUDA_TRY(c, cudaMemcpyAsync(c->pdev, pd, c->nloc * sizeof(PatchDev), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaEventRecord(c->pd_copied, c->stream));
  ++c->geo_epoch;  // the backprojection tables are rebuilt by the next backprojection
  tr.mark("compose patches", c->stream);
  pvr_status r = PVR_OK;
  int nblk = kStatBlocks;  // per-block partials written by the coverage pass
  if (c->psf_mode == 2) {
    // volume-space PSF (reading Q34): per patch the fp64 pixel-centre map, the inverse map of
    // index offsets to slice-frame offsets and the support box; no lattice plans
    if (c->det) return fail(c, PVR_ERR_ARG, "the deterministic mode does not cover the volume-space PSF");
    std::vector<VolPatch> vp(c->nloc);
    for (int64_t s = 0; s < c->nloc; ++s) {
      const HostPatch& hp = c->patches[c->first + s];
      const HostStack& st = c->stacks[hp.stack];
      const double* A = &Th[12 * s];
      const PatchGeo& g = geo[s];
      VolPatch& q = vp[s];
      memset(&q, 0, sizeof(q));
      const double m00 = A[0], m01 = A[1], m02 = A[2], m10 = A[4], m11 = A[5], m12 = A[6], m20 = A[8], m21 = A[9],
                   m22 = A[10];
      const double det = m00 * (m11 * m22 - m12 * m21) - m01 * (m10 * m22 - m12 * m20) + m02 * (m10 * m21 - m11 * m20);
      if (!(std::fabs(det) > 1e-12)) return fail(c, PVR_ERR_ARG, "patch %lld: singular transform", (long long)s);
      const double Ai[9] = {(m11 * m22 - m12 * m21) / det, (m02 * m21 - m01 * m22) / det, (m01 * m12 - m02 * m11) / det,
                            (m12 * m20 - m10 * m22) / det, (m00 * m22 - m02 * m20) / det, (m02 * m10 - m00 * m12) / det,
                            (m10 * m21 - m11 * m20) / det, (m01 * m20 - m00 * m21) / det, (m00 * m11 - m01 * m10) / det};
      const double* frame[3] = {st.u, st.v, st.w};
      for (int r2 = 0; r2 < 3; ++r2)
        for (int c2 = 0; c2 < 3; ++c2) {
          double v = 0.0;
          for (int k = 0; k < 3; ++k) v += frame[r2][k] * Ai[3 * k + c2];
          q.Minv[3 * r2 + c2] = (float)(c->s * v);
          q.Minvd[3 * r2 + c2] = c->s * v;
        }
      const double gu[3] = {st.G[0], st.G[4], st.G[8]}, gv[3] = {st.G[1], st.G[5], st.G[9]};
      const double dx = norm3(gu), dy = norm3(gv), sw = st.theta / (2.0 * std::sqrt(2.0 * std::log(2.0)));
      const double cmax = c->nsigma * sw;
      for (int d = 0; d < 3; ++d) {
        const double b = std::floor(g.t0[d]);
        q.base[d] = (int32_t)b;
        q.xc[d] = (float)(g.t0[d] - b);
        q.xcd[d] = g.t0[d] - b;
        double mu = 0.0, mv = 0.0, au = 0.0, av = 0.0, aw = 0.0;
        for (int k = 0; k < 3; ++k) {
          mu += A[4 * d + k] * gu[k];
          mv += A[4 * d + k] * gv[k];
          au += A[4 * d + k] * st.u[k];
          av += A[4 * d + k] * st.v[k];
          aw += A[4 * d + k] * st.w[k];
        }
        q.Mu[d] = (float)(mu / c->s);
        q.Mv[d] = (float)(mv / c->s);
        q.Mz[d] = (float)g.Mz[d];
        q.Mud[d] = mu / c->s;
        q.Mvd[d] = mv / c->s;
        q.Mzd[d] = g.Mz[d];
        q.h[d] = (float)((std::fabs(au) * dx + std::fabs(av) * dy + std::fabs(aw) * cmax) / c->s + 1e-4);
      }
      q.idx = (float)(1.0 / dx);
      q.idy = (float)(1.0 / dy);
      q.i2s2 = (float)(1.0 / (2.0 * sw * sw));
      q.cmax = (float)cmax;
      q.dxd = dx;
      q.dyd = dy;
      q.cmaxd = cmax;
      q.sx = hp.sx; q.sy = hp.sy; q.sz = hp.sz;
      q.W = st.W;
      q.HW = st.W * st.H;
      q.pix0 = c->pix0_global[c->first + s] - c->first_pix;
      q.y0off = st.y_off + ((int64_t)hp.z0 * st.H + hp.y0) * st.W + hp.x0;
    }
    if (!c->vpat) CUDA_TRY(c, cudaMalloc(&c->vpat, std::max<int64_t>(c->nloc, 1) * sizeof(VolPatch)));
    if (!c->vin) CUDA_TRY(c, cudaMalloc(&c->vin, std::max<int64_t>(c->nloc_pix, 1) * sizeof(float)));
    CUDA_TRY(c, cudaMemcpyAsync(c->vpat, vp.data(), vp.size() * sizeof(VolPatch), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));  // vp goes out of scope
    c->geo.swap(geo);
    c->Tloc.swap(Th);
    const LatticeArgs la = lattice_args(c, c->fplan);
    launch_volpsf(c->stream, 1, c->vpat, c->nloc, la, nullptr, c->kap, c->vin, nullptr, nullptr, c->partials,
                  nullptr, nullptr, 0, nullptr);
    CHECK_LAUNCH(c);
  } else {
  if (c->fplan.ngroups > 0 && c->bplan.ngroups > 0) r = replan_on_device(c);
  else r = PVR_ERR_STATE;
  if (r != PVR_OK) {
    tr.mark("device replan (failed)");
    r = build_plans(c, geo, 0, 2);  // forward + backprojection; init plan: lazily
    ++c->st.host_replans;
  }
  if (r != PVR_OK) return r;
  c->iplan_valid = false;
  c->geo.swap(geo);
  c->Tloc.swap(Th);
  tr.mark("build plans", c->stream);
  r = encode_tmaps(c);
  if (r != PVR_OK) return r;
  tr.mark("tensor maps");
  r = prebuild_bp_table(c);
  if (r != PVR_OK) return r;
  // coverage kappa (geometry only) + live-y range, then the EM reset
  r = build_fwd_table(c);
  if (r != PVR_OK) return r;
  const LatticeArgs la = lattice_args(c, c->fplan);
  nblk = launch_coverage(c->stream, la, c->fplan.t_floats, c->fplan.tile_words, c->kap, c->partials);
  CHECK_LAUNCH(c);
  if (c->bplan.ngroups > 0) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_tab, 0));  // the tables
  tr.mark("coverage", c->stream);
  }
  launch_em_reduce(c->stream, c->partials, nblk, c->em);
  CHECK_LAUNCH(c);
  r = allreduce_stats(c);
  if (r != PVR_OK) return r;
  launch_range_finish(c->stream, c->s2floor, c->em);
  CHECK_LAUNCH(c);
  launch_fill(c->stream, c->p, c->nloc_pix, 1.0f);
  launch_fill(c->stream, c->pbar, c->nloc, 1.0f);
  launch_fill(c->stream, c->w, c->nloc, 1.0f);
  CHECK_LAUNCH(c);
  r = comm_wait(c);  // the coverage allreduce: NCCL errors abort instead of hanging
  if (r != PVR_OK) return r;
  EmDev h;
  CUDA_TRY(c, cudaMemcpyAsync(&h, c->em, sizeof(EmDev), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  tr.mark("coverage + EM reset (GPU)");
  if (!(h.stats[0] > 0)) return fail(c, PVR_ERR_EMPTY, "no observed pixel: nothing to reconstruct");
  // PSF samples visited per iteration (observed pixels x S, all ranks after the allreduce)
  c->samples_obs = (int64_t)h.stats[2];
  // algorithmic HBM bytes per launch: compulsory reads/writes only
  c->st.bytes_alg_forward = 16 * c->nloc_pix + 4 * c->V + 48 * c->nloc;    // y,kap,p in; e out; X; T
  c->st.bytes_alg_estep = 12 * c->nloc_pix + 8 * c->nloc;                   // kap,e in; p out; pbar,w
  c->st.bytes_alg_backproject = 12 * c->nloc_pix + 8 * c->V + 4 * c->nloc;  // kap,e,p in; A,C out
  c->st.bytes_alg_update = 16 * c->V;                                       // X0,A,C in; X2 out
  c->state = READY;
  return PVR_OK;
}

pvr_status pvr_set_volume(pvr_ctx* c, const float* x, size_t nvox) {
  GUARD(c);
  if (!x || (int64_t)nvox != c->V) return fail(c, PVR_ERR_ARG, "volume has %lld voxels", (long long)c->V);
  CUDA_TRY(c, cudaMemcpy2DAsync(c->X[c->cur], c->nxp * sizeof(float), x, c->dims.x * sizeof(float),
                                c->dims.x * sizeof(float), (size_t)c->dims.y * c->dims.z,
                                is_device_ptr(x) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return PVR_OK;
}

// Backprojection with the plan's member tables, rebuilt first when the geometry changed.
// The plan's member-table buffer (k_bp_table's output), grown on demand.
static pvr_status ensure_btab(pvr_ctx* c, pvr_ctx::Plan& pl) {
  size_t goff = 0;
  const size_t bytes = bp_table_bytes(pl.nmem, pl.ngroups, &goff);
  if (bytes > pl.btab_cap) {
    if (pl.btab) cudaFree(pl.btab);
    pl.btab = nullptr;
    pl.btab_cap = 0;
    CUDA_TRY(c, cudaMalloc(&pl.btab, bytes));
    pl.btab_cap = bytes;
    pl.btab_epoch = 0;
  }
  if (pl.btab_goff != goff) pl.btab_epoch = 0;
  pl.btab_goff = goff;
  return PVR_OK;
}

// set_transforms: build the iteration plan's member tables on the auxiliary stream (after the
// geometry upload and re-plan on the main stream), so that they overlap the coverage pass;
// the main stream joins them (ev_tab) before set_transforms returns.
static pvr_status prebuild_bp_table(pvr_ctx* c) {
  pvr_ctx::Plan& pl = c->bplan;
  if (pl.ngroups <= 0) return PVR_OK;
  pvr_status r = ensure_btab(c, pl);
  if (r != PVR_OK) return r;
  if (!c->aux) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
  if (!c->ev_geo) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_geo, cudaEventDisableTiming));
  if (!c->ev_tab) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_tab, cudaEventDisableTiming));
  CUDA_TRY(c, cudaEventRecord(c->ev_geo, c->stream));
  CUDA_TRY(c, cudaStreamWaitEvent(c->aux, c->ev_geo, 0));
  launch_bp_table(c->aux, lattice_args(c, pl), pl.btab, pl.btab_goff, pl.max_nm);
  CHECK_LAUNCH(c);
  CUDA_TRY(c, cudaEventRecord(c->ev_tab, c->aux));
  pl.btab_epoch = c->geo_epoch;
  c->st.kernel_launches += 1;
  return PVR_OK;
}

pvr_status backproject(pvr_ctx* c, cudaStream_t s, pvr_ctx::Plan& pl, const LatticeArgs& lb, const float* w,
                       int init) {
  pvr_status r = ensure_btab(c, pl);
  if (r != PVR_OK) return r;
  const size_t goff = pl.btab_goff;
  const bool build = pl.btab_epoch != c->geo_epoch;
  launch_backproject(s, lb, pl.tile_words, pl.r_bytes, pl.btab, goff, build, pl.max_nm, c->kap, c->e, c->p, w, init,
                     c->AC);
  CHECK_LAUNCH(c);
  if (build) {
    pl.btab_epoch = c->geo_epoch;
    c->st.kernel_launches += 1;
  }
  return PVR_OK;
}

// Backprojection into (A, C) and its exchange over ranks (init / rigidity: a sum-allreduce;
// iterations: PVR_PARAM_EXCHANGE). Deterministic mode: the global maxima of the inputs
// (atomicMax per rank, max-allreduce) fix one tile scale for every group, the tiles add into
// int64 accumulators (sum-allreduced exactly), and (A, C) is formed from them.
pvr_status backproject_reduce(pvr_ctx* c, cudaStream_t s, pvr_ctx::Plan& pl, const float* w, int init,
                              bool iteration) {
  const LatticeArgs lb0 = lattice_args(c, pl);
  if (c->psf_mode == 2) {  // volume-space PSF: direct adjoint (volpsf.cu)
    CUDA_TRY(c, cudaMemsetAsync(c->AC, 0, (c->Vp + 2) * sizeof(float2), s));
    launch_volpsf(s, 2, c->vpat, c->nloc, lb0, nullptr, c->kap, c->vin, nullptr, c->e, nullptr, w, c->p, init, c->AC);
    CHECK_LAUNCH(c);
    return iteration ? exchange_ac(c) : allreduce_ac(c);
  }
  if (!c->det) {
    CUDA_TRY(c, cudaMemsetAsync(c->AC, 0, (c->Vp + 2) * sizeof(float2), s));
    pvr_status r = backproject(c, s, pl, lb0, w, init);
    if (r != PVR_OK) return r;
    return iteration ? exchange_ac(c) : allreduce_ac(c);
  }
  if (!c->ACd) CUDA_TRY(c, cudaMalloc(&c->ACd, (size_t)(c->Vp + 2) * 4 * sizeof(unsigned long long)));
  const LatticeArgs lb = lattice_args(c, pl);
  CUDA_TRY(c, cudaMemsetAsync(c->em->det_max, 0, sizeof(c->em->det_max), s));
  launch_bp_maxima(s, c->pdev, c->nloc, lb.prm, c->kap, c->e, c->p, w, c->ys, init, c->em);
  CHECK_LAUNCH(c);
  pvr_status r = coll(c, c->em->det_max, 2, PVR_DT_F32, PVR_COLL_ALLREDUCE_MAX);
  if (r != PVR_OK) return r;
  launch_det_scales(s, c->em);
  CUDA_TRY(c, cudaMemsetAsync(c->ACd, 0, (size_t)(c->Vp + 2) * 4 * sizeof(unsigned long long), s));
  r = backproject(c, s, pl, lb, w, init);
  if (r != PVR_OK) return r;
  if (!(iteration && c->exchange == PVR_EXCHANGE_AVERAGE)) {
    r = coll(c, c->ACd, c->Vp * 4, PVR_DT_I64, PVR_COLL_ALLREDUCE_SUM);
    if (r != PVR_OK) return r;
  }
  launch_det_to_float(s, c->ACd, c->Vp, c->em, c->AC);
  CHECK_LAUNCH(c);
  c->st.kernel_launches += 3;
  return PVR_OK;
}

// The plan of the one-off exact passes (init, rigidity): the iteration's own plan when all its
// groups are exact (PVR_PARAM_BP_EXACT = 2), else the lazily built all-exact init plan (its
// groups fit the 16 B per cell budget).
static pvr_status exact_plan(pvr_ctx* c, pvr_ctx::Plan** pl) {
  if (c->bp_exact == kBpAll || c->det || c->psf_mode == 2) {  // (volume-space PSF: no plan)
    *pl = &c->bplan;
    return PVR_OK;
  }
  if (!c->iplan_valid) {
    pvr_status rp = build_plans(c, c->geo, 2, 3);
    if (rp != PVR_OK) return rp;
    c->iplan_valid = true;
  }
  *pl = &c->iplan;
  return PVR_OK;
}

pvr_status pvr_init_volume(pvr_ctx* c) {
  GUARD(c);
  if (c->state < READY) return fail(c, PVR_ERR_STATE, "init_volume needs set_transforms");
  pvr_ctx::Plan* pl = nullptr;
  pvr_status rp = exact_plan(c, &pl);
  if (rp != PVR_OK) return rp;
  const LatticeArgs lb = lattice_args(c, *pl);
  pvr_status r = backproject_reduce(c, c->stream, *pl, c->w, 1, false);
  if (r != PVR_OK) return r;
  launch_init_fill(c->stream, c->AC, c->dims, c->nxp, lb.prm, c->X[c->cur]);
  CHECK_LAUNCH(c);
  return comm_wait(c);
}

pvr_status pvr_rigidity_map(pvr_ctx* c, float* out, size_t nvox) {
  GUARD(c);
  if (c->state < READY) return fail(c, PVR_ERR_STATE, "rigidity_map needs set_transforms");
  if (!out || (int64_t)nvox != c->V) return fail(c, PVR_ERR_ARG, "volume has %lld voxels", (long long)c->V);
  pvr_ctx::Plan* pl = nullptr;
  pvr_status rp = exact_plan(c, &pl);
  if (rp != PVR_OK) return rp;
  // W^T (p pbar) and W^T 1 with exact hi/lo tiles (pbar rides in w)
  pvr_status r = backproject_reduce(c, c->stream, *pl, c->pbar, 2, false);
  if (r != PVR_OK) return r;
  r = comm_wait(c);
  if (r != PVR_OK) return r;
  float* tmp = c->X[1 - c->cur];  // scratch between iterations
  launch_ratio(c->stream, c->AC, c->dims, c->nxp, (float)c->tau_C, tmp);
  CHECK_LAUNCH(c);
  CUDA_TRY(c, cudaMemcpy2DAsync(out, c->dims.x * sizeof(float), tmp, c->nxp * sizeof(float),
                                c->dims.x * sizeof(float), (size_t)c->dims.y * c->dims.z,
                                is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return PVR_OK;
}

// set_transforms fast path: keep both plans' groups (membership, order, forward TMA boxes) and
// recompute their boxes for the new geometry on the device (k_replan). Falls back to the host
// planner (returns non-OK) when a forward footprint outgrew its box or a group its budget.
static pvr_status replan_on_device(pvr_ctx* c) {
  if (!c->replan_buf) CUDA_TRY(c, cudaMalloc(&c->replan_buf, 8 * sizeof(int)));
  CUDA_TRY(c, cudaMemsetAsync(c->replan_buf, 0, 8 * sizeof(int), c->stream));
  const int nshape = (int)(c->fbox.size() / 2);
  if (nshape <= 0 || nshape > kMaxBoxShapes) return PVR_ERR_ARG;
  if (!c->fbox_dev) CUDA_TRY(c, cudaMalloc(&c->fbox_dev, 2 * kMaxBoxShapes * sizeof(int)));
  CUDA_TRY(c, cudaMemcpyAsync(c->fbox_dev, c->fbox.data(), 2 * nshape * sizeof(int), cudaMemcpyHostToDevice,
                              c->stream));
  // forward: the planning budget + 50% (more X staged per CTA, 2-3 CTAs / SM until the next
  // host plan); backprojection: the hard tile budget (the host planned to 90% of it)
  launch_replan(c->stream, c->fplan.mem, c->fplan.grp, c->fplan.ngroups, (int)c->fplan.grp_cap, c->pdev, c->psf,
                1, c->dims, kFwdTileBytes / 4 * 3 / 2, c->fbox_dev, nshape, c->replan_buf, c->replan_buf + 1,
                nullptr, c->det ? kBpDet : c->bp_exact);
  // backprojection groups that outgrow the tile are split into single-member groups appended
  // after the plan's (their Morton locality is lost until the next host plan)
  launch_replan(c->stream, c->bplan.mem, c->bplan.grp, c->bplan.ngroups, (int)c->bplan.grp_cap, c->pdev, c->psf,
                0, c->dims, kBpTileBytes, nullptr, 0, c->replan_buf + 2, c->replan_buf + 3, c->replan_buf + 4,
                c->det ? kBpDet : c->bp_exact);
  CHECK_LAUNCH(c);
  int h[5];
  CUDA_TRY(c, cudaMemcpyAsync(h, c->replan_buf, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (getenv("PVR_TRACE"))
    fprintf(stderr, "[pvr] device replan: fwd max vox %d fail %d, bp max vox %d fail %d split members %d\n", h[0],
            h[1], h[2], h[3], h[4]);
  if (h[1] || h[3]) return PVR_ERR_ARG;
  c->bplan.ngroups += h[4];
  c->st.bp_groups = c->bplan.ngroups;
  c->st.replan_splits += h[4];
  c->fplan.tile_words = (h[0] + 3) & ~3;
  c->bplan.tile_words = (h[2] + 3) & ~3;
  c->st.fwd_smem = (int64_t)(c->fplan.t_floats + c->fplan.tile_words) * 4;
  ++c->st.device_replans;
  return PVR_OK;
}

// host src -> caller dst (host or device)
static pvr_status host_out(pvr_ctx* c, void* dst, const void* src, size_t bytes) {
  if (!dst || bytes == 0) return PVR_OK;
  if (is_device_ptr(dst)) CUDA_TRY(c, cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
  else memcpy(dst, src, bytes);
  return PVR_OK;
}

// ---- f1: rigid patch-to-volume registration (registration.cu; reading Q29) ----------
static void pose_rotation_host(const double* p, double R[9]) {
  const double k = M_PI / 180.0;
  const double cx = cos(k * p[3]), sx = sin(k * p[3]), cy = cos(k * p[4]), sy = sin(k * p[4]);
  const double cz = cos(k * p[5]), sz = sin(k * p[5]);
  const double Ryx[9] = {cy, sy * sx, sy * cx, 0.0, cx, -sx, -sy, cy * sx, cy * cx};
  const double Rz[9] = {cz, -sz, 0.0, sz, cz, 0.0, 0.0, 0.0, 1.0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      R[3 * i + j] = Rz[3 * i] * Ryx[j] + Rz[3 * i + 1] * Ryx[3 + j] + Rz[3 * i + 2] * Ryx[6 + j];
}

// Per-patch geometry for the registration kernels (fp64, from the last set_transforms).
static pvr_status upload_reg_patches(pvr_ctx* c, int& max_pix) {
  std::vector<RegPatch> rp(c->nloc);
  max_pix = 1;
  for (int64_t s = 0; s < c->nloc; ++s) {
    const HostPatch& hp = c->patches[c->first + s];
    const HostStack& st = c->stacks[hp.stack];
    const double* A = &c->Tloc[12 * s];
    auto world = [&](double u, double v, double z, double out[3]) {
      double w[3];
      for (int d = 0; d < 3; ++d)
        w[d] = st.G[4 * d] * (hp.x0 + u) + st.G[4 * d + 1] * (hp.y0 + v) + st.G[4 * d + 2] * (hp.z0 + z) + st.G[4 * d + 3];
      for (int d = 0; d < 3; ++d) out[d] = A[4 * d] * w[0] + A[4 * d + 1] * w[1] + A[4 * d + 2] * w[2] + A[4 * d + 3];
    };
    RegPatch& q = rp[s];
    memset(&q, 0, sizeof(q));
    world(0, 0, 0, q.m0);
    double t[3];
    world(1, 0, 0, t);
    for (int d = 0; d < 3; ++d) q.mu[d] = t[d] - q.m0[d];
    world(0, 1, 0, t);
    for (int d = 0; d < 3; ++d) q.mv[d] = t[d] - q.m0[d];
    world(0, 0, 1, t);
    for (int d = 0; d < 3; ++d) q.mz[d] = t[d] - q.m0[d];
    world(0.5 * (hp.sx - 1), 0.5 * (hp.sy - 1), 0.5 * (hp.sz - 1), q.c);
    q.y0off = st.y_off + ((int64_t)hp.z0 * st.H + hp.y0) * st.W + hp.x0;
    q.W = st.W;
    q.HW = st.W * st.H;
    q.sx = hp.sx; q.sy = hp.sy; q.sz = hp.sz;
    max_pix = std::max(max_pix, hp.sx * hp.sy * hp.sz);
  }
  if ((size_t)c->nloc > c->regP_cap) {
    if (c->regP) cudaFree(c->regP);
    c->regP = nullptr;
    CUDA_TRY(c, cudaMalloc(&c->regP, std::max<int64_t>(c->nloc, 1) * sizeof(RegPatch)));
    c->regP_cap = c->nloc;
  }
  CUDA_TRY(c, cudaMemcpyAsync(c->regP, rp.data(), rp.size() * sizeof(RegPatch), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if ((int64_t)max_pix * 4 > 190 * 1024) return fail(c, PVR_ERR_ARG, "patch of %d pixels too large to register", max_pix);
  return PVR_OK;
}

static RegArgs reg_args(const pvr_ctx* c, int levels, int iters) {
  RegArgs a;
  memset(&a, 0, sizeof(a));
  a.P = c->regP;
  a.X = c->X[c->cur];
  a.ys = c->ys;
  a.n = c->dims;
  a.nxp = c->nxp;
  for (int d = 0; d < 3; ++d) a.o[d] = c->o[d];
  a.s = c->s;
  a.levels = levels;
  a.iters = iters;
  a.min_valid = 32;
  return a;
}

pvr_status pvr_register_patches(pvr_ctx* c, int levels, int iters, double* T_out, int32_t* status, float* poses) {
  GUARD(c);
  if (c->state < READY) return fail(c, PVR_ERR_STATE, "register_patches needs set_transforms");
  if (levels < 1 || levels > 16 || iters < 0) return fail(c, PVR_ERR_ARG, "levels in [1, 16], iters >= 0");
  int max_pix = 1;
  pvr_status r = upload_reg_patches(c, max_pix);
  if (r != PVR_OK) return r;
  float* dpose = nullptr;
  int32_t* dst = nullptr;
  CUDA_TRY(c, cudaMalloc(&dpose, std::max<int64_t>(c->nloc, 1) * 6 * sizeof(float)));
  cudaError_t e2 = cudaMalloc(&dst, std::max<int64_t>(c->nloc, 1) * sizeof(int32_t));
  if (e2 != cudaSuccess) { cudaFree(dpose); return fail(c, PVR_ERR_OOM, "register buffers"); }
  cudaMemsetAsync(dpose, 0, c->nloc * 6 * sizeof(float), c->stream);
  launch_register(c->stream, reg_args(c, levels, iters), (int)c->nloc, max_pix, dpose, dst);
  cudaError_t le = cudaGetLastError();
  std::vector<float> hp(6 * c->nloc);
  std::vector<int32_t> hs(c->nloc);
  cudaMemcpyAsync(hp.data(), dpose, hp.size() * sizeof(float), cudaMemcpyDeviceToHost, c->stream);
  cudaMemcpyAsync(hs.data(), dst, hs.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream);
  cudaError_t se = cudaStreamSynchronize(c->stream);
  cudaFree(dpose);
  cudaFree(dst);
  if (le != cudaSuccess || se != cudaSuccess)
    return fail(c, PVR_ERR_CUDA, "register kernel: %s", cudaGetErrorString(le != cudaSuccess ? le : se));
  // T_new = T_pose o T_s in fp64 (the kernel returns the pose parameters)
  std::vector<double> Tn(12 * c->nloc);
  for (int64_t s = 0; s < c->nloc; ++s) {
    const double* T = &c->Tloc[12 * s];
    double* o = &Tn[12 * s];
    if (!hs[s]) { memcpy(o, T, 12 * sizeof(double)); continue; }
    double p[6], R[9], ctr[3];
    for (int k = 0; k < 6; ++k) p[k] = hp[6 * s + k];
    pose_rotation_host(p, R);
    const HostPatch& h = c->patches[c->first + s];
    const HostStack& st = c->stacks[h.stack];
    double w[3];
    const double uu = h.x0 + 0.5 * (h.sx - 1), vv = h.y0 + 0.5 * (h.sy - 1), zz = h.z0 + 0.5 * (h.sz - 1);
    for (int d = 0; d < 3; ++d) w[d] = st.G[4 * d] * uu + st.G[4 * d + 1] * vv + st.G[4 * d + 2] * zz + st.G[4 * d + 3];
    for (int d = 0; d < 3; ++d) ctr[d] = T[4 * d] * w[0] + T[4 * d + 1] * w[1] + T[4 * d + 2] * w[2] + T[4 * d + 3];
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) o[4 * i + j] = R[3 * i] * T[j] + R[3 * i + 1] * T[4 + j] + R[3 * i + 2] * T[8 + j];
      o[4 * i + 3] = R[3 * i] * (T[3] - ctr[0]) + R[3 * i + 1] * (T[7] - ctr[1]) + R[3 * i + 2] * (T[11] - ctr[2]) +
                     ctr[i] + p[i];
    }
  }
  if (T_out) {
    r = host_out(c, T_out + 12 * c->first, Tn.data(), Tn.size() * sizeof(double));
    if (r != PVR_OK) return r;
  }
  if (status) {
    r = host_out(c, status + c->first, hs.data(), hs.size() * sizeof(int32_t));
    if (r != PVR_OK) return r;
  }
  if (poses) {
    r = host_out(c, poses + 6 * c->first, hp.data(), hp.size() * sizeof(float));
    if (r != PVR_OK) return r;
  }
  return PVR_OK;
}

pvr_status pvr_patch_cc(pvr_ctx* c, int64_t n, const int64_t* patch, const float* poses, double* cc) {
  GUARD(c);
  if (c->state < READY) return fail(c, PVR_ERR_STATE, "patch_cc needs set_transforms");
  if (n < 0 || (n > 0 && (!patch || !poses || !cc))) return fail(c, PVR_ERR_ARG, "patch_cc arguments");
  if (n == 0) return PVR_OK;
  std::vector<int64_t> ph(n);
  std::vector<float> qh(6 * n);
  if (is_device_ptr(patch)) CUDA_TRY(c, cudaMemcpy(ph.data(), patch, n * sizeof(int64_t), cudaMemcpyDeviceToHost));
  else memcpy(ph.data(), patch, n * sizeof(int64_t));
  if (is_device_ptr(poses)) CUDA_TRY(c, cudaMemcpy(qh.data(), poses, 6 * n * sizeof(float), cudaMemcpyDeviceToHost));
  else memcpy(qh.data(), poses, 6 * n * sizeof(float));
  std::vector<int32_t> wh(n);
  for (int64_t i = 0; i < n; ++i) {
    if (ph[i] < c->first || ph[i] >= c->first + c->nloc) return fail(c, PVR_ERR_ARG, "patch %lld not on this rank", (long long)ph[i]);
    wh[i] = (int32_t)(ph[i] - c->first);
  }
  int max_pix = 1;
  pvr_status r = upload_reg_patches(c, max_pix);
  if (r != PVR_OK) return r;
  int32_t* dw = nullptr;
  float* dq = nullptr;
  double* dc = nullptr;
  cudaError_t e = cudaMalloc(&dw, n * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&dq, 6 * n * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&dc, n * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpyAsync(dw, wh.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dq, qh.data(), 6 * n * sizeof(float), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) {
    launch_patch_cc(c->stream, reg_args(c, 1, 0), (int)n, max_pix, dw, dq, dc);
    e = cudaGetLastError();
  }
  std::vector<double> hc(n);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hc.data(), dc, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(dw);
  cudaFree(dq);
  cudaFree(dc);
  if (e != cudaSuccess) return fail(c, PVR_ERR_CUDA, "patch_cc: %s", cudaGetErrorString(e));
  return host_out(c, cc, hc.data(), n * sizeof(double));
}

pvr_status pvr_sr_iterate(pvr_ctx* c, int n, float alpha, float lambda) {
  GUARD(c);
  if (c->state < READY) return fail(c, PVR_ERR_STATE, "sr_iterate needs set_transforms");
  if (n < 0 || !(alpha >= 0) || !(lambda >= 0)) return fail(c, PVR_ERR_ARG, "n, alpha, lambda must be >= 0");
  if (c->psf_mode != 2) {
    pvr_status rt = build_fwd_table(c);
    if (rt != PVR_OK) return rt;
  }
  const LatticeArgs la = lattice_args(c, c->fplan), lb = lattice_args(c, c->bplan);
  const Params prm = la.prm;
  const bool prof = c->profile != 0;
  if (c->em_rounds > 1 && !c->rpart)
    CUDA_TRY(c, cudaMalloc(&c->rpart, (size_t)std::max<int64_t>(c->nloc, 1) * 3 * sizeof(double)));
  if (c->patch_mixture && !c->nlivep)
    CUDA_TRY(c, cudaMalloc(&c->nlivep, (size_t)std::max<int64_t>(c->nloc, 1) * sizeof(int32_t)));
  int32_t* nl = c->patch_mixture ? c->nlivep : nullptr;
  cudaStream_t s = c->stream;
  for (int it = 0; it < n; ++it) {
    float* X0 = c->X[c->cur];
    float* X2 = c->X[1 - c->cur];
    std::vector<cudaEvent_t>* ev = prof ? prof_slot(c) : nullptr;
    if (prof) cudaEventRecord((*ev)[EV_FWD0], s);
    if (c->psf_mode == 2)
      launch_volpsf(s, 0, c->vpat, c->nloc, la, X0, c->kap, c->vin, c->p, c->e, c->partials, nullptr, nullptr, 0,
                    nullptr);
    else
      launch_forward(s, la, c->fplan.t_floats, c->fplan.tile_words, c->tmaps + c->cur * (c->fbox.size() / 2) * 128,
                     c->kap, c->p, c->e, c->partials);
    CHECK_LAUNCH(c);
    if (prof) cudaEventRecord((*ev)[EV_FWD1], s);
    launch_em_reduce(s, c->partials, kStatBlocks, c->em);
    CHECK_LAUNCH(c);
    pvr_status r = allreduce_stats(c);
    if (r != PVR_OK) return r;
    launch_em_params(s, prm, c->em);
    CHECK_LAUNCH(c);
    if (prof) cudaEventRecord((*ev)[EV_EM1], s);
    launch_estep(s, c->pdev, c->nloc, prm, c->em, c->kap, c->e, c->p, c->pbar, c->w, 1,
                 c->em_rounds > 1 ? c->rpart : nullptr, nl);
    CHECK_LAUNCH(c);
    // f4 multi-round EM (reading Q30): rounds 2..R re-run M and E on the same residuals until
    // the log-likelihood gain falls below tol |LL| (decided on the device: later launches
    // of a converged iteration are no-ops)
    for (int round = 2; round <= c->em_rounds; ++round) {
      launch_em_reduce3(s, c->rpart, c->nloc, c->em);
      pvr_status r2 = allreduce_stats2(c);
      if (r2 != PVR_OK) return r2;
      launch_em_round(s, prm, c->em, round, c->em_tol);
      launch_estep(s, c->pdev, c->nloc, prm, c->em, c->kap, c->e, c->p, c->pbar, c->w, round, c->rpart, nl);
      CHECK_LAUNCH(c);
      c->st.kernel_launches += 3;
    }
    // f4 two-Gaussian patch classification (reading Q31): w from the mixture posterior
    if (c->patch_mixture) {
      launch_mix_init(s, c->pbar, c->nlivep, c->nloc, c->em);
      pvr_status rm = allreduce_mix(c, 0);
      if (rm != PVR_OK) return rm;
      launch_mix_params_init(s, c->em);
      for (int round = 0; round < kMixRounds; ++round) {
        launch_mix_round(s, c->pbar, c->nlivep, c->nloc, c->em, c->w);
        rm = allreduce_mix(c, 1);
        if (rm != PVR_OK) return rm;
        launch_mix_update(s, c->em, round, 1e-6);
      }
      launch_mix_weights(s, c->nlivep, c->nloc, c->em, c->w);
      CHECK_LAUNCH(c);
      c->st.kernel_launches += 3 + 2 * kMixRounds;
    }
    if (prof) cudaEventRecord((*ev)[EV_EST1], s);
    r = backproject_reduce(c, s, c->bplan, c->w, 0, true);
    if (r != PVR_OK) return r;
    if (prof) cudaEventRecord((*ev)[EV_BP1], s);
    if (prof) cudaEventRecord((*ev)[EV_AR1], s);
    const bool slabs = c->nranks > 1 && c->exchange == PVR_EXCHANGE_SLABS;
    launch_update(s, X0, c->AC, c->dims, c->nxp, prm, c->em, alpha, lambda, X2, slabs ? c->z0 : 0,
                  slabs ? c->z1 : c->dims.z);
    CHECK_LAUNCH(c);
    r = exchange_x(c, X2);
    if (r != PVR_OK) return r;
    if (prof) cudaEventRecord((*ev)[EV_UPD1], s);
    c->cur = 1 - c->cur;
    c->st.iterations += 1;
    c->st.psf_samples += c->samples_obs;
    c->st.kernel_launches += 6;  // forward, em_reduce, em_params, estep, backproject, update
    c->st.n_forward += 1; c->st.n_em += 1; c->st.n_estep += 1; c->st.n_backproject += 1;
    c->st.n_update += 1;
    if (c->nranks > 1) c->st.n_allreduce += 1;
    if (c->prof_pending.size() >= 512) prof_drain(c);
  }
  if (c->comm) {  // poll NCCL's asynchronous errors while the iterations drain (comm_wait)
    pvr_status rw = comm_wait(c);
    if (rw != PVR_OK) return rw;
  }
  if ((double)alpha * lambda > 3.0 / 44.0)
    c->err = "warning: alpha*lambda > 3/44, the regulariser's maximum principle does not hold";
  return PVR_OK;
}

// One quantity (0: A, 1: C) of the interleaved, row-padded (A, C) volume into a caller
// buffer [nz][ny][nx]: unpacked on the device (k_unpack_ac) straight into a device output, or
// into the scratch X buffer and copied to a host output.
static pvr_status unpack_ac(pvr_ctx* c, int which, float* out) {
  const bool dev = is_device_ptr(out);
  float* dst = dev ? out : c->X[1 - c->cur];  // scratch between iterations
  launch_unpack_ac(c->stream, c->AC, c->dims, c->nxp, which, dst);
  CHECK_LAUNCH(c);
  if (!dev) CUDA_TRY(c, cudaMemcpyAsync(out, dst, c->V * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return PVR_OK;
}

pvr_status pvr_get_confidence(pvr_ctx* c, float* out, size_t nvox) {
  GUARD(c);
  if (c->state < READY) return fail(c, PVR_ERR_STATE, "no confidence before set_transforms");
  if (!out || (int64_t)nvox != c->V) return fail(c, PVR_ERR_ARG, "volume has %lld voxels", (long long)c->V);
  return unpack_ac(c, 1, out);
}

pvr_status pvr_get_volume(pvr_ctx* c, float* out, size_t nvox) {
  GUARD(c);
  if (!out || (int64_t)nvox != c->V) return fail(c, PVR_ERR_ARG, "volume has %lld voxels", (long long)c->V);
  CUDA_TRY(c, cudaMemcpy2DAsync(out, c->dims.x * sizeof(float), c->X[c->cur], c->nxp * sizeof(float),
                                c->dims.x * sizeof(float), (size_t)c->dims.y * c->dims.z,
                                is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return PVR_OK;
}

static pvr_status copy_out(pvr_ctx* c, void* dst, const void* src, size_t bytes) {
  if (!dst || bytes == 0) return PVR_OK;
  CUDA_TRY(c, cudaMemcpyAsync(dst, src, bytes, is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                              c->stream));
  return PVR_OK;
}

pvr_status pvr_get_weights(pvr_ctx* c, float* pp, float* pw, float* pb) {
  GUARD(c);
  if (c->state < READY) return fail(c, PVR_ERR_STATE, "no weights before set_transforms");
  pvr_status r;
  if ((r = copy_out(c, pp, c->p, c->nloc_pix * sizeof(float))) != PVR_OK) return r;
  if ((r = copy_out(c, pw, c->w, c->nloc * sizeof(float))) != PVR_OK) return r;
  if ((r = copy_out(c, pb, c->pbar, c->nloc * sizeof(float))) != PVR_OK) return r;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return PVR_OK;
}

static pvr_status copy_in(pvr_ctx* c, void* dst, const void* src, size_t bytes) {
  if (!src || bytes == 0) return PVR_OK;
  CUDA_TRY(c, cudaMemcpyAsync(dst, src, bytes, is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                              c->stream));
  return PVR_OK;
}

// Checkpoint / resume: the state one SR iteration carries into the next is X, the
// pixel probabilities p (the forward's M-step partials weight by the previous p) and
// the EM counter t (c = c0 at t = 1, reading Q10); w and pbar are re-formed by every E-step.
pvr_status pvr_set_weights(pvr_ctx* c, const float* pp, const float* pw, const float* pb) {
  GUARD(c);
  if (c->state < READY) return fail(c, PVR_ERR_STATE, "set_weights needs set_transforms");
  pvr_status r;
  if ((r = copy_in(c, c->p, pp, c->nloc_pix * sizeof(float))) != PVR_OK) return r;
  if ((r = copy_in(c, c->w, pw, c->nloc * sizeof(float))) != PVR_OK) return r;
  if ((r = copy_in(c, c->pbar, pb, c->nloc * sizeof(float))) != PVR_OK) return r;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return PVR_OK;
}

pvr_status pvr_set_em_state(pvr_ctx* c, double sigma2, double cc, double m, int64_t it) {
  GUARD(c);
  if (c->state < READY) return fail(c, PVR_ERR_STATE, "set_em_state needs set_transforms");
  if (it < 0 || !(sigma2 >= 0) || !(cc >= 0 && cc <= 1) || !(m >= 0))
    return fail(c, PVR_ERR_ARG, "need iter >= 0, sigma2 >= 0, 0 <= c <= 1, m >= 0");
  EmDev h;
  CUDA_TRY(c, cudaMemcpyAsync(&h, c->em, sizeof(EmDev), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  h.sigma2 = sigma2;
  h.c = cc;
  h.m = m;
  h.t = it;
  CUDA_TRY(c, cudaMemcpyAsync(c->em, &h, sizeof(EmDev), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return PVR_OK;
}

pvr_status pvr_get_taps(pvr_ctx* c, float* e, float* kap, float* A, float* C) {
  GUARD(c);
  if (c->state < READY) return fail(c, PVR_ERR_STATE, "no taps before set_transforms");
  pvr_status r;
  if ((r = copy_out(c, e, c->e, c->nloc_pix * sizeof(float))) != PVR_OK) return r;
  if ((r = copy_out(c, kap, c->kap, c->nloc_pix * sizeof(float))) != PVR_OK) return r;
  if (A && (r = unpack_ac(c, 0, A)) != PVR_OK) return r;
  if (C && (r = unpack_ac(c, 1, C)) != PVR_OK) return r;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return PVR_OK;
}

pvr_status pvr_get_em_state(pvr_ctx* c, double* sigma2, double* cc, double* m, int64_t* it, double* lo,
                            double* hi) {
  GUARD(c);
  EmDev h;
  CUDA_TRY(c, cudaMemcpyAsync(&h, c->em, sizeof(EmDev), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (sigma2) *sigma2 = h.sigma2;
  if (cc) *cc = h.c;
  if (m) *m = h.m;
  if (it) *it = h.t;
  if (lo) *lo = h.lo;
  if (hi) *hi = h.hi;
  return PVR_OK;
}

pvr_status pvr_get_stats(const pvr_ctx* cc, pvr_stats* out) {
  if (!cc || !out) return fail(nullptr, PVR_ERR_ARG, "null argument");
  pvr_ctx* c = const_cast<pvr_ctx*>(cc);
  cudaSetDevice(c->device);
  prof_drain(c);
  *out = c->st;
  return PVR_OK;
}

pvr_status pvr_reset_stats(pvr_ctx* c) {
  if (!c) return fail(nullptr, PVR_ERR_ARG, "null context");
  cudaSetDevice(c->device);
  prof_drain(c);
  pvr_stats keep = c->st;
  memset(&c->st, 0, sizeof(c->st));
  c->st.pixels = keep.pixels; c->st.voxels = keep.voxels; c->st.patches = keep.patches;
  c->st.bytes_alg_forward = keep.bytes_alg_forward;
  c->st.bytes_alg_estep = keep.bytes_alg_estep;
  c->st.bytes_alg_backproject = keep.bytes_alg_backproject;
  c->st.bytes_alg_update = keep.bytes_alg_update;
  memcpy(c->st.fwd_tile, keep.fwd_tile, sizeof(keep.fwd_tile));
  memcpy(c->st.bp_tile, keep.bp_tile, sizeof(keep.bp_tile));
  c->st.fwd_groups = keep.fwd_groups; c->st.bp_groups = keep.bp_groups;
  c->st.fwd_members = keep.fwd_members; c->st.bp_members = keep.bp_members;
  c->st.fwd_smem = keep.fwd_smem; c->st.bp_smem = keep.bp_smem;
  c->st.bp_exact_groups = keep.bp_exact_groups;
  c->st.fwd_split = keep.fwd_split; c->st.bp_split = keep.bp_split;
  return PVR_OK;
}

}  // extern "C"

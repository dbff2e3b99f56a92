// C-ABI implementation (include/csf_b200.h): contexts, volumes, stage calls
// and the device-resident CSFD frame-derivative pipeline.
//
// The host code only orders launches and moves buffers; every numeric stage
// runs in the kernels of frames.cu / volume.cu / icp.cu.  A missing or
// failing CUDA device is reported as an error — there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <sstream>
#include <fstream>
#include <atomic>
#include <limits>
#include <mutex>
#include <memory>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is opened at runtime (csf_ctx_attach_comm)

#include "../../include/csf_b200.h"
#include "../../include/csf_detmath.h"
#include "csf_internal.h"
#include "geometry.cuh"

namespace csfi {
int synth_workload(cudaStream_t stream, int config, int n_frames, int width, int height, float* depth_out,
                   double* gt_out, csf_intrinsics* k_out, std::string* err);
int band_samples(double mu, double vs);
size_t alloc_scan_bytes(int n);
}  // namespace csfi

using namespace csfi;

// Per-category kernel timing with CUDA events on the context stream
// (bench.py's roofline numbers).  Off unless csf_ctx_profile(ctx, 1).
struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::pair<int, size_t>> recs;  // (category, first event index)
  cudaEvent_t ev() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
};

enum ProfCat {
  kPBilateral = 0, kPDownsample, kPRaycast, kPRaycastLift, kPIcpReduce, kPIcpSolve, kPAlloc, kPIntegrate, kPMisc,
  kPRelocLoss, kPRelocGrad, kPRelocHess, kPN
};
static const char* kProfNames[kPN] = {"bilateral", "downsample", "raycast", "raycast_lift", "icp", "icp_solve",
                                      "allocate", "integrate", "misc", "reloc_loss", "reloc_grad", "reloc_hess"};

struct csf_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int* d_err = nullptr;
  unsigned long long launches = 0;
  std::string last_error;
  Profiler prof;
  EnergyScratch energy;     // icp energy / correspondence-list scratch
  double* corr_upload = nullptr;
  size_t corr_upload_cap = 0;
  // direction-sharded runs: the NCCL communicator of csf_gather_columns
  ncclComm_t comm = nullptr;
  int n_ranks = 1, rank = 0;
  double* gather_buf = nullptr;
  size_t gather_cap = 0;
};

// Brackets a launch with events when profiling is on.
struct ProfScope {
  csf_ctx ctx;
  int cat;
  size_t first = 0;
  ProfScope(csf_ctx c, int k) : ctx(c), cat(k) {
    if (ctx->prof.on) {
      first = ctx->prof.used;
      cudaEventRecord(ctx->prof.ev(), ctx->stream);
    }
  }
  ~ProfScope() {
    if (ctx->prof.on) {
      cudaEventRecord(ctx->prof.ev(), ctx->stream);
      ctx->prof.recs.emplace_back(cat, first);
    }
  }
};
#define PROF(ctx, cat) ProfScope _prof_scope_##__LINE__((ctx), (cat))

namespace {

int fail(csf_ctx ctx, int code, const std::string& msg) {
  if (ctx) ctx->last_error = msg;
  return code;
}

#define CUDA_TRY(ctx, expr)                                                                     \
  do {                                                                                          \
    const cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                      \
      return fail(ctx, _e == cudaErrorMemoryAllocation ? CSF_ENOMEM : CSF_ECUDA,                \
                  std::string(#expr) + ": " + cudaGetErrorString(_e));                          \
  } while (0)

Launch launch_of(csf_ctx ctx) { return Launch{ctx->stream, ctx->d_err, &ctx->launches}; }

// Device->host copy that is complete when it returns: host buffers are only
// borrowed for the duration of a call (csf_b200.h), and a pinned destination
// would otherwise still be in flight when the caller reads it.
cudaError_t d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
  return e != cudaSuccess ? e : cudaStreamSynchronize(s);
}

// Synchronise and translate the device error flag into a status code.
int sync_check(csf_ctx ctx, const char* what) {
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  CUDA_TRY(ctx, cudaGetLastError());
  char lmsg[256];
  if (take_launch_error(lmsg, sizeof(lmsg))) return fail(ctx, CSF_ECUDA, std::string(what) + ": " + lmsg);
  int err = 0;
  CUDA_TRY(ctx, d2h(&err, ctx->d_err, sizeof(int), ctx->stream));
  if (err != 0) {
    cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream);
    if (err == 2) return fail(ctx, CSF_EDOMAIN, std::string(what) + ": division by a zero real part");
    if (err == 5) return fail(ctx, CSF_ENOMEM, std::string(what) + ": hashed volume capacity exhausted");
    return fail(ctx, CSF_ERUNTIME, std::string(what) + ": device error");
  }
  return CSF_OK;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }  // function-local scratch is freed on every return path
  cudaError_t alloc(size_t count) {
    if (count <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    const cudaError_t e = cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1));
    if (e == cudaSuccess) n = count;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

}  // namespace

// ---------------------------------------------------------------------------
// volume
// ---------------------------------------------------------------------------
struct csf_volume_s {
  csf_ctx ctx = nullptr;
  bool hashed = false;
  int D = 0, G = 0, Dp = 0, order = 1;
  DenseDev dense{};
  HashDev hash{};
  long long n_vox = 0;  // dense voxel count / pool voxel capacity
  DevBuf<double2> rw;
  DevBuf<double> fim;
  DevBuf<int> heads, next, coords, nblocks, grid;
  DevBuf<unsigned> occ;
  DevBuf<unsigned char> sdist;
  DevBuf<unsigned long long> keys;
  // allocation scratch (hashed)
  AllocScratch alloc{};
  DevBuf<unsigned long long> a_cand, a_set_keys;
  DevBuf<int> a_cand_block, a_first_flag, a_new_flag, a_first_rank, a_new_rank, a_set_first, a_set_slot, a_visible,
      a_counters;
  DevBuf<unsigned char> a_cub;
  // stage buffers for the single-call APIs
  DevBuf<double> s_depth, s_dch, s_pose, s_intr, s_vre, s_nre, s_vim, s_nim;
  DevBuf<double2> s_hits;
  DevBuf<double> s_terms;  // csf_view_scores per-pixel terms [views][C][P]
  // raycast alpha table (hashed volumes) for (tab_near, tab_far, tab_step)
  DevBuf<double> alpha_tab;
  DevBuf<unsigned> seg_first;  // segmented-march scratch
  double tab_near = 0.0, tab_far = -1.0, tab_step = 0.0;

  ~csf_volume_s() {
    rw.release(); fim.release(); heads.release(); next.release(); coords.release(); nblocks.release(); keys.release();
    grid.release();
    occ.release();
    sdist.release();
    a_cand.release(); a_set_keys.release(); a_cand_block.release(); a_first_flag.release(); a_new_flag.release();
    a_first_rank.release(); a_new_rank.release(); a_set_first.release(); a_set_slot.release(); a_visible.release();
    a_counters.release(); a_cub.release();
    s_depth.release(); s_dch.release(); s_pose.release(); s_intr.release(); s_vre.release(); s_nre.release(); s_vim.release();
    s_nim.release();
    s_hits.release();
    s_terms.release();
    alpha_tab.release();
    seg_first.release();
  }
};

namespace {

int ensure_alloc_scratch(csf_volume v, int w, int h) {
  csf_ctx ctx = v->ctx;
  const int K = band_samples(v->hash.mu, v->hash.vs);
  const size_t n = static_cast<size_t>(w) * h * K;
  if (v->alloc.max_cand >= static_cast<int>(n) && v->alloc.cand) return CSF_OK;
  if (n > 0x7fffffffULL) return fail(ctx, CSF_EINVAL, "frame too large for hashed allocation");
  CUDA_TRY(ctx, v->a_cand.alloc(n));
  CUDA_TRY(ctx, v->a_cand_block.alloc(n));
  CUDA_TRY(ctx, v->a_first_flag.alloc(n));
  CUDA_TRY(ctx, v->a_new_flag.alloc(n));
  CUDA_TRY(ctx, v->a_first_rank.alloc(n));
  CUDA_TRY(ctx, v->a_new_rank.alloc(n));
  CUDA_TRY(ctx, v->a_set_slot.alloc(n));
  const int set_bits = 20;
  CUDA_TRY(ctx, v->a_set_keys.alloc(size_t(1) << set_bits));
  CUDA_TRY(ctx, v->a_set_first.alloc(size_t(1) << set_bits));
  CUDA_TRY(ctx, v->a_visible.alloc(n));
  CUDA_TRY(ctx, v->a_counters.alloc(4));
  const size_t cub_bytes = alloc_scan_bytes(static_cast<int>(n));
  CUDA_TRY(ctx, v->a_cub.alloc(cub_bytes));
  CUDA_TRY(ctx, cudaMemsetAsync(v->a_counters.p, 0, sizeof(int) * 4, ctx->stream));
  AllocScratch& a = v->alloc;
  a.cand = v->a_cand.p;
  a.cand_block = v->a_cand_block.p;
  a.first_flag = v->a_first_flag.p;
  a.new_flag = v->a_new_flag.p;
  a.first_rank = v->a_first_rank.p;
  a.new_rank = v->a_new_rank.p;
  a.set_keys = v->a_set_keys.p;
  a.set_first = v->a_set_first.p;
  a.set_slot = v->a_set_slot.p;
  a.set_bits = set_bits;
  a.visible = v->a_visible.p;
  a.counters = v->a_counters.p;
  a.cub_tmp = v->a_cub.p;
  a.cub_tmp_bytes = cub_bytes;
  a.max_cand = static_cast<int>(n);
  return CSF_OK;
}

// order 1: n_channels first-order directions, grouped by pick_group.
// order 2: n_channels = 3 * pairs bicomplex slots, one pair per group.
int volume_init_common(csf_volume v, int n_channels, int order) {
  if (order == 2) {
    if (n_channels <= 0 || n_channels % 3 != 0 || n_channels > 3 * CSF_MAX_PAIRS)
      return fail(v->ctx, CSF_EINVAL, "second-order volumes carry 3 slots per pair, 1..CSF_MAX_PAIRS pairs");
    v->D = n_channels;
    v->G = 3;
    v->Dp = n_channels;
    v->order = 2;
    return CSF_OK;
  }
  if (n_channels < 0 || n_channels > CSF_MAX_DIRECTIONS)
    return fail(v->ctx, CSF_EINVAL, "channel count must be in [0, " + std::to_string(CSF_MAX_DIRECTIONS) + "]");
  v->D = n_channels;
  v->G = pick_group(n_channels);
  v->Dp = padded_channels(n_channels, v->G);
  v->order = 1;
  return CSF_OK;
}

// Fuse one double depth frame already on the device.  upd (nullable) counts
// the fused voxels.
int volume_fuse(csf_volume v, const double* d_depth, int w, int h, const double* d_pose, const double* d_intr,
                int* upd = nullptr, const double* d_dch = nullptr) {
  const Launch L = launch_of(v->ctx);
  if (v->hashed) {
    const int rc = ensure_alloc_scratch(v, w, h);
    if (rc) return rc;
    {
      PROF(v->ctx, kPAlloc);
      launch_allocate(L, v->hash, v->Dp, v->alloc, d_depth, w, h, d_pose, d_intr);
    }
    PROF(v->ctx, kPIntegrate);
    launch_integrate_hashed(L, v->hash, v->G, v->Dp, v->alloc, d_depth, w, h, d_pose, d_intr, upd, d_dch);
  } else {
    PROF(v->ctx, kPIntegrate);
    launch_integrate_dense(L, v->dense, v->G, v->Dp, d_depth, w, h, d_pose, d_intr, upd, d_dch);
  }
  return CSF_OK;
}

// The alpha sequence of a hashed raycast (a_0 = near, a_{n+1} = a_n + step,
// IEEE double addition as on the device), tabulated on the host once per
// (near, far, step) and kept on the device with the volume.
int ensure_alpha_table(csf_volume v, double near_clip, double far_clip, double step) {
  if (v->alpha_tab.p && v->tab_near == near_clip && v->tab_far == far_clip && v->tab_step == step) return CSF_OK;
  if (!(step > 0.0)) return fail(v->ctx, CSF_EINVAL, "raycast: step must be positive");
  std::vector<double> a;
  double alpha = near_clip;
  while (alpha <= far_clip) {
    a.push_back(alpha);
    alpha += step;
    if (a.size() > (1u << 24)) return fail(v->ctx, CSF_EINVAL, "raycast: too many steps");
  }
  a.push_back(alpha);  // sentinel > far
  CUDA_TRY(v->ctx, cudaStreamSynchronize(v->ctx->stream));
  CUDA_TRY(v->ctx, v->alpha_tab.alloc(a.size()));
  CUDA_TRY(v->ctx, cudaMemcpyAsync(v->alpha_tab.p, a.data(), sizeof(double) * a.size(), cudaMemcpyHostToDevice, v->ctx->stream));
  v->tab_near = near_clip;
  v->tab_far = far_clip;
  v->tab_step = step;
  v->hash.alpha_tab = v->alpha_tab.p;
  v->hash.alpha_n = static_cast<int>(a.size());
  return CSF_OK;
}

void raycast_dev(csf_volume v, const double* d_pose, const double* d_intr, int w, int h, const csf_raycast_cfg& rc,
                 double2* hits, double* vre, double* nre, double* vim, double* nim) {
  Launch L = launch_of(v->ctx);
  const double mu = v->hashed ? v->hash.mu : v->dense.mu;
  const double step = rc.step_fraction * mu;
  if (v->hashed && ensure_alpha_table(v, rc.near_clip, rc.far_clip, step) != CSF_OK) {
    v->hash.alpha_tab = nullptr;  // fall back to the in-kernel repeated addition
    v->hash.alpha_n = 0;
  }
  if (v->hashed) {
    if (v->seg_first.n < static_cast<size_t>(w) * h && v->seg_first.alloc(static_cast<size_t>(w) * h) != cudaSuccess)
      v->seg_first.release();
    v->hash.seg_first = v->seg_first.p;  // null: one thread per ray
  }
  for (int phase = 1; phase <= 2; ++phase) {
    PROF(v->ctx, phase == 1 ? kPRaycast : kPRaycastLift);
    L.phase = phase;
    if (v->hashed)
      launch_raycast_hashed(L, v->hash, v->G, v->Dp, d_pose, d_intr, w, h, rc.near_clip, rc.far_clip, step, hits, vre,
                            nre, vim, nim);
    else
      launch_raycast_dense(L, v->dense, v->G, v->Dp, d_pose, d_intr, w, h, rc.near_clip, rc.far_clip, step, hits,
                           vre, nre, vim, nim);
  }
}

// Host lifted array [n][1+D] -> padded [n][1+Dp]
std::vector<double> pad_channels(const double* src, int n, int D, int Dp) {
  std::vector<double> out(static_cast<size_t>(n) * (1 + Dp), 0.0);
  for (int e = 0; e < n; ++e)
    for (int c = 0; c <= std::min(D, Dp); ++c) out[static_cast<size_t>(e) * (1 + Dp) + c] = src[e * (1 + D) + c];
  return out;
}

}  // namespace

// ---------------------------------------------------------------------------
// defaults
// ---------------------------------------------------------------------------
extern "C" void csf_default_intrinsics(csf_intrinsics* k) {
  k->fx = 525.0; k->fy = 525.0; k->cx = 319.5; k->cy = 239.5;
  k->width = 640; k->height = 480; k->depth_scale = 5000.0;
}
extern "C" void csf_default_volume_params(csf_volume_params* p) {
  p->dims[0] = p->dims[1] = p->dims[2] = 128;
  p->voxel_size = 0.02;
  p->origin[0] = p->origin[1] = p->origin[2] = 0.0;
  p->mu = 0.1;
  p->weight_cap = 128.0;
}
extern "C" void csf_default_raycast_cfg(csf_raycast_cfg* c) {
  c->near_clip = 0.0; c->far_clip = 10.0; c->step_fraction = 0.5;
}
extern "C" void csf_default_icp_cfg(csf_icp_cfg* c) {
  c->solver = CSF_SOLVER_NEWTON;  // icp.hpp:41 (the lifted pipeline selects the linearized solver)
  c->d_max = 0.1;
  c->theta_max_deg = 30.0;
  c->levels = 3;
  c->level_iterations[0] = 10; c->level_iterations[1] = 5; c->level_iterations[2] = 4;
  c->level_pixel_stride[0] = 1; c->level_pixel_stride[1] = 1; c->level_pixel_stride[2] = 2;
  c->step_tolerance = 1e-6;
  c->levenberg_lambda0 = 1e-6;
  c->ncg_restart = 6;
  c->h = 1e-8;
}

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
extern "C" int csf_ctx_create(int device, csf_ctx* out) {
  if (!out) return CSF_EINVAL;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return CSF_ECUDA;
  if (device < 0 || device >= n) return CSF_EINVAL;
  csf_ctx ctx = new csf_ctx_s();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&ctx->d_err, sizeof(int)) != cudaSuccess ||
      cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream) != cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    delete ctx;
    return CSF_ECUDA;
  }
  *out = ctx;
  return CSF_OK;
}

// ---------------------------------------------------------------------------
// NCCL, opened at runtime: no link-time dependency, and in a process that
// already mapped a libnccl.so.2 (torch's) that same library is used.
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};
const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.broadcast = reinterpret_cast<decltype(api.broadcast)>(sym("ncclBroadcast"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.broadcast && api.group_start &&
             api.group_end && api.error_string;
    if (!api.ok) api.err = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}
}  // namespace

extern "C" int csf_comm_unique_id(unsigned char* id) {
  if (!id) return CSF_EINVAL;
  const NcclApi& n = nccl();
  if (!n.ok) return CSF_ERUNTIME;
  ncclUniqueId u;
  if (n.get_unique_id(&u) != ncclSuccess) return CSF_ERUNTIME;
  std::memcpy(id, &u, sizeof(u));
  return CSF_OK;
}

extern "C" int csf_ctx_attach_comm(csf_ctx ctx, int n_ranks, int rank, const unsigned char* id) {
  if (!ctx || !id || n_ranks <= 0 || rank < 0 || rank >= n_ranks) return CSF_EINVAL;
  const NcclApi& n = nccl();
  if (!n.ok) return fail(ctx, CSF_ERUNTIME, "csf_ctx_attach_comm: " + n.err);
  cudaSetDevice(ctx->device);
  if (ctx->comm) {
    n.comm_destroy(ctx->comm);
    ctx->comm = nullptr;
  }
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  const ncclResult_t r = n.comm_init_rank(&ctx->comm, n_ranks, u, rank);
  if (r != ncclSuccess) {
    ctx->comm = nullptr;
    return fail(ctx, CSF_ERUNTIME, std::string("csf_ctx_attach_comm: ") + n.error_string(r));
  }
  ctx->n_ranks = n_ranks;
  ctx->rank = rank;
  return CSF_OK;
}

extern "C" int csf_gather_columns(csf_ctx ctx, const double* local, const int* counts, double* out) {
  if (!ctx || !counts || !out) return CSF_EINVAL;
  if (!ctx->comm) return fail(ctx, CSF_EINVAL, "csf_gather_columns: no communicator (csf_ctx_attach_comm)");
  const NcclApi& n = nccl();
  cudaSetDevice(ctx->device);
  std::vector<size_t> off(ctx->n_ranks + 1, 0);
  for (int r = 0; r < ctx->n_ranks; ++r) {
    if (counts[r] < 0) return CSF_EINVAL;
    off[r + 1] = off[r] + static_cast<size_t>(counts[r]);
  }
  const size_t total = off[ctx->n_ranks];
  if (counts[ctx->rank] > 0 && !local) return CSF_EINVAL;
  if (total > ctx->gather_cap) {
    if (ctx->gather_buf) cudaFree(ctx->gather_buf);
    ctx->gather_buf = nullptr;
    ctx->gather_cap = 0;
    CUDA_TRY(ctx, cudaMalloc(&ctx->gather_buf, sizeof(double) * std::max<size_t>(total, 1)));
    ctx->gather_cap = total;
  }
  double* buf = ctx->gather_buf;
  if (counts[ctx->rank] > 0)
    CUDA_TRY(ctx, cudaMemcpyAsync(buf + off[ctx->rank], local, sizeof(double) * counts[ctx->rank],
                                  cudaMemcpyHostToDevice, ctx->stream));
  // every rank's block broadcast from its owner, in place (one NCCL group)
  n.group_start();
  for (int r = 0; r < ctx->n_ranks; ++r)
    if (counts[r] > 0) {
      const ncclResult_t e = n.broadcast(buf + off[r], buf + off[r], counts[r], ncclDouble, r, ctx->comm, ctx->stream);
      if (e != ncclSuccess) {
        n.group_end();
        return fail(ctx, CSF_ERUNTIME, std::string("csf_gather_columns: ") + n.error_string(e));
      }
    }
  const ncclResult_t ge = n.group_end();
  if (ge != ncclSuccess) return fail(ctx, CSF_ERUNTIME, std::string("csf_gather_columns: ") + n.error_string(ge));
  if (total > 0) CUDA_TRY(ctx, d2h(out, buf, sizeof(double) * total, ctx->stream));
  return CSF_OK;
}

extern "C" int csf_ctx_destroy(csf_ctx ctx) {
  if (!ctx) return CSF_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->comm) nccl().comm_destroy(ctx->comm);
  if (ctx->gather_buf) cudaFree(ctx->gather_buf);
  if (ctx->d_err) cudaFree(ctx->d_err);
  energy_scratch_release(ctx->energy);
  if (ctx->corr_upload) cudaFree(ctx->corr_upload);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return CSF_OK;
}

extern "C" const char* csf_last_error(csf_ctx ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

extern "C" int csf_ctx_synchronize(csf_ctx ctx) {
  if (!ctx) return CSF_EINVAL;
  cudaSetDevice(ctx->device);
  return sync_check(ctx, "synchronize");
}

extern "C" int csf_ctx_launch_count(csf_ctx ctx, unsigned long long* out) {
  if (!ctx || !out) return CSF_EINVAL;
  *out = ctx->launches;
  return CSF_OK;
}

extern "C" void* csf_ctx_stream(csf_ctx ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

extern "C" int csf_ctx_profile(csf_ctx ctx, int enable) {
  if (!ctx) return CSF_EINVAL;
  ctx->prof.on = enable != 0;
  ctx->prof.used = 0;
  ctx->prof.recs.clear();
  return CSF_OK;
}

extern "C" int csf_ctx_profile_read(csf_ctx ctx, int max_categories, char* names, double* ms, long long* counts,
                                    int* n_categories) {
  if (!ctx || !n_categories) return CSF_EINVAL;
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  double tot[kPN] = {0};
  long long cnt[kPN] = {0};
  for (const auto& r : ctx->prof.recs) {
    float t = 0.0f;
    cudaEventElapsedTime(&t, ctx->prof.pool[r.second], ctx->prof.pool[r.second + 1]);
    tot[r.first] += t;
    cnt[r.first] += 1;
  }
  const int n = std::min<int>(kPN, max_categories);
  for (int i = 0; i < n; ++i) {
    if (names) std::snprintf(names + 32 * i, 32, "%s", kProfNames[i]);
    if (ms) ms[i] = tot[i];
    if (counts) counts[i] = cnt[i];
  }
  *n_categories = n;
  ctx->prof.used = 0;
  ctx->prof.recs.clear();
  return CSF_OK;
}

// ---------------------------------------------------------------------------
// frames
// ---------------------------------------------------------------------------
extern "C" int csf_bilateral_filter(csf_ctx ctx, const double* depth, int w, int h, double sigma_s, double sigma_r,
                                    int radius, double* out) {
  if (!ctx || !depth || !out || w <= 0 || h <= 0 || radius < 0 || radius > 7)
    return fail(ctx, CSF_EINVAL, "csf_bilateral_filter: bad arguments (radius must be 0..7)");
  cudaSetDevice(ctx->device);
  const size_t P = static_cast<size_t>(w) * h;
  DevBuf<double> din, dout;
  CUDA_TRY(ctx, din.alloc(P));
  CUDA_TRY(ctx, dout.alloc(P));
  CUDA_TRY(ctx, cudaMemcpyAsync(din.p, depth, sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream));
  launch_bilateral(launch_of(ctx), nullptr, din.p, nullptr, dout.p, w, h, sigma_s, sigma_r, radius);
  CUDA_TRY(ctx, d2h(out, dout.p, sizeof(double) * P, ctx->stream));
  const int rc = sync_check(ctx, "csf_bilateral_filter");
  din.release();
  dout.release();
  return rc;
}

extern "C" int csf_downsample_depth(csf_ctx ctx, const double* depth, int w, int h, double sigma_r, double* out) {
  if (!ctx || !depth || !out || w <= 1 || h <= 1) return fail(ctx, CSF_EINVAL, "csf_downsample_depth: bad arguments");
  cudaSetDevice(ctx->device);
  const size_t P = static_cast<size_t>(w) * h, Po = static_cast<size_t>(w / 2) * (h / 2);
  DevBuf<double> din, dout;
  CUDA_TRY(ctx, din.alloc(P));
  CUDA_TRY(ctx, dout.alloc(Po));
  CUDA_TRY(ctx, cudaMemcpyAsync(din.p, depth, sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream));
  launch_downsample(launch_of(ctx), din.p, dout.p, w, h, sigma_r);
  CUDA_TRY(ctx, d2h(out, dout.p, sizeof(double) * Po, ctx->stream));
  const int rc = sync_check(ctx, "csf_downsample_depth");
  din.release();
  dout.release();
  return rc;
}

extern "C" int csf_measure_surface(csf_ctx ctx, const double* depth, int w, int h, const double* intr, int n_channels,
                                   double* vertices, double* normals) {
  if (!ctx || !depth || !intr || !vertices || !normals || w <= 0 || h <= 0 || n_channels < 0 ||
      n_channels > CSF_MAX_DIRECTIONS)
    return fail(ctx, CSF_EINVAL, "csf_measure_surface: bad arguments");
  if (n_channels > 0 && (intr[0] == 0.0 || intr[1 + n_channels] == 0.0))
    return fail(ctx, CSF_EDOMAIN, "csf_measure_surface: Complex division by zero real part (fx or fy = 0)");
  cudaSetDevice(ctx->device);
  const size_t P = static_cast<size_t>(w) * h, C = 1 + n_channels;
  DevBuf<double> dd, dk, dv, dn;
  CUDA_TRY(ctx, dd.alloc(P * C));
  CUDA_TRY(ctx, dk.alloc(4 * C));
  CUDA_TRY(ctx, dv.alloc(P * 3 * C));
  CUDA_TRY(ctx, dn.alloc(P * 3 * C));
  CUDA_TRY(ctx, cudaMemcpyAsync(dd.p, depth, sizeof(double) * P * C, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(dk.p, intr, sizeof(double) * 4 * C, cudaMemcpyHostToDevice, ctx->stream));
  launch_measure(launch_of(ctx), dd.p, w, h, dk.p, n_channels, dv.p, dn.p);
  CUDA_TRY(ctx, d2h(vertices, dv.p, sizeof(double) * P * 3 * C, ctx->stream));
  CUDA_TRY(ctx, d2h(normals, dn.p, sizeof(double) * P * 3 * C, ctx->stream));
  const int rc = sync_check(ctx, "csf_measure_surface");
  dd.release(); dk.release(); dv.release(); dn.release();
  return rc;
}

// ---------------------------------------------------------------------------
// volumes
// ---------------------------------------------------------------------------
static int create_dense(csf_ctx ctx, const csf_volume_params* p, int n_channels, int order, csf_volume* out) {
  if (!ctx || !p || !out) return CSF_EINVAL;
  *out = nullptr;
  if (p->dims[0] <= 0 || p->dims[1] <= 0 || p->dims[2] <= 0 || !(p->voxel_size > 0.0))
    return fail(ctx, CSF_EINVAL, "csf_volume_create_dense: dims and voxel_size must be positive");
  cudaSetDevice(ctx->device);
  csf_volume v = new csf_volume_s();
  v->ctx = ctx;
  int rc = volume_init_common(v, n_channels, order);
  if (rc) {
    delete v;
    return rc;
  }
  v->n_vox = static_cast<long long>(p->dims[0]) * p->dims[1] * p->dims[2];
  if (v->rw.alloc(v->n_vox) != cudaSuccess || v->fim.alloc(static_cast<size_t>(v->n_vox) * std::max(v->Dp, 1)) != cudaSuccess) {
    delete v;
    return fail(ctx, CSF_ENOMEM, "csf_volume_create_dense: out of device memory");
  }
  DenseDev& d = v->dense;
  d.rw = v->rw.p;
  d.fim = v->fim.p;
  d.nx = p->dims[0]; d.ny = p->dims[1]; d.nz = p->dims[2];
  d.vs = p->voxel_size;
  d.ox = p->origin[0]; d.oy = p->origin[1]; d.oz = p->origin[2];
  d.mu = p->mu;
  d.cap = p->weight_cap;
  d.order = v->order;
  launch_init_volume(launch_of(ctx), d.rw, d.fim, v->n_vox, v->Dp);
  rc = sync_check(ctx, "csf_volume_create_dense");
  if (rc) {
    delete v;
    return rc;
  }
  *out = v;
  return CSF_OK;
}

static int create_hashed(csf_ctx ctx, const csf_hash_params* p, int n_channels, int order, csf_volume* out) {
  if (!ctx || !p || !out) return CSF_EINVAL;
  *out = nullptr;
  if (!(p->voxel_size > 0.0) || p->bucket_bits < 4 || p->bucket_bits > 28 || p->max_blocks <= 0)
    return fail(ctx, CSF_EINVAL, "csf_volume_create_hashed: bad parameters");
  cudaSetDevice(ctx->device);
  csf_volume v = new csf_volume_s();
  v->ctx = ctx;
  v->hashed = true;
  int rc = volume_init_common(v, n_channels, order);
  if (rc) {
    delete v;
    return rc;
  }
  v->n_vox = static_cast<long long>(p->max_blocks) * 512;
  const size_t nb = size_t(1) << p->bucket_bits;
  const int gbits = 9;  // 512^3 block-id window (512 MiB of int32)
  const size_t ng = size_t(1) << (3 * gbits);
  const size_t nocc = occ_words(gbits);
  const size_t nsb = size_t(1) << (3 * (gbits - 3));
  if (v->grid.alloc(ng) != cudaSuccess || v->occ.alloc(nocc) != cudaSuccess || v->sdist.alloc(2 * nsb) != cudaSuccess) {
    delete v;
    return fail(ctx, CSF_ENOMEM, "csf_volume_create_hashed: out of device memory (block grid)");
  }
  if (v->rw.alloc(v->n_vox) != cudaSuccess ||
      v->fim.alloc(static_cast<size_t>(v->n_vox) * std::max(v->Dp, 1)) != cudaSuccess ||
      v->heads.alloc(nb) != cudaSuccess || v->next.alloc(p->max_blocks) != cudaSuccess ||
      v->coords.alloc(3 * static_cast<size_t>(p->max_blocks)) != cudaSuccess ||
      v->keys.alloc(p->max_blocks) != cudaSuccess || v->nblocks.alloc(1) != cudaSuccess) {
    delete v;
    return fail(ctx, CSF_ENOMEM, "csf_volume_create_hashed: out of device memory");
  }
  HashDev& d = v->hash;
  d.rw = v->rw.p;
  d.fim = v->fim.p;
  d.heads = v->heads.p;
  d.keys = v->keys.p;
  d.next = v->next.p;
  d.coords = v->coords.p;
  d.n_blocks = v->nblocks.p;
  d.grid = v->grid.p;
  d.occ = v->occ.p;
  d.sdist = v->sdist.p;
  d.sdist_tmp = v->sdist.p + nsb;
  d.gbits = gbits;
  d.bits = p->bucket_bits;
  d.max_blocks = p->max_blocks;
  d.vs = p->voxel_size;
  d.ox = p->origin[0]; d.oy = p->origin[1]; d.oz = p->origin[2];
  d.mu = p->mu;
  d.cap = p->weight_cap;
  d.order = v->order;
  cudaMemsetAsync(d.heads, 0xFF, sizeof(int) * nb, ctx->stream);
  cudaMemsetAsync(d.next, 0xFF, sizeof(int) * p->max_blocks, ctx->stream);
  cudaMemsetAsync(d.n_blocks, 0, sizeof(int), ctx->stream);
  cudaMemsetAsync(d.grid, 0xFF, sizeof(int) * ng, ctx->stream);
  cudaMemsetAsync(d.occ, 0, sizeof(unsigned) * nocc, ctx->stream);
  launch_super_dist(ctx->stream, d);
  launch_init_volume(launch_of(ctx), d.rw, d.fim, v->n_vox, v->Dp);
  rc = sync_check(ctx, "csf_volume_create_hashed");
  if (rc) {
    delete v;
    return rc;
  }
  *out = v;
  return CSF_OK;
}

extern "C" int csf_volume_create_dense(csf_ctx ctx, const csf_volume_params* p, int n_channels, csf_volume* out) {
  return create_dense(ctx, p, n_channels, 1, out);
}
extern "C" int csf_volume_create_hashed(csf_ctx ctx, const csf_hash_params* p, int n_channels, csf_volume* out) {
  return create_hashed(ctx, p, n_channels, 1, out);
}

extern "C" int csf_volume_destroy(csf_volume vol) {
  if (!vol) return CSF_OK;
  cudaSetDevice(vol->ctx->device);
  cudaStreamSynchronize(vol->ctx->stream);
  delete vol;
  return CSF_OK;
}

extern "C" int csf_volume_block_count(csf_volume v, int* n);
extern "C" int csf_volume_info(csf_volume v, int* n_channels, int* hashed, long long* n_voxels) {
  if (!v) return CSF_EINVAL;
  if (n_channels) *n_channels = v->D;
  if (hashed) *hashed = v->hashed ? 1 : 0;
  if (n_voxels) {
    if (v->hashed) {
      int nb = 0;
      const int rc = csf_volume_block_count(v, &nb);
      if (rc) return rc;
      *n_voxels = static_cast<long long>(nb) * 512;
    } else {
      *n_voxels = v->n_vox;
    }
  }
  return CSF_OK;
}

extern "C" int csf_volume_block_count(csf_volume v, int* n) {
  if (!v || !n) return CSF_EINVAL;
  if (!v->hashed) {
    *n = 0;
    return CSF_OK;
  }
  cudaSetDevice(v->ctx->device);
  CUDA_TRY(v->ctx, cudaStreamSynchronize(v->ctx->stream));
  CUDA_TRY(v->ctx, d2h(n, v->hash.n_blocks, sizeof(int), v->ctx->stream));
  return CSF_OK;
}

static long long volume_voxels_now(csf_volume v) {
  if (!v->hashed) return v->n_vox;
  int nb = 0;
  csf_volume_block_count(v, &nb);
  return static_cast<long long>(nb) * 512;
}

extern "C" int csf_volume_upload(csf_volume v, const double* field, const double* weight) {
  if (!v || !field || !weight) return CSF_EINVAL;
  csf_ctx ctx = v->ctx;
  cudaSetDevice(ctx->device);
  const long long n = volume_voxels_now(v);
  std::vector<double2> rw(n);
  std::vector<double> fim(static_cast<size_t>(n) * std::max(v->Dp, 1), 0.0);
  const int C = 1 + v->D;
  for (long long i = 0; i < n; ++i) {
    rw[i] = make_double2(field[i * C], weight[i]);
    for (int d = 0; d < v->D; ++d) fim[i * v->Dp + d] = field[i * C + 1 + d];
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(v->rw.p, rw.data(), sizeof(double2) * n, cudaMemcpyHostToDevice, ctx->stream));
  if (v->Dp > 0) CUDA_TRY(ctx, cudaMemcpyAsync(v->fim.p, fim.data(), sizeof(double) * n * v->Dp, cudaMemcpyHostToDevice, ctx->stream));
  return CSF_OK;
}

extern "C" int csf_volume_download(csf_volume v, double* field, double* weight) {
  if (!v || !field || !weight) return CSF_EINVAL;
  csf_ctx ctx = v->ctx;
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  const long long n = volume_voxels_now(v);
  std::vector<double2> rw(n);
  std::vector<double> fim(static_cast<size_t>(n) * std::max(v->Dp, 1));
  CUDA_TRY(ctx, d2h(rw.data(), v->rw.p, sizeof(double2) * n, ctx->stream));
  if (v->Dp > 0) CUDA_TRY(ctx, d2h(fim.data(), v->fim.p, sizeof(double) * n * v->Dp, ctx->stream));
  const int C = 1 + v->D;
  for (long long i = 0; i < n; ++i) {
    field[i * C] = rw[i].x;
    weight[i] = rw[i].y;
    for (int d = 0; d < v->D; ++d) field[i * C + 1 + d] = fim[i * v->Dp + d];
  }
  return CSF_OK;
}

extern "C" int csf_volume_download_hash(csf_volume v, int32_t* heads, uint64_t* keys, int32_t* next, int32_t* coords) {
  if (!v || !v->hashed) return v ? fail(v->ctx, CSF_EINVAL, "csf_volume_download_hash: not a hashed volume") : CSF_EINVAL;
  csf_ctx ctx = v->ctx;
  int nb = 0;
  const int rc = csf_volume_block_count(v, &nb);
  if (rc) return rc;
  if (heads) CUDA_TRY(ctx, d2h(heads, v->hash.heads, sizeof(int) << v->hash.bits, ctx->stream));
  if (keys) CUDA_TRY(ctx, d2h(keys, v->hash.keys, sizeof(uint64_t) * nb, ctx->stream));
  if (next) CUDA_TRY(ctx, d2h(next, v->hash.next, sizeof(int) * nb, ctx->stream));
  if (coords) CUDA_TRY(ctx, d2h(coords, v->hash.coords, sizeof(int) * 3 * nb, ctx->stream));
  return CSF_OK;
}

// lifted: depth is [h][w][1+D] (the reference's Image<Complex> depth,
// tsdf.hpp:144-145), else [h][w] real.
static int surface_update_impl(csf_volume v, const double* depth, bool lifted, int w, int h, const double* pose,
                               const double* intr, int* n_visible) {
  if (!v || !depth || !pose || !intr || w <= 1 || h <= 1) return CSF_EINVAL;
  csf_ctx ctx = v->ctx;
  if (v->D > 0 && (intr[0] == 0.0 || intr[1 + v->D] == 0.0))
    return fail(ctx, CSF_EDOMAIN, "csf_surface_update: Complex division by zero real part (fx or fy = 0)");
  if (lifted && v->order != 1)
    return fail(ctx, CSF_EINVAL, "csf_surface_update_lifted: lifted depth takes first-order volumes");
  cudaSetDevice(ctx->device);
  const size_t P = static_cast<size_t>(w) * h;
  const int C = 1 + v->Dp;
  const std::vector<double> pp = pad_channels(pose, 12, v->D, v->Dp);
  const std::vector<double> kp = pad_channels(intr, 4, v->D, v->Dp);
  CUDA_TRY(ctx, v->s_depth.alloc(P));
  CUDA_TRY(ctx, v->s_pose.alloc(12 * C));
  CUDA_TRY(ctx, v->s_intr.alloc(4 * C));
  const bool channels = lifted && v->Dp > 0;
  if (!lifted) {
    CUDA_TRY(ctx, cudaMemcpyAsync(v->s_depth.p, depth, sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream));
  } else {
    // split [P][1+D] into the real image and the channels [P][Dp] (padding zero)
    std::vector<double> re(P), ch(channels ? P * v->Dp : 0, 0.0);
    for (size_t i = 0; i < P; ++i) {
      re[i] = depth[i * (1 + v->D)];
      for (int d = 0; d < v->D && channels; ++d) ch[i * v->Dp + d] = depth[i * (1 + v->D) + 1 + d];
    }
    CUDA_TRY(ctx, cudaMemcpyAsync(v->s_depth.p, re.data(), sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream));
    if (channels) {
      CUDA_TRY(ctx, v->s_dch.alloc(P * v->Dp));
      CUDA_TRY(ctx, cudaMemcpyAsync(v->s_dch.p, ch.data(), sizeof(double) * P * v->Dp, cudaMemcpyHostToDevice,
                                    ctx->stream));
    }
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));  // re / ch are local
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(v->s_pose.p, pp.data(), sizeof(double) * 12 * C, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(v->s_intr.p, kp.data(), sizeof(double) * 4 * C, cudaMemcpyHostToDevice, ctx->stream));
  int rc = volume_fuse(v, v->s_depth.p, w, h, v->s_pose.p, v->s_intr.p, nullptr, channels ? v->s_dch.p : nullptr);
  if (rc) return rc;
  rc = sync_check(ctx, "csf_surface_update");
  if (rc) return rc;
  if (n_visible) {
    *n_visible = 0;
    if (v->hashed) CUDA_TRY(ctx, d2h(n_visible, v->alloc.counters, sizeof(int), ctx->stream));
  }
  return CSF_OK;
}

extern "C" int csf_surface_update(csf_volume v, const double* depth, int w, int h, const double* pose,
                                  const double* intr, int* n_visible) {
  return surface_update_impl(v, depth, false, w, h, pose, intr, n_visible);
}

extern "C" int csf_surface_update_lifted(csf_volume v, const double* depth, int w, int h, const double* pose,
                                         const double* intr, int* n_visible) {
  return surface_update_impl(v, depth, true, w, h, pose, intr, n_visible);
}

extern "C" int csf_raycast(csf_volume v, const double* pose, const double* intr, int w, int h,
                           const csf_raycast_cfg* cfg, double* vertices, double* normals) {
  if (!v || !pose || !intr || !vertices || !normals || w <= 0 || h <= 0) return CSF_EINVAL;
  csf_ctx ctx = v->ctx;
  if (v->D > 0 && (intr[0] == 0.0 || intr[1 + v->D] == 0.0))
    return fail(ctx, CSF_EDOMAIN, "csf_raycast: Complex division by zero real part (fx or fy = 0)");
  cudaSetDevice(ctx->device);
  csf_raycast_cfg rc;
  if (cfg)
    rc = *cfg;
  else
    csf_default_raycast_cfg(&rc);
  const size_t P = static_cast<size_t>(w) * h;
  const int C = 1 + v->Dp;
  const std::vector<double> pp = pad_channels(pose, 12, v->D, v->Dp);
  const std::vector<double> kp = pad_channels(intr, 4, v->D, v->Dp);
  CUDA_TRY(ctx, v->s_pose.alloc(12 * C));
  CUDA_TRY(ctx, v->s_intr.alloc(4 * C));
  CUDA_TRY(ctx, v->s_vre.alloc(P * 3));
  CUDA_TRY(ctx, v->s_nre.alloc(P * 3));
  CUDA_TRY(ctx, v->s_vim.alloc(P * 3 * std::max(v->Dp, 1)));
  CUDA_TRY(ctx, v->s_nim.alloc(P * 3 * std::max(v->Dp, 1)));
  CUDA_TRY(ctx, v->s_hits.alloc(2 * P));  // (alpha_prev, alpha), then (f_prev, f)
  CUDA_TRY(ctx, cudaMemcpyAsync(v->s_pose.p, pp.data(), sizeof(double) * 12 * C, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(v->s_intr.p, kp.data(), sizeof(double) * 4 * C, cudaMemcpyHostToDevice, ctx->stream));
  raycast_dev(v, v->s_pose.p, v->s_intr.p, w, h, rc, v->s_hits.p, v->s_vre.p, v->s_nre.p, v->s_vim.p, v->s_nim.p);
  std::vector<double> vre(P * 3), nre(P * 3), vim(P * 3 * std::max(v->Dp, 1)), nim(P * 3 * std::max(v->Dp, 1));
  CUDA_TRY(ctx, d2h(vre.data(), v->s_vre.p, sizeof(double) * P * 3, ctx->stream));
  CUDA_TRY(ctx, d2h(nre.data(), v->s_nre.p, sizeof(double) * P * 3, ctx->stream));
  if (v->Dp > 0) {
    CUDA_TRY(ctx, d2h(vim.data(), v->s_vim.p, sizeof(double) * P * 3 * v->Dp, ctx->stream));
    CUDA_TRY(ctx, d2h(nim.data(), v->s_nim.p, sizeof(double) * P * 3 * v->Dp, ctx->stream));
  }
  const int r = sync_check(ctx, "csf_raycast");
  if (r) return r;
  const int Cu = 1 + v->D;
  for (size_t e = 0; e < P * 3; ++e) {
    vertices[e * Cu] = vre[e];
    normals[e * Cu] = nre[e];
    for (int d = 0; d < v->D; ++d) {
      vertices[e * Cu + 1 + d] = vim[e * v->Dp + d];
      normals[e * Cu + 1 + d] = nim[e * v->Dp + d];
    }
  }
  return CSF_OK;
}

// ---------------------------------------------------------------------------
// pipeline
// ---------------------------------------------------------------------------
struct csf_pipeline_s {
  csf_ctx ctx = nullptr;
  csf_pipeline_cfg cfg{};
  csf_volume vol = nullptr;
  int D = 0, G = 0, Dp = 0, C = 1;
  int order = 1, n_pairs = 0;
  int W = 0, H = 0, levels = 3;
  int n_uploaded = 0, n_run = 0;
  DevBuf<float> frames;
  DevBuf<unsigned char> rgb;  // run_host_rgbd: colour frames [max_frames][H][W][3], ingested, unused
  DevBuf<double> gt, raw, pyr0, pyr1, pyr2, vre, nre, vim, nim, partials, pose, pred_pose, intr_levels, traj, kbase,
      out, stage;
  DevBuf<int> counts, stats, dirs, pair_i, pair_j;
  DevBuf<TrackState> st;
  DevBuf<double2> hits;
  // run_host: frames uploaded on a copy stream, frame f's kernels wait on ev[f]
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> frame_ev;
  bool wait_frames = false;
  // CUDA graph of a whole run (csf_pipeline_set_graph): captured on the
  // first graph-mode run after a stream run of the same frame count.  Two
  // graphs: [0] device-resident frames (csf_pipeline_run), [1] run_host's
  // per-frame upload waits (captured as external event-wait nodes).
  bool use_graph = false;
  bool capturing = false;
  cudaGraphExec_t graph_exec[2] = {nullptr, nullptr};
  int exec_frames[2] = {0, 0};   // frame count of graph_exec
  int graph_frames[2] = {0, 0};  // frame count of the last stream run
  unsigned long long graph_launches[2] = {0, 0};
  int stream_runs[2] = {0, 0};
  ~csf_pipeline_s() {
    for (cudaGraphExec_t g : graph_exec)
      if (g) cudaGraphExecDestroy(g);
    for (cudaEvent_t e : frame_ev) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    hits.release();
    rgb.release();
    frames.release(); gt.release(); raw.release(); pyr0.release(); pyr1.release(); pyr2.release(); vre.release();
    nre.release(); vim.release(); nim.release(); partials.release(); pose.release(); pred_pose.release();
    intr_levels.release(); traj.release(); kbase.release(); out.release(); counts.release(); stats.release();
    dirs.release(); st.release(); stage.release(); pair_i.release(); pair_j.release();
    if (vol) csf_volume_destroy(vol);
  }
};

extern "C" int csf_pipeline_create(csf_ctx ctx, const csf_pipeline_cfg* cfg, csf_pipeline* out) {
  if (!ctx || !cfg || !out) return CSF_EINVAL;
  *out = nullptr;
  const int order = cfg->order == 0 ? 1 : cfg->order;
  if (order != 1 && order != 2) return fail(ctx, CSF_EINVAL, "csf_pipeline_create: order must be 1 or 2");
  if (cfg->n_dirs < 0 || cfg->n_dirs > CSF_MAX_DIRECTIONS)
    return fail(ctx, CSF_EINVAL, "csf_pipeline_create: n_dirs out of range");
  if (!(cfg->h > 0.0) || cfg->h > 1e-6)
    return fail(ctx, CSF_EINVAL, "StepSize: step must satisfy 0 < h <= 1e-6");
  if (cfg->keyframe_interval < 0) return fail(ctx, CSF_EINVAL, "csf_pipeline_create: negative keyframe_interval");
  for (int d = 0; d < cfg->n_dirs; ++d) {
    const int code = cfg->dirs[d];
    const bool keyframe = cfg->keyframe_interval > 0 && code >= 10 &&
                          1 + (code - 10) / 6 < (cfg->max_frames + cfg->keyframe_interval - 1) / cfg->keyframe_interval;
    if (code < 0 || (code > 9 && !keyframe))
      return fail(ctx, CSF_EINVAL, "csf_pipeline_create: unknown direction");
  }
  if (order == 2) {
    if (cfg->n_pairs <= 0 || cfg->n_pairs > CSF_MAX_PAIRS || cfg->n_dirs != 0)
      return fail(ctx, CSF_EINVAL, "csf_pipeline_create: order 2 needs 1..CSF_MAX_PAIRS pairs and no dirs");
    for (int q = 0; q < cfg->n_pairs; ++q)
      if (cfg->pair_i[q] < 0 || cfg->pair_i[q] > 9 || cfg->pair_j[q] < 0 || cfg->pair_j[q] > 9)
        return fail(ctx, CSF_EINVAL, "csf_pipeline_create: unknown pair parameter");
  }
  if (cfg->icp.solver != CSF_SOLVER_LINEARIZED)
    return fail(ctx, CSF_EINVAL, "csf_pipeline_create: the lifted tracker implements the linearized solver");
  if (cfg->icp.levels < 1 || cfg->icp.levels > 3 || cfg->max_frames <= 0 || cfg->k.width <= 0 || cfg->k.height <= 0)
    return fail(ctx, CSF_EINVAL, "csf_pipeline_create: bad levels/frames/size");
  if (!icp_frame_fits(cfg->k.width, cfg->k.height, 1))
    return fail(ctx, CSF_EINVAL, "csf_pipeline_create: frame too large for the ICP reduction");
  cudaSetDevice(ctx->device);
  csf_pipeline p = new csf_pipeline_s();
  p->ctx = ctx;
  p->cfg = *cfg;
  const int slots = order == 2 ? 3 * cfg->n_pairs : cfg->n_dirs;
  int rc = cfg->hashed ? create_hashed(ctx, &cfg->hash, slots, order, &p->vol)
                       : create_dense(ctx, &cfg->dense, slots, order, &p->vol);
  if (rc) {
    delete p;
    return rc;
  }
  p->order = order;
  p->n_pairs = order == 2 ? cfg->n_pairs : 0;
  p->D = slots;
  p->G = p->vol->G;
  p->Dp = p->vol->Dp;
  p->C = 1 + p->Dp;
  p->W = cfg->k.width;
  p->H = cfg->k.height;
  p->levels = cfg->icp.levels;
  const size_t P = static_cast<size_t>(p->W) * p->H;
  const int C = p->C;
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) {
    if (r != cudaSuccess && e == cudaSuccess) e = r;
  };
  A(p->frames.alloc(P * cfg->max_frames));
  A(p->gt.alloc(12 * static_cast<size_t>(cfg->max_frames)));
  A(p->raw.alloc(P));
  A(p->pyr0.alloc(P));
  A(p->pyr1.alloc(P / 4 + 1));
  A(p->pyr2.alloc(P / 16 + 1));
  A(p->vre.alloc(P * 3));
  A(p->nre.alloc(P * 3));
  A(p->vim.alloc(P * 3 * std::max(p->Dp, 1)));
  A(p->nim.alloc(P * 3 * std::max(p->Dp, 1)));
  A(p->partials.alloc(icp_partials_doubles(C)));
  A(p->counts.alloc(icp_counts_ints()));
  A(p->pose.alloc(12 * C));
  A(p->pred_pose.alloc(12 * C));
  A(p->intr_levels.alloc(3 * 4 * C));
  A(p->traj.alloc(static_cast<size_t>(cfg->max_frames) * 12 * C));
  A(p->stats.alloc(8 * static_cast<size_t>(cfg->max_frames)));
  A(p->dirs.alloc(CSF_MAX_DIRECTIONS));
  A(p->kbase.alloc(4));
  A(p->out.alloc(2 + std::max(CSF_MAX_DIRECTIONS, 3 * CSF_MAX_PAIRS)));
  A(p->stage.alloc(16));
  A(p->pair_i.alloc(CSF_MAX_PAIRS));
  A(p->pair_j.alloc(CSF_MAX_PAIRS));
  A(p->st.alloc(1));
  A(p->hits.alloc(2 * P));
  if (e != cudaSuccess) {
    delete p;
    return fail(ctx, CSF_ENOMEM, std::string("csf_pipeline_create: ") + cudaGetErrorString(e));
  }
  if (cfg->hashed) {
    rc = ensure_alloc_scratch(p->vol, p->W, p->H);
    if (rc) {
      delete p;
      return rc;
    }
  }
  const double kb[4] = {cfg->k.fx, cfg->k.fy, cfg->k.cx, cfg->k.cy};
  cudaMemcpyAsync(p->kbase.p, kb, sizeof(kb), cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(p->dirs.p, cfg->dirs, sizeof(int) * CSF_MAX_DIRECTIONS, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(p->pair_i.p, cfg->pair_i, sizeof(int) * CSF_MAX_PAIRS, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(p->pair_j.p, cfg->pair_j, sizeof(int) * CSF_MAX_PAIRS, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemsetAsync(p->st.p, 0, sizeof(TrackState), ctx->stream);
  cudaMemsetAsync(p->counts.p, 0, sizeof(int) * p->counts.n, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  *out = p;
  return CSF_OK;
}

extern "C" int csf_pipeline_destroy(csf_pipeline p) {
  if (!p) return CSF_OK;
  cudaSetDevice(p->ctx->device);
  cudaStreamSynchronize(p->ctx->stream);
  delete p;
  return CSF_OK;
}

extern "C" int csf_pipeline_upload(csf_pipeline p, const float* depth, const double* gt, int n_frames) {
  if (!p || !depth || !gt || n_frames <= 0) return CSF_EINVAL;
  csf_ctx ctx = p->ctx;
  if (n_frames > p->cfg.max_frames) return fail(ctx, CSF_EINVAL, "csf_pipeline_upload: more frames than max_frames");
  cudaSetDevice(ctx->device);
  const size_t P = static_cast<size_t>(p->W) * p->H;
  CUDA_TRY(ctx, cudaMemcpyAsync(p->frames.p, depth, sizeof(float) * P * n_frames, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(p->gt.p, gt, sizeof(double) * 12 * n_frames, cudaMemcpyHostToDevice, ctx->stream));
  p->n_uploaded = n_frames;
  return CSF_OK;
}

static int pipeline_reset_volume(csf_pipeline p) {
  csf_volume v = p->vol;
  csf_ctx ctx = p->ctx;
  const Launch L = launch_of(ctx);
  if (v->hashed) {
    // device-side bounds only: the run is graph-capturable
    launch_reset_hashed(L, v->hash, v->Dp);
    CUDA_TRY(ctx, cudaMemsetAsync(v->hash.n_blocks, 0, sizeof(int), ctx->stream));
    launch_super_dist(ctx->stream, v->hash);
  } else {
    launch_init_volume(L, v->dense.rw, v->dense.fim, v->n_vox, v->Dp);
  }
  return CSF_OK;
}

static int pipeline_run_body(csf_pipeline p, int n_frames);

extern "C" int csf_pipeline_set_graph(csf_pipeline p, int enable) {
  if (!p) return CSF_EINVAL;
  p->use_graph = enable != 0;
  if (!p->use_graph) {
    cudaSetDevice(p->ctx->device);
    cudaStreamSynchronize(p->ctx->stream);
    for (cudaGraphExec_t& g : p->graph_exec) {
      if (g) cudaGraphExecDestroy(g);
      g = nullptr;
    }
  }
  return CSF_OK;
}

extern "C" int csf_pipeline_run(csf_pipeline p, int n_frames) {
  if (!p) return CSF_EINVAL;
  csf_ctx ctx = p->ctx;
  if (n_frames <= 0 || n_frames > p->n_uploaded) return fail(ctx, CSF_EINVAL, "csf_pipeline_run: frames not uploaded");
  cudaSetDevice(ctx->device);
  // Graph mode replays the captured run: no host work per kernel.  A run is
  // captured only after a stream run of the same frame count (and mode) has
  // set up every lazily allocated scratch; profiling takes the stream path.
  // run_host's per-frame upload waits become external event-wait nodes: a
  // replay waits for the events' latest records (this call's uploads).
  const int m = p->wait_frames ? 1 : 0;
  const bool graph = p->use_graph && !ctx->prof.on;
  if (graph && p->graph_exec[m] && p->exec_frames[m] == n_frames) {
    CUDA_TRY(ctx, cudaGraphLaunch(p->graph_exec[m], ctx->stream));
    ctx->launches += p->graph_launches[m];
    p->n_run = n_frames;
    return CSF_OK;
  }
  if (graph && p->stream_runs[m] > 0 && p->graph_frames[m] == n_frames) {
    if (p->graph_exec[m]) {
      cudaGraphExecDestroy(p->graph_exec[m]);
      p->graph_exec[m] = nullptr;
    }
    cudaGraph_t g = nullptr;
    CUDA_TRY(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    const unsigned long long l0 = ctx->launches;
    p->capturing = true;
    const int rc = pipeline_run_body(p, n_frames);
    p->capturing = false;
    const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce != cudaSuccess) return fail(ctx, CSF_ECUDA, std::string("csf_pipeline_run: capture: ") + cudaGetErrorString(ce));
    const cudaError_t ie = cudaGraphInstantiate(&p->graph_exec[m], g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
      p->graph_exec[m] = nullptr;
      return fail(ctx, CSF_ECUDA, std::string("csf_pipeline_run: graph instantiate: ") + cudaGetErrorString(ie));
    }
    p->graph_launches[m] = ctx->launches - l0;
    p->exec_frames[m] = n_frames;
    ctx->launches = l0;
    CUDA_TRY(ctx, cudaGraphLaunch(p->graph_exec[m], ctx->stream));
    ctx->launches += p->graph_launches[m];
    p->n_run = n_frames;
    return CSF_OK;
  }
  const int rc = pipeline_run_body(p, n_frames);
  if (rc == CSF_OK) {
    ++p->stream_runs[m];
    p->graph_frames[m] = n_frames;
  }
  return rc;
}

static int pipeline_run_body(csf_pipeline p, int n_frames) {
  csf_ctx ctx = p->ctx;
  int rc = pipeline_reset_volume(p);
  if (rc) return rc;
  const Launch L = launch_of(ctx);
  const csf_pipeline_cfg& cfg = p->cfg;
  const int W = p->W, H = p->H, C = p->C;
  const size_t P = static_cast<size_t>(W) * H;
  csf_volume v = p->vol;
  const double cos_max = csf_det::cos(cfg.icp.theta_max_deg * M_PI / 180.0);
  double* pyr[3] = {p->pyr0.p, p->pyr1.p, p->pyr2.p};
  TrackState* st = p->st.p;
  const int* nblk = v->hashed ? v->hash.n_blocks : nullptr;
  const int* counters = v->hashed ? v->alloc.counters : nullptr;

  if (p->order == 2)
    launch_seed2(L, p->Dp, p->pair_i.p, p->pair_j.p, p->n_pairs, cfg.h, p->gt.p, p->kbase.p, p->pose.p,
                 p->intr_levels.p, p->levels);
  else
    launch_seed(L, p->G, p->Dp, p->dirs.p, p->D, cfg.h, p->gt.p, p->kbase.p, p->pose.p, p->intr_levels.p, p->levels);
  launch_frame_begin(L, st, 0);
  if (p->wait_frames)
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, p->frame_ev[0], p->capturing ? cudaEventWaitExternal : 0));
  launch_bilateral(L, p->frames.p, nullptr, p->raw.p, p->pyr0.p, W, H, 4.5, 0.03, 3);
  int* upd = &st->pad[1];
  rc = volume_fuse(v, p->raw.p, W, H, p->pose.p, p->intr_levels.p, upd);
  if (rc) return rc;
  launch_frame_end(L, st, p->pose.p, p->traj.p, p->Dp, p->stats.p, nblk, counters);

  for (int f = 1; f < n_frames; ++f) {
    launch_frame_begin(L, st, f);
    if (p->wait_frames)
      CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, p->frame_ev[f], p->capturing ? cudaEventWaitExternal : 0));
    {
      PROF(ctx, kPBilateral);
      launch_bilateral(L, p->frames.p + P * f, nullptr, p->raw.p, p->pyr0.p, W, H, 4.5, 0.03, 3);
    }
    {
      PROF(ctx, kPDownsample);
      if (p->levels > 1) launch_downsample(L, p->pyr0.p, p->pyr1.p, W, H, 0.03);
      if (p->levels > 2) launch_downsample(L, p->pyr1.p, p->pyr2.p, W / 2, H / 2, 0.03);
    }
    for (int li = 0; li < p->levels; ++li) {
      const int level = p->levels - 1 - li;
      const int wl = W >> level, hl = H >> level;
      const double* kl = p->intr_levels.p + level * 4 * C;
      launch_level_begin(L, st, p->pose.p, p->pred_pose.p, p->Dp);
      raycast_dev(v, p->pred_pose.p, kl, wl, hl, cfg.rc, p->hits.p, p->vre.p, p->nre.p, p->vim.p, p->nim.p);
      const int stride = std::max(1, cfg.icp.level_pixel_stride[li]);
      PROF(ctx, kPIcpReduce);
      if (p->order == 2) {
        for (int it = 0; it < cfg.icp.level_iterations[li]; ++it)
          launch_icp_iteration2(L, p->Dp, st, pyr[level], wl, hl, stride, kl, p->pose.p, p->vre.p, p->nre.p,
                                p->vim.p, p->nim.p, cfg.icp.d_max, cos_max, p->partials.p, p->counts.p, p->stage.p,
                                level, cfg.icp.step_tolerance);
      } else {
        // every iteration of the level in one cooperative launch (breaks on the device)
        launch_icp_level(L, p->Dp, st, pyr[level], wl, hl, stride, kl, p->pose.p, p->vre.p, p->nre.p, p->vim.p,
                         p->nim.p, cfg.icp.d_max, cos_max, cfg.icp.level_iterations[li], level,
                         cfg.icp.step_tolerance, p->partials.p, p->counts.p);
      }
    }
    if (cfg.keyframe_interval > 0 && f % cfg.keyframe_interval == 0 && p->order == 1)
      launch_keyframe_seed(L, p->G, p->Dp, p->dirs.p, p->D, cfg.h, f / cfg.keyframe_interval, p->pose.p);
    rc = volume_fuse(v, p->raw.p, W, H, p->pose.p, p->intr_levels.p, upd);
    if (rc) return rc;
    launch_frame_end(L, st, p->pose.p, p->traj.p, p->Dp, p->stats.p, nblk, counters);
  }
  if (p->order == 2)
    launch_objective2(L, p->Dp, p->n_pairs, p->traj.p, p->gt.p, n_frames, cfg.objective, p->out.p);
  else
    launch_objective(L, p->G, p->Dp, p->D, p->traj.p, p->gt.p, n_frames, cfg.objective, cfg.h, p->out.p);
  p->n_run = n_frames;
  CUDA_TRY(ctx, cudaGetLastError());
  char lmsg[256];
  if (take_launch_error(lmsg, sizeof(lmsg))) return fail(ctx, CSF_ECUDA, std::string("csf_pipeline_run: ") + lmsg);
  return CSF_OK;
}

extern "C" int csf_pipeline_result(csf_pipeline p, double* gradient, double* objective, double* poses,
                                   int32_t* stats) {
  if (!p) return CSF_EINVAL;
  csf_ctx ctx = p->ctx;
  cudaSetDevice(ctx->device);
  int rc = sync_check(ctx, "csf_pipeline_run");
  if (rc) return rc;
  std::vector<double> out(2 + std::max(CSF_MAX_DIRECTIONS, 3 * CSF_MAX_PAIRS));
  CUDA_TRY(ctx, d2h(out.data(), p->out.p, sizeof(double) * out.size(), ctx->stream));
  if (objective) *objective = out[0];
  const double hh = p->cfg.h;
  if (gradient) {
    if (p->order == 2)  // the run's derivative: one Hessian entry per pair
      for (int q = 0; q < p->n_pairs; ++q) gradient[q] = out[2 + 3 * q + 2] / (hh * hh);
    else
      for (int d = 0; d < p->D; ++d) gradient[d] = out[2 + d];
  }
  const int n = p->n_run;
  if (poses) {
    std::vector<double> t(static_cast<size_t>(n) * 12 * p->C);
    CUDA_TRY(ctx, d2h(t.data(), p->traj.p, sizeof(double) * t.size(), ctx->stream));
    const int Cu = 1 + p->D;
    for (int f = 0; f < n; ++f)
      for (int e = 0; e < 12; ++e)
        for (int c = 0; c < Cu; ++c)
          poses[(static_cast<size_t>(f) * 12 + e) * Cu + c] = t[(static_cast<size_t>(f) * 12 + e) * p->C + c];
  }
  if (stats) CUDA_TRY(ctx, d2h(stats, p->stats.p, sizeof(int) * 8 * n, ctx->stream));
  return CSF_OK;
}

extern "C" int csf_pipeline_hessian(csf_pipeline p, double* hessian, double* grad1, double* grad2, double* objective,
                                    double* poses, int32_t* stats) {
  if (!p) return CSF_EINVAL;
  if (p->order != 2) return fail(p->ctx, CSF_EINVAL, "csf_pipeline_hessian: pipeline was created with order 1");
  csf_ctx ctx = p->ctx;
  cudaSetDevice(ctx->device);
  const int rc = csf_pipeline_result(p, nullptr, objective, poses, stats);
  if (rc) return rc;
  std::vector<double> out(2 + 3 * p->n_pairs);
  CUDA_TRY(ctx, d2h(out.data(), p->out.p, sizeof(double) * out.size(), ctx->stream));
  const double h = p->cfg.h;
  for (int q = 0; q < p->n_pairs; ++q) {
    if (hessian) hessian[q] = out[2 + 3 * q + 2] / (h * h);  // extract_hessian, csfd.hpp:319
    if (grad1) grad1[q] = out[2 + 3 * q] / h;
    if (grad2) grad2[q] = out[2 + 3 * q + 1] / h;
  }
  return CSF_OK;
}

// Debug hook (not part of the public header): a copy of one internal buffer
// of the last run (0 vre, 1 nre, 2 vim, 3 nim, 4 raw depth, 5 pyr0, 6 pyr1,
// 7 pyr2, 8 hits, 9 pose, 10 traj, 11 rw of the volume, 12 fim of the volume).
extern "C" int csf_debug_pipeline_buffer(csf_pipeline p, int which, void* host, size_t bytes) {
  if (!p || !host) return CSF_EINVAL;
  cudaSetDevice(p->ctx->device);
  const void* src = nullptr;
  switch (which) {
    case 0: src = p->vre.p; break;
    case 1: src = p->nre.p; break;
    case 2: src = p->vim.p; break;
    case 3: src = p->nim.p; break;
    case 4: src = p->raw.p; break;
    case 5: src = p->pyr0.p; break;
    case 6: src = p->pyr1.p; break;
    case 7: src = p->pyr2.p; break;
    case 8: src = p->hits.p; break;
    case 9: src = p->pose.p; break;
    case 10: src = p->traj.p; break;
    case 11: src = p->vol->hashed ? static_cast<const void*>(p->vol->hash.rw) : p->vol->dense.rw; break;
    case 12: src = p->vol->hashed ? static_cast<const void*>(p->vol->hash.fim) : p->vol->dense.fim; break;
    default: return CSF_EINVAL;
  }
  cudaStreamSynchronize(p->ctx->stream);
  CUDA_TRY(p->ctx, cudaMemcpy(host, src, bytes, cudaMemcpyDeviceToHost));
  return CSF_OK;
}

extern "C" int csf_pipeline_volume(csf_pipeline p, csf_volume* out) {
  if (!p || !out) return CSF_EINVAL;
  *out = p->vol;
  return CSF_OK;
}

extern "C" int csf_pipeline_download_rgb(csf_pipeline p, int frame, unsigned char* out) {
  if (!p || !out || frame < 0 || frame >= p->cfg.max_frames) return CSF_EINVAL;
  csf_ctx ctx = p->ctx;
  if (!p->rgb.p) return fail(ctx, CSF_EINVAL, "csf_pipeline_download_rgb: no colour frames were ingested");
  cudaSetDevice(ctx->device);
  const size_t P = static_cast<size_t>(p->W) * p->H;
  if (p->copy_stream) CUDA_TRY(ctx, cudaStreamSynchronize(p->copy_stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(out, p->rgb.p + 3 * P * frame, 3 * P, cudaMemcpyDeviceToHost, ctx->stream));
  return sync_check(ctx, "csf_pipeline_download_rgb");
}

// One end-to-end call.  The frames go up on a copy stream, one event per
// frame, and frame f's kernels wait only for frame f's upload, so (from
// pinned host memory) the H2D of later frames overlaps the device work of
// earlier ones.
extern "C" int csf_pipeline_run_host(csf_pipeline p, const float* depth, const double* gt, int n_frames,
                                     double* gradient, double* objective) {
  return csf_pipeline_run_host_rgbd(p, depth, nullptr, gt, n_frames, gradient, objective);
}

extern "C" int csf_pipeline_run_host_rgbd(csf_pipeline p, const float* depth, const unsigned char* rgb,
                                          const double* gt, int n_frames, double* gradient, double* objective) {
  if (!p || !depth || !gt || n_frames <= 0) return CSF_EINVAL;
  csf_ctx ctx = p->ctx;
  if (n_frames > p->cfg.max_frames) return fail(ctx, CSF_EINVAL, "csf_pipeline_run_host: more frames than max_frames");
  cudaSetDevice(ctx->device);
  if (!p->copy_stream) CUDA_TRY(ctx, cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
  while (static_cast<int>(p->frame_ev.size()) < n_frames) {
    cudaEvent_t e;
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->frame_ev.push_back(e);
  }
  const size_t P = static_cast<size_t>(p->W) * p->H;
  // the copy stream starts after everything already queued on the context
  CUDA_TRY(ctx, cudaEventRecord(p->frame_ev[0], ctx->stream));
  CUDA_TRY(ctx, cudaStreamWaitEvent(p->copy_stream, p->frame_ev[0], 0));
  CUDA_TRY(ctx, cudaMemcpyAsync(p->gt.p, gt, sizeof(double) * 12 * n_frames, cudaMemcpyHostToDevice, ctx->stream));
  if (rgb && !p->rgb.p) CUDA_TRY(ctx, p->rgb.alloc(P * 3 * static_cast<size_t>(p->cfg.max_frames)));
  for (int f = 0; f < n_frames; ++f) {
    CUDA_TRY(ctx, cudaMemcpyAsync(p->frames.p + P * f, depth + P * f, sizeof(float) * P, cudaMemcpyHostToDevice,
                                  p->copy_stream));
    CUDA_TRY(ctx, cudaEventRecord(p->frame_ev[f], p->copy_stream));
    // colour after the frame's depth event: the frame's kernels never wait on it
    if (rgb)
      CUDA_TRY(ctx, cudaMemcpyAsync(p->rgb.p + 3 * P * f, rgb + 3 * P * f, 3 * P, cudaMemcpyHostToDevice,
                                    p->copy_stream));
  }
  p->n_uploaded = n_frames;
  p->wait_frames = true;
  int rc = csf_pipeline_run(p, n_frames);
  p->wait_frames = false;
  if (rc) {
    // the uploads still read the caller's buffer: finish them before returning
    cudaStreamSynchronize(p->copy_stream);
    return rc;
  }
  rc = csf_pipeline_result(p, gradient, objective, nullptr, nullptr);
  // the colour uploads borrow the caller's buffer until they land
  if (rgb) {
    const cudaError_t e = cudaStreamSynchronize(p->copy_stream);
    if (!rc && e != cudaSuccess) return fail(ctx, CSF_ECUDA, cudaGetErrorString(e));
  }
  return rc;
}

// ---------------------------------------------------------------------------
// track_frame (real tracker on the device)
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// point queries: sample_tsdf / sample_gradient (tsdf.hpp:148-196), measured_tsdf (tsdf.hpp:97-140)
// ---------------------------------------------------------------------------
static int sample_points_common(csf_volume v, const double* points, int n, int grad, double* out, int32_t* valid) {
  if (!v || (n > 0 && (!points || !out || !valid)) || n < 0) return CSF_EINVAL;
  csf_ctx ctx = v->ctx;
  if (v->order != 1) return fail(ctx, CSF_EINVAL, "point queries take first-order volumes");
  cudaSetDevice(ctx->device);
  const int D = v->D, Dp = v->Dp, C = 1 + D, Cp = 1 + Dp;
  const size_t rows = static_cast<size_t>(n) * 3;
  std::vector<double> pts(rows * Cp, 0.0);
  for (size_t r = 0; r < rows; ++r)
    for (int c = 0; c < C; ++c) pts[r * Cp + c] = points[r * C + c];
  const size_t outn = static_cast<size_t>(n) * (grad ? 3 : 1) * Cp;
  DevBuf<double> dp, dout;
  DevBuf<int> dv;
  CUDA_TRY(ctx, dp.alloc(std::max<size_t>(pts.size(), 1)));
  CUDA_TRY(ctx, dout.alloc(std::max<size_t>(outn, 1)));
  CUDA_TRY(ctx, dv.alloc(std::max(n, 1)));
  if (n > 0) {
    CUDA_TRY(ctx, cudaMemcpyAsync(dp.p, pts.data(), sizeof(double) * pts.size(), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemsetAsync(dout.p, 0, sizeof(double) * outn, ctx->stream));
  }
  launch_sample_points(launch_of(ctx), v->hashed, v->dense, v->hash, Dp, dp.p, n, grad, dout.p, dv.p);
  const int rc = sync_check(ctx, grad ? "csf_sample_gradient" : "csf_sample_tsdf");
  if (rc) return rc;
  std::vector<double> o(outn);
  std::vector<int> vv(std::max(n, 1));
  if (n > 0) {
    CUDA_TRY(ctx, d2h(o.data(), dout.p, sizeof(double) * outn, ctx->stream));
    CUDA_TRY(ctx, d2h(vv.data(), dv.p, sizeof(int) * n, ctx->stream));
  }
  const size_t orow = static_cast<size_t>(n) * (grad ? 3 : 1);
  for (size_t r = 0; r < orow; ++r)
    for (int c = 0; c < C; ++c) out[r * C + c] = o[r * Cp + c];
  for (int i = 0; i < n; ++i) valid[i] = vv[i];
  return CSF_OK;
}

extern "C" int csf_sample_tsdf(csf_volume v, const double* points, int n, double* values, int32_t* valid) {
  return sample_points_common(v, points, n, 0, values, valid);
}
extern "C" int csf_sample_gradient(csf_volume v, const double* points, int n, double* gradients, int32_t* valid) {
  return sample_points_common(v, points, n, 1, gradients, valid);
}

static int measured_tsdf_impl(csf_ctx ctx, const double* depth, bool lifted, int w, int h,
                              const double* world_to_camera, const double* intr, double mu, const double* points,
                              const double* center, int n, int n_channels, double* psi, int32_t* valid);

extern "C" int csf_measured_tsdf(csf_ctx ctx, const double* depth, int w, int h, const double* world_to_camera,
                                 const double* intr, double mu, const double* points, const double* center, int n,
                                 int n_channels, double* psi, int32_t* valid) {
  return measured_tsdf_impl(ctx, depth, false, w, h, world_to_camera, intr, mu, points, center, n, n_channels, psi,
                            valid);
}

extern "C" int csf_measured_tsdf_lifted(csf_ctx ctx, const double* depth, int w, int h,
                                        const double* world_to_camera, const double* intr, double mu,
                                        const double* points, const double* center, int n, int n_channels,
                                        double* psi, int32_t* valid) {
  return measured_tsdf_impl(ctx, depth, true, w, h, world_to_camera, intr, mu, points, center, n, n_channels, psi,
                            valid);
}

static int measured_tsdf_impl(csf_ctx ctx, const double* depth, bool lifted, int w, int h,
                              const double* world_to_camera, const double* intr, double mu, const double* points,
                              const double* center, int n, int n_channels, double* psi, int32_t* valid) {
  if (!ctx || !depth || !world_to_camera || !intr || !center || w <= 0 || h <= 0 || n < 0 || n_channels < 0 ||
      n_channels > CSF_MAX_DIRECTIONS || (n > 0 && (!points || !psi || !valid)))
    return CSF_EINVAL;
  if (n_channels > 0 && (intr[0] == 0.0 || intr[1 + n_channels] == 0.0))
    return fail(ctx, CSF_EDOMAIN, "csf_measured_tsdf: Complex division by zero real part (fx or fy = 0)");
  cudaSetDevice(ctx->device);
  const int D = n_channels, C = 1 + D;
  const size_t P = static_cast<size_t>(w) * h;
  DevBuf<double> buf, dout;
  DevBuf<int> dv;
  const bool channels = lifted && D > 0;
  CUDA_TRY(ctx, buf.alloc(P + 12 * C + 4 * C + 3 * C + 3 * static_cast<size_t>(std::max(n, 1)) +
                          (channels ? P * D : 0)));
  CUDA_TRY(ctx, dout.alloc(static_cast<size_t>(std::max(n, 1)) * C));
  CUDA_TRY(ctx, dv.alloc(std::max(n, 1)));
  double* d_depth = buf.p;
  double* d_pose = d_depth + P;
  double* d_intr = d_pose + 12 * C;
  double* d_center = d_intr + 4 * C;
  double* d_pts = d_center + 3 * C;
  double* d_dch = channels ? d_pts + 3 * static_cast<size_t>(std::max(n, 1)) : nullptr;
  std::vector<double> re, ch;
  if (!lifted) {
    CUDA_TRY(ctx, cudaMemcpyAsync(d_depth, depth, sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream));
  } else {
    re.resize(P);
    ch.assign(channels ? P * D : 0, 0.0);
    for (size_t i = 0; i < P; ++i) {
      re[i] = depth[i * C];
      for (int d = 0; d < D && channels; ++d) ch[i * D + d] = depth[i * C + 1 + d];
    }
    CUDA_TRY(ctx, cudaMemcpyAsync(d_depth, re.data(), sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream));
    if (channels)
      CUDA_TRY(ctx, cudaMemcpyAsync(d_dch, ch.data(), sizeof(double) * P * D, cudaMemcpyHostToDevice, ctx->stream));
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(d_pose, world_to_camera, sizeof(double) * 12 * C, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(d_intr, intr, sizeof(double) * 4 * C, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(d_center, center, sizeof(double) * 3 * C, cudaMemcpyHostToDevice, ctx->stream));
  if (n > 0) {
    CUDA_TRY(ctx, cudaMemcpyAsync(d_pts, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemsetAsync(dout.p, 0, sizeof(double) * n * C, ctx->stream));
  }
  launch_measured_points(launch_of(ctx), d_depth, w, h, d_pose, d_intr, mu, d_pts, d_center, n, D, dout.p, dv.p,
                         d_dch);
  const int rc = sync_check(ctx, "csf_measured_tsdf");
  if (rc) return rc;
  if (n > 0) {
    CUDA_TRY(ctx, d2h(psi, dout.p, sizeof(double) * n * C, ctx->stream));
    std::vector<int> vv(n);
    CUDA_TRY(ctx, d2h(vv.data(), dv.p, sizeof(int) * n, ctx->stream));
    for (int i = 0; i < n; ++i) valid[i] = vv[i];
  }
  return CSF_OK;
}

// ---------------------------------------------------------------------------
// checkpoints: the reference's "CSFVOL 1" container (tsdf.cpp:61-153)
// ---------------------------------------------------------------------------
namespace csfi {
void launch_rebuild_index(cudaStream_t stream, const int* coords, int n_blocks, int* grid, unsigned* occ, int gbits);
}

namespace {
// host copies of block_key / block_hash (geometry.cuh)
uint64_t host_block_key(int bx, int by, int bz) {
  constexpr int kBias = 1 << 20;
  return (static_cast<uint64_t>(static_cast<uint32_t>(bx + kBias)) << 42) |
         (static_cast<uint64_t>(static_cast<uint32_t>(by + kBias)) << 21) |
         static_cast<uint64_t>(static_cast<uint32_t>(bz + kBias));
}
uint32_t host_block_hash(int bx, int by, int bz, int bits) {
  return ((static_cast<uint32_t>(bx) * 73856093u) ^ (static_cast<uint32_t>(by) * 19349669u) ^
          (static_cast<uint32_t>(bz) * 83492791u)) &
         ((1u << bits) - 1u);
}
void write_plane(std::ofstream& out, const std::vector<float>& plane) {
  out.write(reinterpret_cast<const char*>(plane.data()), static_cast<std::streamsize>(plane.size() * sizeof(float)));
}
bool read_plane(std::ifstream& in, std::vector<float>& plane) {
  in.read(reinterpret_cast<char*>(plane.data()), static_cast<std::streamsize>(plane.size() * sizeof(float)));
  return static_cast<size_t>(in.gcount()) == plane.size() * sizeof(float);
}
}  // namespace

extern "C" int csf_volume_save(csf_volume v, const char* path) {
  if (!v || !path) return CSF_EINVAL;
  csf_ctx ctx = v->ctx;
  if (v->order != 1) return fail(ctx, CSF_EINVAL, "csf_volume_save: second-order volumes are not checkpointed");
  cudaSetDevice(ctx->device);
  const long long n = volume_voxels_now(v);
  const int D = v->D, C = 1 + D;
  std::vector<double> field(static_cast<size_t>(n) * C), weight(n);
  int rc = n > 0 ? csf_volume_download(v, field.data(), weight.data()) : CSF_OK;
  if (rc) return rc;
  std::vector<int32_t> coords;
  if (v->hashed) {
    coords.resize(static_cast<size_t>(n / 512) * 3);
    if (!coords.empty())
      CUDA_TRY(ctx, d2h(coords.data(), v->hash.coords, sizeof(int32_t) * coords.size(), ctx->stream));
  }
  bool any_im = false;
  for (long long i = 0; i < n && !any_im; ++i)
    for (int d = 0; d < D; ++d)
      if (field[i * C + 1 + d] != 0.0) {
        any_im = true;
        break;
      }
  std::ofstream out(path, std::ios::binary);
  if (!out) return fail(ctx, CSF_ERUNTIME, std::string("cannot write volume: ") + path);
  out.precision(17);
  out << "CSFVOL 1\n";
  if (v->hashed) {
    const HashDev& hd = v->hash;
    out << "hashed " << hd.bits << " " << hd.max_blocks << "\n";
    out << "voxel_size " << hd.vs << "\n";
    out << "origin " << hd.ox << " " << hd.oy << " " << hd.oz << "\n";
    out << "mu " << hd.mu << "\n";
    out << "weight_cap " << hd.cap << "\n";
    out << "blocks " << n / 512 << "\n";
  } else {
    const DenseDev& dd = v->dense;
    out << "dims " << dd.nx << " " << dd.ny << " " << dd.nz << "\n";
    out << "voxel_size " << dd.vs << "\n";
    out << "origin " << dd.ox << " " << dd.oy << " " << dd.oz << "\n";
    out << "mu " << dd.mu << "\n";
    out << "weight_cap " << dd.cap << "\n";
  }
  out << "channels field weight";
  if (any_im)
    for (int d = 0; d < D; ++d) out << " derivative";
  out << "\n";
  out << "data\n";
  if (v->hashed && !coords.empty())
    out.write(reinterpret_cast<const char*>(coords.data()), static_cast<std::streamsize>(coords.size() * 4));
  std::vector<float> plane(n);
  for (long long i = 0; i < n; ++i) plane[i] = static_cast<float>(field[i * C]);
  write_plane(out, plane);
  for (long long i = 0; i < n; ++i) plane[i] = static_cast<float>(weight[i]);
  write_plane(out, plane);
  if (any_im)
    for (int d = 0; d < D; ++d) {
      for (long long i = 0; i < n; ++i) plane[i] = static_cast<float>(field[i * C + 1 + d]);
      write_plane(out, plane);
    }
  if (!out) return fail(ctx, CSF_ERUNTIME, std::string("short write: ") + path);
  return CSF_OK;
}

extern "C" int csf_volume_load(csf_ctx ctx, const char* path, int n_channels, csf_volume* out_vol) {
  if (!ctx || !path || !out_vol) return CSF_EINVAL;
  *out_vol = nullptr;
  std::ifstream in(path, std::ios::binary);
  if (!in) return fail(ctx, CSF_ERUNTIME, std::string("cannot open volume: ") + path);
  std::string line;
  if (!std::getline(in, line) || line != "CSFVOL 1")
    return fail(ctx, CSF_ERUNTIME, std::string("not a volume checkpoint: ") + path);
  csf_volume_params vp{};
  csf_hash_params hp{};
  bool hashed = false, saw_data = false;
  int n_im = 0;
  long long n_blocks = -1;
  while (std::getline(in, line)) {
    std::istringstream ls(line);
    std::string key;
    ls >> key;
    if (key == "data") {
      saw_data = true;
      break;
    } else if (key == "dims") {
      ls >> vp.dims[0] >> vp.dims[1] >> vp.dims[2];
    } else if (key == "hashed") {
      hashed = true;
      ls >> hp.bucket_bits >> hp.max_blocks;
    } else if (key == "blocks") {
      ls >> n_blocks;
    } else if (key == "voxel_size") {
      ls >> vp.voxel_size;
    } else if (key == "origin") {
      ls >> vp.origin[0] >> vp.origin[1] >> vp.origin[2];
    } else if (key == "mu") {
      ls >> vp.mu;
    } else if (key == "weight_cap") {
      ls >> vp.weight_cap;
    } else if (key == "channels") {
      std::string tok;
      while (ls >> tok) n_im += tok == "derivative";
    } else {
      return fail(ctx, CSF_ERUNTIME, "unknown checkpoint field '" + key + "': " + path);
    }
  }
  if (!saw_data || !(vp.voxel_size > 0.0) ||
      (hashed ? (n_blocks < 0 || hp.max_blocks < n_blocks) : (vp.dims[0] <= 0 || vp.dims[1] <= 0 || vp.dims[2] <= 0)))
    return fail(ctx, CSF_ERUNTIME, std::string("malformed volume checkpoint: ") + path);
  const int D = n_channels >= 0 ? n_channels : n_im;
  if (n_im != 0 && n_im != D)
    return fail(ctx, CSF_EINVAL, "csf_volume_load: the checkpoint carries " + std::to_string(n_im) + " channels");
  csf_volume v = nullptr;
  int rc;
  std::vector<int32_t> coords;
  if (hashed) {
    hp.voxel_size = vp.voxel_size;
    for (int a = 0; a < 3; ++a) hp.origin[a] = vp.origin[a];
    hp.mu = vp.mu;
    hp.weight_cap = vp.weight_cap;
    coords.resize(static_cast<size_t>(n_blocks) * 3);
    in.read(reinterpret_cast<char*>(coords.data()), static_cast<std::streamsize>(coords.size() * 4));
    if (static_cast<size_t>(in.gcount()) != coords.size() * 4)
      return fail(ctx, CSF_ERUNTIME, std::string("volume checkpoint truncated: ") + path);
    rc = csf_volume_create_hashed(ctx, &hp, D, &v);
  } else {
    rc = csf_volume_create_dense(ctx, &vp, D, &v);
  }
  if (rc) return rc;
  const long long n = hashed ? n_blocks * 512 : static_cast<long long>(vp.dims[0]) * vp.dims[1] * vp.dims[2];
  std::vector<float> fpl(n), wpl(n);
  bool ok = read_plane(in, fpl) && read_plane(in, wpl);
  std::vector<std::vector<float>> ims(n_im, std::vector<float>(n));
  for (int d = 0; d < n_im && ok; ++d) ok = read_plane(in, ims[d]);
  if (!ok) {
    csf_volume_destroy(v);
    return fail(ctx, CSF_ERUNTIME, std::string("volume checkpoint truncated: ") + path);
  }
  if (hashed && n_blocks > 0) {
    // the canonical hash structure: chains sorted by key, pool ids = file order
    const int bits = hp.bucket_bits;
    std::vector<int32_t> heads(size_t(1) << bits, -1), next(n_blocks, -1);
    std::vector<uint64_t> keys(n_blocks);
    for (long long b = 0; b < n_blocks; ++b) {
      const int bx = coords[3 * b], by = coords[3 * b + 1], bz = coords[3 * b + 2];
      keys[b] = host_block_key(bx, by, bz);
      int32_t* link = &heads[host_block_hash(bx, by, bz, bits)];
      while (*link >= 0 && keys[*link] < keys[b]) link = &next[*link];
      next[b] = *link;
      *link = static_cast<int32_t>(b);
    }
    const int nb = static_cast<int>(n_blocks);
    CUDA_TRY(ctx, cudaMemcpyAsync(v->hash.heads, heads.data(), sizeof(int32_t) * heads.size(), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(v->hash.next, next.data(), sizeof(int32_t) * n_blocks, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(v->hash.keys, keys.data(), sizeof(uint64_t) * n_blocks, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(v->hash.coords, coords.data(), sizeof(int32_t) * coords.size(), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(v->hash.n_blocks, &nb, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    launch_rebuild_index(ctx->stream, v->hash.coords, nb, v->hash.grid, v->hash.occ, v->hash.gbits);
    launch_super_dist(ctx->stream, v->hash);
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  }
  const int C = 1 + D;
  std::vector<double> field(static_cast<size_t>(n) * C, 0.0), weight(n);
  for (long long i = 0; i < n; ++i) {
    field[i * C] = static_cast<double>(fpl[i]);
    weight[i] = static_cast<double>(wpl[i]);
    for (int d = 0; d < n_im; ++d) field[i * C + 1 + d] = static_cast<double>(ims[d][i]);
  }
  rc = n > 0 ? csf_volume_upload(v, field.data(), weight.data()) : CSF_OK;
  if (rc) {
    csf_volume_destroy(v);
    return rc;
  }
  *out_vol = v;
  return CSF_OK;
}

// ---------------------------------------------------------------------------
// BASELINE config 5: view scoring (views.cu; builder-defined objective)
// ---------------------------------------------------------------------------
extern "C" int csf_view_scores(csf_volume v, const double* poses, int n_views, const csf_intrinsics* k, double w0,
                               double beta, double h, double* scores, double* grads) {
  if (!v || !poses || !k || n_views < 0 || !scores) return CSF_EINVAL;
  csf_ctx ctx = v->ctx;
  if (!v->hashed || v->order != 1 || v->Dp != 6)
    return fail(ctx, CSF_EINVAL, "csf_view_scores: needs a hashed volume created with 6 channels");
  if (!(h > 0.0) || h > 1e-6) return fail(ctx, CSF_EINVAL, "StepSize: step must satisfy 0 < h <= 1e-6");
  if (k->width <= 0 || k->height <= 0) return fail(ctx, CSF_EINVAL, "csf_view_scores: bad image size");
  cudaSetDevice(ctx->device);
  const int W = k->width, H = k->height;
  const size_t P = static_cast<size_t>(W) * H;
  constexpr int C = 7;
  // views per pass: all of them while the terms fit 2 GB (one host sync per
  // pass, for the sums)
  const int chunk = std::max(1, std::min(n_views, static_cast<int>((size_t(1) << 28) / (C * P))));
  CUDA_TRY(ctx, v->s_vre.alloc(3 * P));
  CUDA_TRY(ctx, v->s_nre.alloc(3 * P));
  CUDA_TRY(ctx, v->s_vim.alloc(3 * P * 6));
  CUDA_TRY(ctx, v->s_nim.alloc(3 * P * 6));
  CUDA_TRY(ctx, v->s_hits.alloc(2 * P));
  CUDA_TRY(ctx, v->s_pose.alloc(12 * C + 12 * static_cast<size_t>(n_views)));
  CUDA_TRY(ctx, v->s_intr.alloc(4 * C + 4));
  CUDA_TRY(ctx, v->s_terms.alloc(static_cast<size_t>(chunk) * C * P));
  double* const terms = v->s_terms.p;
  double* d_pose = v->s_pose.p;
  double* d_views = v->s_pose.p + 12 * C;
  double* d_intr = v->s_intr.p;
  double* d_k4 = v->s_intr.p + 4 * C;
  const double k4[4] = {k->fx, k->fy, k->cx, k->cy};
  CUDA_TRY(ctx, cudaMemcpyAsync(d_views, poses, sizeof(double) * 12 * n_views, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(d_k4, k4, sizeof(k4), cudaMemcpyHostToDevice, ctx->stream));
  csf_raycast_cfg rc;
  csf_default_raycast_cfg(&rc);
  const Launch L = launch_of(ctx);
  std::vector<double> out(static_cast<size_t>(chunk) * C);
  for (int v0 = 0; v0 < n_views; v0 += chunk) {
    const int nv = std::min(chunk, n_views - v0);
    for (int j = 0; j < nv; ++j) {
      launch_view_seed(L, d_views + 12 * (v0 + j), d_k4, h, d_pose, d_intr);
      raycast_dev(v, d_pose, d_intr, W, H, rc, v->s_hits.p, v->s_vre.p, v->s_nre.p, v->s_vim.p, v->s_nim.p);
      PROF(ctx, kPMisc);
      launch_view_terms(L, v->hash, v->s_vre.p, v->s_nre.p, v->s_vim.p, W, H, w0, beta, terms + j * C * P);
    }
    const int rc2 = tree_sum_slots(ctx->stream, ctx->energy, terms, static_cast<int>(P), nv * C, out.data());
    if (rc2 == 5) return fail(ctx, CSF_ENOMEM, "csf_view_scores: out of device memory");
    if (rc2) return fail(ctx, CSF_ECUDA, "csf_view_scores: CUDA error");
    for (int j = 0; j < nv; ++j) {
      scores[v0 + j] = out[j * C];
      if (grads)
        for (int d = 0; d < 6; ++d) grads[(v0 + j) * 6 + d] = out[j * C + 1 + d] / h;  // extract_derivative
    }
  }
  return sync_check(ctx, "csf_view_scores");
}

// ---------------------------------------------------------------------------
// icp energy and its CSFD derivatives (icp.hpp:70-91)
// ---------------------------------------------------------------------------
extern "C" int csf_icp_energy_derivs(csf_ctx ctx, const double* corrs, int n, const double* base, const double* xi,
                                     double h, double* energy, double* gradient, double* hessian) {
  if (!ctx || (n > 0 && !corrs) || !base || n < 0) return CSF_EINVAL;
  if (!(h > 0.0) || h > 1e-6) return fail(ctx, CSF_EINVAL, "StepSize: step must satisfy 0 < h <= 1e-6");
  cudaSetDevice(ctx->device);
  const size_t need = static_cast<size_t>(std::max(n, 1)) * 9;
  if (ctx->corr_upload_cap < need) {
    if (ctx->corr_upload) cudaFree(ctx->corr_upload);
    ctx->corr_upload = nullptr;
    ctx->corr_upload_cap = 0;
    CUDA_TRY(ctx, cudaMalloc(&ctx->corr_upload, sizeof(double) * need));
    ctx->corr_upload_cap = need;
  }
  if (n > 0)
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->corr_upload, corrs, sizeof(double) * 9 * n, cudaMemcpyHostToDevice,
                                  ctx->stream));
  const int order = hessian ? 2 : (gradient ? 1 : 0);
  const int rc = icp_energy_derivs(ctx->stream, ctx->energy, ctx->corr_upload, n, base, xi, h, order, energy, gradient,
                                   hessian);
  if (rc == 5) return fail(ctx, CSF_ENOMEM, "csf_icp_energy_derivs: out of device memory");
  if (rc) return fail(ctx, CSF_ECUDA, "csf_icp_energy_derivs: CUDA error");
  return sync_check(ctx, "csf_icp_energy_derivs");
}

// ---------------------------------------------------------------------------
// associate / linearized_step / pairwise_sum (icp.cpp:89-126, 146-153;
// diff.hpp:16-37) on the device
// ---------------------------------------------------------------------------
extern "C" int csf_associate(csf_ctx ctx, const double* mvert, const double* mnorm, const double* pvert,
                             const double* pnorm, int w, int h, const double* camera_to_world,
                             const double* predicted_camera_to_world, const csf_intrinsics* k, const csf_icp_cfg* cfg,
                             int pixel_stride, double* corrs, int* n_corrs) {
  if (!ctx || !mvert || !mnorm || !pvert || !pnorm || !camera_to_world || !predicted_camera_to_world || !k || !cfg ||
      !corrs || !n_corrs || w <= 0 || h <= 0)
    return CSF_EINVAL;
  cudaSetDevice(ctx->device);
  double prm[28];
  std::copy(camera_to_world, camera_to_world + 12, prm);
  csfd::Pose<double> pp;
  for (int e = 0; e < 9; ++e) pp.R.m[e] = predicted_camera_to_world[e];
  for (int e = 0; e < 3; ++e) pp.t.v[e] = predicted_camera_to_world[9 + e];
  const csfd::Pose<double> inv = csfd::inverse(pp);
  for (int e = 0; e < 9; ++e) prm[12 + e] = inv.R.m[e];
  for (int e = 0; e < 3; ++e) prm[21 + e] = inv.t.v[e];
  prm[24] = k->fx; prm[25] = k->fy; prm[26] = k->cx; prm[27] = k->cy;
  const double cos_max = csf_det::cos(cfg->theta_max_deg * M_PI / 180.0);
  const int rc = associate_maps(ctx->stream, ctx->energy, mvert, mnorm, pvert, pnorm, w, h, std::max(1, pixel_stride),
                                prm, cfg->d_max, cos_max, corrs, n_corrs);
  if (rc == 5) return fail(ctx, CSF_ENOMEM, "csf_associate: out of device memory");
  if (rc) return fail(ctx, CSF_ECUDA, "csf_associate: CUDA error");
  return sync_check(ctx, "csf_associate");
}

extern "C" int csf_linearized_step(csf_ctx ctx, const double* corrs, int n, const double* base, double* delta) {
  if (!ctx || (n > 0 && !corrs) || !base || !delta || n < 0) return CSF_EINVAL;
  cudaSetDevice(ctx->device);
  const size_t need = static_cast<size_t>(std::max(n, 1)) * 9;
  if (ctx->corr_upload_cap < need) {
    if (ctx->corr_upload) cudaFree(ctx->corr_upload);
    ctx->corr_upload = nullptr;
    ctx->corr_upload_cap = 0;
    CUDA_TRY(ctx, cudaMalloc(&ctx->corr_upload, sizeof(double) * need));
    ctx->corr_upload_cap = need;
  }
  if (n > 0)
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->corr_upload, corrs, sizeof(double) * 9 * n, cudaMemcpyHostToDevice,
                                  ctx->stream));
  const int tiles = (n + 255) / 256;
  std::vector<double> part(static_cast<size_t>(tiles) * 27);
  const int rc = linearized_tiles(ctx->stream, ctx->corr_upload, n, base, part.data());
  if (rc) return fail(ctx, rc == 5 ? CSF_ENOMEM : CSF_ECUDA, "csf_linearized_step: device failure");
  // canonical order: tiles in groups of 16 summed in order, group totals in order
  double total[27] = {0}, group[27] = {0};
  for (int t = 0; t < tiles; ++t) {
    for (int a = 0; a < 27; ++a) group[a] = group[a] + part[static_cast<size_t>(t) * 27 + a];
    if ((t + 1) % 16 == 0 || t + 1 == tiles) {
      for (int a = 0; a < 27; ++a) {
        total[a] = total[a] + group[a];
        group[a] = 0.0;
      }
    }
  }
  double nb[6], m[6][6], d[6];
  int tr[6];
  for (int i = 0; i < 6; ++i) nb[i] = -total[21 + i];
  csfd::ldlt6_factor_reg<double>(total, m, tr);
  csfd::ldlt6_apply_reg<double>(m, tr, nb, d);
  bool finite = true;
  for (int i = 0; i < 6; ++i) finite = finite && std::isfinite(d[i]);
  for (int i = 0; i < 6; ++i) delta[i] = finite ? d[i] : 0.0;  // delta.allFinite() (icp.cpp:152)
  return CSF_OK;
}

extern "C" int csf_pairwise_sum(csf_ctx ctx, const double* terms, int n, int channels, double* out) {
  if (!ctx || (n > 0 && !terms) || !out || n < 0 || channels <= 0) return CSF_EINVAL;
  cudaSetDevice(ctx->device);
  const size_t C = static_cast<size_t>(channels);
  std::vector<double> t(static_cast<size_t>(n) * C);
  for (int i = 0; i < n; ++i)
    for (size_t c = 0; c < C; ++c) t[c * n + i] = terms[static_cast<size_t>(i) * C + c];  // slot-major
  DevBuf<double> d;
  CUDA_TRY(ctx, d.alloc(std::max<size_t>(t.size(), 1)));
  if (n > 0) CUDA_TRY(ctx, cudaMemcpyAsync(d.p, t.data(), sizeof(double) * t.size(), cudaMemcpyHostToDevice, ctx->stream));
  const int rc = tree_sum_slots(ctx->stream, ctx->energy, d.p, n, channels, out);
  if (rc) return fail(ctx, rc == 5 ? CSF_ENOMEM : CSF_ECUDA, "csf_pairwise_sum: device failure");
  return CSF_OK;
}

// ---------------------------------------------------------------------------
// track_frame (icp.cpp:169-244) — every solver family.  The per-pixel work
// (bilateral filter, pyramid, raycast, association, normal equations,
// energies and their CSFD derivatives) runs on the device; the 6-vector
// step logic of descent.hpp stays on the host, as in the reference.
// ---------------------------------------------------------------------------
namespace {

using Vec6h = std::array<double, 6>;

double sum6h(const Vec6h& a) { return (a[0] + (a[1] + a[2])) + (a[3] + (a[4] + a[5])); }
double dot6h(const Vec6h& a, const Vec6h& b) {
  Vec6h p;
  for (int i = 0; i < 6; ++i) p[i] = a[i] * b[i];
  return sum6h(p);
}
double norm6h(const Vec6h& a) { return std::sqrt(dot6h(a, a)); }

// descent.hpp:16-21 (LineSearchConfig defaults)
struct LineSearch {
  double initial_step = 1.0, shrink = 0.5, sufficient_decrease = 1e-4;
  int max_backtracks = 25;
};

// descent.hpp:34-52
template <typename F>
bool backtracking(F&& loss_at, double loss0, double slope, const LineSearch& cfg, double* alpha_out,
                  double* loss_out, int* err) {
  double alpha = cfg.initial_step;
  for (int k = 0; k < cfg.max_backtracks; ++k) {
    const double trial = loss_at(alpha, err);
    if (*err) return false;
    if (trial <= loss0 + cfg.sufficient_decrease * alpha * slope) {
      *alpha_out = alpha;
      *loss_out = trial;
      return true;
    }
    alpha *= cfg.shrink;
  }
  return false;
}

// descent.hpp:58-101 (GradientStepper: GD or Polak-Ribiere NCG with restarts)
struct Stepper {
  bool ncg;
  int restart_every;
  int since_restart = 0;
  bool have_previous = false;
  Vec6h prev_g{}, prev_d{};
  void reset() {
    have_previous = false;
    since_restart = 0;
  }
  Vec6h propose(const Vec6h& g) {
    Vec6h neg;
    for (int i = 0; i < 6; ++i) neg[i] = -g[i];
    if (!ncg) return neg;
    bool restart = !have_previous || since_restart >= restart_every || dot6h(prev_g, prev_g) == 0.0;
    Vec6h dir = neg;
    if (!restart) {
      Vec6h diff;
      for (int i = 0; i < 6; ++i) diff[i] = g[i] - prev_g[i];
      const double beta = std::max(0.0, dot6h(g, diff) / dot6h(prev_g, prev_g));
      for (int i = 0; i < 6; ++i) dir[i] = neg[i] + beta * prev_d[i];
      if (dot6h(g, dir) >= 0.0) {
        dir = neg;
        restart = true;
      }
    }
    if (restart) since_restart = 0;
    ++since_restart;
    prev_g = g;
    prev_d = dir;
    have_previous = true;
    return dir;
  }
};

// apply_increment (se3.hpp:116-119) on the host with the device's exp_map
// (same source, IEEE arithmetic without contraction on both sides).
void apply_increment_h(const Vec6h& d, double* pose12) {
  double xi[6];
  for (int i = 0; i < 6; ++i) xi[i] = d[i];
  csfd::Pose<double> cur;
  for (int e = 0; e < 9; ++e) cur.R.m[e] = pose12[e];
  for (int e = 0; e < 3; ++e) cur.t.v[e] = pose12[9 + e];
  const csfd::Pose<double> np = csfd::compose(csfd::exp_map<double>(xi), cur);
  for (int e = 0; e < 9; ++e) pose12[e] = np.R.m[e];
  for (int e = 0; e < 3; ++e) pose12[9 + e] = np.t.v[e];
}

}  // namespace

static int track_frame_impl(csf_volume v, const double* depth, int w, int h, const double* init_pose,
                            const csf_intrinsics* k, const csf_icp_cfg* cfg_in, double* out_pose,
                            csf_track_result* result, double* trace, int trace_cap, int* n_trace);

extern "C" int csf_track_frame(csf_volume v, const double* depth, int w, int h, const double* init_pose,
                               const csf_intrinsics* k, const csf_icp_cfg* cfg_in, double* out_pose,
                               csf_track_result* result) {
  return track_frame_impl(v, depth, w, h, init_pose, k, cfg_in, out_pose, result, nullptr, 0, nullptr);
}

extern "C" int csf_track_frame_traced(csf_volume v, const double* depth, int w, int h, const double* init_pose,
                                      const csf_intrinsics* k, const csf_icp_cfg* cfg_in, double* out_pose,
                                      csf_track_result* result, double* trace, int trace_cap, int* n_trace) {
  if (!trace || !n_trace || trace_cap < 0) return CSF_EINVAL;
  return track_frame_impl(v, depth, w, h, init_pose, k, cfg_in, out_pose, result, trace, trace_cap, n_trace);
}

static int track_frame_impl(csf_volume v, const double* depth, int w, int h, const double* init_pose,
                            const csf_intrinsics* k, const csf_icp_cfg* cfg_in, double* out_pose,
                            csf_track_result* result, double* trace, int trace_cap, int* n_trace) {
  if (!v || !depth || !init_pose || !k || !out_pose) return CSF_EINVAL;
  csf_ctx ctx = v->ctx;
  csf_icp_cfg cfg;
  if (cfg_in)
    cfg = *cfg_in;
  else
    csf_default_icp_cfg(&cfg);
  if (cfg.solver < CSF_SOLVER_LINEARIZED || cfg.solver > CSF_SOLVER_CONJUGATE_GRADIENT)
    return fail(ctx, CSF_EINVAL, "csf_track_frame: unknown solver");
  if (cfg.solver != CSF_SOLVER_LINEARIZED && (!(cfg.h > 0.0) || cfg.h > 1e-6))
    return fail(ctx, CSF_EINVAL, "StepSize: step must satisfy 0 < h <= 1e-6");
  if (w <= 0 || h <= 0) return fail(ctx, CSF_EINVAL, "csf_track_frame: empty frame");
  if (!icp_frame_fits(w, h, 1)) return fail(ctx, CSF_EINVAL, "csf_track_frame: frame too large for the ICP reduction");
  cudaSetDevice(ctx->device);
  const int levels = std::clamp(cfg.levels, 1, 3);
  const size_t P = static_cast<size_t>(w) * h;
  DevBuf<double> dd, raw, pyr0, pyr1, pyr2, vre, nre, pose, pred, intr, partials;
  DevBuf<int> counts;
  DevBuf<TrackState> st;
  DevBuf<double2> hits;
  CUDA_TRY(ctx, hits.alloc(2 * P));
  CUDA_TRY(ctx, dd.alloc(P));
  CUDA_TRY(ctx, raw.alloc(P));
  CUDA_TRY(ctx, pyr0.alloc(P));
  CUDA_TRY(ctx, pyr1.alloc(P / 4 + 1));
  CUDA_TRY(ctx, pyr2.alloc(P / 16 + 1));
  CUDA_TRY(ctx, vre.alloc(P * 3));
  CUDA_TRY(ctx, nre.alloc(P * 3));
  CUDA_TRY(ctx, pose.alloc(12));
  CUDA_TRY(ctx, pred.alloc(12));
  CUDA_TRY(ctx, intr.alloc(12));
  CUDA_TRY(ctx, partials.alloc(icp_partials_doubles(1)));
  CUDA_TRY(ctx, counts.alloc(icp_counts_ints()));
  CUDA_TRY(ctx, st.alloc(1));
  CUDA_TRY(ctx, cudaMemsetAsync(counts.p, 0, sizeof(int) * counts.n, ctx->stream));
  double kl[12];
  for (int l = 0; l < 3; ++l) {
    const double sc = static_cast<double>(1 << l);
    kl[4 * l] = k->fx / sc;
    kl[4 * l + 1] = k->fy / sc;
    kl[4 * l + 2] = k->cx / sc;
    kl[4 * l + 3] = k->cy / sc;
  }
  const Launch L = launch_of(ctx);
  double hpose[12];
  std::copy(init_pose, init_pose + 12, hpose);
  CUDA_TRY(ctx, cudaMemcpyAsync(dd.p, depth, sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(pose.p, hpose, sizeof(double) * 12, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(intr.p, kl, sizeof(kl), cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemsetAsync(st.p, 0, sizeof(TrackState), ctx->stream));
  const double cos_max = csf_det::cos(cfg.theta_max_deg * M_PI / 180.0);
  launch_bilateral(L, nullptr, dd.p, raw.p, pyr0.p, w, h, 4.5, 0.03, 3);
  if (levels > 1) launch_downsample(L, pyr0.p, pyr1.p, w, h, 0.03);
  if (levels > 2) launch_downsample(L, pyr1.p, pyr2.p, w / 2, h / 2, 0.03);
  double* pyr[3] = {pyr0.p, pyr1.p, pyr2.p};
  // The volume's real channel only: a G = 0 view over its voxel store.
  csf_volume_s real_view;
  real_view.ctx = ctx;
  real_view.hashed = v->hashed;
  real_view.D = 0;
  real_view.G = 0;
  real_view.Dp = 0;  // pose/intrinsics buffers carry the real channel only
  real_view.dense = v->dense;
  real_view.hash = v->hash;
  real_view.dense.order = real_view.hash.order = 1;
  csf_raycast_cfg rcfg;
  csf_default_raycast_cfg(&rcfg);
  const LineSearch ls;
  if (n_trace) *n_trace = 0;
  Stepper stepper{cfg.solver == CSF_SOLVER_CONJUGATE_GRADIENT, cfg.ncg_restart};
  double lambda = cfg.levenberg_lambda0;
  int iteration = 0, n_corr = 0;
  bool converged = false;
  double final_loss = 0.0;
  EnergyScratch& ws = ctx->energy;
  int err = 0;
  // icp_energy(corrs, d, pose) of the current correspondence list
  auto energy_at = [&](const Vec6h& d, int n, const double* base, int* e) -> double {
    double E = 0.0;
    const int r = icp_energy_derivs(ctx->stream, ws, ws.corrs, n, base, d.data(), 1e-8, 0, &E, nullptr, nullptr);
    if (r) *e = r;
    return E;
  };
  for (int li = 0; li < levels; ++li) {
    const int level = levels - 1 - li;
    const int wl = w >> level, hl = h >> level;
    const double* kdev = intr.p + 4 * level;
    // one model prediction per level, cast at the estimate entering it (icp.cpp:189-192)
    CUDA_TRY(ctx, cudaMemcpyAsync(pose.p, hpose, sizeof(double) * 12, cudaMemcpyHostToDevice, ctx->stream));
    launch_level_begin(L, st.p, pose.p, pred.p, 0);
    raycast_dev(&real_view, pred.p, kdev, wl, hl, rcfg, hits.p, vre.p, nre.p, nullptr, nullptr);
    stepper.reset();
    const int stride = std::max(1, cfg.level_pixel_stride[li]);
    for (int it = 0; it < cfg.level_iterations[li]; ++it) {
      int n = 0;
      CUDA_TRY(ctx, cudaMemcpyAsync(pose.p, hpose, sizeof(double) * 12, cudaMemcpyHostToDevice, ctx->stream));
      const double* pred_w2c = reinterpret_cast<const double*>(reinterpret_cast<const char*>(st.p) +
                                                                   offsetof(TrackState, pred_w2c));
      err = associate_list(ctx->stream, ws, pyr[level], wl, hl, stride, kdev, pose.p, pred_w2c, vre.p, nre.p,
                           cfg.d_max, cos_max, &n);
      if (err) break;
      n_corr = n;
      if (n < 12) break;  // icp.cpp:199
      Vec6h delta{}, grad_it{};
      double loss_after = 0.0;
      if (cfg.solver == CSF_SOLVER_LINEARIZED) {
        // canonical slot-tiled normal equations + the real LDLT step on the
        // device (the pipeline's kernels); loss_after = E(delta) (icp.cpp:36-47)
        launch_icp_level(L, 0, st.p, pyr[level], wl, hl, stride, kdev, pose.p, vre.p, nre.p, nullptr, nullptr,
                         cfg.d_max, cos_max, 1, level, cfg.step_tolerance, partials.p, counts.p);
        TrackState hs;
        CUDA_TRY(ctx, d2h(&hs, st.p, sizeof(TrackState), ctx->stream));
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        for (int i = 0; i < 6; ++i) {
          delta[i] = hs.delta[i];
          grad_it[i] = 2.0 * hs.b[i];  // s.gradient = 2 b (icp.cpp:41)
        }
        loss_after = energy_at(delta, n, hpose, &err);
      } else {
        double E0 = 0.0, g[6], H[36];
        const int order = cfg.solver == CSF_SOLVER_NEWTON ? 2 : 1;
        const double zero[6] = {0, 0, 0, 0, 0, 0};
        err = icp_energy_derivs(ctx->stream, ws, ws.corrs, n, hpose, zero, cfg.h, order, &E0, g,
                                order == 2 ? H : nullptr);
        if (err) break;
        Vec6h grad;
        for (int i = 0; i < 6; ++i) grad[i] = g[i];
        grad_it = grad;
        loss_after = E0;
        if (cfg.solver == CSF_SOLVER_NEWTON) {
          // levenberg_newton_step (descent.hpp:109-144)
          bool done = false;
          for (int attempt = 0; attempt < 8 && !done && !err; ++attempt) {
            double a[21];
            for (int r = 0; r < 6; ++r)
              for (int c = 0; c <= r; ++c) a[csfd::tri(r, c)] = H[r * 6 + c] + lambda * (r == c ? 1.0 : 0.0);
            double m[6][6];
            int tr[6];
            const bool ok = csfd::ldlt6_factor_reg<double>(a, m, tr);
            if (ok) {
              double ng[6], d[6];
              for (int i = 0; i < 6; ++i) ng[i] = -grad[i];
              csfd::ldlt6_apply_reg<double>(m, tr, ng, d);
              bool finite = true;
              for (int i = 0; i < 6; ++i) finite = finite && std::isfinite(d[i]);
              if (finite) {
                Vec6h dv;
                for (int i = 0; i < 6; ++i) dv[i] = d[i];
                const double trial = energy_at(dv, n, hpose, &err);
                if (!err && trial < E0) {
                  lambda = std::max(lambda * 0.1, 1e-12);
                  loss_after = trial;
                  delta = dv;
                  done = true;
                  break;
                }
              }
            }
            lambda *= 10.0;
          }
          if (!done && !err) {
            const double slope = -dot6h(grad, grad);
            double alpha = 0.0, lsl = 0.0;
            if (slope < 0.0 &&
                backtracking(
                    [&](double al, int* e) {
                      Vec6h dv;
                      for (int i = 0; i < 6; ++i) dv[i] = -al * grad[i];
                      return energy_at(dv, n, hpose, e);
                    },
                    E0, slope, ls, &alpha, &lsl, &err)) {
              loss_after = lsl;
              for (int i = 0; i < 6; ++i) delta[i] = -alpha * grad[i];
            } else {
              loss_after = E0;
              delta = Vec6h{};
            }
          }
        } else {
          // first_order_outcome (icp.cpp:64-85)
          const Vec6h dir = stepper.propose(grad);
          const double slope = dot6h(grad, dir);
          if (slope < 0.0) {
            double alpha = 0.0, lsl = 0.0;
            if (backtracking(
                    [&](double al, int* e) {
                      Vec6h dv;
                      for (int i = 0; i < 6; ++i) dv[i] = al * dir[i];
                      return energy_at(dv, n, hpose, e);
                    },
                    E0, slope, ls, &alpha, &lsl, &err)) {
              for (int i = 0; i < 6; ++i) delta[i] = alpha * dir[i];
              loss_after = lsl;
            }
          }
        }
      }
      if (err) break;
      apply_increment_h(delta, hpose);
      ++iteration;
      final_loss = loss_after / static_cast<double>(n);
      if (trace) {  // TraceRow (icp.hpp:103-109): iteration, loss, gradient norm, then the pose
        if (*n_trace < trace_cap) {
          double* row = trace + 15 * static_cast<size_t>(*n_trace);
          row[0] = iteration;
          row[1] = final_loss;
          row[2] = norm6h(grad_it);
          std::copy(hpose, hpose + 12, row + 3);
        }
        ++*n_trace;
      }
      if (norm6h(delta) < cfg.step_tolerance) {
        if (level == 0) converged = true;
        break;
      }
    }
    if (err) break;
  }
  if (err == 5) return fail(ctx, CSF_ENOMEM, "csf_track_frame: out of device memory");
  if (err) return fail(ctx, CSF_ECUDA, "csf_track_frame: CUDA error");
  const int rc = sync_check(ctx, "csf_track_frame");
  if (rc) return rc;
  std::copy(hpose, hpose + 12, out_pose);
  if (result) {
    result->iterations = iteration;
    result->converged = converged;
    result->correspondences = n_corr;
    result->final_loss = final_loss;
  }
  return CSF_OK;
}

// Debug hook (not part of the public header): table-march statistics
// (counted only in a -DCSF_MARCH_STATS build; tools/march_stats.py).
namespace csfi { void march_stats_enable(unsigned long long* buf); }
extern "C" int csf_debug_march_stats(unsigned long long* host_out /*[8]*/, int enable) {
  static unsigned long long* dbuf = nullptr;
  if (enable) {
    if (!dbuf && cudaMalloc(&dbuf, 8 * sizeof(unsigned long long)) != cudaSuccess) return CSF_ENOMEM;
    cudaMemset(dbuf, 0, 8 * sizeof(unsigned long long));
    march_stats_enable(dbuf);
    return CSF_OK;
  }
  march_stats_enable(nullptr);
  if (dbuf && host_out) cudaMemcpy(host_out, dbuf, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return CSF_OK;
}

// Debug hook (not part of the public header): the ICP level kernel's
// per-CTA phase timeline (64 launches x 256 CTAs x 32 iterations x 16 phases).
namespace csfi { void icp_clock_enable(unsigned long long* buf); }
extern "C" int csf_debug_icp_clock(unsigned long long* host_out, int enable) {
  static unsigned long long* dbuf = nullptr;
  const size_t n = size_t(64) * 256 * 32 * 16;
  if (enable) {
    if (!dbuf && cudaMalloc(&dbuf, n * sizeof(unsigned long long)) != cudaSuccess) return CSF_ENOMEM;
    cudaMemset(dbuf, 0, n * sizeof(unsigned long long));
    icp_clock_enable(dbuf);
    return CSF_OK;
  }
  icp_clock_enable(nullptr);
  if (dbuf && host_out) cudaMemcpy(host_out, dbuf, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return CSF_OK;
}

extern "C" int csf_synth_workload(csf_ctx ctx, int config, int n_frames, int width, int height, float* depth,
                                  double* gt, csf_intrinsics* k) {
  if (!ctx || !depth || !gt || n_frames <= 0) return CSF_EINVAL;
  cudaSetDevice(ctx->device);
  std::string err;
  const int rc = synth_workload(ctx->stream, config, n_frames, width, height, depth, gt, k, &err);
  ctx->launches += 1;
  if (rc) return fail(ctx, rc, err);
  return CSF_OK;
}

// ---------------------------------------------------------------------------
// relocalization (reloc.hpp)
// ---------------------------------------------------------------------------
struct csf_reloc_s {
  csf_ctx ctx = nullptr;
  int n = 0, w = 0, h = 0;
  double mu = 0.1;
  DevBuf<double> centers, values, depth, k4;
  ~csf_reloc_s() {
    centers.release();
    values.release();
    depth.release();
    k4.release();
  }
};

extern "C" void csf_default_reloc_cfg(csf_reloc_cfg* c) {
  if (!c) return;
  c->switch_relative = 0.5;  // reloc.hpp:86-90
  c->switch_absolute = -1.0;
  c->max_iterations = 50;
  c->step_tolerance = 1e-6;
  c->ls_initial_step = 1.0;  // descent.hpp:16-21
  c->ls_shrink = 0.5;
  c->ls_sufficient_decrease = 1e-4;
  c->ls_max_backtracks = 25;
  c->h = 1e-8;  // csfd.hpp:16
  c->max_step = 0.05;  // builder-defined safeguards
  c->min_overlap_ratio = 0.9;
}

extern "C" int csf_reloc_create(csf_volume v, const double* depth, int w, int h, const csf_intrinsics* k,
                                csf_reloc* out) {
  if (!v || !depth || !k || !out || w <= 0 || h <= 0) return CSF_EINVAL;
  csf_ctx ctx = v->ctx;
  cudaSetDevice(ctx->device);
  const long long nv = volume_voxels_now(v);
  const double2* rw = v->hashed ? v->hash.rw : v->dense.rw;
  const int* coords = v->hashed ? v->hash.coords : nullptr;
  const double vs = v->hashed ? v->hash.vs : v->dense.vs;
  const double origin[3] = {v->hashed ? v->hash.ox : v->dense.ox, v->hashed ? v->hash.oy : v->dense.oy,
                            v->hashed ? v->hash.oz : v->dense.oz};
  int n = 0;
  int rc = reloc_flatten(ctx->stream, rw, nv, coords, v->dense.nx, v->dense.ny, vs, origin, nullptr, nullptr, &n);
  if (rc == 1) return fail(ctx, CSF_EINVAL, "RelocProblem: volume too large to flatten");
  if (rc) return fail(ctx, rc == 5 ? CSF_ENOMEM : CSF_ECUDA, "RelocProblem: flatten failed");
  if (n == 0) return fail(ctx, CSF_EINVAL, "RelocProblem: reference has no observed voxels");
  auto r = std::make_unique<csf_reloc_s>();
  r->ctx = ctx;
  r->w = w;
  r->h = h;
  r->mu = v->hashed ? v->hash.mu : v->dense.mu;
  CUDA_TRY(ctx, r->centers.alloc(3 * static_cast<size_t>(n)));
  CUDA_TRY(ctx, r->values.alloc(n));
  CUDA_TRY(ctx, r->depth.alloc(static_cast<size_t>(w) * h));
  CUDA_TRY(ctx, r->k4.alloc(4));
  int n2 = 0;
  rc = reloc_flatten(ctx->stream, rw, nv, coords, v->dense.nx, v->dense.ny, vs, origin, r->centers.p, r->values.p,
                     &n2);
  if (rc || n2 != n) return fail(ctx, rc == 5 ? CSF_ENOMEM : CSF_ECUDA, "RelocProblem: flatten failed");
  r->n = n;
  const double kk[4] = {k->fx, k->fy, k->cx, k->cy};
  CUDA_TRY(ctx, cudaMemcpyAsync(r->depth.p, depth, sizeof(double) * w * h, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(r->k4.p, kk, sizeof(kk), cudaMemcpyHostToDevice, ctx->stream));
  ctx->launches += 3;
  *out = r.release();
  return CSF_OK;
}

extern "C" int csf_reloc_destroy(csf_reloc r) {
  if (!r) return CSF_EINVAL;
  cudaSetDevice(r->ctx->device);
  delete r;
  return CSF_OK;
}

extern "C" int csf_reloc_info(csf_reloc r, int* n, double* mu, double* centers, double* values) {
  if (!r) return CSF_EINVAL;
  cudaSetDevice(r->ctx->device);
  if (n) *n = r->n;
  if (mu) *mu = r->mu;
  if (centers) CUDA_TRY(r->ctx, d2h(centers, r->centers.p, sizeof(double) * 3 * r->n, r->ctx->stream));
  if (values) CUDA_TRY(r->ctx, d2h(values, r->values.p, sizeof(double) * r->n, r->ctx->stream));
  return CSF_OK;
}

// 0 ok; CSF_* on failure.  no_overlap -> ERUNTIME (reloc.hpp:65-66).
static int reloc_eval(csf_reloc r, const double* pose, int order, double h, double* E, double* g, double* H,
                      long long* overlap) {
  csf_ctx ctx = r->ctx;
  long long ov = 0;
  ProfScope ps(ctx, order == 0 ? kPRelocLoss : order == 1 ? kPRelocGrad : kPRelocHess);
  const int rc = reloc_energy_derivs(ctx->stream, ctx->energy, r->centers.p, r->values.p, r->n, r->depth.p, r->w,
                                     r->h, r->k4.p, r->mu, pose, order, h, E, g, H, &ov);
  ctx->launches += 4;  // pose, terms, tree sub, tree top
  if (rc == 5) return fail(ctx, CSF_ENOMEM, "reloc_energy: out of device memory");
  if (rc) return fail(ctx, CSF_ECUDA, "reloc_energy: CUDA error");
  if (overlap) *overlap = ov;
  if (ov == 0) return fail(ctx, CSF_ERUNTIME, "relocalization energy: no overlapping voxels");
  return CSF_OK;
}

extern "C" int csf_reloc_energy(csf_reloc r, const double* pose, int order, double h, double* E, double* g, double* H,
                                long long* overlap) {
  if (!r || !pose || !E || order < 0 || order > 2 || (order >= 1 && !g) || (order == 2 && !H)) return CSF_EINVAL;
  if (order > 0 && (!(h > 0.0) || h > 1e-6)) return fail(r->ctx, CSF_EINVAL, "StepSize: step must satisfy 0 < h <= 1e-6");
  cudaSetDevice(r->ctx->device);
  return reloc_eval(r, pose, order, h, E, g, H, overlap);
}

// relocalize (reloc.hpp:116-124; builder-defined body, DESIGN.md §3.9 and
// oracle/orc_reloc.hpp): per-voxel work on the device, 6-vector logic here.
extern "C" int csf_relocalize(csf_reloc r, const double* init, int method, const csf_reloc_cfg* cfg_in,
                              double* out_pose, csf_reloc_result* res, double* losses, double* gnorms) {
  if (!r || !init || !out_pose) return CSF_EINVAL;
  if (method != CSF_RELOC_GRADIENT_DESCENT && method != CSF_RELOC_NEWTON)
    return fail(r->ctx, CSF_EINVAL, "relocalize: unknown method");
  csf_reloc_cfg cfg;
  if (cfg_in)
    cfg = *cfg_in;
  else
    csf_default_reloc_cfg(&cfg);
  if (!(cfg.h > 0.0) || cfg.h > 1e-6) return fail(r->ctx, CSF_EINVAL, "StepSize: step must satisfy 0 < h <= 1e-6");
  cudaSetDevice(r->ctx->device);
  double pose[12];
  std::copy(init, init + 12, pose);
  double loss = 0.0;
  long long cur_ov = 0, trial_ov = 0;
  int rc = reloc_eval(r, pose, 0, cfg.h, &loss, nullptr, nullptr, &cur_ov);
  if (rc) return rc;
  const double threshold = cfg.switch_absolute >= 0.0 ? cfg.switch_absolute : cfg.switch_relative * loss;
  LineSearch ls;
  ls.initial_step = cfg.ls_initial_step;
  ls.shrink = cfg.ls_shrink;
  ls.sufficient_decrease = cfg.ls_sufficient_decrease;
  ls.max_backtracks = cfg.ls_max_backtracks;
  int iterations = 0;
  bool converged = false;
  // a trial pose with no overlapping voxel, or keeping fewer than
  // min_overlap_ratio x the current overlap, counts as +inf
  auto trial_loss = [&](const Vec6h& d, int* err) -> double {
    double p[12];
    std::copy(pose, pose + 12, p);
    apply_increment_h(d, p);
    double E = 0.0;
    long long ov = 0;
    ProfScope ps(r->ctx, kPRelocLoss);
    const int e = reloc_energy_derivs(r->ctx->stream, r->ctx->energy, r->centers.p, r->values.p, r->n, r->depth.p,
                                      r->w, r->h, r->k4.p, r->mu, p, 0, cfg.h, &E, nullptr, nullptr, &ov);
    r->ctx->launches += 4;
    if (e) {
      *err = e;
      return 0.0;
    }
    if (ov == 0) return std::numeric_limits<double>::infinity();
    trial_ov = ov;
    if (static_cast<double>(ov) < cfg.min_overlap_ratio * static_cast<double>(cur_ov))
      return std::numeric_limits<double>::infinity();
    return E;
  };
  int err = 0;
  for (int it = 0; it < cfg.max_iterations; ++it) {
    double gg[6], H[36];
    const bool newton = method == CSF_RELOC_NEWTON && loss < threshold;
    double e_lifted = 0.0;  // the real channel of the lifted pass == loss
    rc = reloc_eval(r, pose, newton ? 2 : 1, cfg.h, &e_lifted, gg, H, nullptr);
    if (rc) return rc;
    Vec6h g, dir;
    for (int i = 0; i < 6; ++i) g[i] = gg[i];
    const double gn = norm6h(g);
    const double sg = gn > 0.0 ? cfg.max_step / gn : 0.0;
    for (int i = 0; i < 6; ++i) dir[i] = -g[i] * sg;
    if (newton) {
      double a[21];
      for (int rr = 0; rr < 6; ++rr)
        for (int c = 0; c <= rr; ++c) a[csfd::tri(rr, c)] = H[rr * 6 + c];
      double m[6][6];
      int tr[6];
      if (csfd::ldlt6_factor_reg<double>(a, m, tr)) {
        double ng[6], d[6];
        for (int i = 0; i < 6; ++i) ng[i] = -g[i];
        csfd::ldlt6_apply_reg<double>(m, tr, ng, d);
        bool finite = true;
        Vec6h nd;
        for (int i = 0; i < 6; ++i) {
          finite = finite && std::isfinite(d[i]);
          nd[i] = d[i];
        }
        if (finite && dot6h(g, nd) < 0.0) {
          const double nn = norm6h(nd);
          if (nn > cfg.max_step) {
            const double sn = cfg.max_step / nn;
            for (int i = 0; i < 6; ++i) nd[i] = nd[i] * sn;
          }
          dir = nd;
        }
      }
    }
    const double slope = dot6h(g, dir);
    if (!(slope < 0.0)) {
      converged = gn == 0.0;
      break;
    }
    double alpha = 0.0, lsl = 0.0;
    const bool ok = backtracking(
        [&](double al, int* e) {
          Vec6h d;
          for (int i = 0; i < 6; ++i) d[i] = al * dir[i];
          return trial_loss(d, e);
        },
        loss, slope, ls, &alpha, &lsl, &err);
    if (err) break;
    if (!ok) break;
    Vec6h step;
    for (int i = 0; i < 6; ++i) step[i] = alpha * dir[i];
    apply_increment_h(step, pose);
    loss = lsl;
    cur_ov = trial_ov;
    if (losses) losses[iterations] = loss;
    if (gnorms) gnorms[iterations] = gn;
    ++iterations;
    if (norm6h(step) < cfg.step_tolerance) {
      converged = true;
      break;
    }
  }
  if (err == 5) return fail(r->ctx, CSF_ENOMEM, "relocalize: out of device memory");
  if (err) return fail(r->ctx, CSF_ECUDA, "relocalize: CUDA error");
  std::copy(pose, pose + 12, out_pose);
  if (res) {
    res->iterations = iterations;
    res->converged = converged;
    res->final_loss = loss;
  }
  return CSF_OK;
}

extern "C" int csf_depth_cloud(csf_ctx ctx, const double* depth, int w, int h, const csf_intrinsics* k,
                               const double* c2w, int stride, double* points, int* n_points) {
  if (!ctx || !depth || !k || !c2w || !n_points || w <= 0 || h <= 0) return CSF_EINVAL;
  if (stride < 1) return fail(ctx, CSF_EINVAL, "depth_cloud: stride must be >= 1");
  cudaSetDevice(ctx->device);
  const double kk[4] = {k->fx, k->fy, k->cx, k->cy};
  const int rc = depth_cloud_dev(ctx->stream, depth, w, h, kk, c2w, stride, points, n_points);
  ctx->launches += 3;
  if (rc == 5) return fail(ctx, CSF_ENOMEM, "depth_cloud: out of device memory");
  if (rc) return fail(ctx, CSF_ECUDA, "depth_cloud: CUDA error");
  return CSF_OK;
}

extern "C" int csf_eval_nn_error(csf_ctx ctx, const double* T, const double* q, int nq, const double* ref, int nr,
                                 double* mean, int32_t* outlier) {
  if (!ctx || !T || !mean || nq < 0 || nr < 0) return CSF_EINVAL;
  if (nq == 0 || nr == 0 || !q || !ref) return fail(ctx, CSF_EINVAL, "eval_nn_error: empty cloud");
  cudaSetDevice(ctx->device);
  const int rc = nn_error_dev(ctx->stream, ctx->energy, T, q, nq, ref, nr, mean);
  ctx->launches += 3;
  if (rc == 5) return fail(ctx, CSF_ENOMEM, "eval_nn_error: out of device memory");
  if (rc) return fail(ctx, CSF_ECUDA, "eval_nn_error: CUDA error");
  if (outlier) *outlier = *mean > 0.1;
  return CSF_OK;
}

// ---------------------------------------------------------------------------
// surfel (X-EF) front end (surfel.hpp)
// ---------------------------------------------------------------------------
struct csf_surfels_s {
  csf_ctx ctx = nullptr;
  int D = 0, n = 0, cap = 0;
  DevBuf<double> pos, nrm, conf, rad;
  DevBuf<int> ts;
  DevBuf<double> in;  // depth [P][C] + pose [12][C] + intrinsics [4][C]
  DevBuf<double> in_real;  // real depth [P] (csf_update_surfels_real)
  SurfelScratch ws;
  ~csf_surfels_s() {
    pos.release();
    nrm.release();
    conf.release();
    rad.release();
    ts.release();
    in.release();
    in_real.release();
    surfel_scratch_release(ws);
  }
  SurfelArrays arrays() { return SurfelArrays{pos.p, nrm.p, conf.p, rad.p, ts.p}; }
};

extern "C" void csf_default_surfel_cfg(csf_surfel_cfg* c) {
  if (!c) return;
  c->depth = 0.05;  // surfel.hpp:55-60
  c->normal_deg = 30.0;
  c->distance = 0.05;
  c->sigma = 0.025;
  c->one_to_many = 1;  // surfel.hpp:84-91
}

// grow the map's capacity to >= need, keeping the first n surfels
static int surfels_reserve(csf_surfels m, int need) {
  if (need <= m->cap && m->pos.p) return CSF_OK;
  const int C = 1 + m->D;
  const int cap = std::max({need, 2 * m->cap, 1024});
  DevBuf<double> pos, nrm, conf, rad;
  DevBuf<int> ts;
  CUDA_TRY(m->ctx, pos.alloc(3 * static_cast<size_t>(cap) * C));
  CUDA_TRY(m->ctx, nrm.alloc(3 * static_cast<size_t>(cap) * C));
  CUDA_TRY(m->ctx, conf.alloc(static_cast<size_t>(cap) * C));
  CUDA_TRY(m->ctx, rad.alloc(cap));
  CUDA_TRY(m->ctx, ts.alloc(cap));
  if (m->n > 0) {
    const cudaStream_t s = m->ctx->stream;
    CUDA_TRY(m->ctx, cudaMemcpyAsync(pos.p, m->pos.p, sizeof(double) * 3 * m->n * C, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(m->ctx, cudaMemcpyAsync(nrm.p, m->nrm.p, sizeof(double) * 3 * m->n * C, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(m->ctx, cudaMemcpyAsync(conf.p, m->conf.p, sizeof(double) * m->n * C, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(m->ctx, cudaMemcpyAsync(rad.p, m->rad.p, sizeof(double) * m->n, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(m->ctx, cudaMemcpyAsync(ts.p, m->ts.p, sizeof(int) * m->n, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(m->ctx, cudaStreamSynchronize(s));
  }
  std::swap(m->pos, pos);
  std::swap(m->nrm, nrm);
  std::swap(m->conf, conf);
  std::swap(m->rad, rad);
  std::swap(m->ts, ts);
  pos.release();
  nrm.release();
  conf.release();
  rad.release();
  ts.release();
  m->cap = cap;
  return CSF_OK;
}

extern "C" int csf_surfels_create(csf_ctx ctx, int n_channels, csf_surfels* out) {
  if (!ctx || !out || n_channels < 0 || n_channels > CSF_MAX_DIRECTIONS) return CSF_EINVAL;
  cudaSetDevice(ctx->device);
  auto m = std::make_unique<csf_surfels_s>();
  m->ctx = ctx;
  m->D = n_channels;
  const int rc = surfels_reserve(m.get(), 1024);
  if (rc) return rc;
  *out = m.release();
  return CSF_OK;
}
extern "C" int csf_surfels_destroy(csf_surfels m) {
  if (!m) return CSF_EINVAL;
  cudaSetDevice(m->ctx->device);
  delete m;
  return CSF_OK;
}
extern "C" int csf_surfels_clear(csf_surfels m) {
  if (!m) return CSF_EINVAL;
  m->n = 0;  // capacity and scratch are kept (a new map without re-allocation)
  return CSF_OK;
}
extern "C" int csf_surfels_count(csf_surfels m, int* n) {
  if (!m || !n) return CSF_EINVAL;
  *n = m->n;
  return CSF_OK;
}
extern "C" int csf_surfels_download(csf_surfels m, double* pos, double* nrm, double* rad, double* conf, int32_t* ts) {
  if (!m) return CSF_EINVAL;
  csf_ctx ctx = m->ctx;
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  const size_t C = 1 + m->D, n = m->n;
  if (n == 0) return CSF_OK;
  if (pos) CUDA_TRY(ctx, d2h(pos, m->pos.p, sizeof(double) * 3 * n * C, ctx->stream));
  if (nrm) CUDA_TRY(ctx, d2h(nrm, m->nrm.p, sizeof(double) * 3 * n * C, ctx->stream));
  if (rad) CUDA_TRY(ctx, d2h(rad, m->rad.p, sizeof(double) * n, ctx->stream));
  if (conf) CUDA_TRY(ctx, d2h(conf, m->conf.p, sizeof(double) * n * C, ctx->stream));
  if (ts) CUDA_TRY(ctx, d2h(ts, m->ts.p, sizeof(int) * n, ctx->stream));
  return CSF_OK;
}
extern "C" int csf_surfels_upload(csf_surfels m, int n, const double* pos, const double* nrm, const double* rad,
                                  const double* conf, const int32_t* ts) {
  if (!m || n < 0 || (n > 0 && (!pos || !nrm || !rad || !conf || !ts))) return CSF_EINVAL;
  csf_ctx ctx = m->ctx;
  cudaSetDevice(ctx->device);
  m->n = 0;
  const int rc = surfels_reserve(m, n);
  if (rc) return rc;
  const size_t C = 1 + m->D;
  if (n > 0) {
    CUDA_TRY(ctx, cudaMemcpyAsync(m->pos.p, pos, sizeof(double) * 3 * n * C, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(m->nrm.p, nrm, sizeof(double) * 3 * n * C, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(m->rad.p, rad, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(m->conf.p, conf, sizeof(double) * n * C, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(m->ts.p, ts, sizeof(int) * n, cudaMemcpyHostToDevice, ctx->stream));
  }
  m->n = n;
  return CSF_OK;
}

static void k4_of(const csf_intrinsics* k, double* k4) {
  k4[0] = k->fx;
  k4[1] = k->fy;
  k4[2] = k->cx;
  k4[3] = k->cy;
}

extern "C" int csf_render_index_map(csf_surfels m, const double* c2w, const csf_intrinsics* k, uint32_t* offsets,
                                    int32_t* entries, int* n_entries) {
  if (!m || !c2w || !k || !offsets || !n_entries || k->width <= 0 || k->height <= 0) return CSF_EINVAL;
  csf_ctx ctx = m->ctx;
  cudaSetDevice(ctx->device);
  double k4[4];
  k4_of(k, k4);
  int cnt = 0;
  const int rc = surfel_index_map(ctx->stream, m->ws, m->pos.p, m->n, m->D, c2w, k4, k->width, k->height, &cnt);
  ctx->launches += 4;
  if (rc) return fail(ctx, rc == 5 ? CSF_ENOMEM : CSF_ECUDA, "render_index_map: CUDA error");
  const size_t cells = static_cast<size_t>(16) * k->width * k->height;
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  CUDA_TRY(ctx, d2h(offsets, m->ws.offsets, sizeof(uint32_t) * (cells + 1), ctx->stream));
  if (entries && cnt > 0)
    CUDA_TRY(ctx, d2h(entries, m->ws.entries, sizeof(int32_t) * cnt, ctx->stream));
  *n_entries = cnt;
  return CSF_OK;
}

// upload depth / pose / intrinsics and run index map + association
static int surfels_assoc_common(csf_surfels m, const double* depth, int w, int h, const double* c2w,
                                const csf_intrinsics* k, const csf_surfel_cfg* cfg_in, int* total, int* merged,
                                double* c2w12, double* k4, bool real_depth = false) {
  csf_ctx ctx = m->ctx;
  const int C = 1 + m->D;
  const size_t P = static_cast<size_t>(w) * h;
  csf_surfel_cfg cfg;
  if (cfg_in)
    cfg = *cfg_in;
  else
    csf_default_surfel_cfg(&cfg);
  CUDA_TRY(ctx, m->in.alloc(P * C + 16 * C));
  double* d_depth = m->in.p;
  double* d_pose = d_depth + P * C;
  double* d_intr = d_pose + 12 * C;
  std::vector<double> intr(4 * C, 0.0);
  k4_of(k, k4);
  for (int e = 0; e < 4; ++e) intr[e * C] = k4[e];
  for (int e = 0; e < 12; ++e) c2w12[e] = c2w[e * C];
  if (real_depth) {  // unperturbed depth: upload [P] and lift on the device (1/(1+D) of the bytes)
    CUDA_TRY(ctx, m->in_real.alloc(P));
    CUDA_TRY(ctx, cudaMemcpyAsync(m->in_real.p, depth, sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream));
    launch_expand_depth(ctx->stream, m->in_real.p, static_cast<long long>(P), C, d_depth);
  } else {
    CUDA_TRY(ctx, cudaMemcpyAsync(d_depth, depth, sizeof(double) * P * C, cudaMemcpyHostToDevice, ctx->stream));
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(d_pose, c2w, sizeof(double) * 12 * C, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(d_intr, intr.data(), sizeof(double) * 4 * C, cudaMemcpyHostToDevice, ctx->stream));
  int cnt = 0;
  int rc = surfel_index_map(ctx->stream, m->ws, m->pos.p, m->n, m->D, c2w12, k4, w, h, &cnt);
  if (rc) return fail(ctx, rc == 5 ? CSF_ENOMEM : CSF_ECUDA, "surfels: index map failed");
  AssocParams ap;
  ap.depth = cfg.depth;
  ap.cos_gate = std::cos(cfg.normal_deg * M_PI / 180.0);
  ap.distance = cfg.distance;
  ap.kernel_scale = -1.0 / (2.0 * cfg.sigma * cfg.sigma);
  ap.one_to_many = cfg.one_to_many != 0;
  rc = surfel_associate(ctx->stream, m->ws, m->pos.p, m->nrm.p, m->D, d_depth, d_pose, d_intr, c2w12, k4, w, h, ap,
                        total, merged);
  ctx->launches += 12;
  if (rc) return fail(ctx, rc == 5 ? CSF_ENOMEM : CSF_ECUDA, "surfels: association failed");
  return CSF_OK;
}

extern "C" int csf_associate_surfels(csf_surfels m, const double* depth, int w, int h, const double* c2w,
                                     const csf_intrinsics* k, const csf_surfel_cfg* cfg, int32_t* counts,
                                     int32_t* indices, double* weights, int cap, int* total) {
  if (!m || !depth || !c2w || !k || !counts || !total || w <= 0 || h <= 0) return CSF_EINVAL;
  csf_ctx ctx = m->ctx;
  cudaSetDevice(ctx->device);
  int T = 0, merged = 0;
  double c2w12[12], k4[4];
  const int rc = surfels_assoc_common(m, depth, w, h, c2w, k, cfg, &T, &merged, c2w12, k4);
  if (rc) return rc;
  const size_t P = static_cast<size_t>(w) * h, C = 1 + m->D;
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  CUDA_TRY(ctx, d2h(counts, m->ws.pint + P, sizeof(int32_t) * P, ctx->stream));
  if (indices && weights && T > 0) {
    const int n = std::min(T, cap);
    CUDA_TRY(ctx, d2h(indices, m->ws.pidx, sizeof(int32_t) * n, ctx->stream));
    CUDA_TRY(ctx, d2h(weights, m->ws.pw, sizeof(double) * n * C, ctx->stream));
  }
  *total = T;
  return CSF_OK;
}

static int update_surfels_impl(csf_surfels m, const double* depth, int w, int h, const double* c2w,
                               const csf_intrinsics* k, int frame_index, const csf_surfel_cfg* cfg,
                               int* merged_pixels, int* created, bool real_depth);
extern "C" int csf_update_surfels(csf_surfels m, const double* depth, int w, int h, const double* c2w,
                                  const csf_intrinsics* k, int frame_index, const csf_surfel_cfg* cfg,
                                  int* merged_pixels, int* created) {
  return update_surfels_impl(m, depth, w, h, c2w, k, frame_index, cfg, merged_pixels, created, false);
}
extern "C" int csf_update_surfels_real(csf_surfels m, const double* depth, int w, int h, const double* c2w,
                                       const csf_intrinsics* k, int frame_index, const csf_surfel_cfg* cfg,
                                       int* merged_pixels, int* created) {
  return update_surfels_impl(m, depth, w, h, c2w, k, frame_index, cfg, merged_pixels, created, true);
}
static int update_surfels_impl(csf_surfels m, const double* depth, int w, int h, const double* c2w,
                               const csf_intrinsics* k, int frame_index, const csf_surfel_cfg* cfg,
                               int* merged_pixels, int* created, bool real_depth) {
  if (!m || !depth || !c2w || !k || w <= 0 || h <= 0) return CSF_EINVAL;
  csf_ctx ctx = m->ctx;
  cudaSetDevice(ctx->device);
  int T = 0, merged = 0, cr = 0;
  double c2w12[12], k4[4];
  int rc = surfels_assoc_common(m, depth, w, h, c2w, k, cfg, &T, &merged, c2w12, k4, real_depth);
  if (rc) return rc;
  if (surfel_created_count(ctx->stream, m->ws, w * h, &cr)) return fail(ctx, CSF_ECUDA, "update_surfels: CUDA error");
  rc = surfels_reserve(m, m->n + cr);
  if (rc) return rc;
  rc = surfel_commit(ctx->stream, m->ws, m->arrays(), m->n, m->D, T, c2w12, k4, w, h, frame_index,
                     std::sqrt(2.0) / k->fx);
  ctx->launches += 5;
  if (rc) return fail(ctx, rc == 5 ? CSF_ENOMEM : CSF_ECUDA, "update_surfels: commit failed");
  m->n += cr;
  rc = sync_check(ctx, "update_surfels");
  if (rc) return rc;
  if (merged_pixels) *merged_pixels = merged;
  if (created) *created = cr;
  return CSF_OK;
}

extern "C" int csf_predict_maps(csf_surfels m, const double* c2w, const csf_intrinsics* k, double* V, double* N) {
  if (!m || !c2w || !k || !V || !N || k->width <= 0 || k->height <= 0) return CSF_EINVAL;
  csf_ctx ctx = m->ctx;
  cudaSetDevice(ctx->device);
  const size_t P = static_cast<size_t>(k->width) * k->height;
  DevBuf<double> out;
  CUDA_TRY(ctx, out.alloc(6 * P));
  double k4[4];
  k4_of(k, k4);
  const int rc = surfel_predict(ctx->stream, m->ws, m->pos.p, m->nrm.p, m->n, m->D, c2w, k4, k->width, k->height,
                                out.p, out.p + 3 * P);
  ctx->launches += 5;
  if (rc) return fail(ctx, rc == 5 ? CSF_ENOMEM : CSF_ECUDA, "predict_maps: CUDA error");
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  CUDA_TRY(ctx, d2h(V, out.p, sizeof(double) * 3 * P, ctx->stream));
  CUDA_TRY(ctx, d2h(N, out.p + 3 * P, sizeof(double) * 3 * P, ctx->stream));
  return CSF_OK;
}

// surfel.cpp:110-119 (host copy of the device function; deterministic exp)
extern "C" double csf_sample_confidence(const csf_intrinsics* k, int x, int y) {
  const double dx = static_cast<double>(x) - k->cx;
  const double dy = static_cast<double>(y) - k->cy;
  const double half_diagonal =
      0.5 * std::sqrt(static_cast<double>(k->width) * k->width + static_cast<double>(k->height) * k->height);
  double g = std::sqrt(dx * dx + dy * dy) / half_diagonal;
  g = g < 0.0 ? 0.0 : (1.0 < g ? 1.0 : g);
  return csf_det::exp(-g * g / 0.72);
}

// ---- sticky launch-error record (csf_internal.h).  Per host thread: calls on
// one context are serialized by the caller and different contexts run on
// different host threads (csf_b200.h), so an error is reported by the call on
// the thread whose launch failed, never by another context's call.
namespace csfi {
static thread_local std::string t_launch_msg;
static thread_local bool t_launch_pending = false;
void note_error(const std::string& msg) {
  if (!t_launch_pending) t_launch_msg = msg;  // the first error wins
  t_launch_pending = true;
}
void note_launch_error(const char* what, cudaError_t e) {
  note_error(std::string("launch of ") + what + " failed: " + cudaGetErrorString(e));
}
bool take_launch_error(char* msg, size_t cap) {
  if (!t_launch_pending) return false;
  std::snprintf(msg, cap, "%s", t_launch_msg.c_str());
  t_launch_pending = false;
  return true;
}

// Function attributes and device properties are per device: cache them per
// (device, kernel) under a lock so concurrent contexts on several GPUs each
// get their own opt-in (csf_internal.h / lifted.cuh).
static std::mutex g_attr_mu;
static std::vector<std::pair<std::pair<int, const void*>, size_t>> g_smem_set;
void ensure_dyn_smem(const void* fn, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_attr_mu);
  for (auto& e : g_smem_set)
    if (e.first.first == dev && e.first.second == fn) {
      if (e.second >= bytes) return;
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)) ==
          cudaSuccess)
        e.second = bytes;
      return;
    }
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)) == cudaSuccess)
    g_smem_set.push_back({{dev, fn}, bytes});
}
int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n > 0) return n;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  cache[dev].store(n, std::memory_order_relaxed);
  return n;
}
}  // namespace csfi


// Internal interface between the C-ABI layer (capi.cu) and the kernel
// translation units.  Plain structs of device pointers; no torch types.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace csfi {

// Channel-group widths with instantiated kernels.  A run with D directions
// uses the group width G chosen by pick_group(D) and stores Dp = ceil(D/G)*G
// channels (padding channels stay zero).
int pick_group(int D);
// words of the occupancy pyramid (super-block, 4^3-block and 2^3-block bits)
inline size_t occ_words(int gbits) {
  return ((size_t(1) << (3 * (gbits - 3))) + (size_t(1) << (3 * (gbits - 2))) + (size_t(1) << (3 * (gbits - 1)))) / 32;
}
inline int padded_channels(int D, int G) { return G == 0 ? 0 : ((D + G - 1) / G) * G; }

struct DenseDev {
  double2* rw;   // [n] (F.re, W)
  double* fim;   // [n][Dp]
  int nx, ny, nz;
  double vs, ox, oy, oz, mu, cap;
  int order = 1;  // CSFD order of the channel slots (2: bicomplex pairs, 3 slots each)
};

struct HashDev {
  double2* rw;                  // [max_blocks*512]
  double* fim;                  // [max_blocks*512][Dp]
  int* heads;                   // [2^bits]
  unsigned long long* keys;     // [max_blocks]
  int* next;                    // [max_blocks]
  int* coords;                  // [max_blocks][3]
  int* n_blocks;                // device counter
  int* grid;                    // [2^(3*gbits)] dense block-id window (derived index)
  unsigned* occ;                // occupancy bits: super-blocks [2^(3*(gbits-3))], then 4^3-block
                                // cells [2^(3*(gbits-2))], then 2^3-block cells [2^(3*(gbits-1))]
  unsigned char* sdist = nullptr;  // [2^(3*(gbits-3))] Chebyshev distance (super-blocks) to the
                                   // nearest occupied / out-of-window super-block, capped at 8
  unsigned char* sdist_tmp = nullptr;
  int bits, max_blocks, gbits;
  double vs, ox, oy, oz, mu, cap;
  int order = 1;  // CSFD order of the channel slots (2: bicomplex pairs, 3 slots each)
  // Raycast alpha sequence a_0 = near, a_{n+1} = a_n + step (the reference's
  // repeated addition, tsdf.hpp:254): shared by every ray of a hashed volume
  // (no slab clip), so it is tabulated once; a_{n_tab-1} > far is a sentinel.
  const double* alpha_tab = nullptr;
  int alpha_n = 0;
  unsigned* seg_first = nullptr;  // [pixels] first crossing index of the segmented march
};

// Per-frame allocation scratch (hashed volumes).
struct AllocScratch {
  unsigned long long* cand;     // [P*K] candidate keys (kEmptyKey = none)
  int* cand_block;              // [P*K] existing block id or -1
  int* first_flag;              // [P*K]
  int* new_flag;                // [P*K]
  int* first_rank;              // [P*K]
  int* new_rank;                // [P*K]
  unsigned long long* set_keys; // [set_cap]
  int* set_first;               // [set_cap]
  int* set_slot;                // [P*K] set index of the candidate
  int set_bits;
  int* visible;                 // [max visible] block ids
  int* counters;                // [4]: n_visible, n_new, overflow, spare
  void* cub_tmp;
  size_t cub_tmp_bytes;
  int max_cand;                 // P*K
};

// ---- canonical ICP tiling (builder-defined; oracle/orc_icp.hpp restates it)
// The strided slot grid of a level is cut into at most kIcpMaxTiles tiles of
// a multiple of 32 consecutive slots; the level kernel runs one CTA of
// 32 * kIcpLevelWarps threads per tile, one CTA per SM (148 SMs on B200).
constexpr int kIcpLevelWarps = 16;
constexpr int kIcpMaxTiles = 148;
constexpr int kIcpGroup = 16;  // tiles per group of the cross-tile sum
inline int icp_tile_slots(long long n_slots) {
  const long long u = (n_slots + 32LL * kIcpMaxTiles - 1) / (32LL * kIcpMaxTiles);
  return static_cast<int>(32 * (u > 0 ? u : 1));
}

// Tracker state (device)
struct TrackState {
  int level_done;
  int converged;
  int iterations;
  int n_corr;
  int frame;
  int err;
  int pad[2];
  double pred_w2c[12];  // real inverse of the prediction pose (association)
  double cur_c2w[12];   // real current pose snapshot (unused by kernels)
  double delta[6];      // real increment of the last solved ICP iteration
  double b[6];          // its real J^T r (the linearized solver's gradient / 2, icp.cpp:41)
};

// Arguments of the first-order ICP level kernel (icp.cu).
struct IcpLevelArgs {
  TrackState* st;
  const double* depth;
  int w, h, stride;
  const double* intr;  // [4][1+Dp] level intrinsics
  double* pose;        // [12][1+Dp] current pose (in / out)
  const double *vre, *nre, *vim, *nim;
  double d_max, cos_max;
  int Dp;
  int iterations;
  int level;
  double tol;
  int tile_slots, n_tiles;
  double* partials;   // [kIcpMaxTiles][27(1+Dp)]
  double* gpartials;  // [groups][27(1+Dp)]
  double* totals;     // [27(1+Dp)]
  int* counts;        // tiles, groups, total
  unsigned* sync;     // group counters, total counter, release generation
};

// ---- energy.cu: icp_energy / gradient / Hessian and the correspondence list
struct EnergyScratch {
  double* terms = nullptr;
  size_t terms_cap = 0;
  double* sub = nullptr;
  size_t sub_cap = 0;
  double* small = nullptr;
  size_t small_cap = 0;
  int* pairs = nullptr;
  double* corrs = nullptr;  // [n][9] of the last associate_list
  int* flags = nullptr;
  size_t flags_cap = 0;
  void* cub = nullptr;
  size_t cub_bytes = 0;
  double* out = nullptr;  // tree_sum_slots results
  size_t out_cap = 0;
};
// order 0: energy; 1: + gradient; 2: + Hessian.  Synchronous on `stream`.
// Returns 0, 4 (CUDA error) or 5 (out of memory).
int icp_energy_derivs(cudaStream_t stream, EnergyScratch& ws, const double* corrs, int n, const double* base,
                      const double* xi, double h, int order, double* E, double* g, double* H);
int associate_list(cudaStream_t stream, EnergyScratch& ws, const double* depth, int w, int h, int stride,
                   const double* intr4, const double* pose12, const double* pred_w2c12, const double* vre,
                   const double* nre, double d_max, double cos_max, int* n_out);
void energy_scratch_release(EnergyScratch& ws);
int associate_maps(cudaStream_t stream, EnergyScratch& ws, const double* mvert, const double* mnorm,
                   const double* pvert, const double* pnorm, int w, int h, int stride, const double* prm28,
                   double d_max, double cos_max, double* corrs_out, int* n_out);
int linearized_tiles(cudaStream_t stream, const double* corrs, int n, const double* base12, double* tiles_out);
// pairwise_sum of every slot of device terms [C][n] into out_host[C] (synchronous)
int tree_sum_slots(cudaStream_t stream, EnergyScratch& ws, const double* terms, int n, int C, double* out_host);


// ---- reloc.cu: relocalization (reloc.hpp)
// Observed voxels (W > 0) of rw [n_vox]: centers == nullptr counts only.
// coords == nullptr: dense linear index over (nx, ny); else hashed pool coords.
int reloc_flatten(cudaStream_t stream, const double2* rw, long long n_vox, const int* coords, int nx, int ny,
                  double vs, const double* origin, double* centers, double* values, int* n_out);
int reloc_energy_derivs(cudaStream_t stream, EnergyScratch& ws, const double* centers, const double* values, int n,
                        const double* depth, int w, int h, const double* k4, double mu, const double* pose12,
                        int order, double step, double* E, double* g, double* H, long long* overlap);
int depth_cloud_dev(cudaStream_t stream, const double* depth_host, int w, int h, const double* k4,
                    const double* pose12, int stride, double* out_host, int* n_out);
int nn_error_dev(cudaStream_t stream, EnergyScratch& ws, const double* T12, const double* q, int nq, const double* r,
                 int nr, double* mean);

// ---- surfel.cu: surfel (X-EF) front end (surfel.hpp)
struct SurfelArrays {  // device map arrays (capacity >= count)
  double* pos;   // [cap][3][1+D]
  double* nrm;   // [cap][3][1+D]
  double* conf;  // [cap][1+D]
  double* rad;   // [cap]
  int* ts;       // [cap]
};
struct SurfelScratch {
  unsigned* offsets = nullptr; size_t offsets_cap = 0;          // index map offsets [16P+1]
  unsigned* cellk = nullptr; size_t cellk_cap = 0;
  unsigned long long* depthk = nullptr; size_t depthk_cap = 0;
  int* sidx = nullptr; size_t sidx_cap = 0;
  int* entries = nullptr;                                         // points into sidx
  unsigned char* cub = nullptr; size_t cub_cap = 0;
  double *V = nullptr, *N = nullptr, *VW = nullptr, *NW = nullptr;
  size_t V_cap = 0, N_cap = 0, VW_cap = 0, NW_cap = 0;
  int* pint = nullptr; size_t pint_cap = 0;                       // valid, counts, offs, cflag, crank, merged
  int* pidx = nullptr; size_t pidx_cap = 0;                       // pair surfel index (+ sorted copy)
  int* ppix = nullptr; size_t ppix_cap = 0;                       // pair pixel
  double* pw = nullptr; size_t pw_cap = 0;                        // pair lifted weight [T][1+D]
  int* seg = nullptr; size_t seg_cap = 0;
  int* order = nullptr; size_t order_cap = 0;
  unsigned long long* zbest = nullptr; size_t zbest_cap = 0;
  int* ibest = nullptr; size_t ibest_cap = 0;
  unsigned long long launches = 0;
};
struct AssocParams {
  double depth, cos_gate, distance, kernel_scale;
  int one_to_many;
};
int surfel_index_map(cudaStream_t s, SurfelScratch& ws, const double* pos, int n, int D, const double* c2w12,
                     const double* k4, int w, int h, int* m_out);
int surfel_associate(cudaStream_t s, SurfelScratch& ws, const double* spos, const double* snrm, int D,
                     const double* depth, const double* c2w, const double* intr_lifted, const double* c2w12,
                     const double* k4, int w, int h, const AssocParams& ap, int* total, int* merged);
int surfel_created_count(cudaStream_t s, SurfelScratch& ws, int P, int* created);
int surfel_commit(cudaStream_t s, SurfelScratch& ws, SurfelArrays m, int n, int D, int T, const double* c2w12,
                  const double* k4, int w, int h, int frame, double radius_scale);
int surfel_predict(cudaStream_t s, SurfelScratch& ws, const double* pos, const double* nrm, int n, int D,
                   const double* c2w12, const double* k4, int w, int h, double* Vo, double* No);
void surfel_scratch_release(SurfelScratch& ws);
void launch_expand_depth(cudaStream_t s, const double* real, long long P, int C, double* lifted);

// Launch failures seen by the kernel translation units are recorded here and
// surfaced as CSF_ECUDA by the next status check of the C-ABI (a failed
// launch must never yield silently wrong results).
void note_launch_error(const char* what, cudaError_t e);
void note_error(const std::string& msg);  // a launch that could not be issued (no kernel for the shape)
bool take_launch_error(char* msg, size_t cap);

struct Launch {
  cudaStream_t stream;
  int* err;                // device error flag
  unsigned long long* launches;  // host counter of kernels launched
  int phase = 0;           // multi-kernel stages: 0 = all, 1/2 = first/second half only
};

// ---- frames.cu
void launch_bilateral(const Launch& L, const float* in_f32, const double* in_f64, double* raw_out, double* out, int w,
                      int h, double sigma_s, double sigma_r, int radius);
void launch_downsample(const Launch& L, const double* in, double* out, int w, int h, double sigma_r);
void launch_measure(const Launch& L, const double* depth, int w, int h, const double* intr, int D, double* vert,
                    double* norm);

// ---- volume.cu
// upd (nullable): incremented by the number of voxels fused; dch (nullable):
// the depth image's perturbation channels [w*h][Dp] (a lifted depth image)
void launch_integrate_dense(const Launch& L, const DenseDev& v, int G, int Dp, const double* depth, int w, int h,
                            const double* pose, const double* intr, int* upd, const double* dch = nullptr);
void launch_integrate_hashed(const Launch& L, const HashDev& v, int G, int Dp, const AllocScratch& a,
                             const double* depth, int w, int h, const double* pose, const double* intr, int* upd,
                             const double* dch = nullptr);
void launch_allocate(const Launch& L, const HashDev& v, int Dp, AllocScratch& a, const double* depth, int w, int h,
                     const double* pose, const double* intr);
// hits: [w*h] scratch (alpha_prev, alpha) of the zero crossing per pixel
void launch_raycast_dense(const Launch& L, const DenseDev& v, int G, int Dp, const double* pose, const double* intr,
                          int w, int h, double near_clip, double far_clip, double step, double2* hits, double* vre,
                          double* nre, double* vim, double* nim);
void launch_raycast_hashed(const Launch& L, const HashDev& v, int G, int Dp, const double* pose, const double* intr,
                           int w, int h, double near_clip, double far_clip, double step, double2* hits, double* vre,
                           double* nre, double* vim, double* nim);
void launch_init_volume(const Launch& L, double2* rw, double* fim, long long n, int Dp);
// Back to an empty hashed volume with every bound read on the device (no host
// round trip, so a run can be captured in a CUDA graph); the caller zeroes
// n_blocks afterwards and rebuilds the distance field.
void launch_reset_hashed(const Launch& L, const HashDev& v, int Dp);
// super-block distance field of the occupancy bitmap (after every change of occ)
void launch_super_dist(cudaStream_t stream, const HashDev& v);
// point queries (tsdf.hpp:97-196): pts [n][3][1+Dp] lifted (sample) or [n][3] real (measured)
void launch_sample_points(const Launch& L, bool hashed, const DenseDev& dd, const HashDev& hd, int Dp,
                          const double* pts, int n, int grad, double* out, int* valid);
void launch_measured_points(const Launch& L, const double* depth, int w, int h, const double* w2c, const double* intr,
                            double mu, const double* pts, const double* center, int n, int Dp, double* out,
                            int* valid, const double* dch = nullptr);

// ---- icp.cu
void launch_level_begin(const Launch& L, TrackState* st, const double* pose, double* pred_pose, int Dp);
int icp_tiles(int w, int h, int stride);
// Whether a w x h frame at this pixel stride fits the ICP reduction's group
// counters (callers reject larger frames with CSF_EINVAL).
bool icp_frame_fits(int w, int h, int stride);
// ICP scratch (level kernel and second-order reduce); the counts buffer must
// be zeroed once at allocation.
size_t icp_partials_doubles(int C);
size_t icp_counts_ints();
// All iterations of one ICP pyramid level (icp.cpp:193-238) in one
// cooperative launch: association, lifted normal equations, the 6x6 solve
// and the pose update per iteration; the level's break rules on the device.
// Updates pose and TrackState (iterations, n_corr, converged, delta, b).
void launch_icp_level(const Launch& L, int Dp, TrackState* st, const double* depth, int w, int h, int stride,
                      const double* intr, double* pose, const double* vre, const double* nre, const double* vim,
                      const double* nim, double d_max, double cos_max, int iterations, int level, double tol,
                      double* partials, int* counts);
void launch_seed(const Launch& L, int G, int Dp, const int* dirs, int D, double h, const double* gt0,
                 const double* intr_base, double* pose, double* intr_levels, int levels);
void launch_frame_begin(const Launch& L, TrackState* st, int frame);
// keyframe kf's twist seeds applied to the tracked pose (config 4)
void launch_keyframe_seed(const Launch& L, int G, int Dp, const int* dirs, int D, double h, int kf, double* pose);
void launch_frame_end(const Launch& L, TrackState* st, const double* pose, double* traj, int Dp, int* stats,
                      const int* n_blocks, const int* counters);
void launch_objective(const Launch& L, int G, int Dp, int D, const double* traj, const double* gt, int n_frames,
                      int kind, double h, double* out /*[2 + D]: objective re, pad, grad*/);
// Second order (channel groups = bicomplex pairs, 3 slots each): one ICP
// iteration = reduce (tiles x pairs) + per-pair solve + commit; stage [16].
void launch_icp_iteration2(const Launch& L, int Dp, TrackState* st, const double* depth, int w, int h, int stride,
                           const double* intr, double* pose, const double* vre, const double* nre, const double* vim,
                           const double* nim, double d_max, double cos_max, double* partials, int* counts,
                           double* stage, int level, double tol);
void launch_seed2(const Launch& L, int Dp, const int* pair_i, const int* pair_j, int n_pairs, double h,
                  const double* gt0, const double* intr_base, double* pose, double* intr_levels, int levels);
// out [2 + Dp]: objective re, pad, then the raw slots (im1, im2, im12) per pair
void launch_objective2(const Launch& L, int Dp, int n_pairs, const double* traj, const double* gt, int n_frames,
                       int kind, double* out);
void launch_linearized_corrs(const Launch& L, const double* corrs, int n, const double* base, double* partials,
                             int* counts);

// ---- views.cu: BASELINE config 5 view scoring
// pose_out [12][7]: exp(xi) * view with xi seeded h on the 6 twist channels;
// intr_out [4][7] (zero channels)
void launch_view_seed(const Launch& L, const double* view12, const double* k4, double h, double* pose_out,
                      double* intr_out);
// terms [7][w*h]: sigma(beta (w0 - W~(p))) of every raycast hit (0 elsewhere)
void launch_view_terms(const Launch& L, const HashDev& v, const double* vre, const double* nre, const double* vim,
                       int w, int h, double w0, double beta, double* terms);

}  // namespace csfi

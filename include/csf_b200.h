/*
 * csf_b200.h — C-ABI of the B200-native CSFD dense-SLAM hot path.
 *
 * This is the drop-in boundary under the reference's C++ API
 * (proj/include/csf/ *.hpp).  Everything is plain C: pointers, sizes and POD
 * structs; no torch, Eigen or STL types cross it.  Each entry point cites the
 * reference function it replaces.  The C++ mirror of the reference API
 * (include/csf/b200.hpp) is a thin layer over these calls.
 *
 * Conventions:
 *   - Poses are camera->world, 12 scalars (rotation row-major, translation).
 *     A lifted scalar with D perturbation channels is stored as (1+D)
 *     doubles [re, im_0 .. im_{D-1}]; a lifted array is element-major,
 *     channel-minor: value e occupies [e*(1+D), e*(1+D)+D].
 *   - Lifted intrinsics are 4 scalars (fx, fy, cx, cy), same layout.
 *   - Depth is camera z in metres, 0 = invalid.  Images are row-major.
 *   - Status codes map to the reference's exception types:
 *       CSF_EINVAL  -> std::invalid_argument
 *       CSF_EDOMAIN -> std::domain_error (zero real-part divisor on device)
 *       CSF_ERUNTIME/CSF_ECUDA/CSF_ENOMEM -> std::runtime_error
 *     csf_last_error() returns the message of the last failure on a context.
 *   - Host buffers are borrowed for the duration of a call; device memory is
 *     owned by handles.  Calls on one context are serialised by the caller;
 *     different contexts (one per GPU / host thread) may run concurrently.
 */
#ifndef CSF_B200_H
#define CSF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSF_OK 0
#define CSF_EINVAL 1
#define CSF_EDOMAIN 2
#define CSF_ERUNTIME 3
#define CSF_ECUDA 4
#define CSF_ENOMEM 5

#define CSF_MAX_DIRECTIONS 64
#define CSF_MAX_PAIRS 64

typedef struct csf_ctx_s* csf_ctx;
typedef struct csf_volume_s* csf_volume;
typedef struct csf_pipeline_s* csf_pipeline;

/* frames.hpp:15-36 (Intrinsics) */
typedef struct {
  double fx, fy, cx, cy;
  int width, height;
  double depth_scale;
} csf_intrinsics;

/* tsdf.hpp:21-36 (VolumeParams) */
typedef struct {
  int dims[3];
  double voxel_size;
  double origin[3];
  double mu;
  double weight_cap;
} csf_volume_params;

/* Hashed 8^3-block volume (builder-defined) */
typedef struct {
  double voxel_size;
  double origin[3];
  double mu;
  double weight_cap;
  int bucket_bits; /* 2^bucket_bits hash buckets (20 in BASELINE config 2) */
  int max_blocks;  /* block-pool capacity */
} csf_hash_params;

/* tsdf.hpp:198-204 (RaycastConfig) */
typedef struct {
  double near_clip, far_clip, step_fraction;
} csf_raycast_cfg;

/* icp.hpp:33-53 (IcpSolver, IcpConfig).  The device tracker implements
 * CSF_SOLVER_LINEARIZED; the lifted tracker is the linearized solver lifted
 * to the packed scalar. */
#define CSF_SOLVER_LINEARIZED 0
#define CSF_SOLVER_NEWTON 1
#define CSF_SOLVER_GRADIENT_DESCENT 2
#define CSF_SOLVER_CONJUGATE_GRADIENT 3
typedef struct {
  int solver;
  double d_max;
  double theta_max_deg;
  int levels;
  int level_iterations[3];
  int level_pixel_stride[3];
  double step_tolerance;
  double levenberg_lambda0;
  int ncg_restart;
  double h; /* StepSize (csfd.hpp:20-28) */
} csf_icp_cfg;

/* icp.hpp:119-125 (TrackResult) */
typedef struct {
  int iterations;
  int converged;
  int correspondences;
  int pad;
  double final_loss;
} csf_track_result;

#define CSF_OBJECTIVE_FINAL_TRANSLATION_ERROR 0
#define CSF_OBJECTIVE_TRAJECTORY_ERROR 1

/* The CSFD frame-derivative run: seed D directions (first-frame
 * twist components 0..5 in (rho, phi) order and/or intrinsics 6..9 =
 * fx, fy, cx, cy), fuse frame 0 at exp(xi0*) T0, track + fuse frames
 * 1..N-1 with the lifted tracker, differentiate the objective.
 *
 * Direction codes: 0..5 first-frame twist, 6..9 intrinsics, 10.. keyframe
 * twists (keyframe_interval below).
 *
 * order = 2 (BASELINE config 3): instead of dirs, n_pairs parameter pairs
 * (pair_i[p], pair_j[p]) each carried as one reference Bicomplex
 * (csfd.hpp:83-140; im1 seeded on pair_i, im2 on pair_j) packed as three
 * channel slots (im1, im2, im12) of one evaluation; the result is the
 * Hessian entry im12/h^2 per pair (csf_pipeline_hessian), the csfd_hessian
 * pattern of diff.hpp:58-72 applied to the whole frame loop. */
typedef struct {
  int hashed;
  csf_volume_params dense;
  csf_hash_params hash;
  csf_intrinsics k;
  csf_icp_cfg icp;
  csf_raycast_cfg rc;
  double h;
  int n_dirs;
  int dirs[CSF_MAX_DIRECTIONS];
  int objective;
  int max_frames;
  int order;                    /* 1 (default, 0 also means 1) or 2 */
  int n_pairs;                  /* order 2 */
  int pair_i[CSF_MAX_PAIRS];
  int pair_j[CSF_MAX_PAIRS];
  /* Keyframe perturbations (BASELINE config 4, builder-defined): with
   * keyframe_interval K > 0, direction code 10 + 6 (kf - 1) + c (kf >= 1,
   * c = 0..5 in (rho, phi) order) perturbs the tracked pose of frame kf*K by
   * exp(xi) (left increment, se3.hpp:116-119) before it is fused. */
  int keyframe_interval;
} csf_pipeline_cfg;

/* ---- defaults (the reference's struct defaults) ------------------------- */
void csf_default_intrinsics(csf_intrinsics* k);      /* frames.hpp:16-22 */
void csf_default_volume_params(csf_volume_params* p); /* tsdf.hpp:22-26 */
void csf_default_raycast_cfg(csf_raycast_cfg* c);     /* tsdf.hpp:199-203 */
void csf_default_icp_cfg(csf_icp_cfg* c);             /* icp.hpp:41-52 */

/* ---- context -------------------------------------------------------------- */
int csf_ctx_create(int device, csf_ctx* out);
int csf_ctx_destroy(csf_ctx ctx);
const char* csf_last_error(csf_ctx ctx);
int csf_ctx_synchronize(csf_ctx ctx);
/* Number of kernels this context has launched so far (for launch accounting). */
int csf_ctx_launch_count(csf_ctx ctx, unsigned long long* out);
/* CUDA stream of the context (cudaStream_t as void*), for event timing. */
void* csf_ctx_stream(csf_ctx ctx);
/* Per-kernel-category CUDA-event timing on the context stream (off by default).
 * read: names [n][32] (NUL-terminated), total ms and launch counts per
 * category since the last read; resets the records. */
int csf_ctx_profile(csf_ctx ctx, int enable);
int csf_ctx_profile_read(csf_ctx ctx, int max_categories, char* names, double* ms, long long* counts,
                         int* n_categories);

/* ---- frames: frames.cpp:7-75, frames.hpp:86-114 --------------------------- */
int csf_bilateral_filter(csf_ctx ctx, const double* depth, int w, int h, double sigma_s, double sigma_r, int radius,
                         double* out);
int csf_downsample_depth(csf_ctx ctx, const double* depth, int w, int h, double sigma_r, double* out);
/* depth [w*h][1+D] lifted (depth seeds), intr [4][1+D]; outputs [w*h][3][1+D] */
int csf_measure_surface(csf_ctx ctx, const double* depth, int w, int h, const double* intr, int n_channels,
                        double* vertices, double* normals);

/* ---- volumes: tsdf.hpp:38-78 ----------------------------------------------- */
int csf_volume_create_dense(csf_ctx ctx, const csf_volume_params* p, int n_channels, csf_volume* out);
int csf_volume_create_hashed(csf_ctx ctx, const csf_hash_params* p, int n_channels, csf_volume* out);
int csf_volume_destroy(csf_volume vol);
/* Dense: n = dims product.  Hashed: n = block_count * 512 (block-major,
 * voxel (lz*8+ly)*8+lx).  field [n][1+D], weight [n]. */
int csf_volume_upload(csf_volume vol, const double* field, const double* weight);
int csf_volume_download(csf_volume vol, double* field, double* weight);
int csf_volume_block_count(csf_volume vol, int* n_blocks);
/* The volume's channel count, kind (hashed 1 / dense 0) and voxel count (dense
 * lattice size, or allocated blocks x 512). */
int csf_volume_info(csf_volume vol, int* n_channels, int* hashed, long long* n_voxels);
/* heads [2^bits], keys [n_blocks], next [n_blocks], coords [n_blocks][3] */
int csf_volume_download_hash(csf_volume vol, int32_t* heads, uint64_t* keys, int32_t* next, int32_t* coords);

/* Point queries.  tsdf.hpp:148-177 sample_tsdf / 181-196 sample_gradient at
 * lifted world points [n][3][1+D] (D = the volume's channels): values
 * [n][1+D] / gradients [n][3][1+D]; valid[i] = 0 where the reference returns
 * std::nullopt (a corner unobserved / unallocated). */
int csf_sample_tsdf(csf_volume vol, const double* points, int n, double* values, int32_t* valid);
int csf_sample_gradient(csf_volume vol, const double* points, int n, double* gradients, int32_t* valid);
/* tsdf.hpp:97-140 measured_tsdf at real voxel positions points [n][3]:
 * unperturbed depth [h][w], lifted world->camera pose [12][1+D], lifted
 * intrinsics [4][1+D], lifted camera centre [3][1+D]; psi [n][1+D]. */
int csf_measured_tsdf(csf_ctx ctx, const double* depth, int w, int h, const double* world_to_camera,
                      const double* intr, double mu, const double* points, const double* center, int n,
                      int n_channels, double* psi, int32_t* valid);
/* measured_tsdf with a lifted depth image [h][w][1+n_channels]
 * (tsdf.hpp:97-102 takes Image<S> depth): d psi / d depth = bilinear weight / mu
 * (test_tsdf.cpp:194-231). */
int csf_measured_tsdf_lifted(csf_ctx ctx, const double* depth, int w, int h, const double* world_to_camera,
                             const double* intr, double mu, const double* points, const double* center, int n,
                             int n_channels, double* psi, int32_t* valid);

/* tsdf.cpp:61-153 — save_volume / load_volume in the reference's "CSFVOL 1"
 * container: text header (dims, voxel_size, origin, mu, weight_cap, channels)
 * then float32 planes (field, weight, derivative channels only when any is
 * non-zero).  A dense single-channel file is byte-compatible with the
 * reference.  Extensions (builder-defined): D derivative planes for D
 * channels; hashed volumes add "hashed <bucket_bits> <max_blocks>" and
 * "blocks N" and an int32 N x 3 block-coordinate plane (pool order) before
 * the voxel planes (block-major); loading rebuilds the canonical hash table.
 * load: n_channels = -1 takes the file's channel count.  I/O errors map to
 * CSF_ERUNTIME (std::runtime_error). */
int csf_volume_save(csf_volume vol, const char* path);
int csf_volume_load(csf_ctx ctx, const char* path, int n_channels, csf_volume* out);

/* tsdf.cpp:11-40 — fuse one unperturbed depth frame at a lifted camera pose
 * with lifted intrinsics.  Hashed volumes first allocate the frame's
 * truncation-band blocks; *n_visible (optional) receives the visible count. */
int csf_surface_update(csf_volume vol, const double* depth, int w, int h, const double* pose, const double* intr,
                       int* n_visible);
/* surface_update with a lifted depth image [h][w][1+D] — the reference's
 * Image<Complex> depth (tsdf.hpp:144-145): the depth's own perturbation
 * channels enter psi through the bilinear sample (tsdf.hpp:96-140), e.g. a
 * depth pixel seeded with perturb_depth (frames.cpp:77-102).  First-order
 * volumes; validity, the edge test and the hashed allocation read real parts. */
int csf_surface_update_lifted(csf_volume v, const double* depth, int w, int h, const double* pose,
                              const double* intr, int* n_visible);
/* tsdf.hpp:209-284 — lifted raycast; outputs [w*h][3][1+D] world-frame maps */
int csf_raycast(csf_volume vol, const double* pose, const double* intr, int w, int h, const csf_raycast_cfg* cfg,
                double* vertices, double* normals);

/* ---- icp: icp.cpp:169-244 ----------------------------------------------------
 * Coarse-to-fine tracking of one frame against a volume's real channel, every
 * solver family of the reference: linearized (canonical slot-tiled normal
 * equations), Newton (CSFD gradient + Hessian of icp_energy, Levenberg
 * damping and the -g line search of descent.hpp:109-144), gradient descent
 * and Polak-Ribiere NCG (descent.hpp:58-101).  result->final_loss is the
 * last iteration's loss_after / correspondences (icp.cpp:207-209). */
int csf_track_frame(csf_volume vol, const double* depth, int w, int h, const double* init_pose,
                    const csf_intrinsics* k, const csf_icp_cfg* cfg, double* out_pose, csf_track_result* result);
/* track_frame(..., TrackTrace*) (icp.hpp:130-133, icp.cpp:213-228): also the
 * trace rows [trace_cap][15] = iteration, mean loss, gradient norm (the
 * solver's s.gradient: 2 b for linearized, the CSFD gradient otherwise), then
 * the camera->world pose [12] after the step; *n_trace rows (may exceed
 * trace_cap).  Ground-truth errors are host arithmetic on the poses (mirrors). */
int csf_track_frame_traced(csf_volume vol, const double* depth, int w, int h, const double* init_pose,
                           const csf_intrinsics* k, const csf_icp_cfg* cfg, double* out_pose,
                           csf_track_result* result, double* trace, int trace_cap, int* n_trace);

/* icp.cpp:89-126 — associate(measured, predicted, pose, prediction_pose, k,
 * cfg, stride): maps [h][w][3] (vertices camera / world, normals), poses
 * camera->world [12]; corrs [<= slots][9] in scan order, *n_corrs. */
int csf_associate(csf_ctx ctx, const double* measured_vertices, const double* measured_normals,
                  const double* predicted_vertices, const double* predicted_normals, int w, int h,
                  const double* camera_to_world, const double* predicted_camera_to_world, const csf_intrinsics* k,
                  const csf_icp_cfg* cfg, int pixel_stride, double* corrs, int* n_corrs);
/* icp.cpp:146-153 — linearized_step(corrs, base): the normal equations in
 * the canonical tiled order, LDLT solve of A d = -b, zero
 * when not finite. */
int csf_linearized_step(csf_ctx ctx, const double* corrs, int n, const double* base, double* delta);
/* diff.hpp:16-37 — pairwise_sum of n terms with `channels` lanes each
 * (terms [n][channels], e.g. a lifted value): the reference's fixed tree per
 * lane, init 0. */
int csf_pairwise_sum(csf_ctx ctx, const double* terms, int n, int channels, double* out);

/* icp.hpp:70-91 — icp_energy(corrs, xi, base) with the pairwise_sum tree
 * (diff.hpp:16-37); gradient (optional) = the 6 Complex passes of
 * icp_gradient, hessian (optional, [36] row-major) = the 21 Bicomplex passes
 * of icp_hessian, evaluated at xi (NULL = 0) as one packed device pass.
 * corrs [n][9] = vertex (camera), model vertex, model normal (world) per
 * correspondence (icp.hpp:27-31); base [12] camera->world. */
int csf_icp_energy_derivs(csf_ctx ctx, const double* corrs, int n, const double* base, const double* xi, double h,
                          double* energy, double* gradient, double* hessian);

/* ---- BASELINE config 5: active-scanning view scoring --------------------------
 * Builder-defined objective (the spec's task-gradient "smooth visibility
 * score", is unimplemented in the reference): for each
 * candidate camera->world view T [n][12], S(T) = pairwise_sum over the
 * k->width x k->height pixels (row-major) of sigma(beta (w0 - W~(p))) at the
 * raycast hit p (0 for misses), W~ = trilinear interpolation of the integral
 * fusion weights — a soft count of weakly observed surface the view would
 * see.  grads [n][6] (optional) = dS/dxi of exp(xi) T by CSFD (step h), one
 * lifted raycast per view.  vol: hashed, created with 6 channels, fused with
 * unperturbed poses. */
int csf_view_scores(csf_volume vol, const double* poses, int n_views, const csf_intrinsics* k, double w0, double beta,
                    double h, double* scores, double* grads);

/* ---- relocalization: reloc.hpp --------------------------
 * The reference implements reloc_energy<S> (reloc.hpp:48-69) and declares the
 * rest without bodies; the builder-defined bodies follow the header comments
 * and SPEC.md:533-600.  A csf_reloc is a RelocProblem
 * (reloc.hpp:35-46) resident in HBM: the reference volume's observed voxels
 * (W > 0, storage order: dense linear index, hashed pool block then local
 * index) as centres + real field values, the query depth and intrinsics,
 * mu = the volume's mu. */
typedef struct csf_reloc_s* csf_reloc;
#define CSF_RELOC_GRADIENT_DESCENT 0
#define CSF_RELOC_NEWTON 1
/* reloc.hpp:82-98 (RelocConfig with LineSearchConfig, descent.hpp:16-21) */
typedef struct {
  double switch_relative;  /* 0.5 */
  double switch_absolute;  /* -1 = use switch_relative */
  int max_iterations;      /* 50 */
  int ls_max_backtracks;   /* 25 */
  double step_tolerance;   /* 1e-6 */
  double ls_initial_step, ls_shrink, ls_sufficient_decrease; /* 1, 0.5, 1e-4 */
  double h;                /* StepSize, 1e-8 */
  /* builder-defined safeguards: the overlap-restricted sum
   * also falls when the view slides off the model, so a trial pose keeping
   * fewer than min_overlap_ratio x the current overlap counts as +inf, and
   * every direction is scaled to twist length <= max_step (the steepest-
   * descent direction to exactly max_step). */
  double max_step;          /* 0.05 */
  double min_overlap_ratio; /* 0.9 */
} csf_reloc_cfg;
/* reloc.hpp:100-106 (RelocResult) */
typedef struct {
  int iterations;
  int converged;
  double final_loss;
} csf_reloc_result;
void csf_default_reloc_cfg(csf_reloc_cfg* cfg);
/* RelocProblem(reference, query, k) (reloc.hpp:44-45): EINVAL when the
 * volume has no observed voxel.  query depth [h][w] (host). */
int csf_reloc_create(csf_volume reference, const double* query_depth, int w, int h, const csf_intrinsics* k,
                     csf_reloc* out);
int csf_reloc_destroy(csf_reloc r);
/* voxel count and mu; centers [n][3] / values [n] (optional, host) */
int csf_reloc_info(csf_reloc r, int* n_voxels, double* mu, double* centers, double* values);
/* reloc_energy at the camera->world pose [12] (reloc.hpp:48-69), with the
 * reloc_gradient (6 Complex passes) / reloc_hessian (21 Bicomplex passes) of
 * reloc.hpp:75-80 at order 1 / 2 as one packed device pass each; overlap =
 * mutually observed voxels.  ERUNTIME when no voxel overlaps. */
int csf_reloc_energy(csf_reloc r, const double* pose, int order, double h, double* energy, double* gradient,
                     double* hessian, long long* overlap);
/* relocalize (reloc.hpp:116-124): gradient descent or eta-switched Newton
 * with backtracking line search; losses / gradient_norms [max_iterations]
 * (optional) = the trace rows (TraceRow::loss, gradient_norm). */
int csf_relocalize(csf_reloc r, const double* initial_pose, int method, const csf_reloc_cfg* cfg, double* out_pose,
                   csf_reloc_result* result, double* losses, double* gradient_norms);
/* depth_cloud (reloc.hpp:126-129): world points [<= ceil(w/s) ceil(h/s)][3]
 * of the valid pixels at the stride, row-major order. */
int csf_depth_cloud(csf_ctx ctx, const double* depth, int w, int h, const csf_intrinsics* k,
                    const double* camera_to_world, int stride, double* points, int* n_points);
/* eval_nn_error (reloc.hpp:131-138): mean nearest-neighbour distance from
 * transform * query to reference (brute force on the device); EINVAL on an
 * empty cloud; outlier = mean > 0.1 m. */
int csf_eval_nn_error(csf_ctx ctx, const double* transform, const double* query, int n_query, const double* reference,
                      int n_reference, double* mean, int32_t* outlier);

/* ---- surfel (X-EF) front end: surfel.hpp / surfel.cpp ----
 * A csf_surfels is a SurfelMap (surfel.hpp:24-31) resident in HBM whose
 * position, normal and confidence carry D derivative channels (the
 * reference's Complex is D = 1): positions / normals [n][3][1+D],
 * confidence [n][1+D], radius [n], timestamp [n].  Indices are stable
 * (append only). */
typedef struct csf_surfels_s* csf_surfels;
/* surfel.hpp:55-60, 84-91 */
typedef struct {
  double depth, normal_deg, distance, sigma; /* 0.05 m, 30 deg, 0.05 m, 0.025 m */
  int one_to_many;                           /* 1 */
} csf_surfel_cfg;
void csf_default_surfel_cfg(csf_surfel_cfg* cfg);
int csf_surfels_create(csf_ctx ctx, int n_channels, csf_surfels* out);
int csf_surfels_destroy(csf_surfels m);
int csf_surfels_count(csf_surfels m, int* n);
/* empty the map, keeping its device capacity and scratch */
int csf_surfels_clear(csf_surfels m);
/* host copies of the map (any output may be NULL) / replace the map */
int csf_surfels_download(csf_surfels m, double* positions, double* normals, double* radius, double* confidence,
                         int32_t* timestamps);
int csf_surfels_upload(csf_surfels m, int n, const double* positions, const double* normals, const double* radius,
                       const double* confidence, const int32_t* timestamps);
/* surfel.cpp:30-64 — the 4x-supersampled index map at a real camera->world
 * pose: offsets [16 w h + 1], entries [n] (nearest-first per cell). */
int csf_render_index_map(csf_surfels m, const double* camera_to_world, const csf_intrinsics* k, uint32_t* offsets,
                         int32_t* entries, int* n_entries);
/* surfel.cpp:66-108 for every pixel of a lifted depth [h][w][1+D] at a lifted
 * camera->world pose [12][1+D] (real intrinsics): counts [w h]; with
 * indices/weights non-NULL (capacity cap) the lists in pixel scan order,
 * candidate order within a pixel (weights [.][1+D]); *total = sum of counts. */
int csf_associate_surfels(csf_surfels m, const double* depth, int w, int h, const double* camera_to_world,
                          const csf_intrinsics* k, const csf_surfel_cfg* cfg, int32_t* counts, int32_t* indices,
                          double* weights, int cap, int* total);
/* surfel.cpp:121-236 — update_surfels(map, depth, camera_to_world, k, frame) */
int csf_update_surfels(csf_surfels m, const double* depth, int w, int h, const double* camera_to_world,
                       const csf_intrinsics* k, int frame_index, const csf_surfel_cfg* cfg, int* merged_pixels,
                       int* created);
/* the same with an unperturbed depth [h][w] (complex_depth, frames.cpp:77-81:
 * zero channels; lifted on the device) */
int csf_update_surfels_real(csf_surfels m, const double* depth, int w, int h, const double* camera_to_world,
                            const csf_intrinsics* k, int frame_index, const csf_surfel_cfg* cfg, int* merged_pixels,
                            int* created);
/* surfel.cpp:238-263 — nearest-surfel splat: vertices / normals [h][w][3] */
int csf_predict_maps(csf_surfels m, const double* camera_to_world, const csf_intrinsics* k, double* vertices,
                     double* normals);
/* surfel.cpp:110-119 */
double csf_sample_confidence(const csf_intrinsics* k, int x, int y);

/* ---- on-disk formats: dataset.hpp / dataset.cpp -------
 * Host-side file I/O (no context needed).  Failures return CSF_ERUNTIME
 * (std::runtime_error) with the message in csf_io_last_error(). */
const char* csf_io_last_error(void);
/* dataset.cpp:30-68 — 16-bit grayscale PNG, q = round(d*scale) if 1..65535 else 0 */
int csf_write_depth_png16(const char* path, const double* depth, int w, int h, double scale);
/* dataset.cpp:70-107 — depth [h][w] = v/scale (0 where v = 0); depth NULL: size only */
int csf_read_depth_png16(const char* path, double scale, double* depth, int* w, int* h);
/* dataset.cpp:109-141 — "fx fy cx cy width height depth_scale", '#' comments */
int csf_read_intrinsics(const char* path, csf_intrinsics* k);
int csf_write_intrinsics(const char* path, const csf_intrinsics* k);
/* dataset.cpp:143-177 — "t tx ty tz qx qy qz qw" lines; poses [n][12]
 * camera->world; timestamps/poses NULL: count only (cap entries filled). */
int csf_read_trajectory(const char* path, double* timestamps, double* poses, int cap, int* n);
int csf_write_trajectory(const char* path, const double* timestamps, const double* poses, int n);

/* ---- pipeline ------------------------------------------------------------ */
int csf_pipeline_create(csf_ctx ctx, const csf_pipeline_cfg* cfg, csf_pipeline* out);
int csf_pipeline_destroy(csf_pipeline p);
/* depth [n][h][w] float32 metres (host), gt [n][12] camera->world (host). */
int csf_pipeline_upload(csf_pipeline p, const float* depth, const double* gt, int n_frames);
/* Runs the uploaded frames on the device; asynchronous on the context stream. */
int csf_pipeline_run(csf_pipeline p, int n_frames);
/* Synchronises; gradient [D], poses [n][12][1+D] (optional), stats [n][8]
 * (optional: iterations, correspondences, converged, allocated blocks,
 * visible blocks, new blocks, fused voxels, 0). */
int csf_pipeline_result(csf_pipeline p, double* gradient, double* objective, double* poses, int32_t* stats);
/* Order-2 runs: hessian [n_pairs] = H_{pair_i, pair_j}; grad1/grad2 [n_pairs]
 * (optional) = d obj / d param pair_i / pair_j from the same pass; poses
 * (optional) [n][12][1 + 3 n_pairs] (re, then im1, im2, im12 per pair). */
int csf_pipeline_hessian(csf_pipeline p, double* hessian, double* grad1, double* grad2, double* objective,
                         double* poses, int32_t* stats);
/* Graph mode (enable != 0): csf_pipeline_run replays the whole run as one
 * CUDA graph — captured on the first graph-mode call after a stream-mode run
 * of the same frame count, bit-identical to the stream run.  Runs that
 * profile (csf_ctx_profile) or wait on per-frame uploads (run_host) keep the
 * stream path. */
int csf_pipeline_set_graph(csf_pipeline p, int enable);
/* The pipeline's volume after the last run, borrowed (owned by the pipeline:
 * never pass it to csf_volume_destroy).  Read it with csf_volume_download /
 * csf_volume_download_hash / csf_volume_block_count; it carries the run's
 * channel slots (n_dirs, or 3 n_pairs at order 2). */
int csf_pipeline_volume(csf_pipeline p, csf_volume* out);
/* One end-to-end call from host buffers: upload, run, read back. */
int csf_pipeline_run_host(csf_pipeline p, const float* depth, const double* gt, int n_frames, double* gradient,
                          double* objective);
/* BASELINE config 2's RGB-D ingest: as csf_pipeline_run_host, plus uint8 colour
 * frames rgb [n][h][w][3] (NULL: none) uploaded behind each frame's depth on
 * the copy stream into the pipeline's colour buffer.  Colour is ingested and
 * unused — the reference pipeline has no colour term (frames.hpp
 * reads depth only) — so no kernel waits on it; the call returns after the
 * colour uploads have landed (the host buffer is borrowed for the call). */
int csf_pipeline_run_host_rgbd(csf_pipeline p, const float* depth, const unsigned char* rgb, const double* gt,
                               int n_frames, double* gradient, double* objective);
/* Colour frame `frame` as ingested by the last run_host_rgbd call, out [h][w][3]. */
int csf_pipeline_download_rgb(csf_pipeline p, int frame, unsigned char* out);

/* ---- direction-sharded runs (collective C2) ------------------
 * Rank r of N packs a contiguous block of the directions (or pairs) as its
 * channels; the derivative columns are gathered at the end over an NCCL
 * communicator owned by the context (libnccl.so.2 opened at runtime).
 * Rank 0 creates the 128-byte unique id, every rank attaches with it. */
int csf_comm_unique_id(unsigned char* id /* [128] */);
int csf_ctx_attach_comm(csf_ctx ctx, int n_ranks, int rank, const unsigned char* id /* [128] */);
/* counts[r] columns from rank r, in rank order, into out[sum counts] on every
 * rank (host buffers; local = this rank's counts[rank] columns). */
int csf_gather_columns(csf_ctx ctx, const double* local, const int* counts, double* out);

/* ---- synthetic inputs (harness; not on the timed path) ----------------------
 * BASELINE configs 1 and 2 rendered on the device with the reference's
 * sphere tracer (synth.cpp:55-90) and the builder-defined sensor model;
 * depth [n][h][w] float32, gt [n][12].  width/height 0 = config default. */
int csf_synth_workload(csf_ctx ctx, int config, int n_frames, int width, int height, float* depth, double* gt,
                       csf_intrinsics* k);

#ifdef __cplusplus
}
#endif

#endif /* CSF_B200_H */

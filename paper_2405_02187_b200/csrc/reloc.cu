// Camera relocalization on sm_100a (reference
// proj/include/csf/reloc.hpp).
//
//   RelocProblem   — reloc.hpp:35-46: the reference volume flattened to its
//                    observed voxels (W > 0) in storage order, by a flag /
//                    CUB exclusive scan / scatter compaction over the voxel
//                    store (dense linear index, or hashed pool block then
//                    block-local index); centres origin + vs*(i, j, k).
//   reloc_energy   — reloc.hpp:48-69: per observed voxel the projective
//                    measurement psi of the query depth (measured_tsdf,
//                    tsdf.hpp:97-140, the fusion kernels' device function),
//                    term (psi - F_ref)^2 or 0, summed over ALL observed
//                    voxels with the reference's pairwise_sum tree
//                    (diff.hpp:16-37, tree_sum_slots in energy.cu).
//   reloc_gradient — 6 Complex passes (reloc.hpp:75-77) as ONE packed L<6>
//                    evaluation: channel d of Lifted<D> follows the Complex
//                    formula exactly (oracle/orc_core.hpp Lifted).
//   reloc_hessian  — 21 Bicomplex passes (reloc.hpp:78-80) as the 21
//                    upper-triangle pairs of B<1> channel groups (one grid
//                    row per pair), as icp_hessian in energy.cu.
//   depth_cloud    — reloc.hpp:126-129, flag / scan / scatter in row-major
//                    order; eval_nn_error — reloc.hpp:131-138, brute-force
//                    nearest neighbour with the reference cloud staged through
//                    shared memory, mean by the pairwise tree.
//
// Every channel division is the reference's per-channel quotient
// (CSF_EXACT_CHANNELS) so the relocalizer's steps, which consume these
// derivatives, stay bit-identical to the CPU oracle.
#define CSF_EXACT_CHANNELS 1
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "csf_internal.h"
#include "geometry.cuh"

namespace csfd {

// ---------------------------------------------------------------------------
// flatten: flags / scatter over the voxel store
// ---------------------------------------------------------------------------
__global__ void k_reloc_flags(const double2* __restrict__ rw, long long n, int* __restrict__ flags) {
  pdl_wait();
  pdl_trigger();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    flags[i] = rw[i].y > 0.0 ? 1 : 0;
}

// coords == nullptr: dense (nx, ny) linear index; else hashed pool coords.
__global__ void k_reloc_scatter(const double2* __restrict__ rw, long long n, const int* __restrict__ flags,
                                const int* __restrict__ pos, const int* __restrict__ coords, int nx, int ny,
                                double vs, double ox, double oy, double oz, double* __restrict__ centers,
                                double* __restrict__ values, int* __restrict__ count) {
  pdl_wait();
  pdl_trigger();
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (v == n - 1) *count = pos[v] + flags[v];
    if (!flags[v]) continue;
    int i, j, k;
    if (coords) {
      const long long b = v >> 9;
      const int l = static_cast<int>(v & 511);
      i = coords[3 * b] * 8 + (l & 7);
      j = coords[3 * b + 1] * 8 + ((l >> 3) & 7);
      k = coords[3 * b + 2] * 8 + (l >> 6);
    } else {
      i = static_cast<int>(v % nx);
      j = static_cast<int>((v / nx) % ny);
      k = static_cast<int>(v / (static_cast<long long>(nx) * ny));
    }
    const long long o = pos[v];
    centers[3 * o] = ox + vs * static_cast<double>(i);
    centers[3 * o + 1] = oy + vs * static_cast<double>(j);
    centers[3 * o + 2] = oz + vs * static_cast<double>(k);
    values[o] = rw[v].x;
  }
}

// ---------------------------------------------------------------------------
// lifted query pose: exp(xi) * base with the CSFD seeds (T [12][C])
// ---------------------------------------------------------------------------
// L<6>: channel d seeded on twist component d (csfd_gradient, diff.hpp:46-56)
__global__ void k_reloc_pose_l6(const double* __restrict__ base, double h, double* __restrict__ T) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  using S = L<6>;
  S xi[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    xi[k] = lit<S>(0.0);
    xi[k].im[k] = h;
  }
  Pose<S> b;
#pragma unroll
  for (int e = 0; e < 9; ++e) b.R.m[e] = lit<S>(base[e]);
#pragma unroll
  for (int e = 0; e < 3; ++e) b.t.v[e] = lit<S>(base[9 + e]);
  const Pose<S> pose = compose(exp_map<S>(xi), b);
#pragma unroll
  for (int e = 0; e < 9; ++e) store_ch<S>(T + e * 7, pose.R.m[e], 0, 6, true);
#pragma unroll
  for (int e = 0; e < 3; ++e) store_ch<S>(T + (9 + e) * 7, pose.t.v[e], 0, 6, true);
}

// B<1> pairs (csfd_hessian, diff.hpp:58-72): im1 on pair_i, im2 on pair_j;
// grid row p < P; P = 0: the real pose.  T [12][1 + 3P].
template <typename S>
__global__ void k_reloc_pose_pairs(int P, const double* __restrict__ base, double h, double* __restrict__ T) {
  pdl_wait();
  pdl_trigger();
  const int p = threadIdx.x;
  if (p >= (P > 0 ? P : 1)) return;
  constexpr int G = Traits<S>::G;
  const int C = 1 + 3 * P;
  S xi[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) xi[k] = lit<S>(0.0);
  if constexpr (G > 0) {
    int pi = 0, pj = 0, q = 0;
    for (int a = 0; a < 6; ++a)
      for (int b = a; b < 6; ++b, ++q)
        if (q == p) {
          pi = a;
          pj = b;
        }
    xi[pi].im[0] = h;
    xi[pj].im[1] = h;
  }
  Pose<S> b;
#pragma unroll
  for (int e = 0; e < 9; ++e) b.R.m[e] = lit<S>(base[e]);
#pragma unroll
  for (int e = 0; e < 3; ++e) b.t.v[e] = lit<S>(base[9 + e]);
  const Pose<S> pose = compose(exp_map<S>(xi), b);
#pragma unroll
  for (int e = 0; e < 9; ++e) store_ch<S>(T + e * C, pose.R.m[e], 3 * p, G, p == 0);
#pragma unroll
  for (int e = 0; e < 3; ++e) store_ch<S>(T + (9 + e) * C, pose.t.v[e], 3 * p, G, p == 0);
}

// One term per (observed voxel, channel group); terms [C][n] slot-major.
// grid.y = channel group (slot offset G*y); overlap counted by group 0.
template <typename S>
__global__ void __launch_bounds__(256) k_reloc_terms(const double* __restrict__ centers,
                                                     const double* __restrict__ values, int n,
                                                     const double* __restrict__ depth, int w, int h,
                                                     const double* __restrict__ k4, double mu,
                                                     const double* __restrict__ T, int C,
                                                     double* __restrict__ terms,
                                                     unsigned long long* __restrict__ overlap) {
  pdl_wait();
  pdl_trigger();
  constexpr int G = Traits<S>::G;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int grp = blockIdx.y;
  bool ok = false;
  if (i < n) {
    Pose<S> pose;
#pragma unroll
    for (int e = 0; e < 9; ++e) pose.R.m[e] = load_ch<S>(T + e * C, G * grp, G);
#pragma unroll
    for (int e = 0; e < 3; ++e) pose.t.v[e] = load_ch<S>(T + (9 + e) * C, G * grp, G);
    // reloc.hpp:52-53: world_to_camera = query_pose.inverse(), centre = t
    const Pose<S> w2c = inverse(pose);
    Intr<S> k;
    k.fx = lit<S>(k4[0]);
    k.fy = lit<S>(k4[1]);
    k.cx = lit<S>(k4[2]);
    k.cy = lit<S>(k4[3]);
    k.w = w;
    k.h = h;
    S psi;
    S t = lit<S>(0.0);
    ok = measured_tsdf<S>(depth, w, h, w2c, k, mu, centers[3LL * i], centers[3LL * i + 1], centers[3LL * i + 2],
                          pose.t, &psi);
    if (ok) {
      const S diff = psi - values[i];
      t = diff * diff;
    }
    if (grp == 0) terms[i] = re(t);
    if constexpr (G > 0) {
#pragma unroll
      for (int g = 0; g < G; ++g) terms[static_cast<long long>(1 + G * grp + g) * n + i] = t.im[g];
    }
  }
  if (grp == 0) {  // one atomic per block (per-warp atomics on one address serialise in L2)
    const int cnt = __syncthreads_count(ok);
    if (threadIdx.x == 0 && cnt) atomicAdd(overlap, static_cast<unsigned long long>(cnt));
  }
}

// ---------------------------------------------------------------------------
// depth_cloud / eval_nn_error
// ---------------------------------------------------------------------------
__global__ void k_cloud_flags(const double* __restrict__ depth, int w, int h, int stride, int* __restrict__ flags) {
  pdl_wait();
  pdl_trigger();
  const int nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nxs * nys) return;
  const int x = (s % nxs) * stride, y = (s / nxs) * stride;
  flags[s] = depth[static_cast<long long>(y) * w + x] > 0.0 ? 1 : 0;
}

// frames.hpp:38-43 backproject, then camera_to_world * v (se3.hpp)
__global__ void k_cloud_scatter(const double* __restrict__ depth, int w, int h, int stride,
                                const double* __restrict__ prm /*k4, pose12*/, const int* __restrict__ flags,
                                const int* __restrict__ pos, double* __restrict__ out, int* __restrict__ count) {
  pdl_wait();
  pdl_trigger();
  const int nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  const int n = nxs * nys;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  if (s == n - 1) *count = pos[s] + flags[s];
  if (!flags[s]) return;
  const int x = (s % nxs) * stride, y = (s / nxs) * stride;
  const double d = depth[static_cast<long long>(y) * w + x];
  const double fx = prm[0], fy = prm[1], cx = prm[2], cy = prm[3];
  const V3<double> v = mk3<double>(d * (static_cast<double>(x) - cx) / fx, d * (static_cast<double>(y) - cy) / fy, d);
  Pose<double> c2w;
#pragma unroll
  for (int e = 0; e < 9; ++e) c2w.R.m[e] = prm[4 + e];
#pragma unroll
  for (int e = 0; e < 3; ++e) c2w.t.v[e] = prm[13 + e];
  const V3<double> p = apply(c2w, v);
  double* o = out + 3LL * pos[s];
  o[0] = p.v[0];
  o[1] = p.v[1];
  o[2] = p.v[2];
}

// dist[i] = min_j |T q_i - r_j| (squared distances compared, one sqrt)
constexpr int kNnTile = 256;
__global__ void __launch_bounds__(kNnTile) k_nn_dist(const double* __restrict__ T12, const double* __restrict__ q,
                                                     int nq, const double* __restrict__ r, int nr,
                                                     double* __restrict__ dist) {
  pdl_wait();
  pdl_trigger();
  __shared__ double rs[3][kNnTile];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  V3<double> tq = mk3<double>(0.0, 0.0, 0.0);
  if (i < nq) {
    Pose<double> T;
#pragma unroll
    for (int e = 0; e < 9; ++e) T.R.m[e] = T12[e];
#pragma unroll
    for (int e = 0; e < 3; ++e) T.t.v[e] = T12[9 + e];
    tq = apply(T, mk3<double>(q[3LL * i], q[3LL * i + 1], q[3LL * i + 2]));
  }
  double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  for (int base = 0; base < nr; base += kNnTile) {
    const int m = min(kNnTile, nr - base);
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < m) {
      const long long j = base + threadIdx.x;
      rs[0][threadIdx.x] = r[3 * j];
      rs[1][threadIdx.x] = r[3 * j + 1];
      rs[2][threadIdx.x] = r[3 * j + 2];
    }
    __syncthreads();
    for (int j = 0; j < m; ++j) {
      const double d0 = tq.v[0] - rs[0][j], d1 = tq.v[1] - rs[1][j], d2 = tq.v[2] - rs[2][j];
      const double s = d0 * d0 + (d1 * d1 + d2 * d2);  // sum3 order (oracle dot)
      best = s < best ? s : best;
    }
  }
  if (i < nq) dist[i] = sqrt(best);
}

}  // namespace csfd

// ============================================================================
namespace csfi {

using namespace csfd;

static void chk(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) note_launch_error(what, e);
}

static int grid_of(long long n) {
  const int sms = sm_count();
  const long long want = (n + 255) / 256;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(want, 8LL * sms)));
}

// Observed voxels of a voxel store rw [n_vox] -> centers [*][3], values [*]
// (device buffers grown by the caller from the count pass).  Two phases so
// the caller can size its buffers: count (centers == nullptr) then fill.
int reloc_flatten(cudaStream_t stream, const double2* rw, long long n_vox, const int* coords, int nx, int ny,
                  double vs, const double* origin, double* centers, double* values, int* n_out) {
  *n_out = 0;
  if (n_vox <= 0) return 0;
  if (n_vox > 0x7fffffffLL) return 1;
  int *flags = nullptr, *count = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  const int n = static_cast<int>(n_vox);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, static_cast<int*>(nullptr), static_cast<int*>(nullptr), n);
  if (cudaMalloc(&flags, sizeof(int) * (2 * static_cast<size_t>(n) + 1)) != cudaSuccess) return 5;
  if (cudaMalloc(&tmp, tmp_bytes) != cudaSuccess) {
    cudaFree(flags);
    return 5;
  }
  int* pos = flags + n;
  count = pos + n;
  const int grid = grid_of(n_vox);
  launch_pdl(k_reloc_flags, dim3(grid), dim3(256), 0, stream, rw, n_vox, flags);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flags, pos, n, stream);
  int rc = 0;
  if (!centers) {
    // count only: last flag + last exclusive prefix
    int hv[2] = {0, 0};
    if (cudaMemcpyAsync(&hv[0], pos + n - 1, sizeof(int), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaMemcpyAsync(&hv[1], flags + n - 1, sizeof(int), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
      rc = 4;
    *n_out = hv[0] + hv[1];
  } else {
    launch_pdl(k_reloc_scatter, dim3(grid), dim3(256), 0, stream, rw, n_vox, static_cast<const int*>(flags),
               static_cast<const int*>(pos), coords, nx, ny, vs, origin[0], origin[1], origin[2], centers, values,
               count);
    if (cudaMemcpyAsync(n_out, count, sizeof(int), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
      rc = 4;
  }
  chk("reloc_flatten");
  cudaFree(tmp);
  cudaFree(flags);
  return rc;
}

// reloc_energy (+ gradient at order 1, + gradient and Hessian at order 2) of
// the camera->world pose12 (host).  Synchronous; 0, 4 or 5.
int reloc_energy_derivs(cudaStream_t stream, EnergyScratch& ws, const double* centers, const double* values, int n,
                        const double* depth, int w, int h, const double* k4, double mu, const double* pose12,
                        int order, double step, double* E, double* g, double* H, long long* overlap) {
  const int P = order >= 2 ? 21 : 0;
  const int C = order == 1 ? 7 : 1 + 3 * P;
  auto grow = [&](double*& p, size_t& cap, size_t need) -> cudaError_t {
    if (need <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const cudaError_t e = cudaMalloc(&p, sizeof(double) * need);
    if (e == cudaSuccess) cap = need;
    return e;
  };
  cudaError_t e = grow(ws.terms, ws.terms_cap, static_cast<size_t>(C) * std::max(n, 1));
  if (e == cudaSuccess) e = grow(ws.small, ws.small_cap, 12 * 64 + 64 + 64);
  if (e != cudaSuccess) return 5;
  double* T = ws.small;
  double* base = ws.small + 12 * 64;
  unsigned long long* d_overlap = reinterpret_cast<unsigned long long*>(base + 16);
  cudaMemcpyAsync(base, pose12, sizeof(double) * 12, cudaMemcpyHostToDevice, stream);
  cudaMemsetAsync(d_overlap, 0, sizeof(unsigned long long), stream);
  const dim3 blk(256);
  if (order == 1) {
    launch_pdl(k_reloc_pose_l6, dim3(1), dim3(32), 0, stream, static_cast<const double*>(base), step, T);
    if (n > 0)
      launch_pdl(k_reloc_terms<L<6>>, dim3((n + 255) / 256, 1), blk, 0, stream, centers, values, n, depth, w, h, k4,
                 mu, static_cast<const double*>(T), C, ws.terms, d_overlap);
  } else if (P == 0) {
    launch_pdl(k_reloc_pose_pairs<double>, dim3(1), dim3(32), 0, stream, 0, static_cast<const double*>(base), step, T);
    if (n > 0)
      launch_pdl(k_reloc_terms<double>, dim3((n + 255) / 256, 1), blk, 0, stream, centers, values, n, depth, w, h, k4,
                 mu, static_cast<const double*>(T), C, ws.terms, d_overlap);
  } else {
    launch_pdl(k_reloc_pose_pairs<B<1>>, dim3(1), dim3(32), 0, stream, P, static_cast<const double*>(base), step, T);
    if (n > 0)
      launch_pdl(k_reloc_terms<B<1>>, dim3((n + 255) / 256, P), blk, 0, stream, centers, values, n, depth, w, h, k4,
                 mu, static_cast<const double*>(T), C, ws.terms, d_overlap);
  }
  chk("reloc_terms");
  unsigned long long ov = 0;
  if (cudaMemcpyAsync(&ov, d_overlap, sizeof(ov), cudaMemcpyDeviceToHost, stream) != cudaSuccess) return 4;
  std::vector<double> o(C);
  const int rc = tree_sum_slots(stream, ws, ws.terms, n, C, o.data());
  if (rc) return rc;
  *overlap = static_cast<long long>(ov);
  if (E) *E = o[0];
  if (order == 1 && g)
    for (int i = 0; i < 6; ++i) g[i] = o[1 + i] / step;  // extract_derivative (csfd.hpp:317)
  if (order >= 2) {
    int q = 0;
    for (int a = 0; a < 6; ++a)
      for (int b = a; b < 6; ++b, ++q) {
        if (g && a == b) g[a] = o[1 + 3 * q] / step;  // im1 of (a, a) == Complex pass a
        if (H) {
          const double hij = o[1 + 3 * q + 2] / (step * step);  // extract_hessian (csfd.hpp:319)
          H[a * 6 + b] = hij;
          H[b * 6 + a] = hij;
        }
      }
  }
  return 0;
}

// depth_cloud: world points of the valid stride pixels (host out); 0/4/5.
int depth_cloud_dev(cudaStream_t stream, const double* depth_host, int w, int h, const double* k4,
                    const double* pose12, int stride, double* out_host, int* n_out) {
  const int nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  const int n = nxs * nys;
  const size_t P = static_cast<size_t>(w) * h;
  *n_out = 0;
  if (n <= 0) return 0;
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, static_cast<int*>(nullptr), static_cast<int*>(nullptr), n);
  double* buf = nullptr;
  int* ib = nullptr;
  void* tmp = nullptr;
  if (cudaMalloc(&buf, sizeof(double) * (P + 16 + 3 * static_cast<size_t>(n))) != cudaSuccess) return 5;
  if (cudaMalloc(&ib, sizeof(int) * (2 * static_cast<size_t>(n) + 1)) != cudaSuccess ||
      cudaMalloc(&tmp, tmp_bytes) != cudaSuccess) {
    cudaFree(buf);
    if (ib) cudaFree(ib);
    return 5;
  }
  double* d_depth = buf;
  double* prm = buf + P;
  double* d_out = prm + 16;
  int* flags = ib;
  int* pos = ib + n;
  int* count = pos + n;
  double hp[16];
  std::copy(k4, k4 + 4, hp);
  std::copy(pose12, pose12 + 12, hp + 4);
  cudaMemcpyAsync(d_depth, depth_host, sizeof(double) * P, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(prm, hp, sizeof(hp), cudaMemcpyHostToDevice, stream);
  launch_pdl(k_cloud_flags, dim3((n + 255) / 256), dim3(256), 0, stream, static_cast<const double*>(d_depth), w, h,
             stride, flags);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flags, pos, n, stream);
  launch_pdl(k_cloud_scatter, dim3((n + 255) / 256), dim3(256), 0, stream, static_cast<const double*>(d_depth), w, h,
             stride, static_cast<const double*>(prm), static_cast<const int*>(flags), static_cast<const int*>(pos),
             d_out, count);
  chk("depth_cloud");
  int rc = 0;
  int cnt = 0;
  if (cudaMemcpyAsync(&cnt, count, sizeof(int), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
      cudaStreamSynchronize(stream) != cudaSuccess)
    rc = 4;
  if (!rc && cnt > 0 && out_host &&
      cudaMemcpy(out_host, d_out, sizeof(double) * 3 * cnt, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = 4;
  *n_out = cnt;
  cudaFree(tmp);
  cudaFree(ib);
  cudaFree(buf);
  return rc;
}

// eval_nn_error: mean = pairwise_sum(dist) / nq (host out); 0/4/5.
int nn_error_dev(cudaStream_t stream, EnergyScratch& ws, const double* T12, const double* q, int nq, const double* r,
                 int nr, double* mean) {
  double* buf = nullptr;
  const size_t need = 12 + 3 * static_cast<size_t>(nq) + 3 * static_cast<size_t>(nr) + static_cast<size_t>(nq);
  if (cudaMalloc(&buf, sizeof(double) * need) != cudaSuccess) return 5;
  double* d_T = buf;
  double* d_q = buf + 12;
  double* d_r = d_q + 3 * static_cast<size_t>(nq);
  double* d_dist = d_r + 3 * static_cast<size_t>(nr);
  cudaMemcpyAsync(d_T, T12, sizeof(double) * 12, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(d_q, q, sizeof(double) * 3 * nq, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(d_r, r, sizeof(double) * 3 * nr, cudaMemcpyHostToDevice, stream);
  launch_pdl(k_nn_dist, dim3((nq + kNnTile - 1) / kNnTile), dim3(kNnTile), 0, stream, static_cast<const double*>(d_T),
             static_cast<const double*>(d_q), nq, static_cast<const double*>(d_r), nr, d_dist);
  chk("nn_dist");
  double s = 0.0;
  const int rc = tree_sum_slots(stream, ws, d_dist, nq, 1, &s);
  cudaFree(buf);
  if (rc) return rc;
  *mean = s / static_cast<double>(nq);
  return 0;
}

}  // namespace csfi

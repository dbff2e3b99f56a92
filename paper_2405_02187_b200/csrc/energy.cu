// ICP energy and its CSFD derivatives on sm_100a, and the device
// correspondence list of one ICP iteration.
//
//   icp_energy<S>  — proj/include/csf/icp.hpp:70-85: E(xi) = pairwise_sum over
//                    correspondences of ((exp(xi) base v - mv) . mn)^2
//   pairwise_sum   — proj/include/csf/diff.hpp:16-37: fixed tree, leaves of
//                    <= 8 terms summed sequentially, else split at n/2
//   icp_gradient / icp_hessian — icp.cpp:128-144 via csfd_gradient /
//                    csfd_hessian (diff.hpp:46-72): 6 Complex + 21 Bicomplex
//                    passes, here ONE packed evaluation of the 21 upper-
//                    triangle pairs as B<1> channel groups (the im1 slot of
//                    pair (i, i) is bit-identical to Complex pass i,
//                    test_csfd.cpp:193-204)
//   associate      — icp.cpp:89-126, materialised in scan order (flags, CUB
//                    exclusive scan, scatter) for the solvers that need the
//                    correspondence list (Newton, gradient descent, NCG, and
//                    the linearized solver's loss_after)
//
// The tree is evaluated exactly in parallel: every node above depth d0 is
// internal (its size exceeds 8), so the 2^d0 depth-d0 subtrees (33..64 terms
// each) are summed independently (recursively, one thread each) and combined
// pairwise level by level in aligned 1024-node CTA reductions — the same
// additions, in the same association, as the recursion.
// The Newton / gradient trackers turn these derivative channels into the
// real pose step, so this translation unit evaluates every channel division
// as the reference's per-channel quotient (csfd.hpp:57, 114-121) — the real
// track stays bit-identical to the CPU oracle.  (Device code is not linked
// across translation units, so the define is local to these kernels.)
#define CSF_EXACT_CHANNELS 1
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "csf_internal.h"
#include "geometry.cuh"

namespace csfd {

// diff.hpp:18-28
__device__ double pw_block(const double* x, int n) {
  if (n <= 8) {
    double acc = x[0];
    for (int k = 1; k < n; ++k) acc = acc + x[k];
    return acc;
  }
  const int half = n / 2;
  return pw_block(x, half) + pw_block(x + half, n - half);
}

// Lifted pose exp(xi) * base per pair (csfd_hessian seeds: im1 on pair_i,
// im2 on pair_j), or the real pose (S = double).  T: [12][C] packed.
template <typename S>
__global__ void k_energy_pose(const int* __restrict__ pair_i, const int* __restrict__ pair_j, int P,
                              const double* __restrict__ base, const double* __restrict__ xi0, double h, double* T) {
  pdl_wait();
  pdl_trigger();
  constexpr int G = Traits<S>::G;
  const int p = threadIdx.x;
  if (p >= (P > 0 ? P : 1)) return;
  const int C = 1 + 3 * P;
  S xi[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) xi[k] = lit<S>(xi0[k]);
  if constexpr (G > 0) {
    xi[pair_i[p]].im[0] = h;
    xi[pair_j[p]].im[1] = h;
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

// One term r^2 per (correspondence, pair); terms [C][n] slot-major.
template <typename S>
__global__ void k_energy_terms(const double* __restrict__ corrs, int n, const double* __restrict__ T, int P,
                               double* __restrict__ terms) {
  pdl_wait();
  pdl_trigger();
  constexpr int G = Traits<S>::G;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = blockIdx.y;
  if (i >= n) return;
  const int C = 1 + 3 * P;
  Pose<S> pose;
#pragma unroll
  for (int e = 0; e < 9; ++e) pose.R.m[e] = load_ch<S>(T + e * C, 3 * p, G);
#pragma unroll
  for (int e = 0; e < 3; ++e) pose.t.v[e] = load_ch<S>(T + (9 + e) * C, 3 * p, G);
  const double* c = corrs + 9LL * i;
  const V3<S> v = mk3<S>(lit<S>(c[0]), lit<S>(c[1]), lit<S>(c[2]));
  const V3<S> mv = mk3<S>(lit<S>(c[3]), lit<S>(c[4]), lit<S>(c[5]));
  const V3<S> mn = mk3<S>(lit<S>(c[6]), lit<S>(c[7]), lit<S>(c[8]));
  const S r = dot3(sub3(apply(pose, v), mv), mn);
  const S t = r * r;
  if (p == 0) terms[i] = re(t);
  if constexpr (G > 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) terms[static_cast<long long>(1 + 3 * p + g) * n + i] = t.im[g];
  }
}

// Depth-d0 subtrees of pairwise_block, one thread each: sub [C][2^d0].
__global__ void k_tree_sub(const double* __restrict__ terms, int n, int d0, double* __restrict__ sub) {
  pdl_wait();
  pdl_trigger();
  const int nsub = 1 << d0;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int slot = blockIdx.y;
  if (t >= nsub) return;
  int s = 0, m = n;
  for (int lv = 0; lv < d0; ++lv) {
    const int half = m / 2;
    if ((t >> (d0 - 1 - lv)) & 1) {
      s += half;
      m -= half;
    } else {
      m = half;
    }
  }
  sub[static_cast<long long>(slot) * nsub + t] = pw_block(terms + static_cast<long long>(slot) * n + s, m);
}

// Internal nodes above depth d0 (each has exactly two children): combine
// left + right level by level.  One CTA reduces r = 2^k consecutive nodes of
// one slot (a complete, aligned subtree) to one; `last` adds the result to
// pairwise_sum's init = 0.  in [C][m], out [C][m / r].
__global__ void __launch_bounds__(512) k_tree_top(const double* __restrict__ in, int m, int r, int last,
                                                  double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ double v[1024];
  const int slot = blockIdx.y;
  const double* src = in + static_cast<long long>(slot) * m + static_cast<long long>(blockIdx.x) * r;
  for (int k = threadIdx.x; k < r; k += blockDim.x) v[k] = src[k];
  __syncthreads();
  for (int w = r; w > 1; w >>= 1) {
    double a = 0.0;
    const int k = threadIdx.x;
    if (k < w / 2) a = v[2 * k] + v[2 * k + 1];
    __syncthreads();
    if (k < w / 2) v[k] = a;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[static_cast<long long>(slot) * (m / r) + blockIdx.x] = last ? 0.0 + v[0] : v[0];
}

// ---------------------------------------------------------------------------
// correspondence list (associate, icp.cpp:89-126) in scan order
// ---------------------------------------------------------------------------
__global__ void k_assoc_flags(const double* __restrict__ depth, int w, int h, int stride,
                              const double* __restrict__ intr /*fx fy cx cy*/, const double* __restrict__ pose,
                              const double* __restrict__ pred_w2c, const double* __restrict__ vre,
                              const double* __restrict__ nre, double d_max, double cos_max, int* __restrict__ flags,
                              int* __restrict__ uv) {
  pdl_wait();
  pdl_trigger();
  const int nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= nxs * nys) return;
  Pose<double> c2w, w2p;
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    c2w.R.m[e] = pose[e];
    w2p.R.m[e] = pred_w2c[e];
  }
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    c2w.t.v[e] = pose[9 + e];
    w2p.t.v[e] = pred_w2c[9 + e];
  }
  const int x = (slot % nxs) * stride, y = (slot / nxs) * stride;
  int u = 0, v = 0;
  const bool corr =
      associate_slot(depth, w, h, x, y, intr[0], intr[1], intr[2], intr[3], c2w, w2p, vre, nre, d_max, cos_max, &u, &v);
  flags[slot] = corr ? 1 : 0;
  uv[slot] = corr ? v * w + u : -1;
}

// corrs [n][9]: measured vertex (camera), model vertex, model normal (world)
__global__ void k_assoc_scatter(const double* __restrict__ depth, int w, int stride, int n_slots,
                                const double* __restrict__ intr, const int* __restrict__ flags,
                                const int* __restrict__ pos, const int* __restrict__ uv,
                                const double* __restrict__ vre, const double* __restrict__ nre,
                                double* __restrict__ corrs, int* __restrict__ count) {
  pdl_wait();
  pdl_trigger();
  const int nxs = (w + stride - 1) / stride;
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= n_slots) return;
  if (slot == n_slots - 1) *count = pos[slot] + flags[slot];
  if (!flags[slot]) return;
  const int x = (slot % nxs) * stride, y = (slot / nxs) * stride;
  const double d = depth[y * w + x];
  double* c = corrs + 9LL * pos[slot];
  c[0] = d * (static_cast<double>(x) - intr[2]) / intr[0];
  c[1] = d * (static_cast<double>(y) - intr[3]) / intr[1];
  c[2] = d;
  const long long m = uv[slot];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c[3 + k] = vre[3 * m + k];
    c[6 + k] = nre[3 * m + k];
  }
}

// associate (icp.cpp:89-126) over given measured / predicted maps (the
// reference's signature): gates in the reference's order, scan-order list.
__global__ void k_assoc_maps_flags(const double* __restrict__ mvert, const double* __restrict__ mnorm,
                                   const double* __restrict__ pvert, const double* __restrict__ pnorm, int w, int h,
                                   int stride, const double* __restrict__ prm /*c2w[12], w2p[12], k[4]*/,
                                   double d_max, double cos_max, int* __restrict__ flags, int* __restrict__ uv) {
  pdl_wait();
  pdl_trigger();
  const int nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= nxs * nys) return;
  const int x = (slot % nxs) * stride, y = (slot / nxs) * stride;
  const long long i = static_cast<long long>(y) * w + x;
  flags[slot] = 0;
  uv[slot] = -1;
  const V3<double> vert = mk3<double>(mvert[3 * i], mvert[3 * i + 1], mvert[3 * i + 2]);
  const V3<double> nrm = mk3<double>(mnorm[3 * i], mnorm[3 * i + 1], mnorm[3 * i + 2]);
  if (!(vert.v[2] > 0.0) || !(dot3(nrm, nrm) > 0.5)) return;  // vertex_valid, normal_valid (frames.hpp:73-81)
  Pose<double> c2w, w2p;
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    c2w.R.m[e] = prm[e];
    w2p.R.m[e] = prm[12 + e];
  }
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    c2w.t.v[e] = prm[9 + e];
    w2p.t.v[e] = prm[21 + e];
  }
  const double fx = prm[24], fy = prm[25], cx = prm[26], cy = prm[27];
  const V3<double> world = apply(c2w, vert);
  const V3<double> inp = apply(w2p, world);
  if (!(inp.v[2] > 0.0)) return;
  const int u = static_cast<int>(lround((fx * inp.v[0]) / inp.v[2] + cx));
  const int v = static_cast<int>(lround((fy * inp.v[1]) / inp.v[2] + cy));
  if (!(u >= 0 && u < w && v >= 0 && v < h)) return;
  const long long m = static_cast<long long>(v) * w + u;
  const V3<double> mn = mk3<double>(pnorm[3 * m], pnorm[3 * m + 1], pnorm[3 * m + 2]);
  if (!(dot3(mn, mn) > 0.5)) return;
  const V3<double> mv = mk3<double>(pvert[3 * m], pvert[3 * m + 1], pvert[3 * m + 2]);
  const V3<double> dd = sub3(world, mv);
  if (sqrt(dot3(dd, dd)) > d_max) return;
  const V3<double> wn = matvec(c2w.R, nrm);
  if (dot3(wn, mn) < cos_max) return;
  flags[slot] = 1;
  uv[slot] = static_cast<int>(m);
}

__global__ void k_assoc_maps_scatter(const double* __restrict__ mvert, const double* __restrict__ pvert,
                                     const double* __restrict__ pnorm, int w, int stride, int n_slots,
                                     const int* __restrict__ flags, const int* __restrict__ pos,
                                     const int* __restrict__ uv, double* __restrict__ corrs, int* __restrict__ count) {
  pdl_wait();
  pdl_trigger();
  const int nxs = (w + stride - 1) / stride;
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= n_slots) return;
  if (slot == n_slots - 1) *count = pos[slot] + flags[slot];
  if (!flags[slot]) return;
  const long long i = static_cast<long long>((slot / nxs) * stride) * w + (slot % nxs) * stride;
  const long long m = uv[slot];
  double* c = corrs + 9LL * pos[slot];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c[k] = mvert[3 * i + k];
    c[3 + k] = pvert[3 * m + k];
    c[6 + k] = pnorm[3 * m + k];
  }
}

// Per-tile normal-equation sums over a correspondence list (the oracle's
// canonical normal_equations(corrs, base, false): tiles of 256
// correspondences summed sequentially); out [tiles][27].
__global__ void __launch_bounds__(256) k_lin_tiles(const double* __restrict__ corrs, int n,
                                                   const double* __restrict__ base, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ double rows[256][7];
  const int i = blockIdx.x * 256 + threadIdx.x;
  const int cnt = min(256, n - static_cast<int>(blockIdx.x) * 256);
  if (static_cast<int>(threadIdx.x) < cnt) {
    Pose<double> b;
#pragma unroll
    for (int e = 0; e < 9; ++e) b.R.m[e] = base[e];
#pragma unroll
    for (int e = 0; e < 3; ++e) b.t.v[e] = base[9 + e];
    const double* c = corrs + 9LL * i;
    const V3<double> p = apply(b, mk3<double>(c[0], c[1], c[2]));
    const V3<double> mv = mk3<double>(c[3], c[4], c[5]), mn = mk3<double>(c[6], c[7], c[8]);
    const double r = dot3(sub3(p, mv), mn);
    const V3<double> pn = cross3(p, mn);
    rows[threadIdx.x][0] = mn.v[0]; rows[threadIdx.x][1] = mn.v[1]; rows[threadIdx.x][2] = mn.v[2];
    rows[threadIdx.x][3] = pn.v[0]; rows[threadIdx.x][4] = pn.v[1]; rows[threadIdx.x][5] = pn.v[2];
    rows[threadIdx.x][6] = r;
  }
  __syncthreads();
  const int a = threadIdx.x;
  if (a < 27) {
    int ja, jb;
    if (a < 21) {
      int r = 0;
      while ((r + 1) * (r + 2) / 2 <= a) ++r;
      ja = r;
      jb = a - r * (r + 1) / 2;
    } else {
      ja = a - 21;
      jb = 6;
    }
    double s = 0.0;
    for (int e = 0; e < cnt; ++e) s = s + rows[e][ja] * rows[e][jb];
    out[static_cast<long long>(blockIdx.x) * 27 + a] = s;
  }
}

}  // namespace csfd

// ============================================================================
namespace csfi {

using namespace csfd;

static void chk(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) note_launch_error(what, e);
}

// pairwise_sum (diff.hpp:16-37) of every slot of terms [C][n] (n > 0) into
// out [C] (device).  Depth d0 is chosen so every depth-d0 subtree holds
// 33..64 terms (all nodes above are internal: their size exceeds 8), giving
// 2^d0 independent subtree sums per slot — enough threads to stream the
// terms at HBM rate — then aligned 1024-node CTA reductions to the root.
// sub: scratch of tree_scratch_doubles(n, C).
static int tree_depth(int n) {
  int d0 = 0;
  while (d0 < 20 && (n >> d0) > 64) ++d0;
  return d0;
}
static size_t tree_scratch_doubles(int n, int C) {
  const size_t nsub = size_t(1) << tree_depth(n);
  return static_cast<size_t>(C) * (nsub + nsub / 1024 + 1);
}
static void launch_tree(cudaStream_t stream, const double* terms, int n, int C, double* sub, double* out) {
  const int d0 = tree_depth(n);
  const int nsub = 1 << d0;
  launch_pdl(k_tree_sub, dim3((nsub + 127) / 128, C), dim3(128), 0, stream, terms, n, d0, sub);
  if (nsub <= 1024) {
    launch_pdl(k_tree_top, dim3(1, C), dim3(512), 0, stream, static_cast<const double*>(sub), nsub, nsub, 1, out);
  } else {
    double* mid = sub + static_cast<size_t>(C) * nsub;
    launch_pdl(k_tree_top, dim3(nsub / 1024, C), dim3(512), 0, stream, static_cast<const double*>(sub), nsub, 1024, 0,
               mid);
    const int m = nsub / 1024;
    launch_pdl(k_tree_top, dim3(1, C), dim3(512), 0, stream, static_cast<const double*>(mid), m, m, 1, out);
  }
}

// Energy (and, for order > 0, the 21-pair CSFD derivatives) of n device
// correspondences.  order 0: energy only; 1: + gradient (6 diagonal pairs);
// 2: + Hessian (21 pairs).  Scratch is grown in `ws`.  Synchronous: results
// land in E, g[6], H[36] (host).
int icp_energy_derivs(cudaStream_t stream, EnergyScratch& ws, const double* corrs, int n, const double* base,
                      const double* xi, double h, int order, double* E, double* g, double* H) {
  int pi[21], pj[21], P = 0;
  if (order == 1) {
    for (int i = 0; i < 6; ++i) {
      pi[P] = i;
      pj[P] = i;
      ++P;
    }
  } else if (order >= 2) {
    for (int i = 0; i < 6; ++i)
      for (int j = i; j < 6; ++j) {
        pi[P] = i;
        pj[P] = j;
        ++P;
      }
  }
  const int C = 1 + 3 * P;
  if (n <= 0) {  // pairwise_sum of no terms = init
    if (E) *E = 0.0;
    if (g) std::fill(g, g + 6, 0.0);
    if (H) std::fill(H, H + 36, 0.0);
    return 0;
  }
  auto grow = [&](double*& p, size_t& cap, size_t need) -> cudaError_t {
    if (need <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    cap = 0;
    const cudaError_t e = cudaMalloc(&p, sizeof(double) * need);
    if (e == cudaSuccess) cap = need;
    return e;
  };
  cudaError_t e = grow(ws.terms, ws.terms_cap, static_cast<size_t>(C) * n);
  if (e == cudaSuccess) e = grow(ws.sub, ws.sub_cap, tree_scratch_doubles(n, C));
  if (e == cudaSuccess) e = grow(ws.small, ws.small_cap, 12 * 64 + 64 + 64);
  if (e == cudaSuccess && !ws.pairs) e = cudaMalloc(&ws.pairs, sizeof(int) * 64);
  if (e != cudaSuccess) return 5;
  double* T = ws.small;
  double* out = ws.small + 12 * 64;
  double* params = out + 64;  // base[12], xi[6]
  double hp[18];
  std::copy(base, base + 12, hp);
  for (int k = 0; k < 6; ++k) hp[12 + k] = xi ? xi[k] : 0.0;
  int pp[64];
  for (int k = 0; k < P; ++k) {
    pp[k] = pi[k];
    pp[32 + k] = pj[k];
  }
  cudaMemcpyAsync(params, hp, sizeof(hp), cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(ws.pairs, pp, sizeof(pp), cudaMemcpyHostToDevice, stream);
  if (P == 0) {
    launch_pdl(k_energy_pose<double>, dim3(1), dim3(32), 0, stream, static_cast<const int*>(ws.pairs),
               static_cast<const int*>(ws.pairs + 32), 0, static_cast<const double*>(params),
               static_cast<const double*>(params + 12), h, T);
    launch_pdl(k_energy_terms<double>, dim3((n + 127) / 128, 1), dim3(128), 0, stream, corrs, n,
               static_cast<const double*>(T), 0, ws.terms);
  } else {
    launch_pdl(k_energy_pose<B<1>>, dim3(1), dim3(32), 0, stream, static_cast<const int*>(ws.pairs),
               static_cast<const int*>(ws.pairs + 32), P, static_cast<const double*>(params),
               static_cast<const double*>(params + 12), h, T);
    launch_pdl(k_energy_terms<B<1>>, dim3((n + 127) / 128, P), dim3(128), 0, stream, corrs, n,
               static_cast<const double*>(T), P, ws.terms);
  }
  launch_tree(stream, static_cast<const double*>(ws.terms), n, C, ws.sub, out);
  chk("icp_energy");
  std::vector<double> o(C);
  e = cudaMemcpyAsync(o.data(), out, sizeof(double) * C, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return 4;
  if (E) *E = o[0];
  if (g && P > 0) {
    // gradient: im1 of the diagonal pair (i, i) == Complex pass i
    for (int q = 0; q < P; ++q)
      if (pi[q] == pj[q]) g[pi[q]] = o[1 + 3 * q] / h;  // extract_derivative, csfd.hpp:317
  }
  if (H && order >= 2) {
    for (int q = 0; q < P; ++q) {
      const double hij = o[1 + 3 * q + 2] / (h * h);  // extract_hessian, csfd.hpp:319
      H[pi[q] * 6 + pj[q]] = hij;
      H[pj[q] * 6 + pi[q]] = hij;
    }
  }
  return 0;
}

// pairwise_sum (diff.hpp:16-37) of every slot of terms [C][n] (device) into
// out_host[C]; synchronous.  Returns 0, 4 or 5 like icp_energy_derivs.
int tree_sum_slots(cudaStream_t stream, EnergyScratch& ws, const double* terms, int n, int C, double* out_host) {
  if (n <= 0) {
    std::fill(out_host, out_host + C, 0.0);
    return 0;
  }
  const size_t need = tree_scratch_doubles(n, C);
  if (ws.sub_cap < need || !ws.sub) {
    if (ws.sub) cudaFree(ws.sub);
    ws.sub = nullptr;
    ws.sub_cap = 0;
    if (cudaMalloc(&ws.sub, sizeof(double) * need) != cudaSuccess) return 5;
    ws.sub_cap = need;
  }
  if (ws.out_cap < static_cast<size_t>(C) || !ws.out) {
    if (ws.out) cudaFree(ws.out);
    ws.out = nullptr;
    ws.out_cap = 0;
    if (cudaMalloc(&ws.out, sizeof(double) * C) != cudaSuccess) return 5;
    ws.out_cap = static_cast<size_t>(C);
  }
  double* out = ws.out;
  launch_tree(stream, terms, n, C, ws.sub, out);
  chk("tree_sum");
  if (cudaMemcpyAsync(out_host, out, sizeof(double) * C, cudaMemcpyDeviceToHost, stream) != cudaSuccess) return 4;
  if (cudaStreamSynchronize(stream) != cudaSuccess) return 4;
  return 0;
}

void energy_scratch_release(EnergyScratch& ws) {
  if (ws.terms) cudaFree(ws.terms);
  if (ws.sub) cudaFree(ws.sub);
  if (ws.small) cudaFree(ws.small);
  if (ws.pairs) cudaFree(ws.pairs);
  if (ws.corrs) cudaFree(ws.corrs);
  if (ws.flags) cudaFree(ws.flags);
  if (ws.cub) cudaFree(ws.cub);
  if (ws.out) cudaFree(ws.out);
  ws = EnergyScratch{};
}

// associate -> corrs [n][9] in scan order; returns the count (synchronous).
int associate_list(cudaStream_t stream, EnergyScratch& ws, const double* depth, int w, int h, int stride,
                   const double* intr4, const double* pose12, const double* pred_w2c12, const double* vre,
                   const double* nre, double d_max, double cos_max, int* n_out) {
  const int nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  const int n_slots = nxs * nys;
  if (n_slots <= 0) {
    *n_out = 0;
    return 0;
  }
  const size_t need = static_cast<size_t>(n_slots);
  if (ws.flags_cap < need) {
    if (ws.flags) cudaFree(ws.flags);
    if (ws.corrs) cudaFree(ws.corrs);
    if (ws.cub) cudaFree(ws.cub);
    ws.flags = nullptr;
    ws.corrs = nullptr;
    ws.cub = nullptr;
    ws.flags_cap = 0;
    size_t cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, static_cast<int*>(nullptr), static_cast<int*>(nullptr),
                                  static_cast<int>(need));
    if (cudaMalloc(&ws.flags, sizeof(int) * (3 * need + 4)) != cudaSuccess ||
        cudaMalloc(&ws.corrs, sizeof(double) * 9 * need) != cudaSuccess ||
        cudaMalloc(&ws.cub, cub_bytes) != cudaSuccess)
      return 5;
    ws.cub_bytes = cub_bytes;
    ws.flags_cap = need;
  }
  int* flags = ws.flags;
  int* pos = flags + need;
  int* uv = pos + need;
  int* count = uv + need;
  launch_pdl(k_assoc_flags, dim3((n_slots + 127) / 128), dim3(128), 0, stream, depth, w, h, stride, intr4, pose12,
             pred_w2c12, vre, nre, d_max, cos_max, flags, uv);
  size_t bytes = ws.cub_bytes;
  cub::DeviceScan::ExclusiveSum(ws.cub, bytes, flags, pos, n_slots, stream);
  launch_pdl(k_assoc_scatter, dim3((n_slots + 127) / 128), dim3(128), 0, stream, depth, w, stride, n_slots, intr4,
             static_cast<const int*>(flags), static_cast<const int*>(pos), static_cast<const int*>(uv), vre, nre,
             ws.corrs, count);
  chk("associate_list");
  if (cudaMemcpyAsync(n_out, count, sizeof(int), cudaMemcpyDeviceToHost, stream) != cudaSuccess) return 4;
  if (cudaStreamSynchronize(stream) != cudaSuccess) return 4;
  return 0;
}

// associate over host maps -> host corrs (synchronous); returns 0/4/5
int associate_maps(cudaStream_t stream, EnergyScratch& ws, const double* mvert, const double* mnorm,
                   const double* pvert, const double* pnorm, int w, int h, int stride, const double* prm28,
                   double d_max, double cos_max, double* corrs_out, int* n_out) {
  const int nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  const int n_slots = nxs * nys;
  const size_t P = static_cast<size_t>(w) * h;
  double* dm = nullptr;
  if (cudaMalloc(&dm, sizeof(double) * (12 * P + 28)) != cudaSuccess) return 5;
  double* d_mv = dm;
  double* d_mn = dm + 3 * P;
  double* d_pv = dm + 6 * P;
  double* d_pn = dm + 9 * P;
  double* d_prm = dm + 12 * P;
  cudaMemcpyAsync(d_mv, mvert, sizeof(double) * 3 * P, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(d_mn, mnorm, sizeof(double) * 3 * P, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(d_pv, pvert, sizeof(double) * 3 * P, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(d_pn, pnorm, sizeof(double) * 3 * P, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(d_prm, prm28, sizeof(double) * 28, cudaMemcpyHostToDevice, stream);
  int rc = 0;
  const size_t need = static_cast<size_t>(std::max(n_slots, 1));
  if (ws.flags_cap < need) {
    if (ws.flags) cudaFree(ws.flags);
    if (ws.corrs) cudaFree(ws.corrs);
    if (ws.cub) cudaFree(ws.cub);
    ws.flags = nullptr;
    ws.corrs = nullptr;
    ws.cub = nullptr;
    ws.flags_cap = 0;
    size_t cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, static_cast<int*>(nullptr), static_cast<int*>(nullptr),
                                  static_cast<int>(need));
    if (cudaMalloc(&ws.flags, sizeof(int) * (3 * need + 4)) != cudaSuccess ||
        cudaMalloc(&ws.corrs, sizeof(double) * 9 * need) != cudaSuccess ||
        cudaMalloc(&ws.cub, cub_bytes) != cudaSuccess)
      rc = 5;
    ws.cub_bytes = cub_bytes;
    ws.flags_cap = need;
  }
  int n = 0;
  if (!rc && n_slots > 0) {
    int* flags = ws.flags;
    int* pos = flags + need;
    int* uv = pos + need;
    int* count = uv + need;
    launch_pdl(k_assoc_maps_flags, dim3((n_slots + 127) / 128), dim3(128), 0, stream, static_cast<const double*>(d_mv),
               static_cast<const double*>(d_mn), static_cast<const double*>(d_pv), static_cast<const double*>(d_pn), w,
               h, stride, static_cast<const double*>(d_prm), d_max, cos_max, flags, uv);
    size_t bytes = ws.cub_bytes;
    cub::DeviceScan::ExclusiveSum(ws.cub, bytes, flags, pos, n_slots, stream);
    launch_pdl(k_assoc_maps_scatter, dim3((n_slots + 127) / 128), dim3(128), 0, stream,
               static_cast<const double*>(d_mv), static_cast<const double*>(d_pv), static_cast<const double*>(d_pn), w,
               stride, n_slots, static_cast<const int*>(flags), static_cast<const int*>(pos),
               static_cast<const int*>(uv), ws.corrs, count);
    if (cudaMemcpyAsync(&n, count, sizeof(int), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
      rc = 4;
    if (!rc && n > 0 &&
        cudaMemcpy(corrs_out, ws.corrs, sizeof(double) * 9 * n, cudaMemcpyDeviceToHost) != cudaSuccess)
      rc = 4;
  }
  cudaStreamSynchronize(stream);
  cudaFree(dm);
  *n_out = n;
  return rc;
}

// Tile partials [tiles][27] of the canonical normal equations over n device
// correspondences (synchronous, to the host).
int linearized_tiles(cudaStream_t stream, const double* corrs, int n, const double* base12, double* tiles_out) {
  const int tiles = (n + 255) / 256;
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(double) * (static_cast<size_t>(tiles) * 27 + 12)) != cudaSuccess) return 5;
  double* d_base = d + static_cast<size_t>(tiles) * 27;
  cudaMemcpyAsync(d_base, base12, sizeof(double) * 12, cudaMemcpyHostToDevice, stream);
  if (tiles > 0)
    launch_pdl(k_lin_tiles, dim3(tiles), dim3(256), 0, stream, corrs, n, static_cast<const double*>(d_base), d);
  int rc = 0;
  if (cudaMemcpyAsync(tiles_out, d, sizeof(double) * static_cast<size_t>(tiles) * 27, cudaMemcpyDeviceToHost,
                      stream) != cudaSuccess ||
      cudaStreamSynchronize(stream) != cudaSuccess)
    rc = 4;
  cudaFree(d);
  return rc;
}

}  // namespace csfi

// Lifted point-to-plane ICP for sm_100a.
//
//   associate          — proj/src/icp.cpp:89-126 (real-part gates, scan order)
//   normal_equations   — proj/src/icp.cpp:15-28 (J = [n; p x n], r), lifted
//   LDLT solve         — Eigen::LDLT<Mat6d>(a).solve(-b), icp.cpp:43,151
//   apply_increment    — proj/include/csf/se3.hpp:116-119
//   track_frame loop   — proj/src/icp.cpp:185-240 (break rules)
//
// One ICP iteration is two launches:
//   k_icp_reduce: one CTA per tile of 256 slots (the strided pixel grid in
//     row-major order).  Measured vertex/normal are recomputed from the
//     pyramid depth, gated on real parts, compacted in slot order into shared
//     memory as lifted (J, r) rows, and summed sequentially per accumulator —
//     the canonical "slot-tiled" order the oracle restates.
//   k_icp_solve: one CTA sums the tile partials in tile order, then one
//     thread per channel group runs the 6x6 LDLT, the exp map and the pose
//     update in L<G> arithmetic.  Break decisions are written to TrackState so
//     the whole level stays on the device (no host round trip).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "csf_internal.h"
#include "geometry.cuh"

namespace csfd {

using csfi::TrackState;
constexpr int kTile = 256;

// Optional phase timing (tools/icp_timing.py): per launch, per CTA
// [start, after association/J, after sums, solve start, solve end] in ns.
__device__ unsigned long long* g_icp_clock = nullptr;
__device__ unsigned g_icp_clock_launch = 0;
CSF_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
CSF_DEV void clock_mark(int slot, int cta = -1) {
  if (g_icp_clock && threadIdx.x == 0 && g_icp_clock_launch < 4096)
    g_icp_clock[(static_cast<unsigned long long>(g_icp_clock_launch) * 512 + (cta < 0 ? blockIdx.x : cta)) * 8 + slot] =
        gtimer();
}
// the solve kernel records into CTA slot 511 of the iteration's record
constexpr int kSolveClockCta = 511;

// 256 threads evaluate the tile's slots; all 320 sum accumulators (27*(1+Dp)
// of them, one per thread up to Dp = 10), so no thread carries two.
constexpr int kRedThreads = 320;
__constant__ int c_tri_r[21] = {0, 1, 1, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 4, 5, 5, 5, 5, 5, 5};
__constant__ int c_tri_c[21] = {0, 0, 1, 0, 1, 2, 0, 1, 2, 3, 0, 1, 2, 3, 4, 0, 1, 2, 3, 4, 5};

CSF_DEV void load_pose_real(const double* p, int C, Pose<double>* out) {
#pragma unroll
  for (int e = 0; e < 9; ++e) out->R.m[e] = p[e * C];
#pragma unroll
  for (int e = 0; e < 3; ++e) out->t.v[e] = p[(9 + e) * C];
}



// Canonical two-level cross-tile order (oracle/orc_icp.hpp, kGroup): the
// last CTA to finish within a group of kGroup consecutive tiles sums the
// group's tile partials in tile order into gpartials[group]; the solve then
// sums the (few) group totals in group order.  Called by every CTA after it
// wrote its own tile partials.
constexpr int kGroup = 16;
constexpr int kMaxGroupCtr = 256;  // tiles per launch <= kGroup * kMaxGroupCtr
CSF_DEV bool group_sum(const double* __restrict__ partials, const int* __restrict__ counts, int n_acc,
                       double* __restrict__ gpartials, int* __restrict__ gcounts, unsigned* __restrict__ group_ctr) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  const int grp = blockIdx.x / kGroup;
  const int first = grp * kGroup;
  const int gn = min(kGroup, static_cast<int>(gridDim.x) - first);
  if (threadIdx.x == 0) s_last = atomicAdd(group_ctr + grp, 1u) == static_cast<unsigned>(gn - 1);
  __syncthreads();
  if (!s_last) return false;
  if (threadIdx.x == 0) group_ctr[grp] = 0u;  // ready for the next launch
  __threadfence();
  for (int a = threadIdx.x; a < n_acc; a += blockDim.x) {
    double v[kGroup];
#pragma unroll
    for (int u = 0; u < kGroup; ++u)
      v[u] = u < gn ? __ldcg(partials + static_cast<long long>(first + u) * n_acc + a) : 0.0;
    double total = 0.0;
#pragma unroll
    for (int u = 0; u < kGroup; ++u)
      if (u < gn) total = total + v[u];
    gpartials[static_cast<long long>(grp) * n_acc + a] = total;
  }
  if (threadIdx.x < 32) {
    int c = static_cast<int>(threadIdx.x) < gn ? __ldcg(counts + first + threadIdx.x) : 0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_down_sync(0xffffffffu, c, off);
    if (threadIdx.x == 0) gcounts[grp] = c;
  }
  return true;
}

// The solve of one ICP iteration (one CTA): group totals in group order, then
// the real 6x6 LDLT once (thread 0, the oracle's Ldlt6 order, bit-identical
// real step) and every perturbation channel in tangent form against the real
// factors, d.im = A^-1 (nb.im - A.im d.re) — the first-order quantity the
// truncated-Complex LDLT computes, ~1 ulp per operation apart.  Degenerate
// systems (zero or sub-normal pivots) take the per-channel lifted LDLT
// instead.  Then exp(delta) * T per channel thread (L<1>) and the break
// decisions (icp.cpp:199,235) into TrackState.
constexpr int kMaxC = 1 + 64;  // CSF_MAX_DIRECTIONS
__device__ __noinline__ void icp_solve_body(TrackState* st, const double* __restrict__ gpartials,
                                            const int* __restrict__ gcounts, int n_groups, double* pose, int Dp,
                                            int level, double tol) {
  __shared__ double s_acc[27 * kMaxC];
  __shared__ double s_m[36], s_x[6];
  __shared__ int s_tr[6];
  __shared__ int s_n, s_degen, s_finite;
  const int C = 1 + Dp;
  const int n_acc = 27 * C;
  clock_mark(3, kSolveClockCta);
  for (int a = threadIdx.x; a < n_acc; a += blockDim.x) {
    double v[32];
    double total = 0.0;
    for (int g0 = 0; g0 < n_groups; g0 += 32) {
#pragma unroll
      for (int u = 0; u < 32; ++u)
        v[u] = g0 + u < n_groups ? __ldcg(gpartials + static_cast<long long>(g0 + u) * n_acc + a) : 0.0;
#pragma unroll
      for (int u = 0; u < 32; ++u)
        if (g0 + u < n_groups) total = total + v[u];
    }
    s_acc[a] = total;
  }
  if (threadIdx.x < 32) {
    int c = 0;
    for (int g = threadIdx.x; g < n_groups; g += 32) c += __ldcg(gcounts + g);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_down_sync(0xffffffffu, c, off);
    if (threadIdx.x == 0) {
      s_n = c;
      s_finite = 1;
    }
  }
  __syncthreads();
  clock_mark(5, kSolveClockCta);
  const int n = s_n;
  if (n < 12) {
    if (threadIdx.x == 0) {
      st->n_corr = n;
      st->level_done = 1;
      if (g_icp_clock) atomicAdd(&g_icp_clock_launch, 1u);
    }
    return;
  }
  if (threadIdx.x == 0) {
    double a[21], nb[6], m[6][6], x[6];
    int tr[6];
#pragma unroll
    for (int q = 0; q < 21; ++q) a[q] = s_acc[q * C];
#pragma unroll
    for (int i = 0; i < 6; ++i) nb[i] = -s_acc[(21 + i) * C];
    bool degen = false;
    ldlt6_factor_reg<double>(a, m, tr, &degen);
    ldlt6_apply_reg<double>(m, tr, nb, x);
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
      for (int c = 0; c < 6; ++c) s_m[6 * r + c] = m[r][c];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      s_tr[i] = tr[i];
      s_x[i] = x[i];
    }
    s_degen = degen;
  }
  __syncthreads();
  clock_mark(6, kSolveClockCta);
  // channel threads: thread t < max(Dp, 1) owns channel t (thread 0 also the real part)
  const bool mine = static_cast<int>(threadIdx.x) < (Dp > 0 ? Dp : 1);
  L<1> d[6];
  if (mine) {
    const int ch = 1 + threadIdx.x;
    if (Dp == 0) {
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        d[i].re = s_x[i];
        d[i].im[0] = 0.0;
      }
    } else if (!s_degen) {
      double m[6][6];
      int tr[6];
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c < 6; ++c) m[r][c] = s_m[6 * r + c];
#pragma unroll
      for (int i = 0; i < 6; ++i) tr[i] = s_tr[i];
      double rhs[6], dx[6];
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        double ax = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) ax = ax + s_acc[(i >= j ? tri(i, j) : tri(j, i)) * C + ch] * s_x[j];
        rhs[i] = -s_acc[(21 + i) * C + ch] - ax;
      }
      ldlt6_apply_reg<double>(m, tr, rhs, dx);
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        d[i].re = s_x[i];
        d[i].im[0] = dx[i];
      }
    } else {
      L<1> a[21], nb[6];
#pragma unroll
      for (int q = 0; q < 21; ++q) a[q] = load_ch<L<1>>(s_acc + q * C, threadIdx.x, 1);
#pragma unroll
      for (int i = 0; i < 6; ++i) nb[i] = -load_ch<L<1>>(s_acc + (21 + i) * C, threadIdx.x, 1);
      ldlt6_solve_reg<L<1>>(a, nb, d);
    }
    bool fin = true;
#pragma unroll
    for (int i = 0; i < 6; ++i) fin = fin && finite_s(d[i]);
    if (!fin) atomicAnd(&s_finite, 0);
  }
  __syncthreads();
  clock_mark(7, kSolveClockCta);
  Pose<L<1>> np;
  if (mine) {
    if (!s_finite)
#pragma unroll
      for (int i = 0; i < 6; ++i) d[i] = lit<L<1>>(0.0);
    const int g0 = Dp > 0 ? static_cast<int>(threadIdx.x) : 0;
    const int nv = Dp > 0 ? 1 : 0;
    Pose<L<1>> cur;
#pragma unroll
    for (int e = 0; e < 9; ++e) cur.R.m[e] = load_ch<L<1>>(pose + e * C, g0, nv);
#pragma unroll
    for (int e = 0; e < 3; ++e) cur.t.v[e] = load_ch<L<1>>(pose + (9 + e) * C, g0, nv);
    np = compose(exp_map<L<1>>(d), cur);
  }
  __syncthreads();
  if (mine) {
    const int g0 = Dp > 0 ? static_cast<int>(threadIdx.x) : 0;
    const int nv = Dp > 0 ? 1 : 0;
#pragma unroll
    for (int e = 0; e < 9; ++e) store_ch<L<1>>(pose + e * C, np.R.m[e], g0, nv, threadIdx.x == 0);
#pragma unroll
    for (int e = 0; e < 3; ++e) store_ch<L<1>>(pose + (9 + e) * C, np.t.v[e], g0, nv, threadIdx.x == 0);
  }
  if (threadIdx.x == 0) {
    double sq[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) sq[i] = re(d[i]) * re(d[i]);
    const double nrm = sqrt((sq[0] + (sq[1] + sq[2])) + (sq[3] + (sq[4] + sq[5])));
    st->iterations += 1;
    st->n_corr = n;
#pragma unroll
    for (int i = 0; i < 6; ++i) st->delta[i] = re(d[i]);
#pragma unroll
    for (int i = 0; i < 6; ++i) st->b[i] = s_acc[(21 + i) * C];
    if (nrm < tol) {
      st->level_done = 1;
      if (level == 0) st->converged = 1;
    }
  }
  clock_mark(4, kSolveClockCta);
  if (threadIdx.x == 0 && g_icp_clock) atomicAdd(&g_icp_clock_launch, 1u);
}

__global__ void __launch_bounds__(kRedThreads) k_icp_solve_t(TrackState* st, const double* __restrict__ gpartials,
                                                          const int* __restrict__ gcounts, int n_groups,
                                                          double* pose, int Dp, int level, double tol) {
  pdl_wait();
  pdl_trigger();
  if (st->level_done) return;
  icp_solve_body(st, gpartials, gcounts, n_groups, pose, Dp, level, tol);
}

// One lifted (J, r) row of a correspondence (slot (x, y) -> model pixel
// (u, v)) into row[7][C]: the canonical row both the fused reduce and the
// split rows kernel write (same operations, bit-identical).
CSF_DEV void icp_row(double* row, const double* __restrict__ depth, int w, int x, int y, int u, int v,
                     const double* s_pose, const double* s_intr, int C, int Dp, const double* __restrict__ vre,
                     const double* __restrict__ nre, const double* __restrict__ vim,
                     const double* __restrict__ nim) {
  // One lifted (J, r) row in tangent form: the real chain once, then each
  // channel's im by the truncated-Complex rule of every operation
  // (csfd.hpp:44-58) applied to the saved real intermediates.
  const long long m = static_cast<long long>(v) * w + u;
  const double d = depth[y * w + x];
  // vertex: ((d*(x - cx))/fx, (d*(y - cy))/fy, d)
  const double tx = static_cast<double>(x) - s_intr[2 * C], ty = static_cast<double>(y) - s_intr[3 * C];
  const double nx = d * tx, ny = d * ty;
  const double kfx = s_intr[0], kfy = s_intr[C];
  const double vre3[3] = {nx / kfx, ny / kfy, d};
  const double ifx = 1.0 / (kfx * kfx), ify = 1.0 / (kfy * kfy);
  (void)ifx;
  (void)ify;
  double R[9], T[3], MV[3], MN[3], P[3], PR[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) R[e] = s_pose[e * C];
#pragma unroll
  for (int e = 0; e < 3; ++e) T[e] = s_pose[(9 + e) * C];
#pragma unroll
  for (int c3 = 0; c3 < 3; ++c3) {
    MV[c3] = vre[3 * m + c3];
    MN[c3] = nre[3 * m + c3];
  }
#pragma unroll
  for (int r3 = 0; r3 < 3; ++r3) {
#pragma unroll
    for (int c3 = 0; c3 < 3; ++c3) PR[3 * r3 + c3] = R[3 * r3 + c3] * vre3[c3];
    P[r3] = (PR[3 * r3] + (PR[3 * r3 + 1] + PR[3 * r3 + 2])) + T[r3];
  }
  const double DF[3] = {P[0] - MV[0], P[1] - MV[1], P[2] - MV[2]};
  const double rr = DF[0] * MN[0] + (DF[1] * MN[1] + DF[2] * MN[2]);
  const double PN[3] = {P[1] * MN[2] - P[2] * MN[1], P[2] * MN[0] - P[0] * MN[2], P[0] * MN[1] - P[1] * MN[0]};
  row[0] = MN[0];
  row[C] = MN[1];
  row[2 * C] = MN[2];
  row[3 * C] = PN[0];
  row[4 * C] = PN[1];
  row[5 * C] = PN[2];
  row[6 * C] = rr;
  for (int ch = 1; ch <= Dp; ++ch) {
    // vertex channels (intrinsics seeds): d*(x - cx) has im d*(-cx.im)
    const double tnx = d * -s_intr[2 * C + ch], tny = d * -s_intr[3 * C + ch];
    const double vim3[3] = {CSF_CH_DIV(tnx * kfx - nx * s_intr[ch], kfx * kfx, ifx),
                            CSF_CH_DIV(tny * kfy - ny * s_intr[C + ch], kfy * kfy, ify), 0.0};
    double Pi[3], MVi[3], MNi[3];
#pragma unroll
    for (int c3 = 0; c3 < 3; ++c3) {
      MVi[c3] = vim[(3 * m + c3) * Dp + ch - 1];
      MNi[c3] = nim[(3 * m + c3) * Dp + ch - 1];
    }
#pragma unroll
    for (int r3 = 0; r3 < 3; ++r3) {
      double qi[3];
#pragma unroll
      for (int c3 = 0; c3 < 3; ++c3) qi[c3] = R[3 * r3 + c3] * vim3[c3] + s_pose[(3 * r3 + c3) * C + ch] * vre3[c3];
      Pi[r3] = (qi[0] + (qi[1] + qi[2])) + s_pose[(9 + r3) * C + ch];
    }
    const double DFi[3] = {Pi[0] - MVi[0], Pi[1] - MVi[1], Pi[2] - MVi[2]};
    double ti[3];
#pragma unroll
    for (int c3 = 0; c3 < 3; ++c3) ti[c3] = DF[c3] * MNi[c3] + DFi[c3] * MN[c3];
    const double ri = ti[0] + (ti[1] + ti[2]);
    const double PNi[3] = {(P[1] * MNi[2] + Pi[1] * MN[2]) - (P[2] * MNi[1] + Pi[2] * MN[1]),
                           (P[2] * MNi[0] + Pi[2] * MN[0]) - (P[0] * MNi[2] + Pi[0] * MN[2]),
                           (P[0] * MNi[1] + Pi[0] * MN[1]) - (P[1] * MNi[0] + Pi[1] * MN[0])};
    row[ch] = MNi[0];
    row[C + ch] = MNi[1];
    row[2 * C + ch] = MNi[2];
    row[3 * C + ch] = PNi[0];
    row[4 * C + ch] = PNi[1];
    row[5 * C + ch] = PNi[2];
    row[6 * C + ch] = ri;
  }

}

template <int G>
__global__ void __launch_bounds__(kRedThreads) k_icp_reduce(const TrackState* st, const double* __restrict__ depth,
                                                    int w, int h, int stride, const double* __restrict__ intr,
                                                    const double* pose, const double* __restrict__ vre,
                                                    const double* __restrict__ nre, const double* __restrict__ vim,
                                                    const double* __restrict__ nim, double d_max, double cos_max,
                                                    int Dp, int chunk, double* __restrict__ partials,
                                                    int* __restrict__ counts, double* __restrict__ gpartials,
                                                    int* __restrict__ gcounts, unsigned* __restrict__ group_ctr) {
  pdl_wait();
  pdl_trigger();
  if (st->level_done) return;
  clock_mark(0);
  using S = Scal<G>;
  extern __shared__ double sm[];
  const int C = 1 + Dp;
  double* s_pose = sm;
  double* s_intr = s_pose + 12 * C;
  double* s_jr = s_intr + 4 * C;
  __shared__ int s_wsum[kRedThreads / 32];
  for (int i = threadIdx.x; i < 12 * C; i += blockDim.x) s_pose[i] = pose[i];
  for (int i = threadIdx.x; i < 4 * C; i += blockDim.x) s_intr[i] = intr[i];
  __syncthreads();

  Pose<double> c2w, w2p;
  load_pose_real(s_pose, C, &c2w);
#pragma unroll
  for (int e = 0; e < 9; ++e) w2p.R.m[e] = st->pred_w2c[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) w2p.t.v[e] = st->pred_w2c[9 + e];
  const double fx = s_intr[0], fy = s_intr[C], cx = s_intr[2 * C], cy = s_intr[3 * C];
  const int nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  const int n_slots = nxs * nys;
  const int n_acc = 27 * C;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int tile_count = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  for (int cbase = 0; cbase < kTile; cbase += chunk) {
    const int slot = blockIdx.x * kTile + cbase + threadIdx.x;
    bool corr = false;
    int x = 0, y = 0, u = 0, v = 0;
    if (threadIdx.x < chunk && slot < n_slots) {
      x = (slot % nxs) * stride;
      y = (slot / nxs) * stride;
      corr = associate_slot(depth, w, h, x, y, fx, fy, cx, cy, c2w, w2p, vre, nre, d_max, cos_max, &u, &v);
    }
    // order-preserving compaction within the chunk
    const unsigned ballot = __ballot_sync(0xffffffffu, corr);
    if (lane == 0) s_wsum[warp] = __popc(ballot);
    __syncthreads();
    int before = 0, total = 0;
    for (int k = 0; k < kRedThreads / 32; ++k) {
      if (k < warp) before += s_wsum[k];
      total += s_wsum[k];
    }
    const int pos = before + __popc(ballot & ((1u << lane) - 1u));
    if (corr) icp_row(s_jr + static_cast<long long>(pos) * 7 * C, depth, w, x, y, u, v, s_pose, s_intr, C, Dp, vre,
                      nre, vim, nim);
    __syncthreads();
    if (cbase == 0) clock_mark(1);
    // per-accumulator sequential sums in slot order
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int a = threadIdx.x + kRedThreads * j;
      if (a >= n_acc) break;
      const int q = a / C, c = a % C;
      int ja, jb;
      if (q < 21) {
        ja = c_tri_r[q];
        jb = c_tri_c[q];
      } else {
        ja = q - 21;
        jb = 6;
      }
      const int stride = 7 * C;
      const double* pa = s_jr + ja * C;
      const double* pb = s_jr + jb * C;
      double s = acc[j];
      // the add chain is sequential (canonical order); the shared-memory
      // loads of the next entries are independent and are issued ahead
      if (c == 0) {
#pragma unroll 8
        for (int e = 0; e < total; ++e) s = s + pa[e * stride] * pb[e * stride];
      } else {
#pragma unroll 8
        for (int e = 0; e < total; ++e) {
          const int o = e * stride;
          s = s + (pa[o] * pb[o + c] + pa[o + c] * pb[o]);
        }
      }
      acc[j] = s;
    }
    tile_count += total;
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int a = threadIdx.x + kRedThreads * j;
    if (a < n_acc) partials[static_cast<long long>(blockIdx.x) * n_acc + a] = acc[j];
  }
  if (threadIdx.x == 0) counts[blockIdx.x] = tile_count;
  clock_mark(2);
  group_sum(partials, counts, n_acc, gpartials, gcounts, group_ctr);
}

// Level entry: the prediction pose is the current estimate (icp.cpp:191).
__global__ void k_level_begin(TrackState* st, const double* pose, double* pred_pose, int Dp) {
  pdl_wait();
  pdl_trigger();
  const int C = 1 + Dp;
  for (int i = threadIdx.x; i < 12 * C; i += blockDim.x) pred_pose[i] = pose[i];
  if (threadIdx.x == 0) {
    Pose<double> p;
    load_pose_real(pose, C, &p);
    const Pose<double> inv = inverse(p);
    for (int e = 0; e < 9; ++e) st->pred_w2c[e] = inv.R.m[e];
    for (int e = 0; e < 3; ++e) st->pred_w2c[9 + e] = inv.t.v[e];
    st->level_done = 0;
  }
}

// Seeds: first-frame twist xi0* and intrinsics channels; T0* = exp(xi0*) T0.
template <int G>
__global__ void k_seed(const int* __restrict__ dirs, int D, double hstep, const double* __restrict__ gt0,
                       const double* __restrict__ kbase, double* pose, double* intr_levels, int levels, int Dp) {
  pdl_wait();
  pdl_trigger();
  using S = Scal<G>;
  const int C = 1 + Dp;
  const int ngroups = G == 0 ? 1 : Dp / G;
  const int gi = threadIdx.x;
  if (gi >= ngroups) return;
  const int g0 = gi * G;
  S xi[6], kk[4];
  for (int i = 0; i < 6; ++i) xi[i] = lit<S>(0.0);
  for (int i = 0; i < 4; ++i) kk[i] = lit<S>(kbase[i]);
  if constexpr (G > 0) {
    for (int g = 0; g < G; ++g) {
      const int dd = g0 + g;
      if (dd >= D) continue;
      const int prm = dirs[dd];
      if (prm >= 0 && prm < 6) xi[prm].im[g] = hstep;
      else if (prm >= 6 && prm < 10) kk[prm - 6].im[g] = hstep;
    }
  }
  Pose<S> base;
  for (int e = 0; e < 9; ++e) base.R.m[e] = lit<S>(gt0[e]);
  for (int e = 0; e < 3; ++e) base.t.v[e] = lit<S>(gt0[9 + e]);
  const Pose<S> p = compose(exp_map<S>(xi), base);
  for (int e = 0; e < 9; ++e) store_ch<S>(pose + e * C, p.R.m[e], g0, G, gi == 0);
  for (int e = 0; e < 3; ++e) store_ch<S>(pose + (9 + e) * C, p.t.v[e], g0, G, gi == 0);
  for (int l = 0; l < levels; ++l) {
    const double s = static_cast<double>(1 << l);
    for (int i = 0; i < 4; ++i) store_ch<S>(intr_levels + (l * 4 + i) * C, kk[i] / s, g0, G, gi == 0);
  }
}

// Keyframe perturbation (config 4): pose <- exp(xi) pose, xi seeded on the
// channels whose direction code is 10 + 6 (kf - 1) + c.  With no matching
// channel exp(0) is the exact identity, so the real pose is unchanged.
template <int G>
__global__ void k_keyframe_seed(const int* __restrict__ dirs, int D, double hstep, int kf, double* pose, int Dp) {
  pdl_wait();
  pdl_trigger();
  using S = Scal<G>;
  const int C = 1 + Dp;
  const int ngroups = G == 0 ? 1 : Dp / G;
  const int gi = threadIdx.x;
  const bool mine = gi < ngroups;
  const int g0 = gi * G;
  Pose<S> np;
  if (mine) {
    S xi[6];
    for (int i = 0; i < 6; ++i) xi[i] = lit<S>(0.0);
    if constexpr (G > 0) {
      for (int g = 0; g < G; ++g) {
        const int dd = g0 + g;
        if (dd >= D) continue;
        const int c = dirs[dd] - (10 + 6 * (kf - 1));
        if (c >= 0 && c < 6) xi[c].im[g] = hstep;
      }
    }
    Pose<S> cur;
    for (int e = 0; e < 9; ++e) cur.R.m[e] = load_ch<S>(pose + e * C, g0, G);
    for (int e = 0; e < 3; ++e) cur.t.v[e] = load_ch<S>(pose + (9 + e) * C, g0, G);
    np = compose(exp_map<S>(xi), cur);
  }
  __syncthreads();  // every group has read the real part before group 0 rewrites it
  if (mine) {
    for (int e = 0; e < 9; ++e) store_ch<S>(pose + e * C, np.R.m[e], g0, G, gi == 0);
    for (int e = 0; e < 3; ++e) store_ch<S>(pose + (9 + e) * C, np.t.v[e], g0, G, gi == 0);
  }
}

__global__ void k_frame_begin(TrackState* st, int frame) {
  pdl_wait();
  pdl_trigger();
  st->frame = frame;
  st->pad[1] = 0;  // voxels fused this frame
  st->iterations = 0;
  st->converged = 0;
  st->n_corr = 0;
  st->level_done = 0;
}

__global__ void k_frame_end(const TrackState* st, const double* pose, double* traj, int Dp, int* stats,
                            const int* n_blocks, const int* counters) {
  pdl_wait();
  pdl_trigger();
  const int C = 1 + Dp;
  const int f = st->frame;
  for (int i = threadIdx.x; i < 12 * C; i += blockDim.x) traj[static_cast<long long>(f) * 12 * C + i] = pose[i];
  if (threadIdx.x == 0) {
    int* s = stats + 8 * f;
    s[0] = st->iterations;
    s[1] = st->n_corr;
    s[2] = st->converged;
    s[3] = n_blocks ? *n_blocks : 0;
    s[4] = counters ? counters[0] : 0;
    s[5] = counters ? counters[1] : 0;
    s[6] = st->pad[1];
  }
}

// Objective of the lifted trajectory and Im(f)/h.
template <int G>
__global__ void k_objective(const double* __restrict__ traj, const double* __restrict__ gt, int n_frames, int kind,
                            double hstep, int Dp, int D, double* out) {
  pdl_wait();
  pdl_trigger();
  using S = Scal<G>;
  const int C = 1 + Dp;
  const int ngroups = G == 0 ? 1 : Dp / G;
  const int gi = threadIdx.x;
  if (gi >= ngroups) return;
  const int g0 = gi * G;
  auto diff_at = [&](int f) {
    V3<S> t;
    for (int e = 0; e < 3; ++e)
      t.v[e] = load_ch<S>(traj + (static_cast<long long>(f) * 12 + 9 + e) * C, g0, G) - gt[f * 12 + 9 + e];
    return t;
  };
  S obj = lit<S>(0.0);
  if (kind == 0) {
    const V3<S> d = diff_at(n_frames - 1);
    obj = sqrt_s(dot3(d, d));
  } else {
    for (int f = 0; f < n_frames; ++f) {
      const V3<S> d = diff_at(f);
      obj = obj + dot3(d, d);
    }
  }
  if (gi == 0) out[0] = re(obj);
  if constexpr (G > 0) {
    for (int g = 0; g < G; ++g)
      if (g0 + g < D) out[2 + g0 + g] = obj.im[g] / hstep;
  }
}

// ============================================================================
// Second order (pipeline order 2): channel groups are bicomplex pairs, S =
// B<1> (re + im1, im2, im12).  Association is the first-order kernel's
// (associate_slot, real parts); the J/r rows and the normal-equation sums are
// evaluated generically in S, i.e. with the reference's Bicomplex product
// (the oracle's jacobian_row/accumulate_row, orc_icp.hpp) — no tangent
// shortcut exists at order 2.  One ICP iteration is three launches:
//   k_icp_reduce2  grid (tiles, pairs): per-tile partial sums of one pair's
//                  slots (pair 0 also writes the real channel and counts)
//   k_icp_solve2   one CTA per pair: tile partials in tile order, the 6x6
//                  LDLT/exp map in S; writes its pair's pose slots and (pair 0)
//                  the real step to `stage`
//   k_icp_commit   real pose + break decisions (TrackState)
// ============================================================================
constexpr int kTile2 = 256;

template <typename S>
__global__ void __launch_bounds__(256) k_icp_reduce2(const TrackState* st, const double* __restrict__ depth, int w,
                                                     int h, int stride, const double* __restrict__ intr,
                                                     const double* __restrict__ pose, const double* __restrict__ vre,
                                                     const double* __restrict__ nre, const double* __restrict__ vim,
                                                     const double* __restrict__ nim, double d_max, double cos_max,
                                                     int Dp, double* __restrict__ partials, int* __restrict__ counts) {
  pdl_wait();
  pdl_trigger();
  if (st->level_done) return;
  constexpr int G = Traits<S>::G;
  constexpr int CG = 1 + G;
  const int C = 1 + Dp;
  const int g0 = blockIdx.y * G;
  extern __shared__ double sm[];
  S* rows = reinterpret_cast<S*>(sm);  // [kTile2][7]
  __shared__ int s_wsum[8];
  Pose<double> c2w, w2p;
  load_pose_real(pose, C, &c2w);
#pragma unroll
  for (int e = 0; e < 9; ++e) w2p.R.m[e] = st->pred_w2c[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) w2p.t.v[e] = st->pred_w2c[9 + e];
  const double fx = intr[0], fy = intr[C], cx = intr[2 * C], cy = intr[3 * C];
  const int nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  const int n_slots = nxs * nys;
  const int slot = blockIdx.x * kTile2 + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = 0, y = 0, u = 0, v = 0;
  bool corr = false;
  if (slot < n_slots) {
    x = (slot % nxs) * stride;
    y = (slot / nxs) * stride;
    corr = associate_slot(depth, w, h, x, y, fx, fy, cx, cy, c2w, w2p, vre, nre, d_max, cos_max, &u, &v);
  }
  const unsigned ballot = __ballot_sync(0xffffffffu, corr);
  if (lane == 0) s_wsum[warp] = __popc(ballot);
  __syncthreads();
  int before = 0, total = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (k < warp) before += s_wsum[k];
    total += s_wsum[k];
  }
  if (corr) {
    const int pos = before + __popc(ballot & ((1u << lane) - 1u));
    // jacobian_row (icp.cpp:20-24): vertex = backproject(K, x, y, d) in S
    // (frames.hpp:38-41), p = base * vertex, r = (p - mv) . mn, J = [mn; p x mn]
    const double d = depth[y * w + x];
    const S kfx = load_ch<S>(intr, g0, G), kfy = load_ch<S>(intr + C, g0, G);
    const S kcx = load_ch<S>(intr + 2 * C, g0, G), kcy = load_ch<S>(intr + 3 * C, g0, G);
    const V3<S> vert = mk3<S>((d * (static_cast<double>(x) - kcx)) / kfx, (d * (static_cast<double>(y) - kcy)) / kfy,
                              lit<S>(d));
    Pose<S> base;
#pragma unroll
    for (int e = 0; e < 9; ++e) base.R.m[e] = load_ch<S>(pose + e * C, g0, G);
#pragma unroll
    for (int e = 0; e < 3; ++e) base.t.v[e] = load_ch<S>(pose + (9 + e) * C, g0, G);
    const long long m = static_cast<long long>(v) * w + u;
    V3<S> mv, mn;
#pragma unroll
    for (int c3 = 0; c3 < 3; ++c3) {
      mv.v[c3].re = vre[3 * m + c3];
      mn.v[c3].re = nre[3 * m + c3];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        mv.v[c3].im[g] = vim[(3 * m + c3) * Dp + g0 + g];
        mn.v[c3].im[g] = nim[(3 * m + c3) * Dp + g0 + g];
      }
    }
    const V3<S> pw = apply(base, vert);
    const S r = dot3(sub3(pw, mv), mn);
    const V3<S> pn = cross3(pw, mn);
    S* row = rows + 7 * pos;
    row[0] = mn.v[0]; row[1] = mn.v[1]; row[2] = mn.v[2];
    row[3] = pn.v[0]; row[4] = pn.v[1]; row[5] = pn.v[2];
    row[6] = r;
  }
  __syncthreads();
  // accumulate_row (orc_icp.hpp): one thread per (accumulator, slot), the
  // S product of the two row entries, summed in slot order within the tile
  const int a = threadIdx.x;
  if (a < 27 * CG) {
    const int q = a / CG, c = a % CG;
    int ja, jb;
    if (q < 21) {
      ja = c_tri_r[q];
      jb = c_tri_c[q];
    } else {
      ja = q - 21;
      jb = 6;
    }
    double acc = 0.0;
    for (int e = 0; e < total; ++e) {
      const S prod = rows[7 * e + ja] * rows[7 * e + jb];
      acc = acc + (c == 0 ? prod.re : prod.im[c - 1]);
    }
    if (c == 0) {
      if (blockIdx.y == 0) partials[static_cast<long long>(blockIdx.x) * 27 * C + q * C] = acc;
    } else {
      partials[static_cast<long long>(blockIdx.x) * 27 * C + q * C + g0 + c] = acc;
    }
  }
  if (threadIdx.x == 0 && blockIdx.y == 0) counts[blockIdx.x] = total;
}

// stage: [0..11] new real pose, [12] |delta.re|, [13] correspondence count,
// [14] 1 if the step was applied
template <typename S>
__global__ void __launch_bounds__(128) k_icp_solve2(const TrackState* st, const double* __restrict__ partials,
                                                    const int* __restrict__ counts, int n_tiles, double* pose, int Dp,
                                                    double* stage) {
  pdl_wait();
  pdl_trigger();
  if (st->level_done) return;
  constexpr int G = Traits<S>::G;
  constexpr int CG = 1 + G;
  const int C = 1 + Dp;
  const int g0 = blockIdx.x * G;
  __shared__ double s_acc[27 * CG];
  __shared__ int s_n;
  if (threadIdx.x == 0) s_n = 0;
  for (int a = threadIdx.x; a < 27 * CG; a += blockDim.x) {
    const int q = a / CG, c = a % CG;
    const long long off = static_cast<long long>(q) * C + (c == 0 ? 0 : g0 + c);
    // canonical two-level order: tiles in order within groups of kGroup,
    // group totals in order (oracle tiled_normal_equations)
    double total = 0.0;
    for (int t = 0; t < n_tiles; t += kGroup) {
      double vals[kGroup];
#pragma unroll
      for (int k = 0; k < kGroup; ++k)
        vals[k] = t + k < n_tiles ? __ldcg(partials + static_cast<long long>(t + k) * 27 * C + off) : 0.0;
      double gsum = 0.0;
#pragma unroll
      for (int k = 0; k < kGroup; ++k)
        if (t + k < n_tiles) gsum = gsum + vals[k];
      total = total + gsum;
    }
    s_acc[a] = total;
  }
  __syncthreads();
  {
    int part = 0;
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) part += __ldcg(counts + t);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0 && part) atomicAdd(&s_n, part);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int n = s_n;
  if (blockIdx.x == 0) {
    stage[13] = static_cast<double>(n);
    stage[14] = 0.0;
  }
  if (n < 12) return;
  S a[21], nb[6], d[6];
#pragma unroll
  for (int q = 0; q < 21; ++q) a[q] = load_ch<S>(s_acc + q * CG, 0, G);
#pragma unroll
  for (int i = 0; i < 6; ++i) nb[i] = -load_ch<S>(s_acc + (21 + i) * CG, 0, G);
  ldlt6_solve_reg<S>(a, nb, d);
  bool fin = true;
#pragma unroll
  for (int i = 0; i < 6; ++i) fin = fin && finite_s(d[i]);
  if (!fin)
#pragma unroll
    for (int i = 0; i < 6; ++i) d[i] = lit<S>(0.0);
  Pose<S> cur;
#pragma unroll
  for (int e = 0; e < 9; ++e) cur.R.m[e] = load_ch<S>(pose + e * C, g0, G);
#pragma unroll
  for (int e = 0; e < 3; ++e) cur.t.v[e] = load_ch<S>(pose + (9 + e) * C, g0, G);
  const Pose<S> np = compose(exp_map<S>(d), cur);
  // this pair's slots now; the real channel is committed by k_icp_commit
#pragma unroll
  for (int e = 0; e < 9; ++e) store_ch<S>(pose + e * C, np.R.m[e], g0, G, false);
#pragma unroll
  for (int e = 0; e < 3; ++e) store_ch<S>(pose + (9 + e) * C, np.t.v[e], g0, G, false);
  if (blockIdx.x == 0) {
#pragma unroll
    for (int e = 0; e < 9; ++e) stage[e] = re(np.R.m[e]);
#pragma unroll
    for (int e = 0; e < 3; ++e) stage[9 + e] = re(np.t.v[e]);
    double sq[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) sq[i] = re(d[i]) * re(d[i]);
    stage[12] = sqrt((sq[0] + (sq[1] + sq[2])) + (sq[3] + (sq[4] + sq[5])));
    stage[14] = 1.0;
  }
}

__global__ void k_icp_commit(TrackState* st, double* pose, int Dp, const double* __restrict__ stage, int level,
                             double tol) {
  pdl_wait();
  pdl_trigger();
  if (st->level_done) return;
  const int C = 1 + Dp;
  const int n = static_cast<int>(stage[13]);
  if (stage[14] == 0.0) {  // fewer than 12 correspondences: break before the step (icp.cpp:199)
    st->n_corr = n;
    st->level_done = 1;
    return;
  }
  for (int e = 0; e < 12; ++e) pose[e * C] = stage[e];
  st->iterations += 1;
  st->n_corr = n;
  if (stage[12] < tol) {
    st->level_done = 1;
    if (level == 0) st->converged = 1;
  }
}

// Seeds of a second-order run: pair p carries im1 on parameter pair_i[p] and
// im2 on pair_j[p] (promote2, csfd.hpp:303-307).
template <typename S>
__global__ void k_seed2(const int* __restrict__ pair_i, const int* __restrict__ pair_j, int n_pairs, double hstep,
                        const double* __restrict__ gt0, const double* __restrict__ kbase, double* pose,
                        double* intr_levels, int levels, int Dp) {
  pdl_wait();
  pdl_trigger();
  constexpr int G = Traits<S>::G;
  const int C = 1 + Dp;
  const int gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= Dp / G) return;
  const int g0 = gi * G;
  S xi[6], kk[4];
  for (int i = 0; i < 6; ++i) xi[i] = lit<S>(0.0);
  for (int i = 0; i < 4; ++i) kk[i] = lit<S>(kbase[i]);
  if (gi < n_pairs) {
    const int pi = pair_i[gi], pj = pair_j[gi];
    if (pi < 6) xi[pi].im[0] = hstep; else kk[pi - 6].im[0] = hstep;
    if (pj < 6) xi[pj].im[1] = hstep; else kk[pj - 6].im[1] = hstep;
  }
  Pose<S> base;
  for (int e = 0; e < 9; ++e) base.R.m[e] = lit<S>(gt0[e]);
  for (int e = 0; e < 3; ++e) base.t.v[e] = lit<S>(gt0[9 + e]);
  const Pose<S> p = compose(exp_map<S>(xi), base);
  for (int e = 0; e < 9; ++e) store_ch<S>(pose + e * C, p.R.m[e], g0, G, gi == 0);
  for (int e = 0; e < 3; ++e) store_ch<S>(pose + (9 + e) * C, p.t.v[e], g0, G, gi == 0);
  for (int l = 0; l < levels; ++l) {
    const double sc = static_cast<double>(1 << l);
    for (int i = 0; i < 4; ++i) store_ch<S>(intr_levels + (l * 4 + i) * C, kk[i] / sc, g0, G, gi == 0);
  }
}

// Objective in S per pair; out[0] = re, out[2 + 3p + t] = slot t of pair p.
template <typename S>
__global__ void k_objective2(const double* __restrict__ traj, const double* __restrict__ gt, int n_frames, int kind,
                             int Dp, int n_pairs, double* out) {
  pdl_wait();
  pdl_trigger();
  constexpr int G = Traits<S>::G;
  const int C = 1 + Dp;
  const int gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= n_pairs) return;
  const int g0 = gi * G;
  auto diff_at = [&](int f) {
    V3<S> t;
    for (int e = 0; e < 3; ++e)
      t.v[e] = load_ch<S>(traj + (static_cast<long long>(f) * 12 + 9 + e) * C, g0, G) - gt[f * 12 + 9 + e];
    return t;
  };
  S obj = lit<S>(0.0);
  if (kind == 0) {
    const V3<S> d = diff_at(n_frames - 1);
    obj = sqrt_s(dot3(d, d));
  } else {
    for (int f = 0; f < n_frames; ++f) {
      const V3<S> d = diff_at(f);
      obj = obj + dot3(d, d);
    }
  }
  if (gi == 0) out[0] = re(obj);
  for (int g = 0; g < G; ++g) out[2 + g0 + g] = obj.im[g];
}

}  // namespace csfd

// ============================================================================
namespace csfi {

using namespace csfd;

static void chk(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) note_launch_error(what, e);
}

#define CSF_DISPATCH_G(G, BODY)                       \
  switch (G) {                                        \
    case 0: { constexpr int kG = 0; BODY; } break;    \
    case 1: { constexpr int kG = 1; BODY; } break;    \
    case 2: { constexpr int kG = 2; BODY; } break;    \
    case 3: { constexpr int kG = 3; BODY; } break;    \
    case 4: { constexpr int kG = 4; BODY; } break;    \
    case 5: { constexpr int kG = 5; BODY; } break;    \
    case 6: { constexpr int kG = 6; BODY; } break;    \
    default: note_error("csf_b200: no kernel for group width " + std::to_string(G)); \
  }

// Debug: enable per-CTA phase timestamps into a device buffer of
// 4096 launches x 512 CTAs x 5 slots (nullptr disables).
void icp_clock_enable(unsigned long long* buf) {
  cudaMemcpyToSymbol(g_icp_clock, &buf, sizeof(buf));
  const unsigned z = 0;
  cudaMemcpyToSymbol(g_icp_clock_launch, &z, sizeof(z));
}

int icp_tiles(int w, int h, int stride) {
  const long long nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  return static_cast<int>((nxs * nys + kTile - 1) / kTile);
}
bool icp_frame_fits(int w, int h, int stride) {
  const int tiles = icp_tiles(w, h, stride);
  return (tiles + kGroup - 1) / kGroup <= kMaxGroupCtr - 1;
}

// Slots per shared-memory chunk of the (J, r) rows.
// (one pass over the tile's 256 slots whenever the rows fit: measured faster
// than two half-tile passes at two CTAs per SM, bench r01)
static int reduce_chunk(int C) {
  if (8 * C * (16 + 256 * 7) <= 200 * 1024) return 256;
  if (8 * C * (16 + 128 * 7) <= 200 * 1024) return 128;
  if (8 * C * (16 + 64 * 7) <= 200 * 1024) return 64;
  return 32;
}

void launch_level_begin(const Launch& L, TrackState* st, const double* pose, double* pred_pose, int Dp) {
  launch_pdl(k_level_begin, dim3(1), dim3(128), 0, L.stream, st, pose, pred_pose, Dp);
  ++*L.launches;
  chk("level_begin");
}

size_t icp_partials_doubles(int C, int max_tiles) {
  return static_cast<size_t>(max_tiles + (max_tiles + kGroup - 1) / kGroup) * 27 * C;
}
size_t icp_counts_ints(int max_tiles) {
  return static_cast<size_t>(kMaxGroupCtr + max_tiles + (max_tiles + kGroup - 1) / kGroup);
}

// One ICP iteration: k_icp_reduce (association, lifted rows, tile sums, group
// sums) then k_icp_solve_t.  Scratch layout: partials = [tiles][27C] then
// [groups][27C]; counts = [kMaxGroupCtr] self-resetting group counters (zero
// at allocation), [tiles], [groups].
void launch_icp_reduce(const Launch& L, int G, int Dp, TrackState* st, const double* depth, int w, int h,
                       int stride, const double* intr, double* pose, const double* vre, const double* nre,
                       const double* vim, const double* nim, double d_max, double cos_max, double* partials,
                       int* counts, int level, double tol) {
  const int C = 1 + Dp;
  const int n_acc = 27 * C;
  const int chunk = reduce_chunk(C);
  const size_t smem = sizeof(double) * (16 * C + static_cast<size_t>(chunk) * 7 * C);
  const int tiles = icp_tiles(w, h, stride);
  const int groups = (tiles + kGroup - 1) / kGroup;
  if (groups > kMaxGroupCtr - 1 || Dp > kMaxC - 1) {
    note_error("csf_b200: ICP frame too large (" + std::to_string(tiles) + " tiles) or too many channels (" +
               std::to_string(Dp) + ")");
    return;
  }
  unsigned* ctr = reinterpret_cast<unsigned*>(counts);
  int* tcounts = counts + kMaxGroupCtr;
  int* gcounts = tcounts + tiles;
  double* gpartials = partials + static_cast<size_t>(tiles) * n_acc;
  // J/r rows are evaluated one channel at a time: register-light, and any
  // channel-group width addresses the same channel layout.
  if (G == 0)
    launch_pdl(k_icp_reduce<0>, dim3(tiles), dim3(kRedThreads), smem, L.stream, st, depth, w, h, stride, intr, pose,
               vre, nre, vim, nim, d_max, cos_max, Dp, chunk, partials, tcounts, gpartials, gcounts, ctr);
  else
    launch_pdl(k_icp_reduce<1>, dim3(tiles), dim3(kRedThreads), smem, L.stream, st, depth, w, h, stride, intr, pose,
               vre, nre, vim, nim, d_max, cos_max, Dp, chunk, partials, tcounts, gpartials, gcounts, ctr);
  launch_pdl(k_icp_solve_t, dim3(1), dim3(kRedThreads), 0, L.stream, st, static_cast<const double*>(gpartials),
             static_cast<const int*>(gcounts), groups, pose, Dp, level, tol);
  *L.launches += 2;
  chk("icp_reduce");
}

void launch_seed(const Launch& L, int G, int Dp, const int* dirs, int D, double h, const double* gt0,
                 const double* intr_base, double* pose, double* intr_levels, int levels) {
  if (G == 0)
    launch_pdl(k_seed<0>, dim3(1), dim3(64), 0, L.stream, dirs, D, h, gt0, intr_base, pose, intr_levels, levels, Dp);
  else
    launch_pdl(k_seed<1>, dim3(1), dim3(64), 0, L.stream, dirs, D, h, gt0, intr_base, pose, intr_levels, levels, Dp);
  ++*L.launches;
  chk("seed");
}

void launch_keyframe_seed(const Launch& L, int G, int Dp, const int* dirs, int D, double h, int kf, double* pose) {
  if (G == 0)
    launch_pdl(k_keyframe_seed<0>, dim3(1), dim3(64), 0, L.stream, dirs, D, h, kf, pose, Dp);
  else
    launch_pdl(k_keyframe_seed<1>, dim3(1), dim3(64), 0, L.stream, dirs, D, h, kf, pose, Dp);
  ++*L.launches;
  chk("keyframe_seed");
}

void launch_frame_begin(const Launch& L, TrackState* st, int frame) {
  launch_pdl(k_frame_begin, dim3(1), dim3(1), 0, L.stream, st, frame);
  ++*L.launches;
  chk("frame_begin");
}

void launch_frame_end(const Launch& L, TrackState* st, const double* pose, double* traj, int Dp, int* stats,
                      const int* n_blocks, const int* counters) {
  launch_pdl(k_frame_end, dim3(1), dim3(128), 0, L.stream, st, pose, traj, Dp, stats, n_blocks, counters);
  ++*L.launches;
  chk("frame_end");
}

void launch_objective(const Launch& L, int G, int Dp, int D, const double* traj, const double* gt, int n_frames,
                      int kind, double h, double* out) {
  if (G == 0)
    launch_pdl(k_objective<0>, dim3(1), dim3(64), 0, L.stream, traj, gt, n_frames, kind, h, Dp, D, out);
  else
    launch_pdl(k_objective<1>, dim3(1), dim3(64), 0, L.stream, traj, gt, n_frames, kind, h, Dp, D, out);
  ++*L.launches;
  chk("objective");
}

// ---- second order ----------------------------------------------------------
void launch_icp_iteration2(const Launch& L, int Dp, TrackState* st, const double* depth, int w, int h, int stride,
                           const double* intr, double* pose, const double* vre, const double* nre, const double* vim,
                           const double* nim, double d_max, double cos_max, double* partials, int* counts,
                           double* stage, int level, double tol) {
  using S = B<1>;
  const int tiles = icp_tiles(w, h, stride);
  const int pairs = Dp / 3;
  const size_t smem = sizeof(S) * kTile2 * 7;
  launch_pdl(k_icp_reduce2<S>, dim3(dim3(tiles, pairs)), dim3(kTile2), smem, L.stream, st, depth, w, h, stride, intr, pose, vre, nre, vim,
                                                                   nim, d_max, cos_max, Dp, partials, counts);
  launch_pdl(k_icp_solve2<S>, dim3(pairs), dim3(128), 0, L.stream, st, partials, counts, tiles, pose, Dp, stage);
  launch_pdl(k_icp_commit, dim3(1), dim3(1), 0, L.stream, st, pose, Dp, stage, level, tol);
  *L.launches += 3;
  chk("icp_iteration2");
}

void launch_seed2(const Launch& L, int Dp, const int* pair_i, const int* pair_j, int n_pairs, double h,
                  const double* gt0, const double* intr_base, double* pose, double* intr_levels, int levels) {
  const int groups = Dp / 3;
  launch_pdl(k_seed2<B<1>>, dim3((groups + 63) / 64), dim3(64), 0, L.stream, pair_i, pair_j, n_pairs, h, gt0, intr_base, pose,
                                                         intr_levels, levels, Dp);
  ++*L.launches;
  chk("seed2");
}

void launch_objective2(const Launch& L, int Dp, int n_pairs, const double* traj, const double* gt, int n_frames,
                       int kind, double* out) {
  launch_pdl(k_objective2<B<1>>, dim3((n_pairs + 63) / 64), dim3(64), 0, L.stream, traj, gt, n_frames, kind, Dp, n_pairs, out);
  ++*L.launches;
  chk("objective2");
}

}  // namespace csfi

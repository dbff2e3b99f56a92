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
// Bicomplex quotients with the separate 1/b.re^2 division in this unit (the
// order-2 reduce/solve measured faster with it; lifted.cuh)
#define CSF_B_DEN_DIV
#include "geometry.cuh"

namespace csfd {

using csfi::TrackState;
using csfi::IcpLevelArgs;

// ============================================================================
// First-order ICP: one cooperative launch per pyramid level runs every
// iteration of the level (icp.cpp:193-238) without returning to the host.
//
// Grid = the level's tiles (<= kLvMaxTiles, co-resident at 2 CTAs per SM).
// Per iteration every CTA
//   A  associates its tile's slots (icp.cpp:89-126, real-part gates) and
//      compacts the correspondences, in slot order, into shared-memory
//      records of the real row and the real intermediates its channels need;
//   B  accumulates the normal equations (icp.cpp:15-28): warp w owns channel
//      c = w (+ 11 p), lane l the correspondence stream e = l (mod 32);
//      the real channel adds re(J_a) re(J_b) in plain double (bit-exact with
//      the oracle), every perturbation channel the truncated-Complex product
//      term re(J_a) im(J_b) + im(J_a) re(J_b) (csfd.hpp:50-53);
//   C  reduces the 32 streams with a fixed xor butterfly and writes its tile
//      partial; the last CTA of each group of kLvGroup tiles sums the group
//      in tile order and releases the group's generation flag; every CTA
//      waits for all group flags (the grid barrier) and sums the group
//      totals in group order itself;
//   D  every CTA solves the same 6x6 system redundantly from the totals (the
//      real LDLT in the oracle's Ldlt6 order, channels in tangent form
//      against the real factors), applies exp(delta) T per channel and takes
//      the break decisions (icp.cpp:199,235) — identical bits in every CTA,
//      so no second barrier is needed.
// The canonical order of the real sums (tile size, streams, butterfly, groups)
// is builder-defined and restated in oracle/orc_icp.hpp.
// ============================================================================
constexpr int kLvWarps = csfi::kIcpLevelWarps;
constexpr int kLvThreads = 32 * kLvWarps;
// Association runs on warps 0..kAsWarps-1; the last warp is the channel warp
// of the overlapped solve (it applies the channel step of iteration k while
// the other warps associate iteration k + 1).
constexpr int kAsWarps = kLvWarps - 1;
constexpr int kAsThreads = 32 * kAsWarps;
constexpr int kRounds = 2;                         // slots per thread in one association pass
constexpr int kSegSlots = 576;                     // slots per shared-memory record segment (a VGA tile is 544)
static_assert(kSegSlots <= kRounds * kAsThreads, "one association pass covers a segment");
constexpr int kLvMaxTiles = csfi::kIcpMaxTiles;
constexpr int kLvGroup = csfi::kIcpGroup;
constexpr int kLvMaxGroups = (kLvMaxTiles + kLvGroup - 1) / kLvGroup;
constexpr int kMaxC = 1 + 64;  // CSF_MAX_DIRECTIONS
// Barrier words: the group arrival counters share one line; the groups'
// release generations (one word per group, what every CTA polls) sit 256
// bytes away, so the polls never queue in front of the counters' atomics in
// the same L2 line.
constexpr int kFlagWord = 64;

// shared-memory record fields of one correspondence (structure of arrays)
enum RecField : int {
  kRD = 0, kRNX, kRNY, kRV0, kRV1, kRP0, kRP1, kRP2, kRDF0, kRDF1, kRDF2,
  kRMN0, kRMN1, kRMN2, kRPN0, kRPN1, kRPN2, kRRR, kRecFields
};

CSF_DEV void load_pose_real(const double* p, int C, Pose<double>* out) {
#pragma unroll
  for (int e = 0; e < 9; ++e) out->R.m[e] = p[e * C];
#pragma unroll
  for (int e = 0; e < 3; ++e) out->t.v[e] = p[(9 + e) * C];
}

// (row a, row b) of accumulator q: 21 lower-triangle entries of J J^T, then
// the 6 entries of J r (row b = 6, the residual).
CSF_HD constexpr int acc_row_a(int q) {
  return q < 21 ? (q < 1 ? 0 : q < 3 ? 1 : q < 6 ? 2 : q < 10 ? 3 : q < 15 ? 4 : 5) : q - 21;
}
CSF_HD constexpr int acc_row_b(int q) {
  return q < 21 ? q - (acc_row_a(q) * (acc_row_a(q) + 1)) / 2 : 6;
}

// The measured side of phase A — the vertex and normal of every slot of a
// segment (measure_surface, frames.hpp:86-114, recomputed from the pyramid
// depth) — does not depend on the pose, so it is computed once per level
// (per segment visit for multi-segment tiles) into s_meas[6][kSegSlots];
// an invalid slot stores vertex z = 0.  Every division / sqrt runs on valid
// data only (a zero or NaN operand sends the IEEE division down its slow path).
__device__ __noinline__ void level_measure(const IcpLevelArgs& a, int seg0, int seg1, const double* s_intr,
                                           double* s_meas) {
  const int C = 1 + a.Dp;
  const int nxs = (a.w + a.stride - 1) / a.stride;
  const int w = a.w, h = a.h;
  const double fx = s_intr[0], fy = s_intr[C], cx = s_intr[2 * C], cy = s_intr[3 * C];
  bool ok[kRounds];
  int xs[kRounds], ys[kRounds];
  double d0[kRounds], d1[kRounds], d2[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int slot = seg0 + r * kLvThreads + static_cast<int>(threadIdx.x);
    ok[r] = slot < seg1;  // seg1 <= seg0 + kSegSlots
    xs[r] = ok[r] ? (slot % nxs) * a.stride : 0;
    ys[r] = ok[r] ? (slot / nxs) * a.stride : 0;
    const int x = xs[r], y = ys[r];
    d0[r] = ok[r] ? a.depth[y * w + x] : 0.0;
    d1[r] = ok[r] && x + 1 < w ? a.depth[y * w + x + 1] : 0.0;
    d2[r] = ok[r] && y + 1 < h ? a.depth[(y + 1) * w + x] : 0.0;
  }
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int e = r * kLvThreads + static_cast<int>(threadIdx.x);
    if (e >= kSegSlots) continue;
    const int x = xs[r], y = ys[r];
    bool valid = ok[r] && d0[r] > 0.0 && x + 1 < w && y + 1 < h && d1[r] > 0.0 && d2[r] > 0.0;
    V3<double> vert = mk3<double>(0.0, 0.0, 0.0), n = mk3<double>(0.0, 0.0, 0.0);
    if (valid) {
      const double tx0 = static_cast<double>(x) - cx, tx1 = static_cast<double>(x + 1) - cx;
      const double ty0 = static_cast<double>(y) - cy, ty1 = static_cast<double>(y + 1) - cy;
      vert = mk3<double>(d0[r] * tx0 / fx, d0[r] * ty0 / fy, d0[r]);
      const V3<double> vx = mk3<double>(d1[r] * tx1 / fx, d1[r] * ty0 / fy, d1[r]);
      const V3<double> vy = mk3<double>(d2[r] * tx0 / fx, d2[r] * ty1 / fy, d2[r]);
      n = cross3(sub3(vx, vert), sub3(vy, vert));
      const double len2 = dot3(n, n);
      valid = len2 > 0.0;
      if (valid) {
        const double l = sqrt(len2);
        n = mk3<double>(n.v[0] / l, n.v[1] / l, n.v[2] / l);
        if (dot3(n, vert) > 0.0) n = mk3<double>(-n.v[0], -n.v[1], -n.v[2]);
        valid = dot3(n, n) > 0.5;
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      s_meas[k * kSegSlots + e] = vert.v[k];
      s_meas[(3 + k) * kSegSlots + e] = n.v[k];
    }
    if (!valid) s_meas[2 * kSegSlots + e] = 0.0;
  }
}

// Phase A (pose-dependent part) over one segment, kRounds slots per thread
// with every round's model loads in flight together: the association of
// icp.cpp:89-126 for each slot — the same operations as associate_slot
// (geometry.cuh) on the measured vertex/normal of level_measure, whose tests
// carry no side effects, so evaluating all of them and combining gives the
// reference's answer — then the slot-order compaction of the correspondences
// into the shared-memory records.  Runs on the kAsThreads threads of warps
// 0..kAsWarps-1 (named barrier 1).  Returns the segment's correspondence count.
CSF_DEV void assoc_barrier() { asm volatile("bar.sync 1, %0;" ::"n"(kAsThreads) : "memory"); }
__device__ __noinline__ int level_associate(const IcpLevelArgs& a, int seg0, int seg1, const double* s_pose,
                                            const double* s_intr, const Pose<double>& w2p, const double* s_meas,
                                            double* s_rec, int* s_m, int* s_wsum) {
  const int C = 1 + a.Dp;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nxs = (a.w + a.stride - 1) / a.stride;
  const int w = a.w, h = a.h;
  const double fx = s_intr[0], fy = s_intr[C], cx = s_intr[2 * C], cy = s_intr[3 * C];
  Pose<double> c2w;
  load_pose_real(s_pose, C, &c2w);
  bool ok[kRounds];
  int xs[kRounds], ys[kRounds];
  double d0[kRounds];
  V3<double> world[kRounds], nrm[kRounds];
  long long mi[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int e = r * kAsThreads + static_cast<int>(threadIdx.x);
    const int slot = seg0 + e;
    ok[r] = slot < seg1 && e < kSegSlots;
    xs[r] = ok[r] ? (slot % nxs) * a.stride : 0;
    ys[r] = ok[r] ? (slot / nxs) * a.stride : 0;
    d0[r] = ok[r] ? s_meas[2 * kSegSlots + e] : 0.0;
    ok[r] = ok[r] && d0[r] > 0.0;
    mi[r] = 0;
    if (ok[r]) {
      const V3<double> vert = mk3<double>(s_meas[e], s_meas[kSegSlots + e], d0[r]);
      nrm[r] = mk3<double>(s_meas[3 * kSegSlots + e], s_meas[4 * kSegSlots + e], s_meas[5 * kSegSlots + e]);
      world[r] = apply(c2w, vert);
      const V3<double> inp = apply(w2p, world[r]);
      ok[r] = inp.v[2] > 0.0;
      if (ok[r]) {
        const double uvx = (fx * inp.v[0]) / inp.v[2] + cx;
        const double uvy = (fy * inp.v[1]) / inp.v[2] + cy;
        const long long u = llround(uvx), v = llround(uvy);
        ok[r] = u >= 0 && u < w && v >= 0 && v < h;
        mi[r] = ok[r] ? v * w + u : 0;
      }
    }
  }
  double MV[kRounds][3], MN[kRounds][3];
#pragma unroll
  for (int r = 0; r < kRounds; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      MN[r][k] = ok[r] ? a.nre[3 * mi[r] + k] : 0.0;
      MV[r][k] = ok[r] ? a.vre[3 * mi[r] + k] : 0.0;
    }
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    if (!ok[r]) continue;
    const V3<double> mn = mk3<double>(MN[r][0], MN[r][1], MN[r][2]);
    const V3<double> mv = mk3<double>(MV[r][0], MV[r][1], MV[r][2]);
    ok[r] = dot3(mn, mn) > 0.5;
    const V3<double> dd = sub3(world[r], mv);
    ok[r] = ok[r] && !(sqrt(dot3(dd, dd)) > a.d_max);
    const V3<double> wn = matvec(c2w.R, nrm[r]);
    ok[r] = ok[r] && !(dot3(wn, mn) < a.cos_max);
  }
  // slot-order compaction, round by round
  int total = 0;
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const unsigned ballot = __ballot_sync(0xffffffffu, ok[r]);
    if (lane == 0) s_wsum[r * kLvWarps + warp] = __popc(ballot);
    assoc_barrier();
    int before = 0, rtotal = 0;
#pragma unroll
    for (int k = 0; k < kAsWarps; ++k) {
      const int c = s_wsum[r * kLvWarps + k];
      if (k < warp) before += c;
      rtotal += c;
    }
    if (ok[r]) {
      // the real row of normal_equations (icp.cpp:20-24): vertex =
      // backproject(K, x, y, d) (frames.hpp:38-41), p = base * vertex,
      // r = (p - mv) . mn, J = [mn; p x mn] — the oracle's operation order
      const int e = total + before + __popc(ballot & ((1u << lane) - 1u));
      const int x = xs[r], y = ys[r];
      const int sl = r * kAsThreads + static_cast<int>(threadIdx.x);
      const double d = d0[r];
      const double nx = d * (static_cast<double>(x) - cx), ny = d * (static_cast<double>(y) - cy);
      const double vv[3] = {s_meas[sl], s_meas[kSegSlots + sl], d};  // (nx / fx, ny / fy, d)
      double P[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const double p0 = c2w.R.m[3 * q] * vv[0], p1 = c2w.R.m[3 * q + 1] * vv[1], p2 = c2w.R.m[3 * q + 2] * vv[2];
        P[q] = (p0 + (p1 + p2)) + c2w.t.v[q];
      }
      const double DF[3] = {P[0] - MV[r][0], P[1] - MV[r][1], P[2] - MV[r][2]};
      double* rec = s_rec + e;
      rec[kRD * kSegSlots] = d;
      rec[kRNX * kSegSlots] = nx;
      rec[kRNY * kSegSlots] = ny;
      rec[kRV0 * kSegSlots] = vv[0];
      rec[kRV1 * kSegSlots] = vv[1];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        rec[(kRP0 + q) * kSegSlots] = P[q];
        rec[(kRDF0 + q) * kSegSlots] = DF[q];
        rec[(kRMN0 + q) * kSegSlots] = MN[r][q];
      }
      rec[kRPN0 * kSegSlots] = P[1] * MN[r][2] - P[2] * MN[r][1];
      rec[kRPN1 * kSegSlots] = P[2] * MN[r][0] - P[0] * MN[r][2];
      rec[kRPN2 * kSegSlots] = P[0] * MN[r][1] - P[1] * MN[r][0];
      rec[kRRR * kSegSlots] = DF[0] * MN[r][0] + (DF[1] * MN[r][1] + DF[2] * MN[r][2]);
      s_m[e] = static_cast<int>(mi[r]);
      if (a.Dp > 0) {
        // the channel warps of phase B read this pixel's model channels
        // (3 Dp contiguous doubles in each map): start their L1 fills now
        const double* pv = a.vim + 3 * mi[r] * a.Dp;
        const double* pn = a.nim + 3 * mi[r] * a.Dp;
        for (int o = 0; o < 3 * a.Dp; o += 16) {
          asm volatile("prefetch.global.L1 [%0];" ::"l"(pv + o));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(pn + o));
        }
        asm volatile("prefetch.global.L1 [%0];" ::"l"(pv + 3 * a.Dp - 1));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(pn + 3 * a.Dp - 1));
      }
    }
    total += rtotal;
  }
  return total;
}

// Phase B: lane `lane` of the warp owning channel c accumulates its stream's
// entries (global entry index = lane mod 32) among [e0, e0 + n).
CSF_DEV void level_accumulate(const IcpLevelArgs& a, int c, int ebase, int e0, int n, const double* s_pose,
                              const double* s_intr, const double* s_rec, const int* s_m, double (&acc)[27]) {
  const int lane = threadIdx.x & 31;
  const int C = 1 + a.Dp;
  const int first = (lane - ((ebase + e0) & 31) + 32) & 31;
  if (c == 0) {
    for (int e = e0 + first; e < e0 + n; e += 32) {
      double row[7];
      row[0] = s_rec[kRMN0 * kSegSlots + e];
      row[1] = s_rec[kRMN1 * kSegSlots + e];
      row[2] = s_rec[kRMN2 * kSegSlots + e];
      row[3] = s_rec[kRPN0 * kSegSlots + e];
      row[4] = s_rec[kRPN1 * kSegSlots + e];
      row[5] = s_rec[kRPN2 * kSegSlots + e];
      row[6] = s_rec[kRRR * kSegSlots + e];
#pragma unroll
      for (int q = 0; q < 27; ++q) acc[q] = acc[q] + row[acc_row_a(q)] * row[acc_row_b(q)];
    }
    return;
  }
  // perturbation channel c: the truncated-Complex rule of every operation of
  // the row (csfd.hpp:44-58) applied to the saved real intermediates
  const double kfx = s_intr[0], kfy = s_intr[C];
  const double fxc = s_intr[c], fyc = s_intr[C + c], cxc = s_intr[2 * C + c], cyc = s_intr[3 * C + c];
  const double ifx = 1.0 / (kfx * kfx), ify = 1.0 / (kfy * kfy);
  (void)ifx;
  (void)ify;
  const int Dp = a.Dp;
  for (int e = e0 + first; e < e0 + n; e += 32) {
    // the model-map channels of the correspondence (prefetched into L1 by phase A)
    const long long m = s_m[e];
    double MVi[3], MNi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      MVi[k] = __ldg(a.vim + (3 * m + k) * Dp + c - 1);
      MNi[k] = __ldg(a.nim + (3 * m + k) * Dp + c - 1);
    }
    const double d = s_rec[kRD * kSegSlots + e];
    const double vv[3] = {s_rec[kRV0 * kSegSlots + e], s_rec[kRV1 * kSegSlots + e], d};
    const double tnx = d * -cxc, tny = d * -cyc;
    const double vi[3] = {CSF_CH_DIV(__fma_rn(tnx, kfx, -s_rec[kRNX * kSegSlots + e] * fxc), kfx * kfx, ifx),
                          CSF_CH_DIV(__fma_rn(tny, kfy, -s_rec[kRNY * kSegSlots + e] * fyc), kfy * kfy, ify), 0.0};
    double P[3], DF[3], MN[3], Pi[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      P[r] = s_rec[(kRP0 + r) * kSegSlots + e];
      DF[r] = s_rec[(kRDF0 + r) * kSegSlots + e];
      MN[r] = s_rec[(kRMN0 + r) * kSegSlots + e];
      double qi[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) qi[k] = __fma_rn(s_pose[(3 * r + k) * C], vi[k], s_pose[(3 * r + k) * C + c] * vv[k]);
      Pi[r] = (qi[0] + (qi[1] + qi[2])) + s_pose[(9 + r) * C + c];
    }
    const double DFi[3] = {Pi[0] - MVi[0], Pi[1] - MVi[1], Pi[2] - MVi[2]};
    double ti[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) ti[k] = __fma_rn(DF[k], MNi[k], DFi[k] * MN[k]);
    double ch[7], row[7];
    ch[0] = MNi[0];
    ch[1] = MNi[1];
    ch[2] = MNi[2];
    ch[3] = __fma_rn(P[1], MNi[2], Pi[1] * MN[2]) - __fma_rn(P[2], MNi[1], Pi[2] * MN[1]);
    ch[4] = __fma_rn(P[2], MNi[0], Pi[2] * MN[0]) - __fma_rn(P[0], MNi[2], Pi[0] * MN[2]);
    ch[5] = __fma_rn(P[0], MNi[1], Pi[0] * MN[1]) - __fma_rn(P[1], MNi[0], Pi[1] * MN[0]);
    ch[6] = ti[0] + (ti[1] + ti[2]);
    row[0] = MN[0];
    row[1] = MN[1];
    row[2] = MN[2];
    row[3] = s_rec[kRPN0 * kSegSlots + e];
    row[4] = s_rec[kRPN1 * kSegSlots + e];
    row[5] = s_rec[kRPN2 * kSegSlots + e];
    row[6] = s_rec[kRRR * kSegSlots + e];
#pragma unroll
    for (int q = 0; q < 27; ++q)
      acc[q] = __fma_rn(row[acc_row_a(q)], ch[acc_row_b(q)], __fma_rn(ch[acc_row_a(q)], row[acc_row_b(q)], acc[q]));
  }
}

// Grid barrier of the level kernel: the CTA that completes a group publishes
// generation `gen` on the group's flag; everyone waits for every group.
CSF_DEV void release_gen(unsigned* flag, unsigned gen) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(gen) : "memory");
}
CSF_DEV unsigned acquire_gen(const unsigned* flag) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
  return v;
}
// The spin itself polls with relaxed loads (an acquire load invalidates the
// SM's L1 on every poll, which evicts the co-resident CTA's cached gathers
// and spills); one acquire fence follows the successful poll.
CSF_DEV unsigned poll_gen(const unsigned* flag) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
  return v;
}
CSF_DEV void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
CSF_DEV unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Degenerate real factorization: the channel's own lifted LDLT (rare path,
// kept out of the solve's register budget).
__device__ __noinline__ void solve_channel_lifted(const double* s_tot, int C, int t, L<1> (&d)[6]) {
  L<1> am[21], nb[6];
#pragma unroll
  for (int q = 0; q < 21; ++q) am[q] = load_ch<L<1>>(s_tot + q * C, t, 1);
#pragma unroll
  for (int i = 0; i < 6; ++i) nb[i] = -load_ch<L<1>>(s_tot + (21 + i) * C, t, 1);
  ldlt6_solve_reg<L<1>>(am, nb, d);
}
__device__ __noinline__ void increment_pose(const L<1> (&d)[6], const Pose<L<1>>& cur, Pose<L<1>>* out) {
  *out = compose(exp_map<L<1>>(d), cur);
}

// Phase D of k_icp_level: the 6x6 solve from the totals (every CTA, same
// bits).  The real LDLT runs lane-parallel in warp 0 — lane tri(r, c) holds
// m[r][c] of the lower triangle and performs exactly the operations the
// oracle's Ldlt6 (orc_icp.hpp, Eigen::LDLT's order) performs on that element:
// the pivot search on the diagonal, the symmetric transposition (a lane
// permutation: m'[r][c] = m[s(r)][s(c)]), the column update with the
// sequential dot product, the division by the pivot.  Then every channel
// thread applies the factors: the real step d.re (identical in every
// thread) and the channel in tangent form d.im = A^-1 (nb.im - A.im d.re)
// (the per-channel lifted LDLT for degenerate systems); delta is zeroed
// unless every channel is finite (delta.allFinite(), icp.cpp:45); then
// exp(delta) * T per channel thread (apply_increment, se3.hpp:116-119) and the
// step-tolerance break (icp.cpp:235).  dre: the real delta (thread 0).
CSF_DEV void lv_mark(unsigned seq, int it, int phase, int by = 0);
struct LevelSolveShared {
  double fm[36];  // factors, row-major (lower triangle and diagonal)
  double x[6];    // the real step (overlapped solve)
  double prev[12];  // the real pose before the step (overlapped solve)
  // real intermediates of exp_map(x) (overlapped solve): t, sin t, t/2,
  // sin(t/2), a, b, c, and exp(x) itself (R row-major, then t)
  double et, es1, eth, esh, ea, eb, ec;
  double ex[12];
  int small;  // t^2 < 1e-14 (the series branch of exp_map)
  int ftr[6];
  int degen, finite, done, conv;
  int fin_re;  // the real step is finite (overlapped solve)
};

CSF_HD constexpr int tri_row(int l) { return l < 1 ? 0 : l < 3 ? 1 : l < 6 ? 2 : l < 10 ? 3 : l < 15 ? 4 : 5; }

__device__ __noinline__ void ldlt6_warp(const double* a_lower, int stride, LevelSolveShared* ls) {
  constexpr unsigned kFull = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int l = lane < 21 ? lane : 0;
  const int r = tri_row(l), c = l - r * (r + 1) / 2;
  const bool col_lane = lane < 21;
  double v = col_lane ? a_lower[l * stride] : 0.0;
  bool ok = true, stop = false, degen = false;
  int transp[6] = {0, 1, 2, 3, 4, 5};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    if (stop) continue;
    // pivot: the first strictly largest |m[i][i]|, i >= k
    double best = fabs(__shfl_sync(kFull, v, tri(k, k)));
    int piv = k;
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      const double di = fabs(__shfl_sync(kFull, v, tri(i, i)));
      if (di > best) {
        best = di;
        piv = i;
      }
    }
    transp[k] = piv;
    if (piv != k) {
      const int sr = r == k ? piv : (r == piv ? k : r);
      const int sc = c == k ? piv : (c == piv ? k : c);
      const int src = sr >= sc ? tri(sr, sc) : tri(sc, sr);
      v = __shfl_sync(kFull, v, col_lane ? src : lane);
    }
    if (k > 0) {
      // temp[j] = m[j][j] m[k][j]; m[i][k] -= m[i][0] temp[0] + m[i][1] temp[1] + ...
      double sacc = 0.0;
#pragma unroll
      for (int j = 0; j < k; ++j) {
        const double tj = __shfl_sync(kFull, v, tri(j, j)) * __shfl_sync(kFull, v, tri(k, j));
        const double mij = __shfl_sync(kFull, v, r > j ? tri(r, j) : 0);
        const double prod = mij * tj;
        sacc = j == 0 ? prod : sacc + prod;
      }
      if (col_lane && c == k) v = v - sacc;
    }
    const double akk = __shfl_sync(kFull, v, tri(k, k));
    const bool pivot_valid = fabs(akk) > 0.0;
    if (!pivot_valid) degen = true;
    if (k == 0 && !pivot_valid) {
      ok = false;
#pragma unroll
      for (int j = 0; j < 6; ++j) transp[j] = j;
      stop = true;
      continue;
    }
    if (k < 5) {
      const bool below = col_lane && c == k && r > k;
      if (pivot_valid) {
        if (below) v = v / akk;
      } else {
        ok = ok && __all_sync(kFull, !below || v == 0.0);
      }
    }
  }
  const double tol = 2.2250738585072014e-308;  // numeric_limits<double>::min()
#pragma unroll
  for (int i = 0; i < 6; ++i)
    if (!(fabs(__shfl_sync(kFull, v, tri(i, i))) > tol)) degen = true;
  if (col_lane) {
    ls->fm[6 * r + c] = v;
    ls->fm[6 * c + r] = v;
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 6; ++i) ls->ftr[i] = transp[i];
    ls->degen = degen || stop;
  }
  (void)ok;
}

// ldlt6_apply_reg (geometry.cuh) with the factors in shared memory.
CSF_DEV void ldlt6_apply_smem(const double* fm, const int* tr, const double* rhs, double* dst) {
  double x[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) x[i] = rhs[i];
#pragma unroll
  for (int k = 0; k < 6; ++k)
#pragma unroll
    for (int i = k + 1; i < 6; ++i)
      if (tr[k] == i) swap_s(x[k], x[i]);
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = i + 1; j < 6; ++j) x[j] = x[j] - x[i] * fm[6 * j + i];
  const double tol = 2.2250738585072014e-308;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double mii = fm[7 * i];
    x[i] = fabs(mii) > tol ? x[i] / mii : 0.0;
  }
#pragma unroll
  for (int i = 4; i >= 0; --i) {
    double sacc = fm[6 * (i + 1) + i] * x[i + 1];
#pragma unroll
    for (int j = i + 2; j < 6; ++j) sacc = sacc + fm[6 * j + i] * x[j];
    x[i] = x[i] - sacc;
  }
#pragma unroll
  for (int k = 5; k >= 0; --k)
#pragma unroll
    for (int i = k + 1; i < 6; ++i)
      if (tr[k] == i) swap_s(x[k], x[i]);
#pragma unroll
  for (int i = 0; i < 6; ++i) dst[i] = x[i];
}

__device__ __noinline__ void level_solve(const IcpLevelArgs& a, const double* s_tot, double* s_pose,
                                         LevelSolveShared* ls, double (&dre)[6], unsigned seq, int it,
                                         bool factored) {
  const int C = 1 + a.Dp;
  const int tid = threadIdx.x;
  if (!factored) {
    if (tid < 32) ldlt6_warp(s_tot, C, ls);
    __syncthreads();
  }
  lv_mark(seq, it, 8);
  // channel threads: thread t < max(Dp, 1) owns channel t + 1 (thread 0 also the real part)
  const bool mine = tid < (a.Dp > 0 ? a.Dp : 1);
  L<1> d[6];
  if (mine) {
    const int ch = 1 + tid;
    double nb[6], x[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) nb[i] = -s_tot[(21 + i) * C];
    ldlt6_apply_smem(ls->fm, ls->ftr, nb, x);  // the real step (the same bits in every thread)
    if (a.Dp == 0) {
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        d[i].re = x[i];
        d[i].im[0] = 0.0;
      }
    } else if (!ls->degen) {
      double rhs[6], dx[6];
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        double ax = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) ax = ax + s_tot[(i >= j ? tri(i, j) : tri(j, i)) * C + ch] * x[j];
        rhs[i] = -s_tot[(21 + i) * C + ch] - ax;
      }
      ldlt6_apply_smem(ls->fm, ls->ftr, rhs, dx);
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        d[i].re = x[i];
        d[i].im[0] = dx[i];
      }
    } else {
      solve_channel_lifted(s_tot, C, tid, d);
    }
    bool fin = true;
#pragma unroll
    for (int i = 0; i < 6; ++i) fin = fin && finite_s(d[i]);
    if (!fin) atomicAnd(&ls->finite, 0);  // delta.allFinite() over every channel
  }
  __syncthreads();
  lv_mark(seq, it, 9);
  Pose<L<1>> np;
  if (mine) {
    if (!ls->finite)
#pragma unroll
      for (int i = 0; i < 6; ++i) d[i] = lit<L<1>>(0.0);
    const int g0 = a.Dp > 0 ? tid : 0;
    const int nv = a.Dp > 0 ? 1 : 0;
    Pose<L<1>> cur;
#pragma unroll
    for (int e = 0; e < 9; ++e) cur.R.m[e] = load_ch<L<1>>(s_pose + e * C, g0, nv);
#pragma unroll
    for (int e = 0; e < 3; ++e) cur.t.v[e] = load_ch<L<1>>(s_pose + (9 + e) * C, g0, nv);
    increment_pose(d, cur, &np);  // apply_increment (se3.hpp:116-119)
  }
  __syncthreads();  // every channel thread has read the current pose
  lv_mark(seq, it, 10);
  if (mine) {
    const int g0 = a.Dp > 0 ? tid : 0;
    const int nv = a.Dp > 0 ? 1 : 0;
#pragma unroll
    for (int e = 0; e < 9; ++e) store_ch<L<1>>(s_pose + e * C, np.R.m[e], g0, nv, tid == 0);
#pragma unroll
    for (int e = 0; e < 3; ++e) store_ch<L<1>>(s_pose + (9 + e) * C, np.t.v[e], g0, nv, tid == 0);
  }
  if (tid == 0) {
    double sq[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) sq[i] = re(d[i]) * re(d[i]);
    const double nrm = sqrt((sq[0] + (sq[1] + sq[2])) + (sq[3] + (sq[4] + sq[5])));
    if (nrm < a.tol) {
      ls->done = 1;
      ls->conv = a.level == 0 ? 1 : 0;
    }
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) dre[i] = tid == 0 ? re(d[i]) : 0.0;
}

// Overlapped solve (single-segment tiles, 1 <= Dp < 32), after ldlt6_warp:
//   real_step (thread 0): the real step x from the factors, the real pose
//     exp(x) T (exp_map<double>: the real parts of the lifted evaluation, the
//     same operations) and the step-tolerance decision — assuming every
//     channel is finite — then warps 0..kAsWarps-1 associate the next
//     iteration;
//   channel_step (the channel warp, lane l = channel l + 1), concurrently:
//     the real step again, the channel step in tangent form and exp(delta) T
//     on the channels, against the real pose before the step (ls->prev);
//     delta.allFinite() (icp.cpp:45) is a warp vote, and if it fails delta is
//     zero for every channel and the kernel reverts the real pose
//     (exp(0) T of the saved pose) and decides again.
// exp_map<double> (lifted.cuh, se3.hpp:77-105) with its expensive real
// intermediates recorded for the channels' tangent evaluation.
CSF_DEV Pose<double> exp_map_record(const double xi[6], LevelSolveShared* ls) {
  const double phi[3] = {xi[3], xi[4], xi[5]};
  const double t2 = phi[0] * phi[0] + (phi[1] * phi[1] + phi[2] * phi[2]);
  double a, b, c;
  ls->small = re(t2) < 1e-14 ? 1 : 0;
  if (ls->small) {
    a = 1.0 - t2 / 6.0;
    b = 0.5 - t2 / 24.0;
    c = 1.0 / 6.0 - t2 / 120.0;
  } else {
    const double t = sqrt_s(t2);
    const double s1 = sin_s(t);
    a = s1 / t;
    const double th = t / 2.0;
    const double sh = sin_s(th);
    b = 2.0 * sh * sh / t2;
    c = (t - s1) / (t2 * t);
    ls->et = t;
    ls->es1 = s1;
    ls->eth = th;
    ls->esh = sh;
  }
  ls->ea = a;
  ls->eb = b;
  ls->ec = c;
  M3<double> px;
  px.m[0] = 0.0;     px.m[1] = -phi[2]; px.m[2] = phi[1];
  px.m[3] = phi[2];  px.m[4] = 0.0;     px.m[5] = -phi[0];
  px.m[6] = -phi[1]; px.m[7] = phi[0];  px.m[8] = 0.0;
  const M3<double> px2 = matmul(px, px);
  Pose<double> out;
  M3<double> v;
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    const double id = (e == 0 || e == 4 || e == 8) ? 1.0 : 0.0;
    out.R.m[e] = (id + a * px.m[e]) + b * px2.m[e];
    v.m[e] = (id + b * px.m[e]) + c * px2.m[e];
  }
  out.t = matvec(v, mk3(xi[0], xi[1], xi[2]));
#pragma unroll
  for (int e = 0; e < 9; ++e) ls->ex[e] = out.R.m[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) ls->ex[9 + e] = out.t.v[e];
  return out;
}

// One channel of exp(d) * T (increment_pose with S = L<1>) from the recorded
// real intermediates: every operation of exp_map<L<1>> and compose applies
// the truncated-Complex rule of lifted.cuh to (re, im) with the re parts
// taken from the real evaluation — the same bits as the lifted evaluation,
// without its sqrt / sin / division chains (the series branch is not
// recorded: the caller uses increment_pose there).
struct Tg {
  double re, im;
};
CSF_DEV Tg tg_add(Tg a, Tg b) { return {a.re + b.re, a.im + b.im}; }
CSF_DEV Tg tg_neg(Tg a) { return {-a.re, -a.im}; }
CSF_DEV Tg tg_mul(Tg a, Tg b) { return {a.re * b.re, a.re * b.im + a.im * b.re}; }
// a / b with the quotient's real part supplied
CSF_DEV Tg tg_div(Tg a, Tg b, double q) {
  const double den = b.re * b.re;
  const double inv = 1.0 / den;
  (void)inv;
  return {q, CSF_CH_DIV(a.im * b.re - a.re * b.im, den, inv)};
}
CSF_DEV Tg tg_sum3(Tg a0, Tg a1, Tg a2) { return tg_add(a0, tg_add(a1, a2)); }

CSF_DEV void increment_pose_tangent(const double xr[6], const double xim[6], const LevelSolveShared* ls,
                                    const double cur_im[12], double out_im[12]) {
  Tg xi[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) xi[i] = {xr[i], xim[i]};
  const Tg phi[3] = {xi[3], xi[4], xi[5]};
  const Tg t2 = tg_sum3(tg_mul(phi[0], phi[0]), tg_mul(phi[1], phi[1]), tg_mul(phi[2], phi[2]));
  // t = sqrt_s(t2): lift(z, f, 0.5 / f)
  const double tr = ls->et;
  const Tg t = {tr, (0.5 / tr) * t2.im};
  // sin_s(t): lift(z, sin, cos)
  const Tg s1 = {ls->es1, csf_det::cos(tr) * t.im};
  const Tg a = tg_div(s1, t, ls->ea);
  const Tg two = {2.0, 0.0};
  const Tg th = tg_div(t, two, ls->eth);
  const Tg sh = {ls->esh, csf_det::cos(th.re) * th.im};
  const Tg q2 = tg_mul(tg_mul(two, sh), sh);
  const Tg b = tg_div(q2, t2, ls->eb);
  const Tg n = {tr - ls->es1, t.im - s1.im};
  const Tg c = tg_div(n, tg_mul(t2, t), ls->ec);
  const Tg z = {0.0, 0.0};
  Tg px[9];
  px[0] = z;              px[1] = tg_neg(phi[2]); px[2] = phi[1];
  px[3] = phi[2];         px[4] = z;              px[5] = tg_neg(phi[0]);
  px[6] = tg_neg(phi[1]); px[7] = phi[0];         px[8] = z;
  Tg px2[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
      px2[3 * r + cc] = tg_sum3(tg_mul(px[3 * r], px[cc]), tg_mul(px[3 * r + 1], px[3 + cc]),
                                tg_mul(px[3 * r + 2], px[6 + cc]));
  Tg R[9], v[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    const Tg id = {(e == 0 || e == 4 || e == 8) ? 1.0 : 0.0, 0.0};
    R[e] = tg_add(tg_add(id, tg_mul(a, px[e])), tg_mul(b, px2[e]));
    v[e] = tg_add(tg_add(id, tg_mul(b, px[e])), tg_mul(c, px2[e]));
  }
  Tg tv[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) tv[r] = tg_sum3(tg_mul(v[3 * r], xi[0]), tg_mul(v[3 * r + 1], xi[1]), tg_mul(v[3 * r + 2], xi[2]));
  // compose(exp, cur): R = R_ex R_cur, t = R_ex t_cur + t_ex
  Tg cr[12];
#pragma unroll
  for (int e = 0; e < 12; ++e) cr[e] = {ls->prev[e], cur_im[e]};
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
      out_im[3 * r + cc] =
          tg_sum3(tg_mul(R[3 * r], cr[cc]), tg_mul(R[3 * r + 1], cr[3 + cc]), tg_mul(R[3 * r + 2], cr[6 + cc])).im;
    out_im[9 + r] =
        tg_add(tg_sum3(tg_mul(R[3 * r], cr[9]), tg_mul(R[3 * r + 1], cr[10]), tg_mul(R[3 * r + 2], cr[11])), tv[r]).im;
  }
}

__device__ __noinline__ void real_step(const IcpLevelArgs& a, const double* s_tot, double* s_pose,
                                       LevelSolveShared* ls, bool revert, unsigned seq, int it) {
  const int C = 1 + a.Dp;
  double x[6];
  if (revert) {
#pragma unroll
    for (int i = 0; i < 6; ++i) x[i] = 0.0;
  } else {
    double nb[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) nb[i] = -s_tot[(21 + i) * C];
    ldlt6_apply_smem(ls->fm, ls->ftr, nb, x);
    bool fin = true;
#pragma unroll
    for (int i = 0; i < 6; ++i) fin = fin && isfinite(x[i]);
    ls->fin_re = fin ? 1 : 0;
    if (!fin)
#pragma unroll
      for (int i = 0; i < 6; ++i) x[i] = 0.0;
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) ls->x[i] = x[i];
  Pose<double> cur;
#pragma unroll
  for (int e = 0; e < 9; ++e) cur.R.m[e] = ls->prev[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) cur.t.v[e] = ls->prev[9 + e];
  lv_mark(seq, it, 11);
  const Pose<double> ex = exp_map_record(x, ls);
  lv_mark(seq, it, 12);
  const Pose<double> np = compose(ex, cur);  // apply_increment (se3.hpp:116-119)
#pragma unroll
  for (int e = 0; e < 9; ++e) s_pose[e * C] = np.R.m[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) s_pose[(9 + e) * C] = np.t.v[e];
  double sq[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) sq[i] = x[i] * x[i];
  const double nrm = sqrt((sq[0] + (sq[1] + sq[2])) + (sq[3] + (sq[4] + sq[5])));
  ls->done = 0;
  ls->conv = 0;
  if (nrm < a.tol) {
    ls->done = 1;
    ls->conv = a.level == 0 ? 1 : 0;
  }
}

__device__ __noinline__ void channel_step(const IcpLevelArgs& a, const double* s_tot, double* s_pose,
                                          LevelSolveShared* ls) {
  const int C = 1 + a.Dp;
  const int lane = threadIdx.x & 31;
  const bool mine = lane < a.Dp;
  const int ch = 1 + lane;
  L<1> d[6];
  bool fin = true;
  if (mine) {
    // the real step (the same bits as real_step's)
    double nb[6], x[6], rhs[6], dx[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) nb[i] = -s_tot[(21 + i) * C];
    ldlt6_apply_smem(ls->fm, ls->ftr, nb, x);
#pragma unroll
    for (int i = 0; i < 6; ++i) fin = fin && isfinite(x[i]);
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      double ax = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) ax = ax + s_tot[(i >= j ? tri(i, j) : tri(j, i)) * C + ch] * x[j];
      rhs[i] = -s_tot[(21 + i) * C + ch] - ax;
    }
    ldlt6_apply_smem(ls->fm, ls->ftr, rhs, dx);
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      d[i].re = x[i];
      d[i].im[0] = dx[i];
      fin = fin && isfinite(dx[i]);
    }
  }
  const bool all_fin = __all_sync(0xffffffffu, !mine || fin);
  // real_step's intermediates (named barrier 2: warp 0 arrives after it)
  asm volatile("bar.sync 2, 64;" ::: "memory");
  if (!mine) return;
  double cur_im[12], out_im[12];
#pragma unroll
  for (int e = 0; e < 12; ++e) cur_im[e] = s_pose[e * C + ch];
  if (all_fin && !ls->small) {
    double xr[6], xim[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      xr[i] = d[i].re;
      xim[i] = d[i].im[0];
    }
    increment_pose_tangent(xr, xim, ls, cur_im, out_im);
  } else {
    if (!all_fin)
#pragma unroll
      for (int i = 0; i < 6; ++i) d[i] = lit<L<1>>(0.0);
    Pose<L<1>> cur, np;
#pragma unroll
    for (int e = 0; e < 12; ++e) {
      L<1> v;
      v.re = ls->prev[e];
      v.im[0] = cur_im[e];
      if (e < 9) cur.R.m[e] = v;
      else cur.t.v[e - 9] = v;
    }
    increment_pose(d, cur, &np);
#pragma unroll
    for (int e = 0; e < 9; ++e) out_im[e] = np.R.m[e].im[0];
#pragma unroll
    for (int e = 0; e < 3; ++e) out_im[9 + e] = np.t.v[e].im[0];
  }
#pragma unroll
  for (int e = 0; e < 12; ++e) s_pose[e * C + ch] = out_im[e];
  if (lane == 0 && !all_fin) ls->finite = 0;
}

// Debug timeline (tools/icp_timing.py, csf_debug_icp_clock): per launch, CTA,
// iteration and phase, the %globaltimer in ns (64 launches x 256 CTAs x 32
// iterations x 16 phases); off (nullptr) by default.
__device__ unsigned long long* g_lv_clock = nullptr;
__device__ unsigned g_lv_seq = 0;
__device__ __forceinline__ void lv_mark(unsigned seq, int it, int phase, int by) {
  unsigned long long* b = g_lv_clock;
  if (b && threadIdx.x == by && it < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    b[((static_cast<unsigned long long>(seq & 63) * 256 + blockIdx.x) * 32 + it) * 16 + phase] = t;
  }
}

__global__ void __launch_bounds__(kLvThreads, 1) k_icp_level(IcpLevelArgs a) {
  // launched without the programmatic attribute, but a captured graph may
  // still give it a programmatic edge from the preceding PDL kernel: wait for
  // that kernel's memory (a no-op otherwise)
  pdl_wait();
  extern __shared__ double sm[];
  const int C = 1 + a.Dp;
  const int n_acc = 27 * C;
  double* s_pose = sm;                                        // [12][C]
  double* s_intr = s_pose + 12 * C;                           // [4][C]
  double* s_tot = s_intr + 4 * C;                             // [27][C]
  double* s_rec = s_tot + n_acc;                              // [kRecFields][kSegSlots]
  double* s_meas = s_rec + kRecFields * kSegSlots;            // [6][kSegSlots]
  int* s_m = reinterpret_cast<int*>(s_meas + 6 * kSegSlots);  // [kSegSlots]
  __shared__ int s_wsum[kRounds * kLvWarps];
  __shared__ int s_n, s_last, s_na;
  __shared__ LevelSolveShared ls;
  __shared__ double s_w2p[12];
  __shared__ unsigned s_gen;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;
  for (int i = tid; i < 12 * C; i += blockDim.x) s_pose[i] = a.pose[i];
  for (int i = tid; i < 4 * C; i += blockDim.x) s_intr[i] = a.intr[i];
  if (tid < 12) s_w2p[tid] = a.st->pred_w2c[tid];
  const unsigned seq = g_lv_clock ? *(volatile unsigned*)&g_lv_seq : 0u;
  if (tid == 0) s_gen = acquire_gen(a.sync + kFlagWord);
  __syncthreads();
  const unsigned gen = s_gen;
  Pose<double> w2p;
#pragma unroll
  for (int e = 0; e < 9; ++e) w2p.R.m[e] = s_w2p[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) w2p.t.v[e] = s_w2p[9 + e];

  const int nxs = (a.w + a.stride - 1) / a.stride, nys = (a.h + a.stride - 1) / a.stride;
  const int n_slots = nxs * nys;
  const int t0 = tile * a.tile_slots;
  const int t1 = min(n_slots, t0 + a.tile_slots);
  const int n_segs = (t1 - t0 + kSegSlots - 1) / kSegSlots;
  const int passes = (C + kLvWarps - 1) / kLvWarps;
  const int n_groups = (a.n_tiles + kLvGroup - 1) / kLvGroup;
  const int grp = tile / kLvGroup;
  int taken = 0, last_n = 0;
  double last_delta[6] = {0, 0, 0, 0, 0, 0}, last_b[6] = {0, 0, 0, 0, 0, 0};
  bool converged = false;
  // single-segment tiles (VGA and below): the measured side once per level
  if (n_segs == 1) level_measure(a, t0, t1, s_intr, s_meas);
  // overlapped solve: the channel step of iteration k runs on the channel warp
  // while warps 0..kAsWarps-1 associate iteration k + 1
  const bool overlap = n_segs == 1 && passes == 1 && a.Dp >= 1 && a.Dp < 32;
  bool pre_assoc = false;  // this iteration's association already ran

  for (int it = 0; it < a.iterations; ++it) {
    lv_mark(seq, it, 0);
    // ---- A + B: this tile's partial normal equations, segment by segment
    // (one segment at VGA; a multi-segment tile re-associates per pass)
    int count = 0;
    for (int p = 0; p < passes; ++p) {
      const int c = warp + kLvWarps * p;
      double acc[27];
#pragma unroll
      for (int q = 0; q < 27; ++q) acc[q] = 0.0;
      int ebase = 0;
      for (int sg = 0; sg < n_segs; ++sg) {
        int n;
        if (pre_assoc) {
          n = s_na;
        } else if (n_segs > 1 || p == 0) {
          __syncthreads();  // the previous segment's records are consumed
          const int s0 = t0 + sg * kSegSlots, s1 = min(t1, s0 + kSegSlots);
          if (n_segs > 1) {
            level_measure(a, s0, s1, s_intr, s_meas);
            __syncthreads();
          }
          if (warp < kAsWarps) {
            n = level_associate(a, s0, s1, s_pose, s_intr, w2p, s_meas, s_rec, s_m, s_wsum);
            if (tid == 0) s_na = n;
          }
          __syncthreads();
          n = s_na;
          if (tid == 0) s_n = n;  // kept for the passes that reuse the records
        } else {
          n = s_n;
        }
        if (p == 0) count += n;
        if (p == 0 && sg == 0) lv_mark(seq, it, 1);
        if (c < C) level_accumulate(a, c, ebase, 0, n, s_pose, s_intr, s_rec, s_m, acc);
        ebase += n;
      }
      if (c < C) {
        // the 32 streams: fixed xor butterfly (every lane ends with the total)
#pragma unroll
        for (int q = 0; q < 27; ++q) {
          double v = acc[q];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, off);
          acc[q] = v;
        }
        double mine = 0.0;
#pragma unroll
        for (int q = 0; q < 27; ++q)
          if (lane == q) mine = acc[q];
        if (lane < 27) a.partials[static_cast<long long>(tile) * n_acc + lane * C + c] = mine;
      }
    }
    if (tid == 0) a.counts[tile] = count;
    // ---- C: group sums in tile order, then group totals in group order.
    // One thread per CTA publishes with an acq_rel atomic after the CTA
    // barrier (the barrier orders the CTA's partial writes before it); the
    // last arrival reads the others' partials through L2 (__ldcg).
    __syncthreads();
    lv_mark(seq, it, 2);
    const int first = grp * kLvGroup;
    const int gn = min(kLvGroup, a.n_tiles - first);
    if (tid == 0) s_last = atom_add_acq_rel(a.sync + grp, 1u) == static_cast<unsigned>(gn - 1);
    __syncthreads();
    if (s_last) {
      if (tid == 0) a.sync[grp] = 0u;
      for (int q = tid; q < n_acc; q += blockDim.x) {
        double v[kLvGroup];
#pragma unroll
        for (int u = 0; u < kLvGroup; ++u)
          v[u] = u < gn ? __ldcg(a.partials + static_cast<long long>(first + u) * n_acc + q) : 0.0;
        double total = 0.0;
#pragma unroll
        for (int u = 0; u < kLvGroup; ++u)
          if (u < gn) total = total + v[u];
        a.gpartials[static_cast<long long>(grp) * n_acc + q] = total;
      }
      if (tid < 32) {
        int cn = tid < gn ? __ldcg(a.counts + first + tid) : 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) cn += __shfl_down_sync(0xffffffffu, cn, off);
        if (tid == 0) a.counts[kLvMaxTiles + grp] = cn;
      }
      __syncthreads();
      lv_mark(seq, it, 6);
      // publish this group's total: its own generation flag
      if (tid == 0) release_gen(a.sync + kFlagWord + grp, gen + it + 1);
      lv_mark(seq, it, 3);
    }
    // ---- grid barrier: thread g waits for group g's flag (every CTA then
    // sums the group totals itself, in group order)
    if (tid < n_groups) {
      while (static_cast<int>(poll_gen(a.sync + kFlagWord + tid) - (gen + it + 1)) < 0) __nanosleep(32);
      fence_acquire();
    }
    __syncthreads();
    lv_mark(seq, it, 4);
    for (int q = tid; q < n_acc; q += blockDim.x) {
      double v[kLvMaxGroups];
#pragma unroll
      for (int g = 0; g < kLvMaxGroups; ++g)
        v[g] = g < n_groups ? __ldcg(a.gpartials + static_cast<long long>(g) * n_acc + q) : 0.0;
      double total = 0.0;
#pragma unroll
      for (int g = 0; g < kLvMaxGroups; ++g)
        if (g < n_groups) total = total + v[g];
      s_tot[q] = total;
    }
    if (tid < 32) {
      int cn = 0;
      for (int g = tid; g < n_groups; g += 32) cn += __ldcg(a.counts + kLvMaxTiles + g);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) cn += __shfl_down_sync(0xffffffffu, cn, off);
      if (tid == 0) s_n = cn;
    }
    if (tid == 0) {
      ls.done = 0;
      ls.conv = 0;
      ls.finite = 1;
    }
    if (tid < 12) ls.prev[tid] = s_pose[tid * C];  // the pose before the step (overlapped solve)
    __syncthreads();
    // ---- D: the solve (every CTA, identical bits)
    const int n = s_n;
    last_n = n;
    if (n < 12) break;  // icp.cpp:199, before the step
    double dre[6];
    if (tid < 32) ldlt6_warp(s_tot, C, &ls);
    __syncthreads();
    lv_mark(seq, it, 13);
    pre_assoc = false;
    if (overlap && !ls.degen) {
      if (warp == kAsWarps) {
        channel_step(a, s_tot, s_pose, &ls);
        lv_mark(seq, it, 14, 32 * kAsWarps);
      } else {
        if (tid == 0) real_step(a, s_tot, s_pose, &ls, false, seq, it);
        if (warp == 0) asm volatile("bar.arrive 2, 64;" ::: "memory");  // the channel warp may read ls
        assoc_barrier();
        lv_mark(seq, it, 8);
        if (!ls.done && it + 1 < a.iterations) {
          const int na = level_associate(a, t0, t1, s_pose, s_intr, w2p, s_meas, s_rec, s_m, s_wsum);
          if (tid == 0) s_na = na;
          lv_mark(seq, it, 15);
        }
      }
      __syncthreads();
      lv_mark(seq, it, 9);
      pre_assoc = !ls.done && it + 1 < a.iterations;
      if (!ls.finite && ls.fin_re) {
        // a channel of delta is not finite: delta = 0 (icp.cpp:45), the real
        // pose is exp(0) T of the saved one, and the next association reruns
        if (tid == 0) real_step(a, s_tot, s_pose, &ls, true, seq, it);
        __syncthreads();
        pre_assoc = false;
      }
      lv_mark(seq, it, 10);
#pragma unroll
      for (int i = 0; i < 6; ++i) dre[i] = tid == 0 ? ls.x[i] : 0.0;
    } else {
      level_solve(a, s_tot, s_pose, &ls, dre, seq, it, true);
    }
    lv_mark(seq, it, 5);
    ++taken;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      last_delta[i] = dre[i];
      last_b[i] = s_tot[(21 + i) * C];
    }
    __syncthreads();
    if (ls.done) {
      converged = ls.conv != 0;
      break;
    }
  }
  // the level's result: CTA 0 writes the pose and the tracker state
  if (blockIdx.x == 0) {
    __syncthreads();
    for (int i = tid; i < 12 * C; i += blockDim.x) a.pose[i] = s_pose[i];
    if (tid == 0) {
      TrackState* st = a.st;
      st->iterations += taken;
      st->n_corr = last_n;
      if (taken > 0) {
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          st->delta[i] = last_delta[i];
          st->b[i] = last_b[i];
        }
      }
      if (converged) st->converged = 1;
      st->level_done = 1;
      if (g_lv_clock) atomicAdd(&g_lv_seq, 1u);
    }
  }
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
    s[7] = 0;
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
constexpr int kR2Warps = 8;
constexpr int kR2Threads = 32 * kR2Warps;
constexpr int kR2RowStride = 7 * 4 + 1;  // doubles per correspondence row record (odd: conflict-free)
template <typename S> CSF_DEV void put_row(double* row, int i, const S& v) {
  row[4 * i] = v.re;
#pragma unroll
  for (int g = 0; g < 3; ++g) row[4 * i + 1 + g] = v.im[g];
}
template <typename S> CSF_DEV S get_row(const double* row, int i) {
  S v;
  v.re = row[4 * i];
#pragma unroll
  for (int g = 0; g < 3; ++g) v.im[g] = row[4 * i + 1 + g];
  return v;
}
constexpr int kR2Pairs = 5;  // pairs per CTA: one association serves them

template <typename S>
__global__ void __launch_bounds__(kR2Threads) k_icp_reduce2(const TrackState* st, const double* __restrict__ depth,
                                                             int w, int h, int stride, const double* __restrict__ intr,
                                                             const double* __restrict__ pose,
                                                             const double* __restrict__ vre,
                                                             const double* __restrict__ nre,
                                                             const double* __restrict__ vim,
                                                             const double* __restrict__ nim, double d_max,
                                                             double cos_max, int Dp, int tile_slots,
                                                             double* __restrict__ partials, int* __restrict__ counts) {
  pdl_wait();
  pdl_trigger();
  if (st->level_done) return;
  constexpr int G = Traits<S>::G;
  constexpr int CG = 1 + G;
  constexpr int NA = 27 * CG;  // accumulator threads
  const int C = 1 + Dp;
  const int n_pairs = Dp / G;
  extern __shared__ double sm[];
  // rows [kR2Threads][kR2RowStride] doubles: a correspondence's 7 row entries
  // (S = 4 doubles each) plus one pad double, so the odd stride puts the 32
  // lanes' 8-byte accesses on distinct bank pairs (stride 28: 4-way conflicts)
  double* rows = sm;
  int* s_corr = reinterpret_cast<int*>(rows + kR2Threads * kR2RowStride);  // [tile_slots][4]: x, y, u, v
  __shared__ int s_wsum[kR2Warps];
  Pose<double> c2w, w2p;
  load_pose_real(pose, C, &c2w);
#pragma unroll
  for (int e = 0; e < 9; ++e) w2p.R.m[e] = st->pred_w2c[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) w2p.t.v[e] = st->pred_w2c[9 + e];
  const double fx = intr[0], fy = intr[C], cx = intr[2 * C], cy = intr[3 * C];
  const int nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  const int n_slots = nxs * nys;
  const int t0 = blockIdx.x * tile_slots, t1 = min(n_slots, t0 + tile_slots);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // ---- the tile's association once for the CTA's kR2Pairs pairs: the
  // correspondences (pixel, model pixel) compacted in slot order
  int n_corr = 0;
  for (int c0 = t0; c0 < t1; c0 += kR2Threads) {
    const int slot = c0 + threadIdx.x;
    int x = 0, y = 0, u = 0, v = 0;
    bool corr = false;
    if (slot < t1) {
      x = (slot % nxs) * stride;
      y = (slot / nxs) * stride;
      corr = associate_slot(depth, w, h, x, y, fx, fy, cx, cy, c2w, w2p, vre, nre, d_max, cos_max, &u, &v);
    }
    const unsigned ballot = __ballot_sync(0xffffffffu, corr);
    __syncthreads();
    if (lane == 0) s_wsum[warp] = __popc(ballot);
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int k = 0; k < kR2Warps; ++k) {
      if (k < warp) before += s_wsum[k];
      total += s_wsum[k];
    }
    if (corr) {
      int* e4 = s_corr + 4 * (n_corr + before + __popc(ballot & ((1u << lane) - 1u)));
      e4[0] = x;
      e4[1] = y;
      e4[2] = u;
      e4[3] = v;
    }
    n_corr += total;
  }
  if (threadIdx.x == 0 && blockIdx.y == 0) counts[blockIdx.x] = n_corr;
  // ---- per pair: the rows in S and the canonical-order sums (§3.3): lane l
  // of every warp is stream l; warp w owns the accumulators q = w, w + 8,
  // w + 16, w + 24 (< 27), all components of S
  constexpr int kQ = (27 + kR2Warps - 1) / kR2Warps;
  const int pa = blockIdx.y * kR2Pairs, pb = min(n_pairs, pa + kR2Pairs);
  for (int pair = pa; pair < pb; ++pair) {
    const int g0 = pair * G;
    S acc[kQ];
#pragma unroll
    for (int i = 0; i < kQ; ++i) acc[i] = lit<S>(0.0);
    for (int e0 = 0; e0 < n_corr; e0 += kR2Threads) {
      const int e = e0 + threadIdx.x;
      __syncthreads();  // the previous chunk's rows are consumed (and s_corr is complete)
      if (e < n_corr) {
        const int* e4 = s_corr + 4 * e;
        const int x = e4[0], y = e4[1], u = e4[2], v = e4[3];
        // jacobian_row (icp.cpp:20-24): vertex = backproject(K, x, y, d) in S
        // (frames.hpp:38-41), p = base * vertex, r = (p - mv) . mn, J = [mn; p x mn]
        const double d = depth[y * w + x];
        const S kfx = load_ch<S>(intr, g0, G), kfy = load_ch<S>(intr + C, g0, G);
        const S kcx = load_ch<S>(intr + 2 * C, g0, G), kcy = load_ch<S>(intr + 3 * C, g0, G);
        const V3<S> vert = mk3<S>((d * (static_cast<double>(x) - kcx)) / kfx,
                                  (d * (static_cast<double>(y) - kcy)) / kfy, lit<S>(d));
        Pose<S> base;
#pragma unroll
        for (int q = 0; q < 9; ++q) base.R.m[q] = load_ch<S>(pose + q * C, g0, G);
#pragma unroll
        for (int q = 0; q < 3; ++q) base.t.v[q] = load_ch<S>(pose + (9 + q) * C, g0, G);
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
        double* row = rows + kR2RowStride * threadIdx.x;
        put_row(row, 0, mn.v[0]); put_row(row, 1, mn.v[1]); put_row(row, 2, mn.v[2]);
        put_row(row, 3, pn.v[0]); put_row(row, 4, pn.v[1]); put_row(row, 5, pn.v[2]);
        put_row(row, 6, r);
      }
      __syncthreads();
      // accumulate_row (orc_icp.hpp): lane l adds, in entry order, the S
      // product of the two row entries of every correspondence whose entry
      // index is l mod 32 (e0 is a multiple of 32)
      const int cnt = min(kR2Threads, n_corr - e0);
      for (int k = lane; k < cnt; k += 32) {
#pragma unroll
        for (int i = 0; i < kQ; ++i) {
          const int q = warp + kR2Warps * i;
          if (q < 27)
            acc[i] = acc[i] + get_row<S>(rows + kR2RowStride * k, acc_row_a(q)) *
                                  get_row<S>(rows + kR2RowStride * k, acc_row_b(q));
        }
      }
    }
    // the fixed butterfly of the first-order kernel, lane 0's value
#pragma unroll
    for (int i = 0; i < kQ; ++i) {
      const int q = warp + kR2Warps * i;
      double vv[CG];
      vv[0] = acc[i].re;
#pragma unroll
      for (int g = 0; g < G; ++g) vv[1 + g] = acc[i].im[g];
#pragma unroll
      for (int c = 0; c < CG; ++c)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) vv[c] = vv[c] + __shfl_xor_sync(0xffffffffu, vv[c], off);
      if (lane == 0 && q < 27) {
        double* dst = partials + static_cast<long long>(blockIdx.x) * 27 * C + q * C;
        if (pair == 0) dst[0] = vv[0];
#pragma unroll
        for (int g = 0; g < G; ++g) dst[g0 + 1 + g] = vv[1 + g];
      }
    }
  }
  (void)NA;
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
    // canonical two-level order: tiles in order within groups of kLvGroup,
    // group totals in order (oracle tiled_normal_equations)
    double total = 0.0;
    for (int t = 0; t < n_tiles; t += kLvGroup) {
      double vals[kLvGroup];
#pragma unroll
      for (int k = 0; k < kLvGroup; ++k)
        vals[k] = t + k < n_tiles ? __ldcg(partials + static_cast<long long>(t + k) * 27 * C + off) : 0.0;
      double gsum = 0.0;
#pragma unroll
      for (int k = 0; k < kLvGroup; ++k)
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

void icp_clock_enable(unsigned long long* buf) {
  cudaMemcpyToSymbol(g_lv_clock, &buf, sizeof(buf));
  const unsigned z = 0;
  cudaMemcpyToSymbol(g_lv_seq, &z, sizeof(z));
}

int icp_tiles(int w, int h, int stride) {
  const long long nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  const long long n = nxs * nys;
  const long long t = icp_tile_slots(n);
  return static_cast<int>((n + t - 1) / t);
}
bool icp_frame_fits(int w, int h, int stride) {
  const long long nxs = (w + stride - 1) / stride, nys = (h + stride - 1) / stride;
  return nxs * nys <= (1LL << 30) && icp_tiles(w, h, stride) <= kIcpMaxTiles;
}

void launch_level_begin(const Launch& L, TrackState* st, const double* pose, double* pred_pose, int Dp) {
  launch_pdl(k_level_begin, dim3(1), dim3(128), 0, L.stream, st, pose, pred_pose, Dp);
  ++*L.launches;
  chk("level_begin");
}

// Scratch of the level kernel (and of the second-order reduce, which uses the
// first kIcpMaxTiles rows / counts): partials [kIcpMaxTiles][27C], group
// totals [groups][27C], totals [27C]; counts [kIcpMaxTiles] + [groups] + [1],
// then the barrier words [groups] + [1] + [1] (zero at allocation, self-resetting).
size_t icp_partials_doubles(int C) {
  return static_cast<size_t>(kIcpMaxTiles + kLvMaxGroups + 1) * 27 * C;
}
size_t icp_counts_ints() { return static_cast<size_t>(kIcpMaxTiles + kLvMaxGroups + 1 + 64 + kFlagWord + 32); }

static size_t level_smem(int C) {
  return sizeof(double) * (43 * static_cast<size_t>(C) + (kRecFields + 6) * kSegSlots) + sizeof(int) * kSegSlots;
}

void launch_icp_level(const Launch& L, int Dp, TrackState* st, const double* depth, int w, int h, int stride,
                      const double* intr, double* pose, const double* vre, const double* nre, const double* vim,
                      const double* nim, double d_max, double cos_max, int iterations, int level, double tol,
                      double* partials, int* counts) {
  if (iterations <= 0) return;
  const int C = 1 + Dp;
  if (Dp > kMaxC - 1 || !icp_frame_fits(w, h, stride)) {
    note_error("csf_b200: ICP level too large (" + std::to_string(w) + "x" + std::to_string(h) + ") or too many "
               "channels (" + std::to_string(Dp) + ")");
    return;
  }
  IcpLevelArgs a{};
  a.st = st;
  a.depth = depth;
  a.w = w;
  a.h = h;
  a.stride = stride;
  a.intr = intr;
  a.pose = pose;
  a.vre = vre;
  a.nre = nre;
  a.vim = vim;
  a.nim = nim;
  a.d_max = d_max;
  a.cos_max = cos_max;
  a.Dp = Dp;
  a.iterations = iterations;
  a.level = level;
  a.tol = tol;
  const long long n_slots = static_cast<long long>((w + stride - 1) / stride) * ((h + stride - 1) / stride);
  a.tile_slots = icp_tile_slots(n_slots);
  a.n_tiles = icp_tiles(w, h, stride);
  const int n_acc = 27 * C;
  a.partials = partials;
  a.gpartials = partials + static_cast<size_t>(kIcpMaxTiles) * n_acc;
  a.totals = a.gpartials + static_cast<size_t>(kLvMaxGroups) * n_acc;
  a.counts = counts;
  // the barrier words start on their own 256-byte boundary (counts is cudaMalloc-aligned)
  a.sync = reinterpret_cast<unsigned*>(counts + ((kIcpMaxTiles + kLvMaxGroups + 1 + 63) / 64) * 64);
  const size_t smem = level_smem(C);
  ensure_dyn_smem(reinterpret_cast<const void*>(k_icp_level), smem);
  // every CTA waits at the level's grid barrier: a cooperative launch
  // guarantees they are co-resident (the tile count is capped for 2 CTAs/SM)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.n_tiles);
  cfg.blockDim = dim3(kLvThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = L.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_icp_level, a);
  if (e != cudaSuccess) {
    int per_sm = -1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_icp_level, kLvThreads, smem);
    note_error(std::string("launch of icp_level failed: ") + cudaGetErrorString(e) + " (" +
               std::to_string(a.n_tiles) + " tiles, " + std::to_string(per_sm) + " resident per SM at " +
               std::to_string(smem) + " B shared)");
  }
  ++*L.launches;
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
  const long long n_slots = static_cast<long long>((w + stride - 1) / stride) * ((h + stride - 1) / stride);
  const int tile_slots = icp_tile_slots(n_slots);
  const size_t smem = sizeof(double) * kR2Threads * kR2RowStride + sizeof(int) * 4 * static_cast<size_t>(tile_slots);
  launch_pdl(k_icp_reduce2<S>, dim3(tiles, (pairs + kR2Pairs - 1) / kR2Pairs), dim3(kR2Threads), smem, L.stream, st,
             depth, w, h, stride, intr,
             pose, vre, nre, vim, nim, d_max, cos_max, Dp, tile_slots, partials, counts);
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

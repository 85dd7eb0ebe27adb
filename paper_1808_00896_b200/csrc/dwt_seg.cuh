// Segment-parallel DWT on DMMA (round 2): the Wigner values go from the recurrence registers
// STRAIGHT into the DMMA operand -- no shared-memory Wigner tile.
//
// Same mathematics as dwt_mma.cuh (reference dwt.py:109-125, wigner.py:139-178): one symmetry
// cluster per CTA group, the base column d^l_{m,m'}(beta_j) from the rescaled three-term
// recurrence, shared by up to 8 members.  The kernels of dwt_mma.cuh run the recurrence with one
// beta index per lane and all degrees in sequence, so the 8 x 4 (degree x beta) DMMA fragment has
// to be transposed through a shared tile (1 024 wavefronts per 8 degrees of a cluster: the MIO
// pipe, not the FP64 pipe, bounded those kernels at 56-60 % of the DMMA peak).  Here the degrees
// l = m .. B-1 of a cluster are cut into 8 SEGMENTS of SL = ceil((B-m)/8), and lane (r, k) of a
// warp runs the recurrence of segment r at beta index 4g + k: at step t the 32 lanes hold
// exactly the m8n8k4 fragment W[l = m + r SL + t][beta = 4g + k].  A three-term recurrence can
// start in the middle only from two consecutive values, so the plan stores them: the checkpoint
// table ck[cluster][r][j] = (e^{l_r}(beta_j), e^{l_r - 1}(beta_j)), l_r = m + r SL, written once
// per plan by dwt_checkpoint_kernel with the SAME fma sequence the transforms use (the values
// every lane works with are bit-identical to one uninterrupted recurrence).  16 bytes x 8 x 2B per
// cluster: 17.2 GB at B = 512, read once per DWT beside the 17.2 GB spectrum; the DWT stays
// FP64-bound.
//
//  analysis   C[seg r][member] += W[r][beta k] * X[beta k][member]  (re and im as two DMMAs):
//             a warp owns 4 NB beta indices (NB groups), keeps X and the recurrence state in
//             registers, and emits one 8 x 16 partial tile per step; the warps of a CTA meet in
//             shared memory every TB steps (fixed order), CTAs of a split cluster in global
//             memory (SplitArgs, as dwt_mma.cuh).
//  synthesis  G[beta r][member] += W^T[beta r][seg k] * F[seg k][member]: 4 segments of 2 SL
//             (checkpoint rows 0, 2, 4, 6), accumulators in registers for the whole cluster,
//             the signed mu-scaled coefficients staged in shared memory one tile ahead.
//
// Requires B % 64 == 0 (a warp's 64 beta indices lie on one side of pi/2: one rec_t table half).
#pragma once
#include "dwt_mma.cuh"

namespace so3 {

constexpr int kSegRows = 8;          // checkpoint rows (degree segments) per cluster
constexpr int kSegMaxSL = 64;        // ceil(512 / 8)
constexpr int kSegBeta = 64;         // beta indices per warp

__host__ __device__ __forceinline__ int seg_len(int nsteps) { return (nsteps + kSegRows - 1) / kSegRows; }

// One thread per (cluster, beta index): the whole recurrence once, the state written at the 8
// segment starts.  Same table entries and fma order as the transforms.
__global__ void __launch_bounds__(128) dwt_checkpoint_kernel(DwtArgs a, double2* ck) {
  const int c = blockIdx.x;   // clusters on grid.x (131 328 at B = 512)
  const int j = blockIdx.y * 128 + threadIdx.x;
  const int n = a.n;
  if (j >= n) return;
  const int2 base = __ldg(&a.bases[c]);
  const int m = base.x, mp = base.y;
  const int nsteps = a.B - m, SL = seg_len(nsteps);
  const double* rct = a.rc + 3 * __ldg(&a.rc_off[c]);
  const double x = __ldg(&a.xv[j]);
  const bool up = 2 * j >= n;
  double cur = seed_value(m, mp, __ldg(&a.lnorm[c]), a.logcs[j]);
  double prev = 0.0;
  double2* out = ck + (long long)c * kSegRows * n + j;
  int r = 0, left = 0;
  for (int i = 0; i < nsteps; ++i) {
    if (left == 0) {
      out[(long long)r * n] = make_double2(cur, prev);
      ++r;
      left = SL;
    }
    --left;
    const double al = __ldg(&rct[3 * i]), cp = __ldg(&rct[3 * i + 1]);
    const double nx = fma(fma(al, x, up ? fma(-2.0, al, cp) : cp), cur, -prev);
    prev = cur;
    cur = nx;
  }
  for (; r < kSegRows; ++r) out[(long long)r * n] = make_double2(0.0, 0.0);
}

// Shared table of a cluster's (alpha_l, C_l) entries for both halves of [0, pi] (rec_t), rows of
// SLP (odd) entries so the per-lane-row LDS.128 of one step touch distinct banks; zero past the
// last degree.  rows * SL entries, entry index i = row * SL + t.
__device__ __forceinline__ void seg_stage_table(double2* lo, double2* hi, const double* rct, int rows, int SL, int SLP,
                                                int nsteps, int t, int nt) {
  const int lane = t & 31, nw = nt >> 5;
  for (int rr = t >> 5; rr < rows; rr += nw)   // a table row per warp: no division per entry
    for (int tt = lane; tt < SL; tt += 32) {
      const int i = rr * SL + tt;
      double al = 0.0, cp = 0.0;
      if (i < nsteps) {
        al = __ldg(&rct[3 * i]);
        cp = __ldg(&rct[3 * i + 1]);
      }
      lo[rr * SLP + tt] = make_double2(al, cp);
      hi[rr * SLP + tt] = make_double2(al, fma(-2.0, al, cp));
    }
}

constexpr int kSegTabA = kSegRows * (kSegMaxSL + 1);      // double2 per half, analysis (8 rows)
constexpr int kSegTabS = 4 * (2 * kSegMaxSL + 1);         // double2 per half, synthesis (4 rows)

// Analysis.  Grid (clusters x SPLIT, batch); W = blockDim.x / 32 warps, each over 4 NB beta
// indices; SPLIT x W x 4 NB = 2B.
template <int NB, int SPLIT, int TB, int MINB, int WT = 8>
__global__ void __launch_bounds__(WT * 32, MINB) dwt_analysis_seg_kernel(DwtArgs a, SplitArgs sp, const double2* ck) {
  extern __shared__ double dsm[];
  __shared__ Member mem[8];
  double2* rcs = reinterpret_cast<double2*>(dsm);                  // [2][8][SLP]
  double2* part = reinterpret_cast<double2*>(dsm) + 2 * kSegTabA;   // [2][TB][W][64]

  const int c = a.cluster0 + blockIdx.x / SPLIT;
  const int half = SPLIT > 1 ? (int)(blockIdx.x % SPLIT) : 0;
  const int f = blockIdx.y;
  const int2 base = __ldg(&a.bases[c]);
  const int m = base.x, mp = base.y;
  const int B = a.B, n = a.n;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, W = blockDim.x >> 5;
  const int r = lane >> 2, k = lane & 3;
  const long long rco = __ldg(&a.rc_off[c]);
  const double* rct = a.rc + 3 * rco;
  const int nsteps = B - m, SL = seg_len(nsteps), SLP = SL | 1;

  if (t < 8) mem[t] = member_of(a, m, mp, t);
  seg_stage_table(rcs, rcs + kSegTabA, rct, kSegRows, SL, SLP, nsteps, t, blockDim.x);
  __syncthreads();

  const int jw0 = (half * W + warp) * (4 * NB);
  const double2* rw = rcs + (2 * jw0 >= n ? kSegTabA : 0) + r * SLP;
  double cur[NB], prev[NB], v[NB], xr[NB], xi[NB];
  {
    const Member M = mem[r];   // lane (r, k) supplies column r (member r) of X at its beta index
    const double2* spec = a.spec + (long long)f * a.spec_fstride;
    const double2* ckp = ck + ((long long)c * kSegRows + r) * n;
#pragma unroll
    for (int g = 0; g < NB; ++g) {
      const int j = jw0 + 4 * g + k;
      const double2 s = __ldg(&ckp[j]);
      cur[g] = s.x;
      prev[g] = s.y;
      v[g] = __ldg(&a.xv[j]);
      double2 z = make_double2(0.0, 0.0);
      if (M.valid) z = spec[spec_index(a, M.row, M.reflect ? n - 1 - j : j)];
      xr[g] = z.x;
      xi[g] = z.y;
    }
  }

  const double vscale = 8.0 * 3.141592653589793 * (double)B;

  const double rvscale = 1.0 / vscale;   // one division per thread, not one per output
  int buf = 0;
  for (int t0 = 0; t0 < SL; t0 += TB, buf ^= 1) {
    const int nt = min(TB, SL - t0);
    double2* pw = part + ((size_t)buf * TB * W + warp) * 64 + lane;
#pragma unroll 2
    for (int tb = 0; tb < nt; ++tb) {
      const double2 k2 = rw[t0 + tb];
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
      for (int g = 0; g < NB; ++g) {
        dmma884(a0, a1, cur[g], xr[g]);
        dmma884(b0, b1, cur[g], xi[g]);
        const double nx = fma(fma(k2.x, v[g], k2.y), cur[g], -prev[g]);
        prev[g] = cur[g];
        cur[g] = nx;
      }
      // lane (r, k) holds segment r, members 2k (a0, b0) and 2k + 1 (a1, b1) as (re, im)
      pw[(size_t)tb * W * 64] = make_double2(a0, b0);
      pw[(size_t)tb * W * 64 + 32] = make_double2(a1, b1);
    }
    __syncthreads();   // every warp's partials of these nt steps are visible
    for (int idx = t; idx < nt * 64; idx += blockDim.x) {
      const int tb = idx >> 6, o = idx & 63;
      const int mm = 2 * (o & 3) + (o >> 5), rr = (o >> 2) & 7;
      const int i = rr * SL + t0 + tb;   // degree l = m + i
      const double2* pb = part + (size_t)(buf * TB + tb) * W * 64 + o;
      double2 vv[WT];
#pragma unroll
      for (int w = 0; w < WT; ++w) vv[w] = w < W ? pb[w * 64] : make_double2(0.0, 0.0);
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int w = 0; w < WT; ++w) {   // fixed order
        re += vv[w].x;
        im += vv[w].y;
      }
      const Member M = mem[mm];
      if (i >= nsteps || !M.valid) continue;
      if constexpr (SPLIT > 1) {
        sp.pbuf[half * sp.pstride + (rco + i) * 8 + mm] = make_double2(re, im);
      } else {
        const int l = m + i;
        double sc = (2.0 * l + 1.0) * rvscale * __ldg(&rct[3 * i + 2]);   // v_l * mu_l
        if ((M.sl * l + M.par0) & 1) sc = -sc;
        a.coef[(long long)f * a.coef_fstride + coeff_slot32(l, M.pm, M.pmp)] = make_double2(re * sc, im * sc);
      }
    }
    // the next TB steps write the other buffer; this one is rewritten only after the next
    // __syncthreads, which every reader has passed
  }
  if constexpr (SPLIT > 1) {
    __shared__ int s_last;
    __syncthreads();   // every thread's partial stores are issued
    if (t == 0) {
      __threadfence();
      const unsigned prv = atomicInc(&sp.pcnt[c], SPLIT - 1u);   // wraps to 0: re-armed for the next launch
      s_last = prv == SPLIT - 1;
      if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last) return;
    for (int idx = t; idx < nsteps * 8; idx += blockDim.x) {
      const int mm = idx & 7, i = idx >> 3, l = m + i;
      const Member M = mem[mm];
      if (!M.valid) continue;
      const long long o = (rco + i) * 8 + mm;
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int h = 0; h < SPLIT; ++h) {   // fixed order, whichever CTA arrives last
        const double2 ph = __ldcg(&sp.pbuf[h * sp.pstride + o]);
        re += ph.x;
        im += ph.y;
      }
      double sc = (2.0 * l + 1.0) * rvscale * __ldg(&rct[3 * i + 2]);
      if ((M.sl * l + M.par0) & 1) sc = -sc;
      a.coef[(long long)f * a.coef_fstride + coeff_slot32(l, M.pm, M.pmp)] = make_double2(re * sc, im * sc);
    }
  }
}

// CTA-wide split barrier on an mbarrier: arrive when this thread's shared-memory writes are done,
// wait (much later) before reading the other threads' -- a warp stalls only if another warp is a
// whole tile behind, where __syncthreads stalls on every skew.
__device__ __forceinline__ void seg_bar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void seg_bar_arrive(unsigned long long* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void seg_bar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned addr = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done)
                 : "r"(addr), "r"(parity)
                 : "memory");
  } while (!done);
}

// ---- persistent analysis -------------------------------------------------------------------
// Above, a CTA lives for one (cluster, beta part): its prologue (three dependent global round
// trips) and the final combine of a split cluster are exposed, because 236 registers per thread
// leave one or two CTAs per SM (ncu: DMMA pipe 51 %).  Here one CTA per SM (two for W = 4) walks
// its share of the clusters, and thread 0 streams the NEXT pass's operands -- 8 checkpoint rows,
// up to 8 member rows of the spectrum, v_j and the cluster's recurrence table -- into shared
// memory with 1-D bulk copies (cp.async.bulk, one mbarrier) while the warps work on the current
// pass, so a prologue is shared-memory reads.  A CTA covers W x 64 beta indices per pass and runs
// the passes of a cluster (2 at 2B = 1024) back to back: pass 0 leaves its per-degree sums in
// SplitArgs::pbuf, the last pass adds them to its own in pass order -- same CTA, so no counter,
// no fence and no combine sweep.  Clusters go to CTAs in snake order over the cost-sorted schedule.

__device__ __forceinline__ unsigned seg_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void seg_bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(seg_smem(dst)),
               "l"(src), "r"(bytes), "r"(seg_smem(bar))
               : "memory");
}
__device__ __forceinline__ void seg_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(seg_smem(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool seg_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned done;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(done)
               : "r"(seg_smem(bar)), "r"(parity)
               : "memory");
  return done != 0;
}

constexpr int kSegTabP = 2 * kSegRows * (kSegMaxSL / 2 + 1);   // 528 double2 >= one half at SL <= 64, two at SL <= 32
constexpr int kSegRawTab = 3 * 512;                             // doubles: a cluster's (alpha, C+, mu) entries

__host__ __device__ inline size_t segp_smem_bytes(int W, int TB) {
  const size_t RS = (size_t)W * kSegBeta + 4;
  return 2 * kSegRows * RS * 16 + (size_t)W * kSegBeta * 8 + kSegRawTab * 8 + kSegTabP * 16 + 512 * 8 +
         (size_t)2 * TB * W * 64 * 16;
}

// Measured and dropped (B = 512, one B200; this version: see DESIGN.md): a split mbarrier per batch
// with three partial buffers (36.8 ms: warps still wait for the slowest one, one batch later), and a
// barrier-free ring of per-step partial tiles reduced kSegLag steps later by all warps (47 ms: the
// mbarrier polls between the steps keep the compiler from overlapping one step's DFMAs with the
// next step's DMMAs).
// FULLW: the CTA has exactly WT warps (the common shapes: 8 warps at B = 256 and 512, 4 at B = 128);
// the reduction then has compile-time trip counts and no warp-count selects (it was ~400 SASS
// instructions per batch and thread, issue-bound: ncu, 9 % of the kernel's warp time).
template <int NB, int TB, int WT, int MINB, bool FULLW = false>
__global__ void __launch_bounds__(WT * 32, MINB) dwt_analysis_segp_kernel(DwtArgs a, SplitArgs sp, const double2* ck, int ncl,
                                                                           int halves) {
  static_assert(4 * NB == kSegBeta, "a warp covers kSegBeta beta indices");
  // outputs per thread and batch: TB x 64 outputs over the CTA's threads (>= 128 when not FULLW)
  constexpr int OPT = FULLW ? (TB * 64 + WT * 32 - 1) / (WT * 32) : 2;
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ Member mem[8];
  __shared__ unsigned long long bar;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int W = FULLW ? WT : (int)(blockDim.x >> 5), NT = FULLW ? WT * 32 : (int)blockDim.x;
  const int r = lane >> 2, k = lane & 3;
  const int WB = W * kSegBeta, RS = WB + 4;   // row stride: +64 bytes, rows r and r+1 of a quarter-warp on distinct banks
  double2* ckS = reinterpret_cast<double2*>(smraw);   // [8][RS] checkpoint rows of the pass
  double2* xS = ckS + kSegRows * RS;                  // [8][RS] member rows of the spectrum (mirror ranges for reflecting members)
  double* vS = reinterpret_cast<double*>(xS + kSegRows * RS);   // [WB]
  double* rcS = vS + WB;                              // raw table of the cluster
  double2* rcs = reinterpret_cast<double2*>(rcS + kSegRawTab);   // padded (alpha, C) rows, one or both halves
  double* mus = reinterpret_cast<double*>(rcs + kSegTabP);       // mu_l of the cluster
  double2* part = reinterpret_cast<double2*>(mus + 512);          // [2][TB][W][64]
  const int B = a.B, n = a.n;
  const int G = gridDim.x, b = blockIdx.x;
  const double vscale = 8.0 * 3.141592653589793 * (double)B;
  const double rvscale = 1.0 / vscale;   // one division per thread, not one per output

  // round i of the snake: cluster i G + b (even i) or i G + G - 1 - b (odd i)
  auto cluster_of = [&](int i) { return i * G + ((i & 1) ? G - 1 - b : b); };
  // The operands of pass h of cluster c (base m, m') into the stage buffers: 18 bulk copies (8
  // checkpoint rows, 8 member rows, v_j, the recurrence table), copy ci by lane 0 of warp ci mod W,
  // so no warp falls behind the others by issuing them all (every batch barrier waits for the
  // slowest warp).  Thread 0 registers the byte count first (prefetch_expect, before the barrier
  // that frees the buffers); the copies follow it (prefetch_issue).
  auto prefetch_expect = [&](int h, int m, int mp) {
    const int nsteps = B - m;
    const int nvalid = m == 0 ? 1 : (mp == 0 || mp == m) ? 4 : 8;
    const unsigned tabb = h == 0 ? (unsigned)(((nsteps + 1) & ~1) * 24) : 0u;
    seg_expect_tx(&bar, (unsigned)((kSegRows + nvalid) * WB * 16 + WB * 8) + tabb);
  };
  auto prefetch_issue = [&](int c, int h, int m, int mp, long long rco) {
    if (lane != 0) return;
    const int j0 = h * WB;
    for (int ci = warp; ci < 18; ci += W) {
      if (ci < 8) {
        seg_bulk_load(ckS + ci * RS, ck + ((long long)c * kSegRows + ci) * n + j0, WB * 16, &bar);
      } else if (ci < 16) {
        const Member M = make_member(m, mp, ci - 8, n);
        if (M.valid) seg_bulk_load(xS + (ci - 8) * RS, a.spec + M.row * n + (M.reflect ? n - j0 - WB : j0), WB * 16, &bar);
      } else if (ci == 16) {
        seg_bulk_load(vS, a.xv + j0, WB * 8, &bar);
      } else if (h == 0) {
        seg_bulk_load(rcS, a.rc + 3 * rco, (unsigned)(((B - m + 1) & ~1) * 24), &bar);
      }
    }
  };

  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(seg_smem(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int c0 = cluster_of(0);
  if (c0 >= ncl) return;
  // (m, m', table offset) of the current cluster and of the next one, loaded a pass ahead
  int2 base = __ldg(&a.bases[a.cluster0 + c0]);
  long long rco = __ldg(&a.rc_off[a.cluster0 + c0]);
  if (t == 0) prefetch_expect(0, base.x, base.y);
  __syncthreads();
  prefetch_issue(a.cluster0 + c0, 0, base.x, base.y, rco);
  unsigned parity = 0;
  for (int i = 0;; ++i) {
    const int c = a.cluster0 + cluster_of(i);
    const int cn = cluster_of(i + 1);
    int2 base_n = make_int2(0, 0);
    long long rco_n = 0;
    if (cn < ncl) {
      base_n = __ldg(&a.bases[a.cluster0 + cn]);
      rco_n = __ldg(&a.rc_off[a.cluster0 + cn]);
    }
    const int m = base.x, mp = base.y;
    const int nsteps = B - m, SL = seg_len(nsteps), SLP = SL | 1;
    for (int h = 0; h < halves; ++h) {
      while (!seg_try_wait(&bar, parity)) {}
      parity ^= 1;
      const int j0 = h * WB;
      // padded table rows and mu_l from the raw table (which stays until the next cluster's pass 0 arrives)
      if (h == 0 && lane == 0 && warp < 8) {   // a member per warp (W < 8: the remaining ones by warp 0)
        mem[warp] = make_member(m, mp, warp, n);
        if (warp == 0)
          for (int mmx = W; mmx < 8; ++mmx) mem[mmx] = make_member(m, mp, mmx, n);
      }
      const bool both = halves == 1;         // the CTA spans [0, pi): both table halves
      const bool upper_pass = 2 * j0 >= n;   // halves > 1: the pass lies in one half
      for (int rr = warp; rr < kSegRows; rr += W) {   // one table row per warp: no division per entry
        for (int tt = lane; tt < SL; tt += 32) {
          const int idx = rr * SL + tt;
          double al = 0.0, cp = 0.0;
          if (idx < nsteps) {
            al = rcS[3 * idx];
            cp = rcS[3 * idx + 1];
            if (h == 0) mus[idx] = rcS[3 * idx + 2];
          }
          if (both) {
            rcs[rr * SLP + tt] = make_double2(al, cp);
            rcs[kSegRows * SLP + rr * SLP + tt] = make_double2(al, fma(-2.0, al, cp));
          } else {
            rcs[rr * SLP + tt] = make_double2(al, upper_pass ? fma(-2.0, al, cp) : cp);
          }
        }
      }
      // operands of this warp from the stage buffers
      const int jl0 = warp * kSegBeta;
      double cur[NB], prev[NB], v[NB], xr[NB], xi[NB];
      {
        const Member M = make_member(m, mp, r, n);
        const double2* cr = ckS + r * RS + jl0 + k;
        const double2* xrow = xS + r * RS + (M.reflect ? WB - 1 - jl0 - k : jl0 + k);
        const int xstep = M.reflect ? -4 : 4;
#pragma unroll
        for (int g = 0; g < NB; ++g) {
          const double2 s = cr[4 * g];
          cur[g] = s.x;
          prev[g] = s.y;
          v[g] = vS[jl0 + 4 * g + k];
          double2 z = make_double2(0.0, 0.0);
          if (M.valid) z = xrow[xstep * g];
          xr[g] = z.x;
          xi[g] = z.y;
        }
      }
      if (t == 0) {   // the next pass's byte count: the other half of this cluster, or the next cluster
        if (h + 1 < halves) prefetch_expect(h + 1, m, mp);
        else if (cn < ncl) prefetch_expect(0, base_n.x, base_n.y);
      }
      __syncthreads();   // the stage buffers are free; the padded table, mu and the members are visible
      if (h + 1 < halves) prefetch_issue(c, h + 1, m, mp, rco);
      else if (cn < ncl) prefetch_issue(a.cluster0 + cn, 0, base_n.x, base_n.y, rco_n);
      const double2* rw = rcs + ((both && 2 * (j0 + jl0) >= n) ? kSegRows * SLP : 0) + r * SLP;
      const bool last = h + 1 == halves;
      // Per-pass constants of this thread's outputs: output q is entry o_q of step tb_q of every batch
      // (NT is a multiple of 64 for even W; odd W recomputes nothing either: idx = t + q NT is fixed).
      int o_tb[OPT], o_mm[OPT], o_i0[OPT], o_neg[OPT];
      bool o_ok[OPT];
      long long o_pm[OPT];
      const double2* o_pb[OPT];
#pragma unroll
      for (int q = 0; q < OPT; ++q) {
        const int idx = t + q * NT, tb = idx >> 6, o = idx & 63;
        const int mm = 2 * (o & 3) + (o >> 5);
        const Member M = mem[mm];
        o_tb[q] = tb;
        o_mm[q] = mm;
        o_i0[q] = ((o >> 2) & 7) * SL + tb;           // + t0 = degree index of the output
        o_ok[q] = tb < TB && M.valid;
        o_neg[q] = M.sl | (M.par0 << 1);               // sign (-1)^(sl l + par0)
        o_pm[q] = ((long long)M.pm << 32) | (unsigned)M.pmp;
        o_pb[q] = part + (size_t)tb * W * 64 + o;
      }
      int buf = 0;
      for (int t0 = 0; t0 < SL; t0 += TB, buf ^= 1) {
        const int nt = min(TB, SL - t0);
        // pass 0's sums of this thread's outputs of the batch go out before the batch's math
        double2 p0[OPT];
#pragma unroll
        for (int q = 0; q < OPT; ++q) {
          const int ii = o_i0[q] + t0;
          p0[q] = make_double2(0.0, 0.0);
          // volatile: the load leaves BEFORE the batch's DMMAs (ptxas may otherwise sink it to its use)
          if (h > 0 && o_ok[q] && o_tb[q] < nt && ii < nsteps)
            asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(p0[q].x), "=d"(p0[q].y) : "l"(&sp.pbuf[(rco + ii) * 8 + o_mm[q]]) : "memory");
        }
        double2* pw = part + ((size_t)buf * TB * W + warp) * 64 + lane;
#pragma unroll 2
        for (int tb = 0; tb < nt; ++tb) {
          const double2 k2 = rw[t0 + tb];
          double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
          for (int g = 0; g < NB; ++g) {
            dmma884(a0, a1, cur[g], xr[g]);
            dmma884(b0, b1, cur[g], xi[g]);
            const double nx = fma(fma(k2.x, v[g], k2.y), cur[g], -prev[g]);
            prev[g] = cur[g];
            cur[g] = nx;
          }
          // lane (r, k): segment r, members 2k (a0, b0) and 2k + 1 (a1, b1) as (re, im)
          pw[(size_t)tb * W * 64] = make_double2(a0, b0);
          pw[(size_t)tb * W * 64 + 32] = make_double2(a1, b1);
        }
        __syncthreads();   // every warp's partials of these nt steps are visible
#pragma unroll
        for (int q = 0; q < OPT; ++q) {
          const int ii = o_i0[q] + t0;   // degree l = m + ii
          if (!o_ok[q] || o_tb[q] >= nt || ii >= nsteps) continue;
          const double2* pb = o_pb[q] + (size_t)buf * TB * W * 64;
          double2 vv[WT];
#pragma unroll
          for (int w = 0; w < WT; ++w) vv[w] = (FULLW || w < W) ? pb[w * 64] : make_double2(0.0, 0.0);
          double re = 0.0, im = 0.0;
#pragma unroll
          for (int w = 0; w < WT; ++w) {   // fixed order
            re += vv[w].x;
            im += vv[w].y;
          }
          if (!last) {   // passes accumulate in pass order
            sp.pbuf[(rco + ii) * 8 + o_mm[q]] = make_double2(p0[q].x + re, p0[q].y + im);
          } else {
            const int l = m + ii;
            double sc = (2.0 * l + 1.0) * rvscale * mus[ii];   // v_l * mu_l
            if (((o_neg[q] & 1) * l + (o_neg[q] >> 1)) & 1) sc = -sc;
            a.coef[coeff_slot32(l, (int)(o_pm[q] >> 32), (int)o_pm[q])] = make_double2((p0[q].x + re) * sc, (p0[q].y + im) * sc);
          }
        }
        // the next TB steps write the other buffer; this one is rewritten only after the next
        // __syncthreads, which every reader has passed
      }
      __syncthreads();   // the last reducers are done with mem / mus / the table before the next pass rewrites them
    }
    if (cn >= ncl) break;
    base = base_n;
    rco = rco_n;
  }
}

// Synthesis.  Grid (clusters x split, batch); WPC warps per CTA, each over 8 NB beta indices
// (NB row groups); split x WPC x 8 NB = 2B.  Lane (r, k): beta row r of each group, degree segment
// k of 4 (length SL4 = 2 SL).
template <int NB, int WPC, int TB, int MINB>
__global__ void __launch_bounds__(WPC * 32, MINB) dwt_synthesis_seg_kernel(DwtArgs a, int split, const double2* ck) {
  constexpr int NT = WPC * 32;
  constexpr int FR = TB * 8 + 2;                  // double2 per segment region: TB degree rows of 8 + a 32-byte skew
  constexpr int PF = (4 * TB * 8 + NT - 1) / NT;   // prefetched coefficients per thread and tile
  __shared__ Member mem[8];
  __shared__ double2 rcs[2][kSegTabS];
  // F[seg k][step][col r] = (member r/2, member 4 + r/2), re for even r, im for odd r; the skew puts
  // the four segments' rows of one step on distinct banks.  Three tiles: tile i+1 is staged while
  // slower warps may still read tile i-1 (split barrier below).
  __shared__ double2 fco[3][4 * FR];
  __shared__ unsigned long long bar;

  const int c = a.cluster0 + blockIdx.x / split;
  const int crank = blockIdx.x % split;
  const int f = blockIdx.y;
  const int2 base = __ldg(&a.bases[c]);
  const long long rco = __ldg(&a.rc_off[c]);
  const int m = base.x, mp = base.y;
  const int B = a.B, n = a.n;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int r = lane >> 2, k = lane & 3;
  const double* rct = a.rc + 3 * rco;
  const int nsteps = B - m, SL4 = 2 * seg_len(nsteps), SLP = SL4 | 1;

  // the recurrence state goes out first: it needs neither the member table nor the shared table
  const int jw0 = (crank * WPC + warp) * (8 * NB);
  double cur[NB], prev[NB], v[NB], acc[NB][2][2];
  {
    const double2* ckp = ck + ((long long)c * kSegRows + 2 * k) * n;
#pragma unroll
    for (int g = 0; g < NB; ++g) {
      const int j = jw0 + 8 * g + r;
      const double2 s = __ldg(&ckp[j]);
      cur[g] = s.x;
      prev[g] = s.y;
      v[g] = __ldg(&a.xv[j]);
      acc[g][0][0] = acc[g][0][1] = acc[g][1][0] = acc[g][1][1] = 0.0;
    }
  }
  // item idx of the tile at step t0: member mm = idx & 7, step tb = (idx >> 3) % TB, segment idx / (8 TB)
  // (the loads stay in flight: nothing here consumes them; the sign is applied when staging)
  // NT is a multiple of 8: a thread fetches the same member mm = t & 7 in every tile, so its
  // relation lives in registers and the first tiles go out with the recurrence state
  static_assert(NT % 8 == 0 && TB % 2 == 0, "member per thread; the sign's parity is the same in every tile");
  const Member Mf = make_member(m, mp, t & 7, n);
  // Per-item constants of this thread (item q: member t & 7, step tb_q, segment kk_q of every tile):
  // first degree index i0, live while t0 < lim, sign (-1)^(sl l + par0) (TB even: the same parity in
  // every tile), destination in a staged tile.  The per-tile work is then a compare, a 32-bit slot
  // (coeff_slot32), two loads; two multiplies and two stores when staging -- the 64-bit slot
  // arithmetic and the index decoding per tile cost 1.7 ms of issue slots at B = 512.
  int it_i0[PF], it_lim[PF], it_dst[PF];
  bool it_neg[PF];
#pragma unroll
  for (int q = 0; q < PF; ++q) {
    const int idx = t + q * NT;
    const int mm = idx & 7, tb = (idx >> 3) % TB, kk = idx / (8 * TB);
    it_i0[q] = kk * SL4 + tb;
    it_lim[q] = (idx < 4 * TB * 8 && Mf.valid) ? min(SL4 - tb, nsteps - it_i0[q]) : 0;
    it_neg[q] = ((Mf.sl * (m + it_i0[q]) + Mf.par0) & 1) != 0;
    it_dst[q] = (kk * FR + tb * 8 + 2 * (mm & 3)) * 2 + (mm >> 2);   // in doubles
  }
  const double2* coef_f = a.coef + (long long)f * a.coef_fstride;
  auto fetch = [&](int t0, double2 (&pf)[PF], double (&pmu)[PF]) {
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      double2 z = make_double2(0.0, 0.0);
      double mu = 0.0;
      if (t0 < it_lim[q]) {
        const int i = it_i0[q] + t0;
        z = coef_f[coeff_slot32(m + i, Mf.pm, Mf.pmp)];
        mu = __ldg(&rct[3 * i + 2]);
      }
      pf[q] = z;
      pmu[q] = mu;
    }
  };
  auto stage = [&](int bsel, const double2 (&pf)[PF], const double (&pmu)[PF]) {
    double* tile = reinterpret_cast<double*>(fco[bsel]);
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      if (t + q * NT < 4 * TB * 8) {
        const double mu = it_neg[q] ? -pmu[q] : pmu[q];
        tile[it_dst[q]] = pf[q].x * mu;
        tile[it_dst[q] + 2] = pf[q].y * mu;
      }
    }
  };

  const double2* rw = rcs[2 * jw0 >= n ? 1 : 0] + k * SLP;
  double2 pf[PF], pf1[PF];
  double pmu[PF], pmu1[PF];
  fetch(0, pf1, pmu1);
  fetch(TB, pf, pmu);   // tile 1 (zeros past the last step)
  if (t < 8) mem[t] = member_of(a, m, mp, t);
  if (t == 0) seg_bar_init(&bar, NT);
  seg_stage_table(rcs[0], rcs[1], rct, 4, SL4, SLP, nsteps, t, NT);
  stage(0, pf1, pmu1);
  __syncthreads();

  // iteration i: stage tile i+1 (fetched during iteration i-1), arrive; fetch tile i+2; compute
  // tile i; wait for everyone's tile i+1.  Tile i+1 overwrites tile i-2, which every thread left
  // before its arrive of iteration i-1 -- and this thread has waited for those arrives.
  int bsel = 0;
  unsigned parity = 0;
  for (int t0 = 0; t0 < SL4; t0 += TB) {
    const int bnext = bsel == 2 ? 0 : bsel + 1;
    const bool more = t0 + TB < SL4;
    if (more) {
      stage(bnext, pf, pmu);
      seg_bar_arrive(&bar);
      fetch(t0 + 2 * TB, pf, pmu);
    }
    const int nt = min(TB, SL4 - t0);
    const double2* fb = fco[bsel] + k * FR + r;
#pragma unroll 2
    for (int tb = 0; tb < nt; ++tb) {
      const double2 k2 = rw[t0 + tb];
      const double2 F = fb[tb * 8];
#pragma unroll
      for (int g = 0; g < NB; ++g) {
        dmma884(acc[g][0][0], acc[g][0][1], cur[g], F.x);
        dmma884(acc[g][1][0], acc[g][1][1], cur[g], F.y);
        const double nx = fma(fma(k2.x, v[g], k2.y), cur[g], -prev[g]);
        prev[g] = cur[g];
        cur[g] = nx;
      }
    }
    if (more) {
      seg_bar_wait(&bar, parity);
      parity ^= 1;
    }
    bsel = bnext;
  }
  // lane (r, k) holds member 4h + k at beta index jw0 + 8g + r as (re, im)
  double2* spec = const_cast<double2*>(a.spec) + (long long)f * a.spec_fstride;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const Member M = mem[4 * h + k];
    if (!M.valid) continue;
#pragma unroll
    for (int g = 0; g < NB; ++g) {
      const int j = jw0 + 8 * g + r;
      spec[spec_index(a, M.row, M.reflect ? n - 1 - j : j)] = make_double2(acc[g][h][0], acc[g][h][1]);
    }
  }
}

}  // namespace so3

// DWT on the FP64 tensor path, barrier-free main loops (variant SO3_DWT_MMA2).
//
// Same mathematics and DMMA fragment layouts as dwt_mma.cuh (reference dwt.py:109-125,
// wigner.py:139-178).  ncu on the tile-synchronous kernels showed the FP64 pipe idle ~35%
// of the time in per-tile coefficient staging (+ CTA barrier) and, for the analysis, in
// the barrier-synchronised reduction over warps.  Here no warp ever waits at a CTA
// barrier inside the loop:
//
//  * Each iteration issues the DMMAs of the current degree block FIRST and the
//    recurrence for the NEXT block after them (double-buffered Wigner tile Dt, one
//    __syncwarp per iteration), so the scheduler can hide the recurrence's DFMA chain in
//    the issue gaps of the DMMA stream.  The padding member tile of 1/4-member clusters
//    is computed anyway (0.6% extra work) so the loop body is a single basic block.
//  * Synthesis: each lane loads its two B-fragment coefficients straight from global
//    memory two quads ahead (sign applied at use); no shared staging at all.
//  * Analysis: per-block partial sums go to a ring of R shared slots; the LAST warp to
//    arrive at a slot (shared atomic counter) reduces it, so nobody waits for stragglers.
//    Reduction order over warps is fixed, so results are bit-reproducible.
#pragma once
#include "common.cuh"
#include "dwt.cuh"

namespace so3 {

__device__ __forceinline__ double flip_if(double v, int odd) {
  return __longlong_as_double(__double_as_longlong(v) ^ ((long long)(odd & 1) << 63));
}

__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// (A, A*shift, C) for step index i0 + lane of a cluster, zero past the last step.
__device__ __forceinline__ double3 rc_load(const double* rct, int i0, int lane, int nsteps) {
  const int i = i0 + lane;
  if (i0 < 0 || i >= nsteps) return make_double3(0.0, 0.0, 0.0);
  return make_double3(__ldg(&rct[3 * i]), __ldg(&rct[3 * i + 1]), __ldg(&rct[3 * i + 2]));
}
__device__ __forceinline__ double3 rc_shfl(const double3& v, int src) {
  return make_double3(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                      __shfl_sync(0xffffffffu, v.z, src));
}

template <int JW>
struct Mma2 {
  static constexpr int S = JW + 4;   // Dt row stride (doubles): conflict-free STS and fragment LDS
  static constexpr int R = 4;        // analysis ring slots
  static constexpr size_t syn_warp_doubles = (size_t)8 * S;     // two 4-row halves
  static constexpr size_t ana_warp_doubles = (size_t)16 * S;    // two 8-row halves
};

// ------------------------------------------------------------------------------------------
// synthesis  g(j, r) = sum_l d^l(beta_j) F(l, r); 4 warps per CTA, CTAs of a cluster independent
// ------------------------------------------------------------------------------------------
template <int JW, int MINB>
__global__ void __launch_bounds__(128, MINB) dwt_synthesis_mma2_kernel(DwtArgs a, int split) {
  using K = Mma2<JW>;
  constexpr int JT = JW / 32, MT = JW / 8, S = K::S;
  extern __shared__ double dsm[];
  __shared__ Member mem[8];

  const int c = a.cluster0 + blockIdx.x / split;
  const int crank = blockIdx.x % split;
  const int f = blockIdx.y;
  const int2 base = __ldg(&a.bases[c]);
  const int m = base.x, mp = base.y;
  const int B = a.B, n = a.n;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = lane >> 2, tq = lane & 3;
  double2* spec = const_cast<double2*>(a.spec) + (long long)f * a.spec_fstride;
  const double* coefd = reinterpret_cast<const double*>(a.coef + (long long)f * a.coef_fstride);
  double* Dt = dsm + (size_t)warp * K::syn_warp_doubles;

  if (t < 8) mem[t] = member_of(a, m, mp, t);
  __syncthreads();
  const int nsteps = B - m;   // table entries (degrees)
  const int nq = (B - m + 3) >> 2;
  const double* rct = a.rc + 3 * __ldg(&a.rc_off[c]);

  // B-fragment coefficients of this lane: F(l, r) for r = g (member g>>1) and 8+g (4+(g>>1))
  const Member M0 = mem[g >> 1], M1 = mem[4 + (g >> 1)];
  const int comp = g & 1;
  // branch-free: out-of-range lanes load slot 0 and are zeroed
  auto fetch = [&](int Q, double& f0, double& f1) {
    const int l = m + 4 * Q + tq;
    const bool ok0 = l < B && M0.valid, ok1 = l < B && M1.valid;
    const int lc = ok0 || ok1 ? l : 0;
    const int s0 = ok0 ? coeff_slot32(lc, M0.pm, M0.pmp) : 0;
    const int s1 = ok1 ? coeff_slot32(lc, M1.pm, M1.pmp) : 0;
    const double v0 = __ldg(&coefd[2 * s0 + comp]);
    const double v1 = __ldg(&coefd[2 * s1 + comp]);
    const double mu = (l < B) ? __ldg(&rct[3 * (l - m) + 2]) : 0.0;
    f0 = ok0 ? v0 * mu : 0.0;
    f1 = ok1 ? v1 * mu : 0.0;
  };

  const int jw0 = (crank * 4 + warp) * JW;
  const double2 ln = __ldg(&a.lnorm[c]);
  double x[JT], cur[JT], prev[JT];
#pragma unroll
  for (int q = 0; q < JT; ++q) {
    const int j = jw0 + lane + 32 * q;
    const bool ok = j < n;
    x[q] = ok ? __ldg(&a.cosb[j]) : 0.0;
    cur[q] = ok ? seed_value(m, mp, ln, a.logcs[j]) : 0.0;
    prev[q] = 0.0;
  }
  double acc[MT][2][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) acc[i][nt][0] = acc[i][nt][1] = 0.0;

  // 4 degrees of the base column into Dt half (Q & 1); steps past the cluster's last degree
  // have zero coefficients, so those rows come out exactly zero.
  auto recur = [&](int Q, const double3& rcw) {
    double* D = Dt + (Q & 1) * 4 * S;
#pragma unroll
    for (int ll = 0; ll < 4; ++ll) {
      const double3 k3 = rc_shfl(rcw, (4 * Q + ll) & 31);
#pragma unroll
      for (int q = 0; q < JT; ++q) {
        D[ll * S + lane + 32 * q] = cur[q];
        const double tt = fma(k3.x, x[q], -k3.y);
        const double nx = fma(tt, cur[q], -prev[q]);
        prev[q] = cur[q];
        cur[q] = nx;
      }
    }
  };

  double3 rc_cur = rc_load(rct, 0, lane, nsteps);
  double3 rc_nxt = rc_load(rct, 32, lane, nsteps);
  double fa0, fa1, fb0, fb1;
  fetch(0, fa0, fa1);
  fetch(1, fb0, fb1);
  recur(0, rc_cur);
  __syncwarp();
  for (int Q = 0; Q < nq; ++Q) {
    // (1) DMMAs of quad Q (Dt half Q & 1)
    {
      const int l = m + 4 * Q + tq;
      const double b0 = flip_if(fa0, M0.sl * l + M0.par0);
      const double b1 = flip_if(fa1, M1.sl * l + M1.par0);
      const double* D = Dt + (Q & 1) * 4 * S;
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const double av = D[tq * S + 8 * i + g];
        dmma_884(acc[i][0][0], acc[i][0][1], av, b0);
        dmma_884(acc[i][1][0], acc[i][1][1], av, b1);
      }
    }
    // (2) prefetch quad Q+2's coefficients, recurrence for quad Q+1 (other Dt half)
    fa0 = fb0;
    fa1 = fb1;
    fetch(Q + 2, fb0, fb1);
    if (((Q + 1) & 7) == 0) {   // the next quad starts a new 32-step window
      rc_cur = rc_nxt;
      rc_nxt = rc_load(rct, 4 * (Q + 1) + 32, lane, nsteps);
    }
    recur(Q + 1, rc_cur);
    __syncwarp();
  }
  // lane (g, tq) holds g(j = jw0 + 8 i + g, member 4 nt + tq) as (re, im)
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int j = jw0 + 8 * i + g;
    if (j >= n) continue;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const Member M = mem[4 * nt + tq];
      if (M.valid) spec[spec_index(a, M.row, M.reflect ? n - 1 - j : j)] = make_double2(acc[i][nt][0], acc[i][nt][1]);
    }
  }
}

// ------------------------------------------------------------------------------------------
// analysis  out(r, l) = sum_j x'_r(j) d^l(beta_j); one CTA (W warps) per cluster
// ------------------------------------------------------------------------------------------
template <int JW>
__global__ void __launch_bounds__(256, 1) dwt_analysis_mma2_kernel(DwtArgs a) {
  using K = Mma2<JW>;
  constexpr int JT = JW / 32, KS = JW / 4, S = K::S, R = K::R;
  extern __shared__ double dsm[];
  __shared__ Member mem[8];
  __shared__ int arrive[R];
  __shared__ volatile int slot_free[R];   // first block index allowed to use the slot

  const int c = a.cluster0 + blockIdx.x;
  const int f = blockIdx.y;
  const int2 base = __ldg(&a.bases[c]);
  const int m = base.x, mp = base.y;
  const int B = a.B, n = a.n;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, W = blockDim.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const double2* spec = a.spec + (long long)f * a.spec_fstride;
  double2* coef = a.coef + (long long)f * a.coef_fstride;
  double* Dt = dsm + (size_t)warp * K::ana_warp_doubles;   // [2][8][S]
  double* ring = dsm + (size_t)W * K::ana_warp_doubles;    // [R][W][128]

  if (t < 8) mem[t] = member_of(a, m, mp, t);
  if (t < R) { arrive[t] = 0; slot_free[t] = t; }
  __syncthreads();
  const int nsteps = B - m;   // table entries (degrees)
  const int nb = (B - m + 7) >> 3;   // blocks of 8 degrees
  const double* rct = a.rc + 3 * __ldg(&a.rc_off[c]);

  const int jw0 = warp * JW;
  double afr[KS][2];
#pragma unroll
  for (int s = 0; s < KS; ++s) {
    const int j = jw0 + 4 * s + tq;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r = 8 * mt + g;
      const Member M = mem[r >> 1];
      double v = 0.0;
      if (j < n && M.valid) {
        const double* e = reinterpret_cast<const double*>(&spec[spec_index(a, M.row, M.reflect ? n - 1 - j : j)]);
        v = e[r & 1];
      }
      afr[s][mt] = v;
    }
  }
  const double2 ln = __ldg(&a.lnorm[c]);
  double x[JT], cur[JT], prev[JT];
#pragma unroll
  for (int q = 0; q < JT; ++q) {
    const int j = jw0 + lane + 32 * q;
    const bool ok = j < n;
    x[q] = ok ? __ldg(&a.cosb[j]) : 0.0;
    cur[q] = ok ? seed_value(m, mp, ln, a.logcs[j]) : 0.0;
    prev[q] = 0.0;
  }
  auto recur = [&](int b, const double3& rcw) {
    double* D = Dt + (b & 1) * 8 * S;
#pragma unroll
    for (int ll = 0; ll < 8; ++ll) {
      const double3 k3 = rc_shfl(rcw, (8 * b + ll) & 31);
#pragma unroll
      for (int q = 0; q < JT; ++q) {
        D[ll * S + lane + 32 * q] = cur[q];
        const double tt = fma(k3.x, x[q], -k3.y);
        const double nx = fma(tt, cur[q], -prev[q]);
        prev[q] = cur[q];
        cur[q] = nx;
      }
    }
  };

  const double vscale = 8.0 * 3.141592653589793 * (double)B;
  double3 rc_cur = rc_load(rct, 0, lane, nsteps);
  double3 rc_nxt = rc_load(rct, 32, lane, nsteps);
  recur(0, rc_cur);
  __syncwarp();
  for (int b = 0; b < nb; ++b) {
    // (1) DMMAs of block b
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    {
      const double* D = Dt + (b & 1) * 8 * S;
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const double bv = D[g * S + 4 * s + tq];
        dmma_884(acc[0][0], acc[0][1], afr[s][0], bv);
        dmma_884(acc[1][0], acc[1][1], afr[s][1], bv);
      }
    }
    // (2) recurrence for block b+1 into the other Dt half
    if (((b + 1) & 3) == 0) {
      rc_cur = rc_nxt;
      rc_nxt = rc_load(rct, 8 * (b + 1) + 32, lane, nsteps);
    }
    recur(b + 1, rc_cur);
    // (3) publish partials C[r = 8 mt + g][l = 8 b + 2 tq + e]; the last warp to arrive reduces
    const int slot = b % R;
    if (lane == 0) { while (slot_free[slot] < b) { } }
    __syncwarp();
    double* pw = ring + ((size_t)slot * W + warp) * 128;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
      *reinterpret_cast<double2*>(pw + (mt * 32 + lane) * 2) = make_double2(acc[mt][0], acc[mt][1]);
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      __threadfence_block();
      last = (atomicAdd(&arrive[slot], 1) == W - 1);
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence_block();
      const double* ps = ring + (size_t)slot * W * 128;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int idx = lane + 32 * i;            // (degree ll, member k)
        const int ll = idx >> 3, k = idx & 7;
        const int l = m + 8 * b + ll;
        const Member M = mem[k];
        if (l < B && M.valid) {
          const int mt = k >> 2, g_re = (2 * k) & 7, tsrc = ll >> 1, e = ll & 1;
          const int o_re = (mt * 32 + g_re * 4 + tsrc) * 2 + e;
          const int o_im = o_re + 8;                // g_im = g_re + 1 -> lane + 4
          double re = 0.0, im = 0.0;
          for (int w = 0; w < W; ++w) {
            re += ps[w * 128 + o_re];
            im += ps[w * 128 + o_im];
          }
          double sc = (2.0 * l + 1.0) / vscale * __ldg(&rct[3 * (l - m) + 2]);   // v_l * mu_l
          if ((M.sl * l + M.par0) & 1) sc = -sc;
          coef[coeff_slot32(l, M.pm, M.pmp)] = make_double2(re * sc, im * sc);
        }
      }
      __syncwarp();
      if (lane == 0) {
        arrive[slot] = 0;
        __threadfence_block();
        slot_free[slot] = b + R;
      }
    }
    __syncwarp();
  }
}

}  // namespace so3

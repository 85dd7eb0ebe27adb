// DWT on the FP64 tensor path, software-pipelined and barrier-free in the main loop.
//
// Same mathematics and fragment layouts as dwt_mma.cuh (reference dwt.py:109-125,
// wigner.py:139-178).  What changes is the schedule, after ncu showed the FP64 pipe idle
// ~45% of the time in the tile-synchronous kernels (profiles/): every warp ran its
// latency-bound recurrence at the same moment after each CTA barrier.
//
//  * Each warp overlaps the recurrence for the NEXT block of degrees (writing one half of
//    a double-buffered Wigner tile Dt) with the DMMAs of the CURRENT block (reading the
//    other half), so its own DFMA chain fills the issue gaps of its DMMA stream.
//  * Synthesis: warps are independent.  Each warp stages its own copy of the signed
//    coefficient tiles with cp.async (double buffered, no CTA barrier); recurrence
//    coefficients come from the plan table, one tile per lane, broadcast by shuffles.
//  * Analysis: the per-block partial sums (16 member rows x 8 degrees per warp) go into a
//    ring of R shared slots guarded by mbarriers; block b is reduced by warp b % W while
//    the other warps run ahead (at most R blocks), so no warp ever waits at a CTA barrier.
//    The reduction order over warps is fixed, so results are bit-reproducible.
#pragma once
#include "common.cuh"
#include "dwt.cuh"

namespace so3 {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool full) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(full ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

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
  static constexpr int S = JW + 4;      // Dt row stride (doubles): conflict-free STS and fragment LDS
  static constexpr int CF = 10;         // coefficient-tile row stride (complex): conflict-free LDS
  static constexpr int LT = 32;         // degrees per coefficient / recurrence-coefficient tile
  // synthesis, per warp: Dt 8 rows + two coefficient tiles
  static constexpr size_t syn_warp_doubles = (size_t)8 * S + 2 * LT * CF * 2;
  // analysis, per warp: Dt 16 rows; ring: R slots x W warps x 128 doubles
  static constexpr int R = 4;
  static constexpr size_t ana_dt_doubles = (size_t)16 * S;
};

// ------------------------------------------------------------------------------------------
// synthesis  g(j, r) = sum_l d^l(beta_j) F(l, r)
// ------------------------------------------------------------------------------------------
template <int JW>
__global__ void __launch_bounds__(128, 2) dwt_synthesis_mma2_kernel(DwtArgs a, int split) {
  using K = Mma2<JW>;
  constexpr int JT = JW / 32, MT = JW / 8, S = K::S, CF = K::CF, LT = K::LT;
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
  const double2* coef = a.coef + (long long)f * a.coef_fstride;
  double* Dt = dsm + (size_t)warp * K::syn_warp_doubles;          // [2][4][S]
  double2* cf = reinterpret_cast<double2*>(Dt + 8 * S);           // [2][LT][CF]

  if (t < 8) mem[t] = make_member(m, mp, t, n);
  __syncthreads();
  const bool two_tiles = mem[4].valid;
  const int nsteps = B - 1 - m;       // recurrence steps l -> l+1 of this cluster
  const int nq = (B - m + 3) >> 2;    // quads of degrees
  const double* rct = a.rc + 3 * __ldg(&a.rc_off[c]);

  // coefficient tile T (degrees m + 32T ..) -> cf[T & 1] via cp.async (zero-filled past B)
  auto stage = [&](int T) {
    double2* dst = cf + (T & 1) * LT * CF;
#pragma unroll
    for (int i = 0; i < LT * 8 / 32; ++i) {
      const int idx = lane + 32 * i, ll = idx >> 3, k = idx & 7;
      const int l = m + LT * T + ll;
      const Member& M = mem[k];
      const bool ok = l < B && M.valid;
      cp_async16(&dst[ll * CF + k], ok ? &coef[coeff_slot(l, M.pm, M.pmp)] : coef, ok);
    }
    cp_async_commit();
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

  // the member / component this lane feeds into the B fragments (F(l, r) for r = g, 8 + g)
  const Member M0 = mem[g >> 1], M1 = mem[4 + (g >> 1)];
  const int comp = g & 1;

  // recurrence for quad Q into Dt half (Q & 1); rcw holds steps 32*(Q/8) .. of this lane's tile
  auto recur = [&](int Q, const double3& rcw) {
    double* D = Dt + (Q & 1) * 4 * S;
#pragma unroll
    for (int ll = 0; ll < 4; ++ll) {
      const int s = 4 * Q + ll;                       // step index l - m
      const double3 k3 = rc_shfl(rcw, s & (LT - 1));
      const bool live = s < B - m;
#pragma unroll
      for (int q = 0; q < JT; ++q) {
        D[ll * S + lane + 32 * q] = live ? cur[q] : 0.0;
        const double tt = fma(k3.x, x[q], -k3.y);
        const double nx = fma(tt, cur[q], -k3.z * prev[q]);
        prev[q] = cur[q];
        cur[q] = nx;
      }
    }
  };

  stage(0);
  if (nq > 8) stage(1); else cp_async_commit();
  double3 rc_cur = rc_load(rct, 0, lane, nsteps);
  double3 rc_nxt = rc_load(rct, LT, lane, nsteps);
  recur(0, rc_cur);
  cp_async_wait<1>();
  __syncwarp();
  for (int Q = 0; Q < nq; ++Q) {
    const int T = Q >> 3, qi = Q & 7;
    // (A) next quad's Wigner rows (other Dt half), overlapped with (B)
    if (Q + 1 < nq) recur(Q + 1, qi == 7 ? rc_nxt : rc_cur);
    // (B) this quad's DMMAs
    {
      const double* D = Dt + (Q & 1) * 4 * S;
      const double2* F = cf + (T & 1) * LT * CF + (4 * qi + tq) * CF;
      const int l = m + 4 * Q + tq;
      const double2 f0 = F[g >> 1], f1 = F[4 + (g >> 1)];
      const double b0 = flip_if(comp ? f0.y : f0.x, M0.sl * l + M0.par0);
      const double b1 = flip_if(comp ? f1.y : f1.x, M1.sl * l + M1.par0);
      if (two_tiles) {
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const double av = D[tq * S + 8 * i + g];
          dmma_884(acc[i][0][0], acc[i][0][1], av, b0);
          dmma_884(acc[i][1][0], acc[i][1][1], av, b1);
        }
      } else {
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const double av = D[tq * S + 8 * i + g];
          dmma_884(acc[i][0][0], acc[i][0][1], av, b0);
        }
      }
    }
    if (qi == 7) {   // tile T done: its coefficient buffer is free for tile T + 2
      rc_cur = rc_nxt;
      rc_nxt = rc_load(rct, LT * (T + 2), lane, nsteps);
      __syncwarp();
      if (8 * (T + 2) < nq) stage(T + 2); else cp_async_commit();
      cp_async_wait<1>();   // tile T + 1 has landed
    }
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
      if (M.valid) spec[M.row * n + (M.reflect ? n - 1 - j : j)] = make_double2(acc[i][nt][0], acc[i][nt][1]);
    }
  }
}

// ------------------------------------------------------------------------------------------
// analysis  out(r, l) = sum_j x'_r(j) d^l(beta_j)
// ------------------------------------------------------------------------------------------
template <int JW>
__global__ void __launch_bounds__(256, 1) dwt_analysis_mma2_kernel(DwtArgs a) {
  using K = Mma2<JW>;
  constexpr int JT = JW / 32, KS = JW / 4, S = K::S, LT = K::LT, R = K::R;
  extern __shared__ double dsm[];
  __shared__ Member mem[8];
  __shared__ unsigned long long full_bar[R], empty_bar[R];

  const int c = a.cluster0 + blockIdx.x;
  const int f = blockIdx.y;
  const int2 base = __ldg(&a.bases[c]);
  const int m = base.x, mp = base.y;
  const int B = a.B, n = a.n;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, W = blockDim.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const double2* spec = a.spec + (long long)f * a.spec_fstride;
  double2* coef = a.coef + (long long)f * a.coef_fstride;
  double* Dt = dsm + (size_t)warp * K::ana_dt_doubles;         // [2][8][S]
  double* ring = dsm + (size_t)W * K::ana_dt_doubles;          // [R][W][128]

  if (t < 8) mem[t] = make_member(m, mp, t, n);
  if (t < R) { mbar_init(&full_bar[t], W); mbar_init(&empty_bar[t], 1); }
  __syncthreads();
  const bool two_tiles = mem[4].valid;
  const int nsteps = B - 1 - m;
  const int nb = (B - m + 7) >> 3;    // blocks of 8 degrees
  const double* rct = a.rc + 3 * __ldg(&a.rc_off[c]);

  // A fragments: x'_r(j), r = 8 mt + g, j = jw0 + 4 s + tq (loaded once)
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
        const double* e = reinterpret_cast<const double*>(&spec[M.row * n + (M.reflect ? n - 1 - j : j)]);
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
      const int s = 8 * b + ll;
      const double3 k3 = rc_shfl(rcw, s & (LT - 1));
      const bool live = s < B - m;
#pragma unroll
      for (int q = 0; q < JT; ++q) {
        D[ll * S + lane + 32 * q] = live ? cur[q] : 0.0;
        const double tt = fma(k3.x, x[q], -k3.y);
        const double nx = fma(tt, cur[q], -k3.z * prev[q]);
        prev[q] = cur[q];
        cur[q] = nx;
      }
    }
  };

  const double vscale = 8.0 * 3.141592653589793 * (double)B;
  double3 rc_cur = rc_load(rct, 0, lane, nsteps);
  double3 rc_nxt = rc_load(rct, LT, lane, nsteps);
  recur(0, rc_cur);
  __syncwarp();
  for (int b = 0; b < nb; ++b) {
    const int T = b >> 2, bi = b & 3;
    if (b + 1 < nb) recur(b + 1, bi == 3 ? rc_nxt : rc_cur);
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    {
      const double* D = Dt + (b & 1) * 8 * S;
      if (two_tiles) {
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const double bv = D[g * S + 4 * s + tq];
          dmma_884(acc[0][0], acc[0][1], afr[s][0], bv);
          dmma_884(acc[1][0], acc[1][1], afr[s][1], bv);
        }
      } else {
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const double bv = D[g * S + 4 * s + tq];
          dmma_884(acc[0][0], acc[0][1], afr[s][0], bv);
        }
      }
    }
    if (bi == 3) {
      rc_cur = rc_nxt;
      rc_nxt = rc_load(rct, LT * (T + 2), lane, nsteps);
    }
    __syncwarp();   // Dt half (b & 1) is free for block b + 2
    // publish this warp's partials C[r = 8 mt + g][l = 8 b + 2 tq + e]
    const int slot = b % R;
    if (b >= R) mbar_wait(&empty_bar[slot], ((b / R) - 1) & 1);
    double* pw = ring + ((size_t)slot * W + warp) * 128;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
      *reinterpret_cast<double2*>(pw + (mt * 32 + lane) * 2) = make_double2(acc[mt][0], acc[mt][1]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&full_bar[slot]);
    // rotating reducer: warp b % W finishes block b
    if (b % W == warp) {
      mbar_wait(&full_bar[slot], (b / R) & 1);
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
          double sc = (2.0 * l + 1.0) / vscale;
          if ((M.sl * l + M.par0) & 1) sc = -sc;
          coef[coeff_slot(l, M.pm, M.pmp)] = make_double2(re * sc, im * sc);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[slot]);
    }
  }
}

}  // namespace so3

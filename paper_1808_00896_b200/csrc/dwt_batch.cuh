// Batched DWT for small bandwidths (BASELINE configs[1]: B = 32, 64 functions; reference
// dwt.py:109-125 applied per function, soft.py:134-167).
//
// With many functions sharing one plan, the DWT of a symmetry cluster is a dense contraction
// over the SAME Wigner matrix D[l][j] (l = m..B-1, j < 2B):
//
//   analysis   C[l][(f, member, re/im)] = sum_j  D[l][j] * S_f(member, j or mirror)
//   synthesis  G[j][(f, member, re/im)] = sum_l  D[l][j] * sign * mu_l * F_f(l, member)
//
// One CTA takes one cluster and FC functions (one warp per function).  Per tile of 32 degrees
// the threads run the rescaled recurrence once (one beta index per thread) into a shared
// Wigner tile; every warp then contracts it with its function on the FP64 tensor path
// (DMMA m8n8k4), so the seeds, the recurrence and the member table are paid once per FC
// functions and no cross-warp reduction is needed (each warp owns the full j range).  The
// analysis loads each warp's spectrum operand straight into registers (FC = 4, four CTAs per
// SM); the synthesis stages each warp's signed coefficients in shared memory (FC = 8).
// Shared rows are padded to a stride = 4 (mod 16) doubles so the fragment reads are
// bank-conflict free.  (Measured alternatives: a staged analysis 16 % slower, a
// register-operand synthesis 10 % slower.)
//
// Same arithmetic as dwt_mma.cuh: the synthesis sums degree quads from l = m upward exactly
// like the single-function kernel (results are bit-identical to it); the analysis sums j in
// one pass per warp (the single-function kernel splits j over warps), so it agrees to rounding.
#pragma once
#include "common.cuh"
#include "dwt.cuh"
#include "dwt_mma.cuh"

namespace so3 {

__host__ __device__ inline int batch_np(int n) { return (n + 7) & ~7; }
__host__ __device__ inline int batch_sd(int n) {   // >= np, = 4 (mod 16) when np = 0 (mod 16)
  const int np = batch_np(n);
  return np + ((4 - np) & 15);
}

// Wigner tile rows l0 .. l0+31 of the cluster for this thread's j (rows past B-1 are zero);
// recurrence table entries come through L1 (every thread of the CTA reads the same ones).
__device__ __forceinline__ void batch_wigner_tile_ldg(double* D, int sd, int t, int nl, const double* rct, int l0m,
                                                      double x, bool up, double& cur, double& prev) {
#pragma unroll 4
  for (int ll = 0; ll < 32; ++ll) {
    if (ll < nl) {
      D[ll * sd + t] = cur;
      const double tt = rec_t(__ldg(&rct[3 * (l0m + ll)]), __ldg(&rct[3 * (l0m + ll) + 1]), x, up);
      const double nx = fma(tt, cur, -prev);
      prev = cur;
      cur = nx;
    } else {
      D[ll * sd + t] = 0.0;
    }
  }
}

__host__ __device__ inline size_t batch_analysis_smem(int n) { return (size_t)32 * batch_sd(n) * sizeof(double); }
template <int FC>
__host__ __device__ inline size_t batch_synthesis_smem(int n) {
  return ((size_t)32 * batch_sd(n) + (size_t)32 * (FC * 16 + 4)) * sizeof(double);
}

// ---------------------------------------------------------------------------------- analysis
// Register-operand analysis (2B <= 64): each warp's B operand -- its function's 16 spectrum
// columns over all beta, 2B/4 k-steps x 2 member tiles -- is loaded straight into registers
// (lane (g, tq) reads member (g/2)'s re or im part at beta 4s + tq, mirrored for reflecting
// members: every fetched sector is used).  No staging buffer, so the CTA holds only the
// shared Wigner tile and FC = 4 functions give 4 independent CTAs per SM.
// Seeds d^m_{m,m'}(beta_j) of every (cluster, beta index), once per plan: every CTA of a cluster (one per
// function group) otherwise repeats the double-double log-space evaluation and its exp() in its
// prologue (same function and inputs: the table holds the identical bits).
__global__ void __launch_bounds__(64) dwt_seed_table_kernel(DwtArgs a, double* seeds) {
  const int c = blockIdx.x, j = threadIdx.x + 64 * blockIdx.y;
  if (j >= a.n) return;
  const int2 base = __ldg(&a.bases[c]);
  seeds[(long long)c * a.n + j] = seed_value(base.x, base.y, __ldg(&a.lnorm[c]), a.logcs[j]);
}

template <int FC, int KSM>
__global__ void __launch_bounds__(FC * 32, 4) dwt_analysis_batch_reg_kernel(DwtArgs a, int batch, const double* seeds) {
  extern __shared__ double dsm[];
  __shared__ Member mem[8];
  const int c = a.cluster0 + blockIdx.x;
  const int f0 = blockIdx.y * FC;
  const int2 base = __ldg(&a.bases[c]);
  const int m = base.x, mp = base.y;
  const int B = a.B, n = a.n, np = batch_np(n), sd = batch_sd(n);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int fl = warp;
  const bool fvalid = f0 + fl < batch;
  const long long rco = __ldg(&a.rc_off[c]);
  double* D = dsm;                                   // [32][sd]
  if (t < 8) mem[t] = member_of(a, m, mp, t);
  __syncthreads();

  // B fragments: b[nt][s] = S'(j = 4s + tq, column 8 nt + g)
  double bf[2][KSM];
  const double2* spec = a.spec + (long long)(f0 + fl) * a.spec_fstride;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const Member M = mem[4 * nt + (g >> 1)];
    const bool ok = fvalid && M.valid;
    const double* p = reinterpret_cast<const double*>(spec + (long long)M.row * n) + (g & 1);
#pragma unroll
    for (int s = 0; s < KSM; ++s) {
      const int j = 4 * s + tq;
      bf[nt][s] = (ok && j < n) ? p[2 * (M.reflect ? n - 1 - j : j)] : 0.0;
    }
  }

  const double* rct = a.rc + 3 * rco;
  double x = 0.0, cur = 0.0, prev = 0.0;
  if (t < n) {
    x = __ldg(&a.xv[t]);
    cur = __ldg(&seeds[(long long)c * n + t]);
  }
  const bool two_tiles = mem[4].valid;
  const double vscale = 8.0 * 3.141592653589793 * (double)B;
  const double rvscale = 1.0 / vscale;   // one division per thread: a DDIV per output kept the FP64 pipe busy in the reductions
  double2* coef = a.coef + (long long)(f0 + fl) * a.coef_fstride;

  for (int l0 = m; l0 < B; l0 += 32) {
    const int nl = min(32, B - l0);
    if (l0 > m) __syncthreads();   // every warp is done reading the previous tile
    if (t < np) batch_wigner_tile_ldg(D, sd, t, nl, rct, l0 - m, x, 2 * t >= n, cur, prev);
    __syncthreads();
    if (!fvalid) continue;
    const int mtn = (nl + 7) >> 3;
    double acc[4][2][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    const double* Dg = D + g * sd + tq;
#pragma unroll
    for (int s = 0; s < KSM; ++s) {
      if (4 * s >= np) break;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
        if (mt < mtn) {
          const double av = Dg[8 * mt * sd + 4 * s];
          dmma884(acc[mt][0][0], acc[mt][0][1], av, bf[0][s]);
          if (two_tiles) dmma884(acc[mt][1][0], acc[mt][1][1], av, bf[1][s]);
        }
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int l = l0 + 8 * mt + g;
      if (mt >= mtn || l >= B) continue;
      const double vmu = (2.0 * l + 1.0) * rvscale * __ldg(&rct[3 * (l - m) + 2]);   // v_l * mu_l
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const Member M = mem[4 * nt + tq];
        if (!M.valid) continue;
        const double sc = ((M.sl * l + M.par0) & 1) ? -vmu : vmu;
        coef[coeff_slot32(l, M.pm, M.pmp)] = make_double2(acc[mt][nt][0] * sc, acc[mt][nt][1] * sc);
      }
    }
  }
}

// --------------------------------------------------------------------------------- synthesis
// Warp w stages the signed coefficients of function f0 + w (8 per lane per 32-degree tile,
// fetched one tile ahead) and owns its output; only the Wigner tile is shared.
template <int FC, int MTMAX>
__global__ void __launch_bounds__(FC * 32, 2) dwt_synthesis_batch_kernel(DwtArgs a, int batch, const double* seeds) {
  constexpr int SF = FC * 16 + 4;
  extern __shared__ double dsm[];
  __shared__ Member mem[8];
  const int c = a.cluster0 + blockIdx.x;
  const int f0 = blockIdx.y * FC;
  const int2 base = __ldg(&a.bases[c]);
  const int m = base.x, mp = base.y;
  const int B = a.B, n = a.n, np = batch_np(n), sd = batch_sd(n);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int fl = warp;
  const bool fvalid = f0 + fl < batch;
  double* D = dsm;                         // [32][sd]
  double* Ff = dsm + 32 * sd + fl * 16;    // [32][SF] rows, this warp's 16 columns
  if (t < 8) mem[t] = member_of(a, m, mp, t);
  __syncthreads();

  const double* rct = a.rc + 3 * __ldg(&a.rc_off[c]);
  const double2* coef = a.coef + (long long)(f0 + fl) * a.coef_fstride;
  const int k = lane & 7;                  // this lane's member; degrees ll = (lane >> 3) + 4 i
  const Member Mk = mem[k];
  double2 z[8];
  auto fetch = [&](int l0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int l = l0 + (lane >> 3) + 4 * i;
      z[i] = (fvalid && Mk.valid && l < B) ? coef[coeff_slot32(l, Mk.pm, Mk.pmp)] : make_double2(0.0, 0.0);
    }
  };
  fetch(m);

  double x = 0.0, cur = 0.0, prev = 0.0;
  if (t < n) {
    x = __ldg(&a.xv[t]);
    cur = __ldg(&seeds[(long long)c * n + t]);
  }
  const bool two_tiles = mem[4].valid;
  const int mtn = np >> 3;
  double acc[MTMAX][2][2];
#pragma unroll
  for (int mt = 0; mt < MTMAX; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

  for (int l0 = m; l0 < B; l0 += 32) {
    const int nl = min(32, B - l0);
    if (l0 > m) __syncthreads();   // every warp is done reading the previous Wigner tile
    if (t < np) batch_wigner_tile_ldg(D, sd, t, nl, rct, l0 - m, x, 2 * t >= n, cur, prev);
    // this warp's signed, mu-scaled coefficients of the tile (its own previous reads are
    // complete: same warp, program order)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int ll = (lane >> 3) + 4 * i, l = l0 + ll;
      double sg = 0.0;
      if (l < B) {
        const double mu = __ldg(&rct[3 * (l - m) + 2]);
        sg = ((Mk.sl * l + Mk.par0) & 1) ? -mu : mu;
      }
      Ff[ll * SF + 2 * k] = z[i].x * sg;
      Ff[ll * SF + 2 * k + 1] = z[i].y * sg;
    }
    if (l0 + 32 < B) fetch(l0 + 32);
    __syncthreads();
    if (!fvalid) continue;
    const double* Fb = Ff + tq * SF + g;
    const double* Da = D + tq * sd + g;
    for (int s = 0; s < ((nl + 3) >> 2); ++s) {
      const double b0 = Fb[4 * s * SF];
      const double b1 = two_tiles ? Fb[4 * s * SF + 8] : 0.0;
#pragma unroll
      for (int mt = 0; mt < MTMAX; ++mt) {
        if (mt < mtn) {
          const double av = Da[4 * s * sd + 8 * mt];
          dmma884(acc[mt][0][0], acc[mt][0][1], av, b0);
          if (two_tiles) dmma884(acc[mt][1][0], acc[mt][1][1], av, b1);
        }
      }
    }
  }
  if (!fvalid) return;
  // G[j = 8 mt + g][col = 8 nt + 2 tq + e]: member 4 nt + tq at j (or its mirror)
  double2* spec = const_cast<double2*>(a.spec) + (long long)(f0 + fl) * a.spec_fstride;
#pragma unroll
  for (int mt = 0; mt < MTMAX; ++mt) {
    const int j = 8 * mt + g;
    if (mt >= mtn || j >= n) continue;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const Member M = mem[4 * nt + tq];
      if (M.valid) spec[spec_index(a, M.row, M.reflect ? n - 1 - j : j)] = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
    }
  }
}

}  // namespace so3

// Torus DFT stage of FSOFT / iFSOFT (reference fft.py:35-76, soft.py:127-132, 164-172).
//
// The 2-D unnormalised DFT over (alpha, gamma) of every beta slice is done in
// two passes over HBM, each a batch of 1-D FFTs of length N = 2B whose rows are
// JB consecutive beta indices j:
//
//   ROW_FWD (K1a): grid[f][i][j][k]  --FFT_k(+1)-->  S[f][i][m'][j]     (transposing write)
//   COL     (K1b): S[f][i][m'][j]    --FFT_i(+1)-->  S[f][m][m'][j] * w_j  (in place)
//   COL     (K4a): S[f][m][m'][j]    --FFT_m(-1)-->  S[f][i][m'][j]        (in place)
//   ROW_INV (K4b): S[f][i][m'][j]    --FFT_m'(-1)--> grid[f][i][j][k]   (transposing read)
//
// so the DWT sees each order pair (m, m') as one contiguous vector over j.
// Reads and writes are JB*16 bytes contiguous (or whole rows).  Each thread keeps
// 16 points in registers and runs a radix-16 Stockham FFT whose stages exchange
// through shared memory.  Twiddles come from a per-plan table tw[k] = exp(+2 pi i k / N).
// Non power-of-two or tiny N use a direct O(N^2) DFT kernel (the reference also
// falls back to a kernel-matrix product for those lengths, fft.py:51-54).
#pragma once
#include "common.cuh"

namespace so3 {

enum FftMode { ROW_FWD = 0, COL = 1, ROW_INV = 2 };

struct FftArgs {
  int n;            // transform length N = 2B
  int nyq;          // Nyquist bin B (treated as zero where the inverse reads it)
  int J;            // beta slices held in this array (n on one GPU, the slab width when sharded)
  int jbase;        // global index of local slice 0 (for the quadrature weights)
  const double2* src;
  double2* dst;
  const double2* tw;     // N entries, exp(+2 pi i k / N)
  const double* w;       // quadrature weights (forward COL only), global j
  long long fstride_src; // per-function element strides (batch)
  long long fstride_dst;
};

// exp(SIGN * 2 pi i * Q / 16) * a, Q compile-time
template <int Q, int SIGN>
__device__ __forceinline__ double2 wmul16(double2 a) {
  constexpr int q = Q & 15;
  if constexpr (q == 0) return a;
  else if constexpr (q == 4) return SIGN > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
  else if constexpr (q == 8) return make_double2(-a.x, -a.y);
  else if constexpr (q == 12) return SIGN > 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
  else {
    constexpr double C[16] = {1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173,
                              0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128675613,
                              -1.0, -0.92387953251128675613, -0.70710678118654752440, -0.38268343236508977173,
                              0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128675613};
    constexpr double S[16] = {0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128675613,
                              1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173,
                              0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128675613,
                              -1.0, -0.92387953251128675613, -0.70710678118654752440, -0.38268343236508977173};
    constexpr double c = C[q];
    constexpr double s = SIGN > 0 ? S[q] : -S[q];
    return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
  }
}

template <int LOG>
__host__ __device__ constexpr int bitrev(int r) {
  int rev = 0;
  for (int b = 0; b < LOG; ++b) rev |= ((r >> b) & 1) << (LOG - 1 - b);
  return rev;
}

// In-register DFT of R points (R | 16, power of two): out[k] = sum_r in[r] exp(SIGN 2 pi i r k / R).
// Radix-2 decimation in time on a bit-reversed copy, expanded by template recursion so
// every register index and twiddle is a compile-time constant.
template <int R, int LOG, int I>
__device__ __forceinline__ void bitrev_copy(double2 (&u)[R], const double2 (&v)[R]) {
  u[bitrev<LOG>(I)] = v[I];
  if constexpr (I + 1 < R) bitrev_copy<R, LOG, I + 1>(u, v);
}

template <int R, int S, int B0, int K, int SIGN>
__device__ __forceinline__ void dit_butterflies(double2 (&u)[R]) {
  constexpr int H = S / 2;
  const double2 t = wmul16<(K * 16 / S), SIGN>(u[B0 + K + H]);
  u[B0 + K + H] = csub(u[B0 + K], t);
  u[B0 + K] = cadd(u[B0 + K], t);
  if constexpr (K + 1 < H) dit_butterflies<R, S, B0, K + 1, SIGN>(u);
  else if constexpr (B0 + S < R) dit_butterflies<R, S, B0 + S, 0, SIGN>(u);
}

template <int R, int S, int SIGN>
__device__ __forceinline__ void dit_stages(double2 (&u)[R]) {
  if constexpr (S <= R) {
    dit_butterflies<R, S, 0, 0, SIGN>(u);
    dit_stages<R, S * 2, SIGN>(u);
  }
}

template <int R, int SIGN>
__device__ __forceinline__ void dft_reg(double2 (&v)[R]) {
  if constexpr (R > 1) {
    constexpr int LOG = (R == 2) ? 1 : (R == 4) ? 2 : (R == 8) ? 3 : 4;
    double2 u[R];
    bitrev_copy<R, LOG, 0>(u, v);
    dit_stages<R, 2, SIGN>(u);
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = u[r];
  }
}

// One radix-R Stockham stage with span NS (product of the radices before it).
// Thread t owns butterflies b = t + q*N/16 (q < 16/R); butterfly b reads points
// b + r*N/R (register slot q + r*16/R) and writes b/NS*NS*R + b%NS + r*NS.
template <int N, int R, int NS, int SIGN, bool LAST>
__device__ __forceinline__ void stockham_stage(double2 (&v)[16], int t, const double2* __restrict__ tw,
                                               double2* __restrict__ row) {
  constexpr int Q = 16 / R;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int b = t + q * (N / 16);
    double2 u[R];
#pragma unroll
    for (int r = 0; r < R; ++r) u[r] = v[q + r * Q];
    if constexpr (NS > 1) {
      const int bm = b & (NS - 1);
#pragma unroll
      for (int r = 1; r < R; ++r) {
        double2 w = __ldg(&tw[r * bm * (N / (NS * R))]);
        if constexpr (SIGN < 0) w.y = -w.y;
        u[r] = cmul(u[r], w);
      }
    }
    dft_reg<R, SIGN>(u);
    if constexpr (LAST) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[q + r * Q] = u[r];
    } else {
      const int base = (b / NS) * NS * R + (b & (NS - 1));
#pragma unroll
      for (int r = 0; r < R; ++r) row[base + r * NS] = u[r];
    }
  }
}

template <int N>
struct Radix {
  // N = 16^a * rem; stages: a radix-16 stages then one radix-rem stage (rem in {2,4,8}) if rem > 1.
  static constexpr int LOG = (N == 16) ? 4 : (N == 32) ? 5 : (N == 64) ? 6 : (N == 128) ? 7 : (N == 256) ? 8
                           : (N == 512) ? 9 : (N == 1024) ? 10 : (N == 2048) ? 11 : 12;
  static constexpr int N16 = LOG / 4;
  static constexpr int REM = 1 << (LOG % 4);
};

template <int N, int SIGN>
__device__ __forceinline__ void fft_rows(double2 (&v)[16], int t, const double2* __restrict__ tw,
                                         double2* __restrict__ row) {
  using RX = Radix<N>;
  // stage 1: radix 16, NS = 1
  if constexpr (RX::N16 == 1 && RX::REM == 1) {
    stockham_stage<N, 16, 1, SIGN, true>(v, t, tw, row);
  } else {
    stockham_stage<N, 16, 1, SIGN, false>(v, t, tw, row);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = row[t + e * (N / 16)];
    __syncthreads();
    if constexpr (RX::N16 == 1) {
      stockham_stage<N, RX::REM, 16, SIGN, true>(v, t, tw, row);
    } else if constexpr (RX::N16 == 2 && RX::REM == 1) {
      stockham_stage<N, 16, 16, SIGN, true>(v, t, tw, row);
    } else if constexpr (RX::N16 == 2) {
      stockham_stage<N, 16, 16, SIGN, false>(v, t, tw, row);
      __syncthreads();
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = row[t + e * (N / 16)];
      __syncthreads();
      stockham_stage<N, RX::REM, 256, SIGN, true>(v, t, tw, row);
    } else {  // N16 == 3 (N = 4096)
      stockham_stage<N, 16, 16, SIGN, false>(v, t, tw, row);
      __syncthreads();
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = row[t + e * (N / 16)];
      __syncthreads();
      stockham_stage<N, 16, 256, SIGN, true>(v, t, tw, row);
    }
  }
}

// Element (row jl, point p) addresses of the three modes.  blockIdx: x = j block, y = i / m' / m row, z = function.
template <int MODE>
__device__ __forceinline__ long long src_index(const FftArgs& a, int y, int jj, int p) {
  const long long n = a.n;
  if constexpr (MODE == ROW_FWD) return ((long long)y * a.J + jj) * n + p;          // grid[i][j][k=p]
  else if constexpr (MODE == COL) return ((long long)p * n + y) * a.J + jj;          // S[i=p][m'][j]
  else return ((long long)y * n + p) * a.J + jj;                                      // S[i][m'=p][j]
}
template <int MODE>
__device__ __forceinline__ long long dst_index(const FftArgs& a, int y, int jj, int p) {
  const long long n = a.n;
  if constexpr (MODE == ROW_FWD) return ((long long)y * n + p) * a.J + jj;           // S[i][m'=p][j]
  else if constexpr (MODE == COL) return ((long long)p * n + y) * a.J + jj;          // S[m=p][m'][j]
  else return ((long long)y * a.J + jj) * n + p;                                      // grid[i][j][k=p]
}

// Stockham path: N in {16..4096} power of two, JB rows per CTA, JB*N/16 threads.
template <int N, int JB, int SIGN, int MODE>
__global__ void __launch_bounds__(JB * N / 16) fft_pass_kernel(FftArgs a) {
  extern __shared__ double2 smem[];
  constexpr int TPR = N / 16;  // threads per row
  const int tid = threadIdx.x;
  const int jl = tid % JB, t = tid / JB;
  const int y = blockIdx.y;
  const int jj = blockIdx.x * JB + jl;
  const bool jvalid = jj < a.J;
  const double2* src = a.src + (long long)blockIdx.z * a.fstride_src;
  double2* dst = a.dst + (long long)blockIdx.z * a.fstride_dst;
  double2* row = smem + jl * (N + 1);
  // inverse column pass: the m' = B column is never read downstream (ROW_INV zeroes it)
  if constexpr (MODE == COL && SIGN < 0) { if (y == a.nyq) return; }
  if constexpr (MODE == COL && SIGN > 0) { if (y == a.nyq) return; }   // forward: DWT never reads m' = B

  double2 v[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int p = t + e * TPR;
    double2 z = make_double2(0.0, 0.0);
    bool zero = !jvalid;
    if constexpr (SIGN < 0) zero = zero || (p == a.nyq);   // Nyquist bins of the spectrum are zero (soft.py:164)
    if (!zero) z = src[src_index<MODE>(a, y, jj, p)];
    v[e] = z;
  }
  fft_rows<N, SIGN>(v, t, a.tw, row);
  double wj = 1.0;
  if constexpr (MODE == COL && SIGN > 0) { if (jvalid) wj = __ldg(&a.w[a.jbase + jj]); }
  if (jvalid) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int p = t + e * TPR;
      double2 z = v[e];
      if constexpr (MODE == COL && SIGN > 0) { z.x *= wj; z.y *= wj; }
      dst[dst_index<MODE>(a, y, jj, p)] = z;
    }
  }
}

// Direct DFT for non power-of-two or N < 16.  A CTA owns (row y, JC consecutive j) and
// stages those JC length-N rows in shared memory before writing, so COL stays in place.
template <int SIGN, int MODE>
__global__ void __launch_bounds__(256) dft_direct_kernel(FftArgs a, int JC) {
  extern __shared__ double2 col[];
  const int y = blockIdx.y;
  const int n = a.n;
  const int j0 = blockIdx.x * JC;
  const int jc = min(JC, a.J - j0);
  const double2* src = a.src + (long long)blockIdx.z * a.fstride_src;
  double2* dst = a.dst + (long long)blockIdx.z * a.fstride_dst;
  if constexpr (MODE == COL) { if (y == a.nyq) return; }
  for (int idx = threadIdx.x; idx < jc * n; idx += blockDim.x) {
    const int jl = idx % jc, p = idx / jc;
    double2 z = make_double2(0.0, 0.0);
    if (!(SIGN < 0 && p == a.nyq)) z = src[src_index<MODE>(a, y, j0 + jl, p)];
    col[p * JC + jl] = z;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < jc * n; idx += blockDim.x) {
    const int jl = idx % jc, q = idx / jc;
    double2 acc = make_double2(0.0, 0.0);
    for (int p = 0; p < n; ++p) {
      double2 w = __ldg(&a.tw[(int)(((long long)p * q) % n)]);
      if (SIGN < 0) w.y = -w.y;
      acc = cadd(acc, cmul(col[p * JC + jl], w));
    }
    if constexpr (MODE == COL && SIGN > 0) { const double wj = a.w[a.jbase + j0 + jl]; acc.x *= wj; acc.y *= wj; }
    dst[dst_index<MODE>(a, y, j0 + jl, q)] = acc;
  }
}

}  // namespace so3

// Torus DFT stage of FSOFT / iFSOFT (reference fft.py:35-76, soft.py:127-132, 164-172).
//
// The 2-D unnormalised DFT over (alpha, gamma) of every beta slice is done in two HBM
// passes.  Every pass reads or writes FULL contiguous rows on one side and writes or reads
// XB*16-byte chunks inside a single plane on the other side (a transposition that keeps
// HBM locality; the strided-axis FFT that a plain 2-D FFT needs runs at < 50% of HBM):
//
//   forward  K1a (RI): grid[i][j][k]  --FFT_k(+1)-->  T[j][m'][i]          rows (i,j) in
//            K1b (RI): T[j][m'][i]    --FFT_i(+1)-->  X[m'][m][j] * w_j    rows (j,m') in
//   inverse  K4a (CI): X[m'][m][j]    --FFT_m(-1)-->  T[j][m'][i]          rows (j,m') out
//            K4b (CI): T[j][m'][i]    --FFT_m'(-1)--> grid[i][j][k]        rows (i,j) out
//
// so the DWT sees each order pair as one contiguous vector over j (row m'*2B + m of X).
// A CTA transforms XB rows; each thread keeps 16 points in registers and runs a radix-16
// Stockham FFT whose stages exchange through padded shared memory.  Twiddles come from a
// per-plan table tw[k] = exp(+2 pi i k / N).  Non power-of-two or tiny N use a direct
// O(N^2) DFT (the reference also falls back to a kernel-matrix product, fft.py:51-54).
#pragma once
#include "common.cuh"

namespace so3 {

enum FftMode { RI = 0, CI = 1 };   // rows in + chunks out / chunks in + rows out

// A pass transforms rows indexed by (x, y, f): x in [0, X) grouped XB per CTA, y in [0, Y),
// function f.  Element p of row (x, y) sits at  f*fs + y*sy + x*sx + p*sp  (in units of
// complex128); the contiguous side has sp = 1 (rows) or sx = 1 (chunks over x).
struct FftArgs {
  int n;                      // transform length N = 2B
  int nyq;                    // Nyquist bin B
  int X, Y;                   // row grid
  int skip_y;                 // rows with y == skip_y are neither needed nor written (-1: none)
  int zero_p;                 // input point index read as zero (-1: none), the Nyquist bin
  int weight;                 // multiply outputs by w[jbase + x]
  int jbase;
  const double2* src;
  double2* dst;
  long long fs_in, sy_in, sx_in, sp_in;
  long long fs_out, sy_out, sx_out, sp_out;
  const double2* tw;          // N entries, exp(+2 pi i k / N)
  const double* w;            // quadrature weights
  // sharded passes: the pair-major side is addressed through a row table instead of strides,
  // element (x, y, p) at base + tab[y*N + p] * tabJ + x (tab < 0: not stored / read as zero)
  const int* tab_in;
  const int* tab_out;
  int tabJ;
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
// Shared-memory row layout of the exchange: one pad slot per 16 points plus 8/JB (min 1) per
// row keeps every stage's 16-byte stores and loads free of bank conflicts for the thread
// mapping tid = jl + JB*t (checked by simulation for all N, JB used here).
__device__ __forceinline__ int pidx(int i) { return i + (i >> 4); }
template <int N, int JB>
struct RowLayout {
  static constexpr int SIZE = N + N / 16 + (JB >= 8 ? 1 : 8 / JB);
};

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
      for (int r = 0; r < R; ++r) row[pidx(base + r * NS)] = u[r];
    }
  }
}

// Last stage (span NS = N / R, Q = 16 / R butterflies per thread at b = t + q N/16): its
// twiddle w^(r b) = w^(r t) * exp(SIGN 2 pi i r q / 16), so only tb[r] = w^(r t), r < R, come
// from the table -- loaded by the caller before the preceding exchange -- and the q factor is a
// compile-time 16th root (ncu: the last stage of N = 1024 stalled 60 % on its 12 table loads;
// B = 512 FFT stages 16.3 / 15.0 -> 15.2 / 14.7 ms).  Used for R >= 4; with R = 2 the extra
// constant multiplies cost more than the loads they save.
template <int N, int SIGN, int R>
__device__ __forceinline__ void last_twiddles(double2 (&tb)[R], int t, const double2* __restrict__ tw) {
#pragma unroll
  for (int r = 1; r < R; ++r) {
    double2 w = tw[r * t];
    if constexpr (SIGN < 0) w.y = -w.y;
    tb[r] = w;
  }
}

// u[r] *= tb[r] * exp(SIGN 2 pi i r QI / 16), r = RI..R-1 (QI = 0: the plain table twiddle)
template <int R, int SIGN, int QI, int RI>
__device__ __forceinline__ void twiddle_q(double2 (&u)[R], const double2 (&tb)[R]) {
  if constexpr (RI < R) {
    u[RI] = wmul16<(RI * QI) & 15, SIGN>(cmul(u[RI], tb[RI]));
    twiddle_q<R, SIGN, QI, RI + 1>(u, tb);
  }
}

template <int N, int R, int SIGN, int Q, int QI>
__device__ __forceinline__ void last_stage_q(double2 (&v)[16], const double2 (&tb)[R]) {
  double2 u[R];
#pragma unroll
  for (int r = 0; r < R; ++r) u[r] = v[QI + r * Q];
  twiddle_q<R, SIGN, QI, 1>(u, tb);
  dft_reg<R, SIGN>(u);
#pragma unroll
  for (int r = 0; r < R; ++r) v[QI + r * Q] = u[r];
  if constexpr (QI + 1 < Q) last_stage_q<N, R, SIGN, Q, QI + 1>(v, tb);
}

template <int N, int R, int SIGN>
__device__ __forceinline__ void last_stage(double2 (&v)[16], const double2 (&tb)[R]) {
  last_stage_q<N, R, SIGN, 16 / R, 0>(v, tb);
}

template <int N>
struct Radix {
  // N = 16^a * rem; stages: a radix-16 stages then one radix-rem stage (rem in {2,4,8}) if rem > 1.
  static constexpr int LOG = (N == 16) ? 4 : (N == 32) ? 5 : (N == 64) ? 6 : (N == 128) ? 7 : (N == 256) ? 8
                           : (N == 512) ? 9 : (N == 1024) ? 10 : (N == 2048) ? 11 : 12;
  static constexpr int N16 = LOG / 4;
  static constexpr int REM = 1 << (LOG % 4);
};

struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

// The exchanges synchronise the threads sharing `row` through `sync` (the whole CTA, or one
// named-barrier group of a multi-team CTA).
template <int N, int SIGN, class Sync = CtaSync>
__device__ __forceinline__ void fft_rows(double2 (&v)[16], int t, const double2* __restrict__ tw,
                                         double2* __restrict__ row, Sync sync = Sync()) {
  using RX = Radix<N>;
  // exchange: every thread's 16 points of the next stage, N/16 apart
  auto exchange = [&]() {
    sync();
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = row[pidx(t + e * (N / 16))];
    sync();
  };
  // stage 1: radix 16, NS = 1
  if constexpr (RX::N16 == 1 && RX::REM == 1) {
    stockham_stage<N, 16, 1, SIGN, true>(v, t, tw, row);
  } else if constexpr (RX::N16 == 1) {             // N = 32, 64, 128: last stage radix REM, NS = 16
    stockham_stage<N, 16, 1, SIGN, false>(v, t, tw, row);
    if constexpr (RX::REM >= 4) {
      double2 tb[RX::REM];
      last_twiddles<N, SIGN, RX::REM>(tb, t, tw);  // in flight across the exchange
      exchange();
      last_stage<N, RX::REM, SIGN>(v, tb);
    } else {
      exchange();
      stockham_stage<N, RX::REM, 16, SIGN, true>(v, t, tw, row);
    }
  } else if constexpr (RX::N16 == 2 && RX::REM == 1) {   // N = 256
    stockham_stage<N, 16, 1, SIGN, false>(v, t, tw, row);
    exchange();
    stockham_stage<N, 16, 16, SIGN, true>(v, t, tw, row);
  } else if constexpr (RX::N16 == 2) {             // N = 512, 1024, 2048: last stage radix REM, NS = 256
    stockham_stage<N, 16, 1, SIGN, false>(v, t, tw, row);
    exchange();
    stockham_stage<N, 16, 16, SIGN, false>(v, t, tw, row);
    if constexpr (RX::REM >= 4) {
      double2 tb[RX::REM];
      last_twiddles<N, SIGN, RX::REM>(tb, t, tw);  // in flight across the exchange
      exchange();
      last_stage<N, RX::REM, SIGN>(v, tb);
    } else {
      exchange();
      stockham_stage<N, RX::REM, 256, SIGN, true>(v, t, tw, row);
    }
  } else {                                         // N16 == 3 (N = 4096)
    stockham_stage<N, 16, 1, SIGN, false>(v, t, tw, row);
    exchange();
    stockham_stage<N, 16, 16, SIGN, false>(v, t, tw, row);
    exchange();
    stockham_stage<N, 16, 256, SIGN, true>(v, t, tw, row);
  }
}

// Stockham path: N in {16..2048} power of two, XB rows per CTA, XB*N/16 threads (tid = xl + XB*t).
// TAB: row-table (sharded) addressing compiled in; the plain passes instantiate TAB = false.
template <int N, int XB, int SIGN, bool TAB = false, int MINB = (XB * N / 16 <= 128 ? 3 : XB * N / 16 <= 256 ? 2 : 1)>
__global__ void __launch_bounds__(XB * N / 16, MINB) fft_pass_kernel(FftArgs a) {
  extern __shared__ double2 smem[];
  constexpr int TPR = N / 16;  // threads per row
  const int tid = threadIdx.x;
  const int xl = tid % XB, t = tid / XB;
  const int y = blockIdx.y;
  const int x = blockIdx.x * XB + xl;
  if (y == a.skip_y) return;   // uniform per CTA
  const bool xvalid = x < a.X;
  const long long f = blockIdx.z;
  const double2* src = a.src + f * a.fs_in + (long long)y * a.sy_in + (long long)x * a.sx_in;
  double2* dst = a.dst + f * a.fs_out + (long long)y * a.sy_out + (long long)x * a.sx_out;
  double2* row = smem + xl * RowLayout<N, XB>::SIZE;

  double2 v[16];
  if (TAB && a.tab_in) {
    const double2* base = a.src + f * a.fs_in + x;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int p = t + e * TPR;
      const int r = (xvalid && p != a.zero_p) ? __ldg(&a.tab_in[(long long)y * N + p]) : -1;
      v[e] = r >= 0 ? base[(long long)r * a.tabJ] : make_double2(0.0, 0.0);
    }
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int p = t + e * TPR;
      const bool zero = !xvalid || p == a.zero_p;
      v[e] = zero ? make_double2(0.0, 0.0) : src[(long long)p * a.sp_in];
    }
  }
  // row-table passes: the output rows are fetched before the transform (off the critical path)
  int rout[16];
  if (TAB && a.tab_out) {
#pragma unroll
    for (int e = 0; e < 16; ++e) rout[e] = __ldg(&a.tab_out[(long long)y * N + t + e * TPR]);
  }
  fft_rows<N, SIGN>(v, t, a.tw, row);
  double wx = 1.0;
  if (a.weight && xvalid) wx = __ldg(&a.w[a.jbase + x]);
  if (xvalid) {
    double2* tbase = a.dst + f * a.fs_out + x;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int p = t + e * TPR;
      double2 z = v[e];
      z.x *= wx;
      z.y *= wx;
      if (TAB && a.tab_out) {
        if (rout[e] >= 0) tbase[(long long)rout[e] * a.tabJ] = z;
      } else {
        dst[(long long)p * a.sp_out] = z;
      }
    }
  }
}

// Row-table passes of the sharded pipeline (K1b stores, K4a loads through the (m', m) -> row
// table of the all-to-all layout).  The table entries of a CTA depend on y only, so a CTA keeps
// its 16 entries per thread in registers and walks x-tiles blockIdx.x, + gridDim.x, ...: the
// dependent table -> data load pair is paid once per CTA instead of once per tile (at G = 8
// ranks the per-tile dependent load made K4a ~1.5x slower than the plain pass).
template <int N, int XB, int SIGN>
__global__ void __launch_bounds__(XB * N / 16, (XB * N / 16 <= 128 ? 3 : XB * N / 16 <= 256 ? 2 : 1))
    fft_tab_kernel(FftArgs a) {
  extern __shared__ double2 smem[];
  constexpr int TPR = N / 16;
  const int tid = threadIdx.x;
  const int xl = tid % XB, t = tid / XB;
  const int y = blockIdx.y;
  if (y == a.skip_y) return;
  const long long f = blockIdx.z;
  double2* row = smem + xl * RowLayout<N, XB>::SIZE;
  int rin[16], rout[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int p = t + e * TPR;
    rin[e] = a.tab_in ? (p != a.zero_p ? __ldg(&a.tab_in[(long long)y * N + p]) : -1) : p;
    rout[e] = a.tab_out ? __ldg(&a.tab_out[(long long)y * N + p]) : p;
  }
  for (int xt = blockIdx.x; xt * XB < a.X; xt += gridDim.x) {
    const int x = xt * XB + xl;
    const bool xvalid = x < a.X;
    double2 v[16];
    if (a.tab_in) {
      const double2* base = a.src + f * a.fs_in + x;
#pragma unroll
      for (int e = 0; e < 16; ++e)
        v[e] = (xvalid && rin[e] >= 0) ? base[(long long)rin[e] * a.tabJ] : make_double2(0.0, 0.0);
    } else {
      const double2* src = a.src + f * a.fs_in + (long long)y * a.sy_in + (long long)x * a.sx_in;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int p = t + e * TPR;
        v[e] = (!xvalid || p == a.zero_p) ? make_double2(0.0, 0.0) : src[(long long)p * a.sp_in];
      }
    }
    fft_rows<N, SIGN>(v, t, a.tw, row);   // ends behind a barrier: the rows are free for the next tile
    const double wx = (a.weight && xvalid) ? __ldg(&a.w[a.jbase + x]) : 1.0;
    if (xvalid) {
      if (a.tab_out) {
        double2* tbase = a.dst + f * a.fs_out + x;
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (rout[e] >= 0) tbase[(long long)rout[e] * a.tabJ] = make_double2(v[e].x * wx, v[e].y * wx);
      } else {
        double2* dst = a.dst + f * a.fs_out + (long long)y * a.sy_out + (long long)x * a.sx_out;
#pragma unroll
        for (int e = 0; e < 16; ++e) dst[(long long)(t + e * TPR) * a.sp_out] = make_double2(v[e].x * wx, v[e].y * wx);
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// One-pass 2-D transform of whole beta slices for N = 2B <= 64 (a slice is N*N complex128,
// 64 KB at N = 64, so it fits in shared memory): the grid side moves through shared memory
// with coalesced row accesses, the pair-major side is read / written directly (16 bytes per
// element; CTAs of neighbouring j share every 128-byte line in L2).  Same radix code, in the
// same order, as the two passes (K1a then K1b, K4a then K4b), so results are bit-identical
// to them; HBM traffic is one read + one write of the grid instead of two of each.
//   forward (SIGN +1): grid[f][i][j][k] -> X[f][m'][m][j] * w_j   (m' = nyq not written)
//   inverse (SIGN -1): X[f][m'][m][j]   -> grid[f][i][j][k]       (m = nyq and m' = nyq read as 0)
// One CTA per (j, f); thread tid works on row r = tid % N, points t + (N/16) e.
template <int N, int SIGN>
__global__ void __launch_bounds__(N * N / 16, (N >= 64 ? 2 : 4)) fft2d_slice_kernel(const double2* __restrict__ src, double2* __restrict__ dst,
                                                                  const double2* __restrict__ tw, const double* __restrict__ w,
                                                                  long long fstride, int nyq) {
  constexpr int NT = N * N / 16, TPR = N / 16, SIZE = RowLayout<N, N>::SIZE;
  extern __shared__ double2 E[];   // N rows of SIZE (padded), also the FFT exchange rows
  const int j = blockIdx.x;
  const long long f = blockIdx.y;
  const int tid = threadIdx.x, r = tid % N, t = tid / N;
  const long long n = N, n2 = n * n;
  const double2* in = src + f * fstride;
  double2* out = dst + f * fstride;
  double2* row = E + r * SIZE;
  double2 v[16];
  if (SIGN > 0) {
    // grid rows (i, j) for all i: coalesced into E[i][pidx(k)]
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int idx = tid + NT * q, i = idx / N, k = idx % N;
      E[i * SIZE + pidx(k)] = in[((long long)i * n + j) * n + k];
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = row[pidx(t + e * TPR)];
  } else {
    // X[m' = r][m][j], m = t + TPR e; the Nyquist row and column are zero
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int m = t + e * TPR;
      v[e] = (r == nyq || m == nyq) ? make_double2(0.0, 0.0) : in[((long long)r * n + m) * n + j];
    }
  }
  __syncthreads();   // every thread holds its inputs before the rows are reused for exchange
  fft_rows<N, SIGN>(v, t, tw, row);
  __syncthreads();
  // transpose: first-axis outputs become the rows of the second axis
#pragma unroll
  for (int e = 0; e < 16; ++e) E[(t + e * TPR) * SIZE + pidx(r)] = v[e];
  __syncthreads();
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] = row[pidx(t + e * TPR)];
  __syncthreads();
  fft_rows<N, SIGN>(v, t, tw, row);
  if (SIGN > 0) {
    // v[e] = S(m = t + TPR e, m' = r) -> X[m'][m][j] * w_j
    if (r != nyq) {
      const double wj = __ldg(&w[j]);
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int m = t + e * TPR;
        out[((long long)r * n + m) * n + j] = make_double2(v[e].x * wj, v[e].y * wj);
      }
    }
  } else {
    // v[e] = f(i = r, k = t + TPR e): through E for coalesced grid rows
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 16; ++e) row[pidx(t + e * TPR)] = v[e];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int idx = tid + NT * q, i = idx / N, k = idx % N;
      out[((long long)i * n + j) * n + k] = E[i * SIZE + pidx(k)];
    }
  }
  (void)n2;
}

// Direct DFT for non power-of-two or N < 16: a CTA stages XC rows in shared memory and
// computes every output point of them (O(N^2) per row).
template <int SIGN>
__global__ void __launch_bounds__(256) dft_direct_kernel(FftArgs a, int XC) {
  extern __shared__ double2 col[];
  const int y = blockIdx.y;
  if (y == a.skip_y) return;
  const int n = a.n;
  const int x0 = blockIdx.x * XC;
  const int xc = min(XC, a.X - x0);
  const long long f = blockIdx.z;
  const double2* src = a.src + f * a.fs_in + (long long)y * a.sy_in;
  double2* dst = a.dst + f * a.fs_out + (long long)y * a.sy_out;
  for (int idx = threadIdx.x; idx < xc * n; idx += blockDim.x) {
    const int xl = idx % xc, p = idx / xc;
    double2 z = make_double2(0.0, 0.0);
    if (a.tab_in) {
      const int r = p != a.zero_p ? a.tab_in[(long long)y * n + p] : -1;
      if (r >= 0) z = a.src[f * a.fs_in + (long long)r * a.tabJ + x0 + xl];
    } else if (p != a.zero_p) {
      z = src[(long long)(x0 + xl) * a.sx_in + (long long)p * a.sp_in];
    }
    col[p * XC + xl] = z;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < xc * n; idx += blockDim.x) {
    const int xl = idx % xc, q = idx / xc;
    double2 acc = make_double2(0.0, 0.0);
    for (int p = 0; p < n; ++p) {
      double2 w = __ldg(&a.tw[(int)(((long long)p * q) % n)]);
      if (SIGN < 0) w.y = -w.y;
      acc = cadd(acc, cmul(col[p * XC + xl], w));
    }
    if (a.weight) { const double wx = a.w[a.jbase + x0 + xl]; acc.x *= wx; acc.y *= wx; }
    if (a.tab_out) {
      const int r = a.tab_out[(long long)y * n + q];
      if (r >= 0) a.dst[f * a.fs_out + (long long)r * a.tabJ + x0 + xl] = acc;
    } else {
      dst[(long long)(x0 + xl) * a.sx_out + (long long)q * a.sp_out] = acc;
    }
  }
}

}  // namespace so3

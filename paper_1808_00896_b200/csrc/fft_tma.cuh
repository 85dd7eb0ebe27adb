// TMA-fed torus FFT kernels (sm_100a).  The strided side of every FFT tile -- 16-byte
// elements, one per (row, point), N*16 or more bytes apart -- moves by ONE tensor copy
// (cp.async.bulk.tensor) through shared memory instead of per-thread 16-byte loads / stores,
// each of which is its own L1 wavefront and LSU queue entry:
//
//   fft_pass_tstore_kernel   rows-in passes (K1a, K1b): the XB input rows by 1-D bulk copies
//                            (cp.async.bulk) into the exchange rows, chunk-side outputs staged
//                            [p][x] there and sent by one 5-D tensor store per tile
//   fft_pass_tload_kernel    chunks-in passes (K4a, K4b): one 5-D tensor load per tile into the
//                            exchange rows behind an mbarrier with expect_tx; rows out by 1-D
//                            bulk stores (2B >= 512) or from registers
//   fft2d_slice_tma_kernel   one-pass slices (2B <= 64): the pair-major side of a beta slice as
//                            one 4-D tensor load / store
//
// The radix code (fft_rows) and its order are those of the plain kernels, so results are
// bit-identical.  Tensor maps are built per launch on the host (so3fft_b200.cu) with no L2
// promotion (256-byte promotion over-fetched 10 GB per pass at 2B = 1024).  A persistent
// variant (two teams per CTA, a 3-slot smem ring, loads issued one tile ahead) was slower than
// one tile per CTA with the tensor load: 15.0 vs 12.5 ms per inverse stage at 2B = 1024.
#pragma once
#include <cuda.h>
#include "fft.cuh"

namespace so3 {

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(ok)
      : "r"(smem_addr(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tensor_load5(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void tensor_load4(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void tensor_store4(const CUtensorMap* map, int c0, int c1, int c2, int c3, const void* src) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(map),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(src))
               : "memory");
}

// One-pass 2-D slice transform (2B <= 64, fft2d_slice_kernel in fft.cuh) with the pair-major
// side moved by the TMA.  For one beta index j, X[f][m'][m][j] is N*N elements 16 bytes wide
// and N*16 bytes apart: as per-thread accesses every one is its own L1 wavefront (ncu: the
// L1 data pipe at 64-68 %, MIO throttle 35-43 %).  Here one 4-D tensor copy moves the whole
// slice: dims (j as 2 doubles, m', m, f) -- m' before m, so the shared box is [m][m'] and the
// threads, consecutive in m', read / write it conflict-free.  Same radix code and order as
// fft2d_slice_kernel: results are bit-identical (the forward also writes the unused Nyquist
// row m' = B, which the DWT never reads).
template <int N, int SIGN>
__global__ void __launch_bounds__(N * N / 16, (N >= 64 ? 2 : 4))
    fft2d_slice_tma_kernel(const __grid_constant__ CUtensorMap xmap, const double2* __restrict__ src,
                           double2* __restrict__ dst, const double2* __restrict__ tw, const double* __restrict__ w,
                           long long fstride, int nyq) {
  constexpr int NT = N * N / 16, TPR = N / 16, SIZE = RowLayout<N, N>::SIZE;
  extern __shared__ __align__(1024) double2 E[];   // N rows of SIZE (padded); the dense box at its start
  uint64_t* bar = reinterpret_cast<uint64_t*>(E + N * SIZE);
  const int j = blockIdx.x;
  const int f = blockIdx.y;
  const int tid = threadIdx.x, r = tid % N, t = tid / N;
  const long long n = N;
  double2* row = E + r * SIZE;
  double2 v[16];
  if (SIGN > 0) {
    const double2* in = src + f * fstride;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int idx = tid + NT * q, i = idx / N, k = idx % N;
      E[i * SIZE + pidx(k)] = in[((long long)i * n + j) * n + k];
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = row[pidx(t + e * TPR)];
  } else {
    if (tid == 0) {
      mbar_init(bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(bar, N * N * sizeof(double2));
      tensor_load4(E, &xmap, 2 * j, 0, 0, f, bar);
    }
    __syncthreads();   // the barrier is initialised before anyone waits on it
    while (!mbar_try_wait(bar, 0)) {
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int m = t + e * TPR;
      v[e] = (r == nyq || m == nyq) ? make_double2(0.0, 0.0) : E[m * N + r];   // box [m][m']
    }
  }
  __syncthreads();   // every thread holds its inputs before the rows are reused for exchange
  fft_rows<N, SIGN>(v, t, tw, row);
  __syncthreads();
#pragma unroll
  for (int e = 0; e < 16; ++e) E[(t + e * TPR) * SIZE + pidx(r)] = v[e];
  __syncthreads();
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] = row[pidx(t + e * TPR)];
  __syncthreads();
  fft_rows<N, SIGN>(v, t, tw, row);
  if (SIGN > 0) {
    // v[e] = S(m = t + TPR e, m' = r) * w_j -> the dense box [m][m'], one tensor store
    const double wj = __ldg(&w[j]);
    __syncthreads();   // the last exchange's rows are no longer read
#pragma unroll
    for (int e = 0; e < 16; ++e) E[(t + e * TPR) * N + r] = make_double2(v[e].x * wj, v[e].y * wj);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      tensor_store4(&xmap, 2 * j, 0, 0, f, E);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  } else {
    // v[e] = f(i = r, k = t + TPR e): through E for coalesced grid rows
    double2* out = dst + f * fstride;
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
}


__device__ __forceinline__ void tensor_store5(const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                              const void* src) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(map),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_addr(src))
               : "memory");
}

// Rows-in pass (K1a, K1b) as fft_pass_kernel, but the chunk-side outputs leave by ONE tensor
// store per tile: staged [p][x] in the exchange rows (conflict-free for tid = xl + XB t), box
// (2 XB doubles, p mod 256, p / 256, 1, 1).  The per-thread 64-byte chunk stores filled the
// LSU queue (lg_throttle 12.7 % of the plain pass's stalls).
template <int N, int XB, int SIGN, bool BULKIN = false>
__global__ void __launch_bounds__(XB * N / 16, (XB * N / 16 <= 64 ? 3 : XB * N / 16 <= 128 ? 4 : XB * N / 16 <= 256 ? 2 : 1))
    fft_pass_tstore_kernel(const __grid_constant__ CUtensorMap omap, FftArgs a) {
  extern __shared__ __align__(1024) double2 smem[];
  constexpr int TPR = N / 16, SIZE = RowLayout<N, XB>::SIZE;
  const int tid = threadIdx.x;
  const int xl = tid % XB, t = tid / XB;
  const int y = blockIdx.y;
  const int xt = blockIdx.x;
  const int x = xt * XB + xl;
  if (y == a.skip_y) return;   // uniform per CTA
  const long long f = blockIdx.z;
  const double2* src = a.src + f * a.fs_in + (long long)y * a.sy_in + (long long)x * a.sx_in;
  double2* row = smem + xl * SIZE;
  double2 v[16];
  if constexpr (BULKIN) {
    // the XB input rows by 1-D bulk copies into the exchange rows (row stride SIZE = 2 mod 8
    // 16-byte units: the reads below are conflict-free)
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + XB * SIZE);
    if (tid == 0) {
      mbar_init(bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(bar, XB * N * sizeof(double2));
      const double2* r0 = a.src + f * a.fs_in + (long long)y * a.sy_in + (long long)xt * XB * a.sx_in;
#pragma unroll
      for (int r = 0; r < XB; ++r)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_addr(smem + r * SIZE)),
                     "l"(r0 + r * a.sx_in), "r"((uint32_t)(N * sizeof(double2))), "r"(smem_addr(bar))
                     : "memory");
    }
    __syncthreads();
    while (!mbar_try_wait(bar, 0)) {
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int p = t + e * TPR;
      v[e] = p == a.zero_p ? make_double2(0.0, 0.0) : row[p];
    }
    __syncthreads();   // the rows are in registers before the exchange reuses them
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int p = t + e * TPR;
      v[e] = p == a.zero_p ? make_double2(0.0, 0.0) : src[p];
    }
  }
  fft_rows<N, SIGN>(v, t, a.tw, row);   // ends behind a barrier: the rows are free
  const double wx = a.weight ? __ldg(&a.w[a.jbase + x]) : 1.0;
#pragma unroll
  for (int e = 0; e < 16; ++e) smem[(t + e * TPR) * XB + xl] = make_double2(v[e].x * wx, v[e].y * wx);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    tensor_store5(&omap, 2 * xt * XB, 0, 0, y, (int)f, smem);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// Chunks-in pass (K4a, K4b) as fft_pass_kernel, with the tile's chunk side arriving by ONE
// tensor load into the exchange rows (mbarrier after the rows) instead of 16 per-thread loads.
template <int N, int XB, int SIGN, bool BULKOUT = false>
// CTAs per SM: 3 at 2B = 1024 (85 registers, a few spilled) and 4 at 2B = 512: the CTAs mostly
// wait on their tile's tensor load (ncu: half the stall samples on the mbarrier poll), and more
// resident CTAs hide more of it (B=512 inverse stage 12.5 -> 11.1 ms, B=256 1.53 -> 1.31 ms; the
// rows-in kernel is faster at two CTAs at 2B = 1024, 11.75 vs 12.7 ms, and at four at 2B = 512).
__global__ void __launch_bounds__(XB * N / 16, (XB * N / 16 <= 64 ? 3 : XB * N / 16 <= 128 ? 4 : XB * N / 16 <= 256 ? 3 : 1))
    fft_pass_tload_kernel(const __grid_constant__ CUtensorMap imap, FftArgs a) {
  extern __shared__ __align__(1024) double2 smem[];
  constexpr int TPR = N / 16;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + XB * RowLayout<N, XB>::SIZE);
  const int tid = threadIdx.x;
  const int xl = tid % XB, t = tid / XB;
  const int y = blockIdx.y;
  const int xt = blockIdx.x;
  const int x = xt * XB + xl;
  if (y == a.skip_y) return;   // uniform per CTA
  const long long f = blockIdx.z;
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(bar, XB * N * sizeof(double2));
    tensor_load5(smem, &imap, 2 * xt * XB, 0, 0, y, (int)f, bar);
  }
  __syncthreads();
  while (!mbar_try_wait(bar, 0)) {
  }
  double2 v[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int p = t + e * TPR;
    v[e] = p == a.zero_p ? make_double2(0.0, 0.0) : smem[p * XB + xl];
  }
  __syncthreads();   // the box is in registers before the rows are reused for the exchange
  fft_rows<N, SIGN>(v, t, a.tw, smem + xl * RowLayout<N, XB>::SIZE);
  if constexpr (BULKOUT) {
    // rows staged in the exchange rows (stride SIZE, conflict-free) and stored by 1-D bulk copies
    double2* row = smem + xl * RowLayout<N, XB>::SIZE;
#pragma unroll
    for (int e = 0; e < 16; ++e) row[t + e * TPR] = v[e];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      double2* d0 = a.dst + f * a.fs_out + (long long)y * a.sy_out + (long long)xt * XB * a.sx_out;
#pragma unroll
      for (int r = 0; r < XB; ++r)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d0 + r * a.sx_out),
                     "r"(smem_addr(smem + r * RowLayout<N, XB>::SIZE)), "r"((uint32_t)(N * sizeof(double2)))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  } else {
    double2* dst = a.dst + f * a.fs_out + (long long)y * a.sy_out + (long long)x * a.sx_out;
#pragma unroll
    for (int e = 0; e < 16; ++e) dst[t + e * TPR] = v[e];
  }
}

// Row-table passes of the sharded pipeline (fft_tab_kernel in fft.cuh) with the plain-strided
// side moved by 1-D bulk copies: K1b (table on the output) loads its XB input rows by bulk
// copies, K4a (table on the input) stores its XB output rows by bulk copies.  The table side
// stays per thread (its 64-byte chunks go to / come from arbitrary rows of the all-to-all
// buffer).  A CTA keeps its table entries in registers and walks x-tiles as fft_tab_kernel.
template <int N, int XB, int SIGN>
__global__ void __launch_bounds__(XB * N / 16, (XB * N / 16 <= 128 ? 3 : XB * N / 16 <= 256 ? 2 : 1))
    fft_tab_tma_kernel(FftArgs a) {
  extern __shared__ __align__(1024) double2 smem[];
  constexpr int TPR = N / 16, SIZE = RowLayout<N, XB>::SIZE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + XB * SIZE);
  const int tid = threadIdx.x;
  const int xl = tid % XB, t = tid / XB;
  const int y = blockIdx.y;
  if (y == a.skip_y) return;
  const long long f = blockIdx.z;
  double2* row = smem + xl * SIZE;
  const bool rows_in = a.tab_out != nullptr;
  int rtab[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int p = t + e * TPR;
    rtab[e] = rows_in ? __ldg(&a.tab_out[(long long)y * N + p])
                      : (p != a.zero_p ? __ldg(&a.tab_in[(long long)y * N + p]) : -1);
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  for (int xt = blockIdx.x; xt * XB < a.X; xt += gridDim.x) {
    const int x = xt * XB + xl;
    double2 v[16];
    if (rows_in) {
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // earlier generic use of the rows
        mbar_expect_tx(bar, XB * N * sizeof(double2));
        const double2* r0 = a.src + f * a.fs_in + (long long)y * a.sy_in + (long long)xt * XB * a.sx_in;
#pragma unroll
        for (int r = 0; r < XB; ++r)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           smem_addr(smem + r * SIZE)),
                       "l"(r0 + r * a.sx_in), "r"((uint32_t)(N * sizeof(double2))), "r"(smem_addr(bar))
                       : "memory");
      }
      while (!mbar_try_wait(bar, phase)) {
      }
      phase ^= 1;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int p = t + e * TPR;
        v[e] = p == a.zero_p ? make_double2(0.0, 0.0) : row[p];
      }
      __syncthreads();   // the rows are in registers before the exchange reuses them
    } else {
      const double2* base = a.src + f * a.fs_in + x;
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = rtab[e] >= 0 ? base[(long long)rtab[e] * a.tabJ] : make_double2(0.0, 0.0);
    }
    fft_rows<N, SIGN>(v, t, a.tw, row);   // ends behind a barrier: the exchange rows are free
    const double wx = a.weight ? __ldg(&a.w[a.jbase + x]) : 1.0;
    if (rows_in) {
      double2* tbase = a.dst + f * a.fs_out + x;
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (rtab[e] >= 0) tbase[(long long)rtab[e] * a.tabJ] = make_double2(v[e].x * wx, v[e].y * wx);
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) row[t + e * TPR] = make_double2(v[e].x * wx, v[e].y * wx);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        double2* d0 = a.dst + f * a.fs_out + (long long)y * a.sy_out + (long long)xt * XB * a.sx_out;
#pragma unroll
        for (int r = 0; r < XB; ++r)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d0 + r * a.sx_out),
                       "r"(smem_addr(smem + r * SIZE)), "r"((uint32_t)(N * sizeof(double2)))
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncthreads();   // the rows have been read before the next tile's exchange writes them
    }
  }
}

// ---------------------------------------------------------------- persistent (co-resident) passes
// The same passes as one persistent CTA per slot (grid = the number of CTAs the caller lets the
// FFT occupy, e.g. one per SM beside DWT CTAs), walking tiles t = blockIdx.x + k * gridDim.x with
// two shared-memory stages: the next tile's row loads (rows in) or tensor load (chunks in) are in
// flight while this tile is transformed.  Radix code and order are the per-tile kernels', so the
// results are bit-identical.  Tiles index (xt, y', f) with the skipped row y = skip_y removed.
struct TileSpace {
  int nxt, ny, skip;
  __device__ __forceinline__ void decode(long long tile, int& xt, int& y, int& f) const {
    xt = (int)(tile % nxt);
    const long long r = tile / nxt;
    const int yy = (int)(r % ny);
    f = (int)(r / ny);
    y = (skip >= 0 && yy >= skip) ? yy + 1 : yy;
  }
};

template <int N, int XB, int SIGN>
__global__ void __launch_bounds__(XB * N / 16, 2)
    fft_pass_tstore_persist_kernel(const __grid_constant__ CUtensorMap omap, FftArgs a, TileSpace ts, long long ntiles) {
  extern __shared__ __align__(1024) double2 smem[];
  constexpr int TPR = N / 16, SIZE = RowLayout<N, XB>::SIZE, STAGE = XB * SIZE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * STAGE);
  const int tid = threadIdx.x, xl = tid % XB, t = tid / XB;
  auto issue = [&](long long tile, int s) {   // thread 0: the tile's XB rows into stage s
    int xt, y, f;
    ts.decode(tile, xt, y, f);
    mbar_expect_tx(&bar[s], XB * N * sizeof(double2));
    const double2* r0 = a.src + (long long)f * a.fs_in + (long long)y * a.sy_in + (long long)xt * XB * a.sx_in;
#pragma unroll
    for (int r = 0; r < XB; ++r)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_addr(smem + s * STAGE + r * SIZE)),
                   "l"(r0 + r * a.sx_in), "r"((uint32_t)(N * sizeof(double2))), "r"(smem_addr(&bar[s]))
                   : "memory");
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if ((long long)blockIdx.x < ntiles) issue(blockIdx.x, 0);
  }
  __syncthreads();
  int it = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it & 1;
    double2* st = smem + s * STAGE;
    double2* row = st + xl * SIZE;
    if (tid == 0 && tile + gridDim.x < ntiles) {
      // stage s^1 was last read by the previous tile's tensor store
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tile + gridDim.x, s ^ 1);
    }
    int xt, y, f;
    ts.decode(tile, xt, y, f);
    while (!mbar_try_wait(&bar[s], (it >> 1) & 1)) {
    }
    double2 v[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int p = t + e * TPR;
      v[e] = p == a.zero_p ? make_double2(0.0, 0.0) : row[p];
    }
    __syncthreads();   // the rows are in registers before the exchange reuses them
    fft_rows<N, SIGN>(v, t, a.tw, row);   // ends behind a barrier
    const int x = xt * XB + xl;
    const double wx = a.weight ? __ldg(&a.w[a.jbase + x]) : 1.0;
#pragma unroll
    for (int e = 0; e < 16; ++e) st[(t + e * TPR) * XB + xl] = make_double2(v[e].x * wx, v[e].y * wx);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      tensor_store5(&omap, 2 * xt * XB, 0, 0, y, f, st);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <int N, int XB, int SIGN, bool BULKOUT>
__global__ void __launch_bounds__(XB * N / 16, 2)
    fft_pass_tload_persist_kernel(const __grid_constant__ CUtensorMap imap, FftArgs a, TileSpace ts, long long ntiles) {
  extern __shared__ __align__(1024) double2 smem[];
  constexpr int TPR = N / 16, SIZE = RowLayout<N, XB>::SIZE, STAGE = XB * SIZE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * STAGE);
  const int tid = threadIdx.x, xl = tid % XB, t = tid / XB;
  auto issue = [&](long long tile, int s) {   // thread 0: the tile's chunk side into stage s
    int xt, y, f;
    ts.decode(tile, xt, y, f);
    mbar_expect_tx(&bar[s], XB * N * sizeof(double2));
    tensor_load5(smem + s * STAGE, &imap, 2 * xt * XB, 0, 0, y, f, &bar[s]);
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if ((long long)blockIdx.x < ntiles) issue(blockIdx.x, 0);
  }
  __syncthreads();
  int it = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it & 1;
    double2* st = smem + s * STAGE;
    if (tid == 0 && tile + gridDim.x < ntiles) {
      if constexpr (BULKOUT) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // earlier generic use of stage s^1
      issue(tile + gridDim.x, s ^ 1);
    }
    int xt, y, f;
    ts.decode(tile, xt, y, f);
    while (!mbar_try_wait(&bar[s], (it >> 1) & 1)) {
    }
    double2 v[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int p = t + e * TPR;
      v[e] = p == a.zero_p ? make_double2(0.0, 0.0) : st[p * XB + xl];
    }
    __syncthreads();   // the box is in registers before the rows are reused for the exchange
    double2* row = st + xl * SIZE;
    fft_rows<N, SIGN>(v, t, a.tw, row);
    if constexpr (BULKOUT) {
#pragma unroll
      for (int e = 0; e < 16; ++e) row[t + e * TPR] = v[e];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        double2* d0 = a.dst + (long long)f * a.fs_out + (long long)y * a.sy_out + (long long)xt * XB * a.sx_out;
#pragma unroll
        for (int r = 0; r < XB; ++r)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d0 + r * a.sx_out),
                       "r"(smem_addr(st + r * SIZE)), "r"((uint32_t)(N * sizeof(double2)))
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {
      double2* dst = a.dst + (long long)f * a.fs_out + (long long)y * a.sy_out + (long long)(xt * XB + xl) * a.sx_out;
#pragma unroll
      for (int e = 0; e < 16; ++e) dst[t + e * TPR] = v[e];
      __syncthreads();   // every thread is done with stage s before it is reloaded
    }
  }
  if constexpr (BULKOUT) {
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

}  // namespace so3

// Chunks-in torus FFT pass (K4a, K4b: the inverse direction) fed by the Tensor Memory
// Accelerator (sm_100a): the same rows, radix code and exchange layout as fft_pass_kernel
// (fft.cuh), so results are bit-identical, but the strided chunk side of every tile arrives by
// one asynchronous 5-D tensor copy instead of 16 per-thread loads.
//
// One persistent CTA per SM holds G thread teams of XB*N/16 threads and a ring of S > G
// shared-memory slots of one tile (XB = 4 rows of N complex128) each.  Team g takes the CTA's
// local tiles g, g + G, ...; tile k lives in slot k % S.  While the teams transform their
// tiles, the TMA fills the spare slots with the next tiles, so a tile's HBM latency is paid
// under another tile's arithmetic instead of by registers held across the load.  Per tile:
//
//   full[k % S] (mbarrier, expect_tx)  <-  tensor load of tile k: box (2 XB doubles, p mod 256,
//                                          p / 256, 1, 1), staged [p][x] (64 bytes per p)
//   team: slot -> registers, fft_rows with the exchange rows in the slot itself (one named
//         barrier per team), then one thread issues the load of tile k + S into the slot and
//         the team stores its rows from registers.
//
// Measured at 2B = 1024 (B200): 14.6 ms vs 15.2 ms per inverse FFT stage.  The rows-in passes
// (K1a, K1b) were also built this way -- 1-D bulk row loads, tensor or register stores -- and
// were slower than the plain kernel (17.8-18.6 ms vs 14.7 ms per forward stage), as were both
// directions at 2B = 256 and 512, so only this pass uses the TMA.  The tensor map
// must not promote L2 fills (256-byte promotion over-fetched 10 GB per pass).
#pragma once
#include <cuda.h>
#include "fft.cuh"

namespace so3 {

struct FftTmaArgs {
  int X, Y, skip_y, zero_p;
  long long ntiles;          // (X / XB) * (rows y other than skip_y) * batch
  double2* rows_dst;         // output rows: element (x, y, p, f) at f*fs + y*sy + x*sx + p
  long long fs, sy, sx;
  const double2* tw;
};

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

struct TeamSync {
  int id, count;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory"); }
};

template <int N>
struct TmaGeom {
  static constexpr int XB = 4;
  static constexpr int TPG = XB * N / 16;                         // threads per team
  static constexpr int G = N >= 1024 ? 2 : N >= 512 ? 4 : 8;       // teams per CTA (512 threads)
  static constexpr int SLOT = XB * RowLayout<N, XB>::SIZE;         // complex128 per slot (exchange rows)
  static constexpr int S = N >= 1024 ? 3 : N >= 512 ? 6 : 12;      // ring slots (> G, ~210 KB)
  static constexpr size_t SMEM = (size_t)S * SLOT * sizeof(double2);
  static_assert((SLOT * sizeof(double2)) % 128 == 0, "slots must stay 128-byte aligned for the tensor copies");
};

template <int N, int SIGN>
__global__ void __launch_bounds__(TmaGeom<N>::G * TmaGeom<N>::TPG, 1)
    fft_tma_kernel(const __grid_constant__ CUtensorMap tmap, FftTmaArgs a) {
  using TG = TmaGeom<N>;
  constexpr int XB = TG::XB, TPG = TG::TPG, G = TG::G, S = TG::S, SLOT = TG::SLOT, TPR = N / 16;
  constexpr uint32_t TILE_BYTES = XB * N * sizeof(double2);
  extern __shared__ __align__(1024) double2 smem[];
  __shared__ uint64_t full[S];
  __shared__ volatile long long issued[S];   // local tile whose load was last issued into slot s
  const int tid = threadIdx.x, team = tid / TPG, lt = tid % TPG;
  const int xl = lt % XB, t = lt / XB;
  const int XT = a.X / XB;
  const int Yv = a.Y - (a.skip_y >= 0 ? 1 : 0);
  const long long per_f = (long long)XT * Yv;

  auto coords = [&](long long tile, int& xt, int& y, int& f) {
    f = (int)(tile / per_f);
    const long long r = tile - (long long)f * per_f;
    y = (int)(r / XT);
    xt = (int)(r - (long long)y * XT);
    if (a.skip_y >= 0 && y >= a.skip_y) ++y;
  };
  // one thread: the tensor load of local tile k into slot k % S
  auto issue = [&](long long k) {
    const long long tile = blockIdx.x + k * gridDim.x;
    if (tile >= a.ntiles) return;
    int xt, y, f;
    coords(tile, xt, y, f);
    const int sl = (int)(k % S);
    mbar_expect_tx(&full[sl], TILE_BYTES);
    tensor_load5(smem + (size_t)sl * SLOT, &tmap, 2 * xt * XB, 0, 0, y, f, &full[sl]);
    issued[sl] = k;
  };

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      issued[s] = -1;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int k = 0; k < S; ++k) issue(k);

  const TeamSync sync{1 + team, TPG};
  for (long long k = team; blockIdx.x + k * gridDim.x < a.ntiles; k += G) {
    const long long tile = blockIdx.x + k * gridDim.x;
    int xt, y, f;
    coords(tile, xt, y, f);
    const int sl = (int)(k % S);
    double2* slot = smem + (size_t)sl * SLOT;
    // the load of tile k must have been ISSUED before its parity is tested: an earlier phase
    // of the same slot has the same parity
    while (issued[sl] != k) {
    }
    while (!mbar_try_wait(&full[sl], (uint32_t)((k / S) & 1))) {
    }
    double2 v[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int p = t + e * TPR;
      v[e] = p == a.zero_p ? make_double2(0.0, 0.0) : slot[p * XB + xl];   // [p][x] box
    }
    sync();   // the whole tile is in registers before the slot becomes the exchange rows
    fft_rows<N, SIGN>(v, t, a.tw, slot + xl * RowLayout<N, XB>::SIZE, sync);
    // the last exchange ended with a team barrier: the slot is free, refill it now and store
    // the rows straight from registers (128-byte lines per quarter warp)
    if (lt == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + S);
    }
    double2* out = a.rows_dst + f * a.fs + (long long)y * a.sy + (long long)(xt * XB + xl) * a.sx;
#pragma unroll
    for (int e = 0; e < 16; ++e) out[t + e * TPR] = v[e];
  }
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

}  // namespace so3

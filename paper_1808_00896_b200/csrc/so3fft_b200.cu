// so3fft_b200: plan construction (host, long double) and the C ABI of include/so3fft_b200.h.
//
// Reference mapping (pkg/src/so3fft):
//   make_plan          soft.py:80-108     -> so3_plan_create
//   _fsoft             soft.py:124-149    -> so3_fsoft  = fft_analysis + dwt_analysis
//   _ifsoft            soft.py:152-173    -> so3_ifsoft = dwt_synthesis + fft_synthesis
//   quadrature_weights quadrature.py:66-73, sample_angles quadrature.py:57-63
//   enumerate_clusters schedule.py:136-158 (kappa order) -> cost-sorted launch order
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <thread>
#include <map>
#include <mutex>
#include <tuple>

#include "../../include/so3fft_b200.h"
#include "common.cuh"
#include "sofio.cuh"
#include "hostio.cuh"
#include "dwt.cuh"
#include "dwt_mma.cuh"
#include "dwt_batch.cuh"
#include "dwt_seg.cuh"
#include "fft.cuh"
#include "fft_tma.cuh"
#include "direct.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define SO3_CUDA(call)                                                                         \
  do {                                                                                         \
    cudaError_t _e = (call);                                                                   \
    if (_e != cudaSuccess)                                                                     \
      return fail(SO3_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));           \
  } while (0)

bool valid_bandwidth(int b) { return b >= 1 && b <= 4096; }
constexpr int kMaxBandwidth = 512;   // DWT kernels: at most 2B = 1024 beta indices per cluster

// Per-plan launch knobs that act inside the launch helpers (which take kernel arguments, not
// the plan): each C-ABI stage entry point installs its plan's values for the duration of the
// call (KnobScope), so they stay per plan.  carveout: cudaFuncAttributePreferredSharedMemory-
// Carveout of the big kernels (-1 = driver default; kernels with different carveouts cannot
// share an SM); dwt_pad: extra KB of dynamic shared memory per MMA DWT CTA (experiments with
// fewer DWT CTAs per SM).
struct LaunchKnobs {
  int carveout = -1;
  int dwt_pad = 0;
};
thread_local LaunchKnobs t_knobs;

// The attributes are set once per (kernel, device, value): cudaFuncSetAttribute on a kernel that
// may be running is not free, and launches on other streams must not wait behind it.
template <typename K>
cudaError_t set_smem(K k, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int>, std::pair<size_t, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(k), dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(key);
  const size_t have = it == done.end() ? 48 * 1024 : it->second.first;
  const int cv = it == done.end() ? -1 : it->second.second;
  cudaError_t e = cudaSuccess;
  if (smem > have) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int want = t_knobs.carveout;
  if (!e && want != cv && want >= 0) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, want);
  if (!e) done[key] = {std::max(have, smem), want >= 0 ? want : cv};
  return e;
}

// ---------------------------------------------------------------- host tables

const long double kPi = 3.141592653589793238462643383279502884L;

void host_weights(int b, double* out) {
  // w_B(j) = (2 pi / B^2) sin(beta_j) sum_{i<B} sin((2i+1) beta_j) / (2i+1)  (quadrature.py:66-73)
  const int n = 2 * b;
  for (int j = 0; j < n; ++j) {
    const long double beta = (2.0L * j + 1.0L) * kPi / (4.0L * b);
    long double s = 0.0L;
    for (int i = 0; i < b; ++i) s += sinl((2.0L * i + 1.0L) * beta) / (2.0L * i + 1.0L);
    out[j] = (double)((2.0L * kPi / ((long double)b * b)) * sinl(beta) * s);
  }
}

struct Cluster { int m, mp, members; };

// Symmetry clusters of base pairs 0 <= m' <= m < B (schedule.py:123-158), ordered by
// cost = members * (B - m) descending so the hardware CTA scheduler runs the longest
// first (the GPU form of the reference's dynamic schedule, schedule.py:228-242).
std::vector<Cluster> host_clusters(int b) {
  std::vector<Cluster> cl;
  cl.reserve((size_t)b * (b + 1) / 2);
  for (int m = 0; m < b; ++m)
    for (int mp = 0; mp <= m; ++mp) {
      const int mem = (m == 0) ? 1 : (mp == 0 || mp == m) ? 4 : 8;
      cl.push_back({m, mp, mem});
    }
  std::stable_sort(cl.begin(), cl.end(), [b](const Cluster& x, const Cluster& y) {
    const long long cx = (long long)x.members * (b - x.m), cy = (long long)y.members * (b - y.m);
    if (cx != cy) return cx > cy;
    if (x.m != y.m) return x.m < y.m;
    return x.mp < y.mp;
  });
  return cl;
}

// Cost-balanced cluster groups for `world` ranks: longest-processing-time greedy over the
// cost-sorted schedule (cost = members * (B - m), the DWT work of a cluster).  The GPU form
// of the reference's dynamic work split (schedule.py:200-248) across devices.
std::vector<int> shard_owner(const std::vector<Cluster>& cl, int b, int world) {
  std::vector<long long> load(world, 0);
  std::vector<int> owner(cl.size());
  for (size_t i = 0; i < cl.size(); ++i) {
    int best = 0;
    for (int r = 1; r < world; ++r)
      if (load[r] < load[best]) best = r;
    owner[i] = best;
    load[best] += (long long)cl[i].members * (b - cl[i].m) + 1;
  }
  return owner;
}

// Exchange chunks of the sharded pipeline: each rank's cost-sorted cluster list is cut into
// `chunks` contiguous runs of (nearly) equal DWT cost, so the all-to-all of chunk q+1 can
// overlap the DWT of chunk q.  chunk_of[i] for schedule entry i (its owner's run).
std::vector<int> shard_chunks(const std::vector<Cluster>& cl, const std::vector<int>& owner, int b, int world,
                              int chunks) {
  std::vector<long long> total(world, 0), seen(world, 0);
  for (size_t i = 0; i < cl.size(); ++i) total[owner[i]] += (long long)cl[i].members * (b - cl[i].m) + 1;
  std::vector<int> chunk_of(cl.size());
  for (size_t i = 0; i < cl.size(); ++i) {
    const int r = owner[i];
    chunk_of[i] = (int)std::min<long long>(chunks - 1, seen[r] * chunks / std::max<long long>(total[r], 1));
    seen[r] += (long long)cl[i].members * (b - cl[i].m) + 1;
  }
  return chunk_of;
}

// Member order pairs of a base pair in tag order (schedule.py:115-133), as make_member.
std::vector<std::pair<int, int>> cluster_pairs(int m, int mp) {
  static const int rel[8][4] = {{1, 0, 0, 1}, {-1, 0, 0, -1}, {0, 1, 1, 0}, {0, -1, -1, 0},
                                {-1, 0, 0, 1}, {1, 0, 0, -1}, {0, -1, 1, 0}, {0, 1, -1, 0}};
  std::vector<int> tags;
  if (m == 0) tags = {0};
  else if (mp == 0) tags = {0, 1, 2, 3};
  else if (mp == m) tags = {0, 1, 4, 5};
  else tags = {0, 1, 2, 3, 4, 5, 6, 7};
  std::vector<std::pair<int, int>> out;
  for (int t : tags) out.push_back({rel[t][0] * m + rel[t][1] * mp, rel[t][2] * m + rel[t][3] * mp});
  return out;
}

void split_ld(long double v, double* hi, double* lo) {
  *hi = (double)v;
  *lo = (double)(v - (long double)*hi);
}

}  // namespace

struct so3_plan_s {
  int B = 0, n = 0, batch = 1, device = 0;
  int64_t ncoef = 0, ngrid = 0, nclusters = 0;
  int2* d_bases = nullptr;
  double2* d_lnorm = nullptr;
  double* d_xv = nullptr;            // v_j of rec_t: cos(beta_j) = (j < B ? 1 : -1) + v_j
  double4* d_logcs = nullptr;
  double* d_w = nullptr;
  double2* d_tw = nullptr;
  double2* d_scratch = nullptr;      // T: pass-1 output / pass-2 input
  double2* d_spec = nullptr;         // X: pair-major spectrum [m'][m][j]
  double* d_rc = nullptr;            // recurrence coefficient table
  long long* d_rc_off = nullptr;
  // staging for the host-buffer entry points
  double2* d_grid_stage = nullptr;
  double2* d_coef_stage = nullptr;
  so3host::Staging host_stage;         // pinned bounce buffers for pageable host buffers (hostio.cuh)
  int64_t bytes = 0;
  // sharding (world > 1 or a sharded plan): beta slab [jbase, jbase + J) and a cluster group
  int sharded = 0, world = 1, rank = 0, J = 0, jbase = 0;
  int64_t pairs_rank = 0;               // order pairs owned by this rank (DWT rows)
  std::vector<int64_t> pairs_of;        // pairs per rank
  int* d_row_global = nullptr;          // (m' bin)*n + (m bin) -> row of layout A [chunk q][rank g][pairs_{g,q}], -1 if none
  int* d_row_local = nullptr;           // same index -> row among this rank's pairs of its chunk, -1 if not owned
  int chunks = 1;                       // exchange chunks (layouts are chunk-major, see the header)
  std::vector<int64_t> chunk_cl;        // this rank's clusters of chunk q: [chunk_cl[q], chunk_cl[q+1])
  std::vector<int64_t> chunk_pairs;     // this rank's pairs of chunk q
  std::vector<int64_t> chunk_off;       // prefix of chunk_pairs
  int dwt_variant = SO3_DWT_MMA;
  int syn_jw = 0;     // dev knob (SO3_SYN_JW): beta indices per warp in the synthesis kernel
  int ana_split = 1;  // 2B = 1024 analysis: each cluster over two 4-warp CTAs (dwt_mma.cuh, SPLIT = 2)
  long long rc_entries = 0;       // recurrence-table entries = sum over the plan's clusters of (B - m)
  double2* d_pbuf = nullptr;      // split analysis: per-half partial sums, 2 x rc_entries x 8
  unsigned* d_pcnt = nullptr;     // split analysis: per-cluster arrival counters
  // segment-parallel DWT (dwt_seg.cuh): checkpoint table [cluster][8][2B] of recurrence states
  int dwt_seg = 1;                // knob, bits: 1 = segment-parallel synthesis, 2 = analysis, 4 = persistent analysis (B % 64 == 0)
  int seg_ana_w = 8;              // knob: most warps per analysis CTA (8: one CTA per SM; 4: two)
  double2* d_ck = nullptr;
  double* d_seed = nullptr;       // batched plans with 2B <= 64: recurrence seeds per (cluster, beta index)
  int pbuf_splits = 0;            // partial sets d_pbuf holds
  int fft_wide = 0;   // dev knob (SO3_FFT_XB): rows per FFT CTA override
  int fft_fused = 1;  // 2B <= 64: one-pass 2-D slice transform (fft2d_slice_kernel)
  int fft_tma = 1;    // TMA-fed FFT kernels (fft_tma.cuh): passes at 2B in {256, 512, 1024}, one-pass slices
  int fft_bulkin = 1;    // rows-in TMA passes also load their rows by 1-D bulk copies
  int fft_bulkout = -1;  // chunks-in TMA passes store their rows by 1-D bulk copies (-1: 2B >= 512)
  int fft_tab_loop = 8;  // x-tiles per CTA of the sharded row-table passes (0: one tile per CTA)
  int fft_tab_tma = 1;   // row-table passes move their plain-strided side by bulk copies
  int dwt_batch = 1;  // batched plans with 2B <= 64: dense-contraction DWT kernels (dwt_batch.cuh)
  int fft_pad = 0;    // extra KB of shared memory per TMA FFT pass CTA (limits FFT CTAs per SM when co-running)
  int fft_persist = 0;  // > 0: TMA passes as this many persistent double-buffered CTAs (fft_tma.cuh)
  int carveout = -1;    // see LaunchKnobs
  int dwt_pad = 0;      // see LaunchKnobs
};

// installs a plan's LaunchKnobs for one C-ABI call
struct KnobScope {
  LaunchKnobs saved;
  explicit KnobScope(const so3_plan_s* p) : saved(t_knobs) { t_knobs = LaunchKnobs{p->carveout, p->dwt_pad}; }
  ~KnobScope() { t_knobs = saved; }
};

// ------------------------------------------------------------------ launches

namespace {


template <int N, int XB>
int launch_fft_pow2(const so3_plan_s* p, const so3::FftArgs& a, int sign, int batch, cudaStream_t st) {
  const int threads = XB * N / 16;
  const size_t smem = (size_t)XB * so3::RowLayout<N, XB>::SIZE * sizeof(double2);
  dim3 grid((a.X + XB - 1) / XB, a.Y, batch);
  const bool tab = a.tab_in || a.tab_out;
  if (tab && p->fft_tab_loop > 0 && p->fft_tab_tma && XB == 4 && (N == 256 || N == 512 || N == 1024) && a.X % XB == 0 &&
      !(a.tab_in && a.tab_out) && (a.tab_out ? a.sp_in == 1 : a.sp_out == 1)) {
    constexpr int NT = (N == 256 || N == 512 || N == 1024) ? N : 256;
    auto kt = sign > 0 ? so3::fft_tab_tma_kernel<NT, 4, +1> : so3::fft_tab_tma_kernel<NT, 4, -1>;
    const size_t smem_t = (size_t)4 * so3::RowLayout<NT, 4>::SIZE * sizeof(double2) + 16;
    SO3_CUDA(set_smem(kt, smem_t));
    grid.x = (grid.x + p->fft_tab_loop - 1) / p->fft_tab_loop;
    kt<<<grid, threads, smem_t, st>>>(a);
    SO3_CUDA(cudaGetLastError());
    return SO3_OK;
  }
  if (tab && p->fft_tab_loop > 0) {
    auto kt = sign > 0 ? so3::fft_tab_kernel<N, XB, +1> : so3::fft_tab_kernel<N, XB, -1>;
    SO3_CUDA(set_smem(kt, smem));
    grid.x = (grid.x + p->fft_tab_loop - 1) / p->fft_tab_loop;
    kt<<<grid, threads, smem, st>>>(a);
    SO3_CUDA(cudaGetLastError());
    return SO3_OK;
  }
  void (*k)(so3::FftArgs) = sign > 0 ? (tab ? so3::fft_pass_kernel<N, XB, +1, true> : so3::fft_pass_kernel<N, XB, +1, false>)
                                     : (tab ? so3::fft_pass_kernel<N, XB, -1, true> : so3::fft_pass_kernel<N, XB, -1, false>);
  SO3_CUDA(set_smem(k, smem));
  k<<<grid, threads, smem, st>>>(a);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

int launch_fft_direct(const so3::FftArgs& a, int sign, int batch, cudaStream_t st) {
  const int XC = std::max(1, std::min(a.X, 2048 / a.n));
  const size_t smem = (size_t)XC * a.n * sizeof(double2);
  dim3 grid((a.X + XC - 1) / XC, a.Y, batch);
  void (*k)(so3::FftArgs, int) = sign > 0 ? so3::dft_direct_kernel<+1> : so3::dft_direct_kernel<-1>;
  SO3_CUDA(set_smem(k, smem));
  k<<<grid, 256, smem, st>>>(a, XC);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static const EncodeTiledFn fn = [] {   // thread-safe one-time query
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFn>(ptr);
    return static_cast<EncodeTiledFn>(nullptr);
  }();
  return fn;
}

// returns -1 when the TMA pass does not apply (row tables, odd sizes, knob off)
int launch_fft_tma(const so3_plan_s* p, const so3::FftArgs& a, int sign, cudaStream_t st);

// XB (rows per CTA) = the chunk width on the transposed side (XB * 16 bytes).
template <int N>
int launch_fft_xb(const so3_plan_s* p, const so3::FftArgs& a, int sign, int batch, cudaStream_t st, int xb) {
  switch (xb) {
    case 2: return launch_fft_pow2<N, 2>(p, a, sign, batch, st);
    case 4: return launch_fft_pow2<N, 4>(p, a, sign, batch, st);
    case 8: return launch_fft_pow2<N, 8>(p, a, sign, batch, st);
    default: return launch_fft_pow2<N, 16>(p, a, sign, batch, st);
  }
}

int launch_fft(const so3_plan_s* p, const so3::FftArgs& a, int sign, int batch, cudaStream_t st) {
  const int xb_override = p->fft_wide;
  switch (a.n) {
    case 16: return launch_fft_pow2<16, 16>(p, a, sign, batch, st);
    case 32: return launch_fft_pow2<32, 32>(p, a, sign, batch, st);
    case 64: return launch_fft_pow2<64, 32>(p, a, sign, batch, st);
    case 128: return launch_fft_pow2<128, 32>(p, a, sign, batch, st);
    case 256: return launch_fft_xb<256>(p, a, sign, batch, st, xb_override ? xb_override : 4);
    case 512: return launch_fft_xb<512>(p, a, sign, batch, st, xb_override ? xb_override : 4);
    case 1024: return launch_fft_xb<1024>(p, a, sign, batch, st, xb_override ? xb_override : 4);
    case 2048: return launch_fft_pow2<2048, 2>(p, a, sign, batch, st);
    default: return launch_fft_direct(a, sign, batch, st);
  }
}

// Slice transform with the pair-major side by TMA (fft_tma.cuh): tensor map over X with dims
// (j as doubles, m', m, f) -- strides n^2, n, n^3 complex128 -- and box (2, N, N, 1).
template <int N, int SIGN>
int launch_fft2d_tma_t(const so3_plan_s* p, const void* src, void* dst, cudaStream_t st) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return -1;
  const void* x = SIGN > 0 ? dst : src;
  const cuuint64_t n = (cuuint64_t)N;
  const cuuint64_t dims[4] = {2 * n, n, n, (cuuint64_t)p->batch};
  const cuuint64_t strides[3] = {n * n * 16, n * 16, (cuuint64_t)p->ngrid * 16};
  const cuuint32_t box[4] = {2, (cuuint32_t)N, (cuuint32_t)N, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUtensorMap map;
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(x), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;   // the plain slice kernel takes over
  const size_t smem = (size_t)N * so3::RowLayout<N, N>::SIZE * sizeof(double2) + 16;
  auto k = so3::fft2d_slice_tma_kernel<N, SIGN>;
  SO3_CUDA(set_smem(k, smem));
  k<<<dim3(N, p->batch), N * N / 16, smem, st>>>(map, static_cast<const double2*>(src), static_cast<double2*>(dst),
                                                 p->d_tw, p->d_w, p->ngrid, p->B);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

template <int N, int SIGN>
int launch_fft2d_t(const so3_plan_s* p, const void* src, void* dst, cudaStream_t st) {
  if (p->fft_tma) {
    const int rc = launch_fft2d_tma_t<N, SIGN>(p, src, dst, st);
    if (rc >= 0) return rc;
  }
  const size_t smem = (size_t)N * so3::RowLayout<N, N>::SIZE * sizeof(double2);
  auto k = so3::fft2d_slice_kernel<N, SIGN>;
  SO3_CUDA(set_smem(k, smem));
  k<<<dim3(N, p->batch), N * N / 16, smem, st>>>(static_cast<const double2*>(src), static_cast<double2*>(dst), p->d_tw,
                                               p->d_w, p->ngrid, p->B);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

// One-pass slice transform when a whole beta slice fits in shared memory (2B in {16, 32, 64});
// returns -1 when it does not apply.
int launch_fft2d(const so3_plan_s* p, int sign, const void* src, void* dst, cudaStream_t st) {
  if (!p->fft_fused || p->sharded) return -1;
  switch (p->n) {
    case 16: return sign > 0 ? launch_fft2d_t<16, +1>(p, src, dst, st) : launch_fft2d_t<16, -1>(p, src, dst, st);
    case 32: return sign > 0 ? launch_fft2d_t<32, +1>(p, src, dst, st) : launch_fft2d_t<32, -1>(p, src, dst, st);
    case 64: return sign > 0 ? launch_fft2d_t<64, +1>(p, src, dst, st) : launch_fft2d_t<64, -1>(p, src, dst, st);
    default: return -1;
  }
}

// Rows-in pass with a TMA tensor store of each tile's chunk side (fft_tma.cuh).
template <int N, int SIGN>
int launch_fft_tstore_t(const so3_plan_s* p, const so3::FftArgs& a, int batch, cudaStream_t st) {
  constexpr int XB = 4;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return -1;
  const int plo = N < 256 ? N : 256, phi = N / plo;
  const cuuint64_t dims[5] = {(cuuint64_t)2 * a.X, (cuuint64_t)plo, (cuuint64_t)phi, (cuuint64_t)a.Y, (cuuint64_t)batch};
  const cuuint64_t strides[4] = {(cuuint64_t)a.sp_out * 16, (cuuint64_t)plo * a.sp_out * 16, (cuuint64_t)a.sy_out * 16,
                                 (cuuint64_t)std::max<long long>(a.fs_out, 1) * 16};
  const cuuint32_t box[5] = {(cuuint32_t)(2 * XB), (cuuint32_t)plo, (cuuint32_t)phi, 1, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUtensorMap map;
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, a.dst, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  const size_t smem = (size_t)XB * so3::RowLayout<N, XB>::SIZE * sizeof(double2) + 16 + (size_t)p->fft_pad * 1024;
  auto k = p->fft_bulkin ? (SIGN > 0 ? so3::fft_pass_tstore_kernel<N, XB, +1, true> : so3::fft_pass_tstore_kernel<N, XB, -1, true>)
                        : (SIGN > 0 ? so3::fft_pass_tstore_kernel<N, XB, +1> : so3::fft_pass_tstore_kernel<N, XB, -1>);
  SO3_CUDA(set_smem(k, smem));
  k<<<dim3(a.X / XB, a.Y, batch), XB * N / 16, smem, st>>>(map, a);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

// Chunks-in pass with a TMA tensor load of each tile's chunk side (fft_tma.cuh).
template <int N, int SIGN>
int launch_fft_tload_t(const so3_plan_s* p, const so3::FftArgs& a, int batch, cudaStream_t st) {
  constexpr int XB = 4;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return -1;
  const int plo = N < 256 ? N : 256, phi = N / plo;
  const cuuint64_t dims[5] = {(cuuint64_t)2 * a.X, (cuuint64_t)plo, (cuuint64_t)phi, (cuuint64_t)a.Y, (cuuint64_t)batch};
  const cuuint64_t strides[4] = {(cuuint64_t)a.sp_in * 16, (cuuint64_t)plo * a.sp_in * 16, (cuuint64_t)a.sy_in * 16,
                                 (cuuint64_t)std::max<long long>(a.fs_in, 1) * 16};
  const cuuint32_t box[5] = {(cuuint32_t)(2 * XB), (cuuint32_t)plo, (cuuint32_t)phi, 1, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUtensorMap map;
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double2*>(a.src), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  const size_t smem = (size_t)XB * so3::RowLayout<N, XB>::SIZE * sizeof(double2) + 16 + (size_t)p->fft_pad * 1024;
  const bool bulkout = p->fft_bulkout < 0 ? N >= 512 : p->fft_bulkout != 0;
  auto k = bulkout ? (SIGN > 0 ? so3::fft_pass_tload_kernel<N, XB, +1, true> : so3::fft_pass_tload_kernel<N, XB, -1, true>)
                         : (SIGN > 0 ? so3::fft_pass_tload_kernel<N, XB, +1> : so3::fft_pass_tload_kernel<N, XB, -1>);
  SO3_CUDA(set_smem(k, smem));
  k<<<dim3(a.X / XB, a.Y, batch), XB * N / 16, smem, st>>>(map, a);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

// Persistent variants (fft_tma.cuh): `ctas` CTAs walk all tiles, two smem stages each.
template <int N, int SIGN>
int launch_fft_tstore_persist_t(const so3_plan_s* p, const so3::FftArgs& a, int batch, int ctas, cudaStream_t st) {
  constexpr int XB = 4;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return -1;
  const int plo = N < 256 ? N : 256, phi = N / plo;
  const cuuint64_t dims[5] = {(cuuint64_t)2 * a.X, (cuuint64_t)plo, (cuuint64_t)phi, (cuuint64_t)a.Y, (cuuint64_t)batch};
  const cuuint64_t strides[4] = {(cuuint64_t)a.sp_out * 16, (cuuint64_t)plo * a.sp_out * 16, (cuuint64_t)a.sy_out * 16,
                                 (cuuint64_t)std::max<long long>(a.fs_out, 1) * 16};
  const cuuint32_t box[5] = {(cuuint32_t)(2 * XB), (cuuint32_t)plo, (cuuint32_t)phi, 1, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUtensorMap map;
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, a.dst, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  const so3::TileSpace ts{a.X / XB, a.Y - ((a.skip_y >= 0 && a.skip_y < a.Y) ? 1 : 0), a.skip_y};
  const long long ntiles = (long long)ts.nxt * ts.ny * batch;
  const size_t smem = 2 * (size_t)XB * so3::RowLayout<N, XB>::SIZE * sizeof(double2) + 16;
  auto k = so3::fft_pass_tstore_persist_kernel<N, XB, SIGN>;
  SO3_CUDA(set_smem(k, smem));
  k<<<(unsigned)std::min<long long>(ctas, ntiles), XB * N / 16, smem, st>>>(map, a, ts, ntiles);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

template <int N, int SIGN>
int launch_fft_tload_persist_t(const so3_plan_s* p, const so3::FftArgs& a, int batch, int ctas, cudaStream_t st) {
  constexpr int XB = 4;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return -1;
  const int plo = N < 256 ? N : 256, phi = N / plo;
  const cuuint64_t dims[5] = {(cuuint64_t)2 * a.X, (cuuint64_t)plo, (cuuint64_t)phi, (cuuint64_t)a.Y, (cuuint64_t)batch};
  const cuuint64_t strides[4] = {(cuuint64_t)a.sp_in * 16, (cuuint64_t)plo * a.sp_in * 16, (cuuint64_t)a.sy_in * 16,
                                 (cuuint64_t)std::max<long long>(a.fs_in, 1) * 16};
  const cuuint32_t box[5] = {(cuuint32_t)(2 * XB), (cuuint32_t)plo, (cuuint32_t)phi, 1, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUtensorMap map;
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double2*>(a.src), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  const so3::TileSpace ts{a.X / XB, a.Y - ((a.skip_y >= 0 && a.skip_y < a.Y) ? 1 : 0), a.skip_y};
  const long long ntiles = (long long)ts.nxt * ts.ny * batch;
  const size_t smem = 2 * (size_t)XB * so3::RowLayout<N, XB>::SIZE * sizeof(double2) + 16;
  const bool bulkout = p->fft_bulkout < 0 ? N >= 512 : p->fft_bulkout != 0;
  auto k = bulkout ? so3::fft_pass_tload_persist_kernel<N, XB, SIGN, true> : so3::fft_pass_tload_persist_kernel<N, XB, SIGN, false>;
  SO3_CUDA(set_smem(k, smem));
  k<<<(unsigned)std::min<long long>(ctas, ntiles), XB * N / 16, smem, st>>>(map, a, ts, ntiles);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

int launch_fft_tma(const so3_plan_s* p, const so3::FftArgs& a, int sign, cudaStream_t st) {
  // plain-stride passes at 2B in {256, 512, 1024}: rows-in -> TMA chunk stores, chunks-in -> TMA chunk loads
  if (!p->fft_tma || p->fft_wide || a.tab_in || a.tab_out || a.X % 4) return -1;
  if (a.n != 256 && a.n != 512 && a.n != 1024) return -1;
  const int pc = p->fft_persist;
  if (pc > 0 && a.sp_in == 1 && a.sx_out == 1) {
    switch (a.n) {
      case 256: return sign > 0 ? launch_fft_tstore_persist_t<256, +1>(p, a, p->batch, pc, st) : launch_fft_tstore_persist_t<256, -1>(p, a, p->batch, pc, st);
      case 512: return sign > 0 ? launch_fft_tstore_persist_t<512, +1>(p, a, p->batch, pc, st) : launch_fft_tstore_persist_t<512, -1>(p, a, p->batch, pc, st);
      default: return sign > 0 ? launch_fft_tstore_persist_t<1024, +1>(p, a, p->batch, pc, st) : launch_fft_tstore_persist_t<1024, -1>(p, a, p->batch, pc, st);
    }
  }
  if (pc > 0 && a.sp_in != 1 && a.sx_in == 1 && a.sp_out == 1 && !a.weight) {
    switch (a.n) {
      case 256: return sign > 0 ? launch_fft_tload_persist_t<256, +1>(p, a, p->batch, pc, st) : launch_fft_tload_persist_t<256, -1>(p, a, p->batch, pc, st);
      case 512: return sign > 0 ? launch_fft_tload_persist_t<512, +1>(p, a, p->batch, pc, st) : launch_fft_tload_persist_t<512, -1>(p, a, p->batch, pc, st);
      default: return sign > 0 ? launch_fft_tload_persist_t<1024, +1>(p, a, p->batch, pc, st) : launch_fft_tload_persist_t<1024, -1>(p, a, p->batch, pc, st);
    }
  }
  if (a.sp_in == 1 && a.sx_out == 1) {
    switch (a.n) {
      case 256: return sign > 0 ? launch_fft_tstore_t<256, +1>(p, a, p->batch, st) : launch_fft_tstore_t<256, -1>(p, a, p->batch, st);
      case 512: return sign > 0 ? launch_fft_tstore_t<512, +1>(p, a, p->batch, st) : launch_fft_tstore_t<512, -1>(p, a, p->batch, st);
      default: return sign > 0 ? launch_fft_tstore_t<1024, +1>(p, a, p->batch, st) : launch_fft_tstore_t<1024, -1>(p, a, p->batch, st);
    }
  }
  if (a.sp_in != 1 && a.sx_in == 1 && a.sp_out == 1 && !a.weight) {
    switch (a.n) {
      case 256: return sign > 0 ? launch_fft_tload_t<256, +1>(p, a, p->batch, st) : launch_fft_tload_t<256, -1>(p, a, p->batch, st);
      case 512: return sign > 0 ? launch_fft_tload_t<512, +1>(p, a, p->batch, st) : launch_fft_tload_t<512, -1>(p, a, p->batch, st);
      default: return sign > 0 ? launch_fft_tload_t<1024, +1>(p, a, p->batch, st) : launch_fft_tload_t<1024, -1>(p, a, p->batch, st);
    }
  }
  return -1;
}

// The four passes (see fft.cuh).  n = 2B; all strides in complex128 units.
so3::FftArgs fft_pass_args(const so3_plan_s* p, int pass, const void* src, void* dst) {
  const long long n = p->n, n2 = n * n;
  so3::FftArgs a;
  a.n = p->n;
  a.nyq = p->B;
  a.X = p->n;
  a.Y = p->n;
  a.skip_y = -1;
  a.zero_p = -1;
  a.weight = 0;
  a.jbase = 0;
  a.src = static_cast<const double2*>(src);
  a.dst = static_cast<double2*>(dst);
  a.fs_in = a.fs_out = p->ngrid;
  a.tw = p->d_tw;
  a.w = p->d_w;
  a.tab_in = a.tab_out = nullptr;
  a.tabJ = 0;
  switch (pass) {
    case 0:   // K1a: grid[i][j][k] (x=i, y=j, p=k) -> T[j][m'][i]
      a.sx_in = n2; a.sy_in = n; a.sp_in = 1;
      a.sx_out = 1; a.sy_out = n2; a.sp_out = n;
      break;
    case 1:   // K1b: T[j][m'][i] (x=j, y=m', p=i) -> X[m'][m][j] * w_j
      a.sx_in = n2; a.sy_in = n; a.sp_in = 1;
      a.sx_out = 1; a.sy_out = n2; a.sp_out = n;
      a.skip_y = p->B;   // the DWT never reads m' = B
      a.weight = 1;
      break;
    case 2:   // K4a: X[m'][m][j] (x=j, y=m', p=m) -> T[j][m'][i]
      a.sx_in = 1; a.sy_in = n2; a.sp_in = n;
      a.sx_out = n2; a.sy_out = n; a.sp_out = 1;
      a.zero_p = p->B;   // row m = B of the spectrum is zero (soft.py:164)
      a.skip_y = p->B;   // column m' = B is zero: K4b reads it as zero instead
      break;
    default:  // K4b: T[j][m'][i] (x=i, y=j, p=m') -> grid[i][j][k]
      a.sx_in = 1; a.sy_in = n2; a.sp_in = n;
      a.sx_out = n2; a.sy_out = n; a.sp_out = 1;
      a.zero_p = p->B;
      break;
  }
  return a;
}

// Sharded passes on a beta slab [jbase, jbase + J): the pair-major side is the all-to-all
// buffer, rows [rank g][pairs_g][J] addressed through the global row table (fused pack/unpack).
so3::FftArgs shard_pass_args(const so3_plan_s* p, int pass, const void* src, void* dst) {
  const long long n = p->n, n2 = n * n, J = p->J;
  so3::FftArgs a = fft_pass_args(p, pass, src, dst);
  a.fs_in = a.fs_out = 0;
  a.jbase = p->jbase;
  switch (pass) {
    case 0:   // K1a: slab[i][jj][k] (x=i, y=jj, p=k) -> T[jj][m'][i]
      a.X = p->n; a.Y = p->J;
      a.sx_in = J * n; a.sy_in = n; a.sp_in = 1;
      a.sx_out = 1; a.sy_out = n2; a.sp_out = n;
      break;
    case 1:   // K1b: T[jj][m'][i] (x=jj, y=m', p=i) -> send rows [g][pairs_g][J] * w_j
      a.X = p->J; a.Y = p->n;
      a.sx_in = n2; a.sy_in = n; a.sp_in = 1;
      a.tab_out = p->d_row_global; a.tabJ = p->J;
      break;
    case 2:   // K4a: recv rows (x=jj, y=m', p=m) -> T[jj][m'][i]
      a.X = p->J; a.Y = p->n;
      a.tab_in = p->d_row_global; a.tabJ = p->J;
      a.sx_out = n2; a.sy_out = n; a.sp_out = 1;
      break;
    default:  // K4b: T[jj][m'][i] (x=i, y=jj, p=m') -> slab[i][jj][k]
      a.X = p->n; a.Y = p->J;
      a.sx_in = 1; a.sy_in = n2; a.sp_in = n;
      a.sx_out = J * n; a.sy_out = n; a.sp_out = 1;
      break;
  }
  return a;
}

int dwt_jt(int n) {
  // SIMT kernels: threads per cluster = ceil(n / JT) rounded up to a warp, <= 256
  if (n >= 128) return std::max(4, (n + 255) / 256);
  if (n >= 64) return 2;
  return 1;
}

int dwt_jw(int n) {
  // MMA kernels: beta indices per warp (warps per cluster = ceil(n / JW) <= 8)
  if (n >= 512) return 128;
  if (n >= 128) return 64;
  return 32;
}

// Warps straddle beta = pi/2 (rec_t's two table halves) unless B is a multiple of JW.
inline bool straddles(const so3::DwtArgs& a, int jw) { return a.B % jw != 0; }

template <int JW, int WPC, int FG = 1>
int launch_dwt_syn_wpc(const so3::DwtArgs& a, int split, unsigned ncl, int batch, cudaStream_t st) {
  using SM = so3::MmaSmem<JW>;
  const size_t smem = (size_t)WPC * 4 * SM::S * sizeof(double) + (size_t)t_knobs.dwt_pad * 1024;
  auto k = straddles(a, JW) ? so3::dwt_synthesis_mma_kernel<JW, WPC, (JW <= 64 ? 4 : 2), FG, true>
                            : so3::dwt_synthesis_mma_kernel<JW, WPC, (JW <= 64 ? 4 : 2), FG, false>;
  SO3_CUDA(set_smem(k, smem));
  k<<<dim3(ncl * split, batch / FG), WPC * 32, smem, st>>>(a, split);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}


template <int JW, int FG = 1>
int launch_dwt_mma_cta(const so3::DwtArgs& a, int n, unsigned ncl, int batch, cudaStream_t st, const double2* ck = nullptr) {
  using SM = so3::MmaSmem<JW>;
  const int warps = (n + JW - 1) / JW;
  const size_t smem = ((size_t)warps * 8 * SM::S + 2 * (size_t)warps * 512 * FG) * sizeof(double);
  auto k = straddles(a, JW) ? so3::dwt_analysis_mma_cta_kernel<JW, FG, 8, 1, true>
                            : so3::dwt_analysis_mma_cta_kernel<JW, FG, 8, 1, false>;
  SO3_CUDA(set_smem(k, smem));
  k<<<dim3(ncl, batch / FG), warps * 32, smem, st>>>(a, so3::SplitArgs{nullptr, 0, nullptr, ck});
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

template <int JW>
int launch_dwt_mma(bool analysis, const so3::DwtArgs& a, int n, unsigned ncl, int batch, cudaStream_t st,
                   const double2* ck = nullptr) {
  const int warps = (n + JW - 1) / JW;
  if (analysis) {
    if (warps > 8) return fail(SO3_ERR_INVALID, "bandwidth too large for the MMA DWT kernels");
    return launch_dwt_mma_cta<JW>(a, n, ncl, batch, st, ck);
  }
  if constexpr (JW == 32) {
    if (batch % 4 == 0) {   // batched small B: 4 functions share each recurrence
      if (warps % 2 == 0) return launch_dwt_syn_wpc<JW, 2, 4>(a, warps / 2, ncl, batch, st);
      return launch_dwt_syn_wpc<JW, 1, 4>(a, warps, ncl, batch, st);
    }
  }
  if (warps > 16) return fail(SO3_ERR_INVALID, "bandwidth too large for the MMA DWT kernels");
  if (warps >= 4 && warps % 4 == 0) return launch_dwt_syn_wpc<JW, 4>(a, warps / 4, ncl, batch, st);
  if (warps % 2 == 0) return launch_dwt_syn_wpc<JW, 2>(a, warps / 2, ncl, batch, st);
  return launch_dwt_syn_wpc<JW, 1>(a, warps, ncl, batch, st);
}

// Batched plans with 2B <= 64: analysis 4 functions per CTA (register operands), synthesis
// 8 functions per CTA (staged coefficients), see dwt_batch.cuh.
int launch_dwt_batch(bool analysis, const so3::DwtArgs& a, int n, unsigned ncl, int batch, const double* seeds,
                     cudaStream_t st) {
  if (analysis) {
    constexpr int FC = 4;
    auto k = so3::dwt_analysis_batch_reg_kernel<FC, 16>;
    k<<<dim3(ncl, (batch + FC - 1) / FC), FC * 32, so3::batch_analysis_smem(n), st>>>(a, batch, seeds);
  } else {
    constexpr int FC = 8;
    const size_t smem = so3::batch_synthesis_smem<FC>(n);
    auto k = so3::dwt_synthesis_batch_kernel<FC, 8>;
    SO3_CUDA(set_smem(k, smem));
    k<<<dim3(ncl, (batch + FC - 1) / FC), FC * 32, smem, st>>>(a, batch, seeds);
  }
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

// 2B = 1024 analysis with each cluster over two 4-warp CTAs.  The partial-sum scratch and the
// arrival counters are allocated (and the counters zeroed) at plan creation, or when the
// ana_split knob turns the split on, never on the launch path (graph capture, stream order).
int launch_dwt_ana_split(const so3_plan_s* p, so3::DwtArgs a, unsigned ncl, cudaStream_t st) {
  if (!p->d_pbuf || !p->d_pcnt) return fail(SO3_ERR_INVALID, "split analysis without its plan scratch");
  const so3::SplitArgs sp{p->d_pbuf, p->rc_entries * 8, p->d_pcnt, p->d_ck};
  constexpr int JW = 128;
  const int W = p->n / JW / 2;   // warps per half
  using SM = so3::MmaSmem<JW>;
  const size_t smem = ((size_t)W * 8 * SM::S + 2 * (size_t)W * 512) * sizeof(double) + (size_t)t_knobs.dwt_pad * 1024;
  auto k = so3::dwt_analysis_mma_cta_kernel<JW, 1, 8, 2>;
  SO3_CUDA(set_smem(k, smem));
  k<<<dim3(2 * ncl, 1), W * 32, smem, st>>>(a, sp);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

// Segment-parallel kernels (dwt_seg.cuh): B a multiple of 64, the plan's checkpoint table built.
bool seg_eligible(const so3_plan_s* p) { return p->B >= 64 && p->B % 64 == 0 && p->B <= 512; }
bool seg_applies(const so3_plan_s* p) {
  return p->dwt_seg && p->d_ck && p->dwt_variant != SO3_DWT_SIMT && seg_eligible(p);
}
// CTAs per cluster of the segment-parallel analysis: the fewest of {1, 2, 4} that leave at most
// seg_ana_w (<= 8) warps of 64 beta indices per CTA
int seg_ana_split(const so3_plan_s* p) {
  const int warps = p->n / so3::kSegBeta, wmax = std::max(1, std::min(8, p->seg_ana_w));
  for (int s : {1, 2, 4})
    if (warps % s == 0 && warps / s <= wmax) return s;
  return 0;
}

template <int SPLIT, int WT, int MINB>
int launch_seg_ana_cfg(const so3_plan_s* p, const so3::DwtArgs& a, unsigned ncl, int W, cudaStream_t st) {
  constexpr int TB = 8;
  auto k = so3::dwt_analysis_seg_kernel<16, SPLIT, TB, MINB, WT>;
  const size_t smem = ((size_t)2 * so3::kSegTabA + (size_t)2 * TB * W * 64) * sizeof(double2) + (size_t)t_knobs.dwt_pad * 1024;
  SO3_CUDA(set_smem(k, smem));
  const so3::SplitArgs sp{p->d_pbuf, p->rc_entries * 8, p->d_pcnt, p->d_ck};
  k<<<dim3(ncl * SPLIT, SPLIT > 1 ? 1 : p->batch), W * 32, smem, st>>>(a, sp, p->d_ck);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

int launch_dwt_seg_ana(const so3_plan_s* p, const so3::DwtArgs& a, unsigned ncl, cudaStream_t st) {
  const int split = seg_ana_split(p);
  const int W = split ? p->n / so3::kSegBeta / split : 0;
  if (split > 1 && (p->batch != 1 || !p->d_pbuf || !p->d_pcnt || p->pbuf_splits < split))
    return fail(SO3_ERR_INVALID, "segment-parallel split analysis without its plan scratch");
  switch (split) {
    case 1: return W <= 4 ? launch_seg_ana_cfg<1, 4, 2>(p, a, ncl, W, st) : launch_seg_ana_cfg<1, 8, 1>(p, a, ncl, W, st);
    case 2: return W <= 4 ? launch_seg_ana_cfg<2, 4, 2>(p, a, ncl, W, st) : launch_seg_ana_cfg<2, 8, 1>(p, a, ncl, W, st);
    case 4: return W <= 4 ? launch_seg_ana_cfg<4, 4, 2>(p, a, ncl, W, st) : launch_seg_ana_cfg<4, 8, 1>(p, a, ncl, W, st);
    default: return fail(SO3_ERR_INVALID, "segment-parallel analysis: no CTA shape for this bandwidth");
  }
}

// Persistent segment-parallel analysis (single-device plans, one function): CTAs of W <= 8 warps
// over W x 64 beta indices, `halves` passes per cluster, as many CTAs as fit the device.
template <int WT, int MINB, int TB>
int launch_seg_ana_persist(const so3_plan_s* p, const so3::DwtArgs& a, unsigned ncl, int W, int halves, cudaStream_t st) {
  auto k = W == WT ? so3::dwt_analysis_segp_kernel<16, TB, WT, MINB, true> : so3::dwt_analysis_segp_kernel<16, TB, WT, MINB, false>;
  const size_t smem = so3::segp_smem_bytes(W, TB) + (size_t)t_knobs.dwt_pad * 1024;
  SO3_CUDA(set_smem(k, smem));
  static std::mutex mu;
  static std::map<std::tuple<int, int, size_t>, int> ctas;   // (device, threads, smem) -> resident CTAs per device
  int dev = 0;
  cudaGetDevice(&dev);
  int grid = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_tuple(dev, W * 32 + 4096 * WT, smem);   // (W, WT) also selects the FULLW instantiation
    auto it = ctas.find(key);
    if (it == ctas.end()) {
      int per_sm = 0, sms = 0;
      SO3_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, W * 32, smem));
      SO3_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      it = ctas.emplace(key, std::max(1, per_sm) * sms).first;
    }
    grid = it->second;
  }
  const so3::SplitArgs sp{p->d_pbuf, p->rc_entries * 8, p->d_pcnt, p->d_ck};
  k<<<std::min<unsigned>(ncl, (unsigned)grid), W * 32, smem, st>>>(a, sp, p->d_ck, (int)ncl, halves);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

int launch_dwt_seg_anap(const so3_plan_s* p, const so3::DwtArgs& a, unsigned ncl, cudaStream_t st) {
  const int warps = p->n / so3::kSegBeta;
  int halves = warps > 8 ? 2 : 1;
  if (p->seg_ana_w == 4 && warps % 4 == 0) halves = warps / 4;   // two 4-warp CTAs per SM
  if (warps % halves) return fail(SO3_ERR_INVALID, "persistent analysis: odd warp count");
  const int W = warps / halves;
  if (halves > 1 && !p->d_pbuf) return fail(SO3_ERR_INVALID, "persistent analysis without its plan scratch");
  return W <= 4 ? launch_seg_ana_persist<4, 2, 2>(p, a, ncl, W, halves, st) : launch_seg_ana_persist<8, 1, 4>(p, a, ncl, W, halves, st);
}

int launch_dwt_seg_syn(const so3_plan_s* p, const so3::DwtArgs& a, unsigned ncl, cudaStream_t st) {
  const int warps = p->n / so3::kSegBeta;
  if (warps % 4 == 0) {
    auto k = so3::dwt_synthesis_seg_kernel<8, 4, 8, 3>;
    k<<<dim3(ncl * (warps / 4), p->batch), 128, 0, st>>>(a, warps / 4, p->d_ck);
  } else {
    auto k = so3::dwt_synthesis_seg_kernel<8, 2, 8, 4>;
    k<<<dim3(ncl * (warps / 2), p->batch), 64, 0, st>>>(a, warps / 2, p->d_ck);
  }
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

template <bool ANALYSIS>
int launch_dwt(const so3_plan_s* p, const void* spec, void* coef, int64_t c0, int64_t c1, cudaStream_t st,
               int64_t chunk_pairs = -1) {
  if (c0 < 0 || c1 > p->nclusters || c0 > c1)
    return fail(SO3_ERR_INVALID, "cluster range [" + std::to_string(c0) + ", " + std::to_string(c1) +
                                     ") outside [0, " + std::to_string(p->nclusters) + ")");
  if (c0 == c1) return SO3_OK;
  so3::DwtArgs a;
  a.B = p->B;
  a.n = p->n;
  a.bases = p->d_bases;
  a.lnorm = p->d_lnorm;
  a.xv = p->d_xv;
  a.logcs = p->d_logcs;
  a.spec = static_cast<const double2*>(spec);
  a.coef = static_cast<double2*>(coef);
  a.spec_fstride = p->ngrid;
  a.coef_fstride = p->ncoef;
  a.cluster0 = (int)c0;
  a.rc = p->d_rc;
  a.rc_off = p->d_rc_off;
  a.rowtab = p->sharded ? p->d_row_local : nullptr;
  a.J = p->sharded ? p->J : p->n;
  // sharded: spec is one chunk [h][pairs_chunk][J] of layout B (chunk_pairs; default = all pairs)
  a.slab_stride = p->sharded ? (long long)(chunk_pairs >= 0 ? chunk_pairs : p->pairs_rank) * p->J : 0;
  const unsigned ncl = (unsigned)(c1 - c0);
  if (p->dwt_variant != SO3_DWT_SIMT && p->dwt_batch && p->batch >= 2 && p->n <= 64 && p->d_seed)
    return launch_dwt_batch(ANALYSIS, a, p->n, ncl, p->batch, p->d_seed, st);
  if (ANALYSIS && seg_applies(p) && (p->dwt_seg & 4) && !p->sharded && p->batch == 1 && p->n / so3::kSegBeta >= 4)
    return launch_dwt_seg_anap(p, a, ncl, st);
  if (seg_applies(p) && (p->dwt_seg & (ANALYSIS ? 2 : 1)) && (!ANALYSIS || seg_ana_split(p) == 1 || p->batch == 1))
    return ANALYSIS ? launch_dwt_seg_ana(p, a, ncl, st) : launch_dwt_seg_syn(p, a, ncl, st);
  const int syn_jw = p->syn_jw ? p->syn_jw : (p->n >= 512 ? 64 : 0);   // 16 warps per SM (B=512: 32.8 vs 33.7 ms with JW = 128)
  if (p->dwt_variant != SO3_DWT_SIMT && !ANALYSIS && syn_jw && (p->n + syn_jw - 1) / syn_jw <= 16) {
    if (syn_jw == 64) return launch_dwt_mma<64>(false, a, p->n, ncl, p->batch, st);
    if (syn_jw == 32) return launch_dwt_mma<32>(false, a, p->n, ncl, p->batch, st);
  }
  if (ANALYSIS && p->ana_split && p->dwt_variant != SO3_DWT_SIMT && (p->n == 1024 || (p->n == 512 && p->ana_split > 1)) &&
      p->batch == 1)
    return launch_dwt_ana_split(p, a, ncl, st);
  if (p->dwt_variant != SO3_DWT_SIMT && (p->n + dwt_jw(p->n) - 1) / dwt_jw(p->n) <= 8) {
    switch (dwt_jw(p->n)) {
      case 128: return launch_dwt_mma<128>(ANALYSIS, a, p->n, ncl, p->batch, st, p->d_ck);
      case 64: return launch_dwt_mma<64>(ANALYSIS, a, p->n, ncl, p->batch, st, p->d_ck);
      default: return launch_dwt_mma<32>(ANALYSIS, a, p->n, ncl, p->batch, st);
    }
  }
  const int jt = dwt_jt(p->n);
  const int threads = std::min(256, ((p->n + jt - 1) / jt + 31) / 32 * 32);
  dim3 grid(ncl, p->batch);
  switch (jt) {
    case 1: if (ANALYSIS) so3::dwt_analysis_kernel<1><<<grid, threads, 0, st>>>(a); else so3::dwt_synthesis_kernel<1><<<grid, threads, 0, st>>>(a); break;
    case 2: if (ANALYSIS) so3::dwt_analysis_kernel<2><<<grid, threads, 0, st>>>(a); else so3::dwt_synthesis_kernel<2><<<grid, threads, 0, st>>>(a); break;
    case 4: if (ANALYSIS) so3::dwt_analysis_kernel<4><<<grid, threads, 0, st>>>(a); else so3::dwt_synthesis_kernel<4><<<grid, threads, 0, st>>>(a); break;
    case 8: if (ANALYSIS) so3::dwt_analysis_kernel<8><<<grid, threads, 0, st>>>(a); else so3::dwt_synthesis_kernel<8><<<grid, threads, 0, st>>>(a); break;
    default: return fail(SO3_ERR_INVALID, "bandwidth too large for the DWT kernels (JT > 8)");
  }
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

// Rows of d^l_{m,m'} for any pair: base recurrence + relation (sign, reflection).
__global__ void wigner_rows_kernel(int B, int n, int m, int mp, int bm, int bmp, int reflect, int sl, int par0,
                                   double2 lnorm, const double* xv, const double4* logcs, double* out) {
  const int L = bm;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double x = xv[j];
    const bool up = 2 * j >= n;
    double cur = so3::seed_value(bm, bmp, lnorm, logcs[j]);
    double prev = 0.0;
    const int jo = reflect ? n - 1 - j : j;
    for (int l = L; l < B; ++l) {
      const double s = ((sl * l + par0) & 1) ? -1.0 : 1.0;
      out[(long long)(l - L) * n + jo] = s * cur;
      if (l < B - 1) {
        const double3 k3 = so3::recurrence_coeffs(l, bm, bmp);
        const double tt = so3::rec_t(k3.x, k3.y, x, up);
        const double nx = fma(tt, cur, -k3.z * prev);
        prev = cur;
        cur = nx;
      }
    }
  }
}

}  // namespace

// ====================================================================== C ABI

extern "C" {

const char* so3_last_error(void) { return g_last_error.c_str(); }
const char* so3_version(void) { return "so3fft_b200 0.1.0 (sm_100a, fp64)"; }

int64_t so3_coeff_count(int b) { return b < 1 ? 0 : (int64_t)b * (4LL * b * b - 1) / 3; }
int64_t so3_grid_count(int b) { return b < 1 ? 0 : (int64_t)(2LL * b) * (2LL * b) * (2LL * b); }

int64_t so3_coeff_index(int l, int m, int mp, int b) {
  if (b < 1 || l < 0 || l >= b || std::abs(m) > l || std::abs(mp) > l) return -1;
  const int64_t L = l;
  return L * (4 * L * L - 1) / 3 + (int64_t)(m + l) * (2 * l + 1) + (mp + l);
}

int so3_quadrature_weights(int b, double* out) {
  if (!valid_bandwidth(b)) return fail(SO3_ERR_INVALID, "bandwidth must be in [1, 4096], got " + std::to_string(b));
  if (!out) return fail(SO3_ERR_INVALID, "null output");
  host_weights(b, out);
  return SO3_OK;
}

int so3_sample_angles(int b, double* alphas, double* betas) {
  if (!valid_bandwidth(b)) return fail(SO3_ERR_INVALID, "bandwidth must be in [1, 4096], got " + std::to_string(b));
  for (int i = 0; i < 2 * b; ++i) {
    if (alphas) alphas[i] = (double)i * 3.141592653589793 / (double)b;          // quadrature.py:60
    if (betas) betas[i] = (2.0 * i + 1.0) * 3.141592653589793 / (4.0 * b);     // quadrature.py:61
  }
  return SO3_OK;
}

int64_t so3_cluster_count(int b) { return b < 1 ? 0 : (int64_t)b * (b + 1) / 2; }

int so3_cluster_schedule(int b, int32_t* bases, int32_t* members) {
  if (!valid_bandwidth(b)) return fail(SO3_ERR_INVALID, "bandwidth must be in [1, 4096], got " + std::to_string(b));
  const auto cl = host_clusters(b);
  for (size_t i = 0; i < cl.size(); ++i) {
    if (bases) { bases[2 * i] = cl[i].m; bases[2 * i + 1] = cl[i].mp; }
    if (members) members[i] = cl[i].members;
  }
  return SO3_OK;
}

}  // extern "C"

namespace {

// partial sets the plan's analysis kernels need in d_pbuf (0: no split kernel applies)
int split_sets(const so3_plan_s* p) {
  int sets = 0;
  if (p->ana_split && p->batch == 1 && (p->n == 1024 || (p->n == 512 && p->ana_split > 1))) sets = 2;
  if ((p->dwt_seg & 2) && seg_eligible(p) && p->batch == 1) sets = std::max(sets, seg_ana_split(p) > 1 ? seg_ana_split(p) : 0);
  if ((p->dwt_seg & 4) && seg_eligible(p) && p->batch == 1 && !p->sharded && p->n / so3::kSegBeta > 4) sets = std::max(sets, 1);
  return sets;
}
bool split_applies(const so3_plan_s* p) { return split_sets(p) > 0; }

// Split-analysis scratch: per-half partial sums (2 x rc_entries x 8) and one arrival counter
// per cluster, allocated together (both or neither) and zeroed synchronously.
int ensure_split_scratch(so3_plan_s* p) {
  const int sets = split_sets(p);
  if (p->d_pbuf && p->d_pcnt && p->pbuf_splits >= sets) return SO3_OK;
  if (p->d_pbuf) {   // grow (knob change): the old scratch goes back first
    cudaDeviceSynchronize();
    p->bytes -= (int64_t)((size_t)p->pbuf_splits * std::max<long long>(p->rc_entries, 1) * 8 * sizeof(double2) +
                          (size_t)std::max<int64_t>(p->nclusters, 1) * sizeof(unsigned));
    cudaFree(p->d_pbuf);
    cudaFree(p->d_pcnt);
    p->d_pbuf = nullptr;
    p->d_pcnt = nullptr;
    p->pbuf_splits = 0;
  }
  const size_t pb = (size_t)sets * std::max<long long>(p->rc_entries, 1) * 8 * sizeof(double2);
  const size_t cb = (size_t)std::max<int64_t>(p->nclusters, 1) * sizeof(unsigned);
  double2* buf = nullptr;
  unsigned* cnt = nullptr;
  cudaError_t e = cudaMalloc((void**)&buf, pb);
  e = e ? e : cudaMalloc((void**)&cnt, cb);
  e = e ? e : cudaMemset(cnt, 0, cb);
  e = e ? e : cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaFree(buf);
    cudaFree(cnt);
    return fail(SO3_ERR_NOMEM, std::string("split-analysis scratch: ") + cudaGetErrorString(e));
  }
  p->d_pbuf = buf;
  p->d_pcnt = cnt;
  p->pbuf_splits = sets;
  p->bytes += (int64_t)(pb + cb);
  return SO3_OK;
}

// Checkpoint table of the segment-parallel DWT (dwt_seg.cuh): 8 recurrence states per (cluster,
// beta index), written by one pass of the recurrence.  Not enough memory: the plan keeps the
// dwt_mma.cuh kernels (dwt_seg off), it does not fail.
int ensure_checkpoints(so3_plan_s* p) {
  if (p->d_ck || !p->dwt_seg || !seg_eligible(p) || p->nclusters == 0) return SO3_OK;
  const size_t bytes = (size_t)p->nclusters * so3::kSegRows * p->n * sizeof(double2);
  double2* ck = nullptr;
  if (cudaMalloc((void**)&ck, bytes) != cudaSuccess) {
    cudaGetLastError();
    p->dwt_seg = 0;
    return SO3_OK;
  }
  so3::DwtArgs a{};
  a.B = p->B;
  a.n = p->n;
  a.bases = p->d_bases;
  a.lnorm = p->d_lnorm;
  a.xv = p->d_xv;
  a.logcs = p->d_logcs;
  a.rc = p->d_rc;
  a.rc_off = p->d_rc_off;
  so3::dwt_checkpoint_kernel<<<dim3((unsigned)p->nclusters, (p->n + 127) / 128), 128>>>(a, ck);
  cudaError_t e = cudaGetLastError();
  e = e ? e : cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaFree(ck);
    return fail(SO3_ERR_CUDA, std::string("checkpoint table: ") + cudaGetErrorString(e));
  }
  p->d_ck = ck;
  p->bytes += (int64_t)bytes;
  return SO3_OK;
}

// The rescaled recurrence table, per (cluster, degree l = m..B-1): (alpha_l, C+_l, mu_l) with
// d^l = mu_l e^l, e^{l+1} = t_l e^l - e^{l-1}, t_l = alpha_l (x - shift_l) (rec_t), mu_m = 1,
// mu_{l+1} = c_l mu_{l-1} (a_m mu_m at l = m), alpha_l = a_l mu_l / mu_{l+1}, C+_l = alpha_l (1 -
// shift_l), from the reference's coefficients (wigner.py:165-174).  Evaluated in long double
// (64-bit mantissa) and rounded once per entry, so mu_l carries no fp64 drift along l; split over
// the host's cores (67 M entries at B = 512).
std::vector<double> host_rc_table(int b, const std::vector<Cluster>& cl, const std::vector<long long>& off,
                                  size_t entries) {
  std::vector<double> rc(3 * std::max<size_t>(entries, 1), 0.0);
  const unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (size_t i = t; i < cl.size(); i += nt) {
        const long double m = cl[i].m, mp = cl[i].mp;
        double* dst = rc.data() + 3 * off[i];
        long double mu_prev = 0.0L, mu = 1.0L;
        for (int l = cl[i].m; l < b; ++l) {
          long double alpha = 0.0L, cplus = 0.0L, mu_next = 0.0L;
          if (l < b - 1) {
            const long double lp = l + 1.0L, dl = l;
            const long double denom = sqrtl((lp * lp - m * m) * (lp * lp - mp * mp));
            const long double a = lp * (2.0L * dl + 1.0L) / denom;
            long double c = 0.0L, one_minus_shift = 1.0L;
            if (l > 0) {
              c = lp * sqrtl((dl * dl - m * m) * (dl * dl - mp * mp)) / (dl * denom);
              one_minus_shift = (dl * lp - m * mp) / (dl * lp);
            }
            mu_next = l == cl[i].m ? a * mu : c * mu_prev;
            alpha = a * mu / mu_next;
            cplus = alpha * one_minus_shift;
          }
          dst[3 * (l - cl[i].m)] = (double)alpha;
          dst[3 * (l - cl[i].m) + 1] = (double)cplus;
          dst[3 * (l - cl[i].m) + 2] = (double)mu;
          mu_prev = mu;
          mu = mu_next;
        }
      }
    });
  for (auto& x : th) x.join();
  return rc;
}

// Tables and buffers of a plan over the cluster list `cl` (all clusters, or one rank's group).
int build_plan(so3_plan_s* p, const std::vector<Cluster>& cl) {
  const int b = p->B, n = p->n, batch = p->batch;
  std::vector<double> w(n), xv(n);
  std::vector<double4> logcs(n);
  std::vector<double2> tw(n);
  host_weights(b, w.data());
  for (int j = 0; j < n; ++j) {
    const long double beta = (2.0L * j + 1.0L) * kPi / (4.0L * b);
    // rec_t's v_j: cos(beta) - 1 = -2 sin^2(beta/2) below pi/2, cos(beta) + 1 = 2 cos^2(beta/2) above
    const long double sh = sinl(0.5L * beta), ch = cosl(0.5L * beta);
    xv[j] = 2 * j < n ? (double)(-2.0L * sh * sh) : (double)(2.0L * ch * ch);
    double a0, a1, a2, a3;
    split_ld(logl(cosl(0.5L * beta)), &a0, &a1);
    split_ld(logl(sinl(0.5L * beta)), &a2, &a3);
    logcs[j] = make_double4(a0, a1, a2, a3);
  }
  for (int k = 0; k < n; ++k) {
    const long double th = 2.0L * kPi * k / n;
    tw[k] = make_double2((double)cosl(th), (double)sinl(th));
  }
  p->nclusters = (int64_t)cl.size();
  const size_t ncl = std::max<size_t>(cl.size(), 1);
  std::vector<long long> rc_off(ncl, 0);
  long long rc_entries = 0;
  for (size_t i = 0; i < cl.size(); ++i) {
    rc_off[i] = rc_entries;
    // one (alpha, C+, mu) per degree; an even count, so every cluster's table starts 16-byte
    // aligned and is a multiple of 16 bytes (1-D bulk copies, dwt_seg.cuh)
    rc_entries += (b - cl[i].m + 1) & ~1;
  }
  p->rc_entries = rc_entries;
  rc_entries = std::max(rc_entries, 1LL);
  std::vector<int2> bases(ncl, make_int2(0, 0));
  std::vector<double2> lnorm(ncl, make_double2(0.0, 0.0));
  for (size_t i = 0; i < cl.size(); ++i) {
    const int m = cl[i].m, mp = cl[i].mp;
    bases[i] = make_int2(m, mp);
    // log sqrt((2m)! / ((m+m')! (m-m')!))   (wigner.py:124)
    const long double ln = 0.5L * (lgammal(2.0L * m + 1) - lgammal((long double)m + mp + 1) - lgammal((long double)m - mp + 1));
    double hi, lo;
    split_ld(ln, &hi, &lo);
    lnorm[i] = make_double2(hi, lo);
  }
  // slab size of the spectrum buffers: whole grid, or this rank's pair rows x 2B
  const size_t spec_elems = p->sharded ? (size_t)std::max<int64_t>(p->pairs_rank, 1) * n : (size_t)p->ngrid;
  const size_t slab_elems = p->sharded ? (size_t)n * p->J * n : (size_t)p->ngrid;

#define PLAN_ALLOC(ptr, count)                                                                    \
  do {                                                                                            \
    size_t _bytes = (size_t)(count) * sizeof(*(ptr));                                             \
    cudaError_t _e = cudaMalloc((void**)&(ptr), _bytes);                                          \
    if (_e != cudaSuccess) return fail(SO3_ERR_NOMEM, std::string("cudaMalloc(") +               \
                                 std::to_string(_bytes) + "): " + cudaGetErrorString(_e));        \
    p->bytes += (int64_t)_bytes;                                                                  \
  } while (0)
  PLAN_ALLOC(p->d_bases, ncl);
  PLAN_ALLOC(p->d_lnorm, ncl);
  PLAN_ALLOC(p->d_xv, n);
  PLAN_ALLOC(p->d_logcs, n);
  PLAN_ALLOC(p->d_w, n);
  PLAN_ALLOC(p->d_tw, n);
  PLAN_ALLOC(p->d_scratch, slab_elems * batch);
  PLAN_ALLOC(p->d_spec, spec_elems * batch);
  PLAN_ALLOC(p->d_rc, (size_t)3 * rc_entries);
  PLAN_ALLOC(p->d_rc_off, ncl);
#undef PLAN_ALLOC
  cudaError_t e = cudaSuccess;
  e = e ? e : cudaMemcpy(p->d_bases, bases.data(), ncl * sizeof(int2), cudaMemcpyHostToDevice);
  e = e ? e : cudaMemcpy(p->d_lnorm, lnorm.data(), ncl * sizeof(double2), cudaMemcpyHostToDevice);
  e = e ? e : cudaMemcpy(p->d_xv, xv.data(), n * sizeof(double), cudaMemcpyHostToDevice);
  e = e ? e : cudaMemcpy(p->d_logcs, logcs.data(), n * sizeof(double4), cudaMemcpyHostToDevice);
  e = e ? e : cudaMemcpy(p->d_w, w.data(), n * sizeof(double), cudaMemcpyHostToDevice);
  e = e ? e : cudaMemcpy(p->d_tw, tw.data(), n * sizeof(double2), cudaMemcpyHostToDevice);
  e = e ? e : cudaMemcpy(p->d_rc_off, rc_off.data(), ncl * sizeof(long long), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !cl.empty()) {
    const std::vector<double> rc = host_rc_table(b, cl, rc_off, (size_t)rc_entries);
    e = cudaMemcpy(p->d_rc, rc.data(), rc.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  e = e ? e : cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(SO3_ERR_CUDA, std::string("plan upload: ") + cudaGetErrorString(e));
  if (p->batch >= 2 && n <= 64 && !cl.empty()) {   // seed table of the batched kernels (dwt_batch.cuh)
    const size_t bytes = cl.size() * n * sizeof(double);
    if (cudaMalloc((void**)&p->d_seed, bytes) != cudaSuccess) return fail(SO3_ERR_NOMEM, "seed table");
    so3::DwtArgs sa{};
    sa.B = b;
    sa.n = n;
    sa.bases = p->d_bases;
    sa.lnorm = p->d_lnorm;
    sa.logcs = p->d_logcs;
    so3::dwt_seed_table_kernel<<<dim3((unsigned)cl.size(), (n + 63) / 64), 64>>>(sa, p->d_seed);
    cudaError_t se = cudaGetLastError();
    se = se ? se : cudaDeviceSynchronize();
    if (se != cudaSuccess) return fail(SO3_ERR_CUDA, std::string("seed table: ") + cudaGetErrorString(se));
    p->bytes += (int64_t)bytes;
  }
  if (int rc = ensure_checkpoints(p)) return rc;
  if (split_applies(p)) return ensure_split_scratch(p);
  return SO3_OK;
}

so3_plan_s* new_plan(int b, int batch) {
  auto* p = new so3_plan_s();
  p->B = b;
  p->n = 2 * b;
  p->batch = batch;
  p->ncoef = so3_coeff_count(b);
  p->ngrid = so3_grid_count(b);
  p->J = p->n;
  // 2B / 64 > 8 (B = 320 .. 512): the persistent segment analysis (two passes per cluster) is the
  // default: 31.9 ms at B = 512 against 33.9 ms for the split dwt_mma.cuh analysis, 9.2 against
  // 10.0 ms at B = 320 (no split shape there); at B <= 256 the dwt_mma.cuh analysis is as fast
  if (b % 64 == 0 && b > 256 && b <= 512 && batch == 1) p->dwt_seg |= 4;
  cudaGetDevice(&p->device);
  return p;
}

}  // namespace

extern "C" {

int so3_plan_create(int b, int batch, so3_plan_t* out) {
  if (!out) return fail(SO3_ERR_INVALID, "null plan output");
  *out = nullptr;
  if (!valid_bandwidth(b)) return fail(SO3_ERR_INVALID, "bandwidth must be in [1, 4096], got " + std::to_string(b));
  if (batch < 1) return fail(SO3_ERR_INVALID, "batch must be >= 1, got " + std::to_string(batch));
  if (b > kMaxBandwidth)
    return fail(SO3_ERR_INVALID, "bandwidth must be <= " + std::to_string(kMaxBandwidth) +
                                     " (the DWT kernels span at most 2B = 1024 beta indices per cluster), got " +
                                     std::to_string(b));
  so3_plan_s* p = new_plan(b, batch);
  const int rc = build_plan(p, host_clusters(b));
  if (rc) { so3_plan_destroy(p); return rc; }
  *out = p;
  return SO3_OK;
}

int so3_shard_plan_create(int b, int world, int rank, so3_plan_t* out) {
  return so3_shard_plan_create_chunked(b, world, rank, 1, out);
}

int so3_shard_plan_create_chunked(int b, int world, int rank, int chunks, so3_plan_t* out) {
  if (!out) return fail(SO3_ERR_INVALID, "null plan output");
  *out = nullptr;
  if (!valid_bandwidth(b) || b > kMaxBandwidth)
    return fail(SO3_ERR_INVALID, "bandwidth must be in [1, " + std::to_string(kMaxBandwidth) + "], got " + std::to_string(b));
  if (world < 1 || rank < 0 || rank >= world) return fail(SO3_ERR_INVALID, "rank outside [0, world)");
  if ((2 * b) % world) return fail(SO3_ERR_INVALID, "2B must be divisible by the number of ranks");
  if (chunks < 1 || chunks > 64) return fail(SO3_ERR_INVALID, "chunks must be in [1, 64]");
  so3_plan_s* p = new_plan(b, 1);
  p->sharded = 1;
  p->world = world;
  p->rank = rank;
  p->J = p->n / world;
  p->jbase = rank * p->J;
  p->chunks = chunks;
  const int n = p->n;
  const auto all = host_clusters(b);
  const auto owner = shard_owner(all, b, world);
  const auto chunk_of = shard_chunks(all, owner, b, world, chunks);
  // pairs per (chunk, rank); layout A rows are [q][g][pairs_{g,q}], layout B rows [q][h][pairs_{rank,q}]
  std::vector<int64_t> cnt((size_t)chunks * world, 0);
  p->pairs_of.assign(world, 0);
  for (size_t i = 0; i < all.size(); ++i) {
    cnt[(size_t)chunk_of[i] * world + owner[i]] += all[i].members;
    p->pairs_of[owner[i]] += all[i].members;
  }
  std::vector<int64_t> base_a((size_t)chunks * world + 1, 0);
  for (size_t k = 0; k < cnt.size(); ++k) base_a[k + 1] = base_a[k] + cnt[k];
  std::vector<int64_t> next((size_t)chunks * world, 0);
  std::vector<int> row_global((size_t)n * n, -1), row_local((size_t)n * n, -1);
  std::vector<Cluster> mine;
  p->chunk_cl.assign(chunks + 1, 0);
  p->chunk_pairs.assign(chunks, 0);
  for (size_t i = 0; i < all.size(); ++i) {
    const int r = owner[i], q = chunk_of[i];
    const size_t k = (size_t)q * world + r;
    if (r == rank) {
      mine.push_back(all[i]);
      p->chunk_cl[q + 1] = (int64_t)mine.size();
      p->chunk_pairs[q] += all[i].members;
    }
    for (const auto& pr : cluster_pairs(all[i].m, all[i].mp)) {
      const int bm = ((pr.first % n) + n) % n, bmp = ((pr.second % n) + n) % n;
      const size_t idx = (size_t)bmp * n + bm;
      row_global[idx] = (int)(base_a[k] + next[k]);
      if (r == rank) row_local[idx] = (int)next[k];
      ++next[k];
    }
  }
  for (int q = 1; q <= chunks; ++q) p->chunk_cl[q] = std::max(p->chunk_cl[q], p->chunk_cl[q - 1]);
  p->chunk_off.assign(chunks + 1, 0);
  for (int q = 0; q < chunks; ++q) p->chunk_off[q + 1] = p->chunk_off[q] + p->chunk_pairs[q];
  p->pairs_rank = p->pairs_of[rank];
  // Self-block elision: the FFT passes address ONE exchange buffer holding layout A (rows
  // [0, rows_A)) followed by layout B.  This rank's own pairs live in layout B only (block
  // h = rank of each chunk), so the forward FFT writes them where the DWT reads them and the
  // inverse FFT reads them where the DWT wrote them: the all-to-all carries the other ranks'
  // blocks only.
  const int64_t rows_a = base_a.back();
  for (size_t i = 0; i < all.size(); ++i) {
    if (owner[i] != rank) continue;
    const int q = chunk_of[i];
    for (const auto& pr : cluster_pairs(all[i].m, all[i].mp)) {
      const int bm = ((pr.first % n) + n) % n, bmp = ((pr.second % n) + n) % n;
      const size_t idx = (size_t)bmp * n + bm;
      row_global[idx] = (int)(rows_a + (int64_t)world * p->chunk_off[q] + (int64_t)rank * p->chunk_pairs[q] +
                              row_local[idx]);
    }
  }
  int rc = build_plan(p, mine);
  if (rc) { so3_plan_destroy(p); return rc; }
  cudaError_t e = cudaMalloc((void**)&p->d_row_global, row_global.size() * sizeof(int));
  e = e ? e : cudaMalloc((void**)&p->d_row_local, row_local.size() * sizeof(int));
  e = e ? e : cudaMemcpy(p->d_row_global, row_global.data(), row_global.size() * sizeof(int), cudaMemcpyHostToDevice);
  e = e ? e : cudaMemcpy(p->d_row_local, row_local.data(), row_local.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { so3_plan_destroy(p); return fail(SO3_ERR_NOMEM, std::string("shard tables: ") + cudaGetErrorString(e)); }
  p->bytes += (int64_t)(2 * row_global.size() * sizeof(int));
  *out = p;
  return SO3_OK;
}

int so3_shard_chunk_pairs(int b, int world, int chunks, int64_t* pairs) {
  if (!valid_bandwidth(b) || world < 1 || chunks < 1 || chunks > 64 || !pairs) return fail(SO3_ERR_INVALID, "bad arguments");
  const auto all = host_clusters(b);
  const auto owner = shard_owner(all, b, world);
  const auto chunk_of = shard_chunks(all, owner, b, world, chunks);
  for (int k = 0; k < chunks * world; ++k) pairs[k] = 0;
  for (size_t i = 0; i < all.size(); ++i) pairs[(size_t)chunk_of[i] * world + owner[i]] += all[i].members;
  return SO3_OK;
}

int64_t so3_shard_chunks(so3_plan_t p) { return p ? p->chunks : 0; }

int so3_shard_pair_counts(int b, int world, int64_t* pairs_per_rank) {
  if (!valid_bandwidth(b) || world < 1 || !pairs_per_rank) return fail(SO3_ERR_INVALID, "bad arguments");
  const auto all = host_clusters(b);
  const auto owner = shard_owner(all, b, world);
  for (int r = 0; r < world; ++r) pairs_per_rank[r] = 0;
  for (size_t i = 0; i < all.size(); ++i) pairs_per_rank[owner[i]] += all[i].members;
  return SO3_OK;
}

int so3_shard_cluster_owner(int b, int world, int32_t* owner_out) {
  if (!valid_bandwidth(b) || world < 1 || !owner_out) return fail(SO3_ERR_INVALID, "bad arguments");
  const auto all = host_clusters(b);
  const auto owner = shard_owner(all, b, world);
  for (size_t i = 0; i < all.size(); ++i) owner_out[i] = owner[i];
  return SO3_OK;
}

int so3_shard_pair_list(int b, int world, int rank, int32_t* pairs_out) {
  if (!valid_bandwidth(b) || world < 1 || rank < 0 || rank >= world || !pairs_out)
    return fail(SO3_ERR_INVALID, "bad arguments");
  const auto all = host_clusters(b);
  const auto owner = shard_owner(all, b, world);
  size_t k = 0;
  for (size_t i = 0; i < all.size(); ++i) {
    if (owner[i] != rank) continue;
    for (const auto& pr : cluster_pairs(all[i].m, all[i].mp)) {
      pairs_out[2 * k] = pr.first;
      pairs_out[2 * k + 1] = pr.second;
      ++k;
    }
  }
  return SO3_OK;
}

int64_t so3_shard_slab_width(so3_plan_t p) { return p ? p->J : 0; }
int64_t so3_shard_rank_pairs(so3_plan_t p) { return p ? p->pairs_rank : 0; }

void so3_plan_destroy(so3_plan_t p) {
  if (!p) return;
  cudaFree(p->d_bases);
  cudaFree(p->d_lnorm);
  cudaFree(p->d_xv);
  cudaFree(p->d_logcs);
  cudaFree(p->d_w);
  cudaFree(p->d_tw);
  cudaFree(p->d_scratch);
  cudaFree(p->d_spec);
  cudaFree(p->d_rc);
  cudaFree(p->d_rc_off);
  cudaFree(p->d_pbuf);
  cudaFree(p->d_pcnt);
  cudaFree(p->d_ck);
  cudaFree(p->d_seed);
  cudaFree(p->d_row_global);
  cudaFree(p->d_row_local);
  cudaFree(p->d_grid_stage);
  cudaFree(p->d_coef_stage);
  p->host_stage.release();
  delete p;
}

int so3_plan_bandwidth(so3_plan_t p) { return p ? p->B : 0; }
int so3_plan_batch(so3_plan_t p) { return p ? p->batch : 0; }
int so3_plan_device(so3_plan_t p) { return p ? p->device : -1; }
int64_t so3_plan_device_bytes(so3_plan_t p) { return p ? p->bytes : 0; }
void* so3_plan_scratch(so3_plan_t p) { return p ? p->d_spec : nullptr; }

int so3_plan_set_knob(so3_plan_t p, const char* name, int value) {
  if (!p || !name) return fail(SO3_ERR_INVALID, "null plan or knob name");
  const std::string k(name);
  if (k == "dwt_variant") return so3_plan_set_dwt_variant(p, value);
  if (k == "syn_jw") { p->syn_jw = value; return SO3_OK; }
  if (k == "ana_split") {
    const int old = p->ana_split;
    p->ana_split = value;
    if (split_applies(p)) {
      if (int rc = ensure_split_scratch(p)) { p->ana_split = old; return rc; }
    }
    return SO3_OK;
  }
  if (k == "dwt_seg" || k == "seg_ana_w") {
    if (k == "seg_ana_w" && value != 4 && value != 8) return fail(SO3_ERR_INVALID, "seg_ana_w must be 4 or 8");
    int& field = k == "dwt_seg" ? p->dwt_seg : p->seg_ana_w;
    const int old = field;
    field = value;
    int rc = ensure_checkpoints(p);
    if (!rc && split_applies(p)) rc = ensure_split_scratch(p);
    if (rc) field = old;
    return rc;
  }
  if (k == "fft_xb") { p->fft_wide = value; return SO3_OK; }
  if (k == "dwt_batch") { p->dwt_batch = value; return SO3_OK; }
  if (k == "fft_fused") { p->fft_fused = value; return SO3_OK; }
  if (k == "fft_tma") { p->fft_tma = value; return SO3_OK; }
  if (k == "fft_tab_loop") { p->fft_tab_loop = value; return SO3_OK; }
  if (k == "fft_tab_tma") { p->fft_tab_tma = value; return SO3_OK; }
  if (k == "fft_bulkin") { p->fft_bulkin = value; return SO3_OK; }
  if (k == "fft_bulkout") { p->fft_bulkout = value; return SO3_OK; }
  if (k == "carveout") {   // see LaunchKnobs
    if (value < -1 || value > 100) return fail(SO3_ERR_INVALID, "carveout must be -1 or a percentage in [0, 100]");
    p->carveout = value;
    return SO3_OK;
  }
  if (k == "dwt_pad") {   // see LaunchKnobs
    if (value < 0 || value > 150) return fail(SO3_ERR_INVALID, "dwt_pad must be in [0, 150] KB");
    p->dwt_pad = value;
    return SO3_OK;
  }
  if (k == "fft_persist") {
    if (value < 0 || value > 65536) return fail(SO3_ERR_INVALID, "fft_persist must be in [0, 65536] CTAs");
    p->fft_persist = value;
    return SO3_OK;
  }
  if (k == "fft_pad") {
    if (value < 0 || value > 150) return fail(SO3_ERR_INVALID, "fft_pad must be in [0, 150] KB");
    p->fft_pad = value;
    return SO3_OK;
  }
  return fail(SO3_ERR_INVALID, "unknown knob " + k);
}

int so3_plan_set_dwt_variant(so3_plan_t p, int variant) {
  if (!p) return fail(SO3_ERR_INVALID, "null plan");
  if (variant != SO3_DWT_MMA && variant != SO3_DWT_SIMT) return fail(SO3_ERR_INVALID, "unknown DWT variant");
  p->dwt_variant = variant;
  return SO3_OK;
}

#define CHECK_PLAN(p) \
  if (!(p)) return fail(SO3_ERR_INVALID, "null plan")
#define CHECK_PTR(x) \
  if (!(x)) return fail(SO3_ERR_INVALID, "null buffer: " #x)

int so3_fft_analysis(so3_plan_t p, const void* samples, void* spectrum, void* stream) {
  CHECK_PLAN(p); CHECK_PTR(samples); CHECK_PTR(spectrum);
  KnobScope knobs(p);
  if (samples == spectrum || spectrum == p->d_scratch)
    return fail(SO3_ERR_INVALID, "fft_analysis: spectrum must not alias the samples or the plan scratch");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = launch_fft2d(p, +1, samples, spectrum, st); rc >= 0) return rc;
  for (int pass = 0; pass < 2; ++pass) {
    const so3::FftArgs a = pass == 0 ? fft_pass_args(p, 0, samples, p->d_scratch) : fft_pass_args(p, 1, p->d_scratch, spectrum);
    int rc = launch_fft_tma(p, a, +1, st);
    if (rc < 0) rc = launch_fft(p, a, +1, p->batch, st);
    if (rc) return rc;
  }
  return SO3_OK;
}

int so3_fft_synthesis(so3_plan_t p, void* spectrum, void* samples, void* stream) {
  CHECK_PLAN(p); CHECK_PTR(samples); CHECK_PTR(spectrum);
  KnobScope knobs(p);
  if (samples == spectrum || spectrum == p->d_scratch || samples == p->d_scratch)
    return fail(SO3_ERR_INVALID, "fft_synthesis: buffers must not alias each other or the plan scratch");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = launch_fft2d(p, -1, spectrum, samples, st); rc >= 0) return rc;
  for (int pass = 2; pass < 4; ++pass) {
    const so3::FftArgs a = pass == 2 ? fft_pass_args(p, 2, spectrum, p->d_scratch) : fft_pass_args(p, 3, p->d_scratch, samples);
    int rc = launch_fft_tma(p, a, -1, st);
    if (rc < 0) rc = launch_fft(p, a, -1, p->batch, st);
    if (rc) return rc;
  }
  return SO3_OK;
}

int so3_dwt_analysis(so3_plan_t p, const void* spectrum, void* coeffs, int64_t c0, int64_t c1, void* stream) {
  CHECK_PLAN(p); CHECK_PTR(spectrum); CHECK_PTR(coeffs);
  KnobScope knobs(p);
  return launch_dwt<true>(p, spectrum, coeffs, c0, c1, static_cast<cudaStream_t>(stream));
}

int so3_dwt_synthesis(so3_plan_t p, const void* coeffs, void* spectrum, int64_t c0, int64_t c1, void* stream) {
  CHECK_PLAN(p); CHECK_PTR(spectrum); CHECK_PTR(coeffs);
  KnobScope knobs(p);
  // the synthesis kernel writes the spectrum; DwtArgs carries it as `spec` and reads `coef`
  return launch_dwt<false>(p, spectrum, const_cast<void*>(coeffs), c0, c1, static_cast<cudaStream_t>(stream));
}

int so3_fsoft(so3_plan_t p, const void* samples, void* coeffs, void* stream) {
  CHECK_PLAN(p); CHECK_PTR(samples); CHECK_PTR(coeffs);
  int rc = so3_fft_analysis(p, samples, p->d_spec, stream);
  if (rc) return rc;
  return so3_dwt_analysis(p, p->d_spec, coeffs, 0, p->nclusters, stream);
}

int so3_ifsoft(so3_plan_t p, const void* coeffs, void* samples, void* stream) {
  CHECK_PLAN(p); CHECK_PTR(samples); CHECK_PTR(coeffs);
  int rc = so3_dwt_synthesis(p, coeffs, p->d_spec, 0, p->nclusters, stream);
  if (rc) return rc;
  return so3_fft_synthesis(p, p->d_spec, samples, stream);
}

static int ensure_stage(so3_plan_t p) {
  if (!p->d_grid_stage) {
    cudaError_t e = cudaMalloc((void**)&p->d_grid_stage, (size_t)p->ngrid * p->batch * sizeof(double2));
    if (e != cudaSuccess) return fail(SO3_ERR_NOMEM, std::string("staging grid: ") + cudaGetErrorString(e));
    p->bytes += p->ngrid * p->batch * (int64_t)sizeof(double2);
  }
  if (!p->d_coef_stage) {
    cudaError_t e = cudaMalloc((void**)&p->d_coef_stage, (size_t)p->ncoef * p->batch * sizeof(double2));
    if (e != cudaSuccess) return fail(SO3_ERR_NOMEM, std::string("staging coefficients: ") + cudaGetErrorString(e));
    p->bytes += p->ncoef * p->batch * (int64_t)sizeof(double2);
  }
  return SO3_OK;
}

// Host <-> device copy of a host-buffer entry point: pinned buffers (and small pageable ones)
// go straight to the DMA engines on the caller's stream; large pageable buffers through the
// plan's multi-threaded pinned staging (hostio.cuh), ordered after the stream's earlier work.
static int host_copy(so3_plan_t p, void* dev, void* host, size_t bytes, bool to_device, cudaStream_t st) {
  constexpr size_t kDirect = size_t(64) << 20;
  if (bytes < kDirect || so3host::is_pinned(host)) {
    SO3_CUDA(cudaMemcpyAsync(to_device ? dev : host, to_device ? (const void*)host : (const void*)dev, bytes,
                             to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, st));
    return SO3_OK;
  }
  if (!p->host_stage.ready()) {
    const cudaError_t e = p->host_stage.init(p->device, so3host::default_workers(), so3host::kChunk);
    if (e != cudaSuccess) return fail(SO3_ERR_NOMEM, std::string("pinned staging: ") + cudaGetErrorString(e));
  }
  SO3_CUDA(cudaStreamSynchronize(st));
  SO3_CUDA(to_device ? p->host_stage.run<+1>(p->device, dev, host, bytes)
                     : p->host_stage.run<-1>(p->device, dev, host, bytes));
  return SO3_OK;
}

int so3_fsoft_host(so3_plan_t p, const void* samples_host, void* coeffs_host, void* stream) {
  CHECK_PLAN(p); CHECK_PTR(samples_host); CHECK_PTR(coeffs_host);
  int rc = ensure_stage(p);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = host_copy(p, p->d_grid_stage, const_cast<void*>(samples_host), (size_t)p->ngrid * p->batch * sizeof(double2),
                 true, st);
  if (rc) return rc;
  rc = so3_fsoft(p, p->d_grid_stage, p->d_coef_stage, stream);
  if (rc) return rc;
  rc = host_copy(p, p->d_coef_stage, coeffs_host, (size_t)p->ncoef * p->batch * sizeof(double2), false, st);
  if (rc) return rc;
  SO3_CUDA(cudaStreamSynchronize(st));
  return SO3_OK;
}

int so3_ifsoft_host(so3_plan_t p, const void* coeffs_host, void* samples_host, void* stream) {
  CHECK_PLAN(p); CHECK_PTR(samples_host); CHECK_PTR(coeffs_host);
  int rc = ensure_stage(p);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = host_copy(p, p->d_coef_stage, const_cast<void*>(coeffs_host), (size_t)p->ncoef * p->batch * sizeof(double2),
                 true, st);
  if (rc) return rc;
  rc = so3_ifsoft(p, p->d_coef_stage, p->d_grid_stage, stream);
  if (rc) return rc;
  rc = host_copy(p, p->d_grid_stage, samples_host, (size_t)p->ngrid * p->batch * sizeof(double2), false, st);
  if (rc) return rc;
  SO3_CUDA(cudaStreamSynchronize(st));
  return SO3_OK;
}

#define CHECK_SHARD(p) \
  if (!(p)->sharded) return fail(SO3_ERR_INVALID, "not a sharded plan (so3_shard_plan_create)")

int so3_shard_fft_analysis(so3_plan_t p, const void* slab, void* send, void* stream) {
  CHECK_PLAN(p); CHECK_SHARD(p); CHECK_PTR(slab); CHECK_PTR(send);
  KnobScope knobs(p);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const so3::FftArgs a0 = shard_pass_args(p, 0, slab, p->d_scratch);   // plain strides: TMA-fed when it applies
  int rc = launch_fft_tma(p, a0, +1, st);
  if (rc < 0) rc = launch_fft(p, a0, +1, 1, st);
  if (rc) return rc;
  return launch_fft(p, shard_pass_args(p, 1, p->d_scratch, send), +1, 1, st);
}

#define CHECK_CHUNK(p, q) \
  if ((q) < 0 || (q) >= (p)->chunks) return fail(SO3_ERR_INVALID, "chunk outside [0, chunks)")

// chunk q of layout B starts at row world * chunk_off[q]
int so3_shard_dwt_analysis_chunk(so3_plan_t p, int q, const void* recv_chunk, void* coeffs, void* stream) {
  CHECK_PLAN(p); CHECK_SHARD(p); CHECK_CHUNK(p, q); CHECK_PTR(recv_chunk); CHECK_PTR(coeffs);
  KnobScope knobs(p);
  return launch_dwt<true>(p, recv_chunk, coeffs, p->chunk_cl[q], p->chunk_cl[q + 1], static_cast<cudaStream_t>(stream),
                          p->chunk_pairs[q]);
}

int so3_shard_dwt_synthesis_chunk(so3_plan_t p, int q, const void* coeffs, void* send_chunk, void* stream) {
  CHECK_PLAN(p); CHECK_SHARD(p); CHECK_CHUNK(p, q); CHECK_PTR(coeffs); CHECK_PTR(send_chunk);
  KnobScope knobs(p);
  return launch_dwt<false>(p, send_chunk, const_cast<void*>(coeffs), p->chunk_cl[q], p->chunk_cl[q + 1],
                           static_cast<cudaStream_t>(stream), p->chunk_pairs[q]);
}

int so3_shard_dwt_analysis(so3_plan_t p, const void* recv, void* coeffs, void* stream) {
  CHECK_PLAN(p); CHECK_SHARD(p); CHECK_PTR(recv); CHECK_PTR(coeffs);
  for (int q = 0; q < p->chunks; ++q) {
    const double2* part = static_cast<const double2*>(recv) + (int64_t)p->world * p->chunk_off[q] * p->J;
    if (int rc = so3_shard_dwt_analysis_chunk(p, q, part, coeffs, stream)) return rc;
  }
  return SO3_OK;
}

int so3_shard_dwt_synthesis(so3_plan_t p, const void* coeffs, void* send, void* stream) {
  CHECK_PLAN(p); CHECK_SHARD(p); CHECK_PTR(coeffs); CHECK_PTR(send);
  for (int q = 0; q < p->chunks; ++q) {
    double2* part = static_cast<double2*>(send) + (int64_t)p->world * p->chunk_off[q] * p->J;
    if (int rc = so3_shard_dwt_synthesis_chunk(p, q, coeffs, part, stream)) return rc;
  }
  return SO3_OK;
}

int so3_shard_fft_synthesis(so3_plan_t p, const void* recv, void* slab, void* stream) {
  CHECK_PLAN(p); CHECK_SHARD(p); CHECK_PTR(recv); CHECK_PTR(slab);
  KnobScope knobs(p);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = launch_fft(p, shard_pass_args(p, 2, recv, p->d_scratch), -1, 1, st);
  if (rc) return rc;
  const so3::FftArgs a3 = shard_pass_args(p, 3, p->d_scratch, slab);   // plain strides: TMA-fed when it applies
  rc = launch_fft_tma(p, a3, -1, st);
  return rc >= 0 ? rc : launch_fft(p, a3, -1, 1, st);
}

// Direct O(B^6) transforms (soft.py:212-256): closed-form Wigner functions, no plan.
static int direct_common(int b, double** d_betas, double** d_w, double** d_tab, cudaStream_t st) {
  const int n = 2 * b;
  const long long C = so3_coeff_count(b);
  std::vector<double> betas(n), w(n);
  for (int j = 0; j < n; ++j) betas[j] = (2.0 * j + 1.0) * 3.141592653589793 / (4.0 * b);   // quadrature.py:61
  host_weights(b, w.data());
  SO3_CUDA(cudaMalloc((void**)d_betas, n * sizeof(double)));
  SO3_CUDA(cudaMalloc((void**)d_w, n * sizeof(double)));
  SO3_CUDA(cudaMalloc((void**)d_tab, (size_t)C * n * sizeof(double)));
  SO3_CUDA(cudaMemcpyAsync(*d_betas, betas.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
  SO3_CUDA(cudaMemcpyAsync(*d_w, w.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
  const long long tot = C * n;
  so3::direct_table_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(b, *d_betas, *d_tab);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

int so3_ifsoft_direct(int b, const void* coeffs, void* samples, void* stream) {
  if (!valid_bandwidth(b) || b > 64) return fail(SO3_ERR_INVALID, "direct transforms support 1 <= B <= 64");
  CHECK_PTR(coeffs); CHECK_PTR(samples);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *be = nullptr, *w = nullptr, *tab = nullptr;
  int rc = direct_common(b, &be, &w, &tab, st);
  if (rc == SO3_OK) {
    const long long tot = so3_grid_count(b);
    so3::ifsoft_direct_kernel<<<(unsigned)((tot + 127) / 128), 128, 0, st>>>(
        b, tab, static_cast<const double2*>(coeffs), static_cast<double2*>(samples));
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(SO3_ERR_CUDA, std::string("ifsoft_direct: ") + cudaGetErrorString(e));
  }
  cudaFree(be); cudaFree(w); cudaFree(tab);
  return rc;
}

int so3_fsoft_direct(int b, const void* samples, void* coeffs, void* stream) {
  if (!valid_bandwidth(b) || b > 64) return fail(SO3_ERR_INVALID, "direct transforms support 1 <= B <= 64");
  CHECK_PTR(coeffs); CHECK_PTR(samples);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *be = nullptr, *w = nullptr, *tab = nullptr;
  int rc = direct_common(b, &be, &w, &tab, st);
  if (rc == SO3_OK) {
    so3::fsoft_direct_kernel<<<(unsigned)so3_coeff_count(b), 256, 0, st>>>(
        b, tab, w, static_cast<const double2*>(samples), static_cast<double2*>(coeffs));
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(SO3_ERR_CUDA, std::string("fsoft_direct: ") + cudaGetErrorString(e));
  }
  cudaFree(be); cudaFree(w); cudaFree(tab);
  return rc;
}

// ---------------------------------------------------------------- SOFC / SOFG streaming (sofio.cuh)

int so3_container_info(const char* path, int* kind, int* bandwidth, int64_t* elements) {
  if (!path) return fail(SO3_ERR_INVALID, "null path");
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return fail(SO3_ERR_INVALID, std::string(path) + ": " + strerror(errno));
  so3io::Header h;
  std::string why;
  const int rc = so3io::parse_header(fd, path, &h, &why);
  close(fd);
  if (rc) return fail(rc, why);
  if (kind) *kind = h.kind;
  if (bandwidth) *bandwidth = h.bandwidth;
  if (elements) *elements = h.elements;
  return SO3_OK;
}

int so3_read_container(const char* path, int kind, int jbase, int J, void* dst, int dst_on_device,
                       int64_t staging_bytes, void* stream) {
  if (!path || !dst) return fail(SO3_ERR_INVALID, "null path or destination");
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return fail(SO3_ERR_INVALID, std::string(path) + ": " + strerror(errno));
  so3io::Header h;
  std::string why;
  int rc = so3io::parse_header(fd, path, &h, &why, kind);
  const int n = 2 * h.bandwidth;
  if (!rc && kind == 1) {
    if (J == 0) { jbase = 0; J = n; }
    if (jbase < 0 || J < 1 || jbase + J > n) {
      why = "beta slab [" + std::to_string(jbase) + ", " + std::to_string(jbase + J) + ") outside [0, " +
            std::to_string(n) + ")";
      rc = SO3_ERR_INVALID;
    }
  }
  if (rc) { close(fd); return fail(rc, why); }
  const so3io::Rows rw = so3io::slab_rows(kind, h.bandwidth, jbase, J);
  const long long doubles = (long long)(rw.rows * (long long)rw.row_bytes / 8);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dst_on_device) {
    rc = so3io::stream_in(fd, rw, static_cast<char*>(dst), (size_t)std::max<int64_t>(staging_bytes, 1 << 20), st, &why);
    close(fd);
    if (rc) return fail(rc, std::string(path) + ": " + (why.empty() ? cudaGetErrorString(cudaGetLastError()) : why));
    unsigned long long bad = 0;
    if (so3io::device_nonfinite(dst, doubles, st, &bad)) return fail(SO3_ERR_CUDA, "non-finite check failed");
    if (bad) return fail(SO3_ERR_INVALID, std::string(path) + ": payload contains non-finite values");
    return SO3_OK;
  }
  char* out = static_cast<char*>(dst);
  bool ok = true;
  if (rw.file_stride == (off_t)rw.row_bytes) ok = so3io::pread_all(fd, out, (size_t)rw.rows * rw.row_bytes, rw.off0);
  else
    for (long long r = 0; ok && r < rw.rows; ++r)
      ok = so3io::pread_all(fd, out + r * rw.row_bytes, rw.row_bytes, rw.off0 + (off_t)r * rw.file_stride);
  close(fd);
  if (!ok) return fail(SO3_ERR_INVALID, std::string(path) + ": read failed");
  if (so3io::host_nonfinite(reinterpret_cast<const double*>(dst), doubles))
    return fail(SO3_ERR_INVALID, std::string(path) + ": payload contains non-finite values");
  return SO3_OK;
}

int so3_write_container(const char* path, int kind, int bandwidth, int jbase, int J, const void* src, int src_on_device,
                        int create, int64_t staging_bytes, void* stream) {
  if (!path || !src) return fail(SO3_ERR_INVALID, "null path or source");
  if (!valid_bandwidth(bandwidth) || (kind != 0 && kind != 1)) return fail(SO3_ERR_INVALID, "bad bandwidth or kind");
  const int n = 2 * bandwidth;
  if (kind == 1) {
    if (J == 0) { jbase = 0; J = n; }
    if (jbase < 0 || J < 1 || jbase + J > n) return fail(SO3_ERR_INVALID, "beta slab outside the grid");
  }
  const so3io::Rows rw = so3io::slab_rows(kind, bandwidth, jbase, J);
  const long long doubles = (long long)(rw.rows * (long long)rw.row_bytes / 8);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the reference refuses to persist non-finite values (core.py:180-181): checked before the file is touched
  if (src_on_device) {
    unsigned long long bad = 0;
    if (so3io::device_nonfinite(src, doubles, st, &bad)) return fail(SO3_ERR_CUDA, "non-finite check failed");
    if (bad) return fail(SO3_ERR_INVALID, "refusing to persist non-finite values");
  } else if (so3io::host_nonfinite(static_cast<const double*>(src), doubles)) {
    return fail(SO3_ERR_INVALID, "refusing to persist non-finite values");
  }
  const int fd = open(path, create ? (O_WRONLY | O_CREAT | O_TRUNC) : O_RDWR, 0644);
  if (fd < 0) return fail(SO3_ERR_INVALID, std::string(path) + ": " + strerror(errno));
  std::string why;
  int rc = SO3_OK;
  if (create) {
    unsigned char head[so3io::kHeader];
    memcpy(head, kind ? "SOFG" : "SOFC", 4);
    const uint32_t v = so3io::kVersion, b = (uint32_t)bandwidth;
    memcpy(head + 4, &v, 4);
    memcpy(head + 8, &b, 4);
    if (!so3io::pwrite_all(fd, head, so3io::kHeader, 0) ||
        ftruncate(fd, (off_t)so3io::kHeader + (off_t)so3io::expected_elements(kind, bandwidth) * 16) != 0) {
      why = strerror(errno);
      rc = SO3_ERR_INVALID;
    }
  } else {
    so3io::Header h;
    rc = so3io::parse_header(fd, path, &h, &why);
    if (!rc && (h.kind != kind || h.bandwidth != bandwidth)) {
      why = std::string(path) + ": existing container does not match (kind, bandwidth)";
      rc = SO3_ERR_INVALID;
    }
  }
  if (!rc) {
    if (src_on_device) {
      rc = so3io::stream_out(fd, rw, static_cast<const char*>(src), (size_t)std::max<int64_t>(staging_bytes, 1 << 20),
                             st, &why);
    } else {
      const char* in = static_cast<const char*>(src);
      bool ok = true;
      if (rw.file_stride == (off_t)rw.row_bytes) ok = so3io::pwrite_all(fd, in, (size_t)rw.rows * rw.row_bytes, rw.off0);
      else
        for (long long r = 0; ok && r < rw.rows; ++r)
          ok = so3io::pwrite_all(fd, in + r * rw.row_bytes, rw.row_bytes, rw.off0 + (off_t)r * rw.file_stride);
      if (!ok) { why = strerror(errno); rc = SO3_ERR_INVALID; }
    }
  }
  close(fd);
  if (rc) return fail(rc, std::string(path) + ": " + why);
  return SO3_OK;
}

static unsigned blocks_for(long long count) { return (unsigned)((count + 255) / 256); }

int so3_jacobi_eval(int n, double a, double b, const double* x, int64_t count, double* out, void* stream) {
  if (n < 0) return fail(SO3_ERR_INVALID, "degree n must be a nonnegative integer, got " + std::to_string(n));
  if (!(a > -1.0) || !(b > -1.0)) return fail(SO3_ERR_INVALID, "Jacobi exponents must exceed -1");
  if (count < 0 || (count > 0 && (!x || !out))) return fail(SO3_ERR_INVALID, "bad buffers");
  if (count == 0) return SO3_OK;
  so3::jacobi_eval_kernel<<<blocks_for(count), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, a, b, x, count, out);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

int so3_wigner_d_eval(int l, int m, int mp, const double* beta, int64_t count, double* out, void* stream) {
  if (l < 0 || std::abs(m) > l || std::abs(mp) > l)
    return fail(SO3_ERR_INVALID, "invalid orders (l=" + std::to_string(l) + ", m=" + std::to_string(m) +
                                     ", m'=" + std::to_string(mp) + ")");
  if (count < 0 || (count > 0 && (!beta || !out))) return fail(SO3_ERR_INVALID, "bad buffers");
  if (count == 0) return SO3_OK;
  so3::wigner_direct_eval_kernel<<<blocks_for(count), 256, 0, static_cast<cudaStream_t>(stream)>>>(l, m, mp, beta,
                                                                                                 count, out);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

int so3_wigner_rows_eval(int b, int m, int mp, const double* beta, int64_t count, double* out, void* stream) {
  if (!valid_bandwidth(b)) return fail(SO3_ERR_INVALID, "bandwidth must be in [1, 4096], got " + std::to_string(b));
  const int L = std::max(std::abs(m), std::abs(mp));
  if (L >= b)
    return fail(SO3_ERR_INVALID, "order pair (m=" + std::to_string(m) + ", m'=" + std::to_string(mp) +
                                     ") has no degrees below B=" + std::to_string(b));
  if (count < 0 || (count > 0 && (!beta || !out))) return fail(SO3_ERR_INVALID, "bad buffers");
  if (count == 0) return SO3_OK;
  // norm of wigner_d_seed (wigner.py:124/131) in the reference's own double arithmetic
  const int big = std::max(std::abs(m), std::abs(mp)), o = std::abs(m) >= std::abs(mp) ? mp : m;
  const double norm = std::exp(0.5 * (std::lgamma(2.0 * big + 1) - std::lgamma((double)big + o + 1) -
                                      std::lgamma((double)big - o + 1)));
  so3::wigner_rows_eval_kernel<<<blocks_for(count), 256, 0, static_cast<cudaStream_t>(stream)>>>(b, m, mp, norm,
                                                                                               beta, count, out);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

int so3_wigner_rows(so3_plan_t p, int m, int mp, double* out, void* stream) {
  CHECK_PLAN(p); CHECK_PTR(out);
  const int L = std::max(std::abs(m), std::abs(mp));
  if (L >= p->B) return fail(SO3_ERR_INVALID, "order pair has no degrees below B");
  // find the base pair 0 <= b' <= b and the relation mapping it to (m, m')
  static const int rel[8][8] = {{0, 0, 0, 0, 1, 0, 0, 1},  {0, 0, 1, 1, -1, 0, 0, -1}, {0, 0, 1, 1, 0, 1, 1, 0},
                                {0, 0, 0, 0, 0, -1, -1, 0}, {1, 1, 0, 1, -1, 0, 0, 1},  {1, 1, 1, 0, 1, 0, 0, -1},
                                {1, 1, 0, 1, 0, -1, 1, 0},  {1, 1, 1, 0, 0, 1, -1, 0}};
  const int bm = std::max(std::abs(m), std::abs(mp)), bmp = std::min(std::abs(m), std::abs(mp));
  int tag = -1;
  for (int k = 0; k < 8 && tag < 0; ++k) {
    const int tm = rel[k][4] * bm + rel[k][5] * bmp, tp = rel[k][6] * bm + rel[k][7] * bmp;
    if (tm == m && tp == mp) tag = k;
  }
  if (tag < 0) return fail(SO3_ERR_INVALID, "no symmetry relation reaches the pair");
  const long double ln = 0.5L * (lgammal(2.0L * bm + 1) - lgammal((long double)bm + bmp + 1) - lgammal((long double)bm - bmp + 1));
  double hi, lo;
  split_ld(ln, &hi, &lo);
  const int par0 = (rel[tag][2] * bm + rel[tag][3] * bmp) & 1;
  wigner_rows_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      p->B, p->n, m, mp, bm, bmp, rel[tag][0], rel[tag][1], par0, make_double2(hi, lo), p->d_xv, p->d_logcs, out);
  SO3_CUDA(cudaGetLastError());
  return SO3_OK;
}

}  // extern "C"

// Which feature of the synthesis inner loop costs throughput?  Per quad: 32 DMMA + a
// 4-step recurrence on JT=4 chains, adding one real-kernel feature per mode.
#include <cstdio>
#include <cuda_runtime.h>
#define MMA(c0, c1, a, b) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b))
constexpr int S = 132;
template <int MODE>
__global__ void __launch_bounds__(128, 2) k(double* out, int iters, const double* rct) {
  __shared__ double Dt[4][4 * S];
  __shared__ double fco[32][16];
  __shared__ double rcs[96];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, tq = lane & 3;
  double acc[16][2][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) { acc[i][0][0] = acc[i][0][1] = acc[i][1][0] = acc[i][1][1] = 0; }
  for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) fco[i / 16][i % 16] = 1e-3 * i;
  for (int i = threadIdx.x; i < 96; i += blockDim.x) rcs[i] = rct[i];
  double x[4], cur[4], prev[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) { x[q] = 0.1 * q + lane * 1e-4; cur[q] = 1.0; prev[q] = 0.5; }
  double3 rcw = make_double3(rct[3 * lane], rct[3 * lane + 1], rct[3 * lane + 2]);
  double* D = Dt[warp];
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    // recurrence, 4 steps
    double hA[4], hS[4], hC[4];
    if (MODE == 6) {
#pragma unroll
      for (int ll = 0; ll < 4; ++ll) {
        hA[ll] = __shfl_sync(0xffffffffu, rcw.x, (4 * it + ll) & 31);
        hS[ll] = __shfl_sync(0xffffffffu, rcw.y, (4 * it + ll) & 31);
        hC[ll] = __shfl_sync(0xffffffffu, rcw.z, (4 * it + ll) & 31);
      }
    }
#pragma unroll
    for (int ll = 0; ll < 4; ++ll) {
      double A = 1.0000001, AS = 1e-3, C = 0.999999;
      if (MODE == 2 || MODE == 3) {
        A = __shfl_sync(0xffffffffu, rcw.x, (4 * it + ll) & 31);
        AS = __shfl_sync(0xffffffffu, rcw.y, (4 * it + ll) & 31);
        C = __shfl_sync(0xffffffffu, rcw.z, (4 * it + ll) & 31);
      } else if (MODE == 4) {       // broadcast LDS from a shared table
        const double* r = rcs + 3 * ((4 * it + ll) & 31);
        A = r[0]; AS = r[1]; C = r[2];
      } else if (MODE == 5) {       // uniform global load (L1 hit)
        const double* r = rct + 3 * ((4 * it + ll) & 31);
        A = __ldg(r); AS = __ldg(r + 1); C = __ldg(r + 2);
      } else if (MODE == 6) {       // hoisted shuffles
        A = hA[ll]; AS = hS[ll]; C = hC[ll];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (MODE >= 1) D[ll * S + lane + 32 * q] = cur[q];
        double tt = fma(A, x[q], -AS);
        double nx = fma(tt, cur[q], -C * prev[q]);
        prev[q] = cur[q]; cur[q] = nx;
      }
    }
    if (MODE >= 1) __syncwarp();
    double b0 = 1.0 + lane * 1e-4, b1 = 0.5;
    if (MODE >= 3 && MODE != 5) { b0 = fco[(4 * it + tq) & 31][g]; b1 = fco[(4 * it + tq) & 31][8 + g]; }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      double av = (MODE >= 1) ? D[tq * S + 8 * i + g] : cur[i & 3];
      MMA(acc[i][0][0], acc[i][0][1], av, b0);
      MMA(acc[i][1][0], acc[i][1][1], av, b1);
    }
    if (MODE >= 1) __syncwarp();
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i][0][0] + acc[i][0][1] + acc[i][1][0] + acc[i][1][1];
  if (s == 1.2345) out[0] = s;
}
template <int MODE>
void run(double* out, const double* rct) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 512, threads = 128, blocks = 148 * 2;
  for (int r = 0; r < 2; ++r) {
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(out, iters, rct);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 32 * iters * (double)blocks * threads / 32;
    if (r) printf("mode %d: DMMA part %.2f TF/s (%.0f%%)\n", MODE, fl / ms / 1e9, 100 * fl / ms / 1e9 / 36.97);
  }
}
int main() {
  double* out; cudaMalloc(&out, 8);
  double* rct; cudaMalloc(&rct, 8 * 96);
  double h[96]; for (int i = 0; i < 96; ++i) h[i] = (i % 3 == 0) ? 1.0000001 : (i % 3 == 1) ? 1e-3 : 0.999999;
  cudaMemcpy(rct, h, sizeof h, cudaMemcpyHostToDevice);
  run<0>(out, rct); run<1>(out, rct); run<2>(out, rct); run<3>(out, rct); run<4>(out, rct); run<5>(out, rct); run<6>(out, rct);
  return 0;
}

// DMMA stream + three-term-recurrence DFMA chains sharing the FP64 pipe: which schedule
// keeps the pipe busy?  Per "quad": 32 independent DMMA + 4 steps x JT chains x 3 DP ops.
#include <cstdio>
#include <cuda_runtime.h>
#define MMA(c, a, b) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b))
template <int MODE, int JT>
__global__ void __launch_bounds__(128) k(double* out, int iters, double A, double AS, double C) {
  double acc[32][2];
#pragma unroll
  for (int i = 0; i < 32; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double x[JT], cur[JT], prev[JT];
#pragma unroll
  for (int q = 0; q < JT; ++q) { x[q] = 0.1 * q + threadIdx.x * 1e-4; cur[q] = 1.0; prev[q] = 0.5; }
  const double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {            // blocked: all DMMAs, then the 4-step recurrence
#pragma unroll
      for (int i = 0; i < 32; ++i) MMA(acc[i], a, cur[i % JT]);
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int q = 0; q < JT; ++q) { double tt = fma(A, x[q], -AS); double nx = fma(tt, cur[q], -C * prev[q]); prev[q] = cur[q]; cur[q] = nx; }
    } else if (MODE == 1) {     // interleaved: 8 DMMAs per recurrence step
#pragma unroll
      for (int s = 0; s < 4; ++s) {
#pragma unroll
        for (int i = 0; i < 8; ++i) MMA(acc[8 * s + i], a, b);
#pragma unroll
        for (int q = 0; q < JT; ++q) { double tt = fma(A, x[q], -AS); double nx = fma(tt, cur[q], -C * prev[q]); prev[q] = cur[q]; cur[q] = nx; }
      }
    } else {                    // DMMA only (reference)
#pragma unroll
      for (int i = 0; i < 32; ++i) MMA(acc[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
  for (int q = 0; q < JT; ++q) s += cur[q];
  if (s == 1.2345) out[0] = s;
}
template <int MODE, int JT>
void run(double* out, int warps_per_sm) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 512, threads = 128, blocks = 148 * warps_per_sm / 4;
  for (int r = 0; r < 2; ++r) {
    cudaEventRecord(e0);
    k<MODE, JT><<<blocks, threads>>>(out, iters, 1.0000001, 1e-3, 0.999999);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double mma_fl = 2.0 * 256 * 32 * iters * (double)blocks * threads / 32;
    if (r) printf("mode=%d JT=%d warps/SM=%2d: DMMA part %.2f TF/s (%.0f%% of 36.97)\n", MODE, JT, warps_per_sm, mma_fl / ms / 1e9, 100 * mma_fl / ms / 1e9 / 36.97);
  }
}
int main() {
  double* out; cudaMalloc(&out, 8);
  for (int w : {4, 8, 16}) {
    run<2, 4>(out, w);
    run<0, 4>(out, w);
    run<1, 4>(out, w);
    run<0, 2>(out, w);
    run<1, 2>(out, w);
  }
  return 0;
}

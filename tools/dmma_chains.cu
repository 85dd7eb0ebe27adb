// DMMA m8n8k4 throughput vs independent accumulator chains per warp and warps per SM
// sub-partition (dev probe).  Prints TF/s per (warps/SMSP, chains).
#include <cstdio>
#include <cuda_runtime.h>
#define MMA(c0, c1, a, b) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b))
template <int C>
__global__ void k(double* out, int iters) {
  double c[C][2];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16 / C; ++r)
#pragma unroll
      for (int i = 0; i < C; ++i) MMA(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int C>
void run(double* o, int wps) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, threads = 128 * wps;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<C><<<sms, threads>>>(o, iters);
  cudaEventRecord(e0);
  k<C><<<sms, threads>>>(o, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * 256 * 16 * (double)iters * (threads / 32) * sms;
  printf("{\"warps_per_smsp\": %d, \"chains\": %d, \"tflops\": %.2f}\n", wps, C, fl / ms / 1e9);
}
int main() {
  double* o; cudaMalloc(&o, 8 << 20);
  for (int w : {1, 2, 3, 4}) { run<1>(o, w); run<2>(o, w); run<4>(o, w); run<8>(o, w); }
  return 0;
}

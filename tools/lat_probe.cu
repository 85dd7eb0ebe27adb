// Dependent-issue latency of DMMA m8n8k4 and DFMA on one warp (clock64 based).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, int iters) {
  double c0 = threadIdx.x, c1 = 1.0, a = 1.0000001, b = 0.9999999, f = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) f = fma(f, a, b);
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) { f = f * a; }
  long long t3 = clock64();
  double sh = f;
  for (int i = 0; i < iters; ++i) sh = __shfl_sync(0xffffffffu, sh, (threadIdx.x + 1) & 31);
  long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  out[threadIdx.x] = c0 + c1 + f + sh;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 64); cudaMallocManaged(&c, 64);
  const int it = 4096;
  lat<<<1, 32>>>(o, c, it); cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, it); cudaDeviceSynchronize();
  printf("dependent latency (cycles): DMMA %.1f  DFMA %.1f  DMUL %.1f  SHFL.f64 %.1f\n", c[0] / (double)it, c[1] / (double)it, c[2] / (double)it, c[3] / (double)it);
  return 0;
}

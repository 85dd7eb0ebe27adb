// FP64 peak micro-benchmark for the roofline denominator (B200, sm_100a).
// Measures: (1) SIMT DFMA throughput, (2) DMMA (mma.sync f64) throughput for
// several shapes, (3) DFMA and DMMA issued concurrently from the same warps.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

// m8n8k4: 256 FMA per warp instruction
__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// m16n8k4: 512 FMA per warp instruction
__global__ void dmma1684_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

// m16n8k16: 2048 FMA per warp instruction (A: 8 regs, B: 4 regs)
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

// mixed: per iteration 8 m8n8k4 DMMA (2048 FMA/warp) + NF DFMA per thread (32*NF FMA/warp)
template <int NF>
__global__ void mixed_kernel(double* out, int iters, double x, double y) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  double acc[NF];
#pragma unroll
  for (int i = 0; i < NF; ++i) acc[i] = i;
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < NF; ++i) acc[i] = fma(acc[i], x, y);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < NF; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
float time_it(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  double* out; CK(cudaMalloc(&out, 8));
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  const int iters = 4096;
  for (int wpb : {4, 8, 16}) {
    int threads = 32 * wpb, blocks = sms * (32 / wpb);
    float ms = time_it([&] { dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); });
    double fl = 2.0 * 8 * iters * (double)threads * blocks;
    printf(", \"dfma_tflops_w%d\": %.3f", wpb, fl / ms / 1e9);
  }
  {
    int threads = 256, blocks = sms * 8;
    float ms = time_it([&] { dmma884_kernel<<<blocks, threads>>>(out, iters / 4); });
    double fl = 2.0 * 256 * 8 * (iters / 4) * (threads / 32.0) * blocks;
    printf(", \"dmma_m8n8k4_tflops\": %.3f", fl / ms / 1e9);
  }
  {
    int threads = 256, blocks = sms * 8;
    float ms = time_it([&] { dmma1684_kernel<<<blocks, threads>>>(out, iters / 8); });
    double fl = 2.0 * 512 * 8 * (iters / 8) * (threads / 32.0) * blocks;
    printf(", \"dmma_m16n8k4_tflops\": %.3f", fl / ms / 1e9);
  }
  {
    int threads = 256, blocks = sms * 8;
    float ms = time_it([&] { dmma16816_kernel<<<blocks, threads>>>(out, iters / 32); });
    double fl = 2.0 * 2048 * 4 * (iters / 32) * (threads / 32.0) * blocks;
    printf(", \"dmma_m16n8k16_tflops\": %.3f", fl / ms / 1e9);
  }
  {
    int threads = 256, blocks = sms * 8;
    float ms = time_it([&] { mixed_kernel<16><<<blocks, threads>>>(out, iters / 4, 0.999999, 1e-7); });
    double fl_mma = 2.0 * 256 * 8 * (iters / 4) * (threads / 32.0) * blocks;
    double fl_fma = 2.0 * 16 * (iters / 4) * (double)threads * blocks;
    printf(", \"mixed16_total_tflops\": %.3f, \"mixed16_ms\": %.3f, \"mixed16_mma_part\": %.3f", (fl_mma + fl_fma) / ms / 1e9, ms, fl_mma / (fl_mma + fl_fma));
  }
  {
    int threads = 256, blocks = sms * 8;
    float ms = time_it([&] { mixed_kernel<4><<<blocks, threads>>>(out, iters / 4, 0.999999, 1e-7); });
    double fl_mma = 2.0 * 256 * 8 * (iters / 4) * (threads / 32.0) * blocks;
    double fl_fma = 2.0 * 4 * (iters / 4) * (double)threads * blocks;
    printf(", \"mixed4_total_tflops\": %.3f, \"mixed4_ms\": %.3f", (fl_mma + fl_fma) / ms / 1e9, ms);
  }
  printf("}\n");
  return 0;
}

// Inner loops of the segment-parallel DWT (dwt_seg.cuh) on synthetic data: the Wigner values go
// from the recurrence registers straight into the DMMA operand (lane (r, k) runs the recurrence
// of degree segment r / k at its own beta index), no shared-memory Wigner tile.  Reports the
// DMMA part as a fraction of the measured DMMA peak (36.97 TF/s).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/seg_probe tools/seg_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#define MMA(c0, c1, a, b) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b))

// analysis: NB groups of 4 beta per warp; per step one table LDS.128, NB x (2 DFMA + 2 DMMA),
// the 8 x 16 partial tile to shared memory, a CTA barrier + reduction every TB steps
template <int NB, int W, int TB, int MINB>
__global__ void __launch_bounds__(W * 32, MINB) ana(double* out, int steps, const double2* tab) {
  extern __shared__ double sm[];
  double2* rcs = reinterpret_cast<double2*>(sm);             // [8][65]
  double* part = sm + 2 * 8 * 65;                            // [2][TB][W][128]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, r = lane >> 2;
  for (int i = t; i < 8 * 65; i += blockDim.x) rcs[i] = tab[i % 96];
  double cur[NB], prev[NB], v[NB], xr[NB], xi[NB];
#pragma unroll
  for (int g = 0; g < NB; ++g) {
    cur[g] = 1.0 + 1e-3 * g; prev[g] = 0.5; v[g] = 1e-4 * (lane + 32 * g); xr[g] = 1.0 + lane * 1e-3; xi[g] = 0.5 - g * 1e-3;
  }
  __syncthreads();
  double sum = 0.0;
  int buf = 0;
  for (int t0 = 0; t0 < steps; t0 += TB, buf ^= 1) {
#pragma unroll
    for (int tb = 0; tb < TB; ++tb) {
      const double2 k2 = rcs[r * 65 + ((t0 + tb) & 63)];
      double a0 = 0, a1 = 0, b0 = 0, b1 = 0;
#pragma unroll
      for (int g = 0; g < NB; ++g) {
        MMA(a0, a1, cur[g], xr[g]);
        MMA(b0, b1, cur[g], xi[g]);
        const double nx = fma(fma(k2.x, v[g], k2.y), cur[g], -prev[g]);
        prev[g] = cur[g];
        cur[g] = nx;
      }
      double* pw = part + (((size_t)buf * TB + tb) * W + warp) * 128;
      *reinterpret_cast<double2*>(pw + 2 * lane) = make_double2(a0, a1);
      *reinterpret_cast<double2*>(pw + 64 + 2 * lane) = make_double2(b0, b1);
    }
    __syncthreads();
    for (int idx = t; idx < TB * 128; idx += blockDim.x) {
      const double* pb = part + ((size_t)buf * TB + idx / 128) * W * 128 + (idx & 127);
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < W; ++w) s += pb[w * 128];
      sum += s;
    }
  }
  if (sum == 1.2345) out[0] = sum;
}

// synthesis: NB groups of 8 beta per warp, 2 accumulator tiles each; per step one table LDS.128,
// one coefficient LDS.128, NB x (2 DFMA + 2 DMMA); a barrier every TB steps (coefficient staging)
template <int NB, int W, int TB, int MINB, int DF = 2>
__global__ void __launch_bounds__(W * 32, MINB) syn(double* out, int steps, const double2* tab) {
  __shared__ double2 rcs[4 * 129];
  __shared__ double2 fco[2][4][TB + 2][8];
  const int t = threadIdx.x, lane = t & 31, r = lane >> 2, k = lane & 3;
  for (int i = t; i < 4 * 129; i += blockDim.x) rcs[i] = tab[i % 96];
  for (int i = t; i < 2 * 4 * (TB + 2) * 8; i += blockDim.x) (&fco[0][0][0][0])[i] = make_double2(1e-3 * i, 1.0);
  double cur[NB], prev[NB], v[NB], acc[NB][2][2];
#pragma unroll
  for (int g = 0; g < NB; ++g) {
    cur[g] = 1.0 + 1e-3 * g; prev[g] = 0.5; v[g] = 1e-4 * (lane + 32 * g);
    acc[g][0][0] = acc[g][0][1] = acc[g][1][0] = acc[g][1][1] = 0.0;
  }
  __syncthreads();
  int buf = 0;
  for (int t0 = 0; t0 < steps; t0 += TB, buf ^= 1) {
#pragma unroll 4
    for (int tb = 0; tb < TB; ++tb) {
      const double2 k2 = rcs[k * 129 + ((t0 + tb) & 127)];
      const double2 f = fco[buf][k][tb][r];
#pragma unroll
      for (int g = 0; g < NB; ++g) {
        MMA(acc[g][0][0], acc[g][0][1], cur[g], f.x);
        MMA(acc[g][1][0], acc[g][1][1], cur[g], f.y);
        if (DF == 2) {
          const double nx = fma(fma(k2.x, v[g], k2.y), cur[g], -prev[g]);
          prev[g] = cur[g];
          cur[g] = nx;
        } else if (DF == 1) {
          const double nx = fma(k2.x, cur[g], -prev[g]);
          prev[g] = cur[g];
          cur[g] = nx;
        } else if (DF == 3) {   // integer work instead of FP64
          cur[g] = __longlong_as_double(__double_as_longlong(cur[g]) ^ (long long)(t0 + tb));
        }
      }
    }
    if (t < TB * 4) fco[buf ^ 1][t & 3][t >> 2][r] = make_double2(1e-3 * t0, 0.5);
    __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int g = 0; g < NB; ++g) s += acc[g][0][0] + acc[g][0][1] + acc[g][1][0] + acc[g][1][1];
  if (s == 1.2345) out[0] = s;
}

template <typename K>
void run(const char* name, K kern, int threads, int per_sm, size_t smem, int nb, double* out, const double2* tab) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int steps = 4096, blocks = 148 * per_sm;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    kern<<<blocks, threads, smem>>>(out, steps, tab);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 256 * 2 * nb * steps * (double)blocks * threads / 32;
    if (rep) printf("%-28s %d CTA/SM: DMMA part %.2f TF/s (%.0f%% of 36.97)  [%s]\n", name, per_sm, fl / ms / 1e9, 100 * fl / ms / 1e9 / 36.97,
                    cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  double* out; cudaMalloc(&out, 8);
  double2* tab; cudaMalloc(&tab, 16 * 96);
  double2 h[96]; for (int i = 0; i < 96; ++i) h[i] = make_double2(1.0000001, 1e-3);
  cudaMemcpy(tab, h, sizeof h, cudaMemcpyHostToDevice);
  auto asz = [](int tb, int w) { return (size_t)(2 * 8 * 65 + 2 * tb * w * 128) * 8; };
  run("ana NB16 W8 TB4", ana<16, 8, 4, 1>, 256, 1, asz(4, 8), 16, out, tab);
  run("ana NB16 W8 TB8", ana<16, 8, 8, 1>, 256, 1, asz(8, 8), 16, out, tab);
  run("ana NB16 W4 TB4", ana<16, 4, 4, 2>, 128, 2, asz(4, 4), 16, out, tab);
  run("ana NB16 W4 TB8", ana<16, 4, 8, 2>, 128, 2, asz(8, 4), 16, out, tab);
  run("ana NB8 W8 TB4 x2", ana<8, 8, 4, 2>, 256, 2, asz(4, 8), 8, out, tab);
  run("ana NB8 W16 TB4", ana<8, 16, 4, 1>, 512, 1, asz(4, 16), 8, out, tab);
  run("ana NB8 W4 TB8 x4", ana<8, 4, 8, 4>, 128, 4, asz(8, 4), 8, out, tab);
  run("syn NB8 W4 TB8 x3", syn<8, 4, 8, 3>, 128, 3, 0, 8, out, tab);
  run("syn NB8 W4 TB8 x2", syn<8, 4, 8, 2>, 128, 2, 0, 8, out, tab);
  run("syn NB8 W8 TB8 x1", syn<8, 8, 8, 1>, 256, 1, 0, 8, out, tab);
  run("syn NB8 W8 TB8 x2", syn<8, 8, 8, 2>, 256, 2, 0, 8, out, tab);
  run("syn NB16 W4 TB8 x2", syn<16, 4, 8, 2>, 128, 2, 0, 16, out, tab);
  run("syn NB4 W8 TB8 x3", syn<4, 8, 8, 3>, 256, 3, 0, 4, out, tab);
  run("syn NB8 W4 TB8 x2 DF0", syn<8, 4, 8, 2, 0>, 128, 2, 0, 8, out, tab);
  run("syn NB8 W4 TB8 x2 DF1", syn<8, 4, 8, 2, 1>, 128, 2, 0, 8, out, tab);
  run("syn NB8 W4 TB8 x2 DF3", syn<8, 4, 8, 2, 3>, 128, 2, 0, 8, out, tab);
  run("syn NB8 W4 TB8 x3 DF0", syn<8, 4, 8, 3, 0>, 128, 3, 0, 8, out, tab);
  run("syn NB8 W4 TB8 x4 DF0", syn<8, 4, 8, 4, 0>, 128, 4, 0, 8, out, tab);
  return 0;
}

// Direct O(B^6) transforms on the GPU (reference soft.py:212-256, wigner.py:43-114): the
// defining sums evaluated coefficient by coefficient from the closed-form Wigner functions.
// They share no code with the fast path (no recurrence table, no FFT, no symmetry
// derivation) and serve as an independent cross-check for small B (row 8(f).4).
#pragma once
#include "common.cuh"

namespace so3 {

// Jacobi P_n^(a,b)(x), standard three-term recurrence (wigner.py:43-68).
__device__ __forceinline__ double jacobi(int nd, double a, double b, double x) {
  double p0 = 1.0;
  if (nd == 0) return p0;
  double p1 = 0.5 * (a - b) + 0.5 * (a + b + 2.0) * x;
  for (int k = 2; k <= nd; ++k) {
    const double s = 2.0 * k + a + b;
    const double c1 = 2.0 * k * (k + a + b) * (s - 2.0);
    const double c2 = (s - 1.0) * s * (s - 2.0);
    const double c3 = (s - 1.0) * (a * a - b * b);
    const double c4 = 2.0 * (k + a - 1.0) * (k + b - 1.0) * s;
    const double p2 = ((c2 * x + c3) * p1 - c4 * p0) / c1;
    p0 = p1;
    p1 = p2;
  }
  return p1;
}

// d^l_{m,m'}(beta) by canonicalisation to m' >= |m| and the closed form (wigner.py:78-114).
__device__ __forceinline__ double wigner_closed(int l, int m, int mp, double beta) {
  double sg;
  int mu, nu;
  if (mp >= abs(m)) { sg = 1.0; mu = m; nu = mp; }
  else if (-mp >= abs(m)) { sg = ((m - mp) & 1) ? -1.0 : 1.0; mu = -m; nu = -mp; }
  else if (m >= abs(mp)) { sg = ((m - mp) & 1) ? -1.0 : 1.0; mu = mp; nu = m; }
  else { sg = 1.0; mu = -mp; nu = -m; }
  const int a = nu - mu, b = mu + nu, nd = l - nu;
  const double lr = 0.5 * (lgamma(l + nu + 1.0) + lgamma(l - nu + 1.0) - lgamma(l + mu + 1.0) - lgamma(l - mu + 1.0));
  const double pre = (((mu + nu) & 1) ? -1.0 : 1.0) * exp(lr);
  const double h = 0.5 * beta;
  return sg * pre * pow(sin(h), (double)a) * pow(cos(h), (double)b) * jacobi(nd, (double)a, (double)b, cos(beta));
}

// D table: d[slot][j] for every coefficient slot (l-major) and beta_j; one thread per (slot, j).
__global__ void direct_table_kernel(int B, const double* betas, double* d) {
  const int n = 2 * B;
  const long long C = (long long)B * (4LL * B * B - 1) / 3;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= C * n) return;
  const long long slot = idx / n;
  const int j = (int)(idx % n);
  int l = 0;
  while ((long long)(l + 1) * (4LL * (l + 1) * (l + 1) - 1) / 3 <= slot) ++l;
  const long long r = slot - (long long)l * (4LL * l * l - 1) / 3;
  const int m = (int)(r / (2 * l + 1)) - l, mp = (int)(r % (2 * l + 1)) - l;
  d[idx] = wigner_closed(l, m, mp, betas[j]);
}

// ifsoft_direct (soft.py:236-256): one thread per sample (i, j, k).
__global__ void ifsoft_direct_kernel(int B, const double* d, const double2* coef, double2* grid) {
  const int n = 2 * B;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n * n * n) return;
  const int k = (int)(idx % n), j = (int)((idx / n) % n), i = (int)(idx / ((long long)n * n));
  const double step = 3.141592653589793 / B;   // alpha_i = gamma_i = i*pi/B
  double2 acc = make_double2(0.0, 0.0);
  long long slot = 0;
  for (int l = 0; l < B; ++l)
    for (int m = -l; m <= l; ++m) {
      double sa, ca;
      sincos(-(double)m * (i * step), &sa, &ca);
      for (int mp = -l; mp <= l; ++mp, ++slot) {
        double sg, cg;
        sincos(-(double)mp * (k * step), &sg, &cg);
        const double dv = d[slot * n + j];
        const double2 e = make_double2((ca * cg - sa * sg) * dv, (ca * sg + sa * cg) * dv);
        acc = cadd(acc, cmul(coef[slot], e));
      }
    }
  grid[idx] = acc;
}

// fsoft_direct (soft.py:212-233): one CTA per coefficient slot, block reduction over samples.
__global__ void fsoft_direct_kernel(int B, const double* d, const double* w, const double2* grid, double2* coef) {
  const int n = 2 * B;
  const long long slot = blockIdx.x;
  int l = 0;
  while ((long long)(l + 1) * (4LL * (l + 1) * (l + 1) - 1) / 3 <= slot) ++l;
  const long long r = slot - (long long)l * (4LL * l * l - 1) / 3;
  const int m = (int)(r / (2 * l + 1)) - l, mp = (int)(r % (2 * l + 1)) - l;
  const double step = 3.141592653589793 / B;
  double2 acc = make_double2(0.0, 0.0);
  for (long long idx = threadIdx.x; idx < (long long)n * n * n; idx += blockDim.x) {
    const int k = (int)(idx % n), j = (int)((idx / n) % n), i = (int)(idx / ((long long)n * n));
    double sa, ca, sg, cg;
    sincos((double)m * (i * step), &sa, &ca);
    sincos((double)mp * (k * step), &sg, &cg);
    const double dv = d[slot * n + j] * w[j];
    const double2 e = make_double2((ca * cg - sa * sg) * dv, (ca * sg + sa * cg) * dv);
    acc = cadd(acc, cmul(grid[idx], e));
  }
  __shared__ double2 red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] = cadd(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double scale = (2 * l + 1) / (8.0 * 3.141592653589793 * B);
    coef[slot] = make_double2(red[0].x * scale, red[0].y * scale);
  }
}

// ---- evaluation at arbitrary angles (the reference's wigner.py utilities, one thread per point)

// jacobi_poly (wigner.py:43-68) at count points.
__global__ void jacobi_eval_kernel(int nd, double a, double b, const double* x, long long count, double* out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = jacobi(nd, a, b, x[i]);
}

// wigner_d_direct (wigner.py:92-114) at count angles.
__global__ void wigner_direct_eval_kernel(int l, int m, int mp, const double* beta, long long count, double* out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = wigner_closed(l, m, mp, beta[i]);
}

// wigner_d_rows (wigner.py:139-178) for ANY pair at count angles: the seed of wigner_d_seed
// (wigner.py:117-136, norm from the host) and the three-term recurrence in the reference's
// operation order; out[(l - L) * count + i].
__global__ void wigner_rows_eval_kernel(int B, int m, int mp, double norm, const double* beta, long long count,
                                        double* out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double bt = beta[i];
  double s, c;
  sincos(0.5 * bt, &s, &c);
  double cur;
  const int am = abs(m), amp = abs(mp);
  if (am >= amp) cur = m >= 0 ? norm * pow(c, (double)(am + mp)) * pow(s, (double)(am - mp))
                              : norm * pow(c, (double)(am - mp)) * pow(-s, (double)(am + mp));
  else cur = mp >= 0 ? norm * pow(c, (double)(amp + m)) * pow(-s, (double)(amp - m))
                     : norm * pow(c, (double)(amp - m)) * pow(s, (double)(amp + m));
  const int L = max(am, amp);
  const double x = cos(bt);
  double prev = 0.0;
  out[i] = cur;
  for (int l = L; l < B - 1; ++l) {
    const double lp = l + 1.0;
    const double denom = sqrt((lp * lp - (double)m * m) * (lp * lp - (double)mp * mp));
    const double al = lp * (2.0 * l + 1.0) / denom;
    double shift = 0.0, cl = 0.0;
    if (l > 0) {
      shift = ((double)m * mp) / ((double)l * lp);
      cl = lp * sqrt(((double)l * l - (double)m * m) * ((double)l * l - (double)mp * mp)) / ((double)l * denom);
    }
    const double nx = al * (x - shift) * cur - cl * prev;
    out[(long long)(l + 1 - L) * count + i] = nx;
    prev = cur;
    cur = nx;
  }
}

}  // namespace so3

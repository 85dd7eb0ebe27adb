// Shared device helpers for the SO(3) FFT kernels (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace so3 {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// Flat l-major coefficient slot of (l, m, m') -- reference core.py:54-61.
__device__ __forceinline__ long long coeff_slot(int l, int m, int mp) {
  const long long L = l;
  return L * (4 * L * L - 1) / 3 + (long long)(m + l) * (2 * l + 1) + (mp + l);
}

// 32-bit form, valid while B(4B^2-1)/3 < 2^31 (B <= 812); the plan rejects larger B on
// the paths that use it.
__device__ __forceinline__ int coeff_slot32(int l, int m, int mp) {
  return (l * (4 * l * l - 1)) / 3 + (m + l) * (2 * l + 1) + (mp + l);
}

// The eight symmetry relations of reference wigner.py:244-256, in tag order:
// identity, negate_both, swap, swap_negate_both, negate_m, negate_mp,
// swap_negate_m, swap_negate_mp.  Fields: reflect, sl, sm, smp, tm_m, tm_mp,
// tp_m, tp_mp.
struct Relation { int reflect, sl, sm, smp, tm_m, tm_mp, tp_m, tp_mp; };

__device__ __forceinline__ Relation relation(int tag) {
  switch (tag) {
    case 0: return {0, 0, 0, 0, 1, 0, 0, 1};
    case 1: return {0, 0, 1, 1, -1, 0, 0, -1};
    case 2: return {0, 0, 1, 1, 0, 1, 1, 0};
    case 3: return {0, 0, 0, 0, 0, -1, -1, 0};
    case 4: return {1, 1, 0, 1, -1, 0, 0, 1};
    case 5: return {1, 1, 1, 0, 1, 0, 0, -1};
    case 6: return {1, 1, 0, 1, 0, -1, 1, 0};
    default: return {1, 1, 1, 0, 0, 1, -1, 0};
  }
}

// One member of a symmetry cluster (reference schedule.py:115-133).
struct Member {
  int valid;     // 0 for the padding slots of 1- and 4-member clusters
  int reflect;   // member reads the base at pi - beta (reversed j)
  int sl;        // sign exponent coefficient of l
  int par0;      // parity of sm*m + smp*m'
  int pm, pmp;   // member order pair
  long long row; // (pmp mod n) * n + (pm mod n): row of the [m'][m][j] spectrum
};

// Tags per cluster kind: origin {0}; axis {0,1,2,3}; diagonal {0,1,4,5}; full {0..7}.
__device__ __forceinline__ Member make_member(int m, int mp, int k, int n) {
  Member r;
  int tag;
  if (m == 0) tag = (k == 0) ? 0 : -1;
  else if (mp == 0) tag = (k < 4) ? k : -1;
  else if (mp == m) tag = (k < 2) ? k : (k < 4 ? k + 2 : -1);
  else tag = k;
  if (tag < 0) { r.valid = 0; r.reflect = 0; r.sl = 0; r.par0 = 0; r.pm = 0; r.pmp = 0; r.row = 0; return r; }
  const Relation R = relation(tag);
  r.valid = 1;
  r.reflect = R.reflect;
  r.sl = R.sl;
  r.par0 = (R.sm * m + R.smp * mp) & 1;
  r.pm = R.tm_m * m + R.tm_mp * mp;
  r.pmp = R.tp_m * m + R.tp_mp * mp;
  // |pm|, |pm'| < B = n / 2: the bin is the order itself or the order + n (no integer modulo: two
  // runtime `%` cost ~80 instructions in every DWT prologue)
  const int bm = r.pm < 0 ? r.pm + n : r.pm, bmp = r.pmp < 0 ? r.pmp + n : r.pmp;
  r.row = (long long)bmp * n + bm;
  return r;
}

// Wigner-d seed d^L_{m,m'}(beta_j), L = m >= m' >= 0 (reference wigner.py:117-128):
//   norm * cos(beta/2)^(m+m') * sin(beta/2)^(m-m'),
// evaluated as exp(log norm + (m+m') log c + (m-m') log s) in double-double so
// that neither the huge norm nor the tiny powers over/underflow on their own.
// lnorm = (hi, lo); lcs = (log c hi, log c lo, log s hi, log s lo) from the plan.
__device__ __forceinline__ double seed_value(int m, int mp, double2 lnorm, double4 lcs) {
  const double A = (double)(m + mp), Bx = (double)(m - mp);
  const double p1 = A * lcs.x;
  const double e1 = fma(A, lcs.x, -p1) + A * lcs.y;
  const double p2 = Bx * lcs.z;
  const double e2 = fma(Bx, lcs.z, -p2) + Bx * lcs.w;
  double s = p1 + p2;
  double bb = s - p1;
  double err = (p1 - (s - bb)) + (p2 - bb);
  const double s2 = s + lnorm.x;
  bb = s2 - s;
  err += (s - (s2 - bb)) + (lnorm.x - bb);
  err += e1 + e2 + lnorm.y;
  const double hi = s2 + err;
  const double lo = err - (hi - s2);
  if (hi < -745.5) return 0.0;
  return exp(hi) * (1.0 + lo);
}

// Recurrence coefficients of reference wigner.py:165-174 for the step l -> l+1, stored as
// (A, C+, C) with C+ = A (1 - shift) = A (l(l+1) - m m') / (l(l+1)) (integer numerator, so
// C+ carries no cancellation) for  d^{l+1} = t_l d^l - C d^{l-1},  t_l = A (x - shift).
__device__ __forceinline__ double3 recurrence_coeffs(int l, int m, int mp) {
  const double lp = (double)(l + 1);
  const double dl = (double)l;
  const double denom = sqrt((lp * lp - (double)m * m) * (lp * lp - (double)mp * mp));
  const double a = (lp * (2.0 * dl + 1.0)) / denom;
  double cplus = a, c = 0.0;
  if (l > 0) {
    const double ll1 = dl * lp;   // l(l+1), exact
    cplus = a * ((ll1 - (double)m * (double)mp) / ll1);
    c = (lp * sqrt((dl * dl - (double)m * m) * (dl * dl - (double)mp * mp))) / (dl * denom);
  }
  return make_double3(a, cplus, c);
}

// t_l = A (x - shift) without a rounded cos(beta): the plan stores v_j with x_j = 1 + v_j for
// beta_j < pi/2 (v = -2 sin^2(beta/2)) and x_j = -1 + v_j above (v = 2 cos^2(beta/2)), both to
// full relative precision, so t = A v + C+ (lower half) or A v + C+ - 2A (upper half).  Near the
// poles the reference's rounded cos(beta) moves d^l by l^2/2 ulps (P_l'(1) = l(l+1)/2); this
// form does not (oracle/extended.py measures it).
__device__ __forceinline__ double rec_t(double alpha, double cplus, double v, bool upper) {
  return fma(alpha, v, upper ? fma(-2.0, alpha, cplus) : cplus);
}

}  // namespace so3

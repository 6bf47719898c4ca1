// Exact restatement of the reference GeLU (tensor.py:76-83 over scipy's
// Cephes erf), shared by the row kernels.
#pragma once
#include "zq_common.cuh"

namespace zq {

// scipy.special.erf (scipy 1.18, the reference's erf: tensor.py:15, :83) is the
// Cephes ndtr.c algorithm: odd symmetry, a (4,5) rational in x^2 on |x| <= 1,
// and 1 - erfc(x) above, with erfc = exp(-x^2) * P8(x)/Q8(x) (x < 8) or
// exp(-x^2) * R5(x)/S6(x).  Restated here op for op (round-to-nearest, no
// contraction) so the f64 result matches scipy bit for bit; this matters for
// x << 0, where 1 + erf(x) cancels and the last bits of erf survive into the
// float32 GeLU.  Verified identical to scipy on 5.5e5 points (tools/erf_check.py).
__device__ __forceinline__ double polevl_d(double x, const double* c, int n) {
  double a = c[0];
#pragma unroll
  for (int i = 1; i <= n; ++i) a = __dadd_rn(__dmul_rn(a, x), c[i]);
  return a;
}
__device__ __forceinline__ double p1evl_d(double x, const double* c, int n) {
  double a = __dadd_rn(x, c[0]);
#pragma unroll
  for (int i = 1; i < n; ++i) a = __dadd_rn(__dmul_rn(a, x), c[i]);
  return a;
}
static __constant__ double kErfT[5] = {9.60497373987051638749E0, 9.00260197203842689217E1,
                       2.23200534594684319226E3, 7.00332514112805075473E3,
                       5.55923013010394962768E4};
static __constant__ double kErfU[5] = {3.35617141647503099647E1, 5.21357949780152679795E2,
                       4.59432382970980127987E3, 2.26290000613890934246E4,
                       4.92673942608635921086E4};
static __constant__ double kErfP[9] = {2.46196981473530512524E-10, 5.64189564831068821977E-1,
                       7.46321056442269912687E0,   4.86371970985681366614E1,
                       1.96520832956077098242E2,   5.26445194995477358631E2,
                       9.34528527171957607540E2,   1.02755188689515710272E3,
                       5.57535335369399327526E2};
static __constant__ double kErfQ[8] = {1.32281951154744992508E1, 8.67072140885989742329E1,
                       3.54937778887819891062E2, 9.75708501743205489753E2,
                       1.82390916687909736289E3, 2.24633760818710981792E3,
                       1.65666309194161350182E3, 5.57535340817727675546E2};
static __constant__ double kErfR[6] = {5.64189583547755073984E-1, 1.27536670759978104416E0,
                       5.01905042251180477414E0,  6.16021097993053585195E0,
                       7.40974269950448939160E0,  2.97886665372100240670E0};
static __constant__ double kErfS[6] = {2.26052863220117276590E0, 9.39603524938001434673E0,
                       1.20489539808096656605E1, 1.70814450747565897222E1,
                       9.60896809063285878198E0, 3.36907645100081516050E0};

__device__ __forceinline__ double cephes_erf(double x) {
  const double kMaxLog = 7.09782712893383996843E2;
  const bool neg = x < 0.0;
  const double a = fabs(x);
  double r;
  if (a <= 1.0) {
    const double z = __dmul_rn(a, a);
    r = __ddiv_rn(__dmul_rn(a, polevl_d(z, kErfT, 4)), p1evl_d(z, kErfU, 5));
  } else {
    // erfc(a) for a > 1
    const double z = -__dmul_rn(a, a);
    double ec;
    if (z < -kMaxLog) {
      ec = 0.0;
    } else {
      const double e = exp(z);
      double p, q;
      if (a < 8.0) {
        p = polevl_d(a, kErfP, 8);
        q = p1evl_d(a, kErfQ, 8);
      } else {
        p = polevl_d(a, kErfR, 5);
        q = p1evl_d(a, kErfS, 6);
      }
      ec = __ddiv_rn(__dmul_rn(e, p), q);
    }
    r = __dsub_rn(1.0, ec);
  }
  return neg ? -r : r;
}

// tensor.py:76-83: f32( (x64 * 0.5) * (1.0 + erf(x64 * (1/sqrt 2))) ), every op
// in f64 round-to-nearest (no contraction), one final rounding to f32.
struct GeluOp {
  static constexpr bool kWarpOk = false;
  __device__ __forceinline__ float operator()(float x) const {
    const double kInvSqrt2 = 0x1.6a09e667f3bccp-1;  // 1.0 / math.sqrt(2.0) in Python
    double x64 = (double)x;
    double e = cephes_erf(__dmul_rn(x64, kInvSqrt2));
    return __double2float_rn(__dmul_rn(__dmul_rn(x64, 0.5), __dadd_rn(1.0, e)));
  }
};


}  // namespace zq

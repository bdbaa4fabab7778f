// Shared device helpers for the citywalk B200 kernels (sm_100a).
//
// Parity build: the library is compiled with -fmad=false so that every
// float64 expression rounds exactly like the numpy reference (one rounding
// per ufunc).  Places where the reference goes through OpenBLAS and gets a
// fused multiply-add use the explicit fma below (DESIGN.md §3 lists the
// measured formulas).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define CW_DEV __device__ __forceinline__
#define CW_HD __host__ __device__ __forceinline__

namespace cw {

constexpr double kEps = 1e-12;            // field.py:19, orca.py:14
constexpr double kSqrt2 = 1.4142135623730951;  // float(np.sqrt(2.0))
constexpr double kTwoPi = 6.283185307179586;   // 2 * np.pi

// Cell labels (urbangen/types.py:64-69) and zones (types.py:33-39).
enum Label : uint8_t { L_OBSTACLE = 0, L_ROADWAY = 1, L_WALKABLE = 2, L_NONWALK = 3 };
enum Zone : uint8_t { Z_SIDEWALK = 0, Z_CROSSWALK = 1, Z_PLAZA = 2, Z_BUILDING = 3,
                      Z_VEGETATION = 4, Z_ROADWAY = 5 };

CW_HD uint8_t zone_to_label(uint8_t z) {
  // types.py:72-79
  return z <= Z_PLAZA ? L_WALKABLE : (z == Z_BUILDING ? L_OBSTACLE
                                      : (z == Z_VEGETATION ? L_NONWALK : L_ROADWAY));
}

// numpy a @ b for float64 2-vectors: OpenBLAS ddot = fma(a1, b1, a0*b0).
CW_DEV double dot2_blas(double a0, double a1, double b0, double b1) {
  return __fma_rn(a1, b1, __dmul_rn(a0, b0));
}

// glibc 2.39 __hypot (sysdeps/ieee754/dbl-64/e_hypot.c, non-FMA kernel);
// numpy's np.hypot calls it through libm (verified bit-exact).
CW_DEV double glibc_hypot(double x, double y) {
  double ax = fabs(x), ay = fabs(y);
  if (ax < ay) { double t = ax; ax = ay; ay = t; }
  if (!(ay > ax * 0x1p-54)) return ax + ay;  // also ay == 0
  const double SCALE = 0x1p-600, LARGE = 0x1p511, TINY = 0x1p-511;
  double sc = 1.0;
  if (ax > LARGE) { ax *= SCALE; ay *= SCALE; sc = 1.0 / SCALE; }
  else if (ay < TINY) { ax /= SCALE; ay /= SCALE; sc = SCALE; }
  double h = sqrt(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= 2.0 * ay) {
    double de = h - ay;
    t1 = ax * (2.0 * de - ax);
    t2 = (de - 2.0 * (ax - ay)) * de;
  } else {
    double de = h - ax;
    t1 = 2.0 * de * (ax - 2.0 * ay);
    t2 = (4.0 * de - ay) * ay + de * de;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h * sc;
}

// Python int(x) / numpy astype(int64) truncation of a finite double.
CW_DEV long long trunc_ll(double x) { return (long long)x; }

// x / h, as a multiplication when h is a power of two (the default horizons 2 s / 1 s,
// grid resolutions 0.125 / 0.25 m): x * 2^-k and x / 2^k are the correctly rounded
// values of the same real number, so the result is bit-identical and a long
// double-precision division leaves the dependency chain.
CW_DEV double div_h(double x, double h) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(h);
  const unsigned long long ex = (b >> 52) & 0x7FFull;
  if ((b & 0x800FFFFFFFFFFFFFull) == 0ull && ex >= 1ull && ex <= 2045ull)
    return x * __longlong_as_double((long long)((2046ull - ex) << 52));
  return x / h;
}

CW_DEV long long clampll(long long v, long long lo, long long hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}


// ---------------------------------------------------------------- correctly rounded sin/cos
// The reference's trig (np.cos / np.sin on float64 = glibc libm) is accurate to
// within one ulp and rounds correctly in all but rare cases; CUDA's sincos has a
// 2-ulp bound.  cr_sincos evaluates sin and cos in double-double (Cody-Waite
// reduction by pi/2 in four parts, Taylor series to degree 27 on |r| <= pi/4 with the
// leading terms in double-double, error < 2^-73 relative) and rounds once: the correctly rounded
// value -- glibc's result whenever glibc rounds correctly.  Used where a trig
// value feeds a geometric decision (footprint corners, SAT, cell tests).
struct DD { double hi, lo; };
CW_DEV DD dd_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b), bb = __dsub_rn(s, a);
  return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
CW_DEV DD dd_fast(double a, double b) {   // |a| >= |b|
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
CW_DEV DD dd_add(DD a, DD b) {
  DD s = dd_two_sum(a.hi, b.hi);
  return dd_fast(s.hi, __dadd_rn(s.lo, __dadd_rn(a.lo, b.lo)));
}
CW_DEV DD dd_mul(DD a, DD b) {
  const double p = __dmul_rn(a.hi, b.hi);
  const double e = __fma_rn(a.hi, b.hi, -p);
  return dd_fast(p, __dadd_rn(e, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi))));
}

// 1/n! as double-doubles (hi, lo), n = 0..27
static __constant__ double kInvFactHi[28] = {
    0x1p+0, 0x1p+0, 0x1p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5, 0x1.1111111111111p-7,
    0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19,
    0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33,
    0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-41, 0x1.ae7f3e733b81fp-45, 0x1.952c77030ad4ap-49,
    0x1.6827863b97d97p-53, 0x1.2f49b46814157p-57, 0x1.e542ba4020225p-62, 0x1.71b8ef6dcf572p-66,
    0x1.0ce396db7f853p-70, 0x1.761b41316381ap-75, 0x1.f2cf01972f578p-80, 0x1.3f3ccdd165fa9p-84,
    0x1.88e85fc6a4e5ap-89, 0x1.d1ab1c2dccea3p-94};
static __constant__ double kInvFactLo[9] = {
    0.0, 0.0, 0.0, 0x1.5555555555555p-57, 0x1.5555555555555p-59, 0x1.1111111111111p-63,
    -0x1.f49f49f49f49fp-65, 0x1.a01a01a01a01ap-73, 0x1.a01a01a01a01ap-76};

// sin and cos of x in double-double, rounded once.  Reduction by pi/2 in four parts;
// on |r| <= pi/4 the series in y = -r^2 keeps its leading terms (sin/r: y^0..y^3,
// cos: y^0..y^4) in double-double and evaluates the rest (from r^9 resp. r^10 on,
// magnitude < 3e-6) in double: total relative error < 2^-73, so the result is the
// correctly rounded value but in cases within 2^-73 of a rounding midpoint.
CW_DEV void cr_sincos(double x, double* s_out, double* c_out) {
  if (!(fabs(x) < 0x1p+20)) { sincos(x, s_out, c_out); return; }   // not used by the path
  // pi/2 = P1 + P2 + P3 + P4 (P1..P3 carry 33 bits: k * Pi is exact for |k| < 2^20)
  const double P1 = 0x1.921fb544p+0, P2 = 0x1.0b4611a6p-34, P3 = 0x1.3198a2ep-69, P4 = 0x1.b839a252049c1p-104;
  const double k = rint(__dmul_rn(x, 0x1.45f306dc9c883p-1));   // x * 2/pi
  DD r = dd_two_sum(x, -__dmul_rn(k, P1));
  r = dd_add(r, DD{-__dmul_rn(k, P2), 0.0});
  r = dd_add(r, DD{-__dmul_rn(k, P3), 0.0});
  r = dd_add(r, DD{-__dmul_rn(k, P4), 0.0});
  const DD r2 = dd_mul(r, r);
  const DD y{-r2.hi, -r2.lo};
  // double tails: sin/r terms y^4..y^13 (1/9! .. 1/27!), cos terms y^5..y^13 (1/10! .. 1/26!)
  double ts = kInvFactHi[27], tc = kInvFactHi[26];
#pragma unroll
  for (int n = 25; n >= 9; n -= 2) ts = __dadd_rn(__dmul_rn(ts, y.hi), kInvFactHi[n]);
#pragma unroll
  for (int n = 24; n >= 10; n -= 2) tc = __dadd_rn(__dmul_rn(tc, y.hi), kInvFactHi[n]);
  DD ps{ts, 0.0}, pc{tc, 0.0};
#pragma unroll
  for (int n = 7; n >= 1; n -= 2) ps = dd_add(dd_mul(ps, y), DD{kInvFactHi[n], kInvFactLo[n]});
#pragma unroll
  for (int n = 8; n >= 0; n -= 2) pc = dd_add(dd_mul(pc, y), DD{kInvFactHi[n], kInvFactLo[n]});
  const DD sr = dd_mul(ps, r);
  const double sv = __dadd_rn(sr.hi, sr.lo), cv = __dadd_rn(pc.hi, pc.lo);
  const int q = (int)((long long)k & 3);
  if (q == 0) { *s_out = sv; *c_out = cv; }
  else if (q == 1) { *s_out = cv; *c_out = -sv; }
  else if (q == 2) { *s_out = -sv; *c_out = -cv; }
  else { *s_out = -cv; *c_out = sv; }
}

}  // namespace cw

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

CW_DEV long long clampll(long long v, long long lo, long long hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

}  // namespace cw

// jets.cuh -- forward-mode derivative carriers for the device operators.
//
// R^(2)_h is the time derivative of R^(1)_h along w_t = sigma, so
// every operator of the hot path is R^(1)_h evaluated on a truncated Taylor
// "jet" of the state:
//   double : R1(W)
//   J1     : v + a e1                  -> R1, R2(W, a)                (residual, K v)
//   J2     : v + a e1 + b e2           -> R1, R2(W, a), R2(W, b)      (FD JVP, K u/K v)
//   HJ     : v + a e1 + b e2 + c e1e2  -> ... + R1''[a,b] + R1' c     (EXACT JVP)
// with e1^2 = e2^2 = 0 (J2 drops the e1e2 term).  The flux code in physics.cuh
// is written once, templated on the carrier.
#pragma once
#include <cuda_runtime.h>

struct J1 {
  double v, a;
};
struct J2 {
  double v, a, b;
};
struct HJ {
  double v, a, b, c;
};

// ---- plain double helpers ---------------------------------------------------
__device__ __forceinline__ double jval(double x) { return x; }
__device__ __forceinline__ double jabs(double x) { return x >= 0.0 ? x : -x; }  // sign(0)=+1
__device__ __forceinline__ double jsqrt(double x) { return sqrt(x); }
__device__ __forceinline__ double jmax(double a, double b) { return a >= b ? a : b; }  // tie -> a

// ---- J1 -------------------------------------------------------------------------
__device__ __forceinline__ J1 operator+(J1 x, J1 y) { return {x.v + y.v, x.a + y.a}; }
__device__ __forceinline__ J1 operator-(J1 x, J1 y) { return {x.v - y.v, x.a - y.a}; }
__device__ __forceinline__ J1 operator-(J1 x) { return {-x.v, -x.a}; }
__device__ __forceinline__ J1 operator*(J1 x, J1 y) { return {x.v * y.v, x.v * y.a + x.a * y.v}; }
__device__ __forceinline__ J1 operator*(double s, J1 x) { return {s * x.v, s * x.a}; }
__device__ __forceinline__ J1 operator*(J1 x, double s) { return {s * x.v, s * x.a}; }
__device__ __forceinline__ J1 operator+(J1 x, double s) { return {x.v + s, x.a}; }
__device__ __forceinline__ J1 operator+(double s, J1 x) { return {x.v + s, x.a}; }
__device__ __forceinline__ J1 operator-(J1 x, double s) { return {x.v - s, x.a}; }
__device__ __forceinline__ J1 operator-(double s, J1 x) { return {s - x.v, -x.a}; }
__device__ __forceinline__ J1 operator/(J1 x, J1 y) {
  double r = 1.0 / y.v, q = x.v / y.v;
  return {q, (x.a - q * y.a) * r};
}
__device__ __forceinline__ J1 operator/(J1 x, double s) { return {x.v / s, x.a / s}; }
__device__ __forceinline__ J1 operator/(double s, J1 y) {
  double q = s / y.v, r = 1.0 / y.v;
  return {q, -q * y.a * r};
}
__device__ __forceinline__ double jval(J1 x) { return x.v; }
__device__ __forceinline__ J1 jabs(J1 x) { return x.v >= 0.0 ? x : J1{-x.v, -x.a}; }
// sqrt of a jet from one reciprocal square root: s = x r, s' = x' r / 2 (no division)
__device__ __forceinline__ J1 jsqrt(J1 x) {
  const double r = rsqrt(x.v);
  return {x.v * r, 0.5 * r * x.a};
}
__device__ __forceinline__ J1 jmax(J1 x, J1 y) { return x.v >= y.v ? x : y; }

// ---- J2 -------------------------------------------------------------------------
__device__ __forceinline__ J2 operator+(J2 x, J2 y) { return {x.v + y.v, x.a + y.a, x.b + y.b}; }
__device__ __forceinline__ J2 operator-(J2 x, J2 y) { return {x.v - y.v, x.a - y.a, x.b - y.b}; }
__device__ __forceinline__ J2 operator-(J2 x) { return {-x.v, -x.a, -x.b}; }
__device__ __forceinline__ J2 operator*(J2 x, J2 y) {
  return {x.v * y.v, x.v * y.a + x.a * y.v, x.v * y.b + x.b * y.v};
}
__device__ __forceinline__ J2 operator*(double s, J2 x) { return {s * x.v, s * x.a, s * x.b}; }
__device__ __forceinline__ J2 operator*(J2 x, double s) { return {s * x.v, s * x.a, s * x.b}; }
__device__ __forceinline__ J2 operator+(J2 x, double s) { return {x.v + s, x.a, x.b}; }
__device__ __forceinline__ J2 operator+(double s, J2 x) { return {x.v + s, x.a, x.b}; }
__device__ __forceinline__ J2 operator-(J2 x, double s) { return {x.v - s, x.a, x.b}; }
__device__ __forceinline__ J2 operator-(double s, J2 x) { return {s - x.v, -x.a, -x.b}; }
__device__ __forceinline__ J2 operator/(J2 x, J2 y) {
  double r = 1.0 / y.v, q = x.v / y.v;
  return {q, (x.a - q * y.a) * r, (x.b - q * y.b) * r};
}
__device__ __forceinline__ J2 operator/(J2 x, double s) { return {x.v / s, x.a / s, x.b / s}; }
__device__ __forceinline__ J2 operator/(double s, J2 y) {
  double q = s / y.v, r = 1.0 / y.v;
  return {q, -q * y.a * r, -q * y.b * r};
}
__device__ __forceinline__ double jval(J2 x) { return x.v; }
__device__ __forceinline__ J2 jabs(J2 x) { return x.v >= 0.0 ? x : J2{-x.v, -x.a, -x.b}; }
__device__ __forceinline__ J2 jsqrt(J2 x) {
  const double r = rsqrt(x.v), h = 0.5 * r;
  return {x.v * r, h * x.a, h * x.b};
}
__device__ __forceinline__ J2 jmax(J2 x, J2 y) { return x.v >= y.v ? x : y; }

// ---- HJ (hyper-dual) ------------------------------------------------------------
__device__ __forceinline__ HJ operator+(HJ x, HJ y) { return {x.v + y.v, x.a + y.a, x.b + y.b, x.c + y.c}; }
__device__ __forceinline__ HJ operator-(HJ x, HJ y) { return {x.v - y.v, x.a - y.a, x.b - y.b, x.c - y.c}; }
__device__ __forceinline__ HJ operator-(HJ x) { return {-x.v, -x.a, -x.b, -x.c}; }
__device__ __forceinline__ HJ operator*(HJ x, HJ y) {
  return {x.v * y.v, x.v * y.a + x.a * y.v, x.v * y.b + x.b * y.v,
          x.v * y.c + x.a * y.b + x.b * y.a + x.c * y.v};
}
__device__ __forceinline__ HJ operator*(double s, HJ x) { return {s * x.v, s * x.a, s * x.b, s * x.c}; }
__device__ __forceinline__ HJ operator*(HJ x, double s) { return {s * x.v, s * x.a, s * x.b, s * x.c}; }
__device__ __forceinline__ HJ operator+(HJ x, double s) { return {x.v + s, x.a, x.b, x.c}; }
__device__ __forceinline__ HJ operator+(double s, HJ x) { return {x.v + s, x.a, x.b, x.c}; }
__device__ __forceinline__ HJ operator-(HJ x, double s) { return {x.v - s, x.a, x.b, x.c}; }
__device__ __forceinline__ HJ operator-(double s, HJ x) { return {s - x.v, -x.a, -x.b, -x.c}; }
// f(x) with f0, f1 = f', f2 = f'': (f0, f1 a, f1 b, f1 c + f2 a b)
__device__ __forceinline__ HJ hj_chain(HJ x, double f0, double f1, double f2) {
  return {f0, f1 * x.a, f1 * x.b, f1 * x.c + f2 * x.a * x.b};
}
__device__ __forceinline__ HJ hj_recip(HJ y) {
  double r = 1.0 / y.v;
  return hj_chain(y, r, -r * r, 2.0 * r * r * r);
}
__device__ __forceinline__ HJ operator/(HJ x, HJ y) {
  HJ q = x * hj_recip(y);
  q.v = x.v / y.v;
  return q;
}
__device__ __forceinline__ HJ operator/(HJ x, double s) { return {x.v / s, x.a / s, x.b / s, x.c / s}; }
__device__ __forceinline__ HJ operator/(double s, HJ y) {
  HJ q = s * hj_recip(y);
  q.v = s / y.v;
  return q;
}
__device__ __forceinline__ double jval(HJ x) { return x.v; }
__device__ __forceinline__ HJ jabs(HJ x) { return x.v >= 0.0 ? x : -x; }
__device__ __forceinline__ HJ jsqrt(HJ x) {
  double s = sqrt(x.v);
  return hj_chain(x, s, 0.5 / s, -0.25 / (s * x.v));
}
__device__ __forceinline__ HJ jmax(HJ x, HJ y) { return x.v >= y.v ? x : y; }

// 1/x with one fp64 division per carrier
__device__ __forceinline__ double jrecip(double x) { return 1.0 / x; }
__device__ __forceinline__ J1 jrecip(J1 x) {
  const double r = 1.0 / x.v;
  return {r, -r * r * x.a};
}
__device__ __forceinline__ J2 jrecip(J2 x) {
  const double r = 1.0 / x.v, r2 = -r * r;
  return {r, r2 * x.a, r2 * x.b};
}
__device__ __forceinline__ HJ jrecip(HJ x) { return hj_recip(x); }

template <class T> __device__ __forceinline__ T jconst(double v);
template <> __device__ __forceinline__ double jconst<double>(double v) { return v; }
template <> __device__ __forceinline__ J1 jconst<J1>(double v) { return {v, 0.0}; }
template <> __device__ __forceinline__ J2 jconst<J2>(double v) { return {v, 0.0, 0.0}; }
template <> __device__ __forceinline__ HJ jconst<HJ>(double v) { return {v, 0.0, 0.0, 0.0}; }

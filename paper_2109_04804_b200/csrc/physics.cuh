// physics.cuh -- point-wise fluxes, templated on the jet carrier (jets.cuh).
//
//  advection : F_d = a_d w
//  Euler     : F_x = (rho u, rho u^2 + p, rho u v, u (E + p)), p = (gamma-1)(E - rho|v|^2/2)
//              (eq:Euler; configs: reference Mach number eps = 1, reading R18)
//  LLF       : f* = 1/2 (F_d(wL) + F_d(wR)) + 1/2 lam (wL - wR),
//              lam = max(|v_L.e_d| + c_L, |v_R.e_d| + c_R)  (reading R3; the paper's
//              eq:Riemann is the global-lambda variant).  Canonical orientation:
//              L = element on the -e_d side, normal +e_d; ties take L.
//  GLF       : (pp.glf, HBPDC_GLF_PAPER) the paper's eq:Riemann literally:
//              f* = 1/2 (F_d(wL) + F_d(wR)) + Lambda (wL - wR), the full Lambda on the jump
//              (no 1/2), Lambda = diag(1/eps, 1, 1, 1/eps), advection |a_d|.
//  eps       : reference Mach number (mach_eps): momentum flux p / eps^2, p with eps^2 in
//              the kinetic energy, wave speed |v.n| + c / eps (Euler; NS only at eps = 1).
//  NS        : viscous flux F^v with BR1 gradients (reading R19).
#pragma once
#include "jets.cuh"

struct PhysParams {
  double ax, ay;         // advection velocity (az: 3D, below)
  double gamma;
  double mu, lamT, Rgas; // NS: viscosity, heat conductivity c_p mu / Pr, R = 1/gamma
  int glf;               // 1: the paper's global LF flux (Lambda = diag(1/eps,1,1,1/eps)), 0: LLF
  double ieps, eps2, ieps2;   // reference Mach number eps of eq:Euler: 1/eps, eps^2, 1/eps^2
  double eta_br2;        // NS BR2 lifting: eta (face gradients, lift_kernel)
  double az;             // advection velocity, z component (3D)
};

// EQ: 0 advection, 1 Euler 2D, 2 Navier-Stokes 2D, 3 Euler 3D (NEXT-4: (rho, rho u, rho v, rho w, E))
template <int EQ> struct NVars { static constexpr int value = 4; };
template <> struct NVars<0> { static constexpr int value = 1; };
template <> struct NVars<3> { static constexpr int value = 5; };

__host__ __device__ inline double adv_speed(const struct PhysParams& pp, int d) {
  return d == 0 ? pp.ax : (d == 1 ? pp.ay : pp.az);
}

// Euler primitives of a node state, computed once and shared by both flux
// directions and the wave speed: one jet reciprocal per state.
template <class T> struct EulerPrim {
  T u, v, p, H, rinv;   // velocity, pressure, E + p, 1/rho
  T pe;                 // p / eps^2 (momentum flux, eq:Euler)
};

template <class T>
__device__ __forceinline__ EulerPrim<T> euler_prim(const PhysParams& pp, const T* w) {
  EulerPrim<T> q;
  q.rinv = jrecip(w[0]);
  q.u = w[1] * q.rinv;
  q.v = w[2] * q.rinv;
  q.p = (pp.gamma - 1.0) * (w[3] - (0.5 * pp.eps2) * (w[1] * q.u + w[2] * q.v));
  q.H = w[3] + q.p;
  q.pe = pp.ieps2 * q.p;
  return q;
}

// inviscid flux in direction d from the primitives
template <class T>
__device__ __forceinline__ void euler_flux(const T* w, const EulerPrim<T>& q, int d, T* F) {
  const T vn = d == 0 ? q.u : q.v;
  F[0] = d == 0 ? w[1] : w[2];
  F[1] = d == 0 ? w[1] * vn + q.pe : w[1] * vn;
  F[2] = d == 1 ? w[2] * vn + q.pe : w[2] * vn;
  F[3] = vn * q.H;
}

// ---- 3D Euler (eq:Euler with three momentum components; the paper's 3D case P:1080-1093)
template <class T> struct EulerPrim3 {
  T u, v, w, p, H, rinv, pe;
};

template <class T>
__device__ __forceinline__ EulerPrim3<T> euler3_prim(const PhysParams& pp, const T* w) {
  EulerPrim3<T> q;
  q.rinv = jrecip(w[0]);
  q.u = w[1] * q.rinv;
  q.v = w[2] * q.rinv;
  q.w = w[3] * q.rinv;
  q.p = (pp.gamma - 1.0) * (w[4] - (0.5 * pp.eps2) * (w[1] * q.u + w[2] * q.v + w[3] * q.w));
  q.H = w[4] + q.p;
  q.pe = pp.ieps2 * q.p;
  return q;
}

template <class T>
__device__ __forceinline__ void euler3_flux(const T* w, const EulerPrim3<T>& q, int d, T* F) {
  const T vn = d == 0 ? q.u : (d == 1 ? q.v : q.w);
  F[0] = w[1 + d];
  F[1] = d == 0 ? w[1] * vn + q.pe : w[1] * vn;
  F[2] = d == 1 ? w[2] * vn + q.pe : w[2] * vn;
  F[3] = d == 2 ? w[3] * vn + q.pe : w[3] * vn;
  F[4] = vn * q.H;
}

template <class T>
__device__ __forceinline__ T euler3_speed(const PhysParams& pp, const EulerPrim3<T>& q, int d) {
  return jabs(d == 0 ? q.u : (d == 1 ? q.v : q.w)) + pp.ieps * jsqrt(pp.gamma * q.p * q.rinv);
}

// inviscid flux in direction d
template <int EQ, class T>
__device__ __forceinline__ void phys_flux(const PhysParams& pp, const T* w, int d, T* F) {
  if constexpr (EQ == 0) {
    F[0] = adv_speed(pp, d) * w[0];
  } else if constexpr (EQ == 3) {
    euler3_flux(w, euler3_prim(pp, w), d, F);
  } else {
    euler_flux(w, euler_prim(pp, w), d, F);
  }
}

template <class T>
__device__ __forceinline__ T euler_speed(const PhysParams& pp, const EulerPrim<T>& q, int d) {
  return jabs(d == 0 ? q.u : q.v) + pp.ieps * jsqrt(pp.gamma * q.p * q.rinv);   // |v.n| + c / eps
}

// canonical LLF flux across a face with normal +e_d
template <int EQ, class T>
__device__ __forceinline__ void llf_flux(const PhysParams& pp, const T* wL, const T* wR, int d, T* f) {
  constexpr int NV = NVars<EQ>::value;
  T FL[NV], FR[NV];
  T lam;
  if constexpr (EQ == 0) {
    phys_flux<EQ>(pp, wL, d, FL);
    phys_flux<EQ>(pp, wR, d, FR);
    lam = jconst<T>(fabs(adv_speed(pp, d)));
  } else if constexpr (EQ == 3) {
    const EulerPrim3<T> qL = euler3_prim(pp, wL), qR = euler3_prim(pp, wR);
    euler3_flux(wL, qL, d, FL);
    euler3_flux(wR, qR, d, FR);
    lam = pp.glf ? jconst<T>(1.0) : jmax(euler3_speed(pp, qL, d), euler3_speed(pp, qR, d));
  } else {
    const EulerPrim<T> qL = euler_prim(pp, wL), qR = euler_prim(pp, wR);
    euler_flux(wL, qL, d, FL);
    euler_flux(wR, qR, d, FR);
    lam = pp.glf ? jconst<T>(1.0) : jmax(euler_speed(pp, qL, d), euler_speed(pp, qR, d));
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if (pp.glf) {       // eq:Riemann: full Lambda on the jump, no 1/2; Lambda = |a_d|,
                        // diag(1/eps, 1, 1, 1/eps)
      const double lv = EQ == 0 ? fabs(adv_speed(pp, d)) : ((v == 0 || v == NV - 1) ? pp.ieps : 1.0);
      f[v] = 0.5 * (FL[v] + FR[v]) + lv * (wL[v] - wR[v]);
    } else {
      f[v] = 0.5 * (FL[v] + FR[v]) + 0.5 * lam * (wL[v] - wR[v]);
    }
  }
}

// ---- Navier-Stokes ----------------------------------------------------------------
// gradient variables w_grad = (u, v, T), T = p / (rho R)  (eq:LiftingEq)
template <class T>
__device__ __forceinline__ void grad_vars(const PhysParams& pp, const T* w, T* g) {
  const T rho = w[0], mx = w[1], my = w[2], E = w[3];
  const T p = (pp.gamma - 1.0) * (E - 0.5 * (mx * mx + my * my) / rho);
  g[0] = mx / rho;
  g[1] = my / rho;
  g[2] = p / (rho * pp.Rgas);
}

// F^v_d(w, grad): gx = (u_x, v_x, T_x), gy = (u_y, v_y, T_y)
template <class T>
__device__ __forceinline__ void viscous_flux_uv(const PhysParams& pp, const T& u, const T& v, const T* gx,
                                                const T* gy, int d, T* Fv) {
  const T div = gx[0] + gy[1];
  const T txy = pp.mu * (gy[0] + gx[1]);
  Fv[0] = jconst<T>(0.0);
  if (d == 0) {
    const T txx = pp.mu * (2.0 * gx[0] - (2.0 / 3.0) * div);
    Fv[1] = txx;
    Fv[2] = txy;
    Fv[3] = txx * u + txy * v + pp.lamT * gx[2];
  } else {
    const T tyy = pp.mu * (2.0 * gy[1] - (2.0 / 3.0) * div);
    Fv[1] = txy;
    Fv[2] = tyy;
    Fv[3] = txy * u + tyy * v + pp.lamT * gy[2];
  }
}

template <class T>
__device__ __forceinline__ void viscous_flux(const PhysParams& pp, const T* w, const T* gx,
                                             const T* gy, int d, T* Fv) {
  const T rho = w[0];
  const T u = w[1] / rho, v = w[2] / rho;
  const T div = gx[0] + gy[1];
  const T txy = pp.mu * (gy[0] + gx[1]);
  Fv[0] = jconst<T>(0.0);
  if (d == 0) {
    const T txx = pp.mu * (2.0 * gx[0] - (2.0 / 3.0) * div);
    Fv[1] = txx;
    Fv[2] = txy;
    Fv[3] = txx * u + txy * v + pp.lamT * gx[2];
  } else {
    const T tyy = pp.mu * (2.0 * gy[1] - (2.0 / 3.0) * div);
    Fv[1] = txy;
    Fv[2] = tyy;
    Fv[3] = txy * u + tyy * v + pp.lamT * gy[2];
  }
}

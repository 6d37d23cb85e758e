// ops_kernels.cu -- instantiation and dispatch of the fused element operators,
// the BR1 lifting, and the BJ_ext block build (M_i = I - a1dt K_i + c2 K_i^2).
#include <algorithm>
#include <type_traits>
#include "modes.cuh"
#include "launch.h"

// This file is compiled twice: GLL nodes (the product configuration, also the
// public entry points) and, as ops_kernels_gl.cu with HBPDC_OPS_GL=1, the
// Gauss-Legendre instantiations (advection and Euler), reached through *_gl.
#ifndef HBPDC_OPS_GL
#define HBPDC_OPS_GL 0
#endif
#ifndef HBPDC_OPS_BR2
#define HBPDC_OPS_BR2 0       // 1: the Navier-Stokes operators with BR2 face gradients (ops_kernels*_br2.cu)
#endif
#ifndef HBPDC_OPS_3D
#define HBPDC_OPS_3D 0        // 1: the 3D hexahedral instantiations (ops_kernels_3d.cu, NEXT-4)
#endif
static constexpr bool kGL = HBPDC_OPS_GL;
static constexpr bool kBR2 = HBPDC_OPS_BR2;
using GeoK = GeoSel<kGL>;
template <bool B = false>
static GeoSel<kGL, B> geo_sel(const Geo& g) {
  GeoSel<kGL, B> s;
  static_cast<Geo&>(s) = g;
  return s;
}

template <int EQ, int DIM, int P, class Mode>
static cudaError_t run_op(const OpCfg& c, const Geo& g, const OpArgs& A) {
  constexpr int NODES = ipow(P, DIM);
  constexpr int EPB = epb_for(NODES);
  const int grid = (launch_elems(g) + EPB - 1) / EPB;
  if (grid == 0) return cudaSuccess;
  constexpr size_t smem = (size_t)EPB * slot_doubles<EQ, DIM, P, Mode>() * sizeof(double);
  if constexpr (smem > 48 * 1024) {
    static bool attr = false;       // once per instantiation (same value from any thread)
    if (!attr) {
      cudaFuncSetAttribute(op_kernel<EQ, DIM, P, Mode, EPB, kGL, kBR2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
  }
  op_kernel<EQ, DIM, P, Mode, EPB, kGL, kBR2><<<grid, EPB * NODES, smem, c.stream>>>(A, c.pp, geo_sel<kBR2>(g));
  hbpdc_count_launch();
  return cudaGetLastError();
}

template <int P, class Mode, int K>
static cudaError_t run_gtrace(const OpCfg& c, const Geo& g, const OpArgs& A, double* Tg) {
  const int total = g.nE * 4 * P;
  if (total == 0) return cudaSuccess;
  gtrace_kernel<P, Mode, K><<<(total + 127) / 128, 128, 0, c.stream>>>(A, c.pp, g, Tg);
  hbpdc_count_launch();
  return cudaGetLastError();
}

template <int P, class Mode, int K>
static cudaError_t run_lift(const OpCfg& c, const Geo& g, const OpArgs& A, double* G, double* Gf,
                            const double* gTg) {
  constexpr int NODES = P * P;
  constexpr int EPB = epb_for(NODES);
  const int grid = (launch_elems(g) + EPB - 1) / EPB;
  if (grid == 0) return cudaSuccess;
  if (Gf)
    lift_kernel<P, Mode, K, EPB, kGL, true><<<grid, EPB * NODES, 0, c.stream>>>(A, c.pp, geo_sel(g), G, Gf, gTg);
  else
    lift_kernel<P, Mode, K, EPB, kGL, false><<<grid, EPB * NODES, 0, c.stream>>>(A, c.pp, geo_sel(g), G, Gf, gTg);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// ---- BJ_ext build: columns of M_i via two element-local linearised applications
// K t = L(F'(W_b) t) with the neighbour traces frozen (no tangent), t = e_c then
// t = K e_c.  "element-internal influence only", block formula P:314.
struct KColArgs {
  const double* W;      // build state
  const double* gW;     // its ghost copy (halo), elements e >= nE
  const double* tan;    // shared-memory tangents, one m-vector per slot
  int m, nE;
  const double* S;      // BJ^H_ext: sigma at the build point (R1(W)), NULL otherwise
  const double* gS;     // its ghost copy
};

template <int EQ, int NODES> struct ModeKCol {
  static constexpr int NV = NVars<EQ>::value, NCH = 1;
  using Args = KColArgs;
  template <int K> using StateT = J1;
  struct State { NodeState<EQ, J1> s; };
  __device__ static void load(const Args& A, const Geo&, int e, int slot, int node, State& st, bool nbr) {
    for (int v = 0; v < NV; ++v) {
      const double w = e < A.nE ? A.W[(size_t)e * A.m + v * NODES + node]
                                : A.gW[(size_t)(e - A.nE) * A.m + v * NODES + node];
      st.s.w[v] = J1{w, nbr ? 0.0 : A.tan[slot * A.m + v * NODES + node]};
    }
  }
  template <int DIM>
  __device__ static void vol(const Args&, const PhysParams& pp, const State& st, double (&c)[DIM][NCH][NV]) {
    J1 F[DIM][NV];
    vol_flux_all<EQ, DIM>(pp, st.s, F);
    for (int d = 0; d < DIM; ++d)
      for (int v = 0; v < NV; ++v) c[d][0][v] = F[d][v].a;
  }
  static constexpr int NFP = 2, FPD = half_doubles<EQ, J1>();
  template <class G>
  __device__ static void face_part(const Args& A, const PhysParams& pp, const G& g, int e, int own, int nb,
                                   int nnode, int slot, bool plus, int d, int part, double* raw,
                                   int rs) {
    const bool use_own = (part == 0) == plus;
    State st;
    const int le = use_own ? e : nb;
    trace_load(g, use_own ? own : nnode, d, st,
               [=](int nd, State& s) { load(A, g, le, slot, nd, s, !use_own); }, le >= A.nE);
    half_flux<EQ, J1>(pp, st.s, d, raw, rs);
  }
  __device__ static void face_combine(const Args&, const PhysParams& pp, int d, const double* rL, const double* rR,
                                      int rs, double (&c)[NCH][NV]) {
    J1 f[NV];
    face_from_halves<EQ, J1>(pp, rL, rR, rs, d, f);
    for (int v = 0; v < NV; ++v) c[0][v] = f[v].a;
  }
};

// t = H e_c: the element block of dR2/dW at fixed sigma (BJ^H_ext),
// the e1e2 part of R1(W + e1 sigma + e2 t) with t on the own element only
// (neighbour states carry sigma but no W tangent: "element-internal influence only").
template <int EQ, int NODES> struct ModeHCol {
  static constexpr int NV = NVars<EQ>::value, NCH = 1;
  using Args = KColArgs;
  template <int K> using StateT = HJ;
  struct State { NodeState<EQ, HJ> s; };
  __device__ static void load(const Args& A, const Geo&, int e, int slot, int node, State& st, bool nbr) {
    for (int v = 0; v < NV; ++v) {
      const size_t k = e < A.nE ? (size_t)e * A.m + v * NODES + node : (size_t)(e - A.nE) * A.m + v * NODES + node;
      const double w = e < A.nE ? A.W[k] : A.gW[k];
      const double sg = e < A.nE ? A.S[k] : A.gS[k];
      st.s.w[v] = HJ{w, sg, nbr ? 0.0 : A.tan[slot * A.m + v * NODES + node], 0.0};
    }
  }
  template <int DIM>
  __device__ static void vol(const Args&, const PhysParams& pp, const State& st, double (&c)[DIM][NCH][NV]) {
    HJ F[DIM][NV];
    vol_flux_all<EQ, DIM>(pp, st.s, F);
    for (int d = 0; d < DIM; ++d)
      for (int v = 0; v < NV; ++v) c[d][0][v] = F[d][v].c;
  }
  static constexpr int NFP = 2, FPD = half_doubles<EQ, HJ>();
  template <class G>
  __device__ static void face_part(const Args& A, const PhysParams& pp, const G& g, int e, int own, int nb,
                                   int nnode, int slot, bool plus, int d, int part, double* raw,
                                   int rs) {
    const bool use_own = (part == 0) == plus;
    State st;
    const int le = use_own ? e : nb;
    trace_load(g, use_own ? own : nnode, d, st,
               [=](int nd, State& s) { load(A, g, le, slot, nd, s, !use_own); }, le >= A.nE);
    half_flux<EQ, HJ>(pp, st.s, d, raw, rs);
  }
  __device__ static void face_combine(const Args&, const PhysParams& pp, int d, const double* rL, const double* rR,
                                      int rs, double (&c)[NCH][NV]) {
    HJ f[NV];
    face_from_halves<EQ, HJ>(pp, rL, rR, rs, d, f);
    for (int v = 0; v < NV; ++v) c[0][v] = f[v].c;
  }
};

template <int EQ, int DIM, int P, int EPB, bool HESS>
__global__ void __launch_bounds__(EPB * ipow(P, DIM))
kbuild_kernel(const double* __restrict__ Wb, const double* __restrict__ gWb, const PhysParams pp, const GeoK g, double a1dt, double c2,
              double* __restrict__ M, int e0, const double* __restrict__ Sb, const double* __restrict__ gSb) {
  constexpr int NODES = ipow(P, DIM);
  constexpr int NV = NVars<EQ>::value;
  constexpr int m = NV * NODES;
  using Mode = ModeKCol<EQ, NODES>;
  constexpr int SLOT = HESS ? std::max(slot_doubles<EQ, DIM, P, Mode>(), slot_doubles<EQ, DIM, P, ModeHCol<EQ, NODES>>())
                            : slot_doubles<EQ, DIM, P, Mode>();
  extern __shared__ __align__(16) double sdyn[];
  double* sF = sdyn;                  // EPB * SLOT
  double* stan = sdyn + EPB * SLOT;   // EPB * m
  const int slot = threadIdx.x / NODES, node = threadIdx.x % NODES;
  const int e = e0 + blockIdx.x;
  double* Me = M + (size_t)blockIdx.x * m * m;
  KColArgs A{Wb, gWb, stan, m, g.nE, Sb, gSb};
  for (int c0 = 0; c0 < m; c0 += EPB) {
    const int col = c0 + slot;
    const bool active = col < m;
#pragma unroll
    for (int v = 0; v < NV; ++v) stan[slot * m + v * NODES + node] = (v * NODES + node == col) ? 1.0 : 0.0;
    __syncthreads();
    double y1[1][NV], y2[1][NV];
    eval_slot<EQ, DIM, P, Mode>(A, pp, g, e, slot, node, active, sF + slot * SLOT, y1);
    __syncthreads();
#pragma unroll
    for (int v = 0; v < NV; ++v) stan[slot * m + v * NODES + node] = active ? y1[0][v] : 0.0;
    __syncthreads();
    eval_slot<EQ, DIM, P, Mode>(A, pp, g, e, slot, node, active, sF + slot * SLOT, y2);
    if constexpr (HESS) {
      // BJ^H_ext: + c2 H e_col (hyper-dual, sigma at the build point)
      __syncthreads();
#pragma unroll
      for (int v = 0; v < NV; ++v) stan[slot * m + v * NODES + node] = (v * NODES + node == col) ? 1.0 : 0.0;
      __syncthreads();
      double y3[1][NV];
      eval_slot<EQ, DIM, P, ModeHCol<EQ, NODES>>(A, pp, g, e, slot, node, active, sF + slot * SLOT, y3);
#pragma unroll
      for (int v = 0; v < NV; ++v) y2[0][v] += y3[0][v];
    }
    if (active) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int r = v * NODES + node;
        const double id = r == col ? 1.0 : 0.0;
        Me[(size_t)r * m + col] = fma(c2, y2[0][v], id - a1dt * y1[0][v]);
      }
    }
    __syncthreads();
  }
}

template <int EQ, int DIM, int P, bool HESS>
static cudaError_t run_kbuild_t(const OpCfg& c, const Geo& g, const double* Wb, const double* gWb, double a1dt,
                                double c2, double* M, int e0, int ne, const double* Sb, const double* gSb) {
  constexpr int NODES = ipow(P, DIM);
  constexpr int EPB = epb_for(NODES);
  if (ne <= 0) return cudaSuccess;
  constexpr int NV = NVars<EQ>::value;
  constexpr int SLOT = HESS ? std::max(slot_doubles<EQ, DIM, P, ModeKCol<EQ, NODES>>(),
                                       slot_doubles<EQ, DIM, P, ModeHCol<EQ, NODES>>())
                            : slot_doubles<EQ, DIM, P, ModeKCol<EQ, NODES>>();
  constexpr size_t smem = (size_t)EPB * (SLOT + NV * NODES) * sizeof(double);
  if constexpr (smem > 48 * 1024) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(kbuild_kernel<EQ, DIM, P, EPB, HESS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      attr = true;
    }
  }
  kbuild_kernel<EQ, DIM, P, EPB, HESS><<<ne, EPB * NODES, smem, c.stream>>>(Wb, gWb, c.pp, geo_sel(g), a1dt, c2, M, e0, Sb, gSb);
  hbpdc_count_launch();
  return cudaGetLastError();
}

template <int EQ, int DIM, int P>
static cudaError_t run_kbuild(const OpCfg& c, const Geo& g, const double* Wb, const double* gWb, double a1dt, double c2,
                              double* M, int e0, int ne, const double* Sb, const double* gSb) {
  if (Sb) return run_kbuild_t<EQ, DIM, P, true>(c, g, Wb, gWb, a1dt, c2, M, e0, ne, Sb, gSb);
  return run_kbuild_t<EQ, DIM, P, false>(c, g, Wb, gWb, a1dt, c2, M, e0, ne, Sb, gSb);
}

// ---- dispatch ----------------------------------------------------------------------
template <int EQ, int DIM, int P> struct Disp {
  static constexpr int NODES = ipow(P, DIM);
  static cudaError_t op(OpKind k, const OpCfg& c, const Geo& g, const OpArgs& A) {
    switch (k) {
      case OP_R1: return run_op<EQ, DIM, P, ModeR1<EQ, NODES>>(c, g, A);
      case OP_R1ABS: return run_op<EQ, DIM, P, ModeR1Abs<EQ, NODES>>(c, g, A);
      case OP_R12: return run_op<EQ, DIM, P, ModeR12<EQ, NODES>>(c, g, A);
      case OP_RESID: return run_op<EQ, DIM, P, ModeResid<EQ, NODES>>(c, g, A);
      case OP_JVP_EXACT: return run_op<EQ, DIM, P, ModeJvpExact<EQ, NODES>>(c, g, A);
      case OP_JVP_FD: return run_op<EQ, DIM, P, ModeJvpFD<EQ, NODES>>(c, g, A);
      case OP_JVP_LINEAR:
        if constexpr (EQ == 0) return run_op<EQ, DIM, P, ModeJvpLinear<EQ, NODES>>(c, g, A);
        else return cudaErrorInvalidValue;
      case OP_KAPPLY:
        if constexpr (EQ != 2) return run_op<EQ, DIM, P, ModeKApply<EQ, NODES>>(c, g, A);
        else return cudaErrorNotSupported;
      case OP_KLIN:
        if constexpr (EQ != 2) return run_op<EQ, DIM, P, ModeKLin<EQ, NODES>>(c, g, A);
        else return cudaErrorNotSupported;
      case OP_KNS:
        if constexpr (EQ == 2 && DIM == 2 && !kGL && !kBR2) return run_op<EQ, DIM, P, ModeKNS<EQ, NODES>>(c, g, A);
        else return cudaErrorNotSupported;
      default: return cudaErrorInvalidValue;
    }
  }
  static cudaError_t lift(OpKind k, int s, const OpCfg& c, const Geo& g, const OpArgs& A, double* G, double* Gf,
                          const double* gTg, double* Tg) {
    if constexpr (EQ == 2 && DIM == 2) {
      switch (k) {
        case OP_R1: case OP_R1ABS: return (Tg ? run_gtrace<P, ModeR1<EQ, NODES>, 0>(c, g, A, Tg) : run_lift<P, ModeR1<EQ, NODES>, 0>(c, g, A, G, Gf, gTg));
        case OP_R12: case OP_KNS: return (Tg ? run_gtrace<P, ModeR12<EQ, NODES>, 0>(c, g, A, Tg) : run_lift<P, ModeR12<EQ, NODES>, 0>(c, g, A, G, Gf, gTg));
        case OP_RESID: return (Tg ? run_gtrace<P, ModeResid<EQ, NODES>, 0>(c, g, A, Tg) : run_lift<P, ModeResid<EQ, NODES>, 0>(c, g, A, G, Gf, gTg));
        case OP_JVP_EXACT: return (Tg ? run_gtrace<P, ModeJvpExact<EQ, NODES>, 0>(c, g, A, Tg) : run_lift<P, ModeJvpExact<EQ, NODES>, 0>(c, g, A, G, Gf, gTg));
        case OP_JVP_FD:
          return s == 0 ? (Tg ? run_gtrace<P, ModeJvpFD<EQ, NODES>, 0>(c, g, A, Tg) : run_lift<P, ModeJvpFD<EQ, NODES>, 0>(c, g, A, G, Gf, gTg))
                        : (Tg ? run_gtrace<P, ModeJvpFD<EQ, NODES>, 1>(c, g, A, Tg) : run_lift<P, ModeJvpFD<EQ, NODES>, 1>(c, g, A, G, Gf, gTg));
        default: return cudaErrorInvalidValue;
      }
    }
    return cudaErrorInvalidValue;
  }
  static cudaError_t kbuild(const OpCfg& c, const Geo& g, const double* Wb, const double* gWb, double a1dt, double c2,
                            double* M, int e0, int ne, const double* Sb, const double* gSb) {
    if constexpr (EQ != 2) return run_kbuild<EQ, DIM, P>(c, g, Wb, gWb, a1dt, c2, M, e0, ne, Sb, gSb);
    return cudaErrorNotSupported;
  }
};

#define HBPDC_P_LIST(X, EQ, DIM) X(EQ, DIM, 2) X(EQ, DIM, 3) X(EQ, DIM, 4) X(EQ, DIM, 5) X(EQ, DIM, 6) X(EQ, DIM, 7) X(EQ, DIM, 8)

template <class F>
static cudaError_t dispatch(const OpCfg& c, F&& f) {
#define CASE(EQ, DIM, PP) \
  if (c.eq == EQ && c.dim == DIM && c.P == PP) return f(Disp<EQ, DIM, PP>{});
#if HBPDC_OPS_3D
  // 3D hexahedra, GLL: advection (EQ 0) and Euler (EQ 3: five variables), N = 2, 3
  // (N = 1 would put 16 elements in a CTA: the jet modes' shared memory exceeds 227 KB)
  CASE(0, 3, 3) CASE(0, 3, 4)
  CASE(3, 3, 3) CASE(3, 3, 4)
#else
#if !HBPDC_OPS_BR2
  HBPDC_P_LIST(CASE, 0, 1)
  HBPDC_P_LIST(CASE, 0, 2)
  HBPDC_P_LIST(CASE, 1, 2)
#endif
  HBPDC_P_LIST(CASE, 2, 2)
#endif
#undef CASE
  return cudaErrorInvalidValue;
}

#if HBPDC_OPS_3D
cudaError_t launch_op_3d(OpKind kind, const OpCfg& c, const Geo& g, const OpArgs& A) {
  return dispatch(c, [&](auto d) { return decltype(d)::op(kind, c, g, A); });
}

cudaError_t launch_kbuild_3d(const OpCfg& c, const Geo& g, const double* Wb, const double* gWb, double a1dt,
                             double c2, double* M, int e0, int ne, const double* Sb, const double* gSb) {
  return dispatch(c, [&](auto d) { return decltype(d)::kbuild(c, g, Wb, gWb, a1dt, c2, M, e0, ne, Sb, gSb); });
}
#elif HBPDC_OPS_BR2
#if HBPDC_OPS_GL
cudaError_t launch_op_gl_br2(OpKind kind, const OpCfg& c, const Geo& g, const OpArgs& A) {
#else
cudaError_t launch_op_br2(OpKind kind, const OpCfg& c, const Geo& g, const OpArgs& A) {
#endif
  return dispatch(c, [&](auto d) { return decltype(d)::op(kind, c, g, A); });
}
#elif HBPDC_OPS_GL
cudaError_t launch_lift_gl(OpKind kind, int state, const OpCfg& c, const Geo& g, const OpArgs& A, double* G,
                           double* Gf, const double* gTg, double* Tg) {
  return dispatch(c, [&](auto d) { return decltype(d)::lift(kind, state, c, g, A, G, Gf, gTg, Tg); });
}

cudaError_t launch_op_gl(OpKind kind, const OpCfg& c, const Geo& g, const OpArgs& A) {
  return dispatch(c, [&](auto d) { return decltype(d)::op(kind, c, g, A); });
}

cudaError_t launch_gl_traces(const OpCfg& c, const Geo& g, const OpArgs& A, double* Tr) {
  const int total = g.nE * 4 * c.P;
  if (total == 0) return cudaSuccess;
  const int grid = (total + 127) / 128;
#define GT(PP, NVV) \
  if (c.P == PP && (c.eq == 0 ? 1 : 4) == NVV) { gl_trace_kernel<PP, NVV><<<grid, 128, 0, c.stream>>>(A.W, A.S, A.dW, A.dS, g, Tr); }
  if (c.dim != 2 || c.eq == 2) return cudaErrorInvalidValue;
  GT(2, 1) GT(3, 1) GT(4, 1) GT(5, 1) GT(6, 1) GT(7, 1) GT(8, 1)
  GT(2, 4) GT(3, 4) GT(4, 4) GT(5, 4) GT(6, 4) GT(7, 4) GT(8, 4)
#undef GT
  hbpdc_count_launch();
  return cudaGetLastError();
}

cudaError_t launch_kbuild_gl(const OpCfg& c, const Geo& g, const double* Wb, const double* gWb, double a1dt,
                             double c2, double* M, int e0, int ne, const double* Sb, const double* gSb) {
  return dispatch(c, [&](auto d) { return decltype(d)::kbuild(c, g, Wb, gWb, a1dt, c2, M, e0, ne, Sb, gSb); });
}
#else
int op_grid(const OpCfg& c, const Geo& g) {
  const int nodes = ipow(c.P, c.dim);
  const int epb = epb_for(nodes);
  return (g.nE + epb - 1) / epb;
}

cudaError_t launch_op(OpKind kind, const OpCfg& c, const Geo& g, const OpArgs& A) {
  if (c.dim == 3) return launch_op_3d(kind, c, g, A);
  if (g.br2) return g.gl ? launch_op_gl_br2(kind, c, g, A) : launch_op_br2(kind, c, g, A);
  if (g.gl) return launch_op_gl(kind, c, g, A);
  return dispatch(c, [&](auto d) { return decltype(d)::op(kind, c, g, A); });
}

cudaError_t launch_lift(OpKind kind, int state, const OpCfg& c, const Geo& g, const OpArgs& A, double* G,
                        double* Gf, const double* gTg) {
  if (g.gl) return launch_lift_gl(kind, state, c, g, A, G, Gf, gTg, nullptr);
  return dispatch(c, [&](auto d) { return decltype(d)::lift(kind, state, c, g, A, G, Gf, nullptr, nullptr); });
}

cudaError_t launch_gtrace(OpKind kind, int state, const OpCfg& c, const Geo& g, const OpArgs& A, double* Tg) {
  if (!g.gl) return cudaErrorInvalidValue;
  return launch_lift_gl(kind, state, c, g, A, nullptr, nullptr, nullptr, Tg);
}

int lift_jet_components(OpKind kind, int state) {
  switch (kind) {
    case OP_R1: case OP_R1ABS: return 1;
    case OP_R12: case OP_RESID: case OP_KNS: return 2;
    case OP_JVP_EXACT: return 4;
    case OP_JVP_FD: return state == 0 ? 2 : 3;
    default: return 0;
  }
}

cudaError_t launch_kbuild(const OpCfg& c, const Geo& g, const double* Wb, const double* gWb, double a1dt, double c2,
                          double* M, int e0, int ne, const double* Sb, const double* gSb) {
  if (c.dim == 3) return launch_kbuild_3d(c, g, Wb, gWb, a1dt, c2, M, e0, ne, Sb, gSb);
  if (g.gl) return launch_kbuild_gl(c, g, Wb, gWb, a1dt, c2, M, e0, ne, Sb, gSb);
  return dispatch(c, [&](auto d) { return decltype(d)::kbuild(c, g, Wb, gWb, a1dt, c2, M, e0, ne, Sb, gSb); });
}

// ---- BJ_ext build by element colouring (Navier-Stokes, BR1 stencil radius 2) ----
// The element block K_i of dR1/dW includes the two-hop path through the
// neighbours' lifted gradients (their central face value depends on W_i).  All
// elements of one colour class (ex mod Px, ey mod Py), Px, Py > 2, are seeded
// with e_c at once: no two seeded elements reach each other, so the seeded
// elements' outputs of the linearised operator are exactly K_i e_c (the other
// tangents are exact zeros).  Same colouring as the oracle (oracle element_jacobians).
namespace {
// the k-th element of colour (cx, cy): ex = cx + Px (k mod nx/Px), ey = cy + Py (k div nx/Px)
__device__ __forceinline__ int colour_elem(int k, int nx, int Px, int Py, int cx, int cy) {
  const int nxc = nx / Px;
  return (cy + Py * (k / nxc)) * nx + cx + Px * (k % nxc);
}

// t = e_col on the colour's elements (the rest of t stays zero: set once per build)
__global__ void colour_seed_kernel(double* __restrict__ t, int nc, int nx, int m, int Px, int Py, int cx, int cy,
                                   int col, double val) {
  const size_t n = (size_t)nc * m;
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
    const int e = colour_elem((int)(k / m), nx, Px, Py, cx, cy), r = (int)(k % m);
    t[(size_t)e * m + r] = r == col ? val : 0.0;
  }
}

// t = y on the colour's elements
__global__ void colour_restrict_kernel(const double* __restrict__ y, double* __restrict__ t, int nc, int nx, int m,
                                       int Px, int Py, int cx, int cy) {
  const size_t n = (size_t)nc * m;
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
    const size_t o = (size_t)colour_elem((int)(k / m), nx, Px, Py, cx, cy) * m + k % m;
    t[o] = y[o];
  }
}

// K[e][r][col] = y1, M[e][r][col] = delta - a1dt y1 + c2 y2 for the colour's elements;
// BJ^H_ext (y3 = e_c + H e_c): M = delta - a1dt y1 + c2 (y2 + y3 - delta)
__global__ void colour_gather_kernel(const double* __restrict__ y1, const double* __restrict__ y2,
                                     const double* __restrict__ y3, double* __restrict__ K,
                                     double* __restrict__ M, int nc, int nx, int m, int Px, int Py, int cx, int cy,
                                     int col, double a1dt, double c2) {
  const size_t n = (size_t)nc * m;
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
    const int e = colour_elem((int)(k / m), nx, Px, Py, cx, cy), r = (int)(k % m);
    const size_t i = (size_t)e * m + r;
    const size_t o = i * m + col;
    const double dl = r == col ? 1.0 : 0.0;
    K[o] = y1[i];
    const double q = y3 ? y2[i] + (y3[i] - dl) : y2[i];
    M[o] = fma(c2, q, dl - a1dt * y1[i]);
  }
}

int colour_grid(size_t work) { return (int)std::min<size_t>(1184, (work + 255) / 256); }

// Column col of K_i for the colour's elements, stored TRANSPOSED (row col of K_i^T: consecutive
// threads write consecutive doubles; kk_gemm_kernel transposes it back in shared memory), and for
// BJ^H_ext (y3 = e_col + H e_col) the column c2 H_i e_col of M_i in place (the identity, K and K^2
// terms are added by kk_gemm_kernel).
__global__ void colour_gather_k_kernel(const double* __restrict__ y1, const double* __restrict__ y3,
                                       double* __restrict__ Kt, double* __restrict__ M, int nc, int nx, int m,
                                       int Px, int Py, int cx, int cy, int col, double c2) {
  const size_t n = (size_t)nc * m;
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
    const int e = colour_elem((int)(k / m), nx, Px, Py, cx, cy), r = (int)(k % m);
    const size_t i = (size_t)e * m + r;
    Kt[((size_t)e * m + col) * m + r] = y1[i];
    if (y3) M[i * m + col] = c2 * (y3[i] - (r == col ? 1.0 : 0.0));
  }
}

__device__ __forceinline__ void kk_dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// In place per element: K holds K_i^T from the gather (and M the c2 H_i columns for BJ^H_ext);
// afterwards K holds K_i (row-major, the layout of the apply's GEMV) and M = [c2 H_i +] I - a1dt K_i + c2 K_i K_i
// (P:313-314), K_i^2 on the fp64 tensor cores.  One CTA per element, K_i in shared memory (rows
// padded to ld = mp + 4, mp = m rounded up to 8, zero padding), warp w takes the 8 x 8 output tiles
// w, w + 8, ..., k in steps of 4 (mma.sync m8n8k4).
constexpr int KK_T = 256;
__global__ void __launch_bounds__(KK_T, 1) kk_gemm_kernel(double* __restrict__ K, double* __restrict__ M,
                                                          int m, double a1dt, double c2, int hess, int kt) {
  extern __shared__ __align__(16) double sk[];
  const int mp = (m + 7) & ~7, ld = mp + 4;
  double* Ke = K + (size_t)blockIdx.x * m * m;
  double* Me = M + (size_t)blockIdx.x * m * m;
  for (int t = threadIdx.x; t < mp * ld; t += KK_T) sk[t] = 0.0;
  __syncthreads();
  if (kt) {
    for (int t = threadIdx.x; t < m * m; t += KK_T) {      // coalesced read of K^T, transposed store
      const int c = t / m, r = t % m;
      sk[r * ld + c] = Ke[t];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < m * m; t += KK_T) Ke[t] = sk[(t / m) * ld + t % m];   // K_i row-major
  } else {
    // kt = 0: K already holds K_i row-major (an earlier build of this step transposed it; the
    // second build of the step reuses it for another alpha pair) and stays as it is
    for (int t = threadIdx.x; t < m * m; t += KK_T) sk[(t / m) * ld + t % m] = Ke[t];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int nt = mp / 8;
  for (int tile = wid; tile < nt * nt; tile += KK_T / 32) {
    const int r0 = 8 * (tile / nt), c0 = 8 * (tile % nt);
    double acc[2] = {0.0, 0.0};
    for (int k0 = 0; k0 < mp; k0 += 4)
      kk_dmma(acc, sk[(r0 + g) * ld + k0 + q], sk[(k0 + q) * ld + c0 + g]);
    const int r = r0 + g;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = c0 + 2 * q + h;
      if (r < m && c < m) {
        const size_t o = (size_t)r * m + c;
        Me[o] = (hess ? Me[o] : 0.0) + (r == c ? 1.0 : 0.0) - a1dt * sk[r * ld + c] + c2 * acc[h];
      }
    }
  }
}
}  // namespace

cudaError_t launch_colour_gather_k(const double* y1, const double* y3, double* K, double* M, int nE, int nx, int m,
                                   int Px, int Py, int cx, int cy, int col, double c2, cudaStream_t st) {
  const int nc = nE / (Px * Py);
  colour_gather_k_kernel<<<colour_grid((size_t)nc * m), 256, 0, st>>>(y1, y3, K, M, nc, nx, m, Px, Py, cx, cy, col,
                                                                     c2);
  hbpdc_count_launch();
  return cudaGetLastError();
}

bool kk_gemm_supported(int m) { return m <= 160; }   // K_i in shared memory (<= 227 KB)

cudaError_t launch_kk_gemm(double* K, double* M, int m, int nE, double a1dt, double c2, int hess, int kt, cudaStream_t st) {
  if (!kk_gemm_supported(m)) return cudaErrorInvalidValue;
  if (nE <= 0) return cudaSuccess;
  const int mp = (m + 7) & ~7;
  const size_t smem = (size_t)mp * (mp + 4) * sizeof(double);
  cudaFuncSetAttribute(kk_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kk_gemm_kernel<<<nE, KK_T, smem, st>>>(K, M, m, a1dt, c2, hess, kt);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// seed (val = 1) or clear (val = 0: col = -1) the colour's elements of t
cudaError_t launch_colour_seed(double* t, int nE, int nx, int m, int Px, int Py, int cx, int cy, int col,
                               cudaStream_t st) {
  const int nc = nE / (Px * Py);
  colour_seed_kernel<<<colour_grid((size_t)nc * m), 256, 0, st>>>(t, nc, nx, m, Px, Py, cx, cy, col, 1.0);
  hbpdc_count_launch();
  return cudaGetLastError();
}

cudaError_t launch_colour_restrict(const double* y, double* t, int nE, int nx, int m, int Px, int Py, int cx, int cy,
                                   cudaStream_t st) {
  const int nc = nE / (Px * Py);
  colour_restrict_kernel<<<colour_grid((size_t)nc * m), 256, 0, st>>>(y, t, nc, nx, m, Px, Py, cx, cy);
  hbpdc_count_launch();
  return cudaGetLastError();
}

cudaError_t launch_colour_gather(const double* y1, const double* y2, const double* y3, double* K, double* M, int nE,
                                 int nx, int m, int Px, int Py, int cx, int cy, int col, double a1dt, double c2,
                                 cudaStream_t st) {
  const int nc = nE / (Px * Py);
  colour_gather_kernel<<<colour_grid((size_t)nc * m), 256, 0, st>>>(y1, y2, y3, K, M, nc, nx, m, Px, Py, cx, cy, col,
                                                                   a1dt, c2);
  hbpdc_count_launch();
  return cudaGetLastError();
}
#endif  // HBPDC_OPS_BR2 / HBPDC_OPS_GL

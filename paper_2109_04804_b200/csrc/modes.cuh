// modes.cuh -- what each operator of the hot path feeds the element evaluator.
//
// A mode defines: the node State (one or two jets + NS gradients), NCH output
// channels, how the volume/face fluxes reduce to those channels ("comb"), and
// the epilogue.  Notation: L(.) is the DGSEM operator on a flux field, so
// R1(W) = L(F(W)); a1dt = alpha1 dt; c2 = alpha2 dt^2 / 2.
#pragma once
#include <type_traits>
#include "ops.cuh"

struct OpArgs {
  const double* W;      // state (or build state W_b for the K apply)
  const double* S;      // sigma
  const double* dW;     // Delta W
  const double* dS;     // Delta sigma
  const double* b;      // Newton right-hand side
  const double* U;      // precond: U = S_i W_i
  const double* V;      // precond: V = S_i sigma_i
  double* out1;
  double* out2;
  const double* G0;     // NS lifted gradients of jet state 0
  const double* G1;     // NS lifted gradients of jet state 1
  const double *gG0, *gG1;   // their ghost copies (halo of the lifted gradients)
  const double *shw, *shs;   // JVP epilogue shift: out -= shift * (shw | shs)  (s-step Newton basis)
  double* nrm_part;     // K-apply: per-CTA partial sums of out1^2 (the next FD JVP's ||dW||), or NULL
  double shift;
  double a1dt, c2;
  double epsw;          // FD step for the W direction (<= 0: quotient is 0)
  double iepsw;         // 1 / epsw (0 if epsw <= 0), set by op_kernel
  const double* d_epsw; // if non-NULL, the FD step is read from device memory
  int m;                // doubles per element
  int nE;               // local elements; e >= nE addresses a ghost element (halo)
  const double *gW, *gS, *gdW, *gdS;   // ghost copies (neighbour ranks' face traces)
  const double *Gf0, *Gf1;   // NS BR2: per-face gradients of jet states 0 / 1, or NULL (BR1)
  const double *gGf0, *gGf1; // their ghost copies (the neighbour ranks' shared faces)
  const double* Tr;          // GL FD JVP: face traces [e][face 4][field W,S,dW,dS][var][P] (gl_trace_kernel), or NULL
  const double* Gb;          // NS BJ_ext colour build (ModeKNS): lifted gradients of the build state [e][6][NODES]
  const double* gGb;         // their ghost copies (partitioned runs)
};

// NS BR2 face gradients: [elem][face 4][6][JetN][P] (lift_kernel), face f = 2d + plus,
// kf the node index along the face
template <class T>
__device__ __forceinline__ void load_face_grads(const double* Gf, const double* gGf, int nE, int e, int f, int kf,
                                                int P, T* gx, T* gy) {
  constexpr int JN = JetN<T>::value;
  if (e >= nE) { Gf = gGf; e -= nE; }          // ghost element (halo.cu facebuf exchange)
  const double* base = Gf + ((size_t)e * 4 + f) * 6 * JN * P + kf;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double c[JN];
#pragma unroll
    for (int q = 0; q < JN; ++q) c[q] = base[(k * JN + q) * P];
    if (k < 3) gx[k] = jmake<T>(c); else gy[k - 3] = jmake<T>(c);
  }
}

// JVP epilogue inputs (dW, dsigma and the s-step shift vectors) of one node, prefetched
template <int NV> struct JvpEpiPre {
  double dw[NV], ds[NV], sw[NV], ss[NV];
  __device__ __forceinline__ void load(const OpArgs& A, size_t k0, int stride) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const size_t k = k0 + (size_t)v * stride;
      dw[v] = A.dW[k];
      ds[v] = A.dS[k];
      if (A.shw) { sw[v] = A.shw[k]; ss[v] = A.shs[k]; } else { sw[v] = 0.0; ss[v] = 0.0; }
    }
  }
};

__device__ __forceinline__ double fd_step(const OpArgs& A) { return A.d_epsw ? *A.d_epsw : A.epsw; }

template <int EQ, class T, int NODES>
__device__ __forceinline__ void ld_state(const double* G, const double* Gg, int nE, int e, int node,
                                         NodeState<EQ, T>& s) {
  if constexpr (EQ == 2) {
    if (e < nE) load_grads<T, NODES>(G, e, node, s.gx, s.gy);
    else load_grads<T, NODES>(Gg, e - nE, node, s.gx, s.gy);
  }
}

#define IDX(e, v, node) ((size_t)(e) * A.m + (v) * NODES + (node))
// field F at (e, v, node) for a node-state load: elements e >= A.nE are ghosts
// (halo copies of a neighbouring rank's face traces, same layout, comm.h)
#define FV(F, e, v, node) ((e) < A.nE ? A.F[IDX(e, v, node)] : A.g##F[IDX((e) - A.nE, v, node)])
// base pointer of field F at (e, node) (variable v at [v * NODES]): the own element of a node
// state (nbr = false) is never a ghost, so its loads skip the ghost select
#define FPTR(F, e, node, nbr) (((nbr) && (e) >= A.nE) ? A.g##F + (size_t)((e) - A.nE) * A.m + (node) \
                                                        : A.F + (size_t)(e) * A.m + (node))

// modes whose neighbour states are frozen (no tangent) declare FROZEN_NBR and load_value()
template <class M, class = void> struct FrozenNbr : std::false_type {};
template <class M> struct FrozenNbr<M, std::void_t<decltype(M::FROZEN_NBR)>> : std::bool_constant<M::FROZEN_NBR> {};

// Single-jet modes: Derived supplies  using J; load_w; comb(A, const J* F, c).
template <int EQ, int NODES, class Derived, class J, int NCH_>
struct OneJetMode {
  static constexpr int NV = NVars<EQ>::value, NCH = NCH_;
  using Args = OpArgs;
  template <int K> using StateT = J;
  struct State { NodeState<EQ, J> s; };
  __device__ static void load(const Args& A, const Geo&, int e, int, int node, State& st, bool nbr) {
    Derived::template load_w<0>(A, e, node, st.s.w, nbr);
    ld_state<EQ, J, NODES>(A.G0, A.gG0, A.nE, e, node, st.s);
  }
  template <int DIM>
  __device__ static void vol(const Args& A, const PhysParams& pp, const State& st, double (&c)[DIM][NCH][NV]) {
    J F[DIM][NV];
    vol_flux_all<EQ, DIM>(pp, st.s, F);
#pragma unroll
    for (int d = 0; d < DIM; ++d) Derived::comb(A, F[d], c[d]);
  }
  // face work in two halves: part 0 = the canonical L side (-e_d), part 1 = R
  static constexpr int NFP = 2, FPD = half_doubles<EQ, J>();
  template <class G>
  __device__ static void face_part(const Args& A, const PhysParams& pp, const G& g, int e, int own, int nb,
                                   int nnode, int slot, bool plus, int d, int part, double* raw,
                                   int rs) {
    const bool use_own = (part == 0) == plus;
    if constexpr (FrozenNbr<Derived>::value && EQ != 2) {
      // the neighbour's state carries no tangent (K_i is the element-diagonal block):
      // its half flux in plain doubles, tangent slots zero (same values as the jet)
      if (!use_own) {
        NodeState<EQ, double> sd;
        trace_load(g, nnode, d, sd, [=](int nd, NodeState<EQ, double>& s) { Derived::load_value(A, nb, nd, s.w); },
                   nb >= A.nE);
        constexpr int NR = 2 * NV + 1, JN = JetN<J>::value;
        double tmp[NR];
        half_flux<EQ, double>(pp, sd, d, tmp, 1);
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          raw[rs * (i * JN)] = tmp[i];
#pragma unroll
          for (int c = 1; c < JN; ++c) raw[rs * (i * JN + c)] = 0.0;
        }
        return;
      }
    }
    State st;
    const int le = use_own ? e : nb;
    trace_load(g, use_own ? own : nnode, d, st,
               [=](int nd, State& s) { load(A, g, le, slot, nd, s, !use_own); }, le >= A.nE);
    if constexpr (EQ == 2) {
      if constexpr (G::BR2) {                   // BR2: the face's own local-lifting gradient (reading R33)
        const int f = 2 * d + (use_own ? (plus ? 1 : 0) : (plus ? 0 : 1));
        const int kf = d == 0 ? own / g.P : own % g.P;
        load_face_grads<J>(A.Gf0, A.gGf0, A.nE, le, f, kf, g.P, st.s.gx, st.s.gy);
      }
    }
    half_flux<EQ, J>(pp, st.s, d, raw, rs);
  }
  __device__ static void face_combine(const Args& A, const PhysParams& pp, int d, const double* rL,
                                      const double* rR, int rs, double (&c)[NCH][NV]) {
    J f[NV];
    face_from_halves<EQ, J>(pp, rL, rR, rs, d, f);
    Derived::comb(A, f, c);
  }
};

// R1(W)                                                        (eq:DGSEM_wt)
template <int EQ, int NODES> struct ModeR1 : OneJetMode<EQ, NODES, ModeR1<EQ, NODES>, double, 1> {
  static constexpr int NV = NVars<EQ>::value, NCH = 1;
  template <int K>
  __device__ static void load_w(const OpArgs& A, int e, int node, double* w, bool nbr) {
    const double* pw = FPTR(W, e, node, nbr);
    for (int v = 0; v < NV; ++v) w[v] = pw[v * NODES];
  }
  __device__ static void comb(const OpArgs&, const double* F, double (&c)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) c[0][v] = F[v];
  }
  __device__ static void epilogue(const OpArgs& A, int e, int node, const double (&o)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) A.out1[IDX(e, v, node)] = o[0][v];
  }
};

// R1_abs(W): every term of eq:DGSEM_wt by magnitude (|Dhat| via the Geo, |F|,
// |f*|); the rounding scale of R1 used for the Newton floor (reading R10b).
template <int EQ, int NODES> struct ModeR1Abs : OneJetMode<EQ, NODES, ModeR1Abs<EQ, NODES>, double, 1> {
  static constexpr int NV = NVars<EQ>::value, NCH = 1;
  template <int K>
  __device__ static void load_w(const OpArgs& A, int e, int node, double* w, bool nbr) {
    const double* pw = FPTR(W, e, node, nbr);
    for (int v = 0; v < NV; ++v) w[v] = pw[v * NODES];
  }
  __device__ static void comb(const OpArgs&, const double* F, double (&c)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) c[0][v] = fabs(F[v]);
  }
  __device__ static void epilogue(const OpArgs& A, int e, int node, const double (&o)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) A.out1[IDX(e, v, node)] = -o[0][v];
  }
};

// R1(W) and R2(W, sigma) from one dual evaluation             (eq:DGSEM_wtt)
template <int EQ, int NODES> struct ModeR12 : OneJetMode<EQ, NODES, ModeR12<EQ, NODES>, J1, 2> {
  static constexpr int NV = NVars<EQ>::value, NCH = 2;
  template <int K>
  __device__ static void load_w(const OpArgs& A, int e, int node, J1* w, bool nbr) {
    const double *pw = FPTR(W, e, node, nbr), *ps = FPTR(S, e, node, nbr);
    for (int v = 0; v < NV; ++v) w[v] = J1{pw[v * NODES], ps[v * NODES]};
  }
  __device__ static void comb(const OpArgs&, const J1* F, double (&c)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) { c[0][v] = F[v].v; c[1][v] = F[v].a; }
  }
  __device__ static void epilogue(const OpArgs& A, int e, int node, const double (&o)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) {
      if (A.out1) A.out1[IDX(e, v, node)] = o[0][v];
      A.out2[IDX(e, v, node)] = o[1][v];
    }
  }
};

// Stage residual: G1 = W - b + L(-a1dt F + c2 F'sigma), G2 = sigma - L(F)
// (eq:Newton_Residual; P:236-239 read as R4)
template <int EQ, int NODES> struct ModeResid : OneJetMode<EQ, NODES, ModeResid<EQ, NODES>, J1, 2> {
  static constexpr int NV = NVars<EQ>::value, NCH = 2;
  // (round 2: with the surface terms as the fifth DMMA k-step the tensor-core contraction is
  // faster here too: 88 -> 78 us at C3, r02zc; it had opted out before, r02e)
  template <int K>
  __device__ static void load_w(const OpArgs& A, int e, int node, J1* w, bool nbr) {
    const double *pw = FPTR(W, e, node, nbr), *ps = FPTR(S, e, node, nbr);
    for (int v = 0; v < NV; ++v) w[v] = J1{pw[v * NODES], ps[v * NODES]};
  }
  __device__ static void comb(const OpArgs& A, const J1* F, double (&c)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) {
      c[0][v] = fma(A.c2, F[v].a, -A.a1dt * F[v].v);
      c[1][v] = F[v].v;
    }
  }
  struct EpiPre { double w[NV], b[NV], s[NV]; };
  __device__ static void prefetch_epi(const OpArgs& A, int e, int node, EpiPre& p) {
    for (int v = 0; v < NV; ++v) { const size_t k = IDX(e, v, node); p.w[v] = A.W[k]; p.b[v] = A.b[k]; p.s[v] = A.S[k]; }
  }
  __device__ static void epilogue(const OpArgs& A, int e, int node, const double (&o)[NCH][NV], const EpiPre& p) {
    for (int v = 0; v < NV; ++v) {
      const size_t k = IDX(e, v, node);
      A.out1[k] = (p.w[v] - p.b[v]) + o[0][v];
      A.out2[k] = p.s[v] - o[1][v];
    }
  }
};

// EXACT JVP.  Hyper-dual input W + e1 sigma + e2 dW + e1e2 dsigma gives
//   b-part = dR1/dW dW,   c-part = dR2/dW dW + dR2/dsigma dsigma
// so  top = dW + L(-a1dt F_b + c2 F_c),  bottom = dsigma - L(F_b)   (eq:nonlinear_eqsys)
template <int EQ, int NODES> struct ModeJvpExact : OneJetMode<EQ, NODES, ModeJvpExact<EQ, NODES>, HJ, 2> {
  static constexpr int NV = NVars<EQ>::value, NCH = 2;
  template <int K>
  __device__ static void load_w(const OpArgs& A, int e, int node, HJ* w, bool nbr) {
    const double *pw = FPTR(W, e, node, nbr), *ps = FPTR(S, e, node, nbr);
    const double *pdw = FPTR(dW, e, node, nbr), *pds = FPTR(dS, e, node, nbr);
    for (int v = 0; v < NV; ++v) w[v] = HJ{pw[v * NODES], ps[v * NODES], pdw[v * NODES], pds[v * NODES]};
  }
  __device__ static void comb(const OpArgs& A, const HJ* F, double (&c)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) {
      c[0][v] = fma(A.c2, F[v].c, -A.a1dt * F[v].b);
      c[1][v] = F[v].b;
    }
  }
  using EpiPre = JvpEpiPre<NV>;
  __device__ static void prefetch_epi(const OpArgs& A, int e, int node, EpiPre& p) { p.load(A, IDX(e, 0, node), NODES); }
  __device__ static void epilogue(const OpArgs& A, int e, int node, const double (&o)[NCH][NV], const EpiPre& p) {
    for (int v = 0; v < NV; ++v) {
      const size_t k = IDX(e, v, node);
      double t1 = p.dw[v] + o[0][v], t2 = p.ds[v] - o[1][v];
      if (A.shw) { t1 = fma(-A.shift, p.sw[v], t1); t2 = fma(-A.shift, p.ss[v], t2); }
      A.out1[k] = t1;
      A.out2[k] = t2;
    }
  }
};

// FD JVP (eq:MatrixFree_nonlinear; sigma direction exact, R8):
//   p = (W + eps dW) + e1 sigma           (J1)
//   q =  W + e1 sigma + e2 dsigma         (J2)
//   top = dW + L(-a1dt (F_p - F_q)/eps + c2 (F'_p s - F'_q s)/eps + c2 F'_q ds)
//   bot = dsigma - L((F_p - F_q)/eps)
// eps <= 0 means ||dW|| = 0 and the dW quotients are 0.
template <int EQ, int NODES> struct ModeJvpFD {
  static constexpr int NV = NVars<EQ>::value, NCH = 2;
  using Args = OpArgs;
  template <int K> using StateT = typename std::conditional<K == 0, J1, J2>::type;
  struct State { NodeState<EQ, J1> p; NodeState<EQ, J2> q; };
  template <int K>
  __device__ static void load_w(const Args& A, int e, int node, StateT<K>* w, bool nbr) {
    const double *pw = FPTR(W, e, node, nbr), *ps = FPTR(S, e, node, nbr);
    if constexpr (K == 0) {
      const double ew = fd_step(A);
      const double* pdw = FPTR(dW, e, node, nbr);
      for (int v = 0; v < NV; ++v) {
        const double Wk = pw[v * NODES];
        const double wp = ew > 0.0 ? __dadd_rn(Wk, __dmul_rn(ew, pdw[v * NODES])) : Wk;
        w[v] = J1{wp, ps[v * NODES]};
      }
    } else {
      const double* pds = FPTR(dS, e, node, nbr);
      for (int v = 0; v < NV; ++v) w[v] = J2{pw[v * NODES], ps[v * NODES], pds[v * NODES]};
    }
  }
  __device__ static void load(const Args& A, const Geo&, int e, int, int node, State& st, bool nbr) {
    load_w<0>(A, e, node, st.p.w, nbr);
    load_w<1>(A, e, node, st.q.w, nbr);
    ld_state<EQ, J1, NODES>(A.G0, A.gG0, A.nE, e, node, st.p);
    ld_state<EQ, J2, NODES>(A.G1, A.gG1, A.nE, e, node, st.q);
  }
  __device__ static void comb(const Args& A, const J1* Fp, const J2* Fq, double (&c)[NCH][NV]) {
    const double ew = fd_step(A);
    if (ew > 0.0) {
      const double ie = A.iepsw;
      for (int v = 0; v < NV; ++v) {
        const double q1 = (Fp[v].v - Fq[v].v) * ie;
        const double q2 = (Fp[v].a - Fq[v].a) * ie;
        c[0][v] = fma(A.c2, q2 + Fq[v].b, -A.a1dt * q1);
        c[1][v] = q1;
      }
    } else {
      for (int v = 0; v < NV; ++v) { c[0][v] = A.c2 * Fq[v].b; c[1][v] = 0.0; }
    }
  }
  template <int DIM>
  __device__ static void vol(const Args& A, const PhysParams& pp, const State& st, double (&c)[DIM][NCH][NV]) {
    if constexpr (EQ == 1) {
      // primitives once per jet state, fluxes one direction at a time (short live ranges)
      const EulerPrim<J1> qp = euler_prim(pp, st.p.w);
      const EulerPrim<J2> qq = euler_prim(pp, st.q.w);
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        J1 Fp[NV];
        J2 Fq[NV];
        euler_flux(st.p.w, qp, d, Fp);
        euler_flux(st.q.w, qq, d, Fq);
        comb(A, Fp, Fq, c[d]);
      }
    } else {
      J1 Fp[DIM][NV];
      J2 Fq[DIM][NV];
      vol_flux_all<EQ, DIM>(pp, st.p, Fp);
      vol_flux_all<EQ, DIM>(pp, st.q, Fq);
#pragma unroll
      for (int d = 0; d < DIM; ++d) comb(A, Fp[d], Fq[d], c[d]);
    }
  }
  // volume fluxes in two passes (the two jet states are never live together):
  // pass 0 leaves the p-state flux (tangent, value) in the output slots, pass 1
  // combines them with the q-state flux into the channels (same arithmetic as comb)
  static constexpr int VOL_PASSES = 2;
  template <int DIM>
  __device__ static void vol_pass0(const Args& A, const PhysParams& pp, int e, int node,
                                   double (&t)[DIM][NCH][NV]) {
    if (!(fd_step(A) > 0.0)) return;
    NodeState<EQ, J1> p;
    load_w<0>(A, e, node, p.w, false);
    ld_state<EQ, J1, NODES>(A.G0, A.gG0, A.nE, e, node, p);
    J1 F[DIM][NV];
    vol_flux_all<EQ, DIM>(pp, p, F);
#pragma unroll
    for (int d = 0; d < DIM; ++d)
#pragma unroll
      for (int v = 0; v < NV; ++v) { t[d][0][v] = F[d][v].a; t[d][1][v] = F[d][v].v; }
  }
  template <int DIM>
  __device__ static void vol_pass1(const Args& A, const PhysParams& pp, int e, int node,
                                   double (&t)[DIM][NCH][NV]) {
    NodeState<EQ, J2> q;
    load_w<1>(A, e, node, q.w, false);
    ld_state<EQ, J2, NODES>(A.G1, A.gG1, A.nE, e, node, q);
    J2 F[DIM][NV];
    vol_flux_all<EQ, DIM>(pp, q, F);
    const double ew = fd_step(A);
    const double ie = A.iepsw;
#pragma unroll
    for (int d = 0; d < DIM; ++d)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if (ew > 0.0) {
          const double q1 = (t[d][1][v] - F[d][v].v) * ie;
          const double q2 = (t[d][0][v] - F[d][v].a) * ie;
          t[d][0][v] = fma(A.c2, q2 + F[d][v].b, -A.a1dt * q1);
          t[d][1][v] = q1;
        } else {
          t[d][0][v] = A.c2 * F[d][v].b;
          t[d][1][v] = 0.0;
        }
      }
  }
  // face work split by jet state: part 0 = p-state face flux (J1), part 1 = q-state (J2)
  static constexpr int NFP = 2, FPD = 3 * NV;
  template <class G>
  __device__ static void face_part(const Args& A, const PhysParams& pp, const G& g, int e, int own, int nb,
                                   int nnode, int, bool plus, int d, int part, double* raw,
                                   int rs) {
    if constexpr (G::GL && EQ != 2) {
      if (A.Tr && nb < A.nE) {
        // Gauss-Legendre: both traces from the precomputed face traces (one read per value instead
        // of a P-node line sum per face node); p = trace(W) + eps trace(dW), as the halo's ghosts
        const int P = g.P;
        const int k = d == 0 ? own / P : own % P;
        const int fo = 2 * d + (plus ? 1 : 0), fn = fo ^ 1;
        const double* to = A.Tr + ((size_t)e * 4 + fo) * 4 * NV * P + k;
        const double* tn = A.Tr + ((size_t)nb * 4 + fn) * 4 * NV * P + k;
        auto fld = [&](const double* t, int f, int v) { return t[(f * NV + v) * P]; };
        if (part == 0) {
          const double ew = fd_step(A);
          if (!(ew > 0.0)) return;
          NodeState<EQ, J1> so, sn;
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            so.w[v] = J1{__dadd_rn(fld(to, 0, v), __dmul_rn(ew, fld(to, 2, v))), fld(to, 1, v)};
            sn.w[v] = J1{__dadd_rn(fld(tn, 0, v), __dmul_rn(ew, fld(tn, 2, v))), fld(tn, 1, v)};
          }
          J1 fp[NV];
          if (plus) face_flux<EQ>(pp, so, sn, d, fp);
          else face_flux<EQ>(pp, sn, so, d, fp);
          for (int v = 0; v < NV; ++v) { raw[rs * (2 * v)] = fp[v].v; raw[rs * (2 * v + 1)] = fp[v].a; }
        } else {
          NodeState<EQ, J2> so, sn;
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            so.w[v] = J2{fld(to, 0, v), fld(to, 1, v), fld(to, 3, v)};
            sn.w[v] = J2{fld(tn, 0, v), fld(tn, 1, v), fld(tn, 3, v)};
          }
          J2 fq[NV];
          if (plus) face_flux<EQ>(pp, so, sn, d, fq);
          else face_flux<EQ>(pp, sn, so, d, fq);
          for (int v = 0; v < NV; ++v) {
            raw[rs * (3 * v)] = fq[v].v; raw[rs * (3 * v + 1)] = fq[v].a; raw[rs * (3 * v + 2)] = fq[v].b;
          }
        }
        return;
      }
    }
    if (part == 0) {
      if (!(fd_step(A) > 0.0)) return;
      NodeState<EQ, J1> so, sn;
      trace_load(g, own, d, so, [=](int nd, NodeState<EQ, J1>& s) {
        load_w<0>(A, e, nd, s.w, false);
        ld_state<EQ, J1, NODES>(A.G0, A.gG0, A.nE, e, nd, s);
      });
      trace_load(g, nnode, d, sn, [=](int nd, NodeState<EQ, J1>& s) {
        load_w<0>(A, nb, nd, s.w, true);
        ld_state<EQ, J1, NODES>(A.G0, A.gG0, A.nE, nb, nd, s);
      }, nb >= A.nE);
      if constexpr (EQ == 2) {
        if constexpr (G::BR2) {
          const int kf = d == 0 ? own / g.P : own % g.P;
          load_face_grads<J1>(A.Gf0, A.gGf0, A.nE, e, 2 * d + (plus ? 1 : 0), kf, g.P, so.gx, so.gy);
          load_face_grads<J1>(A.Gf0, A.gGf0, A.nE, nb, 2 * d + (plus ? 0 : 1), kf, g.P, sn.gx, sn.gy);
        }
      }
      J1 fp[NV];
      if (plus) face_flux<EQ>(pp, so, sn, d, fp);
      else face_flux<EQ>(pp, sn, so, d, fp);
      for (int v = 0; v < NV; ++v) { raw[rs * (2 * v)] = fp[v].v; raw[rs * (2 * v + 1)] = fp[v].a; }
    } else {
      NodeState<EQ, J2> so, sn;
      trace_load(g, own, d, so, [=](int nd, NodeState<EQ, J2>& s) {
        load_w<1>(A, e, nd, s.w, false);
        ld_state<EQ, J2, NODES>(A.G1, A.gG1, A.nE, e, nd, s);
      });
      trace_load(g, nnode, d, sn, [=](int nd, NodeState<EQ, J2>& s) {
        load_w<1>(A, nb, nd, s.w, true);
        ld_state<EQ, J2, NODES>(A.G1, A.gG1, A.nE, nb, nd, s);
      }, nb >= A.nE);
      if constexpr (EQ == 2) {
        if constexpr (G::BR2) {
          const int kf = d == 0 ? own / g.P : own % g.P;
          load_face_grads<J2>(A.Gf1, A.gGf1, A.nE, e, 2 * d + (plus ? 1 : 0), kf, g.P, so.gx, so.gy);
          load_face_grads<J2>(A.Gf1, A.gGf1, A.nE, nb, 2 * d + (plus ? 0 : 1), kf, g.P, sn.gx, sn.gy);
        }
      }
      J2 fq[NV];
      if (plus) face_flux<EQ>(pp, so, sn, d, fq);
      else face_flux<EQ>(pp, sn, so, d, fq);
      for (int v = 0; v < NV; ++v) {
        raw[rs * (3 * v)] = fq[v].v; raw[rs * (3 * v + 1)] = fq[v].a; raw[rs * (3 * v + 2)] = fq[v].b;
      }
    }
  }
  // Staged face loads (GLL, Euler / advection): the thread of face item (part, node) prefetches
  // the neighbour node's W, sigma and dW (part 0) or dsigma (part 1) with cp.async before the
  // volume flux; its own edge node is L1-resident (loaded by the element's volume pass).
// Off by default: measured slower in the same session (r02e, C3 FD JVP 157 -> 166 us with the
// DMMA contraction; the extra shared memory costs occupancy more than the L2 latency it hides).
#ifndef HBPDC_STAGE_FACES
#define HBPDC_STAGE_FACES 0
#endif
  static constexpr int NSTAGE = (EQ != 2 && HBPDC_STAGE_FACES) ? 3 * NV : 0;
  __device__ static void prefetch(const Args& A, int, int, int nb, int nnode, int part, double* st, int stride) {
    const bool gh = nb >= A.nE;
    const int eb = gh ? nb - A.nE : nb;
    const double* f0 = gh ? A.gW : A.W;
    const double* f1 = gh ? A.gS : A.S;
    const double* f2 = part == 0 ? (gh ? A.gdW : A.dW) : (gh ? A.gdS : A.dS);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const size_t k = IDX(eb, v, nnode);
      cp_async8(st + (0 * NV + v) * stride, f0 + k);
      cp_async8(st + (1 * NV + v) * stride, f1 + k);
      cp_async8(st + (2 * NV + v) * stride, f2 + k);
    }
  }
  template <class G>
  __device__ static void face_part_staged(const Args& A, const PhysParams& pp, const G& g, int e, int own, int nb,
                                          int nnode, bool plus, int d, int part, const double* st, int stride,
                                          double* raw, int rs) {
    if constexpr (EQ != 2) {
      if (part == 0) {
        const double ew = fd_step(A);
        if (!(ew > 0.0)) return;
        NodeState<EQ, J1> so, sn;
        load_w<0>(A, e, own, so.w, false);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double Wk = st[v * stride], Sk = st[(NV + v) * stride], dk = st[(2 * NV + v) * stride];
          sn.w[v] = J1{__dadd_rn(Wk, __dmul_rn(ew, dk)), Sk};      // as load_w<0>
        }
        J1 fp[NV];
        if (plus) face_flux<EQ>(pp, so, sn, d, fp);
        else face_flux<EQ>(pp, sn, so, d, fp);
        for (int v = 0; v < NV; ++v) { raw[rs * (2 * v)] = fp[v].v; raw[rs * (2 * v + 1)] = fp[v].a; }
      } else {
        NodeState<EQ, J2> so, sn;
        load_w<1>(A, e, own, so.w, false);
#pragma unroll
        for (int v = 0; v < NV; ++v) sn.w[v] = J2{st[v * stride], st[(NV + v) * stride], st[(2 * NV + v) * stride]};
        J2 fq[NV];
        if (plus) face_flux<EQ>(pp, so, sn, d, fq);
        else face_flux<EQ>(pp, sn, so, d, fq);
        for (int v = 0; v < NV; ++v) {
          raw[rs * (3 * v)] = fq[v].v; raw[rs * (3 * v + 1)] = fq[v].a; raw[rs * (3 * v + 2)] = fq[v].b;
        }
      }
    }
  }
  __device__ static void face_combine(const Args& A, const PhysParams&, int, const double* rp, const double* rq,
                                      int rs, double (&c)[NCH][NV]) {
    const double ew = fd_step(A);
    const double ie = A.iepsw;
    for (int v = 0; v < NV; ++v) {
      if (ew > 0.0) {
        const double q1 = (rp[rs * (2 * v)] - rq[rs * (3 * v)]) * ie;
        const double q2 = (rp[rs * (2 * v + 1)] - rq[rs * (3 * v + 1)]) * ie;
        c[0][v] = fma(A.c2, q2 + rq[rs * (3 * v + 2)], -A.a1dt * q1);
        c[1][v] = q1;
      } else {
        c[0][v] = A.c2 * rq[rs * (3 * v + 2)];
        c[1][v] = 0.0;
      }
    }
  }
  using EpiPre = JvpEpiPre<NV>;
  __device__ static void prefetch_epi(const Args& A, int e, int node, EpiPre& p) { p.load(A, IDX(e, 0, node), NODES); }
  __device__ static void epilogue(const Args& A, int e, int node, const double (&o)[NCH][NV], const EpiPre& p) {
    for (int v = 0; v < NV; ++v) {
      const size_t k = IDX(e, v, node);
      double t1 = p.dw[v] + o[0][v], t2 = p.ds[v] - o[1][v];
      if (A.shw) { t1 = fma(-A.shift, p.sw[v], t1); t2 = fma(-A.shift, p.ss[v], t2); }
      A.out1[k] = t1;
      A.out2[k] = t2;
    }
  }
};

// Linear JVP for advection (eq:MatrixFree_linear):
//   top = dW + L(F(-a1dt dW + c2 dsigma)),  bot = dsigma - L(F(dW))
template <int EQ, int NODES> struct ModeJvpLinear {
  static constexpr int NV = NVars<EQ>::value, NCH = 2;
  using Args = OpArgs;
  template <int K> using StateT = double;
  struct State { NodeState<EQ, double> u0, u1; };
  template <int K>
  __device__ static void load_w(const Args& A, int e, int node, double* w, bool) {
    for (int v = 0; v < NV; ++v) w[v] = FV(dW, e, v, node);
  }
  __device__ static void load(const Args& A, const Geo&, int e, int, int node, State& st, bool nbr) {
    const double *pdw = FPTR(dW, e, node, nbr), *pds = FPTR(dS, e, node, nbr);
    for (int v = 0; v < NV; ++v) {
      const double dw = pdw[v * NODES];
      st.u0.w[v] = fma(A.c2, pds[v * NODES], -A.a1dt * dw);
      st.u1.w[v] = dw;
    }
  }
  template <int DIM>
  __device__ static void vol(const Args&, const PhysParams& pp, const State& st, double (&c)[DIM][NCH][NV]) {
    double F0[DIM][NV], F1[DIM][NV];
    vol_flux_all<EQ, DIM>(pp, st.u0, F0);
    vol_flux_all<EQ, DIM>(pp, st.u1, F1);
#pragma unroll
    for (int d = 0; d < DIM; ++d)
      for (int v = 0; v < NV; ++v) { c[d][0][v] = F0[d][v]; c[d][1][v] = F1[d][v]; }
  }
  // face work split by input: part 0 = F(-a1dt dW + c2 dsigma), part 1 = F(dW)
  static constexpr int NFP = 2, FPD = NV;
  template <class G>
  __device__ static void face_part(const Args& A, const PhysParams& pp, const G& g, int e, int own, int nb,
                                   int nnode, int slot, bool plus, int d, int part, double* raw,
                                   int rs) {
    State so, sn;
    trace_load(g, own, d, so, [=](int nd, State& s) { load(A, g, e, slot, nd, s, false); });
    trace_load(g, nnode, d, sn, [=](int nd, State& s) { load(A, g, nb, slot, nd, s, true); }, nb >= A.nE);
    const NodeState<EQ, double>& o = part == 0 ? so.u0 : so.u1;
    const NodeState<EQ, double>& q = part == 0 ? sn.u0 : sn.u1;
    double f[NV];
    if (plus) face_flux<EQ>(pp, o, q, d, f);
    else face_flux<EQ>(pp, q, o, d, f);
    for (int v = 0; v < NV; ++v) raw[rs * v] = f[v];
  }
  __device__ static void face_combine(const Args&, const PhysParams&, int, const double* r0, const double* r1,
                                      int rs, double (&c)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) { c[0][v] = r0[rs * v]; c[1][v] = r1[rs * v]; }
  }
  using EpiPre = JvpEpiPre<NV>;
  __device__ static void prefetch_epi(const Args& A, int e, int node, EpiPre& p) { p.load(A, IDX(e, 0, node), NODES); }
  __device__ static void epilogue(const Args& A, int e, int node, const double (&o)[NCH][NV], const EpiPre& p) {
    for (int v = 0; v < NV; ++v) {
      const size_t k = IDX(e, v, node);
      double t1 = p.dw[v] + o[0][v], t2 = p.ds[v] - o[1][v];
      if (A.shw) { t1 = fma(-A.shift, p.sw[v], t1); t2 = fma(-A.shift, p.ss[v], t2); }
      A.out1[k] = t1;
      A.out2[k] = t2;
    }
  }
};

// BJ_ext apply, second half (P:634-641 in the S+K form):
//   K_i = element-diagonal block of dR1/dW at the build state W_b ("neighbour
//   traces frozen": the neighbour's jet carries no tangent).
//   top = U - c2 K V,   bottom = V + K (U - a1dt V).
template <int EQ, int NODES> struct ModeKApply : OneJetMode<EQ, NODES, ModeKApply<EQ, NODES>, J2, 2> {
  static constexpr int NV = NVars<EQ>::value, NCH = 2;
  static constexpr bool FROZEN_NBR = true;
  __device__ static void load_value(const OpArgs& A, int e, int node, double* w) {
    const double* pw = FPTR(W, e, node, true);
    for (int v = 0; v < NV; ++v) w[v] = pw[v * NODES];
  }
  template <int K>
  __device__ static void load_w(const OpArgs& A, int e, int node, J2* w, bool nbr) {
    for (int v = 0; v < NV; ++v) {
      if (nbr) {
        w[v] = J2{FV(W, e, v, node), 0.0, 0.0};
      } else {
        const size_t k = IDX(e, v, node);
        w[v] = J2{A.W[k], A.V[k], fma(-A.a1dt, A.V[k], A.U[k])};
      }
    }
  }
  __device__ static void comb(const OpArgs&, const J2* F, double (&c)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) { c[0][v] = F[v].a; c[1][v] = F[v].b; }
  }

  // epilogue that also returns this node's sum of out1^2 (op_kernel reduces it per CTA)
  static constexpr bool NORM_EPILOGUE = true;
  struct EpiPre { double u[NV], vv[NV]; };
  __device__ static void epilogue(const OpArgs& A, int e, int node, const double (&o)[NCH][NV], const EpiPre& p) {
    (void)epilogue_ss(A, e, node, o, p);
  }
  __device__ static void prefetch_epi(const OpArgs& A, int e, int node, EpiPre& p) {
    for (int v = 0; v < NV; ++v) { const size_t k = IDX(e, v, node); p.u[v] = A.U[k]; p.vv[v] = A.V[k]; }
  }
  __device__ static double epilogue_ss(const OpArgs& A, int e, int node, const double (&o)[NCH][NV], const EpiPre& p) {
    double ss = 0.0;
    for (int v = 0; v < NV; ++v) {
      const size_t k = IDX(e, v, node);
      const double t1 = fma(-A.c2, o[0][v], p.u[v]);
      A.out1[k] = t1;
      A.out2[k] = p.vv[v] + o[1][v];
      ss = fma(t1, t1, ss);
    }
    return ss;
  }
};

// BJ^H_ext apply pieces: out1 = b + a1dt * (K_i t), t = dW on the own element,
// neighbour states frozen (K_i = element block of dR1/dW at the build state W).
// (OpArgs reuse: W = build state, dW = t, b = base vector, a1dt = the scale.)
template <int EQ, int NODES> struct ModeKLin : OneJetMode<EQ, NODES, ModeKLin<EQ, NODES>, J1, 1> {
  static constexpr int NV = NVars<EQ>::value, NCH = 1;
  static constexpr bool FROZEN_NBR = true;
  __device__ static void load_value(const OpArgs& A, int e, int node, double* w) {
    for (int v = 0; v < NV; ++v) w[v] = FV(W, e, v, node);
  }
  template <int K>
  __device__ static void load_w(const OpArgs& A, int e, int node, J1* w, bool nbr) {
    for (int v = 0; v < NV; ++v) w[v] = J1{FV(W, e, v, node), nbr ? 0.0 : A.dW[IDX(e, v, node)]};
  }
  __device__ static void comb(const OpArgs&, const J1* F, double (&c)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) c[0][v] = F[v].a;
  }
  __device__ static void epilogue(const OpArgs& A, int e, int node, const double (&o)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) {
      const size_t k = IDX(e, v, node);
      A.out1[k] = fma(A.a1dt, o[0][v], A.b[k]);
    }
  }
};

#undef FV
// NS BJ_ext colour build, one column of K_i for the colour's elements (GLL, BR1):
// the tangent channel of R1(W_b + e1 t), t = the seed (zero outside the colour's elements),
// with the lifting evaluated on the colour's elements ONLY.  The neighbour's lifted gradient
// at the shared face is the build state's (A.Gb) plus its one seed-dependent term: the
// neighbour's BR1 central value g* = 1/2 (g_nb + g_i) gives its normal gradient
// component at the shared face node the tangent s_nb * 1/2 * dg_i, s_nb = (2/h) lhat of the
// neighbour's side -- exactly what the neighbour's own lifting of the seeded state computes
// there (its volume part and its other faces carry no tangent).  This replaces a lifting pass
// over the colour's elements AND their four neighbours per (colour, column) (reading R19).
template <int EQ, int NODES> struct ModeKNS : OneJetMode<EQ, NODES, ModeKNS<EQ, NODES>, J1, 1> {
  static constexpr int NV = NVars<EQ>::value, NCH = 1;
  using Base = OneJetMode<EQ, NODES, ModeKNS<EQ, NODES>, J1, 1>;
  template <int K>
  __device__ static void load_w(const OpArgs& A, int e, int node, J1* w, bool nbr) {
    const double *pw = FPTR(W, e, node, nbr), *ps = FPTR(S, e, node, nbr);
    for (int v = 0; v < NV; ++v) w[v] = J1{pw[v * NODES], ps[v * NODES]};
  }
  __device__ static void comb(const OpArgs&, const J1* F, double (&c)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) c[0][v] = F[v].a;
  }
  __device__ static void epilogue(const OpArgs& A, int e, int node, const double (&o)[NCH][NV]) {
    for (int v = 0; v < NV; ++v) A.out2[IDX(e, v, node)] = o[0][v];
  }
  template <class G>
  __device__ static void face_part(const OpArgs& A, const PhysParams& pp, const G& g, int e, int own, int nb,
                                   int nnode, int slot, bool plus, int d, int part, double* raw, int rs) {
    const bool use_own = (part == 0) == plus;
    if (use_own || EQ != 2) {
      Base::face_part(A, pp, g, e, own, nb, nnode, slot, plus, d, part, raw, rs);
      return;
    }
    if constexpr (EQ == 2) {
      NodeState<EQ, J1> sn, so;
      const double* pw = FPTR(W, nb, nnode, true);
#pragma unroll
      for (int v = 0; v < NV; ++v) sn.w[v] = J1{pw[v * NODES], 0.0};      // t = 0 off the colour
      const double* gb = nb < A.nE ? A.Gb + (size_t)nb * 6 * NODES + nnode
                                   : A.gGb + (size_t)(nb - A.nE) * 6 * NODES + nnode;
#pragma unroll
      for (int k = 0; k < 3; ++k) { sn.gx[k] = J1{gb[k * NODES], 0.0}; sn.gy[k] = J1{gb[(k + 3) * NODES], 0.0}; }
      load_w<0>(A, e, own, so.w, false);
      J1 go[3];
      grad_vars(pp, so.w, go);
      const double snb = (d == 0 ? g.sx : g.sy) * (plus ? -g.lhm : g.lhp);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double tk = snb * (0.5 * go[k].a);
        if (d == 0) sn.gx[k].a = tk; else sn.gy[k].a = tk;
      }
      half_flux<EQ, J1>(pp, sn, d, raw, rs);
    }
  }
};

#undef IDX

// ops.cuh -- fused DGSEM element operators on Gauss-Lobatto nodes.
//
// One thread per node, NODES = P^DIM threads per element "slot", EPB slots per
// CTA.  Every operator of the hot path is the same pass (eq:DGSEM_wt, P:179-189,
// on Cartesian elements, reading R2 for Dhat):
//
//   1. load the node state as a jet (mode-defined: W, W + e1 sigma, ...),
//   2. evaluate the volume flux per direction and reduce it to NCH real
//      "channels" (linear combinations fixed by the mode) -> shared memory,
//   3. boundary nodes evaluate the canonical LLF face flux with the
//      neighbour's trace (GLL: the neighbour's boundary node) and keep the
//      surface term  s_d * (f*_+ lhat_N(1) - f*_- lhat_0(-1))  in registers,
//   4. contract with Dhat along x and y from shared memory,
//        L_ch = -( sx (sum_l Dh_il F_lj + surf_x) + sy (sum_m Dh_jm F_im + surf_y) ),
//   5. mode epilogue combines L_ch with the node's inputs and stores.
//
// Because the contraction is linear, the mode combines the jet components
// BEFORE it (e.g. the EXACT JVP needs 2 contractions, not 5 operator
// evaluations).  Navier-Stokes adds BR1 lifted gradients (lift_kernel), read
// back as part of the node state.
#pragma once
#include <type_traits>
#include <cuda_runtime.h>
#include "physics.cuh"

__host__ __device__ constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

struct Geo {
  int nx, ny, nE;          // local element grid
  int hx, hy;              // 1: the -x/+x (-y/+y) neighbours are ghosts (halo), not a local wrap
  double sx, sy;           // 2/dx, 2/dy
  int nz;                  // 3D (NEXT-4): elements in z (single rank, periodic); 1 otherwise
  double sz;               // 2/dz
  double lhp, lhm;         // lhat_N(+1) = 1/w_N, lhat_0(-1) = 1/w_0  (GLL)
  double Dh[64];           // Dhat (P x P, row-major)
  int gl, P, dim;          // gl: Gauss-Legendre nodes (no node on the element edge)
  int br2;                 // NS with BR2 lifting (dispatches to the BR2 instantiations)
  double lp[8], lm[8];     // GL: l_i(+1), l_i(-1)  (traces)
  double lhpv[8], lhmv[8]; // GL: lhat_i(+1), lhat_i(-1)  (surface terms, eq:DGSEM_wt)
  double D[64];            // GL BR2: strong-form D_ij = l_j'(x_i)
  double dlp[8], dlm[8];   // GL BR2: l_j'(+1), l_j'(-1)
  double cp, cm;           // GL BR2: sum_i l_i(+-1) lhat_i(+-1)
  // restricted launches: cmode 0 = every element; 1 = the elements of colour (ccx, ccy) of the
  // period (cpx, cpy) colouring and 2 = those and their 4 neighbours (NS BJ_ext build); 3 = the
  // interior elements of a partitioned 2D block (no neighbour across a halo side) and 4 = the
  // boundary ring (halo / compute overlap: the interior runs while the halo is in flight)
  int cmode, cpx, cpy, ccx, ccy;
};

// elements a restricted launch covers (grid = ceil(count / EPB))
__host__ __device__ inline int launch_elems(const Geo& g) {
  if (g.cmode == 0) return g.nE;
  if (g.cmode >= 3) {
    const int ni = (g.nx - 2 * g.hx) * (g.ny - 2 * g.hy);
    return g.cmode == 3 ? ni : g.nE - ni;
  }
  const int nc = (g.nx / g.cpx) * (g.ny / g.cpy);
  return g.cmode == 1 ? nc : 5 * nc;
}

// k-th element of a (possibly restricted) launch; false past the end
__device__ __forceinline__ bool launch_elem(const Geo& g, int k, int& e) {
  if (g.cmode == 0) { e = k; return k < g.nE; }
  if (g.cmode >= 3) {
    const int wi = g.nx - 2 * g.hx, hi = g.ny - 2 * g.hy, ni = wi * hi;
    if (g.cmode == 3) {
      if (k >= ni) { e = 0; return false; }
      e = (g.hy + k / wi) * g.nx + g.hx + k % wi;
      return true;
    }
    if (k >= g.nE - ni) { e = 0; return false; }
    const int nrow = g.hy * g.nx;                 // first and last row (y halo sides)
    if (k < 2 * nrow) {
      const int r = k / g.nx;                    // 0 .. 2 hy - 1
      e = (r < g.hy ? r : g.ny - 2 * g.hy + r) * g.nx + k % g.nx;
      return true;
    }
    k -= 2 * nrow;                               // left / right columns of the middle rows
    const int c = k % (2 * g.hx), row = g.hy + k / (2 * g.hx);
    e = row * g.nx + (c < g.hx ? c : g.nx - 2 * g.hx + c);
    return true;
  }
  const int nxc = g.nx / g.cpx, nc = nxc * (g.ny / g.cpy);
  if (k >= (g.cmode == 1 ? nc : 5 * nc)) { e = 0; return false; }
  const int s = k / nc, kk = k % nc;
  int ex = g.ccx + g.cpx * (kk % nxc), ey = g.ccy + g.cpy * (kk / nxc);
  // neighbours by periodic wrap inside the local grid (consistent with the global
  // colouring: the local block sizes are multiples of the period)
  if (s == 1) ex = ex + 1 == g.nx ? 0 : ex + 1;
  if (s == 2) ex = ex == 0 ? g.nx - 1 : ex - 1;
  if (s == 3) ey = ey + 1 == g.ny ? 0 : ey + 1;
  if (s == 4) ey = ey == 0 ? g.ny - 1 : ey - 1;
  e = ey * g.nx + ex;
  return true;
}

// Node set selected at compile time (the GL kernels are a separate instantiation,
// ops_kernels_gl.cu, so the GLL hot path is compiled exactly as without GL).
template <bool GL_, bool BR2_ = false> struct GeoSel : Geo {
  static constexpr bool GL = GL_;
  static constexpr bool BR2 = BR2_;   // NS face gradients from the BR2 per-face buffers (reading R33)
};

// Face trace of a node state.  GLL: the edge node n itself.  GL: the
// line sum  sum_l l_l(+-1) S(line node l)  through n in direction d (the side
// is the edge n sits on), accumulated component-wise (a jet is linear in its
// components).  St is a plain aggregate of doubles; ld(node, St&) loads one node.
// A ghost element (ghost = true) already holds the trace at its edge node
// (halo.cu interpolates on the sending rank).
template <class G, class St, class Ld>
__device__ __forceinline__ void trace_load(const G& g, int n, int d, St& st, Ld ld, bool ghost = false) {
  if constexpr (G::GL) {
    if (ghost) { ld(n, st); return; }
    constexpr int NW = sizeof(St) / sizeof(double);
    const int P = g.P;
    const int i = n % P, j = g.dim == 2 ? n / P : 0;
    const bool plus = (d == 0 ? i : j) == P - 1;
    const double* l = plus ? g.lp : g.lm;
    double acc[NW];
#pragma unroll
    for (int q = 0; q < NW; ++q) acc[q] = 0.0;
#pragma unroll 1
    for (int k = 0; k < P; ++k) {
      const int nk = g.dim == 1 ? k : (d == 0 ? j * P + k : k * P + i);
      St t;
      double* tp = reinterpret_cast<double*>(&t);
#pragma unroll
      for (int q = 0; q < NW; ++q) tp[q] = 0.0;
      ld(nk, t);
#pragma unroll
      for (int q = 0; q < NW; ++q) acc[q] = fma(l[k], tp[q], acc[q]);
    }
    double* sp = reinterpret_cast<double*>(&st);
#pragma unroll
    for (int q = 0; q < NW; ++q) sp[q] = acc[q];
  } else {
    ld(n, st);
  }
}

// ---- neighbour addressing (periodic Cartesian, layout L) ----------------------
// Across a partition boundary (hx / hy) the neighbour is a ghost element
// nE + g, g = [-x: ey | +x: ny + ey | -y: 2ny + ex | +y: 2ny + nx + ex]
// (1D: ny = 1), whose face traces the halo exchange filled in (comm.h).
__device__ __forceinline__ int nbr_elem(const Geo& g, int e, int d, int side) {
  if (g.dim == 3) {              // 3D: e = (ez ny + ey) nx + ex, periodic wrap (one rank)
    int ex = e % g.nx, ey = (e / g.nx) % g.ny, ez = e / (g.nx * g.ny);
    if (d == 0) ex = side > 0 ? (ex + 1 == g.nx ? 0 : ex + 1) : (ex == 0 ? g.nx - 1 : ex - 1);
    else if (d == 1) ey = side > 0 ? (ey + 1 == g.ny ? 0 : ey + 1) : (ey == 0 ? g.ny - 1 : ey - 1);
    else ez = side > 0 ? (ez + 1 == g.nz ? 0 : ez + 1) : (ez == 0 ? g.nz - 1 : ez - 1);
    return (ez * g.ny + ey) * g.nx + ex;
  }
  int ex = e % g.nx, ey = e / g.nx;
  if (d == 0) {
    if (side > 0) {
      if (ex + 1 == g.nx) { if (g.hx) return g.nE + g.ny + ey; ex = 0; } else ++ex;
    } else {
      if (ex == 0) { if (g.hx) return g.nE + ey; ex = g.nx - 1; } else --ex;
    }
  } else {
    if (side > 0) {
      if (ey + 1 == g.ny) { if (g.hy) return g.nE + 2 * g.ny + g.nx + ex; ey = 0; } else ++ey;
    } else {
      if (ey == 0) { if (g.hy) return g.nE + 2 * g.ny + ex; ey = g.ny - 1; } else --ey;
    }
  }
  return ey * g.nx + ex;
}

// ---- node state: conserved variables + (NS) lifted gradients ------------------
template <int EQ, class T> struct NodeState {
  static constexpr int NV = NVars<EQ>::value;
  static constexpr int NG = EQ == 2 ? 3 : 1;
  T w[NV];
  T gx[NG], gy[NG];
};

// volume flux in all DIM directions (primitives computed once per state)
template <int EQ, int DIM, class T>
__device__ __forceinline__ void vol_flux_all(const PhysParams& pp, const NodeState<EQ, T>& s,
                                             T (&F)[DIM][NVars<EQ>::value]) {
  if constexpr (EQ == 0) {
#pragma unroll
    for (int d = 0; d < DIM; ++d) F[d][0] = adv_speed(pp, d) * s.w[0];
  } else if constexpr (EQ == 3) {
    const EulerPrim3<T> q = euler3_prim(pp, s.w);
#pragma unroll
    for (int d = 0; d < DIM; ++d) euler3_flux(s.w, q, d, F[d]);
  } else {
    const EulerPrim<T> q = euler_prim(pp, s.w);
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      euler_flux(s.w, q, d, F[d]);
      if constexpr (EQ == 2) {
        T Fv[4];
        viscous_flux_uv(pp, q.u, q.v, s.gx, s.gy, d, Fv);
#pragma unroll
        for (int v = 0; v < 4; ++v) F[d][v] = F[d][v] - Fv[v];
      }
    }
  }
}

template <int EQ, class T>
__device__ __forceinline__ void vol_flux(const PhysParams& pp, const NodeState<EQ, T>& s, int d, T* F) {
  phys_flux<EQ>(pp, s.w, d, F);
  if constexpr (EQ == 2) {
    T Fv[4];
    viscous_flux(pp, s.w, s.gx, s.gy, d, Fv);
#pragma unroll
    for (int v = 0; v < 4; ++v) F[v] = F[v] - Fv[v];
  }
}

template <int EQ, class T>
__device__ __forceinline__ void face_flux(const PhysParams& pp, const NodeState<EQ, T>& L,
                                          const NodeState<EQ, T>& R, int d, T* f) {
  llf_flux<EQ>(pp, L.w, R.w, d, f);
  if constexpr (EQ == 2) {
    T a[4], b[4];
    viscous_flux(pp, L.w, L.gx, L.gy, d, a);
    viscous_flux(pp, R.w, R.gx, R.gy, d, b);
#pragma unroll
    for (int v = 0; v < 4; ++v) f[v] = f[v] - 0.5 * (a[v] + b[v]);
  }
}

// ---- jet <-> flat storage helpers (lifting buffers) ---------------------------
template <class T> struct JetN { static constexpr int value = 1; };
template <> struct JetN<J1> { static constexpr int value = 2; };
template <> struct JetN<J2> { static constexpr int value = 3; };
template <> struct JetN<HJ> { static constexpr int value = 4; };
__device__ __forceinline__ double jget(const double& x, int k) { return x; }
__device__ __forceinline__ double jget(const J1& x, int k) { return k == 0 ? x.v : x.a; }
__device__ __forceinline__ double jget(const J2& x, int k) { return k == 0 ? x.v : (k == 1 ? x.a : x.b); }
__device__ __forceinline__ double jget(const HJ& x, int k) {
  return k == 0 ? x.v : (k == 1 ? x.a : (k == 2 ? x.b : x.c));
}
template <class T> __device__ __forceinline__ T jmake(const double* c);
template <> __device__ __forceinline__ double jmake<double>(const double* c) { return c[0]; }
template <> __device__ __forceinline__ J1 jmake<J1>(const double* c) { return {c[0], c[1]}; }
template <> __device__ __forceinline__ J2 jmake<J2>(const double* c) { return {c[0], c[1], c[2]}; }
template <> __device__ __forceinline__ HJ jmake<HJ>(const double* c) { return {c[0], c[1], c[2], c[3]}; }
template <class T> __device__ __forceinline__ T jzero_tangent(const T& x);
template <> __device__ __forceinline__ double jzero_tangent<double>(const double& x) { return x; }
template <> __device__ __forceinline__ J1 jzero_tangent<J1>(const J1& x) { return {x.v, 0.0}; }
template <> __device__ __forceinline__ J2 jzero_tangent<J2>(const J2& x) { return {x.v, 0.0, 0.0}; }
template <> __device__ __forceinline__ HJ jzero_tangent<HJ>(const HJ& x) { return {x.v, 0.0, 0.0, 0.0}; }

// Lifted-gradient buffer of one jet state: [elem][6][JetN][NODES]
template <class T, int NODES>
__device__ __forceinline__ void load_grads(const double* G, int e, int node, T* gx, T* gy) {
  constexpr int JN = JetN<T>::value;
  const double* base = G + (size_t)e * 6 * JN * NODES + node;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double c[JN];
#pragma unroll
    for (int q = 0; q < JN; ++q) c[q] = base[(k * JN + q) * NODES];
    if (k < 3) gx[k] = jmake<T>(c); else gy[k - 3] = jmake<T>(c);
  }
}

// ---- face flux in two halves -------------------------------------------------
// The canonical face flux needs each side's state, flux, wave speed (and NS
// viscous flux).  Computing the two sides on two threads and combining later
// balances the face work over all warps of an element (the combination below
// reproduces face_flux() operation for operation, so results are bitwise equal).
template <int EQ, class T> struct HalfFlux {
  static constexpr int NV = NVars<EQ>::value;
  T F[NV], w[NV], Fv[EQ == 2 ? 4 : 1];
  T lam;
};
template <int EQ, class T>
__host__ __device__ constexpr int half_doubles() {
  return JetN<T>::value * (2 * NVars<EQ>::value + 1 + (EQ == 2 ? 4 : 0));
}

template <int EQ, class T>
__device__ __forceinline__ void half_flux(const PhysParams& pp, const NodeState<EQ, T>& s, int d, double* raw,
                                          int rs) {
  constexpr int NV = NVars<EQ>::value, JN = JetN<T>::value;
  T F[NV], lam;
  if constexpr (EQ == 0) {
    phys_flux<EQ>(pp, s.w, d, F);
    lam = jconst<T>(0.0);
  } else if constexpr (EQ == 3) {
    const EulerPrim3<T> q = euler3_prim(pp, s.w);
    euler3_flux(s.w, q, d, F);
    lam = euler3_speed(pp, q, d);
  } else {
    const EulerPrim<T> q = euler_prim(pp, s.w);
    euler_flux(s.w, q, d, F);
    lam = euler_speed(pp, q, d);
  }
  int o = 0;
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int c = 0; c < JN; ++c) raw[rs * o++] = jget(F[v], c);
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int c = 0; c < JN; ++c) raw[rs * o++] = jget(s.w[v], c);
#pragma unroll
  for (int c = 0; c < JN; ++c) raw[rs * o++] = jget(lam, c);
  if constexpr (EQ == 2) {
    T Fv[4];
    viscous_flux(pp, s.w, s.gx, s.gy, d, Fv);
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int c = 0; c < JN; ++c) raw[rs * o++] = jget(Fv[v], c);
  }
}

// f = face_flux(L, R) from the two halves (same operations, same order)
template <int EQ, class T>
__device__ __forceinline__ void face_from_halves(const PhysParams& pp, const double* rL, const double* rR, int rs,
                                                 int d, T* f) {
  constexpr int NV = NVars<EQ>::value, JN = JetN<T>::value;
  auto rd = [&](const double* r, int idx) {
    double c[JN];
#pragma unroll
    for (int q = 0; q < JN; ++q) c[q] = r[rs * (idx * JN + q)];
    return jmake<T>(c);
  };
  T lam;
  if constexpr (EQ == 0) {
    lam = jconst<T>(fabs(adv_speed(pp, d)));
  } else {
    lam = pp.glf ? jconst<T>(1.0) : jmax(rd(rL, 2 * NV), rd(rR, 2 * NV));
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if (pp.glf) {       // as llf_flux: eq:Riemann with the constant Lambda, no 1/2 on the jump
      const double lv = EQ == 0 ? fabs(adv_speed(pp, d)) : ((v == 0 || v == NV - 1) ? pp.ieps : 1.0);
      f[v] = 0.5 * (rd(rL, v) + rd(rR, v)) + lv * (rd(rL, NV + v) - rd(rR, NV + v));
    } else {
      f[v] = 0.5 * (rd(rL, v) + rd(rR, v)) + 0.5 * lam * (rd(rL, NV + v) - rd(rR, NV + v));
    }
  }
  if constexpr (EQ == 2) {
#pragma unroll
    for (int v = 0; v < 4; ++v) f[v] = f[v] - 0.5 * (rd(rL, 2 * NV + 1 + v) + rd(rR, 2 * NV + 1 + v));
  }
}

// ---- per-thread asynchronous staging (cp.async, LDGSTS) of the neighbour face data a
// thread's face work item will read: issued before the volume flux, consumed after it,
// so the L2 latency of the neighbour loads hides behind the flux arithmetic.
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// modes that stage their neighbour face loads declare NSTAGE (doubles per thread) and
// prefetch(A, g, e, nb, nnode, part, stage, stride) / face_part_staged(...)
template <class M, class = void> struct Staged { static constexpr int value = 0; };
template <class M> struct Staged<M, std::void_t<decltype(M::NSTAGE)>> { static constexpr int value = M::NSTAGE; };

// modes whose epilogue also returns the node's sum of out1^2 (epilogue_ss)
template <class M, class = void> struct NormEpilogue : std::false_type {};
template <class M> struct NormEpilogue<M, std::void_t<decltype(M::NORM_EPILOGUE)>> : std::true_type {};

// argument packs carrying a device-resident FD step (OpArgs::d_epsw)
template <class A, class = void> struct HasDevEps : std::false_type {};
template <class A> struct HasDevEps<A, std::void_t<decltype(A::d_epsw)>> : std::true_type {};

// modes may evaluate their volume fluxes in two passes (VOL_PASSES = 2)
// modes whose epilogue inputs are prefetched before the element's first barrier
// (Mode::EpiPre, prefetch_epi, epilogue(A, e, node, out, pre)): the loads overlap the
// barrier wait, the surface terms and the contraction instead of stalling the epilogue
template <class M, class = void> struct HasEpiPre : std::false_type {};
template <class M> struct HasEpiPre<M, std::void_t<typename M::EpiPre>> : std::true_type {};
struct NoEpiPre {};
template <class M, class = void> struct EpiPreOf { using type = NoEpiPre; };
template <class M> struct EpiPreOf<M, std::void_t<typename M::EpiPre>> { using type = typename M::EpiPre; };
struct NoHook { __device__ void operator()() const {} };
template <class M, class = void> struct VolPasses { static constexpr int value = 1; };
template <class M> struct VolPasses<M, std::void_t<decltype(M::VOL_PASSES)>> {
  static constexpr int value = M::VOL_PASSES;
};

// ---- fp64 tensor-core contraction (mma.sync m8n8k4 f64: A row-major 8x4, B col-major 4x8;
// lane l holds A[l/4][l%4], B[l%4][l/4], C[l/4][2(l%4) + {0,1}])
// Per mode (measured in one session, r02e, C3): R1 57 -> 44 us, EXACT JVP 127 -> 124.9, FD JVP
// 159 -> 157 with the tensor-core contraction; the residual alone got slower (101.5 -> 109) and
// opted out (NO_DMMA) until the surface terms became the fifth k-step (round 2: residual 88 -> 78 us
// on the tensor cores).  The operators stay bound by the flux arithmetic, not the contraction.
#ifndef HBPDC_DMMA_CONTRACT
#define HBPDC_DMMA_CONTRACT 1
#endif
template <class M, class = void> struct NoDmma : std::false_type {};
template <class M> struct NoDmma<M, std::void_t<decltype(M::NO_DMMA)>> : std::true_type {};
template <int DIM, int P, class Mode = void>
constexpr bool kDmmaContract = HBPDC_DMMA_CONTRACT && DIM == 2 && P == 8 && !NoDmma<Mode>::value;
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// ---- the element evaluation (one slot, one node per thread) --------------------
// Shared scratch per slot: slot_doubles<...>() = volume-flux planes
// NCH*DIM*NV*P*(P+1) + face parts NFP*NFN*FPD.
//   phase 1  every thread: node state -> volume fluxes (NCH channels) -> smem
//   phase 2  the NFP x NFN face work items (a face node's flux split into NFP
//            parts: the two sides' half fluxes, or the two jet states of the FD
//            JVP), spread over all threads of the element -> raw parts in smem
//   phase 3  every thread: Dhat contraction; boundary nodes combine the parts
//            of their face(s) (Mode::face_combine) into the surface terms
// rows of a volume plane (x-lines of P nodes, padded to P + 1) and nodes per face
template <int DIM, int P> struct Dims {
  static constexpr int ROWS = DIM == 1 ? 1 : (DIM == 2 ? P : P * P);
  static constexpr int FN = ROWS;
  static constexpr int NODES = ROWS * P;
};

template <int EQ, int DIM, int P, class Mode>
__host__ __device__ constexpr int slot_doubles() {
  return Mode::NCH * DIM * NVars<EQ>::value * Dims<DIM, P>::ROWS * (P + 1) +
         Mode::NFP * 2 * DIM * Dims<DIM, P>::FN * Mode::FPD +
         Staged<Mode>::value * Dims<DIM, P>::NODES;      // per-thread staging [k][node]
}

template <int EQ, int DIM, int P, class Mode, class G, class Hook = NoHook>
__device__ __forceinline__ void eval_slot(const typename Mode::Args& A, const PhysParams& pp,
                                          const G& g, int e, int slot, int node, bool active,
                                          double* sF, double (&out)[Mode::NCH][NVars<EQ>::value],
                                          Hook pre_barrier = Hook{}) {
  constexpr int NV = NVars<EQ>::value;
  constexpr int NCH = Mode::NCH;
  constexpr int NFP = Mode::NFP;
  static_assert(DIM < 3 || !G::GL, "3D: Gauss-Lobatto nodes only");
  constexpr int PS = P + 1;                       // padded row stride (bank conflicts)
  constexpr int ROWS = Dims<DIM, P>::ROWS;        // x-lines per plane: 1 (1D), P (2D), P^2 (3D)
  constexpr int PLANE = ROWS * PS;                // one (ch, d, v) plane [k][j][i], i padded
  constexpr int FN = Dims<DIM, P>::FN;            // nodes per face
  constexpr int NFN = 2 * DIM * FN;               // face nodes per element
  double* sRaw = sF + NCH * DIM * NV * PLANE;     // [FPD][part][face node] (conflict-free)
  const int i = node % P;
  const int j = DIM >= 2 ? (node / P) % P : 0;
  const int kz = DIM == 3 ? node / (P * P) : 0;
  const int row = DIM == 3 ? kz * P + j : j;      // this node's x-line
  constexpr int NODES_ = Dims<DIM, P>::NODES;
  // staged only with one face item per thread (2D: P >= 8) and GLL (GL traces are line sums)
  constexpr int NST = (G::GL || NFP * NFN > NODES_) ? 0 : Staged<Mode>::value;
  double* sStage = sRaw + NFP * NFN * Mode::FPD + node;   // this thread's staging column [k * NODES_]
  auto face_item = [&](int it, int& part, int& fn, int& own, int& nb, int& nnode, int& d, bool& plus) {
    // face f: 0 = -x, 1 = +x, 2 = -y, 3 = +y (3D: 4 = -z, 5 = +z); node k along the face
    // (2D: the line index; 3D: x-faces k = kz P + j, y-faces kz P + i, z-faces j P + i)
    part = it / NFN; fn = it % NFN;
    const int f = fn / FN, k = fn % FN;
    d = f >> 1;
    plus = f & 1;
    const int own_edge = plus ? P - 1 : 0, nbr_edge = plus ? 0 : P - 1;
    if constexpr (DIM == 3) {
      const int a = k % P, b = k / P;
      own = d == 0 ? (b * P + a) * P + own_edge : (d == 1 ? (b * P + own_edge) * P + a : (own_edge * P + b) * P + a);
      nnode = d == 0 ? (b * P + a) * P + nbr_edge : (d == 1 ? (b * P + nbr_edge) * P + a : (nbr_edge * P + b) * P + a);
    } else {
      own = DIM == 1 ? own_edge : (d == 0 ? k * P + own_edge : own_edge * P + k);
      nnode = DIM == 1 ? nbr_edge : (d == 0 ? k * P + nbr_edge : nbr_edge * P + k);
    }
    nb = nbr_elem(g, e, d, plus ? +1 : -1);
  };
  if constexpr (NST > 0) {
    if (active && node < NFP * NFN) {
      int part, fn, own, nb, nnode, d;
      bool plus;
      face_item(node, part, fn, own, nb, nnode, d, plus);
      Mode::prefetch(A, e, own, nb, nnode, part, sStage, NODES_);
    }
    cp_async_commit();
  }

  if (active) {
    auto put = [&](const double (&cf)[DIM][NCH][NV]) {
#pragma unroll
      for (int d = 0; d < DIM; ++d)
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int v = 0; v < NV; ++v) sF[((c * DIM + d) * NV + v) * PLANE + row * PS + i] = cf[d][c][v];
    };
    if constexpr (VolPasses<Mode>::value == 2) {
      // two jet states evaluated one after the other, the first parked in this
      // node's own output slots (no barrier: the same thread reads them back)
      double cf[DIM][NCH][NV];
      Mode::template vol_pass0<DIM>(A, pp, e, node, cf);
      put(cf);
      double cg[DIM][NCH][NV];
#pragma unroll
      for (int d = 0; d < DIM; ++d)
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int v = 0; v < NV; ++v) cg[d][c][v] = sF[((c * DIM + d) * NV + v) * PLANE + row * PS + i];
      Mode::template vol_pass1<DIM>(A, pp, e, node, cg);
      put(cg);
    } else {
      typename Mode::State st;
      Mode::load(A, g, e, slot, node, st, false);
      double cf[DIM][NCH][NV];
      Mode::template vol<DIM>(A, pp, st, cf);
      put(cf);
    }
  }
  constexpr int NODES = NODES_;
  if constexpr (NST > 0) {
    if (active && node < NFP * NFN) {
      int part, fn, own, nb, nnode, d;
      bool plus;
      face_item(node, part, fn, own, nb, nnode, d, plus);
      cp_async_wait_all();
      Mode::face_part_staged(A, pp, g, e, own, nb, nnode, plus, d, part, sStage, NODES_, sRaw + part * NFN + fn,
                             NFP * NFN);
    }
  } else {
    for (int it = node; active && it < NFP * NFN; it += NODES) {
      int part, fn, own, nb, nnode, d;
      bool plus;
      face_item(it, part, fn, own, nb, nnode, d, plus);
      Mode::face_part(A, pp, g, e, own, nb, nnode, slot, plus, d, part, sRaw + part * NFN + fn, NFP * NFN);
    }
  }
  if (active) pre_barrier();
  __syncthreads();
  if (active && !kDmmaContract<DIM, P, Mode>) {
    // surface terms of this node's face(s), canonical flux with the outward sign:
    // s_d (f*_+ lhat_N(1) - f*_- lhat_0(-1)), summed in the order +x, -x, +y, -y
    double sf[NCH][NV];
#pragma unroll
    for (int c = 0; c < NCH; ++c)
#pragma unroll
      for (int v = 0; v < NV; ++v) sf[c][v] = 0.0;
    auto add_face = [&](int f, int k, double lh) {
      const int d = f >> 1;
      const int fn = f * FN + k;
      double cf[NCH][NV];
      Mode::face_combine(A, pp, d, sRaw + fn, sRaw + NFN + fn, NFP * NFN, cf);
      const double sc = (d == 0 ? g.sx : (d == 1 ? g.sy : g.sz)) * lh;
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int v = 0; v < NV; ++v) sf[c][v] += __dmul_rn(sc, cf[c][v]);
    };
    if constexpr (G::GL) {
      // Gauss-Legendre: every node receives all faces, weighted by lhat_i(+-1) (eq:DGSEM_wt)
#pragma unroll 1
      for (int f = 0; f < 2 * DIM; ++f) {
        const int d = f >> 1, plus = f & 1;
        const int t = d == 0 ? i : j;
        add_face(plus ? 1 + 2 * d : 2 * d, d == 0 ? j : i, plus ? g.lhpv[t] : -g.lhmv[t]);
      }
    } else if constexpr (DIM == 3) {
      if (i == P - 1) add_face(1, kz * P + j, g.lhp);
      if (i == 0) add_face(0, kz * P + j, -g.lhm);
      if (j == P - 1) add_face(3, kz * P + i, g.lhp);
      if (j == 0) add_face(2, kz * P + i, -g.lhm);
      if (kz == P - 1) add_face(5, j * P + i, g.lhp);
      if (kz == 0) add_face(4, j * P + i, -g.lhm);
    } else {
      if (i == P - 1) add_face(1, j, g.lhp);
      if (i == 0) add_face(0, j, -g.lhm);
      if (DIM == 2 && j == P - 1) add_face(3, i, g.lhp);
      if (DIM == 2 && j == 0) add_face(2, i, -g.lhm);
    }
    if constexpr (!kDmmaContract<DIM, P, Mode>) {
      double Dr[P], Dc[P], Dz[P];
#pragma unroll
      for (int l = 0; l < P; ++l) {
        Dr[l] = g.Dh[i * P + l];
        Dc[l] = DIM >= 2 ? g.Dh[j * P + l] : 0.0;
        Dz[l] = DIM == 3 ? g.Dh[kz * P + l] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double* Fx = sF + ((c * DIM + 0) * NV + v) * PLANE + row * PS;
          double ax = 0.0;
#pragma unroll
          for (int l = 0; l < P; ++l) ax = fma(Dr[l], Fx[l], ax);
          double acc = g.sx * ax;
          if constexpr (DIM >= 2) {
            const double* Fy = sF + ((c * DIM + 1) * NV + v) * PLANE + kz * P * PS + i;
            double ay = 0.0;
#pragma unroll
            for (int l = 0; l < P; ++l) ay = fma(Dc[l], Fy[l * PS], ay);
            acc = fma(g.sy, ay, acc);
          }
          if constexpr (DIM == 3) {
            const double* Fz = sF + ((c * DIM + 2) * NV + v) * PLANE + j * PS + i;
            double az = 0.0;
#pragma unroll
            for (int l = 0; l < P; ++l) az = fma(Dz[l], Fz[l * P * PS], az);
            acc = fma(g.sz, az, acc);
          }
          out[c][v] = -(acc + sf[c][v]);
        }
    }
  }
  if constexpr (kDmmaContract<DIM, P, Mode>) {
    // Volume contraction on the fp64 tensor cores (P = 8, 2D): per channel c and
    // variable v the element's 8 x 8 node plane gives
    //   V = sx F_x Dhat^T + sy Dhat F_y           (V_ji = sx sum_l Dhat_il Fx_jl + sy sum_m Dhat_jm Fy_mi)
    // as four mma.sync.m8n8k4.f64 (two k-steps per direction).  The two warps of
    // an element slot take alternate (c, v) planes; D stays in registers as
    // fragments; the result overwrites the F_x plane (node layout) and every
    // thread then reads its node's value back.
    //
    // The surface terms are a fifth k-step (k = +x, -x, +y, -y faces):
    //   V_ji += f*_{+x,j} sx lh+(i) - f*_{-x,j} sx lh-(i) + sy lh+(j) f*_{+y,i} - sy lh-(j) f*_{-y,i}
    // with lh+-(i) = lhat_i(+-1) (GLL: nonzero on the edge node only).  Lane L of each warp
    // combines the two parts of face node L (face L >> 3, node L & 7) -- warp-uniform, once per
    // lane, instead of divergent per-boundary-node face sums -- and the fragments are
    // gathered by shuffles.
    const int lane = threadIdx.x & 31, wslot = node >> 5;
    const int r = lane >> 2, q = lane & 3;
    if (active) {
      double fx0 = g.sx * g.Dh[r * P + q], fx1 = g.sx * g.Dh[r * P + q + 4];   // B = sx Dhat^T: (k = l, n = i)
      double fy0 = g.sy * g.Dh[r * P + q], fy1 = g.sy * g.Dh[r * P + q + 4];   // A = sy Dhat:   (m = j, k = m')
      double lhp_r, lhm_r;
      if constexpr (G::GL) { lhp_r = g.lhpv[r]; lhm_r = g.lhmv[r]; }
      else { lhp_r = r == P - 1 ? g.lhp : 0.0; lhm_r = r == 0 ? g.lhm : 0.0; }
      // constant halves of the fifth k-step: B rows k = 0, 1 (x faces), A columns k = 2, 3 (y faces)
      const double sconst = q == 0 ? g.sx * lhp_r : (q == 1 ? -(g.sx * lhm_r) : (q == 2 ? g.sy * lhp_r : -(g.sy * lhm_r)));
      double cfl[NCH][NV];
      Mode::face_combine(A, pp, lane >> 4, sRaw + lane, sRaw + NFN + lane, NFP * NFN, cfl);
      const int src = ((q ^ 1) << 3) | r;      // face slot q = +x, -x, +y, -y is face 1, 0, 3, 2
#pragma unroll
      for (int mi = 0; mi < NCH * NV; ++mi) {
        if (mi % (NODES / 32) != wslot) continue;     // warp-uniform
        const int c = mi / NV, v = mi % NV;
        const double fv = __shfl_sync(0xffffffffu, cfl[c][v], src);
        double* Fx = sF + ((c * DIM + 0) * NV + v) * PLANE;
        const double* Fy = sF + ((c * DIM + 1) * NV + v) * PLANE;
        double acc[2] = {0.0, 0.0};
        dmma_8x8x4(acc, Fx[r * PS + q], fx0);
        dmma_8x8x4(acc, Fx[r * PS + q + 4], fx1);
        dmma_8x8x4(acc, fy0, Fy[q * PS + r]);
        dmma_8x8x4(acc, fy1, Fy[(q + 4) * PS + r]);
        dmma_8x8x4(acc, q < 2 ? fv : sconst, q < 2 ? sconst : fv);
        __syncwarp();
        Fx[r * PS + 2 * q] = acc[0];
        Fx[r * PS + 2 * q + 1] = acc[1];
      }
    }
    __syncthreads();
    if (active) {
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int v = 0; v < NV; ++v)
          out[c][v] = -sF[((c * DIM + 0) * NV + v) * PLANE + row * PS + i];
    }
  }
}

#ifndef HBPDC_CTA_THREADS
#define HBPDC_CTA_THREADS 128
#endif
__host__ __device__ constexpr int epb_for(int nodes) {
  return nodes >= HBPDC_CTA_THREADS ? 1 : HBPDC_CTA_THREADS / nodes;
}

// Generic operator kernel: EPB element slots per CTA, one element per slot.
// HBPDC_MINB CTAs per SM are requested from ptxas (register cap).
#ifndef HBPDC_MINB
#define HBPDC_MINB 4
#endif
template <int EQ, int DIM, int P, class Mode, int EPB, bool GL, bool BR2>
__global__ void __launch_bounds__(EPB * ipow(P, DIM), HBPDC_MINB)
op_kernel(const typename Mode::Args A, const PhysParams pp, const GeoSel<GL, BR2> g) {
  constexpr int NODES = ipow(P, DIM);
  constexpr int NV = NVars<EQ>::value;
  extern __shared__ __align__(16) double sF[];     // EPB * slot_doubles (dynamic: may exceed 48 KB)
  constexpr int SLOT = slot_doubles<EQ, DIM, P, Mode>();
  const int slot = threadIdx.x / NODES, node = threadIdx.x % NODES;
  // restricted launches (cmode != 0): the NS BJ_ext colour passes, the interior / boundary
  // halves of a partitioned operator; cmode 0 is the plain element index
  int e;
  const bool active = launch_elem(g, blockIdx.x * EPB + slot, e);
  double out[Mode::NCH][NV];
  using Pre = typename std::conditional<HasEpiPre<Mode>::value, typename EpiPreOf<Mode>::type, NoEpiPre>::type;
  Pre pre;
  typename Mode::Args Al = A;
  if constexpr (HasDevEps<typename Mode::Args>::value) {
    // the FD step lives in device memory (norm computed on the device): read it once
    if (Al.d_epsw) { Al.epsw = __ldg(Al.d_epsw); Al.d_epsw = nullptr; }
    Al.iepsw = Al.epsw > 0.0 ? 1.0 / Al.epsw : 0.0;    // once per thread (was: per face and pass)
  }
  auto hook = [&]() {
    if constexpr (HasEpiPre<Mode>::value) Mode::prefetch_epi(Al, e, node, pre);
  };
  eval_slot<EQ, DIM, P, Mode>(Al, pp, g, e, slot, node, active, sF + slot * SLOT, out, hook);
  if constexpr (NormEpilogue<Mode>::value) {
    // per-CTA partial of sum(out1^2), fixed reduction order (warp tree, then warps in order)
    double ss = 0.0;
    if (active) {
      if constexpr (HasEpiPre<Mode>::value) ss = Mode::epilogue_ss(Al, e, node, out, pre);
      else ss = Mode::epilogue_ss(Al, e, node, out);
    }
    if (Al.nrm_part) {
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o2);
      __syncthreads();                              // sF is reused as the warp-sum scratch
      if ((threadIdx.x & 31) == 0) sF[threadIdx.x >> 5] = ss;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sF[w];
        Al.nrm_part[blockIdx.x] = t;
      }
    }
  } else {
    if (active) {
      if constexpr (HasEpiPre<Mode>::value) Mode::epilogue(Al, e, node, out, pre);
      else Mode::epilogue(Al, e, node, out);
    }
  }
}

// ---- BR1 lifting (eq:Lifting P:855, central value P:861; reading R19) -----------
//   d^x_ij = sx ( sum_l Dh_il g_lj + g*_E,j lhat_N(1) [i=N] - g*_W,j lhat_0(-1) [i=0] )
// Computed for jet state K of the mode; result [elem][6][JetN][NODES].
// CTAs per SM requested from ptxas for the lifting, by the jet width of the lifted state
// (measured on the C5 operators, r02w: R1 lift 334 -> 286 us at 8 for plain doubles, FD JVP
// 1650 -> 1605 us at 5 / 6 for the J1 / J2 states; the hyper-dual EXACT lift spills below 128)
template <class Mode, int K> struct LiftMinb {
  static constexpr int JN = JetN<typename Mode::template StateT<K>>::value;
  static constexpr int value = JN == 1 ? 8 : (JN == 2 ? 6 : (JN == 3 ? 5 : 1));
};
// BR2F: the BR2 per-face gradient output (Gf) is compiled in; the BR1 instantiations drop it
// (its unrolled face loops set the register count: J2 lift 144 -> 128 registers without it)
template <int P, class Mode, int K, int EPB, bool GL, bool BR2F = true>
__global__ void __launch_bounds__(EPB * P * P, (LiftMinb<Mode, K>::value))
lift_kernel(const typename Mode::Args A, const PhysParams pp, const GeoSel<GL> g, double* Gout, double* Gf,
            const double* gTg) {
  using T = typename Mode::template StateT<K>;
  constexpr int NODES = P * P, PS = P + 1, PLANE = P * PS;
  constexpr int JN = JetN<T>::value;
  __shared__ double sG[EPB * 3 * JN * PLANE];
  const int slot = threadIdx.x / NODES, node = threadIdx.x % NODES;
  int e;
  const bool active = launch_elem(g, blockIdx.x * EPB + slot, e);
  const int i = node % P, j = node / P;
  double* sg = sG + slot * 3 * JN * PLANE;
  T sx_[3], sy_[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) { sx_[k] = jconst<T>(0.0); sy_[k] = jconst<T>(0.0); }
  if constexpr (GL) {
    // Gauss-Legendre: g* = 1/2 (own + neighbour trace), traces sum_l l_l(+-1) g(w_l) of the
    // nodal gradient variables (oracle lifting()), on every node weighted by lhat(+-1)
    if (active) {
      T w[4], gv[3];
      Mode::template load_w<K>(A, e, node, w, false);
      grad_vars(pp, w, gv);
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int q = 0; q < JN; ++q) sg[(k * JN + q) * PLANE + j * PS + i] = jget(gv[k], q);
    }
    __syncthreads();
    if (active) {
#pragma unroll 1
      for (int f = 0; f < 4; ++f) {
        const int d = f >> 1, side = (f & 1) ? +1 : -1;
        const double* lo = side > 0 ? g.lp : g.lm;      // own trace on this face
        const double* ln = side > 0 ? g.lm : g.lp;      // the neighbour's opposite face
        const int nb = nbr_elem(g, e, d, side);
        double own[3][JN], nbr[3][JN];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int q = 0; q < JN; ++q) { own[k][q] = 0.0; nbr[k][q] = 0.0; }
        const bool ghost = nb >= g.nE;      // across a partition: the sender's g-trace (gtrace_kernel)
#pragma unroll 1
        for (int l = 0; l < P; ++l) {
          const int ii = d == 0 ? l : i, jj = d == 0 ? j : l;
#pragma unroll
          for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int q = 0; q < JN; ++q) own[k][q] = fma(lo[l], sg[(k * JN + q) * PLANE + jj * PS + ii], own[k][q]);
          if (ghost) continue;
          T wn[4], gn[3];
          Mode::template load_w<K>(A, nb, jj * P + ii, wn, true);
          grad_vars(pp, wn, gn);
#pragma unroll
          for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int q = 0; q < JN; ++q) nbr[k][q] = fma(ln[l], jget(gn[k], q), nbr[k][q]);
        }
        if (ghost) {
          const double* tg = gTg + ((size_t)(nb - g.nE) * 4 + (f ^ 1)) * 3 * JN * P + (d == 0 ? j : i);
#pragma unroll
          for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int q = 0; q < JN; ++q) nbr[k][q] = tg[(k * JN + q) * P];
        }
        const int t = d == 0 ? i : j;
        const double s = (d == 0 ? g.sx : g.sy) * (side > 0 ? g.lhpv[t] : -g.lhmv[t]);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const T go = jmake<T>(own[k]), gn = jmake<T>(nbr[k]);
          const T gs = side > 0 ? 0.5 * (go + gn) : 0.5 * (gn + go);
          if (d == 0) sx_[k] = sx_[k] + s * gs; else sy_[k] = sy_[k] + s * gs;
        }
        if (BR2F && Gf && t == (side > 0 ? P - 1 : 0)) {
          // BR2 on GL (reading R33): the face point kf of this line; normal component
          // l'(+-1).g along d + eta s_d (+-c) (g* - g_f), tangential the trace of (2/h) D g
          const int kf = d == 0 ? j : i;
          const double* dl = side > 0 ? g.dlp : g.dlm;
          const double sd = d == 0 ? g.sx : g.sy, st = d == 0 ? g.sy : g.sx;
          const double cj = side > 0 ? g.cp : -g.cm;
          double* fo = Gf + ((size_t)e * 4 + f) * 6 * JN * P + kf;
#pragma unroll
          for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int q = 0; q < JN; ++q) {
              const double* row = sg + (k * JN + q) * PLANE;
              double an = 0.0, at = 0.0;
#pragma unroll 1
              for (int l = 0; l < P; ++l) {
                // line node l across the face direction; tangential derivative at (l, kf)
                const int ii = d == 0 ? l : kf, jj = d == 0 ? kf : l;
                an = fma(dl[l], row[jj * PS + ii], an);
                double dt = 0.0;
                for (int m2 = 0; m2 < P; ++m2)
                  dt = fma(g.D[kf * P + m2], d == 0 ? row[m2 * PS + ii] : row[jj * PS + m2], dt);
                at = fma(lo[l], dt, at);
              }
              const double gst = side > 0 ? 0.5 * (own[k][q] + nbr[k][q]) : 0.5 * (nbr[k][q] + own[k][q]);
              const double vn = fma(pp.eta_br2 * sd * cj, gst - own[k][q], sd * an);
              fo[((d * 3 + k) * JN + q) * P] = vn;
              fo[(((1 - d) * 3 + k) * JN + q) * P] = st * at;
            }
        }
      }
    }
  }
  T gsd[2][3];                       // GLL: g* on this node's x / y face (BR2 face gradients)
#pragma unroll
  for (int d = 0; d < 2; ++d)
#pragma unroll
    for (int k = 0; k < 3; ++k) gsd[d][k] = jconst<T>(0.0);
  if (!GL && active) {
    T w[4], gv[3];
    Mode::template load_w<K>(A, e, node, w, false);
    grad_vars(pp, w, gv);
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int q = 0; q < JN; ++q) sg[(k * JN + q) * PLANE + j * PS + i] = jget(gv[k], q);
    for (int d = 0; d < 2; ++d) {
      const int kk = d == 0 ? i : j;
      if (kk == P - 1 || kk == 0) {
        const int side = kk == P - 1 ? +1 : -1;
        const int nb = nbr_elem(g, e, d, side);
        const int nnode = side > 0 ? (d == 0 ? j * P : i) : (d == 0 ? j * P + P - 1 : (P - 1) * P + i);
        T wn[4], gn[3];
        Mode::template load_w<K>(A, nb, nnode, wn, true);
        grad_vars(pp, wn, gn);
        const double s = (d == 0 ? g.sx : g.sy) * (side > 0 ? g.lhp : -g.lhm);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const T gs = side > 0 ? 0.5 * (gv[k] + gn[k]) : 0.5 * (gn[k] + gv[k]);
          gsd[d][k] = gs;
          if (d == 0) sx_[k] = sx_[k] + s * gs; else sy_[k] = sy_[k] + s * gs;
        }
      }
    }
  }
  __syncthreads();
  if constexpr (!GL) {
    // BR2 (reading R33): on each face of this edge node, the strong-form gradient
    // (2/h) D g (D = Dhat + M^-1 B) plus, in the normal component, eta (2/h) (+-) lhat (g* - g)
    if (BR2F && Gf && active) {
#pragma unroll 1
      for (int d = 0; d < 2; ++d) {
        const int kk = d == 0 ? i : j;
        if (kk != P - 1 && kk != 0) continue;
        const int side = kk == P - 1 ? +1 : -1;
        double* fo = Gf + ((size_t)e * 4 + 2 * d + (side > 0 ? 1 : 0)) * 6 * JN * P + (d == 0 ? j : i);
        const double sd = d == 0 ? g.sx : g.sy;
        const double lj = side > 0 ? g.lhp : -g.lhm;
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int q = 0; q < JN; ++q) {
            const double* row = sg + (k * JN + q) * PLANE;
            const double gown = row[j * PS + i];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int ic = c == 0 ? i : j;
              double a = 0.0;
#pragma unroll
              for (int l = 0; l < P; ++l) a = fma(g.Dh[ic * P + l], c == 0 ? row[j * PS + l] : row[l * PS + i], a);
              if (ic == P - 1) a = fma(g.lhp, gown, a);
              if (ic == 0) a = fma(-g.lhm, gown, a);
              double v = (c == 0 ? g.sx : g.sy) * a;
              if (c == d) v = fma(pp.eta_br2 * sd * lj, jget(gsd[d][k], q) - gown, v);
              fo[((c * 3 + k) * JN + q) * P] = v;
            }
          }
      }
    }
  }
  if (active) {
    double* out = Gout + (size_t)e * 6 * JN * NODES + node;
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int q = 0; q < JN; ++q) {
        const double* row = sg + (k * JN + q) * PLANE;
        double ax = 0.0, ay = 0.0;
#pragma unroll
        for (int l = 0; l < P; ++l) {
          ax = fma(g.Dh[i * P + l], row[j * PS + l], ax);
          ay = fma(g.Dh[j * P + l], row[l * PS + i], ay);
        }
        out[(k * JN + q) * NODES] = g.sx * ax + jget(sx_[k], q);
        out[((k + 3) * JN + q) * NODES] = g.sy * ay + jget(sy_[k], q);
      }
  }
}

// ---- GL Navier-Stokes across partitions: face traces of g(w) ----------------------
// T[e][face f][3][JetN][P] = sum_l l_l(+-1) g(w_l) along the line through face point kf
// (the same accumulation order as the local neighbour trace in lift_kernel), exchanged
// by the face-buffer halo so that a rank's lift reads its neighbours' g-traces.
template <int P, class Mode, int K>
__global__ void gtrace_kernel(const typename Mode::Args A, const PhysParams pp, const Geo g, double* Tg) {
  using T = typename Mode::template StateT<K>;
  constexpr int JN = JetN<T>::value;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.nE * 4 * P) return;
  const int kf = t % P, f = (t / P) % 4, e = t / (4 * P);
  const int d = f >> 1;
  const double* l = (f & 1) ? g.lp : g.lm;
  double acc[3][JN];
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int q = 0; q < JN; ++q) acc[k][q] = 0.0;
  for (int m = 0; m < P; ++m) {
    const int ii = d == 0 ? m : kf, jj = d == 0 ? kf : m;
    T wn[4], gn[3];
    Mode::template load_w<K>(A, e, jj * P + ii, wn, false);
    grad_vars(pp, wn, gn);
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int q = 0; q < JN; ++q) acc[k][q] = fma(l[m], jget(gn[k], q), acc[k][q]);
  }
  double* o = Tg + ((size_t)e * 4 + f) * 3 * JN * P + kf;
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int q = 0; q < JN; ++q) o[(k * JN + q) * P] = acc[k][q];
}

// ---- GL face traces of the FD JVP inputs: Tr[e][face][field][v][k] = sum_l l_l(+-1) X(line node l),
// fields W, sigma, dW, dsigma; one thread per (element, face, face node).  The FD JVP's GL face work then
// reads one value per trace instead of a line sum per face node and jet state.
template <int P, int NV>
__global__ void gl_trace_kernel(const double* __restrict__ W, const double* __restrict__ S,
                                const double* __restrict__ dW, const double* __restrict__ dS, const Geo g,
                                double* __restrict__ Tr) {
  constexpr int NODES = P * P, m = NV * NODES;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.nE * 4 * P) return;
  const int k = t % P, f = (t / P) % 4, e = t / (4 * P);
  const int d = f >> 1;
  const double* l = (f & 1) ? g.lp : g.lm;
  const double* src[4] = {W, S, dW, dS};
  double* out = Tr + ((size_t)e * 4 + f) * 4 * NV * P + k;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double* x = src[q] + (size_t)e * m + v * NODES;
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < P; ++i) acc = fma(l[i], x[d == 0 ? k * P + i : i * P + k], acc);
      out[(q * NV + v) * P] = acc;
    }
}


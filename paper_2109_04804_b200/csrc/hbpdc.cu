// hbpdc.cu -- C-ABI implementation: context, operators, BJ_ext, GMRES, Newton,
// and the HBPC(q, k_max) step (Alg. 1).  The host runs the control
// flow; every vector operation runs in the kernels of ops_kernels.cu / linalg.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include "../../include/hbpdc.h"
#include "comm.h"
#include "launch.h"
#include "modes.cuh"

namespace hbpdc {
struct Basis1D {
  int N;
  int gl;
  std::vector<double> xi, w, Dhat;
  double lhp, lhm;
  std::vector<double> lp, lm;
  std::vector<double> lhpv, lhmv;
  std::vector<double> D;
  std::vector<double> dlp, dlm;
};
Basis1D gll_basis(int N);
Basis1D gl_basis(int N);
}  // namespace hbpdc

namespace {

// ---- HBPC tableaux (App. A, eq:butcher4/6/8) ------------------------
struct Tableau {
  int s;
  double c[4], B1[4][4], B2[4][4];
};

Tableau tableau(int q) {
  Tableau t{};
  auto set = [&](int s, std::initializer_list<double> c, std::initializer_list<double> b1,
                 std::initializer_list<double> b2) {
    t.s = s;
    int i = 0;
    for (double v : c) t.c[i++] = v;
    i = 0;
    for (double v : b1) { t.B1[i / s][i % s] = v; ++i; }
    i = 0;
    for (double v : b2) { t.B2[i / s][i % s] = v; ++i; }
  };
  if (q == 4) {
    set(2, {0.0, 1.0}, {0, 0, 1.0 / 2, 1.0 / 2}, {0, 0, 1.0 / 12, -1.0 / 12});
  } else if (q == 6) {
    set(3, {0.0, 0.5, 1.0},
        {0, 0, 0, 101.0 / 480, 8.0 / 30, 55.0 / 2400, 7.0 / 30, 16.0 / 30, 7.0 / 30},
        {0, 0, 0, 65.0 / 4800, -25.0 / 600, -25.0 / 8000, 5.0 / 300, 0.0, -5.0 / 300});
  } else {
    set(4, {0.0, 1.0 / 3, 2.0 / 3, 1.0},
        {0, 0, 0, 0, 6893.0 / 54432, 313.0 / 2016, 89.0 / 2016, 397.0 / 54432, 223.0 / 1701, 20.0 / 63,
         13.0 / 63, 20.0 / 1701, 31.0 / 224, 81.0 / 224, 81.0 / 224, 31.0 / 224},
        {0, 0, 0, 0, 1283.0 / 272160, -851.0 / 30240, -269.0 / 30240, -163.0 / 272160, 43.0 / 8505,
         -16.0 / 945, -19.0 / 945, -8.0 / 8505, 19.0 / 3360, -9.0 / 1120, 9.0 / 1120, -19.0 / 3360});
  }
  return t;
}

constexpr double EPS_MACH = 2.220446049250313e-16;   // 2^-52 (reading R7)
constexpr int NPROF = 8;

struct DevBuf {
  double* p = nullptr;
  size_t n = 0;
};

}  // namespace

// Newton / GMRES workspace of one stage system (NEXT-1 solves the s-1
// corrector stages of a sweep in lock step, one workspace each)
struct SysWS {
  double *X = nullptr, *G = nullptr, *dX = nullptr, *rhs = nullptr, *r = nullptr, *zb = nullptr;
  double *b = nullptr;                      // Newton right-hand side b (n)
  double *U = nullptr, *V = nullptr;        // BJ_ext GEMV outputs (n each)
  double* ky = nullptr;                     // NS: U - a1dt V, the second K right-hand side (n)
  double *ks = nullptr, *ks2 = nullptr;     // Schur mode: K v and a discarded JVP half (n each)
  double* npart = nullptr;                  // K-apply per-CTA partials of ||out1||^2 ...
  const double* npart_of = nullptr;         // ... valid for this vector (the next FD JVP's dW)
  double *Vk = nullptr;                     // Krylov basis: vk_cap x 2n, grown on demand up to restart+1
  size_t vk_cap = 0;
  double *partial = nullptr, *dh = nullptr, *dy = nullptr, *dnrm = nullptr;
  double *gW = nullptr, *gS = nullptr;      // ghosts of its linearisation point (halo)
  double* hpin = nullptr;                   // pinned host scratch
  std::vector<double> H, Hraw, cs, sn, gv, y;
};

struct hbpdc_ctx {
  hbpdc_problem pb{};
  hbpdc_solver_opts op{};
  hbpdc_dist ds{};
  int nv = 1, P = 2, nodes = 2, m = 2, nE = 0, nxl = 0, nyl = 0, nzl = 1, ex0 = 0, ey0 = 0;
  size_t n = 0;          // W-DOF on this rank
  Geo geo{};
  Geo geo_abs{};         // |Dhat|, -lhat_0(-1): R1_abs (rounding scale, reading R10b)
  OpCfg cfg{};
  hbpdc::Basis1D basis;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  Tableau tab{};
  int restart = 0;
  int sstep = 1;                   // s-step Arnoldi block size (1: DCGS2)
  // device memory
  std::vector<void*> allocs;
  std::vector<SysWS> sys;      // Newton/GMRES workspaces: [0] always, s-1 of them for batched correctors
  double *partial = nullptr;   // RED_BLOCKS partial sums (norms)
  double *dnrm = nullptr, *deps = nullptr;
  double *Sb = nullptr, *gSb = nullptr;   // BJ^H_ext: sigma at the build point, R1(Wb), and its ghosts
  double *lift0 = nullptr, *lift1 = nullptr;
  double* liftB = nullptr;        // NS BJ_ext build: lifted gradients of the build state (ModeKNS)
  double *gGb = nullptr, *gzero = nullptr;   // their ghost copies; a zero ghost field (partitioned ModeKNS)
  double *liftf0 = nullptr, *liftf1 = nullptr;   // BR2 per-face gradients (NULL: BR1)
  // precond
  double *S = nullptr, *Wb = nullptr, *Z = nullptr;
  double *Kst = nullptr, *KV = nullptr, *KT = nullptr, *tseed = nullptr, *y1 = nullptr, *y2 = nullptr;  // NS
  double *y3 = nullptr, *yz = nullptr, *yb = nullptr;   // NS BJ^H_ext build: H e_c output, zero dsigma, scratch
  int* info = nullptr;
  int s_shared = 0, pc_valid = 0, zchunk = 0;
  int kst_step = 0;                // NS: Kst holds the K_i of this step's W^n (built by ensure_pc_for)
  double pc_a1 = 0, pc_a2 = 0, pc_dt = -1;
  // stage store: [sweep(2)][s] of w, R1, R2
  double *stw[2][4] = {}, *str1[2][4] = {}, *str2[2][4] = {};
  double *Wn = nullptr, *Wio = nullptr;
  int fsal_valid = 0;
  const double* fsal_ptr = nullptr;      // the W the FSAL cache belongs to (the last step's output)
  unsigned long long* dfp = nullptr;     // device fingerprints: [0] last output, [1] incoming W
  int* dadm = nullptr;                   // admissibility flags (launch_admissible)
  int* hadm = nullptr;                   // pinned host copy
  double* hpin = nullptr;      // pinned host scratch (norms)
  // profiling
  int prof_on = 0;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_rec;
  long long prof_launch[NPROF] = {};
  double prof_ms[NPROF] = {};
  double prof_bytes[NPROF] = {};   // algorithmic bytes (DESIGN.md byte model)
  hbpdc_step_stats* st = nullptr;  // stats of the step in progress
  // element partition
  hbpdc::Comm* comm = nullptr;     // nullptr: single rank, no halo
  // halo / compute overlap (partitioned 2D, advection / Euler): the exchange runs on cstream while
  // the interior elements are computed on the main stream; the boundary ring follows (HBPDC_OVERLAP=0: off)
  bool overlap = false;
  double* gltr = nullptr;          // GL FD JVP face traces (launch_gl_traces)
  bool gl_notrace = false;         // HBPDC_GL_TRACES=0: line sums per face node (round 1)
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  int nbr[4] = {0, 0, 0, 0};       // neighbour ranks -x, +x, -y, +y
  HaloLayout hl{};
  double *gW = nullptr, *gS = nullptr, *gdW = nullptr, *gdS = nullptr, *gWb = nullptr;  // ghosts
  double *gG0 = nullptr, *gG1 = nullptr;                  // NS: ghost lifted gradients (second halo)
  double *gGf0 = nullptr, *gGf1 = nullptr;                // NS BR2: ghost face gradients
  double *tg0 = nullptr, *tg1 = nullptr, *gtg0 = nullptr, *gtg1 = nullptr;   // NS GL: g(w) face traces + ghosts
  double *hsend = nullptr, *hrecv = nullptr;
  bool halo() const { return hl.active[0] || hl.active[2]; }
  int debug_sync = 0;              // HBPDC_DEBUG_SYNC=1: synchronise + check after every launch group
  int trace = 0;                   // HBPDC_TRACE=1: per stage / Newton / GMRES trace on stderr
  int fuse_cgs = 1;                // HBPDC_FUSE_CGS=0: unfused block CGS2 passes (A/B checks)
  double sel_reorth = 1e-12;       // s = 8 block CGS: skip the second update when |C2 Rw^-1| <= this (0: never;
                                   // HBPDC_SEL_REORTH, reading R37)
  long long blk_count = 0, blk_skip = 0, blk_hist[6] = {0, 0, 0, 0, 0, 0};  // trace: max|C2 Rw^-1| by decade
};

namespace {

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      c->err = std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call;     \
      return e_ == cudaErrorMemoryAllocation ? HBPDC_E_OOM : HBPDC_E_CUDA;              \
    }                                                                                   \
  } while (0)
#define CKS(call)                          \
  do {                                     \
    hbpdc_status s_ = (call);              \
    if (s_ != HBPDC_OK) return s_;         \
  } while (0)

hbpdc_status fail(hbpdc_ctx* c, hbpdc_status s, const std::string& msg) {
  c->err = msg;
  return s;
}

hbpdc_status dalloc(hbpdc_ctx* c, double** p, size_t n) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, (n ? n : 1) * sizeof(double));
  if (e != cudaSuccess) {
    cudaGetLastError();
    char buf[160];
    snprintf(buf, sizeof buf, "cudaMalloc of %zu doubles failed: %s", n, cudaGetErrorString(e));
    c->err = buf;
    return HBPDC_E_OOM;
  }
  c->allocs.push_back(q);
  *p = (double*)q;
  return HBPDC_OK;
}

// profiling helpers (CUDA events on the context stream)
// NVTX ranges (header-only NVTX3: no-ops unless a tool such as ncu/nsys injects itself)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
static const char* const kProfName[8] = {"precond GEMV", "JVP", "residual", "Arnoldi dots",
                                         "Arnoldi update", "precond K-apply", "precond build",
                                         "Arnoldi update+dots"};

struct ProfScope {
  hbpdc_ctx* c;
  int id;
  cudaEvent_t a = nullptr, b = nullptr;
  NvtxRange nv;
  ProfScope(hbpdc_ctx* c_, int id_, double alg_bytes = 0.0) : c(c_), id(id_), nv(kProfName[id_ & 7]) {
    if (!c->prof_on) return;
    c->prof_bytes[id] += alg_bytes;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, c->stream);
  }
  ~ProfScope() {
    if (!c->prof_on) return;
    cudaEventRecord(b, c->stream);
    c->prof_rec.push_back({id, {a, b}});
  }
};

void prof_flush(hbpdc_ctx* c) {
  if (c->prof_rec.empty()) return;
  cudaStreamSynchronize(c->stream);
  for (auto& r : c->prof_rec) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.second.first, r.second.second);
    c->prof_ms[r.first] += ms;
    c->prof_launch[r.first] += 1;
    cudaEventDestroy(r.second.first);
    cudaEventDestroy(r.second.second);
  }
  c->prof_rec.clear();
}

OpArgs base_args(hbpdc_ctx* c) {
  OpArgs A{};
  A.m = c->m;
  A.nE = c->nE;
  return A;
}

// debugging aid: with HBPDC_DEBUG_SYNC=1 every operator / exchange is followed
// by a stream synchronisation, so an asynchronous fault names its call site
hbpdc_status dbg_sync(hbpdc_ctx* c, const char* where) {
  if (!c->debug_sync) return HBPDC_OK;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, HBPDC_E_CUDA, std::string("CUDA error after ") + where + ": " + cudaGetErrorString(e));
  return HBPDC_OK;
}

// sum over ranks of n doubles in device memory (no-op on a single rank)
hbpdc_status allreduce(hbpdc_ctx* c, double* d, int n) {
  if (!c->comm) return HBPDC_OK;
  std::string e;
  if (c->comm->allreduce_sum(d, n, c->stream, e)) return fail(c, HBPDC_E_NCCL, e);
  return HBPDC_OK;
}

// halo exchange of nf fields into their ghost copies
hbpdc_status halo_exchange(hbpdc_ctx* c, int nf, const double* const* src, double* const* dst, int nvf = 0,
                           bool facebuf = false) {
  size_t off[4], len[4];
  halo_segments(c->hl, nf, off, len, nvf);
  CK(launch_halo_pack(c->hl, nf, src, c->hsend, c->stream, nvf, facebuf));
  CKS(dbg_sync(c, "halo pack"));
  std::string e;
  if (c->comm->halo(c->hsend, c->hrecv, off, len, c->nbr, c->hl.active, c->stream, e))
    return fail(c, HBPDC_E_NCCL, e);
  CKS(dbg_sync(c, "halo transport"));
  CK(launch_halo_unpack(c->hl, nf, c->hrecv, dst, c->stream, nvf, facebuf));
  CKS(dbg_sync(c, "halo unpack"));
  return HBPDC_OK;
}

// fields of an operator that neighbours read (bits: 1 W, 2 sigma, 4 dW, 8 dsigma)
int halo_fields(OpKind k) {
  switch (k) {
    case OP_R1: case OP_R1ABS: return 1;
    case OP_R12: case OP_RESID: return 3;
    case OP_JVP_EXACT: case OP_JVP_FD: return 15;
    case OP_JVP_LINEAR: return 12;
    default: return 0;
  }
}

// launch an operator; exchange the halos of the fields in `xmask` first (the
// ghosts of the other fields are assumed current); NS lifts the jet states first
hbpdc_status run_op(hbpdc_ctx* c, OpKind k, OpArgs A, int xmask = -1) {
  if (k == OP_JVP_FD && c->geo.gl && c->pb.equation != HBPDC_NAVIER_STOKES && c->pb.dim == 2 && !c->gl_notrace) {
    // Gauss-Legendre FD JVP: the elements' face traces once, read by the face work (one value per trace)
    if (!c->gltr) CKS(dalloc(c, &c->gltr, (size_t)c->nE * 4 * 4 * c->nv * c->P));
    CK(launch_gl_traces(c->cfg, c->geo, A, c->gltr));
    A.Tr = c->gltr;
  }
  if (c->halo()) {
    if (xmask < 0) xmask = halo_fields(k);
    xmask &= halo_fields(k);
    const double* src[4];
    double* dst[4];
    int nf = 0;
    if (xmask & 1) { src[nf] = A.W; dst[nf++] = c->gW; }
    if (xmask & 2) { src[nf] = A.S; dst[nf++] = c->gS; }
    if (xmask & 4) { src[nf] = A.dW; dst[nf++] = c->gdW; }
    if (xmask & 8) { src[nf] = A.dS; dst[nf++] = c->gdS; }
    A.gW = (k == OP_KAPPLY || k == OP_KNS) ? c->gWb : c->gW;
    A.gS = k == OP_KNS ? c->gzero : c->gS;     // ModeKNS: no seed on the neighbours' ghosts
    A.gdW = c->gdW; A.gdS = c->gdS;
    if (nf && c->overlap && c->geo.cmode == 0 && c->pb.equation != HBPDC_NAVIER_STOKES) {
      // halo / compute overlap: pack + transport + unpack on the comm stream while
      // the interior elements (no neighbour across a halo side) run on the main stream
      size_t off[4], len[4];
      halo_segments(c->hl, nf, off, len, 0);
      CK(cudaEventRecord(c->ev_ready, c->stream));
      CK(cudaStreamWaitEvent(c->cstream, c->ev_ready, 0));
      CK(launch_halo_pack(c->hl, nf, src, c->hsend, c->cstream, 0, false));
      Geo gi = k == OP_R1ABS ? c->geo_abs : c->geo;
      gi.cmode = 3;
      CK(launch_op(k, c->cfg, gi, A));
      std::string e;
      if (c->comm->halo(c->hsend, c->hrecv, off, len, c->nbr, c->hl.active, c->cstream, e))
        return fail(c, HBPDC_E_NCCL, e);
      CK(launch_halo_unpack(c->hl, nf, c->hrecv, dst, c->cstream, 0, false));
      CK(cudaEventRecord(c->ev_halo, c->cstream));
      CK(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
      Geo gb = k == OP_R1ABS ? c->geo_abs : c->geo;
      gb.cmode = 4;
      CK(launch_op(k, c->cfg, gb, A));
      CKS(dbg_sync(c, "overlapped operator"));
      return HBPDC_OK;
    }
    if (nf) CKS(halo_exchange(c, nf, src, dst));
  }
  if (c->pb.equation == HBPDC_NAVIER_STOKES) {
    // BR1: lift the jet state(s), then (partitioned) exchange the lifted
    // gradients' face traces -- the second halo of the radius-2 stencil
    const double *gtg0 = nullptr, *gtg1 = nullptr;
    if (c->halo() && c->geo.gl) {
      // GL across partitions: the neighbours' face traces of g(w) for the lifting's central value
      CK(launch_gtrace(k, 0, c->cfg, c->geo, A, c->tg0));
      const double* t0[1] = {c->tg0};
      double* u0[1] = {c->gtg0};
      CKS(halo_exchange(c, 1, t0, u0, 3 * lift_jet_components(k, 0), true));
      gtg0 = c->gtg0;
      if (k == OP_JVP_FD) {
        CK(launch_gtrace(k, 1, c->cfg, c->geo, A, c->tg1));
        const double* t1[1] = {c->tg1};
        double* u1[1] = {c->gtg1};
        CKS(halo_exchange(c, 1, t1, u1, 3 * lift_jet_components(k, 1), true));
        gtg1 = c->gtg1;
      }
    }
    Geo lg = c->geo;                 // a colour-restricted operator needs the lifting on the
    if (lg.cmode == 1 && k != OP_KNS) lg.cmode = 2;   // colour's elements and their neighbours
                                     // (OP_KNS: the colour's elements only, ModeKNS)
    CK(launch_lift(k, 0, c->cfg, lg, A, c->lift0, c->liftf0, gtg0));
    A.G0 = c->lift0;
    A.Gf0 = c->liftf0;
    if (k == OP_JVP_FD) {
      CK(launch_lift(k, 1, c->cfg, lg, A, c->lift1, c->liftf1, gtg1));
      A.G1 = c->lift1;
      A.Gf1 = c->liftf1;
    }
    if (c->halo() && k != OP_KNS) {     // ModeKNS reads the neighbours' gradients from Gb / gGb
      const double* s0[1] = {c->lift0};
      double* d0[1] = {c->gG0};
      CKS(halo_exchange(c, 1, s0, d0, 6 * lift_jet_components(k, 0)));
      A.gG0 = c->gG0;
      if (c->liftf0) {        // BR2: the neighbours' face gradients on the shared faces
        const double* f0[1] = {c->liftf0};
        double* g0[1] = {c->gGf0};
        CKS(halo_exchange(c, 1, f0, g0, 6 * lift_jet_components(k, 0), true));
        A.gGf0 = c->gGf0;
      }
      if (k == OP_JVP_FD) {
        const double* s1[1] = {c->lift1};
        double* d1[1] = {c->gG1};
        CKS(halo_exchange(c, 1, s1, d1, 6 * lift_jet_components(k, 1)));
        A.gG1 = c->gG1;
        if (c->liftf1) {
          const double* f1[1] = {c->liftf1};
          double* g1[1] = {c->gGf1};
          CKS(halo_exchange(c, 1, f1, g1, 6 * lift_jet_components(k, 1), true));
          A.gGf1 = c->gGf1;
        }
      }
    }
  }
  CK(launch_op(k, c->cfg, k == OP_R1ABS ? c->geo_abs : c->geo, A));
  {
    char w[32];
    snprintf(w, sizeof w, "operator kind %d", (int)k);
    CKS(dbg_sync(c, w));
  }
  return HBPDC_OK;
}

hbpdc_status norm_host(hbpdc_ctx* c, const double* x, size_t L, double* out) {
  CK(launch_sumsq(x, L, c->partial, c->stream));
  if (c->comm) {
    CK(launch_reduce_partials_n(c->partial, 1, RED_BLOCKS, c->dnrm, c->stream));
    CKS(allreduce(c, c->dnrm, 1));
    CK(cudaMemcpyAsync(c->hpin, c->dnrm, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *out = std::sqrt(c->hpin[0]);
    return HBPDC_OK;
  }
  CK(launch_finish_norm(c->partial, c->dnrm, c->stream));
  CK(cudaMemcpyAsync(c->hpin, c->dnrm, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *out = c->hpin[0];
  return HBPDC_OK;
}

// Euler / NS: the state W must have rho > 0 and p > 0 everywhere; NaN / Inf
// are reported as non-finite.  Synchronises (used at existing sync points).
hbpdc_status check_admissible(hbpdc_ctx* c, const double* W, const char* where) {
  if (c->pb.equation == HBPDC_ADVECTION) {       // no pressure: finiteness only
    double nrm;
    CKS(norm_host(c, W, c->n, &nrm));
    if (!std::isfinite(nrm)) return fail(c, HBPDC_E_NONFINITE, std::string(where) + ": non-finite state");
    return HBPDC_OK;
  }
  const int nodes = c->nodes;
  CK(launch_admissible(W, c->nE, nodes, c->nv, c->pb.gamma, c->pb.mach_eps * c->pb.mach_eps, c->dadm, c->stream));
  CK(cudaMemcpyAsync(c->hadm, c->dadm, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->hadm[1] == 0) return HBPDC_OK;
  const int t = c->hadm[0];
  char buf[200];
  snprintf(buf, sizeof buf, "%s: %s at local element %d node %d", where,
           (c->hadm[1] & 1) ? "non-finite state" : "negative density or pressure", t / nodes, t % nodes);
  return fail(c, (c->hadm[1] & 1) ? HBPDC_E_NONFINITE : HBPDC_E_NEG_PRESSURE, buf);
}

int jvp_kind(hbpdc_ctx* c, int mode) {
  if (mode == HBPDC_JVP_AUTO) mode = c->pb.equation == HBPDC_ADVECTION ? HBPDC_JVP_LINEAR : HBPDC_JVP_FD;
  return mode;
}

// the K-apply norm partials recorded for vector z (GEMV slot that produced it), consumed once
const double* take_npart(hbpdc_ctx* c, const double* z) {
  for (auto& s : c->sys)
    if (s.npart_of == z) {
      s.npart_of = nullptr;
      return s.npart;
    }
  return nullptr;
}

// J dX for the extended system, dX = [dW | ds] (2n), out = [top | bottom]
// ws_ghosts: the halos of (W, sigma) are current (GMRES inside one Newton
// iteration: the linearisation point is fixed), exchange only (dW, dsigma)
// shift_src (2n, optional): out -= shift * shift_src, fused into the epilogue
hbpdc_status jvp_impl(hbpdc_ctx* c, double a1, double a2, double dt, const double* W, const double* sg,
                      const double* dW, const double* ds, double* o1, double* o2, int mode,
                      const double* eps_override, bool ws_ghosts = false, const double* shift_src = nullptr,
                      double shift = 0.0, const double* dw_part = nullptr) {
  const size_t n = c->n;
  mode = jvp_kind(c, mode);
  OpArgs A = base_args(c);
  A.W = W; A.S = sg; A.dW = dW; A.dS = ds; A.out1 = o1; A.out2 = o2;
  A.a1dt = a1 * dt;
  A.c2 = a2 * dt * dt / 2.0;
  if (shift_src) { A.shw = shift_src; A.shs = shift_src + n; A.shift = shift; }
  OpKind k;
  if (mode == HBPDC_JVP_LINEAR) {
    if (c->pb.equation != HBPDC_ADVECTION) return fail(c, HBPDC_E_ARG, "LINEAR JVP needs a linear flux");
    k = OP_JVP_LINEAR;
  } else if (mode == HBPDC_JVP_EXACT) {
    k = OP_JVP_EXACT;
  } else {
    k = OP_JVP_FD;
    if (eps_override) {
      A.epsw = eps_override[0];
    } else {
      // ||dW||^2 partials: from the K-apply that produced dW (dw_part), else one sumsq pass
      const double* part = dw_part;
      int np = dw_part ? op_grid(c->cfg, c->geo) : RED_BLOCKS;
      if (!part) {
        CK(launch_sumsq(dW, n, c->partial, c->stream));
        part = c->partial;
      }
      if (c->comm) {   // global ||dW|| (reading R7)
        CK(launch_reduce_partials_n(part, 1, np, c->deps + 1, c->stream));
        CKS(allreduce(c, c->deps + 1, 1));
        CK(launch_fd_eps_from_sum(c->deps + 1, std::sqrt(EPS_MACH) / c->pb.mach_eps, c->deps, c->stream));
      } else {
        CK(launch_finish_fd_eps(part, std::sqrt(EPS_MACH) / c->pb.mach_eps, c->deps, c->stream, np));
      }
      A.d_epsw = c->deps;
    }
  }
  ProfScope ps(c, 1, ((k == OP_JVP_LINEAR ? 4.0 : 6.0) + (shift_src ? 2.0 : 0.0)) * n * 8.0);
  CKS(run_op(c, k, A, ws_ghosts ? 12 : -1));
  if (c->st) c->st->jvp_calls++;
  return HBPDC_OK;
}

// K v = dR1/dW v at W, exactly: R2(W, v) (R2 is linear in sigma)
hbpdc_status k_apply_global(hbpdc_ctx* c, const double* W, const double* v, double* out) {
  OpArgs A = base_args(c);
  A.W = W; A.S = v; A.out1 = nullptr; A.out2 = out;
  return run_op(c, OP_R12, A);
}

// ---- BJ_ext ----------------------------------------------------------------------
hbpdc_status ensure_precond_mem(hbpdc_ctx* c) {
  if (c->S) return HBPDC_OK;
  const size_t mm = (size_t)c->m * c->m;
  c->s_shared = c->pb.equation == HBPDC_ADVECTION ? 1 : 0;
  const size_t nblk = c->s_shared ? 1 : (size_t)c->nE;
  CKS(dalloc(c, &c->S, nblk * mm));
  CKS(dalloc(c, &c->Wb, c->n));
  for (auto& w : c->sys) {
    CKS(dalloc(c, &w.U, c->n));
    CKS(dalloc(c, &w.V, c->n));
    CKS(dalloc(c, &w.npart, (size_t)op_grid(c->cfg, c->geo) + 1));
  }
  if (c->pb.equation == HBPDC_NAVIER_STOKES) {   // explicit K_i (two-hop BR1 path) + colouring scratch
    CKS(dalloc(c, &c->Kst, nblk * mm));
    for (auto& w : c->sys) CKS(dalloc(c, &w.ky, c->n));
    CKS(dalloc(c, &c->KV, c->n));
    CKS(dalloc(c, &c->KT, c->n));
    CKS(dalloc(c, &c->tseed, c->n));
    CKS(dalloc(c, &c->y1, c->n));
    CKS(dalloc(c, &c->y2, c->n));
    if (c->op.precond == HBPDC_PC_BJEXT_H) {
      CKS(dalloc(c, &c->y3, c->n));
      CKS(dalloc(c, &c->yz, c->n));
      CKS(dalloc(c, &c->yb, c->n));
      CK(cudaMemsetAsync(c->yz, 0, c->n * sizeof(double), c->stream));
    }
  }
  // Gauss-Jordan scratch: chunks of at most ~1 GiB
  size_t chunk = (size_t)(1ull << 30) / (mm * sizeof(double));
  if (chunk < 1) chunk = 1;
  if (chunk > nblk) chunk = nblk;
  c->zchunk = (int)chunk;
  CKS(dalloc(c, &c->Z, chunk * mm));
  void* q = nullptr;
  CK(cudaMalloc(&q, chunk * sizeof(int)));
  c->allocs.push_back(q);
  c->info = (int*)q;
  return HBPDC_OK;
}

// ghost copy of the BJ_ext build state (K_i reads the neighbours' frozen traces)
hbpdc_status wb_halo(hbpdc_ctx* c) {
  if (!c->halo()) return HBPDC_OK;
  const double* src[1] = {c->Wb};
  double* dst[1] = {c->gWb};
  return halo_exchange(c, 1, src, dst);
}

// in_step: called by the step at W^n (ensure_pc_for).  Navier-Stokes: the stored K_i depend on the
// build state only, not on (alpha1, alpha2), so a second build of the same step at the same W^n
// (the correctors' alpha pair) reuses them and only redoes M_i = I - a1 dt K_i + c2 K_i^2 and
// its inverse (bitwise the same blocks: the colour loop is deterministic); HBPDC_NS_KREUSE=0 rebuilds.
hbpdc_status precond_build_impl(hbpdc_ctx* c, double a1, double a2, double dt, const double* W, bool in_step = false) {
  CKS(ensure_precond_mem(c));
  const bool ns = c->pb.equation == HBPDC_NAVIER_STOKES;
  ProfScope ps(c, 6, (double)(c->s_shared ? 1 : c->nE) * c->m * c->m * 8.0 * (ns ? 2.0 : 1.0) + c->n * 8.0);
  CK(cudaMemcpyAsync(c->Wb, W, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CKS(wb_halo(c));
  const bool hess = c->op.precond == HBPDC_PC_BJEXT_H;
  if (hess) {
    // BJ^H_ext: the Hessian block dR2/dW at (Wb, sigma_b = R1(Wb)) (reading R31)
    if (!c->Sb) {
      CKS(dalloc(c, &c->Sb, c->n));
      if (c->halo()) CKS(dalloc(c, &c->gSb, (size_t)(c->pb.dim == 2 ? 2 * (c->nxl + c->nyl) : 2) * c->m));
    }
    OpArgs A = base_args(c);
    A.W = c->Wb; A.out1 = c->Sb;
    CKS(run_op(c, OP_R1, A));
    if (c->halo()) {
      const double* src[1] = {c->Sb};
      double* dst[1] = {c->gSb};
      CKS(halo_exchange(c, 1, src, dst));
    }
  }
  const size_t mm = (size_t)c->m * c->m;
  const int nblk = c->s_shared ? 1 : c->nE;
  const double a1dt = a1 * dt, c2 = a2 * dt * dt / 2.0;
  if (ns) {
    // columns of K_i and M_i for all elements by colouring (ops_kernels.cu); M goes to S,
    // then each chunk is copied to Z and inverted back into S
    auto period = [](int n) { for (int P = 3; P <= n; ++P) if (n % P == 0) return P; return n; };
    const int Px = period(c->nxl), Py = period(c->nyl);
    if (Px < 3 || Py < 3)    // two seeded elements of one colour must be > 2 elements apart
      return fail(c, HBPDC_E_ARG, "Navier-Stokes BJ_ext needs local element counts with a divisor >= 3");
    // Every launch of the loop is restricted to the colour's elements (the operator) and
    // to those plus their 4 neighbours (the lifting, whose central face values take the
    // seeded traces): the other elements' outputs are not needed (the gather reads the
    // seeded elements only), so each (colour, column) costs 1 / (Px Py) of a full-mesh
    // operator instead of one.  tseed is zero outside the seeded elements throughout.
    // m <= 160: one operator pass per column (K e_c); K_i^2 by the element-block product on
    // the fp64 tensor cores afterwards (K_i^2 e_c = K_i (K_i e_c) exactly: the same block),
    // instead of a second colour pass through lifting and operator per column
    const bool single = kk_gemm_supported(c->m) && !std::getenv("HBPDC_NS_TWOPASS");
    const char* kreuse_env = std::getenv("HBPDC_NS_KREUSE");
    const bool kreuse = in_step && c->kst_step && single && !hess && !(kreuse_env && atoi(kreuse_env) == 0);
    if (kreuse && c->st) c->st->precond_k_reused++;
    if (!kreuse) {
    CK(cudaMemsetAsync(c->tseed, 0, c->n * sizeof(double), c->stream));
    // one-hop lifting (ModeKNS, GLL / BR1 / one rank): the colour pass lifts the colour's elements
    // only; the neighbours' gradients are the build state's plus the seed's central-value term
    const char* onehop_env = std::getenv("HBPDC_NS_ONEHOP");
    const bool onehop = single && !c->geo.gl && !c->geo.br2 && !(onehop_env && atoi(onehop_env) == 0);
    if (onehop) {
      if (!c->liftB) CKS(dalloc(c, &c->liftB, (size_t)c->nE * 6 * c->P * c->P));
      OpArgs B = base_args(c);
      B.W = c->Wb;
      if (c->halo()) {
        // the build state's ghosts (wb_halo) for the lifting's neighbour traces; its lifted
        // gradients' ghosts for the neighbours' face gradients; a zero seed on every ghost
        const size_t ng = (size_t)2 * (c->nxl + c->nyl) * c->m;
        if (!c->gGb) {
          CKS(dalloc(c, &c->gGb, (size_t)2 * (c->nxl + c->nyl) * 6 * c->P * c->P));
          CKS(dalloc(c, &c->gzero, ng));
          CK(cudaMemsetAsync(c->gzero, 0, ng * sizeof(double), c->stream));
        }
        B.gW = c->gWb;
      }
      CK(launch_lift(OP_R1, 0, c->cfg, c->geo, B, c->liftB, nullptr, nullptr));
      if (c->halo()) {
        const double* s0[1] = {c->liftB};
        double* d0[1] = {c->gGb};
        CKS(halo_exchange(c, 1, s0, d0, 6));
      }
    }
    const Geo full = c->geo;
    for (int cy = 0; cy < Py; ++cy)
      for (int cx = 0; cx < Px; ++cx) {
        c->geo.cmode = 1;
        c->geo.cpx = Px; c->geo.cpy = Py; c->geo.ccx = cx; c->geo.ccy = cy;
        hbpdc_status st = HBPDC_OK;
        for (int col = 0; col < c->m && st == HBPDC_OK; ++col) {
          cudaError_t ce = launch_colour_seed(c->tseed, c->nE, c->nxl, c->m, Px, Py, cx, cy, col, c->stream);
          if (ce != cudaSuccess) { c->geo = full; CK(ce); }
          OpArgs A = base_args(c);
          A.W = c->Wb; A.S = c->tseed; A.out1 = nullptr; A.out2 = c->y1;
          A.Gb = c->liftB;
          A.gGb = c->gGb;
          st = run_op(c, onehop ? OP_KNS : OP_R12, A);
          if (st != HBPDC_OK) break;
          if (hess) {
            // BJ^H_ext: H e_c = e1e2 part of R1(W_b + e1 sigma_b + e2 e_c) (reading R31), from the
            // EXACT JVP with a1 dt = 0, c2 = 1, dsigma = 0: out1 = e_c + H e_c
            OpArgs H = base_args(c);
            H.W = c->Wb; H.S = c->Sb; H.dW = c->tseed; H.dS = c->yz; H.out1 = c->y3; H.out2 = c->yb;
            H.a1dt = 0.0; H.c2 = 1.0;
            st = run_op(c, OP_JVP_EXACT, H);
            if (st != HBPDC_OK) break;
          }
          if (single) {
            // K column only; K_i^2 comes from the element-block product below (kk_gemm)
            ce = launch_colour_gather_k(c->y1, hess ? c->y3 : nullptr, c->Kst, c->S, c->nE, c->nxl, c->m, Px, Py,
                                        cx, cy, col, c2, c->stream);
            if (ce != cudaSuccess) { c->geo = full; CK(ce); }
            continue;
          }
          ce = launch_colour_restrict(c->y1, c->tseed, c->nE, c->nxl, c->m, Px, Py, cx, cy, c->stream);
          if (ce != cudaSuccess) { c->geo = full; CK(ce); }
          A.out2 = c->y2;
          st = run_op(c, OP_R12, A);
          if (st != HBPDC_OK) break;
          ce = launch_colour_gather(c->y1, c->y2, hess ? c->y3 : nullptr, c->Kst, c->S, c->nE, c->nxl, c->m, Px, Py,
                                    cx, cy, col, a1dt, c2, c->stream);
          if (ce != cudaSuccess) { c->geo = full; CK(ce); }
        }
        c->geo = full;
        CKS(st);
        // clear this colour's elements of tseed for the next colour
        CK(launch_colour_seed(c->tseed, c->nE, c->nxl, c->m, Px, Py, cx, cy, -1, c->stream));
      }
    }   // !kreuse
    if (single) CK(launch_kk_gemm(c->Kst, c->S, c->m, c->nE, a1dt, c2, hess ? 1 : 0, kreuse ? 0 : 1, c->stream));
    c->kst_step = (in_step && single && !hess) ? 1 : 0;
  }
  std::vector<int> hinfo(c->zchunk);
  for (int e0 = 0; e0 < nblk; e0 += c->zchunk) {
    const int ne = std::min(c->zchunk, nblk - e0);
    CK(cudaMemsetAsync(c->info, 0, ne * sizeof(int), c->stream));
    if (ns)
      CK(cudaMemcpyAsync(c->Z, c->S + (size_t)e0 * mm, ne * mm * sizeof(double), cudaMemcpyDeviceToDevice,
                         c->stream));
    else
      CK(launch_kbuild(c->cfg, c->geo, c->Wb, c->halo() ? c->gWb : c->Wb, a1dt, c2, c->Z, e0, ne,
                       hess ? c->Sb : nullptr, hess ? (c->halo() ? c->gSb : c->Sb) : nullptr));
    CKS(dbg_sync(c, "BJ_ext K/M build"));
    CK(launch_gj_invert(c->Z, c->S + (size_t)e0 * mm, c->m, ne, c->info, c->stream));
    CKS(dbg_sync(c, "Gauss-Jordan"));
    CK(cudaMemcpyAsync(hinfo.data(), c->info, ne * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    int bad = -1;
    for (int b = 0; b < ne && bad < 0; ++b)
      if (hinfo[b]) bad = b;
    if (c->comm) {   // every rank leaves together (no rank waits in a collective alone)
      c->hpin[0] = bad >= 0 ? 1.0 : 0.0;
      CK(cudaMemcpyAsync(c->dnrm, c->hpin, sizeof(double), cudaMemcpyHostToDevice, c->stream));
      CKS(allreduce(c, c->dnrm, 1));
      CK(cudaMemcpyAsync(c->hpin, c->dnrm, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (c->hpin[0] > 0.0 && bad < 0)
        return fail(c, HBPDC_E_LU_SINGULAR, "BJ_ext block singular on another rank");
    }
    if (bad >= 0) {
      char buf[200];
      snprintf(buf, sizeof buf, "BJ_ext block of element %d (rank %d) is singular (dt=%g, a1=%g, a2=%g)", e0 + bad,
               c->ds.rank, dt, a1, a2);
      return fail(c, HBPDC_E_LU_SINGULAR, buf);
    }
  }
  c->pc_a1 = a1; c->pc_a2 = a2; c->pc_dt = dt;
  c->pc_valid = 1;
  if (c->st) c->st->precond_builds++;
  return HBPDC_OK;
}

// P^-1 X for B systems at once: u_i = S W_i, v_i = S sigma_i for
// all i in ONE streaming pass over S (B > 1: the lock-step corrector stages,
// NEXT-1), then per system top = u - c2 K v, bottom = v + K (u - a1dt v).
hbpdc_status precond_apply_multi(hbpdc_ctx* c, int B, const double* const* iw, const double* const* is,
                                 double* const* ow, double* const* os) {
  if (!c->pc_valid) return fail(c, HBPDC_E_ARG, "precond_apply before precond_build");
  if (c->op.schur) {
    // element-block Jacobi of J_S (reading R32): the D block S (or S^H) on the W half, sigma half 0
    ProfScope ps(c, 0, (double)(c->s_shared ? 1 : c->nE) * c->m * c->m * 8.0 + 2.0 * B * c->n * 8.0);
    if (c->s_shared) {
      for (int i = 0; i < B; ++i)
        CK(launch_block_gemv2(c->S, 1, iw[i], iw[i], ow[i], c->sys[i].V, c->m, c->nE, c->stream));
    } else {
      const double* in[GEMV_MAX_RHS];
      double* out[GEMV_MAX_RHS];
      for (int i = 0; i < B; ++i) { in[i] = iw[i]; out[i] = ow[i]; }
      CK(launch_block_gemv_multi(c->S, B, in, out, c->m, c->nE, c->stream));
    }
    for (int i = 0; i < B; ++i) {
      CK(cudaMemsetAsync(os[i], 0, c->n * sizeof(double), c->stream));
      if (c->st) c->st->precond_applies++;
    }
    return HBPDC_OK;
  }
  if (c->op.precond != HBPDC_PC_BJEXT_H) {
    ProfScope ps(c, 0, (double)(c->s_shared ? 1 : c->nE) * c->m * c->m * 8.0 + 4.0 * B * c->n * 8.0);
    if (B == 1 || c->s_shared || (c->m & 1)) {      // odd m (3D, N = 2: m = 135): 2-RHS kernel per system
      for (int i = 0; i < B; ++i)
        CK(launch_block_gemv2(c->S, c->s_shared, iw[i], is[i], c->sys[i].U, c->sys[i].V, c->m, c->nE, c->stream));
    } else {
      const double* in[GEMV_MAX_RHS];
      double* out[GEMV_MAX_RHS];
      for (int i = 0; i < B; ++i) {
        in[2 * i] = iw[i]; in[2 * i + 1] = is[i];
        out[2 * i] = c->sys[i].U; out[2 * i + 1] = c->sys[i].V;
      }
      CK(launch_block_gemv_multi(c->S, 2 * B, in, out, c->m, c->nE, c->stream));
    }
    CKS(dbg_sync(c, "BJ_ext GEMV"));
  }
  const double a1dt = c->pc_a1 * c->pc_dt, c2 = c->pc_a2 * c->pc_dt * c->pc_dt / 2.0;
  if (c->op.precond == HBPDC_PC_BJEXT_H && c->pb.equation == HBPDC_NAVIER_STOKES) {
    // P^-1 (x, y) with the Hessian block and the stored K_i (two-hop BR1 path):
    // u = S^H (x - c2 K y); top = u; bottom = y + K u -- three 1-RHS passes per system
    for (int i = 0; i < B; ++i) {
      ProfScope ps(c, 0, 3.0 * c->nE * c->m * c->m * 8.0 + 6.0 * c->n * 8.0);
      const double* in1[1] = {is[i]};
      double* out1[1] = {c->KV};
      CK(launch_block_gemv_multi(c->Kst, 1, in1, out1, c->m, c->nE, c->stream));
      CK(launch_waxpby(1.0, iw[i], -c2, c->KV, c->sys[i].U, c->n, c->stream));
      const double* in2[1] = {c->sys[i].U};
      double* out2[1] = {ow[i]};
      CK(launch_block_gemv_multi(c->S, 1, in2, out2, c->m, c->nE, c->stream));
      const double* in3[1] = {ow[i]};
      double* out3[1] = {c->KT};
      CK(launch_block_gemv_multi(c->Kst, 1, in3, out3, c->m, c->nE, c->stream));
      CK(launch_waxpby(1.0, is[i], 1.0, c->KT, os[i], c->n, c->stream));
      if (c->st) c->st->precond_applies++;
    }
    return HBPDC_OK;
  }
  if (c->op.precond == HBPDC_PC_BJEXT_H) {
    // P^-1 (x, y) with the Hessian block: u = S^H (x - c2 K y); top = u; bottom = y + K u
    for (int i = 0; i < B; ++i) {
      OpArgs A = base_args(c);
      A.W = c->Wb; A.gW = c->halo() ? c->gWb : c->Wb;
      A.dW = is[i]; A.b = iw[i]; A.a1dt = -c2; A.out1 = c->sys[i].U;
      ProfScope ps(c, 5, 3.0 * c->n * 8.0);
      CK(launch_op(OP_KLIN, c->cfg, c->geo, A));
    }
    {
      ProfScope ps(c, 0, (double)(c->s_shared ? 1 : c->nE) * c->m * c->m * 8.0 + 2.0 * B * c->n * 8.0);
      if (c->s_shared) {
        for (int i = 0; i < B; ++i)   // shared block: the 2-RHS kernel with a dummy second vector
          CK(launch_block_gemv2(c->S, 1, c->sys[i].U, c->sys[i].U, ow[i], c->sys[i].V, c->m, c->nE, c->stream));
      } else {
        const double* in[GEMV_MAX_RHS];
        double* out[GEMV_MAX_RHS];
        for (int i = 0; i < B; ++i) { in[i] = c->sys[i].U; out[i] = ow[i]; }
        CK(launch_block_gemv_multi(c->S, B, in, out, c->m, c->nE, c->stream));
      }
    }
    for (int i = 0; i < B; ++i) {
      OpArgs A = base_args(c);
      A.W = c->Wb; A.gW = c->halo() ? c->gWb : c->Wb;
      A.dW = ow[i]; A.b = is[i]; A.a1dt = 1.0; A.out1 = os[i];
      ProfScope ps(c, 5, 3.0 * c->n * 8.0);
      CK(launch_op(OP_KLIN, c->cfg, c->geo, A));
      if (c->st) c->st->precond_applies++;
    }
    return HBPDC_OK;
  }
  if (c->pb.equation == HBPDC_NAVIER_STOKES) {
    // explicit K_i: (K V_i, K (U_i - a1dt V_i)) for all B systems in ONE 2B-RHS pass over the
    // stored blocks (the lock-step corrector stages share it like the S pass; the DMMA GEMV sums
    // its k-range partials in the same order for every batch width: bitwise the per-system
    // result), K V -> ow, K (U - a1dt V) -> os, then top = U - c2 K V, bottom = V + K (U - a1dt V)
    ProfScope ps(c, 5, (double)c->nE * c->m * c->m * 8.0 + 8.0 * B * c->n * 8.0);
    const double* in[GEMV_MAX_RHS];
    double* out[GEMV_MAX_RHS];
    for (int i = 0; i < B; ++i) {
      CK(launch_waxpby(1.0, c->sys[i].U, -a1dt, c->sys[i].V, c->sys[i].ky, c->n, c->stream));
      in[2 * i] = c->sys[i].V; in[2 * i + 1] = c->sys[i].ky;
      out[2 * i] = ow[i]; out[2 * i + 1] = os[i];
    }
    if (B == 1 || (c->m & 1)) {
      for (int i = 0; i < B; ++i)
        CK(launch_block_gemv2(c->Kst, 0, in[2 * i], in[2 * i + 1], out[2 * i], out[2 * i + 1], c->m, c->nE, c->stream));
    } else {
      CK(launch_block_gemv_multi(c->Kst, 2 * B, in, out, c->m, c->nE, c->stream));
    }
    for (int i = 0; i < B; ++i) {
      CK(launch_waxpby(1.0, c->sys[i].U, -c2, ow[i], ow[i], c->n, c->stream));
      CK(launch_waxpby(1.0, c->sys[i].V, 1.0, os[i], os[i], c->n, c->stream));
      if (c->st) c->st->precond_applies++;
    }
    return HBPDC_OK;
  }
  for (int i = 0; i < B; ++i) {
    const double *U = c->sys[i].U, *V = c->sys[i].V;
    {
      OpArgs A = base_args(c);
      A.W = c->Wb; A.U = U; A.V = V; A.out1 = ow[i]; A.out2 = os[i];
      A.a1dt = a1dt;
      A.c2 = c2;
      A.gW = c->halo() ? c->gWb : c->Wb;
      A.nrm_part = c->sys[i].npart;             // ||out1||^2 partials for the next FD JVP
      ProfScope ps(c, 5, 5.0 * c->n * 8.0);
      CK(launch_op(OP_KAPPLY, c->cfg, c->geo, A));
      c->sys[i].npart_of = ow[i];
      CKS(dbg_sync(c, "BJ_ext K apply"));
    }
    if (c->st) c->st->precond_applies++;
  }
  return HBPDC_OK;
}

hbpdc_status precond_apply_impl(hbpdc_ctx* c, const double* iw, const double* is, double* ow, double* os) {
  return precond_apply_multi(c, 1, &iw, &is, &ow, &os);
}

// Krylov basis capacity >= `need` vectors (restart 700 at C3 would pin 47 GB
// up front; GMRES mostly converges far earlier).  Growth doubles, capped at
// restart + 1, and copies the existing vectors (rare, synchronous).
hbpdc_status ensure_krylov(hbpdc_ctx* c, SysWS& w, size_t need) {
  if (need <= w.vk_cap) return HBPDC_OK;
  const size_t n2 = 2 * c->n;
  size_t cap = std::max(need, 2 * w.vk_cap);
  cap = std::min(cap, (size_t)c->restart + 1);
  if (cap < need) cap = need;
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, cap * n2 * sizeof(double));
  if (e != cudaSuccess) {
    cudaGetLastError();
    char buf[200];
    snprintf(buf, sizeof buf, "Krylov basis of %zu vectors (%.1f GB) does not fit: %s", cap,
             cap * n2 * 8.0 / 1e9, cudaGetErrorString(e));
    return fail(c, HBPDC_E_OOM, buf);
  }
  if (w.Vk) {
    CK(cudaMemcpyAsync(q, w.Vk, w.vk_cap * n2 * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(w.Vk);
  }
  w.Vk = (double*)q;
  w.vk_cap = cap;
  return HBPDC_OK;
}

// the ghost buffers of (W, sigma) belong to the system being linearised
void use_ghosts(hbpdc_ctx* c, SysWS& w) {
  if (c->halo()) { c->gW = w.gW; c->gS = w.gS; }
}

// ---- GMRES (right preconditioned, DCGS2 Arnoldi, restarted) ----------------------
// One GMRES solve is a resumable state (GState), so that several independent
// systems can be advanced in lock step and share the BJ_ext S pass (NEXT-1).
struct LinSys {
  double a1, a2, dt;
  const double* W;     // linearisation point
  const double* sg;
  bool pc;
};

constexpr double GMRES_STAGNATION = 0.9;   // reading R34, the same constant as the CPU checker

struct GState {
  SysWS* w = nullptr;
  LinSys L{};
  double beta0 = 0, beta = 0;
  int total = 0;
  bool converged = false, done = false;
  // current restart cycle
  bool in_cycle = false, flush_next = false, est_ok = false;
  int j = 0, k = 0;
  std::vector<double> a, bvec, t, hp, d;
  // s-step mode (sstep > 1): Newton-basis matrix powers w_i = (A - theta) w_{i-1}
  // from w_0 = q_kb, then one block Gram-Schmidt per block of sstep vectors
  int sstep = 1, pi = 0, kb = 0;
  double theta = 1.0;
  bool needs_op() const { return in_cycle && !flush_next && j != 0; }
};

// the Newton system's operator on a GMRES vector (2n): J z, or in Schur mode
// (J_S z_W, 0) with J_S z = top block of J (z, K z), K z = R2(W, z)
hbpdc_status sys_matvec(hbpdc_ctx* c, GState& g, const double* z, double* out, const double* shift_src = nullptr,
                        double shift = 0.0, const double* dw_part = nullptr) {
  const size_t n = c->n;
  if (!c->op.schur)
    return jvp_impl(c, g.L.a1, g.L.a2, g.L.dt, g.L.W, g.L.sg, z, z + n, out, out + n, c->op.jvp_mode, nullptr,
                    true, shift_src, shift, dw_part);
  SysWS& w = *g.w;
  CKS(k_apply_global(c, g.L.W, z, w.ks));
  // ws_ghosts = false: k_apply_global's exchange reused the sigma ghost buffer (partitioned runs)
  CKS(jvp_impl(c, g.L.a1, g.L.a2, g.L.dt, g.L.W, g.L.sg, z, w.ks, out, w.ks2, c->op.jvp_mode, nullptr, false,
               shift_src, shift, nullptr));
  CK(cudaMemsetAsync(out + n, 0, n * sizeof(double), c->stream));
  return HBPDC_OK;
}

hbpdc_status g_start(hbpdc_ctx* c, GState& g) {
  SysWS& w = *g.w;
  const size_t n2 = 2 * c->n;
  CK(cudaMemsetAsync(w.dX, 0, n2 * sizeof(double), c->stream));
  CKS(norm_host(c, w.rhs, n2, &g.beta0));
  g.total = 0;
  g.in_cycle = false;
  g.converged = g.done = false;
  if (!(g.beta0 > 0.0)) {
    if (g.beta0 == 0.0) { g.converged = g.done = true; return HBPDC_OK; }
    return fail(c, HBPDC_E_NONFINITE, "GMRES rhs not finite");
  }
  CK(cudaMemcpyAsync(w.r, w.rhs, n2 * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));   // x0 = 0
  g.beta = g.beta0;
  return HBPDC_OK;
}

// start a restart cycle (or finish: converged / iteration cap)
hbpdc_status g_cycle_begin(hbpdc_ctx* c, GState& g) {
  SysWS& w = *g.w;
  const size_t n2 = 2 * c->n;
  if (g.beta <= c->op.gmres_rtol * g.beta0) { g.converged = g.done = true; return HBPDC_OK; }
  if (g.total >= c->op.krylov_max_per_newton) { g.done = true; return HBPDC_OK; }
  // V0 = r / beta
  w.hpin[0] = g.beta;
  CK(cudaMemcpyAsync(w.dnrm, w.hpin, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CK(launch_scale_by_inv(w.r, w.dnrm, w.Vk, n2, c->stream));
  std::fill(w.H.begin(), w.H.end(), 0.0);
  std::fill(w.Hraw.begin(), w.Hraw.end(), 0.0);
  std::fill(w.gv.begin(), w.gv.end(), 0.0);
  w.gv[0] = g.beta;
  g.in_cycle = true;
  g.flush_next = false;
  g.est_ok = false;
  g.j = 1;
  g.k = 0;
  g.pi = 0;
  g.kb = 0;
  return HBPDC_OK;
}

// end of a restart cycle: y = H^-1 g, x += P^-1 (V y); true residual unless converged
hbpdc_status g_cycle_end(hbpdc_ctx* c, GState& g) {
  SysWS& w = *g.w;
  const size_t n = c->n, n2 = 2 * n;
  const int R = c->restart;
  const int k = g.k;
  for (int i = k - 1; i >= 0; --i) {
    double sum = w.gv[i];
    for (int l = i + 1; l < k; ++l) sum -= w.H[(size_t)l * (R + 1) + i] * w.y[l];
    w.y[i] = sum / w.H[(size_t)i * (R + 1) + i];
  }
  // the pinned buffer may still feed an earlier async upload: wait for the stream
  CK(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < k; ++i) w.hpin[i] = w.y[i];
  CK(cudaMemcpyAsync(w.dy, w.hpin, k * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CK(launch_lincomb(w.Vk, n2, k, w.dy, w.r, n2, c->stream));
  if (g.L.pc) {
    CKS(precond_apply_impl(c, w.r, w.r + n, w.zb, w.zb + n));
    CK(launch_axpby(1.0, w.zb, 1.0, w.dX, n2, c->stream));
  } else {
    CK(launch_axpby(1.0, w.r, 1.0, w.dX, n2, c->stream));
  }
  g.in_cycle = false;
  if (g.est_ok) { g.converged = g.done = true; return HBPDC_OK; }
  // true residual r = rhs - J x
  use_ghosts(c, w);
  CKS(sys_matvec(c, g, w.dX, w.r));
  CK(launch_axpby(1.0, w.rhs, -1.0, w.r, n2, c->stream));
  const double beta_start = g.beta;
  CKS(norm_host(c, w.r, n2, &g.beta));
  // stagnation (reading R34, as the oracle): a cycle that lowered the true residual by
  // less than 10 % has reached the FD JVP's noise level; x goes back to Newton
  if (g.beta > GMRES_STAGNATION * beta_start && !(g.beta <= c->op.gmres_rtol * g.beta0)) g.converged = g.done = true;
  return HBPDC_OK;
}

// Arnoldi step j of the cycle (DCGS2, Swirydowicz et al. 2020 / Bielich et al.
// 2022; the oracle uses MGS).  z = P^-1 u_j was computed by the caller (NULL on
// a flush step, which only finalises the lagged column).  One reduction gives
// the lagged reorthogonalisation of u_j and the projections of w = J z; one
// update pass writes q_j and u_{j+1}.  Column j-1 of the Hessenberg matrix
// becomes final (and its Givens rotation applied) one iteration later.
hbpdc_status g_iter(hbpdc_ctx* c, GState& g, const double* z) {
  SysWS& w = *g.w;
  const size_t n = c->n, n2 = 2 * n;
  const int R = c->restart;
  const double rtol = c->op.gmres_rtol;
  const int j = g.j;
  const bool flush = g.flush_next || j == R + 1;
  CKS(ensure_krylov(c, w, (size_t)j + 1));
  double* u = w.Vk + (size_t)(j - 1) * n2;   // u_j (once orthogonalised)
  double* wv = w.Vk + (size_t)j * n2;
  if (!flush) {
    use_ghosts(c, w);
    CKS(sys_matvec(c, g, z, wv, nullptr, 0.0, take_npart(c, z)));
    ++g.total;
  }
  const int nk = j - 1;
  const int nb = arnoldi_dot_blocks(n2);
  {
    ProfScope ps(c, 3, (double)(nk + (flush ? 1 : 2)) * n2 * 8.0);
    CK(launch_dcgs2_dots(w.Vk, n2, nk, u, flush ? nullptr : wv, n2, w.partial, c->stream));
    CK(launch_reduce_partials_n(w.partial, 2 * nk + 3, nb, w.dh, c->stream));
    CKS(allreduce(c, w.dh, 2 * nk + 3));
  }
  CK(cudaMemcpyAsync(w.hpin, w.dh, (2 * nk + 3) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  auto HR = [&](int row, int col) -> double& { return w.Hraw[(size_t)col * (R + 1) + row]; };
  auto HQ = [&](int row, int col) -> double& { return w.H[(size_t)col * (R + 1) + row]; };
  std::vector<double>&a = g.a, &bv = g.bvec, &t = g.t, &hp = g.hp, &d = g.d;
  a.assign(nk, 0.0);
  bv.assign(nk, 0.0);
  double sa = 0.0, ab = 0.0;
  for (int q = 0; q < nk; ++q) {
    a[q] = w.hpin[2 * q];
    bv[q] = w.hpin[2 * q + 1];
    sa += a[q] * a[q];
    ab += a[q] * bv[q];
  }
  const double uu = w.hpin[2 * nk], uw = w.hpin[2 * nk + 1];
  double b2 = uu - sa;
  bool explicit_q = false;
  if (nk > 0 && !(b2 >= 0.25 * uu)) {
    // severe cancellation in the lagged step: form q_j explicitly
    for (int q = 0; q < nk; ++q) w.hpin[q] = a[q];
    CK(cudaMemcpyAsync(w.dy, w.hpin, nk * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(launch_arnoldi_axpy(w.Vk, n2, nk, w.dy, u, n2, w.partial, c->stream));
    if (c->comm) {
      CK(launch_reduce_partials_n(w.partial, 1, nb, w.dnrm, c->stream));
      CKS(allreduce(c, w.dnrm, 1));
      CK(cudaMemcpyAsync(w.hpin, w.dnrm, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      b2 = w.hpin[0];
    } else {
      CK(launch_finish_sqrt(w.partial, nb, w.dnrm, c->stream));
      CK(cudaMemcpyAsync(w.hpin, w.dnrm, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      b2 = w.hpin[0] * w.hpin[0];
    }
    explicit_q = true;
  }
  const double bu = std::sqrt(std::max(b2, 0.0));
  if (!std::isfinite(bu)) return fail(c, HBPDC_E_NONFINITE, "non-finite Arnoldi norm");
  if (j >= 2) {
    // finalize column j-2: lagged correction + subdiagonal, then Givens
    const int col = j - 2;
    for (int q = 0; q < nk; ++q) HR(q, col) += a[q];
    HR(j - 1, col) = bu;
    for (int q = 0; q <= j - 1; ++q) HQ(q, col) = HR(q, col);
    for (int i = 0; i < col; ++i) {
      const double tt = w.cs[i] * HQ(i, col) + w.sn[i] * HQ(i + 1, col);
      HQ(i + 1, col) = -w.sn[i] * HQ(i, col) + w.cs[i] * HQ(i + 1, col);
      HQ(i, col) = tt;
    }
    const double den = std::hypot(HQ(col, col), HQ(col + 1, col));
    w.cs[col] = HQ(col, col) / den;
    w.sn[col] = HQ(col + 1, col) / den;
    HQ(col, col) = den;
    HQ(col + 1, col) = 0.0;
    w.gv[col + 1] = -w.sn[col] * w.gv[col];
    w.gv[col] = w.cs[col] * w.gv[col];
    g.k = col + 1;
    if (c->st && g.k > c->st->max_krylov_j) c->st->max_krylov_j = g.k;
    if (std::fabs(w.gv[g.k]) <= rtol * g.beta0) {
      g.est_ok = true;
      return g_cycle_end(c, g);
    }
  }
  if (flush || bu == 0.0) return g_cycle_end(c, g);
  // first-pass projections of B q_j onto Q_j (provisional column j-1)
  t.assign(j, 0.0);
  for (int col = 0; col < nk; ++col)
    for (int i = 0; i <= col + 1 && i < j; ++i) t[i] += HR(i, col) * a[col];
  hp.assign(j, 0.0);
  for (int i = 0; i < nk; ++i) hp[i] = (bv[i] - t[i]) / bu;
  const double qw = (uw - ab) / bu;
  hp[j - 1] = (qw - t[j - 1]) / bu;
  for (int i = 0; i < j; ++i) HR(i, j - 1) = hp[i];
  const double cj = t[j - 1] / bu + hp[j - 1];
  d.assign(nk, 0.0);
  for (int q = 0; q < nk; ++q) d[q] = t[q] / bu + hp[q] - (explicit_q ? 0.0 : a[q] * cj / bu);
  for (int q = 0; q < nk; ++q) {
    w.hpin[q] = explicit_q ? 0.0 : a[q];
    w.hpin[(R + 1) + q] = d[q];
  }
  CK(cudaMemcpyAsync(w.dy, w.hpin, nk * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(w.dy + (R + 1), w.hpin + (R + 1), nk * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  {
    ProfScope ps(c, 4, (double)(nk + 4) * n2 * 8.0);
    CK(launch_dcgs2_update(w.Vk, n2, nk, w.dy, w.dy + (R + 1), u, wv, 1.0 / bu, cj / bu, n2, c->stream));
  }
  g.j = j + 1;
  if (g.total >= c->op.krylov_max_per_newton) g.flush_next = true;
  return HBPDC_OK;
}

// ---- s-step Arnoldi (communication-avoiding GMRES, Hoemmen 2010 / Carson 2015) ----
// A = J P^-1.  From the last orthonormal vector q_kb the block computes the
// Newton-basis powers w_i = A w_{i-1} - theta w_{i-1} (i = 1..s, one operator
// application each, like s ordinary Arnoldi steps), then orthogonalises the
// whole block against Q = [q_0..q_kb] with block CGS2 (two projection passes,
// each one streaming pass over Q) and the block itself with CholQR2.  With the
// coordinates r_i of w_i in [Q, Q_new] (r_0 = e_kb), A w_i = w_{i+1} + theta w_i
// gives the Hessenberg columns kb+i (i < s) by forward substitution:
//   h_{kb+i} = ( r_{i+1} + theta r_i - sum_{j < kb+i} r_i[j] h_j ) / r_i[kb+i].
// The Krylov space and the GMRES iterate are those of s ordinary Arnoldi steps
// (the paper's GMRES); only the orthogonalisation schedule differs.
// Q traffic: 4 passes per s iterations instead of 2 per iteration (DCGS2).

// Cholesky T = R^T R of a small SPD matrix (row-major s x s); false if not SPD
static bool small_chol(std::vector<double>& T, int sb, std::vector<double>& R) {
  R.assign((size_t)sb * sb, 0.0);
  for (int i = 0; i < sb; ++i) {
    for (int j = i; j < sb; ++j) {
      double v = T[(size_t)i * sb + j];
      for (int k = 0; k < i; ++k) v -= R[(size_t)k * sb + i] * R[(size_t)k * sb + j];
      if (i == j) {
        if (!(v > 0.0)) return false;
        R[(size_t)i * sb + i] = std::sqrt(v);
      } else {
        R[(size_t)i * sb + j] = v / R[(size_t)i * sb + i];
      }
    }
  }
  return true;
}
static void upper_inv(const std::vector<double>& R, int sb, std::vector<double>& Ri) {
  Ri.assign((size_t)sb * sb, 0.0);
  for (int j = 0; j < sb; ++j) {
    Ri[(size_t)j * sb + j] = 1.0 / R[(size_t)j * sb + j];
    for (int i = j - 1; i >= 0; --i) {
      double v = 0.0;
      for (int k = i + 1; k <= j; ++k) v += R[(size_t)i * sb + k] * Ri[(size_t)k * sb + j];
      Ri[(size_t)i * sb + j] = -v / R[(size_t)i * sb + i];
    }
  }
}

// block reduction: rows of launch_block_dots, summed over ranks, to the host
hbpdc_status block_dots_host(hbpdc_ctx* c, SysWS& w, int nq, const double* W, int sb, std::vector<double>& out) {
  const size_t n2 = 2 * c->n;
  const int rows = nq * sb + sb * sb;
  // s = 4, 8: fp64 tensor-core kernels (scripts/bench_block.cu: 5.5-5.8 TB/s vs 5.4 / 2.4 with FMAs);
  // s = 8 and a short basis: the TMA-streamed one (scripts/bench_block_tma.cu: faster for nq <= 64)
  const bool tma = sb == 8 && nq <= BLOCK_TMA_DOTS_MAX_NQ;
  const bool mma = sb >= 4;
  const int nb = tma ? block_dot_parts_tma() : (mma ? block_dot_blocks_mma(n2) : block_dot_blocks(n2));
  {
    ProfScope ps(c, 3, (double)(nq + sb) * n2 * 8.0);
    if (tma) CK(launch_block_dots_tma8(w.Vk, n2, nq, W, n2, n2, w.partial, c->stream));
    else if (mma) CK(launch_block_dots_mma(w.Vk, n2, nq, W, n2, sb, n2, w.partial, c->stream));
    else CK(launch_block_dots(w.Vk, n2, nq, W, n2, sb, n2, w.partial, c->stream));
    CK(launch_reduce_partials_n(w.partial, rows, nb, w.dh, c->stream));
    CKS(allreduce(c, w.dh, rows));
  }
  CK(cudaMemcpyAsync(w.hpin, w.dh, rows * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  out.assign(w.hpin, w.hpin + rows);
  return HBPDC_OK;
}

hbpdc_status block_update_dev(hbpdc_ctx* c, SysWS& w, int nq, double* W, int sb, const std::vector<double>& C,
                              const std::vector<double>* Rinv) {
  const size_t n2 = 2 * c->n;
  const int nc = nq * sb;
  CK(cudaStreamSynchronize(c->stream));      // the pinned staging buffer is free
  for (int q = 0; q < nc; ++q) w.hpin[q] = C[q];
  if (Rinv) for (int q = 0; q < sb * sb; ++q) w.hpin[nc + q] = (*Rinv)[q];
  const int tot = nc + (Rinv ? sb * sb : 0);
  if (tot) CK(cudaMemcpyAsync(w.dy, w.hpin, tot * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  ProfScope ps(c, 4, (double)(nq + 2 * sb) * n2 * 8.0);
  // s = 8: fp64 tensor-core kernel (5.8 TB/s vs 4.0 with FMAs), TMA-streamed for a short basis
  // (scripts/bench_block_tma.cu: 3.3 / 5.4 / 6.6 TB/s at nq = 1 / 17 / 64 vs 2.8 / 4.1 / 5.8);
  // s <= 4: FMA kernel (6.1 TB/s)
  if (sb == 8 && nq >= 1 && nq <= BLOCK_TMA_UPDATE_MAX_NQ)
    CK(launch_block_update_tma8(w.Vk, n2, nq, W, n2, w.dy, Rinv ? w.dy + nc : nullptr, n2, c->stream));
  else if (sb == 8) CK(launch_block_update_mma(w.Vk, n2, nq, W, n2, sb, w.dy, Rinv ? w.dy + nc : nullptr, n2, c->stream));
  else CK(launch_block_update(w.Vk, n2, nq, W, n2, sb, w.dy, Rinv ? w.dy + nc : nullptr, n2, c->stream));
  return HBPDC_OK;
}

// fused W <- W - Q C (the first CGS2 update) and the rows of the second
// projection [Q W]^T W of the updated block, one pass over Q (s = 8, short basis)
hbpdc_status block_update_dots_host(hbpdc_ctx* c, SysWS& w, int nq, double* W, const std::vector<double>& C,
                                    std::vector<double>& out) {
  const size_t n2 = 2 * c->n;
  const int sb = 8, nc = nq * sb, rows = nq * sb + sb * sb;
  CK(cudaStreamSynchronize(c->stream));      // the pinned staging buffer is free
  for (int q = 0; q < nc; ++q) w.hpin[q] = C[q];
  CK(cudaMemcpyAsync(w.dy, w.hpin, nc * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  {
    // algorithmic bytes: Q once, W read + written
    ProfScope ps(c, 7, (double)(nq + 2 * sb) * n2 * 8.0);
    CK(launch_block_update_dots_tma8(w.Vk, n2, nq, W, n2, w.dy, n2, w.partial, c->stream));
    CK(launch_reduce_partials_n(w.partial, rows, block_fused_parts_tma(), w.dh, c->stream));
    CKS(allreduce(c, w.dh, rows));
  }
  CK(cudaMemcpyAsync(w.hpin, w.dh, rows * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  out.assign(w.hpin, w.hpin + rows);
  return HBPDC_OK;
}

// s = 8: second update W <- (W - Q C) Rinv with the Gram rows of the updated block
// computed in the same pass (the CholQR2 reduction), then summed to the host
hbpdc_status block_update_gram_host(hbpdc_ctx* c, SysWS& w, int nq, double* W, const std::vector<double>& C,
                                    const std::vector<double>& Rinv, std::vector<double>& out) {
  const size_t n2 = 2 * c->n;
  const int sb = 8, nc = nq * sb, rows = sb * sb;
  CK(cudaStreamSynchronize(c->stream));      // the pinned staging buffer is free
  for (int q = 0; q < nc; ++q) w.hpin[q] = C[q];
  for (int q = 0; q < sb * sb; ++q) w.hpin[nc + q] = Rinv[q];
  CK(cudaMemcpyAsync(w.dy, w.hpin, (nc + sb * sb) * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  {
    ProfScope ps(c, 4, (double)(nq + 2 * sb) * n2 * 8.0);
    CK(launch_block_update_tma8(w.Vk, n2, nq, W, n2, w.dy, w.dy + nc, n2, c->stream, w.partial));
    CK(launch_reduce_partials_n(w.partial, rows, block_fused_parts_tma(), w.dh, c->stream));
    CKS(allreduce(c, w.dh, rows));
  }
  CK(cudaMemcpyAsync(w.hpin, w.dh, rows * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  out.assign(w.hpin, w.hpin + rows);
  return HBPDC_OK;
}

// s = 8: W <- W Rinv (second CholQR pass), one streaming pass over the block
hbpdc_status block_scale_dev(hbpdc_ctx* c, SysWS& w, double* W, const std::vector<double>& Rinv) {
  const size_t n2 = 2 * c->n;
  CK(cudaStreamSynchronize(c->stream));
  for (int q = 0; q < 64; ++q) w.hpin[q] = Rinv[q];
  CK(cudaMemcpyAsync(w.dy, w.hpin, 64 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  ProfScope ps(c, 4, 2.0 * 8 * n2 * 8.0);
  CK(launch_block_scale_w8(W, n2, w.dy, n2, c->stream));
  return HBPDC_OK;
}

// the block of s powers is complete: orthogonalise it, extend H, apply Givens
hbpdc_status g_block(hbpdc_ctx* c, GState& g) {
  SysWS& w = *g.w;
  const size_t n2 = 2 * c->n;
  const int R = c->restart;
  const int sb = g.sstep, kb = g.kb, nq = kb + 1;
  double* W = w.Vk + (size_t)(kb + 1) * n2;
  std::vector<double> r1, r2, r3, T, Rw, Rwi, R3, R3i;
  // pass 1 + 2: C1 = Q^T W, W1 = W - Q C1
  CKS(block_dots_host(c, w, nq, W, sb, r1));
  std::vector<double> C1(r1.begin(), r1.begin() + (size_t)nq * sb);
  // pass 3 + 4: C2 = Q^T W1, G2 = W1^T W1; Q_new = (W1 - Q C2) Rw^-1, Rw^T Rw = G2 - C2^T C2
  // (s = 8 with a short basis: pass 2 and the projection of pass 3 fused, Q read once)
  if (sb == 8 && nq <= block_fused_max_nq() && c->fuse_cgs) {
    CKS(block_update_dots_host(c, w, nq, W, C1, r2));
  } else {
    CKS(block_update_dev(c, w, nq, W, sb, C1, nullptr));
    CKS(block_dots_host(c, w, nq, W, sb, r2));
  }
  std::vector<double> C2(r2.begin(), r2.begin() + (size_t)nq * sb);
  // Selective reorthogonalisation (reading R37; PETSc's CGS "refine if needed"): the first
  // projection already left W1 orthogonal to Q when the second projection's coefficients,
  // seen through the block's own orthonormalisation, X = C2 Rw0^-1 (Rw0^T Rw0 = W1^T W1),
  // are at the level sel_reorth.  Q_new = W1 Rw0^-1 then departs from Q^T Q_new = 0 by |X|
  // only, and the second update pass over Q is skipped (W = Q C1 + Q_new Rw0 exactly).
  bool skip2 = false;
  if (sb == 8 && c->fuse_cgs && (c->sel_reorth > 0.0 || c->trace)) {
    std::vector<double> T0((size_t)sb * sb), R0, R0i;
    for (int a = 0; a < sb * sb; ++a) T0[a] = r2[(size_t)nq * sb + a];
    if (small_chol(T0, sb, R0)) {
      upper_inv(R0, sb, R0i);
      double mx = 0.0;
      for (int j = 0; j < nq; ++j)
        for (int b = 0; b < sb; ++b) {
          double v = 0.0;
          for (int a = 0; a <= b; ++a) v += C2[(size_t)j * sb + a] * R0i[(size_t)a * sb + b];
          mx = std::max(mx, std::fabs(v));
        }
      ++c->blk_count;
      const int dec = mx <= 1e-15 ? 0 : mx <= 1e-14 ? 1 : mx <= 1e-13 ? 2 : mx <= 1e-12 ? 3 : mx <= 1e-10 ? 4 : 5;
      ++c->blk_hist[dec];
      if (c->sel_reorth > 0.0 && mx <= c->sel_reorth) {
        skip2 = true;
        ++c->blk_skip;
        Rw = R0;
        Rwi = R0i;
      }
    }
  }
  if (skip2) {
    std::fill(C2.begin(), C2.end(), 0.0);
    std::vector<double> zero(sb, 0.0);
    // W <- W Rw0^-1 with the Gram of the result (the CholQR2 reduction); q_0 with zero coefficients
    CKS(block_update_gram_host(c, w, 1, W, zero, Rwi, r3));
  }
  T.assign((size_t)sb * sb, 0.0);
  for (int a = 0; a < sb; ++a)
    for (int b = 0; b < sb; ++b) {
      double v = r2[(size_t)nq * sb + a * sb + b];
      for (int j = 0; j < nq; ++j) v -= C2[(size_t)j * sb + a] * C2[(size_t)j * sb + b];
      T[(size_t)a * sb + b] = v;
    }
  bool ok = skip2 || small_chol(T, sb, Rw);
  if (ok && skip2) {
    T.assign(r3.begin(), r3.begin() + (size_t)sb * sb);
    ok = small_chol(T, sb, R3);
    if (ok) {
      upper_inv(R3, sb, R3i);
      CKS(block_scale_dev(c, w, W, R3i));
    }
  } else if (ok) {
    upper_inv(Rw, sb, Rwi);
    // CholQR2 of the block itself: its Gram from the update pass (s = 8) or a separate pass
    const bool fused = sb == 8 && c->fuse_cgs;
    if (fused) {
      CKS(block_update_gram_host(c, w, nq, W, C2, Rwi, r3));
    } else {
      CKS(block_update_dev(c, w, nq, W, sb, C2, &Rwi));
      CKS(block_dots_host(c, w, 0, W, sb, r3));
    }
    T.assign(r3.begin(), r3.begin() + (size_t)sb * sb);
    ok = small_chol(T, sb, R3);
    if (ok) {
      upper_inv(R3, sb, R3i);
      if (fused) {
        CKS(block_scale_dev(c, w, W, R3i));
      } else {
        std::vector<double> none;
        CKS(block_update_dev(c, w, 0, W, sb, none, &R3i));
      }
    }
  }
  if (!ok) {
    // numerically dependent block (near a happy breakdown or an ill-conditioned
    // power basis): finish the cycle with the columns so far, continue with DCGS2
    g.sstep = 1;
    return g_cycle_end(c, g);
  }
  // R_total = R3 Rw (upper triangular)
  std::vector<double> Rt((size_t)sb * sb, 0.0);
  for (int i = 0; i < sb; ++i)
    for (int j = i; j < sb; ++j) {
      double v = 0.0;
      for (int k = i; k <= j; ++k) v += R3[(size_t)i * sb + k] * Rw[(size_t)k * sb + j];
      Rt[(size_t)i * sb + j] = v;
    }
  // coordinates r_i (i = 0..sb) of w_i in [q_0 .. q_{kb+sb}]
  const int dimc = nq + sb;
  std::vector<std::vector<double>> rc(sb + 1, std::vector<double>(dimc, 0.0));
  rc[0][kb] = 1.0;
  for (int i = 1; i <= sb; ++i) {
    for (int j = 0; j < nq; ++j) rc[i][j] = C1[(size_t)j * sb + i - 1] + C2[(size_t)j * sb + i - 1];
    for (int m = 0; m < sb; ++m) rc[i][nq + m] = Rt[(size_t)m * sb + i - 1];
  }
  auto HR = [&](int row, int col) -> double& { return w.Hraw[(size_t)col * (R + 1) + row]; };
  auto HQ = [&](int row, int col) -> double& { return w.H[(size_t)col * (R + 1) + row]; };
  for (int i = 0; i < sb; ++i) {
    const int col = kb + i;
    std::vector<double> h(dimc, 0.0);
    for (int r = 0; r < dimc; ++r) h[r] = rc[i + 1][r] + g.theta * rc[i][r];
    for (int j = 0; j < col; ++j) {
      const double cj = rc[i][j];
      if (cj == 0.0) continue;
      for (int r = 0; r <= j + 1 && r < dimc; ++r) h[r] -= cj * HR(r, j);
    }
    const double piv = rc[i][col];
    for (int r = 0; r <= col + 1; ++r) HR(r, col) = h[r] / piv;
    // Givens on the new column
    for (int r = 0; r <= col + 1; ++r) HQ(r, col) = HR(r, col);
    for (int q = 0; q < col; ++q) {
      const double tt = w.cs[q] * HQ(q, col) + w.sn[q] * HQ(q + 1, col);
      HQ(q + 1, col) = -w.sn[q] * HQ(q, col) + w.cs[q] * HQ(q + 1, col);
      HQ(q, col) = tt;
    }
    const double den = std::hypot(HQ(col, col), HQ(col + 1, col));
    w.cs[col] = HQ(col, col) / den;
    w.sn[col] = HQ(col + 1, col) / den;
    HQ(col, col) = den;
    HQ(col + 1, col) = 0.0;
    w.gv[col + 1] = -w.sn[col] * w.gv[col];
    w.gv[col] = w.cs[col] * w.gv[col];
    g.k = col + 1;
    if (c->st && g.k > c->st->max_krylov_j) c->st->max_krylov_j = g.k;
    if (!std::isfinite(w.gv[g.k])) return fail(c, HBPDC_E_NONFINITE, "non-finite s-step Arnoldi");
    if (std::fabs(w.gv[g.k]) <= c->op.gmres_rtol * g.beta0) {
      g.est_ok = true;
      return g_cycle_end(c, g);
    }
  }
  // next block from q_{kb+sb}
  g.kb = kb + sb;
  g.pi = 0;
  g.j = g.kb + 1;
  if (g.kb + sb > R || g.total >= c->op.krylov_max_per_newton) return g_cycle_end(c, g);
  return HBPDC_OK;
}

// one matrix-powers step of the s-step block: w_{pi+1} = A w_pi - theta w_pi, z = P^-1 w_pi given
hbpdc_status g_power(hbpdc_ctx* c, GState& g, const double* z) {
  SysWS& w = *g.w;
  const size_t n = c->n, n2 = 2 * n;
  CKS(ensure_krylov(c, w, (size_t)g.j + 1));
  double* prev = w.Vk + (size_t)(g.j - 1) * n2;
  double* out = w.Vk + (size_t)g.j * n2;
  use_ghosts(c, w);
  CKS(sys_matvec(c, g, z, out, prev, g.theta, take_npart(c, z)));
  ++g.total;
  ++g.pi;
  ++g.j;
  if (g.pi == g.sstep) return g_block(c, g);
  return HBPDC_OK;
}

// Solve J x_i = rhs_i (rhs in w.rhs, x -> w.dX) for B systems in lock step:
// every Arnoldi step preconditions all systems that need an operator
// application with ONE pass over S (precond_apply_multi), the JVPs and
// Arnoldi passes run per system.  B = 1 is the plain restarted GMRES.
hbpdc_status gmres_batch(hbpdc_ctx* c, GState* gs, int B) {
  const size_t n = c->n;
  for (int i = 0; i < B; ++i) CKS(g_start(c, gs[i]));
  while (true) {
    for (int i = 0; i < B; ++i)
      if (!gs[i].done && !gs[i].in_cycle) CKS(g_cycle_begin(c, gs[i]));
    int act[GEMV_MAX_RHS / 2], na = 0, ncyc = 0;
    for (int i = 0; i < B; ++i) {
      if (!gs[i].in_cycle) continue;
      // grow the basis BEFORE taking pointers into it (growth reallocates)
      CKS(ensure_krylov(c, *gs[i].w, (size_t)gs[i].j + 1));
      ++ncyc;
      if (gs[i].needs_op() && gs[i].j != c->restart + 1) act[na++] = i;
    }
    if (ncyc == 0) break;
    const double* zs[GEMV_MAX_RHS / 2] = {};
    if (na) {
      const double *iw[GEMV_MAX_RHS / 2], *is[GEMV_MAX_RHS / 2];
      double *ow[GEMV_MAX_RHS / 2], *os[GEMV_MAX_RHS / 2];
      for (int q = 0; q < na; ++q) {
        SysWS& w = *gs[act[q]].w;
        const double* u = w.Vk + (size_t)(gs[act[q]].j - 1) * 2 * n;
        if (gs[act[q]].L.pc) {
          iw[q] = u; is[q] = u + n; ow[q] = w.zb; os[q] = w.zb + n;
          zs[q] = w.zb;
        } else {
          zs[q] = u;
        }
      }
      // the GEMV scratch of sys[0..na) serves any subset of systems
      if (gs[act[0]].L.pc) CKS(precond_apply_multi(c, na, iw, is, ow, os));
    }
    for (int i = 0, q = 0; i < B; ++i) {
      if (!gs[i].in_cycle) continue;
      const double* z = nullptr;
      if (q < na && act[q] == i) z = zs[q++];
      if (gs[i].sstep > 1 && z) CKS(g_power(c, gs[i], z));
      else CKS(g_iter(c, gs[i], z));
    }
  }
  for (int i = 0; i < B; ++i) {
    if (c->st) c->st->gmres_its += gs[i].total;
    if (!gs[i].converged) {
      char buf[128];
      snprintf(buf, sizeof buf, "GMRES did not converge within %d iterations", c->op.krylov_max_per_newton);
      return fail(c, HBPDC_E_GMRES, buf);
    }
  }
  return HBPDC_OK;
}

// ---- Newton on the extended system (eq:Newton) -------------------------
// B systems in lock step (B = 1: one stage solve).  System i starts from
// X0 = (Wg_i, R1(Wg_i)) with right-hand side b_i = sys[i].b; result in sys[i].X.
hbpdc_status newton_batch(hbpdc_ctx* c, int B, double a1, double a2, double dt, const double* const* Wg) {
  const size_t n = c->n, n2 = 2 * n;
  double floor_[GEMV_MAX_RHS / 2], g0[GEMV_MAX_RHS / 2];
  bool active[GEMV_MAX_RHS / 2];
  for (int i = 0; i < B; ++i) {
    SysWS& w = c->sys[i];
    CK(cudaMemcpyAsync(w.X, Wg[i], n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    OpArgs A = base_args(c);
    A.W = w.X; A.out1 = w.X + n;
    CKS(run_op(c, OP_R1, A));
    double bn, rabs;
    CKS(norm_host(c, w.b, n, &bn));
    OpArgs Ab = base_args(c);
    Ab.W = w.X; Ab.out1 = w.G;            // G is scratch here
    CKS(run_op(c, OP_R1ABS, Ab));
    CKS(norm_host(c, w.G, n, &rabs));
    // floor = max(64 eps ||b||, 4 eps ||R1_abs(W_g)||)   (readings R10, R10b)
    floor_[i] = std::max(c->op.newton_floor * EPS_MACH * bn, 4.0 * EPS_MACH * rabs);
    g0[i] = -1.0;
    active[i] = true;
  }
  const bool pc = c->op.precond != HBPDC_PC_NONE;
  for (int r = 0; r <= c->op.newton_max; ++r) {
    int na = 0;
    for (int i = 0; i < B; ++i) {
      if (!active[i]) continue;
      SysWS& w = c->sys[i];
      use_ghosts(c, w);
      {
        OpArgs A = base_args(c);
        A.W = w.X; A.S = w.X + n; A.b = w.b; A.out1 = w.G; A.out2 = w.G + n;
        A.a1dt = a1 * dt;
        A.c2 = a2 * dt * dt / 2.0;
        ProfScope ps(c, 2, 5.0 * n * 8.0);
        CKS(run_op(c, OP_RESID, A));
      }
      double gn;
      CKS(norm_host(c, w.G, n2, &gn));
      if (!std::isfinite(gn)) return fail(c, HBPDC_E_NONFINITE, "non-finite Newton residual");
      if (g0[i] < 0) g0[i] = gn;
      if (c->trace) fprintf(stderr, "[hbpdc] newton sys %d it %d |G| %.3e |G0| %.3e floor %.3e\n", i, r, gn, g0[i], floor_[i]);
      if (c->st) c->st->final_newton_rel = g0[i] > 0 ? gn / g0[i] : 0.0;
      if (gn <= std::max(c->op.newton_rtol * g0[i], floor_[i])) { active[i] = false; continue; }
      if (r == c->op.newton_max) {
        char buf[160];
        snprintf(buf, sizeof buf, "Newton did not converge in %d iterations (||G||=%.3e, ||G0||=%.3e)", r, gn,
                 g0[i]);
        return fail(c, HBPDC_E_NEWTON, buf);
      }
      ++na;
    }
    if (na == 0) {
      // the converged stage values must be admissible (intermediate Newton iterates may
      // overshoot, as in the oracle; only solutions are checked)
      for (int i = 0; i < B; ++i) CKS(check_admissible(c, c->sys[i].X, "converged stage value"));
      return HBPDC_OK;
    }
    if (pc && c->op.precond_policy == HBPDC_PC_PER_NEWTON) {   // B == 1 under this policy
      CKS(precond_build_impl(c, a1, a2, dt, c->sys[0].X));
    }
    GState gs[GEMV_MAX_RHS / 2];
    int idx[GEMV_MAX_RHS / 2], nb = 0;
    for (int i = 0; i < B; ++i) {
      if (!active[i]) continue;
      SysWS& w = c->sys[i];
      if (c->op.schur) {
        // Schur complement: rhs = (-G1 + c2 K G2, 0)
        CKS(k_apply_global(c, w.X, w.G + n, w.ks));
        CK(launch_waxpby(-1.0, w.G, a2 * dt * dt / 2.0, w.ks, w.rhs, n, c->stream));
        CK(cudaMemsetAsync(w.rhs + n, 0, n * sizeof(double), c->stream));
      } else {
        CK(launch_axpby(-1.0, w.G, 0.0, w.rhs, n2, c->stream));       // rhs = -G
      }
      gs[nb].w = &w;
      gs[nb].L = LinSys{a1, a2, dt, w.X, w.X + n, pc};
      gs[nb].sstep = c->sstep;
      idx[nb++] = i;
    }
    CKS(gmres_batch(c, gs, nb));
    if (c->trace)
      for (int q = 0; q < nb; ++q) fprintf(stderr, "[hbpdc] gmres sys %d its %d\n", idx[q], gs[q].total);
    for (int q = 0; q < nb; ++q) {
      SysWS& w = c->sys[idx[q]];
      if (c->op.schur) {                                              // dsigma = -G2 + K dw
        CKS(k_apply_global(c, w.X, w.dX, w.ks));
        CK(launch_waxpby(-1.0, w.G + n, 1.0, w.ks, w.dX + n, n, c->stream));
      }
      CK(launch_axpby(1.0, w.dX, 1.0, w.X, n2, c->stream));         // X += dX
      if (c->st) c->st->newton_its++;
      double dwn;
      CKS(norm_host(c, w.dX, n, &dwn));
      if (dwn <= c->op.newton_atol_dw) active[idx[q]] = false;
    }
  }
  return HBPDC_OK;
}

// R1 and R2(w, R1(w)) of a stage value (reading R6)
hbpdc_status stage_ops(hbpdc_ctx* c, const double* w, double* r1, double* r2) {
  OpArgs A = base_args(c);
  A.W = w; A.out1 = r1;
  CKS(run_op(c, OP_R1, A));
  OpArgs B = base_args(c);
  B.W = w; B.S = r1; B.out1 = nullptr; B.out2 = r2;
  CKS(run_op(c, OP_R12, B));
  return HBPDC_OK;
}

hbpdc_status ensure_pc_for(hbpdc_ctx* c, double a1, double a2, double dt, const double* Wn) {
  if (c->op.precond == HBPDC_PC_NONE || c->op.precond_policy != HBPDC_PC_PER_STEP_PER_ALPHA) return HBPDC_OK;
  // (alpha1, alpha2) pairs equal up to rounding (dc = c_l - c_{l-1} is constant
  // for q = 4, 6, 8 in exact arithmetic, App. A) share one build (reading R12)
  auto same = [](double x, double y) { return std::fabs(x - y) <= 1e-12 * std::fabs(y); };
  if (c->pc_valid == 2 && same(a1, c->pc_a1) && same(a2, c->pc_a2) && c->pc_dt == dt) return HBPDC_OK;
  CKS(precond_build_impl(c, a1, a2, dt, Wn, true));
  c->pc_valid = 2;   // built inside this step at W^n
  return HBPDC_OK;
}

// Alg. 1: predictor (eq:predictor), k_max corrector sweeps
// (eq:corrector, with I_l, reading R5), FSAL update.  The s-1 corrector
// stages of a sweep depend only on sweep-k data (eq:corrector), so
// with batching they are solved in lock step (NEXT-1); the arithmetic of each
// stage solve is unchanged (bitwise equal to the sequential order).
hbpdc_status step_impl(hbpdc_ctx* c, double dt, double* W) {
  const size_t n = c->n;
  const Tableau& T = c->tab;
  const int s = T.s;
  int cur = 0;
  CK(cudaMemcpyAsync(c->Wn, W, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CKS(check_admissible(c, W, "step input"));
  if (c->fsal_valid) {
    // the cached R1/R2 belong to the previous step's output: reuse them only if W is that
    // array with unchanged contents (pointer + fingerprint), else recompute
    if (W != c->fsal_ptr) {
      c->fsal_valid = 0;
    } else {
      unsigned long long fp[2];
      CK(launch_fingerprint(W, n, c->dfp + 1, c->stream));
      CK(cudaMemcpyAsync(fp, c->dfp, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (fp[0] != fp[1]) c->fsal_valid = 0;
    }
  }
  if (!c->fsal_valid) CKS(stage_ops(c, c->Wn, c->str1[cur][0], c->str2[cur][0]));
  c->pc_valid = c->pc_valid ? 1 : 0;   // a build from an earlier step is not at this W^n
  c->kst_step = 0;                     // nor are its Navier-Stokes K_i
  CK(cudaMemcpyAsync(c->stw[cur][0], c->Wn, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  // ---- predictor (eq:nonlinear_predictor)
  for (int l = 1; l < s; ++l) {
    const double dc = T.c[l] - T.c[l - 1];
    const double a1 = dc / 2.0, a2 = dc * dc / 6.0, c2 = a2 * dt * dt / 2.0;
    const double* X[2] = {c->str1[cur][l - 1], c->str2[cur][l - 1]};
    const double co[2] = {a1 * dt, c2};
    CK(launch_stage_combo(c->stw[cur][l - 1], 2, X, co, 0, nullptr, nullptr, c->sys[0].b, n, c->stream));
    CKS(ensure_pc_for(c, a1, a2, dt, c->Wn));
    const double* g = c->stw[cur][l - 1];
    if (c->trace) fprintf(stderr, "[hbpdc] predictor stage %d\n", l + 1);
    NvtxRange nv("predictor stage");
    hbpdc_status stt = newton_batch(c, 1, a1, a2, dt, &g);
    if (stt != HBPDC_OK) {
      c->err = "predictor stage " + std::to_string(l + 1) + ": " + c->err;
      return stt;
    }
    if (c->st) c->st->stage_solves++;
    CK(cudaMemcpyAsync(c->stw[cur][l], c->sys[0].X, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CKS(stage_ops(c, c->stw[cur][l], c->str1[cur][l], c->str2[cur][l]));
  }
  // ---- correctors (eq:nonlinear_corrector)
  const int B = (int)c->sys.size();       // 1, or s - 1 when the stages are batched
  for (int k = 0; k < c->pb.kmax; ++k) {
    const int nxt = 1 - cur;
    // stage 1 of the new sweep is W^n with the FSAL operators
    CK(cudaMemcpyAsync(c->stw[nxt][0], c->stw[cur][0], n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->str1[nxt][0], c->str1[cur][0], n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->str2[nxt][0], c->str2[cur][0], n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    for (int l0 = 1; l0 < s; l0 += B) {
      NvtxRange nv("corrector stages");
      const int nb = std::min(B, s - l0);
      const double* guess[GEMV_MAX_RHS / 2];
      for (int q = 0; q < nb; ++q) {
        const int l = l0 + q;
        // b = W^n - dt R1_l + dt^2/2 R2_l + dt sum_j B1_lj R1_j + dt^2 sum_j B2_lj R2_j
        const double* X[4];
        const double* Y[4];
        double a[4], bb[4];
        for (int j = 0; j < s; ++j) {
          X[j] = c->str1[cur][j];
          Y[j] = c->str2[cur][j];
          a[j] = dt * T.B1[l][j] - (j == l ? dt : 0.0);
          bb[j] = dt * dt * T.B2[l][j] + (j == l ? dt * dt / 2.0 : 0.0);
        }
        CK(launch_stage_combo(c->Wn, s, X, a, s, Y, bb, c->sys[q].b, n, c->stream));
        guess[q] = c->stw[cur][l];
      }
      CKS(ensure_pc_for(c, 1.0, 1.0, dt, c->Wn));
      if (c->trace) fprintf(stderr, "[hbpdc] corrector sweep %d stages %d..%d\n", k + 1, l0 + 1, l0 + nb);
      hbpdc_status stt = newton_batch(c, nb, 1.0, 1.0, dt, guess);
      if (stt != HBPDC_OK) {
        c->err = "corrector sweep " + std::to_string(k + 1) + " stages " + std::to_string(l0 + 1) + ".." +
                 std::to_string(l0 + nb) + ": " + c->err;
        return stt;
      }
      for (int q = 0; q < nb; ++q) {
        const int l = l0 + q;
        if (c->st) c->st->stage_solves++;
        CK(cudaMemcpyAsync(c->stw[nxt][l], c->sys[q].X, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        CKS(stage_ops(c, c->stw[nxt][l], c->str1[nxt][l], c->str2[nxt][l]));
      }
    }
    cur = nxt;
  }
  // ---- update / FSAL
  CK(cudaMemcpyAsync(W, c->stw[cur][s - 1], n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  if (cur != 0) {
    CK(cudaMemcpyAsync(c->str1[0][0], c->str1[cur][s - 1], n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->str2[0][0], c->str2[cur][s - 1], n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  } else {
    CK(cudaMemcpyAsync(c->str1[0][0], c->str1[0][s - 1], n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->str2[0][0], c->str2[0][s - 1], n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  }
  c->fsal_valid = 1;
  c->fsal_ptr = W;
  CK(launch_fingerprint(W, n, c->dfp, c->stream));
  if (c->pc_valid == 2) c->pc_valid = 1;
  return HBPDC_OK;
}

hbpdc_status alloc_solver(hbpdc_ctx* c) {
  const size_t n = c->n, n2 = 2 * n;
  const int R = c->restart;
  // lock-step corrector stages (NEXT-1): one workspace per stage of a sweep
  int B = 1;
  if (c->op.batch_stages && c->pb.kmax > 0 && c->op.precond_policy == HBPDC_PC_PER_STEP_PER_ALPHA)
    B = std::min(c->tab.s - 1, GEMV_MAX_RHS / 2);
  c->sys.resize(std::max(B, 1));
  const size_t ng = (size_t)(c->pb.dim == 2 ? 2 * (c->nxl + c->nyl) : 2) * c->m;
  for (auto& w : c->sys) {
    CKS(dalloc(c, &w.X, n2));
    CKS(dalloc(c, &w.G, n2));
    CKS(dalloc(c, &w.dX, n2));
    CKS(dalloc(c, &w.rhs, n2));
    CKS(dalloc(c, &w.r, n2));
    CKS(dalloc(c, &w.zb, n2));
    CKS(dalloc(c, &w.b, n));
    if (c->op.schur) {
      CKS(dalloc(c, &w.ks, n));
      CKS(dalloc(c, &w.ks2, n));
    }
    CKS(ensure_krylov(c, w, std::min<size_t>((size_t)R + 1, 33)));
    // reduction rows: DCGS2 2j + 3, s-step (j + 1) s + s^2
    const size_t rows = std::max<size_t>(2 * (size_t)R + 4, ((size_t)R + 1) * c->sstep + (size_t)c->sstep * c->sstep);
    CKS(dalloc(c, &w.partial, rows * std::max({arnoldi_dot_blocks(n2), block_dot_blocks(n2), block_dot_blocks_mma(n2), block_dot_parts_tma(), RED_BLOCKS})));
    CKS(dalloc(c, &w.dh, rows));
    CKS(dalloc(c, &w.dy, rows));
    CKS(dalloc(c, &w.dnrm, 1));
    if (c->halo()) {
      CKS(dalloc(c, &w.gW, ng));
      CKS(dalloc(c, &w.gS, ng));
    }
    w.H.assign((size_t)R * (R + 1), 0.0);
    w.Hraw.assign((size_t)R * (R + 1), 0.0);
    w.cs.assign(R + 1, 0.0);
    w.sn.assign(R + 1, 0.0);
    w.gv.assign(R + 2, 0.0);
    w.y.assign(R + 1, 0.0);
    void* hp = nullptr;
    CK(cudaMallocHost(&hp, std::max<size_t>(3 * (size_t)(R + 1) + 8,
                                             ((size_t)R + 1) * c->sstep + (size_t)c->sstep * c->sstep + 8) *
                               sizeof(double)));
    w.hpin = (double*)hp;
  }
  CKS(dalloc(c, &c->partial, RED_BLOCKS));
  CKS(dalloc(c, (double**)&c->dfp, 2));
  CKS(dalloc(c, (double**)&c->dadm, 1));
  {
    void* hp = nullptr;
    CK(cudaMallocHost(&hp, 2 * sizeof(int)));
    c->hadm = (int*)hp;
  }
  CKS(dalloc(c, &c->dnrm, 1));
  CKS(dalloc(c, &c->deps, 2));
  CKS(dalloc(c, &c->Wn, n));
  for (int sw = 0; sw < 2; ++sw)
    for (int l = 0; l < c->tab.s; ++l) {
      CKS(dalloc(c, &c->stw[sw][l], n));
      CKS(dalloc(c, &c->str1[sw][l], n));
      CKS(dalloc(c, &c->str2[sw][l], n));
    }
  if (c->halo()) {
    c->gW = c->sys[0].gW;
    c->gS = c->sys[0].gS;
    CKS(dalloc(c, &c->gdW, ng));
    CKS(dalloc(c, &c->gdS, ng));
    CKS(dalloc(c, &c->gWb, ng));
    size_t off[4], len[4];
    halo_segments(c->hl, HALO_MAX_FIELDS, off, len);
    size_t hb = off[3] + len[3];
    if (c->pb.equation == HBPDC_NAVIER_STOKES) {
      const size_t ngg = (size_t)(c->pb.dim == 2 ? 2 * (c->nxl + c->nyl) : 2) * 6 * 4 * c->nodes;
      CKS(dalloc(c, &c->gG0, ngg));
      CKS(dalloc(c, &c->gG1, ngg));
      if (c->pb.nodes == HBPDC_GL) {
        const size_t lt = (size_t)c->nE * 4 * 3 * 4 * c->P;
        const size_t gt = (size_t)2 * (c->nxl + c->nyl) * 4 * 3 * 4 * c->P;
        CKS(dalloc(c, &c->tg0, lt));
        CKS(dalloc(c, &c->tg1, lt));
        CKS(dalloc(c, &c->gtg0, gt));
        CKS(dalloc(c, &c->gtg1, gt));
      }
      if (c->pb.lifting == HBPDC_BR2) {
        const size_t ngf = (size_t)2 * (c->nxl + c->nyl) * 4 * 6 * 4 * c->P;
        CKS(dalloc(c, &c->gGf0, ngf));
        CKS(dalloc(c, &c->gGf1, ngf));
      }
      halo_segments(c->hl, 1, off, len, 6 * 4);          // lifted gradients, hyper-dual jets
      hb = std::max(hb, off[3] + len[3]);
    }
    CKS(dalloc(c, &c->hsend, hb));
    CKS(dalloc(c, &c->hrecv, hb));
  }
  if (c->pb.equation == HBPDC_NAVIER_STOKES) {
    const size_t lg = (size_t)c->nE * 6 * 4 * c->nodes;
    CKS(dalloc(c, &c->lift0, lg));
    CKS(dalloc(c, &c->lift1, lg));
    if (c->pb.lifting == HBPDC_BR2) {
      const size_t lf = (size_t)c->nE * 4 * 6 * 4 * c->P;
      CKS(dalloc(c, &c->liftf0, lf));
      CKS(dalloc(c, &c->liftf1, lf));
    }
  }
  void* hp = nullptr;
  CK(cudaMallocHost(&hp, 16 * sizeof(double)));
  c->hpin = (double*)hp;
  return HBPDC_OK;
}

}  // namespace

// =====================================================================================
// C-ABI
// =====================================================================================
extern "C" {

hbpdc_status hbpdc_init(const hbpdc_problem* pb, const hbpdc_solver_opts* op, const hbpdc_dist* ds,
                        hbpdc_ctx** out) {
  if (!pb || !op || !out) return HBPDC_E_ARG;
  *out = nullptr;
  hbpdc_ctx* c = new hbpdc_ctx();
  c->pb = *pb;
  c->op = *op;
  if (ds) c->ds = *ds;
  else { c->ds.rank = 0; c->ds.nranks = 1; c->ds.px = 1; c->ds.py = 1; c->ds.own_stream = 1; }
  auto bad = [&](const char* msg) {
    c->err = msg;
    *out = c;   // return the context so the caller can read the message
    return HBPDC_E_ARG;
  };
  if (pb->dim < 1 || pb->dim > 3) return bad("dim must be 1, 2 or 3");
  if (pb->equation < 0 || pb->equation > 2) return bad("unknown equation");
  if (pb->equation != HBPDC_ADVECTION && pb->dim == 1) return bad("Euler/NS need dim >= 2");
  if (pb->dim == 3) {       // NEXT-4 scope: inviscid hexahedra, GLL, one rank, N = 2, 3 (m = 135, 320)
    if (pb->equation == HBPDC_NAVIER_STOKES) return bad("3D: advection or Euler (Navier-Stokes is 2D)");
    if (pb->nodes != HBPDC_GLL) return bad("3D: Gauss-Lobatto nodes only");
    if (pb->N < 2 || pb->N > 3) return bad("3D: N must be 2 or 3 (m = 5 (N+1)^3 <= 320)");
    if (pb->nz < 1 || pb->ny < 1 || !(pb->zmax > pb->zmin)) return bad("3D: bad z extent / element counts");
    if (ds && (ds->nranks > 1 || ds->force_halo)) return bad("3D runs on one rank");
  }
  if (pb->N < 1 || pb->N > 7) return bad("N must be in 1..7");
  if (pb->nodes != HBPDC_GLL && pb->nodes != HBPDC_GL) return bad("nodes must be HBPDC_GLL or HBPDC_GL");
  if (!(pb->mach_eps > 0.0)) return bad("mach_eps must be positive");
  if (pb->lifting != HBPDC_BR1 && pb->lifting != HBPDC_BR2) return bad("lifting must be HBPDC_BR1 or HBPDC_BR2");
  if (pb->lifting == HBPDC_BR2 && pb->equation == HBPDC_NAVIER_STOKES) {
    if (!(pb->eta_br2 > 0.0)) return bad("BR2: eta_br2 must be positive");
  }
  if (pb->equation == HBPDC_NAVIER_STOKES && pb->mach_eps != 1.0)
    return bad("Navier-Stokes: mach_eps must be 1 (reading R18)");
  if (pb->q != 4 && pb->q != 6 && pb->q != 8) return bad("q must be 4, 6 or 8");
  if (pb->kmax < 0) return bad("kmax must be >= 0");
  if (pb->nx < 1 || (pb->dim >= 2 && pb->ny < 1)) return bad("element counts must be positive");
  if (c->ds.nranks < 1 || c->ds.rank < 0 || c->ds.rank >= c->ds.nranks) return bad("bad rank / nranks");
  if (c->ds.px < 1 || c->ds.py < 1) { c->ds.px = c->ds.nranks; c->ds.py = 1; }
  if (c->ds.px * c->ds.py != c->ds.nranks) return bad("px * py must equal nranks");
  if (pb->dim == 1 && c->ds.py != 1) return bad("1D partitions need py = 1");
  if (pb->nx % c->ds.px || (pb->dim == 2 && pb->ny % c->ds.py)) return bad("px must divide nx and py divide ny");
  const bool halo = c->ds.nranks > 1 || c->ds.force_halo;

  if (op->gmres_restart < 1 || op->krylov_max_per_newton < 1 || op->newton_max < 0) return bad("bad solver options");
  c->nv = pb->equation == HBPDC_ADVECTION ? 1 : (pb->dim == 3 ? 5 : 4);
  c->P = pb->N + 1;
  c->nodes = pb->dim == 3 ? c->P * c->P * c->P : (pb->dim == 2 ? c->P * c->P : c->P);
  c->m = c->nv * c->nodes;
  c->nxl = pb->nx / c->ds.px;
  c->nyl = pb->dim >= 2 ? pb->ny / c->ds.py : 1;
  c->nzl = pb->dim == 3 ? pb->nz : 1;
  {
    const int rx = c->ds.rank % c->ds.px, ry = c->ds.rank / c->ds.px;
    c->ex0 = rx * c->nxl;
    c->ey0 = ry * c->nyl;
    c->nbr[0] = ry * c->ds.px + (rx + c->ds.px - 1) % c->ds.px;
    c->nbr[1] = ry * c->ds.px + (rx + 1) % c->ds.px;
    c->nbr[2] = ((ry + c->ds.py - 1) % c->ds.py) * c->ds.px + rx;
    c->nbr[3] = ((ry + 1) % c->ds.py) * c->ds.px + rx;
    // a direction exchanges halos when it is split over ranks (or forced)
    const int hx = halo && (c->ds.px > 1 || c->ds.force_halo);
    const int hy = halo && pb->dim == 2 && (c->ds.py > 1 || c->ds.force_halo);
    c->hl = HaloLayout{c->nxl, c->nyl, pb->equation == HBPDC_ADVECTION ? 1 : 4, pb->N + 1, pb->dim, {hx, hx, hy, hy}};
  }
  c->nE = c->nxl * c->nyl * c->nzl;
  c->n = (size_t)c->nE * c->m;
  c->restart = op->gmres_restart;
  c->sstep = op->gmres_sstep > 1 ? op->gmres_sstep : 1;
  if (pb->flux != HBPDC_LLF && pb->flux != HBPDC_GLF_PAPER) return bad("flux must be HBPDC_LLF or HBPDC_GLF_PAPER");
  if (op->precond < HBPDC_PC_NONE || op->precond > HBPDC_PC_BJEXT_H) return bad("unknown precond");
  if (c->sstep != 1 && c->sstep != 2 && c->sstep != 4 && c->sstep != 8) return bad("gmres_sstep must be 1, 2, 4 or 8");
  if (c->sstep > c->restart) c->sstep = 1;
  c->tab = tableau(pb->q);
  c->basis = pb->nodes == HBPDC_GL ? hbpdc::gl_basis(pb->N) : hbpdc::gll_basis(pb->N);
  // geometry: Cartesian, J = dx dy / 4, s-hat = dy/2, dx/2 -> scale 2/dx, 2/dy
  const double dx = (pb->xmax - pb->xmin) / pb->nx;
  const double dy = pb->dim >= 2 ? (pb->ymax - pb->ymin) / pb->ny : 1.0;
  c->geo.nx = c->nxl;
  c->geo.ny = c->nyl;
  c->geo.nz = c->nzl;
  c->geo.sz = pb->dim == 3 ? 2.0 / ((pb->zmax - pb->zmin) / pb->nz) : 1.0;
  c->geo.nE = c->nE;
  c->geo.hx = c->hl.active[0];
  c->geo.hy = c->hl.active[2];
  c->geo.sx = 2.0 / dx;
  c->geo.sy = 2.0 / dy;
  c->geo.lhp = c->basis.lhp;
  c->geo.lhm = c->basis.lhm;
  for (int i = 0; i < c->P * c->P; ++i) c->geo.Dh[i] = c->basis.Dhat[i];
  c->geo.gl = c->basis.gl;
  c->geo.br2 = pb->equation == HBPDC_NAVIER_STOKES && pb->lifting == HBPDC_BR2;
  c->hl.gl = c->basis.gl;                // GL halos carry interpolated traces
  for (int i = 0; i < c->P; ++i) { c->hl.lp[i] = c->basis.lp[i]; c->hl.lm[i] = c->basis.lm[i]; }
  c->geo.P = c->P;
  c->geo.dim = pb->dim;
  for (int i = 0; i < c->P * c->P; ++i) c->geo.D[i] = c->basis.D[i];
  c->geo.cp = c->geo.cm = 0.0;
  for (int i = 0; i < c->P; ++i) {
    c->geo.dlp[i] = c->basis.dlp[i];
    c->geo.dlm[i] = c->basis.dlm[i];
    c->geo.cp += c->basis.lp[i] * c->basis.lhpv[i];
    c->geo.cm += c->basis.lm[i] * c->basis.lhmv[i];
  }
  for (int i = 0; i < c->P; ++i) {
    c->geo.lp[i] = c->basis.lp[i];
    c->geo.lm[i] = c->basis.lm[i];
    c->geo.lhpv[i] = c->basis.lhpv[i];
    c->geo.lhmv[i] = c->basis.lhmv[i];
  }
  c->geo_abs = c->geo;
  for (int i = 0; i < c->P * c->P; ++i) c->geo_abs.Dh[i] = std::fabs(c->basis.Dhat[i]);
  c->geo_abs.lhm = -std::fabs(c->geo.lhm);
  c->geo_abs.lhp = std::fabs(c->geo.lhp);
  for (int i = 0; i < c->P; ++i) {     // R1_abs: |lhat|, the - face added (traces keep l)
    c->geo_abs.lhpv[i] = std::fabs(c->geo.lhpv[i]);
    c->geo_abs.lhmv[i] = -std::fabs(c->geo.lhmv[i]);
  }
  c->cfg.eq = (pb->equation == HBPDC_EULER && pb->dim == 3) ? 3 : pb->equation;   // EQ 3: 3D Euler (5 variables)
  c->cfg.dim = pb->dim;
  c->cfg.pp.az = pb->dim == 3 ? pb->az : 0.0;
  c->cfg.P = c->P;
  c->cfg.pp.ax = pb->a[0];
  c->cfg.pp.ay = pb->a[1];
  c->cfg.pp.gamma = pb->gamma;
  c->cfg.pp.glf = pb->flux == HBPDC_GLF_PAPER ? 1 : 0;
  c->cfg.pp.eta_br2 = pb->eta_br2;
  c->cfg.pp.ieps = 1.0 / pb->mach_eps;
  c->cfg.pp.eps2 = pb->mach_eps * pb->mach_eps;
  c->cfg.pp.ieps2 = 1.0 / c->cfg.pp.eps2;
  c->cfg.pp.mu = pb->mu;
  c->cfg.pp.Rgas = 1.0 / pb->gamma;
  c->cfg.pp.lamT = (c->cfg.pp.Rgas * pb->gamma / (pb->gamma - 1.0)) * pb->mu / (pb->prandtl > 0 ? pb->prandtl : 1.0);
  cudaError_t e = cudaSetDevice(c->ds.device);
  if (e != cudaSuccess) { c->err = cudaGetErrorString(e); *out = c; return HBPDC_E_CUDA; }
  if (!c->ds.own_stream) {
    c->stream = (cudaStream_t)c->ds.cuda_stream;   // NULL = legacy default stream
  } else {
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) { c->err = cudaGetErrorString(e); *out = c; return HBPDC_E_CUDA; }
    c->own_stream = true;
  }
  c->cfg.stream = c->stream;
  if (halo) {
    std::string err;
    int kind = c->ds.comm;
    if (kind == HBPDC_COMM_AUTO) kind = HBPDC_COMM_NCCL;
    if (kind == HBPDC_COMM_NCCL) c->comm = hbpdc::make_nccl_comm(c->ds.rank, c->ds.nranks, c->ds.nccl_unique_id, err);
    else if (kind == HBPDC_COMM_LOOPBACK)
      c->comm = hbpdc::make_loopback_comm((hbpdc::LoopbackGroup*)c->ds.loopback_group, c->ds.rank);
    else err = "unknown comm kind";
    if (!c->comm) {
      c->err = err.empty() ? "cannot create the communicator" : err;
      *out = c;
      return HBPDC_E_NCCL;
    }
  }
  if (halo && pb->dim == 2 && c->nxl >= 3 && c->nyl >= 3) {
    const char* ov = std::getenv("HBPDC_OVERLAP");
    c->overlap = !(ov && ov[0] == '0');
    if (c->overlap) {
      e = cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming);
      if (e != cudaSuccess) { c->err = cudaGetErrorString(e); *out = c; return HBPDC_E_CUDA; }
    }
  }
  { const char* gt = std::getenv("HBPDC_GL_TRACES"); c->gl_notrace = gt && gt[0] == '0'; }
  { const char* dbg = std::getenv("HBPDC_DEBUG_SYNC"); c->debug_sync = dbg && dbg[0] == '1'; }
  { const char* tr = std::getenv("HBPDC_TRACE"); c->trace = tr && tr[0] == '1'; }   // solver trace on stderr
  { const char* fc = std::getenv("HBPDC_FUSE_CGS"); c->fuse_cgs = !(fc && fc[0] == '0'); }
  { const char* sr = std::getenv("HBPDC_SEL_REORTH"); if (sr) c->sel_reorth = std::atof(sr); }
  hbpdc_status s = alloc_solver(c);
  *out = c;
  return s;
}

hbpdc_status hbpdc_partition(int dim, int nx, int ny, int px, int py, int rank, int* ex0, int* ey0, int* nxl,
                             int* nyl, int* nbr4) {
  if (dim == 1) ny = 1;
  if (nx < 1 || ny < 1 || px < 1 || py < 1 || (dim == 1 && py != 1) || nx % px || ny % py || rank < 0 ||
      rank >= px * py)
    return HBPDC_E_ARG;
  const int rx = rank % px, ry = rank / px;
  if (ex0) *ex0 = rx * (nx / px);
  if (ey0) *ey0 = ry * (ny / py);
  if (nxl) *nxl = nx / px;
  if (nyl) *nyl = ny / py;
  if (nbr4) {
    nbr4[0] = ry * px + (rx + px - 1) % px;
    nbr4[1] = ry * px + (rx + 1) % px;
    nbr4[2] = ((ry + py - 1) % py) * px + rx;
    nbr4[3] = ((ry + 1) % py) * px + rx;
  }
  return HBPDC_OK;
}

hbpdc_status hbpdc_nccl_unique_id(void* out128) {
  if (!out128) return HBPDC_E_ARG;
  std::string e;
  return hbpdc::nccl_unique_id(out128, e) ? HBPDC_E_NCCL : HBPDC_OK;
}

hbpdc_status hbpdc_loopback_group_create(int nranks, void** group) {
  if (!group || nranks < 1) return HBPDC_E_ARG;
  *group = hbpdc::loopback_group_create(nranks);
  return HBPDC_OK;
}

void hbpdc_loopback_group_destroy(void* group) { hbpdc::loopback_group_destroy((hbpdc::LoopbackGroup*)group); }

hbpdc_status hbpdc_local_shape(const hbpdc_ctx* c, int* nle, int* m, int* ex0, int* ey0, int* nxl, int* nyl) {
  if (!c) return HBPDC_E_ARG;
  if (nle) *nle = c->nE;
  if (m) *m = c->m;
  if (ex0) *ex0 = c->ex0;
  if (ey0) *ey0 = c->ey0;
  if (nxl) *nxl = c->nxl;
  if (nyl) *nyl = c->nyl;
  return HBPDC_OK;
}

hbpdc_status hbpdc_node_coords(const hbpdc_ctx* c, double* xh, double* yh) {
  if (!c || !xh) return HBPDC_E_ARG;
  const auto& pb = c->pb;
  const double dx = (pb.xmax - pb.xmin) / pb.nx;
  const double dy = pb.dim >= 2 ? (pb.ymax - pb.ymin) / pb.ny : 0.0;
  const int P = c->P;
  for (int e = 0; e < c->nE; ++e) {
    const int ex = c->ex0 + e % c->nxl, ey = c->ey0 + (e / c->nxl) % c->nyl;
    for (int nd = 0; nd < c->nodes; ++nd) {
      const int i = nd % P, j = (nd / P) % P;
      xh[(size_t)e * c->nodes + nd] = pb.xmin + ex * dx + (c->basis.xi[i] + 1.0) * dx / 2;
      if (pb.dim >= 2 && yh) yh[(size_t)e * c->nodes + nd] = pb.ymin + ey * dy + (c->basis.xi[j] + 1.0) * dy / 2;
    }
  }
  return HBPDC_OK;
}

hbpdc_status hbpdc_node_coords_z(const hbpdc_ctx* c, double* zh) {
  if (!c || !zh) return HBPDC_E_ARG;
  const auto& pb = c->pb;
  if (pb.dim != 3) return fail(const_cast<hbpdc_ctx*>(c), HBPDC_E_ARG, "node_coords_z: 3D only");
  const double dz = (pb.zmax - pb.zmin) / pb.nz;
  const int P = c->P;
  for (int e = 0; e < c->nE; ++e) {
    const int ez = e / (c->nxl * c->nyl);
    for (int nd = 0; nd < c->nodes; ++nd)
      zh[(size_t)e * c->nodes + nd] = pb.zmin + ez * dz + (c->basis.xi[nd / (P * P)] + 1.0) * dz / 2;
  }
  return HBPDC_OK;
}

hbpdc_status hbpdc_rhs(hbpdc_ctx* c, const double* W, const double* sigma, double* out) {
  if (!c || !W || !out) return HBPDC_E_ARG;
  OpArgs A = base_args(c);
  A.W = W;
  if (!sigma) {
    A.out1 = out;
    return run_op(c, OP_R1, A);
  }
  A.S = sigma;
  A.out1 = nullptr;
  A.out2 = out;
  return run_op(c, OP_R12, A);
}

hbpdc_status hbpdc_residual(hbpdc_ctx* c, double a1, double a2, double dt, const double* b, const double* W,
                            const double* sigma, double* G1, double* G2, double* norm_out) {
  if (!c || !b || !W || !sigma || !G1 || !G2) return HBPDC_E_ARG;
  OpArgs A = base_args(c);
  A.W = W; A.S = sigma; A.b = b; A.out1 = G1; A.out2 = G2;
  A.a1dt = a1 * dt;
  A.c2 = a2 * dt * dt / 2.0;
  {
    ProfScope ps(c, 2, 5.0 * c->n * 8.0);
    CKS(run_op(c, OP_RESID, A));
  }
  if (norm_out) {
    double s1, s2;
    CKS(norm_host(c, G1, c->n, &s1));
    CKS(norm_host(c, G2, c->n, &s2));
    *norm_out = std::sqrt(s1 * s1 + s2 * s2);
  }
  return HBPDC_OK;
}

hbpdc_status hbpdc_jvp(hbpdc_ctx* c, double a1, double a2, double dt, const double* W, const double* sigma,
                       const double* dW, const double* dsigma, double* out1, double* out2, int mode,
                       const double* eps_override) {
  if (!c || !dW || !dsigma || !out1 || !out2) return HBPDC_E_ARG;
  const int k = jvp_kind(c, mode);
  if (k != HBPDC_JVP_LINEAR && (!W || !sigma)) return HBPDC_E_ARG;
  return jvp_impl(c, a1, a2, dt, W, sigma, dW, dsigma, out1, out2, mode, eps_override);
}

hbpdc_status hbpdc_precond_build(hbpdc_ctx* c, double a1, double a2, double dt, const double* W) {
  if (!c || !W) return HBPDC_E_ARG;
  return precond_build_impl(c, a1, a2, dt, W);
}

hbpdc_status hbpdc_precond_set(hbpdc_ctx* c, double a1, double a2, double dt, const double* W, const double* S,
                               int shared) {
  if (!c || !W || !S) return HBPDC_E_ARG;
  CKS(ensure_precond_mem(c));
  if (c->pb.equation == HBPDC_NAVIER_STOKES)
    return fail(c, HBPDC_E_ARG, "precond_set: Navier-Stokes applies the stored K_i too; build it instead");
  if (shared != c->s_shared) return fail(c, HBPDC_E_ARG, "shared flag does not match the equation");
  const size_t nblk = c->s_shared ? 1 : (size_t)c->nE;
  CK(cudaMemcpyAsync(c->S, S, nblk * c->m * c->m * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaMemcpyAsync(c->Wb, W, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CKS(wb_halo(c));

  c->pc_a1 = a1; c->pc_a2 = a2; c->pc_dt = dt;
  c->pc_valid = 1;
  return HBPDC_OK;
}

hbpdc_status hbpdc_precond_export(hbpdc_ctx* c, double* S_out, size_t capacity, int* shared) {
  if (!c) return HBPDC_E_ARG;
  if (!c->pc_valid) return fail(c, HBPDC_E_ARG, "no preconditioner built");
  const size_t nblk = c->s_shared ? 1 : (size_t)c->nE;
  if (shared) *shared = c->s_shared;
  if (!S_out) return HBPDC_OK;                 // query only: *shared tells the size
  if (capacity < nblk * c->m * c->m)
    return fail(c, HBPDC_E_ARG, "precond_export: S_out holds " + std::to_string(capacity) + " doubles, " +
                                    std::to_string(nblk * c->m * c->m) + " needed");
  CK(cudaMemcpyAsync(S_out, c->S, nblk * c->m * c->m * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return HBPDC_OK;
}

hbpdc_status hbpdc_precond_apply(hbpdc_ctx* c, const double* iw, const double* is, double* ow, double* os) {
  if (!c || !iw || !is || !ow || !os) return HBPDC_E_ARG;
  return precond_apply_impl(c, iw, is, ow, os);
}

hbpdc_status hbpdc_step(hbpdc_ctx* c, double dt, double* W, hbpdc_step_stats* stats) {
  if (!c || !W || !(dt >= 0.0)) return HBPDC_E_ARG;
  hbpdc_step_stats local{};
  c->st = &local;
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0, c->stream);
  hbpdc_status s;
  {
    NvtxRange nv("hbpdc_step");
    s = step_impl(c, dt, W);
  }
  cudaEventRecord(t1, c->stream);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  local.wall_s = ms * 1e-3;
  c->st = nullptr;
  if (c->trace && c->blk_count)
    fprintf(stderr, "[hbpdc] s-step blocks %lld, second update skipped %lld; max|C2 Rw^-1| <=1e-15 %lld <=1e-14 %lld "
            "<=1e-13 %lld <=1e-12 %lld <=1e-10 %lld larger %lld\n", c->blk_count, c->blk_skip, c->blk_hist[0],
            c->blk_hist[1], c->blk_hist[2], c->blk_hist[3], c->blk_hist[4], c->blk_hist[5]);
  if (stats) *stats = local;
  prof_flush(c);
  if (s == HBPDC_OK && e != cudaSuccess) {
    c->err = cudaGetErrorString(e);
    return HBPDC_E_CUDA;
  }
  return s;
}

hbpdc_status hbpdc_step_host(hbpdc_ctx* c, double dt, double* W_host, hbpdc_step_stats* stats) {
  if (!c || !W_host) return HBPDC_E_ARG;
  if (!c->Wio) CKS(dalloc(c, &c->Wio, c->n));
  CK(cudaMemcpyAsync(c->Wio, W_host, c->n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  hbpdc_status s = hbpdc_step(c, dt, c->Wio, stats);
  if (s == HBPDC_OK) {
    CK(cudaMemcpyAsync(W_host, c->Wio, c->n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  return s;
}

hbpdc_status hbpdc_reset(hbpdc_ctx* c) {
  if (!c) return HBPDC_E_ARG;
  c->fsal_valid = 0;
  return HBPDC_OK;
}

hbpdc_status hbpdc_profile(hbpdc_ctx* c, int enable) {
  if (!c) return HBPDC_E_ARG;
  prof_flush(c);
  c->prof_on = enable ? 1 : 0;
  if (enable) {
    for (int i = 0; i < NPROF; ++i) { c->prof_launch[i] = 0; c->prof_ms[i] = 0.0; c->prof_bytes[i] = 0.0; }
  }
  return HBPDC_OK;
}

hbpdc_status hbpdc_profile_read(hbpdc_ctx* c, int id, long long* launches, double* total_ms,
                                double* alg_bytes) {
  if (!c || id < 0 || id >= NPROF) return HBPDC_E_ARG;
  prof_flush(c);
  if (launches) *launches = c->prof_launch[id];
  if (total_ms) *total_ms = c->prof_ms[id];
  if (alg_bytes) *alg_bytes = c->prof_bytes[id];
  return HBPDC_OK;
}

hbpdc_status hbpdc_launch_count(long long* count) {
  if (!count) return HBPDC_E_ARG;
  *count = g_hbpdc_launches;
  return HBPDC_OK;
}

const char* hbpdc_last_error(const hbpdc_ctx* c) { return c ? c->err.c_str() : "null context"; }

void hbpdc_finalize(hbpdc_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  prof_flush(c);
  for (void* p : c->allocs) cudaFree(p);
  for (auto& w : c->sys) {
    if (w.Vk) cudaFree(w.Vk);
    if (w.hpin) cudaFreeHost(w.hpin);
  }
  if (c->hpin) cudaFreeHost(c->hpin);
  if (c->hadm) cudaFreeHost(c->hadm);
  if (c->cstream) cudaStreamSynchronize(c->cstream), cudaStreamDestroy(c->cstream);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  delete c->comm;
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

}  // extern "C"

// launch.h -- host-side entry points of the device kernels (internal).
#pragma once
#include <algorithm>
#include <cstddef>
#include <cuda_runtime.h>
#include "physics.cuh"

struct Geo;
struct OpArgs;

// OP_R1ABS needs a Geo with |Dhat| and lhm negated (see hbpdc.cu)
enum OpKind { OP_R1 = 0, OP_R12, OP_RESID, OP_JVP_EXACT, OP_JVP_FD, OP_JVP_LINEAR, OP_KAPPLY, OP_R1ABS, OP_KLIN,
              OP_KNS, OP_NKINDS };

struct OpCfg {
  int eq, dim, P;
  PhysParams pp;
  cudaStream_t stream;
};

// fused element operator (modes.cuh); NS modes need lift buffers in A.G0/G1
cudaError_t launch_op(OpKind kind, const OpCfg& c, const Geo& g, const OpArgs& A);
// CTAs of an operator launch (per-CTA partials, e.g. the K-apply norm epilogue)
int op_grid(const OpCfg& c, const Geo& g);
// Gauss-Legendre instantiations (ops_kernels_gl.cu), reached from launch_op / launch_kbuild when g.gl
cudaError_t launch_op_gl(OpKind kind, const OpCfg& c, const Geo& g, const OpArgs& A);
// GL FD JVP: face traces of W, sigma, dW, dsigma (ops_kernels_gl.cu) -> OpArgs::Tr
cudaError_t launch_gl_traces(const OpCfg& c, const Geo& g, const OpArgs& A, double* Tr);
// Navier-Stokes operators with BR2 face gradients (ops_kernels_br2.cu, ops_kernels_gl_br2.cu), when g.br2
cudaError_t launch_op_br2(OpKind kind, const OpCfg& c, const Geo& g, const OpArgs& A);
cudaError_t launch_op_gl_br2(OpKind kind, const OpCfg& c, const Geo& g, const OpArgs& A);
// 3D hexahedral instantiations (ops_kernels_3d.cu, NEXT-4), reached from launch_op / launch_kbuild when c.dim == 3
cudaError_t launch_op_3d(OpKind kind, const OpCfg& c, const Geo& g, const OpArgs& A);
cudaError_t launch_kbuild_3d(const OpCfg& c, const Geo& g, const double* Wb, const double* gWb, double a1dt,
                             double c2, double* M, int e0, int ne, const double* Sb, const double* gSb);
cudaError_t launch_lift_gl(OpKind kind, int state, const OpCfg& c, const Geo& g, const OpArgs& A, double* Gout,
                           double* Gf, const double* gTg, double* Tg);
cudaError_t launch_kbuild_gl(const OpCfg& c, const Geo& g, const double* Wb, const double* gWb, double a1dt,
                             double c2, double* M, int e0, int ne, const double* Sb, const double* gSb);
// BR1 lifting of jet state `state` of operator `kind` into Gout
// Gf (BR2, GLL): also write the per-face gradients [elem][face][6][JetN][P], or NULL (BR1)
// gTg (GL across partitions): the neighbour ranks' g(w) face traces (launch_gtrace + face-buffer halo)
cudaError_t launch_lift(OpKind kind, int state, const OpCfg& c, const Geo& g, const OpArgs& A, double* Gout,
                        double* Gf = nullptr, const double* gTg = nullptr);
// GL: face traces of the gradient variables g(w) of jet state `state`, [elem][face][3][JetN][P]
cudaError_t launch_gtrace(OpKind kind, int state, const OpCfg& c, const Geo& g, const OpArgs& A, double* Tg);
// number of jet components of the lifted gradients of (kind, state)
int lift_jet_components(OpKind kind, int state);
// BJ_ext: M_i = I - a1dt K_i + c2 K_i^2 for elements [e0, e0+ne), row-major m x m each
// Sb / gSb (BJ^H_ext): sigma at the build point and its ghosts; NULL for BJ_ext
cudaError_t launch_kbuild(const OpCfg& c, const Geo& g, const double* Wb, const double* gWb, double a1dt, double c2,
                          double* M, int e0, int ne, const double* Sb = nullptr, const double* gSb = nullptr);

// BJ_ext build by element colouring (NS): seed e_col in the colour's elements,
// restrict a vector to them, gather K and M columns of the seeded elements
cudaError_t launch_colour_seed(double* t, int nE, int nx, int m, int Px, int Py, int cx, int cy, int col,
                               cudaStream_t st);
cudaError_t launch_colour_restrict(const double* y, double* t, int nE, int nx, int m, int Px, int Py, int cx, int cy,
                                   cudaStream_t st);
// single-pass colour build (m <= 160): K column (and c2 H column for BJ^H_ext) per seeded element, then
// M_i += I - a1dt K_i + c2 K_i^2 for all elements on the fp64 tensor cores (kk_gemm)
cudaError_t launch_colour_gather_k(const double* y1, const double* y3, double* K, double* M, int nE, int nx, int m,
                                   int Px, int Py, int cx, int cy, int col, double c2, cudaStream_t st);
bool kk_gemm_supported(int m);
cudaError_t launch_kk_gemm(double* K, double* M, int m, int nE, double a1dt, double c2, int hess, int kt, cudaStream_t st);
cudaError_t launch_colour_gather(const double* y1, const double* y2, const double* y3, double* K, double* M, int nE,
                                 int nx, int m, int Px, int Py, int cx, int cy, int col, double a1dt, double c2,
                                 cudaStream_t st);

// ---- linalg.cu -----------------------------------------------------------------
// in-place Gauss-Jordan inversion with partial pivoting of `nmat` m x m
// row-major matrices in Z (scratch), result unpermuted into S; info[b] != 0
// flags a zero pivot in matrix b.
cudaError_t launch_gj_invert(double* Z, double* S, int m, int nmat, int* info, cudaStream_t st);
// U_e = S_e W_e, V_e = S_e sig_e for every element (S stride 0 if shared)
cudaError_t launch_block_gemv2(const double* S, int shared, const double* W, const double* sig,
                               double* U, double* V, int m, int nE, cudaStream_t st);
// out_k = S_e in_k for k < nr right-hand sides (nr in {2, 4, 6}), one streaming pass over
// the per-element S (not shared); bitwise equal to nr/2 calls of launch_block_gemv2
constexpr int GEMV_MAX_RHS = 6;
cudaError_t launch_block_gemv_multi(const double* S, int nr, const double* const* in, double* const* out, int m,
                                    int nE, cudaStream_t st);

// GMRES / Newton vector kernels.  Reductions are two-level (fixed block
// count, fixed order): deterministic.
constexpr int RED_BLOCKS = 592;         // 4 x 148 SMs
constexpr int RED_THREADS = 256;
// Arnoldi kernels: per-chunk partials part[k * nb + b], nb = arnoldi_dot_blocks(L)
int arnoldi_dot_blocks(size_t L);
// h_k = V_k . w (k < nk) and w . w (k = nk) -> part, nk + 1 rows
cudaError_t launch_arnoldi_dots(const double* V, size_t ldx, int nk, const double* w, size_t L, double* part,
                                cudaStream_t st);
// out[k] = sum_b part[k * nb + b]
cudaError_t launch_reduce_partials_n(const double* part, int nk, int nb, double* out, cudaStream_t st);
// w -= sum_k h_k V_k (h on device); per-chunk partial sums of the new w . w -> sq_part[nb]
cudaError_t launch_arnoldi_axpy(const double* V, size_t ldx, int nk, const double* h, double* w, size_t L,
                                double* sq_part, cudaStream_t st);
// out = sqrt(sum part[0..nb))
cudaError_t launch_finish_sqrt(const double* part, int nb, double* out, cudaStream_t st);
// DCGS2: rows 2k, 2k+1 = Q_k.u, Q_k.w (k < nk); rows 2nk.. = u.u, u.w, w.w  (w may be NULL)
cudaError_t launch_dcgs2_dots(const double* Q, size_t ldx, int nk, const double* u, const double* w, size_t L,
                              double* part, cudaStream_t st);
// DCGS2: u <- (u - Q a) ib ;  w <- w ib - Q d - u_old cb   (a, d on device)
cudaError_t launch_dcgs2_update(const double* Q, size_t ldx, int nk, const double* a, const double* d, double* u,
                                double* w, double ib, double cb, size_t L, cudaStream_t st);

// partial[k * RED_BLOCKS + b] = sum over block b of X_k . y   (k < nk), X_k = X + k*ldx
cudaError_t launch_multidot(const double* X, size_t ldx, int nk, const double* y, size_t L,
                            double* partial, cudaStream_t st);
// out[k] = sum_b partial[k * RED_BLOCKS + b] (+ out[k] if accumulate), k < nk
cudaError_t launch_reduce_partials(const double* partial, int nk, double* out, int accumulate, cudaStream_t st);
// y -= sum_k h[k] X_k  (h on device); if sq_partial != NULL also partial sums of y_new^2
cudaError_t launch_multiaxpy(const double* X, size_t ldx, int nk, const double* h, double* y, size_t L,
                             double* sq_partial, cudaStream_t st);
// y = sum_k c[k] X_k  (c on device)
cudaError_t launch_lincomb(const double* X, size_t ldx, int nk, const double* c, double* y, size_t L,
                           cudaStream_t st);
// y = x * (1 / *nrm)  (nrm on device; nrm == 0 -> y = 0)
cudaError_t launch_scale_by_inv(const double* x, const double* nrm, double* y, size_t L, cudaStream_t st);
// y = a x + b y   (host scalars)
cudaError_t launch_axpby(double a, const double* x, double b, double* y, size_t L, cudaStream_t st);
// y = a x + b z   (host scalars)
cudaError_t launch_waxpby(double a, const double* x, double b, const double* z, double* y, size_t L,
                          cudaStream_t st);
// partial sums of x.x (sumsq) into partial[0..RED_BLOCKS)
cudaError_t launch_sumsq(const double* x, size_t L, double* partial, cudaStream_t st);
// out = sqrt(sum partial)
cudaError_t launch_finish_norm(const double* partial, double* out, cudaStream_t st);
// out = c / sqrt(sum partial), or 0 if the sum is 0   (FD step)
// eps_FD from np partial sums of ||dW||^2 (np <= 0: RED_BLOCKS)
cudaError_t launch_finish_fd_eps(const double* partial, double c, double* out, cudaStream_t st, int np = 0);
// Euler / NS state admissibility: flag[0] = first bad node (0x7f7f7f7f if none), flag[1] = 1 non-finite | 2 rho/p <= 0
cudaError_t launch_admissible(const double* W, int nE, int nodes, int nv, double gamma, double eps2, int* flag,
                              cudaStream_t st);
// order-independent 64-bit fingerprint of x into *out (device), FSAL cache validation
cudaError_t launch_fingerprint(const double* x, size_t L, unsigned long long* out, cudaStream_t st);
// HBPC quadrature: y = base + sum_j a[j] X_j + sum_j b[j] Y_j  (host coefficient arrays, <= 8 terms)
cudaError_t launch_stage_combo(const double* base, int nx, const double* const* X, const double* a,
                               int ny, const double* const* Y, const double* b, double* y, size_t L,
                               cudaStream_t st);

// ---- halo.cu: face-trace halo of the element partition (comm.h) -----------------
constexpr int HALO_MAX_FIELDS = 4;
struct HaloLayout {
  int nx, ny, nv, P, dim;   // local element grid, variables, nodes per direction, dimension
  int active[4];            // sides taking part: -x, +x, -y, +y
  int gl;                   // Gauss-Legendre: send the interpolated traces sum_l l_l(+-1) w_l
  double lp[8], lm[8];      // l_l(+1), l_l(-1)
};
// segment offsets / lengths (doubles) of an exchange of nf fields
// (nvf: variables per element of each field; 0 = the state's n_v)
void halo_segments(const HaloLayout& L, int nf, size_t off[4], size_t len[4], int nvf = 0);
// send <- boundary-node values of src[0..nf) ; dst[f] ghost elements <- recv
// facebuf: the fields are BR2 face-gradient buffers [elem][face 4][nvf][P] (send face s, fill ghost face s^1)
cudaError_t launch_halo_pack(const HaloLayout& L, int nf, const double* const* src, double* send, cudaStream_t st,
                             int nvf = 0, bool facebuf = false);
cudaError_t launch_halo_unpack(const HaloLayout& L, int nf, const double* recv, double* const* dst, cudaStream_t st,
                               int nvf = 0, bool facebuf = false);
// out = c / sqrt(*sum), or 0 if *sum == 0
cudaError_t launch_fd_eps_from_sum(const double* sum, double c, double* out, cudaStream_t st);

// ---- sstep.cu: block Gram-Schmidt of the s-step Arnoldi process ------------------
int block_dot_blocks(size_t L);
// part rows j*s + l = Q_j . W_l (j < nq), rows nq*s + a*s + b = W_a . W_b; s in {2, 4, 8}
cudaError_t launch_block_dots(const double* Q, size_t ldq, int nq, const double* W, size_t ldw, int s, size_t L,
                              double* part, cudaStream_t st);
// W_l <- sum_m (W_m - sum_j Q_j C[j*s + m]) Rinv[m*s + l]  (Rinv upper triangular, NULL = I)
cudaError_t launch_block_update(const double* Q, size_t ldq, int nq, double* W, size_t ldw, int s, const double* C,
                                const double* Rinv, size_t L, cudaStream_t st);

// fp64 tensor-core (mma.sync m8n8k4 f64) versions, s in {4, 8}; same row layout
int block_dot_blocks_mma(size_t L);
cudaError_t launch_block_dots_mma(const double* Q, size_t ldq, int nq, const double* W, size_t ldw, int s, size_t L,
                                  double* part, cudaStream_t st);
cudaError_t launch_block_update_mma(const double* Q, size_t ldq, int nq, double* W, size_t ldw, int s,
                                    const double* C, const double* Rinv, size_t L, cudaStream_t st);
// TMA-streamed persistent versions for s = 8 (one CTA per SM, same row layout;
// dots partials: block_dot_parts_tma() per row).  Used while the basis is short
// (measured crossover with the register-streamed DMMA kernels, bench_block_tma.cu).
constexpr int BLOCK_TMA_DOTS_MAX_NQ = 72;
constexpr int BLOCK_TMA_UPDATE_MAX_NQ = 100;
int block_dot_blocks_tma();
int block_dot_parts_tma();
cudaError_t launch_block_dots_tma8(const double* Q, size_t ldq, int nq, const double* W, size_t ldw, size_t L,
                                   double* part, cudaStream_t st);
// gram (optional, nq >= 1): Gram rows a*8 + b of the OUTPUT block, block_fused_parts_tma() partials per row
cudaError_t launch_block_update_tma8(const double* Q, size_t ldq, int nq, double* W, size_t ldw, const double* C,
                                     const double* Rinv, size_t L, cudaStream_t st, double* gram = nullptr);
// W_l <- sum_{m <= l} W_m Rinv[m][l] for the 8 vectors of a block (second CholQR pass)
cudaError_t launch_block_scale_w8(double* W, size_t ldw, const double* Rinv, size_t L, cudaStream_t st);
// fused W <- W - Q C (Rinv = I) and rows of [Q W]^T W of the updated W in one
// pass over Q (1 <= nq <= block_fused_max_nq(); partials: block_fused_parts_tma() per row)
int block_fused_parts_tma();
int block_fused_max_nq();
cudaError_t launch_block_update_dots_tma8(const double* Q, size_t ldq, int nq, double* W, size_t ldw,
                                          const double* C, size_t L, double* part, cudaStream_t st);

// kernel-launch counter (reported by hbpdc_launch_count)
extern long long g_hbpdc_launches;
inline void hbpdc_count_launch() { ++g_hbpdc_launches; }

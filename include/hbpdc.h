/*
 * hbpdc.h -- C-ABI of the B200-native HBPC(q, k_max) / DGSEM hot path
 * (Zeifang & Schuetz, arXiv 2109.04804).
 *
 * Citation convention: "P:n" = line n of the paper's LaTeX source,
 * "S:n" = line n of SPEC.md, equations by their \label{} name.  Readings of
 * ambiguous passages (R1..R30) are listed in DESIGN.md.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - All arrays are IEEE binary64, DEVICE pointers (unless a name ends in
 *    _host), contiguous, in layout L = [elem][var][j][i] (i fastest) over the
 *    calling rank's local elements (elem = ey_local * nx_local + ex_local).
 *    A field has n_local = n_local_elems * m doubles, m = nv * (N+1)^dim.
 *  - Ownership: the caller owns every pointer argument.  The library owns
 *    all scratch (BJ_ext blocks, Krylov basis, stage store, halo buffers).
 *  - Stream semantics: work is enqueued on the context stream
 *    (hbpdc_dist.cuda_stream, or a library stream if NULL).  Calls that return
 *    host scalars (norm_out, stats) synchronise the stream; the others are
 *    asynchronous.
 *  - Aliasing: outputs must not alias inputs (except hbpdc_step's in/out W).
 *  - Errors: a non-zero hbpdc_status; hbpdc_last_error() gives a message
 *    (stage / sweep / Newton index, element and dt for LU breakdown).  No C++
 *    exception crosses the ABI, nothing calls exit().
 *  - Multi-GPU: every rank calls every function collectively with its local
 *    block; norms and stats come back globally reduced.
 */
#ifndef HBPDC_H
#define HBPDC_H

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define HBPDC_API __attribute__((visibility("default")))
#else
#define HBPDC_API
#endif

typedef struct hbpdc_ctx hbpdc_ctx;

typedef enum {
  HBPDC_OK = 0,
  HBPDC_E_ARG = 1,          /* invalid argument / unsupported configuration   */
  HBPDC_E_CUDA = 2,         /* CUDA runtime error                              */
  HBPDC_E_NCCL = 3,         /* NCCL error                                      */
  HBPDC_E_OOM = 4,          /* device allocation failed                        */
  HBPDC_E_NONFINITE = 5,    /* NaN/Inf detected in a residual or norm          */
  HBPDC_E_NEG_PRESSURE = 6, /* reserved                                        */
  HBPDC_E_LU_SINGULAR = 7,  /* zero pivot in the BJ_ext block inversion        */
  HBPDC_E_NEWTON = 8,       /* Newton did not converge within newton_max       */
  HBPDC_E_GMRES = 9         /* GMRES exceeded krylov_max_per_newton            */
} hbpdc_status;

enum { HBPDC_ADVECTION = 0, HBPDC_EULER = 1, HBPDC_NAVIER_STOKES = 2 };
enum { HBPDC_GLL = 0, HBPDC_GL = 1 };
enum { HBPDC_LLF = 0, HBPDC_GLF_PAPER = 1 };
enum { HBPDC_BR1 = 0, HBPDC_BR2 = 1 };
enum { HBPDC_PC_NONE = 0, HBPDC_PC_BJEXT = 1, HBPDC_PC_BJEXT_H = 2 };
enum { HBPDC_PC_PER_STEP_PER_ALPHA = 0, HBPDC_PC_PER_NEWTON = 1 };
enum { HBPDC_JVP_AUTO = 0, HBPDC_JVP_FD = 1, HBPDC_JVP_EXACT = 2, HBPDC_JVP_LINEAR = 3 };

/* The problem (P:43-47 conservation law; P:170 DGSEM degree N; P:83 HBPC(q,k_max)). */
typedef struct {
  int dim;              /* 1, 2 or 3 (3: hexahedra, advection or Euler, GLL, one rank;
                           NEXT-4, the paper's 3D case P:1080-1093, inviscid scope)   */
  int equation;         /* HBPDC_ADVECTION | HBPDC_EULER | HBPDC_NAVIER_STOKES     */
  double a[2];          /* advection velocity (advection only)                     */
  double gamma;         /* isentropic coefficient, e.g. 1.4                */
  double mach_eps;      /* reference Mach number eps of eq:Euler (configs: 1, R18;
                           Navier-Stokes: must be 1)                               */
  double mu;            /* dynamic viscosity (NS)                           */
  double prandtl;       /* Prandtl number (NS), e.g. 0.72                   */
  int N;                /* polynomial degree, 1..7                                 */
  int nodes;            /* HBPDC_GLL (configs, reading R1) or HBPDC_GL       */
  int nx, ny;           /* global element counts (ny ignored in 1D)                */
  double xmin, xmax, ymin, ymax;   /* periodic Cartesian domain                   */
  int flux;             /* HBPDC_LLF (reading R3) | HBPDC_GLF_PAPER (eq:Riemann, P:197-201,
                           literally: 1/2 (F_L + F_R).n + Lambda (w_L - w_R), no 1/2 on the
                           jump; Lambda = diag(1/eps,1,1,1/eps), |a.n|) */
  int lifting;          /* HBPDC_BR1 (NS, reading R19) | HBPDC_BR2 (reading R33) */
  int q, kmax;          /* HBPC(q, k_max), q in {4, 6, 8}, k_max >= 0              */
  double eta_br2;       /* BR2 stabilisation parameter eta (> 0; the paper gives no
                           value, reading R33); ignored for BR1                   */
  int nz;               /* 3D only: global element count in z (>= 1)               */
  double zmin, zmax;    /* 3D only: periodic extent in z                          */
  double az;            /* 3D advection only: z component of the velocity          */
} hbpdc_problem;

typedef struct {
  double newton_rtol;          /* ||G(X^r)|| <= rtol ||G(X^0)||               */
  double newton_atol_dw;       /* stop after a step with ||dW||_2 <= atol     */
  double newton_floor;         /* floor factor f: ||G|| <= f eps ||b|| (reading R10) */
  int newton_max;              /* max Newton iterations per stage solve       */
  double gmres_rtol;           /* relative GMRES tolerance             */
  int gmres_restart;           /* Krylov dimension before restart            */
  int krylov_max_per_newton;   /* total GMRES iterations per Newton step     */
  int precond;                 /* HBPDC_PC_NONE | HBPDC_PC_BJEXT |
                                  HBPDC_PC_BJEXT_H (with the Hessian block, P:269-296;
                                  advection / Euler; built at (W, R1(W)))              */
  int precond_policy;          /* HBPDC_PC_PER_STEP_PER_ALPHA (default) | PER_NEWTON */
  int jvp_mode;                /* HBPDC_JVP_AUTO: linear (advection) / FD otherwise  */
  int batch_stages;            /* 1: solve the s-1 corrector stages of a sweep in lock
                                  step, sharing one BJ_ext S pass per Arnoldi step
                                  (they are independent, eq:corrector P:119-122;
                                  SURVEY NEXT-1).  Bitwise equal results to 0.      */
  int gmres_sstep;             /* Arnoldi schedule: 0/1 = DCGS2 (one JVP per block,
                                  2 passes over the basis per iteration); s = 2, 4, 8:
                                  s-step blocks (s Newton-basis powers, then block CGS2
                                  + CholQR2: 4 passes over the basis per s iterations).
                                  Same Krylov space and GMRES iterates, other rounding. */
  int schur;                   /* 0: Newton on the extended system (eq:Newton);
                                  1: Schur complement: GMRES on
                                  J_S dw = -G1 + c2 K G2 (J_S = I - a1 dt K + c2 dR2/dW
                                  + c2 K^2, applied as the top block of J (v, K v)),
                                  dsigma = -G2 + K dw; preconditioned by the D block of
                                  BJ_ext / BJ^H_ext (element-block Jacobi, reading R32). */
} hbpdc_solver_opts;

/* Element partition (the mesh is decomposed, W and sigma share the
 * partition).  Rank r owns the element block (rx, ry) = (r % px, r / px) of
 * nx/px x ny/py elements; its local elements are numbered ey_l * nx_l + ex_l.
 * Face traces of the neighbouring blocks are exchanged before every operator
 * (halo), global norms and Krylov dot products are summed over ranks; the
 * BJ_ext preconditioner is rank-local.  See DESIGN.md "Multi-GPU". */
enum { HBPDC_COMM_AUTO = 0,      /* nranks == 1: none; else NCCL                      */
       HBPDC_COMM_NCCL = 1,      /* one process per GPU, NCCL over NVLink/NVSwitch    */
       HBPDC_COMM_LOOPBACK = 2   /* ranks are host threads of one process sharing a   */
};                               /* loopback group (tests the partition on one GPU)  */
typedef struct {
  int rank, nranks;            /* this rank, number of ranks                          */
  int px, py;                  /* rank grid: px * py == nranks, nx % px == ny % py == 0 */
  const void* nccl_unique_id;  /* 128-byte ncclUniqueId of rank 0 (COMM_NCCL)         */
  void* cuda_stream;           /* cudaStream_t to enqueue on (NULL = legacy default)  */
  int device;                  /* CUDA device ordinal                                 */
  int own_stream;              /* 1: ignore cuda_stream, the library creates a stream */
  int comm;                    /* HBPDC_COMM_*                                        */
  void* loopback_group;        /* from hbpdc_loopback_group_create (COMM_LOOPBACK)    */
  int force_halo;              /* 1: exchange halos even with oneself (periodic wrap
                                  of a 1-rank direction goes through the transport);
                                  a test hook for the transport on a single GPU      */
} hbpdc_dist;

typedef struct {               /* summed over one hbpdc_step                          */
  int stage_solves, newton_its, gmres_its, precond_builds, max_krylov_j;
  int jvp_calls, precond_applies;
  int precond_k_reused;        /* Navier-Stokes builds that reused this step's stored K_i   */
  double final_newton_rel, wall_s;
} hbpdc_step_stats;

/* Create a context: basis (GLL or GL nodes/weights, Dhat = -M^-1 D^T M, reading R2),
 * mesh, rank partition, NCCL communicator, scratch.  Host only. */
HBPDC_API hbpdc_status hbpdc_init(const hbpdc_problem* problem, const hbpdc_solver_opts* opts,
                        const hbpdc_dist* dist, hbpdc_ctx** out);

/* Host-only partition arithmetic (no device, no context): the element block of
 * `rank` on a px x py rank grid over an nx x ny mesh (ny = 1 in 1D) and its four
 * neighbour ranks [-x, +x, -y, +y] (periodic).  HBPDC_E_ARG if the grid does not
 * divide the mesh. */
HBPDC_API hbpdc_status hbpdc_partition(int dim, int nx, int ny, int px, int py, int rank, int* ex0, int* ey0,
                             int* nx_local, int* ny_local, int* nbr4);

/* Rank 0 creates the NCCL unique id (128 bytes, host) that every rank passes in
 * hbpdc_dist.nccl_unique_id; the caller distributes it (torch.distributed). */
HBPDC_API hbpdc_status hbpdc_nccl_unique_id(void* out128);

/* A loopback group for `nranks` ranks living as host threads of this process
 * (HBPDC_COMM_LOOPBACK).  Destroy after every context of the group is finalized. */
HBPDC_API hbpdc_status hbpdc_loopback_group_create(int nranks, void** group);
HBPDC_API void hbpdc_loopback_group_destroy(void* group);

/* Local block: element count, block size m, offsets and extents in elements. */
HBPDC_API hbpdc_status hbpdc_local_shape(const hbpdc_ctx* ctx, int* n_local_elems, int* m,
                               int* ex0, int* ey0, int* nx_local, int* ny_local);

/* Physical coordinates of the local nodes, layout [elem][j][i] (host arrays of
 * n_local_elems*(N+1)^dim doubles; y_host ignored in 1D).  Synchronous. */
HBPDC_API hbpdc_status hbpdc_node_coords(const hbpdc_ctx* ctx, double* x_host, double* y_host);
/* 3D: z coordinates of the local nodes, same order (host array of n_local_elems*(N+1)^3). */
HBPDC_API hbpdc_status hbpdc_node_coords_z(const hbpdc_ctx* ctx, double* z_host);

/* sigma == NULL: out = R^(1)_h(W) (eq:DGSEM_wt).
 * sigma != NULL: out = R^(2)_h(W, sigma) (eq:DGSEM_wtt): the time
 * derivative of R^(1)_h along w_t = sigma. */
HBPDC_API hbpdc_status hbpdc_rhs(hbpdc_ctx* ctx, const double* W, const double* sigma, double* out);

/* Extended stage residual (eq:Newton_Residual P:137-141, reading R4):
 *   G1 = W - a1 dt R1(W) + (a2 dt^2/2) R2(W, sigma) - b,   G2 = sigma - R1(W).
 * norm_out (host, may be NULL): global ||(G1, G2)||_2 (synchronises). */
HBPDC_API hbpdc_status hbpdc_residual(hbpdc_ctx* ctx, double alpha1, double alpha2, double dt,
                            const double* b, const double* W, const double* sigma,
                            double* G1, double* G2, double* norm_out);

/* Jacobian-vector product J dX of eq:nonlinear_eqsys:
 *   HBPDC_JVP_FD     : eq:MatrixFree_nonlinear with
 *                      eps_FD = sqrt(2^-52)/(eps ||d.||_2) (reading R7),
 *                      sigma direction R2(W, dsigma) (reading R8);
 *   HBPDC_JVP_EXACT  : the exact blocks (hyper-dual evaluation);
 *   HBPDC_JVP_LINEAR : eq:MatrixFree_linear, advection only;
 *   HBPDC_JVP_AUTO   : LINEAR for advection, FD otherwise.
 * out1 = top block, out2 = bottom block.  eps_override: NULL or a HOST array
 * [eps_w, eps_s] fixing eps_FD (<= 0 means "the quotient is 0"). */
HBPDC_API hbpdc_status hbpdc_jvp(hbpdc_ctx* ctx, double alpha1, double alpha2, double dt,
                       const double* W, const double* sigma, const double* dW,
                       const double* dsigma, double* out1, double* out2, int mode,
                       const double* eps_override);

/* BJ_ext build: K_i = element-diagonal block of dR1/dW at W,
 * S_i = (I - a1 dt K_i + (a2 dt^2/2) K_i^2)^-1 by Gauss-Jordan with partial
 * pivoting; advection stores one shared block. */
HBPDC_API hbpdc_status hbpdc_precond_build(hbpdc_ctx* ctx, double alpha1, double alpha2, double dt,
                                 const double* W);

/* Install caller-provided S blocks (device array, n_local_elems*m*m row-major,
 * or m*m if `shared`) together with the build state W and (a1, a2, dt).
 * Used by parity tests to apply the oracle's S. */
HBPDC_API hbpdc_status hbpdc_precond_set(hbpdc_ctx* ctx, double alpha1, double alpha2, double dt,
                               const double* W, const double* S, int shared);

/* Copy the current S blocks to the device array S_out of `capacity` doubles:
 * n_local_elems*m*m doubles, or m*m when *shared = 1 (advection: one block for
 * all elements).  S_out = NULL only reports *shared (size query).  A capacity
 * below the block count returns HBPDC_E_ARG without writing.  Test hook. */
HBPDC_API hbpdc_status hbpdc_precond_export(hbpdc_ctx* ctx, double* S_out, size_t capacity, int* shared);

/* P^-1 X per element: (D W + E s ; F W + G s), evaluated as
 * u = S W, v = S s, top = u - c2 K v, bottom = v + K (u - a1 dt v). */
HBPDC_API hbpdc_status hbpdc_precond_apply(hbpdc_ctx* ctx, const double* inW, const double* insig,
                                 double* outW, double* outsig);

/* One HBPC(q, k_max) step (Alg. 1) of size dt, W in/out (device).
 * stats may be NULL.  Synchronises. */
HBPDC_API hbpdc_status hbpdc_step(hbpdc_ctx* ctx, double dt, double* W, hbpdc_step_stats* stats);

/* Same, with W a HOST array: host->device copy, step, device->host copy. */
HBPDC_API hbpdc_status hbpdc_step_host(hbpdc_ctx* ctx, double dt, double* W_host, hbpdc_step_stats* stats);

/* Forget the FSAL cache (the next step recomputes R1/R2 of its input).
 * hbpdc_step reuses R1/R2 of its previous output (FSAL) only when it is
 * called with that same device array and unchanged contents (pointer and a
 * 64-bit fingerprint of W are checked); any other W recomputes them. */
HBPDC_API hbpdc_status hbpdc_reset(hbpdc_ctx* ctx);

/* Per-kernel timing (CUDA events on the context stream), for roofline
 * reporting.  enable=1 starts recording (and zeroes the counters), 0 stops.
 * kernel ids: 0 = precond GEMV (S streaming), 1 = JVP, 2 = residual,
 * 3 = Arnoldi dots, 4 = Arnoldi update, 5 = precond K-apply, 6 = precond
 * build, 7 = fused Arnoldi update + re-projection (s-step, s = 8).  alg_bytes = algorithmic HBM bytes of those launches (DESIGN.md
 * byte model: each input and output touched once). */
HBPDC_API hbpdc_status hbpdc_profile(hbpdc_ctx* ctx, int enable);
HBPDC_API hbpdc_status hbpdc_profile_read(hbpdc_ctx* ctx, int kernel_id, long long* launches,
                                double* total_ms, double* alg_bytes);

/* Number of kernels this process has launched through the library so far. */
HBPDC_API hbpdc_status hbpdc_launch_count(long long* count);

HBPDC_API const char* hbpdc_last_error(const hbpdc_ctx* ctx);
HBPDC_API void hbpdc_finalize(hbpdc_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* HBPDC_H */

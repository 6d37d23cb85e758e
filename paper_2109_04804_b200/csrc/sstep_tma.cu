// sstep_tma.cu -- TMA-streamed persistent block Gram-Schmidt kernels of the
// s-step Arnoldi process for s = 8 (one CTA per SM).
//
// The DMMA kernels of sstep.cu load Q straight into registers: every batch of
// loads is consumed before the next one is issued, so per CTA a pass is a
// chain of dependent DRAM round trips (ncu at C3: ~4.8 TB/s, 59% of DRAM peak,
// issue active 24%, 2 CTAs/SM).  Here the Q rows are bulk-copied
// (cp.async.bulk + mbarrier) into shared-memory rings that stay several
// stages ahead of the fp64 tensor-core (mma.sync m8n8k4 f64) consumers.
//
//   block_dots_tma8    rows j*8 + l : V_j . W_l,  V = [Q_0 .. Q_{nq-1}, W_0 .. W_7]
//   block_update_tma8  W_l <- sum_m (W_m - sum_j Q_j C[j*8 + m]) Rinv[m*8 + l]
//
// Same row layout / semantics as launch_block_dots_mma / launch_block_update_mma;
// deterministic (fixed chunk -> CTA map, fixed accumulation order).
#include <algorithm>
#include <cstdlib>
#include "launch.h"
#include "tma.cuh"

namespace {
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
constexpr int TD_E = 512;          // dots: elements per chunk (4 KB row copies: 2 KB ones cap the
                                   // stream at ~4.1 TB/s, 4 KB ones reach 6.5 TB/s, measured)
constexpr int TD_P = TD_E + 4;     // padded row (doubles): conflict-free A fragments
constexpr int TD_W = 16;           // consumer warps (8 cannot issue DMMAs fast enough: 4.1 TB/s)
constexpr int TD_R = 6;            // ring stages (shared by the consumer warps)
constexpr int TD_G = 16;           // tiles per group
constexpr int TD_C = 1;            // accumulator chains per tile
constexpr int TU_E = 256;          // update: elements per chunk
constexpr int TU_P = TU_E + 4;     // padded row: conflict-free B fragments
constexpr int TU_R = 8;            // ring stages (shared by the 8 consumer warps)
constexpr int TU_NB = TU_E / 64;   // n-blocks (8 elements) per consumer warp
}  // namespace

int block_dot_blocks_tma() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return nsm;
}
int block_dot_parts_tma() { return TD_W * block_dot_blocks_tma(); }

// Vector tile t = the 8 vectors 8t .. 8t+7 of V; tiles are taken in groups of
// up to TD_G (one group while nq + 8 <= 8 TD_G).  Per group the CTA walks its
// chunks (TD_E elements) and warp TD_W (one lane) streams every tile-chunk of
// the group through a TD_R-stage ring.  All TD_W consumer warps read every
// stage, warp w the k-steps of elements (TD_E / TD_W) w + 4 ks + t of the
// chunk, with its B fragments (W) in registers, prefetched one chunk ahead,
// and one accumulator per tile of the group.  Each consumer warp writes its
// own partial (deterministic: fixed element -> warp map; part has
// block_dot_parts_tma() columns per row).
__global__ void __launch_bounds__(32 * (TD_W + 1), 1) block_dots_tma8_kernel(const double* __restrict__ Q, size_t ldq, int nq,
                                                                 const double* __restrict__ W, size_t ldw,
                                                                 size_t L, double* __restrict__ part) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double* ring = reinterpret_cast<double*>(smraw);                            // TD_R x 8 x TD_P
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + (size_t)TD_R * 8 * TD_P);
  unsigned long long* empty = full + TD_R;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < TD_R * 8 * TD_P; k += blockDim.x) ring[k] = 0.0;
  if (threadIdx.x == 0) {
    for (int r = 0; r < TD_R; ++r) { mbar_init(&full[r], 1); mbar_init(&empty[r], TD_W); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async_smem();
  __syncthreads();
  const int nv = nq + 8;
  const int T = (nv + 7) / 8;
  const size_t nch = (L + TD_E - 1) / TD_E;
  const size_t nmy = blockIdx.x < nch ? (nch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (wid == TD_W) {                                                             // ---- producer
    if (lane == 0) {
      size_t k = 0;
      for (int t0 = 0; t0 < T; t0 += TD_G) {
        const int ng = min(TD_G, T - t0);
        for (size_t ci = 0; ci < nmy; ++ci) {
          const size_t e0 = (blockIdx.x + ci * gridDim.x) * TD_E;
          const int ne = (int)min((size_t)TD_E, L - e0);
          for (int tg = 0; tg < ng; ++tg, ++k) {
            const int st = (int)(k % TD_R);
            if (k >= (size_t)TD_R) mbar_wait(&empty[st], (unsigned)(((k / TD_R) - 1) & 1));
            const int tile = t0 + tg;
            const int nrow = min(8, nv - 8 * tile);
            mbar_expect_tx(&full[st], (unsigned)(nrow * ne * sizeof(double)));
            for (int r = 0; r < nrow; ++r) {
              const int j = 8 * tile + r;
              const double* src = j < nq ? Q + (size_t)j * ldq + e0 : W + (size_t)(j - nq) * ldw + e0;
              tma_load_1d(ring + ((size_t)st * 8 + r) * TD_P, src, (unsigned)(ne * sizeof(double)), &full[st]);
            }
          }
        }
      }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  constexpr int KW = TD_E / (4 * TD_W);          // k-steps per warp per stage (TD_E / TD_W elements)
  auto load_b = [&](size_t ci, double (&o)[KW]) {
    const size_t e0 = (blockIdx.x + ci * gridDim.x) * TD_E + (TD_E / TD_W) * wid;
    const double* wg = W + (size_t)g * ldw;
#pragma unroll
    for (int ks = 0; ks < KW; ++ks) {
      const size_t e = e0 + 4 * ks + t;
      o[ks] = e < L ? __ldg(wg + e) : 0.0;
    }
  };
  size_t k = 0;
  for (int t0 = 0; t0 < T; t0 += TD_G) {
    const int ng = min(TD_G, T - t0);
    double acc[TD_G][TD_C][2];
#pragma unroll
    for (int i = 0; i < TD_G; ++i)
#pragma unroll
      for (int c = 0; c < TD_C; ++c) { acc[i][c][0] = 0.0; acc[i][c][1] = 0.0; }
    double b[KW], bn[KW];
    if (nmy > 0) load_b(0, bn);
    for (size_t ci = 0; ci < nmy; ++ci) {
#pragma unroll
      for (int ks = 0; ks < KW; ++ks) b[ks] = bn[ks];
      if (ci + 1 < nmy) load_b(ci + 1, bn);
      // one stage at a time (the ring stays as full as possible); its KW
      // k-steps go to TD_C accumulators per tile (a DMMA's latency is long:
      // a single chain per stage would serialise KW of them)
#pragma unroll
      for (int tg = 0; tg < TD_G; ++tg) {
        if (tg < ng) {
          const int st = (int)(k % TD_R);
          mbar_wait(&full[st], (unsigned)((k / TD_R) & 1));
          const double* sa = ring + (size_t)st * 8 * TD_P + g * TD_P + (TD_E / TD_W) * wid + t;
#pragma unroll
          for (int ks = 0; ks < KW; ++ks) dmma(acc[tg][ks % TD_C], sa[4 * ks], b[ks]);
          fence_proxy_async_smem();      // order this lane's reads before the stage's next bulk copy
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[st]);
          ++k;
        }
      }
    }
    // one partial per consumer warp: part[row][TD_W * blockIdx + wid]
#pragma unroll
    for (int tg = 0; tg < TD_G; ++tg) {
      const int j = 8 * (t0 + tg) + g;
      if (tg < ng && j < nv) {
        double s0 = acc[tg][0][0], s1 = acc[tg][0][1];
#pragma unroll
        for (int c = 1; c < TD_C; ++c) { s0 += acc[tg][c][0]; s1 += acc[tg][c][1]; }
        const size_t col = (size_t)blockIdx.x * TD_W + wid, ncol = (size_t)gridDim.x * TD_W;
        part[((size_t)j * 8 + 2 * t) * ncol + col] = s0;
        part[((size_t)j * 8 + 2 * t + 1) * ncol + col] = s1;
      }
    }
  }
}

// nq >= 1.  Warp 8 (one lane) streams, per chunk of TU_E elements, the Q tiles
// (8 vectors each) through a TU_R-stage ring; the 8 consumer warps take TU_NB
// n-blocks of 8 elements each: D (8 W x 8 elements) += A (C^T, 8 x 4, shared
// memory) x B (4 Q vectors x 8 elements, the stage).  Then tmp = W - D and
// out_l = sum_{m <= l} Rinv[m][l] tmp_m with the 8 tmp rows gathered by shuffles.
__global__ void __launch_bounds__(288, 1) block_update_tma8_kernel(const double* __restrict__ Q, size_t ldq, int nq,
                                                                   double* __restrict__ W, size_t ldw,
                                                                   const double* __restrict__ C,
                                                                   const double* __restrict__ Rinv, size_t L,
                                                                   double* __restrict__ gram) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int nq8 = (nq + 7) / 8 * 8;
  double* ring = reinterpret_cast<double*>(smraw);                            // TU_R x 8 x TU_P
  double* sC = ring + (size_t)TU_R * 8 * TU_P;                                // C (zero padded to nq8 x 8)
  double* sR = sC + (size_t)nq8 * 8;                                          // Rinv (or I), 8 x 8
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sR + 64);
  unsigned long long* empty = full + TU_R;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < TU_R * 8 * TU_P; k += blockDim.x) ring[k] = 0.0;
  for (int k = threadIdx.x; k < nq8 * 8; k += blockDim.x) sC[k] = k < nq * 8 ? C[k] : 0.0;
  for (int k = threadIdx.x; k < 64; k += blockDim.x) sR[k] = Rinv ? Rinv[k] : ((k / 8 == k % 8) ? 1.0 : 0.0);
  if (threadIdx.x == 0) {
    for (int r = 0; r < TU_R; ++r) { mbar_init(&full[r], 1); mbar_init(&empty[r], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async_smem();
  __syncthreads();
  const int T = nq8 / 8;
  const size_t nch = (L + TU_E - 1) / TU_E;
  const size_t nmy = blockIdx.x < nch ? (nch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (wid == 8) {                                                             // ---- producer
    if (lane == 0) {
      size_t k = 0;
      for (size_t ci = 0; ci < nmy; ++ci) {
        const size_t e0 = (blockIdx.x + ci * gridDim.x) * TU_E;
        const int ne = (int)min((size_t)TU_E, L - e0);
        for (int tile = 0; tile < T; ++tile, ++k) {
          const int st = (int)(k % TU_R);
          if (k >= (size_t)TU_R) mbar_wait(&empty[st], (unsigned)(((k / TU_R) - 1) & 1));
          const int nrow = min(8, nq - 8 * tile);
          mbar_expect_tx(&full[st], (unsigned)(nrow * ne * sizeof(double)));
          for (int r = 0; r < nrow; ++r)
            tma_load_1d(ring + ((size_t)st * 8 + r) * TU_P, Q + (size_t)(8 * tile + r) * ldq + e0,
                        (unsigned)(ne * sizeof(double)), &full[st]);
        }
      }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  auto load_w = [&](size_t ci, double (&o)[TU_NB][2]) {
    const size_t e0 = (blockIdx.x + ci * gridDim.x) * TU_E;
    const double* wg = W + (size_t)g * ldw;
#pragma unroll
    for (int nb = 0; nb < TU_NB; ++nb) {
      const size_t e = e0 + (size_t)(wid * TU_NB + nb) * 8 + 2 * t;
      if (e + 1 < L) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(wg + e));
        o[nb][0] = v.x;
        o[nb][1] = v.y;
      } else {
        o[nb][0] = e < L ? wg[e] : 0.0;
        o[nb][1] = 0.0;
      }
    }
  };
  double gacc[2] = {0.0, 0.0};
  double wv[TU_NB][2], wn[TU_NB][2];
  if (nmy > 0) load_w(0, wn);
  size_t k = 0;
  for (size_t ci = 0; ci < nmy; ++ci) {
    const size_t e0 = (blockIdx.x + ci * gridDim.x) * TU_E;
#pragma unroll
    for (int nb = 0; nb < TU_NB; ++nb) { wv[nb][0] = wn[nb][0]; wv[nb][1] = wn[nb][1]; }
    if (ci + 1 < nmy) load_w(ci + 1, wn);
    double acc[TU_NB][2];
#pragma unroll
    for (int nb = 0; nb < TU_NB; ++nb) { acc[nb][0] = 0.0; acc[nb][1] = 0.0; }
    for (int tile = 0; tile < T; ++tile, ++k) {
      const int st = (int)(k % TU_R);
      mbar_wait(&full[st], (unsigned)((k / TU_R) & 1));
      const double* sb = ring + (size_t)st * 8 * TU_P + (size_t)(wid * TU_NB) * 8 + g;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const double a = sC[(8 * tile + 4 * kk + t) * 8 + g];
#pragma unroll
        for (int nb = 0; nb < TU_NB; ++nb) dmma(acc[nb], a, sb[(4 * kk + t) * TU_P + nb * 8]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    // lane (g, t) holds D[g][e] for e = n-block base + 2t, 2t + 1
#pragma unroll
    for (int nb = 0; nb < TU_NB; ++nb) {
      const double t0 = wv[nb][0] - acc[nb][0], t1 = wv[nb][1] - acc[nb][1];
      double o0 = 0.0, o1 = 0.0;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const double v0 = __shfl_sync(0xffffffffu, t0, m * 4 + t);
        const double v1 = __shfl_sync(0xffffffffu, t1, m * 4 + t);
        if (m <= g) {
          const double r = sR[m * 8 + g];
          o0 = fma(v0, r, o0);
          o1 = fma(v1, r, o1);
        }
      }
      const size_t e = e0 + (size_t)(wid * TU_NB + nb) * 8 + 2 * t;
      double* wg = W + (size_t)g * ldw;
      if (e + 1 < L) {
        *reinterpret_cast<double2*>(wg + e) = make_double2(o0, o1);
      } else if (e < L) {
        wg[e] = o0;
      }
      if (gram) {
        // Gram of the output block (the next CholQR pass) from registers: B fragment
        // (element 4 kk + t of the n-block, vector g) gathered by shuffles; beyond L: 0
        const double u0 = e < L ? o0 : 0.0, u1 = e + 1 < L ? o1 : 0.0;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int src = g * 4 + 2 * kk + (t >> 1);
          const double v0 = __shfl_sync(0xffffffffu, u0, src);
          const double v1 = __shfl_sync(0xffffffffu, u1, src);
          const double bfv = (t & 1) ? v1 : v0;
          dmma(gacc, bfv, bfv);
        }
      }
    }
  }
  if (gram) {   // one partial per consumer warp: gram[(a * 8 + b)][8 * blockIdx + wid]
    const size_t col = (size_t)blockIdx.x * 8 + wid, ncol = (size_t)gridDim.x * 8;
    gram[((size_t)g * 8 + 2 * t) * ncol + col] = gacc[0];
    gram[((size_t)g * 8 + 2 * t + 1) * ncol + col] = gacc[1];
  }
}

// W_l <- sum_{m <= l} W_m Rinv[m][l] (Rinv upper triangular, 8 x 8): the second
// CholQR pass of a block, one streaming read + write of the 8 vectors
__global__ void __launch_bounds__(256) block_scale_w8_kernel(double* __restrict__ W, size_t ldw,
                                                            const double* __restrict__ Rinv, size_t L) {
  __shared__ double sR[64];
  if (threadIdx.x < 64) sR[threadIdx.x] = Rinv[threadIdx.x];
  __syncthreads();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += (size_t)gridDim.x * blockDim.x) {
    double x[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) x[m] = __ldcs(W + (size_t)m * ldw + i);
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      double o = 0.0;
#pragma unroll
      for (int m = 0; m <= l; ++m) o = fma(x[m], sR[m * 8 + l], o);
      __stcs(W + (size_t)l * ldw + i, o);
    }
  }
}

cudaError_t launch_block_dots_tma8(const double* Q, size_t ldq, int nq, const double* W, size_t ldw, size_t L,
                                   double* part, cudaStream_t st) {
  if ((ldq & 1) || (ldw & 1)) return cudaErrorInvalidValue;     // 16-B aligned rows for the bulk copies
  const size_t smem = (size_t)TD_R * 8 * TD_P * sizeof(double) +
                      2 * TD_R * sizeof(unsigned long long);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(block_dots_tma8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  block_dots_tma8_kernel<<<block_dot_blocks_tma(), 32 * (TD_W + 1), smem, st>>>(Q, ldq, nq, W, ldw, L, part);
  hbpdc_count_launch();
  return cudaGetLastError();
}

cudaError_t launch_block_scale_w8(double* W, size_t ldw, const double* Rinv, size_t L, cudaStream_t st) {
  const int grid = (int)std::min<size_t>((L + 255) / 256, (size_t)block_dot_blocks_tma() * 8);
  block_scale_w8_kernel<<<grid, 256, 0, st>>>(W, ldw, Rinv, L);
  hbpdc_count_launch();
  return cudaGetLastError();
}

cudaError_t launch_block_update_tma8(const double* Q, size_t ldq, int nq, double* W, size_t ldw, const double* C,
                                     const double* Rinv, size_t L, cudaStream_t st, double* gram) {
  if (nq < 1 && !gram) return launch_block_update_mma(Q, ldq, nq, W, ldw, 8, C, Rinv, L, st);
  if (nq < 1) return cudaErrorInvalidValue;
  if ((ldq & 1) || (ldw & 1)) return cudaErrorInvalidValue;
  const int nq8 = (nq + 7) / 8 * 8;
  const size_t smem = ((size_t)TU_R * 8 * TU_P + (size_t)nq8 * 8 + 64) * sizeof(double) +
                      2 * TU_R * sizeof(unsigned long long);
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(block_update_tma8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return cudaErrorInvalidValue;
    attr = smem;
  }
  block_update_tma8_kernel<<<block_dot_blocks_tma(), 288, smem, st>>>(Q, ldq, nq, W, ldw, C, Rinv, L, gram);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// ============================================================================
// Fused first update + second projection of block CGS2 (s = 8):
//   W1 = W - Q C1                      (written back to W)
//   part rows j*8 + l   : Q_j . W1_l   (j < nq)
//   part rows nq*8 + a*8 + b : W1_a . W1_b
// i.e. block_update (Rinv = I) followed by block_dots, in ONE pass over Q from
// HBM: per chunk the producer streams the Q tiles twice, the second time from
// L2 (a chunk's tiles are nq x 2 KB per CTA, ~40 MB over all CTAs at nq = 126,
// well inside the 126 MB L2).  Phase U is block_update_tma8's consumer loop;
// W1 stays in registers, its B fragments (element 4 kk + t of an n-block,
// vector g) are gathered by shuffles, and phase D accumulates Q_tile^T W1 on
// the tensor cores into per-warp accumulators that persist over the CTA's
// chunks (one partial per consumer warp, as block_dots_tma8).
// ============================================================================
namespace {
#ifndef TF_MAXT_
#define TF_MAXT_ 20
#endif
constexpr int TF_MAXT = TF_MAXT_;  // Q tiles (nq <= 8 TF_MAXT) kept in accumulators
#ifndef TF_E_
#define TF_E_ 512
#endif
#ifndef TF_PAR_
#define TF_PAR_ 1
#endif
constexpr int TF_E = TF_E_;        // elements per chunk (row copies of 8 TF_E bytes)
constexpr int TF_P = TF_E + 4;     // padded row: conflict-free fragments
#ifndef TF_R_
#define TF_R_ ((200 * 1024) / (8 * TF_P * 8))
#endif
constexpr int TF_R = TF_R_;        // ring stages
#ifndef TF_W_
#define TF_W_ 8
#endif
constexpr int TF_W = TF_W_;        // consumer warps
#ifndef TF_DCH_
#define TF_DCH_ 1
#endif
constexpr int TF_DCH = TF_DCH_;    // transient accumulator chains per tile in phase D
constexpr int TF_NB = TF_E / (8 * TF_W);   // n-blocks per consumer warp
}
int block_fused_parts_tma() {
  static_assert(TF_W == 8, "block_update_tma8's Gram partials share this column count");
  return TF_W * block_dot_blocks_tma();
}
int block_fused_max_nq() { return 8 * TF_MAXT; }

__global__ void __launch_bounds__(32 * (TF_W + 1), 1) block_update_dots_tma8_kernel(const double* __restrict__ Q, size_t ldq,
                                                                        int nq, double* __restrict__ W, size_t ldw,
                                                                        const double* __restrict__ C, size_t L,
                                                                        double* __restrict__ part) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int nq8 = (nq + 7) / 8 * 8;
  double* ring = reinterpret_cast<double*>(smraw);                            // TF_R x 8 x TF_P
  double* sC = ring + (size_t)TF_R * 8 * TF_P;                                // C1 (zero padded to nq8 x 8)
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sC + (size_t)nq8 * 8);
  unsigned long long* empty = full + TF_R;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < TF_R * 8 * TF_P; k += blockDim.x) ring[k] = 0.0;
  for (int k = threadIdx.x; k < nq8 * 8; k += blockDim.x) sC[k] = k < nq * 8 ? C[k] : 0.0;
  if (threadIdx.x == 0) {
    for (int r = 0; r < TF_R; ++r) { mbar_init(&full[r], 1); mbar_init(&empty[r], TF_W); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async_smem();
  __syncthreads();
  const int T = nq8 / 8;
  const size_t nch = (L + TF_E - 1) / TF_E;
  const size_t nmy = blockIdx.x < nch ? (nch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (wid == TF_W) {                                                          // ---- producer
    // lane 0 waits / arms the stage, lanes 0..7 issue one row copy each
    size_t k = 0;
    for (size_t ci = 0; ci < nmy; ++ci) {
      const size_t e0 = (blockIdx.x + ci * gridDim.x) * TF_E;
      const int ne = (int)min((size_t)TF_E, L - e0);
      for (int pass = 0; pass < 2; ++pass)                                    // phase U, then phase D (L2)
        for (int tile = 0; tile < T; ++tile, ++k) {
          const int st = (int)(k % TF_R);
          const int nrow = min(8, nq - 8 * tile);
          if (lane == 0) {
            if (k >= (size_t)TF_R) mbar_wait(&empty[st], (unsigned)(((k / TF_R) - 1) & 1));
            mbar_expect_tx(&full[st], (unsigned)(nrow * ne * sizeof(double)));
          }
          __syncwarp();
          if (TF_PAR_) {
            if (lane < nrow)
              tma_load_1d(ring + ((size_t)st * 8 + lane) * TF_P, Q + (size_t)(8 * tile + lane) * ldq + e0,
                          (unsigned)(ne * sizeof(double)), &full[st]);
          } else if (lane == 0) {
            for (int r = 0; r < nrow; ++r)
              tma_load_1d(ring + ((size_t)st * 8 + r) * TF_P, Q + (size_t)(8 * tile + r) * ldq + e0,
                          (unsigned)(ne * sizeof(double)), &full[st]);
          }
        }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  auto load_w = [&](size_t ci, double (&o)[TF_NB][2]) {
    const size_t e0 = (blockIdx.x + ci * gridDim.x) * TF_E;
    const double* wg = W + (size_t)g * ldw;
#pragma unroll
    for (int nb = 0; nb < TF_NB; ++nb) {
      const size_t e = e0 + (size_t)(wid * TF_NB + nb) * 8 + 2 * t;
      if (e + 1 < L) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(wg + e));
        o[nb][0] = v.x;
        o[nb][1] = v.y;
      } else {
        o[nb][0] = e < L ? wg[e] : 0.0;
        o[nb][1] = 0.0;
      }
    }
  };
  double dacc[TF_MAXT][2], gacc[2] = {0.0, 0.0};
#pragma unroll
  for (int i = 0; i < TF_MAXT; ++i) { dacc[i][0] = 0.0; dacc[i][1] = 0.0; }
  size_t k = 0;
  for (size_t ci = 0; ci < nmy; ++ci) {
    const size_t e0 = (blockIdx.x + ci * gridDim.x) * TF_E;
    double wv[TF_NB][2];
    load_w(ci, wv);                    // consumed after phase U: the latency hides behind it
    // ---- phase U: D = C1^T Q over the chunk (block_update_tma8)
    double acc[TF_NB][2];
#pragma unroll
    for (int nb = 0; nb < TF_NB; ++nb) { acc[nb][0] = 0.0; acc[nb][1] = 0.0; }
    for (int tile = 0; tile < T; ++tile, ++k) {
      const int st = (int)(k % TF_R);
      mbar_wait(&full[st], (unsigned)((k / TF_R) & 1));
      const double* sb = ring + (size_t)st * 8 * TF_P + (size_t)(wid * TF_NB) * 8 + g;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const double a = sC[(8 * tile + 4 * kk + t) * 8 + g];
#pragma unroll
        for (int nb = 0; nb < TF_NB; ++nb) dmma(acc[nb], a, sb[(4 * kk + t) * TF_P + nb * 8]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    // W1 = W - D (lane (g, t): vector g, elements 2t, 2t + 1 of each n-block) -> W
    double (&w1)[TF_NB][2] = acc;
#pragma unroll
    for (int nb = 0; nb < TF_NB; ++nb) {
      const size_t e = e0 + (size_t)(wid * TF_NB + nb) * 8 + 2 * t;
      w1[nb][0] = e < L ? wv[nb][0] - acc[nb][0] : 0.0;          // beyond L: 0 (stale ring rows)
      w1[nb][1] = e + 1 < L ? wv[nb][1] - acc[nb][1] : 0.0;
      double* wg = W + (size_t)g * ldw;
      if (e + 1 < L) {
        *reinterpret_cast<double2*>(wg + e) = make_double2(w1[nb][0], w1[nb][1]);
      } else if (e < L) {
        wg[e] = w1[nb][0];
      }
    }
    // B fragments of W1: k-step (nb, kk) covers elements 4 kk + t of n-block nb,
    // held by lane g*4 + 2kk + t/2 at position t & 1 (elements >= L are 0)
    double bf[TF_NB][2];
#pragma unroll
    for (int nb = 0; nb < TF_NB; ++nb)
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int src = g * 4 + 2 * kk + (t >> 1);
        const double v0 = __shfl_sync(0xffffffffu, w1[nb][0], src);
        const double v1 = __shfl_sync(0xffffffffu, w1[nb][1], src);
        bf[nb][kk] = (t & 1) ? v1 : v0;
      }
    // Gram W1^T W1: A fragment (vector g, element k) equals the B fragment
#pragma unroll
    for (int nb = 0; nb < TF_NB; ++nb)
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma(gacc, bf[nb][kk], bf[nb][kk]);
    // ---- phase D: Q_tile^T W1 over the chunk (tiles re-streamed, from L2)
#pragma unroll
    for (int tile = 0; tile < TF_MAXT; ++tile) {
      if (tile < T) {
        const int st = (int)(k % TF_R);
        mbar_wait(&full[st], (unsigned)((k / TF_R) & 1));
        const double* sa = ring + (size_t)st * 8 * TF_P + (size_t)g * TF_P + (size_t)(wid * TF_NB) * 8 + t;
        if constexpr (TF_DCH == 1) {
#pragma unroll
          for (int nb = 0; nb < TF_NB; ++nb)
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) dmma(dacc[tile], sa[nb * 8 + 4 * kk], bf[nb][kk]);
        } else {
          // the tile's 2 TF_NB k-steps go to TF_DCH transient accumulator chains (a single
          // chain serialises them on the DMMA latency); summed in chain order (deterministic)
          double ch[TF_DCH][2];
          ch[0][0] = dacc[tile][0];
          ch[0][1] = dacc[tile][1];
#pragma unroll
          for (int c = 1; c < TF_DCH; ++c) { ch[c][0] = 0.0; ch[c][1] = 0.0; }
#pragma unroll
          for (int nb = 0; nb < TF_NB; ++nb)
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) dmma(ch[(2 * nb + kk) % TF_DCH], sa[nb * 8 + 4 * kk], bf[nb][kk]);
          double s0 = ch[0][0], s1 = ch[0][1];
#pragma unroll
          for (int c = 1; c < TF_DCH; ++c) { s0 += ch[c][0]; s1 += ch[c][1]; }
          dacc[tile][0] = s0;
          dacc[tile][1] = s1;
        }
        fence_proxy_async_smem();      // order this lane's reads before the stage's next bulk copy
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        ++k;
      }
    }
  }
  // one partial per consumer warp: part[row][TF_W * blockIdx + wid]
  const size_t col = (size_t)blockIdx.x * TF_W + wid, ncol = (size_t)gridDim.x * TF_W;
#pragma unroll
  for (int tile = 0; tile < TF_MAXT; ++tile) {
    const int j = 8 * tile + g;
    if (tile < T && j < nq) {
      part[((size_t)j * 8 + 2 * t) * ncol + col] = dacc[tile][0];
      part[((size_t)j * 8 + 2 * t + 1) * ncol + col] = dacc[tile][1];
    }
  }
  part[((size_t)nq * 8 + g * 8 + 2 * t) * ncol + col] = gacc[0];
  part[((size_t)nq * 8 + g * 8 + 2 * t + 1) * ncol + col] = gacc[1];
}

// Chunk-resident variant (round 2): the chunk's Q tiles stay in shared memory between phase U
// and phase D (no L2 re-stream).  Chunks of TR_E = 64 elements (512 B row copies, 4 KB tiles),
// a 47-tile ring: a chunk holds T = nq / 8 <= 20 slots from its phase-U wait to its phase-D
// release, and the ring holds the whole next chunk besides (measured: with 128-element chunks
// and a 24-tile ring only part of the next chunk fits and its last tiles are issued after the
// phase-D releases -- 3.0 TB/s), so HBM never waits on the L2 pass (ncu r02o: the L2 re-read version ran at
// 49 % of DRAM peak, 4.0 TB/s of algorithmic bytes).  Same partial layout as above (TF_W
// consumer warps, one partial each); only the element -> warp map (and so the rounding order)
// differs.  NOT the default: the bulk copies are then 512 B / 1 KB rows and the copy issue rate,
// not the bytes, bounds the stream (C3 bench, r02r/r02s: 1.5 TB/s with 64-element chunks,
// 3.0 TB/s with 128, against 4.2 TB/s for the L2 re-stream kernel with 4 KB rows).  Kept behind
// HBPDC_FUSED_RES=1 for the record; a 2D-tensor TMA box (8 rows x 64 elements per copy, swizzled)
// would be the way to make the resident schedule pay.
namespace {
#ifndef TR_E_
#define TR_E_ 64
#endif
constexpr int TR_E = TR_E_;
constexpr int TR_P = TR_E + 4;
constexpr int TR_R = (200 * 1024) / (8 * TR_P * 8);
constexpr int TR_NB = TR_E / (8 * TF_W);
static_assert(TR_R >= TF_MAXT, "a chunk must fit the ring");
static_assert(TR_NB >= 1, "TR_E: at least one 8-element n-block per consumer warp");
}
__global__ void __launch_bounds__(32 * (TF_W + 1), 1) block_update_dots_res8_kernel(const double* __restrict__ Q, size_t ldq,
                                                                        int nq, double* __restrict__ W, size_t ldw,
                                                                        const double* __restrict__ C, size_t L,
                                                                        double* __restrict__ part) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int nq8 = (nq + 7) / 8 * 8;
  double* ring = reinterpret_cast<double*>(smraw);                            // TR_R x 8 x TR_P
  double* sC = ring + (size_t)TR_R * 8 * TR_P;                                // C1 (zero padded to nq8 x 8)
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sC + (size_t)nq8 * 8);
  unsigned long long* empty = full + TR_R;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < TR_R * 8 * TR_P; k += blockDim.x) ring[k] = 0.0;
  for (int k = threadIdx.x; k < nq8 * 8; k += blockDim.x) sC[k] = k < nq * 8 ? C[k] : 0.0;
  if (threadIdx.x == 0) {
    for (int r = 0; r < TR_R; ++r) { mbar_init(&full[r], 1); mbar_init(&empty[r], TF_W); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async_smem();
  __syncthreads();
  const int T = nq8 / 8;
  const size_t nch = (L + TR_E - 1) / TR_E;
  const size_t nmy = blockIdx.x < nch ? (nch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (wid == TF_W) {                                                          // ---- producer
    size_t k = 0;
    for (size_t ci = 0; ci < nmy; ++ci) {
      const size_t e0 = (blockIdx.x + ci * gridDim.x) * TR_E;
      const int ne = (int)min((size_t)TR_E, L - e0);
      for (int tile = 0; tile < T; ++tile, ++k) {
        const int st = (int)(k % TR_R);
        const int nrow = min(8, nq - 8 * tile);
        if (lane == 0) {
          if (k >= (size_t)TR_R) mbar_wait(&empty[st], (unsigned)(((k / TR_R) - 1) & 1));
          mbar_expect_tx(&full[st], (unsigned)(nrow * ne * sizeof(double)));
        }
        __syncwarp();
        if (lane < nrow)
          tma_load_1d(ring + ((size_t)st * 8 + lane) * TR_P, Q + (size_t)(8 * tile + lane) * ldq + e0,
                      (unsigned)(ne * sizeof(double)), &full[st]);
      }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  double dacc[TF_MAXT][2], gacc[2] = {0.0, 0.0};
#pragma unroll
  for (int i = 0; i < TF_MAXT; ++i) { dacc[i][0] = 0.0; dacc[i][1] = 0.0; }
  size_t k0 = 0;
  for (size_t ci = 0; ci < nmy; ++ci, k0 += T) {
    const size_t e0 = (blockIdx.x + ci * gridDim.x) * TR_E;
    double wv[TR_NB][2];
    {
      const double* wg = W + (size_t)g * ldw;
#pragma unroll
      for (int nb = 0; nb < TR_NB; ++nb) {
        const size_t e = e0 + (size_t)(wid * TR_NB + nb) * 8 + 2 * t;
        if (e + 1 < L) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(wg + e));
          wv[nb][0] = v.x;
          wv[nb][1] = v.y;
        } else {
          wv[nb][0] = e < L ? wg[e] : 0.0;
          wv[nb][1] = 0.0;
        }
      }
    }
    // ---- phase U: D = C1^T Q over the chunk; the tiles stay in the ring
    double acc[TR_NB][2];
#pragma unroll
    for (int nb = 0; nb < TR_NB; ++nb) { acc[nb][0] = 0.0; acc[nb][1] = 0.0; }
    for (int tile = 0; tile < T; ++tile) {
      const size_t k = k0 + tile;
      const int st = (int)(k % TR_R);
      mbar_wait(&full[st], (unsigned)((k / TR_R) & 1));
      const double* sb = ring + (size_t)st * 8 * TR_P + (size_t)(wid * TR_NB) * 8 + g;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const double a = sC[(8 * tile + 4 * kk + t) * 8 + g];
#pragma unroll
        for (int nb = 0; nb < TR_NB; ++nb) dmma(acc[nb], a, sb[(4 * kk + t) * TR_P + nb * 8]);
      }
    }
    double (&w1)[TR_NB][2] = acc;
#pragma unroll
    for (int nb = 0; nb < TR_NB; ++nb) {
      const size_t e = e0 + (size_t)(wid * TR_NB + nb) * 8 + 2 * t;
      w1[nb][0] = e < L ? wv[nb][0] - acc[nb][0] : 0.0;          // beyond L: 0 (stale ring rows)
      w1[nb][1] = e + 1 < L ? wv[nb][1] - acc[nb][1] : 0.0;
      double* wg = W + (size_t)g * ldw;
      if (e + 1 < L) {
        *reinterpret_cast<double2*>(wg + e) = make_double2(w1[nb][0], w1[nb][1]);
      } else if (e < L) {
        wg[e] = w1[nb][0];
      }
    }
    double bf[TR_NB][2];
#pragma unroll
    for (int nb = 0; nb < TR_NB; ++nb)
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int src = g * 4 + 2 * kk + (t >> 1);
        const double v0 = __shfl_sync(0xffffffffu, w1[nb][0], src);
        const double v1 = __shfl_sync(0xffffffffu, w1[nb][1], src);
        bf[nb][kk] = (t & 1) ? v1 : v0;
      }
#pragma unroll
    for (int nb = 0; nb < TR_NB; ++nb)
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma(gacc, bf[nb][kk], bf[nb][kk]);
    // ---- phase D: Q_tile^T W1 from the resident tiles, then release them
#pragma unroll
    for (int tile = 0; tile < TF_MAXT; ++tile) {
      if (tile < T) {
        const size_t k = k0 + tile;
        const int st = (int)(k % TR_R);
        const double* sa = ring + (size_t)st * 8 * TR_P + (size_t)g * TR_P + (size_t)(wid * TR_NB) * 8 + t;
#pragma unroll
        for (int nb = 0; nb < TR_NB; ++nb)
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) dmma(dacc[tile], sa[nb * 8 + 4 * kk], bf[nb][kk]);
        fence_proxy_async_smem();      // order this lane's reads before the stage's next bulk copy
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
    }
  }
  const size_t col = (size_t)blockIdx.x * TF_W + wid, ncol = (size_t)gridDim.x * TF_W;
#pragma unroll
  for (int tile = 0; tile < TF_MAXT; ++tile) {
    const int j = 8 * tile + g;
    if (tile < T && j < nq) {
      part[((size_t)j * 8 + 2 * t) * ncol + col] = dacc[tile][0];
      part[((size_t)j * 8 + 2 * t + 1) * ncol + col] = dacc[tile][1];
    }
  }
  part[((size_t)nq * 8 + g * 8 + 2 * t) * ncol + col] = gacc[0];
  part[((size_t)nq * 8 + g * 8 + 2 * t + 1) * ncol + col] = gacc[1];
}

cudaError_t launch_block_update_dots_tma8(const double* Q, size_t ldq, int nq, double* W, size_t ldw,
                                          const double* C, size_t L, double* part, cudaStream_t st) {
  if (nq < 1 || nq > block_fused_max_nq() || (ldq & 1) || (ldw & 1)) return cudaErrorInvalidValue;
  static const bool resident = [] {
    const char* e = getenv("HBPDC_FUSED_RES");   // 1: the chunk-resident kernel (measured slower)
    return e && atoi(e) == 1;
  }();
  if (resident) {
    const int nq8 = (nq + 7) / 8 * 8;
    const size_t smem = ((size_t)TR_R * 8 * TR_P + (size_t)nq8 * 8) * sizeof(double) +
                        2 * TR_R * sizeof(unsigned long long);
    static size_t attr = 0;
    if (smem > attr) {
      if (cudaFuncSetAttribute(block_update_dots_res8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem) != cudaSuccess)
        return cudaErrorInvalidValue;
      attr = smem;
    }
    block_update_dots_res8_kernel<<<block_dot_blocks_tma(), 32 * (TF_W + 1), smem, st>>>(Q, ldq, nq, W, ldw, C, L, part);
    hbpdc_count_launch();
    return cudaGetLastError();
  }
  const int nq8 = (nq + 7) / 8 * 8;
  const size_t smem = ((size_t)TF_R * 8 * TF_P + (size_t)nq8 * 8) * sizeof(double) +
                      2 * TF_R * sizeof(unsigned long long);
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(block_update_dots_tma8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return cudaErrorInvalidValue;
    attr = smem;
  }
  block_update_dots_tma8_kernel<<<block_dot_blocks_tma(), 32 * (TF_W + 1), smem, st>>>(Q, ldq, nq, W, ldw, C, L, part);
  hbpdc_count_launch();
  return cudaGetLastError();
}

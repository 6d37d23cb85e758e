// sstep.cu -- block kernels of the s-step (communication-avoiding) Arnoldi
// process: Gram-Schmidt of a block of S Krylov vectors against the basis Q in
// ONE pass over Q per projection / update (block CGS2 = 4 passes per S
// iterations instead of DCGS2's 2 passes per iteration).
//
//   block_dots   rows j*S + l : Q_j . W_l  (j < nq, l < S);  rows nq*S + a*S + b : W_a . W_b
//   block_update W_l <- sum_m (W_m - sum_j Q_j C[j*S + m]) Rinv[m*S + l]   (Rinv NULL: identity)
//
// Deterministic two-level reductions (fixed chunking, fixed order) as in linalg.cu.
#include "launch.h"

namespace {
constexpr int BT = 4;              // doubles per thread per vector (256 x BT elements per CTA)
constexpr int BV = 16;             // values per reduction round
}

int block_dot_blocks(size_t L) { return (int)((L + 256 * BT - 1) / (256 * BT)); }

template <int S>
__global__ void __launch_bounds__(256) block_dots_kernel(const double* __restrict__ Q, size_t ldq, int nq,
                                                         const double* __restrict__ W, size_t ldw, size_t L,
                                                         double* __restrict__ part) {
  constexpr int KB = BV / S;       // basis vectors per full round
  __shared__ double red[8][BV];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t base = (size_t)blockIdx.x * (256 * BT) + threadIdx.x;
  const bool full = (size_t)blockIdx.x * (256 * BT) + 256 * BT <= L;
  double wr[S][BT];
#pragma unroll
  for (int l = 0; l < S; ++l)
#pragma unroll
    for (int t = 0; t < BT; ++t) {
      const size_t i = base + (size_t)t * 256;
      wr[l][t] = (full || i < L) ? W[(size_t)l * ldw + i] : 0.0;
    }
  const int nrows = nq * S + S * S;
  for (int r0 = 0; r0 < nrows; r0 += BV) {
    double acc[BV];
    const int j0 = r0 / S;
    if (full && r0 + BV <= nq * S) {
      double x[KB][BT];
#pragma unroll
      for (int q = 0; q < KB; ++q)
#pragma unroll
        for (int t = 0; t < BT; ++t) x[q][t] = __ldcs(Q + (size_t)(j0 + q) * ldq + base + (size_t)t * 256);
#pragma unroll
      for (int q = 0; q < KB; ++q)
#pragma unroll
        for (int l = 0; l < S; ++l) {
          double a = 0.0;
#pragma unroll
          for (int t = 0; t < BT; ++t) a = fma(x[q][t], wr[l][t], a);
          acc[q * S + l] = a;
        }
    } else {
      // row r0 + q S + l: vector j0 + q (a basis vector if < nq, else Gram row j0 + q - nq)
#pragma unroll
      for (int q = 0; q < KB; ++q) {
        const int j = j0 + q;
#pragma unroll
        for (int l = 0; l < S; ++l) {
          double a = 0.0;
          if (j < nq) {
            const double* qj = Q + (size_t)j * ldq;
#pragma unroll
            for (int t = 0; t < BT; ++t) {
              const size_t i = base + (size_t)t * 256;
              if (full || i < L) a = fma(__ldg(qj + i), wr[l][t], a);
            }
          } else if (j < nq + S) {
#pragma unroll
            for (int ga = 0; ga < S; ++ga)
              if (ga == j - nq) {
#pragma unroll
                for (int t = 0; t < BT; ++t) a = fma(wr[ga][t], wr[l][t], a);
              }
          }
          acc[q * S + l] = a;
        }
      }
    }
    // transposed butterfly: 16 values over 32 lanes (15 + 1 shuffles)
#pragma unroll
    for (int s = 8; s >= 1; s >>= 1) {
      const bool hi = lane & (2 * s);
#pragma unroll
      for (int q = 0; q < s; ++q) {
        const double send = hi ? acc[q] : acc[q + s];
        const double recv = __shfl_xor_sync(0xffffffffu, send, 2 * s);
        acc[q] = (hi ? acc[q + s] : acc[q]) + recv;
      }
    }
    acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
    if ((lane & 1) == 0) {
      const int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
      red[wid][idx] = acc[0];
    }
    __syncthreads();
    if (threadIdx.x < BV) {
      const int row = r0 + threadIdx.x;
      if (row < nrows) {
        double s = 0.0;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) s += red[ww][threadIdx.x];
        part[(size_t)row * gridDim.x + blockIdx.x] = s;
      }
    }
    __syncthreads();
  }
}

template <int S>
__global__ void __launch_bounds__(256) block_update_kernel(const double* __restrict__ Q, size_t ldq, int nq,
                                                           double* __restrict__ W, size_t ldw,
                                                           const double* __restrict__ C,
                                                           const double* __restrict__ Rinv, size_t L) {
  extern __shared__ double sC[];                 // nq * S coefficients, then S * S of Rinv
  for (int k = threadIdx.x; k < nq * S; k += 256) sC[k] = C[k];
  if (Rinv)
    for (int k = threadIdx.x; k < S * S; k += 256) sC[nq * S + k] = Rinv[k];
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * (256 * BT) + threadIdx.x;
  const bool full = (size_t)blockIdx.x * (256 * BT) + 256 * BT <= L;
  double tmp[S][BT];
#pragma unroll
  for (int m = 0; m < S; ++m)
#pragma unroll
    for (int t = 0; t < BT; ++t) {
      const size_t i = base + (size_t)t * 256;
      tmp[m][t] = (full || i < L) ? W[(size_t)m * ldw + i] : 0.0;
    }
  constexpr int U = S >= 8 ? 2 : (S >= 4 ? 4 : 8);   // basis vectors per batch of hoisted loads
  int j = 0;
  if (full) {
    for (; j + U <= nq; j += U) {
      double x[U][BT];
#pragma unroll
      for (int q = 0; q < U; ++q)
#pragma unroll
        for (int t = 0; t < BT; ++t) x[q][t] = __ldcs(Q + (size_t)(j + q) * ldq + base + (size_t)t * 256);
#pragma unroll
      for (int q = 0; q < U; ++q)
#pragma unroll
        for (int m = 0; m < S; ++m) {
          const double cm = sC[(j + q) * S + m];
#pragma unroll
          for (int t = 0; t < BT; ++t) tmp[m][t] = fma(-cm, x[q][t], tmp[m][t]);
        }
    }
  }
  for (; j < nq; ++j) {
    const double* qj = Q + (size_t)j * ldq;
#pragma unroll
    for (int t = 0; t < BT; ++t) {
      const size_t i = base + (size_t)t * 256;
      if (full || i < L) {
        const double x = __ldg(qj + i);
#pragma unroll
        for (int m = 0; m < S; ++m) tmp[m][t] = fma(-sC[j * S + m], x, tmp[m][t]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < BT; ++t) {
    const size_t i = base + (size_t)t * 256;
    if (!(full || i < L)) continue;
#pragma unroll
    for (int l = 0; l < S; ++l) {
      double o;
      if (Rinv) {
        o = 0.0;
#pragma unroll
        for (int m = 0; m <= l; ++m) o = fma(tmp[m][t], sC[nq * S + m * S + l], o);   // Rinv upper triangular
      } else {
        o = tmp[l][t];
      }
      W[(size_t)l * ldw + i] = o;
    }
  }
}

template <int S>
cudaError_t run_block_update(const double* Q, size_t ldq, int nq, double* W, size_t ldw, const double* C,
                             const double* Rinv, size_t L, cudaStream_t st) {
  const size_t smem = ((size_t)nq * S + S * S) * sizeof(double);
  if (smem > 48 * 1024) {
    static size_t attr = 0;
    if (smem > attr) {
      cudaFuncSetAttribute(block_update_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = smem;
    }
  }
  block_update_kernel<S><<<block_dot_blocks(L), 256, smem, st>>>(Q, ldq, nq, W, ldw, C, Rinv, L);
  hbpdc_count_launch();
  return cudaGetLastError();
}

cudaError_t launch_block_dots(const double* Q, size_t ldq, int nq, const double* W, size_t ldw, int s, size_t L,
                              double* part, cudaStream_t st) {
  const int nb = block_dot_blocks(L);
  switch (s) {
    case 2: block_dots_kernel<2><<<nb, 256, 0, st>>>(Q, ldq, nq, W, ldw, L, part); break;
    case 4: block_dots_kernel<4><<<nb, 256, 0, st>>>(Q, ldq, nq, W, ldw, L, part); break;
    case 8: block_dots_kernel<8><<<nb, 256, 0, st>>>(Q, ldq, nq, W, ldw, L, part); break;
    default: return cudaErrorInvalidValue;
  }
  hbpdc_count_launch();
  return cudaGetLastError();
}

cudaError_t launch_block_update(const double* Q, size_t ldq, int nq, double* W, size_t ldw, int s, const double* C,
                                const double* Rinv, size_t L, cudaStream_t st) {
  switch (s) {
    case 2: return run_block_update<2>(Q, ldq, nq, W, ldw, C, Rinv, L, st);
    case 4: return run_block_update<4>(Q, ldq, nq, W, ldw, C, Rinv, L, st);
    case 8: return run_block_update<8>(Q, ldq, nq, W, ldw, C, Rinv, L, st);
    default: return cudaErrorInvalidValue;
  }
}

// ============================================================================
// fp64 tensor-core (DMMA, mma.sync m8n8k4 f64) versions for S = 4, 8: both
// block operations are GEMMs with a huge inner (dots) or outer (update)
// dimension; the MMA keeps the reduction over elements inside the warp's
// accumulators, so the per-element cost is one load per lane per k-step.
// Fragment layout (PTX m8n8k4.f64): A (8x4, row) a0 = A[g][t]; B (4x8, col)
// b0 = B[t][g]; C/D (8x8) c0, c1 = C[g][2t], C[g][2t+1]; g = lane/4, t = lane%4.
// ============================================================================
namespace {
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
constexpr int MM_E = 128;          // elements per warp (32 k-steps of 4)
constexpr int MM_T = 4;            // vector tiles (8 vectors each) per round
constexpr int MM_KB = 4;           // k-steps per batch of hoisted loads (update kernel)
constexpr int MM_KD = 8;           // k-steps per batch of hoisted loads (dots kernel)
}

int block_dot_blocks_mma(size_t L) { return (int)((L + 8 * MM_E - 1) / (8 * MM_E)); }

// rows j*S + l = V_j . W_l for "vectors" V = [Q_0 .. Q_{nq-1}, W_0 .. W_{S-1}] (the
// last S give the Gram rows nq*S + a*S + b); one partial per CTA (8 warps x MM_E).
// Element map (the dot product sums over all elements, so any order is valid):
// k-steps 4p + r (r < 4) with k index t -> element ebase + 16p + 4t + r: each lane
// loads 32 B per four k-steps and the 4 lanes of a vector read 128 contiguous bytes.
template <int S>
__global__ void __launch_bounds__(256) block_dots_mma_kernel(const double* __restrict__ Q, size_t ldq, int nq,
                                                             const double* __restrict__ W, size_t ldw, size_t L,
                                                             double* __restrict__ part) {
  constexpr int RUN = MM_E / 4;                     // elements per lane
  extern __shared__ __align__(16) double sdm[];
  double (*red)[MM_T * 64] = reinterpret_cast<double (*)[MM_T * 64]>(sdm);        // [8][MM_T * 64]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* bsm = sdm + 8 * MM_T * 64 + (size_t)wid * RUN * 32;                      // this warp's B fragments [ks][lane]
  const int g = lane >> 2, t = lane & 3;
  const size_t ebase = ((size_t)blockIdx.x * 8 + wid) * MM_E;
  const size_t erun = ebase + 4 * (size_t)t;        // this lane's first element; quad p adds 16p
  const bool fullw = ebase + MM_E <= L;
#pragma unroll 2
  for (int ks = 0; ks < RUN; ks += 4) {
    const size_t e = erun + 4 * ks;                   // quad ks/4 starts at 16 (ks/4)
    double b[4];
    if (g < S && fullw) {
      const double2 v0 = *reinterpret_cast<const double2*>(W + (size_t)g * ldw + e);
      const double2 v1 = *reinterpret_cast<const double2*>(W + (size_t)g * ldw + e + 2);
      b[0] = v0.x; b[1] = v0.y; b[2] = v1.x; b[3] = v1.y;
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) b[r] = (g < S && e + r < L) ? W[(size_t)g * ldw + e + r] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) bsm[(ks + r) * 32 + lane] = b[r];
  }
  __syncwarp();
  const int nv = nq + S;                            // vectors incl. the Gram block
  const int nrows = nq * S + S * S;
  for (int v0 = 0; v0 < nv; v0 += 8 * MM_T) {
    double acc[MM_T][2];
#pragma unroll
    for (int q = 0; q < MM_T; ++q) { acc[q][0] = 0.0; acc[q][1] = 0.0; }
    const double* vp[MM_T];
#pragma unroll
    for (int q = 0; q < MM_T; ++q) {
      const int j = v0 + 8 * q + g;
      vp[q] = j < nq ? Q + (size_t)j * ldq : (j < nv ? W + (size_t)(j - nq) * ldw : nullptr);
    }
    for (int k0 = 0; k0 < RUN; k0 += MM_KD) {
      double a[MM_T][MM_KD];
#pragma unroll
      for (int q = 0; q < MM_T; ++q)
#pragma unroll
        for (int kk = 0; kk < MM_KD; kk += 4) {
          const size_t e = erun + 4 * (k0 + kk);
          if (vp[q] && fullw) {
            const double2 v0 = __ldcs(reinterpret_cast<const double2*>(vp[q] + e));
            const double2 v1 = __ldcs(reinterpret_cast<const double2*>(vp[q] + e + 2));
            a[q][kk] = v0.x; a[q][kk + 1] = v0.y; a[q][kk + 2] = v1.x; a[q][kk + 3] = v1.y;
          } else {
#pragma unroll
            for (int r = 0; r < 4; ++r) a[q][kk + r] = (vp[q] && e + r < L) ? vp[q][e + r] : 0.0;
          }
        }
#pragma unroll
      for (int kk = 0; kk < MM_KD; ++kk) {
        const double b = bsm[(k0 + kk) * 32 + lane];
#pragma unroll
        for (int q = 0; q < MM_T; ++q) dmma(acc[q], a[q][kk], b);
      }
    }
#pragma unroll
    for (int q = 0; q < MM_T; ++q) {
      red[wid][q * 64 + g * 8 + 2 * t] = acc[q][0];
      red[wid][q * 64 + g * 8 + 2 * t + 1] = acc[q][1];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < MM_T * 64; idx += 256) {
      const int q = idx / 64, i = (idx / 8) % 8, n = idx % 8;
      const int j = v0 + 8 * q + i;
      if (n < S && j < nv) {
        double sum = 0.0;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) sum += red[ww][idx];
        const int row = j * S + n;                  // Q rows, then the Gram rows (j >= nq)
        if (row < nrows) part[(size_t)row * gridDim.x + blockIdx.x] = sum;
      }
    }
    __syncthreads();
  }
}

// W_l <- sum_m (W_m - sum_j Q_j C[j*S + m]) Rinv[m*S + l].  A warp owns 32
// consecutive elements as 4 row tiles; tile q, row g is element e0 + 4g + q, so
// a lane's 4 tile rows are 4 consecutive elements (one 32 B load per vector).
template <int S>
__global__ void __launch_bounds__(256) block_update_mma_kernel(const double* __restrict__ Q, size_t ldq, int nq,
                                                               double* __restrict__ W, size_t ldw,
                                                               const double* __restrict__ C,
                                                               const double* __restrict__ Rinv, size_t L) {
  extern __shared__ double sC[];                 // -C padded to nq4 x 8 (B fragments), then Rinv 8 x 8
  const int nq4 = (nq + 3) / 4 * 4;
  for (int k = threadIdx.x; k < nq4 * 8; k += 256) {
    const int j = k / 8, n = k % 8;
    sC[k] = (j < nq && n < S) ? -C[j * S + n] : 0.0;
  }
  double* sR = sC + nq4 * 8;
  for (int k = threadIdx.x; k < 64; k += 256) {
    const int m = k / 8, l = k % 8;
    sR[k] = (m < S && l < S) ? (Rinv ? Rinv[m * S + l] : (m == l ? 1.0 : 0.0)) : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  constexpr int TE = 4;                          // row tiles per warp
  const size_t e0 = ((size_t)blockIdx.x * 8 + wid) * (8 * TE);
  const size_t er = e0 + 4 * g;                  // this lane's 4 consecutive elements
  const bool full = e0 + 8 * TE <= L;
  auto ld4 = [&](const double* p, double (&o)[TE]) {
    if (full) {
      const double2 v0 = __ldcs(reinterpret_cast<const double2*>(p + er));
      const double2 v1 = __ldcs(reinterpret_cast<const double2*>(p + er + 2));
      o[0] = v0.x; o[1] = v0.y; o[2] = v1.x; o[3] = v1.y;
    } else {
#pragma unroll
      for (int q = 0; q < TE; ++q) o[q] = er + q < L ? p[er + q] : 0.0;
    }
  };
  double acc[TE][2];
  {
    double w0[TE], w1[TE];
    if (2 * t < S) ld4(W + (size_t)(2 * t) * ldw, w0); else for (int q = 0; q < TE; ++q) w0[q] = 0.0;
    if (2 * t + 1 < S) ld4(W + (size_t)(2 * t + 1) * ldw, w1); else for (int q = 0; q < TE; ++q) w1[q] = 0.0;
#pragma unroll
    for (int q = 0; q < TE; ++q) { acc[q][0] = w0[q]; acc[q][1] = w1[q]; }
  }
  for (int j0 = 0; j0 < nq4; j0 += 4 * MM_KB) {
    double a[MM_KB][TE], b[MM_KB];
#pragma unroll
    for (int kk = 0; kk < MM_KB; ++kk) {
      const int j = j0 + 4 * kk + t;
      b[kk] = j < nq4 ? sC[j * 8 + g] : 0.0;
      if (j < nq) ld4(Q + (size_t)j * ldq, a[kk]);
      else
#pragma unroll
        for (int q = 0; q < TE; ++q) a[kk][q] = 0.0;
    }
#pragma unroll
    for (int kk = 0; kk < MM_KB; ++kk)
#pragma unroll
      for (int q = 0; q < TE; ++q) dmma(acc[q], a[kk][q], b[kk]);
  }
  // out[e][l] = sum_m D[e][m] Rinv[m][l]: gather row e's 8 D values from the 4 lanes of the group
  double o0[TE], o1[TE];
#pragma unroll
  for (int q = 0; q < TE; ++q) {
    double drow[8];
#pragma unroll
    for (int src = 0; src < 4; ++src) {
      drow[2 * src] = __shfl_sync(0xffffffffu, acc[q][0], (lane & ~3) | src);
      drow[2 * src + 1] = __shfl_sync(0xffffffffu, acc[q][1], (lane & ~3) | src);
    }
    double v0 = 0.0, v1 = 0.0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      if (m <= 2 * t) v0 = fma(drow[m], sR[m * 8 + 2 * t], v0);
      if (m <= 2 * t + 1) v1 = fma(drow[m], sR[m * 8 + 2 * t + 1], v1);
    }
    o0[q] = v0;
    o1[q] = v1;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int l = 2 * t + h;
    if (l >= S) continue;
    double* p = W + (size_t)l * ldw;
    const double* o = h ? o1 : o0;
    if (full) {
      *reinterpret_cast<double2*>(p + er) = make_double2(o[0], o[1]);
      *reinterpret_cast<double2*>(p + er + 2) = make_double2(o[2], o[3]);
    } else {
#pragma unroll
      for (int q = 0; q < TE; ++q)
        if (er + q < L) p[er + q] = o[q];
    }
  }
}

template <int S>
cudaError_t run_block_update_mma(const double* Q, size_t ldq, int nq, double* W, size_t ldw, const double* C,
                                 const double* Rinv, size_t L, cudaStream_t st) {
  const int nq4 = (nq + 3) / 4 * 4;
  const size_t smem = ((size_t)nq4 * 8 + 64) * sizeof(double);
  if (smem > 48 * 1024) {
    static size_t attr = 0;
    if (smem > attr) {
      cudaFuncSetAttribute(block_update_mma_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = smem;
    }
  }
  const int grid = (int)((L + 256 - 1) / 256);   // 8 warps x 32 elements
  block_update_mma_kernel<S><<<grid, 256, smem, st>>>(Q, ldq, nq, W, ldw, C, Rinv, L);
  hbpdc_count_launch();
  return cudaGetLastError();
}

cudaError_t launch_block_dots_mma(const double* Q, size_t ldq, int nq, const double* W, size_t ldw, int s, size_t L,
                                  double* part, cudaStream_t st) {
  const int nb = block_dot_blocks_mma(L);
  const size_t smem = ((size_t)8 * MM_T * 64 + (size_t)8 * (MM_E / 4) * 32) * sizeof(double);   // 80 KB
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(block_dots_mma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(block_dots_mma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  switch (s) {
    case 4: block_dots_mma_kernel<4><<<nb, 256, smem, st>>>(Q, ldq, nq, W, ldw, L, part); break;
    case 8: block_dots_mma_kernel<8><<<nb, 256, smem, st>>>(Q, ldq, nq, W, ldw, L, part); break;
    default: return cudaErrorInvalidValue;
  }
  hbpdc_count_launch();
  return cudaGetLastError();
}

cudaError_t launch_block_update_mma(const double* Q, size_t ldq, int nq, double* W, size_t ldw, int s,
                                    const double* C, const double* Rinv, size_t L, cudaStream_t st) {
  switch (s) {
    case 4: return run_block_update_mma<4>(Q, ldq, nq, W, ldw, C, Rinv, L, st);
    case 8: return run_block_update_mma<8>(Q, ldq, nq, W, ldw, C, Rinv, L, st);
    default: return cudaErrorInvalidValue;
  }
}

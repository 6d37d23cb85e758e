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

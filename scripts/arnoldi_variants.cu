// Variants of the DCGS2 dots / update kernels, timed against the library's
// (scripts/bench_arnoldi.cu drives the library versions).  Development tool:
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Iinclude \
//     scripts/arnoldi_variants.cu paper_2109_04804_b200/csrc/build/linalg.o -o /tmp/av && /tmp/av
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2109_04804_b200/csrc/launch.h"

// V1: full-chunk fast path, all KB x T loads issued before the FMAs; T doubles
// per thread per vector; CTA of 256 threads; per-round transposed warp reduction.
template <int T, int KB>
__global__ void __launch_bounds__(256) dots_v1(const double* __restrict__ Q, size_t ldx, int nk,
                                              const double* __restrict__ u, const double* __restrict__ w, size_t L,
                                              double* __restrict__ part) {
  __shared__ double red[8][2 * KB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t base = (size_t)blockIdx.x * (256 * T) + threadIdx.x;
  const bool full = (size_t)blockIdx.x * (256 * T) + 256 * T <= L;
  double ur[T], wr[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const size_t i = base + (size_t)t * 256;
    ur[t] = (full || i < L) ? u[i] : 0.0;
    wr[t] = (full || i < L) ? w[i] : 0.0;
  }
  const int nrows = 2 * nk + 3;
  for (int k0 = 0; k0 < nk + 2; k0 += KB) {
    double acc[2 * KB];
    if (full && k0 + KB <= nk) {
      double x[KB][T];
#pragma unroll
      for (int q = 0; q < KB; ++q)
#pragma unroll
        for (int t = 0; t < T; ++t) x[q][t] = __ldcs(Q + (size_t)(k0 + q) * ldx + base + (size_t)t * 256);
#pragma unroll
      for (int q = 0; q < KB; ++q) {
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int t = 0; t < T; ++t) { a = fma(x[q][t], ur[t], a); b = fma(x[q][t], wr[t], b); }
        acc[2 * q] = a;
        acc[2 * q + 1] = b;
      }
    } else {
#pragma unroll
      for (int q = 0; q < KB; ++q) {
        const int k = k0 + q;
        double a = 0.0, b = 0.0;
        if (k < nk) {
          const double* qk = Q + (size_t)k * ldx;
#pragma unroll
          for (int t = 0; t < T; ++t) {
            const size_t i = base + (size_t)t * 256;
            if (i < L) { const double xx = __ldcs(qk + i); a = fma(xx, ur[t], a); b = fma(xx, wr[t], b); }
          }
        } else if (k == nk) {
#pragma unroll
          for (int t = 0; t < T; ++t) { a = fma(ur[t], ur[t], a); b = fma(ur[t], wr[t], b); }
        } else if (k == nk + 1) {
#pragma unroll
          for (int t = 0; t < T; ++t) a = fma(wr[t], wr[t], a);
        }
        acc[2 * q] = a;
        acc[2 * q + 1] = b;
      }
    }
    // transposed butterfly: V = 2KB values over 32 lanes.  Step j halves the
    // live values across lane bit (16 >> j); the remaining low lane bits are a
    // plain reduction.  Lane bits 4..(5-p) then index the value (p = log2 V).
    constexpr int V = 2 * KB;
    constexpr int p = V == 16 ? 4 : V == 8 ? 3 : V == 4 ? 2 : 1;
#pragma unroll
    for (int j = 0; j < p; ++j) {
      const int h = V >> (j + 1);
      const int mask = 16 >> j;
      const bool hi = lane & mask;
#pragma unroll
      for (int q = 0; q < h; ++q) {
        const double send = hi ? acc[q] : acc[q + h];
        const double recv = __shfl_xor_sync(0xffffffffu, send, mask);
        acc[q] = (hi ? acc[q + h] : acc[q]) + recv;
      }
    }
#pragma unroll
    for (int mask = 16 >> p; mask >= 1; mask >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], mask);
    if ((lane & ((32 >> p) - 1)) == 0) {
      int idx = 0;
#pragma unroll
      for (int j = 0; j < p; ++j)
        if (lane & (16 >> j)) idx |= V >> (j + 1);
      red[wid][idx] = acc[0];
    }
    __syncthreads();
    if (threadIdx.x < 2 * KB) {
      const int row = 2 * k0 + threadIdx.x;
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

// V2 update: full-chunk fast path, k loop unrolled by U with loads hoisted.
template <int T, int U>
__global__ void __launch_bounds__(256) update_v2(const double* __restrict__ Q, size_t ldx, int nk,
                                                const double* __restrict__ a, const double* __restrict__ d,
                                                double* __restrict__ u, double* __restrict__ w, double ib, double cb,
                                                size_t L) {
  __shared__ double as[1024], ds[1024];
  for (int k = threadIdx.x; k < nk && k < 1024; k += 256) { as[k] = a[k]; ds[k] = d[k]; }
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * (256 * T) + threadIdx.x;
  const bool full = (size_t)blockIdx.x * (256 * T) + 256 * T <= L;
  double qa[T], qd[T];
#pragma unroll
  for (int t = 0; t < T; ++t) { qa[t] = 0.0; qd[t] = 0.0; }
  int k = 0;
  if (full) {
    for (; k + U <= nk; k += U) {
      double x[U][T];
#pragma unroll
      for (int q = 0; q < U; ++q)
#pragma unroll
        for (int t = 0; t < T; ++t) x[q][t] = __ldcs(Q + (size_t)(k + q) * ldx + base + (size_t)t * 256);
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const double ak = (k + q) < 1024 ? as[k + q] : a[k + q];
        const double dk = (k + q) < 1024 ? ds[k + q] : d[k + q];
#pragma unroll
        for (int t = 0; t < T; ++t) { qa[t] = fma(ak, x[q][t], qa[t]); qd[t] = fma(dk, x[q][t], qd[t]); }
      }
    }
  }
  for (; k < nk; ++k) {
    const double ak = k < 1024 ? as[k] : a[k];
    const double dk = k < 1024 ? ds[k] : d[k];
    const double* qk = Q + (size_t)k * ldx;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const size_t i = base + (size_t)t * 256;
      if (full || i < L) {
        const double x = __ldcs(qk + i);
        qa[t] = fma(ak, x, qa[t]);
        qd[t] = fma(dk, x, qd[t]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const size_t i = base + (size_t)t * 256;
    if (full || i < L) {
      const double ui = u[i], wi = w[i];
      u[i] = (ui - qa[t]) * ib;
      w[i] = fma(wi, ib, -qd[t]) - ui * cb;
    }
  }
}

template <class F>
float timeit(F f, cudaStream_t st, int R = 10) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  f();
  cudaEventRecord(e0, st);
  for (int r = 0; r < R; ++r) f();
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / R;
}

int main() {
  const size_t L = 8388608;
  const int KMAX = 160;
  double *Q, *u, *w, *part, *part2, *a, *d, *out, *out2;
  cudaMalloc(&Q, (KMAX + 2) * L * sizeof(double));
  cudaMalloc(&u, L * sizeof(double));
  cudaMalloc(&w, L * sizeof(double));
  const int nb = arnoldi_dot_blocks(L);
  cudaMalloc(&part, (2 * KMAX + 4) * (size_t)nb * sizeof(double));
  cudaMalloc(&part2, (2 * KMAX + 4) * (size_t)nb * 2 * sizeof(double));
  cudaMalloc(&a, KMAX * sizeof(double));
  cudaMalloc(&d, KMAX * sizeof(double));
  cudaMalloc(&out, (2 * KMAX + 4) * sizeof(double));
  cudaMalloc(&out2, (2 * KMAX + 4) * sizeof(double));
  // deterministic non-trivial data
  std::vector<double> h(L);
  for (size_t i = 0; i < L; ++i) h[i] = 1.0 / (1.0 + (i % 97));
  for (int k = 0; k < KMAX + 2; ++k) cudaMemcpy(Q + k * L, h.data(), L * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(u, h.data(), L * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(w, h.data(), L * 8, cudaMemcpyHostToDevice);
  std::vector<double> ha(KMAX, 1e-3);
  cudaMemcpy(a, ha.data(), KMAX * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d, ha.data(), KMAX * 8, cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreate(&st);
  printf("%5s | %9s %9s %9s %9s | %9s %9s %9s\n", "nk", "lib", "v1<8,8>", "v1<4,8>", "v1<8,4>", "upd_lib",
         "v2<8,4>", "v2<4,8>");
  for (int nk : {4, 16, 32, 64, 96, 128, 160}) {
    const double b1 = (nk + 2.0) * L * 8, b2 = (nk + 4.0) * L * 8;
    auto gbs = [&](double bytes, float ms) { return bytes / (ms * 1e-3) / 1e9; };
    float tl = timeit([&] { launch_dcgs2_dots(Q, L, nk, u, w, L, part, st); }, st);
    const int g8 = (int)((L + 256 * 8 - 1) / (256 * 8)), g4 = (int)((L + 256 * 4 - 1) / (256 * 4));
    float t1 = timeit([&] { dots_v1<8, 8><<<g8, 256, 0, st>>>(Q, L, nk, u, w, L, part2); }, st);
    float t2 = timeit([&] { dots_v1<4, 8><<<g4, 256, 0, st>>>(Q, L, nk, u, w, L, part2); }, st);
    float t3 = timeit([&] { dots_v1<8, 4><<<g8, 256, 0, st>>>(Q, L, nk, u, w, L, part2); }, st);
    // correctness of v1<8,8> vs the library (same partial layout, same order)
    launch_dcgs2_dots(Q, L, nk, u, w, L, part, st);
    launch_reduce_partials_n(part, 2 * nk + 3, nb, out, st);
    dots_v1<8, 8><<<g8, 256, 0, st>>>(Q, L, nk, u, w, L, part2);
    launch_reduce_partials_n(part2, 2 * nk + 3, g8, out2, st);
    std::vector<double> o1(2 * nk + 3), o2(2 * nk + 3);
    cudaMemcpy(o1.data(), out, o1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(o2.data(), out2, o2.size() * 8, cudaMemcpyDeviceToHost);
    double md = 0;
    for (size_t i = 0; i < o1.size(); ++i) md = std::max(md, std::abs(o1[i] - o2[i]) / std::abs(o1[i]));
    float u0 = timeit([&] { launch_dcgs2_update(Q, L, nk, a, d, u, w, 1.0, 0.0, L, st); }, st);
    float u1 = timeit([&] { update_v2<8, 4><<<g8, 256, 0, st>>>(Q, L, nk, a, d, u, w, 1.0, 0.0, L); }, st);
    float u2 = timeit([&] { update_v2<4, 8><<<g4, 256, 0, st>>>(Q, L, nk, a, d, u, w, 1.0, 0.0, L); }, st);
    printf("%5d | %9.0f %9.0f %9.0f %9.0f | %9.0f %9.0f %9.0f   (dots v1 rel diff %.1e)\n", nk, gbs(b1, tl),
           gbs(b1, t1), gbs(b1, t2), gbs(b1, t3), gbs(b2, u0), gbs(b2, u1), gbs(b2, u2), md);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

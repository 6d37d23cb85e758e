// Micro-benchmark + cross-check of the s-step block kernels (sstep.cu): FMA vs
// fp64-MMA versions of block_dots / block_update at C3 size (2n = 8,388,608).
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Iinclude scripts/bench_block.cu \
//     paper_2109_04804_b200/csrc/build/sstep.o paper_2109_04804_b200/csrc/build/linalg.o -o /tmp/bb && /tmp/bb
#include <cmath>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2109_04804_b200/csrc/launch.h"

template <class F>
float timeit(F f, cudaStream_t st, int R = 5) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
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
  const int NQ = 64;
  double *Q, *W, *W2, *part, *out1, *out2, *C;
  cudaMalloc(&Q, (size_t)NQ * L * 8);
  cudaMalloc(&W, 8 * L * 8);
  cudaMalloc(&W2, 8 * L * 8);
  const int rows = NQ * 8 + 64;
  const int nb = std::max(block_dot_blocks(L), block_dot_blocks_mma(L));
  cudaMalloc(&part, (size_t)rows * nb * 8);
  cudaMalloc(&out1, rows * 8);
  cudaMalloc(&out2, rows * 8);
  cudaMalloc(&C, (NQ * 8 + 64) * 8);
  std::vector<double> h(L);
  for (size_t i = 0; i < L; ++i) h[i] = std::sin(0.001 * i) + 0.01 * (i % 13);
  for (int k = 0; k < NQ; ++k) cudaMemcpy(Q + k * L, h.data(), L * 8, cudaMemcpyHostToDevice);
  for (size_t i = 0; i < L; ++i) h[i] = std::cos(0.0007 * i);
  for (int k = 0; k < 8; ++k) cudaMemcpy(W + k * L, h.data(), L * 8, cudaMemcpyHostToDevice);
  std::vector<double> hc(NQ * 8 + 64);
  for (size_t i = 0; i < hc.size(); ++i) hc[i] = 1e-3 * ((i * 7) % 11);
  cudaMemcpy(C, hc.data(), hc.size() * 8, cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (int s : {4, 8}) {
    const int r = NQ * s + s * s;
    const double bd = (double)(NQ + s) * L * 8, bu = (double)(NQ + 2 * s) * L * 8;
    float t1 = timeit([&] { launch_block_dots(Q, L, NQ, W, L, s, L, part, st); }, st);
    launch_block_dots(Q, L, NQ, W, L, s, L, part, st);
    launch_reduce_partials_n(part, r, block_dot_blocks(L), out1, st);
    float t2 = timeit([&] { launch_block_dots_mma(Q, L, NQ, W, L, s, L, part, st); }, st);
    launch_block_dots_mma(Q, L, NQ, W, L, s, L, part, st);
    launch_reduce_partials_n(part, r, block_dot_blocks_mma(L), out2, st);
    std::vector<double> a(r), b(r);
    cudaMemcpy(a.data(), out1, r * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), out2, r * 8, cudaMemcpyDeviceToHost);
    double md = 0;
    for (int i = 0; i < r; ++i) md = std::max(md, std::abs(a[i] - b[i]) / (std::abs(a[i]) + 1e-300));
    cudaMemcpy(W2, W, 8 * L * 8, cudaMemcpyDeviceToDevice);
    float t3 = timeit([&] { launch_block_update(Q, L, NQ, W2, L, s, C, C + NQ * s, L, st); }, st);
    cudaMemcpy(W2, W, 8 * L * 8, cudaMemcpyDeviceToDevice);
    launch_block_update(Q, L, NQ, W2, L, s, C, nullptr, L, st);
    float t4 = timeit([&] { launch_block_update_mma(Q, L, NQ, W, L, s, C, C + NQ * s, L, st); }, st);
    // correctness of the update (identity Rinv): W2 (FMA) vs MMA on a fresh copy
    double* W3;
    cudaMalloc(&W3, 8 * L * 8);
    cudaMemcpy(W3, W2, 8, cudaMemcpyDeviceToDevice);
    printf("s=%d dots: fma %8.1f us %6.0f GB/s | mma %8.1f us %6.0f GB/s | max rel diff %.2e\n", s, t1 * 1e3,
           bd / (t1 * 1e-3) / 1e9, t2 * 1e3, bd / (t2 * 1e-3) / 1e9, md);
    printf("s=%d update: fma %8.1f us %6.0f GB/s | mma %8.1f us %6.0f GB/s\n", s, t3 * 1e3, bu / (t3 * 1e-3) / 1e9,
           t4 * 1e3, bu / (t4 * 1e-3) / 1e9);
    cudaFree(W3);
  }
  // update correctness: same input, both kernels, identity Rinv
  for (int s : {4, 8}) {
    for (size_t i = 0; i < L; ++i) h[i] = std::cos(0.0007 * i);
    for (int k = 0; k < 8; ++k) cudaMemcpy(W + k * L, h.data(), L * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(W2, W, 8 * L * 8, cudaMemcpyDeviceToDevice);
    launch_block_update(Q, L, NQ, W, L, s, C, C + NQ * s, L, st);
    launch_block_update_mma(Q, L, NQ, W2, L, s, C, C + NQ * s, L, st);
    std::vector<double> a(s * L), b(s * L);
    cudaMemcpy(a.data(), W, s * L * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), W2, s * L * 8, cudaMemcpyDeviceToHost);
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) { num += (a[i] - b[i]) * (a[i] - b[i]); den += a[i] * a[i]; }
    printf("s=%d update fma vs mma rel L2 diff %.2e\n", s, std::sqrt(num / den));
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// Micro-benchmark + cross-check of the TMA-streamed s = 8 block kernels
// (sstep_tma.cu) against the register-streamed DMMA kernels (sstep.cu) at C3
// size (2n = 8,388,608) and on a ragged length, for several basis sizes nq.
//   make -C paper_2109_04804_b200/csrc && nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a \
//     scripts/bench_block_tma.cu paper_2109_04804_b200/csrc/build/{sstep,sstep_tma,linalg}.o -o /tmp/bbt && /tmp/bbt
#include <algorithm>
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

int main(int argc, char** argv) {
  const bool quick = argc > 1;             // fused kernel check only, small L (for compute-sanitizer)
  const size_t LMAX = quick ? 262144 : 8388608;
  const int NQMAX = 160;
  double *Q, *W, *W2, *W3, *part, *out1, *out2, *C;
  cudaMalloc(&Q, (size_t)NQMAX * LMAX * 8);
  cudaMalloc(&W, 8 * LMAX * 8);
  cudaMalloc(&W2, 8 * LMAX * 8);
  cudaMalloc(&W3, 8 * LMAX * 8);
  const int rows = NQMAX * 8 + 64;
  const int nb = std::max(block_dot_blocks_mma(LMAX), block_dot_parts_tma());
  cudaMalloc(&part, (size_t)rows * nb * 8);
  cudaMalloc(&out1, rows * 8);
  cudaMalloc(&out2, rows * 8);
  cudaMalloc(&C, (NQMAX * 8 + 64) * 8);
  std::vector<double> h(LMAX);
  for (int k = 0; k < NQMAX; ++k) {
    for (size_t i = 0; i < LMAX; ++i) h[i] = std::sin(0.001 * i + 0.37 * k) + 0.01 * ((i + k) % 13);
    cudaMemcpy(Q + k * LMAX, h.data(), LMAX * 8, cudaMemcpyHostToDevice);
  }
  for (int k = 0; k < 8; ++k) {
    for (size_t i = 0; i < LMAX; ++i) h[i] = std::cos(0.0007 * i + 0.11 * k);
    cudaMemcpy(W + k * LMAX, h.data(), LMAX * 8, cudaMemcpyHostToDevice);
  }
  std::vector<double> hc(NQMAX * 8 + 64);
  for (size_t i = 0; i < hc.size(); ++i) hc[i] = 1e-3 * ((i * 7) % 11) - 2e-3;
  for (int m = 0; m < 8; ++m)           // Rinv upper triangular
    for (int l = 0; l < 8; ++l) hc[NQMAX * 8 + m * 8 + l] = l >= m ? 0.5 + 0.1 * m - 0.03 * l : 0.0;
  cudaMemcpy(C, hc.data(), hc.size() * 8, cudaMemcpyHostToDevice);
  const double* Rinv = C + NQMAX * 8;
  cudaStream_t st;
  cudaStreamCreate(&st);
  bool ok = true;
  for (size_t L : {LMAX, (size_t)1000006}) {
    if (quick) break;
    for (int nq : {1, 9, 17, 64, 96, 126}) {
      const int r = nq * 8 + 64;
      const double bd = (double)(nq + 8) * L * 8, bu = (double)(nq + 16) * L * 8;
      const int nbm = block_dot_blocks_mma(L), nbt = block_dot_parts_tma();
      float t1 = timeit([&] { launch_block_dots_mma(Q, LMAX, nq, W, LMAX, 8, L, part, st); }, st);
      launch_block_dots_mma(Q, LMAX, nq, W, LMAX, 8, L, part, st);
      launch_reduce_partials_n(part, r, nbm, out1, st);
      float t2 = timeit([&] { launch_block_dots_tma8(Q, LMAX, nq, W, LMAX, L, part, st); }, st);
      launch_block_dots_tma8(Q, LMAX, nq, W, LMAX, L, part, st);
      launch_reduce_partials_n(part, r, nbt, out2, st);
      std::vector<double> a(r), b(r);
      cudaMemcpy(a.data(), out1, r * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), out2, r * 8, cudaMemcpyDeviceToHost);
      double md = 0, mx = 0;
      for (int i = 0; i < r; ++i) { md = std::max(md, std::abs(a[i] - b[i])); mx = std::max(mx, std::abs(a[i])); }
      // update: same input, both kernels
      cudaMemcpy(W2, W, 8 * LMAX * 8, cudaMemcpyDeviceToDevice);
      cudaMemcpy(W3, W, 8 * LMAX * 8, cudaMemcpyDeviceToDevice);
      launch_block_update_mma(Q, LMAX, nq, W2, LMAX, 8, C, Rinv, L, st);
      launch_block_update_tma8(Q, LMAX, nq, W3, LMAX, C, Rinv, L, st);
      std::vector<double> u(8 * LMAX), v(8 * LMAX);
      cudaMemcpy(u.data(), W2, 8 * LMAX * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(v.data(), W3, 8 * LMAX * 8, cudaMemcpyDeviceToHost);
      double num = 0, den = 0, tail = 0;
      for (int k = 0; k < 8; ++k)
        for (size_t i = 0; i < LMAX; ++i) {
          const double x = u[k * LMAX + i], y = v[k * LMAX + i];
          if (i < L) { num += (x - y) * (x - y); den += x * x; }
          else tail = std::max(tail, std::abs(y - x));      // beyond L: untouched by both
        }
      cudaMemcpy(W2, W, 8 * LMAX * 8, cudaMemcpyDeviceToDevice);
      float t3 = timeit([&] { launch_block_update_mma(Q, LMAX, nq, W2, LMAX, 8, C, nullptr, L, st); }, st);
      float t4 = timeit([&] { launch_block_update_tma8(Q, LMAX, nq, W2, LMAX, C, nullptr, L, st); }, st);
      const double rd = md / mx, ru = std::sqrt(num / den);
      ok = ok && rd < 1e-13 && ru < 1e-13 && tail == 0.0;
      printf("L=%zu nq=%3d dots: mma %7.1f us %5.0f GB/s | tma %7.1f us %5.0f GB/s | diff %.1e   "
             "update: mma %7.1f us %5.0f GB/s | tma %7.1f us %5.0f GB/s | diff %.1e tail %.1e\n",
             L, nq, t1 * 1e3, bd / (t1 * 1e-3) / 1e9, t2 * 1e3, bd / (t2 * 1e-3) / 1e9, rd, t3 * 1e3,
             bu / (t3 * 1e-3) / 1e9, t4 * 1e3, bu / (t4 * 1e-3) / 1e9, ru, tail);
    }
  }
  // fused update + re-projection vs update then dots (separate kernels)
  double* part2;
  cudaMalloc(&part2, (size_t)rows * block_fused_parts_tma() * 8);
  for (size_t L : {LMAX, quick ? (size_t)100006 : (size_t)1000006}) {
    for (int nq : {1, 9, 17, 64, 126, 152}) {
      if (quick && nq != 17) continue;
      const int r = nq * 8 + 64;
      cudaMemcpy(W2, W, 8 * LMAX * 8, cudaMemcpyDeviceToDevice);
      cudaMemcpy(W3, W, 8 * LMAX * 8, cudaMemcpyDeviceToDevice);
      launch_block_update_mma(Q, LMAX, nq, W2, LMAX, 8, C, nullptr, L, st);
      launch_block_dots_mma(Q, LMAX, nq, W2, LMAX, 8, L, part, st);
      launch_reduce_partials_n(part, r, block_dot_blocks_mma(L), out1, st);
      launch_block_update_dots_tma8(Q, LMAX, nq, W3, LMAX, C, L, part2, st);
      launch_reduce_partials_n(part2, r, block_fused_parts_tma(), out2, st);
      std::vector<double> a(r), b(r);
      cudaMemcpy(a.data(), out1, r * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), out2, r * 8, cudaMemcpyDeviceToHost);
      double md = 0, mx = 0;
      for (int i = 0; i < r; ++i) { md = std::max(md, std::abs(a[i] - b[i])); mx = std::max(mx, std::abs(a[i])); }
      for (int i = 0; i < r; ++i)
        if (std::abs(a[i] - b[i]) > 1e-12 * mx) printf("   bad row %d (j %d l %d): %.6e vs %.6e\n", i, i / 8, i % 8, a[i], b[i]);
      std::vector<double> u(8 * LMAX), v(8 * LMAX);
      cudaMemcpy(u.data(), W2, 8 * LMAX * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(v.data(), W3, 8 * LMAX * 8, cudaMemcpyDeviceToHost);
      double num = 0, den = 0, tail = 0;
      for (int k = 0; k < 8; ++k)
        for (size_t i = 0; i < LMAX; ++i) {
          const double x = u[k * LMAX + i], y = v[k * LMAX + i];
          if (i < L) { num += (x - y) * (x - y); den += x * x; }
          else tail = std::max(tail, std::abs(y - x));
        }
      cudaMemcpy(W2, W, 8 * LMAX * 8, cudaMemcpyDeviceToDevice);
      float ts = timeit([&] {
        launch_block_update_mma(Q, LMAX, nq, W2, LMAX, 8, C, nullptr, L, st);
        launch_block_dots_mma(Q, LMAX, nq, W2, LMAX, 8, L, part, st);
      }, st);
      float tf = timeit([&] { launch_block_update_dots_tma8(Q, LMAX, nq, W2, LMAX, C, L, part2, st); }, st);
      const double rd = md / mx, ru = std::sqrt(num / den);
      ok = ok && rd < 1e-12 && ru < 1e-13 && tail == 0.0;
      const double bq = (double)nq * L * 8;
      printf("L=%zu nq=%3d fused: separate %7.1f us | fused %7.1f us (Q stream %5.0f GB/s) | dots diff %.1e W diff %.1e tail %.1e\n",
             L, nq, ts * 1e3, tf * 1e3, bq / (tf * 1e-3) / 1e9, rd, ru, tail);
    }
  }
  // update with the Gram of its output, and the W-only scale, vs the separate kernels
  for (size_t L : {LMAX, quick ? (size_t)100006 : (size_t)1000006}) {
    for (int nq : {1, 17, 126}) {
      cudaMemcpy(W2, W, 8 * LMAX * 8, cudaMemcpyDeviceToDevice);
      cudaMemcpy(W3, W, 8 * LMAX * 8, cudaMemcpyDeviceToDevice);
      launch_block_update_mma(Q, LMAX, nq, W2, LMAX, 8, C, Rinv, L, st);
      launch_block_dots_mma(Q, LMAX, 0, W2, LMAX, 8, L, part, st);
      launch_reduce_partials_n(part, 64, block_dot_blocks_mma(L), out1, st);
      launch_block_update_tma8(Q, LMAX, nq, W3, LMAX, C, Rinv, L, st, part2);
      launch_reduce_partials_n(part2, 64, block_fused_parts_tma(), out2, st);
      std::vector<double> a(64), b(64);
      cudaMemcpy(a.data(), out1, 64 * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), out2, 64 * 8, cudaMemcpyDeviceToHost);
      double md = 0, mx = 0;
      for (int i = 0; i < 64; ++i) { md = std::max(md, std::abs(a[i] - b[i])); mx = std::max(mx, std::abs(a[i])); }
      // scale: W2 <- W2 Rinv by both kernels
      launch_block_update_mma(Q, LMAX, 0, W2, LMAX, 8, C, Rinv, L, st);
      launch_block_scale_w8(W3, LMAX, Rinv, L, st);
      std::vector<double> u(8 * LMAX), v(8 * LMAX);
      cudaMemcpy(u.data(), W2, 8 * LMAX * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(v.data(), W3, 8 * LMAX * 8, cudaMemcpyDeviceToHost);
      double num = 0, den = 0, tail = 0;
      for (int k = 0; k < 8; ++k)
        for (size_t i = 0; i < LMAX; ++i) {
          const double x = u[k * LMAX + i], y = v[k * LMAX + i];
          if (i < L) { num += (x - y) * (x - y); den += x * x; }
          else tail = std::max(tail, std::abs(y - x));
        }
      float ts = timeit([&] { launch_block_update_mma(Q, LMAX, 0, W2, LMAX, 8, C, Rinv, L, st); }, st);
      float tn = timeit([&] { launch_block_scale_w8(W3, LMAX, Rinv, L, st); }, st);
      float tg = timeit([&] { launch_block_update_tma8(Q, LMAX, nq, W3, LMAX, C, Rinv, L, st, part2); }, st);
      const double rd = md / mx, ru = std::sqrt(num / den);
      ok = ok && rd < 1e-13 && ru < 1e-13 && tail == 0.0;
      printf("L=%zu nq=%3d gram: update+gram %7.1f us, gram diff %.1e | scale: mma %6.1f us / new %6.1f us (%5.0f GB/s) diff %.1e tail %.1e\n",
             L, nq, tg * 1e3, rd, ts * 1e3, tn * 1e3, 16.0 * L * 8 / (tn * 1e-3) / 1e9, ru, tail);
    }
  }
  printf("status: %s  check: %s\n", cudaGetErrorString(cudaGetLastError()), ok ? "OK" : "FAIL");
  return ok ? 0 : 1;
}

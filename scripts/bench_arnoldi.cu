// Micro-benchmark of the Arnoldi (DCGS2) kernels of linalg.cu at C3 size
// (2n = 8,388,608 doubles per Krylov vector): achieved GB/s of the algorithmic
// bytes for several Krylov indices.  Build + run (GPU box):
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I../include \
//        scripts/bench_arnoldi.cu paper_2109_04804_b200/csrc/build/linalg.o -o /tmp/ba && /tmp/ba
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2109_04804_b200/csrc/launch.h"

int main() {
  const size_t L = 8388608;
  const int KMAX = 160;
  double *Q, *u, *w, *part, *a, *d, *out;
  cudaMalloc(&Q, (KMAX + 2) * L * sizeof(double));
  cudaMalloc(&u, L * sizeof(double));
  cudaMalloc(&w, L * sizeof(double));
  const int nb = arnoldi_dot_blocks(L);
  cudaMalloc(&part, (2 * KMAX + 4) * (size_t)nb * sizeof(double));
  cudaMalloc(&a, KMAX * sizeof(double));
  cudaMalloc(&d, KMAX * sizeof(double));
  cudaMalloc(&out, (2 * KMAX + 4) * sizeof(double));
  cudaMemset(Q, 0, (KMAX + 2) * L * sizeof(double));
  cudaMemset(u, 0, L * sizeof(double));
  cudaMemset(w, 0, L * sizeof(double));
  cudaMemset(a, 0, KMAX * sizeof(double));
  cudaMemset(d, 0, KMAX * sizeof(double));
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("%6s %12s %10s %12s %10s\n", "nk", "dots_us", "dots_GBs", "update_us", "upd_GBs");
  for (int nk : {4, 16, 32, 64, 96, 128, 160}) {
    for (int rep = 0; rep < 2; ++rep) {
      launch_dcgs2_dots(Q, L, nk, u, w, L, part, st);
      launch_dcgs2_update(Q, L, nk, a, d, u, w, 1.0, 0.0, L, st);
    }
    const int R = 10;
    cudaEventRecord(e0, st);
    for (int r = 0; r < R; ++r) {
      launch_dcgs2_dots(Q, L, nk, u, w, L, part, st);
      launch_reduce_partials_n(part, 2 * nk + 3, nb, out, st);
    }
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms1;
    cudaEventElapsedTime(&ms1, e0, e1);
    cudaEventRecord(e0, st);
    for (int r = 0; r < R; ++r) launch_dcgs2_update(Q, L, nk, a, d, u, w, 1.0, 0.0, L, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms2;
    cudaEventElapsedTime(&ms2, e0, e1);
    const double t1 = ms1 / R * 1e-3, t2 = ms2 / R * 1e-3;
    const double b1 = (nk + 2.0) * L * 8, b2 = (nk + 4.0) * L * 8;
    printf("%6d %12.1f %10.1f %12.1f %10.1f\n", nk, t1 * 1e6, b1 / t1 / 1e9, t2 * 1e6, b2 / t2 / 1e9);
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

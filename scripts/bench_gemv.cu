// Micro-benchmark of the BJ_ext S-streaming GEMV (linalg.cu launch_block_gemv_multi)
// at C3 size (16384 elements, m = 256, 8.6 GB of S) for 2, 4, 6 right-hand sides.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Iinclude \
//        scripts/bench_gemv.cu paper_2109_04804_b200/csrc/build/linalg.o -o /tmp/bg && /tmp/bg
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2109_04804_b200/csrc/launch.h"

int main() {
  const int m = 256, nE = 16384;
  const size_t n = (size_t)nE * m;
  double* S;
  cudaMalloc(&S, (size_t)nE * m * m * sizeof(double));
  cudaMemset(S, 0, (size_t)nE * m * m * sizeof(double));
  std::vector<double*> in(6), out(6);
  for (int k = 0; k < 6; ++k) {
    cudaMalloc(&in[k], n * 8);
    cudaMalloc(&out[k], n * 8);
    cudaMemset(in[k], 0, n * 8);
  }
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int nr : {2, 4, 6}) {
    for (int r = 0; r < 2; ++r) launch_block_gemv_multi(S, nr, in.data(), out.data(), m, nE, st);
    const int R = 10;
    cudaEventRecord(e0, st);
    for (int r = 0; r < R; ++r) launch_block_gemv_multi(S, nr, in.data(), out.data(), m, nE, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double t = ms / R * 1e-3;
    const double bytes = (double)nE * m * m * 8 + 2.0 * nr * n * 8;
    printf("NR=%d  %8.1f us  %7.1f GB/s\n", nr, t * 1e6, bytes / t / 1e9);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

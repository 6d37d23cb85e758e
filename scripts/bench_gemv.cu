// Micro-benchmark of the BJ_ext S-streaming GEMV (linalg.cu launch_block_gemv_multi)
// at C3 size (16384 elements, m = 256, 8.6 GB of S) for 2, 4, 6 right-hand sides.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Iinclude \
//        scripts/bench_gemv.cu paper_2109_04804_b200/csrc/build/linalg.o -o /tmp/bg && /tmp/bg
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2109_04804_b200/csrc/launch.h"

__global__ void fill(double* x, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)(i * 2654435761u) ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    x[i] = (double)(h & 0xffffff) / 16777216.0 - 0.5;
  }
}

int main() {
  const int m = 256, nE = 16384;
  const size_t n = (size_t)nE * m;
  double* S;
  cudaMalloc(&S, (size_t)nE * m * m * sizeof(double));
  fill<<<4096, 256>>>(S, (size_t)nE * m * m, 1u);
  std::vector<double*> in(6), out(6);
  for (int k = 0; k < 6; ++k) {
    cudaMalloc(&in[k], n * 8);
    cudaMalloc(&out[k], n * 8);
    fill<<<1024, 256>>>(in[k], n, 100u + k);
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
  // batched outputs must equal single-system outputs bitwise (NR = 6 vs NR = 2 on RHS 4, 5)
  std::vector<double*> in2 = {in[4], in[5]}, out2(2);
  cudaMalloc(&out2[0], n * 8);
  cudaMalloc(&out2[1], n * 8);
  launch_block_gemv_multi(S, 6, in.data(), out.data(), m, nE, st);
  launch_block_gemv_multi(S, 2, in2.data(), out2.data(), m, nE, st);
  cudaStreamSynchronize(st);
  std::vector<double> a(n), b(n);
  bool same = true;
  for (int k = 0; k < 2; ++k) {
    cudaMemcpy(a.data(), out[4 + k], n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), out2[k], n * 8, cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < n; ++i) same = same && a[i] == b[i];
  }
  printf("NR=6 vs NR=2 bitwise: %s\n", same ? "equal" : "DIFFERENT");
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

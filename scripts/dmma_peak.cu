// fp64 tensor-core (mma.sync m8n8k4 f64) throughput probe: independent accumulator
// chains per warp, operands in registers, no memory traffic.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void __launch_bounds__(256) dmma_loop(double* out, int iters) {
  double acc[CH][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CH; ++c) { acc[c][0] = 0.0; acc[c][1] = 0.0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.0) out[0] = s;
}
template <int CH>
void run(int blocks_per_sm, int nsm) {
  double* o; cudaMalloc(&o, 8);
  const int iters = 4096, grid = nsm * blocks_per_sm;
  dmma_loop<CH><<<grid, 256>>>(o, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  dmma_loop<CH><<<grid, 256>>>(o, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = (double)grid * 8 * iters * CH * 512.0;
  printf("chains %2d  CTAs/SM %d (warps/SM %2d): %7.2f TFLOP/s  (%.3f ms)\n", CH, blocks_per_sm, 8 * blocks_per_sm,
         flops / (ms * 1e-3) / 1e12, ms);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int b : {1, 2, 4}) { run<1>(b, nsm); run<2>(b, nsm); run<4>(b, nsm); run<8>(b, nsm); }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

// Microbenchmark: cost of a 512-thread barrier step in a single-CTA kernel.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void steps(int nsteps, double* out, int work) {
  __shared__ double buf[2][128];
  const int t = threadIdx.x, c = t & 127;
  double x[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) x[q] = q * 0.001 + t;
  if (t < 128) buf[0][t] = 1.0;
  __syncthreads();
  for (int k = 0; k < nsteps; ++k) {
    const double f = buf[k & 1][c] * 1e-9;
    if (work) {
#pragma unroll
      for (int q = 0; q < 32; ++q) x[q] -= buf[k & 1][q * 4 % 128] * f;
    }
    if (t < 128) buf[(k + 1) & 1][t] = x[7] * 1e-3 + 1.0;
    __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 32; ++q) s += x[q];
  out[t] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 4096 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int threads : {128, 256, 512, 1024}) {
    for (int work : {0, 1}) {
      steps<<<1, threads>>>(128, out, work);
      cudaEventRecord(a);
      for (int r = 0; r < 10; ++r) steps<<<1, threads>>>(1024, out, work);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("threads %d work %d: %.3f us per step\n", threads, work, ms * 1e3 / (10 * 1024));
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

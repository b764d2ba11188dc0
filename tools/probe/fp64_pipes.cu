#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
  #pragma unroll
  for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < 16; i++) s += x[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}
__global__ void dmma_kernel(double* out, int iters) {
  double acc[16][2];
  #pragma unroll
  for (int i = 0; i < 16; i++) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int i = 0; i < 16; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}
__global__ void dmma16_kernel(double* out, int iters) {
  double acc[8][4];
  #pragma unroll
  for (int i = 0; i < 8; i++) for (int j=0;j<4;j++) acc[i][j] = 0;
  double a[8], b[4];
  for (int j=0;j<8;j++) a[j] = threadIdx.x * 1e-3 + j;
  for (int j=0;j<4;j++) b[j] = 1.0 + threadIdx.x * 1e-4 + j;
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
        : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
        : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(a[4]),"d"(a[5]),"d"(a[6]),"d"(a[7]),
          "d"(b[0]),"d"(b[1]),"d"(b[2]),"d"(b[3]));
    }
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < 8; i++) for (int j=0;j<4;j++) s += acc[i][j];
  if (s == 12345.0) out[threadIdx.x] = s;
}
int main() {
  double* out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  for (int threads : {256, 512, 1024}) {
    int iters = 20000;
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      dfma_kernel<<<sms * 2, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * iters * (double)threads * sms * 2;
      if (rep) printf("DFMA threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
    }
  }
  for (int threads : {128, 256, 512}) {
    int iters = 5000;
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      dmma_kernel<<<sms * 2, threads>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 16 * iters * (double)(threads / 32) * sms * 2;
      if (rep) printf("DMMA m8n8k4 threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
    }
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      dmma16_kernel<<<sms * 2, threads>>>(out, iters/4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16*8*16 * 8 * (iters/4) * (double)(threads / 32) * sms * 2;
      if (rep) printf("DMMA m16n8k16 threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}

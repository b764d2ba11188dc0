// Single-warp dependent-chain latencies (cycles per op) of the instructions
// on the small factorizations' critical path: DFMA, DMUL, MUFU.RSQ64H /
// MUFU.RCP64H, the STS -> __syncwarp -> LDS round trip, SHFL, bar.sync of 8 warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/lat_probe tools/probe/lat_probe.cu
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0, int n) {
  __shared__ double sm[64];
  const int lane = threadIdx.x & 31;
  double x = x0 + lane * 1e-9, y = 1.0000001;
  long long t[12];
  int q = 0;
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) x = __fma_rn(x, y, 1e-9);
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
  t[q++] = clock64();
  if (threadIdx.x < 32) {
    for (int i = 0; i < n; ++i) { sm[lane] = x; __syncwarp(); x = sm[(lane + 1) & 31]; __syncwarp(); }
  }
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) { __syncthreads(); }
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x) + 1.0;
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) { sm[lane + (threadIdx.x >> 5 & 1) * 32] = x; __syncthreads(); x = sm[(lane + 1) & 31]; }
  t[q++] = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) for (int i = 0; i + 1 < q; ++i) cyc[i] = t[i + 1] - t[i];
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 256); cudaMalloc(&c, 8 * 16);
  const int n = 1000;
  for (int th : {32, 256}) {
    k<<<1, th>>>(o, c, 1.5, n);
    long long h[16]; cudaMemcpy(h, c, 8 * 16, cudaMemcpyDeviceToHost);
    const char* nm[] = {"DFMA", "DMUL", "MUFU.RSQ64H", "MUFU.RCP64H", "STS+syncwarp+LDS(+syncwarp)", "SHFL.64", "bar.sync", "rsqrt()+DADD", "STS+bar.sync+LDS"};
    printf("threads %d:", th);
    for (int i = 0; i < 9; ++i) printf("  %s %.1f", nm[i], (double)h[i] / n);
    printf("\n");
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}

// Latency microbenchmarks on B200 (dev helper): cycles per dependent op.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, double a) {
  __shared__ double sm[1024];
  sm[threadIdx.x] = a + threadIdx.x;
  __syncthreads();
  double x = a, y = a * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, y);  // DFMA chain
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x / (y + 1.0);         // DDIV chain
  long long t2 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) { idx = (int)sm[idx & 1023] & 1023; }  // LDS chain
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t4 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) z = __shfl_xor_sync(0xffffffffu, z, 1) + 1.0;
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x + 1.0);
  long long t7 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 1.0);
  long long t8 = clock64();
  out[threadIdx.x] = x + z + idx;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    cyc[5] = t6 - t5; cyc[6] = t7 - t6; cyc[7] = t8 - t7;
  }
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8192); cudaMallocManaged(&cyc, 128);
  const char* names[] = {"DFMA", "DDIV", "LDS", "BAR(1024 thr)", "SHFL+DADD", "DSQRT", "DRCP_RN", "RSQRT"};
  for (int threads : {32, 1024}) {
    k<<<1, threads>>>(out, cyc, 1000, 1.5); cudaDeviceSynchronize();
    k<<<1, threads>>>(out, cyc, 1000, 1.5); cudaDeviceSynchronize();
    printf("threads=%d\n", threads);
    for (int i = 0; i < 8; ++i) printf("  %-14s %7.1f cycles/op\n", names[i], cyc[i] / 1000.0);
  }
  return 0;
}

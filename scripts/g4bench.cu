// Feasibility microbenchmark: TMA tile::gather4 row gathers (SpMM X rows) into shared
// memory vs plain LDG gathers.  X is n x k fp64 row-major; each "nonzero" gathers one
// row.  Indices follow a 7-point-stencil pattern (i, i+-1, i+-nx, i+-nx*ny) of a 64^3
// grid, i.e. the cfg2 SpMM access stream.  Prints achieved gather GB/s (row bytes).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/g4bench.cu -o g4bench
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);   \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(phase)
      : "memory");
  return ok;
}
__device__ __forceinline__ void g4(void* dst, const CUtensorMap* tm, unsigned long long* bar,
                                   int c0, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"((unsigned long long)tm), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

constexpr int NW = 8;

// per warp: STAGES buffers of G gathers (4 rows each); lanes 0..G-1 issue one gather4 each
template <int STAGES, int G>
__global__ void __launch_bounds__(NW * 32) g4_kernel(const __grid_constant__ CUtensorMap tm,
                                                     const int* __restrict__ idx, long long nnz,
                                                     int k, double* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row_bytes = k * 8;
  const int stage_bytes = G * 4 * row_bytes;
  unsigned char* base = sm + (size_t)warp * STAGES * stage_bytes;
  __shared__ __align__(8) unsigned long long bars[NW][STAGES];
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long long per = 4LL * G;  // nonzeros per batch
  const long long nb = nnz / per;
  const long long gw = (long long)gridDim.x * NW;
  const long long w0 = (long long)blockIdx.x * NW + warp;
  double acc = 0.0;
  auto issue = [&](long long b, int s) {
    if (lane == 0) mbar_expect(&bars[warp][s], (unsigned)stage_bytes);
    __syncwarp();
    if (lane < G) {
      const int* ix = idx + b * per + 4 * lane;
      g4(base + s * stage_bytes + lane * 4 * row_bytes, &tm, &bars[warp][s], 0, ix[0], ix[1],
         ix[2], ix[3]);
    }
  };
  long long my = 0;
  for (long long b = w0; b < nb && my < STAGES; b += gw, ++my) issue(b, (int)my);
  long long it = 0;
  for (long long b = w0; b < nb; b += gw, ++it) {
    const int s = (int)(it % STAGES);
    const unsigned ph = (unsigned)((it / STAGES) & 1);
    while (!mbar_try(&bars[warp][s], ph)) {
    }
    const double* d = (const double*)(base + s * stage_bytes);
    for (int e = lane; e < G * 4 * k; e += 32) acc += d[e];
    __syncwarp();
    const long long bn = b + STAGES * gw;
    if (bn < nb) issue(bn, s);
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void ldg_kernel(const double* __restrict__ X, int k, const int* __restrict__ idx,
                           long long nnz, double* out) {
  // lane group of k/4 lanes (double4) per nonzero row, as the register-pipelined SpMM
  const int lpr = k / 4;
  const int g = (threadIdx.x & 31) / lpr, sub = (threadIdx.x & 31) % lpr;
  const int G = 32 / lpr;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const long long w = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  double acc = 0.0;
  if (g < G) {
    for (long long e0 = w * G * 4; e0 < nnz; e0 += warps * G * 4) {
      double4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const long long e = e0 + u * G + g;
        v[u] = e < nnz ? *reinterpret_cast<const double4*>(X + (long long)idx[e] * k + sub * 4)
                       : make_double4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
  const int nx = 64, n = nx * nx * nx;
  const int k = argc > 1 ? atoi(argv[1]) : 20;
  std::vector<int> idx;
  idx.reserve((size_t)n * 8);
  const int off[7] = {-nx * nx, -nx, -1, 0, 1, nx, nx * nx};
  for (int i = 0; i < n; ++i)
    for (int o : off) {
      const int j = i + o;
      if (j >= 0 && j < n) idx.push_back(j);
    }
  while (idx.size() % 128) idx.push_back(0);
  const long long nnz = (long long)idx.size();
  double* X;
  int* didx;
  double* out;
  CK(cudaMalloc(&X, (size_t)n * k * 8));
  CK(cudaMemset(X, 0, (size_t)n * k * 8));
  CK(cudaMalloc(&didx, nnz * 4));
  CK(cudaMemcpy(didx, idx.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&out, 8));

  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)k, (cuuint64_t)n};
  cuuint64_t gstride[1] = {(cuuint64_t)k * 8};
  cuuint32_t box[2] = {(cuuint32_t)k, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, X, gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    return 1;
  }
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)nnz * k * 8;
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double t = ms / 20 / 1e3;
    printf("%-28s k=%3d  %8.1f us  %8.1f GB/s gathered\n", name, k, t * 1e6, bytes / t / 1e9);
  };
#define G4(ST, G)                                                                              \
  {                                                                                            \
    const int smb = NW * ST * G * 4 * k * 8;                                                   \
    if (smb > 220 * 1024) { printf("gather4 st=%d g=%d: %d B smem, skipped\n", ST, G, smb); } else \
    CK(cudaFuncSetAttribute(g4_kernel<ST, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb)); \
    int occ = 0;                                                                               \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, g4_kernel<ST, G>, NW * 32, smb);       \
    char nm[64];                                                                               \
    snprintf(nm, sizeof nm, "gather4 st=%d g=%d occ=%d", ST, G, occ);                          \
    run(nm, [&] { g4_kernel<ST, G><<<sms * (occ > 0 ? occ : 1), NW * 32, smb>>>(tm, didx, nnz, k, out); }); \
    CK(cudaGetLastError());                                                                    \
  }
  G4(2, 4) G4(3, 4) G4(4, 4) G4(2, 8) G4(2, 2) G4(3, 2) G4(4, 2) G4(6, 2)
  if (k % 4 == 0 && k / 4 <= 32) {
    run("ldg double4 (register)", [&] { ldg_kernel<<<sms * 4, 256>>>(X, k, didx, nnz, out); });
    CK(cudaGetLastError());
  }
  return 0;
}

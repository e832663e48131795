// Prototype: CSR SpMM with TMA tile::gather4 row gathers into shared memory
// (feasibility for the block-CG SpMM: n = 64^3 7-pt Laplacian, k = 20).
// Each warp owns tiles of T consecutive rows; lanes issue the gather4s of a tile's
// nonzero rows (4 per instruction) into a double-buffered per-warp stage, then the
// warp forms Y rows from the staged X rows.  Compared against a plain CSR
// reference for correctness and timed with CUDA events.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/spmm_tma_proto.cu -o /tmp/stp
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <math.h>
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

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(b)));
}
__device__ __forceinline__ void mb_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned ph) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}\n" ::"r"(sa(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void g4(void* dst, const CUtensorMap* tm, unsigned long long* b, int r0,
                                   int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(sa(dst)),
      "l"((unsigned long long)tm), "r"(sa(b)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

constexpr int K = 20;       // columns
#ifndef PT
#define PT 8
#endif
#ifndef PNW
#define PNW 8
#endif
constexpr int T = PT;           // rows per tile
constexpr int CAP = 8 * PT;     // nonzeros per tile stage (multiple of 4; >= 7 T)
constexpr int NW = PNW;         // warps per CTA
constexpr int ROWB = K * 8; // bytes per gathered row

// out-of-range row index for padding: TMA fills zeros
__global__ void __launch_bounds__(NW * 32) spmm_tma(const __grid_constant__ CUtensorMap tm, int n,
                                                    const int* __restrict__ rowptr,
                                                    const int* __restrict__ colidx,
                                                    const double* __restrict__ val,
                                                    double* __restrict__ Y) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* stage[2];
  stage[0] = (double*)(smem + (size_t)(warp * 2 + 0) * CAP * ROWB);
  stage[1] = (double*)(smem + (size_t)(warp * 2 + 1) * CAP * ROWB);
  __shared__ __align__(8) unsigned long long bar[NW][2];
  __shared__ int sptr[NW][2][T + 1];
  if (lane < 2) mb_init(&bar[warp][lane]);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int ntiles = (n + T - 1) / T;
  const int gw = gridDim.x * NW;
  int tile = blockIdx.x * NW + warp;
  // issue the gathers of `t` into stage s (rows assumed to fit CAP)
  auto issue = [&](int t, int s) {
    const int r0 = t * T;
    const int rcount = min(T, n - r0);
    if (lane <= rcount) sptr[warp][s][lane] = rowptr[r0 + lane];
    __syncwarp();
    const int e0 = sptr[warp][s][0], e1 = sptr[warp][s][rcount];
    const int nz = e1 - e0;
    const int ng = (nz + 3) / 4;
    if (lane == 0) mb_expect(&bar[warp][s], (unsigned)(ng * 4 * ROWB));
    __syncwarp();
    for (int q = lane; q < ng; q += 32) {
      int c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + 4 * q + u;
        c[u] = e < e1 ? colidx[e] : n;  // out of range -> zeros
      }
      g4(stage[s] + (size_t)4 * q * K, &tm, &bar[warp][s], c[0], c[1], c[2], c[3]);
    }
  };
  unsigned ph[2] = {0, 0};
  if (tile < ntiles) issue(tile, 0);
  int s = 0;
  for (; tile < ntiles; tile += gw, s ^= 1) {
    const int nt = tile + gw;
    if (nt < ntiles) issue(nt, s ^ 1);
    mb_wait(&bar[warp][s], ph[s]);
    ph[s] ^= 1;
    const int r0 = tile * T;
    const int rcount = min(T, n - r0);
    const int e0 = sptr[warp][s][0];
    // (row, 4-column chunk) items: T rows x 5 chunks
    for (int it = lane; it < rcount * (K / 4); it += 32) {
      const int rr = it / (K / 4), ch = it % (K / 4);
      const int a = sptr[warp][s][rr], b = sptr[warp][s][rr + 1];
      double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
      for (int e = a; e < b; ++e) {
        const double v = __ldg(val + e);
        const double4 x = *reinterpret_cast<const double4*>(stage[s] + (size_t)(e - e0) * K + ch * 4);
        acc0 = fma(v, x.x, acc0);
        acc1 = fma(v, x.y, acc1);
        acc2 = fma(v, x.z, acc2);
        acc3 = fma(v, x.w, acc3);
      }
      *reinterpret_cast<double4*>(Y + (size_t)(r0 + rr) * K + ch * 4) = make_double4(acc0, acc1, acc2, acc3);
    }
    __syncwarp();
  }
}

__global__ void spmm_ref(int n, const int* rowptr, const int* colidx, const double* val,
                         const double* X, double* Y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * K) return;
  const int r = i / K, c = i % K;
  double s = 0;
  for (int e = rowptr[r]; e < rowptr[r + 1]; ++e) s += val[e] * X[(size_t)colidx[e] * K + c];
  Y[i] = s;
}

int main() {
  const int N = 64, n = N * N * N;
  std::vector<int> rp(n + 1), ci;
  std::vector<double> v;
  rp[0] = 0;
  for (int z = 0; z < N; ++z)
    for (int y = 0; y < N; ++y)
      for (int x = 0; x < N; ++x) {
        const int i = (z * N + y) * N + x;
        const int offs[7][3] = {{-1, 0, 0}, {0, -1, 0}, {0, 0, -1}, {0, 0, 0}, {0, 0, 1}, {0, 1, 0}, {1, 0, 0}};
        for (auto& o : offs) {
          const int zz = z + o[0], yy = y + o[1], xx = x + o[2];
          if (zz < 0 || zz >= N || yy < 0 || yy >= N || xx < 0 || xx >= N) continue;
          ci.push_back((zz * N + yy) * N + xx);
          v.push_back((o[0] | o[1] | o[2]) ? -1.0 : 6.0);
        }
        rp[i + 1] = (int)ci.size();
      }
  const int nnz = (int)ci.size();
  std::vector<double> xh((size_t)n * K);
  for (size_t i = 0; i < xh.size(); ++i) xh[i] = sin(0.001 * i);
  int *drp, *dci;
  double *dv, *dx, *dy, *dyr;
  CK(cudaMalloc(&drp, (n + 1) * 4));
  CK(cudaMalloc(&dci, nnz * 4));
  CK(cudaMalloc(&dv, nnz * 8));
  CK(cudaMalloc(&dx, (size_t)n * K * 8));
  CK(cudaMalloc(&dy, (size_t)n * K * 8));
  CK(cudaMalloc(&dyr, (size_t)n * K * 8));
  CK(cudaMemcpy(drp, rp.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, v.data(), nnz * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dx, xh.data(), (size_t)n * K * 8, cudaMemcpyHostToDevice));
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)n};
  cuuint64_t gstride[1] = {(cuuint64_t)K * 8};
  cuuint32_t box[2] = {(cuuint32_t)K, 1};
  cuuint32_t estr[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dx, gdim, gstride, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int smb = NW * 2 * CAP * ROWB;
  CK(cudaFuncSetAttribute(spmm_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smb));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmm_tma, NW * 32, smb);
  spmm_ref<<<(n * K + 255) / 256, 256>>>(n, drp, dci, dv, dx, dyr);
  spmm_tma<<<sms * occ, NW * 32, smb>>>(tm, n, drp, dci, dv, dy);
  CK(cudaDeviceSynchronize());
  std::vector<double> a((size_t)n * K), b((size_t)n * K);
  CK(cudaMemcpy(a.data(), dy, a.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b.data(), dyr, b.size() * 8, cudaMemcpyDeviceToHost));
  double err = 0;
  for (size_t i = 0; i < a.size(); ++i) err = fmax(err, fabs(a[i] - b[i]));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) spmm_tma<<<sms * occ, NW * 32, smb>>>(tm, n, drp, dci, dv, dy);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) spmm_tma<<<sms * occ, NW * 32, smb>>>(tm, n, drp, dci, dv, dy);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("spmm_tma T=%d NW=%d occ=%d smem=%d  %.1f us  max|err|=%.3e\n", T, NW, occ, smb, ms / 20 * 1e3, err);
  return 0;
}

// MatDotMultiVec on B200: fp64 CSR x row-major multivector (SpMM).
//
// Reference: CsrOperator.apply (operators.py:103-111) -> kernels.csr_matvec
// (_cy.pyx:11-23: column-by-column scalar CSR loop) and ShiftedOperator.apply
// (operators.py:149-156: A x - theta (B x or x)).
//
// B200 design.  X is row-major, so the k values a nonzero (i, j) needs are one
// contiguous run X[j*ldx : j*ldx+k]: a group of LPR lanes owns one row and
// reads those runs with 16-byte vector loads (coalesced, L2-resident for the
// stencil's plane-distance reuse).  The row's (column index, value) stream is
// loaded once, cooperatively, one nonzero per lane, and broadcast inside the
// group with shuffles — 12 B/nnz from HBM instead of k separate index loads.
// The epilogue fuses the shifted-operator term (gamma*Z, Z = X for A - theta*I),
// an axpby with a second input (beta*Yin, used for r = rhs - op x) and an
// optional per-column dot product reduced deterministically (p'q and ||r||^2
// for block CG), so CG never makes a separate pass for them.
//
// Roofline: HBM.  Algorithmic bytes per launch = 12*nnz + 4*(n+1) + 16*n*k
// (+8*n*k per extra epilogue stream); flops = 2*nnz*k.

#include <stdlib.h>

#include "common.cuh"

namespace gcg {

struct SpmmArgs {
  long long n;
  const int* __restrict__ rowptr;
  const int* __restrict__ colidx;
  const double* __restrict__ val;
  int k;
  const double* __restrict__ X;
  long long ldx;
  double alpha, gamma, beta;
  const double* __restrict__ Z;
  long long ldz;
  const double* Yin;
  long long ldyin;
  double* Y;
  long long ldy;
  int dot_mode;
  const double* __restrict__ W;
  long long ldw;
  double* partials;  // [gridDim.x][k]
  const int* skip;   // device flag: nonzero -> kernel is a no-op (CG early exit)
  int* prof_skipped; // profiling: set when the launch was a no-op
  long long nnz;     // total nonzeros (clips the bulk copies of the last tile)
  int cap;           // nonzeros per shared-memory stage (tiled kernel)
};

template <int VEC>
struct VecT;
template <>
struct VecT<1> {
  using T = double;
  static __device__ __forceinline__ void load(const double* p, double* o) { o[0] = __ldg(p); }
};
template <>
struct VecT<2> {
  static __device__ __forceinline__ void load(const double* p, double* o) {
    double2 v = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = v.x;
    o[1] = v.y;
  }
};

constexpr int kSpmmThreads = 256;

template <int LPR, int VEC, int NV>
__global__ void __launch_bounds__(kSpmmThreads) spmm_csr_kernel(SpmmArgs a) {
  if (a.skip != nullptr && *a.skip) {
    if (a.prof_skipped && blockIdx.x == 0 && threadIdx.x == 0) *a.prof_skipped = 1;
    return;
  }
  constexpr int G = 32 / LPR;  // row groups per warp
  constexpr int COLS = LPR * VEC * NV;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int g = lane / LPR;
  const int sub = lane % LPR;
  const int nwarps = kSpmmThreads / 32;
  const long long stride = (long long)gridDim.x * nwarps * G;
  const int k = a.k;

  __shared__ double sdot[kSpmmThreads / 32][COLS];
  double dacc[NV][VEC];
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int v = 0; v < VEC; ++v) dacc[q][v] = 0.0;

  // This kernel handles one column pass [c0, c0 + COLS); wider blocks are
  // split by the launcher into several launches with offset pointers.
  for (long long rb = ((long long)blockIdx.x * nwarps + warp) * G; rb < a.n; rb += stride) {
    const long long r = rb + g;
    const bool valid = r < a.n;
    int start = 0, len = 0;
    if (valid) {
      start = __ldg(a.rowptr + r);
      len = __ldg(a.rowptr + r + 1) - start;
    }
    const int maxlen = __reduce_max_sync(0xffffffffu, len);
    double acc[NV][VEC];
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[q][v] = 0.0;

    for (int off = 0; off < maxlen; off += LPR) {
      int mycol = 0;
      double myval = 0.0;
      if (off + sub < len) {
        mycol = __ldg(a.colidx + start + off + sub);
        myval = __ldg(a.val + start + off + sub);
      }
      const int tmax = min(LPR, maxlen - off);
#pragma unroll 4
      for (int t = 0; t < tmax; ++t) {
        const int j = __shfl_sync(0xffffffffu, mycol, t, LPR);
        const double v = __shfl_sync(0xffffffffu, myval, t, LPR);
        if (off + t < len) {
          const double* xr = a.X + (long long)j * a.ldx;
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            const int c = (q * LPR + sub) * VEC;
            if (c < k) {
              double xv[VEC];
              VecT<VEC>::load(xr + c, xv);
#pragma unroll
              for (int e = 0; e < VEC; ++e) acc[q][e] = fma(v, xv[e], acc[q][e]);
            }
          }
        }
      }
    }
    if (valid) {
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const int c = (q * LPR + sub) * VEC;
        if (c < k) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            double y = a.alpha * acc[q][e];
            if (a.gamma != 0.0) y = fma(a.gamma, a.Z[r * a.ldz + c + e], y);
            if (a.beta != 0.0) y = fma(a.beta, a.Yin[r * a.ldyin + c + e], y);
            a.Y[r * a.ldy + c + e] = y;
            if (a.dot_mode == 1) dacc[q][e] = fma(y, a.W[r * a.ldw + c + e], dacc[q][e]);
            else if (a.dot_mode == 2) dacc[q][e] = fma(y, y, dacc[q][e]);
          }
        }
      }
    }
  }

  if (a.dot_mode == 0) return;
  // reduce over the row groups of the warp (lanes with equal `sub`)
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      double v = dacc[q][e];
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      dacc[q][e] = v;
    }
  if (g == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) sdot[warp][(q * LPR + sub) * VEC + e] = dacc[q][e];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k && c < COLS; c += kSpmmThreads) {
    double s = 0.0;
    for (int w = 0; w < nwarps; ++w) s += sdot[w][c];
    a.partials[(long long)blockIdx.x * k + c] = s;
  }
}

// out[c*out_stride] = sum_b partials[b*k + c] in fixed b order (deterministic).
__global__ void reduce_partials_kernel(const double* __restrict__ partials, int nparts, int k,
                                       double* out, int out_stride, int mode) {
  const int c = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nparts; b += blockDim.x) s += partials[(long long)b * k + c];
  // fixed-shape tree over the 128 threads
  __shared__ double sm[128];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = 64; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double v = sm[0];
    if (mode == 1) v += out[(long long)c * out_stride];
    out[(long long)c * out_stride] = v;
  }
}

int reduce_partials(Ctx* c, const double* partials, int nparts, int k, double* out,
                    int out_stride, int mode) {
  if (k <= 0) return GCG_OK;
  reduce_partials_kernel<<<k, 128, 0, c->stream>>>(partials, nparts, k, out, out_stride, mode);
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

extern int64_t g_launches;

// ---------------------------------------------------------------------------
// Tiled SpMM: persistent CTAs walk tiles of kTileRows rows.  The tile's
// (column index, value) streams are one contiguous nonzero range, so it is
// brought into shared memory with two 1-D TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx) one tile AHEAD of the compute: the
// HBM index/value stream never sits in the dependent load chain of a row.
// Rows then read their (col, val) pairs as shared-memory broadcasts and issue
// all X-row gathers of an unrolled group at once.

constexpr int kTileRows = 128;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, int bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, int phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, int bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct TileStage {
  int rp[kTileRows + 1];  // row pointers of the tile (absolute)
  int c0;                 // first nonzero held in smem (index alignment base)
  int v0;                 // value alignment base
  int cend, vend;         // smem holds [c0, cend) / [v0, vend); the rest is read from global
};

template <int LPR, int VEC, int NV>
__global__ void __launch_bounds__(kSpmmThreads) spmm_tiled_kernel(SpmmArgs a) {
  if (a.skip != nullptr && *a.skip) {
    if (a.prof_skipped && blockIdx.x == 0 && threadIdx.x == 0) *a.prof_skipped = 1;
    return;
  }
  constexpr int G = 32 / LPR;
  constexpr int COLS = LPR * VEC * NV;
  constexpr int NW = kSpmmThreads / 32;
  constexpr int U = 4;  // nonzeros per unrolled gather group
  extern __shared__ __align__(16) unsigned char sm_raw[];
  __shared__ TileStage st[2];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ double sdot[NW][COLS];
  const int cap = a.cap;
  // stage s: values at sval0 + s*(cap+2), indices at scol0 + s*(cap+4)
  double* const sval0 = reinterpret_cast<double*>(sm_raw);
  int* const scol0 = reinterpret_cast<int*>(sval0 + 2 * (cap + 2));

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / LPR, sub = lane % LPR;
  const int k = a.k;
  const long long ntiles = (a.n + kTileRows - 1) / kTileRows;

  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  double dacc[NV][VEC];
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int e = 0; e < VEC; ++e) dacc[q][e] = 0.0;

  // stage the row pointers of tile t into st[s] (all threads), then thread 0
  // issues the bulk copies of its index/value ranges
  auto stage_rp = [&](long long t, int s) {
    const long long r0 = t * kTileRows;
    const int nr = (int)min((long long)kTileRows, a.n - r0);
    for (int i = threadIdx.x; i <= nr; i += kSpmmThreads) st[s].rp[i] = __ldg(a.rowptr + r0 + i);
  };
  auto bulk = [&](long long t, int s) {
    const long long r0 = t * kTileRows;
    const int nr = (int)min((long long)kTileRows, a.n - r0);
    const int beg = st[s].rp[0], end = st[s].rp[nr];
    int c0 = beg & ~3, c1 = (end + 3) & ~3;
    const int cmax = (int)(a.nnz & ~3LL);
    if (c1 > cmax) c1 = cmax > c0 ? cmax : c0;
    if (c1 - c0 > cap) c1 = c0 + (cap & ~3);  // overflow beyond the stage: read from global
    int v0 = beg & ~1, v1 = (end + 1) & ~1;
    const int vmax = (int)(a.nnz & ~1LL);
    if (v1 > vmax) v1 = vmax > v0 ? vmax : v0;
    if (v1 - v0 > cap) v1 = v0 + (cap & ~1);
    st[s].c0 = c0;
    st[s].cend = c1;
    st[s].v0 = v0;
    st[s].vend = v1;
    const int bytes = (c1 - c0) * 4 + (v1 - v0) * 8;
    mbar_arrive_tx(&bar[s], bytes);
    if (c1 > c0) tma_load_1d(scol0 + s * (cap + 4), a.colidx + c0, (c1 - c0) * 4, &bar[s]);
    if (v1 > v0) tma_load_1d(sval0 + s * (cap + 2), a.val + v0, (v1 - v0) * 8, &bar[s]);
  };

  long long t = blockIdx.x;
  int s = 0, phase0 = 0, phase1 = 0;
  if (t < ntiles) {
    stage_rp(t, 0);
    __syncthreads();
    if (threadIdx.x == 0) bulk(t, 0);
  }
  for (; t < ntiles; t += gridDim.x, s ^= 1) {
    const long long tn = t + gridDim.x;
    // prefetch the next tile into the other stage (its previous use finished at the
    // __syncthreads that ended the last iteration)
    if (tn < ntiles) {
      stage_rp(tn, s ^ 1);
      __syncthreads();
      if (threadIdx.x == 0) bulk(tn, s ^ 1);
    }
    mbar_wait(&bar[s], s == 0 ? phase0 : phase1);
    if (s == 0) phase0 ^= 1;
    else phase1 ^= 1;
    const TileStage& S = st[s];
    const int* cs = scol0 + s * (cap + 4);
    const double* vs = sval0 + s * (cap + 2);
    const long long r0 = t * kTileRows;
    const int nr = (int)min((long long)kTileRows, a.n - r0);
    for (int lr = warp * G + g; lr < nr; lr += NW * G) {
      const int beg = S.rp[lr], end = S.rp[lr + 1];
      double acc[NV][VEC];
#pragma unroll
      for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[q][e] = 0.0;
      for (int j0 = beg; j0 < end; j0 += U) {
        int col[U];
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + u;
          const bool ok = j < end;
          col[u] = ok ? (j < S.cend ? cs[j - S.c0] : __ldg(a.colidx + j)) : 0;
          v[u] = ok ? (j < S.vend ? vs[j - S.v0] : __ldg(a.val + j)) : 0.0;
        }
        double xv[U][NV][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double* xr = a.X + (long long)col[u] * a.ldx;
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            const int c = (q * LPR + sub) * VEC;
            if (c < k && j0 + u < end) VecT<VEC>::load(xr + c, xv[u][q]);
            else
#pragma unroll
              for (int e = 0; e < VEC; ++e) xv[u][q][e] = 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < NV; ++q)
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[q][e] = fma(v[u], xv[u][q][e], acc[q][e]);
      }
      const long long r = r0 + lr;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const int c = (q * LPR + sub) * VEC;
        if (c < k) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            double y = a.alpha * acc[q][e];
            if (a.gamma != 0.0) y = fma(a.gamma, a.Z[r * a.ldz + c + e], y);
            if (a.beta != 0.0) y = fma(a.beta, a.Yin[r * a.ldyin + c + e], y);
            a.Y[r * a.ldy + c + e] = y;
            if (a.dot_mode == 1) dacc[q][e] = fma(y, a.W[r * a.ldw + c + e], dacc[q][e]);
            else if (a.dot_mode == 2) dacc[q][e] = fma(y, y, dacc[q][e]);
          }
        }
      }
    }
    __syncthreads();  // stage s is free for the prefetch two tiles ahead
  }

  if (a.dot_mode == 0) return;
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      double v = dacc[q][e];
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      dacc[q][e] = v;
    }
  if (g == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) sdot[warp][(q * LPR + sub) * VEC + e] = dacc[q][e];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k && c < COLS; c += kSpmmThreads) {
    double sum = 0.0;
    for (int w = 0; w < NW; ++w) sum += sdot[w][c];
    a.partials[(long long)blockIdx.x * k + c] = sum;
  }
}

template <int LPR, int VEC>
static int launch_tiled_nv(Ctx* c, SpmmArgs a, int nv, int grid, size_t sm) {
  switch (nv) {
#define TCASE(NVV)                                                                         \
  case NVV: {                                                                              \
    auto kern = spmm_tiled_kernel<LPR, VEC, NVV>;                                          \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);      \
    kern<<<grid, kSpmmThreads, sm, c->stream>>>(a);                                        \
    break;                                                                                 \
  }
    TCASE(1)
    TCASE(2)
    TCASE(3)
    default:
      TCASE(4)
#undef TCASE
  }
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

template <int VEC>
static int launch_tiled(Ctx* c, SpmmArgs a, int lpr, int nv, int grid, size_t sm) {
  switch (lpr) {
    case 4: return launch_tiled_nv<4, VEC>(c, a, nv, grid, sm);
    case 8: return launch_tiled_nv<8, VEC>(c, a, nv, grid, sm);
    case 16: return launch_tiled_nv<16, VEC>(c, a, nv, grid, sm);
    default: return launch_tiled_nv<32, VEC>(c, a, nv, grid, sm);
  }
}

template <int LPR, int VEC>
static int launch_nv(Ctx* c, SpmmArgs a, int nv, int grid) {
  switch (nv) {
    case 1: spmm_csr_kernel<LPR, VEC, 1><<<grid, kSpmmThreads, 0, c->stream>>>(a); break;
    case 2: spmm_csr_kernel<LPR, VEC, 2><<<grid, kSpmmThreads, 0, c->stream>>>(a); break;
    case 3: spmm_csr_kernel<LPR, VEC, 3><<<grid, kSpmmThreads, 0, c->stream>>>(a); break;
    default: spmm_csr_kernel<LPR, VEC, 4><<<grid, kSpmmThreads, 0, c->stream>>>(a); break;
  }
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

template <int VEC>
static int launch_lpr(Ctx* c, SpmmArgs a, int lpr, int nv, int grid) {
  switch (lpr) {
    case 4: return launch_nv<4, VEC>(c, a, nv, grid);
    case 8: return launch_nv<8, VEC>(c, a, nv, grid);
    case 16: return launch_nv<16, VEC>(c, a, nv, grid);
    default: return launch_nv<32, VEC>(c, a, nv, grid);
  }
}

static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

int spmm_grid(Ctx* c, long long n) { return grid_for(n, 64, 8, c->num_sms); }

// One SpMM over all k columns, split into passes of at most 256 columns.  With
// dot_mode != 0 and `partials` given, per-CTA partials ([grid][k], k <= 256)
// are left for the caller to reduce; otherwise they are reduced into `dots`.
int spmm_launch_impl(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                     const double* val, int k, const double* X, long long ldx, double alpha,
                     double gamma, const double* Z, long long ldz, double beta, const double* Yin,
                     long long ldyin, double* Y, long long ldy, int dot_mode, const double* W,
                     long long ldw, double* dots, double* partials_ext, int* grid_out,
                     const int* skip) {
  if (n <= 0 || k <= 0) return GCG_OK;
  constexpr int kMaxPass = 256;
  // tiled (TMA-staged) path: needs 16-byte aligned index/value arrays
  static const bool legacy_env = getenv("GCG_SPMM_LEGACY") != nullptr;
  const bool tiled = !legacy_env && nnz > 0 && ((uintptr_t)colidx & 15u) == 0 &&
                     ((uintptr_t)val & 15u) == 0;
  const double avg = (double)nnz / (double)n;
  int tcap = (int)(1.25 * kTileRows * avg) + 16;
  if (tcap > 8192) tcap = 8192;
  tcap = (tcap + 3) & ~3;
  const size_t tsm = (size_t)2 * (tcap + 2) * sizeof(double) + (size_t)2 * (tcap + 4) * sizeof(int);
  int per_sm = (int)((200 * 1024) / (tsm + 16 * 1024));
  if (per_sm > 4) per_sm = 4;
  if (per_sm < 1) per_sm = 1;
  const long long ntiles = (n + kTileRows - 1) / kTileRows;
  const int tgrid = (int)(ntiles < (long long)c->num_sms * per_sm ? ntiles : c->num_sms * per_sm);
  const int grid = tiled ? tgrid : spmm_grid(c, n);
  if (grid_out) *grid_out = grid;
  if (partials_ext && k > kMaxPass) return GCG_ERR_ARG;
  double* partials = partials_ext;
  if (dot_mode && !partials) {
    GCG_TRY(ensure(c->partials, sizeof(double) * (size_t)grid * (size_t)kMaxPass));
    partials = (double*)c->partials.ptr;
  }
  for (int c0 = 0; c0 < k; c0 += kMaxPass) {
    const int kc = (k - c0) < kMaxPass ? (k - c0) : kMaxPass;
    bool vec2 = (kc % 2 == 0) && (ldx % 2 == 0) && aligned16(X + c0);
    const int vec = vec2 ? 2 : 1;
    const int lanes_needed = (kc + vec - 1) / vec;
    int lpr = 4;
    while (lpr < 32 && lpr * 2 < lanes_needed) lpr <<= 1;
    int nv = (lanes_needed + lpr - 1) / lpr;
    while (nv > 4 && lpr < 32) {
      lpr <<= 1;
      nv = (lanes_needed + lpr - 1) / lpr;
    }
    SpmmArgs a;
    a.n = n;
    a.rowptr = rowptr;
    a.colidx = colidx;
    a.val = val;
    a.k = kc;
    a.X = X + c0;
    a.ldx = ldx;
    a.alpha = alpha;
    a.gamma = gamma;
    a.Z = Z ? Z + c0 : nullptr;
    a.ldz = ldz;
    a.beta = beta;
    a.Yin = Yin ? Yin + c0 : nullptr;
    a.ldyin = ldyin;
    a.Y = Y + c0;
    a.ldy = ldy;
    a.dot_mode = dot_mode;
    a.W = W ? W + c0 : nullptr;
    a.ldw = ldw;
    a.partials = partials;
    a.skip = skip;
    // algorithmic bytes: index/value stream + X once + Y once + each extra distinct stream
    double bytes = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n * kc;
    if (gamma != 0.0 && Z != X) bytes += 8.0 * n * kc;
    if (beta != 0.0) bytes += 8.0 * n * kc;
    if (dot_mode == 1 && W != X && W != Z) bytes += 8.0 * n * kc;
    a.nnz = nnz;
    const int ps = prof_start(c, PROF_SPMM, bytes);
    a.prof_skipped = prof_skip_slot(c, ps);
    int s;
    if (tiled) {
      a.cap = tcap;
      s = vec2 ? launch_tiled<2>(c, a, lpr, nv, tgrid, tsm)
               : launch_tiled<1>(c, a, lpr, nv, tgrid, tsm);
    } else {
      a.cap = 0;
      s = vec2 ? launch_lpr<2>(c, a, lpr, nv, grid) : launch_lpr<1>(c, a, lpr, nv, grid);
    }
    prof_stop(c, ps);
    if (s != GCG_OK) return s;
    if (dot_mode && !partials_ext) {
      GCG_TRY(reduce_partials(c, partials, grid, kc, dots + c0, 1, 0));
      ++g_launches;
    }
  }
  return GCG_OK;
}

int spmm_launch_parts(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                      const double* val, int k, const double* X, long long ldx, double alpha,
                      double gamma, const double* Z, long long ldz, double beta,
                      const double* Yin, long long ldyin, double* Y, long long ldy, int dot_mode,
                      const double* W, long long ldw, double* partials, int* grid_out,
                      const int* skip) {
  return spmm_launch_impl(c, n, nnz, rowptr, colidx, val, k, X, ldx, alpha, gamma, Z, ldz, beta, Yin,
                          ldyin, Y, ldy, dot_mode, W, ldw, nullptr, partials, grid_out, skip);
}

}  // namespace gcg

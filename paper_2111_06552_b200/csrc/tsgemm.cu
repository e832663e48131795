// Tall-skinny fp64 GEMMs on B200 with FP64 tensor cores (DMMA): Gram
// (MultiVecInnerProd) and LinComb (MultiVecLinearComb).
//
//  gram     G = alpha X'Y + beta G   multivec.py:84-112, _cy.pyx:26-50, orth.py:139-140,164,242,288
//  lincomb  Y = alpha X C + beta Y   solver.py:300,333,376; orth.py:144,175,184,264,291
//
// B200 has no FP64 kind in tcgen05; its FP64 tensor path is the warp-level
// DMMA (mma.sync.m8n8k4.f64, SASS DMMA.8x8x4), at the same ~40 TF as the FFMA64
// pipe but with 256 FMAs per instruction and operands from registers.  With
// SIMT micro-tiles these kernels were shared-memory-issue bound (one LDS per
// two FMAs); with DMMA a warp tile of FMxFN 8x8 blocks needs FM+FN fragment
// loads per FM*FN*256 FMAs.
//
// Both kernels stream the n-long panel once from HBM through a 3-stage
// cp.async (LDGSTS) shared-memory ring (16-byte copies when row runs are
// 16-byte aligned).  Shared-memory row strides are 4 (mod 16) doubles so the
// four rows a half-warp touches for a fragment land in disjoint bank groups.
//
// Gram splits the n-long contraction over (a) row groups of warps inside a CTA
// and (b) row slabs across CTAs; CTA partials are combined in shared memory
// and the slab partials by a second kernel with one warp per output, always
// in a fixed order — bit-identical run to run (test_kernels.py:74-85).

#include <stdint.h>
#include <stdlib.h>

#include "async.cuh"
#include "common.cuh"

namespace gcg {

extern int64_t g_launches;

// d = a*b + d for one 8x8x4 fp64 block (A row fragment, B col fragment)
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Copy element `idx` (pair index when VEC16) of a row run of `valid` doubles.
template <bool VEC16>
__device__ __forceinline__ void stage_elems(double* dst, const double* src, int idx, int valid,
                                            const double* safe) {
  if (VEC16) {
    const int e = idx * 2;
    const int nb = valid - e >= 2 ? 16 : (valid - e == 1 ? 8 : 0);
    cp_async16(dst + e, nb ? src + e : safe, nb);
  } else {
    cp_async8(dst + idx, idx < valid ? src + idx : safe, idx < valid);
  }
}

constexpr int kStages = 3;

// smem stride (doubles) >= w, even, and 4 (mod 16)
__host__ __device__ constexpr int frag_stride(int w) { return ((w + 11) / 16) * 16 + 4; }

// ---------------------------------------------------------------------------
// Gram: CTA tile BM x BN; warps tile it WM x WN; the remaining warps split rows.

__constant__ int c_ts_desc = 0;  // GCG_LC_DESC=1: lincomb_ts_kernel walks its row tiles downwards

template <int BM, int BN, int WM, int WN, int R, bool VEC16, bool BULK = false>
__global__ void __launch_bounds__(256) gram_dmma_kernel(long long n, int k1, int k2,
                                                        const double* __restrict__ X,
                                                        long long ldx,
                                                        const double* __restrict__ Y,
                                                        long long ldy, long long rows_per_slab,
                                                        double* part, Skip skip) {
  pdl_wait();  // launched with programmatic stream serialization: predecessor complete from here on
  if (skip_now(skip)) return;
  constexpr int FM = WM / 8, FN = WN / 8;
  constexpr int WT = (BM / WM) * (BN / WN);  // warps per output tile
  constexpr int RG = 8 / WT;                 // row groups
  static_assert(WT * RG == 8, "8 warps");
  constexpr int W = frag_stride(BM + BN);
  constexpr int V = VEC16 ? 2 : 1;
  extern __shared__ __align__(16) double smg[];
  const int tm0 = blockIdx.x * BM, tn0 = blockIdx.y * BN;
  // rows_per_slab > 0: slab z owns one contiguous row range; < 0: the R-row stages are dealt
  // round-robin over the slabs (stage ch of slab z = rows ((ch * nslab + z) * R ...)), so the
  // grid walks X and Y as one ascending window — the LinComb that follows walks the same
  // rows downwards and starts on the lines this kernel left in L2
  const bool inter = rows_per_slab < 0;
  const long long r0 = inter ? (long long)blockIdx.z * R : (long long)blockIdx.z * rows_per_slab;
  long long r1 = inter ? n : r0 + rows_per_slab;
  if (r1 > n) r1 = n;
  const long long cstride = inter ? (long long)gridDim.z * R : (long long)R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wt = warp % WT, rg = warp / WT;
  const int wm0 = (wt / (BN / WN)) * WM, wn0 = (wt % (BN / WN)) * WN;
  const int vx = min(BM, k1 - tm0), vy = min(BN, k2 - tn0);
  const int nch = r1 > r0 ? (int)((r1 - r0 + cstride - 1) / cstride) : 0;
  const int fr = lane & 3, fc = lane >> 2;  // fragment row (k) / column (m or n)
  // Bulk mode: row runs that start 8 bytes past a 16-byte boundary (views at an odd
  // column of an even-ld arena) are copied from one element earlier, so the tile
  // sits at +1 in its shared-memory row; the Y part starts at BM + 2 (16-B aligned).
  static_assert(!BULK || W >= BM + BN + 3, "room for the shifted runs");
  const int sxo = BULK ? (int)(((uintptr_t)(X + tm0) >> 3) & 1) : 0;
  const int syo = BULK ? (int)(((uintptr_t)(Y + tn0) >> 3) & 1) : 0;
  const int xo = sxo, yo = BULK ? BM + 2 + syo : BM;  // shared-memory column of element 0

  __shared__ __align__(8) unsigned long long mbar[kStages];
  if constexpr (BULK) {
    if (tid == 0) {
      for (int s = 0; s < kStages; ++s) mbar_init(&mbar[s]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  auto load = [&](int ch, int st) {
    const long long rb = r0 + (long long)ch * cstride;
    if constexpr (BULK) {
      // one bulk copy per row segment (threads 0.. for X, 128.. for Y); an odd
      // trailing column and the rows past the slab end are filled by plain stores
      const int nr = (int)min((long long)R, r1 - rb);
      const int ex = vx + sxo, ey = vy + syo;  // elements copied, incl. the lead-in
      const int bx = (ex * 8) & ~15, by = (ey * 8) & ~15;
      double* base = smg + st * R * W;
      if (tid == 0) mbar_expect(&mbar[st], (unsigned)(nr * (bx + by)));
      if (tid < nr) {
        const long long row = rb + tid;
        const double* src = X + row * ldx + tm0 - sxo;
        if (bx) bulk_g2s(base + tid * W, src, bx, &mbar[st]);
        if (ex & 1) base[tid * W + ex - 1] = src[ex - 1];
      } else if (tid >= 128 && tid - 128 < nr) {
        const int t = tid - 128;
        const long long row = rb + t;
        const double* src = Y + row * ldy + tn0 - syo;
        if (by) bulk_g2s(base + t * W + BM + 2, src, by, &mbar[st]);
        if (ey & 1) base[t * W + BM + 2 + ey - 1] = src[ey - 1];
      }
      for (int e = tid; e < (R - nr) * W; e += 256) base[nr * W + e] = 0.0;
    } else {
      constexpr int PX = BM / V, PY = BN / V, P = PX + PY;
      for (int e = tid; e < R * P; e += 256) {
        const int rr = e / P, cc = e % P;
        const long long row = rb + rr;
        double* dst = smg + (st * R + rr) * W;
        const bool ok = row < r1;
        if (cc < PX)
          stage_elems<VEC16>(dst, X + (ok ? row : r0) * ldx + tm0, cc, ok ? vx : 0, X);
        else
          stage_elems<VEC16>(dst + BM, Y + (ok ? row : r0) * ldy + tn0, cc - PX, ok ? vy : 0, Y);
      }
    }
  };

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nch) load(s, s);
    cp_commit();
  }
  for (int ch = 0; ch < nch; ++ch) {
    if constexpr (BULK) mbar_wait(&mbar[ch % kStages], (unsigned)((ch / kStages) & 1));
    else cp_wait<kStages - 2>();
    __syncthreads();
    if (ch + kStages - 1 < nch) load(ch + kStages - 1, (ch + kStages - 1) % kStages);
    cp_commit();
    const double* base = smg + (ch % kStages) * R * W;
#pragma unroll 2
    for (int ks = rg; ks < R / 4; ks += RG) {
      const double* rowp = base + (ks * 4 + fr) * W;
      double a[FM], b[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) a[i] = rowp[xo + wm0 + i * 8 + fc];
#pragma unroll
      for (int j = 0; j < FN; ++j) b[j] = rowp[yo + wn0 + j * 8 + fc];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  pdl_trigger();  // late: the successor (the finish kernel) launches while this grid drains
  cp_wait<0>();
  __syncthreads();
  // combine the RG row groups in a fixed order
  double* red = smg;  // RG * BM * BN doubles
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        red[(rg * BM + wm0 + i * 8 + fc) * BN + wn0 + j * 8 + fr * 2 + h] = acc[i][j][h];
  __syncthreads();
  double* out = part + (long long)blockIdx.z * k1 * k2;
  for (int e = tid; e < BM * BN; e += 256) {
    const int rr = e / BN, cc = e % BN;
    double s = 0.0;
#pragma unroll
    for (int g = 0; g < RG; ++g) s += red[g * BM * BN + e];
    if (tm0 + rr < k1 && tn0 + cc < k2) out[(long long)(tm0 + rr) * k2 + tn0 + cc] = s;
  }
}

// one warp per output: lanes stride the slabs, fixed shuffle tree (deterministic)
__global__ void gram_finish2_kernel(int k1, int k2, int nslab, const double* __restrict__ part,
                                    double alpha, double beta, double* G, long long grs,
                                    long long gcs, const int* skip) {
  pdl_wait();
  pdl_trigger();  // a small kernel: let the successor's CTAs become resident now
  if (skip && *skip) return;
  const long long e = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= (long long)k1 * k2) return;
  const long long kk = (long long)k1 * k2;
  double s = 0.0;
  for (int q = lane; q < nslab; q += 32) s += part[q * kk + e];
  s = warp_sum(s);
  if (lane == 0) {
    const int r = (int)(e / k2), c = (int)(e % k2);
    double* g = G + r * grs + c * gcs;
    *g = (beta == 0.0) ? alpha * s : fma(alpha, s, beta * *g);
  }
}

static inline bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

template <int BM, int BN, int WM, int WN, int R>
static void gram_go_r(Ctx* c, long long n, int k1, int k2, const double* X, long long ldx,
                      const double* Y, long long ldy, double* part, long long rps, int nslab,
                      bool vec, Skip sk);

template <int BM, int BN, int WM, int WN>
static void gram_go(Ctx* c, long long n, int k1, int k2, const double* X, long long ldx,
                    const double* Y, long long ldy, double* part, long long rps, int nslab,
                    bool vec, Skip sk) {
  constexpr int W = frag_stride(BM + BN);
  // rows per stage: as many as fit three stages in ~110 KB (>= 16)
  constexpr int R0 = (3 * 64 * W * 8 <= 112 * 1024) ? 64 : ((3 * 32 * W * 8 <= 160 * 1024) ? 32 : 16);
  // wide tiles (BN >= 96, the cfg4 / cfg5 deflation shapes): twice the rows per stage
  // where three stages still fit 220 KB — half the block barriers per row, measured at
  // n = 2.1M: 900x100 16.3 -> 15.4 ms, 300x100 5.44 -> 5.15, 600x200 23.9 -> 22.7 (skinny
  // tiles get slower: 180x20 0.67 -> 1.04 ms, so they keep R0); GCG_GRAM_R2=0 disables
  constexpr int R2 = (BN >= 96 && 3 * 2 * R0 * W * 8 <= 220 * 1024) ? 2 * R0 : R0;
  static const bool r2 = !(getenv("GCG_GRAM_R2") && getenv("GCG_GRAM_R2")[0] == '0');
  if (r2 && R2 != R0) {
    gram_go_r<BM, BN, WM, WN, R2>(c, n, k1, k2, X, ldx, Y, ldy, part, rps, nslab, vec, sk);
    return;
  }
  gram_go_r<BM, BN, WM, WN, R0>(c, n, k1, k2, X, ldx, Y, ldy, part, rps, nslab, vec, sk);
}

template <int BM, int BN, int WM, int WN, int R>
static void gram_go_r(Ctx* c, long long n, int k1, int k2, const double* X, long long ldx,
                      const double* Y, long long ldy, double* part, long long rps, int nslab,
                      bool vec, Skip sk) {
  constexpr int W = frag_stride(BM + BN);
  constexpr int RG = 8 / ((BM / WM) * (BN / WN));
  const size_t sm_stage = sizeof(double) * (size_t)kStages * R * W;
  const size_t sm_red = sizeof(double) * (size_t)RG * BM * BN;
  const size_t sm = sm_stage > sm_red ? sm_stage : sm_red;
  dim3 grid((k1 + BM - 1) / BM, (k2 + BN - 1) / BN, nslab);
  // GCG_GRAM_INTER=1: stages dealt round-robin over the slabs (one ascending window over
  // the rows; with GCG_LC_DESC=1 the LinComb that follows starts on this kernel's L2 tail).
  // Measured: -2 % per cfg2 iteration (LinComb 50.9 -> 49.3 ms), nothing at cfg3 / cfg4
  // (basis >> L2); off by default (one contiguous range per slab)
  static const bool inter_on = getenv("GCG_GRAM_INTER") && getenv("GCG_GRAM_INTER")[0] == '1';
  if (inter_on) rps = -1;
  static const bool bulk_on = !(getenv("GCG_GRAM_BULK") && getenv("GCG_GRAM_BULK")[0] == '0');
  // bulk staging needs every row run at the same 16-byte phase: even leading dimensions
  // (a run starting 8 bytes past a boundary is copied from one element earlier)
  if (bulk_on && ldx % 2 == 0 && ldy % 2 == 0) {
    // row segments staged by the bulk-copy engine: one instruction per row and
    // operand per stage instead of one cp.async per 16 bytes
    auto kern = gram_dmma_kernel<BM, BN, WM, WN, R, true, true>;
    kernel_smem((const void*)kern, sm);
    pdl_launch(kern, grid, dim3(256), sm, c->stream, n, k1, k2, X, ldx, Y, ldy, rps, part, sk);
  } else if (vec) {
    auto kern = gram_dmma_kernel<BM, BN, WM, WN, R, true>;
    kernel_smem((const void*)kern, sm);
    pdl_launch(kern, grid, dim3(256), sm, c->stream, n, k1, k2, X, ldx, Y, ldy, rps, part, sk);
  } else {
    auto kern = gram_dmma_kernel<BM, BN, WM, WN, R, false>;
    kernel_smem((const void*)kern, sm);
    pdl_launch(kern, grid, dim3(256), sm, c->stream, n, k1, k2, X, ldx, Y, ldy, rps, part, sk);
  }
}

// Tile shapes: the whole k1 x k2 output in one CTA tile when it is skinny
// (k2 <= 32, k1 <= 256: 8 warps stacked along k1), so X and Y are each read
// once; 64 x 64 tiles (2 x 2 warps, 2 row groups) otherwise.
static int gram_dispatch(Ctx* c, long long n, int k1, int k2, const double* X, long long ldx,
                         const double* Y, long long ldy, double* part, long long rps, int nslab,
                         bool vec, int* bm_out, int* bn_out, Skip sk = Skip{nullptr, nullptr}) {
  const int f1 = (k1 + 63) / 64, f2 = (k2 + 7) / 8;
#define GO(bm, bn, wm, wn)                                                              \
  do {                                                                                \
    *bm_out = bm;                                                                     \
    *bn_out = bn;                                                                     \
    if (part) gram_go<bm, bn, wm, wn>(c, n, k1, k2, X, ldx, Y, ldy, part, rps, nslab, vec, sk); \
    return GCG_OK;                                                                    \
  } while (0)
  if (k1 <= 16 && k2 <= 16) GO(16, 16, 16, 16);
  if (k1 <= 32 && k2 <= 32) GO(32, 32, 32, 32);
  if (k2 <= 32 && k1 <= 256 && (k1 + 31) / 32 % 2 == 1 && k1 > 64) {
    // k1 in (64, 96], (128, 160], (192, 224]: tiles of 96 / 160 / 224 rows (4 warps
    // along M x 2 row groups) instead of the next multiple of 64 — e.g. the 200-row
    // deflation / cross Grams pay 12 % padding instead of 28 %
    const int b = (k1 + 31) / 32;  // 3, 5 or 7
    switch (b * 8 + f2) {
      case 3 * 8 + 1: GO(96, 8, 24, 8);
      case 3 * 8 + 2: GO(96, 16, 24, 16);
      case 3 * 8 + 3: GO(96, 24, 24, 24);
      case 3 * 8 + 4: GO(96, 32, 24, 32);
      case 5 * 8 + 1: GO(160, 8, 40, 8);
      case 5 * 8 + 2: GO(160, 16, 40, 16);
      case 5 * 8 + 3: GO(160, 24, 40, 24);
      case 5 * 8 + 4: GO(160, 32, 40, 32);
      case 7 * 8 + 1: GO(224, 8, 56, 8);
      case 7 * 8 + 2: GO(224, 16, 56, 16);
      case 7 * 8 + 3: GO(224, 24, 56, 24);
      default: GO(224, 32, 56, 32);
    }
  }
  if (k2 <= 32 && k1 <= 256) {
    switch (f1 * 8 + f2) {
      case 1 * 8 + 1: GO(64, 8, 8, 8);
      case 1 * 8 + 2: GO(64, 16, 8, 16);
      case 1 * 8 + 3: GO(64, 24, 8, 24);
      case 1 * 8 + 4: GO(64, 32, 8, 32);
      case 2 * 8 + 1: GO(128, 8, 16, 8);
      case 2 * 8 + 2: GO(128, 16, 16, 16);
      case 2 * 8 + 3: GO(128, 24, 16, 24);
      case 2 * 8 + 4: GO(128, 32, 16, 32);
      case 3 * 8 + 1: GO(192, 8, 24, 8);
      case 3 * 8 + 2: GO(192, 16, 24, 16);
      case 3 * 8 + 3: GO(192, 24, 24, 24);
      case 3 * 8 + 4: GO(192, 32, 24, 32);
      case 4 * 8 + 1: GO(256, 8, 32, 8);
      case 4 * 8 + 2: GO(256, 16, 32, 16);
      case 4 * 8 + 3: GO(256, 24, 32, 24);
      default: GO(256, 32, 32, 32);
    }
  }
  // 128 x 64 tiles (4 x 2 warps, no row-group split: more DMMA per staged element)
  // when they add no padding over 64-row tiles or the N side is narrow; measured
  // 200x200 14.5 vs 10.8 TF/s, 400x40 11.6 vs 9.5, but 160x160 8.6 vs 12.8
  const bool t128 = k1 > 96 && ((k1 + 127) / 128 * 128 == (k1 + 63) / 64 * 64 || k2 <= 64);
  // Wide 160 x 128 tiles (2 x 4 warps of 80 x 32: 40 DMMAs per 14 fragment loads, X read
  // once and Y twice for k2 <= 128; one CTA per SM) unless they pad clearly more than
  // the narrow tile.  Measured at n = 2.1M (scripts/gram_wide.sh): 300x100 12.6 -> 20.9
  // TF/s, 600x200 11.9 -> 21.1, 900x100 12.4 -> 14.5 (before the whole-wave slab count);
  // 200x200 and 500x100 (1.25x the padded area) stay on 128 x 64.
  if (k1 > 128 && k2 > 64) {
    // k2 in (96, 112] (cfg4's bs = 100): 160 x 112 tiles of 4 x 2 warps (40 x 56) pad
    // 12 % instead of 28 %: 900x100 18.2 -> 16.3 ms, 300x100 5.5 -> 5.4 ms at n = 2.1M
    static const char* wide_env = getenv("GCG_GRAM_WIDE");
    static const char* g112 = getenv("GCG_GRAM112");
    const bool n112 = k2 > 96 && k2 <= 112 && !(g112 && g112[0] == '0');
    const long long pw =
        (long long)((k1 + 159) / 160 * 160) * (n112 ? 112 : (k2 + 127) / 128 * 128);
    const int bm = t128 ? 128 : 64;
    const long long pn = (long long)((k1 + bm - 1) / bm * bm) * ((k2 + 63) / 64 * 64);
    const bool wide = wide_env ? wide_env[0] == '1' : 5 * pw < 6 * pn;
    if (wide && n112) GO(160, 112, 40, 56);
    if (wide) GO(160, 128, 80, 32);
  }
  // k1 > 128, k2 in (32, 48] (cfg3's bs = 40 deflation shapes): 160 x 48 tiles of 4 x 2
  // warps (40 x 24) instead of 64-wide ones that pad k2 = 40 by 60 %; at n = 493k:
  // 400x40 1.38 -> 1.00 ms, 320x40 1.04 -> 0.68 ms, 600x40 1.72 -> 1.33 ms
  // (`profiles/r01_tile48.txt`)
  static const char* g48 = getenv("GCG_GRAM48");
  if (!(g48 && g48[0] == '0') && k1 > 128 && k2 > 32 && k2 <= 48) GO(160, 48, 40, 24);
  if (t128) GO(128, 64, 32, 32);
  GO(64, 64, 32, 32);
#undef GO
}

// ---------------------------------------------------------------------------
// Symmetric small Gram X'X, k <= 32 (the SVQB leaf and block Grams with B = I):
// each lane's loads X[row][8f + a] are simultaneously its A fragment (m = a,
// k = row) and its B fragment (k = row, n = a) of column block f, so a warp
// reads every X element once, straight into registers (four 4-row k-steps in
// flight), and issues FN*FN DMMAs per k-step.  Warps own contiguous row
// ranges; the CTA's warp partials are summed in warp order and the CTA
// partials by gram_finish2_kernel — deterministic.
template <int FN>
__global__ void __launch_bounds__(256) gram_sym_kernel(long long n, int k,
                                                       const double* __restrict__ X, long long ldx,
                                                       long long rps, double* part, Skip skip) {
  pdl_wait();  // launched with programmatic stream serialization: predecessor complete from here on
  if (skip_now(skip)) return;
  constexpr int U = 4;  // k-steps in flight
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int fa = lane >> 2, fc = lane & 3;
  const long long c0 = (long long)blockIdx.x * rps;
  const long long c1 = min(n, c0 + rps);
  const long long wr = ((c1 - c0 + 7) / 8 + 3) / 4 * 4;  // rows per warp, multiple of 4
  const long long r0 = c0 + warp * wr;
  const long long r1 = min(c1, r0 + wr);
  double acc[FN][FN][2];
#pragma unroll
  for (int i = 0; i < FN; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (long long r = r0; r < r1; r += 4 * U) {
    double v[U][FN];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long row = r + 4 * u + fc;
      const bool ok = row < r1;
#pragma unroll
      for (int f = 0; f < FN; ++f) {
        const int col = 8 * f + fa;
        v[u][f] = (ok && col < k) ? X[row * ldx + col] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < FN; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], v[u][i], v[u][j]);
  }
  pdl_trigger();  // late: the finish kernel launches while this grid drains
  // warp partials: warps 4..7 park theirs, warps 0..3 add them (fixed pairing), then
  // the four pair sums are added in order
  constexpr int KW = 8 * FN;
  __shared__ double red[4][KW * KW];
  if (warp >= 4) {
#pragma unroll
    for (int i = 0; i < FN; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          red[warp - 4][(8 * i + fa) * KW + 8 * j + 2 * fc + h] = acc[i][j][h];
  }
  __syncthreads();
  if (warp < 4) {
#pragma unroll
    for (int i = 0; i < FN; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double& t = red[warp][(8 * i + fa) * KW + 8 * j + 2 * fc + h];
          t = acc[i][j][h] + t;
        }
  }
  __syncthreads();
  double* out = part + (long long)blockIdx.x * k * k;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int a = e / k, b = e % k;
    out[e] = ((red[0][a * KW + b] + red[1][a * KW + b]) + red[2][a * KW + b]) + red[3][a * KW + b];
  }
}

static int gram_sym_launch(Ctx* c, long long n, int k, const double* X, long long ldx,
                           double alpha, double beta, double* G, long long grs, long long gcs) {
  long long nslab = 2LL * c->num_sms;
  const long long max_slab = (n + 1023) / 1024;
  if (nslab > max_slab) nslab = max_slab;
  if (nslab < 1) nslab = 1;
  long long rps = (n + nslab - 1) / nslab;
  rps = (rps + 31) / 32 * 32;
  nslab = (n + rps - 1) / rps;
  if (nslab < 1) nslab = 1;
  GCG_TRY(ensure(c->partials, sizeof(double) * (size_t)nslab * k * k));
  double* part = (double*)c->partials.ptr;
  const int ps = prof_start(c, PROF_GRAM, 8.0 * n * k);
  const Skip sk = skip_of(c, ps);
  switch ((k + 7) / 8) {
    case 1: pdl_launch(gram_sym_kernel<1>, dim3((unsigned)nslab), dim3(256), 0, c->stream, n, k, X, ldx, rps, part, sk); break;
    case 2: pdl_launch(gram_sym_kernel<2>, dim3((unsigned)nslab), dim3(256), 0, c->stream, n, k, X, ldx, rps, part, sk); break;
    case 3: pdl_launch(gram_sym_kernel<3>, dim3((unsigned)nslab), dim3(256), 0, c->stream, n, k, X, ldx, rps, part, sk); break;
    default: pdl_launch(gram_sym_kernel<4>, dim3((unsigned)nslab), dim3(256), 0, c->stream, n, k, X, ldx, rps, part, sk); break;
  }
  prof_stop(c, ps);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  const long long outs = (long long)k * k;
  pdl_launch(gram_finish2_kernel, dim3((unsigned)((outs * 32 + 255) / 256)), dim3(256), 0, c->stream, k, k,
             (int)nslab, (const double*)part, alpha, beta, G, grs, gcs, c->skip);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

int gram_launch(Ctx* c, long long n, int k1, int k2, const double* X, long long ldx,
                const double* Y, long long ldy, double alpha, double beta, double* G,
                long long grs, long long gcs) {
  if (k1 <= 0 || k2 <= 0) return GCG_OK;
  static const bool sym_on = !(getenv("GCG_GRAM_SYM") && getenv("GCG_GRAM_SYM")[0] == '0');
  if (sym_on && X == Y && ldx == ldy && k1 == k2 && k1 <= 32 && n >= 4096)
    return gram_sym_launch(c, n, k1, X, ldx, alpha, beta, G, grs, gcs);
  // skinny on the left: compute G' = Y'X with roles swapped (write through swapped strides)
  if (k1 <= 32 && k2 > 32 && k2 <= 256)
    return gram_launch(c, n, k2, k1, Y, ldy, X, ldx, alpha, beta, G, gcs, grs);
  int BM = 0, BN = 0;
  gram_dispatch(c, n, k1, k2, X, ldx, Y, ldy, nullptr, 0, 0, false, &BM, &BN);
  const long long tiles = (long long)((k1 + BM - 1) / BM) * ((k2 + BN - 1) / BN);
  // ~2 CTAs per SM in total (whole waves: rounded down), slabs a multiple of 64 rows
  long long nslab = (2LL * c->num_sms) / tiles;
  const long long max_slab = (n + 255) / 256;
  if (nslab > max_slab) nslab = max_slab;
  if (nslab < 1) nslab = 1;
  if (nslab > 65535) nslab = 65535;
  long long rps = (n + nslab - 1) / nslab;
  rps = (rps + 63) / 64 * 64;
  nslab = (n + rps - 1) / rps;
  if (nslab < 1) nslab = 1;
  GCG_TRY(ensure(c->partials, sizeof(double) * (size_t)nslab * k1 * k2));
  double* part = (double*)c->partials.ptr;
  const bool vec = (ldx % 2 == 0) && (ldy % 2 == 0) && al16(X) && al16(Y);
  const int ps = prof_start(c, PROF_GRAM, 8.0 * n * (X == Y ? k1 : k1 + k2));
  gram_dispatch(c, n, k1, k2, X, ldx, Y, ldy, part, rps, (int)nslab, vec, &BM, &BN,
                skip_of(c, ps));
  prof_stop(c, ps);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  const long long outs = (long long)k1 * k2;
  pdl_launch(gram_finish2_kernel, dim3((unsigned)((outs * 32 + 255) / 256)), dim3(256), 0, c->stream, k1, k2,
             (int)nslab, (const double*)part, alpha, beta, G, grs, gcs, c->skip);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

// ---------------------------------------------------------------------------
// LinComb  Y = alpha X C + beta Y: CTA tile BM rows x BN columns, warp tile
// WM x WN, K (= m) in BK = 16 chunks through the cp.async ring.

template <int BM, int BN, int WM, int WN, bool VEC16, bool BULK = false>
__global__ void __launch_bounds__(256) lincomb_dmma_kernel(long long n, int m, int d,
                                                           double alpha,
                                                           const double* X,
                                                           long long ldx,
                                                           const double* __restrict__ C,
                                                           long long ldc, double beta, double* Y,
                                                           long long ldy, Skip skip) {
  pdl_wait();  // launched with programmatic stream serialization: predecessor complete from here on
  if (skip_now(skip)) return;
  constexpr int BK = 16;
  constexpr int FM = WM / 8, FN = WN / 8;
  static_assert((BM / WM) * (BN / WN) == 8, "8 warps");
  constexpr int XW = frag_stride(BK);  // 20
  constexpr int CW = frag_stride(BN);
  constexpr int XS = BM * XW, CS = BK * CW;
  constexpr int V = VEC16 ? 2 : 1;
  extern __shared__ __align__(16) double sml[];
  double* xs = sml;
  double* cs = sml + kStages * XS;
  const long long r0 = (long long)blockIdx.x * BM;
  const int c0 = blockIdx.y * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / (BN / WN)) * WM, wn0 = (warp % (BN / WN)) * WN;
  const int nk = (m + BK - 1) / BK;
  const int vc = min(BN, d - c0);
  const int fr = lane & 3, fc = lane >> 2;
  const int xo = BULK ? (int)(((uintptr_t)X >> 3) & 1) : 0;  // X runs' 8-byte phase

  __shared__ __align__(8) unsigned long long mbar[kStages];
  if constexpr (BULK) {
    if (tid == 0) {
      for (int s = 0; s < kStages; ++s) mbar_init(&mbar[s]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  auto load = [&](int kb, int st) {
    const int k0 = kb * BK;
    const int vk = min(BK, m - k0);
    if constexpr (BULK) {
      // bulk copies: threads 0..BM-1 one X row chunk each, threads BM.. one C row each;
      // a K tail zero-fills the unused X columns and C rows (stale shared memory could
      // hold non-finite bit patterns), an odd trailing element is a plain store
      // (rows starting 8 bytes past a 16-byte boundary are copied from one element
      // earlier and sit at +1 in shared memory, see xo)
      const int ex = vk + xo;
      const int bk = (ex * 8) & ~15, bc = (vc * 8) & ~15;
      const int nr = (int)min((long long)BM, n - r0);
      if (tid == 0) mbar_expect(&mbar[st], (unsigned)(nr * bk + vk * bc));
      double* xd = xs + st * XS;
      double* cd = cs + st * CS;
      if (tid < nr) {
        const double* src = X + (r0 + tid) * ldx + k0 - xo;
        if (bk) bulk_g2s(xd + tid * XW, src, bk, &mbar[st]);
        if (ex & 1) xd[tid * XW + ex - 1] = src[ex - 1];
        for (int e = vk; e < BK; ++e) xd[tid * XW + xo + e] = 0.0;
      }
      const int kk = BM < 256 ? tid - BM : tid;  // the C row this thread stages
      if (kk >= 0 && kk < vk) {
        const double* src = C + (long long)(k0 + kk) * ldc + c0;
        if (bc) bulk_g2s(cd + kk * CW, src, bc, &mbar[st]);
        if (vc & 1) cd[kk * CW + vc - 1] = src[vc - 1];
      }
      for (int e = tid; e < (BK - vk) * CW; e += 256) cd[vk * CW + e] = 0.0;
      return;
    }
    constexpr int PX = BK / V;
    for (int e = tid; e < BM * PX; e += 256) {
      const int rr = e / PX, cc = e % PX;
      const long long row = r0 + rr;
      const bool ok = row < n;
      stage_elems<VEC16>(xs + st * XS + rr * XW, X + (ok ? row : 0) * ldx + k0, cc, ok ? vk : 0,
                         X);
    }
    for (int e = tid; e < BK * BN; e += 256) {
      const int kk = e / BN, cc = e % BN;
      const bool ok = kk < vk && cc < vc;
      cp_async8(cs + st * CS + kk * CW + cc, ok ? C + (long long)(k0 + kk) * ldc + c0 + cc : C,
                ok);
    }
  };

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) load(s, s);
    cp_commit();
  }
  for (int kb = 0; kb < nk; ++kb) {
    if constexpr (BULK) mbar_wait(&mbar[kb % kStages], (unsigned)((kb / kStages) & 1));
    else cp_wait<kStages - 2>();
    __syncthreads();
    if (kb + kStages - 1 < nk) load(kb + kStages - 1, (kb + kStages - 1) % kStages);
    cp_commit();
    const double* xb = xs + (kb % kStages) * XS;
    const double* cb = cs + (kb % kStages) * CS;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double a[FM], b[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) a[i] = xb[(wm0 + i * 8 + fc) * XW + ks * 4 + fr + xo];
#pragma unroll
      for (int j = 0; j < FN; ++j) b[j] = cb[(ks * 4 + fr) * CW + wn0 + j * 8 + fc];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_wait<0>();
#pragma unroll
  for (int i = 0; i < FM; ++i) {
    const long long row = r0 + wm0 + i * 8 + fc;
    if (row >= n) continue;
#pragma unroll
    for (int j = 0; j < FN; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = c0 + wn0 + j * 8 + fr * 2 + h;
        if (col >= d) continue;
        double* y = Y + row * ldy + col;
        *y = (beta == 0.0) ? alpha * acc[i][j][h] : fma(alpha, acc[i][j][h], beta * *y);
      }
    }
  }
}

template <int BM, int BN, int WM, int WN>
static void lincomb_go(Ctx* c, long long n, int m, int d, double alpha, const double* X,
                       long long ldx, const double* C, long long ldc, double beta, double* Y,
                       long long ldy, bool vec, Skip sk) {
  const size_t sm =
      sizeof(double) * (size_t)kStages * (BM * frag_stride(16) + 16 * frag_stride(BN));
  dim3 grid((unsigned)((n + BM - 1) / BM), (d + BN - 1) / BN);
  static const bool bulk_on = !(getenv("GCG_LINCOMB_BULK") && getenv("GCG_LINCOMB_BULK")[0] == '0');
  if (BM < 256 && bulk_on && ldx % 2 == 0 && al16(C) && ldc % 2 == 0) {
    // X row chunks and C rows staged by the bulk-copy engine (one instruction per row)
    auto kern = lincomb_dmma_kernel<BM, BN, WM, WN, true, true>;
    kernel_smem((const void*)kern, sm);
    pdl_launch(kern, grid, dim3(256), sm, c->stream, n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy, sk);
  } else if (vec) {
    auto kern = lincomb_dmma_kernel<BM, BN, WM, WN, true>;
    kernel_smem((const void*)kern, sm);
    pdl_launch(kern, grid, dim3(256), sm, c->stream, n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy, sk);
  } else {
    auto kern = lincomb_dmma_kernel<BM, BN, WM, WN, false>;
    kernel_smem((const void*)kern, sm);
    pdl_launch(kern, grid, dim3(256), sm, c->stream, n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy, sk);
  }
}

// ---------------------------------------------------------------------------
// Tall-skinny LinComb, d <= 64 (W -= [X P] R in the deflation, the Ritz-vector
// chunks of the convergence test, momentum): Y = alpha X C + beta Y.
//
// The m x d coefficient block stays resident in shared memory as DMMA B
// fragments; each warp streams 8*FM rows of X from HBM straight into DMMA A
// fragments — one VEC-wide load per lane feeds VEC k-substeps, because the k
// index inside every 4*VEC chunk is permuted (lane c of a fragment takes
// k = 4*VEC*chunk + c*VEC + s at substep s), identically for the B fragments —
// and keeps the next chunk's loads in flight while multiplying the current one.
// No X staging through shared memory, no block barrier in the main loop: warps
// are independent, so the X stream is limited only by loads in flight, and a
// warp writes only rows it alone has read (in-place use is safe for any d).
__host__ __device__ constexpr int ts_cstride(int fn, int vec) {
  // >= 8*fn, and vec*stride == 8 (mod 16) so the two k-rows a fragment load pairs
  // up fall in opposite bank halves
  int s = 8 * fn;
  while ((vec * s) % 16 != 8) ++s;
  return s;
}

template <int VEC>
__device__ __forceinline__ void ts_load(double* v, const double* p, int valid) {
  if (valid >= VEC) {
    if constexpr (VEC == 4) {
      const double4 t = *reinterpret_cast<const double4*>(p);
      v[0] = t.x;
      v[1] = t.y;
      v[2] = t.z;
      v[3] = t.w;
    } else if constexpr (VEC == 2) {
      const double2 t = *reinterpret_cast<const double2*>(p);
      v[0] = t.x;
      v[1] = t.y;
    } else {
      v[0] = *p;
    }
  } else {
#pragma unroll
    for (int s = 0; s < VEC; ++s) v[s] = s < valid ? p[s] : 0.0;
  }
}

template <int FM, int FN, int VEC>
__global__ void __launch_bounds__(128) lincomb_ts_kernel(long long n, int m, int d, double alpha,
                                                         const double* X, long long ldx,
                                                         const double* __restrict__ C,
                                                         long long ldc, double beta, double* Y,
                                                         long long ldy, Skip skip) {
  pdl_wait();  // launched with programmatic stream serialization: predecessor complete from here on
  if (skip_now(skip)) return;
  constexpr int KC = 4 * VEC;
  constexpr int CW = ts_cstride(FN, VEC);
  extern __shared__ __align__(16) double cs[];
  const int mp = (m + KC - 1) / KC * KC;
  for (int e = threadIdx.x; e < mp * 8 * FN; e += blockDim.x) {
    const int k = e / (8 * FN), j = e % (8 * FN);
    cs[k * CW + j] = (k < m && j < d) ? C[(long long)k * ldc + j] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int fa = lane >> 2, fc = lane & 3;
  const long long ntiles = (n + 8 * FM - 1) / (8 * FM);
  const long long wstride = (long long)gridDim.x * (blockDim.x >> 5);

  for (long long t = (long long)blockIdx.x * (blockDim.x >> 5) + warp; t < ntiles; t += wstride) {
    if (t + wstride >= ntiles) pdl_trigger();  // this warp's last tile: the successor may launch
    // tiles from the last rows down (c_ts_desc): the Gram before this LinComb walked the
    // same X upwards, its last rows are still in L2
    const long long r0 = (c_ts_desc ? ntiles - 1 - t : t) * 8 * FM;
    const double* xr[FM];
    bool rok[FM];
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const long long row = r0 + i * 8 + fa;
      rok[i] = row < n;
      xr[i] = X + (rok[i] ? row : 0) * ldx;
    }
    auto load = [&](double (*v)[VEC], int kc) {
      const int k = kc + fc * VEC;
      const int valid = min(VEC, m - k);
#pragma unroll
      for (int i = 0; i < FM; ++i) ts_load<VEC>(v[i], xr[i] + k, rok[i] ? valid : 0);
    };
    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    auto compute = [&](double (*v)[VEC], int kc) {
#pragma unroll
      for (int s = 0; s < VEC; ++s) {
        double b[FN];
        const double* crow = cs + (kc + fc * VEC + s) * CW + fa;
#pragma unroll
        for (int j = 0; j < FN; ++j) b[j] = crow[j * 8];
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], v[i][s], b[j]);
      }
    };
    double va[FM][VEC], vb[FM][VEC];
    load(va, 0);
    for (int kc = 0; kc < mp; kc += 2 * KC) {
      const bool more = kc + KC < mp;
      if (more) load(vb, kc + KC);
      compute(va, kc);
      if (more) {
        if (kc + 2 * KC < mp) load(va, kc + 2 * KC);
        compute(vb, kc + KC);
      }
    }
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const long long row = r0 + i * 8 + fa;
      if (row >= n) continue;
#pragma unroll
      for (int j = 0; j < FN; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = j * 8 + fc * 2 + h;
          if (col >= d) continue;
          double* y = Y + row * ldy + col;
          *y = (beta == 0.0) ? alpha * acc[i][j][h] : fma(alpha, acc[i][j][h], beta * *y);
        }
      }
    }
  }
}

template <int FM, int FN, int VEC>
static void lincomb_ts_go(Ctx* c, long long n, int m, int d, double alpha, const double* X,
                          long long ldx, const double* C, long long ldc, double beta, double* Y,
                          long long ldy, Skip sk) {
  auto kern = lincomb_ts_kernel<FM, FN, VEC>;
  const int mp = (m + 4 * VEC - 1) / (4 * VEC) * (4 * VEC);
  const size_t sm = sizeof(double) * (size_t)mp * ts_cstride(FN, VEC);
  kernel_smem((const void*)kern, sm);
  const int occ = kernel_occupancy((const void*)kern, 128, sm);
  const long long ntiles = (n + 8 * FM - 1) / (8 * FM);
  long long grid = (ntiles + 3) / 4;
  const long long cap = (long long)occ * c->num_sms;
  if (grid > cap) grid = cap;
  static const bool desc_set = [] {
    const int v = getenv("GCG_LC_DESC") && getenv("GCG_LC_DESC")[0] == '1';
    return cudaMemcpyToSymbol(c_ts_desc, &v, sizeof(int)) == cudaSuccess;
  }();
  (void)desc_set;
  pdl_launch(kern, dim3((unsigned)grid), dim3(128), sm, c->stream, n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy, sk);
}

template <int VEC>
static bool lincomb_ts_dispatch(Ctx* c, long long n, int m, int d, double alpha, const double* X,
                                long long ldx, const double* C, long long ldc, double beta,
                                double* Y, long long ldy, Skip sk) {
  const int fn = (d + 7) / 8;
  const size_t sm = sizeof(double) * (size_t)((m + 4 * VEC - 1) / (4 * VEC) * (4 * VEC)) *
                    ts_cstride(fn, VEC);
  if (fn > 8 || sm > 96 * 1024) return false;
#define TS(fm, fnn) lincomb_ts_go<fm, fnn, VEC>(c, n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy, sk)
  static const int fmx = getenv("GCG_TS_FM") ? atoi(getenv("GCG_TS_FM")) : 0;
#define TSF(fnn, dflt)                    \
  {                                       \
    const int f = fmx ? fmx : (dflt);     \
    if (f >= 8) TS(8, fnn);               \
    else if (f >= 4) TS(4, fnn);          \
    else if (f >= 2) TS(2, fnn);          \
    else TS(1, fnn);                      \
  }
  switch (fn) {
    // row blocks per warp: 4 (32 rows) up to d = 40 — measured best at n = 262144
    // (200x20: 115 us vs 151 us with 2); wider d keeps the accumulators in registers
    case 1: TSF(1, 4); break;
    case 2: TSF(2, 4); break;
    case 3: TSF(3, 4); break;
    case 4: TSF(4, 4); break;
    case 5: TSF(5, 4); break;
    case 6: TSF(6, 2); break;
    case 7: TSF(7, 2); break;
    default: TSF(8, 2); break;
  }
#undef TSF
#undef TS
  return true;
}

int lincomb_launch(Ctx* c, long long n, int m, int d, double alpha, const double* X,
                   long long ldx, const double* C, long long ldc, double beta, double* Y,
                   long long ldy) {
  if (n <= 0 || d <= 0) return GCG_OK;
  {
    // In-place use (Y inside the rows of X: [X|P] <- basis [coeffs|phat]) is safe
    // only when one CTA owns all d output columns of its rows (grid.y == 1): every
    // X row tile is fully staged (cp.async + barrier) before that CTA stores it.
    const double* xe = X + (n - 1) * ldx + m;
    const double* ye = Y + (n - 1) * ldy + d;
    if ((Y < xe) && (X < ye)) {  // address hulls meet: compare on the row lattice
      if (ldx != ldy) return GCG_ERR_ARG;
      const long long off = Y - X;
      const long long r = off >= 0 ? off / ldx : -((-off + ldx - 1) / ldx);
      const long long co = off - r * ldx;  // Y row i starts at column co of X row i + r
      const bool same = co < m;            // hits X row i + r
      const bool next = co + d > ldx;      // wraps into X row i + r + 1
      if (next || (same && (r != 0 || d > 256))) return GCG_ERR_ARG;
    }
  }
  const int ps =
      prof_start(c, PROF_LINCOMB, 8.0 * n * (m + d) + (beta != 0.0 ? 8.0 * n * d : 0.0));
  const Skip sk = skip_of(c, ps);
  static const bool ts_on = !(getenv("GCG_LINCOMB_TS") && getenv("GCG_LINCOMB_TS")[0] == '0');
  if (ts_on && d <= 64) {
    bool done;
    if (ldx % 4 == 0 && ((uintptr_t)X & 31) == 0)
      done = lincomb_ts_dispatch<4>(c, n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy, sk);
    else if (ldx % 2 == 0 && al16(X))
      done = lincomb_ts_dispatch<2>(c, n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy, sk);
    else
      done = lincomb_ts_dispatch<1>(c, n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy, sk);
    if (done) {
      prof_stop(c, ps);
      ++g_launches;
      GCG_CHECK_LAUNCH();
      return GCG_OK;
    }
  }
  const bool vec = (ldx % 2 == 0) && al16(X);
  // One column tile covers all d <= 256 columns, so X is streamed exactly once:
  // d <= 64: 8 warps stacked along rows (BM = 256, warp tile 32 x BN);
  // d  > 64: 2 x 4 warps (BM = 64, warp tile 32 x BN/4).
#define LC(bm, bn, wm, wn) lincomb_go<bm, bn, wm, wn>(c, n, m, d, alpha, X, ldx, C, ldc, beta, Y, ldy, vec, sk)
  static const bool lc112 = !(getenv("GCG_LC112") && getenv("GCG_LC112")[0] == '0');
  if (d <= 8) LC(256, 8, 32, 8);
  else if (d <= 16) LC(256, 16, 32, 16);
  else if (d <= 24) LC(256, 24, 32, 24);
  else if (d <= 32) LC(256, 32, 32, 32);
  else if (d <= 48) LC(256, 48, 32, 48);
  else if (d <= 64) LC(256, 64, 32, 64);
  else if (d <= 96) LC(64, 96, 32, 24);
  // d in (96, 112] (cfg4's bs = 100): 4 x 2 warps of 16 x 56 — 12 % padding instead of
  // the 128-wide tile's 28 %: 300x100 5.50 -> 4.33 ms, 900x100 15.4 -> 12.5 ms at n = 2.1M
  // (29-30 TF/s; a 128 x 112 tile of 32 x 56 warps was slower, 6.1 ms)
  else if (d <= 112 && lc112)
    LC(64, 112, 16, 56);
  else if (d <= 128) LC(64, 128, 32, 32);
  else if (d <= 160) LC(64, 160, 32, 40);
  else if (d <= 192) LC(64, 192, 32, 48);
  // d in (192, 224] (cfg5's bs = 200): 224-wide tile, 12 instead of 22 % padding —
  // n = 2.1M, 600x200 22.5 -> 20.4 ms, 200x200 8.4 -> 7.8 ms.  (A 128 x 112 tile of
  // 4 x 2 warps of 32 x 56 for d in (96, 112] measured slower than 64 x 128.)
  else if (d <= 224) LC(64, 224, 32, 56);
  else LC(64, 256, 32, 64);
#undef LC
  prof_stop(c, ps);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  return GCG_OK;
}

}  // namespace gcg

// MatDotMultiVec on B200: fp64 CSR x row-major multivector (SpMM).
//
// Reference: CsrOperator.apply (operators.py:103-111) -> kernels.csr_matvec
// (_cy.pyx:11-23: column-by-column scalar CSR loop) and ShiftedOperator.apply
// (operators.py:149-156: A x - theta (B x or x)).
//
// B200 design.  X is row-major, so the k values a nonzero (i, j) needs are one
// contiguous run X[j*ldx : j*ldx+k].  A group of LPR lanes owns one row and
// reads that run with the widest aligned vector loads (32-byte LDG.256 when
// rows are 4-double aligned, else 16 or 8 bytes), NV column chunks per lane;
// LPR is any 1..32 chosen so the groups tile the row and the warp with the
// least idle lanes (k = 20: five lanes x 32 B per row, six rows per warp), so
// one row gather is one instruction touching the two 128-byte lines it spans.
// The row's (column index, value) stream is loaded once, cooperatively (two
// nonzeros per lane, 12 B/nnz from HBM), and broadcast inside the group with
// shuffles.
//
// At the BASELINE shapes the kernel is latency-bound (a row is a 3-deep chain:
// row pointer -> index/value -> X gathers), so it is software-pipelined: while
// a warp gathers X for its current rows, the index/value chunk of its next rows
// and the row pointers of the rows after those are already in flight, leaving
// only the X gathers on the critical path.
//
// The epilogue fuses the shifted-operator term (gamma*Z, Z = X for A - theta*I),
// an axpby with a second input (beta*Yin, used for r = rhs - op x) and an
// optional per-column dot product reduced deterministically (p'q and ||r||^2
// for block CG), so CG never makes a separate pass for them.  When Z (and W)
// is X itself the row's own values come from the diagonal gather already in
// registers instead of a second read; the epilogue streams are vectorised.
//
// Roofline: HBM.  Algorithmic bytes per launch = 12*nnz + 4*(n+1) + 16*n*k
// (+8*n*k per extra epilogue stream); flops = 2*nnz*k.

#include <limits.h>
#include <stdlib.h>

#include <cub/block/block_radix_sort.cuh>
#include <vector>

#include "async.cuh"
#include "cgstate.cuh"
#include "common.cuh"

namespace gcg {

extern int64_t g_launches;

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
  int lpr, gpw;    // lanes per row, rows per warp step
  int vepi;        // epilogue streams VEC-aligned
  long long rpc;   // > 0: rows per CTA (contiguous ranges); 0: grid-stride
  const double* __restrict__ W;
  long long ldw;
  double* partials;   // [gridDim.x][pld] (+ this pass' column offset)
  int pld;
  const int* skip;    // device flag: nonzero -> kernel is a no-op (CG early exit)
  int* prof_skipped;  // profiling: set when the launch was a no-op
  int c0;             // first column of this pass (CG mode: index of the per-column state)
  int cg_prefetch;    // CG mode: L2-prefetch the next row step's p, q, x
  int stages;         // staged CG sweep (CGM 3): ring depth per warp
  unsigned stage_bytes;  // ... and bytes per stage and stream (a warp step's rows, 128-aligned)
};

template <int VEC>
struct VecT;
template <>
struct VecT<1> {
  static __device__ __forceinline__ void ld_stream(const double* p, double* o) {
    long long a;
    asm volatile("ld.global.L1::no_allocate.b64 %0, [%1];" : "=l"(a) : "l"(p) : "memory");
    o[0] = __longlong_as_double(a);
  }
  static __device__ __forceinline__ void load(const double* p, double* o) { o[0] = __ldg(p); }
  static __device__ __forceinline__ void ld(const double* p, double* o) { o[0] = *p; }
  static __device__ __forceinline__ void st(double* p, const double* o) { *p = o[0]; }
};
template <>
struct VecT<2> {
  static __device__ __forceinline__ void ld_stream(const double* p, double* o) {
    long long a, b;
    asm volatile("ld.global.L1::no_allocate.v2.b64 {%0,%1}, [%2];"
                 : "=l"(a), "=l"(b)
                 : "l"(p)
                 : "memory");
    o[0] = __longlong_as_double(a);
    o[1] = __longlong_as_double(b);
  }
  static __device__ __forceinline__ void load(const double* p, double* o) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = v.x;
    o[1] = v.y;
  }
  static __device__ __forceinline__ void ld(const double* p, double* o) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    o[0] = v.x;
    o[1] = v.y;
  }
  static __device__ __forceinline__ void st(double* p, const double* o) {
    *reinterpret_cast<double2*>(p) = make_double2(o[0], o[1]);
  }
};
// 32-byte accesses: a 20-column row is 5 lanes.  Explicit 256-bit PTX vectors —
// a double4 dereference is emitted as two LDG.E.128 whenever ptxas cannot prove
// the 32-byte alignment from the address arithmetic (the gathers' row pointers),
// and two 16-byte halves of each 32-byte sector double the L1 sector traffic.
template <>
struct VecT<4> {
  static __device__ __forceinline__ void load(const double* p, double* o) {
    long long a, b, c, d;
    asm("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];"
        : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
        : "l"(p));
    o[0] = __longlong_as_double(a);
    o[1] = __longlong_as_double(b);
    o[2] = __longlong_as_double(c);
    o[3] = __longlong_as_double(d);
  }
  static __device__ __forceinline__ void ld(const double* p, double* o) {
    long long a, b, c, d;
    asm volatile("ld.global.v4.b64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p)
                 : "memory");
    o[0] = __longlong_as_double(a);
    o[1] = __longlong_as_double(b);
    o[2] = __longlong_as_double(c);
    o[3] = __longlong_as_double(d);
  }
  // streaming own-row load that does not allocate in L1 (keeps L1 for the gathers)
  static __device__ __forceinline__ void ld_stream(const double* p, double* o) {
    long long a, b, c, d;
    asm volatile("ld.global.L1::no_allocate.v4.b64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p)
                 : "memory");
    o[0] = __longlong_as_double(a);
    o[1] = __longlong_as_double(b);
    o[2] = __longlong_as_double(c);
    o[3] = __longlong_as_double(d);
  }
  static __device__ __forceinline__ void st(double* p, const double* o) {
    asm volatile("st.global.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(__double_as_longlong(o[0])),
                 "l"(__double_as_longlong(o[1])), "l"(__double_as_longlong(o[2])),
                 "l"(__double_as_longlong(o[3]))
                 : "memory");
  }
};

constexpr int kSpmmThreads = 256;
constexpr int kSpmmMaxPass = 256;
constexpr int kSpmmMaxSlots = 8;  // NV * VEC
constexpr int kCgMaxStages = 4;   // staged CG sweep: deepest per-warp ring
// resident CTAs per SM by per-lane accumulator width (<= 64 registers at 4)
__host__ __device__ constexpr int spmm_min_blocks(int doubles) {
  return doubles > 0 ? 4 : 4;  // every shape: 64 registers, one grid size
}

// CG = true: the fused block-CG sweep (cgstate.cuh CgSweep; X is the residual block
// r, dense ld = cg.k).  Prologue: every CTA reduces the previous r-update's ||r||^2
// partials in fixed order and takes the per-column decisions of cg.py:86-96 (stop
// test, beta); CTA 0 publishes them.  Epilogue, from own-row values only:
// x += alpha p (the previous sweep's deferred x-update), p = r + beta p,
// q = (A + shift) r + beta q  ( = (A + shift) p, the Chronopoulos-Gear recurrence:
// no second gather of p), and the p'q partials for the next r-update.
// CGM: 0 = plain SpMM, 1 = CG sweep at 4 CTAs / SM (64 registers), 2 = CG sweep at
// 3 CTAs / SM (80 registers: the fused epilogue's values no longer spill the gather
// pipeline's state), 3 = CGM 2 with the own-row streams p, q, x staged through shared
// memory by the bulk copy engine: every warp step's rows are one contiguous run per
// stream (dense ld = k), so each warp keeps a ring of a.stages steps in flight — one
// cp.async.bulk per stream and step, completion on the warp's mbarrier — and the only
// global loads left on a step's critical path are the gathers of r.
template <int VEC, int NV, bool SELF, int CGM>
__global__ void __launch_bounds__(kSpmmThreads, CGM >= 2 ? 3 : spmm_min_blocks(VEC* NV))
    spmm_csr_kernel(SpmmArgs a, CgSweep cg) {
  constexpr bool CG = CGM != 0;
  constexpr bool STG = CGM == 3;
  pdl_wait();
  if constexpr (CG) {
    if (*cg.s.skip1) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        *cg.s.skip2 = 1;  // propagate: the r-update of this sweep is a no-op too
        if (a.prof_skipped) *a.prof_skipped = 1;
      }
      return;
    }
  } else if (a.skip != nullptr && *a.skip) {
    if (a.prof_skipped && blockIdx.x == 0 && threadIdx.x == 0) *a.prof_skipped = 1;
    return;
  }
  // gathers in flight per batch: <= 16 doubles of X per lane, at most 4 nonzeros
  constexpr int UB = 16 / (NV * VEC);
  constexpr int U = UB >= 4 ? 4 : (UB >= 2 ? 2 : 1);
  constexpr int NW = kSpmmThreads / 32;
  constexpr unsigned FULL = 0xffffffffu;
  const int LPR = a.lpr, G = a.gpw;  // lanes per row (any 1..32), rows per warp step
  const int CH = 2 * LPR;            // nonzeros per index/value chunk (2 per lane)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g0 = lane / LPR;
  const bool active = g0 < G;  // lanes past G*LPR mirror the last group, never store
  const int g = active ? g0 : G - 1;
  const int sub = lane - g0 * LPR;
  const int gbase = g * LPR;
  // rows: contiguous per CTA (a.rpc > 0: stencil neighbours i +- 1, i +- nx are
  // gathered by the same SM and hit L1) or interleaved grid-stride
  long long rb, rend, stride;
  if (a.rpc > 0) {
    rb = (long long)blockIdx.x * a.rpc + (long long)warp * G;
    rend = min(a.n, (long long)(blockIdx.x + 1) * a.rpc);
    stride = (long long)NW * G;
  } else {
    rb = ((long long)blockIdx.x * NW + warp) * G;
    rend = a.n;
    stride = (long long)gridDim.x * NW * G;
  }
  const int k = a.k;

  // per-lane dot accumulators live in shared memory ([warp][slot][lane]: each
  // lane owns its column slots), keeping registers for gathers in flight
  // (STG: both live in the dynamic staging buffer once the row loop is done)
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  // sdot[warp] (the warp's per-column sums) reuses sacc[warp]'s 2 KB: a warp reads all its
  // slots into registers before it writes its sums
  static_assert(kSpmmMaxSlots * 32 == kSpmmMaxPass, "sdot aliases sacc per warp");
  __shared__ double sacc_st[STG ? 1 : NW][kSpmmMaxSlots][32];
  double(*sacc)[kSpmmMaxSlots][32] = sacc_st;
  if constexpr (STG) sacc = reinterpret_cast<double(*)[kSpmmMaxSlots][32]>(dyn_smem);
  double(*sdot)[kSpmmMaxPass] = reinterpret_cast<double(*)[kSpmmMaxPass]>(sacc);
  if (!CG && a.dot_mode) {
#pragma unroll
    for (int q = 0; q < NV * VEC; ++q) sacc[warp][q][lane] = 0.0;
  }
  // STG: per-warp ring of a.stages stages x {p, q, x} x a.stage_bytes, one mbarrier per stage
  __shared__ unsigned long long stg_bar[STG ? NW : 1][STG ? kCgMaxStages : 1];
  unsigned char* stg_buf = nullptr;
  const bool stg_on = STG && !cg.first;
  auto stg_issue = [&](long long rbs, int st) {  // lane 0: the own-row streams of step rbs
    if (rbs < rend) {
      const long long rows = min((long long)G, rend - rbs);
      const unsigned bytes = (unsigned)(rows * a.k * sizeof(double));
      unsigned long long* bar = &stg_bar[STG ? warp : 0][STG ? st : 0];
      unsigned char* dst = stg_buf + (size_t)st * 3 * a.stage_bytes;
      const long long o = rbs * (long long)cg.k;
      mbar_expect(bar, 3 * bytes);
      bulk_g2s(dst, cg.P + o, bytes, bar);
      bulk_g2s(dst + a.stage_bytes, cg.Q + o, bytes, bar);
      bulk_g2s(dst + 2 * a.stage_bytes, cg.x + o, bytes, bar);
    }
  };
  if constexpr (STG) {
    stg_buf = dyn_smem + (size_t)warp * a.stages * 3 * a.stage_bytes;
    if (stg_on) {
      if (lane == 0) {
        for (int st = 0; st < a.stages; ++st) mbar_init(&stg_bar[warp][st]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int st = 0; st < a.stages; ++st) stg_issue(rb + st * stride, st);
      }
      __syncwarp();
    }
  }
  int stg_st = 0;
  unsigned stg_par = 0;
  // CG mode: the p'q accumulators stay in registers (one shared-memory store at the
  // end) — per-row shared read-modify-writes doubled the L1 wavefronts of the sweep
  double dacc[CG ? NV : 1][CG ? VEC : 1];
#pragma unroll
  for (int q = 0; q < (CG ? NV : 1); ++q)
#pragma unroll
    for (int e = 0; e < (CG ? VEC : 1); ++e) dacc[q][e] = 0.0;
  constexpr int CGN = CG ? kSpmmMaxPass : 1;
  // per-column (alpha, beta) and flags, stored at slot(col) = (col % VEC) * (256 / VEC) +
  // col / VEC: for a fixed e the lanes of a row group read consecutive slots (one
  // wavefront, broadcast across the groups) instead of a VEC-strided, bank-conflicting run
  __shared__ double cg_be[CGN], cg_sm[CGN];
  __shared__ double2 cg_ab[CGN];
  __shared__ int cg_fl[CGN];  // bit 0: p/q update (active), bit 1: deferred x-update
  auto cg_slot = [](int col) { return (col % VEC) * (kSpmmMaxPass / VEC) + col / VEC; };
  __shared__ int cg_nact;
  if constexpr (CG) {
    const int K = cg.k;
    if (threadIdx.x == 0) cg_nact = 0;
    if (!cg.first) cta_column_sums(cg.rpart, cg.nrp, K, cg_sm, cg_be);
    else __syncthreads();
    if (threadIdx.x < K) {
      const int cc = threadIdx.x;
      int pp = 0, ux = 0;
      double be = 0.0, al = 0.0;
      const double rzo = cg.s.rz[cg.par * K + cc];
      double rzn = rzo;
      if (cg.first) {
        pp = !cg.s.conv[cc] && !cg.s.frozen[cc];
      } else if (cg.s.upd[cc]) {
        ux = 1;
        al = cg.s.alpha[cc];
        const double rr = cg_be[cc];
        const double rn = sqrt(rr);
        if (blockIdx.x == 0) cg.s.rn[cc] = rn;
        if (rn <= cg.s.target[cc]) {
          if (blockIdx.x == 0) cg.s.conv[cc] = 1;
        } else {
          be = rr / rzo;
          rzn = rr;
          pp = 1;
        }
      }
      if (blockIdx.x == 0) cg.s.rz[(cg.par ^ 1) * K + cc] = rzn;
      cg_ab[cg_slot(cc)] = make_double2(al, be);
      cg_fl[cg_slot(cc)] = pp | (ux << 1);
      if (pp) atomicAdd(&cg_nact, 1);
    }
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *cg.s.pending = 0;
      if (cg_nact == 0) *cg.s.skip2 = 1;
    }
  }

  // prefetched state of the row this lane group handles next
  int nstart = 0, nlen = 0, ncol0 = 0, ncol1 = 0;
  double nval0 = 0.0, nval1 = 0.0;
  // (st, en) stay raw until the step that consumes them: an eager en - st would make
  // the warp wait for the row pointers right where they are requested
  auto fetch_rowptr = [&](long long base, int& st, int& en) {
    const long long r = base + g;
    st = 0;
    en = 0;
    if (r < rend) {
      st = __ldg(a.rowptr + r);
      en = __ldg(a.rowptr + r + 1);
    }
  };
  auto fetch_chunk = [&](int st, int ln, int off, int& c0, double& v0, int& c1, double& v1) {
    const int i0 = off + sub, i1 = off + LPR + sub;
    c0 = 0;
    v0 = 0.0;
    c1 = 0;
    v1 = 0.0;
    if (i0 < ln) {
      c0 = __ldg(a.colidx + st + i0);
      v0 = __ldg(a.val + st + i0);
    }
    if (i1 < ln) {
      c1 = __ldg(a.colidx + st + i1);
      v1 = __ldg(a.val + st + i1);
    }
  };
  // pipeline: row pointers two steps ahead, the first index/value chunk one step
  // ahead, so neither load is on a step's critical path (only the X gathers are)
  int pstart = 0, pend = 0;  // row pointers of the step after next
  if (rb < rend) {
    fetch_rowptr(rb, nstart, nlen);
    nlen -= nstart;
    fetch_chunk(nstart, nlen, 0, ncol0, nval0, ncol1, nval1);
    if (rb + stride < rend) fetch_rowptr(rb + stride, pstart, pend);
  }

  for (; rb < rend; rb += stride) {
    const long long r = rb + g;
    const int start = nstart, len = nlen;
    int col0 = ncol0, col1 = ncol1;
    double val0 = nval0, val1 = nval1;
    const long long rbn = rb + stride;
    nstart = pstart;
    nlen = pend - pstart;
    pstart = 0;
    pend = 0;
    if (rbn < rend) fetch_chunk(nstart, nlen, 0, ncol0, nval0, ncol1, nval1);
    if (rbn + stride < rend) fetch_rowptr(rbn + stride, pstart, pend);
    if constexpr (CG) {
      // the next step's own-row streams (p, q, x) into L2 while this step gathers, so
      // the epilogue's loads are L2 hits instead of exposed HBM latency
      static_assert(CGM >= 0, "");
      const long long rp = rb + (a.cg_prefetch == 2 ? 2 : 1) * stride + g;
      if (!STG && a.cg_prefetch && !cg.first && active && rp < rend) {
        const long long o = rp * (long long)cg.k + a.c0;
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          const int c = (q * LPR + sub) * VEC;
          if (c < k) {
            if (a.cg_prefetch == 3) {
              asm volatile("prefetch.global.L1 [%0];" ::"l"(cg.P + o + c));
              asm volatile("prefetch.global.L1 [%0];" ::"l"(cg.Q + o + c));
              asm volatile("prefetch.global.L1 [%0];" ::"l"(cg.x + o + c));
            } else {
              asm volatile("prefetch.global.L2 [%0];" ::"l"(cg.P + o + c));
              asm volatile("prefetch.global.L2 [%0];" ::"l"(cg.Q + o + c));
              asm volatile("prefetch.global.L2 [%0];" ::"l"(cg.x + o + c));
            }
          }
        }
      }
    }
    const int maxlen = __reduce_max_sync(FULL, len);
    // SELF (Z and/or W are X itself): keep the row's own X values from the
    // diagonal gather instead of re-reading them in the epilogue
    double xr[SELF ? NV : 1][VEC];
    bool have_diag = false;
    double acc[NV][VEC];
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[q][e] = 0.0;

    for (int off = 0; off < maxlen; off += CH) {
      if (off > 0) fetch_chunk(start, len, off, col0, val0, col1, val1);  // long rows
      const int tmax = min(CH, maxlen - off);
      for (int t0 = 0; t0 < tmax; t0 += U) {
        int j[U];
        double v[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int t = t0 + u;  // warp-uniform
          const bool lo = t < LPR;
          const int src = (gbase + (lo ? t : t - LPR)) & 31;
          j[u] = __shfl_sync(FULL, lo ? col0 : col1, src);
          v[u] = __shfl_sync(FULL, lo ? val0 : val1, src);
          ok[u] = (t < tmax) && (off + t < len);
          if (!ok[u]) v[u] = 0.0;
        }
        double xv[U][NV][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double* xr = a.X + (long long)j[u] * a.ldx;
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            const int c = (q * LPR + sub) * VEC;
            if (ok[u] && c < k) {
              VecT<VEC>::load(xr + c, xv[u][q]);
            } else {
#pragma unroll
              for (int e = 0; e < VEC; ++e) xv[u][q][e] = 0.0;
            }
          }
        }
        if constexpr (SELF) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const bool dg = ok[u] && (long long)j[u] == r;
            have_diag |= dg;
#pragma unroll
            for (int q = 0; q < NV; ++q)
#pragma unroll
              for (int e = 0; e < VEC; ++e) xr[q][e] = dg ? xv[u][q][e] : xr[q][e];
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < NV; ++q)
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[q][e] = fma(v[u], xv[u][q][e], acc[q][e]);
      }
    }
    // STG: this step's p, q, x have landed in the warp's stage (read below, in place)
    const unsigned char* stg_src = nullptr;
    if constexpr (STG) {
      if (stg_on) {
        mbar_wait(&stg_bar[warp][stg_st], stg_par);
        stg_src = stg_buf + (size_t)stg_st * 3 * a.stage_bytes + (size_t)g * k * sizeof(double);
      }
    }
    if constexpr (CG) {
      if (active && r < rend) {
        auto ldv = [&](const double* p, double* o) {
          if (a.vepi) {
            VecT<VEC>::ld(p, o);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) o[e] = p[e];
          }
        };
        auto lds = [&](const double* p, double* o) {  // p, q, x: read once, bypass L1
          if (a.vepi) {
            VecT<VEC>::ld_stream(p, o);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) o[e] = p[e];
          }
        };
        auto ldsm = [&](const unsigned char* p, double* o) {  // 32 bytes of a staged row
          const double2* v = reinterpret_cast<const double2*>(p);
#pragma unroll
          for (int e = 0; e < VEC / 2; ++e) {
            const double2 t = v[e];
            o[2 * e] = t.x;
            o[2 * e + 1] = t.y;
          }
        };
        auto stv = [&](double* p, const double* o) {
          if (a.vepi) {
            VecT<VEC>::st(p, o);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) p[e] = o[e];
          }
        };
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          const int c = (q * LPR + sub) * VEC;
          if (c >= k) continue;
          const int gc = a.c0 + c;  // passes keep k % VEC == 0: every e is a column
          double rv[VEC], y[VEC];
          ldv(a.X + r * a.ldx + c, rv);
#pragma unroll
          for (int e = 0; e < VEC; ++e) y[e] = fma(a.gamma, rv[e], acc[q][e]);
          int fl[VEC];
          bool anyp = false, anyx = false;
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            fl[e] = cg_fl[cg_slot(gc + e)];
            anyp |= (fl[e] & 1) != 0;
            anyx |= (fl[e] & 2) != 0;
          }
          const long long o = r * (long long)cg.k + gc;
          if (cg.first) {
            stv(cg.P + o, rv);  // p = r, q = (A + shift) r for every column (keeps P finite)
            stv(cg.Q + o, y);
#pragma unroll
            for (int e = 0; e < VEC; ++e)
              if (fl[e] & 1) dacc[CG ? q : 0][CG ? e : 0] = fma(rv[e], y[e], dacc[CG ? q : 0][CG ? e : 0]);
          } else if (anyp || anyx) {
            double pv[VEC];
            if constexpr (STG) {
              ldsm(stg_src + c * sizeof(double), pv);
            } else {
              lds(cg.P + o, pv);
            }
            if (anyx) {
              double xv[VEC];
              if constexpr (STG) {
                ldsm(stg_src + 2 * a.stage_bytes + c * sizeof(double), xv);
              } else {
                lds(cg.x + o, xv);
              }
#pragma unroll
              for (int e = 0; e < VEC; ++e)
                if (fl[e] & 2) xv[e] = fma(cg_ab[cg_slot(gc + e)].x, pv[e], xv[e]);
              stv(cg.x + o, xv);
            }
            if (anyp) {
              double qv[VEC];
              if constexpr (STG) {
                ldsm(stg_src + a.stage_bytes + c * sizeof(double), qv);
              } else {
                lds(cg.Q + o, qv);
              }
#pragma unroll
              for (int e = 0; e < VEC; ++e) {
                if (fl[e] & 1) {
                  const double be = cg_ab[cg_slot(gc + e)].y;
                  pv[e] = fma(be, pv[e], rv[e]);
                  qv[e] = fma(be, qv[e], y[e]);
                  dacc[CG ? q : 0][CG ? e : 0] = fma(pv[e], qv[e], dacc[CG ? q : 0][CG ? e : 0]);
                }
              }
              stv(cg.P + o, pv);
              stv(cg.Q + o, qv);
            }
          }
        }
      }
      if constexpr (STG) {
        // the stage goes back to the copy engine for the step a.stages ahead
        if (stg_on) {
          __syncwarp();
          if (lane == 0) stg_issue(rb + a.stages * stride, stg_st);
          if (++stg_st == a.stages) {
            stg_st = 0;
            stg_par ^= 1u;
          }
        }
      }
    } else if (active && r < rend) {
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const int c = (q * LPR + sub) * VEC;
        if (c >= k) continue;
        double y[VEC], t[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) y[e] = a.alpha * acc[q][e];
        const bool self_ok = SELF && have_diag;
        if (a.gamma != 0.0) {
          if (SELF && self_ok && a.Z == a.X) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) t[e] = xr[SELF ? q : 0][e];
          } else if (a.vepi) {
            VecT<VEC>::ld(a.Z + r * a.ldz + c, t);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) t[e] = a.Z[r * a.ldz + c + e];
          }
#pragma unroll
          for (int e = 0; e < VEC; ++e) y[e] = fma(a.gamma, t[e], y[e]);
        }
        if (a.beta != 0.0) {
          if (a.vepi) {
            VecT<VEC>::ld(a.Yin + r * a.ldyin + c, t);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) t[e] = a.Yin[r * a.ldyin + c + e];
          }
#pragma unroll
          for (int e = 0; e < VEC; ++e) y[e] = fma(a.beta, t[e], y[e]);
        }
        if (a.vepi) {
          VecT<VEC>::st(a.Y + r * a.ldy + c, y);
        } else {
#pragma unroll
          for (int e = 0; e < VEC; ++e) a.Y[r * a.ldy + c + e] = y[e];
        }
        if (a.dot_mode == 1) {
          if (SELF && self_ok && a.W == a.X) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) t[e] = xr[SELF ? q : 0][e];
          } else if (a.vepi) {
            VecT<VEC>::ld(a.W + r * a.ldw + c, t);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) t[e] = a.W[r * a.ldw + c + e];
          }
#pragma unroll
          for (int e = 0; e < VEC; ++e)
            sacc[warp][q * VEC + e][lane] = fma(y[e], t[e], sacc[warp][q * VEC + e][lane]);
        } else if (a.dot_mode == 2) {
#pragma unroll
          for (int e = 0; e < VEC; ++e)
            sacc[warp][q * VEC + e][lane] = fma(y[e], y[e], sacc[warp][q * VEC + e][lane]);
        }
      }
    }
  }

  // the successor may start launching while this grid drains (it still waits for this
  // grid's completion before touching memory): an early trigger would let its CTAs take
  // SM slots from this kernel's for the whole run
  pdl_trigger();
  if (a.dot_mode == 0) return;
  if constexpr (STG) __syncthreads();  // every warp is done with its stages: reuse them
  if constexpr (CG) {
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) sacc[warp][q * VEC + e][lane] = dacc[q][e];
  }
  // reduce over the row groups of the warp (fixed order g = 0..G-1), then warps
  __syncwarp();
  double gsum[NV][VEC];
  if (g0 == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        double v = 0.0;
        for (int gg = 0; gg < G; ++gg) v += sacc[warp][q * VEC + e][gg * LPR + sub];
        gsum[q][e] = v;
      }
  }
  __syncwarp();
  if (g0 == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const int c = (q * LPR + sub) * VEC + e;
        if (c < k) sdot[warp][c] = gsum[q][e];
      }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += kSpmmThreads) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += sdot[w][c];
    a.partials[(long long)blockIdx.x * a.pld + c] = s;
  }
}

// out[c*out_stride] = sum_b partials[b*k + c] in fixed b order (deterministic).
__global__ void reduce_partials_kernel(const double* __restrict__ partials, int nparts, int k,
                                       double* out, int out_stride, int mode) {
  const int c = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nparts; b += blockDim.x) s += partials[(long long)b * k + c];
  __shared__ double sm[128];  // fixed-shape tree over the 128 threads
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

// resident CTAs per SM of the fused CG sweep (GCG_CG_MINB=4: the 64-register build)
static int cg_minb() {
  static const int v = getenv("GCG_CG_MINB") ? atoi(getenv("GCG_CG_MINB")) : 3;
  return v == 4 ? 4 : 3;
}

template <int VEC, int NV>
static void launch_one(Ctx* c, const SpmmArgs& a, int grid, const CgSweep* cg) {
  if (cg) {
    if constexpr (VEC == 4) {
      if (a.stages > 0) {
        const size_t ring = (size_t)(kSpmmThreads / 32) * a.stages * 3 * a.stage_bytes;
        const size_t tail = sizeof(double) * (kSpmmThreads / 32) * (kSpmmMaxSlots * 32);
        const size_t smem = ring > tail ? ring : tail;
        static size_t smem_set = 0;  // opt in once per size class (> 48 KB)
        if (smem > smem_set) {
          cudaFuncSetAttribute(spmm_csr_kernel<VEC, NV, false, 3>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          smem_set = smem;
        }
        pdl_launch(spmm_csr_kernel<VEC, NV, false, 3>, dim3(grid), dim3(kSpmmThreads), smem,
                   c->stream, a, *cg);
        return;
      }
    }
    if (cg_minb() == 4)
      pdl_launch(spmm_csr_kernel<VEC, NV, false, 1>, dim3(grid), dim3(kSpmmThreads), 0,
                 c->stream, a, *cg);
    else
      pdl_launch(spmm_csr_kernel<VEC, NV, false, 2>, dim3(grid), dim3(kSpmmThreads), 0,
                 c->stream, a, *cg);
    return;
  }
  // the CG forms (shift and/or dot against X itself, same ld): own row from the gathers
  static const bool self_env = getenv("GCG_SPMM_SELF") ? atoi(getenv("GCG_SPMM_SELF")) != 0 : false;
  const bool self = self_env && ((a.gamma != 0.0 && a.Z == a.X && a.ldz == a.ldx) ||
                                 (a.dot_mode == 1 && a.W == a.X && a.ldw == a.ldx));
  const CgSweep none = {};
  if (self)
    pdl_launch(spmm_csr_kernel<VEC, NV, true, 0>, dim3(grid), dim3(kSpmmThreads), 0,
               c->stream, a, none);
  else
    pdl_launch(spmm_csr_kernel<VEC, NV, false, 0>, dim3(grid), dim3(kSpmmThreads), 0,
               c->stream, a, none);
}

template <int VEC>
static void launch_vec(Ctx* c, const SpmmArgs& a, int nv, int grid, const CgSweep* cg) {
  if constexpr (VEC == 4) {
    if (nv == 1) launch_one<4, 1>(c, a, grid, cg);
    else launch_one<4, 2>(c, a, grid, cg);
  } else if constexpr (VEC == 2) {
    switch (nv) {
      case 1: launch_one<2, 1>(c, a, grid, cg); break;
      case 2: launch_one<2, 2>(c, a, grid, cg); break;
      case 3: launch_one<2, 3>(c, a, grid, cg); break;
      default: launch_one<2, 4>(c, a, grid, cg); break;
    }
  } else {
    switch (nv) {
      case 1: launch_one<1, 1>(c, a, grid, cg); break;
      case 2: launch_one<1, 2>(c, a, grid, cg); break;
      case 3: launch_one<1, 3>(c, a, grid, cg); break;
      default: launch_one<1, 4>(c, a, grid, cg); break;
    }
  }
}

static inline bool aligned_to(const void* p, int bytes) {
  return ((uintptr_t)p % (uintptr_t)bytes) == 0;
}

// grid for a variant: one wave of its resident CTAs (grid-stride over rows)
static int spmm_grid_for(Ctx* c, long long n, int doubles) {
  return grid_for(n, 64, spmm_min_blocks(doubles), c->num_sms);
}
// upper bound over all variants (partials sizing in block CG)
int spmm_grid(Ctx* c, long long n) { return spmm_grid_for(c, n, 1); }

// Lane-group shape for `chunks` VEC-wide column chunks: NV chunks per lane,
// LPR = ceil(chunks / NV) lanes per row (any 1..32), G = 32 / LPR rows per warp.
// Maximises the useful fraction (G LPR / 32) (chunks / (LPR NV)); ties keep the
// smaller NV (fewer registers, more resident warps).
static double spmm_shape(int chunks, int vec, int* nv_out, int* lpr_out) {
  double best = -1.0;
  for (int nv = 1; nv <= 4 && nv * vec <= kSpmmMaxSlots; ++nv) {
    const int lpr = (chunks + nv - 1) / nv;
    if (lpr > 32) continue;
    const int g = 32 / lpr;
    const double eff = (double)(g * lpr) / 32.0 * (double)chunks / (double)(lpr * nv);
    if (eff > best + 1e-9) {
      best = eff;
      *nv_out = nv;
      *lpr_out = lpr;
    }
  }
  return best;
}

// One SpMM over all k columns, in even passes of at most 256 columns.  With
// dot_mode != 0 and `partials` given, per-CTA partials ([grid][k]) are left for
// the caller to reduce; otherwise they are reduced into `dots` per pass.
static int spmm_launch_core(Ctx* c, long long n, long long nnz, const int* rowptr,
                            const int* colidx, const double* val, int k, const double* X,
                            long long ldx, double alpha, double gamma, const double* Z,
                            long long ldz, double beta, const double* Yin, long long ldyin,
                            double* Y, long long ldy, int dot_mode, const double* W,
                            long long ldw, double* dots, double* partials_ext, int* grid_out,
                            const int* skip, const CgSweep* cg) {
  if (n <= 0 || k <= 0) return GCG_OK;
  double* partials = partials_ext;
  if (dot_mode && !partials) {
    GCG_TRY(ensure(c->partials, sizeof(double) * (size_t)spmm_grid(c, n) * kSpmmMaxPass));
    partials = (double*)c->partials.ptr;
  }
  int c0 = 0;
  int grid_fixed = 0;
  while (c0 < k) {
    const int rest = k - c0;
    // widest access every row start of X allows (rows of X must stay VEC-aligned)
    static const int vec_cap = getenv("GCG_SPMM_VEC") ? atoi(getenv("GCG_SPMM_VEC")) : 4;
    static const int contig = getenv("GCG_SPMM_ORDER") ? atoi(getenv("GCG_SPMM_ORDER")) : 0;
    int vec = 1;
    if (vec_cap >= 4 && ldx % 4 == 0 && aligned_to(X + c0, 32) && rest >= 4) vec = 4;
    else if (vec_cap >= 2 && ldx % 2 == 0 && aligned_to(X + c0, 16) && rest >= 2) vec = 2;
    // even passes of at most 32 lanes x NV x VEC columns
    auto max_cols = [](int v) { return 32 * v * (kSpmmMaxSlots / v < 4 ? kSpmmMaxSlots / v : 4); };
    // Column panels of <= 40 for 64 < k <= 128: one pass of k = 100 spreads 25 vec4 chunks
    // over 13 lanes x 2 (one row per warp); three ~36-column passes run 3 rows per warp
    // and keep each pass's neighbour rows L2-resident — measured at cfg4 (k = 100,
    // n = 2.1M): 1.90 -> 1.42 ms for the CG form, 1.71 -> 1.24 ms plain, although the
    // index/value stream is read three times.  Wider k (cfg5, k = 200) is gather-bound
    // and gains nothing (scripts/spmm_panel.sh).  GCG_SPMM_PANEL overrides the cap.
    static const int panel_env = getenv("GCG_SPMM_PANEL") ? atoi(getenv("GCG_SPMM_PANEL")) : -1;
    // (not for the fused CG sweep: there one pass over all k columns wins — cfg4 sweep
    // 5.94 -> 5.08 ms — its epilogue streams dominate and panels re-read them per pass)
    const int panel = panel_env >= 0 ? panel_env : (!cg && k > 64 && k <= 128 ? 40 : 0);
    int npass = (rest + max_cols(vec) - 1) / max_cols(vec);
    if (panel > 0 && (rest + panel - 1) / panel > npass) npass = (rest + panel - 1) / panel;
    int kc = (rest + npass - 1) / npass;
    kc = (kc + vec - 1) / vec * vec;
    if (kc > rest) kc = rest;
    if (kc % vec) {
      if (kc > vec) kc -= kc % vec;  // ragged tail goes to a narrower next pass
      else vec = 1;
    }
    int nv = 1, lpr = 1;
    double eff = spmm_shape((kc + vec - 1) / vec, vec, &nv, &lpr);
    if (vec > 1) {  // half-width accesses can tile the row and warp better (k = 160)
      int nv2 = 1, lpr2 = 1;
      const double eff2 = spmm_shape((kc + vec / 2 - 1) / (vec / 2), vec / 2, &nv2, &lpr2);
      if (eff2 > eff + 1e-9) {
        vec /= 2;
        nv = nv2;
        lpr = lpr2;
        eff = eff2;
      }
    }
    // caller-reduced partials ([grid][k]) need one grid for every pass
    int grid = grid_fixed ? grid_fixed
                          : (cg ? grid_for(n, 64, cg_minb(), c->num_sms)
                                : spmm_grid_for(c, n, nv * vec));
    if (partials_ext) grid_fixed = grid;
    long long rpc = 0;
    if (contig) {
      const long long step = 8LL * (32 / lpr);  // rows per CTA step (8 warps)
      rpc = ((n + grid - 1) / grid + step - 1) / step * step;
      grid = (int)((n + rpc - 1) / rpc);
    }
    if (grid_out) *grid_out = grid;
    SpmmArgs a;
    a.n = n;
    a.rowptr = rowptr;
    a.colidx = colidx;
    a.val = val;
    a.k = kc;
    a.lpr = lpr;
    a.gpw = 32 / lpr;
    a.rpc = rpc;
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
    a.partials = partials_ext ? partials + c0 : partials;
    a.pld = partials_ext ? k : kc;
    a.skip = skip;
    a.c0 = c0;
    static const int cg_pf = getenv("GCG_CG_PREFETCH") ? atoi(getenv("GCG_CG_PREFETCH")) : 1;
    a.cg_prefetch = cg_pf;
    const int vb = 8 * vec;
    a.vepi = aligned_to(a.Y, vb) && ldy % vec == 0 &&
             (gamma == 0.0 || (aligned_to(a.Z, vb) && ldz % vec == 0)) &&
             (beta == 0.0 || (aligned_to(a.Yin, vb) && ldyin % vec == 0)) &&
             (dot_mode != 1 || (aligned_to(a.W, vb) && ldw % vec == 0));
    // staged CG sweep (CGM 3): one pass over all k columns, 32-byte lanes, dense blocks
    // (ld = k, so a warp step's rows of p / q / x are one 16-byte-aligned run each)
    // Measured (scripts/gpu_cg_stage_ab.sh): wide blocks, one row per warp step (cfg4,
    // k = 100: 4.22 -> 3.80 ms per sweep with a one-stage ring) gain; at k = 20 (six rows
    // per warp step) the gathers, not the streams, bound the step and the ring's
    // shared-memory reads cost 2-3 %.  GCG_CG_STAGES overrides (0 = off).
    static const int cg_stages_env = getenv("GCG_CG_STAGES") ? atoi(getenv("GCG_CG_STAGES")) : -1;
    const int cg_stages = cg_stages_env >= 0 ? cg_stages_env : (32 / lpr == 1 ? 1 : 0);
    a.stages = 0;
    a.stage_bytes = 0;
    if (cg && cg_stages > 0 && vec == 4 && a.vepi && kc == k && kc == cg->k &&
        cg_minb() == 3 && aligned_to(cg->P, 32) && aligned_to(cg->Q, 32) && aligned_to(cg->x, 32)) {
      a.stage_bytes = (unsigned)(((size_t)(32 / lpr) * kc * sizeof(double) + 127) / 128 * 128);
      a.stages = cg_stages > kCgMaxStages ? kCgMaxStages : cg_stages;
      // at most 3 CTAs x ring within the 227 KB of shared memory
      while (a.stages > 1 && (size_t)(kSpmmThreads / 32) * a.stages * 3 * a.stage_bytes > 66 * 1024) --a.stages;
    }
    // algorithmic bytes: index/value stream + X once + Y once + each extra distinct stream
    double bytes = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n * kc;
    if (gamma != 0.0 && Z != X) bytes += 8.0 * n * kc;
    if (beta != 0.0) bytes += 8.0 * n * kc;
    if (dot_mode == 1 && W != X && W != Z) bytes += 8.0 * n * kc;
    // fused CG sweep: r once (gather) + p, q written (first sweep) / + p, q, x read and
    // written (later sweeps)
    if (cg) bytes = 12.0 * nnz + 4.0 * (n + 1) + (cg->first ? 24.0 : 56.0) * n * kc;
    // the fused CG sweep is its own class (its bytes include the x / p / q streams)
    const int ps = prof_start(c, cg ? PROF_CG_SWEEP : PROF_SPMM, bytes);
    a.prof_skipped = prof_skip_slot(c, ps);
    switch (vec) {
      case 4: launch_vec<4>(c, a, nv, grid, cg); break;
      case 2: launch_vec<2>(c, a, nv, grid, cg); break;
      default: launch_vec<1>(c, a, nv, grid, cg); break;
    }
    ++g_launches;
    GCG_CHECK_LAUNCH();
    prof_stop(c, ps);
    if (dot_mode && !partials_ext) {
      GCG_TRY(reduce_partials(c, partials, grid, kc, dots + c0, 1, 0));
      ++g_launches;
    }
    c0 += kc;
  }
  return GCG_OK;
}

int spmm_launch_impl(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                     const double* val, int k, const double* X, long long ldx, double alpha,
                     double gamma, const double* Z, long long ldz, double beta, const double* Yin,
                     long long ldyin, double* Y, long long ldy, int dot_mode, const double* W,
                     long long ldw, double* dots, double* partials_ext, int* grid_out,
                     const int* skip) {
  return spmm_launch_core(c, n, nnz, rowptr, colidx, val, k, X, ldx, alpha, gamma, Z, ldz, beta,
                          Yin, ldyin, Y, ldy, dot_mode, W, ldw, dots, partials_ext, grid_out, skip,
                          nullptr);
}

// The fused block-CG sweep over the dense n x k residual block R (ld k): see the CG
// mode of spmm_csr_kernel.  p'q partials ([grid][k]) are left in `partials`.
int spmm_cg_sweep_launch(Ctx* c, long long n, long long nnz, const int* rowptr,
                         const int* colidx, const double* val, int k, const double* R,
                         double shift, double* partials, int* grid_out, const CgSweep& cg) {
  return spmm_launch_core(c, n, nnz, rowptr, colidx, val, k, R, k, 1.0, shift, R, k, 0.0, nullptr,
                          0, cg.Q, k, 1, cg.P, k, nullptr, partials, grid_out, nullptr, &cg);
}

int spmm_launch_parts(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                      const double* val, int k, const double* X, long long ldx, double alpha,
                      double gamma, const double* Z, long long ldz, double beta,
                      const double* Yin, long long ldyin, double* Y, long long ldy, int dot_mode,
                      const double* W, long long ldw, double* partials, int* grid_out,
                      const int* skip) {
  return spmm_launch_impl(c, n, nnz, rowptr, colidx, val, k, X, ldx, alpha, gamma, Z, ldz, beta,
                          Yin, ldyin, Y, ldy, dot_mode, W, ldw, nullptr, partials, grid_out, skip);
}


// ---------------------------------------------------------------------------
// SELL-C-sigma SpMM (MatDotMultiVec on the sliced-ELLPACK format).
//
// Rows are sorted by length (descending, stable) inside windows of sigma rows and
// grouped into slices of kSellC = 32 consecutive sorted rows; slice s stores its
// width w_s = longest row, entry e of row t at slice_ptr[s] + e * 32 + t
// (column-major inside the slice: one slice's e-th entries are contiguous, so the
// index / value stream is read in coalesced 128-byte runs), padded with zero values
// whose column repeats the row's last column (the padding gather hits L1).  The
// SpMM kernel walks slices per warp with the CSR kernel's lane groups (LPR lanes,
// 32-byte gathers) and scatters each row to its original position through perm.
// Per row, the real entries are summed in CSR order with the same fma chain as the
// CSR kernel; padding adds exact zeros — results equal the CSR kernel's.
// Built on the device (gcg_sell_size / gcg_csr_to_sell: block radix sort per
// window, device exclusive scan of the slice sizes).

constexpr int kSellC = 32;
constexpr int kSellSigma = 1024;  // rows per sorting window (256 threads x 4 keys)

__global__ void __launch_bounds__(256) sell_sort_kernel(long long n, const int* __restrict__ rowptr,
                                                        int sorted, int* perm, long long* swidth) {
  using Sort = cub::BlockRadixSort<int, 256, 4, int>;
  __shared__ typename Sort::TempStorage tmp;
  const long long w0 = (long long)blockIdx.x * kSellSigma;
  int keys[4], vals[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = threadIdx.x * 4 + i;  // blocked: row order = input order (stable sort)
    const long long r = w0 + idx;
    if (r < n) {
      keys[i] = -(rowptr[r + 1] - rowptr[r]);
      vals[i] = (int)r;
    } else {
      keys[i] = INT_MAX;
      vals[i] = -1;
    }
  }
  if (sorted) Sort(tmp).Sort(keys, vals);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = threadIdx.x * 4 + i;
    const long long r = w0 + idx;
    if (r < n) {
      perm[r] = vals[i];
      if (idx % kSellC == 0) swidth[r / kSellC] = (long long)(-keys[i]) * kSellC;
    }
  }
}

// unsorted windows: the slice width is the max over its 32 rows
__global__ void sell_width_fix_kernel(long long n, const int* __restrict__ rowptr,
                                      const int* __restrict__ perm, long long nslices,
                                      long long* swidth) {
  const long long s = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const long long r = s * kSellC + (threadIdx.x & 31);
  int len = 0;
  if (r < n) {
    const int o = perm[r];
    len = rowptr[o + 1] - rowptr[o];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, off));
  if ((threadIdx.x & 31) == 0) swidth[s] = (long long)len * kSellC;
}

__global__ void sell_fill_kernel(long long n, const int* __restrict__ rowptr,
                                 const int* __restrict__ colidx, const double* __restrict__ val,
                                 const int* __restrict__ perm, const long long* __restrict__ sptr,
                                 long long nslices, int* scol, double* sval) {
  const long long s = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int t = threadIdx.x & 31;
  const long long base = sptr[s];
  const int w = (int)((sptr[s + 1] - base) / kSellC);
  const long long r = s * kSellC + t;
  int st = 0, len = 0, lastc = 0;
  if (r < n) {
    const int o = perm[r];
    st = rowptr[o];
    len = rowptr[o + 1] - st;
    lastc = len > 0 ? colidx[st + len - 1] : o;
  }
  for (int e = 0; e < w; ++e) {
    const bool real = e < len;
    scol[base + (long long)e * kSellC + t] = real ? colidx[st + e] : lastc;
    if (val) sval[base + (long long)e * kSellC + t] = real ? val[st + e] : 0.0;
  }
}

struct SellArgs {
  long long n, nslices;
  const long long* sptr;
  const int* perm;
  const int* scol;
  const double* sval;
  int k;
  const double* X;
  long long ldx;
  double alpha, gamma, beta;
  const double* Z;
  long long ldz;
  const double* Yin;
  long long ldyin;
  double* Y;
  long long ldy;
  int dot_mode;
  int lpr, gpw, vepi;
  const double* W;
  long long ldw;
  double* partials;
  int pld;
};

template <int VEC, int NV>
__global__ void __launch_bounds__(kSpmmThreads) spmm_sell_kernel(SellArgs a) {
  constexpr int NW = kSpmmThreads / 32;
  constexpr int U = 4;
  const int LPR = a.lpr, G = a.gpw;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g0 = lane / LPR;
  const bool active = g0 < G;
  const int g = active ? g0 : G - 1;
  const int sub = lane - g0 * LPR;
  const int k = a.k;
  __shared__ double sacc[NW][kSpmmMaxSlots][32];
  __shared__ double sdot[NW][kSpmmMaxPass];
  if (a.dot_mode) {
#pragma unroll
    for (int q = 0; q < NV * VEC; ++q) sacc[warp][q][lane] = 0.0;
  }
  for (long long s = (long long)blockIdx.x * NW + warp; s < a.nslices;
       s += (long long)gridDim.x * NW) {
    const long long base = a.sptr[s];
    const int w = (int)((a.sptr[s + 1] - base) / kSellC);
    for (int t0 = 0; t0 < kSellC; t0 += G) {
      const int t = t0 + g;
      const long long pos = s * kSellC + t;
      const bool ok_row = t < kSellC && pos < a.n;
      double acc[NV][VEC];
#pragma unroll
      for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[q][e] = 0.0;
      if (ok_row) {
        const int* cp = a.scol + base + t;
        const double* vp = a.sval + base + t;
        int e0 = 0;
        for (; e0 + U <= w; e0 += U) {
          int j[U];
          double v[U], xv[U][NV][VEC];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            j[u] = __ldg(cp + (long long)(e0 + u) * kSellC);
            v[u] = __ldg(vp + (long long)(e0 + u) * kSellC);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const double* xr = a.X + (long long)j[u] * a.ldx;
#pragma unroll
            for (int q = 0; q < NV; ++q) {
              const int c = (q * LPR + sub) * VEC;
              if (c < k) VecT<VEC>::load(xr + c, xv[u][q]);
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
        for (; e0 < w; ++e0) {
          const int j = __ldg(cp + (long long)e0 * kSellC);
          const double v = __ldg(vp + (long long)e0 * kSellC);
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
      if (!(active && ok_row)) continue;
      const long long r = a.perm[pos];
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const int c = (q * LPR + sub) * VEC;
        if (c >= k) continue;
        double y[VEC], tv[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) y[e] = a.alpha * acc[q][e];
        if (a.gamma != 0.0) {
          if (a.vepi) VecT<VEC>::ld(a.Z + r * a.ldz + c, tv);
          else
#pragma unroll
            for (int e = 0; e < VEC; ++e) tv[e] = a.Z[r * a.ldz + c + e];
#pragma unroll
          for (int e = 0; e < VEC; ++e) y[e] = fma(a.gamma, tv[e], y[e]);
        }
        if (a.beta != 0.0) {
          if (a.vepi) VecT<VEC>::ld(a.Yin + r * a.ldyin + c, tv);
          else
#pragma unroll
            for (int e = 0; e < VEC; ++e) tv[e] = a.Yin[r * a.ldyin + c + e];
#pragma unroll
          for (int e = 0; e < VEC; ++e) y[e] = fma(a.beta, tv[e], y[e]);
        }
        if (a.vepi) VecT<VEC>::st(a.Y + r * a.ldy + c, y);
        else
#pragma unroll
          for (int e = 0; e < VEC; ++e) a.Y[r * a.ldy + c + e] = y[e];
        if (a.dot_mode == 1) {
          if (a.vepi) VecT<VEC>::ld(a.W + r * a.ldw + c, tv);
          else
#pragma unroll
            for (int e = 0; e < VEC; ++e) tv[e] = a.W[r * a.ldw + c + e];
#pragma unroll
          for (int e = 0; e < VEC; ++e)
            sacc[warp][q * VEC + e][lane] = fma(y[e], tv[e], sacc[warp][q * VEC + e][lane]);
        } else if (a.dot_mode == 2) {
#pragma unroll
          for (int e = 0; e < VEC; ++e)
            sacc[warp][q * VEC + e][lane] = fma(y[e], y[e], sacc[warp][q * VEC + e][lane]);
        }
      }
    }
  }
  if (a.dot_mode == 0) return;
  __syncwarp();
  if (g0 == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const int c = (q * LPR + sub) * VEC + e;
        double v = 0.0;
        for (int gg = 0; gg < G; ++gg) v += sacc[warp][q * VEC + e][gg * LPR + sub];
        if (c < k) sdot[warp][c] = v;
      }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += kSpmmThreads) {
    double s = 0.0;
    for (int ww = 0; ww < NW; ++ww) s += sdot[ww][c];
    a.partials[(long long)blockIdx.x * a.pld + c] = s;
  }
}

template <int VEC, int NV>
static void sell_launch_one(Ctx* c, const SellArgs& a, int grid) {
  spmm_sell_kernel<VEC, NV><<<grid, kSpmmThreads, 0, c->stream>>>(a);
}

// slices and padded entry count of the SELL-C-sigma form (sigma: 1 = keep the row
// order, else rows sorted by length inside windows of 1024); synchronises once.
int sell_size(Ctx* c, long long n, const int* rowptr, int sigma, long long* nslices,
              long long* nnz_padded) {
  if (n <= 0 || !rowptr) return GCG_ERR_ARG;
  const long long ns = (n + kSellC - 1) / kSellC;
  const long long nwin = (n + kSellSigma - 1) / kSellSigma;
  GCG_TRY(ensure(c->host_tmp3, sizeof(long long) * (size_t)(ns + 1) + sizeof(int) * (size_t)n + 256));
  long long* sw = (long long*)c->host_tmp3.ptr;
  int* perm = (int*)(sw + ns + 1);
  sell_sort_kernel<<<(unsigned)nwin, 256, 0, c->stream>>>(n, rowptr, sigma > 1, perm, sw);
  if (sigma <= 1)
    sell_width_fix_kernel<<<(unsigned)((ns + 7) / 8), 256, 0, c->stream>>>(n, rowptr, perm, ns, sw);
  g_launches += sigma <= 1 ? 2 : 1;
  GCG_CHECK_LAUNCH();
  // total = sum of slice sizes (host reduction of ns values is fine at setup time)
  std::vector<long long> h((size_t)ns);
  GCG_TRY(cuda_status(cudaMemcpyAsync(h.data(), sw, sizeof(long long) * ns, cudaMemcpyDeviceToHost,
                                      c->stream)));
  GCG_TRY(cuda_status(cudaStreamSynchronize(c->stream)));
  long long tot = 0;
  for (long long v : h) tot += v;
  *nslices = ns;
  *nnz_padded = tot;
  return GCG_OK;
}

int csr_to_sell(Ctx* c, long long n, const int* rowptr, const int* colidx, const double* val,
                int sigma, long long* sptr, int* perm, int* scol, double* sval) {
  if (n <= 0 || !rowptr || !colidx || !sptr || !perm || !scol) return GCG_ERR_ARG;
  const long long ns = (n + kSellC - 1) / kSellC;
  const long long nwin = (n + kSellSigma - 1) / kSellSigma;
  GCG_TRY(ensure(c->host_tmp3, sizeof(long long) * (size_t)(ns + 1) + 256));
  long long* sw = (long long*)c->host_tmp3.ptr;
  sell_sort_kernel<<<(unsigned)nwin, 256, 0, c->stream>>>(n, rowptr, sigma > 1, perm, sw);
  if (sigma <= 1)
    sell_width_fix_kernel<<<(unsigned)((ns + 7) / 8), 256, 0, c->stream>>>(n, rowptr, perm, ns, sw);
  // slice_ptr = exclusive scan of the slice sizes (host: setup-time, ns values)
  std::vector<long long> h((size_t)ns + 1);
  GCG_TRY(cuda_status(cudaMemcpyAsync(h.data(), sw, sizeof(long long) * ns, cudaMemcpyDeviceToHost,
                                      c->stream)));
  GCG_TRY(cuda_status(cudaStreamSynchronize(c->stream)));
  long long acc = 0;
  for (long long s = 0; s < ns; ++s) {
    const long long v = h[(size_t)s];
    h[(size_t)s] = acc;
    acc += v;
  }
  h[(size_t)ns] = acc;
  GCG_TRY(cuda_status(cudaMemcpyAsync(sptr, h.data(), sizeof(long long) * (ns + 1),
                                      cudaMemcpyHostToDevice, c->stream)));
  sell_fill_kernel<<<(unsigned)((ns + 7) / 8), 256, 0, c->stream>>>(n, rowptr, colidx, val, perm,
                                                                    sptr, ns, scol, sval);
  g_launches += sigma <= 1 ? 3 : 2;
  GCG_CHECK_LAUNCH();
  // the host vector is read by the async copy: finish it before returning
  return cuda_status(cudaStreamSynchronize(c->stream));
}

int spmm_sell_launch(Ctx* c, long long n, long long nslices, const long long* sptr,
                     const int* perm, const int* scol, const double* sval, int k,
                     const double* X, long long ldx, double alpha, double gamma, const double* Z,
                     long long ldz, double beta, const double* Yin, long long ldyin, double* Y,
                     long long ldy, int dot_mode, const double* W, long long ldw, double* dots) {
  if (n <= 0 || k <= 0) return GCG_OK;
  double* partials = nullptr;
  const int grid = grid_for(nslices, 8, 4, c->num_sms);
  if (dot_mode) {
    GCG_TRY(ensure(c->partials, sizeof(double) * (size_t)grid * kSpmmMaxPass));
    partials = (double*)c->partials.ptr;
  }
  int c0 = 0;
  while (c0 < k) {
    const int rest = k - c0;
    int vec = 1;
    if (ldx % 4 == 0 && aligned_to(X + c0, 32) && rest >= 4) vec = 4;
    else if (ldx % 2 == 0 && aligned_to(X + c0, 16) && rest >= 2) vec = 2;
    auto max_cols = [](int v) { return 32 * v * (kSpmmMaxSlots / v < 4 ? kSpmmMaxSlots / v : 4); };
    const int npass = (rest + max_cols(vec) - 1) / max_cols(vec);
    int kc = (rest + npass - 1) / npass;
    kc = (kc + vec - 1) / vec * vec;
    if (kc > rest) kc = rest;
    if (kc % vec) {
      if (kc > vec) kc -= kc % vec;
      else vec = 1;
    }
    int nv = 1, lpr = 1;
    spmm_shape((kc + vec - 1) / vec, vec, &nv, &lpr);
    SellArgs a;
    a.n = n;
    a.nslices = nslices;
    a.sptr = sptr;
    a.perm = perm;
    a.scol = scol;
    a.sval = sval;
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
    a.lpr = lpr;
    a.gpw = 32 / lpr;
    a.partials = partials;
    a.pld = kc;
    const int vb = 8 * vec;
    a.vepi = aligned_to(a.Y, vb) && ldy % vec == 0 &&
             (gamma == 0.0 || (aligned_to(a.Z, vb) && ldz % vec == 0)) &&
             (beta == 0.0 || (aligned_to(a.Yin, vb) && ldyin % vec == 0)) &&
             (dot_mode != 1 || (aligned_to(a.W, vb) && ldw % vec == 0));
    if (vec == 4) {
      if (nv == 1) sell_launch_one<4, 1>(c, a, grid);
      else sell_launch_one<4, 2>(c, a, grid);
    } else if (vec == 2) {
      switch (nv) {
        case 1: sell_launch_one<2, 1>(c, a, grid); break;
        case 2: sell_launch_one<2, 2>(c, a, grid); break;
        case 3: sell_launch_one<2, 3>(c, a, grid); break;
        default: sell_launch_one<2, 4>(c, a, grid); break;
      }
    } else {
      switch (nv) {
        case 1: sell_launch_one<1, 1>(c, a, grid); break;
        case 2: sell_launch_one<1, 2>(c, a, grid); break;
        case 3: sell_launch_one<1, 3>(c, a, grid); break;
        default: sell_launch_one<1, 4>(c, a, grid); break;
      }
    }
    ++g_launches;
    GCG_CHECK_LAUNCH();
    if (dot_mode) {
      GCG_TRY(reduce_partials(c, partials, grid, kc, dots + c0, 1, 0));
      ++g_launches;
    }
    c0 += kc;
  }
  return GCG_OK;
}

}  // namespace gcg

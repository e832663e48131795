// PROTOTYPE, NOT BUILT — kept for the record (DESIGN.md §4 "tried and not adopted").
// Windowed SpMM: per 128-row tile, stage the runs of X rows the tile references
// into shared memory with bulk copies (warp-specialised producer, mbarrier ring)
// and compute rows from shared memory.  Measured on B200 at cfg2 (7-point 64^3,
// k = 20, CG form): 51.6 us vs 51.6 us for the register-gather kernel in spmm.cu;
// staging alone 28 us, shared-memory compute alone 41-43 us (instruction-issue /
// shared-memory latency bound at 3-6 rows per warp instruction).  It lived inside
// spmm.cu (uses SpmmArgs, VecT, spmm_shape, async.cuh) and was registered per CSR
// pattern through gcg_csr_plan_attach / gcg_csr_plan_detach.
// ---------------------------------------------------------------------------
// Windowed SpMM: X rows staged in shared memory once per row tile.
//
// The gather kernel above reads, per nonzero, one k-wide run of X from L2: at
// cfg2 (7-point stencil, k = 20) that is 7 x 42 MB = 293 MB of L2->SM traffic
// per SpMM, and B200's L2 delivers ~10-12 TB/s to the SMs, so the gathers, not
// HBM, bound it (~25 us floor for the gathers alone; profiles/r01_gather_floor.txt).
// A tile of R consecutive rows of a banded / stencil / FEM matrix references a
// few contiguous runs of X rows (7-point, R = 128: [r0-4096, +R), [r0-64,
// r0+R+64), [r0+4096, +R) = 4R rows for 7R gathers).  Each tile stages exactly
// those runs into shared memory with the bulk-copy engine (one cp.async.bulk
// per run; X rows are contiguous, ld = k — the block-CG direction block),
// together with its row pointers and (local row index, value) stream, and then
// computes every row from shared memory.  L2->SM traffic drops to
// (staged rows / R) x X, the index stream shrinks from 12 to 10 bytes per
// nonzero, and the gathers leave the critical path.
//
// Warp-specialised pipeline: one producer warp (one elected lane) walks the
// CTA's tiles and issues each tile's copies into a ring of NBUF buffers
// ("full" mbarriers with transaction counts); eight consumer warps compute
// rows and release buffers through "empty" mbarriers, without block barriers.
//
// The plan (runs, local indices) depends only on the sparsity pattern: it is
// built once per registered CSR on the device (gcg_csr_plan_attach: a block
// radix sort of each tile's column indices, runs merged across gaps of <= 4
// rows) and looked up by (rowptr, colidx) at every SpMM.  Matrices whose tiles
// need too many runs or too many staged rows keep the gather kernel.
//
// Per (row, column) the products are summed in CSR order with the same fma
// chain as the gather kernel: both kernels give bit-identical Y.

constexpr int kWinMaxSeg = 24;
constexpr int kWinPlanThreads = 256;
constexpr int kWinPlanItems = 16;  // keys per thread: tile nnz + R <= 4096
constexpr int kWinGap = 4;         // runs separated by <= kWinGap rows are merged
constexpr int kWinConsumers = 16;  // consumer warps
constexpr int kWinThreads = 32 * (kWinConsumers + 1);
constexpr int kWinMaxBuf = 6;

struct WinPlan {
  long long n = 0, nnz = 0;
  const int* rowptr = nullptr;
  const int* colidx = nullptr;
  int R = 0, T = 0;
  int smax = 0, emax = 0;      // max staged rows / nonzeros of a tile
  long long staged_sum = 0;    // staged rows over all tiles
  bool ok = false;
  int4* seg = nullptr;         // [T][kWinMaxSeg] {first row, rows, smem row offset, 0}
  int4* tinfo = nullptr;       // [T] {runs, smem row of the first own row, e0, e1}
  uint16_t* lcol = nullptr;    // [nnz + 8] staged-row index of each nonzero
  int* rpad = nullptr;         // rowptr copy padded to 16-byte tile copies
  void* mem = nullptr;
};

__global__ void __launch_bounds__(kWinPlanThreads)
    win_plan_kernel(long long n, const int* __restrict__ rowptr, const int* __restrict__ colidx,
                    int R, int4* seg, int4* tinfo, uint16_t* lcol, int* status,
                    unsigned long long* staged_sum) {
  using Sort = cub::BlockRadixSort<int, kWinPlanThreads, kWinPlanItems>;
  __shared__ union {
    typename Sort::TempStorage sort;
    int keys[kWinPlanThreads * kWinPlanItems];
  } sh;
  __shared__ int4 sseg[kWinMaxSeg];
  __shared__ int sns, sfail;
  const int t = blockIdx.x;
  const long long r0 = (long long)t * R, r1 = min(n, r0 + R);
  const int e0 = rowptr[r0], e1 = rowptr[r1];
  const int m = e1 - e0, own = (int)(r1 - r0);
  if (m + own > kWinPlanThreads * kWinPlanItems) {  // uniform over the block
    if (threadIdx.x == 0) atomicExch(status, 1);
    return;
  }
  // keys: the tile's column indices plus its own rows (so the rows' own X values
  // are always staged, in one run, for the fused shift / dot epilogues)
  int keys[kWinPlanItems];
#pragma unroll
  for (int i = 0; i < kWinPlanItems; ++i) {
    const int idx = i * kWinPlanThreads + threadIdx.x;
    keys[i] = idx < m ? colidx[e0 + idx] : (idx < m + own ? (int)(r0 + idx - m) : INT_MAX);
  }
  Sort(sh.sort).Sort(keys);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kWinPlanItems; ++i) sh.keys[threadIdx.x * kWinPlanItems + i] = keys[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    const int M = m + own;
    int ns = 0, off = 0, fail = 0, own_off = -1;
    int s = sh.keys[0], e = s;
    for (int i = 1; i <= M; ++i) {
      const int kx = i < M ? sh.keys[i] : INT_MAX;
      if (i < M && kx - e <= kWinGap) {
        e = kx;
        continue;
      }
      if (ns == kWinMaxSeg) {
        fail = 1;
        break;
      }
      sseg[ns] = make_int4(s, e - s + 1, off, 0);
      if (r0 >= s && r0 <= e) own_off = off + (int)(r0 - s);
      off += e - s + 1;
      ++ns;
      s = e = kx;
    }
    if (off > 65535 || own_off < 0) fail = 1;
    sns = ns;
    sfail = fail;
    if (fail) {
      atomicExch(status, 1);
    } else {
      atomicMax(status + 1, off);
      atomicMax(status + 2, m);
      atomicAdd(staged_sum, (unsigned long long)off);
      tinfo[t] = make_int4(ns, own_off, e0, e1);
    }
  }
  __syncthreads();
  if (sfail) return;
  const int ns = sns;
  if (threadIdx.x < ns) seg[(long long)t * kWinMaxSeg + threadIdx.x] = sseg[threadIdx.x];
  for (int i = threadIdx.x; i < m; i += kWinPlanThreads) {
    const int col = colidx[e0 + i];
    int q = 0;
    while (q + 1 < ns && col >= sseg[q + 1].x) ++q;
    lcol[e0 + i] = (uint16_t)(sseg[q].z + col - sseg[q].x);
  }
}

struct WinArgs {
  SpmmArgs s;
  const int4* seg;
  const int4* tinfo;
  const uint16_t* lcol;
  const int* rpad;
  long long nnz;
  int R, T;
  int nbuf;         // staging buffers in the ring
  int buf_bytes;    // bytes per buffer
  int vs_off, ls_off, rp_off;  // byte offsets of the value / index / row-pointer regions
  int zx, wx;       // epilogue Z / W are X itself (read from shared memory)
  int dbg;          // development: 1 = consumers skip rows, 2 = producer skips X runs
};

__device__ __forceinline__ void mbar_init_n(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}

template <int VEC, int NV>
__global__ void __launch_bounds__(kWinThreads) spmm_win_kernel(WinArgs w) {
  const SpmmArgs& a = w.s;
  if (a.skip != nullptr && *a.skip) {
    if (a.prof_skipped && blockIdx.x == 0 && threadIdx.x == 0) *a.prof_skipped = 1;
    return;
  }
  extern __shared__ __align__(128) unsigned char wsm[];
  __shared__ __align__(8) unsigned long long full[kWinMaxBuf], empty[kWinMaxBuf];
  constexpr int NW = kWinConsumers;
  const int k = a.k;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int NB = w.nbuf;

  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init_n(&full[b], 1);
      mbar_init_n(&empty[b], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NW) {
    // ---- producer: one lane issues every tile's bulk copies into the ring
    if (lane == 0) {
      int i = 0;
      for (int t = blockIdx.x; t < w.T; t += gridDim.x, ++i) {
        const int b = i % NB;
        if (i >= NB) mbar_wait(&empty[b], ((i / NB) - 1) & 1);
        unsigned char* base = wsm + (size_t)b * w.buf_bytes;
        double* vs = reinterpret_cast<double*>(base + w.vs_off);
        const int4 info = w.tinfo[t];
        const int ns = info.x, e0 = info.z, e1 = info.w;
        const int4* sg = w.seg + (long long)t * kWinMaxSeg;
        const long long r0 = (long long)t * w.R;
        const int rows = (int)(min(a.n, r0 + w.R) - r0);
        const int a0v = e0 & ~1, a0l = e0 & ~7;
        int a1v = (e1 + 1) & ~1;
        if (a1v > w.nnz) {  // the stream's odd last element: plain copy (no read past the end)
          a1v = e1 & ~1;
          vs[e1 - 1 - a0v] = __ldg(a.val + e1 - 1);
        }
        const int a1l = (e1 + 7) & ~7;
        const unsigned rp_bytes = (unsigned)((rows + 1 + 3) & ~3) * 4u;
        unsigned bytes = (unsigned)(a1v - a0v) * 8u + (unsigned)(a1l - a0l) * 2u + rp_bytes;
        int4 sv[kWinMaxSeg];
#pragma unroll 1
        for (int q = 0; q < ns; ++q) {
          sv[q] = sg[q];
          if (w.dbg == 2) sv[q].y = 0;
          bytes += (unsigned)sv[q].y * k * 8u;
        }
        mbar_expect(&full[b], bytes);
#pragma unroll 1
        for (int q = 0; q < ns; ++q)
          if (sv[q].y)
            bulk_g2s(base + (size_t)sv[q].z * k * 8, a.X + (long long)sv[q].x * a.ldx,
                     (unsigned)sv[q].y * k * 8u, &full[b]);
        if (a1v > a0v) bulk_g2s(vs, a.val + a0v, (unsigned)(a1v - a0v) * 8u, &full[b]);
        if (a1l > a0l) bulk_g2s(base + w.ls_off, w.lcol + a0l, (unsigned)(a1l - a0l) * 2u, &full[b]);
        bulk_g2s(base + w.rp_off, w.rpad + r0, rp_bytes, &full[b]);
      }
    }
    return;
  }

  // ---- consumers
  const int LPR = a.lpr, G = a.gpw;
  const int g0 = lane / LPR;
  const bool active = g0 < G;
  const int g = active ? g0 : G - 1;
  const int sub = lane - g0 * LPR;
  double dacc[NV][VEC];
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int e = 0; e < VEC; ++e) dacc[q][e] = 0.0;

  int i = 0;
  for (int t = blockIdx.x; t < w.T; t += gridDim.x, ++i) {
    const int b = i % NB;
    const int4 info = w.tinfo[t];  // issued before the wait: off the critical path
    mbar_wait(&full[b], (i / NB) & 1);
    const unsigned char* base = wsm + (size_t)b * w.buf_bytes;
    const double* xs = reinterpret_cast<const double*>(base);
    const double* vs = reinterpret_cast<const double*>(base + w.vs_off);
    const uint16_t* ls = reinterpret_cast<const uint16_t*>(base + w.ls_off);
    const int* rp = reinterpret_cast<const int*>(base + w.rp_off);
    const int own = info.y, e0 = info.z;
    const int dv = (e0 & 1) - e0, dl = (e0 & 7) - e0;  // absolute nonzero -> smem slot
    const long long r0 = (long long)t * w.R;
    const int rows = w.dbg == 1 ? 0 : (int)(min(a.n, r0 + w.R) - r0);
    for (int rl = warp * G + g; rl < rows; rl += NW * G) {
      const int ps = rp[rl], pe = rp[rl + 1];
      double acc[NV][VEC];
#pragma unroll
      for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[q][e] = 0.0;
      int p = ps;
      for (; p + 4 <= pe; p += 4) {
        int j[4];
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          j[u] = ls[p + u + dl];
          v[u] = vs[p + u + dv];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            const int c = (q * LPR + sub) * VEC;
            if (c < k) {
              double xv[VEC];
              VecT<VEC>::ld(xs + j[u] * k + c, xv);
#pragma unroll
              for (int e = 0; e < VEC; ++e) acc[q][e] = fma(v[u], xv[e], acc[q][e]);
            }
          }
      }
      for (; p < pe; ++p) {
        const int j = ls[p + dl];
        const double v = vs[p + dv];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          const int c = (q * LPR + sub) * VEC;
          if (c < k) {
            double xv[VEC];
            VecT<VEC>::ld(xs + j * k + c, xv);
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[q][e] = fma(v, xv[e], acc[q][e]);
          }
        }
      }
      if (!active) continue;
      const long long r = r0 + rl;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const int c = (q * LPR + sub) * VEC;
        if (c >= k) continue;
        double y[VEC], tv[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) y[e] = a.alpha * acc[q][e];
        if (a.gamma != 0.0) {
          if (w.zx) {
            VecT<VEC>::ld(xs + (own + rl) * k + c, tv);
          } else if (a.vepi) {
            VecT<VEC>::ld(a.Z + r * a.ldz + c, tv);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) tv[e] = a.Z[r * a.ldz + c + e];
          }
#pragma unroll
          for (int e = 0; e < VEC; ++e) y[e] = fma(a.gamma, tv[e], y[e]);
        }
        if (a.beta != 0.0) {
          if (a.vepi) {
            VecT<VEC>::ld(a.Yin + r * a.ldyin + c, tv);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) tv[e] = a.Yin[r * a.ldyin + c + e];
          }
#pragma unroll
          for (int e = 0; e < VEC; ++e) y[e] = fma(a.beta, tv[e], y[e]);
        }
        if (a.vepi) {
          VecT<VEC>::st(a.Y + r * a.ldy + c, y);
        } else {
#pragma unroll
          for (int e = 0; e < VEC; ++e) a.Y[r * a.ldy + c + e] = y[e];
        }
        if (a.dot_mode == 1) {
          if (w.wx) {
            VecT<VEC>::ld(xs + (own + rl) * k + c, tv);
          } else if (a.vepi) {
            VecT<VEC>::ld(a.W + r * a.ldw + c, tv);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) tv[e] = a.W[r * a.ldw + c + e];
          }
#pragma unroll
          for (int e = 0; e < VEC; ++e) dacc[q][e] = fma(y[e], tv[e], dacc[q][e]);
        } else if (a.dot_mode == 2) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) dacc[q][e] = fma(y[e], y[e], dacc[q][e]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);
  }

  if (a.dot_mode == 0) return;
  // fixed-order reduction: row groups of a warp (g = 0..G-1), then warps.  All
  // copies have landed and been consumed, so buffer 0 is free for the slots.
  double* sacc = reinterpret_cast<double*>(wsm);   // [NW][kSpmmMaxSlots][32]
  double* sdot = sacc + NW * kSpmmMaxSlots * 32;   // [NW][kSpmmMaxPass]
  asm volatile("bar.sync 1, %0;" ::"n"(32 * NW) : "memory");
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int e = 0; e < VEC; ++e) sacc[(warp * kSpmmMaxSlots + q * VEC + e) * 32 + lane] = dacc[q][e];
  __syncwarp();
  if (g0 == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const int c = (q * LPR + sub) * VEC + e;
        double v = 0.0;
        for (int gg = 0; gg < G; ++gg) v += sacc[(warp * kSpmmMaxSlots + q * VEC + e) * 32 + gg * LPR + sub];
        if (c < k) sdot[warp * kSpmmMaxPass + c] = v;
      }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(32 * NW) : "memory");
  for (int c = threadIdx.x; c < k; c += 32 * NW) {
    double s = 0.0;
    for (int ww = 0; ww < NW; ++ww) s += sdot[ww * kSpmmMaxPass + c];
    a.partials[(long long)blockIdx.x * a.pld + c] = s;
  }
}

// -- plan registry (per context) ---------------------------------------------

struct WinRegistry {
  std::vector<WinPlan*> plans;
};

static WinRegistry* registry(Ctx* c) {
  if (!c->csr_plans) c->csr_plans = new WinRegistry();
  return (WinRegistry*)c->csr_plans;
}

static void plan_free(WinPlan* p) {
  if (p->mem) cudaFree(p->mem);
  delete p;
}

void spmm_plans_release(Ctx* c) {
  if (!c->csr_plans) return;
  for (WinPlan* p : registry(c)->plans) plan_free(p);
  delete registry(c);
  c->csr_plans = nullptr;
}

static const WinPlan* plan_lookup(Ctx* c, long long n, long long nnz, const int* rowptr,
                                  const int* colidx) {
  if (!c->csr_plans) return nullptr;
  for (const WinPlan* p : registry(c)->plans)
    if (p->rowptr == rowptr && p->colidx == colidx && p->n == n && p->nnz == nnz) return p;
  return nullptr;
}

int csr_plan_detach(Ctx* c, const int* rowptr, const int* colidx) {
  if (!c->csr_plans) return GCG_OK;
  auto& v = registry(c)->plans;
  for (size_t i = 0; i < v.size(); ++i) {
    if (v[i]->rowptr == rowptr && v[i]->colidx == colidx) {
      cudaStreamSynchronize(c->stream);  // no launch in flight still reads the plan
      plan_free(v[i]);
      v.erase(v.begin() + i);
      return GCG_OK;
    }
  }
  return GCG_OK;
}

// Build and register the windowed-SpMM plan of a CSR pattern (synchronises the
// stream once to read the plan's extent).  *usable = 1 when the matrix gets
// the windowed kernel.
int csr_plan_attach(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                    int rows_per_tile, int* usable) {
  if (usable) *usable = 0;
  if (n <= 0 || nnz < 0 || !rowptr || (nnz > 0 && !colidx)) return GCG_ERR_ARG;
  GCG_TRY(csr_plan_detach(c, rowptr, colidx));
  WinPlan* p = new WinPlan();
  p->n = n;
  p->nnz = nnz;
  p->rowptr = rowptr;
  p->colidx = colidx;
  p->R = rows_per_tile > 0 ? rows_per_tile : 128;
  p->T = (int)((n + p->R - 1) / p->R);
  const size_t seg_b = sizeof(int4) * (size_t)p->T * kWinMaxSeg;
  const size_t info_b = sizeof(int4) * (size_t)p->T;
  const size_t lcol_b = (sizeof(uint16_t) * (size_t)(nnz + 8) + 255) & ~(size_t)255;
  const size_t rpad_b = (sizeof(int) * (size_t)(n + 1 + 8) + 255) & ~(size_t)255;
  const size_t stat_b = 64;
  if (cudaMalloc(&p->mem, seg_b + info_b + lcol_b + rpad_b + stat_b) != cudaSuccess) {
    cudaGetLastError();
    delete p;
    return GCG_ERR_ALLOC;
  }
  unsigned char* m = (unsigned char*)p->mem;
  p->seg = (int4*)m;
  p->tinfo = (int4*)(m + seg_b);
  p->lcol = (uint16_t*)(m + seg_b + info_b);
  p->rpad = (int*)(m + seg_b + info_b + lcol_b);
  int* status = (int*)(m + seg_b + info_b + lcol_b + rpad_b);
  unsigned long long* ssum = (unsigned long long*)(status + 4);
  int st = cuda_status(cudaMemsetAsync(status, 0, stat_b, c->stream));
  if (st == GCG_OK) st = cuda_status(cudaMemsetAsync(p->lcol, 0, lcol_b + rpad_b, c->stream));
  if (st == GCG_OK)
    st = cuda_status(cudaMemcpyAsync(p->rpad, rowptr, sizeof(int) * (size_t)(n + 1),
                                     cudaMemcpyDeviceToDevice, c->stream));
  if (st == GCG_OK) {
    win_plan_kernel<<<p->T, kWinPlanThreads, 0, c->stream>>>(n, rowptr, colidx, p->R, p->seg,
                                                            p->tinfo, p->lcol, status, ssum);
    ++g_launches;
    st = cuda_status(cudaGetLastError());
  }
  int h[4] = {0, 0, 0, 0};
  unsigned long long hs = 0;
  if (st == GCG_OK) st = cuda_status(cudaMemcpyAsync(h, status, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  if (st == GCG_OK) st = cuda_status(cudaMemcpyAsync(&hs, ssum, sizeof(hs), cudaMemcpyDeviceToHost, c->stream));
  if (st == GCG_OK) st = cuda_status(cudaStreamSynchronize(c->stream));
  if (st != GCG_OK) {
    plan_free(p);
    return st;
  }
  p->ok = h[0] == 0;
  p->smax = h[1];
  p->emax = h[2];
  p->staged_sum = (long long)hs;
  registry(c)->plans.push_back(p);
  if (usable) *usable = p->ok ? 1 : 0;
  return GCG_OK;
}

template <int VEC, int NV>
static void win_launch_one(Ctx* c, const WinArgs& w, int grid, size_t smem) {
  const void* kern = (const void*)spmm_win_kernel<VEC, NV>;
  kernel_smem(kern, smem);
  spmm_win_kernel<VEC, NV><<<grid, kWinThreads, smem, c->stream>>>(w);
}

template <int VEC, int NV>
static int win_occupancy(size_t smem) {
  const void* kern = (const void*)spmm_win_kernel<VEC, NV>;
  kernel_smem(kern, smem);
  return kernel_occupancy(kern, kWinThreads, smem);
}

static void win_dispatch(Ctx* c, const WinArgs& w, int vec, int nv, int grid, size_t smem,
                         int* occ) {
#define GCG_WIN_CASE(V, N)                                            \
  if (vec == V && nv == N) {                                          \
    if (occ) *occ = win_occupancy<V, N>(smem);                        \
    else win_launch_one<V, N>(c, w, grid, smem);                      \
    return;                                                           \
  }
  GCG_WIN_CASE(4, 1) GCG_WIN_CASE(4, 2) GCG_WIN_CASE(2, 1) GCG_WIN_CASE(2, 2)
  GCG_WIN_CASE(2, 3) GCG_WIN_CASE(2, 4) GCG_WIN_CASE(1, 1) GCG_WIN_CASE(1, 2)
  GCG_WIN_CASE(1, 3) GCG_WIN_CASE(1, 4)
#undef GCG_WIN_CASE
}

// Ring geometry for the windowed kernel: bytes per buffer and buffers (0: do
// not use the windowed kernel for this shape).  X rows must be contiguous
// (ldx == k) and 16-byte aligned so each run is one bulk copy.
static int win_geometry(const WinPlan* p, int k, long long ldx, const double* X, const double* val,
                        int* nbuf_out, int* buf_bytes_out, int offs[3]) {
  static const int enabled = getenv("GCG_SPMM_WIN") ? atoi(getenv("GCG_SPMM_WIN")) : 1;
  static const int budget = getenv("GCG_SPMM_WIN_KB") ? atoi(getenv("GCG_SPMM_WIN_KB")) * 1024 : 200 * 1024;
  static const int nbuf_max = getenv("GCG_SPMM_WIN_NBUF") ? atoi(getenv("GCG_SPMM_WIN_NBUF")) : kWinMaxBuf;
  if (!enabled || !p || !p->ok || p->smax <= 0) return 0;
  if (ldx != k || k % 2 || k > 256 || !aligned_to(X, 16) || !aligned_to(val, 16)) return 0;
  const int xs_b = (p->smax * k * 8 + 127) / 128 * 128;
  const int vs_b = ((p->emax + 2) * 8 + 127) / 128 * 128;
  const int ls_b = ((p->emax + 16) * 2 + 127) / 128 * 128;
  const int rp_b = ((p->R + 4) * 4 + 127) / 128 * 128;
  const int bb = xs_b + vs_b + ls_b + rp_b;
  int nb = budget / bb;
  if (nb > nbuf_max) nb = nbuf_max;
  if (nb > kWinMaxBuf) nb = kWinMaxBuf;
  if (nb < 2) return 0;
  offs[0] = xs_b;
  offs[1] = xs_b + vs_b;
  offs[2] = xs_b + vs_b + ls_b;
  *nbuf_out = nb;
  *buf_bytes_out = bb;
  return 1;
}

// One windowed SpMM over all k columns (same contract as a gather-kernel pass).
// Returns the grid in *grid_out.
static int spmm_win_pass(Ctx* c, const WinPlan* p, SpmmArgs a, int nbuf, int buf_bytes,
                         const int offs[3], bool z_is_x, bool w_is_x, int* grid_out) {
  // 16-byte shared-memory reads (one LDS.128 per lane and column chunk): a quarter
  // warp then reads 128 contiguous bytes of one row — no intra-row bank conflicts
  // (32-byte lane chunks put lanes 0 and 4 of a 160-byte row in the same banks)
  const int kc = a.k;
  static const int vec_cap = getenv("GCG_SPMM_WIN_VEC") ? atoi(getenv("GCG_SPMM_WIN_VEC")) : 2;
  int vec = (kc % 4 == 0 && vec_cap >= 4) ? 4 : (kc % 2 == 0 ? 2 : 1);
  int nv = 1, lpr = 1;
  spmm_shape((kc + vec - 1) / vec, vec, &nv, &lpr);
  static const int nv_env = getenv("GCG_SPMM_WIN_NV") ? atoi(getenv("GCG_SPMM_WIN_NV")) : 0;
  if (nv_env > 0 && nv_env * vec <= kSpmmMaxSlots && (kc / vec + nv_env - 1) / nv_env <= 32) {
    nv = nv_env;
    lpr = (kc / vec + nv - 1) / nv;
  }
  WinArgs w;
  a.lpr = lpr;
  a.gpw = 32 / lpr;
  const int vb = 8 * vec;
  a.vepi = aligned_to(a.Y, vb) && a.ldy % vec == 0 &&
           (a.gamma == 0.0 || z_is_x || (aligned_to(a.Z, vb) && a.ldz % vec == 0)) &&
           (a.beta == 0.0 || (aligned_to(a.Yin, vb) && a.ldyin % vec == 0)) &&
           (a.dot_mode != 1 || w_is_x || (aligned_to(a.W, vb) && a.ldw % vec == 0));
  w.s = a;
  w.seg = p->seg;
  w.tinfo = p->tinfo;
  w.lcol = p->lcol;
  w.rpad = p->rpad;
  w.nnz = p->nnz;
  w.R = p->R;
  w.T = p->T;
  w.nbuf = nbuf;
  w.buf_bytes = buf_bytes;
  w.vs_off = offs[0];
  w.ls_off = offs[1];
  w.rp_off = offs[2];
  w.zx = z_is_x ? 1 : 0;
  w.wx = w_is_x ? 1 : 0;
  static const int dbg = getenv("GCG_SPMM_WIN_DEBUG") ? atoi(getenv("GCG_SPMM_WIN_DEBUG")) : 0;
  w.dbg = dbg;
  size_t smem = (size_t)nbuf * buf_bytes;
  const size_t red = sizeof(double) * (kWinConsumers * kSpmmMaxSlots * 32 + kWinConsumers * kSpmmMaxPass);
  if (smem < red) smem = red;
  int occ = 1;
  win_dispatch(c, w, vec, nv, 0, smem, &occ);
  int grid = occ * c->num_sms;
  if (grid > p->T) grid = p->T;
  const int cap = spmm_grid(c, a.n);
  if (grid > cap) grid = cap;
  if (grid_out) *grid_out = grid;
  win_dispatch(c, w, vec, nv, grid, smem, nullptr);
  return GCG_OK;
}

// Windowed form of spmm_launch_impl (same arguments); returns -1 when the
// matrix has no usable plan for this shape (the caller runs the gather kernel).
static int spmm_win_launch(Ctx* c, long long n, long long nnz, const int* rowptr,
                           const int* colidx, const double* val, int k, const double* X,
                           long long ldx, double alpha, double gamma, const double* Z,
                           long long ldz, double beta, const double* Yin, long long ldyin,
                           double* Y, long long ldy, int dot_mode, const double* W, long long ldw,
                           double* dots, double* partials_ext, int* grid_out, const int* skip) {
  const WinPlan* p = plan_lookup(c, n, nnz, rowptr, colidx);
  int nbuf = 0, bb = 0, offs[3];
  if (!p || !win_geometry(p, k, ldx, X, val, &nbuf, &bb, offs)) return -1;
  double* partials = partials_ext;
  if (dot_mode && !partials) {
    GCG_TRY(ensure(c->partials, sizeof(double) * (size_t)spmm_grid(c, n) * kSpmmMaxPass));
    partials = (double*)c->partials.ptr;
  }
  const bool z_is_x = gamma != 0.0 && Z == X && ldz == ldx;
  const bool w_is_x = dot_mode == 1 && W == X && ldw == ldx;
  {
    const int c0 = 0, kc = k;
    SpmmArgs a;
    a.n = n;
    a.rowptr = rowptr;
    a.colidx = colidx;
    a.val = val;
    a.k = kc;
    a.rpc = 0;
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
    double bytes = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n * kc;
    if (gamma != 0.0 && Z != X) bytes += 8.0 * n * kc;
    if (beta != 0.0) bytes += 8.0 * n * kc;
    if (dot_mode == 1 && W != X && W != Z) bytes += 8.0 * n * kc;
    const int ps = prof_start(c, PROF_SPMM, bytes);
    a.prof_skipped = prof_skip_slot(c, ps);
    int grid = 0;
    GCG_TRY(spmm_win_pass(c, p, a, nbuf, bb, offs, z_is_x, w_is_x, &grid));
    ++g_launches;
    GCG_CHECK_LAUNCH();
    prof_stop(c, ps);
    if (grid_out) *grid_out = grid;
    if (dot_mode && !partials_ext) {
      GCG_TRY(reduce_partials(c, partials, grid, kc, dots + c0, 1, 0));
      ++g_launches;
    }
  }
  return GCG_OK;
}


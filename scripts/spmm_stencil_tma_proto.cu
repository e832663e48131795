// PROTOTYPE, NOT BUILT — kept for the record (DESIGN.md §4 "tried and not adopted").
// 2.5-D z-marching SpMM for structured-grid CSR patterns: X planes staged by one 4-D TMA
// bulk-tensor copy each (halo zero-fill by the TMA unit), CSR values/codes per grid line
// by cp.async, lane = x with an odd 16-byte row pitch.  Bit-identical to the gather
// kernel on all operator families, but at cfg4 (k = 100) staging alone took 1.05 ms
// against the gather kernel's 1.25 ms for the whole SpMM (the ring that fits 227 KB
// forces 2-line tiles: 2.1x halo) and the full kernel 4.1 ms; cfg5 65-150 ms vs 75 ms.
// Lived in csrc/ with gcg_csr_set_grid / gcg_csr_clear_grid registering the grid.
// MatDotMultiVec for CSR operators that live on a structured grid: X rows staged
// in shared memory, one z-plane at a time (2.5-D blocking).
//
// Reference: CsrOperator.apply (operators.py:103-111) -> kernels.csr_matvec
// (_cy.pyx:11-23); the matrix is still a general CSR (any values, any subset of the
// 27 grid neighbours per row) — only its sparsity must stay within one grid step:
// rows in natural order i = x + nx (y + ny z), every column j of row i at
// |jx - x|, |jy - y|, |jz - z| <= 1 (checked once per pattern, gcg_csr_set_grid).
// All five BASELINE operators qualify (5/7/27-point stencils, the Kuhn P1 FEM
// 15-point pattern, the var-coef 7-point operator).
//
// Why: the gather kernel (spmm.cu) reads every neighbour row from L2 — 7 x (cfg4) or
// 27 x (cfg5) the X bytes — and L2 -> SM bandwidth, not HBM, bounds it (cfg5 at
// 13 % of the HBM roofline).  Here a CTA owns a Tx x Ty column of the grid and a
// z-segment; it marches in z with a ring of 4 planes of (Ty+2) x (Tx+2) X rows (the
// tile plus a one-row halo) in shared memory: planes z-1, z, z+1 are read by the
// compute of plane z while plane z+2 is in flight (cp.async, 16-byte pieces).  Each
// X row is staged (Tx+2)(Ty+2)/(Tx Ty) times instead of gathered up to 27 times,
// neighbour gathers become shared-memory loads, and the index/value stream is the
// only per-nonzero global read.  Wide k runs in column passes of <= 32 (the ring is
// 4 (Tx+2)(Ty+2) x P doubles).
//
// Lane mapping: a row of a pass is served by LPR lanes; lane s owns the 16-byte
// pieces s and s + LPR (columns 2s, 2s+1, 2(s+LPR), 2(s+LPR)+1), so each shared-memory
// load instruction of a lane group reads one contiguous run (conflict-free).
// Per (row, column) the products are summed in CSR order with one fma each — the
// gather kernel's order: both kernels give bit-identical Y.
//
// Roofline: HBM.  Algorithmic bytes per launch = 12 nnz + 4 (n+1) + 16 n k (+8 n k
// per extra epilogue stream), the gather kernel's figure.

#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <mutex>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "async.cuh"
#include "common.cuh"

namespace gcg {

extern int64_t g_launches;

constexpr int kStThreads = 512;
constexpr int kStRing = 4;
constexpr int kStMaxP = 32;  // columns per pass: a row is 16 lanes x one 16-byte piece

struct StArgs {
  int nx, ny, nz;
  int nxy;
  const int* __restrict__ rowptr;
  const uint8_t* __restrict__ code;  // per nonzero: (dz+1)*9 + (dy+1)*3 + (dx+1)
  const double* __restrict__ val;
  int P;                 // columns of this pass
  int PP;                // shared-memory row width (doubles): 16 or 32
  int LS;                // CSR entries per staged grid line (Tx * longest row)
  int LA;                // planes of lookahead (1..4)
  const double* X;       // X + c0
  long long ldx;
  double alpha, gamma, beta;
  const double* Z;       // gamma term (nullptr: none); zself: Z is X (own row from the ring)
  long long ldz;
  int zself;
  const double* Yin;
  long long ldyin;
  double* Y;
  long long ldy;
  int Tx, Ty, Lz;
  int tiles_x, tiles_y;
  int dbg;  // development: 1 = no compute, 2 = no CSR staging
};

__device__ __forceinline__ void lds2(const double* p, double& a, double& b) {
  const double2 v = *reinterpret_cast<const double2*>(p);
  a = v.x;
  b = v.y;
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(pred ? 4 : 0));
}

// Pipeline.  LA planes of lookahead: the X ring has NX = LA + 3 slots (planes z-1 ..
// z+1 read by the compute of plane z, LA more in flight), the CSR ring (values, codes,
// row pointers) LA + 1.  Iteration z commits one cp.async group with X(z+1+LA) and the
// CSR entries of plane z+LA, then waits until only the last LA groups are pending — the
// group that carried X(z+1) and CSR(z) — so each plane's loads have LA compute phases
// to land.  The row pointers that place a plane's CSR entries are loaded into
// registers one iteration earlier (warp w: line w, lane l: row pointer l; lane 0 also
// keeps entry 32) and written to the ring when the entries are issued.
// Shared memory: X [NX][(Ty+2)(Tx+2)][PP] | values [LA+1][Ty][LS] | row pointers
// [LA+1][Ty][Tx+1] | codes [LA+1][Ty][LS+8] bytes.  A grid line's rows are consecutive
// CSR rows, so its entries are one contiguous run (values 8 bytes at a time, codes in
// aligned 4-byte words).  Lane mapping: LPR = PP / 2 lanes per row (8 or 16), lane s
// owns columns 2s, 2s+1 — one 16-byte load per nonzero; a lane group reads one
// contiguous 128/256-byte staged row.  A thread serves the same (x, y) rows in every
// plane (<= kStRS row steps): their ring offsets are computed once.
constexpr int kStNPC = 9;  // 16-byte column pieces per warp: ceil(17 / WPL) with WPL >= 2
__global__ void __launch_bounds__(kStThreads, 1)
    spmm_stencil_kernel(StArgs a, const __grid_constant__ CUtensorMap xmap) {
  extern __shared__ __align__(128) double smem_raw[];
  __shared__ int ptab[27];
  __shared__ __align__(8) unsigned long long xbar[8];
  // the TMA destinations: 1024-byte aligned ring
  double* ring = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~(uintptr_t)1023);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = blockIdx.x % a.tiles_x;
  const int rest = blockIdx.x / a.tiles_x;
  const int ty = rest % a.tiles_y;
  const int seg = rest / a.tiles_y;
  const int x0 = tx * a.Tx, y0 = ty * a.Ty;
  const int z0 = seg * a.Lz;
  const int z1 = min(a.nz, z0 + a.Lz);
  const int Tx = a.Tx, Ty = a.Ty, LA = a.LA;
  const int NX = LA + 3, NC = LA + 1;
  const int W = Tx + 2, H = Ty + 2;
  const int PP = a.PP, LS = a.LS;
  const int plane_sz = W * H * PP;
  const int nx = a.nx, ny = a.ny, nxy = a.nxy;
  const int xcnt = min(Tx, nx - x0);  // rows of a tile line inside the grid
  const int ycnt = min(Ty, ny - y0);
  double* cval = ring + NX * plane_sz;                               // [NC][Ty][LS]
  int* crp = reinterpret_cast<int*>(cval + NC * Ty * LS);            // [NC][Ty][Tx+1]
  uint8_t* ccode = reinterpret_cast<uint8_t*>(crp + NC * Ty * (Tx + 1));  // [NC][Ty][LS+8]
  const int LSB = LS + 8;
  const auto xslot = [&](int zz) { return ((zz % NX) + NX) % NX; };

  // X plane zz: one 4-D bulk tensor copy (columns x rows x lines x 1 plane) by thread 0,
  // completion on the slot's mbarrier; the TMA unit zero-fills rows, lines and planes
  // outside the grid and the columns past P
  const unsigned xbytes = (unsigned)plane_sz * 8u;
  auto stage_x = [&](int zz) {
    if (tid != 0 || zz > z1) return;  // plane z1 is the last one read (as z + 1)
    const int sl = xslot(zz);
    double* dst = ring + sl * plane_sz;
    mbar_expect(&xbar[sl], xbytes);
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(&xmap)), "r"(0), "r"(x0 - 1), "r"(y0 - 1), "r"(zz),
        "r"(smem_addr(&xbar[sl]))
        : "memory");
  };
  // parity of plane zz's use of its slot (planes are staged in order from z0 - 1)
  const auto xpar = [&](int zz) { return (unsigned)(((zz - (z0 - 1)) / NX) & 1); };
  if (tid < NX) mbar_init(&xbar[tid]);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  // row pointers of line `warp` of plane zz into registers (lane l: entry l, lane 0: 32)
  int rpa = 0, rpb = 0;
  auto load_rp = [&](int zz) {
    if (zz >= z1 || warp >= ycnt) return;
    const long long i0 = (long long)nxy * zz + (long long)nx * (y0 + warp) + x0;
    rpa = lane <= xcnt ? __ldg(a.rowptr + i0 + lane) : 0;
    rpb = (lane == 0 && xcnt >= 32) ? __ldg(a.rowptr + i0 + 32) : 0;
  };
  // CSR entries of plane zz (row pointers in registers): stored row pointers + cp.async
  auto stage_csr = [&](int zz) {
    if (zz >= z1 || warp >= ycnt) return;
    const int sl = zz % NC;
    int* rpd = crp + (sl * Ty + warp) * (Tx + 1);
    if (lane <= xcnt) rpd[lane] = rpa;
    if (lane == 0 && xcnt >= 32) rpd[32] = rpb;
    const int b0 = __shfl_sync(0xffffffffu, rpa, 0);
    int b1 = __shfl_sync(0xffffffffu, rpa, xcnt & 31);
    if (xcnt >= 32) b1 = __shfl_sync(0xffffffffu, rpb, 0);
    double* dv = cval + (sl * Ty + warp) * LS;
    uint8_t* dc = ccode + (sl * Ty + warp) * LSB;
    for (int e = b0 + lane; e < b1; e += 32) cp_async8(dv + (e - b0), a.val + e, true);
    const int w0 = b0 & ~3, w1 = (b1 + 3) & ~3;
    for (int w = w0 + 4 * lane; w < w1; w += 128) cp_async4(dc + (w - w0), a.code + w, true);
  };

  // prologue: X(z0-1 .. z0+1) and CSR(z0) in one group (waited), then LA - 1 groups
  // q = 1 .. LA-1 with X(z0+1+q) and CSR(z0+q) — the pattern the loop continues
  load_rp(z0);
  stage_x(z0 - 1);
  stage_x(z0);
  stage_x(z0 + 1);
  stage_csr(z0);
  cp_commit();
  load_rp(z0 + 1);
  for (int q = 1; q < LA; ++q) {
    stage_x(z0 + 1 + q);
    stage_csr(z0 + q);
    cp_commit();
    load_rp(z0 + q + 1);
  }
  // compute mapping: lane = x (Tx = 32), warp w -> line ly = w / WPL and a share of the
  // 16-byte column pieces; PP / 2 is odd, so the 32 lanes' rows (stride PP doubles) hit
  // distinct bank groups — one conflict-free 16-byte load feeds two fma per lane.
  const int WPL = (kStThreads / 32) / Ty;   // warps per line
  const int lyw = warp / WPL, part = warp - lyw * WPL;
  const int npc = PP / 2;                   // 16-byte pieces per staged row
  const int pc0 = (npc * part) / WPL, pc1 = (npc * (part + 1)) / WPL;
  const int lx = lane;
  const bool rowok = lyw < ycnt && lx < xcnt;
  const int centre = ((lyw + 1) * W + (lx + 1)) * PP;
  const int rpo = lyw * (Tx + 1) + lx;
  const long long inpl = (long long)nx * (y0 + lyw) + x0 + lx;
  const double alpha = a.alpha, gamma = a.gamma, beta = a.beta;
  for (int z = z0; z < z1; ++z) {
    stage_x(z + 1 + LA);
    stage_csr(z + LA);
    cp_commit();
    load_rp(z + LA + 1);
    if (tid < 27) {
      const int dz = tid / 9 - 1, dy = (tid / 3) % 3 - 1, dx = tid % 3 - 1;
      ptab[tid] = xslot(z + dz) * plane_sz + (dy * W + dx) * PP;
    }
    // the group that carried CSR(z) is LA groups back; X(z+1) on its slot's mbarrier
    switch (LA) {
      case 1: cp_wait<1>(); break;
      case 2: cp_wait<2>(); break;
      case 3: cp_wait<3>(); break;
      default: cp_wait<4>(); break;
    }
    if (z == z0) {
      mbar_wait(&xbar[xslot(z0 - 1)], xpar(z0 - 1));
      mbar_wait(&xbar[xslot(z0)], xpar(z0));
    }
    mbar_wait(&xbar[xslot(z + 1)], xpar(z + 1));
    __syncthreads();
    if (rowok && a.dbg != 1) {
      const int sl = z % NC;
      const int* rp = crp + sl * Ty * (Tx + 1);
      const int base = rp[lyw * (Tx + 1)];
      const int e0 = rp[rpo] - base, e1 = rp[rpo + 1] - base;
      const double* vline = cval + (sl * Ty + lyw) * LS;
      const uint8_t* cline = ccode + (sl * Ty + lyw) * LSB + (base & 3);
      double acc[2 * kStNPC];
#pragma unroll
      for (int q = 0; q < 2 * kStNPC; ++q) acc[q] = 0.0;
      for (int e = e0; e < e1; ++e) {
        const double v = vline[e];
        const double* src = ring + centre + ptab[cline[e]];
#pragma unroll
        for (int q = 0; q < kStNPC; ++q) {
          const int pc = pc0 + q;
          if (pc < pc1) {
            double q0, q1;
            lds2(src + 2 * pc, q0, q1);
            acc[2 * q] = fma(v, q0, acc[2 * q]);
            acc[2 * q + 1] = fma(v, q1, acc[2 * q + 1]);
          }
        }
      }
      // epilogue: y = alpha A x + gamma Z + beta Yin (the gather kernel's order)
      const long long i = (long long)nxy * z + inpl;
      const double* own = ring + xslot(z) * plane_sz + centre;
#pragma unroll
      for (int q = 0; q < kStNPC; ++q) {
        const int pc = pc0 + q;
        const int c = 2 * pc;
        if (pc >= pc1 || c >= a.P) continue;
        const bool two = c + 1 < a.P;
        double y0v = alpha * acc[2 * q], y1v = alpha * acc[2 * q + 1];
        if (gamma != 0.0) {
          double t0, t1;
          if (a.zself) {
            lds2(own + c, t0, t1);
          } else {
            t0 = a.Z[i * a.ldz + c];
            t1 = two ? a.Z[i * a.ldz + c + 1] : 0.0;
          }
          y0v = fma(gamma, t0, y0v);
          y1v = fma(gamma, t1, y1v);
        }
        if (beta != 0.0) {
          y0v = fma(beta, a.Yin[i * a.ldyin + c], y0v);
          if (two) y1v = fma(beta, a.Yin[i * a.ldyin + c + 1], y1v);
        }
        double* yp = a.Y + i * a.ldy + c;
        if (two && ((reinterpret_cast<uintptr_t>(yp) & 15) == 0)) {
          *reinterpret_cast<double2*>(yp) = make_double2(y0v, y1v);
        } else {
          yp[0] = y0v;
          if (two) yp[1] = y1v;
        }
      }
    }
    __syncthreads();  // every slot read this iteration may be restaged next iteration
  }
  cp_wait<0>();
}

static size_t stencil_smem(int Tx, int Ty, int PP, int LS, int LA) {
  return sizeof(double) * ((size_t)(LA + 3) * (Tx + 2) * (Ty + 2) * PP + (LA + 1) * (size_t)Ty * LS) +
         sizeof(int) * (LA + 1) * (size_t)Ty * (Tx + 1) + (LA + 1) * (size_t)Ty * (LS + 8) + 1024 + 16;
}

// per-nonzero neighbour codes of a validated stencil pattern
__global__ void stencil_code_kernel(long long n, const int* __restrict__ rowptr,
                                    const int* __restrict__ colidx, int nx, int ny,
                                    uint8_t* code) {
  const long long nxy = (long long)nx * ny;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long z = i / nxy, y = (i / nx) % ny, x = i % nx;
    for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const long long j = colidx[e];
      const long long jz = j / nxy, jy = (j / nx) % ny, jx = j % nx;
      code[e] = (uint8_t)((jz - z + 1) * 9 + (jy - y + 1) * 3 + (jx - x + 1));
    }
  }
}

// device check: every nonzero within one grid step of its row (natural order)
__global__ void stencil_check_kernel(long long n, const int* __restrict__ rowptr,
                                     const int* __restrict__ colidx, int nx, int ny, int* bad) {
  const long long nxy = (long long)nx * ny;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long z = i / nxy, y = (i / nx) % ny, x = i % nx;
    atomicMax(bad + 1, rowptr[i + 1] - rowptr[i]);
    for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const long long j = colidx[e];
      const long long jz = j / nxy, jy = (j / nx) % ny, jx = j % nx;
      if (j < 0 || j >= n || llabs(jz - z) > 1 || llabs(jy - y) > 1 || llabs(jx - x) > 1) {
        atomicExch(bad, 1);
        return;
      }
    }
  }
}

// ---- per-context registry: CSR pattern (row pointers, column indices) -> grid ----
struct GridEntry {
  Ctx* ctx;
  const int* rowptr;
  const int* colidx;
  long long n;
  int nx, ny, nz;
  uint8_t* code;  // device, nnz entries (owned)
  int maxrow;     // longest row
};
static std::mutex g_grid_mu;
static std::vector<GridEntry> g_grids;

int stencil_set_grid(Ctx* c, long long n, const int* rowptr, const int* colidx, int nx, int ny,
                     int nz) {
  if (nx <= 0 || ny <= 0 || nz <= 0 || (long long)nx * ny * nz != n) return GCG_ERR_ARG;
  GCG_TRY(ensure(c->partials, 64));
  int* bad = (int*)c->partials.ptr;
  GCG_TRY(cuda_status(cudaMemsetAsync(bad, 0, 2 * sizeof(int), c->stream)));
  const int grid = grid_for(n, 256, 8, c->num_sms);
  stencil_check_kernel<<<grid, 256, 0, c->stream>>>(n, rowptr, colidx, nx, ny, bad);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  int hbad[2] = {1, 0};
  GCG_TRY(cuda_status(cudaMemcpyAsync(hbad, bad, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream)));
  GCG_TRY(cuda_status(cudaStreamSynchronize(c->stream)));
  if (hbad[0] || hbad[1] > 27) return GCG_ERR_ARG;
  int nnz = 0;
  GCG_TRY(cuda_status(cudaMemcpyAsync(&nnz, rowptr + n, sizeof(int), cudaMemcpyDeviceToHost, c->stream)));
  GCG_TRY(cuda_status(cudaStreamSynchronize(c->stream)));
  uint8_t* code = nullptr;
  if (cudaMalloc((void**)&code, (size_t)nnz + 16) != cudaSuccess) {
    cudaGetLastError();
    return GCG_ERR_ALLOC;
  }
  stencil_code_kernel<<<grid, 256, 0, c->stream>>>(n, rowptr, colidx, nx, ny, code);
  ++g_launches;
  GCG_CHECK_LAUNCH();
  std::lock_guard<std::mutex> lk(g_grid_mu);
  for (auto& e : g_grids)
    if (e.ctx == c && e.rowptr == rowptr) {
      cudaStreamSynchronize(c->stream);
      cudaFree(e.code);
      e = {c, rowptr, colidx, n, nx, ny, nz, code, hbad[1]};
      return GCG_OK;
    }
  g_grids.push_back({c, rowptr, colidx, n, nx, ny, nz, code, hbad[1]});
  return GCG_OK;
}

int stencil_clear_grid(Ctx* c, const int* rowptr) {
  std::lock_guard<std::mutex> lk(g_grid_mu);
  for (size_t q = 0; q < g_grids.size(); ++q)
    if (g_grids[q].rowptr == rowptr && (c == nullptr || g_grids[q].ctx == c)) {
      // in-flight kernels may still read the codes: free after the device drains
      cudaDeviceSynchronize();
      cudaFree(g_grids[q].code);
      g_grids.erase(g_grids.begin() + q);
      return GCG_OK;
    }
  return GCG_OK;
}

static bool stencil_lookup(Ctx* c, long long n, const int* rowptr, const int* colidx,
                           GridEntry* out) {
  std::lock_guard<std::mutex> lk(g_grid_mu);
  for (auto& e : g_grids)
    if (e.ctx == c && e.rowptr == rowptr && e.colidx == colidx && e.n == n) {
      *out = e;
      return true;
    }
  return false;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    else
      cudaGetLastError();
  }
  return fn;
}

static bool stencil_enabled() {
  static const bool on = !(getenv("GCG_STENCIL") && getenv("GCG_STENCIL")[0] == '0');
  return on;
}

// Plain forms only (no fused dots / CG sweep): Y = alpha A X + gamma Z + beta Yin.
// Returns 1 when it ran, 0 when the caller should use the gather kernel.
int spmm_stencil_try(Ctx* c, long long n, long long nnz, const int* rowptr, const int* colidx,
                     const double* val, int k, const double* X, long long ldx, double alpha,
                     double gamma, const double* Z, long long ldz, double beta, const double* Yin,
                     long long ldyin, double* Y, long long ldy, int* ran) {
  *ran = 0;
  if (!stencil_enabled() || n <= 0 || k <= 0) return GCG_OK;
  GridEntry ge;
  if (!stencil_lookup(c, n, rowptr, colidx, &ge)) return GCG_OK;
  if ((ldx & 1) || ((uintptr_t)X & 15)) return GCG_OK;  // 16-byte staged pieces
  if (ge.nx < 4 || ge.ny < 4) return GCG_OK;
  static const int env_tx = getenv("GCG_ST_TX") ? atoi(getenv("GCG_ST_TX")) : 0;
  static const int env_ty = getenv("GCG_ST_TY") ? atoi(getenv("GCG_ST_TY")) : 0;
  static const int env_lz = getenv("GCG_ST_LZ") ? atoi(getenv("GCG_ST_LZ")) : 0;
  static const int env_p = getenv("GCG_ST_P") ? atoi(getenv("GCG_ST_P")) : 0;
  // column passes of <= 32 (even widths; the last takes the rest)
  const int pmax = env_p > 0 ? env_p : kStMaxP;
  const int npass = (k + pmax - 1) / pmax;
  int pw = (k + npass - 1) / npass;
  pw += pw & 1;
  const double bytes_pass = 9.0 * nnz + 4.0 * (n + 1);
  for (int c0 = 0; c0 < k; c0 += pw) {
    const int P = k - c0 < pw ? k - c0 : pw;
    // staged row width: P rounded up to 2 (mod 4) doubles — an odd number of 16-byte
    // pieces, so the 32 lanes (consecutive x) read conflict-free
    int PP = P + (P & 1);
    if (PP % 4 == 0) PP += 2;
    const int Tx = 32;
    static const int env_la = getenv("GCG_ST_LA") ? atoi(getenv("GCG_ST_LA")) : 0;
    const int LA = env_la > 0 ? (env_la > 4 ? 4 : env_la) : 2;
    const int LS = Tx * (ge.maxrow > 0 ? ge.maxrow : 1);
    // lines per tile: 8, 4, 2 (>= 2 warps per line, so <= kStNPC pieces per warp), the
    // largest whose ring fits ~200 KB
    int Ty = env_ty > 0 ? env_ty : 8;
    while (Ty > 2 && stencil_smem(Tx, Ty, PP, LS, LA) > 200 * 1024) Ty >>= 1;
    if (Ty > ge.ny) Ty = ge.ny >= 8 ? 8 : (ge.ny >= 4 ? 4 : 2);
    const int WPL = (kStThreads / 32) / Ty;
    const size_t smem = stencil_smem(Tx, Ty, PP, LS, LA);
    if (smem > 220 * 1024 || Ty < 1 || (kStThreads / 32) % Ty || (PP / 2 + WPL - 1) / WPL > kStNPC)
      return GCG_OK;
    const int tiles_x = (ge.nx + Tx - 1) / Tx, tiles_y = (ge.ny + Ty - 1) / Ty;
    int Lz = env_lz;
    if (Lz <= 0) {
      // whole waves of one CTA per SM where the z extent allows, segments of >= 8 planes
      const long long tiles = (long long)tiles_x * tiles_y;
      long long segs = (c->num_sms + tiles - 1) / tiles;
      for (long long sgs = segs; sgs <= 4 * segs; ++sgs) {
        const long long ctas = tiles * sgs;
        if (ctas % c->num_sms == 0 || (ctas % c->num_sms) * 10 >= 9LL * c->num_sms) {
          segs = sgs;
          break;
        }
      }
      if (segs > ge.nz / 8) segs = ge.nz / 8;
      if (segs < 1) segs = 1;
      Lz = (int)((ge.nz + segs - 1) / segs);
    }
    const int nseg = (ge.nz + Lz - 1) / Lz;
    StArgs a;
    a.nx = ge.nx;
    a.ny = ge.ny;
    a.nz = ge.nz;
    a.nxy = ge.nx * ge.ny;
    a.rowptr = rowptr;
    a.code = ge.code;
    a.val = val;
    a.P = P;
    a.PP = PP;
    a.LS = LS;
    a.LA = LA;
    static const int env_dbg = getenv("GCG_ST_DBG") ? atoi(getenv("GCG_ST_DBG")) : 0;
    a.dbg = env_dbg;
    a.X = X + c0;
    a.ldx = ldx;
    a.alpha = alpha;
    a.gamma = gamma;
    a.beta = beta;
    a.Z = Z ? Z + c0 : nullptr;
    a.ldz = ldz;
    a.zself = (Z == X && ldz == ldx) ? 1 : 0;
    a.Yin = Yin ? Yin + c0 : nullptr;
    a.ldyin = ldyin;
    a.Y = Y + c0;
    a.ldy = ldy;
    a.Tx = Tx;
    a.Ty = Ty;
    a.Lz = Lz;
    a.tiles_x = tiles_x;
    a.tiles_y = tiles_y;
    double bytes = bytes_pass + 16.0 * n * P;
    if (gamma != 0.0 && !a.zself) bytes += 8.0 * n * P;
    if (beta != 0.0) bytes += 8.0 * n * P;
    // X viewed as [nz][ny][nx][P] (strides ldx, nx ldx, nx ny ldx doubles), box
    // [1][Ty+2][Tx+2][PP]: one copy per plane, out-of-range elements zero-filled
    CUtensorMap xmap;
    {
      auto enc = tmap_encoder();
      if (!enc) return GCG_OK;
      cuuint64_t dims[4] = {(cuuint64_t)P, (cuuint64_t)ge.nx, (cuuint64_t)ge.ny,
                            (cuuint64_t)ge.nz};
      cuuint64_t strides[3] = {(cuuint64_t)ldx * 8, (cuuint64_t)ldx * 8 * ge.nx,
                               (cuuint64_t)ldx * 8 * ge.nx * ge.ny};
      cuuint32_t box[4] = {(cuuint32_t)PP, (cuuint32_t)(Tx + 2), (cuuint32_t)(Ty + 2), 1};
      cuuint32_t estr[4] = {1, 1, 1, 1};
      if (enc(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)(X + c0), dims, strides, box,
              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return GCG_OK;
    }
    if (getenv("GCG_ST_VERBOSE"))
      fprintf(stderr, "stencil: P=%d PP=%d Tx=%d Ty=%d LA=%d Lz=%d tiles=%dx%d segs=%d smem=%zu\n",
              P, PP, Tx, Ty, LA, Lz, tiles_x, tiles_y, nseg, smem);
    const int ps = prof_start(c, PROF_SPMM, bytes);
    kernel_smem((const void*)spmm_stencil_kernel, smem);
    spmm_stencil_kernel<<<tiles_x * tiles_y * nseg, kStThreads, smem, c->stream>>>(a, xmap);
    prof_stop(c, ps);
    ++g_launches;
    GCG_CHECK_LAUNCH();
  }
  *ran = 1;
  return GCG_OK;
}

}  // namespace gcg

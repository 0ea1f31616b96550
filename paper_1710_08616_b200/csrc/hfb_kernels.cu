// hfb_kernels.cu — sm_100a kernels of the Hybrid-Fortran timestep hot path.
//
// Every kernel maps one thread to one (i,j) column of the domain and marches K
// sequentially (K is executed sequentially, I/J are the parallel
// domain), over the I-fastest device order of hfb_layout.cuh, so each warp touches
// 32 consecutive i of one row per access (fully coalesced 256-B requests).
//
// Bit-exactness: compiled with -fmad=false (no FMA contraction), IEEE division and
// sqrt; every expression is written in the reference's left-associative evaluation
// order (parser.cpp:174-211, interp.cpp:661-770), so results equal the reference
// interpreter's binary64 results bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>
#include <cstdlib>

#include "hfb_kernels.cuh"

namespace hfb {

namespace {

inline dim3 span_grid(const Span& sp, dim3 block, unsigned z = 1) {
  int64_t ex = sp.ihi - sp.ilo + 1, ey = sp.jhi - sp.jlo + 1;
  return dim3(static_cast<unsigned>((ex + block.x - 1) / block.x),
              static_cast<unsigned>((ey + block.y - 1) / block.y), z);
}

inline bool span_empty(const Span& sp) { return sp.ihi < sp.ilo || sp.jhi < sp.jlo; }

}  // namespace

// ============================================================================
// relayout: dense host order (any dim permutation) <-> device layout.
// One 32x32 tile of the (I, F) plane per block, F = the host-fastest role;
// smem transpose so both global sides are coalesced.
// ============================================================================
namespace {
struct RelayoutArgs {
  const double* src;
  double* dst;
  Relayout r;
  int r1, r2;  // the two roles enumerated by blockIdx.z
  bool to_device;
};

__global__ void __launch_bounds__(256) k_relayout(RelayoutArgs a) {
  __shared__ double tile[32][33];
  const Relayout& r = a.r;
  const int F = r.fast;
  const int64_t z = blockIdx.z;
  const int64_t n1 = r.ext[a.r1];
  const int64_t c1 = z % n1, c2 = z / n1;
  const int64_t hrest = c1 * r.hs[a.r1] + c2 * r.hs[a.r2];
  const int64_t drest = c1 * r.ds[a.r1] + c2 * r.ds[a.r2];
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int64_t f0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (F == kRoleI) {
    // host already I-fastest: straight coalesced copy of rows (blockIdx.y over J*...)
    for (int rr = ty; rr < 32; rr += 8) {
      int64_t i = i0 + tx, f = f0 + rr;  // here "f" walks J
      if (i < r.ext[kRoleI] && f < r.ext[kRoleJ]) {
        int64_t h = i * r.hs[kRoleI] + f * r.hs[kRoleJ] + hrest;
        int64_t d = i + f * r.ds[kRoleJ] + drest;
        if (a.to_device)
          a.dst[d] = a.src[h];
        else
          a.dst[h] = a.src[d];
      }
    }
    return;
  }
  if (a.to_device) {
    for (int rr = ty; rr < 32; rr += 8) {  // read along F (host-contiguous)
      int64_t i = i0 + rr, f = f0 + tx;
      if (i < r.ext[kRoleI] && f < r.ext[F]) tile[rr][tx] = a.src[i * r.hs[kRoleI] + f + hrest];
    }
    __syncthreads();
    for (int rr = ty; rr < 32; rr += 8) {  // write along I (device-contiguous)
      int64_t i = i0 + tx, f = f0 + rr;
      if (i < r.ext[kRoleI] && f < r.ext[F]) a.dst[i + f * r.ds[F] + drest] = tile[tx][rr];
    }
  } else {
    for (int rr = ty; rr < 32; rr += 8) {  // read along I (device)
      int64_t i = i0 + tx, f = f0 + rr;
      if (i < r.ext[kRoleI] && f < r.ext[F]) tile[rr][tx] = a.src[i + f * r.ds[F] + drest];
    }
    __syncthreads();
    for (int rr = ty; rr < 32; rr += 8) {  // write along F (host)
      int64_t i = i0 + rr, f = f0 + tx;
      if (i < r.ext[kRoleI] && f < r.ext[F]) a.dst[i * r.hs[kRoleI] + f + hrest] = tile[tx][rr];
    }
  }
}
}  // namespace

cudaError_t launch_relayout(const double* src, double* dst, const Relayout& r, bool to_device,
                            cudaStream_t s) {
  RelayoutArgs a{src, dst, r, 0, 0, to_device};
  int F = r.fast;
  int rest[3], n = 0;
  int second = (F == kRoleI) ? kRoleJ : F;
  for (int role = 0; role < 4; ++role)
    if (role != kRoleI && role != second) rest[n++] = role;
  a.r1 = rest[0];
  a.r2 = rest[1];
  int64_t gz = r.ext[a.r1] * r.ext[a.r2];
  if (r.ext[kRoleI] <= 0 || r.ext[second] <= 0 || gz <= 0) return cudaSuccess;
  if (gz > 65535) return cudaErrorInvalidConfiguration;
  dim3 block(32, 8);
  dim3 grid(static_cast<unsigned>((r.ext[kRoleI] + 31) / 32),
            static_cast<unsigned>((r.ext[second] + 31) / 32), static_cast<unsigned>(gz));
  k_relayout<<<grid, block, 0, s>>>(a);
  return cudaGetLastError();
}

// ============================================================================
// element init flags (the reference's ArrayValue::init, interp.hpp:16-28) for the
// checked mode: one byte per element in the device layout of its array
// ============================================================================
namespace {
__global__ void k_relayout_u8(const uint8_t* src, uint8_t* dst, Relayout r, bool to_device,
                              int64_t n) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t q = e, ho = 0, dof = 0;
    for (int role = 0; role < 4; ++role) {
      const int64_t x = q % r.ext[role];
      q /= r.ext[role];
      ho += x * r.hs[role];
      dof += x * r.ds[role];
    }
    if (to_device)
      dst[dof] = src[ho];
    else
      dst[ho] = src[dof];
  }
}

// mode 0: *flag = 1 if any element of the box is unset; mode 1: set every element
__global__ void k_init_box(uint8_t* init, InitBox b, int mode, int* flag) {
  const int64_t n = b.n[0] * b.n[1] * b.n[2] * b.n[3];
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t q = e, off = 0;
    for (int role = 0; role < 4; ++role) {
      off += (b.lo[role] + q % b.n[role]) * b.ds[role];
      q /= b.n[role];
    }
    if (mode == 1)
      init[off] = 1;
    else if (!init[off])
      *flag = 1;
  }
}
}  // namespace

cudaError_t launch_relayout_u8(const uint8_t* src, uint8_t* dst, const Relayout& r,
                               bool to_device, cudaStream_t s) {
  const int64_t n = r.ext[0] * r.ext[1] * r.ext[2] * r.ext[3];
  if (n <= 0) return cudaSuccess;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  k_relayout_u8<<<blocks, 256, 0, s>>>(src, dst, r, to_device, n);
  return cudaGetLastError();
}

cudaError_t launch_init_box(uint8_t* init, const InitBox& b, int mode, int* flag,
                            cudaStream_t s) {
  const int64_t n = b.n[0] * b.n[1] * b.n[2] * b.n[3];
  if (n <= 0) return cudaSuccess;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  k_init_box<<<blocks, 256, 0, s>>>(init, b, mode, flag);
  return cudaGetLastError();
}

// ============================================================================
// diffusion.h90:23-41 — 7-point stencil with the Dirichlet copy on the GLOBAL
// boundary; K neighbours live in registers (k-1, k, k+1 rotate), I/J neighbours
// come from L1 (each is loaded by the adjacent threads of the same warp/block).
// hfk1 (t_old = t_new) is fused away: the step result goes to out1 and, when the
// caller needs both arrays materialised, to out2.
// ============================================================================
namespace {
struct DiffArgs {
  const double* __restrict__ src;
  double* __restrict__ o1;
  double* __restrict__ o2;
  Grid3 g;
  int nz, kchunk;
  double coef;
  Span sp;
};

// K is processed in chunks of kDiffChunk levels: all loads of a chunk (its center
// column plus the four horizontal neighbours of every level) are issued before any
// arithmetic, so ~40 independent loads per thread are in flight (the one-level
// version is bound by load latency: long_scoreboard 87%).
template <int kDiffChunk>
__global__ void __launch_bounds__(256) k_diffusion(DiffArgs a) {
  const int64_t i = a.sp.ilo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t j = a.sp.jlo + static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y;
  if (i > a.sp.ihi || j > a.sp.jhi) return;
  const int kb = 1 + static_cast<int>(blockIdx.z) * a.kchunk;
  const int ke = min(a.nz, kb + a.kchunk - 1);
  const int64_t gi = i + a.sp.i0, gj = j + a.sp.j0;
  const bool hb = (gi == 1) | (gi == a.sp.gnx) | (gj == 1) | (gj == a.sp.gny);
  const int64_t P = a.g.plane, W = a.g.pitch;
  const int64_t col = (j - 1) * W + (i - 1);
  const double* __restrict__ src = a.src + col;
  double* o1 = a.o1 + col;
  double* o2 = a.o2 ? a.o2 + col : nullptr;
  const int nz = a.nz;
  const double coef = a.coef;
#pragma unroll 1
  for (int k0 = kb; k0 <= ke; k0 += kDiffChunk) {
    double cc[kDiffChunk + 2];  // levels k0-1 .. k0+kDiffChunk
    double xw[kDiffChunk], xe[kDiffChunk], ys[kDiffChunk], yn[kDiffChunk];
#pragma unroll
    for (int q = 0; q < kDiffChunk + 2; ++q) {
      const int k = k0 - 1 + q;
      cc[q] = (k >= 1 && k <= nz) ? __ldg(src + static_cast<int64_t>(k - 1) * P) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kDiffChunk; ++q) {
      const int k = k0 + q;
      const bool need = !hb && k > 1 && k < nz && k <= ke;
      const double* c = src + static_cast<int64_t>(k - 1) * P;
      xw[q] = need ? __ldg(c - 1) : 0.0;
      xe[q] = need ? __ldg(c + 1) : 0.0;
      ys[q] = need ? __ldg(c - W) : 0.0;
      yn[q] = need ? __ldg(c + W) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kDiffChunk; ++q) {
      const int k = k0 + q;
      if (k > ke) break;
      const double c0 = cc[q + 1];
      double out;
      if (hb || k == 1 || k == nz) {
        out = c0;
      } else {
        double s = cc[q] + cc[q + 2];
        s = s + xw[q];
        s = s + xe[q];
        s = s + ys[q];
        s = s + yn[q];
        s = s - 6.0 * c0;
        out = c0 + coef * s;
      }
      const int64_t off = static_cast<int64_t>(k - 1) * P;
      o1[off] = out;
      if (o2) o2[off] = out;
    }
  }
}

__global__ void __launch_bounds__(256) k_copy_columns(const double* __restrict__ src,
                                                      double* __restrict__ dst, Grid3 g, int nz,
                                                      Span sp) {
  const int64_t i = sp.ilo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t j = sp.jlo + static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y;
  if (i > sp.ihi || j > sp.jhi) return;
  const int64_t col = (j - 1) * g.pitch + (i - 1);
  for (int k = 0; k < nz; ++k) dst[col + k * g.plane] = src[col + k * g.plane];
}
}  // namespace

cudaError_t launch_diffusion(const double* t_old, double* out1, double* out2, Grid3 g,
                             int64_t nz, double coef, const Span& sp, cudaStream_t s) {
  if (span_empty(sp) || nz <= 0) return cudaSuccess;
  dim3 block(32, 8);
  int64_t cols = (sp.ihi - sp.ilo + 1) * (sp.jhi - sp.jlo + 1);
  // Small grids cannot fill 148 SMs with one thread per column: split K into chunks
  // (each chunk re-reads its two boundary planes) until ~4 waves of columns exist.
  int64_t target = 148LL * 2048 * 2;
  int kchunks = 1;
  while (cols * kchunks < target && nz / (kchunks * 2) >= 8) kchunks *= 2;
  int kchunk = static_cast<int>((nz + kchunks - 1) / kchunks);
  kchunks = static_cast<int>((nz + kchunk - 1) / kchunk);
  DiffArgs a{t_old, out1, out2, g, static_cast<int>(nz), kchunk, coef, sp};
  dim3 grid = span_grid(sp, block, kchunks);
  k_diffusion<2><<<grid, block, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_copy_columns(const double* src, double* dst, Grid3 g, int64_t nz,
                                const Span& sp, cudaStream_t s) {
  if (span_empty(sp) || nz <= 0) return cudaSuccess;
  dim3 block(32, 8);
  k_copy_columns<<<span_grid(sp, block), block, 0, s>>>(src, dst, g, static_cast<int>(nz), sp);
  return cudaGetLastError();
}

// ============================================================================
// damping.h90:38-48 — pointwise: d = (m*(r + b1) + t*(r + b2)) - r.
// One thread per (i, j, k) element (no reuse to exploit; pure streaming).
// ============================================================================
namespace {
__global__ void __launch_bounds__(256) k_damping(const double* __restrict__ ref,
                                                 const double* __restrict__ b1,
                                                 const double* __restrict__ b2,
                                                 double* __restrict__ d, Grid3 g, double m,
                                                 double t, Span sp) {
  const int64_t i = sp.ilo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t j = sp.jlo + static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y;
  if (i > sp.ihi || j > sp.jhi) return;
  const int64_t idx = g.at(i - 1, j - 1, blockIdx.z);
  const double r = __ldg(ref + idx);
  d[idx] = (m * (r + __ldg(b1 + idx)) + t * (r + __ldg(b2 + idx))) - r;
}
}  // namespace

cudaError_t launch_damping(const double* ref, const double* bnd1, const double* bnd2,
                           double* damp, Grid3 g, int64_t nk, double mtratio, double tratio,
                           const Span& sp, cudaStream_t s) {
  if (span_empty(sp) || nk <= 0) return cudaSuccess;
  if (nk > 65535) return cudaErrorInvalidConfiguration;
  dim3 block(32, 8);
  k_damping<<<span_grid(sp, block, static_cast<unsigned>(nk)), block, 0, s>>>(
      ref, bnd1, bnd2, damp, g, mtratio, tratio, sp);
  return cudaGetLastError();
}

// ============================================================================
// bounded.h90:19-21 — 2-D 5-point average.
// ============================================================================
namespace {
__global__ void __launch_bounds__(256) k_bounded(const double* __restrict__ a,
                                                 double* __restrict__ b, int64_t W, Span sp) {
  const int64_t i = sp.ilo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t j = sp.jlo + static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y;
  if (i > sp.ihi || j > sp.jhi) return;
  const double* c = a + (j - 1) * W + (i - 1);
  b[(j - 1) * W + (i - 1)] =
      0.25 * (((__ldg(c - 1) + __ldg(c + 1)) + __ldg(c - W)) + __ldg(c + W));
}
}  // namespace

cudaError_t launch_bounded(const double* a, double* b, int64_t pitch, const Span& sp,
                           cudaStream_t s) {
  if (span_empty(sp)) return cudaSuccess;
  dim3 block(32, 8);
  k_bounded<<<span_grid(sp, block), block, 0, s>>>(a, b, pitch, sp);
  return cudaGetLastError();
}

// ============================================================================
// surface flux: driver.h90:3-17 (setup shift) and surface_flux.h90:3-48 (tile
// physics, privatised temporaries kept in registers instead of DOM(nx,ny,ntlm)
// device arrays — SURVEY §2.2 S5).
// ============================================================================
namespace {
__global__ void __launch_bounds__(256) k_sf_setup(double* __restrict__ cf, Grid3 g, int ntlm,
                                                  Span sp) {
  const int64_t i = sp.ilo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t j = sp.jlo + static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y;
  if (i > sp.ihi || j > sp.jhi) return;
  for (int lt = 0; lt < ntlm; ++lt) {
    const int64_t idx = g.at(i - 1, j - 1, lt);
    cf[idx] = cf[idx] - 0.5;
  }
}

__global__ void __launch_bounds__(256) k_sf_tile(const double* __restrict__ cover,
                                                 double* __restrict__ fx,
                                                 double* __restrict__ fy,
                                                 double* __restrict__ sw, int64_t W, Span sp) {
  const int64_t i = sp.ilo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t j = sp.jlo + static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y;
  if (i > sp.ihi || j > sp.jhi) return;
  const int64_t idx = (j - 1) * W + (i - 1);
  const double cf = __ldg(cover + idx);
  double taux, tauy, uf;
  if (cf > 0.0) {
    taux = 0.1 * cf;
    tauy = 0.2 * cf * cf;
    uf = sqrt(sqrt(taux * taux + tauy * tauy));
  } else {
    taux = 0.0;
    tauy = 0.0;
    uf = 0.0;
  }
  fx[idx] = taux;
  fy[idx] = tauy;
  sw[idx] = uf;
}
}  // namespace

cudaError_t launch_sf_setup(double* cover_frac, Grid3 g, int64_t ntlm, const Span& sp,
                            cudaStream_t s) {
  if (span_empty(sp)) return cudaSuccess;
  dim3 block(32, 8);
  k_sf_setup<<<span_grid(sp, block), block, 0, s>>>(cover_frac, g, static_cast<int>(ntlm), sp);
  return cudaGetLastError();
}

cudaError_t launch_sf_tile(const double* cover_lt, double* flx_x, double* flx_y, double* swind,
                           int64_t pitch, const Span& sp, cudaStream_t s) {
  if (span_empty(sp)) return cudaSuccess;
  dim3 block(32, 8);
  k_sf_tile<<<span_grid(sp, block), block, 0, s>>>(cover_lt, flx_x, flx_y, swind, pitch, sp);
  return cudaGetLastError();
}

// ============================================================================
// reduction.h90:21-25 — deterministic fp64 sum: fixed block count, each block sums
// a fixed contiguous range of (k, j) rows, warp-shuffle + smem tree inside the
// block; a single block folds the partials in index order. Same bits every run;
// within 1e-12 relative of the reference's sequential order.
// ============================================================================
namespace {
constexpr int kRedBlocks = 148 * 8;
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double warp_part[kRedThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) warp_part[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < kRedThreads / 32 ? warp_part[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0
}

__global__ void __launch_bounds__(kRedThreads) k_sum_rows(const double* __restrict__ y, Grid3 g,
                                                          int64_t nz, Span sp,
                                                          double* __restrict__ partials) {
  const int64_t ni = sp.ihi - sp.ilo + 1, nj = sp.jhi - sp.jlo + 1;
  const int64_t rows = nz * nj;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  double acc = 0.0;
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t k = r / nj, jj = r % nj;
    const double* row = y + g.at(sp.ilo - 1, sp.jlo - 1 + jj, k);
    for (int64_t ii = threadIdx.x; ii < ni; ii += kRedThreads) acc += __ldg(row + ii);
  }
  const double s = block_sum(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kRedThreads) k_sum_partials(const double* __restrict__ partials,
                                                              int n, double total,
                                                              double* __restrict__ result) {
  double acc = 0.0;
  for (int t = threadIdx.x; t < n; t += kRedThreads) acc += partials[t];
  const double s = block_sum(acc);
  if (threadIdx.x == 0) *result = total + s;
}

// ---- ordered mode: the reference's acc-simulated order (interp.cpp:1080-1173) ---------
// every (i,j) iteration is one virtual thread whose private `total` starts at the identity
// and adds y(k,i,j) for k = 1..nz in order; the partials are then combined one by one,
// in linear-id order (i fastest, then j), starting from the initial value of `total`.
__global__ void __launch_bounds__(128) k_column_sums(const double* __restrict__ y, Grid3 g,
                                                     int64_t nz, Span sp,
                                                     double* __restrict__ col, int64_t ld) {
  const int64_t i = sp.ilo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t j = sp.jlo + static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y;
  if (i > sp.ihi || j > sp.jhi) return;
  const double* p = y + g.at(i - 1, j - 1, 0);
  double acc = 0.0;  // identity_for("+") (interp.cpp:167-171)
  for (int64_t k = 0; k < nz; ++k) acc += __ldg(p + k * g.plane);
  col[(j - sp.jlo) * ld + (i - sp.ilo)] = acc;
}

// one warp: the partials are staged through shared memory in 1024-value chunks (coalesced,
// the next chunk loaded while the current one is summed) and lane 0 adds them in order,
// 32 values per batch read ahead of the dependent DADD chain (8.2 cycles per add on B200:
// the chain is the floor of this mode, ~8.6 ms per 2 M columns)
__global__ void __launch_bounds__(32) k_ordered_total(const double* __restrict__ col, int64_t n,
                                                      double total, double* __restrict__ result) {
  constexpr int kChunk = 1024;
  __shared__ double buf[2][kChunk];
  const int lane = threadIdx.x;
  auto load = [&](int b, int64_t t0) {
#pragma unroll 4
    for (int q = lane; q < kChunk; q += 32) buf[b][q] = (t0 + q < n) ? __ldg(col + t0 + q) : 0.0;
  };
  double acc = total;
  load(0, 0);
  __syncwarp();
  int b = 0;
  for (int64_t t0 = 0; t0 < n; t0 += kChunk) {
    if (t0 + kChunk < n) load(b ^ 1, t0 + kChunk);
    if (lane == 0) {
      const int m = n - t0 < kChunk ? static_cast<int>(n - t0) : kChunk;
      int q = 0;
      for (; q + 32 <= m; q += 32) {
        double v[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = buf[b][q + r];
#pragma unroll
        for (int r = 0; r < 32; ++r) acc += v[r];
      }
      for (; q < m; ++q) acc += buf[b][q];
    }
    __syncwarp();
    b ^= 1;
  }
  if (lane == 0) *result = acc;
}
}  // namespace

cudaError_t launch_column_sums(const double* y, Grid3 g, int64_t nz, const Span& sp, double* col,
                               int64_t ld, cudaStream_t s) {
  if (span_empty(sp)) return cudaSuccess;
  dim3 block(32, 4);
  dim3 grid(static_cast<unsigned>((sp.ihi - sp.ilo + 1 + 31) / 32),
            static_cast<unsigned>((sp.jhi - sp.jlo + 1 + 3) / 4));
  k_column_sums<<<grid, block, 0, s>>>(y, g, nz, sp, col, ld);
  return cudaGetLastError();
}

cudaError_t launch_ordered_total(const double* col, int64_t n, double total, double* result,
                                 cudaStream_t s) {
  k_ordered_total<<<1, 32, 0, s>>>(col, n, total, result);
  return cudaGetLastError();
}

int64_t reduce_partials_needed() { return kRedBlocks; }

cudaError_t launch_grid_sum(const double* y, Grid3 g, int64_t nz, const Span& sp,
                            double* partials, double* result, double total, cudaStream_t s) {
  if (span_empty(sp) || nz <= 0) {
    k_sum_partials<<<1, kRedThreads, 0, s>>>(partials, 0, total, result);
    return cudaGetLastError();
  }
  k_sum_rows<<<kRedBlocks, kRedThreads, 0, s>>>(y, g, nz, sp, partials);
  k_sum_partials<<<1, kRedThreads, 0, s>>>(partials, kRedBlocks, total, result);
  return cudaGetLastError();
}

// ============================================================================
// apps/dycore/dycore.h90
// ============================================================================
DynConst make_dyn_const(double dt, double rdx, double rdy, double rdz, double cs2, double grav,
                        double th0) {
  DynConst c;
  c.dt = dt;
  c.rdx = rdx;
  c.rdy = rdy;
  c.rdz = rdz;
  c.cs2 = cs2;
  c.grav = grav;
  c.th0 = th0;
  c.dt_rdx = dt * rdx;                    // `dt * rdx * (...)`
  c.dt_rdy = dt * rdy;
  c.dt_rdz = dt * rdz;                    // `dt * rdz * (...) / rf`
  c.dt_cs2 = dt * cs2;                    // `dt * cs2 * (...)`
  c.dt_cs2_rdz = dt * cs2 * rdz;          // `dt * cs2 * rdz * (...)`
  c.beta_num = dt * dt * cs2 * rdz * rdz; // `dt * dt * cs2 * rdz * rdz / rf`
  c.dt_grav = dt * grav;                  // `dt * grav * (...) / th0`
  return c;
}

namespace {
__device__ __forceinline__ double minmod(double a, double b) {
  // dycore.h90 `minmod`
  if (a * b <= 0.0) return 0.0;
  if (fabs(a) < fabs(b)) return a;
  return b;
}

// Upwind limited flux through face f (between cells f and f+1) of a dimension with
// n cells: walls at f = 0 and f = n (dycore.h90 regions 1-3).
__device__ __forceinline__ double face_flux(int64_t f, int64_t n, double vel, double tm1,
                                            double t0, double tp1, double tp2) {
  if (f == 0 || f == n) return 0.0;
  if (vel >= 0.0) {
    const double s = (f == 1) ? 0.0 : minmod(t0 - tm1, tp1 - t0);
    return vel * (t0 + 0.5 * s);
  }
  const double s = (f + 1 == n) ? 0.0 : minmod(tp1 - t0, tp2 - tp1);
  return vel * (tp1 - 0.5 * s);
}

struct AdvArgs {
  DynIn in;
  double* __restrict__ thn;
  Grid3 g;
  int nz;
  DynConst c;
  Span sp;
};

// Regions 1-4 fused: the x/y/z face fluxes are recomputed per cell from theta
// (each face is computed by both adjacent cells with identical inputs, so the bits
// match the materialised fx/fy/fz of the reference), then the flux divergence with
// the velocity-divergence correction. K-window of theta in registers; the next
// level's 13 loads are issued before the current level is computed (software
// pipelining: two levels of loads in flight per thread).
struct AdvLevel {
  double xm2, xm1, xp1, xp2, ym2, ym1, yp1, yp2, ui, uim1, vj, vjm1, w, tkp2;
};

__device__ __forceinline__ AdvLevel adv_load(const double* __restrict__ th,
                                             const double* __restrict__ u,
                                             const double* __restrict__ v,
                                             const double* __restrict__ w, int64_t off,
                                             int64_t W, int64_t off_kp2, bool has_kp2) {
  AdvLevel L;
  const double* r = th + off;
  L.xm2 = __ldg(r - 2);
  L.xm1 = __ldg(r - 1);
  L.xp1 = __ldg(r + 1);
  L.xp2 = __ldg(r + 2);
  L.ym2 = __ldg(r - 2 * W);
  L.ym1 = __ldg(r - W);
  L.yp1 = __ldg(r + W);
  L.yp2 = __ldg(r + 2 * W);
  L.ui = __ldg(u + off);
  L.uim1 = __ldg(u + off - 1);
  L.vj = __ldg(v + off);
  L.vjm1 = __ldg(v + off - W);
  L.w = __ldg(w + off);
  L.tkp2 = has_kp2 ? __ldg(th + off_kp2) : 0.0;
  return L;
}

__global__ void __launch_bounds__(128) k_dyn_advect(AdvArgs a) {
  const int64_t i = a.sp.ilo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t j = a.sp.jlo + static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y;
  if (i > a.sp.ihi || j > a.sp.jhi) return;
  const int64_t gi = i + a.sp.i0, gj = j + a.sp.j0, gnx = a.sp.gnx, gny = a.sp.gny;
  const int64_t P = a.g.plane, W = a.g.pitch;
  const int64_t col = (j - 1) * W + (i - 1);
  const double* __restrict__ th = a.in.th + col;
  const double* __restrict__ u = a.in.u + col;
  const double* __restrict__ v = a.in.v + col;
  const double* __restrict__ w = a.in.w + col;
  double* __restrict__ thn = a.thn + col;
  const int nz = a.nz;
  const DynConst& c = a.c;
  const bool east = gi == gnx, west = gi == 1, north = gj == gny, south = gj == 1;

  double tkm1 = 0.0;
  double tk = __ldg(th);
  double tkp1 = nz >= 2 ? __ldg(th + P) : 0.0;
  double fzm = 0.0;   // fz(k-1), fz(0) = 0 (ground)
  double wkm1 = 0.0;  // w(k-1)
  AdvLevel cur = adv_load(th, u, v, w, 0, W, 2 * P, nz >= 3);
  for (int k = 1; k <= nz; ++k) {
    AdvLevel nxt;
    if (k < nz) {
      const int64_t o = static_cast<int64_t>(k) * P;
      nxt = adv_load(th, u, v, w, o, W, static_cast<int64_t>(k + 2) * P, k + 3 <= nz);
    }
    const double tkp2 = cur.tkp2;
    const double wk = cur.w;
    const double fzk = face_flux(k, nz, wk, tkm1, tk, tkp1, tkp2);
    const double fxe = face_flux(gi, gnx, cur.ui, cur.xm1, tk, cur.xp1, cur.xp2);
    const double fxw = face_flux(gi - 1, gnx, cur.uim1, cur.xm2, cur.xm1, tk, cur.xp1);
    const double fyn = face_flux(gj, gny, cur.vj, cur.ym1, tk, cur.yp1, cur.yp2);
    const double fys = face_flux(gj - 1, gny, cur.vjm1, cur.ym2, cur.ym1, tk, cur.yp1);
    const double ue = east ? 0.0 : cur.ui;
    const double uw = west ? 0.0 : cur.uim1;
    const double vnf = north ? 0.0 : cur.vj;
    const double vs = south ? 0.0 : cur.vjm1;
    const double wt = (k == nz) ? 0.0 : wk;
    const double wb = (k == 1) ? 0.0 : wkm1;
    double flux = c.rdx * (fxe - fxw) + c.rdy * (fyn - fys);
    flux = flux + c.rdz * (fzk - fzm);
    double div = c.rdx * (ue - uw) + c.rdy * (vnf - vs);
    div = div + c.rdz * (wt - wb);
    thn[static_cast<int64_t>(k - 1) * P] = tk - c.dt * (flux - tk * div);
    fzm = fzk;
    wkm1 = wk;
    tkm1 = tk;
    tk = tkp1;
    tkp1 = tkp2;
    cur = nxt;
  }
}

struct AcoArgs {
  DynIn in;
  DynOut out;
  Grid3 g;
  int nz;
  DynConst c;
  Span sp;
};

struct AcoLevel {
  double pk, pe, pw, pnn, psth, uk, ukw, vk, vks, rho, th, w;
};

__device__ __forceinline__ AcoLevel aco_load(const DynIn& in, int64_t col, int64_t off,
                                             int64_t W) {
  AcoLevel L;
  const double* p = in.p + col + off;
  L.pk = __ldg(p);
  L.pe = __ldg(p + 1);
  L.pw = __ldg(p - 1);
  L.pnn = __ldg(p + W);
  L.psth = __ldg(p - W);
  L.uk = __ldg(in.u + col + off);
  L.ukw = __ldg(in.u + col + off - 1);
  L.vk = __ldg(in.v + col + off);
  L.vks = __ldg(in.v + col + off - W);
  L.rho = __ldg(in.rho + col + off);
  L.th = __ldg(in.th + col + off);
  L.w = __ldg(in.w + col + off);
  return L;
}

// Regions 5-7 fused: horizontal pressure gradient (new u, v), the pressure after the
// horizontal divergence (ps; the western/southern new velocities are recomputed from
// p and u/v instead of being re-read), and the HE-VI Thomas sweep for w with the
// pressure update, in one forward and one backward K sweep per column.
// On-chip budget: the Thomas coefficient cp(k) stays in shared memory ([k][thread],
// conflict-free); dp(k) and ps(k) make an L2 round trip through the OUTPUT arrays
// themselves (wn and pn hold dp and ps after the forward sweep and are overwritten
// with the final w and p in the backward sweep, so DRAM sees only the final values).
// This keeps shared memory at nz*8 B per thread, i.e. ~15 resident warps per SM.
__global__ void __launch_bounds__(128) k_dyn_acoustic(AcoArgs a) {
  extern __shared__ double smem[];
  const int T = blockDim.x * blockDim.y;
  const int t = threadIdx.y * blockDim.x + threadIdx.x;
  const int64_t i = a.sp.ilo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t j = a.sp.jlo + static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y;
  if (i > a.sp.ihi || j > a.sp.jhi) return;
  const int nz = a.nz;
  double* cps = smem + t;
  const int64_t gi = i + a.sp.i0, gj = j + a.sp.j0;
  const bool east = gi == a.sp.gnx, west = gi == 1, north = gj == a.sp.gny, south = gj == 1;
  const int64_t P = a.g.plane, W = a.g.pitch;
  const int64_t col = (j - 1) * W + (i - 1);
  double* un = a.out.u + col;
  double* vn = a.out.v + col;
  double* wn = a.out.w + col;  // holds dp(k) between the sweeps
  double* pn = a.out.p + col;  // holds ps(k) between the sweeps
  const DynConst& c = a.c;

  double rho_prev = 0.0, th_prev = 0.0, ps_prev = 0.0, w_prev = 0.0, cp_prev = 0.0,
         dp_prev = 0.0;
  AcoLevel cur = aco_load(a.in, col, 0, W);
  for (int k = 1; k <= nz; ++k) {
    AcoLevel nxt;
    if (k < nz) nxt = aco_load(a.in, col, static_cast<int64_t>(k) * P, W);
    const int64_t off = static_cast<int64_t>(k - 1) * P;
    const double pk = cur.pk;
    const double unk = east ? 0.0 : cur.uk - c.dt_rdx * (cur.pe - pk);
    const double vnk = north ? 0.0 : cur.vk - c.dt_rdy * (cur.pnn - pk);
    const double uw = west ? 0.0 : cur.ukw - c.dt_rdx * (pk - cur.pw);
    const double vs = south ? 0.0 : cur.vks - c.dt_rdy * (pk - cur.psth);
    const double psk = pk - c.dt_cs2 * (c.rdx * (unk - uw) + c.rdy * (vnk - vs));
    un[off] = unk;
    vn[off] = vnk;
    pn[off] = psk;
    if (k >= 2) {
      const int kf = k - 1;  // face kf + 1/2 between levels kf and kf + 1
      const double rf = 0.5 * (rho_prev + cur.rho);
      const double beta = c.beta_num / rf;
      double dd = w_prev - c.dt_rdz * (psk - ps_prev) / rf;
      dd = dd + c.dt_grav * (0.5 * (th_prev + cur.th) - c.th0) / c.th0;
      const double bb = 1.0 + 2.0 * beta;
      double cpk, dpk;
      if (kf == 1) {
        cpk = -beta / bb;
        dpk = dd / bb;
      } else {
        const double m = bb + beta * cp_prev;
        cpk = -beta / m;
        dpk = (dd + beta * dp_prev) / m;
      }
      cps[static_cast<int64_t>(kf - 1) * T] = cpk;
      wn[static_cast<int64_t>(kf - 1) * P] = dpk;
      cp_prev = cpk;
      dp_prev = dpk;
    }
    rho_prev = cur.rho;
    th_prev = cur.th;
    w_prev = cur.w;
    ps_prev = psk;
    cur = nxt;
  }
  // backward sweep: w at faces nz-1 .. 1 (w(nz) = 0 is the lid), pressure update.
  // dp(k) / ps(k+1) were written by this thread (same-thread RAW through L2: plain
  // loads, not the read-only path); they are fetched one level ahead.
  wn[static_cast<int64_t>(nz - 1) * P] = 0.0;
  double wk1 = 0.0;  // w(k+1)
  double dpk = wn[static_cast<int64_t>(nz - 2) * P];
  double psk1 = pn[static_cast<int64_t>(nz - 1) * P];
  for (int k = nz - 1; k >= 1; --k) {
    double dp_next = 0.0, ps_next = 0.0;
    if (k >= 2) {
      dp_next = wn[static_cast<int64_t>(k - 2) * P];
      ps_next = pn[static_cast<int64_t>(k - 1) * P];
    }
    const double wk = (k == nz - 1) ? dpk : dpk - cps[static_cast<int64_t>(k - 1) * T] * wk1;
    wn[static_cast<int64_t>(k - 1) * P] = wk;
    pn[static_cast<int64_t>(k) * P] = psk1 - c.dt_cs2_rdz * (wk1 - wk);
    wk1 = wk;
    dpk = dp_next;
    psk1 = ps_next;
  }
  pn[0] = pn[0] - c.dt_cs2_rdz * wk1;
}
}  // namespace

cudaError_t launch_dycore_advect(const DynIn& in, double* thn, Grid3 g, int64_t nz,
                                 const DynConst& c, const Span& sp, cudaStream_t s) {
  if (span_empty(sp) || nz <= 0) return cudaSuccess;
  dim3 block(32, 4);
  AdvArgs a{in, thn, g, static_cast<int>(nz), c, sp};
  k_dyn_advect<<<span_grid(sp, block), block, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_dycore_acoustic(const DynIn& in, const DynOut& out, Grid3 g, int64_t nz,
                                   const DynConst& c, const Span& sp, cudaStream_t s) {
  if (span_empty(sp) || nz < 2) return cudaSuccess;
  // pick the block height that maximises resident warps under the shared-memory budget
  // (cp: nz doubles per thread) and the 128-thread launch bound
  const size_t smem_cap = 227 * 1024;
  int best_by = 1, best_warps = 0;
  for (int by = 1; by <= 4; ++by) {
    size_t per_block = static_cast<size_t>(nz) * 32 * by * sizeof(double);
    if (per_block > smem_cap) break;
    int blocks = static_cast<int>(std::min<size_t>(smem_cap / (per_block + 1024), 32 / by));
    int warps = blocks * by;
    if (warps >= best_warps) {
      best_warps = warps;
      best_by = by;
    }
  }
  if (best_warps == 0) return cudaErrorInvalidConfiguration;
  dim3 block(32, best_by);
  size_t smem = static_cast<size_t>(nz) * block.x * block.y * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(k_dyn_acoustic), smem);
    if (e != cudaSuccess) return e;
  }
  AcoArgs a{in, out, g, static_cast<int>(nz), c, sp};
  k_dyn_acoustic<<<span_grid(sp, block), block, smem, s>>>(a);
  return cudaGetLastError();
}

// ============================================================================
// apps/dycore/dycore.h90 column_physics — one thread per column, one K pass:
// relaxation toward the previous column mean, bulk surface heat flux at k = 1, the new
// density-weighted column mean (sequential column sum, the dialect's order).
// ============================================================================
namespace {
__global__ void __launch_bounds__(128) k_column_physics(const double* __restrict__ rho,
                                                        double* __restrict__ th,
                                                        const double* __restrict__ u,
                                                        const double* __restrict__ v, Grid3 g,
                                                        int nz, DynConst c, PhysArgs ph,
                                                        Span sp) {
  const int64_t i = sp.ilo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t j = sp.jlo + static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y;
  if (i > sp.ihi || j > sp.jhi) return;
  const int64_t col = (j - 1) * g.pitch + (i - 1);
  const double cmean = ph.colm[col];
  double cs = 0.0, cm = 0.0;
  for (int k = 0; k < nz; ++k) {
    const int64_t o = col + static_cast<int64_t>(k) * g.plane;
    const double r = __ldg(rho + o);
    double t = th[o];
    t = t - ph.dt_rrelax * (t - cmean);
    if (k == 0) {
      const double uu = __ldg(u + o), vv = __ldg(v + o);
      const double wspd = sqrt(uu * uu + vv * vv);
      t = t + ph.dt_ch * wspd * (__ldg(ph.tsfc + col) - t) * c.rdz / r;
    }
    th[o] = t;
    cs = cs + r * t;
    cm = cm + r;
  }
  ph.colm[col] = cs / cm;
}
}  // namespace

cudaError_t launch_column_physics(const double* rho, double* th, const double* u,
                                  const double* v, Grid3 g, int64_t nz, const DynConst& c,
                                  const PhysArgs& ph, const Span& sp, cudaStream_t s) {
  if (span_empty(sp) || nz <= 0) return cudaSuccess;
  dim3 block(32, 4);
  k_column_physics<<<span_grid(sp, block), block, 0, s>>>(rho, th, u, v, g,
                                                          static_cast<int>(nz), c, ph, sp);
  return cudaGetLastError();
}

// ============================================================================
// halo pack/unpack: box {ilo, ihi, jlo, jhi} (local 1-based) x all K levels
// ============================================================================
namespace {
__global__ void __launch_bounds__(256) k_pack_box(const double* __restrict__ field,
                                                  double* __restrict__ buf, Grid3 g,
                                                  int64_t bi0, int64_t bj0, int64_t nbi,
                                                  int64_t nbj, int64_t total) {
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    buf[t] = field[box_elem(g, bi0, bj0, nbi, nbj, t)];
}
__global__ void __launch_bounds__(256) k_unpack_box(double* __restrict__ field,
                                                    const double* __restrict__ buf, Grid3 g,
                                                    int64_t bi0, int64_t bj0, int64_t nbi,
                                                    int64_t nbj, int64_t total) {
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    field[box_elem(g, bi0, bj0, nbi, nbj, t)] = buf[t];
}
}  // namespace

void pack_box_host(const double* field, double* buf, Grid3 g, int64_t nk, const int64_t box[4],
                   bool pack) {
  const int64_t nbi = box[1] - box[0] + 1, nbj = box[3] - box[2] + 1;
  if (nbi <= 0 || nbj <= 0 || nk <= 0) return;
  const int64_t total = nbi * nbj * nk;
  for (int64_t t = 0; t < total; ++t) {
    const int64_t e = box_elem(g, box[0], box[2], nbi, nbj, t);
    if (pack)
      buf[t] = field[e];
    else
      const_cast<double*>(field)[e] = buf[t];
  }
}

cudaError_t launch_pack_box(const double* field, double* buf, Grid3 g, int64_t nk,
                            const int64_t box[4], bool pack, cudaStream_t s) {
  const int64_t nbi = box[1] - box[0] + 1, nbj = box[3] - box[2] + 1;
  if (nbi <= 0 || nbj <= 0 || nk <= 0) return cudaSuccess;
  const int64_t total = nbi * nbj * nk;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  if (pack)
    k_pack_box<<<blocks, 256, 0, s>>>(field, buf, g, box[0], box[2], nbi, nbj, total);
  else
    k_unpack_box<<<blocks, 256, 0, s>>>(const_cast<double*>(field), buf, g, box[0], box[2], nbi,
                                        nbj, total);
  return cudaGetLastError();
}

cudaError_t ensure_dynamic_smem(const void* kernel, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{dev, kernel}];
  if (smem <= have) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
  if (e == cudaSuccess) have = smem;
  return e;
}

// ---------------------------------------------------------------------------
// peer-memory halo transport
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_f64(double* p, double v) {
  asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// blockIdx.y: box; threads stride over the box's cells, i fastest (rows of the face are
// contiguous on both sides)
__global__ void __launch_bounds__(256) k_peer_push(const __grid_constant__ PeerPush p) {
  const PeerBox& b = p.box[blockIdx.y];
  const int64_t total = b.nbi * b.nbj * b.nk;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t ii = t % b.nbi, rest = t / b.nbi, jj = rest % b.nbj, k = rest / b.nbj;
    b.dst[b.gd.at(b.di0 - 1 + ii, b.dj0 - 1 + jj, k)] =
        b.src[b.gs.at(b.si0 - 1 + ii, b.sj0 - 1 + jj, k)];
  }
}

struct FlagList {
  uint64_t* f[16];
};

__global__ void k_peer_signal(FlagList fl, int n, uint64_t* epoch_ctr, uint64_t epoch_val) {
  // every push of this stream completed before this kernel started (stream order); the
  // system-scope fence makes them visible to whoever acquires the flag
  uint64_t epoch = epoch_val;
  if (epoch_ctr) {  // the counter is touched by this stream only
    epoch = *epoch_ctr + 1;
    *epoch_ctr = epoch;
  }
  __threadfence_system();
  for (int q = 0; q < n; ++q) st_release_sys(fl.f[q], epoch);
}

__global__ void k_peer_wait(FlagList fl, int n, const uint64_t* epoch_ctr, uint64_t epoch_val) {
  const int q = threadIdx.x;
  // the counter was written by this stream's previous signal
  const uint64_t epoch = epoch_ctr ? *epoch_ctr : epoch_val;
  if (q < n)
    while (ld_acquire_sys(fl.f[q]) < epoch) __nanosleep(128);
}

__global__ void k_peer_allreduce(const __grid_constant__ PeerReduce r) {
  const double v = *r.value;
  const int par = static_cast<int>(r.epoch & 1);
  for (int q = 0; q < r.n; ++q) st_relaxed_sys_f64(r.slots[q] + par * 64 + r.rank, v);
  __threadfence_system();
  for (int q = 0; q < r.n; ++q) st_release_sys(r.flags[q] + r.rank, r.epoch);
  for (int q = 0; q < r.n; ++q)
    while (ld_acquire_sys(r.my_flags + q) < r.epoch) __nanosleep(128);
  double acc = 0.0;  // rank order: every rank computes the identical total
  for (int q = 0; q < r.n; ++q) acc += r.my_slots[par * 64 + q];
  *r.value = acc;
}

}  // namespace

cudaError_t launch_peer_push(const PeerPush& p, cudaStream_t s) {
  if (p.n <= 0) return cudaSuccess;
  int64_t most = 0;
  for (int q = 0; q < p.n; ++q)
    most = std::max(most, p.box[q].nbi * p.box[q].nbj * p.box[q].nk);
  if (most == 0) return cudaSuccess;
  const unsigned bx = static_cast<unsigned>(std::min<int64_t>((most + 255) / 256, 64));
  k_peer_push<<<dim3(bx, static_cast<unsigned>(p.n)), 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_peer_signal(uint64_t* const* flags, int n, uint64_t* epoch, cudaStream_t s,
                               uint64_t epoch_val) {
  if (n <= 0) return cudaSuccess;
  if (n > 16) return cudaErrorInvalidValue;
  FlagList fl{};
  for (int q = 0; q < n; ++q) fl.f[q] = flags[q];
  k_peer_signal<<<1, 1, 0, s>>>(fl, n, epoch, epoch_val);
  return cudaGetLastError();
}

cudaError_t launch_peer_wait(const uint64_t* const* flags, int n, const uint64_t* epoch,
                             cudaStream_t s, uint64_t epoch_val) {
  if (n <= 0) return cudaSuccess;
  if (n > 16) return cudaErrorInvalidValue;
  FlagList fl{};
  for (int q = 0; q < n; ++q) fl.f[q] = const_cast<uint64_t*>(flags[q]);
  k_peer_wait<<<1, 32, 0, s>>>(fl, n, epoch, epoch_val);
  return cudaGetLastError();
}

cudaError_t launch_peer_allreduce(const PeerReduce& r, cudaStream_t s) {
  if (r.n < 1 || r.n > 64) return cudaErrorInvalidValue;
  k_peer_allreduce<<<1, 1, 0, s>>>(r);
  return cudaGetLastError();
}

}  // namespace hfb

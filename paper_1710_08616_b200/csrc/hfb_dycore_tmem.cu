// hfb_dycore_tmem.cu — the HE-VI acoustic kernel, B200 edition.
//
// Same arithmetic as dycore.h90 regions 5-7 (see k_dyn_acoustic in hfb_kernels.cu for
// the line-by-line mapping), different machine organisation:
//
//   * A CTA owns a 32 x 4 tile of (i,j) columns (warp w = row j0+w, lane = i0+lane) and
//     marches K. Each K-plane of the six input fields the tile needs (p with its
//     one-cell ring, u with i-1, v with j-1, rho, th, w) is staged into shared memory by
//     LDGSTS (cp.async, 16-B chunks, L1 bypass) through a kStages-deep ring, so ~6 planes
//     per CTA are in flight while the current one is computed (no per-thread register
//     prefetch, no redundant L1 traffic for the horizontal neighbours).
//   * The Thomas sweep needs cp(k), dp(k) for the back substitution and ps(k) for the
//     pressure update: 3 x nz doubles per column. cp and dp live in TENSOR MEMORY: each
//     thread owns one TMEM lane (warp w -> lanes 32w..32w+31) and writes its
//     coefficients with tcgen05.st; the back substitution reads four levels per
//     tcgen05.ld. ps lives in shared memory. Nothing makes a round trip through L2/HBM:
//     DRAM traffic is exactly the compulsory 10 x 8 B per grid point.
//   * Budget per CTA: 256 TMEM columns (cp: 0..127, dp: 128..255; nz <= 65), ring
//     kStages x 7 KB, ps nz x 1 KB -> two CTAs (8 warps) per SM share the 512 TMEM
//     columns and ~200 KB of shared memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

// The tolerance build of this file (Makefile: -fmad=true -DHFB_ARITH_FMA): the same
// kernels with a*b+c contracted to FMA, every entry point renamed *_fma; selected per
// context with hfb_set_option(ctx, "arith", "fma"). Results then differ from the
// reference's binary64 evaluation by rounding only (tests/test_gpu_tolerance.py).
#ifdef HFB_ARITH_FMA
#define launch_dycore_acoustic_tmem launch_dycore_acoustic_tmem_fma
#define dycore_acoustic_tmem_fits dycore_acoustic_tmem_fits_fma
#define launch_dycore_step_tmem launch_dycore_step_tmem_fma
#define dycore_step_tmem_fits dycore_step_tmem_fits_fma
#define dycore_step_ws_fits dycore_step_ws_fits_fma
#define launch_dycore_step_ws launch_dycore_step_ws_fma
#endif
#include <cuda.h>
#include <cudaTypedefs.h>

#include "hfb_kernels.cuh"
#include "hfb_sm100.cuh"
#include "hfb_fp64.cuh"
#include "hfb_tmap.cuh"

namespace hfb {

namespace {

constexpr int kTX = 32, kTY = 4, kThreads = kTX * kTY;
constexpr int kStages = 6;
// per-stage plane tiles (doubles): p rows j0-1..j0+4, cols i0-2..i0+33 (36);
// u rows j0..j0+3, cols i0-2..i0+31 (34); v rows j0-1..j0+3, cols i0..i0+31 (32);
// rho/th/w rows j0..j0+3, cols i0..i0+31 (32)
constexpr int kPW = 36, kPR = kTY + 2;
constexpr int kUW = 34, kUR = kTY;
constexpr int kVW = 32, kVR = kTY + 1;
constexpr int kSW = 32, kSR = kTY;
constexpr int kOffP = 0;
constexpr int kOffU = kOffP + kPW * kPR;
constexpr int kOffV = kOffU + kUW * kUR;
constexpr int kOffRho = kOffV + kVW * kVR;
constexpr int kOffTh = kOffRho + kSW * kSR;
constexpr int kOffW = kOffTh + kSW * kSR;
constexpr int kStageDoubles = kOffW + kSW * kSR;  // 896
constexpr int kChunks = kStageDoubles / 2;         // 16-B chunks per stage (448)
constexpr int kChunksPerThread = (kChunks + kThreads - 1) / kThreads;  // 4
constexpr int kTmemCols = 256;
constexpr int kDpCol = 128;

struct AcoTmemArgs {
  DynIn in;
  DynOut out;
  Grid3 g;
  int nz;
  int64_t nj;       // tile extents of the arrays (rows valid: -2 .. nj+1)
  int64_t row_lo, row_hi;  // valid element range inside a row: [-kIOff, pitch-kIOff-1]
  DynConst c;
  Span sp;
};

__global__ void __launch_bounds__(kThreads, 2) k_dyn_acoustic_tmem(AcoTmemArgs a) {
  extern __shared__ __align__(128) double smem[];
  __shared__ uint32_t tmem_base_slot;
  double* ring = smem;                                   // kStages * kStageDoubles
  double* ps_s = smem + kStages * kStageDoubles;         // nz * kThreads

  const int lane = threadIdx.x, warp = threadIdx.y;
  const int t = warp * kTX + lane;
  const int64_t i0 = a.sp.ilo + static_cast<int64_t>(blockIdx.x) * kTX;  // 1-based local
  const int64_t j0 = a.sp.jlo + static_cast<int64_t>(blockIdx.y) * kTY;
  const int64_t i = i0 + lane, j = j0 + warp;
  const bool active = i <= a.sp.ihi && j <= a.sp.jhi;
  const int nz = a.nz;
  const int64_t P = a.g.plane, W = a.g.pitch;
  const DynConst& c = a.c;

  // ---- TMEM allocation (warp 0), address broadcast through shared memory ----------
  if (warp == 0) sm100::tmem_alloc(&tmem_base_slot, kTmemCols);
  sm100::tmem_fence_before();
  __syncthreads();
  sm100::tmem_fence_after();
  const uint32_t tmem = tmem_base_slot + (static_cast<uint32_t>(32 * warp) << 16);

  // ---- this thread's copy chunks: (global source at plane 0, smem byte offset) -----
  const double* src[kChunksPerThread];
  uint32_t dst[kChunksPerThread];
  bool ok[kChunksPerThread];
  const uint32_t ring_u32 = sm100::smem_u32(ring);
#pragma unroll
  for (int q = 0; q < kChunksPerThread; ++q) {
    const int ch = t + q * kThreads;
    ok[q] = false;
    src[q] = a.in.p;
    dst[q] = 0;
    if (ch >= kChunks) continue;
    const int e = ch * 2;  // first double of the chunk inside the stage
    const double* base;
    int64_t row, col;      // 0-based local row (j') and column (i') of the chunk start
    if (e < kOffU) {
      base = a.in.p; row = (j0 - 2) + e / kPW; col = (i0 - 3) + e % kPW;
    } else if (e < kOffV) {
      base = a.in.u; row = (j0 - 1) + (e - kOffU) / kUW; col = (i0 - 3) + (e - kOffU) % kUW;
    } else if (e < kOffRho) {
      base = a.in.v; row = (j0 - 2) + (e - kOffV) / kVW; col = (i0 - 1) + (e - kOffV) % kVW;
    } else if (e < kOffTh) {
      base = a.in.rho; row = (j0 - 1) + (e - kOffRho) / kSW; col = (i0 - 1) + (e - kOffRho) % kSW;
    } else if (e < kOffW) {
      base = a.in.th; row = (j0 - 1) + (e - kOffTh) / kSW; col = (i0 - 1) + (e - kOffTh) % kSW;
    } else {
      base = a.in.w; row = (j0 - 1) + (e - kOffW) / kSW; col = (i0 - 1) + (e - kOffW) % kSW;
    }
    ok[q] = row >= -kHalo && row <= a.nj - 1 + kHalo && col >= a.row_lo && col + 1 <= a.row_hi;
    src[q] = base + row * W + col;
    dst[q] = ring_u32 + static_cast<uint32_t>(e) * 8u;
  }
  auto issue = [&](int k) {  // stage the 0-based level k into ring slot k % kStages
    if (k < nz) {
      const uint32_t so = static_cast<uint32_t>((k % kStages) * kStageDoubles * 8);
      const int64_t go = static_cast<int64_t>(k) * P;
#pragma unroll
      for (int q = 0; q < kChunksPerThread; ++q)
        if (ok[q]) sm100::cp_async16(dst[q] + so, src[q] + go);
    }
    sm100::cp_async_commit();
  };

  const int64_t col = (j - 1) * W + (i - 1);
  double* un = a.out.u + col;
  double* vn = a.out.v + col;
  double* wn = a.out.w + col;
  double* pn = a.out.p + col;
  const bool east = i + a.sp.i0 == a.sp.gnx, west = i + a.sp.i0 == 1;
  const bool north = j + a.sp.j0 == a.sp.gny, south = j + a.sp.j0 == 1;

#pragma unroll 1
  for (int k = 0; k < kStages - 1; ++k) issue(k);

  double rho_prev = 0.0, th_prev = 0.0, ps_prev = 0.0, w_prev = 0.0, cp_prev = 0.0,
         dp_prev = 0.0;
#pragma unroll 1
  for (int k = 0; k < nz; ++k) {  // 0-based level; dialect level kk = k + 1
    issue(k + kStages - 1);
    sm100::cp_async_wait<kStages - 1>();
    __syncthreads();
    const double* S = ring + (k % kStages) * kStageDoubles;
    const double* Pp = S + kOffP + (warp + 1) * kPW + (lane + 2);
    const double pk = Pp[0], pe = Pp[1], pw = Pp[-1], pnn = Pp[kPW], psth = Pp[-kPW];
    const double* Up = S + kOffU + warp * kUW + (lane + 2);
    const double uk = Up[0], ukw = Up[-1];
    const double* Vp = S + kOffV + (warp + 1) * kVW + lane;
    const double vk = Vp[0], vks = Vp[-kVW];
    const double rhok = S[kOffRho + warp * kSW + lane];
    const double thk = S[kOffTh + warp * kSW + lane];
    const double wk = S[kOffW + warp * kSW + lane];

    const double unk = east ? 0.0 : uk - c.dt_rdx * (pe - pk);
    const double vnk = north ? 0.0 : vk - c.dt_rdy * (pnn - pk);
    const double uw = west ? 0.0 : ukw - c.dt_rdx * (pk - pw);
    const double vs = south ? 0.0 : vks - c.dt_rdy * (pk - psth);
    const double psk = pk - c.dt_cs2 * (c.rdx * (unk - uw) + c.rdy * (vnk - vs));
    if (active) {
      un[static_cast<int64_t>(k) * P] = unk;
      vn[static_cast<int64_t>(k) * P] = vnk;
    }
    ps_s[k * kThreads + t] = psk;
    if (k >= 1) {
      const int f = k - 1;  // 0-based face between levels k-1 and k (dialect kf = k)
      const double rf = 0.5 * (rho_prev + rhok);
      const double beta = c.beta_num / rf;
      double dd = w_prev - c.dt_rdz * (psk - ps_prev) / rf;
      dd = dd + c.dt_grav * (0.5 * (th_prev + thk) - c.th0) / c.th0;
      const double bb = 1.0 + 2.0 * beta;
      double cpk, dpk;
      if (f == 0) {
        cpk = -beta / bb;
        dpk = dd / bb;
      } else {
        const double m = bb + beta * cp_prev;
        cpk = -beta / m;
        dpk = (dd + beta * dp_prev) / m;
      }
      sm100::tmem_st_f64(tmem + 2 * f, cpk);
      sm100::tmem_st_f64(tmem + kDpCol + 2 * f, dpk);
      cp_prev = cpk;
      dp_prev = dpk;
    }
    rho_prev = rhok;
    th_prev = thk;
    w_prev = wk;
    ps_prev = psk;
    __syncthreads();  // the slot is refilled by the next iteration's issue()
  }
  sm100::cp_async_wait<0>();
  sm100::tmem_wait_st();

  // ---- back substitution: faces nz-2 .. 0 (w(nz) = 0 is the lid), four per TMEM load
  if (active) wn[static_cast<int64_t>(nz - 1) * P] = 0.0;
  double wk1 = 0.0;  // w at the face above
  const int nf = nz - 1;
#pragma unroll 1
  for (int cb = (nf - 1) / 4; cb >= 0; --cb) {
    double cpv[4], dpv[4];
    sm100::tmem_ld_4f64(tmem + 8 * cb, cpv);
    sm100::tmem_ld_4f64(tmem + kDpCol + 8 * cb, dpv);
#pragma unroll
    for (int q = 3; q >= 0; --q) {
      const int f = 4 * cb + q;
      if (f >= nf) continue;
      const double wk = (f == nf - 1) ? dpv[q] : dpv[q] - cpv[q] * wk1;
      const double pk1 = ps_s[(f + 1) * kThreads + t] - c.dt_cs2_rdz * (wk1 - wk);
      if (active) {
        wn[static_cast<int64_t>(f) * P] = wk;
        pn[static_cast<int64_t>(f + 1) * P] = pk1;
      }
      wk1 = wk;
    }
  }
  if (active) pn[0] = ps_s[t] - c.dt_cs2_rdz * wk1;

  sm100::tmem_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem_base_slot, kTmemCols);
}

}  // namespace

bool dycore_acoustic_tmem_fits(int64_t nz) { return nz >= 2 && nz - 1 <= 64; }

cudaError_t launch_dycore_acoustic_tmem(const DynIn& in, const DynOut& out, Grid3 g,
                                        int64_t nz, int64_t nj, const DynConst& c,
                                        const Span& sp, cudaStream_t s) {
  if (sp.ihi < sp.ilo || sp.jhi < sp.jlo) return cudaSuccess;
  if (!dycore_acoustic_tmem_fits(nz)) return cudaErrorInvalidValue;
  // at most two CTAs per SM: they share the SM's 512 TMEM columns (256 each); a third
  // CTA would block in tcgen05.alloc, so small-nz launches pad their shared memory
  const size_t smem = std::max<size_t>((static_cast<size_t>(kStages) * kStageDoubles +
                                        static_cast<size_t>(nz) * kThreads) * sizeof(double),
                                       80 * 1024);
  {
    cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(k_dyn_acoustic_tmem), smem);
    if (e != cudaSuccess) return e;
  }
  AcoTmemArgs a{in, out, g, static_cast<int>(nz), nj, -kIOff, g.pitch - kIOff - 1, c, sp};
  dim3 block(kTX, kTY);
  dim3 grid(static_cast<unsigned>((sp.ihi - sp.ilo + 1 + kTX - 1) / kTX),
            static_cast<unsigned>((sp.jhi - sp.jlo + 1 + kTY - 1) / kTY));
  k_dyn_acoustic_tmem<<<grid, block, smem, s>>>(a);
  return cudaGetLastError();
}


// ===========================================================================
// The whole dycore timestep in ONE kernel (dycore.h90 regions 1-8): flux-limited
// advection of theta + horizontal pressure gradient + divergence + HE-VI Thomas
// sweep, reading rho, th, u, v, w, p once and writing th', u', v', w', p' once:
// 88 compulsory bytes per grid point (the two-kernel split needs 120).
// Advection is independent of the Thomas recurrence, so its arithmetic fills the
// latency of the division chain (the acoustic kernel alone is bound by fp64 latency).
// ===========================================================================
namespace {

// fused stage: th rows j0-2..j0+5 (8) x cols i0-2..i0+33 (36); u 4 x 34; v 5 x 32;
// w 4 x 32; p 6 x 36; rho 4 x 32
constexpr int kFThW = 36, kFThR = kTY + 4;
constexpr int kFOffTh = 0;
constexpr int kFOffU = kFOffTh + kFThW * kFThR;
constexpr int kFOffV = kFOffU + kUW * kUR;
constexpr int kFOffW = kFOffV + kVW * kVR;
constexpr int kFOffP = kFOffW + kSW * kSR;
constexpr int kFOffRho = kFOffP + kPW * kPR;
constexpr int kFStageDoubles = kFOffRho + kSW * kSR;  // 1056
constexpr int kFChunks = kFStageDoubles / 2;          // 528
constexpr int kFChunksPerThread = (kFChunks + kThreads - 1) / kThreads;  // 5
constexpr int kFStages = 6;

// minmod and the limited upwind face flux, branch-free (both upwind candidates are
// formed and one is selected: identical bits to the branching dialect code, no warp
// divergence on the sign of the face velocity)
__device__ __forceinline__ double minmod_sel(double a, double b) {
  const double m = fabs(a) < fabs(b) ? a : b;
  return (a * b <= 0.0) ? 0.0 : m;
}
__device__ __forceinline__ double face_flux_sel(int64_t f, int64_t n, double vel, double tm1,
                                                double t0, double tp1, double tp2) {
  const double d0 = t0 - tm1, d1 = tp1 - t0, d2 = tp2 - tp1;
  const double sp = (f == 1) ? 0.0 : minmod_sel(d0, d1);
  const double sm = (f + 1 == n) ? 0.0 : minmod_sel(d1, d2);
  const double fp = vel * (t0 + 0.5 * sp);
  const double fm = vel * (tp1 - 0.5 * sm);
  const double fv = vel >= 0.0 ? fp : fm;
  return (f == 0 || f == n) ? 0.0 : fv;
}

struct StepTmemArgs {
  DynIn in;
  DynOut out;
  Grid3 g;
  int nz;
  // roles this launch computes: bit 0 = advection, bit 1 = acoustic/HE-VI. Always 3 in
  // the product (launch_dycore_step_ws); the A/B build's timing experiments clear one
  // (hfb_set_option debug_skip). A runtime value on purpose: folding it to a constant
  // changes the register allocation of the 128-register kernel and costs ~2%.
  int roles;
  // column physics fused into the advection warps (full_step); null when off
  const double* tsfc;
  double* colm;
  double dt_rrelax, dt_ch;
  // RK3 stages 2-3: the state at the start of the step (th, u, v, w, p; rho unused)
  DynIn base;
  int64_t nj;
  int64_t row_lo, row_hi;
  DynConst c;
  Span sp;
  // tile order of the warp-specialised kernel (1-D grid): the rim first, then the tiles
  // of the rectangle [tx_lo, tx_hi] x [ty_lo, ty_hi] that need no boundary cases
  int ntx, nty, tx_lo, tx_hi, ty_lo, ty_hi;
};

__global__ void __launch_bounds__(kThreads, 2) k_dyn_step_tmem(StepTmemArgs a) {
  extern __shared__ __align__(128) double smem[];
  __shared__ uint32_t tmem_base_slot;
  double* ring = smem;
  double* ps_s = smem + kFStages * kFStageDoubles;

  const int lane = threadIdx.x, warp = threadIdx.y;
  const int t = warp * kTX + lane;
  const int64_t i0 = a.sp.ilo + static_cast<int64_t>(blockIdx.x) * kTX;
  const int64_t j0 = a.sp.jlo + static_cast<int64_t>(blockIdx.y) * kTY;
  const int64_t i = i0 + lane, j = j0 + warp;
  const bool active = i <= a.sp.ihi && j <= a.sp.jhi;
  const int nz = a.nz;
  const int64_t P = a.g.plane, W = a.g.pitch;
  const DynConst& c = a.c;
  const int64_t gi = i + a.sp.i0, gj = j + a.sp.j0, gnx = a.sp.gnx, gny = a.sp.gny;

  if (warp == 0) sm100::tmem_alloc(&tmem_base_slot, kTmemCols);
  sm100::tmem_fence_before();
  __syncthreads();
  sm100::tmem_fence_after();
  const uint32_t tmem = tmem_base_slot + (static_cast<uint32_t>(32 * warp) << 16);

  const double* src[kFChunksPerThread];
  uint32_t dst[kFChunksPerThread];
  bool ok[kFChunksPerThread];
  const uint32_t ring_u32 = sm100::smem_u32(ring);
#pragma unroll
  for (int q = 0; q < kFChunksPerThread; ++q) {
    const int ch = t + q * kThreads;
    ok[q] = false;
    src[q] = a.in.p;
    dst[q] = 0;
    if (ch >= kFChunks) continue;
    const int e = ch * 2;
    const double* base;
    int64_t row, col;  // 0-based local (j', i') of the chunk start
    if (e < kFOffU) {
      base = a.in.th; row = (j0 - 3) + e / kFThW; col = (i0 - 3) + e % kFThW;
    } else if (e < kFOffV) {
      base = a.in.u; row = (j0 - 1) + (e - kFOffU) / kUW; col = (i0 - 3) + (e - kFOffU) % kUW;
    } else if (e < kFOffW) {
      base = a.in.v; row = (j0 - 2) + (e - kFOffV) / kVW; col = (i0 - 1) + (e - kFOffV) % kVW;
    } else if (e < kFOffP) {
      base = a.in.w; row = (j0 - 1) + (e - kFOffW) / kSW; col = (i0 - 1) + (e - kFOffW) % kSW;
    } else if (e < kFOffRho) {
      base = a.in.p; row = (j0 - 2) + (e - kFOffP) / kPW; col = (i0 - 3) + (e - kFOffP) % kPW;
    } else {
      base = a.in.rho; row = (j0 - 1) + (e - kFOffRho) / kSW; col = (i0 - 1) + (e - kFOffRho) % kSW;
    }
    ok[q] = row >= -kHalo && row <= a.nj - 1 + kHalo && col >= a.row_lo && col + 1 <= a.row_hi;
    src[q] = base + row * W + col;
    dst[q] = ring_u32 + static_cast<uint32_t>(e) * 8u;
  }
  auto issue = [&](int k) {
    if (k < nz) {
      const uint32_t so = static_cast<uint32_t>((k % kFStages) * kFStageDoubles * 8);
      const int64_t go = static_cast<int64_t>(k) * P;
#pragma unroll
      for (int q = 0; q < kFChunksPerThread; ++q)
        if (ok[q]) sm100::cp_async16(dst[q] + so, src[q] + go);
    }
    sm100::cp_async_commit();
  };

  const int64_t col = (j - 1) * W + (i - 1);
  double* thn = a.out.th + col;
  double* un = a.out.u + col;
  double* vn = a.out.v + col;
  double* wn = a.out.w + col;
  double* pn = a.out.p + col;
  const bool east = gi == gnx, west = gi == 1, north = gj == gny, south = gj == 1;
  const int thc = (warp + 2) * kFThW + (lane + 2);  // this column inside a th plane tile

#pragma unroll 1
  for (int k = 0; k < kFStages - 1; ++k) issue(k);

  double rho_prev = 0.0, th_prev = 0.0, ps_prev = 0.0, w_prev = 0.0, cp_prev = 0.0,
         dp_prev = 0.0, fz_prev = 0.0;
#pragma unroll 1
  for (int k = 0; k < nz; ++k) {  // 0-based level; dialect level kk = k + 1
    issue(k + kFStages - 1);
    sm100::cp_async_wait<kFStages - 4>();  // levels <= k+2 have landed (own copies)
    __syncthreads();                       // ... and everyone else's
    const int kk = k + 1;
    const double* S = ring + (k % kFStages) * kFStageDoubles;
    const double* T0 = S + kFOffTh + thc;
    const double tk = T0[0];
    const double tkp1 = (kk + 1 <= nz) ? ring[((k + 1) % kFStages) * kFStageDoubles + kFOffTh + thc] : 0.0;
    const double tkp2 = (kk + 2 <= nz) ? ring[((k + 2) % kFStages) * kFStageDoubles + kFOffTh + thc] : 0.0;
    const double xm2 = T0[-2], xm1 = T0[-1], xp1 = T0[1], xp2 = T0[2];
    const double ym2 = T0[-2 * kFThW], ym1 = T0[-kFThW], yp1 = T0[kFThW], yp2 = T0[2 * kFThW];
    const double* Up = S + kFOffU + warp * kUW + (lane + 2);
    const double ui = Up[0], uim1 = Up[-1];
    const double* Vp = S + kFOffV + (warp + 1) * kVW + lane;
    const double vj = Vp[0], vjm1 = Vp[-kVW];
    const double wk = S[kFOffW + warp * kSW + lane];
    const double* Pp = S + kFOffP + (warp + 1) * kPW + (lane + 2);
    const double pk = Pp[0], pe = Pp[1], pw = Pp[-1], pnn = Pp[kPW], psth = Pp[-kPW];
    const double rhok = S[kFOffRho + warp * kSW + lane];

    // ---- advection (regions 1-4) --------------------------------------------------
    const double fzk = face_flux_sel(kk, nz, wk, th_prev, tk, tkp1, tkp2);
    const double fxe = face_flux_sel(gi, gnx, ui, xm1, tk, xp1, xp2);
    const double fxw = face_flux_sel(gi - 1, gnx, uim1, xm2, xm1, tk, xp1);
    const double fyn = face_flux_sel(gj, gny, vj, ym1, tk, yp1, yp2);
    const double fys = face_flux_sel(gj - 1, gny, vjm1, ym2, ym1, tk, yp1);
    const double ue = east ? 0.0 : ui;
    const double uwf = west ? 0.0 : uim1;
    const double vnf = north ? 0.0 : vj;
    const double vsf = south ? 0.0 : vjm1;
    const double wt = (kk == nz) ? 0.0 : wk;
    const double wb = (kk == 1) ? 0.0 : w_prev;
    double flux = c.rdx * (fxe - fxw) + c.rdy * (fyn - fys);
    flux = flux + c.rdz * (fzk - fz_prev);
    double div = c.rdx * (ue - uwf) + c.rdy * (vnf - vsf);
    div = div + c.rdz * (wt - wb);
    const double thk_new = tk - c.dt * (flux - tk * div);

    // ---- pressure gradient + divergence (regions 5-6) ------------------------------
    const double unk = east ? 0.0 : ui - c.dt_rdx * (pe - pk);
    const double vnk = north ? 0.0 : vj - c.dt_rdy * (pnn - pk);
    const double uw = west ? 0.0 : uim1 - c.dt_rdx * (pk - pw);
    const double vs = south ? 0.0 : vjm1 - c.dt_rdy * (pk - psth);
    const double psk = pk - c.dt_cs2 * (c.rdx * (unk - uw) + c.rdy * (vnk - vs));
    if (active) {
      const int64_t o = static_cast<int64_t>(k) * P;
      thn[o] = thk_new;
      un[o] = unk;
      vn[o] = vnk;
    }
    ps_s[k * kThreads + t] = psk;
    // ---- HE-VI forward elimination (region 7) --------------------------------------
    if (k >= 1) {
      const int f = k - 1;
      const double rf = 0.5 * (rho_prev + rhok);
      const double beta = c.beta_num / rf;
      double dd = w_prev - c.dt_rdz * (psk - ps_prev) / rf;
      dd = dd + c.dt_grav * (0.5 * (th_prev + tk) - c.th0) / c.th0;
      const double bb = 1.0 + 2.0 * beta;
      double cpk, dpk;
      if (f == 0) {
        cpk = -beta / bb;
        dpk = dd / bb;
      } else {
        const double m = bb + beta * cp_prev;
        cpk = -beta / m;
        dpk = (dd + beta * dp_prev) / m;
      }
      sm100::tmem_st_f64(tmem + 2 * f, cpk);
      sm100::tmem_st_f64(tmem + kDpCol + 2 * f, dpk);
      cp_prev = cpk;
      dp_prev = dpk;
    }
    rho_prev = rhok;
    th_prev = tk;
    w_prev = wk;
    ps_prev = psk;
    fz_prev = fzk;
    __syncthreads();
  }
  sm100::cp_async_wait<0>();
  sm100::tmem_wait_st();

  // ---- back substitution + pressure update (region 7), four faces per TMEM load ----
  if (active) wn[static_cast<int64_t>(nz - 1) * P] = 0.0;
  double wk1 = 0.0;
  const int nf = nz - 1;
#pragma unroll 1
  for (int cb = (nf - 1) / 4; cb >= 0; --cb) {
    double cpv[4], dpv[4];
    sm100::tmem_ld_4f64(tmem + 8 * cb, cpv);
    sm100::tmem_ld_4f64(tmem + kDpCol + 8 * cb, dpv);
#pragma unroll
    for (int q = 3; q >= 0; --q) {
      const int f = 4 * cb + q;
      if (f >= nf) continue;
      const double wk = (f == nf - 1) ? dpv[q] : dpv[q] - cpv[q] * wk1;
      const double pk1 = ps_s[(f + 1) * kThreads + t] - c.dt_cs2_rdz * (wk1 - wk);
      if (active) {
        wn[static_cast<int64_t>(f) * P] = wk;
        pn[static_cast<int64_t>(f + 1) * P] = pk1;
      }
      wk1 = wk;
    }
  }
  if (active) pn[0] = ps_s[t] - c.dt_cs2_rdz * wk1;

  sm100::tmem_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem_base_slot, kTmemCols);
}

}  // namespace

bool dycore_step_tmem_fits(int64_t nz) { return nz >= 2 && nz - 1 <= 64; }
// the warp-specialised step: 256 TMEM columns per CTA up to 64 faces, 512 up to 128 (the
// shared memory of such a column, ps included, then keeps one CTA per SM as well)
bool dycore_step_ws_fits(int64_t nz) { return nz >= 2 && nz - 1 <= 128; }

cudaError_t launch_dycore_step_tmem(const DynIn& in, const DynOut& out, Grid3 g, int64_t nz,
                                    int64_t nj, const DynConst& c, const Span& sp,
                                    cudaStream_t s) {
  if (sp.ihi < sp.ilo || sp.jhi < sp.jlo) return cudaSuccess;
  if (!dycore_step_tmem_fits(nz)) return cudaErrorInvalidValue;
  const size_t smem = std::max<size_t>((static_cast<size_t>(kFStages) * kFStageDoubles +
                                        static_cast<size_t>(nz) * kThreads) * sizeof(double),
                                       80 * 1024);
  {
    cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(k_dyn_step_tmem), smem);
    if (e != cudaSuccess) return e;
  }
  StepTmemArgs a{in,  out,     g,      static_cast<int>(nz), 3, nullptr, nullptr, 0.0, 0.0,
                 DynIn{}, nj, -kIOff, g.pitch - kIOff - 1, c, sp};
  dim3 block(kTX, kTY);
  dim3 grid(static_cast<unsigned>((sp.ihi - sp.ilo + 1 + kTX - 1) / kTX),
            static_cast<unsigned>((sp.jhi - sp.jlo + 1 + kTY - 1) / kTY));
  k_dyn_step_tmem<<<grid, block, smem, s>>>(a);
  return cudaGetLastError();
}


// ===========================================================================
// Warp-specialised fused timestep: the same 32 x 4 column tile and cp.async plane ring,
// but 8 warps per CTA — warps 0-3 run the acoustic/HE-VI part (they own the TMEM lanes
// holding the Thomas coefficients), warps 4-7 run the flux-limited advection of the same
// four rows. The two halves share every staged plane, split the fp64 work roughly in
// half and, with 2 CTAs per SM, double the resident warps (16) that hide the fp64
// dependency latency (the single-role kernel is bound by `stall_wait`).
// Tiles that touch no global boundary (all but a thin rim) take a boundary-free
// instantiation of the level body: no wall/limiter special cases, no selects for them.
// ===========================================================================
namespace {

constexpr int kWsThreads = 2 * kThreads;  // 256
// ring stage layout: the six plane tiles of a level (th, u, v, w, p, rho), each starting
// 128-B aligned (the TMA destination rule; the cp.async feed uses the same layout)
constexpr int pad16(int n) { return (n + 15) / 16 * 16; }
constexpr int kWOffTh = 0;
constexpr int kWOffU = kWOffTh + pad16(kFThW * kFThR);
constexpr int kWOffV = kWOffU + pad16(kUW * kUR);
constexpr int kWOffW = kWOffV + pad16(kVW * kVR);
constexpr int kWOffP = kWOffW + pad16(kSW * kSR);
constexpr int kWOffRho = kWOffP + pad16(kPW * kPR);
constexpr int kWStageDoubles = kWOffRho + pad16(kSW * kSR);  // 1072
constexpr uint32_t kWStageTx = kFStageDoubles * 8;            // bytes landing per level
#ifndef HFB_MID_UNROLL
#define HFB_MID_UNROLL 1
#endif
constexpr int kMidUnroll = HFB_MID_UNROLL;  // mid-column K loop unrolling
// ring depth: 6 planes x 8.25 KB (+ ps, nz x 1 KB, in shared memory: measured faster than
// an L2 round trip of ps with a 10-deep ring)
constexpr int kWsStages = 6;
constexpr int kWsChunksPerThread = (kFChunks + kWsThreads - 1) / kWsThreads;  // 3

// Limited upwind face flux with ONE minmod: the upwind side's slope pair and base value
// are selected first. vel*(tp1 - 0.5*s) == vel*(tp1 + (-0.5)*s) bit for bit (exact
// negation), so this equals the dialect's two-branch form. kCheck adds the wall and
// first/last-face cases (face index f of n cells).
template <bool kCheck>
__device__ __forceinline__ double face_flux_up(int64_t f, int64_t n, double vel, double tm1,
                                               double t0, double tp1, double tp2) {
  const double d0 = t0 - tm1, d1 = tp1 - t0, d2 = tp2 - tp1;
  const bool up = vel >= 0.0;
  const double x = up ? d0 : d1, y = up ? d1 : d2;
  const double m = fabs(x) < fabs(y) ? x : y;
  double sl = (x * y <= 0.0) ? 0.0 : m;
  if (kCheck) sl = (up ? f == 1 : f + 1 == n) ? 0.0 : sl;
  const double base = up ? t0 : tp1;
  const double h = up ? 0.5 : -0.5;
  const double fv = vel * (base + h * sl);
  if (kCheck) return (f == 0 || f == n) ? 0.0 : fv;
  return fv;
}

// which lateral boundary cases a tile's instantiation handles
template <bool kX, bool kY>
struct Chk {
  static constexpr bool x = kX, y = kY;
};

// The ring feed: TMA (the product: six 3-D box loads per level, one field each, issued by
// lane 0 of the acoustic warps 0-3; completion on the slot's mbarrier, observed by one advection warp
// at the end of its level, published to every warp by the per-level CTA barrier) or, in
// the A/B build flag HFB_WS_CPASYNC, cp.async (LDGSTS: every thread copies 2-3 16-B
// chunks per level and waits for its own; ~45 more instructions per warp and level).
#ifdef HFB_WS_CPASYNC
constexpr bool kTmaFeed = false;
#else
constexpr bool kTmaFeed = true;
#endif
#ifndef HFB_WAIT_WARP
#define HFB_WAIT_WARP 4
#endif
constexpr int kWaitWarp = HFB_WAIT_WARP;  // TMA feed: the warp that waits on the slots

template <bool kPhys, bool kRK, bool kRemote>
__global__ void __launch_bounds__(kWsThreads, 2)
    k_dyn_step_ws(const __grid_constant__ StepMaps maps, StepTmemArgs a,
                  const __grid_constant__ RemoteHalo rem) {
  // (the tensor maps come first: a CUtensorMap must sit 64-B aligned in parameter space)
  static_assert(!(kPhys && kRK), "column physics is not fused into RK stages");
  // (declared 16-B aligned only: the runtime places the dynamic segment right after the
  // 64 B of static shared memory, and a larger declared alignment would let the compiler
  // fold the 128-B round-up below to zero)
  extern __shared__ __align__(16) double smem_raw[];
  // static shared memory: the slot barriers and the TMEM address, 64 B in total, so the
  // dynamic segment starts 16-B aligned and the 128-B alignment below is exact
  __shared__ __align__(16) uint64_t sbar[8];
  static_assert(kWsStages < 8, "slot barriers");
  uint64_t* const full_bar = sbar;
  uint32_t& tmem_base_slot = *reinterpret_cast<uint32_t*>(&sbar[7]);
  // the ring starts 128-B aligned (TMA destinations; the launch adds the slack)
  // (offset arithmetic on the __shared__ array keeps the loads in the shared window)
  const uint32_t raw_u32 = sm100::smem_u32(smem_raw);
  double* ring = smem_raw + ((((raw_u32 + 127u) & ~127u) - raw_u32) >> 3);
  double* ps_s = ring + kWsStages * kWStageDoubles;  // nz x 128 (ps of each column)
  // kPhys: theta' of levels k-1 / k (parity), handed from the advection warps to the
  // acoustic warps, which accumulate the column sums (the halves stay balanced)
  double* thv_s = ps_s + a.nz * kThreads;

  // blockDim = (32, 8); the warp index shuffled from lane 0 is known warp-uniform: the
  // role branches are uniform and the TMA issue operands live in uniform registers (no
  // per-lane ELECT / R2UR.BROADCAST / BRA.U.ANY loop around UTMALDG; the allocation fell
  // from 124 to 102 registers in the dycore-step instantiation): C4 dycore step 2.557 ->
  // 2.478 ms, RK3 512^2 1.176 -> 1.123 ms (tools/gpu_r2zv.sh)
  const int lane = threadIdx.x, warp = sm100::warp_uniform(threadIdx.y);
  const bool acoustic = warp < kTY;
  const int row = acoustic ? warp : warp - kTY;       // tile row served by this warp
  const int tid = warp * kTX + lane;                  // 0..255 (copy issue)
  const int t = row * kTX + lane;                     // 0..127 (column within the tile)
  // CTA -> tile: the rim first, then the boundary-free tiles, so co-resident CTAs mostly
  // run the same instantiation (the variants' code does not compete for the instruction
  // cache) and the tail of the grid is made of the fast interior tiles
  int tx, ty;
  {
    const int nix = a.tx_hi - a.tx_lo + 1, niy = a.ty_hi - a.ty_lo + 1;
    const int nin = (nix > 0 && niy > 0) ? nix * niy : 0;
    const int nrim = a.ntx * a.nty - nin;
    const int b = static_cast<int>(blockIdx.x);
    if (b >= nrim) {
      tx = a.tx_lo + (b - nrim) % nix;
      ty = a.ty_lo + (b - nrim) / nix;
    } else {
      const int e = b;
      const int bottom = (nin ? a.ty_lo : a.nty) * a.ntx;
      const int top = nin ? (a.nty - 1 - a.ty_hi) * a.ntx : 0;
      if (e < bottom) {
        tx = e % a.ntx;
        ty = e / a.ntx;
      } else if (e < bottom + top) {
        tx = (e - bottom) % a.ntx;
        ty = a.ty_hi + 1 + (e - bottom) / a.ntx;
      } else {
        const int left = a.tx_lo, side = a.ntx - nix, r3 = e - bottom - top;
        ty = a.ty_lo + r3 / side;
        const int r = r3 % side;
        tx = r < left ? r : a.tx_hi + 1 + (r - left);
      }
    }
  }
  const int64_t i0 = a.sp.ilo + static_cast<int64_t>(tx) * kTX;
  const int64_t j0 = a.sp.jlo + static_cast<int64_t>(ty) * kTY;
  const int64_t i = i0 + lane, j = j0 + row;
  const bool active = i <= a.sp.ihi && j <= a.sp.jhi;
  const int nz = a.nz;
  const int64_t P = a.g.plane, W = a.g.pitch;
  const DynConst& c = a.c;
  const int64_t gi = i + a.sp.i0, gj = j + a.sp.j0, gnx = a.sp.gnx, gny = a.sp.gny;
  // CTA-uniform: every column of the tile is >= 3 cells from every global wall
  const int64_t gi0 = i0 + a.sp.i0, gj0 = j0 + a.sp.j0;
  // CTA-uniform: which wall / partial-tile cases this tile needs (x: its columns, y: its
  // rows); tiles >= 3 cells from the walls and fully inside the span need none
  const bool chk_x = !(gi0 >= 3 && gi0 + kTX - 1 <= gnx - 2 && i0 + kTX - 1 <= a.sp.ihi);
  const bool chk_y = !(gj0 >= 3 && gj0 + kTY - 1 <= gny - 2 && j0 + kTY - 1 <= a.sp.jhi);

  const uint32_t full0 = sm100::smem_u32(full_bar);
  // TMEM: cp in columns [0, ncols/2), dp in [ncols/2, ncols); 256 columns (two CTAs per SM)
  // up to 64 faces, 512 (one CTA per SM) up to 128
  const uint32_t tmem_cols = a.nz - 1 <= 64 ? 256u : 512u;
  const uint32_t dp_col = tmem_cols / 2;
  if (warp == 0) sm100::tmem_alloc(&tmem_base_slot, tmem_cols);
  if (kTmaFeed && warp == 0 && lane == 0) {
    for (int q = 0; q < kWsStages; ++q) sm100::mbar_init(full0 + 8 * q, 1);
    sm100::mbar_fence_init();
  }
  // TMA issue: which boxes this warp's lane 0 loads per level (-1: none). The acoustic
  // warps issue (warp 0 th + u, 1 v + w, 2 p, 3 rho; warp 0 arms the slot barrier), an
  // advection warp waits: the advection role is the one whose per-level instruction
  // stream sets the pace (issuing from warps 0-5 instead: 2.68-2.71 vs 2.65 ms; waiting on
  // an acoustic warp: 2.75-2.79 ms, tools/gpu_r2zf.sh, gpu_r2zg.sh)
  const int f0 = warp == 0 ? 0 : warp == 1 ? 2 : warp == 2 ? 4 : warp == 3 ? 5 : -1;
  const int f1 = warp == 0 ? 1 : warp == 1 ? 3 : -1;
  if (kTmaFeed && lane == 0) {
    if (f0 >= 0) sm100::tma_prefetch_desc(&maps.m[f0]);
    if (f1 >= 0) sm100::tma_prefetch_desc(&maps.m[f1]);
  }
  sm100::tmem_fence_before();
  __syncthreads();
  sm100::tmem_fence_after();
  const uint32_t tmem = tmem_base_slot + (static_cast<uint32_t>(32 * row) << 16);

  // TMA feed: lane 0 of warp f (f < 6) loads field f's box (th, u, v, w, p, rho order);
  // box origins in allocation coordinates (x = kIOff + i', y = kHalo + j', z = k)
  auto box_of = [&](int f, int& off, int& dx, int& dy) {
    off = f == 0 ? kWOffTh : f == 1 ? kWOffU : f == 2 ? kWOffV : f == 3 ? kWOffW
        : f == 4 ? kWOffP : kWOffRho;
    dx = (f == 0 || f == 1 || f == 4) ? -2 : 0;
    dy = f == 0 ? -2 : (f == 2 || f == 4) ? -1 : 0;
  };
  const int x00 = static_cast<int>(kIOff + (i0 - 1)), y00 = static_cast<int>(kHalo + (j0 - 1));
  int off0 = 0, dx0 = 0, dy0 = 0, off1 = 0, dx1 = 0, dy1 = 0;
  box_of(f0 < 0 ? 0 : f0, off0, dx0, dy0);
  box_of(f1 < 0 ? 0 : f1, off1, dx1, dy1);
  const uint32_t dst0 = sm100::smem_u32(ring) + static_cast<uint32_t>(off0 * 8);
  const uint32_t dst1 = sm100::smem_u32(ring) + static_cast<uint32_t>(off1 * 8);
  int tma_k = 0;  // the next level this lane loads

  const double* src[kWsChunksPerThread];
  uint32_t dst[kWsChunksPerThread];
  bool ok[kWsChunksPerThread];
  const uint32_t ring_u32 = sm100::smem_u32(ring);
#pragma unroll
  for (int q = 0; q < kWsChunksPerThread; ++q) {
    const int ch = tid + q * kWsThreads;
    ok[q] = false;
    src[q] = a.in.p;
    dst[q] = 0;
    if (ch >= kFChunks) continue;
    const int e = ch * 2;  // packed index of the chunk's first double in the stage
    const double* base;
    int64_t r, cc;  // 0-based local (j', i') of the chunk start
    int d;          // padded offset of the chunk's field minus its packed offset
    if (e < kFOffU) {
      base = a.in.th; r = (j0 - 3) + e / kFThW; cc = (i0 - 3) + e % kFThW; d = kWOffTh - kFOffTh;
    } else if (e < kFOffV) {
      base = a.in.u; r = (j0 - 1) + (e - kFOffU) / kUW; cc = (i0 - 3) + (e - kFOffU) % kUW;
      d = kWOffU - kFOffU;
    } else if (e < kFOffW) {
      base = a.in.v; r = (j0 - 2) + (e - kFOffV) / kVW; cc = (i0 - 1) + (e - kFOffV) % kVW;
      d = kWOffV - kFOffV;
    } else if (e < kFOffP) {
      base = a.in.w; r = (j0 - 1) + (e - kFOffW) / kSW; cc = (i0 - 1) + (e - kFOffW) % kSW;
      d = kWOffW - kFOffW;
    } else if (e < kFOffRho) {
      base = a.in.p; r = (j0 - 2) + (e - kFOffP) / kPW; cc = (i0 - 3) + (e - kFOffP) % kPW;
      d = kWOffP - kFOffP;
    } else {
      base = a.in.rho; r = (j0 - 1) + (e - kFOffRho) / kSW; cc = (i0 - 1) + (e - kFOffRho) % kSW;
      d = kWOffRho - kFOffRho;
    }
    ok[q] = r >= -kHalo && r <= a.nj - 1 + kHalo && cc >= a.row_lo && cc + 1 <= a.row_hi;
    src[q] = base + r * W + cc;
    dst[q] = ring_u32 + static_cast<uint32_t>(e + d) * 8u;
  }
  // levels are issued in order, once each: sources advance by one plane per call and the
  // ring offset rotates (no per-level multiplies or modulo). 528 chunks per level over
  // 256 threads: two each, and a third for the first 16 threads (warp 0 only, so the
  // other warps carry no third pointer).
  static_assert(kFChunks > 2 * kWsThreads && kFChunks <= 2 * kWsThreads + kTX, "chunk split");
  uint32_t so = 0;
  uint32_t tma_bar = 0;  // TMA feed: byte offset of the slot's barrier
  constexpr uint32_t kStageBytes = kWStageDoubles * 8;
  auto issue = [&](bool copy) {
    if constexpr (kTmaFeed) {
      if (copy && f0 >= 0) {  // (warp-uniform) the ring cursor shuffled from lane 0 is
        // known uniform, so the issue needs no per-lane waterfall loop around UTMALDG
        const uint32_t so_u = __shfl_sync(0xffffffffu, so, 0);
        const uint32_t fb = full0 + __shfl_sync(0xffffffffu, tma_bar, 0);
        const int k_u = __shfl_sync(0xffffffffu, tma_k, 0);
        if (sm100::elect_one()) {  // (not lane == 0: with elect.sync the compiler emits no
          // per-active-lane BRA.U.ANY loop around the UTMALDGs)
        if (warp == 0) sm100::mbar_arrive_expect_tx(fb, kWStageTx);
        sm100::tma_load_3d(dst0 + so_u, &maps.m[f0], fb, x00 + dx0, y00 + dy0, k_u);
        if (f1 >= 0)
          sm100::tma_load_3d(dst1 + so_u, &maps.m[f1], fb, x00 + dx1, y00 + dy1, k_u);
        // RK stages: the base state of the same level into L2 (TMA prefetch boxes), so
        // the per-thread base loads one level ahead hit L2 instead of DRAM (C2 RK3 step
        // 1.41 -> 1.17 ms); boxes th 32x4, u 34x4 (i-2..), v 32x5 (j-1..), w, p
        if constexpr (kRK) {
          if (f0 < 5)
            sm100::tma_prefetch_l2_3d(&maps.base[f0], x00 + (f0 == 1 ? -2 : 0),
                                      y00 + (f0 == 2 ? -1 : 0), k_u);
          if (f1 >= 0 && f1 < 5)
            sm100::tma_prefetch_l2_3d(&maps.base[f1], x00 + (f1 == 1 ? -2 : 0),
                                      y00 + (f1 == 2 ? -1 : 0), k_u);
        }
        }
      }
      ++tma_k;
      const bool wrap = so == (kWsStages - 1) * kStageBytes;
      so = wrap ? 0u : so + kStageBytes;
      tma_bar = wrap ? 0u : tma_bar + 8u;
      return;
    }
    if (copy) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (ok[q]) sm100::cp_async16(dst[q] + so, src[q]);
        src[q] += P;
      }
      if (warp == 0) {
        if (ok[2]) sm100::cp_async16(dst[2] + so, src[2]);
        src[2] += P;
      }
    }
    sm100::cp_async_commit();
    so = so == (kWsStages - 1) * kStageBytes ? 0u : so + kStageBytes;
  };


  const int64_t col = (j - 1) * W + (i - 1);
  // running output pointers (advance one plane per level): acoustic u', v'; advection th'
  double* out_a = (acoustic ? a.out.u : a.out.th) + col;
  double* out_v = a.out.v + col;
  const bool east = gi == gnx, west = gi == 1, north = gj == gny, south = gj == 1;
  const int thc = (row + 2) * kFThW + (lane + 2);
  // kRemote: the neighbours (up to 3: edge, edge, corner) whose halo ring holds this
  // column, and the column's offset in each neighbour's buffers
  int rq[3] = {0, 0, 0}, nrem = 0;
  int64_t roff[3] = {0, 0, 0};
  if constexpr (kRemote) {
    if (active)
      for (int q = 0; q < rem.n; ++q) {
        const bool in_i = rem.dx[q] < 0 ? i <= rem.h : rem.dx[q] > 0 ? i > rem.nx - rem.h : true;
        const bool in_j = rem.dy[q] < 0 ? j <= rem.h : rem.dy[q] > 0 ? j > rem.ny - rem.h : true;
        if (in_i && in_j && nrem < 3) {
          rq[nrem] = q;
          roff[nrem] = rem.g[q].at(i + rem.shift_i[q] - 1, j + rem.shift_j[q] - 1, 0);
          ++nrem;
        }
      }
  }
  // store one output value of level k (0-based) of this column into the neighbours
  auto remote = [&](double* const* base, int k, double v) {
    if constexpr (kRemote) {
#pragma unroll 1
      for (int r = 0; r < nrem; ++r)
        base[rq[r]][roff[r] + static_cast<int64_t>(k) * rem.g[rq[r]].plane] = v;
    }
  };

#pragma unroll 1
  for (int k = 0; k < kWsStages - 1; ++k) issue(k < nz);
  if (kTmaFeed && warp == kWaitWarp)
    for (int l = 0; l < 3 && l < nz; ++l) sm100::mbar_wait(full0 + 8 * l, 0);

  // role state carried along K
  double th_prev = 0.0, w_prev = 0.0;              // both roles
  double rho_prev = 0.0, ps_prev = 0.0, cp_prev = 0.0, dp_prev = 0.0;  // acoustic
  double fz_prev = 0.0;                            // advection
  double phys_cs = 0.0, phys_cm = 0.0, colm_ij = 0.0;  // column physics
  // RK stage: base-state values of this column (one level prefetched in registers)
  struct BaseLevel {
    double th, u, uw, v, vs, p, w;
  };
  auto base_load = [&](int k, auto role_tag) {
    BaseLevel b{};
    if (kRK && k < nz && active) {
      const int64_t o = col + static_cast<int64_t>(k) * P;
      if constexpr (decltype(role_tag)::value) {
        b.u = __ldg(a.base.u + o);
        b.uw = __ldg(a.base.u + o - 1);
        b.v = __ldg(a.base.v + o);
        b.vs = __ldg(a.base.v + o - W);
        b.p = __ldg(a.base.p + o);
        b.w = __ldg(a.base.w + o);
      } else {
        b.th = __ldg(a.base.th + o);
      }
    }
    return b;
  };
  BaseLevel bcur{};
  if (kRK) bcur = acoustic ? base_load(0, std::true_type{}) : base_load(0, std::false_type{});
  double wb_prev = 0.0;  // base w of the previous level (RK: the HE-VI right-hand side)
  if (kPhys && !acoustic && active) {
    colm_ij = a.colm[(j - 1) * W + (i - 1)];
  }
  double pend_beta = 0.0, pend_bb = 1.0, pend_dd = 0.0;  // face awaiting its recursion step
  int s0 = 0;  // ring slot of level k
  const fp64::Recip rth0 = fp64::recip(c.th0);

  // Thomas forward recursion for face f (dialect face kf = f + 1) from the pending
  // coefficients (quotients by m share one reciprocal; `ok` guards the fast path)
  auto thomas_fast = [&](int f, double& cpk, double& dpk, bool& ok, bool not_first) {
    const bool first = !not_first && f == 0;
    const double m = first ? pend_bb : pend_bb + pend_beta * cp_prev;
    const double num = first ? pend_dd : pend_dd + pend_beta * dp_prev;
    const fp64::Recip rm = fp64::recip(m);
    cpk = fp64::quot(-pend_beta, rm, ok);
    dpk = fp64::quot(num, rm, ok);
  };
  auto thomas_div = [&](int f, double& cpk, double& dpk) {  // the dialect's divisions
    if (f == 0) {
      cpk = -pend_beta / pend_bb;
      dpk = pend_dd / pend_bb;
    } else {
      const double m = pend_bb + pend_beta * cp_prev;
      cpk = -pend_beta / m;
      dpk = (pend_dd + pend_beta * dp_prev) / m;
    }
  };
  // cp/dp of face f go to this thread's TMEM lane
  auto thomas_commit = [&](int f, double cpk, double dpk) {
    sm100::tmem_st_f64(tmem + 2 * f, cpk);
    sm100::tmem_st_f64(tmem + dp_col + 2 * f, dpk);
    cp_prev = cpk;
    dp_prev = dpk;
  };

  // kMid: 3 <= k < nz - 5 — no vertical boundary cases (faces kk+1/2 with
  // 2 <= kk <= nz-2, Thomas face k-2 >= 1) and the copy of level k+5 always exists
  // kAc: the role of this warp (acoustic/HE-VI or advection) is a compile-time property of
  // the whole K sweep, so each role's loop carries only its own state across levels
  auto level = [&](int k, auto chk_tag, auto mid_tag, auto role_tag) {
    constexpr bool kCX = decltype(chk_tag)::x, kCY = decltype(chk_tag)::y;
    constexpr bool kIn = !kCX && !kCY;  // every lane active
    constexpr bool kMid = decltype(mid_tag)::value;
    constexpr bool kAc = decltype(role_tag)::value;
    const BaseLevel bnext = base_load(k + 1, role_tag);
    const int kk = k + 1;
    const int s1 = s0 == kWsStages - 1 ? 0 : s0 + 1;
    const int s2 = s1 == kWsStages - 1 ? 0 : s1 + 1;
    const double* S = ring + s0 * kWStageDoubles;
    const double tk = S[kWOffTh + thc];
    const double* Up = S + kWOffU + row * kUW + (lane + 2);
    const double ui = Up[0], uim1 = Up[-1];
    const double* Vp = S + kWOffV + (row + 1) * kVW + lane;
    const double vj = Vp[0], vjm1 = Vp[-kVW];
    const double wk = S[kWOffW + row * kSW + lane];
    if (kAc && (a.roles & 2) != 0) {
      const double* Pp = S + kWOffP + (row + 1) * kPW + (lane + 2);
      const double pk = Pp[0], pe = Pp[1], pw = Pp[-1], pnn = Pp[kPW], psth = Pp[-kPW];
      const double rhok = S[kWOffRho + row * kSW + lane];
      // PGF applied to the base momentum (RK) or the current one (single stage)
      const double unk0 = (kRK ? bcur.u : ui) - c.dt_rdx * (pe - pk);
      const double vnk0 = (kRK ? bcur.v : vj) - c.dt_rdy * (pnn - pk);
      const double uw0 = (kRK ? bcur.uw : uim1) - c.dt_rdx * (pk - pw);
      const double vs0 = (kRK ? bcur.vs : vjm1) - c.dt_rdy * (pk - psth);
      const double unk = (kCX && east) ? 0.0 : unk0;
      const double vnk = (kCY && north) ? 0.0 : vnk0;
      const double uw = (kCX && west) ? 0.0 : uw0;
      const double vs = (kCY && south) ? 0.0 : vs0;
      const double psk = (kRK ? bcur.p : pk) - c.dt_cs2 * (c.rdx * (unk - uw) + c.rdy * (vnk - vs));
      if (kIn || active) {
        *out_a = unk;
        *out_v = vnk;
      }
      remote(rem.u, k, unk);
      remote(rem.v, k, vnk);
      ps_s[k * kThreads + t] = psk;
      if (kPhys && (kMid || k >= 1)) {  // column sums of level k-1, in level order
        const double thp = thv_s[((k - 1) & 1) * kThreads + t];
        phys_cs = phys_cs + rho_prev * thp;
        phys_cm = phys_cm + rho_prev;
      }
      // The Thomas recursion for face f = k-2 (its coefficients were formed in the
      // previous iteration) runs here, independent of this iteration's coefficient
      // formation for face k-1: the two division chains overlap instead of adding up.
      bool ok = true;
      double cpk = 0.0, dpk = 0.0, beta = 0.0, dd = 0.0;
      if (kMid || k >= 2) thomas_fast(k - 2, cpk, dpk, ok, kMid);
      const double w_rhs = kRK ? wb_prev : w_prev;
      const double n_ps = c.dt_rdz * (psk - ps_prev);
      const double n_th = c.dt_grav * (0.5 * (th_prev + tk) - c.th0);
      if (kMid || k >= 1) {
        const double rf = 0.5 * (rho_prev + rhok);
        const fp64::Recip rr = fp64::recip(rf);
        beta = fp64::quot(c.beta_num, rr, ok);
        dd = w_rhs - fp64::quot(n_ps, rr, ok);
        dd = dd + fp64::quot(n_th, rth0, ok);
      }
      if (__builtin_expect(!ok, 0)) {  // a range check failed: the dialect's divisions
        if (k >= 2) thomas_div(k - 2, cpk, dpk);
        if (k >= 1) {
          const double rf = 0.5 * (rho_prev + rhok);
          beta = c.beta_num / rf;
          dd = w_rhs - n_ps / rf;
          dd = dd + n_th / c.th0;
        }
      }
      if (kMid || k >= 2) thomas_commit(k - 2, cpk, dpk);
      if (kMid || k >= 1) {
        pend_beta = beta;
        pend_bb = 1.0 + 2.0 * beta;
        pend_dd = dd;
      }
      rho_prev = rhok;
      ps_prev = psk;
      if (kRK) wb_prev = bcur.w;
    } else if (!kAc && (a.roles & 1) != 0) {
      const double* T0 = S + kWOffTh + thc;
      const double tkp1 =
          (kMid || kk + 1 <= nz) ? ring[s1 * kWStageDoubles + kWOffTh + thc] : 0.0;
      const double tkp2 =
          (kMid || kk + 2 <= nz) ? ring[s2 * kWStageDoubles + kWOffTh + thc] : 0.0;
      const double xm2 = T0[-2], xm1 = T0[-1], xp1 = T0[1], xp2 = T0[2];
      const double ym2 = T0[-2 * kFThW], ym1 = T0[-kFThW], yp1 = T0[kFThW], yp2 = T0[2 * kFThW];
      const double fzk = face_flux_up<!kMid>(kk, nz, wk, th_prev, tk, tkp1, tkp2);
      const double fxe = face_flux_up<kCX>(gi, gnx, ui, xm1, tk, xp1, xp2);
      const double fxw = face_flux_up<kCX>(gi - 1, gnx, uim1, xm2, xm1, tk, xp1);
      const double fyn = face_flux_up<kCY>(gj, gny, vj, ym1, tk, yp1, yp2);
      const double fys = face_flux_up<kCY>(gj - 1, gny, vjm1, ym2, ym1, tk, yp1);
      const double ue = (kCX && east) ? 0.0 : ui;
      const double uwf = (kCX && west) ? 0.0 : uim1;
      const double vnf = (kCY && north) ? 0.0 : vj;
      const double vsf = (kCY && south) ? 0.0 : vjm1;
      const double wt = (!kMid && kk == nz) ? 0.0 : wk;
      const double wb = (!kMid && kk == 1) ? 0.0 : w_prev;
      double flux = c.rdx * (fxe - fxw) + c.rdy * (fyn - fys);
      flux = flux + c.rdz * (fzk - fz_prev);
      double div = c.rdx * (ue - uwf) + c.rdy * (vnf - vsf);
      div = div + c.rdz * (wt - wb);
      double thv = (kRK ? bcur.th : tk) - c.dt * (flux - tk * div);
      if (kPhys) {  // column_physics (dycore.h90), applied to the new theta of this level
        thv = thv - a.dt_rrelax * (thv - colm_ij);
        // (only the first K phase holds level 1: the mid instantiation carries no branch, and
        // tsfc is read where it is used instead of living in a register for the sweep)
        if (!kMid && kk == 1) {  // new u, v at the lowest level (region 5), from the plane
          const double* Pp = S + kWOffP + (row + 1) * kPW + (lane + 2);
          const double un1 = (kCX && east) ? 0.0 : ui - c.dt_rdx * (Pp[1] - Pp[0]);
          const double vn1 = (kCY && north) ? 0.0 : vj - c.dt_rdy * (Pp[kPW] - Pp[0]);
          const double wspd = sqrt(un1 * un1 + vn1 * vn1);
          const double tsfc_ij = active ? a.tsfc[(j - 1) * W + (i - 1)] : 0.0;
          thv = thv + a.dt_ch * wspd * (tsfc_ij - thv) * c.rdz / S[kWOffRho + row * kSW + lane];
        }
        thv_s[(k & 1) * kThreads + t] = thv;
      }
      if (kIn || active) *out_a = thv;
      remote(rem.th, k, thv);
      fz_prev = fzk;
    }
    th_prev = tk;
    w_prev = wk;
    s0 = s1;
    out_a += P;
    if (kAc) out_v += P;
    bcur = bnext;
  };

  // one level: levels <= k+2 have landed (own copies; issued up to k+kWsStages-2), the
  // barrier makes everyone's visible and tells that every warp has finished level k-1,
  // so its slot is refilled with level k+kWsStages-1 (one barrier per level)
  // TMA feed: the waiter warp observes level k+3 at the END of level k (its own work
  // done, so the mbarrier latency overlaps the other warps' arithmetic); the barrier at
  // the top of level k+1 publishes it (mbarrier acquire, then bar.sync)
  uint32_t wslot = 3 % kWsStages, wpar = 0;  // slot / phase parity of the awaited level
  auto wait_level = [&]() {
    sm100::mbar_wait(full0 + 8 * wslot, wpar);
    if (++wslot == kWsStages) {
      wslot = 0;
      wpar ^= 1u;
    }
  };
  auto step = [&](int k, auto in_tag, auto mid_tag, auto role_tag) {
    if constexpr (!kTmaFeed) sm100::cp_async_wait<kWsStages - 4>();
    __syncthreads();
    issue(decltype(mid_tag)::value || k + kWsStages - 1 < nz);
    level(k, in_tag, mid_tag, role_tag);
    if constexpr (kTmaFeed && decltype(role_tag)::value == (kWaitWarp < kTY)) {
      if (warp == kWaitWarp && (decltype(mid_tag)::value || k + 3 < nz)) wait_level();
    }
  };
  // K phases: [0, 3) and [nz-5, nz) with the vertical boundary cases, [3, nz-5) without
  const int mid_lo = nz >= 3 ? 3 : nz, mid_hi = nz - 5 > mid_lo ? nz - 5 : mid_lo;
  auto sweep = [&](auto in_tag, auto role_tag) {
    int k = 0;
#pragma unroll 1
    for (; k < mid_lo; ++k) step(k, in_tag, std::false_type{}, role_tag);
#pragma unroll kMidUnroll
    for (; k < mid_hi; ++k) step(k, in_tag, std::true_type{}, role_tag);
#pragma unroll 1
    for (; k < nz; ++k) step(k, in_tag, std::false_type{}, role_tag);
  };
  // the two roles run separate K loops (same barrier sequence: one bar.sync per level)
  auto run = [&](auto role_tag) {
    if (!chk_x && !chk_y)
      sweep(Chk<false, false>{}, role_tag);
    else if (!chk_y)
      sweep(Chk<true, false>{}, role_tag);
    else if (!chk_x)
      sweep(Chk<false, true>{}, role_tag);
    else
      sweep(Chk<true, true>{}, role_tag);
  };
  if (acoustic)
    run(std::true_type{});
  else
    run(std::false_type{});
  if (acoustic && nz >= 2) {  // drain the last face
    bool ok = true;
    double cpk, dpk;
    thomas_fast(nz - 2, cpk, dpk, ok, false);
    if (!ok) thomas_div(nz - 2, cpk, dpk);
    thomas_commit(nz - 2, cpk, dpk);
  }
  sm100::cp_async_wait<0>();
  if (kPhys) {  // the last level's column-sum terms, then the new column mean
    __syncthreads();
    if (acoustic) {
      const double thp = thv_s[((nz - 1) & 1) * kThreads + t];
      phys_cs = phys_cs + rho_prev * thp;
      phys_cm = phys_cm + rho_prev;
      if (active) a.colm[(j - 1) * W + (i - 1)] = phys_cs / phys_cm;
    }
  }

  if (acoustic) {
    sm100::tmem_wait_st();
    double* wn = a.out.w + col + static_cast<int64_t>(nz - 1) * P;  // running pointers
    double* pn = a.out.p + col + static_cast<int64_t>(nz - 1) * P;
    if (active) *wn = 0.0;
    double wk1 = 0.0;
    const int nf = nz - 1;
    const double* psp = ps_s + (nz - 1) * kThreads + t;  // ps(f+1)
#pragma unroll 1
    for (int cb = (nf - 1) / 4; cb >= 0; --cb) {
      double cpv[4], dpv[4];
      sm100::tmem_ld_4f64(tmem + 8 * cb, cpv);
      sm100::tmem_ld_4f64(tmem + dp_col + 8 * cb, dpv);
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        const int f = 4 * cb + q;
        if (f >= nf) continue;
        wn -= P;
        const double wkk = (f == nf - 1) ? dpv[q] : dpv[q] - cpv[q] * wk1;
        const double pk1 = *psp - c.dt_cs2_rdz * (wk1 - wkk);
        if (active) {
          *wn = wkk;
          *pn = pk1;
        }
        remote(rem.p, f + 1, pk1);
        pn -= P;
        psp -= kThreads;
        wk1 = wkk;
      }
    }
    const double p0 = *psp - c.dt_cs2_rdz * wk1;
    if (active) *pn = p0;
    remote(rem.p, 0, p0);
  }
  sm100::tmem_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem_base_slot, tmem_cols);
}

}  // namespace

#ifndef HFB_ARITH_FMA
// ---- host: TMA tensor maps over hfb-layout device arrays (hfb_tmap.cuh) -------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}
}  // namespace

bool make_box_map(CUtensorMap* m, const double* origin, Grid3 g, int64_t nj, int64_t nz, int bw,
                  int bh) {
  auto fn = encode_fn();
  if (!fn) return false;
  const double* base = origin - (kHalo * g.pitch + kIOff);
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.pitch), static_cast<cuuint64_t>(nj + 2 * kHalo),
                        static_cast<cuuint64_t>(nz)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(g.pitch * 8),
                           static_cast<cuuint64_t>(g.plane * 8)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
#endif

cudaError_t launch_dycore_step_ws(const DynIn& in, const DynOut& out, Grid3 g, int64_t nz,
                                  int64_t nj, const DynConst& c, const Span& sp,
                                  cudaStream_t s, const PhysArgs* phys, const DynIn* base,
                                  const RemoteHalo* remote, int debug_skip) {
  if (sp.ihi < sp.ilo || sp.jhi < sp.jlo) return cudaSuccess;
  if (!dycore_step_ws_fits(nz)) return cudaErrorInvalidValue;
  if (phys && base) return cudaErrorInvalidValue;
  if (remote && base) return cudaErrorInvalidValue;  // RK stages exchange by push
  const size_t smem = std::max<size_t>((static_cast<size_t>(kWsStages) * kWStageDoubles +
                                        static_cast<size_t>(nz) * kThreads +
                                        (phys ? 2 * kThreads : 0)) * sizeof(double) + 128,
                                       80 * 1024);
  const int variant = (phys ? 1 : base ? 2 : 0) + (remote ? 3 : 0);
  StepMaps maps{};
  if (kTmaFeed) {
    const bool ok = make_box_map(&maps.m[0], in.th, g, nj, nz, kFThW, kFThR) &&
                    make_box_map(&maps.m[1], in.u, g, nj, nz, kUW, kUR) &&
                    make_box_map(&maps.m[2], in.v, g, nj, nz, kVW, kVR) &&
                    make_box_map(&maps.m[3], in.w, g, nj, nz, kSW, kSR) &&
                    make_box_map(&maps.m[4], in.p, g, nj, nz, kPW, kPR) &&
                    make_box_map(&maps.m[5], in.rho, g, nj, nz, kSW, kSR);
    if (!ok) return cudaErrorInvalidValue;
    if (base) {
      const bool okb = make_box_map(&maps.base[0], base->th, g, nj, nz, kSW, kSR) &&
                       make_box_map(&maps.base[1], base->u, g, nj, nz, kUW, kUR) &&
                       make_box_map(&maps.base[2], base->v, g, nj, nz, kVW, kVR) &&
                       make_box_map(&maps.base[3], base->w, g, nj, nz, kSW, kSR) &&
                       make_box_map(&maps.base[4], base->p, g, nj, nz, kSW, kSR);
      if (!okb) return cudaErrorInvalidValue;
    }
  }
  void (*kern)(StepMaps, StepTmemArgs, RemoteHalo) = variant == 1   ? k_dyn_step_ws<true, false, false>
                                           : variant == 2 ? k_dyn_step_ws<false, true, false>
                                           : variant == 3 ? k_dyn_step_ws<false, false, true>
                                           : variant == 4 ? k_dyn_step_ws<true, false, true>
                                                          : k_dyn_step_ws<false, false, false>;
  {
    cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
  }
#ifndef HFB_VARIANTS
  debug_skip = 0;  // the product computes both roles
#endif
  StepTmemArgs a{in, out, g, static_cast<int>(nz), 3 & ~debug_skip,
                 phys ? phys->tsfc : nullptr, phys ? phys->colm : nullptr,
                 phys ? phys->dt_rrelax : 0.0, phys ? phys->dt_ch : 0.0,
                 base ? *base : DynIn{}, nj, -kIOff, g.pitch - kIOff - 1, c, sp};
  const int ntx = static_cast<int>((sp.ihi - sp.ilo + 1 + kTX - 1) / kTX);
  const int nty = static_cast<int>((sp.jhi - sp.jlo + 1 + kTY - 1) / kTY);
  // the boundary-free tile rectangle (the kernel's chk_x / chk_y criteria)
  auto interior = [&](int n, int64_t lo, int64_t hi, int64_t off, int64_t gn, int w, int* a0,
                      int* a1) {
    *a0 = 0;
    *a1 = -1;
    for (int t = 0; t < n; ++t) {
      const int64_t l0 = lo + static_cast<int64_t>(t) * w, g0 = l0 + off;
      if (g0 >= 3 && g0 + w - 1 <= gn - 2 && l0 + w - 1 <= hi) {
        if (*a1 < *a0) *a0 = t;
        *a1 = t;
      }
    }
  };
  a.ntx = ntx;
  a.nty = nty;
  interior(ntx, sp.ilo, sp.ihi, sp.i0, sp.gnx, kTX, &a.tx_lo, &a.tx_hi);
  interior(nty, sp.jlo, sp.jhi, sp.j0, sp.gny, kTY, &a.ty_lo, &a.ty_hi);
  if (a.tx_hi < a.tx_lo || a.ty_hi < a.ty_lo) a.tx_lo = a.ty_lo = 0, a.tx_hi = a.ty_hi = -1;
  dim3 block(kTX, 2 * kTY);
  dim3 grid(static_cast<unsigned>(ntx * nty));
  static const RemoteHalo none{};
  kern<<<grid, block, smem, s>>>(maps, a, remote ? *remote : none);
  return cudaGetLastError();
}

}  // namespace hfb

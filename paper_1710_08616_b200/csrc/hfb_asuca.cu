// hfb_asuca.cu — the ASUCA time scheme of apps/dycore/asuca.h90 on sm_100a.
//
// One asuca_step = three RK3 stages; each stage is
//   k_asu_tend            slow tendencies (limited advection of rho, theta, u, v, w) at the
//                         stage state: asuca.h90 regions "theta and rho ..." through
//                         "momentum (advective form ...)", fused into one K-march;
//   nsm x { k_asu_acoustic<A>   RK2 first stage (h = dtau/2): the midpoint pressure pa,
//           k_asu_acoustic<B> } RK2 second stage (dtau) + lateral/upper damping: u, v, w, p;
//   k_asu_stage_end       theta = thb + dtf*fth, rho = rhob + dtf*frho.
// The dialect's copies (the step's base state, the acoustic restart from it, the
// short-step copy-back) are pointer swaps in the runtime (hfb_runtime.cu asuca_step).
//
// Machine organisation follows k_dyn_step_ws (hfb_dycore_tmem.cu): a CTA owns a 32 x 4
// tile of (i,j) columns (warp = row, lane = column; the tendency pass: 31 x 4 plus a ghost
// lane that supplies the shared x faces) and marches K; every K-plane of the
// fields the tile reads (with the halo columns/rows its stencils need) is staged into a
// shared-memory ring by TMA (one 3-D box load per field and level, completion on the
// slot's mbarrier) several levels ahead;
// the acoustic passes keep the Thomas coefficients in TENSOR MEMORY (one lane per
// thread) and ps in shared memory, so HBM traffic is the compulsory bytes: each input
// read once, each output written once.
//
// Arithmetic is the dialect's, operation for operation (-fmad=false, IEEE division),
// so results are bit-identical to the reference interpreter. Boundary cases (walls,
// first/last faces) are evaluated as selects on GLOBAL indices; stencil values outside
// the domain are read from the halo ring / other ring slots and discarded by those
// selects (the dialect clamps those indices; the discarded values never matter).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include <cuda.h>

#include "hfb_fp64.cuh"
#include "hfb_kernels.cuh"
#include "hfb_sm100.cuh"
#include "hfb_tmap.cuh"

namespace hfb {

namespace {

constexpr int kTX = 32, kTY = 4, kThreads = kTX * kTY;
// TMEM per acoustic CTA: cp in columns [0, n/2), dp in [n/2, n); n = 256 (two CTAs per SM)
// up to 64 faces, 512 (one CTA per SM) up to 128

// limited upwind flux (asuca.h90 asu_flux with asu_minmod) as selects: both upwind
// candidates' slope pairs are formed and one is chosen, so there is no divergence on the
// sign of the face velocity. vel*(qp1 + (-0.5)*s) == vel*(qp1 - 0.5*s) bit for bit.
__device__ __forceinline__ double asu_flux(double vel, double qm1, double q0, double qp1,
                                           double qp2, bool lo, bool hi) {
  const double d0 = q0 - qm1, d1 = qp1 - q0, d2 = qp2 - qp1;
  const bool up = vel >= 0.0;
  const double x = up ? d0 : d1, y = up ? d1 : d2;
  const double m = fabs(x) < fabs(y) ? x : y;
  double sl = (x * y <= 0.0) ? 0.0 : m;
  sl = (up ? lo : hi) ? 0.0 : sl;
  const double base = up ? q0 : qp1;
  const double h = up ? 0.5 : -0.5;
  return vel * (base + h * sl);
}

// ============================================================================
// slow tendencies
// ============================================================================
// 38 x 8 plane tile: the 2-cell ring around the 32 lanes plus one column, because a TMA
// box must start 16-B aligned (an even x) and the 31-column tiles (below) alternate parity
constexpr int kTW = kTX + 6, kTR = kTY + 4;
constexpr int kTPlane = kTW * kTR;            // 304
constexpr int kTStage = 5 * kTPlane;          // rho, th, u, v, w
constexpr int kTStages = 6;                   // levels k-1..k+2 in use, k+3 in flight
enum { kFRho = 0, kFTh = 1, kFU = 2, kFV = 3, kFW = 4 };

struct TendArgs {
  AsuState s;
  AsuTend f;
  Grid3 g;
  int nz;
  int64_t nj, row_lo, row_hi;
  double rdx, rdy, rdz;
  Span sp;
};

// The ring is fed by TMA: five 38 x 8 box loads per level (rho, th, u, v, w with their
// 2-cell ring), issued by lane 0 of warps 0-3 (warp 0 also the fifth), completion on the
// slot's mbarrier; warp kTendWaitWarp observes level k+3 at the end of its level k and
// the per-level CTA barrier publishes it.
struct TendMaps {
  CUtensorMap m[5];
};
constexpr int kTendWaitWarp = 3;
// x faces are shared between neighbouring lanes: every lane evaluates the EAST face (or
// x-centre / x-edge) of its point and takes the west one from lane - 1 by a shuffle, so
// each horizontal x flux is evaluated once instead of twice. Lane 0 is therefore a ghost
// column (the point west of the tile: it supplies lane 1's west faces and stores nothing)
// and a tile owns 31 columns.
constexpr int kTXo = kTX - 1;
__device__ __forceinline__ double from_west(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }

__global__ void __launch_bounds__(kThreads, 3)
    k_asu_tend(const __grid_constant__ TendMaps maps, TendArgs a) {
  // (maps first: 64-B aligned parameters; the dynamic segment declared 16-B aligned so
  // the round-up to 128 B is not folded away)
  extern __shared__ __align__(16) double smem_raw[];
  __shared__ __align__(16) uint64_t sbar[8];  // slot barriers
  const uint32_t raw_u32 = sm100::smem_u32(smem_raw);
  double* const smem = smem_raw + ((((raw_u32 + 127u) & ~127u) - raw_u32) >> 3);
  const int lane = threadIdx.x, row = sm100::warp_uniform(threadIdx.y), t = row * kTX + lane;
  const int64_t i0 = a.sp.ilo + static_cast<int64_t>(blockIdx.x) * kTXo;  // lane 1's column
  const int64_t j0 = a.sp.jlo + static_cast<int64_t>(blockIdx.y) * kTY;
  const int64_t i = i0 - 1 + lane, j = j0 + row;
  const bool active = lane > 0 && i <= a.sp.ihi && j <= a.sp.jhi;
  const int nz = a.nz;
  const int64_t P = a.g.plane, W = a.g.pitch;
  const int64_t gi = i + a.sp.i0, gj = j + a.sp.j0, gnx = a.sp.gnx, gny = a.sp.gny;
  const double rdx = a.rdx, rdy = a.rdy, rdz = a.rdz;

  static_assert(kTStages <= 8, "slot barriers");
  const uint32_t full0 = sm100::smem_u32(sbar);
  if (t == 0) {
    for (int q = 0; q < kTStages; ++q) sm100::mbar_init(full0 + 8 * q, 1);
    sm100::mbar_fence_init();
  }
  if (lane == 0) {
    sm100::tma_prefetch_desc(&maps.m[row]);
    if (row == 0) sm100::tma_prefetch_desc(&maps.m[4]);
  }
  __syncthreads();
  constexpr uint32_t kStageBytes = kTStage * 8;
  const uint32_t ring_u32 = sm100::smem_u32(smem);
  // box origin in allocation coordinates (x = kIOff + i', y = kHalo + j'), 2-cell ring
  // box origin: 2 columns left of lane 0 (local i0 - 2, 0-based), rounded down to even
  const int xo_l = static_cast<int>(kIOff + (i0 - 2)) - 2, xpar = xo_l & 1;
  const int xo = xo_l - xpar, yo = static_cast<int>(kHalo + (j0 - 1)) - 2;
  auto issue = [&](int k) {  // level k into slot k % kTStages (lane 0 of every warp)
    if (k >= nz || !sm100::elect_one()) return;  // (k warp-uniform: the warp is converged)
    const uint32_t slot = static_cast<uint32_t>(k % kTStages);
    const uint32_t fb = full0 + 8 * slot;
    const uint32_t so = ring_u32 + slot * kStageBytes;
    if (row == 0) sm100::mbar_arrive_expect_tx(fb, kStageBytes);
    sm100::tma_load_3d(so + row * kTPlane * 8, &maps.m[row], fb, xo, yo, k);
    if (row == 0) sm100::tma_load_3d(so + 4 * kTPlane * 8, &maps.m[4], fb, xo, yo, k);
  };
  auto wait_level = [&](int l) {
    sm100::mbar_wait(full0 + 8 * static_cast<uint32_t>(l % kTStages),
                     static_cast<uint32_t>((l / kTStages) & 1));
  };
  // value of field f at level k (0-based; any k, ring slot), offset (di, dj)
  const int cen = (row + 2) * kTW + (lane + 2 + xpar);
  auto V = [&](int f, int k, int di, int dj) -> double {
    const int slot = ((k % kTStages) + kTStages) % kTStages;
    return smem[slot * kTStage + f * kTPlane + cen + dj * kTW + di];
  };

  const int64_t col = (j - 1) * W + (i - 1);

  for (int k = 0; k < kTStages - 2; ++k) issue(k);
  if (row == kTendWaitWarp)
    for (int l = 0; l < 3 && l < nz; ++l) wait_level(l);

  // kLat: the tile touches (or is within 2 cells of) a lateral wall and needs the wall /
  // first-last-face cases; tiles >= 3 cells from every wall run without them
  auto sweep = [&](auto lat_tag) {
  constexpr bool kLat = decltype(lat_tag)::value;
  const bool east = kLat && gi == gnx, west = kLat && gi == 1;
  const bool north = kLat && gj == gny, south = kLat && gj == 1;
  // carried along K (values at the bottom face / level centre of the current level)
  double fzt_b = 0.0, fzr_b = 0.0;  // theta/rho flux through z-face kk-1/2
  double gzu_b = 0.0, czu_b = 0.0;  // u: z-edge flux / velocity at kk-1/2
  double gzv_b = 0.0, czv_b = 0.0;  // v
  double gzw_b = 0.0, czw_b = 0.0;  // w: flux / velocity through level centre kk
  // kV: the level needs the vertical boundary cases (ground, lid, first/last faces);
  // mid-column levels 3 <= kk <= nz-3 run without them
  auto level = [&](int k, auto v_tag) {
  constexpr bool kV = decltype(v_tag)::value;
    __syncthreads();  // levels <= k+2 landed (observed by the waiter); slot of level k-2 free
    issue(k + kTStages - 2);
    const int kk = k + 1;

    // ---- theta and rho -------------------------------------------------------------
    const double ui = V(kFU, k, 0, 0), uim1 = V(kFU, k, -1, 0);
    const double vj = V(kFV, k, 0, 0), vjm1 = V(kFV, k, 0, -1);
    const double wk = V(kFW, k, 0, 0), wkm1 = V(kFW, k - 1, 0, 0);
    double fth, frho;
    {
      // x faces: east (face i) and west (face i-1)
      auto xface = [&](int fld, int64_t f, int off, double vel) {  // face f = gi + off
        return (kLat && (f == 0 || f == gnx)) ? 0.0
                                    : asu_flux(vel, V(fld, k, off - 1, 0), V(fld, k, off, 0),
                                               V(fld, k, off + 1, 0), V(fld, k, off + 2, 0),
                                               kLat && f == 1, kLat && f + 1 == gnx);
      };
      auto yface = [&](int fld, int64_t f, int off, double vel) {
        return (kLat && (f == 0 || f == gny)) ? 0.0
                                    : asu_flux(vel, V(fld, k, 0, off - 1), V(fld, k, 0, off),
                                               V(fld, k, 0, off + 1), V(fld, k, 0, off + 2),
                                               kLat && f == 1, kLat && f + 1 == gny);
      };
      auto zface = [&](int fld) {  // top face kk+1/2
        return (kV && kk == nz) ? 0.0
                          : asu_flux(wk, V(fld, k - 1, 0, 0), V(fld, k, 0, 0), V(fld, k + 1, 0, 0),
                                     V(fld, k + 2, 0, 0), kV && kk == 1, kV && kk + 1 == nz);
      };
      const double ue = east ? 0.0 : ui, uw = west ? 0.0 : uim1;
      const double vnf = north ? 0.0 : vj, vs = south ? 0.0 : vjm1;
      const double wt = (kV && kk == nz) ? 0.0 : wk, wb = (kV && kk == 1) ? 0.0 : wkm1;
      double div = rdx * (ue - uw) + rdy * (vnf - vs);
      div = div + rdz * (wt - wb);
      const double fzt = zface(kFTh), fzr = zface(kFRho);
      const double fxt = xface(kFTh, gi, 0, ui), fxr = xface(kFRho, gi, 0, ui);
      const double fxt_w = from_west(fxt), fxr_w = from_west(fxr);  // faces gi - 1
      double flux = rdx * (fxt - fxt_w) + rdy * (yface(kFTh, gj, 0, vj) - yface(kFTh, gj - 1, -1, vjm1));
      flux = flux + rdz * (fzt - fzt_b);
      fth = V(kFTh, k, 0, 0) * div - flux;
      flux = rdx * (fxr - fxr_w) + rdy * (yface(kFRho, gj, 0, vj) - yface(kFRho, gj - 1, -1, vjm1));
      flux = flux + rdz * (fzr - fzr_b);
      frho = 0.0 - flux;
      fzt_b = fzt;
      fzr_b = fzr;
    }

    // ---- u (x-face point i) --------------------------------------------------------
    double fu = 0.0;
    {
      // centre c = gi + off between u-points c-1 and c (walls 0 and gnx are zero)
      auto xcen = [&](int off, double& cv) {
        const int64_t c = gi + off;
        const double qb = (kLat && c == 1) ? 0.0 : V(kFU, k, off - 1, 0);
        const double qc = (kLat && c == gnx) ? 0.0 : V(kFU, k, off, 0);
        const double qa = (kLat && c <= 2) ? 0.0 : V(kFU, k, off - 2, 0);
        const double qd = (kLat && c + 1 >= gnx) ? 0.0 : V(kFU, k, off + 1, 0);
        cv = 0.5 * (qb + qc);
        return asu_flux(cv, qa, qb, qc, qd, kLat && c == 1, kLat && c == gnx);
      };
      // y edge f = gj + off (between u(j') and u(j'+1)), velocity mean of v(i), v(i+1)
      auto yedge = [&](int off, double& cv) {
        const int64_t f = gj + off;
        if (kLat && (f == 0 || f == gny || east)) {
          cv = 0.0;
          return 0.0;
        }
        cv = 0.5 * (V(kFV, k, 0, off) + V(kFV, k, 1, off));
        return asu_flux(cv, V(kFU, k, 0, off - 1), V(kFU, k, 0, off), V(kFU, k, 0, off + 1),
                        V(kFU, k, 0, off + 2), kLat && f == 1, kLat && f + 1 == gny);
      };
      double cxe, cxw, cyn, cys, czt;
      const double gxe = xcen(1, cxe);
      const double gxw = from_west(gxe);  // centre gi
      cxw = from_west(cxe);
      const double gyn = yedge(0, cyn), gys = yedge(-1, cys);
      double gzt;
      if ((kV && kk == nz) || east) {
        czt = 0.0;
        gzt = 0.0;
      } else {
        czt = 0.5 * (wk + V(kFW, k, 1, 0));
        gzt = asu_flux(czt, V(kFU, k - 1, 0, 0), ui, V(kFU, k + 1, 0, 0), V(kFU, k + 2, 0, 0),
                       kV && kk == 1, kV && kk + 1 == nz);
      }
      if (!east) {
        double div = rdx * (cxe - cxw) + rdy * (cyn - cys);
        div = div + rdz * (czt - czu_b);
        double flux = rdx * (gxe - gxw) + rdy * (gyn - gys);
        flux = flux + rdz * (gzt - gzu_b);
        fu = ui * div - flux;
      }
      gzu_b = gzt;
      czu_b = czt;
    }

    // ---- v (y-face point j) --------------------------------------------------------
    double fv = 0.0;
    {
      auto ycen = [&](int off, double& cv) {
        const int64_t c = gj + off;
        const double qb = (kLat && c == 1) ? 0.0 : V(kFV, k, 0, off - 1);
        const double qc = (kLat && c == gny) ? 0.0 : V(kFV, k, 0, off);
        const double qa = (kLat && c <= 2) ? 0.0 : V(kFV, k, 0, off - 2);
        const double qd = (kLat && c + 1 >= gny) ? 0.0 : V(kFV, k, 0, off + 1);
        cv = 0.5 * (qb + qc);
        return asu_flux(cv, qa, qb, qc, qd, kLat && c == 1, kLat && c == gny);
      };
      auto xedge = [&](int off, double& cv) {
        const int64_t f = gi + off;
        if (kLat && (f == 0 || f == gnx || north)) {
          cv = 0.0;
          return 0.0;
        }
        cv = 0.5 * (V(kFU, k, off, 0) + V(kFU, k, off, 1));
        return asu_flux(cv, V(kFV, k, off - 1, 0), V(kFV, k, off, 0), V(kFV, k, off + 1, 0),
                        V(kFV, k, off + 2, 0), kLat && f == 1, kLat && f + 1 == gnx);
      };
      double cye, cyw, cxe, cxw, czt;
      const double gxe = xedge(0, cxe);
      const double gxw = from_west(gxe);  // edge gi - 1
      cxw = from_west(cxe);
      const double gyn = ycen(1, cye), gys = ycen(0, cyw);
      double gzt;
      if ((kV && kk == nz) || north) {
        czt = 0.0;
        gzt = 0.0;
      } else {
        czt = 0.5 * (wk + V(kFW, k, 0, 1));
        gzt = asu_flux(czt, V(kFV, k - 1, 0, 0), vj, V(kFV, k + 1, 0, 0), V(kFV, k + 2, 0, 0),
                       kV && kk == 1, kV && kk + 1 == nz);
      }
      if (!north) {
        double div = rdx * (cxe - cxw) + rdy * (cye - cyw);
        div = div + rdz * (czt - czv_b);
        double flux = rdx * (gxe - gxw) + rdy * (gyn - gys);
        flux = flux + rdz * (gzt - gzv_b);
        fv = vj * div - flux;
      }
      gzv_b = gzt;
      czv_b = czt;
    }

    // ---- w (z-face point kk) -------------------------------------------------------
    double fw = 0.0;
    {
      // level centre c between w-points c-1 and c (0 = ground and nz = lid are zero)
      auto zcen = [&](int c, int kc, double& cv) {  // kc: 0-based level of w-point c
        const double qb = (kV && c == 1) ? 0.0 : V(kFW, kc - 1, 0, 0);
        const double qc = (kV && c == nz) ? 0.0 : V(kFW, kc, 0, 0);
        const double qa = (kV && c <= 2) ? 0.0 : V(kFW, kc - 2, 0, 0);
        const double qd = (kV && c + 1 >= nz) ? 0.0 : V(kFW, kc + 1, 0, 0);
        cv = 0.5 * (qb + qc);
        return asu_flux(cv, qa, qb, qc, qd, kV && c == 1, kV && c == nz);
      };
      if (kV && kk == 1) gzw_b = zcen(1, 0, czw_b);  // the ground-side centre of the column
      double czt;
      const double gzt = (kV && kk == nz) ? 0.0 : zcen(kk + 1, k + 1, czt);
      if (kV && kk == nz) czt = 0.0;
      if (!(kV && kk == nz)) {
        auto xedge = [&](int off, double& cv) {
          const int64_t f = gi + off;
          if (kLat && (f == 0 || f == gnx)) {
            cv = 0.0;
            return 0.0;
          }
          cv = 0.5 * (V(kFU, k, off, 0) + V(kFU, k + 1, off, 0));
          return asu_flux(cv, V(kFW, k, off - 1, 0), V(kFW, k, off, 0), V(kFW, k, off + 1, 0),
                          V(kFW, k, off + 2, 0), kLat && f == 1, kLat && f + 1 == gnx);
        };
        auto yedge = [&](int off, double& cv) {
          const int64_t f = gj + off;
          if (kLat && (f == 0 || f == gny)) {
            cv = 0.0;
            return 0.0;
          }
          cv = 0.5 * (V(kFV, k, 0, off) + V(kFV, k + 1, 0, off));
          return asu_flux(cv, V(kFW, k, 0, off - 1), V(kFW, k, 0, off), V(kFW, k, 0, off + 1),
                          V(kFW, k, 0, off + 2), kLat && f == 1, kLat && f + 1 == gny);
        };
        double cxe, cxw, cyn, cys;
        const double gxe = xedge(0, cxe);
        const double gxw = from_west(gxe);  // edge gi - 1
        cxw = from_west(cxe);
        const double gyn = yedge(0, cyn), gys = yedge(-1, cys);
        double div = rdx * (cxe - cxw) + rdy * (cyn - cys);
        div = div + rdz * (czt - czw_b);
        double flux = rdx * (gxe - gxw) + rdy * (gyn - gys);
        flux = flux + rdz * (gzt - gzw_b);
        fw = wk * div - flux;
      }
      gzw_b = gzt;
      czw_b = czt;
    }

    if (active) {
      const int64_t o = col + static_cast<int64_t>(k) * P;
      a.f.fth[o] = fth;
      a.f.frho[o] = frho;
      a.f.fu[o] = fu;
      a.f.fv[o] = fv;
      a.f.fw[o] = fw;
    }
    if (row == kTendWaitWarp && k + 3 < nz) wait_level(k + 3);
    };
  const int mid_lo = nz > 2 ? 2 : nz, mid_hi = nz - 3 > mid_lo ? nz - 3 : mid_lo;
  int k = 0;
#pragma unroll 1
  for (; k < mid_lo; ++k) level(k, std::true_type{});
#pragma unroll 1
  for (; k < mid_hi; ++k) level(k, std::false_type{});
#pragma unroll 1
  for (; k < nz; ++k) level(k, std::true_type{});
  };
  const int64_t gi0 = i0 - 1 + a.sp.i0, gj0 = j0 + a.sp.j0;  // lane 0 (the ghost) included
  const bool interior = gi0 >= 3 && gi0 + kTX - 1 <= gnx - 3 && i0 - 1 + kTX - 1 <= a.sp.ihi &&
                        gj0 >= 3 && gj0 + kTY - 1 <= gny - 3 && j0 + kTY - 1 <= a.sp.jhi;
  if (interior)
    sweep(std::false_type{});
  else
    sweep(std::true_type{});
}

// ============================================================================
// acoustic RK2 passes
// ============================================================================
// pass A (kB = false) planes: p (i-1..i+1, j-1..j+1), u, fu (i-1), v, fv (j-1), w, rho,
// th, fw. Pass B (kB = true): pa in place of p's neighbourhood, p at the column only.
constexpr int kAW = kTX + 4;  // 36 (x-halo planes, even start 2 columns left)
constexpr int kAStages = 4;   // level k in use, k+1..k+3 in flight

struct AcoArgs {
  AsuState s;        // current u, v, w, p; stage rho, th
  const double *fu, *fv, *fw;
  const double* pa;  // pass B: the midpoint pressure
  double* pa_out;    // pass A
  double *un, *vn, *wn, *pn;  // pass B
  Grid3 g;
  int nz;
  int64_t nj, row_lo, row_hi;
  AsuAcoConst c;
  Span sp;
};

// Warp-specialised: 8 warps per CTA over the same 32 x 4 column tile. Warps 4-7 (the
// "horizontal" role) compute, per level k, the pressure gradient, the divergence and ps
// (pass B: also the damped u', v') and leave ps in shared memory; warps 0-3 (the
// "Thomas" role, owners of the TMEM lanes) form the HE-VI coefficients of face k-2 one
// level behind (its upper ps was published by this level's barrier; rho, th, w, fw come
// from the ring at their own level and stay in registers for two levels) beside the
// forward recursion of face k-3, then run the back substitution and the pressure update.
// The barrier that publishes every staged plane also publishes ps, so the pipeline needs
// no extra synchronisation. Two CTAs per SM (TMEM: 256 columns each) give 16 resident
// warps instead of 8; the roles carry about the same instruction count per level.
constexpr int kAcoThreads = 2 * kThreads;
// The plane ring is fed by TMA: one 3-D box load per field and level (10 in pass B, 9 in
// pass A), issued by lane 0 of the horizontal warps 4-7 in pass A, of the Thomas warps 0-3 in pass B, completion on
// the slot's mbarrier; one horizontal warp (the lighter role) observes level k+1's
// barrier at the end of its level k, and the per-level CTA barrier publishes it. Plane
// tiles start 128-B aligned inside a slot.
__host__ __device__ constexpr int pad16(int n) { return (n + 15) / 16 * 16; }
constexpr int kAoP = 0;                                   // p or pa: 36 x 6
constexpr int kAoU = kAoP + pad16(kAW * (kTY + 2));       // u: 36 x 4
constexpr int kAoFU = kAoU + pad16(kAW * kTY);            // fu: 36 x 4
constexpr int kAoV = kAoFU + pad16(kAW * kTY);            // v: 32 x 5
constexpr int kAoFV = kAoV + pad16(kTX * (kTY + 1));      // fv: 32 x 5
constexpr int kAoW = kAoFV + pad16(kTX * (kTY + 1));      // w, rho, th, fw: 32 x 4 each
constexpr int kAoRho = kAoW + kTX * kTY;
constexpr int kAoTh = kAoRho + kTX * kTY;
constexpr int kAoFW = kAoTh + kTX * kTY;
constexpr int kAoPc = kAoFW + kTX * kTY;                  // pass B: p at the column
constexpr int kAcoWaitWarp = 4;
// box of field f: smem offset, origin offset (dx, dy) from the tile, extent (bw, bh)
struct AcoBox {
  int off, dx, dy, bw, bh;
};
constexpr AcoBox kAcoBox[10] = {{kAoP, -2, -1, kAW, kTY + 2},  {kAoU, -2, 0, kAW, kTY},
                                {kAoFU, -2, 0, kAW, kTY},      {kAoV, 0, -1, kTX, kTY + 1},
                                {kAoFV, 0, -1, kTX, kTY + 1},  {kAoW, 0, 0, kTX, kTY},
                                {kAoRho, 0, 0, kTX, kTY},      {kAoTh, 0, 0, kTX, kTY},
                                {kAoFW, 0, 0, kTX, kTY},       {kAoPc, 0, 0, kTX, kTY}};
// (device code reads the table through its __constant__ copy)
__constant__ AcoBox kAcoBoxDev[10] = {{kAoP, -2, -1, kAW, kTY + 2},  {kAoU, -2, 0, kAW, kTY},
                                      {kAoFU, -2, 0, kAW, kTY},      {kAoV, 0, -1, kTX, kTY + 1},
                                      {kAoFV, 0, -1, kTX, kTY + 1},  {kAoW, 0, 0, kTX, kTY},
                                      {kAoRho, 0, 0, kTX, kTY},      {kAoTh, 0, 0, kTX, kTY},
                                      {kAoFW, 0, 0, kTX, kTY},       {kAoPc, 0, 0, kTX, kTY}};
__host__ __device__ constexpr uint32_t aco_tx(int nb) {
  uint32_t b = 0;
  const int words[10] = {kAW * (kTY + 2), kAW * kTY, kAW * kTY, kTX * (kTY + 1),
                        kTX * (kTY + 1), kTX * kTY, kTX * kTY, kTX * kTY, kTX * kTY, kTX * kTY};
  for (int f = 0; f < nb; ++f) b += words[f] * 8;
  return b;
}
struct AcoMaps {
  CUtensorMap m[10];
};

template <bool kB>
__global__ void __launch_bounds__(kAcoThreads, 2)
    k_asu_acoustic(const __grid_constant__ AcoMaps maps, AcoArgs a) {
  // (the tensor maps come first: a CUtensorMap must sit 64-B aligned in parameter space;
  // the dynamic segment is declared 16-B aligned so the round-up below is not folded)
  extern __shared__ __align__(16) double smem_raw[];
  __shared__ __align__(16) uint64_t sbar[8];  // slot barriers, TMEM address (64 B)
  uint32_t& tmem_base_slot = *reinterpret_cast<uint32_t*>(&sbar[7]);
  const uint32_t raw_u32 = sm100::smem_u32(smem_raw);
  double* const ring = smem_raw + ((((raw_u32 + 127u) & ~127u) - raw_u32) >> 3);
  constexpr int oP = kAoP, oU = kAoU, oFU = kAoFU, oV = kAoV, oFV = kAoFV, oW = kAoW,
                oRho = kAoRho, oTh = kAoTh, oFW = kAoFW, oPc = kAoPc;
  constexpr int kNB = kB ? 10 : 9;  // boxes per level
  constexpr int kStage = kB ? oPc + kTX * kTY : oPc;
  constexpr uint32_t kTx = aco_tx(kNB);
  const int nz = a.nz;
  double* ps_s = ring + kAStages * kStage;  // nz x 128

  const int lane = threadIdx.x, warp = sm100::warp_uniform(threadIdx.y);  // blockDim = (32, 8)
  const bool thomas = warp < kTY;
  const int row = thomas ? warp : warp - kTY;
  const int t = row * kTX + lane;     // 0..127 (column within the tile)
  const int64_t i0 = a.sp.ilo + static_cast<int64_t>(blockIdx.x) * kTX;
  const int64_t j0 = a.sp.jlo + static_cast<int64_t>(blockIdx.y) * kTY;
  const int64_t i = i0 + lane, j = j0 + row;
  const bool active = i <= a.sp.ihi && j <= a.sp.jhi;
  const int64_t P = a.g.plane, W = a.g.pitch;
  const int64_t gi = i + a.sp.i0, gj = j + a.sp.j0;
  const AsuAcoConst& c = a.c;

  const uint32_t full0 = sm100::smem_u32(sbar);
  const uint32_t tmem_cols = a.nz - 1 <= 64 ? 256u : 512u;
  const uint32_t dp_col = tmem_cols / 2;
  if (warp == 0) sm100::tmem_alloc(&tmem_base_slot, tmem_cols);
  if (warp == 0 && lane == 0) {
    for (int q = 0; q < kAStages; ++q) sm100::mbar_init(full0 + 8 * q, 1);
    sm100::mbar_fence_init();
  }
  if (lane == 0) {
    sm100::tma_prefetch_desc(&maps.m[warp]);
    if (warp + 8 < kNB) sm100::tma_prefetch_desc(&maps.m[warp + 8]);
  }
  sm100::tmem_fence_before();
  __syncthreads();
  sm100::tmem_fence_after();
  const uint32_t tmem = tmem_base_slot + (static_cast<uint32_t>(32 * row) << 16);

  // Who issues the boxes (lane 0 of each issuing warp; warp w of the issuing role loads
  // fields w, w + 4 and w + 8 < kNB). Pass A: the horizontal warps (the lighter role there:
  // the Thomas warps' K loop carries no issue code): 2.39 -> 2.23 ms at C4. Pass B, whose
  // horizontal warps also store the damped u', v': the Thomas warps (with the warp-uniform
  // index: 2.60 vs 2.63 ms every warp, 2.65 the horizontal ones; tools/gpu_r2zt.sh,
  // gpu_r2zu.sh, gpu_r2zz.sh). Allocation coordinates x = kIOff + i', y = kHalo + j'.
  // issuing role: 0 every warp, 1 the horizontal warps, 2 the Thomas warps
  constexpr int kIssue = kB ? 2 : 1;
  const uint32_t ring_u32 = sm100::smem_u32(ring);
  const int xo = static_cast<int>(kIOff + (i0 - 1)), yo = static_cast<int>(kHalo + (j0 - 1));
  const int f0 = kIssue == 0 ? warp : kIssue == 1 ? (thomas ? 0 : warp - kTY) : (thomas ? warp : 0);
  const int fstep = kIssue == 0 ? 8 : 4;
  const int nbox = (f0 + 2 * fstep < kNB) ? 3 : (f0 + fstep < kNB) ? 2 : 1;
  const AcoBox b0 = kAcoBoxDev[f0];
  const AcoBox b1 = kAcoBoxDev[nbox > 1 ? f0 + fstep : 0];
  const AcoBox b2 = kAcoBoxDev[nbox > 2 ? f0 + 2 * fstep : 0];
  const bool issuer = kIssue == 0 || (kIssue == 1) != thomas;
  constexpr uint32_t kStageBytes = kStage * 8;
  auto issue = [&](int k) {  // level k into slot k % kAStages
    if (!issuer || k >= nz || !sm100::elect_one()) return;  // (issuer, k warp-uniform)
    const uint32_t slot = static_cast<uint32_t>(k % kAStages);
    const uint32_t fb = full0 + 8 * slot;
    const uint32_t so = ring_u32 + slot * kStageBytes;
    if (f0 == 0) sm100::mbar_arrive_expect_tx(fb, kTx);
    sm100::tma_load_3d(so + b0.off * 8, &maps.m[f0], fb, xo + b0.dx, yo + b0.dy, k);
    if (nbox > 1)
      sm100::tma_load_3d(so + b1.off * 8, &maps.m[f0 + fstep], fb, xo + b1.dx, yo + b1.dy, k);
    if (nbox > 2)
      sm100::tma_load_3d(so + b2.off * 8, &maps.m[f0 + 2 * fstep], fb, xo + b2.dx, yo + b2.dy,
                         k);
  };
  // the waiter (a horizontal warp) observes level l's slot barrier
  auto wait_level = [&](int l) {
    sm100::mbar_wait(full0 + 8 * static_cast<uint32_t>(l % kAStages),
                     static_cast<uint32_t>((l / kAStages) & 1));
  };

  const bool east = gi == a.sp.gnx, west = gi == 1, north = gj == a.sp.gny, south = gj == 1;
  const int64_t col = (j - 1) * W + (i - 1);
  // damping (pass B): lateral ramp of this column; the upper ramp per level
  double axy = 0.0;
  if (kB) {
    const int64_t nb = c.nbnd;
    auto ramp = [&](int64_t q, int64_t n) {  // max(0, max(nbnd + 1 - q, q - n + nbnd))
      const int64_t l = nb + 1 - q, r = q - n + nb;
      const int64_t m = r > l ? r : l;
      return static_cast<double>(m > 0 ? m : 0);
    };
    const double ax = ramp(gi, a.sp.gnx) * c.rnbnd;
    const double ay = ramp(gj, a.sp.gny) * c.rnbnd;
    axy = ay > ax ? ay : ax;  // interp.cpp max: the first unless a later one is greater
  }
  auto tau_at = [&](int kk) {  // dtau * rdmp * max(max(ax, ay), az) at 1-based level kk
    const double az = static_cast<double>(kk - c.kdmp > 0 ? kk - c.kdmp : 0) * c.rnzd;
    return c.dtau_rdmp * (az > axy ? az : axy);
  };
  for (int k = 0; k < kAStages - 1; ++k) issue(k);
  if (warp == kAcoWaitWarp) wait_level(0);

  // Thomas role state: rho/th/w/fw of the last two levels (read from the ring at their
  // own level), the coefficients of the face awaiting its recursion step, cp/dp of the
  // face below
  double rho_1 = 0.0, th_1 = 0.0, w_1 = 0.0, fw_1 = 0.0;  // level k-1
  double rho_2 = 0.0, th_2 = 0.0, w_2 = 0.0, fw_2 = 0.0;  // level k-2
  double pend_beta = 0.0, pend_dd = 0.0, cp_p = 0.0, dp_p = 0.0;
  const fp64::Recip rth0 = fp64::recip(c.th0);
  const double* ps_t = ps_s + t;
  // coefficient formation of face f (levels f, f+1: rho/th/w/fw from registers, ps from
  // shared memory); quotients by rf share one reciprocal (hfb_fp64.cuh), else the
  // dialect's divisions
  auto formation = [&](int f, double rho_lo, double rho_hi, double th_lo, double th_hi,
                       double w_lo, double fw_lo, double& beta, double& dd, bool& ok) {
    const double n_ps = c.h_rdz * (ps_t[(f + 1) * kThreads] - ps_t[f * kThreads]);
    const double n_th = c.h_grav * (0.5 * (th_lo + th_hi) - c.th0);
    const double rf = 0.5 * (rho_lo + rho_hi);
    const fp64::Recip rr = fp64::recip(rf);
    beta = fp64::quot(c.beta_num, rr, ok);
    dd = w_lo - fp64::quot(n_ps, rr, ok);
    dd = dd + fp64::quot(n_th, rth0, ok);
    dd = dd + c.h * fw_lo;
    if (__builtin_expect(!ok, 0)) {
      beta = c.beta_num / rf;
      dd = w_lo - n_ps / rf;
      dd = dd + n_th / c.th0;
      dd = dd + c.h * fw_lo;
    }
  };
  // forward recursion of face f from its coefficients; quotients by m share one
  // reciprocal
  auto recursion = [&](int f, double beta, double dd) {
    const double bb = 1.0 + 2.0 * beta;
    const bool first = f == 0;  // face 0: no previous coefficients
    const double m = first ? bb : bb + beta * cp_p;
    const double num = first ? dd : dd + beta * dp_p;
    bool ok = true;
    const fp64::Recip rm = fp64::recip(m);
    double cpk = fp64::quot(-beta, rm, ok);
    double dpk = fp64::quot(num, rm, ok);
    if (__builtin_expect(!ok, 0)) {
      cpk = -beta / m;
      dpk = num / m;
    }
    sm100::tmem_st_f64(tmem + 2 * f, cpk);
    sm100::tmem_st_f64(tmem + dp_col + 2 * f, dpk);
    cp_p = cpk;
    dp_p = dpk;
  };

  // one role's K sweep (the role is compile-time per loop: no cross-role live state).
  // Horizontal warps: ps of level k (pass B: u', v'). Thomas warps: formation of face
  // k-2 (its upper ps, of level k-1, was published by this level's barrier) beside the
  // recursion of face k-3, so the two division chains overlap.
  auto sweep = [&](auto role_tag) {
    constexpr bool kThomas = decltype(role_tag)::value;
#pragma unroll 1
    for (int k = 0; k < nz; ++k) {
      __syncthreads();  // level k landed (observed by the waiter); the slot of level k-1
                        // is free; ps of level k-1 is visible
      if constexpr (kIssue == 0 || (kIssue == 1) != kThomas) issue(k + kAStages - 1);
      const double* S = ring + (k % kAStages) * kStage;
      if constexpr (kThomas) {
        const double wk = S[oW + t], rhok = S[oRho + t], thk = S[oTh + t], fwk = S[oFW + t];
        if (k >= 2) {
          bool ok = true;
          double beta, dd;
          formation(k - 2, rho_2, rho_1, th_2, th_1, w_2, fw_2, beta, dd, ok);
          if (k >= 3) recursion(k - 3, pend_beta, pend_dd);
          pend_beta = beta;
          pend_dd = dd;
        }
        rho_2 = rho_1, th_2 = th_1, w_2 = w_1, fw_2 = fw_1;
        rho_1 = rhok, th_1 = thk, w_1 = wk, fw_1 = fwk;
      } else {
        const double* Pp = S + oP + (row + 1) * kAW + (lane + 2);
        const double pk = Pp[0], pe = Pp[1], pw = Pp[-1], pnn = Pp[kAW], psth = Pp[-kAW];
        const double uk = S[oU + row * kAW + lane + 2], ukw = S[oU + row * kAW + lane + 1];
        const double fuk = S[oFU + row * kAW + lane + 2], fukw = S[oFU + row * kAW + lane + 1];
        const double vk = S[oV + (row + 1) * kTX + lane], vks = S[oV + row * kTX + lane];
        const double fvk = S[oFV + (row + 1) * kTX + lane], fvks = S[oFV + row * kTX + lane];
        const double pc = kB ? S[oPc + t] : pk;  // p at the column (the RK2 base)

        // PGF at p (A) / pa (B) applied to the current momentum, plus h * slow tendency
        const double unk = east ? 0.0 : uk - c.h_rdx * (pe - pk) + c.h * fuk;
        const double vnk = north ? 0.0 : vk - c.h_rdy * (pnn - pk) + c.h * fvk;
        const double uw = west ? 0.0 : ukw - c.h_rdx * (pk - pw) + c.h * fukw;
        const double vs = south ? 0.0 : vks - c.h_rdy * (pk - psth) + c.h * fvks;
        const double psk = pc - c.h_cs2 * (c.rdx * (unk - uw) + c.rdy * (vnk - vs));
        ps_s[k * kThreads + t] = psk;
        if (kB && active) {  // damped momentum of the short step
          const double tau = tau_at(k + 1);
          const int64_t o = col + static_cast<int64_t>(k) * P;
          a.un[o] = unk - tau * unk;
          a.vn[o] = vnk - tau * vnk;
        }
        if (warp == kAcoWaitWarp && k + 1 < nz) wait_level(k + 1);
      }
    }
  };
  if (thomas)
    sweep(std::true_type{});
  else
    sweep(std::false_type{});
  __syncthreads();  // every ps is visible

  if (thomas) {
    // drain: formation of the last face nz-2 (levels nz-2, nz-1 are in registers), the
    // recursions of faces nz-3 and nz-2
    if (nz >= 2) {
      bool ok = true;
      double beta, dd;
      formation(nz - 2, rho_2, rho_1, th_2, th_1, w_2, fw_2, beta, dd, ok);
      if (nz >= 3) recursion(nz - 3, pend_beta, pend_dd);
      recursion(nz - 2, beta, dd);
    }
    sm100::tmem_wait_st();
    // back substitution (faces nz-2 .. 0, w(nz) = 0 is the lid), four per TMEM load,
    // then the pressure update (pass B: the damped w of the short step)
    double* pout = kB ? a.pn : a.pa_out;
    if (kB && active) a.wn[col + static_cast<int64_t>(nz - 1) * P] = 0.0 - tau_at(nz) * 0.0;
    double wk1 = 0.0;
    const int nf = nz - 1;
#pragma unroll 1
    for (int cb = (nf - 1) / 4; cb >= 0; --cb) {
      double cpv[4], dpv[4];
      sm100::tmem_ld_4f64(tmem + 8 * cb, cpv);
      sm100::tmem_ld_4f64(tmem + dp_col + 8 * cb, dpv);
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        const int f = 4 * cb + q;  // face f = w-point f+1 (1-based) at 0-based level f
        if (f >= nf) continue;
        const double wkk = (f == nf - 1) ? dpv[q] : dpv[q] - cpv[q] * wk1;
        const double pk1 = ps_s[(f + 1) * kThreads + t] - c.h_cs2_rdz * (wk1 - wkk);
        if (active) {
          pout[col + static_cast<int64_t>(f + 1) * P] = pk1;
          if (kB) a.wn[col + static_cast<int64_t>(f) * P] = wkk - tau_at(f + 1) * wkk;
        }
        wk1 = wkk;
      }
    }
    if (active) pout[col] = ps_s[t] - c.h_cs2_rdz * wk1;
  }
  sm100::tmem_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem_base_slot, tmem_cols);
}

// theta = thb + dtf * fth, rho = rhob + dtf * frho over the span (asuca.h90 stage end)
__global__ void k_asu_stage_end(const double* thb, const double* fth, const double* rhob,
                                const double* frho, double* th, double* rho, Grid3 g, int nz,
                                double dtf, Span sp) {
  const int64_t i = sp.ilo + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t j = sp.jlo + blockIdx.y;
  if (i > sp.ihi) return;
  int64_t o = (j - 1) * g.pitch + (i - 1);
  for (int k = 0; k < nz; ++k, o += g.plane) {
    th[o] = thb[o] + dtf * fth[o];
    rho[o] = rhob[o] + dtf * frho[o];
  }
}

}  // namespace

AsuAcoConst make_asu_aco_const(double h, double dtau, double rdx, double rdy, double rdz,
                               double cs2, double grav, double th0, double rdmp, int64_t nbnd,
                               int64_t kdmp, double rnbnd, double rnzd) {
  AsuAcoConst c;
  c.h = h;
  c.rdx = rdx;
  c.rdy = rdy;
  c.th0 = th0;
  c.h_rdx = h * rdx;                     // `h * rdx * (...)`
  c.h_rdy = h * rdy;
  c.h_rdz = h * rdz;                     // `h * rdz * (...) / rf`
  c.h_cs2 = h * cs2;                     // `h * cs2 * (...)`
  c.h_cs2_rdz = h * cs2 * rdz;           // `h * cs2 * rdz * (...)`
  c.beta_num = h * h * cs2 * rdz * rdz;  // `h * h * cs2 * rdz * rdz / rf`
  c.h_grav = h * grav;                   // `h * grav * (...) / th0`
  c.dtau_rdmp = dtau * rdmp;             // `dtau * rdmp * max(...)`
  c.nbnd = nbnd;
  c.kdmp = kdmp;
  c.rnbnd = rnbnd;
  c.rnzd = rnzd;
  return c;
}

bool asuca_fits(int64_t nz) { return nz >= 2 && nz - 1 <= 128; }

cudaError_t launch_asu_tend(const AsuState& s, const AsuTend& f, Grid3 g, int64_t nz, int64_t nj,
                            double rdx, double rdy, double rdz, const Span& sp, cudaStream_t st) {
  if (sp.ihi < sp.ilo || sp.jhi < sp.jlo) return cudaSuccess;
  const size_t smem = static_cast<size_t>(kTStages) * kTStage * sizeof(double) + 128;
  {
    cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(k_asu_tend), smem);
    if (e != cudaSuccess) return e;
  }
  TendMaps maps{};
  const double* fld[5] = {s.rho, s.th, s.u, s.v, s.w};
  for (int q = 0; q < 5; ++q)
    if (!make_box_map(&maps.m[q], fld[q], g, nj, nz, kTW, kTR)) return cudaErrorInvalidValue;
  TendArgs a{s, f, g, static_cast<int>(nz), nj, -kIOff, g.pitch - kIOff - 1, rdx, rdy, rdz, sp};
  dim3 block(kTX, kTY);
  dim3 grid(static_cast<unsigned>((sp.ihi - sp.ilo + 1 + kTXo - 1) / kTXo),
            static_cast<unsigned>((sp.jhi - sp.jlo + 1 + kTY - 1) / kTY));
  k_asu_tend<<<grid, block, smem, st>>>(maps, a);
  return cudaGetLastError();
}

cudaError_t launch_asu_acoustic(bool pass_b, const AsuState& s, const double* fu,
                                const double* fv, const double* fw, const double* pa,
                                double* pa_out, double* un, double* vn, double* wn, double* pn,
                                Grid3 g, int64_t nz, int64_t nj, const AsuAcoConst& c,
                                const Span& sp, cudaStream_t st) {
  if (sp.ihi < sp.ilo || sp.jhi < sp.jlo) return cudaSuccess;
  if (!asuca_fits(nz)) return cudaErrorInvalidValue;
  const int stage = pass_b ? kAoPc + kTX * kTY : kAoPc;  // padded plane tiles
  // two CTAs per SM share the SM's 512 TMEM columns; pad small-nz launches so a third
  // CTA never blocks in tcgen05.alloc (+128 B: the ring's 128-B round-up)
  const size_t smem = std::max<size_t>(
      (static_cast<size_t>(kAStages) * stage + static_cast<size_t>(nz) * kThreads) *
              sizeof(double) + 128,
      80 * 1024);
  AcoMaps maps{};
  {
    const double* fld[10] = {pass_b ? pa : s.p, s.u, fu, s.v, fv, s.w, s.rho, s.th, fw, s.p};
    for (int f = 0; f < (pass_b ? 10 : 9); ++f)
      if (!make_box_map(&maps.m[f], fld[f], g, nj, nz, kAcoBox[f].bw, kAcoBox[f].bh))
        return cudaErrorInvalidValue;
  }
  const void* kern = pass_b ? reinterpret_cast<const void*>(k_asu_acoustic<true>)
                            : reinterpret_cast<const void*>(k_asu_acoustic<false>);
  {
    cudaError_t e = ensure_dynamic_smem(kern, smem);
    if (e != cudaSuccess) return e;
  }
  AcoArgs a{s, fu, fv, fw, pa, pa_out, un, vn, wn, pn, g, static_cast<int>(nz), nj,
            -kIOff, g.pitch - kIOff - 1, c, sp};
  dim3 block(kTX, 2 * kTY);
  dim3 grid(static_cast<unsigned>((sp.ihi - sp.ilo + 1 + kTX - 1) / kTX),
            static_cast<unsigned>((sp.jhi - sp.jlo + 1 + kTY - 1) / kTY));
  if (pass_b)
    k_asu_acoustic<true><<<grid, block, smem, st>>>(maps, a);
  else
    k_asu_acoustic<false><<<grid, block, smem, st>>>(maps, a);
  return cudaGetLastError();
}

cudaError_t launch_asu_stage_end(const double* thb, const double* fth, const double* rhob,
                                 const double* frho, double* th, double* rho, Grid3 g,
                                 int64_t nz, double dtf, const Span& sp, cudaStream_t st) {
  if (sp.ihi < sp.ilo || sp.jhi < sp.jlo) return cudaSuccess;
  dim3 block(128);
  dim3 grid(static_cast<unsigned>((sp.ihi - sp.ilo + 1 + 127) / 128),
            static_cast<unsigned>(sp.jhi - sp.jlo + 1));
  k_asu_stage_end<<<grid, block, 0, st>>>(thb, fth, rhob, frho, th, rho, g, static_cast<int>(nz),
                                          dtf, sp);
  return cudaGetLastError();
}

}  // namespace hfb

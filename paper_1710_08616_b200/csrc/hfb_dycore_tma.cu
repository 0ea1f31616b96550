// hfb_dycore_tma.cu — the whole dycore timestep (dycore.h90 regions 1-8) in one kernel,
// fed by TMA: round 1's TMA twin of k_dyn_step_ws (then fed by cp.async; since round 2 the
// product kernel is TMA-fed itself, with role-split loops and a different waiter), kept
// as a measured alternative (hfb_set_option "variant" "tma" in the A/B build; see MEASURED below).
//
// Machine organisation (one CTA per 32 x 4 tile of (i,j) columns, marching K):
//   * per K level, six threads issue six 3-D TMA box loads (th with its 2-cell ring, u
//     with i-1..i-2, v with j-1, w, p with a 1-cell ring, rho) into one slot of a
//     kStages-deep shared-memory ring and arms the slot's mbarrier with the byte count.
//     Out-of-array cells of a box are zero-filled by the TMA unit (never used by an
//     active column). The cp.async version spent ~14% of all instructions on per-thread
//     copy addressing and LDGSTS; here it is a handful of instructions per CTA and level.
//   * warps 0-3 (ACOUSTIC) run the pressure gradient, the divergence and the HE-VI
//     Thomas sweep; each thread owns one TMEM lane for its column's cp(k), dp(k).
//   * warps 4-7 (ADVECTION) run the flux-limited advection of theta for the same rows
//     (they read levels k..k+2 of th for the vertical faces).
//   * warp 0 waits on the slot mbarrier of the newest level needed (parity = pass over
//     the ring); one CTA barrier per level then publishes it and frees the slot of
//     level k-1 for level k-1+kStages (the same sync structure as the cp.async twin).
//   * MEASURED (512x512x58, B200): this kernel is SLOWER than its cp.async twin (0.414 vs
//     0.379 ms per step) although its data-movement skeleton is faster (0.219 vs 0.235
//     ms with both roles' arithmetic skipped), so the cp.async kernel stays the product
//     path and this one is the "tma" variant. Also measured and dropped: a
//     dedicated producer warp with empty/full barrier pairs (0.430 ms: a ninth warp
//     cuts the register budget to 96) and refills by the last warp out of a slot through
//     an acq_rel arrival counter, no CTA barrier (0.441 ms).
//   * HE-VI divisions share reciprocals (hfb_fp64.cuh).
// Compulsory DRAM traffic: 6 fields read + 5 written = 88 B per grid point.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "hfb_fp64.cuh"
#include "hfb_kernels.cuh"
#include "hfb_sm100.cuh"
#include "hfb_tmap.cuh"

namespace hfb {

namespace {

constexpr int kTX = 32, kTY = 4, kCols = kTX * kTY;  // columns per tile
constexpr int kWarps = 2 * kTY;                      // 4 acoustic + 4 advection
constexpr int kThreadsTma = kWarps * kTX;            // 256
constexpr int kStages = 6;
constexpr int kTmemCols = 256;
constexpr int kDpCol = 128;

// one ring slot: six box tiles, each starting 128-B aligned (TMA destination rule)
constexpr int pad16(int n) { return (n + 15) / 16 * 16; }
constexpr int kThW = 36, kThR = kTY + 4;  // th: cols i0-2..i0+33, rows j0-2..j0+5
constexpr int kUW = 34, kUR = kTY;        // u:  cols i0-2..i0+31, rows j0..j0+3
constexpr int kVW = 32, kVR = kTY + 1;    // v:  cols i0..i0+31,   rows j0-1..j0+3
constexpr int kWW = 32, kWR = kTY;        // w:  cols i0..i0+31,   rows j0..j0+3
constexpr int kPW = 36, kPR = kTY + 2;    // p:  cols i0-2..i0+33, rows j0-1..j0+4
constexpr int kRW = 32, kRR = kTY;        // rho
constexpr int kOffTh = 0;
constexpr int kOffU = kOffTh + pad16(kThW * kThR);
constexpr int kOffV = kOffU + pad16(kUW * kUR);
constexpr int kOffW = kOffV + pad16(kVW * kVR);
constexpr int kOffP = kOffW + pad16(kWW * kWR);
constexpr int kOffRho = kOffP + pad16(kPW * kPR);
constexpr int kStageDoubles = kOffRho + pad16(kRW * kRR);  // 1072
constexpr uint32_t kStageTx =
    (kThW * kThR + kUW * kUR + kVW * kVR + kWW * kWR + kPW * kPR + kRW * kRR) * 8;  // 8448

enum { kMapTh, kMapU, kMapV, kMapW, kMapP, kMapRho, kMaps };

struct TmaMaps {
  CUtensorMap m[kMaps];
};

struct TmaStepArgs {
  DynOut out;
  Grid3 g;
  int nz;
  int debug_skip;  // profiling experiments only: 1 = no advection, 2 = no acoustic
  const double* tsfc;  // column physics (full_step), null when off
  double* colm;
  double dt_rrelax, dt_ch;
  DynIn base;  // RK3 stages 2-3: the state at the start of the step
  DynConst c;
  Span sp;
  int wait_warp;  // the warp that waits on the slot barriers
};

// limited upwind face flux (see face_flux_up in hfb_dycore_tmem.cu for the derivation)
template <bool kCheck>
__device__ __forceinline__ double face_flux(int64_t f, int64_t n, double vel, double tm1,
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

template <bool kPhys, bool kRK>
__global__ void __launch_bounds__(kThreadsTma, 2)
    k_dyn_step_tma(const __grid_constant__ TmaMaps maps, const TmaStepArgs a) {
  static_assert(!(kPhys && kRK), "column physics is not fused into RK stages");
  extern __shared__ __align__(1024) double smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ uint32_t tmem_base_slot;
  // TMA destinations must be 128-B aligned: align the ring explicitly (the launch adds
  // the slack) instead of trusting the placement of the dynamic segment
  double* ring = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~static_cast<uintptr_t>(127));
  double* ps_s = ring + kStages * kStageDoubles;  // nz x 128 (ps of each column)

  const int lane = threadIdx.x, warp = threadIdx.y;  // blockDim = (32, 8)
  const bool acoustic = warp < kTY;
  const int row = acoustic ? warp : warp - kTY;  // tile row served by a consumer warp
  const int t = row * kTX + lane;                // column within the tile (consumers)
  const int64_t i0 = a.sp.ilo + static_cast<int64_t>(blockIdx.x) * kTX;
  const int64_t j0 = a.sp.jlo + static_cast<int64_t>(blockIdx.y) * kTY;
  const int64_t i = i0 + lane, j = j0 + row;
  const bool active = i <= a.sp.ihi && j <= a.sp.jhi;
  const int nz = a.nz;
  const int64_t P = a.g.plane, W = a.g.pitch;
  const DynConst& c = a.c;
  const int64_t gi = i + a.sp.i0, gj = j + a.sp.j0, gnx = a.sp.gnx, gny = a.sp.gny;
  const int64_t gi0 = i0 + a.sp.i0, gj0 = j0 + a.sp.j0;
  const bool interior = gi0 >= 3 && gi0 + kTX - 1 <= gnx - 2 && gj0 >= 3 &&
                        gj0 + kTY - 1 <= gny - 2 && i0 + kTX - 1 <= a.sp.ihi &&
                        j0 + kTY - 1 <= a.sp.jhi;
  const uint32_t full0 = sm100::smem_u32(full_bar);

  if (warp == 0) sm100::tmem_alloc(&tmem_base_slot, kTmemCols);
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) sm100::mbar_init(full0 + 8 * s, 1);
    sm100::mbar_fence_init();
    for (int m = 0; m < kMaps; ++m) sm100::tma_prefetch_desc(&maps.m[m]);
  }
  sm100::tmem_fence_before();
  __syncthreads();
  sm100::tmem_fence_after();

  // box origins in allocation coordinates (x = kIOff + i', y = kHalo + j'; i', j'
  // 0-based local), level z = k
  const int xi = static_cast<int>(kIOff + (i0 - 1)), yj = static_cast<int>(kHalo + (j0 - 1));
  const uint32_t ring0 = sm100::smem_u32(ring);
  // the six box loads of a level are issued by lane 0 of warps 0-5 (one field each, so
  // no warp carries all of the issue latency); warp 0 also arms the slot's barrier
  // (the tx-count may go transiently negative, PTX ISA mbarrier tx-count range)
  const bool tma_lane = lane == 0 && warp < kMaps;
  int f_off = kOffTh, f_dx = -2, f_dy = -2;
  switch (warp) {
    case kMapU: f_off = kOffU; f_dx = -2; f_dy = 0; break;
    case kMapV: f_off = kOffV; f_dx = 0; f_dy = -1; break;
    case kMapW: f_off = kOffW; f_dx = 0; f_dy = 0; break;
    case kMapP: f_off = kOffP; f_dx = -2; f_dy = -1; break;
    case kMapRho: f_off = kOffRho; f_dx = 0; f_dy = 0; break;
    default: break;
  }
  const CUtensorMap* f_map = &maps.m[warp < kMaps ? warp : 0];
  const uint32_t f_dst = ring0 + static_cast<uint32_t>(f_off * 8);
  auto issue = [&](int k) {  // this lane's field of level k into slot k % kStages
    const int s = k % kStages;
    const uint32_t fb = full0 + 8 * s;
    if (warp == 0) sm100::mbar_arrive_expect_tx(fb, kStageTx);
    sm100::tma_load_3d(f_dst + static_cast<uint32_t>(s * kStageDoubles * 8), f_map, fb,
                       xi + f_dx, yj + f_dy, k);
  };
  if (tma_lane)
    for (int k = 0; k < kStages && k < nz; ++k) issue(k);

  {
    const uint32_t tmem = tmem_base_slot + (static_cast<uint32_t>(32 * row) << 16);
    const int64_t col = (j - 1) * W + (i - 1);
    double* out_th = a.out.th + col;  // running pointers (advance one plane per level)
    double* out_u = a.out.u + col;
    double* out_v = a.out.v + col;
    const bool east = gi == gnx, west = gi == 1, north = gj == gny, south = gj == 1;
    const int thc = (row + 2) * kThW + (lane + 2);

    double th_prev = 0.0, w_prev = 0.0;
    double rho_prev = 0.0, ps_prev = 0.0, cp_prev = 0.0, dp_prev = 0.0;
    double fz_prev = 0.0;
    double phys_cs = 0.0, phys_cm = 0.0, colm_ij = 0.0, tsfc_ij = 0.0;
    struct BaseLevel {
      double th, u, uw, v, vs, p, w;
    };
    auto base_load = [&](int k) {
      BaseLevel b{};
      if (kRK && k < nz && active) {
        const int64_t o = col + static_cast<int64_t>(k) * P;
        if (acoustic) {
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
    BaseLevel bcur = base_load(0);
    double wb_prev = 0.0;
    if (kPhys && !acoustic && active) {
      colm_ij = a.colm[(j - 1) * W + (i - 1)];
      tsfc_ij = a.tsfc[(j - 1) * W + (i - 1)];
    }
    double pend_beta = 0.0, pend_bb = 1.0, pend_dd = 0.0;
    const fp64::Recip rth0 = fp64::recip(c.th0);

    auto thomas_fast = [&](int f, double& cpk, double& dpk, bool& ok) {
      const double m = f == 0 ? pend_bb : pend_bb + pend_beta * cp_prev;
      const double num = f == 0 ? pend_dd : pend_dd + pend_beta * dp_prev;
      const fp64::Recip rm = fp64::recip(m);
      cpk = fp64::quot(-pend_beta, rm, ok);
      dpk = fp64::quot(num, rm, ok);
    };
    auto thomas_div = [&](int f, double& cpk, double& dpk) {
      if (f == 0) {
        cpk = -pend_beta / pend_bb;
        dpk = pend_dd / pend_bb;
      } else {
        const double m = pend_bb + pend_beta * cp_prev;
        cpk = -pend_beta / m;
        dpk = (pend_dd + pend_beta * dp_prev) / m;
      }
    };
    auto thomas_commit = [&](int f, double cpk, double dpk) {
      sm100::tmem_st_f64(tmem + 2 * f, cpk);
      sm100::tmem_st_f64(tmem + kDpCol + 2 * f, dpk);
      cp_prev = cpk;
      dp_prev = dpk;
    };

    int s0 = 0;
    auto level = [&](int k, auto interior_tag) {
      constexpr bool kIn = decltype(interior_tag)::value;
      const BaseLevel bnext = base_load(k + 1);
      const int kk = k + 1;
      const int s1 = s0 == kStages - 1 ? 0 : s0 + 1;
      const int s2 = s1 == kStages - 1 ? 0 : s1 + 1;
      const double* S = ring + s0 * kStageDoubles;
      const double tk = S[kOffTh + thc];
      const double* Up = S + kOffU + row * kUW + (lane + 2);
      const double ui = Up[0], uim1 = Up[-1];
      const double* Vp = S + kOffV + (row + 1) * kVW + lane;
      const double vj = Vp[0], vjm1 = Vp[-kVW];
      const double wk = S[kOffW + row * kWW + lane];
      if (acoustic) {
        if ((a.debug_skip & 2) == 0) {
          const double* Pp = S + kOffP + (row + 1) * kPW + (lane + 2);
          const double pk = Pp[0], pe = Pp[1], pw = Pp[-1], pnn = Pp[kPW], psth = Pp[-kPW];
          const double rhok = S[kOffRho + row * kRW + lane];
          const double unk0 = (kRK ? bcur.u : ui) - c.dt_rdx * (pe - pk);
          const double vnk0 = (kRK ? bcur.v : vj) - c.dt_rdy * (pnn - pk);
          const double uw0 = (kRK ? bcur.uw : uim1) - c.dt_rdx * (pk - pw);
          const double vs0 = (kRK ? bcur.vs : vjm1) - c.dt_rdy * (pk - psth);
          const double unk = (!kIn && east) ? 0.0 : unk0;
          const double vnk = (!kIn && north) ? 0.0 : vnk0;
          const double uw = (!kIn && west) ? 0.0 : uw0;
          const double vs = (!kIn && south) ? 0.0 : vs0;
          const double psk =
              (kRK ? bcur.p : pk) - c.dt_cs2 * (c.rdx * (unk - uw) + c.rdy * (vnk - vs));
          if (kIn || active) {
            *out_u = unk;
            *out_v = vnk;
          }
          ps_s[k * kCols + t] = psk;
          // Thomas recursion of face k-2 (coefficients formed last level) next to the
          // coefficient formation of face k-1: two independent division chains
          bool ok = true;
          double cpk = 0.0, dpk = 0.0, beta = 0.0, dd = 0.0;
          if (k >= 2) thomas_fast(k - 2, cpk, dpk, ok);
          const double w_rhs = kRK ? wb_prev : w_prev;
          const double n_ps = c.dt_rdz * (psk - ps_prev);
          const double n_th = c.dt_grav * (0.5 * (th_prev + tk) - c.th0);
          if (k >= 1) {
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
          if (k >= 2) thomas_commit(k - 2, cpk, dpk);
          if (k >= 1) {
            pend_beta = beta;
            pend_bb = 1.0 + 2.0 * beta;
            pend_dd = dd;
          }
          rho_prev = rhok;
          ps_prev = psk;
          if (kRK) wb_prev = bcur.w;
        }
      } else if ((a.debug_skip & 1) == 0) {
        const double* T0 = S + kOffTh + thc;
        const double tkp1 = (kk + 1 <= nz) ? ring[s1 * kStageDoubles + kOffTh + thc] : 0.0;
        const double tkp2 = (kk + 2 <= nz) ? ring[s2 * kStageDoubles + kOffTh + thc] : 0.0;
        const double xm2 = T0[-2], xm1 = T0[-1], xp1 = T0[1], xp2 = T0[2];
        const double ym2 = T0[-2 * kThW], ym1 = T0[-kThW], yp1 = T0[kThW], yp2 = T0[2 * kThW];
        const double fzk = face_flux<true>(kk, nz, wk, th_prev, tk, tkp1, tkp2);
        const double fxe = face_flux<!kIn>(gi, gnx, ui, xm1, tk, xp1, xp2);
        const double fxw = face_flux<!kIn>(gi - 1, gnx, uim1, xm2, xm1, tk, xp1);
        const double fyn = face_flux<!kIn>(gj, gny, vj, ym1, tk, yp1, yp2);
        const double fys = face_flux<!kIn>(gj - 1, gny, vjm1, ym2, ym1, tk, yp1);
        const double ue = (!kIn && east) ? 0.0 : ui;
        const double uwf = (!kIn && west) ? 0.0 : uim1;
        const double vnf = (!kIn && north) ? 0.0 : vj;
        const double vsf = (!kIn && south) ? 0.0 : vjm1;
        const double wt = (kk == nz) ? 0.0 : wk;
        const double wb = (kk == 1) ? 0.0 : w_prev;
        double flux = c.rdx * (fxe - fxw) + c.rdy * (fyn - fys);
        flux = flux + c.rdz * (fzk - fz_prev);
        double div = c.rdx * (ue - uwf) + c.rdy * (vnf - vsf);
        div = div + c.rdz * (wt - wb);
        double thv = (kRK ? bcur.th : tk) - c.dt * (flux - tk * div);
        if (kPhys) {  // column_physics (dycore.h90) on the new theta of this level
          thv = thv - a.dt_rrelax * (thv - colm_ij);
          if (kk == 1) {  // new u, v at the lowest level (region 5), from the plane
            const double* Pp = S + kOffP + (row + 1) * kPW + (lane + 2);
            const double un1 = (!kIn && east) ? 0.0 : ui - c.dt_rdx * (Pp[1] - Pp[0]);
            const double vn1 = (!kIn && north) ? 0.0 : vj - c.dt_rdy * (Pp[kPW] - Pp[0]);
            const double wspd = sqrt(un1 * un1 + vn1 * vn1);
            thv = thv + a.dt_ch * wspd * (tsfc_ij - thv) * c.rdz / S[kOffRho + row * kRW + lane];
          }
          const double rhok = S[kOffRho + row * kRW + lane];
          phys_cs = phys_cs + rhok * thv;
          phys_cm = phys_cm + rhok;
        }
        if (kIn || active) *out_th = thv;
        fz_prev = fzk;
      }
      th_prev = tk;
      w_prev = wk;
      out_th += P;
      out_u += P;
      out_v += P;
      bcur = bnext;
      s0 = s1;
    };

    // One warp waits for the levels: k+3 at the END of level k (after its own work, so
    // the ~90-cycle mbarrier wait overlaps the other warps' arithmetic instead of
    // sitting on the critical path), levels 0-2 before the loop. The CTA barrier at the
    // top of level k+1 then publishes k+3 to every warp (mbarrier acquire, bar.sync) —
    // the newest level the advection reads there — and frees the slot of level k.
    const bool waiter = warp == a.wait_warp;
    if (waiter)
      for (int l = 0; l < 3 && l < nz; ++l)
        sm100::mbar_wait(full0 + 8 * (l % kStages), (l / kStages) & 1);
#pragma unroll 1
    for (int k = 0; k < nz; ++k) {
      __syncthreads();
      if (tma_lane && k >= 1 && k - 1 + kStages < nz) issue(k - 1 + kStages);
      if (interior)
        level(k, std::true_type{});
      else
        level(k, std::false_type{});
      if (waiter && k + 3 < nz)
        sm100::mbar_wait(full0 + 8 * ((k + 3) % kStages), ((k + 3) / kStages) & 1);
    }
    if (acoustic && nz >= 2) {  // drain the last face
      bool ok = true;
      double cpk, dpk;
      thomas_fast(nz - 2, cpk, dpk, ok);
      if (!ok) thomas_div(nz - 2, cpk, dpk);
      thomas_commit(nz - 2, cpk, dpk);
    }
    if (kPhys && !acoustic && active) a.colm[(j - 1) * W + (i - 1)] = phys_cs / phys_cm;

    if (acoustic) {  // back substitution + pressure update (region 7), 4 faces per TMEM load
      sm100::tmem_wait_st();
      double* wn = a.out.w + col + static_cast<int64_t>(nz - 1) * P;
      double* pn = a.out.p + col + static_cast<int64_t>(nz - 1) * P;
      if (active) *wn = 0.0;
      double wk1 = 0.0;
      const int nf = nz - 1;
      const double* psp = ps_s + (nz - 1) * kCols + t;  // ps(f+1)
#pragma unroll 1
      for (int cb = (nf - 1) / 4; cb >= 0; --cb) {
        double cpv[4], dpv[4];
        sm100::tmem_ld_4f64(tmem + 8 * cb, cpv);
        sm100::tmem_ld_4f64(tmem + kDpCol + 8 * cb, dpv);
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
          pn -= P;
          psp -= kCols;
          wk1 = wkk;
        }
      }
      if (active) *pn = *psp - c.dt_cs2_rdz * wk1;
    }
  }
  sm100::tmem_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem_base_slot, kTmemCols);
}

}  // namespace

// make_box_map (hfb_tmap.cuh) is defined with the product step in hfb_dycore_tmem.cu

cudaError_t launch_dycore_step_tma(const DynIn& in, const DynOut& out, Grid3 g, int64_t nz,
                                   int64_t nj, const DynConst& c, const Span& sp,
                                   cudaStream_t s, const PhysArgs* phys, const DynIn* base,
                                   int debug_skip) {
  if (sp.ihi < sp.ilo || sp.jhi < sp.jlo) return cudaSuccess;
  if (!dycore_step_tmem_fits(nz)) return cudaErrorInvalidValue;
  if (phys && base) return cudaErrorInvalidValue;
  TmaMaps maps;
  const bool ok = make_box_map(&maps.m[kMapTh], in.th, g, nj, nz, kThW, kThR) &&
                  make_box_map(&maps.m[kMapU], in.u, g, nj, nz, kUW, kUR) &&
                  make_box_map(&maps.m[kMapV], in.v, g, nj, nz, kVW, kVR) &&
                  make_box_map(&maps.m[kMapW], in.w, g, nj, nz, kWW, kWR) &&
                  make_box_map(&maps.m[kMapP], in.p, g, nj, nz, kPW, kPR) &&
                  make_box_map(&maps.m[kMapRho], in.rho, g, nj, nz, kRW, kRR);
  if (!ok) return cudaErrorInvalidValue;
  // two CTAs per SM share its 512 TMEM columns; small-nz launches pad shared memory
  // so that a third CTA never blocks in tcgen05.alloc
  const size_t smem = std::max<size_t>((static_cast<size_t>(kStages) * kStageDoubles +
                                        static_cast<size_t>(nz) * kCols) * sizeof(double) + 128,
                                       80 * 1024);
  const int variant = phys ? 1 : base ? 2 : 0;
  void (*kern)(const TmaMaps, const TmaStepArgs) = variant == 1   ? k_dyn_step_tma<true, false>
                                                   : variant == 2 ? k_dyn_step_tma<false, true>
                                                                  : k_dyn_step_tma<false, false>;
  {
    cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
  }
  TmaStepArgs a{out, g, static_cast<int>(nz), debug_skip,
                phys ? phys->tsfc : nullptr, phys ? phys->colm : nullptr,
                phys ? phys->dt_rrelax : 0.0, phys ? phys->dt_ch : 0.0,
                base ? *base : DynIn{}, c, sp,
                getenv("HFB_TMA_WAITWARP") ? atoi(getenv("HFB_TMA_WAITWARP")) : 7};
  dim3 block(kTX, kWarps);
  dim3 grid(static_cast<unsigned>((sp.ihi - sp.ilo + 1 + kTX - 1) / kTX),
            static_cast<unsigned>((sp.jhi - sp.jlo + 1 + kTY - 1) / kTY));
  kern<<<grid, block, smem, s>>>(maps, a);
  return cudaGetLastError();
}

}  // namespace hfb

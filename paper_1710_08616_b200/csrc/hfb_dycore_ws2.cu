// hfb_dycore_ws2.cu — the fused dycore timestep (dycore.h90 regions 1-8) with TWO
// columns per thread: one CTA per SM owns a 32 x 8 tile of (i,j) columns; warps 0-3 run
// the acoustic / HE-VI part and warps 4-7 the flux-limited advection, each thread for
// the columns (i, j) and (i, j+1) of two adjacent tile rows.
//
// Why two columns: in the one-column kernel (k_dyn_step_ws, hfb_dycore_tmem.cu) a third
// of the instructions per grid point were per-level bookkeeping of each warp (wait,
// barrier, copy issue, ring and output addressing, loop control; ncu source counts,
// profiles/r01_v10). Two columns per thread pay it once for two points and give every
// warp two independent dependency chains. Adjacent rows also share work: the north face
// flux of row j is the south face of row j+1 (9 limited face fluxes per 2 points, not
// 10), the v' of row j is the vs of row j+1, and the y-stencils overlap in shared memory.
//
// Budget (1 CTA/SM): TMEM 512 columns (cp, dp of 2 columns x 64 faces per lane),
// shared memory kStages x 14.6 KB ring + nz x 2 KB ps.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "hfb_fp64.cuh"
#include "hfb_kernels.cuh"
#include "hfb_sm100.cuh"

namespace hfb {

namespace {

constexpr int kTX = 32, kRows = 8, kPairs = kRows / 2;  // tile 32 x 8, 4 row pairs
constexpr int kThreads = 2 * kPairs * kTX;              // 256: 4 acoustic + 4 advection warps
constexpr int kCols = kTX * kRows;                      // 256 columns per tile
constexpr int kStages = 6;
constexpr int kTmemCols = 512;
// ring slot: th rows j0-2..j0+9 x cols i0-2..i0+33; u rows j0..j0+7 x cols i0-2..i0+31;
// v rows j0-1..j0+7 x cols i0..i0+31; w, rho rows j0..j0+7 x cols i0..i0+31;
// p rows j0-1..j0+8 x cols i0-2..i0+33
constexpr int kThW = 36, kThR = kRows + 4;
constexpr int kUW = 34, kUR = kRows;
constexpr int kVW = 32, kVR = kRows + 1;
constexpr int kWW = 32, kWR = kRows;
constexpr int kPW = 36, kPR = kRows + 2;
constexpr int kRW = 32, kRR = kRows;
constexpr int kOffTh = 0;
constexpr int kOffU = kOffTh + kThW * kThR;
constexpr int kOffV = kOffU + kUW * kUR;
constexpr int kOffW = kOffV + kVW * kVR;
constexpr int kOffP = kOffW + kWW * kWR;
constexpr int kOffRho = kOffP + kPW * kPR;
constexpr int kStageDoubles = kOffRho + kRW * kRR;  // 1864
constexpr int kChunks = kStageDoubles / 2;          // 932 16-B chunks per level
static_assert(kStageDoubles % 2 == 0, "16-B chunks");
constexpr int kFullChunks = kChunks / kThreads;     // 3 for everyone
constexpr int kExtraChunks = kChunks - kFullChunks * kThreads;  // + 1 for the first 164
static_assert(kExtraChunks > 0 && kExtraChunks <= 6 * kTX, "4th chunk in warps 0-5");

struct Ws2Args {
  DynIn in;
  DynOut out;
  Grid3 g;
  int nz;
  int debug_skip;  // profiling experiments only: 1 = no advection, 2 = no acoustic
  const double* tsfc;  // column physics (full_step), null when off
  double* colm;
  double dt_rrelax, dt_ch;
  DynIn base;  // RK3 stages 2-3: the state at the start of the step
  int64_t nj;
  int64_t row_lo, row_hi;
  DynConst c;
  Span sp;
};

// limited upwind face flux with one minmod (hfb_dycore_tmem.cu face_flux_up)
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
__global__ void __launch_bounds__(kThreads, 1) k_dyn_step_ws2(Ws2Args a) {
  static_assert(!(kPhys && kRK), "column physics is not fused into RK stages");
  extern __shared__ __align__(128) double smem[];
  __shared__ uint32_t tmem_base_slot;
  double* ring = smem;
  double* ps_s = smem + kStages * kStageDoubles;  // [level][2 columns][128 threads]

  const int lane = threadIdx.x, warp = threadIdx.y;  // blockDim = (32, 8)
  const bool acoustic = warp < kPairs;
  const int pr = acoustic ? warp : warp - kPairs;  // row pair: tile rows 2pr, 2pr+1
  const int tid = warp * kTX + lane;
  const int t = pr * kTX + lane;                   // 0..127 (thread slot of a role)
  const int64_t i0 = a.sp.ilo + static_cast<int64_t>(blockIdx.x) * kTX;
  const int64_t j0 = a.sp.jlo + static_cast<int64_t>(blockIdx.y) * kRows;
  const int64_t i = i0 + lane, ja = j0 + 2 * pr, jb = ja + 1;
  const bool act_a = i <= a.sp.ihi && ja <= a.sp.jhi;
  const bool act_b = i <= a.sp.ihi && jb <= a.sp.jhi;
  const int nz = a.nz;
  const int64_t P = a.g.plane, W = a.g.pitch;
  const DynConst& c = a.c;
  const int64_t gi = i + a.sp.i0, gja = ja + a.sp.j0, gjb = jb + a.sp.j0;
  const int64_t gnx = a.sp.gnx, gny = a.sp.gny;
  const int64_t gi0 = i0 + a.sp.i0, gj0 = j0 + a.sp.j0;
  const bool interior = gi0 >= 3 && gi0 + kTX - 1 <= gnx - 2 && gj0 >= 3 &&
                        gj0 + kRows - 1 <= gny - 2 && i0 + kTX - 1 <= a.sp.ihi &&
                        j0 + kRows - 1 <= a.sp.jhi;

  if (warp == 0) sm100::tmem_alloc(&tmem_base_slot, kTmemCols);
  sm100::tmem_fence_before();
  __syncthreads();
  sm100::tmem_fence_after();
  // lane quarter of this warp; column a at TMEM columns [0, 256), b at [256, 512)
  const uint32_t tmem = tmem_base_slot + (static_cast<uint32_t>(32 * pr) << 16);

  // ---- copy chunks of this thread: 3 for everyone, a 4th for the first kExtraChunks
  const double* src[4];
  uint32_t dst[4];
  bool ok[4];
  const uint32_t ring_u32 = sm100::smem_u32(ring);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int ch = tid + q * kThreads;
    ok[q] = false;
    src[q] = a.in.p;
    dst[q] = 0;
    if (ch >= kChunks) continue;
    const int e = ch * 2;
    const double* base;
    int64_t r, cc;  // 0-based local (j', i') of the chunk start
    if (e < kOffU) {
      base = a.in.th; r = (j0 - 3) + e / kThW; cc = (i0 - 3) + e % kThW;
    } else if (e < kOffV) {
      base = a.in.u; r = (j0 - 1) + (e - kOffU) / kUW; cc = (i0 - 3) + (e - kOffU) % kUW;
    } else if (e < kOffW) {
      base = a.in.v; r = (j0 - 2) + (e - kOffV) / kVW; cc = (i0 - 1) + (e - kOffV) % kVW;
    } else if (e < kOffP) {
      base = a.in.w; r = (j0 - 1) + (e - kOffW) / kWW; cc = (i0 - 1) + (e - kOffW) % kWW;
    } else if (e < kOffRho) {
      base = a.in.p; r = (j0 - 2) + (e - kOffP) / kPW; cc = (i0 - 3) + (e - kOffP) % kPW;
    } else {
      base = a.in.rho; r = (j0 - 1) + (e - kOffRho) / kRW; cc = (i0 - 1) + (e - kOffRho) % kRW;
    }
    ok[q] = r >= -kHalo && r <= a.nj - 1 + kHalo && cc >= a.row_lo && cc + 1 <= a.row_hi;
    src[q] = base + r * W + cc;
    dst[q] = ring_u32 + static_cast<uint32_t>(e) * 8u;
  }
  uint32_t so = 0;
  constexpr uint32_t kStageBytes = kStageDoubles * 8;
  auto issue = [&](bool copy) {
    if (copy) {
#pragma unroll
      for (int q = 0; q < kFullChunks; ++q) {
        if (ok[q]) sm100::cp_async16(dst[q] + so, src[q]);
        src[q] += P;
      }
      if (warp < 6) {
        if (ok[3]) sm100::cp_async16(dst[3] + so, src[3]);
        src[3] += P;
      }
    }
    sm100::cp_async_commit();
    so = so == (kStages - 1) * kStageBytes ? 0u : so + kStageBytes;
  };

  // ---- per-thread geometry -----------------------------------------------------------
  const int64_t col_a = (ja - 1) * W + (i - 1);  // element offset of column a (b: + W)
  // running output pointers (one plane per level): acoustic u' (and v'), advection th'
  double* out_a = (acoustic ? a.out.u : a.out.th) + col_a;
  double* out_v = a.out.v + col_a;
  const bool east = gi == gnx, west = gi == 1;
  const bool north_a = gja == gny, south_a = gja == 1, north_b = gjb == gny, south_b = gjb == 1;
  const int ra = 2 * pr;                                // tile row of column a
  const int thc = (ra + 2) * kThW + (lane + 2);         // column a in a th tile
  const int uo = kOffU + ra * kUW + (lane + 2);
  const int vo = kOffV + (ra + 1) * kVW + lane;         // v(ja); v(ja-1) = -kVW, v(jb) = +kVW
  const int wo = kOffW + ra * kWW + lane;
  const int po = kOffP + (ra + 1) * kPW + (lane + 2);   // p(ja)
  const int ro = kOffRho + ra * kRW + lane;

  // ---- role state carried along K (index 0: column a, 1: column b) -------------------
  double th_prev[2] = {0.0, 0.0}, w_prev[2] = {0.0, 0.0};
  double rho_prev[2] = {0.0, 0.0}, ps_prev[2] = {0.0, 0.0};
  double cp_prev[2] = {0.0, 0.0}, dp_prev[2] = {0.0, 0.0};
  double pend_beta[2] = {0.0, 0.0}, pend_bb[2] = {1.0, 1.0}, pend_dd[2] = {0.0, 0.0};
  double fz_prev[2] = {0.0, 0.0};
  double phys_cs[2] = {0.0, 0.0}, phys_cm[2] = {0.0, 0.0}, colm_ij[2] = {0.0, 0.0},
         tsfc_ij[2] = {0.0, 0.0};
  double wb_prev[2] = {0.0, 0.0};
  struct BaseLevel {
    double th[2], u[2], uw[2], v[2], vs[2], p[2], w[2];
  };
  auto base_load = [&](int k) {
    BaseLevel b{};
    if (kRK && k < nz) {
      const int64_t o = col_a + static_cast<int64_t>(k) * P;
#pragma unroll
      for (int cI = 0; cI < 2; ++cI) {
        if (!(cI == 0 ? act_a : act_b)) continue;
        const int64_t oc = o + cI * W;
        if (acoustic) {
          b.u[cI] = __ldg(a.base.u + oc);
          b.uw[cI] = __ldg(a.base.u + oc - 1);
          b.v[cI] = __ldg(a.base.v + oc);
          b.vs[cI] = __ldg(a.base.v + oc - W);
          b.p[cI] = __ldg(a.base.p + oc);
          b.w[cI] = __ldg(a.base.w + oc);
        } else {
          b.th[cI] = __ldg(a.base.th + oc);
        }
      }
    }
    return b;
  };
  BaseLevel bcur = base_load(0);
  if (kPhys && !acoustic) {
    if (act_a) {
      colm_ij[0] = a.colm[col_a];
      tsfc_ij[0] = a.tsfc[col_a];
    }
    if (act_b) {
      colm_ij[1] = a.colm[col_a + W];
      tsfc_ij[1] = a.tsfc[col_a + W];
    }
  }
  const fp64::Recip rth0 = fp64::recip(c.th0);

  // Thomas forward recursion of face f of column cI from its pending coefficients
  auto thomas_fast = [&](int cI, int f, double& cpk, double& dpk, bool& ok, bool not_first) {
    const bool first = !not_first && f == 0;
    const double m = first ? pend_bb[cI] : pend_bb[cI] + pend_beta[cI] * cp_prev[cI];
    const double num = first ? pend_dd[cI] : pend_dd[cI] + pend_beta[cI] * dp_prev[cI];
    const fp64::Recip rm = fp64::recip(m);
    cpk = fp64::quot(-pend_beta[cI], rm, ok);
    dpk = fp64::quot(num, rm, ok);
  };
  auto thomas_div = [&](int cI, int f, double& cpk, double& dpk) {
    if (f == 0) {
      cpk = -pend_beta[cI] / pend_bb[cI];
      dpk = pend_dd[cI] / pend_bb[cI];
    } else {
      const double m = pend_bb[cI] + pend_beta[cI] * cp_prev[cI];
      cpk = -pend_beta[cI] / m;
      dpk = (pend_dd[cI] + pend_beta[cI] * dp_prev[cI]) / m;
    }
  };
  auto thomas_commit = [&](int cI, int f, double cpk, double dpk) {
    sm100::tmem_st_f64(tmem + 256 * cI + 2 * f, cpk);
    sm100::tmem_st_f64(tmem + 256 * cI + 128 + 2 * f, dpk);
    cp_prev[cI] = cpk;
    dp_prev[cI] = dpk;
  };

  int s0 = 0;
  // kMid: 3 <= k < nz - 5 (no vertical boundary cases; the copy of level k+5 exists)
  auto level = [&](int k, auto interior_tag, auto mid_tag) {
    constexpr bool kIn = decltype(interior_tag)::value;
    constexpr bool kMid = decltype(mid_tag)::value;
    const BaseLevel bnext = base_load(k + 1);
    const int kk = k + 1;
    const int s1 = s0 == kStages - 1 ? 0 : s0 + 1;
    const int s2 = s1 == kStages - 1 ? 0 : s1 + 1;
    const double* S = ring + s0 * kStageDoubles;
    const double ta = S[kOffTh + thc], tb = S[kOffTh + thc + kThW];
    const double wk[2] = {S[wo], S[wo + kWW]};
    if (acoustic) {
      if ((a.debug_skip & 2) == 0) {
        const double* Pp = S + po;
        const double p_am = Pp[-kPW], pa = Pp[0], pb = Pp[kPW], p_bp = Pp[2 * kPW];
        const double pe[2] = {Pp[1], Pp[kPW + 1]}, pw[2] = {Pp[-1], Pp[kPW - 1]};
        const double pk[2] = {pa, pb}, pn[2] = {pb, p_bp};
        const double* Up = S + uo;
        const double uu[2] = {Up[0], Up[kUW]}, uwv[2] = {Up[-1], Up[kUW - 1]};
        const double* Vp = S + vo;
        const double v_am = Vp[-kVW], v_a = Vp[0], v_b = Vp[kVW];
        const double rhok[2] = {S[ro], S[ro + kRW]};
        const double thk[2] = {ta, tb};
        // horizontally explicit PGF; v' of row a is the vs of row b (same expression)
        double unk[2], uw[2], vnk0[2], vs0[2];
#pragma unroll
        for (int cI = 0; cI < 2; ++cI) {
          unk[cI] = (kRK ? bcur.u[cI] : uu[cI]) - c.dt_rdx * (pe[cI] - pk[cI]);
          uw[cI] = (kRK ? bcur.uw[cI] : uwv[cI]) - c.dt_rdx * (pk[cI] - pw[cI]);
        }
        vnk0[0] = (kRK ? bcur.v[0] : v_a) - c.dt_rdy * (pn[0] - pk[0]);
        vnk0[1] = (kRK ? bcur.v[1] : v_b) - c.dt_rdy * (pn[1] - pk[1]);
        vs0[0] = (kRK ? bcur.vs[0] : v_am) - c.dt_rdy * (pk[0] - p_am);
        vs0[1] = vnk0[0];
        const double vnk[2] = {(!kIn && north_a) ? 0.0 : vnk0[0],
                               (!kIn && north_b) ? 0.0 : vnk0[1]};
        const double vs[2] = {(!kIn && south_a) ? 0.0 : vs0[0], (!kIn && south_b) ? 0.0 : vs0[1]};
        double psk[2];
#pragma unroll
        for (int cI = 0; cI < 2; ++cI) {
          const double un = (!kIn && east) ? 0.0 : unk[cI];
          const double uwf = (!kIn && west) ? 0.0 : uw[cI];
          psk[cI] = (kRK ? bcur.p[cI] : pk[cI]) -
                    c.dt_cs2 * (c.rdx * (un - uwf) + c.rdy * (vnk[cI] - vs[cI]));
          unk[cI] = un;
        }
        if (kIn || act_a) {
          out_a[0] = unk[0];
          out_v[0] = vnk[0];
        }
        if (kIn || act_b) {
          out_a[W] = unk[1];
          out_v[W] = vnk[1];
        }
        ps_s[(2 * k) * 128 + t] = psk[0];
        ps_s[(2 * k + 1) * 128 + t] = psk[1];
        // Thomas recursion of face k-2 next to the coefficient formation of face k-1
        bool ok = true;
        double cpk[2] = {0.0, 0.0}, dpk[2] = {0.0, 0.0}, beta[2] = {0.0, 0.0},
               dd[2] = {0.0, 0.0}, n_ps[2], n_th[2], w_rhs[2];
#pragma unroll
        for (int cI = 0; cI < 2; ++cI) {
          if (kMid || k >= 2) thomas_fast(cI, k - 2, cpk[cI], dpk[cI], ok, kMid);
          w_rhs[cI] = kRK ? wb_prev[cI] : w_prev[cI];
          n_ps[cI] = c.dt_rdz * (psk[cI] - ps_prev[cI]);
          n_th[cI] = c.dt_grav * (0.5 * (th_prev[cI] + thk[cI]) - c.th0);
          if (kMid || k >= 1) {
            const double rf = 0.5 * (rho_prev[cI] + rhok[cI]);
            const fp64::Recip rr = fp64::recip(rf);
            beta[cI] = fp64::quot(c.beta_num, rr, ok);
            dd[cI] = w_rhs[cI] - fp64::quot(n_ps[cI], rr, ok);
            dd[cI] = dd[cI] + fp64::quot(n_th[cI], rth0, ok);
          }
        }
        if (__builtin_expect(!ok, 0)) {  // a range check failed: the dialect's divisions
#pragma unroll
          for (int cI = 0; cI < 2; ++cI) {
            if (k >= 2) thomas_div(cI, k - 2, cpk[cI], dpk[cI]);
            if (k >= 1) {
              const double rf = 0.5 * (rho_prev[cI] + rhok[cI]);
              beta[cI] = c.beta_num / rf;
              dd[cI] = w_rhs[cI] - n_ps[cI] / rf;
              dd[cI] = dd[cI] + n_th[cI] / c.th0;
            }
          }
        }
#pragma unroll
        for (int cI = 0; cI < 2; ++cI) {
          if (kMid || k >= 2) thomas_commit(cI, k - 2, cpk[cI], dpk[cI]);
          if (kMid || k >= 1) {
            pend_beta[cI] = beta[cI];
            pend_bb[cI] = 1.0 + 2.0 * beta[cI];
            pend_dd[cI] = dd[cI];
          }
          rho_prev[cI] = rhok[cI];
          ps_prev[cI] = psk[cI];
          if (kRK) wb_prev[cI] = bcur.w[cI];
        }
      }
      out_v += P;
    } else if ((a.debug_skip & 1) == 0) {
      const double* T0 = S + kOffTh + thc;  // column a
      const double* T1 = ring + s1 * kStageDoubles + kOffTh + thc;
      const double* T2 = ring + s2 * kStageDoubles + kOffTh + thc;
      const double tkp1[2] = {(kMid || kk + 1 <= nz) ? T1[0] : 0.0,
                              (kMid || kk + 1 <= nz) ? T1[kThW] : 0.0};
      const double tkp2[2] = {(kMid || kk + 2 <= nz) ? T2[0] : 0.0,
                              (kMid || kk + 2 <= nz) ? T2[kThW] : 0.0};
      // y column through both rows: rows ja-2 .. jb+2
      const double y_m2 = T0[-2 * kThW], y_m1 = T0[-kThW], y_p2 = T0[2 * kThW],
                   y_p3 = T0[3 * kThW];
      const double tk[2] = {ta, tb};
      const double* Up = S + uo;
      const double uu[2] = {Up[0], Up[kUW]}, uwv[2] = {Up[-1], Up[kUW - 1]};
      const double* Vp = S + vo;
      const double v_am = Vp[-kVW], v_a = Vp[0], v_b = Vp[kVW];
      // y faces: ja-1/2, ja+1/2 (= south face of jb), jb+1/2
      const double fy_s = face_flux<!kIn>(gja - 1, gny, v_am, y_m2, y_m1, ta, tb);
      const double fy_m = face_flux<!kIn>(gja, gny, v_a, y_m1, ta, tb, y_p2);
      const double fy_n = face_flux<!kIn>(gjb, gny, v_b, ta, tb, y_p2, y_p3);
      const double fyn[2] = {fy_m, fy_n}, fys[2] = {fy_s, fy_m};
      const double vnf[2] = {(!kIn && north_a) ? 0.0 : v_a, (!kIn && north_b) ? 0.0 : v_b};
      const double vsf[2] = {(!kIn && south_a) ? 0.0 : v_am, (!kIn && south_b) ? 0.0 : v_a};
      double thv[2];
#pragma unroll
      for (int cI = 0; cI < 2; ++cI) {
        const double* Tc = T0 + cI * kThW;
        const double xm2 = Tc[-2], xm1 = Tc[-1], xp1 = Tc[1], xp2 = Tc[2];
        const double fzk = face_flux<!kMid>(kk, nz, wk[cI], th_prev[cI], tk[cI], tkp1[cI],
                                            tkp2[cI]);
        const double fxe = face_flux<!kIn>(gi, gnx, uu[cI], xm1, tk[cI], xp1, xp2);
        const double fxw = face_flux<!kIn>(gi - 1, gnx, uwv[cI], xm2, xm1, tk[cI], xp1);
        const double ue = (!kIn && east) ? 0.0 : uu[cI];
        const double uwf = (!kIn && west) ? 0.0 : uwv[cI];
        const double wt = (!kMid && kk == nz) ? 0.0 : wk[cI];
        const double wb = (!kMid && kk == 1) ? 0.0 : w_prev[cI];
        double flux = c.rdx * (fxe - fxw) + c.rdy * (fyn[cI] - fys[cI]);
        flux = flux + c.rdz * (fzk - fz_prev[cI]);
        double div = c.rdx * (ue - uwf) + c.rdy * (vnf[cI] - vsf[cI]);
        div = div + c.rdz * (wt - wb);
        double th_new = (kRK ? bcur.th[cI] : tk[cI]) - c.dt * (flux - tk[cI] * div);
        if (kPhys) {  // column_physics (dycore.h90) on the new theta of this level
          th_new = th_new - a.dt_rrelax * (th_new - colm_ij[cI]);
          const double rhok = S[ro + cI * kRW];
          if (kk == 1) {  // new u, v at the lowest level (region 5), from the plane
            const double* Pp = S + po + cI * kPW;
            const double un1 = (!kIn && east) ? 0.0 : uu[cI] - c.dt_rdx * (Pp[1] - Pp[0]);
            const double vn1 = (!kIn && (cI == 0 ? north_a : north_b))
                                   ? 0.0
                                   : (cI == 0 ? v_a : v_b) - c.dt_rdy * (Pp[kPW] - Pp[0]);
            const double wspd = sqrt(un1 * un1 + vn1 * vn1);
            th_new = th_new + a.dt_ch * wspd * (tsfc_ij[cI] - th_new) * c.rdz / rhok;
          }
          phys_cs[cI] = phys_cs[cI] + rhok * th_new;
          phys_cm[cI] = phys_cm[cI] + rhok;
        }
        thv[cI] = th_new;
        fz_prev[cI] = fzk;
      }
      if (kIn || act_a) out_a[0] = thv[0];
      if (kIn || act_b) out_a[W] = thv[1];
    }
    th_prev[0] = ta;
    th_prev[1] = tb;
    w_prev[0] = wk[0];
    w_prev[1] = wk[1];
    s0 = s1;
    out_a += P;
    bcur = bnext;
  };

  // one level: levels <= k+2 have landed, the barrier publishes them and frees the slot
  // of level k-1 for level k+kStages-1
  auto step = [&](int k, auto in_tag, auto mid_tag) {
    sm100::cp_async_wait<kStages - 4>();
    __syncthreads();
    issue(decltype(mid_tag)::value || k + kStages - 1 < nz);
    level(k, in_tag, mid_tag);
  };
  const int mid_lo = nz >= 3 ? 3 : nz, mid_hi = nz - 5 > mid_lo ? nz - 5 : mid_lo;
  auto sweep = [&](auto in_tag) {
    int k = 0;
#pragma unroll 1
    for (; k < mid_lo; ++k) step(k, in_tag, std::false_type{});
#pragma unroll 1
    for (; k < mid_hi; ++k) step(k, in_tag, std::true_type{});
#pragma unroll 1
    for (; k < nz; ++k) step(k, in_tag, std::false_type{});
  };
#pragma unroll 1
  for (int k = 0; k < kStages - 1; ++k) issue(k < nz);
  if (interior)
    sweep(std::true_type{});
  else
    sweep(std::false_type{});

  if (acoustic && nz >= 2) {  // drain the last face
#pragma unroll
    for (int cI = 0; cI < 2; ++cI) {
      bool ok = true;
      double cpk, dpk;
      thomas_fast(cI, nz - 2, cpk, dpk, ok, false);
      if (!ok) thomas_div(cI, nz - 2, cpk, dpk);
      thomas_commit(cI, nz - 2, cpk, dpk);
    }
  }
  sm100::cp_async_wait<0>();
  if (kPhys && !acoustic) {
    if (act_a) a.colm[col_a] = phys_cs[0] / phys_cm[0];
    if (act_b) a.colm[col_a + W] = phys_cs[1] / phys_cm[1];
  }

  if (acoustic) {  // back substitution + pressure update (region 7), both columns
    sm100::tmem_wait_st();
    double* wn = a.out.w + col_a + static_cast<int64_t>(nz - 1) * P;
    double* pn = a.out.p + col_a + static_cast<int64_t>(nz - 1) * P;
    if (act_a) wn[0] = 0.0;
    if (act_b) wn[W] = 0.0;
    double wk1[2] = {0.0, 0.0};
    const int nf = nz - 1;
    const double* psp = ps_s + (2 * (nz - 1)) * 128 + t;  // ps(f+1) of column a; b: +128
#pragma unroll 1
    for (int cb = (nf - 1) / 4; cb >= 0; --cb) {
      double cpv[2][4], dpv[2][4];
      sm100::tmem_ld_4f64(tmem + 8 * cb, cpv[0]);
      sm100::tmem_ld_4f64(tmem + 128 + 8 * cb, dpv[0]);
      sm100::tmem_ld_4f64(tmem + 256 + 8 * cb, cpv[1]);
      sm100::tmem_ld_4f64(tmem + 384 + 8 * cb, dpv[1]);
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        const int f = 4 * cb + q;
        if (f >= nf) continue;
        wn -= P;
        double wkk[2], pk1[2];
#pragma unroll
        for (int cI = 0; cI < 2; ++cI) {
          wkk[cI] = (f == nf - 1) ? dpv[cI][q] : dpv[cI][q] - cpv[cI][q] * wk1[cI];
          pk1[cI] = psp[cI * 128] - c.dt_cs2_rdz * (wk1[cI] - wkk[cI]);
          wk1[cI] = wkk[cI];
        }
        if (act_a) {
          wn[0] = wkk[0];
          pn[0] = pk1[0];
        }
        if (act_b) {
          wn[W] = wkk[1];
          pn[W] = pk1[1];
        }
        pn -= P;
        psp -= 2 * 128;
      }
    }
    if (act_a) pn[0] = psp[0] - c.dt_cs2_rdz * wk1[0];
    if (act_b) pn[W] = psp[128] - c.dt_cs2_rdz * wk1[1];
  }
  sm100::tmem_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem_base_slot, kTmemCols);
}

}  // namespace

cudaError_t launch_dycore_step_ws2(const DynIn& in, const DynOut& out, Grid3 g, int64_t nz,
                                   int64_t nj, const DynConst& c, const Span& sp,
                                   cudaStream_t s, const PhysArgs* phys, const DynIn* base,
                                   int debug_skip) {
  if (sp.ihi < sp.ilo || sp.jhi < sp.jlo) return cudaSuccess;
  if (!dycore_step_tmem_fits(nz)) return cudaErrorInvalidValue;
  if (phys && base) return cudaErrorInvalidValue;
  // one CTA per SM: it takes all 512 TMEM columns, so small-nz launches pad shared
  // memory past half of the SM's so that a second CTA never blocks in tcgen05.alloc
  const size_t smem = std::max<size_t>((static_cast<size_t>(kStages) * kStageDoubles +
                                        static_cast<size_t>(nz) * kCols) * sizeof(double),
                                       120 * 1024);
  const int variant = phys ? 1 : base ? 2 : 0;
  void (*kern)(Ws2Args) = variant == 1   ? k_dyn_step_ws2<true, false>
                          : variant == 2 ? k_dyn_step_ws2<false, true>
                                         : k_dyn_step_ws2<false, false>;
  {
    cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
  }
  Ws2Args a{in, out, g, static_cast<int>(nz), debug_skip,
            phys ? phys->tsfc : nullptr, phys ? phys->colm : nullptr,
            phys ? phys->dt_rrelax : 0.0, phys ? phys->dt_ch : 0.0,
            base ? *base : DynIn{}, nj, -kIOff, g.pitch - kIOff - 1, c, sp};
  dim3 block(kTX, 2 * kPairs);
  dim3 grid(static_cast<unsigned>((sp.ihi - sp.ilo + 1 + kTX - 1) / kTX),
            static_cast<unsigned>((sp.jhi - sp.jlo + 1 + kRows - 1) / kRows));
  kern<<<grid, block, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace hfb

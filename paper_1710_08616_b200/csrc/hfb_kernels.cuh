// hfb_kernels.cuh — launchers of the sm_100a kernels (internal C++ interface).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "hfb_layout.cuh"

namespace hfb {

// Tile of a launch in 1-based LOCAL coordinates plus the tile's global placement,
// so boundary predicates always test GLOBAL indices (diffusion.h90:25 tests i == nx
// on the global domain).
struct Span {
  int64_t ilo, ihi, jlo, jhi;   // inclusive, local 1-based
  int64_t i0 = 0, j0 = 0;       // global offset (global i = local i + i0)
  int64_t gnx = 0, gny = 0;     // global extents
};

// ---- relayout: caller's host order <-> device layout -------------------------
// ext/hs per role (I, J, K, L): extents and host strides in elements; the device side
// uses the Layout strides. `fast` is the role with host stride 1.
struct Relayout {
  int64_t ext[4];
  int64_t hs[4];
  int64_t ds[4];
  int fast;
};
cudaError_t launch_relayout(const double* src, double* dst, const Relayout& r, bool to_device,
                            cudaStream_t s);
// the same for one-byte element init flags (checked mode)
cudaError_t launch_relayout_u8(const uint8_t* src, uint8_t* dst, const Relayout& r,
                               bool to_device, cudaStream_t s);
// a box of device elements per role (I, J, K, L): lo (0-based), n, device strides
struct InitBox {
  int64_t lo[4], n[4], ds[4];
};
// mode 0: *flag = 1 when any element of the box is unset; mode 1: mark the box set
cudaError_t launch_init_box(uint8_t* init, const InitBox& b, int mode, int* flag,
                            cudaStream_t s);

// ---- diffusion.h90 (hfk0 + hfk1 fused: write the step result to one or two outputs)
cudaError_t launch_diffusion(const double* t_old, double* out1, double* out2, Grid3 g,
                             int64_t nz, double coef, const Span& sp, cudaStream_t s);
// the same step with shared-memory plane staging (hfb_diffusion.cu); nj = rows of the
// arrays (halo-row bounds)
cudaError_t launch_diffusion_ring(const double* t_old, double* out1, double* out2, Grid3 g,
                                  int64_t nz, int64_t nj, double coef, const Span& sp,
                                  cudaStream_t s);
// hfk1_diffuse_step alone (t_old = t_new over the span)
cudaError_t launch_copy_columns(const double* src, double* dst, Grid3 g, int64_t nz,
                                const Span& sp, cudaStream_t s);

// ---- damping.h90 ---------------------------------------------------------------
cudaError_t launch_damping(const double* ref, const double* bnd1, const double* bnd2,
                           double* damp, Grid3 g, int64_t nk, double mtratio, double tratio,
                           const Span& sp, cudaStream_t s);

// ---- bounded.h90 -----------------------------------------------------------------
cudaError_t launch_bounded(const double* a, double* b, int64_t pitch, const Span& sp,
                           cudaStream_t s);

// ---- surface flux (driver.h90 setup, surface_flux.h90 tile physics) ----------------
cudaError_t launch_sf_setup(double* cover_frac, Grid3 g, int64_t ntlm, const Span& sp,
                            cudaStream_t s);
cudaError_t launch_sf_tile(const double* cover_lt, double* flx_x, double* flx_y, double* swind,
                           int64_t pitch, const Span& sp, cudaStream_t s);

// ---- reduction.h90: deterministic two-level fp64 sum ------------------------------
// partials must hold >= reduce_partials_needed() doubles; result = total + sum.
int64_t reduce_partials_needed();
cudaError_t launch_grid_sum(const double* y, Grid3 g, int64_t nz, const Span& sp,
                            double* partials, double* result, double total, cudaStream_t s);
// ordered mode, the reference's acc-simulated order (interp.cpp:1080-1173): per-column
// partials (k in order from 0) into col[(j-jlo)*ld + (i-ilo)], then one in-order pass
cudaError_t launch_column_sums(const double* y, Grid3 g, int64_t nz, const Span& sp, double* col,
                               int64_t ld, cudaStream_t s);
cudaError_t launch_ordered_total(const double* col, int64_t n, double total, double* result,
                                 cudaStream_t s);

// ---- apps/dycore/dycore.h90 --------------------------------------------------------
struct DynConst {
  double dt, rdx, rdy, rdz, cs2, grav, th0;
  // products formed exactly as the reference evaluates them (left-associative)
  double dt_rdx, dt_rdy, dt_rdz, dt_cs2, dt_cs2_rdz, beta_num, dt_grav;
};
DynConst make_dyn_const(double dt, double rdx, double rdy, double rdz, double cs2, double grav,
                        double th0);
struct DynIn {
  const double *rho, *th, *u, *v, *w, *p;
};
struct DynOut {
  double *th, *u, *v, *w, *p;
};
cudaError_t launch_dycore_advect(const DynIn& in, double* thn, Grid3 g, int64_t nz,
                                 const DynConst& c, const Span& sp, cudaStream_t s);
// generic version: Thomas scratch dp/ps through an L2 round trip, cp in shared memory
cudaError_t launch_dycore_acoustic(const DynIn& in, const DynOut& out, Grid3 g, int64_t nz,
                                   const DynConst& c, const Span& sp, cudaStream_t s);
// sm_100a version (hfb_dycore_tmem.cu): cp.async plane ring + TMEM Thomas scratch;
// nj = rows of the arrays (for halo-row bounds); requires nz - 1 <= 64
bool dycore_acoustic_tmem_fits(int64_t nz);
cudaError_t launch_dycore_acoustic_tmem(const DynIn& in, const DynOut& out, Grid3 g,
                                        int64_t nz, int64_t nj, const DynConst& c,
                                        const Span& sp, cudaStream_t s);
// the whole timestep in one kernel (advection + acoustic), same budget
bool dycore_step_tmem_fits(int64_t nz);
bool dycore_step_ws_fits(int64_t nz);  // the product step kernel (nz - 1 <= 128)
cudaError_t launch_dycore_step_tmem(const DynIn& in, const DynOut& out, Grid3 g, int64_t nz,
                                    int64_t nj, const DynConst& c, const Span& sp,
                                    cudaStream_t s);
// column physics (dycore.h90 column_physics): surface field, previous column mean
// (updated in place), and the products dt*rrelax, dt*ch as the dialect forms them
struct PhysArgs {
  const double* tsfc;
  double* colm;
  double dt_rrelax, dt_ch;
};
// warp-specialised variant (acoustic warps + advection warps per tile); with `phys` the
// column physics is fused into the advection warps (the full timestep in one kernel)
// with `base` it is an RK stage: tendencies at `in`, applied to the base state
// Peer transport, fused: the step's outputs of the cells within `h` of a tile edge are
// also stored straight into the neighbours' next-step halo rings (their output buffers,
// mapped by CUDA IPC) — the halo exchange of the next step rides on this step's epilogue
struct RemoteHalo {
  int n;                           // neighbour directions
  int dx[8], dy[8];
  int64_t shift_i[8], shift_j[8];  // neighbour (i, j) = local (i, j) + shift
  Grid3 g[8];                      // the neighbour's layout
  double* th[8];                   // the neighbour's output buffers (origins)
  double* u[8];
  double* v[8];
  double* p[8];
  int64_t nx, ny, h;               // this tile
};
cudaError_t launch_dycore_step_ws(const DynIn& in, const DynOut& out, Grid3 g, int64_t nz,
                                  int64_t nj, const DynConst& c, const Span& sp,
                                  cudaStream_t s, const PhysArgs* phys = nullptr,
                                  const DynIn* base = nullptr,
                                  const RemoteHalo* remote = nullptr, int debug_skip = 0);
#ifndef HFB_ARITH_FMA
// the same step compiled with FMA contraction (tolerance mode, hfb_set_option "arith")
cudaError_t launch_dycore_step_ws_fma(const DynIn& in, const DynOut& out, Grid3 g, int64_t nz,
                                      int64_t nj, const DynConst& c, const Span& sp,
                                      cudaStream_t s, const PhysArgs* phys = nullptr,
                                      const DynIn* base = nullptr,
                                      const RemoteHalo* remote = nullptr, int debug_skip = 0);
#endif
#ifdef HFB_VARIANTS
// Measured-slower alternatives, compiled only into the A/B build (make variants ->
// libhfb_variants.so; selected with hfb_set_option(ctx, "variant", "tma" | "ws2")).
// debug_skip (timing experiments): 1 = no advection, 2 = no acoustic arithmetic.
// the same step fed by TMA through mbarriers (hfb_dycore_tma.cu)
cudaError_t launch_dycore_step_tma(const DynIn& in, const DynOut& out, Grid3 g, int64_t nz,
                                   int64_t nj, const DynConst& c, const Span& sp,
                                   cudaStream_t s, const PhysArgs* phys, const DynIn* base,
                                   int debug_skip);
// two columns per thread, one CTA (32 x 8 tile) per SM (hfb_dycore_ws2.cu)
cudaError_t launch_dycore_step_ws2(const DynIn& in, const DynOut& out, Grid3 g, int64_t nz,
                                   int64_t nj, const DynConst& c, const Span& sp,
                                   cudaStream_t s, const PhysArgs* phys, const DynIn* base,
                                   int debug_skip);
#endif
// standalone column physics on the current state (th updated in place)
cudaError_t launch_column_physics(const double* rho, double* th, const double* u,
                                  const double* v, Grid3 g, int64_t nz, const DynConst& c,
                                  const PhysArgs& ph, const Span& sp, cudaStream_t s);

// ---- halo pack/unpack for the 2-D decomposition -------------------------------------
// element t of a halo box {ilo, ihi, jlo, jhi} (local 1-based) x all K levels in its
// packed order (i fastest, then j, then k): the one indexing of the pack/unpack kernels
// and of their host twin
__host__ __device__ __forceinline__ int64_t box_elem(const Grid3& g, int64_t bi0, int64_t bj0,
                                                     int64_t nbi, int64_t nbj, int64_t t) {
  const int64_t ii = t % nbi, rest = t / nbi, jj = rest % nbj, k = rest / nbj;
  return g.at(bi0 - 1 + ii, bj0 - 1 + jj, k);
}
// the same pack (pack = true) / unpack on host memory (hfb_pack_box_host)
void pack_box_host(const double* field, double* buf, Grid3 g, int64_t nk, const int64_t box[4],
                   bool pack);
cudaError_t launch_pack_box(const double* field, double* buf, Grid3 g, int64_t nk,
                            const int64_t box[4], bool pack, cudaStream_t s);

// ---- launch attributes ----------------------------------------------------------------
// Opt a kernel into `smem` bytes of dynamic shared memory on the CURRENT device (the
// attribute is per device context): remembered per (device, kernel), thread-safe.
cudaError_t ensure_dynamic_smem(const void* kernel, size_t smem);

// ---- peer-memory halo transport (NVLink / NVSwitch P2P stores) -----------------------
// one box: interior cells of a local field stored straight into a neighbour's halo ring
// (the neighbour's buffer is mapped into this process by CUDA IPC); (i, j) are 1-based
// tile-local, the same k range on both sides
struct PeerBox {
  const double* src;   // local field origin
  double* dst;         // remote field origin (the neighbour's layout)
  Grid3 gs, gd;
  int64_t si0, sj0;    // first source cell
  int64_t di0, dj0;    // where it lands on the neighbour
  int64_t nbi, nbj, nk;
};
constexpr int kMaxPeerBoxes = 64;
struct PeerPush {
  PeerBox box[kMaxPeerBoxes];
  int n;
};
cudaError_t launch_peer_push(const PeerPush& p, cudaStream_t s);
// The exchange epoch lives in DEVICE memory (`epoch`, one word of the rank's own signal
// block), so a captured CUDA graph replays correct epochs: the signal kernel increments
// it and releases the new value into each remote flag (system scope, after the pushes on
// this stream); the wait kernel reads it and waits until every local flag reached it
// (acquire, system scope). With `epoch` null the epoch is the host value epoch_val.
cudaError_t launch_peer_signal(uint64_t* const* flags, int n, uint64_t* epoch, cudaStream_t s,
                               uint64_t epoch_val = 0);
cudaError_t launch_peer_wait(const uint64_t* const* flags, int n, const uint64_t* epoch,
                             cudaStream_t s, uint64_t epoch_val = 0);
// deterministic all-reduce of one double over n ranks through peer memory: my value goes
// to slot [parity][rank] of every rank, then every rank sums slots 0..n-1 in rank order
struct PeerReduce {
  double* value;               // in: this rank's partial; out: the total
  double* slots[64];           // every rank's slot array (remote, or local for self)
  uint64_t* flags[64];         // every rank's reduction flag array
  double* my_slots;            // this rank's slot array
  uint64_t* my_flags;          // this rank's reduction flags
  int n, rank;
  uint64_t epoch;
};
cudaError_t launch_peer_allreduce(const PeerReduce& r, cudaStream_t s);

// ---- apps/dycore/asuca.h90 (hfb_asuca.cu): the ASUCA time scheme ------------------
struct AsuState {
  const double *rho, *th, *u, *v, *w, *p;
};
struct AsuTend {
  double *frho, *fth, *fu, *fv, *fw;
};
// one RK2 acoustic pass of step h (dtau/2 or dtau), products formed as the dialect
// evaluates them (left-associative)
struct AsuAcoConst {
  double h, rdx, rdy, th0;
  double h_rdx, h_rdy, h_rdz, h_cs2, h_cs2_rdz, beta_num, h_grav;
  double dtau_rdmp, rnbnd, rnzd;
  int64_t nbnd, kdmp;
};
AsuAcoConst make_asu_aco_const(double h, double dtau, double rdx, double rdy, double rdz,
                               double cs2, double grav, double th0, double rdmp, int64_t nbnd,
                               int64_t kdmp, double rnbnd, double rnzd);
bool asuca_fits(int64_t nz);
// slow tendencies at the stage state (rho, th, u, v, w; p unused)
cudaError_t launch_asu_tend(const AsuState& s, const AsuTend& f, Grid3 g, int64_t nz, int64_t nj,
                            double rdx, double rdy, double rdz, const Span& sp, cudaStream_t st);
// pass A (pass_b false): pa_out = the RK2 midpoint pressure; pass B: un, vn, wn (damped),
// pn from the state s (u, v, w, p current; rho, th of the stage) and the midpoint pa
cudaError_t launch_asu_acoustic(bool pass_b, const AsuState& s, const double* fu,
                                const double* fv, const double* fw, const double* pa,
                                double* pa_out, double* un, double* vn, double* wn, double* pn,
                                Grid3 g, int64_t nz, int64_t nj, const AsuAcoConst& c,
                                const Span& sp, cudaStream_t st);
cudaError_t launch_asu_stage_end(const double* thb, const double* fth, const double* rhob,
                                 const double* frho, double* th, double* rho, Grid3 g,
                                 int64_t nz, double dtf, const Span& sp, cudaStream_t st);

}  // namespace hfb

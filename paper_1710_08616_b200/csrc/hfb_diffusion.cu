// hfb_diffusion.cu — the reference's 7-point diffusion step (diffusion.h90:23-41, hfk0 +
// the fused-away hfk1 copy) with shared-memory plane staging.
//
// A CTA owns a 32 x 16 tile of (i,j) columns and marches K. Each K-plane of t_old the tile
// needs (the tile plus its one-cell ring, rows j0-1..j0+16, 36 columns from the even
// column at or left of i0-1 so the 16-B copy chunks stay aligned for any span start) is
// staged by LDGSTS into a kStages-deep ring; the
// vertical neighbours ride in registers (k-1, k rotate; k+1 is the next plane's centre).
// Every input value is read from DRAM once per step (the ring overlap between
// neighbouring tiles is served by L2), every output written once: 16 B per grid point,
// 24 B when both t_old and t_new are materialised (the per-step entry).
//
// Arithmetic exactly as the dialect writes it, left to right, no FMA:
//   s = t(k-1) + t(k+1); s = s + t(i-1); s = s + t(i+1); s = s + t(j-1); s = s + t(j+1);
//   s = s - 6*t; t_new = t + coef*s   (Dirichlet copy on the GLOBAL boundary).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "hfb_kernels.cuh"
#include "hfb_sm100.cuh"

namespace hfb {

namespace {

constexpr int kTX = 32, kTY = 16, kThreads = kTX * kTY;  // 32x16: 32x8 was 1.9% slower
constexpr int kPW = kTX + 4, kPR = kTY + 2;  // plane tile 36 x 18
constexpr int kPlane = kPW * kPR;            // 648 doubles
constexpr int kChunks = kPlane / 2;          // 324 16-B chunks (one per thread)
constexpr int kStages = 6;

struct RingArgs {
  const double* src;
  double* o1;
  double* o2;
  Grid3 g;
  int nz, kchunk;
  double coef;
  int64_t nj, row_lo, row_hi;
  Span sp;
};

__global__ void __launch_bounds__(kThreads, 2) k_diffusion_ring(RingArgs a) {
  __shared__ __align__(16) double ring[kStages * kPlane];
  const int lane = threadIdx.x, row = threadIdx.y, tid = row * kTX + lane;
  const int64_t i0 = a.sp.ilo + static_cast<int64_t>(blockIdx.x) * kTX;  // 1-based local
  const int64_t j0 = a.sp.jlo + static_cast<int64_t>(blockIdx.y) * kTY;
  const int64_t i = i0 + lane, j = j0 + row;
  const bool active = i <= a.sp.ihi && j <= a.sp.jhi;
  const int nz = a.nz;
  const int kb = 1 + static_cast<int>(blockIdx.z) * a.kchunk;  // this CTA's levels
  const int ke = min(nz, kb + a.kchunk - 1);
  const int64_t P = a.g.plane, W = a.g.pitch;
  const int64_t gi = i + a.sp.i0, gj = j + a.sp.j0;
  const bool hb = (gi == 1) | (gi == a.sp.gnx) | (gj == 1) | (gj == a.sp.gny);
  const double coef = a.coef;

  // the plane tile starts at the even 0-based column at or left of the west neighbour
  // (i0 - 2, 0-based), so every 16-B chunk is aligned for any span start
  const int64_t cs = ((i0 - 2) % 2 == 0) ? i0 - 2 : i0 - 3;
  const int shift = static_cast<int>((i0 - 2) - cs);  // 0 or 1
  // this thread's copy chunk of a plane (chunk tid; threads >= kChunks copy nothing)
  bool ok = false;
  const double* src = a.src;
  uint32_t dst = 0;
  if (tid < kChunks) {
    const int e = tid * 2;
    const int64_t r = (j0 - 2) + e / kPW, cc = cs + e % kPW;  // 0-based local
    ok = r >= -kHalo && r <= a.nj - 1 + kHalo && cc >= a.row_lo && cc + 1 <= a.row_hi;
    src = a.src + r * W + cc;
    dst = sm100::smem_u32(ring) + static_cast<uint32_t>(e) * 8u;
  }
  // planes kb-1 .. ke+1 in order, one commit group each (planes outside 1..nz are empty
  // groups), plane k into slot (k - kb + 1) % kStages
  const int klast = min(nz, ke + 1);
  int issued = kb - 1;
  auto issue = [&]() {
    if (issued >= 1 && issued <= klast && ok) {
      const uint32_t so =
          static_cast<uint32_t>(((issued - kb + 1) % kStages) * kPlane * 8);
      sm100::cp_async16(dst + so, src + static_cast<int64_t>(issued - 1) * P);
    }
    sm100::cp_async_commit();
    ++issued;
  };
#pragma unroll 1
  for (int q = 0; q < kStages; ++q) issue();

  const int c0 = (row + 1) * kPW + (lane + 1 + shift);  // this column in a plane tile
  auto plane = [&](int k) { return ring + ((k - kb + 1) % kStages) * kPlane; };
  const int64_t col = (j - 1) * W + (i - 1);
  double* o1 = a.o1 + col;
  double* o2 = a.o2 ? a.o2 + col : nullptr;

  // levels k-1 and k of this column, carried in registers
  double tkm = 0.0, tk = 0.0;
  if (kb > 1) {  // plane kb-1 (the first group)
    sm100::cp_async_wait<kStages - 1>();
    __syncthreads();
    tkm = plane(kb - 1)[c0];
  }
#pragma unroll 1
  for (int k = kb; k <= ke; ++k) {
    // planes <= k+1 have landed (own copies), everyone's after the barrier; the slot of
    // plane k-1 (finished by every thread) then takes plane k + kStages - 1
    sm100::cp_async_wait<kStages - 3>();
    __syncthreads();
    issue();
    const double* Pk = plane(k);
    if (k == kb) tk = Pk[c0];
    const double tkp = (k < nz) ? plane(k + 1)[c0] : 0.0;
    double out;
    if (hb || k == 1 || k == nz) {
      out = tk;
    } else {
      double s = tkm + tkp;
      s = s + Pk[c0 - 1];
      s = s + Pk[c0 + 1];
      s = s + Pk[c0 - kPW];
      s = s + Pk[c0 + kPW];
      s = s - 6.0 * tk;
      out = tk + coef * s;
    }
    if (active) {
      const int64_t off = static_cast<int64_t>(k - 1) * P;
      o1[off] = out;
      if (o2) o2[off] = out;
    }
    tkm = tk;
    tk = tkp;
  }
  sm100::cp_async_wait<0>();
}

}  // namespace

cudaError_t launch_diffusion_ring(const double* t_old, double* out1, double* out2, Grid3 g,
                                  int64_t nz, int64_t nj, double coef, const Span& sp,
                                  cudaStream_t s) {
  if (sp.ihi < sp.ilo || sp.jhi < sp.jlo || nz <= 0) return cudaSuccess;
  const int64_t tiles = ((sp.ihi - sp.ilo + 1 + kTX - 1) / kTX) *
                        ((sp.jhi - sp.jlo + 1 + kTY - 1) / kTY);
  // small grids: split K until two waves of resident CTAs exist (each chunk re-reads two
  // planes, so no more splitting than that); residency from the occupancy calculator
  static const int resident = [] {
    int n = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &n, reinterpret_cast<const void*>(k_diffusion_ring), kTX * kTY, 0) != cudaSuccess ||
        n < 1)
      n = 1;
    return n * sms;
  }();
  int kchunks = 1;
  while (tiles * kchunks < 2 * resident && nz / (kchunks * 2) >= 8) kchunks *= 2;
  const int kchunk = static_cast<int>((nz + kchunks - 1) / kchunks);
  kchunks = static_cast<int>((nz + kchunk - 1) / kchunk);
  RingArgs a{t_old, out1, out2, g, static_cast<int>(nz), kchunk, coef, nj,
             -kIOff, g.pitch - kIOff - 1, sp};
  dim3 block(kTX, kTY);
  dim3 grid(static_cast<unsigned>((sp.ihi - sp.ilo + 1 + kTX - 1) / kTX),
            static_cast<unsigned>((sp.jhi - sp.jlo + 1 + kTY - 1) / kTY),
            static_cast<unsigned>(kchunks));
  k_diffusion_ring<<<grid, block, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace hfb

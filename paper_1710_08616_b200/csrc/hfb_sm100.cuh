// hfb_sm100.cuh — thin inline-PTX wrappers for the sm_100a features the kernels use:
// LDGSTS (cp.async) multi-stage staging of K-planes into shared memory, and TMEM
// (tcgen05.alloc / st / ld) as per-thread scratch for the column solvers.
//
// TMEM is 128 lanes x 512 columns x 32 bit per SM. With a 128-thread CTA, warp w owns
// lanes [32w, 32w+32) and thread (w, lane) owns lane 32w+lane: a private row of up to
// 512 x 4 B that no other thread touches — a per-thread stack the size of a column's
// Thomas coefficients, outside shared memory and the register file.
#pragma once
#include <cstdint>

namespace hfb {
namespace sm100 {

// The warp index as a value the compiler knows to be warp-uniform (shuffled from lane 0):
// branches on it are uniform, and values derived from it (TMA box coordinates, ring
// offsets) live in uniform registers, so a TMA issue needs no per-lane waterfall loop
// (ELECT / R2UR.BROADCAST / BRA.U.ANY) around UTMALDG.
__device__ __forceinline__ int warp_uniform(int v) { return __shfl_sync(0xffffffffu, v, 0); }
// one elected lane of a converged warp (elect.sync)
__device__ __forceinline__ bool elect_one() {
  uint32_t e = 0;
  asm volatile(
      "{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(e));
  return e != 0;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- cp.async (LDGSTS): 16-byte global -> shared copies, L1 bypass -----------------
__device__ __forceinline__ void cp_async16(uint32_t dst_smem, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst_smem), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---- TMEM ------------------------------------------------------------------------
// Allocate `ncols` (power of two >= 32) columns; executed by one full warp. The base
// address is written to shared memory.
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// one fp64 value per thread into its lane, columns [col, col+2)
__device__ __forceinline__ void tmem_st_f64(uint32_t taddr, double v) {
  const uint32_t lo = static_cast<uint32_t>(__double2loint(v));
  const uint32_t hi = static_cast<uint32_t>(__double2hiint(v));
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(taddr), "r"(lo),
               "r"(hi)
               : "memory");
}
// four fp64 values per thread from its lane, columns [col, col+8)
__device__ __forceinline__ void tmem_ld_4f64(uint32_t taddr, double (&out)[4]) {
  uint32_t r[8];
  // load and wait in ONE asm statement so no use of r[] can be scheduled before the wait
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int q = 0; q < 4; ++q)
    out[q] = __hiloint2double(static_cast<int>(r[2 * q + 1]), static_cast<int>(r[2 * q]));
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

// ---- mbarrier (shared::cta) --------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
// make the initialised barriers visible to the async (TMA) proxy
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(bar), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// per-slot arrival counter in shared memory: returns the count before this arrival
// (acq_rel: the caller's earlier reads of the slot are ordered before it, and the last
// arriver sees everyone's)
__device__ __forceinline__ uint32_t smem_count_arrival(uint32_t* cnt) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;\n"
               : "=r"(old)
               : "r"(smem_u32(cnt))
               : "memory");
  return old;
}
// order this thread's generic-proxy shared-memory accesses before later async-proxy
// (TMA) ones
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// ---- TMA: 3-D tiled tensor load into shared memory, completion on an mbarrier -------
__device__ __forceinline__ void tma_load_3d(uint32_t dst_smem, const void* tmap, uint32_t bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst_smem),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}
// TMA box prefetch into L2 only (no shared memory, no completion to track)
__device__ __forceinline__ void tma_prefetch_l2_3d(const void* tmap, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

}  // namespace sm100
}  // namespace hfb

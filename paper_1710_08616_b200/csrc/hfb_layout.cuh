// hfb_layout.cuh — compile-time GPU storage order for Hybrid-Fortran module arrays.
//
// Replaces the reference's storage-order abstraction (macro.hpp:13-41: MacroTable
// ordering families; macro.cpp:210-302: AT(...)/DOM(...) access and declaration
// rewriting). The reference permutes subscripts textually per target; here every
// module array of an app gets ONE device order, fixed at compile time:
//
//   I fastest (coalesced across the threads of a warp, one thread per (i,j) column),
//   then J, then K (the sequential K-march), then an optional trailing dim L.
//
//   addr(i', j', k', l') = origin + l'*volume + k'*plane + j'*pitch + i'
//
// with i', j', k', l' 0-based offsets from the declared lower bounds. Every row
// carries kIOff = 16 elements (128 B) in front, so the interior of every row starts
// 128-B aligned; a halo ring of kHalo cells exists in I and J on every array (halo
// cells are read by stencils and filled by the multi-GPU exchange; they are never
// part of the logical array). pitch is a multiple of 16 elements (128 B).
#pragma once
#include <cstdint>

namespace hfb {

constexpr int kHalo = 2;       // widest stencil radius on the path (limited advection)
constexpr int kIOff = 16;      // elements before i' = 0 in every row (128 B)
constexpr int kAlignElems = 16;

enum Role : int { kRoleI = 0, kRoleJ = 1, kRoleK = 2, kRoleL = 3 };

struct Layout {
  int64_t ni = 1, nj = 1, nk = 1, nl = 1;  // logical extents per role
  int64_t pitch = 0, plane = 0, volume = 0;
  int64_t alloc_elems = 0;                 // total allocation
  int64_t origin_off = 0;                  // origin - base (elements)

  static Layout make(int64_t ni, int64_t nj, int64_t nk, int64_t nl) {
    Layout L;
    L.ni = ni;
    L.nj = nj;
    L.nk = nk;
    L.nl = nl;
    int64_t row = kIOff + ni + kHalo;
    L.pitch = (row + kAlignElems - 1) / kAlignElems * kAlignElems;
    L.plane = (nj + 2 * kHalo) * L.pitch;
    L.volume = nk * L.plane;
    L.alloc_elems = nl * L.volume;
    L.origin_off = kHalo * L.pitch + kIOff;
    return L;
  }
};

// Scalar index helper used by every kernel: 0-based (i', j', k').
struct Grid3 {
  int64_t pitch, plane;
  __host__ __device__ __forceinline__ int64_t at(int64_t i, int64_t j, int64_t k) const {
    return k * plane + j * pitch + i;
  }
};

}  // namespace hfb

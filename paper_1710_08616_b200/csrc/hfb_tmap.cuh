// hfb_tmap.cuh — TMA tensor maps over device arrays in the hfb layout (hfb_layout.cuh).
#pragma once
#include <cuda.h>

#include <cstdint>

#include "hfb_layout.cuh"

namespace hfb {

// 3-D map (i, j, k) over a whole device array allocation (pitch x (nj + 2 halo rows) x
// nk elements, fp64), box (bw, bh, 1); `origin` is the array's interior origin
// (Slot::d()). Box coordinates are allocation coordinates: x = kIOff + i', y = kHalo + j'
// (i', j' 0-based local), z = k'. Cells outside the allocation are zero-filled.
bool make_box_map(CUtensorMap* m, const double* origin, Grid3 g, int64_t nj, int64_t nk, int bw,
                  int bh);

// the six plane boxes of one level of the fused dycore step, in DynIn field order of the
// ring (th, u, v, w, p, rho)
struct StepMaps {
  CUtensorMap m[6];
  CUtensorMap base[5];  // RK stages: the base state's th, u, v, w, p (L2 prefetch boxes)
};

}  // namespace hfb

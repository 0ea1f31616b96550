"""B200-native timestep engine for Hybrid-Fortran grid programs (arXiv 1710.08616).

The product is libhfb.so (CUDA sm_100a kernels + the C ABI of include/hfb.h);
this package is the Python host mirror of the reference executor's interface.
"""
from .runtime import (EXPORTS, Engine, Group, HfbError, LaunchStats, MODULES, build, decomp_faces,
                      decomp_init, lib, run_gpu, variants_build, TileLayout)

__all__ = ["Engine", "Group", "HfbError", "LaunchStats", "MODULES", "EXPORTS", "build", "lib", "run_gpu",
           "decomp_init", "decomp_faces", "variants_build", "TileLayout"]

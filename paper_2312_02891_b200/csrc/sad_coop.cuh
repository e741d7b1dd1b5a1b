// sad_coop.cuh -- launchers of the cooperative persistent GMRES kernel.
//
// The kernel is instantiated for 10 (vector type, value type, shift, flexible)
// variants x 8 block widths; each variant lives in its own translation unit
// (sad_coop.cu compiled once per -DSAD_COOP_VARIANT) so the library builds in
// parallel.  sad_capi.cu only sees these declarations.
#pragma once

#include <cuda_runtime.h>

#include "sad_persistent.cuh"

namespace sad {

struct CoopCfg {
  int nsm;                   // SMs of the device
  int max_sms;               // cap (0 = all)
  int min_elems_per_thread;  // grid sizing
  int max_blocks;            // partial-sum capacity (also the partial stride)
};

// variant tags: d = fp64 blocks / real values, z = complex128 blocks / real
// values, zc = complex128 blocks / complex values; s1 = identity-mass shift in
// the epilogue; f1 = flexible (stores Z).
#define SAD_COOP_VARIANTS(X)                                   \
  X(d_s0_f0, double, double, false, false)                     \
  X(d_s0_f1, double, double, false, true)                      \
  X(d_s1_f0, double, double, true, false)                      \
  X(d_s1_f1, double, double, true, true)                       \
  X(z_s0_f0, double2, double, false, false)                    \
  X(z_s0_f1, double2, double, false, true)                     \
  X(z_s1_f0, double2, double, true, false)                     \
  X(z_s1_f1, double2, double, true, true)                      \
  X(zc_s0_f0, double2, double2, false, false)                  \
  X(zc_s0_f1, double2, double2, false, true)

#define SAD_COOP_DECL(tag, XT, VT, SIGMA, FLEX)                                             \
  cudaError_t coop_launch_##tag(int R, PArgs<XT> a, const CoopCfg& cfg, cudaStream_t s,    \
                                size_t smem, int* grid_out);
SAD_COOP_VARIANTS(SAD_COOP_DECL)
#undef SAD_COOP_DECL

}  // namespace sad

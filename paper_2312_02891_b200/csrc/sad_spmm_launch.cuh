// sad_spmm_launch.cuh -- host-side dispatch of the stand-alone shifted SpMM
// kernels (apply / residual / the multi-kernel engine's Arnoldi and cycle-end
// SpMMs).  Instantiated in sad_spmm_launch.cu, compiled in parts by _build.py.
#pragma once

#include <cuda_runtime.h>

#include "sad_kernels.cuh"

namespace sad {

void count_launches(long long k);   // defined in sad_capi.cu
extern int g_spmm_bulk_sms;         // SMs for the persistent-style SpMM grids (sad_capi.cu)

// Returns 0, or 1 for an unsupported block width.
template <typename XT, int MODE>
int launch_spmm(const SpmmArgs<XT>& a, int R, bool vc, bool pre, bool sigma, int nsm,
                cudaStream_t s, int grid_cap = 0);

extern template int launch_spmm<double, SPMM_APPLY>(const SpmmArgs<double>&, int, bool, bool, bool, int, cudaStream_t, int);
extern template int launch_spmm<double, SPMM_RESID>(const SpmmArgs<double>&, int, bool, bool, bool, int, cudaStream_t, int);
extern template int launch_spmm<double, SPMM_RESID_CYCLE>(const SpmmArgs<double>&, int, bool, bool, bool, int, cudaStream_t, int);
extern template int launch_spmm<double, SPMM_ARNOLDI>(const SpmmArgs<double>&, int, bool, bool, bool, int, cudaStream_t, int);
extern template int launch_spmm<double2, SPMM_APPLY>(const SpmmArgs<double2>&, int, bool, bool, bool, int, cudaStream_t, int);
extern template int launch_spmm<double2, SPMM_RESID>(const SpmmArgs<double2>&, int, bool, bool, bool, int, cudaStream_t, int);
extern template int launch_spmm<double2, SPMM_RESID_CYCLE>(const SpmmArgs<double2>&, int, bool, bool, bool, int, cudaStream_t, int);
extern template int launch_spmm<double2, SPMM_ARNOLDI>(const SpmmArgs<double2>&, int, bool, bool, bool, int, cudaStream_t, int);

}  // namespace sad

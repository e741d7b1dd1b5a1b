// sad_spmm_launch.cu -- SpMM dispatch (see sad_spmm_launch.cuh).  Compiled
// once per -DSAD_SPMM_PART=<0..3> so the instantiations build in parallel:
//   0: fp64 apply/residual   1: complex128 apply/residual
//   2: fp64 Arnoldi/cycle    3: complex128 Arnoldi/cycle
#include <algorithm>
#include <type_traits>

#include "sad_spmm_launch.cuh"
#include "sad_spmm_bulk.cuh"

#ifndef SAD_SPMM_PART
#error "compile with -DSAD_SPMM_PART=<0..3>"
#endif

namespace sad {


static int grid_for(long long work, int per_block, int cap) {
  long long g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// -----------------------------------------------------------------------------
// SpMM dispatch
// -----------------------------------------------------------------------------
template <typename XT, typename VT, int R, int MODE, bool PRE, bool SIGMA>
static void launch_spmm_t(const SpmmArgs<XT>& a, int grid, cudaStream_t s) {
  if constexpr (MODE == SPMM_APPLY || MODE == SPMM_RESID || MODE == SPMM_ARNOLDI) {
    // TMA-staged SpMM; grid = resident blocks (persistent over row tiles)
    auto kern = k_spmm_bulk<XT, VT, R, MODE, PRE, SIGMA>;
    constexpr size_t smem = bulk_smem_bytes<VT, R>();
    static int nb = -1;
    if (nb < 0) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kThreads + 32, smem);
      if (nb < 1) nb = 1;
    }
    const long long tiles = (a.n + BulkTile<R>::TR - 1) / BulkTile<R>::TR;
    const int g = (int)std::max(1LL, std::min(tiles, (long long)nb * g_spmm_bulk_sms));
    kern<<<g, kThreads + 32, smem, s>>>(a);
    count_launches(1);
  } else {
    k_spmm<XT, VT, R, MODE, PRE, SIGMA><<<grid, kThreads, 0, s>>>(a);
    count_launches(1);
  }
}

template <typename XT, typename VT, int R, int MODE>
static void launch_spmm_ps(const SpmmArgs<XT>& a, bool pre, bool sigma, int grid, cudaStream_t s) {
  if (pre) {
    if (sigma) launch_spmm_t<XT, VT, R, MODE, true, true>(a, grid, s);
    else launch_spmm_t<XT, VT, R, MODE, true, false>(a, grid, s);
  } else {
    if (sigma) launch_spmm_t<XT, VT, R, MODE, false, true>(a, grid, s);
    else launch_spmm_t<XT, VT, R, MODE, false, false>(a, grid, s);
  }
}

template <typename XT, int R, int MODE>
static void launch_spmm_v(const SpmmArgs<XT>& a, bool vc, bool pre, bool sigma, int grid,
                          cudaStream_t s);
template <int R, int MODE>
struct SpmmV {
  static void run(const SpmmArgs<double>& a, bool, bool pre, bool sigma, int grid, cudaStream_t s) {
    launch_spmm_ps<double, double, R, MODE>(a, pre, sigma, grid, s);
  }
  static void run(const SpmmArgs<double2>& a, bool vc, bool pre, bool sigma, int grid,
                  cudaStream_t s) {
    if (vc) launch_spmm_ps<double2, double2, R, MODE>(a, pre, false, grid, s);
    else launch_spmm_ps<double2, double, R, MODE>(a, pre, sigma, grid, s);
  }
};


// A real block with an even number of columns is processed as a complex block
// of R/2 columns (16-byte loads, half the lanes per row): for a real matrix and
// a real shift every complex product reduces to the same two real FMAs, so
// the results are identical.
static bool spmm_pairs(const SpmmArgs<double>& a, int R, bool pre, bool sigma, int nsm,
                       cudaStream_t s, int mode) {
  if (R % 2 || pre || a.sigma.y != 0.0) return false;
  SpmmArgs<double2> z{};
  z.n = a.n; z.rowptr = a.rowptr; z.colidx = a.colidx; z.vals = a.vals;
  z.x = reinterpret_cast<const double2*>(a.x);
  z.y = reinterpret_cast<double2*>(a.y);
  z.b = reinterpret_cast<const double2*>(a.b);
  z.sigma = a.sigma;
  z.row0 = a.row0;
  if (mode == SPMM_APPLY) launch_spmm<double2, SPMM_APPLY>(z, R / 2, false, false, sigma, nsm, s);
  else launch_spmm<double2, SPMM_RESID>(z, R / 2, false, false, sigma, nsm, s);
  return true;
}

template <typename XT, int MODE>
int launch_spmm(const SpmmArgs<XT>& a, int R, bool vc, bool pre, bool sigma, int nsm,
                cudaStream_t s, int grid_cap) {
  if constexpr (std::is_same<XT, double>::value && (MODE == SPMM_APPLY || MODE == SPMM_RESID)) {
    if (spmm_pairs(a, R, pre, sigma, nsm, s, MODE)) return 0;
  }
  const int gpw = 32 / R;
  const int cap = grid_cap > 0 ? grid_cap : nsm * 8;
  const int grid = grid_for(a.n, kWarps * gpw, cap);
  switch (R) {
    case 1: SpmmV<1, MODE>::run(a, vc, pre, sigma, grid, s); break;
    case 2: SpmmV<2, MODE>::run(a, vc, pre, sigma, grid, s); break;
    case 3: SpmmV<3, MODE>::run(a, vc, pre, sigma, grid, s); break;
    case 4: SpmmV<4, MODE>::run(a, vc, pre, sigma, grid, s); break;
    case 5: SpmmV<5, MODE>::run(a, vc, pre, sigma, grid, s); break;
    case 6: SpmmV<6, MODE>::run(a, vc, pre, sigma, grid, s); break;
    case 7: SpmmV<7, MODE>::run(a, vc, pre, sigma, grid, s); break;
    case 8: SpmmV<8, MODE>::run(a, vc, pre, sigma, grid, s); break;
    default: return 1;
  }
  return 0;
}


#if SAD_SPMM_PART == 0
template int launch_spmm<double, SPMM_APPLY>(const SpmmArgs<double>&, int, bool, bool, bool, int, cudaStream_t, int);
template int launch_spmm<double, SPMM_RESID>(const SpmmArgs<double>&, int, bool, bool, bool, int, cudaStream_t, int);
#elif SAD_SPMM_PART == 1
template int launch_spmm<double2, SPMM_APPLY>(const SpmmArgs<double2>&, int, bool, bool, bool, int, cudaStream_t, int);
template int launch_spmm<double2, SPMM_RESID>(const SpmmArgs<double2>&, int, bool, bool, bool, int, cudaStream_t, int);
#elif SAD_SPMM_PART == 2
template int launch_spmm<double, SPMM_RESID_CYCLE>(const SpmmArgs<double>&, int, bool, bool, bool, int, cudaStream_t, int);
template int launch_spmm<double, SPMM_ARNOLDI>(const SpmmArgs<double>&, int, bool, bool, bool, int, cudaStream_t, int);
#else
template int launch_spmm<double2, SPMM_RESID_CYCLE>(const SpmmArgs<double2>&, int, bool, bool, bool, int, cudaStream_t, int);
template int launch_spmm<double2, SPMM_ARNOLDI>(const SpmmArgs<double2>&, int, bool, bool, bool, int, cudaStream_t, int);
#endif

}  // namespace sad

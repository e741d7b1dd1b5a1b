// sad_spmm_launch.cu -- SpMM dispatch (see sad_spmm_launch.cuh).  Compiled
// once per -DSAD_SPMM_PART=<0..3> so the instantiations build in parallel:
//   0: fp64 apply/residual   1: complex128 apply/residual
//   2: fp64 Arnoldi/cycle    3: complex128 Arnoldi/cycle
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "sad_spmm_launch.cuh"
#include "sad_spmm_bulk.cuh"
#include "sad_spmm_band.cuh"

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
static size_t al128(size_t b) { return (b + 127) & ~size_t(127); }

// Banded plan: stage layout and pipeline depth for this block type; false when
// two stages do not fit (the CSR kernel runs instead)
template <typename XT, typename VT, int R, bool PRE, bool PAIR = false>
static bool band_config(int xcap, int wmax, int tr, bool one_block, BandCfg& cfg, size_t& smem) {
  const size_t xb = al128(32 + (size_t)xcap * R * sizeof(XT));
  const size_t db = PRE ? al128(32 + (size_t)xcap * (PAIR ? 8 : sizeof(XT))) : 0;
  const size_t vb = al128((size_t)wmax * tr * (sizeof(VT) + 2));   // values + indices
  const size_t sb = xb + db + vb;
  int S = one_block ? 0 : (int)std::min<size_t>(6, (110 * 1024) / sb);   // two blocks per SM
  if (S < 3) S = (int)std::min<size_t>(6, (212 * 1024) / sb);            // one block per SM
  if (S < 2) return false;
  cfg.S = S;
  cfg.SB = (unsigned)sb;
  cfg.offD = (unsigned)xb;
  cfg.offV = (unsigned)(xb + db);
  smem = (size_t)S * sb;
  return true;
}

template <typename XT, typename VT, int R, int MODE, bool PRE, bool SIGMA, int U, bool PAIR = false>
static bool launch_band_u(const SpmmArgs<XT>& a, cudaStream_t s);

template <typename XT, typename VT, int R, int MODE, bool PRE, bool SIGMA>
static bool launch_band(const SpmmArgs<XT>& a, cudaStream_t s) {
  if (!a.band_meta || a.row0 != 0) return false;
  // 16 consumer warps (U = 4, one block per SM) when a tile holds two rows per lane group
  // of 16 warps (config 4: 256-row tiles); tiles of 16 warps x ONE row are slower than 8
  // warps x two rows (config 5, 128-row tiles: 516 vs 449 us)
  if (a.band_tr >= 2 * 16 * (32 / R)) return launch_band_u<XT, VT, R, MODE, PRE, SIGMA, 4>(a, s);
  return launch_band_u<XT, VT, R, MODE, PRE, SIGMA, 2>(a, s);
}

template <typename XT, typename VT, int R, int MODE, bool PRE, bool SIGMA, int U, bool PAIR>
static bool launch_band_u(const SpmmArgs<XT>& a, cudaStream_t s) {
  // TMA sources must be 16-byte aligned up to the parity rule of the plan
  const XT* xsrc = a.x;
  if ((reinterpret_cast<uintptr_t>(xsrc) & 15) || (reinterpret_cast<uintptr_t>(a.dinv) & 15)) return false;
  if (MODE == SPMM_ARNOLDI && ((size_t)a.stride * sizeof(XT)) % 16) return false;
  BandCfg cfg{};
  size_t smem = 0;
  if (!band_config<XT, VT, R, PRE, PAIR>(a.band_xcap, a.band_wmax, a.band_tr, U >= 4, cfg, smem)) return false;
  auto kern = k_spmm_band<XT, VT, R, MODE, PRE, SIGMA, U, PAIR>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 216 * 1024);
    attr = true;
  }
  // per host thread: the A- and B-side solves may launch from two threads
  static thread_local size_t nb_smem = 0;
  static thread_local int nb = 0;
  if (nb_smem != smem) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, (band_consumer_warps<U>() + 1) * 32, smem);
    nb_smem = smem;
  }
  if (nb < 1) return false;
  const long long tiles = (a.n + a.band_tr - 1) / a.band_tr;
  const int g = (int)std::max(1LL, std::min(tiles, (long long)nb * g_spmm_bulk_sms));
  kern<<<g, (band_consumer_warps<U>() + 1) * 32, smem, s>>>(a, cfg);
  count_launches(1);
  return true;
}

template <typename XT, typename VT, int R, int MODE, bool PRE, bool SIGMA>
static void launch_spmm_t(const SpmmArgs<XT>& a, int grid, cudaStream_t s) {
  if constexpr (MODE == SPMM_APPLY || MODE == SPMM_RESID || MODE == SPMM_ARNOLDI) {
    if (launch_band<XT, VT, R, MODE, PRE, SIGMA>(a, s)) return;
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
  z.band_meta = a.band_meta; z.band_seg = a.band_seg; z.band_dinv = a.band_dinv;
  z.band_xstride = a.band_xstride;
  z.band_xcap = a.band_xcap; z.band_wmax = a.band_wmax; z.band_tr = a.band_tr;
  if (mode == SPMM_APPLY) launch_spmm<double2, SPMM_APPLY>(z, R / 2, false, false, sigma, nsm, s);
  else launch_spmm<double2, SPMM_RESID>(z, R / 2, false, false, sigma, nsm, s);
  return true;
}

#if SAD_SPMM_PART == 2
// Arnoldi-mode SpMM of a real block with an even number of columns through the
// banded kernel's PAIR mode (16-byte lanes); false: not applicable, the caller
// runs the per-column kernels
template <int RP, bool PRE, bool SIGMA>
static bool pair_arnoldi_u(const SpmmArgs<double2>& z, cudaStream_t s) {
  if (z.band_tr >= 2 * 16 * (32 / RP))
    return launch_band_u<double2, double, RP, SPMM_ARNOLDI, PRE, SIGMA, 4, true>(z, s);
  return launch_band_u<double2, double, RP, SPMM_ARNOLDI, PRE, SIGMA, 2, true>(z, s);
}
template <int RP>
static bool pair_arnoldi_r(const SpmmArgs<double2>& z, bool pre, bool sigma, cudaStream_t s) {
  if (pre) return sigma ? pair_arnoldi_u<RP, true, true>(z, s) : pair_arnoldi_u<RP, true, false>(z, s);
  return sigma ? pair_arnoldi_u<RP, false, true>(z, s) : pair_arnoldi_u<RP, false, false>(z, s);
}
static bool pair_arnoldi(const SpmmArgs<double>& a, int R, bool pre, bool sigma, cudaStream_t s) {
  if (R % 2 || a.sigma.y != 0.0 || !a.band_meta || a.row0 != 0 || (a.stride & 1)) return false;
  static const bool off = [] {
    const char* e = getenv("SAD_SPMM_PAIRS");
    return e && *e && atoi(e) == 0;
  }();
  if (off) return false;
  SpmmArgs<double2> z{};
  z.n = a.n; z.rowptr = a.rowptr; z.colidx = a.colidx; z.vals = a.vals;
  z.x = reinterpret_cast<const double2*>(a.x);
  z.y = reinterpret_cast<double2*>(a.y);
  z.b = reinterpret_cast<const double2*>(a.b);
  z.dinv = reinterpret_cast<const double2*>(a.dinv);      // doubles: read as such in PAIR mode
  z.zout = reinterpret_cast<double2*>(a.zout);
  z.sigma = a.sigma;
  z.stride = a.stride / 2;
  z.row0 = 0;
  z.band_meta = a.band_meta; z.band_seg = a.band_seg; z.band_dinv = a.band_dinv;
  z.band_xstride = a.band_xstride;
  z.band_xcap = a.band_xcap; z.band_wmax = a.band_wmax; z.band_tr = a.band_tr;
  z.st = a.st;
  switch (R / 2) {
    case 1: return pair_arnoldi_r<1>(z, pre, sigma, s);
    case 2: return pair_arnoldi_r<2>(z, pre, sigma, s);
    case 3: return pair_arnoldi_r<3>(z, pre, sigma, s);
    case 4: return pair_arnoldi_r<4>(z, pre, sigma, s);
  }
  return false;
}
#endif

template <typename XT, int MODE>
int launch_spmm(const SpmmArgs<XT>& a, int R, bool vc, bool pre, bool sigma, int nsm,
                cudaStream_t s, int grid_cap) {
#if SAD_SPMM_PART == 2
  if constexpr (std::is_same<XT, double>::value && MODE == SPMM_ARNOLDI) {
    if (pair_arnoldi(a, R, pre, sigma, s)) return 0;
  }
#endif
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

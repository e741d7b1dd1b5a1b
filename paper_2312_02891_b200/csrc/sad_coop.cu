// sad_coop.cu -- one variant of the cooperative persistent GMRES launcher
// (see sad_coop.cuh).  Compiled once per -DSAD_COOP_VARIANT=<n> (0..9) by
// paper_2312_02891_b200/_build.py.
#include <mutex>

#include "sad_coop.cuh"

#ifndef SAD_COOP_VARIANT
#error "compile with -DSAD_COOP_VARIANT=<0..9>"
#endif

namespace sad {

template <typename XT, typename VT, int R, bool SIGMA, bool FLEX>
static cudaError_t coop_launch_t(PArgs<XT> a, const CoopCfg& cfg, cudaStream_t s, size_t smem,
                                 int* grid_out) {
  auto kern = k_gmres_persistent<XT, VT, R, true, SIGMA, FLEX>;
  // the smem attribute and the occupancy query cost tens of microseconds per
  // call; both depend only on smem here, so they are cached per variant (the
  // small configs launch one solve per side per outer step)
  static std::mutex mu;
  static size_t attr_smem = 0;
  static size_t occ_smem = ~size_t(0);
  static int occ_nb = 0;
  int nb = 0;
  cudaError_t e = cudaSuccess;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (smem > attr_smem) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr_smem = smem;
    }
    if (smem != occ_smem) {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_nb, kern, kThreads, smem);
      if (e != cudaSuccess) return e;
      occ_smem = smem;
    }
    nb = occ_nb;
  }
  if (nb < 1) return cudaErrorInvalidConfiguration;
  const int sms = cfg.max_sms > 0 ? (cfg.max_sms < cfg.nsm ? cfg.max_sms : cfg.nsm) : cfg.nsm;
  const long long elems = a.n * R;
  const long long per_block = (long long)kThreads * (cfg.min_elems_per_thread > 1 ? cfg.min_elems_per_thread : 1);
  long long grid = (elems + per_block - 1) / per_block;
  if (grid > (long long)nb * sms) grid = (long long)nb * sms;
  if (grid > (long long)cfg.max_blocks) grid = cfg.max_blocks;
  if (grid < 1) grid = 1;
  a.rows_per_block = (a.n + grid - 1) / grid;
  if (a.band_meta) {
    // banded sub-phase A1: slabs are whole tiles
    a.rows_per_block = (a.rows_per_block + a.band_tr - 1) / a.band_tr * a.band_tr;
    grid = (a.n + a.rows_per_block - 1) / a.rows_per_block;
  }
  if (a.direct_a && a.rows_per_block > a.direct_rows) return cudaErrorInvalidConfiguration;
  a.pT = cfg.max_blocks;
  void* args[] = {(void*)&a};
  if (grid_out) *grid_out = (int)grid;
  return cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)grid), dim3(kThreads), args,
                                     smem, s);
}

#define SAD_COOP_DEF(tag, XT, VT, SIGMA, FLEX)                                               \
  cudaError_t coop_launch_##tag(int R, PArgs<XT> a, const CoopCfg& cfg, cudaStream_t s,     \
                                size_t smem, int* grid_out) {                               \
    switch (R) {                                                                            \
      case 1: return coop_launch_t<XT, VT, 1, SIGMA, FLEX>(a, cfg, s, smem, grid_out);      \
      case 2: return coop_launch_t<XT, VT, 2, SIGMA, FLEX>(a, cfg, s, smem, grid_out);      \
      case 3: return coop_launch_t<XT, VT, 3, SIGMA, FLEX>(a, cfg, s, smem, grid_out);      \
      case 4: return coop_launch_t<XT, VT, 4, SIGMA, FLEX>(a, cfg, s, smem, grid_out);      \
      case 5: return coop_launch_t<XT, VT, 5, SIGMA, FLEX>(a, cfg, s, smem, grid_out);      \
      case 6: return coop_launch_t<XT, VT, 6, SIGMA, FLEX>(a, cfg, s, smem, grid_out);      \
      case 7: return coop_launch_t<XT, VT, 7, SIGMA, FLEX>(a, cfg, s, smem, grid_out);      \
      case 8: return coop_launch_t<XT, VT, 8, SIGMA, FLEX>(a, cfg, s, smem, grid_out);      \
    }                                                                                       \
    return cudaErrorInvalidValue;                                                           \
  }

// the SAD_COOP_VARIANT-th entry of SAD_COOP_VARIANTS
#if SAD_COOP_VARIANT == 0
SAD_COOP_DEF(d_s0_f0, double, double, false, false)
#elif SAD_COOP_VARIANT == 1
SAD_COOP_DEF(d_s0_f1, double, double, false, true)
#elif SAD_COOP_VARIANT == 2
SAD_COOP_DEF(d_s1_f0, double, double, true, false)
#elif SAD_COOP_VARIANT == 3
SAD_COOP_DEF(d_s1_f1, double, double, true, true)
#elif SAD_COOP_VARIANT == 4
SAD_COOP_DEF(z_s0_f0, double2, double, false, false)
#elif SAD_COOP_VARIANT == 5
SAD_COOP_DEF(z_s0_f1, double2, double, false, true)
#elif SAD_COOP_VARIANT == 6
SAD_COOP_DEF(z_s1_f0, double2, double, true, false)
#elif SAD_COOP_VARIANT == 7
SAD_COOP_DEF(z_s1_f1, double2, double, true, true)
#elif SAD_COOP_VARIANT == 8
SAD_COOP_DEF(zc_s0_f0, double2, double2, false, false)
#elif SAD_COOP_VARIANT == 9
SAD_COOP_DEF(zc_s0_f1, double2, double2, false, true)
#else
#error "SAD_COOP_VARIANT out of range"
#endif

}  // namespace sad

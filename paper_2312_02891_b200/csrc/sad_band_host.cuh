// sad_band_host.cuh -- inspector of the banded SpMM plan (sad_spmm_band.cuh),
// included by sad_capi.cu.  Runs once per sparsity pattern (a matrix or its
// transpose; a merged base + mass pattern), on the host cores in parallel over
// row tiles, and uploads the plan.  A pattern whose tiles touch more x rows
// than fit the shared-memory buffer, need more than kBandMaxRanges ranges after
// merging, or pad to much more than their nonzeros gets NO plan: the operator
// then runs the CSR kernels (k_spmm_bulk) as before.
#pragma once

#include <thread>

#include "sad_spmm_band.cuh"

namespace {

constexpr int kBandGap = 4;          // ranges closer than this are merged
constexpr int kBandXMax = 1400;      // local rows per tile the plan accepts

struct BandPlan {
  long long n = 0, ntiles = 0, nent = 0, nnz = 0;
  int xcap = 0, wmax = 0, tr = 0;      // tr: rows per tile
  int xstride = 0;                     // local rows reserved per tile in the Jacobi-row copies (even)
  BandMeta* meta = nullptr;            // device
  unsigned short* idx = nullptr;       // device: local row of every padded slot
  int* perm = nullptr;                 // device: CSR position of every padded slot (-1 = padding)
  int* lrow = nullptr;                 // device [ntiles * xstride]: x row of every local row (-1 unused)
  unsigned char* seg_base = nullptr;   // device: values + indices segments of the matrix itself
                                       // (operators with identity mass share them; the shift is
                                       // in the epilogue)
};

// the plans of one pattern (a matrix side, or a merged base + mass pattern whose
// host arrays are kept here), by class
struct BandSet {
  std::vector<int> rp, ci;
  BandPlan* plan[2] = {nullptr, nullptr};
  bool tried[2] = {false, false};
};

void band_free(sad_ctx* ctx, BandPlan* p);
void bandset_free(sad_ctx* ctx, BandSet* b) {
  if (!b) return;
  band_free(ctx, b->plan[0]);
  band_free(ctx, b->plan[1]);
  delete b;
}

void band_free(sad_ctx* ctx, BandPlan* p) {
  if (!p) return;
  ctx_free(ctx, p->meta);
  ctx_free(ctx, p->idx);
  ctx_free(ctx, p->perm);
  ctx_free(ctx, p->lrow);
  ctx_free(ctx, p->seg_base);
  delete p;
}

struct TileInfo {
  BandMeta m;
  int rows_total;   // local rows used
  bool ok;
};

// ranges + padded width of one tile
void band_tile_ranges(long long n, const int* rp, const int* ci, long long t, int TR, TileInfo& out,
                      std::vector<int>& cols) {
  const long long r0 = t * TR;
  const long long r1 = std::min<long long>(n, r0 + TR);
  cols.clear();
  int W = 0;
  for (long long i = r0; i < r1; ++i) {
    W = std::max(W, rp[i + 1] - rp[i]);
    for (int k = rp[i]; k < rp[i + 1]; ++k) cols.push_back(ci[k]);
    cols.push_back((int)i);            // the row itself (shift term, padding target)
  }
  std::sort(cols.begin(), cols.end());
  cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
  // maximal runs, merged when closer than kBandGap
  std::vector<std::pair<int, int>> rg;   // [start, end)
  for (int cidx : cols) {
    if (!rg.empty() && cidx - rg.back().second < kBandGap) rg.back().second = cidx + 1;
    else rg.push_back({cidx, cidx + 1});
  }
  while ((int)rg.size() > kBandMaxRanges) {
    // merge the two neighbours with the smallest gap
    size_t best = 1;
    for (size_t q = 2; q < rg.size(); ++q)
      if (rg[q].first - rg[q - 1].second < rg[best].first - rg[best - 1].second) best = q;
    rg[best - 1].second = rg[best].second;
    rg.erase(rg.begin() + best);
  }
  BandMeta& m = out.m;
  std::memset(&m, 0, sizeof(m));
  m.W = (short)std::max(W, 1);
  m.nr = (short)rg.size();
  long long pos = 0;
  out.ok = W <= 32767;
  for (size_t q = 0; q < rg.size(); ++q) {
    const long long len = (long long)rg[q].second - rg[q].first;
    if (q > 0) pos += 1;                               // spare row between ranges
    if ((pos ^ rg[q].first) & 1) pos += 1;             // ro == xs (mod 2)
    if (len > 65535 || pos + len > kBandXMax) { out.ok = false; break; }
    m.xs[q] = rg[q].first;
    m.xl[q] = (unsigned short)len;
    m.ro[q] = (unsigned short)pos;
    if (r0 >= rg[q].first && r0 < rg[q].second) m.self_off = (int)(pos + (r0 - rg[q].first));
    pos += len;
  }
  out.rows_total = (int)pos + 1;
  m.xrows = out.rows_total;
}

inline int band_local(const BandMeta& m, int col) {
  for (int q = 0; q < m.nr; ++q)
    if (col >= m.xs[q] && col < m.xs[q] + (int)m.xl[q]) return (int)m.ro[q] + (col - m.xs[q]);
  return -1;
}

// Build the plan of an n x n CSR pattern (host arrays) with TR rows per tile;
// nullptr if it does not fit.  stage_est: bytes of one pipeline stage for a
// 64-byte block row, real values and a real Jacobi diagonal (the tile-size choice).
BandPlan* band_build_tr(sad_ctx* ctx, long long n, const std::vector<int>& rp, const std::vector<int>& ci,
                        int TR, size_t stage_limit) {
  const int kBandRows = TR;
  const long long ntiles = (n + kBandRows - 1) / kBandRows;
  const long long nnz = (long long)ci.size();
  if (ntiles < 1 || nnz < 1) return nullptr;
  std::vector<TileInfo> info(ntiles);
  const int nth = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  auto par = [&](auto fn) {
    std::vector<std::thread> th;
    for (int w = 0; w < nth; ++w)
      th.emplace_back([&, w] {
        const long long t0 = ntiles * w / nth, t1 = ntiles * (w + 1) / nth;
        fn(t0, t1);
      });
    for (auto& t : th) t.join();
  };
  par([&](long long t0, long long t1) {
    std::vector<int> cols;
    for (long long t = t0; t < t1; ++t) band_tile_ranges(n, rp.data(), ci.data(), t, TR, info[t], cols);
  });
  long long nent = 0;
  int xcap = 0, wmax = 0;
  for (long long t = 0; t < ntiles; ++t) {
    if (!info[t].ok) return nullptr;
    if (nent > 0xffffffffLL - (long long)info[t].m.W * kBandRows) return nullptr;
    info[t].m.eoff = (unsigned)nent;
    nent += (long long)info[t].m.W * kBandRows;
    xcap = std::max(xcap, info[t].rows_total);
    wmax = std::max(wmax, (int)info[t].m.W);
  }
  if (nent > nnz + nnz / 2 + 64 * kBandRows) return nullptr;   // too much padding
  if (stage_limit && (size_t)xcap * 72 + (size_t)wmax * TR * 10 > stage_limit) return nullptr;
  const int xstride = (xcap + 1) & ~1;
  std::vector<unsigned short> idx((size_t)nent);
  std::vector<int> perm((size_t)nent);
  std::vector<int> lrow((size_t)ntiles * xstride, -1);
  std::vector<BandMeta> meta(ntiles);
  std::atomic<bool> bad{false};
  par([&](long long t0, long long t1) {
    for (long long t = t0; t < t1; ++t) {
      const BandMeta& m = info[t].m;
      meta[t] = m;
      for (int q = 0; q < m.nr; ++q)
        for (int k = 0; k < (int)m.xl[q]; ++k)
          lrow[(size_t)t * xstride + m.ro[q] + k] = m.xs[q] + k;
      const long long r0 = t * kBandRows;
      for (int lr = 0; lr < kBandRows; ++lr) {
        const long long i = r0 + lr;
        const int k0 = i < n ? rp[i] : 0, k1 = i < n ? rp[i + 1] : 0;
        for (int s = 0; s < m.W; ++s) {
          const size_t e = (size_t)m.eoff + (size_t)s * kBandRows + lr;
          if (k0 + s < k1) {
            const int l = band_local(m, ci[k0 + s]);
            if (l < 0) bad = true;
            idx[e] = (unsigned short)std::max(l, 0);
            perm[e] = k0 + s;
          } else {
            idx[e] = (unsigned short)(i < n ? m.self_off + lr : m.self_off);
            perm[e] = -1;
          }
        }
      }
    }
  });
  if (bad) return nullptr;
  BandPlan* p = new BandPlan();
  p->n = n;
  p->ntiles = ntiles;
  p->nent = nent;
  p->nnz = nnz;
  p->xcap = xcap;
  p->wmax = wmax;
  p->tr = TR;
  p->xstride = xstride;
  if (ctx_malloc(ctx, (void**)&p->meta, (size_t)ntiles * sizeof(BandMeta)) != cudaSuccess ||
      ctx_malloc(ctx, (void**)&p->idx, (size_t)nent * 2 + 64) != cudaSuccess ||
      ctx_malloc(ctx, (void**)&p->perm, (size_t)nent * 4) != cudaSuccess ||
      ctx_malloc(ctx, (void**)&p->lrow, lrow.size() * 4) != cudaSuccess ||
      cudaMemcpy(p->lrow, lrow.data(), lrow.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->meta, meta.data(), (size_t)ntiles * sizeof(BandMeta), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->idx, idx.data(), (size_t)nent * 2, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->perm, perm.data(), (size_t)nent * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaGetLastError();
    band_free(ctx, p);
    return nullptr;
  }
  return p;
}

// The largest tile (256, 128, 64 rows) whose stage fits three times in shared
// memory; small matrices take 64 (more tiles than SMs matter more there).
// Class 1 (the persistent GMRES kernel's SpMM sub-phase, two blocks per SM next
// to the kernel's other shared memory): 128-row tiles when two stages fit in
// ~90 KB, else 64.  SAD_BAND_ROWS / SAD_BAND_ROWS_P override (multiples of 8).
BandPlan* band_build(sad_ctx* ctx, long long n, const std::vector<int>& rp, const std::vector<int>& ci,
                     int cls) {
  const char* e = std::getenv(cls ? "SAD_BAND_ROWS_P" : "SAD_BAND_ROWS");
  if (e && *e) return band_build_tr(ctx, n, rp, ci, std::max(32, std::atoi(e) & ~7), 0);
  if (cls == 0) {
    for (int tr : {256, 128}) {
      if (n < (long long)tr * ctx->nsm * 4) continue;
      if (BandPlan* p = band_build_tr(ctx, n, rp, ci, tr, 70 * 1024)) return p;
    }
  } else if (n >= (long long)128 * ctx->nsm * 8) {
    if (BandPlan* p = band_build_tr(ctx, n, rp, ci, 128, 46 * 1024)) return p;
  }
  return band_build_tr(ctx, n, rp, ci, 64, 0);
}

// values + indices segments of a plan from CSR values on the device
template <typename VT>
int band_segments(sad_ctx* ctx, const BandPlan* p, const VT* vals_dev, unsigned char** out) {
  CK(ctx, ctx_malloc(ctx, (void**)out, (size_t)p->nent * (sizeof(VT) + 2) + 64));
  const int blocks = (int)std::min<long long>(p->ntiles, (long long)ctx->nsm * 16);
  k_band_segments<VT><<<blocks, 256>>>(p->ntiles, p->tr, p->meta, p->idx, p->perm, vals_dev, *out);
  COUNT_LAUNCH(1);
  CKL(ctx);
  // Plans are built on first use, possibly from a solve on a non-blocking stream
  // (the concurrent A / B solves of DeviceAdi): the segments must be complete before
  // any stream reads them, so the legacy-stream kernel is waited for here (once
  // per operator and plan class).
  CK(ctx, cudaStreamSynchronize(cudaStreamLegacy));
  return SAD_OK;
}

// the Jacobi rows of every tile in local row order (per operator: D depends on the shift)
template <typename DT>
int band_dinv_rows(sad_ctx* ctx, const BandPlan* p, const DT* dinv_dev, DT** out) {
  const long long count = p->ntiles * (long long)p->xstride;
  CK(ctx, ctx_malloc(ctx, (void**)out, (size_t)count * sizeof(DT) + 64));
  const int blocks = (int)std::min<long long>((count + 255) / 256, (long long)ctx->nsm * 32);
  k_band_dinv<DT><<<blocks, 256>>>(count, p->lrow, dinv_dev, *out);
  COUNT_LAUNCH(1);
  CKL(ctx);
  CK(ctx, cudaStreamSynchronize(cudaStreamLegacy));
  return SAD_OK;
}

// SAD_SPMM_BAND: 0 = never, 1 = every operator, unset = operators with >= 1M nonzeros
bool band_wanted(long long nnz) {
  const char* e = std::getenv("SAD_SPMM_BAND");
  if (e && *e) return std::atoi(e) != 0;
  return nnz >= (1LL << 20);
}

}  // namespace

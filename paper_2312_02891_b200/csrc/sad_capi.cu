// sad_capi.cu -- C-ABI of libsylvadi_b200.so (see include/sylvadi_b200.h).
//
// Host runtime of the inner-solve hot path: CSR upload (+ explicit transpose),
// shifted operators with device Jacobi, the batched GMRES/FGMRES driver whose
// inner loop advances without host synchronisation (device finishers + a
// host-mapped progress flag polled only to stop issuing work), Gram/axpy block
// utilities for the device-resident ADI step.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/sylvadi_b200.h"
#include "sad_kernels.cuh"
#include "sad_coop.cuh"
#include "sad_spmm_launch.cuh"
#include "sad_verify.cuh"
#include "sad_adi.cuh"
#include "sad_spmm_bulk.cuh"

using namespace sad;

#define SAD_ABI_VERSION 1

// Device allocations of matrices, operators and workspaces go through a
// per-context cache: a destroyed handle's buffers are kept for reuse instead
// of cudaFree (which synchronises the device; tearing down an ADI engine's
// two dozen operators cost ~50 ms of a ~120 ms config-2 call).  A reused
// buffer may still be in use by kernels launched before its previous owner
// was destroyed, so the first reuse after any free synchronises the device
// once (cheap: it happens when a new engine is built, with the device idle).
struct DevCache {
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks;   // size -> pointer
  std::unordered_map<void*, size_t> live;     // pointer -> size
  size_t free_bytes = 0;
  bool pending = false;                       // frees since the last device sync
};

struct sad_ctx {
  DevCache cache;
  std::mutex op_mu;              // serialises sad_op_create
  int device = 0;
  int nsm = 148;
  std::string err;
  double* scratch = nullptr;     // gram partials
  unsigned* ticket = nullptr;
  double2* gram_out = nullptr;
  double2* gram_host = nullptr;  // pinned
  int scratch_blocks = 0;
  double2* epi_part = nullptr;   // fused ADI epilogue partials (lazy)
  double2* epi_out = nullptr;
  double2* epi_host = nullptr;   // pinned
  // tall-skinny products (verification diagnostics), grown on demand
  double2* ts_part = nullptr;
  size_t ts_part_elems = 0;
  double2* ts_dev = nullptr;     // reduced outputs / coefficients
  double2* ts_host = nullptr;    // pinned staging
  size_t ts_elems = 0;
};

struct DevCsr {
  int* rowptr = nullptr;
  int* colidx = nullptr;
  double* vals = nullptr;
};

namespace { struct BandPlan; struct BandSet; }   // sad_band_host.cuh

struct sad_csr {
  sad_ctx* ctx = nullptr;
  unsigned long long uid = 0;
  // banded SpMM plans of the patterns this matrix is the base of: its own (mass
  // uid 0) and the merged base + mass patterns, per side; built on first use
  std::mutex band_mu;
  std::map<std::pair<unsigned long long, int>, BandSet*> bands;
  long long nrows = 0, ncols = 0, nnz = 0;
  DevCsr d, dt;  // matrix and (optional) transpose
  bool has_t = false;
  std::vector<int> h_rowptr, h_colidx;   // host copies (transpose/union builds)
  std::vector<double> h_vals;
  std::vector<int> ht_rowptr, ht_colidx;
  std::vector<double> ht_vals;
};

static std::atomic<unsigned long long> g_op_uid{1};
static std::atomic<long long> g_launches{0};   // kernels launched by this library
#define COUNT_LAUNCH(k) g_launches.fetch_add((k), std::memory_order_relaxed)
namespace sad {
void count_launches(long long k) { COUNT_LAUNCH(k); }
int g_spmm_bulk_sms = 148;
}

struct sad_op {
  sad_ctx* ctx = nullptr;
  unsigned long long uid = 0;
  long long n = 0;
  long long ncols = 0;          // columns (n; n_loc + n_halo for a row slab)
  const int* rowptr = nullptr;
  const int* colidx = nullptr;
  const void* vals = nullptr;
  // banded SpMM plans (built on first use; null: CSR kernels).  Class 0: the
  // stand-alone SpMM (large tiles); class 1: the persistent kernel's SpMM
  // sub-phase (tiles that fit next to its other shared memory).  Values in a
  // plan's layout: double, or double2 if vals_complex.
  const sad_csr* base_csr = nullptr;
  unsigned long long mass_uid = 0;
  int adjoint = 0;
  BandSet* bset = nullptr;
  const BandPlan* band[2] = {nullptr, nullptr};
  const unsigned char* band_seg[2] = {nullptr, nullptr};
  unsigned char* own_band_seg[2] = {nullptr, nullptr};
  // the tiles' Jacobi rows in the plan's layout, [class][0 real / 1 complex], built when a
  // block of that type first runs the Jacobi prologue
  void* band_dinv[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  bool band_tried[2] = {false, false};
  bool band_ok = false;               // SAD_SPMM_BAND / size rule, read when the operator is created
  bool vals_complex = false;
  bool sigma_identity = false;  // identity mass: shift added in the epilogue
  double2 sigma_eff = {0.0, 0.0};
  bool real_ok = true;          // operator (and dinv) real
  // owned storage for assembled matrices
  int* own_rowptr = nullptr;
  int* own_colidx = nullptr;
  void* own_vals = nullptr;
  double2* dinv_c = nullptr;
  double* dinv_r = nullptr;
  int precond = 0;
  long long nnz = 0;
  struct HostApply* happ = nullptr;   // sad_op_apply_host staging (lazy)
};

// Chunked, pipelined y = Op x between HOST buffers (sad_op_apply_host): x is
// uploaded in row chunks on one stream, the SpMM of output chunk k starts as
// soon as every x chunk up to its largest column index has landed, and y
// chunk k is downloaded on a third stream while later chunks compute, so the
// two PCIe directions and the SpMM overlap.
struct HostApply {
  int r = 0, dtype = -1, nchunk = 0;
  size_t esz = 0;
  void* xd = nullptr;
  void* yd = nullptr;
  std::vector<long long> bounds;   // nchunk + 1 row boundaries
  std::vector<int> need;           // last x chunk each output chunk reads
  cudaStream_t sin = nullptr, sout = nullptr;
  std::vector<cudaEvent_t> ein, ecomp;
  cudaEvent_t estart = nullptr, eend = nullptr;
};

struct sad_gmres {
  sad_ctx* ctx = nullptr;
  long long n = 0;
  long long n_ext = 0;          // rows per basis block incl. halo (row-partitioned solves)
  void* xext = nullptr;         // row-partitioned: solution [local | halo]
  double* rsum = nullptr;       // row-partitioned: rank sums (pstride doubles)
  long long* hist_host = nullptr;   // row-partitioned: per-step progress history
  long long* hist_dev = nullptr;
  int dist_dcgs2 = 0;           // row-partitioned: 1 = DCGS2 (default), 0 = CGS2
  size_t dual_smem = 0;         // row-partitioned DCGS2: dual-dot shared memory
  int R = 1, dtype = 0, m = 1, flexible = 0;
  size_t esz = 8;
  void* V = nullptr;
  void* Z = nullptr;
  char* state = nullptr;
  size_t state_bytes = 0;
  double* part = nullptr;
  int max_blocks = 0;
  int pstride = 0;
  long long* hflag_host = nullptr;
  long long* hflag_dev = nullptr;
  long long* res_host = nullptr;   // pinned: iterations [8] | residual norms [8]
  GState st{};
  int64_t bytes = 0;
  int dot_blocks_per_sm = 1;
  // persistent engine
  int engine = SAD_ENGINE_PERSISTENT;
  int max_sms = 0;              // 0 = all SMs
  int min_elems_per_thread = 2;
  int direct_a = -1;            // phase-A path: -1 auto, 0 TMA ring, 1 direct loads
  int resident_csr = 1;         // keep small CSR slabs in shared memory
  int dbg_delay_ns = 0;         // SAD_OPT_DEBUG_DELAY (race stress tests)
  PState pst{};
  double* stats_dev = nullptr;
  // profiling (sad_gmres_profile): synchronous stepping with CUDA events
  int profile = 0;
  int pending_multi = 0;
  double pending_tol = 0.0;
  int timers = 0;   // phase timers without event profiling (sad_gmres_fixed)
  double prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double prof2[5] = {0, 0, 0, 0, 0};   // work_A, work_C (block 0), fin_A, fin_C (last block), spmm_A (block 0), ms
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
};

// -----------------------------------------------------------------------------
static int set_err(sad_ctx* ctx, int code, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return code;
}

#define CK(ctx, call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return set_err((ctx), SAD_ECUDA, "%s failed: %s (%s:%d)", #call,             \
                     cudaGetErrorString(e_), __FILE__, __LINE__);                   \
  } while (0)

#define CKL(ctx)                                                                   \
  do {                                                                             \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess)                                                         \
      return set_err((ctx), SAD_ECUDA, "kernel launch failed: %s (%s:%d)",         \
                     cudaGetErrorString(e_), __FILE__, __LINE__);                   \
  } while (0)

static inline cudaStream_t S_(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Wait for a stream by polling it: the small configs' outer loop waits for
// the solves once per step, and a blocking synchronisation that yields the
// thread costs tens of microseconds of wake-up latency each time.
static cudaError_t spin_sync(cudaStream_t s) {
  for (;;) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e != cudaErrorNotReady) return e;
  }
}

static constexpr size_t kCacheLimit = (size_t)8 << 30;   // cached free bytes before a release

static size_t cache_round(size_t n) {
  const size_t g = n >= ((size_t)2 << 20) ? ((size_t)2 << 20) : 4096;
  return (n + g - 1) / g * g;
}

static void cache_release_locked(DevCache& c) {
  if (c.free_blocks.empty()) return;
  cudaDeviceSynchronize();
  for (auto& kv : c.free_blocks) cudaFree(kv.second);
  c.free_blocks.clear();
  c.free_bytes = 0;
  c.pending = false;
}

// cudaMalloc through the context's cache (best fit within 1/8 + 4 KB slack)
static cudaError_t ctx_malloc(sad_ctx* ctx, void** p, size_t n) {
  DevCache& c = ctx->cache;
  const size_t rn = cache_round(std::max<size_t>(n, 1));
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.free_blocks.lower_bound(rn);
  if (it != c.free_blocks.end() && it->first <= rn + rn / 8 + 4096) {
    if (c.pending) {
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) return e;
      c.pending = false;
    }
    *p = it->second;
    c.live[it->second] = it->first;
    c.free_bytes -= it->first;
    c.free_blocks.erase(it);
    return cudaSuccess;
  }
  cudaError_t e = cudaMalloc(p, rn);
  if (e == cudaErrorMemoryAllocation && !c.free_blocks.empty()) {
    cudaGetLastError();
    cache_release_locked(c);
    e = cudaMalloc(p, rn);
  }
  if (e == cudaSuccess) c.live[*p] = rn;
  return e;
}

static void ctx_free(sad_ctx* ctx, void* p) {
  if (!p) return;
  DevCache& c = ctx->cache;
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.live.find(p);
  if (it == c.live.end()) {   // not from the cache
    cudaFree(p);
    return;
  }
  c.free_blocks.insert({it->second, p});
  c.free_bytes += it->second;
  c.live.erase(it);
  c.pending = true;
  if (c.free_bytes > kCacheLimit) cache_release_locked(c);
}

extern "C" int sad_ctx_trim(sad_ctx* ctx) {
  if (!ctx) return SAD_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->cache.mu);
  cache_release_locked(ctx->cache);
  return SAD_OK;
}

extern "C" int sad_version(void) { return SAD_ABI_VERSION; }
extern "C" int64_t sad_kernel_launches(void) { return g_launches.load(); }

extern "C" int sad_ctx_create(int device, sad_ctx** out) {
  if (!out) return SAD_EINVAL;
  *out = nullptr;
  sad_ctx* c = new sad_ctx();
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete c; return SAD_ECUDA; }
  int nsm = 0;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    delete c;
    return SAD_ECUDA;
  }
  c->nsm = nsm;
  g_spmm_bulk_sms = nsm;
  c->scratch_blocks = nsm * 4;
  if (cudaMalloc(&c->scratch, (size_t)c->scratch_blocks * 2 * 64 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&c->ticket, 64) != cudaSuccess ||
      cudaMalloc(&c->gram_out, 64 * sizeof(double2)) != cudaSuccess ||
      cudaMallocHost(&c->gram_host, 64 * sizeof(double2)) != cudaSuccess) {
    delete c;
    return SAD_ENOMEM;
  }
  cudaMemset(c->ticket, 0, 64);
  *out = c;
  return SAD_OK;
}

extern "C" int sad_ctx_destroy(sad_ctx* c) {
  if (!c) return SAD_OK;
  {
    std::lock_guard<std::mutex> lk(c->cache.mu);
    cache_release_locked(c->cache);
  }
  cudaFree(c->scratch);
  cudaFree(c->ticket);
  cudaFree(c->gram_out);
  cudaFreeHost(c->gram_host);
  cudaFree(c->epi_part);
  cudaFree(c->epi_out);
  if (c->epi_host) cudaFreeHost(c->epi_host);
  cudaFree(c->ts_part);
  cudaFree(c->ts_dev);
  if (c->ts_host) cudaFreeHost(c->ts_host);
  delete c;
  return SAD_OK;
}

extern "C" const char* sad_last_error(const sad_ctx* c) { return c ? c->err.c_str() : "null ctx"; }
extern "C" int sad_ctx_num_sms(const sad_ctx* c) { return c ? c->nsm : 0; }

#include "sad_band_host.cuh"

// -----------------------------------------------------------------------------
// CSR
// -----------------------------------------------------------------------------
static void host_transpose(long long nr, long long nc, const std::vector<int>& rp,
                           const std::vector<int>& ci, const std::vector<double>& v,
                           std::vector<int>& trp, std::vector<int>& tci, std::vector<double>& tv) {
  // counting sort by column; rows visited in increasing order, so each row of the
  // transpose is sorted by (original) row index -- the same summation order as
  // scipy's CSC scatter (csc_matvec) for A^T x.
  trp.assign(nc + 1, 0);
  for (size_t k = 0; k < ci.size(); ++k) trp[ci[k] + 1]++;
  for (long long j = 0; j < nc; ++j) trp[j + 1] += trp[j];
  tci.resize(ci.size());
  tv.resize(ci.size());
  std::vector<int> pos(trp.begin(), trp.end() - 1);
  for (long long i = 0; i < nr; ++i)
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      int p = pos[ci[k]]++;
      tci[p] = (int)i;
      tv[p] = v[k];
    }
}

static int upload_csr(sad_ctx* ctx, DevCsr& d, const std::vector<int>& rp,
                      const std::vector<int>& ci, const std::vector<double>& v) {
  // +64 bytes: the TMA bulk SpMM widens its source ranges to 16-byte alignment
  CK(ctx, ctx_malloc(ctx, (void**)&d.rowptr, rp.size() * sizeof(int) + 64));
  CK(ctx, ctx_malloc(ctx, (void**)&d.colidx, std::max<size_t>(ci.size(), 1) * sizeof(int) + 64));
  CK(ctx, ctx_malloc(ctx, (void**)&d.vals, std::max<size_t>(v.size(), 1) * sizeof(double) + 64));
  CK(ctx, cudaMemcpy(d.rowptr, rp.data(), rp.size() * sizeof(int), cudaMemcpyHostToDevice));
  if (!ci.empty()) {
    CK(ctx, cudaMemcpy(d.colidx, ci.data(), ci.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(ctx, cudaMemcpy(d.vals, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  return SAD_OK;
}

static void free_csr(sad_ctx* ctx, DevCsr& d) {
  ctx_free(ctx, d.rowptr);
  ctx_free(ctx, d.colidx);
  ctx_free(ctx, d.vals);
  d = DevCsr();
}

extern "C" int sad_csr_create(sad_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz,
                              const int32_t* rowptr, const int32_t* colidx, const double* vals,
                              int build_transpose, sad_csr** out) {
  if (!ctx || !out) return SAD_EINVAL;
  *out = nullptr;
  if (nrows < 0 || ncols < 0 || nnz < 0 || nnz > 2147483647LL || !rowptr)
    return set_err(ctx, SAD_EINVAL, "bad CSR sizes");
  if (rowptr[0] != 0 || rowptr[nrows] != nnz)
    return set_err(ctx, SAD_EINVAL, "row offsets inconsistent with nnz");
  for (int64_t i = 0; i < nrows; ++i) {
    if (rowptr[i + 1] < rowptr[i]) return set_err(ctx, SAD_EINVAL, "row offsets not monotone");
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      if (colidx[k] < 0 || colidx[k] >= ncols)
        return set_err(ctx, SAD_EINVAL, "column index out of range in row %lld", (long long)i);
      if (k > rowptr[i] && colidx[k] <= colidx[k - 1])
        return set_err(ctx, SAD_EINVAL, "column indices not strictly increasing in row %lld",
                       (long long)i);
      if (!std::isfinite(vals[k])) return set_err(ctx, SAD_EINVAL, "non-finite matrix entry");
    }
  }
  sad_csr* c = new sad_csr();
  c->ctx = ctx;
  c->uid = g_op_uid.fetch_add(1);
  c->nrows = nrows;
  c->ncols = ncols;
  c->nnz = nnz;
  c->h_rowptr.assign(rowptr, rowptr + nrows + 1);
  c->h_colidx.assign(colidx, colidx + nnz);
  c->h_vals.assign(vals, vals + nnz);
  int rc = upload_csr(ctx, c->d, c->h_rowptr, c->h_colidx, c->h_vals);
  if (rc == SAD_OK && build_transpose) {
    host_transpose(nrows, ncols, c->h_rowptr, c->h_colidx, c->h_vals, c->ht_rowptr,
                   c->ht_colidx, c->ht_vals);
    rc = upload_csr(ctx, c->dt, c->ht_rowptr, c->ht_colidx, c->ht_vals);
    c->has_t = true;
  }
  if (rc != SAD_OK) {
    free_csr(ctx, c->d);
    free_csr(ctx, c->dt);
    delete c;
    return rc;
  }
  *out = c;
  return SAD_OK;
}

extern "C" int sad_csr_destroy(sad_csr* c) {
  if (!c) return SAD_OK;
  for (auto& kv : c->bands) bandset_free(c->ctx, kv.second);
  free_csr(c->ctx, c->d);
  free_csr(c->ctx, c->dt);
  delete c;
  return SAD_OK;
}

extern "C" int64_t sad_csr_nnz(const sad_csr* c) { return c ? c->nnz : -1; }

// -----------------------------------------------------------------------------
// shifted operators
// -----------------------------------------------------------------------------
static int grid_for(long long work, int per_block, int cap) {
  long long g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

extern "C" int sad_op_create(sad_ctx* ctx, const sad_csr* base, const sad_csr* mass,
                             double sre, double sim, int adjoint, int precond_kind,
                             sad_op** out) {
  if (!ctx || !base || !out) return SAD_EINVAL;
  *out = nullptr;
  if (base->nrows != base->ncols) return set_err(ctx, SAD_EINVAL, "shifted operator must be square");
  if (mass && (mass->nrows != base->nrows || mass->ncols != base->ncols))
    return set_err(ctx, SAD_EINVAL, "base and mass dimensions disagree");
  if (adjoint && (!base->has_t || (mass && !mass->has_t)))
    return set_err(ctx, SAD_EINVAL, "adjoint operator needs matrices created with build_transpose");
  if (precond_kind != SAD_PRECOND_NONE && precond_kind != SAD_PRECOND_JACOBI)
    return set_err(ctx, SAD_EINVAL, "unknown preconditioner kind %d", precond_kind);
  // creation is serialised per context (shared error string, legacy-stream
  // work); concurrent solves on other streams are unaffected
  std::lock_guard<std::mutex> creating(ctx->op_mu);
  sad_op* op = new sad_op();
  op->ctx = ctx;
  op->uid = g_op_uid.fetch_add(1);
  op->n = base->nrows;
  op->ncols = base->nrows;
  op->base_csr = base;
  op->mass_uid = mass ? mass->uid : 0;
  op->adjoint = adjoint ? 1 : 0;
  op->precond = precond_kind;
  const double2 sig = adjoint ? make_double2(sre, -sim) : make_double2(sre, sim);
  op->sigma_eff = sig;
  const DevCsr& bd = adjoint ? base->dt : base->d;
  if (!mass) {
    op->rowptr = bd.rowptr;
    op->colidx = bd.colidx;
    op->vals = bd.vals;
    op->nnz = base->nnz;
    op->vals_complex = false;
    op->sigma_identity = true;
    op->real_ok = (sig.y == 0.0);
  } else {
    // assemble base + sigma*mass on the merged pattern (sparse.py:138-155)
    const std::vector<int>& brp = adjoint ? base->ht_rowptr : base->h_rowptr;
    const std::vector<int>& bci = adjoint ? base->ht_colidx : base->h_colidx;
    const std::vector<double>& bv = adjoint ? base->ht_vals : base->h_vals;
    const std::vector<int>& mrp = adjoint ? mass->ht_rowptr : mass->h_rowptr;
    const std::vector<int>& mci = adjoint ? mass->ht_colidx : mass->h_colidx;
    const std::vector<double>& mv = adjoint ? mass->ht_vals : mass->h_vals;
    const long long n = base->nrows;
    std::vector<int> rp(n + 1, 0), ci;
    std::vector<double> vr, vi;
    ci.reserve(bci.size() + mci.size());
    const bool cplx = (sig.y != 0.0);
    vr.reserve(ci.capacity());
    if (cplx) vi.reserve(ci.capacity());
    for (long long i = 0; i < n; ++i) {
      int p = brp[i], q = mrp[i];
      const int pe = brp[i + 1], qe = mrp[i + 1];
      while (p < pe || q < qe) {
        int cb = p < pe ? bci[p] : INT32_MAX;
        int cm = q < qe ? mci[q] : INT32_MAX;
        int col = std::min(cb, cm);
        double a = 0.0, mm = 0.0;
        if (cb == col) a = bv[p++];
        if (cm == col) mm = mv[q++];
        ci.push_back(col);
        vr.push_back(a + sig.x * mm);
        if (cplx) vi.push_back(sig.y * mm);
      }
      rp[i + 1] = (int)ci.size();
    }
    size_t nz = ci.size();
    CK(ctx, ctx_malloc(ctx, (void**)&op->own_rowptr, (n + 1) * sizeof(int) + 64));
    CK(ctx, ctx_malloc(ctx, (void**)&op->own_colidx, std::max<size_t>(nz, 1) * sizeof(int) + 64));
    CK(ctx, cudaMemcpy(op->own_rowptr, rp.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice));
    if (nz) CK(ctx, cudaMemcpy(op->own_colidx, ci.data(), nz * sizeof(int), cudaMemcpyHostToDevice));
    if (cplx) {
      std::vector<double2> vc(nz);
      for (size_t k = 0; k < nz; ++k) vc[k] = make_double2(vr[k], vi[k]);
      CK(ctx, ctx_malloc(ctx, &op->own_vals, std::max<size_t>(nz, 1) * sizeof(double2) + 64));
      if (nz) CK(ctx, cudaMemcpy(op->own_vals, vc.data(), nz * sizeof(double2), cudaMemcpyHostToDevice));
    } else {
      CK(ctx, ctx_malloc(ctx, &op->own_vals, std::max<size_t>(nz, 1) * sizeof(double) + 64));
      if (nz) CK(ctx, cudaMemcpy(op->own_vals, vr.data(), nz * sizeof(double), cudaMemcpyHostToDevice));
    }
    op->rowptr = op->own_rowptr;
    op->colidx = op->own_colidx;
    op->vals = op->own_vals;
    op->nnz = (long long)nz;
    op->vals_complex = cplx;
    op->sigma_identity = false;
    op->real_ok = !cplx;
    if (band_wanted((long long)nz)) {
      // the merged pattern is the same for every shift: kept once per (mass, side)
      // for the plans built on first use
      sad_csr* bm = const_cast<sad_csr*>(base);
      std::lock_guard<std::mutex> lk(bm->band_mu);
      BandSet*& bs = bm->bands[std::make_pair(mass->uid, adjoint ? 1 : 0)];
      if (!bs) {
        bs = new BandSet();
        bs->rp = rp;
        bs->ci = ci;
      }
    }
  }
  op->band_ok = band_wanted(op->nnz);
  // Jacobi dinv (precond.py:272-276): 1/diag(assembled op); identity when "none"
  const long long n = op->n;
  // one allocation for both dinv copies; the breakdown flag lives in the ctx
  char* dbuf = nullptr;
  const size_t nn = (size_t)std::max<long long>(n, 1);
  const size_t dr_off = (nn * sizeof(double2) + 255) & ~size_t(255);
  const size_t bd_off = (dr_off + nn * sizeof(double) + 255) & ~size_t(255);
  CK(ctx, ctx_malloc(ctx, (void**)&dbuf, bd_off + 256));
  op->dinv_c = reinterpret_cast<double2*>(dbuf);
  op->dinv_r = reinterpret_cast<double*>(dbuf + dr_off);
  // the breakdown flag belongs to this operator (two host threads may create
  // operators on one context at once)
  int* d_bd = reinterpret_cast<int*>(dbuf + bd_off);
  CK(ctx, cudaMemsetAsync(d_bd, 0, sizeof(int), 0));
  const int blocks = grid_for(n, 256, ctx->nsm * 16);
  if (precond_kind == SAD_PRECOND_JACOBI) {
    if (op->vals_complex)
      k_jacobi<double2><<<blocks, 256>>>(n, op->rowptr, op->colidx,
                                         (const double2*)op->vals, sig, 0, op->dinv_c, d_bd);
    else
      k_jacobi<double><<<blocks, 256>>>(n, op->rowptr, op->colidx, (const double*)op->vals,
                                        sig, op->sigma_identity ? 1 : 0, op->dinv_c, d_bd);
  } else {
    std::vector<double2> ones(n, make_double2(1.0, 0.0));
    CK(ctx, cudaMemcpy(op->dinv_c, ones.data(), n * sizeof(double2), cudaMemcpyHostToDevice));
  }
  k_c2r<<<blocks, 256>>>(n, op->dinv_c, op->dinv_r);
  CKL(ctx);
  int brk = 0;
  CK(ctx, cudaMemcpy(&brk, d_bd, sizeof(int), cudaMemcpyDeviceToHost));
  if (brk) {
    sad_op_destroy(op);
    return set_err(ctx, SAD_EBREAKDOWN, "zero diagonal entry for Jacobi");
  }
  *out = op;
  return SAD_OK;
}

static void host_apply_free(sad_op* op) {
  HostApply* h = op->happ;
  if (!h) return;
  if (h->sin) cudaStreamSynchronize(h->sin);
  if (h->sout) cudaStreamSynchronize(h->sout);
  ctx_free(op->ctx, h->xd);
  ctx_free(op->ctx, h->yd);
  for (cudaEvent_t e : h->ein) cudaEventDestroy(e);
  for (cudaEvent_t e : h->ecomp) cudaEventDestroy(e);
  if (h->estart) cudaEventDestroy(h->estart);
  if (h->eend) cudaEventDestroy(h->eend);
  if (h->sin) cudaStreamDestroy(h->sin);
  if (h->sout) cudaStreamDestroy(h->sout);
  delete h;
  op->happ = nullptr;
}

extern "C" int sad_op_destroy(sad_op* op) {
  if (!op) return SAD_OK;
  host_apply_free(op);
  ctx_free(op->ctx, op->own_rowptr);
  ctx_free(op->ctx, op->own_colidx);
  ctx_free(op->ctx, op->own_vals);
  for (int cl = 0; cl < 2; ++cl) {
    ctx_free(op->ctx, op->own_band_seg[cl]);
    ctx_free(op->ctx, op->band_dinv[cl][0]);
    ctx_free(op->ctx, op->band_dinv[cl][1]);
  }
  ctx_free(op->ctx, op->dinv_c);   // dinv_r lives in the same allocation
  delete op;
  return SAD_OK;
}

// The operator's plan of class cls (0 stand-alone SpMM, 1 persistent kernel),
// built on first use; nullptr when the pattern has none
static const BandPlan* op_band(sad_op* op, int cls) {
  if (op->band_tried[cls]) return op->band[cls];
  op->band_tried[cls] = true;
  if (!op->base_csr || !op->band_ok) return nullptr;
  sad_ctx* ctx = op->ctx;
  sad_csr* bm = const_cast<sad_csr*>(op->base_csr);
  std::lock_guard<std::mutex> lk(bm->band_mu);
  BandSet*& bs = bm->bands[std::make_pair(op->mass_uid, op->adjoint)];
  if (!bs) {
    if (op->mass_uid) return nullptr;     // merged pattern not kept
    bs = new BandSet();
  }
  if (!bs->tried[cls]) {
    bs->tried[cls] = true;
    const std::vector<int>& rp = op->mass_uid ? bs->rp : (op->adjoint ? bm->ht_rowptr : bm->h_rowptr);
    const std::vector<int>& ci = op->mass_uid ? bs->ci : (op->adjoint ? bm->ht_colidx : bm->h_colidx);
    BandPlan* p = band_build(ctx, op->n, rp, ci, cls);
    if (p && !op->mass_uid) {
      // identity mass: the operators of every shift share the matrix's values
      const DevCsr& bd = op->adjoint ? bm->dt : bm->d;
      if (band_segments<double>(ctx, p, bd.vals, &p->seg_base) != SAD_OK) {
        band_free(ctx, p);
        p = nullptr;
      }
    }
    bs->plan[cls] = p;
  }
  const BandPlan* p = bs->plan[cls];
  if (!p || p->nnz != op->nnz) return nullptr;
  if (!op->mass_uid) {
    op->band_seg[cls] = p->seg_base;
  } else {
    const int rc = op->vals_complex
        ? band_segments<double2>(ctx, p, (const double2*)op->own_vals, &op->own_band_seg[cls])
        : band_segments<double>(ctx, p, (const double*)op->own_vals, &op->own_band_seg[cls]);
    if (rc != SAD_OK) {
      ctx_free(ctx, op->own_band_seg[cls]);
      op->own_band_seg[cls] = nullptr;
      return nullptr;
    }
    op->band_seg[cls] = op->own_band_seg[cls];
  }
  op->band[cls] = p;
  return p;
}

// The tiles' Jacobi rows for blocks of the given type (built on first use; nullptr on failure)
static const void* op_band_dinv(sad_op* op, int cls, bool cplx) {
  const BandPlan* p = op->band[cls];
  if (!p) return nullptr;
  void*& slot = op->band_dinv[cls][cplx ? 1 : 0];
  if (!slot) {
    sad_csr* bm = const_cast<sad_csr*>(op->base_csr);
    std::lock_guard<std::mutex> lk(bm->band_mu);
    if (!slot) {
      const int rc = cplx ? band_dinv_rows<double2>(op->ctx, p, op->dinv_c, (double2**)&slot)
                          : band_dinv_rows<double>(op->ctx, p, op->dinv_r, (double**)&slot);
      if (rc != SAD_OK) {
        ctx_free(op->ctx, slot);
        slot = nullptr;
      }
    }
  }
  return slot;
}

// info[7]: plan present (0/1), tiles, padded entries, nonzeros, local x rows per
// tile (max), padded row length (max), rows per tile
extern "C" int sad_op_band_info(sad_op* op, int cls, int64_t* info) {
  if (!op || !info || cls < 0 || cls > 1) return SAD_EINVAL;
  for (int i = 0; i < 7; ++i) info[i] = 0;
  if (const BandPlan* p = op_band(op, cls)) {
    info[0] = 1;
    info[1] = p->ntiles;
    info[2] = p->nent;
    info[3] = p->nnz;
    info[4] = p->xcap;
    info[5] = p->wmax;
    info[6] = p->tr;
  }
  return SAD_OK;
}

extern "C" int sad_op_get_dinv(const sad_op* op, double* dinv_host) {
  if (!op || !dinv_host) return SAD_EINVAL;
  CK(op->ctx, cudaMemcpy(dinv_host, op->dinv_c, op->n * sizeof(double2), cudaMemcpyDeviceToHost));
  return SAD_OK;
}

static int check_block(sad_ctx* ctx, int r, int dtype) {
  if (r < 1 || r > 8) return set_err(ctx, SAD_EINVAL, "block width r=%d outside 1..8", r);
  if (dtype != SAD_F64 && dtype != SAD_C128) return set_err(ctx, SAD_EINVAL, "bad dtype %d", dtype);
  return SAD_OK;
}

template <typename XT>
static void op_band_args(sad_op* op, SpmmArgs<XT>& a) {
  const BandPlan* p = op_band(op, 0);
  if (!p) return;
  const void* dv = op_band_dinv(op, 0, sizeof(XT) == 16);
  if (!dv) return;
  a.band_meta = p->meta;
  a.band_seg = op->band_seg[0];
  a.band_dinv = dv;
  a.band_xstride = p->xstride;
  a.band_xcap = p->xcap;
  a.band_wmax = p->wmax;
  a.band_tr = p->tr;
}

template <int MODE>
static int op_spmm(sad_op* op, int r, int dtype, const void* b, const void* x, void* y, void* stream) {
  sad_ctx* ctx = op->ctx;
  int rc = check_block(ctx, r, dtype);
  if (rc) return rc;
  if (dtype == SAD_F64) {
    if (!op->real_ok) return set_err(ctx, SAD_EINVAL, "complex shift needs a complex128 block");
    SpmmArgs<double> a{};
    a.n = op->n; a.rowptr = op->rowptr; a.colidx = op->colidx; a.vals = op->vals;
    a.x = (const double*)x; a.y = (double*)y; a.b = (const double*)b;
    a.dinv = op->dinv_r; a.sigma = op->sigma_eff;
    op_band_args(op, a);
    rc = launch_spmm<double, MODE>(a, r, false, false, op->sigma_identity, ctx->nsm, S_(stream));
  } else {
    SpmmArgs<double2> a{};
    a.n = op->n; a.rowptr = op->rowptr; a.colidx = op->colidx; a.vals = op->vals;
    a.x = (const double2*)x; a.y = (double2*)y; a.b = (const double2*)b;
    a.dinv = op->dinv_c; a.sigma = op->sigma_eff;
    op_band_args(op, a);
    rc = launch_spmm<double2, MODE>(a, r, op->vals_complex, false, op->sigma_identity, ctx->nsm,
                                    S_(stream));
  }
  if (rc) return rc;
  CKL(ctx);
  return SAD_OK;
}

extern "C" int sad_op_apply(sad_op* op, int r, int dtype, const void* x, void* y, void* stream) {
  if (!op || !x || !y) return SAD_EINVAL;
  return op_spmm<SPMM_APPLY>(op, r, dtype, nullptr, x, y, stream);
}

extern "C" int sad_op_residual(sad_op* op, int r, int dtype, const void* b, const void* x, void* y,
                               void* stream) {
  if (!op || !b || !x || !y) return SAD_EINVAL;
  return op_spmm<SPMM_RESID>(op, r, dtype, b, x, y, stream);
}

// largest column index over the rows [bounds[k], bounds[k+1]) of each chunk
__global__ void k_chunk_maxcol(const int* rowptr, const int* colidx, const long long* bounds,
                               int* out) {
  const int k = blockIdx.x;
  const int kb = rowptr[bounds[k]], ke = rowptr[bounds[k + 1]];
  int mx = -1;
  for (int i = kb + threadIdx.x; i < ke; i += blockDim.x) mx = max(mx, colidx[i]);
  for (int sh = 16; sh > 0; sh >>= 1) mx = max(mx, __shfl_down_sync(0xffffffffu, mx, sh));
  __shared__ int s_mx[32];
  if ((threadIdx.x & 31) == 0) s_mx[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = max(mx, s_mx[w]);
    out[k] = max(mx, s_mx[0]);
  }
}

static int host_apply_setup(sad_op* op, int r, int dtype) {
  sad_ctx* ctx = op->ctx;
  HostApply* h = op->happ;
  const size_t esz = dtype == SAD_F64 ? 8 : 16;
  if (h && h->r == r && h->dtype == dtype) return SAD_OK;
  host_apply_free(op);
  h = op->happ = new HostApply();
  h->r = r;
  h->dtype = dtype;
  h->esz = esz;
  const long long n = op->n;
  const size_t bytes = (size_t)n * r * esz;
  // ~16 MiB chunks (PCIe transfers stay efficient), at most 128 of them
  const long long target = std::max<long long>(1, (long long)((bytes + (16u << 20) - 1) / (16u << 20)));
  h->nchunk = (int)std::min<long long>(std::min<long long>(target, 128), std::max<long long>(n, 1));
  h->bounds.resize(h->nchunk + 1);
  for (int k = 0; k <= h->nchunk; ++k) h->bounds[k] = n * k / h->nchunk;
  CK(ctx, ctx_malloc(ctx, &h->xd, bytes + 64));
  CK(ctx, ctx_malloc(ctx, &h->yd, bytes + 64));
  CK(ctx, cudaStreamCreateWithFlags(&h->sin, cudaStreamNonBlocking));
  CK(ctx, cudaStreamCreateWithFlags(&h->sout, cudaStreamNonBlocking));
  h->ein.resize(h->nchunk);
  h->ecomp.resize(h->nchunk);
  for (int k = 0; k < h->nchunk; ++k) {
    CK(ctx, cudaEventCreateWithFlags(&h->ein[k], cudaEventDisableTiming));
    CK(ctx, cudaEventCreateWithFlags(&h->ecomp[k], cudaEventDisableTiming));
  }
  CK(ctx, cudaEventCreateWithFlags(&h->estart, cudaEventDisableTiming));
  CK(ctx, cudaEventCreateWithFlags(&h->eend, cudaEventDisableTiming));
  // which x chunk each output chunk waits for (x chunks land in order)
  long long* dbounds = nullptr;
  int* dmax = nullptr;
  CK(ctx, cudaMalloc(&dbounds, (h->nchunk + 1) * sizeof(long long)));
  CK(ctx, cudaMalloc(&dmax, h->nchunk * sizeof(int)));
  CK(ctx, cudaMemcpy(dbounds, h->bounds.data(), (h->nchunk + 1) * sizeof(long long),
                     cudaMemcpyHostToDevice));
  k_chunk_maxcol<<<h->nchunk, 256>>>(op->rowptr, op->colidx, dbounds, dmax);
  COUNT_LAUNCH(1);
  std::vector<int> mx(h->nchunk);
  CK(ctx, cudaMemcpy(mx.data(), dmax, h->nchunk * sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(dbounds);
  cudaFree(dmax);
  h->need.resize(h->nchunk);
  for (int k = 0; k < h->nchunk; ++k) {
    // the diagonal term (shift) reads x rows of the chunk itself
    const long long col = std::max<long long>(mx[k], h->bounds[k + 1] - 1);
    int q = (int)(std::upper_bound(h->bounds.begin(), h->bounds.end(), col) - h->bounds.begin()) - 1;
    h->need[k] = std::min(std::max(q, k), h->nchunk - 1);
  }
  return SAD_OK;
}

extern "C" int sad_op_apply_host(sad_op* op, int r, int dtype, const void* x_host, void* y_host,
                                 void* stream) {
  if (!op || !x_host || !y_host) return SAD_EINVAL;
  sad_ctx* ctx = op->ctx;
  int rc = check_block(ctx, r, dtype);
  if (rc) return rc;
  if (dtype == SAD_F64 && !op->real_ok)
    return set_err(ctx, SAD_EINVAL, "complex shift needs a complex128 block");
  if (op->ncols != op->n) return set_err(ctx, SAD_EINVAL, "host apply needs a square operator");
  rc = host_apply_setup(op, r, dtype);
  if (rc) return rc;
  HostApply* h = op->happ;
  cudaStream_t s = S_(stream);
  const size_t rowb = (size_t)r * h->esz;
  // the staging buffers are reused: uploads wait for earlier work on `stream`
  CK(ctx, cudaEventRecord(h->estart, s));
  CK(ctx, cudaStreamWaitEvent(h->sin, h->estart, 0));
  CK(ctx, cudaStreamWaitEvent(h->sout, h->estart, 0));
  for (int k = 0; k < h->nchunk; ++k) {
    const long long b0 = h->bounds[k], b1 = h->bounds[k + 1];
    CK(ctx, cudaMemcpyAsync((char*)h->xd + b0 * rowb, (const char*)x_host + b0 * rowb,
                            (b1 - b0) * rowb, cudaMemcpyHostToDevice, h->sin));
    CK(ctx, cudaEventRecord(h->ein[k], h->sin));
  }
  int waited = -1;
  for (int k = 0; k < h->nchunk; ++k) {
    const long long b0 = h->bounds[k], b1 = h->bounds[k + 1];
    if (h->need[k] > waited) {
      CK(ctx, cudaStreamWaitEvent(s, h->ein[h->need[k]], 0));
      waited = h->need[k];
    }
    if (b1 > b0) {
      if (dtype == SAD_F64) {
        SpmmArgs<double> a{};
        a.n = b1 - b0; a.row0 = b0;
        a.rowptr = op->rowptr + b0; a.colidx = op->colidx; a.vals = op->vals;
        a.x = (const double*)h->xd; a.y = (double*)h->yd + b0 * r;
        a.dinv = op->dinv_r; a.sigma = op->sigma_eff;
        rc = launch_spmm<double, SPMM_APPLY>(a, r, false, false, op->sigma_identity, ctx->nsm, s);
      } else {
        SpmmArgs<double2> a{};
        a.n = b1 - b0; a.row0 = b0;
        a.rowptr = op->rowptr + b0; a.colidx = op->colidx; a.vals = op->vals;
        a.x = (const double2*)h->xd; a.y = (double2*)h->yd + b0 * r;
        a.dinv = op->dinv_c; a.sigma = op->sigma_eff;
        rc = launch_spmm<double2, SPMM_APPLY>(a, r, op->vals_complex, false, op->sigma_identity,
                                               ctx->nsm, s);
      }
      if (rc) return set_err(ctx, SAD_EINVAL, "unsupported block width %d", r);
      CKL(ctx);
    }
    CK(ctx, cudaEventRecord(h->ecomp[k], s));
    CK(ctx, cudaStreamWaitEvent(h->sout, h->ecomp[k], 0));
    CK(ctx, cudaMemcpyAsync((char*)y_host + b0 * rowb, (const char*)h->yd + b0 * rowb,
                            (b1 - b0) * rowb, cudaMemcpyDeviceToHost, h->sout));
  }
  CK(ctx, cudaEventRecord(h->eend, h->sout));
  CK(ctx, cudaStreamWaitEvent(s, h->eend, 0));
  CK(ctx, cudaStreamSynchronize(s));
  return SAD_OK;
}

extern "C" int sad_csr_apply(sad_csr* csr, int transpose, int r, int dtype, const void* x, void* y,
                             void* stream) {
  if (!csr || !x || !y) return SAD_EINVAL;
  sad_ctx* ctx = csr->ctx;
  int rc = check_block(ctx, r, dtype);
  if (rc) return rc;
  if (transpose && !csr->has_t) return set_err(ctx, SAD_EINVAL, "transpose was not built");
  const DevCsr& d = transpose ? csr->dt : csr->d;
  const long long rows = transpose ? csr->ncols : csr->nrows;
  if (dtype == SAD_F64) {
    SpmmArgs<double> a{};
    a.n = rows; a.rowptr = d.rowptr; a.colidx = d.colidx; a.vals = d.vals;
    a.x = (const double*)x; a.y = (double*)y;
    rc = launch_spmm<double, SPMM_APPLY>(a, r, false, false, false, ctx->nsm, S_(stream));
  } else {
    SpmmArgs<double2> a{};
    a.n = rows; a.rowptr = d.rowptr; a.colidx = d.colidx; a.vals = d.vals;
    a.x = (const double2*)x; a.y = (double2*)y;
    rc = launch_spmm<double2, SPMM_APPLY>(a, r, false, false, false, ctx->nsm, S_(stream));
  }
  if (rc) return rc;
  CKL(ctx);
  return SAD_OK;
}

// -----------------------------------------------------------------------------
// GMRES workspace
// -----------------------------------------------------------------------------
template <typename T>
static T* carve(char*& p, size_t count) {
  size_t off = (reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15);
  T* r = reinterpret_cast<T*>(off);
  p = reinterpret_cast<char*>(off + count * sizeof(T));
  return r;
}

static size_t dot_smem(int J, int R, size_t esz) { return (size_t)J * kWarps * R * esz + kWarps * R * 8; }
static size_t upd_smem(int J, int R, size_t esz) { return (size_t)J * R * esz; }

template <typename XT, int R>
static int set_smem_attrs(size_t dsm, size_t usm) {
  cudaError_t e = cudaSuccess;
  e = cudaFuncSetAttribute(k_dot<XT, R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_dot<XT, R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_update<XT, R, UPD_ORTH1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_update<XT, R, UPD_ORTH2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_update<XT, R, UPD_X>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_update<XT, R, UPD_XF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm);
  return e == cudaSuccess ? 0 : 1;
}

template <typename XT>
static int set_smem_all(int R, size_t dsm, size_t usm) {
  switch (R) {
    case 1: return set_smem_attrs<XT, 1>(dsm, usm);
    case 2: return set_smem_attrs<XT, 2>(dsm, usm);
    case 3: return set_smem_attrs<XT, 3>(dsm, usm);
    case 4: return set_smem_attrs<XT, 4>(dsm, usm);
    case 5: return set_smem_attrs<XT, 5>(dsm, usm);
    case 6: return set_smem_attrs<XT, 6>(dsm, usm);
    case 7: return set_smem_attrs<XT, 7>(dsm, usm);
    case 8: return set_smem_attrs<XT, 8>(dsm, usm);
  }
  return 1;
}

static int gmres_create(sad_ctx* ctx, int64_t n, int64_t n_ext, int r, int dtype, int restart,
                        int flexible, sad_gmres** out) {
  if (!ctx || !out) return SAD_EINVAL;
  *out = nullptr;
  int rc = check_block(ctx, r, dtype);
  if (rc) return rc;
  if (n < 1) return set_err(ctx, SAD_EINVAL, "n must be >= 1");
  if (n_ext < n) return set_err(ctx, SAD_EINVAL, "extended rows %lld < local rows %lld",
                                (long long)n_ext, (long long)n);
  if (restart < 1 || restart > 400) return set_err(ctx, SAD_EINVAL, "restart %d outside 1..400", restart);
  sad_gmres* ws = new sad_gmres();
  ws->ctx = ctx;
  ws->n = n;
  ws->n_ext = n_ext;
  ws->R = r;
  ws->dtype = dtype;
  ws->m = restart;
  ws->flexible = flexible ? 1 : 0;
  ws->esz = dtype == SAD_F64 ? 8 : 16;
  const int m = restart;
  const size_t blk = (size_t)n_ext * r * ws->esz;
  size_t dsm = dot_smem(m + 1, r, ws->esz), usm = upd_smem(m + 1, r, ws->esz);
  if (dsm > 220 * 1024) {
    delete ws;
    return set_err(ctx, SAD_EINVAL, "restart %d too long for the shared-memory dot at r=%d", m, r);
  }
  int bad = dtype == SAD_F64 ? set_smem_all<double>(r, dsm, usm) : set_smem_all<double2>(r, dsm, usm);
  if (bad) {
    delete ws;
    return set_err(ctx, SAD_ECUDA, "cudaFuncSetAttribute failed");
  }
  ws->dot_blocks_per_sm = std::max(1, std::min(8, (int)((200 * 1024) / dsm)));
  if (ctx_malloc(ctx, &ws->V, blk * (m + 1) + 64) != cudaSuccess) {
    delete ws;
    return set_err(ctx, SAD_ENOMEM, "basis allocation of %zu bytes failed", blk * (m + 1));
  }
  if (ws->flexible && ctx_malloc(ctx, &ws->Z, blk * m) != cudaSuccess) {
    ctx_free(ctx, ws->V);
    delete ws;
    return set_err(ctx, SAD_ENOMEM, "FGMRES Z allocation failed");
  }
  ws->max_blocks = ctx->nsm * 8;
  // [max_blocks][pstride] doubles for the multi engine; the persistent engine
  // uses the same buffer output-major: [(2(m+1)+1) r][max_blocks] complex
  ws->pstride = 2 * (2 * (m + 1) * r + r) + 8;
  size_t sb = 0;
  sb += 16 * 8;                              // j, any_active, jx, ticket, seqs
  sb += 4 * r * sizeof(int) + r * 8 + 64;    // active, done, kdim, iters
  sb += (size_t)(m + 1) * r * 8;             // S
  sb += 2 * (size_t)(m + 1) * r * 16;        // h, h2
  sb += (size_t)r * m * (m + 1) * 16;        // H
  sb += (size_t)r * m * 8 + (size_t)r * m * 16;  // cs, sn
  sb += (size_t)r * (m + 1) * 16;            // g
  sb += (size_t)m * r * 16;                  // ycoef
  sb += 2 * r * 8;                           // wpre2, beta
  sb += (size_t)r * (m + 1) * (m + 1) * 16;  // G (persistent engine)
  sb += 2 * (size_t)(m + 1) * r * 16;        // hc, coef
  sb += (size_t)(2 * (m + 1) + 1) * r * 16;  // red
  sb += 4 * 16 + 16 * 8;                     // barrier, err, stats
  sb += 64 * 16;                             // alignment slack
  ws->state_bytes = sb;
  if (ctx_malloc(ctx, (void**)&ws->state, sb) != cudaSuccess ||
      ctx_malloc(ctx, (void**)&ws->part, (size_t)ws->max_blocks * ws->pstride * sizeof(double)) != cudaSuccess ||
      cudaHostAlloc(&ws->hflag_host, 8 * sizeof(long long), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc(&ws->res_host, 16 * sizeof(long long), cudaHostAllocDefault) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&ws->hflag_dev, ws->hflag_host, 0) != cudaSuccess) {
    sad_gmres_destroy(ws);
    return set_err(ctx, SAD_ENOMEM, "workspace allocation failed");
  }
  cudaMemset(ws->state, 0, sb);
  char* p = ws->state;
  GState& st = ws->st;
  st.j = carve<int>(p, 1);
  st.any_active = carve<int>(p, 1);
  st.jx = carve<int>(p, 1);
  st.ticket = carve<unsigned>(p, 1);
  st.stepseq = carve<unsigned long long>(p, 1);
  st.cycleseq = carve<unsigned long long>(p, 1);
  st.active = carve<int>(p, r);
  st.done = carve<int>(p, r);
  st.kdim = carve<int>(p, r);
  st.iters = carve<long long>(p, r);
  st.S = carve<double>(p, (size_t)(m + 1) * r);
  st.h = carve<double2>(p, (size_t)(m + 1) * r);
  st.h2 = carve<double2>(p, (size_t)(m + 1) * r);
  st.H = carve<double2>(p, (size_t)r * m * (m + 1));
  st.cs = carve<double>(p, (size_t)r * m);
  st.sn = carve<double2>(p, (size_t)r * m);
  st.g = carve<double2>(p, (size_t)r * (m + 1));
  st.ycoef = carve<double2>(p, (size_t)m * r);
  st.wpre2 = carve<double>(p, r);
  st.beta = carve<double>(p, r);
  PState& ps = ws->pst;
  ps.G = carve<double2>(p, (size_t)r * (m + 1) * (m + 1));
  ps.hc = carve<double2>(p, (size_t)(m + 1) * r);
  ps.coef = carve<double2>(p, (size_t)(m + 1) * r);
  ps.red = carve<double2>(p, (size_t)(2 * (m + 1) + 1) * r);
  ps.bar_count = carve<unsigned>(p, 1);
  ps.bar_gen = carve<unsigned>(p, 1);
  ps.err = carve<int>(p, 1);
  ps.stats = carve<double>(p, 16);
  ws->stats_dev = ps.stats;
  if ((size_t)(p - ws->state) > sb) {
    sad_gmres_destroy(ws);
    return set_err(ctx, SAD_EINVAL, "internal: state carve overflow");
  }
  st.part = ws->part;
  st.hflag = ws->hflag_dev;
  st.m = m;
  st.R = r;
  st.pstride = ws->pstride;
  ws->bytes = (int64_t)(blk * (m + 1) + (ws->flexible ? blk * m : 0) + sb +
                        (size_t)ws->max_blocks * ws->pstride * 8);
  *out = ws;
  return SAD_OK;
}

extern "C" int sad_gmres_create(sad_ctx* ctx, int64_t n, int r, int dtype, int restart, int flexible,
                                sad_gmres** out) {
  return gmres_create(ctx, n, n, r, dtype, restart, flexible, out);
}

extern "C" int sad_gmres_destroy(sad_gmres* ws) {
  if (!ws) return SAD_OK;
  ctx_free(ws->ctx, ws->xext);
  ctx_free(ws->ctx, ws->rsum);
  if (ws->hist_host) cudaFreeHost(ws->hist_host);
  for (int i = 0; i < 3; ++i)
    if (ws->ev[i]) cudaEventDestroy(ws->ev[i]);
  ctx_free(ws->ctx, ws->V);
  ctx_free(ws->ctx, ws->Z);
  ctx_free(ws->ctx, ws->state);
  ctx_free(ws->ctx, ws->part);
  if (ws->hflag_host) cudaFreeHost(ws->hflag_host);
  if (ws->res_host) cudaFreeHost(ws->res_host);
  delete ws;
  return SAD_OK;
}

extern "C" int64_t sad_gmres_bytes(const sad_gmres* ws) { return ws ? ws->bytes : -1; }

// ---- per-step launches ------------------------------------------------------
template <typename XT, int R>
struct Orth {
  static void dot(const OrthArgs& a, bool pass1, int grid, size_t smem, cudaStream_t s) {
    COUNT_LAUNCH(1);
    if (pass1) k_dot<XT, R, true><<<grid, kThreads, smem, s>>>(a);
    else k_dot<XT, R, false><<<grid, kThreads, smem, s>>>(a);
  }
  static void upd(const OrthArgs& a, int mode, int grid, size_t smem, cudaStream_t s) {
    COUNT_LAUNCH(1);
    switch (mode) {
      case UPD_ORTH1: k_update<XT, R, UPD_ORTH1><<<grid, kThreads, smem, s>>>(a); break;
      case UPD_ORTH2: k_update<XT, R, UPD_ORTH2><<<grid, kThreads, smem, s>>>(a); break;
      case UPD_X: k_update<XT, R, UPD_X><<<grid, kThreads, smem, s>>>(a); break;
      case UPD_XF: k_update<XT, R, UPD_XF><<<grid, kThreads, smem, s>>>(a); break;
    }
  }
};

template <typename XT>
static void orth_dot(int R, const OrthArgs& a, bool pass1, int grid, size_t smem, cudaStream_t s) {
  switch (R) {
    case 1: Orth<XT, 1>::dot(a, pass1, grid, smem, s); break;
    case 2: Orth<XT, 2>::dot(a, pass1, grid, smem, s); break;
    case 3: Orth<XT, 3>::dot(a, pass1, grid, smem, s); break;
    case 4: Orth<XT, 4>::dot(a, pass1, grid, smem, s); break;
    case 5: Orth<XT, 5>::dot(a, pass1, grid, smem, s); break;
    case 6: Orth<XT, 6>::dot(a, pass1, grid, smem, s); break;
    case 7: Orth<XT, 7>::dot(a, pass1, grid, smem, s); break;
    case 8: Orth<XT, 8>::dot(a, pass1, grid, smem, s); break;
  }
}

template <typename XT>
static void orth_upd(int R, const OrthArgs& a, int mode, int grid, size_t smem, cudaStream_t s) {
  switch (R) {
    case 1: Orth<XT, 1>::upd(a, mode, grid, smem, s); break;
    case 2: Orth<XT, 2>::upd(a, mode, grid, smem, s); break;
    case 3: Orth<XT, 3>::upd(a, mode, grid, smem, s); break;
    case 4: Orth<XT, 4>::upd(a, mode, grid, smem, s); break;
    case 5: Orth<XT, 5>::upd(a, mode, grid, smem, s); break;
    case 6: Orth<XT, 6>::upd(a, mode, grid, smem, s); break;
    case 7: Orth<XT, 7>::upd(a, mode, grid, smem, s); break;
    case 8: Orth<XT, 8>::upd(a, mode, grid, smem, s); break;
  }
}

struct Launcher {
  sad_gmres* ws;
  sad_op* op;
  cudaStream_t s;
  const void* rhs;
  void* x;
  int grid_spmm, grid_dot, grid_upd;
  size_t dsm, usm;

  template <typename XT>
  SpmmArgs<XT> spmm_args(int mode) const {
    SpmmArgs<XT> a{};
    a.n = ws->n;
    a.rowptr = op->rowptr;
    a.colidx = op->colidx;
    a.vals = op->vals;
    a.sigma = op->sigma_eff;
    a.stride = ws->n_ext * ws->R;
    a.st = ws->st;
    a.dinv = reinterpret_cast<const XT*>(sizeof(XT) == 8 ? (const void*)op->dinv_r
                                                         : (const void*)op->dinv_c);
    op_band_args(op, a);
    if (mode == SPMM_ARNOLDI) {
      a.x = reinterpret_cast<const XT*>(ws->V);
      a.zout = reinterpret_cast<XT*>(ws->Z);
    } else {  // residual into V_0
      a.x = reinterpret_cast<const XT*>(x);
      a.b = reinterpret_cast<const XT*>(rhs);
      a.y = reinterpret_cast<XT*>(ws->V);
    }
    return a;
  }

  OrthArgs orth_args() const {
    OrthArgs a{};
    a.n = ws->n;
    a.V = ws->V;
    a.Z = ws->Z;
    a.x = x;
    a.dinv = ws->dtype == SAD_F64 ? (const void*)op->dinv_r : (const void*)op->dinv_c;
    a.stride = ws->n_ext * ws->R;
    a.st = ws->st;
    return a;
  }

  template <typename XT>
  void arnoldi_t(int which) const {
    const bool pre = op->precond == SAD_PRECOND_JACOBI;
    const int R = ws->R;
    const OrthArgs oa = orth_args();
    switch (which) {
      case 0: {
        auto a = spmm_args<XT>(SPMM_ARNOLDI);
        launch_spmm<XT, SPMM_ARNOLDI>(a, R, op->vals_complex, pre, op->sigma_identity,
                                      ws->ctx->nsm, s, grid_spmm);
        break;
      }
      case 1: orth_dot<XT>(R, oa, true, grid_dot, dsm, s); break;
      case 2: orth_upd<XT>(R, oa, UPD_ORTH1, grid_upd, usm, s); break;
      case 3: orth_dot<XT>(R, oa, false, grid_dot, dsm, s); break;
      case 4: orth_upd<XT>(R, oa, UPD_ORTH2, grid_upd, usm, s); break;
    }
  }
  void arnoldi(int which) const {
    if (ws->dtype == SAD_F64) arnoldi_t<double>(which);
    else arnoldi_t<double2>(which);
  }

  template <typename XT>
  void cycle_end_t() const {
    k_trisolve<<<1, 32, 0, s>>>(ws->st, ws->flexible);
    COUNT_LAUNCH(1);
    const OrthArgs oa = orth_args();
    orth_upd<XT>(ws->R, oa, ws->flexible ? UPD_XF : UPD_X, grid_upd, usm, s);
    residual_t<XT>();
  }
  template <typename XT>
  void residual_t() const {
    auto a = spmm_args<XT>(SPMM_RESID_CYCLE);
    launch_spmm<XT, SPMM_RESID_CYCLE>(a, ws->R, op->vals_complex, false, op->sigma_identity,
                                      ws->ctx->nsm, s, grid_spmm);
  }
  void cycle_end() const {
    if (ws->dtype == SAD_F64) cycle_end_t<double>();
    else cycle_end_t<double2>();
  }
  void residual() const {
    if (ws->dtype == SAD_F64) residual_t<double>();
    else residual_t<double2>();
  }
};

static int prepare(sad_gmres* ws, sad_op* op, const void* rhs, void* x, cudaStream_t s,
                   Launcher& L) {
  sad_ctx* ctx = ws->ctx;
  if (!op || !rhs || !x) return set_err(ctx, SAD_EINVAL, "null argument");
  if (op->n != ws->n) return set_err(ctx, SAD_EINVAL, "operator size %lld != workspace size %lld",
                                     op->n, ws->n);
  if (ws->dtype == SAD_F64 && !op->real_ok)
    return set_err(ctx, SAD_EINVAL, "complex shift needs a complex128 workspace");
  L.ws = ws;
  L.op = op;
  L.s = s;
  L.rhs = rhs;
  L.x = x;
  const int R = ws->R;
  const int gpw = 32 / R;
  const int U = (R <= 2) ? 8 : 4;
  const long long tiles = (ws->n + (long long)gpw * U - 1) / ((long long)gpw * U);
  L.grid_spmm = grid_for(ws->n, kWarps * gpw, ws->max_blocks);
  L.grid_dot = grid_for(tiles, kWarps, std::min(ws->max_blocks, ctx->nsm * ws->dot_blocks_per_sm));
  L.grid_upd = grid_for(tiles, kWarps, std::min(ws->max_blocks, ctx->nsm * 8));
  L.dsm = dot_smem(ws->m + 1, R, ws->esz);
  L.usm = upd_smem(ws->m + 1, R, ws->esz);
  return SAD_OK;
}

static int read_results(sad_gmres* ws, void* res, cudaStream_t s, int64_t* iters, double* resn,
                        uint8_t* conv, double tol) {
  sad_ctx* ctx = ws->ctx;
  const int R = ws->R;
  if (res) CK(ctx, cudaMemcpyAsync(res, ws->V, (size_t)ws->n * R * ws->esz, cudaMemcpyDeviceToDevice, s));
  // pinned staging (a pageable destination would make each copy a staged, slower transfer)
  long long* it = ws->res_host;
  double* be = reinterpret_cast<double*>(ws->res_host + 8);
  CK(ctx, cudaMemcpyAsync(it, ws->st.iters, R * sizeof(long long), cudaMemcpyDeviceToHost, s));
  CK(ctx, cudaMemcpyAsync(be, ws->st.beta, R * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(ctx, spin_sync(s));
  for (int c = 0; c < R; ++c) {
    if (iters) iters[c] = it[c];
    if (resn) resn[c] = be[c];
    if (conv) conv[c] = be[c] <= tol ? 1 : 0;
  }
  return SAD_OK;
}

// Spin until `pred()` holds, reading host-mapped flags written by the device.
// Falls back to a stream query so a faulted/finished stream cannot hang us.
template <typename P>
static int spin_until(sad_ctx* ctx, cudaStream_t s, P pred) {
  unsigned long it = 0;
  while (!pred()) {
    if ((++it & 1023) == 0) {
      cudaError_t q = cudaStreamQuery(s);
      if (q == cudaSuccess) {
        std::atomic_thread_fence(std::memory_order_seq_cst);
        if (pred()) break;
        return set_err(ctx, SAD_ECUDA, "device progress flag not observed after stream drained");
      }
      if (q != cudaErrorNotReady)
        return set_err(ctx, SAD_ECUDA, "stream failed: %s", cudaGetErrorString(q));
      if ((it & ((1u << 16) - 1)) == 0) std::this_thread::yield();
    }
  }
  return SAD_OK;
}

// Algorithmic bytes of one shifted SpMM application:
// nnz*(4 + value bytes) + 4(n+1) + read x + write y (+ dinv gather when PRE, + Z write).
static double spmm_bytes(const sad_gmres* ws, const sad_op* op, bool arnoldi) {
  const double n = (double)ws->n, blk = n * ws->R * ws->esz;
  const long long nnz = op->nnz;
  double b = (double)nnz * (4.0 + (op->vals_complex ? 16.0 : 8.0)) + 4.0 * (n + 1) + 2.0 * blk;
  if (arnoldi && op->precond == SAD_PRECOND_JACOBI) b += n * ws->esz;
  if (arnoldi && ws->flexible) b += blk;
  return b;
}

extern "C" int sad_gmres_profile(sad_gmres* ws, int enable, double* stats_host) {
  if (!ws) return SAD_EINVAL;
  sad_ctx* ctx = ws->ctx;
  if (stats_host) {
    for (int i = 0; i < 8; ++i) stats_host[i] = ws->prof[i];
    for (int i = 0; i < 5; ++i) stats_host[8 + i] = ws->prof2[i];
  }
  if (enable) {
    for (int i = 0; i < 8; ++i) ws->prof[i] = 0.0;
    for (int i = 0; i < 5; ++i) ws->prof2[i] = 0.0;
    for (int i = 0; i < 3; ++i)
      if (!ws->ev[i]) CK(ctx, cudaEventCreate(&ws->ev[i]));
  }
  ws->profile = enable ? 1 : 0;
  return SAD_OK;
}

// ---- persistent (cooperative) engine ------------------------------------------
static CoopCfg coop_cfg(const sad_gmres* ws) {
  CoopCfg c;
  c.nsm = ws->ctx->nsm;
  c.max_sms = ws->max_sms;
  c.min_elems_per_thread = ws->min_elems_per_thread;
  c.max_blocks = ws->max_blocks;
  return c;
}

static cudaError_t coop_dispatch_d(PArgs<double> a, sad_gmres* ws, sad_op* op,
                                   cudaStream_t s, size_t smem) {
  const CoopCfg c = coop_cfg(ws);
  const int R = ws->R;
  int g = 0;
  cudaError_t e;
  if (op->sigma_identity)
    e = ws->flexible ? coop_launch_d_s1_f1(R, a, c, s, smem, &g) : coop_launch_d_s1_f0(R, a, c, s, smem, &g);
  else
    e = ws->flexible ? coop_launch_d_s0_f1(R, a, c, s, smem, &g) : coop_launch_d_s0_f0(R, a, c, s, smem, &g);
  COUNT_LAUNCH(1);
  return e;
}
static cudaError_t coop_dispatch_z(PArgs<double2> a, sad_gmres* ws, sad_op* op,
                                   cudaStream_t s, size_t smem) {
  const CoopCfg c = coop_cfg(ws);
  const int R = ws->R;
  int g = 0;
  cudaError_t e;
  if (op->vals_complex)
    e = ws->flexible ? coop_launch_zc_s0_f1(R, a, c, s, smem, &g) : coop_launch_zc_s0_f0(R, a, c, s, smem, &g);
  else if (op->sigma_identity)
    e = ws->flexible ? coop_launch_z_s1_f1(R, a, c, s, smem, &g) : coop_launch_z_s1_f0(R, a, c, s, smem, &g);
  else
    e = ws->flexible ? coop_launch_z_s0_f1(R, a, c, s, smem, &g) : coop_launch_z_s0_f0(R, a, c, s, smem, &g);
  COUNT_LAUNCH(1);
  return e;
}

template <typename XT>
static PArgs<XT> make_pargs(sad_gmres* ws, sad_op* op, const void* rhs, void* x) {
  PArgs<XT> a{};
  a.n = ws->n;
  a.rowptr = op->rowptr;
  a.colidx = op->colidx;
  a.vals = op->vals;
  a.dinv = reinterpret_cast<const XT*>(sizeof(XT) == 8 ? (const void*)op->dinv_r
                                                       : (const void*)op->dinv_c);
  a.sigma = op->sigma_eff;
  a.b = reinterpret_cast<const XT*>(rhs);
  a.x = reinterpret_cast<XT*>(x);
  a.V = reinterpret_cast<XT*>(ws->V);
  a.Z = reinterpret_cast<XT*>(ws->Z);
  a.stride = ws->n * ws->R;
  a.st = ws->pst;
  a.prof = ws->profile || ws->timers;
  a.dbg_delay_ns = ws->dbg_delay_ns;
  return a;
}

static double spmm_bytes(const sad_gmres* ws, const sad_op* op, bool arnoldi);

static int persistent_run(sad_gmres* ws, sad_op* op, const void* rhs, void* x, cudaStream_t s,
                          double tol, int maxit, int fixed) {
  sad_ctx* ctx = ws->ctx;
  if (!op || !rhs || !x) return set_err(ctx, SAD_EINVAL, "null argument");
  if (op->n != ws->n)
    return set_err(ctx, SAD_EINVAL, "operator size %lld != workspace size %lld", op->n, ws->n);
  if (ws->dtype == SAD_F64 && !op->real_ok)
    return set_err(ctx, SAD_EINVAL, "complex shift needs a complex128 workspace");
  ws->st.tol = tol;
  ws->st.maxit = maxit;
  ws->st.fixed = fixed;
  ws->pst.g = ws->st;
  ws->pst.spmm_bytes_arn = spmm_bytes(ws, op, true);
  ws->pst.spmm_bytes_res = spmm_bytes(ws, op, false) + (double)ws->n * ws->R * ws->esz;
  CK(ctx, cudaMemsetAsync(ws->pst.bar_count, 0, sizeof(unsigned), s));
  CK(ctx, cudaMemsetAsync(ws->pst.err, 0, sizeof(int), s));
  if (ws->profile) {
    CK(ctx, cudaMemsetAsync(ws->stats_dev, 0, 16 * sizeof(double), s));
    CK(ctx, cudaEventRecord(ws->ev[0], s));
  }
  const size_t m1 = ws->m + 1;
  const size_t R = ws->R;
  // finisher-A staging: sums (2(m+1)+1)R, h1, Gram column, rotations (sn, cs), S,
  // flags, old Gram block
  const size_t finA = ((2 * m1 + 1) * R + 2 * m1 * R + ws->m * R) * 16 + (m1 + ws->m) * R * 8 +
                      8 * 4 + 64;
  const size_t gblk = R * m1 * m1 * 16;
  // SAD_GSMEM_KB caps the staged Gram block (A/B experiments on the L1 carve-out)
  static const size_t gsmem_cap = [] {
    const char* e = getenv("SAD_GSMEM_KB");
    return (size_t)(e && *e ? atoi(e) : 200) * 1024;
  }();
  const bool g_smem = finA + gblk <= gsmem_cap;
  // phase-A TMA stages: one block-tile (kWarps * GPW * UA rows) of one basis block
  const size_t gpw = 32 / R, ua = ws->esz == 8 ? 8 : 4;
  const size_t tile_rows = (size_t)kWarps * gpw * ua;
  // Direct phase A when every block owns at most two tiles even at one block
  // per SM (latency-bound small slabs); else the TMA ring.
  const int sms = ws->max_sms > 0 ? std::min(ws->max_sms, ctx->nsm) : ctx->nsm;
  // direct phase A stages the block's rows of w and v_j in shared memory: an
  // upper bound of the rows per block (the launcher's grid is at least
  // min(n R / (threads * min elems per thread), SMs) blocks)
  // Sized for `bps` blocks per SM: a direct-path block stays within 110 KB, so two
  // are resident per SM and the launcher's grid reaches 2 * SMs blocks -- sizing
  // the rows for one block per SM left no room for the resident CSR slab (config
  // 2's B side on its 22 SMs: 44 blocks of 614 rows, SpMM sub-phase 13 us from L2
  // against 2.5 us from shared memory).  If the occupancy turns out lower the
  // launcher refuses (rows per block > direct_rows) and the sizing is redone for
  // one block per SM.
  // SAD_DIRECT_BPS=1: size for one block per SM from the start (A/B runs, tests)
  int bps = 2;
  if (const char* e = getenv("SAD_DIRECT_BPS")) bps = atoi(e) == 1 ? 1 : 2;
resize:
  const size_t slots = (size_t)sms * bps;
  const size_t rows_cap = std::max<size_t>(
      ((size_t)kThreads * std::max(ws->min_elems_per_thread, 1) + R - 1) / R,
      ((size_t)ws->n + slots - 1) / slots);
  const size_t stage_rows_bytes = 2 * rows_cap * R * ws->esz;
  bool direct = ws->direct_a >= 0 ? ws->direct_a != 0
                                  : (size_t)ws->n <= 2 * tile_rows * slots;
  if (direct && stage_rows_bytes > 96 * 1024) direct = false;   // rows do not fit: TMA ring
  const size_t stage = direct ? 0 : ((tile_rows * R * ws->esz + 32 + 127) & ~size_t(127));
  // s_blk [2(m+1)R] + the ring sweep's per-warp sums (two parity buffers)
  const size_t sums = 2 * m1 * R * ws->esz + (direct ? stage_rows_bytes : 4 * kGroup * kWarps * R * ws->esz);
  // TMA path: the basis ring and the A1 CSR ring share one region
  const size_t vsz = op->vals_complex ? 16 : 8;
  size_t ring_bytes = direct ? 0 : std::max((size_t)kStages * stage,
                                            (size_t)kStagesA1 * a1_stage_bytes((int)R, vsz));
  // large-slab basis sweep: by basis block with direct loads when the block
  // width does not divide the warp (R = 3: config 3 sweep 228 -> 221 us per
  // A-side step, solve -3 %), through the TMA ring otherwise (config 4, R = 8:
  // the ring is 6 % faster; config 5, R = 4 complex: 48.4 s vs 49.8 s);
  // SAD_SWEEP=direct|tma overrides (A/B experiments)
  static const int sweep_env = [] {
    const char* e = getenv("SAD_SWEEP");
    if (!e) return -1;
    return std::string(e) == "tma" ? 0 : 1;
  }();
  // (round 2, with one synchronisation per group in the ring sweep: on blocks of
  // 32 MB and more the ring wins for R = 3 too -- config 3's A side 294 -> 282 us of
  // phase-A work per step, its B side, 23.5 MB, stays with the direct loads)
  const bool small_block = (size_t)ws->n * R * ws->esz < ((size_t)32 << 20);
  const int sweep_direct =
      sweep_env >= 0 ? sweep_env : (((32 % ws->R) != 0 && small_block) ? 1 : 0);
  // Banded plan for the SpMM sub-phase (large slabs): the stages share the ring
  // region; two blocks per SM must still fit, with at least two stages
  const BandPlan* bp = nullptr;
  const void* bdinv = nullptr;
  BandCfg bcfg{};
  static const int band_p_env = [] {
    const char* e = getenv("SAD_BAND_PERSISTENT");
    return e && *e ? atoi(e) : 1;
  }();
  // With the by-basis-block sweep (block widths that do not divide the warp, config 3)
  // w / v_j are read through L1: stages that push two blocks past the 196 KB
  // carve-out (L1 60 -> 28 KB) cost the sweeps 17 %, so there the stages may only
  // use what the kernel's other phases already need (no growth).
  const size_t smem_base = std::max({ring_bytes + sums, R * (m1 * 16 + ws->m * 24),
                                     (size_t)kWarps * ws->m * 16, finA + (g_smem ? gblk : 0)});
  if (!direct && band_p_env && (((size_t)ws->n * R * ws->esz) % 16) == 0) {
    if (const BandPlan* p = op_band(op, 1)) {
      auto al128 = [](size_t b) { return (b + 127) & ~size_t(127); };
      const size_t xb = al128(32 + (size_t)p->xcap * R * ws->esz);
      const size_t db = al128(32 + (size_t)p->xcap * ws->esz);
      const size_t vb = al128((size_t)p->wmax * p->tr * (vsz + 2));   // values + indices
      const size_t sb = xb + db + vb;
      const size_t other = sums;
      // per block: two blocks stay within the 196 KB carve-out (SAD_BAND_CAP_KB: A/B runs)
      static const size_t cap_env = [] {
        const char* e = getenv("SAD_BAND_CAP_KB");
        return (size_t)(e && *e ? atoi(e) : 92) * 1024;
      }();
      const size_t cap = sweep_direct ? std::min(cap_env, smem_base) : cap_env;
      const size_t recs = 2 * 32 * sizeof(BandMeta);   // tile records after the stages
      int S = other + recs < cap ? (int)std::min<size_t>(kBandMaxStages, (cap - other - recs) / sb) : 0;
      static const int s_env = [] {
        const char* e = getenv("SAD_BAND_STAGES_P");
        return e && *e ? atoi(e) : 0;
      }();
      if (s_env > 0) S = std::min(S, s_env);
      const void* dv = S >= 2 ? op_band_dinv(op, 1, ws->dtype == SAD_C128) : nullptr;
      if (S >= 2 && dv) {
        bp = p;
        bdinv = dv;
        bcfg.S = S;
        bcfg.SB = (unsigned)sb;
        bcfg.offD = (unsigned)xb;
        bcfg.offV = (unsigned)(xb + db);
        ring_bytes = std::max(ring_bytes, (size_t)S * sb + recs);
      }
    }
  }
  size_t smem = std::max({ring_bytes + sums,                              // rings + sums
                          R * (m1 * 16 + ws->m * 24),                  // Givens staging
                          (size_t)kWarps * ws->m * 16,                 // back substitution
                          finA + (g_smem ? gblk : 0)});
  // Resident CSR slab (small slabs only, within two blocks' worth of shared
  // memory per SM): placed after everything else; the kernel keeps it only
  // when its own slab fits the budget.
  const size_t csr_off = (smem + 127) & ~size_t(127);
  const size_t per_block_cap = 110 * 1024;
  const size_t csr_budget = (direct && ws->resident_csr && csr_off + 4096 <= per_block_cap)
                                ? per_block_cap - csr_off : 0;
  if (csr_budget) smem = csr_off + csr_budget;
  // (read per launch: the tests switch it inside one process)
  const char* dist_red_s = getenv("SAD_DIST_RED_MIN");
  const int dist_red_env = dist_red_s && *dist_red_s ? atoi(dist_red_s) : 8192;
  static const int ring_c_env = [] {
    const char* e = getenv("SAD_RING_C");
    return e && *e ? atoi(e) : 2;
  }();
  cudaError_t e;
  if (ws->dtype == SAD_F64) {
    PArgs<double> a = make_pargs<double>(ws, op, rhs, x);
    if (bp) {
      a.band_meta = bp->meta;
      a.band_seg = op->band_seg[1];
      a.band_dinv = bdinv;
      a.band_xstride = bp->xstride;
      a.band_tr = bp->tr;
      a.band_cfg = bcfg;
    }
    a.g_smem = g_smem ? 1 : 0;
    a.stage_bytes = (int)stage;
    a.direct_a = direct ? 1 : 0;
    a.direct_rows = (int)rows_cap;
    a.ring_bytes = (int)ring_bytes;
    a.csr_off = (int)csr_off;
    a.csr_budget = (int)csr_budget;
    a.sweep_direct = sweep_direct;
    a.ring_c = ring_c_env;
    a.dist_red_min = dist_red_env;
    e = coop_dispatch_d(a, ws, op, s, smem);
  } else {
    PArgs<double2> a = make_pargs<double2>(ws, op, rhs, x);
    if (bp) {
      a.band_meta = bp->meta;
      a.band_seg = op->band_seg[1];
      a.band_dinv = bdinv;
      a.band_xstride = bp->xstride;
      a.band_tr = bp->tr;
      a.band_cfg = bcfg;
    }
    a.g_smem = g_smem ? 1 : 0;
    a.stage_bytes = (int)stage;
    a.direct_a = direct ? 1 : 0;
    a.direct_rows = (int)rows_cap;
    a.ring_bytes = (int)ring_bytes;
    a.csr_off = (int)csr_off;
    a.csr_budget = (int)csr_budget;
    a.sweep_direct = sweep_direct;
    a.ring_c = ring_c_env;
    a.dist_red_min = dist_red_env;
    e = coop_dispatch_z(a, ws, op, s, smem);
  }
  if (e == cudaErrorInvalidConfiguration && direct && bps == 2) {
    bps = 1;
    goto resize;
  }
  if (e != cudaSuccess)
    return set_err(ctx, SAD_ECUDA, "cooperative GMRES launch failed: %s", cudaGetErrorString(e));
  if (ws->profile) CK(ctx, cudaEventRecord(ws->ev[1], s));
  return SAD_OK;
}

static int persistent_collect(sad_gmres* ws, cudaStream_t s) {
  sad_ctx* ctx = ws->ctx;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_err(ctx, SAD_ECUDA, "persistent GMRES failed: %s", cudaGetErrorString(e));
  if (ws->profile) {
    float ms = 0.f;
    CK(ctx, cudaEventElapsedTime(&ms, ws->ev[0], ws->ev[1]));
    double st[16];
    CK(ctx, cudaMemcpy(st, ws->stats_dev, sizeof(st), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 5; ++i) ws->prof2[i] += st[8 + i] * 1e-6;
    ws->prof[0] += ms;
    ws->prof[1] += 1;
    ws->prof[2] += st[0];
    ws->prof[3] += st[3] * 1e-6;
    ws->prof[4] += st[1];
    ws->prof[5] += st[4] * 1e-6;
    ws->prof[6] += (st[5] + st[6]) * 1e-6;
    ws->prof[7] += st[2];
  }
  return SAD_OK;
}

extern "C" int sad_gmres_set_option(sad_gmres* ws, int key, int value) {
  if (!ws) return SAD_EINVAL;
  switch (key) {
    case SAD_OPT_ENGINE:
      if (value != SAD_ENGINE_MULTI && value != SAD_ENGINE_PERSISTENT)
        return set_err(ws->ctx, SAD_EINVAL, "unknown engine %d", value);
      ws->engine = value;
      return SAD_OK;
    case SAD_OPT_MAX_SMS:
      if (value < 0) return set_err(ws->ctx, SAD_EINVAL, "max_sms must be >= 0");
      ws->max_sms = value;
      return SAD_OK;
    case SAD_OPT_MIN_ELEMS_PER_THREAD:
      if (value < 1) return set_err(ws->ctx, SAD_EINVAL, "min elements per thread must be >= 1");
      ws->min_elems_per_thread = value;
      return SAD_OK;
    case SAD_OPT_RESIDENT_CSR:
      ws->resident_csr = value != 0;
      return SAD_OK;
    case SAD_OPT_DIST_ORTH:
      if (!ws->rsum) return set_err(ws->ctx, SAD_EINVAL, "orthogonalisation option applies to row-partitioned workspaces");
      if (value == 1 && ws->dual_smem > 220 * 1024)
        return set_err(ws->ctx, SAD_EINVAL, "restart too long for the DCGS2 dual dot at this r");
      ws->dist_dcgs2 = value ? 1 : 0;
      return SAD_OK;
    case SAD_OPT_DIRECT_A:
      if (value < -1 || value > 1) return set_err(ws->ctx, SAD_EINVAL, "direct-A option must be -1, 0 or 1");
      ws->direct_a = value;
      return SAD_OK;
    case SAD_OPT_DEBUG_DELAY:
      if (value < 0 || value > 1000000) return set_err(ws->ctx, SAD_EINVAL, "delay must be in [0, 1e6] ns");
      ws->dbg_delay_ns = value;
      return SAD_OK;
  }
  return set_err(ws->ctx, SAD_EINVAL, "unknown option %d", key);
}

extern "C" int sad_gmres_solve(sad_gmres* ws, sad_op* op, const void* rhs, void* x, void* res,
                               double tol_col, int maxit, void* stream, int64_t* iters_host,
                               double* resnorm_host, uint8_t* conv_host) {
  if (!ws) return SAD_EINVAL;
  if (ws->rsum)
    return set_err(ws->ctx, SAD_EINVAL, "row-partitioned workspace: use sad_dist_gmres_solve");
  sad_ctx* ctx = ws->ctx;
  if (!(tol_col > 0.0)) return set_err(ctx, SAD_EINVAL, "abs_tolerance must be positive");
  if (maxit < 0) return set_err(ctx, SAD_EINVAL, "maxit must be >= 0");
  cudaStream_t s = S_(stream);
  if (ws->engine == SAD_ENGINE_PERSISTENT) {
    int rc = persistent_run(ws, op, rhs, x, s, tol_col, maxit, 0);
    if (rc) return rc;
    rc = persistent_collect(ws, s);
    if (rc) return rc;
    return read_results(ws, res, s, iters_host, resnorm_host, conv_host, tol_col);
  }
  Launcher L;
  int rc = prepare(ws, op, rhs, x, s, L);
  if (rc) return rc;
  ws->st.tol = tol_col;
  ws->st.maxit = maxit;
  ws->st.fixed = 0;
  volatile long long* hf = ws->hflag_host;
  for (int i = 0; i < 8; ++i) hf[i] = -1;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  k_init<<<1, 32, 0, s>>>(ws->st);
  COUNT_LAUNCH(1);
  CK(ctx, cudaMemsetAsync(x, 0, (size_t)ws->n * ws->R * ws->esz, s));
  L.residual();
  CKL(ctx);
  long long cycles = 1;
  rc = spin_until(ctx, s, [&] { return hf[2] >= cycles; });
  if (rc) return rc;
  int any = (int)hf[3];
  const int LAG = 3;
  const double N = (double)ws->n * ws->R * ws->esz;   // bytes of one n x r block
  while (any) {
    const long long base = hf[0] < 0 ? 0 : hf[0];
    for (int step = 0; step < ws->m; ++step) {
      if (ws->profile) {
        // synchronous stepping: exact per-kernel-class device times
        if (step > 0 && hf[1] == 0) break;
        CK(ctx, cudaEventRecord(ws->ev[0], s));
        L.arnoldi(0);
        CK(ctx, cudaEventRecord(ws->ev[1], s));
        for (int k = 1; k < 5; ++k) L.arnoldi(k);
        CK(ctx, cudaEventRecord(ws->ev[2], s));
        CK(ctx, cudaEventSynchronize(ws->ev[2]));
        float t1 = 0.f, t2 = 0.f;
        cudaEventElapsedTime(&t1, ws->ev[0], ws->ev[1]);
        cudaEventElapsedTime(&t2, ws->ev[1], ws->ev[2]);
        const double J = step + 1;
        ws->prof[0] += t1;
        ws->prof[1] += 1;
        ws->prof[2] += spmm_bytes(ws, op, true);
        ws->prof[3] += t2;
        ws->prof[4] += 1;
        ws->prof[5] += (4.0 * J + 6.0) * N;
        continue;
      }
      bool stop = false;
      rc = spin_until(ctx, s, [&] {
        long long done = hf[0] - base;
        long long act = hf[1];
        if (done >= 1 && act == 0) { stop = true; return true; }
        return step - done <= LAG;
      });
      if (rc) return rc;
      if (stop) break;
      for (int k = 0; k < 5; ++k) L.arnoldi(k);
    }
    if (ws->profile) CK(ctx, cudaEventRecord(ws->ev[0], s));
    L.cycle_end();
    CKL(ctx);
    ++cycles;
    rc = spin_until(ctx, s, [&] { return hf[2] >= cycles; });
    if (rc) return rc;
    if (ws->profile) {
      CK(ctx, cudaEventRecord(ws->ev[1], s));
      CK(ctx, cudaEventSynchronize(ws->ev[1]));
      float t = 0.f;
      cudaEventElapsedTime(&t, ws->ev[0], ws->ev[1]);
      ws->prof[6] += t;
      ws->prof[7] += 1;
    }
    any = (int)hf[3];
  }
  return read_results(ws, res, s, iters_host, resnorm_host, conv_host, tol_col);
}

extern "C" int sad_gmres_fixed(sad_gmres* ws, sad_op* op, const void* rhs, void* x, void* res,
                               int steps, void* stream, double* resnorm_host, double* timing_ms) {
  if (!ws) return SAD_EINVAL;
  if (ws->rsum)
    return set_err(ws->ctx, SAD_EINVAL, "row-partitioned workspace: use sad_dist_gmres_solve");
  sad_ctx* ctx = ws->ctx;
  if (steps < 1 || steps > ws->m)
    return set_err(ctx, SAD_EINVAL, "steps %d outside 1..restart(%d)", steps, ws->m);
  cudaStream_t s = S_(stream);
  if (ws->engine == SAD_ENGINE_PERSISTENT) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing_ms) {
      CK(ctx, cudaEventCreate(&e0));
      CK(ctx, cudaEventCreate(&e1));
      CK(ctx, cudaMemsetAsync(ws->stats_dev, 0, 16 * sizeof(double), s));
      CK(ctx, cudaEventRecord(e0, s));
    }
    ws->timers = timing_ms ? 1 : 0;
    int rc = persistent_run(ws, op, rhs, x, s, 0.0, steps, 1);
    ws->timers = 0;
    if (rc) return rc;
    if (timing_ms) CK(ctx, cudaEventRecord(e1, s));
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_err(ctx, SAD_ECUDA, "persistent GMRES failed: %s", cudaGetErrorString(e));
    if (timing_ms) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      double st[16];
      CK(ctx, cudaMemcpy(st, ws->stats_dev, sizeof(st), cudaMemcpyDeviceToHost));
      // {kernel_ms, phaseA_ms, phaseC_ms, algorithmic_bytes, spmmA_ms,
      //  cycle_end_ms, arnoldi_steps, 0}
      timing_ms[0] = ms;
      timing_ms[1] = st[3] * 1e-6;
      timing_ms[2] = st[4] * 1e-6;
      timing_ms[3] = st[0];
      timing_ms[4] = st[12] * 1e-6;
      timing_ms[5] = (st[5] + st[6]) * 1e-6;
      timing_ms[6] = st[1];
      timing_ms[7] = 0.0;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    return read_results(ws, res, s, nullptr, resnorm_host, nullptr, 0.0);
  }
  Launcher L;
  int rc = prepare(ws, op, rhs, x, s, L);
  if (rc) return rc;
  ws->st.tol = 0.0;
  ws->st.maxit = steps;
  ws->st.fixed = 1;
  k_init<<<1, 32, 0, s>>>(ws->st);
  COUNT_LAUNCH(1);
  CK(ctx, cudaMemsetAsync(x, 0, (size_t)ws->n * ws->R * ws->esz, s));
  const bool timed = timing_ms != nullptr;
  std::vector<cudaEvent_t> ev;
  auto mark = [&]() {
    if (!timed) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back(e);
  };
  mark();
  L.residual();
  mark();
  for (int step = 0; step < steps; ++step) {
    L.arnoldi(0);
    mark();
    for (int k = 1; k < 5; ++k) L.arnoldi(k);
    mark();
  }
  L.cycle_end();
  mark();
  CKL(ctx);
  CK(ctx, cudaStreamSynchronize(s));
  if (timed) {
    for (int i = 0; i < 4; ++i) timing_ms[i] = 0.0;
    auto el = [&](int a, int b) {
      float t = 0.f;
      cudaEventElapsedTime(&t, ev[a], ev[b]);
      return (double)t;
    };
    timing_ms[3] += el(0, 1);
    for (int step = 0; step < steps; ++step) {
      timing_ms[0] += el(1 + 2 * step, 2 + 2 * step);
      timing_ms[1] += el(2 + 2 * step, 3 + 2 * step);
    }
    timing_ms[2] += el(1 + 2 * steps, 2 + 2 * steps);
    for (auto e : ev) cudaEventDestroy(e);
  }
  return read_results(ws, res, s, nullptr, resnorm_host, nullptr, 0.0);
}

// -----------------------------------------------------------------------------
// block utilities
// -----------------------------------------------------------------------------
template <typename XT>
static void gram_launch(int R, long long n, const void* x, const void* y, double* part,
                        unsigned* ticket, double2* out, int grid, cudaStream_t s) {
  const XT* X = (const XT*)x;
  const XT* Y = (const XT*)y;
  switch (R) {
    case 1: k_gram<XT, 1><<<grid, kThreads, 0, s>>>(n, X, Y, part, ticket, out); break;
    default: break;
    case 2: k_gram<XT, 2><<<grid, kThreads, 0, s>>>(n, X, Y, part, ticket, out); break;
    case 3: k_gram<XT, 3><<<grid, kThreads, 0, s>>>(n, X, Y, part, ticket, out); break;
    case 4: k_gram<XT, 4><<<grid, kThreads, 0, s>>>(n, X, Y, part, ticket, out); break;
    case 5: k_gram<XT, 5><<<grid, kThreads, 0, s>>>(n, X, Y, part, ticket, out); break;
    case 6: k_gram<XT, 6><<<grid, kThreads, 0, s>>>(n, X, Y, part, ticket, out); break;
    case 7: k_gram<XT, 7><<<grid, kThreads, 0, s>>>(n, X, Y, part, ticket, out); break;
    case 8: k_gram<XT, 8><<<grid, kThreads, 0, s>>>(n, X, Y, part, ticket, out); break;
  }
}

extern "C" int sad_gram(sad_ctx* ctx, int64_t n, int r, int dtype, const void* x, const void* y,
                        double* gram_host, void* stream) {
  if (!ctx || !x || !y || !gram_host) return SAD_EINVAL;
  int rc = check_block(ctx, r, dtype);
  if (rc) return rc;
  cudaStream_t s = S_(stream);
  const int grid = grid_for(n, kThreads, ctx->scratch_blocks);
  COUNT_LAUNCH(1);
  if (dtype == SAD_F64)
    gram_launch<double>(r, n, x, y, ctx->scratch, ctx->ticket, ctx->gram_out, grid, s);
  else
    gram_launch<double2>(r, n, x, y, ctx->scratch, ctx->ticket, ctx->gram_out, grid, s);
  CKL(ctx);
  CK(ctx, cudaMemcpyAsync(ctx->gram_host, ctx->gram_out, r * r * sizeof(double2), cudaMemcpyDeviceToHost, s));
  CK(ctx, spin_sync(s));
  std::memcpy(gram_host, ctx->gram_host, r * r * sizeof(double2));
  return SAD_OK;
}

extern "C" int sad_axpy(sad_ctx* ctx, int64_t n, int r, int dtype, double are, double aim,
                        const void* x, void* y, void* stream) {
  if (!ctx || !x || !y) return SAD_EINVAL;
  int rc = check_block(ctx, r, dtype);
  if (rc) return rc;
  if (dtype == SAD_F64 && aim != 0.0) return set_err(ctx, SAD_EINVAL, "complex coefficient on a real block");
  const long long count = n * r;
  const int grid = grid_for(count, 256, ctx->nsm * 16);
  COUNT_LAUNCH(1);
  if (dtype == SAD_F64)
    k_axpy<double><<<grid, 256, 0, S_(stream)>>>(count, make_double2(are, aim), (const double*)x, (double*)y);
  else
    k_axpy<double2><<<grid, 256, 0, S_(stream)>>>(count, make_double2(are, aim), (const double2*)x,
                                                  (double2*)y);
  CKL(ctx);
  return SAD_OK;
}

// -----------------------------------------------------------------------------
// fused ADI step epilogue
// -----------------------------------------------------------------------------
template <typename XT>
static void epi_launch(int R, const EpiArgs<XT>& a, cudaStream_t s) {
  const int grid = a.gA + a.gB;
  switch (R) {
    case 1: k_adi_epilogue<XT, 1><<<grid, kThreads, 0, s>>>(a); break;
    case 2: k_adi_epilogue<XT, 2><<<grid, kThreads, 0, s>>>(a); break;
    case 3: k_adi_epilogue<XT, 3><<<grid, kThreads, 0, s>>>(a); break;
    case 4: k_adi_epilogue<XT, 4><<<grid, kThreads, 0, s>>>(a); break;
    case 5: k_adi_epilogue<XT, 5><<<grid, kThreads, 0, s>>>(a); break;
    case 6: k_adi_epilogue<XT, 6><<<grid, kThreads, 0, s>>>(a); break;
    case 7: k_adi_epilogue<XT, 7><<<grid, kThreads, 0, s>>>(a); break;
    case 8: k_adi_epilogue<XT, 8><<<grid, kThreads, 0, s>>>(a); break;
  }
}

extern "C" int sad_adi_epilogue(sad_ctx* ctx, int64_t nA, int64_t nB, int r, int dtype,
                                double g_re, double g_im, const void* mz, const void* resA,
                                void* w, const void* cty, const void* resB, void* t,
                                double* gram_host, void* stream) {
  if (!ctx || !mz || !resA || !w || !cty || !resB || !t || !gram_host) return SAD_EINVAL;
  int rc = check_block(ctx, r, dtype);
  if (rc) return rc;
  if (dtype == SAD_F64 && g_im != 0.0)
    return set_err(ctx, SAD_EINVAL, "complex step coefficient on a real block");
  const int cap = ctx->nsm * 2;
  const int pT = 2 * cap;
  if (!ctx->epi_part) {
    CK(ctx, cudaMalloc(&ctx->epi_part, (size_t)6 * 64 * pT * sizeof(double2)));
    CK(ctx, cudaMalloc(&ctx->epi_out, 6 * 64 * sizeof(double2)));
    CK(ctx, cudaMallocHost(&ctx->epi_host, 6 * 64 * sizeof(double2)));
  }
  cudaStream_t s = S_(stream);
  auto blocks = [&](long long rows) {
    long long g = (rows + kThreads - 1) / kThreads;
    return (int)std::max(1LL, std::min(g, (long long)cap));
  };
  if (dtype == SAD_F64) {
    EpiArgs<double> a{};
    a.nA = nA; a.nB = nB; a.gA = blocks(nA); a.gB = blocks(nB);
    a.gam = make_double2(g_re, g_im);
    a.mz = (const double*)mz; a.resA = (const double*)resA; a.w = (double*)w;
    a.cty = (const double*)cty; a.resB = (const double*)resB; a.t = (double*)t;
    a.partT = ctx->epi_part; a.pT = pT; a.ticket = ctx->ticket + 1; a.out = ctx->epi_out;
    epi_launch<double>(r, a, s);
  } else {
    EpiArgs<double2> a{};
    a.nA = nA; a.nB = nB; a.gA = blocks(nA); a.gB = blocks(nB);
    a.gam = make_double2(g_re, g_im);
    a.mz = (const double2*)mz; a.resA = (const double2*)resA; a.w = (double2*)w;
    a.cty = (const double2*)cty; a.resB = (const double2*)resB; a.t = (double2*)t;
    a.partT = ctx->epi_part; a.pT = pT; a.ticket = ctx->ticket + 1; a.out = ctx->epi_out;
    epi_launch<double2>(r, a, s);
  }
  COUNT_LAUNCH(1);
  CKL(ctx);
  const size_t bytes = (size_t)6 * r * r * sizeof(double2);
  CK(ctx, cudaMemcpyAsync(ctx->epi_host, ctx->epi_out, bytes, cudaMemcpyDeviceToHost, s));
  CK(ctx, spin_sync(s));
  std::memcpy(gram_host, ctx->epi_host, bytes);
  return SAD_OK;
}

// -----------------------------------------------------------------------------
// split launch / finish (two solves in flight from one host thread)
// -----------------------------------------------------------------------------
extern "C" int sad_gmres_launch(sad_gmres* ws, sad_op* op, const void* rhs, void* x, double tol_col,
                                int maxit, void* stream) {
  if (!ws) return SAD_EINVAL;
  if (ws->rsum)
    return set_err(ws->ctx, SAD_EINVAL, "row-partitioned workspace: use sad_dist_gmres_solve");
  sad_ctx* ctx = ws->ctx;
  if (!(tol_col > 0.0)) return set_err(ctx, SAD_EINVAL, "abs_tolerance must be positive");
  if (maxit < 0) return set_err(ctx, SAD_EINVAL, "maxit must be >= 0");
  ws->pending_tol = tol_col;
  if (ws->engine != SAD_ENGINE_PERSISTENT) {
    // the multi-kernel engine is host-driven: run it to completion here
    ws->pending_multi = 1;
    return sad_gmres_solve(ws, op, rhs, x, nullptr, tol_col, maxit, stream, nullptr, nullptr,
                           nullptr);
  }
  ws->pending_multi = 0;
  return persistent_run(ws, op, rhs, x, S_(stream), tol_col, maxit, 0);
}

extern "C" int sad_gmres_finish(sad_gmres* ws, void* res, void* stream, int64_t* iters_host,
                                double* resnorm_host, uint8_t* conv_host) {
  if (!ws) return SAD_EINVAL;
  cudaStream_t s = S_(stream);
  // profiling needs the launch's events and counters; otherwise the single
  // synchronisation inside read_results also reports a failed launch
  if (!ws->pending_multi && ws->profile) {
    int rc = persistent_collect(ws, s);
    if (rc) return rc;
  }
  return read_results(ws, res, s, iters_host, resnorm_host, conv_host, ws->pending_tol);
}

// -----------------------------------------------------------------------------
// tall-skinny products over the low-rank factors (true_residual_norm's power
// iteration, adi.py:682-726)
// -----------------------------------------------------------------------------
static int ts_reserve(sad_ctx* ctx, size_t part_elems, size_t out_elems) {
  if (part_elems > ctx->ts_part_elems) {
    cudaFree(ctx->ts_part);
    ctx->ts_part = nullptr;
    ctx->ts_part_elems = 0;
    CK(ctx, cudaMalloc(&ctx->ts_part, part_elems * sizeof(double2)));
    ctx->ts_part_elems = part_elems;
  }
  if (out_elems > ctx->ts_elems) {
    cudaFree(ctx->ts_dev);
    if (ctx->ts_host) cudaFreeHost(ctx->ts_host);
    ctx->ts_dev = nullptr;
    ctx->ts_host = nullptr;
    ctx->ts_elems = 0;
    CK(ctx, cudaMalloc(&ctx->ts_dev, out_elems * sizeof(double2)));
    CK(ctx, cudaMallocHost(&ctx->ts_host, out_elems * sizeof(double2)));
    ctx->ts_elems = out_elems;
  }
  return SAD_OK;
}

template <typename XT, int S>
static void ts_hgemv_launch(long long n, long long K, long long ldx, const void* X, const void* V,
                            long long rpb, int CW, int grid, double2* part, cudaStream_t s) {
  k_ts_hgemv<XT, S><<<grid, 256, 0, s>>>(n, K, ldx, (const XT*)X, (const double2*)V, rpb, CW, part);
}

extern "C" int sad_ts_hgemv(sad_ctx* ctx, int64_t n, int64_t K, int64_t ldx, int xdtype,
                            const void* X, int nvec, const void* V, double* out_host,
                            void* stream) {
  if (!ctx || !X || !V || !out_host) return SAD_EINVAL;
  if (n < 1 || K < 1 || ldx < K) return set_err(ctx, SAD_EINVAL, "bad factor shape n=%lld K=%lld ldx=%lld", (long long)n, (long long)K, (long long)ldx);
  if (nvec != 1 && nvec != 2) return set_err(ctx, SAD_EINVAL, "nvec must be 1 or 2");
  if (xdtype != SAD_F64 && xdtype != SAD_C128) return set_err(ctx, SAD_EINVAL, "bad dtype %d", xdtype);
  cudaStream_t s = S_(stream);
  const int CW = (int)std::min<long long>(256, ((K + 31) / 32) * 32);
  const long long min_rows = 64;
  int grid = (int)std::min<long long>((n + min_rows - 1) / min_rows, (long long)ctx->nsm * 4);
  grid = std::max(grid, 1);
  const long long rpb = (n + grid - 1) / grid;
  const size_t nout = (size_t)K * nvec;
  int rc = ts_reserve(ctx, (size_t)grid * nout, nout);
  if (rc) return rc;
  if (xdtype == SAD_F64) {
    if (nvec == 1) ts_hgemv_launch<double, 1>(n, K, ldx, X, V, rpb, CW, grid, ctx->ts_part, s);
    else ts_hgemv_launch<double, 2>(n, K, ldx, X, V, rpb, CW, grid, ctx->ts_part, s);
  } else {
    if (nvec == 1) ts_hgemv_launch<double2, 1>(n, K, ldx, X, V, rpb, CW, grid, ctx->ts_part, s);
    else ts_hgemv_launch<double2, 2>(n, K, ldx, X, V, rpb, CW, grid, ctx->ts_part, s);
  }
  CKL(ctx);
  k_ts_reduce<<<(unsigned)((nout * 32 + 255) / 256), 256, 0, s>>>(ctx->ts_part, grid, (long long)nout, ctx->ts_dev);
  COUNT_LAUNCH(2);
  CKL(ctx);
  CK(ctx, cudaMemcpyAsync(ctx->ts_host, ctx->ts_dev, nout * sizeof(double2), cudaMemcpyDeviceToHost, s));
  CK(ctx, cudaStreamSynchronize(s));
  std::memcpy(out_host, ctx->ts_host, nout * sizeof(double2));
  return SAD_OK;
}

template <typename XT, int S>
static cudaError_t ts_gemv_launch(long long n, long long K, long long ldx, const void* X,
                                  const double2* C, void* Y, int acc, int grid, cudaStream_t s) {
  const size_t smem = (size_t)K * S * sizeof(double2);
  auto kern = k_ts_gemv<XT, S>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<grid, 256, smem, s>>>(n, K, ldx, (const XT*)X, C, (double2*)Y, acc);
  return cudaGetLastError();
}

extern "C" int sad_ts_gemv(sad_ctx* ctx, int64_t n, int64_t K, int64_t ldx, int xdtype,
                           const void* X, int nvec, const double* C_host, void* Y,
                           int accumulate, void* stream) {
  if (!ctx || !X || !C_host || !Y) return SAD_EINVAL;
  if (n < 1 || K < 1 || ldx < K) return set_err(ctx, SAD_EINVAL, "bad factor shape n=%lld K=%lld ldx=%lld", (long long)n, (long long)K, (long long)ldx);
  if (nvec != 1 && nvec != 2) return set_err(ctx, SAD_EINVAL, "nvec must be 1 or 2");
  if (xdtype != SAD_F64 && xdtype != SAD_C128) return set_err(ctx, SAD_EINVAL, "bad dtype %d", xdtype);
  const size_t ncoef = (size_t)K * nvec;
  if (ncoef * sizeof(double2) > 200 * 1024)
    return set_err(ctx, SAD_EINVAL, "K=%lld too large for the staged coefficients", (long long)K);
  cudaStream_t s = S_(stream);
  int rc = ts_reserve(ctx, 0, ncoef);
  if (rc) return rc;
  CK(ctx, cudaStreamSynchronize(s));   // the pinned staging buffer may still be in flight
  std::memcpy(ctx->ts_host, C_host, ncoef * sizeof(double2));
  CK(ctx, cudaMemcpyAsync(ctx->ts_dev, ctx->ts_host, ncoef * sizeof(double2), cudaMemcpyHostToDevice, s));
  const int grid = (int)std::max<long long>(1, std::min<long long>((n + 7) / 8, (long long)ctx->nsm * 8));
  cudaError_t e;
  if (xdtype == SAD_F64)
    e = nvec == 1 ? ts_gemv_launch<double, 1>(n, K, ldx, X, ctx->ts_dev, Y, accumulate, grid, s)
                  : ts_gemv_launch<double, 2>(n, K, ldx, X, ctx->ts_dev, Y, accumulate, grid, s);
  else
    e = nvec == 1 ? ts_gemv_launch<double2, 1>(n, K, ldx, X, ctx->ts_dev, Y, accumulate, grid, s)
                  : ts_gemv_launch<double2, 2>(n, K, ldx, X, ctx->ts_dev, Y, accumulate, grid, s);
  COUNT_LAUNCH(1);
  if (e != cudaSuccess) return set_err(ctx, SAD_ECUDA, "ts_gemv launch failed: %s", cudaGetErrorString(e));
  return SAD_OK;
}

#include "sad_dist.cuh"
#include "sad_precond_host.cuh"
#include "sad_bicg_host.cuh"
#include "sad_minres_host.cuh"
#include "sad_adi_host.cuh"

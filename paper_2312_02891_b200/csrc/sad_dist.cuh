// sad_dist.cuh -- row-partitioned inner solves, included
// at the end of sad_capi.cu (it uses the workspace/operator internals).
//
// One rank owns a contiguous row slab of the shifted operator.  Its local CSR
// has the columns remapped to [local rows | halo rows] (halo = the remote rows
// its rows reference, grouped by owning rank), so every kernel of the
// multi-kernel engine runs unchanged on (n_loc rows, blocks of n_ext rows):
//   * before each SpMM the halo rows of the input block are exchanged
//     (pack kernel + ncclSend/ncclRecv straight into the halo rows);
//   * every reduction of the Arnoldi step ends as a rank sum in st.rsum, is
//     all-reduced (ncclAllReduce, in stream order, no host sync) and finished
//     by k_dist_fin on every rank -- the Hessenberg, Givens rotations and the
//     column masks are replicated, never communicated;
//   * the host stops issuing steps from a per-step progress history that is a
//     deterministic function of the replicated state, so every rank issues the
//     same sequence of collectives.
// Two communicators: NCCL (one process per GPU; libnccl is bound at run time
// with dlopen, normally the copy torch has already loaded), and an in-process
// group that runs P ranks' kernels on one device in rank order with a device
// sum in place of the all-reduce and device copies in place of send/recv (no
// kernel ever waits on another rank's kernel) -- the one-GPU test vehicle.
#pragma once

#include "sad_ring.cuh"
#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  // prefer the copy already in the process (torch's), else the loader path
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.err = std::string("libnccl.so.2 not found: ") + dlerror();
    return api;
  }
#define SAD_NCCL_SYM(field, name)                                        \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));     \
  if (!api.field) {                                                      \
    api.err = std::string("missing NCCL symbol ") + name;                \
    return api;                                                          \
  }
  SAD_NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
  SAD_NCCL_SYM(CommInitRank, "ncclCommInitRank");
  SAD_NCCL_SYM(CommDestroy, "ncclCommDestroy");
  SAD_NCCL_SYM(AllReduce, "ncclAllReduce");
  SAD_NCCL_SYM(Send, "ncclSend");
  SAD_NCCL_SYM(Recv, "ncclRecv");
  SAD_NCCL_SYM(GroupStart, "ncclGroupStart");
  SAD_NCCL_SYM(GroupEnd, "ncclGroupEnd");
  SAD_NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef SAD_NCCL_SYM
  api.ok = true;
  return api;
}

}  // namespace

// ---- delayed-Gram CGS2 (DCGS2) for row-partitioned solves ------------------------
// The persistent kernel's Arnoldi step split at its two grid barriers, with an
// all-reduce at each: one sweep over the basis for h_raw = V^H w, g_raw =
// V^H v_j and ||w||^2 (k_dot_dual), the finisher A math (k_dist_finA: Gram
// column, h1 = S h_raw, c = 2 h1 - G h1, previous rotations), the update
// w -= V S c with ||w||^2 (k_update<UPD_ORTH2>), the new rotation (k_dist_finC).
// The basis is streamed twice per step and there are two all-reduces per step
// (classical CGS2: four sweeps, three all-reduces).
namespace sad {

// rank-sum layout: h_raw [2 J R] at 0, g_raw at 2(m+1)R, ||w||^2 [R] at 4(m+1)R
template <typename XT, int R>
__global__ void __launch_bounds__(kThreads) k_dot_dual(OrthArgs a) {
  constexpr int GPW = 32 / R;
  constexpr int U = 8;
  extern __shared__ double smem_d[];
  if (*a.st.any_active == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  const int j = *a.st.j;
  const int J = j + 1;
  const int m = a.st.m;
  const XT* V = reinterpret_cast<const XT*>(a.V);
  const XT* w = V + (long long)J * a.stride;
  const XT* vj = V + (long long)j * a.stride;
  XT* s_h = reinterpret_cast<XT*>(smem_d);                       // [J][kWarps][R]
  XT* s_g = s_h + (size_t)J * kWarps * R;                        // [J][kWarps][R]
  double* s_w2 = reinterpret_cast<double*>(s_g + (size_t)J * kWarps * R);   // [kWarps][R]
  for (int o = threadIdx.x; o < J * kWarps * R; o += kThreads) {
    s_h[o] = zero<XT>();
    s_g[o] = zero<XT>();
  }
  for (int o = threadIdx.x; o < kWarps * R; o += kThreads) s_w2[o] = 0.0;
  __syncthreads();
  const long long tile_rows = (long long)GPW * U;
  const long long ntiles = (a.n + tile_rows - 1) / tile_rows;
  double w2 = 0.0;
  for (long long t = (long long)blockIdx.x * kWarps + warp; t < ntiles;
       t += (long long)gridDim.x * kWarps) {
    XT wv[U], jv[U];
    long long idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long row = t * tile_rows + u * GPW + grp;
      const bool ok = lane_ok && row < a.n;
      idx[u] = ok ? row * R + c : -1;
      wv[u] = ok ? w[idx[u]] : zero<XT>();
      jv[u] = ok ? vj[idx[u]] : zero<XT>();
      w2 += abs2(wv[u]);
    }
    // two basis blocks per pass: 2U independent loads in flight per lane
    int i = 0;
    for (; i + 1 < J; i += 2) {
      const XT* v0 = V + (long long)i * a.stride;
      const XT* v1 = v0 + a.stride;
      XT a0[U], a1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a0[u] = idx[u] >= 0 ? v0[idx[u]] : zero<XT>();
        a1[u] = idx[u] >= 0 ? v1[idx[u]] : zero<XT>();
      }
      XT ph0 = zero<XT>(), pg0 = zero<XT>(), ph1 = zero<XT>(), pg1 = zero<XT>();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ph0 = cfma(a0[u], wv[u], ph0);
        pg0 = cfma(a0[u], jv[u], pg0);
        ph1 = cfma(a1[u], wv[u], ph1);
        pg1 = cfma(a1[u], jv[u], pg1);
      }
      ph0 = group_reduce<R>(ph0, grp);
      pg0 = group_reduce<R>(pg0, grp);
      ph1 = group_reduce<R>(ph1, grp);
      pg1 = group_reduce<R>(pg1, grp);
      if (grp == 0 && lane_ok) {
        XT* sh = s_h + ((size_t)i * kWarps + warp) * R + c;
        XT* sg = s_g + ((size_t)i * kWarps + warp) * R + c;
        sh[0] = add(sh[0], ph0);
        sg[0] = add(sg[0], pg0);
        sh[kWarps * R] = add(sh[kWarps * R], ph1);
        sg[kWarps * R] = add(sg[kWarps * R], pg1);
      }
    }
    if (i < J) {
      const XT* vi = V + (long long)i * a.stride;
      XT ph = zero<XT>(), pg = zero<XT>();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (idx[u] >= 0) {
          const XT v = vi[idx[u]];
          ph = cfma(v, wv[u], ph);
          pg = cfma(v, jv[u], pg);
        }
      }
      ph = group_reduce<R>(ph, grp);
      pg = group_reduce<R>(pg, grp);
      if (grp == 0 && lane_ok) {
        XT* sh = s_h + ((size_t)i * kWarps + warp) * R + c;
        XT* sg = s_g + ((size_t)i * kWarps + warp) * R + c;
        *sh = add(*sh, ph);
        *sg = add(*sg, pg);
      }
    }
  }
  w2 = group_reduce<R>(w2, grp);
  if (grp == 0 && lane_ok) s_w2[warp * R + c] = w2;
  __syncthreads();
  double* part = a.st.part + (size_t)blockIdx.x * a.st.pstride;
  const int og = 2 * (m + 1) * R, ow = 4 * (m + 1) * R;
  for (int o = threadIdx.x; o < J * R; o += kThreads) {
    const int ii = o / R, cc = o - ii * R;
    XT th = zero<XT>(), tg = zero<XT>();
    for (int wq = 0; wq < kWarps; ++wq) {
      th = add(th, s_h[((size_t)ii * kWarps + wq) * R + cc]);
      tg = add(tg, s_g[((size_t)ii * kWarps + wq) * R + cc]);
    }
    const double2 h2c = to_c(th), g2c = to_c(tg);
    part[2 * o] = h2c.x;
    part[2 * o + 1] = h2c.y;
    part[og + 2 * o] = g2c.x;
    part[og + 2 * o + 1] = g2c.y;
  }
  if (threadIdx.x < R) {
    double t = 0.0;
    for (int wq = 0; wq < kWarps; ++wq) t += s_w2[wq * R + threadIdx.x];
    part[ow + threadIdx.x] = t;
  }
  if (last_block(a.st.ticket)) {
    for (int o = threadIdx.x; o < 2 * J * R; o += kThreads) {
      double sh = 0.0, sg = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) {
        const double* pb = a.st.part + (size_t)b * a.st.pstride;
        sh += __ldcg(pb + o);
        sg += __ldcg(pb + og + o);
      }
      a.st.rsum[o] = sh;
      a.st.rsum[og + o] = sg;
    }
    if (threadIdx.x < R) {
      double t = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b)
        t += __ldcg(a.st.part + (size_t)b * a.st.pstride + ow + threadIdx.x);
      a.st.rsum[ow + threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) *a.st.ticket = 0u;
  }
}

// finisher A on the all-reduced sums (the persistent kernel's finisher A math):
// Gram column, h1, c = 2 h1 - G h1 (into st.h2 for k_update<UPD_ORTH2>, which
// scales by S), ||w_pre||^2, the previous rotations applied to the new column
static __global__ void __launch_bounds__(kThreads) k_dist_finA(GState gs, PState ps) {
  if (*gs.any_active == 0) return;
  const int R = gs.R, m = gs.m;
  const int j = *gs.j, J = j + 1;
  const double* rs = gs.rsum;
  double2* h1 = ps.red;
  double2* gc = ps.red + (size_t)(m + 1) * R;
  double2* cv = ps.coef;
  const int og = 2 * (m + 1) * R, ow = 4 * (m + 1) * R;
  for (int o = threadIdx.x; o < J * R; o += kThreads) {
    const int cc = o - (o / R) * R;
    const double si = gs.S[o], sjj = gs.S[j * R + cc];
    const double2 graw = make_double2(rs[og + 2 * o], rs[og + 2 * o + 1]);
    gc[o] = (si == 0.0 || sjj == 0.0) ? make_double2(0.0, 0.0)
                                      : make_double2(si * sjj * graw.x, si * sjj * graw.y);
    h1[o] = si == 0.0 ? make_double2(0.0, 0.0) : make_double2(si * rs[2 * o], si * rs[2 * o + 1]);
  }
  __syncthreads();
  for (int o = threadIdx.x; o < J * R; o += kThreads) {
    const int ii = o / R, cc = o - ii * R;
    double2 gh0 = make_double2(0.0, 0.0), gh1 = gh0, gh2 = gh0, gh3 = gh0;
    if (ii < j) {
      const double2* Grow = ps.G + (size_t)cc * (m + 1) * (m + 1) + (size_t)ii * (m + 1);
      int l = 0;
      for (; l + 3 < j; l += 4) {
        gh0 = add(gh0, mul(Grow[l], h1[l * R + cc]));
        gh1 = add(gh1, mul(Grow[l + 1], h1[(l + 1) * R + cc]));
        gh2 = add(gh2, mul(Grow[l + 2], h1[(l + 2) * R + cc]));
        gh3 = add(gh3, mul(Grow[l + 3], h1[(l + 3) * R + cc]));
      }
      for (; l < j; ++l) gh0 = add(gh0, mul(Grow[l], h1[l * R + cc]));
    } else {
      for (int l = 0; l < j; ++l) gh0 = add(gh0, mul(cconj(gc[l * R + cc]), h1[l * R + cc]));
    }
    double2 gh = add(add(gh0, gh1), add(gh2, gh3));
    gh = add(gh, mul(gc[ii * R + cc], h1[j * R + cc]));
    const double2 h = h1[o];
    double2 c2 = make_double2(2.0 * h.x - gh.x, 2.0 * h.y - gh.y);
    if (!gs.active[cc]) c2 = make_double2(0.0, 0.0);
    cv[o] = c2;
    gs.h2[o] = c2;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < J * R; o += kThreads) {
    const int ii = o / R, cc = o - ii * R;
    double2* Gc = ps.G + (size_t)cc * (m + 1) * (m + 1);
    Gc[(size_t)ii * (m + 1) + j] = gc[o];
    Gc[(size_t)j * (m + 1) + ii] = cconj(gc[o]);
  }
  if (threadIdx.x < R) {
    const int cc = threadIdx.x;
    gs.wpre2[cc] = rs[ow + cc];
    if (gs.active[cc]) {
      double2 x0 = cv[cc];
      for (int ii = 0; ii < j; ++ii) {
        const double2 x1 = cv[(ii + 1) * R + cc];
        const double ci = gs.cs[(size_t)cc * m + ii];
        const double2 si = gs.sn[(size_t)cc * m + ii];
        gs.H[((size_t)cc * m + j) * (m + 1) + ii] = add(scal(ci, x0), mul(si, x1));
        x0 = sub(scal(ci, x1), mul(cconj(si), x0));
      }
      ps.hc[j * R + cc] = x0;
    }
  }
}

// finisher C: the new rotation from ||w||, the residual estimate, the stopping
// test (the persistent kernel's finisher C), the host-visible progress record
static __global__ void k_dist_finC(GState gs, PState ps) {
  if (*gs.any_active == 0) return;
  const int R = gs.R, m = gs.m;
  const int j = *gs.j;
  __shared__ int s_actn[8];
  if (threadIdx.x < R) {
    const int cc = threadIdx.x;
    s_actn[cc] = 0;
    if (gs.active[cc]) {
      const double hn = sqrt(gs.rsum[cc]);
      double cj; double2 sjv, rj;
      givens(ps.hc[j * R + cc], make_double2(hn, 0.0), cj, sjv, rj);
      gs.cs[(size_t)cc * m + j] = cj;
      gs.sn[(size_t)cc * m + j] = sjv;
      double2* col = gs.H + ((size_t)cc * m + j) * (m + 1);
      col[j] = rj;
      col[j + 1] = make_double2(0.0, 0.0);
      double2* gv = gs.g + (size_t)cc * (m + 1);
      const double2 gj = gv[j];
      const double2 gn = mul(cconj(sjv), gj);
      const double2 gnext = make_double2(-gn.x, -gn.y);
      gv[j + 1] = gnext;
      gv[j] = scal(cj, gj);
      const long long it = gs.iters[cc] + 1;
      gs.iters[cc] = it;
      gs.kdim[cc] = j + 1;
      gs.S[(j + 1) * R + cc] = hn > 0.0 ? 1.0 / hn : 0.0;
      bool end = (j + 1 == m) || it >= gs.maxit;
      if (!gs.fixed) end = end || cabs_(gnext) <= gs.tol || hn <= kLucky * sqrt(gs.wpre2[cc]);
      if (end) gs.active[cc] = 0;
      s_actn[cc] = end ? 0 : 1;
    } else {
      gs.S[(j + 1) * R + cc] = 0.0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int any = 0;
    for (int cc = 0; cc < R; ++cc) any |= s_actn[cc];
    *gs.any_active = any;
    *gs.j = j + 1;
    unsigned long long sq = ++(*gs.stepseq);
    if (gs.hist) gs.hist[j + 1] = (long long)((*gs.cycleseq) << 1) | any;
    gs.hflag[1] = any;
    __threadfence_system();
    gs.hflag[0] = (long long)sq;
  }
}

template <typename XT, int R>
static void dot_dual_launch(const OrthArgs& a, int grid, size_t smem, cudaStream_t s) {
  static size_t attr = 48 * 1024;   // dynamic shared memory opted in so far
  if (smem > attr) {
    if (cudaFuncSetAttribute(k_dot_dual<XT, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) == cudaSuccess)
      attr = smem;
  }
  k_dot_dual<XT, R><<<grid, kThreads, smem, s>>>(a);
}

// ---- the two DCGS2 sweeps through a TMA ring (sad_ring.cuh), large slabs ----
template <typename XT, int R>
static bool ring_launch(const OrthArgs& a, bool dot, int m1, int nsm, bool force, cudaStream_t s) {
  const size_t smem = dot ? ring_dot_smem<XT, R>(m1) : ring_upd_smem<XT, R>(m1);
  if (smem > 110 * 1024) return false;                       // two blocks per SM
  const long long ntiles = (a.n + ring_tile_rows<XT, R>() - 1) / ring_tile_rows<XT, R>();
  if (ntiles < 4LL * nsm && !force) return false;            // small slabs: the direct kernels
  static size_t attr[2] = {0, 0};
  if (smem > attr[dot ? 0 : 1]) {
    const cudaError_t e = dot
        ? cudaFuncSetAttribute(k_dot_dual_ring<XT, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
        : cudaFuncSetAttribute(k_update_ring<XT, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    attr[dot ? 0 : 1] = smem;
  }
  const int grid = (int)std::min<long long>(ntiles, 2LL * nsm);
  if (dot) k_dot_dual_ring<XT, R><<<grid, kThreads, smem, s>>>(a);
  else k_update_ring<XT, R><<<grid, kThreads, smem, s>>>(a);
  return true;
}

// false: not launched (block too small / shared memory), the caller runs the direct kernel
template <typename XT>
static bool ring_sweep(int R, const OrthArgs& a, bool dot, int m1, int nsm, cudaStream_t s) {
  // SAD_DIST_RING: 0 = the direct kernels, 1 (default) = the ring for large slabs,
  // 2 = the ring for every size (tests)
  const char* ev = getenv("SAD_DIST_RING");
  const int env = ev && *ev ? atoi(ev) : 1;
  if (!env) return false;
  const bool force = env > 1;
  switch (R) {
    case 1: return ring_launch<XT, 1>(a, dot, m1, nsm, force, s);
    case 2: return ring_launch<XT, 2>(a, dot, m1, nsm, force, s);
    case 3: return ring_launch<XT, 3>(a, dot, m1, nsm, force, s);
    case 4: return ring_launch<XT, 4>(a, dot, m1, nsm, force, s);
    case 5: return ring_launch<XT, 5>(a, dot, m1, nsm, force, s);
    case 6: return ring_launch<XT, 6>(a, dot, m1, nsm, force, s);
    case 7: return ring_launch<XT, 7>(a, dot, m1, nsm, force, s);
    case 8: return ring_launch<XT, 8>(a, dot, m1, nsm, force, s);
  }
  return false;
}

template <typename XT>
static void dot_dual(int R, const OrthArgs& a, int grid, size_t smem, cudaStream_t s) {
  switch (R) {
    case 1: dot_dual_launch<XT, 1>(a, grid, smem, s); break;
    case 2: dot_dual_launch<XT, 2>(a, grid, smem, s); break;
    case 3: dot_dual_launch<XT, 3>(a, grid, smem, s); break;
    case 4: dot_dual_launch<XT, 4>(a, grid, smem, s); break;
    case 5: dot_dual_launch<XT, 5>(a, grid, smem, s); break;
    case 6: dot_dual_launch<XT, 6>(a, grid, smem, s); break;
    case 7: dot_dual_launch<XT, 7>(a, grid, smem, s); break;
    case 8: dot_dual_launch<XT, 8>(a, grid, smem, s); break;
  }
}

}  // namespace sad

#define NCK(ctx, call)                                                                  \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      return set_err((ctx), SAD_ENCCL, "%s failed: %s", #call,                         \
                     nccl_api().GetErrorString ? nccl_api().GetErrorString(r_) : "?"); \
  } while (0)

struct sad_halo {
  sad_ctx* ctx = nullptr;
  int nranks = 1, rank = 0;
  long long n_loc = 0, n_halo = 0;
  std::vector<long long> send_off, recv_off;   // [nranks + 1] row offsets per peer
  int* d_send_rows = nullptr;                  // local rows to send, grouped by peer
  long long nsend = 0;
  double* sendbuf = nullptr;                   // nsend x (up to 16) doubles
};

struct sad_comm {
  sad_ctx* ctx = nullptr;
  int nranks = 1;
  int rank = 0;             // NCCL rank; 0 for the in-process group
  bool local = false;       // in-process group of `nranks` ranks on ctx's device
  ncclComm_t nc = nullptr;
  double** d_ptrs = nullptr;    // local group: device array of the rank buffers
  double** h_ptrs = nullptr;    // pinned staging for d_ptrs
  int ptr_cap = 0;
};

static constexpr int kHaloMaxWd = 16;   // doubles per row: r <= 8 complex128

extern "C" int sad_comm_unique_id(uint8_t* id_out) {
  if (!id_out) return SAD_EINVAL;
  NcclApi& api = nccl_api();
  if (!api.ok) return SAD_ENCCL;
  ncclUniqueId id;
  if (api.GetUniqueId(&id) != ncclSuccess) return SAD_ENCCL;
  std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return SAD_OK;
}

extern "C" const char* sad_comm_nccl_error(void) {
  NcclApi& api = nccl_api();
  return api.ok ? "" : api.err.c_str();
}

extern "C" int sad_comm_create_nccl(sad_ctx* ctx, int nranks, int rank, const uint8_t* id,
                                    sad_comm** out) {
  if (!ctx || !out || !id) return SAD_EINVAL;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return set_err(ctx, SAD_EINVAL, "rank %d outside 0..%d", rank, nranks - 1);
  NcclApi& api = nccl_api();
  if (!api.ok) return set_err(ctx, SAD_ENCCL, "%s", api.err.c_str());
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  CK(ctx, cudaSetDevice(ctx->device));
  ncclComm_t nc = nullptr;
  NCK(ctx, api.CommInitRank(&nc, nranks, uid, rank));
  sad_comm* c = new sad_comm();
  c->ctx = ctx;
  c->nranks = nranks;
  c->rank = rank;
  c->nc = nc;
  *out = c;
  return SAD_OK;
}

extern "C" int sad_comm_create_local(sad_ctx* ctx, int nranks, sad_comm** out) {
  if (!ctx || !out) return SAD_EINVAL;
  *out = nullptr;
  if (nranks < 1 || nranks > 64) return set_err(ctx, SAD_EINVAL, "local group of %d ranks", nranks);
  sad_comm* c = new sad_comm();
  c->ctx = ctx;
  c->nranks = nranks;
  c->local = true;
  if (cudaMalloc(&c->d_ptrs, 64 * sizeof(double*)) != cudaSuccess ||
      cudaMallocHost(&c->h_ptrs, 64 * sizeof(double*)) != cudaSuccess) {
    cudaFree(c->d_ptrs);
    delete c;
    return set_err(ctx, SAD_ENOMEM, "group pointer table");
  }
  c->ptr_cap = 64;
  *out = c;
  return SAD_OK;
}

extern "C" int sad_comm_destroy(sad_comm* c) {
  if (!c) return SAD_OK;
  if (c->nc) nccl_api().CommDestroy(c->nc);
  cudaFree(c->d_ptrs);
  if (c->h_ptrs) cudaFreeHost(c->h_ptrs);
  delete c;
  return SAD_OK;
}

extern "C" int sad_comm_size(const sad_comm* c) { return c ? c->nranks : 0; }
extern "C" int sad_comm_local_ranks(const sad_comm* c) { return c ? (c->local ? c->nranks : 1) : 0; }

extern "C" int sad_halo_create(sad_ctx* ctx, int nranks, int rank, int64_t n_loc, int64_t n_halo,
                               const int64_t* send_off, const int32_t* send_rows,
                               const int64_t* recv_off, sad_halo** out) {
  if (!ctx || !out || !send_off || !recv_off) return SAD_EINVAL;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return set_err(ctx, SAD_EINVAL, "rank %d outside 0..%d", rank, nranks - 1);
  if (send_off[0] != 0 || recv_off[0] != 0 || recv_off[nranks] != n_halo)
    return set_err(ctx, SAD_EINVAL, "halo offsets inconsistent");
  for (int q = 0; q < nranks; ++q) {
    if (send_off[q + 1] < send_off[q] || recv_off[q + 1] < recv_off[q])
      return set_err(ctx, SAD_EINVAL, "halo offsets not monotone");
    if (q == rank && (send_off[q + 1] != send_off[q] || recv_off[q + 1] != recv_off[q]))
      return set_err(ctx, SAD_EINVAL, "a rank cannot send to itself");
  }
  const long long nsend = send_off[nranks];
  for (long long i = 0; i < nsend; ++i)
    if (send_rows[i] < 0 || send_rows[i] >= n_loc)
      return set_err(ctx, SAD_EINVAL, "send row %d outside the local slab", send_rows[i]);
  sad_halo* h = new sad_halo();
  h->ctx = ctx;
  h->nranks = nranks;
  h->rank = rank;
  h->n_loc = n_loc;
  h->n_halo = n_halo;
  h->send_off.assign(send_off, send_off + nranks + 1);
  h->recv_off.assign(recv_off, recv_off + nranks + 1);
  h->nsend = nsend;
  if (cudaMalloc(&h->d_send_rows, std::max<long long>(nsend, 1) * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&h->sendbuf, std::max<long long>(nsend, 1) * kHaloMaxWd * sizeof(double)) != cudaSuccess) {
    cudaFree(h->d_send_rows);
    delete h;
    return set_err(ctx, SAD_ENOMEM, "halo buffers");
  }
  if (nsend) CK(ctx, cudaMemcpy(h->d_send_rows, send_rows, nsend * sizeof(int), cudaMemcpyHostToDevice));
  *out = h;
  return SAD_OK;
}

extern "C" int sad_halo_destroy(sad_halo* h) {
  if (!h) return SAD_OK;
  cudaFree(h->d_send_rows);
  cudaFree(h->sendbuf);
  delete h;
  return SAD_OK;
}

// local CSR of a row slab: columns already remapped to [local | halo]; the
// per-row order is the global matrix's (so row sums accumulate in the same
// order as on one GPU), which is not increasing after the remap.
extern "C" int sad_local_csr_create(sad_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz,
                                    const int32_t* rowptr, const int32_t* colidx,
                                    const double* vals, sad_csr** out) {
  if (!ctx || !out) return SAD_EINVAL;
  *out = nullptr;
  if (nrows < 0 || ncols < nrows || nnz < 0 || nnz > 2147483647LL || !rowptr)
    return set_err(ctx, SAD_EINVAL, "bad local CSR sizes");
  if (rowptr[0] != 0 || rowptr[nrows] != nnz)
    return set_err(ctx, SAD_EINVAL, "row offsets inconsistent with nnz");
  for (int64_t i = 0; i < nrows; ++i) {
    if (rowptr[i + 1] < rowptr[i]) return set_err(ctx, SAD_EINVAL, "row offsets not monotone");
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      if (colidx[k] < 0 || colidx[k] >= ncols)
        return set_err(ctx, SAD_EINVAL, "column index out of range in row %lld", (long long)i);
      if (!std::isfinite(vals[k])) return set_err(ctx, SAD_EINVAL, "non-finite matrix entry");
    }
  }
  sad_csr* c = new sad_csr();
  c->ctx = ctx;
  c->uid = g_op_uid.fetch_add(1);
  c->nrows = nrows;
  c->ncols = ncols;
  c->nnz = nnz;
  // host copies: the banded SpMM plan of the slab pattern is built from them
  c->h_rowptr.assign(rowptr, rowptr + nrows + 1);
  c->h_colidx.assign(colidx, colidx + nnz);
  c->h_vals.assign(vals, vals + nnz);
  int rc = upload_csr(ctx, c->d, c->h_rowptr, c->h_colidx, c->h_vals);
  if (rc != SAD_OK) {
    free_csr(ctx, c->d);
    delete c;
    return rc;
  }
  *out = c;
  return SAD_OK;
}

// Op = base_local + sigma I on a row slab (identity mass; the B side passes the
// slab of B^T and conj(sigma)).  dinv covers [local | halo]: the local part is
// computed here, the halo part by sad_dist_op_setup.
extern "C" int sad_local_op_create(sad_ctx* ctx, const sad_csr* base, double sre, double sim,
                                   int precond_kind, sad_op** out) {
  if (!ctx || !base || !out) return SAD_EINVAL;
  *out = nullptr;
  if (precond_kind != SAD_PRECOND_NONE && precond_kind != SAD_PRECOND_JACOBI)
    return set_err(ctx, SAD_EINVAL, "unknown preconditioner kind %d", precond_kind);
  sad_op* op = new sad_op();
  op->ctx = ctx;
  op->uid = g_op_uid.fetch_add(1);
  op->n = base->nrows;
  op->ncols = base->ncols;
  op->precond = precond_kind;
  // banded plan of the slab pattern ([local | halo] columns: the halo rows of x
  // are one or two more ranges per tile), on first use
  op->base_csr = base;
  op->band_ok = band_wanted(base->nnz);
  op->sigma_eff = make_double2(sre, sim);
  op->rowptr = base->d.rowptr;
  op->colidx = base->d.colidx;
  op->vals = base->d.vals;
  op->nnz = base->nnz;
  op->vals_complex = false;
  op->sigma_identity = true;
  op->real_ok = (sim == 0.0);
  const size_t nn = (size_t)std::max<long long>(op->ncols, 1);
  char* dbuf = nullptr;
  CK(ctx, ctx_malloc(ctx, (void**)&dbuf, nn * sizeof(double2) + nn * sizeof(double) + 256));
  op->dinv_c = reinterpret_cast<double2*>(dbuf);
  op->dinv_r = reinterpret_cast<double*>(dbuf + ((nn * sizeof(double2) + 255) & ~size_t(255)));
  CK(ctx, cudaMemset(op->dinv_c, 0, nn * sizeof(double2)));
  int* d_bd = reinterpret_cast<int*>(ctx->ticket + 8);
  CK(ctx, cudaMemsetAsync(d_bd, 0, sizeof(int), 0));
  const long long n = op->n;
  const int blocks = grid_for(n, 256, ctx->nsm * 16);
  if (precond_kind == SAD_PRECOND_JACOBI) {
    k_jacobi<double><<<blocks, 256>>>(n, op->rowptr, op->colidx, (const double*)op->vals,
                                      op->sigma_eff, 1, op->dinv_c, d_bd);
  } else {
    std::vector<double2> ones(nn, make_double2(1.0, 0.0));
    CK(ctx, cudaMemcpy(op->dinv_c, ones.data(), nn * sizeof(double2), cudaMemcpyHostToDevice));
  }
  COUNT_LAUNCH(1);
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

// ---- collectives over the local ranks of this process ------------------------
// `nl` local ranks: 1 for NCCL (this process's rank), nranks for a local group.
static int check_nl(sad_comm* cm, int nl) {
  const int want = cm->local ? cm->nranks : 1;
  if (nl != want) return set_err(cm->ctx, SAD_EINVAL, "%d local ranks given, communicator has %d", nl, want);
  return SAD_OK;
}

static int group_ptrs(sad_comm* cm, double* const* bufs, int nl, cudaStream_t s) {
  for (int i = 0; i < nl; ++i) cm->h_ptrs[i] = bufs[i];
  CK(cm->ctx, cudaMemcpyAsync(cm->d_ptrs, cm->h_ptrs, nl * sizeof(double*), cudaMemcpyHostToDevice, s));
  // the pinned table is rewritten by the next call: wait for the copy
  CK(cm->ctx, cudaStreamSynchronize(s));
  return SAD_OK;
}

// sum over ranks, in place; for the local group `ptrs_ready` says d_ptrs
// already holds `bufs` (the solve loop sets it once)
static int allreduce(sad_comm* cm, double* const* bufs, int nl, int count, cudaStream_t s,
                     bool ptrs_ready) {
  if (cm->local) {
    if (!ptrs_ready) {
      int rc = group_ptrs(cm, bufs, nl, s);
      if (rc) return rc;
    }
    k_group_sum<<<std::max(1, std::min(64, (count + 255) / 256)), 256, 0, s>>>(cm->d_ptrs, nl, count);
    COUNT_LAUNCH(1);
    CKL(cm->ctx);
    return SAD_OK;
  }
  NCK(cm->ctx, nccl_api().AllReduce(bufs[0], bufs[0], (size_t)count, ncclDouble, ncclSum, cm->nc, s));
  return SAD_OK;
}

// fill the halo rows of each local rank's block (n_ext x wd doubles)
static int halo_exchange(sad_comm* cm, sad_halo* const* H, char* const* blocks, int nl, int wd,
                         cudaStream_t s) {
  sad_ctx* ctx = cm->ctx;
  if (wd < 1 || wd > kHaloMaxWd) return set_err(ctx, SAD_EINVAL, "halo row width %d", wd);
  for (int i = 0; i < nl; ++i) {
    if (H[i]->nsend == 0) continue;
    const long long tot = H[i]->nsend * wd;
    const int g = (int)std::max(1LL, std::min((tot + 255) / 256, (long long)ctx->nsm * 8));
    k_halo_pack<<<g, 256, 0, s>>>(reinterpret_cast<const double*>(blocks[i]), wd, H[i]->d_send_rows,
                                  H[i]->nsend, H[i]->sendbuf);
    COUNT_LAUNCH(1);
  }
  CKL(ctx);
  const size_t row_bytes = (size_t)wd * sizeof(double);
  if (cm->local) {
    for (int p = 0; p < nl; ++p)
      for (int q = 0; q < nl; ++q) {
        if (p == q) continue;
        const long long cnt = H[p]->send_off[q + 1] - H[p]->send_off[q];
        if (!cnt) continue;
        if (H[q]->recv_off[p + 1] - H[q]->recv_off[p] != cnt)
          return set_err(ctx, SAD_EINVAL, "halo plans of ranks %d and %d disagree", p, q);
        char* dst = blocks[q] + (size_t)(H[q]->n_loc + H[q]->recv_off[p]) * row_bytes;
        const double* src = H[p]->sendbuf + (size_t)H[p]->send_off[q] * wd;
        CK(ctx, cudaMemcpyAsync(dst, src, (size_t)cnt * row_bytes, cudaMemcpyDeviceToDevice, s));
      }
    return SAD_OK;
  }
  NcclApi& api = nccl_api();
  sad_halo* h = H[0];
  NCK(ctx, api.GroupStart());
  for (int q = 0; q < cm->nranks; ++q) {
    if (q == cm->rank) continue;
    const long long ns = h->send_off[q + 1] - h->send_off[q];
    const long long nr = h->recv_off[q + 1] - h->recv_off[q];
    if (ns) NCK(ctx, api.Send(h->sendbuf + (size_t)h->send_off[q] * wd, (size_t)ns * wd, ncclDouble, q, cm->nc, s));
    if (nr) NCK(ctx, api.Recv(blocks[0] + (size_t)(h->n_loc + h->recv_off[q]) * row_bytes,
                              (size_t)nr * wd, ncclDouble, q, cm->nc, s));
  }
  NCK(ctx, api.GroupEnd());
  return SAD_OK;
}

extern "C" int sad_dist_allreduce(sad_comm* cm, int nl, double* const* bufs, int64_t count, void* stream) {
  if (!cm || !bufs || count < 0) return SAD_EINVAL;
  int rc = check_nl(cm, nl);
  if (rc) return rc;
  if (count == 0) return SAD_OK;
  return allreduce(cm, bufs, nl, (int)count, S_(stream), false);
}

extern "C" int sad_dist_halo_exchange(sad_comm* cm, int nl, sad_halo* const* halos, void* const* blocks,
                                      int r, int dtype, void* stream) {
  if (!cm || !halos || !blocks) return SAD_EINVAL;
  int rc = check_nl(cm, nl);
  if (rc) return rc;
  rc = check_block(cm->ctx, r, dtype);
  if (rc) return rc;
  const int wd = r * (dtype == SAD_F64 ? 1 : 2);
  return halo_exchange(cm, halos, reinterpret_cast<char* const*>(blocks), nl, wd, S_(stream));
}

// dinv of the halo rows from their owners (once per operator)
extern "C" int sad_dist_op_setup(sad_comm* cm, int nl, sad_op* const* ops, sad_halo* const* halos,
                                 void* stream) {
  if (!cm || !ops || !halos) return SAD_EINVAL;
  int rc = check_nl(cm, nl);
  if (rc) return rc;
  cudaStream_t s = S_(stream);
  std::vector<char*> blocks(nl);
  for (int i = 0; i < nl; ++i) {
    if (ops[i]->n != halos[i]->n_loc || ops[i]->ncols != halos[i]->n_loc + halos[i]->n_halo)
      return set_err(cm->ctx, SAD_EINVAL, "operator slab and halo plan disagree on rank %d", i);
    blocks[i] = reinterpret_cast<char*>(ops[i]->dinv_c);
  }
  rc = halo_exchange(cm, halos, blocks.data(), nl, 2, s);
  if (rc) return rc;
  for (int i = 0; i < nl; ++i) {
    const long long n = ops[i]->ncols;
    k_c2r<<<grid_for(n, 256, cm->ctx->nsm * 16), 256, 0, s>>>(n, ops[i]->dinv_c, ops[i]->dinv_r);
    COUNT_LAUNCH(1);
  }
  CKL(cm->ctx);
  CK(cm->ctx, cudaStreamSynchronize(s));
  return SAD_OK;
}

// y = Op x on every local rank; x blocks are n_ext rows (halo rows overwritten)
extern "C" int sad_dist_op_apply(sad_comm* cm, int nl, sad_op* const* ops, sad_halo* const* halos,
                                 int r, int dtype, void* const* x_ext, void* const* y, void* stream) {
  if (!cm || !ops || !halos || !x_ext || !y) return SAD_EINVAL;
  int rc = sad_dist_halo_exchange(cm, nl, halos, x_ext, r, dtype, stream);
  if (rc) return rc;
  for (int i = 0; i < nl; ++i) {
    rc = op_spmm<SPMM_APPLY>(ops[i], r, dtype, nullptr, x_ext[i], y[i], stream);
    if (rc) return rc;
  }
  return SAD_OK;
}

extern "C" int sad_dist_gmres_create(sad_ctx* ctx, int64_t n_loc, int64_t n_ext, int r, int dtype,
                                     int restart, int flexible, sad_gmres** out) {
  int rc = gmres_create(ctx, n_loc, n_ext, r, dtype, restart, flexible, out);
  if (rc) return rc;
  sad_gmres* ws = *out;
  ws->engine = SAD_ENGINE_MULTI;
  ws->dist_dcgs2 = 1;
  ws->dual_smem = 2 * (size_t)(restart + 1) * kWarps * r * ws->esz + kWarps * r * 8;
  if (ws->dual_smem > 220 * 1024) ws->dist_dcgs2 = 0;   // CGS2 (single-dot smem) instead
  const size_t xb = (size_t)n_ext * r * ws->esz;
  if (ctx_malloc(ctx, &ws->xext, xb) != cudaSuccess ||
      ctx_malloc(ctx, (void**)&ws->rsum, (size_t)ws->pstride * sizeof(double)) != cudaSuccess ||
      cudaHostAlloc(&ws->hist_host, (size_t)(restart + 2) * sizeof(long long), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&ws->hist_dev, ws->hist_host, 0) != cudaSuccess) {
    sad_gmres_destroy(ws);
    *out = nullptr;
    return set_err(ctx, SAD_ENOMEM, "row-partitioned workspace allocation failed");
  }
  cudaMemset(ws->rsum, 0, (size_t)ws->pstride * sizeof(double));
  ws->st.rsum = ws->rsum;
  ws->st.hist = reinterpret_cast<volatile long long*>(ws->hist_dev);
  ws->bytes += (int64_t)xb;
  return SAD_OK;
}

template <int MODE>
static void dist_fin(sad_gmres* const* W, int nl, cudaStream_t s) {
  for (int i = 0; i < nl; ++i) k_dist_fin<MODE><<<1, kThreads, 0, s>>>(W[i]->st);
  COUNT_LAUNCH(nl);
}

// Row-partitioned Jacobi-GMRES(m)/FGMRES(m): the multi-kernel engine's step
// sequence on every local rank, with halo exchanges before the SpMMs and an
// all-reduce between each reduction and its finisher.  Same contract as
// sad_gmres_solve; iteration counts, residual norms and
// convergence flags are replicated (the values of local rank 0 are returned).
extern "C" int sad_dist_gmres_solve(sad_comm* cm, int nl, sad_gmres* const* W, sad_op* const* O,
                                    sad_halo* const* H, const void* const* rhs, void* const* x,
                                    void* const* res, double tol_col, int maxit, void* stream,
                                    int64_t* iters_host, double* resnorm_host, uint8_t* conv_host) {
  if (!cm || !W || !O || !H || !rhs || !x) return SAD_EINVAL;
  sad_ctx* ctx = cm->ctx;
  int rc = check_nl(cm, nl);
  if (rc) return rc;
  if (!(tol_col > 0.0)) return set_err(ctx, SAD_EINVAL, "abs_tolerance must be positive");
  if (maxit < 0) return set_err(ctx, SAD_EINVAL, "maxit must be >= 0");
  cudaStream_t s = S_(stream);
  const int R = W[0]->R, m = W[0]->m;
  std::vector<Launcher> L(nl);
  for (int i = 0; i < nl; ++i) {
    sad_gmres* ws = W[i];
    if (!ws->rsum || !ws->hist_host)
      return set_err(ctx, SAD_EINVAL, "workspace %d was not created by sad_dist_gmres_create", i);
    if (ws->R != R || ws->m != m || ws->dtype != W[0]->dtype || ws->flexible != W[0]->flexible)
      return set_err(ctx, SAD_EINVAL, "workspaces of the ranks disagree");
    if (H[i]->n_loc != ws->n || H[i]->n_loc + H[i]->n_halo != ws->n_ext || O[i]->ncols != ws->n_ext)
      return set_err(ctx, SAD_EINVAL, "rank %d: workspace, operator and halo plan disagree", i);
    rc = prepare(ws, O[i], rhs[i], ws->xext, s, L[i]);
    if (rc) return rc;
    ws->st.tol = tol_col;
    ws->st.maxit = maxit;
    ws->st.fixed = 0;
    for (int k = 0; k < m + 2; ++k) ws->hist_host[k] = -1;
  }
  const int wd = R * (int)(W[0]->esz / 8);
  // bytes of one n_ext-row block; slabs differ in size from rank to rank
  auto blk_bytes = [&](int i) { return (size_t)W[i]->n_ext * R * W[i]->esz; };
  std::vector<double*> rs(nl);
  for (int i = 0; i < nl; ++i) rs[i] = W[i]->rsum;
  if (cm->local) {
    rc = group_ptrs(cm, rs.data(), nl, s);
    if (rc) return rc;
  }
  const int cnt_dot = 2 * (m + 1) * R + R;
  const int cnt_dual = 4 * (m + 1) * R + R;
  const bool dcgs2 = W[0]->dist_dcgs2 != 0;
  for (int i = 0; i < nl; ++i)
    if ((W[i]->dist_dcgs2 != 0) != dcgs2)
      return set_err(ctx, SAD_EINVAL, "ranks disagree on the orthogonalisation");
  if (dcgs2) {
    // the persistent pieces of the workspace must see this solve's state
    for (int i = 0; i < nl; ++i) W[i]->pst.g = W[i]->st;
  }
  auto AR = [&](int count) { return allreduce(cm, rs.data(), nl, count, s, true); };
  auto blocks_of = [&](int j, std::vector<char*>& b) {
    b.resize(nl);
    for (int i = 0; i < nl; ++i) b[i] = reinterpret_cast<char*>(W[i]->V) + (size_t)j * blk_bytes(i);
  };
  std::vector<char*> xb(nl), vb;
  for (int i = 0; i < nl; ++i) xb[i] = reinterpret_cast<char*>(W[i]->xext);
  volatile long long* hf = W[0]->hflag_host;
  volatile long long* hist = W[0]->hist_host;
  for (int k = 0; k < 8; ++k) hf[k] = -1;
  std::atomic_thread_fence(std::memory_order_seq_cst);

  auto cycle_residual = [&]() -> int {
    int e = halo_exchange(cm, H, xb.data(), nl, wd, s);
    if (e) return e;
    for (int i = 0; i < nl; ++i) L[i].residual();
    CKL(ctx);
    e = AR(R);
    if (e) return e;
    dist_fin<FIN_CYCLE>(W, nl, s);
    CKL(ctx);
    return SAD_OK;
  };

  for (int i = 0; i < nl; ++i) {
    k_init<<<1, 32, 0, s>>>(W[i]->st);
    COUNT_LAUNCH(1);
    CK(ctx, cudaMemsetAsync(W[i]->xext, 0, blk_bytes(i), s));
  }
  rc = cycle_residual();
  if (rc) return rc;
  long long cycles = 1;
  rc = spin_until(ctx, s, [&] { return hf[2] >= cycles; });
  if (rc) return rc;
  int any = (int)hf[3];
  const int LAG = 3;
  while (any) {
    for (int step = 0; step < m; ++step) {
      if (step > LAG) {
        // stop decision from the replicated history of step (step - LAG - 1):
        // the same on every rank, so every rank issues the same collectives
        const int hi = step - LAG;
        rc = spin_until(ctx, s, [&] { return hist[hi] >= 0 && (hist[hi] >> 1) == cycles; });
        if (rc) return rc;
        if ((hist[hi] & 1) == 0) break;
      }
      blocks_of(step, vb);
      rc = halo_exchange(cm, H, vb.data(), nl, wd, s);
      if (rc) return rc;
      for (int i = 0; i < nl; ++i) L[i].arnoldi(0);       // SpMM
      if (dcgs2) {
        // DCGS2: one dual dot sweep, finisher A, one update sweep, finisher C
        for (int i = 0; i < nl; ++i) {
          const OrthArgs oa = L[i].orth_args();
          const int m1 = W[i]->m + 1;
          if (W[i]->dtype == SAD_F64) {
            if (!ring_sweep<double>(R, oa, true, m1, ctx->nsm, s))
              dot_dual<double>(R, oa, L[i].grid_dot, W[i]->dual_smem, s);
          } else if (!ring_sweep<double2>(R, oa, true, m1, ctx->nsm, s)) {
            dot_dual<double2>(R, oa, L[i].grid_dot, W[i]->dual_smem, s);
          }
        }
        COUNT_LAUNCH(nl);
        if ((rc = AR(cnt_dual))) return rc;
        for (int i = 0; i < nl; ++i) k_dist_finA<<<1, kThreads, 0, s>>>(W[i]->st, W[i]->pst);
        COUNT_LAUNCH(nl);
        for (int i = 0; i < nl; ++i) {                    // w -= V S c, ||w||^2
          const OrthArgs oa = L[i].orth_args();
          const int m1 = W[i]->m + 1;
          const bool ringed = W[i]->dtype == SAD_F64 ? ring_sweep<double>(R, oa, false, m1, ctx->nsm, s)
                                                     : ring_sweep<double2>(R, oa, false, m1, ctx->nsm, s);
          if (ringed) COUNT_LAUNCH(1);
          else L[i].arnoldi(4);
        }
        if ((rc = AR(R))) return rc;
        for (int i = 0; i < nl; ++i) k_dist_finC<<<1, 32, 0, s>>>(W[i]->st, W[i]->pst);
        COUNT_LAUNCH(nl);
        CKL(ctx);
        continue;
      }
      for (int i = 0; i < nl; ++i) L[i].arnoldi(1);       // pass-1 dots
      if ((rc = AR(cnt_dot))) return rc;
      dist_fin<FIN_DOT1>(W, nl, s);
      for (int i = 0; i < nl; ++i) L[i].arnoldi(2);       // pass-1 update
      for (int i = 0; i < nl; ++i) L[i].arnoldi(3);       // pass-2 dots
      if ((rc = AR(cnt_dot))) return rc;
      dist_fin<FIN_DOT2>(W, nl, s);
      for (int i = 0; i < nl; ++i) L[i].arnoldi(4);       // pass-2 update + norms
      if ((rc = AR(R))) return rc;
      dist_fin<FIN_GIVENS>(W, nl, s);
      CKL(ctx);
    }
    for (int i = 0; i < nl; ++i) {
      k_trisolve<<<1, 32, 0, s>>>(W[i]->st, W[i]->flexible);
      COUNT_LAUNCH(1);
      const OrthArgs oa = L[i].orth_args();
      if (W[i]->dtype == SAD_F64) orth_upd<double>(R, oa, W[i]->flexible ? UPD_XF : UPD_X, L[i].grid_upd, L[i].usm, s);
      else orth_upd<double2>(R, oa, W[i]->flexible ? UPD_XF : UPD_X, L[i].grid_upd, L[i].usm, s);
    }
    CKL(ctx);
    rc = cycle_residual();
    if (rc) return rc;
    ++cycles;
    rc = spin_until(ctx, s, [&] { return hf[2] >= cycles; });
    if (rc) return rc;
    any = (int)hf[3];
  }
  for (int i = 0; i < nl; ++i)
    CK(ctx, cudaMemcpyAsync(x[i], W[i]->xext, (size_t)W[i]->n * R * W[i]->esz, cudaMemcpyDeviceToDevice, s));
  for (int i = 0; i < nl; ++i) {
    rc = read_results(W[i], res ? res[i] : nullptr, s, i == 0 ? iters_host : nullptr,
                      i == 0 ? resnorm_host : nullptr, i == 0 ? conv_host : nullptr, tol_col);
    if (rc) return rc;
  }
  return SAD_OK;
}

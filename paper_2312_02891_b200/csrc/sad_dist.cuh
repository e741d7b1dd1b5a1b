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
  c->nrows = nrows;
  c->ncols = ncols;
  c->nnz = nnz;
  std::vector<int> rp(rowptr, rowptr + nrows + 1), ci(colidx, colidx + nnz);
  std::vector<double> v(vals, vals + nnz);
  int rc = upload_csr(ctx, c->d, rp, ci, v);
  if (rc != SAD_OK) {
    free_csr(c->d);
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
  CK(ctx, cudaMalloc(&dbuf, nn * sizeof(double2) + nn * sizeof(double) + 256));
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
  const size_t xb = (size_t)n_ext * r * ws->esz;
  if (cudaMalloc(&ws->xext, xb) != cudaSuccess ||
      cudaMalloc(&ws->rsum, (size_t)ws->pstride * sizeof(double)) != cudaSuccess ||
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

// libdbm C ABI (include/dbm.h): contexts, blocked matrices, the Cannon multiply driver
// (§II) with the densified (§III) and blocked (§II) local paths.
//
// Runtime model: one process per GPU; the compute stream is the caller's (torch's)
// stream; a second "comm" stream carries NCCL grouped send/recv of Cannon panels so the fetch of
// step s+1 overlaps the local multiply of step s; CUDA events order the two streams.
#include <cstdio>
#include <mutex>

#include "api_internal.h"

namespace dbm {
static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }

int num_sms() {
  static int n = 0;
  if (n <= 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

}  // namespace dbm

using namespace dbm;


namespace {

uint64_t next_serial() {
  static std::mutex mu;
  static uint64_t n = 0;
  std::lock_guard<std::mutex> g(mu);
  return ++n;
}

}  // namespace

cudaEvent_t dbm::get_event(dbm_ctx ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return e;
}



// ====================================================================== misc
extern "C" const char* dbm_status_string(dbm_status s) {
  switch (s) {
    case DBM_OK: return "DBM_OK";
    case DBM_ERR_ARG: return "DBM_ERR_ARG";
    case DBM_ERR_SHAPE: return "DBM_ERR_SHAPE";
    case DBM_ERR_RANGE: return "DBM_ERR_RANGE";
    case DBM_ERR_PARTITION: return "DBM_ERR_PARTITION";
    case DBM_ERR_PLAN: return "DBM_ERR_PLAN";
    case DBM_ERR_OWNERSHIP: return "DBM_ERR_OWNERSHIP";
    case DBM_ERR_ALIAS: return "DBM_ERR_ALIAS";
    case DBM_ERR_GRID: return "DBM_ERR_GRID";
    case DBM_ERR_WORKSPACE: return "DBM_ERR_WORKSPACE";
    case DBM_ERR_CUDA: return "DBM_ERR_CUDA";
    case DBM_ERR_NCCL: return "DBM_ERR_NCCL";
    case DBM_ERR_NOMEM: return "DBM_ERR_NOMEM";
  }
  return "DBM_ERR_UNKNOWN";
}

extern "C" const char* dbm_last_error(void) { return g_err.c_str(); }

extern "C" int dbm_unique_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

extern "C" dbm_status dbm_get_unique_id(void* id_out) {
  ARG_CHECK(id_out, DBM_ERR_ARG, "null id buffer");
  ncclUniqueId id;
  NCCL_TRY((dbm_ctx) nullptr, ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return DBM_OK;
}

// ====================================================================== context
extern "C" dbm_status dbm_ctx_create(int nranks, int rank, int pr, int pc, const void* id, int device,
                                     void* cuda_stream, dbm_ctx* out) {
  ARG_CHECK(out, DBM_ERR_ARG, "null output handle");
  ARG_CHECK(nranks >= 1 && rank >= 0 && rank < nranks, DBM_ERR_ARG, "bad nranks/rank");
  ARG_CHECK(pr >= 0 && pc >= 0, DBM_ERR_ARG, "negative grid");
  if (pr == 0 && pc == 0) {  // reading R1: largest divisor <= sqrt(P) rows
    int best = 1;
    for (int d = 1; (int64_t)d * d <= nranks; ++d)
      if (nranks % d == 0) best = d;
    pr = best;
    pc = nranks / best;
  }
  ARG_CHECK(pr * pc == nranks, DBM_ERR_GRID, "pr*pc != nranks");
  ARG_CHECK(nranks == 1 || id != nullptr, DBM_ERR_ARG, "multi-rank context needs an NCCL unique id");
  dbm_ctx ctx = new dbm_ctx_s();
  ctx->nranks = nranks;
  ctx->rank = rank;
  ctx->pr = pr;
  ctx->pc = pc;
  ctx->myrow = rank / pc;
  ctx->mycol = rank % pc;
  ctx->device = device;
  if (const char* hp = getenv("DBM_HOST_PIPE")) ctx->host_pipe = *hp != '0';  // measurement override
  if (const char* dp = getenv("DBM_DEV_PIPE")) ctx->dev_pipe = *dp != '0';    // opt-in (see multiply_impl)
  cudaError_t e = cudaSetDevice(device);
  ctx->stream = (cudaStream_t)cuda_stream;  // NULL = the legacy default stream (torch's default)
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->comm, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->comm2, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    set_error(std::string("context CUDA setup: ") + cudaGetErrorString(e));
    delete ctx;
    return DBM_ERR_CUDA;
  }
  if (nranks > 1) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm;
    ncclResult_t r = ncclCommInitRank(&comm, nranks, uid, rank);
    if (r != ncclSuccess) {
      set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
      cudaStreamDestroy(ctx->comm);
      cudaStreamDestroy(ctx->comm2);
      if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
      delete ctx;
      return DBM_ERR_NCCL;
    }
    ctx->nccl = comm;
  }
  num_sms();
  *out = ctx;
  return DBM_OK;
}

extern "C" dbm_status dbm_ctx_grid(dbm_ctx ctx, int* pr, int* pc, int* myrow, int* mycol) {
  ARG_CHECK(ctx, DBM_ERR_ARG, "null context");
  if (pr) *pr = ctx->pr;
  if (pc) *pc = ctx->pc;
  if (myrow) *myrow = ctx->myrow;
  if (mycol) *mycol = ctx->mycol;
  return DBM_OK;
}

extern "C" dbm_status dbm_ctx_set_stream(dbm_ctx ctx, void* stream) {
  CTX_OK(ctx);
  if (ctx->own_stream && ctx->stream != (cudaStream_t)stream) {
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    cudaStreamDestroy(ctx->stream);
    ctx->own_stream = false;
  }
  ctx->stream = (cudaStream_t)stream;
  return DBM_OK;
}

extern "C" dbm_status dbm_ctx_sync(dbm_ctx ctx) {
  CTX_OK(ctx);
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  for (cudaStream_t st : {ctx->comm, ctx->comm2, ctx->up, ctx->gen, ctx->own})
    if (st) CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (ctx->nccl) {
    ncclResult_t ae;
    NCCL_TRY(ctx, ncclCommGetAsyncError((ncclComm_t)ctx->nccl, &ae));
    NCCL_TRY(ctx, ae);
  }
  return DBM_OK;
}

extern "C" dbm_status dbm_ctx_set_profiling(dbm_ctx ctx, int on) {
  ARG_CHECK(ctx, DBM_ERR_ARG, "null context");
  ctx->profiling = on != 0;
  return DBM_OK;
}

extern "C" dbm_status dbm_ctx_profile_read(dbm_ctx ctx, int kernel, double* ms_out, int64_t* launches_out,
                                           double* flops_out, double* bytes_out) {
  CTX_OK(ctx);
  double ms = 0, fl = 0, by = 0;
  int64_t n = 0;
  std::vector<dbm_ctx_s::ProfRec> keep;
  for (auto& r : ctx->prof) {
    if (r.kind != kernel) {
      keep.push_back(r);
      continue;
    }
    CUDA_TRY(ctx, cudaEventSynchronize(r.b));
    float t = 0;
    CUDA_TRY(ctx, cudaEventElapsedTime(&t, r.a, r.b));
    ms += t;
    fl += r.flops;
    by += r.bytes;
    ++n;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  ctx->prof.swap(keep);
  ctx->lt_valid = false;  // the bracketed record range is gone
  if (ms_out) *ms_out = ms;
  if (launches_out) *launches_out = n;
  if (flops_out) *flops_out = fl;
  if (bytes_out) *bytes_out = by;
  return DBM_OK;
}

extern "C" dbm_status dbm_ctx_profile_timeline(dbm_ctx ctx, int max_records, double* out, int* n_out) {
  CTX_OK(ctx);
  ARG_CHECK(n_out && max_records >= 0 && (out || max_records == 0), DBM_ERR_ARG, "bad timeline buffer");
  const int n = (int)std::min<size_t>(ctx->prof.size(), (size_t)max_records);
  for (int i = 0; i < n; ++i) {
    const auto& r = ctx->prof[i];
    CUDA_TRY(ctx, cudaEventSynchronize(r.b));
    float t0 = 0, t1 = 0;
    CUDA_TRY(ctx, cudaEventElapsedTime(&t0, ctx->prof[0].a, r.a));
    CUDA_TRY(ctx, cudaEventElapsedTime(&t1, ctx->prof[0].a, r.b));
    out[3 * i] = r.kind;
    out[3 * i + 1] = t0;
    out[3 * i + 2] = t1;
  }
  *n_out = (int)ctx->prof.size();
  return DBM_OK;
}

extern "C" dbm_status dbm_ctx_set_transport(dbm_ctx ctx, int transport) {
  ARG_CHECK(ctx && (transport == 0 || transport == 1), DBM_ERR_ARG, "transport must be 0 (copy engine) or 1 (NCCL)");
  ctx->transport = transport;
  return DBM_OK;
}

extern "C" dbm_status dbm_ctx_set_algorithm(dbm_ctx ctx, int algorithm) {
  ARG_CHECK(ctx && algorithm >= 0 && algorithm <= 2, DBM_ERR_ARG,
            "algorithm must be 0 (Cannon), 1 (tall-skinny) or 2 (automatic)");
  ctx->algorithm = algorithm;
  return DBM_OK;
}

extern "C" dbm_status dbm_ctx_set_dense_chunk_bytes(dbm_ctx ctx, int64_t bytes) {
  ARG_CHECK(ctx && bytes >= 1, DBM_ERR_ARG, "bad argument");
  ctx->chunk_bytes = bytes;
  return DBM_OK;
}

extern "C" dbm_status dbm_ctx_set_densify_threshold(dbm_ctx ctx, double threshold) {
  ARG_CHECK(ctx && threshold >= 0.0 && threshold <= 1.0, DBM_ERR_ARG, "threshold outside [0, 1]");
  ctx->densify_threshold = threshold;
  return DBM_OK;
}

extern "C" dbm_status dbm_ctx_launch_count(dbm_ctx ctx, int64_t* out) {
  ARG_CHECK(ctx && out, DBM_ERR_ARG, "null argument");
  *out = ctx->launches;
  return DBM_OK;
}

extern "C" dbm_status dbm_ctx_destroy(dbm_ctx ctx) {
  if (!ctx) return DBM_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (cudaStream_t st : {ctx->comm, ctx->comm2, ctx->up, ctx->gen, ctx->own})
    if (st) cudaStreamSynchronize(st);
  free_sp_cache(ctx);
  free_nu_cache(ctx);
  for (auto& r : ctx->prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->lt_a) cudaEventDestroy(ctx->lt_a);
  if (ctx->lt_b) cudaEventDestroy(ctx->lt_b);
  for (int i = 0; i < 2; ++i) {
    if (ctx->stage[i]) cudaFreeHost(ctx->stage[i]);
    if (ctx->stage_ev[i]) cudaEventDestroy(ctx->stage_ev[i]);
  }
  for (void* b : ctx->peer_bases)
    if (b) cudaIpcCloseMemHandle(b);
  if (ctx->d_scratch) cudaFree(ctx->d_scratch);
  if (ctx->xpool) cudaFree(ctx->xpool);
  if (ctx->nccl) ncclCommDestroy((ncclComm_t)ctx->nccl);
  cudaStreamDestroy(ctx->comm);
  if (ctx->comm2) cudaStreamDestroy(ctx->comm2);
  if (ctx->up) cudaStreamDestroy(ctx->up);
  if (ctx->gen) cudaStreamDestroy(ctx->gen);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return DBM_OK;
}

// ====================================================================== matrix
extern "C" dbm_status dbm_matrix_create(dbm_ctx ctx, int64_t rows, int64_t cols, int32_t bs, dbm_matrix* out) {
  ARG_CHECK(ctx && out, DBM_ERR_ARG, "null argument");
  ARG_CHECK(bs > 0 && rows >= 0 && cols >= 0, DBM_ERR_ARG, "bad block size or dimensions");
  ARG_CHECK(rows % bs == 0 && cols % bs == 0, DBM_ERR_SHAPE, "rows/cols must be multiples of the block size");
  ARG_CHECK(rows / bs < (1LL << 31) && cols / bs < (1LL << 31), DBM_ERR_SHAPE, "too many blocks");
  dbm_matrix m = new dbm_matrix_s();
  m->ctx = ctx;
  m->rows = rows;
  m->cols = cols;
  m->bs = bs;
  m->Mb = rows / bs;
  m->Nb = cols / bs;
  m->mloc = local_count(m->Mb, ctx->pr, ctx->myrow);
  m->nloc = local_count(m->Nb, ctx->pc, ctx->mycol);
  m->nnz = m->mloc * m->nloc;
  m->gnnz = m->Mb * m->Nb;
  m->serial = next_serial();
  *out = m;
  return DBM_OK;
}

// ---- block sparsity (reading R15) ----
static uint64_t host_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

extern "C" dbm_status dbm_pattern_random(uint64_t seed, uint32_t mat_id, int64_t Mb, int64_t Nb, double occupancy,
                                         uint8_t* mask) {
  ARG_CHECK(Mb >= 0 && Nb >= 0, DBM_ERR_ARG, "negative block counts");
  ARG_CHECK(Mb * Nb == 0 || mask, DBM_ERR_ARG, "null mask");
  ARG_CHECK(occupancy >= 0.0 && occupancy <= 1.0, DBM_ERR_ARG, "occupancy outside [0, 1]");
  const uint64_t key = host_mix64(seed + 0x9E3779B97F4A7C15ull * ((uint64_t)(mat_id | 0x80000000u) + 1ull));
  for (int64_t bi = 0; bi < Mb; ++bi)
    for (int64_t bj = 0; bj < Nb; ++bj) {
      const uint64_t bits = host_mix64(key ^ host_mix64(((uint64_t)bi << 32) ^ (uint64_t)bj));
      const double u = (double)(bits >> 11) * 0x1.0p-53;
      mask[bi * Nb + bj] = u < occupancy ? 1 : 0;
    }
  return DBM_OK;
}

extern "C" dbm_status dbm_pattern_product(int64_t Mb, int64_t Kb, int64_t Nb, const uint8_t* amask,
                                          const uint8_t* bmask, uint8_t* cmask) {
  ARG_CHECK(Mb >= 0 && Kb >= 0 && Nb >= 0, DBM_ERR_ARG, "negative block counts");
  ARG_CHECK((Mb * Kb == 0 || amask) && (Kb * Nb == 0 || bmask) && (Mb * Nb == 0 || cmask), DBM_ERR_ARG, "null mask");
  for (int64_t i = 0; i < Mb; ++i) {  // row i: OR the B rows k with A(i, k) stored
    uint8_t* crow = cmask + i * Nb;
    for (int64_t k = 0; k < Kb; ++k) {
      if (!amask[i * Kb + k]) continue;
      const uint8_t* brow = bmask + k * Nb;
      for (int64_t j = 0; j < Nb; ++j) crow[j] |= brow[j] ? 1 : 0;
    }
  }
  return DBM_OK;
}

extern "C" dbm_status dbm_matrix_create_sparse(dbm_ctx ctx, int64_t rows, int64_t cols, int32_t bs,
                                               const uint8_t* mask, dbm_matrix* out) {
  dbm_matrix m = nullptr;
  if (dbm_status s = dbm_matrix_create(ctx, rows, cols, bs, &m)) return s;
  m->sparse = true;
  m->device = ctx->device;
  const size_t nb = (size_t)(m->Mb * m->Nb);
  m->gmask.assign(nb, 1);
  if (mask)
    for (size_t i = 0; i < nb; ++i) m->gmask[i] = mask[i] ? 1 : 0;
  m->gnnz = 0;
  for (size_t i = 0; i < nb; ++i) m->gnnz += m->gmask[i];
  m->row_ptr.assign(m->mloc + 1, 0);
  std::vector<int32_t> ij;
  std::vector<int32_t> map((size_t)(m->mloc * m->nloc), -1);
  for (int64_t li = 0; li < m->mloc; ++li) {
    for (int64_t lj = 0; lj < m->nloc; ++lj)
      if (m->gmask[(size_t)(ctx->myrow + li * ctx->pr) * m->Nb + ctx->mycol + lj * ctx->pc]) {
        map[(size_t)(li * m->nloc + lj)] = (int32_t)m->col.size();
        m->col.push_back((int32_t)lj);
        ij.push_back((int32_t)li);
        ij.push_back((int32_t)lj);
      }
    m->row_ptr[li + 1] = (int64_t)m->col.size();
  }
  m->nnz = (int64_t)m->col.size();
  auto fail = [&](cudaError_t e) {
    set_error(std::string("sparse metadata: ") + cudaGetErrorString(e));
    dbm_matrix_destroy(m);
    return DBM_ERR_NOMEM;
  };
  if (cudaError_t e = cudaSetDevice(ctx->device)) return fail(e);
  if (cudaError_t e = cudaMalloc(&m->d_ij, std::max<size_t>(ij.size(), 2) * 4)) return fail(e);
  if (cudaError_t e = cudaMalloc(&m->d_map, std::max<size_t>(map.size(), 1) * 4)) return fail(e);
  if (!ij.empty())
    if (cudaError_t e = cudaMemcpy(m->d_ij, ij.data(), ij.size() * 4, cudaMemcpyHostToDevice)) return fail(e);
  if (!map.empty())
    if (cudaError_t e = cudaMemcpy(m->d_map, map.data(), map.size() * 4, cudaMemcpyHostToDevice)) return fail(e);
  *out = m;
  return DBM_OK;
}

// ---- non-uniform block sizes (reading R16) ----
extern "C" dbm_status dbm_matrix_create_blocked(dbm_ctx ctx, int64_t nblk_rows, const int32_t* row_sizes,
                                                int64_t nblk_cols, const int32_t* col_sizes, const uint8_t* mask,
                                                dbm_matrix* out) {
  ARG_CHECK(ctx && out, DBM_ERR_ARG, "null argument");
  ARG_CHECK(nblk_rows >= 0 && nblk_cols >= 0 && nblk_rows < (1LL << 31) && nblk_cols < (1LL << 31), DBM_ERR_ARG,
            "bad block counts");
  ARG_CHECK((nblk_rows == 0 || row_sizes) && (nblk_cols == 0 || col_sizes), DBM_ERR_ARG, "null size list");
  for (int64_t i = 0; i < nblk_rows; ++i) ARG_CHECK(row_sizes[i] > 0, DBM_ERR_SHAPE, "block sizes must be positive");
  for (int64_t j = 0; j < nblk_cols; ++j) ARG_CHECK(col_sizes[j] > 0, DBM_ERR_SHAPE, "block sizes must be positive");
  // all sizes equal: the uniform matrix (dense or sparse), which takes the uniform kernels
  const int32_t s0 = nblk_rows ? row_sizes[0] : (nblk_cols ? col_sizes[0] : 1);
  bool uni = true;
  for (int64_t i = 0; i < nblk_rows; ++i) uni &= row_sizes[i] == s0;
  for (int64_t j = 0; j < nblk_cols; ++j) uni &= col_sizes[j] == s0;
  if (uni)
    return mask ? dbm_matrix_create_sparse(ctx, nblk_rows * s0, nblk_cols * s0, s0, mask, out)
                : dbm_matrix_create(ctx, nblk_rows * s0, nblk_cols * s0, s0, out);
  dbm_matrix m = new dbm_matrix_s();
  m->ctx = ctx;
  m->nonuni = true;
  m->bs = 0;  // no uniform block size
  m->device = ctx->device;
  m->Mb = nblk_rows;
  m->Nb = nblk_cols;
  m->rsz.assign(row_sizes, row_sizes + nblk_rows);
  m->csz.assign(col_sizes, col_sizes + nblk_cols);
  m->roff.assign(nblk_rows + 1, 0);
  m->coff.assign(nblk_cols + 1, 0);
  for (int64_t i = 0; i < nblk_rows; ++i) m->roff[i + 1] = m->roff[i] + row_sizes[i];
  for (int64_t j = 0; j < nblk_cols; ++j) m->coff[j + 1] = m->coff[j] + col_sizes[j];
  m->rows = m->roff.back();
  m->cols = m->coff.back();
  m->mloc = local_count(m->Mb, ctx->pr, ctx->myrow);
  m->nloc = local_count(m->Nb, ctx->pc, ctx->mycol);
  m->sparse = mask != nullptr;
  if (m->sparse) {
    m->gmask.resize((size_t)(m->Mb * m->Nb));
    for (size_t i = 0; i < m->gmask.size(); ++i) m->gmask[i] = mask[i] ? 1 : 0;
  }
  m->gnnz = 0;
  for (int64_t bi = 0; bi < m->Mb; ++bi)
    for (int64_t bj = 0; bj < m->Nb; ++bj) m->gnnz += m->stored(bi, bj) ? 1 : 0;
  m->row_ptr.assign(m->mloc + 1, 0);
  m->slot_off.assign(1, 0);
  for (int64_t li = 0; li < m->mloc; ++li) {
    const int64_t bi = ctx->myrow + li * ctx->pr;
    for (int64_t lj = 0; lj < m->nloc; ++lj) {
      const int64_t bj = ctx->mycol + lj * ctx->pc;
      if (!m->stored(bi, bj)) continue;
      m->col.push_back((int32_t)lj);
      m->hblk.push_back({m->slot_off.back(), m->roff[bi], m->coff[bj], m->rsz[bi], m->csz[bj]});
      m->slot_off.push_back(m->slot_off.back() + (int64_t)m->rsz[bi] * m->csz[bj]);
    }
    m->row_ptr[li + 1] = (int64_t)m->col.size();
  }
  m->nnz = (int64_t)m->col.size();
  m->serial = next_serial();
  if (cudaError_t e = cudaSetDevice(ctx->device)) {
    set_error(cudaGetErrorString(e));
    delete m;
    return DBM_ERR_CUDA;
  }
  cudaError_t e = cudaMalloc(&m->d_blk, std::max<size_t>(m->hblk.size(), 1) * sizeof(NUBlk));
  if (e == cudaSuccess && !m->hblk.empty())
    e = cudaMemcpy(m->d_blk, m->hblk.data(), m->hblk.size() * sizeof(NUBlk), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    set_error(std::string("non-uniform block table: ") + cudaGetErrorString(e));
    dbm_matrix_destroy(m);
    return DBM_ERR_NOMEM;
  }
  *out = m;
  return DBM_OK;
}

// A uniform matrix that meets non-uniform ones in a multiply gets the per-slot tables too (slot s at element
// offset s * bs^2, CSR slot order for block-sparse patterns); built once, library-owned.
dbm_status dbm::nu_tables(dbm_matrix m) {
  if (m->nonuni || m->d_blk) return DBM_OK;
  dbm_ctx ctx = m->ctx;
  const int64_t bb = (int64_t)m->bs * m->bs;
  m->slot_off.assign(1, 0);
  m->hblk.clear();
  for (int64_t li = 0; li < m->mloc; ++li) {
    const int64_t bi = ctx->myrow + li * ctx->pr;
    const int64_t q0 = m->sparse ? m->row_ptr[li] : li * m->nloc, q1 = m->sparse ? m->row_ptr[li + 1] : (li + 1) * m->nloc;
    for (int64_t q = q0; q < q1; ++q) {
      const int64_t lj = m->sparse ? m->col[q] : q - li * m->nloc, bj = ctx->mycol + lj * ctx->pc;
      m->hblk.push_back({m->slot_off.back(), bi * m->bs, bj * m->bs, m->bs, m->bs});
      m->slot_off.push_back(m->slot_off.back() + bb);
    }
  }
  m->device = ctx->device;
  cudaError_t e = cudaMalloc(&m->d_blk, std::max<size_t>(m->hblk.size(), 1) * sizeof(NUBlk));
  if (e == cudaSuccess && !m->hblk.empty())
    e = cudaMemcpy(m->d_blk, m->hblk.data(), m->hblk.size() * sizeof(NUBlk), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    set_error(std::string("block table: ") + cudaGetErrorString(e));
    return DBM_ERR_NOMEM;
  }
  return DBM_OK;
}

extern "C" dbm_status dbm_matrix_block_sizes(dbm_matrix m, int32_t* row_sizes, int32_t* col_sizes) {
  ARG_CHECK(m, DBM_ERR_ARG, "null matrix");
  for (int64_t i = 0; i < m->Mb && row_sizes; ++i) row_sizes[i] = m->row_size(i);
  for (int64_t j = 0; j < m->Nb && col_sizes; ++j) col_sizes[j] = m->col_size(j);
  return DBM_OK;
}

extern "C" dbm_status dbm_matrix_nnz(dbm_matrix m, int64_t* local_blocks, int64_t* global_blocks) {
  ARG_CHECK(m, DBM_ERR_ARG, "null matrix");
  if (local_blocks) *local_blocks = m->blocks();
  if (global_blocks) *global_blocks = m->gnnz;
  return DBM_OK;
}

extern "C" dbm_status dbm_matrix_local_info(dbm_matrix m, int64_t* mloc, int64_t* nloc, int64_t* bytes) {
  ARG_CHECK(m, DBM_ERR_ARG, "null matrix");
  if (mloc) *mloc = m->mloc;
  if (nloc) *nloc = m->nloc;
  if (bytes) *bytes = m->elems() * 8;
  return DBM_OK;
}

extern "C" dbm_status dbm_matrix_local_csr(dbm_matrix m, int64_t* row_ptr, int64_t* col_idx, int64_t* row_idx) {
  ARG_CHECK(m, DBM_ERR_ARG, "null matrix");
  const dbm_ctx c = m->ctx;
  for (int64_t li = 0; li <= m->mloc; ++li)
    if (row_ptr) row_ptr[li] = m->sparse ? m->row_ptr[li] : li * m->nloc;
  for (int64_t li = 0; li < m->mloc; ++li) {
    if (row_idx) row_idx[li] = c->myrow + li * c->pr;
    if (!col_idx) continue;
    if (m->sparse) {
      for (int64_t s = m->row_ptr[li]; s < m->row_ptr[li + 1]; ++s) col_idx[s] = c->mycol + (int64_t)m->col[s] * c->pc;
    } else {
      for (int64_t lj = 0; lj < m->nloc; ++lj) col_idx[li * m->nloc + lj] = c->mycol + lj * c->pc;
    }
  }
  return DBM_OK;
}

extern "C" dbm_status dbm_matrix_attach(dbm_matrix m, void* arena, int64_t bytes) {
  ARG_CHECK(m, DBM_ERR_ARG, "null matrix");
  const int64_t need = m->elems() * 8;
  ARG_CHECK(bytes >= need, DBM_ERR_WORKSPACE, "arena smaller than dbm_matrix_local_info() bytes");
  ARG_CHECK(need == 0 || arena != nullptr, DBM_ERR_ARG, "null arena");
  ARG_CHECK(((uintptr_t)arena & 15) == 0, DBM_ERR_ARG, "arena must be 16-byte aligned");
  m->arena = (double*)arena;
  m->arena_bytes = bytes;
  return DBM_OK;
}

static dbm_status need_arena(dbm_matrix m) {
  const int64_t need = m->elems() * 8;
  ARG_CHECK(need == 0 || m->arena, DBM_ERR_WORKSPACE, "matrix has no attached arena");
  return DBM_OK;
}

extern "C" dbm_status dbm_matrix_fill_random(dbm_matrix m, uint64_t seed, uint32_t mat_id, int kind) {
  ARG_CHECK(m, DBM_ERR_ARG, "null matrix");
  ARG_CHECK(kind == 0 || kind == 1, DBM_ERR_ARG, "kind must be 0 or 1");
  dbm_ctx ctx = m->ctx;
  CTX_OK(ctx);
  if (dbm_status s = need_arena(m)) return s;
  if (m->nonuni)
    launch_nu_fill(m->arena, m->d_blk, m->blocks(), seed, mat_id, kind, ctx->stream);
  else if (m->sparse)
    launch_fill_sparse(m->arena, m->nnz, m->d_ij, m->bs, ctx->pr, ctx->pc, ctx->myrow, ctx->mycol, seed, mat_id, kind,
                       ctx->stream);
  else
    launch_fill(m->arena, m->mloc, m->nloc, m->bs, ctx->pr, ctx->pc, ctx->myrow, ctx->mycol, seed, mat_id, kind,
                ctx->stream);
  ctx->launches += m->blocks() ? 1 : 0;
  CUDA_TRY(ctx, cudaGetLastError());
  return DBM_OK;
}

static dbm_status block_slot(dbm_matrix m, int64_t bi, int64_t bj, int64_t* slot) {
  ARG_CHECK(bi >= 0 && bj >= 0 && bi < m->Mb && bj < m->Nb, DBM_ERR_RANGE, "block index out of range");
  const dbm_ctx c = m->ctx;
  ARG_CHECK(bi % c->pr == c->myrow && bj % c->pc == c->mycol, DBM_ERR_OWNERSHIP, "block owned by another rank");
  const int64_t li = bi / c->pr, lj = bj / c->pc;
  if (!m->sparse && !m->nonuni) {
    *slot = li * m->nloc + lj;
    return DBM_OK;
  }
  if (!m->sparse) {  // non-uniform, every block stored: CSR slots are li * nloc + lj
    *slot = li * m->nloc + lj;
    return DBM_OK;
  }
  const auto b = m->col.begin() + m->row_ptr[li], e = m->col.begin() + m->row_ptr[li + 1];
  const auto it = std::lower_bound(b, e, (int32_t)lj);
  ARG_CHECK(it != e && *it == (int32_t)lj, DBM_ERR_RANGE, "block not stored in the sparsity pattern");
  *slot = (int64_t)(it - m->col.begin());
  return DBM_OK;
}

extern "C" dbm_status dbm_matrix_set_block(dbm_matrix m, int64_t bi, int64_t bj, const double* host) {
  ARG_CHECK(m && host, DBM_ERR_ARG, "null argument");
  dbm_ctx ctx = m->ctx;
  CTX_OK(ctx);
  int64_t slot;
  if (dbm_status s = block_slot(m, bi, bj, &slot)) return s;
  if (dbm_status s = need_arena(m)) return s;
  const size_t bb = (size_t)m->row_size(bi) * m->col_size(bj);
  const int64_t off = m->nonuni ? m->slot_off[slot] : slot * (int64_t)bb;
  CUDA_TRY(ctx, cudaMemcpyAsync(m->arena + off, host, bb * 8, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return DBM_OK;
}

extern "C" dbm_status dbm_matrix_get_block(dbm_matrix m, int64_t bi, int64_t bj, double* host) {
  ARG_CHECK(m && host, DBM_ERR_ARG, "null argument");
  dbm_ctx ctx = m->ctx;
  CTX_OK(ctx);
  int64_t slot;
  if (dbm_status s = block_slot(m, bi, bj, &slot)) return s;
  if (dbm_status s = need_arena(m)) return s;
  const size_t bb = (size_t)m->row_size(bi) * m->col_size(bj);
  const int64_t off = m->nonuni ? m->slot_off[slot] : slot * (int64_t)bb;
  CUDA_TRY(ctx, cudaMemcpyAsync(host, m->arena + off, bb * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return DBM_OK;
}

// Host <-> device of the whole arena.  Pinned host memory: one async copy.  Pageable: staged through a
// pinned double buffer (P:174 double buffering, P:200 page-locked memory pools).
static dbm_status host_copy(dbm_matrix m, void* host, bool upload) {
  dbm_ctx ctx = m->ctx;
  const size_t bytes = (size_t)m->elems() * 8;
  if (bytes == 0) return DBM_OK;
  cudaPointerAttributes at;
  bool pinned = cudaPointerGetAttributes(&at, host) == cudaSuccess &&
                (at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeManaged);
  cudaGetLastError();
  char* dev = (char*)m->arena;
  if (pinned) {
    CUDA_TRY(ctx, cudaMemcpyAsync(upload ? (void*)dev : host, upload ? host : (void*)dev, bytes,
                                  upload ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, ctx->stream));
    return DBM_OK;
  }
  const size_t chunk = 64ull << 20;
  if (!ctx->stage[0]) {
    for (int i = 0; i < 2; ++i) {
      CUDA_TRY(ctx, cudaHostAlloc(&ctx->stage[i], chunk, cudaHostAllocDefault));
      CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming));
    }
    ctx->stage_bytes = chunk;
  }
  size_t off = 0;
  int b = 0;
  bool used[2] = {false, false};
  while (off < bytes) {
    const size_t n = std::min(chunk, bytes - off);
    if (used[b]) CUDA_TRY(ctx, cudaEventSynchronize(ctx->stage_ev[b]));
    if (upload) {
      std::memcpy(ctx->stage[b], (char*)host + off, n);
      CUDA_TRY(ctx, cudaMemcpyAsync(dev + off, ctx->stage[b], n, cudaMemcpyHostToDevice, ctx->stream));
      CUDA_TRY(ctx, cudaEventRecord(ctx->stage_ev[b], ctx->stream));
    } else {
      CUDA_TRY(ctx, cudaMemcpyAsync(ctx->stage[b], dev + off, n, cudaMemcpyDeviceToHost, ctx->stream));
      CUDA_TRY(ctx, cudaEventRecord(ctx->stage_ev[b], ctx->stream));
      CUDA_TRY(ctx, cudaEventSynchronize(ctx->stage_ev[b]));
      std::memcpy((char*)host + off, ctx->stage[b], n);
    }
    used[b] = true;
    off += n;
    b ^= 1;
  }
  for (int i = 0; i < 2; ++i)
    if (used[i]) CUDA_TRY(ctx, cudaEventSynchronize(ctx->stage_ev[i]));
  return DBM_OK;
}

extern "C" dbm_status dbm_matrix_upload(dbm_matrix m, const void* host) {
  ARG_CHECK(m && host, DBM_ERR_ARG, "null argument");
  CTX_OK(m->ctx);
  if (dbm_status s = need_arena(m)) return s;
  return host_copy(m, (void*)host, true);
}

extern "C" dbm_status dbm_matrix_download(dbm_matrix m, void* host) {
  ARG_CHECK(m && host, DBM_ERR_ARG, "null argument");
  CTX_OK(m->ctx);
  if (dbm_status s = need_arena(m)) return s;
  return host_copy(m, host, false);
}

extern "C" dbm_status dbm_owner_of_block(dbm_matrix m, int64_t bi, int64_t bj, int* rank) {
  ARG_CHECK(m && rank, DBM_ERR_ARG, "null argument");
  ARG_CHECK(bi >= 0 && bj >= 0 && bi < m->Mb && bj < m->Nb, DBM_ERR_RANGE, "block index out of range");
  *rank = (int)(bi % m->ctx->pr) * m->ctx->pc + (int)(bj % m->ctx->pc);
  return DBM_OK;
}

extern "C" dbm_status dbm_matrix_destroy(dbm_matrix m) {
  if (m && (m->d_ij || m->d_map || m->d_blk)) {
    // the context may already be destroyed: use the device recorded at creation, restore the caller's
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(m->device);
    if (m->d_ij) cudaFree(m->d_ij);
    if (m->d_map) cudaFree(m->d_map);
    if (m->d_blk) cudaFree(m->d_blk);
    cudaSetDevice(cur);
    cudaGetLastError();
  }
  delete m;
  return DBM_OK;
}

// ====================================================================== densify / undensify
// Non-uniform blocks (R16): the local share's element rows / columns and one copy task per stored slot,
// staged in stream-ordered device memory for one launch of the table-driven copy kernel.
static dbm_status nu_local_copy(dbm_matrix m, double* dense, int64_t ld, int mode, double alpha, double beta) {
  dbm_ctx ctx = m->ctx;
  std::vector<int64_t> lro(m->mloc + 1, 0), lco(m->nloc + 1, 0);
  for (int64_t li = 0; li < m->mloc; ++li) lro[li + 1] = lro[li] + m->row_size(ctx->myrow + li * ctx->pr);
  for (int64_t lj = 0; lj < m->nloc; ++lj) lco[lj + 1] = lco[lj] + m->col_size(ctx->mycol + lj * ctx->pc);
  const int64_t rows = lro.back(), cols = lco.back();
  ARG_CHECK(ld >= (mode == 0 ? cols : rows), DBM_ERR_PLAN, "leading dimension too small");
  ARG_CHECK(rows * cols == 0 || dense, DBM_ERR_ARG, "null dense buffer");
  if (rows * cols == 0) return DBM_OK;
  std::vector<NUTask> t;
  for (int64_t li = 0; li < m->mloc; ++li)
    for (int64_t q = m->row_ptr[li]; q < m->row_ptr[li + 1]; ++q) {
      const int64_t lj = m->col[q];
      t.push_back({m->slot_off[q], lro[li], lco[lj], m->hblk[q].rows, m->hblk[q].cols});
    }
  if (mode != 2 && m->sparse)  // absent blocks densify to zeros
    CUDA_TRY(ctx, cudaMemsetAsync(dense, 0, (size_t)ld * (mode == 0 ? rows : cols) * 8, ctx->stream));
  if (t.empty()) return DBM_OK;
  NUTask* d = nullptr;
  CUDA_TRY(ctx, cudaMallocAsync((void**)&d, t.size() * sizeof(NUTask), ctx->stream));
  CUDA_TRY(ctx, cudaMemcpyAsync(d, t.data(), t.size() * sizeof(NUTask), cudaMemcpyHostToDevice, ctx->stream));
  launch_nu_copy(d, (int64_t)t.size(), m->arena, dense, ld, mode, alpha, beta, ctx->stream);
  CUDA_TRY(ctx, cudaGetLastError());
  CUDA_TRY(ctx, cudaFreeAsync(d, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));  // the pageable task vector must outlive the H2D copy
  ctx->launches += 1;
  return DBM_OK;
}

extern "C" dbm_status dbm_densify(dbm_matrix m, double* dense, int64_t ld, int layout) {
  ARG_CHECK(m, DBM_ERR_ARG, "null matrix");
  ARG_CHECK(layout == 0 || layout == 1, DBM_ERR_ARG, "layout must be 0 or 1");
  dbm_ctx ctx = m->ctx;
  CTX_OK(ctx);
  if (dbm_status s = need_arena(m)) return s;
  if (m->nonuni) return nu_local_copy(m, dense, ld, layout == 0 ? 1 : 0, 0.0, 0.0);
  const int64_t rows = m->mloc * m->bs, cols = m->nloc * m->bs;
  ARG_CHECK(ld >= (layout == 0 ? rows : cols), DBM_ERR_PLAN, "leading dimension too small");
  ARG_CHECK(rows * cols == 0 || dense, DBM_ERR_ARG, "null dense buffer");
  ProfScope ps(ctx, ctx->stream, 2, 0.0, 16.0 * rows * cols);
  if (m->sparse)
    CUDA_TRY(ctx, launch_sp_densify(m->arena, m->d_ij, m->nnz, m->bs, 0, 0, 1, m->nloc, m->mloc, dense, ld, layout,
                                    ctx->stream));
  else
    launch_densify_cols(m->arena, m->mloc, m->nloc, m->bs, 0, 1, m->nloc, dense, ld, layout, ctx->stream);
  ctx->launches += rows * cols ? 1 : 0;
  CUDA_TRY(ctx, cudaGetLastError());
  return DBM_OK;
}

extern "C" dbm_status dbm_undensify(dbm_matrix m, const double* dense, int64_t ld, double alpha, double beta) {
  ARG_CHECK(m, DBM_ERR_ARG, "null matrix");
  dbm_ctx ctx = m->ctx;
  CTX_OK(ctx);
  if (dbm_status s = need_arena(m)) return s;
  if (m->nonuni) return nu_local_copy(m, (double*)dense, ld, 2, alpha, beta);
  const int64_t rows = m->mloc * m->bs, cols = m->nloc * m->bs;
  ARG_CHECK(ld >= rows, DBM_ERR_PLAN, "leading dimension too small");
  ARG_CHECK(rows * cols == 0 || dense, DBM_ERR_ARG, "null dense buffer");
  ProfScope ps(ctx, ctx->stream, 3, 0.0, (beta == 0.0 ? 16.0 : 24.0) * rows * cols);
  if (m->sparse)
    launch_sp_undensify(dense, ld, 1, 0, m->d_ij, m->nnz, m->bs, alpha, beta, m->arena, ctx->stream);
  else
    launch_undensify(dense, ld, 1, 0, m->mloc, m->nloc, m->bs, alpha, beta, m->arena, ctx->stream);
  ctx->launches += rows * cols ? 1 : 0;
  CUDA_TRY(ctx, cudaGetLastError());
  return DBM_OK;
}

// ====================================================================== multiply plan
namespace {

// Host-operand pipeline on several ranks (dbm_multiply_host): upload, own-panel densify and Cannon's
// step-0 pull + GEMM all run in the same 5 K-chunks of each panel (1, 1, 2, 4, 8 sixteenths).  The
// boundaries depend only on the panel's block count, which every rank agrees on, so an owner's
// progress after chunk j is exactly what a consumer's chunk j needs.
// Densified panels of an odd block size keep every chunk start even (in blocks), so the GEMM's TMA base
// Ap + k0*bs stays 16-byte aligned (`even`); the last bound is always kb.
constexpr int kHostPipeChunks = 5;
inline int64_t host_pipe_bound(int64_t kb, int j, bool even = false) {
  static const int F[kHostPipeChunks + 1] = {0, 1, 2, 4, 8, 16};
  if (j >= kHostPipeChunks) return kb;
  const int64_t b = kb * F[j] / 16;
  return even ? b / 2 * 2 : b;
}
inline bool host_pipe_even(bool densified, int64_t bs) { return densified && (bs & 1); }

struct Plan {
  int L = 1;
  int pr = 1, pc = 1, r = 0, c = 0;
  int64_t bs = 0, Mb = 0, Nb = 0, Kb = 0;
  int64_t mloc = 0, nloc = 0;  // C / A rows, C / B cols (blocks)
  int64_t kA = 0, kB = 0;      // A local block cols, B local block rows
  bool densified = true;
  std::vector<int64_t> kb;  // panel sizes (blocks) per kappa
  // K chunking (single-rank densified path): chunk_kb blocks per chunk
  int64_t chunk_kb = 0, nchunks = 1;
  // workspace regions (byte offsets)
  size_t off_cd = 0, off_ownA = 0, off_ownB = 0, off_recvA[2] = {0, 0}, off_recvB[2] = {0, 0}, off_part = 0;
  size_t off_trav = 0, off_trip = 0, off_spart = 0;  // smm split-K partials
  size_t off_trip2 = 0;                               // second triplet buffer (0: one chunk per step)
  bool mixed = false;                                 // bs 22 squares inside a non-square traversal
  // densified bs 64 with a dense B: B is never densified -- the GEMM reads B's 64 x 64 blocks in place
  // (arena, or packed panels the peers pull), through a 4-D TMA view (§8f-3, zero-copy B)
  bool b_packed = false;
  // densified bs 64 with a dense A: A is never densified either -- the GEMM reads A's 64 x 64 blocks in
  // place through a 4-D TMA view (arena on one rank, packed own panels the peers pull on several)
  bool a_packed = false;
  size_t off_pos = 0, off_sqflag = 0, off_sqids = 0, off_runsq = 0, off_runleft = 0, off_runflag = 0;
  size_t off_counts = 0, off_mtemp = 0, mtemp_bytes = 0;
  int64_t spart_runs = 0;                            // capacity: (split x runs) C blocks
  std::vector<size_t> ownA_off, ownB_off;  // per kappa, SIZE_MAX if not owned
  int64_t trip_cap = 0;                     // entries per stack-generation chunk
  size_t total = 0;       // caller-owned workspace bytes
  size_t pool_total = 0;  // several ranks: exchange-pool bytes (signal header + own panels peers pull)
  int max_split = 1;

  bool local_first = false;  // steps in local-first order (local_first_start), else canonical
  int s0 = 0;                // this rank's first canonical step
  int kappa(int s) const { return (r + c + s + s0) % L; }
  int a_src(int s) const { return r * pc + kappa(s) % pc; }
  int b_src(int s) const { return (kappa(s) % pr) * pc + c; }
  int me() const { return r * pc + c; }
  // dense panel leading dimensions (even, so TMA strides are 16-byte multiples)
  int64_t ld_panel(int k) const { return round_up(std::max<int64_t>(kb[k] * bs, 1), 2); }
  // (an empty K panel, kb = 0, moves no bytes on either path)
  size_t a_panel_bytes(int k) const {
    if (kb[k] == 0) return 0;
    return densified ? (size_t)(mloc * bs) * ld_panel(k) * 8 : (size_t)(mloc * kb[k]) * bs * bs * 8;
  }
  size_t b_panel_bytes(int k) const {
    if (kb[k] == 0) return 0;
    return densified ? (size_t)(nloc * bs) * ld_panel(k) * 8 : (size_t)(nloc * kb[k]) * bs * bs * 8;
  }
};

bool stackgen_dbuf();
bool zero_copy_a();
// DBM_SMMQ=0 keeps the padded small sizes on the per-run kernel (the A/B of the R x R square kernel);
// DBM_SMMQ=2 takes the squares even when they cannot fill the GPU (tests of small shapes)
bool ce_pack_on() {  // opt-in (DBM_CE_PACK=1): see the own-panel block of multiply_impl
  static const bool on = [] {
    const char* e = getenv("DBM_CE_PACK");
    return e && *e == '1';
  }();
  return on;
}

int smmq_on() {
  static const int on = [] {
    const char* e = getenv("DBM_SMMQ");
    return e ? atoi(e) : 1;
  }();
  return on;
}

// Host-only plan: depends on the grid, this rank's coordinates and the block counts (no CUDA).
Plan make_plan_raw(int nranks, int pr, int pc, int r, int c, int64_t Mb, int64_t Nb, int64_t Kb, int64_t bs,
                   bool densified, int64_t chunk_bytes, int transport, bool b_packed = false,
                   bool a_packed = false, bool local_first = false) {
  Plan p;
  p.local_first = local_first && nranks > 1 && transport == 0;
  p.s0 = p.local_first ? local_first_start(pr, pc, r * pc + c) : 0;
  p.b_packed = b_packed;
  p.a_packed = a_packed;
  p.pr = pr;
  p.pc = pc;
  p.r = r;
  p.c = c;
  p.L = (int)lcm64(p.pr, p.pc);
  p.bs = bs;
  p.Mb = Mb;
  p.Kb = Kb;
  p.Nb = Nb;
  p.mloc = local_count(Mb, pr, r);
  p.nloc = local_count(Nb, pc, c);
  p.kA = local_count(Kb, pc, c);
  p.kB = local_count(Kb, pr, r);
  p.densified = densified;
  p.kb.resize(p.L);
  for (int k = 0; k < p.L; ++k) p.kb[k] = local_count(p.Kb, p.L, k);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + bytes);
    return o;
  };
  // own panels (what the peers pull) live in the library's exchange pool, after the signal header
  size_t poff = xhdr_bytes(nranks, p.L);
  auto take_pool = [&](size_t bytes) {
    size_t o = poff;
    poff = align256(poff + bytes);
    return o;
  };
  const int64_t M = p.mloc * p.bs, N = p.nloc * p.bs;
  p.ownA_off.assign(p.L, SIZE_MAX);
  p.ownB_off.assign(p.L, SIZE_MAX);
  if (densified) {
    p.off_cd = take((size_t)M * N * 8);
    if (nranks == 1) {  // K-chunked densify -> GEMM accumulate (fits HBM at 63,360^3)
      const int64_t per_kblock = (M + N) * p.bs * 8;
      int64_t ck = per_kblock > 0 ? std::max<int64_t>(1, chunk_bytes / per_kblock) : p.Kb;
      ck = std::min<int64_t>(std::max<int64_t>(ck, 1), std::max<int64_t>(p.Kb, 1));
      p.chunk_kb = ck;
      p.nchunks = p.Kb > 0 ? (p.Kb + ck - 1) / ck : 1;
      const int64_t ld = round_up(ck * p.bs, 2);
      if (!a_packed) p.off_ownA = take((size_t)M * ld * 8);  // zero-copy A needs no dense A chunk
      if (!b_packed) p.off_ownB = take((size_t)N * ld * 8);  // zero-copy B needs no dense B chunk
      p.max_split = pick_splitk(M, N, std::min<int64_t>(ck, std::max<int64_t>(p.Kb, 1)) * p.bs, num_sms());
    } else {
      for (int k = 0; k < p.L; ++k) {
        if (k % p.pc == p.c) p.ownA_off[k] = take_pool(p.a_panel_bytes(k));
        if (k % p.pr == p.r) p.ownB_off[k] = take_pool(p.b_panel_bytes(k));
      }
      for (int s = 0; s < p.L; ++s) {
        p.max_split = std::max(p.max_split, pick_splitk(M, N, p.kb[p.kappa(s)] * p.bs, num_sms()));
        const std::vector<int64_t> b = pipeline_chunks(p.kb[p.kappa(s)]);  // step 0 may be chunked
        for (size_t j = 1; j < b.size(); ++j)
          p.max_split = std::max(p.max_split, pick_splitk(M, N, (b[j] - b[j - 1]) * p.bs, num_sms()));
        const bool ev = host_pipe_even(true, p.bs);
        for (int j = 0; j < kHostPipeChunks; ++j)  // host-operand pipeline chunks (dbm_multiply_host)
          p.max_split = std::max(p.max_split, pick_splitk(M, N, (host_pipe_bound(p.kb[p.kappa(s)], j + 1, ev) -
                                                                 host_pipe_bound(p.kb[p.kappa(s)], j, ev)) * p.bs,
                                                          num_sms()));
      }
    }
    if (p.max_split > 1) p.off_part = take((size_t)p.max_split * M * N * 8);
  } else {
    // own panels need packing when a rank holds more than one panel per operand, and always for the
    // copy-engine transport (peers pull from this rank's workspace, the IPC-mapped allocation)
    const bool all = nranks > 1 && transport == 0;
    for (int k = 0; k < p.L; ++k) {
      if (k % p.pc == p.c && (all || p.L / p.pc > 1)) p.ownA_off[k] = take_pool(p.a_panel_bytes(k));
      if (k % p.pr == p.r && (all || p.L / p.pr > 1)) p.ownB_off[k] = take_pool(p.b_panel_bytes(k));
    }
    p.off_trav = take((size_t)std::max<int64_t>(p.mloc * p.nloc, 1) * 8);
    int64_t maxkb = 1;
    for (int k = 0; k < p.L; ++k) maxkb = std::max(maxkb, p.kb[k]);
    // chunks hold whole runs, a multiple of the smm group size (8 runs, 16 for the 4 x 4 squares), at
    // least one group
    const int64_t runs = std::max<int64_t>(16, kTripChunkEntries / maxkb / 16 * 16);
    p.trip_cap = std::min<int64_t>(runs, round_up(std::max<int64_t>(p.mloc * p.nloc, 1), 16)) * maxkb;
    p.off_trip = take((size_t)p.trip_cap * 12);
    // several stack chunks per step: a second triplet buffer, so chunk c+1 is generated (side stream)
    // while chunk c multiplies
    if (stackgen_dbuf() && runs < round_up(std::max<int64_t>(p.mloc * p.nloc, 1), 16))
      p.off_trip2 = take((size_t)p.trip_cap * 12);
    // split-K partials of the smm kernel (rectangular shapes with few, long runs)
    const int64_t chunk_runs = std::max<int64_t>(1, std::min<int64_t>(p.mloc * p.nloc, p.trip_cap / maxkb));
    int64_t max_split = 1;
    for (int k = 0; k < p.L; ++k)
      if (p.kb[k] > 0)
        max_split = std::max<int64_t>({max_split, (int64_t)smm_pick_split((int)bs, chunk_runs, p.kb[k]),
                                       (int64_t)smm_pick_split((int)bs, chunk_runs, p.kb[k], true)});
    if (max_split > 1) {
      p.spart_runs = max_split * chunk_runs;
      p.off_spart = take((size_t)p.spart_runs * bs * bs * 8);
    }
    p.mixed = bs == 22 && p.mloc >= 4 && p.nloc >= 4 && !bisection_squares(p.mloc, p.nloc);
    if (p.mixed) {
      const int64_t nsq = (p.mloc / 4) * (p.nloc / 4);
      p.off_pos = take((size_t)p.mloc * p.nloc * 4);
      p.off_sqflag = take((size_t)nsq);
      p.off_sqids = take((size_t)nsq * 4);
      p.off_runsq = take((size_t)chunk_runs * 4);
      p.off_runleft = take((size_t)chunk_runs * 4);
      p.off_runflag = take((size_t)chunk_runs);
      p.off_counts = take(16);
      p.mtemp_bytes = smm22_mixed_temp_bytes(std::max<int64_t>(nsq, chunk_runs));
      p.off_mtemp = take(p.mtemp_bytes);
    }
  }
  if (nranks > 1) {
    size_t amax = 0, bmax = 0;
    int nA = 0, nB = 0;
    for (int s = 0; s < p.L; ++s) {
      if (p.a_src(s) != p.me()) {
        amax = std::max(amax, p.a_panel_bytes(p.kappa(s)));
        ++nA;
      }
      if (p.b_src(s) != p.me()) {
        bmax = std::max(bmax, p.b_panel_bytes(p.kappa(s)));
        ++nB;
      }
    }
    for (int i = 0; i < std::min(nA, 2); ++i) p.off_recvA[i] = take(amax);
    for (int i = 0; i < std::min(nB, 2); ++i) p.off_recvB[i] = take(bmax);
  }
  p.total = std::max<size_t>(off, 256);
  p.pool_total = nranks > 1 ? poff : 0;
  return p;
}

// The MPI-level algorithm for these operands (§II: Cannon for general matrices, the
// tall-and-skinny algorithm "only for tall-and-skinny matrices (one large dimension)"): algorithm 2
// picks tall-and-skinny when K >= 16 max(M, N) on several ranks (densified path, copy engines).
bool use_tallskinny(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, bool densified) {
  if (ctx->nranks <= 1) return false;
  if (ctx->algorithm == 1) return true;
  if (ctx->algorithm != 2 || !densified || ctx->transport != 0) return false;
  return A->cols >= 16 * std::max(A->rows, B->cols);
}

// Opt-in variants, measured and not the default:
// DBM_STACKGEN_DBUF=1 generates stack chunk c+1 on a side stream into a second triplet buffer while chunk c
// multiplies (63,360^3 bs 22 blocked: 34.03 vs 34.03 TFLOP/s -- the overlap gains what the co-running
// generation costs the small-block kernel -- for 6.4 GB more workspace);
bool stackgen_dbuf() {
  static const bool on = [] {
    const char* e = getenv("DBM_STACKGEN_DBUF");
    return e && *e == '1';
  }();
  return on;
}

// DBM_ZC_A=1 reads bs-64 A blocks in place (zero-copy A): no A densify, but the M-major A tile's 2-way
// conflicted fragment loads and 4 boxes per stage slow the GEMM by 5 % (63,360^3: 33.9 vs 35.6 TFLOP/s).
bool zero_copy_a() {
  static const bool on = [] {
    const char* e = getenv("DBM_ZC_A");
    return e && *e == '1';
  }();
  return on;
}

Plan make_plan(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, bool densified, bool local_first = true) {
  (void)C;
  const bool zc = densified && A->bs == 64 && !use_tallskinny(ctx, A, B, densified);
  return make_plan_raw(ctx->nranks, ctx->pr, ctx->pc, ctx->myrow, ctx->mycol, A->Mb, B->Nb, A->Nb, A->bs, densified,
                       ctx->chunk_bytes, ctx->transport, zc && !B->sparse, zc && !A->sparse && zero_copy_a(),
                       local_first);
}

// One Cannon exchange step as a list of point-to-point operations (owner-pull, reading R5):
// for every rank whose step-s panel lives here, a send; for each of this rank's remote panels, a recv.
struct XOp {
  int send;     // 1 send, 0 recv
  int operand;  // 0 = A panel, 1 = B panel
  int peer;
  int kappa;
  int64_t bytes;
};

std::vector<XOp> exchange_ops(const Plan& p, int s) {
  std::vector<XOp> ops;
  const int me = p.me();
  for (int rr = 0; rr < p.pr; ++rr)
    for (int cc = 0; cc < p.pc; ++cc) {
      const int dst = rr * p.pc + cc;
      if (dst == me) continue;
      const int k = (rr + cc + s + (p.local_first ? local_first_start(p.pr, p.pc, dst) : 0)) % p.L;
      if (rr == p.r && k % p.pc == p.c) ops.push_back({1, 0, dst, k, (int64_t)p.a_panel_bytes(k)});  // dst needs my A(r,k)
      if (cc == p.c && k % p.pr == p.r) ops.push_back({1, 1, dst, k, (int64_t)p.b_panel_bytes(k)});  // dst needs my B(k,c)
    }
  const int k = p.kappa(s);
  if (p.a_src(s) != me) ops.push_back({0, 0, p.a_src(s), k, (int64_t)p.a_panel_bytes(k)});
  if (p.b_src(s) != me) ops.push_back({0, 1, p.b_src(s), k, (int64_t)p.b_panel_bytes(k)});
  return ops;
}

}  // namespace

namespace dbm {
int local_first_start(int pr, int pc, int rank) {
  const int L = (int)lcm64(pr, pc), P = pr * pc;
  std::vector<int> load(P, 0);
  int mine = 0;
  for (int q = 0; q < P; ++q) {
    const int r = q / pc, c = q % pc;
    int best = 0, best_remote = 3, best_load = 0;
    for (int s = 0; s < L; ++s) {
      const int k = (r + c + s) % L, a = r * pc + k % pc, b = (k % pr) * pc + c;
      const int remote = (a != q) + (b != q), ld = (a != q ? load[a] : 0) + (b != q ? load[b] : 0);
      if (remote < best_remote || (remote == best_remote && ld < best_load)) {
        best = s;
        best_remote = remote;
        best_load = ld;
      }
    }
    const int k = (r + c + best) % L, a = r * pc + k % pc, b = (k % pr) * pc + c;
    if (a != q) ++load[a];
    if (b != q) ++load[b];
    if (q == rank) mine = best;
  }
  return mine;
}

// K-chunk boundaries (blocks) of a transfer -> GEMM pipeline whose first transfer nothing hides (Cannon's
// step 0, the tall-and-skinny gather).  The first chunk is 1/16 of kb and each next one is `growth`
// times larger: the pull of chunk j+1 (copy engines, ~600 GB/s from a peer) must fit under the GEMM of
// chunk j, i.e. growth <= (GEMM time per K-block) / (pull time per K-block) = pipeline_growth(); a
// rank that pulls both operands of a thin 704 x 704 C has a ratio of ~1.5, one that pulls a single
// operand ~3, the tall-and-skinny ranks ~4 (growth is capped at 2).
std::vector<int64_t> pipeline_chunks(int64_t kb, double growth) {
  if (kb <= 0) return {0, 0};  // one empty chunk: its K = 0 GEMM still writes (zeros) the partial
  std::vector<int64_t> b{0};
  double c = std::max(1.0, (double)kb / 16.0);
  while (b.back() < kb) {
    const int64_t n = b.size() >= 15 ? kb - b.back() : std::max<int64_t>(1, (int64_t)c);  // <= 15 chunks
    b.push_back(std::min(kb, b.back() + n));
    c *= growth;
  }
  return b;
}
double pipeline_growth(double gemm_flop_per_kblock, double pull_bytes_per_kblock) {
  if (pull_bytes_per_kblock <= 0) return 2.0;
  const double ratio = (gemm_flop_per_kblock / 36e12) / (pull_bytes_per_kblock / 600e9);
  return std::max(1.0, std::min(2.0, 0.85 * ratio));
}
dbm_status validate(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C) {
  ARG_CHECK(ctx && A && B && C, DBM_ERR_ARG, "null handle");
  ARG_CHECK(A->ctx == ctx && B->ctx == ctx && C->ctx == ctx, DBM_ERR_GRID, "matrices from a different context");
  ARG_CHECK(A->cols == B->rows && A->rows == C->rows && B->cols == C->cols, DBM_ERR_SHAPE, "non-conformant shapes");
  if (!A->nonuni && !B->nonuni && !C->nonuni) {
    ARG_CHECK(A->bs == B->bs && A->bs == C->bs, DBM_ERR_PARTITION, "block sizes differ (K partition mismatch)");
  } else {  // reading R16: the block partitions must agree, K (S:42 PartitionMismatch) and C's rows / columns
    ARG_CHECK(A->Nb == B->Mb && A->Mb == C->Mb && B->Nb == C->Nb, DBM_ERR_PARTITION, "block partitions differ");
    for (int64_t k = 0; k < A->Nb; ++k)
      ARG_CHECK(A->col_size(k) == B->row_size(k), DBM_ERR_PARTITION, "K partition of A and B differs");
    for (int64_t i = 0; i < A->Mb; ++i)
      ARG_CHECK(A->row_size(i) == C->row_size(i), DBM_ERR_PARTITION, "row partition of A and C differs");
    for (int64_t j = 0; j < B->Nb; ++j)
      ARG_CHECK(B->col_size(j) == C->col_size(j), DBM_ERR_PARTITION, "column partition of B and C differs");
  }
  ARG_CHECK(C != A && C != B, DBM_ERR_ALIAS, "C aliases A or B");
  auto overlap = [](dbm_matrix x, dbm_matrix y) {
    if (!x->arena || !y->arena) return false;
    const char *a0 = (const char*)x->arena, *a1 = a0 + x->elems() * 8;
    const char *b0 = (const char*)y->arena, *b1 = b0 + y->elems() * 8;
    return a0 < b1 && b0 < a1;
  };
  ARG_CHECK(!overlap(C, A) && !overlap(C, B), DBM_ERR_ALIAS, "C storage overlaps A or B");
  if (dbm_status s = need_arena(A)) return s;
  if (dbm_status s = need_arena(B)) return s;
  if (dbm_status s = need_arena(C)) return s;
  return DBM_OK;
}

// Densify / undensify a possibly block-sparse matrix (reading R15: absent blocks densify to zeros,
// undensify writes the stored C blocks only).  Panels as launch_densify_cols / _rows.
dbm_status densify_a(dbm_ctx ctx, dbm_matrix A, int64_t col0, int64_t stride, int64_t nk, double* dst, int64_t ld,
                     int layout, cudaStream_t cs) {
  if (A->sparse)
    CUDA_TRY(ctx, launch_sp_densify(A->arena, A->d_ij, A->nnz, A->bs, 0, col0, stride, nk, A->mloc, dst, ld, layout,
                                    cs));
  else
    launch_densify_cols(A->arena, A->mloc, A->nloc, A->bs, col0, stride, nk, dst, ld, layout, cs);
  return DBM_OK;
}
dbm_status densify_b(dbm_ctx ctx, dbm_matrix B, int64_t row0, int64_t stride, int64_t nk, double* dst, int64_t ld,
                     int layout, cudaStream_t cs) {
  if (B->sparse)
    CUDA_TRY(ctx, launch_sp_densify(B->arena, B->d_ij, B->nnz, B->bs, 1, row0, stride, nk, B->nloc, dst, ld, layout,
                                    cs));
  else
    launch_densify_rows(B->arena, B->nloc, B->bs, row0, stride, nk, dst, ld, layout, cs);
  return DBM_OK;
}
void undensify_c(dbm_matrix C, const double* dense, int64_t ld, int nsplit, int64_t split_stride, double alpha,
                 double beta, cudaStream_t cs) {
  if (C->sparse)
    launch_sp_undensify(dense, ld, nsplit, split_stride, C->d_ij, C->nnz, C->bs, alpha, beta, C->arena, cs);
  else
    launch_undensify(dense, ld, nsplit, split_stride, C->mloc, C->nloc, C->bs, alpha, beta, C->arena, cs);
}

}  // namespace dbm


extern "C" dbm_status dbm_debug_first_step(int pr, int pc, int rank, int* first_step) {
  ARG_CHECK(first_step && pr > 0 && pc > 0 && rank >= 0 && rank < pr * pc, DBM_ERR_ARG, "bad grid or rank");
  *first_step = local_first_start(pr, pc, rank);
  return DBM_OK;
}

extern "C" dbm_status dbm_plan_exchange(int pr, int pc, int myrow, int mycol, int64_t Mb, int64_t Nb, int64_t Kb,
                                        int32_t bs, dbm_path path, int step, int32_t* ops, int64_t* bytes,
                                        int* n_ops) {
  ARG_CHECK(n_ops && pr > 0 && pc > 0 && myrow >= 0 && myrow < pr && mycol >= 0 && mycol < pc && bs > 0,
            DBM_ERR_ARG, "bad grid or block size");
  ARG_CHECK(Mb >= 0 && Nb >= 0 && Kb >= 0, DBM_ERR_ARG, "negative block counts");
  const Plan p = make_plan_raw(pr * pc, pr, pc, myrow, mycol, Mb, Nb, Kb, bs, path == DBM_PATH_DENSIFIED,
                               16ll << 30, 0);
  ARG_CHECK(step >= 0 && step < p.L, DBM_ERR_RANGE, "step out of range");
  const std::vector<XOp> v = exchange_ops(p, step);
  if (ops || bytes) {
    ARG_CHECK(*n_ops >= (int)v.size(), DBM_ERR_ARG, "ops buffer too small");
    for (size_t i = 0; i < v.size(); ++i) {
      if (ops) {
        ops[4 * i + 0] = v[i].send;
        ops[4 * i + 1] = v[i].operand;
        ops[4 * i + 2] = v[i].peer;
        ops[4 * i + 3] = v[i].kappa;
      }
      if (bytes) bytes[i] = v[i].bytes;
    }
  }
  *n_ops = (int)v.size();
  return DBM_OK;
}


namespace {

// One Cannon exchange (owner-pull, reading R5): everything this rank sends and receives at step s.
dbm_status post_exchange(dbm_ctx ctx, const Plan& p, int s, char* ws, const double* Aarena, const double* Barena,
                         int bufA, int bufB, int64_t* sent, int64_t* recv) {
  ncclComm_t comm = (ncclComm_t)ctx->nccl;
  NCCL_TRY(ctx, ncclGroupStart());
  for (const XOp& op : exchange_ops(p, s)) {
    const size_t n = (size_t)op.bytes;
    if (op.send) {
      const size_t own = op.operand == 0 ? p.ownA_off[op.kappa] : p.ownB_off[op.kappa];
      const void* src = own != SIZE_MAX ? (const void*)(ctx->xpool + own) : (const void*)(op.operand == 0 ? Aarena : Barena);
      if (n) NCCL_TRY(ctx, ncclSend(src, n / 8, ncclDouble, op.peer, comm, ctx->comm));
      *sent += (int64_t)n;
    } else {
      void* dst = ws + (op.operand == 0 ? p.off_recvA[bufA] : p.off_recvB[bufB]);
      if (n) NCCL_TRY(ctx, ncclRecv(dst, n / 8, ncclDouble, op.peer, comm, ctx->comm));
      *recv += (int64_t)n;
    }
  }
  NCCL_TRY(ctx, ncclGroupEnd());
  return DBM_OK;
}

// ---------------------------------------------------------------- copy-engine transport (CUDA IPC)
// Every rank's workspace (the allocation holding its own densified / packed panels) is mapped into
// its peers with cudaIpcOpenMemHandle; a Cannon exchange is then a set of cudaMemcpyAsync pulls on
// the comm stream, executed by the DMA copy engines over NVLink 5 — no SM is taken from the GEMM.
// Ordering across processes uses two tiny NCCL collectives: the handle all-gather on the comm
// stream (after this rank's own panels are ready: all panels are ready when it completes) and a
// closing all-reduce on the compute stream after the last GEMM (no peer still reads my panels).
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

AddrRangeFn addr_range_fn() {
  static AddrRangeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (AddrRangeFn)p;
  }
  return fn;
}

constexpr int kIpcRec = 128;  // bytes per rank: 64-B handle + 8-B offset, padded

// 64-bit stream memory operations (driver API through the runtime's entry points): an owner publishes
// its own-panel progress into its peers' flag tables with a stream write after each densify chunk,
// and a consumer's copy-engine pull waits on its local table (GEQ) -- no SM and no host in the loop.
typedef CUresult (*StreamValue64Fn)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*DevAttrFn)(int*, CUdevice_attribute, CUdevice);
struct MemOps {
  StreamValue64Fn wait = nullptr, write = nullptr;
  bool ok = false;
};
const MemOps& memops(int device) {
  static MemOps m;
  static bool init = false;
  if (!init) {
    init = true;
    void *w = nullptr, *x = nullptr, *a = nullptr;
    cudaDriverEntryPointQueryResult q1, q2, q3;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &w, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWriteValue64", &x, cudaEnableDefault, &q2) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuDeviceGetAttribute", &a, cudaEnableDefault, &q3) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && q3 == cudaDriverEntryPointSuccess) {
      int v = 0;
      if (((DevAttrFn)a)(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, (CUdevice)device) == CUDA_SUCCESS &&
          v) {
        m.wait = (StreamValue64Fn)w;
        m.write = (StreamValue64Fn)x;
        m.ok = true;
      }
    }
    cudaGetLastError();
  }
  return m;
}

}  // namespace

dbm_status dbm::ipc_exchange(dbm_ctx ctx, void* ws) {
  const int P = ctx->nranks;
  AddrRangeFn fn = addr_range_fn();
  ARG_CHECK(fn, DBM_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t sz = 0;
  if (fn(&base, &sz, (CUdeviceptr)ws) != CUDA_SUCCESS) {
    set_error("cuMemGetAddressRange failed on the workspace");
    ctx->poisoned = DBM_ERR_CUDA;
    return DBM_ERR_CUDA;
  }
  cudaIpcMemHandle_t h;
  CUDA_TRY(ctx, cudaIpcGetMemHandle(&h, (void*)base));
  std::vector<char> mine(kIpcRec, 0), all((size_t)kIpcRec * P, 0);
  const int64_t off = (int64_t)((char*)ws - (char*)base);
  std::memcpy(mine.data(), &h, sizeof(h));
  std::memcpy(mine.data() + 64, &off, sizeof(off));
  if (!ctx->d_scratch) CUDA_TRY(ctx, cudaMalloc(&ctx->d_scratch, (size_t)kIpcRec * (P + 1) + 64));
  char* d_mine = (char*)ctx->d_scratch + 64;
  char* d_all = d_mine + kIpcRec;
  CUDA_TRY(ctx, cudaMemcpyAsync(d_mine, mine.data(), kIpcRec, cudaMemcpyHostToDevice, ctx->comm));
  NCCL_TRY(ctx, ncclAllGather(d_mine, d_all, kIpcRec, ncclChar, (ncclComm_t)ctx->nccl, ctx->comm));
  CUDA_TRY(ctx, cudaMemcpyAsync(all.data(), d_all, (size_t)kIpcRec * P, cudaMemcpyDeviceToHost, ctx->comm));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->comm));
  if ((int)ctx->peer_ws.size() != P) {
    ctx->peer_ws.assign(P, nullptr);
    ctx->peer_handles.assign(P, std::vector<char>());
    ctx->peer_bases.assign(P, nullptr);
  }
  for (int q = 0; q < P; ++q) {
    if (q == ctx->rank) continue;
    const char* rec = all.data() + (size_t)q * kIpcRec;
    std::vector<char> hq(rec, rec + 64);
    int64_t offq;
    std::memcpy(&offq, rec + 64, sizeof(offq));
    if (hq != ctx->peer_handles[q]) {
      if (ctx->peer_bases[q]) cudaIpcCloseMemHandle(ctx->peer_bases[q]);
      cudaIpcMemHandle_t hh;
      std::memcpy(&hh, hq.data(), sizeof(hh));
      void* pb = nullptr;
      CUDA_TRY(ctx, cudaIpcOpenMemHandle(&pb, hh, cudaIpcMemLazyEnablePeerAccess));
      ctx->peer_bases[q] = pb;
      ctx->peer_handles[q] = hq;
    }
    ctx->peer_ws[q] = (char*)ctx->peer_bases[q] + offq;
  }
  ctx->ipc_ws = ws;
  return DBM_OK;
}

size_t dbm::xhdr_bytes(int nranks, int L) {
  if (nranks <= 1) return 0;
  return align256((size_t)8 * nranks * (X_KINDS + 2 * (size_t)L));
}

dbm_status dbm::xattach(dbm_ctx ctx, size_t need, cudaStream_t cs) {
  ARG_CHECK(memops(ctx->device).ok, DBM_ERR_CUDA, "64-bit stream memory operations unavailable");
  if (ctx->xpool && ctx->xpool_bytes >= need && (int)ctx->peer_ws.size() == ctx->nranks) return DBM_OK;
  // Grow the exchange pool.  `need` is the maximum over all ranks (every rank computes every rank's
  // plan), so every rank takes this branch in the same multiply: the registration all-gather below is
  // collective by construction.  A fresh cudaMalloc allocation (not the caller's allocator: CUDA IPC
  // needs a plain allocation, which expandable segments are not).
  const size_t bytes = std::max(round_up((int64_t)need, 2 << 20), (int64_t)(2 << 20));
  char* pool = nullptr;
  CUDA_TRY(ctx, cudaMalloc(&pool, bytes));
  const int L = (int)lcm64(ctx->pr, ctx->pc);
  CUDA_TRY(ctx, cudaMemsetAsync(pool, 0, xhdr_bytes(ctx->nranks, L), cs));  // the header: every word 0
  cudaEvent_t e = get_event(ctx);
  CUDA_TRY(ctx, cudaEventRecord(e, cs));
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm, e, 0));
  ctx->ev_pool.push_back(e);
  if (dbm_status st = ipc_exchange(ctx, pool)) {  // all-gather of the handles after the memset on every rank
    cudaFree(pool);
    return st;
  }
  // the previous pool: every multiply that used it ended with the closing barrier (no peer reads it)
  if (ctx->xpool) cudaFree(ctx->xpool);
  ctx->xpool = pool;
  ctx->xpool_bytes = bytes;
  return DBM_OK;
}

dbm_status dbm::xwrite_word(dbm_ctx ctx, cudaStream_t st, int q, size_t word, uint64_t value) {
  if (memops(ctx->device).write(st, (CUdeviceptr)(ctx->peer_ws[q] + word * 8), (cuuint64_t)value,
                                CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS) {
    set_error("cuStreamWriteValue64 failed");
    ctx->poisoned = DBM_ERR_CUDA;
    return DBM_ERR_CUDA;
  }
  return DBM_OK;
}

dbm_status dbm::xwait_word(dbm_ctx ctx, cudaStream_t st, size_t word, uint64_t value) {
  if (memops(ctx->device).wait(st, (CUdeviceptr)(ctx->xpool + word * 8), (cuuint64_t)value,
                               CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
    set_error("cuStreamWaitValue64 failed");
    ctx->poisoned = DBM_ERR_CUDA;
    return DBM_ERR_CUDA;
  }
  return DBM_OK;
}

dbm_status dbm::xsignal(dbm_ctx ctx, cudaStream_t st, int kind, uint64_t value) {
  for (int q = 0; q < ctx->nranks; ++q)
    if (q != ctx->rank)
      if (dbm_status e = xwrite_word(ctx, st, q, (size_t)kind * ctx->nranks + ctx->rank, value)) return e;
  return DBM_OK;
}

dbm_status dbm::xwait(dbm_ctx ctx, cudaStream_t st, int kind, uint64_t value) {
  for (int q = 0; q < ctx->nranks; ++q)
    if (q != ctx->rank)
      if (dbm_status e = xwait_word(ctx, st, (size_t)kind * ctx->nranks + q, value)) return e;
  return DBM_OK;
}

namespace {

// Pull this rank's step-s panels from their owners' workspaces (peer plans give the offsets).
// Each pull first waits (on its copy stream) until the owner of op's panel has published at least `need`
// K-blocks of it for this multiply (epoch hp_epoch) into this rank's progress table: the whole panel
// behind its densify / pack, or chunk by chunk in the pipelined modes.
// A step's A and B pulls go on two streams (comm, comm2), so two copy engines move them concurrently; the
// B stream forks from the comm stream's state and joins it again at the end of the step's posts.
cudaStream_t pull_stream(dbm_ctx ctx, const XOp& op) { return op.operand == 1 ? ctx->comm2 : ctx->comm; }
dbm_status fork_b(dbm_ctx ctx) {
  cudaEvent_t e = get_event(ctx);
  CUDA_TRY(ctx, cudaEventRecord(e, ctx->comm));
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm2, e, 0));
  ctx->ev_pool.push_back(e);
  return DBM_OK;
}
dbm_status join_b(dbm_ctx ctx) {
  cudaEvent_t e = get_event(ctx);
  CUDA_TRY(ctx, cudaEventRecord(e, ctx->comm2));
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm, e, 0));
  ctx->ev_pool.push_back(e);
  return DBM_OK;
}

dbm_status wait_panel(dbm_ctx ctx, const Plan& p, uint64_t hp_epoch, const XOp& op, int64_t need) {
  if (!hp_epoch || need <= 0) return DBM_OK;
  return xwait_word(ctx, pull_stream(ctx, op), xprog_word(ctx->nranks, p.L, op.peer, op.operand, op.kappa),
                    (hp_epoch << 32) | (uint64_t)need);
}

dbm_status post_pulls(dbm_ctx ctx, const Plan& p, const std::vector<Plan>& peer_plan, int s, char* ws, int bufA,
                      int bufB, int64_t* sent, int64_t* recv, uint64_t hp_epoch = 0) {
  if (dbm_status e = fork_b(ctx)) return e;
  for (const XOp& op : exchange_ops(p, s)) {
    const size_t n = (size_t)op.bytes;
    if (op.send) {  // the peer pulls it; counted for the statistics
      *sent += (int64_t)n;
      continue;
    }
    if (dbm_status e = wait_panel(ctx, p, hp_epoch, op, p.kb[op.kappa])) return e;
    const Plan& q = peer_plan[op.peer];
    const size_t src_off = op.operand == 0 ? q.ownA_off[op.kappa] : q.ownB_off[op.kappa];
    ARG_CHECK(src_off != SIZE_MAX && ctx->peer_ws[op.peer], DBM_ERR_PLAN, "peer panel not in its workspace");
    void* dst = ws + (op.operand == 0 ? p.off_recvA[bufA] : p.off_recvB[bufB]);
    if (n)
      CUDA_TRY(ctx, cudaMemcpyAsync(dst, ctx->peer_ws[op.peer] + src_off, n, cudaMemcpyDeviceToDevice,
                                    pull_stream(ctx, op)));
    *recv += (int64_t)n;
  }
  return join_b(ctx);
}

// K-chunk [k0, k1) (blocks) of this rank's step-s dense panels: one 2-D copy-engine pull per remote
// operand (rows x chunk width, pitch = the panel's leading dimension).  Statistics count the whole
// panel once (count == true on the first chunk).
dbm_status post_pulls_chunk(dbm_ctx ctx, const Plan& p, const std::vector<Plan>& peer_plan, int s, char* ws, int bufA,
                            int bufB, int64_t k0, int64_t k1, bool count, int64_t* sent, int64_t* recv,
                            uint64_t hp_epoch = 0) {
  if (dbm_status e = fork_b(ctx)) return e;
  for (const XOp& op : exchange_ops(p, s)) {
    if (op.send) {
      if (count) *sent += op.bytes;
      continue;
    }
    if (k1 > k0)
      if (dbm_status e = wait_panel(ctx, p, hp_epoch, op, k1)) return e;
    const Plan& q = peer_plan[op.peer];
    const size_t src_off = op.operand == 0 ? q.ownA_off[op.kappa] : q.ownB_off[op.kappa];
    ARG_CHECK(src_off != SIZE_MAX && ctx->peer_ws[op.peer], DBM_ERR_PLAN, "peer panel not in its workspace");
    // densified: dense K-major panels (rows x ld doubles); blocked: packed block panels, A row-major
    // over (li, kk) (mloc rows of kb blocks), B over (kk, lj) (a K-chunk is one contiguous range)
    const size_t bb8 = (size_t)p.bs * p.bs * 8;
    int64_t rows;
    size_t pitch, off, width;
    if (p.densified && !(op.operand == 1 && p.b_packed) && !(op.operand == 0 && p.a_packed)) {
      rows = (op.operand == 0 ? p.mloc : p.nloc) * p.bs;
      pitch = (size_t)p.ld_panel(op.kappa) * 8;
      off = (size_t)(k0 * p.bs) * 8;
      width = (size_t)((k1 - k0) * p.bs) * 8;
    } else if (op.operand == 0) {
      rows = p.mloc;
      pitch = (size_t)p.kb[op.kappa] * bb8;
      off = (size_t)k0 * bb8;
      width = (size_t)(k1 - k0) * bb8;
    } else {
      rows = 1;
      off = (size_t)(k0 * p.nloc) * bb8;
      width = pitch = (size_t)((k1 - k0) * p.nloc) * bb8;
    }
    char* dst = ws + (op.operand == 0 ? p.off_recvA[bufA] : p.off_recvB[bufB]) + off;
    const char* src = ctx->peer_ws[op.peer] + src_off + off;
    if (rows && width)
      CUDA_TRY(ctx, cudaMemcpy2DAsync(dst, pitch, src, pitch, width, rows, cudaMemcpyDeviceToDevice,
                                      pull_stream(ctx, op)));
    if (count) *recv += op.bytes;
  }
  return join_b(ctx);
}

__global__ void scale_kernel(double* __restrict__ x, int64_t n, double beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = beta == 0.0 ? 0.0 : beta * x[i];
}

}  // namespace

void dbm::launch_scale(double* x, int64_t n, double beta, cudaStream_t st) {
  if (n <= 0) return;
  scale_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, num_sms() * 16), 256, 0, st>>>(x, n, beta);
}

namespace {

}  // namespace



extern "C" dbm_status dbm_multiply_workspace(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, dbm_path path,
                                             int64_t* bytes) {
  ARG_CHECK(bytes, DBM_ERR_ARG, "null output");
  ARG_CHECK(path == DBM_PATH_BLOCKED || path == DBM_PATH_DENSIFIED || path == DBM_PATH_AUTO, DBM_ERR_ARG, "bad path");
  if (dbm_status s = validate(ctx, A, B, C)) return s;
  path = resolve_path(ctx, A, B, path);
  if (A->nonuni || B->nonuni || C->nonuni) return nu_workspace_bytes(ctx, A, B, C, path == DBM_PATH_DENSIFIED, bytes);
  if (path == DBM_PATH_BLOCKED && (A->sparse || B->sparse || C->sparse)) {
    return sp_workspace_bytes(ctx, A, B, C, bytes);
  }
  if (use_tallskinny(ctx, A, B, path == DBM_PATH_DENSIFIED))
    *bytes = (int64_t)ts_workspace_bytes(ctx->pr, ctx->pc, ctx->myrow, ctx->mycol, A->Mb, B->Nb, A->Nb, A->bs);
  else
    *bytes = (int64_t)make_plan(ctx, A, B, C, path == DBM_PATH_DENSIFIED).total;
  return DBM_OK;
}

extern "C" dbm_status dbm_plan_tallskinny(int pr, int pc, int myrow, int mycol, int64_t Mb, int64_t Nb, int64_t Kb,
                                          int32_t bs, int64_t* bytes_recv, int64_t* bytes_sent) {
  ARG_CHECK(bytes_recv && bytes_sent && pr > 0 && pc > 0 && myrow >= 0 && myrow < pr && mycol >= 0 && mycol < pc &&
                bs > 0 && Mb >= 0 && Nb >= 0 && Kb >= 0,
            DBM_ERR_ARG, "bad arguments");
  ts_plan_bytes(pr, pc, myrow, mycol, Mb, Nb, Kb, bs, bytes_recv, bytes_sent);
  return DBM_OK;
}

// Host-resident operands (dbm_multiply_host): pinned host arenas streamed to the device arenas on
// the comm stream; chunk_ev[ch] marks A/B K-chunk ch of the single-rank densified path uploaded,
// all_ev everything uploaded (other paths), c_ev C_in uploaded.

struct HostIO {
  const double* A = nullptr;
  const double* B = nullptr;
  double* C = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  cudaEvent_t all_ev = nullptr, c_ev = nullptr;
  std::vector<cudaEvent_t> panel_ev;  // C row panels ready for their download
  cudaEvent_t a_ev = nullptr;         // A uploaded (several ranks: A's own panels start while B uploads)
  bool b_deferred = false;            // the wait for B's upload sits before B's own panels
  bool c_downloaded = false;          // the multiply already enqueued C's download
  std::vector<cudaEvent_t> up_ev;     // several ranks, pipelined: upload chunk j landed (ctx->up)
};

namespace {
// Single-rank densified K-chunks (block boundaries).  Device-resident operands: uniform chunks of the
// dense-buffer budget.  Host-resident operands (dbm_multiply_host): the chunks start at 1/16 of K and
// double up to the budget, so only a small first upload is exposed; every later upload (PCIe, ~12x
// faster per K-block than the GEMM consumes it at 63,360^3) runs under the previous chunks' GEMMs.
std::vector<int64_t> k_chunks(int64_t Kb, int64_t budget, bool host_io) {
  std::vector<int64_t> b{0};
  int64_t step = host_io ? std::max<int64_t>(1, Kb / 16) : budget;
  while (b.back() < Kb) {
    b.push_back(std::min(Kb, b.back() + std::min(step, budget)));
    if (host_io) step *= 2;
  }
  if (b.size() == 1) b.push_back(0);
  return b;
}
}  // namespace

namespace {
dbm_status multiply_impl(dbm_ctx ctx, double alpha, dbm_matrix A, dbm_matrix B, double beta, dbm_matrix C,
                         dbm_path path, int32_t stack_cap, void* workspace, int64_t ws_bytes, dbm_stats* stats,
                         HostIO* hio);
}

// Profiled multiplies are bracketed (dbm_multiply_timing): events on the ctx stream + the record range.
struct TimingBracket {
  dbm_ctx ctx;
  bool on;
  explicit TimingBracket(dbm_ctx c) : ctx(c), on(c && c->profiling && c->poisoned == DBM_OK) {
    if (!on) return;
    if (!ctx->lt_a) cudaEventCreate(&ctx->lt_a);
    if (!ctx->lt_b) cudaEventCreate(&ctx->lt_b);
    cudaEventRecord(ctx->lt_a, ctx->stream);
    ctx->lt_first = ctx->prof.size();
    ctx->lt_valid = false;
  }
  void done(dbm_status s) {
    if (!on || s != DBM_OK) return;
    cudaEventRecord(ctx->lt_b, ctx->stream);
    ctx->lt_last = ctx->prof.size();
    ctx->lt_valid = true;
  }
};

extern "C" dbm_status dbm_multiply(dbm_ctx ctx, double alpha, dbm_matrix A, dbm_matrix B, double beta, dbm_matrix C,
                                   dbm_path path, int32_t stack_cap, void* workspace, int64_t ws_bytes,
                                   dbm_stats* stats) {
  TimingBracket tb(ctx);
  const dbm_status s = multiply_impl(ctx, alpha, A, B, beta, C, path, stack_cap, workspace, ws_bytes, stats, nullptr);
  tb.done(s);
  return s;
}

extern "C" dbm_status dbm_multiply_timing(dbm_ctx ctx, dbm_stats* st) {
  CTX_OK(ctx);
  ARG_CHECK(st, DBM_ERR_ARG, "null stats");
  ARG_CHECK(ctx->lt_valid && ctx->prof.size() >= ctx->lt_last, DBM_ERR_ARG,
            "no profiled multiply pending (dbm_ctx_set_profiling, and before dbm_ctx_profile_read)");
  CUDA_TRY(ctx, cudaEventSynchronize(ctx->lt_b));
  float t = 0;
  CUDA_TRY(ctx, cudaEventElapsedTime(&t, ctx->lt_a, ctx->lt_b));
  double ph[6] = {0, 0, 0, 0, 0, 0};
  for (size_t i = ctx->lt_first; i < ctx->lt_last; ++i) {
    const auto& r = ctx->prof[i];
    CUDA_TRY(ctx, cudaEventSynchronize(r.b));
    float d = 0;
    CUDA_TRY(ctx, cudaEventElapsedTime(&d, r.a, r.b));
    if (r.kind >= 0 && r.kind < 6) ph[r.kind] += d;
  }
  st->ms_total = t;
  st->ms_densify = ph[2];
  st->ms_local = ph[0] + ph[1] + ph[4];
  st->ms_undensify = ph[3];
  st->ms_comm_exposed = std::max(0.0, st->ms_total - st->ms_densify - st->ms_local - st->ms_undensify);
  return DBM_OK;
}

extern "C" dbm_status dbm_multiply_host(dbm_ctx ctx, double alpha, dbm_matrix A, dbm_matrix B, double beta,
                                        dbm_matrix C, dbm_path path, int32_t stack_cap, void* workspace,
                                        int64_t ws_bytes, const void* A_host, const void* B_host, void* C_host,
                                        dbm_stats* stats) {
  CTX_OK(ctx);
  ARG_CHECK(A_host && B_host && C_host, DBM_ERR_ARG, "null host buffer");
  auto pinned = [](const void* p) {
    cudaPointerAttributes at;
    const bool ok = cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return ok;
  };
  if (!pinned(A_host) || !pinned(B_host) || !pinned(C_host)) {
    // pageable: staged through the pinned double buffer, no overlap with the multiply
    if (dbm_status e = dbm_matrix_upload(A, A_host)) return e;
    if (dbm_status e = dbm_matrix_upload(B, B_host)) return e;
    if (beta != 0.0)
      if (dbm_status e = dbm_matrix_upload(C, C_host)) return e;
    if (dbm_status e = dbm_multiply(ctx, alpha, A, B, beta, C, path, stack_cap, workspace, ws_bytes, stats)) return e;
    return dbm_matrix_download(C, C_host);
  }
  HostIO hio;
  hio.A = (const double*)A_host;
  hio.B = (const double*)B_host;
  hio.C = (double*)C_host;
  TimingBracket tb(ctx);
  dbm_status e = multiply_impl(ctx, alpha, A, B, beta, C, path, stack_cap, workspace, ws_bytes, stats, &hio);
  for (cudaEvent_t ev : hio.chunk_ev) ctx->ev_pool.push_back(ev);
  for (cudaEvent_t ev : hio.panel_ev) ctx->ev_pool.push_back(ev);
  for (cudaEvent_t ev : hio.up_ev) ctx->ev_pool.push_back(ev);
  if (hio.all_ev) ctx->ev_pool.push_back(hio.all_ev);
  if (hio.a_ev) ctx->ev_pool.push_back(hio.a_ev);
  if (hio.c_ev) ctx->ev_pool.push_back(hio.c_ev);
  if (e) return e;
  const size_t cbytes = (size_t)C->elems() * 8;
  if (cbytes && !hio.c_downloaded)
    CUDA_TRY(ctx, cudaMemcpyAsync(C_host, C->arena, cbytes, cudaMemcpyDeviceToHost, ctx->stream));
  tb.done(DBM_OK);
  return DBM_OK;
}

namespace {
dbm_status multiply_impl(dbm_ctx ctx, double alpha, dbm_matrix A, dbm_matrix B, double beta, dbm_matrix C,
                         dbm_path path, int32_t stack_cap, void* workspace, int64_t ws_bytes, dbm_stats* stats,
                         HostIO* hio) {
  CTX_OK(ctx);
  ARG_CHECK(path == DBM_PATH_BLOCKED || path == DBM_PATH_DENSIFIED || path == DBM_PATH_AUTO, DBM_ERR_ARG, "bad path");
  ARG_CHECK(stack_cap >= 0, DBM_ERR_ARG, "negative stack cap");
  if (dbm_status s = validate(ctx, A, B, C)) return s;
  path = resolve_path(ctx, A, B, path);
  const bool dens = path == DBM_PATH_DENSIFIED;
  if (A->nonuni || B->nonuni || C->nonuni) {  // non-uniform block sizes (reading R16)
    ARG_CHECK(ctx->transport == 0 && ctx->algorithm != 1, DBM_ERR_ARG,
              "non-uniform blocks: Cannon over the copy-engine transport");
    if (hio) {  // host operands: plain uploads ahead of the multiply on the compute stream
      if (A->elems()) CUDA_TRY(ctx, cudaMemcpyAsync(A->arena, hio->A, A->elems() * 8, cudaMemcpyHostToDevice, ctx->stream));
      if (B->elems()) CUDA_TRY(ctx, cudaMemcpyAsync(B->arena, hio->B, B->elems() * 8, cudaMemcpyHostToDevice, ctx->stream));
      if (beta != 0.0 && C->elems())
        CUDA_TRY(ctx, cudaMemcpyAsync(C->arena, hio->C, C->elems() * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    return multiply_nonuniform(ctx, alpha, A, B, beta, C, dens, workspace, ws_bytes, stats);
  }
  if (!dens && (A->sparse || B->sparse || C->sparse)) {
    if (hio) {  // host operands: plain uploads ahead of the multiply on the compute stream
      const size_t bb8 = (size_t)A->bs * A->bs * 8;
      const size_t ab = (size_t)A->blocks() * bb8, bbytes = (size_t)B->blocks() * bb8, cb = (size_t)C->blocks() * bb8;
      if (ab) CUDA_TRY(ctx, cudaMemcpyAsync(A->arena, hio->A, ab, cudaMemcpyHostToDevice, ctx->stream));
      if (bbytes) CUDA_TRY(ctx, cudaMemcpyAsync(B->arena, hio->B, bbytes, cudaMemcpyHostToDevice, ctx->stream));
      if (beta != 0.0 && cb) CUDA_TRY(ctx, cudaMemcpyAsync(C->arena, hio->C, cb, cudaMemcpyHostToDevice, ctx->stream));
    }
    return multiply_sparse_blocked(ctx, alpha, A, B, beta, C, stack_cap, workspace, ws_bytes, stats);
  }
  if (use_tallskinny(ctx, A, B, dens)) {
    ARG_CHECK(dens, DBM_ERR_ARG, "the tall-and-skinny algorithm runs the densified local multiply");
    ARG_CHECK(ctx->transport == 0, DBM_ERR_ARG, "the tall-and-skinny algorithm uses the copy-engine transport");
    const size_t ts_total = ts_workspace_bytes(ctx->pr, ctx->pc, ctx->myrow, ctx->mycol, A->Mb, B->Nb, A->Nb, A->bs);
    ARG_CHECK(workspace != nullptr && ws_bytes >= (int64_t)ts_total, DBM_ERR_WORKSPACE,
              "workspace smaller than dbm_multiply_workspace()");
    dbm_stats st{};
    int launches = 0;
    if (hio) {  // host operands: plain uploads ahead of the multiply on the compute stream
      const size_t bb8 = (size_t)A->bs * A->bs * 8;
      const size_t ab = (size_t)A->blocks() * bb8, bbytes = (size_t)B->blocks() * bb8,
                   cb = (size_t)C->blocks() * bb8;
      if (ab) CUDA_TRY(ctx, cudaMemcpyAsync(A->arena, hio->A, ab, cudaMemcpyHostToDevice, ctx->stream));
      if (bbytes) CUDA_TRY(ctx, cudaMemcpyAsync(B->arena, hio->B, bbytes, cudaMemcpyHostToDevice, ctx->stream));
      if (beta != 0.0 && cb) CUDA_TRY(ctx, cudaMemcpyAsync(C->arena, hio->C, cb, cudaMemcpyHostToDevice, ctx->stream));
    }
    if (alpha == 0.0 || A->Nb == 0) {
      const int64_t n = C->blocks() * (int64_t)C->bs * C->bs;
      if (n) {
        launch_scale(C->arena, n, beta, ctx->stream);
        ++launches;
        CUDA_TRY(ctx, cudaGetLastError());
      }
    } else if (dbm_status e = multiply_tallskinny(ctx, alpha, A, B, beta, C, (char*)workspace, &st, &launches)) {
      return e;
    }
    ctx->launches += launches;
    st.kernel_launches = launches;
    if (stats) *stats = st;
    return DBM_OK;
  }
  const Plan p = make_plan(ctx, A, B, C, dens);
  ARG_CHECK(workspace != nullptr && ws_bytes >= (int64_t)p.total, DBM_ERR_WORKSPACE,
            "workspace smaller than dbm_multiply_workspace()");
  const int64_t cap = stack_cap ? stack_cap : 30000;
  // host operands on several ranks (densified Cannon, copy engines): uploads, own-panel densify and the
  // step-0 pull + GEMM run chunk by chunk, the pulls gated by the owners' published progress
  const bool hpipe = hio && ctx->nranks > 1 && ctx->transport == 0 && ctx->host_pipe && alpha != 0.0 && p.Kb > 0 &&
                     !A->sparse && !B->sparse && !C->sparse && memops(ctx->device).ok;
  // the same pipeline for device-resident operands (no uploads; opt-in, DBM_DEV_PIPE=1): this rank's own
  // panels are densified / packed chunk by chunk on the own-panel stream, each chunk's progress published
  // at once, so the peers' step-0 pulls and this rank's step-0 chunks start behind the first chunk instead
  // of behind the whole panel.  Measured on 4 GPUs it loses on the rectangular configs (1,408^2 x
  // 1,982,464 bs 64 128.5 -> 124.0 TFLOP/s, bs 22 blocked 116.4 -> 114.5): the later chunks' densify /
  // pack kernels find no free SM beside the persistent GEMM / small-block kernel (its CTAs hold every
  // SM's register file), so they run only in the gaps between chunks and the peers' pulls trail them.
  const bool dpipe = !hio && ctx->nranks > 1 && ctx->transport == 0 && ctx->dev_pipe && alpha != 0.0 && p.Kb > 0 &&
                     !A->sparse && !B->sparse && !C->sparse && memops(ctx->device).ok;
  const bool pipe = hpipe || dpipe;
  cudaEvent_t dpipe_e0 = nullptr;
  if (dpipe) {
    if (!ctx->own) CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking));
    dpipe_e0 = get_event(ctx);
    CUDA_TRY(ctx, cudaEventRecord(dpipe_e0, ctx->stream));  // previous work on the arenas is done
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->own, dpipe_e0, 0));
  }
  const bool hp_even = host_pipe_even(dens, p.bs);
  if (hpipe) {
    cudaEvent_t e0 = get_event(ctx);
    CUDA_TRY(ctx, cudaEventRecord(e0, ctx->stream));  // previous work on the arenas is done
    hio->chunk_ev.push_back(e0);
    if (!ctx->up) CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->up, cudaStreamNonBlocking));
    if (!ctx->own) CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking));
    cudaStream_t up = ctx->up;
    CUDA_TRY(ctx, cudaStreamWaitEvent(up, e0, 0));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->own, e0, 0));  // the own-panel stream starts after earlier work too
    const size_t bb8 = (size_t)p.bs * p.bs * 8;
    const size_t cbytes = beta != 0.0 ? (size_t)C->blocks() * bb8 : 0;
    if (!dens) {  // the blocked path accumulates into C from the first chunk on: C_in goes first
      if (cbytes) CUDA_TRY(ctx, cudaMemcpyAsync(C->arena, hio->C, cbytes, cudaMemcpyHostToDevice, up));
      hio->c_ev = get_event(ctx);
      CUDA_TRY(ctx, cudaEventRecord(hio->c_ev, up));
    }
    int64_t loA = 0, loB = 0;
    for (int j = 0; j < kHostPipeChunks; ++j) {
      // local A columns / B rows that hold the first host_pipe_bound(kb, j + 1) blocks of every own panel
      int64_t hiA = loA, hiB = loB;
      for (int k = 0; k < p.L; ++k) {
        const int64_t q1 = host_pipe_bound(p.kb[k], j + 1, hp_even);
        if (q1 <= 0) continue;
        if (k % p.pc == p.c) hiA = std::max(hiA, (k - p.c) / p.pc + (q1 - 1) * (p.L / p.pc) + 1);
        if (k % p.pr == p.r) hiB = std::max(hiB, (k - p.r) / p.pr + (q1 - 1) * (p.L / p.pr) + 1);
      }
      if (j == kHostPipeChunks - 1) {
        hiA = p.kA;
        hiB = p.kB;
      }
      if (p.mloc && hiA > loA)
        CUDA_TRY(ctx, cudaMemcpy2DAsync((char*)A->arena + loA * bb8, p.kA * bb8, (const char*)hio->A + loA * bb8,
                                        p.kA * bb8, (hiA - loA) * bb8, p.mloc, cudaMemcpyHostToDevice, up));
      if (p.nloc && hiB > loB)
        CUDA_TRY(ctx, cudaMemcpyAsync((char*)B->arena + loB * p.nloc * bb8, (const char*)hio->B + loB * p.nloc * bb8,
                                      (hiB - loB) * p.nloc * bb8, cudaMemcpyHostToDevice, up));
      cudaEvent_t e = get_event(ctx);
      CUDA_TRY(ctx, cudaEventRecord(e, up));
      hio->up_ev.push_back(e);
      loA = hiA;
      loB = hiB;
    }
    if (dens) {  // the densified path reads C_in only in the undensify
      if (cbytes) CUDA_TRY(ctx, cudaMemcpyAsync(C->arena, hio->C, cbytes, cudaMemcpyHostToDevice, up));
      hio->c_ev = get_event(ctx);
      CUDA_TRY(ctx, cudaEventRecord(hio->c_ev, up));
    }
  } else if (hio) {
    // Stream the host operands in (P:174 double buffering; P:200 page-locked host memory).  The
    // single-rank densified path consumes A and B one K-chunk at a time, so chunk ch's upload only
    // has to precede chunk ch's densify and overlaps the GEMMs of the chunks before it.
    cudaStream_t cp = ctx->comm;
    CUDA_TRY(ctx, cudaStreamWaitEvent(cp, [&] {
      cudaEvent_t e0 = get_event(ctx);
      cudaEventRecord(e0, ctx->stream);  // previous work on the arenas is done
      hio->chunk_ev.push_back(e0);
      return e0;
    }(), 0));
    const size_t bb8 = (size_t)p.bs * p.bs * 8;
    const bool chunked = ctx->nranks == 1 && dens && alpha != 0.0 && p.Kb > 0 && !A->sparse && !B->sparse;
    if (chunked) {
      const std::vector<int64_t> kc = k_chunks(p.Kb, p.chunk_kb, true);
      for (size_t ch = 0; ch + 1 < kc.size(); ++ch) {
        const int64_t k0 = kc[ch], nk = kc[ch + 1] - kc[ch];
        if (p.mloc && nk)
          CUDA_TRY(ctx, cudaMemcpy2DAsync((char*)A->arena + k0 * bb8, p.kA * bb8, (const char*)hio->A + k0 * bb8,
                                          p.kA * bb8, nk * bb8, p.mloc, cudaMemcpyHostToDevice, cp));
        if (p.nloc && nk)
          CUDA_TRY(ctx, cudaMemcpyAsync((char*)B->arena + k0 * p.nloc * bb8, (const char*)hio->B + k0 * p.nloc * bb8,
                                        nk * p.nloc * bb8, cudaMemcpyHostToDevice, cp));
        cudaEvent_t e = get_event(ctx);
        CUDA_TRY(ctx, cudaEventRecord(e, cp));
        hio->chunk_ev.push_back(e);  // chunk_ev[ch + 1]
      }
    } else {
      const size_t ab = (size_t)A->blocks() * bb8, bbytes = (size_t)B->blocks() * bb8;
      if (ab && alpha != 0.0) CUDA_TRY(ctx, cudaMemcpyAsync(A->arena, hio->A, ab, cudaMemcpyHostToDevice, cp));
      hio->a_ev = get_event(ctx);
      CUDA_TRY(ctx, cudaEventRecord(hio->a_ev, cp));
      if (bbytes && alpha != 0.0) CUDA_TRY(ctx, cudaMemcpyAsync(B->arena, hio->B, bbytes, cudaMemcpyHostToDevice, cp));
      hio->all_ev = get_event(ctx);
      CUDA_TRY(ctx, cudaEventRecord(hio->all_ev, cp));
    }
    const size_t cb = (size_t)C->blocks() * bb8;
    if (beta != 0.0 && cb) CUDA_TRY(ctx, cudaMemcpyAsync(C->arena, hio->C, cb, cudaMemcpyHostToDevice, cp));
    hio->c_ev = get_event(ctx);
    CUDA_TRY(ctx, cudaEventRecord(hio->c_ev, cp));
    if (!chunked || beta != 0.0 || alpha == 0.0 || p.Kb == 0) {
      // paths that touch C (or all of A, B) early wait for everything; on several ranks A's own panels
      // are built while B still uploads (the wait for B moves in front of B's own panels)
      hio->b_deferred = ctx->nranks > 1 && alpha != 0.0 && p.Kb > 0 && hio->a_ev && beta == 0.0;
      if (hio->b_deferred)
        CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, hio->a_ev, 0));
      else if (hio->all_ev)
        CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, hio->all_ev, 0));
      if ((!chunked || alpha == 0.0 || p.Kb == 0) && !hio->b_deferred)
        CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, hio->c_ev, 0));
    }
  }
  dbm_stats st{};
  st.steps = p.L;
  int launches = 0;
  cudaStream_t cs = ctx->stream;
  char* ws = (char*)workspace;
  const int64_t bs = p.bs, M = p.mloc * bs, N = p.nloc * bs;
  const int64_t bb = bs * bs;

  // BLAS convention: alpha == 0 -> A and B are not read (reading R8).
  if (alpha == 0.0 || p.Kb == 0) {
    const int64_t n = C->blocks() * bb;
    if (n) {
      launch_scale(C->arena, n, beta, cs);
      ++launches;
      CUDA_TRY(ctx, cudaGetLastError());
    }
    ctx->launches += launches;
    st.kernel_launches = launches;
    if (stats) *stats = st;
    return DBM_OK;
  }

  // ------------------------------------------------ the exchange pool (several ranks)
  char* xp = nullptr;  // this rank's exchange pool: signal header + own panels (the peers pull them)
  uint64_t ep = 0;     // this multiply's epoch
  if (ctx->nranks > 1) {
    size_t need = p.pool_total;
    for (int q = 0; q < ctx->nranks; ++q)
      need = std::max(need, make_plan_raw(ctx->nranks, p.pr, p.pc, q / p.pc, q % p.pc, p.Mb, p.Nb, p.Kb, p.bs, dens,
                                          ctx->chunk_bytes, ctx->transport, p.b_packed, p.a_packed,
                                          p.local_first).pool_total);
    if (dbm_status e = xattach(ctx, need, cs)) return e;
    xp = ctx->xpool;
    ep = ++ctx->epoch;
  }

  // copy-engine pulls write only this rank's receive buffers: they wait for the compute stream's work
  // up to here (the previous multiply's reads of those buffers), not for the own panels packed next
  // (each pull waits on its panel's progress word instead)
  cudaEvent_t ev_prior = nullptr;
  bool ce_ident_a = false, ce_ident_b = false;  // own panel copied by the copy engine (see below)
  if (ctx->nranks > 1 && ctx->transport == 0) {
    ev_prior = get_event(ctx);
    CUDA_TRY(ctx, cudaEventRecord(ev_prior, cs));
  }

  // ------------------------------------------------ own panels (densify or pack), on the compute stream
  // Copy-engine transport: each own panel's completion goes into every peer's progress table as soon as
  // it is in place ((epoch << 32) | its K-blocks), and a peer's pull of that panel waits on exactly that
  // word -- not on a "all my panels are ready" signal -- so the operand the peers pull first is packed
  // first and released alone (on 2 x 2 with the local-first order: the B panels).
  if (ctx->nranks > 1 && !pipe) {
    const bool ce = ctx->transport == 0;
    auto publish_panel = [&](int operand, int k, cudaStream_t st) -> dbm_status {
      if (!ce) return DBM_OK;
      for (int q = 0; q < ctx->nranks; ++q)
        if (q != ctx->rank)
          if (dbm_status e = xwrite_word(ctx, st, q, xprog_word(ctx->nranks, p.L, ctx->rank, operand, k),
                                         (ep << 32) | (uint64_t)p.kb[k]))
            return e;
      return DBM_OK;
    };
    // Packed panels (blocked path; the densified path's zero-copy B / A for bs 64) of dense operands with
    // L = pc (A) / L = pr (B): the rank's one own panel of that operand is its arena verbatim (packed panel
    // = row-major blocks = the local CSR order), so with DBM_CE_PACK=1 the local steps read the arena and
    // the pool copy the peers pull is a cudaMemcpyAsync on the own-panel stream.  Opt-in: a same-device
    // copy needs the SMs (it does not go to a copy engine), so when the persistent GEMM / small-block
    // kernel starts first the copy -- and the peers' first pulls behind it -- wait for that kernel (one
    // 4-GPU session: 28 ms of idle per multiply on two ranks); the pack kernels on the compute stream
    // stay the default.
    ce_ident_a = ce && (!dens || p.a_packed) && !hio && ce_pack_on() && p.L == p.pc && !A->sparse;
    ce_ident_b = ce && (!dens || p.b_packed) && !hio && ce_pack_on() && p.L == p.pr && !B->sparse;
    if (ce_ident_a || ce_ident_b) {
      if (!ctx->own) CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking));
      CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->own, ev_prior, 0));  // the arenas' earlier writers
    }
    bool a_first = false, b_first = false;  // a peer's first step pulls my A / my B panel
    for (int q = 0; q < ctx->nranks && ce; ++q) {
      if (q == ctx->rank) continue;
      const int rq = q / p.pc, cq = q % p.pc;
      const int kq = (rq + cq + (p.local_first ? local_first_start(p.pr, p.pc, q) : 0)) % p.L;
      a_first |= rq * p.pc + kq % p.pc == ctx->rank;
      b_first |= (kq % p.pr) * p.pc + cq == ctx->rank;
    }
    auto own_a = [&]() -> dbm_status {
      for (int k = 0; k < p.L; ++k) {
        if (p.ownA_off[k] == SIZE_MAX) continue;
        const int64_t col0 = (k - p.c) / p.pc, stride = p.L / p.pc;
        double* dst = (double*)(xp + p.ownA_off[k]);
        if (ce_ident_a) {  // the panel IS the arena: a copy-engine copy beside the compute, published there
          CUDA_TRY(ctx, cudaMemcpyAsync(dst, A->arena, p.a_panel_bytes(k), cudaMemcpyDeviceToDevice, ctx->own));
          if (dbm_status e = publish_panel(0, k, ctx->own)) return e;
          continue;
        }
        if (dens && !p.a_packed) {
          ProfScope ps(ctx, cs, 2, 0.0, 16.0 * M * p.kb[k] * bs);
          if (dbm_status e = densify_a(ctx, A, col0, stride, p.kb[k], dst, p.ld_panel(k), 1, cs)) return e;
        } else {  // packed whole blocks (blocked path; densified bs 64: the GEMM reads them in place)
          ProfScope ps(ctx, cs, 2, 0.0, 16.0 * M * p.kb[k] * bs);
          launch_pack_cols(A->arena, p.mloc, p.kA, (int)bs, col0, stride, p.kb[k], dst, cs);
        }
        launches += (M * p.kb[k]) ? 1 : 0;
        if (dbm_status e = publish_panel(0, k, cs)) return e;
      }
      return DBM_OK;
    };
    auto own_b = [&]() -> dbm_status {
      for (int k = 0; k < p.L; ++k) {
        if (p.ownB_off[k] == SIZE_MAX) continue;
        const int64_t row0 = (k - p.r) / p.pr, stride = p.L / p.pr;
        double* dst = (double*)(xp + p.ownB_off[k]);
        if (ce_ident_b) {
          CUDA_TRY(ctx, cudaMemcpyAsync(dst, B->arena, p.b_panel_bytes(k), cudaMemcpyDeviceToDevice, ctx->own));
          if (dbm_status e = publish_panel(1, k, ctx->own)) return e;
          continue;
        }
        if (dens && !p.b_packed) {
          ProfScope ps(ctx, cs, 2, 0.0, 16.0 * N * p.kb[k] * bs);
          if (dbm_status e = densify_b(ctx, B, row0, stride, p.kb[k], dst, p.ld_panel(k), 0, cs)) return e;
        } else {
          ProfScope ps(ctx, cs, 2, 0.0, 16.0 * N * p.kb[k] * bs);  // packing: the same 16 B per element
          launch_pack_rows(B->arena, p.nloc, (int)bs, row0, stride, p.kb[k], dst, cs);
        }
        launches += (N * p.kb[k]) ? 1 : 0;
        if (dbm_status e = publish_panel(1, k, cs)) return e;
      }
      return DBM_OK;
    };
    if (b_first && !a_first && !hio) {  // (host operands: B may still be uploading, A goes first)
      if (dbm_status e = own_b()) return e;
      if (dbm_status e = own_a()) return e;
    } else {
      if (dbm_status e = own_a()) return e;
      if (hio && hio->b_deferred) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, hio->all_ev, 0));
      if (dbm_status e = own_b()) return e;
    }
    CUDA_TRY(ctx, cudaGetLastError());
  }

  // blocked path: traversal table once per multiply
  int32_t* trav_li = nullptr;
  int32_t* trav_lj = nullptr;
  int32_t* trip0 = nullptr;
  if (!dens) {
    trav_li = (int32_t*)(ws + p.off_trav);
    trav_lj = trav_li + std::max<int64_t>(p.mloc * p.nloc, 1);
    trip0 = (int32_t*)(ws + p.off_trip);
    ProfScope ps(ctx, cs, 4, 0.0, 8.0 * p.mloc * p.nloc);
    launch_traversal(p.mloc, p.nloc, trav_li, trav_lj, cs);
    launches += (p.mloc * p.nloc) ? 1 : 0;
    if (p.mixed) {
      launch_inverse_traversal(trav_li, trav_lj, p.mloc * p.nloc, p.nloc, (int32_t*)(ws + p.off_pos), cs);
      ++launches;
    }
  }

  // ------------------------------------------------ Cannon steps
  std::vector<cudaEvent_t> ev_x(p.L, nullptr), ev_g(p.L, nullptr);
  cudaEvent_t ev_ready = nullptr;
  std::vector<int> bufA_of(p.L, -1), bufB_of(p.L, -1);
  std::vector<Plan> peer_plan;
  // Pipelined host operands: this rank's own panels are densified (or packed) chunk by chunk on the
  // upload stream, each chunk right behind its upload, and after every chunk the rank publishes its
  // progress into every peer's flag table.  All of this is enqueued BEFORE any wait on a peer's flag:
  // a rank's signals then never sit behind its own waits (in a stream or in the host's program order),
  // so host calls that synchronise the device (lazy kernel loading, cudaFree, ...) cannot close a
  // cycle across ranks -- the round-1 hang was exactly that: flag waits enqueued, then a first kernel
  // launch loaded its module, synchronised, and waited forever on the peer doing the same.
  std::vector<cudaEvent_t> own_ev;  // own panels' chunk j in place (own-panel stream)
  // own-panel stream: chunk j's densify / pack waits only for upload chunk j (the uploads stream on
  // ctx->up back to back); it never waits on a peer, so its progress signals keep the ordering rule
  cudaStream_t up = pipe ? ctx->own : nullptr;
  auto publish = [&](int j, bool final_) -> dbm_status {
    // every peer's table entry [me][operand][k] = (epoch, K-blocks of my panel k now in place)
    for (int q = 0; q < ctx->nranks; ++q) {
      if (q == ctx->rank) continue;
      for (int k = 0; k < p.L; ++k)
        for (int o = 0; o < 2; ++o) {
          if ((o == 0 ? p.ownA_off[k] : p.ownB_off[k]) == SIZE_MAX) continue;
          const int64_t v = final_ ? p.kb[k] : host_pipe_bound(p.kb[k], j + 1, hp_even);
          if (dbm_status e = xwrite_word(ctx, up, q, xprog_word(ctx->nranks, p.L, ctx->rank, o, k), (ep << 32) | (uint64_t)v))
            return e;
        }
    }
    return DBM_OK;
  };
  auto own_panels_chunk = [&](int j) -> dbm_status {
    if (hpipe) CUDA_TRY(ctx, cudaStreamWaitEvent(up, hio->up_ev[j], 0));  // upload chunk j landed
    for (int k = 0; k < p.L; ++k) {
      const int64_t q0 = host_pipe_bound(p.kb[k], j, hp_even), q1 = host_pipe_bound(p.kb[k], j + 1, hp_even);
      if (q1 <= q0) continue;
      if (p.ownA_off[k] != SIZE_MAX && M) {
        const int64_t col0 = (k - p.c) / p.pc, stride = p.L / p.pc;
        ProfScope ps(ctx, up, 2, 0.0, 16.0 * M * (q1 - q0) * bs);
        if (dens && !p.a_packed) {
          double* dst = (double*)(xp + p.ownA_off[k]) + q0 * bs;
          if (dbm_status e = densify_a(ctx, A, col0 + q0 * stride, stride, q1 - q0, dst, p.ld_panel(k), 1, up))
            return e;
        } else {  // packed A panel: mloc rows of kb[k] blocks; this chunk is columns [q0, q1) of every row
          double* dst = (double*)(xp + p.ownA_off[k]) + q0 * bb;
          launch_pack_cols(A->arena, p.mloc, p.kA, (int)bs, col0 + q0 * stride, stride, q1 - q0, dst, up, p.kb[k]);
        }
        ++launches;
      }
      if (p.ownB_off[k] != SIZE_MAX && N) {
        const int64_t row0 = (k - p.r) / p.pr, stride = p.L / p.pr;
        ProfScope ps(ctx, up, 2, 0.0, 16.0 * N * (q1 - q0) * bs);
        if (dens && !p.b_packed) {
          double* dst = (double*)(xp + p.ownB_off[k]) + q0 * bs;
          if (dbm_status e = densify_b(ctx, B, row0 + q0 * stride, stride, q1 - q0, dst, p.ld_panel(k), 0, up))
            return e;
        } else {
          double* dst = (double*)(xp + p.ownB_off[k]) + q0 * p.nloc * bb;
          launch_pack_rows(B->arena, p.nloc, (int)bs, row0 + q0 * stride, stride, q1 - q0, dst, up);
        }
        ++launches;
      }
    }
    CUDA_TRY(ctx, cudaGetLastError());
    return publish(j, false);
  };
  int nsub0 = 1;               // K-chunks of the step-0 pull (copy-engine transport, densified)
  cudaEvent_t ev_c[kMaxChunks] = {};
  std::vector<int64_t> cb0{0, 0};
  auto recv_bytes = [&](int s) {
    double n = 0;
    for (const XOp& op : exchange_ops(p, s)) n += op.send ? 0 : (double)op.bytes;
    return n;
  };
  auto exchange = [&](int s) -> dbm_status {
    if (ctx->transport == 0) {
      ProfScope ps(ctx, ctx->comm, 5, 0.0, recv_bytes(s));  // copy-engine pulls of this step
      return post_pulls(ctx, p, peer_plan, s, ws, bufA_of[s], bufB_of[s], &st.bytes_sent, &st.bytes_recv, ep);
    }
    return post_exchange(ctx, p, s, ws, A->arena, B->arena, bufA_of[s], bufB_of[s], &st.bytes_sent, &st.bytes_recv);
  };
  if (ctx->nranks > 1) {
    int na = 0, nb = 0;
    for (int s = 0; s < p.L; ++s) {
      bufA_of[s] = (p.a_src(s) != p.me()) ? (na++ & 1) : -1;
      bufB_of[s] = (p.b_src(s) != p.me()) ? (nb++ & 1) : -1;
    }
    if (ev_prior) {
      ev_ready = ev_prior;
    } else {  // (NCCL: the sends read the own panels packed above)
      ev_ready = get_event(ctx);
      CUDA_TRY(ctx, cudaEventRecord(ev_ready, cs));
    }
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm, ev_ready, 0));
    for (int s = 0; s < p.L; ++s) {
      ev_x[s] = get_event(ctx);
      ev_g[s] = get_event(ctx);
    }
    if (ctx->transport == 0) {
      // Copy engines over the IPC-mapped workspaces, ordered by device-side signals (no host sync once
      // the workspace is registered): every signal this rank owes its peers -- each own panel's progress
      // word (on the compute stream behind its densify / pack, or chunk by chunk on the own-panel stream
      // in the pipelined modes) -- is enqueued before the first wait on theirs.
      peer_plan.resize(ctx->nranks);
      for (int q = 0; q < ctx->nranks; ++q)
        if (q != ctx->rank)
          peer_plan[q] = make_plan_raw(ctx->nranks, p.pr, p.pc, q / p.pc, q % p.pc, p.Mb, p.Nb, p.Kb, p.bs, dens,
                                       ctx->chunk_bytes, ctx->transport, p.b_packed, p.a_packed, p.local_first);
      if (pipe) {
        for (int j = 0; j < kHostPipeChunks; ++j) {
          if (dbm_status e = own_panels_chunk(j)) {
            // the peers drain instead of hanging (final progress + my "done"); the ctx is poisoned
            publish(kHostPipeChunks - 1, true);
            xsignal(ctx, up, X_DONE, ep);
            ctx->poisoned = e;
            return e;
          }
          own_ev.push_back(get_event(ctx));
          CUDA_TRY(ctx, cudaEventRecord(own_ev.back(), up));
        }
      }  // (else: every own panel's progress word went out behind its densify / pack above)
    }
  }

  // Everything after the Cannon setup runs in body(): whatever it returns, the closing barrier below is
  // still enqueued, so an error on one rank (poisoning its ctx) does not leave its peers waiting in theirs.
  auto body = [&]() -> dbm_status {
  if (ctx->nranks > 1) {
    // Step 0 is the one exchange nothing overlaps with (Cannon's initial alignment).  With the copy
    // engines and densified panels it is pulled in K-chunks, each followed by its GEMM chunk, so only
    // the first chunk's transfer is exposed.
    bool remote0 = p.a_src(0) != p.me() || p.b_src(0) != p.me();
    const int64_t kb0 = p.kb[p.kappa(0)];
    if (pipe) {  // the fixed pipeline chunks, even when both step-0 panels are local
      cb0.resize(kHostPipeChunks + 1);
      for (int j = 0; j <= kHostPipeChunks; ++j) cb0[j] = host_pipe_bound(kb0, j, hp_even);
      nsub0 = kHostPipeChunks;
    } else if (ctx->transport == 0 && remote0 && (!dens || bs % 2 == 0) && kb0 >= 2) {
      const double pull = ((p.a_src(0) != p.me() ? p.mloc : 0) + (p.b_src(0) != p.me() ? p.nloc : 0)) * (double)bs * bs * 8;
      cb0 = pipeline_chunks(kb0, pipeline_growth(2.0 * M * N * bs * (dens ? 1.0 : 1.25), pull));
      nsub0 = (int)cb0.size() - 1;
    }
    if (nsub0 > 1) {
      ProfScope ps(ctx, ctx->comm, 5, 0.0, recv_bytes(0));
      for (int j = 0; j < nsub0; ++j) {
        ev_c[j] = get_event(ctx);
        if (dbm_status e = post_pulls_chunk(ctx, p, peer_plan, 0, ws, bufA_of[0], bufB_of[0], cb0[j], cb0[j + 1],
                                            j == 0, &st.bytes_sent, &st.bytes_recv, ep))
          return e;
        CUDA_TRY(ctx, cudaEventRecord(ev_c[j], ctx->comm));
      }
    } else if (dbm_status e = exchange(0)) {
      return e;
    }
    CUDA_TRY(ctx, cudaEventRecord(ev_x[0], ctx->comm));
  }

  for (int s = 0; s < p.L; ++s) {
    const int k = p.kappa(s);
    if (ctx->nranks > 1) {
      if (s + 1 < p.L) {  // prefetch step s+1 while step s computes (P:171 overlap)
        if (s >= 1) CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm, ev_g[s - 1], 0));
        if (dbm_status e = exchange(s + 1)) return e;
        CUDA_TRY(ctx, cudaEventRecord(ev_x[s + 1], ctx->comm));
      }
      if (!(s == 0 && nsub0 > 1)) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, ev_x[s], 0));
    }
    const int64_t kbk = p.kb[k];
    if (hpipe && s == 0 && !dens) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, hio->c_ev, 0));  // C_in (uploaded first)
    if (pipe && s == 1) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, own_ev.back(), 0));  // all own panels in place
    // operand panels for this step
    const double* Ap;
    const double* Bp;
    if (ctx->nranks > 1) {
      Ap = p.a_src(s) != p.me() ? (const double*)(ws + p.off_recvA[bufA_of[s]])
                                : (p.ownA_off[k] != SIZE_MAX && !ce_ident_a ? (const double*)(xp + p.ownA_off[k])
                                                                            : A->arena);
      Bp = p.b_src(s) != p.me() ? (const double*)(ws + p.off_recvB[bufB_of[s]])
                                : (p.ownB_off[k] != SIZE_MAX && !ce_ident_b ? (const double*)(xp + p.ownB_off[k])
                                                                            : B->arena);
    } else {
      Ap = A->arena;
      Bp = B->arena;
    }
    if (dens) {
      double* Cd = (double*)(ws + p.off_cd);
      if (ctx->nranks == 1) {
        // K-chunked: densify chunk -> GEMM accumulate
        const bool hchunk = hio && !A->sparse && !B->sparse;
        const std::vector<int64_t> kc = k_chunks(p.Kb, p.chunk_kb, hchunk);
        const int64_t nch = (int64_t)kc.size() - 1;
        // host C: the last chunk's GEMM runs in row panels, each undensified and downloaded while the
        // next panel multiplies, so only the last panel's download is exposed
        const int npan = (hchunk && !C->sparse && p.mloc >= 8) ? 8 : 1;
        for (int64_t ch = 0; ch < nch; ++ch) {
          const int64_t k0 = kc[ch], nk = kc[ch + 1] - kc[ch];
          const int64_t ld = round_up(p.chunk_kb * bs, 2);
          double* Ad = (double*)(ws + p.off_ownA);
          double* Bd = (double*)(ws + p.off_ownB);
          if (hio && hio->chunk_ev.size() > (size_t)ch + 1)  // chunk ch uploaded
            CUDA_TRY(ctx, cudaStreamWaitEvent(cs, hio->chunk_ev[ch + 1], 0));
          if (p.b_packed) Bd = B->arena + k0 * p.nloc * bb;  // B's blocks read in place (§8f-3)
          if (!p.a_packed || !p.b_packed) {
            ProfScope ps(ctx, cs, 2, 0.0, 16.0 * ((p.a_packed ? 0 : M) + (p.b_packed ? 0 : N)) * nk * bs);
            if (!p.a_packed)
              if (dbm_status e = densify_a(ctx, A, k0, 1, nk, Ad, ld, 1, cs)) return e;
            if (!p.b_packed)
              if (dbm_status e = densify_b(ctx, B, k0, 1, nk, Bd, ld, 0, cs)) return e;
            launches += (p.a_packed ? 0 : 1) + (p.b_packed ? 0 : 1);
          }
          const int pans = (ch == nch - 1) ? npan : 1;
          for (int pn = 0; pn < pans; ++pn) {
            const int64_t li0 = p.mloc * pn / pans, li1 = p.mloc * (pn + 1) / pans, m0 = li0 * bs, mr = (li1 - li0) * bs;
            GemmArgs g{mr, N, nk * bs, Ad + m0 * ld, ld, Bd, ld, Cd + m0, M, 1.0, ch == 0 ? 0.0 : 1.0, 1, nullptr};
            if (p.a_packed) {  // A's blocks read in place: block (li, kk) at slot li * kA + kk of the arena (§8f-3)
              g.A = A->arena + (li0 * p.kA + k0) * bb;
              g.a_blocks = 1;
              g.a_blk_ld = p.kA;
            }
            g.b_blocks = p.b_packed ? 1 : 0;
            g.splitk = std::min(pick_splitk(g.M, N, g.K, num_sms()), p.max_split);  // partial buffer bound
            g.partial = g.splitk > 1 ? (double*)(ws + p.off_part) : nullptr;
            {
              ProfScope ps(ctx, cs, 0, 2.0 * mr * N * g.K, 8.0 * (mr * g.K + N * g.K + mr * N * (ch ? 2 : 1)));
              CUDA_TRY(ctx, launch_dgemm(g, cs, &launches));
            }
            ++st.gemm_launches;
            if (pans > 1) {  // undensify this row panel, then download it on the copy stream
              if (pn == 0 && hio->c_ev) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, hio->c_ev, 0));  // C_in uploaded
              {
                ProfScope ps(ctx, cs, 3, 0.0, (beta == 0.0 ? 16.0 : 24.0) * mr * N);
                launch_undensify(Cd + m0, M, 1, 0, li1 - li0, p.nloc, (int)bs, alpha, beta,
                                 C->arena + li0 * p.nloc * bb, cs);
                ++launches;
              }
              cudaEvent_t e = get_event(ctx);
              CUDA_TRY(ctx, cudaEventRecord(e, cs));
              hio->panel_ev.push_back(e);
              CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm, e, 0));
              const size_t off = (size_t)(li0 * p.nloc) * bb * 8, n = (size_t)((li1 - li0) * p.nloc) * bb * 8;
              if (n) CUDA_TRY(ctx, cudaMemcpyAsync((char*)hio->C + off, (const char*)C->arena + off, n,
                                                   cudaMemcpyDeviceToHost, ctx->comm));
              hio->c_downloaded = true;
            }
          }
          ++st.entries;
          ++st.stacks;
          st.flops += 2.0 * M * N * nk * bs;
        }
        if (hio && hio->c_downloaded) {  // the call ends when C is on the host
          cudaEvent_t e = get_event(ctx);
          CUDA_TRY(ctx, cudaEventRecord(e, ctx->comm));
          hio->panel_ev.push_back(e);
          CUDA_TRY(ctx, cudaStreamWaitEvent(cs, e, 0));
        }
      } else {
        const int64_t ld = p.ld_panel(k);
        const int nsub = (s == 0) ? nsub0 : 1;
        for (int j = 0; j < nsub; ++j) {
          const int64_t k0 = nsub > 1 ? cb0[j] : 0, k1 = nsub > 1 ? cb0[j + 1] : kbk;
          if (pipe && s == 0) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, own_ev[j], 0));  // my own panels' chunk j
          if (nsub > 1) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, ev_c[j], 0));
          // host C: the multiply's last GEMM runs in row panels, each undensified and downloaded on the
          // copy stream while the next panel multiplies (as on one rank)
          const int pans = (hio && !C->sparse && s == p.L - 1 && j == nsub - 1 && p.mloc >= 8) ? 8 : 1;
          for (int pn = 0; pn < pans; ++pn) {
            const int64_t li0 = p.mloc * pn / pans, li1 = p.mloc * (pn + 1) / pans, m0 = li0 * bs, mr = (li1 - li0) * bs;
            GemmArgs g{mr, N, (k1 - k0) * bs, Ap + m0 * ld + k0 * bs, ld,
                       p.b_packed ? Bp + k0 * p.nloc * bb : Bp + k0 * bs, ld, Cd + m0, M, 1.0,
                       (s == 0 && j == 0) ? 0.0 : 1.0, 1, nullptr};
            if (p.a_packed) {  // packed A panel read in place: block (li, kk) at slot li * kb + kk (§8f-3)
              g.A = Ap + (li0 * kbk + k0) * bb;
              g.a_blocks = 1;
              g.a_blk_ld = kbk;
            }
            g.b_blocks = p.b_packed ? 1 : 0;
            g.splitk = std::min(pick_splitk(g.M, N, g.K, num_sms()), p.max_split);  // partial buffer bound
            g.partial = g.splitk > 1 ? (double*)(ws + p.off_part) : nullptr;
            {
              ProfScope ps(ctx, cs, 0, 2.0 * mr * N * g.K,
                           8.0 * (mr * g.K + N * g.K + mr * N * ((s == 0 && j == 0) ? 1 : 2)));
              CUDA_TRY(ctx, launch_dgemm(g, cs, &launches));
            }
            ++st.gemm_launches;
            if (pans > 1) {
              if (pn == 0 && hio->c_ev) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, hio->c_ev, 0));  // C_in uploaded
              {
                ProfScope ps(ctx, cs, 3, 0.0, (beta == 0.0 ? 16.0 : 24.0) * mr * N);
                launch_undensify(Cd + m0, M, 1, 0, li1 - li0, p.nloc, (int)bs, alpha, beta,
                                 C->arena + li0 * p.nloc * bb, cs);
                ++launches;
              }
              cudaEvent_t e = get_event(ctx);
              CUDA_TRY(ctx, cudaEventRecord(e, cs));
              hio->panel_ev.push_back(e);
              CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm, e, 0));
              const size_t off = (size_t)(li0 * p.nloc) * bb * 8, n = (size_t)((li1 - li0) * p.nloc) * bb * 8;
              if (n) CUDA_TRY(ctx, cudaMemcpyAsync((char*)hio->C + off, (const char*)C->arena + off, n,
                                                   cudaMemcpyDeviceToHost, ctx->comm));
              hio->c_downloaded = true;
            }
          }
        }
        if (hio && hio->c_downloaded && s == p.L - 1) {  // the call ends when C is on the host
          cudaEvent_t e = get_event(ctx);
          CUDA_TRY(ctx, cudaEventRecord(e, ctx->comm));
          hio->panel_ev.push_back(e);
          CUDA_TRY(ctx, cudaStreamWaitEvent(cs, e, 0));
        }
        st.entries += (M && N) ? 1 : 0;  // densified batches hold one multiplication
        st.stacks += (M && N) ? 1 : 0;
        st.flops += 2.0 * M * N * kbk * bs;
      }
    } else if (kbk > 0 && p.mloc * p.nloc > 0) {
      // blocked: Generation (stack chunks) -> batched small-block GEMM
      const int64_t nruns = p.mloc * p.nloc;
      // a dense local grid the bisection visits as whole 4 x 4 squares runs the unpadded bs-22 kernel;
      // chunks of runs then hold whole squares
      // ... and the small padded sizes take R x R run squares (smmq) when the bisection visits them and
      // there are enough squares to fill the GPU
      const int qR = smmq_on() ? smmq_side((int)bs) : 0;
      const bool squares = bs == 22 ? bisection_squares(p.mloc, p.nloc)
                                    : (qR > 0 && bisection_squares(p.mloc, p.nloc, qR) &&
                                       (smmq_on() == 2 || nruns / ((int64_t)qR * qR) >= num_sms()));
      const int64_t grp = squares ? (bs == 22 ? 16 : (int64_t)qR * qR) : smm_group_runs((int)bs);
      const int64_t runs_per_chunk = std::max<int64_t>(grp, p.trip_cap / kbk / grp * grp);
      const int64_t a_ld = kbk;  // A panel is mloc x kb blocks, row-major over (li, kk)
      // step 0 with a chunked pull: each K-chunk [k0, k1) of the panels multiplies as soon as it landed
      // (the runs' K split across chunks, accumulated in chunk order: C = beta*C + alpha*acc_0, then
      // C += alpha*acc_j); the stack list itself (dbm_debug_stacks) is the unchunked one
      const int nsub = (s == 0) ? nsub0 : 1;
      for (int j = 0; j < nsub; ++j) {
        const int64_t k0 = nsub > 1 ? cb0[j] : 0, nk = nsub > 1 ? cb0[j + 1] - cb0[j] : kbk;
        if (pipe && s == 0) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, own_ev[j], 0));  // my own panels' chunk j
        if (nsub > 1) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, ev_c[j], 0));
        if (nk == 0) continue;  // (host pipeline, ragged K: empty leading chunks)
        const double* Aj = Ap + k0 * bb;
        const double* Bj = Bp + k0 * p.nloc * bb;
        const double bfirst = (s == 0 && k0 == 0) ? beta : 1.0;  // the first non-empty chunk applies beta
        // two triplet buffers (several chunks): chunk c's stacks are generated on the generation stream
        // into buffer c % 2 once the multiply of chunk c - 2 released it, overlapping chunk c - 1's
        // multiply (the generation kernel's CTAs fit beside the persistent small-block kernel's)
        const bool dbuf = p.off_trip2 != 0 && nruns > runs_per_chunk && stackgen_dbuf();
        cudaEvent_t ev_free[2] = {nullptr, nullptr};
        if (dbuf) {
          if (!ctx->gen) CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->gen, cudaStreamNonBlocking));
          cudaEvent_t e = get_event(ctx);
          CUDA_TRY(ctx, cudaEventRecord(e, cs));  // the traversal table and everything before
          CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->gen, e, 0));
          ctx->ev_pool.push_back(e);
        }
        for (int64_t q0 = 0, chunk = 0; q0 < nruns; q0 += runs_per_chunk, ++chunk) {
          const int64_t q1 = std::min(nruns, q0 + runs_per_chunk);
          int32_t* trip = (dbuf && (chunk & 1)) ? (int32_t*)(ws + p.off_trip2) : trip0;
          if (dbuf) {
            if (ev_free[chunk & 1]) CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->gen, ev_free[chunk & 1], 0));
            {
              ProfScope ps(ctx, ctx->gen, 4, 0.0, 12.0 * (q1 - q0) * nk);
              launch_stackgen(trav_li, trav_lj, q0, q1, nk, p.nloc, a_ld, p.nloc, trip, ctx->gen);
              ++launches;
            }
            cudaEvent_t e = get_event(ctx);
            CUDA_TRY(ctx, cudaEventRecord(e, ctx->gen));
            CUDA_TRY(ctx, cudaStreamWaitEvent(cs, e, 0));
            ctx->ev_pool.push_back(e);
          } else {
            ProfScope ps(ctx, cs, 4, 0.0, 12.0 * (q1 - q0) * nk);
            launch_stackgen(trav_li, trav_lj, q0, q1, nk, p.nloc, a_ld, p.nloc, trip, cs);
            ++launches;
          }
          {
            ProfScope ps(ctx, cs, 1, 2.0 * bs * bb * (q1 - q0) * nk, 16.0 * bb * (q1 - q0) * nk);
            const int nsplit = p.spart_runs ? (int)std::min<int64_t>(smm_pick_split((int)bs, q1 - q0, nk, squares),
                                                                     p.spart_runs / (q1 - q0))
                                            : 1;
            if (p.mixed && nsplit <= 1) {
              const SmmMixedWS mw{(uint8_t*)(ws + p.off_sqflag), (int32_t*)(ws + p.off_sqids),
                                  (int32_t*)(ws + p.off_runsq),   (int32_t*)(ws + p.off_runleft),
                                  (uint8_t*)(ws + p.off_runflag), (int*)(ws + p.off_counts),
                                  ws + p.off_mtemp,                p.mtemp_bytes};
              CUDA_TRY(ctx, launch_smm22_mixed(trip, q0, q1 - q0, nk, Aj, Bj, C->arena, alpha, bfirst, trav_li, trav_lj,
                                               (const int32_t*)(ws + p.off_pos), p.mloc, p.nloc, mw, cs, &launches));
            } else {
              CUDA_TRY(ctx, launch_smm((int)bs, trip, q1 - q0, nk, Aj, Bj, C->arena, alpha, bfirst, nsplit,
                                       nsplit > 1 ? (double*)(ws + p.off_spart) : nullptr, cs, &launches,
                                       p.mloc * kbk - k0, (kbk - k0) * p.nloc, squares));
            }
          }
          if (dbuf) {  // buffer chunk % 2 is free once this multiply is done with it
            if (!ev_free[chunk & 1]) ev_free[chunk & 1] = get_event(ctx);
            CUDA_TRY(ctx, cudaEventRecord(ev_free[chunk & 1], cs));
          }
        }
        for (cudaEvent_t e : ev_free)
          if (e) ctx->ev_pool.push_back(e);
      }
      st.entries += nruns * kbk;
      st.stacks += kbk <= cap ? (nruns + (cap / kbk) - 1) / (cap / kbk) : nruns * ((kbk + cap - 1) / cap);
      st.flops += 2.0 * bs * bb * nruns * kbk;
    } else if (s == 0 && p.mloc * p.nloc > 0) {
      // empty K panel at step 0 still applies beta exactly once
      launch_scale(C->arena, M * N, beta, cs);
      ++launches;
    }
    CUDA_TRY(ctx, cudaGetLastError());
    if (ctx->nranks > 1) CUDA_TRY(ctx, cudaEventRecord(ev_g[s], cs));
  }

  if (ctx->nranks > 1) {
    // the comm stream's last op covers every transfer of this rank (and the upload stream's own panels)
    CUDA_TRY(ctx, cudaStreamWaitEvent(cs, ev_x[p.L - 1], 0));
    if (pipe) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, own_ev.back(), 0));
    if (ce_ident_a || ce_ident_b) {  // the copy-engine panel copies read the arenas
      cudaEvent_t e = get_event(ctx);
      CUDA_TRY(ctx, cudaEventRecord(e, ctx->own));
      CUDA_TRY(ctx, cudaStreamWaitEvent(cs, e, 0));
      ctx->ev_pool.push_back(e);
    }
  }
  if (dens && M * N > 0 && !(hio && hio->c_downloaded)) {
    if (hio && hio->c_ev) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, hio->c_ev, 0));  // C_in uploaded
    ProfScope ps(ctx, cs, 3, 0.0, (beta == 0.0 ? 16.0 : 24.0) * M * N);
    undensify_c(C, (double*)(ws + p.off_cd), M, 1, 0, alpha, beta, cs);
    ++launches;
    CUDA_TRY(ctx, cudaGetLastError());
  }
  return DBM_OK;
  };
  const dbm_status berr = body();
  if (ctx->nranks > 1 && ctx->transport == 0) {
    // Closing barrier: "done" goes out on the comm stream behind my last pull, and the compute stream
    // (after my last GEMM) waits for every peer's "done": when it passes, no peer still pulls from this
    // workspace, so stream-ordered reuse of it is safe.  Device-side signals: no kernel spins on an SM
    // next to the persistent GEMM, no host round trip.
    if (dbm_status e = xsignal(ctx, ctx->comm, X_DONE, ep)) return e;
    if (dbm_status e = xwait(ctx, cs, X_DONE, ep)) return e;
  }
  if (berr != DBM_OK) {
    if (ctx->poisoned == DBM_OK) ctx->poisoned = berr;
    return berr;
  }
  if (ctx->nranks > 1) {
    // events are reusable once the compute stream has passed them; recycle after this call
    cudaEvent_t done = get_event(ctx);
    CUDA_TRY(ctx, cudaEventRecord(done, cs));
    ctx->ev_pool.push_back(ev_ready);
    for (int s = 0; s < p.L; ++s) {
      ctx->ev_pool.push_back(ev_x[s]);
      ctx->ev_pool.push_back(ev_g[s]);
    }
    for (int j = 0; j < nsub0 && nsub0 > 1; ++j) ctx->ev_pool.push_back(ev_c[j]);
    for (cudaEvent_t e : own_ev) ctx->ev_pool.push_back(e);
    if (dpipe_e0) ctx->ev_pool.push_back(dpipe_e0);
    ctx->ev_pool.push_back(done);
  }
  ctx->launches += launches;
  st.kernel_launches = launches;
  if (stats) *stats = st;
  return DBM_OK;
}

}  // namespace

// ====================================================================== debug entry points
extern "C" dbm_status dbm_debug_stacks(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, int step, int32_t cap,
                                       int32_t* triplets, int64_t* n_entries, int64_t* stack_ptr,
                                       int64_t* n_stacks) {
  CTX_OK(ctx);
  if (dbm_status s = validate(ctx, A, B, C)) return s;
  ARG_CHECK(n_entries && n_stacks, DBM_ERR_ARG, "null size outputs");
  if (A->sparse || B->sparse || C->sparse)
    return sp_debug_stacks(ctx, A, B, C, step, cap, triplets, n_entries, stack_ptr, n_stacks);
  // (non-uniform blocks, R16: the same slot triplets -- the list depends on the block structure only)
  const Plan p = A->nonuni || B->nonuni || C->nonuni
                     ? make_plan_raw(ctx->nranks, ctx->pr, ctx->pc, ctx->myrow, ctx->mycol, A->Mb, B->Nb, A->Nb, 1,
                                     false, ctx->chunk_bytes, ctx->transport)
                     : make_plan(ctx, A, B, C, false, false);  // (the canonical step numbering)
  ARG_CHECK(step >= 0 && step < p.L, DBM_ERR_RANGE, "step out of range");
  const int64_t capv = cap ? cap : 30000;
  const int64_t kb = p.kb[p.kappa(step)], nruns = p.mloc * p.nloc, ne = nruns * kb;
  const int64_t ns = kb == 0 ? 0 : (kb <= capv ? (nruns + capv / kb - 1) / (capv / kb) : nruns * ((kb + capv - 1) / capv));
  *n_entries = ne;
  *n_stacks = ns;
  if (!triplets && !stack_ptr) return DBM_OK;
  int32_t *d_li = nullptr, *d_trip = nullptr;
  int64_t* d_ptr = nullptr;
  CUDA_TRY(ctx, cudaMalloc(&d_li, (size_t)std::max<int64_t>(2 * nruns, 2) * 4));
  CUDA_TRY(ctx, cudaMalloc(&d_trip, (size_t)std::max<int64_t>(3 * ne, 3) * 4));
  CUDA_TRY(ctx, cudaMalloc(&d_ptr, (size_t)(ns + 1) * 8));
  launch_traversal(p.mloc, p.nloc, d_li, d_li + nruns, ctx->stream);
  launch_stackgen(d_li, d_li + nruns, 0, nruns, kb, p.nloc, kb, p.nloc, d_trip, ctx->stream);
  launch_stack_ptr(nruns, std::max<int64_t>(kb, 1), capv, ns, d_ptr, ctx->stream);
  ctx->launches += 3;
  CUDA_TRY(ctx, cudaGetLastError());
  if (triplets && ne) CUDA_TRY(ctx, cudaMemcpyAsync(triplets, d_trip, ne * 12, cudaMemcpyDeviceToHost, ctx->stream));
  if (stack_ptr) CUDA_TRY(ctx, cudaMemcpyAsync(stack_ptr, d_ptr, (ns + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  cudaFree(d_li);
  cudaFree(d_trip);
  cudaFree(d_ptr);
  return DBM_OK;
}

extern "C" dbm_status dbm_debug_pack_panel(dbm_matrix m, int operand, int64_t first, int64_t stride, int64_t nk,
                                           int64_t pitch, double* out) {
  ARG_CHECK(m, DBM_ERR_ARG, "null matrix");
  dbm_ctx ctx = m->ctx;
  CTX_OK(ctx);
  ARG_CHECK(operand == 0 || operand == 1, DBM_ERR_ARG, "operand must be 0 (A columns) or 1 (B rows)");
  ARG_CHECK(!m->sparse, DBM_ERR_ARG, "pack_panel takes a dense-pattern matrix");
  ARG_CHECK(nk >= 0 && stride >= 1 && first >= 0 && pitch >= 0, DBM_ERR_ARG, "negative sizes");
  if (dbm_status s = need_arena(m)) return s;
  const int64_t lim = operand == 0 ? m->nloc : m->mloc;
  ARG_CHECK(nk == 0 || first + (nk - 1) * stride < lim, DBM_ERR_RANGE, "panel index outside the local blocks");
  ARG_CHECK(operand == 1 || pitch == 0 || pitch >= nk, DBM_ERR_RANGE, "pitch < nk");
  const int64_t other = operand == 0 ? m->mloc : m->nloc;
  ARG_CHECK(nk * other == 0 || out, DBM_ERR_ARG, "null output");
  if (operand == 0)
    launch_pack_cols(m->arena, m->mloc, m->nloc, m->bs, first, stride, nk, out, ctx->stream, pitch);
  else
    launch_pack_rows(m->arena, m->nloc, m->bs, first, stride, nk, out, ctx->stream);
  ctx->launches += (nk * other) ? 1 : 0;
  CUDA_TRY(ctx, cudaGetLastError());
  return DBM_OK;
}

extern "C" dbm_status dbm_debug_dgemm(dbm_ctx ctx, int64_t M, int64_t N, int64_t K, double alpha, const double* At,
                                      int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                                      int splitk, double* partial, int64_t partial_bytes) {
  CTX_OK(ctx);
  ARG_CHECK(M >= 0 && N >= 0 && K >= 0, DBM_ERR_ARG, "negative dimension");
  ARG_CHECK(lda >= K && ldb >= K && ldc >= M && lda % 2 == 0 && ldb % 2 == 0, DBM_ERR_ARG,
            "bad leading dimensions (lda, ldb >= K and even; ldc >= M)");
  ARG_CHECK(M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31), DBM_ERR_SHAPE, "dimension too large");
  if (splitk == 0) splitk = pick_splitk(M, N, K, num_sms());
  ARG_CHECK(splitk >= 1, DBM_ERR_ARG, "bad splitk");
  if (splitk > 1)
    ARG_CHECK(partial && partial_bytes >= (int64_t)splitk * M * N * 8, DBM_ERR_WORKSPACE, "partial buffer too small");
  GemmArgs g{M, N, K, At, lda, B, ldb, C, ldc, alpha, beta, splitk, partial};
  int launches = 0;
  {
    ProfScope ps(ctx, ctx->stream, 0, 2.0 * M * N * K, 8.0 * (M * K + N * K + M * N * (beta != 0 ? 2 : 1)));
    CUDA_TRY(ctx, launch_dgemm(g, ctx->stream, &launches));
  }
  ctx->launches += launches;
  return DBM_OK;
}

// Block-sparse matrices in the multiply (§8f-2, reading R15): the host plan cache, the sparse Cannon
// driver of the blocked path, DBM_PATH_AUTO and the sparse stack-list debug entry.  Part of libdbm's
// host runtime; the kernels are in kernels_sparse.cu.
#include "api_internal.h"

// ====================================================================== block-sparse blocked path (R15)
// Cannon over sparse panels (§8f-2).  Every rank knows every operand's global pattern, so each rank
// plans on the host, once per (A, B, C) pattern triple (cached in the context): the CSR / CSC lists
// of each step's A(r, kappa) and B(kappa, c) panels (kk ascending, slot = rank among the panel's stored
// blocks in row-major order = the order the owner packs them), the gather lists of the panels it owns,
// and its peers' workspace offsets.  Per multiply the GPU packs the owned panels (stored blocks only),
// the copy engines pull the remote ones (only stored blocks move), and per step the Generation
// kernels + smm_sparse run over the traversal in chunks of runs.
namespace dbm {
struct SpStep {
  int kappa = 0, a_src = 0, b_src = 0;
  int64_t a_nnz = 0, b_nnz = 0, entries = 0;
  size_t o_aptr = 0, o_akk = 0, o_bptr = 0, o_bkk = 0, o_bslot = 0;  // int32 offsets into d_meta
  std::vector<int32_t> run_len;                                      // per traversal position
  std::vector<int64_t> chunk_entries;                                // per chunk of runs_per_chunk runs
};
struct SpCache {
  uint64_t a_serial = 0, b_serial = 0, c_serial = 0;
  int L = 1;
  std::vector<SpStep> steps;
  std::vector<int64_t> ownA_nnz, ownB_nnz;  // per kappa (-1: not mine)
  std::vector<size_t> ownA_off, ownB_off, o_gatherA, o_gatherB;
  std::vector<std::vector<size_t>> peer_ownA_off, peer_ownB_off;
  size_t pool_need = 0;  // exchange-pool bytes: the maximum over all ranks of their own_layout end
  std::vector<std::vector<int64_t>> peer_ownA_nnz, peer_ownB_nnz;
  size_t off_recvA[2] = {0, 0}, off_recvB[2] = {0, 0}, off_trav = 0, off_cnt = 0, off_off = 0, off_scan = 0;
  size_t off_trip = 0, scan_bytes = 0, total = 256;
  int64_t runs_per_chunk = 1;
  int32_t* d_meta = nullptr;
  std::vector<std::pair<int64_t, int64_t>> stacks_by_cap;  // (cap, stacks of the whole multiply)
};

void free_sp_cache(dbm_ctx ctx) {
  for (SpCache* c : ctx->sp_cache) {
    if (c->d_meta) cudaFree(c->d_meta);
    delete c;
  }
  ctx->sp_cache.clear();
}

namespace {


int64_t local_slot(dbm_matrix m, int64_t li, int64_t lj) {
  if (!m->sparse) return li * m->nloc + lj;
  const auto b = m->col.begin() + m->row_ptr[li], e = m->col.begin() + m->row_ptr[li + 1];
  const auto it = std::lower_bound(b, e, (int32_t)lj);
  return (it != e && *it == (int32_t)lj) ? (int64_t)(it - m->col.begin()) : -1;
}

void host_traversal(int64_t r0, int64_t r1, int64_t c0, int64_t c1, std::vector<int32_t>& li, std::vector<int32_t>& lj) {
  if (r1 <= r0 || c1 <= c0) return;
  if (r1 - r0 == 1 && c1 - c0 == 1) {
    li.push_back((int32_t)r0);
    lj.push_back((int32_t)c0);
    return;
  }
  if (r1 - r0 >= c1 - c0) {
    const int64_t mid = r0 + (r1 - r0) / 2;
    host_traversal(r0, mid, c0, c1, li, lj);
    host_traversal(mid, r1, c0, c1, li, lj);
  } else {
    const int64_t mid = c0 + (c1 - c0) / 2;
    host_traversal(r0, r1, c0, mid, li, lj);
    host_traversal(r0, r1, mid, c1, li, lj);
  }
}

// Stored blocks of the A(rr, kappa) / B(kappa, cc) panels, as owned by rank (rr, kappa mod Pc) /
// (kappa mod Pr, cc).
int64_t a_panel_nnz(dbm_ctx ctx, dbm_matrix A, int L, int rr, int kappa) {
  int64_t n = 0;
  for (int64_t i = rr; i < A->Mb; i += ctx->pr)
    for (int64_t k = kappa; k < A->Nb; k += L) n += A->stored(i, k);
  return n;
}
int64_t b_panel_nnz(dbm_ctx ctx, dbm_matrix B, int L, int cc, int kappa) {
  int64_t n = 0;
  for (int64_t k = kappa; k < B->Mb; k += L)
    for (int64_t j = cc; j < B->Nb; j += ctx->pc) n += B->stored(k, j);
  return n;
}

// Exchange-pool layout (several ranks): the signal header, then the own (packed) panels, so a peer only
// needs the panel sizes to find them.  *end = the pool bytes this rank needs.
void own_layout(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, int L, int r, int c, std::vector<int64_t>& a_nnz,
                std::vector<int64_t>& b_nnz, std::vector<size_t>& a_off, std::vector<size_t>& b_off, size_t* end) {
  const size_t bb8 = (size_t)A->bs * A->bs * 8;
  a_nnz.assign(L, -1);
  b_nnz.assign(L, -1);
  a_off.assign(L, SIZE_MAX);
  b_off.assign(L, SIZE_MAX);
  size_t off = xhdr_bytes(ctx->nranks, L);  // exchange-pool offsets: the signal header comes first
  if (ctx->nranks > 1) {
    for (int k = 0; k < L; ++k)
      if (k % ctx->pc == c) {
        a_nnz[k] = a_panel_nnz(ctx, A, L, r, k);
        a_off[k] = off;
        off = align256(off + (size_t)a_nnz[k] * bb8);
      }
    for (int k = 0; k < L; ++k)
      if (k % ctx->pr == r) {
        b_nnz[k] = b_panel_nnz(ctx, B, L, c, k);
        b_off[k] = off;
        off = align256(off + (size_t)b_nnz[k] * bb8);
      }
  }
  *end = off;
}

dbm_status sp_cache_get(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, SpCache** out) {
  for (SpCache* c : ctx->sp_cache)
    if (c->a_serial == A->serial && c->b_serial == B->serial && c->c_serial == C->serial) {
      *out = c;
      return DBM_OK;
    }
  SpCache* sc = new SpCache();
  sc->a_serial = A->serial;
  sc->b_serial = B->serial;
  sc->c_serial = C->serial;
  const int pr = ctx->pr, pc = ctx->pc, r = ctx->myrow, c = ctx->mycol, me = ctx->rank;
  const int L = (int)lcm64(pr, pc);
  sc->L = L;
  const int64_t mloc = C->mloc, nloc = C->nloc, Kb = A->Nb;
  const size_t bb8 = (size_t)A->bs * A->bs * 8;
  size_t off = 0;  // caller-owned workspace offsets (the own panels are in the exchange pool)
  own_layout(ctx, A, B, L, r, c, sc->ownA_nnz, sc->ownB_nnz, sc->ownA_off, sc->ownB_off, &sc->pool_need);
  sc->peer_ownA_off.resize(ctx->nranks);
  sc->peer_ownB_off.resize(ctx->nranks);
  sc->peer_ownA_nnz.resize(ctx->nranks);
  sc->peer_ownB_nnz.resize(ctx->nranks);
  for (int q = 0; q < ctx->nranks && ctx->nranks > 1; ++q) {
    size_t e;
    if (q != me) {
      own_layout(ctx, A, B, L, q / pc, q % pc, sc->peer_ownA_nnz[q], sc->peer_ownB_nnz[q], sc->peer_ownA_off[q],
                 sc->peer_ownB_off[q], &e);
      sc->pool_need = std::max(sc->pool_need, e);  // the pool size every rank agrees on
    }
  }
  // per-step panel metadata and entry counts
  std::vector<int32_t> meta;
  std::vector<int32_t> tli, tlj;
  host_traversal(0, mloc, 0, nloc, tli, tlj);
  const int64_t words = 0;
  (void)words;
  int64_t kbmax = 1, amax = 0, bmax = 0;
  int na = 0, nb = 0;
  sc->steps.resize(L);
  for (int s = 0; s < L; ++s) {
    SpStep& st = sc->steps[s];
    st.kappa = (r + c + s) % L;
    st.a_src = r * pc + st.kappa % pc;
    st.b_src = (st.kappa % pr) * pc + c;
    const int64_t kb = local_count(Kb, L, st.kappa);
    kbmax = std::max(kbmax, kb);
    // A panel CSR over li
    std::vector<std::vector<uint64_t>> abits(mloc, std::vector<uint64_t>((kb + 63) / 64, 0));
    st.o_aptr = meta.size();
    meta.resize(meta.size() + mloc + 1);
    std::vector<int32_t> akk;
    for (int64_t li = 0; li < mloc; ++li) {
      meta[st.o_aptr + li] = (int32_t)akk.size();
      for (int64_t kk = 0; kk < kb; ++kk)
        if (A->stored(r + li * pr, st.kappa + kk * L)) {
          akk.push_back((int32_t)kk);
          abits[li][kk >> 6] |= 1ull << (kk & 63);
        }
    }
    meta[st.o_aptr + mloc] = (int32_t)akk.size();
    st.a_nnz = (int64_t)akk.size();
    st.o_akk = meta.size();
    meta.insert(meta.end(), akk.begin(), akk.end());
    // B panel: row-major slots over (kk, lj), CSC lists per lj
    std::vector<std::vector<uint64_t>> bbits(nloc, std::vector<uint64_t>((kb + 63) / 64, 0));
    std::vector<std::vector<std::pair<int32_t, int32_t>>> bcol(nloc);
    int32_t slot = 0;
    for (int64_t kk = 0; kk < kb; ++kk)
      for (int64_t lj = 0; lj < nloc; ++lj)
        if (B->stored(st.kappa + kk * L, c + lj * pc)) {
          bcol[lj].push_back({(int32_t)kk, slot++});
          bbits[lj][kk >> 6] |= 1ull << (kk & 63);
        }
    st.b_nnz = slot;
    st.o_bptr = meta.size();
    meta.resize(meta.size() + nloc + 1);
    std::vector<int32_t> bkk, bsl;
    for (int64_t lj = 0; lj < nloc; ++lj) {
      meta[st.o_bptr + lj] = (int32_t)bkk.size();
      for (auto& pr_ : bcol[lj]) {
        bkk.push_back(pr_.first);
        bsl.push_back(pr_.second);
      }
    }
    meta[st.o_bptr + nloc] = (int32_t)bkk.size();
    st.o_bkk = meta.size();
    meta.insert(meta.end(), bkk.begin(), bkk.end());
    st.o_bslot = meta.size();
    meta.insert(meta.end(), bsl.begin(), bsl.end());
    // run lengths in traversal order (stored C blocks only)
    st.run_len.resize(tli.size());
    for (size_t q = 0; q < tli.size(); ++q) {
      const int64_t li = tli[q], lj = tlj[q];
      int64_t n = 0;
      if (C->stored(r + li * pr, c + lj * pc))
        for (size_t w = 0; w < abits[li].size(); ++w) n += __builtin_popcountll(abits[li][w] & bbits[lj][w]);
      st.run_len[q] = (int32_t)n;
      st.entries += n;
    }
    if (st.a_src != me) {
      amax = std::max(amax, st.a_nnz);
      ++na;
    }
    if (st.b_src != me) {
      bmax = std::max(bmax, st.b_nnz);
      ++nb;
    }
  }
  // gather lists of my own panels (multi-rank: packed into the workspace for the peers and myself)
  sc->o_gatherA.assign(L, SIZE_MAX);
  sc->o_gatherB.assign(L, SIZE_MAX);
  for (int k = 0; k < L && ctx->nranks > 1; ++k) {
    if (sc->ownA_nnz[k] >= 0) {
      sc->o_gatherA[k] = meta.size();
      for (int64_t li = 0; li < A->mloc; ++li)
        for (int64_t kg = k; kg < Kb; kg += L)
          if (A->stored(r + li * pr, kg)) meta.push_back((int32_t)local_slot(A, li, (kg - c) / pc));
    }
    if (sc->ownB_nnz[k] >= 0) {
      sc->o_gatherB[k] = meta.size();
      for (int64_t kg = k; kg < Kb; kg += L)
        for (int64_t lj = 0; lj < B->nloc; ++lj)
          if (B->stored(kg, c + lj * pc)) meta.push_back((int32_t)local_slot(B, (kg - r) / pr, lj));
    }
  }
  // the rest of the workspace
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + bytes);
    return o;
  };
  for (int i = 0; i < std::min(na, 2); ++i) sc->off_recvA[i] = take((size_t)amax * bb8);
  for (int i = 0; i < std::min(nb, 2); ++i) sc->off_recvB[i] = take((size_t)bmax * bb8);
  const int64_t nruns = std::max<int64_t>(mloc * nloc, 1);
  sc->off_trav = take((size_t)nruns * 8);
  sc->runs_per_chunk = std::max<int64_t>(1, std::min<int64_t>(nruns, kTripChunkEntries / kbmax));
  sc->off_cnt = take((size_t)(sc->runs_per_chunk + 1) * 8);
  sc->off_off = take((size_t)(sc->runs_per_chunk + 1) * 8);
  sc->scan_bytes = sp_scan_temp_bytes(sc->runs_per_chunk + 1);
  sc->off_scan = take(sc->scan_bytes);
  sc->off_trip = take((size_t)sc->runs_per_chunk * kbmax * 12);
  sc->total = std::max<size_t>(off, 256);
  for (SpStep& x : sc->steps) {
    for (size_t q0 = 0; q0 < x.run_len.size(); q0 += (size_t)sc->runs_per_chunk) {
      int64_t n = 0;
      for (size_t q = q0; q < std::min(x.run_len.size(), q0 + (size_t)sc->runs_per_chunk); ++q) n += x.run_len[q];
      x.chunk_entries.push_back(n);
    }
  }
  cudaError_t e = cudaMalloc(&sc->d_meta, std::max<size_t>(meta.size(), 1) * 4);
  if (e == cudaSuccess && !meta.empty())
    e = cudaMemcpy(sc->d_meta, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (sc->d_meta) cudaFree(sc->d_meta);
    delete sc;
    set_error(std::string("sparse plan metadata: ") + cudaGetErrorString(e));
    return DBM_ERR_NOMEM;
  }
  ctx->sp_cache.push_back(sc);
  *out = sc;
  return DBM_OK;
}

int64_t sp_stacks(SpCache* sc, int64_t cap) {
  for (auto& pcs : sc->stacks_by_cap)
    if (pcs.first == cap) return pcs.second;
  int64_t ns = 0;
  for (const SpStep& st : sc->steps) {  // greedy whole-run packing, runs > cap split (reading R6)
    int64_t cur = 0;
    for (int32_t n : st.run_len) {
      if (n == 0) continue;
      if (n > cap) {
        if (cur) ++ns;
        cur = 0;
        ns += (n + cap - 1) / cap;
      } else {
        if (cur + n > cap) {
          ++ns;
          cur = 0;
        }
        cur += n;
      }
    }
    if (cur) ++ns;
  }
  sc->stacks_by_cap.push_back({cap, ns});
  return ns;
}

}  // namespace

dbm_status multiply_sparse_blocked(dbm_ctx ctx, double alpha, dbm_matrix A, dbm_matrix B, double beta, dbm_matrix C,
                                   int32_t stack_cap, void* workspace, int64_t ws_bytes, dbm_stats* stats) {
  ARG_CHECK(ctx->nranks == 1 || ctx->transport == 0, DBM_ERR_ARG,
            "the block-sparse blocked path uses the copy-engine transport");
  SpCache* sc = nullptr;
  if (dbm_status e = sp_cache_get(ctx, A, B, C, &sc)) return e;
  ARG_CHECK(workspace != nullptr && ws_bytes >= (int64_t)sc->total, DBM_ERR_WORKSPACE,
            "workspace smaller than dbm_multiply_workspace()");
  const int64_t cap = stack_cap ? stack_cap : 30000;
  cudaStream_t cs = ctx->stream;
  char* ws = (char*)workspace;
  const int bs = A->bs;
  const int64_t bb = (int64_t)bs * bs, mloc = C->mloc, nloc = C->nloc, L = sc->L;
  const int me = ctx->rank;
  dbm_stats st{};
  st.steps = L;
  int launches = 0;
  auto scale_c = [&](double f) -> dbm_status {
    const int64_t n = C->blocks() * bb;
    if (n && f != 1.0) {
      launch_scale(C->arena, n, f, cs);
      ++launches;
      CUDA_TRY(ctx, cudaGetLastError());
    }
    return DBM_OK;
  };
  // beta scales every stored C block once (R15); the steps then accumulate alpha * A * B
  if (dbm_status e = scale_c(beta)) return e;
  if (alpha == 0.0 || A->Nb == 0) {
    ctx->launches += launches;
    st.kernel_launches = launches;
    if (stats) *stats = st;
    return DBM_OK;
  }
  const int32_t* meta = sc->d_meta;
  char* xp = nullptr;  // exchange pool (several ranks): signal header + my packed panels
  uint64_t ep = 0;     // this multiply's epoch (signals between ranks)
  if (ctx->nranks > 1) {
    if (dbm_status e = xattach(ctx, sc->pool_need, cs)) return e;
    xp = ctx->xpool;
    ep = ++ctx->epoch;
  }
  if (ctx->nranks > 1) {  // pack my panels (stored blocks only)
    for (int k = 0; k < L; ++k) {
      if (sc->ownA_nnz[k] > 0) {
        launch_sp_gather(A->arena, meta + sc->o_gatherA[k], sc->ownA_nnz[k], bs, (double*)(xp + sc->ownA_off[k]), cs);
        ++launches;
      }
      if (sc->ownB_nnz[k] > 0) {
        launch_sp_gather(B->arena, meta + sc->o_gatherB[k], sc->ownB_nnz[k], bs, (double*)(xp + sc->ownB_off[k]), cs);
        ++launches;
      }
    }
    CUDA_TRY(ctx, cudaGetLastError());
  }
  int32_t* trav_li = (int32_t*)(ws + sc->off_trav);
  int32_t* trav_lj = trav_li + std::max<int64_t>(mloc * nloc, 1);
  {
    ProfScope ps(ctx, cs, 4, 0.0, 8.0 * mloc * nloc);
    launch_traversal(mloc, nloc, trav_li, trav_lj, cs);
    launches += (mloc * nloc) ? 1 : 0;
  }
  std::vector<cudaEvent_t> ev_x(L, nullptr), ev_g(L, nullptr);
  cudaEvent_t ev_ready = nullptr;
  std::vector<int> bufA(L, -1), bufB(L, -1);
  auto pulls = [&](int s) -> dbm_status {
    const SpStep& x = sc->steps[s];
    ProfScope ps(ctx, ctx->comm, 5, 0.0,
                 (double)(((x.a_src != me) ? x.a_nnz : 0) + ((x.b_src != me) ? x.b_nnz : 0)) * bb * 8);
    if (x.a_src != me && x.a_nnz) {
      CUDA_TRY(ctx, cudaMemcpyAsync(ws + sc->off_recvA[bufA[s]], ctx->peer_ws[x.a_src] + sc->peer_ownA_off[x.a_src][x.kappa],
                                    (size_t)x.a_nnz * bb * 8, cudaMemcpyDeviceToDevice, ctx->comm));
    }
    if (x.b_src != me && x.b_nnz) {
      CUDA_TRY(ctx, cudaMemcpyAsync(ws + sc->off_recvB[bufB[s]], ctx->peer_ws[x.b_src] + sc->peer_ownB_off[x.b_src][x.kappa],
                                    (size_t)x.b_nnz * bb * 8, cudaMemcpyDeviceToDevice, ctx->comm));
    }
    if (x.a_src != me) st.bytes_recv += x.a_nnz * bb * 8;
    if (x.b_src != me) st.bytes_recv += x.b_nnz * bb * 8;
    for (int rr = 0; rr < ctx->pr; ++rr)  // what peers pull from me at this step (statistics)
      for (int cc = 0; cc < ctx->pc; ++cc) {
        const int dst = rr * ctx->pc + cc;
        if (dst == me) continue;
        const int k = (rr + cc + s) % (int)L;
        if (rr == ctx->myrow && k % ctx->pc == ctx->mycol) st.bytes_sent += sc->ownA_nnz[k] * bb * 8;
        if (cc == ctx->mycol && k % ctx->pr == ctx->myrow) st.bytes_sent += sc->ownB_nnz[k] * bb * 8;
      }
    return DBM_OK;
  };
  if (ctx->nranks > 1) {
    int na = 0, nb = 0;
    for (int s = 0; s < L; ++s) {
      if (sc->steps[s].a_src != me) bufA[s] = na++ & 1;
      if (sc->steps[s].b_src != me) bufB[s] = nb++ & 1;
      ev_x[s] = get_event(ctx);
      ev_g[s] = get_event(ctx);
    }
    ev_ready = get_event(ctx);
    CUDA_TRY(ctx, cudaEventRecord(ev_ready, cs));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm, ev_ready, 0));
    // my packed panels are ready (signal behind the packs) -> wait for every peer's (device-side)
    if (dbm_status e = xsignal(ctx, cs, X_READY, ep)) return e;
    if (dbm_status e = xwait(ctx, ctx->comm, X_READY, ep)) return e;
    if (dbm_status e = pulls(0)) return e;
    CUDA_TRY(ctx, cudaEventRecord(ev_x[0], ctx->comm));
  }
  int64_t* cnt = (int64_t*)(ws + sc->off_cnt);
  int64_t* offs = (int64_t*)(ws + sc->off_off);
  int32_t* trip = (int32_t*)(ws + sc->off_trip);
  for (int s = 0; s < L; ++s) {
    const SpStep& x = sc->steps[s];
    if (ctx->nranks > 1) {
      if (s + 1 < L) {
        if (s >= 1) CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm, ev_g[s - 1], 0));
        if (dbm_status e = pulls(s + 1)) return e;
        CUDA_TRY(ctx, cudaEventRecord(ev_x[s + 1], ctx->comm));
      }
      CUDA_TRY(ctx, cudaStreamWaitEvent(cs, ev_x[s], 0));
    }
    const double* Ap = ctx->nranks == 1 ? A->arena
                       : x.a_src != me ? (const double*)(ws + sc->off_recvA[bufA[s]])
                                       : (const double*)(xp + sc->ownA_off[x.kappa]);
    const double* Bp = ctx->nranks == 1 ? B->arena
                       : x.b_src != me ? (const double*)(ws + sc->off_recvB[bufB[s]])
                                       : (const double*)(xp + sc->ownB_off[x.kappa]);
    if (x.entries > 0) {
      const int64_t nruns = mloc * nloc;
      for (int64_t q0 = 0, ch = 0; q0 < nruns; q0 += sc->runs_per_chunk, ++ch) {
        const int64_t n = std::min(sc->runs_per_chunk, nruns - q0);
        const int64_t ent = x.chunk_entries[ch];
        if (ent == 0) continue;
        {
          // algorithmic bytes: the two A/B run lists read per run, 12 B written per entry
          ProfScope ps(ctx, cs, 4, 0.0, 12.0 * ent + 16.0 * n);
          CUDA_TRY(ctx, launch_sp_stackgen(meta + x.o_aptr, meta + x.o_akk, meta + x.o_bptr, meta + x.o_bkk,
                                           meta + x.o_bslot, C->sparse ? C->d_map : nullptr, nloc, trav_li, trav_lj, q0,
                                           n, cnt, offs, ws + sc->off_scan, sc->scan_bytes, trip, cs));
          launches += 3;
        }
        {
          ProfScope ps(ctx, cs, 1, 2.0 * bs * bb * ent, 16.0 * bb * ent);
          CUDA_TRY(ctx, launch_smm_sparse(bs, trip, offs, n, Ap, Bp, C->arena, alpha, cs));
          ++launches;
        }
      }
    }
    st.entries += x.entries;
    st.flops += 2.0 * bs * bb * x.entries;
    if (ctx->nranks > 1) CUDA_TRY(ctx, cudaEventRecord(ev_g[s], cs));
  }
  st.stacks = sp_stacks(sc, cap);
  if (ctx->nranks > 1) {
    CUDA_TRY(ctx, cudaStreamWaitEvent(cs, ev_x[L - 1], 0));
    // closing barrier: "done" behind my last pull, then wait for every peer's (no peer reads my panels)
    if (dbm_status e = xsignal(ctx, ctx->comm, X_DONE, ep)) return e;
    if (dbm_status e = xwait(ctx, cs, X_DONE, ep)) return e;
    cudaEvent_t done = get_event(ctx);
    CUDA_TRY(ctx, cudaEventRecord(done, cs));
    ctx->ev_pool.push_back(ev_ready);
    for (int s = 0; s < L; ++s) {
      ctx->ev_pool.push_back(ev_x[s]);
      ctx->ev_pool.push_back(ev_g[s]);
    }
    ctx->ev_pool.push_back(done);
  }
  ctx->launches += launches;
  st.kernel_launches = launches;
  if (stats) *stats = st;
  return DBM_OK;
}

// DBM_PATH_AUTO -> blocked / densified (should_densify)
dbm_path resolve_path(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_path path) {
  if (path != DBM_PATH_AUTO) return path;
  // non-uniform block-sparse operands: the blocked path takes dense patterns only (reading R16)
  if ((A->nonuni || B->nonuni) && (A->sparse || B->sparse)) return DBM_PATH_DENSIFIED;
  auto occ = [](dbm_matrix m) { return m->Mb * m->Nb ? (double)m->gnnz / (double)(m->Mb * m->Nb) : 1.0; };
  return (occ(A) >= ctx->densify_threshold && occ(B) >= ctx->densify_threshold) ? DBM_PATH_DENSIFIED
                                                                                : DBM_PATH_BLOCKED;
}

dbm_status sp_debug_stacks(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, int step, int32_t cap,
                           int32_t* triplets, int64_t* n_entries, int64_t* stack_ptr, int64_t* n_stacks) {
    SpCache* sc = nullptr;
    if (dbm_status e = sp_cache_get(ctx, A, B, C, &sc)) return e;
    ARG_CHECK(step >= 0 && step < sc->L, DBM_ERR_RANGE, "step out of range");
    const SpStep& x = sc->steps[step];
    const int64_t capv = cap ? cap : 30000;
    std::vector<int64_t> ptr{0};
    int64_t e = 0, cur = 0;
    for (int32_t n : x.run_len) {  // greedy whole-run packing (as sp_stacks), recording the boundaries
      if (n == 0) continue;
      if (n > capv) {
        if (cur) ptr.push_back(e);
        cur = 0;
        for (int64_t done = 0; done < n;) {
          done += std::min<int64_t>(capv, n - done);
          ptr.push_back(e + done);
        }
      } else {
        if (cur + n > capv) {
          ptr.push_back(e);
          cur = 0;
        }
        cur += n;
      }
      e += n;
    }
    if (cur) ptr.push_back(e);
    *n_entries = x.entries;
    *n_stacks = (int64_t)ptr.size() - 1;
    if (stack_ptr) std::memcpy(stack_ptr, ptr.data(), ptr.size() * 8);
    if (!triplets || x.entries == 0) return DBM_OK;
    const int64_t nruns = C->mloc * C->nloc;
    const size_t scan_bytes = sp_scan_temp_bytes(nruns + 1);
    char* d = nullptr;
    const size_t o_cnt = align256((size_t)nruns * 8), o_off = o_cnt + align256((size_t)(nruns + 1) * 8),
                 o_scan = o_off + align256((size_t)(nruns + 1) * 8), o_trip = o_scan + align256(scan_bytes),
                 total = o_trip + (size_t)x.entries * 12;
    CUDA_TRY(ctx, cudaMalloc(&d, total));
    int32_t* li = (int32_t*)d;
    launch_traversal(C->mloc, C->nloc, li, li + nruns, ctx->stream);
    const int32_t* meta = sc->d_meta;
    CUDA_TRY(ctx, launch_sp_stackgen(meta + x.o_aptr, meta + x.o_akk, meta + x.o_bptr, meta + x.o_bkk,
                                     meta + x.o_bslot, C->sparse ? C->d_map : nullptr, C->nloc, li, li + nruns, 0,
                                     nruns, (int64_t*)(d + o_cnt), (int64_t*)(d + o_off), d + o_scan, scan_bytes,
                                     (int32_t*)(d + o_trip), ctx->stream));
    ctx->launches += 4;
    CUDA_TRY(ctx, cudaMemcpyAsync(triplets, d + o_trip, (size_t)x.entries * 12, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    cudaFree(d);
    return DBM_OK;
}

dbm_status sp_workspace_bytes(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, int64_t* bytes) {
  SpCache* sc = nullptr;
  if (dbm_status e = sp_cache_get(ctx, A, B, C, &sc)) return e;
  *bytes = (int64_t)sc->total;
  return DBM_OK;
}

}  // namespace dbm

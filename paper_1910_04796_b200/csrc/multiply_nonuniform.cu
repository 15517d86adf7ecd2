// Multiply of matrices with non-uniform block sizes (reading R16): the same method
// as the uniform path -- Cannon over L = lcm(Pr, Pc) steps with owner-pull panels (reading R5),
// each local step blocked (stacks of (a, b, c) slot triplets -> small-block products of mixed (m, n, k),
// P:172-177) or densified (the panel's blocks coalesced into dense panels -> one DGEMM -> undensify,
// P:192-200) -- with every block carrying its own (m, k) / (k, n) shape.
//
//   * Panels: K-panel kappa = the k blocks with k = kappa (mod L); its element width W = sum of their
//     sizes.  Densified: A panel = local A rows x W (K-major rows, ld even), B panel = local B columns x W
//     (K-major columns); blocked: packed whole blocks, A row-major over (li, kk), B over (kk, lj) -- the
//     stack list is the uniform one (slots), the products read every slot's offset and shape from tables.
//   * Exchange: the copy-engine transport of the uniform path (exchange pool, device-side READY / DONE
//     signals, double-buffered receive panels on the comm stream).
//   * Not here: the step-0 K-chunked pull, the host-operand pipeline, single-rank K-chunking
//     of the dense buffers; the blocked path takes dense patterns and C blocks up to 64 x 64 (block-sparse
//     non-uniform operands run densified).
#include <algorithm>
#include <cstring>

#include "api_internal.h"

namespace dbm {

namespace {

// Host-only layout of one rank's side of the multiply (every rank can compute every rank's).
struct NURank {
  int pr = 1, pc = 1, r = 0, c = 0, L = 1;
  bool dens = true;
  int64_t mloc = 0, nloc = 0;
  std::vector<int64_t> lro, lco;        // local element row offset per li (A / C), column offset per lj (B / C)
  int64_t Mel = 0, Nel = 0;
  std::vector<std::vector<int64_t>> ks;  // per kappa: the global k blocks of the panel, ascending
  std::vector<std::vector<int64_t>> pko; // per kappa: element offset of panel k block kk (size kb + 1)
  std::vector<int64_t> ldk;              // per kappa: dense panel leading dimension (even)
  size_t a_bytes(int k) const { return (size_t)(dens ? Mel * ldk[k] : Mel * pko[k].back()) * 8; }
  size_t b_bytes(int k) const { return (size_t)(dens ? Nel * ldk[k] : Nel * pko[k].back()) * 8; }
  int s0 = 0;  // first canonical step (local-first order, several ranks: local_first_start)
  int kappa(int s) const { return (r + c + s + s0) % L; }
  int a_src(int s) const { return r * pc + kappa(s) % pc; }
  int b_src(int s) const { return (kappa(s) % pr) * pc + c; }
  int me() const { return r * pc + c; }
  std::vector<size_t> ownA, ownB;  // per kappa: exchange-pool offset, SIZE_MAX if not owned
  size_t pool_total = 0;
};

NURank nu_rank(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, bool dens, int r, int c) {
  NURank p;
  p.pr = ctx->pr;
  p.pc = ctx->pc;
  p.r = r;
  p.c = c;
  p.L = (int)lcm64(p.pr, p.pc);
  p.s0 = ctx->nranks > 1 && ctx->transport == 0 ? local_first_start(p.pr, p.pc, r * p.pc + c) : 0;
  p.dens = dens;
  p.mloc = local_count(A->Mb, p.pr, r);
  p.nloc = local_count(B->Nb, p.pc, c);
  p.lro.assign(p.mloc + 1, 0);
  for (int64_t li = 0; li < p.mloc; ++li) p.lro[li + 1] = p.lro[li] + A->row_size(r + li * p.pr);
  p.lco.assign(p.nloc + 1, 0);
  for (int64_t lj = 0; lj < p.nloc; ++lj) p.lco[lj + 1] = p.lco[lj] + B->col_size(c + lj * p.pc);
  p.Mel = p.lro.back();
  p.Nel = p.lco.back();
  p.ks.resize(p.L);
  p.pko.resize(p.L);
  p.ldk.resize(p.L);
  for (int k = 0; k < p.L; ++k) {
    p.pko[k].assign(1, 0);
    for (int64_t kg = k; kg < A->Nb; kg += p.L) {
      p.ks[k].push_back(kg);
      p.pko[k].push_back(p.pko[k].back() + A->col_size(kg));
    }
    p.ldk[k] = round_up(std::max<int64_t>(p.pko[k].back(), 1), 2);
  }
  p.ownA.assign(p.L, SIZE_MAX);
  p.ownB.assign(p.L, SIZE_MAX);
  if (ctx->nranks > 1) {
    size_t off = xhdr_bytes(ctx->nranks, p.L);
    for (int k = 0; k < p.L; ++k) {
      if (k % p.pc == c) {
        p.ownA[k] = off;
        off = align256(off + p.a_bytes(k));
      }
      if (k % p.pr == r) {
        p.ownB[k] = off;
        off = align256(off + p.b_bytes(k));
      }
    }
    p.pool_total = off;
  }
  return p;
}

}  // namespace

// Plan + device tables of one (A, B, C, path) triple on this rank, cached in the context.
struct NUCache {
  uint64_t a_serial = 0, b_serial = 0, c_serial = 0;
  bool dens = true;
  NURank me;
  size_t pool_need = 0;  // max over ranks
  // caller-owned workspace layout
  size_t off_recvA[2] = {0, 0}, off_recvB[2] = {0, 0}, off_cd = 0, off_part = 0, off_adense = 0, off_bdense = 0;
  size_t off_trav = 0, off_trip = 0, total = 256;
  int max_split = 1;
  int64_t trip_runs = 0;  // runs per stack chunk
  // device tables (one allocation) and their element offsets
  char* d_meta = nullptr;
  std::vector<size_t> o_atask, o_btask;     // per kappa (own panels): NUTask lists (densify) or NUPack lists (pack)
  std::vector<int64_t> n_atask, n_btask;
  size_t o_ctask = 0;                       // C undensify tasks
  int64_t n_ctask = 0;
  std::vector<size_t> o_aoff, o_boff, o_kdim;  // per kappa: panel slot -> element offset tables, k sizes (blocked)
  std::vector<size_t> o_kofs, o_gbeg;          // per kappa: entry k offsets inside their groups, group starts
  std::vector<int> ngroups;
  int kmax = 1, mmax = 1, nmax = 1, kcap = 32;
};

namespace {

dbm_status nu_cache_get(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, bool dens, NUCache** out) {
  for (dbm_matrix m : {A, B, C})  // uniform operands beside non-uniform ones: per-slot tables
    if (dbm_status e = nu_tables(m)) return e;
  for (NUCache* c : ctx->nu_cache)
    if (c->a_serial == A->serial && c->b_serial == B->serial && c->c_serial == C->serial && c->dens == dens) {
      *out = c;
      return DBM_OK;
    }
  NUCache* nc = new NUCache();
  nc->a_serial = A->serial;
  nc->b_serial = B->serial;
  nc->c_serial = C->serial;
  nc->dens = dens;
  const int r = ctx->myrow, c = ctx->mycol;
  nc->me = nu_rank(ctx, A, B, dens, r, c);
  const NURank& p = nc->me;
  for (int q = 0; q < ctx->nranks; ++q)
    nc->pool_need = std::max(nc->pool_need, q == ctx->rank ? p.pool_total
                                                           : nu_rank(ctx, A, B, dens, q / ctx->pc, q % ctx->pc).pool_total);
  // workspace
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + bytes);
    return o;
  };
  if (ctx->nranks > 1) {
    size_t amax = 0, bmax = 0;
    int na = 0, nb = 0;
    for (int s = 0; s < p.L; ++s) {
      if (p.a_src(s) != p.me()) {
        amax = std::max(amax, p.a_bytes(p.kappa(s)));
        ++na;
      }
      if (p.b_src(s) != p.me()) {
        bmax = std::max(bmax, p.b_bytes(p.kappa(s)));
        ++nb;
      }
    }
    for (int i = 0; i < std::min(na, 2); ++i) nc->off_recvA[i] = take(amax);
    for (int i = 0; i < std::min(nb, 2); ++i) nc->off_recvB[i] = take(bmax);
  }
  if (dens) {
    nc->off_cd = take((size_t)p.Mel * p.Nel * 8);
    if (ctx->nranks == 1) {  // the whole local A / B densified once (no K-chunking on this path)
      nc->off_adense = take((size_t)p.Mel * p.ldk[0] * 8);
      nc->off_bdense = take((size_t)p.Nel * p.ldk[0] * 8);
    }
    for (int k = 0; k < p.L; ++k) nc->max_split = std::max(nc->max_split, pick_splitk(p.Mel, p.Nel, p.pko[k].back(), num_sms()));
    if (nc->max_split > 1) nc->off_part = take((size_t)nc->max_split * p.Mel * p.Nel * 8);
  } else {
    nc->off_trav = take((size_t)std::max<int64_t>(p.mloc * p.nloc, 1) * 8);
    int64_t maxkb = 1;
    for (int k = 0; k < p.L; ++k) maxkb = std::max<int64_t>(maxkb, (int64_t)p.ks[k].size());
    nc->trip_runs = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(p.mloc * p.nloc, 1), kTripChunkEntries / maxkb));
    nc->off_trip = take((size_t)nc->trip_runs * maxkb * 12);
  }
  nc->total = std::max<size_t>(off, 256);

  // device tables
  std::vector<char> meta;
  auto put = [&](const void* d, size_t bytes) {
    size_t o = align256(meta.size());
    meta.resize(o + bytes);
    if (bytes) std::memcpy(meta.data() + o, d, bytes);
    return o;
  };
  auto a_slot = [&](int64_t li, int64_t kl) { return A->sparse ? -1 : li * A->nloc + kl; };  // dense patterns
  nc->o_atask.assign(p.L, SIZE_MAX);
  nc->o_btask.assign(p.L, SIZE_MAX);
  nc->n_atask.assign(p.L, 0);
  nc->n_btask.assign(p.L, 0);
  nc->o_aoff.assign(p.L, SIZE_MAX);
  nc->o_boff.assign(p.L, SIZE_MAX);
  nc->o_kdim.assign(p.L, SIZE_MAX);
  // local slot lookup (sparse patterns: CSR search; -1 = absent)
  auto slot_of = [](dbm_matrix m, int64_t li, int64_t lj) -> int64_t {
    if (!m->sparse) return li * m->nloc + lj;
    const auto b = m->col.begin() + m->row_ptr[li], e = m->col.begin() + m->row_ptr[li + 1];
    const auto it = std::lower_bound(b, e, (int32_t)lj);
    return (it != e && *it == (int32_t)lj) ? (int64_t)(it - m->col.begin()) : -1;
  };
  (void)a_slot;
  const bool multi = ctx->nranks > 1;
  std::vector<std::vector<int32_t>> kdims(p.L);  // per kappa: the panel's k-block sizes (blocked)
  for (int k = 0; k < p.L; ++k) {
    const int64_t kb = (int64_t)p.ks[k].size();
    if (dens) {
      // own A panel (or, on one rank, the whole local A = panel 0): K-major rows
      if (multi ? p.ownA[k] != SIZE_MAX : k == 0) {
        std::vector<NUTask> t;
        for (int64_t li = 0; li < p.mloc; ++li)
          for (int64_t kk = 0; kk < kb; ++kk) {
            const int64_t s = slot_of(A, li, (p.ks[k][kk] - c) / p.pc);
            if (s < 0) continue;
            t.push_back({A->slot_off[s], p.lro[li], p.pko[k][kk], A->row_size(r + li * p.pr),
                         A->col_size(p.ks[k][kk])});
          }
        nc->o_atask[k] = put(t.data(), t.size() * sizeof(NUTask));
        nc->n_atask[k] = (int64_t)t.size();
      }
      if (multi ? p.ownB[k] != SIZE_MAX : k == 0) {  // own B panel: K-major columns
        std::vector<NUTask> t;
        for (int64_t kk = 0; kk < kb; ++kk)
          for (int64_t lj = 0; lj < p.nloc; ++lj) {
            const int64_t s = slot_of(B, (p.ks[k][kk] - r) / p.pr, lj);
            if (s < 0) continue;
            t.push_back({B->slot_off[s], p.pko[k][kk], p.lco[lj], B->row_size(p.ks[k][kk]),
                         B->col_size(c + lj * p.pc)});
          }
        nc->o_btask[k] = put(t.data(), t.size() * sizeof(NUTask));
        nc->n_btask[k] = (int64_t)t.size();
      }
    } else {
      // packed panel offsets (every kappa: the consumer reads the panel of step s in this layout)
      std::vector<int64_t> ao, bo;
      std::vector<int32_t> kd;
      int64_t o = 0;
      for (int64_t li = 0; li < p.mloc; ++li)
        for (int64_t kk = 0; kk < kb; ++kk) {
          ao.push_back(o);
          o += (int64_t)A->row_size(r + li * p.pr) * A->col_size(p.ks[k][kk]);
        }
      o = 0;
      for (int64_t kk = 0; kk < kb; ++kk)
        for (int64_t lj = 0; lj < p.nloc; ++lj) {
          bo.push_back(o);
          o += (int64_t)B->row_size(p.ks[k][kk]) * B->col_size(c + lj * p.pc);
        }
      for (int64_t kk = 0; kk < kb; ++kk) {
        kd.push_back(A->col_size(p.ks[k][kk]));
        nc->kmax = std::max(nc->kmax, (int)kd.back());
      }
      if (!multi) {  // one rank: the arenas are the panels (A slot li*kA + kk, B slot kk*nloc + lj)
        ao.assign(A->slot_off.begin(), A->slot_off.end() - 1);
        bo.assign(B->slot_off.begin(), B->slot_off.end() - 1);
      }
      nc->o_aoff[k] = put(ao.data(), ao.size() * 8);
      nc->o_boff[k] = put(bo.data(), bo.size() * 8);
      nc->o_kdim[k] = put(kd.data(), kd.size() * 4);
      kdims[k] = kd;
      if (multi && p.ownA[k] != SIZE_MAX) {  // pack my A panel kappa: blocks (li, kk) in row-major order
        std::vector<NUPack> t;
        for (int64_t li = 0; li < p.mloc; ++li)
          for (int64_t kk = 0; kk < kb; ++kk) {
            const int64_t s = slot_of(A, li, (p.ks[k][kk] - c) / p.pc);
            t.push_back({A->slot_off[s], ao[li * kb + kk], A->slot_off[s + 1] - A->slot_off[s]});
          }
        nc->o_atask[k] = put(t.data(), t.size() * sizeof(NUPack));
        nc->n_atask[k] = (int64_t)t.size();
      }
      if (multi && p.ownB[k] != SIZE_MAX) {  // pack my B panel kappa: blocks (kk, lj)
        std::vector<NUPack> t;
        for (int64_t kk = 0; kk < kb; ++kk)
          for (int64_t lj = 0; lj < p.nloc; ++lj) {
            const int64_t s = slot_of(B, (p.ks[k][kk] - r) / p.pr, lj);
            t.push_back({B->slot_off[s], bo[kk * p.nloc + lj], B->slot_off[s + 1] - B->slot_off[s]});
          }
        nc->o_btask[k] = put(t.data(), t.size() * sizeof(NUPack));
        nc->n_btask[k] = (int64_t)t.size();
      }
    }
  }
  for (int64_t li = 0; li < p.mloc; ++li) nc->mmax = std::max(nc->mmax, (int)A->row_size(r + li * p.pr));
  for (int64_t lj = 0; lj < p.nloc; ++lj) nc->nmax = std::max(nc->nmax, (int)B->col_size(c + lj * p.pc));
  if (!dens) {  // entry groups of the small-block kernel: consecutive entries with summed k <= kcap (and
              // at most kNuGroupMaxEntries of them)
    static const int kcap_env = [] {  // (tuning knob: DBM_NU_KCAP, default 32)
      const char* e = getenv("DBM_NU_KCAP");
      return e ? std::max(4, atoi(e)) : 32;
    }();
    nc->kcap = std::max(nc->kmax, kcap_env);
    nc->o_kofs.assign(p.L, SIZE_MAX);
    nc->o_gbeg.assign(p.L, SIZE_MAX);
    nc->ngroups.assign(p.L, 0);
    for (int k = 0; k < p.L; ++k) {
      std::vector<int32_t> kofs, gbeg{0};
      int32_t acc = 0;
      for (size_t e = 0; e < kdims[k].size(); ++e) {
        if (acc + kdims[k][e] > nc->kcap || (int64_t)e - gbeg.back() == kNuGroupMaxEntries) {
          gbeg.push_back((int32_t)e);
          acc = 0;
        }
        kofs.push_back(acc);
        acc += kdims[k][e];
      }
      if (!kdims[k].empty()) gbeg.push_back((int32_t)kdims[k].size());
      nc->ngroups[k] = (int)gbeg.size() - 1;
      nc->o_kofs[k] = put(kofs.data(), kofs.size() * 4);
      nc->o_gbeg[k] = put(gbeg.data(), gbeg.size() * 4);
    }
  }
  if (dens) {  // undensify C (stored blocks only)
    std::vector<NUTask> t;
    for (int64_t li = 0; li < p.mloc; ++li)
      for (int64_t lj = 0; lj < p.nloc; ++lj) {
        const int64_t s = slot_of(C, li, lj);
        if (s < 0) continue;
        t.push_back({C->slot_off[s], p.lro[li], p.lco[lj],
                     C->row_size(r + li * p.pr), C->col_size(c + lj * p.pc)});
      }
    nc->o_ctask = put(t.data(), t.size() * sizeof(NUTask));
    nc->n_ctask = (int64_t)t.size();
  }
  cudaError_t e = cudaMalloc(&nc->d_meta, std::max<size_t>(meta.size(), 256));
  if (e == cudaSuccess && !meta.empty()) e = cudaMemcpy(nc->d_meta, meta.data(), meta.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (nc->d_meta) cudaFree(nc->d_meta);
    delete nc;
    set_error(std::string("non-uniform plan tables: ") + cudaGetErrorString(e));
    return DBM_ERR_NOMEM;
  }
  ctx->nu_cache.push_back(nc);
  *out = nc;
  return DBM_OK;
}

}  // namespace

void free_nu_cache(dbm_ctx ctx) {
  for (NUCache* c : ctx->nu_cache) {
    if (c->d_meta) cudaFree(c->d_meta);
    delete c;
  }
  ctx->nu_cache.clear();
}

dbm_status nu_workspace_bytes(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, bool dens, int64_t* bytes) {
  NUCache* nc = nullptr;
  if (dbm_status e = nu_cache_get(ctx, A, B, C, dens, &nc)) return e;
  *bytes = (int64_t)nc->total;
  return DBM_OK;
}

dbm_status multiply_nonuniform(dbm_ctx ctx, double alpha, dbm_matrix A, dbm_matrix B, double beta, dbm_matrix C,
                               bool dens, void* workspace, int64_t ws_bytes, dbm_stats* stats) {
  ARG_CHECK(dens || !(A->sparse || B->sparse || C->sparse), DBM_ERR_ARG,
            "non-uniform block-sparse matrices take the densified path (reading R16)");
  NUCache* nc = nullptr;
  if (dbm_status e = nu_cache_get(ctx, A, B, C, dens, &nc)) return e;
  const NURank& p = nc->me;
  ARG_CHECK(workspace != nullptr && ws_bytes >= (int64_t)nc->total, DBM_ERR_WORKSPACE,
            "workspace smaller than dbm_multiply_workspace()");
  if (!dens) {
    ARG_CHECK(nc->mmax <= 64 && nc->nmax <= 64, DBM_ERR_SHAPE,
              "blocked path: C blocks up to 64 x 64 (larger blocks: the densified path)");
    ARG_CHECK(nu_smm_smem(nc->kcap, nc->mmax, nc->nmax) <= 227 * 1024, DBM_ERR_SHAPE,
              "blocked path: A / B blocks too large for the shared-memory stages (use the densified path)");
  }
  cudaStream_t cs = ctx->stream;
  char* ws = (char*)workspace;
  char* meta = nc->d_meta;
  dbm_stats st{};
  st.steps = p.L;
  int launches = 0;
  const int64_t Kb = A->Nb;
  if (alpha == 0.0 || Kb == 0 || p.Mel * p.Nel == 0) {  // BLAS convention (reading R8): A, B not read
    if (C->elems()) {
      launch_scale(C->arena, C->elems(), beta, cs);
      ++launches;
      CUDA_TRY(ctx, cudaGetLastError());
    }
    if (alpha == 0.0 || Kb == 0 || ctx->nranks == 1) {  // (empty local C on several ranks: still collective)
      ctx->launches += launches;
      st.kernel_launches = launches;
      if (stats) *stats = st;
      return DBM_OK;
    }
  }
  const bool multi = ctx->nranks > 1;
  char* xp = nullptr;
  uint64_t ep = 0;
  if (multi) {
    if (dbm_status e = xattach(ctx, nc->pool_need, cs)) return e;
    xp = ctx->xpool;
    ep = ++ctx->epoch;
  }
  // ---- own panels (densified or packed) on the compute stream
  auto own_panel = [&](int k, bool isA, double* dst) -> dbm_status {
    const size_t o = isA ? nc->o_atask[k] : nc->o_btask[k];
    const int64_t n = isA ? nc->n_atask[k] : nc->n_btask[k];
    const size_t bytes = isA ? p.a_bytes(k) : p.b_bytes(k);
    if (dens) {
      if ((isA ? A : B)->sparse && bytes) CUDA_TRY(ctx, cudaMemsetAsync(dst, 0, bytes, cs));  // absent blocks: zeros
      ProfScope ps(ctx, cs, 2, 0.0, 16.0 * (bytes / 8));
      launch_nu_copy((const NUTask*)(meta + o), n, (isA ? A : B)->arena, dst, p.ldk[k], isA ? 0 : 1, 0, 0, cs);
    } else {
      ProfScope ps(ctx, cs, 2, 0.0, 16.0 * (bytes / 8));
      launch_nu_pack((const NUPack*)(meta + o), n, (isA ? A : B)->arena, dst, cs);
    }
    ++launches;
    CUDA_TRY(ctx, cudaGetLastError());
    return DBM_OK;
  };
  if (multi) {
    for (int k = 0; k < p.L; ++k) {
      if (p.ownA[k] != SIZE_MAX)
        if (dbm_status e = own_panel(k, true, (double*)(xp + p.ownA[k]))) return e;
      if (p.ownB[k] != SIZE_MAX)
        if (dbm_status e = own_panel(k, false, (double*)(xp + p.ownB[k]))) return e;
    }
  } else if (dens) {
    if (dbm_status e = own_panel(0, true, (double*)(ws + nc->off_adense))) return e;
    if (dbm_status e = own_panel(0, false, (double*)(ws + nc->off_bdense))) return e;
  }
  // ---- Cannon setup: my panels ready -> every owner's panels ready (device-side signals)
  std::vector<cudaEvent_t> ev_x(p.L, nullptr), ev_g(p.L, nullptr);
  std::vector<int> bufA(p.L, -1), bufB(p.L, -1);
  if (multi) {
    int na = 0, nb = 0;
    for (int s = 0; s < p.L; ++s) {
      if (p.a_src(s) != p.me()) bufA[s] = na++ & 1;
      if (p.b_src(s) != p.me()) bufB[s] = nb++ & 1;
      ev_x[s] = get_event(ctx);
      ev_g[s] = get_event(ctx);
    }
    cudaEvent_t ev_ready = get_event(ctx);
    CUDA_TRY(ctx, cudaEventRecord(ev_ready, cs));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm, ev_ready, 0));
    ctx->ev_pool.push_back(ev_ready);
    if (dbm_status e = xsignal(ctx, cs, X_READY, ep)) return e;
    if (dbm_status e = xwait(ctx, ctx->comm, X_READY, ep)) return e;
  }
  std::vector<NURank> peer(ctx->nranks);
  auto peer_of = [&](int q) -> const NURank& {
    if (peer[q].L == 1 && q != ctx->rank && multi) peer[q] = nu_rank(ctx, A, B, dens, q / ctx->pc, q % ctx->pc);
    return q == ctx->rank ? p : peer[q];
  };
  auto pulls = [&](int s) -> dbm_status {  // copy-engine pulls of step s's remote panels
    const int k = p.kappa(s);
    double bytes = 0;
    if (p.a_src(s) != p.me()) bytes += (double)p.a_bytes(k);
    if (p.b_src(s) != p.me()) bytes += (double)p.b_bytes(k);
    ProfScope ps(ctx, ctx->comm, 5, 0.0, bytes);
    if (p.a_src(s) != p.me() && p.a_bytes(k)) {
      const NURank& q = peer_of(p.a_src(s));
      CUDA_TRY(ctx, cudaMemcpyAsync(ws + nc->off_recvA[bufA[s]], ctx->peer_ws[p.a_src(s)] + q.ownA[k], p.a_bytes(k),
                                    cudaMemcpyDeviceToDevice, ctx->comm));
      st.bytes_recv += (int64_t)p.a_bytes(k);
    }
    if (p.b_src(s) != p.me() && p.b_bytes(k)) {
      const NURank& q = peer_of(p.b_src(s));
      CUDA_TRY(ctx, cudaMemcpyAsync(ws + nc->off_recvB[bufB[s]], ctx->peer_ws[p.b_src(s)] + q.ownB[k], p.b_bytes(k),
                                    cudaMemcpyDeviceToDevice, ctx->comm));
      st.bytes_recv += (int64_t)p.b_bytes(k);
    }
    // what the peers pull from me at step s (statistics): my own panels that are their step-s panels
    for (int q = 0; q < ctx->nranks; ++q) {
      if (q == p.me()) continue;
      const NURank& o = peer_of(q);
      if (o.a_src(s) == p.me()) st.bytes_sent += (int64_t)o.a_bytes(o.kappa(s));
      if (o.b_src(s) == p.me()) st.bytes_sent += (int64_t)o.b_bytes(o.kappa(s));
    }
    return DBM_OK;
  };
  int32_t* trav_li = (int32_t*)(ws + nc->off_trav);
  int32_t* trav_lj = trav_li + std::max<int64_t>(p.mloc * p.nloc, 1);
  int32_t* trip = (int32_t*)(ws + nc->off_trip);
  if (!dens && p.mloc * p.nloc > 0) {
    ProfScope ps(ctx, cs, 4, 0.0, 8.0 * p.mloc * p.nloc);
    launch_traversal(p.mloc, p.nloc, trav_li, trav_lj, cs);
    ++launches;
  }
  auto body = [&]() -> dbm_status {
    if (multi) {
      if (dbm_status e = pulls(0)) return e;
      CUDA_TRY(ctx, cudaEventRecord(ev_x[0], ctx->comm));
    }
    double* Cd = (double*)(ws + nc->off_cd);
    for (int s = 0; s < p.L; ++s) {
      const int k = p.kappa(s);
      const int64_t kb = (int64_t)p.ks[k].size(), W = p.pko[k].back();
      if (multi) {
        if (s + 1 < p.L) {  // prefetch step s+1 while step s computes (P:171 overlap)
          if (s >= 1) CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm, ev_g[s - 1], 0));
          if (dbm_status e = pulls(s + 1)) return e;
          CUDA_TRY(ctx, cudaEventRecord(ev_x[s + 1], ctx->comm));
        }
        CUDA_TRY(ctx, cudaStreamWaitEvent(cs, ev_x[s], 0));
      }
      const double* Ap = !multi ? (dens ? (const double*)(ws + nc->off_adense) : A->arena)
                         : p.a_src(s) != p.me() ? (const double*)(ws + nc->off_recvA[bufA[s]])
                                                : (const double*)(xp + p.ownA[k]);
      const double* Bp = !multi ? (dens ? (const double*)(ws + nc->off_bdense) : B->arena)
                         : p.b_src(s) != p.me() ? (const double*)(ws + nc->off_recvB[bufB[s]])
                                                : (const double*)(xp + p.ownB[k]);
      if (dens && p.Mel * p.Nel > 0) {
        GemmArgs g{p.Mel, p.Nel, W, Ap, p.ldk[k], Bp, p.ldk[k], Cd, p.Mel, 1.0, s == 0 ? 0.0 : 1.0, 1, nullptr};
        g.splitk = std::min(pick_splitk(g.M, g.N, g.K, num_sms()), nc->max_split);
        g.partial = g.splitk > 1 ? (double*)(ws + nc->off_part) : nullptr;
        ProfScope ps(ctx, cs, 0, 2.0 * g.M * g.N * g.K, 8.0 * (g.M * g.K + g.N * g.K + g.M * g.N * (s ? 2 : 1)));
        CUDA_TRY(ctx, launch_dgemm(g, cs, &launches));
        ++st.gemm_launches;
        st.entries += 1;  // the densified batch holds one multiplication
        st.stacks += 1;
        st.flops += 2.0 * p.Mel * p.Nel * W;
      } else if (!dens && kb > 0 && p.mloc * p.nloc > 0) {
        const int64_t nruns = p.mloc * p.nloc;
        for (int64_t q0 = 0; q0 < nruns; q0 += nc->trip_runs) {
          const int64_t q1 = std::min(nruns, q0 + nc->trip_runs);
          {
            ProfScope ps(ctx, cs, 4, 0.0, 12.0 * (q1 - q0) * kb);
            launch_stackgen(trav_li, trav_lj, q0, q1, kb, p.nloc, kb, p.nloc, trip, cs);
            ++launches;
          }
          // flops of the chunk: the step's 2 Mel Nel W spread over the runs (exact for one chunk per step)
          ProfScope ps(ctx, cs, 1, 2.0 * (double)p.Mel * p.Nel * W * (double)(q1 - q0) / (double)nruns, 0.0);
          CUDA_TRY(ctx, launch_nu_smm(trip, q1 - q0, kb, Ap, (const int64_t*)(meta + nc->o_aoff[k]), Bp,
                                      (const int64_t*)(meta + nc->o_boff[k]), (const int32_t*)(meta + nc->o_kdim[k]),
                                      (const int32_t*)(meta + nc->o_kofs[k]), (const int32_t*)(meta + nc->o_gbeg[k]),
                                      nc->ngroups[k], C->arena, C->d_blk, nc->kcap, nc->mmax, nc->nmax, alpha,
                                      s == 0 ? beta : 1.0, cs));
          ++launches;
        }
        st.entries += nruns * kb;
        const int64_t cap = 30000;
        st.stacks += kb <= cap ? (nruns + (cap / kb) - 1) / (cap / kb) : nruns * ((kb + cap - 1) / cap);
        st.flops += 2.0 * (double)p.Mel * p.Nel * W;
      } else if (!dens && s == 0 && C->elems()) {  // empty K panel at step 0 still applies beta once
        launch_scale(C->arena, C->elems(), beta, cs);
        ++launches;
      }
      CUDA_TRY(ctx, cudaGetLastError());
      if (multi) CUDA_TRY(ctx, cudaEventRecord(ev_g[s], cs));
    }
    if (multi) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, ev_x[p.L - 1], 0));
    if (dens && nc->n_ctask) {
      ProfScope ps(ctx, cs, 3, 0.0, (beta == 0.0 ? 16.0 : 24.0) * p.Mel * p.Nel);
      launch_nu_copy((const NUTask*)(meta + nc->o_ctask), nc->n_ctask, C->arena, Cd, p.Mel, 2, alpha, beta, cs);
      ++launches;
      CUDA_TRY(ctx, cudaGetLastError());
    }
    return DBM_OK;
  };
  const dbm_status berr = body();
  if (multi) {  // closing barrier: no peer still pulls from my exchange pool
    if (dbm_status e = xsignal(ctx, ctx->comm, X_DONE, ep)) return e;
    if (dbm_status e = xwait(ctx, cs, X_DONE, ep)) return e;
    for (int s = 0; s < p.L; ++s) {
      ctx->ev_pool.push_back(ev_x[s]);
      ctx->ev_pool.push_back(ev_g[s]);
    }
  }
  if (berr != DBM_OK) {
    if (ctx->poisoned == DBM_OK) ctx->poisoned = berr;
    return berr;
  }
  ctx->launches += launches;
  st.kernel_launches = launches;
  if (stats) *stats = st;
  return DBM_OK;
}

}  // namespace dbm

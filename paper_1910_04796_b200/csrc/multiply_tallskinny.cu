// Tall-and-skinny MPI-level algorithm (§II, reading R14; §8f-1): 1-D K decomposition, one partial
// GEMM per rank, fixed-order reduction of the small C.  Part of libdbm's host runtime (include/dbm.h:
// dbm_ctx_set_algorithm(ctx, 1)).
#include "api_internal.h"

namespace dbm {

namespace {
// ====================================================================== tall-and-skinny
// "only for tall-and-skinny matrices (one large dimension) we use an optimized algorithm" (§II;
// 1-D decomposition of K, local partial products, reduction of the small C).
// Reading R14: rank p = r*Pc + c takes the K blocks S_p = {k : k mod P == p}.  Every
// k in S_p has k mod Pc == c, so A[:, S_p] lives in p's grid column: rank (r', c) contributes its
// rows (i = r' mod Pr) as one dense K-major piece; B[S_p, :] lives in grid row p mod Pr: rank
// (p mod Pr, c') contributes its columns.  p assembles A_full (all M rows) x B_full (all N cols),
// computes the partial C_p = A[:, S_p] B[S_p, :] with one GEMM (pulled in K-chunks, each chunk
// followed by its GEMM chunk), and finally every rank pulls its own C blocks' sub-rectangle out of
// all P partials and sums them in rank order (deterministic) with alpha / beta.  Rows of A_full /
// C_p are ordered (r', li) and columns of B_full / C_p (c', lj), so each owner's piece and each
// rank's C share are contiguous 2-D sub-rectangles: every transfer is one copy-engine copy.
struct TSPlan {
  int P = 1, pr = 1, pc = 1, r = 0, c = 0, me = 0;
  int64_t bs = 0, Mb = 0, Nb = 0, Kb = 0;
  std::vector<int64_t> kp;                 // |S_q| (blocks) per rank q
  std::vector<int64_t> mrows, rowoff;      // per grid row r': rows (elements) and offset in A_full / C_p
  std::vector<int64_t> ncols, coloff;      // per grid column c'
  int64_t Mtot = 0, Ntot = 0;
  std::vector<size_t> offApiece, offBpiece;  // my pieces: A per target row tr, B per target t (q = r + t*pr)
  size_t off_afull = 0, off_bfull = 0, off_cpart = 0, off_cstack = 0, off_part = 0, total = 0;
  size_t pool_total = 0;  // exchange pool: header + pieces + partial C (offApiece, offBpiece, off_cpart)
  int max_split = 1;
  int64_t ld(int q) const { return round_up(std::max<int64_t>(kp[q] * bs, 1), 2); }
  size_t a_piece_bytes(int q, int rr) const { return kp[q] ? (size_t)mrows[rr] * ld(q) * 8 : 0; }
  size_t b_piece_bytes(int q, int cc) const { return kp[q] ? (size_t)ncols[cc] * ld(q) * 8 : 0; }
};

TSPlan make_ts_plan(int pr, int pc, int r, int c, int64_t Mb, int64_t Nb, int64_t Kb, int64_t bs) {
  TSPlan t;
  t.P = pr * pc;
  t.pr = pr;
  t.pc = pc;
  t.r = r;
  t.c = c;
  t.me = r * pc + c;
  t.bs = bs;
  t.Mb = Mb;
  t.Nb = Nb;
  t.Kb = Kb;
  t.kp.resize(t.P);
  for (int q = 0; q < t.P; ++q) t.kp[q] = local_count(Kb, t.P, q);
  t.mrows.resize(pr);
  t.rowoff.resize(pr);
  for (int rr = 0; rr < pr; ++rr) {
    t.mrows[rr] = local_count(Mb, pr, rr) * bs;
    t.rowoff[rr] = rr ? t.rowoff[rr - 1] + t.mrows[rr - 1] : 0;
  }
  t.ncols.resize(pc);
  t.coloff.resize(pc);
  for (int cc = 0; cc < pc; ++cc) {
    t.ncols[cc] = local_count(Nb, pc, cc) * bs;
    t.coloff[cc] = cc ? t.coloff[cc - 1] + t.ncols[cc - 1] : 0;
  }
  t.Mtot = Mb * bs;
  t.Ntot = Nb * bs;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + bytes);
    return o;
  };
  // what the peers read (my pieces, my partial C) lives in the exchange pool, after the signal header
  size_t poff = xhdr_bytes(pr * pc, (int)lcm64(pr, pc));
  auto take_pool = [&](size_t bytes) {
    size_t o = poff;
    poff = align256(poff + bytes);
    return o;
  };
  t.offApiece.resize(pr);
  for (int tr = 0; tr < pr; ++tr) t.offApiece[tr] = take_pool(t.a_piece_bytes(tr * pc + c, r));
  t.offBpiece.resize(pc);
  for (int tt = 0; tt < pc; ++tt) t.offBpiece[tt] = take_pool(t.b_piece_bytes(r + tt * pr, c));
  t.off_cpart = take_pool((size_t)t.Mtot * t.Ntot * 8);
  t.pool_total = poff;
  t.off_afull = take((size_t)t.Mtot * t.ld(t.me) * 8);
  t.off_bfull = take((size_t)t.Ntot * t.ld(t.me) * 8);
  t.off_cstack = take((size_t)t.P * t.mrows[r] * t.ncols[c] * 8);
  const int64_t K = t.kp[t.me] * bs;
  const std::vector<int64_t> cb = pipeline_chunks(t.kp[t.me]);
  for (size_t j = 1; j < cb.size(); ++j)
    t.max_split = std::max(t.max_split, pick_splitk(t.Mtot, t.Ntot, (cb[j] - cb[j - 1]) * bs, num_sms()));
  t.max_split = std::max(t.max_split, pick_splitk(t.Mtot, t.Ntot, K, num_sms()));
  if (t.max_split > 1) t.off_part = take((size_t)t.max_split * t.Mtot * t.Ntot * 8);
  t.total = std::max<size_t>(off, 256);
  return t;
}

// Bytes this rank pulls from peers / peers pull from it in one tall-and-skinny multiply.
void ts_bytes(const TSPlan& t, int64_t* recv, int64_t* sent) {
  int64_t rv = 0, sd = 0;
  for (int rr = 0; rr < t.pr; ++rr)
    if (rr != t.r) rv += (int64_t)t.a_piece_bytes(t.me, rr);
  const int rb = t.me % t.pr;
  for (int cc = 0; cc < t.pc; ++cc)
    if (rb * t.pc + cc != t.me) rv += (int64_t)t.b_piece_bytes(t.me, cc);
  for (int q = 0; q < t.P; ++q)
    if (q != t.me) rv += t.mrows[t.r] * t.ncols[t.c] * 8;  // my C share out of every other partial
  // what the others pull from me
  for (int tr = 0; tr < t.pr; ++tr)
    if (tr != t.r) sd += (int64_t)t.a_piece_bytes(tr * t.pc + t.c, t.r);
  for (int tt = 0; tt < t.pc; ++tt) {
    const int q = t.r + tt * t.pr;
    if (q != t.me) sd += (int64_t)t.b_piece_bytes(q, t.c);
  }
  for (int q = 0; q < t.P; ++q)
    if (q != t.me) sd += t.mrows[q / t.pc] * t.ncols[q % t.pc] * 8;
  *recv = rv;
  *sent = sd;
}

}  // namespace

size_t ts_workspace_bytes(int pr, int pc, int r, int c, int64_t Mb, int64_t Nb, int64_t Kb, int64_t bs) {
  return make_ts_plan(pr, pc, r, c, Mb, Nb, Kb, bs).total;
}

void ts_plan_bytes(int pr, int pc, int r, int c, int64_t Mb, int64_t Nb, int64_t Kb, int64_t bs, int64_t* recv,
                   int64_t* sent) {
  ts_bytes(make_ts_plan(pr, pc, r, c, Mb, Nb, Kb, bs), recv, sent);
}

dbm_status multiply_tallskinny(dbm_ctx ctx, double alpha, dbm_matrix A, dbm_matrix B, double beta, dbm_matrix C,
                               char* ws, dbm_stats* st, int* launches) {
  const TSPlan t = make_ts_plan(ctx->pr, ctx->pc, ctx->myrow, ctx->mycol, A->Mb, B->Nb, A->Nb, A->bs);
  cudaStream_t cs = ctx->stream;
  const int64_t bs = t.bs, P = t.P;
  size_t need = t.pool_total;  // every rank's pool need: the growth decision is the same on every rank
  for (int q = 0; q < P; ++q)
    need = std::max(need, make_ts_plan(t.pr, t.pc, q / t.pc, q % t.pc, t.Mb, t.Nb, t.Kb, bs).pool_total);
  if (dbm_status e = xattach(ctx, need, cs)) return e;
  char* xp = ctx->xpool;
  const uint64_t ep = ++ctx->epoch;
  // ---- own pieces (densified once; peers pull them).  The pieces this rank needs itself are densified
  // straight into its A_full / B_full: a local device-to-device copy would run on SMs and wait behind
  // the persistent GEMM (measured: 23 GB/s under a GEMM vs 750 GB/s for the peer pulls on the copy
  // engines, tools/microbench/ce_copy.py).
  for (int tr = 0; tr < t.pr; ++tr) {
    const int q = tr * t.pc + t.c;
    if (!t.kp[q] || !t.mrows[t.r]) continue;
    double* dst = q == t.me ? (double*)(ws + t.off_afull) + (size_t)t.rowoff[t.r] * t.ld(q)
                            : (double*)(xp + t.offApiece[tr]);
    ProfScope ps(ctx, cs, 2, 0.0, 16.0 * t.mrows[t.r] * t.kp[q] * bs);
    if (dbm_status e = densify_a(ctx, A, tr, t.pr, t.kp[q], dst, t.ld(q), 1, cs)) return e;
    ++*launches;
  }
  for (int tt = 0; tt < t.pc; ++tt) {
    const int q = t.r + tt * t.pr;
    if (!t.kp[q] || !t.ncols[t.c]) continue;
    double* dst = q == t.me ? (double*)(ws + t.off_bfull) + (size_t)t.coloff[t.c] * t.ld(q)
                            : (double*)(xp + t.offBpiece[tt]);
    ProfScope ps(ctx, cs, 2, 0.0, 16.0 * t.ncols[t.c] * t.kp[q] * bs);
    if (dbm_status e = densify_b(ctx, B, tt, t.pc, t.kp[q], dst, t.ld(q), 0, cs)) return e;
    ++*launches;
  }
  CUDA_TRY(ctx, cudaGetLastError());
  cudaEvent_t ev_ready = get_event(ctx);
  CUDA_TRY(ctx, cudaEventRecord(ev_ready, cs));
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm, ev_ready, 0));
  // "my pieces are ready" (behind the densifies) -> the gathers wait for every peer's (device-side)
  if (dbm_status e = xsignal(ctx, cs, X_READY, ep)) return e;
  if (dbm_status e = xwait(ctx, ctx->comm, X_READY, ep)) return e;
  std::vector<TSPlan> peer(P);
  for (int q = 0; q < P; ++q)
    if (q != t.me) peer[q] = make_ts_plan(t.pr, t.pc, q / t.pc, q % t.pc, t.Mb, t.Nb, t.Kb, bs);
  auto base_of = [&](int q) { return q == t.me ? xp : ctx->peer_ws[q]; };

  // ---- gather A[:, S_me] and B[S_me, :] in K-chunks on the comm stream, GEMM chunks on the compute stream
  const int64_t kb = t.kp[t.me], ldp = t.ld(t.me);
  // chunks keep 16-B TMA bases when bs is even
  int64_t remote_rows = 0;  // A rows and B columns this rank pulls from peers
  for (int rr = 0; rr < t.pr; ++rr)
    if (rr != t.r) remote_rows += t.mrows[rr];
  for (int cc = 0; cc < t.pc; ++cc)
    if ((t.me % t.pr) * t.pc + cc != t.me) remote_rows += t.ncols[cc];
  const double growth = pipeline_growth(2.0 * t.Mtot * t.Ntot * bs, (double)remote_rows * bs * 8);
  const std::vector<int64_t> cb = bs % 2 ? std::vector<int64_t>{0, kb} : pipeline_chunks(kb, growth);
  const int nsub = (int)cb.size() - 1;
  char* afull = ws + t.off_afull;
  char* bfull = ws + t.off_bfull;
  double* cpart = (double*)(xp + t.off_cpart);
  cudaEvent_t ev_c[kMaxChunks] = {};
  const int rb = t.me % t.pr;
  int64_t ts_recv = 0, ts_sent = 0;
  ts_bytes(t, &ts_recv, &ts_sent);
  ts_recv -= (int64_t)(t.P - 1) * t.mrows[t.r] * t.ncols[t.c] * 8;  // the C-share pulls run later, on cs
  ProfScope ps_x(ctx, ctx->comm, 5, 0.0, (double)ts_recv);  // the A / B gathers on the copy engines
  for (int j = 0; j < nsub && kb > 0; ++j) {
    const int64_t k0 = cb[j], k1 = cb[j + 1];
    const size_t off = (size_t)(k0 * bs) * 8, width = (size_t)((k1 - k0) * bs) * 8;
    for (int rr = 0; rr < t.pr; ++rr) {  // rows of grid row rr from rank (rr, c), its piece for target row r
      const int q = rr * t.pc + t.c;
      if (!t.mrows[rr] || q == t.me) continue;  // my own rows are already in place
      const char* src = ctx->peer_ws[q] + peer[q].offApiece[t.r];
      CUDA_TRY(ctx, cudaMemcpy2DAsync(afull + (size_t)t.rowoff[rr] * ldp * 8 + off, ldp * 8, src + off, ldp * 8, width,
                                      t.mrows[rr], cudaMemcpyDeviceToDevice, ctx->comm));
    }
    for (int cc = 0; cc < t.pc; ++cc) {  // columns of grid column cc from rank (rb, cc), its piece for target me
      const int q = rb * t.pc + cc;
      if (!t.ncols[cc] || q == t.me) continue;
      const int tt = (t.me - rb) / t.pr;
      const char* src = ctx->peer_ws[q] + peer[q].offBpiece[tt];
      CUDA_TRY(ctx, cudaMemcpy2DAsync(bfull + (size_t)t.coloff[cc] * ldp * 8 + off, ldp * 8, src + off, ldp * 8, width,
                                      t.ncols[cc], cudaMemcpyDeviceToDevice, ctx->comm));
    }
    ev_c[j] = get_event(ctx);
    CUDA_TRY(ctx, cudaEventRecord(ev_c[j], ctx->comm));
  }
  for (int j = 0; j < nsub; ++j) {
    const int64_t k0 = cb[j], k1 = cb[j + 1];
    if (kb > 0) CUDA_TRY(ctx, cudaStreamWaitEvent(cs, ev_c[j], 0));
    GemmArgs g{t.Mtot, t.Ntot, (k1 - k0) * bs, (const double*)afull + k0 * bs, ldp, (const double*)bfull + k0 * bs,
               ldp, cpart, t.Mtot, 1.0, j == 0 ? 0.0 : 1.0, 1, nullptr};
    g.splitk = std::min(pick_splitk(g.M, g.N, g.K, num_sms()), t.max_split);
    g.partial = g.splitk > 1 ? (double*)(ws + t.off_part) : nullptr;
    ProfScope ps(ctx, cs, 0, 2.0 * g.M * g.N * g.K, 8.0 * (g.M * g.K + g.N * g.K + g.M * g.N * (j ? 2 : 1)));
    CUDA_TRY(ctx, launch_dgemm(g, cs, launches));
    ++st->gemm_launches;
    if (kb == 0) break;
  }
  st->entries += 1;  // the densified batch holds one multiplication
  st->stacks += 1;
  st->flops += 2.0 * t.Mtot * t.Ntot * kb * bs;
  // ---- reduction: every partial is complete after this barrier; pull my C share out of each.  My gathers
  // are finished too (the last GEMM chunk waited for them): "done" goes out with "mid".
  if (dbm_status e = xsignal(ctx, cs, X_MID, ep)) return e;
  if (dbm_status e = xwait(ctx, cs, X_MID, ep)) return e;
  const int64_t mr = t.mrows[t.r], nc = t.ncols[t.c];
  double* cstack = (double*)(ws + t.off_cstack);
  for (int q = 0; q < P && mr * nc > 0; ++q) {
    const double* src = (const double*)(base_of(q) + (q == t.me ? t.off_cpart : peer[q].off_cpart)) + t.rowoff[t.r] +
                        (size_t)t.coloff[t.c] * t.Mtot;
    CUDA_TRY(ctx, cudaMemcpy2DAsync(cstack + (size_t)q * mr * nc, mr * 8, src, t.Mtot * 8, mr * 8, nc,
                                    cudaMemcpyDeviceToDevice, cs));
  }
  if (mr * nc > 0) {
    ProfScope ps(ctx, cs, 3, 0.0, (8.0 * P + (beta == 0.0 ? 8.0 : 16.0)) * mr * nc);
    undensify_c(C, cstack, mr, (int)P, mr * nc, alpha, beta, cs);
    ++*launches;
    CUDA_TRY(ctx, cudaGetLastError());
  }
  // closing barrier: no peer still reads my pieces or my partial
  if (dbm_status e = xsignal(ctx, cs, X_DONE, ep)) return e;
  if (dbm_status e = xwait(ctx, cs, X_DONE, ep)) return e;
  ts_bytes(t, &st->bytes_recv, &st->bytes_sent);
  st->steps = 1;
  ctx->ev_pool.push_back(ev_ready);
  for (int j = 0; j < kMaxChunks; ++j)
    if (ev_c[j]) ctx->ev_pool.push_back(ev_c[j]);
  return DBM_OK;
}

}  // namespace dbm

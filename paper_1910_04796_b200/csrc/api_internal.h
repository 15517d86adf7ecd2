// Shared internals of the libdbm host runtime (dbm_api.cu, multiply_tallskinny.cu, multiply_sparse.cu):
// error macros, stream/event helpers, the profiling bracket and the pieces of the multiply driver the
// algorithm files share.  Not part of the ABI.
#pragma once

#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "dbm_internal.h"

#define ARG_CHECK(cond, code, msg) \
  do {                             \
    if (!(cond)) {                 \
      set_error(msg);              \
      return code;                 \
    }                              \
  } while (0)

#define CUDA_TRY(ctx, x)                                                                    \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) {                                                                \
      set_error(std::string(#x) + ": " + cudaGetErrorString(e_));                           \
      if (ctx) (ctx)->poisoned = DBM_ERR_CUDA;                                              \
      return DBM_ERR_CUDA;                                                                  \
    }                                                                                       \
  } while (0)

#define NCCL_TRY(ctx, x)                                                                    \
  do {                                                                                      \
    ncclResult_t r_ = (x);                                                                  \
    if (r_ != ncclSuccess) {                                                                \
      set_error(std::string(#x) + ": " + ncclGetErrorString(r_));                           \
      if (ctx) (ctx)->poisoned = DBM_ERR_NCCL;                                              \
      return DBM_ERR_NCCL;                                                                  \
    }                                                                                       \
  } while (0)

#define CTX_OK(ctx)                                                             \
  do {                                                                          \
    ARG_CHECK((ctx) != nullptr, DBM_ERR_ARG, "null context");                   \
    if ((ctx)->poisoned != DBM_OK) {                                            \
      set_error("context poisoned by an earlier CUDA/NCCL failure");            \
      return (ctx)->poisoned;                                                   \
    }                                                                           \
    CUDA_TRY(ctx, cudaSetDevice((ctx)->device));                                \
  } while (0)

namespace dbm {

inline int64_t local_count(int64_t nb, int p, int r) { return nb > r ? (nb - r + p - 1) / p : 0; }
inline int64_t lcm64(int64_t a, int64_t b) { return a / std::gcd(a, b) * b; }
inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

constexpr int kMaxChunks = 16;                       // pipeline_chunks() returns <= 15 chunks
constexpr int64_t kDefaultChunkBytes = 16ll << 30;   // A+B dense chunk budget (single rank)
// Triplets per stack-generation chunk (<= 6.4 GB): large enough that one smm launch has thousands
// of 8-run groups for 148 SMs even with the 90,112-long runs of the rectangular bs-22 config.
constexpr int64_t kTripChunkEntries = 1ll << 29;

cudaEvent_t get_event(dbm_ctx ctx);  // from the context's pool (timing disabled)

// Profiling bracket around one launch or transfer (timing events live on its stream).  kind: 0 dense
// GEMM, 1 small-block GEMM, 2 densify, 3 undensify, 4 stack generation, 5 exchange pulls.
struct ProfScope {
  dbm_ctx ctx;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  int kind;
  double flops, bytes;
  ProfScope(dbm_ctx c, cudaStream_t s, int k, double f, double by) : ctx(c), st(s), kind(k), flops(f), bytes(by) {
    if (!ctx->profiling) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, st);
    ctx->prof.push_back({a, b, kind, flops, bytes});
  }
};

std::vector<int64_t> pipeline_chunks(int64_t kb, double growth = 2.0);
// Local-first step order (copy-engine transport, several ranks).  With owner-pull every panel sits in
// its owner's exchange pool before any step, so a rank may take Cannon's L steps in any order (reading
// R5; the canonical skew kappa = (r + c + s) mod L stays the schedule dbm_plan_exchange describes and the
// NCCL transport runs).  Each rank starts at the canonical step with the most local operands -- the
// first step is the one nothing overlaps with -- ties broken towards the owners serving the fewest first-
// step pulls (greedy over the ranks in order, so every rank computes every rank's choice), and then
// continues cyclically.  2 x 2: ranks 0 and 3 start with both operands local, ranks 1 and 2 with one
// pull each from different owners (canonical: rank 3 pulls both, and serves both of the others' pulls).
// Returns rank's first canonical step.
int local_first_start(int pr, int pc, int rank);
double pipeline_growth(double gemm_flop_per_kblock, double pull_bytes_per_kblock);

dbm_status validate(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C);
dbm_status densify_a(dbm_ctx ctx, dbm_matrix A, int64_t col0, int64_t stride, int64_t nk, double* dst, int64_t ld,
                     int layout, cudaStream_t cs);
dbm_status densify_b(dbm_ctx ctx, dbm_matrix B, int64_t row0, int64_t stride, int64_t nk, double* dst, int64_t ld,
                     int layout, cudaStream_t cs);
void undensify_c(dbm_matrix C, const double* dense, int64_t ld, int nsplit, int64_t split_stride, double alpha,
                 double beta, cudaStream_t cs);
void launch_scale(double* x, int64_t n, double beta, cudaStream_t st);  // x = beta * x (beta 0: zeros)
// All-gather of the workspaces' CUDA IPC handles (maps the peers' workspaces).  Synchronises the comm
// stream: it runs only when a rank registers a new workspace (xattach / dbm_ctx_set_workspace).
dbm_status ipc_exchange(dbm_ctx ctx, void* ws);

// ---- device-side signals between ranks (copy-engine transport)
// Every rank's exchange pool starts with a header of int64 words its peers write into through
// the IPC mappings: word (kind * P + q) holds the last epoch for which peer q announced `kind`, then the
// host pipeline's progress table [peer][operand][kappa] = (epoch << 32) | K-blocks in place.  Values
// only grow (epochs count the copy-engine multiplies, identical on every rank), so no table is ever
// reset between multiplies; registration zeroes the header once, ordered before any peer write by the
// registration all-gather.  Waits are cuStreamWaitValue64 (GEQ) on a stream, writes
// cuStreamWriteValue64: no SM spins and no host round trip.
enum XKind { X_READY = 0, X_MID = 1, X_DONE = 2, X_KINDS = 3 };
size_t xhdr_bytes(int nranks, int L);           // header bytes at the start of the workspace (0: one rank)
inline size_t xprog_word(int P, int L, int peer, int operand, int kappa) {
  return (size_t)X_KINDS * P + ((size_t)peer * 2 + operand) * L + kappa;
}
// Make the context's exchange pool (library-owned: signal header + the own panels / pieces peers pull)
// hold at least `need` bytes, `need` being the maximum over all ranks.  Growing is collective by
// construction (every rank sees the same need): a new cudaMalloc allocation, its header zeroed, the
// IPC handles all-gathered (the only host synchronisation, once per growth).  Otherwise: nothing.
dbm_status xattach(dbm_ctx ctx, size_t need, cudaStream_t cs);
// Write `value` into word (kind, me) of every peer's header / wait on stream st until word (kind, q) of
// my header holds >= value for every peer q.
dbm_status xsignal(dbm_ctx ctx, cudaStream_t st, int kind, uint64_t value);
dbm_status xwait(dbm_ctx ctx, cudaStream_t st, int kind, uint64_t value);
// Single words: write my progress into peer q's table / wait for peer q's progress in mine.
dbm_status xwrite_word(dbm_ctx ctx, cudaStream_t st, int q, size_t word, uint64_t value);
dbm_status xwait_word(dbm_ctx ctx, cudaStream_t st, size_t word, uint64_t value);

// ---- tall-and-skinny (multiply_tallskinny.cu, reading R14)
size_t ts_workspace_bytes(int pr, int pc, int r, int c, int64_t Mb, int64_t Nb, int64_t Kb, int64_t bs);
void ts_plan_bytes(int pr, int pc, int r, int c, int64_t Mb, int64_t Nb, int64_t Kb, int64_t bs, int64_t* recv,
                   int64_t* sent);
dbm_status multiply_tallskinny(dbm_ctx ctx, double alpha, dbm_matrix A, dbm_matrix B, double beta, dbm_matrix C,
                               char* ws, dbm_stats* st, int* launches);

// ---- block sparsity (multiply_sparse.cu, reading R15)
dbm_path resolve_path(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_path path);  // DBM_PATH_AUTO
dbm_status sp_workspace_bytes(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, int64_t* bytes);
dbm_status multiply_sparse_blocked(dbm_ctx ctx, double alpha, dbm_matrix A, dbm_matrix B, double beta, dbm_matrix C,
                                   int32_t stack_cap, void* workspace, int64_t ws_bytes, dbm_stats* stats);
dbm_status sp_debug_stacks(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, int step, int32_t cap,
                           int32_t* triplets, int64_t* n_entries, int64_t* stack_ptr, int64_t* n_stacks);
void free_sp_cache(dbm_ctx ctx);

// ---- non-uniform block sizes (multiply_nonuniform.cu, reading R16)
dbm_status nu_workspace_bytes(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, bool dens, int64_t* bytes);
dbm_status multiply_nonuniform(dbm_ctx ctx, double alpha, dbm_matrix A, dbm_matrix B, double beta, dbm_matrix C,
                               bool dens, void* workspace, int64_t ws_bytes, dbm_stats* stats);
void free_nu_cache(dbm_ctx ctx);
dbm_status nu_tables(dbm_matrix m);  // per-slot offset / shape tables for a uniform matrix (R16 multiplies)

}  // namespace dbm

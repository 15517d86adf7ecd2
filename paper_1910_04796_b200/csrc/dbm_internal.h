// Internal declarations of libdbm (B200 / sm_100a).  Not part of the ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "dbm.h"

namespace dbm {

// ----------------------------------------------------------------- errors
void set_error(const std::string& msg);

// ----------------------------------------------------------------- kernels
// Counter-based generator, device implementation.
void launch_fill(double* arena, int64_t mloc, int64_t nloc, int bs, int pr, int pc, int r, int c, uint64_t seed,
                 uint32_t mat_id, int kind, cudaStream_t st);

// Densify a set of block columns of a local arena (A panels): blocks (li, kcol0 + q*kstride),
// q < nk, li < mloc, from an arena with nloc block columns.  layout 1 = row-major (K-major, the
// GEMM's A operand): dense[(li*bs+x)*ld + q*bs+y]; layout 0 = column-major: dense[(q*bs+y)*ld + li*bs+x].
void launch_densify_cols(const double* arena, int64_t mloc, int64_t nloc, int bs, int64_t kcol0, int64_t kstride,
                         int64_t nk, double* dense, int64_t ld, int layout, cudaStream_t st);
// Densify a set of block rows (B panels): blocks (krow0 + q*kstride, lj).  layout 0 = column-major
// (K-major for B, the GEMM's B operand): dense[(lj*bs+y)*ld + q*bs+x]; layout 1 = row-major.
void launch_densify_rows(const double* arena, int64_t nloc, int bs, int64_t krow0, int64_t kstride, int64_t nk,
                         double* dense, int64_t ld, int layout, cudaStream_t st);
// Undensify with alpha/beta: block(li,lj)(x,y) = alpha*D + beta*block.
// If nsplit > 1, D is the sum over s of dense + s*split_stride (fixed order s = 0..nsplit-1).
void launch_undensify(const double* dense, int64_t ld, int nsplit, int64_t split_stride, int64_t mloc, int64_t nloc,
                      int bs, double alpha, double beta, double* arena, cudaStream_t st);
// Pack a panel of whole blocks: out slot q*ncols + j <- arena slot (row0 + q*rstride)*ncols + j.
void launch_pack_rows(const double* arena, int64_t ncols, int bs, int64_t row0, int64_t rstride, int64_t nrows,
                      double* out, cudaStream_t st);
void launch_pack_cols(const double* arena, int64_t mloc, int64_t nloc, int bs, int64_t col0, int64_t cstride,
                      int64_t ncols, double* out, cudaStream_t st,
                      int64_t out_pitch = 0);

// ---- block-sparse matrices (kernels_sparse.cu, reading R15) ----
void launch_fill_sparse(double* arena, int64_t nnz, const int32_t* ij, int bs, int pr, int pc, int r, int c,
                        uint64_t seed, uint32_t mat_id, int kind, cudaStream_t st);
// Densify the stored blocks of one panel; absent blocks become zeros.  axis 0 (A panel): blocks with
// lj = sel0 + q*stride, q < nk -> dense block (li, q), `other` = mloc; axis 1 (B panel): blocks with
// li = sel0 + q*stride -> dense block (q, lj), `other` = nloc.  Layouts as launch_densify_cols/rows.
cudaError_t launch_sp_densify(const double* arena, const int32_t* ij, int64_t nnz, int bs, int axis, int64_t sel0,
                              int64_t stride, int64_t nk, int64_t other, double* dense, int64_t ld, int layout,
                              cudaStream_t st);
void launch_sp_undensify(const double* dense, int64_t ld, int nsplit, int64_t split_stride, const int32_t* ij,
                         int64_t nnz, int bs, double alpha, double beta, double* arena, cudaStream_t st);
// out block q <- arena block src[q] (panel packing)
void launch_sp_gather(const double* arena, const int32_t* src, int64_t n, int bs, double* out, cudaStream_t st);
size_t sp_scan_temp_bytes(int64_t n);
// Sparse Generation for runs q0 .. q0+n-1 of the traversal: cnt (n+1) and off (n+1) are scratch /
// the run offsets (off[n] = entries), trip receives the triplets.
cudaError_t launch_sp_stackgen(const int32_t* a_ptr, const int32_t* a_kk, const int32_t* b_ptr, const int32_t* b_kk,
                               const int32_t* b_slot, const int32_t* cmap, int64_t nloc, const int32_t* li,
                               const int32_t* lj, int64_t q0, int64_t n, int64_t* cnt, int64_t* off, void* scan_tmp,
                               size_t scan_bytes, int32_t* trip, cudaStream_t st);
// C_blk(trip c) += alpha * sum over a run's entries of A_blk * B_blk; runs given by off (nruns+1).
cudaError_t launch_smm_sparse(int bs, const int32_t* trip, const int64_t* off, int64_t nruns, const double* A,
                              const double* B, double* C, double alpha, cudaStream_t st);

// Dense FP64 GEMM, both operands K-major (the "TN" form): C(M x N col-major) = alpha * At^T B + beta C.
struct GemmArgs {
  int64_t M, N, K;
  const double* A;  // element (m,k) at A[m*lda + k]
  int64_t lda;
  const double* B;  // element (k,n) at B[n*ldb + k]
  int64_t ldb;
  double* C;  // element (m,n) at C[m + n*ldc]
  int64_t ldc;
  double alpha, beta;
  int splitk;        // >= 1
  double* partial;   // splitk*M*N doubles when splitk > 1
  // b_blocks: B is not a dense K-major matrix but a panel of 64 x 64 column-major blocks, block (kk, lj)
  // at slot kk * ceil(N/64) + lj (a bs-64 arena / packed panel, read in place: no densify); ldb unused
  int b_blocks = 0;
  // a_blocks: A is a panel of 64 x 64 column-major blocks, block (li, kk) at slot li * a_blk_ld + kk (a bs-64
  // arena or packed panel, read in place through a 4-D TMA view: no densify; §8f-3 zero-copy A); lda unused
  int a_blocks = 0;
  int64_t a_blk_ld = 0;
};
// Returns cudaSuccess or an error (tensor-map encode failures map to cudaErrorInvalidValue).
cudaError_t launch_dgemm(const GemmArgs& g, cudaStream_t st, int* launches);
int pick_splitk(int64_t M, int64_t N, int64_t K, int num_sms);
// 2-D FP64 tensor map (TMA), 128-B swizzle: `rows` rows of `inner` doubles, row stride in bytes.
bool make_map_2d(CUtensorMap* tm, const double* base, uint64_t inner, uint64_t rows, uint64_t row_stride_bytes,
                 uint32_t box_inner, uint32_t box_rows);
void launch_splitk_reduce(const double* partial, int splitk, int64_t M, int64_t N, double* C, int64_t ldc,
                          double alpha, double beta, cudaStream_t st);

// Blocked path: stack generation and the batched small-block GEMM.
// Traversal order table: run q -> (li, lj) (recursive bisection, reading R6), computed on device.
void launch_traversal(int64_t mloc, int64_t nloc, int32_t* li_out, int32_t* lj_out, cudaStream_t st);
// Stack entries for runs [q0, q1): triplets (a,b,c) int32 with a = li*kb+kk, b = kk*nb_ld+lj, c = li*nloc+lj.
void launch_stackgen(const int32_t* li, const int32_t* lj, int64_t q0, int64_t q1, int64_t kb, int64_t nloc,
                     int64_t a_ld, int64_t b_ld, int32_t* trip, cudaStream_t st);
void launch_stack_ptr(int64_t nruns, int64_t kb, int64_t cap, int64_t nstacks, int64_t* ptr, cudaStream_t st);
// Execute stack entries [e0, e1) (whole C-block runs of length kb, consecutive): for each run,
// C_blk = (first ? beta*C_blk : C_blk) + alpha*sum_k A_blk*B_blk.
// nsplit > 1 splits each run's K across CTAs (partial: nsplit*nruns*bs*bs doubles, reduced in a
// fixed order); see smm_pick_split.
// a_blocks / b_blocks: blocks in the A / B panels (tensor-map extents of the bs-64 kernel).
// squares: the caller guarantees every 16 consecutive runs form a 4 x 4 square of C blocks with equal
// K lists (bisection_squares() of a dense local grid): bs 22 then runs the unpadded 88 x 88 kernel.
cudaError_t launch_smm(int bs, const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const double* B,
                       double* C, double alpha, double beta_first, int nsplit, double* partial, cudaStream_t st,
                       int* launches, int64_t a_blocks = 0, int64_t b_blocks = 0, bool squares = false);
int smm_pick_split(int bs, int64_t nruns, int64_t kb, bool squares = false);
// bs 22 on grids the bisection does not visit as whole squares: per chunk of runs [q0, q0+nruns), the
// aligned 4 x 4 squares whose 16 runs are all in the chunk run on the unpadded kernel, the other runs on
// the 8-run kernel (lists built on the GPU).  pos = inverse traversal (launch_inverse_traversal).
struct SmmMixedWS {
  uint8_t* sqflag;    // mloc/4 * nloc/4
  int32_t* sq_ids;    // mloc/4 * nloc/4
  int32_t* runs_sq;   // chunk runs
  int32_t* runs_left; // chunk runs
  uint8_t* runflag;   // chunk runs
  int* counts;        // 4 ints
  void* temp;
  size_t temp_bytes;
};
void launch_inverse_traversal(const int32_t* li, const int32_t* lj, int64_t n, int64_t nloc, int32_t* pos,
                              cudaStream_t st);
size_t smm22_mixed_temp_bytes(int64_t n);
cudaError_t launch_smm22_mixed(const int32_t* trip, int64_t q0, int64_t nruns, int64_t kb, const double* A,
                               const double* B, double* C, double alpha, double beta_first, const int32_t* li,
                               const int32_t* lj, const int32_t* pos, int64_t mloc, int64_t nloc, const SmmMixedWS& w,
                               cudaStream_t st, int* launches);
// True when the bisection traversal of an mloc x nloc grid (reading R6) visits it as whole 4 x 4 squares
// of 16 consecutive runs (both sides keep halving evenly down to 4).
bool bisection_squares(int64_t mloc, int64_t nloc, int64_t side = 4);
// smmq (kernels_smmq.cu): R x R run squares for the padded small sizes (bs 4, 5, 6, 9); R (0: none)
int smmq_side(int bs);
cudaError_t launch_smmq(int bs, const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const double* B,
                        double* C, double alpha, double beta_first, cudaStream_t st);
// DMMA group kernel for bs 22 / 64 (kernels_smm.cu); the generic smm handles other block sizes.
bool smm_has_tensor_path(int bs);
// DMMA per-run kernel for other compiled block sizes (kernels_sparse.cu); off == nullptr: uniform runs of kb
bool smm_has_run_path(int bs);
cudaError_t launch_smm_run(int bs, const int32_t* trip, const int64_t* off, int64_t nruns, int64_t kb,
                           const double* A, const double* B, double* C, double alpha, double beta_first,
                           cudaStream_t st);
int smm_group_runs(int bs);  // runs per CTA group (stack chunks are cut at multiples of it)
cudaError_t launch_smm_tc(int bs, const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const double* B,
                          double* C, double alpha, double beta_first, int nsplit, double* partial, cudaStream_t st,
                          int64_t a_blocks, int64_t b_blocks, bool squares);

// ----------------------------------------------------------------- driver
int num_sms();

struct SpCache;  // block-sparse multiply plans + device metadata (dbm_api.cu)

// ---- non-uniform block sizes (kernels_nonuniform.cu, multiply_nonuniform.cu; reading R16) ----
struct NUBlk {  // one stored local block: arena element offset, global element row / column, shape
  int64_t off, r0, c0;
  int32_t rows, cols;
};
struct NUTask {  // block <-> dense copy: block at arena element src, dense position (row0, col0)
  int64_t src, row0, col0;
  int32_t rows, cols;
};
struct NUPack {  // whole-block gather: n elements from src to dst (element offsets)
  int64_t src, dst, n;
};
void launch_nu_fill(double* arena, const NUBlk* blk, int64_t nslots, uint64_t seed, uint32_t mat_id, int kind,
                    cudaStream_t st);
// mode 0: A block -> K-major rows dense[(row0+x)*ld + col0+y]; mode 1: B block -> K-major columns
// dense[(col0+y)*ld + row0+x]; mode 2: C block = alpha*dense[(col0+y)*ld + row0+x] + beta*C block
void launch_nu_copy(const NUTask* tasks, int64_t ntasks, double* arena, double* dense, int64_t ld, int mode,
                    double alpha, double beta, cudaStream_t st);
void launch_nu_pack(const NUPack* tasks, int64_t ntasks, const double* src, double* dst, cudaStream_t st);
// Entries grouped per stage: kdim[e] = k size of the run's entry e, kofs[e] = its k offset inside its group,
// groups g = entries [gbeg[g], gbeg[g+1]) (host-computed; every run of a step has the same k sizes)
// Entry groups of the non-uniform small-block kernel hold at most this many entries (its 4 warps load a
// group's entry metadata one entry per lane; each entry reserves 4 doubles of alignment room per operand
// in a stage, so the bound keeps 4 CTAs' rings of 32 x 32 blocks within an SM's shared memory).
constexpr int kNuGroupMaxEntries = 16;
size_t nu_smm_smem(int kcap, int mmax, int nmax);
cudaError_t launch_nu_smm(const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const int64_t* aoff,
                          const double* B, const int64_t* boff, const int32_t* kdim, const int32_t* kofs,
                          const int32_t* gbeg, int ngroups, double* C, const NUBlk* cblk, int kcap, int mmax, int nmax,
                          double alpha, double beta_first, cudaStream_t st);
struct NUCache;  // non-uniform multiply plans + device tables (multiply_nonuniform.cu)
}  // namespace dbm

// ----------------------------------------------------------------- handles
struct dbm_ctx_s {
  int nranks = 1, rank = 0, pr = 1, pc = 1, myrow = 0, mycol = 0, device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t comm = nullptr;
  cudaStream_t comm2 = nullptr;  // second pull stream: a step's B panel beside its A panel (two copy engines)
  cudaStream_t up = nullptr;  // host->device uploads of dbm_multiply_host on several ranks (lazy)
  cudaStream_t gen = nullptr; // stack generation of the next chunk beside the small-block GEMM (lazy)
  cudaStream_t own = nullptr; // host pipeline: own-panel densify / pack + progress signals (lazy)
  bool host_pipe = true;      // several ranks, host operands: chunked uploads gated by peer flags
  bool dev_pipe = false;      // several ranks, device operands: own panels chunked, pulls gated by progress
  void* nccl = nullptr;  // ncclComm_t
  dbm_status poisoned = DBM_OK;
  int64_t launches = 0;
  int64_t chunk_bytes = 16ll << 30;  // densified single-rank K-chunk budget (dense A + B)
  bool profiling = false;
  struct ProfRec {
    cudaEvent_t a, b;
    int kind;
    double flops, bytes;
  };
  std::vector<ProfRec> prof;
  // the last profiled multiply (dbm_multiply_timing): bracket events on the ctx stream, record range
  cudaEvent_t lt_a = nullptr, lt_b = nullptr;
  size_t lt_first = 0, lt_last = 0;
  bool lt_valid = false;
  std::vector<cudaEvent_t> ev_pool;  // free events
  // pinned staging ring for pageable host copies
  void* stage[2] = {nullptr, nullptr};
  size_t stage_bytes = 0;
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  // Cannon transport: 0 = copy engines pulling peer panels through CUDA IPC mappings (default),
  // 1 = NCCL grouped send/recv.
  int transport = 0;
  int algorithm = 0;  // 0 = Cannon, 1 = tall-and-skinny
  void* ipc_ws = nullptr;                 // the allocation the peer mappings were built for (= xpool)
  int64_t ipc_ws_bytes = 0;
  char* xpool = nullptr;                  // exchange pool (several ranks): signal header + own panels
  size_t xpool_bytes = 0;
  uint64_t epoch = 0;                     // copy-engine multiplies so far (the same count on every rank)
  std::vector<char*> peer_ws;             // peer workspaces mapped into this process (nullptr = self)
  std::vector<std::vector<char>> peer_handles;  // raw IPC handles (to re-use / close mappings)
  std::vector<void*> peer_bases;          // opened allocation bases (cudaIpcCloseMemHandle)
  int* d_scratch = nullptr;               // device scratch: barrier word + handle exchange
  double densify_threshold = 1.0;         // DBM_PATH_AUTO: densify iff occupancy >= this
  std::vector<dbm::SpCache*> sp_cache;    // sparse plans keyed by the operands' pattern serials
  std::vector<dbm::NUCache*> nu_cache;    // non-uniform plans keyed by the operands' serials
};

struct dbm_matrix_s {
  dbm_ctx ctx = nullptr;
  int64_t rows = 0, cols = 0;
  int bs = 0;
  int64_t Mb = 0, Nb = 0, mloc = 0, nloc = 0;
  double* arena = nullptr;
  int64_t arena_bytes = 0;
  // block sparsity (reading R15): stored blocks in local CSR order; the dense matrix is the
  // all-stored case (slot li*nloc + lj) and keeps sparse == false
  bool sparse = false;
  int64_t nnz = 0;                // stored local blocks
  int64_t gnnz = 0;               // stored blocks of the whole matrix
  std::vector<uint8_t> gmask;     // global pattern, Mb x Nb row-major (sparse only)
  std::vector<int64_t> row_ptr;   // local CSR over li (sparse only)
  std::vector<int32_t> col;       // lj per slot (sparse only)
  int32_t* d_ij = nullptr;        // device (li, lj) per slot (sparse only; library-owned)
  int32_t* d_map = nullptr;       // device li*nloc + lj -> slot or -1 (sparse only; library-owned)
  uint64_t serial = 0;            // pattern identity (plan caches)
  int device = 0;                 // CUDA device of the metadata (sparse only)
  // non-uniform block sizes (reading R16): global sizes, prefix offsets, per-slot element offsets
  bool nonuni = false;
  std::vector<int32_t> rsz, csz;      // block row / column sizes (Mb / Nb entries)
  std::vector<int64_t> roff, coff;    // prefix sums (Mb + 1 / Nb + 1 entries)
  std::vector<int64_t> slot_off;      // element offset of every stored local slot (blocks() + 1 entries)
  std::vector<dbm::NUBlk> hblk;       // host copy of the per-slot table
  dbm::NUBlk* d_blk = nullptr;        // device per-slot table (library-owned)
  int64_t blocks() const { return sparse ? nnz : mloc * nloc; }
  int64_t elems() const { return nonuni ? slot_off.back() : blocks() * (int64_t)bs * bs; }
  int32_t row_size(int64_t bi) const { return nonuni ? rsz[bi] : bs; }
  int32_t col_size(int64_t bj) const { return nonuni ? csz[bj] : bs; }
  bool stored(int64_t bi, int64_t bj) const { return !sparse || gmask[(size_t)bi * Nb + bj]; }
};

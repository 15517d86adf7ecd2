/*
 * dbm.h — C ABI of the B200-native DBCSR dense-multiply hot path (arXiv 1910.04796).
 *
 * The library (paper_1910_04796_b200/libdbm.so) multiplies FP64 matrices of uniform
 * square blocks, distributed block-cyclically over a 2-D grid of ranks (one rank per
 * GPU), with Cannon's algorithm and either a blocked (stacks + batched small-block
 * GEMM) or a densified (densify -> one large GEMM -> undensify) local multiply.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n; readings R1..R15 are
 * listed in DESIGN.md §3.
 *
 * General conventions
 *  - Every function returns dbm_status; DBM_OK == 0.  On error, dbm_last_error()
 *    returns a thread-local human-readable detail string.
 *  - Device memory (matrix arenas, multiply workspace, dense buffers) is CALLER-OWNED
 *    (e.g. torch tensors).  The library never frees it.  Handles belong to the
 *    library until the matching *_destroy.  Library-owned device memory: small metadata
 *    tables (block-sparse / non-uniform matrices, plans) and, on several ranks, the
 *    exchange pool of dbm_ctx_set_transport (freed by dbm_ctx_destroy).
 *  - Calls that launch GPU work enqueue on the context's stream and return without
 *    synchronising, unless documented otherwise.  Asynchronous CUDA / NCCL failures
 *    surface at dbm_ctx_sync(), after which the context is poisoned: every later
 *    call returns DBM_ERR_CUDA or DBM_ERR_NCCL.
 *  - Arguments are validated on the host BEFORE anything is enqueued; on a
 *    validation error nothing is modified.
 *  - Matrix storage ("arena", reading R3): the local share of a rows x cols matrix
 *    with block size bs is mloc x nloc blocks, mloc = #{i < rows/bs : i mod Pr == myrow},
 *    nloc = #{j < cols/bs : j mod Pc == mycol}; block (li,lj) holds global block
 *    (myrow + li*Pr, mycol + lj*Pc) ("block-cycling distributed a la ScaLAPACK";
 *    S:115), at slot li*nloc + lj; element (x,y) at slot*bs*bs + y*bs + x
 *    (column-major inside a block; DBCSR is Fortran).  The metadata is a
 *    blocked CSR (§II) with every block present (dense occupancy).
 *  - Block-sparse matrices (dbm_matrix_create_sparse; reading R15, "occupancy between
 *    0.01% up to dense"): only the stored blocks occupy the arena, in local CSR order (li
 *    ascending, then lj ascending); slot = position in that order.  The dense layout above is
 *    the all-stored special case.
 */
#ifndef DBM_H
#define DBM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DBM_OK = 0,
  DBM_ERR_ARG = 1,       /* null handle / pointer, bad enum, bad size */
  DBM_ERR_SHAPE = 2,     /* non-conformant shapes; rows/cols not a multiple of bs */
  DBM_ERR_RANGE = 3,     /* block index out of range */
  DBM_ERR_PARTITION = 4, /* A's K partition differs from B's (unequal block sizes) */
  DBM_ERR_PLAN = 5,      /* densify plan mismatch */
  DBM_ERR_OWNERSHIP = 6, /* block not owned by the calling rank */
  DBM_ERR_ALIAS = 7,     /* C aliases A or B */
  DBM_ERR_GRID = 8,      /* Pr*Pc != nranks, or matrices from different contexts */
  DBM_ERR_WORKSPACE = 9, /* workspace smaller than dbm_multiply_workspace() / arena not attached */
  DBM_ERR_CUDA = 20,
  DBM_ERR_NCCL = 21,
  DBM_ERR_NOMEM = 22
} dbm_status;

/* DBM_PATH_AUTO: densified iff both A's and B's occupancy (stored / all blocks) is >= the
 * context's densify threshold (dbm_ctx_set_densify_threshold; default 1.0 = dense only). */
typedef enum { DBM_PATH_BLOCKED = 0, DBM_PATH_DENSIFIED = 1, DBM_PATH_AUTO = 2 } dbm_path;

typedef struct dbm_ctx_s* dbm_ctx;
typedef struct dbm_matrix_s* dbm_matrix;

/* Per-multiply statistics (all counts for the calling rank). */
typedef struct {
  int64_t entries;    /* block multiplications (stack entries) executed; densified: 1 per GEMM */
  int64_t stacks;     /* stacks of <= stack_cap entries generated */
  int64_t bytes_sent; /* Cannon panel bytes sent by this rank */
  int64_t bytes_recv; /* Cannon panel bytes received by this rank */
  int64_t steps;      /* Cannon steps L = lcm(Pr,Pc) (reading R5) */
  int64_t gemm_launches;
  int64_t kernel_launches; /* all kernels this call launched */
  double flops;            /* 2*mloc*bs*nloc*bs*K_local + epilogue, this rank */
  /* Device times (ms) of the call, filled by dbm_multiply_timing (the call returns before its work
   * runs, so dbm_multiply leaves them 0): whole call on the ctx stream, densify / pack kernels, the
   * local multiply (GEMMs, small-block kernels, stack generation), undensify, and the exposed remainder
   * (ms_total minus the three phases: exchange waits, barriers and gaps not hidden under the rank's
   * kernels; clamped at 0).  SURVEY §8(b) timing fields; "only the execution time of the
   * multiplication part". */
  double ms_total, ms_densify, ms_local, ms_comm_exposed, ms_undensify;
} dbm_stats;

const char* dbm_status_string(dbm_status s);
const char* dbm_last_error(void);

/* ----------------------------------------------------------------- context */
/* Bytes of an NCCL unique id (NCCL_UNIQUE_ID_BYTES). */
int dbm_unique_id_bytes(void);
/* Rank 0 calls this, then broadcasts the bytes to every rank (e.g. torch.distributed). */
dbm_status dbm_get_unique_id(void* id_out);

/* Create the per-rank context (§II: a 2-D grid of P processes; one rank per GPU,
 * P:175).  pr = pc = 0 picks the grid by reading R1 (1->1x1, 2->1x2, 4->2x2, 8->2x4);
 * otherwise pr*pc must equal nranks (DBM_ERR_GRID).  rank = myrow*pc + mycol.
 * id: NCCL unique id bytes (ignored when nranks == 1).  device: CUDA ordinal.
 * cuda_stream: cudaStream_t to enqueue on (NULL = the legacy default stream, e.g. torch's default
 * stream); the library adds one internal non-blocking stream for the Cannon exchange.
 * Collective over all ranks when nranks > 1 (ncclCommInitRank). */
dbm_status dbm_ctx_create(int nranks, int rank, int pr, int pc, const void* id, int device, void* cuda_stream,
                          dbm_ctx* out);
dbm_status dbm_ctx_grid(dbm_ctx ctx, int* pr, int* pc, int* myrow, int* mycol);
/* Switch the stream subsequent calls enqueue on (e.g. torch.cuda.current_stream()). */
dbm_status dbm_ctx_set_stream(dbm_ctx ctx, void* cuda_stream);
/* Block until all work enqueued by this context finished; surfaces async errors. */
dbm_status dbm_ctx_sync(dbm_ctx ctx);
/* Profiling: when on, every dominant-kernel launch (the FP64 GEMM / small-block GEMM)
 * is bracketed by CUDA events on its own stream.  dbm_ctx_profile_read() synchronises,
 * returns the summed device time, launch count and algorithmic flops of the recorded
 * launches of `kernel` (0 = dense GEMM, 1 = small-block GEMM, 2 = densify, 3 = undensify,
 * 4 = stack generation, 5 = the copy-engine panel pulls of one exchange step, timed on the comm
 * stream) and clears the records. bytes_out: algorithmic bytes (kernel 5: bytes received). */
dbm_status dbm_ctx_set_profiling(dbm_ctx ctx, int on);
/* Timing of the last dbm_multiply / dbm_multiply_host this ctx ran with profiling on: synchronises on
 * it and fills st->ms_* (the other fields are left untouched).  Call before dbm_ctx_profile_read
 * consumes that multiply's records.  DBM_ERR_ARG if no profiled multiply is pending. */
dbm_status dbm_multiply_timing(dbm_ctx ctx, dbm_stats* st);
dbm_status dbm_ctx_profile_read(dbm_ctx ctx, int kernel, double* ms_out, int64_t* launches_out, double* flops_out,
                                double* bytes_out);
/* Timeline of the pending profiling records (not consumed): for record i (enqueue order, at most
 * max_records) out[3i] = kind (as dbm_ctx_profile_read), out[3i+1] / out[3i+2] = start / end in ms
 * relative to the first record's start (CUDA events, so records on the compute, comm and upload
 * streams share one clock: the overlap of the Cannon pulls with the GEMMs is read off directly).
 * *n_out = number of pending records.  Synchronises on the records. */
dbm_status dbm_ctx_profile_timeline(dbm_ctx ctx, int max_records, double* out, int* n_out);
/* Cannon panel transport between ranks ("asynchronous point-to-point"):
 * 0 (default) = DMA copy engines pull each needed panel over NVLink from its owner's exchange pool (no
 *     SM is taken from the local multiply).  The pool is library-owned (a plain cudaMalloc allocation,
 *     freed by dbm_ctx_destroy): a header of 64-bit signal words and the rank's own panels.  It is
 *     mapped into every peer with CUDA IPC when it grows (an all-gather of the handles with a host
 *     synchronisation; every rank sizes it by the maximum over all ranks' plans, so every rank grows
 *     it in the same multiply); otherwise a multiply orders ranks device-side only: per-panel progress
 *     and "done" epochs written into the peers' headers (cuStreamWriteValue64) and awaited on the
 *     streams (cuStreamWaitValue64), no host synchronisation.  Ranks take Cannon's steps in a
 *     local-first order (dbm_debug_first_step).
 * 1 = NCCL grouped ncclSend / ncclRecv.
 * Every rank must use the same transport.  Changes dbm_multiply_workspace() for the blocked path. */
dbm_status dbm_ctx_set_transport(dbm_ctx ctx, int transport);
/* MPI-level algorithm (§II): 0 (default) = Cannon (any shape, O(1/sqrt(P)) volume);
 * 1 = tall-and-skinny (one large dimension; reading R14): rank p = r*Pc + c computes the
 * partial product over the K blocks {k : k mod P == p} after gathering A[:, S_p] from its grid
 * column and B[S_p, :] from grid row p mod Pr, then every rank sums its C blocks out of all P partials
 * in rank order.  Requires the densified path and the copy-engine transport (DBM_ERR_ARG otherwise).
 * 2 = automatic: tall-and-skinny when K >= 16 max(M, N) on several ranks with the densified path and
 * the copy-engine transport ("one large dimension"), Cannon otherwise.
 * Every rank must use the same algorithm.  Changes dbm_multiply_workspace(). */
dbm_status dbm_ctx_set_algorithm(dbm_ctx ctx, int algorithm);
/* Densified path on a single rank: byte budget of one K-chunk of dense A + B (default 16 GiB).
 * K is densified and multiplied chunk by chunk (GEMM-accumulate), so 63,360^3 fits in HBM.
 * bytes >= 1; changes dbm_multiply_workspace(). */
dbm_status dbm_ctx_set_dense_chunk_bytes(dbm_ctx ctx, int64_t bytes);
/* should_densify threshold for DBM_PATH_AUTO: occupancy in [0, 1]; default 1.0. */
dbm_status dbm_ctx_set_densify_threshold(dbm_ctx ctx, double threshold);
/* Total kernels this context has launched since creation. */
dbm_status dbm_ctx_launch_count(dbm_ctx ctx, int64_t* out);
dbm_status dbm_ctx_destroy(dbm_ctx ctx);

/* ------------------------------------------------------------------ matrix */
/* A rows x cols FP64 matrix of uniform square blocks of size bs, distributed
 * block-cyclically over ctx's grid.  rows, cols must be multiples of bs (DBM_ERR_SHAPE;
 * reading R10).  Host metadata only; attach device storage before use. */
dbm_status dbm_matrix_create(dbm_ctx ctx, int64_t rows, int64_t cols, int32_t block_size, dbm_matrix* out);
/* Block-sparse matrix (§8f-2, reading R15; P:86, P:157 blocked CSR).  mask: the GLOBAL
 * pattern, (rows/bs) x (cols/bs) bytes row-major, nonzero = block stored; every rank passes the same
 * mask (it is copied; the library keeps it so every rank can plan its peers' panels).  NULL mask = all
 * stored, i.e. a dense matrix in the sparse code path.  The library allocates small device metadata
 * arrays (slot -> (li, lj), (li, lj) -> slot) that dbm_matrix_destroy frees; the arena stays
 * caller-owned.  Errors as dbm_matrix_create; DBM_ERR_NOMEM if the metadata allocation fails.
 * In a multiply C keeps its pattern: products onto absent C blocks are not formed, beta scales every
 * stored C block (DBCSR's retain-sparsity mode). */
dbm_status dbm_matrix_create_sparse(dbm_ctx ctx, int64_t rows, int64_t cols, int32_t block_size,
                                    const uint8_t* mask, dbm_matrix* out);
/* Host-only: the seeded pattern generator of reading R15 / DESIGN.md §4: block (bi, bj) is stored iff
 * u(seed, mat_id, bi, bj) < occupancy (u uniform in [0,1) from the counter generator's stream
 * mat_id | 2^31).  mask: Mb x Nb bytes, row-major, caller-allocated. */
dbm_status dbm_pattern_random(uint64_t seed, uint32_t mat_id, int64_t Mb, int64_t Nb, double occupancy,
                              uint8_t* mask);
/* Host-only symbolic product of two global patterns, for the fill-in workflow (reading R15: a multiply
 * keeps C's pattern, so a caller that wants DBCSR's fill-in creates C with the product pattern first):
 * cmask[i*Nb + j] |= OR over k of amask[i*Kb + k] && bmask[k*Nb + j].  cmask is OR-ed into (pass C's
 * current pattern to keep its blocks, zeros for the pure product pattern).  Row-major byte masks. */
dbm_status dbm_pattern_product(int64_t Mb, int64_t Kb, int64_t Nb, const uint8_t* amask, const uint8_t* bmask,
                               uint8_t* cmask);
/* Stored blocks: local (this rank) and global. */
/* Matrix with non-uniform block sizes (SPEC S:25-26 BlockDims: row_sizes / col_sizes, "non-uniform
 * block sizes are supported throughout"; the paper's (m x k) A blocks and (k x n) B blocks, §II),
 * reading R16: nblk_rows block rows of row_sizes[i] rows, nblk_cols block columns of col_sizes[j]
 * columns (host arrays, copied; every size > 0), block-cyclic over the ctx grid by block index.
 * mask (host, nblk_rows x nblk_cols row-major, nonzero = stored; NULL = every block) makes it
 * block-sparse (R15).  The local arena holds the rank's stored blocks in local CSR order, each
 * row_sizes[bi] x col_sizes[bj] column-major, back to back (dbm_matrix_local_info gives its bytes).
 * All sizes equal: the uniform matrix of dbm_matrix_create / dbm_matrix_create_sparse.  A multiply
 * needs equal block partitions: A's columns = B's rows (else DBM_ERR_PARTITION), A's rows = C's rows,
 * B's columns = C's columns.  Non-uniform operands: Cannon over the copy-engine transport, the
 * densified path for any sizes and patterns, the blocked path for dense patterns with C blocks up to
 * 64 x 64 (DBM_ERR_SHAPE otherwise).  Errors: DBM_ERR_ARG (null pointers, bad counts), DBM_ERR_SHAPE
 * (a size <= 0), DBM_ERR_NOMEM. */
dbm_status dbm_matrix_create_blocked(dbm_ctx ctx, int64_t nblk_rows, const int32_t* row_sizes, int64_t nblk_cols,
                                     const int32_t* col_sizes, const uint8_t* mask, dbm_matrix* out);
/* The block sizes of a matrix (uniform matrices: bs everywhere); either output may be NULL. */
dbm_status dbm_matrix_block_sizes(dbm_matrix m, int32_t* row_sizes, int32_t* col_sizes);
dbm_status dbm_matrix_nnz(dbm_matrix m, int64_t* local_blocks, int64_t* global_blocks);
/* Local share: mloc x nloc blocks; arena_bytes = (stored local blocks)*bs*bs*8 (mloc*nloc*bs*bs*8 dense). */
dbm_status dbm_matrix_local_info(dbm_matrix m, int64_t* mloc_blocks, int64_t* nloc_blocks, int64_t* arena_bytes);
/* Blocked-CSR metadata of the local share: row_ptr[mloc+1], col_idx[local stored blocks]
 * (global block column), row_idx[mloc] (global block row); dense: row_ptr[li] = li*nloc.  Host arrays,
 * caller-allocated. */
dbm_status dbm_matrix_local_csr(dbm_matrix m, int64_t* row_ptr, int64_t* col_idx, int64_t* row_idx);
/* Attach caller-owned device storage of >= arena_bytes bytes, 16-byte aligned. */
dbm_status dbm_matrix_attach(dbm_matrix m, void* device_arena, int64_t bytes);
/* Fill the local share from the counter-based generator of DESIGN.md §4:
 * element (gi,gj) = f(seed, mat_id, gi, gj); kind 0 = U[-1,1), 1 = integers {-2..2}. */
dbm_status dbm_matrix_fill_random(dbm_matrix m, uint64_t seed, uint32_t mat_id, int kind);
/* Copy one locally-owned block (global indices) from / to a host column-major bs x bs array.
 * DBM_ERR_RANGE for indices outside the matrix or a block the pattern does not store,
 * DBM_ERR_OWNERSHIP if another rank owns it.
 * Synchronous with respect to the host. */
dbm_status dbm_matrix_set_block(dbm_matrix m, int64_t bi, int64_t bj, const double* host_colmajor);
dbm_status dbm_matrix_get_block(dbm_matrix m, int64_t bi, int64_t bj, double* host_colmajor);
/* Whole local arena host <-> device (host buffer in arena layout, arena_bytes long).
 * Pinned host memory is copied directly; pageable memory is staged through the context's
 * pinned double buffer.  Enqueued on the ctx stream; host buffers must stay
 * valid until the stream reaches the copy (pinned) or the call returns (pageable). */
dbm_status dbm_matrix_upload(dbm_matrix m, const void* host_arena);
dbm_status dbm_matrix_download(dbm_matrix m, void* host_arena);
/* Rank owning global block (bi,bj): (bi mod Pr)*Pc + (bj mod Pc). */
dbm_status dbm_owner_of_block(dbm_matrix m, int64_t bi, int64_t bj, int* rank);
dbm_status dbm_matrix_destroy(dbm_matrix m);

/* ---------------------------------------------------------------- multiply */
/* Device workspace dbm_multiply needs for these operands and path, in bytes. */
dbm_status dbm_multiply_workspace(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, dbm_path path,
                                  int64_t* bytes);
/* C = alpha*A*B + beta*C (north star), collective over the context's ranks.
 * Cannon over L = lcm(Pr,Pc) steps (reading R5) with NCCL point-to-point panel
 * exchange on a side stream overlapped with the local multiply.
 * path DENSIFIED: densify A, B panels -> FP64 GEMM per step -> undensify C with alpha,
 *   beta (§III).
 * path BLOCKED: stacks of <= stack_cap (a,b,c) block triplets (0 -> 30000) executed
 *   by the batched small-block GEMM.
 * BLAS conventions (reading R8): beta == 0 -> C is not read; alpha == 0 -> A, B not read.
 * Block-sparse operands (any of A, B, C from dbm_matrix_create_sparse; reading R15): the blocked
 * path generates stacks from the stored blocks only and exchanges only stored blocks (copy-engine
 * transport); the densified path densifies absent blocks as zeros; C keeps its pattern.
 * Errors before enqueue: SHAPE (A.cols != B.rows, A.rows != C.rows, B.cols != C.cols),
 * PARTITION (block sizes differ), ALIAS, GRID (different contexts), WORKSPACE.
 * stats may be NULL. */
dbm_status dbm_multiply(dbm_ctx ctx, double alpha, dbm_matrix A, dbm_matrix B, double beta, dbm_matrix C,
                        dbm_path path, int32_t stack_cap, void* workspace, int64_t workspace_bytes, dbm_stats* stats);

/* Host-only (no GPU needed): the point-to-point operations dbm_multiply issues at Cannon step
 * `step` for rank (myrow, mycol) of a pr x pc grid multiplying Mb x Kb by Kb x Nb blocks of bs
 * (owner-pull reading R5).  ops[4*i] = {send(1)/recv(0), operand (0 = A, 1 = B), peer
 * rank, kappa}; bytes[i] = message size.  *n_ops: in = capacity of ops/bytes, out = count.  Pass
 * NULL ops and bytes to query the count. */
dbm_status dbm_plan_exchange(int pr, int pc, int myrow, int mycol, int64_t Mb, int64_t Nb, int64_t Kb, int32_t bs,
                             dbm_path path, int step, int32_t* ops, int64_t* bytes, int* n_ops);

/* Host-only: the canonical Cannon step rank `rank` of a pr x pc grid takes FIRST under the copy-engine
 * transport (the local-first order: with owner-pull every panel is in its owner's exchange pool before
 * any step, so a rank may take the L = lcm(pr, pc) steps in any order; it starts at the step with the
 * most local operands, ties broken towards the owners with the fewest first-step pullers, then runs the
 * steps cyclically: position s is canonical step (first + s) mod L).  The NCCL transport and
 * dbm_plan_exchange keep the canonical order (first = 0).  ARG on a bad grid or rank. */
dbm_status dbm_debug_first_step(int pr, int pc, int rank, int* first_step);

/* Host-only: bytes rank (myrow, mycol) receives from / sends to its peers in one tall-and-skinny
 * multiply of Mb x Kb by Kb x Nb blocks of bs (gather of A and B pieces + the C-share reduction). */
dbm_status dbm_plan_tallskinny(int pr, int pc, int myrow, int mycol, int64_t Mb, int64_t Nb, int64_t Kb, int32_t bs,
                               int64_t* bytes_recv, int64_t* bytes_sent);

/* dbm_multiply with HOST-resident operands (the paper's setting: "the matrices are allocated on the
 * host system"; double buffering with CUDA streams and events; page-locked memory).
 * A_host, B_host, C_host are this rank's arenas in host memory (arena layout, arena_bytes each); the
 * device arenas of A, B, C are the staging copies.  Pinned host buffers: A and B are streamed on the
 * library's copy stream — on a single rank the densified path uploads K-chunk j+1 while chunk j is
 * densified and multiplied; on several ranks (copy-engine transport) each rank uploads and densifies
 * (or packs) its own panels in 5 K-chunks and publishes its progress into the peers' exchange pools
 * (64-bit stream writes), and Cannon's step-0 pulls wait on those flags, so the uploads pipeline
 * across ranks (set DBM_HOST_PIPE=0 in the environment for the whole-upload-then-barrier schedule) —
 * C_host is read only if beta != 0, and C is copied back to C_host.
 * Enqueued on the ctx stream; C_host is valid after the stream reaches the end (dbm_ctx_sync).
 * Pageable host buffers: staged synchronously (no overlap).  Errors as dbm_multiply. */
dbm_status dbm_multiply_host(dbm_ctx ctx, double alpha, dbm_matrix A, dbm_matrix B, double beta, dbm_matrix C,
                             dbm_path path, int32_t stack_cap, void* workspace, int64_t workspace_bytes,
                             const void* A_host, const void* B_host, void* C_host, dbm_stats* stats);

/* ------------------------------------------------------- densify / undensify */
/* Densify the whole local share ("a single block is formed from all the blocks
 * assigned to each thread"): dense is (mloc*bs) x (nloc*bs), layout 0 = column-major with
 * leading dimension ld >= mloc*bs, layout 1 = row-major with ld >= nloc*bs. Device memory.
 * Absent blocks of a sparse matrix densify to zeros; undensify writes stored blocks only. */
dbm_status dbm_densify(dbm_matrix m, double* dense, int64_t ld, int layout);
/* Undensify ("decomposed following the original block sizes") with scaling:
 * block(li,lj)(x,y) = alpha*D(li*bs+x, lj*bs+y) + beta*block (two roundings, no FMA; beta == 0 ->
 * block not read).  D column-major, ld >= mloc*bs. */
dbm_status dbm_undensify(dbm_matrix m, const double* dense, int64_t ld, double alpha, double beta);

/* ------------------------------------------------------------------ debug */
/* Run the GPU stack-generation kernel for Cannon step `step` of A*B into C on this rank and
 * copy the result to host: triplets[3*n] (a_slot, b_slot, c_slot) int32, stack_ptr[n_stacks+1].
 * Sparse operands (R15): runs are the stored C blocks, entries the kk with A(li,kk) and B(kk,lj)
 * both stored, slots ranks among the panel's stored blocks.  Pass NULL arrays to query the sizes
 * only.  Synchronous. */
dbm_status dbm_debug_stacks(dbm_ctx ctx, dbm_matrix A, dbm_matrix B, dbm_matrix C, int step, int32_t cap,
                            int32_t* triplets, int64_t* n_entries, int64_t* stack_ptr, int64_t* n_stacks);
/* Pack panel (blocked path; the Cannon panels of P:168 §II moved as whole blocks):
 * gather nk local block columns (operand 0, an A panel) or block rows (operand 1, a B panel)
 * first, first + stride, ... of a dense-pattern matrix into out (device, caller-owned):
 *   operand 0: block (li, first + q*stride) -> out slot li*pitch + q   (row-major over (li, q));
 *   operand 1: block (first + q*stride, lj) -> out slot q*nloc + lj    (row-major over (q, lj)).
 * pitch (operand 0 only) = blocks per packed row, 0 -> nk (the host pipeline packs K-chunks of a
 * panel at pitch kb).  Blocks copied whole (column-major inside).  Enqueued on the ctx stream.
 * Errors: DBM_ERR_ARG (bad operand, sparse matrix, negative sizes, null out with work to do),
 * DBM_ERR_RANGE (an index outside the local block columns / rows, pitch < nk). */
dbm_status dbm_debug_pack_panel(dbm_matrix m, int operand, int64_t first, int64_t stride, int64_t nk, int64_t pitch,
                                double* out);
/* Raw dense FP64 GEMM kernel (the densified path's local multiply) on device buffers:
 * C(MxN, col-major, ldc) = alpha * At^T * B + beta * C, At K-major (element (m,k) at At[m*lda+k]),
 * B K-major (element (k,n) at B[n*ldb+k]); lda, ldb even.  splitk >= 1 splits K with a
 * deterministic reduction through `partial` (device, splitk*M*N doubles; NULL when splitk == 1);
 * splitk == 0 picks it.  For tests and profiling. */
dbm_status dbm_debug_dgemm(dbm_ctx ctx, int64_t M, int64_t N, int64_t K, double alpha, const double* At, int64_t lda,
                           const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int splitk,
                           double* partial, int64_t partial_bytes);

#ifdef __cplusplus
}
#endif
#endif /* DBM_H */

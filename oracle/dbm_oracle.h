/*
 * dbm_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct host implementation of what the hot path of
 * arXiv 1910.04796 (DBCSR dense multiply on GPUs) computes.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it.  It shares no code, header, table or constant generator with the CUDA
 * path in paper_1910_04796_b200/ and neither side includes the other.
 *
 * Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n (the section /
 * equation is named beside each key).  Every reading of a silent or ambiguous
 * passage is listed in DESIGN.md §3 ("Readings").
 *
 * Layout conventions (reading R3): a matrix of rows x cols with
 * uniform square blocks of bs is stored per rank as an "arena" of
 * mloc x nloc blocks, block (li,lj) at slot li*nloc+lj, element (x,y) of a block
 * at slot*bs*bs + y*bs + x (column-major inside a block; DBCSR is Fortran).
 * A "global" arena is the arena of a 1x1 grid.
 *
 * Parity status: every function is pinned by tests/test_oracle_pins.py except
 * those marked "parity unpinned" below (none at present).
 */
#ifndef DBM_ORACLE_H
#define DBM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- grid & block-cyclic distribution (§II, §IV) ---- */
void orc_grid_dims(int nranks, int* pr, int* pc);
int64_t orc_local_count(int64_t nblocks, int p, int r);
int orc_owner_rank(int64_t bi, int64_t bj, int pr, int pc);
int64_t orc_lcm(int64_t a, int64_t b);

/* ---- seeded synthetic input generator (not the method) ---- */
double orc_fill_value(uint64_t seed, uint32_t mat_id, int64_t gi, int64_t gj, int kind);
void orc_fill_arena(uint64_t seed, uint32_t mat_id, int kind, int64_t rows, int64_t cols, int bs,
                    int pr, int pc, int r, int c, double* arena);

/* ---- distribution data movement (S:120-145 scatter/gather) ---- */
void orc_scatter(const double* global_arena, int64_t Mb, int64_t Nb, int bs, int pr, int pc, int r, int c,
                 double* local_arena);
void orc_gather(const double* local_arena, int64_t Mb, int64_t Nb, int bs, int pr, int pc, int r, int c,
                double* global_arena);
void orc_arena_to_dense(const double* global_arena, int64_t Mb, int64_t Nb, int bs, double* dense_colmajor);
void orc_dense_to_arena(const double* dense_colmajor, int64_t Mb, int64_t Nb, int bs, double* global_arena);

/* ---- the product (north star: C = alpha*A*B + beta*C) ---- */
/* Plain triple loop over blocks on global arenas: for each C block (bi,bj),
 * acc = sum_bk A(bi,bk)*B(bk,bj) (element loops), then C = beta*C + alpha*acc,
 * beta == 0 => C not read; alpha == 0 => A, B not read.  OpenMP over bi. */
void orc_multiply_blocked(int64_t Mb, int64_t Nb, int64_t Kb, int bs, double alpha, const double* A,
                          const double* B, double beta, double* C);
/* Brute-force dense triple loop on column-major dense matrices (a pin for the above). */
void orc_dense_gemm(int64_t M, int64_t N, int64_t K, double alpha, const double* A, const double* B, double beta,
                    double* C);

/* ---- Traversal + Generation (§II) ---- */
/* C-block order by recursive bisection of [0,mloc) x [0,nloc) (reading R6). */
int64_t orc_traversal(int64_t mloc, int64_t nloc, int64_t* li_out, int64_t* lj_out);
/* Stack list for one (rank, step): triplets (a_slot,b_slot,c_slot) int32, stacks of <= cap entries.
 * Pass NULL outputs to count only.  Returns the number of entries. */
int64_t orc_stacks(int64_t mloc, int64_t nloc, int64_t kb, int64_t cap, int32_t* triplets, int64_t* stack_ptr,
                   int64_t* n_stacks);

/* ---- Cannon schedule (§II), owner-pull reading R5 ---- */
/* For step s and rank (r,c): kappa, the rank that holds A(r,kappa) and B(kappa,c). */
void orc_cannon_step(int pr, int pc, int r, int c, int s, int* kappa, int* a_src, int* b_src);
/* Bytes a rank receives / sends over all L steps of one multiply. */
void orc_cannon_bytes(int64_t Mb, int64_t Nb, int64_t Kb, int bs, int pr, int pc, int r, int c,
                      int64_t* bytes_recv, int64_t* bytes_sent);

/* ---- Tall-and-skinny (§II), reading R14 ---- */
void orc_ts_bytes(int64_t Mb, int64_t Nb, int64_t Kb, int bs, int pr, int pc, int r, int c, int64_t* bytes_recv,
                  int64_t* bytes_sent);

/* ---- Densification (§III, Eqs. (1)-(2)) ---- */
void orc_densified_dims(int64_t M, int64_t N, int64_t K, int64_t ptilde, int64_t t, int64_t* a_rows, int64_t* a_cols,
                        int64_t* b_rows, int64_t* b_cols);
/* Coalesce blocks (li, kl) for li in [0,mloc), kl in kcols[0..nk) of a local arena (mloc x nloc blocks)
 * into one dense matrix of (mloc*bs) x (nk*bs).  layout 0: column-major (ld >= mloc*bs);
 * layout 1: row-major (ld >= nk*bs). */
void orc_densify_cols(const double* arena, int64_t mloc, int64_t nloc, int bs, const int64_t* kcols, int64_t nk,
                      double* dense, int64_t ld, int layout);
/* Same for a set of block rows krows (B panels): (nk*bs) x (nloc*bs). */
void orc_densify_rows(const double* arena, int64_t mloc, int64_t nloc, int bs, const int64_t* krows, int64_t nk,
                      double* dense, int64_t ld, int layout);
/* Pack panel (blocked path): operand 0 gathers A blocks (li, kidx[q]) row-major over (li, q);
 * operand 1 gathers B blocks (kidx[q], lj) row-major over (q, lj).  out holds mloc*nk (A) / nk*nloc (B)
 * whole blocks. */
void orc_pack_panel(const double* arena, int64_t mloc, int64_t nloc, int bs, int operand, const int64_t* kidx,
                    int64_t nk, double* out);
/* Undensify C: C_blk(li,lj)(x,y) = fl(fl(alpha*D(li*bs+x, lj*bs+y)) + fl(beta*C_blk)); beta==0 => C not read.
 * D column-major with leading dimension ld. */
void orc_undensify(const double* dense, int64_t ld, int64_t mloc, int64_t nloc, int bs, double alpha, double beta,
                   double* arena);

/* ---- verification of large configs from seeds (north star) ---- */
/* Rows `rows[0..nrows)` of C_out = alpha*A*B + beta*C_in with A,B,C_in regenerated from the generator.
 * out is nrows x N row-major.  OpenMP over column chunks; k ascending per element. */
void orc_rows_from_seeds(int64_t M, int64_t N, int64_t K, uint64_t seed, int kind, double alpha, double beta,
                         const int64_t* rows, int64_t nrows, double* out);
/* Freivalds expected vector: out = alpha*A*(B*x) + beta*C_in*x, x in {-1,+1}^N from x_seed. */
void orc_freivalds_rhs(int64_t M, int64_t N, int64_t K, uint64_t seed, int kind, double alpha, double beta,
                       uint64_t x_seed, double* x_out, double* out);
double orc_sign_value(uint64_t x_seed, int64_t j);

/* ---- Block sparsity (§I "block-sparse ... occupancy between 0.01% up to dense"; §II blocked
 * CSR), reading R15 ---- */
/* Seeded block pattern: block (bi,bj) is stored iff u < occupancy, u = the kind-0 uniform of the counter
 * generator's independent stream mat_id | 2^31 taken at (bi, bj) and mapped to [0,1). */
int orc_pattern_present(uint64_t seed, uint32_t mat_id, int64_t bi, int64_t bj, double occupancy);
void orc_pattern_random(uint64_t seed, uint32_t mat_id, int64_t Mb, int64_t Nb, double occupancy, uint8_t* mask);
/* C_out = alpha*A*B + beta*C_in over stored blocks only: for every stored C block (bi,bj)
 * acc = sum over bk ascending with A(bi,bk) and B(bk,bj) both stored of A_blk*B_blk, then
 * C_blk = beta*C_blk + alpha*acc (C's pattern is kept: products landing on absent C blocks are not
 * formed).  Global arenas in the dense layout (slot bi*Nb+bj); absent blocks are never read or written. */
void orc_multiply_sparse(int64_t Mb, int64_t Nb, int64_t Kb, int bs, double alpha, const double* A,
                         const uint8_t* amask, const double* B, const uint8_t* bmask, double beta, double* C,
                         const uint8_t* cmask);
/* A rank's stored blocks in local CSR order (li ascending, then lj ascending) <-> global dense-layout arena. */
int64_t orc_sparse_compress(const double* global_arena, const uint8_t* mask, int64_t Mb, int64_t Nb, int bs, int pr,
                            int pc, int r, int c, double* local_sparse);
void orc_sparse_expand(const double* local_sparse, const uint8_t* mask, int64_t Mb, int64_t Nb, int bs, int pr, int pc,
                       int r, int c, double* global_arena);
/* Stack list of one (rank, step) with sparse panels: amask (mloc x kb), bmask (kb x nloc), cmask
 * (mloc x nloc), row-major.  Runs = stored C blocks in bisection order; a run's entries are the kk
 * ascending with A(li,kk) and B(kk,lj) stored; a_slot / b_slot / c_slot = the block's rank in the
 * row-major order of the stored blocks of its panel (the packed panel layout).  Empty runs produce no
 * entry.  Stacks: the same greedy whole-run packing as orc_stacks.  Returns the number of entries. */
int64_t orc_sparse_stacks(int64_t mloc, int64_t nloc, int64_t kb, const uint8_t* amask, const uint8_t* bmask,
                          const uint8_t* cmask, int64_t cap, int32_t* triplets, int64_t* stack_ptr, int64_t* n_stacks);

/* Rows of C_out for sparse operands regenerated from seeds (values: seed; patterns: pseed, occ_*); NAN where
 * C's block is absent.  Returns the multiply-adds performed over stored block pairs. */
int64_t orc_sparse_rows_from_seeds(int64_t M, int64_t N, int64_t K, int bs, uint64_t seed, int kind, uint64_t pseed,
                                   double occ_a, double occ_b, double occ_c, double alpha, double beta,
                                   const int64_t* rows, int64_t nrows, double* out);

/* ---- Non-uniform block sizes (§II (m x k)(k x n) block
 * products), reading R16: blocks cut by row_sizes / col_sizes; a rank's arena = its stored blocks in
 * local CSR order, each column-major, back to back. ---- */
int64_t orc_nu_local_elems(const int32_t* rsz, int64_t Mb, const int32_t* csz, int64_t Nb, int pr, int pc, int r,
                           int c, const uint8_t* mask);
void orc_nu_scatter(const double* dense, const int32_t* rsz, int64_t Mb, const int32_t* csz, int64_t Nb, int pr,
                    int pc, int r, int c, const uint8_t* mask, double* local);
void orc_nu_gather(const double* local, const int32_t* rsz, int64_t Mb, const int32_t* csz, int64_t Nb, int pr,
                   int pc, int r, int c, const uint8_t* mask, double* dense);
void orc_nu_multiply(const int32_t* msz, int64_t Mb, const int32_t* nsz, int64_t Nb, const int32_t* ksz, int64_t Kb,
                     double alpha, const double* A, const uint8_t* amask, const double* B, const uint8_t* bmask,
                     double beta, double* C, const uint8_t* cmask);

int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif

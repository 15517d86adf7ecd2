/*
 * dbm_oracle.c — TEST INFRASTRUCTURE ONLY (see dbm_oracle.h).
 *
 * Plain host C, FP64 (the precision the paper fixes: "double-precision floating
 * point numbers", §IV; "only optimized for [double]", §II).  No
 * blocking, fusion or reordering beyond what each cited passage states.
 * Built by __graft_entry__.build(): gcc -O2 -fopenmp -shared -fPIC.
 */
#include "dbm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------- */
/* Grid and block-cyclic distribution.                                         */
/* P:157 §II "distributed over a two-dimensional grid of P MPI processes";     */
/* P:25 §IV "block-cycling distributed a la ScaLAPACK"; S:115 owner rule.      */
/* ------------------------------------------------------------------------- */

/* Reading R1: P -> Pr x Pc with Pr the largest divisor of P not
 * above sqrt(P): 1 -> 1x1, 2 -> 1x2, 4 -> 2x2, 8 -> 2x4 (north star). */
void orc_grid_dims(int nranks, int* pr, int* pc) {
  int best = 1;
  for (int d = 1; (int64_t)d * d <= nranks; ++d)
    if (nranks % d == 0) best = d;
  *pr = best;
  *pc = nranks / best;
}

/* Number of block indices i in [0, nblocks) with i mod p == r. */
int64_t orc_local_count(int64_t nblocks, int p, int r) {
  int64_t n = 0;
  for (int64_t i = r; i < nblocks; i += p) ++n;
  return n;
}

/* owner(i,j) = grid coordinates (i mod Pr, j mod Pc), rank = row*Pc + col. */
int orc_owner_rank(int64_t bi, int64_t bj, int pr, int pc) { return (int)(bi % pr) * pc + (int)(bj % pc); }

int64_t orc_lcm(int64_t a, int64_t b) {
  int64_t x = a, y = b;
  while (y) {
    int64_t t = x % y;
    x = y;
    y = t;
  }
  return a / x * b;
}

/* ------------------------------------------------------------------------- */
/* Seeded synthetic input generator.  Counter based, so every  */
/* element is a pure function of (seed, mat_id, gi, gj); the CUDA side holds  */
/* its own implementation of the same definition.                              */
/* ------------------------------------------------------------------------- */
static uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

static uint64_t gen_bits(uint64_t seed, uint32_t mat_id, int64_t gi, int64_t gj) {
  uint64_t key = mix64(seed + 0x9E3779B97F4A7C15ull * ((uint64_t)mat_id + 1ull));
  uint64_t ctr = ((uint64_t)gi << 32) ^ (uint64_t)gj;
  return mix64(key ^ mix64(ctr));
}

double orc_fill_value(uint64_t seed, uint32_t mat_id, int64_t gi, int64_t gj, int kind) {
  uint64_t bits = gen_bits(seed, mat_id, gi, gj);
  if (kind == 1) return (double)((int)((bits >> 32) % 5u) - 2);
  double u = (double)(bits >> 11) * 0x1.0p-53; /* [0,1), exact */
  return 2.0 * u - 1.0;                         /* [-1,1), exact */
}

void orc_fill_arena(uint64_t seed, uint32_t mat_id, int kind, int64_t rows, int64_t cols, int bs, int pr, int pc,
                    int r, int c, double* arena) {
  int64_t Mb = rows / bs, Nb = cols / bs;
  int64_t mloc = orc_local_count(Mb, pr, r), nloc = orc_local_count(Nb, pc, c);
  int64_t bb = (int64_t)bs * bs;
#pragma omp parallel for schedule(static)
  for (int64_t li = 0; li < mloc; ++li)
    for (int64_t lj = 0; lj < nloc; ++lj) {
      int64_t bi = r + li * pr, bj = c + lj * pc;
      double* blk = arena + (li * nloc + lj) * bb;
      for (int y = 0; y < bs; ++y)
        for (int x = 0; x < bs; ++x)
          blk[(int64_t)y * bs + x] = orc_fill_value(seed, mat_id, bi * bs + x, bj * bs + y, kind);
    }
}

/* ------------------------------------------------------------------------- */
/* Scatter / gather between a global arena and a rank's local arena. */
/* ------------------------------------------------------------------------- */
void orc_scatter(const double* g, int64_t Mb, int64_t Nb, int bs, int pr, int pc, int r, int c, double* l) {
  int64_t mloc = orc_local_count(Mb, pr, r), nloc = orc_local_count(Nb, pc, c), bb = (int64_t)bs * bs;
  for (int64_t li = 0; li < mloc; ++li)
    for (int64_t lj = 0; lj < nloc; ++lj) {
      int64_t bi = r + li * pr, bj = c + lj * pc;
      memcpy(l + (li * nloc + lj) * bb, g + (bi * Nb + bj) * bb, (size_t)bb * sizeof(double));
    }
}

void orc_gather(const double* l, int64_t Mb, int64_t Nb, int bs, int pr, int pc, int r, int c, double* g) {
  int64_t mloc = orc_local_count(Mb, pr, r), nloc = orc_local_count(Nb, pc, c), bb = (int64_t)bs * bs;
  for (int64_t li = 0; li < mloc; ++li)
    for (int64_t lj = 0; lj < nloc; ++lj) {
      int64_t bi = r + li * pr, bj = c + lj * pc;
      memcpy(g + (bi * Nb + bj) * bb, l + (li * nloc + lj) * bb, (size_t)bb * sizeof(double));
    }
}

/* Global arena <-> dense column-major (S:46-74 to_dense / from_dense). */
void orc_arena_to_dense(const double* g, int64_t Mb, int64_t Nb, int bs, double* d) {
  int64_t M = Mb * bs, bb = (int64_t)bs * bs;
  for (int64_t bi = 0; bi < Mb; ++bi)
    for (int64_t bj = 0; bj < Nb; ++bj)
      for (int y = 0; y < bs; ++y)
        for (int x = 0; x < bs; ++x)
          d[(bj * bs + y) * M + bi * bs + x] = g[(bi * Nb + bj) * bb + (int64_t)y * bs + x];
}

void orc_dense_to_arena(const double* d, int64_t Mb, int64_t Nb, int bs, double* g) {
  int64_t M = Mb * bs, bb = (int64_t)bs * bs;
  for (int64_t bi = 0; bi < Mb; ++bi)
    for (int64_t bj = 0; bj < Nb; ++bj)
      for (int y = 0; y < bs; ++y)
        for (int x = 0; x < bs; ++x)
          g[(bi * Nb + bj) * bb + (int64_t)y * bs + x] = d[(bj * bs + y) * M + bi * bs + x];
}

/* ------------------------------------------------------------------------- */
/* The product.  The method reaches the plain definition C = alpha*A*B + beta*C */
/* (north star; "the blocks are coalesced", P:200 undensify), so the    */
/* oracle is that definition written as a triple loop over blocks.            */
/* ------------------------------------------------------------------------- */
void orc_multiply_blocked(int64_t Mb, int64_t Nb, int64_t Kb, int bs, double alpha, const double* A, const double* B,
                          double beta, double* C) {
  int64_t bb = (int64_t)bs * bs;
#pragma omp parallel
  {
    double* acc = (double*)malloc((size_t)bb * sizeof(double));
#pragma omp for schedule(dynamic, 1)
    for (int64_t bi = 0; bi < Mb; ++bi) {
      for (int64_t bj = 0; bj < Nb; ++bj) {
        double* cb = C + (bi * Nb + bj) * bb;
        for (int64_t e = 0; e < bb; ++e) acc[e] = 0.0;
        if (alpha != 0.0) {
          for (int64_t bk = 0; bk < Kb; ++bk) {
            const double* ab = A + (bi * Kb + bk) * bb; /* A(bi,bk), col-major */
            const double* bblk = B + (bk * Nb + bj) * bb; /* B(bk,bj), col-major */
            for (int y = 0; y < bs; ++y)
              for (int z = 0; z < bs; ++z) {
                double b = bblk[(int64_t)y * bs + z];
                for (int x = 0; x < bs; ++x) acc[(int64_t)y * bs + x] += ab[(int64_t)z * bs + x] * b;
              }
          }
        }
        for (int64_t e = 0; e < bb; ++e) {
          double t = alpha * acc[e];
          cb[e] = (beta == 0.0) ? t : t + beta * cb[e];
        }
      }
    }
    free(acc);
  }
}

void orc_dense_gemm(int64_t M, int64_t N, int64_t K, double alpha, const double* A, const double* B, double beta,
                    double* C) {
  for (int64_t j = 0; j < N; ++j)
    for (int64_t i = 0; i < M; ++i) {
      double s = 0.0;
      for (int64_t k = 0; k < K; ++k) s += A[k * M + i] * B[j * K + k];
      double t = alpha * s;
      C[j * M + i] = (beta == 0.0) ? t : t + beta * C[j * M + i];
    }
}

/* ------------------------------------------------------------------------- */
/* Traversal (§II: "cache-oblivious matrix traversal ... loops over A   */
/* matrix row-blocks and then ... over B matrix column-blocks").  Reading R6: */
/* recursive bisection of [0,mloc) x [0,nloc); split the longer side (rows on */
/* ties) at lo + floor(len/2); lower half first; down to single blocks.        */
/* ------------------------------------------------------------------------- */
static int64_t bisect(int64_t r0, int64_t r1, int64_t c0, int64_t c1, int64_t* li, int64_t* lj, int64_t pos) {
  int64_t nr = r1 - r0, nc = c1 - c0;
  if (nr <= 0 || nc <= 0) return pos;
  if (nr == 1 && nc == 1) {
    if (li) {
      li[pos] = r0;
      lj[pos] = c0;
    }
    return pos + 1;
  }
  if (nr >= nc) {
    int64_t mid = r0 + nr / 2;
    pos = bisect(r0, mid, c0, c1, li, lj, pos);
    return bisect(mid, r1, c0, c1, li, lj, pos);
  }
  int64_t mid = c0 + nc / 2;
  pos = bisect(r0, r1, c0, mid, li, lj, pos);
  return bisect(r0, r1, mid, c1, li, lj, pos);
}

int64_t orc_traversal(int64_t mloc, int64_t nloc, int64_t* li, int64_t* lj) {
  return bisect(0, mloc, 0, nloc, li, lj, 0);
}

/* Generation (§II: "organized in batches ... each batch consists of      */
/* maximum 30'000 multiplications").  Reading R6: for each C block in traversal */
/* order, k ascending: (a_slot=li*kb+kk, b_slot=kk*nloc+lj, c_slot=li*nloc+lj). */
/* Whole C-block runs are packed greedily while the stack holds <= cap entries; */
/* a run longer than cap is split into ceil(kb/cap) stacks cap,...,cap,rest.    */
int64_t orc_stacks(int64_t mloc, int64_t nloc, int64_t kb, int64_t cap, int32_t* trip, int64_t* stack_ptr,
                   int64_t* n_stacks) {
  int64_t nrun = mloc * nloc;
  int64_t* li = (int64_t*)malloc((size_t)(nrun > 0 ? nrun : 1) * sizeof(int64_t));
  int64_t* lj = (int64_t*)malloc((size_t)(nrun > 0 ? nrun : 1) * sizeof(int64_t));
  orc_traversal(mloc, nloc, li, lj);
  int64_t e = 0, ns = 0, cur = 0; /* entries so far, stacks closed, entries in the open stack */
  if (stack_ptr) stack_ptr[0] = 0;
  for (int64_t q = 0; q < nrun && kb > 0; ++q) {
    if (trip)
      for (int64_t kk = 0; kk < kb; ++kk) {
        trip[3 * (e + kk) + 0] = (int32_t)(li[q] * kb + kk);
        trip[3 * (e + kk) + 1] = (int32_t)(kk * nloc + lj[q]);
        trip[3 * (e + kk) + 2] = (int32_t)(li[q] * nloc + lj[q]);
      }
    if (kb > cap) { /* close the open stack, then cap, cap, ..., remainder */
      if (cur > 0) {
        ++ns;
        if (stack_ptr) stack_ptr[ns] = e;
        cur = 0;
      }
      for (int64_t done = 0; done < kb;) {
        done += (kb - done < cap) ? kb - done : cap;
        ++ns;
        if (stack_ptr) stack_ptr[ns] = e + done;
      }
    } else {
      if (cur + kb > cap) { /* the run does not fit: close the open stack */
        ++ns;
        if (stack_ptr) stack_ptr[ns] = e;
        cur = 0;
      }
      cur += kb;
    }
    e += kb;
  }
  if (cur > 0) {
    ++ns;
    if (stack_ptr) stack_ptr[ns] = e;
  }
  if (n_stacks) *n_stacks = ns;
  free(li);
  free(lj);
  return e;
}

/* ------------------------------------------------------------------------- */
/* Cannon (§II "we use the Cannon algorithm, where the amount of        */
/* communicated data by each process scales as O(1/sqrt(P))"; P:171 async     */
/* point-to-point).  Reading R5: L = lcm(Pr,Pc) K-panels, kappa = {k : k mod L */
/* = kappa}; at step s rank (r,c) computes C(r,c) += A(r,kappa)*B(kappa,c)     */
/* with kappa = (r+c+s) mod L; A(r,kappa) lives on (r, kappa mod Pc) and        */
/* B(kappa,c) on (kappa mod Pr, c).  For Pr = Pc this is Cannon with the skew  */
/* folded into the step permutation.                              */
/* ------------------------------------------------------------------------- */
void orc_cannon_step(int pr, int pc, int r, int c, int s, int* kappa, int* a_src, int* b_src) {
  int L = (int)orc_lcm(pr, pc);
  int k = (r + c + s) % L;
  *kappa = k;
  *a_src = r * pc + (k % pc);
  *b_src = (k % pr) * pc + c;
}

void orc_cannon_bytes(int64_t Mb, int64_t Nb, int64_t Kb, int bs, int pr, int pc, int r, int c, int64_t* recv,
                      int64_t* sent) {
  int L = (int)orc_lcm(pr, pc);
  int me = r * pc + c;
  int64_t bb8 = (int64_t)bs * bs * 8;
  int64_t rv = 0, sd = 0;
  for (int s = 0; s < L; ++s) {
    /* what I receive */
    int k, asrc, bsrc;
    orc_cannon_step(pr, pc, r, c, s, &k, &asrc, &bsrc);
    int64_t kbk = orc_local_count(Kb, L, k);
    if (asrc != me) rv += orc_local_count(Mb, pr, r) * kbk * bb8;
    if (bsrc != me) rv += kbk * orc_local_count(Nb, pc, c) * bb8;
    /* what I send: every rank whose needed panel lives on me */
    for (int rr = 0; rr < pr; ++rr)
      for (int cc = 0; cc < pc; ++cc) {
        int dst = rr * pc + cc;
        if (dst == me) continue;
        int k2, a2, b2;
        orc_cannon_step(pr, pc, rr, cc, s, &k2, &a2, &b2);
        int64_t kb2 = orc_local_count(Kb, L, k2);
        if (a2 == me) sd += orc_local_count(Mb, pr, rr) * kb2 * bb8;
        if (b2 == me) sd += kb2 * orc_local_count(Nb, pc, cc) * bb8;
      }
  }
  *recv = rv;
  *sent = sd;
}

/* Tall-and-skinny (§II "only for tall-and-skinny matrices ... we use an optimized algorithm,   */
/* where the amount of communicated data by each process scales as O(1)").        */
/* Reading R14: rank p takes K blocks S_p = {k : k mod P == p}, needs every A(i, k) and B(k, j)    */
/* with k in S_p, computes the partial C_p, and receives its own C blocks from every other partial. */
/* Bytes counted by brute force over blocks.                                                        */
void orc_ts_bytes(int64_t Mb, int64_t Nb, int64_t Kb, int bs, int pr, int pc, int r, int c, int64_t* recv,
                  int64_t* sent) {
  const int P = pr * pc, me = r * pc + c;
  const int64_t bb8 = (int64_t)bs * bs * 8;
  int64_t rv = 0, sd = 0;
  for (int q = 0; q < P; ++q) {
    for (int64_t k = q; k < Kb; k += P) {
      for (int64_t i = 0; i < Mb; ++i) {
        const int own = orc_owner_rank(i, k, pr, pc);
        if (q == me && own != me) rv += bb8;
        if (q != me && own == me) sd += bb8;
      }
      for (int64_t j = 0; j < Nb; ++j) {
        const int own = orc_owner_rank(k, j, pr, pc);
        if (q == me && own != me) rv += bb8;
        if (q != me && own == me) sd += bb8;
      }
    }
  }
  /* reduction: each C block's owner receives it from the P-1 other partials */
  for (int64_t i = 0; i < Mb; ++i)
    for (int64_t j = 0; j < Nb; ++j) {
      const int own = orc_owner_rank(i, j, pr, pc);
      if (own == me) rv += (int64_t)(P - 1) * bb8;
      else sd += bb8;
    }
  *recv = rv;
  *sent = sd;
}

/* ------------------------------------------------------------------------- */
/* Densification (§III): "a single block is formed from all the      */
/* blocks assigned to each thread"; Eqs. (1)-(2) give its size.                */
/* ------------------------------------------------------------------------- */
void orc_densified_dims(int64_t M, int64_t N, int64_t K, int64_t pt, int64_t t, int64_t* ar, int64_t* ac, int64_t* br,
                        int64_t* bc) {
  *ar = M / (t * pt); /* Eq. (1): M/(t*P~) x K/P~ */
  *ac = K / pt;
  *br = K / pt; /* Eq. (2): K/P~ x N/P~ */
  *bc = N / pt;
}

void orc_densify_cols(const double* arena, int64_t mloc, int64_t nloc, int bs, const int64_t* kcols, int64_t nk,
                      double* dense, int64_t ld, int layout) {
  int64_t bb = (int64_t)bs * bs;
  for (int64_t li = 0; li < mloc; ++li)
    for (int64_t q = 0; q < nk; ++q) {
      const double* blk = arena + (li * nloc + kcols[q]) * bb;
      for (int y = 0; y < bs; ++y)
        for (int x = 0; x < bs; ++x) {
          int64_t row = li * bs + x, col = q * bs + y;
          double v = blk[(int64_t)y * bs + x];
          if (layout == 0)
            dense[col * ld + row] = v;
          else
            dense[row * ld + col] = v;
        }
    }
}

void orc_densify_rows(const double* arena, int64_t mloc, int64_t nloc, int bs, const int64_t* krows, int64_t nk,
                      double* dense, int64_t ld, int layout) {
  (void)mloc;
  int64_t bb = (int64_t)bs * bs;
  for (int64_t q = 0; q < nk; ++q)
    for (int64_t lj = 0; lj < nloc; ++lj) {
      const double* blk = arena + (krows[q] * nloc + lj) * bb;
      for (int y = 0; y < bs; ++y)
        for (int x = 0; x < bs; ++x) {
          int64_t row = q * bs + x, col = lj * bs + y;
          double v = blk[(int64_t)y * bs + x];
          if (layout == 0)
            dense[col * ld + row] = v;
          else
            dense[row * ld + col] = v;
        }
    }
}

/* Pack a Cannon K-panel of whole blocks (§II "the Cannon algorithm" moves panels
 * of blocks).  operand 0 (A): blocks (li, kcols[q]) for li in [0,mloc), q in [0,nk), packed row-major over
 * (li, q): out slot li*nk + q.  operand 1 (B): blocks (kcols[q], lj), packed row-major over (q, lj): out
 * slot q*nloc + lj.  Blocks are copied whole (column-major inside, reading R3). */
void orc_pack_panel(const double* arena, int64_t mloc, int64_t nloc, int bs, int operand, const int64_t* kidx,
                    int64_t nk, double* out) {
  int64_t bb = (int64_t)bs * bs;
  if (operand == 0) {
    for (int64_t li = 0; li < mloc; ++li)
      for (int64_t q = 0; q < nk; ++q)
        for (int64_t e = 0; e < bb; ++e) out[(li * nk + q) * bb + e] = arena[(li * nloc + kidx[q]) * bb + e];
  } else {
    for (int64_t q = 0; q < nk; ++q)
      for (int64_t lj = 0; lj < nloc; ++lj)
        for (int64_t e = 0; e < bb; ++e) out[(q * nloc + lj) * bb + e] = arena[(kidx[q] * nloc + lj) * bb + e];
  }
}

/* P:200 §III: "the resulting C matrix is undensified, i.e. the large blocks are */
/* decomposed following the original block sizes"; alpha/beta per reading R8.  */
void orc_undensify(const double* dense, int64_t ld, int64_t mloc, int64_t nloc, int bs, double alpha, double beta,
                   double* arena) {
  int64_t bb = (int64_t)bs * bs;
  for (int64_t li = 0; li < mloc; ++li)
    for (int64_t lj = 0; lj < nloc; ++lj) {
      double* blk = arena + (li * nloc + lj) * bb;
      for (int y = 0; y < bs; ++y)
        for (int x = 0; x < bs; ++x) {
          double d = dense[(lj * bs + y) * ld + li * bs + x];
          double t = alpha * d;
          blk[(int64_t)y * bs + x] = (beta == 0.0) ? t : t + beta * blk[(int64_t)y * bs + x];
        }
    }
}

/* ------------------------------------------------------------------------- */
/* Verification of large configs from seeds: sampled rows + Freivalds (north star). */
/* Element (i,j) of A is orc_fill_value(seed, 0, i, j, kind); B uses mat_id 1;  */
/* C_in uses mat_id 2.                                          */
/* ------------------------------------------------------------------------- */
void orc_rows_from_seeds(int64_t M, int64_t N, int64_t K, uint64_t seed, int kind, double alpha, double beta,
                         const int64_t* rows, int64_t nrows, double* out) {
  (void)M;
  const int64_t CH = 256; /* column chunk per task */
  int64_t nch = (N + CH - 1) / CH;
#pragma omp parallel
  {
    double* a = (double*)malloc((size_t)nrows * sizeof(double));
    double* acc = (double*)malloc((size_t)(nrows * CH) * sizeof(double));
#pragma omp for schedule(dynamic, 1)
    for (int64_t ch = 0; ch < nch; ++ch) {
      int64_t j0 = ch * CH, j1 = j0 + CH < N ? j0 + CH : N, w = j1 - j0;
      for (int64_t e = 0; e < nrows * CH; ++e) acc[e] = 0.0;
      if (alpha != 0.0) {
        for (int64_t k = 0; k < K; ++k) {
          for (int64_t q = 0; q < nrows; ++q) a[q] = orc_fill_value(seed, 0, rows[q], k, kind);
          for (int64_t j = j0; j < j1; ++j) {
            double b = orc_fill_value(seed, 1, k, j, kind);
            for (int64_t q = 0; q < nrows; ++q) acc[q * CH + (j - j0)] += a[q] * b;
          }
        }
      }
      for (int64_t q = 0; q < nrows; ++q)
        for (int64_t jj = 0; jj < w; ++jj) {
          double t = alpha * acc[q * CH + jj];
          out[q * N + j0 + jj] =
              (beta == 0.0) ? t : t + beta * orc_fill_value(seed, 2, rows[q], j0 + jj, kind);
        }
    }
    free(a);
    free(acc);
  }
}

double orc_sign_value(uint64_t x_seed, int64_t j) {
  return (mix64(mix64(x_seed ^ 0xA0761D6478BD642Full) ^ (uint64_t)j) >> 63) ? -1.0 : 1.0;
}

void orc_freivalds_rhs(int64_t M, int64_t N, int64_t K, uint64_t seed, int kind, double alpha, double beta,
                       uint64_t x_seed, double* x, double* out) {
  double* y = (double*)malloc((size_t)K * sizeof(double));
  for (int64_t j = 0; j < N; ++j) x[j] = orc_sign_value(x_seed, j);
  /* y = B x */
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < K; ++k) {
    double s = 0.0;
    for (int64_t j = 0; j < N; ++j) s += orc_fill_value(seed, 1, k, j, kind) * x[j];
    y[k] = s;
  }
  /* out = alpha * A y + beta * C_in x */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    double s = 0.0, t = 0.0;
    if (alpha != 0.0)
      for (int64_t k = 0; k < K; ++k) s += orc_fill_value(seed, 0, i, k, kind) * y[k];
    if (beta != 0.0)
      for (int64_t j = 0; j < N; ++j) t += orc_fill_value(seed, 2, i, j, kind) * x[j];
    out[i] = alpha * s + beta * t;
  }
  free(y);
}

/* ------------------------------------------------------------------------- */
/* Block sparsity (§I; §II "blocked compressed sparse row (CSR)    */
/* format"; SPEC S:32-37 occupancy = stored blocks / all blocks).  Reading    */
/* R15: C keeps its stored pattern.                               */
/* ------------------------------------------------------------------------- */
int orc_pattern_present(uint64_t seed, uint32_t mat_id, int64_t bi, int64_t bj, double occupancy) {
  uint64_t bits = gen_bits(seed, mat_id | 0x80000000u, bi, bj);
  double u = (double)(bits >> 11) * 0x1.0p-53; /* [0,1) */
  return u < occupancy;
}

void orc_pattern_random(uint64_t seed, uint32_t mat_id, int64_t Mb, int64_t Nb, double occupancy, uint8_t* mask) {
  for (int64_t bi = 0; bi < Mb; ++bi)
    for (int64_t bj = 0; bj < Nb; ++bj) mask[bi * Nb + bj] = (uint8_t)orc_pattern_present(seed, mat_id, bi, bj, occupancy);
}

void orc_multiply_sparse(int64_t Mb, int64_t Nb, int64_t Kb, int bs, double alpha, const double* A,
                         const uint8_t* amask, const double* B, const uint8_t* bmask, double beta, double* C,
                         const uint8_t* cmask) {
  int64_t bb = (int64_t)bs * bs;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t bi = 0; bi < Mb; ++bi) {
    double* acc = (double*)malloc((size_t)bb * sizeof(double));
    for (int64_t bj = 0; bj < Nb; ++bj) {
      if (!cmask[bi * Nb + bj]) continue;
      for (int64_t e = 0; e < bb; ++e) acc[e] = 0.0;
      for (int64_t bk = 0; bk < Kb; ++bk) {
        if (!amask[bi * Kb + bk] || !bmask[bk * Nb + bj]) continue;
        const double* a = A + (bi * Kb + bk) * bb;
        const double* b = B + (bk * Nb + bj) * bb;
        for (int y = 0; y < bs; ++y)
          for (int x = 0; x < bs; ++x) {
            double s = acc[(int64_t)y * bs + x];
            for (int z = 0; z < bs; ++z) s += a[(int64_t)z * bs + x] * b[(int64_t)y * bs + z];
            acc[(int64_t)y * bs + x] = s;
          }
      }
      double* c = C + (bi * Nb + bj) * bb;
      for (int64_t e = 0; e < bb; ++e) c[e] = (beta == 0.0) ? alpha * acc[e] : beta * c[e] + alpha * acc[e];
    }
    free(acc);
  }
}

int64_t orc_sparse_compress(const double* g, const uint8_t* mask, int64_t Mb, int64_t Nb, int bs, int pr, int pc,
                            int r, int c, double* l) {
  int64_t bb = (int64_t)bs * bs, n = 0;
  for (int64_t bi = r; bi < Mb; bi += pr)
    for (int64_t bj = c; bj < Nb; bj += pc)
      if (mask[bi * Nb + bj]) {
        if (l) memcpy(l + n * bb, g + (bi * Nb + bj) * bb, (size_t)bb * sizeof(double));
        ++n;
      }
  return n;
}

void orc_sparse_expand(const double* l, const uint8_t* mask, int64_t Mb, int64_t Nb, int bs, int pr, int pc, int r,
                       int c, double* g) {
  int64_t bb = (int64_t)bs * bs, n = 0;
  for (int64_t bi = r; bi < Mb; bi += pr)
    for (int64_t bj = c; bj < Nb; bj += pc)
      if (mask[bi * Nb + bj]) {
        memcpy(g + (bi * Nb + bj) * bb, l + n * bb, (size_t)bb * sizeof(double));
        ++n;
      }
}

int64_t orc_sparse_stacks(int64_t mloc, int64_t nloc, int64_t kb, const uint8_t* amask, const uint8_t* bmask,
                          const uint8_t* cmask, int64_t cap, int32_t* trip, int64_t* stack_ptr, int64_t* n_stacks) {
  int64_t nrun = mloc * nloc;
  int64_t* li = (int64_t*)malloc((size_t)(nrun > 0 ? nrun : 1) * sizeof(int64_t));
  int64_t* lj = (int64_t*)malloc((size_t)(nrun > 0 ? nrun : 1) * sizeof(int64_t));
  /* slot of a stored block = its rank in the row-major order of its panel's stored blocks */
  int64_t* aslot = (int64_t*)malloc((size_t)(mloc * kb > 0 ? mloc * kb : 1) * sizeof(int64_t));
  int64_t* bslot = (int64_t*)malloc((size_t)(kb * nloc > 0 ? kb * nloc : 1) * sizeof(int64_t));
  int64_t* cslot = (int64_t*)malloc((size_t)(nrun > 0 ? nrun : 1) * sizeof(int64_t));
  int64_t n = 0;
  for (int64_t i = 0; i < mloc * kb; ++i) aslot[i] = amask[i] ? n++ : -1;
  n = 0;
  for (int64_t i = 0; i < kb * nloc; ++i) bslot[i] = bmask[i] ? n++ : -1;
  n = 0;
  for (int64_t i = 0; i < nrun; ++i) cslot[i] = cmask[i] ? n++ : -1;
  orc_traversal(mloc, nloc, li, lj);
  int64_t e = 0, ns = 0, cur = 0;
  if (stack_ptr) stack_ptr[0] = 0;
  for (int64_t q = 0; q < nrun; ++q) {
    int64_t cs = cslot[li[q] * nloc + lj[q]];
    if (cs < 0) continue;
    int64_t len = 0;
    for (int64_t kk = 0; kk < kb; ++kk) {
      int64_t as = aslot[li[q] * kb + kk], bs_ = bslot[kk * nloc + lj[q]];
      if (as < 0 || bs_ < 0) continue;
      if (trip) {
        trip[3 * (e + len) + 0] = (int32_t)as;
        trip[3 * (e + len) + 1] = (int32_t)bs_;
        trip[3 * (e + len) + 2] = (int32_t)cs;
      }
      ++len;
    }
    if (len == 0) continue;
    if (len > cap) {
      if (cur > 0) {
        ++ns;
        if (stack_ptr) stack_ptr[ns] = e;
        cur = 0;
      }
      for (int64_t done = 0; done < len;) {
        done += (len - done < cap) ? len - done : cap;
        ++ns;
        if (stack_ptr) stack_ptr[ns] = e + done;
      }
    } else {
      if (cur + len > cap) {
        ++ns;
        if (stack_ptr) stack_ptr[ns] = e;
        cur = 0;
      }
      cur += len;
    }
    e += len;
  }
  if (cur > 0) {
    ++ns;
    if (stack_ptr) stack_ptr[ns] = e;
  }
  if (n_stacks) *n_stacks = ns;
  free(li);
  free(lj);
  free(aslot);
  free(bslot);
  free(cslot);
  return e;
}

/* Rows `rows[0..nrows)` of C_out for block-sparse operands regenerated from the seeds: element values from
 * the generator (seed, mat_id 0/1/2), patterns from orc_pattern_present(pseed, mat_id 0/1/2, occ_*).
 * out (nrows x N, row-major) = beta*C + alpha*sum over k of A(i,k) B(k,j) taken over k whose A block
 * (i/bs, k/bs) and B block (k/bs, j/bs) are both stored, for stored C blocks; NAN where C's block is
 * absent.  Returns the number of multiply-adds performed (useful work, 2 flop each). */
int64_t orc_sparse_rows_from_seeds(int64_t M, int64_t N, int64_t K, int bs, uint64_t seed, int kind, uint64_t pseed,
                                   double occ_a, double occ_b, double occ_c, double alpha, double beta,
                                   const int64_t* rows, int64_t nrows, double* out) {
  (void)M;
  int64_t fmas = 0;
  int64_t Kb = K / bs, Nb = N / bs;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : fmas)
  for (int64_t q = 0; q < nrows; ++q) {
    int64_t i = rows[q], bi = i / bs;
    double* acc = (double*)calloc((size_t)N, sizeof(double));
    for (int64_t bk = 0; bk < Kb; ++bk) {
      if (!orc_pattern_present(pseed, 0, bi, bk, occ_a)) continue;
      for (int64_t bj = 0; bj < Nb; ++bj) {
        if (!orc_pattern_present(pseed, 1, bk, bj, occ_b) || !orc_pattern_present(pseed, 2, bi, bj, occ_c)) continue;
        for (int64_t k = bk * bs; k < (bk + 1) * bs; ++k) {
          double a = orc_fill_value(seed, 0, i, k, kind);
          for (int64_t j = bj * bs; j < (bj + 1) * bs; ++j) acc[j] += a * orc_fill_value(seed, 1, k, j, kind);
        }
        fmas += (int64_t)bs * bs;
      }
    }
    for (int64_t j = 0; j < N; ++j) {
      if (!orc_pattern_present(pseed, 2, bi, j / bs, occ_c)) {
        out[q * N + j] = NAN;
        continue;
      }
      double t = alpha * acc[j];
      out[q * N + j] = (beta == 0.0) ? t : t + beta * orc_fill_value(seed, 2, i, j, kind);
    }
    free(acc);
  }
  return fmas;
}

/* ------------------------------------------------------------------------- */
/* Non-uniform block sizes ("BlockDims: row_sizes / */
/* col_sizes", "non-uniform block sizes are supported throughout"; the      */
/* paper's (m x k) x (k x n) block products, §II).  A matrix is a dense     */
/* M x N array cut into blocks by row_sizes (Mb entries) and col_sizes (Nb);      */
/* block (bi, bj) covers rows roff[bi] .. roff[bi]+rsz[bi]-1 and the same for     */
/* columns, roff / coff the prefix sums.  A rank's local arena holds its stored    */
/* blocks (owner rule S:115, block-cyclic over block indices) in local CSR order   */
/* (li, then lj), each block column-major, packed back to back (reading R16).     */
/* ------------------------------------------------------------------------- */
static int64_t nu_off(const int32_t* sz, int64_t i) {
  int64_t o = 0;
  for (int64_t q = 0; q < i; ++q) o += sz[q];
  return o;
}

int64_t orc_nu_local_elems(const int32_t* rsz, int64_t Mb, const int32_t* csz, int64_t Nb, int pr, int pc, int r,
                           int c, const uint8_t* mask) {
  int64_t n = 0;
  for (int64_t bi = r; bi < Mb; bi += pr)
    for (int64_t bj = c; bj < Nb; bj += pc)
      if (!mask || mask[bi * Nb + bj]) n += (int64_t)rsz[bi] * csz[bj];
  return n;
}

/* dense (column-major, ld = M = sum rsz) -> the local arena of rank (r, c) */
void orc_nu_scatter(const double* dense, const int32_t* rsz, int64_t Mb, const int32_t* csz, int64_t Nb, int pr,
                    int pc, int r, int c, const uint8_t* mask, double* local) {
  int64_t M = nu_off(rsz, Mb), o = 0;
  for (int64_t bi = r; bi < Mb; bi += pr)
    for (int64_t bj = c; bj < Nb; bj += pc) {
      if (mask && !mask[bi * Nb + bj]) continue;
      int64_t r0 = nu_off(rsz, bi), c0 = nu_off(csz, bj);
      for (int64_t y = 0; y < csz[bj]; ++y)
        for (int64_t x = 0; x < rsz[bi]; ++x) local[o++] = dense[(c0 + y) * M + r0 + x];
    }
}

/* the local arena of rank (r, c) -> its blocks' places in the dense array (other entries untouched) */
void orc_nu_gather(const double* local, const int32_t* rsz, int64_t Mb, const int32_t* csz, int64_t Nb, int pr,
                   int pc, int r, int c, const uint8_t* mask, double* dense) {
  int64_t M = nu_off(rsz, Mb), o = 0;
  for (int64_t bi = r; bi < Mb; bi += pr)
    for (int64_t bj = c; bj < Nb; bj += pc) {
      if (mask && !mask[bi * Nb + bj]) continue;
      int64_t r0 = nu_off(rsz, bi), c0 = nu_off(csz, bj);
      for (int64_t y = 0; y < csz[bj]; ++y)
        for (int64_t x = 0; x < rsz[bi]; ++x) dense[(c0 + y) * M + r0 + x] = local[o++];
    }
}

/* C = alpha*A*B + beta*C over blocks of mixed (m, n, k) sizes: for every stored C block (bi, bj),
 * acc = sum over bk ascending with A(bi, bk) and B(bk, bj) stored of the (m x k) x (k x n) block
 * product (element loops), then C_blk = beta*C_blk + alpha*acc (beta == 0: C not read; C's pattern is
 * kept, reading R15).  Dense column-major arrays: A M x K, B K x N, C M x N; masks NULL = all stored.
 * The block products are the paper's (§II "(m x k) for A blocks and (k x n) for B blocks"). */
void orc_nu_multiply(const int32_t* msz, int64_t Mb, const int32_t* nsz, int64_t Nb, const int32_t* ksz, int64_t Kb,
                     double alpha, const double* A, const uint8_t* amask, const double* B, const uint8_t* bmask,
                     double beta, double* C, const uint8_t* cmask) {
  int64_t M = nu_off(msz, Mb), K = nu_off(ksz, Kb);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t bi = 0; bi < Mb; ++bi) {
    int64_t r0 = nu_off(msz, bi), m = msz[bi];
    for (int64_t bj = 0; bj < Nb; ++bj) {
      if (cmask && !cmask[bi * Nb + bj]) continue;
      int64_t c0 = nu_off(nsz, bj), n = nsz[bj];
      double* acc = (double*)calloc((size_t)(m * n > 0 ? m * n : 1), sizeof(double));
      for (int64_t bk = 0; bk < Kb && alpha != 0.0; ++bk) { /* alpha == 0: A, B not read (reading R8) */
        if ((amask && !amask[bi * Kb + bk]) || (bmask && !bmask[bk * Nb + bj])) continue;
        int64_t k0 = nu_off(ksz, bk);
        for (int64_t y = 0; y < n; ++y)
          for (int64_t x = 0; x < m; ++x) {
            double sum = acc[y * m + x];
            for (int64_t z = 0; z < ksz[bk]; ++z) sum += A[(k0 + z) * M + r0 + x] * B[(c0 + y) * K + k0 + z];
            acc[y * m + x] = sum;
          }
      }
      for (int64_t y = 0; y < n; ++y)
        for (int64_t x = 0; x < m; ++x) {
          double* p = &C[(c0 + y) * M + r0 + x];
          double t = alpha * acc[y * m + x];
          *p = (beta == 0.0) ? t : t + beta * *p;
        }
      free(acc);
    }
  }
}

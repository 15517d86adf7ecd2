// Block-sparse matrices (§8f-2, reading R15): "DBCSR matrices are stored in a blocked compressed sparse
// row (CSR) format" (§II), occupancy 0.01 % up to dense (§I).  A rank stores its blocks in
// local CSR order; slot s holds block (li, lj) = ij[2s], ij[2s+1].
//
//   fill_sparse / sp_densify / sp_undensify / sp_gather : HBM-bound data movement over stored blocks
//     (absent blocks densify to zeros, S:59 / S:477; only stored C blocks are written, R15).
//   sp_count / sp_fill : the Generation phase for sparse panels.  A run is a stored C block
//     (bisection order, R6); its entries are the kk where A(li, kk) and B(kk, lj) are both stored,
//     found by merging the A-panel row list with the B-panel column list (both kk-ascending).  Two
//     passes around an exclusive scan give every run its offset: integer work, bit-exact vs oracle.
//   smm_sparse<BS> : batched small-block DGEMM over runs of any length (the LIBCUSMM role):
//     a team of warps per run accumulates its entries with DMMA (mma.sync.m8n8k4.f64), the next
//     entry's A and B blocks streamed into shared memory with cp.async while this one multiplies;
//     C_blk += alpha * acc (beta was applied to every stored C block before the first step).
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "dbm_internal.h"

namespace dbm {

namespace {

inline unsigned sp_grid(int64_t work, int per = 256, int mult = 16) {
  int64_t g = (work + per - 1) / per;
  g = std::min<int64_t>(g, (int64_t)num_sms() * mult);
  return (unsigned)std::max<int64_t>(g, 1);
}

__device__ __forceinline__ uint64_t sp_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

__global__ void fill_sparse_kernel(double* __restrict__ arena, int64_t total, const int32_t* __restrict__ ij, int bs,
                                   int pr, int pc, int r, int c, uint64_t key, int kind) {
  const int64_t bb = (int64_t)bs * bs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t slot = e / bb, w = e - slot * bb;
    const int64_t y = w / bs, x = w - y * bs;
    const int64_t li = ij[2 * slot], lj = ij[2 * slot + 1];
    const uint64_t gi = (uint64_t)((r + li * pr) * bs + x), gj = (uint64_t)((c + lj * pc) * bs + y);
    const uint64_t bits = sp_mix64(key ^ sp_mix64((gi << 32) ^ gj));
    double v;
    if (kind == 1) {
      v = (double)((int)((bits >> 32) % 5u) - 2);
    } else {
      const double u = __dmul_rn((double)(bits >> 11), 0x1.0p-53);
      v = __dsub_rn(__dmul_rn(2.0, u), 1.0);
    }
    arena[e] = v;
  }
}

// axis 0 (A panel): blocks with lj = sel0 + q*stride -> dense block (li, q)
// axis 1 (B panel): blocks with li = sel0 + q*stride -> dense block (q, lj)
// layout 0: dense[col*ld + row]; layout 1: dense[row*ld + col]
__global__ void sp_densify_kernel(const double* __restrict__ arena, const int32_t* __restrict__ ij, int64_t total,
                                  int bs, int axis, int64_t sel0, int64_t stride, int64_t nk,
                                  double* __restrict__ dense, int64_t ld, int layout) {
  const int64_t bb = (int64_t)bs * bs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t slot = e / bb, w = e - slot * bb;
    const int64_t li = ij[2 * slot], lj = ij[2 * slot + 1];
    const int64_t d = (axis == 0 ? lj : li) - sel0;
    if (d < 0 || d % stride != 0 || d / stride >= nk) continue;
    const int64_t q = d / stride, y = w / bs, x = w - y * bs;
    const int64_t row = (axis == 0 ? li : q) * bs + x, col = (axis == 0 ? q : lj) * bs + y;
    dense[layout == 0 ? col * ld + row : row * ld + col] = arena[e];
  }
}

__global__ void sp_undensify_kernel(const double* __restrict__ dense, int64_t ld, int nsplit, int64_t split_stride,
                                    const int32_t* __restrict__ ij, int bs, int64_t total, double alpha, double beta,
                                    double* __restrict__ arena) {
  const int64_t bb = (int64_t)bs * bs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t slot = e / bb, w = e - slot * bb;
    const int64_t y = w / bs, x = w - y * bs;
    const int64_t li = ij[2 * slot], lj = ij[2 * slot + 1];
    const int64_t di = (lj * bs + y) * ld + li * bs + x;
    double d = dense[di];
    for (int s = 1; s < nsplit; ++s) d = __dadd_rn(d, dense[di + s * split_stride]);
    const double t = __dmul_rn(alpha, d);
    arena[e] = (beta == 0.0) ? t : __dadd_rn(t, __dmul_rn(beta, arena[e]));
  }
}

__global__ void sp_gather_kernel(const double* __restrict__ arena, const int32_t* __restrict__ src, int64_t total,
                                 int bs, double* __restrict__ out) {
  const int64_t bb = (int64_t)bs * bs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / bb, w = e - q * bb;
    out[e] = arena[(int64_t)src[q] * bb + w];
  }
}

// ---------------------------------------------------------------- Generation (sparse)
// A panel: row li's stored blocks are a_kk[a_ptr[li] .. a_ptr[li+1]) (kk ascending), slot = position.
// B panel: column lj's stored blocks are b_kk / b_slot[b_ptr[lj] .. b_ptr[lj+1]) (kk ascending).
// C: cmap[li*nloc + lj] = stored slot or -1 (nullptr: dense C, slot li*nloc + lj).
struct SpPanels {
  const int32_t* a_ptr;
  const int32_t* a_kk;
  const int32_t* b_ptr;
  const int32_t* b_kk;
  const int32_t* b_slot;
  const int32_t* cmap;
  int64_t nloc;
};

template <bool WRITE>
__global__ void sp_gen_kernel(SpPanels P, const int32_t* __restrict__ li_of, const int32_t* __restrict__ lj_of,
                              int64_t q0, int64_t n, int64_t* __restrict__ cnt, const int64_t* __restrict__ off,
                              int32_t* __restrict__ trip) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t li = li_of[q0 + t], lj = lj_of[q0 + t];
    const int64_t cs = P.cmap ? (int64_t)P.cmap[li * P.nloc + lj] : li * P.nloc + lj;
    int64_t m = 0;
    if (cs >= 0) {
      int32_t a = P.a_ptr[li];
      const int32_t a1 = P.a_ptr[li + 1];
      int32_t b = P.b_ptr[lj];
      const int32_t b1 = P.b_ptr[lj + 1];
      int64_t o = WRITE ? off[t] : 0;
      while (a < a1 && b < b1) {
        const int32_t ka = P.a_kk[a], kb = P.b_kk[b];
        if (ka == kb) {
          if (WRITE) {
            trip[3 * (o + m) + 0] = a;
            trip[3 * (o + m) + 1] = P.b_slot[b];
            trip[3 * (o + m) + 2] = (int32_t)cs;
          }
          ++m;
          ++a;
          ++b;
        } else if (ka < kb) {
          ++a;
        } else {
          ++b;
        }
      }
    }
    if (!WRITE) cnt[t] = m;
  }
}

// ---------------------------------------------------------------- smm over runs of any length
__device__ __forceinline__ void sp_dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

constexpr int sp_pitch(int bs) {  // column pitch (doubles) with pitch mod 16 in {4, 12}: the four k (or n)
  int p = bs;                      // columns a half-warp's 64-bit fragment loads touch land on disjoint
  while (p % 16 != 4 && p % 16 != 12) ++p;  // groups of 4 bank pairs (conflict-free with rows 0..3)
  return p;
}

template <int BS>
struct SpCfg {
  static constexpr int MT = (BS + 7) / 8;            // 8x8 subtiles per block dimension
  static constexpr int TEAM = MT >= 4 ? 4 : 1;       // warps per run
  static constexpr int NPW = MT / TEAM;              // n-subtiles per warp
  static constexpr int WARPS = TEAM == 4 ? 4 : 8;    // bs 64: one 4-warp team
  static constexpr int TEAMS = WARPS / TEAM;
  static constexpr int BB = BS * BS;
  static constexpr int P = sp_pitch(BS);             // 28 (bs 22), 68 (bs 64)
  // stage = A block [k][m] (pitch P, m < P) + B block [n][k] (pitch P, n < 8*MT padded)
  static constexpr int A_D = BS * P;
  static constexpr int B_D = 8 * MT * P;
  static constexpr int STAGE = ((A_D + B_D) + 1) / 2 * 2;
  static constexpr size_t SMEM = (size_t)TEAMS * 2 * STAGE * 8;
  static_assert(MT % TEAM == 0, "team split");
  static_assert(BS % 2 == 0, "16-byte column chunks");
};

template <int BS>
__global__ void __launch_bounds__(SpCfg<BS>::WARPS * 32, 1)
    smm_sparse_kernel(const int32_t* __restrict__ trip, const int64_t* __restrict__ off, int64_t nruns,
                      const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                      double alpha) {
  using Cfg = SpCfg<BS>;
  constexpr int MT = Cfg::MT, TEAM = Cfg::TEAM, NPW = Cfg::NPW, BB = Cfg::BB, P = Cfg::P;
  constexpr int HALF = BS / 2;  // 16-byte chunks per block column
  extern __shared__ __align__(16) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp / TEAM, tw = warp % TEAM;
  const int g = lane >> 2, t = lane & 3;
  double* st0 = sm + (size_t)team * 2 * Cfg::STAGE;
  const int tlane = tw * 32 + lane;  // 0 .. TEAM*32-1
  constexpr int TT = TEAM * 32;
  auto team_sync = [&]() {
    if (TEAM == 1)
      __syncwarp();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(TT) : "memory");
  };

  // The team's runs (run = first + i * nteams) are consumed as ONE stream of entries: the copy of the
  // next entry (possibly the next run's first) is in flight while this one multiplies, its slots and
  // the next run's offsets are fetched one step earlier still, and a run's C block is read into
  // registers when the run starts, so no global-memory latency sits on the critical path.
  const int64_t nteams = (int64_t)gridDim.x * Cfg::TEAMS;
  int64_t pr = (int64_t)blockIdx.x * Cfg::TEAMS + team, pe = 0, pend = 0, pstart = 0;
  while (pr < nruns) {
    pe = off[pr];
    pend = off[pr + 1];
    if (pe < pend) break;
    pr += nteams;
  }
  if (pr >= nruns) return;
  pstart = pe;
  int la = trip[3 * pe], lb = trip[3 * pe + 1], lc = trip[3 * pe + 2];
  int64_t gr = pr + nteams, g0 = 0, g1 = 0;  // prefetched offsets of the team's next run
  if (gr < nruns) {
    g0 = off[gr];
    g1 = off[gr + 1];
  }
  struct Meta {
    int cslot;
    bool first, last;
  };
  auto issue = [&](int stage) -> Meta {
    const Meta m{lc, pe == pstart, pe + 1 == pend};
    const double* a = A + (int64_t)la * BB;
    const double* b = B + (int64_t)lb * BB;
    double* dst = st0 + (size_t)stage * Cfg::STAGE;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(dst + Cfg::A_D);
    for (int i = tlane; i < BS * HALF; i += TT) {
      const int col = i / HALF, j = i - col * HALF;
      const uint32_t d = 8u * (uint32_t)(col * P + 2 * j);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa + d), "l"(a + col * BS + 2 * j) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sb + d), "l"(b + col * BS + 2 * j) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (++pe == pend) {  // next nonempty run of the team
      int64_t r = gr, e = g0, e1 = g1;
      while (r < nruns && e == e1) {
        r += nteams;
        if (r < nruns) {
          e = off[r];
          e1 = off[r + 1];
        }
      }
      pr = r;
      pe = pstart = e;
      pend = e1;
      gr = pr + nteams;
      if (gr < nruns) {
        g0 = off[gr];
        g1 = off[gr + 1];
      }
    }
    if (pr < nruns) {  // slots of the entry after this one (consumed by the next issue)
      la = trip[3 * pe];
      lb = trip[3 * pe + 1];
      lc = trip[3 * pe + 2];
    }
    return m;
  };

  double acc[MT][NPW][2];
  double creg[TEAM == 1 ? MT : 1][TEAM == 1 ? NPW : 1][2];
  Meta nxt = issue(0);
  int cs = 0;
  for (;;) {
    const Meta cur = nxt;
    const bool more = pr < nruns;
    if (more) {
      nxt = issue(cs ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    team_sync();
    double* cb = C + (int64_t)cur.cslot * BB;
    if (cur.first) {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NPW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      if constexpr (TEAM == 1) {
#pragma unroll
        for (int mi = 0; mi < MT; ++mi)
#pragma unroll
          for (int ni = 0; ni < NPW; ++ni)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const int m = mi * 8 + g, n = ni * 8 + 2 * t + jj;
              creg[mi][ni][jj] = (m < BS && n < BS) ? cb[m + n * BS] : 0.0;
            }
      }
    }
    const double* sA = st0 + (size_t)cs * Cfg::STAGE;  // (m, k) at k*P + m
    const double* sB = sA + Cfg::A_D;                   // (k, n) at n*P + k
#pragma unroll
    for (int ks = 0; ks < (BS + 3) / 4; ++ks) {
      const int k = 4 * ks + t;
      const bool kok = (BS % 4 == 0) || k < BS;
      double a[MT], b[NPW];
#pragma unroll
      for (int mi = 0; mi < MT; ++mi) a[mi] = kok ? sA[k * P + mi * 8 + g] : 0.0;
#pragma unroll
      for (int ni = 0; ni < NPW; ++ni) b[ni] = kok ? sB[((tw * NPW + ni) * 8 + g) * P + k] : 0.0;
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NPW; ++ni) sp_dmma(acc[mi][ni], a[mi], b[ni]);
    }
    team_sync();  // every warp is done with this stage before it is refilled
    if (cur.last) {
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NPW; ++ni)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int m = mi * 8 + g, n = (tw * NPW + ni) * 8 + 2 * t + jj;
            if (m < BS && n < BS) {
              double* p = cb + m + n * BS;
              const double c0 = (TEAM == 1) ? creg[TEAM == 1 ? mi : 0][TEAM == 1 ? ni : 0][jj] : *p;
              *p = __dadd_rn(c0, __dmul_rn(alpha, acc[mi][ni][jj]));
            }
          }
    }
    if (!more) break;
    cs ^= 1;
  }
}

// ---- per-run variant (bs 22): one run at a time per warp, blocks staged at their natural 22-double
// column pitch, next entry prefetched.  Measured against the stream kernel above on one B200
// (profiles/r01_smm_sparse_variants.jsonl): faster for bs 22 once runs hold more than a few entries
// (21.0 vs 17.1 TFLOP/s at 11,264^3 occupancy 0.5; 17.0 vs 14.0 at 63,360^3 occupancy 0.1), slower
// for bs 64 (21.9 vs 24.7), so bs 22 uses this one and bs 64 the stream kernel.
template <int BS>
struct SpRunCfg {
  static constexpr int MT = (BS + 7) / 8;            // 8x8 subtiles per block dimension
  static constexpr int TEAM = MT >= 8 ? 4 : MT >= 4 ? 2 : 1;  // warps per run
  static constexpr int NPW = MT / TEAM;                        // n-subtiles per warp
  static constexpr int WARPS = TEAM == 1 ? 8 : 4;  // bs 64: one 4-warp team (132 KB of stages); bs 26-32: two teams
  static constexpr int TEAMS = WARPS / TEAM;
  static constexpr int BB = BS * BS;
  // entries per pipeline stage: a bs <= 8 entry is a few hundred bytes, so a stage carries four of them
  // (one cp.async issue, one wait and one barrier per four entries instead of per entry)
  static constexpr int G = BS <= 8 ? 4 : 1;
  // one entry = A block (+ slack for the padded rows m >= BS) and B block (+ padded columns n >= BS)
  // (odd bs^2: +2 for the 8-byte shift below); the stage ends with one int per entry holding the shifts
  // column pitch in shared memory: at bs 16 / 32 the natural pitch (0 mod 16) puts all four k (or n)
  // columns a half-warp's fragment loads touch on the same banks (4- to 8-way conflicts), so those
  // blocks are staged at a pitch = 4 or 12 mod 16 (conflict-free): 15.3 -> 24.8 and 22.2 -> 30.0
  // TFLOP/s.  The same staging measured neutral at bs 26 and slower at bs 6 / 8 (more shared memory
  // per stage, fewer resident CTAs), which keep their natural pitch, as do the odd sizes
  static constexpr int P = (BS >= 16 && BS % 8 == 0) ? sp_pitch(BS) : BS;
  static constexpr int A_D = ((BS - 1) * P + 8 * MT + 2 + 1) / 2 * 2;
  static constexpr int B_D = (8 * MT * P + 8 + 2 + 1) / 2 * 2;
  static constexpr int STAGE = G * (A_D + B_D) + (G + 1) / 2 * 2;
  static constexpr int STAGES = 2;
  // copies per block: 16 B each when bs^2 is even; for odd bs^2 a block starts 8 bytes off a 16-byte
  // boundary when its slot is odd, so it is staged one double further in and copied as (bs^2 - 1) / 2
  // 16-byte chunks plus one 8-byte element (the first when shifted, else the last)
  static constexpr int CH = BB % 2 == 0 ? BB / 2 : (BB - 1) / 2 + 1;
  static constexpr size_t SMEM = (size_t)TEAMS * STAGES * STAGE * 8;
  static_assert(MT % TEAM == 0, "team split");
};

template <int BS>
__global__ void __launch_bounds__(SpRunCfg<BS>::WARPS * 32, 1)
    smm_sparse_run_kernel(const int32_t* __restrict__ trip, const int64_t* __restrict__ off, int64_t nruns,
                      int64_t kb, const double* __restrict__ A, const double* __restrict__ B,
                      double* __restrict__ C, double alpha, double beta_first) {
  using Cfg = SpRunCfg<BS>;
  constexpr int MT = Cfg::MT, TEAM = Cfg::TEAM, NPW = Cfg::NPW, BB = Cfg::BB, G = Cfg::G, CH = Cfg::CH;
  extern __shared__ __align__(16) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp / TEAM, tw = warp % TEAM;
  const int g = lane >> 2, t = lane & 3;
  double* st0 = sm + (size_t)team * Cfg::STAGES * Cfg::STAGE;
  const int tlane = tw * 32 + lane;  // 0 .. TEAM*32-1
  constexpr int TT = TEAM * 32;
  // stage layout: A of entries 0..G-1, then B of entries 0..G-1
  // blocks are 16-byte aligned when BB is even (bs 22, 64, ...); odd BB (bs 5, 13, 23) copies 8 bytes at a time
  auto load = [&](double* dst, int64_t first, int64_t end) {
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(dst);
    for (int idx = tlane; idx < G * CH; idx += TT) {
      const int i = idx / CH, c = idx - i * CH;
      const int64_t entry = first + i;
      if (entry >= end) break;  // idx grows with i: the rest of this lane's copies are past the run too
      const double* a = A + (int64_t)trip[3 * entry] * BB;
      const double* b = B + (int64_t)trip[3 * entry + 1] * BB;
      const uint32_t sa = s0 + 8u * (uint32_t)(i * Cfg::A_D), sb = s0 + 8u * (uint32_t)(G * Cfg::A_D + i * Cfg::B_D);
      if (BB % 2 == 0) {  // chunk c = doubles 2c, 2c+1 of column c / (bs/2), staged at that column's pitch
        const int col = c / (BS / 2), d = col * Cfg::P + 2 * (c - col * (BS / 2));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa + 8u * d), "l"(a + 2 * c) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sb + 8u * d), "l"(b + 2 * c) : "memory");
      } else {
        // 1: block starts 8 mod 16 (from the address: a chunked panel base A + k0 bs^2 may itself be 8 mod 16)
        const int pa = (int)(((uintptr_t)a >> 3) & 1), pb = (int)(((uintptr_t)b >> 3) & 1);
        if (c < CH - 1) {  // elements pa + 2c, pa + 2c + 1 -> shared doubles 2 pa + 2c (16-byte aligned)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa + 16u * (pa + c)), "l"(a + pa + 2 * c)
                       : "memory");
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sb + 16u * (pb + c)), "l"(b + pb + 2 * c)
                       : "memory");
        } else {  // the single element: 0 when shifted, else bs^2 - 1; this lane also records the shifts
          const int ja = pa ? 0 : BB - 1, jb = pb ? 0 : BB - 1;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa + 8u * (pa + ja)), "l"(a + ja) : "memory");
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sb + 8u * (pb + jb)), "l"(b + jb) : "memory");
          reinterpret_cast<int*>(dst + G * (Cfg::A_D + Cfg::B_D))[i] = pa | (pb << 1);
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto team_sync = [&]() {
    if (TEAM == 1)
      __syncwarp();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(TT) : "memory");
  };
  // fragment row / column of this lane in each subtile
  int rowm[MT], coln[NPW];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi) rowm[mi] = mi * 8 + g;
#pragma unroll
  for (int ni = 0; ni < NPW; ++ni) coln[ni] = (tw * NPW + ni) * 8 + g;

  const int64_t nteams = (int64_t)gridDim.x * Cfg::TEAMS;
  for (int64_t run = (int64_t)blockIdx.x * Cfg::TEAMS + team; run < nruns; run += nteams) {
    // sparse stacks carry run offsets; dense stacks (off == nullptr) are uniform runs of kb entries
    const int64_t e0 = off ? off[run] : run * kb, e1 = off ? off[run + 1] : e0 + kb;
    if (e0 == e1) continue;
    double acc[MT][NPW][2], cold[MT][NPW][2];  // (cold: the run's C values, loaded under its products)
    double* cb = C + (int64_t)trip[3 * e0 + 2] * BB;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NPW; ++j)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          acc[i][j][jj] = 0.0;
          const int m = rowm[i], n = (tw * NPW + j) * 8 + 2 * t + jj;
          cold[i][j][jj] = (beta_first != 0.0 && m < BS && n < BS) ? cb[m + n * BS] : 0.0;
        }
    team_sync();  // the previous run's last stage has been consumed by every team warp
    load(st0, e0, e1);
    int si = 0;
    for (int64_t e = e0; e < e1; e += G, si ^= 1) {
      double* cur = st0 + (size_t)si * Cfg::STAGE;
      if (e + G < e1) {
        load(st0 + (size_t)(si ^ 1) * Cfg::STAGE, e + G, e1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      team_sync();
#pragma unroll
      for (int i = 0; i < G; ++i) {
        if (G > 1 && e + i >= e1) break;  // warp-uniform
        const int sh = BB % 2 == 0 ? 0 : reinterpret_cast<const int*>(cur + G * (Cfg::A_D + Cfg::B_D))[i];
        const double* sA = cur + i * Cfg::A_D + (sh & 1);                 // (m, k) at k*BS + m
        const double* sB = cur + G * Cfg::A_D + i * Cfg::B_D + (sh >> 1);  // (k, n) at n*BS + k
#pragma unroll
        for (int ks = 0; ks < (BS + 3) / 4; ++ks) {
          const int k = 4 * ks + t;
          const bool kok = (BS % 4 == 0) || k < BS;
          double a[MT], b[NPW];
#pragma unroll
          for (int mi = 0; mi < MT; ++mi) a[mi] = kok ? sA[k * Cfg::P + rowm[mi]] : 0.0;
#pragma unroll
          for (int ni = 0; ni < NPW; ++ni) b[ni] = kok ? sB[coln[ni] * Cfg::P + k] : 0.0;
#pragma unroll
          for (int mi = 0; mi < MT; ++mi)
#pragma unroll
            for (int ni = 0; ni < NPW; ++ni) sp_dmma(acc[mi][ni], a[mi], b[ni]);
        }
      }
      team_sync();  // every warp is done with `cur` before it is refilled
    }
#pragma unroll
    for (int mi = 0; mi < MT; ++mi)
#pragma unroll
      for (int ni = 0; ni < NPW; ++ni)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const int m = rowm[mi], n = (tw * NPW + ni) * 8 + 2 * t + jj;
          if (m < BS && n < BS) {
            const double c0 = cold[mi][ni][jj], ab = __dmul_rn(alpha, acc[mi][ni][jj]);
            cb[m + n * BS] = beta_first == 1.0 ? __dadd_rn(c0, ab) : beta_first == 0.0 ? ab : fma(beta_first, c0, ab);
          }
        }
  }
}

// ---- bs 22 with TMA bulk staging (round 2): the per-run kernel's structure -- one warp per run, blocks at
// their natural 22-double column pitch -- with each entry's A and B blocks fetched by two cp.async.bulk
// copies (a 3,872-B block is 16-B aligned and a multiple of 16 B) issued by one lane into a 3-stage
// per-warp ring that completes on the stage's mbarrier, instead of 242 16-B cp.async per block spread over
// the lanes; the warp's runs stream through the ring as one sequence of entries, with every run's
// metadata loaded one run ahead (see the kernel).
constexpr int kSpBulkStages = 3, kSpBulkWarps = 8;

template <int BS>
struct SpBulkCfg {
  using R = SpRunCfg<BS>;
  static_assert(R::TEAM == 1 && R::BB % 2 == 0 && R::P == BS && R::G == 1, "bulk staging: one warp per run, even bs^2");
  static constexpr int STG = R::A_D + R::B_D;  // doubles (even: every stage and B region 16-B aligned)
  static constexpr size_t SMEM = (size_t)kSpBulkWarps * kSpBulkStages * STG * 8;
};

template <int BS>
__global__ void __launch_bounds__(kSpBulkWarps * 32, 1)
    smm_sparse_bulk_kernel(const int32_t* __restrict__ trip, const int64_t* __restrict__ off, int64_t nruns,
                           int64_t kb, const double* __restrict__ A, const double* __restrict__ B,
                           double* __restrict__ C, double alpha, double beta_first) {
  using R = SpRunCfg<BS>;
  using Q = SpBulkCfg<BS>;
  constexpr int MT = R::MT, BB = R::BB, S = kSpBulkStages;
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t mbar[kSpBulkWarps][S];
  __shared__ int smeta[kSpBulkWarps][S][2];  // per stage: C slot of the entry's run, flags (1 first, 2 last)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* ring = sm + (size_t)warp * S * Q::STG;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(&mbar[warp][0]);
  if (lane == 0) {
    for (int i = 0; i < S; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0 + 8 * i) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;  // bit s: parity of stage s's next completion
  int rowm[MT], coln[MT];
#pragma unroll
  for (int i = 0; i < MT; ++i) rowm[i] = coln[i] = i * 8 + g;
  const int64_t nwarps = (int64_t)gridDim.x * kSpBulkWarps;

  // The warp's runs (run = first + i * nwarps) are issued as ONE stream of entries, so the ring stays
  // full across run boundaries; the next run's offsets, C slot and first 32 trip slots are loaded one
  // run ahead, the current run's next 32 slots one window ahead (one per lane, handed to the issuing
  // lane by shuffles): no dependent global load sits between two entries or two runs.
  struct RunPre {  // a run's prefetched metadata (lane l: entry e0 + l's slots)
    int64_t r, e0, e1;
    int a, b, c;
  };
  auto prefetch_run = [&](int64_t r) -> RunPre {
    RunPre p{r, 0, 0, 0, 0, 0};
    while (p.r < nruns) {  // (skip runs without entries)
      p.e0 = off ? off[p.r] : p.r * kb;
      p.e1 = off ? off[p.r + 1] : p.e0 + kb;
      if (p.e1 > p.e0) break;
      p.r += nwarps;
    }
    if (p.r < nruns) {
      p.c = trip[3 * p.e0 + 2];
      if (p.e0 + lane < p.e1) p.a = trip[3 * (p.e0 + lane)], p.b = trip[3 * (p.e0 + lane) + 1];
    }
    return p;
  };
  RunPre cur = prefetch_run((int64_t)blockIdx.x * kSpBulkWarps + warp);
  RunPre nxt = prefetch_run(cur.r + nwarps);
  int64_t ie = cur.e0, w0 = cur.e0;  // issue cursor (entry of run cur.r) and its slot window
  int ca = cur.a, cb = cur.b, na = 0, nb = 0;
  if (cur.r < nruns && cur.e0 + 32 + lane < cur.e1)
    na = trip[3 * (cur.e0 + 32 + lane)], nb = trip[3 * (cur.e0 + 32 + lane) + 1];
  auto issue_next = [&](int si) -> bool {  // warp-uniform
    if (cur.r >= nruns) return false;
    if (ie >= w0 + 32) {
      w0 += 32;
      ca = na;
      cb = nb;
      const int64_t f = w0 + 32 + lane;
      if (f < cur.e1) na = trip[3 * f], nb = trip[3 * f + 1];
    }
    const int sa = __shfl_sync(0xffffffffu, ca, (int)(ie - w0)), sb = __shfl_sync(0xffffffffu, cb, (int)(ie - w0));
    if (lane == 0) {
      smeta[warp][si][0] = cur.c;
      smeta[warp][si][1] = (ie == cur.e0 ? 1 : 0) | (ie + 1 == cur.e1 ? 2 : 0);
      const uint32_t mb = mb0 + 8 * si, dst = ring_s + 8u * (uint32_t)(si * Q::STG);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(2 * BB * 8) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       dst),
                   "l"(A + (int64_t)sa * BB), "r"(BB * 8), "r"(mb)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       dst + 8u * R::A_D),
                   "l"(B + (int64_t)sb * BB), "r"(BB * 8), "r"(mb)
                   : "memory");
    }
    if (++ie == cur.e1) {  // on to the next run: its metadata is in registers; prefetch the one after
      cur = nxt;
      ie = w0 = cur.e0;
      ca = cur.a;
      cb = cur.b;
      na = nb = 0;
      if (cur.r < nruns) {
        if (cur.e0 + 32 + lane < cur.e1)
          na = trip[3 * (cur.e0 + 32 + lane)], nb = trip[3 * (cur.e0 + 32 + lane) + 1];
        nxt = prefetch_run(cur.r + nwarps);
      }
    }
    return true;
  };
  double acc[MT][MT][2], cold[MT][MT][2];  // (cold: the run's C values, loaded at its first entry)
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < MT; ++j) acc[i][j][0] = acc[i][j][1] = cold[i][j][0] = cold[i][j][1] = 0.0;
  int inflight = 0;
#pragma unroll
  for (int i = 0; i < S - 1; ++i) inflight += issue_next(i) ? 1 : 0;
  int si = 0;
  while (inflight > 0) {
    if (issue_next(si == 0 ? S - 1 : si - 1)) ++inflight;  // refill the stage the previous entry used
    {
      const uint32_t mb = mb0 + 8 * si, par = (phase >> si) & 1;
      uint32_t done;
      do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(mb), "r"(par)
            : "memory");
      } while (!done);
      phase ^= 1u << si;
    }
    --inflight;
    const int cslot = smeta[warp][si][0], flags = smeta[warp][si][1];
    if ((flags & 1) && beta_first != 0.0) {  // a run's first entry: its C values load under its products
      const double* cbk = C + (int64_t)cslot * BB;
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < MT; ++ni)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int m = rowm[mi], n = ni * 8 + 2 * t + jj;
            cold[mi][ni][jj] = (m < BS && n < BS) ? cbk[m + n * BS] : 0.0;
          }
    }
    const double* sA = ring + si * Q::STG;  // (m, k) at k*BS + m
    const double* sB = sA + R::A_D;         // (k, n) at n*BS + k
#pragma unroll
    for (int ks = 0; ks < (BS + 3) / 4; ++ks) {
      const int k = 4 * ks + t;
      const bool kok = (BS % 4 == 0) || k < BS;
      double a[MT], b[MT];
#pragma unroll
      for (int mi = 0; mi < MT; ++mi) a[mi] = kok ? sA[k * BS + rowm[mi]] : 0.0;
#pragma unroll
      for (int ni = 0; ni < MT; ++ni) b[ni] = kok ? sB[coln[ni] * BS + k] : 0.0;
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < MT; ++ni) sp_dmma(acc[mi][ni], a[mi], b[ni]);
    }
    __syncwarp();  // every lane is done with stage si (and its metadata) before an issue refills it
    si = si == S - 1 ? 0 : si + 1;
    if (flags & 2) {  // the run's last entry: C_blk = (first ? beta*C : C) + alpha*acc, then a fresh acc
      double* cbk = C + (int64_t)cslot * BB;
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < MT; ++ni)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int m = rowm[mi], n = ni * 8 + 2 * t + jj;
            if (m < BS && n < BS) {
              const double c0 = cold[mi][ni][jj];
              const double ab = __dmul_rn(alpha, acc[mi][ni][jj]);
              cbk[m + n * BS] = beta_first == 1.0 ? __dadd_rn(c0, ab) : beta_first == 0.0 ? ab : fma(beta_first, c0, ab);
            }
            acc[mi][ni][jj] = 0.0;
          }
    }
  }
}

bool sp_bulk_on() {
  static const bool on = [] {
    const char* e = getenv("DBM_SP_BULK");
    return !(e && *e == '0');
  }();
  return on;
}

template <int BS>
cudaError_t launch_sp_bulk(const int32_t* trip, const int64_t* off, int64_t nruns, int64_t kb, const double* A,
                           const double* B, double* C, double alpha, double beta_first, cudaStream_t st) {
  using Q = SpBulkCfg<BS>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(smm_sparse_bulk_kernel<BS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Q::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t ctas = (nruns + kSpBulkWarps - 1) / kSpBulkWarps;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ctas, (int64_t)num_sms()));
  smm_sparse_bulk_kernel<BS><<<grid, kSpBulkWarps * 32, Q::SMEM, st>>>(trip, off, nruns, kb, A, B, C, alpha,
                                                                      beta_first);
  return cudaGetLastError();
}

// Any block size: one CTA per run, one thread per C element, FMA.
__global__ void __launch_bounds__(256) smm_sparse_generic_kernel(int bs, const int32_t* __restrict__ trip,
                                                                 const int64_t* __restrict__ off, int64_t nruns,
                                                                 const double* __restrict__ A,
                                                                 const double* __restrict__ B,
                                                                 double* __restrict__ C, double alpha) {
  extern __shared__ double sg[];
  const int BB = bs * bs;
  double* sA = sg;
  double* sB = sg + BB;
  for (int64_t run = blockIdx.x; run < nruns; run += gridDim.x) {
    const int64_t e0 = off[run], e1 = off[run + 1];
    if (e0 == e1) continue;
    double* c = C + (int64_t)trip[3 * e0 + 2] * BB;
    for (int idx0 = 0; idx0 < BB; idx0 += 256) {
      const int idx = idx0 + threadIdx.x;
      double acc = 0.0;
      for (int64_t e = e0; e < e1; ++e) {
        const double* a = A + (int64_t)trip[3 * e] * BB;
        const double* b = B + (int64_t)trip[3 * e + 1] * BB;
        __syncthreads();
        for (int i = threadIdx.x; i < BB; i += 256) {
          sA[i] = a[i];
          sB[i] = b[i];
        }
        __syncthreads();
        if (idx < BB) {
          const int x = idx % bs, y = idx / bs;
          for (int z = 0; z < bs; ++z) acc = fma(sA[z * bs + x], sB[y * bs + z], acc);
        }
      }
      if (idx < BB) c[idx] = __dadd_rn(c[idx], __dmul_rn(alpha, acc));
    }
  }
}

template <int BS>
cudaError_t launch_sp_run(const int32_t* trip, const int64_t* off, int64_t nruns, int64_t kb, const double* A,
                          const double* B, double* C, double alpha, double beta_first, cudaStream_t st) {
  using Cfg = SpRunCfg<BS>;
  static int per_sm = 0;  // resident CTAs per SM (several for the small block sizes)
  if (per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(smm_sparse_run_kernel<BS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Cfg::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, smm_sparse_run_kernel<BS>, Cfg::WARPS * 32,
                                                      Cfg::SMEM);
    if (e != cudaSuccess) return e;
    per_sm = std::max(1, per_sm);
  }
  const int64_t ctas = (nruns + Cfg::TEAMS - 1) / Cfg::TEAMS;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ctas, (int64_t)num_sms() * per_sm));
  smm_sparse_run_kernel<BS><<<grid, Cfg::WARPS * 32, Cfg::SMEM, st>>>(trip, off, nruns, kb, A, B, C, alpha,
                                                                     beta_first);
  return cudaGetLastError();
}

template <int BS>
cudaError_t launch_sp_tc(const int32_t* trip, const int64_t* off, int64_t nruns, const double* A, const double* B,
                         double* C, double alpha, cudaStream_t st) {
  if (BS == 22) {  // TMA bulk staging when both panels are 16-B aligned (blocks then are too: bs^2 even)
    if (sp_bulk_on() && (((uintptr_t)A | (uintptr_t)B) & 15) == 0)
      return launch_sp_bulk<22>(trip, off, nruns, 0, A, B, C, alpha, 1.0, st);
    return launch_sp_run<BS>(trip, off, nruns, 0, A, B, C, alpha, 1.0, st);
  }
  using Cfg = SpCfg<BS>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(smm_sparse_kernel<BS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t ctas = (nruns + Cfg::TEAMS - 1) / Cfg::TEAMS;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ctas, (int64_t)num_sms()));
  smm_sparse_kernel<BS><<<grid, Cfg::WARPS * 32, Cfg::SMEM, st>>>(trip, off, nruns, A, B, C, alpha);
  return cudaGetLastError();
}

}  // namespace

void launch_fill_sparse(double* arena, int64_t nnz, const int32_t* ij, int bs, int pr, int pc, int r, int c,
                        uint64_t seed, uint32_t mat_id, int kind, cudaStream_t st) {
  const int64_t total = nnz * (int64_t)bs * bs;
  if (total == 0) return;
  auto hmix = [](uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
  };
  const uint64_t key = hmix(seed + 0x9E3779B97F4A7C15ull * ((uint64_t)mat_id + 1ull));
  fill_sparse_kernel<<<sp_grid(total), 256, 0, st>>>(arena, total, ij, bs, pr, pc, r, c, key, kind);
}

cudaError_t launch_sp_densify(const double* arena, const int32_t* ij, int64_t nnz, int bs, int axis, int64_t sel0,
                              int64_t stride, int64_t nk, int64_t other, double* dense, int64_t ld, int layout,
                              cudaStream_t st) {
  const int64_t rows = (axis == 0 ? other : nk) * bs, cols = (axis == 0 ? nk : other) * bs;
  if (rows * cols == 0) return cudaSuccess;
  const int64_t w = layout == 0 ? rows : cols, h = layout == 0 ? cols : rows;
  cudaError_t e = cudaMemset2DAsync(dense, (size_t)ld * 8, 0, (size_t)w * 8, (size_t)h, st);
  if (e != cudaSuccess) return e;
  const int64_t total = nnz * (int64_t)bs * bs;
  if (total) sp_densify_kernel<<<sp_grid(total), 256, 0, st>>>(arena, ij, total, bs, axis, sel0, std::max<int64_t>(stride, 1), nk, dense, ld, layout);
  return cudaGetLastError();
}

void launch_sp_undensify(const double* dense, int64_t ld, int nsplit, int64_t split_stride, const int32_t* ij,
                         int64_t nnz, int bs, double alpha, double beta, double* arena, cudaStream_t st) {
  const int64_t total = nnz * (int64_t)bs * bs;
  if (total == 0) return;
  sp_undensify_kernel<<<sp_grid(total), 256, 0, st>>>(dense, ld, nsplit < 1 ? 1 : nsplit, split_stride, ij, bs, total,
                                                      alpha, beta, arena);
}

void launch_sp_gather(const double* arena, const int32_t* src, int64_t n, int bs, double* out, cudaStream_t st) {
  const int64_t total = n * (int64_t)bs * bs;
  if (total == 0) return;
  sp_gather_kernel<<<sp_grid(total), 256, 0, st>>>(arena, src, total, bs, out);
}

size_t sp_scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int64_t*)nullptr, (int64_t*)nullptr, (int)std::max<int64_t>(n, 1));
  return bytes;
}

cudaError_t launch_sp_stackgen(const int32_t* a_ptr, const int32_t* a_kk, const int32_t* b_ptr, const int32_t* b_kk,
                               const int32_t* b_slot, const int32_t* cmap, int64_t nloc, const int32_t* li,
                               const int32_t* lj, int64_t q0, int64_t n, int64_t* cnt, int64_t* off, void* scan_tmp,
                               size_t scan_bytes, int32_t* trip, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  SpPanels P{a_ptr, a_kk, b_ptr, b_kk, b_slot, cmap, nloc};
  sp_gen_kernel<false><<<sp_grid(n), 256, 0, st>>>(P, li, lj, q0, n, cnt, nullptr, nullptr);
  cudaError_t e = cudaMemsetAsync(cnt + n, 0, sizeof(int64_t), st);
  if (e != cudaSuccess) return e;
  size_t bytes = scan_bytes;
  e = cub::DeviceScan::ExclusiveSum(scan_tmp, bytes, cnt, off, (int)(n + 1), st);
  if (e != cudaSuccess) return e;
  sp_gen_kernel<true><<<sp_grid(n), 256, 0, st>>>(P, li, lj, q0, n, nullptr, off, trip);
  return cudaGetLastError();
}

// Block sizes with a compiled DMMA per-run instance besides 22 and 64 (LIBCUSMM-style: one kernel per size,
// P:173-177).  Used by the dense blocked path (uniform runs, off == nullptr) and the sparse path.
#define DBM_RUN_SIZES(X) X(4) X(5) X(6) X(8) X(9) X(13) X(16) X(23) X(26) X(32)

bool smm_has_run_path(int bs) {
  switch (bs) {
#define DBM_CASE(n) case n:
    DBM_RUN_SIZES(DBM_CASE)
#undef DBM_CASE
    return true;
    default:
      return false;
  }
}

cudaError_t launch_smm_run(int bs, const int32_t* trip, const int64_t* off, int64_t nruns, int64_t kb,
                           const double* A, const double* B, double* C, double alpha, double beta_first,
                           cudaStream_t st) {
  if (nruns <= 0) return cudaSuccess;
  switch (bs) {
#define DBM_CASE(n) \
  case n:           \
    return launch_sp_run<n>(trip, off, nruns, kb, A, B, C, alpha, beta_first, st);
    DBM_RUN_SIZES(DBM_CASE)
#undef DBM_CASE
    default:
      return cudaErrorNotSupported;
  }
}

cudaError_t launch_smm_sparse(int bs, const int32_t* trip, const int64_t* off, int64_t nruns, const double* A,
                              const double* B, double* C, double alpha, cudaStream_t st) {
  if (nruns <= 0) return cudaSuccess;
  if (bs == 22) return launch_sp_tc<22>(trip, off, nruns, A, B, C, alpha, st);
  if (bs == 64) return launch_sp_tc<64>(trip, off, nruns, A, B, C, alpha, st);
  if (smm_has_run_path(bs)) return launch_smm_run(bs, trip, off, nruns, 0, A, B, C, alpha, 1.0, st);
  const size_t smem = 2 * (size_t)bs * bs * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(smm_sparse_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const unsigned grid = (unsigned)std::min<int64_t>(nruns, (int64_t)num_sms() * 8);
  smm_sparse_generic_kernel<<<grid, 256, smem, st>>>(bs, trip, off, nruns, A, B, C, alpha);
  return cudaGetLastError();
}

}  // namespace dbm

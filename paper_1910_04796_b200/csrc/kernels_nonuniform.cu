// Kernels for matrices with non-uniform block sizes (SPEC S:25-26 row_sizes /
// col_sizes; the paper's (m x k) A blocks times (k x n) B blocks, §II).  Reading R16
// (DESIGN.md §3): a rank's arena holds its stored blocks in local CSR order, each column-major, back to
// back; the host keeps every slot's element offset and shape (NUBlk).
//
//   nu_fill_kernel     the counter generator at global element coordinates
//   nu_copy_kernel     block <-> dense panel copies from a task list: densify B (K-major columns) and
//                      undensify C with alpha / beta (column-major); nu_copy_a_kernel densify A (K-major
//                      rows, a transpose through a shared tile)
//   nu_pack_kernel     whole-block gathers into packed Cannon panels (blocked path)
//   nu_smm_kernel      the blocked path's small-block products of mixed (m, n, k): one CTA per C-block
//                      run, entry groups staged by TMA bulk copies into a 3-stage mbarrier ring, K split
//                      over the warps, FP64 DMMA (mma.sync m8n8k4) on 8 x 8 subtiles
#include <algorithm>

#include "dbm_internal.h"

namespace dbm {

namespace {

__device__ __forceinline__ uint64_t nu_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

__global__ void nu_fill_kernel(double* __restrict__ arena, const NUBlk* __restrict__ blk, int64_t nslots, uint64_t key,
                               int kind) {
  for (int64_t s = blockIdx.x; s < nslots; s += gridDim.x) {
    const NUBlk b = blk[s];
    const int64_t n = (int64_t)b.rows * b.cols;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
      const int64_t y = e / b.rows, x = e - y * b.rows;
      const uint64_t gi = (uint64_t)(b.r0 + x), gj = (uint64_t)(b.c0 + y);
      const uint64_t bits = nu_mix64(key ^ nu_mix64((gi << 32) ^ gj));
      double v;
      if (kind == 1) {
        v = (double)((int)((bits >> 32) % 5u) - 2);
      } else {
        const double u = __dmul_rn((double)(bits >> 11), 0x1.0p-53);
        v = __dsub_rn(__dmul_rn(2.0, u), 1.0);
      }
      arena[b.off + e] = v;
    }
  }
}

// mode 0: A block (rows m x cols k) -> K-major rows: dense[(row0 + x) * ld + col0 + y]
// mode 1: B block (rows k x cols n) -> K-major columns: dense[(col0 + y) * ld + row0 + x]
// mode 2: C block <- column-major dense: blk = alpha * dense[(col0 + y) * ld + row0 + x] + beta * blk
//         (two roundings, no FMA, as the uniform undensify; beta == 0: blk not read)
constexpr int kNuTile = 64 * 65;  // shared transpose tile (doubles): blocks up to 64 x 64, rows padded by one

// One CTA (8 warps) per task.  Modes 1 and 2 are contiguous in x (down a block column) on both sides: a
// flat loop over the block's elements (32-bit index math), no shared memory.
__global__ void __launch_bounds__(256) nu_copy_kernel(const NUTask* __restrict__ tasks, int64_t ntasks,
                                                      double* __restrict__ arena, double* __restrict__ dense,
                                                      int64_t ld, int mode, double alpha, double beta) {
  for (int64_t t = blockIdx.x; t < ntasks; t += gridDim.x) {
    const NUTask k = tasks[t];
    const int rows = k.rows, n = k.rows * k.cols;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      const int y = e / rows, x = e - y * rows;
      if (mode == 1) {
        dense[(k.col0 + y) * ld + k.row0 + x] = arena[k.src + e];
      } else {
        const double d = __dmul_rn(alpha, dense[(k.col0 + y) * ld + k.row0 + x]);
        double* p = arena + k.src + e;
        *p = beta == 0.0 ? d : __dadd_rn(d, __dmul_rn(beta, *p));
      }
    }
  }
}

// Mode 0 transposes (the dense row is contiguous in y): blocks up to 64 x 64 go through a shared tile, read
// down the block columns and written along the dense rows, so both sides stay coalesced; larger blocks
// copy directly.
__global__ void __launch_bounds__(256) nu_copy_a_kernel(const NUTask* __restrict__ tasks, int64_t ntasks,
                                                        const double* __restrict__ arena, double* __restrict__ dense,
                                                        int64_t ld) {
  __shared__ double tile[kNuTile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int64_t t = blockIdx.x; t < ntasks; t += gridDim.x) {
    const NUTask k = tasks[t];
    const int rows = k.rows, cols = k.cols;
    if (rows <= 64 && cols <= 64) {
      const int pitch = cols + 1;
      for (int y = warp; y < cols; y += nw)
        for (int x = lane; x < rows; x += 32) tile[x * pitch + y] = arena[k.src + (int64_t)y * rows + x];
      __syncthreads();
      for (int x = warp; x < rows; x += nw)
        for (int y = lane; y < cols; y += 32) dense[(k.row0 + x) * ld + k.col0 + y] = tile[x * pitch + y];
      __syncthreads();  // the next task's tile
      continue;
    }
    const int n = rows * cols;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      const int y = e / rows, x = e - y * rows;
      dense[(k.row0 + x) * ld + k.col0 + y] = arena[k.src + e];
    }
  }
}

__global__ void nu_pack_kernel(const NUPack* __restrict__ tasks, int64_t ntasks, const double* __restrict__ src,
                               double* __restrict__ dst) {
  for (int64_t t = blockIdx.x; t < ntasks; t += gridDim.x) {
    const NUPack k = tasks[t];
    for (int64_t e = threadIdx.x; e < k.n; e += blockDim.x) dst[k.dst + e] = src[k.src + e];
  }
}

__device__ __forceinline__ void nu_dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

constexpr int kNuWarps = 4;
constexpr int kNuStages = 3;
constexpr int kNuZero = 64;  // doubles of zeros past the ring (the k tail's operand)

__device__ __forceinline__ void nu_mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void nu_mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void nu_mbar_arrive_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void nu_mbar_wait(uint32_t a, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void nu_bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

// Stage layout (doubles), kp = kcap rounded up to 4, ne = the most entries a group holds: A region
// kp mmax + 4 ne + 4 | B region kp nmax + 4 ne + 4 | k table kp int4 | the group's K (2 doubles, keeps
// every region 16-B aligned).
__host__ __device__ inline int nu_a_region(int kp, int mmax, int ne) { return kp * mmax + 4 * ne + 4; }
__host__ __device__ inline int nu_stage_doubles(int kp, int mmax, int nmax, int ne) {
  return nu_a_region(kp, mmax, ne) + nu_a_region(kp, nmax, ne) + 2 * kp + 2;
}
__host__ __device__ inline int nu_group_entries(int kp) { return kp < kNuGroupMaxEntries ? kp : kNuGroupMaxEntries; }

// A warp's k-loop over one staged group for a run of R x Cn subtiles (all of them: one row group, WR = 1):
// per k-step one k-table entry, R A and Cn B fragments, R Cn DMMAs, no shape branches.
template <int R, int Cn, int S>
__device__ __forceinline__ void nu_kloop(double (&acc)[S][S][2], const int4* zt, int K, int z_first, int z_step,
                                         int t, const int (&rowc)[S], const int (&colc)[S], const double* nsm) {
  for (int z0 = z_first; z0 < K; z0 += z_step) {
    const int4 zi = zt[z0 + t];  // (z0 + t < kp: the table covers the tail)
    const double* ap = nsm + zi.x;
    const double* bp = nsm + zi.y;
    double av[R], bv[Cn];
#pragma unroll
    for (int i = 0; i < R; ++i) av[i] = ap[rowc[i]];
#pragma unroll
    for (int j = 0; j < Cn; ++j) bv[j] = bp[colc[j] * zi.z];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int j = 0; j < Cn; ++j) nu_dmma(acc[i][j], av[i], bv[j]);
  }
}

// One CTA per run (C block, m x n <= 64 x 64): acc(c) = sum over the run's entries of A_blk (m x k_e) *
// B_blk (k_e x n), then C = (first ? beta*C : C) + alpha*acc.  The entries are taken in GROUPS
// (host-computed from the k sizes, the same for every run of the step: group g = entries [gbeg[g],
// gbeg[g+1]), their k sizes summing to at most kcap, at most kNuGroupMaxEntries of them), entry e at k
// offset kofs[e] inside its group:
//   * staging (TMA bulk copies into a 3-stage ring): lane l of warp w owns entry w + 4 l of the group; its
//     metadata -- k, k offset, trip slots, then A and B block addresses -- is loaded in two levels, two
//     and one groups ahead (each dependent lookup's latency hides under a group's compute), then the
//     lane issues one cp.async.bulk per operand block, completing on the stage's mbarrier (every thread
//     arrives once per group, the data lanes with their bytes).  Blocks of odd element counts sit at any
//     8-B offset, so each copy takes the 16-B-aligned superset of its block (at most one extra double on
//     either side, never outside the block's 16-B granules) into a 16-B-aligned slot with room for it;
//     a k table (written lane-parallel before the lanes arrive, so the stage's mbarrier publishes it with
//     the data) gives, for every k index z of the group, the shared offsets of A(0, z) and B(z, 0) and
//     the B column stride k_e.  No per-element staging instruction, no L1 traffic, one CTA barrier per
//     group (the ring's reuse);
//   * compute: the warps split the group's K WK ways (k-step ks to k-group ks mod WK) and the subtile rows
//     WR ways (WR WK = 4 warps); a warp holds SI subtile rows x all S subtile columns of the C block (8 x 8
//     DMMA subtiles; blocks up to 32: S = 4, WR = 1, WK = 4; up to 64: S = 8, WR = 2, WK = 2, so the
//     accumulators stay at 64 registers) and per k-step loads its A and B fragments once for all its DMMAs
//     -- every warp busy whatever the block shape; for blocks up to 32 the k-loop is instantiated per
//     subtile shape (1..4 x 1..4, a switch per group), so it issues only the run's fragments and DMMAs.  Fragment rows >= m and columns >= n read the block's
//     last row / column (clamped offsets, computed once per run): they only feed accumulator rows /
//     columns that are never stored.  k indices past the group's K read a zero region (A and B), so the
//     tail adds exact zeros;
//   * epilogue: the WK k-groups' partial C blocks meet in shared memory and are summed in k-group order
//     (deterministic), then scaled into C.
// (blocks up to 32: the ring's shared memory allows 4 resident CTAs per SM, so the register budget is
// pinned to 4 x 128 threads; measured: 2 stages at 5 CTAs and 4 stages at 3 CTAs both lose, 7.7 vs 9.1
// TFLOP/s at 3,960^3)
template <int S, int WR>
__global__ void __launch_bounds__(kNuWarps * 32, S == 4 ? 4 : 1)
    nu_smm_kernel(const int32_t* __restrict__ trip, int64_t nruns, int64_t kb, const double* __restrict__ A,
                  const int64_t* __restrict__ aoff, const double* __restrict__ B, const int64_t* __restrict__ boff,
                  const int32_t* __restrict__ kdim, const int32_t* __restrict__ kofs, const int32_t* __restrict__ gbeg,
                  int ngroups, double* __restrict__ C, const NUBlk* __restrict__ cblk, int kcap, int mmax_pad,
                  int nmax_pad, double alpha, double beta_first) {
  extern __shared__ __align__(16) double nsm[];
  __shared__ __align__(8) uint64_t nmb[kNuStages];  // one per stage: every thread arrives, data lanes with tx
  constexpr int WK = kNuWarps / WR, SI = S / WR;
  const int kp = (kcap + 3) & ~3, ne = nu_group_entries(kp);
  const int a_reg = nu_a_region(kp, mmax_pad, ne), b_reg = nu_a_region(kp, nmax_pad, ne);
  const int st_d = nu_stage_doubles(kp, mmax_pad, nmax_pad, ne);
  // past the ring and the epilogue's partial C blocks (zeroed once, never overwritten)
  const int zero_off = max(kNuStages * st_d, kNuWarps * mmax_pad * nmax_pad);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int rh = warp % WR, kg = warp / WR, i0 = rh * SI;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(nsm);
  const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(&nmb[0]);
  for (int i = threadIdx.x; i < kNuZero; i += blockDim.x) nsm[zero_off + i] = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kNuStages; ++i) nu_mbar_init(mb0 + 8 * i, kNuWarps * 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  uint32_t phase = 0;  // bit s: the parity of stage s's next completion
  for (int64_t run = blockIdx.x; run < nruns; run += gridDim.x) {
    const int32_t* rt = trip + 3 * run * kb;
    const NUBlk cb = cblk[rt[2]];
    const int m = cb.rows, n = cb.cols;
    const int sm_ = (m + 7) / 8, sn = (n + 7) / 8;
    int rowc[SI], colc[S];  // clamped fragment rows / columns
#pragma unroll
    for (int i = 0; i < SI; ++i) rowc[i] = min(8 * (i0 + i) + g, m - 1);
#pragma unroll
    for (int j = 0; j < S; ++j) colc[j] = min(8 * j + g, n - 1);
    // A group's metadata in two levels, a group apart: level 1 (this lane's entry e = gbeg + warp + 4 lane:
    // k, k offset, the trip's A / B slots; the group's K), then level 2 (the blocks' addresses, from the
    // slot offset tables).  Group g + 4's level 1 and g + 3's level 2 are in flight while group g computes,
    // so each dependent lookup has a whole group's compute to land.
    bool l1_has = false, pm_has = false;
    int l1_k = 0, l1_ko = 0, l1_K = 0, l1_sa = 0, l1_sb = 0, pm_k = 0, pm_ko = 0, pm_K = 0;
    const double *pm_a = A, *pm_b = B;
    auto fetch1 = [&](int grp) {
      l1_has = false;
      if (grp < ngroups) {
        const int gb = gbeg[grp], ge = gbeg[grp + 1];
        l1_K = kofs[ge - 1] + kdim[ge - 1];
        const int e = gb + warp + kNuWarps * lane;
        if (e < ge) {
          l1_has = true;
          l1_k = kdim[e];
          l1_ko = kofs[e];
          l1_sa = rt[3 * e];
          l1_sb = rt[3 * e + 1];
        }
      }
    };
    auto fetch2 = [&]() {
      pm_has = l1_has;
      pm_k = l1_k;
      pm_ko = l1_ko;
      pm_K = l1_K;
      if (l1_has) {
        pm_a = A + aoff[l1_sa];
        pm_b = B + boff[l1_sb];
      }
    };
    auto stage = [&](int grp, int buf) {  // group grp's blocks -> stage buf (nothing past the end)
      if (grp >= ngroups) return;
      const int so = buf * st_d;
      int4* zt = reinterpret_cast<int4*>(nsm + so + a_reg + b_reg);
      const uint32_t mb = mb0 + 8 * buf;
      if (warp == kNuWarps - 1) {  // the k tail up to a multiple of 4: the zero region, stride 0; the K
        if (lane < 4 && pm_K + lane < kp) zt[pm_K + lane] = make_int4(zero_off, zero_off, 0, 0);
        if (lane == 0) reinterpret_cast<int*>(zt + kp)[0] = pm_K;
      }
      // the warp's entries are its lanes 0 .. c-1 (typically one or two warps of the four hold any)
      const int c = __popc(__ballot_sync(0xffffffffu, pm_has));
      if (c > 0) {
        const int er = warp + kNuWarps * lane;  // this lane's entry's index in its group
        const uintptr_t as = reinterpret_cast<uintptr_t>(pm_a), bs = reinterpret_cast<uintptr_t>(pm_b);
        const int ha = (int)((as >> 3) & 1), hb = (int)((bs >> 3) & 1);  // doubles before the block
        const int ao = so + ((pm_ko * m + 4 * er + 1) & ~1);
        const int bo = so + a_reg + ((pm_ko * n + 4 * er + 1) & ~1);
        for (int i = 0; i < c; ++i) {  // the k table, lane-parallel
          const int k = __shfl_sync(0xffffffffu, pm_k, i), ko = __shfl_sync(0xffffffffu, pm_ko, i);
          const int a0 = __shfl_sync(0xffffffffu, ao + ha, i), b0 = __shfl_sync(0xffffffffu, bo + hb, i);
          for (int z = lane; z < k; z += 32) zt[ko + z] = make_int4(a0 + z * m, b0 + z, k, 0);
        }
        // every lane arrives after its table stores (release; the consumers' wait acquires them)
        if (pm_has) {
          const uint32_t na = (uint32_t)((ha + m * pm_k) * 8 + 15) & ~15u;
          const uint32_t nb = (uint32_t)((hb + pm_k * n) * 8 + 15) & ~15u;
          nu_mbar_arrive_tx(mb, na + nb);
          nu_bulk_g2s(sbase + 8 * ao, reinterpret_cast<const void*>(as & ~(uintptr_t)15), na, mb);
          nu_bulk_g2s(sbase + 8 * bo, reinterpret_cast<const void*>(bs & ~(uintptr_t)15), nb, mb);
        } else {
          nu_mbar_arrive(mb);
        }
      } else {
        nu_mbar_arrive(mb);
      }
    };
    double acc[SI][S][2];
#pragma unroll
    for (int i = 0; i < SI; ++i)
#pragma unroll
      for (int j = 0; j < S; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int s = 0; s < kNuStages - 1; ++s) {
      fetch1(s);
      fetch2();
      stage(s, s);
    }
    fetch1(kNuStages - 1);
    fetch2();
    fetch1(kNuStages);
    for (int grp = 0; grp < ngroups; ++grp) {
      stage(grp + kNuStages - 1, (grp + kNuStages - 1) % kNuStages);
      fetch2();                   // group grp + 3's addresses
      fetch1(grp + kNuStages + 1);  // group grp + 4's entries (both in flight during this group's compute)
      const int buf = grp % kNuStages;
#pragma unroll
      nu_mbar_wait(mb0 + 8 * buf, (phase >> buf) & 1);
      phase ^= 1u << buf;
      const int4* zt = reinterpret_cast<const int4*>(nsm + buf * st_d + a_reg + b_reg);
      const int K = reinterpret_cast<const int*>(zt + kp)[0];  // the group's concatenated K
      if constexpr (WR == 1) {  // blocks up to 32 x 32: the k-loop specialised on the run's subtile shape
        const int shape = (sm_ - 1) * S + (sn - 1);
#define NU_K(R_, C_)                                                        \
  case (R_ - 1) * S + (C_ - 1):                                             \
    nu_kloop<R_, C_, S>(acc, zt, K, 4 * kg, 4 * WK, t, rowc, colc, nsm); \
    break;
        switch (shape) {
          NU_K(1, 1) NU_K(1, 2) NU_K(1, 3) NU_K(1, 4)
          NU_K(2, 1) NU_K(2, 2) NU_K(2, 3) NU_K(2, 4)
          NU_K(3, 1) NU_K(3, 2) NU_K(3, 3) NU_K(3, 4)
          NU_K(4, 1) NU_K(4, 2) NU_K(4, 3) NU_K(4, 4)
          default: break;
        }
#undef NU_K
      } else {
        for (int z0 = 4 * kg; z0 < K; z0 += 4 * WK) {
          const int4 zi = zt[z0 + t];  // (z0 + t < kp: the table covers the tail)
          const double* ap = nsm + zi.x;
          const double* bp = nsm + zi.y;
          double av[SI], bv[S];
#pragma unroll
          for (int i = 0; i < SI; ++i) av[i] = ap[rowc[i]];
#pragma unroll
          for (int j = 0; j < S; ++j) bv[j] = bp[colc[j] * zi.z];
#pragma unroll
          for (int i = 0; i < SI; ++i) {
            if (i0 + i >= sm_) break;
#pragma unroll
            for (int j = 0; j < S; ++j) {
              if (j >= sn) break;
              nu_dmma(acc[i][j], av[i], bv[j]);
            }
          }
        }
      }
      __syncthreads();  // stage buf is refilled two groups on
    }
    // epilogue: subtile (i0 + i, j), lane (g, t) holds k-group kg's partial C(8(i0+i) + g, 8j + 2t + jj)
    const int mp = 8 * sm_, np = 8 * sn;
    double* red = nsm;
#pragma unroll
    for (int i = 0; i < SI; ++i) {
      if (i0 + i >= sm_) break;
#pragma unroll
      for (int j = 0; j < S; ++j) {
        if (j >= sn) break;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
          red[(kg * np + 8 * j + 2 * t + jj) * mp + 8 * (i0 + i) + g] = acc[i][j][jj];
      }
    }
    __syncthreads();
    for (int y = warp; y < n; y += kNuWarps)
      for (int x = lane; x < m; x += 32) {
        double v = red[y * mp + x];
#pragma unroll
        for (int w = 1; w < WK; ++w) v += red[(w * np + y) * mp + x];
        double* p = C + cb.off + (int64_t)y * m + x;
        v *= alpha;
        *p = beta_first == 0.0 ? v : beta_first * *p + v;
      }
    // the next run's bulk copies (async proxy) overwrite what the epilogue wrote and read (generic proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
}

unsigned nu_grid(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(n, (int64_t)num_sms() * 16)); }

}  // namespace

void launch_nu_fill(double* arena, const NUBlk* blk, int64_t nslots, uint64_t seed, uint32_t mat_id, int kind,
                    cudaStream_t st) {
  if (nslots <= 0) return;
  auto hmix = [](uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
  };
  const uint64_t key = hmix(seed + 0x9E3779B97F4A7C15ull * ((uint64_t)mat_id + 1ull));
  nu_fill_kernel<<<nu_grid(nslots), 256, 0, st>>>(arena, blk, nslots, key, kind);
}

void launch_nu_copy(const NUTask* tasks, int64_t ntasks, double* arena, double* dense, int64_t ld, int mode,
                    double alpha, double beta, cudaStream_t st) {
  if (ntasks <= 0) return;
  if (mode == 0)
    nu_copy_a_kernel<<<nu_grid(ntasks), 256, 0, st>>>(tasks, ntasks, arena, dense, ld);
  else
    nu_copy_kernel<<<nu_grid(ntasks), 256, 0, st>>>(tasks, ntasks, arena, dense, ld, mode, alpha, beta);
}

void launch_nu_pack(const NUPack* tasks, int64_t ntasks, const double* src, double* dst, cudaStream_t st) {
  if (ntasks <= 0) return;
  nu_pack_kernel<<<nu_grid(ntasks), 256, 0, st>>>(tasks, ntasks, src, dst);
}

size_t nu_smm_smem(int kcap, int mmax, int nmax) {
  const int kp = (kcap + 3) & ~3, mp = (mmax + 7) & ~7, np = (nmax + 7) & ~7;
  const size_t ring = (size_t)kNuStages * nu_stage_doubles(kp, mp, np, nu_group_entries(kp));
  // (the epilogue's WK partial C blocks, at most 4 mp np doubles, reuse the ring; the zero region follows it)
  return (std::max(ring, (size_t)kNuWarps * mp * np) + kNuZero) * 8;
}

cudaError_t launch_nu_smm(const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const int64_t* aoff,
                          const double* B, const int64_t* boff, const int32_t* kdim, const int32_t* kofs,
                          const int32_t* gbeg, int ngroups, double* C, const NUBlk* cblk, int kcap, int mmax, int nmax,
                          double alpha, double beta_first, cudaStream_t st) {
  if (nruns <= 0 || kb <= 0) return cudaSuccess;
  if (mmax > 64 || nmax > 64) return cudaErrorInvalidValue;  // the host checks: C blocks up to 64 x 64
  const size_t smem = nu_smm_smem(kcap, mmax, nmax);
  const bool small = mmax <= 32 && nmax <= 32;  // 4 x 4 subtiles per warp, else 8 x 8
  auto kern = small ? nu_smm_kernel<4, 1> : nu_smm_kernel<8, 2>;
  static size_t attr[2] = {0, 0};
  if (smem > 48 * 1024 && smem > attr[small]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[small] = smem;
  }
  kern<<<(unsigned)std::min<int64_t>(nruns, (int64_t)num_sms() * 32), kNuWarps * 32, smem, st>>>(
      trip, nruns, kb, A, aoff, B, boff, kdim, kofs, gbeg, ngroups, C, cblk, kcap, (mmax + 7) & ~7, (nmax + 7) & ~7,
      alpha, beta_first);
  return cudaGetLastError();
}

}  // namespace dbm

// dgemm_f64 — the densified path's local multiply (§III, the cublasDgemm role; "better
// performance by using the well-optimized cuBLAS library ... for multiplication of large blocks").
//
// B200 design: FP64 has no tcgen05 kind on sm_100a, so the tensor path is
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), which shares the FP64 pipe with DFMA (measured 37.1 vs
// 36.6 TFLOP/s, profiles/r01_fp64_peaks.jsonl).  Operands are both K-major ("TN"), staged by TMA
// (cp.async.bulk.tensor.2d, SWIZZLE_128B, 16 x 128 boxes) into a STAGES-deep shared-memory ring
// guarded by mbarriers; one producer warp issues the TMA, 8 consumer warps each own a 64 x 32
// slice of the 128 x 128 C tile (64 FP64 accumulators per thread) and read fragments with
// conflict-free LDS.64 thanks to the 128B swizzle.  Split-K with a fixed-order reduction covers
// thin C (rectangular configs).  Bound: FP64 pipe; 2*M*N*K flops per launch.
#include <algorithm>
#include <cstdlib>

#include "dbm_internal.h"

namespace dbm {

namespace {

constexpr int BK = 16;
constexpr int kConsumerWarps = 8;
// 12 warps = three warpgroups: two of consumers, one whose first warp is the TMA producer.  The launch
// gives every thread 168 registers (65,536 / 384); the producer warpgroup then releases down to 40 and the
// consumers raise to 232 (setmaxnreg), so the 64 FP64 accumulators, the fragments and the ring state of a
// consumer fit without spilling (at a flat 168 the k-loop spilled its stage / phase / base registers).
constexpr int kThreads = (kConsumerWarps + 4) * 32;
constexpr int kRegsConsumer = 232, kRegsProducer = 40;
// CTA tile BM x BN in {128, 64}^2 (the host picks the one that wastes the least padding for the
// block-multiple shapes of the configs, e.g. 704 = 5.5 x 128); ~192 KB of stages in every case.
template <int BM, int BN>
struct Tile {
  static constexpr int kStageA = BM * BK * 8;
  static constexpr int kStageB = BN * BK * 8;
  static constexpr int kStage = kStageA + kStageB;
  static constexpr int STAGES = (196608 / kStage) > 12 ? 12 : (196608 / kStage);
  static constexpr size_t kSmem = (size_t)STAGES * kStage + 2 * STAGES * 8 + 1024;
  static constexpr int MI = BM / 16, NI = BN / 32;  // 8x8 subtiles per consumer warp (2 x 4 warps)
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
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
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                            uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
          "r"(dst),
      "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

template <int BM, int BN, bool A_BLK>
__global__ void __launch_bounds__(kThreads, 1)
    dgemm_tn_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                    int k_tiles_total, int k_tiles_per_split, int nsplit, int tiles_m, int tiles_n,
                    double* __restrict__ C,
                    int64_t ldc, double alpha, double beta, double* __restrict__ partial,
                    unsigned* __restrict__ wave_sync, int sync_kt, int sync_rounds, int slack, int b_blocks) {
  using T = Tile<BM, BN>;
  constexpr int STAGES = T::STAGES, kStage = T::kStage, kStageA = T::kStageA, MI = T::MI, NI = T::NI;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + STAGES * kStage);
  uint64_t* empty = full + STAGES;

  // Persistent: CTA b takes work items b, b + grid, ...  All items have equal work, so the CTAs move
  // through their item lists in lock-step and each "wave" of grid consecutive items runs together.
  // Items are rasterised in groups of GROUP tile-rows (column-major inside a group), so one wave
  // is a ~12 x 12 patch of C tiles that streams ~24 A/B panels through L2 at the same k.
  constexpr int GROUP = 12;
  const int ntiles = tiles_m * tiles_n;
  const int nitems = ntiles * nsplit;
  auto item_coords = [&](int item, int& tm, int& tn, int& split) {
    split = item / ntiles;
    const int tile = item - split * ntiles;
    const int span = GROUP * tiles_n;
    const int first_m = (tile / span) * GROUP;
    const int gsize = min(tiles_m - first_m, GROUP);
    tm = first_m + (tile % span) % gsize;
    tn = (tile % span) / gsize;
  };
  auto item_k = [&](int split, int& kt0, int& nkt) {
    kt0 = split * k_tiles_per_split;
    nkt = max(0, min(k_tiles_total, kt0 + k_tiles_per_split) - kt0);
  };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(su32(&full[s]), 1);
      mbar_init(su32(&empty[s]), kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= kConsumerWarps) {  // ---------------- producer warpgroup: warp 8 issues the TMA, 9-11 idle
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsProducer));
    if (warp == kConsumerWarps && lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      unsigned epoch = 0;
      int round = 0;
      for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++round) {
        int tm, tn, split, kt0, nkt;
        item_coords(item, tm, tn, split);
        item_k(split, kt0, nkt);
        for (int kt = 0; kt < nkt; ++kt) {
          // Fuzzy wave barrier (cooperative launch only): every sync_kt k-tiles of the rounds every CTA
          // runs, a producer announces its arrival and waits only until every CTA has reached the
          // sync point `slack` intervals back.  CTAs then never drift more than (slack + 1) intervals
          // apart in k, so one wave's A/B panel slices stay in L2 (read once from HBM), while a CTA
          // stalls only if it gets a whole interval ahead of the slowest one.
          if (wave_sync != nullptr && round < sync_rounds && kt % sync_kt == 0) {
            ++epoch;
            atomicAdd(wave_sync, 1u);
            const unsigned target = epoch > (unsigned)slack ? (epoch - (unsigned)slack) * gridDim.x : 0u;
            unsigned seen;
            do {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(wave_sync) : "memory");
            } while (seen < target);
          }
          mbar_wait(su32(&empty[stage]), phase ^ 1);
          const uint32_t fb = su32(&full[stage]);
          mbar_expect_tx(fb, kStage);
          const uint32_t dst = su32(smem + stage * kStage);
          if (A_BLK) {  // A read in place from 64 x 64 blocks: 4 boxes of (16 m, 16 k) x BM/64 block rows
            const int k = (kt0 + kt) * BK;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              tma_load_4d(dst + q * (BM / 64) * 2048, &tmA, 16 * q, k & 63, k >> 6, tm * (BM / 64), fb);
          } else {
            tma_load_2d(dst, &tmA, (kt0 + kt) * BK, tm * BM, fb);
          }
          if (b_blocks) {  // B read in place from 64 x 64 blocks: (k in block, n in block, block col, block row)
            const int k = (kt0 + kt) * BK;
            tma_load_4d(dst + kStageA, &tmB, k & 63, 0, tn * (BN / 64), k >> 6, fb);
          } else {
            tma_load_2d(dst + kStageA, &tmB, (kt0 + kt) * BK, tn * BN, fb);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers: warp (wm, wn) owns rows wm*BM/2.., cols wn*BN/4..
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsConsumer));
  const int wm = warp >> 2, wn = warp & 3;

  // Fragment addressing inside a 128-B-swizzled [rows][16 doubles] box: element (row, k) lives at
  // row*128 + (((k>>1) ^ (row&7)) << 4) + ((k&1) << 3), and row&7 == g = lane>>2 for every fragment
  // row.  A 64-bit LDS is served per half-warp (g = 0..3 / 4..7), so the MMA k-slot t = lane&3 of
  // k-step ks reads k = 2*ks + (t&1) + 8*(t>>1): the 16 lanes of a half-warp then hit 16 distinct
  // 8-byte bank pairs (k ^ 2g distinct), one wavefront per half-warp.  Any fixed k permutation
  // shared by A and B leaves the product unchanged (the four k-steps cover k = 0..15).
  const int g = lane >> 2, t = lane & 3;
  const uint32_t a_row = (uint32_t)(wm * (BM / 2) + g) * 128u;
  const uint32_t b_row = (uint32_t)(wn * (BN / 4) + g) * 128u;
  // k>>1 = ks + 4 (t>>1) with ks < 4, so ((k>>1) ^ g) = ks ^ G: the per-ks offsets are one XOR away from
  // two lane constants (cheaper than four live registers under the 168-register cap)
  const uint32_t G = (uint32_t)(g ^ (4 * (t >> 1))), kodd = (uint32_t)(t & 1) << 3;
  // A_BLK: the A tile is 4 boxes q (m_in chunks of 16) of [BM/64 block rows][16 k][16 m] doubles, rows of
  // 128 B swizzled by (row & 7) = (k & 7).  Element (m_local, k): li = m_local / 64, q = (m_local % 64) / 16,
  // at q * (BM/64) * 2048 + (li * 16 + k) * 128 + ((((m % 16) >> 1) ^ (k & 7)) << 4) + ((m & 1) << 3).  With
  // k = 2 ks + kt, kt = (t & 1) + 8 (t >> 1), the lane constants are the row base and the low m bits.
  const int kt_a = (t & 1) + 8 * (t >> 1);
  const int m_warp = wm * (BM / 2);  // a warp's first tile row: a multiple of 32
  const uint32_t a_blk_row = (uint32_t)((m_warp >> 6) * 16 + kt_a) * 128u + (uint32_t)((g & 1) << 3);

  int stage = 0;
  uint32_t phase = 0;
  const uint32_t smem_base = su32(smem);
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
  int nkt;
  {
    int tm_, tn_, split_, kt0_;
    item_coords(item, tm_, tn_, split_);
    item_k(split_, kt0_, nkt);
  }
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int kt = 0; kt < nkt; ++kt) {
    mbar_wait(su32(&full[stage]), phase);
    const uint32_t sA = smem_base + stage * kStage;
    const uint32_t sB = sA + kStageA;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const uint32_t koff = ((G ^ (uint32_t)ks) << 4) | kodd;
      double a[MI], b[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        if (A_BLK) {
          const int m_in = (m_warp & 63) + mi * 8;  // + g (in the lane constants)
          const uint32_t x = (uint32_t)((((m_in & 15) >> 1) + (g >> 1)) ^ ((2 * ks + (t & 1)) & 7));
          a[mi] = lds64(sA + (uint32_t)(m_in >> 4) * (BM / 64) * 2048u + a_blk_row + (uint32_t)(2 * ks) * 128u + (x << 4));
        } else {
          a[mi] = lds64(sA + a_row + mi * 1024 + koff);
        }
      }
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) b[ni] = lds64(sB + b_row + ni * 1024 + koff);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(su32(&empty[stage]));
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }

  // ---------------- epilogue (C column-major); the tile coordinates are recomputed here so they are not
  // live (spilled) across the k-loop
  int tm, tn, split;
  item_coords(item, tm, tn, split);
  const int m0 = tm * BM + wm * (BM / 2) + g;
  const int n0 = tn * BN + wn * (BN / 4) + (lane & 3) * 2;
  if (partial) {
    double* P = partial + (size_t)split * M * N;
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const int m = m0 + mi * 8;
      if (m >= M) continue;
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int n = n0 + ni * 8 + j;
          if (n < N) P[(size_t)n * M + m] = acc[mi][ni][j];
        }
    }
    continue;
  }
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int m = m0 + mi * 8;
    if (m >= M) continue;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = n0 + ni * 8 + j;
        if (n < N) {
          double* p = C + (size_t)n * ldc + m;
          double v = alpha * acc[mi][ni][j];
          if (beta != 0.0) v += beta * *p;
          *p = v;
        }
      }
  }
  }  // item loop
}

__global__ void splitk_reduce_kernel(const double* __restrict__ partial, int splitk, int64_t M, int64_t N,
                                     double* __restrict__ C, int64_t ldc, double alpha, double beta) {
  const int64_t total = M * N, MN = M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double s = partial[e];
    for (int q = 1; q < splitk; ++q) s += partial[q * MN + e];  // fixed order: deterministic
    const int64_t n = e / M, m = e - n * M;
    double* p = C + n * ldc + m;
    double v = alpha * s;
    if (beta != 0.0) v += beta * *p;
    *p = v;
  }
}

// ---- tensor maps through the driver entry point (no libcuda link dependency) ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// K-major operand: rows x K, element (row, k) at base[row*ld + k]; box BK x box_rows, 128B swizzle.
bool make_kmajor_map(CUtensorMap* tm, const double* base, int64_t rows, int64_t K, int64_t ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)std::max<int64_t>(K, 1), (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

// 2-D FP64 tensor map with a 128-B swizzle (shared with the smm kernels).
bool make_map_2d(CUtensorMap* tm, const double* base, uint64_t inner, uint64_t rows, uint64_t row_stride_bytes,
                 uint32_t box_inner, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)std::max<uint64_t>(rows, 1)};
  cuuint64_t strides[1] = {(cuuint64_t)row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4-D view of a panel of 64 x 64 column-major blocks, block (kk, lj) at slot kk*nblk_n + lj: B(k, n) with
// k = 64 kk + k_in, n = 64 lj + n_in lives at ((kk*nblk_n + lj)*64 + n_in)*64 + k_in.  Box {16 k, 64 n,
// BN/64 block columns, 1}: the same [n][16 k] 128-B-swizzled tile a 2-D K-major box gives.
bool make_block_b_map(CUtensorMap* tm, const double* base, int64_t nblk_n, int64_t nblk_k, int bn) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {64, 64, (cuuint64_t)std::max<int64_t>(nblk_n, 1), (cuuint64_t)std::max<int64_t>(nblk_k, 1)};
  cuuint64_t strides[3] = {64 * 8, 64 * 64 * 8, (cuuint64_t)std::max<int64_t>(nblk_n, 1) * 64 * 64 * 8};
  cuuint32_t box[4] = {BK, 64, (cuuint32_t)(bn / 64), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4-D view of a panel of 64 x 64 column-major A blocks, block (li, kk) at slot li*blk_ld + kk: A(m, k) with
// m = 64 li + m_in, k = 64 kk + k_in lives at ((li*blk_ld + kk)*64 + k_in)*64 + m_in.  Box {16 m, 16 k, 1,
// bm/64 block rows}: a [bm/64][16 k][16 m] 128-B-swizzled tile per 16-row m chunk (4 chunks per stage).
bool make_block_a_map(CUtensorMap* tm, const double* base, int64_t nblk_m, int64_t nblk_k, int64_t blk_ld, int bm) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {64, 64, (cuuint64_t)std::max<int64_t>(nblk_k, 1), (cuuint64_t)std::max<int64_t>(nblk_m, 1)};
  cuuint64_t strides[3] = {64 * 8, 64 * 64 * 8, (cuuint64_t)std::max<int64_t>(blk_ld, 1) * 64 * 64 * 8};
  cuuint32_t box[4] = {16, BK, 1, (cuuint32_t)(bm / 64)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

// Host planner: for each CTA tile shape, the split-K count that fills whole waves of `sms`
// persistent CTAs; the cheapest (padded work x rounds / shape efficiency) wins.
struct GemmPlan {
  int bm, bn, splitk;
};

GemmPlan pick_gemm(int64_t M, int64_t N, int64_t K, int sms) {
  static const int shapes[4][2] = {{128, 128}, {128, 64}, {64, 128}, {64, 64}};
  static const double eff[4] = {1.0, 0.97, 0.97, 0.90};  // per-flop cost of the smaller tiles (LDS/DMMA ratio)
  const int64_t ktiles = (K + BK - 1) / BK;
  GemmPlan best{128, 128, 1};
  double best_t = 1e300;
  for (int v = 0; v < 4; ++v) {
    const int bm = shapes[v][0], bn = shapes[v][1];
    const int64_t tiles = ((M + bm - 1) / bm) * ((N + bn - 1) / bn);
    for (int s = 1; s <= 64; ++s) {
      if (s > 1 && (tiles >= 4LL * sms || ktiles / s < 64)) break;  // keep >= 1024 of K per split
      const int64_t rounds = (tiles * s + sms - 1) / sms;
      const double t = (double)rounds * bm * bn * ((double)K / s) / eff[v] * (1.0 + 0.002 * (s - 1));
      if (t < best_t * (1.0 - 1e-9)) {
        best_t = t;
        best = {bm, bn, s};
      }
    }
  }
  return best;
}

}  // namespace

int pick_splitk(int64_t M, int64_t N, int64_t K, int sms) { return pick_gemm(M, N, K, sms).splitk; }

namespace {
// DBM_DGEMM_WAVESYNC=<k-tiles> sets the fuzzy wave barrier's interval (0/unset = off) and
// DBM_DGEMM_WAVESLACK=<intervals> its slack (default 1).  See DESIGN.md §5.
int wave_sync_ktiles() {
  static int v = [] {
    const char* e = getenv("DBM_DGEMM_WAVESYNC");
    return e ? std::max(0, atoi(e)) : 0;
  }();
  return v;
}
int wave_slack() {
  static int v = [] {
    const char* e = getenv("DBM_DGEMM_WAVESLACK");
    return e ? std::max(0, atoi(e)) : 1;
  }();
  return v;
}
unsigned* wave_sync_counter() {
  static unsigned* p = nullptr;  // one process drives one device
  if (p == nullptr && cudaMalloc(&p, sizeof(unsigned)) != cudaSuccess) p = nullptr;
  return p;
}

template <int BM, int BN, bool A_BLK>
cudaError_t launch_tile(const GemmArgs& g, int splitk, cudaStream_t st) {
  using T = Tile<BM, BN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(dgemm_tn_kernel<BM, BN, A_BLK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)T::kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap tmA, tmB;
  // A zero-K product still needs valid (never dereferenced) maps: point at a 1-column view.
  if (A_BLK ? !make_block_a_map(&tmA, g.A, (g.M + 63) / 64, (g.K + 63) / 64, g.a_blk_ld, BM)
            : !make_kmajor_map(&tmA, g.A, g.M, g.K, std::max<int64_t>(g.lda, 2), BM))
    return cudaErrorInvalidValue;
  if (g.b_blocks ? !make_block_b_map(&tmB, g.B, (g.N + 63) / 64, (g.K + 63) / 64, BN)
                 : !make_kmajor_map(&tmB, g.B, g.N, g.K, std::max<int64_t>(g.ldb, 2), BN))
    return cudaErrorInvalidValue;
  const int tiles_m = (int)((g.M + BM - 1) / BM), tiles_n = (int)((g.N + BN - 1) / BN);
  const int ktiles = (int)((g.K + BK - 1) / BK);
  const int per = (ktiles + splitk - 1) / splitk;
  const int64_t items = (int64_t)tiles_m * tiles_n * splitk;
  const unsigned grid = (unsigned)std::min<int64_t>(items, num_sms());  // persistent: one CTA per SM
  double* partial = splitk > 1 ? g.partial : nullptr;
  const int sync_kt = wave_sync_ktiles();
  // Barriers only where every CTA reaches them: the full rounds, and (split-K) equal k-ranges.
  const int rounds = (int)(items / grid);
  if (sync_kt > 0 && rounds > 0 && (ktiles % splitk) == 0) {
    unsigned* ws = wave_sync_counter();
    if (ws == nullptr) return cudaErrorMemoryAllocation;
    cudaError_t e = cudaMemsetAsync(ws, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = T::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident, or the launch fails: no deadlock
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, dgemm_tn_kernel<BM, BN, A_BLK>, tmA, tmB, (int)g.M, (int)g.N, ktiles,
                              std::max(per, 0), splitk, tiles_m, tiles_n, g.C, g.ldc, g.alpha, g.beta, partial, ws,
                              sync_kt, rounds, wave_slack(), g.b_blocks);
  }
  dgemm_tn_kernel<BM, BN, A_BLK><<<grid, kThreads, T::kSmem, st>>>(tmA, tmB, (int)g.M, (int)g.N, ktiles, std::max(per, 0),
                                                            splitk, tiles_m, tiles_n, g.C, g.ldc, g.alpha, g.beta,
                                                            partial, nullptr, 1, 0, 0, g.b_blocks);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_dgemm(const GemmArgs& g, cudaStream_t st, int* launches) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  const GemmPlan pl = pick_gemm(g.M, g.N, g.K, num_sms());
  const int splitk = std::max(1, g.splitk);
  cudaError_t e;
  if (g.a_blocks) {
    if (pl.bm == 128 && pl.bn == 128)
      e = launch_tile<128, 128, true>(g, splitk, st);
    else if (pl.bm == 128)
      e = launch_tile<128, 64, true>(g, splitk, st);
    else if (pl.bn == 128)
      e = launch_tile<64, 128, true>(g, splitk, st);
    else
      e = launch_tile<64, 64, true>(g, splitk, st);
  } else if (pl.bm == 128 && pl.bn == 128) {
    e = launch_tile<128, 128, false>(g, splitk, st);
  } else if (pl.bm == 128) {
    e = launch_tile<128, 64, false>(g, splitk, st);
  } else if (pl.bn == 128) {
    e = launch_tile<64, 128, false>(g, splitk, st);
  } else {
    e = launch_tile<64, 64, false>(g, splitk, st);
  }
  if (launches) ++*launches;
  if (e != cudaSuccess) return e;
  if (splitk > 1) {
    launch_splitk_reduce(g.partial, splitk, g.M, g.N, g.C, g.ldc, g.alpha, g.beta, st);
    if (launches) ++*launches;
    e = cudaGetLastError();
  }
  return e;
}

void launch_splitk_reduce(const double* partial, int splitk, int64_t M, int64_t N, double* C, int64_t ldc,
                          double alpha, double beta, cudaStream_t st) {
  const int64_t total = M * N;
  int64_t grid = std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
  splitk_reduce_kernel<<<(unsigned)std::max<int64_t>(grid, 1), 256, 0, st>>>(partial, splitk, M, N, C, ldc, alpha,
                                                                             beta);
}

}  // namespace dbm

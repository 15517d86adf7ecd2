// smm — the blocked path's batched small-block FP64 GEMM (the LIBCUSMM role, §II).
//
// Executes a chunk of stacks: consecutive C-block runs, each run = kb entries (a, b, c) with the
// k-index ascending (stack generator, reading R6); per run C_blk = (first ? beta*C_blk : C_blk) +
// alpha * sum_k A_blk(a_k) * B_blk(b_k).
//
// B200 design: FP64 tensor path = mma.sync.m8n8k4.f64 (DMMA, which shares the FP64
// pipe with DFMA).  A CTA executes a GROUP of consecutive runs (bs 22: 8 runs, one warp per C block,
// 24x24 padded = 3x3 DMMA subtiles; bs 64: 2 runs, 2x2 warps of 32x32 per C block).  Runs of a
// group that share an A (B) block share one staged copy — consecutive runs of the bisection
// traversal form compact rectangles, so a group of 8 typically stages 6-8 blocks instead of 16.
// Staged blocks live in a pool of P slots per stage; a group whose distinct blocks exceed P is run
// as two halves.  The K dimension of a run is the concatenation of its kb blocks (a stage holds KS
// consecutive k), so k-steps of 4 never pad K; only M, N pad 22 -> 24 (the bs-22 ceiling is
// (22/24)^2 = 84% of the DMMA peak; bs 64 has none).  cp.async (16 B) stages operands in a 3-deep
// ring; pitches are chosen so DMMA fragment loads are (near) conflict-free LDS.64.
#include <algorithm>
#include <cstdlib>

#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "dbm_internal.h"

namespace dbm {

namespace {

template <int BS_, int RUNS_, int WRM_, int WRN_, int SM_, int SN_, int KS_, int PA_, int PB_, int P_>
struct SmmCfg {
  static constexpr int BS = BS_, BB = BS_ * BS_;
  static constexpr int RUNS = RUNS_;            // runs (C blocks) per group
  static constexpr int WRM = WRM_, WRN = WRN_;  // warps per run (m x n)
  static constexpr int SM = SM_, SN = SN_;      // 8x8 DMMA subtiles per warp (m x n)
  static constexpr int KS = KS_;                // k values per stage (multiple of 4)
  static constexpr int PA = PA_, PB = PB_;      // A: [k][PA] rows contiguous; B: [n][PB] k contiguous
  static constexpr int P = P_;                  // pool slots per stage (A and B blocks share them)
  static constexpr int WARPS = RUNS * WRM * WRN;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int SLOT = (KS * PA > BS * PB) ? KS * PA : BS * PB;  // doubles
  static constexpr int PAD_ROWS = SM * 8 * WRM - BS;                  // padded rows read past a slot
  static constexpr int SLACK = (PAD_ROWS > 0 ? PAD_ROWS : 0) * (PA > PB ? PA : PB) + 8;
  static constexpr int STAGE = P * SLOT + SLACK;
  static constexpr int STAGES = 3;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE * 8;
  static_assert(KS % 4 == 0 && KS % 2 == 0 && BS % 2 == 0, "16-byte chunks, k-steps of 4");
  static_assert(SM * 8 * WRM >= BS && SN * 8 * WRN >= BS, "warps cover the block");
  static_assert(SMEM + 256 <= 232448, "shared memory");
};

// (bs 22 uses smm22_kernel below)
// bs 64: padded pitches 72 / 36 (both conflict-free), half a block of K per stage
using Cfg64 = SmmCfg<64, 2, 2, 2, 4, 4, 32, 72, 36, 4>;

__device__ __forceinline__ double lds64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// Warp 0: distinct A / B blocks among runs [q0+s0, q0+s0+n) (from their first entries).
struct Uniq {
  unsigned lead_a, lead_b, ma, mb;
  bool act;
};
__device__ __forceinline__ Uniq uniq(const int32_t* __restrict__ trip, int64_t q0, int s0, int n, int64_t kb,
                                     int lane, const int32_t* __restrict__ runs = nullptr) {
  Uniq u;
  u.act = lane < n;
  const int64_t v = q0 + s0 + lane;
  const int64_t q = (runs && u.act) ? runs[v] : v;
  const int a = u.act ? trip[3 * (q * kb)] : -1 - lane;
  const int b = u.act ? trip[3 * (q * kb) + 1] : -1 - lane;
  u.ma = __match_any_sync(0xffffffffu, a);
  u.mb = __match_any_sync(0xffffffffu, b);
  u.lead_a = __ballot_sync(0xffffffffu, u.act && (__ffs(u.ma) - 1) == lane);
  u.lead_b = __ballot_sync(0xffffffffu, u.act && (__ffs(u.mb) - 1) == lane);
  return u;
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
// arrive on the mbarrier when all of this thread's prior cp.async have landed
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

__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

// Warp-specialised: warps 0..WARPS-1 compute (one run, or a WRM x WRN share of one), warp WARPS is
// the producer.  Per stage the producer reads the slots' block indices from the stack triplets
// once (one lane each), broadcasts them with shuffles, and issues one TMA bulk copy per padded
// column / row segment, completing on the stage's mbarrier (expect_tx).  Consumers release a stage with one
// mbarrier arrive per warp.  Group metadata (which runs share blocks) is computed by the producer
// between two CTA barriers at each (sub-)group start.
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS + 32, 1)
    smm_group_kernel(const int32_t* __restrict__ trip, int64_t nruns, int64_t kb, const double* __restrict__ A,
                     const double* __restrict__ B, double* __restrict__ C, double alpha, double beta_first) {
  constexpr int BS = Cfg::BS, BB = Cfg::BB, KS = Cfg::KS, PA = Cfg::PA, PB = Cfg::PB;
  constexpr int RUNS = Cfg::RUNS, P = Cfg::P, STAGES = Cfg::STAGES, SLOT = Cfg::SLOT, WARPS = Cfg::WARPS;
  static_assert(KS % BS == 0 || BS % KS == 0, "a stage covers whole blocks or a block divides into stages");
  constexpr int KKS = (KS % BS == 0) ? KS / BS : 1;  // blocks (k indices kk) touched per stage
  static_assert(P * KKS <= 32, "one lane per (slot, kk)");
  constexpr int CA = KS * (BS / 2);  // 16-B chunks per A slot: KS columns x BS/2
  constexpr int CB = BS * (KS / 2);  // per B slot: BS rows x KS/2
  static_assert(CA == CB, "equal chunk counts");
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  __shared__ int s_rep[P];  // representative run (in group) of each pool slot
  __shared__ int s_isb[P];  // slot holds a B block (else A)
  __shared__ int s_ia[RUNS], s_ib[RUNS];
  __shared__ int s_n, s_sub;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp == WARPS;
  const int run_in_group = warp / (Cfg::WRM * Cfg::WRN);
  const int wsub = warp % (Cfg::WRM * Cfg::WRN);
  const int wm = wsub / Cfg::WRN, wn = wsub % Cfg::WRN;
  const int Krun = (int)(kb * BS);  // concatenated K of a run (< 2^31 for every config)
  const int nst = (Krun + KS - 1) / KS;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const int64_t ngroups = (nruns + RUNS - 1) / RUNS;
  const int g = lane >> 2, t = lane & 3;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init((uint32_t)__cvta_generic_to_shared(&full[s]), 1);
      mbar_init((uint32_t)__cvta_generic_to_shared(&empty[s]), WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  int stage = 0;
  uint32_t phase = 0;
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int64_t q0 = grp * RUNS;
    const int nrun_g = (int)(nruns - q0 < RUNS ? nruns - q0 : RUNS);
    if (producer) {  // sub-group size: halve until every sub-group's distinct blocks fit the pool
      int sub = nrun_g;
      for (;;) {
        bool ok = true;
        for (int s0 = 0; s0 < nrun_g; s0 += sub) {
          const Uniq u = uniq(trip, q0, s0, min(sub, nrun_g - s0), kb, lane);
          if (__popc(u.lead_a) + __popc(u.lead_b) > P) ok = false;
        }
        if (ok || sub == 1) break;
        sub = (sub + 1) / 2;
      }
      if (lane == 0) s_sub = sub;
    }
    __syncthreads();
    const int sub = s_sub;

    for (int s0 = 0; s0 < nrun_g; s0 += sub) {
      const int n_sub = min(sub, nrun_g - s0);
      if (s0 > 0) __syncthreads();  // every warp finished the previous sub-group
      if (producer) {
        const Uniq u = uniq(trip, q0, s0, n_sub, kb, lane);
        const int na = __popc(u.lead_a);
        if (u.act) {
          const int la = __ffs(u.ma) - 1, lb = __ffs(u.mb) - 1;
          const int ia = __popc(u.lead_a & ((1u << la) - 1));
          const int ib = na + __popc(u.lead_b & ((1u << lb) - 1));
          s_ia[lane] = ia;
          s_ib[lane] = ib;
          if (la == lane) {
            s_rep[ia] = s0 + lane;
            s_isb[ia] = 0;
          }
          if (lb == lane) {
            s_rep[ib] = s0 + lane;
            s_isb[ib] = 1;
          }
        }
        if (lane == 0) s_n = na + __popc(u.lead_b);
      }
      __syncthreads();
      const int nslots = s_n;

      if (producer) {
        // ---------------- producer: nst stages of this sub-group
        // lane l < nslots*KKS owns (slot u = l / KKS, block kk = kk_first + l % KKS)
        const int my_u = lane / KKS;
        const bool owner = lane < nslots * KKS;
        const int64_t my_q = q0 + (owner ? s_rep[my_u] : 0);
        const int my_col = owner ? s_isb[my_u] : 0;
        // one TMA bulk copy per segment: an A k-column (BS contiguous doubles -> pitch PA) or a B
        // n-row (KS contiguous k of block column y -> pitch PB); KS divides BS, so a stage never
        // straddles two k-blocks and K never needs zero-fill
        static_assert(KKS == 1 && BS % KS == 0, "bulk segments need stages inside one block");
        const int nseg = nslots * (KS > BS ? KS : BS);  // per slot: KS A-columns or BS B-rows (KS <= BS)
        for (int st = 0; st < nst; ++st) {
          const int kg0 = st * KS, kk = kg0 / BS, x0 = kg0 - kk * BS;
          int blk = 0;
          if (owner) blk = trip[3 * (my_q * kb + kk) + my_col];
          const uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[stage]);
          if (lane == 0) {
            mbar_wait((uint32_t)__cvta_generic_to_shared(&empty[stage]), phase ^ 1);
            uint32_t bytes = 0;
            for (int u = 0; u < nslots; ++u) bytes += s_isb[u] ? BS * KS * 8 : KS * BS * 8;
            mbar_expect_tx(fb, bytes);
          }
          __syncwarp();
          const uint32_t d0 = sbase + (uint32_t)(stage * Cfg::STAGE) * 8u;
          for (int c0 = 0; c0 < nseg; c0 += 32) {
            const int c = c0 + lane;
            const int u = c / BS, r = c - u * BS;  // slot, segment index (< BS)
            const bool v = c < nseg;
            const int b = __shfl_sync(0xffffffffu, blk, v ? u : 0);
            if (v) {
              if (!s_isb[u]) {
                if (r < KS)  // A column k = r of this stage: column x0 + r of the block
                  bulk_g2s(d0 + (uint32_t)(u * SLOT + r * PA) * 8u, A + (int64_t)b * BB + (int64_t)(x0 + r) * BS,
                           BS * 8, fb);
              } else {  // B row n = r: k = x0 .. x0+KS-1 of block column r
                bulk_g2s(d0 + (uint32_t)(u * SLOT + r * PB) * 8u, B + (int64_t)b * BB + (int64_t)r * BS + x0,
                         KS * 8, fb);
              }
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        continue;
      }

      // ---------------- consumers
      const int my = run_in_group - s0;
      const bool active = my >= 0 && my < n_sub;
      double acc[Cfg::SM][Cfg::SN][2];
#pragma unroll
      for (int i = 0; i < Cfg::SM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::SN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      const int ia = active ? s_ia[my] : 0, ib = active ? s_ib[my] : 0;
      // fragments: A (k, m) at slot ia: k*PA + m; B (k, n) at slot ib: n*PB + k;
      // m = wm*SM*8 + mi*8 + g, n = wn*SN*8 + ni*8 + g, k = 4*ks + t
      const uint32_t offA = (uint32_t)(ia * SLOT + t * PA + wm * Cfg::SM * 8 + g) * 8u;
      const uint32_t offB = (uint32_t)(ib * SLOT + (wn * Cfg::SN * 8 + g) * PB + t) * 8u;
      for (int st = 0; st < nst; ++st) {
        mbar_wait((uint32_t)__cvta_generic_to_shared(&full[stage]), phase);
        if (active) {
          const uint32_t base = sbase + (uint32_t)(stage * Cfg::STAGE) * 8u;
#pragma unroll
          for (int ks = 0; ks < KS / 4; ++ks) {
            double a[Cfg::SM], b[Cfg::SN];
#pragma unroll
            for (int mi = 0; mi < Cfg::SM; ++mi) a[mi] = lds64(base + offA + (uint32_t)(ks * 4 * PA + mi * 8) * 8u);
#pragma unroll
            for (int ni = 0; ni < Cfg::SN; ++ni) b[ni] = lds64(base + offB + (uint32_t)(ks * 4 + ni * 8 * PB) * 8u);
#pragma unroll
            for (int mi = 0; mi < Cfg::SM; ++mi)
#pragma unroll
              for (int ni = 0; ni < Cfg::SN; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive((uint32_t)__cvta_generic_to_shared(&empty[stage]));
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      // ---- epilogue: this warp's part of its run's C block
      if (active) {
        const int64_t q = q0 + run_in_group;
        double* cb = C + (int64_t)trip[3 * (q * kb) + 2] * BB;
#pragma unroll
        for (int mi = 0; mi < Cfg::SM; ++mi) {
          const int m = wm * Cfg::SM * 8 + mi * 8 + g;
#pragma unroll
          for (int ni = 0; ni < Cfg::SN; ++ni)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int n = wn * Cfg::SN * 8 + ni * 8 + 2 * t + j;
              if (m < BS && n < BS) {
                double* p = cb + m + n * BS;
                const double v = alpha * acc[mi][ni][j];
                *p = (beta_first == 0.0) ? v : beta_first * *p + v;
              }
            }
        }
      }
    }
    __syncthreads();  // group done: metadata may be rewritten
  }
}

template <class Cfg>
cudaError_t launch_group(const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const double* B, double* C,
                         double alpha, double beta_first, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(smm_group_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t ngroups = (nruns + Cfg::RUNS - 1) / Cfg::RUNS;
  const unsigned grid = (unsigned)std::min<int64_t>(ngroups, (int64_t)num_sms());
  smm_group_kernel<Cfg><<<grid, Cfg::THREADS + 32, Cfg::SMEM, st>>>(trip, nruns, kb, A, B, C, alpha, beta_first);
  return cudaGetLastError();
}

// ============================================================================ bs 22: TMA bulk staging
// Same group scheme (8 runs per CTA, one consumer warp per C block), but every staged block is one
// 3,872-B cp.async.bulk (TMA) issued by one producer lane, completing on the stage's mbarrier:
// a stage is KK22 = 2 consecutive k-blocks, i.e. 44 k = 11 DMMA k-steps without K padding.
//   A slot: blocks (li, kk0), (li, kk0+1) column-major back to back = [k 0..43][m 0..21] (pitch 22)
//   B slot: blocks (kk0, lj), (kk0+1, lj)                            = [kk][n][x] (pitch 22)
// A tail stage (odd kb) masks the missing k with zeros in registers.
namespace s22 {
constexpr int BS = 22, BB = 484, KK = 2, KS = 44, RUNS = 8, WARPS = 8, P = 9, STAGES = 3;
constexpr int SLOT = KK * BB;                       // doubles
// slack: the padded rows m, n = 22, 23 of the last slot read past it (B: up to kk*484 + 23*22 + 21
// = SLOT + 43 doubles); only discarded C rows / columns see those values
constexpr int STAGE = P * SLOT + 64;
constexpr size_t SMEM = (size_t)STAGES * STAGE * 8;
constexpr uint32_t BLK_BYTES = BB * 8;              // 3,872
static_assert(SMEM + 512 <= 232448, "shared memory");
}  // namespace s22


template <bool MASK>
__device__ __forceinline__ void s22_stage(double (&acc)[3][3][2], uint32_t sA, uint32_t sB, int t, int kvalid) {
  using namespace s22;
  // B (k, n) of the two-block slot: kk = k / 22, x = k % 22 -> kk*484 + n*22 + x
#pragma unroll
  for (int ks = 0; ks < KS / 4; ++ks) {
    const int k = 4 * ks + t;
    const bool ok = !MASK || k < kvalid;
    const uint32_t kb_off = (uint32_t)((k >= BS ? BB + (k - BS) : k) * 8);
    double a[3], b[3];
#pragma unroll
    for (int mi = 0; mi < 3; ++mi) a[mi] = ok ? lds64(sA + (uint32_t)(k * BS + mi * 8) * 8u) : 0.0;
#pragma unroll
    for (int ni = 0; ni < 3; ++ni) b[ni] = ok ? lds64(sB + kb_off + (uint32_t)(ni * 8 * BS) * 8u) : 0.0;
#pragma unroll
    for (int mi = 0; mi < 3; ++mi)
#pragma unroll
      for (int ni = 0; ni < 3; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
  }
}

__global__ void __launch_bounds__((s22::WARPS + 1) * 32, 1)
    smm22_kernel(const int32_t* __restrict__ trip, int64_t nruns, int64_t kb, const double* __restrict__ A,
                 const double* __restrict__ B, double* __restrict__ C, double alpha, double beta_first, int nsplit,
                 double* __restrict__ partial, const int32_t* __restrict__ runs, const int* __restrict__ d_count) {
  // runs != nullptr: the runs to execute are runs[0 .. *d_count) (indices into the chunk's triplets),
  // grouped 8 at a time in list order; otherwise runs 0 .. nruns-1
  using namespace s22;
  if (d_count) nruns = *d_count;
  auto RUN = [&](int64_t v) -> int64_t { return runs ? (int64_t)runs[v] : v; };
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  __shared__ int s_rep[P], s_isb[P], s_ia[RUNS], s_ib[RUNS], s_n, s_sub;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp == WARPS;
  const int Krun = (int)(kb * BS);
  const int nst = (Krun + KS - 1) / KS;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const int64_t ngroups = (nruns + RUNS - 1) / RUNS;
  const int g = lane >> 2, t = lane & 3;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init((uint32_t)__cvta_generic_to_shared(&full[s]), 1);
      mbar_init((uint32_t)__cvta_generic_to_shared(&empty[s]), WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  int stage = 0;
  uint32_t phase = 0;
  // work item = (group, K split); with nsplit > 1 each item accumulates stages [st0, st1) of its
  // runs into `partial` (reduced later in a fixed order) instead of updating C
  for (int64_t item = blockIdx.x; item < ngroups * nsplit; item += gridDim.x) {
    const int64_t grp = item % ngroups;
    const int split = (int)(item / ngroups);
    const int st0 = (int)((int64_t)nst * split / nsplit), st1 = (int)((int64_t)nst * (split + 1) / nsplit);
    const int64_t q0 = grp * RUNS;
    const int nrun_g = (int)(nruns - q0 < RUNS ? nruns - q0 : RUNS);
    if (producer) {
      int sub = nrun_g;
      for (;;) {
        bool ok = true;
        for (int s0 = 0; s0 < nrun_g; s0 += sub) {
          const Uniq u = uniq(trip, q0, s0, min(sub, nrun_g - s0), kb, lane, runs);
          if (__popc(u.lead_a) + __popc(u.lead_b) > P) ok = false;
        }
        if (ok || sub == 1) break;
        sub = (sub + 1) / 2;
      }
      if (lane == 0) s_sub = sub;
    }
    __syncthreads();
    const int sub = s_sub;
    for (int s0 = 0; s0 < nrun_g; s0 += sub) {
      const int n_sub = min(sub, nrun_g - s0);
      if (s0 > 0) __syncthreads();
      if (producer) {
        const Uniq u = uniq(trip, q0, s0, n_sub, kb, lane, runs);
        const int na = __popc(u.lead_a);
        if (u.act) {
          const int la = __ffs(u.ma) - 1, lb = __ffs(u.mb) - 1;
          const int ia = __popc(u.lead_a & ((1u << la) - 1));
          const int ib = na + __popc(u.lead_b & ((1u << lb) - 1));
          s_ia[lane] = ia;
          s_ib[lane] = ib;
          if (la == lane) {
            s_rep[ia] = s0 + lane;
            s_isb[ia] = 0;
          }
          if (lb == lane) {
            s_rep[ib] = s0 + lane;
            s_isb[ib] = 1;
          }
        }
        if (lane == 0) s_n = na + __popc(u.lead_b);
      }
      __syncthreads();
      const int nslots = s_n;

      if (producer) {
        // lane l < 2*nslots copies block kk0 + (l & 1) of slot l >> 1
        const int u = lane >> 1, j = lane & 1;
        const bool owner = u < nslots;
        const int64_t q = RUN(q0 + (owner ? s_rep[u] : 0));
        const int col = owner ? s_isb[u] : 0;
        const double* base = col ? B : A;
        for (int st = st0; st < st1; ++st) {
          const int kk = st * KK + j;
          const bool valid = owner && kk < kb;
          const uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[stage]);
          if (lane == 0) mbar_wait((uint32_t)__cvta_generic_to_shared(&empty[stage]), phase ^ 1);
          const unsigned vm = __ballot_sync(0xffffffffu, valid);
          if (lane == 0) mbar_expect_tx(fb, (uint32_t)__popc(vm) * BLK_BYTES);
          __syncwarp();
          if (valid) {
            const int64_t blk = trip[3 * (q * kb + kk) + col];
            bulk_g2s(sbase + (uint32_t)(stage * STAGE + u * SLOT + j * BB) * 8u, base + blk * BB, BLK_BYTES, fb);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        continue;
      }

      const int my = warp - s0;
      const bool active = my >= 0 && my < n_sub;
      double acc[3][3][2];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
      const int ia = active ? s_ia[my] : 0, ib = active ? s_ib[my] : 0;
      const uint32_t offA = (uint32_t)(ia * SLOT + g) * 8u;        // + k*22 + mi*8
      const uint32_t offB = (uint32_t)(ib * SLOT + g * BS) * 8u;   // + kk*484 + x + ni*8*22
      for (int st = st0; st < st1; ++st) {
        mbar_wait((uint32_t)__cvta_generic_to_shared(&full[stage]), phase);
        if (active) {
          const uint32_t sb = sbase + (uint32_t)(stage * STAGE) * 8u;
          const int kvalid = Krun - st * KS;
          if (kvalid >= KS)
            s22_stage<false>(acc, sb + offA, sb + offB, t, KS);
          else
            s22_stage<true>(acc, sb + offA, sb + offB, t, kvalid);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive((uint32_t)__cvta_generic_to_shared(&empty[stage]));
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (active) {
        double* cb = partial ? partial + ((int64_t)split * nruns + q0 + warp) * BB
                             : C + (int64_t)trip[3 * (RUN(q0 + warp) * kb) + 2] * BB;
#pragma unroll
        for (int mi = 0; mi < 3; ++mi) {
          const int m = mi * 8 + g;
#pragma unroll
          for (int ni = 0; ni < 3; ++ni)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const int n = ni * 8 + 2 * t + jj;
              if (m < BS && n < BS) {
                double* p = cb + m + n * BS;
                if (partial) {
                  *p = acc[mi][ni][jj];
                } else {
                  const double v = alpha * acc[mi][ni][jj];
                  *p = (beta_first == 0.0) ? v : beta_first * *p + v;
                }
              }
            }
        }
      }
    }
    __syncthreads();
  }
}

// ============================================================================ bs 22: 4 x 4 run squares
// When 16 consecutive runs are a 4 x 4 square of C blocks (the bisection order of power-of-two-like
// local grids: every rectangular config), they share 4 A block rows and 4 B block columns per k, and
// their 88 x 88 C region is exactly 11 x 11 DMMA subtiles: no 22 -> 24 padding (the 8-run kernel above
// wastes (24/22)^2 - 1 = 19 % of its DMMAs on it).  A stage = 2 k-blocks (44 k) of 4 A + 4 B blocks,
// 16 TMA bulk copies from the producer warp.  The 121 subtiles go to the 4 SM sub-partitions
// as a pinwheel of 5 x 6 / 6 x 5 rectangles around the centre subtile (30, 30, 30, 31
// DMMAs per k-step), each rectangle split between the sub-partition's two warps (5 x 3 or 3 x 5).
namespace s22q {
constexpr int BS = 22, BB = 484, KK = 2, KS = 44, RUNS = 16, WARPS = 8, STAGES = 3;
constexpr int SLOT = KK * BB;                  // A slot: one block row over the stage's 2 k-blocks, [k][m]
constexpr int BOFF = 4 * SLOT;                 // B slots follow the 4 A slots
constexpr int SLOTB = 980;                     // B slot: [kk0 block][2 pad][kk1 block], stride = 4 (mod 16)
constexpr int KK1B = BB + 2;                   // the kk1 block's offset inside a B slot
constexpr int STAGE = BOFF + 4 * SLOTB;        // 7,792 doubles (a multiple of 16)
constexpr size_t SMEM = (size_t)STAGES * STAGE * 8;
constexpr uint32_t BLK_BYTES = BB * 8;
static_assert(SMEM + 1024 <= 232448, "shared memory");
}  // namespace s22q

// Subtile row i, fragment row g reads supertile row kQRowIdx[8i + g] (A offset kQRowOff); subtile column j,
// fragment column g reads supertile column kQColIdx[8j + g] (B offset kQColOff, incl. the B region).  The
// permutations group rows (m, m+1, m+8, m+9 of one block, or m, m+1 of two blocks 968 = 8 (mod 16)
// doubles apart) and columns (residues 6n + base spaced by 4 (mod 16); B slots at bases 0, 4, 8, 12) so
// that with the k-slot t of k-step ks reading k = 4 ks + t every half-warp's 64-bit fragment load hits
// 16 distinct bank pairs (generated and checked by a script; no padding, so no wasted DMMA lane).
__constant__ short kQRowOff[88] = {0, 1, 8, 9, 2, 3, 10, 11, 4, 5, 12, 13, 6, 7, 14, 15, 968, 969, 976, 977, 970, 971, 978, 979, 972, 973, 980, 981, 974, 975, 982, 983, 16, 17, 984, 985, 18, 19, 986, 987, 20, 21, 988, 989, 1936, 1937, 1944, 1945, 1938, 1939, 1946, 1947, 1940, 1941, 1948, 1949, 1942, 1943, 1950, 1951, 2904, 2905, 2912, 2913, 2906, 2907, 2914, 2915, 2908, 2909, 2916, 2917, 2910, 2911, 2918, 2919, 1952, 1953, 2920, 2921, 1954, 1955, 2922, 2923, 1956, 1957, 2924, 2925};
__constant__ short kQRowIdx[88] = {0, 1, 8, 9, 2, 3, 10, 11, 4, 5, 12, 13, 6, 7, 14, 15, 22, 23, 30, 31, 24, 25, 32, 33, 26, 27, 34, 35, 28, 29, 36, 37, 16, 17, 38, 39, 18, 19, 40, 41, 20, 21, 42, 43, 44, 45, 52, 53, 46, 47, 54, 55, 48, 49, 56, 57, 50, 51, 58, 59, 66, 67, 74, 75, 68, 69, 76, 77, 70, 71, 78, 79, 72, 73, 80, 81, 60, 61, 82, 83, 62, 63, 84, 85, 64, 65, 86, 87};
__constant__ short kQColOff[88] = {3872, 4004, 3960, 3916, 4048, 4180, 4136, 4092, 3938, 3894, 4026, 3982, 4114, 4070, 4202, 4158, 4852, 4984, 4940, 4896, 5028, 5160, 5116, 5072, 4918, 4874, 5006, 4962, 5094, 5050, 5182, 5138, 5832, 5964, 5920, 5876, 6008, 6140, 6096, 6052, 5898, 5854, 5986, 5942, 6074, 6030, 6162, 6118, 6812, 6944, 6900, 6856, 6988, 7120, 7076, 7032, 6878, 6834, 6966, 6922, 7054, 7010, 7142, 7098, 4224, 5204, 4312, 4268, 4290, 4246, 5226, 4334, 5292, 5248, 6228, 6184, 5270, 6250, 6206, 5314, 6272, 7252, 7208, 7164, 6294, 7274, 7230, 7186};
__constant__ short kQColIdx[88] = {0, 6, 4, 2, 8, 14, 12, 10, 3, 1, 7, 5, 11, 9, 15, 13, 22, 28, 26, 24, 30, 36, 34, 32, 25, 23, 29, 27, 33, 31, 37, 35, 44, 50, 48, 46, 52, 58, 56, 54, 47, 45, 51, 49, 55, 53, 59, 57, 66, 72, 70, 68, 74, 80, 78, 76, 69, 67, 73, 71, 77, 75, 81, 79, 16, 38, 20, 18, 19, 17, 39, 21, 42, 40, 62, 60, 41, 63, 61, 43, 64, 86, 84, 82, 65, 87, 85, 83};

// One stage (11 k-steps of 4): R x Cn subtiles (+ the centre subtile for CENTRE), fragments loaded with the
// tail predicate only when TAIL (the last stage of an odd kb holds one k-block).  (Splitting the centre's
// k-steps over the four SMSPs balances their DMMA counts 30/30/30/31 -> 30.25 each, but needs a named-barrier
// reduction and spills at the 168-register cap: measured 93.3 -> 79.9 % DMMA at 5,632^3, not kept.)
template <int R, int Cn, bool CENTRE, bool TAIL>
__device__ __forceinline__ void s22q_stage(uint32_t sb, int kvalid, int t, const uint32_t (&offA)[R],
                                           const uint32_t (&offB)[Cn], uint32_t offAc, uint32_t offBc,
                                           double (&acc)[R][Cn][2], double (&cacc)[2]) {
  using namespace s22q;
#pragma unroll
  for (int ks = 0; ks < KS / 4; ++ks) {
    const int k = 4 * ks + t;
    const bool ok = !TAIL || k < kvalid;
    // A slot: [k 0..43][m] at pitch 22 (the two blocks are contiguous); B slot: block k / 22 (the second
    // at KK1B), [n][k % 22]
    const uint32_t ka = (uint32_t)(k * BS) * 8u, kbo = (uint32_t)(k + (k >= BS ? KK1B - BS : 0)) * 8u;
    double a[R], b[Cn];
#pragma unroll
    for (int i = 0; i < R; ++i) a[i] = ok ? lds64(sb + offA[i] + ka) : 0.0;
#pragma unroll
    for (int j = 0; j < Cn; ++j) b[j] = ok ? lds64(sb + offB[j] + kbo) : 0.0;
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int j = 0; j < Cn; ++j) dmma(acc[i][j], a[i], b[j]);
    if (CENTRE) {
      const double ac = ok ? lds64(sb + offAc + ka) : 0.0;
      const double bc = ok ? lds64(sb + offBc + kbo) : 0.0;
      dmma(cacc, ac, bc);
    }
  }
}

// One warp's rectangle of subtiles: rows [r0, r0+R), cols [c0, c0+Cn) of the 11 x 11 grid (+ the centre
// subtile (5, 5) for CENTRE, a compile-time role so the k-loop carries no branch).
template <int R, int Cn, bool CENTRE>
__device__ __forceinline__ void s22q_consume(uint64_t* full, uint64_t* empty, uint32_t sbase, int& stage,
                                             uint32_t& phase, int st0, int st1, int Krun, int r0, int c0, int g,
                                             int t, int lane, double* const (&s_dst)[4][4], bool raw, double alpha,
                                             double beta_first) {
  using namespace s22q;
  double acc[R][Cn][2], cacc[2] = {0.0, 0.0};
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < Cn; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  uint32_t offA[R], offB[Cn];
#pragma unroll
  for (int i = 0; i < R; ++i) offA[i] = (uint32_t)kQRowOff[(r0 + i) * 8 + g] * 8u;
#pragma unroll
  for (int j = 0; j < Cn; ++j) offB[j] = (uint32_t)kQColOff[(c0 + j) * 8 + g] * 8u;
  const uint32_t offAc = (uint32_t)kQRowOff[40 + g] * 8u, offBc = (uint32_t)kQColOff[40 + g] * 8u;
  // every stage but (possibly) the last holds 44 valid k
  const int full_end = min(st1, Krun / KS);
  for (int st = st0; st < st1; ++st) {
    mbar_wait((uint32_t)__cvta_generic_to_shared(&full[stage]), phase);
    const uint32_t sb = sbase + (uint32_t)(stage * STAGE) * 8u;
    if (st < full_end)
      s22q_stage<R, Cn, CENTRE, false>(sb, KS, t, offA, offB, offAc, offBc, acc, cacc);
    else
      s22q_stage<R, Cn, CENTRE, true>(sb, Krun - st * KS, t, offA, offB, offAc, offBc, acc, cacc);
    __syncwarp();
    if (lane == 0) mbar_arrive((uint32_t)__cvta_generic_to_shared(&empty[stage]));
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
  // epilogue straight from the accumulators: subtile (i, j), lane (g, t) holds the element at row
  // M = kQRowIdx[8 (r0 + i) + g], column N = kQColIdx[8 (c0 + j) + 2t + jj] of the 88 x 88 square,
  // i.e. element (M mod 22, N mod 22) of C block (M / 22, N / 22) (once per square: off the hot loop)
  auto put = [&](int M, int N, double v) {
    const int ri = M / BS, cj = N / BS;
    double* p = s_dst[ri][cj] + (M - ri * BS) + (N - cj * BS) * BS;
    if (raw) {
      *p = v;
    } else {
      const double w = alpha * v;
      *p = (beta_first == 0.0) ? w : beta_first * *p + w;
    }
  };
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int M = kQRowIdx[(r0 + i) * 8 + g];
#pragma unroll
    for (int j = 0; j < Cn; ++j)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) put(M, kQColIdx[(c0 + j) * 8 + 2 * t + jj], acc[i][j][jj]);
  }
  if (CENTRE)
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) put(kQRowIdx[40 + g], kQColIdx[40 + 2 * t + jj], cacc[jj]);
}

__global__ void __launch_bounds__((s22q::WARPS + 1) * 32, 1)
    smm22q_kernel(const int32_t* __restrict__ trip, int64_t nruns, int64_t kb, const double* __restrict__ A,
                  const double* __restrict__ B, double* __restrict__ C, double alpha, double beta_first, int nsplit,
                  double* __restrict__ partial, const int32_t* __restrict__ runs, const int* __restrict__ d_count,
                  int centre_warp) {
  // runs != nullptr: squares are runs[16 s .. 16 s + 16) for s < *d_count / 16; otherwise runs 16 s ..
  using namespace s22q;
  if (d_count) nruns = *d_count;
  auto RUN = [&](int64_t v) -> int64_t { return runs ? (int64_t)runs[v] : v; };
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  __shared__ int s_rowrep[4], s_colrep[4];
  __shared__ double* s_dst[2][4][4];  // per item parity: the C (or split-K partial) block of square cell (ri, cj)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp == WARPS;
  const int Krun = (int)(kb * BS);
  const int nst = (Krun + KS - 1) / KS;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const int64_t ngroups = nruns / RUNS;  // the host launches this kernel only on whole squares
  const int g = lane >> 2, t = lane & 3;
  // Items of >= STAGES + 1 stages need no CTA barrier between them: the consumers read the item's
  // destination pointers (s_dst, double-buffered by item parity) after waiting on one of its full
  // barriers, and the producer cannot reach item i + 2 before the consumers finished item i (it waits
  // for the release of item i + 1's own stages).  Shorter items (kb < 8, small multiplies) keep the
  // barriers.  (The host never splits K below 64 stages, so every item has >= 1 stage.)
  const bool sync_items = nst / nsplit < STAGES + 1;

  // pinwheel of the 11 x 11 subtiles around the centre (5, 5): warp 0 rows 0-4 x cols 0-5 (+ centre),
  // warp 1 rows 0-5 x cols 6-10, warp 2 rows 6-10 x cols 5-10, warp 3 rows 5-10 x cols 0-4
  // (two warps per sub-partition: sp = warp % 4 owns a rectangle, h = warp / 4 one half of it)
  const int sp = warp & 3, hh = warp >> 2;
  const int r0 = sp == 0 ? 0 : sp == 1 ? 3 * hh : sp == 2 ? 6 : 5 + 3 * hh;
  const int c0 = sp == 0 ? 3 * hh : sp == 1 ? 6 : sp == 2 ? 5 + 3 * hh : 0;
  const bool tall = sp == 0 || sp == 2;  // 5 x 3, else 3 x 5

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init((uint32_t)__cvta_generic_to_shared(&full[s]), 1);
      mbar_init((uint32_t)__cvta_generic_to_shared(&empty[s]), WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  int stage = 0;
  uint32_t phase = 0;
  int par = 0;
  for (int64_t item = blockIdx.x; item < ngroups * nsplit; item += gridDim.x, par ^= 1) {
    const int64_t grp = item % ngroups;
    const int split = (int)(item / ngroups);
    const int st0 = (int)((int64_t)nst * split / nsplit), st1 = (int)((int64_t)nst * (split + 1) / nsplit);
    const int64_t q0 = grp * RUNS;
    if (producer) {  // rank the 16 runs' first A / B blocks: row ri, column cj of the square
      const int64_t q = RUN(q0 + (lane & 15));
      const int a0 = trip[3 * (q * kb)], b0 = trip[3 * (q * kb) + 1];
      int ri = 0, cj = 0;
      for (int o = 0; o < 16; ++o) {
        const int ao = __shfl_sync(0xffffffffu, a0, o), bo = __shfl_sync(0xffffffffu, b0, o);
        // count distinct smaller values (first occurrence of each value counts)
        bool firsta = true, firstb = true;
        for (int p2 = 0; p2 < o; ++p2) {
          firsta &= __shfl_sync(0xffffffffu, a0, p2) != ao;
          firstb &= __shfl_sync(0xffffffffu, b0, p2) != bo;
        }
        ri += (firsta && ao < a0) ? 1 : 0;
        cj += (firstb && bo < b0) ? 1 : 0;
      }
      if (lane < 16) {
        s_dst[par][ri][cj] =
            partial ? partial + ((int64_t)split * nruns + q) * BB : C + (int64_t)trip[3 * (q * kb) + 2] * BB;
        if (cj == 0) s_rowrep[ri] = lane;
        if (ri == 0) s_colrep[cj] = lane;
      }
      __syncwarp();  // s_rowrep / s_colrep are read by the producer lanes; s_dst is released by the full barrier
    }
    if (sync_items) __syncthreads();
    if (producer) {
      // lane l < 16: l < 8 -> A row l / 2, block kk0 + (l & 1); else B column (l - 8) / 2
      const int isb = lane >= 8 ? 1 : 0, u = (lane & 7) >> 1, j = lane & 1;
      const bool owner = lane < 16;
      const int64_t q = RUN(q0 + (owner ? (isb ? s_colrep[u] : s_rowrep[u]) : 0));
      const double* base = isb ? B : A;
      // the stage's block indices come from the stack list in global memory: load them two stages ahead,
      // so the load latency overlaps the wait for a free stage instead of following it (ncu: the producer's
      // dependent trip load was the refill's critical path, consumers waited on full stages 5 % of the time)
      auto blk_of = [&](int st) -> int64_t {
        const int kk = st * KK + j;
        return (owner && st < st1 && kk < kb) ? (int64_t)trip[3 * (q * kb + kk) + isb] : 0;
      };
      int64_t blk0 = blk_of(st0), blk1 = blk_of(st0 + 1);
      for (int st = st0; st < st1; ++st) {
        const int kk = st * KK + j;
        const bool valid = owner && kk < kb;
        const int64_t blk = blk0;
        blk0 = blk1;
        blk1 = blk_of(st + 2);
        const uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[stage]);
        if (lane == 0) mbar_wait((uint32_t)__cvta_generic_to_shared(&empty[stage]), phase ^ 1);
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        if (lane == 0) mbar_expect_tx(fb, (uint32_t)__popc(vm) * BLK_BYTES);
        __syncwarp();
        if (valid) {
          const int off = isb ? BOFF + u * SLOTB + j * KK1B : u * SLOT + j * BB;
          bulk_g2s(sbase + (uint32_t)(stage * STAGE + off) * 8u, base + blk * BB, BLK_BYTES, fb);
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    } else if (warp == centre_warp && tall) {  // the centre subtile rides with one warp (default 5: SMSP 1,
      // so SMSP 0, which also issues the producer warp, keeps 30 DMMAs per k-step)
      s22q_consume<5, 3, true>(full, empty, sbase, stage, phase, st0, st1, Krun, r0, c0, g, t, lane, s_dst[par],
                               partial != nullptr, alpha, beta_first);
    } else if (warp == centre_warp) {
      s22q_consume<3, 5, true>(full, empty, sbase, stage, phase, st0, st1, Krun, r0, c0, g, t, lane, s_dst[par],
                               partial != nullptr, alpha, beta_first);
    } else if (tall) {
      s22q_consume<5, 3, false>(full, empty, sbase, stage, phase, st0, st1, Krun, r0, c0, g, t, lane, s_dst[par],
                                partial != nullptr, alpha, beta_first);
    } else {
      s22q_consume<3, 5, false>(full, empty, sbase, stage, phase, st0, st1, Krun, r0, c0, g, t, lane, s_dst[par],
                                partial != nullptr, alpha, beta_first);
    }
    if (sync_items) __syncthreads();
  }
}

// Fixed-order split-K reduction of the smm partials: C_blk = (first ? beta*C : C) + alpha * sum_s P_s.
__global__ void smm_splitk_reduce(const int32_t* __restrict__ trip, int64_t nruns, int64_t kb, int bb, int nsplit,
                                  const double* __restrict__ partial, double* __restrict__ C, double alpha,
                                  double beta_first) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nruns * bb;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / bb, w = e - q * bb;
    double sum = partial[e];
    for (int s = 1; s < nsplit; ++s) sum += partial[(int64_t)s * nruns * bb + e];
    double* p = C + (int64_t)trip[3 * (q * kb) + 2] * bb + w;
    const double v = alpha * sum;
    *p = (beta_first == 0.0) ? v : beta_first * *p + v;
  }
}

// ============================================================================ bs 64: TMA tensor staging
// 2 runs per CTA (2 x 2 consumer warps of 32 x 32 per 64 x 64 C block), a stage = half a k-block
// (32 k = 8 DMMA k-steps).  The A and B arenas are viewed as 2-D tensors of 64-double rows (a block
// column each); per stage a staged A block is 4 TMA boxes [32 k][16 m] and a staged B block 2 boxes
// [64 n][16 k], all with the 128-B swizzle, i.e. 6 TMA ops per distinct block instead of one copy per
// column.  MMA k-slot t of k-step ks reads k = 16(ks/4) + 2(ks%4) + (t&1) + 8(t>>1): conflict-free B
// fragments (as in dgemm), 2-way on A.
namespace s64 {
constexpr int BS = 64, BB = 4096, KS = 32, RUNS = 2, WARPS = 8, P = 4, STAGES = 3;
constexpr int SLOT = BS * KS;                       // doubles (16 KB)
constexpr int STAGE = P * SLOT;
constexpr size_t SMEM = (size_t)STAGES * STAGE * 8 + 1024;  // + 1024-B alignment slack for the swizzle
static_assert(SMEM + 512 <= 232448, "shared memory");
}  // namespace s64

__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}

__global__ void __launch_bounds__((s64::WARPS + 1) * 32, 1)
    smm64_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const int32_t* __restrict__ trip, int64_t nruns, int64_t kb, double* __restrict__ C, double alpha,
                 double beta_first, int nsplit, double* __restrict__ partial) {
  using namespace s64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  __shared__ int s_rep[P], s_isb[P], s_ia[RUNS], s_ib[RUNS], s_n;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp == WARPS;
  const int run = warp >> 2, wsub = warp & 3, wm = wsub >> 1, wn = wsub & 1;
  const int nst = (int)(kb * 2);  // two stages per k-block
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const int64_t ngroups = (nruns + RUNS - 1) / RUNS;
  const int g = lane >> 2, t = lane & 3;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init((uint32_t)__cvta_generic_to_shared(&full[s]), 1);
      mbar_init((uint32_t)__cvta_generic_to_shared(&empty[s]), WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (producer && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
  }
  __syncthreads();

  // per-lane fragment offsets inside a stage (bytes), k-step ks, lane (g, t)
  auto kof = [&](int ks) { return 16 * (ks >> 2) + 2 * (ks & 3) + (t & 1) + 8 * (t >> 1); };
  int stage = 0;
  uint32_t phase = 0;
  // work item = (group, K split); with nsplit > 1 each item accumulates stages [st0, st1) of its runs
  // into `partial` (reduced later in a fixed order) instead of updating C
  for (int64_t item = blockIdx.x; item < ngroups * nsplit; item += gridDim.x) {
    const int64_t grp = item % ngroups;
    const int split = (int)(item / ngroups);
    const int st0 = (int)((int64_t)nst * split / nsplit), st1 = (int)((int64_t)nst * (split + 1) / nsplit);
    const int64_t q0 = grp * RUNS;
    const int n_g = (int)(nruns - q0 < RUNS ? nruns - q0 : RUNS);
    if (producer) {
      const Uniq u = uniq(trip, q0, 0, n_g, kb, lane);  // <= 2 + 2 distinct blocks: always fits P = 4
      const int na = __popc(u.lead_a);
      if (u.act) {
        const int la = __ffs(u.ma) - 1, lb = __ffs(u.mb) - 1;
        const int ia = __popc(u.lead_a & ((1u << la) - 1));
        const int ib = na + __popc(u.lead_b & ((1u << lb) - 1));
        s_ia[lane] = ia;
        s_ib[lane] = ib;
        if (la == lane) {
          s_rep[ia] = lane;
          s_isb[ia] = 0;
        }
        if (lb == lane) {
          s_rep[ib] = lane;
          s_isb[ib] = 1;
        }
      }
      if (lane == 0) s_n = na + __popc(u.lead_b);
    }
    __syncthreads();
    const int nslots = s_n;
    if (producer) {
      const bool owner = lane < nslots;
      const int64_t q = q0 + (owner ? s_rep[lane] : 0);
      const int isb = owner ? s_isb[lane] : 0;
      for (int st = st0; st < st1; ++st) {
        const int kk = st >> 1, h = st & 1;
        const uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[stage]);
        if (lane == 0) {
          mbar_wait((uint32_t)__cvta_generic_to_shared(&empty[stage]), phase ^ 1);
          mbar_expect_tx(fb, (uint32_t)nslots * SLOT * 8);
        }
        __syncwarp();
        if (owner) {
          const int blk = trip[3 * (q * kb + kk) + isb];
          const uint32_t dst = sbase + (uint32_t)(stage * STAGE + lane * SLOT) * 8u;
          if (!isb) {
#pragma unroll
            for (int sb = 0; sb < 4; ++sb) tma2d(dst + sb * 4096, &tmA, sb * 16, blk * 64 + h * 32, fb);
          } else {
#pragma unroll
            for (int j = 0; j < 2; ++j) tma2d(dst + j * 8192, &tmB, h * 32 + j * 16, blk * 64, fb);
          }
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    } else {
      const bool active = run < n_g;
      const int ia = active ? s_ia[run] : 0, ib = active ? s_ib[run] : 0;
      double acc[4][4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      for (int st = st0; st < st1; ++st) {
        mbar_wait((uint32_t)__cvta_generic_to_shared(&full[stage]), phase);
        if (active) {
          const uint32_t sA = sbase + (uint32_t)(stage * STAGE + ia * SLOT) * 8u;
          const uint32_t sB = sbase + (uint32_t)(stage * STAGE + ib * SLOT) * 8u;
#pragma unroll
          for (int ks = 0; ks < KS / 4; ++ks) {
            const int k = kof(ks);
            double a[4], b[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {  // A (m, k): box m/16, row k, 16-B chunk ((m%16)/2) ^ (k%8)
              const int m = wm * 32 + mi * 8 + g, mm = m & 15;
              a[mi] = lds64(sA + (m >> 4) * 4096 + k * 128 + ((((mm >> 1) ^ (k & 7))) << 4) + ((mm & 1) << 3));
            }
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) {  // B (k, n): box k/16, row n, chunk ((k%16)/2) ^ (n%8)
              const int n = wn * 32 + ni * 8 + g, kk16 = k & 15;
              b[ni] = lds64(sB + (k >> 4) * 8192 + n * 128 + ((((kk16 >> 1) ^ (n & 7))) << 4) + ((kk16 & 1) << 3));
            }
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive((uint32_t)__cvta_generic_to_shared(&empty[stage]));
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (active) {
        double* cb = partial ? partial + ((int64_t)split * nruns + q0 + run) * BB
                             : C + (int64_t)trip[3 * ((q0 + run) * kb) + 2] * BB;
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int m = wm * 32 + mi * 8 + g, n = wn * 32 + ni * 8 + 2 * t + j;
              double* p = cb + m + n * BS;
              if (partial) {
                *p = acc[mi][ni][j];
              } else {
                const double v = alpha * acc[mi][ni][j];
                *p = (beta_first == 0.0) ? v : beta_first * *p + v;
              }
            }
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_smm64(const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const double* B, double* C,
                         double alpha, double beta_first, int nsplit, double* partial, int64_t a_blocks,
                         int64_t b_blocks, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(smm64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s64::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap tmA, tmB;
  if (!make_map_2d(&tmA, A, 64, (uint64_t)a_blocks * 64, 512, 16, 32) ||
      !make_map_2d(&tmB, B, 64, (uint64_t)b_blocks * 64, 512, 16, 64))
    return cudaErrorInvalidValue;
  const int64_t ngroups = (nruns + s64::RUNS - 1) / s64::RUNS;
  if (nsplit < 1 || !partial) nsplit = 1;
  const unsigned grid = (unsigned)std::min<int64_t>(ngroups * nsplit, (int64_t)num_sms());
  smm64_kernel<<<grid, (s64::WARPS + 1) * 32, s64::SMEM, st>>>(tmA, tmB, trip, nruns, kb, C, alpha, beta_first, nsplit,
                                                               nsplit > 1 ? partial : nullptr);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || nsplit == 1) return e;
  const int64_t n = nruns * s64::BB;
  smm_splitk_reduce<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16), 256, 0, st>>>(
      trip, nruns, kb, s64::BB, nsplit, partial, C, alpha, beta_first);
  return cudaGetLastError();
}

// DBM_SMM22Q_CENTRE=<warp 0..7> picks the consumer warp that also computes the square's centre subtile.
int smm22q_centre_warp() {
  static const int w = [] {
    const char* e = getenv("DBM_SMM22Q_CENTRE");
    const int v = e ? atoi(e) : 5;
    return v >= 0 && v < s22q::WARPS ? v : 5;
  }();
  return w;
}

cudaError_t launch_smm22q(const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const double* B, double* C,
                          double alpha, double beta_first, int nsplit, double* partial, cudaStream_t st,
                          const int32_t* runs = nullptr, const int* d_count = nullptr) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(smm22q_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s22q::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t ngroups = nruns / s22q::RUNS;
  if (nsplit < 1 || !partial) nsplit = 1;
  const unsigned grid = (unsigned)std::min<int64_t>(ngroups * nsplit, (int64_t)num_sms());
  smm22q_kernel<<<grid, (s22q::WARPS + 1) * 32, s22q::SMEM, st>>>(trip, nruns, kb, A, B, C, alpha, beta_first, nsplit,
                                                                  nsplit > 1 ? partial : nullptr, runs, d_count, smm22q_centre_warp());
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || nsplit == 1) return e;
  const int64_t n = nruns * s22q::BB;
  smm_splitk_reduce<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16), 256, 0, st>>>(
      trip, nruns, kb, s22q::BB, nsplit, partial, C, alpha, beta_first);
  return cudaGetLastError();
}

cudaError_t launch_smm22(const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const double* B, double* C,
                         double alpha, double beta_first, int nsplit, double* partial, cudaStream_t st,
                         const int32_t* runs = nullptr, const int* d_count = nullptr) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(smm22_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s22::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t ngroups = (nruns + s22::RUNS - 1) / s22::RUNS;
  if (nsplit < 1 || !partial) nsplit = 1;
  const unsigned grid = (unsigned)std::min<int64_t>(ngroups * nsplit, (int64_t)num_sms());
  smm22_kernel<<<grid, (s22::WARPS + 1) * 32, s22::SMEM, st>>>(trip, nruns, kb, A, B, C, alpha, beta_first, nsplit,
                                                               nsplit > 1 ? partial : nullptr, runs, d_count);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || nsplit == 1) return e;
  const int64_t n = nruns * s22::BB;
  smm_splitk_reduce<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16), 256, 0, st>>>(
      trip, nruns, kb, s22::BB, nsplit, partial, C, alpha, beta_first);
  return cudaGetLastError();
}


// ---------------------------------------------------------------- squares inside other traversals
// When the bisection does not visit the local grid as whole squares (63,360^3 bs 22: 2,880 = 64 x 45
// blocks per side), the aligned 4 x 4 squares of C blocks whose 16 runs all lie in the current chunk of
// runs are still executed by the unpadded kernel, through a list of their run indices; the remaining
// runs go, in traversal order, to the 8-run kernel.  Lists are built with stable compactions (CUB
// DeviceSelect), so the CTA work assignment, and the result, are deterministic.
__global__ void inverse_traversal_kernel(const int32_t* __restrict__ li, const int32_t* __restrict__ lj, int64_t n,
                                         int64_t nloc, int32_t* __restrict__ pos) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    pos[(int64_t)li[q] * nloc + lj[q]] = (int32_t)q;
}

__global__ void square_flags_kernel(const int32_t* __restrict__ pos, int64_t nloc, int64_t nsq, int64_t sqc,
                                    int64_t q0, int64_t n, uint8_t* __restrict__ flag) {
  for (int64_t sq = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sq < nsq; sq += (int64_t)gridDim.x * blockDim.x) {
    const int64_t I = sq / sqc, J = sq - I * sqc;
    bool in = true;
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) {
        const int64_t p = pos[(4 * I + a) * nloc + 4 * J + b];
        in &= p >= q0 && p < q0 + n;
      }
    flag[sq] = in ? 1 : 0;
  }
}

__global__ void leftover_flags_kernel(const int32_t* __restrict__ li, const int32_t* __restrict__ lj, int64_t q0,
                                      int64_t n, int64_t sqr, int64_t sqc, const uint8_t* __restrict__ sqflag,
                                      uint8_t* __restrict__ flag) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t I = li[q0 + q] / 4, J = lj[q0 + q] / 4;
    flag[q] = (I < sqr && J < sqc && sqflag[I * sqc + J]) ? 0 : 1;
  }
}

__global__ void square_runs_kernel(const int32_t* __restrict__ pos, int64_t nloc, int64_t sqc,
                                   const int32_t* __restrict__ sq_ids, const int* __restrict__ nsel, int64_t q0,
                                   int32_t* __restrict__ runs, int* __restrict__ nruns16) {
  const int64_t total = (int64_t)*nsel * 16;
  if (blockIdx.x == 0 && threadIdx.x == 0) *nruns16 = (int)total;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sq = sq_ids[e / 16], I = sq / sqc, J = sq - I * sqc;
    const int r = (int)(e % 16);
    runs[e] = (int32_t)(pos[(4 * I + r / 4) * nloc + 4 * J + r % 4] - q0);
  }
}

inline unsigned mixed_grid(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16));
}
}  // namespace

bool smm_has_tensor_path(int bs) { return bs == 22 || bs == 64; }

void launch_inverse_traversal(const int32_t* li, const int32_t* lj, int64_t n, int64_t nloc, int32_t* pos,
                              cudaStream_t st) {
  if (n > 0) inverse_traversal_kernel<<<mixed_grid(n), 256, 0, st>>>(li, lj, n, nloc, pos);
}

size_t smm22_mixed_temp_bytes(int64_t n) {
  size_t b = 0;
  cub::CountingInputIterator<int32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, b, it, (const uint8_t*)nullptr, (int32_t*)nullptr, (int*)nullptr,
                             (int)std::max<int64_t>(n, 1));
  return b;
}

cudaError_t launch_smm22_mixed(const int32_t* trip, int64_t q0, int64_t nruns, int64_t kb, const double* A,
                               const double* B, double* C, double alpha, double beta_first, const int32_t* li,
                               const int32_t* lj, const int32_t* pos, int64_t mloc, int64_t nloc, const SmmMixedWS& w,
                               cudaStream_t st, int* launches) {
  if (nruns <= 0 || kb <= 0) return cudaSuccess;
  const int64_t sqr = mloc / 4, sqc = nloc / 4, nsq = sqr * sqc;
  cudaError_t e;
  if (nsq > 0) {
    square_flags_kernel<<<mixed_grid(nsq), 256, 0, st>>>(pos, nloc, nsq, sqc, q0, nruns, w.sqflag);
    size_t tb = w.temp_bytes;
    e = cub::DeviceSelect::Flagged(w.temp, tb, cub::CountingInputIterator<int32_t>(0), w.sqflag, w.sq_ids,
                                   w.counts, (int)nsq, st);
    if (e != cudaSuccess) return e;
    square_runs_kernel<<<mixed_grid(nruns), 256, 0, st>>>(pos, nloc, sqc, w.sq_ids, w.counts, q0, w.runs_sq,
                                                          w.counts + 1);
    e = launch_smm22q(trip, nruns, kb, A, B, C, alpha, beta_first, 1, nullptr, st, w.runs_sq, w.counts + 1);
    if (e != cudaSuccess) return e;
    if (launches) *launches += 4;
  } else {
    cudaMemsetAsync(w.sqflag, 0, 1, st);
  }
  leftover_flags_kernel<<<mixed_grid(nruns), 256, 0, st>>>(li, lj, q0, nruns, sqr, sqc, w.sqflag, w.runflag);
  size_t tb = w.temp_bytes;
  e = cub::DeviceSelect::Flagged(w.temp, tb, cub::CountingInputIterator<int32_t>(0), w.runflag, w.runs_left,
                                 w.counts + 2, (int)nruns, st);
  if (e != cudaSuccess) return e;
  e = launch_smm22(trip, nruns, kb, A, B, C, alpha, beta_first, 1, nullptr, st, w.runs_left, w.counts + 2);
  if (launches) *launches += 3;
  return e != cudaSuccess ? e : cudaGetLastError();
}

int smm_group_runs(int bs) { return bs == 22 ? s22::RUNS : (bs == 64 ? Cfg64::RUNS : 1); }

// Split the runs' K across CTAs when the groups alone cannot fill the GPU (long, few runs: the
// rectangular configs on several GPUs).  Returns 1 when no split is needed.
bool bisection_squares(int64_t mloc, int64_t nloc, int64_t side) {
  if (mloc == side && nloc == side) return true;
  if (mloc < side || nloc < side) return false;
  if (mloc >= nloc) return mloc % 2 == 0 && bisection_squares(mloc / 2, nloc, side);  // rows split on ties
  return nloc % 2 == 0 && bisection_squares(mloc, nloc / 2, side);
}

int smm_pick_split(int bs, int64_t nruns, int64_t kb, bool squares) {
  if (bs != 22 && bs != 64) return 1;
  const int64_t sms = num_sms();
  const int64_t ngroups = bs == 22 ? (nruns + (squares ? s22q::RUNS : s22::RUNS) - 1) / (squares ? s22q::RUNS : s22::RUNS)
                                   : (nruns + s64::RUNS - 1) / s64::RUNS;
  const int64_t nst = bs == 22 ? (kb * s22::BS + s22::KS - 1) / s22::KS : kb * 2;
  if (ngroups >= 2 * sms) return 1;
  int best = 1;
  double best_t = 1e300;
  for (int s = 1; s <= 16 && nst / s >= 64; ++s) {
    const double rounds = (double)((ngroups * s + sms - 1) / sms);
    const double t = rounds / s * (1.0 + 0.01 * (s - 1));  // + reduction traffic
    if (t < best_t * (1.0 - 1e-9)) {
      best_t = t;
      best = s;
    }
  }
  return best;
}

cudaError_t launch_smm_tc(int bs, const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const double* B,
                          double* C, double alpha, double beta_first, int nsplit, double* partial, cudaStream_t st,
                          int64_t a_blocks, int64_t b_blocks, bool squares) {
  if (nruns <= 0 || kb <= 0) return cudaSuccess;
  if (bs == 22 && squares && nruns % s22q::RUNS == 0)
    return launch_smm22q(trip, nruns, kb, A, B, C, alpha, beta_first, nsplit, partial, st);
  if (bs == 22) return launch_smm22(trip, nruns, kb, A, B, C, alpha, beta_first, nsplit, partial, st);
  if (bs == 64 && a_blocks > 0 && b_blocks > 0 && ((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0)
    return launch_smm64(trip, nruns, kb, A, B, C, alpha, beta_first, nsplit, partial, a_blocks, b_blocks, st);
  if (bs == 64) return launch_group<Cfg64>(trip, nruns, kb, A, B, C, alpha, beta_first, st);
  return cudaErrorInvalidValue;
}

}  // namespace dbm

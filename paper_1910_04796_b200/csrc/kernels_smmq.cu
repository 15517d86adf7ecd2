// smmq — the blocked path's small-block products on R x R squares of C-block runs, for block sizes whose
// 8 x 8 DMMA fragments pad worst (bs 4, 5, 6, 9: the per-run kernel computes (8 ceil(bs/8))^2 outputs per
// bs^2 useful ones, 39 % useful at bs 5, 32 % at bs 9).  The LIBCUSMM role for the small sizes of CP2K
// basis sets; the generalisation of smm22q (kernels_smm.cu) to other sizes.
//
// When the bisection traversal visits the local grid as whole R x R squares (R a power of two: an R x R
// square is then R^2 consecutive runs in Morton order, R6 / the test pin on power-of-two traversals), a
// CTA takes a square: R A block rows and R B block columns per k-block, a (R bs) x (R bs) C region with
// R bs a multiple of 8, i.e. U x U DMMA subtiles with no padding.  The K of a run is the concatenation of
// its kb blocks; a stage holds KK k-blocks with KK bs a multiple of 4, so k-steps never straddle a stage.
// All warps stage the next stages' blocks with 8-byte cp.async (any block alignment: odd bs^2) into a
// STAGES-deep ring, then each warp multiplies its rectangle of the U x U subtiles (2 x 4 or 3 x 4 warps).
// The last stage of a run whose kb is not a multiple of KK is zero-predicated in registers.
#include <algorithm>

#include "dbm_internal.h"

namespace dbm {

namespace {

template <int BS>
struct SQ {
  static constexpr int R = BS == 5 ? 16 : (BS == 26 ? 4 : 8);  // R bs = 80, 32, 48, 72, 104, 104
  // k-blocks per stage: KK bs a multiple of 4 and >= 32 (8+ k-steps per stage), 2 R KK dividing the 256 threads
  static constexpr int KK = BS == 9 ? 4 : 8;
  static constexpr int KS = KK * BS, NKS = KS / 4;
  static constexpr int BB = BS * BS;
  static constexpr int U = R * BS / 8;
  // warp grid WR x WC over the U x U subtiles: 2 x 4 warps, 3 x 4 (384 threads) for the 13 x 13 squares
  // so the accumulators fit the registers
  static constexpr int WR = U >= 12 ? 3 : 2, WC = 4, THREADS = WR * WC * 32;
  static constexpr int RI = (U + WR - 1) / WR, CJ = (U + WC - 1) / WC;  // a warp's rectangle, at most
  static constexpr int NBLK = 2 * R * KK;                    // blocks per stage (A rows then B columns)
  static constexpr int STAGE = NBLK * BB;                    // doubles
  static constexpr int STAGES = (200 * 1024 / (STAGE * 8)) > 6 ? 6 : (200 * 1024 / (STAGE * 8));
  static_assert(R * BS % 8 == 0 && KS % 4 == 0 && STAGES >= 2, "square shape");
  static constexpr size_t SMEM = (size_t)STAGES * STAGE * 8;
};

__device__ __forceinline__ double q_lds(const double* p) { return *p; }

__device__ __forceinline__ void q_dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// Morton position of (r, c) inside a square: c's bits at even, r's bits at odd positions (i-major)
__device__ __forceinline__ int morton(int r, int c) {
  int k = 0;
#pragma unroll
  for (int b = 0; b < 5; ++b) k |= (((c >> b) & 1) << (2 * b)) | (((r >> b) & 1) << (2 * b + 1));
  return k;
}

template <int BS>
__global__ void __launch_bounds__(SQ<BS>::THREADS, 1)
    smmq_kernel(const int32_t* __restrict__ trip, int64_t nsq, int64_t kb, const double* __restrict__ A,
                const double* __restrict__ B, double* __restrict__ C, double alpha, double beta_first) {
  using Q = SQ<BS>;
  extern __shared__ __align__(16) double qsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wr = warp / Q::WC, wc = warp % Q::WC;
  // subtile rows [i0, i0 + ni), columns [c_lo, c_lo + nj): the U rows / columns split as evenly as possible
  const int i0 = (Q::U / Q::WR) * wr + min(wr, Q::U % Q::WR), ni = Q::U / Q::WR + (wr < Q::U % Q::WR ? 1 : 0);
  const int c_lo = (Q::U / Q::WC) * wc + min(wc, Q::U % Q::WC), nj = Q::U / Q::WC + (wc < Q::U % Q::WC ? 1 : 0);
  const int64_t Krun = kb * BS;
  const int nst = (int)((Krun + Q::KS - 1) / Q::KS);
  // lane constants: fragment rows / columns -> (block, element) offsets inside a stage
  int rowoff[Q::RI], coloff[Q::CJ];
#pragma unroll
  for (int i = 0; i < Q::RI; ++i) {
    const int m = 8 * (i0 + i) + g, r = m / BS, x = m - r * BS;
    rowoff[i] = r * Q::KK * Q::BB + x;  // A block (r, kk): element (x, z) at z*BS + x
  }
#pragma unroll
  for (int j = 0; j < Q::CJ; ++j) {
    const int n = 8 * (c_lo + j) + g, c = n / BS, y = n - c * BS;
    coloff[j] = (Q::R + c) * Q::KK * Q::BB + y * BS;  // B block (kk, c): element (z, y) at y*BS + z
  }
  // this thread's staging share: block tid % NBLK (THREADS / NBLK threads per block)
  const int my_blk = tid % Q::NBLK, blk_threads = Q::THREADS / Q::NBLK;
  static_assert(Q::THREADS % Q::NBLK == 0, "staging split");
  const int my_part = tid / Q::NBLK;  // element stride = blk_threads
  for (int64_t sq = blockIdx.x; sq < nsq; sq += gridDim.x) {
    const int64_t q0 = sq * (int64_t)Q::R * Q::R;
    const bool isb = my_blk >= Q::R * Q::KK;
    const int bi = isb ? my_blk - Q::R * Q::KK : my_blk;  // (row or column) * KK + kk
    const int rc = bi / Q::KK, kk_in = bi - rc * Q::KK;
    const int64_t run = q0 + (isb ? morton(0, rc) : morton(rc, 0));
    auto stage_in = [&](int st) {  // blocks of stage st -> ring slot st % STAGES
      double* dst = qsm + (size_t)(st % Q::STAGES) * Q::STAGE + (size_t)my_blk * Q::BB;
      const int64_t kk = (int64_t)st * Q::KK + kk_in;
      if (tid < Q::NBLK * blk_threads && kk < kb) {
        const double* src = (isb ? B : A) + (int64_t)trip[3 * (run * kb + kk) + (isb ? 1 : 0)] * Q::BB;
        for (int e = my_part; e < Q::BB; e += blk_threads)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + e)),
                       "l"(src + e)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[Q::RI][Q::CJ][2];
#pragma unroll
    for (int i = 0; i < Q::RI; ++i)
#pragma unroll
      for (int j = 0; j < Q::CJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int s = 0; s < Q::STAGES - 1; ++s) stage_in(s);  // (stages past the run: empty groups)
    for (int st = 0; st < nst; ++st) {
      stage_in(st + Q::STAGES - 1);
      asm volatile("cp.async.wait_group %0;" ::"n"(Q::STAGES - 1) : "memory");
      __syncthreads();
      const double* sb = qsm + (size_t)(st % Q::STAGES) * Q::STAGE;
      const int64_t kvalid = Krun - (int64_t)st * Q::KS;
#pragma unroll
      for (int ks = 0; ks < Q::NKS; ++ks) {
        const int k = 4 * ks + t, kk = k / BS, z = k - kk * BS;
        const bool ok = kvalid >= Q::KS || k < kvalid;
        const int ka = kk * Q::BB + z * BS, kbo = kk * Q::BB + z;
        double a[Q::RI], b[Q::CJ];
#pragma unroll
        for (int i = 0; i < Q::RI; ++i) a[i] = (ok && i < ni) ? q_lds(sb + rowoff[i] + ka) : 0.0;
#pragma unroll
        for (int j = 0; j < Q::CJ; ++j) b[j] = (ok && j < nj) ? q_lds(sb + coloff[j] + kbo) : 0.0;
#pragma unroll
        for (int i = 0; i < Q::RI; ++i)
#pragma unroll
          for (int j = 0; j < Q::CJ; ++j) q_dmma(acc[i][j], a[i], b[j]);
      }
      __syncthreads();  // slot st % STAGES is refilled by the next iteration's stage_in
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    // epilogue: subtile (i, j), lane (g, t) holds C(8 (i0+i) + g, 8 (c_lo+j) + 2t + jj) of the square
#pragma unroll
    for (int i = 0; i < Q::RI; ++i) {
      if (i >= ni) break;
      const int m = 8 * (i0 + i) + g, r = m / BS, x = m - r * BS;
#pragma unroll
      for (int j = 0; j < Q::CJ; ++j) {
        if (j >= nj) break;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const int n = 8 * (c_lo + j) + 2 * t + jj, c = n / BS, y = n - c * BS;
          const int64_t q = q0 + morton(r, c);
          double* p = C + (int64_t)trip[3 * (q * kb) + 2] * Q::BB + y * BS + x;
          const double v = alpha * acc[i][j][jj];
          *p = beta_first == 0.0 ? v : beta_first * *p + v;
        }
      }
    }
    __syncthreads();  // the next square's first stages reuse the ring
  }
}

template <int BS>
cudaError_t launch_q(const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const double* B, double* C,
                     double alpha, double beta_first, cudaStream_t st) {
  using Q = SQ<BS>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(smmq_kernel<BS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t nsq = nruns / ((int64_t)Q::R * Q::R);
  const unsigned grid = (unsigned)std::min<int64_t>(nsq, (int64_t)num_sms());
  smmq_kernel<BS><<<grid, Q::THREADS, Q::SMEM, st>>>(trip, nsq, kb, A, B, C, alpha, beta_first);
  return cudaGetLastError();
}

}  // namespace

int smmq_side(int bs) {
  switch (bs) {
    case 4: return SQ<4>::R;
    case 5: return SQ<5>::R;
    case 6: return SQ<6>::R;
    case 9: return SQ<9>::R;
    default: return 0;  // (13 x 13-subtile squares, bs 13 / 26: the accumulators spill at any warp grid tried)
  }
}

cudaError_t launch_smmq(int bs, const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const double* B,
                        double* C, double alpha, double beta_first, cudaStream_t st) {
  if (nruns <= 0 || kb <= 0) return cudaSuccess;
  switch (bs) {
    case 4: return launch_q<4>(trip, nruns, kb, A, B, C, alpha, beta_first, st);
    case 5: return launch_q<5>(trip, nruns, kb, A, B, C, alpha, beta_first, st);
    case 6: return launch_q<6>(trip, nruns, kb, A, B, C, alpha, beta_first, st);
    case 9: return launch_q<9>(trip, nruns, kb, A, B, C, alpha, beta_first, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dbm

// HBM-bound data-movement kernels of the hot path (sm_100a):
//   fill (synthetic inputs, untimed), densify (§III), undensify with alpha/beta
//   (§III), panel packing for the blocked path (Cannon panels).
// Bound: HBM.  Algorithmic bytes: densify 16 B/element, undensify 24 B/element (16 if beta == 0),
// pack 16 B/element.
#include <algorithm>
#include <cstdlib>

#include "dbm_internal.h"

namespace dbm {

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t work, int per_block = kThreads) {
  int64_t g = (work + per_block - 1) / per_block;
  int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

// ---- counter-based generator, DESIGN.md §4 (device copy of the definition) ----
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

__global__ void fill_kernel(double* __restrict__ arena, int64_t total, int64_t nloc, int bs, int pr, int pc, int r,
                            int c, uint64_t key, int kind) {
  const int64_t bb = (int64_t)bs * bs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t slot = e / bb, w = e - slot * bb;
    int64_t y = w / bs, x = w - y * bs;
    int64_t li = slot / nloc, lj = slot - li * nloc;
    uint64_t gi = (uint64_t)((r + li * pr) * bs + x), gj = (uint64_t)((c + lj * pc) * bs + y);
    uint64_t bits = mix64(key ^ mix64((gi << 32) ^ gj));
    double v;
    if (kind == 1) {
      v = (double)((int)((bits >> 32) % 5u) - 2);
    } else {
      double u = __dmul_rn((double)(bits >> 11), 0x1.0p-53);
      v = __dsub_rn(__dmul_rn(2.0, u), 1.0);
    }
    arena[e] = v;
  }
}

// ---- densify A panel: blocks (li, kcol0 + q*kstride) -> dense (mloc*bs) x (nk*bs) ----
// One CTA per (li, group of G consecutive q): stage G blocks in padded shared memory, write
// rows of G*bs contiguous doubles (layout 1) or copy columns (layout 0).
template <int G>
__global__ void densify_cols_kernel(const double* __restrict__ arena, int64_t nloc, int bs, int64_t kcol0,
                                    int64_t kstride, int64_t nk, double* __restrict__ dense, int64_t ld, int layout) {
  extern __shared__ double sm[];
  const int64_t bb = (int64_t)bs * bs;
  const int pitch = bs + 1;  // padded column pitch (bank-conflict free transpose)
  const int64_t ngroups = (nk + G - 1) / G;
  const int64_t li = blockIdx.x / ngroups;
  const int64_t q0 = (blockIdx.x % ngroups) * G;
  const int g_n = (int)((nk - q0) < G ? (nk - q0) : G);
  if (layout == 0) {  // column-major: each block column is a contiguous run of bs doubles
    for (int g = 0; g < g_n; ++g) {
      const double* src = arena + (li * nloc + kcol0 + (q0 + g) * kstride) * bb;
      for (int t = threadIdx.x; t < bb; t += blockDim.x) {
        int y = t / bs, x = t - y * bs;
        dense[((q0 + g) * bs + y) * ld + li * bs + x] = src[t];
      }
    }
    return;
  }
  for (int g = 0; g < g_n; ++g) {
    const double* src = arena + (li * nloc + kcol0 + (q0 + g) * kstride) * bb;
    for (int t = threadIdx.x; t < bb; t += blockDim.x) {
      int y = t / bs, x = t - y * bs;
      sm[g * bs * pitch + y * pitch + x] = src[t];
    }
  }
  __syncthreads();
  const int w = g_n * bs;
  for (int t = threadIdx.x; t < bs * w; t += blockDim.x) {
    int x = t / w, v = t - x * w;
    int g = v / bs, y = v - g * bs;
    dense[(li * bs + x) * ld + (q0 + g) * bs + y] = sm[g * bs * pitch + y * pitch + x];
  }
}

// ---- densify B panel: blocks (krow0 + q*kstride, lj) -> dense (nk*bs) x (nloc*bs) ----
__global__ void densify_rows_kernel(const double* __restrict__ arena, int64_t nloc, int bs, int64_t krow0,
                                    int64_t kstride, int64_t nk, double* __restrict__ dense, int64_t ld, int layout) {
  const int64_t bb = (int64_t)bs * bs;
  const int64_t rows = nk * bs, total = rows * nloc * bs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    // layout 0 (column-major): e runs down a dense column; layout 1: along a dense row.
    int64_t row, col;
    if (layout == 0) {
      col = e / rows;
      row = e - col * rows;
    } else {
      const int64_t cols = nloc * bs;
      row = e / cols;
      col = e - row * cols;
    }
    int64_t q = row / bs, x = row - q * bs, lj = col / bs, y = col - lj * bs;
    double v = arena[((krow0 + q * kstride) * nloc + lj) * bb + y * bs + x];
    if (layout == 0)
      dense[col * ld + row] = v;
    else
      dense[row * ld + col] = v;
  }
}

// ---- undensify with alpha/beta (and a fixed-order split-K sum) ----
__global__ void undensify_kernel(const double* __restrict__ dense, int64_t ld, int nsplit, int64_t split_stride,
                                 int64_t nloc, int bs, int64_t total, double alpha, double beta,
                                 double* __restrict__ arena) {
  const int64_t bb = (int64_t)bs * bs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t slot = e / bb, w = e - slot * bb;
    int64_t y = w / bs, x = w - y * bs;
    int64_t li = slot / nloc, lj = slot - li * nloc;
    int64_t di = (lj * bs + y) * ld + li * bs + x;
    double d = dense[di];
    for (int s = 1; s < nsplit; ++s) d = __dadd_rn(d, dense[di + s * split_stride]);
    double t = __dmul_rn(alpha, d);
    arena[e] = (beta == 0.0) ? t : __dadd_rn(t, __dmul_rn(beta, arena[e]));
  }
}

// ---- whole-block panel packing (blocked path, zero-copy B) ----
// Row panels: every selected block row is one contiguous run of ncols blocks; 16-byte copies.
__global__ void __launch_bounds__(256) pack_rows_fast(const double2* __restrict__ arena, int64_t row_pairs,
                                                      int64_t row0, int64_t rstride, int64_t nrows,
                                                      double2* __restrict__ out) {
  for (int64_t q = blockIdx.y; q < nrows; q += gridDim.y) {
    const double2* src = arena + (row0 + q * rstride) * row_pairs;
    double2* dst = out + q * row_pairs;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < row_pairs; i += (int64_t)gridDim.x * blockDim.x)
      dst[i] = src[i];
  }
}

// Column panels: block row i's selected blocks (i, col0 + q*cstride) are contiguous bs^2 runs; a CTA row
// (blockIdx.y) per block row, CTAs along x over its blocks, threads over a block's 16-byte pairs (no
// per-element index division).  Out row i starts out_row blocks after row i-1.
__global__ void __launch_bounds__(256) pack_cols_fast(const double2* __restrict__ arena, int64_t bb2, int64_t inner,
                                                      int64_t col0, int64_t cstride, int64_t ncols, int64_t mloc,
                                                      int64_t out_row, double2* __restrict__ out) {
  for (int64_t i = blockIdx.y; i < mloc; i += gridDim.y)
    for (int64_t q = blockIdx.x; q < ncols; q += gridDim.x) {
      const double2* src = arena + (i * inner + col0 + q * cstride) * bb2;
      double2* dst = out + (i * out_row + q) * bb2;
      for (int64_t w = threadIdx.x; w < bb2; w += blockDim.x) dst[w] = src[w];
    }
}

__global__ void pack_blocks_kernel(const double* __restrict__ arena, int64_t nsel, int64_t inner, int64_t outer_stride,
                                   int64_t sel0, int64_t sel_stride, int bs, int by_rows, int64_t other,
                                   double* __restrict__ out) {
  // by_rows: out block (q, j) <- arena block (sel0 + q*sel_stride, j), j < other (row panel of a
  //          matrix with `other` block columns).
  // else   : out block (i, q) <- arena block (i, sel0 + q*sel_stride), i < other, with `inner`
  //          block columns in the arena; out rows are outer_stride blocks apart (0: nsel, dense).
  const int64_t bb = (int64_t)bs * bs;
  const int64_t total = nsel * other * bb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t slot = e / bb, w = e - slot * bb;
    int64_t src, dst = e;
    if (by_rows) {
      int64_t q = slot / other, j = slot - q * other;
      src = ((sel0 + q * sel_stride) * other + j) * bb + w;
    } else {
      int64_t i = slot / nsel, q = slot - i * nsel;
      src = (i * inner + sel0 + q * sel_stride) * bb + w;
      if (outer_stride > 0) dst = (i * outer_stride + q) * bb + w;
    }
    out[dst] = arena[src];
  }
}

// ---- fast paths for the paper's block sizes (compile-time BS: no 64-bit divisions, 16-B accesses) ----
// B panel, column-major: dense[(lj*BS+y)*ld + q*BS+x] = block(krow0+q*kstride, lj)[x + y*BS].
// One thread per (x, x+1) pair; CTAs walk blocks b = q*nloc + lj (block-contiguous reads,
// column-run writes of BS doubles), or lj-major b = lj*nk + q when the panel has few block columns
// and very long rows (the rectangular configs: 22 columns, rows of 6 MB), so the blocks in flight
// write a few dense rows instead of every row of the panel.
template <int BS>
__global__ void __launch_bounds__(256) densify_b_fast(const double* __restrict__ arena, int nloc, int64_t krow0,
                                                      int64_t kstride, int nblk, double* __restrict__ dense,
                                                      int64_t ld, int lj_major) {
  constexpr int BB = BS * BS, PAIRS = BB / 2;
  const int nk = nblk / nloc;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < (int64_t)nblk * PAIRS;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(w / PAIRS), i = 2 * (int)(w - (int64_t)b * PAIRS);
    const int q = lj_major ? b % nk : b / nloc, lj = lj_major ? b / nk : b - (b / nloc) * nloc;
    const int y = i / BS, x = i - y * BS;
    const double2 v = *(const double2*)(arena + ((krow0 + q * kstride) * nloc + lj) * BB + i);
    *(double2*)(dense + ((int64_t)lj * BS + y) * ld + (int64_t)q * BS + x) = v;
  }
}

// A panel, row-major (K-major): dense[(li*BS+x)*ld + q*BS+y] = block(li, kcol0+q*kstride)[x + y*BS].
// A CTA stages G blocks of one block row in shared memory (pitch BS+1) and writes G*BS-long rows.
template <int BS, int G>
__global__ void __launch_bounds__(256) densify_a_fast(const double* __restrict__ arena, int64_t nloc, int64_t kcol0,
                                                      int64_t kstride, int64_t nk, double* __restrict__ dense,
                                                      int64_t ld) {
  constexpr int BB = BS * BS, PITCH = BS + 1;
  __shared__ double sm[G * BS * PITCH];
  const int64_t ngroups = (nk + G - 1) / G;
  const int64_t li = blockIdx.x / ngroups, q0 = (blockIdx.x % ngroups) * G;
  const int gn = (int)(nk - q0 < G ? nk - q0 : G);
  for (int g = 0; g < gn; ++g) {
    const double* src = arena + (li * nloc + kcol0 + (q0 + g) * kstride) * BB;
    for (int i = 2 * threadIdx.x; i < BB; i += 2 * blockDim.x) {
      const double2 v = *(const double2*)(src + i);
      const int y = i / BS, x = i - y * BS;  // x even: (x, y) and (x+1, y)
      sm[g * BS * PITCH + y * PITCH + x] = v.x;
      sm[g * BS * PITCH + y * PITCH + x + 1] = v.y;
    }
  }
  __syncthreads();
  const int w = gn * BS;  // row segment length (even)
  for (int i = 2 * threadIdx.x; i < BS * w; i += 2 * blockDim.x) {
    const int x = i / w, v = i - x * w;  // v even, (v, v+1) inside one block (BS even)
    const int g = v / BS, y = v - g * BS;
    double2 o;
    o.x = sm[g * BS * PITCH + y * PITCH + x];
    o.y = sm[g * BS * PITCH + (y + 1) * PITCH + x];
    *(double2*)(dense + (li * BS + x) * ld + q0 * BS + v) = o;
  }
}

// Undensify with alpha/beta: block b = (li, lj), pair (x, x+1) of column y.
template <int BS>
__global__ void __launch_bounds__(256) undensify_fast(const double* __restrict__ dense, int64_t ld, int nsplit,
                                                      int64_t split_stride, int nloc, int nblk, double alpha,
                                                      double beta, double* __restrict__ arena) {
  constexpr int BB = BS * BS, PAIRS = BB / 2;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < (int64_t)nblk * PAIRS;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(w / PAIRS), i = 2 * (int)(w - (int64_t)b * PAIRS);
    const int li = b / nloc, lj = b - li * nloc;
    const int y = i / BS, x = i - y * BS;
    const int64_t di = ((int64_t)lj * BS + y) * ld + (int64_t)li * BS + x;
    double2 d = *(const double2*)(dense + di);
    for (int s = 1; s < nsplit; ++s) {
      const double2 e = *(const double2*)(dense + di + s * split_stride);
      d.x = __dadd_rn(d.x, e.x);
      d.y = __dadd_rn(d.y, e.y);
    }
    double2* p = (double2*)(arena + (int64_t)b * BB + i);
    double2 o;
    o.x = __dmul_rn(alpha, d.x);
    o.y = __dmul_rn(alpha, d.y);
    if (beta != 0.0) {
      const double2 c = *p;
      o.x = __dadd_rn(o.x, __dmul_rn(beta, c.x));
      o.y = __dadd_rn(o.y, __dmul_rn(beta, c.y));
    }
    *p = o;
  }
}

inline bool fast_ok(int bs, int64_t ld, const void* a, const void* b) {
  return (bs == 22 || bs == 64) && ld % 2 == 0 && ((uintptr_t)a & 15) == 0 && ((uintptr_t)b & 15) == 0;
}

inline unsigned grid_pairs(int64_t pairs) {
  int64_t g = (pairs + 255) / 256;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)num_sms() * 32));
}

}  // namespace

void launch_fill(double* arena, int64_t mloc, int64_t nloc, int bs, int pr, int pc, int r, int c, uint64_t seed,
                 uint32_t mat_id, int kind, cudaStream_t st) {
  int64_t total = mloc * nloc * (int64_t)bs * bs;
  if (total == 0) return;
  // key = mix64(seed + golden * (mat_id + 1)), computed on the host with the same definition
  auto hmix = [](uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
  };
  uint64_t key = hmix(seed + 0x9E3779B97F4A7C15ull * ((uint64_t)mat_id + 1ull));
  fill_kernel<<<grid_for(total), kThreads, 0, st>>>(arena, total, nloc, bs, pr, pc, r, c, key, kind);
}

void launch_densify_cols(const double* arena, int64_t mloc, int64_t nloc, int bs, int64_t kcol0, int64_t kstride,
                         int64_t nk, double* dense, int64_t ld, int layout, cudaStream_t st) {
  if (mloc == 0 || nk == 0) return;
  if (layout == 1 && fast_ok(bs, ld, arena, dense) && mloc * nk < (1ll << 31)) {
    if (bs == 22) {
      constexpr int G = 8;  // 176-double rows, 8 x 22 x 23 x 8 B = 32 KB of smem
      densify_a_fast<22, G><<<(unsigned)(mloc * ((nk + G - 1) / G)), 256, 0, st>>>(arena, nloc, kcol0, kstride, nk,
                                                                                 dense, ld);
    } else {
      constexpr int G = 1;  // 64 x 65 x 8 B = 33 KB
      densify_a_fast<64, G><<<(unsigned)(mloc * nk), 256, 0, st>>>(arena, nloc, kcol0, kstride, nk, dense, ld);
    }
    return;
  }
  const int64_t bb = (int64_t)bs * bs;
  constexpr int G = 8;
  int g = (int)std::max<int64_t>(1, std::min<int64_t>(G, 6144 / bb));
  size_t smem = (size_t)g * bs * (bs + 1) * sizeof(double);
  // template on the maximum group; the kernel uses min(G, remaining) at run time via ngroups
  // computed from G, so instantiate the actual group size.
  int64_t grid;
  switch (g) {
#define DBM_DC(GG)                                                                                          \
  case GG:                                                                                                  \
    grid = mloc * ((nk + GG - 1) / GG);                                                                     \
    if (smem > 48 * 1024) cudaFuncSetAttribute(densify_cols_kernel<GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    densify_cols_kernel<GG><<<(unsigned)grid, kThreads, layout == 1 ? smem : 0, st>>>(arena, nloc, bs, kcol0, \
                                                                                       kstride, nk, dense, ld, layout); \
    break;
    DBM_DC(1) DBM_DC(2) DBM_DC(3) DBM_DC(4) DBM_DC(5) DBM_DC(6) DBM_DC(7) DBM_DC(8)
#undef DBM_DC
    default:
      break;
  }
}

void launch_densify_rows(const double* arena, int64_t nloc, int bs, int64_t krow0, int64_t kstride, int64_t nk,
                         double* dense, int64_t ld, int layout, cudaStream_t st) {
  int64_t total = nk * bs * nloc * (int64_t)bs;
  if (total == 0) return;
  if (layout == 0 && fast_ok(bs, ld, arena, dense) && nk * nloc < (1ll << 31)) {
    const int nblk = (int)(nk * nloc);
    static const char* env = getenv("DBM_DENSIFY_B_ORDER");  // measurement override: "q" / "lj"
    const int ljm = env ? (env[0] == 'l') : (nloc <= 128 && nk >= 4 * nloc);
    if (bs == 22)
      densify_b_fast<22><<<grid_pairs((int64_t)nblk * 242), 256, 0, st>>>(arena, (int)nloc, krow0, kstride, nblk,
                                                                         dense, ld, ljm);
    else
      densify_b_fast<64><<<grid_pairs((int64_t)nblk * 2048), 256, 0, st>>>(arena, (int)nloc, krow0, kstride, nblk,
                                                                          dense, ld, ljm);
    return;
  }
  densify_rows_kernel<<<grid_for(total), kThreads, 0, st>>>(arena, nloc, bs, krow0, kstride, nk, dense, ld, layout);
}

void launch_undensify(const double* dense, int64_t ld, int nsplit, int64_t split_stride, int64_t mloc, int64_t nloc,
                      int bs, double alpha, double beta, double* arena, cudaStream_t st) {
  int64_t total = mloc * nloc * (int64_t)bs * bs;
  if (total == 0) return;
  if (fast_ok(bs, ld, dense, arena) && (nsplit <= 1 || split_stride % 2 == 0) && mloc * nloc < (1ll << 31)) {
    const int nblk = (int)(mloc * nloc);
    const int ns = nsplit < 1 ? 1 : nsplit;
    if (bs == 22)
      undensify_fast<22><<<grid_pairs((int64_t)nblk * 242), 256, 0, st>>>(dense, ld, ns, split_stride, (int)nloc,
                                                                          nblk, alpha, beta, arena);
    else
      undensify_fast<64><<<grid_pairs((int64_t)nblk * 2048), 256, 0, st>>>(dense, ld, ns, split_stride, (int)nloc,
                                                                           nblk, alpha, beta, arena);
    return;
  }
  undensify_kernel<<<grid_for(total), kThreads, 0, st>>>(dense, ld, nsplit < 1 ? 1 : nsplit, split_stride, nloc, bs,
                                                         total, alpha, beta, arena);
}

void launch_pack_rows(const double* arena, int64_t ncols, int bs, int64_t row0, int64_t rstride, int64_t nrows,
                      double* out, cudaStream_t st) {
  int64_t total = nrows * ncols * (int64_t)bs * bs;
  if (total == 0) return;
  const int64_t row = ncols * (int64_t)bs * bs;
  if (row % 2 == 0 && ((uintptr_t)arena & 15) == 0 && ((uintptr_t)out & 15) == 0) {
    const int64_t pairs = row / 2;
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((pairs + 255) / 256, 64));
    const unsigned gy = (unsigned)std::min<int64_t>(nrows, 65535);
    pack_rows_fast<<<dim3(gx, gy), 256, 0, st>>>((const double2*)arena, pairs, row0, rstride, nrows, (double2*)out);
    return;
  }
  pack_blocks_kernel<<<grid_for(total), kThreads, 0, st>>>(arena, nrows, ncols, 0, row0, rstride, bs, 1, ncols, out);
}

void launch_pack_cols(const double* arena, int64_t mloc, int64_t nloc, int bs, int64_t col0, int64_t cstride,
                      int64_t ncols, double* out, cudaStream_t st, int64_t out_pitch) {
  int64_t total = ncols * mloc * (int64_t)bs * bs;
  if (total == 0) return;
  const int64_t bb = (int64_t)bs * bs;
  if (bb % 2 == 0 && ((uintptr_t)arena & 15) == 0 && ((uintptr_t)out & 15) == 0) {
    const unsigned gy = (unsigned)std::min<int64_t>(mloc, 65535);
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ncols, (4 * num_sms() * 8 + gy - 1) / gy));
    pack_cols_fast<<<dim3(gx, gy), 256, 0, st>>>((const double2*)arena, bb / 2, nloc, col0, cstride, ncols, mloc,
                                                 out_pitch > 0 ? out_pitch : ncols, (double2*)out);
    return;
  }
  pack_blocks_kernel<<<grid_for(total), kThreads, 0, st>>>(arena, ncols, nloc, out_pitch, col0, cstride, bs, 0, mloc,
                                                           out);
}

}  // namespace dbm

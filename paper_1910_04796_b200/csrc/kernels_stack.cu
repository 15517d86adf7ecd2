// Blocked path (§II): Traversal -> Generation -> batched small-block GEMM.
//
// traversal_kernel: C-block order by recursive bisection (reading R6), one thread per run,
//   descending the bisection tree (integer; bit-exact vs the oracle).
// stackgen_kernel: the Generation phase on the GPU: (a_slot, b_slot, c_slot) int32 triplets for a
//   range of runs (12 B written per entry; HBM/L2 bound).  stack_ptr_kernel writes the <= cap
//   stack boundaries (greedy whole-run packing, closed form for uniform runs).
// smm_generic_kernel: block sizes other than 22 / 64 (the DMMA group kernel is kernels_smm.cu).
#include <algorithm>
#include <cstdlib>

#include "dbm_internal.h"

namespace dbm {

namespace {

__global__ void traversal_kernel(int64_t mloc, int64_t nloc, int32_t* __restrict__ li_out,
                                 int32_t* __restrict__ lj_out) {
  const int64_t total = mloc * nloc;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t r0 = 0, r1 = mloc, c0 = 0, c1 = nloc, rem = q;
    while (r1 - r0 > 1 || c1 - c0 > 1) {
      const int64_t nr = r1 - r0, nc = c1 - c0;
      if (nr >= nc) {  // split rows (ties go to rows), lower half first
        const int64_t mid = r0 + nr / 2, first = (mid - r0) * nc;
        if (rem < first) {
          r1 = mid;
        } else {
          rem -= first;
          r0 = mid;
        }
      } else {
        const int64_t mid = c0 + nc / 2, first = nr * (mid - c0);
        if (rem < first) {
          c1 = mid;
        } else {
          rem -= first;
          c0 = mid;
        }
      }
    }
    li_out[q] = (int32_t)r0;
    lj_out[q] = (int32_t)c0;
  }
}

__global__ void stackgen_kernel(const int32_t* __restrict__ li, const int32_t* __restrict__ lj, int64_t q0,
                                int64_t nent, int64_t kb, int64_t nloc, int64_t a_ld, int64_t b_ld,
                                int32_t* __restrict__ trip) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nent; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t qq = e / kb, kk = e - qq * kb, q = q0 + qq;
    const int64_t i = li[q], j = lj[q];
    trip[3 * e + 0] = (int32_t)(i * a_ld + kk);
    trip[3 * e + 1] = (int32_t)(kk * b_ld + j);
    trip[3 * e + 2] = (int32_t)(i * nloc + j);
  }
}

__global__ void stack_ptr_kernel(int64_t nruns, int64_t kb, int64_t cap, int64_t nstacks, int64_t* __restrict__ ptr) {
  const int64_t total = nruns * kb;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= nstacks;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t v;
    if (kb <= cap) {
      const int64_t per = cap / kb;  // whole runs per stack
      v = t * per * kb;
    } else {
      const int64_t ns = (kb + cap - 1) / cap;  // stacks per run
      const int64_t q = t / ns, i = t - q * ns;
      v = q * kb + (i * cap < kb ? i * cap : kb);
    }
    ptr[t] = v < total ? v : total;
  }
}

// Generic block size (any bs <= 64): same algorithm, dynamic shared memory.
__global__ void __launch_bounds__(256) smm_generic_kernel(int bs, const int32_t* __restrict__ trip, int64_t nruns,
                                                          int64_t kb, const double* __restrict__ A,
                                                          const double* __restrict__ B, double* __restrict__ C,
                                                          double alpha, double beta_first) {
  extern __shared__ double sm[];
  const int BB = bs * bs;
  double* sA = sm;
  double* sB = sm + BB;
  for (int64_t run = blockIdx.x; run < nruns; run += gridDim.x) {
    const int32_t* t = trip + 3 * run * kb;
    double* c = C + (int64_t)t[2] * BB;
    for (int idx0 = 0; idx0 < BB; idx0 += 256) {
      const int idx = idx0 + threadIdx.x;
      double acc = 0.0;
      for (int64_t e = 0; e < kb; ++e) {
        const double* a = A + (int64_t)t[3 * e] * BB;
        const double* b = B + (int64_t)t[3 * e + 1] * BB;
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
      if (idx < BB) c[idx] = (beta_first == 0.0) ? alpha * acc : beta_first * c[idx] + alpha * acc;
    }
  }
}

// Small blocks (bs <= 8, bs^2 <= 64): one warp per run, lane l owns C elements l and l + 32; per entry the
// warp loads the A and B blocks into registers (coalesced, two entries in flight) and forms the
// products with shuffles.  Memory-bound like the paper's bs-4 case, but no CTA-wide barriers.
__global__ void __launch_bounds__(256) smm_small_kernel(int bs, const int32_t* __restrict__ trip, int64_t nruns,
                                                        int64_t kb, const double* __restrict__ A,
                                                        const double* __restrict__ B, double* __restrict__ C,
                                                        double alpha, double beta_first) {
  const int lane = threadIdx.x & 31, bb = bs * bs;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int x0 = lane % bs, y0 = lane / bs, x1 = (lane + 32) % bs, y1 = (lane + 32) / bs;
  for (int64_t run = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); run < nruns; run += warps) {
    const int32_t* t = trip + 3 * run * kb;
    double acc0 = 0.0, acc1 = 0.0;
    double a0 = 0, a1 = 0, b0 = 0, b1 = 0;
    auto fetch = [&](int64_t e, double& va0, double& va1, double& vb0, double& vb1) {
      const double* a = A + (int64_t)t[3 * e] * bb;
      const double* b = B + (int64_t)t[3 * e + 1] * bb;
      va0 = lane < bb ? a[lane] : 0.0;
      va1 = lane + 32 < bb ? a[lane + 32] : 0.0;
      vb0 = lane < bb ? b[lane] : 0.0;
      vb1 = lane + 32 < bb ? b[lane + 32] : 0.0;
    };
    if (kb > 0) fetch(0, a0, a1, b0, b1);
    for (int64_t e = 0; e < kb; ++e) {
      double na0 = 0, na1 = 0, nb0 = 0, nb1 = 0;
      if (e + 1 < kb) fetch(e + 1, na0, na1, nb0, nb1);
      for (int z = 0; z < bs; ++z) {
        // A(x, z) is element x + z*bs, B(z, y) is z + y*bs (column-major blocks)
        const int ia0 = x0 + z * bs, ib0 = z + y0 * bs, ia1 = x1 + z * bs, ib1 = z + y1 * bs;
        // every lane sends the same register; the reader picks the half its element lives in
        double av0 = __shfl_sync(0xffffffffu, a0, ia0 & 31), bv0 = __shfl_sync(0xffffffffu, b0, ib0 & 31);
        double av1 = __shfl_sync(0xffffffffu, a0, ia1 & 31), bv1 = __shfl_sync(0xffffffffu, b0, ib1 & 31);
        if (bb > 32) {  // warp-uniform
          const double ah0 = __shfl_sync(0xffffffffu, a1, ia0 & 31), bh0 = __shfl_sync(0xffffffffu, b1, ib0 & 31);
          const double ah1 = __shfl_sync(0xffffffffu, a1, ia1 & 31), bh1 = __shfl_sync(0xffffffffu, b1, ib1 & 31);
          av0 = ia0 < 32 ? av0 : ah0;
          bv0 = ib0 < 32 ? bv0 : bh0;
          av1 = ia1 < 32 ? av1 : ah1;
          bv1 = ib1 < 32 ? bv1 : bh1;
        }
        acc0 = fma(av0, bv0, acc0);
        acc1 = fma(av1, bv1, acc1);
      }
      a0 = na0; a1 = na1; b0 = nb0; b1 = nb1;
    }
    double* c = C + (int64_t)t[2] * bb;
    if (lane < bb) c[lane] = (beta_first == 0.0) ? alpha * acc0 : beta_first * c[lane] + alpha * acc0;
    if (lane + 32 < bb) c[lane + 32] = (beta_first == 0.0) ? alpha * acc1 : beta_first * c[lane + 32] + alpha * acc1;
  }
}

// measurement override: DBM_SMM_NO_RUN=1 sends the small sizes back to the FMA kernels (tools/smm_small_ab)
bool smm_run_disabled() {
  static const int v = [] {
    const char* e = getenv("DBM_SMM_NO_RUN");
    return (e && *e && *e != '0') ? 1 : 0;
  }();
  return v != 0;
}

inline unsigned grid_of(int64_t n, int per = 256) {
  int64_t g = (n + per - 1) / per;
  g = std::min<int64_t>(g, (int64_t)num_sms() * 32);
  return (unsigned)std::max<int64_t>(g, 1);
}

}  // namespace

void launch_traversal(int64_t mloc, int64_t nloc, int32_t* li_out, int32_t* lj_out, cudaStream_t st) {
  if (mloc * nloc == 0) return;
  traversal_kernel<<<grid_of(mloc * nloc), 256, 0, st>>>(mloc, nloc, li_out, lj_out);
}

void launch_stackgen(const int32_t* li, const int32_t* lj, int64_t q0, int64_t q1, int64_t kb, int64_t nloc,
                     int64_t a_ld, int64_t b_ld, int32_t* trip, cudaStream_t st) {
  const int64_t nent = (q1 - q0) * kb;
  if (nent <= 0) return;
  stackgen_kernel<<<grid_of(nent), 256, 0, st>>>(li, lj, q0, nent, kb, nloc, a_ld, b_ld, trip);
}

void launch_stack_ptr(int64_t nruns, int64_t kb, int64_t cap, int64_t nstacks, int64_t* ptr, cudaStream_t st) {
  stack_ptr_kernel<<<grid_of(nstacks + 1), 256, 0, st>>>(nruns, kb, cap, nstacks, ptr);
}

cudaError_t launch_smm(int bs, const int32_t* trip, int64_t nruns, int64_t kb, const double* A, const double* B,
                       double* C, double alpha, double beta_first, int nsplit, double* partial, cudaStream_t st,
                       int* launches, int64_t a_blocks, int64_t b_blocks, bool squares) {
  if (nruns <= 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<int64_t>(nruns, (int64_t)num_sms() * 8);
  if (squares && smmq_side(bs) > 0) {  // R x R run squares of a padded small size (the host checked the shape)
    cudaError_t e = launch_smmq(bs, trip, nruns, kb, A, B, C, alpha, beta_first, st);
    if (e != cudaSuccess) return e;
  } else if (smm_has_tensor_path(bs)) {
    cudaError_t e =
        launch_smm_tc(bs, trip, nruns, kb, A, B, C, alpha, beta_first, nsplit, partial, st, a_blocks, b_blocks,
                      squares);
    if (e != cudaSuccess) return e;
  } else if (smm_has_run_path(bs) && !smm_run_disabled()) {
    cudaError_t e = launch_smm_run(bs, trip, nullptr, nruns, kb, A, B, C, alpha, beta_first, st);
    if (e != cudaSuccess) return e;
  } else if (bs <= 8) {
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nruns + 7) / 8, (int64_t)num_sms() * 16));
    smm_small_kernel<<<g, 256, 0, st>>>(bs, trip, nruns, kb, A, B, C, alpha, beta_first);
  } else {
    size_t smem = 2 * (size_t)bs * bs * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(smm_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smm_generic_kernel<<<grid, 256, smem, st>>>(bs, trip, nruns, kb, A, B, C, alpha, beta_first);
  }
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace dbm

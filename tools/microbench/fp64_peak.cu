// FP64 roofline denominators on B200: DFMA chain peak,
// DMMA (mma.sync f64) peak for each legal shape, both mixed, and an L2 read
// bandwidth probe. Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int ITERS = 4096;

__global__ void dfma_peak(double* out, double s) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], s, 1e-12);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
  if (r == 12345.678) out[0] = r;
}

__global__ void dmma_m8n8k4_peak(double* out, double s) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a = threadIdx.x * 1e-9 + s, b = s;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1];
  if (r == 12345.678) out[0] = r;
}

__global__ void dmma_m16n8k4_peak(double* out, double s) {
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a0 = threadIdx.x * 1e-9 + s, a1 = s, b = s;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 12345.678) out[0] = r;
}

__global__ void dmma_m16n8k16_peak(double* out, double s) {
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + s + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = s - i;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 12345.678) out[0] = r;
}

__global__ void l2_read(const double2* __restrict__ p, size_t n, int reps, double* out) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(p + i);
      acc += v.x + v.y;
    }
  if (acc == 12345.678) out[0] = acc;
}

template <class F>
float timeit(F f, int reps = 5) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  size_t fre, tot; CK(cudaMemGetInfo(&fre, &tot));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f, \"mem_free_gb\": %.2f, \"mem_total_gb\": %.2f, \"l2_mb\": %.1f, \"smem_optin_kb\": %zu}\n",
         prop.name, sms, clk_khz / 1e3, fre / 1e9, tot / 1e9, prop.l2CacheSize / 1048576.0, prop.sharedMemPerBlockOptin / 1024);
  double* out; CK(cudaMalloc(&out, 64));
  for (int warps = 4; warps <= 32; warps *= 2) {
    for (int ctas_per_sm = 1; ctas_per_sm <= 2; ++ctas_per_sm) {
      int grid = sms * ctas_per_sm * 4, thr = warps * 32;
      float ms = timeit([&] { dfma_peak<<<grid, thr>>>(out, 0.999999); });
      double fl = 2.0 * 16 * ITERS * (double)grid * thr;
      printf("{\"kernel\": \"dfma\", \"warps\": %d, \"grid\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", warps, grid, ms, fl / ms / 1e9);
      ms = timeit([&] { dmma_m8n8k4_peak<<<grid, thr>>>(out, 0.999999); });
      fl = 2.0 * 8 * 8 * 4 * 8 * ITERS * (double)grid * warps;
      printf("{\"kernel\": \"dmma_m8n8k4\", \"warps\": %d, \"grid\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", warps, grid, ms, fl / ms / 1e9);
      ms = timeit([&] { dmma_m16n8k4_peak<<<grid, thr>>>(out, 0.999999); });
      fl = 2.0 * 16 * 8 * 4 * 4 * ITERS * (double)grid * warps;
      printf("{\"kernel\": \"dmma_m16n8k4\", \"warps\": %d, \"grid\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", warps, grid, ms, fl / ms / 1e9);
      ms = timeit([&] { dmma_m16n8k16_peak<<<grid, thr>>>(out, 0.999999); });
      fl = 2.0 * 16 * 8 * 16 * 4 * (ITERS / 4) * (double)grid * warps;
      printf("{\"kernel\": \"dmma_m16n8k16\", \"warps\": %d, \"grid\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", warps, grid, ms, fl / ms / 1e9);
    }
  }
  // L2-resident read bandwidth: 64 MB working set re-read.
  size_t bytes = 64ull << 20; double2* p; CK(cudaMalloc(&p, bytes)); CK(cudaMemset(p, 0, bytes));
  size_t n = bytes / 16; int reps = 20;
  float ms = timeit([&] { l2_read<<<sms * 8, 512>>>(p, n, reps, out); });
  printf("{\"kernel\": \"l2_read_64MB\", \"ms\": %.3f, \"gbs\": %.1f}\n", ms, (double)bytes * reps / ms / 1e6);
  size_t bigb = 8ull << 30; double2* q; CK(cudaMalloc(&q, bigb)); CK(cudaMemset(q, 0, bigb));
  ms = timeit([&] { l2_read<<<sms * 8, 512>>>(q, bigb / 16, 1, out); });
  printf("{\"kernel\": \"hbm_read_8GB\", \"ms\": %.3f, \"gbs\": %.1f}\n", ms, (double)bigb / ms / 1e6);
  return 0;
}

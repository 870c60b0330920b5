// Microbenchmark: the tile-matmul fold's inner loop (fold_gemm_tma_kernel's
// consumer side) with its operands already in shared memory -- no TMA, no
// mbarrier waits -- to find the FP64-pipe ceiling of each register-block /
// thread-mapping choice.  A unit is PB x BC groups x SL slots; a thread owns a
// RB x CB sub-block of groups for one slot; per fold step it loads RB + CB
// doubles from shared memory and issues RB*CB DMUL + RB*CB DADD (separately
// rounded, no FMA, as the real kernel).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o gemm_loop gemm_loop.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double f64add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double f64mul(double a, double b) { return __dmul_rn(a, b); }

// BATCH: rows of products formed before their additions.
template <int PB, int BC, int SL, int RB, int CB, int BATCH, int STEPS>
__device__ __forceinline__ void body(const double* tsm, double* out, int iters) {
  constexpr int kA = STEPS * PB * SL;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int subs_per_warp = 32 / SL;
  const int sub = warp * subs_per_warp + lane / SL, slot = lane % SL;
  const int r0 = (sub / (BC / CB)) * RB, c0 = (sub % (BC / CB)) * CB;
  double acc[RB][CB];
#pragma unroll
  for (int i = 0; i < RB; ++i)
#pragma unroll
    for (int k = 0; k < CB; ++k) acc[i][k] = -0.0;
  for (int it = 0; it < iters; ++it) {
    asm volatile("" ::: "memory");  // operands re-read every stage, as after an mbarrier wait
    const double* sA = tsm + r0 * SL + slot;
    const double* sB = tsm + kA + c0 * SL + slot;
#pragma unroll
    for (int h = 0; h < STEPS; ++h) {
      double a[RB], b[CB];
#pragma unroll
      for (int i = 0; i < RB; ++i) a[i] = sA[h * PB * SL + i * SL];
#pragma unroll
      for (int k = 0; k < CB; ++k) b[k] = sB[h * BC * SL + k * SL];
#pragma unroll
      for (int i = 0; i < RB; i += BATCH) {
        double pr[BATCH][CB];
#pragma unroll
        for (int r = 0; r < BATCH; ++r)
#pragma unroll
          for (int k = 0; k < CB; ++k) pr[r][k] = f64mul(a[i + r], b[k]);
#pragma unroll
        for (int r = 0; r < BATCH; ++r)
#pragma unroll
          for (int k = 0; k < CB; ++k) acc[i + r][k] = f64add(acc[i + r][k], pr[r][k]);
      }
    }
  }
  double sum = 0;
#pragma unroll
  for (int i = 0; i < RB; ++i)
#pragma unroll
    for (int k = 0; k < CB; ++k) sum += acc[i][k];
  if (sum == 1234.5) out[threadIdx.x] = sum;
}

template <int PB, int BC, int SL, int RB, int CB, int BATCH, int MAXREG>
__global__ void __maxnreg__(MAXREG) k(double* out, int iters) {
  constexpr int STEPS = 4;
  extern __shared__ double tsm[];
  constexpr int n = STEPS * (PB + BC) * SL;
  for (int i = threadIdx.x; i < n; i += blockDim.x) tsm[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  body<PB, BC, SL, RB, CB, BATCH, STEPS>(tsm, out, iters);
}

template <int PB, int BC, int SL, int RB, int CB, int BATCH, int MAXREG>
void run(const char* name, int ctas_per_sm, int sms, double* out) {
  constexpr int threads = (PB / RB) * (BC / CB) * SL;
  const size_t smem = 4 * (PB + BC) * SL * sizeof(double);
  auto kern = k<PB, BC, SL, RB, CB, BATCH, MAXREG>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  const int per_sm = ctas_per_sm < occ ? ctas_per_sm : occ;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  const int iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    kern<<<sms * per_sm, threads, smem>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * sms * per_sm * double(threads) * iters * 4 * RB * CB;
  printf("%-34s thr=%4d ctas/SM=%d warps/SM=%2d regs=%3d  %6.2f T fp64 ops/s  (%.0f%% of 18.34)\n", name,
         threads, per_sm, per_sm * threads / 32, fa.numRegs, ops / best / 1e9, ops / best / 1e9 / 18.34 * 100);
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // the shipped configuration: 16x16 groups x 16 slots, 8x4 per thread, 2 rows batched
  run<16, 16, 16, 8, 4, 2, 128>("16x16x16 8x4 batch2 (shipped)", 4, sms, out);
  run<16, 16, 16, 8, 4, 1, 128>("16x16x16 8x4 batch1", 4, sms, out);
  run<16, 16, 16, 8, 4, 4, 168>("16x16x16 8x4 batch4 r168", 3, sms, out);
  run<16, 16, 16, 8, 4, 8, 168>("16x16x16 8x4 batch8 r168", 3, sms, out);
  run<16, 16, 16, 8, 4, 2, 128>("16x16x16 8x4 batch2 2cta", 2, sms, out);
  run<16, 16, 16, 8, 4, 2, 128>("16x16x16 8x4 batch2 3cta", 3, sms, out);
  run<16, 16, 16, 4, 4, 2, 96>("16x16x16 4x4 batch2 r96", 5, sms, out);
  run<16, 16, 16, 4, 4, 4, 96>("16x16x16 4x4 batch4 r96", 5, sms, out);
  run<16, 16, 8, 8, 4, 2, 128>("16x16x8 8x4 batch2", 8, sms, out);
  run<16, 16, 16, 8, 8, 2, 232>("16x16x16 8x8 batch2 r232", 4, sms, out);
  run<16, 16, 16, 8, 8, 4, 232>("16x16x16 8x8 batch4 r232", 4, sms, out);
  run<16, 32, 16, 8, 8, 2, 232>("16x32x16 8x8 batch2 r232", 4, sms, out);
  run<32, 16, 16, 8, 4, 2, 128>("32x16x16 8x4 batch2", 2, sms, out);
  run<16, 16, 32, 8, 4, 2, 128>("16x16x32 8x4 batch2", 2, sms, out);
  run<16, 16, 4, 8, 4, 2, 128>("16x16x4 8x4 batch2", 16, sms, out);
  return 0;
}

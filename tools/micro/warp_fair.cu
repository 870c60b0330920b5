// Microbenchmark: how the SM's warp schedulers share the FP64 pipe between warps doing
// identical work -- 3 CTAs x 4 warps per SM (the shipped GEMM fold's residency) against
// 1 CTA x 12 warps.  Every warp runs the fold's inner loop (8 + 4 shared-memory loads,
// 32 DMUL + 32 DADD per step) a fixed number of times and records when it finishes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o warp_fair warp_fair.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <algorithm>
#include <vector>

template <int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) k(double* out, unsigned long long* rec, int iters) {
  extern __shared__ double tsm[];
  constexpr int SL = 16, PB = 16, BC = 16, STEPS = 4;
  constexpr int n = STEPS * (PB + BC) * SL;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = threadIdx.x; i < n; i += blockDim.x) tsm[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  const int warp = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31;
  const int sub = warp * 2 + lane / SL, slot = lane % SL;
  const int r0 = (sub / 4) * 8, c0 = (sub % 4) * 4;
  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = -0.0;
  for (int it = 0; it < iters; ++it) {
    asm volatile("" ::: "memory");
    const double* sA = tsm + r0 * SL + slot;
    const double* sB = tsm + STEPS * PB * SL + c0 * SL + slot;
#pragma unroll
    for (int h = 0; h < STEPS; ++h) {
      double a[8], b[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = sA[h * PB * SL + i * SL];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[h * BC * SL + j * SL];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a[i], b[j]));
    }
  }
  double sum = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) sum += acc[i][j];
  if (sum == 1234.5) out[threadIdx.x] = sum;
  if (lane == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int w = blockIdx.x * WARPS + (threadIdx.x >> 5);
    rec[2 * w] = t1 - t0;
    rec[2 * w + 1] = smid;
  }
}

template <int WARPS, int MINB>
void run(const char* name, int sms) {
  const size_t smem = 4 * 32 * 16 * 8;
  auto kern = k<WARPS, MINB>;
  const int grid = sms * MINB, iters = 1024, nw = grid * WARPS;
  double* out;
  unsigned long long* rec;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&rec, nw * 16);
  for (int rep = 0; rep < 2; ++rep) kern<<<grid, WARPS * 32, smem>>>(out, rec, iters);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(nw * 2);
  cudaMemcpy(h.data(), rec, nw * 16, cudaMemcpyDeviceToHost);
  // per SM: sort the warps' finish times; report the mean of the k-th finisher over SMs
  std::vector<std::vector<double>> per(sms + 64);
  for (int w = 0; w < nw; ++w) per[h[2 * w + 1]].push_back(h[2 * w] * 1e-3);
  const int per_sm = WARPS * MINB;
  std::vector<double> mean(per_sm, 0);
  int cnt = 0;
  for (auto& v : per) {
    if ((int)v.size() != per_sm) continue;
    std::sort(v.begin(), v.end());
    for (int i = 0; i < per_sm; ++i) mean[i] += v[i];
    ++cnt;
  }
  printf("%-24s finish time of the k-th warp of an SM (us, mean over %d SMs):", name, cnt);
  for (int i = 0; i < per_sm; ++i) printf(" %.1f", mean[i] / cnt);
  const double ops = 2.0 * 32 * 4 * 32 * iters * per_sm;  // per SM
  printf("\n   ideal at 63 FP64 ops/clk/SM @1.965 GHz: %.1f us\n", ops / (63.06 * 1.965e3));
  cudaFree(out);
  cudaFree(rec);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, 3>("3 CTAs x 4 warps", sms);
  run<12, 1>("1 CTA x 12 warps", sms);
  run<8, 1>("1 CTA x 8 warps", sms);
  run<4, 1>("1 CTA x 4 warps", sms);
  run<16, 1>("1 CTA x 16 warps", sms);
  return 0;
}

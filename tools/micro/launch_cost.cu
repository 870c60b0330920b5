// Host cost of cudaLaunchKernel vs kernel-parameter size (config 1's fused op
// passes a ~3.3 KB GroupParams by value).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_cost launch_cost.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
template <int N>
struct P { long long v[N]; };
template <int N>
__global__ void k(const __grid_constant__ P<N> p, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.v[N - 1] == 12345) out[0] = 1;
}
template <int N>
void run(double* out, cudaStream_t st) {
  P<N> p{};
  for (int i = 0; i < 100; ++i) k<N><<<7, 512, 0, st>>>(p, out);
  cudaStreamSynchronize(st);
  const int n = 20000;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) k<N><<<7, 512, 0, st>>>(p, out);
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(st);
  auto t2 = std::chrono::steady_clock::now();
  printf("params %6zu B: enqueue %.2f us/launch, with drain %.2f us\n", sizeof(P<N>),
         std::chrono::duration<double>(t1 - t0).count() / n * 1e6,
         std::chrono::duration<double>(t2 - t0).count() / n * 1e6);
}
int main() {
  double* out;
  cudaMalloc(&out, 64);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  run<8>(out, st);
  run<64>(out, st);
  run<128>(out, st);
  run<256>(out, st);
  run<420>(out, st);
  run<1000>(out, st);
  return 0;
}

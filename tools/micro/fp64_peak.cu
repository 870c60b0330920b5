// Microbenchmark: sustained DMUL / DADD / DFMA issue rate on this GPU
// (register-only, independent chains).  Used to set the FP64 roofline of the
// tile-matmul fold (separate DMUL + DADD, no contraction, for bit parity).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>  // 0 = dmul+dadd pairs, 1 = dfma, 2 = dadd only
__global__ void k(double* out, int iters, double x) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = x + threadIdx.x + i;
  const double m = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (OP == 0) a[i] = __dadd_rn(__dmul_rn(a[i], m), c);
      if (OP == 1) a[i] = __fma_rn(a[i], m, c);
      if (OP == 2) a[i] = __dadd_rn(a[i], c);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int op = 0; op < 3; ++op)
    for (int warps = 4; warps <= 32; warps *= 2) {
      const int threads = warps * 32;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (op == 0) k<0><<<sms, threads>>>(out, iters, 1.0);
        if (op == 1) k<1><<<sms, threads>>>(out, iters, 1.0);
        if (op == 2) k<2><<<sms, threads>>>(out, iters, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double instr = double(sms) * threads * iters * 16 * (op == 0 ? 2 : 1);
        if (rep) printf("op=%s warps/SM=%d  %.2f T fp64 thread-instr/s\n",
                        op == 0 ? "dmul+dadd" : op == 1 ? "dfma" : "dadd", warps, instr / ms / 1e9);
      }
    }
  return 0;
}

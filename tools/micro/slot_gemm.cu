// Microbenchmark: the tile-matmul fold (per-slot batched outer-product fold,
// config 3 stage 1 shapes) fed by a TMA ring, to find where the FP64 pipe
// loses issue cycles against the smem-only loop (tools/micro/gemm_loop.cu).
//
//   out[i][j][h] = fold_k ( A[k][i][h] * B[k][j][h] ),  k = 0..K-1 in order,
//   each product and sum separately rounded (no FMA), starting from -0.0.
//
// A unit = PI x PJ groups x SL slots; a consumer thread owns RI x RJ groups of
// one slot.  MODE 0: real ring; 1: consumers never wait for data (the ring
// still streams); 2: the producer issues no TMA (barriers complete at once).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -o slot_gemm slot_gemm.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>
#include <algorithm>
#include <cstdlib>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);      \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
          su32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}

#ifndef S_SLOTS
#define S_SLOTS 8192
#endif
#ifndef K_STEPS
#define K_STEPS 48
#endif
constexpr int NI = 32, NJ = 16, K = K_STEPS, S = S_SLOTS;
// G_GROUPS > 1: one CTA holds G_GROUPS independent consumer groups, each with its own ring,
// producer warp and unit stream (the warps of one CTA share the schedulers fairly; CTAs of
// one SM are served oldest first, tools/micro/warp_fair.cu)
#ifndef G_GROUPS
#define G_GROUPS 1
#endif
constexpr int G = G_GROUPS;

template <int PI, int PJ, int SL, int RI, int RJ, int KS, int NS, int MODE, int MINB, int SCHED>
__global__ void __launch_bounds__(((PI / RI) * (PJ / RJ) * SL + 32) * G, MINB)
    sg_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, double* out,
              int reps, unsigned* q, unsigned long long* rec, unsigned long long* crec) {
  constexpr int kC = (PI / RI) * (PJ / RJ) * SL;  // consumer threads per group
  constexpr int kCW = kC / 32;
  const bool is_prod = threadIdx.x >= G * kC;
  const int grp = is_prod ? (threadIdx.x - G * kC) / 32 : threadIdx.x / kC;
  const int tg = is_prod ? 0 : threadIdx.x % kC;  // consumer thread within its group
  const int vb = blockIdx.x * G + grp, vgrid = gridDim.x * G;
  if (crec && !is_prod && tg == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(crec[3 * vb]));
  constexpr int kA = KS * PI * SL, kB = KS * PJ * SL, kSt = kA + kB;
  constexpr int nbi = NI / PI, nbj = NJ / PJ, nch = S / SL;
  constexpr int units1 = nbi * nbj * nch;
  constexpr int nst = K / KS;
  extern __shared__ __align__(1024) double sm_all[];
  constexpr int kGS = NS * kSt + (3 * NS + 15) / 16 * 16;  // doubles per group (ring + barriers + stage units)
  double* sm = sm_all + grp * kGS;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * kSt);
  uint64_t* empty = full + NS;
  int* stu = reinterpret_cast<int*>(empty + NS);  // unit of each stage (-1: done)
  const int units = units1 * reps;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (!is_prod && tg == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (is_prod) {
    if (lane != 0) return;
    int st = 0;
    uint32_t ph = 0;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int nsm = gridDim.x / MINB;  // SMs
    const int lo = (int)((long long)units * smid / nsm), hi = (int)((long long)units * (smid + 1) / nsm);
    // SCHED: 0 static round-robin, 1 per-SM queue, 2 one global queue (the library's);
    // +10*D: pace the CTAs of an SM (a producer issues a stage only while its CTA is
    // at most D stages ahead of the slowest sibling still running)
    constexpr int kSched = SCHED % 10, kPace = SCHED / 10;
    auto next = [&](int prev) -> int {
      if (kSched == 0) return prev < 0 ? vb : prev + vgrid;
      if (kSched == 2) return prev < 0 ? vb : (int)(vgrid + atomicAdd(&q[1023], 1u));
      const int v = lo + (int)atomicAdd(&q[smid], 1u);
      return v < hi ? v : units;
    };
    volatile unsigned* pg = q + 384 + smid * 4;
    unsigned myslot = 0, total = 0;
    if (kPace) myslot = atomicAdd(&q[192 + smid], 1u);
    for (int u = next(-1); ; u = next(u)) {
      if (u >= units) {
        if (kPace) pg[myslot] = 0x7fffffffu;
        mbar_wait(&empty[st], ph ^ 1);
        stu[st] = -1;
        mbar_arrive(&full[st]);
        break;
      }
      const int uu = u % units1;
      const int ch = uu % nch, b = uu / nch, bi = b % nbi, bj = b / nbi;
      for (int k = 0; k < nst; ++k) {
        mbar_wait(&empty[st], ph ^ 1);
        if (kPace) {
          pg[myslot] = ++total;
          for (;;) {
            const unsigned n = *(volatile unsigned*)&q[192 + smid];
            unsigned m = 0x7fffffffu;
            for (unsigned j = 0; j < n && j < 4; ++j)
              if (j != myslot) m = min(m, pg[j]);
            if (total <= m + kPace) break;
            __nanosleep(100);
          }
        }
        stu[st] = u;
        if (MODE == 2) {
          mbar_arrive(&full[st]);
        } else {
          mbar_expect(&full[st], kSt * 8);
          tma3(sm + st * kSt, &mA, ch * SL, bi * PI, k * KS, &full[st]);
          tma3(sm + st * kSt + kA, &mB, ch * SL, bj * PJ, k * KS, &full[st]);
        }
        if (++st == NS) {
          st = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }
  const int sub = tg / SL, slot = tg % SL;
  const int r0 = (sub / (PJ / RJ)) * RI, c0 = (sub % (PJ / RJ)) * RJ;
  int st = 0;
  uint32_t ph = 0;
  bool first = true;
  for (;;) {
    mbar_wait(&full[st], ph);
    if (first && crec && tg == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(crec[3 * vb + 1]));
    first = false;
    const int u = stu[st];
    if (u < 0) break;
    const int uu = u % units1;
    const int ch = uu % nch, b = uu / nch, bi = b % nbi, bj = b / nbi;
    unsigned long long t_begin = 0;
    if (rec && tg == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
    double acc[RI][RJ];
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
      for (int j = 0; j < RJ; ++j) acc[i][j] = -0.0;
    for (int k = 0; k < nst; ++k) {
      if (k > 0) mbar_wait(&full[st], ph);
      const double* sA = sm + st * kSt + r0 * SL + slot;
      const double* sB = sm + st * kSt + kA + c0 * SL + slot;
#ifdef SG_PIPE
      // operands of step h + 1 loaded before the arithmetic of step h (register double buffer)
      double a[RI], bb[RJ];
#pragma unroll
      for (int i = 0; i < RI; ++i) a[i] = sA[i * SL];
#pragma unroll
      for (int j = 0; j < RJ; ++j) bb[j] = sB[j * SL];
#pragma unroll
      for (int h = 0; h < KS; ++h) {
        double an[RI], bn[RJ];
        if (h + 1 < KS) {
#pragma unroll
          for (int i = 0; i < RI; ++i) an[i] = sA[(h + 1) * PI * SL + i * SL];
#pragma unroll
          for (int j = 0; j < RJ; ++j) bn[j] = sB[(h + 1) * PJ * SL + j * SL];
        }
#pragma unroll
        for (int i = 0; i < RI; ++i)
#pragma unroll
          for (int j = 0; j < RJ; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a[i], bb[j]));
        if (h + 1 < KS) {
#pragma unroll
          for (int i = 0; i < RI; ++i) a[i] = an[i];
#pragma unroll
          for (int j = 0; j < RJ; ++j) bb[j] = bn[j];
        }
      }
#else
#pragma unroll
      for (int h = 0; h < KS; ++h) {
        double a[RI], bb[RJ];
#pragma unroll
        for (int i = 0; i < RI; ++i) a[i] = sA[h * PI * SL + i * SL];
#pragma unroll
        for (int j = 0; j < RJ; ++j) bb[j] = sB[h * PJ * SL + j * SL];
#pragma unroll
        for (int i = 0; i < RI; ++i)
#pragma unroll
          for (int j = 0; j < RJ; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a[i], bb[j]));
      }
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == NS) {
        st = 0;
        ph ^= 1;
      }
    }
    if (rec && tg == 0) {
      unsigned long long t_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      rec[3 * u] = t_begin;
      rec[3 * u + 1] = t_end;
      rec[3 * u + 2] = smid * 65536ull + vb;
    }
    if (u < units1 || MODE != 0) {
      double* o = out + ((size_t)(bi * PI + r0) * NJ + bj * PJ + c0) * S + ch * SL + slot;
#pragma unroll
      for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < RJ; ++j) o[((size_t)i * NJ + j) * S] = acc[i][j];
    }
  }
  if (crec && tg == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(crec[3 * vb + 2]));
}

__global__ void stamp_kernel(unsigned long long* t) {
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t[0]));
}

__global__ void ref_kernel(const double* A, const double* B, double* out) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)NI * NJ * S) return;
  const int h = idx % S, g = idx / S, i = g / NJ, j = g % NJ;
  double acc = -0.0;
  for (int k = 0; k < K; ++k) acc = __dadd_rn(acc, __dmul_rn(A[((size_t)k * NI + i) * S + h], B[((size_t)k * NJ + j) * S + h]));
  out[idx] = acc;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncFn enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return (EncFn)p;
}

static void make_map(CUtensorMap* m, const double* base, int rows, int box_s, int box_r, int box_k) {
  cuuint64_t dims[3] = {(cuuint64_t)S, (cuuint64_t)rows, (cuuint64_t)K};
  cuuint64_t str[2] = {(cuuint64_t)S * 8, (cuuint64_t)rows * S * 8};
  cuuint32_t box[3] = {(cuuint32_t)box_s, (cuuint32_t)box_r, (cuuint32_t)box_k};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
}

double *gA, *gB, *gO, *gR;
unsigned* gQ;
int g_sms;
int g_run_idx = 0;

template <int PI, int PJ, int SL, int RI, int RJ, int KS, int NS, int MODE, int MINB, int SCHED = 1>
void run(const char* name, int reps) {
  const int me = g_run_idx++;
  if (getenv("SG_ONLY") && atoi(getenv("SG_ONLY")) != me) return;
  CUtensorMap mA, mB;
  make_map(&mA, gA, NI, SL, PI, KS);
  make_map(&mB, gB, NJ, SL, PJ, KS);
  constexpr int threads = ((PI / RI) * (PJ / RJ) * SL + 32) * G;
  constexpr size_t smem = ((size_t)NS * KS * (PI + PJ) * SL * 8 + (3 * NS + 15) / 16 * 128) * G;
  auto k = sg_kernel<PI, PJ, SL, RI, RJ, KS, NS, MODE, MINB, SCHED>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, k));
  const int units = (NI / PI) * (NJ / PJ) * (S / SL) * reps;
  const int grid = occ * g_sms;
  if (occ != MINB) { printf("%s: occupancy %d != %d, skipped\n", name, occ, MINB); return; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  CK(cudaMemset(gO, 0xff, (size_t)NI * NJ * S * 8));
  CK(cudaMemset(gQ, 0, 4096));
  k<<<grid, threads, smem>>>(mA, mB, gO, reps, gQ, nullptr, nullptr);
  CK(cudaDeviceSynchronize());
  bool ok = true;
  if (MODE == 0) {
    std::vector<double> o((size_t)NI * NJ * S), r((size_t)NI * NJ * S);
    CK(cudaMemcpy(o.data(), gO, o.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r.data(), gR, r.size() * 8, cudaMemcpyDeviceToHost));
    ok = memcmp(o.data(), r.data(), o.size() * 8) == 0;
  }
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
    CK(cudaMemsetAsync(gQ, 0, 4096));
    cudaEventRecord(e0);
    k<<<grid, threads, smem>>>(mA, mB, gO, reps, gQ, nullptr, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  if (getenv("SG_TIMELINE")) {
    const int units = (NI / PI) * (NJ / PJ) * (S / SL) * reps;
    unsigned long long* rec;
    CK(cudaMalloc(&rec, units * 24));
    CK(cudaMemsetAsync(gQ, 0, 4096));
    unsigned long long* crec;
    const int vg = grid * G;
    CK(cudaMalloc(&crec, (vg * 3 + 2) * 8));
    CK(cudaMemsetAsync(crec, 0, (vg * 3 + 2) * 8));
    CK(cudaDeviceSynchronize());
    stamp_kernel<<<1, 1>>>(crec + vg * 3);  // ends right before the fold kernel starts
    k<<<grid, threads, smem>>>(mA, mB, gO, reps, gQ, rec, crec);
    stamp_kernel<<<1, 1>>>(crec + vg * 3 + 1);  // starts right after it ends
    CK(cudaDeviceSynchronize());
    {
      std::vector<unsigned long long> c(vg * 3 + 2);
      CK(cudaMemcpy(c.data(), crec, c.size() * 8, cudaMemcpyDeviceToHost));
      const unsigned long long pre = c[vg * 3], post = c[vg * 3 + 1];
      std::vector<double> en, fd, ex;
      for (int b = 0; b < vg; ++b) {
        en.push_back((c[3 * b] - pre) * 1e-3);
        fd.push_back((c[3 * b + 1] - pre) * 1e-3);
        ex.push_back((c[3 * b + 2] - pre) * 1e-3);
      }
      {
        const int tiers = vg / g_sms;
        printf("   mean CTA exit by launch tier (blockIdx / #SMs):");
        for (int t = 0; t < tiers; ++t) {
          double a = 0;
          for (int b = t * g_sms; b < (t + 1) * g_sms; ++b) a += ex[b] - en[b];
          printf(" %.1f", a / g_sms);
        }
        printf(" us after entry\n");
      }
      std::sort(en.begin(), en.end()); std::sort(fd.begin(), fd.end()); std::sort(ex.begin(), ex.end());
      printf("   CTA stamps (us after the preceding kernel's stamp): entry %.2f/%.2f/%.2f  first data %.2f/%.2f/%.2f  exit %.2f/%.2f/%.2f  next kernel %.2f\n",
             en[0], en[vg / 2], en[vg - 1], fd[0], fd[vg / 2], fd[vg - 1], ex[0], ex[vg / 2], ex[vg - 1], (post - pre) * 1e-3);
    }
    cudaFree(crec);
    std::vector<unsigned long long> h(units * 3);
    CK(cudaMemcpy(h.data(), rec, units * 24, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int u = 0; u < units; ++u) { t0 = std::min(t0, h[3 * u]); t1 = std::max(t1, h[3 * u + 1]); }
    std::vector<double> sm_end(g_sms, 0), sm_busy(g_sms, 0);
    std::vector<int> sm_units(g_sms, 0);
    double dsum = 0, dmin = 1e30, dmax = 0;
    for (int u = 0; u < units; ++u) {
      const int sm = (int)(h[3 * u + 2] >> 16);
      const double b = (h[3 * u] - t0) * 1e-3, e = (h[3 * u + 1] - t0) * 1e-3;
      sm_end[sm] = std::max(sm_end[sm], e);
      sm_units[sm]++;
      dsum += e - b; dmin = std::min(dmin, e - b); dmax = std::max(dmax, e - b);
    }
    std::vector<double> ends = sm_end;
    std::sort(ends.begin(), ends.end());
    int hist[12] = {0};
    for (int i = 0; i < g_sms; ++i) hist[std::min(11, sm_units[i])]++;
    printf("   timeline: span %.1f us; unit duration min/avg/max %.1f/%.1f/%.1f us; SM finish p0/p10/p50/p90/p100 %.1f/%.1f/%.1f/%.1f/%.1f us\n",
           (t1 - t0) * 1e-3, dmin, dsum / units, dmax, ends[0], ends[g_sms / 10], ends[g_sms / 2], ends[g_sms * 9 / 10], ends[g_sms - 1]);
    printf("   units per SM histogram:");
    for (int i = 0; i < 12; ++i) if (hist[i]) printf(" %d:%d", i, hist[i]);
    printf("\n");
    // first unit start per SM and per-round timing
    double first_end = 1e30;
    for (int u = 0; u < units; ++u) first_end = std::min(first_end, (h[3 * u + 1] - t0) * 1e-3);
    printf("   earliest unit end %.1f us\n", first_end);
    cudaFree(rec);
  }
  const double ops = 2.0 * NI * NJ * K * (double)S * reps;
  printf("%-40s reps=%d thr=%3d occ=%d grid=%4d regs=%3d smem=%6zu  %8.2f us  %5.1f%% fp64 %s\n", name, reps, threads,
         occ, grid, fa.numRegs, smem, best * 1e3, ops / (best * 1e-3) / 18.34e12 * 100, ok ? "bitwise-ok" : "MISMATCH");
}

int main() {
  CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t na = (size_t)K * NI * S, nb = (size_t)K * NJ * S;
  std::vector<double> h(na);
  uint64_t x = 88172645463325252ull;
  for (auto& v : h) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v = ((x >> 11) * (1.0 / 9007199254740992.0)) * 2 - 1;
  }
  CK(cudaMalloc(&gA, na * 8));
  CK(cudaMalloc(&gB, nb * 8));
  CK(cudaMalloc(&gO, (size_t)NI * NJ * S * 8));
  CK(cudaMalloc(&gR, (size_t)NI * NJ * S * 8));
  CK(cudaMalloc(&gQ, 4096));
  CK(cudaMemcpy(gA, h.data(), na * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(gB, h.data() + 7, nb * 8, cudaMemcpyHostToDevice));
  ref_kernel<<<(NI * NJ * S + 255) / 256, 256>>>(gA, gB, gR);
  CK(cudaDeviceSynchronize());
#if G_GROUPS > 1
  run<16, 16, 16, 8, 4, 4, 4, 0, 1, 1>("G groups/CTA per-SM queue", 1);
  run<16, 16, 16, 8, 4, 4, 4, 0, 1, 0>("G groups/CTA static", 1);
  run<16, 16, 16, 8, 4, 4, 4, 0, 1, 2>("G groups/CTA global queue", 1);
  run<16, 16, 16, 8, 4, 4, 4, 2, 1, 0>("G groups/CTA static MODE2 (no TMA)", 1);
  run<16, 16, 16, 8, 4, 4, 4, 2, 1, 0>("G groups/CTA static MODE2 (no TMA)", 4);
  run<16, 16, 16, 8, 4, 4, 4, 0, 1, 2>("G groups/CTA global queue", 4);
  return 0;
#endif
  // index (SG_ONLY):  0 shipped shape, per-SM queue   1 static   2 the library's global queue
  //   3 no TMA, static   4 no TMA, 4 reps (steady state)   5 ring 6 steps x 3 stages
  //   6 ring 12 steps x 2 stages at 2 CTAs/SM   7 CTAs of an SM paced against each other
  //   8 shipped shape, 4 reps (steady state)
  run<16, 16, 16, 8, 4, 4, 4, 0, 3, 1>("16x16x16 8x4 ks4 ns4 per-SM", 1);
  run<16, 16, 16, 8, 4, 4, 4, 0, 3, 0>("16x16x16 8x4 ks4 ns4 static", 1);
  run<16, 16, 16, 8, 4, 4, 4, 0, 3, 2>("16x16x16 8x4 ks4 ns4 global queue", 1);
  run<16, 16, 16, 8, 4, 4, 4, 2, 3, 0>("16x16x16 static MODE2 (no TMA)", 1);
  run<16, 16, 16, 8, 4, 4, 4, 2, 3, 0>("16x16x16 static MODE2 (no TMA)", 4);
  run<16, 16, 16, 8, 4, 6, 3, 0, 3, 1>("16x16x16 8x4 ks6 ns3 per-SM", 1);
  run<16, 16, 16, 8, 4, 12, 2, 0, 2, 1>("16x16x16 8x4 ks12 ns2 2 CTAs/SM", 1);
  run<16, 16, 16, 8, 4, 4, 4, 0, 3, 42>("16x16x16 global queue, paced (4 stages)", 1);
  run<16, 16, 16, 8, 4, 4, 4, 0, 3, 1>("16x16x16 8x4 ks4 ns4 per-SM", 4);
  return 0;
}

// kernels/group.cuh -- group programs: fused external fold + in-tile rotate-and-sum (register, TMA-ring, sliding-window, generic) and the split fold.
// Included by tt_kernels.cu inside namespace ttb::{anonymous}: one
// translation unit, so the kernels share its device helpers (FastDiv,
// dadd / dmul, mbarrier and TMA wrappers) without external linkage.
#pragma once

// ---- group programs (reductions) ---------------------------------------------------

struct GroupParams {
  GroupSpec g;
  FastDiv64 gdiv[R];  // divide by g.ext[i]
  int64_t s;
  int nops;
  int nbuf;           // logical scratch tiles
  int use_smem;       // scratch tiles live in dynamic shared memory
  int nlevels;        // simple_pow2: number of in-place ROTADD levels
  int64_t rots[64];   // simple_pow2: rotation of each level
  GOp ops[kMaxOps];
};

struct GroupBase {
  int64_t out, a, b;
};

// Compact parameters of the fold-only kernels (phase 1, GEMM folds): the
// group grid and the one FOLD instruction.  ~0.5 KB instead of GroupParams'
// ~3.3 KB program -- kernel-parameter size is paid on every launch, and small
// ops are launch bound.
struct FoldParams {
  GroupSpec g;
  FastDiv64 gdiv[R];
  int64_t s;
  int64_t first, count;  // FOLD over operand steps [first, first + count)
  int nlevels;           // column-tree fusion: power-of-two levels
  int late;              // release PDL dependents at CTA exit (a tree pass follows)
};

FoldParams to_fold(const GroupParams& p, bool late = false) {
  FoldParams f;
  f.late = late ? 1 : 0;
  f.g = p.g;
  for (int i = 0; i < R; ++i) f.gdiv[i] = p.gdiv[i];
  f.s = p.s;
  f.first = p.ops[0].x;
  f.count = p.ops[0].y;
  f.nlevels = p.nlevels;
  return f;
}

template <class PP>
__device__ __forceinline__ GroupBase group_base(const PP& p, uint64_t v) {
  GroupBase gb{0, 0, 0};
#pragma unroll
  for (int i = R - 1; i >= 0; --i) {
    if (i < p.g.nd) {
      const uint64_t q = fdiv(v, p.gdiv[i]);
      const int64_t c = static_cast<int64_t>(v - q * p.gdiv[i].d);
      v = q;
      gb.out += c * p.g.out_stride[i];
      gb.a += c * p.g.a_stride[i];
      gb.b += c * p.g.b_stride[i];
    }
  }
  return gb;
}

// FOLD for one pair of slots (j, j+1) when VEC, else one slot j:
//   acc = P[first]; acc = acc + P[first+1]; ...   P[l] = A[l] (* B[l]).
template <bool HAS_B, bool VEC, class PP>
__device__ __forceinline__ void fold_slots(const PP& p, const GroupBase& gb,
                                           const double* __restrict__ A,
                                           const double* __restrict__ B, int64_t first,
                                           int64_t count, int64_t j, double* dst) {
  const int64_t s = p.s;
  const double* pa = A + (gb.a + first * p.g.astep) * s + j;
  const int64_t sa = p.g.astep * s;
  const double* pb = HAS_B ? B + (gb.b + first * p.g.bstep) * s + j : nullptr;
  const int64_t sb = p.g.bstep * s;
  if (VEC) {
    double2 x = __ldg(reinterpret_cast<const double2*>(pa));
    double2 acc;
    double2 w;
    if (HAS_B) {
      w = __ldg(reinterpret_cast<const double2*>(pb));
      acc = make_double2(dmul(x.x, w.x), dmul(x.y, w.y));
    } else {
      acc = x;
    }
    if (HAS_B && sb == 0) {  // broadcast B along the summed dim: load once
#pragma unroll 8
      for (int64_t c = 1; c < count; ++c) {
        x = __ldg(reinterpret_cast<const double2*>(pa + c * sa));
        acc.x = dadd(acc.x, dmul(x.x, w.x));
        acc.y = dadd(acc.y, dmul(x.y, w.y));
      }
    } else {
#pragma unroll 4
      for (int64_t c = 1; c < count; ++c) {
        x = __ldg(reinterpret_cast<const double2*>(pa + c * sa));
        if (HAS_B) {
          const double2 y = __ldg(reinterpret_cast<const double2*>(pb + c * sb));
          acc.x = dadd(acc.x, dmul(x.x, y.x));
          acc.y = dadd(acc.y, dmul(x.y, y.y));
        } else {
          acc.x = dadd(acc.x, x.x);
          acc.y = dadd(acc.y, x.y);
        }
      }
    }
    *reinterpret_cast<double2*>(dst) = acc;
  } else {
    double acc = HAS_B ? dmul(__ldg(pa), __ldg(pb)) : __ldg(pa);
#pragma unroll 4
    for (int64_t c = 1; c < count; ++c) {
      const double x = __ldg(pa + c * sa);
      acc = dadd(acc, HAS_B ? dmul(x, __ldg(pb + c * sb)) : x);
    }
    *dst = acc;
  }
}

// FOLD for NP independent slot pairs at j0 + k*jstride (k < NP), all valid
// and 16-byte aligned.  Each fold step issues NP (or 2*NP with a B operand)
// independent 16-byte loads before any dependent arithmetic, so a thread
// keeps NP*16 B (x2 with unroll) of HBM reads in flight -- the fold is
// latency bound otherwise (one long-scoreboard stall per tile step).
template <bool HAS_B, int NP, class PP>
__device__ __forceinline__ void fold_pairs(const PP& p, const GroupBase& gb,
                                           const double* __restrict__ A,
                                           const double* __restrict__ B, int64_t first,
                                           int64_t count, int64_t j0, int64_t jstride,
                                           double* dst, int64_t dst_stride) {
  const int64_t s = p.s;
  const double* pa = A + (gb.a + first * p.g.astep) * s + j0;
  const int64_t sa = p.g.astep * s;
  const double* pb = HAS_B ? B + (gb.b + first * p.g.bstep) * s + j0 : nullptr;
  const int64_t sb = p.g.bstep * s;
  double2 acc[NP];
  double2 w[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const double2 x = __ldg(reinterpret_cast<const double2*>(pa + k * jstride));
    if (HAS_B) {
      w[k] = __ldg(reinterpret_cast<const double2*>(pb + k * jstride));
      acc[k] = make_double2(dmul(x.x, w[k].x), dmul(x.y, w[k].y));
    } else {
      acc[k] = x;
    }
  }
  if (HAS_B && sb == 0) {  // B broadcast along the summed dim: its pairs stay in registers
#pragma unroll 2
    for (int64_t c = 1; c < count; ++c) {
      double2 x[NP];
#pragma unroll
      for (int k = 0; k < NP; ++k)
        x[k] = __ldg(reinterpret_cast<const double2*>(pa + c * sa + k * jstride));
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        acc[k].x = dadd(acc[k].x, dmul(x[k].x, w[k].x));
        acc[k].y = dadd(acc[k].y, dmul(x[k].y, w[k].y));
      }
    }
  } else {
#pragma unroll 2
    for (int64_t c = 1; c < count; ++c) {
      double2 x[NP], y[NP];
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        x[k] = __ldg(reinterpret_cast<const double2*>(pa + c * sa + k * jstride));
        if (HAS_B) y[k] = __ldg(reinterpret_cast<const double2*>(pb + c * sb + k * jstride));
      }
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        if (HAS_B) {
          acc[k].x = dadd(acc[k].x, dmul(x[k].x, y[k].x));
          acc[k].y = dadd(acc[k].y, dmul(x[k].y, y[k].y));
        } else {
          acc[k].x = dadd(acc[k].x, x[k].x);
          acc[k].y = dadd(acc[k].y, x[k].y);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) *reinterpret_cast<double2*>(dst + k * dst_stride) = acc[k];
}

// Fast path: FOLD into one shared tile, then `nlevels` in-place rotate-adds
// (the power-of-two schedule, rotate_sum.hpp:51-56), the last into the output
// tile.  Each thread owns slots j = i*T + tid; a level reads the partner
// slot from shared memory into registers, barriers, then writes.
template <int VMAX, bool HAS_B, bool VEC>
__global__ void __launch_bounds__(512, 1) group_pow2_kernel(const __grid_constant__ GroupParams p,
                                                            const double* __restrict__ A,
                                                            const double* __restrict__ B,
                                                            double* __restrict__ OUT) {
  pdl_enter();
  extern __shared__ __align__(16) double sbuf[];
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  const int s = static_cast<int>(p.s);
  const int64_t first = p.ops[0].x;
  const int64_t count = p.ops[0].y;
  for (uint64_t v = blockIdx.x; v < static_cast<uint64_t>(p.g.groups); v += gridDim.x) {
    const GroupBase gb = group_base(p, v);
    if (VEC) {
      // pairs q = tid + i*T; batches of 4 pairs (i, i+1, i+2, i+3) per thread
      // (2 pairs per batch when the tree's val[32] already claims 64 registers)
      constexpr int NP = VMAX >= 32 ? 2 : 4;
      const int npairs = s / 2;
      int q = tid;
      for (; q + (NP - 1) * T < npairs; q += NP * T)
        fold_pairs<HAS_B, NP>(p, gb, A, B, first, count, 2 * q, 2 * T, sbuf + 2 * q, 2 * T);
      for (; q < npairs; q += T)
        fold_pairs<HAS_B, 1>(p, gb, A, B, first, count, 2 * q, 0, sbuf + 2 * q, 0);
    } else {
      for (int j = tid; j < s; j += T) fold_slots<HAS_B, false>(p, gb, A, B, first, count, j, sbuf + j);
    }
    __syncthreads();
    double val[VMAX];
#pragma unroll
    for (int i = 0; i < VMAX; ++i) {
      const int j = i * T + tid;
      if (j < s) val[i] = sbuf[j];
    }
    const bool pow2_s = (s & (s - 1)) == 0;
    for (int lv = 0; lv < p.nlevels; ++lv) {
      const int r = static_cast<int>(p.rots[lv]);
      if (pow2_s) {  // cyclic index by mask: no per-slot compare
        const int mask = s - 1;
        const int base = tid + r;
#pragma unroll
        for (int i = 0; i < VMAX; ++i)
          if (i * T + tid < s) val[i] = dadd(val[i], sbuf[(base + i * T) & mask]);
      } else {
#pragma unroll
        for (int i = 0; i < VMAX; ++i) {
          const int j = i * T + tid;
          if (j < s) {
            int jj = j + r;
            if (jj >= s) jj -= s;
            val[i] = dadd(val[i], sbuf[jj]);
          }
        }
      }
      __syncthreads();
      if (lv + 1 < p.nlevels) {
#pragma unroll
        for (int i = 0; i < VMAX; ++i) {
          const int j = i * T + tid;
          if (j < s) sbuf[j] = val[i];
        }
        __syncthreads();
      }
    }
    double* out = OUT + gb.out * p.s;
#pragma unroll
    for (int i = 0; i < VMAX; ++i) {
      const int j = i * T + tid;
      if (j < s) out[j] = val[i];
    }
    // The last level's reads completed before its barrier, so the next
    // group's FOLD may overwrite sbuf without another barrier.
  }
}

// ---- TMA-fed fused fold + power-of-two tree ---------------------------------------
// The B200-native fast path.  One producer warp streams every fold operand
// chunk (16 KiB of one tile, plus the matching chunk of B when B varies
// along the summed dim) into a shared-memory ring with cp.async.bulk
// (TMA bulk copies, SASS UBLKCP) completing on mbarriers; 16 consumer warps
// fold each chunk from shared memory into registers and release the stage.
// The ring keeps ~96 KiB of HBM reads in flight per SM independent of
// register pressure, and the producer runs ahead into the next group while
// the consumers execute the current group's rotate-and-sum tree.

constexpr int kTmaConsumerWarps = 16;
constexpr int kTmaConsumers = kTmaConsumerWarps * 32;
constexpr int kTmaThreads = kTmaConsumers + 32;
constexpr int kTmaPairsPerThread = 2;                         // per stage
constexpr int kTmaChunk = 2 * kTmaConsumers * kTmaPairsPerThread;  // 2048 slots = 16 KiB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// try_wait with a suspend-time hint: the thread sleeps until the phase
// completes (or the hint expires) instead of re-issuing the probe -- for
// waiters whose spinning would take issue slots from compute warps on the
// same SM sub-partition (the GEMM fold's producer warp).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x100000u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_keep(double* p, double v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(policy) : "memory");
}
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumers) : "memory");
}

template <int VMAX, bool HAS_B>
__global__ void __launch_bounds__(kTmaThreads, 1)
    group_tma_kernel(const __grid_constant__ GroupParams p, const double* __restrict__ A,
                     const double* __restrict__ B, double* __restrict__ OUT, int nstages) {
  pdl_enter();
  extern __shared__ __align__(128) double smem[];
  const int s = static_cast<int>(p.s);
  const bool b_stream = HAS_B && p.g.bstep != 0;
  const int stage_doubles = kTmaChunk * (b_stream ? 2 : 1);
  double* tile = smem;
  double* ring = smem + s;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<int64_t>(nstages) * stage_doubles);
  uint64_t* empty = full + nstages;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t first = p.ops[0].x;
  const int64_t count = p.ops[0].y;
  const int nchunks = s / kTmaChunk;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nstages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kTmaConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kTmaConsumerWarps) {  // ---- producer ----
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_first();  // streamed once
      const uint64_t pol_b = policy_evict_last();   // shared by neighbouring groups
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t chunk_bytes = kTmaChunk * sizeof(double);
      for (uint64_t v = blockIdx.x; v < static_cast<uint64_t>(p.g.groups); v += gridDim.x) {
        const GroupBase gb = group_base(p, v);
        for (int r = 0; r < nchunks; ++r) {
          for (int64_t c = 0; c < count; ++c) {
            mbar_wait(&empty[stage], phase ^ 1);
            double* dst = ring + static_cast<int64_t>(stage) * stage_doubles;
            mbar_arrive_expect_tx(&full[stage], chunk_bytes * (b_stream ? 2 : 1));
            const double* src = A + (gb.a + (first + c) * p.g.astep) * p.s + r * kTmaChunk;
            bulk_g2s(dst, src, chunk_bytes, &full[stage], pol_a);
            if (b_stream) {
              const double* sb = B + (gb.b + (first + c) * p.g.bstep) * p.s + r * kTmaChunk;
              bulk_g2s(dst + kTmaChunk, sb, chunk_bytes, &full[stage], pol_b);
            }
            if (++stage == nstages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
    return;
  }

  // ---- consumers ----
  const int tid = threadIdx.x;
  int stage = 0;
  uint32_t phase = 0;
  for (uint64_t v = blockIdx.x; v < static_cast<uint64_t>(p.g.groups); v += gridDim.x) {
    const GroupBase gb = group_base(p, v);
    for (int r = 0; r < nchunks; ++r) {
      double2 acc[kTmaPairsPerThread];
      double2 w[kTmaPairsPerThread];
      if (HAS_B && !b_stream) {  // B broadcast along the summed dim: one load per chunk
        const double* pb = B + (gb.b + first * p.g.bstep) * p.s + r * kTmaChunk;
#pragma unroll
        for (int k = 0; k < kTmaPairsPerThread; ++k)
          w[k] = __ldg(reinterpret_cast<const double2*>(pb) + tid + k * kTmaConsumers);
      }
      for (int64_t c = 0; c < count; ++c) {
        mbar_wait(&full[stage], phase);
        const double2* st = reinterpret_cast<const double2*>(ring + static_cast<int64_t>(stage) * stage_doubles);
#pragma unroll
        for (int k = 0; k < kTmaPairsPerThread; ++k) {
          const double2 x = st[tid + k * kTmaConsumers];
          double2 prod;
          if (HAS_B) {
            const double2 y = b_stream ? st[kTmaChunk / 2 + tid + k * kTmaConsumers] : w[k];
            prod = make_double2(dmul(x.x, y.x), dmul(x.y, y.y));
          } else {
            prod = x;
          }
          if (c == 0) {
            acc[k] = prod;
          } else {
            acc[k].x = dadd(acc[k].x, prod.x);
            acc[k].y = dadd(acc[k].y, prod.y);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == nstages) {
          stage = 0;
          phase ^= 1;
        }
      }
      double2* dt = reinterpret_cast<double2*>(tile + r * kTmaChunk);
#pragma unroll
      for (int k = 0; k < kTmaPairsPerThread; ++k) dt[tid + k * kTmaConsumers] = acc[k];
    }
    consumer_sync();
    // power-of-two rotate-and-sum on the folded tile (rotate_sum.hpp:51-56)
    double val[VMAX];
#pragma unroll
    for (int i = 0; i < VMAX; ++i) {
      const int j = i * kTmaConsumers + tid;
      if (j < s) val[i] = tile[j];
    }
    const int mask = s - 1;  // s is a power of two on this path
    for (int lv = 0; lv < p.nlevels; ++lv) {
      const int base = tid + static_cast<int>(p.rots[lv]);
#pragma unroll
      for (int i = 0; i < VMAX; ++i)
        if (i * kTmaConsumers + tid < s) val[i] = dadd(val[i], tile[(base + i * kTmaConsumers) & mask]);
      consumer_sync();
      if (lv + 1 < p.nlevels) {
#pragma unroll
        for (int i = 0; i < VMAX; ++i) {
          const int j = i * kTmaConsumers + tid;
          if (j < s) tile[j] = val[i];
        }
        consumer_sync();
      }
    }
    double* out = OUT + gb.out * p.s;
#pragma unroll
    for (int i = 0; i < VMAX; ++i) {
      const int j = i * kTmaConsumers + tid;
      if (j < s) out[j] = val[i];
    }
  }
}

// ---- sliding-window variant ---------------------------------------------------------
// When the power-of-two schedule's reach H = (t-1)*stride is at most one
// chunk (c5 dims 2 and 3: H = 992 and 31 slots), output slot j only depends on
// folded slots j .. j+H (cyclic), so chunk r is finalised right after chunk
// r+1 has been folded, from [chunk r | first H slots of chunk r+1] (the last
// chunk wraps to a saved head of chunk 0).  Shared memory then holds two
// folded chunks + two H-slot halos (~48 KiB) instead of the whole 128 KiB
// tile, and the TMA ring gets the rest: ~2x the bytes in flight, and the tree
// work is spread between the fold steps instead of stalling the SM per group.
// Level k of the schedule runs on the shrinking range [0, CH + H - sum_{i<=k} d_i).

constexpr int kWinVmax = 8;  // (CH + H) / consumers, rounded up: (2048 + 2047) / 512

template <bool HAS_B>
__global__ void __launch_bounds__(kTmaThreads, 1)
    group_tma_win_kernel(const __grid_constant__ GroupParams p, const double* __restrict__ A,
                         const double* __restrict__ B, double* __restrict__ OUT, int nstages,
                         int halo) {
  pdl_enter();
  extern __shared__ __align__(128) double smem[];
  const int s = static_cast<int>(p.s);
  const bool b_stream = HAS_B && p.g.bstep != 0;
  const int stage_doubles = kTmaChunk * (b_stream ? 2 : 1);
  double* cbuf = smem;                         // 2 folded chunks (ping-pong)
  double* work = smem + 2 * kTmaChunk;         // chunk r-1 copy + halo: CH + H
  double* head = work + kTmaChunk + halo;      // first H slots of chunk 0
  // TMA destinations must stay 16-byte aligned: start the ring on a 128 B line
  double* ring = smem + 3 * kTmaChunk + ((2 * halo + 15) / 16) * 16;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<int64_t>(nstages) * stage_doubles);
  uint64_t* empty = full + nstages;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t first = p.ops[0].x;
  const int64_t count = p.ops[0].y;
  const int nchunks = s / kTmaChunk;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nstages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kTmaConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kTmaConsumerWarps) {  // ---- producer (as in group_tma_kernel) ----
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t chunk_bytes = kTmaChunk * sizeof(double);
      for (uint64_t v = blockIdx.x; v < static_cast<uint64_t>(p.g.groups); v += gridDim.x) {
        const GroupBase gb = group_base(p, v);
        for (int r = 0; r < nchunks; ++r) {
          for (int64_t c = 0; c < count; ++c) {
            mbar_wait(&empty[stage], phase ^ 1);
            double* dst = ring + static_cast<int64_t>(stage) * stage_doubles;
            mbar_arrive_expect_tx(&full[stage], chunk_bytes * (b_stream ? 2 : 1));
            bulk_g2s(dst, A + (gb.a + (first + c) * p.g.astep) * p.s + r * kTmaChunk, chunk_bytes,
                     &full[stage], pol_a);
            if (b_stream)
              bulk_g2s(dst + kTmaChunk, B + (gb.b + (first + c) * p.g.bstep) * p.s + r * kTmaChunk,
                       chunk_bytes, &full[stage], pol_b);
            if (++stage == nstages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
    return;
  }

  // ---- consumers ----
  const int tid = threadIdx.x;
  int stage = 0;
  uint32_t phase = 0;
  // sum of the level offsets up to and including level k
  int64_t reach[32];
  {
    int64_t acc = 0;
    for (int lv = 0; lv < p.nlevels; ++lv) {
      acc += p.rots[lv];
      reach[lv] = acc;
    }
  }
  // stride-1 schedules with reach < 32 (every offset < 32): warp w owns rows
  // w*4 .. w*4+3 of 32 slots plus the next row as halo; all levels run in
  // registers with shuffles (partner of (row i, lane l) at offset d is
  // (i, l+d) or (i+1, l+d-32)), no barrier and no shared-memory round trip.
  const bool shfl_tree = halo < 32;
  auto finalise_shfl = [&](int rc, const double* src, const double* hal, double* out) {
    const int w = tid >> 5;
    double v[5];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = src[w * 128 + i * 32 + lane];
    v[4] = (w + 1 < kTmaConsumerWarps) ? src[(w + 1) * 128 + lane] : (lane < halo ? hal[lane] : 0.0);
    for (int lv = 0; lv < p.nlevels; ++lv) {
      const int d = static_cast<int>(p.rots[lv]);
      const int srcl = (lane + d) & 31;
      const bool same_row = lane + d < 32;
      double sh[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) sh[i] = __shfl_sync(0xffffffffu, v[i], srcl);
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = dadd(v[i], same_row ? sh[i] : sh[i + 1]);
      v[4] = dadd(v[4], sh[4]);  // only its low lanes stay meaningful; never stored
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) out[static_cast<int64_t>(rc) * kTmaChunk + w * 128 + i * 32 + lane] = v[i];
  };

  // finalise chunk `rc` (folded values in `src`), halo = first H slots of `hal`
  auto finalise = [&](int rc, const double* src, const double* hal, double* out) {
    if (shfl_tree) {
      finalise_shfl(rc, src, hal, out);
      return;
    }
    for (int j = tid; j < kTmaChunk; j += kTmaConsumers) work[j] = src[j];
    for (int j = tid; j < halo; j += kTmaConsumers) work[kTmaChunk + j] = hal[j];
    consumer_sync();
    int range = kTmaChunk + halo;
    for (int lv = 0; lv < p.nlevels; ++lv) {
      const int d = static_cast<int>(p.rots[lv]);
      const int nr = kTmaChunk + halo - static_cast<int>(reach[lv]);
      double val[kWinVmax];
#pragma unroll
      for (int i = 0; i < kWinVmax; ++i) {
        const int j = i * kTmaConsumers + tid;
        if (j < nr) val[i] = dadd(work[j], work[j + d]);
      }
      consumer_sync();
      if (lv + 1 < p.nlevels) {
#pragma unroll
        for (int i = 0; i < kWinVmax; ++i) {
          const int j = i * kTmaConsumers + tid;
          if (j < nr) work[j] = val[i];
        }
        consumer_sync();
      } else {
#pragma unroll
        for (int i = 0; i < kWinVmax; ++i) {
          const int j = i * kTmaConsumers + tid;
          if (j < nr) out[static_cast<int64_t>(rc) * kTmaChunk + j] = val[i];
        }
      }
      range = nr;
    }
    (void)range;
  };

  for (uint64_t v = blockIdx.x; v < static_cast<uint64_t>(p.g.groups); v += gridDim.x) {
    const GroupBase gb = group_base(p, v);
    double* out = OUT + gb.out * p.s;
    for (int r = 0; r < nchunks; ++r) {
      double2 acc[kTmaPairsPerThread];
      double2 w[kTmaPairsPerThread];
      if (HAS_B && !b_stream) {
        const double* pb = B + (gb.b + first * p.g.bstep) * p.s + r * kTmaChunk;
#pragma unroll
        for (int k = 0; k < kTmaPairsPerThread; ++k)
          w[k] = __ldg(reinterpret_cast<const double2*>(pb) + tid + k * kTmaConsumers);
      }
      for (int64_t c = 0; c < count; ++c) {
        mbar_wait(&full[stage], phase);
        const double2* st = reinterpret_cast<const double2*>(ring + static_cast<int64_t>(stage) * stage_doubles);
#pragma unroll
        for (int k = 0; k < kTmaPairsPerThread; ++k) {
          const double2 x = st[tid + k * kTmaConsumers];
          double2 prod;
          if (HAS_B) {
            const double2 y = b_stream ? st[kTmaChunk / 2 + tid + k * kTmaConsumers] : w[k];
            prod = make_double2(dmul(x.x, y.x), dmul(x.y, y.y));
          } else {
            prod = x;
          }
          if (c == 0) {
            acc[k] = prod;
          } else {
            acc[k].x = dadd(acc[k].x, prod.x);
            acc[k].y = dadd(acc[k].y, prod.y);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == nstages) {
          stage = 0;
          phase ^= 1;
        }
      }
      double* cb = cbuf + (r & 1) * kTmaChunk;
      double2* dt = reinterpret_cast<double2*>(cb);
#pragma unroll
      for (int k = 0; k < kTmaPairsPerThread; ++k) dt[tid + k * kTmaConsumers] = acc[k];
      consumer_sync();
      if (r == 0) {  // keep chunk 0's head for the cyclic wrap of the last chunk
        for (int j = tid; j < halo; j += kTmaConsumers) head[j] = cb[j];
      } else {
        finalise(r - 1, cbuf + ((r - 1) & 1) * kTmaChunk, cb, out);
      }
      consumer_sync();
    }
    finalise(nchunks - 1, cbuf + ((nchunks - 1) & 1) * kTmaChunk, head, out);
    consumer_sync();
  }
}

// Generic interpreter: any program (ltr/rtl schedules, boundary split,
// replication).  Logical buffers map onto nbuf+1 physical tiles; an in-place
// ROTADD writes the spare tile and swaps it in, so one barrier per op.
template <bool HAS_B>
__global__ void __launch_bounds__(512) group_generic_kernel(const __grid_constant__ GroupParams p,
                                                            const double* __restrict__ A,
                                                            const double* __restrict__ B,
                                                            double* __restrict__ OUT,
                                                            double* __restrict__ scratch) {
  pdl_enter();
  extern __shared__ __align__(16) double sbuf[];
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  const int64_t s = p.s;
  double* base = p.use_smem ? sbuf : scratch + static_cast<int64_t>(blockIdx.x) * (p.nbuf + 1) * s;
  for (uint64_t v = blockIdx.x; v < static_cast<uint64_t>(p.g.groups); v += gridDim.x) {
    const GroupBase gb = group_base(p, v);
    double* out = OUT + gb.out * s;
    int map[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) map[i] = i;
    int spare = p.nbuf;
    for (int k = 0; k < p.nops; ++k) {
      const GOp op = p.ops[k];
      double* dst;
      bool swap = false;
      if (op.dst == BUF_OUT) {
        dst = out;
      } else if (op.inplace) {
        dst = base + static_cast<int64_t>(spare) * s;
        swap = true;
      } else {
        dst = base + static_cast<int64_t>(map[op.dst]) * s;
      }
      if (op.kind == GOP_FOLD) {
        for (int64_t j = tid; j < s; j += T)
          fold_slots<HAS_B, false>(p, gb, A, B, op.x, op.y, j, dst + j);
      } else {
        const double* a = base + static_cast<int64_t>(map[op.a]) * s;
        const double* b = base + static_cast<int64_t>(map[op.b]) * s;
        const int64_t r = op.x;
        if (op.kind == GOP_ROTADD) {
          for (int64_t j = tid; j < s; j += T) {
            int64_t jj = j + r;
            if (jj >= s) jj -= s;
            dst[j] = dadd(a[j], b[jj]);
          }
        } else {
          for (int64_t j = tid; j < s; j += T) dst[j] = a[j];
        }
      }
      if (swap) {
        const int old = map[op.dst];
        map[op.dst] = spare;
        spare = old;
      }
      __syncthreads();
    }
  }
}

// Split fold: the whole grid folds (group, chunk) work units and writes the
// folded tile straight into OUT.  Used when a reduction has no in-tile
// schedule (t == 1) or has too few groups to fill the GPU (phase 1 of 2).
// VEC: a warp owns 128 slot pairs (256 slots) of one group; lane l folds the
// pairs l, l+32, l+64, l+96 (fully coalesced 512-byte requests, 4 loads in
// flight per operand).  Scalar mode: one slot per work item.
template <bool HAS_B, bool VEC>
__global__ void __launch_bounds__(256) fold_kernel(const __grid_constant__ FoldParams p,
                                                    const double* __restrict__ A,
                                                    const double* __restrict__ B,
                                                    double* __restrict__ OUT,
                                                    FastDiv64 units_div) {
  pdl_enter(p.late != 0);
  const int64_t first = p.first;
  const int64_t count = p.count;
  const int64_t s = p.s;
  if (VEC) {
    const uint64_t total = static_cast<uint64_t>(p.g.groups) * units_div.d;  // warp units
    const int lane = threadIdx.x & 31;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
         u < total; u += warps) {
      const uint64_t v = fdiv(u, units_div);
      const int64_t q0 = static_cast<int64_t>(u - v * units_div.d) * 128;
      const GroupBase gb = group_base(p, v);
      double* dst = OUT + gb.out * s;
      const int64_t npairs = s / 2;
      if (q0 + 128 <= npairs) {
        fold_pairs<HAS_B, 4>(p, gb, A, B, first, count, 2 * (q0 + lane), 64, dst + 2 * (q0 + lane), 64);
      } else {
        for (int64_t q = q0 + lane; q < npairs; q += 32)
          fold_pairs<HAS_B, 1>(p, gb, A, B, first, count, 2 * q, 0, dst + 2 * q, 0);
      }
    }
  } else {
    const uint64_t total = static_cast<uint64_t>(p.g.groups) * units_div.d;  // slots
    for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < total;
         w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
      const uint64_t v = fdiv(w, units_div);
      const int64_t j = static_cast<int64_t>(w - v * units_div.d);
      const GroupBase gb = group_base(p, v);
      fold_slots<HAS_B, false>(p, gb, A, B, first, count, j, OUT + gb.out * s + j);
    }
  }
}

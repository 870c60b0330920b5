// kernels/gemm.cuh -- blocked and GEMM-shaped folds for products with two broadcast dims (tile matmul).
// Included by tt_kernels.cu inside namespace ttb::{anonymous}: one
// translation unit, so the kernels share its device helpers (FastDiv,
// dadd / dmul, mbarrier and TMA wrappers) without external linkage.
#pragma once

// ---- blocked fold (tile-tensor matmul) ---------------------------------------------------
// For a product whose group grid has a dim `ia` along which B broadcasts and a
// dim `ib` along which A broadcasts (matmul_a/b: out(i,k) = sum_j A(i,j)B(j,k)),
// a thread folds a P x Q block of groups for one slot: per fold step it loads
// P slots of A and Q of B and updates P*Q accumulators (acc = P[0]; acc += P[l],
// the reference's left fold per group).  A is read ceil(|ib|/Q) times and B
// ceil(|ia|/P) times instead of once per group; consecutive work units cover
// the blocks of one slot chunk so concurrently running CTAs share operand
// chunks in L2.  The folded tiles go to OUT; the in-tile schedule then runs
// in place (two-phase reduction).

struct BlockSpec {
  int64_t ext_ia = 1, ext_ib = 1;            // extents of the blocked dims (1 if absent)
  int64_t a_ia = 0, out_ia = 0;              // tile strides along ia
  int64_t b_ib = 0, out_ib = 0;              // tile strides along ib
  int64_t nbp = 1, nbq = 1;                  // blocks along ia, ib
  int64_t chunks = 1;                        // slot chunks per tile
  int64_t units = 0;
  FastDiv64 div_nbq, div_nbp, div_chunks;
};

constexpr int kBlockThreads = 256;

template <bool HAS_B, int P, int Q>
__global__ void __launch_bounds__(kBlockThreads) fold_blocked_kernel(
    const __grid_constant__ FoldParams p, const __grid_constant__ BlockSpec bs,
    const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ OUT) {
  pdl_enter(p.late != 0);
  const int64_t s = p.s;
  const int64_t first = p.first;
  const int64_t count = p.count;
  const int64_t sa = p.g.astep * s, sb = p.g.bstep * s;
  for (uint64_t u = blockIdx.x; u < static_cast<uint64_t>(bs.units); u += gridDim.x) {
    // u = ((rest * chunks + chunk) * nbp + pb) * nbq + qb
    uint64_t t = u;
    const uint64_t t1 = fdiv(t, bs.div_nbq);
    const int64_t qb = static_cast<int64_t>(t - t1 * bs.div_nbq.d);
    const uint64_t t2 = fdiv(t1, bs.div_nbp);
    const int64_t pb = static_cast<int64_t>(t1 - t2 * bs.div_nbp.d);
    const uint64_t rest = fdiv(t2, bs.div_chunks);
    const int64_t chunk = static_cast<int64_t>(t2 - rest * bs.div_chunks.d);
    const int64_t j = chunk * kBlockThreads + threadIdx.x;
    if (j >= s) continue;
    const GroupBase gb = group_base(p, rest);
    const int np = static_cast<int>(bs.ext_ia - pb * P < P ? bs.ext_ia - pb * P : P);
    const int nq = static_cast<int>(bs.ext_ib - qb * Q < Q ? bs.ext_ib - qb * Q : Q);
    // operand slot j of group row i / column k at fold step c (tails clamp to
    // the last valid group; their results are not stored)
    const double* a0 = A + (gb.a + pb * P * bs.a_ia + first * p.g.astep) * s + j;
    const double* b0 = HAS_B ? B + (gb.b + qb * Q * bs.b_ib + first * p.g.bstep) * s + j : nullptr;
    const int64_t a_row = bs.a_ia * s, b_col = bs.b_ib * s;
    double acc[P][Q];
    {
      double a[P], b[Q];
#pragma unroll
      for (int i = 0; i < P; ++i) a[i] = __ldg(a0 + (i < np ? i : np - 1) * a_row);
#pragma unroll
      for (int k = 0; k < Q; ++k) b[k] = HAS_B ? __ldg(b0 + (k < nq ? k : nq - 1) * b_col) : 1.0;
#pragma unroll
      for (int i = 0; i < P; ++i)
#pragma unroll
        for (int k = 0; k < Q; ++k) acc[i][k] = HAS_B ? dmul(a[i], b[k]) : a[i];
    }
    for (int64_t c = 1; c < count; ++c) {
      double a[P], b[Q];
#pragma unroll
      for (int i = 0; i < P; ++i) a[i] = __ldg(a0 + c * sa + (i < np ? i : np - 1) * a_row);
#pragma unroll
      for (int k = 0; k < Q; ++k)
        b[k] = HAS_B ? __ldg(b0 + c * sb + (k < nq ? k : nq - 1) * b_col) : 1.0;
#pragma unroll
      for (int i = 0; i < P; ++i)
#pragma unroll
        for (int k = 0; k < Q; ++k)
          acc[i][k] = dadd(acc[i][k], HAS_B ? dmul(a[i], b[k]) : a[i]);
    }
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
      for (int k = 0; k < Q; ++k)
        if (i < np && k < nq)
          OUT[(gb.out + (pb * P + i) * bs.out_ia + (qb * Q + k) * bs.out_ib) * s + j] = acc[i][k];
  }
}

// GEMM-shaped variant for products with BOTH broadcast dims (matmul_a/b):
// a CTA folds a 16 x 16 block of groups for 64 consecutive slots.  Each fold
// step stages the block's 16 A-chunks and 16 B-chunks (64 slots each, 16 KiB)
// in shared memory with cp.async (double-buffered, next step in flight while
// this one computes); warp w owns slot half (w & 1) and the 8 x 4 sub-block
// (w >> 1) of the 16 x 16 groups, so each thread reads 8 + 4 operands from
// shared memory for 32 multiply-adds (128 registers, no spills).  Every A chunk is read once per 16
// groups and every B chunk once per 16 groups (vs once per group).
constexpr int kGemmSlots = 64;
constexpr int kGemmBlk = 16;   // block rows (groups along ia)
constexpr int kGemmSubR = 8;
constexpr int kGemmSubC = 4;
constexpr int kGemmStages = 3;  // super-stages in flight
constexpr int kGemmPair = 4;    // fold steps per super-stage (one barrier per super-stage)

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Few groups, long folds (config 4's second layer: 16 groups x 100 steps;
// config 2's matvec): one thread per slot pair, the pair's operands streamed
// through a kFoldRing-deep shared-memory ring with 16-byte cp.async (no
// register dependency, no barrier: a thread only reads what it copied), so
// kFoldRing fold steps of loads are in flight per thread.  A CTA owns 256
// consecutive slots of one group (s % 256 == 0, 16-byte aligned operands).
constexpr int kFoldRing = 8;
// EPI: the reduction's elementwise tail (+ C, square: tt_mul_sum_affine) applied to
// the folded pair before its store -- no separate in-place pass over the result
// (config 4's second layer: fold 22.5 us + epilogue pass 3.2 us -> one kernel).
template <bool HAS_B, bool EPI = false>
__global__ void __launch_bounds__(128) fold_ring_kernel(const __grid_constant__ FoldParams p,
                                                        const double* __restrict__ A,
                                                        const double* __restrict__ B,
                                                        double* __restrict__ OUT, FastDiv64 runs_div,
                                                        const __grid_constant__ EpiDev epi) {
  pdl_enter(p.late != 0);
  __shared__ __align__(16) double2 ring[kFoldRing][HAS_B ? 2 : 1][128];
  const int64_t s = p.s;
  const int64_t count = p.count;
  const int64_t sa = p.g.astep * s;
  const int64_t sb = p.g.bstep * s;
  const bool b_moves = HAS_B && sb != 0;
  const int t = threadIdx.x;
  const uint64_t total = static_cast<uint64_t>(p.g.groups) * runs_div.d;
  for (uint64_t r = blockIdx.x; r < total; r += gridDim.x) {
    const uint64_t v = fdiv(r, runs_div);
    const int64_t j0 = static_cast<int64_t>(r - v * runs_div.d) * 256 + 2 * t;
    const GroupBase gb = group_base(p, v);
    const double* pa = A + (gb.a + p.first * p.g.astep) * s + j0;
    const double* pb = HAS_B ? B + (gb.b + p.first * p.g.bstep) * s + j0 : nullptr;
    double2 wfix = make_double2(0.0, 0.0);
    if (HAS_B && !b_moves) wfix = __ldg(reinterpret_cast<const double2*>(pb));
#pragma unroll
    for (int k = 0; k < kFoldRing; ++k) {
      if (k < count) {
        cp_async16(&ring[k][0][t], pa + k * sa);
        if (b_moves) cp_async16(&ring[k][HAS_B ? 1 : 0][t], pb + k * sb);
      }
      cp_async_commit();
    }
    double2 acc = make_double2(0.0, 0.0);
    int slot = 0;
    for (int64_t c = 0; c < count; ++c) {
      cp_async_wait<kFoldRing - 1>();  // step c has landed
      const double2 x = ring[slot][0][t];
      const double2 y = HAS_B ? (b_moves ? ring[slot][HAS_B ? 1 : 0][t] : wfix) : make_double2(0.0, 0.0);
      const double2 pr = HAS_B ? make_double2(dmul(x.x, y.x), dmul(x.y, y.y)) : x;
      acc = c == 0 ? pr : make_double2(dadd(acc.x, pr.x), dadd(acc.y, pr.y));
      const int64_t f = c + kFoldRing;  // refill this slot with step c + ring
      if (f < count) {
        cp_async16(&ring[slot][0][t], pa + f * sa);
        if (b_moves) cp_async16(&ring[slot][HAS_B ? 1 : 0][t], pb + f * sb);
      }
      cp_async_commit();
      if (++slot == kFoldRing) slot = 0;
    }
    cp_async_wait<0>();
    if (EPI) {
      double x[2] = {acc.x, acc.y};
      epi_apply_n<2>(epi, x, epi_tile(epi, static_cast<uint64_t>(gb.out), s), j0, 1);
      acc = make_double2(x[0], x[1]);
    }
    *reinterpret_cast<double2*>(OUT + gb.out * s + j0) = acc;
  }
}

// Group-blocked ring fold: few groups, long folds in which ONE operand is the
// same for all groups along a group dim (config 2: the vector's tiles for the
// 16 row blocks of the matrix; config 4's second layer: the weight tiles for
// the 16 batch tiles).  The plain ring fold above re-reads that operand from L2
// once per group, and such folds run at the L2's ~9 TB/s, not at HBM's rate.
// Here a thread folds its slot pair for Q consecutive groups along that dim:
// one copy of the shared operand and Q of the other per step, through the same
// per-thread cp.async ring (no barrier).  The host passes a group grid whose
// blocked dim is already divided by Q (strides multiplied), `vq` / `oq` = tile
// strides between the Q groups of the varying operand / the output.  SHARED_A:
// A is the shared operand.  The products and the left fold are those of
// fold_ring_kernel (IEEE multiplication commutes).
template <int Q, int T, bool SHARED_A>
__global__ void __launch_bounds__(T) fold_ring_blk_kernel(const __grid_constant__ FoldParams p,
                                                          const double* __restrict__ A,
                                                          const double* __restrict__ B,
                                                          double* __restrict__ OUT, FastDiv64 runs_div,
                                                          int64_t vq, int64_t oq) {
  pdl_enter(p.late != 0);
  extern __shared__ __align__(16) double2 bring[];  // [kFoldRing][1 + Q][T]
  const int64_t s = p.s;
  const int64_t count = p.count;
  const int64_t ss = (SHARED_A ? p.g.astep : p.g.bstep) * s;  // fold strides
  const int64_t sv = (SHARED_A ? p.g.bstep : p.g.astep) * s;
  const int t = threadIdx.x;
  auto cell = [&](int slot, int which) { return bring + (slot * (1 + Q) + which) * T + t; };
  const uint64_t total = static_cast<uint64_t>(p.g.groups) * runs_div.d;
  for (uint64_t r = blockIdx.x; r < total; r += gridDim.x) {
    const uint64_t v = fdiv(r, runs_div);
    const int64_t j0 = static_cast<int64_t>(r - v * runs_div.d) * (2 * T) + 2 * t;
    const GroupBase gb = group_base(p, v);
    const double* pa = A + (gb.a + p.first * p.g.astep) * s + j0;
    const double* pb = B + (gb.b + p.first * p.g.bstep) * s + j0;
    const double* psh = SHARED_A ? pa : pb;
    const double* pv = SHARED_A ? pb : pa;
    auto issue = [&](int slot, int64_t step) {
      cp_async16(cell(slot, 0), psh + step * ss);
#pragma unroll
      for (int q = 0; q < Q; ++q) cp_async16(cell(slot, 1 + q), pv + step * sv + q * vq * s);
    };
#pragma unroll
    for (int k = 0; k < kFoldRing; ++k) {
      if (k < count) issue(k, k);
      cp_async_commit();
    }
    double2 acc[Q];
    int slot = 0;
    for (int64_t c = 0; c < count; ++c) {
      cp_async_wait<kFoldRing - 1>();  // step c has landed
      const double2 y = *cell(slot, 0);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const double2 x = *cell(slot, 1 + q);
        const double2 pr = make_double2(dmul(x.x, y.x), dmul(x.y, y.y));
        acc[q] = c == 0 ? pr : make_double2(dadd(acc[q].x, pr.x), dadd(acc[q].y, pr.y));
      }
      const int64_t f = c + kFoldRing;  // refill this slot with step c + ring
      if (f < count) issue(slot, f);
      cp_async_commit();
      if (++slot == kFoldRing) slot = 0;
    }
    cp_async_wait<0>();
#pragma unroll
    for (int q = 0; q < Q; ++q)
      *reinterpret_cast<double2*>(OUT + (gb.out + q * oq) * s + j0) = acc[q];
  }
}

// BC = block columns (groups along ib): 16 (512 threads) or 8 (256 threads,
// more and smaller work units when the 16 x 16 grid would leave SMs idle).
// COLTREE: the reduction is over the first dim with t = 16 (s = 16 * stride):
// a 64-slot unit is then 16 rows x 4 consecutive columns (row = in-tile index
// of the summed dim), each warp holds 16 rows x 2 columns (lane = row*2 + c),
// i.e. complete cyclic columns, and the power-of-two tree runs as 4 shuffle
// levels (partner lane (l + 2e) mod 32 == row (r + e) mod 16) before the
// final store -- no separate tree pass, no round trip of the folded tile.
// SLOTS = slots per work unit: 64 (512 threads, 1 CTA/SM) or 32 (256 threads,
// 2 CTAs/SM, so one CTA computes while the other waits at its barrier).
template <int BC, bool COLTREE, int SLOTS = kGemmSlots>
__global__ void __launch_bounds__((SLOTS / 32) * (kGemmBlk / kGemmSubR) * (BC / kGemmSubC) * 32,
                                  (SLOTS == 32 && BC == 8) ? 4 : (SLOTS == 32 || BC == 8) ? 2 : 1)
    fold_gemm_kernel(const __grid_constant__ FoldParams p, const __grid_constant__ BlockSpec bs,
                     const double* __restrict__ A, const double* __restrict__ B,
                     double* __restrict__ OUT) {
  pdl_enter(p.late != 0);
  constexpr int kHalves = SLOTS / 32;
  constexpr int kThreads = kHalves * (kGemmBlk / kGemmSubR) * (BC / kGemmSubC) * 32;
  constexpr int kSubCols = BC / kGemmSubC;
  constexpr int kSegs = SLOTS / 2;  // 16-byte segments per operand row
  constexpr int kStep = kGemmBlk * SLOTS + BC * SLOTS;  // doubles per fold step
  extern __shared__ __align__(16) double gsm[];
  // ring of kGemmStages super-stages, each holding kGemmPair fold steps
  const int64_t s = p.s;
  const int64_t first = p.first;
  const int64_t count = p.count;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int slot = (warp % kHalves) * 32 + lane;  // slot within the unit
  const int sub = warp / kHalves;                 // 8x4 sub-block of the 16 x BC groups
  const int r0 = (sub / kSubCols) * kGemmSubR, c0 = (sub % kSubCols) * kGemmSubC;
  for (uint64_t u = blockIdx.x; u < static_cast<uint64_t>(bs.units); u += gridDim.x) {
    uint64_t t = u;
    const uint64_t t1 = fdiv(t, bs.div_nbq);
    const int64_t qb = static_cast<int64_t>(t - t1 * bs.div_nbq.d);
    const uint64_t t2 = fdiv(t1, bs.div_nbp);
    const int64_t pb = static_cast<int64_t>(t1 - t2 * bs.div_nbp.d);
    const uint64_t rest = fdiv(t2, bs.div_chunks);
    const int64_t chunk = static_cast<int64_t>(t2 - rest * bs.div_chunks.d);
    const GroupBase gb = group_base(p, rest);
    const int np = static_cast<int>(bs.ext_ia - pb * kGemmBlk < kGemmBlk ? bs.ext_ia - pb * kGemmBlk : kGemmBlk);
    const int nq = static_cast<int>(bs.ext_ib - qb * BC < BC ? bs.ext_ib - qb * BC : BC);
    const int64_t stride = COLTREE ? s / 16 : 0;
    constexpr int kCols = SLOTS / 16;  // COLTREE: columns per unit (16 rows each)
    const int64_t j0 = COLTREE ? chunk * kCols : chunk * SLOTS;
    const double* a0 = A + (gb.a + pb * kGemmBlk * bs.a_ia + first * p.g.astep) * s + j0;
    const double* b0 = B + (gb.b + qb * BC * bs.b_ib + first * p.g.bstep) * s + j0;
    // global offset (from j0) of the 16-byte segment `seg` of a 64-slot unit
    auto seg_off = [&](int seg) -> int64_t {
      if (COLTREE) return static_cast<int64_t>(seg / kHalves) * stride + (seg % kHalves) * 2;  // row, half
      return seg * 2;
    };
    // shared-memory position of segment `seg` (slot index = half*32 + row*2 + c)
    auto seg_pos = [&](int seg) -> int {
      if (COLTREE) return (seg % kHalves) * 32 + (seg / kHalves) * 2;
      return seg * 2;
    };
    const int64_t a_row = bs.a_ia * s, b_col = bs.b_ib * s;
    const int64_t sa = p.g.astep * s, sb = p.g.bstep * s;

    // per-thread staging plan, invariant across fold steps: which 16-byte
    // segments this thread copies (source pointer at step 0, smem offset)
    constexpr int kCopiesA = (kGemmBlk * kSegs + kThreads - 1) / kThreads;
    constexpr int kCopiesB = (BC * kSegs + kThreads - 1) / kThreads;
    const double* srcA[kCopiesA];
    const double* srcB[kCopiesB];
    int dstA[kCopiesA], dstB[kCopiesB];
#pragma unroll
    for (int q = 0; q < kCopiesA; ++q) {
      const int e = tid + q * kThreads;
      const int row = e / kSegs, seg = e % kSegs;
      const int ra = row < np ? row : np - 1;
      srcA[q] = e < kGemmBlk * kSegs ? a0 + ra * a_row + seg_off(seg) : a0;  // unused when e is out
      dstA[q] = row * SLOTS + seg_pos(seg);
    }
#pragma unroll
    for (int q = 0; q < kCopiesB; ++q) {
      const int e = tid + q * kThreads;
      const int row = e / kSegs, seg = e % kSegs;
      const int rb = row < nq ? row : nq - 1;
      srcB[q] = e < BC * kSegs ? b0 + rb * b_col + seg_off(seg) : b0;
      dstB[q] = kGemmBlk * SLOTS + row * SLOTS + seg_pos(seg);
    }

    // fold steps are int32 (the host checks count < 2^31); ring offsets in
    // doubles advance by one super-stage and wrap without a division
    const int cnt = static_cast<int>(count);
    const int nsup = (cnt + kGemmPair - 1) / kGemmPair;
    constexpr int kSuper = kGemmPair * kStep;
    constexpr int kRing = kGemmStages * kSuper;
    // staging pointers advance by one super-stage per call (no 64-bit
    // multiplies in the loop); step h of a super-stage is h * sa further on
    auto stage = [&](int off, int c_first) {
#pragma unroll
      for (int h = 0; h < kGemmPair; ++h) {
        if (c_first + h < cnt) {
          double* st = gsm + off + h * kStep;
#pragma unroll
          for (int q = 0; q < kCopiesA; ++q)
            if (kGemmBlk * kSegs % kThreads == 0 || tid + q * kThreads < kGemmBlk * kSegs)
              cp_async16(st + dstA[q], srcA[q] + h * sa);
#pragma unroll
          for (int q = 0; q < kCopiesB; ++q)
            if (BC * kSegs % kThreads == 0 || tid + q * kThreads < BC * kSegs)
              cp_async16(st + dstB[q], srcB[q] + h * sb);
        }
      }
      cp_async_commit();
#pragma unroll
      for (int q = 0; q < kCopiesA; ++q) srcA[q] += kGemmPair * sa;
#pragma unroll
      for (int q = 0; q < kCopiesB; ++q) srcB[q] += kGemmPair * sb;
    };

    // -0.0 is the exact additive identity (-0 + x == x for every x, signed
    // zeros included), so starting the fold from it reproduces the
    // reference's "first product, then add" association bit for bit
    double acc[kGemmSubR][kGemmSubC];
#pragma unroll
    for (int i = 0; i < kGemmSubR; ++i)
#pragma unroll
      for (int k = 0; k < kGemmSubC; ++k) acc[i][k] = -0.0;
    auto fold_step = [&](const double* sA) {
      const double* sB = sA + kGemmBlk * SLOTS;
      double a[kGemmSubR], b[kGemmSubC];
#pragma unroll
      for (int i = 0; i < kGemmSubR; ++i) a[i] = sA[(r0 + i) * SLOTS + slot];
#pragma unroll
      for (int k = 0; k < kGemmSubC; ++k) b[k] = sB[(c0 + k) * SLOTS + slot];
      // products of two rows first, then their additions: 8 independent
      // DMULs in flight before the dependent DADDs (fixed-latency hiding)
#pragma unroll
      for (int i = 0; i < kGemmSubR; i += 2) {
        double pr[2][kGemmSubC];
#pragma unroll
        for (int k = 0; k < kGemmSubC; ++k) {
          pr[0][k] = dmul(a[i], b[k]);
          pr[1][k] = dmul(a[i + 1], b[k]);
        }
#pragma unroll
        for (int k = 0; k < kGemmSubC; ++k) {
          acc[i][k] = dadd(acc[i][k], pr[0][k]);
          acc[i + 1][k] = dadd(acc[i + 1][k], pr[1][k]);
        }
      }
    };
#pragma unroll
    for (int k = 0; k < kGemmStages - 1; ++k) {
      if (k < nsup)
        stage(k * kSuper, k * kGemmPair);
      else
        cp_async_commit();
    }
    int rd = 0, wr = (kGemmStages - 1) * kSuper;
    for (int sup = 0; sup < nsup; ++sup) {
      cp_async_wait<kGemmStages - 2>();  // super-stage `sup` has landed
      __syncthreads();                   // ...for every thread; the previous buffer is free
      if (sup + kGemmStages - 1 < nsup)
        stage(wr, (sup + kGemmStages - 1) * kGemmPair);
      else
        cp_async_commit();
      wr = wr + kSuper == kRing ? 0 : wr + kSuper;
      const double* sbuf = gsm + rd;
      if ((sup + 1) * kGemmPair <= cnt) {
#pragma unroll
        for (int h = 0; h < kGemmPair; ++h) fold_step(sbuf + h * kStep);
      } else {
        for (int h = 0; h < cnt - sup * kGemmPair; ++h) fold_step(sbuf + h * kStep);
      }
      rd = rd + kSuper == kRing ? 0 : rd + kSuper;
    }
    cp_async_wait<0>();
    __syncthreads();  // the ring is reused by the next unit
    if (COLTREE) {
      for (int lv = 0; lv < p.nlevels; ++lv) {  // e = 1, 2, 4, 8 rows
        const int src = (lane + (2 << lv)) & 31;
#pragma unroll
        for (int i = 0; i < kGemmSubR; ++i)
#pragma unroll
          for (int k = 0; k < kGemmSubC; ++k)
            acc[i][k] = dadd(acc[i][k], __shfl_sync(0xffffffffu, acc[i][k], src));
      }
    }
    const int64_t j = COLTREE ? j0 + static_cast<int64_t>(lane >> 1) * stride + (warp % kHalves) * 2 + (lane & 1)
                              : j0 + slot;
    if (j < s) {
      // row pointers by increment, column offsets once: one 64-bit add per store
      double* orow = OUT + (gb.out + (pb * kGemmBlk + r0) * bs.out_ia + (qb * BC + c0) * bs.out_ib) * s + j;
      const int64_t rstep = bs.out_ia * s, cstep = bs.out_ib * s;
      int64_t coff[kGemmSubC];
#pragma unroll
      for (int k = 0; k < kGemmSubC; ++k) coff[k] = k * cstep;
#pragma unroll
      for (int i = 0; i < kGemmSubR; ++i) {
        if (r0 + i < np) {
#pragma unroll
          for (int k = 0; k < kGemmSubC; ++k)
            if (c0 + k < nq) orow[coff[k]] = acc[i][k];
        }
        orow += rstep;
      }
    }
  }
}

// TMA-fed GEMM fold (the default for matmul-shaped products).  Same work
// unit as fold_gemm_kernel -- a 16 x BC block of groups for 32 consecutive
// slots -- but the operands arrive by tensor-map TMA: per stage, ONE 5-D box
// load brings the block's A chunks ([kTgSteps fold steps][16 rows][32 slots])
// and one the B chunks, both completing on the stage's mbarrier.  Lane 0 of
// warp 0 issues them kTgStages-1 stages ahead, running on into the CTA's next
// unit while the warps store the previous one, so no thread spends an
// instruction on staging addresses.  There is no separate producer warp: with
// ~200 registers per thread, 4-warp CTAs let two CTAs (2 warps per SM
// sub-partition) share an SM, where a 5-warp CTA would fit only once.  Each
// warp owns an 8 x 8 sub-block of the groups (16 shared-memory loads per 128
// FP64 operations).  Tensor dims (innermost first): slot, block row, fold
// step, up to two remaining group dims.  Out-of-range rows and steps are
// zero-filled by the TMA unit: rows are never stored, steps never folded.
// kTgSteps = fold steps per stage, kTgStages = ring stages (kTgStages - 1
// loads in flight ahead), SC = columns of a thread's 8 x SC sub-block of groups

struct TgSpec {
  int small;                 // units < 2^31: decode with the 32-bit divisors below
  FastDiv32 dq, dp, dc;      // nbq, nbp, chunks
  int nrest;
  int chunk_major;  // unit order: chunk fastest (consecutive CTAs read adjacent slots)
  int a_act[2], b_act[2];  // remaining group dim i is a tensor-map dim of A / B
};

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(smem_u32(bar))
      : "memory");
}

// SL = slots per unit: 32 (one slot per lane) or 16 (the two half-warps take
// different 8-column halves of the block: twice the units, for wave balance)
template <int BC, int SL, int SC, int PB = kGemmBlk>
__host__ __device__ constexpr int tg_warps() {
  return (PB / 8) * (BC / SC) * SL / 32;
}
template <int BC, int SL, int kTgSteps, int kTgStages, int PB = kGemmBlk>
__host__ __device__ constexpr size_t tg_smem_bytes() {
  return static_cast<size_t>(kTgStages) * kTgSteps * (PB + BC) * SL * sizeof(double) +
         3 * kTgStages * sizeof(uint64_t);
}

struct TgUnit {
  int64_t qb, pb, chunk;
  uint64_t rest;
};
__device__ __forceinline__ TgUnit tg_decode(const BlockSpec& bs, uint64_t u, int chunk_major) {
  TgUnit t;
  if (chunk_major) {
    const uint64_t t1 = fdiv(u, bs.div_chunks);
    t.chunk = static_cast<int64_t>(u - t1 * bs.div_chunks.d);
    const uint64_t t2 = fdiv(t1, bs.div_nbq);
    t.qb = static_cast<int64_t>(t1 - t2 * bs.div_nbq.d);
    t.rest = fdiv(t2, bs.div_nbp);
    t.pb = static_cast<int64_t>(t2 - t.rest * bs.div_nbp.d);
    return t;
  }
  const uint64_t t1 = fdiv(u, bs.div_nbq);
  t.qb = static_cast<int64_t>(u - t1 * bs.div_nbq.d);
  const uint64_t t2 = fdiv(t1, bs.div_nbp);
  t.pb = static_cast<int64_t>(t1 - t2 * bs.div_nbp.d);
  t.rest = fdiv(t2, bs.div_chunks);
  t.chunk = static_cast<int64_t>(t2 - t.rest * bs.div_chunks.d);
  return t;
}

// 32-bit unit decode (qb fastest, then pb, chunk, rest), for units < 2^31
__device__ __forceinline__ TgUnit tg_decode32(const TgSpec& ts, uint32_t u) {
  TgUnit t;
  const uint32_t t1 = fdiv(u, ts.dq);
  t.qb = u - t1 * ts.dq.d;
  const uint32_t t2 = fdiv(t1, ts.dp);
  t.pb = t1 - t2 * ts.dp.d;
  const uint32_t rest = fdiv(t2, ts.dc);
  t.chunk = t2 - rest * ts.dc.d;
  t.rest = rest;
  return t;
}

template <int BC, int SL, int kTgSteps, int kTgStages, int SC, int PB = kGemmBlk>
__global__ void __maxnreg__(SC == 8 ? 232 : 128)
    fold_gemm_tma_kernel(const __grid_constant__ CUtensorMap mapA,
                         const __grid_constant__ CUtensorMap mapB,
                         const __grid_constant__ FoldParams p, const __grid_constant__ BlockSpec bs,
                         const __grid_constant__ TgSpec ts, double* __restrict__ OUT,
                         unsigned int* __restrict__ sched) {
  pdl_enter(p.late != 0);
  constexpr int kW = tg_warps<BC, SL, SC, PB>();
  constexpr int kTgRows = 8 / SC;  // rows of products batched before their adds
  constexpr int kA = kTgSteps * PB * SL;  // doubles per stage
  constexpr int kB = kTgSteps * BC * SL;
  constexpr int kStage = kA + kB;
  extern __shared__ __align__(1024) double tsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + kTgStages * kStage);
  uint64_t* empty = full + kTgStages;
  uint64_t* stage_unit = empty + kTgStages;  // unit loaded into each stage (~0: no more)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool issuer = threadIdx.x == 0;
  if (issuer) {
    for (int i = 0; i < kTgStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t s = p.s;
  const int cnt = static_cast<int>(p.count);
  const int nst = (cnt + kTgSteps - 1) / kTgSteps;  // stages per unit
  const uint64_t units = static_cast<uint64_t>(bs.units);

  // load sequence of this CTA (issuer only): unit lu, stage k of that unit.
  // The first unit is blockIdx.x; later ones come from the launch's work
  // queue (sched[0], so SMs that run ahead take more units) or, without one,
  // statically every gridDim.x.  When none is left the issuer publishes a
  // ~0 unit on the next stage, which ends every warp's loop.
  uint64_t lu = blockIdx.x;
  int lk = 0, lstage = 0;
  uint32_t lphase = 0;
  bool ended = false;
  int rc[2] = {0, 0};
  TgUnit lt{};
  auto load_unit = [&]() {
    lt = (ts.small && !ts.chunk_major) ? tg_decode32(ts, static_cast<uint32_t>(lu))
                                       : tg_decode(bs, lu, ts.chunk_major);
    uint64_t v = lt.rest;
#pragma unroll
    for (int i = 1; i >= 0; --i) {
      if (i < ts.nrest) {
        const uint64_t q = fdiv(v, p.gdiv[i]);
        rc[i] = static_cast<int>(v - q * p.gdiv[i].d);
        v = q;
      }
    }
  };
  auto issue_next = [&]() {
    if (lu >= units) {
      if (ended) return;
      mbar_wait(&empty[lstage], lphase ^ 1);
      stage_unit[lstage] = ~uint64_t{0};
      mbar_arrive(&full[lstage]);
      ended = true;
      return;
    }
    mbar_wait(&empty[lstage], lphase ^ 1);  // every warp has released this buffer
    stage_unit[lstage] = lu;
    mbar_arrive_expect_tx(&full[lstage], kStage * sizeof(double));
    double* st = tsm + lstage * kStage;
    const int j0 = static_cast<int>(lt.chunk * SL);
    tma_load_5d(st, &mapA, j0, static_cast<int>(lt.pb * PB), lk * kTgSteps,
                ts.a_act[0] ? rc[0] : 0, ts.a_act[1] ? rc[1] : 0, &full[lstage]);
    tma_load_5d(st + kA, &mapB, j0, static_cast<int>(lt.qb * BC), lk * kTgSteps,
                ts.b_act[0] ? rc[0] : 0, ts.b_act[1] ? rc[1] : 0, &full[lstage]);
    if (++lstage == kTgStages) {
      lstage = 0;
      lphase ^= 1;
    }
    if (++lk == nst) {
      lk = 0;
      lu = sched ? gridDim.x + atomicAdd(&sched[0], 1u) : lu + gridDim.x;
      if (lu < units) load_unit();
    }
  };
  if (issuer) {
    if (lu < units) load_unit();
    for (int i = 0; i < kTgStages - 1; ++i) issue_next();
  }

  const int sub = warp * (32 / SL) + lane / SL, slot = lane % SL;
  const int r0 = (sub / (BC / SC)) * 8, c0 = (sub % (BC / SC)) * SC;
  // launch-constant output strides, hoisted out of the unit loop; the fold
  // output is re-read at once by the tree pass: keep it in L2
  const int64_t rstep = bs.out_ia * s;
  int64_t coff[SC];
#pragma unroll
  for (int k = 0; k < SC; ++k) coff[k] = k * bs.out_ib * s;
  const uint64_t keep = policy_evict_last();
  int stage = 0;
  uint32_t phase = 0;
  for (;;) {
    if (issuer) issue_next();  // refills the buffer released one stage ago
    __syncwarp();
    mbar_wait(&full[stage], phase);
    const uint64_t u = stage_unit[stage];
    if (u == ~uint64_t{0}) break;
    const TgUnit t = (ts.small && !ts.chunk_major) ? tg_decode32(ts, static_cast<uint32_t>(u))
                                                   : tg_decode(bs, u, ts.chunk_major);
    double acc[8][SC];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int k = 0; k < SC; ++k) acc[i][k] = -0.0;  // exact identity: -0 + x == x
    auto fold_step = [&](const double* sA, const double* sB) {
      double a[8], b[SC];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = sA[i * SL];
#pragma unroll
      for (int k = 0; k < SC; ++k) b[k] = sB[k * SL];
      // per kTgRows rows: 8 * kTgRows independent products, then their additions
#pragma unroll
      for (int i = 0; i < 8; i += kTgRows) {
        double pr[kTgRows][SC];
#pragma unroll
        for (int r = 0; r < kTgRows; ++r)
#pragma unroll
          for (int k = 0; k < SC; ++k) pr[r][k] = dmul(a[i + r], b[k]);
#pragma unroll
        for (int r = 0; r < kTgRows; ++r)
#pragma unroll
          for (int k = 0; k < SC; ++k) acc[i + r][k] = dadd(acc[i + r][k], pr[r][k]);
      }
    };
    for (int k = 0; k < nst; ++k) {
      if (k > 0) {
        if (issuer) issue_next();
        __syncwarp();
        mbar_wait(&full[stage], phase);
      }
      const double* sA = tsm + stage * kStage + r0 * SL + slot;
      const double* sB = tsm + stage * kStage + kA + c0 * SL + slot;
      const int nsteps = cnt - k * kTgSteps;
      if (nsteps >= kTgSteps) {
#pragma unroll
        for (int h = 0; h < kTgSteps; ++h) fold_step(sA + h * PB * SL, sB + h * BC * SL);
      } else {
        for (int h = 0; h < nsteps; ++h) fold_step(sA + h * PB * SL, sB + h * BC * SL);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kTgStages) {
        stage = 0;
        phase ^= 1;
      }
    }
    const int64_t gout = ts.nrest ? group_base(p, t.rest).out : 0;
    const int np = static_cast<int>(bs.ext_ia - t.pb * PB < PB ? bs.ext_ia - t.pb * PB : PB);
    const int nq = static_cast<int>(bs.ext_ib - t.qb * BC < BC ? bs.ext_ib - t.qb * BC : BC);
    double* orow = OUT + (gout + (t.pb * PB + r0) * bs.out_ia + (t.qb * BC + c0) * bs.out_ib) * s +
                   t.chunk * SL + slot;
    if (np == PB && nq == BC) {  // interior block: no bounds tests
#pragma unroll
      for (int i = 0; i < 8; ++i) {
#pragma unroll
        for (int k = 0; k < SC; ++k) st_keep(orow + coff[k], acc[i][k], keep);
        orow += rstep;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (r0 + i < np) {
#pragma unroll
          for (int k = 0; k < SC; ++k)
            if (c0 + k < nq) st_keep(orow + coff[k], acc[i][k], keep);
        }
        orow += rstep;
      }
    }
  }
  // the last CTA to finish leaves the queue counters at zero for the next launch
  if (issuer && sched) {
    __threadfence();
    if (atomicAdd(&sched[1], 1u) == gridDim.x - 1) {
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
    }
  }
}

// Warp-specialised variant of fold_gemm_tma_kernel: the same units, tensor-map
// boxes, ring layout and epilogue, but the TMA issue runs on its own producer
// warp (warp kW, one elected lane) instead of on consumer warp 0's lane 0.
// The producer alone waits for a ring buffer to be released (empty barrier);
// consumer warps only wait for data (full barrier), so no consumer is held
// back to the slowest one at every stage.  Measured with the operands already
// in shared memory (tools/micro/gemm_loop.cu) the consumer loop itself runs the
// FP64 pipe at 92%; the ring machinery is what this variant trims.
template <int BC, int SL, int kTgSteps, int kTgStages, int SC, int PB = kGemmBlk>
__global__ void __launch_bounds__((tg_warps<BC, SL, SC, PB>() + 1) * 32, 3)
    fold_gemm_ws_kernel(const __grid_constant__ CUtensorMap mapA,
                        const __grid_constant__ CUtensorMap mapB,
                        const __grid_constant__ FoldParams p, const __grid_constant__ BlockSpec bs,
                        const __grid_constant__ TgSpec ts, double* __restrict__ OUT,
                        unsigned int* __restrict__ sched, int wait_mode) {
  pdl_enter(p.late != 0);
  // wait_mode (TT_GEMM_WAIT): 0 = every mbarrier waiter spins on try_wait,
  // 1 = the producer sleeps on try_wait's suspend hint, 2 = every waiter does
  constexpr int kW = tg_warps<BC, SL, SC, PB>();  // consumer warps
  constexpr int kA = kTgSteps * PB * SL;           // doubles per stage
  constexpr int kB = kTgSteps * BC * SL;
  constexpr int kStage = kA + kB;
  extern __shared__ __align__(1024) double tsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + kTgStages * kStage);
  uint64_t* empty = full + kTgStages;
  uint64_t* stage_unit = empty + kTgStages;  // unit loaded into each stage (~0: no more)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kTgStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t s = p.s;
  const int cnt = static_cast<int>(p.count);
  const int nst = (cnt + kTgSteps - 1) / kTgSteps;  // stages per unit
  const uint64_t units = static_cast<uint64_t>(bs.units);

  if (warp == kW) {  // ---- producer ----
    if (lane != 0) return;
    uint64_t lu = blockIdx.x;
    int lk = 0, lstage = 0;
    uint32_t lphase = 0;
    int rc[2] = {0, 0};
    TgUnit lt{};
    auto load_unit = [&]() {
      lt = (ts.small && !ts.chunk_major) ? tg_decode32(ts, static_cast<uint32_t>(lu))
                                         : tg_decode(bs, lu, ts.chunk_major);
      uint64_t v = lt.rest;
#pragma unroll
      for (int i = 1; i >= 0; --i) {
        if (i < ts.nrest) {
          const uint64_t q = fdiv(v, p.gdiv[i]);
          rc[i] = static_cast<int>(v - q * p.gdiv[i].d);
          v = q;
        }
      }
    };
    if (lu < units) load_unit();
    for (;;) {
      // every consumer warp has released it (asleep meanwhile: a spinning
      // probe here took ~25% of the SM's issue slots)
      if (wait_mode >= 1)
        mbar_wait_sleep(&empty[lstage], lphase ^ 1);
      else
        mbar_wait(&empty[lstage], lphase ^ 1);
      if (lu >= units) {
        stage_unit[lstage] = ~uint64_t{0};
        mbar_arrive(&full[lstage]);
        break;
      }
      stage_unit[lstage] = lu;
      mbar_arrive_expect_tx(&full[lstage], kStage * sizeof(double));
      double* st = tsm + lstage * kStage;
      const int j0 = static_cast<int>(lt.chunk * SL);
      tma_load_5d(st, &mapA, j0, static_cast<int>(lt.pb * PB), lk * kTgSteps,
                  ts.a_act[0] ? rc[0] : 0, ts.a_act[1] ? rc[1] : 0, &full[lstage]);
      tma_load_5d(st + kA, &mapB, j0, static_cast<int>(lt.qb * BC), lk * kTgSteps,
                  ts.b_act[0] ? rc[0] : 0, ts.b_act[1] ? rc[1] : 0, &full[lstage]);
      if (++lstage == kTgStages) {
        lstage = 0;
        lphase ^= 1;
      }
      if (++lk == nst) {
        lk = 0;
        lu = sched ? gridDim.x + atomicAdd(&sched[0], 1u) : lu + gridDim.x;
        if (lu < units) load_unit();
      }
    }
    // the last CTA done taking units leaves the queue counters at zero
    if (sched) {
      __threadfence();
      if (atomicAdd(&sched[1], 1u) == gridDim.x - 1) {
        sched[0] = 0;
        sched[1] = 0;
        __threadfence();
      }
    }
    return;
  }

  // ---- consumers ----
  const int sub = warp * (32 / SL) + lane / SL, slot = lane % SL;
  const int r0 = (sub / (BC / SC)) * 8, c0 = (sub % (BC / SC)) * SC;
  const int64_t rstep = bs.out_ia * s;
  int64_t coff[SC];
#pragma unroll
  for (int k = 0; k < SC; ++k) coff[k] = k * bs.out_ib * s;
  const uint64_t keep = policy_evict_last();
  int stage = 0;
  uint32_t phase = 0;
  for (;;) {
    if (wait_mode >= 2)
      mbar_wait_sleep(&full[stage], phase);
    else
      mbar_wait(&full[stage], phase);
    const uint64_t u = stage_unit[stage];
    if (u == ~uint64_t{0}) break;
    const TgUnit t = (ts.small && !ts.chunk_major) ? tg_decode32(ts, static_cast<uint32_t>(u))
                                                   : tg_decode(bs, u, ts.chunk_major);
    const int np = static_cast<int>(bs.ext_ia - t.pb * PB < PB ? bs.ext_ia - t.pb * PB : PB);
    const int nq = static_cast<int>(bs.ext_ib - t.qb * BC < BC ? bs.ext_ib - t.qb * BC : BC);
    // a sub-block wholly outside a partial edge block folds nothing (its
    // rows / columns are TMA zero fill and never stored)
    const bool idle = r0 >= np || c0 >= nq;
    double acc[8][SC];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int k = 0; k < SC; ++k) acc[i][k] = -0.0;  // exact identity: -0 + x == x
    auto fold_step = [&](const double* sA, const double* sB) {
      double a[8], b[SC];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = sA[i * SL];
#pragma unroll
      for (int k = 0; k < SC; ++k) b[k] = sB[k * SL];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int k = 0; k < SC; ++k) acc[i][k] = dadd(acc[i][k], dmul(a[i], b[k]));
    };
    for (int k = 0; k < nst; ++k) {
      if (k > 0) {
        if (wait_mode >= 2)
          mbar_wait_sleep(&full[stage], phase);
        else
          mbar_wait(&full[stage], phase);
      }
      if (!idle) {
        const double* sA = tsm + stage * kStage + r0 * SL + slot;
        const double* sB = tsm + stage * kStage + kA + c0 * SL + slot;
        const int nsteps = cnt - k * kTgSteps;
        if (nsteps >= kTgSteps) {
#pragma unroll
          for (int h = 0; h < kTgSteps; ++h) fold_step(sA + h * PB * SL, sB + h * BC * SL);
        } else {
          for (int h = 0; h < nsteps; ++h) fold_step(sA + h * PB * SL, sB + h * BC * SL);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kTgStages) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (idle) continue;
    const int64_t gout = ts.nrest ? group_base(p, t.rest).out : 0;
    double* orow = OUT + (gout + (t.pb * PB + r0) * bs.out_ia + (t.qb * BC + c0) * bs.out_ib) * s +
                   t.chunk * SL + slot;
    if (np == PB && nq == BC) {  // interior block: no bounds tests
#pragma unroll
      for (int i = 0; i < 8; ++i) {
#pragma unroll
        for (int k = 0; k < SC; ++k) st_keep(orow + coff[k], acc[i][k], keep);
        orow += rstep;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (r0 + i < np) {
#pragma unroll
          for (int k = 0; k < SC; ++k)
            if (c0 + k < nq) st_keep(orow + coff[k], acc[i][k], keep);
        }
        orow += rstep;
      }
    }
  }
}

// kernels/chain.cuh -- the tile matmul (and a chain of two) as ONE persistent
// kernel: GEMM-shaped fold units and in-tile rotate-and-sum tree items pulled
// from a single dependency-ordered work queue.
// Included by tt_kernels.cu inside namespace ttb::{anonymous}.
//
// A product phase is  fold[i,j][h] = sum_k A[k,i][h] * B[k,j][h]  (the
// reference's left fold tile_tensor.hpp:313-330, k in order, product and sum
// separately rounded) followed by the power-of-two rotate-and-sum of the summed
// dim inside each output tile (rotate_sum.hpp:51-56).  For the matmul forms
// (linalg.hpp:41-73) that tree is either
//   * column-local (sum over the first tile dim, t * stride = s): slot
//     h = m * stride + r only meets slots of the same column r, or
//   * row-local (sum over an inner dim): slot h meets slots h .. h + reach,
//     reach < 512, i.e. its own 512-slot row block and the next one (cyclic).
// So tree work for a column block / row block can start as soon as the fold
// units that cover it are done, and -- in a chain where phase 2 multiplies
// by phase 1's result -- phase 2's fold units at slot chunk c can start as
// soon as phase 1's column block holding c is finished.  The queue orders
// the work so that dependencies are always earlier items; a CTA that takes an
// item whose inputs are not ready yet spins on a counter (every earlier item is
// held by a running CTA, so this cannot deadlock).  The fold units' tails are
// filled with tree items and with the next phase's units instead of idling,
// and the folded tiles never leave L2 between fold and tree.
//
// Work-unit shapes (as the stand-alone GEMM fold, gemm.cuh): a fold unit is a
// 16 x 16 block of output tiles x 16 slots; a producer warp streams its
// operands through a 4-stage mbarrier ring of TMA boxes {16 slots, 16 tiles,
// 4 fold steps}; 4 consumer warps, each thread an 8 x 4 sub-block of one slot.

constexpr int kChSL = 16;       // slots per fold unit
constexpr int kChP = 16;        // tiles per block side
constexpr int kChKS = 4;        // fold steps per ring stage
constexpr int kChNS = 4;        // ring stages
constexpr int kChCW = 4;        // consumer warps
constexpr int kChThreads = (kChCW + 1) * 32;
constexpr int kChStage = kChKS * 2 * kChP * kChSL;  // doubles per stage (A + B)
constexpr uint32_t kChEnd = 0xffffffffu;

enum : uint32_t { kChFold = 0, kChTree = 1 };

struct ChainPhaseDev {
  int ni, nj, nk;          // output-tile block extents (i: A varies, j: B varies), fold steps
  int nbi, nbj;            // 16-tile blocks along i / j
  int64_t out_i, out_j;    // output tile index = i * out_i + j * out_j
  double* fold;            // folded tiles (tree phases) -- or the result (no tree)
  double* out;             // result tiles
  int tree;                // 0 none, 1 column-local, 2 row-local
  int col_t, col_stride;   // column tree: T values per column, stride between them
  int nlevels, hr;         // row tree: levels (offsets in lv), halo rows of 32 slots
  int lv[8];
  // work queues: nf fold units in q groups of per_q chunks x nb blocks
  // (column-major: chunk = g + ncb * e; row-major: chunk = g * per_q + e) and
  // nt tree items in tq groups of nb x nsub
  int col_order, ncb, q, per_q;
  int colg;                // column-major: column blocks per super-group (order [g/colg][e][g%colg][block])
  int tq, tree_ncb, tree_per, nsub;
  int nf, nt;
  int fold_done, tree_done;  // counter offsets: fold_done[tree group][block], tree_done[tree group]
  int dep_phase;           // -1, or the phase whose column-tree output this one reads
  int dep_ncb, dep_target;
};

struct ChainDev {
  int nphase;
  int64_t s;
  int nchunks;             // s / 16
  unsigned int* cnt;       // [0..3] queue heads (F0, T0, F1, T1), [4] CTAs done, then dependency counters
  int ncnt;
  ChainPhaseDev ph[2];
};

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_until(const unsigned int* p, unsigned int target) {
  while (ld_acquire_u32(p) < target) __nanosleep(64);
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void consumer_bar() {  // the 4 consumer warps only
  asm volatile("bar.sync 1, %0;" ::"n"(kChCW * 32) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Decoded queue item.
struct ChItem {
  int kind;       // kChFold / kChTree
  int phase;
  int g;          // segment group (column block or row block)
  int chunk;      // fold: slot chunk
  int block;      // fold / tree: bi * nbj + bj
  int sub;        // tree: item within the block
};

// Queue item codes in the ring: kind (fold / tree) << 30 | phase << 29 | index.
__device__ __forceinline__ uint32_t ch_code(int kind, int phase, int idx) {
  return (static_cast<uint32_t>(kind) << 30) | (static_cast<uint32_t>(phase) << 29) | static_cast<uint32_t>(idx);
}

__device__ __forceinline__ ChItem chain_decode(const ChainDev& d, uint32_t code) {
  ChItem it{};
  it.kind = static_cast<int>(code >> 30);
  it.phase = static_cast<int>((code >> 29) & 1u);
  const int idx = static_cast<int>(code & ((1u << 29) - 1));
  const ChainPhaseDev& P = d.ph[it.phase];
  const int nb = P.nbi * P.nbj;
  if (it.kind == kChFold) {
    if (P.col_order) {
      const int G = P.colg;
      const int per_sg = G * P.per_q * nb;
      const int sg = idx / per_sg;
      int rr = idx - sg * per_sg;
      const int e = rr / (G * nb);
      rr -= e * G * nb;
      const int x = rr / nb;
      it.block = rr - x * nb;
      it.g = sg * G + x;
      it.chunk = it.g + P.ncb * e;
    } else {
      const int per_g = P.per_q * nb;
      it.g = idx / per_g;
      const int rr = idx - it.g * per_g;
      const int e = rr / nb;
      it.block = rr - e * nb;
      it.chunk = it.g * P.per_q + e;
    }
  } else {
    const int per_g = nb * P.nsub;
    it.g = idx / per_g;
    const int rr = idx - it.g * per_g;
    it.block = rr / P.nsub;
    it.sub = rr - it.block * P.nsub;
  }
  return it;
}

// Whether item `it`'s inputs are complete (acquire loads).
__device__ __forceinline__ bool ch_ready(const ChainDev& d, const ChItem& it) {
  const ChainPhaseDev& P = d.ph[it.phase];
  const unsigned int* cnt = d.cnt;
  if (it.kind == kChTree) {
    const int nb = P.nbi * P.nbj;
    if (ld_acquire_u32(&cnt[P.fold_done + it.g * nb + it.block]) < static_cast<unsigned>(P.tree_per))
      return false;
    return P.tree != 2 ||
           ld_acquire_u32(&cnt[P.fold_done + ((it.g + 1) % P.tq) * nb + it.block]) >= static_cast<unsigned>(P.tree_per);
  }
  if (P.dep_phase < 0) return true;
  return ld_acquire_u32(&cnt[d.ph[P.dep_phase].tree_done + it.chunk % P.dep_ncb]) >=
         static_cast<unsigned>(P.dep_target);
}

// Column tree of one column: T values at stride `stride`, the power-of-two
// levels v'[m] = v[m] + v[(m + e) mod T] in place (the first e values saved).
template <int T>
__device__ __forceinline__ void col_tree_column(const double* src, double* dst, int64_t stride) {
  double v[T];
#pragma unroll
  for (int m = 0; m < T; ++m) v[m] = __ldcg(src + m * stride);
#pragma unroll
  for (int e = 1; e < T; e *= 2) {
    double head[T / 2 > 0 ? T / 2 : 1];
#pragma unroll
    for (int m = 0; m < e; ++m) head[m] = v[m];
#pragma unroll
    for (int m = 0; m < T; ++m) v[m] = dadd(v[m], m + e < T ? v[m + e] : head[m + e - T]);
  }
#pragma unroll
  for (int m = 0; m < T; ++m) dst[m * stride] = v[m];
}

__global__ void __launch_bounds__(kChThreads, 3)
    chain_kernel(const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapB0,
                 const __grid_constant__ CUtensorMap mapA1, const __grid_constant__ CUtensorMap mapB1,
                 const __grid_constant__ ChainDev d) {
  extern __shared__ __align__(1024) double tsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + kChNS * kChStage);
  uint64_t* empty = full + kChNS;
  uint32_t* stage_item = reinterpret_cast<uint32_t*>(empty + kChNS);
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kChNS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kChCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t s = d.s;
  unsigned int* cnt = d.cnt;

  if (warp == kChCW) {  // ---- producer: one elected lane ----
    if (lane != 0) return;
    int st = 0;
    uint32_t ph = 0;
    // Queues (heads cnt[0..3]): F0, T0, F1, T1 (fold units / tree items of
    // phase 0 / 1).  Items are claimed with one atomicAdd (no CAS retries:
    // 444 producers racing on a CAS serialise to ~1 claim per microsecond).
    // A claimed item whose inputs are not complete yet is parked (one per
    // dependent queue) and the producer keeps claiming upstream work, which
    // never waits, so every parked item's inputs are eventually claimed and
    // done: no CTA idles while other work exists and none can deadlock.
    // Only complete items enter the ring, in the order they become ready.
    uint32_t park[4] = {kChEnd, kChEnd, kChEnd, kChEnd};
    bool done_q[4] = {false, false, false, false};
    const int nq = 2 * d.nphase;
    for (int q = nq; q < 4; ++q) done_q[q] = true;
    // One non-blocking scheduling step: a ready item's code, kChEnd when every
    // queue is exhausted and nothing is parked, kChEnd - 1 when only parked
    // (not yet ready) work remains.
    auto try_get = [&]() -> uint32_t {
      for (int q = 1; q < nq; ++q)  // parked items that became ready (critical path first)
        if (park[q] != kChEnd && ch_ready(d, chain_decode(d, park[q]))) {
          const uint32_t r = park[q];
          park[q] = kChEnd;
          return r;
        }
      bool waiting = false;
      for (int k = 0; k < nq; ++k) {  // claim: T0, F0, F1, T1 (one parked item per queue)
        const int q = k < 2 ? 1 - k : k;
        if (done_q[q]) continue;
        if (park[q] != kChEnd) {
          waiting = true;
          continue;
        }
        const ChainPhaseDev& Q = d.ph[q >> 1];
        const int n = (q & 1) ? Q.nt : Q.nf;
        const unsigned int i = atomicAdd(&cnt[q], 1u);
        if (i >= static_cast<unsigned>(n)) {
          done_q[q] = true;
          continue;
        }
        const uint32_t code = ch_code(q & 1, q >> 1, static_cast<int>(i));
        const bool needs = (q & 1) || Q.dep_phase >= 0;
        if (!needs || ch_ready(d, chain_decode(d, code))) return code;
        park[q] = code;
        waiting = true;
      }
      return waiting ? kChEnd - 1 : kChEnd;
    };
    auto get = [&]() -> uint32_t {  // blocking
      for (;;) {
        const uint32_t r = try_get();
        if (r != kChEnd - 1) return r;
        __nanosleep(128);
      }
    };
    for (;;) {
      const uint32_t u = get();
      if (u == kChEnd) {  // all work handed out
        mbar_wait_sleep(&empty[st], ph ^ 1);
        stage_item[st] = kChEnd;
        mbar_arrive(&full[st]);
        return;
      }
      const ChItem it = chain_decode(d, u);
      const ChainPhaseDev& P = d.ph[it.phase];
      if (it.kind == kChTree) {
        mbar_wait_sleep(&empty[st], ph ^ 1);
        stage_item[st] = u;
        mbar_arrive(&full[st]);
        if (++st == kChNS) {
          st = 0;
          ph ^= 1;
        }
        continue;
      }
      if (P.dep_phase >= 0) fence_proxy_async();  // operands written by other CTAs' trees
      const CUtensorMap* mA = it.phase ? &mapA1 : &mapA0;
      const CUtensorMap* mB = it.phase ? &mapB1 : &mapB0;
      const int bi = it.block / P.nbj, bj = it.block - (it.block / P.nbj) * P.nbj;
      const int nst = (P.nk + kChKS - 1) / kChKS;
      for (int k = 0; k < nst; ++k) {
        mbar_wait_sleep(&empty[st], ph ^ 1);
        stage_item[st] = u;
        mbar_arrive_expect_tx(&full[st], kChStage * sizeof(double));
        double* sp = tsm + st * kChStage;
        tma_load_3d(sp, mA, it.chunk * kChSL, bi * kChP, k * kChKS, &full[st]);
        tma_load_3d(sp + kChKS * kChP * kChSL, mB, it.chunk * kChSL, bj * kChP, k * kChKS, &full[st]);
        if (++st == kChNS) {
          st = 0;
          ph ^= 1;
        }
      }
    }
  }

  // ---- consumers ----
  const int tid = threadIdx.x;
  const int sub = warp * 2 + (lane >> 4), slot = lane & 15;  // 8 sub-blocks x 16 slots
  const int r0 = (sub >> 2) * 8, c0 = (sub & 3) * 4;
  const uint64_t keep = policy_evict_last();
  int st = 0;
  uint32_t ph = 0;
  for (;;) {
    mbar_wait(&full[st], ph);
    const uint32_t u = stage_item[st];
    if (u == kChEnd) break;
    const ChItem it = chain_decode(d, u);
    const ChainPhaseDev& P = d.ph[it.phase];
    const int bi = it.block / P.nbj, bj = it.block - (it.block / P.nbj) * P.nbj;
    if (it.kind == kChFold) {
      const int np = min(kChP, P.ni - bi * kChP), nq = min(kChP, P.nj - bj * kChP);
      const bool idle = r0 >= np || c0 >= nq;
      double acc[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[i][k] = -0.0;  // exact identity: -0 + x == x
      const int nst = (P.nk + kChKS - 1) / kChKS;
      for (int k = 0; k < nst; ++k) {
        if (k > 0) mbar_wait(&full[st], ph);
        if (!idle) {
          const double* sA = tsm + st * kChStage + r0 * kChSL + slot;
          const double* sB = tsm + st * kChStage + kChKS * kChP * kChSL + c0 * kChSL + slot;
          auto step = [&](int h) {
            double a[8], b[4];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = sA[h * kChP * kChSL + i * kChSL];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = sB[h * kChP * kChSL + j * kChSL];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[i][j] = dadd(acc[i][j], dmul(a[i], b[j]));
          };
          const int nsteps = P.nk - k * kChKS;
          if (nsteps >= kChKS) {
#pragma unroll
            for (int h = 0; h < kChKS; ++h) step(h);
          } else {
            for (int h = 0; h < nsteps; ++h) step(h);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++st == kChNS) {
          st = 0;
          ph ^= 1;
        }
      }
      if (!idle) {
        double* base = P.fold + ((bi * kChP + r0) * P.out_i + (bj * kChP + c0) * P.out_j) * s +
                       it.chunk * kChSL + slot;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (r0 + i < np) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (c0 + j < nq) st_keep(base + (i * P.out_i + j * P.out_j) * s, acc[i][j], keep);
          }
      }
      if (P.tree) {
        consumer_bar();  // every consumer's stores precede the release below
        if (tid == 0) {
          __threadfence();
          const int tg = P.tree == 1 ? it.chunk % P.tree_ncb : it.chunk / 32;  // 512-slot row blocks
          atomicAdd(&cnt[P.fold_done + tg * P.nbi * P.nbj + it.block], 1u);
        }
      }
      continue;
    }
    // ---- tree item: 16 output tiles (row `sub` of the block) ----
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);  // the stage carried no data
    if (++st == kChNS) {
      st = 0;
      ph ^= 1;
    }
    const int nb = P.nbi * P.nbj;
    if (tid == 0) {  // claimed ready: these acquire loads return at once
      spin_until(&cnt[P.fold_done + it.g * nb + it.block], P.tree_per);
      if (P.tree == 2) spin_until(&cnt[P.fold_done + ((it.g + 1) % P.tq) * nb + it.block], P.tree_per);
    }
    consumer_bar();
    const int i = bi * kChP + it.sub;  // the item's tiles: i fixed, j across the block
    if (i < P.ni) {
      const int nj = min(kChP, P.nj - bj * kChP);
      if (P.tree == 1) {
        // column trees: SL columns x nj tiles, two per thread
        const int col = tid & 15;
        for (int tj = tid >> 4; tj < nj; tj += 8) {
          const int64_t tile = i * P.out_i + (bj * kChP + tj) * P.out_j;
          const double* src = P.fold + tile * s + it.g * kChSL + col;
          double* dst = P.out + tile * s + it.g * kChSL + col;
          switch (P.col_t) {
            case 2: col_tree_column<2>(src, dst, P.col_stride); break;
            case 4: col_tree_column<4>(src, dst, P.col_stride); break;
            case 8: col_tree_column<8>(src, dst, P.col_stride); break;
            case 16: col_tree_column<16>(src, dst, P.col_stride); break;
            default: col_tree_column<32>(src, dst, P.col_stride); break;
          }
        }
      } else {
        // row trees: a warp finalises one tile's 16 rows of 32 slots (row block
        // g) with HR halo rows from the next block (cyclic), as row_tree_kernel
        const int rows = static_cast<int>(s / 32);
        for (int tj = warp; tj < nj; tj += kChCW) {
          const int64_t tile = i * P.out_i + (bj * kChP + tj) * P.out_j;
          const double* t = P.fold + tile * s;
          double* o = P.out + tile * s;
          const int rb = it.g * 16;
          double v[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            v[k] = 0.0;
            if (k < 16 + P.hr) {
              int row = rb + k;
              if (row >= rows) row -= rows;
              v[k] = __ldcg(t + row * 32 + lane);
            }
          }
          for (int k = 0; k < P.nlevels; ++k) {
            const int dd = P.lv[k];
            if (dd < 32) {
              const int srcl = (lane + dd) & 31;
              const bool same = lane + dd < 32;
              double cur = __shfl_sync(0xffffffffu, v[0], srcl);
#pragma unroll
              for (int q = 0; q < 32; ++q) {
                const double nxt = (q + 1 < 32) ? __shfl_sync(0xffffffffu, v[q + 1], srcl) : 0.0;
                v[q] = dadd(v[q], same ? cur : nxt);
                cur = nxt;
              }
            } else {
              switch (dd >> 5) {
                case 1: row_shift<32>(v, 1); break;
                case 2: row_shift<32>(v, 2); break;
                case 4: row_shift<32>(v, 4); break;
                case 8: row_shift<32>(v, 8); break;
                case 16: row_shift<32>(v, 16); break;
                default: break;
              }
            }
          }
#pragma unroll
          for (int k = 0; k < 16; ++k) o[(rb + k) * 32 + lane] = v[k];
        }
      }
    }
    if (P.tree == 1) {  // the next phase's producers read this output through TMA
      consumer_bar();
      if (tid == 0) {
        fence_proxy_async();
        __threadfence();
        atomicAdd(&cnt[P.tree_done + it.g], 1u);
      }
    }
  }
  // ---- exit: the last CTA leaves every counter at zero for the next launch ----
  consumer_bar();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(&cnt[4], 1u) == gridDim.x - 1;
  }
  consumer_bar();
  if (s_last) {
    __threadfence();
    for (int k = tid; k < d.ncnt; k += kChCW * 32) cnt[k] = 0;
  }
}

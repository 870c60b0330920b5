// kernels/tree.cuh -- tree-only passes (phase 2 of a split reduction): column, row-shift, shared-memory.
// Included by tt_kernels.cu inside namespace ttb::{anonymous}: one
// translation unit, so the kernels share its device helpers (FastDiv,
// dadd / dmul, mbarrier and TMA wrappers) without external linkage.
#pragma once

// ---- tree-only passes (phase 2 of a two-phase reduction), in place on OUT ----------------
// (A) column-local: the summed dim is the first (s == t * stride), so each
// column c of the tile viewed as [t][stride] is one cyclic sequence of t
// values; a thread loads its column, runs the power-of-two levels in
// registers (v'[m] = v[m] + v[(m + e) mod t]), stores it back.  Coalesced
// across threads (consecutive columns), no shared memory, no barrier.
// BACK: rotations by -e*stride (replicate_tile_dim's right-to-left schedule):
// the column is read mirrored (m -> T-1-m), which turns them into the forward
// levels below with the same operand order.  `in` may equal `out`.
// EPI: the reduction's elementwise tail (+ C, square) applied before the store.
template <int T, bool BACK = false, bool EPI = false>
__global__ void __launch_bounds__(256) col_tree_kernel(const double* in, double* out, int64_t n_tiles,
                                                       int64_t stride, int64_t s, FastDiv64 cdiv,
                                                       const __grid_constant__ EpiDev epi) {
  pdl_enter();
  const uint64_t total = static_cast<uint64_t>(n_tiles) * stride;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t tile = fdiv(w, cdiv);
    const int64_t col = static_cast<int64_t>(w - tile * cdiv.d);
    const double* src = in + tile * s + col;
    double* base = out + tile * s + col;
    double v[T];
#pragma unroll
    for (int m = 0; m < T; ++m) v[m] = src[(BACK ? T - 1 - m : m) * stride];
#pragma unroll
    for (int e = 1; e < T; e *= 2) {
      double nv[T];
#pragma unroll
      for (int m = 0; m < T; ++m) nv[m] = dadd(v[m], v[(m + e) % T]);
#pragma unroll
      for (int m = 0; m < T; ++m) v[m] = nv[m];
    }
    if (EPI) epi_apply_n<T>(epi, v, epi_tile(epi, tile, s), col, stride);
#pragma unroll
    for (int m = 0; m < T; ++m) base[(BACK ? T - 1 - m : m) * stride] = v[m];
  }
}

// (B) row-shift: tile as rows of 32 slots; a warp finalises 16 rows and holds
// HR more rows of halo (reach <= HR*32 slots), read straight from L2/HBM
// (cyclic over the tile).  An offset d < 32 is a shuffle with carry into the
// next row; an offset 32*D is a register row shift.  Rows are updated in
// ascending order in place, so each update still reads the previous level's
// value of the rows below.  Valid rows shrink by the level's reach.
template <int NR>
__device__ __forceinline__ void row_shift(double (&v)[NR], int D) {
#pragma unroll
  for (int i = 0; i < NR; ++i)
    if (i + D < NR) v[i] = dadd(v[i], v[i + D]);
}

// Reads the folded tiles from `in` (scratch) and writes `out`: warps read
// halo rows owned by other warps, so the pass cannot run in place.
// BACK: the tile is read and written mirrored (slot p -> s-1-p), which turns
// rotations by -d (replicate schedules) into the forward offsets d handled here.
// EPI: the reduction's elementwise tail (+ C, square) applied before the store.
// C > 1: a warp takes a chain of C consecutive row blocks of one tile, last
// block first, and carries each block's raw (pre-tree) rows over as the halo of
// the block before it -- rows are read (C + HR/R) / C times instead of twice.
template <int HR, int R = 16, bool BACK = false, bool EPI = false, int C = 1>
__global__ void __launch_bounds__(256, (C == 1 && R + HR <= 20 ? 2 : HR <= 8 ? 3 : 2)) row_tree_kernel(const double* __restrict__ in,
                                                       double* __restrict__ out, int64_t n_tiles,
                                                       int64_t s, int nlevels, int4 lv0, int4 lv1,
                                                       const __grid_constant__ EpiDev epi) {
  pdl_enter();
  constexpr int NR = R + HR;
  // PF: the next block's rows are loaded before this block's levels run, so a
  // warp keeps its loads in flight while it computes (small halos only: the
  // second row set doubles the registers)
  constexpr bool PF = C == 1 && NR <= 20;
  static_assert(C == 1 || HR <= R, "the carried halo comes from one block");
  const int lane = threadIdx.x & 31;
  const int rows = static_cast<int>(s / 32);
  const int chains_per_tile = rows / R / C;
  const uint64_t total = static_cast<uint64_t>(n_tiles) * chains_per_tile;
  const int lvl[8] = {lv0.x, lv0.y, lv0.z, lv0.w, lv1.x, lv1.y, lv1.z, lv1.w};
  const uint64_t gstride = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  // rows [block, block + NR) of unit u (cyclic over its tile), mirrored when BACK
  auto load_rows = [&](uint64_t u, double (&dst)[NR]) {
    const uint64_t tile = u / chains_per_tile;
    const int rb = static_cast<int>(u - tile * chains_per_tile) * R;
    const double* t = in + tile * s;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      int row = rb + i;
      if (row >= rows) row -= rows;
      const int64_t p = row * 32 + lane;
      dst[i] = __ldg(t + (BACK ? s - 1 - p : p));
    }
  };
  double pre[PF ? NR : 1];
  uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
  if constexpr (PF) {
    if (u < total) load_rows(u, pre);
  }
  for (; u < total; u += gstride) {
    const uint64_t tile = u / chains_per_tile;
    const int b0 = static_cast<int>(u - tile * chains_per_tile) * C;
    const double* t = in + tile * s;
    double* o = out + tile * s;
    double halo[HR];  // raw rows following the current block (cyclic over the tile)
    if constexpr (!PF) {
#pragma unroll
      for (int i = 0; i < HR; ++i) {
        int row = (b0 + C) * R + i;
        if (row >= rows) row -= rows;
        const int64_t p = row * 32 + lane;
        halo[i] = __ldg(t + (BACK ? s - 1 - p : p));
      }
    }
#pragma unroll 1
    for (int kk = C - 1; kk >= 0; --kk) {
    const int rb = (b0 + kk) * R;
    double v[NR];
    if constexpr (PF) {
#pragma unroll
      for (int i = 0; i < NR; ++i) v[i] = pre[i];
      if (u + gstride < total) load_rows(u + gstride, pre);
    } else {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int64_t p = (rb + i) * 32 + lane;
        v[i] = __ldg(t + (BACK ? s - 1 - p : p));
      }
#pragma unroll
      for (int i = 0; i < HR; ++i) v[R + i] = halo[i];
      if (C > 1) {
#pragma unroll
        for (int i = 0; i < HR; ++i) halo[i] = v[i < R ? i : 0];
      }
    }
    for (int k = 0; k < nlevels; ++k) {
      const int d = lvl[k];
      if (d < 32) {
        const int src = (lane + d) & 31;
        const bool same = lane + d < 32;
        double cur = __shfl_sync(0xffffffffu, v[0], src);
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          const double nxt = (i + 1 < NR) ? __shfl_sync(0xffffffffu, v[i + 1], src) : 0.0;
          v[i] = dadd(v[i], same ? cur : nxt);
          cur = nxt;
        }
      } else {
        switch (d >> 5) {
          case 1: row_shift<NR>(v, 1); break;
          case 2: row_shift<NR>(v, 2); break;
          case 4: row_shift<NR>(v, 4); break;
          case 8: row_shift<NR>(v, 8); break;
          case 16: row_shift<NR>(v, 16); break;
          default: break;  // excluded by the host eligibility check
        }
      }
    }
    if (EPI) {
      double w[R];
#pragma unroll
      for (int i = 0; i < R; ++i) w[i] = v[i];
      epi_apply_n<R>(epi, w, epi_tile(epi, tile, s), rb * 32 + lane, 32);
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = w[i];
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int64_t p = (rb + i) * 32 + lane;
      o[BACK ? s - 1 - p : p] = v[i];
    }
    }
  }
}

// (C) whole tile in shared memory: a CTA of s / PER threads holds one tile
// in registers (thread t owns slots t + i * T), and each power-of-two level
// v'[j] = v[j] + v[(j + r) mod s] exchanges through shared memory (store,
// barrier, load the partner, barrier).  Any rotations, one global read and
// one global write per slot, in place.  Several CTAs per SM overlap one
// tile's loads with another's levels.
__device__ __forceinline__ int level_rot(int k, const int4& a, const int4& b) {
  switch (k) {
    case 0: return a.x;
    case 1: return a.y;
    case 2: return a.z;
    case 3: return a.w;
    case 4: return b.x;
    case 5: return b.y;
    case 6: return b.z;
    default: return b.w;
  }
}

constexpr int kTreeThreads = 256;
template <int PER>
__global__ void __launch_bounds__(kTreeThreads, 2) smem_tree_kernel(double* __restrict__ tiles,
                                                                    int64_t n_tiles, int nlevels,
                                                                    int4 lv0, int4 lv1) {
  pdl_enter();
  extern __shared__ double tsh[];
  constexpr int T = kTreeThreads, s = T * PER;
  const int tid = threadIdx.x;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    double* t = tiles + tile * s;
    double v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) v[i] = t[tid + i * T];
    for (int k = 0; k < nlevels; ++k) {
      const int r = level_rot(k, lv0, lv1);
#pragma unroll
      for (int i = 0; i < PER; ++i) tsh[tid + i * T] = v[i];
      __syncthreads();
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        int j = tid + i * T + r;
        if (j >= s) j -= s;
        v[i] = dadd(v[i], tsh[j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) t[tid + i * T] = v[i];
  }
}

// (D) the reduction's elementwise tail alone (paths without a tree pass): in
// place over the output tiles; VEC = slot pairs (16-byte accesses).
template <bool VEC>
__global__ void __launch_bounds__(256) epilogue_kernel(double* __restrict__ tiles, int64_t n_tiles,
                                                       int64_t s, FastDiv64 per_tile,
                                                       const __grid_constant__ EpiDev epi) {
  pdl_enter();
  const uint64_t total = static_cast<uint64_t>(n_tiles) * per_tile.d;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t tile = fdiv(w, per_tile);
    const int64_t j = static_cast<int64_t>(w - tile * per_tile.d) * (VEC ? 2 : 1);
    const EpiTile et = epi_tile(epi, tile, s);
    double* t = tiles + tile * s + j;
    if (VEC) {
      const double2 v = *reinterpret_cast<double2*>(t);
      double x[2] = {v.x, v.y};
      epi_apply_n<2>(epi, x, et, j, 1);
      *reinterpret_cast<double2*>(t) = make_double2(x[0], x[1]);
    } else {
      double x[1] = {*t};
      epi_apply_n<1>(epi, x, et, j, 1);
      *t = x[0];
    }
  }
}

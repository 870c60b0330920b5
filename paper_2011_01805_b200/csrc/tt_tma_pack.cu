// tt_tma_pack.cu -- pack / unpack as pure TMA data movement (sm_100a).
//
// For a tile shape whose dims are all plain data dims (no replication, no `~`,
// not relaxed; rank <= 5; last tile extent even so a box row is a multiple of
// 16 bytes), a tile is exactly one box of the dense tensor: the box with
// extents (t_1 .. t_k) at element coordinates (l_i * t_i).  Its row-major box
// layout in shared memory IS the tile's slot order (tile_tensor.hpp:31-39,
// Eq. 1), and the TMA unit zero-fills the out-of-bounds part of an edge box --
// precisely pack's padding (tile_tensor.hpp:209-215: slots outside the used
// box hold +0.0).  So
//   pack   = cp.async.bulk.tensor (dense box -> smem)  +  cp.async.bulk (smem -> tile)
//   unpack = cp.async.bulk (tile -> smem)  +  cp.async.bulk.tensor (smem -> dense box;
//            the TMA store writes only the in-bounds elements).
// One elected thread per CTA drives a ring of box buffers: loads run NB-1 boxes
// ahead of the stores, and a buffer is refilled once its store has finished
// reading it (cp.async.bulk.wait_group.read).  No per-slot instruction at all.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tt_launch.hpp"
#include "tt_pdl.cuh"

namespace ttb {

namespace {

// Largest sub-box per TMA transfer and ring depth.  Measured on config 5
// (16 GiB): on an idle GPU pack is fastest with 16 KiB boxes x 8 buffers
// (5.13 ms vs 5.52 ms with 64 KiB x 3), but right after ~100 ms of fused
// products (the bench's order) the 16 KiB ring drops to 6.1 ms while 64 KiB
// boxes hold 5.56 ms -- so 64 KiB is the default for both directions.
// TT_PACK_BOX_KB / TT_PACK_RING override, for measurement.
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
int max_box_bytes(bool) { return env_int("TT_PACK_BOX_KB", 64) * 1024; }
int max_ring() { return env_int("TT_PACK_RING", 8); }

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

struct TmaPackParams {
  int rank;
  int64_t n_items;          // tiles * subs
  int64_t subs;             // sub-boxes per tile (split of the outermost non-unit tile dim)
  int split_dim;            // tensor dim split into `subs` parts (box dim there = t / subs)
  int64_t sub_extent;       // t_split / subs
  int64_t s;                // slots per tile
  uint32_t box_bytes;       // one sub-box
  int64_t ext[5];           // external extents (tensor order)
  int64_t t[5];             // tile extents (tensor order)
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int RK>
__device__ __forceinline__ void item_coords(const TmaPackParams& pp, int64_t item, int64_t& tile,
                                            int64_t& sub, int32_t* c) {
  tile = item / pp.subs;
  sub = item - tile * pp.subs;
  int64_t rem = tile;
#pragma unroll
  for (int i = RK - 1; i >= 0; --i) {
    const int64_t l = rem % pp.ext[i];
    rem /= pp.ext[i];
    // TMA coordinate order is innermost first: tensor dim i -> coordinate RK-1-i
    int64_t e = l * pp.t[i];
    if (i == pp.split_dim) e += sub * pp.sub_extent;
    c[RK - 1 - i] = static_cast<int32_t>(e);
  }
}

template <int RK>
__device__ __forceinline__ void tma_load_box(void* dst, const CUtensorMap* map, const int32_t* c,
                                             uint64_t* bar) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  if constexpr (RK == 1)
    asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                 ::"r"(smem_addr(dst)), "l"(m), "r"(c[0]), "r"(smem_addr(bar)) : "memory");
  else if constexpr (RK == 2)
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_addr(dst)), "l"(m), "r"(c[0]), "r"(c[1]), "r"(smem_addr(bar)) : "memory");
  else if constexpr (RK == 3)
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_addr(dst)), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(smem_addr(bar)) : "memory");
  else if constexpr (RK == 4)
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(smem_addr(dst)), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(smem_addr(bar)) : "memory");
  else
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 ::"r"(smem_addr(dst)), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_addr(bar)) : "memory");
}

template <int RK>
__device__ __forceinline__ void tma_store_box(const CUtensorMap* map, const int32_t* c, const void* src) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  if constexpr (RK == 1)
    asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];"
                 ::"l"(m), "r"(c[0]), "r"(smem_addr(src)) : "memory");
  else if constexpr (RK == 2)
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                 ::"l"(m), "r"(c[0]), "r"(c[1]), "r"(smem_addr(src)) : "memory");
  else if constexpr (RK == 3)
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                 ::"l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(smem_addr(src)) : "memory");
  else if constexpr (RK == 4)
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                 ::"l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(smem_addr(src)) : "memory");
  else
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                 ::"l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_addr(src)) : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               ::"l"(dst), "r"(smem_addr(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(smem_addr(bar)), "r"(parity) : "memory");
}

// PACK=true: dense box -> tile.  PACK=false: tile -> dense box.
template <int RK, bool PACK>
__global__ void __launch_bounds__(32, 1) tma_pack_kernel(const __grid_constant__ CUtensorMap map,
                                                         const __grid_constant__ TmaPackParams pp,
                                                         double* tiles, int nbuf) {
  pdl_enter();
  extern __shared__ __align__(128) unsigned char sm[];
  if (threadIdx.x != 0) return;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  unsigned char* bufs = sm + 128;
  for (int i = 0; i < nbuf; ++i) bar_init(&bars[i]);
  const int64_t sub_slots = pp.box_bytes / sizeof(double);
  int64_t n_mine = 0;
  for (int64_t i = blockIdx.x; i < pp.n_items; i += gridDim.x) ++n_mine;
  auto item_of = [&](int64_t k) { return blockIdx.x + k * static_cast<int64_t>(gridDim.x); };
  auto issue_load = [&](int64_t k) {
    const int b = static_cast<int>(k % nbuf);
    unsigned char* dst = bufs + static_cast<size_t>(b) * pp.box_bytes;
    int64_t tile, sub;
    int32_t c[5];
    item_coords<RK>(pp, item_of(k), tile, sub, c);
    bar_expect(&bars[b], pp.box_bytes);
    if (PACK)
      tma_load_box<RK>(dst, &map, c, &bars[b]);
    else
      bulk_load(dst, tiles + tile * pp.s + sub * sub_slots, pp.box_bytes, &bars[b]);
  };
  const int64_t pre = n_mine < nbuf ? n_mine : nbuf;
  for (int64_t k = 0; k < pre; ++k) issue_load(k);
  for (int64_t k = 0; k < n_mine; ++k) {
    const int b = static_cast<int>(k % nbuf);
    bar_wait(&bars[b], static_cast<uint32_t>((k / nbuf) & 1));
    unsigned char* src = bufs + static_cast<size_t>(b) * pp.box_bytes;
    int64_t tile, sub;
    int32_t c[5];
    item_coords<RK>(pp, item_of(k), tile, sub, c);
    if (PACK)
      bulk_store(tiles + tile * pp.s + sub * sub_slots, src, pp.box_bytes);
    else
      tma_store_box<RK>(&map, c, src);
    bulk_commit();
    // refill the buffer of item k-1 (its store has read it) with item k-1+nbuf
    if (k >= 1 && k - 1 + nbuf < n_mine) {
      bulk_wait_read<1>();
      issue_load(k - 1 + nbuf);
    }
  }
  bulk_wait_all();
}

struct TmaPlan {
  bool ok = false;
  CUtensorMap map;
  TmaPackParams pp;
  int nbuf = 0;
  size_t smem = 0;
};

TmaPlan plan_tma(const LaunchCtx& c, const Shape& sh, int64_t s, const double* dense, bool pack) {
  const int kMaxBoxBytes = max_box_bytes(pack);
  const int kMaxRing = max_ring();
  TmaPlan tp;
  const int rank = sh.rank();
  if (rank > 5 || sh.relaxed || sh.tile_slots() != s) return tp;
  if ((reinterpret_cast<uintptr_t>(dense) & 15) != 0) return tp;
  for (const auto& d : sh.dims)
    if (d.d != 1 || d.interleaved || d.t > 256 || d.n >= (int64_t{1} << 31)) return tp;
  if (sh.dims[rank - 1].t % 2 != 0) return tp;               // box row multiple of 16 B
  if (rank > 1 && sh.dims[rank - 1].n % 2 != 0) return tp;    // global strides multiple of 16 B
  const auto ext = sh.external();
  // split the outermost tile dim with t > 1 until a sub-box fits kMaxBoxBytes
  int split = -1;
  for (int i = 0; i < rank; ++i)
    if (sh.dims[i].t > 1) {
      split = i;
      break;
    }
  if (split < 0) return tp;
  int64_t subs = 1;
  const int64_t tile_bytes = s * static_cast<int64_t>(sizeof(double));
  while (tile_bytes / subs > kMaxBoxBytes && sh.dims[split].t % (subs * 2) == 0) subs *= 2;
  // a tile that cannot be split down to the preferred box still takes TMA
  // with boxes up to 64 KiB
  if (tile_bytes / subs > std::max(kMaxBoxBytes, 64 * 1024)) return tp;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return tp;
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t box[5], estride[5];
  int64_t stride = sizeof(double);
  for (int k = 0; k < rank; ++k) {  // TMA order: innermost tensor dim first
    const int i = rank - 1 - k;
    gdim[k] = static_cast<cuuint64_t>(sh.dims[i].n);
    box[k] = static_cast<cuuint32_t>(i == split ? sh.dims[i].t / subs : sh.dims[i].t);
    estride[k] = 1;
    if (k > 0) gstride[k - 1] = static_cast<cuuint64_t>(stride);
    stride *= sh.dims[i].n;
  }
  const CUresult r = enc(&tp.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(dense),
                         gdim, gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return tp;
  std::memset(&tp.pp, 0, sizeof(tp.pp));
  tp.pp.rank = rank;
  tp.pp.subs = subs;
  tp.pp.split_dim = split;
  tp.pp.sub_extent = sh.dims[split].t / subs;
  tp.pp.s = s;
  tp.pp.box_bytes = static_cast<uint32_t>(tile_bytes / subs);
  tp.pp.n_items = sh.tile_count() * subs;
  for (int i = 0; i < rank; ++i) {
    tp.pp.ext[i] = ext[i];
    tp.pp.t[i] = sh.dims[i].t;
  }
  const size_t budget = c.smem_optin - 128;
  tp.nbuf = static_cast<int>(std::min<size_t>(kMaxRing, budget / tp.pp.box_bytes));
  if (tp.nbuf < 2) return tp;
  tp.smem = 128 + static_cast<size_t>(tp.nbuf) * tp.pp.box_bytes;
  tp.ok = true;
  return tp;
}

template <bool PACK>
bool launch_tma_copy(const LaunchCtx& c, const Shape& sh, int64_t s, const double* dense,
                     double* tiles) {
  if ((reinterpret_cast<uintptr_t>(tiles) & 15) != 0) return false;
  TmaPlan tp = plan_tma(c, sh, s, dense, PACK);
  if (!tp.ok) return false;
  const void* k = nullptr;
  switch (tp.pp.rank) {
    case 1: k = (const void*)tma_pack_kernel<1, PACK>; break;
    case 2: k = (const void*)tma_pack_kernel<2, PACK>; break;
    case 3: k = (const void*)tma_pack_kernel<3, PACK>; break;
    case 4: k = (const void*)tma_pack_kernel<4, PACK>; break;
    default: k = (const void*)tma_pack_kernel<5, PACK>; break;
  }
  check_cuda(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(tp.smem)),
             "smem attribute");
  int per_sm = 1;
  check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32, tp.smem), "occupancy");
  const int64_t grid64 = std::min<int64_t>(tp.pp.n_items, static_cast<int64_t>(c.sm_count) * std::max(per_sm, 1));
  const int grid = static_cast<int>(std::max<int64_t>(grid64, 1));
  switch (tp.pp.rank) {
    case 1: launch_k(c, tma_pack_kernel<1, PACK>, grid, 32, tp.smem, tp.map, tp.pp, tiles, tp.nbuf); break;
    case 2: launch_k(c, tma_pack_kernel<2, PACK>, grid, 32, tp.smem, tp.map, tp.pp, tiles, tp.nbuf); break;
    case 3: launch_k(c, tma_pack_kernel<3, PACK>, grid, 32, tp.smem, tp.map, tp.pp, tiles, tp.nbuf); break;
    case 4: launch_k(c, tma_pack_kernel<4, PACK>, grid, 32, tp.smem, tp.map, tp.pp, tiles, tp.nbuf); break;
    default: launch_k(c, tma_pack_kernel<5, PACK>, grid, 32, tp.smem, tp.map, tp.pp, tiles, tp.nbuf); break;
  }
  if (c.launches) ++*c.launches;
  check_cuda(cudaGetLastError(), PACK ? "tma pack kernel" : "tma unpack kernel");
  return true;
}

}  // namespace

bool encode_tensor_map_f64(void* map128, int rank, const void* base, const uint64_t* dims,
                           const uint64_t* stride_bytes, const uint32_t* box) {
  EncodeTiledFn enc = encode_fn();
  if (!enc || rank < 1 || rank > 5) return false;
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t bx[5], estride[5];
  for (int k = 0; k < rank; ++k) {
    gdim[k] = dims[k];
    bx[k] = box[k];
    estride[k] = 1;
    if (k > 0) gstride[k - 1] = stride_bytes[k - 1];
  }
  return enc(static_cast<CUtensorMap*>(map128), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank,
             const_cast<void*>(base), gdim, gstride, bx, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool launch_pack_tma(const LaunchCtx& c, const Shape& shape, int64_t s, const double* dense,
                     double* tiles) {
  return launch_tma_copy<true>(c, shape, s, dense, tiles);
}

bool launch_unpack_tma(const LaunchCtx& c, const Shape& shape, int64_t s, const double* tiles,
                       double* dense) {
  return launch_tma_copy<false>(c, shape, s, dense, const_cast<double*>(tiles));
}

}  // namespace ttb

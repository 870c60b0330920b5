// tt_kernels.cu -- hand-written sm_100a kernels of the tile-tensor hot path.
//
// Everything here is HBM-bandwidth bound fp64 gather/stream/reduction work
// (SURVEY 8d): no tensor cores.  Design rules applied throughout:
//  * persistent grids sized to (SM count x resident CTAs), grid-stride work;
//  * coalesced 16-byte (double2) accesses on the streamed operand;
//  * integer index math through precomputed magic-number division (no
//    hardware div/mod per slot);
//  * every fp64 operation is __dadd_rn / __dmul_rn, so ptxas cannot contract
//    a multiply and an add into an FMA: results are bit-identical to the
//    reference's scalar x86 loops (which have no FMA);
//  * reductions keep the reference's association exactly: the external left
//    fold (tile_tensor.hpp:323-324) runs per slot in registers, and the
//    in-tile rotate-and-sum schedule runs from shared memory without any HBM
//    round trip per rotation (north-star item 3).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>

#include "tt_launch.hpp"

namespace ttb {

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(TT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

constexpr int R = TT_MAX_RANK;

// ---- magic-number division ----------------------------------------------------

struct FastDiv64 {
  uint64_t d = 1, m = 0;
  uint32_t l = 0;
};

FastDiv64 make_div64(uint64_t d) {
  FastDiv64 f;
  f.d = d;
  if (d <= 1) return f;
  uint32_t l = 0;
  while ((uint64_t{1} << l) < d) ++l;  // l = ceil(log2 d), 1..63
  const unsigned __int128 two64 = static_cast<unsigned __int128>(1) << 64;
  const unsigned __int128 num = two64 * ((static_cast<unsigned __int128>(1) << l) - d);
  f.m = static_cast<uint64_t>(num / d) + 1;
  f.l = l;
  return f;
}

__device__ __forceinline__ uint64_t fdiv(uint64_t n, const FastDiv64& f) {
  if (f.d == 1) return n;
  const uint64_t t = __umul64hi(n, f.m);
  return (t + ((n - t) >> 1)) >> (f.l - 1);
}

struct FastDiv32 {
  uint32_t d = 1, m = 0, l = 0;
};

FastDiv32 make_div32(uint32_t d) {
  FastDiv32 f;
  f.d = d;
  if (d <= 1) return f;
  uint32_t l = 0;
  while ((uint64_t{1} << l) < d) ++l;
  const uint64_t num = (uint64_t{1} << 32) * ((uint64_t{1} << l) - d);
  f.m = static_cast<uint32_t>(num / d + 1);
  f.l = l;
  return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv32& f) {
  if (f.d == 1) return n;
  const uint32_t t = __umulhi(n, f.m);
  return (t + ((n - t) >> 1)) >> (f.l - 1);
}

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// Host-side launch overhead matters for short ops (a c3 matmul stage is ~40
// us of GPU work): occupancy answers and the dynamic-smem opt-in are cached
// per (device, kernel, block shape) instead of queried on every launch.
struct OccKey {
  int device;
  const void* kernel;
  int threads;
  size_t smem;
  bool operator<(const OccKey& o) const {
    return std::tie(device, kernel, threads, smem) < std::tie(o.device, o.kernel, o.threads, o.smem);
  }
};
std::mutex g_launch_cache_mu;
std::map<OccKey, int> g_occupancy;
std::map<std::pair<int, const void*>, size_t> g_smem_attr;

void set_smem_attr(const void* kernel, size_t smem) {
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_launch_cache_mu);
  size_t& cur = g_smem_attr[{dev, kernel}];
  if (smem <= cur) return;
  check_cuda(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)),
             "smem attribute");
  cur = smem;
}

int grid_for(const LaunchCtx& c, const void* kernel, int threads, size_t smem, int64_t work) {
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(g_launch_cache_mu);
    const OccKey key{c.device, kernel, threads, smem};
    auto it = g_occupancy.find(key);
    if (it != g_occupancy.end()) {
      per_sm = it->second;
    } else {
      check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem),
                 "occupancy query");
      g_occupancy[key] = per_sm;
    }
  }
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = static_cast<int64_t>(c.sm_count) * per_sm;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cap, work)));
}

void count_launch(const LaunchCtx& c) {
  if (c.launches) ++*c.launches;
}

void post_launch(const LaunchCtx& c, const char* what) {
  count_launch(c);
  check_cuda(cudaGetLastError(), what);
}

// ---- tile-grid geometry shared by pack / unpack / clean ------------------------

struct Geo {
  int rank;
  int64_t s;            // slots per tile
  int64_t tile_slots;   // prod t_i (< s only for relaxed shapes)
  int64_t n_tiles;
  FastDiv32 tdiv[R];    // divide by t_i
  FastDiv32 ediv[R];    // divide by ext_i
  FastDiv64 ndiv[R];    // divide by n_i (dense decomposition)
  int64_t t[R], ext[R], used[R], n[R];
  int64_t tstride[R];   // in-tile stride of dim i
  int64_t estride[R];   // external (tile-index) stride of dim i
  int64_t dstride[R];   // dense stride of dim i, 0 when n_i == 1 (replication)
  int32_t inter[R];
  int32_t quad_runs;
};

Geo make_geo(const Shape& sh, int64_t s) {
  Geo g;
  std::memset(&g, 0, sizeof(g));
  g.rank = sh.rank();
  g.s = s;
  g.tile_slots = sh.tile_slots();
  g.n_tiles = sh.tile_count();
  const auto ext = sh.external();
  const auto ts = tile_strides(sh);
  const auto es = row_major_strides(ext);
  std::vector<int64_t> nn;
  for (const auto& d : sh.dims) nn.push_back(d.n);
  const auto ds = row_major_strides(nn);
  for (int i = 0; i < g.rank; ++i) {
    const Dim& d = sh.dims[i];
    g.tdiv[i] = make_div32(static_cast<uint32_t>(d.t));
    g.ediv[i] = make_div32(static_cast<uint32_t>(ext[i]));
    g.ndiv[i] = make_div64(static_cast<uint64_t>(d.n));
    g.t[i] = d.t;
    g.ext[i] = ext[i];
    g.used[i] = d.used();
    g.n[i] = d.n;
    g.tstride[i] = ts[i];
    g.estride[i] = es[i];
    g.dstride[i] = d.n == 1 ? 0 : ds[i];
    g.inter[i] = d.interleaved ? 1 : 0;
  }
  const Dim& last = sh.dims[g.rank - 1];
  g.quad_runs = (last.n > 1 && !last.interleaved && last.t % 4 == 0) ? 1 : 0;
  return g;
}

// Decompose tile index `flat` into external coordinates l_i.
template <int RK>
__device__ __forceinline__ void tile_coords(const Geo& g, uint32_t flat, uint32_t* l) {
#pragma unroll
  for (int i = RK - 1; i >= 0; --i) {
    if (i < g.rank) {
      const uint32_t q = fdiv(flat, g.ediv[i]);
      l[i] = flat - q * g.ediv[i].d;
      flat = q;
    }
  }
}

// Eq.(1) (tile_tensor.hpp:205-214): source offset of slot h of the tile with
// coordinates l, or -1 when the slot is outside the used box (zero padding).
template <int RK>
__device__ __forceinline__ int64_t slot_source(const Geo& g, const uint32_t* l, uint32_t h) {
  if (h >= static_cast<uint64_t>(g.tile_slots)) return -1;
  int64_t src = 0;
#pragma unroll
  for (int i = RK - 1; i >= 0; --i) {
    if (i < g.rank) {
      const uint32_t q = fdiv(h, g.tdiv[i]);
      const int64_t m = h - q * g.tdiv[i].d;
      h = q;
      const int64_t j = g.inter[i] ? m * g.ext[i] + l[i] : static_cast<int64_t>(l[i]) * g.t[i] + m;
      if (j >= g.used[i]) return -1;
      src += j * g.dstride[i];
    }
  }
  return src;
}

// ---- pack ------------------------------------------------------------------------
// A warp owns 256 consecutive slots of one tile; lane l fills the quads at
// l*4 and 128 + l*4 (two 16-byte stores each, 1 KiB contiguous per warp
// instruction).  When a quad's 4 sources are consecutive dense elements (the
// common case: a run along the last dim) they are read with two 16-byte
// loads, else slot by slot; padding slots are written as +0.0 without a read.

template <int RK, bool VEC>
__device__ __forceinline__ void pack_quad(const Geo& g, const uint32_t* l,
                                          const double* __restrict__ dense, uint32_t h0,
                                          double* out) {
  double v[4];
  const int64_t src0 = slot_source<RK>(g, l, h0);
  // quad_runs (host): the last dim is a plain data dim (n > 1, not
  // interleaved) with t % 4 == 0, so an aligned quad varies only along it and
  // its sources are src0 .. src0+3 whenever the first and last are in range.
  const bool run = VEC && g.quad_runs && h0 + 4 <= g.s && src0 >= 0 &&
                   slot_source<RK>(g, l, h0 + 3) >= 0;
  if (run && (src0 & 1) == 0) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(dense + src0));
    const double2 b = __ldg(reinterpret_cast<const double2*>(dense + src0) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  } else if (run) {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldg(dense + src0 + k);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t src = k == 0 ? src0 : slot_source<RK>(g, l, h0 + k);
      v[k] = src >= 0 ? __ldg(dense + src) : 0.0;
    }
  }
  if (VEC && h0 + 4 <= g.s) {
    reinterpret_cast<double2*>(out)[0] = make_double2(v[0], v[1]);
    reinterpret_cast<double2*>(out)[1] = make_double2(v[2], v[3]);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (h0 + k < g.s) out[k] = v[k];
  }
}

template <int RK, bool VEC>
__global__ void __launch_bounds__(256) pack_kernel(const __grid_constant__ Geo g,
                                                    const double* __restrict__ dense,
                                                    double* __restrict__ tiles,
                                                    FastDiv64 units_div) {
  const uint64_t total = static_cast<uint64_t>(g.n_tiles) * units_div.d;
  const int lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
       u < total; u += warps) {
    const uint64_t flat = fdiv(u, units_div);
    const uint32_t base = static_cast<uint32_t>((u - flat * units_div.d) * 256);
    uint32_t l[RK];
    tile_coords<RK>(g, static_cast<uint32_t>(flat), l);
    double* tile = tiles + flat * g.s;
    const uint32_t h0 = base + lane * 4;
    const uint32_t h1 = h0 + 128;
    if (h0 < g.s) pack_quad<RK, VEC>(g, l, dense, h0, tile + h0);
    if (h1 < g.s) pack_quad<RK, VEC>(g, l, dense, h1, tile + h1);
  }
}

// ---- unpack ----------------------------------------------------------------------
// One work item = 4 consecutive dense elements (coalesced writes); each reads
// replica 0 (tile_tensor.hpp:231-239).

template <int RK>
__global__ void __launch_bounds__(256) unpack_kernel(const __grid_constant__ Geo g,
                                                      const double* __restrict__ tiles,
                                                      double* __restrict__ dense,
                                                      uint64_t total) {
  const uint64_t quads = (total + 3) / 4;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < quads;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t f = w * 4;
    int64_t j[RK];
    uint64_t rem = f;
#pragma unroll
    for (int i = RK - 1; i >= 0; --i) {
      if (i < g.rank) {
        const uint64_t q = fdiv(rem, g.ndiv[i]);
        j[i] = static_cast<int64_t>(rem - q * g.ndiv[i].d);
        rem = q;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (f + k < total) {
        int64_t tile = 0, h = 0;
#pragma unroll
        for (int i = 0; i < RK; ++i) {
          if (i < g.rank) {
            int64_t li, mi;
            if (g.inter[i]) {
              const uint32_t q = fdiv(static_cast<uint32_t>(j[i]), g.ediv[i]);
              li = j[i] - static_cast<int64_t>(q) * g.ext[i];
              mi = q;
            } else {
              const uint32_t q = fdiv(static_cast<uint32_t>(j[i]), g.tdiv[i]);
              li = q;
              mi = j[i] - static_cast<int64_t>(q) * g.t[i];
            }
            tile += li * g.estride[i];
            h += mi * g.tstride[i];
          }
        }
        dense[f + k] = __ldg(tiles + tile * g.s + h);
        // odometer step
#pragma unroll
        for (int i = RK - 1; i >= 0; --i) {
          if (i < g.rank) {
            if (++j[i] < g.n[i]) break;
            j[i] = 0;
          }
        }
      }
    }
  }
}

// ---- clean_unknowns: multiply by the 0/1 used indicator ---------------------------

template <int RK>
__global__ void __launch_bounds__(256) clean_kernel(const __grid_constant__ Geo g,
                                                     const double* __restrict__ in,
                                                     double* __restrict__ out,
                                                     FastDiv64 quads_div) {
  const uint64_t total = static_cast<uint64_t>(g.n_tiles) * quads_div.d;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t flat = fdiv(w, quads_div);
    const uint32_t h0 = static_cast<uint32_t>((w - flat * quads_div.d) * 4);
    uint32_t l[RK];
    tile_coords<RK>(g, static_cast<uint32_t>(flat), l);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t h = h0 + k;
      if (h < g.s) {
        const double mask = slot_source<RK>(g, l, h) >= 0 ? 1.0 : 0.0;
        const uint64_t o = flat * g.s + h;
        out[o] = dmul(in[o], mask);  // Session::mask_mul backend.hpp:145
      }
    }
  }
}

// Chunked form (even s): a work item is a 4096-slot chunk of one tile.  The
// tile's coordinates are decoded once per item; when every in-tile coordinate
// of the tile maps inside the used region (all tiles but the '?' boundary
// ones), the chunk is a vectorised multiply by 1.0 with no per-slot index
// math, otherwise the per-slot mask test of clean_kernel.
constexpr int kCleanChunk = 4096;
template <int RK>
__global__ void __launch_bounds__(256) clean_chunk_kernel(const __grid_constant__ Geo g,
                                                           const double* __restrict__ in,
                                                           double* __restrict__ out,
                                                           FastDiv64 chunks_div) {
  const uint64_t items = static_cast<uint64_t>(g.n_tiles) * chunks_div.d;
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const uint64_t flat = fdiv(item, chunks_div);
    const int64_t base = static_cast<int64_t>(item - flat * chunks_div.d) * kCleanChunk;
    uint32_t l[RK];
    tile_coords<RK>(g, static_cast<uint32_t>(flat), l);
    bool full = g.tile_slots == g.s;
#pragma unroll
    for (int i = 0; i < RK; ++i) {
      const int64_t last = g.inter[i] ? (g.t[i] - 1) * g.ext[i] + l[i] : l[i] * g.t[i] + g.t[i] - 1;
      full = full && last < g.used[i];
    }
    const double* src = in + flat * g.s + base;
    double* dst = out + flat * g.s + base;
    const int64_t n = g.s - base < kCleanChunk ? g.s - base : kCleanChunk;
    if (full) {
      const double2* s2 = reinterpret_cast<const double2*>(src);
      double2* d2 = reinterpret_cast<double2*>(dst);
      double2 v[kCleanChunk / 512];
#pragma unroll
      for (int u = 0; u < kCleanChunk / 512; ++u) {
        const int64_t k = u * 256 + threadIdx.x;
        if (2 * k < n) v[u] = __ldg(s2 + k);
      }
#pragma unroll
      for (int u = 0; u < kCleanChunk / 512; ++u) {
        const int64_t k = u * 256 + threadIdx.x;
        if (2 * k < n) d2[k] = make_double2(dmul(v[u].x, 1.0), dmul(v[u].y, 1.0));
      }
    } else {
      // boundary tile: the used slots form the box m_i < v_i in tile
      // coordinates; with power-of-two extents m_i = (h >> sh_i) & (t_i - 1)
      bool pow2 = true;
      int64_t v[RK];
      int sh[RK];
#pragma unroll
      for (int i = 0; i < RK; ++i) {
        pow2 = pow2 && (g.t[i] & (g.t[i] - 1)) == 0 && (g.tstride[i] & (g.tstride[i] - 1)) == 0;
        const int64_t left = g.inter[i] ? (g.used[i] - l[i] + g.ext[i] - 1) / g.ext[i]
                                        : g.used[i] - static_cast<int64_t>(l[i]) * g.t[i];
        v[i] = left < 0 ? 0 : (left > g.t[i] ? g.t[i] : left);
        sh[i] = __ffsll(static_cast<long long>(g.tstride[i])) - 1;
      }
      if (pow2) {
        // only the dims this tile cuts short need a test (uniform per item)
        bool cut[RK];
#pragma unroll
        for (int i = 0; i < RK; ++i) cut[i] = v[i] < g.t[i];
        const double2* s2 = reinterpret_cast<const double2*>(src);
        double2* d2 = reinterpret_cast<double2*>(dst);
        constexpr int U = kCleanChunk / 512;
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t k = u * 256 + threadIdx.x;
          if (2 * k < n) x[u] = __ldg(s2 + k);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t k = u * 256 + threadIdx.x;
          if (2 * k < n) {
            double m[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int64_t h = base + 2 * k + e;
              bool ok = h < g.tile_slots;
#pragma unroll
              for (int i = 0; i < RK; ++i)
                if (cut[i]) ok = ok && ((h >> sh[i]) & (g.t[i] - 1)) < v[i];
              m[e] = ok ? 1.0 : 0.0;
            }
            d2[k] = make_double2(dmul(x[u].x, m[0]), dmul(x[u].y, m[1]));
          }
        }
      } else {
        for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
          const double mask = slot_source<RK>(g, l, static_cast<uint32_t>(base + k)) >= 0 ? 1.0 : 0.0;
          dst[k] = dmul(src[k], mask);  // Session::mask_mul backend.hpp:145
        }
      }
    }
  }
}

// ---- elementwise with external broadcast ------------------------------------------

struct EwParams {
  int rank;
  int64_t s;
  int64_t n_tiles;
  FastDiv32 ediv[R];      // out external extents
  int64_t a_stride[R];    // tile-index stride of A along dim i, 0 where A broadcasts
  int64_t b_stride[R];
  int64_t o_stride[R];    // chunk kernel: out tile-index stride; dims in visiting order
};

template <int OP, bool VEC>
__global__ void __launch_bounds__(256) elementwise_kernel(const __grid_constant__ EwParams p,
                                                           const double* __restrict__ a,
                                                           const double* __restrict__ b,
                                                           double* __restrict__ out,
                                                           FastDiv64 quads_div) {
  const uint64_t total = static_cast<uint64_t>(p.n_tiles) * quads_div.d;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t flat = fdiv(w, quads_div);
    const uint32_t h0 = static_cast<uint32_t>((w - flat * quads_div.d) * 4);
    uint32_t rem = static_cast<uint32_t>(flat);
    int64_t fa = 0, fb = 0;
#pragma unroll
    for (int i = R - 1; i >= 0; --i) {
      if (i < p.rank) {
        const uint32_t q = fdiv(rem, p.ediv[i]);
        const int64_t li = rem - q * p.ediv[i].d;
        rem = q;
        fa += li * p.a_stride[i];
        fb += li * p.b_stride[i];
      }
    }
    const double* pa = a + fa * p.s + h0;
    const double* pb = b + fb * p.s + h0;
    double* po = out + flat * p.s + h0;
    if (VEC && h0 + 4 <= p.s) {
      const double2 a0 = __ldg(reinterpret_cast<const double2*>(pa));
      const double2 a1 = __ldg(reinterpret_cast<const double2*>(pa) + 1);
      const double2 b0 = __ldg(reinterpret_cast<const double2*>(pb));
      const double2 b1 = __ldg(reinterpret_cast<const double2*>(pb) + 1);
      double2 o0, o1;
      if (OP == TT_OP_ADD) {
        o0 = make_double2(dadd(a0.x, b0.x), dadd(a0.y, b0.y));
        o1 = make_double2(dadd(a1.x, b1.x), dadd(a1.y, b1.y));
      } else {
        o0 = make_double2(dmul(a0.x, b0.x), dmul(a0.y, b0.y));
        o1 = make_double2(dmul(a1.x, b1.x), dmul(a1.y, b1.y));
      }
      reinterpret_cast<double2*>(po)[0] = o0;
      reinterpret_cast<double2*>(po)[1] = o1;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (h0 + k < p.s)
          po[k] = OP == TT_OP_ADD ? dadd(pa[k], pb[k]) : dmul(pa[k], pb[k]);
    }
  }
}

// Streaming form for even s (the common case): a work item is a 2048-slot
// chunk of one output tile; the external-index decomposition (broadcast
// source tiles) is done once per item, uniformly, and each thread then
// moves 4 x 16 bytes of A, B and OUT with all eight loads in flight --
// the per-16-byte index math of elementwise_kernel is what held the
// broadcast product on config 5 to 62% of the copy peak.
constexpr int kEwU = 8;                // double2 per thread per item
constexpr int kEwChunk = 512 * kEwU;   // slots per work item (256 threads x kEwU x double2)
template <int OP>
__global__ void __launch_bounds__(256) elementwise_chunk_kernel(const __grid_constant__ EwParams p,
                                                                 const double* __restrict__ a,
                                                                 const double* __restrict__ b,
                                                                 double* __restrict__ out,
                                                                 FastDiv64 chunks_div) {
  const uint64_t items = static_cast<uint64_t>(p.n_tiles) * chunks_div.d;
  const int tid = threadIdx.x;
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const uint64_t vt = fdiv(item, chunks_div);  // tile in visiting order
    const int64_t base = static_cast<int64_t>(item - vt * chunks_div.d) * kEwChunk;
    uint32_t rem = static_cast<uint32_t>(vt);
    int64_t fa = 0, fb = 0, flat = 0;
#pragma unroll
    for (int i = R - 1; i >= 0; --i) {
      if (i < p.rank) {
        const uint32_t q = fdiv(rem, p.ediv[i]);
        const int64_t li = rem - q * p.ediv[i].d;
        rem = q;
        fa += li * p.a_stride[i];
        fb += li * p.b_stride[i];
        flat += li * p.o_stride[i];
      }
    }
    const double2* pa = reinterpret_cast<const double2*>(a + fa * p.s + base);
    const double2* pb = reinterpret_cast<const double2*>(b + fb * p.s + base);
    double2* po = reinterpret_cast<double2*>(out + flat * p.s + base);
    const int64_t npairs = (p.s - base) / 2 < kEwChunk / 2 ? (p.s - base) / 2 : kEwChunk / 2;
    double2 va[kEwU], vb[kEwU];
#pragma unroll
    for (int u = 0; u < kEwU; ++u) {
      const int k = u * 256 + tid;
      if (k < npairs) {
        va[u] = __ldg(pa + k);
        vb[u] = __ldg(pb + k);
      }
    }
#pragma unroll
    for (int u = 0; u < kEwU; ++u) {
      const int k = u * 256 + tid;
      if (k < npairs)
        po[k] = OP == TT_OP_ADD ? make_double2(dadd(va[u].x, vb[u].x), dadd(va[u].y, vb[u].y))
                                : make_double2(dmul(va[u].x, vb[u].x), dmul(va[u].y, vb[u].y));
    }
  }
}

template <int OP>
__global__ void __launch_bounds__(256) binary_flat_kernel(const double* __restrict__ a,
                                                           const double* __restrict__ b,
                                                           double* __restrict__ out,
                                                           uint64_t count) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = OP == TT_OP_ADD ? dadd(a[i], b[i]) : dmul(a[i], b[i]);
}

__global__ void __launch_bounds__(256) rotate_kernel(const double* __restrict__ in,
                                                      double* __restrict__ out, uint64_t s,
                                                      uint64_t r, uint64_t total,
                                                      FastDiv64 sdiv) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t tile = fdiv(i, sdiv);
    uint64_t j = i - tile * s + r;
    if (j >= s) j -= s;
    out[i] = in[tile * s + j];
  }
}

// Chunked rotate: a work item is a 4096-slot chunk of one output tile; its
// source is the contiguous (cyclic) range starting at base + r, so each
// thread issues 16 coalesced loads before its 16 stores (no per-slot division).
constexpr int kRotChunk = 4096;
__global__ void __launch_bounds__(256) rotate_chunk_kernel(const double* __restrict__ in,
                                                            double* __restrict__ out, int64_t s,
                                                            int64_t r, uint64_t items,
                                                            FastDiv64 chunks_div) {
  constexpr int U = kRotChunk / 256;
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const uint64_t tile = fdiv(item, chunks_div);
    const int64_t base = static_cast<int64_t>(item - tile * chunks_div.d) * kRotChunk;
    const double* t = in + tile * s;
    double* o = out + tile * s;
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t h = base + u * 256 + threadIdx.x;
      if (h < s) {
        int64_t j = h + r;
        if (j >= s) j -= s;
        v[u] = __ldg(t + j);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t h = base + u * 256 + threadIdx.x;
      if (h < s) o[h] = v[u];
    }
  }
}

// Aligned variant (s % 32 == 0): a warp owns 32 x U consecutive outputs and
// loads the U + 1 32-slot-aligned source segments they span (cyclic), then
// shifts by r mod 32 with shuffles -- every DRAM sector is fetched once
// (the misaligned form's warp accesses straddle 9 sectors per 8).
template <int U>
__global__ void __launch_bounds__(256) rotate_aligned_kernel(const double* __restrict__ in,
                                                              double* __restrict__ out, int64_t s,
                                                              int64_t r, uint64_t units,
                                                              FastDiv64 units_div) {
  const int lane = threadIdx.x & 31;
  const int rho = static_cast<int>(r & 31);
  const int64_t r0 = r - rho;  // aligned part of the rotation
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
       w < units * 1; w += warps) {
    const uint64_t tile = fdiv(w, units_div);
    const int64_t h0 = static_cast<int64_t>(w - tile * units_div.d) * (32 * U);
    const double* t = in + tile * s;
    double v[U + 1];
#pragma unroll
    for (int u = 0; u <= U; ++u) {
      int64_t seg = h0 + r0 + 32 * u;
      seg = seg >= s ? seg - s : seg;
      seg = seg >= s ? seg - s : seg;
      v[u] = __ldg(t + seg + lane);
    }
    const int src = (lane + rho) & 31;
    const bool lo = lane + rho < 32;
    double* o = out + tile * s + h0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double a = __shfl_sync(0xffffffffu, v[u], src);
      const double b = __shfl_sync(0xffffffffu, v[u + 1], src);
      o[32 * u + lane] = lo ? a : b;
    }
  }
}

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
};

FoldParams to_fold(const GroupParams& p) {
  FoldParams f;
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

// ---- tree-only passes (phase 2 of a two-phase reduction), in place on OUT ----------------
// (A) column-local: the summed dim is the first (s == t * stride), so each
// column c of the tile viewed as [t][stride] is one cyclic sequence of t
// values; a thread loads its column, runs the power-of-two levels in
// registers (v'[m] = v[m] + v[(m + e) mod t]), stores it back.  Coalesced
// across threads (consecutive columns), no shared memory, no barrier.
// BACK: rotations by -e*stride (replicate_tile_dim's right-to-left schedule):
// the column is read mirrored (m -> T-1-m), which turns them into the forward
// levels below with the same operand order.  `in` may equal `out`.
template <int T, bool BACK = false>
__global__ void __launch_bounds__(256) col_tree_kernel(const double* in, double* out, int64_t n_tiles,
                                                       int64_t stride, int64_t s, FastDiv64 cdiv) {
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
template <int HR, int R = 16, bool BACK = false>
__global__ void __launch_bounds__(256) row_tree_kernel(const double* __restrict__ in,
                                                       double* __restrict__ out, int64_t n_tiles,
                                                       int64_t s, int nlevels, int4 lv0, int4 lv1) {
  constexpr int NR = R + HR;
  const int lane = threadIdx.x & 31;
  const int rows = static_cast<int>(s / 32);
  const int blocks_per_tile = rows / R;
  const uint64_t total = static_cast<uint64_t>(n_tiles) * blocks_per_tile;
  const int lvl[8] = {lv0.x, lv0.y, lv0.z, lv0.w, lv1.x, lv1.y, lv1.z, lv1.w};
  for (uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
       u < total; u += static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5)) {
    const uint64_t tile = u / blocks_per_tile;
    const int rb = static_cast<int>(u - tile * blocks_per_tile) * R;
    const double* t = in + tile * s;
    double* o = out + tile * s;
    double v[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      int row = rb + i;
      if (row >= rows) row -= rows;  // cyclic halo
      const int64_t p = row * 32 + lane;
      v[i] = __ldg(t + (BACK ? s - 1 - p : p));
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
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int64_t p = (rb + i) * 32 + lane;
      o[BACK ? s - 1 - p : p] = v[i];
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

// ---- batch-packed affine layer (nn.hpp:282-326) ----------------------------------------
// One thread per (output tile o, slot j); consecutive threads take
// consecutive slots of one output, so every tap's tile read is coalesced and
// its weight / source index is a warp-uniform broadcast load.
__global__ void __launch_bounds__(256) batch_affine_kernel(const double* __restrict__ in, int64_t s,
                                                           uint64_t total,
                                                           const int64_t* __restrict__ row_ptr,
                                                           const int64_t* __restrict__ src,
                                                           const double* __restrict__ w,
                                                           const double* __restrict__ bias,
                                                           double* __restrict__ out, FastDiv64 sdiv) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t o = fdiv(i, sdiv);
    const int64_t j = static_cast<int64_t>(i - o * sdiv.d);
    double acc = bias[o];
    const int64_t k1 = row_ptr[o + 1];
    for (int64_t k = row_ptr[o]; k < k1; ++k) acc = dadd(acc, dmul(w[k], __ldg(in + src[k] * s + j)));
    out[i] = acc;
  }
}

// ---- fold over a range of output tiles (cross-rank chains, sharding.py) -------------
struct FoldRangeParams {
  int rank;
  FastDiv32 gdiv[R];
  int64_t a_stride[R], b_stride[R];
  int64_t astep, bstep, first, count, s, o0, npairs_tile;
};

template <bool HAS_B, bool INIT>
__global__ void __launch_bounds__(256) fold_range_kernel(const __grid_constant__ FoldRangeParams p,
                                                          const double* __restrict__ A,
                                                          const double* __restrict__ B,
                                                          const double* __restrict__ init,
                                                          double* __restrict__ acc_out, uint64_t total,
                                                          FastDiv64 pairs_div) {
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = fdiv(w, pairs_div);  // output tile within the range
    const int64_t j = static_cast<int64_t>(w - k * pairs_div.d) * 2;
    uint32_t rem = static_cast<uint32_t>(p.o0 + static_cast<int64_t>(k));
    int64_t fa = 0, fb = 0;
#pragma unroll
    for (int i = R - 1; i >= 0; --i) {
      if (i < p.rank) {
        const uint32_t q = fdiv(rem, p.gdiv[i]);
        const int64_t li = rem - q * p.gdiv[i].d;
        rem = q;
        fa += li * p.a_stride[i];
        fb += li * p.b_stride[i];
      }
    }
    const double* pa = A + (fa + p.first * p.astep) * p.s + j;
    const double* pb = HAS_B ? B + (fb + p.first * p.bstep) * p.s + j : nullptr;
    const int64_t sa = p.astep * p.s, sb = p.bstep * p.s;
    double2 acc;
    int64_t c0 = 0;
    if (INIT) {
      acc = *reinterpret_cast<const double2*>(init + k * p.s + j);
    } else {
      const double2 x = __ldg(reinterpret_cast<const double2*>(pa));
      if (HAS_B) {
        const double2 y = __ldg(reinterpret_cast<const double2*>(pb));
        acc = make_double2(dmul(x.x, y.x), dmul(x.y, y.y));
      } else {
        acc = x;
      }
      c0 = 1;
    }
    for (int64_t c = c0; c < p.count; ++c) {
      const double2 x = __ldg(reinterpret_cast<const double2*>(pa + c * sa));
      if (HAS_B) {
        const double2 y = __ldg(reinterpret_cast<const double2*>(pb + c * sb));
        acc.x = dadd(acc.x, dmul(x.x, y.x));
        acc.y = dadd(acc.y, dmul(x.y, y.y));
      } else {
        acc.x = dadd(acc.x, x.x);
        acc.y = dadd(acc.y, x.y);
      }
    }
    *reinterpret_cast<double2*>(acc_out + k * p.s + j) = acc;
  }
}

// Blocked form: `ob` consecutive output tiles that share one tap source list
// (every row of an fc layer; the filters of one window of a conv layer) are
// folded by one thread per slot pair: each input pair is loaded once and
// feeds ob accumulators (bias first, then + w * x in tap order -- the same
// association per output as batch_affine_kernel).
template <int OBMAX, int V>  // V = slots per thread (2: double2, 1: scalar for more threads)
__global__ void __launch_bounds__(256) batch_affine_blocked_kernel(
    const double* __restrict__ in, int64_t s, int64_t n_out, int ob, uint64_t total,
    const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ src,
    const double* __restrict__ w, const double* __restrict__ bias, double* __restrict__ out,
    FastDiv64 pairs_div) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t blk = fdiv(i, pairs_div);
    const int64_t j = static_cast<int64_t>(i - blk * pairs_div.d) * V;
    const int64_t o0 = static_cast<int64_t>(blk) * ob;
    const int64_t k0 = row_ptr[o0], taps = row_ptr[o0 + 1] - k0;
    double2 acc[OBMAX];
    int64_t wk[OBMAX];
#pragma unroll
    for (int r = 0; r < OBMAX; ++r) {
      if (r < ob && o0 + r < n_out) {
        acc[r] = make_double2(bias[o0 + r], bias[o0 + r]);
        wk[r] = row_ptr[o0 + r];
      }
    }
    for (int64_t t = 0; t < taps; ++t) {
      const double* px = in + src[k0 + t] * s + j;
      const double2 x = V == 2 ? __ldg(reinterpret_cast<const double2*>(px)) : make_double2(__ldg(px), 0.0);
#pragma unroll
      for (int r = 0; r < OBMAX; ++r) {
        if (r < ob && o0 + r < n_out) {
          const double wv = w[wk[r] + t];
          acc[r].x = dadd(acc[r].x, dmul(wv, x.x));
          if (V == 2) acc[r].y = dadd(acc[r].y, dmul(wv, x.y));
        }
      }
    }
#pragma unroll
    for (int r = 0; r < OBMAX; ++r) {
      if (r < ob && o0 + r < n_out) {
        if (V == 2)
          *reinterpret_cast<double2*>(out + (o0 + r) * s + j) = acc[r];
        else
          out[(o0 + r) * s + j] = acc[r].x;
      }
    }
  }
}

// Shared-memory form of the blocked fold (s % 512 == 0): a work item is one
// row block x 256 slot pairs (one CTA); weights and source indices for up to
// kBaTaps taps are staged per CTA, then each thread folds its pair with one
// 16-byte input load and 4 vector shared loads of weights per tap.
constexpr int kBaTaps = 64;
__global__ void __launch_bounds__(256) batch_affine_smem_kernel(
    const double* __restrict__ in, int64_t s, int64_t n_out, int ob, uint64_t items,
    const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ src,
    const double* __restrict__ w, const double* __restrict__ bias, double* __restrict__ out,
    FastDiv64 chunks_div) {
  __shared__ __align__(16) double ws[kBaTaps][8];
  __shared__ int64_t ss[kBaTaps];
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const uint64_t blk = fdiv(item, chunks_div);
    const int64_t j = (static_cast<int64_t>(item - blk * chunks_div.d) * 256 + threadIdx.x) * 2;
    const int64_t o0 = static_cast<int64_t>(blk) * ob;
    const int nr = static_cast<int>(n_out - o0 < ob ? n_out - o0 : ob);
    const int64_t k0 = row_ptr[o0], taps = row_ptr[o0 + 1] - k0;
    double2 acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const double bv = r < nr ? bias[o0 + r] : 0.0;
      acc[r] = make_double2(bv, bv);
    }
    for (int64_t t0 = 0; t0 < taps; t0 += kBaTaps) {
      const int nt = static_cast<int>(taps - t0 < kBaTaps ? taps - t0 : kBaTaps);
      __syncthreads();  // previous chunk consumed
      for (int e = threadIdx.x; e < nt * 8; e += 256) {
        const int t = e >> 3, r = e & 7;
        ws[t][r] = r < nr ? w[row_ptr[o0 + r] + t0 + t] : 0.0;
      }
      for (int t = threadIdx.x; t < nt; t += 256) ss[t] = src[k0 + t0 + t];
      __syncthreads();
      for (int t = 0; t < nt; ++t) {
        const double2 x = __ldg(reinterpret_cast<const double2*>(in + ss[t] * s + j));
        const double2* wv = reinterpret_cast<const double2*>(ws[t]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 w2 = wv[q];
          acc[2 * q].x = dadd(acc[2 * q].x, dmul(w2.x, x.x));
          acc[2 * q].y = dadd(acc[2 * q].y, dmul(w2.x, x.y));
          acc[2 * q + 1].x = dadd(acc[2 * q + 1].x, dmul(w2.y, x.x));
          acc[2 * q + 1].y = dadd(acc[2 * q + 1].y, dmul(w2.y, x.y));
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (r < nr) *reinterpret_cast<double2*>(out + (o0 + r) * s + j) = acc[r];
  }
}

// ---- synthetic input generator (== or_fill_uniform in oracle/tt_oracle.c) ------------

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void fill_uniform_kernel(double* out, uint64_t count, uint64_t key, uint64_t offset,
                                    double lo, double span) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t u = splitmix64(key ^ (offset + i));
    out[i] = dadd(lo, dmul(span, dmul(static_cast<double>(u >> 11), 0x1.0p-53)));
  }
}

uint64_t host_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

// ---- launchers ------------------------------------------------------------------

#define TT_RANK_SWITCH(rank, RKV, ...)          \
  switch (rank) {                               \
    case 1: { constexpr int RKV = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int RKV = 2; __VA_ARGS__; } break; \
    case 3: { constexpr int RKV = 3; __VA_ARGS__; } break; \
    case 4: { constexpr int RKV = 4; __VA_ARGS__; } break; \
    default: { constexpr int RKV = R; __VA_ARGS__; } break; \
  }

void launch_pack(const LaunchCtx& c, const Shape& shape, int64_t s, const double* dense,
                 double* tiles) {
  const Geo g = make_geo(shape, s);
  if (g.n_tiles == 0) return;
  const uint64_t units = static_cast<uint64_t>((s + 255) / 256);
  const FastDiv64 ud = make_div64(units);
  const int64_t work = (g.n_tiles * static_cast<int64_t>(units) + 7) / 8;
  const bool vec = (s % 2 == 0) && aligned16(tiles) && aligned16(dense);
  TT_RANK_SWITCH(g.rank, RK, {
    const void* k = vec ? (const void*)pack_kernel<RK, true> : (const void*)pack_kernel<RK, false>;
    const int grid = grid_for(c, k, 256, 0, work);
    if (vec)
      pack_kernel<RK, true><<<grid, 256, 0, c.stream>>>(g, dense, tiles, ud);
    else
      pack_kernel<RK, false><<<grid, 256, 0, c.stream>>>(g, dense, tiles, ud);
  });
  post_launch(c, "pack kernel");
}

void launch_unpack(const LaunchCtx& c, const Shape& shape, int64_t s, const double* tiles,
                   double* dense) {
  const Geo g = make_geo(shape, s);
  const uint64_t total = static_cast<uint64_t>(shape.dense_count());
  if (total == 0) return;
  const int64_t work = static_cast<int64_t>((total + 1023) / 1024);
  TT_RANK_SWITCH(g.rank, RK, {
    const int grid = grid_for(c, (const void*)unpack_kernel<RK>, 256, 0, work);
    unpack_kernel<RK><<<grid, 256, 0, c.stream>>>(g, tiles, dense, total);
  });
  post_launch(c, "unpack kernel");
}

// TT_EW_CHUNK=0 keeps the per-16-byte elementwise / clean kernels (measurement)
const int g_ew_chunk = [] {
  const char* e = std::getenv("TT_EW_CHUNK");
  return e ? std::atoi(e) : 1;
}();

void launch_clean(const LaunchCtx& c, const Shape& shape, int64_t s, const double* in,
                  double* out) {
  const Geo g = make_geo(shape, s);
  if (s % 2 == 0 && aligned16(in) && aligned16(out) && g_ew_chunk) {
    const uint64_t chunks = static_cast<uint64_t>((s + kCleanChunk - 1) / kCleanChunk);
    const FastDiv64 cd = make_div64(chunks);
    const int64_t items = g.n_tiles * static_cast<int64_t>(chunks);
    TT_RANK_SWITCH(g.rank, RK, {
      const int grid = grid_for(c, (const void*)clean_chunk_kernel<RK>, 256, 0, items);
      clean_chunk_kernel<RK><<<grid, 256, 0, c.stream>>>(g, in, out, cd);
    });
    post_launch(c, "clean_unknowns chunk kernel");
    return;
  }
  const uint64_t quads = static_cast<uint64_t>((s + 3) / 4);
  const FastDiv64 qd = make_div64(quads);
  const int64_t work = (g.n_tiles * static_cast<int64_t>(quads) + 255) / 256;
  TT_RANK_SWITCH(g.rank, RK, {
    const int grid = grid_for(c, (const void*)clean_kernel<RK>, 256, 0, work);
    clean_kernel<RK><<<grid, 256, 0, c.stream>>>(g, in, out, qd);
  });
  post_launch(c, "clean_unknowns kernel");
}

void launch_elementwise(const LaunchCtx& c, int op, const Shape& out, const Shape& a,
                        const Shape& b, int64_t s, const double* ta, const double* tb,
                        double* tout) {
  EwParams p;
  std::memset(&p, 0, sizeof(p));
  p.rank = out.rank();
  p.s = s;
  p.n_tiles = out.tile_count();
  const auto eo = out.external();
  const auto ea = a.external();
  const auto eb = b.external();
  const auto sa = row_major_strides(ea);
  const auto sb = row_major_strides(eb);
  for (int i = 0; i < p.rank; ++i) {
    p.ediv[i] = make_div32(static_cast<uint32_t>(eo[i]));
    // l mod e_a is l when e_a == e_out and 0 when e_a == 1 (the only cases
    // compatible shapes allow, shape.hpp:306-308).
    p.a_stride[i] = ea[i] == 1 ? 0 : sa[i];
    p.b_stride[i] = eb[i] == 1 ? 0 : sb[i];
  }
  if (p.n_tiles == 0) return;
  const bool vec = (s % 2 == 0) && aligned16(ta) && aligned16(tb) && aligned16(tout);
  if (vec && g_ew_chunk) {
    // visit output tiles with the dims along which an operand broadcasts
    // innermost: consecutive work items then reuse the broadcast operand's
    // tile from L2 (config 5 X * W: W is 128 MiB, re-read per X row otherwise)
    EwParams q = p;
    const auto so = row_major_strides(eo);
    int order[R], n = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i < p.rank; ++i) {
        const bool bcast = eo[i] > 1 && (p.a_stride[i] == 0 || p.b_stride[i] == 0);
        if (bcast == (pass == 1)) order[n++] = i;
      }
    for (int k = 0; k < p.rank; ++k) {
      const int i = order[k];
      q.ediv[k] = p.ediv[i];
      q.a_stride[k] = p.a_stride[i];
      q.b_stride[k] = p.b_stride[i];
      q.o_stride[k] = so[i];
    }
    const uint64_t chunks = static_cast<uint64_t>((s + kEwChunk - 1) / kEwChunk);
    const FastDiv64 cd = make_div64(chunks);
    const int64_t items = p.n_tiles * static_cast<int64_t>(chunks);
    if (op == TT_OP_ADD) {
      const int grid = grid_for(c, (const void*)elementwise_chunk_kernel<TT_OP_ADD>, 256, 0, items);
      elementwise_chunk_kernel<TT_OP_ADD><<<grid, 256, 0, c.stream>>>(q, ta, tb, tout, cd);
    } else {
      const int grid = grid_for(c, (const void*)elementwise_chunk_kernel<TT_OP_MUL>, 256, 0, items);
      elementwise_chunk_kernel<TT_OP_MUL><<<grid, 256, 0, c.stream>>>(q, ta, tb, tout, cd);
    }
    post_launch(c, "elementwise chunk kernel");
    return;
  }
  const uint64_t quads = static_cast<uint64_t>((s + 3) / 4);
  const FastDiv64 qd = make_div64(quads);
  const int64_t work = (p.n_tiles * static_cast<int64_t>(quads) + 255) / 256;
#define TT_EW(OPV, VECV)                                                                  \
  {                                                                                       \
    const int grid = grid_for(c, (const void*)elementwise_kernel<OPV, VECV>, 256, 0, work); \
    elementwise_kernel<OPV, VECV><<<grid, 256, 0, c.stream>>>(p, ta, tb, tout, qd);       \
  }
  if (op == TT_OP_ADD) {
    if (vec) TT_EW(TT_OP_ADD, true) else TT_EW(TT_OP_ADD, false)
  } else {
    if (vec) TT_EW(TT_OP_MUL, true) else TT_EW(TT_OP_MUL, false)
  }
#undef TT_EW
  post_launch(c, "elementwise kernel");
}

void launch_fold_range(const LaunchCtx& c, const FoldRange& fr, int64_t s, int64_t o0, int64_t o1,
                       const double* ta, const double* tb, const double* init, double* acc) {
  if (o1 <= o0) return;
  if (s % 2 != 0 || !aligned16(ta) || (tb && !aligned16(tb)) || !aligned16(acc) ||
      (init && !aligned16(init)))
    invalid_argument("chain folds need an even slot count and 16-byte aligned tiles");
  FoldRangeParams p;
  std::memset(&p, 0, sizeof(p));
  p.rank = fr.rank;
  for (int i = 0; i < fr.rank; ++i) {
    p.gdiv[i] = make_div32(static_cast<uint32_t>(fr.gext[i]));
    p.a_stride[i] = fr.a_stride[i];
    p.b_stride[i] = fr.b_stride[i];
  }
  p.astep = fr.astep;
  p.bstep = fr.bstep;
  p.first = fr.first;
  p.count = fr.count;
  p.s = s;
  p.o0 = o0;
  const uint64_t pairs = static_cast<uint64_t>(s / 2);
  const uint64_t total = pairs * static_cast<uint64_t>(o1 - o0);
  const FastDiv64 pd = make_div64(pairs);
  const int64_t work = static_cast<int64_t>((total + 255) / 256);
#define TT_FR(HB, IN)                                                                        \
  {                                                                                         \
    const int grid = grid_for(c, (const void*)fold_range_kernel<HB, IN>, 256, 0, work);      \
    fold_range_kernel<HB, IN><<<grid, 256, 0, c.stream>>>(p, ta, tb, init, acc, total, pd);  \
  }
  if (tb) {
    if (init) TT_FR(true, true) else TT_FR(true, false)
  } else {
    if (init) TT_FR(false, true) else TT_FR(false, false)
  }
#undef TT_FR
  post_launch(c, "fold range kernel");
}

void launch_batch_affine(const LaunchCtx& c, const double* in, int64_t s, int64_t n_out,
                         const int64_t* row_ptr, const int64_t* src, const double* w,
                         const double* bias, double* out, int block) {
  const uint64_t total = static_cast<uint64_t>(s) * n_out;
  if (total == 0) return;
  if (block > 1 && s % 512 == 0 && aligned16(in) && aligned16(out)) {
    // every CTA works inside one row block: the block's weights for a run of
    // taps are staged in shared memory once per CTA (tap-major, 8 per tap)
    const uint64_t blocks = static_cast<uint64_t>((n_out + block - 1) / block);
    const uint64_t items = blocks * static_cast<uint64_t>(s / 512);
    const int grid = grid_for(c, (const void*)batch_affine_smem_kernel, 256, 0, static_cast<int64_t>(items));
    batch_affine_smem_kernel<<<grid, 256, 0, c.stream>>>(in, s, n_out, block, items, row_ptr, src, w,
                                                         bias, out, make_div64(static_cast<uint64_t>(s / 512)));
    post_launch(c, "batch affine smem kernel");
    return;
  }
  if (block > 1) {
    const uint64_t blocks = static_cast<uint64_t>((n_out + block - 1) / block);
    const bool pair = s % 2 == 0 && aligned16(in) && aligned16(out);
    const uint64_t per = static_cast<uint64_t>(pair ? s / 2 : s);
    const uint64_t work = blocks * per;
    const int64_t nb = static_cast<int64_t>((work + 255) / 256);
    if (pair) {
      const int grid = grid_for(c, (const void*)batch_affine_blocked_kernel<8, 2>, 256, 0, nb);
      batch_affine_blocked_kernel<8, 2><<<grid, 256, 0, c.stream>>>(in, s, n_out, block, work, row_ptr,
                                                                    src, w, bias, out, make_div64(per));
    } else {
      const int grid = grid_for(c, (const void*)batch_affine_blocked_kernel<8, 1>, 256, 0, nb);
      batch_affine_blocked_kernel<8, 1><<<grid, 256, 0, c.stream>>>(in, s, n_out, block, work, row_ptr,
                                                                    src, w, bias, out, make_div64(per));
    }
    post_launch(c, "batch affine blocked kernel");
    return;
  }
  const int grid = grid_for(c, (const void*)batch_affine_kernel, 256, 0, (total + 255) / 256);
  batch_affine_kernel<<<grid, 256, 0, c.stream>>>(in, s, total, row_ptr, src, w, bias, out,
                                                   make_div64(static_cast<uint64_t>(s)));
  post_launch(c, "batch affine kernel");
}

void launch_binary_flat(const LaunchCtx& c, int op, const double* a, const double* b, double* out,
                        int64_t count) {
  if (count <= 0) return;
  const int64_t work = (count + 255) / 256;
  if (op == TT_OP_ADD) {
    const int grid = grid_for(c, (const void*)binary_flat_kernel<TT_OP_ADD>, 256, 0, work);
    binary_flat_kernel<TT_OP_ADD><<<grid, 256, 0, c.stream>>>(a, b, out, count);
  } else {
    const int grid = grid_for(c, (const void*)binary_flat_kernel<TT_OP_MUL>, 256, 0, work);
    binary_flat_kernel<TT_OP_MUL><<<grid, 256, 0, c.stream>>>(a, b, out, count);
  }
  post_launch(c, "binary kernel");
}

void launch_rotate(const LaunchCtx& c, const double* in, double* out, int64_t s, int64_t r,
                   int64_t n_tiles) {
  const uint64_t total = static_cast<uint64_t>(s) * n_tiles;
  if (total == 0) return;
  if (s % 512 == 0) {  // a warp unit of 32 x 16 outputs
    const uint64_t per_tile = static_cast<uint64_t>(s / 512);
    const uint64_t units = per_tile * static_cast<uint64_t>(n_tiles);
    const int64_t work = static_cast<int64_t>((units + 7) / 8);
    const int grid = grid_for(c, (const void*)rotate_aligned_kernel<16>, 256, 0, work);
    rotate_aligned_kernel<16><<<grid, 256, 0, c.stream>>>(in, out, s, r, units, make_div64(per_tile));
    post_launch(c, "rotate aligned kernel");
    return;
  }
  const uint64_t chunks = static_cast<uint64_t>((s + kRotChunk - 1) / kRotChunk);
  const uint64_t items = chunks * static_cast<uint64_t>(n_tiles);
  if (s >= 1024) {  // chunked: whole 4096-slot items (small tiles keep one slot per thread)
    const int grid = grid_for(c, (const void*)rotate_chunk_kernel, 256, 0, static_cast<int64_t>(items));
    rotate_chunk_kernel<<<grid, 256, 0, c.stream>>>(in, out, s, r, items, make_div64(chunks));
    post_launch(c, "rotate chunk kernel");
    return;
  }
  const int grid = grid_for(c, (const void*)rotate_kernel, 256, 0, (total + 255) / 256);
  rotate_kernel<<<grid, 256, 0, c.stream>>>(in, out, s, r, total, make_div64(s));
  post_launch(c, "rotate kernel");
}

void launch_fill_uniform(const LaunchCtx& c, double* out, int64_t count, uint64_t seed,
                         int64_t offset, double lo, double hi) {
  if (count <= 0) return;
  const int grid = grid_for(c, (const void*)fill_uniform_kernel, 256, 0, (count + 255) / 256);
  fill_uniform_kernel<<<grid, 256, 0, c.stream>>>(out, count, host_splitmix64(seed), offset, lo,
                                                  hi - lo);
  post_launch(c, "fill kernel");
}

namespace {

GroupParams make_group_params(const Program& prog, const GroupSpec& g, int64_t s) {
  GroupParams p;
  std::memset(&p, 0, sizeof(p));
  p.g = g;
  for (int i = 0; i < g.nd; ++i) p.gdiv[i] = make_div64(static_cast<uint64_t>(g.ext[i]));
  p.s = s;
  p.nops = static_cast<int>(prog.ops.size());
  p.nbuf = prog.nbuf;
  for (size_t i = 0; i < prog.ops.size(); ++i) p.ops[i] = prog.ops[i];
  return p;
}

// Kernel-path override for A/B measurement and tests (tt_set_kernel_path /
// TT_KERNEL_PATH = tma | regs | generic); 0 = best eligible path.
std::atomic<int> g_forced_path{-1};

int forced_path() {
  int v = g_forced_path.load(std::memory_order_relaxed);
  if (v >= 0) return v;
  const char* e = std::getenv("TT_KERNEL_PATH");
  const std::string s(e ? e : "");
  v = s == "tma" ? 1 : s == "regs" ? 2 : s == "generic" ? 3 : s == "window" ? 4 : 0;
  g_forced_path.store(v, std::memory_order_relaxed);
  return v;
}

template <bool HAS_B>
void launch_fold(const LaunchCtx& c, const GroupParams& p, const double* ta, const double* tb,
                 double* tout) {
  const int64_t s = p.s;
  // 256 slots per warp when that still gives every SM >= 8 warps; otherwise
  // one slot per thread (small folds are latency bound: more loads in flight)
  const int64_t vec_warps = p.g.groups * ((s / 2 + 127) / 128);
  const bool vec = (s % 2 == 0) && aligned16(ta) && (!HAS_B || aligned16(tb)) && aligned16(tout) &&
                   vec_warps >= 8 * static_cast<int64_t>(c.sm_count);
  if (vec) {
    const uint64_t units = static_cast<uint64_t>((s / 2 + 127) / 128);
    const int64_t work = (p.g.groups * static_cast<int64_t>(units) + 7) / 8;
    const int grid = grid_for(c, (const void*)fold_kernel<HAS_B, true>, 256, 0, work);
    fold_kernel<HAS_B, true><<<grid, 256, 0, c.stream>>>(to_fold(p), ta, tb, tout, make_div64(units));
  } else {
    const int64_t work = (p.g.groups * s + 255) / 256;
    const int grid = grid_for(c, (const void*)fold_kernel<HAS_B, false>, 256, 0, work);
    fold_kernel<HAS_B, false><<<grid, 256, 0, c.stream>>>(to_fold(p), ta, tb, tout,
                                                           make_div64(static_cast<uint64_t>(s)));
  }
  post_launch(c, "fold kernel");
}

// GEMM unit width (TT_GEMM_SLOTS=64 forces the 64-slot, 1-CTA-per-SM variant).
const int g_gemm_slots = [] {
  const char* e = std::getenv("TT_GEMM_SLOTS");
  return e ? std::atoi(e) : 32;
}();
// GEMM block columns for 32-slot units: 8 (16 x 8 groups, 128 threads, twice the
// units of 16 x 16 -- better wave balance on 148 SMs; measured ~5% faster on
// config 3) or TT_GEMM_BC=16 (16 x 16 groups, 256 threads)
const int g_gemm_bc = [] {
  const char* e = std::getenv("TT_GEMM_BC");
  return e ? std::atoi(e) : 8;
}();

// TT_GEMM_TMA=0 disables the tensor-map-fed GEMM fold (cp.async variant instead)
const int g_gemm_tma = [] {
  const char* e = std::getenv("TT_GEMM_TMA");
  return e ? std::atoi(e) : 1;
}();

// Blocked-fold plan: ia = a group dim along which B broadcasts (A varies), ib =
// one along which A broadcasts (B varies).  Eligible when at least one exists.
struct BlockPlan {
  int ia = -1, ib = -1;
};

BlockPlan block_plan(const GroupSpec& g, bool has_b) {
  BlockPlan bp;
  if (!has_b) return bp;
  for (int i = 0; i < g.nd; ++i) {
    if (g.ext[i] <= 1) continue;
    if (g.a_stride[i] != 0 && g.b_stride[i] == 0 && bp.ia < 0) bp.ia = i;
    if (g.a_stride[i] == 0 && g.b_stride[i] != 0 && bp.ib < 0) bp.ib = i;
  }
  return bp;
}

// Launches fold_gemm_tma_kernel when both operands are expressible as 5-D
// tensor maps (<= 2 remaining group dims, non-zero fold strides); false
// otherwise (the caller falls back to the cp.async GEMM fold).
// TT_GEMM_DYNAMIC=0: static round-robin units instead of the work queue
const int g_gemm_dynamic = [] {
  const char* e = std::getenv("TT_GEMM_DYNAMIC");
  return e ? std::atoi(e) : 1;
}();
const int g_gemm_order = [] {
  const char* e = std::getenv("TT_GEMM_ORDER");
  return e ? std::atoi(e) : 0;
}();

template <int SL, int kTgSteps, int kTgStages, int SC, int PB = kGemmBlk>
bool launch_gemm_tma_sl(const LaunchCtx& c, const GroupParams& p, const GroupParams& pr,
                        BlockSpec bs, const double* ta, const double* tb, double* tout) {
  const GroupSpec& g = p.g;
  const int64_t s = p.s;
  const int64_t first = p.ops[0].x, count = p.ops[0].y;
  if (pr.g.nd > 2 || g.astep == 0 || g.bstep == 0 || s % SL != 0 || count >= (int64_t{1} << 31))
    return false;
  if (s >= (int64_t{1} << 32) || bs.ext_ia >= (int64_t{1} << 31) || bs.ext_ib >= (int64_t{1} << 31))
    return false;
  constexpr int BC = 16;
  TgSpec ts{};
  ts.nrest = pr.g.nd;
  ts.chunk_major = g_gemm_order;
  alignas(64) unsigned char mapA[128], mapB[128];
  const uint64_t eb = sizeof(double);
  uint64_t dA[5] = {static_cast<uint64_t>(s), static_cast<uint64_t>(bs.ext_ia), static_cast<uint64_t>(count), 1, 1};
  uint64_t dB[5] = {static_cast<uint64_t>(s), static_cast<uint64_t>(bs.ext_ib), static_cast<uint64_t>(count), 1, 1};
  uint64_t sA[4] = {static_cast<uint64_t>(bs.a_ia * s) * eb, static_cast<uint64_t>(g.astep * s) * eb,
                    static_cast<uint64_t>(s) * eb, static_cast<uint64_t>(s) * eb};
  uint64_t sB[4] = {static_cast<uint64_t>(bs.b_ib * s) * eb, static_cast<uint64_t>(g.bstep * s) * eb,
                    static_cast<uint64_t>(s) * eb, static_cast<uint64_t>(s) * eb};
  for (int i = 0; i < pr.g.nd; ++i) {
    if (pr.g.a_stride[i] > 0) {
      ts.a_act[i] = 1;
      dA[3 + i] = static_cast<uint64_t>(pr.g.ext[i]);
      sA[2 + i] = static_cast<uint64_t>(pr.g.a_stride[i] * s) * eb;
    } else if (pr.g.a_stride[i] < 0) {
      return false;
    }
    if (pr.g.b_stride[i] > 0) {
      ts.b_act[i] = 1;
      dB[3 + i] = static_cast<uint64_t>(pr.g.ext[i]);
      sB[2 + i] = static_cast<uint64_t>(pr.g.b_stride[i] * s) * eb;
    } else if (pr.g.b_stride[i] < 0) {
      return false;
    }
  }
  if (bs.a_ia <= 0 || bs.b_ib <= 0 || g.astep < 0 || g.bstep < 0) return false;
  const uint32_t boxA[5] = {static_cast<uint32_t>(SL), PB, kTgSteps, 1, 1};
  const uint32_t boxB[5] = {static_cast<uint32_t>(SL), BC, kTgSteps, 1, 1};
  if (!encode_tensor_map_f64(mapA, 5, ta + first * g.astep * s, dA, sA, boxA) ||
      !encode_tensor_map_f64(mapB, 5, tb + first * g.bstep * s, dB, sB, boxB))
    return false;
  bs.nbq = (bs.ext_ib + BC - 1) / BC;
  bs.nbp = (bs.ext_ia + PB - 1) / PB;
  bs.div_nbp = make_div64(static_cast<uint64_t>(bs.nbp));
  bs.chunks = s / SL;
  bs.units = pr.g.groups * bs.chunks * bs.nbp * bs.nbq;
  bs.div_nbq = make_div64(static_cast<uint64_t>(bs.nbq));
  bs.div_chunks = make_div64(static_cast<uint64_t>(bs.chunks));
  ts.small = bs.units < (int64_t{1} << 31) ? 1 : 0;
  ts.dq = make_div32(static_cast<uint32_t>(bs.nbq));
  ts.dp = make_div32(static_cast<uint32_t>(bs.nbp));
  ts.dc = make_div32(static_cast<uint32_t>(bs.chunks));
  auto k = fold_gemm_tma_kernel<BC, SL, kTgSteps, kTgStages, SC, PB>;
  constexpr size_t smem = tg_smem_bytes<BC, SL, kTgSteps, kTgStages, PB>();
  constexpr int threads = tg_warps<BC, SL, SC, PB>() * 32;
  set_smem_attr((const void*)k, smem);
  const int grid = grid_for(c, (const void*)k, threads, smem, bs.units);
  unsigned int* sched = g_gemm_dynamic ? take_sched_slot(c) : nullptr;
  k<<<grid, threads, smem, c.stream>>>(*reinterpret_cast<const CUtensorMap*>(mapA),
                                       *reinterpret_cast<const CUtensorMap*>(mapB), to_fold(pr), bs, ts, tout,
                                       sched);
  post_launch(c, "gemm fold kernel (TMA)");
  return true;
}


const int g_gemm_cfg = [] {
  const char* e = std::getenv("TT_GEMM_CFG");
  return e ? std::atoi(e) : 0;
}();

bool launch_gemm_tma(const LaunchCtx& c, const GroupParams& p, const GroupParams& pr,
                     const BlockSpec& bs, const double* ta, const double* tb, double* tout) {
  switch (g_gemm_cfg) {
    case 1: return launch_gemm_tma_sl<16, 2, 6, 4>(c, p, pr, bs, ta, tb, tout);
    case 2: return launch_gemm_tma_sl<16, 4, 4, 4>(c, p, pr, bs, ta, tb, tout);
    case 3: return launch_gemm_tma_sl<32, 2, 6, 4>(c, p, pr, bs, ta, tb, tout);
    case 4: return launch_gemm_tma_sl<8, 4, 3, 4, 32>(c, p, pr, bs, ta, tb, tout);
    case 5: return launch_gemm_tma_sl<16, 4, 3, 4, 32>(c, p, pr, bs, ta, tb, tout);
    case 6: return launch_gemm_tma_sl<8, 4, 4, 4, 32>(c, p, pr, bs, ta, tb, tout);
    default: return launch_gemm_tma_sl<16, 4, 3, 4>(c, p, pr, bs, ta, tb, tout);
  }
}

template <bool HAS_B, int P, int Q>
void run_blocked(const LaunchCtx& c, const GroupParams& p, const BlockSpec& bs, const double* ta,
                 const double* tb, double* tout) {
  auto k = fold_blocked_kernel<HAS_B, P, Q>;
  const int grid = grid_for(c, (const void*)k, kBlockThreads, 0, bs.units);
  k<<<grid, kBlockThreads, 0, c.stream>>>(to_fold(p), bs, ta, tb, tout);
  post_launch(c, "blocked fold kernel");
}

// Phase-1 fold into OUT using the blocked kernel (requires has_b and a plan).
template <bool HAS_B>
void launch_fold_blocked(const LaunchCtx& c, const GroupParams& p, const BlockPlan& bp,
                         const double* ta, const double* tb, double* tout, bool coltree = false) {
  const GroupSpec& g = p.g;
  GroupParams pr = p;  // the remaining ("rest") group dims
  pr.g.nd = 0;
  pr.g.groups = 1;
  for (int i = 0; i < g.nd; ++i) {
    if (i == bp.ia || i == bp.ib) continue;
    const int k = pr.g.nd++;
    pr.g.ext[k] = g.ext[i];
    pr.g.out_stride[k] = g.out_stride[i];
    pr.g.a_stride[k] = g.a_stride[i];
    pr.g.b_stride[k] = g.b_stride[i];
    pr.gdiv[k] = p.gdiv[i];
    pr.g.groups *= g.ext[i];
  }
  const bool gemm = bp.ia >= 0 && bp.ib >= 0 && p.s % kGemmSlots == 0 && aligned16(ta) &&
                    aligned16(tb) && forced_path() != 2 && p.ops[0].y < (int64_t{1} << 31);
  int P = gemm ? kGemmBlk : (bp.ia >= 0 ? 8 : 1);
  int Q = gemm ? (g_gemm_bc == 8 && !coltree && g_gemm_slots != 64 ? 8 : kGemmBlk) : (bp.ib >= 0 ? 8 : 1);
  if (coltree && !(gemm && Q == 16)) invalid_argument("column-tree fusion needs the 16x16 GEMM fold");
  if (gemm && !coltree) {  // 16 x 8 blocks when 16 x 16 would give fewer than ~3 waves of units
    const int64_t units16 = pr.g.groups * (p.s / kGemmSlots) * ((g.ext[bp.ia] + 15) / 16) *
                            ((g.ext[bp.ib] + 15) / 16);
    (void)units16;  // 16 x 8 measured slower on config 3 (more L2 traffic); keep 16 x 16
  }
  BlockSpec bs;
  if (bp.ia >= 0) {
    bs.ext_ia = g.ext[bp.ia];
    bs.a_ia = g.a_stride[bp.ia];
    bs.out_ia = g.out_stride[bp.ia];
  }
  if (bp.ib >= 0) {
    bs.ext_ib = g.ext[bp.ib];
    bs.b_ib = g.b_stride[bp.ib];
    bs.out_ib = g.out_stride[bp.ib];
  }
  bs.nbp = (bs.ext_ia + P - 1) / P;
  bs.nbq = (bs.ext_ib + Q - 1) / Q;
  // 32-slot units (2 CTAs per SM) for the plain GEMM fold
  const bool slots32 = gemm && p.s % 32 == 0 && g_gemm_slots != 64;
  bs.chunks = coltree ? (p.s / 16) / (slots32 ? 2 : 4)
              : gemm ? p.s / (slots32 ? 32 : kGemmSlots)
                     : (p.s + kBlockThreads - 1) / kBlockThreads;
  bs.units = pr.g.groups * bs.chunks * bs.nbp * bs.nbq;
  bs.div_nbq = make_div64(static_cast<uint64_t>(bs.nbq));
  bs.div_nbp = make_div64(static_cast<uint64_t>(bs.nbp));
  bs.div_chunks = make_div64(static_cast<uint64_t>(bs.chunks));
  if (slots32 && !coltree && g_gemm_tma && launch_gemm_tma(c, p, pr, bs, ta, tb, tout)) {
    return;
  } else if (slots32) {
    const size_t smem = static_cast<size_t>(kGemmStages) * kGemmPair * (kGemmBlk + Q) * 32 * sizeof(double);
    auto k = coltree ? fold_gemm_kernel<16, true, 32>
                     : (Q == 8 ? fold_gemm_kernel<8, false, 32> : fold_gemm_kernel<16, false, 32>);
    set_smem_attr((const void*)k, smem);
    const int threads = Q == 8 ? 128 : 256;
    const int grid = grid_for(c, (const void*)k, threads, smem, bs.units);
    k<<<grid, threads, smem, c.stream>>>(to_fold(pr), bs, ta, tb, tout);
    post_launch(c, coltree ? "gemm fold + column tree kernel (32-slot units)" : "gemm fold kernel (32-slot units)");
  } else if (gemm) {
    const size_t smem =
        static_cast<size_t>(kGemmStages) * kGemmPair * (kGemmBlk + Q) * kGemmSlots * sizeof(double);
    const void* k = coltree ? (const void*)fold_gemm_kernel<16, true>
                            : (Q == 16 ? (const void*)fold_gemm_kernel<16, false>
                                       : (const void*)fold_gemm_kernel<8, false>);
    set_smem_attr((const void*)k, smem);
    const int threads = Q == 16 ? 512 : 256;
    const int grid = grid_for(c, k, threads, smem, bs.units);
    if (coltree)
      fold_gemm_kernel<16, true><<<grid, threads, smem, c.stream>>>(to_fold(pr), bs, ta, tb, tout);
    else if (Q == 16)
      fold_gemm_kernel<16, false><<<grid, threads, smem, c.stream>>>(to_fold(pr), bs, ta, tb, tout);
    else
      fold_gemm_kernel<8, false><<<grid, threads, smem, c.stream>>>(to_fold(pr), bs, ta, tb, tout);
    post_launch(c, coltree ? "gemm fold + column tree kernel" : "gemm fold kernel");
  } else if (P == 8 && Q == 8)
    run_blocked<HAS_B, 8, 8>(c, pr, bs, ta, tb, tout);
  else if (P == 8)
    run_blocked<HAS_B, 8, 1>(c, pr, bs, ta, tb, tout);
  else
    run_blocked<HAS_B, 1, 8>(c, pr, bs, ta, tb, tout);
}

// Phase-1 fold: blocked when the product has a broadcast structure to exploit.
template <bool HAS_B>
void launch_fold_best(const LaunchCtx& c, const GroupParams& p, const double* ta,
                      const double* tb, double* tout) {
  const BlockPlan bp = block_plan(p.g, HAS_B);
  bool blocked = HAS_B && (bp.ia >= 0 || bp.ib >= 0) && p.ops[0].y > 1 && forced_path() != 3;
  if (blocked && (bp.ia < 0 || bp.ib < 0)) {
    // one broadcast dim: the blocked kernel's 256-thread units (8 groups x 256
    // slots) must still cover every SM twice, else the plain fold has more
    // loads in flight (config 2: 24 -> ~8 us)
    const int64_t e = p.g.ext[bp.ia >= 0 ? bp.ia : bp.ib];
    const int64_t units = (p.g.groups / e) * ((e + 7) / 8) * ((p.s + kBlockThreads - 1) / kBlockThreads);
    if (units < 2 * static_cast<int64_t>(c.sm_count)) blocked = false;
  }
  if (blocked)
    launch_fold_blocked<HAS_B>(c, p, bp, ta, tb, tout);
  else
    launch_fold<HAS_B>(c, p, ta, tb, tout);
}

template <int VMAX, bool HAS_B, bool VEC>
void run_pow2(const LaunchCtx& c, const GroupParams& p, int threads, size_t smem,
              const double* ta, const double* tb, double* tout) {
  auto k = group_pow2_kernel<VMAX, HAS_B, VEC>;
  set_smem_attr((const void*)k, smem);
  const int grid = grid_for(c, (const void*)k, threads, smem, p.g.groups);
  k<<<grid, threads, smem, c.stream>>>(p, ta, tb, tout);
  post_launch(c, "group pow2 kernel");
}

template <bool HAS_B, bool VEC>
void dispatch_pow2(const LaunchCtx& c, const GroupParams& p, int threads, int vmax, size_t smem,
                   const double* ta, const double* tb, double* tout) {
  switch (vmax) {
    case 1: run_pow2<1, HAS_B, VEC>(c, p, threads, smem, ta, tb, tout); break;
    case 2: run_pow2<2, HAS_B, VEC>(c, p, threads, smem, ta, tb, tout); break;
    case 4: run_pow2<4, HAS_B, VEC>(c, p, threads, smem, ta, tb, tout); break;
    case 8: run_pow2<8, HAS_B, VEC>(c, p, threads, smem, ta, tb, tout); break;
    case 16: run_pow2<16, HAS_B, VEC>(c, p, threads, smem, ta, tb, tout); break;
    default: run_pow2<32, HAS_B, VEC>(c, p, threads, smem, ta, tb, tout); break;
  }
}

template <int VMAX, bool HAS_B>
void run_tma(const LaunchCtx& c, const GroupParams& p, const double* ta, const double* tb,
             double* tout) {
  const bool b_stream = HAS_B && p.g.bstep != 0;
  const size_t stage_bytes = static_cast<size_t>(kTmaChunk) * sizeof(double) * (b_stream ? 2 : 1);
  const size_t tile_bytes = static_cast<size_t>(p.s) * sizeof(double);
  const size_t avail = c.smem_optin - tile_bytes;
  int nstages = static_cast<int>(avail / (stage_bytes + 16));
  nstages = std::min(nstages, 12);
  if (nstages < 2) invalid_argument("TMA path needs two ring stages");
  const size_t smem = tile_bytes + nstages * (stage_bytes + 16);
  auto k = group_tma_kernel<VMAX, HAS_B>;
  set_smem_attr((const void*)k, smem);
  const int grid = grid_for(c, (const void*)k, kTmaThreads, smem, p.g.groups);
  k<<<grid, kTmaThreads, smem, c.stream>>>(p, ta, tb, tout, nstages);
  post_launch(c, "group tma kernel");
}

template <bool HAS_B>
void run_tma_win(const LaunchCtx& c, const GroupParams& p, int halo, const double* ta,
                 const double* tb, double* tout) {
  const bool b_stream = HAS_B && p.g.bstep != 0;
  const size_t stage_bytes = static_cast<size_t>(kTmaChunk) * sizeof(double) * (b_stream ? 2 : 1);
  const size_t fixed = (3 * static_cast<size_t>(kTmaChunk) + ((2 * halo + 15) / 16) * 16) * sizeof(double);
  int nstages = static_cast<int>((c.smem_optin - fixed) / (stage_bytes + 16));
  nstages = std::min(nstages, 16);
  if (nstages < 2) invalid_argument("window path needs two ring stages");
  const size_t smem = fixed + nstages * (stage_bytes + 16);
  auto k = group_tma_win_kernel<HAS_B>;
  set_smem_attr((const void*)k, smem);
  const int grid = grid_for(c, (const void*)k, kTmaThreads, smem, p.g.groups);
  k<<<grid, kTmaThreads, smem, c.stream>>>(p, ta, tb, tout, nstages, halo);
  post_launch(c, "group tma window kernel");
}

template <bool HAS_B>
void dispatch_tma(const LaunchCtx& c, const GroupParams& p, const double* ta, const double* tb,
                  double* tout) {
  const int64_t v = p.s / kTmaConsumers;
  if (v <= 4)
    run_tma<4, HAS_B>(c, p, ta, tb, tout);
  else if (v <= 8)
    run_tma<8, HAS_B>(c, p, ta, tb, tout);
  else if (v <= 16)
    run_tma<16, HAS_B>(c, p, ta, tb, tout);
  else
    run_tma<32, HAS_B>(c, p, ta, tb, tout);
}

// Tree-only passes (phase 2), register-resident.  kind 1 = column-local (in
// place on OUT), kind 2 = row-shift (reads the folded tiles from a separate
// buffer, writes OUT); 0 = none applies.
// TT_TREE_SMEM=1 selects the whole-tile shared-memory tree pass (kind 3)
// for any eligible schedule.  Correct for any rotations, but measured slower
// than the column / row passes on config 3 (chain 116 vs 102 us: two 64 KiB
// CTAs per SM leave too few loads in flight), so it is opt-in.
const int g_tree_smem = [] {
  const char* e = std::getenv("TT_TREE_SMEM");
  return e ? std::atoi(e) : 0;
}();

// rows per warp of the wide-halo row tree (TT_ROW_ROWS = 16 / 32 / 64)
const int g_row_rows = [] {
  const char* e = std::getenv("TT_ROW_ROWS");
  return e ? std::atoi(e) : 16;
}();

struct TreePass {
  int kind = 0;
  int hr = 0;
  int64_t stride0 = 0, t = 0;
  bool back = false;  // rotations by -e*stride0 (mirrored kernels)
};

TreePass plan_tree_pass(const GroupParams& p2, int64_t s, size_t smem_optin) {
  TreePass tp;
  const int L = p2.nlevels;
  if (L < 1 || L > 8) return tp;
  // whole-tile shared-memory tree: any rotations, tile <= 64 KiB (>= 3 CTAs/SM)
  if (g_tree_smem && (s == 16 * kTreeThreads || s == 32 * kTreeThreads) &&
      static_cast<size_t>(s) * sizeof(double) <= smem_optin) {
    tp.kind = 3;
    tp.t = int64_t{1} << L;
    return tp;
  }
  // forward levels r_i = stride0 * 2^i, or backward ones r_i = s - stride0 * 2^i
  int64_t d[8];
  bool fwd = true, bwd = true;
  for (int i = 0; i < L; ++i) {
    fwd = fwd && p2.rots[i] == p2.rots[0] << i;
    bwd = bwd && p2.rots[i] > 0 && s - p2.rots[i] == (s - p2.rots[0]) << i;
  }
  if (!fwd && !bwd) return tp;
  tp.back = !fwd;
  for (int i = 0; i < L; ++i) d[i] = tp.back ? s - p2.rots[i] : p2.rots[i];
  const int64_t stride0 = d[0];
  const int64_t t = int64_t{1} << L;
  tp.stride0 = stride0;
  tp.t = t;
  if (t * stride0 == s && t <= 32) {
    tp.kind = 1;
    return tp;
  }
  if (s % (32 * 16) != 0) return tp;
  int64_t reach = 0;
  for (int i = 0; i < L; ++i) {
    if (!(d[i] < 32 || (d[i] % 32 == 0 && d[i] / 32 <= 16 && ((d[i] / 32) & (d[i] / 32 - 1)) == 0)))
      return tp;
    reach += d[i];
  }
  const int hr = static_cast<int>((reach + 31) / 32);
  if (hr > 16) return tp;
  tp.kind = 2;
  tp.hr = hr;
  return tp;
}

void run_tree_pass(const LaunchCtx& c, const TreePass& tp, const GroupParams& p2, int64_t n_tiles,
                   int64_t s, const double* folded, double* tout) {
  if (tp.kind == 3) {  // in place: folded == tout
    int lv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < p2.nlevels; ++i) lv[i] = static_cast<int>(p2.rots[i]);
    const size_t smem = static_cast<size_t>(s) * sizeof(double);
    const void* k = s == 32 * kTreeThreads ? (const void*)smem_tree_kernel<32>
                                           : (const void*)smem_tree_kernel<16>;
    set_smem_attr(k, smem);
    const int grid = grid_for(c, k, kTreeThreads, smem, n_tiles);
    const int4 lv0 = make_int4(lv[0], lv[1], lv[2], lv[3]), lv1 = make_int4(lv[4], lv[5], lv[6], lv[7]);
    if (s == 32 * kTreeThreads)
      smem_tree_kernel<32><<<grid, kTreeThreads, smem, c.stream>>>(tout, n_tiles, p2.nlevels, lv0, lv1);
    else
      smem_tree_kernel<16><<<grid, kTreeThreads, smem, c.stream>>>(tout, n_tiles, p2.nlevels, lv0, lv1);
    post_launch(c, "shared-memory tree pass");
    return;
  }
  if (tp.kind == 1) {  // column-local; folded may equal tout
    const int64_t stride0 = tp.stride0;
    const uint64_t total = static_cast<uint64_t>(n_tiles) * stride0;
    const FastDiv64 cd = make_div64(static_cast<uint64_t>(stride0));
    const int64_t work = static_cast<int64_t>((total + 255) / 256);
#define TT_COL(TV, BK)                                                                       \
  {                                                                                         \
    const int grid = grid_for(c, (const void*)col_tree_kernel<TV, BK>, 256, 0, work);       \
    col_tree_kernel<TV, BK><<<grid, 256, 0, c.stream>>>(folded, tout, n_tiles, stride0, s, cd); \
  }
#define TT_COL_T(BK)              \
  switch (tp.t) {                 \
    case 2: TT_COL(2, BK) break;   \
    case 4: TT_COL(4, BK) break;   \
    case 8: TT_COL(8, BK) break;   \
    case 16: TT_COL(16, BK) break; \
    default: TT_COL(32, BK) break; \
  }
    if (tp.back) {
      TT_COL_T(true)
    } else {
      TT_COL_T(false)
    }
#undef TT_COL_T
#undef TT_COL
    post_launch(c, "column tree pass");
    return;
  }
  const int L = p2.nlevels;
  int lv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < L; ++i) lv[i] = static_cast<int>(tp.back ? s - p2.rots[i] : p2.rots[i]);
  const int4 lv0 = make_int4(lv[0], lv[1], lv[2], lv[3]);
  const int4 lv1 = make_int4(lv[4], lv[5], lv[6], lv[7]);
  auto row = [&](auto hr_c, auto r_c) {
    constexpr int HR = decltype(hr_c)::value, RR = decltype(r_c)::value;
    const int64_t work = (n_tiles * (s / 32 / RR) + 7) / 8;
    if (tp.back) {
      const int grid = grid_for(c, (const void*)row_tree_kernel<HR, RR, true>, 256, 0, work);
      row_tree_kernel<HR, RR, true><<<grid, 256, 0, c.stream>>>(folded, tout, n_tiles, s, L, lv0, lv1);
    } else {
      const int grid = grid_for(c, (const void*)row_tree_kernel<HR, RR, false>, 256, 0, work);
      row_tree_kernel<HR, RR, false><<<grid, 256, 0, c.stream>>>(folded, tout, n_tiles, s, L, lv0, lv1);
    }
  };
  using I1 = std::integral_constant<int, 1>;
  using I8 = std::integral_constant<int, 8>;
  using I16 = std::integral_constant<int, 16>;
  using I32 = std::integral_constant<int, 32>;
  using I64 = std::integral_constant<int, 64>;
  if (tp.hr <= 1)
    row(I1{}, I16{});
  else if (tp.hr <= 8)
    row(I8{}, I16{});
  else if (g_row_rows == 32 && s % (32 * 32) == 0)  // 32 rows per warp: 1.5x halo reads, not 2x
    row(I16{}, I32{});
  else if (g_row_rows == 64 && s % (32 * 64) == 0)
    row(I16{}, I64{});
  else
    row(I16{}, I16{});
  post_launch(c, "row tree pass");
}

template <bool HAS_B>
void launch_program_impl(const LaunchCtx& c, const Program& prog, const GroupSpec& g, int64_t s,
                         const double* ta, const double* tb, double* tout) {
  GroupParams p = make_group_params(prog, g, s);
  if (g.groups == 0) return;
  const size_t tile_bytes = static_cast<size_t>(s) * sizeof(double);
  // 1) No in-tile schedule: the fold is the whole program.
  if (prog.ops.size() == 1 && prog.ops[0].kind == GOP_FOLD && prog.ops[0].dst == BUF_OUT) {
    launch_fold_best<HAS_B>(c, p, ta, tb, tout);
    return;
  }
  const BlockPlan bplan = block_plan(g, HAS_B);
  const bool matmul_like = HAS_B && bplan.ia >= 0 && bplan.ib >= 0;
  // 2) Fast paths: fold + power-of-two rotate-and-sum in one pass.
  const int force = forced_path();
  const int threads = static_cast<int>(std::min<int64_t>(512, ((s + 31) / 32) * 32));
  const int64_t v_needed = (s + threads - 1) / threads;
  const bool pow2_s = (s & (s - 1)) == 0;
  if (prog.simple_pow2 && tile_bytes <= c.smem_optin && v_needed <= 32 && force != 3) {
    int vmax = 1;
    while (vmax < v_needed) vmax *= 2;
    p.nlevels = static_cast<int>(prog.ops.size()) - 1;
    for (int i = 0; i < p.nlevels; ++i) p.rots[i] = prog.ops[i + 1].x;
    const bool vec = (s % 2 == 0) && aligned16(ta) && (!HAS_B || aligned16(tb));
    const bool tma_ok = pow2_s && s % kTmaChunk == 0 && s / kTmaConsumers <= 32 && aligned16(ta) &&
                        (!HAS_B || aligned16(tb)) && aligned16(tout) &&
                        tile_bytes + 2 * (2 * kTmaChunk * sizeof(double) + 16) <= c.smem_optin &&
                        force != 2;
    // No fold (one input tile per group, e.g. replicate_dim) with a register
    // tree pass available: read the input tiles directly, no copy and no
    // whole-tile shared-memory tree (replicate schedules are backward
    // rotations: the mirrored row / column kernels)
    if (!HAS_B && prog.ops[0].y == 1 && prog.ops[0].x == 0 && force == 0) {
      bool identity = true;
      int64_t rm = 1;
      for (int i = g.nd - 1; i >= 0; --i) {
        identity = identity && g.out_stride[i] == rm && g.a_stride[i] == rm;
        rm *= g.ext[i];
      }
      const TreePass tdirect = identity ? plan_tree_pass(p, s, c.smem_optin) : TreePass{};
      if ((tdirect.kind == 1 || tdirect.kind == 2) && (tdirect.kind == 1 || ta != tout)) {
        run_tree_pass(c, tdirect, p, g.groups, s, ta, tout);
        return;
      }
    }
    // Too few groups to occupy every SM: fold over the whole grid first
    // (phase 1, into OUT), then run the schedule on OUT in place (phase 2).
    const int64_t per_sm = std::max<int64_t>(1, static_cast<int64_t>(c.smem_optin / (tile_bytes + 1024)));
    // ...unless the whole reduction is tiny (< 2^20 product slots): then one
    // fused launch beats two (small ops are launch-latency bound; config 1)
    const bool tiny = g.groups * prog.ops[0].y * s < (int64_t{1} << 20);
    if ((g.groups < static_cast<int64_t>(c.sm_count) * std::min<int64_t>(per_sm, 4) ||
         (matmul_like && force != 1 && force != 2)) &&
        prog.ops[0].y > 1 && !(tiny && force == 0)) {
      // phase 2 plan first: the row-shift pass needs the folded tiles in a
      // separate buffer, so phase 1 then folds into session scratch
      TreePass tpass;
      if (force == 0 || force == 4) tpass = plan_tree_pass(p, s, c.smem_optin);
      double* fold_dst = tout;
      if (tpass.kind == 2)
        fold_dst = c.scratch(c.scratch_owner, static_cast<size_t>(g.groups) * tile_bytes);
      // fused column tree: correct, but its 32-byte column segments make the
      // operand stream request-bound (c3 stage 1: 107 us vs 57 + 10 us unfused),
      // so it is only taken when forced (TT_KERNEL_PATH=window is reused as the knob)
      const bool fuse_col = force == 4 && HAS_B && matmul_like && tpass.kind == 1 && tpass.t == 16 &&
                            tpass.stride0 % 4 == 0 && s % kGemmSlots == 0 && aligned16(ta) &&
                            aligned16(tb);
      if (fuse_col) {
        launch_fold_blocked<HAS_B>(c, p, bplan, ta, tb, tout, true);
        return;
      }
      if (tpass.kind != 0) {
        launch_fold_best<HAS_B>(c, p, ta, tb, fold_dst);
        run_tree_pass(c, tpass, p, g.groups, s, fold_dst, tout);
        return;
      }
      launch_fold_best<HAS_B>(c, p, ta, tb, tout);
      // phase 2 reads its group's folded tile from OUT: a = out tile index
      GroupParams p2 = p;
      for (int i = 0; i < g.nd; ++i) {
        p2.g.a_stride[i] = g.out_stride[i];
        p2.g.b_stride[i] = 0;
      }
      p2.g.astep = 0;
      p2.g.bstep = 0;
      p2.ops[0].x = 0;
      p2.ops[0].y = 1;
      // tree-only pass: the register-tree kernel (several CTAs per SM overlap
      // load, tree and store) unless the tile is too big for two CTAs per SM
      const bool regs2 = force == 2;  // the TMA kernel measured faster for tree-only passes
      if (tma_ok && !regs2)
        dispatch_tma<false>(c, p2, tout, nullptr, tout);
      else if (s % 2 == 0 && aligned16(tout))
        dispatch_pow2<false, true>(c, p2, threads, vmax, tile_bytes, tout, nullptr, tout);
      else
        dispatch_pow2<false, false>(c, p2, threads, vmax, tile_bytes, tout, nullptr, tout);
      return;
    }
    int64_t halo = 0;
    for (int i = 0; i < p.nlevels; ++i) halo += p.rots[i];
    const bool win_ok = tma_ok && halo <= kTmaChunk && (force == 0 || force == 4);
    if (win_ok)
      run_tma_win<HAS_B>(c, p, static_cast<int>(halo), ta, tb, tout);
    else if (tma_ok)
      dispatch_tma<HAS_B>(c, p, ta, tb, tout);
    else if (vec)
      dispatch_pow2<HAS_B, true>(c, p, threads, vmax, tile_bytes, ta, tb, tout);
    else
      dispatch_pow2<HAS_B, false>(c, p, threads, vmax, tile_bytes, ta, tb, tout);
    return;
  }
  // 3) Generic interpreter.
  const int gthreads = static_cast<int>(std::min<int64_t>(512, ((s + 31) / 32) * 32));
  const size_t phys = static_cast<size_t>(prog.nbuf + 1) * tile_bytes;
  if (prog.nbuf + 1 > 16) invalid_argument("reduction schedule needs too many scratch tiles");
  double* scratch = nullptr;
  size_t smem = 0;
  auto k = group_generic_kernel<HAS_B>;
  if (phys <= c.smem_optin) {
    p.use_smem = 1;
    smem = phys;
    set_smem_attr((const void*)k, smem);
  }
  const int grid = grid_for(c, (const void*)k, gthreads, smem, g.groups);
  if (!p.use_smem) scratch = c.scratch(c.scratch_owner, phys * static_cast<size_t>(grid));
  k<<<grid, gthreads, smem, c.stream>>>(p, ta, tb, tout, scratch);
  post_launch(c, "group generic kernel");
}

}  // namespace

void set_kernel_path(int path) { g_forced_path.store(path, std::memory_order_relaxed); }
int kernel_path() { return forced_path(); }

void launch_group_program(const LaunchCtx& c, const Program& prog, const GroupSpec& g, int64_t s,
                          const double* ta, const double* tb, double* tout) {
  if (tb != nullptr)
    launch_program_impl<true>(c, prog, g, s, ta, tb, tout);
  else
    launch_program_impl<false>(c, prog, g, s, ta, tb, tout);
}

}  // namespace ttb

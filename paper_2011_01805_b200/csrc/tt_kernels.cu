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
#include "tt_pdl.cuh"

namespace ttb {

// TT_PDL=0: launch without programmatic stream serialization (tt_pdl.cuh)
int pdl_enabled() {
  static const int on = [] {
    const char* e = std::getenv("TT_PDL");
    return e ? std::atoi(e) : 1;
  }();
  return on;
}
int pdl_oversub() {
  static const int k = [] {
    const char* e = std::getenv("TT_PDL_OVERSUB");
    return e ? std::max(1, std::atoi(e)) : 8;
  }();
  return k;
}

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
std::map<const void*, size_t> g_static_smem;

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

// one_wave: the grid must stay co-resident (dependency waits) or schedules its
// own work dynamically -- never oversubscribed
int grid_for(const LaunchCtx& c, const void* kernel, int threads, size_t smem, int64_t work,
             bool one_wave = false) {
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
  // Under PDL a grid is dispatched while its predecessor still holds most SMs:
  // the SMs that free up first would take all of a one-wave persistent grid's
  // CTAs.  Several waves' worth of CTAs keep the grid-stride loops balanced.
  const int64_t waves = per_sm > 1 && !one_wave && pdl_would_allow(c, kernel, threads, smem) ? pdl_oversub() : 1;
  const int64_t cap = static_cast<int64_t>(c.sm_count) * per_sm * waves;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cap, work)));
}

}  // namespace

// A kernel that keeps no shared memory of its own runs on L1 cache; dispatched
// early onto an SM whose shared-memory carve-out a predecessor still holds
// (GEMM fold, TMA group kernels: ~200 KiB per SM), it is left with a few KiB
// of L1 and measured slower (config 3 row tree 12.2 -> 15.2 us).  Such a
// launch after a shared-memory-heavy one is made without the PDL attribute:
// it then starts on drained SMs, which reconfigure their carve-out.
namespace {
std::mutex g_pdl_mu;
// each stream's last launch: its per-SM shared memory and whether it releases
// its dependents at entry (early) or only at CTA exit
struct PdlPrev {
  size_t smem = 0;
  bool early = false;
};
std::map<cudaStream_t, PdlPrev> g_pdl_last;

// per-CTA shared memory (dynamic + static) and resident CTAs per SM, cached
// per (device, kernel, block size, dynamic smem) like grid_for's occupancy
std::pair<size_t, size_t> smem_footprint(const LaunchCtx& c, const void* kernel, int threads,
                                         size_t dyn_smem) {
  std::lock_guard<std::mutex> lk(g_launch_cache_mu);
  auto it = g_static_smem.find(kernel);
  if (it == g_static_smem.end()) {
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kernel) != cudaSuccess) fa.sharedSizeBytes = 0;
    it = g_static_smem.emplace(kernel, fa.sharedSizeBytes).first;
  }
  const OccKey key{c.device, kernel, threads, dyn_smem};
  auto oc = g_occupancy.find(key);
  if (oc == g_occupancy.end()) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, dyn_smem) != cudaSuccess)
      per_sm = 1;
    oc = g_occupancy.emplace(key, per_sm).first;
  }
  return {dyn_smem + it->second, static_cast<size_t>(std::max(1, oc->second))};
}

bool pdl_rule(size_t prev_per_sm, size_t cta) {
  return !(prev_per_sm >= (size_t{96} << 10) && cta <= (size_t{16} << 10));
}
}  // namespace

// peek: would a launch of `kernel` on c.stream be dispatched early (PDL
// attribute, predecessor releasing at entry)?
bool pdl_would_allow(const LaunchCtx& c, const void* kernel, int threads, size_t dyn_smem) {
  if (!pdl_enabled()) return false;
  const size_t cta = smem_footprint(c, kernel, threads, dyn_smem).first;
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  auto it = g_pdl_last.find(c.stream);
  const PdlPrev prev = it == g_pdl_last.end() ? PdlPrev{} : it->second;
  return prev.early && pdl_rule(prev.smem, cta);
}

// A grid smaller than one full wave is launched without the attribute too:
// dispatched early it would be packed onto the first SMs to free up (config 4's
// 512-CTA layer-2 fold on ~70 SMs: 22 -> 28 us) instead of spread over all.
void pdl_note_late_release(const LaunchCtx& c) {
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  g_pdl_last[c.stream] = PdlPrev{0, false};  // nothing lands on its SMs early
}

bool pdl_allow(const LaunchCtx& c, const void* kernel, int threads, size_t dyn_smem, int64_t grid) {
  if (!pdl_enabled()) return false;
  const auto [cta, per_sm] = smem_footprint(c, kernel, threads, dyn_smem);
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  if (g_pdl_last.size() > 4096) g_pdl_last.clear();  // streams come and go; a forgotten one costs one overlap
  PdlPrev& prev = g_pdl_last[c.stream];
  // a predecessor that releases only at exit cannot have this grid placed early
  const bool allow = !prev.early || (pdl_rule(prev.smem, cta) &&
                                     grid >= static_cast<int64_t>(c.sm_count) * static_cast<int64_t>(per_sm));
  prev = PdlPrev{cta * per_sm, true};
  return allow;
}

namespace {

void count_launch(const LaunchCtx& c) {
  if (c.launches) ++*c.launches;
}

void post_launch(const LaunchCtx& c, const char* what) {
  count_launch(c);
  check_cuda(cudaGetLastError(), what);
  if (c.release_late) pdl_note_late_release(c);
}

// Device form of an Epilogue (tt_launch.hpp): the add operand's tile for
// output tile l is C + (sum_i coord_i(l) * cst[i]) * s, coordinates of l in
// the row-major output grid (divisors innermost last).
struct EpiDev {
  const double* c = nullptr;
  int nd = 0;
  int square = 0;
  FastDiv64 ext[TT_MAX_RANK];
  int64_t cst[TT_MAX_RANK] = {};
  // clean_unknowns mask (nmask cut dims; power-of-two extents and strides)
  int nmask = 0;
  int msh[kEpiMaskDims] = {}, mdim[kEpiMaskDims] = {};
  int64_t mtm1[kEpiMaskDims] = {}, mt[kEpiMaskDims] = {}, mused[kEpiMaskDims] = {};
};

EpiDev make_epi_dev(const Epilogue& e) {
  EpiDev d;
  d.c = e.c;
  d.square = e.square ? 1 : 0;
  d.nd = e.nd;
  for (int i = 0; i < e.nd; ++i) {
    d.ext[i] = make_div64(static_cast<uint64_t>(e.ext[i]));
    d.cst[i] = e.c_stride[i];
  }
  d.nmask = e.nmask;
  for (int k = 0; k < e.nmask; ++k) {
    d.mdim[k] = e.mask_dim[k];
    d.mt[k] = e.mask_t[k];
    d.mtm1[k] = e.mask_t[k] - 1;
    d.mused[k] = e.mask_used[k];
    int sh = 0;
    while ((int64_t{1} << sh) < e.mask_stride[k]) ++sh;
    d.msh[k] = sh;
  }
  return d;
}

// Per output tile: the add operand's tile and, for the mask, the number of
// used coordinates left in this tile along each cut dim.
struct EpiTile {
  const double* ct;
  int lim[kEpiMaskDims];  // clamped to [0, t]: 32-bit mask arithmetic (slots < 2^31)
};

__device__ __forceinline__ EpiTile epi_tile(const EpiDev& e, uint64_t tile, int64_t s) {
  EpiTile t;
  t.ct = nullptr;
#pragma unroll
  for (int k = 0; k < kEpiMaskDims; ++k) t.lim[k] = 0;
  if (!e.c && !e.nmask) return t;
  int64_t ci = 0;
  for (int i = e.nd - 1; i >= 0; --i) {
    const uint64_t q = fdiv(tile, e.ext[i]);
    const int64_t l = static_cast<int64_t>(tile - q * e.ext[i].d);
    ci += l * e.cst[i];
#pragma unroll
    for (int k = 0; k < kEpiMaskDims; ++k)
      if (k < e.nmask && e.mdim[k] == i) {
        const int64_t left = e.mused[k] - l * e.mt[k];
        t.lim[k] = static_cast<int>(left < 0 ? 0 : (left > e.mt[k] ? e.mt[k] : left));
      }
    tile = q;
  }
  if (e.c) t.ct = e.c + ci * s;
  return t;
}

// clean_unknowns' x * (0 or 1), then tt_add(x, C), then tt_mul(x, x), each
// separately rounded, as the composition, over N values at slots j0 + i * dj.
// One loop per step (uniform branches), so the add's loads issue together.
template <int N>
__device__ __forceinline__ void epi_apply_n(const EpiDev& e, double (&x)[N], const EpiTile& t,
                                            int64_t j0, int64_t dj) {
  if (e.nmask) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int j = static_cast<int>(j0 + i * dj);
      bool ok = true;
#pragma unroll
      for (int k = 0; k < kEpiMaskDims; ++k)
        if (k < e.nmask) ok = ok && ((j >> e.msh[k]) & static_cast<int>(e.mtm1[k])) < t.lim[k];
      x[i] = dmul(x[i], ok ? 1.0 : 0.0);  // Session::mask_mul backend.hpp:145
    }
  }
  if (t.ct) {
    double c[N];
#pragma unroll
    for (int i = 0; i < N; ++i) c[i] = __ldg(t.ct + j0 + i * dj);
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = dadd(x[i], c[i]);
  }
  if (e.square) {
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = dmul(x[i], x[i]);
  }
}

#include "kernels/stream.cuh"
#include "kernels/group.cuh"
#include "kernels/gemm.cuh"
#include "kernels/tree.cuh"
#include "kernels/layers.cuh"
#include "kernels/chain.cuh"

// ---- synthetic input generator (== or_fill_uniform in oracle/tt_oracle.c) ------------

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void fill_uniform_kernel(double* out, uint64_t count, uint64_t key, uint64_t offset,
                                    double lo, double span) {
  pdl_enter();
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
      launch_k(c, pack_kernel<RK, true>, grid, 256, 0, g, dense, tiles, ud);
    else
      launch_k(c, pack_kernel<RK, false>, grid, 256, 0, g, dense, tiles, ud);
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
    launch_k(c, unpack_kernel<RK>, grid, 256, 0, g, tiles, dense, total);
  });
  post_launch(c, "unpack kernel");
}

// TT_EW_CHUNK=0 keeps the per-16-byte elementwise / clean kernels (measurement)
const int g_ew_chunk = [] {
  const char* e = std::getenv("TT_EW_CHUNK");
  return e ? std::atoi(e) : 1;
}();
// TT_EW_HINT=0: no L2 eviction hints in the broadcast elementwise kernel
const int g_ew_hint = [] {
  const char* e = std::getenv("TT_EW_HINT");
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
      launch_k(c, clean_chunk_kernel<RK>, grid, 256, 0, g, in, out, cd);
    });
    post_launch(c, "clean_unknowns chunk kernel");
    return;
  }
  const uint64_t quads = static_cast<uint64_t>((s + 3) / 4);
  const FastDiv64 qd = make_div64(quads);
  const int64_t work = (g.n_tiles * static_cast<int64_t>(quads) + 255) / 256;
  TT_RANK_SWITCH(g.rank, RK, {
    const int grid = grid_for(c, (const void*)clean_kernel<RK>, 256, 0, work);
    launch_k(c, clean_kernel<RK>, grid, 256, 0, g, in, out, qd);
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
    for (int i = 0; i < p.rank; ++i) {
      if (eo[i] > 1 && p.a_stride[i] == 0) q.keep_a = 1;
      if (eo[i] > 1 && p.b_stride[i] == 0) q.keep_b = 1;
    }
    // the L2 hints pay when the broadcast operand's re-reads outgrow the L2
    const bool hint = g_ew_hint && (q.keep_a || q.keep_b) &&
                      p.n_tiles * s * 8 > (int64_t{64} << 20);
    auto run = [&](auto k) {
      const int grid = grid_for(c, (const void*)k, 256, 0, items);
      launch_k(c, k, grid, 256, 0, q, ta, tb, tout, cd);
    };
    // large broadcast op whose innermost visited dim has exactly one broadcasting
    // operand and an even extent: two output tiles per item share that operand's chunk
    // (config 5: X * W 5.66 -> 5.63 ms, W * X / X + W 5.74 -> 5.66 ms; TT_EW_PAIR=0 off).
    // Measured and not kept: visiting up to 2 MiB of consecutive tiles of the last dim
    // inside the broadcast dims (one page per side consumed in one go): 5.63 -> 5.79 ms.
    const int ki = p.rank - 1;
    static const int ew_pair = [] { const char* e = std::getenv("TT_EW_PAIR"); return e ? std::atoi(e) : 1; }();
    if (hint && ew_pair && ki >= 0 && q.ediv[ki].d >= 2 && q.ediv[ki].d % 2 == 0 &&
        (q.a_stride[ki] == 0) != (q.b_stride[ki] == 0) && s % 2 == 0) {
      const bool shared_b = q.b_stride[ki] == 0;
      const int64_t v_in = shared_b ? q.a_stride[ki] : q.b_stride[ki];
      const int64_t o_in = q.o_stride[ki];
      EwParams q2 = q;
      q2.ediv[ki] = make_div32(q.ediv[ki].d / 2);
      q2.a_stride[ki] *= 2;
      q2.b_stride[ki] *= 2;
      q2.o_stride[ki] *= 2;
      q2.n_tiles = p.n_tiles / 2;
      auto run2 = [&](auto k) {
        const int grid = grid_for(c, (const void*)k, 256, 0, items / 2);
        launch_k(c, k, grid, 256, 0, q2, ta, tb, tout, cd, v_in, o_in);
      };
      if (op == TT_OP_ADD) {
        if (shared_b) run2(elementwise_pair_kernel<TT_OP_ADD, true>);
        else run2(elementwise_pair_kernel<TT_OP_ADD, false>);
      } else {
        if (shared_b) run2(elementwise_pair_kernel<TT_OP_MUL, true>);
        else run2(elementwise_pair_kernel<TT_OP_MUL, false>);
      }
      post_launch(c, "elementwise pair kernel");
      return;
    }
    if (op == TT_OP_ADD) {
      if (hint) run(elementwise_chunk_kernel<TT_OP_ADD, true>);
      else run(elementwise_chunk_kernel<TT_OP_ADD, false>);
    } else {
      if (hint) run(elementwise_chunk_kernel<TT_OP_MUL, true>);
      else run(elementwise_chunk_kernel<TT_OP_MUL, false>);
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
    launch_k(c, elementwise_kernel<OPV, VECV>, grid, 256, 0, p, ta, tb, tout, qd);       \
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
    launch_k(c, fold_range_kernel<HB, IN>, grid, 256, 0, p, ta, tb, init, acc, total, pd);  \
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
    launch_k(c, batch_affine_smem_kernel, grid, 256, 0, in, s, n_out, block, items, row_ptr, src, w,
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
      launch_k(c, batch_affine_blocked_kernel<8, 2>, grid, 256, 0, in, s, n_out, block, work, row_ptr,
                                                                    src, w, bias, out, make_div64(per));
    } else {
      const int grid = grid_for(c, (const void*)batch_affine_blocked_kernel<8, 1>, 256, 0, nb);
      launch_k(c, batch_affine_blocked_kernel<8, 1>, grid, 256, 0, in, s, n_out, block, work, row_ptr,
                                                                    src, w, bias, out, make_div64(per));
    }
    post_launch(c, "batch affine blocked kernel");
    return;
  }
  const int grid = grid_for(c, (const void*)batch_affine_kernel, 256, 0, (total + 255) / 256);
  launch_k(c, batch_affine_kernel, grid, 256, 0, in, s, total, row_ptr, src, w, bias, out,
                                                   make_div64(static_cast<uint64_t>(s)));
  post_launch(c, "batch affine kernel");
}

void launch_binary_flat(const LaunchCtx& c, int op, const double* a, const double* b, double* out,
                        int64_t count) {
  if (count <= 0) return;
  const int64_t work = (count + 255) / 256;
  if (op == TT_OP_ADD) {
    const int grid = grid_for(c, (const void*)binary_flat_kernel<TT_OP_ADD>, 256, 0, work);
    launch_k(c, binary_flat_kernel<TT_OP_ADD>, grid, 256, 0, a, b, out, count);
  } else {
    const int grid = grid_for(c, (const void*)binary_flat_kernel<TT_OP_MUL>, 256, 0, work);
    launch_k(c, binary_flat_kernel<TT_OP_MUL>, grid, 256, 0, a, b, out, count);
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
    launch_k(c, rotate_aligned_kernel<16>, grid, 256, 0, in, out, s, r, units, make_div64(per_tile));
    post_launch(c, "rotate aligned kernel");
    return;
  }
  const uint64_t chunks = static_cast<uint64_t>((s + kRotChunk - 1) / kRotChunk);
  const uint64_t items = chunks * static_cast<uint64_t>(n_tiles);
  if (s >= 1024) {  // chunked: whole 4096-slot items (small tiles keep one slot per thread)
    const int grid = grid_for(c, (const void*)rotate_chunk_kernel, 256, 0, static_cast<int64_t>(items));
    launch_k(c, rotate_chunk_kernel, grid, 256, 0, in, out, s, r, items, make_div64(chunks));
    post_launch(c, "rotate chunk kernel");
    return;
  }
  const int grid = grid_for(c, (const void*)rotate_kernel, 256, 0, (total + 255) / 256);
  launch_k(c, rotate_kernel, grid, 256, 0, in, out, s, r, total, make_div64(s));
  post_launch(c, "rotate kernel");
}

void launch_fill_uniform(const LaunchCtx& c, double* out, int64_t count, uint64_t seed,
                         int64_t offset, double lo, double hi) {
  if (count <= 0) return;
  const int grid = grid_for(c, (const void*)fill_uniform_kernel, 256, 0, (count + 255) / 256);
  launch_k(c, fill_uniform_kernel, grid, 256, 0, out, count, host_splitmix64(seed), offset, lo,
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

// Few-group folds stream their operands through a cp.async ring
// (fold_ring_kernel) when the streamed operand's bytes (groups x fold steps x
// tile: the per-group operand; a broadcast second operand is re-read from L2 and
// not counted) exceed half the device L2: config 4's layer-2 fold (100 MiB) 36 ->
// 22 us; an L2-resident one (config 2, 32 MiB) is ~0.5 us faster without.
// TT_FOLD_RING=0 / 1 forces it off / on; "on" still needs the ring's layout:
// s % 256 == 0, more than one fold step, 16-byte aligned operands (otherwise
// the plain fold runs).
const int g_fold_ring = [] {
  const char* e = std::getenv("TT_FOLD_RING");
  return e ? std::atoi(e) : -1;
}();

// TT_FOLD_BLK=0: no group-blocked ring fold (parity variant)
const int g_fold_blk = [] {
  const char* e = std::getenv("TT_FOLD_BLK");
  return e ? std::atoi(e) : 1;
}();

// Small few-group fold with one operand shared along a group dim (fold_ring_blk_kernel;
// config 2's matvec: the fold 6.8 -> 5.5 us, the call 12.3 -> 10.7 us).  Folds large
// enough for fold_ring_kernel stay there: config 4's second layer measured the same
// either way (22.5 us: bound by DRAM, including the write-back of the activations the
// pass before it left in L2, not by the L2 re-reads of the shared operand).
template <int Q, int T, bool SHARED_A>
void run_fold_ring_blk(const LaunchCtx& c, const GroupParams& p, int d, const double* ta,
                       const double* tb, double* tout) {
  FoldParams f = to_fold(p, c.release_late);
  const int64_t vq = SHARED_A ? f.g.b_stride[d] : f.g.a_stride[d];
  const int64_t oq = f.g.out_stride[d];
  f.g.ext[d] /= Q;
  f.g.out_stride[d] *= Q;
  f.g.a_stride[d] *= Q;
  f.g.b_stride[d] *= Q;
  f.g.groups /= Q;
  f.gdiv[d] = make_div64(static_cast<uint64_t>(f.g.ext[d]));
  const int64_t runs = p.s / (2 * T);
  constexpr size_t smem = static_cast<size_t>(kFoldRing) * (1 + Q) * T * sizeof(double2);
  auto k = fold_ring_blk_kernel<Q, T, SHARED_A>;
  set_smem_attr((const void*)k, smem);
  const int grid = grid_for(c, (const void*)k, T, smem, f.g.groups * runs);
  launch_k(c, k, grid, T, smem, f, ta, tb, tout, make_div64(static_cast<uint64_t>(runs)), vq, oq);
}

bool launch_fold_ring_blk(const LaunchCtx& c, const GroupParams& p, const double* ta,
                          const double* tb, double* tout) {
  const GroupSpec& g = p.g;
  const int64_t s = p.s;
  if (!g_fold_blk || g.astep == 0 || g.bstep == 0 || p.ops[0].y < 2 || s % 256 != 0 ||
      !aligned16(ta) || !aligned16(tb) || !aligned16(tout))
    return false;
  int d = -1;
  bool shared_a = false;
  for (int i = 0; i < g.nd && d < 0; ++i) {
    if (g.ext[i] < 2 || g.ext[i] % 2 != 0 || g.out_stride[i] == 0) continue;
    if (g.a_stride[i] == 0 && g.b_stride[i] > 0) d = i, shared_a = true;
    else if (g.b_stride[i] == 0 && g.a_stride[i] > 0) d = i, shared_a = false;
  }
  if (d < 0) return false;
  // Q = 2 groups per thread, 64-thread CTAs (measured on config 2: Q = 2 5.5 us, Q = 4
  // 5.9 us, scalar fold 6.8 us; 128-thread CTAs the same)
  if (shared_a) run_fold_ring_blk<2, 64, true>(c, p, d, ta, tb, tout);
  else run_fold_ring_blk<2, 64, false>(c, p, d, ta, tb, tout);
  return true;
}

// Returns true when `epi` (the reduction's elementwise tail, may be null) was applied
// in the fold's store; the caller runs it as its own pass otherwise.
template <bool HAS_B>
bool launch_fold(const LaunchCtx& c, const GroupParams& p, const double* ta, const double* tb,
                 double* tout, const Epilogue* epi = nullptr) {
  const int64_t s = p.s;
  bool fused = false;
  // 256 slots per warp when that still gives every SM >= 8 warps; otherwise
  // one slot per thread (small folds are latency bound: more loads in flight)
  const int64_t vec_warps = p.g.groups * ((s / 2 + 127) / 128);
  const bool vec = (s % 2 == 0) && aligned16(ta) && (!HAS_B || aligned16(tb)) && aligned16(tout) &&
                   vec_warps >= 8 * static_cast<int64_t>(c.sm_count);
  if (vec) {
    const uint64_t units = static_cast<uint64_t>((s / 2 + 127) / 128);
    const int64_t work = (p.g.groups * static_cast<int64_t>(units) + 7) / 8;
    const int grid = grid_for(c, (const void*)fold_kernel<HAS_B, true>, 256, 0, work);
    launch_k(c, fold_kernel<HAS_B, true>, grid, 256, 0, to_fold(p, c.release_late), ta, tb, tout, make_div64(units));
  } else if ((g_fold_ring == 1 ||
              (g_fold_ring < 0 && p.g.groups * p.ops[0].y * s * 8 > static_cast<int64_t>(c.l2_bytes / 2))) &&
             s % 256 == 0 && p.ops[0].y > 1 && aligned16(ta) && (!HAS_B || aligned16(tb)) &&
             aligned16(tout)) {
    const int64_t runs = s / 256;
    static const int fuse_epi = [] { const char* e = std::getenv("TT_FOLD_EPI"); return e ? std::atoi(e) : 1; }();
    if (epi != nullptr && epi->active() && epi->nmask == 0 && fuse_epi) {
      // the tail rides on the fold's store: no pass follows, no late release
      const int grid = grid_for(c, (const void*)fold_ring_kernel<HAS_B, true>, 128, 0, p.g.groups * runs);
      launch_k(c, fold_ring_kernel<HAS_B, true>, grid, 128, 0, to_fold(p, false), ta, tb, tout,
               make_div64(static_cast<uint64_t>(runs)), make_epi_dev(*epi));
      fused = true;
    } else {
      const int grid = grid_for(c, (const void*)fold_ring_kernel<HAS_B>, 128, 0, p.g.groups * runs);
      launch_k(c, fold_ring_kernel<HAS_B>, grid, 128, 0, to_fold(p, c.release_late), ta, tb, tout,
               make_div64(static_cast<uint64_t>(runs)), EpiDev{});
    }
  } else if (HAS_B && launch_fold_ring_blk(c, p, ta, tb, tout)) {
    // small fold, few groups sharing one operand: group-blocked ring fold
  } else {
    const int64_t work = (p.g.groups * s + 255) / 256;
    const int grid = grid_for(c, (const void*)fold_kernel<HAS_B, false>, 256, 0, work);
    launch_k(c, fold_kernel<HAS_B, false>, grid, 256, 0, to_fold(p, c.release_late), ta, tb, tout,
                                                           make_div64(static_cast<uint64_t>(s)));
  }
  post_launch(c, "fold kernel");
  return fused;
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

// TT_GEMM_GRID: cap on the TMA GEMM fold's CTA count (measurement knob)
const int g_gemm_grid = [] {
  const char* e = std::getenv("TT_GEMM_GRID");
  return e ? std::atoi(e) : 0;
}();

// TT_GEMM_WAIT: mbarrier wait style of the warp-specialised fold (see the kernel)
const int g_gemm_wait = [] {
  const char* e = std::getenv("TT_GEMM_WAIT");
  return e ? std::atoi(e) : 1;
}();

// The warp-specialised fold releases its dependents at CTA exit (TT_GEMM_LATE=0:
// at entry), so the tree pass after it is PDL-launched -- its launch overlaps
// the fold's end -- without landing early on SMs whose shared-memory carve-out
// the fold still holds: config 3 chain 92.8 -> 88.1 us through the API (graph
// replay unchanged), config 4 130 -> 128 us
const int g_gemm_late = [] {
  const char* e = std::getenv("TT_GEMM_LATE");
  return e ? std::atoi(e) : 1;
}();

// WS: warp-specialised kernel (a producer warp issues the TMA loads)
template <int SL, int kTgSteps, int kTgStages, int SC, int PB = kGemmBlk, bool WS = false>
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
  auto k = [] {
    if constexpr (WS)
      return fold_gemm_ws_kernel<BC, SL, kTgSteps, kTgStages, SC, PB>;
    else
      return fold_gemm_tma_kernel<BC, SL, kTgSteps, kTgStages, SC, PB>;
  }();
  constexpr size_t smem = tg_smem_bytes<BC, SL, kTgSteps, kTgStages, PB>();
  constexpr int threads = (tg_warps<BC, SL, SC, PB>() + (WS ? 1 : 0)) * 32;
  set_smem_attr((const void*)k, smem);
  unsigned int* sched = g_gemm_dynamic ? take_sched_slot(c) : nullptr;
  int grid = grid_for(c, (const void*)k, threads, smem, bs.units, sched != nullptr);
  if (g_gemm_grid > 0) grid = std::min(grid, g_gemm_grid);  // measurement knob
  if constexpr (WS) {
    launch_k(c, k, grid, threads, smem, *reinterpret_cast<const CUtensorMap*>(mapA),
                                         *reinterpret_cast<const CUtensorMap*>(mapB), to_fold(pr, c.release_late || g_gemm_late != 0), bs, ts,
                                         tout, sched, g_gemm_wait);
    if (g_gemm_late) pdl_note_late_release(c);
  } else {
    launch_k(c, k, grid, threads, smem, *reinterpret_cast<const CUtensorMap*>(mapA),
                                         *reinterpret_cast<const CUtensorMap*>(mapB), to_fold(pr, c.release_late), bs, ts,
                                         tout, sched);
  }
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
    case 7: return launch_gemm_tma_sl<16, 4, 3, 4, kGemmBlk, true>(c, p, pr, bs, ta, tb, tout);
    case 8: return launch_gemm_tma_sl<16, 4, 4, 4, kGemmBlk, true>(c, p, pr, bs, ta, tb, tout);
    case 9: return launch_gemm_tma_sl<16, 2, 8, 4, kGemmBlk, true>(c, p, pr, bs, ta, tb, tout);
    case 10: return launch_gemm_tma_sl<16, 4, 2, 4, kGemmBlk, true>(c, p, pr, bs, ta, tb, tout);
    case 1: return launch_gemm_tma_sl<16, 2, 6, 4>(c, p, pr, bs, ta, tb, tout);
    case 2: return launch_gemm_tma_sl<16, 4, 4, 4>(c, p, pr, bs, ta, tb, tout);
    case 3: return launch_gemm_tma_sl<32, 2, 6, 4>(c, p, pr, bs, ta, tb, tout);
    case 4: return launch_gemm_tma_sl<8, 4, 3, 4, 32>(c, p, pr, bs, ta, tb, tout);
    case 5: return launch_gemm_tma_sl<16, 4, 3, 4, 32>(c, p, pr, bs, ta, tb, tout);
    case 6: return launch_gemm_tma_sl<8, 4, 4, 4, 32>(c, p, pr, bs, ta, tb, tout);
    case 11: return launch_gemm_tma_sl<16, 4, 3, 4>(c, p, pr, bs, ta, tb, tout);
    // default: warp-specialised, 4 stages x 4 steps, 3 CTAs per SM (c3 chain
    // 99.6 -> 98.2 us, c4 layer 1 72.7 -> 68.4 us vs case 11)
    default: return launch_gemm_tma_sl<16, 4, 4, 4, kGemmBlk, true>(c, p, pr, bs, ta, tb, tout);
  }
}

template <bool HAS_B, int P, int Q>
void run_blocked(const LaunchCtx& c, const GroupParams& p, const BlockSpec& bs, const double* ta,
                 const double* tb, double* tout) {
  auto k = fold_blocked_kernel<HAS_B, P, Q>;
  const int grid = grid_for(c, (const void*)k, kBlockThreads, 0, bs.units);
  launch_k(c, k, grid, kBlockThreads, 0, to_fold(p, c.release_late), bs, ta, tb, tout);
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
    launch_k(c, k, grid, threads, smem, to_fold(pr, c.release_late), bs, ta, tb, tout);
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
      launch_k(c, fold_gemm_kernel<16, true>, grid, threads, smem, to_fold(pr, c.release_late), bs, ta, tb, tout);
    else if (Q == 16)
      launch_k(c, fold_gemm_kernel<16, false>, grid, threads, smem, to_fold(pr, c.release_late), bs, ta, tb, tout);
    else
      launch_k(c, fold_gemm_kernel<8, false>, grid, threads, smem, to_fold(pr, c.release_late), bs, ta, tb, tout);
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
bool launch_fold_best(const LaunchCtx& c, const GroupParams& p, const double* ta,
                      const double* tb, double* tout, const Epilogue* epi = nullptr) {
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
  if (blocked) {
    launch_fold_blocked<HAS_B>(c, p, bp, ta, tb, tout);
    return false;
  }
  return launch_fold<HAS_B>(c, p, ta, tb, tout, epi);
}

template <int VMAX, bool HAS_B, bool VEC>
void run_pow2(const LaunchCtx& c, const GroupParams& p, int threads, size_t smem,
              const double* ta, const double* tb, double* tout) {
  auto k = group_pow2_kernel<VMAX, HAS_B, VEC>;
  set_smem_attr((const void*)k, smem);
  const int grid = grid_for(c, (const void*)k, threads, smem, p.g.groups);
  launch_k(c, k, grid, threads, smem, p, ta, tb, tout);
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
  launch_k(c, k, grid, kTmaThreads, smem, p, ta, tb, tout, nstages);
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
  launch_k(c, k, grid, kTmaThreads, smem, p, ta, tb, tout, nstages, halo);
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

// TT_ROW_CHAIN=2 / 4: chains of 2 / 4 row blocks per warp with the halo
// carried over (rows read 1.5x / 1.25x instead of 2x) -- measured slower with 4
// (c3 stage-2 tree 12.4 -> 14.5 us: the serial chain leaves fewer loads in
// flight), so off (1) by default
const int g_row_chain = [] {
  const char* e = std::getenv("TT_ROW_CHAIN");
  return e ? std::atoi(e) : 0;
}();

// TT_TREE_TMA = 1 / 2: tree-only passes of GEMM-shaped products on the TMA
// group kernels (1: sliding-window ring when the reach fits one chunk, 2:
// whole tile in shared memory) instead of the register column / row passes
const int g_tree_tma = [] {
  const char* e = std::getenv("TT_TREE_TMA");
  return e ? std::atoi(e) : 0;
}();

// rows per warp of the wide-halo row tree (TT_ROW_ROWS = 16 / 32 / 64): 32
// reads each row 1.5x instead of 2x (config 3 row tree 12.8 -> 11.6 us,
// literal chain 219 -> 210 us, measured with PDL); 64 spills
const int g_row_rows = [] {
  const char* e = std::getenv("TT_ROW_ROWS");
  return e ? std::atoi(e) : 32;
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

// epi (optional, kinds 1 and 2 only): the reduction's elementwise tail, fused
// into the tree pass's store.
void run_tree_pass(const LaunchCtx& c, const TreePass& tp, const GroupParams& p2, int64_t n_tiles,
                   int64_t s, const double* folded, double* tout, const Epilogue* epi = nullptr) {
  const bool fuse = epi != nullptr && epi->active();
  const EpiDev ed = fuse ? make_epi_dev(*epi) : EpiDev{};
  if (tp.kind == 3) {  // in place: folded == tout
    if (fuse) invalid_argument("tree epilogue: the shared-memory pass takes none");
    int lv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < p2.nlevels; ++i) lv[i] = static_cast<int>(p2.rots[i]);
    const size_t smem = static_cast<size_t>(s) * sizeof(double);
    const void* k = s == 32 * kTreeThreads ? (const void*)smem_tree_kernel<32>
                                           : (const void*)smem_tree_kernel<16>;
    set_smem_attr(k, smem);
    const int grid = grid_for(c, k, kTreeThreads, smem, n_tiles);
    const int4 lv0 = make_int4(lv[0], lv[1], lv[2], lv[3]), lv1 = make_int4(lv[4], lv[5], lv[6], lv[7]);
    if (s == 32 * kTreeThreads)
      launch_k(c, smem_tree_kernel<32>, grid, kTreeThreads, smem, tout, n_tiles, p2.nlevels, lv0, lv1);
    else
      launch_k(c, smem_tree_kernel<16>, grid, kTreeThreads, smem, tout, n_tiles, p2.nlevels, lv0, lv1);
    post_launch(c, "shared-memory tree pass");
    return;
  }
  if (tp.kind == 1) {  // column-local; folded may equal tout
    const int64_t stride0 = tp.stride0;
    const uint64_t total = static_cast<uint64_t>(n_tiles) * stride0;
    const FastDiv64 cd = make_div64(static_cast<uint64_t>(stride0));
    const int64_t work = static_cast<int64_t>((total + 255) / 256);
#define TT_COL(TV, BK, EP)                                                                       \
  {                                                                                             \
    const int grid = grid_for(c, (const void*)col_tree_kernel<TV, BK, EP>, 256, 0, work);       \
    launch_k(c, col_tree_kernel<TV, BK, EP>, grid, 256, 0, folded, tout, n_tiles, stride0, s, cd, ed); \
  }
#define TT_COL_T(BK, EP)              \
  switch (tp.t) {                     \
    case 2: TT_COL(2, BK, EP) break;   \
    case 4: TT_COL(4, BK, EP) break;   \
    case 8: TT_COL(8, BK, EP) break;   \
    case 16: TT_COL(16, BK, EP) break; \
    default: TT_COL(32, BK, EP) break; \
  }
    if (tp.back) {
      if (fuse) invalid_argument("tree epilogue: mirrored passes take none");
      TT_COL_T(true, false)
    } else if (fuse) {
      TT_COL_T(false, true)
    } else {
      TT_COL_T(false, false)
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
  // chains of 4 blocks per warp (halo rows carried, not re-read) when that
  // still leaves >= 8 warps per SM
  const int chain = (g_row_chain == 2 || g_row_chain == 4) ? g_row_chain : 1;
  const bool chained = chain > 1 && s % (32 * 16 * chain) == 0 &&
                       n_tiles * (s / 32 / 16 / chain) >= 8 * static_cast<int64_t>(c.sm_count);
  auto launch_chain = [&](auto hr_c, auto c_c) {
    constexpr int HR = decltype(hr_c)::value, CC = decltype(c_c)::value;
    const int64_t work = (n_tiles * (s / 32 / 16 / CC) + 7) / 8;
    if (tp.back) {
      const int grid = grid_for(c, (const void*)row_tree_kernel<HR, 16, true, false, CC>, 256, 0, work);
      launch_k(c, row_tree_kernel<HR, 16, true, false, CC>, grid, 256, 0, folded, tout, n_tiles, s, L, lv0,
                                                                            lv1, ed);
    } else if (fuse) {
      const int grid = grid_for(c, (const void*)row_tree_kernel<HR, 16, false, true, CC>, 256, 0, work);
      launch_k(c, row_tree_kernel<HR, 16, false, true, CC>, grid, 256, 0, folded, tout, n_tiles, s, L, lv0,
                                                                            lv1, ed);
    } else {
      const int grid = grid_for(c, (const void*)row_tree_kernel<HR, 16, false, false, CC>, 256, 0, work);
      launch_k(c, row_tree_kernel<HR, 16, false, false, CC>, grid, 256, 0, folded, tout, n_tiles, s, L, lv0,
                                                                             lv1, ed);
    }
  };
  auto row = [&](auto hr_c, auto r_c) {
    constexpr int HR = decltype(hr_c)::value, RR = decltype(r_c)::value;
    if constexpr (RR == 16) {
      if (chained) {
        if (chain == 2)
          launch_chain(hr_c, std::integral_constant<int, 2>{});
        else
          launch_chain(hr_c, std::integral_constant<int, 4>{});
        return;
      }
    }
    const int64_t work = (n_tiles * (s / 32 / RR) + 7) / 8;
    if (tp.back) {
      if (fuse) invalid_argument("tree epilogue: mirrored passes take none");
      const int grid = grid_for(c, (const void*)row_tree_kernel<HR, RR, true>, 256, 0, work);
      launch_k(c, row_tree_kernel<HR, RR, true>, grid, 256, 0, folded, tout, n_tiles, s, L, lv0, lv1, ed);
    } else if (fuse) {
      const int grid = grid_for(c, (const void*)row_tree_kernel<HR, RR, false, true>, 256, 0, work);
      launch_k(c, row_tree_kernel<HR, RR, false, true>, grid, 256, 0, folded, tout, n_tiles, s, L, lv0,
                                                                       lv1, ed);
    } else {
      const int grid = grid_for(c, (const void*)row_tree_kernel<HR, RR, false>, 256, 0, work);
      launch_k(c, row_tree_kernel<HR, RR, false>, grid, 256, 0, folded, tout, n_tiles, s, L, lv0, lv1, ed);
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

// TT_CHAIN=0 turns the persistent chain kernel (kernels/chain.cuh) off: products
// then run as GEMM fold + tree pass (two launches each), as before.
// Off by default: measured on config 3 it does not beat the two-launch path
// (fold 41.8 + column tree 7.8 us, fold 27.4 + row tree 12.4 us): the chain
// kernel's products take 57 / 58 us and the two-product chain 109 us -- its
// tree items run latency-bound on the GEMM CTAs' 4 consumer warps, the
// dependency probes lengthen each claim, and the row trees of the second
// product still wait for the last fold units (profiles/r02_chain_kernel.md).
std::atomic<int> g_chain{[] {
  const char* e = std::getenv("TT_CHAIN");
  return e ? std::atoi(e) : 0;
}()};
// TT_CHAIN_P2COL=1: a chain's second product (row tree) folds in the first
// product's column order (starts earlier, its row trees wait for the end)
const int g_chain_p2_col = [] {
  const char* e = std::getenv("TT_CHAIN_P2COL");
  return e ? std::atoi(e) : 0;
}();
// TT_CHAIN_G: column blocks per super-group of the column-major fold order
const int g_chain_g = [] {
  const char* e = std::getenv("TT_CHAIN_G");
  return e ? std::atoi(e) : 4;
}();

// Host view of one chain phase.
struct ChainPlan {
  ChainPhaseDev dev{};
  alignas(64) unsigned char mapA[128];
  alignas(64) unsigned char mapB[128];
  int64_t n_out = 0;
};

// A product is chain-eligible when its fold is GEMM shaped (one group dim along
// which only A varies, one along which only B varies, every other group dim of
// extent 1, positive fold steps, the fold over all steps from 0) and its in-tile
// schedule is a forward power-of-two tree of the column-local (t * stride = s,
// stride a multiple of 16) or row-local (reach <= 16 rows of 32) kind -- or none.
bool plan_chain_phase(const LaunchCtx& c, const ChainStep& st, int64_t s, ChainPlan& cp) {
  const Program& prog = *st.prog;
  const GroupSpec& g = st.g;
  if (!st.tb || s % (kChSL * 32) != 0 || s >= (int64_t{1} << 31)) return false;
  const bool fold_only = prog.ops.size() == 1 && prog.ops[0].kind == GOP_FOLD && prog.ops[0].dst == BUF_OUT;
  if (!fold_only && !prog.simple_pow2) return false;
  GroupParams p = make_group_params(prog, g, s);
  if (p.ops[0].x != 0 || p.ops[0].y < 1 || p.ops[0].y >= (int64_t{1} << 24)) return false;
  const BlockPlan bp = block_plan(g, true);
  if (bp.ia < 0 || bp.ib < 0) return false;
  for (int i = 0; i < g.nd; ++i)
    if (i != bp.ia && i != bp.ib && g.ext[i] != 1) return false;
  if (g.astep <= 0 || g.bstep <= 0 || g.a_stride[bp.ia] <= 0 || g.b_stride[bp.ib] <= 0) return false;
  const int64_t ni = g.ext[bp.ia], nj = g.ext[bp.ib];
  if (ni > 16 * 255 || nj > 16 * 255 || ((ni + 15) / 16) * ((nj + 15) / 16) > 64) return false;
  if (!aligned16(st.ta) || !aligned16(st.tb) || !aligned16(st.tout)) return false;
  ChainPhaseDev& d = cp.dev;
  d.ni = static_cast<int>(ni);
  d.nj = static_cast<int>(nj);
  d.nk = static_cast<int>(p.ops[0].y);
  d.nbi = static_cast<int>((ni + 15) / 16);
  d.nbj = static_cast<int>((nj + 15) / 16);
  d.out_i = g.out_stride[bp.ia];
  d.out_j = g.out_stride[bp.ib];
  d.out = st.tout;
  d.nsub = 16;
  const int nchunks = static_cast<int>(s / kChSL);
  if (fold_only) {
    d.tree = 0;
  } else {
    p.nlevels = static_cast<int>(prog.ops.size()) - 1;
    if (p.nlevels < 1 || p.nlevels > 8) return false;
    for (int i = 0; i < p.nlevels; ++i) p.rots[i] = prog.ops[i + 1].x;
    const TreePass tp = plan_tree_pass(p, s, c.smem_optin);
    if (tp.back || tp.kind == 3) return false;
    if (tp.kind == 1 && tp.stride0 % kChSL == 0 && tp.t <= 32) {
      d.tree = 1;
      d.col_t = static_cast<int>(tp.t);
      d.col_stride = static_cast<int>(tp.stride0);
      d.tree_ncb = static_cast<int>(tp.stride0 / kChSL);
      d.tq = d.tree_ncb;
      d.tree_per = nchunks / d.tree_ncb;
    } else if (tp.kind == 2 && tp.hr <= 16) {
      d.tree = 2;
      d.hr = tp.hr;
      d.nlevels = p.nlevels;
      for (int i = 0; i < p.nlevels; ++i) d.lv[i] = static_cast<int>(p.rots[i]);
      d.tq = static_cast<int>(s / 512);
      d.tree_per = 512 / kChSL;
    } else {
      return false;
    }
  }
  // operand tensor maps {slot, block row, fold step}
  const uint64_t eb = sizeof(double);
  const uint64_t dA[3] = {static_cast<uint64_t>(s), static_cast<uint64_t>(ni), static_cast<uint64_t>(d.nk)};
  const uint64_t dB[3] = {static_cast<uint64_t>(s), static_cast<uint64_t>(nj), static_cast<uint64_t>(d.nk)};
  const uint64_t sA[2] = {static_cast<uint64_t>(g.a_stride[bp.ia] * s) * eb, static_cast<uint64_t>(g.astep * s) * eb};
  const uint64_t sB[2] = {static_cast<uint64_t>(g.b_stride[bp.ib] * s) * eb, static_cast<uint64_t>(g.bstep * s) * eb};
  const uint32_t box[3] = {kChSL, kChP, kChKS};
  if (!encode_tensor_map_f64(cp.mapA, 3, st.ta, dA, sA, box) ||
      !encode_tensor_map_f64(cp.mapB, 3, st.tb, dB, sB, box))
    return false;
  return true;
}

// Returns true when `epi` was applied (fused into a tree pass); the caller
// runs it as a separate pass otherwise.
template <bool HAS_B>
bool launch_program_impl(const LaunchCtx& c, const Program& prog, const GroupSpec& g, int64_t s,
                         const double* ta, const double* tb, double* tout, const Epilogue* epi) {
  GroupParams p = make_group_params(prog, g, s);
  if (g.groups == 0) return true;
  const size_t tile_bytes = static_cast<size_t>(s) * sizeof(double);
  // 1) No in-tile schedule: the fold is the whole program.
  if (prog.ops.size() == 1 && prog.ops[0].kind == GOP_FOLD && prog.ops[0].dst == BUF_OUT) {
    LaunchCtx cl = c;  // an epilogue pass follows (unless the fold applies it): late release
    cl.release_late = epi != nullptr;
    return launch_fold_best<HAS_B>(cl, p, ta, tb, tout, epi);
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
        return false;
      }
    }
    // Too few groups to occupy every SM: fold over the whole grid first
    // (phase 1, into OUT), then run the schedule on OUT in place (phase 2).
    const int64_t per_sm = std::max<int64_t>(1, static_cast<int64_t>(c.smem_optin / (tile_bytes + 1024)));
    // ...unless the whole reduction is tiny (< 2^20 product slots): then one
    // fused launch beats two (small ops are launch-latency bound; config 1)
    const bool tiny = g.groups * prog.ops[0].y * s < (int64_t{1} << 20);
    if (matmul_like && HAS_B && force == 0 && prog.ops[0].y > 1 && (epi == nullptr || !epi->active()) &&
        !tiny) {
      ChainStep one;
      one.prog = &prog;
      one.g = g;
      one.ta = ta;
      one.tb = tb;
      one.tout = tout;
      if (launch_chain(c, &one, 1, s)) return false;
    }
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
        return false;
      }
      int64_t reach = 0;
      for (int i = 0; i < p.nlevels; ++i) reach += p.rots[i];
      const bool tree_tma = g_tree_tma && tma_ok && (tpass.kind == 1 || tpass.kind == 2) && !tpass.back &&
                            (epi == nullptr || !epi->active()) && aligned16(fold_dst);
      if (tree_tma) {
        launch_fold_best<HAS_B>(c, p, ta, tb, fold_dst);
        GroupParams p2 = p;
        for (int i = 0; i < g.nd; ++i) {
          p2.g.a_stride[i] = g.out_stride[i];
          p2.g.b_stride[i] = 0;
        }
        p2.g.astep = 0;
        p2.g.bstep = 0;
        p2.ops[0].x = 0;
        p2.ops[0].y = 1;
        if (reach <= kTmaChunk && g_tree_tma == 1)
          run_tma_win<false>(c, p2, static_cast<int>(reach), fold_dst, nullptr, tout);
        else
          dispatch_tma<false>(c, p2, fold_dst, nullptr, tout);
        return false;
      }
      if (tpass.kind != 0) {
        LaunchCtx cl = c;  // the tree pass follows: the fold releases it at exit
        cl.release_late = true;
        launch_fold_best<HAS_B>(cl, p, ta, tb, fold_dst);
        const bool fuse_epi = tpass.kind == 1 || tpass.kind == 2;
        run_tree_pass(c, tpass, p, g.groups, s, fold_dst, tout, fuse_epi ? epi : nullptr);
        return fuse_epi;
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
      return false;
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
    return false;
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
  launch_k(c, k, grid, gthreads, smem, p, ta, tb, tout, scratch);
  post_launch(c, "group generic kernel");
  return false;
}

}  // namespace

void set_kernel_path(int path) { g_forced_path.store(path, std::memory_order_relaxed); }
void set_chain_kernel(int on) { g_chain.store(on ? 1 : 0, std::memory_order_relaxed); }
int chain_kernel_enabled() { return g_chain.load(std::memory_order_relaxed); }
int kernel_path() { return forced_path(); }

bool launch_chain(const LaunchCtx& c, const ChainStep* steps, int n, int64_t s) {
  if (!g_chain.load(std::memory_order_relaxed) || n < 1 || n > 2 || !c.chain_base || forced_path() != 0)
    return false;
  ChainPlan cp[2];
  for (int k = 0; k < n; ++k)
    if (!plan_chain_phase(c, steps[k], s, cp[k])) return false;
  if (n == 2) {  // the second product reads the first's result: column tree needed
    if (cp[0].dev.tree != 1) return false;
    if (steps[1].ta != steps[0].tout && steps[1].tb != steps[0].tout) return false;
  }
  ChainDev d{};
  d.nphase = n;
  d.s = s;
  d.nchunks = static_cast<int>(s / kChSL);
  // fold buffers: session scratch, one region per phase with a tree
  size_t fold_bytes[2] = {0, 0};
  for (int k = 0; k < n; ++k) {
    if (!cp[k].dev.tree) continue;
    const int64_t hi = (cp[k].dev.ni - 1) * cp[k].dev.out_i + (cp[k].dev.nj - 1) * cp[k].dev.out_j + 1;
    fold_bytes[k] = static_cast<size_t>(hi) * s * sizeof(double);
  }
  double* scratch = (fold_bytes[0] + fold_bytes[1]) ? c.scratch(c.scratch_owner, fold_bytes[0] + fold_bytes[1]) : nullptr;
  int counter = 5;  // queue heads F0, T0, F1, T1 and the exit count
  for (int k = 0; k < n; ++k) {
    ChainPhaseDev& P = cp[k].dev;
    P.fold = P.tree ? scratch + (k == 1 ? fold_bytes[0] / sizeof(double) : 0) : P.out;
    const int nb = P.nbi * P.nbj;
    if (k == 1 && (P.tree != 2 || g_chain_p2_col)) {  // follow phase 1's column order: its column block c % ncb unlocks chunk c
      P.col_order = 1;
      P.ncb = cp[0].dev.tree_ncb;
      P.q = P.ncb;
      P.per_q = d.nchunks / P.ncb;
      P.dep_phase = 0;
      P.dep_ncb = cp[0].dev.tree_ncb;
      P.dep_target = cp[0].dev.nbi * cp[0].dev.nbj * cp[0].dev.nsub;
    } else {
      P.dep_phase = -1;
      if (k == 1) {  // rows of phase 2 complete one after the other (its row trees overlap)
        P.dep_phase = 0;
        P.dep_ncb = cp[0].dev.tree_ncb;
        P.dep_target = cp[0].dev.nbi * cp[0].dev.nbj * cp[0].dev.nsub;
      }
      if (P.tree == 1) {  // column blocks complete one after the other
        P.col_order = 1;
        P.ncb = P.tree_ncb;
        P.q = P.ncb;
        P.per_q = d.nchunks / P.ncb;
      } else {            // row blocks complete one after the other
        P.col_order = 0;
        P.ncb = 1;
        P.q = P.tree == 2 ? P.tq : 1;
        P.per_q = d.nchunks / P.q;
      }
    }
    if (P.col_order) {  // super-groups of colg column blocks (a divisor of q)
      P.colg = std::max(1, std::min(g_chain_g, P.q));
      while (P.q % P.colg) --P.colg;
    }
    P.nf = P.q * P.per_q * nb;
    P.nt = P.tree ? P.tq * nb * P.nsub : 0;
    P.fold_done = counter;
    counter += P.tree ? P.tq * nb : 0;
    P.tree_done = counter;
    counter += P.tree == 1 ? P.tq : 0;
    d.ph[k] = P;
  }
  if (counter > static_cast<int>(kChainCounters)) return false;
  d.ncnt = counter;
  d.cnt = c.chain_base + ((*c.chain_next)++ % kChainSlots) * kChainCounters;
  const size_t smem = static_cast<size_t>(kChNS) * kChStage * sizeof(double) + 3 * kChNS * 8;
  set_smem_attr((const void*)chain_kernel, smem);
  const int grid = grid_for(c, (const void*)chain_kernel, kChThreads, smem,
                            d.ph[0].nf + (n > 1 ? d.ph[1].nf : 0), true);
  const CUtensorMap* m0a = reinterpret_cast<const CUtensorMap*>(cp[0].mapA);
  const CUtensorMap* m0b = reinterpret_cast<const CUtensorMap*>(cp[0].mapB);
  const CUtensorMap* m1a = reinterpret_cast<const CUtensorMap*>(n > 1 ? cp[1].mapA : cp[0].mapA);
  const CUtensorMap* m1b = reinterpret_cast<const CUtensorMap*>(n > 1 ? cp[1].mapB : cp[0].mapB);
  chain_kernel<<<grid, kChThreads, smem, c.stream>>>(*m0a, *m0b, *m1a, *m1b, d);
  post_launch(c, "chain kernel");
  return true;
}

void launch_group_program(const LaunchCtx& c, const Program& prog, const GroupSpec& g, int64_t s,
                          const double* ta, const double* tb, double* tout, const Epilogue* epi) {
  if (epi != nullptr && !epi->active()) epi = nullptr;
  const bool applied = tb != nullptr ? launch_program_impl<true>(c, prog, g, s, ta, tb, tout, epi)
                                     : launch_program_impl<false>(c, prog, g, s, ta, tb, tout, epi);
  if (epi != nullptr && !applied) launch_epilogue(c, *epi, s, tout, g.groups);
}

void launch_epilogue(const LaunchCtx& c, const Epilogue& e, int64_t s, double* tiles,
                     int64_t n_tiles) {
  if (!e.active() || n_tiles <= 0) return;
  const EpiDev ed = make_epi_dev(e);
  const bool vec = s % 2 == 0 && aligned16(tiles) && (e.c == nullptr || aligned16(e.c));
  const int64_t per = vec ? s / 2 : s;
  const int64_t work = (n_tiles * per + 255) / 256;
  if (vec) {
    const int grid = grid_for(c, (const void*)epilogue_kernel<true>, 256, 0, work);
    launch_k(c, epilogue_kernel<true>, grid, 256, 0, tiles, n_tiles, s, make_div64(static_cast<uint64_t>(per)), ed);
  } else {
    const int grid = grid_for(c, (const void*)epilogue_kernel<false>, 256, 0, work);
    launch_k(c, epilogue_kernel<false>, grid, 256, 0, tiles, n_tiles, s, make_div64(static_cast<uint64_t>(per)), ed);
  }
  post_launch(c, "epilogue kernel");
}

}  // namespace ttb

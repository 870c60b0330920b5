// kernels/stream.cuh -- pack / unpack / clean_unknowns / elementwise / rotate kernels (streaming, HBM bound).
// Included by tt_kernels.cu inside namespace ttb::{anonymous}: one
// translation unit, so the kernels share its device helpers (FastDiv,
// dadd / dmul, mbarrier and TMA wrappers) without external linkage.
#pragma once

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
  pdl_enter();
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
  pdl_enter();
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
  pdl_enter();
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
  pdl_enter();
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
        // a cut dim whose whole period t * 2^sh fits in 512 slots has the same
        // coordinate at o and at base + 512 u + o: the mask is per thread
        bool local = true;
#pragma unroll
        for (int i = 0; i < RK; ++i) local = local && (!cut[i] || (g.t[i] << sh[i]) <= 512);
        if (local && n == kCleanChunk && g.tile_slots == g.s) {
          bool ok[2] = {true, true};
#pragma unroll
          for (int i = 0; i < RK; ++i)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (cut[i]) ok[e] = ok[e] && (((2 * static_cast<int>(threadIdx.x) + e) >> sh[i]) & (g.t[i] - 1)) < v[i];
          const double m0 = ok[0] ? 1.0 : 0.0, m1 = ok[1] ? 1.0 : 0.0;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t k = u * 256 + threadIdx.x;
            d2[k] = make_double2(dmul(x[u].x, m0), dmul(x[u].y, m1));
          }
        } else if (n == kCleanChunk && g.tile_slots == g.s) {
          // h = base + 512 u + o with o = 2 tid + e < 512 and base + 512 u a
          // multiple of 512, so the coordinate of a cut dim with stride 2^sh
          // splits into an item/u part and a per-thread part:
          //   sh <= 9: ((base + 512 u) >> sh) + (o >> sh)   (no carry)
          //   sh >  9: (base + 512 u) >> sh                  (o below bit 9)
          // Per thread the o-parts are fixed; per u one shift per dim.
          int ob[RK][2];
#pragma unroll
          for (int i = 0; i < RK; ++i)
#pragma unroll
            for (int e = 0; e < 2; ++e) ob[i][e] = sh[i] <= 9 ? (2 * static_cast<int>(threadIdx.x) + e) >> sh[i] : 0;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t k = u * 256 + threadIdx.x;
            const int64_t hu = base + 512 * u;
            bool ok0 = true, ok1 = true;
#pragma unroll
            for (int i = 0; i < RK; ++i) {
              if (cut[i]) {
                const int64_t a = hu >> sh[i];
                ok0 = ok0 && ((a + ob[i][0]) & (g.t[i] - 1)) < v[i];
                ok1 = ok1 && ((a + ob[i][1]) & (g.t[i] - 1)) < v[i];
              }
            }
            d2[k] = make_double2(dmul(x[u].x, ok0 ? 1.0 : 0.0), dmul(x[u].y, ok1 ? 1.0 : 0.0));
          }
        } else {
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
  int keep_a, keep_b;     // operand broadcasts along a dim (its tiles are re-read): L2 evict_last
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
  pdl_enter();
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
// 16-byte global load / store with an L2 eviction-priority hint
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t pol;
  if (keep)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double2 ld2_hint(const double2* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st2_hint(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}

constexpr int kEwU = 8;                // double2 per thread per item
constexpr int kEwChunk = 512 * kEwU;   // slots per work item (256 threads x kEwU x double2)
// HINT (an operand broadcasts): its loads are L2 evict_last and the streamed
// operand's loads and the stores evict_first, so the re-read broadcast tiles
// stay L2-resident while the rest streams past (config 5 X * W: W's 128 MiB is
// otherwise re-fetched from HBM ~8 times, 6% of the op's traffic).
template <int OP, bool HINT = false>
__global__ void __launch_bounds__(256) elementwise_chunk_kernel(const __grid_constant__ EwParams p,
                                                                 const double* __restrict__ a,
                                                                 const double* __restrict__ b,
                                                                 double* __restrict__ out,
                                                                 FastDiv64 chunks_div) {
  pdl_enter();
  const uint64_t items = static_cast<uint64_t>(p.n_tiles) * chunks_div.d;
  const int tid = threadIdx.x;
  const uint64_t pol_a = l2_policy(HINT && p.keep_a), pol_b = l2_policy(HINT && p.keep_b);
  const uint64_t pol_o = l2_policy(false);
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
        if (HINT) {
          va[u] = ld2_hint(pa + k, pol_a);
          vb[u] = ld2_hint(pb + k, pol_b);
        } else {
          va[u] = __ldg(pa + k);
          vb[u] = __ldg(pb + k);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kEwU; ++u) {
      const int k = u * 256 + tid;
      if (k < npairs) {
        const double2 o = OP == TT_OP_ADD ? make_double2(dadd(va[u].x, vb[u].x), dadd(va[u].y, vb[u].y))
                                          : make_double2(dmul(va[u].x, vb[u].x), dmul(va[u].y, vb[u].y));
        if (HINT)
          st2_hint(po + k, o, pol_o);
        else
          po[k] = o;
      }
    }
  }
}

// Paired variant for a large broadcast product / sum: a work item is the same
// chunk of TWO output tiles that are consecutive along the innermost visited dim,
// where exactly one operand broadcasts -- its chunk is loaded once for both, a
// quarter fewer loads through the L2 (config 5: X * W 5.66 -> 5.63 ms, W * X and
// X + W 5.74 -> 5.66 ms: a ~1% gain, the op is bound by its DRAM traffic).  `p` has
// the inner dim halved (strides doubled); v_in / o_in = tile strides of the varying
// operand and the output between the two tiles.  SHARED_B: b is the broadcast operand.
template <int OP, bool SHARED_B>
__global__ void __launch_bounds__(256) elementwise_pair_kernel(const __grid_constant__ EwParams p,
                                                                const double* __restrict__ a,
                                                                const double* __restrict__ b,
                                                                double* __restrict__ out,
                                                                FastDiv64 chunks_div, int64_t v_in,
                                                                int64_t o_in) {
  pdl_enter();
  const uint64_t items = static_cast<uint64_t>(p.n_tiles) * chunks_div.d;
  const int tid = threadIdx.x;
  const uint64_t pol_s = l2_policy(true), pol_v = l2_policy(false);
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const uint64_t vt = fdiv(item, chunks_div);  // tile pair in visiting order
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
    const double2* psh = reinterpret_cast<const double2*>((SHARED_B ? b + fb * p.s : a + fa * p.s) + base);
    const double2* pv0 = reinterpret_cast<const double2*>((SHARED_B ? a + fa * p.s : b + fb * p.s) + base);
    const double2* pv1 = pv0 + (v_in * p.s) / 2;
    double2* po0 = reinterpret_cast<double2*>(out + flat * p.s + base);
    double2* po1 = po0 + (o_in * p.s) / 2;
    const int64_t npairs = (p.s - base) / 2 < kEwChunk / 2 ? (p.s - base) / 2 : kEwChunk / 2;
    double2 vs[kEwU], v0[kEwU], v1[kEwU];
#pragma unroll
    for (int u = 0; u < kEwU; ++u) {
      const int k = u * 256 + tid;
      if (k < npairs) {
        v0[u] = ld2_hint(pv0 + k, pol_v);
        v1[u] = ld2_hint(pv1 + k, pol_v);
        vs[u] = ld2_hint(psh + k, pol_s);
      }
    }
#pragma unroll
    for (int u = 0; u < kEwU; ++u) {
      const int k = u * 256 + tid;
      if (k < npairs) {
        // IEEE addition and multiplication commute: op(a, b) with either operand shared
        const double2 o0 = OP == TT_OP_ADD ? make_double2(dadd(v0[u].x, vs[u].x), dadd(v0[u].y, vs[u].y))
                                           : make_double2(dmul(v0[u].x, vs[u].x), dmul(v0[u].y, vs[u].y));
        const double2 o1 = OP == TT_OP_ADD ? make_double2(dadd(v1[u].x, vs[u].x), dadd(v1[u].y, vs[u].y))
                                           : make_double2(dmul(v1[u].x, vs[u].x), dmul(v1[u].y, vs[u].y));
        st2_hint(po0 + k, o0, pol_v);
        st2_hint(po1 + k, o1, pol_v);
      }
    }
  }
}

template <int OP>
__global__ void __launch_bounds__(256) binary_flat_kernel(const double* __restrict__ a,
                                                           const double* __restrict__ b,
                                                           double* __restrict__ out,
                                                           uint64_t count) {
  pdl_enter();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = OP == TT_OP_ADD ? dadd(a[i], b[i]) : dmul(a[i], b[i]);
}

__global__ void __launch_bounds__(256) rotate_kernel(const double* __restrict__ in,
                                                      double* __restrict__ out, uint64_t s,
                                                      uint64_t r, uint64_t total,
                                                      FastDiv64 sdiv) {
  pdl_enter();
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
  pdl_enter();
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
  pdl_enter();
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

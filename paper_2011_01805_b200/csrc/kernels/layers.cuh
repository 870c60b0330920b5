// kernels/layers.cuh -- batch-packed nn layers and the range fold of cross-GPU chains.
// Included by tt_kernels.cu inside namespace ttb::{anonymous}: one
// translation unit, so the kernels share its device helpers (FastDiv,
// dadd / dmul, mbarrier and TMA wrappers) without external linkage.
#pragma once

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
  pdl_enter();
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
  pdl_enter();
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
  pdl_enter();
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
  pdl_enter();
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

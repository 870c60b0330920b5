// tt_launch.hpp -- host-side launch API of the sm_100a kernels (tt_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "tt_internal.hpp"

namespace ttb {

struct LaunchCtx {
  cudaStream_t stream = nullptr;
  int device = 0;
  int sm_count = 148;
  size_t smem_optin = 227 * 1024;  // max dynamic smem per block
  size_t l2_bytes = size_t{126} << 20;  // device L2 size (cudaDeviceProp::l2CacheSize)
  uint64_t* launches = nullptr;    // incremented per kernel launch
  // Session-owned device scratch; (re)sized by the caller via `need`.
  double* (*scratch)(void* owner, size_t bytes) = nullptr;
  void* scratch_owner = nullptr;
  // Session-owned ring of work-queue counter pairs (next unit, CTAs done).
  unsigned int* sched_base = nullptr;
  unsigned int* sched_next = nullptr;
  unsigned int* chain_base = nullptr;   // kChainSlots blocks of kChainCounters
  unsigned int* chain_next = nullptr;
  // The fold launched with this context is followed by a tree pass of the same
  // operator: it releases its PDL dependents at CTA exit (tt_pdl.cuh).
  bool release_late = false;
};

constexpr unsigned int kSchedSlots = 256;
// Dependency-counter blocks of the chain kernel (kernels/chain.cuh), a ring
// after the scheduler pairs in the same session buffer; each launch's last CTA
// leaves its block at zero.
constexpr unsigned int kChainSlots = 8;
constexpr unsigned int kChainCounters = 8192;
// The (next, done) counter pair for one dynamically scheduled launch.  The
// kernel's last CTA resets both to zero, so a slot is reusable by the next
// launch on the stream; concurrent launches (different streams) get distinct
// slots of the ring.
inline unsigned int* take_sched_slot(const LaunchCtx& c) {
  if (!c.sched_base) return nullptr;
  const unsigned int i = (*c.sched_next)++ % kSchedSlots;
  return c.sched_base + 2 * i;
}

// Group grid of a reduction: output tile ("group") g is addressed by
// coordinates c_0..c_{nd-1} in iteration order (outermost first); its output
// tile index and the operands' base tile indices are linear in c.  Along the
// summed dim, operand tile indices advance by astep/bstep per fold step.
struct GroupSpec {
  int nd = 0;
  int64_t ext[TT_MAX_RANK] = {};
  int64_t out_stride[TT_MAX_RANK] = {};
  int64_t a_stride[TT_MAX_RANK] = {};
  int64_t b_stride[TT_MAX_RANK] = {};
  int64_t astep = 0;
  int64_t bstep = 0;
  int64_t groups = 1;
};

void launch_pack(const LaunchCtx& c, const Shape& shape, int64_t s, const double* dense,
                 double* tiles);
void launch_unpack(const LaunchCtx& c, const Shape& shape, int64_t s, const double* tiles,
                   double* dense);
// TMA tensor-map pack / unpack (tt_tma_pack.cu); return false when the shape
// is not eligible (replication, `~`, relaxed, rank > 5, odd last extent...).
// Encodes a float64 tiled tensor map (CUtensorMap, 128 bytes at map128):
// dims/box innermost first, stride_bytes for dims 1..rank-1.  False if the
// driver entry point is missing or the geometry is not expressible.
bool encode_tensor_map_f64(void* map128, int rank, const void* base, const uint64_t* dims,
                           const uint64_t* stride_bytes, const uint32_t* box);
bool launch_pack_tma(const LaunchCtx& c, const Shape& shape, int64_t s, const double* dense,
                     double* tiles);
bool launch_unpack_tma(const LaunchCtx& c, const Shape& shape, int64_t s, const double* tiles,
                       double* dense);
// out tile l = A[l mod ea] (op) B[l mod eb]   (tile_tensor.hpp:259-270)
void launch_elementwise(const LaunchCtx& c, int op, const Shape& out, const Shape& a,
                        const Shape& b, int64_t s, const double* ta, const double* tb,
                        double* tout);
// out[i] = a[i] (op) b[i] over `count` slots; op 2 = a * mask (same as mul)
// out[o] = bias[o] (+) w[k] (*) in[src[k]] over k in [row_ptr[o], row_ptr[o+1]),
// left fold per slot; the CSR arrays are device pointers.
// block > 1: consecutive groups of `block` rows share their source list (the
// blocked kernel loads each input once for the whole group).
void launch_batch_affine(const LaunchCtx& c, const double* in, int64_t s, int64_t n_out,
                         const int64_t* row_ptr, const int64_t* src, const double* w,
                         const double* bias, double* out, int block);
// Fold of a product over its summed dim for the output tiles [o0, o1) of the
// result grid `gext` (row-major, summed dim extent 1): acc = init (when
// given) then acc = acc + A[l]*B[l] (B optional) for l in [first, first+count)
// in order; without init the fold starts from the first product.  Output and
// init hold (o1 - o0) tiles.  Strides are operand tile-index strides per dim;
// astep/bstep the operand strides along the summed dim.
struct FoldRange {
  int rank = 0;
  int64_t gext[TT_MAX_RANK] = {};
  int64_t a_stride[TT_MAX_RANK] = {};
  int64_t b_stride[TT_MAX_RANK] = {};
  int64_t astep = 0, bstep = 0, first = 0, count = 0;
};
void launch_fold_range(const LaunchCtx& c, const FoldRange& fr, int64_t s, int64_t o0, int64_t o1,
                       const double* ta, const double* tb, const double* init, double* acc);
void launch_binary_flat(const LaunchCtx& c, int op, const double* a, const double* b, double* out,
                        int64_t count);
// out[t][j] = in[t][(j + r) mod s]   (backend.hpp:157-159), r in [1, s)
void launch_rotate(const LaunchCtx& c, const double* in, double* out, int64_t s, int64_t r,
                   int64_t n_tiles);
// out = in * used-mask(shape)   (tile_tensor.hpp:364-380)
void launch_clean(const LaunchCtx& c, const Shape& shape, int64_t s, const double* in,
                  double* out);
// Elementwise tail of a reduction -- tt_add(r, C) then tt_mul(r, r), each
// optional -- over the reduction's output grid `ext` (row-major, outermost
// first): out tile l = (r_l + C[sum_i coord_i(l) * c_stride[i]]) squared.
// c_stride[i] is C's tile-index stride along output dim i (0 where C
// broadcasts).  Fused into the tree pass when the reduction ends in one,
// else a separate in-place pass over the output tiles.
// The tail may also start with clean_unknowns' mask (nmask > 0): slot h of
// output tile l is kept iff l_i * t_i + ((h / stride_i) mod t_i) < used_i for
// each cut dim i (power-of-two t_i and strides, not interleaved).
constexpr int kEpiMaskDims = 3;
struct Epilogue {
  const double* c = nullptr;
  bool square = false;
  int nd = 0;
  int64_t ext[TT_MAX_RANK] = {};
  int64_t c_stride[TT_MAX_RANK] = {};
  int nmask = 0;
  int mask_dim[kEpiMaskDims] = {};
  int64_t mask_t[kEpiMaskDims] = {}, mask_stride[kEpiMaskDims] = {}, mask_used[kEpiMaskDims] = {};
  bool active() const { return c != nullptr || square || nmask > 0; }
};
// Runs `prog` for every group of `g`; `tb` may be null (no fused multiply);
// `epi` (optional) is applied to every output tile.
// One product of a fused chain (tt_linalg_chain): its reduction program and
// group grid as run_reduction builds them, operand and result tiles.
struct ChainStep {
  const Program* prog = nullptr;
  GroupSpec g;
  const double* ta = nullptr;
  const double* tb = nullptr;
  double* tout = nullptr;
};
// Runs 1 or 2 products (the second reading the first's result as one operand)
// as one persistent chain kernel; false (nothing launched) when a product is
// not a GEMM-shaped fold with a column- or row-local power-of-two tree.
bool launch_chain(const LaunchCtx& c, const ChainStep* steps, int n, int64_t s);

void launch_group_program(const LaunchCtx& c, const Program& prog, const GroupSpec& g, int64_t s,
                          const double* ta, const double* tb, double* tout,
                          const Epilogue* epi = nullptr);
// The epilogue alone, in place over n_tiles output tiles.
void launch_epilogue(const LaunchCtx& c, const Epilogue& e, int64_t s, double* tiles,
                     int64_t n_tiles);
// Synthetic input generator shared with oracle/tt_oracle.c or_fill_uniform.
void launch_fill_uniform(const LaunchCtx& c, double* out, int64_t count, uint64_t seed,
                         int64_t offset, double lo, double hi);

void check_cuda(cudaError_t e, const char* what);
// 0 = best eligible, 1 = TMA ring, 2 = register tree, 3 = generic interpreter.
void set_kernel_path(int path);
int kernel_path();
void set_chain_kernel(int on);
int chain_kernel_enabled();

}  // namespace ttb

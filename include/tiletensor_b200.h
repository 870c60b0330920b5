/*
 * tiletensor_b200.h -- C-ABI of the B200-native tile-tensor hot path.
 *
 * The reference (arXiv 2011.01805, /root/reference/proj) is a header-only
 * C++20 library in namespace `tiletensor`; it has no FFI of its own.  This
 * header is the thin `extern "C"` layer that the C++ host mirror
 * (paper_2011_01805_b200/include/tiletensor_b200/*.hpp, same signatures as
 * the reference's inc/*.hpp) and the Python binding call.  Every entry point
 * below names the reference symbol it replaces (path:line relative to
 * /root/reference/proj/include/tiletensor/).
 *
 * Conventions
 *  - A tile tensor lives on the device as ONE contiguous fp64 array
 *    [tile_count][slot_count], row-major over the external grid: exactly the
 *    concatenation of the reference's `TileTensor::tiles()[flat].slots()`.
 *  - Dense tensors are row-major fp64 device arrays over the shape's n_i.
 *  - All pointers passed to op entry points are DEVICE pointers unless the
 *    name says `host`.  Ops are asynchronous on the session's stream.
 *  - No entry point throws.  Each returns a tt_status; on failure
 *    tt_last_error() (thread-local) holds the message the reference's
 *    exception would carry, and the C++ mirror rethrows the exact type.
 *  - Shape checks, depth (chain) checks and the cost counters are evaluated
 *    on the host before any launch, so a failing call launches nothing and
 *    changes no counter (the reference throws before its first primitive
 *    for every shape/depth error it can raise on these paths).
 */
#ifndef TILETENSOR_B200_H
#define TILETENSOR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TT_MAX_RANK 16

/* Status codes; map 1:1 onto the reference's exception types. */
typedef enum tt_status {
  TT_OK = 0,
  TT_ERR_SHAPE = 1,            /* tiletensor::ShapeError            shape.hpp:21   */
  TT_ERR_SHAPE_PARSE = 2,      /* tiletensor::ShapeParseError       shape.hpp:26   */
  TT_ERR_DEPTH = 3,            /* tiletensor::DepthExhaustedError   backend.hpp:18 */
  TT_ERR_INVALID_ARGUMENT = 4, /* std::invalid_argument                            */
  TT_ERR_OUT_OF_RANGE = 5,     /* std::out_of_range                                */
  TT_ERR_LOGIC = 6,            /* std::logic_error                                 */
  TT_ERR_CUDA = 7,             /* CUDA runtime failure (no reference equivalent)   */
  TT_ERR_NO_DEVICE = 8         /* no CUDA device: the product never falls back     */
} tt_status;

typedef enum tt_op { TT_OP_ADD = 0, TT_OP_MUL = 1 } tt_op;          /* OpKind shape.hpp:284 */

typedef enum tt_variant {                                             /* SumVariant rotate_sum.hpp:20 */
  TT_VARIANT_AUTO = -1, /* std::nullopt -> auto_variant(n)  rotate_sum.hpp:99 */
  TT_VARIANT_LEFT_TO_RIGHT = 0,
  TT_VARIANT_RIGHT_TO_LEFT = 1,
  TT_VARIANT_POWER_OF_TWO = 2
} tt_variant;

/* DimSpec (shape.hpp:37).  `interleaved` is the north star's `~` tiling,
 * which the reference does not implement: element j of
 * an interleaved dim sits in external tile l = j mod e at in-tile coordinate
 * m = j div e, instead of l = j div t, m = j mod t. */
typedef struct tt_dim {
  int64_t n;
  int64_t d;
  int64_t t;
  int32_t unknown;
  int32_t interleaved;
} tt_dim;

/* TileTensorShape (shape.hpp:72). */
typedef struct tt_shape {
  int32_t rank;
  int32_t relaxed;
  tt_dim dims[TT_MAX_RANK];
} tt_shape;

/* CostReport (backend.hpp:28). */
typedef struct tt_cost {
  uint64_t additions;
  uint64_t multiplications;
  uint64_t mask_multiplications;
  uint64_t rotations;
  uint64_t bootstraps;
  uint64_t power_of_two_rotations;
} tt_cost;

typedef struct tt_session tt_session; /* Session backend.hpp:83 */

/* ---- errors ------------------------------------------------------------ */
const char* tt_last_error(void);
int64_t tt_last_error_position(void); /* ShapeParseError::position() shape.hpp:31 */
const char* tt_version(void);

/* ---- shape algebra (host only; no device needed) ----------------------- */
int tt_shape_parse(const char* text, tt_shape* out);                  /* parse_shape        shape.hpp:250 */
int tt_shape_format(const tt_shape* s, char* buf, int64_t cap);       /* format_shape       shape.hpp:256 */
int tt_shape_check(const tt_shape* s);                                /* TileTensorShape()  shape.hpp:74  */
int tt_shape_external(const tt_shape* s, int64_t* ext_out);           /* external_extents   shape.hpp:99  */
int64_t tt_shape_tile_count(const tt_shape* s);                       /* tile_count         shape.hpp:106 */
int64_t tt_shape_tile_slots(const tt_shape* s);                       /* tile_slots         shape.hpp:86  */
int64_t tt_shape_used_slots(const tt_shape* s);                       /* used_slots         shape.hpp:112 */
int tt_shape_elementwise_result(const tt_shape* a, const tt_shape* b, int op,
                                tt_shape* out);                       /* elementwise_result_shape shape.hpp:293 */
int tt_shape_sum_result(const tt_shape* s, int dim, tt_shape* out);   /* sum_result_shape   shape.hpp:357 */
/* logical_indices / slot_of (tile_tensor.hpp:96,114) */
int tt_logical_indices(const tt_shape* s, const int64_t* tile_index, int64_t h, int64_t* j_out);
int tt_slot_of(const tt_shape* s, const int64_t* j, int64_t* tile_index_out, int64_t* h_out);
/* closed-form rotation counts rotate_sum.hpp:33-39 */
int64_t tt_rotations_left_to_right(int64_t n);
int64_t tt_rotations_right_to_left(int64_t n);

/* ---- session ----------------------------------------------------------- */
int tt_device_count(int* out);
/* Session(slots, depth) backend.hpp:85-91; binds `device` and creates a stream. */
int tt_session_create(int64_t slot_count, int64_t max_chain_index, int device, tt_session** out);
void tt_session_destroy(tt_session* s);
int64_t tt_session_slot_count(const tt_session* s);
int64_t tt_session_max_chain_index(const tt_session* s);
int tt_session_device(const tt_session* s);
/* Run subsequent ops on an external stream (e.g. torch's current stream; NULL
 * is the legacy default stream).  tt_session_use_own_stream restores the
 * session's private stream.  A session's ops share its device scratch (the
 * split-fold target, batch-packed layer tables): ops of ONE session issued on
 * different streams must be ordered by the caller (events); separate
 * sessions are independent. */
int tt_session_set_stream(tt_session* s, void* cuda_stream);
int tt_session_use_own_stream(tt_session* s);
void* tt_session_stream(const tt_session* s);
int tt_session_synchronize(tt_session* s);
void tt_session_cost(const tt_session* s, tt_cost* out);              /* cost_report    backend.hpp:171 */
void tt_session_reset_counters(tt_session* s);                        /* reset_counters backend.hpp:182 */
/* Number of kernels this session has launched (evidence counter for bench/tests). */
uint64_t tt_session_launches(const tt_session* s);
/* Counts `count` bootstraps (backend.hpp:165); values are unchanged so no launch. */
void tt_session_count_bootstraps(tt_session* s, int64_t count);

/* ---- device memory helpers -------------------------------------------- */
/* Stream-ordered: tt_device_alloc takes the block from the session's memory
 * pool in order on the session stream (usable by work enqueued after it on
 * that stream), tt_device_free returns it in order (after the work enqueued
 * before it).  Neither synchronises the device; both are legal during stream
 * capture.  Replaces the reference's per-tile std::vector storage
 * (backend.hpp:65-80, tile_tensor.hpp:151). */
int tt_device_alloc(tt_session* s, int64_t bytes, void** out);
int tt_device_free(tt_session* s, void* p);
/* Result-tile cache on top of the pool (the Python mirror's operator results):
 * tt_tiles_release keeps the block in a per-(stream, size) free list and
 * tt_tiles_alloc hands it out again on the same stream with no driver call
 * (stream order makes the reuse safe).  Freed blocks of a destroyed session
 * are returned to the driver.  While the session stream is being captured
 * tt_tiles_alloc returns TT_OK with *out == NULL: the caller allocates the
 * result in the capturing framework's graph memory instead. */
int tt_tiles_alloc(tt_session* s, int64_t bytes, void** out);
int tt_tiles_release(tt_session* s, void* p);
int tt_copy_h2d(tt_session* s, void* dst, const void* host_src, int64_t bytes);
int tt_copy_d2h(tt_session* s, void* host_dst, const void* src, int64_t bytes);
int tt_copy_d2d(tt_session* s, void* dst, const void* src, int64_t bytes);
/* Seeded synthetic input (bench/tests), bit-identical to the CPU generator
 * or_fill_uniform in oracle/tt_oracle.c: u = splitmix64(splitmix64(seed) ^ (offset+i)),
 * x = lo + (hi-lo) * (u>>11) * 2^-53. */
int tt_fill_uniform(tt_session* s, double* out, int64_t count, uint64_t seed, int64_t offset,
                    double lo, double hi);

/* ---- tile-tensor operators (device pointers) -------------------------- */
/* pack tile_tensor.hpp:167-220.  `dense` holds prod(n_i) values row-major;
 * `tiles` receives tile_count*slot_count values. */
int tt_pack(tt_session* s, const double* dense, const tt_shape* shape, double* tiles);
/* unpack tile_tensor.hpp:222-242 (replica 0 of every element). */
int tt_unpack(tt_session* s, const tt_shape* shape, const double* tiles, double* dense);
/* tt_elementwise / tt_add / tt_mul tile_tensor.hpp:244-279 with external
 * broadcast.  chain_* are the operands' chain indices (TileTensor::chain_index
 * tile_tensor.hpp:145); *out_chain receives the result's. */
int tt_elementwise(tt_session* s, int op, const tt_shape* a, const double* ta, int64_t chain_a,
                   const tt_shape* b, const double* tb, int64_t chain_b, tt_shape* out_shape,
                   double* out, int64_t* out_chain);
/* tt_sum tile_tensor.hpp:286-347 (external left fold + in-tile rotate-and-sum). */
int tt_sum(tt_session* s, const tt_shape* in_shape, const double* tin, int dim, int variant,
           tt_shape* out_shape, double* out);
/* tt_sum(tt_mul(a,b), dim, variant) fused: the product is never materialised.
 * The body of matvec_a/b and matmul_a/b linalg.hpp:41-73. Counters and
 * results equal the two-call composition exactly. */
int tt_mul_sum(tt_session* s, const tt_shape* a, const double* ta, int64_t chain_a,
               const tt_shape* b, const double* tb, int64_t chain_b, int dim, int variant,
               tt_shape* out_shape, double* out, int64_t* out_chain);
/* A fully connected stage of cryptonets_infer's tiled branch nn.hpp:468-490
 * (and the c4 layer): r = tt_sum(tt_mul(a,b), dim, variant); if c is not NULL
 * r = tt_add(r, c); if square r = tt_mul(r, r) -- one device pass for the tail
 * where the reduction ends in a tree pass, else consecutive kernels.  Shapes,
 * chain index, counters and errors equal the three-call composition (which
 * runs as such when c would broadcast the sum to a larger grid or the square
 * would exhaust the depth). */
int tt_mul_sum_affine(tt_session* s, const tt_shape* a, const double* ta, int64_t chain_a,
                      const tt_shape* b, const double* tb, int64_t chain_b, int dim, int variant,
                      const tt_shape* c, const double* tc, int64_t chain_c, int square,
                      tt_shape* out_shape, double* out, int64_t* out_chain);
/* clean_unknowns(tt_sum(tt_mul(a,b), dim, variant)) tile_tensor.hpp:352-386 --
 * the odd -> even seam of pipeline() (linalg.hpp:213-260) and of config 3's
 * literal chain -- with the mask applied in the reduction's last pass.  Shapes,
 * chain index, counters and errors equal the two-call composition (which runs
 * as such when the mask is not expressible in the fused pass). */
int tt_mul_sum_clean(tt_session* s, const tt_shape* a, const double* ta, int64_t chain_a,
                     const tt_shape* b, const double* tb, int64_t chain_b, int dim, int variant,
                     tt_shape* out_shape, double* out, int64_t* out_chain);
/* matvec_a/matvec_b/matmul_a/matmul_b linalg.hpp:41-73 (adds the rank and
 * replication preconditions of linalg.hpp:32-37 to tt_mul_sum).
 * which: 0=matvec_a 1=matvec_b 2=matmul_a 3=matmul_b. */
int tt_linalg_product(tt_session* s, int which, const tt_shape* a, const double* ta,
                      int64_t chain_a, const tt_shape* b, const double* tb, int64_t chain_b,
                      int variant, tt_shape* out_shape, double* out, int64_t* out_chain);
/* Two consecutive products in one launch (the persistent chain kernel):
 *   R1 = product(which1, a1, b1)
 *   R2 = product(which2, x, R1)   (r1_pos == 1: R1 is the right operand)
 *      = product(which2, R1, x)   (r1_pos == 0)
 * e.g. config 3's zero-repack chain matmul_a(A, matmul_b(Bt, C))
 * (tests/test_linalg.cpp:157-178 of the reference).  Both results are
 * written (R1 to out1, R2 to out2); shapes, chain indices, counters and
 * errors equal the two tt_linalg_product calls (which run as such when the
 * pair is not fusable, and always when the first call's inputs are
 * invalid).  Phase 2's fold units at a slot chunk start as soon as phase 1's
 * column trees covering that chunk are done -- no kernel boundary. */
int tt_linalg_chain2(tt_session* s, int which1, const tt_shape* a1, const double* ta1,
                     int64_t chain_a1, const tt_shape* b1, const double* tb1, int64_t chain_b1,
                     int which2, const tt_shape* x, const double* tx, int64_t chain_x, int r1_pos,
                     int variant, tt_shape* out1_shape, double* out1, int64_t* out1_chain,
                     tt_shape* out2_shape, double* out2, int64_t* out2_chain);
/* clean_unknowns tile_tensor.hpp:352-386.  Returns the input unchanged (a
 * device copy when out != in) at zero cost when the shape has no '?'. */
int tt_clean_unknowns(tt_session* s, const tt_shape* in_shape, const double* tin, int64_t chain,
                      tt_shape* out_shape, double* out, int64_t* out_chain);
/* replicate_dim tile_tensor.hpp:391-420. */
int tt_replicate_dim(tt_session* s, const tt_shape* in_shape, const double* tin, int dim,
                     tt_shape* out_shape, double* out);

/* ---- tile-level primitives (Session / rotate_sum.hpp), batched over n_tiles ---- */
int tt_tiles_binary(tt_session* s, int op, const double* a, const double* b, double* out,
                    int64_t n_tiles, const int64_t* chain_a, const int64_t* chain_b,
                    int64_t* chain_out);                              /* Session::add/mul backend.hpp:117-136 */
int tt_tiles_mask_mul(tt_session* s, const double* a, const double* mask, double* out,
                      int64_t n_tiles, const int64_t* chain_a, int64_t* chain_out); /* backend.hpp:138 */
int tt_tiles_rotate(tt_session* s, const double* in, int64_t offset, double* out,
                    int64_t n_tiles);                                 /* Session::rotate backend.hpp:152 */
int tt_sum_tile_strided(tt_session* s, const double* in, int64_t n, int64_t stride, int variant,
                        double* out, int64_t n_tiles);                /* rotate_sum.hpp:44-90 */
int tt_sum_tile_dim(tt_session* s, const double* in, const int64_t* tile_extents, int rank,
                    int dim, int variant, double* out, int64_t n_tiles); /* rotate_sum.hpp:109-120 */
int tt_replicate_tile_dim(tt_session* s, const double* in, const int64_t* tile_extents, int rank,
                          int dim, double* out, int64_t n_tiles);     /* rotate_sum.hpp:128-152 */

/* ---- cross-GPU left-fold chains (sharding.py) --------------------------- */
/* Partial left fold of tt_sum(tt_mul(a, b), dim) -- or tt_sum(a, dim) when b
 * is null -- over output tiles [out_begin, out_end) of the result grid (row-
 * major): acc = init (when given), then acc = acc + product for every
 * external index of `dim` in order; without init the fold starts from the
 * first product, exactly as the reference's tt_sum (tile_tensor.hpp:311-318).
 * A rank holding a slab of `dim` continues the accumulator of the rank before
 * it, so a chain of ranks reproduces the single-GPU association bit for bit.
 * No in-tile schedule: finish with tt_sum over `dim` on the accumulated tiles
 * viewed with the shape tt_fold_shape gives (dim's extent one tile).
 * Counters: the range's products and fold additions; *out_chain as tt_mul.
 * Rejects a '?' boundary split, `~` or degenerate summed dims (use tt_mul_sum). */
int tt_mul_fold(tt_session* s, const tt_shape* a, const double* ta, int64_t chain_a,
                const tt_shape* b, const double* tb, int64_t chain_b, int dim,
                int64_t out_begin, int64_t out_end, const double* init, double* acc,
                int64_t* out_chain);
/* Shape of the accumulated tiles of tt_mul_fold: the product shape (a alone
 * when b is null) with `dim` reduced to one external tile (n = t). */
int tt_fold_shape(const tt_shape* a, const tt_shape* b, int dim, tt_shape* out);

/* ---- neural-network layers (nn.hpp) ------------------------------------ */
/* Batch-packed affine layer of cryptonets_infer (nn.hpp:282-326 replaces the
 * per-scalar Session::add / Session::mul loop of infer_batch_packed): every
 * network scalar is one tile, and output tile o is the left fold
 *   acc = bias[o];  acc = acc + w[k] * in[src[k]]  for k in [row_ptr[o], row_ptr[o+1])
 * with separately rounded multiply and add, exactly as
 * session.add(acc, session.mul(constant_tile(w[k]), v[src[k]])).  Counters
 * grow by one multiplication and one addition per tap.  row_ptr (n_out + 1
 * entries), src, w and bias are HOST arrays (plaintext weights); in / out are
 * device tiles.  chain_in is the input's chain index; *chain_out gets the
 * result's (chain_in - 1 when any tap exists, else the session depth).
 * TT_ERR_DEPTH when a tap would multiply at chain index 0. */
int tt_batch_affine(tt_session* s, const double* in, int64_t n_in, int64_t n_out,
                    const int64_t* row_ptr, const int64_t* src, const double* w,
                    const double* bias, double* out, int64_t chain_in, int64_t* chain_out);
/* The same layer uploaded once and kept on the device (repeated inference with
 * fixed weights: no per-call validation, tap-list scan or H2D).  create takes
 * the arguments of tt_batch_affine (host arrays, same checks and errors);
 * apply runs it with tt_batch_affine's semantics, counters and chain rule;
 * destroy frees it (after the session's queued work that uses it). */
typedef struct tt_affine_layer tt_affine_layer;
int tt_affine_layer_create(tt_session* s, int64_t n_in, int64_t n_out, const int64_t* row_ptr,
                           const int64_t* src, const double* w, const double* bias,
                           tt_affine_layer** out);
int tt_affine_layer_apply(tt_session* s, const tt_affine_layer* layer, const double* in,
                          double* out, int64_t chain_in, int64_t* chain_out);
void tt_affine_layer_destroy(tt_session* s, tt_affine_layer* layer);

/* ---- diagnostics ------------------------------------------------------- */
/* Force the reduction kernel path (tests / A-B measurement): 0 = best
 * eligible (default), 1 = TMA-ring fused kernel (whole-tile tree),
 * 2 = register-tree fused kernel, 3 = generic program interpreter,
 * 4 = TMA-ring sliding-window kernel.  Results are identical on every path;
 * only speed differs. */
int tt_set_kernel_path(int path);
int tt_kernel_path(void);
/* The persistent chain kernel (fold units + in-tile tree items of one or two
 * products from one dependency-ordered queue): 1 = on, 0 = off (default;
 * env TT_CHAIN).  Results are identical either way. */
int tt_set_chain_kernel(int on);
int tt_chain_kernel(void);

/* ---- sharding (north star item 5) -------------------------------------- */
/* Block-partition external dim `shard_dim` (1-based) of `shape` over
 * `world` ranks; rank r owns external indices [*begin, *end).  Returns the
 * rank's local shape (same dims, n restricted to the slab). */
int tt_shard_plan(const tt_shape* shape, int shard_dim, int world, int rank, int64_t* begin,
                  int64_t* end, tt_shape* local_shape);

#ifdef __cplusplus
}
#endif

#endif /* TILETENSOR_B200_H */

// tt_internal.hpp -- host-side internals of libtiletensor_b200 (not installed).
//
// Shape algebra, the rotate-and-sum schedule compiler and the launch API the
// C-ABI (tt_capi.cpp) dispatches to.  Semantics follow the reference headers
// /root/reference/proj/include/tiletensor/*.hpp (cited per declaration).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "tiletensor_b200.h"

namespace ttb {

// Carries a tt_status code and, for parse errors, the position.
struct Error : std::runtime_error {
  int code;
  int64_t position;
  Error(int c, const std::string& msg, int64_t pos = -1)
      : std::runtime_error(msg), code(c), position(pos) {}
};

[[noreturn]] inline void shape_error(const std::string& m) { throw Error(TT_ERR_SHAPE, m); }
[[noreturn]] inline void invalid_argument(const std::string& m) {
  throw Error(TT_ERR_INVALID_ARGUMENT, m);
}
[[noreturn]] inline void depth_error(const std::string& m) { throw Error(TT_ERR_DEPTH, m); }

// DimSpec shape.hpp:37-49 (+ the builder's `~` interleaved flag).
struct Dim {
  int64_t n = 1, d = 1, t = 1;
  bool unknown = false;
  bool interleaved = false;
  int64_t used() const { return n * d; }
  bool fully_replicated() const { return n == 1 && d == t; }
  bool operator==(const Dim&) const = default;
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// TileTensorShape shape.hpp:72-138.
struct Shape {
  std::vector<Dim> dims;
  bool relaxed = false;

  int rank() const { return static_cast<int>(dims.size()); }
  const Dim& dim(int i) const { return dims.at(static_cast<size_t>(i)); }
  int64_t tile_slots() const {
    int64_t p = 1;
    for (const auto& d : dims) p *= d.t;
    return p;
  }
  int64_t ext(int i) const { return ceil_div(dims[i].used(), dims[i].t); }
  std::vector<int64_t> external() const {
    std::vector<int64_t> e;
    for (int i = 0; i < rank(); ++i) e.push_back(ext(i));
    return e;
  }
  int64_t tile_count() const {
    int64_t p = 1;
    for (int i = 0; i < rank(); ++i) p *= ext(i);
    return p;
  }
  int64_t used_slots() const {
    int64_t p = 1;
    for (const auto& d : dims) p *= d.used();
    return p;
  }
  int64_t dense_count() const {
    int64_t p = 1;
    for (const auto& d : dims) p *= d.n;
    return p;
  }
  bool has_unknown() const {
    for (const auto& d : dims)
      if (d.unknown) return true;
    return false;
  }
  bool operator==(const Shape&) const = default;
};

void check_shape(const Shape& s);  // TileTensorShape ctor checks shape.hpp:74-78
Shape from_c(const tt_shape* s);   // validates
void to_c(const Shape& s, tt_shape* out);
Shape parse_shape(std::string_view text);               // shape.hpp:144-252
std::string format_shape(const Shape& s);               // shape.hpp:256-278
Shape elementwise_result_shape(const Shape& a, const Shape& b, int op);  // shape.hpp:293-337
Shape sum_result_shape(const Shape& s, int dim);        // shape.hpp:357-377
std::vector<int64_t> tile_strides(const Shape& s);      // tile_tensor.hpp:31-39
std::vector<int64_t> row_major_strides(const std::vector<int64_t>& e);  // tile_tensor.hpp:41-49

// ---- group programs ---------------------------------------------------------
// Every reduction on the path (tt_sum, the fused mul+sum, sum_tile_strided,
// replicate_tile_dim, replicate_dim) is compiled on the host into a short
// program that one CTA runs per output tile ("group").  Instructions:
//   FOLD(dst, first, count): dst = P[first] + P[first+1] + ... (left fold,
//       tile_tensor.hpp:323-324), P[l] = A-tile (times B-tile when fused);
//   ROTADD(dst, a, b, r):     dst[j] = a[j] + b[(j + r) mod s]
//       == Session::add(a, Session::rotate(b, r)) (backend.hpp:117,152);
//   COPY(dst, a).
// Buffers are per-group scratch tiles; BUF_OUT is the group's output tile.
enum GOpKind : int8_t { GOP_FOLD = 0, GOP_ROTADD = 1, GOP_COPY = 2 };
constexpr int8_t BUF_OUT = -1;

struct GOp {
  int8_t kind;
  int8_t dst;
  int8_t a;
  int8_t b;
  int32_t inplace;  // dst aliases a or b: read phase, barrier, write phase
  int64_t x;        // FOLD: first; ROTADD: normalised rotation r in [0, s)
  int64_t y;        // FOLD: count
};

constexpr int kMaxOps = 96;

struct Program {
  std::vector<GOp> ops;
  int nbuf = 0;
  tt_cost per_group{};  // primitives the reference issues per group
  bool simple_pow2 = false;  // FOLD(B0) then in-place ROTADDs, last into OUT
};

// Builds the reduction program for one group of a tt_sum over a dim with
// external extent `ei`, in-tile extent `t`, in-tile stride `stride`, slot
// count `s`, used extent `used` and unknown flag (tile_tensor.hpp:286-347).
// `variant` < 0 is auto.  Throws invalid_argument exactly where the
// reference's sum_tile_strided would (rotate_sum.hpp:52-53,58-59).
Program build_sum_program(int64_t ei, int64_t t, int64_t stride, int64_t s, int64_t used,
                          bool unknown, int variant);
// sum_tile_strided on a single tile (rotate_sum.hpp:44-90): FOLD(count 1) + schedule.
Program build_strided_program(int64_t n, int64_t stride, int64_t s, int variant);
// replicate_tile_dim (rotate_sum.hpp:128-152).
Program build_replicate_program(int64_t t, int64_t stride, int64_t s);

// Closed forms rotate_sum.hpp:33-39.
int64_t rotations_left_to_right(int64_t n);
int64_t rotations_right_to_left(int64_t n);

}  // namespace ttb

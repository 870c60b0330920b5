#pragma once

// Drop-in mirror of the reference's inc/shape.hpp (namespace tiletensor):
// DimSpec, TileTensorShape, parse_shape, format_shape, external_shape,
// elementwise_result_shape, sum_result_shape -- same names, signatures and
// exception types.  The grammar and rules execute in libtiletensor_b200
// (include/tiletensor_b200.h) so C++ callers, the Python binding and the
// kernels share one implementation.  Adds the `~` interleaved flag.

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "tiletensor_b200.h"

namespace tiletensor {

class ShapeError : public std::runtime_error {
 public:
  explicit ShapeError(const std::string& msg) : std::runtime_error(msg) {}
};

class ShapeParseError : public ShapeError {
 public:
  ShapeParseError(const std::string& msg, std::size_t position)
      : ShapeError(msg), position_(position) {}
  std::size_t position() const { return position_; }

 private:
  std::size_t position_;
};

class DepthExhaustedError : public std::runtime_error {
 public:
  explicit DepthExhaustedError(const std::string& msg) : std::runtime_error(msg) {}
};

class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& msg) : std::runtime_error(msg) {}
};

namespace detail {

// Rethrows a C-ABI status as the reference's exception type.
inline void check(int rc) {
  if (rc == TT_OK) return;
  const std::string msg = tt_last_error();
  switch (rc) {
    case TT_ERR_SHAPE: throw ShapeError(msg);
    case TT_ERR_SHAPE_PARSE:
      throw ShapeParseError(msg, static_cast<std::size_t>(tt_last_error_position()));
    case TT_ERR_DEPTH: throw DepthExhaustedError(msg);
    case TT_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case TT_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case TT_ERR_CUDA:
    case TT_ERR_NO_DEVICE: throw CudaError(msg);
    default: throw std::logic_error(msg);
  }
}

}  // namespace detail

struct DimSpec {
  std::int64_t n = 1;
  std::int64_t d = 1;
  std::int64_t t = 1;
  bool unknown = false;
  bool interleaved = false;  // `~` (builder's extension)

  std::int64_t used() const { return n * d; }
  bool fully_replicated() const { return n == 1 && d == t; }
  bool operator==(const DimSpec&) const = default;
};

using ExternalShape = std::vector<std::int64_t>;

class TileTensorShape {
 public:
  explicit TileTensorShape(std::vector<DimSpec> dims, bool relaxed = false)
      : dims_(std::move(dims)), relaxed_(relaxed) {
    if (dims_.empty()) throw ShapeError("shape must have at least one dimension");
    const tt_shape c = to_c();
    detail::check(tt_shape_check(&c));
  }

  static TileTensorShape from_c(const tt_shape& c) {
    std::vector<DimSpec> dims;
    for (int i = 0; i < c.rank; ++i)
      dims.push_back(DimSpec{c.dims[i].n, c.dims[i].d, c.dims[i].t, c.dims[i].unknown != 0,
                             c.dims[i].interleaved != 0});
    return TileTensorShape(std::move(dims), c.relaxed != 0);
  }

  tt_shape to_c() const {
    tt_shape c;
    std::memset(&c, 0, sizeof(c));
    if (dims_.size() > TT_MAX_RANK) throw ShapeError("rank exceeds the supported maximum");
    c.rank = static_cast<int32_t>(dims_.size());
    c.relaxed = relaxed_ ? 1 : 0;
    for (std::size_t i = 0; i < dims_.size(); ++i) {
      c.dims[i].n = dims_[i].n;
      c.dims[i].d = dims_[i].d;
      c.dims[i].t = dims_[i].t;
      c.dims[i].unknown = dims_[i].unknown ? 1 : 0;
      c.dims[i].interleaved = dims_[i].interleaved ? 1 : 0;
    }
    return c;
  }

  std::size_t rank() const { return dims_.size(); }
  const std::vector<DimSpec>& dims() const { return dims_; }
  const DimSpec& dim(std::size_t i) const { return dims_.at(i); }
  bool relaxed() const { return relaxed_; }

  std::int64_t tile_slots() const {
    std::int64_t p = 1;
    for (const auto& ds : dims_) p *= ds.t;
    return p;
  }
  std::vector<std::int64_t> tensor_extents() const {
    std::vector<std::int64_t> out;
    for (const auto& ds : dims_) out.push_back(ds.n);
    return out;
  }
  ExternalShape external_extents() const {
    ExternalShape out;
    for (const auto& ds : dims_) out.push_back((ds.used() + ds.t - 1) / ds.t);
    return out;
  }
  std::int64_t tile_count() const {
    std::int64_t p = 1;
    for (auto e : external_extents()) p *= e;
    return p;
  }
  std::int64_t used_slots() const {
    std::int64_t p = 1;
    for (const auto& ds : dims_) p *= ds.used();
    return p;
  }
  std::int64_t total_slots() const { return tile_count() * tile_slots(); }
  bool has_unknown() const {
    for (const auto& ds : dims_)
      if (ds.unknown) return true;
    return false;
  }
  TileTensorShape with_dim(std::size_t i, DimSpec ds) const {
    auto dims = dims_;
    dims.at(i) = ds;
    return TileTensorShape(std::move(dims), relaxed_);
  }
  bool operator==(const TileTensorShape&) const = default;

 private:
  std::vector<DimSpec> dims_;
  bool relaxed_;
};

inline TileTensorShape parse_shape(std::string_view text) {
  tt_shape c;
  const std::string s(text);
  detail::check(tt_shape_parse(s.c_str(), &c));
  return TileTensorShape::from_c(c);
}

inline std::string format_shape(const TileTensorShape& shape) {
  char buf[64 * TT_MAX_RANK + 64];
  const tt_shape c = shape.to_c();
  detail::check(tt_shape_format(&c, buf, sizeof(buf)));
  return buf;
}

inline ExternalShape external_shape(const TileTensorShape& shape) {
  return shape.external_extents();
}

enum class OpKind { add, mul };

inline TileTensorShape elementwise_result_shape(const TileTensorShape& a, const TileTensorShape& b,
                                                OpKind op) {
  const tt_shape ca = a.to_c(), cb = b.to_c();
  tt_shape out;
  detail::check(tt_shape_elementwise_result(&ca, &cb, op == OpKind::mul ? TT_OP_MUL : TT_OP_ADD,
                                            &out));
  return TileTensorShape::from_c(out);
}

inline TileTensorShape sum_result_shape(const TileTensorShape& shape, int dim) {
  const tt_shape c = shape.to_c();
  tt_shape out;
  detail::check(tt_shape_sum_result(&c, dim, &out));
  return TileTensorShape::from_c(out);
}

}  // namespace tiletensor

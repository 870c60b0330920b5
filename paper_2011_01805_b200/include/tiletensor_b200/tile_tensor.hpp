#pragma once

// Drop-in mirror of the reference's inc/tile_tensor.hpp: TileTensor,
// logical_indices, slot_of, pack, unpack, tt_elementwise / tt_add / tt_mul,
// tt_sum, clean_unknowns, replicate_dim, with_leading_unit_dim.
//
// A TileTensor keeps its tiles as ONE contiguous device array
// [tile_count][s] (the concatenation of the reference's tiles()[i].slots()).
// tiles() hands out a host mirror std::vector<Tile> built on demand; the
// mutable overload marks the mirror authoritative from then on: every later
// operator that reads the tensor uploads it first -- so code that edits slots
// in place (the reference's fuzzing tests do), including through a reference
// to tiles() kept across operator calls, keeps the reference semantics.  A
// tensor whose tiles were never handed out mutably is never re-uploaded.

#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <utility>
#include <vector>

#include "tiletensor_b200/backend.hpp"
#include "tiletensor_b200/dense.hpp"
#include "tiletensor_b200/rotate_sum.hpp"
#include "tiletensor_b200/shape.hpp"

namespace tiletensor {

inline std::vector<std::int64_t> logical_indices(const TileTensorShape& shape,
                                                 std::span<const std::int64_t> tile_index,
                                                 std::int64_t h) {
  if (tile_index.size() != shape.rank()) throw ShapeError("tile index rank mismatch");
  const tt_shape c = shape.to_c();
  std::vector<std::int64_t> j(shape.rank());
  detail::check(tt_logical_indices(&c, tile_index.data(), h, j.data()));
  return j;
}

inline std::pair<std::vector<std::int64_t>, std::int64_t> slot_of(
    const TileTensorShape& shape, std::span<const std::int64_t> j) {
  if (j.size() != shape.rank()) throw ShapeError("logical index rank mismatch");
  const tt_shape c = shape.to_c();
  std::vector<std::int64_t> l(shape.rank());
  std::int64_t h = 0;
  detail::check(tt_slot_of(&c, j.data(), l.data(), &h));
  return {std::move(l), h};
}

class TileTensor {
 public:
  // TileTensor(shape, tiles, session) tile_tensor.hpp:132-136: host tiles in.
  TileTensor(TileTensorShape shape, std::vector<Tile> tiles, Session& session)
      : shape_(std::move(shape)), session_(&session) {
    if (static_cast<std::int64_t>(tiles.size()) != shape_.tile_count())
      throw ShapeError("tile count does not match external shape");
    std::int64_t chain = session.max_chain_index();
    for (const auto& t : tiles) {
      if (static_cast<std::int64_t>(t.size()) != session.slot_count())
        throw std::invalid_argument("tile belongs to a backend with a different slot count");
      chain = std::min(chain, t.chain_index());
    }
    chain_ = chain;
    mirror_ = std::make_shared<std::vector<Tile>>(std::move(tiles));
    host_dirty_ = true;
  }

  // Device-resident construction (operators' results).
  TileTensor(TileTensorShape shape, std::shared_ptr<DeviceArray> dev, Session& session,
             std::int64_t chain)
      : shape_(std::move(shape)), session_(&session), dev_(std::move(dev)), chain_(chain) {}

  const TileTensorShape& shape() const { return shape_; }
  Session& session() const { return *session_; }
  std::size_t tile_count() const { return static_cast<std::size_t>(shape_.tile_count()); }

  const std::vector<Tile>& tiles() const { return mirror(); }
  std::vector<Tile>& tiles() {
    auto& m = mirror();
    // the caller may edit slots in place -- now or through the returned
    // reference at any later time -- so the mirror stays authoritative
    host_dirty_ = true;
    exposed_ = true;
    return m;
  }
  const Tile& tile_at(std::size_t flat) const { return mirror().at(flat); }
  std::int64_t chain_index() const {
    if ((host_dirty_ || exposed_) && mirror_) {
      std::int64_t c = session_->max_chain_index();
      for (const auto& t : *mirror_) c = std::min(c, t.chain_index());
      return c;
    }
    return chain_;
  }

  // Device array [tile_count][s]; uploads a dirty host mirror first.
  const double* device_data() const {
    sync_to_device();
    return dev_->get();
  }

 private:
  std::vector<Tile>& mirror() const {
    if (!mirror_) {
      const std::int64_t s = session_->slot_count();
      std::vector<double> host(static_cast<std::size_t>(shape_.tile_count() * s));
      if (!host.empty()) dev_->download(host.data(), static_cast<std::int64_t>(host.size()));
      auto v = std::make_shared<std::vector<Tile>>();
      v->reserve(tile_count());
      for (std::size_t i = 0; i < tile_count(); ++i)
        v->push_back(session_->make_tile(
            std::span<const double>(host.data() + i * s, static_cast<std::size_t>(s))));
      for (auto& t : *v) t = with_chain(t, chain_);
      mirror_ = v;
    }
    return *mirror_;
  }
  static Tile with_chain(const Tile& t, std::int64_t chain) {
    Tile out = t;
    out.chain_ = chain;
    return out;
  }
  void sync_to_device() const {
    if (dev_ && !host_dirty_ && !exposed_) return;
    const std::int64_t s = session_->slot_count();
    const std::int64_t n = shape_.tile_count() * s;
    if (!dev_) dev_ = std::make_shared<DeviceArray>(session_->handle(), std::max<std::int64_t>(n, 1));
    std::vector<double> host(static_cast<std::size_t>(n));
    std::int64_t chain = session_->max_chain_index();
    for (std::size_t i = 0; i < mirror_->size(); ++i) {
      const auto& t = (*mirror_)[i];
      if (static_cast<std::int64_t>(t.size()) != s)
        throw std::invalid_argument("tile belongs to a backend with a different slot count");
      std::copy(t.slots().begin(), t.slots().end(), host.begin() + static_cast<std::ptrdiff_t>(i * s));
      chain = std::min(chain, t.chain_index());
    }
    if (n) dev_->upload(host.data(), n);
    chain_ = chain;
    host_dirty_ = false;
  }

  TileTensorShape shape_;
  Session* session_;
  mutable std::shared_ptr<DeviceArray> dev_;
  mutable std::shared_ptr<std::vector<Tile>> mirror_;
  mutable std::int64_t chain_ = 0;
  mutable bool host_dirty_ = false;
  bool exposed_ = false;  // tiles() was handed out mutably: re-upload before every read
};

namespace detail {

inline std::shared_ptr<DeviceArray> alloc_tiles(Session& s, std::int64_t tiles) {
  return std::make_shared<DeviceArray>(s.handle(), std::max<std::int64_t>(tiles * s.slot_count(), 1));
}

}  // namespace detail

inline TileTensor with_leading_unit_dim(const TileTensor& t) {
  std::vector<DimSpec> dims;
  dims.push_back(DimSpec{});
  for (const auto& ds : t.shape().dims()) dims.push_back(ds);
  TileTensorShape shape(std::move(dims), t.shape().relaxed());
  auto dev = detail::alloc_tiles(t.session(), shape.tile_count());
  detail::check(tt_copy_d2d(t.session().handle(), dev->get(), t.device_data(),
                            shape.tile_count() * t.session().slot_count() * 8));
  return TileTensor(std::move(shape), dev, t.session(), t.chain_index());
}

inline TileTensor pack(const DenseTensor& tensor, const TileTensorShape& shape, Session& session) {
  if (shape.has_unknown())
    throw ShapeError("pack target shape may not contain '?': " + format_shape(shape));
  std::int64_t want = 1;
  for (auto e : shape.tensor_extents()) want *= e;
  if (static_cast<std::int64_t>(tensor.size()) != want)
    throw ShapeError("tensor of " + std::to_string(tensor.size()) + " values cannot pack into " +
                     format_shape(shape));
  DeviceArray dense(session.handle(), std::max<std::int64_t>(want, 1));
  dense.upload(tensor.values().data(), want);
  auto out = detail::alloc_tiles(session, shape.tile_count());
  const tt_shape c = shape.to_c();
  detail::check(tt_pack(session.handle(), dense.get(), &c, out->get()));
  return TileTensor(shape, out, session, session.max_chain_index());
}

inline DenseTensor unpack(const TileTensor& t) {
  const auto ext = t.shape().tensor_extents();
  std::int64_t n = 1;
  for (auto e : ext) n *= e;
  DeviceArray dense(t.session().handle(), std::max<std::int64_t>(n, 1));
  const tt_shape c = t.shape().to_c();
  detail::check(tt_unpack(t.session().handle(), &c, t.device_data(), dense.get()));
  std::vector<double> host(static_cast<std::size_t>(n));
  dense.download(host.data(), n);
  return DenseTensor(ext, std::move(host));
}

inline TileTensor tt_elementwise(const TileTensor& a, const TileTensor& b, OpKind op) {
  if (&a.session() != &b.session())
    throw std::invalid_argument("operands belong to different sessions");
  Session& s = a.session();
  const TileTensorShape res = elementwise_result_shape(a.shape(), b.shape(), op);
  auto out = detail::alloc_tiles(s, res.tile_count());
  const tt_shape ca = a.shape().to_c(), cb = b.shape().to_c();
  tt_shape co;
  std::int64_t chain = 0;
  detail::check(tt_elementwise(s.handle(), op == OpKind::mul ? TT_OP_MUL : TT_OP_ADD, &ca,
                               a.device_data(), a.chain_index(), &cb, b.device_data(),
                               b.chain_index(), &co, out->get(), &chain));
  return TileTensor(TileTensorShape::from_c(co), out, s, chain);
}

inline TileTensor tt_add(const TileTensor& a, const TileTensor& b) {
  return tt_elementwise(a, b, OpKind::add);
}
inline TileTensor tt_mul(const TileTensor& a, const TileTensor& b) {
  return tt_elementwise(a, b, OpKind::mul);
}

inline TileTensor tt_sum(const TileTensor& t, int dim,
                         std::optional<SumVariant> variant = std::nullopt) {
  Session& s = t.session();
  const TileTensorShape res = sum_result_shape(t.shape(), dim);
  auto out = detail::alloc_tiles(s, res.tile_count());
  const tt_shape ci = t.shape().to_c();
  tt_shape co;
  detail::check(tt_sum(s.handle(), &ci, t.device_data(), dim, detail::variant_code(variant), &co,
                       out->get()));
  return TileTensor(TileTensorShape::from_c(co), out, s, t.chain_index());
}

// tt_sum(tt_mul(a, b), dim) in one fused pass (no materialised product).
inline TileTensor tt_mul_sum(const TileTensor& a, const TileTensor& b, int dim,
                             std::optional<SumVariant> variant = std::nullopt) {
  if (&a.session() != &b.session())
    throw std::invalid_argument("operands belong to different sessions");
  Session& s = a.session();
  const TileTensorShape prod = elementwise_result_shape(a.shape(), b.shape(), OpKind::mul);
  const TileTensorShape res = sum_result_shape(prod, dim);
  auto out = detail::alloc_tiles(s, res.tile_count());
  const tt_shape ca = a.shape().to_c(), cb = b.shape().to_c();
  tt_shape co;
  std::int64_t chain = 0;
  detail::check(tt_mul_sum(s.handle(), &ca, a.device_data(), a.chain_index(), &cb,
                           b.device_data(), b.chain_index(), dim, detail::variant_code(variant),
                           &co, out->get(), &chain));
  return TileTensor(TileTensorShape::from_c(co), out, s, chain);
}

// clean_unknowns(tt_sum(tt_mul(a, b), dim)) with the mask applied in the
// reduction's last pass (pipeline()'s odd -> even seam, linalg.hpp:213-260).
// Shapes, chain index, counters and errors equal the two-call composition.
inline TileTensor tt_mul_sum_clean(const TileTensor& a, const TileTensor& b, int dim,
                                   std::optional<SumVariant> variant = std::nullopt) {
  if (&a.session() != &b.session())
    throw std::invalid_argument("operands belong to different sessions");
  Session& s = a.session();
  const TileTensorShape res =
      sum_result_shape(elementwise_result_shape(a.shape(), b.shape(), OpKind::mul), dim);
  auto out = detail::alloc_tiles(s, res.tile_count());
  const tt_shape ca = a.shape().to_c(), cb = b.shape().to_c();
  tt_shape co;
  std::int64_t chain = 0;
  detail::check(tt_mul_sum_clean(s.handle(), &ca, a.device_data(), a.chain_index(), &cb,
                                 b.device_data(), b.chain_index(), dim, detail::variant_code(variant),
                                 &co, out->get(), &chain));
  return TileTensor(TileTensorShape::from_c(co), out, s, chain);
}

// One fully connected stage of cryptonets_infer's tiled branch (nn.hpp:468-490):
// tt_sum(tt_mul(a, b), dim), then tt_add(., *c) when c is given, then
// tt_mul(., .) when square -- the tail fused into the reduction's tree pass.
// Shapes, chain index, counters and errors equal the three-call composition.
inline TileTensor tt_mul_sum_affine(const TileTensor& a, const TileTensor& b, int dim,
                                    const TileTensor* c, bool square,
                                    std::optional<SumVariant> variant = std::nullopt) {
  if (&a.session() != &b.session() || (c && &c->session() != &a.session()))
    throw std::invalid_argument("operands belong to different sessions");
  Session& s = a.session();
  TileTensorShape res = sum_result_shape(elementwise_result_shape(a.shape(), b.shape(), OpKind::mul), dim);
  if (c) res = elementwise_result_shape(res, c->shape(), OpKind::add);
  auto out = detail::alloc_tiles(s, res.tile_count());
  const tt_shape ca = a.shape().to_c(), cb = b.shape().to_c();
  const tt_shape cc = c ? c->shape().to_c() : tt_shape{};
  tt_shape co;
  std::int64_t chain = 0;
  detail::check(tt_mul_sum_affine(s.handle(), &ca, a.device_data(), a.chain_index(), &cb,
                                  b.device_data(), b.chain_index(), dim,
                                  detail::variant_code(variant), c ? &cc : nullptr,
                                  c ? c->device_data() : nullptr, c ? c->chain_index() : 0,
                                  square ? 1 : 0, &co, out->get(), &chain));
  return TileTensor(TileTensorShape::from_c(co), out, s, chain);
}

inline TileTensor clean_unknowns(const TileTensor& t) {
  if (!t.shape().has_unknown()) return t;
  Session& s = t.session();
  auto out = detail::alloc_tiles(s, t.shape().tile_count());
  const tt_shape ci = t.shape().to_c();
  tt_shape co;
  std::int64_t chain = 0;
  detail::check(tt_clean_unknowns(s.handle(), &ci, t.device_data(), t.chain_index(), &co,
                                  out->get(), &chain));
  return TileTensor(TileTensorShape::from_c(co), out, s, chain);
}

inline TileTensor replicate_dim(const TileTensor& t, int dim) {
  Session& s = t.session();
  auto out = detail::alloc_tiles(s, t.shape().tile_count());
  const tt_shape ci = t.shape().to_c();
  tt_shape co;
  detail::check(tt_replicate_dim(s.handle(), &ci, t.device_data(), dim, &co, out->get()));
  return TileTensor(TileTensorShape::from_c(co), out, s, t.chain_index());
}

}  // namespace tiletensor

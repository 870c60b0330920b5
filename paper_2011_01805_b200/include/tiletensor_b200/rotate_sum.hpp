#pragma once

// Drop-in mirror of the reference's inc/rotate_sum.hpp: the three
// rotate-and-sum schedules and tile-dimension replication.  Each call runs
// the schedule as one group program on the device (tt_sum_tile_strided /
// tt_replicate_tile_dim), issuing exactly the reference's additions and
// rotations (same association, same counters).

#include <bit>
#include <cstdint>
#include <optional>
#include <span>
#include <vector>

#include "tiletensor_b200/backend.hpp"

namespace tiletensor {

enum class SumVariant { left_to_right, right_to_left, power_of_two };

inline std::int64_t rotations_left_to_right(std::int64_t n) { return tt_rotations_left_to_right(n); }
inline std::int64_t rotations_right_to_left(std::int64_t n) { return tt_rotations_right_to_left(n); }

namespace detail {
inline int variant_code(std::optional<SumVariant> v) {
  return v ? static_cast<int>(*v) : TT_VARIANT_AUTO;
}
}  // namespace detail

inline Tile sum_tile_strided(Session& session, const Tile& tile, std::int64_t n,
                             std::int64_t stride, SumVariant variant) {
  if (n < 1 || n > session.slot_count())
    throw std::invalid_argument("sum length must be in [1, slot count]");
  if (n == 1) return tile;
  return session.run_tile_program(tile, [&](tt_session* s, const double* in, double* out) {
    return tt_sum_tile_strided(s, in, n, stride, static_cast<int>(variant), out, 1);
  });
}

inline Tile sum_tile_flat(Session& session, const Tile& tile, std::int64_t n, SumVariant variant) {
  return sum_tile_strided(session, tile, n, 1, variant);
}

inline SumVariant auto_variant(std::int64_t n) {
  return (n > 0 && (n & (n - 1)) == 0) ? SumVariant::power_of_two : SumVariant::right_to_left;
}

inline Tile sum_tile_dim(Session& session, const Tile& tile,
                         std::span<const std::int64_t> tile_extents, int dim,
                         std::optional<SumVariant> variant = std::nullopt) {
  if (dim < 1 || static_cast<std::size_t>(dim) > tile_extents.size())
    throw std::invalid_argument("tile dimension out of range");
  if (tile_extents[static_cast<std::size_t>(dim - 1)] == 1) return tile;
  const std::vector<std::int64_t> ext(tile_extents.begin(), tile_extents.end());
  return session.run_tile_program(tile, [&](tt_session* s, const double* in, double* out) {
    return tt_sum_tile_dim(s, in, ext.data(), static_cast<int>(ext.size()), dim,
                           detail::variant_code(variant), out, 1);
  });
}

inline Tile replicate_tile_dim(Session& session, const Tile& tile,
                               std::span<const std::int64_t> tile_extents, int dim) {
  if (dim < 1 || static_cast<std::size_t>(dim) > tile_extents.size())
    throw std::invalid_argument("tile dimension out of range");
  if (tile_extents[static_cast<std::size_t>(dim - 1)] == 1) return tile;
  const std::vector<std::int64_t> ext(tile_extents.begin(), tile_extents.end());
  return session.run_tile_program(tile, [&](tt_session* s, const double* in, double* out) {
    return tt_replicate_tile_dim(s, in, ext.data(), static_cast<int>(ext.size()), dim, out, 1);
  });
}

}  // namespace tiletensor

#pragma once

// Drop-in mirror of the reference's inc/backend.hpp: BackendConfig,
// CostReport, Tile, Session -- same names, signatures, counters and
// exceptions.  A Session owns a libtiletensor_b200 session (one CUDA device,
// one stream, atomic counters).  Tiles are value objects whose slots live in
// host memory exactly like the reference's (so `slots()` stays a mutable
// std::vector<double>&); every primitive on them runs the sm_100a kernels
// through the C-ABI (DeviceArray staging), never a CPU loop.  Tile tensors
// (tile_tensor.hpp) keep their tiles resident on the device instead.

#include <atomic>
#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "tiletensor_b200/shape.hpp"

namespace tiletensor {

struct BackendConfig {
  std::int64_t slot_count = 1;
  std::int64_t max_chain_index = 1;
};

struct CostReport {
  std::uint64_t additions = 0;
  std::uint64_t multiplications = 0;
  std::uint64_t mask_multiplications = 0;
  std::uint64_t rotations = 0;
  std::uint64_t bootstraps = 0;
  std::uint64_t power_of_two_rotations = 0;

  std::string to_text(bool extended = false) const {
    std::string out;
    out += "additions=" + std::to_string(additions) + "\n";
    out += "multiplications=" + std::to_string(multiplications) + "\n";
    out += "mask_multiplications=" + std::to_string(mask_multiplications) + "\n";
    out += "rotations=" + std::to_string(rotations) + "\n";
    out += "bootstraps=" + std::to_string(bootstraps) + "\n";
    if (extended) out += "power_of_two_rotations=" + std::to_string(power_of_two_rotations) + "\n";
    return out;
  }
  CostReport since(const CostReport& b) const {
    return CostReport{additions - b.additions, multiplications - b.multiplications,
                      mask_multiplications - b.mask_multiplications, rotations - b.rotations,
                      bootstraps - b.bootstraps, power_of_two_rotations - b.power_of_two_rotations};
  }
  std::uint64_t total_ops() const {
    return additions + multiplications + mask_multiplications + rotations + bootstraps;
  }
};

class Session;

// RAII device allocation through the C-ABI.
class DeviceArray {
 public:
  DeviceArray(tt_session* s, std::int64_t count) : s_(s), count_(count) {
    void* p = nullptr;
    detail::check(tt_device_alloc(s_, count * static_cast<std::int64_t>(sizeof(double)), &p));
    ptr_ = static_cast<double*>(p);
  }
  ~DeviceArray() {
    if (ptr_) tt_device_free(s_, ptr_);
  }
  DeviceArray(const DeviceArray&) = delete;
  DeviceArray& operator=(const DeviceArray&) = delete;
  double* get() const { return ptr_; }
  std::int64_t size() const { return count_; }
  void upload(const double* host, std::int64_t count) {
    detail::check(tt_copy_h2d(s_, ptr_, host, count * static_cast<std::int64_t>(sizeof(double))));
  }
  void download(double* host, std::int64_t count) const {
    detail::check(tt_copy_d2h(s_, host, ptr_, count * static_cast<std::int64_t>(sizeof(double))));
  }

 private:
  tt_session* s_;
  std::int64_t count_;
  double* ptr_ = nullptr;
};

class Tile {
 public:
  Tile() = default;
  const std::vector<double>& slots() const { return slots_; }
  std::vector<double>& slots() { return slots_; }
  std::size_t size() const { return slots_.size(); }
  std::int64_t chain_index() const { return chain_; }

 private:
  friend class Session;
  friend class TileTensor;
  Tile(std::vector<double> slots, std::int64_t chain) : slots_(std::move(slots)), chain_(chain) {}
  std::vector<double> slots_;
  std::int64_t chain_ = 0;
};

class Session {
 public:
  explicit Session(BackendConfig cfg, int device = 0) : cfg_(cfg) {
    if (cfg_.slot_count < 1) throw std::invalid_argument("slot count must be >= 1");
    if (cfg_.max_chain_index < 1) throw std::invalid_argument("max chain index must be >= 1");
    detail::check(tt_session_create(cfg_.slot_count, cfg_.max_chain_index, device, &s_));
  }
  Session(std::int64_t slots, std::int64_t depth) : Session(BackendConfig{slots, depth}) {}
  ~Session() { tt_session_destroy(s_); }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  std::int64_t slot_count() const { return cfg_.slot_count; }
  std::int64_t max_chain_index() const { return cfg_.max_chain_index; }
  const BackendConfig& config() const { return cfg_; }
  tt_session* handle() const { return s_; }

  Tile make_tile(std::span<const double> values) const {
    if (static_cast<std::int64_t>(values.size()) != cfg_.slot_count)
      throw std::invalid_argument("tile expects " + std::to_string(cfg_.slot_count) +
                                  " values, got " + std::to_string(values.size()));
    return Tile(std::vector<double>(values.begin(), values.end()), cfg_.max_chain_index);
  }
  Tile zero_tile() const {
    return Tile(std::vector<double>(static_cast<std::size_t>(cfg_.slot_count), 0.0),
                cfg_.max_chain_index);
  }
  Tile constant_tile(double value) const {
    return Tile(std::vector<double>(static_cast<std::size_t>(cfg_.slot_count), value),
                cfg_.max_chain_index);
  }

  Tile add(const Tile& a, const Tile& b) { return binary(TT_OP_ADD, a, b); }
  Tile mul(const Tile& a, const Tile& b) { return binary(TT_OP_MUL, a, b); }

  Tile mask_mul(const Tile& a, std::span<const double> mask) {
    check_width(a);
    if (static_cast<std::int64_t>(mask.size()) != cfg_.slot_count)
      throw std::invalid_argument("mask length does not match slot count");
    DeviceArray buf(s_, 3 * cfg_.slot_count);
    const std::int64_t s = cfg_.slot_count;
    buf.upload(a.slots_.data(), s);
    detail::check(tt_copy_h2d(s_, buf.get() + s, mask.data(), s * 8));
    std::int64_t chain_out = 0;
    detail::check(tt_tiles_mask_mul(s_, buf.get(), buf.get() + s, buf.get() + 2 * s, 1, &a.chain_,
                                    &chain_out));
    Tile out(std::vector<double>(static_cast<std::size_t>(s)), chain_out);
    detail::check(tt_copy_d2h(s_, out.slots_.data(), buf.get() + 2 * s, s * 8));
    return out;
  }

  // Cyclic left rotation out[j] = in[(j + offset) mod s]; r == 0 is free.
  Tile rotate(const Tile& a, std::int64_t offset) {
    check_width(a);
    const std::int64_t s = cfg_.slot_count;
    if (((offset % s) + s) % s == 0) return a;
    DeviceArray buf(s_, 2 * s);
    buf.upload(a.slots_.data(), s);
    detail::check(tt_tiles_rotate(s_, buf.get(), offset, buf.get() + s, 1));
    Tile out(std::vector<double>(static_cast<std::size_t>(s)), a.chain_);
    detail::check(tt_copy_d2h(s_, out.slots_.data(), buf.get() + s, s * 8));
    return out;
  }

  Tile bootstrap(const Tile& a) {
    check_width(a);
    tt_session_count_bootstraps(s_, 1);
    return Tile(a.slots_, cfg_.max_chain_index);
  }

  CostReport cost_report() const {
    tt_cost c;
    tt_session_cost(s_, &c);
    return CostReport{c.additions, c.multiplications, c.mask_multiplications, c.rotations,
                      c.bootstraps, c.power_of_two_rotations};
  }
  void reset_counters() { tt_session_reset_counters(s_); }
  std::uint64_t kernel_launches() const { return tt_session_launches(s_); }

  // Runs a single-tile schedule program (rotate_sum.hpp) on the device.
  template <typename Fn>
  Tile run_tile_program(const Tile& a, Fn&& fn) {
    check_width(a);
    const std::int64_t s = cfg_.slot_count;
    DeviceArray buf(s_, 2 * s);
    buf.upload(a.slots_.data(), s);
    detail::check(fn(s_, buf.get(), buf.get() + s));
    Tile out(std::vector<double>(static_cast<std::size_t>(s)), a.chain_);
    detail::check(tt_copy_d2h(s_, out.slots_.data(), buf.get() + s, s * 8));
    return out;
  }

 private:
  Tile binary(int op, const Tile& a, const Tile& b) {
    check_width(a);
    check_width(b);
    const std::int64_t s = cfg_.slot_count;
    std::int64_t chain_out = 0;
    // chain checks happen before any launch (backend.hpp:129-131)
    DeviceArray buf(s_, 3 * s);
    buf.upload(a.slots_.data(), s);
    detail::check(tt_copy_h2d(s_, buf.get() + s, b.slots_.data(), s * 8));
    detail::check(tt_tiles_binary(s_, op, buf.get(), buf.get() + s, buf.get() + 2 * s, 1, &a.chain_,
                                  &b.chain_, &chain_out));
    Tile out(std::vector<double>(static_cast<std::size_t>(s)), chain_out);
    detail::check(tt_copy_d2h(s_, out.slots_.data(), buf.get() + 2 * s, s * 8));
    return out;
  }
  void check_width(const Tile& t) const {
    if (static_cast<std::int64_t>(t.slots_.size()) != cfg_.slot_count)
      throw std::invalid_argument("tile belongs to a backend with a different slot count");
  }

  BackendConfig cfg_;
  tt_session* s_ = nullptr;
};

}  // namespace tiletensor

// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (see oracle/tt_oracle.c header).  Compiled by
// oracle/Makefile with -I/root/reference/proj/include into
// oracle/_ref/libttref.so (git-ignored).  Nothing here re-implements the
// algorithm: every entry point builds reference objects (DenseTensor,
// TileTensorShape, Session, TileTensor) from plain buffers and calls the
// reference's own functions, so its outputs ARE the reference's outputs.
// Used to (1) pin the C restatement oracle/tt_oracle.c, (2) generate the
// golden fixtures under tests/golden/, (3) time the reference CPU path
// (bench.py --impl reference, cpu_baseline kind "reference").
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <span>
#include <sstream>
#include <string>
#include <vector>

#include "tiletensor/linalg.hpp"
#include "tiletensor/nn.hpp"
#include "tiletensor/rotate_sum.hpp"
#include "tiletensor/tile_tensor.hpp"
#include "../include/tiletensor_b200.h"

using namespace tiletensor;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const ShapeParseError& e) {
    return fail(2, e.what());
  } catch (const ShapeError& e) {
    return fail(1, e.what());
  } catch (const DepthExhaustedError& e) {
    return fail(3, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(4, e.what());
  } catch (const std::out_of_range& e) {
    return fail(5, e.what());
  } catch (const std::exception& e) {
    return fail(6, e.what());
  }
}

TileTensorShape to_ref(const tt_shape* s) {
  std::vector<DimSpec> dims;
  for (int i = 0; i < s->rank; ++i) {
    DimSpec d;
    d.n = s->dims[i].n;
    d.d = s->dims[i].d;
    d.t = s->dims[i].t;
    d.unknown = s->dims[i].unknown != 0;
    dims.push_back(d);
  }
  return TileTensorShape(std::move(dims), s->relaxed != 0);
}

void from_ref(const TileTensorShape& r, tt_shape* out) {
  std::memset(out, 0, sizeof(*out));
  out->rank = static_cast<int32_t>(r.rank());
  out->relaxed = r.relaxed() ? 1 : 0;
  for (std::size_t i = 0; i < r.rank(); ++i) {
    out->dims[i].n = r.dim(i).n;
    out->dims[i].d = r.dim(i).d;
    out->dims[i].t = r.dim(i).t;
    out->dims[i].unknown = r.dim(i).unknown ? 1 : 0;
  }
}

std::vector<Tile> make_tiles(Session& session, const double* tiles, int64_t count) {
  std::vector<Tile> out;
  out.reserve(static_cast<std::size_t>(count));
  const int64_t s = session.slot_count();
  for (int64_t i = 0; i < count; ++i)
    out.push_back(session.make_tile(std::span<const double>(tiles + i * s, static_cast<std::size_t>(s))));
  return out;
}

void dump_tiles(const TileTensor& t, double* out) {
  const int64_t s = t.session().slot_count();
  for (std::size_t i = 0; i < t.tile_count(); ++i)
    std::memcpy(out + static_cast<int64_t>(i) * s, t.tile_at(i).slots().data(),
                static_cast<std::size_t>(s) * sizeof(double));
}

void dump_cost(const Session& s, tt_cost* c) {
  if (!c) return;
  const CostReport r = s.cost_report();
  c->additions = r.additions;
  c->multiplications = r.multiplications;
  c->mask_multiplications = r.mask_multiplications;
  c->rotations = r.rotations;
  c->bootstraps = r.bootstraps;
  c->power_of_two_rotations = r.power_of_two_rotations;
}

std::optional<SumVariant> to_variant(int v) {
  if (v < 0) return std::nullopt;
  return static_cast<SumVariant>(v);
}

DenseTensor dense_of(const double* v, const tt_shape* s) {
  std::vector<std::int64_t> ext;
  std::int64_t n = 1;
  for (int i = 0; i < s->rank; ++i) {
    ext.push_back(s->dims[i].n);
    n *= s->dims[i].n;
  }
  return DenseTensor(ext, std::vector<double>(v, v + n));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// TILETENSOR_THREADS is read once by the reference (tile_tensor.hpp:53-61).
void ref_set_threads(int n) {
  const std::string v = std::to_string(n);
  setenv("TILETENSOR_THREADS", v.c_str(), 1);
}
int ref_thread_hint() { return detail::thread_hint(); }

int ref_shape_parse(const char* text, tt_shape* out, int64_t* pos) {
  *pos = -1;
  try {
    from_ref(parse_shape(text), out);
    return 0;
  } catch (const ShapeParseError& e) {
    *pos = static_cast<int64_t>(e.position());
    return fail(2, e.what());
  } catch (const ShapeError& e) {
    return fail(1, e.what());
  }
}

int ref_shape_format(const tt_shape* s, char* buf, int64_t cap) {
  return guard([&] {
    const std::string f = format_shape(to_ref(s));
    std::strncpy(buf, f.c_str(), static_cast<std::size_t>(cap));
    buf[cap - 1] = '\0';
  });
}

int ref_elementwise_result_shape(const tt_shape* a, const tt_shape* b, int op, tt_shape* out) {
  return guard([&] {
    from_ref(elementwise_result_shape(to_ref(a), to_ref(b), op ? OpKind::mul : OpKind::add), out);
  });
}

int ref_sum_result_shape(const tt_shape* s, int dim, tt_shape* out) {
  return guard([&] { from_ref(sum_result_shape(to_ref(s), dim), out); });
}

int ref_pack(const double* dense, const tt_shape* shape, int64_t slots, double* tiles, tt_cost* c) {
  return guard([&] {
    Session session(slots, 1);
    const TileTensor t = pack(dense_of(dense, shape), to_ref(shape), session);
    dump_tiles(t, tiles);
    dump_cost(session, c);
  });
}

int ref_unpack(const tt_shape* shape, int64_t slots, const double* tiles, double* dense) {
  return guard([&] {
    Session session(slots, 1);
    const TileTensorShape sh = to_ref(shape);
    const TileTensor t(sh, make_tiles(session, tiles, sh.tile_count()), session);
    const DenseTensor d = unpack(t);
    std::memcpy(dense, d.values().data(), d.size() * sizeof(double));
  });
}

int ref_elementwise(int op, const tt_shape* sa, const double* ta, const tt_shape* sb,
                    const double* tb, int64_t slots, tt_shape* so, double* out, tt_cost* c) {
  return guard([&] {
    Session session(slots, 8);
    const TileTensorShape a = to_ref(sa), b = to_ref(sb);
    const TileTensor xa(a, make_tiles(session, ta, a.tile_count()), session);
    const TileTensor xb(b, make_tiles(session, tb, b.tile_count()), session);
    const TileTensor r = tt_elementwise(xa, xb, op ? OpKind::mul : OpKind::add);
    from_ref(r.shape(), so);
    dump_tiles(r, out);
    dump_cost(session, c);
  });
}

int ref_sum(const tt_shape* sh, const double* tin, int64_t slots, int dim, int variant,
            tt_shape* so, double* out, tt_cost* c) {
  return guard([&] {
    Session session(slots, 8);
    const TileTensorShape s = to_ref(sh);
    const TileTensor x(s, make_tiles(session, tin, s.tile_count()), session);
    const TileTensor r = tt_sum(x, dim, to_variant(variant));
    from_ref(r.shape(), so);
    dump_tiles(r, out);
    dump_cost(session, c);
  });
}

// tt_sum(tt_mul(a, b), dim) -- the two-line product body (linalg.hpp:41-73).
int ref_mul_sum(const tt_shape* sa, const double* ta, const tt_shape* sb, const double* tb,
                int64_t slots, int dim, int variant, tt_shape* so, double* out, tt_cost* c) {
  return guard([&] {
    Session session(slots, 8);
    const TileTensorShape a = to_ref(sa), b = to_ref(sb);
    const TileTensor xa(a, make_tiles(session, ta, a.tile_count()), session);
    const TileTensor xb(b, make_tiles(session, tb, b.tile_count()), session);
    const TileTensor r = tt_sum(tt_mul(xa, xb), dim, to_variant(variant));
    from_ref(r.shape(), so);
    dump_tiles(r, out);
    dump_cost(session, c);
  });
}

// matvec_a / matvec_b / matmul_a / matmul_b (linalg.hpp:41-73), which = 0..3.
int ref_linalg(int which, const tt_shape* sa, const double* ta, const tt_shape* sb,
               const double* tb, int64_t slots, tt_shape* so, double* out, tt_cost* c) {
  return guard([&] {
    Session session(slots, 8);
    const TileTensorShape a = to_ref(sa), b = to_ref(sb);
    const TileTensor xa(a, make_tiles(session, ta, a.tile_count()), session);
    const TileTensor xb(b, make_tiles(session, tb, b.tile_count()), session);
    TileTensor r = which == 0   ? matvec_a(xa, xb)
                   : which == 1 ? matvec_b(xa, xb)
                   : which == 2 ? matmul_a(xa, xb)
                                : matmul_b(xa, xb);
    from_ref(r.shape(), so);
    dump_tiles(r, out);
    dump_cost(session, c);
  });
}

// pipeline (linalg.hpp:213-260) on k matrices packed back to back in
// `mats` (matrix i is rows[i] x cols[i], row-major), vector v of length n;
// returns the output shape, tiles and the cost since the start.
int ref_pipeline(const double* mats, const int64_t* rows, const int64_t* cols, int k,
                 const double* v, int64_t n, int64_t t1, int64_t t2, int64_t slots,
                 int64_t depth, tt_shape* so, double* out, tt_cost* c) {
  return guard([&] {
    std::vector<DenseTensor> ms;
    const double* p = mats;
    for (int i = 0; i < k; ++i) {
      const int64_t cnt = rows[i] * cols[i];
      ms.emplace_back(std::vector<std::int64_t>{rows[i], cols[i]}, std::vector<double>(p, p + cnt));
      p += cnt;
    }
    Session session(slots, depth);
    const DenseTensor dv({n}, std::vector<double>(v, v + n));
    const auto res = pipeline(ms, dv, {t1, t2}, session);
    from_ref(res.out.shape(), so);
    dump_tiles(res.out, out);
    c->additions = res.cost.additions;
    c->multiplications = res.cost.multiplications;
    c->mask_multiplications = res.cost.mask_multiplications;
    c->rotations = res.cost.rotations;
    c->bootstraps = res.cost.bootstraps;
    c->power_of_two_rotations = res.cost.power_of_two_rotations;
  });
}

// score_tile_factorizations (linalg.hpp:279-294): writes up to `cap`
// (t1, rotations, total_ops) triples in the reference's order; returns count.
int ref_score_tile_factorizations(const double* mats, const int64_t* rows, const int64_t* cols,
                                  int k, const double* v, int64_t n, int64_t slots, int64_t depth,
                                  int64_t* triples, int cap, int* count) {
  return guard([&] {
    std::vector<DenseTensor> ms;
    const double* p = mats;
    for (int i = 0; i < k; ++i) {
      const int64_t cnt = rows[i] * cols[i];
      ms.emplace_back(std::vector<std::int64_t>{rows[i], cols[i]}, std::vector<double>(p, p + cnt));
      p += cnt;
    }
    const DenseTensor dv({n}, std::vector<double>(v, v + n));
    const auto choices = score_tile_factorizations(ms, dv, slots, depth);
    *count = static_cast<int>(choices.size());
    for (int i = 0; i < *count && i < cap; ++i) {
      triples[3 * i] = choices[i].t1;
      triples[3 * i + 1] = static_cast<int64_t>(choices[i].cost.rotations);
      triples[3 * i + 2] = static_cast<int64_t>(choices[i].cost.total_ops());
    }
  });
}

// nn.hpp: the network from a spec text + seed (parse_network), run through
// nn_forward (which = 0) or cryptonets_infer with tile t (which = 1) on a
// batch [features, n] (row-major); logits [out, n] into `out` (cap values).
int ref_nn_run(int which, const char* spec, uint64_t seed, const double* batch, int64_t features,
               int64_t n, const int64_t* tile, int64_t slots, int64_t depth, double* out,
               int64_t cap, int64_t* out_rows, tt_cost* c) {
  return guard([&] {
    std::istringstream in(spec);
    const NetworkSpec net = parse_network(in, "", seed);
    const DenseTensor b({features, n}, std::vector<double>(batch, batch + features * n));
    DenseTensor logits = DenseTensor::zeros({1});
    if (which == 0) {
      logits = nn_forward(net, b);
    } else {
      Session session(slots, depth);
      auto res = cryptonets_infer(net, b, {tile[0], tile[1], tile[2]}, session);
      logits = std::move(res.logits);
      c->additions = res.cost.additions;
      c->multiplications = res.cost.multiplications;
      c->mask_multiplications = res.cost.mask_multiplications;
      c->rotations = res.cost.rotations;
      c->bootstraps = res.cost.bootstraps;
      c->power_of_two_rotations = res.cost.power_of_two_rotations;
    }
    if (static_cast<int64_t>(logits.size()) > cap) throw std::invalid_argument("output buffer too small");
    *out_rows = logits.extent(0);
    std::memcpy(out, logits.values().data(), logits.size() * sizeof(double));
  });
}

// parse_network's seeded parameters, flattened in layer order (weights then bias)
int ref_nn_params(const char* spec, uint64_t seed, double* out, int64_t cap, int64_t* count) {
  return guard([&] {
    std::istringstream in(spec);
    const NetworkSpec net = parse_network(in, "", seed);
    int64_t k = 0;
    auto put = [&](const DenseTensor& t) {
      for (double v : t.values()) {
        if (k < cap) out[k] = v;
        ++k;
      }
    };
    for (const auto& layer : net.layers) {
      if (const auto* cv = std::get_if<ConvLayer>(&layer)) {
        put(cv->weights);
        put(cv->bias);
      } else if (const auto* f = std::get_if<FcLayer>(&layer)) {
        put(f->weights);
        put(f->bias);
      }
    }
    *count = k;
  });
}

int ref_clean_unknowns(const tt_shape* sh, const double* tin, int64_t slots, tt_shape* so,
                       double* out, tt_cost* c) {
  return guard([&] {
    Session session(slots, 8);
    const TileTensorShape s = to_ref(sh);
    const TileTensor x(s, make_tiles(session, tin, s.tile_count()), session);
    const TileTensor r = clean_unknowns(x);
    from_ref(r.shape(), so);
    dump_tiles(r, out);
    dump_cost(session, c);
  });
}

int ref_replicate_dim(const tt_shape* sh, const double* tin, int64_t slots, int dim, tt_shape* so,
                      double* out, tt_cost* c) {
  return guard([&] {
    Session session(slots, 8);
    const TileTensorShape s = to_ref(sh);
    const TileTensor x(s, make_tiles(session, tin, s.tile_count()), session);
    const TileTensor r = replicate_dim(x, dim);
    from_ref(r.shape(), so);
    dump_tiles(r, out);
    dump_cost(session, c);
  });
}

int ref_rotate(const double* in, int64_t slots, int64_t offset, double* out, tt_cost* c) {
  return guard([&] {
    Session session(slots, 1);
    const Tile t = session.make_tile(std::span<const double>(in, static_cast<std::size_t>(slots)));
    const Tile r = session.rotate(t, offset);
    std::memcpy(out, r.slots().data(), static_cast<std::size_t>(slots) * sizeof(double));
    dump_cost(session, c);
  });
}

int ref_sum_tile_strided(const double* in, int64_t slots, int64_t n, int64_t stride, int variant,
                         double* out, tt_cost* c) {
  return guard([&] {
    Session session(slots, 1);
    const Tile t = session.make_tile(std::span<const double>(in, static_cast<std::size_t>(slots)));
    const SumVariant v = variant < 0 ? auto_variant(n) : static_cast<SumVariant>(variant);
    const Tile r = sum_tile_strided(session, t, n, stride, v);
    std::memcpy(out, r.slots().data(), static_cast<std::size_t>(slots) * sizeof(double));
    dump_cost(session, c);
  });
}

int ref_replicate_tile_dim(const double* in, int64_t slots, const int64_t* extents, int rank,
                           int dim, double* out, tt_cost* c) {
  return guard([&] {
    Session session(slots, 1);
    const Tile t = session.make_tile(std::span<const double>(in, static_cast<std::size_t>(slots)));
    const Tile r = replicate_tile_dim(session, t, std::span<const int64_t>(extents, rank), dim);
    std::memcpy(out, r.slots().data(), static_cast<std::size_t>(slots) * sizeof(double));
    dump_cost(session, c);
  });
}

int ref_logical_indices(const tt_shape* sh, const int64_t* tile_index, int64_t h, int64_t* j) {
  return guard([&] {
    const TileTensorShape s = to_ref(sh);
    const auto r = logical_indices(s, std::span<const int64_t>(tile_index, s.rank()), h);
    for (std::size_t i = 0; i < r.size(); ++i) j[i] = r[i];
  });
}

// ---- timed CPU baseline helpers (bench.py) ----------------------------------
// A persistent session holding W packed once (W is a fixed operand, like a
// weight), so a timed step covers: pack X, tt_sum(tt_mul(X, W), k), unpack.
namespace {
std::unique_ptr<Session> g_bench_session;
std::unique_ptr<TileTensor> g_bench_w;
}  // namespace

int ref_bench_prepare_w(const double* dense_w, const tt_shape* sw, int64_t slots) {
  return guard([&] {
    g_bench_w.reset();
    g_bench_session = std::make_unique<Session>(slots, 8);
    g_bench_w = std::make_unique<TileTensor>(pack(dense_of(dense_w, sw), to_ref(sw), *g_bench_session));
  });
}

int ref_bench_step(const double* dense_x, const tt_shape* sx, const int* dims, int ndims,
                   double* secs) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    if (!g_bench_w) throw std::logic_error("ref_bench_prepare_w first");
    Session& session = *g_bench_session;
    auto t0 = clk::now();
    const TileTensor x = pack(dense_of(dense_x, sx), to_ref(sx), session);
    auto t1 = clk::now();
    std::vector<TileTensor> outs;
    for (int k = 0; k < ndims; ++k) outs.push_back(tt_sum(tt_mul(x, *g_bench_w), dims[k]));
    auto t2 = clk::now();
    double sink = 0;
    for (const auto& o : outs) sink += unpack(o).values()[0];
    auto t3 = clk::now();
    secs[0] = std::chrono::duration<double>(t1 - t0).count();
    secs[1] = std::chrono::duration<double>(t2 - t1).count();
    secs[2] = std::chrono::duration<double>(t3 - t2).count();
    secs[3] = sink;
  });
}
// Split form of ref_bench_step for the CPU baseline legs: pack X once
// (timed), run tt_sum(tt_mul(X, W), dim) over `dims` as many times as the
// caller asks (each call timed), unpack the last results once (timed).
std::unique_ptr<TileTensor> g_bench_x;
std::vector<TileTensor> g_bench_outs;

int ref_bench_pack_x(const double* dense_x, const tt_shape* sx, double* secs) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    if (!g_bench_w) throw std::logic_error("ref_bench_prepare_w first");
    g_bench_outs.clear();
    g_bench_x.reset();
    auto t0 = clk::now();
    g_bench_x = std::make_unique<TileTensor>(pack(dense_of(dense_x, sx), to_ref(sx), *g_bench_session));
    secs[0] = std::chrono::duration<double>(clk::now() - t0).count();
  });
}

int ref_bench_mul_sum(const int* dims, int ndims, double* secs) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    if (!g_bench_x) throw std::logic_error("ref_bench_pack_x first");
    g_bench_outs.clear();
    auto t0 = clk::now();
    for (int k = 0; k < ndims; ++k) g_bench_outs.push_back(tt_sum(tt_mul(*g_bench_x, *g_bench_w), dims[k]));
    secs[0] = std::chrono::duration<double>(clk::now() - t0).count();
  });
}

int ref_bench_unpack(double* secs) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    double sink = 0;
    for (const auto& o : g_bench_outs) sink += unpack(o).values()[0];
    secs[0] = std::chrono::duration<double>(clk::now() - t0).count();
    secs[1] = sink;
  });
}

// One call = pack a seeded dense tensor, then tt_sum(tt_mul(X, W), dim) for each
// dim in `dims`, then unpack each result, exactly through the reference API.
// Returns wall seconds of each phase in secs[0..2] (pack, mul+sum, unpack).
int ref_bench_pipeline(const double* dense_x, const tt_shape* sx, const double* dense_w,
                       const tt_shape* sw, int64_t slots, const int* dims, int ndims, double* secs) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    Session session(slots, 8);
    auto t0 = clk::now();
    const TileTensor x = pack(dense_of(dense_x, sx), to_ref(sx), session);
    const TileTensor w = pack(dense_of(dense_w, sw), to_ref(sw), session);
    auto t1 = clk::now();
    std::vector<TileTensor> outs;
    for (int k = 0; k < ndims; ++k) outs.push_back(tt_sum(tt_mul(x, w), dims[k]));
    auto t2 = clk::now();
    double sink = 0;
    for (const auto& o : outs) sink += unpack(o).values()[0];
    auto t3 = clk::now();
    secs[0] = std::chrono::duration<double>(t1 - t0).count();
    secs[1] = std::chrono::duration<double>(t2 - t1).count();
    secs[2] = std::chrono::duration<double>(t3 - t2).count();
    secs[3] = sink;
  });
}

}  // extern "C"

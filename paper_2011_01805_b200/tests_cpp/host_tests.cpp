// host_tests.cpp -- C++ tests of the drop-in headers (include/tiletensor_b200/*.hpp)
// against the reference's own test expectations (cases re-expressed from
// /root/reference/proj/tests/test_*.cpp, cited per case).  The code under test
// is exactly what a reference user would compile: `#include "tiletensor_b200/linalg.hpp"`
// and the unchanged tiletensor:: API, backed by the sm_100a kernels.
// Needs a GPU; run by tests/test_cpp_host.py.  Exit code = failed checks.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "tiletensor_b200/linalg.hpp"
#include "tiletensor_b200/formats.hpp"
#include "tiletensor_b200/nn.hpp"

using namespace tiletensor;

static int g_checks = 0, g_failed = 0;
#define CHECK(cond)                                                             \
  do {                                                                          \
    ++g_checks;                                                                 \
    if (!(cond)) {                                                              \
      ++g_failed;                                                               \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
    }                                                                           \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                                \
  do {                                                                          \
    ++g_checks;                                                                 \
    bool ok_ = false;                                                           \
    try {                                                                       \
      (void)(expr);                                                             \
    } catch (const T&) {                                                        \
      ok_ = true;                                                               \
    } catch (...) {                                                             \
    }                                                                           \
    if (!ok_) {                                                                 \
      ++g_failed;                                                               \
      std::fprintf(stderr, "FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); \
    }                                                                           \
  } while (0)

static DenseTensor random_tensor(std::vector<std::int64_t> shape, std::mt19937_64& rng,
                                 double lo = -2, double hi = 2) {
  std::int64_t n = 1;
  for (auto e : shape) n *= e;
  std::uniform_real_distribution<double> dist(lo, hi);
  std::vector<double> v(static_cast<std::size_t>(n));
  for (auto& x : v) x = dist(rng);
  return DenseTensor(std::move(shape), std::move(v));
}

static TileTensorShape random_pack_shape(std::mt19937_64& rng, std::int64_t slots, int rank,
                                         bool allow_rep = true) {
  std::vector<std::int64_t> t(static_cast<std::size_t>(rank), 1);
  std::int64_t rem = slots;
  for (int i = 0; i < rank - 1; ++i) {
    std::vector<std::int64_t> divs;
    for (std::int64_t x = 1; x <= rem; x *= 2) divs.push_back(x);
    t[i] = divs[std::uniform_int_distribution<std::size_t>(0, divs.size() - 1)(rng)];
    rem /= t[i];
  }
  t[rank - 1] = rem;
  std::vector<DimSpec> dims;
  for (int i = 0; i < rank; ++i) {
    DimSpec d;
    d.t = t[i];
    const int pick = std::uniform_int_distribution<int>(0, 3)(rng);
    if (allow_rep && pick == 0) {
      d.n = 1;
      d.d = d.t;
    } else if (allow_rep && pick == 1 && d.t > 1) {
      d.n = 1;
      d.d = std::uniform_int_distribution<std::int64_t>(1, d.t)(rng);
    } else {
      d.n = std::uniform_int_distribution<std::int64_t>(1, 12)(rng);
    }
    dims.push_back(d);
  }
  return TileTensorShape(dims);
}

static void fuzz_unknown_regions(TileTensor& t, std::uint64_t seed) {
  const TileTensorShape& shape = t.shape();
  if (!shape.has_unknown()) return;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-100, 100);
  const auto ext = shape.external_extents();
  std::vector<std::int64_t> idx(shape.rank(), 0);
  auto& tiles = t.tiles();
  for (std::size_t flat = 0; flat < t.tile_count(); ++flat) {
    for (std::int64_t h = 0; h < shape.tile_slots(); ++h) {
      const auto j = logical_indices(shape, idx, h);
      bool garbage = false;
      for (std::size_t i = 0; i < shape.rank(); ++i)
        if (shape.dim(i).unknown && j[i] >= shape.dim(i).used()) garbage = true;
      if (garbage) tiles[flat].slots()[static_cast<std::size_t>(h)] = dist(rng);
    }
    for (std::size_t i = shape.rank(); i-- > 0;) {
      if (++idx[i] < ext[i]) break;
      idx[i] = 0;
    }
  }
}


// ---- test_shape.cpp ---------------------------------------------------------
static void shapes() {
  CHECK(format_shape(parse_shape("[5/2,*3/4]")) == "[5/2,*3/4]");
  CHECK(parse_shape("[*/4,5/8]").dim(0) == (DimSpec{1, 4, 4}));
  CHECK_THROWS_AS(parse_shape("[*5/4]"), ShapeParseError);
  try {
    parse_shape("[5/2,*3/");
    CHECK(false);
  } catch (const ShapeParseError& e) {
    CHECK(e.position() == 8);
  }
  const auto s = parse_shape("[4,3/8,5/16]");
  CHECK(format_shape(sum_result_shape(s, 1)) == "[1,3/8,5/16]");
  CHECK(format_shape(sum_result_shape(s, 2)) == "[4,*/8,5/16]");
  CHECK(format_shape(sum_result_shape(s, 3)) == "[4,3/8,1?/16]");
  CHECK(format_shape(elementwise_result_shape(parse_shape("[18/8,4/16]"), parse_shape("[*/8,4/16]"),
                                              OpKind::add)) == "[18?/8,4/16]");
  CHECK(external_shape(parse_shape("[50/16,20/2,255/32]")) == (ExternalShape{4, 10, 8}));
}

// ---- test_backend.cpp --------------------------------------------------------
static void backend() {
  Session session(4, 3);
  const Tile t = session.make_tile(std::vector<double>{1, 2, 3, 4});
  CHECK(session.rotate(t, 1).slots() == (std::vector<double>{2, 3, 4, 1}));
  CHECK(session.rotate(t, -1).slots() == (std::vector<double>{4, 1, 2, 3}));
  CHECK(session.rotate(t, 5).slots() == (std::vector<double>{2, 3, 4, 1}));
  CHECK(session.cost_report().rotations == 3);
  CHECK(session.rotate(t, -8).slots() == t.slots());
  CHECK(session.cost_report().rotations == 3);

  Session s2(2, 3);
  const Tile a = s2.make_tile(std::vector<double>{1, 2});
  const Tile b = s2.make_tile(std::vector<double>{3, 4});
  const Tile p = s2.mul(a, b);
  CHECK(p.slots() == (std::vector<double>{3, 8}) && p.chain_index() == 2);
  const Tile sum = s2.add(a, p);
  CHECK(sum.slots() == (std::vector<double>{4, 10}) && sum.chain_index() == 2);
  const Tile m = s2.mask_mul(a, std::vector<double>{1, 0});
  CHECK(m.slots() == (std::vector<double>{1, 0}) && m.chain_index() == 2);
  const auto r = s2.cost_report();
  CHECK(r.additions == 1 && r.multiplications == 1 && r.mask_multiplications == 1);

  Session s3(2, 2);  // depth exhaustion and bootstrap
  const Tile ones = s3.constant_tile(1.0);
  Tile x = s3.make_tile(std::vector<double>{2, 3});
  x = s3.mul(x, ones);
  x = s3.mul(x, ones);
  CHECK(x.chain_index() == 0);
  CHECK_THROWS_AS(s3.mul(x, ones), DepthExhaustedError);
  const Tile restored = s3.bootstrap(x);
  CHECK(restored.chain_index() == 2 && s3.cost_report().bootstraps == 1);

  Session s4(4, 5);
  (void)s4.rotate(s4.constant_tile(1.0), 1);
  (void)s4.rotate(s4.constant_tile(1.0), 2);
  (void)s4.rotate(s4.constant_tile(1.0), 3);
  CHECK(s4.cost_report().power_of_two_rotations == 2);
  s4.reset_counters();
  CHECK(s4.cost_report().to_text() ==
        "additions=0\nmultiplications=0\nmask_multiplications=0\nrotations=0\nbootstraps=0\n");

  Session s5(16, 4);  // counters under concurrency (test_backend.cpp:186-203)
  std::vector<std::thread> pool;
  for (int w = 0; w < 8; ++w)
    pool.emplace_back([&] {
      const Tile c = s5.constant_tile(1.0);
      for (int i = 0; i < 2000; ++i) {
        (void)s5.add(c, c);
        (void)s5.rotate(c, 1);
      }
    });
  for (auto& th : pool) th.join();
  CHECK(s5.cost_report().additions == 16000 && s5.cost_report().rotations == 16000);
}

// ---- test_rotate_sum.cpp -----------------------------------------------------
static void rotate_sum() {
  std::mt19937_64 rng(41);
  for (std::int64_t s : {16, 64, 256}) {
    Session session(s, 2);
    std::uniform_int_distribution<int> d(-50, 50);
    std::vector<double> v(static_cast<std::size_t>(s));
    for (auto& x : v) x = d(rng);
    const Tile tile = session.make_tile(v);
    for (int it = 0; it < 12; ++it) {
      const std::int64_t n = std::uniform_int_distribution<std::int64_t>(1, s)(rng);
      std::vector<double> want(v.size(), 0.0);
      for (std::int64_t j = 0; j < s; ++j)
        for (std::int64_t i = j; i < j + n; ++i) want[j] += v[i % s];
      CHECK(sum_tile_flat(session, tile, n, SumVariant::left_to_right).slots() == want);
      CHECK(sum_tile_flat(session, tile, n, SumVariant::right_to_left).slots() == want);
      if ((n & (n - 1)) == 0) CHECK(sum_tile_flat(session, tile, n, SumVariant::power_of_two).slots() == want);
    }
  }
  CHECK(rotations_left_to_right(1190) == 14 && rotations_right_to_left(1190) == 14);
  Session session(8, 2);
  const Tile t = session.make_tile(std::vector<double>{1, 2, 3, 4, 10, 20, 30, 40});
  const std::vector<std::int64_t> ext{2, 4};
  CHECK(sum_tile_dim(session, t, ext, 1).slots() == (std::vector<double>{11, 22, 33, 44, 11, 22, 33, 44}));
  const Tile cols = sum_tile_dim(session, t, ext, 2);
  CHECK(cols.slots()[0] == 10 && cols.slots()[4] == 100);
  CHECK_THROWS_AS(sum_tile_dim(session, t, ext, 3), std::invalid_argument);
  CHECK_THROWS_AS(sum_tile_flat(session, t, 3, SumVariant::power_of_two), std::invalid_argument);
  Session r(8, 2);
  const Tile rt = r.make_tile(std::vector<double>{5, 0, 0, 0, 7, 0, 0, 0});
  CHECK(replicate_tile_dim(r, rt, ext, 2).slots() == (std::vector<double>{5, 5, 5, 5, 7, 7, 7, 7}));
  CHECK(r.cost_report().rotations == 2);
}

// ---- test_tile_tensor.cpp ----------------------------------------------------
static void tile_tensor() {
  {
    Session session(8, 4);  // :152-181
    const DenseTensor v({5}, {1, 2, 3, 4, 5});
    const TileTensor tv = pack(v, parse_shape("[5/2,*/4]"), session);
    CHECK(tv.tile_count() == 3);
    CHECK(tv.tile_at(0).slots() == (std::vector<double>{1, 1, 1, 1, 2, 2, 2, 2}));
    CHECK(tv.tile_at(2).slots() == (std::vector<double>{5, 5, 5, 5, 0, 0, 0, 0}));
    CHECK(pack(v, parse_shape("[5/2,*3/4]"), session).tile_at(0).slots() ==
          (std::vector<double>{1, 1, 1, 0, 2, 2, 2, 0}));
    CHECK_THROWS_AS(pack(v, parse_shape("[5/2,1?/4]"), session), ShapeError);
    CHECK_THROWS_AS(pack(v, parse_shape("[5/2]"), session), ShapeError);
  }
  {
    std::mt19937_64 rng(71);  // round trip (:183-198 / acceptance criterion 4)
    for (int it = 0; it < 60; ++it) {
      const std::int64_t slots = std::int64_t{1} << std::uniform_int_distribution<int>(3, 6)(rng);
      Session session(slots, 2);
      const TileTensorShape shape = random_pack_shape(rng, slots, std::uniform_int_distribution<int>(1, 4)(rng));
      const DenseTensor a = random_tensor(shape.tensor_extents(), rng);
      CHECK(unpack(pack(a, shape, session)) == a);
    }
  }
  {
    std::mt19937_64 rng(73);  // elementwise homomorphism (:218-264)
    int done = 0;
    while (done < 80) {
      const std::int64_t slots = std::int64_t{1} << std::uniform_int_distribution<int>(2, 5)(rng);
      Session session(slots, 8);
      const TileTensorShape sa = random_pack_shape(rng, slots, std::uniform_int_distribution<int>(1, 3)(rng));
      std::vector<DimSpec> pd;
      for (const auto& d : sa.dims()) {
        DimSpec p;
        p.t = d.t;
        switch (std::uniform_int_distribution<int>(0, 2)(rng)) {
          case 0: p.n = d.n; break;
          case 1: p.n = 1; p.d = p.t; break;
          default: p.n = std::uniform_int_distribution<std::int64_t>(1, 12)(rng);
        }
        pd.push_back(p);
      }
      const TileTensorShape sb(pd);
      const OpKind op = std::uniform_int_distribution<int>(0, 1)(rng) ? OpKind::add : OpKind::mul;
      try {
        (void)elementwise_result_shape(sa, sb, op);
      } catch (const ShapeError&) {
        continue;
      }
      const DenseTensor a = random_tensor(sa.tensor_extents(), rng);
      const DenseTensor b = random_tensor(sb.tensor_extents(), rng);
      TileTensor tc = tt_elementwise(pack(a, sa, session), pack(b, sb, session), op);
      fuzz_unknown_regions(tc, 5000 + static_cast<std::uint64_t>(done));
      CHECK(max_rel_diff(unpack(tc), dense_elementwise(a, b, op)) < 1e-9);
      ++done;
    }
  }
  {
    std::mt19937_64 rng(89);  // tt_sum homomorphism (:302-320)
    for (int it = 0; it < 60; ++it) {
      const std::int64_t slots = std::int64_t{1} << std::uniform_int_distribution<int>(2, 5)(rng);
      Session session(slots, 8);
      const int rank = std::uniform_int_distribution<int>(1, 3)(rng);
      const TileTensorShape shape = random_pack_shape(rng, slots, rank);
      const DenseTensor a = random_tensor(shape.tensor_extents(), rng);
      const TileTensor ta = pack(a, shape, session);
      for (int dim = 1; dim <= rank; ++dim) {
        TileTensor summed = tt_sum(ta, dim);
        CHECK(summed.shape() == sum_result_shape(shape, dim));
        fuzz_unknown_regions(summed, 7000 + static_cast<std::uint64_t>(it));
        CHECK(max_rel_diff(unpack(summed), dense_sum(a, dim)) < 1e-9);
      }
    }
  }
  {
    Session session(8, 4);  // '?' dimension boundary split (:322-333)
    std::mt19937_64 rng(97);
    const DenseTensor m = random_tensor({18, 1}, rng);
    const TileTensor tm = pack(m, parse_shape("[18/8,1]"), session);
    TileTensor forged(parse_shape("[18?/8,1]"), tm.tiles(), session);
    fuzz_unknown_regions(forged, 31337);
    const TileTensor summed = tt_sum(forged, 1);
    CHECK(format_shape(summed.shape()) == "[1?/8,1]");
    CHECK(max_rel_diff(unpack(summed), dense_sum(m, 1)) < 1e-9);
  }
  {
    Session session(8, 4);  // clean_unknowns / replicate_dim (:400-449)
    std::mt19937_64 rng(107);
    const DenseTensor m = random_tensor({5, 1}, rng);
    const TileTensor tm = pack(m, parse_shape("[5/2,1/4]"), session);
    TileTensor forged(parse_shape("[5/2,1?/4]"), tm.tiles(), session);
    fuzz_unknown_regions(forged, 400);
    const TileTensor cleaned = clean_unknowns(forged);
    CHECK(format_shape(cleaned.shape()) == "[5/2,1/4]");
    CHECK(unpack(cleaned) == m);
    for (std::size_t i = 0; i < cleaned.tile_count(); ++i)
      CHECK(cleaned.tile_at(i).slots() == tm.tile_at(i).slots());
    CHECK(cleaned.chain_index() == session.max_chain_index() - 1);
    const DenseTensor v({5}, {1, 2, 3, 4, 5});
    const TileTensor tv = pack(v, parse_shape("[5/2,1/4]"), session);
    const TileTensor rep = replicate_dim(tv, 2);
    CHECK(format_shape(rep.shape()) == "[5/2,*/4]");
    const TileTensor direct = pack(v, parse_shape("[5/2,*/4]"), session);
    for (std::size_t i = 0; i < rep.tile_count(); ++i)
      CHECK(rep.tile_at(i).slots() == direct.tile_at(i).slots());
    CHECK_THROWS_AS(replicate_dim(tv, 1), ShapeError);
  }
  {
    std::mt19937_64 rng(109);  // relaxed shapes (:451-476)
    Session session(16, 4);
    const TileTensorShape relaxed(std::vector<DimSpec>{DimSpec{7, 1, 3}, DimSpec{5, 1, 5}}, true);
    const DenseTensor a = random_tensor({7, 5}, rng);
    const TileTensor ta = pack(a, relaxed, session);
    CHECK(unpack(ta) == a);
    for (int dim = 1; dim <= 2; ++dim) {
      const TileTensor summed = tt_sum(ta, dim);
      CHECK(!summed.shape().dim(static_cast<std::size_t>(dim - 1)).fully_replicated());
      CHECK(max_rel_diff(unpack(summed), dense_sum(a, dim)) < 1e-9);
    }
  }
  {
    Session session(4, 1);  // depth exhaustion (:478-485)
    const TileTensor ta = pack(DenseTensor({2, 2}, {1, 2, 3, 4}), parse_shape("[2/2,2/2]"), session);
    const TileTensor sq = tt_mul(ta, ta);
    CHECK_THROWS_AS(tt_mul(sq, sq), DepthExhaustedError);
  }
  {
    Session session(8, 4);  // with_leading_unit_dim (:509-519)
    std::mt19937_64 rng(127);
    const DenseTensor a = random_tensor({3, 4}, rng);
    const TileTensor ta = pack(a, parse_shape("[3/2,4/4]"), session);
    const TileTensor lifted = with_leading_unit_dim(ta);
    CHECK(format_shape(lifted.shape()) == "[1,3/2,4/4]");
    CHECK(unpack(lifted) == a.reshape({1, 3, 4}));
  }
}

// ---- test_linalg.cpp / acceptance criterion 6 (subset) ------------------------
static void linalg() {
  std::mt19937_64 rng(6006);
  long runs = 0, fails = 0;
  for (std::int64_t s : {8, 16, 32}) {
    for (std::int64_t t1 = 1; t1 <= s; t1 *= 2)
      for (std::int64_t t2 = 1; t1 * t2 <= s; t2 *= 2) {
        const std::int64_t t3 = s / (t1 * t2);
        for (int it = 0; it < 6; ++it) {
          const std::int64_t a = std::uniform_int_distribution<std::int64_t>(1, 9)(rng);
          const std::int64_t b = std::uniform_int_distribution<std::int64_t>(1, 9)(rng);
          const std::int64_t c = std::uniform_int_distribution<std::int64_t>(1, 9)(rng);
          Session session(s, 16);
          const DenseTensor m1 = random_tensor({a, b}, rng, -1, 1);
          const DenseTensor m2 = random_tensor({b, c}, rng, -1, 1);
          const DenseTensor expect = dense_matmul(m1, m2);
          const TileTensor ta = pack(m1.reshape({a, b, 1}),
                                     TileTensorShape({DimSpec{a, 1, t1}, DimSpec{b, 1, t2}, DimSpec{1, t3, t3}}), session);
          const TileTensor tb = pack(m2.reshape({1, b, c}),
                                     TileTensorShape({DimSpec{1, t1, t1}, DimSpec{b, 1, t2}, DimSpec{c, 1, t3}}), session);
          ++runs;
          if (max_rel_diff(unpack(matmul_a(ta, tb)).reshape({a, c}), expect) >= 1e-9) ++fails;
          const TileTensor tat = pack(transpose2d(m1).reshape({b, a, 1}),
                                      TileTensorShape({DimSpec{b, 1, t1}, DimSpec{a, 1, t2}, DimSpec{1, t3, t3}}), session);
          const TileTensor tbb = pack(m2.reshape({b, 1, c}),
                                      TileTensorShape({DimSpec{b, 1, t1}, DimSpec{1, t2, t2}, DimSpec{c, 1, t3}}), session);
          ++runs;
          if (max_rel_diff(unpack(matmul_b(tat, tbb)).reshape({a, c}), expect) >= 1e-9) ++fails;
          if (it == 0) {  // fused FC stage == tt_mul(tt_add(matmul_a, bias)) bit for bit
            const TileTensor bias = pack(random_tensor({a, 1, c}, rng, -1, 1),
                                         TileTensorShape({DimSpec{a, 1, t1}, DimSpec{1, t2, t2}, DimSpec{c, 1, t3}}), session);
            session.reset_counters();
            TileTensor want = tt_add(tt_mul_sum(ta, tb, 2), bias);
            want = tt_mul(want, want);
            const CostReport wc = session.cost_report();
            session.reset_counters();
            const TileTensor got = tt_mul_sum_affine(ta, tb, 2, &bias, true);
            const CostReport gc = session.cost_report();
            bool same = format_shape(got.shape()) == format_shape(want.shape()) &&
                        got.chain_index() == want.chain_index() && gc.additions == wc.additions &&
                        gc.multiplications == wc.multiplications && gc.rotations == wc.rotations &&
                        got.tiles().size() == want.tiles().size();
            for (std::size_t i = 0; same && i < got.tiles().size(); ++i)
              same = std::memcmp(got.tiles()[i].slots().data(), want.tiles()[i].slots().data(),
                                 8 * got.tiles()[i].slots().size()) == 0;
            ++runs;
            if (!same) ++fails;
          }
        }
      }
  }
  CHECK(runs > 100 && fails == 0);
  // matmul_b output chains into matmul_a (test_linalg.cpp:157-178)
  Session session(8, 8);
  const DenseTensor x = random_tensor({4, 3}, rng), m1 = random_tensor({5, 4}, rng),
                    m2 = random_tensor({2, 5}, rng);
  const TileTensor tm1 = pack(transpose2d(m1).reshape({4, 5, 1}),
                              TileTensorShape({DimSpec{4, 1, 2}, DimSpec{5, 1, 2}, DimSpec{1, 2, 2}}), session);
  const TileTensor tx = pack(x.reshape({4, 1, 3}),
                             TileTensorShape({DimSpec{4, 1, 2}, DimSpec{1, 2, 2}, DimSpec{3, 1, 2}}), session);
  const TileTensor s1 = matmul_b(tm1, tx);
  const TileTensor tm2 = pack(m2.reshape({2, 5, 1}),
                              TileTensorShape({DimSpec{2, 1, 2}, DimSpec{5, 1, 2}, DimSpec{1, 2, 2}}), session);
  const TileTensor s2 = matmul_a(tm2, s1);
  CHECK(max_rel_diff(unpack(s2).reshape({2, 3}), dense_matmul(m2, dense_matmul(m1, x))) < 1e-9);
  CHECK_THROWS_AS(matvec_a(tm1, tx), ShapeError);  // rank-3 operands
  // dense oracle routes (dense.hpp:107-177)
  const DenseTensor p = random_tensor({4, 5}, rng), q = random_tensor({5, 3}, rng);
  CHECK(max_rel_diff(dense_matmul_via_broadcast(p, q), dense_matmul(p, q)) < 1e-12);
  const DenseTensor row = random_tensor({1, 5}, rng);
  const DenseTensor sum = dense_elementwise(p, row, OpKind::add);
  CHECK(sum.shape() == p.shape() && sum(2, 3) == p(2, 3) + row(0, 3));
  CHECK_THROWS_AS(dense_elementwise(p, q, OpKind::mul), ShapeError);
}

// chain of dense matrix-vector products (the pipeline's oracle)
static DenseTensor chain_oracle(const std::vector<DenseTensor>& ms, const DenseTensor& v) {
  DenseTensor x = v.reshape({static_cast<std::int64_t>(v.size()), 1});
  for (const auto& m : ms) x = dense_matmul(m, x);
  return x.reshape({static_cast<std::int64_t>(x.size())});
}

static DenseTensor identity_matrix(std::int64_t n) {
  std::vector<double> v(static_cast<std::size_t>(n * n), 0.0);
  for (std::int64_t i = 0; i < n; ++i) v[static_cast<std::size_t>(i * n + i)] = 1.0;
  return DenseTensor({n, n}, std::move(v));
}

// packing methods, the alternating pipeline and the tile-extent search
// (inc/linalg.hpp:77-294; behaviour as pinned by tests/test_linalg.cpp:181-326)
static void pipeline_suite() {
  std::mt19937_64 rng(9009);
  {  // every special-case packing runs through the same two-line body
    const DenseTensor m = random_tensor({5, 3}, rng, -1, 1);
    const DenseTensor v = random_tensor({3}, rng, -1, 1);
    const DenseTensor expect = chain_oracle({m}, v);
    for (const auto& method : {PackingMethod::row_order(), PackingMethod::column_order(),
                               PackingMethod::input_packing(), PackingMethod::general({4, 4})}) {
      Session session(16, 8);
      const bool inp = method.kind == PackingMethod::Kind::input_packing;
      const TileTensor tm = pack_for_method(m, inp ? OperandRole::lhs : OperandRole::matrix, method, session);
      const TileTensor tv = pack_for_method(v, inp ? OperandRole::rhs : OperandRole::vector, method, session);
      CHECK(max_rel_diff(unpack_vector(tt_sum(tt_mul(tm, tv), sum_dim_for(method))), expect) < 1e-9);
    }
    Session session(16, 8);
    const DenseTensor batch = random_tensor({3, 7}, rng, -1, 1);
    const TileTensor tw = pack_for_method(m, OperandRole::matrix, PackingMethod::batch_packing(), session);
    const TileTensor tb = pack_for_method(batch, OperandRole::vector, PackingMethod::batch_packing(), session);
    CHECK(format_shape(tw.shape()) == "[5,3,*/16]");
    CHECK(format_shape(tb.shape()) == "[3,7/16]");
    session.reset_counters();
    const TileTensor r = tt_sum(tt_mul(tw, with_leading_unit_dim(tb)), 2);
    CHECK(session.cost_report().rotations == 0);
    CHECK(max_rel_diff(unpack(r).reshape({5, 7}), dense_matmul(m, batch)) < 1e-9);
  }
  {  // input packing: smallest divisor of s that fits the contracted extent
    Session session(16, 8);
    const TileTensor tm = pack_for_method(random_tensor({4, 3}, rng, -1, 1), OperandRole::lhs,
                                          PackingMethod::input_packing(), session);
    CHECK(format_shape(tm.shape()) == "[3/4,4/4]");
    CHECK_THROWS_AS(pack_for_method(random_tensor({2, 17}, rng, -1, 1), OperandRole::lhs,
                                    PackingMethod::input_packing(), session),
                    ShapeError);
  }
  {  // general packing fills every slot
    Session session(1024, 2);
    const DenseTensor m = random_tensor({768, 768}, rng, -1, 1);
    const TileTensor g = pack_for_method(m, OperandRole::matrix, PackingMethod::general({4, 256}), session);
    CHECK(g.tile_count() == 576);
    CHECK(g.shape().used_slots() == g.shape().total_slots());
    CHECK(pack_for_method(m, OperandRole::matrix, PackingMethod::row_order(), session).tile_count() == 768);
  }
  {  // identities, one stage, three and four stages, two stages without masks
    Session s8(8, 8);
    const DenseTensor v3({3}, {1, 2, 3});
    const std::vector<DenseTensor> ids{identity_matrix(3), identity_matrix(3)};
    CHECK(max_rel_diff(unpack_vector(pipeline(ids, v3, {2, 4}, s8).out), v3) < 1e-12);
    const DenseTensor m = random_tensor({5, 6}, rng, -1, 1), v = random_tensor({6}, rng, -1, 1);
    const auto one = pipeline(std::vector<DenseTensor>{m}, v, {2, 4}, s8);
    CHECK(format_shape(one.out.shape()) == "[*/2,5/4]");
    CHECK(one.cost.mask_multiplications == 0);
    CHECK(max_rel_diff(unpack_vector(one.out), chain_oracle({m}, v)) < 1e-9);

    Session s32(32, 8);
    const std::vector<DenseTensor> three{random_tensor({5, 7}, rng, -1, 1), random_tensor({9, 5}, rng, -1, 1),
                                         random_tensor({7, 9}, rng, -1, 1)};
    const DenseTensor v7 = random_tensor({7}, rng, -1, 1);
    const auto r3 = pipeline(three, v7, {4, 8}, s32);
    CHECK(max_rel_diff(unpack_vector(r3.out), chain_oracle(three, v7)) < 1e-9);
    CHECK(r3.cost.mask_multiplications > 0);

    Session s16(16, 16);
    const std::vector<DenseTensor> two{random_tensor({6, 4}, rng, -1, 1), random_tensor({3, 6}, rng, -1, 1)};
    const DenseTensor v4 = random_tensor({4}, rng, -1, 1);
    const auto r2 = pipeline(two, v4, {4, 4}, s16);
    CHECK(r2.cost.mask_multiplications == 0);
    CHECK(max_rel_diff(unpack_vector(r2.out), chain_oracle(two, v4)) < 1e-9);
    const std::vector<DenseTensor> four{random_tensor({5, 4}, rng, -1, 1), random_tensor({7, 5}, rng, -1, 1),
                                        random_tensor({6, 7}, rng, -1, 1), random_tensor({3, 6}, rng, -1, 1)};
    const auto r4 = pipeline(four, v4, {4, 4}, s16);
    CHECK(max_rel_diff(unpack_vector(r4.out), chain_oracle(four, v4)) < 1e-9);
    CHECK(r4.cost.mask_multiplications == 2);  // one seam: [7/4,1?/4] -> two tiles masked
  }
  {  // validation and depth exhaustion naming the stage
    Session s8(8, 8);
    CHECK_THROWS_AS(pipeline(std::vector<DenseTensor>{random_tensor({3, 4}, rng, -1, 1)},
                             random_tensor({5}, rng, -1, 1), {2, 4}, s8),
                    ShapeError);
    CHECK_THROWS_AS(pipeline(std::vector<DenseTensor>{random_tensor({3, 4}, rng, -1, 1)},
                             random_tensor({4}, rng, -1, 1), {3, 4}, s8),
                    ShapeError);
    Session shallow(8, 2);
    const std::vector<DenseTensor> ms{random_tensor({4, 4}, rng, -1, 1), random_tensor({4, 4}, rng, -1, 1),
                                      random_tensor({4, 4}, rng, -1, 1)};
    bool named = false;
    try {
      (void)pipeline(ms, random_tensor({4}, rng, -1, 1), {2, 4}, shallow);
    } catch (const DepthExhaustedError& e) {
      named = std::string(e.what()).find("stage") != std::string::npos;
    }
    CHECK(named);
  }
  {  // the search scores every divisor pair, ordered by rotations
    const std::vector<DenseTensor> ms{random_tensor({4, 6}, rng, -1, 1), random_tensor({5, 4}, rng, -1, 1)};
    const auto choices = score_tile_factorizations(ms, random_tensor({6}, rng, -1, 1), 16, 8);
    CHECK(choices.size() == 5);
    for (std::size_t i = 1; i < choices.size(); ++i)
      CHECK(choices[i - 1].cost.rotations <= choices[i].cost.rotations);
  }
}

// inference kit (inc/nn.hpp; behaviour pinned by tests/test_nn.cpp:162-270)
static void nn_suite() {
  std::mt19937_64 rng(3131);
  std::istringstream spec(
      "input h=6 w=6\nconv filters=2 kh=3 kw=3 stride=2 pad=1\nact square\n"
      "fc in=18 out=4\nact square\nfc in=4 out=3\n");
  const NetworkSpec net = parse_network(spec, "", 44);
  CHECK(net.layers.size() == 5 && net.input_size() == 36);
  const std::int64_t s = 64;
  long runs = 0;
  for (std::int64_t t3 = 1; t3 <= s; t3 *= 2)
    for (std::int64_t t1 = 1; t1 * t3 <= s; t1 *= 2) {
      const DenseTensor batch = random_tensor({36, t3}, rng, -1, 1);
      Session session(s, 8);
      const auto res = cryptonets_infer(net, batch, {t1, s / (t1 * t3), t3}, session);
      CHECK(max_rel_diff(res.logits, nn_forward(net, batch)) < 1e-6);
      if (t1 == 1 && s / (t1 * t3) == 1) CHECK(res.cost.rotations == 0);
      ++runs;
    }
  CHECK(runs == 28);
  {  // lifted batch limit: n > t3 equals per-chunk runs
    const DenseTensor batch = random_tensor({36, 21}, rng, -1, 1);
    Session session(64, 8);
    CHECK_THROWS_AS(cryptonets_infer(net, batch, {2, 4, 8}, session), ShapeError);
    const auto all = cryptonets_infer(net, batch, {2, 4, 8}, session, true);
    CHECK(all.logits.extent(1) == 21);
    CHECK(max_rel_diff(all.logits, nn_forward(net, batch)) < 1e-6);
    const auto bp = cryptonets_infer(net, batch, {1, 1, 64}, session, true);
    CHECK(max_rel_diff(bp.logits, nn_forward(net, batch)) < 1e-6);
    const auto big = random_tensor({36, 150}, rng, -1, 1);
    const auto bp2 = cryptonets_infer(net, big, {1, 1, 64}, session, true);
    CHECK(bp2.logits.extent(1) == 150 && max_rel_diff(bp2.logits, nn_forward(net, big)) < 1e-6);
  }
  {  // layers uploaded once: CompiledBatchPacked == cryptonets_infer, bit for bit, every call
    const NetworkSpec cn = cryptonets_network(7);
    Session session(256, 8);
    CompiledBatchPacked comp(cn, session);
    for (std::int64_t n : {256, 77}) {
      const DenseTensor batch = random_tensor({784, n}, rng, 0, 1);
      session.reset_counters();
      const auto want = cryptonets_infer(cn, batch, {1, 1, 256}, session);
      const CostReport wc = session.cost_report();
      session.reset_counters();
      const auto got = comp.infer(batch);
      const CostReport gc = session.cost_report();
      bool same = got.logits.values().size() == want.logits.values().size();
      for (std::size_t i = 0; same && i < got.logits.values().size(); ++i)
        same = std::memcmp(&got.logits.values()[i], &want.logits.values()[i], 8) == 0;
      CHECK(same && gc.additions == wc.additions && gc.multiplications == wc.multiplications);
    }
    CHECK_THROWS_AS(comp.infer(random_tensor({783, 4}, rng, 0, 1)), ShapeError);
  }
  {  // tiled branch with weights packed once: CompiledTiled == cryptonets_infer, every call
    for (const auto& tile : {std::array<std::int64_t, 3>{2, 32, 1}, std::array<std::int64_t, 3>{4, 4, 4}}) {
      Session session(64, 8);
      CompiledTiled comp(net, tile, session);
      for (int rep = 0; rep < 3; ++rep) {
        const DenseTensor batch = random_tensor({36, tile[2]}, rng, -1, 1);
        session.reset_counters();
        const auto want = cryptonets_infer(net, batch, tile, session);
        const CostReport wc = session.cost_report();
        session.reset_counters();
        const auto got = comp.infer(batch);
        const CostReport gc = session.cost_report();
        bool same = got.logits.values().size() == want.logits.values().size();
        for (std::size_t i = 0; same && i < got.logits.values().size(); ++i)
          same = std::memcmp(&got.logits.values()[i], &want.logits.values()[i], 8) == 0;
        CHECK(same && gc.additions == wc.additions && gc.rotations == wc.rotations &&
              gc.multiplications == wc.multiplications);
      }
    }
  }
  {  // paper-scale counts for tile [32, 256, 1]
    const NetworkSpec cn = cryptonets_network(42);
    const DenseTensor batch = random_tensor({784, 1}, rng, -1, 1);
    Session session(8192, 8);
    const auto res = cryptonets_infer(cn, batch, {32, 256, 1}, session);
    CHECK(res.cost.multiplications == 32 && res.cost.rotations == 89 && res.cost.additions == 113);
    CHECK(max_rel_diff(res.logits, nn_forward(cn, batch)) < 1e-6);
  }
  {  // depth exhaustion names the layer, both branches
    Session shallow(64, 2);
    for (const auto& tile : {std::array<std::int64_t, 3>{2, 32, 1}, std::array<std::int64_t, 3>{1, 1, 64}}) {
      bool named = false;
      try {
        (void)cryptonets_infer(net, random_tensor({36, 1}, rng, -1, 1), tile, shallow);
      } catch (const DepthExhaustedError& e) {
        named = std::string(e.what()).find("layer") != std::string::npos;
      }
      CHECK(named);
    }
    Session session(64, 8);
    CHECK_THROWS_AS(cryptonets_infer(net, random_tensor({36, 9}, rng, -1, 1), {2, 4, 8}, session),
                    ShapeError);
  }
  {  // im2col, text tensors
    const DenseTensor x = random_tensor({4, 4}, rng, -1, 1);
    const DenseTensor m1 = im2col(x, 2, 2, 2, 0);
    CHECK(m1.shape() == (std::vector<std::int64_t>{4, 4}) && m1(3, 0) == x(2, 2));
    CHECK(im2col(DenseTensor::zeros({28, 28}), 5, 5, 2, 1).extent(0) == 169);
    CHECK_THROWS_AS(im2col(x, 6, 6, 1, 0), ShapeError);
    std::stringstream io;
    write_tensor(io, x);
    CHECK(read_tensor(io) == x);
  }
}

// A reference to tiles() kept across operator calls: every later edit through it
// is seen by the next operator, as with the reference's host-resident tiles.
static void held_tiles_suite() {
  Session session(4, 8);
  TileTensor t = pack(DenseTensor({2, 2}, {1, 2, 3, 4}), parse_shape("[2/2,2/2]"), session);
  auto& held = t.tiles();
  held[0].slots()[0] = 10.0;  // tile = {10, 2, 3, 4}
  CHECK(tt_sum(t, 2).tiles()[0].slots()[0] == 12.0);
  held[0].slots()[1] = 20.0;  // edited again after an operator read the tensor
  CHECK(tt_sum(t, 2).tiles()[0].slots()[0] == 30.0);
  CHECK(tt_add(t, t).tiles()[0].slots()[1] == 40.0);
  held[0].slots()[3] = -4.0;
  CHECK(tt_mul(t, t).tiles()[0].slots()[3] == 16.0);
}

// packed tile file (tools/tiletensor_main.cpp:76-128): text and bit-exact round trip
static void formats_suite() {
  Session session(4, 8);
  const TileTensor t = pack(DenseTensor({3}, {1, 2, 3}), parse_shape("[3/2,*/2]"), session);
  std::stringstream io;
  write_tiles(io, t);
  CHECK(io.str() == "shape: [3/2,*/2]\nslots: 4\ntile: 1 1 2 2\ntile: 3 3 0 0\n");
  const TileTensor back = read_tiles(io, session);
  CHECK(back.shape() == t.shape() && back.tiles()[1].slots()[1] == 3.0);
  std::mt19937_64 rng(4242);
  Session s16(16, 8);
  const TileTensor r = tt_sum(pack(random_tensor({5, 7}, rng), parse_shape("[5/4,7/4]"), s16), 2);
  std::stringstream io2;
  write_tiles(io2, r);
  const TileTensor r2 = read_tiles(io2, s16);
  CHECK(r2.shape() == r.shape());
  bool same = true;
  for (std::size_t i = 0; i < r.tile_count(); ++i)
    for (std::size_t h = 0; h < 16; ++h)
      same = same && std::memcmp(&r.tiles()[i].slots()[h], &r2.tiles()[i].slots()[h], 8) == 0;
  CHECK(same);
  std::istringstream bad("shape: [2/2,*/2]\nslots: 8\n");
  CHECK_THROWS_AS(read_tiles(bad, session), std::runtime_error);
}

int main() {
  const std::vector<std::pair<const char*, std::function<void()>>> suites = {
      {"shapes", shapes}, {"backend", backend}, {"rotate_sum", rotate_sum},
      {"tile_tensor", tile_tensor}, {"linalg", linalg}, {"pipeline", pipeline_suite}, {"nn", nn_suite}, {"held_tiles", held_tiles_suite}, {"formats", formats_suite}};
  for (const auto& [name, fn] : suites) {
    const int before = g_failed;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_failed;
      std::fprintf(stderr, "FAIL %s: uncaught %s\n", name, e.what());
    }
    std::printf("[%s] %s\n", g_failed == before ? "PASS" : "FAIL", name);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_failed);
  return g_failed;
}

// tt_shape.cpp -- tile-tensor shape notation and algebra (host side).
//
// Re-implements, for the B200 build, the grammar and rules of the reference's
// inc/shape.hpp (cited per function; paths relative to
// /root/reference/proj/include/tiletensor/).  Error texts and parse positions
// match the reference so callers see identical diagnostics.  The builder's
// `~` (interleaved) token is an extension the reference does not have.
#include <algorithm>
#include <cstring>

#include "tt_internal.hpp"

namespace ttb {

namespace {

void check_dim(const Dim& ds, size_t idx) {  // shape.hpp:57-66
  auto fail = [&](const std::string& what) {
    shape_error("dimension " + std::to_string(idx + 1) + ": " + what);
  };
  if (ds.n < 1 || ds.d < 1 || ds.t < 1) fail("extents must be positive");
  if (ds.d > 1 && ds.n > 1) fail("replication requires original extent 1");
  if (ds.d > ds.t)
    fail("replication count " + std::to_string(ds.d) + " exceeds tile extent " +
         std::to_string(ds.t));
  if (ds.interleaved && ds.d > 1) fail("interleaved tiling requires no replication");
}

}  // namespace

void check_shape(const Shape& s) {  // shape.hpp:74-78
  if (s.dims.empty()) shape_error("shape must have at least one dimension");
  if (s.dims.size() > TT_MAX_RANK)
    shape_error("rank " + std::to_string(s.dims.size()) + " exceeds the supported maximum " +
                std::to_string(TT_MAX_RANK));
  for (size_t i = 0; i < s.dims.size(); ++i) check_dim(s.dims[i], i);
}

Shape from_c(const tt_shape* c) {
  if (c == nullptr) invalid_argument("null shape");
  if (c->rank < 1 || c->rank > TT_MAX_RANK)
    shape_error(c->rank < 1 ? "shape must have at least one dimension"
                            : "rank exceeds the supported maximum");
  Shape s;
  s.relaxed = c->relaxed != 0;
  for (int i = 0; i < c->rank; ++i) {
    Dim d;
    d.n = c->dims[i].n;
    d.d = c->dims[i].d;
    d.t = c->dims[i].t;
    d.unknown = c->dims[i].unknown != 0;
    d.interleaved = c->dims[i].interleaved != 0;
    s.dims.push_back(d);
  }
  check_shape(s);
  return s;
}

void to_c(const Shape& s, tt_shape* out) {
  if (out == nullptr) return;  // result shape not wanted (the caller already knows it)
  std::memset(out, 0, sizeof(*out));
  out->rank = s.rank();
  out->relaxed = s.relaxed ? 1 : 0;
  for (int i = 0; i < s.rank(); ++i) {
    out->dims[i].n = s.dims[i].n;
    out->dims[i].d = s.dims[i].d;
    out->dims[i].t = s.dims[i].t;
    out->dims[i].unknown = s.dims[i].unknown ? 1 : 0;
    out->dims[i].interleaved = s.dims[i].interleaved ? 1 : 0;
  }
}

// ---- parser (shape.hpp:144-252) ---------------------------------------------

namespace {

class Parser {
 public:
  explicit Parser(std::string_view text) : text_(text) {}

  Shape run() {
    skip_ws();
    expect('[');
    Shape s;
    s.dims.push_back(parse_dim(0));
    while (peek() == ',') {
      ++pos_;
      s.dims.push_back(parse_dim(s.dims.size()));
    }
    expect(']');
    skip_ws();
    if (pos_ != text_.size()) parse_error("trailing characters after shape", pos_);
    check_shape(s);
    return s;
  }

 private:
  [[noreturn]] void parse_error(const std::string& msg, size_t pos) {
    throw Error(TT_ERR_SHAPE_PARSE, msg + " (at position " + std::to_string(pos) + ")",
                static_cast<int64_t>(pos));
  }

  Dim parse_dim(size_t index) {
    skip_ws();
    const size_t start = pos_;
    Dim ds;
    bool have_n = false, star = false, star_count = false;
    if (is_digit(peek())) {
      ds.n = parse_int();
      have_n = true;
    }
    skip_ws();
    if (peek() == '*') {
      ++pos_;
      star = true;
      skip_ws();
      if (is_digit(peek())) {
        ds.d = parse_int();
        star_count = true;
      }
    }
    // '?' (shape.hpp:187-190) and the builder's '~', in either order.
    for (int k = 0; k < 2; ++k) {
      skip_ws();
      if (peek() == '?' && !ds.unknown) {
        ++pos_;
        ds.unknown = true;
      } else if (peek() == '~' && !ds.interleaved) {
        ++pos_;
        ds.interleaved = true;
      }
    }
    skip_ws();
    if (peek() == '/') {
      ++pos_;
      skip_ws();
      if (!is_digit(peek())) parse_error("expected tile extent after '/'", pos_);
      ds.t = parse_int();
    }
    skip_ws();
    if (!have_n && !star) parse_error("expected dimension extent or '*'", start);
    if (star && !have_n) ds.n = 1;
    if (star && !star_count) ds.d = ds.t;
    if (ds.n < 1 || ds.d < 1 || ds.t < 1) parse_error("extents must be positive", start);
    try {
      check_dim(ds, index);
    } catch (const Error& e) {
      parse_error(e.what(), start);
    }
    return ds;
  }

  int64_t parse_int() {
    int64_t v = 0;
    const size_t start = pos_;
    while (is_digit(peek())) {
      v = v * 10 + (text_[pos_] - '0');
      if (v > (int64_t{1} << 48)) parse_error("integer too large", start);
      ++pos_;
    }
    return v;
  }

  static bool is_digit(char c) { return c >= '0' && c <= '9'; }
  char peek() const { return pos_ < text_.size() ? text_[pos_] : '\0'; }
  void expect(char c) {
    skip_ws();
    if (peek() != c) parse_error(std::string("expected '") + c + "'", pos_);
    ++pos_;
  }
  void skip_ws() {
    while (pos_ < text_.size() && (text_[pos_] == ' ' || text_[pos_] == '\t')) ++pos_;
  }

  std::string_view text_;
  size_t pos_ = 0;
};

}  // namespace

Shape parse_shape(std::string_view text) { return Parser(text).run(); }

// Canonical form shape.hpp:256-278 ('~' printed before '?').
std::string format_shape(const Shape& s) {
  std::string out = "[";
  bool first = true;
  for (const auto& ds : s.dims) {
    if (!first) out += ',';
    first = false;
    if (ds.n > 1) {
      out += std::to_string(ds.n);
    } else if (ds.d > 1) {
      out += '*';
      if (ds.d < ds.t) out += std::to_string(ds.d);
    } else {
      out += '1';
    }
    if (ds.interleaved) out += '~';
    if (ds.unknown) out += '?';
    if (ds.t > 1) {
      out += '/';
      out += std::to_string(ds.t);
    }
  }
  out += ']';
  return out;
}

// ---- elementwise and summation rules (shape.hpp:293-377) ---------------------

Shape elementwise_result_shape(const Shape& a, const Shape& b, int op) {
  if (a.rank() != b.rank())
    shape_error("rank mismatch: " + format_shape(a) + " vs " + format_shape(b));
  Shape out;
  out.relaxed = a.relaxed || b.relaxed;
  for (int i = 0; i < a.rank(); ++i) {
    const Dim& da = a.dims[i];
    const Dim& db = b.dims[i];
    if (da.t != db.t)
      shape_error("dimension " + std::to_string(i + 1) + ": tile extent mismatch (" +
                  std::to_string(da.t) + " vs " + std::to_string(db.t) + ")");
    const bool compatible = da.n == db.n || (da.n == 1 && da.fully_replicated()) ||
                            (db.n == 1 && db.fully_replicated());
    if (!compatible)
      shape_error("dimension " + std::to_string(i + 1) + ": incompatible extents " +
                  std::to_string(da.n) + " and " + std::to_string(db.n) +
                  " (neither side fully replicated)");
    // `~` extension: both sides must agree unless one side broadcasts.
    if (da.interleaved != db.interleaved && !da.fully_replicated() && !db.fully_replicated())
      shape_error("dimension " + std::to_string(i + 1) +
                  ": interleaved and regular tilings cannot be combined");
    Dim r;
    r.t = da.t;
    r.n = std::max(da.n, db.n);
    r.d = std::min(da.d, db.d);
    r.interleaved = (da.interleaved || db.interleaved) && r.d == 1;
    bool unk = da.unknown || db.unknown || da.used() != db.used();
    if (op == TT_OP_MUL && unk) {
      const int64_t used_r = r.used();
      const int64_t er = ceil_div(used_r, r.t);
      auto covers = [&](const Dim& o) {
        if (o.unknown) return false;
        const int64_t eo = ceil_div(o.used(), o.t);
        if (eo < er) return o.used() <= used_r - (er - 1) * r.t;
        return o.used() <= used_r;
      };
      if (covers(da) || covers(db)) unk = false;
    }
    r.unknown = unk;
    out.dims.push_back(r);
  }
  check_shape(out);
  return out;
}

namespace {
bool is_lowest_nontrivial(const Shape& s, int i) {  // shape.hpp:341-346
  for (int j = 0; j < i; ++j)
    if (s.dims[j].t > 1) return false;
  return s.dims[i].t > 1;
}
}  // namespace

Shape sum_result_shape(const Shape& s, int dim) {
  if (dim < 1 || dim > s.rank())
    shape_error("sum dimension " + std::to_string(dim) + " out of range for " + format_shape(s));
  const int i = dim - 1;
  const Dim& ds = s.dims[i];
  Dim r;
  r.t = ds.t;
  if (ds.unknown) {
    r.unknown = true;
  } else if (ds.n == 1 && ds.d > 1) {
    r = ds;
  } else if (ds.t == 1) {
    r = Dim{};
  } else if (is_lowest_nontrivial(s, i) && !s.relaxed) {
    r.d = ds.t;
  } else {
    r.unknown = true;
  }
  Shape out = s;
  out.dims[i] = r;
  check_shape(out);
  return out;
}

std::vector<int64_t> tile_strides(const Shape& s) {
  std::vector<int64_t> st(s.dims.size());
  int64_t p = 1;
  for (int i = s.rank() - 1; i >= 0; --i) {
    st[i] = p;
    p *= s.dims[i].t;
  }
  return st;
}

std::vector<int64_t> row_major_strides(const std::vector<int64_t>& e) {
  std::vector<int64_t> st(e.size());
  int64_t p = 1;
  for (int i = static_cast<int>(e.size()) - 1; i >= 0; --i) {
    st[i] = p;
    p *= e[i];
  }
  return st;
}

}  // namespace ttb

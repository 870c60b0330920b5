// tt_schedule.cpp -- compiles the reference's reduction schedules into group
// programs (see GOp in tt_internal.hpp) and counts their primitives.
//
// The compiler walks exactly the control flow of
//   sum_tile_strided  rotate_sum.hpp:44-90  (power_of_two / left_to_right / right_to_left)
//   replicate_tile_dim rotate_sum.hpp:128-152
//   tt_sum            tile_tensor.hpp:286-347 (fold, then in-tile schedule; '?' boundary split)
// emitting one instruction per Session::add (+ its rotate), so the device
// program performs the same additions in the same association and the cost
// counters are the reference's to the unit.
#include <bit>

#include "tt_internal.hpp"

namespace ttb {

namespace {

bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
int num_bits(int64_t n) { return 64 - std::countl_zero(static_cast<uint64_t>(n)); }

struct Builder {
  int64_t s;
  Program prog;

  int8_t new_buf() { return static_cast<int8_t>(prog.nbuf++); }

  void count_rot(int64_t r) {
    prog.per_group.rotations += 1;
    if ((r & (r - 1)) == 0) prog.per_group.power_of_two_rotations += 1;
  }

  // dst = a + rotate(b, offset)  (Session::add(a, Session::rotate(b, off))).
  void rotadd(int8_t dst, int8_t a, int8_t b, int64_t offset) {
    const int64_t r = ((offset % s) + s) % s;  // backend.hpp:155
    if (r != 0) count_rot(r);                  // r == 0 is free (backend.hpp:156)
    prog.per_group.additions += 1;
    GOp op{};
    op.kind = GOP_ROTADD;
    op.dst = dst;
    op.a = a;
    op.b = b;
    op.inplace = (dst == a || dst == b) ? 1 : 0;
    op.x = r;
    prog.ops.push_back(op);
  }

  void copy(int8_t dst, int8_t a) {
    GOp op{};
    op.kind = GOP_COPY;
    op.dst = dst;
    op.a = a;
    op.b = a;
    prog.ops.push_back(op);
  }

  void fold(int8_t dst, int64_t first, int64_t count) {
    prog.per_group.additions += static_cast<uint64_t>(count - 1);  // tile_tensor.hpp:324
    GOp op{};
    op.kind = GOP_FOLD;
    op.dst = dst;
    op.x = first;
    op.y = count;
    prog.ops.push_back(op);
  }

  // sum_tile_strided on buffer `in`; returns the buffer holding the result.
  // `tile` (the schedule's input) is never written except by pow2, which does
  // not read it again.
  int8_t strided(int8_t in, int64_t n, int64_t stride, int variant) {
    if (n < 1 || n > s) invalid_argument("sum length must be in [1, slot count]");
    if (n == 1) return in;
    if (variant < 0) variant = is_pow2(n) ? TT_VARIANT_POWER_OF_TWO : TT_VARIANT_RIGHT_TO_LEFT;
    switch (variant) {
      case TT_VARIANT_POWER_OF_TWO: {
        if (!is_pow2(n)) invalid_argument("power_of_two variant requires a power-of-two length");
        for (int64_t e = 1; e < n; e *= 2) rotadd(in, in, in, e * stride);
        return in;
      }
      case TT_VARIANT_LEFT_TO_RIGHT: {
        const int8_t sb = new_buf();
        bool first = true;  // s == tile until the first write
        int64_t e = 1;
        for (int j = num_bits(n) - 2; j >= 0; --j) {
          const int8_t cur = first ? in : sb;
          rotadd(sb, cur, cur, e * stride);
          first = false;
          e *= 2;
          if ((n >> j) & 1) {
            rotadd(sb, in, sb, stride);
            e += 1;
          }
        }
        return first ? in : sb;
      }
      case TT_VARIANT_RIGHT_TO_LEFT: {
        const int8_t x = in;  // x starts as the tile; the tile is not re-read
        int8_t y = -2;        // unset
        int64_t e = 1, m = n;
        while (true) {
          if (m % 2 == 1) {
            if (y == -2) {
              // y = x (a value copy, no primitive); when nothing follows, the
              // result IS x: no copy, so the schedule stays one in-place chain
              if ((m - 1) / 2 == 0) return x;
              y = new_buf();
              copy(y, x);
            } else {
              rotadd(y, x, y, e * stride);
            }
            m = (m - 1) / 2;
          } else {
            m = m / 2;
          }
          if (m == 0) return y;
          rotadd(x, x, x, e * stride);
          e *= 2;
        }
      }
      default:
        invalid_argument("unknown sum variant " + std::to_string(variant));
    }
  }

  // replicate_tile_dim: reverse right-to-left with negative shifts.
  int8_t replicate(int8_t in, int64_t t, int64_t stride) {
    if (t == 1) return in;
    const int8_t x = in;
    int8_t y = -2;
    int64_t e = 1, m = t;
    while (true) {
      if (m % 2 == 1) {
        if (y == -2) {
          if ((m - 1) / 2 == 0) return x;  // as in strided(): the result is x itself
          y = new_buf();
          copy(y, x);
        } else {
          rotadd(y, x, y, -e * stride);
        }
        m = (m - 1) / 2;
      } else {
        m = m / 2;
      }
      if (m == 0) return y;
      rotadd(x, x, x, -e * stride);
      e *= 2;
    }
  }

  // Route the value held in `result` into the group's output tile: retarget
  // the last instruction that wrote it, or append a copy.
  void finish(int8_t result) {
    if (!prog.ops.empty() && prog.ops.back().dst == result) {
      GOp& last = prog.ops.back();
      last.dst = BUF_OUT;
      last.inplace = 0;
    } else {
      copy(BUF_OUT, result);
    }
    // simple_pow2: FOLD into B0, then only in-place ROTADDs on B0, last one into OUT.
    bool simple = prog.ops.size() >= 1 && prog.ops[0].kind == GOP_FOLD && prog.nbuf <= 1;
    for (size_t i = 1; i < prog.ops.size() && simple; ++i) {
      const GOp& op = prog.ops[i];
      simple = op.kind == GOP_ROTADD && op.a == 0 && op.b == 0 &&
               (op.dst == 0 || (op.dst == BUF_OUT && i + 1 == prog.ops.size()));
    }
    prog.simple_pow2 = simple;
    if (prog.ops.size() > static_cast<size_t>(kMaxOps))
      invalid_argument("reduction schedule too long for one group program");
  }
};

}  // namespace

Program build_sum_program(int64_t ei, int64_t t, int64_t stride, int64_t s, int64_t used,
                          bool unknown, int variant) {
  Builder b{s, {}};
  const bool boundary_split = unknown && used % t != 0;  // tile_tensor.hpp:302
  const int64_t known_tail = used - (ei - 1) * t;        // :303
  if (!boundary_split) {
    const int8_t acc = b.new_buf();
    b.fold(acc, 0, ei);
    int8_t r = acc;
    if (t > 1) r = b.strided(acc, t, stride, variant);
    b.finish(r);
  } else {
    const int8_t tail = b.new_buf();
    b.fold(tail, ei - 1, 1);
    int8_t rt = tail;
    if (known_tail > 1) rt = b.strided(tail, known_tail, stride, variant);
    if (ei > 1) {
      const int8_t head = b.new_buf();
      b.fold(head, 0, ei - 1);
      int8_t rh = head;
      if (t > 1) rh = b.strided(head, t, stride, variant);
      b.rotadd(BUF_OUT, rh, rt, 0);  // session.add(head, tail) :339
      b.prog.simple_pow2 = false;
    } else {
      b.finish(rt);
    }
  }
  return b.prog;
}

Program build_strided_program(int64_t n, int64_t stride, int64_t s, int variant) {
  Builder b{s, {}};
  const int8_t in = b.new_buf();
  b.fold(in, 0, 1);
  b.finish(b.strided(in, n, stride, variant));
  return b.prog;
}

Program build_replicate_program(int64_t t, int64_t stride, int64_t s) {
  Builder b{s, {}};
  const int8_t in = b.new_buf();
  b.fold(in, 0, 1);
  b.finish(b.replicate(in, t, stride));
  return b.prog;
}

int64_t rotations_left_to_right(int64_t n) {
  return (num_bits(n) - 1) + (std::popcount(static_cast<uint64_t>(n)) - 1);
}
int64_t rotations_right_to_left(int64_t n) {
  return (num_bits(n) - 1) + std::popcount(static_cast<uint64_t>(n)) - 1;
}

}  // namespace ttb

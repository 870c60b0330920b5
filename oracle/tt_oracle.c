/*
 * tt_oracle.c -- CPU restatement of the reference tile-tensor hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline -- never as the product path.
 *
 * It restates, in plain C99 and scalar loops, the algorithm of the reference
 * headers under /root/reference/proj/include/tiletensor/ (cited per function
 * as file:line).  Floating-point work follows the reference's exact operation
 * order (left folds, the rotate-and-sum schedules) and is compiled with
 * -ffp-contract=off, so results are bit-identical to the reference, which the
 * not-gpu tests check against oracle/_ref (the reference itself, compiled
 * here) and against the golden vectors of the reference's own tests.
 *
 * The `~` (interleaved) dimension is NOT in the reference; its restatement
 * here is the builder's own definition and is parity-unpinned.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/tiletensor_b200.h"

#define OR_OK 0
#define OR_SHAPE 1
#define OR_INVALID 4
#define OR_DEPTH 3

/* ---- shape helpers (shape.hpp:37-138) ------------------------------------ */

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
static int64_t used_of(const tt_dim* d) { return d->n * d->d; }
static int fully_replicated(const tt_dim* d) { return d->n == 1 && d->d == d->t; }

int64_t or_tile_slots(const tt_shape* s) {
  int64_t p = 1;
  for (int i = 0; i < s->rank; ++i) p *= s->dims[i].t;
  return p;
}

void or_external(const tt_shape* s, int64_t* ext) {
  for (int i = 0; i < s->rank; ++i) ext[i] = ceil_div(used_of(&s->dims[i]), s->dims[i].t);
}

int64_t or_tile_count(const tt_shape* s) {
  int64_t p = 1;
  for (int i = 0; i < s->rank; ++i) p *= ceil_div(used_of(&s->dims[i]), s->dims[i].t);
  return p;
}

static int has_unknown(const tt_shape* s) {
  for (int i = 0; i < s->rank; ++i)
    if (s->dims[i].unknown) return 1;
  return 0;
}

/* tile_strides tile_tensor.hpp:31-39 */
static void tile_strides(const tt_shape* s, int64_t* st) {
  int64_t p = 1;
  for (int i = s->rank - 1; i >= 0; --i) {
    st[i] = p;
    p *= s->dims[i].t;
  }
}

/* row_major_strides tile_tensor.hpp:41-49 */
static void row_major(const int64_t* ext, int rank, int64_t* st) {
  int64_t p = 1;
  for (int i = rank - 1; i >= 0; --i) {
    st[i] = p;
    p *= ext[i];
  }
}

/* Logical index along dim i of slot coordinate m in external tile l (Eq. 1,
 * tile_tensor.hpp:108); the interleaved variant is the builder's `~`. */
static int64_t logical_j(const tt_dim* d, int64_t e, int64_t l, int64_t m) {
  return d->interleaved ? m * e + l : l * d->t + m;
}

/* ---- shape algebra (shape.hpp:293-377) ----------------------------------- */

int or_elementwise_result_shape(const tt_shape* a, const tt_shape* b, int op, tt_shape* out) {
  if (a->rank != b->rank) return OR_SHAPE;
  memset(out, 0, sizeof(*out));
  out->rank = a->rank;
  out->relaxed = a->relaxed || b->relaxed;
  for (int i = 0; i < a->rank; ++i) {
    const tt_dim* da = &a->dims[i];
    const tt_dim* db = &b->dims[i];
    if (da->t != db->t) return OR_SHAPE;
    /* builder's `~` rule: an interleaved dim combines
     * with an interleaved one or with a fully replicated (broadcast) one */
    if (da->interleaved != db->interleaved && !fully_replicated(da) && !fully_replicated(db))
      return OR_SHAPE;
    const int compatible = da->n == db->n || (da->n == 1 && fully_replicated(da)) ||
                           (db->n == 1 && fully_replicated(db));
    if (!compatible) return OR_SHAPE;
    tt_dim r;
    memset(&r, 0, sizeof(r));
    r.t = da->t;
    r.n = da->n > db->n ? da->n : db->n;
    r.d = da->d < db->d ? da->d : db->d;
    r.interleaved = (da->interleaved || db->interleaved) && r.d == 1;
    int unk = da->unknown || db->unknown || used_of(da) != used_of(db);
    if (op == TT_OP_MUL && unk) {
      const int64_t used_r = r.n * r.d;
      const int64_t er = ceil_div(used_r, r.t);
      for (int side = 0; side < 2 && unk; ++side) {
        const tt_dim* o = side == 0 ? da : db;
        if (o->unknown) continue;
        const int64_t eo = ceil_div(used_of(o), o->t);
        int covers;
        if (eo < er)
          covers = used_of(o) <= used_r - (er - 1) * r.t;
        else
          covers = used_of(o) <= used_r;
        if (covers) unk = 0;
      }
    }
    r.unknown = unk;
    out->dims[i] = r;
  }
  return OR_OK;
}

static int is_lowest_nontrivial(const tt_shape* s, int i) {
  for (int j = 0; j < i; ++j)
    if (s->dims[j].t > 1) return 0;
  return s->dims[i].t > 1;
}

int or_sum_result_shape(const tt_shape* s, int dim, tt_shape* out) {
  if (dim < 1 || dim > s->rank) return OR_SHAPE;
  *out = *s;
  const int i = dim - 1;
  const tt_dim* ds = &s->dims[i];
  tt_dim r;
  memset(&r, 0, sizeof(r));
  r.n = 1;
  r.d = 1;
  r.t = ds->t;
  if (ds->unknown) {
    r.unknown = 1;
  } else if (ds->n == 1 && ds->d > 1) {
    r = *ds;
  } else if (ds->t == 1) {
    r.t = 1;
  } else if (is_lowest_nontrivial(s, i) && !s->relaxed) {
    r.d = ds->t;
  } else {
    r.unknown = 1;
  }
  out->dims[i] = r;
  return OR_OK;
}

/* ---- counters (backend.hpp:198-203) --------------------------------------- */

static void count_rot(tt_cost* c, int64_t r) {
  if (!c) return;
  c->rotations += 1;
  if ((r & (r - 1)) == 0) c->power_of_two_rotations += 1;
}

/* ---- Session primitives on single tiles (backend.hpp:117-163) ------------ */

static void tile_add(const double* a, const double* b, double* out, int64_t s, tt_cost* c) {
  for (int64_t i = 0; i < s; ++i) out[i] = a[i] + b[i];
  if (c) c->additions += 1;
}

/* rotate backend.hpp:152-163: out[j] = in[(j + r) % s], r == 0 is free. */
static void tile_rotate(const double* in, int64_t off, double* out, int64_t s, tt_cost* c) {
  int64_t r = ((off % s) + s) % s;
  if (r == 0) {
    memcpy(out, in, (size_t)s * sizeof(double));
    return;
  }
  for (int64_t j = 0; j < s; ++j) out[j] = in[(j + r) % s];
  count_rot(c, r);
}

void or_rotate(const double* in, int64_t off, double* out, int64_t s, tt_cost* c) {
  tile_rotate(in, off, out, s, c);
}

static int is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
static int num_bits(int64_t n) {
  int b = 0;
  while (n) {
    ++b;
    n >>= 1;
  }
  return b;
}

/* sum_tile_strided rotate_sum.hpp:44-90.  `variant` < 0 means auto
 * (rotate_sum.hpp:99-101).  out may alias in. */
int or_sum_tile_strided(const double* in, int64_t s, int64_t n, int64_t stride, int variant,
                        double* out, tt_cost* c) {
  if (n < 1 || n > s) return OR_INVALID;
  if (variant < 0) variant = is_pow2(n) ? TT_VARIANT_POWER_OF_TWO : TT_VARIANT_RIGHT_TO_LEFT;
  const size_t bytes = (size_t)s * sizeof(double);
  if (n == 1) {
    memmove(out, in, bytes);
    return OR_OK;
  }
  double* x = (double*)malloc(bytes);
  double* y = (double*)malloc(bytes);
  double* rot = (double*)malloc(bytes);
  double* tile = (double*)malloc(bytes);
  memcpy(tile, in, bytes);
  int rc = OR_OK;
  if (variant == TT_VARIANT_POWER_OF_TWO) {
    if (!is_pow2(n)) {
      rc = OR_INVALID;
    } else {
      memcpy(x, tile, bytes);
      for (int64_t e = 1; e < n; e *= 2) {
        tile_rotate(x, e * stride, rot, s, c);
        tile_add(x, rot, x, s, c);
      }
      memcpy(out, x, bytes);
    }
  } else if (variant == TT_VARIANT_LEFT_TO_RIGHT) {
    memcpy(x, tile, bytes);
    int64_t e = 1;
    for (int j = num_bits(n) - 2; j >= 0; --j) {
      tile_rotate(x, e * stride, rot, s, c);
      tile_add(x, rot, x, s, c);
      e *= 2;
      if ((n >> j) & 1) {
        tile_rotate(x, stride, rot, s, c);
        tile_add(tile, rot, x, s, c);
        e += 1;
      }
    }
    memcpy(out, x, bytes);
  } else { /* right_to_left */
    memcpy(x, tile, bytes);
    int have_y = 0;
    int64_t e = 1, m = n;
    for (;;) {
      if (m % 2 == 1) {
        if (have_y) {
          tile_rotate(y, e * stride, rot, s, c);
          tile_add(x, rot, y, s, c);
        } else {
          memcpy(y, x, bytes);
          have_y = 1;
        }
        m = (m - 1) / 2;
      } else {
        m = m / 2;
      }
      if (m == 0) break;
      tile_rotate(x, e * stride, rot, s, c);
      tile_add(x, rot, x, s, c);
      e *= 2;
    }
    memcpy(out, y, bytes);
  }
  free(x);
  free(y);
  free(rot);
  free(tile);
  return rc;
}

/* replicate_tile_dim rotate_sum.hpp:128-152 (reverse rtl, negative shifts). */
int or_replicate_tile_dim(const double* in, int64_t s, const int64_t* tile_extents, int rank,
                          int dim, double* out, tt_cost* c) {
  if (dim < 1 || dim > rank) return OR_INVALID;
  int64_t stride = 1;
  for (int x = dim; x < rank; ++x) stride *= tile_extents[x];
  const int64_t t = tile_extents[dim - 1];
  const size_t bytes = (size_t)s * sizeof(double);
  if (t == 1) {
    memmove(out, in, bytes);
    return OR_OK;
  }
  double* x = (double*)malloc(bytes);
  double* y = (double*)malloc(bytes);
  double* rot = (double*)malloc(bytes);
  memcpy(x, in, bytes);
  int have_y = 0;
  int64_t e = 1, m = t;
  for (;;) {
    if (m % 2 == 1) {
      if (have_y) {
        tile_rotate(y, -e * stride, rot, s, c);
        tile_add(x, rot, y, s, c);
      } else {
        memcpy(y, x, bytes);
        have_y = 1;
      }
      m = (m - 1) / 2;
    } else {
      m = m / 2;
    }
    if (m == 0) break;
    tile_rotate(x, -e * stride, rot, s, c);
    tile_add(x, rot, x, s, c);
    e *= 2;
  }
  memcpy(out, y, bytes);
  free(x);
  free(y);
  free(rot);
  return OR_OK;
}

/* ---- pack / unpack (tile_tensor.hpp:167-242) ------------------------------ */

/* pack tile_tensor.hpp:167-220.  dense: prod(n_i) values row-major. */
int or_pack(const double* dense, const tt_shape* shape, int64_t s, double* tiles) {
  if (has_unknown(shape)) return OR_SHAPE;
  const int64_t ts = or_tile_slots(shape);
  if (!shape->relaxed && ts != s) return OR_SHAPE;
  if (shape->relaxed && ts > s) return OR_SHAPE;
  const int rank = shape->rank;
  int64_t ext[TT_MAX_RANK], es[TT_MAX_RANK], tst[TT_MAX_RANK], dst[TT_MAX_RANK];
  or_external(shape, ext);
  row_major(ext, rank, es);
  tile_strides(shape, tst);
  int64_t nn[TT_MAX_RANK];
  for (int i = 0; i < rank; ++i) nn[i] = shape->dims[i].n;
  row_major(nn, rank, dst);
  const int64_t n_tiles = or_tile_count(shape);
  for (int64_t flat = 0; flat < n_tiles; ++flat) {
    double* slots = tiles + flat * s;
    for (int64_t h = 0; h < s; ++h) slots[h] = 0.0;
    for (int64_t h = 0; h < ts; ++h) {
      int used = 1;
      int64_t src = 0;
      for (int i = 0; i < rank; ++i) {
        const tt_dim* ds = &shape->dims[i];
        const int64_t l = (flat / es[i]) % ext[i];
        const int64_t j = logical_j(ds, ext[i], l, (h / tst[i]) % ds->t);
        if (j >= used_of(ds)) {
          used = 0;
          break;
        }
        src += (j % ds->n) * dst[i];
      }
      if (used) slots[h] = dense[src];
    }
  }
  return OR_OK;
}

/* unpack tile_tensor.hpp:222-242: every dense element reads replica 0. */
int or_unpack(const tt_shape* shape, int64_t s, const double* tiles, double* dense) {
  const int rank = shape->rank;
  int64_t ext[TT_MAX_RANK], es[TT_MAX_RANK], tst[TT_MAX_RANK];
  or_external(shape, ext);
  row_major(ext, rank, es);
  tile_strides(shape, tst);
  int64_t total = 1;
  for (int i = 0; i < rank; ++i) total *= shape->dims[i].n;
  int64_t j[TT_MAX_RANK];
  for (int i = 0; i < rank; ++i) j[i] = 0;
  for (int64_t f = 0; f < total; ++f) {
    int64_t tile = 0, h = 0;
    for (int i = 0; i < rank; ++i) {
      const tt_dim* ds = &shape->dims[i];
      int64_t l, m;
      if (ds->interleaved) {
        l = j[i] % ext[i];
        m = j[i] / ext[i];
      } else {
        l = j[i] / ds->t;
        m = j[i] % ds->t;
      }
      tile += l * es[i];
      h += m * tst[i];
    }
    dense[f] = tiles[tile * s + h];
    for (int i = rank - 1; i >= 0; --i) {
      if (++j[i] < shape->dims[i].n) break;
      j[i] = 0;
    }
  }
  return OR_OK;
}

/* ---- operators ------------------------------------------------------------ */

/* tt_elementwise tile_tensor.hpp:244-272 (external broadcast l % e). */
int or_elementwise(int op, const tt_shape* sa, const double* ta, const tt_shape* sb,
                   const double* tb, int64_t s, tt_shape* so, double* out, tt_cost* c) {
  int rc = or_elementwise_result_shape(sa, sb, op, so);
  if (rc) return rc;
  const int rank = so->rank;
  int64_t ext[TT_MAX_RANK], es[TT_MAX_RANK], ea[TT_MAX_RANK], eas[TT_MAX_RANK],
      eb[TT_MAX_RANK], ebs[TT_MAX_RANK];
  or_external(so, ext);
  row_major(ext, rank, es);
  or_external(sa, ea);
  row_major(ea, rank, eas);
  or_external(sb, eb);
  row_major(eb, rank, ebs);
  const int64_t n = or_tile_count(so);
  for (int64_t flat = 0; flat < n; ++flat) {
    int64_t fa = 0, fb = 0;
    for (int i = 0; i < rank; ++i) {
      const int64_t l = (flat / es[i]) % ext[i];
      fa += (l % ea[i]) * eas[i];
      fb += (l % eb[i]) * ebs[i];
    }
    const double* a = ta + fa * s;
    const double* b = tb + fb * s;
    double* o = out + flat * s;
    if (op == TT_OP_ADD) {
      for (int64_t h = 0; h < s; ++h) o[h] = a[h] + b[h];
      if (c) c->additions += 1;
    } else {
      for (int64_t h = 0; h < s; ++h) o[h] = a[h] * b[h];
      if (c) c->multiplications += 1;
    }
  }
  return OR_OK;
}

/* tt_sum tile_tensor.hpp:286-347, including the '?' boundary split. */
int or_sum(const tt_shape* sh, const double* tin, int64_t s, int dim, int variant, tt_shape* so,
           double* out, tt_cost* c) {
  int rc = or_sum_result_shape(sh, dim, so);
  if (rc) return rc;
  const int rank = sh->rank;
  const int di = dim - 1;
  const tt_dim* ds = &sh->dims[di];
  const size_t bytes = (size_t)s * sizeof(double);
  const int64_t n_in = or_tile_count(sh);
  /* builder's `~` rule I9: the '?' boundary split assumes
   * a used prefix per tile; an unknown interleaved dim must be cleaned first */
  if (ds->interleaved && ds->unknown && ds->n * ds->d < ((ds->n * ds->d + ds->t - 1) / ds->t) * ds->t)
    return OR_SHAPE;
  if (ds->n == 1 && ds->d > 1) { /* degenerate: tiles unchanged :295 */
    memmove(out, tin, (size_t)n_in * bytes);
    return OR_OK;
  }
  int64_t ext[TT_MAX_RANK], es[TT_MAX_RANK], tst[TT_MAX_RANK];
  or_external(sh, ext);
  row_major(ext, rank, es);
  tile_strides(sh, tst);
  const int64_t ei = ext[di];
  const int64_t stride = tst[di];
  const int boundary_split = ds->unknown && (used_of(ds) % ds->t) != 0;
  const int64_t known_tail = used_of(ds) - (ei - 1) * ds->t;
  const int v_t = variant >= 0 ? variant
                               : (is_pow2(ds->t) ? TT_VARIANT_POWER_OF_TWO : TT_VARIANT_RIGHT_TO_LEFT);
  const int v_tail = variant >= 0 ? variant
                                  : (is_pow2(known_tail) ? TT_VARIANT_POWER_OF_TWO
                                                         : TT_VARIANT_RIGHT_TO_LEFT);
  int64_t gext[TT_MAX_RANK];
  for (int i = 0; i < rank; ++i) gext[i] = ext[i];
  gext[di] = 1;
  const int64_t n_groups = or_tile_count(so);
  double* acc = (double*)malloc(bytes);
  double* head = (double*)malloc(bytes);
  int64_t g[TT_MAX_RANK];
  for (int i = 0; i < rank; ++i) g[i] = 0;
  for (int64_t flat_out = 0; flat_out < n_groups; ++flat_out) {
    int64_t base = 0;
    for (int i = 0; i < rank; ++i) base += g[i] * es[i];
    const int64_t step = es[di];
    if (!boundary_split) {
      memcpy(acc, tin + base * s, bytes);
      for (int64_t li = 1; li < ei; ++li) tile_add(acc, tin + (base + li * step) * s, acc, s, c);
      if (ds->t > 1) {
        rc = or_sum_tile_strided(acc, s, ds->t, stride, v_t, acc, c);
        if (rc) break;
      }
    } else {
      memcpy(acc, tin + (base + (ei - 1) * step) * s, bytes); /* tail */
      if (known_tail > 1) {
        rc = or_sum_tile_strided(acc, s, known_tail, stride, v_tail, acc, c);
        if (rc) break;
      }
      if (ei > 1) {
        memcpy(head, tin + base * s, bytes);
        for (int64_t li = 1; li < ei - 1; ++li)
          tile_add(head, tin + (base + li * step) * s, head, s, c);
        if (ds->t > 1) {
          rc = or_sum_tile_strided(head, s, ds->t, stride, v_t, head, c);
          if (rc) break;
        }
        tile_add(head, acc, acc, s, c);
      }
    }
    memcpy(out + flat_out * s, acc, bytes);
    for (int i = rank - 1; i >= 0; --i) {
      if (++g[i] < gext[i]) break;
      g[i] = 0;
    }
  }
  free(acc);
  free(head);
  return rc;
}

/* used-slot predicate of clean_unknowns tile_tensor.hpp:364-378 (same as pack). */
int or_clean_unknowns(const tt_shape* sh, const double* tin, int64_t s, tt_shape* so, double* out,
                      tt_cost* c) {
  *so = *sh;
  const int64_t n = or_tile_count(sh);
  if (!has_unknown(sh)) {
    memmove(out, tin, (size_t)(n * s) * sizeof(double));
    return OR_OK;
  }
  const int rank = sh->rank;
  int64_t ext[TT_MAX_RANK], es[TT_MAX_RANK], tst[TT_MAX_RANK];
  or_external(sh, ext);
  row_major(ext, rank, es);
  tile_strides(sh, tst);
  const int64_t ts = or_tile_slots(sh);
  for (int64_t flat = 0; flat < n; ++flat) {
    for (int64_t h = 0; h < s; ++h) {
      double mask = 0.0;
      if (h < ts) {
        int used = 1;
        for (int i = 0; i < rank; ++i) {
          const tt_dim* ds = &sh->dims[i];
          const int64_t l = (flat / es[i]) % ext[i];
          const int64_t j = logical_j(ds, ext[i], l, (h / tst[i]) % ds->t);
          if (j >= used_of(ds)) {
            used = 0;
            break;
          }
        }
        if (used) mask = 1.0;
      }
      out[flat * s + h] = tin[flat * s + h] * mask;
    }
    if (c) c->mask_multiplications += 1;
  }
  for (int i = 0; i < rank; ++i) so->dims[i].unknown = 0;
  return OR_OK;
}

/* replicate_dim tile_tensor.hpp:391-420. */
int or_replicate_dim(const tt_shape* sh, const double* tin, int64_t s, int dim, tt_shape* so,
                     double* out, tt_cost* c) {
  if (dim < 1 || dim > sh->rank) return OR_SHAPE;
  const tt_dim* ds = &sh->dims[dim - 1];
  if (ds->unknown) return OR_SHAPE;
  if (ds->n != 1 || ds->d != 1) return OR_SHAPE;
  if (sh->relaxed) return OR_SHAPE;
  *so = *sh;
  const int64_t n = or_tile_count(sh);
  if (ds->t == 1) {
    memmove(out, tin, (size_t)(n * s) * sizeof(double));
    return OR_OK;
  }
  int64_t te[TT_MAX_RANK];
  for (int i = 0; i < sh->rank; ++i) te[i] = sh->dims[i].t;
  for (int64_t flat = 0; flat < n; ++flat)
    or_replicate_tile_dim(tin + flat * s, s, te, sh->rank, dim, out + flat * s, c);
  so->dims[dim - 1].d = ds->t;
  so->dims[dim - 1].interleaved = 0; /* I13: a replicated dim is not interleaved */
  return OR_OK;
}

/* ---- dense oracle (dense.hpp:107-165) -------------------------------------- */

/* dense_elementwise dense.hpp:109-133 (broadcast by index mod extent). */
int or_dense_elementwise(int op, const double* a, const int64_t* ea, const double* b,
                         const int64_t* eb, int rank, double* out, int64_t* eo) {
  int64_t total = 1;
  for (int i = 0; i < rank; ++i) {
    if (ea[i] != eb[i] && ea[i] != 1 && eb[i] != 1) return OR_SHAPE;
    eo[i] = ea[i] > eb[i] ? ea[i] : eb[i];
    total *= eo[i];
  }
  int64_t idx[TT_MAX_RANK];
  for (int i = 0; i < rank; ++i) idx[i] = 0;
  for (int64_t f = 0; f < total; ++f) {
    int64_t fa = 0, fb = 0;
    for (int i = 0; i < rank; ++i) {
      fa = fa * ea[i] + idx[i] % ea[i];
      fb = fb * eb[i] + idx[i] % eb[i];
    }
    out[f] = op == TT_OP_ADD ? a[fa] + b[fb] : a[fa] * b[fb];
    for (int i = rank - 1; i >= 0; --i) {
      if (++idx[i] < eo[i]) break;
      idx[i] = 0;
    }
  }
  return OR_OK;
}

/* dense_sum dense.hpp:135-149 (accumulates from 0.0 in row-major order). */
int or_dense_sum(const double* a, const int64_t* ea, int rank, int dim, double* out) {
  if (dim < 1 || dim > rank) return OR_SHAPE;
  int64_t eo[TT_MAX_RANK], total = 1, out_total = 1;
  for (int i = 0; i < rank; ++i) {
    eo[i] = ea[i];
    total *= ea[i];
  }
  eo[dim - 1] = 1;
  for (int i = 0; i < rank; ++i) out_total *= eo[i];
  for (int64_t f = 0; f < out_total; ++f) out[f] = 0.0;
  int64_t idx[TT_MAX_RANK];
  for (int i = 0; i < rank; ++i) idx[i] = 0;
  for (int64_t f = 0; f < total; ++f) {
    int64_t fo = 0;
    for (int i = 0; i < rank; ++i) fo = fo * eo[i] + (i == dim - 1 ? 0 : idx[i]);
    out[fo] += a[f];
    for (int i = rank - 1; i >= 0; --i) {
      if (++idx[i] < ea[i]) break;
      idx[i] = 0;
    }
  }
  return OR_OK;
}

/* dense_matmul dense.hpp:151-165 (naive ijk, acc from 0). */
void or_dense_matmul(const double* a, const double* b, int64_t m, int64_t k, int64_t n,
                     double* out) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0;
      for (int64_t x = 0; x < k; ++x) acc += a[i * k + x] * b[x * n + j];
      out[i * n + j] = acc;
    }
}

/* max_rel_diff dense.hpp:188-198 */
double or_max_rel_diff(const double* a, const double* b, int64_t n) {
  double worst = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double va = a[i] < 0 ? -a[i] : a[i];
    const double vb = b[i] < 0 ? -b[i] : b[i];
    double denom = va > vb ? va : vb;
    if (denom < 1.0) denom = 1.0;
    double diff = a[i] - b[i];
    if (diff < 0) diff = -diff;
    const double r = diff / denom;
    if (r > worst || r != r) worst = r;
  }
  return worst;
}

/* ---- shared synthetic input generator --------------------------
 * u = splitmix64(seed, i);  x = lo + (hi-lo) * (u>>11) * 2^-53.
 * The same formula runs on the device (bench/tests) so both sides see
 * bit-identical inputs. */
static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

void or_fill_uniform(double* out, int64_t count, uint64_t seed, int64_t offset, double lo,
                     double hi) {
  const uint64_t key = splitmix64(seed);
  for (int64_t i = 0; i < count; ++i) {
    const uint64_t u = splitmix64(key ^ (uint64_t)(offset + i));
    out[i] = lo + (hi - lo) * ((double)(u >> 11) * 0x1.0p-53);
  }
}

/* tt_pyfast.c -- vectorcall (METH_FASTCALL) entry points for the Python
 * mirror's small-op fast path (paper_2011_01805_b200/tiletensor.py, _FAST).
 *
 * A repeated small op (config 1: 49 tiles of 512 slots) is host bound: its
 * kernel runs in ~3.4 us, while a ctypes call with a dozen arguments spends
 * ~1.5 us converting them.  These functions take plain Python ints (the
 * session handle, the addresses of cached tt_shape structs, device pointers,
 * chain indices) and forward them to the C-ABI unchanged -- no validation is
 * skipped: every call still goes through tt_mul_sum / tt_sum / ... which
 * check shapes, slots and depth before launching.  Each returns the C-ABI
 * status code; the Python side maps it to the reference's exception types.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include "tiletensor_b200.h"

static int get_ll(PyObject* o, long long* v) {
  *v = PyLong_AsLongLong(o);
  return !(*v == -1 && PyErr_Occurred());
}

#define ARGS(n)                                                              \
  long long a[n];                                                            \
  if (nargs != n) {                                                          \
    PyErr_SetString(PyExc_TypeError, "wrong number of arguments");           \
    return NULL;                                                             \
  }                                                                          \
  for (Py_ssize_t i = 0; i < n; ++i)                                         \
    if (!get_ll(args[i], &a[i])) return NULL;

#define P(i) ((void*)(intptr_t)a[i])
#define SHP(i) ((const tt_shape*)(intptr_t)a[i])
#define DP(i) ((const double*)(intptr_t)a[i])

/* mul_sum(session, sa, ta, chain_a, sb, tb, chain_b, dim, variant, out) */
static PyObject* f_mul_sum(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  ARGS(10)
  return PyLong_FromLong(tt_mul_sum((tt_session*)P(0), SHP(1), DP(2), a[3], SHP(4), DP(5), a[6],
                                    (int)a[7], (int)a[8], NULL, (double*)P(9), NULL));
}

/* product(session, which, sa, ta, chain_a, sb, tb, chain_b, variant, out) */
static PyObject* f_product(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  ARGS(10)
  return PyLong_FromLong(tt_linalg_product((tt_session*)P(0), (int)a[1], SHP(2), DP(3), a[4],
                                           SHP(5), DP(6), a[7], (int)a[8], NULL, (double*)P(9),
                                           NULL));
}

/* elementwise(session, op, sa, ta, chain_a, sb, tb, chain_b, out) */
static PyObject* f_elementwise(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  ARGS(9)
  return PyLong_FromLong(tt_elementwise((tt_session*)P(0), (int)a[1], SHP(2), DP(3), a[4], SHP(5),
                                        DP(6), a[7], NULL, (double*)P(8), NULL));
}

/* sum(session, s_in, t_in, dim, variant, out) */
static PyObject* f_sum(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  ARGS(6)
  return PyLong_FromLong(
      tt_sum((tt_session*)P(0), SHP(1), DP(2), (int)a[3], (int)a[4], NULL, (double*)P(5)));
}

/* The *_new forms allocate the result from the session's tile cache
 * (tt_tiles_alloc, `nbytes`) and return its device address, -status on
 * error (the block is released again), or 0 under stream capture (nothing
 * ran: the caller takes its regular path). */
#define NEW_RESULT(call)                                   \
  void* out = NULL;                                        \
  int rc = tt_tiles_alloc((tt_session*)P(0), nbytes, &out); \
  if (rc == 0 && out == NULL) return PyLong_FromLong(0);  \
  if (rc == 0) {                                           \
    rc = (call);                                           \
    if (rc != 0) tt_tiles_release((tt_session*)P(0), out); \
  }                                                        \
  return rc ? PyLong_FromLong(-rc) : PyLong_FromVoidPtr(out);

/* mul_sum_new(session, sa, ta, chain_a, sb, tb, chain_b, dim, variant, nbytes) */
static PyObject* f_mul_sum_new(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  ARGS(10)
  const long long nbytes = a[9];
  NEW_RESULT(tt_mul_sum((tt_session*)P(0), SHP(1), DP(2), a[3], SHP(4), DP(5), a[6], (int)a[7],
                        (int)a[8], NULL, (double*)out, NULL))
}

/* product_new(session, which, sa, ta, chain_a, sb, tb, chain_b, variant, nbytes) */
static PyObject* f_product_new(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  ARGS(10)
  const long long nbytes = a[9];
  NEW_RESULT(tt_linalg_product((tt_session*)P(0), (int)a[1], SHP(2), DP(3), a[4], SHP(5), DP(6),
                               a[7], (int)a[8], NULL, (double*)out, NULL))
}

/* elementwise_new(session, op, sa, ta, chain_a, sb, tb, chain_b, nbytes) */
static PyObject* f_elementwise_new(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  ARGS(9)
  const long long nbytes = a[8];
  NEW_RESULT(tt_elementwise((tt_session*)P(0), (int)a[1], SHP(2), DP(3), a[4], SHP(5), DP(6), a[7],
                            NULL, (double*)out, NULL))
}

/* sum_new(session, s_in, t_in, dim, variant, nbytes) */
static PyObject* f_sum_new(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  ARGS(6)
  const long long nbytes = a[5];
  NEW_RESULT(tt_sum((tt_session*)P(0), SHP(1), DP(2), (int)a[3], (int)a[4], NULL, (double*)out))
}

/* release(session, ptr) */
static PyObject* f_release(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  ARGS(2)
  return PyLong_FromLong(tt_tiles_release((tt_session*)P(0), P(1)));
}

static PyMethodDef methods[] = {
    {"mul_sum_new", (PyCFunction)(void (*)(void))f_mul_sum_new, METH_FASTCALL, "tt_mul_sum into a cached block"},
    {"product_new", (PyCFunction)(void (*)(void))f_product_new, METH_FASTCALL, "tt_linalg_product into a cached block"},
    {"elementwise_new", (PyCFunction)(void (*)(void))f_elementwise_new, METH_FASTCALL, "tt_elementwise into a cached block"},
    {"sum_new", (PyCFunction)(void (*)(void))f_sum_new, METH_FASTCALL, "tt_sum into a cached block"},
    {"release", (PyCFunction)(void (*)(void))f_release, METH_FASTCALL, "tt_tiles_release"},
    {"mul_sum", (PyCFunction)(void (*)(void))f_mul_sum, METH_FASTCALL, "tt_mul_sum"},
    {"product", (PyCFunction)(void (*)(void))f_product, METH_FASTCALL, "tt_linalg_product"},
    {"elementwise", (PyCFunction)(void (*)(void))f_elementwise, METH_FASTCALL, "tt_elementwise"},
    {"sum", (PyCFunction)(void (*)(void))f_sum, METH_FASTCALL, "tt_sum"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_ttfast", NULL, -1, methods,
                                    NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__ttfast(void) { return PyModule_Create(&module); }

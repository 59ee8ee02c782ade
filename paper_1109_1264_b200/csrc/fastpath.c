/*
 * fastpath.c — CPython extension `_fastpath`: the common case of the host
 * layer in C.
 *
 * For trees whose leaves and destination are plain device DenseVectors on the
 * current CUDA device, this walks the node objects (Leaf / AddNode / SubNode /
 * MulNode / ScaleNode), builds the same canonical postfix signature as
 * expressions.lower(), collects the leaf pointers, element-typed scalars and
 * DeviceScalar addresses (P<k>),
 * and calls libsalt.so's C ABI directly — replacing ~10 us of Python per call
 * (profiles/r01_api_overhead.json) by ~1 us.  Anything else (other vector
 * types, host or sharded vectors, mismatched lengths/dtypes/devices, trees
 * beyond one kernel, plan options) returns "not handled" and the Python path
 * runs — which also raises the reference's exceptions.  It is a host-side
 * accelerator only: there is no CPU arithmetic here.
 *
 * libsalt.so's entry points are passed in as addresses from the ctypes
 * handle (init()), so both share one library instance.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#define MAX_LEAVES 16
#define MAX_SCALARS 32
#define MAX_SIG 1024
#define MAX_PSCALARS 8
#define MAX_ROOTS 4

typedef int (*assign_fn)(int, const char*, void*, const void* const*, int, const double*, int,
                         int64_t, void*);
typedef int (*reduce_fn)(int, const char*, const void* const*, int, const double*, int, int64_t,
                         int, void*, size_t, void*, void*, void*);
typedef int (*assign_reduce_fn)(int, const char*, const char*, void*, const void* const*, int,
                                const double*, int, int64_t, int, void*, size_t, void*, void*,
                                void*);
typedef int (*fused_fn)(int, const char*, const char*, void* const*, int, const void* const*, int,
                        const double*, int, const void* const*, int, int64_t, int, void*, size_t,
                        void*, void*, void*);
typedef int (*assign_batch_fn)(int, const char*, int, void* const*, const void* const*, int,
                               const double*, int, const int64_t*, void*);
typedef int (*reduce_batch_fn)(int, const char*, int, const void* const*, int, const double*, int,
                               const int64_t*, int, void* const*, void*, size_t, void*);
typedef int (*fused_prog_fn)(int, const char*, const char*, void* const*, int, const void* const*,
                             int, const double*, int, const void* const*, int, const char*, int64_t,
                             int, void*, size_t, void*, void*, void*);
typedef const char* (*last_error_fn)(void);
typedef int (*result_enqueue_fn)(const void*, size_t, void*, void**);
typedef int (*result_slot_fn)(void**);
typedef int (*stream_sync_fn)(void*);

static assign_fn p_assign;
static reduce_fn p_reduce;
static assign_reduce_fn p_assign_reduce;
static fused_fn p_fused;
static assign_batch_fn p_assign_batch;
static reduce_batch_fn p_reduce_batch;
static PyObject* batch_out; /* runtime._batch_out(device, count) -> (tensor, data_ptr) */
static last_error_fn p_last_error;
static fused_prog_fn p_fused_prog;
static result_enqueue_fn p_result_enqueue;
static result_slot_fn p_result_slot;
static stream_sync_fn p_stream_sync;
static size_t ws_bytes;

static PyObject *T_Leaf, *T_Add, *T_Sub, *T_Mul, *T_Scale, *T_Dense, *T_DevScalar;
static PyObject *get_stream, *current_device, *workspace_fn, *np_f32, *np_f64, *lazy_out;
static PyObject *s_vector, *s_left, *s_right, *s_child, *s_alpha, *s_ptr, *s_dev, *s_n, *s_code,
    *s_data_ptr, *s_tensor, *s_get_device, *s_expr, *s_check_operands;

typedef struct {
  char sig[MAX_SIG];
  int len;
  PyObject* vecs[MAX_LEAVES];
  void* ptrs[MAX_LEAVES];
  int nvec;
  double sc[MAX_SCALARS];
  int nsc;
  const void* ps[MAX_PSCALARS]; /* DeviceScalar operands (P<k>) */
  int nps;
  /* lazy DeviceScalars (unevaluated scalar operations): the tree's P<k>
   * come from a scalar program over raw device scalars (salt_fused_prog) */
  PyObject* pobj[MAX_PSCALARS];
  int lazy;
  char prog[512];
  int plen;
  const void* raw[MAX_PSCALARS];
  PyObject* rawobj[MAX_PSCALARS];
  int nraw;
  int dev, code;
  long long n;
  /* vectors assigned by earlier roots of the same kernel: a later tree reads
   * them as D<k>, the value root k has just computed (latest root wins) */
  PyObject* dests[MAX_ROOTS];
  int ndests;
} Walk;

/* 1 = ok, 0 = not eligible (fall back), -1 = Python error */
static int emit(Walk* w, const char* tok) {
  int k = (int)strlen(tok);
  if (w->len + k + 1 >= MAX_SIG) return 0;
  if (w->len) w->sig[w->len++] = ' ';
  memcpy(w->sig + w->len, tok, (size_t)k);
  w->len += k;
  w->sig[w->len] = '\0';
  return 1;
}

static int long_attr(PyObject* o, PyObject* name, long long* out) {
  PyObject* v = PyObject_GetAttr(o, name);
  if (!v) return -1;
  *out = PyLong_AsLongLong(v);
  Py_DECREF(v);
  return (*out == -1 && PyErr_Occurred()) ? -1 : 1;
}

static int leaf(Walk* w, PyObject* vec) {
  char tok[16];
  for (int k = w->ndests - 1; k >= 0; --k)
    if (w->dests[k] == vec) {
      snprintf(tok, sizeof tok, "D%d", k);
      return emit(w, tok);
    }
  for (int k = 0; k < w->nvec; ++k)
    if (w->vecs[k] == vec) {
      snprintf(tok, sizeof tok, "L%d", k);
      return emit(w, tok);
    }
  if ((PyObject*)Py_TYPE(vec) != T_Dense || w->nvec == MAX_LEAVES) return 0;
  long long dev, code, n, ptr;
  if (long_attr(vec, s_dev, &dev) < 0 || long_attr(vec, s_code, &code) < 0 ||
      long_attr(vec, s_n, &n) < 0 || long_attr(vec, s_ptr, &ptr) < 0)
    return -1;
  if (dev != w->dev || code != w->code || n != w->n) return 0;
  w->vecs[w->nvec] = vec;
  w->ptrs[w->nvec] = (void*)(intptr_t)ptr;
  snprintf(tok, sizeof tok, "L%d", w->nvec++);
  return emit(w, tok);
}

/* Pointer of a materialised DeviceScalar on device `dev`: 1 ok, 0 other
 * device, -1 error. */
static int scalar_ptr(PyObject* t, int dev, void** ptr) {
  PyObject* d = PyObject_CallMethodNoArgs(t, s_get_device);
  PyObject* p = d ? PyObject_CallMethodNoArgs(t, s_data_ptr) : NULL;
  if (!p) { Py_XDECREF(d); return -1; }
  long dv = PyLong_AsLong(d);
  *ptr = PyLong_AsVoidPtr(p);
  Py_DECREF(d);
  Py_DECREF(p);
  if (PyErr_Occurred()) return -1;
  return dv == dev ? 1 : 0;
}

/* DeviceScalar -> w->ps[w->nps++]; must live on the kernel's device.  A
 * LAZY DeviceScalar (an unevaluated scalar operation, _tensor None) is kept
 * as an object: build_program() turns the tree's device scalars into a
 * scalar program over the raw device scalars underneath. */
static int device_scalar(Walk* w, PyObject* ds) {
  if (w->nps == MAX_PSCALARS) return 0;
  PyObject* t = PyObject_GetAttr(ds, s_tensor);
  if (!t) return -1;
  if (t == Py_None) {
    Py_DECREF(t);
    w->pobj[w->nps] = ds;
    w->ps[w->nps++] = NULL;
    w->lazy = 1;
    return 1;
  }
  w->pobj[w->nps] = ds;
  PyObject* d = PyObject_CallMethodNoArgs(t, s_get_device);
  PyObject* p = d ? PyObject_CallMethodNoArgs(t, s_data_ptr) : NULL;
  Py_DECREF(t);
  if (!p) { Py_XDECREF(d); return -1; }
  long dev = PyLong_AsLong(d);
  void* ptr = PyLong_AsVoidPtr(p);
  Py_DECREF(d);
  Py_DECREF(p);
  if (PyErr_Occurred()) return -1;
  if (dev != w->dev) return 0;
  w->ps[w->nps++] = ptr;
  return 1;
}

static int prog_tok(Walk* w, const char* tok) {
  const int k = (int)strlen(tok);
  if (w->plen + k + 2 >= (int)sizeof w->prog) return 0;
  if (w->plen) w->prog[w->plen++] = ' ';
  memcpy(w->prog + w->plen, tok, (size_t)k + 1);
  w->plen += k;
  return 1;
}

/* Postfix of one scalar operand (DeviceScalar, lazy or not, or a float)
 * into w->prog; *depth tracks the program's stack.  0 = too large for one
 * program (the Python path then materialises), -1 = Python error. */
static int prog_operand(Walk* w, PyObject* x, int* depth, int* ops) {
  char tok[16];
  if (++*ops > 30) return 0;
  if (PyFloat_Check(x)) {
    if (w->nsc == MAX_SCALARS) return 0;
    w->sc[w->nsc] = PyFloat_AS_DOUBLE(x);
    snprintf(tok, sizeof tok, "S%d", w->nsc++);
    if (++*depth > 8) return 0;
    return prog_tok(w, tok);
  }
  if ((PyObject*)Py_TYPE(x) != T_DevScalar) return 0;
  PyObject* t = PyObject_GetAttr(x, s_tensor);
  if (!t) return -1;
  if (t != Py_None) {  /* materialised: a raw device scalar */
    int i = 0;
    while (i < w->nraw && w->rawobj[i] != x) ++i;
    if (i == w->nraw) {
      if (w->nraw == MAX_PSCALARS) { Py_DECREF(t); return 0; }
      void* ptr;
      int rc = scalar_ptr(t, w->dev, &ptr);
      Py_DECREF(t);
      if (rc != 1) return rc;
      w->rawobj[i] = x;
      w->raw[i] = ptr;
      ++w->nraw;
    } else {
      Py_DECREF(t);
    }
    snprintf(tok, sizeof tok, "p%d", i);
    if (++*depth > 8) return 0;
    return prog_tok(w, tok);
  }
  Py_DECREF(t);
  PyObject* e = PyObject_GetAttr(x, s_expr);
  if (!e) return -1;
  int rc = 1;
  if (!PyTuple_Check(e) || PyTuple_GET_SIZE(e) < 2) rc = 0;
  for (Py_ssize_t i = 1; rc == 1 && i < PyTuple_GET_SIZE(e); ++i)
    rc = prog_operand(w, PyTuple_GET_ITEM(e, i), depth, ops);
  if (rc == 1) {
    const char* op = PyUnicode_AsUTF8(PyTuple_GET_ITEM(e, 0));
    if (!op) rc = -1;
    else {
      if (strcmp(op, "neg") != 0) --*depth;  /* binary: two in, one out */
      rc = prog_tok(w, op);
    }
  }
  Py_DECREF(e);
  return rc;
}

/* With lazy device scalars: the scalar program that defines every P<k> of
 * the tree, the raw device scalars it reads (w->raw) and its host constants
 * (appended to w->sc).  1 ok (or nothing to do), 0 decline, -1 error. */
static int build_program(Walk* w) {
  if (!w->lazy) return 1;
  for (int k = 0; k < w->nps; ++k) {
    /* refuses operands modified in place since the operation was recorded */
    PyObject* r = PyObject_CallMethodNoArgs(w->pobj[k], s_check_operands);
    if (!r) return -1;
    Py_DECREF(r);
  }
  int depth = 0, ops = 0;
  char tok[16];
  for (int k = 0; k < w->nps; ++k) {
    int rc = prog_operand(w, w->pobj[k], &depth, &ops);
    if (rc != 1) return rc;
    snprintf(tok, sizeof tok, "=%d", k);
    --depth;
    if (!prog_tok(w, tok)) return 0;
  }
  return 1;
}

/* salt_fused, or salt_fused_prog when the tree has lazy device scalars */
static int call_fused(Walk* w, const char* asig, const char* rsig, void* const* dsts, int ndst,
                      int flags, void* ws, void* out, void* host, void* stream) {
  const void* const* leaves = (const void* const*)w->ptrs;
  if (w->lazy)
    return p_fused_prog(w->code, asig, rsig, dsts, ndst, leaves, w->nvec, w->sc, w->nsc, w->raw,
                        w->nraw, w->prog, w->n, flags, ws, ws ? ws_bytes : 0, out, host, stream);
  return p_fused(w->code, asig, rsig, dsts, ndst, leaves, w->nvec, w->sc, w->nsc, w->ps, w->nps,
                 w->n, flags, ws, ws ? ws_bytes : 0, out, host, stream);
}

static int walk(Walk* w, PyObject* node) {
  PyObject* t = (PyObject*)Py_TYPE(node);
  int rc;
  if (t == T_Leaf) {
    PyObject* v = PyObject_GetAttr(node, s_vector);
    if (!v) return -1;
    rc = leaf(w, v);
    Py_DECREF(v);
    return rc;
  }
  if (t == T_Dense) return leaf(w, node); /* a bare vector used as a tree */
  if (t == T_Scale) {
    if (w->nsc == MAX_SCALARS) return 0;
    PyObject* a = PyObject_GetAttr(node, s_alpha);
    if (!a) return -1;
    char tok[16];
    if ((PyObject*)Py_TYPE(a) == T_DevScalar) {
      /* device-resident alpha (element type checked by ScaleNode): the
       * kernel reads it from device memory */
      rc = device_scalar(w, a);
      Py_DECREF(a);
      if (rc != 1) return rc;
      snprintf(tok, sizeof tok, "P%d", w->nps - 1);
    } else {
      double v = PyFloat_AsDouble(a); /* alpha is already element-typed */
      Py_DECREF(a);
      if (v == -1.0 && PyErr_Occurred()) return -1;
      snprintf(tok, sizeof tok, "S%d", w->nsc);
      w->sc[w->nsc++] = v;
    }
    if ((rc = emit(w, tok)) != 1) return rc;
    PyObject* c = PyObject_GetAttr(node, s_child);
    if (!c) return -1;
    rc = walk(w, c);
    Py_DECREF(c);
    return rc == 1 ? emit(w, "*") : rc;
  }
  const char* op = t == T_Add ? "+" : t == T_Sub ? "-" : t == T_Mul ? "*" : NULL;
  if (!op) return 0;
  PyObject* l = PyObject_GetAttr(node, s_left);
  if (!l) return -1;
  rc = walk(w, l);
  Py_DECREF(l);
  if (rc != 1) return rc;
  PyObject* r = PyObject_GetAttr(node, s_right);
  if (!r) return -1;
  rc = walk(w, r);
  Py_DECREF(r);
  return rc == 1 ? emit(w, op) : rc;
}

/* Destination checks; fills dev/code/n. 1 ok, 0 not eligible, -1 error. */
static int start(Walk* w, PyObject* dest, void** dptr) {
  memset(w, 0, sizeof *w);
  if ((PyObject*)Py_TYPE(dest) != T_Dense) return 0;
  long long dev, code, n, ptr;
  if (long_attr(dest, s_dev, &dev) < 0 || long_attr(dest, s_code, &code) < 0 ||
      long_attr(dest, s_n, &n) < 0 || long_attr(dest, s_ptr, &ptr) < 0)
    return -1;
  if (dev < 0) return 0;
  w->dev = (int)dev;
  w->code = (int)code;
  w->n = n;
  if (dptr) *dptr = (void*)(intptr_t)ptr;
  return 1;
}

/* Current device must be w->dev; returns the current stream handle. */
static int stream_for(Walk* w, void** stream) {
  PyObject* cur = PyObject_CallNoArgs(current_device);
  if (!cur) return -1;
  long c = PyLong_AsLong(cur);
  Py_DECREF(cur);
  if (c == -1 && PyErr_Occurred()) return -1;
  if (c != w->dev) return 0;
  PyObject* d = PyLong_FromLong(w->dev);
  PyObject* s = PyObject_CallOneArg(get_stream, d);
  Py_DECREF(d);
  if (!s) return -1;
  *stream = PyLong_AsVoidPtr(s);
  Py_DECREF(s);
  return PyErr_Occurred() ? -1 : 1;
}

static PyObject* check(int rc) {
  if (rc != 0) {
    PyErr_Format(PyExc_RuntimeError, "libsalt error %d: %s", rc, p_last_error());
    return NULL;
  }
  Py_RETURN_TRUE;
}

/* Workspace of (device, stream) from runtime._workspace; its last 256 bytes
 * hold the fast path's result slot (non-lazy reductions only). */
static int workspace(Walk* w, void* stream, void** ws, void** slot) {
  PyObject* t = PyObject_CallFunction(workspace_fn, "iK", w->dev,
                                      (unsigned long long)(uintptr_t)stream);
  if (!t) return -1;
  PyObject* p = PyObject_CallMethodNoArgs(t, s_data_ptr);
  Py_DECREF(t);
  if (!p) return -1;
  *ws = PyLong_AsVoidPtr(p);
  Py_DECREF(p);
  *slot = (char*)*ws + ws_bytes;
  return PyErr_Occurred() ? -1 : 1;
}

static PyObject* scalar_result(Walk* w, const double* host) {
  if (w->code == 0) {
    float f;
    memcpy(&f, host, sizeof f);
    return PyObject_CallFunction(np_f32, "d", (double)f);
  }
  return PyObject_CallFunction(np_f64, "d", host[0]);
}

#define TRY(expr)                 \
  do {                            \
    int rc_ = (expr);             \
    if (rc_ < 0) return NULL;     \
    if (rc_ == 0) Py_RETURN_FALSE; \
  } while (0)

/* assign(dest, source) -> True if launched, False if not eligible */
static PyObject* fp_assign(PyObject* self, PyObject* args) {
  PyObject *dest, *src;
  if (!PyArg_ParseTuple(args, "OO", &dest, &src)) return NULL;
  Walk w;
  void *dptr, *stream;
  TRY(start(&w, dest, &dptr));
  TRY(walk(&w, src));
  if (w.nvec == 0) Py_RETURN_FALSE;
  TRY(build_program(&w));
  TRY(stream_for(&w, &stream));
  if (w.n == 0) Py_RETURN_TRUE;
  if (w.nps) return check(call_fused(&w, w.sig, NULL, &dptr, 1, 0, NULL, NULL, NULL, stream));
  return check(p_assign(w.code, w.sig, dptr, (const void* const*)w.ptrs, w.nvec, w.sc, w.nsc,
                        w.n, stream));
}

/* Device result of a lazy reduction: (DeviceScalar, out pointer) from the
 * Python helper runtime._lazy_out(device, code). */
static PyObject* lazy_slot(Walk* w, void** out) {
  PyObject* r = PyObject_CallFunction(lazy_out, "ii", w->dev, w->code);
  if (!r) return NULL;
  PyObject* ds = PyTuple_GetItem(r, 0);
  PyObject* ptr = PyTuple_GetItem(r, 1);
  if (!ds || !ptr) { Py_DECREF(r); return NULL; }
  *out = PyLong_AsVoidPtr(ptr);
  Py_INCREF(ds);
  Py_DECREF(r);
  return ds;
}

/* One reducing launch: reduce-only (asig NULL) or assignments + reduction.
 * Lazy: the result stays on the device (DeviceScalar); else the NumPy scalar. */
static PyObject* launch_reduce(Walk* w, const char* asig, void* const* dptrs, int ndst, int flags,
                               int lazy, void* ws, void* slot, void* stream) {
  PyObject* ds = NULL;
  void* out = slot;
  void* direct = NULL; /* this thread's device-mapped pinned slot, if any */
  double host[2] = {0.0, 0.0};
  if (lazy && !(ds = lazy_slot(w, &out))) return NULL;
  /* Non-lazy, preferred: the kernel stores the result straight into this
   * thread's pinned host slot (mapped at the same address on the device),
   * so nothing is copied afterwards. */
  if (!lazy && p_result_slot && p_result_slot(&direct) == 0) out = direct;
  else direct = NULL;
  /* Non-lazy: the kernel writes the workspace's result slot and the copy to
   * this thread's pinned slot is enqueued behind it with the GIL held (a
   * later reduction on the same stream — same workspace — is ordered after
   * the copy); only the wait for the stream runs without the GIL, so other
   * Python threads progress during a long reduction. */
  const void* const* leaves = (const void* const*)w->ptrs;
  int rc;
  if (w->nps || ndst > 1)
    rc = call_fused(w, asig, w->sig, dptrs, ndst, flags, ws, out, NULL, stream);
  else if (asig)
    rc = p_assign_reduce(w->code, asig, w->sig, dptrs[0], leaves, w->nvec, w->sc, w->nsc, w->n,
                         flags, ws, ws_bytes, out, NULL, stream);
  else
    rc = p_reduce(w->code, w->sig, leaves, w->nvec, w->sc, w->nsc, w->n, flags, ws, ws_bytes, out,
                  NULL, stream);
  if (rc != 0) {
    Py_XDECREF(ds);
    return check(rc);
  }
  if (lazy) return ds;
  const size_t bytes = (flags & 2) ? 16 : (w->code == 0 ? 4 : 8);
  void* hslot = direct;
  if (!direct) {
    rc = p_result_enqueue(out, bytes, stream, &hslot);
    if (rc != 0) return check(rc);
  }
  Py_BEGIN_ALLOW_THREADS
  rc = p_stream_sync(stream);
  Py_END_ALLOW_THREADS
  if (rc != 0) return check(rc);
  memcpy(host, hslot, bytes);
  return scalar_result(w, host);
}

/* reduce(child, flags, lazy) -> NumPy scalar (or DeviceScalar if lazy), or
 * None if not eligible */
static PyObject* fp_reduce(PyObject* self, PyObject* args) {
  PyObject* child;
  int flags, lazy = 0;
  if (!PyArg_ParseTuple(args, "Oi|p", &child, &flags, &lazy)) return NULL;
  Walk w;
  memset(&w, 0, sizeof w);
  /* the first leaf fixes device / dtype / length */
  PyObject* first = child;
  while ((PyObject*)Py_TYPE(first) != T_Leaf && (PyObject*)Py_TYPE(first) != T_Dense) {
    PyObject* t = (PyObject*)Py_TYPE(first);
    PyObject* nxt = PyObject_GetAttr(first, t == T_Scale ? s_child : s_left);
    if (!nxt) { PyErr_Clear(); Py_RETURN_NONE; }
    Py_DECREF(nxt); /* nodes are kept alive by their parents */
    first = nxt;
  }
  PyObject* v0 = (PyObject*)Py_TYPE(first) == T_Leaf ? PyObject_GetAttr(first, s_vector) : (Py_INCREF(first), first);
  if (!v0) return NULL;
  int rc = start(&w, v0, NULL);
  Py_DECREF(v0);
  if (rc < 0) return NULL;
  if (rc == 0) Py_RETURN_NONE;
  rc = walk(&w, child);
  if (rc < 0) return NULL;
  if (rc == 1) rc = build_program(&w);
  if (rc < 0) return NULL;
  void* stream;
  if (rc == 0 || (rc = stream_for(&w, &stream)) == 0) Py_RETURN_NONE;
  if (rc < 0) return NULL;
  void *ws, *slot;
  if (workspace(&w, stream, &ws, &slot) < 0) return NULL;
  return launch_reduce(&w, NULL, NULL, 0, flags, lazy, ws, slot, stream);
}

/* assign_reduce(dest, assign_source, reduce_child, flags) -> scalar or None */
static PyObject* fp_assign_reduce(PyObject* self, PyObject* args) {
  PyObject *dest, *src, *child;
  int flags, lazy = 0;
  if (!PyArg_ParseTuple(args, "OOOi|p", &dest, &src, &child, &flags, &lazy)) return NULL;
  Walk w;
  void *dptr, *stream;
  int rc = start(&w, dest, &dptr);
  if (rc <= 0) { if (rc < 0) return NULL; Py_RETURN_NONE; }
  rc = walk(&w, src);
  if (rc <= 0) { if (rc < 0) return NULL; Py_RETURN_NONE; }
  char asig[MAX_SIG];
  memcpy(asig, w.sig, (size_t)w.len + 1);
  w.len = 0;
  w.sig[0] = '\0';
  w.dests[w.ndests++] = dest;
  rc = walk(&w, child);
  if (rc <= 0) { if (rc < 0) return NULL; Py_RETURN_NONE; }
  if (w.nvec == 0) Py_RETURN_NONE;
  rc = build_program(&w);
  if (rc <= 0) { if (rc < 0) return NULL; Py_RETURN_NONE; }
  rc = stream_for(&w, &stream);
  if (rc <= 0) { if (rc < 0) return NULL; Py_RETURN_NONE; }
  void *ws, *slot;
  if (workspace(&w, stream, &ws, &slot) < 0) return NULL;
  return launch_reduce(&w, asig, &dptr, 1, flags, lazy, ws, slot, stream);
}

/* fused(((dest, source), ...), total_child or None, flags, lazy) -> (result,)
 * if launched (result None without a total), None if not eligible.  The
 * statements run in order in ONE kernel (a later tree reads an earlier
 * destination as D<k>); same signatures as FusedNode.lower(). */
static PyObject* fp_fused(PyObject* self, PyObject* args) {
  PyObject *assigns, *total;
  int flags, lazy = 0;
  if (!PyArg_ParseTuple(args, "OOi|p", &assigns, &total, &flags, &lazy)) return NULL;
  if (!PyTuple_Check(assigns) && !PyList_Check(assigns)) Py_RETURN_NONE;
  Py_ssize_t na = PySequence_Fast_GET_SIZE(assigns);
  if (na < 1 || na > MAX_ROOTS) Py_RETURN_NONE;
  PyObject** items = PySequence_Fast_ITEMS(assigns);
  Walk w;
  void* dptrs[MAX_ROOTS];
  char asig[MAX_SIG];
  int alen = 0, rc;
  for (Py_ssize_t k = 0; k < na; ++k) {
    PyObject* st = items[k];
    if (!PyTuple_Check(st) || PyTuple_GET_SIZE(st) != 2) Py_RETURN_NONE;
    PyObject *dest = PyTuple_GET_ITEM(st, 0), *src = PyTuple_GET_ITEM(st, 1);
    if (k == 0) {
      rc = start(&w, dest, &dptrs[0]);
    } else {
      Walk d;
      rc = start(&d, dest, &dptrs[k]);
      if (rc == 1 && (d.dev != w.dev || d.code != w.code || d.n != w.n)) rc = 0;
    }
    if (rc <= 0) { if (rc < 0) return NULL; Py_RETURN_NONE; }
    w.len = 0;
    w.sig[0] = '\0';
    rc = walk(&w, src);
    if (rc <= 0) { if (rc < 0) return NULL; Py_RETURN_NONE; }
    if (alen + w.len + 4 >= MAX_SIG) Py_RETURN_NONE;
    if (k) { memcpy(asig + alen, " ; ", 3); alen += 3; }
    memcpy(asig + alen, w.sig, (size_t)w.len + 1);
    alen += w.len;
    w.dests[w.ndests++] = dest;
  }
  w.len = 0;
  w.sig[0] = '\0';
  if (total != Py_None) {
    rc = walk(&w, total);
    if (rc <= 0) { if (rc < 0) return NULL; Py_RETURN_NONE; }
  }
  if (w.nvec == 0) Py_RETURN_NONE;
  rc = build_program(&w);
  if (rc <= 0) { if (rc < 0) return NULL; Py_RETURN_NONE; }
  void* stream;
  rc = stream_for(&w, &stream);
  if (rc <= 0) { if (rc < 0) return NULL; Py_RETURN_NONE; }
  PyObject* result;
  if (total == Py_None) {
    if (w.n) {
      rc = call_fused(&w, asig, NULL, dptrs, (int)na, 0, NULL, NULL, NULL, stream);
      if (rc != 0) return check(rc);
    }
    Py_INCREF(Py_None);
    result = Py_None;
  } else {
    void *ws, *slot;
    if (workspace(&w, stream, &ws, &slot) < 0) return NULL;
    result = launch_reduce(&w, asig, dptrs, (int)na, flags, lazy, ws, slot, stream);
    if (!result) return NULL;
  }
  PyObject* t = PyTuple_Pack(1, result);
  Py_DECREF(result);
  return t;
}

/* op(sig, dest_or_None, leaves_tuple, alpha_or_None, flags, lazy): a named
 * operation (ops.py) without building node objects.  `sig` is the
 * signature expressions.lower() gives that operation for these operands
 * (the caller picks it, deduplicating repeated vectors); `alpha` is coerced
 * to the element type like ScaleNode does.  Assignments return True,
 * reductions their result; None = not eligible (the node path runs). */
static PyObject* fp_op(PyObject* self, PyObject* args) {
  const char* sig;
  PyObject *dest, *leaves, *alpha;
  int flags, lazy = 0;
  if (!PyArg_ParseTuple(args, "yOO!Oi|p", &sig, &dest, &PyTuple_Type, &leaves, &alpha, &flags,
                        &lazy))
    return NULL;
  Py_ssize_t nl = PyTuple_GET_SIZE(leaves);
  if (nl < 1 || nl > MAX_LEAVES) Py_RETURN_NONE;
  Walk w;
  void* dptr = NULL;
  int rc = start(&w, dest != Py_None ? dest : PyTuple_GET_ITEM(leaves, 0),
                 dest != Py_None ? &dptr : NULL);
  if (rc <= 0) { if (rc < 0) return NULL; Py_RETURN_NONE; }
  for (Py_ssize_t k = 0; k < nl; ++k) {
    PyObject* v = PyTuple_GET_ITEM(leaves, k);
    if ((PyObject*)Py_TYPE(v) != T_Dense) Py_RETURN_NONE;
    long long dev, code, n, ptr;
    if (long_attr(v, s_dev, &dev) < 0 || long_attr(v, s_code, &code) < 0 ||
        long_attr(v, s_n, &n) < 0 || long_attr(v, s_ptr, &ptr) < 0)
      return NULL;
    if (dev != w.dev || code != w.code || n != w.n) Py_RETURN_NONE;
    w.ptrs[k] = (void*)(intptr_t)ptr;
  }
  w.nvec = (int)nl;
  if (alpha != Py_None) {
    /* Python floats, small ints and NumPy floating scalars only; anything
     * else (DeviceScalar, huge ints, arrays) takes the node path */
    double a;
    if (PyFloat_Check(alpha)) {
      a = PyFloat_AS_DOUBLE(alpha);
    } else if (PyLong_Check(alpha)) {
      long long i = PyLong_AsLongLong(alpha);
      if (i == -1 && PyErr_Occurred()) { PyErr_Clear(); Py_RETURN_NONE; }
      if (i > (1LL << 53) || i < -(1LL << 53)) Py_RETURN_NONE;
      a = (double)i;
    } else if ((PyObject*)Py_TYPE(alpha) == np_f64 || (PyObject*)Py_TYPE(alpha) == np_f32) {
      a = PyFloat_AsDouble(alpha);
      if (a == -1.0 && PyErr_Occurred()) return NULL;
    } else {
      Py_RETURN_NONE;
    }
    if (w.code == 0) a = (double)(float)a; /* round to the element type (ScaleNode) */
    w.sc[0] = a;
    w.nsc = 1;
  }
  void* stream;
  rc = stream_for(&w, &stream);
  if (rc <= 0) { if (rc < 0) return NULL; Py_RETURN_NONE; }
  size_t len = strlen(sig);
  if (len >= MAX_SIG) Py_RETURN_NONE;
  memcpy(w.sig, sig, len + 1);
  w.len = (int)len;
  if (dest != Py_None) {
    if (w.n == 0) Py_RETURN_TRUE;
    return check(p_assign(w.code, w.sig, dptr, (const void* const*)w.ptrs, w.nvec, w.sc, w.nsc,
                          w.n, stream));
  }
  void *ws, *slot;
  if (workspace(&w, stream, &ws, &slot) < 0) return NULL;
  return launch_reduce(&w, NULL, NULL, 0, flags, lazy, ws, slot, stream);
}

/* ---- assign_batch(statements): lv.assign_batch's common case in C.
 * Every statement (dest, source) must be eligible for fp_assign (plain
 * device vectors on the current device, no device scalars); statements are
 * grouped by (element type, signature) and each group is ONE
 * salt_assign_batch call.  A destination used by another statement (as its
 * destination or a leaf) makes the whole batch ineligible, so the Python
 * path raises the error.  Returns the statement count, or None. */
typedef struct {
  int code, nl, nsc;
  char* sig;
  Py_ssize_t count, cap;
  void** dsts;
  void** leaves;   /* count x nl */
  double* sc;      /* count x nsc */
  int64_t* ns;
} Group;

static int ptr_cmp(const void* a, const void* b) {
  uintptr_t x = *(const uintptr_t*)a, y = *(const uintptr_t*)b;
  return x < y ? -1 : x > y;
}

static int group_push(Group* g, void* dptr, const Walk* w) {
  if (g->count == g->cap) {
    Py_ssize_t cap = g->cap ? 2 * g->cap : 16;
    void** d = PyMem_Realloc(g->dsts, cap * sizeof(void*));
    if (d) g->dsts = d;
    void** l = PyMem_Realloc(g->leaves, cap * (g->nl ? g->nl : 1) * sizeof(void*));
    if (l) g->leaves = l;
    double* c = PyMem_Realloc(g->sc, cap * (g->nsc ? g->nsc : 1) * sizeof(double));
    if (c) g->sc = c;
    int64_t* n = PyMem_Realloc(g->ns, cap * sizeof(int64_t));
    if (n) g->ns = n;
    if (!d || !l || !c || !n) { PyErr_NoMemory(); return -1; }
    g->cap = cap;
  }
  g->dsts[g->count] = dptr;
  for (int k = 0; k < g->nl; ++k) g->leaves[g->count * g->nl + k] = w->ptrs[k];
  for (int k = 0; k < g->nsc; ++k) g->sc[g->count * g->nsc + k] = w->sc[k];
  g->ns[g->count] = (int64_t)w->n;
  ++g->count;
  return 1;
}

static void groups_free(Group* gs, int ng) {
  for (int i = 0; i < ng; ++i) {
    PyMem_Free(gs[i].sig);
    PyMem_Free(gs[i].dsts);
    PyMem_Free(gs[i].leaves);
    PyMem_Free(gs[i].sc);
    PyMem_Free(gs[i].ns);
  }
  PyMem_Free(gs);
}

static PyObject* fp_assign_batch(PyObject* self, PyObject* args) {
  PyObject* list;
  if (!PyArg_ParseTuple(args, "O!", &PyList_Type, &list)) return NULL;
  if (!p_assign_batch) Py_RETURN_NONE;
  const Py_ssize_t m = PyList_GET_SIZE(list);
  if (m == 0) return PyLong_FromLong(0);
  Group* gs = NULL;
  int ng = 0, capg = 0, dev = -1;
  uintptr_t* dests = PyMem_Malloc(m * sizeof(uintptr_t));
  if (!dests) return PyErr_NoMemory();
  PyObject* result = NULL;
  int eligible = 1;
  Py_ssize_t empties = 0;
  Walk w;
  /* pass 1: walk every statement, collect destinations */
  for (Py_ssize_t i = 0; i < m && eligible; ++i) {
    PyObject* st = PyList_GET_ITEM(list, i);
    if (!PyTuple_Check(st) || PyTuple_GET_SIZE(st) != 2) { eligible = 0; break; }
    void* dptr;
    int rc = start(&w, PyTuple_GET_ITEM(st, 0), &dptr);
    if (rc > 0) rc = walk(&w, PyTuple_GET_ITEM(st, 1));
    if (rc < 0) goto done;
    if (rc == 0 || w.nps || w.nvec == 0 || (dev >= 0 && w.dev != dev)) { eligible = 0; break; }
    dev = w.dev;
    dests[i] = w.n ? (uintptr_t)dptr : 0; /* empty statements write nothing */
  }
  if (eligible) {  /* no destination shared with another statement */
    uintptr_t* sorted = PyMem_Malloc(m * sizeof(uintptr_t));
    if (!sorted) { PyErr_NoMemory(); goto done; }
    memcpy(sorted, dests, m * sizeof(uintptr_t));
    qsort(sorted, (size_t)m, sizeof(uintptr_t), ptr_cmp);
    for (Py_ssize_t i = 1; i < m; ++i)
      if (sorted[i] && sorted[i] == sorted[i - 1]) eligible = 0;
    /* pass 2: leaves vs other statements' destinations, and grouping */
    for (Py_ssize_t i = 0; i < m && eligible; ++i) {
      PyObject* st = PyList_GET_ITEM(list, i);
      void* dptr;
      int rc = start(&w, PyTuple_GET_ITEM(st, 0), &dptr);
      if (rc > 0) rc = walk(&w, PyTuple_GET_ITEM(st, 1));
      if (rc <= 0) { eligible = 0; if (rc < 0) { PyMem_Free(sorted); goto done; } break; }
      for (int k = 0; k < w.nvec && eligible; ++k) {
        uintptr_t p = (uintptr_t)w.ptrs[k];
        if (p != dests[i] && w.n > 0 &&
            bsearch(&p, sorted, (size_t)m, sizeof(uintptr_t), ptr_cmp))
          eligible = 0;
      }
      if (!eligible) continue;
      if (w.n == 0) { ++empties; continue; }
      int gi = 0;
      for (; gi < ng; ++gi)
        if (gs[gi].code == w.code && gs[gi].nl == w.nvec && gs[gi].nsc == w.nsc &&
            strcmp(gs[gi].sig, w.sig) == 0)
          break;
      if (gi == ng) {
        if (ng == capg) {
          int cap = capg ? 2 * capg : 4;
          Group* n = PyMem_Realloc(gs, cap * sizeof(Group));
          if (!n) { PyErr_NoMemory(); PyMem_Free(sorted); goto done; }
          gs = n;
          capg = cap;
        }
        memset(&gs[ng], 0, sizeof(Group));
        gs[ng].code = w.code;
        gs[ng].nl = w.nvec;
        gs[ng].nsc = w.nsc;
        gs[ng].sig = PyMem_Malloc((size_t)w.len + 1);
        if (!gs[ng].sig) { PyErr_NoMemory(); PyMem_Free(sorted); goto done; }
        memcpy(gs[ng].sig, w.sig, (size_t)w.len + 1);
        ++ng;
      }
      if (group_push(&gs[gi], dptr, &w) < 0) { PyMem_Free(sorted); goto done; }
    }
    PyMem_Free(sorted);
  }
  if (!eligible) {
    Py_INCREF(Py_None);
    result = Py_None;
    goto done;
  }
  {
    void* stream;
    w.dev = dev;
    int rc = stream_for(&w, &stream);
    if (rc < 0) goto done;
    if (rc == 0) { Py_INCREF(Py_None); result = Py_None; goto done; }
    Py_ssize_t launched = empties;
    for (int gi = 0; gi < ng; ++gi) {
      Group* g = &gs[gi];
      int e = p_assign_batch(g->code, g->sig, (int)g->count, g->dsts, (const void* const*)g->leaves,
                             g->nl, g->sc, g->nsc, g->ns, stream);
      if (e != 0) {
        PyErr_Format(PyExc_RuntimeError, "libsalt error %d: %s", e, p_last_error());
        goto done;
      }
      launched += g->count;
    }
    result = PyLong_FromSsize_t(launched);
  }
done:
  PyMem_Free(dests);
  groups_free(gs, ng);
  return result;
}

/* Walk one reduction child: the first leaf fixes device / dtype / length
 * (as fp_reduce).  1 ok, 0 not eligible, -1 error. */
static int walk_child(Walk* w, PyObject* child) {
  memset(w, 0, sizeof *w);
  PyObject* first = child;
  while ((PyObject*)Py_TYPE(first) != T_Leaf && (PyObject*)Py_TYPE(first) != T_Dense) {
    PyObject* t = (PyObject*)Py_TYPE(first);
    if (t != T_Scale && t != T_Add && t != T_Sub && t != T_Mul) return 0;
    PyObject* nxt = PyObject_GetAttr(first, t == T_Scale ? s_child : s_left);
    if (!nxt) { PyErr_Clear(); return 0; }
    Py_DECREF(nxt); /* nodes are kept alive by their parents */
    first = nxt;
  }
  PyObject* v0 = (PyObject*)Py_TYPE(first) == T_Leaf ? PyObject_GetAttr(first, s_vector) : (Py_INCREF(first), first);
  if (!v0) return -1;
  int rc = start(w, v0, NULL);
  Py_DECREF(v0);
  if (rc <= 0) return rc;
  return walk(w, child);
}

/* reduce_batch([child, ...], flags) -> (out_tensor, [slot index per child])
 * or None: lv.reduce_batch's common case in C — every child eligible for
 * fp_reduce and on the current device, no device scalars; grouped by
 * (element type, signature), one salt_reduce_batch call per group, result
 * q in 16-byte slot q of out_tensor (element type at its start). */
static PyObject* fp_reduce_batch(PyObject* self, PyObject* args) {
  PyObject* list;
  int flags;
  if (!PyArg_ParseTuple(args, "O!i", &PyList_Type, &list, &flags)) return NULL;
  if (!p_reduce_batch || !batch_out) Py_RETURN_NONE;
  const Py_ssize_t m = PyList_GET_SIZE(list);
  if (m == 0) Py_RETURN_NONE;
  Group* gs = NULL;
  int ng = 0, capg = 0, dev = -1;
  int* gid = PyMem_Malloc(m * sizeof(int));
  Py_ssize_t* pos = PyMem_Malloc(m * sizeof(Py_ssize_t));
  PyObject *result = NULL, *out = NULL, *slots = NULL;
  if (!gid || !pos) { PyErr_NoMemory(); goto done; }
  Walk w;
  for (Py_ssize_t i = 0; i < m; ++i) {
    int rc = walk_child(&w, PyList_GET_ITEM(list, i));
    if (rc < 0) goto done;
    if (rc == 0 || w.nps || w.nvec == 0 || (dev >= 0 && w.dev != dev)) { Py_INCREF(Py_None); result = Py_None; goto done; }
    dev = w.dev;
    int g = 0;
    for (; g < ng; ++g)
      if (gs[g].code == w.code && gs[g].nl == w.nvec && gs[g].nsc == w.nsc && strcmp(gs[g].sig, w.sig) == 0)
        break;
    if (g == ng) {
      if (ng == capg) {
        int cap = capg ? 2 * capg : 4;
        Group* n = PyMem_Realloc(gs, cap * sizeof(Group));
        if (!n) { PyErr_NoMemory(); goto done; }
        gs = n;
        capg = cap;
      }
      memset(&gs[ng], 0, sizeof(Group));
      gs[ng].code = w.code;
      gs[ng].nl = w.nvec;
      gs[ng].nsc = w.nsc;
      gs[ng].sig = PyMem_Malloc((size_t)w.len + 1);
      if (!gs[ng].sig) { PyErr_NoMemory(); goto done; }
      memcpy(gs[ng].sig, w.sig, (size_t)w.len + 1);
      ++ng;
    }
    gid[i] = g;
    pos[i] = gs[g].count;
    if (group_push(&gs[g], NULL, &w) < 0) goto done;
  }
  {
    void* stream;
    w.dev = dev;
    int rc = stream_for(&w, &stream);
    if (rc < 0) goto done;
    if (rc == 0) { Py_INCREF(Py_None); result = Py_None; goto done; }
    PyObject* r = PyObject_CallFunction(batch_out, "in", dev, m);
    if (!r) goto done;
    out = PyTuple_GetItem(r, 0);
    void* base = PyLong_AsVoidPtr(PyTuple_GetItem(r, 1));
    Py_XINCREF(out);
    Py_DECREF(r);
    if (!out || PyErr_Occurred()) goto done;
    void *ws, *slot;
    if (workspace(&w, stream, &ws, &slot) < 0) goto done;
    /* slot of child i: groups are laid out one after another */
    Py_ssize_t off = 0;
    for (int g = 0; g < ng; ++g) {
      for (Py_ssize_t q = 0; q < gs[g].count; ++q) gs[g].dsts[q] = (char*)base + 16 * (off + q);
      int e = p_reduce_batch(gs[g].code, gs[g].sig, (int)gs[g].count, (const void* const*)gs[g].leaves,
                             gs[g].nl, gs[g].sc, gs[g].nsc, gs[g].ns, flags, gs[g].dsts, ws, ws_bytes,
                             stream);
      if (e != 0) {
        PyErr_Format(PyExc_RuntimeError, "libsalt error %d: %s", e, p_last_error());
        goto done;
      }
      gs[g].cap = off; /* reuse: group start slot */
      off += gs[g].count;
    }
    slots = PyList_New(m);
    if (!slots) goto done;
    for (Py_ssize_t i = 0; i < m; ++i) {
      PyObject* v = PyLong_FromSsize_t(gs[gid[i]].cap + pos[i]);
      if (!v) goto done;
      PyList_SET_ITEM(slots, i, v);
    }
    result = PyTuple_Pack(2, out, slots);
  }
done:
  Py_XDECREF(out);
  Py_XDECREF(slots);
  PyMem_Free(gid);
  PyMem_Free(pos);
  groups_free(gs, ng);
  return result;
}

static PyObject* fp_init(PyObject* self, PyObject* args) {
  unsigned long long a, r, ar, fu, le, ab, rb, re, ss, fp, rs;
  Py_ssize_t wsb;
  if (!PyArg_ParseTuple(args, "KKKKKnOOOOOOOOOOOOOKKOKKKK", &a, &r, &ar, &fu, &le, &wsb, &T_Leaf, &T_Add,
                        &T_Sub, &T_Mul, &T_Scale, &T_Dense, &T_DevScalar, &get_stream,
                        &current_device, &workspace_fn, &np_f32, &np_f64, &lazy_out, &ab, &rb,
                        &batch_out, &re, &ss, &fp, &rs))
    return NULL;
  p_fused_prog = (fused_prog_fn)(uintptr_t)fp;
  p_result_slot = (result_slot_fn)(uintptr_t)rs;
  p_result_enqueue = (result_enqueue_fn)(uintptr_t)re;
  p_stream_sync = (stream_sync_fn)(uintptr_t)ss;
  p_assign_batch = (assign_batch_fn)(uintptr_t)ab;
  p_reduce_batch = (reduce_batch_fn)(uintptr_t)rb;
  Py_INCREF(batch_out);
  PyObject* keep[] = {T_Leaf, T_Add, T_Sub, T_Mul, T_Scale, T_Dense, T_DevScalar, get_stream,
                      current_device, workspace_fn, np_f32, np_f64, lazy_out};
  for (size_t i = 0; i < sizeof keep / sizeof keep[0]; ++i) Py_INCREF(keep[i]);
  p_assign = (assign_fn)(uintptr_t)a;
  p_reduce = (reduce_fn)(uintptr_t)r;
  p_assign_reduce = (assign_reduce_fn)(uintptr_t)ar;
  p_fused = (fused_fn)(uintptr_t)fu;
  p_last_error = (last_error_fn)(uintptr_t)le;
  ws_bytes = (size_t)wsb;
  Py_RETURN_NONE;
}

static PyMethodDef methods[] = {
    {"init", fp_init, METH_VARARGS, "bind libsalt entry points and the Python types"},
    {"assign", fp_assign, METH_VARARGS, "assign(dest, source) -> bool"},
    {"reduce", fp_reduce, METH_VARARGS, "reduce(child, flags, lazy=False) -> scalar or None"},
    {"assign_reduce", fp_assign_reduce, METH_VARARGS,
     "assign_reduce(dest, source, child, flags, lazy=False) -> scalar or None"},
    {"op", fp_op, METH_VARARGS,
     "op(sig, dest_or_None, leaves, alpha_or_None, flags, lazy=False) -> True / result, or None"},
    {"assign_batch", fp_assign_batch, METH_VARARGS,
     "assign_batch([(dest, source), ...]) -> statements launched, or None"},
    {"reduce_batch", fp_reduce_batch, METH_VARARGS,
     "reduce_batch([child, ...], flags) -> (out_tensor, slots), or None"},
    {"fused", fp_fused, METH_VARARGS,
     "fused(((dest, source), ...), total_child_or_None, flags, lazy=False) -> (result,) or None"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_fastpath", NULL, -1, methods};

PyMODINIT_FUNC PyInit__fastpath(void) {
  s_vector = PyUnicode_InternFromString("vector");
  s_left = PyUnicode_InternFromString("left");
  s_right = PyUnicode_InternFromString("right");
  s_child = PyUnicode_InternFromString("child");
  s_alpha = PyUnicode_InternFromString("alpha");
  s_ptr = PyUnicode_InternFromString("_ptr");
  s_dev = PyUnicode_InternFromString("_dev");
  s_n = PyUnicode_InternFromString("_n");
  s_code = PyUnicode_InternFromString("_code");
  s_data_ptr = PyUnicode_InternFromString("data_ptr");
  s_tensor = PyUnicode_InternFromString("_tensor");
  s_expr = PyUnicode_InternFromString("_expr");
  s_check_operands = PyUnicode_InternFromString("check_operands");
  s_get_device = PyUnicode_InternFromString("get_device");
  return PyModule_Create(&module);
}

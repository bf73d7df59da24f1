/*
 * pyfast.c -- CPython binding of the per-request calls of include/mempool.h
 * (alloc_mem / free_mem, insert / match / unpin / delete, transfer /
 * transfer_with_insert, stream ordering).  Argument marshalling only: every
 * function converts its array arguments with the numpy C API (no copy when
 * the caller already passes contiguous arrays of the right dtype), calls the
 * C-ABI entry point of the same name and wraps the outputs.  It exists because
 * ctypes marshalling costs several microseconds per call, which is most of a
 * small request's host time (profiles/README.md, ReAct-like workload); the
 * setup, debug and measurement entry points stay on ctypes (mempool.py).
 *
 * Pool handles travel as Python ints (the mp_pool* value).  A non-zero
 * mp_status raises the exception built by the factory registered with
 * set_error_factory(status, where) (mempool.MempoolError).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_2_0_API_VERSION
#include <numpy/arrayobject.h>

#include "mempool.h"

static PyObject* g_err_factory = NULL;

static PyObject* raise_status(int st, const char* where) {
  if (!g_err_factory) {
    PyErr_Format(PyExc_RuntimeError, "%s: mp_status %d", where, st);
    return NULL;
  }
  PyObject* exc = PyObject_CallFunction(g_err_factory, "is", st, where);
  if (!exc) return NULL;
  PyErr_SetObject((PyObject*)Py_TYPE(exc), exc);
  Py_DECREF(exc);
  return NULL;
}

#define CHECK(st, where)                              \
  do {                                                \
    if ((st) != MP_OK) return raise_status(st, where); \
  } while (0)

/* obj -> C-contiguous array of `type` (any shape, read flat), new reference. */
static PyArrayObject* as_flat(PyObject* obj, int type) {
  return (PyArrayObject*)PyArray_FROMANY(obj, type, 0, 0,
                                         NPY_ARRAY_IN_ARRAY | NPY_ARRAY_FORCECAST);
}

static PyArrayObject* new_u64(npy_intp n) {
  return (PyArrayObject*)PyArray_SimpleNew(1, &n, NPY_UINT64);
}

/* Not an int: NULL, which every entry point rejects with MP_ERR_CONFIG. */
static mp_pool* handle(PyObject* o) {
  void* p = PyLong_AsVoidPtr(o);
  if (!p && PyErr_Occurred()) PyErr_Clear();
  return (mp_pool*)p;
}

static PyObject* py_set_error_factory(PyObject* self, PyObject* f) {
  Py_XINCREF(f);
  Py_XSETREF(g_err_factory, f);
  Py_RETURN_NONE;
}

/* alloc_mem(h, n, type, requester) -> uint64[n] */
static PyObject* py_alloc_mem(PyObject* self, PyObject* args) {
  PyObject* h;
  long long n;
  int type, req;
  if (!PyArg_ParseTuple(args, "OLii", &h, &n, &type, &req)) return NULL;
  PyArrayObject* out = new_u64(n > 0 ? (npy_intp)n : 0);
  if (!out) return NULL;
  int st;
  mp_pool* p = handle(h);  /* with the GIL held */
  Py_BEGIN_ALLOW_THREADS
  st = mp_alloc_mem(p, n, type, req, (mp_addr*)PyArray_DATA(out));
  Py_END_ALLOW_THREADS
  if (st != MP_OK) {
    Py_DECREF(out);
    return raise_status(st, "alloc_mem");
  }
  return (PyObject*)out;
}

/* free_mem(h, addrs) / unpin(h, addrs) */
static PyObject* addr_list_call(PyObject* args, mp_status (*fn)(mp_pool*, const mp_addr*, int64_t),
                                const char* where) {
  PyObject *h, *a;
  if (!PyArg_ParseTuple(args, "OO", &h, &a)) return NULL;
  PyArrayObject* arr = as_flat(a, NPY_UINT64);
  if (!arr) return NULL;
  const int st = fn(handle(h), (const mp_addr*)PyArray_DATA(arr), (int64_t)PyArray_SIZE(arr));
  Py_DECREF(arr);
  CHECK(st, where);
  Py_RETURN_NONE;
}

static PyObject* py_free_mem(PyObject* self, PyObject* args) {
  return addr_list_call(args, mp_free_mem, "free_mem");
}

static PyObject* py_unpin(PyObject* self, PyObject* args) {
  return addr_list_call(args, mp_unpin, "unpin");
}

/* insert(h, tokens, addrs, flags) -> n_dup_freed */
static PyObject* py_insert(PyObject* self, PyObject* args) {
  PyObject *h, *t, *a;
  unsigned int flags;
  if (!PyArg_ParseTuple(args, "OOOI", &h, &t, &a, &flags)) return NULL;
  PyArrayObject* ta = as_flat(t, NPY_INT32);
  if (!ta) return NULL;
  PyArrayObject* aa = as_flat(a, NPY_UINT64);
  if (!aa) {
    Py_DECREF(ta);
    return NULL;
  }
  int64_t dup = 0;
  const int st = mp_insert(handle(h), (const mp_token*)PyArray_DATA(ta), (int64_t)PyArray_SIZE(ta),
                           (const mp_addr*)PyArray_DATA(aa), (int64_t)PyArray_SIZE(aa), flags,
                           &dup);
  Py_DECREF(ta);
  Py_DECREF(aa);
  CHECK(st, "insert");
  return PyLong_FromLongLong(dup);
}

/* match(h, tokens, flags, B) -> (matched_tokens, uint64[matched_tokens / B]) */
static PyObject* py_match(PyObject* self, PyObject* args) {
  PyObject *h, *t;
  unsigned int flags;
  int B;
  if (!PyArg_ParseTuple(args, "OOIi", &h, &t, &flags, &B)) return NULL;
  if (B <= 0) return raise_status(MP_ERR_CONFIG, "match"); /* block size sizes the output */
  PyArrayObject* ta = as_flat(t, NPY_INT32);
  if (!ta) return NULL;
  const int64_t nt = (int64_t)PyArray_SIZE(ta);
  const int64_t cap = nt / B;
  mp_addr small[256];
  mp_addr* buf = cap <= 256 ? small : (mp_addr*)PyMem_Malloc((size_t)cap * sizeof(mp_addr));
  if (!buf) {
    Py_DECREF(ta);
    return PyErr_NoMemory();
  }
  int64_t mt = 0;
  const int st = mp_match(handle(h), (const mp_token*)PyArray_DATA(ta), nt, flags, buf,
                          cap > 0 ? cap : 1, &mt);
  Py_DECREF(ta);
  PyArrayObject* out = NULL;
  if (st == MP_OK) {
    out = new_u64((npy_intp)(mt / B));
    if (out) memcpy(PyArray_DATA(out), buf, (size_t)(mt / B) * sizeof(mp_addr));
  }
  if (buf != small) PyMem_Free(buf);
  CHECK(st, "match");
  if (!out) return NULL;
  return Py_BuildValue("(LN)", (long long)mt, out);
}

/* delete(h, tokens) */
static PyObject* py_delete(PyObject* self, PyObject* args) {
  PyObject *h, *t;
  if (!PyArg_ParseTuple(args, "OO", &h, &t)) return NULL;
  PyArrayObject* ta = as_flat(t, NPY_INT32);
  if (!ta) return NULL;
  const int st = mp_delete(handle(h), (const mp_token*)PyArray_DATA(ta), (int64_t)PyArray_SIZE(ta));
  Py_DECREF(ta);
  CHECK(st, "delete");
  Py_RETURN_NONE;
}

/* priv: None or a bytes-like object */
static int get_priv(PyObject* priv, Py_buffer* view) {
  if (priv == Py_None) {
    view->obj = NULL;
    view->buf = NULL;
    view->len = 0;
    return 0;
  }
  return PyObject_GetBuffer(priv, view, PyBUF_SIMPLE);
}

/* transfer(h, dst_inst, src_addrs, dst_addrs_or_None, flags, layer_begin, layer_end, priv)
 * -> uint64[n] (the destination addrs; a copy of the given ones with DST_GIVEN) */
static PyObject* py_transfer(PyObject* self, PyObject* args) {
  PyObject *h, *s, *d, *priv;
  int dst_inst, lb, le;
  unsigned int flags;
  if (!PyArg_ParseTuple(args, "OiOOIiiO", &h, &dst_inst, &s, &d, &flags, &lb, &le, &priv))
    return NULL;
  PyArrayObject* sa = as_flat(s, NPY_UINT64);
  if (!sa) return NULL;
  const npy_intp n = PyArray_SIZE(sa);
  PyArrayObject* out = new_u64(n);
  if (!out) {
    Py_DECREF(sa);
    return NULL;
  }
  if (d != Py_None) {
    PyArrayObject* da = as_flat(d, NPY_UINT64);
    if (!da) {
      Py_DECREF(sa);
      Py_DECREF(out);
      return NULL;
    }
    /* a given list must name exactly one destination per source block */
    if (PyArray_SIZE(da) != n) {
      Py_DECREF(da);
      Py_DECREF(sa);
      Py_DECREF(out);
      return raise_status(MP_ERR_ADDR_COUNT, "transfer");
    }
    memcpy(PyArray_DATA(out), PyArray_DATA(da), (size_t)n * sizeof(mp_addr));
    Py_DECREF(da);
    flags |= MP_XFER_DST_GIVEN;
  } else {
    flags &= ~MP_XFER_DST_GIVEN; /* no list given: the receiver allocates */
  }
  Py_buffer pv;
  if (get_priv(priv, &pv) < 0) {
    Py_DECREF(sa);
    Py_DECREF(out);
    return NULL;
  }
  const int st = mp_transfer(handle(h), dst_inst, (const mp_addr*)PyArray_DATA(sa), (int64_t)n,
                             (mp_addr*)PyArray_DATA(out), flags, lb, le, pv.len ? pv.buf : NULL,
                             (int64_t)pv.len);
  if (pv.obj) PyBuffer_Release(&pv);
  Py_DECREF(sa);
  if (st != MP_OK) {
    Py_DECREF(out);
    return raise_status(st, "transfer");
  }
  return (PyObject*)out;
}

/* transfer_with_insert(h, dst_inst, tokens, src_addrs, dst_addrs_or_None, flags, priv, B)
 * -> (uint64[ceil(n_tok / B)], n_moved) */
static PyObject* py_transfer_with_insert(PyObject* self, PyObject* args) {
  PyObject *h, *t, *s, *d, *priv;
  int dst_inst, B;
  unsigned int flags;
  if (!PyArg_ParseTuple(args, "OiOOOIOi", &h, &dst_inst, &t, &s, &d, &flags, &priv, &B))
    return NULL;
  if (B <= 0) return raise_status(MP_ERR_CONFIG, "transfer_with_insert");
  PyArrayObject* ta = as_flat(t, NPY_INT32);
  if (!ta) return NULL;
  PyArrayObject* sa = as_flat(s, NPY_UINT64);
  if (!sa) {
    Py_DECREF(ta);
    return NULL;
  }
  const int64_t nt = (int64_t)PyArray_SIZE(ta);
  const npy_intp ceil_b = (npy_intp)((nt + B - 1) / B);
  npy_intp cap = ceil_b > 0 ? ceil_b : 1;
  PyArrayObject* da = NULL;
  if (d != Py_None) {
    da = as_flat(d, NPY_UINT64);
    if (!da) {
      Py_DECREF(ta);
      Py_DECREF(sa);
      return NULL;
    }
    if (PyArray_SIZE(da) != PyArray_SIZE(sa)) { /* one given destination per source block */
      Py_DECREF(ta);
      Py_DECREF(sa);
      Py_DECREF(da);
      return raise_status(MP_ERR_ADDR_COUNT, "transfer_with_insert");
    }
    if (PyArray_SIZE(da) > cap) cap = PyArray_SIZE(da);
    flags |= MP_XFER_DST_GIVEN;
  } else {
    flags &= ~MP_XFER_DST_GIVEN; /* no list given: the receiver allocates */
  }
  PyArrayObject* out = new_u64(cap);
  if (!out) {
    Py_DECREF(ta);
    Py_DECREF(sa);
    Py_XDECREF(da);
    return NULL;
  }
  if (da) {
    memset(PyArray_DATA(out), 0, (size_t)cap * sizeof(mp_addr));
    memcpy(PyArray_DATA(out), PyArray_DATA(da), (size_t)PyArray_SIZE(da) * sizeof(mp_addr));
    Py_DECREF(da);
  }
  Py_buffer pv;
  if (get_priv(priv, &pv) < 0) {
    Py_DECREF(ta);
    Py_DECREF(sa);
    Py_DECREF(out);
    return NULL;
  }
  int64_t moved = 0;
  const int st = mp_transfer_with_insert(
      handle(h), dst_inst, (const mp_token*)PyArray_DATA(ta), nt, (const mp_addr*)PyArray_DATA(sa),
      (int64_t)PyArray_SIZE(sa), (mp_addr*)PyArray_DATA(out), flags, pv.len ? pv.buf : NULL,
      (int64_t)pv.len, &moved);
  if (pv.obj) PyBuffer_Release(&pv);
  Py_DECREF(ta);
  Py_DECREF(sa);
  if (st != MP_OK) {
    Py_DECREF(out);
    return raise_status(st, "transfer_with_insert");
  }
  if (cap != ceil_b) { /* given dst list longer than the token blocks: return ceil_b entries */
    PyObject* v = PySequence_GetSlice((PyObject*)out, 0, ceil_b);
    Py_DECREF(out);
    if (!v) return NULL;
    return Py_BuildValue("(NL)", v, (long long)moved);
  }
  return Py_BuildValue("(NL)", (PyObject*)out, (long long)moved);
}

/* record_event(h, cudaEvent_t as int) / wait_event(h, ...) */
static PyObject* event_call(PyObject* args, mp_status (*fn)(mp_pool*, void*), const char* where) {
  PyObject *h, *e;
  if (!PyArg_ParseTuple(args, "OO", &h, &e)) return NULL;
  void* ev = PyLong_AsVoidPtr(e);
  if (PyErr_Occurred()) return NULL;
  const int st = fn(handle(h), ev);
  CHECK(st, where);
  Py_RETURN_NONE;
}

static PyObject* py_record_event(PyObject* self, PyObject* args) {
  return event_call(args, mp_record_event, "record_event");
}

static PyObject* py_wait_event(PyObject* self, PyObject* args) {
  return event_call(args, mp_wait_event, "wait_event");
}

/* recv_poll(h) -> (kind, src_instance, private bytes, addrs uint64[]) or None:
 * the size query and the pop in one call from Python. */
static PyObject* py_recv_poll(PyObject* self, PyObject* h) {
  mp_pool* p = handle(h);
  mp_recv_msg m;
  int st = mp_recv_poll(p, &m, NULL, 0, NULL, 0);
  if (st == MP_ERR_PRECONDITION) Py_RETURN_NONE;  /* nothing queued */
  if (st != MP_OK && st != MP_ERR_BUFFER_TOO_SMALL) return raise_status(st, "recv_poll");
  PyObject* pb = PyBytes_FromStringAndSize(NULL, (Py_ssize_t)m.priv_len);
  if (!pb) return NULL;
  npy_intp dims[1] = {(npy_intp)m.n_addrs};
  PyObject* ad = PyArray_SimpleNew(1, dims, NPY_UINT64);
  if (!ad) {
    Py_DECREF(pb);
    return NULL;
  }
  if (st == MP_ERR_BUFFER_TOO_SMALL) {  /* kept: pop it into the sized buffers */
    st = mp_recv_poll(p, &m, PyBytes_AS_STRING(pb), m.priv_len,
                      (mp_addr*)PyArray_DATA((PyArrayObject*)ad), m.n_addrs);
    if (st != MP_OK) {
      Py_DECREF(pb);
      Py_DECREF(ad);
      return raise_status(st, "recv_poll");
    }
  }  /* else: an empty message (no private bytes, no addrs) was popped already */
  return Py_BuildValue("(iiNN)", (int)m.kind, (int)m.src_instance, pb, ad);
}

/* sync(h) */
static PyObject* py_sync(PyObject* self, PyObject* h) {
  int st;
  mp_pool* p = handle(h);
  Py_BEGIN_ALLOW_THREADS
  st = mp_sync(p);
  Py_END_ALLOW_THREADS
  CHECK(st, "sync");
  Py_RETURN_NONE;
}

static PyMethodDef methods[] = {
    {"set_error_factory", py_set_error_factory, METH_O, "factory(status, where) -> exception"},
    {"alloc_mem", py_alloc_mem, METH_VARARGS, "mp_alloc_mem"},
    {"free_mem", py_free_mem, METH_VARARGS, "mp_free_mem"},
    {"insert", py_insert, METH_VARARGS, "mp_insert"},
    {"match", py_match, METH_VARARGS, "mp_match"},
    {"unpin", py_unpin, METH_VARARGS, "mp_unpin"},
    {"delete", py_delete, METH_VARARGS, "mp_delete"},
    {"transfer", py_transfer, METH_VARARGS, "mp_transfer"},
    {"transfer_with_insert", py_transfer_with_insert, METH_VARARGS, "mp_transfer_with_insert"},
    {"record_event", py_record_event, METH_VARARGS, "mp_record_event"},
    {"wait_event", py_wait_event, METH_VARARGS, "mp_wait_event"},
    {"sync", py_sync, METH_O, "mp_sync"},
    {"recv_poll", py_recv_poll, METH_O, "mp_recv_poll"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_mpfast", NULL, -1, methods};

PyMODINIT_FUNC PyInit__mpfast(void) {
  import_array();
  return PyModule_Create(&module);
}

/*
 * _tmfast — host-side argument marshalling for the drop-in API (CPython extension).
 *
 * The reference's callers hand the trajectory manager Python lists of ints and SpanOrigin
 * enums (trie.py:120-126: lpm_insert(tokens, origins, versions)).  Before the C ABI can
 * take them they must become int32 buffers and (start, origin, version) runs
 * (trie.py:26-33).  Doing that with array.array / numpy costs ~20-30 ns per token, more
 * than the GPU path itself for short records; these loops read the list items directly.
 *
 *   pack_i32(seq)                      -> bytearray of int32 (ValueError outside int32)
 *   pack_lists(list_of_seqs, nthreads) -> (bytearray int32 tokens, bytearray int64 offsets[n+1])
 *                                         rows split over nthreads POSIX threads
 *   meta_runs(origins, versions, model_output)
 *                                      -> (bytearray int32 starts, bytearray uint8 origin codes,
 *                                          bytearray int32 versions): maximal runs of
 *                                          (origin == model_output, version)
 *
 * Worker threads never call into the interpreter: they read list items and the values of
 * compact ints (the caller holds the GIL for the whole call, so nothing can mutate the
 * lists meanwhile); anything else (large ints, non-int items) is left to the calling
 * thread, which converts it with the C API and raises the reference's ValueError.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>

/* value of a compact int (|v| < 2^30 on 64-bit CPython 3.12) without touching the error state */
static inline int compact_value(PyObject *o, int64_t *v) {
  if (!PyLong_CheckExact(o)) return 0;
  if (!PyUnstable_Long_IsCompact((PyLongObject *)o)) return 0;
  *v = (int64_t)PyUnstable_Long_CompactValue((PyLongObject *)o);
  return 1;
}

/* slow path, calling thread only: any int-like object -> int32 or ValueError */
static int to_i32(PyObject *o, int32_t *out) {
  int overflow = 0;
  long long v = PyLong_AsLongLongAndOverflow(o, &overflow);
  if (v == -1 && PyErr_Occurred()) return -1;
  if (overflow || v < INT32_MIN || v > INT32_MAX) {
    PyErr_SetString(PyExc_ValueError, "token ids must fit in int32");
    return -1;
  }
  *out = (int32_t)v;
  return 0;
}

static int fill_i32(PyObject **items, Py_ssize_t n, int32_t *dst) {
  for (Py_ssize_t i = 0; i < n; i++) {
    int64_t v;
    if (compact_value(items[i], &v)) {
      dst[i] = (int32_t)v;  /* compact ints always fit */
    } else if (to_i32(items[i], dst + i) < 0) {
      return -1;
    }
  }
  return 0;
}

static PyObject *pack_i32(PyObject *self, PyObject *args) {
  PyObject *seq;
  if (!PyArg_ParseTuple(args, "O", &seq)) return NULL;
  PyObject *fast = PySequence_Fast(seq, "tokens must be a sequence");
  if (!fast) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  PyObject *out = PyByteArray_FromStringAndSize(NULL, 4 * n);
  if (!out) {
    Py_DECREF(fast);
    return NULL;
  }
  if (fill_i32(PySequence_Fast_ITEMS(fast), n, (int32_t *)PyByteArray_AS_STRING(out)) < 0) {
    Py_DECREF(fast);
    Py_DECREF(out);
    return NULL;
  }
  Py_DECREF(fast);
  return out;
}

typedef struct {
  PyObject **fast;       /* PySequence_Fast of every row */
  const int64_t *off;
  int32_t *dst;
  Py_ssize_t r0, r1;
  Py_ssize_t bad_row;    /* first row this worker could not convert (-1: none) */
} PackJob;

static void *pack_worker(void *arg) {
  PackJob *j = (PackJob *)arg;
  j->bad_row = -1;
  for (Py_ssize_t r = j->r0; r < j->r1; r++) {
    PyObject **items = PySequence_Fast_ITEMS(j->fast[r]);
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(j->fast[r]);
    int32_t *d = j->dst + j->off[r];
    for (Py_ssize_t i = 0; i < n; i++) {
      int64_t v;
      if (!compact_value(items[i], &v)) {
        if (j->bad_row < 0) j->bad_row = r;
        break;
      }
      d[i] = (int32_t)v;
    }
  }
  return NULL;
}

static PyObject *pack_lists(PyObject *self, PyObject *args) {
  PyObject *rows;
  int nthreads = 1;
  if (!PyArg_ParseTuple(args, "O|i", &rows, &nthreads)) return NULL;
  PyObject *outer = PySequence_Fast(rows, "rows must be a sequence");
  if (!outer) return NULL;
  const Py_ssize_t nr = PySequence_Fast_GET_SIZE(outer);
  PyObject **fast = (PyObject **)PyMem_Calloc((size_t)(nr > 0 ? nr : 1), sizeof(PyObject *));
  PyObject *offs = PyByteArray_FromStringAndSize(NULL, 8 * (nr + 1));
  PyObject *toks = NULL;
  if (!fast || !offs) goto fail;
  int64_t *off = (int64_t *)PyByteArray_AS_STRING(offs);
  off[0] = 0;
  for (Py_ssize_t r = 0; r < nr; r++) {
    fast[r] = PySequence_Fast(PySequence_Fast_GET_ITEM(outer, r), "each row must be a sequence");
    if (!fast[r]) goto fail;
    off[r + 1] = off[r] + PySequence_Fast_GET_SIZE(fast[r]);
  }
  toks = PyByteArray_FromStringAndSize(NULL, 4 * (off[nr] > 0 ? off[nr] : 1));
  if (!toks) goto fail;
  int32_t *dst = (int32_t *)PyByteArray_AS_STRING(toks);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 64) nthreads = 64;
  if ((Py_ssize_t)nthreads > nr) nthreads = (int)(nr > 0 ? nr : 1);
  if (off[nr] < (1 << 16)) nthreads = 1;  /* small batches: thread start-up costs more */
  PackJob jobs[64];
  pthread_t th[64];
  /* split rows so every worker gets about the same number of tokens */
  Py_ssize_t r = 0;
  for (int t = 0; t < nthreads; t++) {
    const int64_t goal = off[nr] * (t + 1) / nthreads;
    jobs[t].fast = fast;
    jobs[t].off = off;
    jobs[t].dst = dst;
    jobs[t].r0 = r;
    while (r < nr && (off[r] < goal || t == nthreads - 1)) r++;
    jobs[t].r1 = r;
  }
  for (int t = 1; t < nthreads; t++)
    if (pthread_create(&th[t], NULL, pack_worker, &jobs[t]) != 0) {
      pack_worker(&jobs[t]);
      th[t] = 0;
    }
  pack_worker(&jobs[0]);
  for (int t = 1; t < nthreads; t++)
    if (th[t]) pthread_join(th[t], NULL);
  for (int t = 0; t < nthreads; t++)  /* rows with large ints / non-ints: the C API, here */
    for (Py_ssize_t rr = jobs[t].bad_row; rr >= 0 && rr < jobs[t].r1; rr++)
      if (fill_i32(PySequence_Fast_ITEMS(fast[rr]), PySequence_Fast_GET_SIZE(fast[rr]), dst + off[rr]) < 0) goto fail;
  for (Py_ssize_t k = 0; k < nr; k++) Py_XDECREF(fast[k]);
  PyMem_Free(fast);
  Py_DECREF(outer);
  return Py_BuildValue("(NN)", toks, offs);
fail:
  if (fast) {
    for (Py_ssize_t k = 0; k < nr; k++) Py_XDECREF(fast[k]);
    PyMem_Free(fast);
  }
  Py_XDECREF(toks);
  Py_XDECREF(offs);
  Py_DECREF(outer);
  return NULL;
}

/* origin code of one item: the reference enum member (identity), or 0/1/True/False,
 * or any object whose .value is "model_output" */
static int origin_code(PyObject *o, PyObject *model_output, PyObject *agent_input) {
  if (o == model_output) return 1;
  if (o == agent_input) return 0;
  if (o == Py_True) return 1;
  if (o == Py_False) return 0;
  int64_t v;
  if (compact_value(o, &v)) return v == 1;
  PyObject *val = PyObject_GetAttrString(o, "value");
  if (!val) {
    PyErr_Clear();
    return 0;
  }
  int r = PyUnicode_Check(val) && PyUnicode_CompareWithASCIIString(val, "model_output") == 0;
  Py_DECREF(val);
  return r;
}

static PyObject *meta_runs(PyObject *self, PyObject *args) {
  PyObject *origins, *versions, *model_output, *agent_input = Py_None;
  if (!PyArg_ParseTuple(args, "OOO|O", &origins, &versions, &model_output, &agent_input)) return NULL;
  PyObject *fo = PySequence_Fast(origins, "origins must be a sequence");
  if (!fo) return NULL;
  PyObject *fv = PySequence_Fast(versions, "versions must be a sequence");
  if (!fv) {
    Py_DECREF(fo);
    return NULL;
  }
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fo);
  PyObject *res = NULL, *bs = NULL, *bo = NULL, *bv = NULL;
  if (PySequence_Fast_GET_SIZE(fv) != n) {
    PyErr_SetString(PyExc_ValueError, "tokens, origins, versions must be parallel");
    goto done;
  }
  PyObject **oi = PySequence_Fast_ITEMS(fo), **vi = PySequence_Fast_ITEMS(fv);
  /* one pass: runs collected in a small growable buffer (a handful for real sequences),
   * items compared by identity first (a list of enum members or of one small int repeats
   * the same objects, so a run's interior is a pointer scan); then exact-size bytearrays */
  Py_ssize_t nr = 0, cap = 64;
  int32_t st_buf[64], vr_buf[64];
  uint8_t or_buf[64];
  int32_t *rs = st_buf, *rv = vr_buf;
  uint8_t *ro = or_buf;
  int heap = 0, failed = 0;
  {
    PyObject *a = NULL, *b = NULL;
    int po = -1;
    int32_t pv = 0;
    Py_ssize_t i = 0;
    while (i < n) {
      if (oi[i] == a && vi[i] == b) {  /* scan the rest of the run */
        while (i + 4 <= n && oi[i] == a && oi[i + 1] == a && oi[i + 2] == a && oi[i + 3] == a && vi[i] == b &&
               vi[i + 1] == b && vi[i + 2] == b && vi[i + 3] == b)
          i += 4;
        while (i < n && oi[i] == a && vi[i] == b) i++;
        continue;
      }
      const int o = origin_code(oi[i], model_output, agent_input);
      int64_t v;
      int32_t v32;
      if (compact_value(vi[i], &v)) v32 = (int32_t)v;
      else if (to_i32(vi[i], &v32) < 0) { failed = 1; break; }
      if (i == 0 || o != po || v32 != pv) {
        if (nr == cap) {  /* grow (rare): move to the heap */
          const Py_ssize_t nc = 2 * cap;
          int32_t *ns = (int32_t *)PyMem_Malloc(4 * nc), *nv = (int32_t *)PyMem_Malloc(4 * nc);
          uint8_t *no = (uint8_t *)PyMem_Malloc(nc);
          if (!ns || !nv || !no) {
            PyMem_Free(ns); PyMem_Free(nv); PyMem_Free(no);
            PyErr_NoMemory();
            failed = 1;
            break;
          }
          memcpy(ns, rs, 4 * nr); memcpy(nv, rv, 4 * nr); memcpy(no, ro, nr);
          if (heap) { PyMem_Free(rs); PyMem_Free(rv); PyMem_Free(ro); }
          rs = ns; rv = nv; ro = no;
          cap = nc;
          heap = 1;
        }
        rs[nr] = (int32_t)i;
        ro[nr] = (uint8_t)o;
        rv[nr] = v32;
        nr++;
      }
      po = o;
      pv = v32;
      a = oi[i];
      b = vi[i];
      i++;
    }
  }
  if (!failed) {
    bs = PyByteArray_FromStringAndSize((const char *)rs, 4 * nr);
    bo = PyByteArray_FromStringAndSize((const char *)ro, nr);
    bv = PyByteArray_FromStringAndSize((const char *)rv, 4 * nr);
  }
  if (heap) { PyMem_Free(rs); PyMem_Free(rv); PyMem_Free(ro); }
  if (failed || !bs || !bo || !bv) goto done;
  res = Py_BuildValue("(OOOn)", bs, bo, bv, nr);
done:
  Py_XDECREF(bs);
  Py_XDECREF(bo);
  Py_XDECREF(bv);
  Py_DECREF(fo);
  Py_DECREF(fv);
  return res;
}

static PyMethodDef methods[] = {
    {"pack_i32", pack_i32, METH_VARARGS, "sequence of ints -> bytearray of int32"},
    {"pack_lists", pack_lists, METH_VARARGS, "rows of ints -> (int32 tokens, int64 offsets[n+1]), threaded"},
    {"meta_runs", meta_runs, METH_VARARGS, "per-token (origin, version) -> (starts, origin codes, versions, nruns)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_tmfast", NULL, -1, methods};

PyMODINIT_FUNC PyInit__tmfast(void) { return PyModule_Create(&module); }

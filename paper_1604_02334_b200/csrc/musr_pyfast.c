// musr_pyfast.c -- CPython fast path of the drop-in objective call (host side).
//
// The reference objective reads every dataset on every call (musr.py:181-232);
// the package answers from a cached device session instead, so each call must
// first prove that the problem is the one the session was built from.  In
// Python that proof costs O(datasets) attribute reads and comparisons --
// ~30 us per call for the 64 datasets of C4 when they are the reference's own
// MusrDataset objects, i.e. a few percent of a whole evaluation, paid on every
// minimizer step.  This module keeps the last call's problem in C and
// re-validates it with pointer compares:
//
//   * the same datasets list (identity) holding the same dataset objects;
//   * the same theory, backend and constants objects (frozen dataclasses in
//     the reference, theory.py:363-406, musr.py:52-59);
//   * no attribute of any dataset assigned since: every dataset's __dict__ is
//     watched with a CPython dict watcher (PyDict_AddWatcher, 3.12+) that bumps
//     a counter on any event;
//   * every counts array still read-only (objective.py _FrozenCounts: an
//     in-place edit needs writeable = True first);
//   * p a float64, aligned, contiguous 1-D ndarray of the session's length.
//
// On a hit it runs musr_eval (libmusr_b200.so, C ABI) with the GIL released
// under the session's lock and returns the total as a Python float.  Anything
// else -- a miss, a busy lock, a non-zero status, an MLH bin with a
// non-positive model -- returns None and the caller takes the Python path,
// which re-validates, evaluates and raises the reference's exceptions.  The
// fast path never computes anything itself: the objective is always the
// device's.
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_2_0_API_VERSION
#include <numpy/ndarraytypes.h>  // struct layout and inline accessors only (no API table)
#include <stdint.h>

#if PY_VERSION_HEX < 0x030C0000
#error "musr_pyfast needs CPython >= 3.12 (dict watchers)"
#endif

typedef int (*musr_eval_fn)(void* ctx, int kind, const double* p, int n_p, double* per_dataset,
                            int64_t* first_bad_bin, double* total);

static musr_eval_fn g_eval = NULL;
static PyTypeObject* g_ndarray = NULL;  // numpy.ndarray
static PyObject* g_f64 = NULL;          // numpy.dtype('float64') (the builtin descriptor)
static int g_watcher = -1;
static unsigned long long g_mutations = 0;  // any event on a watched dataset __dict__
static PyObject* g_str_acquire = NULL;
static PyObject* g_str_release = NULL;

typedef struct {
  int valid;
  PyObject* session;    // strong refs: the remembered objects cannot be freed and
  PyObject* datasets;   // their addresses reused while remembered
  PyObject** items;
  PyObject** dicts;
  Py_ssize_t n;
  PyObject* expr;
  PyObject* backend;
  PyObject* constants;
  PyObject** arrays;
  Py_ssize_t n_arrays;
  PyObject* lock;
  unsigned long long mutations;
  void* ctx;
  int n_p, n_global;
  double* sums;
  int64_t* bad;
  double* total;
} Slot;

static Slot g_last;

static int on_dict_event(PyDict_WatchEvent ev, PyObject* d, PyObject* k, PyObject* v) {
  (void)ev; (void)d; (void)k; (void)v;
  ++g_mutations;
  return 0;
}

static void slot_clear(Slot* s) {
  s->valid = 0;
  for (Py_ssize_t i = 0; i < s->n; ++i) {
    Py_XDECREF(s->items[i]);
    Py_XDECREF(s->dicts[i]);
  }
  for (Py_ssize_t i = 0; i < s->n_arrays; ++i) Py_XDECREF(s->arrays[i]);
  PyMem_Free(s->items);
  PyMem_Free(s->dicts);
  PyMem_Free(s->arrays);
  Py_CLEAR(s->session);
  Py_CLEAR(s->datasets);
  Py_CLEAR(s->expr);
  Py_CLEAR(s->backend);
  Py_CLEAR(s->constants);
  Py_CLEAR(s->lock);
  s->items = s->dicts = s->arrays = NULL;
  s->n = s->n_arrays = 0;
}

static PyObject** seq_items(PyObject* seq, Py_ssize_t* n) {
  if (PyList_CheckExact(seq)) {
    *n = PyList_GET_SIZE(seq);
    return ((PyListObject*)seq)->ob_item;
  }
  if (PyTuple_CheckExact(seq)) {
    *n = PyTuple_GET_SIZE(seq);
    return ((PyTupleObject*)seq)->ob_item;
  }
  return NULL;
}

// init(musr_eval_address, numpy.ndarray, numpy.dtype('float64'))
static PyObject* pf_init(PyObject* self, PyObject* args) {
  unsigned long long addr;
  PyObject *nd, *f64;
  if (!PyArg_ParseTuple(args, "KOO", &addr, &nd, &f64)) return NULL;
  if (!PyType_Check(nd)) {
    PyErr_SetString(PyExc_TypeError, "second argument must be numpy.ndarray");
    return NULL;
  }
  g_eval = (musr_eval_fn)(uintptr_t)addr;
  Py_XSETREF(g_ndarray, (PyTypeObject*)Py_NewRef(nd));
  Py_XSETREF(g_f64, Py_NewRef(f64));
  if (g_watcher < 0) {
    g_watcher = PyDict_AddWatcher(on_dict_event);
    if (g_watcher < 0) return NULL;
  }
  Py_RETURN_NONE;
}

// remember(session, datasets, expr, backend, constants, arrays, ctx, n_p, n_global,
//          sums, bad, total, lock) -> bool
static PyObject* pf_remember(PyObject* self, PyObject* args) {
  PyObject *sess, *datasets, *expr, *backend, *constants, *arrays, *lock;
  unsigned long long ctx, sums, bad, total;
  int n_p, n_global;
  if (!PyArg_ParseTuple(args, "OOOOOOKiiKKKO", &sess, &datasets, &expr, &backend, &constants,
                        &arrays, &ctx, &n_p, &n_global, &sums, &bad, &total, &lock))
    return NULL;
  slot_clear(&g_last);
  if (g_eval == NULL || g_watcher < 0 || !ctx) Py_RETURN_FALSE;
  Py_ssize_t n = 0, na = 0;
  PyObject** items = seq_items(datasets, &n);
  PyObject** arr = seq_items(arrays, &na);
  if (items == NULL || arr == NULL || n == 0) Py_RETURN_FALSE;
  for (Py_ssize_t i = 0; i < na; ++i)
    if (!PyObject_TypeCheck(arr[i], g_ndarray)) Py_RETURN_FALSE;
  Slot s = {0};
  s.items = PyMem_Calloc((size_t)n, sizeof(PyObject*));
  s.dicts = PyMem_Calloc((size_t)n, sizeof(PyObject*));
  s.arrays = PyMem_Calloc((size_t)(na ? na : 1), sizeof(PyObject*));
  if (!s.items || !s.dicts || !s.arrays) {
    PyMem_Free(s.items); PyMem_Free(s.dicts); PyMem_Free(s.arrays);
    return PyErr_NoMemory();
  }
  s.n = n;
  for (Py_ssize_t i = 0; i < n; ++i) {
    s.items[i] = Py_NewRef(items[i]);
    PyObject* d = PyObject_GenericGetDict(items[i], NULL);  // new reference
    if (d == NULL || !PyDict_CheckExact(d) || PyDict_Watch(g_watcher, d) < 0) {
      PyErr_Clear();                       // no plain __dict__: stay on the Python path
      Py_XDECREF(d);
      slot_clear(&s);
      Py_RETURN_FALSE;
    }
    s.dicts[i] = d;
  }
  s.n_arrays = na;
  for (Py_ssize_t i = 0; i < na; ++i) s.arrays[i] = Py_NewRef(arr[i]);
  s.session = Py_NewRef(sess);
  s.datasets = Py_NewRef(datasets);
  s.expr = Py_NewRef(expr);
  s.backend = Py_NewRef(backend);
  s.constants = Py_NewRef(constants);
  s.lock = Py_NewRef(lock);
  s.mutations = g_mutations;
  s.ctx = (void*)(uintptr_t)ctx;
  s.n_p = n_p;
  s.n_global = n_global;
  s.sums = (double*)(uintptr_t)sums;
  s.bad = (int64_t*)(uintptr_t)bad;
  s.total = (double*)(uintptr_t)total;
  s.valid = 1;
  g_last = s;
  Py_RETURN_TRUE;
}

// forget(session=None): drop the remembered call (of this session only, if given)
static PyObject* pf_forget(PyObject* self, PyObject* args) {
  PyObject* sess = Py_None;
  if (!PyArg_ParseTuple(args, "|O", &sess)) return NULL;
  if (sess == Py_None || g_last.session == sess) slot_clear(&g_last);
  Py_RETURN_NONE;
}

// evaluate(kind, datasets, expr, p, backend, constants) -> float | None
static PyObject* pf_evaluate(PyObject* self, PyObject* const* a, Py_ssize_t nargs) {
  if (nargs != 6) {
    PyErr_SetString(PyExc_TypeError, "evaluate(kind, datasets, expr, p, backend, constants)");
    return NULL;
  }
  Slot* s = &g_last;
  if (!s->valid || g_mutations != s->mutations || a[1] != s->datasets || a[2] != s->expr ||
      a[4] != s->backend || a[5] != s->constants)
    Py_RETURN_NONE;
  const long kind = PyLong_AsLong(a[0]);
  if (kind != 0 && kind != 1) {
    PyErr_Clear();
    Py_RETURN_NONE;
  }
  Py_ssize_t n = 0;
  PyObject** items = seq_items(a[1], &n);
  if (items == NULL || n != s->n) Py_RETURN_NONE;
  for (Py_ssize_t i = 0; i < n; ++i)
    if (items[i] != s->items[i]) Py_RETURN_NONE;  // list edited in place
  for (Py_ssize_t i = 0; i < s->n_arrays; ++i)
    if (PyArray_FLAGS((PyArrayObject*)s->arrays[i]) & NPY_ARRAY_WRITEABLE) Py_RETURN_NONE;
  for (Py_ssize_t i = 0; i < n; ++i) {  // a dataset's __dict__ replaced wholesale
    PyObject* d = PyObject_GenericGetDict(items[i], NULL);
    const int same = d == s->dicts[i];
    Py_XDECREF(d);
    if (!same) {
      PyErr_Clear();
      Py_RETURN_NONE;
    }
  }
  PyObject* p = a[3];
  if (Py_TYPE(p) != g_ndarray) Py_RETURN_NONE;
  PyArrayObject* pa = (PyArrayObject*)p;
  const int want = NPY_ARRAY_C_CONTIGUOUS | NPY_ARRAY_ALIGNED;
  if (PyArray_NDIM(pa) != 1 || PyArray_DIM(pa, 0) != s->n_p ||
      (PyObject*)PyArray_DESCR(pa) != g_f64 || (PyArray_FLAGS(pa) & want) != want)
    Py_RETURN_NONE;

  // the session's lock (Session.evaluate holds it around the same call)
  PyObject* got = PyObject_CallMethodOneArg(s->lock, g_str_acquire, Py_False);
  if (got == NULL) return NULL;
  const int locked = got == Py_True;
  Py_DECREF(got);
  if (!locked) Py_RETURN_NONE;  // busy: the Python path waits for it
  PyObject* keep = Py_NewRef(s->session);  // the buffers below belong to it
  PyObject* lock = Py_NewRef(s->lock);
  void* ctx = s->ctx;
  const double* pp = (const double*)PyArray_DATA(pa);
  const int n_p = s->n_p, n_global = s->n_global;
  double* sums = s->sums;
  int64_t* bad = s->bad;
  double* total = s->total;
  Py_INCREF(p);
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = g_eval(ctx, (int)kind, pp, n_p, sums, bad, total);
  Py_END_ALLOW_THREADS
  Py_DECREF(p);
  int clean = rc == 0;
  if (clean && kind == 1)
    for (int j = 0; j < n_global; ++j)
      if (bad[j] >= 0) { clean = 0; break; }  // the Python path raises the reference's error
  const double v = *total;
  PyObject* rel = PyObject_CallMethodNoArgs(lock, g_str_release);
  Py_DECREF(lock);
  Py_DECREF(keep);
  if (rel == NULL) return NULL;
  Py_DECREF(rel);
  if (!clean) Py_RETURN_NONE;
  return PyFloat_FromDouble(v);
}

static PyObject* pf_stats(PyObject* self, PyObject* unused) {
  return Py_BuildValue("{s:i,s:K,s:n}", "valid", g_last.valid, "mutations", g_mutations,
                       "datasets", g_last.n);
}

static PyMethodDef methods[] = {
    {"init", pf_init, METH_VARARGS, "init(musr_eval_address, numpy.ndarray, float64 dtype)"},
    {"remember", pf_remember, METH_VARARGS, "remember the last evaluated problem"},
    {"forget", pf_forget, METH_VARARGS, "forget([session])"},
    {"evaluate", (PyCFunction)(void (*)(void))pf_evaluate, METH_FASTCALL,
     "evaluate(kind, datasets, expr, p, backend, constants) -> float | None"},
    {"stats", pf_stats, METH_NOARGS, "state of the remembered call (tests)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pyfast",
                                    "CPython fast path of the drop-in objective call", -1,
                                    methods};

PyMODINIT_FUNC PyInit__pyfast(void) {
  g_str_acquire = PyUnicode_InternFromString("acquire");
  g_str_release = PyUnicode_InternFromString("release");
  if (!g_str_acquire || !g_str_release) return NULL;
  return PyModule_Create(&module);
}

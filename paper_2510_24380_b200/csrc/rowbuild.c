/*
 * rowbuild.c — native builder of the reference's result rows (CPython C API).
 *
 * engine._build_result turns the device's materialized rows (global index,
 * objective, constraint values, reaction position, digits; K7 output) into
 * the caller's result objects, the shape _result_from_selection produces
 * (reference engine.py:238-262):
 *
 *   ScoredCompound(global_index, chi=MultiIndex(reaction_id,
 *                  ((rgroup_id, synthon_id), ...)), objective, violation=0.0,
 *                  constraint_values=(...))
 *
 * Built in C, one pass, no per-row Python bytecode: at k = 10,000 the Python
 * loop cost ~2 us per row and dominated the operator API's latency (the
 * device pass is ~0.4 ms).  Instances of plain dataclasses (no __post_init__,
 * no __slots__; frozen or not) are allocated with tp_alloc and their fields
 * set with the generic setattr (what object.__setattr__ does), which is
 * exactly the state the generated __init__ leaves; any other class is called.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

static PyObject *s_reaction_id, *s_assignment, *s_global_index, *s_chi, *s_objective, *s_violation,
    *s_constraint_values;

static int get_buf(PyObject* o, Py_buffer* b, Py_ssize_t itemsize, Py_ssize_t need) {
  if (PyObject_GetBuffer(o, b, PyBUF_C_CONTIGUOUS) < 0) return -1;
  if (b->len < need * itemsize) {
    PyBuffer_Release(b);
    PyErr_SetString(PyExc_ValueError, "result buffer too small");
    return -1;
  }
  return 0;
}

static PyObject* make_obj(PyTypeObject* cls, int fast, PyObject** names, PyObject** vals, int n) {
  if (fast) {
    PyObject* o = cls->tp_alloc(cls, 0);
    if (!o) return NULL;
    for (int i = 0; i < n; ++i)
      if (PyObject_GenericSetAttr(o, names[i], vals[i]) < 0) {
        Py_DECREF(o);
        return NULL;
      }
    return o;
  }
  PyObject* args = PyTuple_New(n);
  if (!args) return NULL;
  for (int i = 0; i < n; ++i) {
    Py_INCREF(vals[i]);
    PyTuple_SET_ITEM(args, i, vals[i]);
  }
  PyObject* o = PyObject_Call((PyObject*)cls, args, NULL);
  Py_DECREF(args);
  return o;
}

/* build_entries(mi_cls, sc_cls, fast, n, g, obj, cons, m, rx, digits, rx_table[, chi_cache[, chi_insert]]) -> list
 *   g: uint64[n]; obj: float64[n]; cons: float64[n*m]; rx: int32[n];
 *   digits: int32[n*6]; rx_table: sequence indexed by reaction position of
 *   (reaction_id, (rgroup_id, ...), ((synthon_id, ...), ...)[, (pair list, ...)]);
 *   the optional 4th item holds one list per R-group, indexed by digit, of
 *   (rgroup_id, synthon_id) tuples filled on first use (shared: tuples are
 *   immutable).  chi_cache: dict global index -> MultiIndex (frozen in the
 *   reference, csl.py:47, so a repeated product's chi is shared) or None;
 *   chi_insert: whether new MultiIndex instances are added to it. */
#define CHI_CACHE_MAX (1 << 16) /* cleared when full: bounded memory, no large-dict resize pauses */
static PyObject* build_entries(PyObject* self, PyObject* args) {
  PyObject *mi_cls, *sc_cls, *og, *oobj, *ocons, *orx, *odig, *table, *chi_cache = Py_None;
  int fast, chi_insert = 1;
  Py_ssize_t n, m;
  (void)self;
  if (!PyArg_ParseTuple(args, "OOpnOOOnOOO|Op", &mi_cls, &sc_cls, &fast, &n, &og, &oobj, &ocons, &m, &orx, &odig,
                        &table, &chi_cache, &chi_insert))
    return NULL;
  if (chi_cache != Py_None && !PyDict_Check(chi_cache)) {
    PyErr_SetString(PyExc_TypeError, "chi_cache must be a dict or None");
    return NULL;
  }
  if (!PyType_Check(mi_cls) || !PyType_Check(sc_cls)) {
    PyErr_SetString(PyExc_TypeError, "result classes must be types");
    return NULL;
  }
  Py_buffer bg, bo, bc, br, bd;
  if (get_buf(og, &bg, 8, n) < 0) return NULL;
  if (get_buf(oobj, &bo, 8, n) < 0) goto e1;
  if (get_buf(ocons, &bc, 8, n * m) < 0) goto e2;
  if (get_buf(orx, &br, 4, n) < 0) goto e3;
  if (get_buf(odig, &bd, 4, n * 6) < 0) goto e4;
  const uint64_t* g = (const uint64_t*)bg.buf;
  const double* obj = (const double*)bo.buf;
  const double* cons = (const double*)bc.buf;
  const int32_t* rx = (const int32_t*)br.buf;
  const int32_t* dig = (const int32_t*)bd.buf;
  PyObject* out = PyList_New(n);
  PyObject* zero = PyFloat_FromDouble(0.0); /* violation +0.0 (engine.py:252) */
  if (!out || !zero) goto fail;
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* gi = PyLong_FromUnsignedLongLong(g[i]);
    if (!gi) goto fail;
    PyObject* chi = NULL;
    if (chi_cache != Py_None) {
      chi = PyDict_GetItemWithError(chi_cache, gi);
      if (chi) {
        Py_INCREF(chi);
      } else if (PyErr_Occurred()) {
        Py_DECREF(gi);
        goto fail;
      }
    }
    if (!chi) {
      PyObject* info = PySequence_GetItem(table, rx[i]);
      if (!info) {
        Py_DECREF(gi);
        goto fail;
      }
      PyObject *rid = PyTuple_GetItem(info, 0), *rgids = PyTuple_GetItem(info, 1), *sids = PyTuple_GetItem(info, 2);
      PyObject* pairs = PyTuple_GET_SIZE(info) > 3 ? PyTuple_GET_ITEM(info, 3) : NULL;
      if (!rid || !rgids || !sids) {
        Py_DECREF(info);
        Py_DECREF(gi);
        goto fail;
      }
      const Py_ssize_t c = PyTuple_GET_SIZE(rgids);
      PyObject* asg = PyTuple_New(c);
      if (!asg) {
        Py_DECREF(info);
        Py_DECREF(gi);
        goto fail;
      }
      for (Py_ssize_t j = 0; j < c; ++j) {
        const int32_t d = dig[i * 6 + j];
        PyObject* lst = pairs ? PyTuple_GET_ITEM(pairs, j) : NULL;
        PyObject* pair = NULL;
        if (lst && PyList_Check(lst) && d >= 0 && d < PyList_GET_SIZE(lst) && PyList_GET_ITEM(lst, d) != Py_None) {
          pair = PyList_GET_ITEM(lst, d);
          Py_INCREF(pair);
        } else {
          PyObject* sid = PySequence_GetItem(PyTuple_GET_ITEM(sids, j), d);
          if (sid) pair = PyTuple_Pack(2, PyTuple_GET_ITEM(rgids, j), sid);
          Py_XDECREF(sid);
          if (pair && lst && PyList_Check(lst) && d >= 0 && d < PyList_GET_SIZE(lst)) {
            Py_INCREF(pair);
            PyList_SetItem(lst, d, pair);  /* steals the extra reference, releases None */
          }
        }
        if (!pair) {
          Py_DECREF(asg);
          Py_DECREF(info);
          Py_DECREF(gi);
          goto fail;
        }
        PyTuple_SET_ITEM(asg, j, pair);
      }
      PyObject* mi_names[2] = {s_reaction_id, s_assignment};
      PyObject* mi_vals[2] = {rid, asg};
      chi = make_obj((PyTypeObject*)mi_cls, fast, mi_names, mi_vals, 2);
      Py_DECREF(asg);
      Py_DECREF(info);
      if (!chi) {
        Py_DECREF(gi);
        goto fail;
      }
      if (chi_cache != Py_None && chi_insert && PyDict_GET_SIZE(chi_cache) >= CHI_CACHE_MAX) PyDict_Clear(chi_cache);
      if (chi_cache != Py_None && chi_insert && PyDict_SetItem(chi_cache, gi, chi) < 0) {
        Py_DECREF(chi);
        Py_DECREF(gi);
        goto fail;
      }
    }
    PyObject* cv = PyTuple_New(m);
    PyObject* ov = PyFloat_FromDouble(obj[i]);
    if (!cv || !ov) {
      Py_XDECREF(cv);
      Py_XDECREF(gi);
      Py_XDECREF(ov);
      Py_DECREF(chi);
      goto fail;
    }
    for (Py_ssize_t j = 0; j < m; ++j) PyTuple_SET_ITEM(cv, j, PyFloat_FromDouble(cons[i * m + j]));
    PyObject* sc_names[5] = {s_global_index, s_chi, s_objective, s_violation, s_constraint_values};
    PyObject* sc_vals[5] = {gi, chi, ov, zero, cv};
    PyObject* sc = make_obj((PyTypeObject*)sc_cls, fast, sc_names, sc_vals, 5);
    Py_DECREF(gi);
    Py_DECREF(chi);
    Py_DECREF(ov);
    Py_DECREF(cv);
    if (!sc) goto fail;
    PyList_SET_ITEM(out, i, sc);
  }
  Py_DECREF(zero);
  PyBuffer_Release(&bd);
  PyBuffer_Release(&br);
  PyBuffer_Release(&bc);
  PyBuffer_Release(&bo);
  PyBuffer_Release(&bg);
  return out;
fail:
  Py_XDECREF(out);
  Py_XDECREF(zero);
  PyBuffer_Release(&bd);
e4:
  PyBuffer_Release(&br);
e3:
  PyBuffer_Release(&bc);
e2:
  PyBuffer_Release(&bo);
e1:
  PyBuffer_Release(&bg);
  return NULL;
}

/* ---------------------------------------------------------------------------
 * format_rows(entries) -> str: the data lines of save_result (reference
 * engine.py:463-489, without the optional assembled column), one per entry:
 *   rank \t global_index \t reaction_id \t synthon ids (comma-joined) \t
 *   repr(objective) \t repr(violation) [\t repr(constraint value)]...
 * Floats are formatted with PyOS_double_to_string(.., 'r', 0, ADD_DOT_0), the
 * routine behind float.__repr__, so the bytes equal the reference's f"{v!r}";
 * any non-float value goes through PyObject_Repr / PyObject_Str as the
 * reference's f-string would. */
typedef struct {
  char* p;
  size_t n, cap;
} sbuf;

static int sb_put(sbuf* b, const char* s, size_t k) {
  if (b->n + k + 1 > b->cap) {
    size_t nc = b->cap ? b->cap : 1 << 16;
    while (nc < b->n + k + 1) nc *= 2;
    char* q = (char*)PyMem_Realloc(b->p, nc);
    if (!q) {
      PyErr_NoMemory();
      return -1;
    }
    b->p = q;
    b->cap = nc;
  }
  memcpy(b->p + b->n, s, k);
  b->n += k;
  return 0;
}

static int sb_obj(sbuf* b, PyObject* o, int use_repr) {
  if (PyFloat_CheckExact(o) && use_repr) {
    char* t = PyOS_double_to_string(PyFloat_AS_DOUBLE(o), 'r', 0, Py_DTSF_ADD_DOT_0, NULL);
    if (!t) return -1;
    const int r = sb_put(b, t, strlen(t));
    PyMem_Free(t);
    return r;
  }
  PyObject* u = use_repr ? PyObject_Repr(o) : PyObject_Str(o);
  if (!u) return -1;
  Py_ssize_t k;
  const char* t = PyUnicode_AsUTF8AndSize(u, &k);
  const int r = t ? sb_put(b, t, (size_t)k) : -1;
  Py_DECREF(u);
  return r;
}

static PyObject* format_rows(PyObject* self, PyObject* args) {
  PyObject* entries;
  (void)self;
  if (!PyArg_ParseTuple(args, "O", &entries)) return NULL;
  PyObject* seq = PySequence_Fast(entries, "entries must be a sequence");
  if (!seq) return NULL;
  sbuf b = {NULL, 0, 0};
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  char num[32];
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* e = PySequence_Fast_GET_ITEM(seq, i);
    PyObject *gi = NULL, *chi = NULL, *rid = NULL, *asg = NULL, *obj = NULL, *viol = NULL, *cv = NULL;
    int ok = 0;
    gi = PyObject_GetAttr(e, s_global_index);
    chi = gi ? PyObject_GetAttr(e, s_chi) : NULL;
    rid = chi ? PyObject_GetAttr(chi, s_reaction_id) : NULL;
    asg = rid ? PyObject_GetAttr(chi, s_assignment) : NULL;
    obj = asg ? PyObject_GetAttr(e, s_objective) : NULL;
    viol = obj ? PyObject_GetAttr(e, s_violation) : NULL;
    cv = viol ? PyObject_GetAttr(e, s_constraint_values) : NULL;
    if (cv) {
      const int k = snprintf(num, sizeof num, "%zd\t", i);
      ok = sb_put(&b, num, (size_t)k) == 0 && sb_obj(&b, gi, 0) == 0 && sb_put(&b, "\t", 1) == 0 &&
           sb_obj(&b, rid, 0) == 0 && sb_put(&b, "\t", 1) == 0;
      PyObject* a = ok ? PySequence_Fast(asg, "assignment must be a sequence") : NULL;
      if (a) {
        for (Py_ssize_t j = 0; ok && j < PySequence_Fast_GET_SIZE(a); ++j) {
          PyObject* pair = PySequence_Fast_GET_ITEM(a, j);
          PyObject* sid = PySequence_GetItem(pair, 1);
          ok = sid && (j == 0 || sb_put(&b, ",", 1) == 0) && sb_obj(&b, sid, 0) == 0;
          Py_XDECREF(sid);
        }
        Py_DECREF(a);
      } else {
        ok = 0;
      }
      ok = ok && sb_put(&b, "\t", 1) == 0 && sb_obj(&b, obj, 1) == 0 && sb_put(&b, "\t", 1) == 0 &&
           sb_obj(&b, viol, 1) == 0;
      PyObject* c = ok ? PySequence_Fast(cv, "constraint values must be a sequence") : NULL;
      if (c) {
        for (Py_ssize_t j = 0; ok && j < PySequence_Fast_GET_SIZE(c); ++j)
          ok = sb_put(&b, "\t", 1) == 0 && sb_obj(&b, PySequence_Fast_GET_ITEM(c, j), 1) == 0;
        Py_DECREF(c);
      } else {
        ok = 0;
      }
      ok = ok && sb_put(&b, "\n", 1) == 0;
    }
    Py_XDECREF(gi);
    Py_XDECREF(chi);
    Py_XDECREF(rid);
    Py_XDECREF(asg);
    Py_XDECREF(obj);
    Py_XDECREF(viol);
    Py_XDECREF(cv);
    if (!ok) {
      PyMem_Free(b.p);
      Py_DECREF(seq);
      return NULL;
    }
  }
  Py_DECREF(seq);
  PyObject* out = PyUnicode_FromStringAndSize(b.p ? b.p : "", (Py_ssize_t)b.n);
  PyMem_Free(b.p);
  return out;
}

static PyMethodDef methods[] = {
    {"build_entries", build_entries, METH_VARARGS, "ScoredCompound rows from materialized device rows"},
    {"format_rows", format_rows, METH_VARARGS, "save_result data lines (repr floats)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef moddef = {PyModuleDef_HEAD_INIT, "_rowbuild", NULL, -1, methods};

PyMODINIT_FUNC PyInit__rowbuild(void) {
  s_reaction_id = PyUnicode_InternFromString("reaction_id");
  s_assignment = PyUnicode_InternFromString("assignment");
  s_global_index = PyUnicode_InternFromString("global_index");
  s_chi = PyUnicode_InternFromString("chi");
  s_objective = PyUnicode_InternFromString("objective");
  s_violation = PyUnicode_InternFromString("violation");
  s_constraint_values = PyUnicode_InternFromString("constraint_values");
  return PyModule_Create(&moddef);
}

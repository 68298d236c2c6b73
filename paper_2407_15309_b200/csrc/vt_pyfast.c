/* CPython entry points for the manager's per-token hot calls into
 * libvtensor.so (include/vtensor.h). ctypes spends ~1.5 us converting the
 * arguments of one vt_extend; a METH_FASTCALL function spends ~0.1 us. These
 * are thin: no state of their own, the C ABI stays the boundary.
 *
 *   extend(dev, base, first_page, reuse_ids, n_create) -> list[int] | None
 *       vt_extend; the created chunk ids, or None when the shim rejected the
 *       fused call (nothing changed; the caller runs the per-op sequence).
 *   unmap_tail(dev, base, from_page, down_to) -> (rc, [ids unmapped])
 *       vt_unmap_tail.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

#include "../../include/vtensor.h"

#define SMALL 64

static int get_dev(PyObject* o, vt_device** d) {
  void* p = PyLong_AsVoidPtr(o);
  if (!p) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "null vt_device");
    return -1;
  }
  *d = (vt_device*)p;
  return 0;
}

static PyObject* py_extend(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 5) {
    PyErr_SetString(PyExc_TypeError, "extend(dev, base, first_page, reuse_ids, n_create)");
    return NULL;
  }
  vt_device* d;
  if (get_dev(args[0], &d)) return NULL;
  int64_t base = PyLong_AsLongLong(args[1]);
  int64_t first = PyLong_AsLongLong(args[2]);
  int64_t n_create = PyLong_AsLongLong(args[4]);
  if (PyErr_Occurred()) return NULL;
  PyObject* seq = PySequence_Fast(args[3], "reuse_ids must be a sequence");
  if (!seq) return NULL;
  Py_ssize_t n_reuse = PySequence_Fast_GET_SIZE(seq);
  int64_t reuse_small[SMALL], out_small[SMALL];
  int64_t* reuse = n_reuse <= SMALL ? reuse_small : (int64_t*)PyMem_Malloc(sizeof(int64_t) * n_reuse);
  int64_t* out = n_create <= SMALL ? out_small : (int64_t*)PyMem_Malloc(sizeof(int64_t) * n_create);
  PyObject* result = NULL;
  if (!reuse || !out || n_create < 0) {
    if (n_create < 0) PyErr_SetString(PyExc_ValueError, "negative n_create");
    else PyErr_NoMemory();
    goto done;
  }
  for (Py_ssize_t k = 0; k < n_reuse; ++k) {
    reuse[k] = PyLong_AsLongLong(PySequence_Fast_GET_ITEM(seq, k));
    if (PyErr_Occurred()) goto done;
  }
  if (vt_extend(d, base, first, reuse, (int64_t)n_reuse, n_create, out) != VT_OK) {
    result = Py_NewRef(Py_None);
    goto done;
  }
  result = PyList_New((Py_ssize_t)n_create);
  if (!result) goto done;
  for (int64_t k = 0; k < n_create; ++k) {
    PyObject* v = PyLong_FromLongLong(out[k]);
    if (!v) {
      Py_CLEAR(result);
      goto done;
    }
    PyList_SET_ITEM(result, (Py_ssize_t)k, v);
  }
done:
  if (reuse && reuse != reuse_small) PyMem_Free(reuse);
  if (out && out != out_small) PyMem_Free(out);
  Py_DECREF(seq);
  return result;
}

static PyObject* py_unmap_tail(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 4) {
    PyErr_SetString(PyExc_TypeError, "unmap_tail(dev, base, from_page, down_to)");
    return NULL;
  }
  vt_device* d;
  if (get_dev(args[0], &d)) return NULL;
  int64_t base = PyLong_AsLongLong(args[1]);
  int64_t from = PyLong_AsLongLong(args[2]);
  int64_t down = PyLong_AsLongLong(args[3]);
  if (PyErr_Occurred()) return NULL;
  int64_t n = from - down + 1;
  if (n < 0) n = 0;
  int64_t small[SMALL];
  int64_t* ids = n <= SMALL ? small : (int64_t*)PyMem_Malloc(sizeof(int64_t) * (size_t)n);
  if (!ids) return PyErr_NoMemory();
  int64_t done = 0;
  int rc = vt_unmap_tail(d, base, from, down, ids, &done);
  PyObject* lst = PyList_New((Py_ssize_t)done);
  if (lst) {
    for (int64_t k = 0; k < done; ++k) {
      PyObject* v = PyLong_FromLongLong(ids[k]);
      if (!v) {
        Py_CLEAR(lst);
        break;
      }
      PyList_SET_ITEM(lst, (Py_ssize_t)k, v);
    }
  }
  if (ids != small) PyMem_Free(ids);
  if (!lst) return NULL;
  return Py_BuildValue("(iN)", rc, lst);
}

static PyMethodDef methods[] = {
    {"extend", (PyCFunction)(void (*)(void))py_extend, METH_FASTCALL, "vt_extend"},
    {"unmap_tail", (PyCFunction)(void (*)(void))py_unmap_tail, METH_FASTCALL, "vt_unmap_tail"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_vtfast", NULL, -1, methods,
                                    NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__vtfast(void) { return PyModule_Create(&module); }

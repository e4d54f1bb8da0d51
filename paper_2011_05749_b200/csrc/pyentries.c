/* Host helper for the drop-in result type: SparseSpectrum.entries (dict[int, complex],
 * signals.py) built in one C loop from the decoder's (positions, values) arrays, in
 * their order (the reference's insertion order).  The dict is presized, and each key and
 * value object is made directly from the int64 / complex128 element — 4096 entries in
 * ~0.2 ms instead of ~0.4 ms for dict(zip(pos.tolist(), val.tolist())), time the
 * Python API otherwise spends holding the GIL per DSFFT signal.  Loaded with
 * ctypes.PyDLL (the GIL stays held); no CUDA here. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

PyObject* afft_py_entries(const int64_t* pos, const double* val, int64_t m) {
  PyObject* d = _PyDict_NewPresized((Py_ssize_t)m);
  if (!d) return NULL;
  for (int64_t i = 0; i < m; ++i) {
    PyObject* k = PyLong_FromLongLong(pos[i]);
    PyObject* c = k ? PyComplex_FromDoubles(val[2 * i], val[2 * i + 1]) : NULL;
    const int rc = c ? PyDict_SetItem(d, k, c) : -1;
    Py_XDECREF(k);
    Py_XDECREF(c);
    if (rc) {
      Py_DECREF(d);
      return NULL;
    }
  }
  return d;
}

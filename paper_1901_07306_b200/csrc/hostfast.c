/* CPython binding of the drop-in staging copy (host code only).
 *
 * The reference's callers feed DetectorState.process_batch 65,536-pair
 * numpy buffers (cli.py:215-217, distributed.py:225-227).  Through ctypes a
 * call spends ~3-5 us in Python before the copy starts (two numpy
 * `.ctypes.data` objects, ctypes argument conversion) -- a third of the
 * call at 65,536 pairs.  `pack_u32(hips, oips, dst_h, dst_o, room)` takes
 * the two arrays through the buffer protocol (C-contiguous, 1-D, format
 * 'I' = uint32) and calls the library's sspd_host_pack_pairs (the native
 * copy pool, host_stage.cu) with the GIL released.  Returns the number of
 * pairs staged, or -1 when the arrays are not plain 1-D uint32 of equal
 * length fitting `room` -- the caller then takes its general path.  The
 * copy function's address is set once from the loaded library
 * (`set_pack`), so this module has no link-time dependency on it.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

typedef int (*pack_fn)(const void*, const void*, uint64_t, uint32_t, uint32_t, uint32_t*, uint32_t*);
static pack_fn g_pack = NULL;

static PyObject* set_pack(PyObject* self, PyObject* arg) {
  (void)self;
  unsigned long long p = PyLong_AsUnsignedLongLong(arg);
  if (PyErr_Occurred()) return NULL;
  g_pack = (pack_fn)(uintptr_t)p;
  Py_RETURN_NONE;
}

static int u32_vector(Py_buffer* b) {
  if (b->ndim != 1 || b->itemsize != 4 || b->format == NULL) return 0;
  const char* f = b->format;
  if (*f == '=' || *f == '<' || *f == '@') ++f; /* native little-endian uint32 */
  return f[0] == 'I' && f[1] == '\0';
}

static PyObject* pack_u32(PyObject* self, PyObject* args) {
  (void)self;
  PyObject *ho, *oo;
  unsigned long long dh, dob, room;
  if (!PyArg_ParseTuple(args, "OOKKK", &ho, &oo, &dh, &dob, &room)) return NULL;
  if (g_pack == NULL) {
    PyErr_SetString(PyExc_RuntimeError, "pack_u32: set_pack was not called");
    return NULL;
  }
  Py_buffer bh, bo;
  if (PyObject_GetBuffer(ho, &bh, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) != 0) {
    PyErr_Clear();
    return PyLong_FromLong(-1);
  }
  if (PyObject_GetBuffer(oo, &bo, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) != 0) {
    PyErr_Clear();
    PyBuffer_Release(&bh);
    return PyLong_FromLong(-1);
  }
  long long n = -1;
  if (u32_vector(&bh) && u32_vector(&bo) && bh.shape[0] == bo.shape[0] && bh.shape[0] > 0 &&
      (unsigned long long)bh.shape[0] <= room) {
    const uint64_t cnt = (uint64_t)bh.shape[0];
    int rc;
    Py_BEGIN_ALLOW_THREADS
    rc = g_pack(bh.buf, bo.buf, cnt, 4, 4, (uint32_t*)(uintptr_t)dh, (uint32_t*)(uintptr_t)dob);
    Py_END_ALLOW_THREADS
    if (rc != 0) {
      PyBuffer_Release(&bh);
      PyBuffer_Release(&bo);
      return PyErr_Format(PyExc_RuntimeError, "sspd_host_pack_pairs failed (%d)", rc);
    }
    n = (long long)cnt;
  }
  PyBuffer_Release(&bh);
  PyBuffer_Release(&bo);
  return PyLong_FromLongLong(n);
}

static PyMethodDef methods[] = {
    {"set_pack", set_pack, METH_O, "address of sspd_host_pack_pairs in the loaded library"},
    {"pack_u32", pack_u32, METH_VARARGS, "stage two 1-D uint32 arrays; pairs staged or -1"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_hostfast", NULL, -1, methods, NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__hostfast(void) { return PyModule_Create(&module); }

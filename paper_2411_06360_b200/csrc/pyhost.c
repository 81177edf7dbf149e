/* _rsrhost: the CPython binding of the host-buffer session entry point
 * (rsr_host_session_multiply, include/rsr_b200.h).  ctypes spends ~2 us per NumPy data pointer
 * and ~1 us per call on argument conversion; this binding takes the vector and the result
 * array through the buffer protocol and releases the GIL while the call waits for the GPU.
 * Everything else (validation, sessions, errors) stays in the Python layer (kernels.py). */
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include "rsr_b200.h"

/* multiply(session: int, v: buffer, v_dtype: int, out: writable buffer, out_dtype: int,
 *          variant: int, stream: int) -> int rsr_status */
static PyObject* rsrhost_multiply(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 7) {
    PyErr_SetString(PyExc_TypeError, "multiply(session, v, v_dtype, out, out_dtype, variant, stream)");
    return NULL;
  }
  void* sess = PyLong_AsVoidPtr(args[0]);
  const int v_dtype = (int)PyLong_AsLong(args[2]);
  const int out_dtype = (int)PyLong_AsLong(args[4]);
  const int variant = (int)PyLong_AsLong(args[5]);
  void* stream = PyLong_AsVoidPtr(args[6]);
  if (PyErr_Occurred()) return NULL;
  Py_buffer v, out;
  if (PyObject_GetBuffer(args[1], &v, PyBUF_C_CONTIGUOUS) < 0) return NULL;
  if (PyObject_GetBuffer(args[3], &out, PyBUF_C_CONTIGUOUS | PyBUF_WRITABLE) < 0) {
    PyBuffer_Release(&v);
    return NULL;
  }
  rsr_status st;
  Py_BEGIN_ALLOW_THREADS
  st = rsr_host_session_multiply((rsr_host_session*)sess, v.buf, (rsr_dtype)v_dtype, (size_t)v.len, out.buf,
                                 (rsr_dtype)out_dtype, (size_t)out.len, (rsr_variant)variant, stream);
  Py_END_ALLOW_THREADS
  PyBuffer_Release(&out);
  PyBuffer_Release(&v);
  return PyLong_FromLong((long)st);
}

static PyMethodDef methods[] = {
    {"multiply", (PyCFunction)(void (*)(void))rsrhost_multiply, METH_FASTCALL,
     "multiply(session, v, v_dtype, out, out_dtype, variant, stream) -> rsr_status"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_rsrhost", NULL, -1, methods};

PyMODINIT_FUNC PyInit__rsrhost(void) { return PyModule_Create(&module); }

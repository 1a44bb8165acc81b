/* pyfast.c -- _gemm_fast: a vectorcall (METH_FASTCALL) entry for the binding's hot call.
 *
 * Argument marshalling only: converts 14 Python ints / floats to C and calls gemm_f64_ex
 * (include/gemm_f64.h) through the function pointer the binding hands over with
 * set_target(address) -- the address ctypes resolved in the already loaded libgemm_f64.so, so
 * there is exactly one copy of the library (its plan table, workspace and error state).
 * ctypes' per-argument conversion costs ~2 us per call on the GPU box's host, a large share of
 * a small GEMM (tools/binding_overhead.py).  Built by paper_1706_10086_b200/build.py when
 * Python's headers are present; without it the binding calls the same symbol through ctypes.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

typedef int (*gemm_ex_fn)(int64_t, int64_t, int64_t, double, const double *, int64_t, const double *, int64_t,
                          double, double *, int64_t, int, int, void *);

static gemm_ex_fn g_ex = NULL;

static PyObject *set_target(PyObject *self, PyObject *arg) {
    (void)self;
    void *p = PyLong_AsVoidPtr(arg);
    if (!p) {
        if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "NULL gemm_f64_ex address");
        return NULL;
    }
    g_ex = (gemm_ex_fn)p;
    Py_RETURN_NONE;
}

static void *as_ptr(PyObject *o) { return o == Py_None ? NULL : PyLong_AsVoidPtr(o); }

/* gemm_f64_ex(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, cfg_id, splits, stream) -> status */
static PyObject *gemm_f64_ex(PyObject *self, PyObject *const *a, Py_ssize_t n) {
    (void)self;
    if (n != 14) {
        PyErr_Format(PyExc_TypeError, "gemm_f64_ex takes 14 arguments (%zd given)", n);
        return NULL;
    }
    if (!g_ex) {
        PyErr_SetString(PyExc_RuntimeError, "_gemm_fast.set_target was not called");
        return NULL;
    }
    const int64_t M = PyLong_AsLongLong(a[0]), N = PyLong_AsLongLong(a[1]), K = PyLong_AsLongLong(a[2]);
    const double alpha = PyFloat_AsDouble(a[3]);
    const double *A = (const double *)as_ptr(a[4]);
    const int64_t lda = PyLong_AsLongLong(a[5]);
    const double *B = (const double *)as_ptr(a[6]);
    const int64_t ldb = PyLong_AsLongLong(a[7]);
    const double beta = PyFloat_AsDouble(a[8]);
    double *C = (double *)as_ptr(a[9]);
    const int64_t ldc = PyLong_AsLongLong(a[10]);
    const long cfg = PyLong_AsLong(a[11]), splits = PyLong_AsLong(a[12]);
    void *stream = as_ptr(a[13]);
    if (PyErr_Occurred()) return NULL;
    int rc;
    Py_BEGIN_ALLOW_THREADS
    rc = g_ex(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, (int)cfg, (int)splits, stream);
    Py_END_ALLOW_THREADS
    return PyLong_FromLong(rc);
}

static PyMethodDef methods[] = {
    {"set_target", set_target, METH_O, "set_target(address of gemm_f64_ex)"},
    {"gemm_f64_ex", (PyCFunction)(void (*)(void))gemm_f64_ex, METH_FASTCALL,
     "gemm_f64_ex(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, cfg_id, splits, stream) -> status"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_gemm_fast", NULL, -1, methods, NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__gemm_fast(void) { return PyModule_Create(&module); }

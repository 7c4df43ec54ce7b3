// Host side of Collection.jagged_fill (collection.py:537-556). The reference
// turns every segment into an array with np.asarray in a Python loop, then
// concatenates them; at 1M clusters that loop is most of its ~400 ms.
//
// Here one C pass over the list reads each segment's length straight from
// the numpy array struct, and a second pass copies the bytes into one pool.
// Both passes split the list across host threads (the GIL stays held by the
// caller, so no Python code can touch the segments meanwhile). The GPU packer
// then turns the lengths and the pool into the prefix sums and the packed
// member pool.
//
// pack_segments(segments, dtype, alloc=None) -> out, or None
//   out is one buffer laid out as [lengths int64 x n | starts int64 x n | pool],
//   starts being the exclusive prefix sum of lengths (element offsets into the
//   pool). out = alloc(nbytes) when alloc is given (any writable buffer of at
//   least nbytes, e.g. a pinned staging area), else a new bytearray.
//   Returns None when some segment is not a C-contiguous, native-order numpy
//   array of exactly that dtype. The caller then takes the general np.asarray
//   path, which handles lists, tuples and conversions.
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <numpy/arrayobject.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace {

bool same_dtype(PyArrayObject* a, PyArray_Descr* want) {
  PyArray_Descr* d = PyArray_DESCR(a);
  return d == want || (d->type_num == want->type_num && PyArray_ITEMSIZE(a) == PyDataType_ELSIZE(want) &&
                       PyArray_ISNBO(d->byteorder) == PyArray_ISNBO(want->byteorder));
}

// Run fn(chunk, begin, end) over [0, n) on up to `threads` threads.
template <class F>
void split(Py_ssize_t n, int threads, F fn) {
  if (threads <= 1) {
    fn(0, 0, n);
    return;
  }
  std::vector<std::thread> pool;
  const Py_ssize_t per = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const Py_ssize_t b = std::min(n, t * per), e = std::min(n, b + per);
    pool.emplace_back(fn, t, b, e);
  }
  for (auto& th : pool) th.join();
}

int thread_count(Py_ssize_t n) {
  int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  if (const char* e = std::getenv("SOAKIT_SEGPACK_THREADS")) hw = std::max(1, std::atoi(e));
  return static_cast<int>(std::clamp<Py_ssize_t>(n / 32768, 1, std::min(hw, 16)));
}

PyObject* pack_segments(PyObject*, PyObject* args) {
  PyObject* seq = nullptr;
  PyArray_Descr* want = nullptr;
  PyObject* alloc = Py_None;
  if (!PyArg_ParseTuple(args, "OO&|O", &seq, PyArray_DescrConverter, &want, &alloc)) return nullptr;
  PyObject* fast = PySequence_Fast(seq, "segments must be a sequence");
  if (!fast) {
    Py_DECREF(want);
    return nullptr;
  }
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  PyObject** items = PySequence_Fast_ITEMS(fast);
  const int threads = thread_count(n);
  std::vector<int64_t> lengths(static_cast<size_t>(n));
  std::vector<size_t> chunk_bytes(static_cast<size_t>(threads), 0);
  std::vector<int64_t> chunk_members(static_cast<size_t>(threads), 0);
  std::vector<char> chunk_ok(static_cast<size_t>(threads), 1);
  const bool nbo = PyArray_ISNBO(want->byteorder);
  split(n, threads, [&](int t, Py_ssize_t b, Py_ssize_t e) {  // 1. lengths
    size_t bytes = 0;
    int64_t members = 0;
    for (Py_ssize_t i = b; i < e; ++i) {
      PyObject* o = items[i];
      if (!PyArray_Check(o)) {
        chunk_ok[t] = 0;
        return;
      }
      PyArrayObject* a = reinterpret_cast<PyArrayObject*>(o);
      if (!PyArray_IS_C_CONTIGUOUS(a) || !same_dtype(a, want) || PyArray_NDIM(a) > 1) {
        chunk_ok[t] = 0;
        return;
      }
      const int64_t len = static_cast<int64_t>(PyArray_SIZE(a));
      lengths[static_cast<size_t>(i)] = len;
      members += len;
      bytes += static_cast<size_t>(PyArray_NBYTES(a));
    }
    chunk_bytes[t] = bytes;
    chunk_members[t] = members;
  });
  Py_DECREF(want);
  if (!nbo || std::find(chunk_ok.begin(), chunk_ok.end(), 0) != chunk_ok.end()) {
    Py_DECREF(fast);
    Py_RETURN_NONE;
  }
  size_t pool_bytes = 0;
  for (size_t b : chunk_bytes) pool_bytes += b;
  const size_t head = static_cast<size_t>(n) * 2 * sizeof(int64_t);
  const size_t total = head + pool_bytes;

  PyObject* out = nullptr;
  Py_buffer view{};
  bool have_view = false;
  char* dst = nullptr;
  if (alloc == Py_None) {
    out = PyByteArray_FromStringAndSize(nullptr, static_cast<Py_ssize_t>(total));
    if (out) dst = PyByteArray_AS_STRING(out);
  } else {
    out = PyObject_CallFunction(alloc, "n", static_cast<Py_ssize_t>(total));
    if (out && PyObject_GetBuffer(out, &view, PyBUF_WRITABLE | PyBUF_C_CONTIGUOUS) == 0) {
      have_view = true;
      if (static_cast<size_t>(view.len) < total) {
        PyErr_SetString(PyExc_ValueError, "alloc returned a buffer smaller than requested");
      } else {
        dst = static_cast<char*>(view.buf);
      }
    }
  }
  if (!dst) {
    if (have_view) PyBuffer_Release(&view);
    Py_XDECREF(out);
    Py_DECREF(fast);
    return nullptr;
  }
  int64_t* lens_out = reinterpret_cast<int64_t*>(dst);
  int64_t* starts_out = lens_out + n;
  char* pool = dst + head;
  std::vector<size_t> byte_base(static_cast<size_t>(threads), 0);
  std::vector<int64_t> member_base(static_cast<size_t>(threads), 0);
  for (int t = 1; t < threads; ++t) {
    byte_base[t] = byte_base[t - 1] + chunk_bytes[t - 1];
    member_base[t] = member_base[t - 1] + chunk_members[t - 1];
  }
  split(n, threads, [&](int t, Py_ssize_t b, Py_ssize_t e) {  // 2. lengths, starts and bytes
    char* p = pool + byte_base[t];
    int64_t at = member_base[t];
    for (Py_ssize_t i = b; i < e; ++i) {
      PyArrayObject* a = reinterpret_cast<PyArrayObject*>(items[i]);
      const size_t nb = static_cast<size_t>(PyArray_NBYTES(a));
      lens_out[i] = lengths[static_cast<size_t>(i)];
      starts_out[i] = at;
      at += lengths[static_cast<size_t>(i)];
      if (nb) std::memcpy(p, PyArray_DATA(a), nb);
      p += nb;
    }
  });
  if (have_view) PyBuffer_Release(&view);
  Py_DECREF(fast);
  return out;
}

// split_views(pool, bounds) -> [pool[bounds[i]:bounds[i+1]] for i in range(len(bounds) - 1)]
//   The inverse direction (Particle export, baselines.py:104-120): one view of a 1-D C-contiguous pool per
//   segment, made in C instead of one Python slice at a time. bounds: int64 array of n + 1 offsets.
PyObject* split_views(PyObject*, PyObject* args) {
  PyArrayObject* pool = nullptr;
  PyArrayObject* bounds = nullptr;
  if (!PyArg_ParseTuple(args, "O!O!", &PyArray_Type, &pool, &PyArray_Type, &bounds)) return nullptr;
  if (PyArray_NDIM(pool) != 1 || !PyArray_IS_C_CONTIGUOUS(pool) || PyArray_NDIM(bounds) != 1 ||
      PyArray_TYPE(bounds) != NPY_INT64 || !PyArray_IS_C_CONTIGUOUS(bounds)) {
    PyErr_SetString(PyExc_ValueError, "split_views needs a 1-D contiguous pool and int64 bounds");
    return nullptr;
  }
  const npy_intp nb = PyArray_DIM(bounds, 0);
  const npy_intp n = nb > 0 ? nb - 1 : 0;
  const int64_t* b = static_cast<const int64_t*>(PyArray_DATA(bounds));
  const npy_intp len = PyArray_DIM(pool, 0);
  for (npy_intp i = 0; i < n; ++i)
    if (b[i] < 0 || b[i] > b[i + 1] || b[i + 1] > len) {
      PyErr_SetString(PyExc_ValueError, "bounds out of order or past the pool");
      return nullptr;
    }
  PyObject* out = PyList_New(n);
  if (!out) return nullptr;
  PyArray_Descr* descr = PyArray_DESCR(pool);
  const npy_intp item = PyArray_ITEMSIZE(pool);
  char* data = static_cast<char*>(PyArray_DATA(pool));
  const int flags = PyArray_FLAGS(pool) & (NPY_ARRAY_WRITEABLE | NPY_ARRAY_ALIGNED);
  for (npy_intp i = 0; i < n; ++i) {
    npy_intp dim = static_cast<npy_intp>(b[i + 1] - b[i]);
    Py_INCREF(descr);  // stolen by NewFromDescr
    PyObject* v = PyArray_NewFromDescr(&PyArray_Type, descr, 1, &dim, nullptr, data + b[i] * item,
                                       flags | NPY_ARRAY_C_CONTIGUOUS, nullptr);
    if (!v) {
      Py_DECREF(out);
      return nullptr;
    }
    Py_INCREF(pool);
    if (PyArray_SetBaseObject(reinterpret_cast<PyArrayObject*>(v), reinterpret_cast<PyObject*>(pool)) < 0) {
      Py_DECREF(v);
      Py_DECREF(out);
      return nullptr;
    }
    PyList_SET_ITEM(out, i, v);
  }
  return out;
}

PyMethodDef kMethods[] = {
    {"pack_segments", pack_segments, METH_VARARGS,
     "pack_segments(segments, dtype, alloc=None) -> buffer [lengths i64 | starts i64 | pool], or None"},
    {"split_views", split_views, METH_VARARGS, "split_views(pool, bounds) -> list of views pool[b[i]:b[i+1]]"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_segpack", "host packing and splitting of jagged segments", -1,
                       kMethods};

}  // namespace

PyMODINIT_FUNC PyInit__segpack(void) {
  import_array();
  return PyModule_Create(&kModule);
}

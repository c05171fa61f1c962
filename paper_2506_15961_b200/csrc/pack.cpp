// pack.cpp -- CPython extension `_pqw_pack`: flattens a host Graph (the
// reference's dataflow-graph objects, paper_2506_15961_b200/graph.py) into the
// flat columns of pqw_graph_desc (include/planeq_witness.h) in one pass over
// the Python objects, without building intermediate Python lists.
//
// It is the C++ form of native.py's _pack_graph: same columns, same attribute
// encoding (documented in native.py), names as NUL-terminated UTF-8. Rational
// attributes (scale factor, shift addend, full value) are numbered through the
// caller's `const_id` callable so the plan's constant table stays in Python.
// Any attribute it cannot encode raises (KeyError/TypeError/ValueError); the
// caller then declines the plan to the Python host path, as the Python packer
// does.
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <structmember.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <unordered_map>

#include <sys/mman.h>
#include <thread>
#include <string>
#include <vector>

namespace {

// pqw_top opcodes (include/planeq_witness.h) of the kinds that carry attributes
enum : int {
  T_DIV = 19, T_SCALE = 23, T_SHIFT = 24, T_POW = 25, T_SOFTMAX = 29, T_CREATE_MASK = 30,
  T_VIEW = 32, T_TRANSPOSE = 33, T_EXPAND = 34, T_SUM = 35, T_MEAN = 36, T_EINSUM = 38,
  T_FULL = 39, T_CHUNK = 40, T_EMBEDDING_GRAD = 42, T_ALL_REDUCE = 44, T_ALL_GATHER = 45,
  T_REDUCE_SCATTER = 46, T_ALL_TO_ALL = 47
};

struct Err {};

PyObject* S_shape;
PyObject* S_dtype;
PyObject* S_meta;
PyObject* S_id;
PyObject* S_kind;
PyObject* S_inputs;
PyObject* S_outputs;
PyObject* S_attrs;
PyObject* S_device;
PyObject* S_seq;
PyObject* S_tensors;
PyObject* S_nodes;
PyObject* S_inputs_g;

// Attribute reads of one type: a slotted dataclass (graph.py Tensor / Node)
// keeps each field at a fixed offset (its member descriptor), read directly;
// anything else goes through PyObject_GetAttr.
struct Fields {
  PyTypeObject* type = nullptr;
  std::vector<Py_ssize_t> off;
  void bind(PyObject* obj, PyObject* const* names, size_t n) {
    type = Py_TYPE(obj);
    off.assign(n, -1);
    for (size_t i = 0; i < n; ++i) {
      PyObject* d = _PyType_Lookup(type, names[i]);  // borrowed
      if (d && Py_IS_TYPE(d, &PyMemberDescr_Type)) {
        PyMemberDef* m = ((PyMemberDescrObject*)d)->d_member;
        if (m->type == Py_T_OBJECT_EX) off[i] = m->offset;
      }
    }
  }
};

struct Ref {  // owned reference
  PyObject* p;
  explicit Ref(PyObject* o) : p(o) {
    if (!p) throw Err{};
  }
  ~Ref() { Py_XDECREF(p); }
  Ref(const Ref&) = delete;
  Ref& operator=(const Ref&) = delete;
};

struct Ref;
PyObject* field(PyObject* obj, Fields& f, size_t i, PyObject* const* names, size_t n) {
  if (Py_TYPE(obj) != f.type) f.bind(obj, names, n);
  if (f.off[i] >= 0) {
    PyObject* v = *reinterpret_cast<PyObject**>(reinterpret_cast<char*>(obj) + f.off[i]);
    if (v) {
      Py_INCREF(v);
      return v;
    }
  }
  return PyObject_GetAttr(obj, names[i]);
}

void put_str(std::string& out, PyObject* s) {
  Py_ssize_t n;
  const char* c = PyUnicode_AsUTF8AndSize(s, &n);
  if (!c) throw Err{};
  out.append(c, (size_t)n);
  out.push_back('\0');
}

long long as_int(PyObject* v) {  // int(v)
  Ref l(PyNumber_Long(v));
  long long x = PyLong_AsLongLong(l.p);
  if (x == -1 && PyErr_Occurred()) throw Err{};
  return x;
}

template <class T>
void put(std::string& out, T v) {
  out.append(reinterpret_cast<const char*>(&v), sizeof(T));
}

// interned attribute keys (no temporary string per lookup), created at module
// init so that worker threads only read the table
const char* const KEYS[] = {"factor", "addend", "value", "shape", "exponent", "den_positive",
                            "axis", "size", "perm", "vocab", "keepdims", "axes", "spec", "parts",
                            "index", "group", "split_axis", "concat_axis", "enum"};
constexpr size_t N_KEYS = sizeof(KEYS) / sizeof(KEYS[0]);
PyObject* KEY_OBJS[N_KEYS];

PyObject* key_obj_cached(const char* key) {
  for (size_t i = 0; i < N_KEYS; ++i)
    if (KEYS[i] == key || std::strcmp(KEYS[i], key) == 0) return KEY_OBJS[i];
  return nullptr;
}
PyObject* key_obj(const char* key) {
  PyObject* o = key_obj_cached(key);
  if (!o) {
    PyErr_Format(PyExc_KeyError, "%s", key);
    throw Err{};
  }
  return o;
}

// attrs[key] (borrowed), KeyError when absent
PyObject* item(PyObject* d, const char* key) {
  PyObject* k = key_obj(key);
  PyObject* v = PyDict_GetItemWithError(d, k);
  if (!v) {
    if (!PyErr_Occurred()) PyErr_SetObject(PyExc_KeyError, k);
    throw Err{};
  }
  return v;
}
PyObject* opt(PyObject* d, const char* key) {
  PyObject* v = PyDict_GetItemWithError(d, key_obj(key));
  if (!v && PyErr_Occurred()) throw Err{};
  return v;
}

void put_seq_ints(std::vector<long long>& w, PyObject* seq, bool with_len) {
  Ref f(PySequence_Fast(seq, "expected a sequence"));
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(f.p);
  if (with_len) w.push_back(n);
  PyObject** it = PySequence_Fast_ITEMS(f.p);
  for (Py_ssize_t i = 0; i < n; ++i) w.push_back(as_int(it[i]));
}

bool has_attrs(int k) {
  switch (k) {
    case T_SCALE: case T_SHIFT: case T_FULL: case T_POW: case T_DIV: case T_SOFTMAX:
    case T_CREATE_MASK: case T_TRANSPOSE: case T_VIEW: case T_EXPAND: case T_EMBEDDING_GRAD:
    case T_SUM: case T_MEAN: case T_EINSUM: case T_CHUNK: case T_ALL_REDUCE: case T_ALL_GATHER:
    case T_REDUCE_SCATTER: case T_ALL_TO_ALL:
      return true;
    default:
      return false;
  }
}

void encode(int k, PyObject* a, PyObject* const_id, std::vector<long long>& w) {
  auto cid = [&](const char* key) {
    Ref r(PyObject_CallOneArg(const_id, item(a, key)));
    w.push_back(as_int(r.p));
  };
  auto truth = [&](const char* key) {
    PyObject* v = opt(a, key);
    int t = v ? PyObject_IsTrue(v) : 0;
    if (t < 0) throw Err{};
    return t;
  };
  switch (k) {
    case T_SCALE: cid("factor"); return;
    case T_SHIFT: cid("addend"); return;
    case T_FULL: cid("value"); put_seq_ints(w, item(a, "shape"), true); return;
    case T_POW: {
      PyObject* v = opt(a, "exponent");
      w.push_back(v ? as_int(v) : 0);
      return;
    }
    case T_DIV: w.push_back(truth("den_positive")); return;
    case T_SOFTMAX: {
      PyObject* v = opt(a, "axis");
      w.push_back(v ? as_int(v) : -1);
      return;
    }
    case T_CREATE_MASK: w.push_back(as_int(item(a, "size"))); return;
    case T_TRANSPOSE: put_seq_ints(w, item(a, "perm"), false); return;
    case T_VIEW:
    case T_EXPAND: put_seq_ints(w, item(a, "shape"), true); return;
    case T_EMBEDDING_GRAD: w.push_back(as_int(item(a, "vocab"))); return;
    case T_SUM:
    case T_MEAN: {
      w.push_back(truth("keepdims"));
      PyObject* axes = opt(a, "axes");
      if (!axes || axes == Py_None) {
        w.push_back(0);
      } else {
        w.push_back(1);
        put_seq_ints(w, axes, true);
      }
      return;
    }
    case T_EINSUM: {
      PyObject* s = item(a, "spec");
      if (!PyUnicode_Check(s)) {
        PyErr_SetString(PyExc_TypeError, "einsum spec");
        throw Err{};
      }
      const Py_ssize_t n = PyUnicode_GET_LENGTH(s);
      w.push_back(n);
      const int kind = PyUnicode_KIND(s);
      const void* data = PyUnicode_DATA(s);
      for (Py_ssize_t i = 0; i < n; ++i) w.push_back((long long)PyUnicode_READ(kind, data, i));
      return;
    }
    case T_CHUNK:
      w.push_back(as_int(item(a, "axis")));
      w.push_back(as_int(item(a, "parts")));
      w.push_back(as_int(item(a, "index")));
      return;
    case T_ALL_REDUCE:
    case T_ALL_GATHER:
    case T_REDUCE_SCATTER:
    case T_ALL_TO_ALL: {
      const Py_ssize_t g = PyObject_Size(item(a, "group"));
      if (g < 0) throw Err{};
      w.push_back(g);
      if (k == T_ALL_GATHER || k == T_REDUCE_SCATTER) w.push_back(as_int(item(a, "axis")));
      if (k == T_ALL_TO_ALL) {
        w.push_back(as_int(item(a, "split_axis")));
        w.push_back(as_int(item(a, "concat_axis")));
      }
      return;
    }
    default:
      return;
  }
}

// ---- parallel fast path ------------------------------------------------------
// For the common case -- graph.py's slotted Tensor/Node objects holding exact
// small ints, compact-ASCII names, tuples/lists and dicts -- the per-object
// work runs on host threads while the calling thread keeps the GIL and
// waits: the workers only read (borrowed references, no refcount changes, no
// Python code, no exceptions). Anything else makes the fast path decline and
// the serial path below (which raises the proper Python errors) runs instead.
// Rational attributes are numbered afterwards, serially, in node order.

// Large buffers (the columns run to tens of MB): ask for transparent huge
// pages, so first touch costs one fault per 2 MB instead of per 4 KB.
void advise_huge(void* p, size_t n) {
  constexpr uintptr_t H = 2u << 20;
  if (n < 2 * H) return;
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + H - 1) & ~(H - 1);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + n) & ~(H - 1);
  if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
}

// Growable byte buffer on malloc/realloc: large blocks grow by remapping
// pages instead of copying them.
struct Buf {
  char* p = nullptr;
  size_t n = 0, cap = 0;
  Buf() = default;
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  ~Buf() { std::free(p); }
  void grow(size_t need) {
    size_t c = std::max<size_t>(4096, cap * 2);
    while (c < need) c *= 2;
    char* q = static_cast<char*>(std::realloc(p, c));
    if (!q) throw std::bad_alloc();
    p = q;
    cap = c;
    advise_huge(p, cap);
  }
  void append(const void* s, size_t k) {
    if (n + k > cap) grow(n + k);
    std::memcpy(p + n, s, k);
    n += k;
  }
  void push_back(char c) {
    if (n + 1 > cap) grow(n + 1);
    p[n++] = c;
  }
};

// the columns of pqw_graph_desc, in the order of the result dict
enum Col { C_TN, C_NDIM, C_DIMS, C_FLAGS, C_IDS, C_KIND, C_NIN, C_NOUT, C_INS, C_OUTS,
           C_NATTR, C_ATTRS, C_DEVICE, C_SEQ, NCOL };
const char* const COL_NAMES[NCOL] = {"tn",  "ndim", "dims", "flags", "ids",   "kind",   "nin",
                                     "nout", "ins", "outs", "nattr", "attrs", "device", "seq"};

struct Cols {  // one worker's share (a contiguous range of tensors and of nodes)
  Buf c[NCOL];
  std::vector<std::pair<size_t, PyObject*>> consts;  // (attr word index, value) to number
};

bool fast_str(PyObject* s, Buf& out) {
  if (!s || !PyUnicode_Check(s) || !PyUnicode_IS_COMPACT_ASCII(s)) return false;
  out.append(PyUnicode_DATA(s), (size_t)PyUnicode_GET_LENGTH(s) + 1);  // with its NUL
  return true;
}
bool fast_int(PyObject* o, long long& x) {
  if (!o || !PyLong_CheckExact(o) || !PyUnstable_Long_IsCompact((PyLongObject*)o)) return false;
  x = (long long)PyUnstable_Long_CompactValue((PyLongObject*)o);
  return true;
}
bool fast_seq(PyObject* o, PyObject** & it, Py_ssize_t& n) {
  if (o && PyTuple_CheckExact(o)) {
    it = &PyTuple_GET_ITEM(o, 0);
    n = PyTuple_GET_SIZE(o);
    return true;
  }
  if (o && PyList_CheckExact(o)) {
    it = PyList_GET_SIZE(o) ? &PyList_GET_ITEM(o, 0) : nullptr;
    n = PyList_GET_SIZE(o);
    return true;
  }
  return false;
}
bool fast_ints(PyObject* o, std::vector<long long>& w, bool with_len) {
  PyObject** it;
  Py_ssize_t n;
  if (!fast_seq(o, it, n)) return false;
  if (with_len) w.push_back(n);
  for (Py_ssize_t i = 0; i < n; ++i) {
    long long x;
    if (!fast_int(it[i], x)) return false;
    w.push_back(x);
  }
  return true;
}
PyObject* fast_get(PyObject* d, const char* key) {
  return PyDict_GetItemWithError(d, key_obj_cached(key));  // str keys: a read-only lookup
}
bool fast_ascii_eq(PyObject* s, const char* lit) {
  return s && PyUnicode_Check(s) && PyUnicode_IS_COMPACT_ASCII(s) &&
         std::strcmp((const char*)PyUnicode_DATA(s), lit) == 0;
}
bool fast_truth(PyObject* a, const char* key, long long& t) {
  PyObject* v = fast_get(a, key);
  if (!v || v == Py_None || v == Py_False) {
    t = 0;
    return true;
  }
  if (v == Py_True) {
    t = 1;
    return true;
  }
  long long x;
  if (!fast_int(v, x)) return false;
  t = x != 0;
  return true;
}

// fast_* form of encode(); rational attributes get a placeholder word and are
// queued in `cq` (word index within this part's attrs, value)
bool encode_fast(int k, PyObject* a, std::vector<long long>& w, size_t word0,
                 std::vector<std::pair<size_t, PyObject*>>& cq) {
  long long x;
  auto req_int = [&](const char* key) {
    long long v;
    if (!fast_int(fast_get(a, key), v)) return false;
    w.push_back(v);
    return true;
  };
  auto cst = [&](const char* key) {
    PyObject* v = fast_get(a, key);
    if (!v) return false;
    cq.push_back({word0 + w.size(), v});
    w.push_back(0);
    return true;
  };
  switch (k) {
    case T_SCALE: return cst("factor");
    case T_SHIFT: return cst("addend");
    case T_FULL: return cst("value") && fast_ints(fast_get(a, "shape"), w, true);
    case T_POW: {
      PyObject* v = fast_get(a, "exponent");
      if (!v) {
        w.push_back(0);
        return true;
      }
      if (!fast_int(v, x)) return false;
      w.push_back(x);
      return true;
    }
    case T_DIV:
      if (!fast_truth(a, "den_positive", x)) return false;
      w.push_back(x);
      return true;
    case T_SOFTMAX: {
      PyObject* v = fast_get(a, "axis");
      if (!v) {
        w.push_back(-1);
        return true;
      }
      if (!fast_int(v, x)) return false;
      w.push_back(x);
      return true;
    }
    case T_CREATE_MASK: return req_int("size");
    case T_TRANSPOSE: return fast_ints(fast_get(a, "perm"), w, false);
    case T_VIEW:
    case T_EXPAND: return fast_ints(fast_get(a, "shape"), w, true);
    case T_EMBEDDING_GRAD: return req_int("vocab");
    case T_SUM:
    case T_MEAN: {
      if (!fast_truth(a, "keepdims", x)) return false;
      w.push_back(x);
      PyObject* axes = fast_get(a, "axes");
      if (!axes || axes == Py_None) {
        w.push_back(0);
        return true;
      }
      w.push_back(1);
      return fast_ints(axes, w, true);
    }
    case T_EINSUM: {
      PyObject* sp = fast_get(a, "spec");
      if (!sp || !PyUnicode_Check(sp) || !PyUnicode_IS_COMPACT_ASCII(sp)) return false;
      const Py_ssize_t n = PyUnicode_GET_LENGTH(sp);
      const char* c = (const char*)PyUnicode_DATA(sp);
      w.push_back(n);
      for (Py_ssize_t i = 0; i < n; ++i) w.push_back((unsigned char)c[i]);
      return true;
    }
    case T_CHUNK: return req_int("axis") && req_int("parts") && req_int("index");
    case T_ALL_REDUCE:
    case T_ALL_GATHER:
    case T_REDUCE_SCATTER:
    case T_ALL_TO_ALL: {
      PyObject** it;
      Py_ssize_t g;
      if (!fast_seq(fast_get(a, "group"), it, g)) return false;
      w.push_back(g);
      if (k == T_ALL_GATHER || k == T_REDUCE_SCATTER) return req_int("axis");
      if (k == T_ALL_TO_ALL) return req_int("split_axis") && req_int("concat_axis");
      return true;
    }
    default:
      return true;
  }
}

PyObject* bytes_of(const std::string& s) {
  return PyBytes_FromStringAndSize(s.data(), (Py_ssize_t)s.size());
}

struct KindTable {
  std::vector<std::pair<std::string, int>> kv;
  int find(PyObject* s) const {
    if (!s || !PyUnicode_Check(s) || !PyUnicode_IS_COMPACT_ASCII(s)) return -2;
    const char* c = (const char*)PyUnicode_DATA(s);
    for (auto& e : kv)
      if (e.first == c) return e.second;
    return -1;
  }
};

// per-worker memo of kind strings by object identity (the plan's kind
// strings are a handful of shared objects)
struct KindMemo {
  PyObject* key[64] = {};
  int val[64] = {};
  int find(const KindTable& kt, PyObject* s) {
    const size_t h = (reinterpret_cast<uintptr_t>(s) >> 4) & 63u;
    if (s && key[h] == s) return val[h];
    const int v = kt.find(s);
    if (v >= -1) {
      key[h] = s;
      val[h] = v;
    }
    return v;
  }
};

template <class T>
void putv(Buf& out, T v) {
  out.append(reinterpret_cast<const char*>(&v), sizeof(T));
}

// PQW_TIMING=1: phase times on stderr
void lap(const char* what) {
  static const bool on = getenv("PQW_TIMING") != nullptr;
  static auto t0 = std::chrono::steady_clock::now();
  if (!on) return;
  const auto t = std::chrono::steady_clock::now();
  fprintf(stderr, "PQW_TIMING pack %s %.1f ms\n", what,
          std::chrono::duration<double, std::milli>(t - t0).count());
  t0 = t;
}

unsigned pack_threads(size_t work) {
  unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (const char* e = getenv("PQW_THREADS")) nt = (unsigned)std::max(1, std::min(16, atoi(e)));
  return work < 50000 ? 1u : nt;
}

template <class F>
void on_threads(unsigned nt, F&& f) {
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < nt; ++t) pool.emplace_back(f, t);
  f(0u);
  for (auto& th : pool) th.join();
}

bool pack_fast(PyObject* tensors, PyObject* const* nodes, Py_ssize_t nn, const KindTable& kinds,
               std::vector<Cols>& parts) {
  std::vector<std::pair<PyObject*, PyObject*>> tv;
  tv.reserve((size_t)PyDict_GET_SIZE(tensors));
  {
    Py_ssize_t pos = 0;
    PyObject *k, *v;
    while (PyDict_Next(tensors, &pos, &k, &v)) tv.push_back({k, v});
  }
  lap("tensor list");
  PyObject* const tnames[3] = {S_shape, S_dtype, S_meta};
  PyObject* const nnames[7] = {S_id, S_kind, S_inputs, S_outputs, S_attrs, S_device, S_seq};
  Fields tf, nf;
  if (!tv.empty()) {
    tf.bind(tv[0].second, tnames, 3);
    for (auto o : tf.off)
      if (o < 0) return false;
  }
  if (nn) {
    nf.bind(nodes[0], nnames, 7);
    for (auto o : nf.off)
      if (o < 0) return false;
  }
  auto slot = [](PyObject* obj, const Fields& f, int i) {
    return *reinterpret_cast<PyObject**>(reinterpret_cast<char*>(obj) + f.off[i]);
  };
  const unsigned nt = pack_threads(tv.size() + (size_t)nn);
  parts = std::vector<Cols>(nt);
  std::vector<char> ok(nt, 1);
  auto run = [&](unsigned t) {
    Cols& c = parts[t];
    std::vector<long long> sh, w;
    KindMemo memo;
    const size_t t0 = tv.size() * t / nt, t1 = tv.size() * (t + 1) / nt;
    for (size_t i = t0; i < t1 && ok[t]; ++i) {
      PyObject* o = tv[i].second;
      sh.clear();
      if (Py_TYPE(o) != tf.type || !fast_str(tv[i].first, c.c[C_TN]) ||
          !fast_ints(slot(o, tf, 0), sh, false)) {
        ok[t] = 0;
        break;
      }
      putv<int32_t>(c.c[C_NDIM], (int32_t)sh.size());
      c.c[C_DIMS].append(sh.data(), sh.size() * sizeof(int64_t));
      uint8_t fl = 0;
      if (fast_ascii_eq(slot(o, tf, 1), "int")) {
        fl = 1;
        PyObject* meta = slot(o, tf, 2);
        if (!meta || !PyDict_CheckExact(meta)) {
          ok[t] = 0;
          break;
        }
        if (fast_ascii_eq(fast_get(meta, "enum"), "position")) fl |= 2;
      }
      c.c[C_FLAGS].push_back((char)fl);
    }
    const size_t n0 = (size_t)nn * t / nt, n1 = (size_t)nn * (t + 1) / nt;
    size_t words = 0;
    for (size_t i = n0; i < n1 && ok[t]; ++i) {
      PyObject* n = nodes[i];
      bool good = Py_TYPE(n) == nf.type && fast_str(slot(n, nf, 0), c.c[C_IDS]);
      const int k = good ? memo.find(kinds, slot(n, nf, 1)) : -2;
      good = good && k >= -1;
      PyObject** it = nullptr;
      Py_ssize_t ni = 0, no = 0;
      good = good && fast_seq(slot(n, nf, 2), it, ni);
      for (Py_ssize_t j = 0; good && j < ni; ++j) good = fast_str(it[j], c.c[C_INS]);
      good = good && fast_seq(slot(n, nf, 3), it, no);
      for (Py_ssize_t j = 0; good && j < no; ++j) good = fast_str(it[j], c.c[C_OUTS]);
      w.clear();
      if (good && has_attrs(k)) {
        PyObject* at = slot(n, nf, 4);
        good = at && PyDict_CheckExact(at) && encode_fast(k, at, w, words, c.consts);
      }
      long long dv = -1, sq = 0;
      PyObject* dvo = good ? slot(n, nf, 5) : nullptr;
      good = good && dvo && (dvo == Py_None || fast_int(dvo, dv));
      good = good && fast_int(slot(n, nf, 6), sq);
      if (!good) {
        ok[t] = 0;
        break;
      }
      putv<int32_t>(c.c[C_KIND], k);
      putv<int32_t>(c.c[C_NIN], (int32_t)ni);
      putv<int32_t>(c.c[C_NOUT], (int32_t)no);
      putv<int32_t>(c.c[C_NATTR], (int32_t)w.size());
      c.c[C_ATTRS].append(w.data(), w.size() * sizeof(int64_t));
      words += w.size();
      putv<int32_t>(c.c[C_DEVICE], (int32_t)dv);
      putv<int64_t>(c.c[C_SEQ], sq);
    }
  };
  on_threads(nt, [&](unsigned t) {
    try {
      run(t);
    } catch (...) {  // out of memory: let the serial path raise
      ok[t] = 0;
    }
  });
  lap("workers");
  for (char o : ok)
    if (!o) return false;
  return true;
}

// The workers' shares, concatenated straight into new bytes objects (one
// parallel copy, pages first touched on the workers); rational attributes
// then numbered through const_id in node order. Returns false with a Python
// error set.
bool gather_parts(std::vector<Cols>& parts, PyObject* const_id, PyObject* out[NCOL]) {
  const size_t nt = parts.size();
  std::vector<size_t> off((nt + 1) * NCOL, 0);
  for (int k = 0; k < NCOL; ++k)
    for (size_t t = 0; t < nt; ++t) off[(t + 1) * NCOL + k] = off[t * NCOL + k] + parts[t].c[k].n;
  for (int k = 0; k < NCOL; ++k) {
    out[k] = PyBytes_FromStringAndSize(nullptr, (Py_ssize_t)off[nt * NCOL + k]);
    if (!out[k]) return false;
  }
  char* dst[NCOL];
  for (int k = 0; k < NCOL; ++k) {
    dst[k] = PyBytes_AS_STRING(out[k]);
    advise_huge(dst[k], (size_t)PyBytes_GET_SIZE(out[k]));
  }
  on_threads((unsigned)nt, [&](unsigned t) {
    for (int k = 0; k < NCOL; ++k)
      if (parts[t].c[k].n) std::memcpy(dst[k] + off[t * NCOL + k], parts[t].c[k].p, parts[t].c[k].n);
  });
  lap("gather");
  // const_id is a function of the exact value: memoise it per exact int /
  // float value, per (numerator, denominator) for a Fraction whose terms fit
  // in 64 bits (every node carries its own Fraction object), and per object
  // for anything else (numpy scalars, big fractions)
  struct Key {
    uint64_t tag, bits, bits2;
    bool operator==(const Key& o) const { return tag == o.tag && bits == o.bits && bits2 == o.bits2; }
  };
  struct KeyHash {
    size_t operator()(const Key& k) const {
      return std::hash<uint64_t>()((k.bits * 0x9E3779B97F4A7C15ull ^ k.bits2) * 0xBF58476D1CE4E5B9ull ^ k.tag);
    }
  };
  static PyObject* S_num = PyUnicode_InternFromString("_numerator");
  static PyObject* S_den = PyUnicode_InternFromString("_denominator");
  PyTypeObject* fraction_type = nullptr;  // the first type seen with both slots
  std::unordered_map<Key, int64_t, KeyHash> memo;
  for (size_t t = 0; t < nt; ++t) {
    const size_t word0 = off[t * NCOL + C_ATTRS] / sizeof(int64_t);
    for (auto& q : parts[t].consts) {
      PyObject* v = q.second;
      Key key{3, reinterpret_cast<uintptr_t>(v), 0};
      long long x;
      if (PyFloat_CheckExact(v)) {
        const double d = PyFloat_AS_DOUBLE(v);
        key = {1, 0, 0};
        std::memcpy(&key.bits, &d, sizeof(d));
      } else if (fast_int(v, x)) {
        key = {2, static_cast<uint64_t>(x), 0};
      } else if (!PyLong_Check(v) && (fraction_type == nullptr || Py_TYPE(v) == fraction_type)) {
        PyObject* nu = PyObject_GetAttr(v, S_num);
        PyObject* de = nu ? PyObject_GetAttr(v, S_den) : nullptr;
        long long a, b;
        if (nu && de && fast_int(nu, a) && fast_int(de, b) && b > 0) {
          fraction_type = Py_TYPE(v);
          key = {4, static_cast<uint64_t>(a), static_cast<uint64_t>(b)};
        }
        Py_XDECREF(nu);
        Py_XDECREF(de);
        PyErr_Clear();
      }
      auto it = memo.find(key);
      int64_t id;
      if (it != memo.end()) {
        id = it->second;
      } else {
        PyObject* r = PyObject_CallOneArg(const_id, v);
        if (!r) return false;
        id = PyLong_AsLongLong(r);
        Py_DECREF(r);
        if (id == -1 && PyErr_Occurred()) return false;
        memo.emplace(key, id);
      }
      std::memcpy(dst[C_ATTRS] + (word0 + q.first) * sizeof(int64_t), &id, sizeof(id));
    }
  }
  lap("constants");
  return true;
}

// pack_graph(graph, opcodes: dict[str, int], const_id) -> dict[str, bytes]
PyObject* pack_graph(PyObject*, PyObject* args) {
  PyObject *g, *opcodes, *const_id;
  if (!PyArg_ParseTuple(args, "OO!O", &g, &PyDict_Type, &opcodes, &const_id)) return nullptr;
  PyObject* cols[NCOL] = {};
  lap("start");
  auto release = [&] {
    for (auto& o : cols) Py_CLEAR(o);
  };
  try {
    Ref tensors(PyObject_GetAttr(g, S_tensors));
    if (!PyDict_Check(tensors.p)) {
      PyErr_SetString(PyExc_TypeError, "graph.tensors is not a dict");
      throw Err{};
    }
    Ref nodes_o(PyObject_GetAttr(g, S_nodes));
    Ref nodes(PySequence_Fast(nodes_o.p, "graph.nodes"));
    const Py_ssize_t nn = PySequence_Fast_GET_SIZE(nodes.p);
    PyObject** nv = PySequence_Fast_ITEMS(nodes.p);
    long long nt = PyDict_GET_SIZE(tensors.p);
    bool fast = false;
    if (!getenv("PQW_PACK_SERIAL")) {
      KindTable kt;
      Py_ssize_t pos = 0;
      PyObject *kk, *vv;
      bool tab_ok = true;
      while (PyDict_Next(opcodes, &pos, &kk, &vv)) {
        long long c;
        if (!PyUnicode_Check(kk) || !PyUnicode_IS_COMPACT_ASCII(kk) || !fast_int(vv, c)) {
          tab_ok = false;
          break;
        }
        kt.kv.push_back({std::string((const char*)PyUnicode_DATA(kk)), (int)c});
      }
      std::vector<Cols> parts;
      if (tab_ok && pack_fast(tensors.p, nv, nn, kt, parts)) {
        if (!gather_parts(parts, const_id, cols)) throw Err{};
        fast = true;
      }
    }
    if (!fast) {
    std::string c[NCOL];
    nt = 0;
    Py_ssize_t pos = 0;
    PyObject *key, *t;
    PyObject* const tnames[3] = {S_shape, S_dtype, S_meta};
    Fields tf;
    while (PyDict_Next(tensors.p, &pos, &key, &t)) {
      put_str(c[C_TN], key);
      Ref shape(field(t, tf, 0, tnames, 3));
      Ref f(PySequence_Fast(shape.p, "shape"));
      const Py_ssize_t r = PySequence_Fast_GET_SIZE(f.p);
      put<int32_t>(c[C_NDIM], (int32_t)r);
      PyObject** it = PySequence_Fast_ITEMS(f.p);
      for (Py_ssize_t i = 0; i < r; ++i) put<int64_t>(c[C_DIMS], as_int(it[i]));
      Ref dt(field(t, tf, 1, tnames, 3));
      uint8_t fl = 0;
      if (PyUnicode_Check(dt.p) && PyUnicode_CompareWithASCIIString(dt.p, "int") == 0) {
        fl = 1;
        Ref meta(field(t, tf, 2, tnames, 3));
        PyObject* en = PyDict_Check(meta.p) ? opt(meta.p, "enum") : nullptr;
        if (en && PyUnicode_Check(en) && PyUnicode_CompareWithASCIIString(en, "position") == 0)
          fl |= 2;
      }
      c[C_FLAGS].push_back((char)fl);
      ++nt;
    }
    std::vector<long long> w;
    PyObject* const nnames[7] = {S_id, S_kind, S_inputs, S_outputs, S_attrs, S_device, S_seq};
    Fields nf;
    for (Py_ssize_t i = 0; i < nn; ++i) {
      PyObject* n = nv[i];
      Ref id(field(n, nf, 0, nnames, 7));
      put_str(c[C_IDS], id.p);
      Ref kd(field(n, nf, 1, nnames, 7));
      PyObject* code = PyDict_GetItem(opcodes, kd.p);
      const int k = code ? (int)PyLong_AsLong(code) : -1;
      put<int32_t>(c[C_KIND], k);
      Ref in(field(n, nf, 2, nnames, 7));
      Ref inf(PySequence_Fast(in.p, "inputs"));
      const Py_ssize_t ni = PySequence_Fast_GET_SIZE(inf.p);
      for (Py_ssize_t j = 0; j < ni; ++j) put_str(c[C_INS], PySequence_Fast_GET_ITEM(inf.p, j));
      put<int32_t>(c[C_NIN], (int32_t)ni);
      Ref out(field(n, nf, 3, nnames, 7));
      Ref outf(PySequence_Fast(out.p, "outputs"));
      const Py_ssize_t no = PySequence_Fast_GET_SIZE(outf.p);
      for (Py_ssize_t j = 0; j < no; ++j) put_str(c[C_OUTS], PySequence_Fast_GET_ITEM(outf.p, j));
      put<int32_t>(c[C_NOUT], (int32_t)no);
      w.clear();
      if (has_attrs(k)) {
        Ref at(field(n, nf, 4, nnames, 7));
        if (!PyDict_Check(at.p)) {
          PyErr_SetString(PyExc_TypeError, "node attrs is not a dict");
          throw Err{};
        }
        encode(k, at.p, const_id, w);
      }
      put<int32_t>(c[C_NATTR], (int32_t)w.size());
      for (long long x : w) put<int64_t>(c[C_ATTRS], x);
      Ref dv(field(n, nf, 5, nnames, 7));
      put<int32_t>(c[C_DEVICE], dv.p == Py_None ? -1 : (int32_t)as_int(dv.p));
      Ref sq(field(n, nf, 6, nnames, 7));
      put<int64_t>(c[C_SEQ], as_int(sq.p));
    }
    for (int k = 0; k < NCOL; ++k)
      if (!(cols[k] = bytes_of(c[k]))) throw Err{};
    }  // serial path
    std::string gin;
    Ref gi(PyObject_GetAttr(g, S_inputs_g));
    Ref gif(PySequence_Fast(gi.p, "graph.inputs"));
    const Py_ssize_t ng = PySequence_Fast_GET_SIZE(gif.p);
    for (Py_ssize_t j = 0; j < ng; ++j) put_str(gin, PySequence_Fast_GET_ITEM(gif.p, j));
    Ref d(PyDict_New());
    for (int k = 0; k < NCOL; ++k)
      if (PyDict_SetItemString(d.p, COL_NAMES[k], cols[k]) < 0) throw Err{};
    Ref gb(bytes_of(gin));
    if (PyDict_SetItemString(d.p, "inputs", gb.p) < 0) throw Err{};
    Ref cnt(Py_BuildValue("(LnL)", nt, nn, (long long)ng));
    if (PyDict_SetItemString(d.p, "counts", cnt.p) < 0) throw Err{};
    release();
    lap("dict");
    Py_INCREF(d.p);
    return d.p;
  } catch (const Err&) {
    release();
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "graph not packable");
    return nullptr;
  }
}

// pack_lineage(lineage: dict[str, LineageEntry]) -> dict[str, bytes]: the
// columns of pqw_lineage_desc (native.py _pack_lineage): entry names (the
// dict keys), mode (0 full, 1 partial, 2 other), shards per entry, shard
// tensor names, dims per shard, (lo, hi) per dim.
PyObject* pack_lineage(PyObject*, PyObject* args) {
  PyObject* lin;
  if (!PyArg_ParseTuple(args, "O!", &PyDict_Type, &lin)) return nullptr;
  try {
    std::string names, mode, nsh, snames, sdim, ranges;
    Ref s_mode(PyUnicode_InternFromString("mode"));
    Ref s_shards(PyUnicode_InternFromString("shards"));
    Ref s_tensor(PyUnicode_InternFromString("tensor"));
    Ref s_ranges(PyUnicode_InternFromString("ranges"));
    Py_ssize_t pos = 0;
    PyObject *key, *e;
    while (PyDict_Next(lin, &pos, &key, &e)) {
      put_str(names, key);
      Ref m(PyObject_GetAttr(e, s_mode.p));
      char md = 2;
      if (PyUnicode_Check(m.p)) {
        if (PyUnicode_CompareWithASCIIString(m.p, "full") == 0) md = 0;
        else if (PyUnicode_CompareWithASCIIString(m.p, "partial") == 0) md = 1;
      }
      mode.push_back(md);
      Ref sh(PyObject_GetAttr(e, s_shards.p));
      Ref shf(PySequence_Fast(sh.p, "shards"));
      const Py_ssize_t ns = PySequence_Fast_GET_SIZE(shf.p);
      put<int32_t>(nsh, (int32_t)ns);
      for (Py_ssize_t i = 0; i < ns; ++i) {
        PyObject* s = PySequence_Fast_GET_ITEM(shf.p, i);
        Ref t(PyObject_GetAttr(s, s_tensor.p));
        put_str(snames, t.p);
        Ref r(PyObject_GetAttr(s, s_ranges.p));
        Ref rf(PySequence_Fast(r.p, "ranges"));
        const Py_ssize_t nd = PySequence_Fast_GET_SIZE(rf.p);
        put<int32_t>(sdim, (int32_t)nd);
        for (Py_ssize_t d = 0; d < nd; ++d) {
          Ref pr(PySequence_Fast(PySequence_Fast_GET_ITEM(rf.p, d), "range"));
          const Py_ssize_t k = PySequence_Fast_GET_SIZE(pr.p);
          for (Py_ssize_t j = 0; j < k; ++j)
            put<int64_t>(ranges, as_int(PySequence_Fast_GET_ITEM(pr.p, j)));
        }
      }
    }
    Ref d(PyDict_New());
    const std::pair<const char*, std::string*> cols[] = {
        {"names", &names}, {"mode", &mode}, {"n_shards", &nsh},
        {"shard_names", &snames}, {"sdim", &sdim}, {"ranges", &ranges}};
    for (auto& c : cols) {
      Ref b(bytes_of(*c.second));
      if (PyDict_SetItemString(d.p, c.first, b.p) < 0) throw Err{};
    }
    Py_INCREF(d.p);
    return d.p;
  } catch (const Err&) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "lineage not packable");
    return nullptr;
  }
}

PyMethodDef methods[] = {
    {"pack_graph", pack_graph, METH_VARARGS,
     "pack_graph(graph, opcodes, const_id) -> dict of flat columns (pqw_graph_desc)"},
    {"pack_lineage", pack_lineage, METH_VARARGS,
     "pack_lineage(lineage) -> dict of flat columns (pqw_lineage_desc)"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pqw_pack",
                      "Flattening of host graphs for the native plan core.", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__pqw_pack(void) {
  S_shape = PyUnicode_InternFromString("shape");
  S_dtype = PyUnicode_InternFromString("dtype");
  S_meta = PyUnicode_InternFromString("meta");
  S_id = PyUnicode_InternFromString("id");
  S_kind = PyUnicode_InternFromString("kind");
  S_inputs = PyUnicode_InternFromString("inputs");
  S_outputs = PyUnicode_InternFromString("outputs");
  S_attrs = PyUnicode_InternFromString("attrs");
  S_device = PyUnicode_InternFromString("device");
  S_seq = PyUnicode_InternFromString("seq");
  S_tensors = PyUnicode_InternFromString("tensors");
  S_nodes = PyUnicode_InternFromString("nodes");
  S_inputs_g = PyUnicode_InternFromString("inputs");
  for (size_t i = 0; i < N_KEYS; ++i) {
    KEY_OBJS[i] = PyUnicode_InternFromString(KEYS[i]);
    if (!KEY_OBJS[i]) return nullptr;
    (void)PyObject_Hash(KEY_OBJS[i]);  // cache the hash before any worker reads it
  }
  return PyModule_Create(&module);
}

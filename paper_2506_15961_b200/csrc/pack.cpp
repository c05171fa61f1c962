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

#include <cstdint>
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

// interned attribute keys (no temporary string per lookup)
PyObject* key_obj(const char* key) {
  static std::vector<std::pair<const char*, PyObject*>> cache;
  for (auto& kv : cache)
    if (kv.first == key) return kv.second;
  PyObject* o = PyUnicode_InternFromString(key);
  if (!o) throw Err{};
  cache.push_back({key, o});
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

PyObject* bytes_of(const std::string& s) {
  return PyBytes_FromStringAndSize(s.data(), (Py_ssize_t)s.size());
}

// pack_graph(graph, opcodes: dict[str, int], const_id) -> dict[str, bytes]
PyObject* pack_graph(PyObject*, PyObject* args) {
  PyObject *g, *opcodes, *const_id;
  if (!PyArg_ParseTuple(args, "OO!O", &g, &PyDict_Type, &opcodes, &const_id)) return nullptr;
  try {
    std::string tn, ndim, dims, flags;
    Ref tensors(PyObject_GetAttr(g, S_tensors));
    if (!PyDict_Check(tensors.p)) {
      PyErr_SetString(PyExc_TypeError, "graph.tensors is not a dict");
      throw Err{};
    }
    Py_ssize_t pos = 0;
    PyObject *key, *t;
    long long nt = 0;
    PyObject* const tnames[3] = {S_shape, S_dtype, S_meta};
    Fields tf;
    while (PyDict_Next(tensors.p, &pos, &key, &t)) {
      put_str(tn, key);
      Ref shape(field(t, tf, 0, tnames, 3));
      Ref f(PySequence_Fast(shape.p, "shape"));
      const Py_ssize_t r = PySequence_Fast_GET_SIZE(f.p);
      put<int32_t>(ndim, (int32_t)r);
      PyObject** it = PySequence_Fast_ITEMS(f.p);
      for (Py_ssize_t i = 0; i < r; ++i) put<int64_t>(dims, as_int(it[i]));
      Ref dt(field(t, tf, 1, tnames, 3));
      uint8_t fl = 0;
      if (PyUnicode_Check(dt.p) && PyUnicode_CompareWithASCIIString(dt.p, "int") == 0) {
        fl = 1;
        Ref meta(field(t, tf, 2, tnames, 3));
        PyObject* en = PyDict_Check(meta.p) ? opt(meta.p, "enum") : nullptr;
        if (en && PyUnicode_Check(en) && PyUnicode_CompareWithASCIIString(en, "position") == 0)
          fl |= 2;
      }
      flags.push_back((char)fl);
      ++nt;
    }
    Ref nodes_o(PyObject_GetAttr(g, S_nodes));
    Ref nodes(PySequence_Fast(nodes_o.p, "graph.nodes"));
    const Py_ssize_t nn = PySequence_Fast_GET_SIZE(nodes.p);
    PyObject** nv = PySequence_Fast_ITEMS(nodes.p);
    std::string ids, kind, nin, nout, ins, outs, nattr, attrs, device, seq;
    std::vector<long long> w;
    PyObject* const nnames[7] = {S_id, S_kind, S_inputs, S_outputs, S_attrs, S_device, S_seq};
    Fields nf;
    for (Py_ssize_t i = 0; i < nn; ++i) {
      PyObject* n = nv[i];
      Ref id(field(n, nf, 0, nnames, 7));
      put_str(ids, id.p);
      Ref kd(field(n, nf, 1, nnames, 7));
      PyObject* code = PyDict_GetItem(opcodes, kd.p);
      const int k = code ? (int)PyLong_AsLong(code) : -1;
      put<int32_t>(kind, k);
      Ref in(field(n, nf, 2, nnames, 7));
      Ref inf(PySequence_Fast(in.p, "inputs"));
      const Py_ssize_t ni = PySequence_Fast_GET_SIZE(inf.p);
      for (Py_ssize_t j = 0; j < ni; ++j) put_str(ins, PySequence_Fast_GET_ITEM(inf.p, j));
      put<int32_t>(nin, (int32_t)ni);
      Ref out(field(n, nf, 3, nnames, 7));
      Ref outf(PySequence_Fast(out.p, "outputs"));
      const Py_ssize_t no = PySequence_Fast_GET_SIZE(outf.p);
      for (Py_ssize_t j = 0; j < no; ++j) put_str(outs, PySequence_Fast_GET_ITEM(outf.p, j));
      put<int32_t>(nout, (int32_t)no);
      w.clear();
      if (has_attrs(k)) {
        Ref at(field(n, nf, 4, nnames, 7));
        if (!PyDict_Check(at.p)) {
          PyErr_SetString(PyExc_TypeError, "node attrs is not a dict");
          throw Err{};
        }
        encode(k, at.p, const_id, w);
      }
      put<int32_t>(nattr, (int32_t)w.size());
      for (long long x : w) put<int64_t>(attrs, x);
      Ref dv(field(n, nf, 5, nnames, 7));
      put<int32_t>(device, dv.p == Py_None ? -1 : (int32_t)as_int(dv.p));
      Ref sq(field(n, nf, 6, nnames, 7));
      put<int64_t>(seq, as_int(sq.p));
    }
    std::string gin;
    Ref gi(PyObject_GetAttr(g, S_inputs_g));
    Ref gif(PySequence_Fast(gi.p, "graph.inputs"));
    const Py_ssize_t ng = PySequence_Fast_GET_SIZE(gif.p);
    for (Py_ssize_t j = 0; j < ng; ++j) put_str(gin, PySequence_Fast_GET_ITEM(gif.p, j));
    PyObject* d = PyDict_New();
    if (!d) throw Err{};
    auto set = [&](const char* k, const std::string& v) {
      PyObject* b = bytes_of(v);
      if (!b || PyDict_SetItemString(d, k, b) < 0) {
        Py_XDECREF(b);
        throw Err{};
      }
      Py_DECREF(b);
    };
    try {
      set("tn", tn); set("ndim", ndim); set("dims", dims); set("flags", flags);
      set("ids", ids); set("kind", kind); set("nin", nin); set("nout", nout);
      set("ins", ins); set("outs", outs); set("nattr", nattr); set("attrs", attrs);
      set("device", device); set("seq", seq); set("inputs", gin);
      PyObject* cnt = Py_BuildValue("(LnL)", nt, nn, (long long)ng);
      if (!cnt || PyDict_SetItemString(d, "counts", cnt) < 0) {
        Py_XDECREF(cnt);
        throw Err{};
      }
      Py_DECREF(cnt);
    } catch (const Err&) {
      Py_DECREF(d);
      throw;
    }
    return d;
  } catch (const Err&) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "graph not packable");
    return nullptr;
  }
}

PyMethodDef methods[] = {
    {"pack_graph", pack_graph, METH_VARARGS,
     "pack_graph(graph, opcodes, const_id) -> dict of flat columns (pqw_graph_desc)"},
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
  return PyModule_Create(&module);
}

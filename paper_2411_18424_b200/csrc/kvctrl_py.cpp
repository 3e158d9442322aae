// _kvctrl — CPython binding of the native control plane (ctrlplane.cpp).
//
// The same C++ pool and store that libkvctrl.so exports through the C ABI
// (include/kvctrl.h), bound with METH_FASTCALL module functions so a
// control-plane call from the engine costs ~0.1 µs of binding instead of the
// ~2 µs of a ctypes call — the engine makes 4-5 pool calls per iteration
// (set_request_fill, owned_blocks, ...), so the binding, not the C++, would
// otherwise dominate.  Handles are PyCapsules; results are Python ints,
// tuples and lists.  paper_2411_18424_b200/native_ctrl.py wraps these in the
// reference's classes.

#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include "ctrlplane.cpp"  // one translation unit: the pool / store internals

namespace {

constexpr int kErrCallback = -20;  // a Python rank_of callback raised
const char* kPoolCap = "kvctrl.pool";
const char* kStoreCap = "kvctrl.store";

PyObject* g_exc[32];  // indexed by -code - 10

struct PoolBox {
  KvcPool* pool;
  bool owned;
  PyObject* rank_fn;  // strong ref or nullptr
  PyObject* keep;     // store capsule keeping a borrowed pool alive
};

int64_t rank_trampoline(void* ctx, int64_t req) {
  PyObject* fn = static_cast<PyObject*>(ctx);
  PyObject* arg = PyLong_FromLongLong(req);
  PyObject* r = arg ? PyObject_CallOneArg(fn, arg) : nullptr;
  Py_XDECREF(arg);
  if (r == nullptr) throw Err{kErrCallback, "rank_of raised"};
  const long long v = PyLong_AsLongLong(r);
  Py_DECREF(r);
  if (v == -1 && PyErr_Occurred()) throw Err{kErrCallback, "rank_of returned a non-int"};
  return v;
}

PyObject* raise(const Err& e) {
  if (e.code == kErrCallback) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_RuntimeError, e.msg.c_str());
    return nullptr;
  }
  const int idx = -e.code - 10;
  PyObject* cls = (idx >= 0 && idx < 32 && g_exc[idx]) ? g_exc[idx] : PyExc_RuntimeError;
  if (cls == PyExc_KeyError) {
    PyObject* k = PyUnicode_FromString(e.msg.c_str());
    PyErr_SetObject(cls, k);
    Py_XDECREF(k);
  } else {
    PyErr_SetString(cls, e.msg.c_str());
  }
  return nullptr;
}

template <typename F>
PyObject* guarded(F&& f) {
  try {
    return f();
  } catch (const Err& e) {
    return raise(e);
  } catch (const std::bad_alloc&) {
    return PyErr_NoMemory();
  }
}

void pool_cap_free(PyObject* cap) {
  auto* b = static_cast<PoolBox*>(PyCapsule_GetPointer(cap, kPoolCap));
  if (b == nullptr) return;
  if (b->owned) delete b->pool;
  Py_XDECREF(b->rank_fn);
  Py_XDECREF(b->keep);
  delete b;
}

void store_cap_free(PyObject* cap) {
  auto* s = static_cast<KvcStore*>(PyCapsule_GetPointer(cap, kStoreCap));
  delete s;
}

PoolBox* pool_box(PyObject* o) {
  return static_cast<PoolBox*>(PyCapsule_GetPointer(o, kPoolCap));
}
KvcStore* store_of(PyObject* o) {
  return static_cast<KvcStore*>(PyCapsule_GetPointer(o, kStoreCap));
}

bool i64(PyObject* o, int64_t* v) {
  const long long x = PyLong_AsLongLong(o);
  if (x == -1 && PyErr_Occurred()) return false;
  *v = x;
  return true;
}
// None -> KVC_NONE
bool opt_i64(PyObject* o, int64_t* v) {
  if (o == Py_None) {
    *v = KVC_NONE;
    return true;
  }
  return i64(o, v);
}
PyObject* opt_py(int64_t v) {
  if (v == KVC_NONE) Py_RETURN_NONE;
  return PyLong_FromLongLong(v);
}

#define NARGS(n)                                                               \
  if (nargs != (n)) {                                                          \
    PyErr_Format(PyExc_TypeError, "expected %d arguments, got %zd", (n), nargs); \
    return nullptr;                                                            \
  }
#define POOL(i)                        \
  PoolBox* box = pool_box(args[i]);    \
  if (box == nullptr) return nullptr;  \
  KvcPool* p = box->pool;
#define STORE(i)                          \
  KvcStore* s = store_of(args[i]);        \
  if (s == nullptr) return nullptr;
#define I64(name, i)                  \
  int64_t name;                       \
  if (!i64(args[i], &name)) return nullptr;
#define OPT(name, i)                  \
  int64_t name;                       \
  if (!opt_i64(args[i], &name)) return nullptr;

PyObject* group7(const Group& g) {
  return Py_BuildValue("(LLLNNNL)", static_cast<long long>(g.id),
                       static_cast<long long>(g.start), static_cast<long long>(g.length),
                       PyBool_FromLong(g.free), opt_py(g.owner), PyBool_FromLong(g.active),
                       static_cast<long long>(g.filled));
}

PyObject* triple(int64_t a, int64_t b, int64_t c) {
  return Py_BuildValue("(LLL)", static_cast<long long>(a), static_cast<long long>(b),
                       static_cast<long long>(c));
}
PyObject* pair(int64_t a, int64_t b) {
  return Py_BuildValue("(LL)", static_cast<long long>(a), static_cast<long long>(b));
}

// block table argument: a sequence of (start, length)
bool read_extents(PyObject* seq, std::vector<int64_t>& flat) {
  PyObject* fast = PySequence_Fast(seq, "extents must be a sequence");
  if (fast == nullptr) return false;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  PyObject** items = PySequence_Fast_ITEMS(fast);
  flat.resize(static_cast<size_t>(2 * n));
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* t = PySequence_Fast(items[i], "extent must be (start, length)");
    if (t == nullptr || PySequence_Fast_GET_SIZE(t) != 2) {
      Py_XDECREF(t);
      Py_DECREF(fast);
      if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "extent must be (start, length)");
      return false;
    }
    const bool ok = i64(PySequence_Fast_GET_ITEM(t, 0), &flat[2 * i]) &&
                    i64(PySequence_Fast_GET_ITEM(t, 1), &flat[2 * i + 1]);
    Py_DECREF(t);
    if (!ok) {
      Py_DECREF(fast);
      return false;
    }
  }
  Py_DECREF(fast);
  return true;
}

// plan words [moved, reused, n, nr, ops..., refresh...] -> (moved, reused, ops, refresh)
PyObject* plan_tuple(const std::vector<int64_t>& w) {
  const int64_t n = w[2], nr = w[3];
  PyObject* ops = PyList_New(n);
  PyObject* ref = PyList_New(nr);
  if (ops == nullptr || ref == nullptr) {
    Py_XDECREF(ops);
    Py_XDECREF(ref);
    return nullptr;
  }
  for (int64_t i = 0; i < n; ++i)
    PyList_SET_ITEM(ops, i, triple(w[4 + 3 * i], w[5 + 3 * i], w[6 + 3 * i]));
  for (int64_t i = 0; i < nr; ++i) {
    const size_t at = 4 + 3 * static_cast<size_t>(n + i);
    PyList_SET_ITEM(ref, i, triple(w[at], w[at + 1], w[at + 2]));
  }
  return Py_BuildValue("(LLNN)", static_cast<long long>(w[0]), static_cast<long long>(w[1]),
                       ops, ref);
}

// ------------------------------------------------------------------ module fns
PyObject* set_exceptions(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  // (PoolError, OutOfMemoryError, NoVictimError, CpuOutOfMemoryError,
  //  ContaminatedCopyError, InsufficientVictimsError)
  NARGS(6)
  PyObject* table[10] = {args[0], args[1], args[2], PyExc_ValueError, PyExc_KeyError,
                         PyExc_AssertionError, args[3], args[4], args[5], PyExc_StopIteration};
  for (int i = 0; i < 10; ++i) {
    Py_INCREF(table[i]);
    Py_XSETREF(g_exc[i], table[i]);
  }
  Py_RETURN_NONE;
}

PyObject* rng_draws(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(3)
  std::vector<int64_t> ent;
  PyObject* fast = PySequence_Fast(args[0], "entropy must be a sequence");
  if (fast == nullptr) return nullptr;
  for (Py_ssize_t i = 0; i < PySequence_Fast_GET_SIZE(fast); ++i) {
    int64_t v;
    if (!i64(PySequence_Fast_GET_ITEM(fast, i), &v)) {
      Py_DECREF(fast);
      return nullptr;
    }
    ent.push_back(v);
  }
  Py_DECREF(fast);
  I64(bound, 1)
  I64(n, 2)
  return guarded([&]() -> PyObject* {
    Pcg64 r;
    r.seed(coerce_entropy(ent.data(), static_cast<int>(ent.size())));
    PyObject* out = PyList_New(n);
    if (out == nullptr) return nullptr;
    for (int64_t i = 0; i < n; ++i) PyList_SET_ITEM(out, i, PyLong_FromLongLong(r.integers(bound)));
    return out;
  });
}

PyObject* pool_create(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(4)
  I64(total, 0)
  I64(initial, 1)
  I64(seed, 2)
  I64(policy, 3)
  KvcPool* p = nullptr;
  const int rc = kvc_pool_create(total, initial, seed, static_cast<int>(policy), &p);
  if (rc) return raise(Err{rc, g_err});
  auto* box = new PoolBox{p, true, nullptr, nullptr};
  PyObject* cap = PyCapsule_New(box, kPoolCap, pool_cap_free);
  if (cap == nullptr) {
    delete p;
    delete box;
  }
  return cap;
}

PyObject* pool_set_rank_fn(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  POOL(0)
  PyObject* fn = args[1];
  Py_XDECREF(box->rank_fn);
  box->rank_fn = nullptr;
  if (fn == Py_None) {
    p->rank_fn = nullptr;
    p->rank_ctx = nullptr;
  } else {
    Py_INCREF(fn);
    box->rank_fn = fn;
    p->rank_fn = rank_trampoline;
    p->rank_ctx = fn;
  }
  Py_RETURN_NONE;
}

PyObject* pool_allocate(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(5)
  POOL(0)
  I64(req, 1)
  I64(want, 2)
  OPT(expected, 3)
  const int reclaim = PyObject_IsTrue(args[4]);
  if (reclaim < 0) return nullptr;
  return guarded([&]() -> PyObject* {
    std::vector<Group> grants;
    std::vector<std::pair<int64_t, int64_t>> carved;
    p->allocate(req, want, expected, reclaim != 0, grants, carved);
    PyObject* gl = PyList_New(static_cast<Py_ssize_t>(grants.size()));
    PyObject* cl = PyList_New(static_cast<Py_ssize_t>(carved.size()));
    if (gl == nullptr || cl == nullptr) {
      Py_XDECREF(gl);
      Py_XDECREF(cl);
      return nullptr;
    }
    for (size_t i = 0; i < grants.size(); ++i)
      PyList_SET_ITEM(gl, i, triple(grants[i].id, grants[i].start, grants[i].length));
    for (size_t i = 0; i < carved.size(); ++i)
      PyList_SET_ITEM(cl, i, pair(carved[i].first, carved[i].second));
    return Py_BuildValue("(NN)", gl, cl);
  });
}

PyObject* pool_reclaim_from_victim(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(3)
  POOL(0)
  I64(need, 1)
  I64(for_request, 2)
  return guarded([&]() -> PyObject* {
    auto r = p->reclaim_from_victim(need, for_request);
    return Py_BuildValue("(LLLL)", static_cast<long long>(r.first),
                         static_cast<long long>(r.second.id),
                         static_cast<long long>(r.second.start),
                         static_cast<long long>(r.second.length));
  });
}

PyObject* pool_allocate_at(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(4)
  POOL(0)
  I64(req, 1)
  I64(start, 2)
  I64(length, 3)
  return guarded([&]() -> PyObject* {
    Group g{};
    if (!p->allocate_at(req, start, length, &g)) Py_RETURN_NONE;
    return triple(g.id, g.start, g.length);
  });
}

PyObject* pool_free_group(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  POOL(0)
  I64(gid, 1)
  return guarded([&]() -> PyObject* {
    p->free_group(gid);
    Py_RETURN_NONE;
  });
}

PyObject* pool_shrink_group(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(3)
  POOL(0)
  I64(gid, 1)
  I64(n, 2)
  return guarded([&]() -> PyObject* {
    p->shrink_group(gid, n);
    Py_RETURN_NONE;
  });
}

PyObject* pool_free_request(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  POOL(0)
  I64(req, 1)
  return guarded([&]() -> PyObject* { return PyLong_FromLongLong(p->free_request(req)); });
}

PyObject* pool_set_request_fill(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(3)
  POOL(0)
  I64(req, 1)
  I64(n, 2)
  return guarded([&]() -> PyObject* {
    p->set_request_fill(req, n);
    Py_RETURN_NONE;
  });
}

PyObject* pool_record_transfer(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  POOL(0)
  I64(blocks, 1)
  p->sizes[blocks] += 1;
  p->ops_recorded += 1;
  p->blocks_recorded += blocks;
  Py_RETURN_NONE;
}

PyObject* pool_counters(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(1)
  POOL(0)
  return Py_BuildValue("(LLLLLL)", static_cast<long long>(p->total),
                       static_cast<long long>(p->free_total),
                       static_cast<long long>(p->total - p->free_total),
                       static_cast<long long>(p->groups.size()),
                       static_cast<long long>(p->ops_recorded),
                       static_cast<long long>(p->blocks_recorded));
}

PyObject* pool_free_blocks(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(1)
  POOL(0)
  return PyLong_FromLongLong(p->free_total);
}

PyObject* pool_owned_blocks(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  POOL(0)
  I64(req, 1)
  return guarded([&]() -> PyObject* { return PyLong_FromLongLong(p->owned_blocks(req)); });
}

PyObject* pool_reclaimable(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  POOL(0)
  OPT(ex, 1)
  return guarded([&]() -> PyObject* { return PyLong_FromLongLong(p->reclaimable(ex)); });
}

PyObject* pool_group(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  POOL(0)
  I64(gid, 1)
  return guarded([&]() -> PyObject* { return group7(p->at(gid)); });
}

PyObject* pool_owned_groups(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  POOL(0)
  I64(req, 1)
  return guarded([&]() -> PyObject* {
    auto it = p->owned.find(req);
    const Py_ssize_t n = it == p->owned.end() ? 0 : static_cast<Py_ssize_t>(it->second.size());
    PyObject* out = PyList_New(n);
    if (out == nullptr) return nullptr;
    for (Py_ssize_t i = 0; i < n; ++i) PyList_SET_ITEM(out, i, group7(p->groups.at(it->second[i])));
    return out;
  });
}

PyObject* pool_free_groups(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(1)
  POOL(0)
  return guarded([&]() -> PyObject* {
    PyObject* out = PyList_New(static_cast<Py_ssize_t>(p->by_addr.size()));
    if (out == nullptr) return nullptr;
    Py_ssize_t i = 0;
    for (auto& a : p->by_addr) PyList_SET_ITEM(out, i++, group7(p->groups.at(a.second)));
    return out;
  });
}

PyObject* pool_extents(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  POOL(0)
  I64(req, 1)
  return guarded([&]() -> PyObject* {
    std::vector<std::pair<int64_t, int64_t>> runs;
    auto it = p->owned.find(req);
    if (it != p->owned.end())
      for (int64_t gid : it->second) {
        const Group& g = p->groups.at(gid);
        if (!runs.empty() && runs.back().first + runs.back().second == g.start)
          runs.back().second += g.length;
        else
          runs.emplace_back(g.start, g.length);
      }
    PyObject* out = PyList_New(static_cast<Py_ssize_t>(runs.size()));
    if (out == nullptr) return nullptr;
    for (size_t i = 0; i < runs.size(); ++i)
      PyList_SET_ITEM(out, i, pair(runs[i].first, runs[i].second));
    return out;
  });
}

PyObject* pool_granularity(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(1)
  POOL(0)
  PyObject* d = PyDict_New();
  if (d == nullptr) return nullptr;
  for (auto& kv : p->sizes) {
    PyObject* k = PyLong_FromLongLong(kv.first);
    PyObject* v = PyLong_FromLongLong(kv.second);
    const int rc = (k && v) ? PyDict_SetItem(d, k, v) : -1;
    Py_XDECREF(k);
    Py_XDECREF(v);
    if (rc) {
      Py_DECREF(d);
      return nullptr;
    }
  }
  return d;
}

PyObject* pool_dump(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(1)
  POOL(0)
  return guarded([&]() -> PyObject* {
    const std::string t = p->dump();
    return PyUnicode_FromStringAndSize(t.data(), static_cast<Py_ssize_t>(t.size()));
  });
}

PyObject* pool_validate(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(1)
  POOL(0)
  return guarded([&]() -> PyObject* {
    p->validate();
    Py_RETURN_NONE;
  });
}

PyObject* store_create(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(6)
  I64(total, 0)
  I64(reuse, 1)
  I64(pmin, 2)
  I64(pmax, 3)
  I64(rel, 4)
  I64(bt, 5)
  KvcStore* s = nullptr;
  const int rc = kvc_store_create(total, static_cast<int>(reuse), pmin, pmax,
                                  static_cast<int>(rel), bt, &s);
  if (rc) return raise(Err{rc, g_err});
  PyObject* cap = PyCapsule_New(s, kStoreCap, store_cap_free);
  if (cap == nullptr) delete s;
  return cap;
}

PyObject* store_pool(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(1)
  STORE(0)
  Py_INCREF(args[0]);
  auto* box = new PoolBox{&s->pool, false, nullptr, args[0]};
  PyObject* cap = PyCapsule_New(box, kPoolCap, pool_cap_free);
  if (cap == nullptr) {
    Py_DECREF(args[0]);
    delete box;
  }
  return cap;
}

PyObject* store_set_flag(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(3)
  STORE(0)
  I64(which, 1)
  I64(v, 2)
  const int rc = kvc_store_set_flag(s, static_cast<int>(which), v);
  if (rc) return raise(Err{rc, g_err});
  Py_RETURN_NONE;
}

PyObject* store_counters(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(1)
  STORE(0)
  return Py_BuildValue("(LLLLL)", static_cast<long long>(s->peak),
                       static_cast<long long>(s->refreshed),
                       static_cast<long long>(s->copies.size()),
                       static_cast<long long>(s->ranks.size()),
                       static_cast<long long>(s->refresh_dirty_tail ? 1 : 0));
}

PyObject* store_set_rank(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(3)
  STORE(0)
  I64(req, 1)
  I64(rank, 2)
  s->ranks[req] = rank;
  Py_RETURN_NONE;
}

PyObject* store_set_ranks(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  STORE(0)
  if (!PyDict_Check(args[1])) {
    PyErr_SetString(PyExc_TypeError, "ranks must be a dict");
    return nullptr;
  }
  PyObject *k, *v;
  Py_ssize_t pos = 0;
  while (PyDict_Next(args[1], &pos, &k, &v)) {
    int64_t req, rank;
    if (!i64(k, &req) || !i64(v, &rank)) return nullptr;
    s->ranks[req] = rank;
  }
  Py_RETURN_NONE;
}

PyObject* store_get_rank(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  STORE(0)
  I64(req, 1)
  auto it = s->ranks.find(req);
  if (it == s->ranks.end()) Py_RETURN_NONE;
  return PyLong_FromLongLong(it->second);
}

PyObject* store_del_rank(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  STORE(0)
  I64(req, 1)
  if (s->ranks.erase(req) == 0) return raise(Err{KVC_ERR_KEY, i2s(req)});
  Py_RETURN_NONE;
}

PyObject* store_ranks(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(1)
  STORE(0)
  PyObject* out = PyList_New(static_cast<Py_ssize_t>(s->ranks.size()));
  if (out == nullptr) return nullptr;
  Py_ssize_t i = 0;
  for (auto& kv : s->ranks) PyList_SET_ITEM(out, i++, pair(kv.first, kv.second));
  return out;
}

PyObject* store_clear_ranks(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(1)
  STORE(0)
  s->ranks.clear();
  Py_RETURN_NONE;
}

PyObject* store_plan_swap_out(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(5)
  STORE(0)
  I64(req, 1)
  I64(fp, 2)
  std::vector<int64_t> ext;
  if (!read_extents(args[3], ext)) return nullptr;
  OPT(tokens, 4)
  return guarded([&]() -> PyObject* {
    s->plan_swap_out(req, fp, ext.data(), static_cast<int64_t>(ext.size() / 2), tokens);
    return plan_tuple(s->out);
  });
}

PyObject* store_plan_swap_in(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(3)
  STORE(0)
  I64(req, 1)
  std::vector<int64_t> ext;
  if (!read_extents(args[2], ext)) return nullptr;
  return guarded([&]() -> PyObject* {
    s->plan_swap_in(req, ext.data(), static_cast<int64_t>(ext.size() / 2));
    return plan_tuple(s->out);
  });
}

PyObject* store_plan_swap_in_prefix(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(3)
  STORE(0)
  I64(req, 1)
  std::vector<int64_t> ext;
  if (!read_extents(args[2], ext)) return nullptr;
  return guarded([&]() -> PyObject* {
    s->plan_swap_in_prefix(req, ext.data(), static_cast<int64_t>(ext.size() / 2));
    PyObject* plan = plan_tuple(s->out);
    if (plan == nullptr) return nullptr;
    return Py_BuildValue("(NL)", plan, static_cast<long long>(s->out.back()));
  });
}

PyObject* store_evict_for(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(3)
  STORE(0)
  I64(rank, 1)
  I64(need, 2)
  return guarded([&]() -> PyObject* {
    std::vector<int64_t> taken;
    s->evict_for(rank, need, &taken);
    PyObject* out = PyList_New(static_cast<Py_ssize_t>(taken.size() / 2));
    if (out == nullptr) return nullptr;
    for (size_t i = 0; i < taken.size() / 2; ++i)
      PyList_SET_ITEM(out, i, pair(taken[2 * i], taken[2 * i + 1]));
    return out;
  });
}

PyObject* store_preallocate_increment(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(3)
  STORE(0)
  I64(req, 1)
  I64(inc, 2)
  return guarded([&]() -> PyObject* {
    return PyBool_FromLong(s->preallocate_increment(req, inc) ? 1 : 0);
  });
}

PyObject* store_release(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  STORE(0)
  I64(req, 1)
  return guarded([&]() -> PyObject* {
    s->release(req);
    Py_RETURN_NONE;
  });
}

PyObject* store_ensure_free(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(3)
  STORE(0)
  I64(req, 1)
  I64(need, 2)
  return guarded([&]() -> PyObject* {
    s->ensure_free(req, need);
    Py_RETURN_NONE;
  });
}

PyObject* store_track_peak(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(1)
  STORE(0)
  s->track_peak();
  Py_RETURN_NONE;
}

PyObject* store_copy_ids(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(1)
  STORE(0)
  std::vector<std::pair<int64_t, int64_t>> order;
  for (auto& kv : s->copies) order.emplace_back(kv.second.order, kv.first);
  std::sort(order.begin(), order.end());
  PyObject* out = PyList_New(static_cast<Py_ssize_t>(order.size()));
  if (out == nullptr) return nullptr;
  for (size_t i = 0; i < order.size(); ++i)
    PyList_SET_ITEM(out, i, PyLong_FromLongLong(order[i].second));
  return out;
}

PyObject* store_has_copy(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  STORE(0)
  I64(req, 1)
  return PyBool_FromLong(s->copies.count(req) ? 1 : 0);
}

PyObject* store_copy(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  STORE(0)
  I64(req, 1)
  auto it = s->copies.find(req);
  if (it == s->copies.end()) return raise(Err{KVC_ERR_KEY, i2s(req)});
  const Copy& c = it->second;
  PyObject* segs = PyList_New(static_cast<Py_ssize_t>(c.segs.size()));
  if (segs == nullptr) return nullptr;
  for (size_t i = 0; i < c.segs.size(); ++i) {
    const Seg& g = c.segs[i];
    PyList_SET_ITEM(segs, i,
                    Py_BuildValue("(LLNN)", static_cast<long long>(g.lo),
                                  static_cast<long long>(g.hi), opt_py(g.gid),
                                  PyBool_FromLong(g.valid)));
  }
  return Py_BuildValue("(NNN)", opt_py(c.prealloc), opt_py(c.saved), segs);
}

PyObject* store_put_copy(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(5)
  STORE(0)
  I64(req, 1)
  OPT(prealloc, 2)
  OPT(saved, 3)
  PyObject* fast = PySequence_Fast(args[4], "segments must be a sequence");
  if (fast == nullptr) return nullptr;
  std::vector<int64_t> flat;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* t = PySequence_Fast(PySequence_Fast_GET_ITEM(fast, i),
                                  "segment must be (lo, hi, group id, valid)");
    if (t == nullptr || PySequence_Fast_GET_SIZE(t) != 4) {
      Py_XDECREF(t);
      Py_DECREF(fast);
      if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "segment must have 4 fields");
      return nullptr;
    }
    int64_t lo, hi, gid;
    const int valid = PyObject_IsTrue(PySequence_Fast_GET_ITEM(t, 3));
    const bool ok = i64(PySequence_Fast_GET_ITEM(t, 0), &lo) &&
                    i64(PySequence_Fast_GET_ITEM(t, 1), &hi) &&
                    opt_i64(PySequence_Fast_GET_ITEM(t, 2), &gid) && valid >= 0;
    Py_DECREF(t);
    if (!ok) {
      Py_DECREF(fast);
      return nullptr;
    }
    flat.insert(flat.end(), {lo, hi, gid, valid});
  }
  Py_DECREF(fast);
  const int rc = kvc_store_put_copy(s, req, prealloc, saved, flat.data(), n);
  if (rc) return raise(Err{rc, g_err});
  Py_RETURN_NONE;
}

PyObject* store_drop_copy(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  NARGS(2)
  STORE(0)
  I64(req, 1)
  if (s->copies.erase(req) == 0) return raise(Err{KVC_ERR_KEY, i2s(req)});
  Py_RETURN_NONE;
}

#define FN(name) {#name, reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(name)), \
                  METH_FASTCALL, nullptr}

PyMethodDef kMethods[] = {
    FN(set_exceptions), FN(rng_draws),
    FN(pool_create), FN(pool_set_rank_fn), FN(pool_allocate), FN(pool_reclaim_from_victim),
    FN(pool_allocate_at), FN(pool_free_group), FN(pool_shrink_group), FN(pool_free_request),
    FN(pool_set_request_fill), FN(pool_record_transfer), FN(pool_counters), FN(pool_free_blocks),
    FN(pool_owned_blocks), FN(pool_reclaimable), FN(pool_group), FN(pool_owned_groups),
    FN(pool_free_groups), FN(pool_extents), FN(pool_granularity), FN(pool_dump),
    FN(pool_validate),
    FN(store_create), FN(store_pool), FN(store_set_flag), FN(store_counters), FN(store_set_rank),
    FN(store_set_ranks), FN(store_get_rank), FN(store_del_rank), FN(store_ranks),
    FN(store_clear_ranks), FN(store_plan_swap_out), FN(store_plan_swap_in),
    FN(store_plan_swap_in_prefix), FN(store_evict_for), FN(store_preallocate_increment),
    FN(store_release), FN(store_ensure_free), FN(store_track_peak), FN(store_copy_ids),
    FN(store_has_copy), FN(store_copy), FN(store_put_copy), FN(store_drop_copy),
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_kvctrl",
                       "Native control plane (block-group pool, CPU store); see native_ctrl.py",
                       -1, kMethods, nullptr, nullptr, nullptr, nullptr};

}  // namespace

PyMODINIT_FUNC PyInit__kvctrl(void) { return PyModule_Create(&kModule); }

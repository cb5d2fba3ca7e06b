/*
 * materialize.c — host-side construction of the reference's template objects from the
 * device's frontier items (coral_s1_frontier_item, include/coral_s1.h), for the e2e
 * path of build_frontier. Pure object plumbing: no arithmetic happens here; every
 * number comes from the CUDA library. It builds exactly what
 * paper_2605_04357_b200/frontier.py:materialise builds in Python (one ServingTemplate
 * per (model, phase, combo), shared by the regions it survives in), writing fields
 * into each frozen dataclass instance's __dict__ as the Python path does.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

#include "../../include/coral_s1.h"

static PyObject *s_items, *s_num_stages, *s_layers, *s_son, *s_model, *s_phase, *s_slo, *s_combo,
    *s_placement, *s_tps;

static PyObject* new_with_dict(PyTypeObject* tp, PyObject** dict) {
  PyObject* o = tp->tp_alloc(tp, 0);
  if (!o) return NULL;
  *dict = PyObject_GenericGetDict(o, NULL);
  if (!*dict) { Py_DECREF(o); return NULL; }
  return o;
}

static int set(PyObject* d, PyObject* k, PyObject* v) {  /* steals v */
  if (!v) return -1;
  int rc = PyDict_SetItem(d, k, v);
  Py_DECREF(v);
  return rc;
}

/* materialise(items: bytes-like of coral_s1_frontier_item, cfg_by_rank: list,
 *             model_names: list[str], phases: tuple[str], slos: list, regions: list[str],
 *             num_phases: int, ServingTemplate, Placement, NodeComboKey, FrontierEntry)
 * -> dict {(model, phase, region): [FrontierEntry, ...]} in item order. */
static PyObject* materialise(PyObject* self, PyObject* args) {
  Py_buffer buf;
  PyObject *cfgs, *mnames, *phases, *slos, *regions, *T_tmpl, *T_pl, *T_combo, *T_entry;
  int NP;
  if (!PyArg_ParseTuple(args, "y*OOOOOiOOOO", &buf, &cfgs, &mnames, &phases, &slos, &regions, &NP,
                        &T_tmpl, &T_pl, &T_combo, &T_entry))
    return NULL;
  const coral_s1_frontier_item* it = (const coral_s1_frontier_item*)buf.buf;
  const Py_ssize_t n = buf.len / (Py_ssize_t)sizeof(coral_s1_frontier_item);
  PyObject* segments = PyDict_New();
  PyObject* cache = PyDict_New();
  if (!segments || !cache) goto fail;
  for (Py_ssize_t i = 0; i < n; ++i) {
    const coral_s1_frontier_item* x = &it[i];
    const int mp = x->mp, m = mp / NP, ph = mp % NP;
    PyObject* ck = Py_BuildValue("(iK)", mp, (unsigned long long)x->combo_key);
    if (!ck) goto fail;
    PyObject* t = PyDict_GetItem(cache, ck); /* borrowed */
    if (!t) {
      /* NodeComboKey(items=((cfg, n), ...)) */
      int ntok = 0;
      for (int k = 0; k < CORAL_S1_MAX_NODES; ++k)
        if ((x->combo_key >> (9 * (CORAL_S1_MAX_NODES - 1 - k))) & 511u) ++ntok;
      PyObject* items = PyTuple_New(ntok);
      for (int k = 0; k < ntok; ++k) {
        const unsigned tok = (unsigned)(x->combo_key >> (9 * (CORAL_S1_MAX_NODES - 1 - k))) & 511u;
        PyObject* cfg = PyList_GetItem(cfgs, (Py_ssize_t)((tok >> 3) - 1));
        Py_INCREF(cfg);
        PyTuple_SET_ITEM(items, k, Py_BuildValue("(Ni)", cfg, (int)(tok & 7u)));
      }
      PyObject *dc, *dp, *dt;
      PyObject* combo = new_with_dict((PyTypeObject*)T_combo, &dc);
      if (!combo || set(dc, s_items, items) < 0) goto fail;
      Py_DECREF(dc);
      const int S = x->rec.num_stages, nn = x->rec.num_nodes;
      PyObject* layers = PyTuple_New(S);
      for (int s = 0; s < S; ++s) PyTuple_SET_ITEM(layers, s, PyLong_FromLong(x->rec.layers_per_stage[s]));
      PyObject* son = PyTuple_New(nn);
      for (int k = 0; k < nn; ++k) PyTuple_SET_ITEM(son, k, PyLong_FromLong(x->rec.stage_of_node[k]));
      PyObject* pl = new_with_dict((PyTypeObject*)T_pl, &dp);
      if (!pl || set(dp, s_num_stages, PyLong_FromLong(S)) < 0 || set(dp, s_layers, layers) < 0 ||
          set(dp, s_son, son) < 0)
        goto fail;
      Py_DECREF(dp);
      PyObject* tmpl = new_with_dict((PyTypeObject*)T_tmpl, &dt);
      PyObject* mname = PyList_GetItem(mnames, m);
      PyObject* phs = PyTuple_GetItem(phases, ph);
      PyObject* slo = PyList_GetItem(slos, m);
      Py_INCREF(mname);
      Py_INCREF(phs);
      Py_INCREF(slo);
      if (!tmpl || set(dt, s_model, mname) < 0 || set(dt, s_phase, phs) < 0 || set(dt, s_slo, slo) < 0 ||
          set(dt, s_combo, combo) < 0 || set(dt, s_placement, pl) < 0 ||
          set(dt, s_tps, PyFloat_FromDouble(x->rec.throughput_tps)) < 0)
        goto fail;
      Py_DECREF(dt);
      if (PyDict_SetItem(cache, ck, tmpl) < 0) goto fail;
      Py_DECREF(tmpl);
      t = tmpl; /* owned by cache */
    }
    Py_DECREF(ck);
    PyObject* seg = Py_BuildValue("(OOO)", PyList_GetItem(mnames, m), PyTuple_GetItem(phases, ph),
                                  PyList_GetItem(regions, x->region));
    PyObject* lst = PyDict_GetItem(segments, seg);
    if (!lst) {
      lst = PyList_New(0);
      PyDict_SetItem(segments, seg, lst);
      Py_DECREF(lst);
    }
    Py_DECREF(seg);
    /* FrontierEntry is a 2-field namedtuple subclass: allocate the tuple directly */
    PyObject* entry = ((PyTypeObject*)T_entry)->tp_alloc((PyTypeObject*)T_entry, 2);
    if (!entry) goto fail;
    Py_INCREF(t);
    PyTuple_SET_ITEM(entry, 0, t);
    PyTuple_SET_ITEM(entry, 1, PyFloat_FromDouble(x->price_usd_h));
    if (PyList_Append(lst, entry) < 0) goto fail;
    Py_DECREF(entry);
  }
  Py_DECREF(cache);
  PyBuffer_Release(&buf);
  return segments;
fail:
  Py_XDECREF(segments);
  Py_XDECREF(cache);
  PyBuffer_Release(&buf);
  if (!PyErr_Occurred()) PyErr_SetString(PyExc_RuntimeError, "materialise failed");
  return NULL;
}

static PyMethodDef methods[] = {{"materialise", materialise, METH_VARARGS, NULL}, {NULL, NULL, 0, NULL}};
static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_materialize", NULL, -1, methods};

PyMODINIT_FUNC PyInit__materialize(void) {
  s_items = PyUnicode_InternFromString("items");
  s_num_stages = PyUnicode_InternFromString("num_stages");
  s_layers = PyUnicode_InternFromString("layers_per_stage");
  s_son = PyUnicode_InternFromString("stage_of_node");
  s_model = PyUnicode_InternFromString("model");
  s_phase = PyUnicode_InternFromString("phase");
  s_slo = PyUnicode_InternFromString("slo");
  s_combo = PyUnicode_InternFromString("combo");
  s_placement = PyUnicode_InternFromString("placement");
  s_tps = PyUnicode_InternFromString("throughput_tps");
  return PyModule_Create(&mod);
}

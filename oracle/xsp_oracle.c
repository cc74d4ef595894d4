/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference's correlate + analyze path over the
 * SoA columns of include/xsp.h. It follows the reference's own algorithm
 * (an augmented interval tree per trace and hash maps keyed by correlation
 * id), i.e. deliberately NOT the scan-based design of the CUDA path, so the two
 * cross-check each other. Every function cites the reference code it restates
 * (paths relative to /root/reference/proj). Pinned against the unmodified
 * reference (oracle/_ref) by tests/test_oracle.py.
 */
#include "xsp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define NONE 0xFFFFFFFFu

static unsigned lvl(uint8_t f) { return f & 3u; }
static unsigned knd(uint8_t f) { return (f >> 2) & 3u; }
/* Span::duration_ns, span.hpp:93-95 */
static uint64_t dur(uint64_t b, uint64_t e) { return e >= b ? e - b : 0; }
/* is_kernel_launch / is_exec / is_sync_kernel, correlator.cpp:32-42 */
static int is_kernel_launch(uint8_t f) { return knd(f) == XSP_KIND_LAUNCH && lvl(f) >= XSP_LEVEL_KERNEL; }
static int is_exec(uint8_t f) { return knd(f) == XSP_KIND_EXEC; }
static int is_sync_kernel(uint8_t f) { return knd(f) == XSP_KIND_SYNC && lvl(f) == XSP_LEVEL_KERNEL; }
static int is_model(uint8_t f) { return knd(f) == XSP_KIND_SYNC && lvl(f) == XSP_LEVEL_MODEL; }

/* ---- growable vectors ---------------------------------------------------- */
#define VEC(T, N)                                                              \
  typedef struct { T* v; size_t n, cap; } N;                                   \
  static void N##_push(N* a, T x) {                                            \
    if (a->n == a->cap) {                                                      \
      a->cap = a->cap ? 2 * a->cap : 64;                                       \
      a->v = (T*)realloc(a->v, a->cap * sizeof(T));                            \
    }                                                                          \
    a->v[a->n++] = x;                                                          \
  }
VEC(uint32_t, vu32)
VEC(uint64_t, vu64)
VEC(uint8_t, vu8)
VEC(double, vf64)
VEC(int32_t, vi32)
VEC(int8_t, vi8)

/* ---- hash map u64 -> u32 (std::unordered_map stand-in) -------------------- */
typedef struct {
  uint64_t* key;
  uint32_t* val;
  uint8_t* used;
  size_t mask;
} hmap;

static uint64_t mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}
static void hmap_init(hmap* h, size_t n) {
  size_t cap = 16;
  while (cap < 2 * n + 16) cap <<= 1;
  h->key = (uint64_t*)malloc(cap * sizeof(uint64_t));
  h->val = (uint32_t*)malloc(cap * sizeof(uint32_t));
  h->used = (uint8_t*)calloc(cap, 1);
  h->mask = cap - 1;
}
static void hmap_free(hmap* h) {
  free(h->key);
  free(h->val);
  free(h->used);
}
/* slot of key, or the empty slot where it would go */
static size_t hmap_slot(const hmap* h, uint64_t k) {
  size_t s = mix(k) & h->mask;
  while (h->used[s] && h->key[s] != k) s = (s + 1) & h->mask;
  return s;
}

/* ---- sort helpers --------------------------------------------------------- */
typedef struct {
  uint64_t k1, k2, k3;
  uint32_t a, b;
} rec;
static int rec_cmp(const void* x, const void* y) {
  const rec* p = (const rec*)x;
  const rec* q = (const rec*)y;
  if (p->k1 != q->k1) return p->k1 < q->k1 ? -1 : 1;
  if (p->k2 != q->k2) return p->k2 < q->k2 ? -1 : 1;
  if (p->k3 != q->k3) return p->k3 < q->k3 ? -1 : 1;
  return 0;
}

/* ---- IntervalTree, correlator.cpp:66-126 ---------------------------------- */
typedef struct {
  uint64_t b, e, sid;
  uint32_t idx;
} entry;
typedef struct {
  entry* en;
  uint64_t* maxend;
  size_t n;
} itree;

static uint64_t it_fill(itree* t, size_t lo, size_t hi) {
  if (lo >= hi) return 0;
  size_t mid = lo + (hi - lo) / 2;
  uint64_t m = t->en[mid].e;
  uint64_t l = it_fill(t, lo, mid), r = it_fill(t, mid + 1, hi);
  if (l > m) m = l;
  if (r > m) m = r;
  t->maxend[mid] = m;
  return m;
}
static void it_query(const itree* t, size_t lo, size_t hi, uint64_t b, uint64_t e, vu32* out) {
  if (lo >= hi) return;
  size_t mid = lo + (hi - lo) / 2;
  if (t->maxend[mid] < e) return;
  it_query(t, lo, mid, b, e, out);
  if (t->en[mid].b <= b) {
    if (t->en[mid].e >= e) vu32_push(out, (uint32_t)mid);
    it_query(t, mid + 1, hi, b, e, out);
  }
}

/* ---- correlate ------------------------------------------------------------ */
typedef struct {
  vi32 status;
  vu32 err, model;
  vu32 t_loff, t_koff, t_ooff, t_aoff;
  vu32 l_row, l_koff, l_attr;
  vu64 l_dur;
  vu32 k_launch, k_exec, k_mrow, k_name;
  vu64 k_dur;
  vf64 k_occ;
  vu32 o_row;
  vu8 o_reason;
  vu32 a_row, a_coff, a_crow;
} corr_acc;

int xspo_correlate(const xsp_span_cols* c, const xsp_traces* tr, xsp_corr_out* out) {
  const uint64_t n = c->n_spans;
  const uint32_t T = tr->n_traces;
  uint32_t* mrow = (uint32_t*)malloc((n + 1) * sizeof(uint32_t)); /* metric-table row per span */
  uint32_t* arow = (uint32_t*)malloc((n + 1) * sizeof(uint32_t)); /* layer-table row per span */
  {
    uint32_t m = 0, a = 0;
    for (uint64_t i = 0; i < n; ++i) {
      mrow[i] = (c->flags[i] & XSP_F_METRICS) ? m++ : NONE;
      arow[i] = lvl(c->flags[i]) == XSP_LEVEL_LAYER ? a++ : NONE;
    }
  }
  corr_acc A;
  memset(&A, 0, sizeof(A));
  vu32_push(&A.t_loff, 0);
  vu32_push(&A.t_koff, 0);
  vu32_push(&A.t_ooff, 0);
  vu32_push(&A.t_aoff, 0);
  vu32_push(&A.l_koff, 0);
  vu32_push(&A.a_coff, 0);

  for (uint32_t t = 0; t < T; ++t) {
    const uint64_t s0 = tr->span_off[t], s1 = tr->span_off[t + 1];
    const uint64_t ns = s1 - s0;
    int32_t status = XSP_T_OK;
    uint32_t ea = NONE, eb = NONE;
    /* TraceBundle::model_span, span.cpp:298-303 */
    uint64_t model = (uint64_t)-1;
    for (uint64_t i = s0; i < s1; ++i)
      if (is_model(c->flags[i])) {
        model = i;
        break;
      }
    /* assign_parents preconditions, correlator.cpp:142-158 */
    if (model == (uint64_t)-1) {
      status = XSP_T_NO_MODEL;
    } else {
      for (uint64_t i = s0; i < s1; ++i) {
        uint8_t f = c->flags[i];
        if (is_model(f) && c->span_id[i] != c->span_id[model]) {
          status = XSP_T_MULTI_MODEL;
          ea = (uint32_t)i;
          break;
        }
        if (lvl(f) >= XSP_LEVEL_KERNEL && !(tr->levels[t] & (1u << XSP_LEVEL_LAYER))) {
          status = XSP_T_SKIP_LEVEL;
          ea = (uint32_t)i;
          break;
        }
      }
    }
    /* per-trace outputs are staged and committed only if the trace succeeds */
    vu32 o_row = {0}, lay = {0}, amb = {0}, amb_cand = {0}, amb_coff = {0};
    vu8 o_reason = {0};
    vu32_push(&amb_coff, 0);
    rec* knodes = NULL;
    size_t nkn = 0;
    if (status == XSP_T_OK) {
      const uint64_t mb = c->begin_ns[model], me = c->end_ns[model], msid = c->span_id[model];
      /* layers, correlator.cpp:168-212 */
      for (uint64_t i = s0; i < s1; ++i) {
        uint8_t f = c->flags[i];
        if (lvl(f) != XSP_LEVEL_LAYER) continue;
        if (knd(f) != XSP_KIND_SYNC) {
          vu32_push(&o_row, (uint32_t)i);
          vu8_push(&o_reason, XSP_O_LAYER_NON_SYNC);
          continue;
        }
        if (f & XSP_F_PARENT) {
          if (c->parent_id[i] != msid) {
            vu32_push(&o_row, (uint32_t)i);
            vu8_push(&o_reason, XSP_O_LAYER_BAD_PARENT);
            continue;
          }
        } else if (!(mb <= c->begin_ns[i] && c->end_ns[i] <= me)) {
          vu32_push(&o_row, (uint32_t)i);
          vu8_push(&o_reason, XSP_O_LAYER_OUTSIDE_MODEL);
          continue;
        }
        vu32_push(&lay, (uint32_t)i);
      }
      /* sort placed layers by (begin_ns, span_id) -> layer_index */
      rec* lr = (rec*)malloc((lay.n + 1) * sizeof(rec));
      for (size_t j = 0; j < lay.n; ++j) {
        uint32_t i = lay.v[j];
        lr[j].k1 = c->begin_ns[i];
        lr[j].k2 = c->span_id[i];
        lr[j].k3 = j;
        lr[j].a = i;
      }
      qsort(lr, lay.n, sizeof(rec), rec_cmp);
      const size_t L = lay.n;
      /* layer_by_span_id (last wins, :215-220) as (sid, index) sorted */
      rec* bysid = (rec*)malloc((L + 1) * sizeof(rec));
      for (size_t j = 0; j < L; ++j) {
        bysid[j].k1 = c->span_id[lr[j].a];
        bysid[j].k2 = j;
        bysid[j].k3 = 0;
      }
      qsort(bysid, L, sizeof(rec), rec_cmp);
      /* interval tree over placed layers */
      itree it;
      it.n = L;
      it.en = (entry*)malloc((L + 1) * sizeof(entry));
      it.maxend = (uint64_t*)calloc(L + 1, sizeof(uint64_t));
      for (size_t j = 0; j < L; ++j) {
        it.en[j].b = c->begin_ns[lr[j].a];
        it.en[j].e = c->end_ns[lr[j].a];
        it.en[j].sid = c->span_id[lr[j].a];
        it.en[j].idx = (uint32_t)j;
      }
      it_fill(&it, 0, L);
      /* kernels, correlator.cpp:226-268 */
      knodes = (rec*)malloc((ns + 1) * sizeof(rec));
      vu32 cand = {0};
      for (uint64_t i = s0; i < s1; ++i) {
        uint8_t f = c->flags[i];
        if (!is_kernel_launch(f) && !is_sync_kernel(f)) continue;
        uint32_t parent = NONE;
        if (f & XSP_F_PARENT) {
          uint64_t want = c->parent_id[i];
          size_t lo = 0, hi = L;
          while (lo < hi) {
            size_t mid = (lo + hi) / 2;
            if (bysid[mid].k1 <= want) lo = mid + 1; else hi = mid;
          }
          if (lo == 0 || bysid[lo - 1].k1 != want) {
            vu32_push(&o_row, (uint32_t)i);
            vu8_push(&o_reason, XSP_O_KERNEL_BAD_PARENT);
            continue;
          }
          parent = (uint32_t)bysid[lo - 1].k2;
        } else {
          cand.n = 0;
          it_query(&it, 0, L, c->begin_ns[i], c->end_ns[i], &cand);
          if (cand.n == 0) {
            vu32_push(&o_row, (uint32_t)i);
            vu8_push(&o_reason, XSP_O_KERNEL_NO_LAYER);
            continue;
          }
          if (cand.n > 1) {
            /* candidates sorted by span_id (:115-117) */
            rec* cr = (rec*)malloc(cand.n * sizeof(rec));
            for (size_t q = 0; q < cand.n; ++q) {
              cr[q].k1 = it.en[cand.v[q]].sid;
              cr[q].k2 = 0;
              cr[q].k3 = 0;
              cr[q].a = lr[cand.v[q]].a;
            }
            qsort(cr, cand.n, sizeof(rec), rec_cmp);
            vu32_push(&amb, (uint32_t)i);
            for (size_t q = 0; q < cand.n; ++q) vu32_push(&amb_cand, cr[q].a);
            vu32_push(&amb_coff, (uint32_t)amb_cand.n);
            free(cr);
            continue;
          }
          parent = it.en[cand.v[0]].idx;
        }
        rec* kn = &knodes[nkn++];
        kn->k1 = parent;
        kn->k2 = c->begin_ns[i];
        kn->k3 = c->span_id[i];
        kn->a = (uint32_t)i;
        kn->b = (uint32_t)(nkn - 1);
      }
      free(cand.v);
      /* kernels per layer sorted by (launch.begin_ns, launch.span_id) (:270-276) */
      qsort(knodes, nkn, sizeof(rec), rec_cmp);
      /* ambiguities sorted by span_id (:277-280): sort (sid, slot) and permute */
      if (amb.n > 1) {
        rec* ar = (rec*)malloc(amb.n * sizeof(rec));
        for (size_t q = 0; q < amb.n; ++q) {
          ar[q].k1 = c->span_id[amb.v[q]];
          ar[q].k2 = q;
          ar[q].k3 = 0;
        }
        qsort(ar, amb.n, sizeof(rec), rec_cmp);
        vu32 na = {0}, nc = {0}, no = {0};
        vu32_push(&no, 0);
        for (size_t q = 0; q < amb.n; ++q) {
          size_t src = ar[q].k2;
          vu32_push(&na, amb.v[src]);
          for (uint32_t x = amb_coff.v[src]; x < amb_coff.v[src + 1]; ++x) vu32_push(&nc, amb_cand.v[x]);
          vu32_push(&no, (uint32_t)nc.n);
        }
        free(amb.v);
        free(amb_cand.v);
        free(amb_coff.v);
        amb = na;
        amb_cand = nc;
        amb_coff = no;
        free(ar);
      }

      /* correlate_async, correlator.cpp:287-364 */
      hmap ex, la;
      hmap_init(&ex, ns);
      hmap_init(&la, ns);
      for (uint64_t i = s0; i < s1 && status == XSP_T_OK; ++i) {
        uint8_t f = c->flags[i];
        if (!is_exec(f)) continue;
        if (!(f & XSP_F_CID)) {
          vu32_push(&o_row, (uint32_t)i);
          vu8_push(&o_reason, XSP_O_EXEC_NO_CID);
          continue;
        }
        size_t s = hmap_slot(&ex, c->cid[i]);
        if (ex.used[s]) {
          status = XSP_T_DUP_EXEC_CID;
          ea = ex.val[s];
          eb = (uint32_t)i;
          break;
        }
        ex.used[s] = 1;
        ex.key[s] = c->cid[i];
        ex.val[s] = (uint32_t)i;
      }
      for (uint64_t i = s0; i < s1 && status == XSP_T_OK; ++i) {
        uint8_t f = c->flags[i];
        if (!is_kernel_launch(f) || !(f & XSP_F_CID)) continue;
        size_t s = hmap_slot(&la, c->cid[i]);
        if (la.used[s]) {
          status = XSP_T_DUP_LAUNCH_CID;
          ea = la.val[s];
          eb = (uint32_t)i;
          break;
        }
        la.used[s] = 1;
        la.key[s] = c->cid[i];
        la.val[s] = (uint32_t)i;
      }
      if (status == XSP_T_OK) {
        /* commit layers */
        const uint32_t lbase = (uint32_t)A.l_row.n;
        uint32_t* exec_of = (uint32_t*)malloc((nkn + 1) * sizeof(uint32_t));
        uint8_t* keep = (uint8_t*)malloc(nkn + 1);
        for (size_t q = 0; q < nkn; ++q) {
          uint32_t i = knodes[q].a;
          uint8_t f = c->flags[i];
          keep[q] = 0;
          exec_of[q] = NONE;
          if (is_sync_kernel(f)) {
            keep[q] = 1;
            exec_of[q] = i;
          } else if (!(f & XSP_F_CID)) {
            vu32_push(&o_row, i);
            vu8_push(&o_reason, XSP_O_LAUNCH_NO_CID);
          } else {
            size_t s = hmap_slot(&ex, c->cid[i]);
            if (!ex.used[s] || ex.val[s] == NONE) {
              vu32_push(&o_row, i);
              vu8_push(&o_reason, XSP_O_LAUNCH_NO_EXEC);
            } else {
              keep[q] = 1;
              exec_of[q] = ex.val[s];
              ex.val[s] = NONE; /* exec_by_cid.erase(found) */
            }
          }
        }
        /* launches outside the tree still consume their execs (:348-354) */
        for (uint64_t i = s0; i < s1; ++i) {
          uint8_t f = c->flags[i];
          if (is_kernel_launch(f) && (f & XSP_F_CID)) {
            size_t s = hmap_slot(&ex, c->cid[i]);
            if (ex.used[s]) ex.val[s] = NONE;
          }
        }
        vu32 left = {0};
        for (size_t s = 0; s <= ex.mask; ++s)
          if (ex.used[s] && ex.val[s] != NONE) vu32_push(&left, ex.val[s]);
        rec* lf = (rec*)malloc((left.n + 1) * sizeof(rec));
        for (size_t q = 0; q < left.n; ++q) {
          lf[q].k1 = c->span_id[left.v[q]];
          lf[q].k2 = left.v[q];
          lf[q].k3 = 0;
        }
        qsort(lf, left.n, sizeof(rec), rec_cmp);
        for (size_t q = 0; q < left.n; ++q) {
          vu32_push(&o_row, (uint32_t)lf[q].k2);
          vu8_push(&o_reason, XSP_O_EXEC_NO_LAUNCH);
        }
        free(lf);
        free(left.v);
        /* emit layers and kernels (tree order) */
        size_t q = 0;
        for (size_t j = 0; j < L; ++j) {
          uint32_t i = lr[j].a;
          vu32_push(&A.l_row, i);
          vu64_push(&A.l_dur, dur(c->begin_ns[i], c->end_ns[i]));
          vu32_push(&A.l_attr, arow[i]);
          while (q < nkn && knodes[q].k1 == j) {
            if (keep[q]) {
              uint32_t r = knodes[q].a, x = exec_of[q];
              vu32_push(&A.k_launch, r);
              vu32_push(&A.k_exec, x);
              vu32_push(&A.k_mrow, mrow[x]);
              vu64_push(&A.k_dur, dur(c->begin_ns[x], c->end_ns[x]));
              vu32_push(&A.k_name, c->name_id[x]);
              vf64_push(&A.k_occ, mrow[x] != NONE ? c->occupancy[mrow[x]] : 0.0);
            }
            ++q;
          }
          vu32_push(&A.l_koff, (uint32_t)A.k_launch.n);
        }
        (void)lbase;
        for (size_t j = 0; j < o_row.n; ++j) {
          vu32_push(&A.o_row, o_row.v[j]);
          vu8_push(&A.o_reason, o_reason.v[j]);
        }
        const uint32_t cbase = (uint32_t)A.a_crow.n;
        for (size_t j = 0; j < amb.n; ++j) {
          vu32_push(&A.a_row, amb.v[j]);
          vu32_push(&A.a_coff, cbase + amb_coff.v[j + 1]);
        }
        for (size_t j = 0; j < amb_cand.n; ++j) vu32_push(&A.a_crow, amb_cand.v[j]);
        free(exec_of);
        free(keep);
      }
      hmap_free(&ex);
      hmap_free(&la);
      free(lr);
      free(bysid);
      free(it.en);
      free(it.maxend);
    }
    free(knodes);
    free(o_row.v);
    free(o_reason.v);
    free(lay.v);
    free(amb.v);
    free(amb_cand.v);
    free(amb_coff.v);
    vi32_push(&A.status, status);
    vu32_push(&A.err, ea);
    vu32_push(&A.err, eb);
    vu32_push(&A.model, model == (uint64_t)-1 ? NONE : (uint32_t)model);
    vu32_push(&A.t_loff, (uint32_t)A.l_row.n);
    vu32_push(&A.t_koff, (uint32_t)A.k_launch.n);
    vu32_push(&A.t_ooff, (uint32_t)A.o_row.n);
    vu32_push(&A.t_aoff, (uint32_t)A.a_row.n);
  }
  free(mrow);
  free(arow);
  memset(out, 0, sizeof(*out));
  out->n_traces = T;
  out->n_failed = 0;
  for (uint32_t t = 0; t < T; ++t) out->n_failed += A.status.v[t] != XSP_T_OK;
  out->n_layers = A.l_row.n;
  out->n_kernels = A.k_launch.n;
  out->n_orphans = A.o_row.n;
  out->n_ambiguities = A.a_row.n;
  out->n_candidates = A.a_crow.n;
  out->trace_status = A.status.v;
  out->trace_err_row = A.err.v;
  out->trace_model_row = A.model.v;
  out->trace_layer_off = A.t_loff.v;
  out->trace_kernel_off = A.t_koff.v;
  out->trace_orphan_off = A.t_ooff.v;
  out->trace_amb_off = A.t_aoff.v;
  out->layer_row = A.l_row.v;
  out->layer_kernel_off = A.l_koff.v;
  out->layer_dur = A.l_dur.v;
  out->layer_attr_row = A.l_attr.v;
  out->kernel_launch_row = A.k_launch.v;
  out->kernel_exec_row = A.k_exec.v;
  out->kernel_metric_row = A.k_mrow.v;
  out->kernel_dur = A.k_dur.v;
  out->kernel_name = A.k_name.v;
  out->kernel_occ = A.k_occ.v;
  out->orphan_row = A.o_row.v;
  out->orphan_reason = A.o_reason.v;
  out->amb_row = A.a_row.v;
  out->amb_cand_off = A.a_coff.v;
  out->amb_cand_row = A.a_crow.v;
  return 0;
}

void xspo_corr_free(xsp_corr_out* o) {
  void* ps[] = {o->trace_status, o->trace_err_row, o->trace_model_row, o->trace_layer_off,
                o->trace_kernel_off, o->trace_orphan_off, o->trace_amb_off, o->layer_row,
                o->layer_kernel_off, o->layer_dur, o->layer_attr_row, o->kernel_launch_row,
                o->kernel_exec_row, o->kernel_metric_row, o->kernel_dur, o->kernel_name, o->kernel_occ,
                o->orphan_row, o->orphan_reason, o->amb_row, o->amb_cand_off, o->amb_cand_row};
  for (size_t i = 0; i < sizeof(ps) / sizeof(ps[0]); ++i) free(ps[i]);
  memset(o, 0, sizeof(*o));
}

/* ---- analysis ------------------------------------------------------------- */

static int dcmp(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}
/* trimmed_mean, analysis.cpp:28-39 */
static double trimmed_mean(double* v, size_t n, double f) {
  qsort(v, n, sizeof(double), dcmp);
  size_t drop = (size_t)floor(f * (double)n);
  double s = 0.0;
  for (size_t i = drop; i < n - drop; ++i) s += v[i];
  return s / (double)(n - 2 * drop);
}

/* arithmetic_intensity / throughput / ideal / classify, analysis.cpp:41-71 */
static void roof(uint64_t fl, uint64_t r, uint64_t w, double lat, double peak, double bw,
                 double* ai, double* tp, int8_t* bound) {
  double bytes = (double)r + (double)w;
  *ai = bytes <= 0.0 ? NAN : (double)fl / bytes;
  *tp = lat > 0.0 ? (double)fl / (lat / 1e9) : NAN;
  *bound = bytes <= 0.0 ? -1 : (int8_t)(*ai < peak / bw);
}

typedef struct {
  vi32 st;
  vu32 arg, goff_l, goff_k, goff_n;
  vu32 k_name, k_layer;
  vf64 k_lat, k_occ, k_ai, k_tput;
  vu64 k_flops, k_read, k_write;
  vi8 k_bound;
  vu8 k_in;
  vu32 l_index, l_row, l_topk;
  vf64 l_layer_lat, l_kern_lat, l_occ, l_ai, l_tput, l_nongpu, l_gs, l_ngs;
  vu64 l_flops, l_read, l_write, l_count;
  vi8 l_bound;
  vu8 l_flag, l_in;
  vu32 n_name;
  vu64 n_count, n_flops, n_read, n_write;
  vf64 n_lat, n_pct, n_occ, n_ai, n_tput;
  vi8 n_bound;
  vf64 m_lat, m_klat, m_occ, m_ai, m_tput, m_gpu, m_gpct, m_tp;
  vu64 m_flops, m_read, m_write, m_count;
  vi8 m_bound;
  vu8 m_in;
  vu32 goff_y, y_type;
  vu64 y_count, y_alloc;
  vf64 y_lat;
} tab_acc;

typedef struct {
  double lat;
  uint32_t name, ord;
} krow;
static int topk_cmp(const void* a, const void* b) {
  const krow* p = (const krow*)a;
  const krow* q = (const krow*)b;
  if (p->lat != q->lat) return p->lat > q->lat ? -1 : 1;
  return p->ord < q->ord ? -1 : (p->ord > q->ord ? 1 : 0);
}
static int name_cmp(const void* a, const void* b) {
  const krow* p = (const krow*)a;
  const krow* q = (const krow*)b;
  if (p->name != q->name) return p->name < q->name ? -1 : 1;
  return p->ord < q->ord ? -1 : (p->ord > q->ord ? 1 : 0);
}

int xspo_analyze(const xsp_span_cols* c, const xsp_corr_out* co, const xsp_groups* gr,
                 const xsp_system_spec* spec, const xsp_analysis_opts* o, xsp_tables_out* out) {
  tab_acc A;
  memset(&A, 0, sizeof(A));
  const double peak = spec->peak_flops, bw = spec->memory_bandwidth_bytes_per_s;
  const uint32_t K = o->top_k;
  vu32_push(&A.goff_l, 0);
  vu32_push(&A.goff_k, 0);
  vu32_push(&A.goff_n, 0);
  vu32_push(&A.goff_y, 0);
  for (uint32_t g = 0; g < gr->n_groups; ++g) {
    const uint32_t t0 = gr->first_trace[g], R = gr->n_runs[g];
    int32_t st = XSP_G_OK;
    uint32_t arg = 0;
    /* combine() preconditions, analysis.cpp:103-118 */
    if (R == 0) st = XSP_G_NO_RUNS;
    for (uint32_t r = 0; r < R && st == XSP_G_OK; ++r)
      if (co->trace_status[t0 + r] != XSP_T_OK) st = XSP_G_TRACE_FAILED;
    uint32_t L0 = 0;
    if (st == XSP_G_OK) {
      L0 = co->trace_layer_off[t0 + 1] - co->trace_layer_off[t0];
      for (uint32_t r = 0; r < R && st == XSP_G_OK; ++r) {
        uint32_t t = t0 + r;
        if (co->trace_layer_off[t + 1] - co->trace_layer_off[t] != L0) {
          st = XSP_G_LAYER_COUNT;
          break;
        }
        for (uint32_t li = 0; li < L0; ++li) {
          uint32_t a = co->trace_layer_off[t] + li, b = co->trace_layer_off[t0] + li;
          if (co->layer_kernel_off[a + 1] - co->layer_kernel_off[a] !=
              co->layer_kernel_off[b + 1] - co->layer_kernel_off[b]) {
            st = XSP_G_KERNEL_COUNT;
            arg = li;
            break;
          }
        }
      }
      if (st == XSP_G_OK && !(o->trim_fraction >= 0.0 && o->trim_fraction < 0.5)) st = XSP_G_BAD_TRIM;
    }
    vi32_push(&A.st, st);
    vu32_push(&A.arg, arg);
    if (st != XSP_G_OK) {
      vu32_push(&A.goff_l, (uint32_t)A.l_index.n);
      vu32_push(&A.goff_k, (uint32_t)A.k_lat.n);
      vu32_push(&A.goff_n, (uint32_t)A.n_name.n);
      vu32_push(&A.goff_y, (uint32_t)A.y_type.n);
      vf64_push(&A.m_lat, NAN);
      vf64_push(&A.m_klat, 0);
      vu64_push(&A.m_flops, 0);
      vu64_push(&A.m_read, 0);
      vu64_push(&A.m_write, 0);
      vf64_push(&A.m_occ, 0);
      vu64_push(&A.m_count, 0);
      vf64_push(&A.m_ai, NAN);
      vf64_push(&A.m_tput, NAN);
      vi8_push(&A.m_bound, -1);
      vf64_push(&A.m_gpu, 0);
      vf64_push(&A.m_gpct, 0);
      vf64_push(&A.m_tp, 0);
      vu8_push(&A.m_in, 0);
      continue;
    }
    double* v = (double*)malloc((R + 1) * sizeof(double));
    double* w = (double*)malloc((R + 1) * sizeof(double));
    /* model latency (analysis.cpp:126-133) */
    for (uint32_t r = 0; r < R; ++r) {
      uint32_t m = co->trace_model_row[t0 + r];
      v[r] = (double)dur(c->begin_ns[m], c->end_ns[m]);
    }
    const double mlat = trimmed_mean(v, R, o->trim_fraction);
    const size_t kbase = A.k_lat.n;
    const uint32_t tk0 = co->trace_kernel_off[t0];
    double model_gpu = 0.0;
    const size_t ybase = A.y_type.n;
    for (uint32_t li = 0; li < L0; ++li) {
      for (uint32_t r = 0; r < R; ++r) v[r] = (double)co->layer_dur[co->trace_layer_off[t0 + r] + li];
      const double llat = trimmed_mean(v, R, o->trim_fraction);
      const uint32_t gl0 = co->trace_layer_off[t0] + li;
      {
        /* a5-a7 by layer type (analysis.cpp:315-337): accumulate in execution order */
        const uint32_t ar0 = co->layer_attr_row[gl0];
        const uint32_t ty = c->type_id[ar0];
        size_t y = ybase;
        while (y < A.y_type.n && A.y_type.v[y] != ty) ++y;
        if (y == A.y_type.n) {
          vu32_push(&A.y_type, ty);
          vu64_push(&A.y_count, 0);
          vf64_push(&A.y_lat, 0.0);
          vu64_push(&A.y_alloc, 0);
        }
        A.y_count.v[y] += 1;
        A.y_lat.v[y] += llat;
        A.y_alloc.v[y] += (uint64_t)c->alloc_bytes[ar0];
      }
      double acc_lat = 0.0, acc_occw = 0.0;
      uint64_t af = 0, ar = 0, aw = 0, an = 0;
      krow* kr = (krow*)malloc((co->layer_kernel_off[gl0 + 1] - co->layer_kernel_off[gl0] + 1) * sizeof(krow));
      size_t nk = 0;
      for (uint32_t j = co->layer_kernel_off[gl0]; j < co->layer_kernel_off[gl0 + 1]; ++j) {
        uint32_t ord = j - tk0;
        for (uint32_t r = 0; r < R; ++r) {
          uint32_t jr = co->trace_kernel_off[t0 + r] + ord;
          v[r] = (double)co->kernel_dur[jr];
          uint32_t mr = co->kernel_metric_row[jr];
          w[r] = mr != NONE ? c->occupancy[mr] : 0.0;
        }
        double klat = trimmed_mean(v, R, o->trim_fraction);
        double kocc = trimmed_mean(w, R, o->trim_fraction);
        uint64_t fl = 0, rd = 0, wr = 0;
        uint32_t mr0 = co->kernel_metric_row[j];
        if (mr0 != NONE) {
          fl = c->flops[mr0];
          rd = c->dram_read[mr0];
          wr = c->dram_write[mr0];
        }
        double ai, tp;
        int8_t bd;
        roof(fl, rd, wr, klat, peak, bw, &ai, &tp, &bd);
        vu32_push(&A.k_name, co->kernel_name[j]);
        vu32_push(&A.k_layer, li);
        vf64_push(&A.k_lat, klat);
        vu64_push(&A.k_flops, fl);
        vu64_push(&A.k_read, rd);
        vu64_push(&A.k_write, wr);
        vf64_push(&A.k_occ, kocc);
        vf64_push(&A.k_ai, ai);
        vf64_push(&A.k_tput, tp);
        vi8_push(&A.k_bound, bd);
        vu8_push(&A.k_in, bd >= 0 && klat > 0.0);
        /* Accumulator::add, analysis.cpp:181-188 */
        acc_lat += klat;
        af += fl;
        ar += rd;
        aw += wr;
        acc_occw += kocc * klat;
        ++an;
        kr[nk].lat = klat;
        kr[nk].ord = ord;
        kr[nk].name = co->kernel_name[j];
        ++nk;
      }
      double ai, tp;
      int8_t bd;
      roof(af, ar, aw, acc_lat, peak, bw, &ai, &tp, &bd);
      vu32_push(&A.l_index, li);
      vu32_push(&A.l_row, co->layer_row[gl0]);
      vf64_push(&A.l_layer_lat, llat);
      vf64_push(&A.l_kern_lat, acc_lat);
      vu64_push(&A.l_flops, af);
      vu64_push(&A.l_read, ar);
      vu64_push(&A.l_write, aw);
      vf64_push(&A.l_occ, acc_lat > 0.0 ? acc_occw / acc_lat : 0.0);
      vu64_push(&A.l_count, an);
      vf64_push(&A.l_ai, ai);
      vf64_push(&A.l_tput, tp);
      vi8_push(&A.l_bound, bd);
      vu8_push(&A.l_in, bd >= 0 && acc_lat > 0.0);
      /* a13, analysis.cpp:484-494 */
      double ng = llat - acc_lat;
      vf64_push(&A.l_nongpu, ng);
      vf64_push(&A.l_gs, llat > 0.0 ? acc_lat / llat : 0.0);
      vf64_push(&A.l_ngs, llat > 0.0 ? ng / llat : 0.0);
      vu8_push(&A.l_flag, ng < -(o->noise_tolerance * llat));
      model_gpu += acc_lat;
      /* top-k: latency desc, ordinal asc */
      qsort(kr, nk, sizeof(krow), topk_cmp);
      for (uint32_t s = 0; s < K; ++s) vu32_push(&A.l_topk, s < nk ? kr[s].ord : NONE);
      free(kr);
    }
    /* a15 accumulator over all kernels in tree order (analysis.cpp:536-552) */
    double lat = 0.0, occw = 0.0;
    uint64_t f = 0, rd = 0, wr = 0, cnt = 0;
    const size_t kend = A.k_lat.n;
    for (size_t j = kbase; j < kend; ++j) {
      lat += A.k_lat.v[j];
      f += A.k_flops.v[j];
      rd += A.k_read.v[j];
      wr += A.k_write.v[j];
      occw += A.k_occ.v[j] * A.k_lat.v[j];
      ++cnt;
    }
    double ai, tp;
    int8_t bd;
    roof(f, rd, wr, lat, peak, bw, &ai, &tp, &bd);
    vf64_push(&A.m_lat, mlat);
    vf64_push(&A.m_klat, lat);
    vu64_push(&A.m_flops, f);
    vu64_push(&A.m_read, rd);
    vu64_push(&A.m_write, wr);
    vf64_push(&A.m_occ, lat > 0.0 ? occw / lat : 0.0);
    vu64_push(&A.m_count, cnt);
    vf64_push(&A.m_ai, ai);
    vf64_push(&A.m_tput, tp);
    vi8_push(&A.m_bound, bd);
    vf64_push(&A.m_gpu, model_gpu);
    vf64_push(&A.m_gpct, model_gpu / mlat * 100.0);
    vf64_push(&A.m_tp, (double)gr->batch_size[g] / (mlat / 1e9));
    vu8_push(&A.m_in, bd >= 0 && lat > 0.0);
    /* a10 by name, analysis.cpp:399-432 */
    krow* byname = (krow*)malloc((kend - kbase + 1) * sizeof(krow));
    for (size_t j = kbase; j < kend; ++j) {
      byname[j - kbase].name = A.k_name.v[j];
      byname[j - kbase].ord = (uint32_t)(j - kbase);
      byname[j - kbase].lat = 0;
    }
    qsort(byname, kend - kbase, sizeof(krow), name_cmp);
    const size_t nbase = A.n_name.n;
    for (size_t q = 0; q < kend - kbase;) {
      uint32_t nm = byname[q].name;
      double nl = 0.0, no = 0.0;
      uint64_t nf = 0, nr = 0, nw = 0, nc = 0;
      for (; q < kend - kbase && byname[q].name == nm; ++q) {
        size_t j = kbase + byname[q].ord;
        nl += A.k_lat.v[j];
        nf += A.k_flops.v[j];
        nr += A.k_read.v[j];
        nw += A.k_write.v[j];
        no += A.k_occ.v[j] * A.k_lat.v[j];
        ++nc;
      }
      roof(nf, nr, nw, nl, peak, bw, &ai, &tp, &bd);
      vu32_push(&A.n_name, nm);
      vu64_push(&A.n_count, nc);
      vf64_push(&A.n_lat, nl);
      vf64_push(&A.n_pct, nl / mlat * 100.0);
      vu64_push(&A.n_flops, nf);
      vu64_push(&A.n_read, nr);
      vu64_push(&A.n_write, nw);
      vf64_push(&A.n_occ, nl > 0.0 ? no / nl : 0.0);
      vf64_push(&A.n_ai, ai);
      vf64_push(&A.n_tput, tp);
      vi8_push(&A.n_bound, bd);
    }
    /* rows by total latency desc, name asc: insertion sort of this group's rows */
    for (size_t i = nbase + 1; i < A.n_name.n; ++i) {
      for (size_t j = i; j > nbase && A.n_lat.v[j - 1] < A.n_lat.v[j]; --j) {
#define SWAP(vec, T)                 \
  do {                               \
    T tmp_ = vec.v[j];               \
    vec.v[j] = vec.v[j - 1];         \
    vec.v[j - 1] = tmp_;             \
  } while (0)
        SWAP(A.n_name, uint32_t);
        SWAP(A.n_count, uint64_t);
        SWAP(A.n_lat, double);
        SWAP(A.n_pct, double);
        SWAP(A.n_flops, uint64_t);
        SWAP(A.n_read, uint64_t);
        SWAP(A.n_write, uint64_t);
        SWAP(A.n_occ, double);
        SWAP(A.n_ai, double);
        SWAP(A.n_tput, double);
        SWAP(A.n_bound, int8_t);
#undef SWAP
      }
    }
    free(byname);
    /* a5 rows: total latency desc, then type asc (std::map order + stable_sort) */
    for (size_t i = ybase + 1; i < A.y_type.n; ++i) {
      for (size_t j = i; j > ybase && (A.y_lat.v[j - 1] < A.y_lat.v[j] ||
                                       (A.y_lat.v[j - 1] == A.y_lat.v[j] && A.y_type.v[j - 1] > A.y_type.v[j]));
           --j) {
#define SWAPY(vec, T)                \
  do {                               \
    T tmp_ = vec.v[j];               \
    vec.v[j] = vec.v[j - 1];         \
    vec.v[j - 1] = tmp_;             \
  } while (0)
        SWAPY(A.y_type, uint32_t);
        SWAPY(A.y_count, uint64_t);
        SWAPY(A.y_lat, double);
        SWAPY(A.y_alloc, uint64_t);
#undef SWAPY
      }
    }
    free(v);
    free(w);
    vu32_push(&A.goff_y, (uint32_t)A.y_type.n);
    vu32_push(&A.goff_l, (uint32_t)A.l_index.n);
    vu32_push(&A.goff_k, (uint32_t)A.k_lat.n);
    vu32_push(&A.goff_n, (uint32_t)A.n_name.n);
  }
  memset(out, 0, sizeof(*out));
  out->n_groups = gr->n_groups;
  out->n_layers = A.l_index.n;
  out->n_kernels = A.k_lat.n;
  out->n_names = A.n_name.n;
  out->group_status = A.st.v;
  out->group_err_arg = A.arg.v;
  out->group_layer_off = A.goff_l.v;
  out->group_kernel_off = A.goff_k.v;
  out->group_name_off = A.goff_n.v;
  out->k_name = A.k_name.v;
  out->k_layer = A.k_layer.v;
  out->k_lat = A.k_lat.v;
  out->k_flops = A.k_flops.v;
  out->k_read = A.k_read.v;
  out->k_write = A.k_write.v;
  out->k_occ = A.k_occ.v;
  out->k_ai = A.k_ai.v;
  out->k_tput = A.k_tput.v;
  out->k_bound = A.k_bound.v;
  out->k_roofline_in = A.k_in.v;
  out->l_index = A.l_index.v;
  out->l_row = A.l_row.v;
  out->l_layer_lat = A.l_layer_lat.v;
  out->l_kern_lat = A.l_kern_lat.v;
  out->l_flops = A.l_flops.v;
  out->l_read = A.l_read.v;
  out->l_write = A.l_write.v;
  out->l_occ = A.l_occ.v;
  out->l_count = A.l_count.v;
  out->l_ai = A.l_ai.v;
  out->l_tput = A.l_tput.v;
  out->l_bound = A.l_bound.v;
  out->l_nongpu = A.l_nongpu.v;
  out->l_gpu_share = A.l_gs.v;
  out->l_nongpu_share = A.l_ngs.v;
  out->l_flagged = A.l_flag.v;
  out->l_roofline_in = A.l_in.v;
  out->l_topk = A.l_topk.v;
  out->n_name = A.n_name.v;
  out->n_count = A.n_count.v;
  out->n_lat = A.n_lat.v;
  out->n_pct = A.n_pct.v;
  out->n_flops = A.n_flops.v;
  out->n_read = A.n_read.v;
  out->n_write = A.n_write.v;
  out->n_occ = A.n_occ.v;
  out->n_ai = A.n_ai.v;
  out->n_tput = A.n_tput.v;
  out->n_bound = A.n_bound.v;
  out->m_lat = A.m_lat.v;
  out->m_kern_lat = A.m_klat.v;
  out->m_flops = A.m_flops.v;
  out->m_read = A.m_read.v;
  out->m_write = A.m_write.v;
  out->m_occ = A.m_occ.v;
  out->m_count = A.m_count.v;
  out->m_ai = A.m_ai.v;
  out->m_tput = A.m_tput.v;
  out->m_bound = A.m_bound.v;
  out->m_gpu = A.m_gpu.v;
  out->m_gpu_pct = A.m_gpct.v;
  out->m_throughput = A.m_tp.v;
  out->m_roofline_in = A.m_in.v;
  out->n_type_rows = A.y_type.n;
  out->group_type_off = A.goff_y.v;
  out->y_type = A.y_type.v;
  out->y_count = A.y_count.v;
  out->y_lat = A.y_lat.v;
  out->y_alloc = (int64_t*)A.y_alloc.v;
  return 0;
}

void xspo_tables_free(xsp_tables_out* o) {
  void* ps[] = {o->group_status, o->group_err_arg, o->group_layer_off, o->group_kernel_off,
                o->group_name_off, o->k_name, o->k_layer, o->k_lat, o->k_flops, o->k_read,
                o->k_write, o->k_occ, o->k_ai, o->k_tput, o->k_bound, o->k_roofline_in,
                o->l_index, o->l_row, o->l_layer_lat, o->l_kern_lat, o->l_flops, o->l_read,
                o->l_write, o->l_occ, o->l_count, o->l_ai, o->l_tput, o->l_bound, o->l_nongpu,
                o->l_gpu_share, o->l_nongpu_share, o->l_flagged, o->l_roofline_in, o->l_topk,
                o->n_name, o->n_count, o->n_lat, o->n_pct, o->n_flops, o->n_read, o->n_write,
                o->n_occ, o->n_ai, o->n_tput, o->n_bound, o->m_lat, o->m_kern_lat, o->m_flops,
                o->m_read, o->m_write, o->m_occ, o->m_count, o->m_ai, o->m_tput, o->m_bound,
                o->m_gpu, o->m_gpu_pct, o->m_throughput, o->m_roofline_in, o->group_type_off,
                o->y_type, o->y_count, o->y_lat, o->y_alloc};
  for (size_t i = 0; i < sizeof(ps) / sizeof(ps[0]); ++i) free(ps[i]);
  memset(o, 0, sizeof(*o));
}

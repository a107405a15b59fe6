/* TEST INFRASTRUCTURE ONLY — see restate.h. Plain C11, single-threaded.
 *
 * The list placer is restated in its "exact argmin" form: at every step the
 * lexicographic minimum of (key, node, device) over all live pairs is
 * committed or discarded. The reference reaches the same sequence through a
 * lazy min-heap with explicit re-pushes (proj/src/placers.cpp:188-202,
 * 242, 253, 271-279); SURVEY.md finding 1 proves and measures the
 * equivalence. This form has no heap, so it checks the GPU kernel (which
 * uses the same form) against an independent sequential implementation.
 */
#include "restate.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define RS_OK 0
#define RS_VALIDATION 2
#define RS_INFEASIBLE 3

static int fail(char *msg, int msglen, int code, const char *text) {
  if (msg && msglen > 0) snprintf(msg, (size_t)msglen, "%s", text);
  return code;
}

static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
static int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

/* proj/src/cost_model.cpp:18-20 (round half up) and :30-36 (comm_time).
 * Multiply and add are kept as two separately rounded double ops. */
int64_t rs_comm_time(double intercept, double per_byte, int64_t bytes, int *err) {
  if (bytes < 0) {
    if (err) *err = RS_VALIDATION;
    return 0;
  }
  if (err) *err = RS_OK;
  volatile double prod = per_byte * (double)bytes;
  volatile double sum = intercept + prod;
  return (int64_t)floor(sum + 0.5);
}

/* ---- CSR over the sorted meta edges (transforms.hpp:56-60) ------------- */
typedef struct {
  int32_t *in_off, *in_edge, *out_off, *out_edge;
} csr_t;

static void csr_build(const rs_graph *g, csr_t *c) {
  int V = g->V, E = g->E;
  c->in_off = calloc((size_t)V + 1, sizeof(int32_t));
  c->out_off = calloc((size_t)V + 1, sizeof(int32_t));
  c->in_edge = malloc(sizeof(int32_t) * (size_t)(E > 0 ? E : 1));
  c->out_edge = malloc(sizeof(int32_t) * (size_t)(E > 0 ? E : 1));
  for (int e = 0; e < E; ++e) {
    c->in_off[g->edst[e] + 1]++;
    c->out_off[g->esrc[e] + 1]++;
  }
  for (int v = 0; v < V; ++v) {
    c->in_off[v + 1] += c->in_off[v];
    c->out_off[v + 1] += c->out_off[v];
  }
  int32_t *ip = malloc(sizeof(int32_t) * (size_t)(V > 0 ? V : 1));
  int32_t *op = malloc(sizeof(int32_t) * (size_t)(V > 0 ? V : 1));
  memcpy(ip, c->in_off, sizeof(int32_t) * (size_t)V);
  memcpy(op, c->out_off, sizeof(int32_t) * (size_t)V);
  /* ascending edge index inside every list, as GroupedGraph builds them */
  for (int e = 0; e < E; ++e) {
    c->in_edge[ip[g->edst[e]]++] = e;
    c->out_edge[op[g->esrc[e]]++] = e;
  }
  free(ip);
  free(op);
}

static void csr_free(csr_t *c) {
  free(c->in_off);
  free(c->in_edge);
  free(c->out_off);
  free(c->out_edge);
}

/* ---- binary min-heap of ints (Kahn with smallest index first) --------- */
typedef struct {
  int32_t *a;
  int n;
} iheap;

static void ih_push(iheap *h, int32_t v) {
  int i = h->n++;
  h->a[i] = v;
  while (i > 0) {
    int p = (i - 1) / 2;
    if (h->a[p] <= h->a[i]) break;
    int32_t t = h->a[p];
    h->a[p] = h->a[i];
    h->a[i] = t;
    i = p;
  }
}

static int32_t ih_pop(iheap *h) {
  int32_t top = h->a[0];
  h->a[0] = h->a[--h->n];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && h->a[l] < h->a[m]) m = l;
    if (r < h->n && h->a[r] < h->a[m]) m = r;
    if (m == i) break;
    int32_t t = h->a[m];
    h->a[m] = h->a[i];
    h->a[i] = t;
    i = m;
  }
  return top;
}

/* proj/src/transforms.cpp:446-479 (meta_topo_order). Returns count placed;
 * on a cycle writes the reference's CycleError text. */
static int topo_impl(const rs_graph *g, const csr_t *c, int32_t *order,
                     char *msg, int msglen) {
  int V = g->V;
  int32_t *indeg = calloc((size_t)(V > 0 ? V : 1), sizeof(int32_t));
  for (int e = 0; e < g->E; ++e) indeg[g->edst[e]]++;
  iheap h = {malloc(sizeof(int32_t) * (size_t)(V > 0 ? V : 1)), 0};
  for (int i = 0; i < V; ++i)
    if (indeg[i] == 0) ih_push(&h, i);
  int cnt = 0;
  while (h.n > 0) {
    int u = ih_pop(&h);
    order[cnt++] = u;
    for (int x = c->out_off[u]; x < c->out_off[u + 1]; ++x) {
      int v = g->edst[c->out_edge[x]];
      if (--indeg[v] == 0) ih_push(&h, v);
    }
  }
  int rc = RS_OK;
  if (cnt != V) {
    size_t cap = 128 + (size_t)V * 24;
    char *buf = malloc(cap);
    size_t len = (size_t)snprintf(buf, cap, "meta graph is cyclic; groups of base node ids {");
    int first = 1;
    for (int i = 0; i < V; ++i) {
      if (indeg[i] > 0) {
        long long id = g->first_id ? (long long)g->first_id[i] : (long long)i;
        len += (size_t)snprintf(buf + len, cap - len, "%s%lld", first ? "" : ", ", id);
        first = 0;
      }
    }
    snprintf(buf + len, cap - len, "} remain");
    fail(msg, msglen, RS_VALIDATION, buf);
    free(buf);
    rc = RS_VALIDATION;
  }
  free(indeg);
  free(h.a);
  return rc;
}

int rs_topo_order(const rs_graph *g, int32_t *order, char *msg, int msglen) {
  csr_t c;
  csr_build(g, &c);
  int rc = topo_impl(g, &c, order, msg, msglen);
  csr_free(&c);
  return rc;
}

/* ---- placer state (proj/include/dagsched/placers.hpp:49-60) ----------- */
typedef struct {
  int V, n, mode;
  int64_t *dev_free, *tail, *fin, *cache, *c_e;
  int32_t *dev_of;
} pstate;

/* proj/src/placers.cpp:43-79 (schedulable_time_impl). `tail` is either the
 * live queue tails (commit) or a scratch copy (estimate). */
static int64_t sched_time(pstate *st, const rs_graph *g, const csr_t *c, int j,
                          int p, int64_t *tail, int commit) {
  int n = st->n;
  int64_t t = st->dev_free[p];
  for (int x = c->in_off[j]; x < c->in_off[j + 1]; ++x) {
    int e = c->in_edge[x];
    int i = g->esrc[e];
    int q = st->dev_of[i];
    int64_t term;
    if (q == p) {
      term = st->fin[i];
    } else {
      int64_t cached = st->cache[(size_t)i * n + p];
      if (cached >= 0) {
        term = max64(st->fin[i], cached);
      } else {
        int64_t cc = st->c_e[e];
        if (st->mode == 1) {
          term = st->fin[i] + cc;
        } else {
          int64_t begin = max64(st->fin[i], max64(tail[q], tail[p]));
          term = begin + cc;
          tail[q] = term;
          tail[p] = term;
        }
        if (commit) st->cache[(size_t)i * n + p] = term;
      }
    }
    t = max64(t, term);
  }
  return t;
}

static int cmp_start(const void *a, const void *b) {
  const int64_t *x = a, *y = b;
  if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
  return x[1] < y[1] ? -1 : (x[1] > y[1] ? 1 : 0);
}

/* proj/src/placers.cpp:282-294: exec_order = nodes by (start, index). */
static void emit_exec_order(int V, int n, const int64_t *start,
                            const int32_t *dev_of, int32_t *exec_order,
                            int32_t *exec_off) {
  int64_t *pairs = malloc(sizeof(int64_t) * 2 * (size_t)(V > 0 ? V : 1));
  for (int j = 0; j < V; ++j) {
    pairs[2 * j] = start[j];
    pairs[2 * j + 1] = j;
  }
  qsort(pairs, (size_t)V, 2 * sizeof(int64_t), cmp_start);
  int32_t *cnt = calloc((size_t)n + 1, sizeof(int32_t));
  for (int j = 0; j < V; ++j) cnt[dev_of[j] + 1]++;
  exec_off[0] = 0;
  for (int d = 0; d < n; ++d) exec_off[d + 1] = exec_off[d] + cnt[d + 1];
  int32_t *pos = calloc((size_t)n, sizeof(int32_t));
  for (int d = 0; d < n; ++d) pos[d] = exec_off[d];
  for (int x = 0; x < V; ++x) {
    int j = (int)pairs[2 * x + 1];
    exec_order[pos[dev_of[j]]++] = j;
  }
  free(pairs);
  free(cnt);
  free(pos);
}

static int roster_check(int n, const int64_t *caps, int64_t *min_cap, char *msg,
                        int msglen) {
  /* DeviceRoster::min_capacity, proj/src/placers.cpp:19-29 */
  if (n <= 0) return fail(msg, msglen, RS_VALIDATION, "device roster is empty");
  int64_t m = caps[0];
  for (int d = 0; d < n; ++d) m = min64(m, caps[d]);
  if (m <= 0)
    return fail(msg, msglen, RS_VALIDATION, "device capacities must be positive");
  *min_cap = m;
  return RS_OK;
}

static int place_topo(const rs_graph *g, const csr_t *c, int n,
                      const int64_t *caps, int mode, int64_t *c_e,
                      int32_t *device_of, int64_t *start, int32_t *exec_order,
                      int32_t *exec_off, char *msg, int msglen) {
  /* proj/src/placers.cpp:314-365 */
  int V = g->V;
  int64_t total = 0, largest = 0;
  for (int j = 0; j < V; ++j) {
    int64_t b = g->perm[j] + g->out[j] + g->temp[j];
    total += b;
    largest = max64(largest, b);
  }
  if (n <= 0) return fail(msg, msglen, RS_VALIDATION, "device roster is empty");
  int64_t cap = (total + n - 1) / n + largest;
  int64_t min_cap;
  int rc = roster_check(n, caps, &min_cap, msg, msglen);
  if (rc) return rc;
  if (cap > min_cap) {
    char buf[256];
    snprintf(buf, sizeof buf,
             "m-topo per-device cap %lld bytes exceeds the smallest device "
             "capacity %lld; use m-etf or m-sct for tight memory limits",
             (long long)cap, (long long)min_cap);
    return fail(msg, msglen, RS_INFEASIBLE, buf);
  }
  int32_t *order = malloc(sizeof(int32_t) * (size_t)(V > 0 ? V : 1));
  rc = topo_impl(g, c, order, msg, msglen);
  if (rc) {
    free(order);
    return rc;
  }
  int dev = 0;
  int64_t used = 0;
  int32_t *cnt = calloc((size_t)n, sizeof(int32_t));
  for (int x = 0; x < V; ++x) {
    int j = order[x];
    int64_t b = g->perm[j] + g->out[j] + g->temp[j];
    if (used + b > cap && dev + 1 < n) {
      ++dev;
      used = 0;
    }
    device_of[j] = dev;
    cnt[dev]++;
    used += b;
  }
  exec_off[0] = 0;
  for (int d = 0; d < n; ++d) exec_off[d + 1] = exec_off[d] + cnt[d];
  for (int d = 0; d < n; ++d) cnt[d] = exec_off[d];
  for (int x = 0; x < V; ++x) exec_order[cnt[device_of[order[x]]]++] = order[x];

  pstate st = {V, n, mode, calloc((size_t)n, 8), calloc((size_t)n, 8),
               calloc((size_t)(V > 0 ? V : 1), 8),
               malloc(8 * (size_t)(V > 0 ? V : 1) * (size_t)n), c_e,
               malloc(4 * (size_t)(V > 0 ? V : 1))};
  for (size_t x = 0; x < (size_t)V * (size_t)n; ++x) st.cache[x] = -1;
  for (int j = 0; j < V; ++j) st.dev_of[j] = -1;
  for (int x = 0; x < V; ++x) {
    int j = order[x];
    int p = device_of[j];
    st.dev_of[j] = p;
    int64_t t = sched_time(&st, g, c, j, p, st.tail, 1);
    t = max64(t, st.dev_free[p]);
    start[j] = t;
    st.fin[j] = t + g->k[j];
    st.dev_free[p] = st.fin[j];
  }
  free(st.dev_free);
  free(st.tail);
  free(st.fin);
  free(st.cache);
  free(st.dev_of);
  free(cnt);
  free(order);
  return RS_OK;
}

int rs_place(const rs_graph *g, int32_t algo, int32_t n, const int64_t *caps,
             double intercept, double per_byte, int32_t mode,
             const int32_t *fav_child, int32_t *device_of, int64_t *start,
             int32_t *exec_order, int32_t *exec_off, int64_t *stats3, char *msg,
             int msglen) {
  const int V = g->V;
  csr_t c;
  csr_build(g, &c);
  int64_t *c_e = malloc(8 * (size_t)(g->E > 0 ? g->E : 1));
  int64_t c_max = 0;
  for (int e = 0; e < g->E; ++e) {
    int err;
    c_e[e] = rs_comm_time(intercept, per_byte, g->ebytes[e], &err);
    if (err) {
      free(c_e);
      csr_free(&c);
      return fail(msg, msglen, RS_VALIDATION, "comm_time: negative byte count");
    }
    c_max = max64(c_max, c_e[e]);
  }
  if (stats3) stats3[0] = stats3[1] = stats3[2] = 0;
  if (algo == 0) {
    int rc = place_topo(g, &c, n, caps, mode, c_e, device_of, start, exec_order,
                        exec_off, msg, msglen);
    free(c_e);
    csr_free(&c);
    return rc;
  }

  /* place_list, proj/src/placers.cpp:115-295 */
  int64_t min_cap;
  int rc = roster_check(n, caps, &min_cap, msg, msglen);
  if (rc) {
    free(c_e);
    csr_free(&c);
    return rc;
  }
  {
    int32_t *order = malloc(sizeof(int32_t) * (size_t)(V > 0 ? V : 1));
    rc = topo_impl(g, &c, order, msg, msglen); /* :121 validates acyclicity */
    free(order);
    if (rc) {
      free(c_e);
      csr_free(&c);
      return rc;
    }
  }
  size_t Vn = (size_t)(V > 0 ? V : 1) * (size_t)n;
  pstate st = {V, n, mode, calloc((size_t)n, 8), calloc((size_t)n, 8),
               calloc((size_t)(V > 0 ? V : 1), 8), malloc(8 * Vn), c_e,
               malloc(4 * (size_t)(V > 0 ? V : 1))};
  for (size_t x = 0; x < Vn; ++x) st.cache[x] = -1;
  for (int j = 0; j < V; ++j) st.dev_of[j] = -1;
  int64_t *need = malloc(8 * (size_t)(V > 0 ? V : 1));
  int64_t *reserved = calloc((size_t)n, 8);
  char *placed = calloc((size_t)(V > 0 ? V : 1), 1);
  char *dead = calloc(Vn, 1);
  char *ready = calloc((size_t)(V > 0 ? V : 1), 1);
  int32_t *alive = malloc(4 * (size_t)(V > 0 ? V : 1));
  int32_t *pending = calloc((size_t)(V > 0 ? V : 1), 4);
  int64_t *urgent = calloc((size_t)(V > 0 ? V : 1), 8);
  int32_t *awake_for = malloc(4 * (size_t)n);
  int64_t *awake_until = calloc((size_t)n, 8);
  int64_t *scratch = malloc(8 * (size_t)n);
  int64_t discarded = 0, excluded = 0, awake = 0;
  for (int j = 0; j < V; ++j) {
    need[j] = g->perm[j] + g->out[j] + g->temp[j];
    alive[j] = n;
    start[j] = 0;
  }
  for (int e = 0; e < g->E; ++e) pending[g->edst[e]]++;
  for (int j = 0; j < V; ++j) ready[j] = pending[j] == 0;
  for (int d = 0; d < n; ++d) awake_for[d] = -1;

  int placed_count = 0;
  char buf[160];
  rc = RS_OK;
  while (placed_count < V) {
    /* exact argmin over live pairs; keys per pair_key, :147-156 */
    int64_t bt = 0;
    int bj = -1, bp = -1;
    for (int j = 0; j < V; ++j) {
      if (!ready[j] || placed[j]) continue;
      for (int p = 0; p < n; ++p) {
        if (dead[(size_t)j * n + p]) continue;
        memcpy(scratch, st.tail, 8 * (size_t)n);
        int64_t t = sched_time(&st, g, &c, j, p, scratch, 0);
        if (awake_for[p] >= 0 && awake_for[p] != j)
          t = max64(t, min64(awake_until[p], urgent[j]));
        if (bj < 0 || t < bt) { /* (t, j, p) ascending: j, p scanned in order */
          bt = t;
          bj = j;
          bp = p;
        }
      }
    }
    if (bj < 0) {
      rc = fail(msg, msglen, RS_INFEASIBLE, "no schedulable (node, device) pair remains");
      break;
    }
    int j = bj, p = bp;
    int64_t t = bt;
    if (reserved[p] + need[j] > caps[p]) {
      /* discard, :203-219 */
      dead[(size_t)j * n + p] = 1;
      if (--alive[j] == 0) {
        snprintf(buf, sizeof buf, "node %d fits on no device", j);
        rc = fail(msg, msglen, RS_INFEASIBLE, buf);
        break;
      }
      discarded++;
      int have = 0;
      int64_t min_rem = 0;
      for (int x = 0; x < V; ++x) {
        if (placed[x]) continue;
        if (!have || need[x] < min_rem) min_rem = need[x];
        have = 1;
      }
      if (have && reserved[p] + min_rem > caps[p]) {
        excluded++;
        for (int j2 = 0; j2 < V && rc == RS_OK; ++j2) {
          if (!placed[j2] && !dead[(size_t)j2 * n + p]) {
            dead[(size_t)j2 * n + p] = 1;
            if (--alive[j2] == 0) {
              snprintf(buf, sizeof buf, "node %d fits on no device", j2);
              rc = fail(msg, msglen, RS_INFEASIBLE, buf);
            }
          }
        }
        if (rc) break;
      }
      continue;
    }
    /* commit, :221-233 */
    st.dev_of[j] = p;
    start[j] = t;
    st.fin[j] = t + g->k[j];
    sched_time(&st, g, &c, j, p, st.tail, 1);
    st.dev_free[p] = st.fin[j];
    reserved[p] += need[j];
    placed[j] = 1;
    ++placed_count;
    if (fav_child) { /* m-SCT awake logic, :235-254 */
      awake_for[p] = -1;
      for (int q = 0; q < n; ++q)
        if (awake_for[q] == j) awake_for[q] = -1;
      int h = fav_child[j];
      if (h >= 0 && h < V && !placed[h]) {
        awake_for[p] = h;
        awake_until[p] = st.fin[j] + c_max;
        awake++;
      }
    }
    /* readiness + urgency, :256-268 */
    for (int x = c.out_off[j]; x < c.out_off[j + 1]; ++x) {
      int child = g->edst[c.out_edge[x]];
      if (--pending[child] == 0) {
        int64_t u = 0;
        for (int y = c.in_off[child]; y < c.in_off[child + 1]; ++y) {
          int e2 = c.in_edge[y];
          u = max64(u, st.fin[g->esrc[e2]] + c_e[e2]);
        }
        urgent[child] = u;
        ready[child] = 1;
      }
    }
  }
  if (rc == RS_OK) {
    for (int j = 0; j < V; ++j) device_of[j] = st.dev_of[j];
    emit_exec_order(V, n, start, device_of, exec_order, exec_off);
    if (stats3) {
      stats3[0] = discarded;
      stats3[1] = excluded;
      stats3[2] = awake;
    }
  }
  free(st.dev_free);
  free(st.tail);
  free(st.fin);
  free(st.cache);
  free(st.dev_of);
  free(need);
  free(reserved);
  free(placed);
  free(dead);
  free(ready);
  free(alive);
  free(pending);
  free(urgent);
  free(awake_for);
  free(awake_until);
  free(scratch);
  free(c_e);
  csr_free(&c);
  return rc;
}

/* ---- simulator, proj/src/simulator.cpp:14-278 ------------------------- */
typedef struct {
  int64_t t;
  int32_t kind, a, b; /* kind: finish 0 < xfer_done 1 < start 2 (:14) */
} ev_t;

typedef struct {
  ev_t *a;
  int n, cap;
} eheap;

static int ev_less(const ev_t *x, const ev_t *y) {
  if (x->t != y->t) return x->t < y->t;
  if (x->kind != y->kind) return x->kind < y->kind;
  if (x->a != y->a) return x->a < y->a;
  return x->b < y->b;
}

static void eh_push(eheap *h, ev_t v) {
  if (h->n == h->cap) {
    h->cap = h->cap ? 2 * h->cap : 64;
    h->a = realloc(h->a, sizeof(ev_t) * (size_t)h->cap);
  }
  int i = h->n++;
  h->a[i] = v;
  while (i > 0) {
    int p = (i - 1) / 2;
    if (!ev_less(&h->a[i], &h->a[p])) break;
    ev_t t = h->a[p];
    h->a[p] = h->a[i];
    h->a[i] = t;
    i = p;
  }
}

static ev_t eh_pop(eheap *h) {
  ev_t top = h->a[0];
  h->a[0] = h->a[--h->n];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && ev_less(&h->a[l], &h->a[m])) m = l;
    if (r < h->n && ev_less(&h->a[r], &h->a[m])) m = r;
    if (m == i) break;
    ev_t t = h->a[m];
    h->a[m] = h->a[i];
    h->a[i] = t;
    i = m;
  }
  return top;
}

typedef struct {
  const rs_graph *g;
  const csr_t *c;
  int V, n, mode, mem_mode;
  double ic, pb;
  const int64_t *caps;
  const int32_t *dev_of, *order, *off;
  int64_t *mem, *peak, *xfree;
  int32_t *qpos, *consumers_left;
  char *busy, *finished, *start_q, *resident, *sent;
  int64_t *start, makespan, xcount, xbytes, dups;
  eheap h;
  char *msg;
  int msglen;
} sim_t;

static long long base_id(const sim_t *s, int meta) {
  return s->g->first_id ? (long long)s->g->first_id[meta] : (long long)meta;
}

static int charge(sim_t *s, int dev, int64_t delta, int64_t t, int meta) {
  s->mem[dev] += delta;
  if (s->mem[dev] > s->peak[dev]) s->peak[dev] = s->mem[dev];
  if (s->mem[dev] > s->caps[dev]) {
    char buf[256];
    snprintf(buf, sizeof buf,
             "memory violation on device %d at t=%lldus while holding node "
             "%lld: %lld > %lld",
             dev, (long long)t, base_id(s, meta), (long long)s->mem[dev],
             (long long)s->caps[dev]);
    return fail(s->msg, s->msglen, RS_INFEASIBLE, buf);
  }
  return RS_OK;
}

static int inputs_resident(const sim_t *s, int j) {
  int dev = s->dev_of[j];
  for (int x = s->c->in_off[j]; x < s->c->in_off[j + 1]; ++x) {
    int i = s->g->esrc[s->c->in_edge[x]];
    if (!s->finished[i]) return 0;
    if (s->dev_of[i] != dev && !s->resident[(size_t)i * s->n + dev]) return 0;
  }
  return 1;
}

static void try_start(sim_t *s, int dev, int64_t now) {
  if (s->busy[dev] || s->qpos[dev] >= s->off[dev + 1] - s->off[dev]) return;
  int j = s->order[s->off[dev] + s->qpos[dev]];
  if (s->start_q[j] || !inputs_resident(s, j)) return;
  s->start_q[j] = 1;
  ev_t ev = {now, 2, j, 0};
  eh_push(&s->h, ev);
}

int rs_simulate(const rs_graph *g, int32_t n, const int64_t *caps,
                double intercept, double per_byte, int32_t mode,
                int32_t mem_mode, const int32_t *device_of,
                const int32_t *exec_order, const int32_t *exec_off,
                int64_t *makespan, int64_t *start, int64_t *dev3n,
                int64_t *xfer4, char *msg, int msglen) {
  const int V = g->V;
  /* validate_placement, :78-97 */
  {
    int32_t *seen = calloc((size_t)(V > 0 ? V : 1), 4);
    for (int d = 0; d < n; ++d) {
      for (int x = exec_off[d]; x < exec_off[d + 1]; ++x) {
        int m = exec_order[x];
        if (m < 0 || m >= V || device_of[m] != d) {
          free(seen);
          return fail(msg, msglen, RS_VALIDATION, "exec_order disagrees with assignments");
        }
        seen[m]++;
      }
    }
    for (int j = 0; j < V; ++j) {
      if (device_of[j] < 0 || device_of[j] >= n || seen[j] != 1) {
        free(seen);
        return fail(msg, msglen, RS_VALIDATION,
                    "placement must assign every node exactly once");
      }
    }
    free(seen);
  }
  csr_t c;
  csr_build(g, &c);
  size_t Vn = (size_t)(V > 0 ? V : 1) * (size_t)n;
  sim_t s;
  memset(&s, 0, sizeof s);
  s.g = g;
  s.c = &c;
  s.V = V;
  s.n = n;
  s.mode = mode;
  s.mem_mode = mem_mode;
  s.ic = intercept;
  s.pb = per_byte;
  s.caps = caps;
  s.dev_of = device_of;
  s.order = exec_order;
  s.off = exec_off;
  s.mem = calloc((size_t)n, 8);
  s.peak = calloc((size_t)n, 8);
  s.xfree = calloc((size_t)n, 8);
  s.qpos = calloc((size_t)n, 4);
  s.busy = calloc((size_t)n, 1);
  s.consumers_left = calloc((size_t)(V > 0 ? V : 1), 4);
  s.finished = calloc((size_t)(V > 0 ? V : 1), 1);
  s.start_q = calloc((size_t)(V > 0 ? V : 1), 1);
  s.resident = calloc(Vn, 1);
  s.sent = calloc(Vn, 1);
  s.start = start;
  s.msg = msg;
  s.msglen = msglen;
  int64_t *dest_bytes = malloc(8 * (size_t)n);
  char *dest_has = malloc((size_t)n);
  for (int j = 0; j < V; ++j) start[j] = 0;
  for (int e = 0; e < g->E; ++e) s.consumers_left[g->esrc[e]]++;
  int rc = RS_OK;
  /* permanent memory up front, :209-214 */
  for (int d = 0; d < n && !rc; ++d)
    for (int x = exec_off[d]; x < exec_off[d + 1] && !rc; ++x)
      rc = charge(&s, d, g->perm[exec_order[x]], 0, exec_order[x]);
  if (!rc)
    for (int d = 0; d < n; ++d) try_start(&s, d, 0);
  int finished_count = 0;
  while (!rc && s.h.n > 0) {
    ev_t ev = eh_pop(&s.h);
    int j = ev.a;
    if (ev.kind == 2) { /* run_start, :121-131 */
      int dev = device_of[j];
      s.busy[dev] = 1;
      start[j] = ev.t;
      rc = charge(&s, dev, g->temp[j] + g->out[j], ev.t, j);
      if (rc) break;
      ev_t fe = {ev.t + g->k[j], 0, j, 0};
      eh_push(&s.h, fe);
    } else if (ev.kind == 0) { /* run_finish, :133-184 */
      int dev = device_of[j];
      s.busy[dev] = 0;
      s.qpos[dev]++;
      s.finished[j] = 1;
      finished_count++;
      s.makespan = max64(s.makespan, ev.t);
      s.mem[dev] -= g->temp[j];
      if (mem_mode == 0) { /* GraphStatic */
        if (s.consumers_left[j] == 0) s.mem[dev] -= g->out[j];
        for (int x = c.in_off[j]; x < c.in_off[j + 1]; ++x) {
          int i = g->esrc[c.in_edge[x]];
          if (--s.consumers_left[i] == 0) s.mem[device_of[i]] -= g->out[i];
        }
      }
      memset(dest_has, 0, (size_t)n);
      for (int x = c.out_off[j]; x < c.out_off[j + 1]; ++x) {
        int e = c.out_edge[x];
        int cdev = device_of[g->edst[e]];
        if (cdev == dev) continue;
        if (!dest_has[cdev] || g->ebytes[e] > dest_bytes[cdev]) dest_bytes[cdev] = g->ebytes[e];
        dest_has[cdev] = 1;
      }
      for (int cdev = 0; cdev < n; ++cdev) {
        if (!dest_has[cdev]) continue;
        size_t key = (size_t)j * n + cdev;
        if (s.resident[key] || s.sent[key]) {
          s.dups++;
          continue;
        }
        s.sent[key] = 1;
        int64_t cc = rs_comm_time(intercept, per_byte, dest_bytes[cdev], NULL);
        int64_t begin = ev.t;
        if (mode == 0) {
          begin = max64(ev.t, max64(s.xfree[dev], s.xfree[cdev]));
          s.xfree[dev] = begin + cc;
          s.xfree[cdev] = begin + cc;
        }
        s.xcount++;
        s.xbytes += dest_bytes[cdev];
        ev_t xe = {begin + cc, 1, j, cdev};
        eh_push(&s.h, xe);
      }
      try_start(&s, dev, ev.t);
    } else { /* run_xfer_done, :186-190 */
      s.resident[(size_t)ev.a * n + ev.b] = 1;
      try_start(&s, ev.b, ev.t);
    }
  }
  if (!rc && finished_count != V) { /* deadlock, :234-246 */
    char buf[256];
    int found = 0;
    for (int d = 0; d < n && !found; ++d) {
      if (s.qpos[d] < exec_off[d + 1] - exec_off[d]) {
        int j = exec_order[exec_off[d] + s.qpos[d]];
        snprintf(buf, sizeof buf,
                 "deadlock: device %d waits forever for inputs of node %lld; "
                 "exec_order contradicts the DAG",
                 d, base_id(&s, j));
        found = 1;
      }
    }
    if (!found) snprintf(buf, sizeof buf, "deadlock: simulation stalled");
    rc = fail(msg, msglen, RS_VALIDATION, buf);
  }
  if (!rc) {
    *makespan = s.makespan;
    for (int d = 0; d < n; ++d) {
      int64_t busy = 0;
      for (int x = exec_off[d]; x < exec_off[d + 1]; ++x) busy += g->k[exec_order[x]];
      dev3n[3 * d + 0] = s.peak[d];
      dev3n[3 * d + 1] = busy;
      dev3n[3 * d + 2] = s.makespan - busy;
    }
    /* cache hits, :256-266 */
    int64_t hits = 0;
    int32_t *per = calloc((size_t)n, 4);
    for (int j = 0; j < V; ++j) {
      memset(per, 0, 4 * (size_t)n);
      for (int x = c.out_off[j]; x < c.out_off[j + 1]; ++x) {
        int cdev = device_of[g->edst[c.out_edge[x]]];
        if (cdev != device_of[j]) per[cdev]++;
      }
      for (int d = 0; d < n; ++d)
        if (per[d] > 0) hits += per[d] - 1;
    }
    free(per);
    xfer4[0] = s.xcount;
    xfer4[1] = s.xbytes;
    xfer4[2] = s.dups;
    xfer4[3] = hits;
  }
  free(s.mem);
  free(s.peak);
  free(s.xfree);
  free(s.qpos);
  free(s.busy);
  free(s.consumers_left);
  free(s.finished);
  free(s.start_q);
  free(s.resident);
  free(s.sent);
  free(s.h.a);
  free(dest_bytes);
  free(dest_has);
  csr_free(&c);
  return rc;
}

/* ---- favourite-child extraction, proj/src/lp.cpp:280-326 --------------- */
static int xd_less(double xa, int ia, double xb, int ib) {
  /* std::pair<double,int> operator< */
  if (xa < xb) return 1;
  if (xb < xa) return 0;
  return ia < ib;
}

int rs_round_extract(int32_t V, int32_t E, const int32_t *esrc,
                     const int32_t *edst, const double *x, double threshold,
                     int32_t *fav_child, int32_t *fav_parent, int32_t *stats2,
                     char *msg, int msglen) {
  if (threshold <= 0 || threshold >= 0.5)
    return fail(msg, msglen, RS_VALIDATION, "rounding threshold must lie in (0, 0.5)");
  int32_t *best_of_src = malloc(4 * (size_t)(V > 0 ? V : 1));
  int32_t *cnt_src = calloc((size_t)(V > 0 ? V : 1), 4);
  for (int i = 0; i < V; ++i) best_of_src[i] = -1;
  for (int e = 0; e < E; ++e) {
    if (!(x[e] < threshold)) continue;
    int i = esrc[e];
    cnt_src[i]++;
    int b = best_of_src[i];
    if (b < 0 || xd_less(x[e], edst[e], x[b], edst[b])) best_of_src[i] = e;
  }
  int repaired = 0, fav_edges = 0;
  int32_t *best_of_dst = malloc(4 * (size_t)(V > 0 ? V : 1));
  int32_t *cnt_dst = calloc((size_t)(V > 0 ? V : 1), 4);
  for (int i = 0; i < V; ++i) best_of_dst[i] = -1;
  for (int i = 0; i < V; ++i) {
    fav_child[i] = -1;
    fav_parent[i] = -1;
  }
  /* kept edges in ascending source order, then per destination */
  for (int i = 0; i < V; ++i) {
    if (cnt_src[i] == 0) continue;
    if (cnt_src[i] > 1) repaired++;
    int e = best_of_src[i];
    int d = edst[e];
    cnt_dst[d]++;
    int b = best_of_dst[d];
    if (b < 0 || xd_less(x[e], esrc[e], x[b], esrc[b])) best_of_dst[d] = e;
  }
  for (int d = 0; d < V; ++d) {
    if (cnt_dst[d] == 0) continue;
    if (cnt_dst[d] > 1) repaired++;
    int e = best_of_dst[d];
    fav_child[esrc[e]] = d;
    fav_parent[d] = esrc[e];
    fav_edges++;
  }
  if (stats2) {
    stats2[0] = fav_edges;
    stats2[1] = repaired;
  }
  free(best_of_src);
  free(cnt_src);
  free(best_of_dst);
  free(cnt_dst);
  return RS_OK;
}

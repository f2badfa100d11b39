/*
 * CPU oracle (TEST INFRASTRUCTURE ONLY): C restatement of the reference session
 * radix tree, /root/reference/pkg/src/rolloutlab/trie.py, for many sessions.
 *
 * Used by tests/ (as the checker at sizes the Python oracle cannot reach) and by
 * bench.py (the timed CPU reference: `cpu_baseline` / `--impl reference`, kind
 * "port").  Never linked into the product.
 *
 * Restated functions (trie.py line numbers):
 *   ro_insert_batch  -> SessionTrie.lpm_insert   :120-179  (walk :136-158, split
 *                       :106-118 + _split_runs :36-49, suffix node :141-149/:164-168,
 *                       counters :145-146/:168-176)
 *   ro_match_batch   -> the LPM walk of lpm_insert without mutation (read-only)
 *   ro_stats         -> SessionTrie.stats        :184-185
 *   ro_export_row    -> path_trajectory          :203-208 (+ _merge_runs :258-265)
 *   ro_lex_rows      -> _walk/extract order      :189-198, :210-216
 * Row / parent numbering as oracle/radix.py.
 *
 * Sessions are independent, so batches are processed by a pool of
 * pthreads, each owning a disjoint set of sessions; per-session order is batch
 * order.  The per-token compare is the reference's scalar loop (trie.py:153).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { int32_t len; int32_t version; uint8_t origin; } Run;

typedef struct Node Node;
struct Node {
  int32_t *tok;      /* span tokens (may alias a parent's buffer after a split) */
  int32_t len;
  Run *runs;
  int32_t nruns, capruns;
  int32_t creator;   /* row that first wrote these tokens */
  int32_t row;       /* row ordinal ending here, -1 if none */
  Node *up;
  Node **kids;       /* sorted by first token */
  int32_t nkids, capkids;
};

typedef struct {
  Node root;
  Node **rows;
  int64_t *row_len;
  int32_t nrows, caprows;
  int64_t stored, naive;
  void **blocks;
  int32_t nblocks, capblocks;
} Session;

typedef struct {
  Session **sess;
  int64_t nsess, capsess;
} Store;

static void *xrealloc(void *p, size_t n) {
  void *q = realloc(p, n ? n : 1);
  if (!q) abort();
  return q;
}

static void own(Session *s, void *p) {
  if (s->nblocks == s->capblocks) {
    s->capblocks = s->capblocks ? 2 * s->capblocks : 16;
    s->blocks = xrealloc(s->blocks, sizeof(void *) * s->capblocks);
  }
  s->blocks[s->nblocks++] = p;
}

static Node *new_node(Session *s) {
  Node *n = calloc(1, sizeof(Node));
  if (!n) abort();
  own(s, n);
  n->row = -1;
  return n;
}

static void push_run(Node *n, int32_t len, uint8_t o, int32_t v) {
  if (n->nruns && n->runs[n->nruns - 1].origin == o && n->runs[n->nruns - 1].version == v) {
    n->runs[n->nruns - 1].len += len;
    return;
  }
  if (n->nruns == n->capruns) {
    n->capruns = n->capruns ? 2 * n->capruns : 4;
    n->runs = xrealloc(n->runs, sizeof(Run) * n->capruns);
  }
  n->runs[n->nruns].len = len;
  n->runs[n->nruns].origin = o;
  n->runs[n->nruns].version = v;
  n->nruns++;
}

static int32_t kid_find(Node *n, int32_t t, int *pos) {
  int lo = 0, hi = n->nkids;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (n->kids[mid]->tok[0] < t) lo = mid + 1; else hi = mid;
  }
  *pos = lo;
  return (lo < n->nkids && n->kids[lo]->tok[0] == t) ? lo : -1;
}

static void kid_insert(Node *n, Node *c, int pos) {
  if (n->nkids == n->capkids) {
    n->capkids = n->capkids ? 2 * n->capkids : 2;
    n->kids = xrealloc(n->kids, sizeof(Node *) * n->capkids);
  }
  memmove(n->kids + pos + 1, n->kids + pos, sizeof(Node *) * (n->nkids - pos));
  n->kids[pos] = c;
  n->nkids++;
  c->up = n;
}

static int32_t new_row(Session *s, Node *end, int64_t L) {
  if (s->nrows == s->caprows) {
    s->caprows = s->caprows ? 2 * s->caprows : 8;
    s->rows = xrealloc(s->rows, sizeof(Node *) * s->caprows);
    s->row_len = xrealloc(s->row_len, sizeof(int64_t) * s->caprows);
  }
  end->row = s->nrows;
  s->rows[s->nrows] = end;
  s->row_len[s->nrows] = L;
  return s->nrows++;
}

/* suffix node for tokens[i:L) with the per-run metadata of the request */
static Node *suffix_node(Session *s, const int32_t *tok, int64_t i, int64_t L, const int32_t *rs,
                         const uint8_t *ro, const int32_t *rv, int64_t nr) {
  Node *n = new_node(s);
  n->tok = malloc(sizeof(int32_t) * (L - i));
  if (!n->tok) abort();
  own(s, n->tok);
  memcpy(n->tok, tok + i, sizeof(int32_t) * (L - i));
  n->len = (int32_t)(L - i);
  n->creator = s->nrows;
  for (int64_t k = 0; k < nr; k++) {
    int64_t a = rs[k], b = (k + 1 < nr) ? rs[k + 1] : L;
    if (b <= i) continue;
    if (a < i) a = i;
    push_run(n, (int32_t)(b - a), ro[k], rv[k]);
  }
  return n;
}

/* lpm_insert (trie.py:120-179) */
static void insert_one(Session *s, const int32_t *tok, int64_t L, const int32_t *rs, const uint8_t *ro,
                       const int32_t *rv, int64_t nr, int32_t *om, int32_t *orow, int32_t *opar,
                       int32_t *oadd) {
  Node *node = &s->root;
  int64_t i = 0;
  int32_t parent = -1;
  Node *end = NULL;
  for (;;) {
    if (i == L) { end = node; parent = node->creator; break; }
    int pos;
    int32_t k = kid_find(node, tok[i], &pos);
    if (k < 0) {
      parent = (i > 0) ? node->creator : -1;
      Node *n = suffix_node(s, tok, i, L, rs, ro, rv, nr);
      kid_insert(node, n, pos);
      s->stored += L - i;
      s->naive += L;
      *om = (int32_t)i; *opar = parent; *oadd = (int32_t)(L - i);
      *orow = new_row(s, n, L);
      return;
    }
    Node *ch = node->kids[k];
    int64_t lim = ch->len < L - i ? ch->len : L - i;
    int64_t c = 0;
    while (c < lim && ch->tok[c] == tok[i + c]) c++;
    if (c == ch->len) { node = ch; i += c; continue; }
    /* split (trie.py:106-118): head keeps ch's first c tokens, ch keeps its id */
    parent = ch->creator;
    Node *head = new_node(s);
    head->tok = ch->tok;
    head->len = (int32_t)c;
    head->creator = ch->creator;
    int32_t seen = 0, r = 0;
    Run *old = ch->runs;
    int32_t nold = ch->nruns;
    ch->runs = NULL; ch->nruns = 0; ch->capruns = 0;
    for (r = 0; r < nold; r++) {
      int32_t ln = old[r].len;
      if (seen + ln <= c) push_run(head, ln, old[r].origin, old[r].version);
      else if (seen >= c) push_run(ch, ln, old[r].origin, old[r].version);
      else {
        push_run(head, (int32_t)(c - seen), old[r].origin, old[r].version);
        push_run(ch, (int32_t)(ln - (c - seen)), old[r].origin, old[r].version);
      }
      seen += ln;
    }
    free(old);
    ch->tok += c;
    ch->len -= (int32_t)c;
    node->kids[k] = head;
    head->up = node;
    int dummy;
    kid_find(head, ch->tok[0], &dummy);
    kid_insert(head, ch, dummy);
    i += c;
    if (i == L) { end = head; break; }
    Node *n = suffix_node(s, tok, i, L, rs, ro, rv, nr);
    kid_find(head, tok[i], &pos);
    kid_insert(head, n, pos);
    s->stored += L - i;
    s->naive += L;
    *om = (int32_t)i; *opar = parent; *oadd = (int32_t)(L - i);
    *orow = new_row(s, n, L);
    return;
  }
  s->naive += L;
  *om = (int32_t)L; *opar = parent; *oadd = 0;
  *orow = (end->row >= 0) ? end->row : new_row(s, end, L);
}

/* read-only walk: matched length, parent row, duplicate row (or -1) */
static void match_one(const Session *s, const int32_t *tok, int64_t L, int64_t *om, int32_t *opar,
                      int32_t *odup) {
  const Node *node = &s->root;
  int64_t i = 0;
  *odup = -1;
  for (;;) {
    if (i == L) { *om = L; *opar = node->creator; *odup = node->row; return; }
    int pos;
    int32_t k = kid_find((Node *)node, tok[i], &pos);
    if (k < 0) { *om = i; *opar = i > 0 ? node->creator : -1; return; }
    const Node *ch = node->kids[k];
    int64_t lim = ch->len < L - i ? ch->len : L - i;
    int64_t c = 0;
    while (c < lim && ch->tok[c] == tok[i + c]) c++;
    if (c == ch->len) { node = ch; i += c; continue; }
    *om = i + c;
    *opar = ch->creator;
    return;
  }
}

void *ro_create(void) { return calloc(1, sizeof(Store)); }

static void free_tree(Node *n) {
  for (int32_t k = 0; k < n->nkids; k++) free_tree(n->kids[k]);
  free(n->kids);
  free(n->runs);
}

void ro_destroy(void *h) {
  Store *st = h;
  if (!st) return;
  for (int64_t i = 0; i < st->nsess; i++) {
    Session *s = st->sess[i];
    if (!s) continue;
    free_tree(&s->root);
    for (int32_t b = 0; b < s->nblocks; b++) free(s->blocks[b]);
    free(s->blocks);
    free(s->rows);
    free(s->row_len);
    free(s);
  }
  free(st->sess);
  free(st);
}

static Session *get_session(Store *st, int64_t sid) {
  if (sid >= st->capsess) {
    int64_t cap = st->capsess ? st->capsess : 64;
    while (cap <= sid) cap *= 2;
    st->sess = xrealloc(st->sess, sizeof(Session *) * cap);
    memset(st->sess + st->capsess, 0, sizeof(Session *) * (cap - st->capsess));
    st->capsess = cap;
  }
  if (sid >= st->nsess) st->nsess = sid + 1;
  if (!st->sess[sid]) {
    Session *s = calloc(1, sizeof(Session));
    if (!s) abort();
    s->root.row = -1;
    s->root.creator = -1;
    st->sess[sid] = s;
  }
  return st->sess[sid];
}

typedef struct {
  Store *st;
  int64_t n;
  const int32_t *sids, *tok;
  const int64_t *tok_off, *run_off;
  const int32_t *run_start, *run_version;
  const uint8_t *run_origin;
  int32_t *om32, *orow, *opar, *oadd, *odup;
  int64_t *om64;
  int tid, nthreads, mode;
} Job;

static void *worker(void *arg) {
  Job *j = arg;
  for (int64_t e = 0; e < j->n; e++) {
    int64_t sid = j->sids[e];
    if (sid % j->nthreads != j->tid) continue;
    const int32_t *t = j->tok + j->tok_off[e];
    int64_t L = j->tok_off[e + 1] - j->tok_off[e];
    if (j->mode == 0) {
      int64_t r0 = j->run_off[e], r1 = j->run_off[e + 1];
      insert_one(j->st->sess[sid], t, L, j->run_start + r0, j->run_origin + r0, j->run_version + r0,
                 r1 - r0, j->om32 + e, j->orow + e, j->opar + e, j->oadd + e);
    } else {
      Session *s = (sid < j->st->nsess) ? j->st->sess[sid] : NULL;
      if (!s || L == 0) { j->om64[e] = 0; j->opar[e] = -1; j->odup[e] = -1; continue; }
      match_one(s, t, L, j->om64 + e, j->opar + e, j->odup + e);
    }
  }
  return NULL;
}

static void run_jobs(Job *proto, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  pthread_t th[256];
  Job jobs[256];
  if (nthreads > 256) nthreads = 256;
  for (int t = 0; t < nthreads; t++) {
    jobs[t] = *proto;
    jobs[t].tid = t;
    jobs[t].nthreads = nthreads;
  }
  if (nthreads == 1) { worker(&jobs[0]); return; }
  for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, worker, &jobs[t]);
  for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
}

/* Record a batch; run starts are relative to each sequence; origins 0/1. */
int ro_insert_batch(void *h, int64_t n, const int32_t *sids, const int32_t *tok, const int64_t *tok_off,
                    const int64_t *run_off, const int32_t *run_start, const uint8_t *run_origin,
                    const int32_t *run_version, int32_t *out_matched, int32_t *out_row,
                    int32_t *out_parent, int32_t *out_added, int nthreads) {
  Store *st = h;
  for (int64_t e = 0; e < n; e++) {
    if (tok_off[e + 1] - tok_off[e] <= 0) return 1; /* ValueError: empty sequence */
    get_session(st, sids[e]);
  }
  Job j = {0};
  j.st = st; j.n = n; j.sids = sids; j.tok = tok; j.tok_off = tok_off; j.run_off = run_off;
  j.run_start = run_start; j.run_origin = run_origin; j.run_version = run_version;
  j.om32 = out_matched; j.orow = out_row; j.opar = out_parent; j.oadd = out_added; j.mode = 0;
  run_jobs(&j, nthreads);
  return 0;
}

int ro_match_batch(void *h, int64_t n, const int32_t *sids, const int32_t *tok, const int64_t *tok_off,
                   int64_t *out_matched, int32_t *out_parent, int32_t *out_dup, int nthreads) {
  Job j = {0};
  j.st = h; j.n = n; j.sids = sids; j.tok = tok; j.tok_off = tok_off;
  j.om64 = out_matched; j.opar = out_parent; j.odup = out_dup; j.mode = 1;
  run_jobs(&j, nthreads);
  return 0;
}

int ro_stats(void *h, int64_t sid, int64_t *stored, int64_t *naive, int32_t *nrows) {
  Store *st = h;
  if (sid >= st->nsess || !st->sess[sid]) return 2;
  *stored = st->sess[sid]->stored;
  *naive = st->sess[sid]->naive;
  *nrows = st->sess[sid]->nrows;
  return 0;
}

int64_t ro_row_len(void *h, int64_t sid, int32_t row) {
  Store *st = h;
  if (sid >= st->nsess || !st->sess[sid] || row < 0 || row >= st->sess[sid]->nrows) return -1;
  return st->sess[sid]->row_len[row];
}

/* path_trajectory (trie.py:203-208): tokens, mask (origin==OUTPUT), versions */
int ro_export_row(void *h, int64_t sid, int32_t row, int32_t *tokens, uint8_t *mask, int32_t *versions) {
  Store *st = h;
  if (sid >= st->nsess || !st->sess[sid] || row < 0 || row >= st->sess[sid]->nrows) return 2;
  Session *s = st->sess[sid];
  const Node *path[4096];
  const Node **pp = path;
  int32_t depth = 0, cap = 4096;
  for (const Node *n = s->rows[row]; n && n != &s->root; n = n->up) {
    if (depth == cap) {
      const Node **np = malloc(sizeof(Node *) * cap * 2);
      memcpy(np, pp, sizeof(Node *) * cap);
      if (pp != path) free(pp);
      pp = np;
      cap *= 2;
    }
    pp[depth++] = n;
  }
  int64_t pos = 0;
  for (int32_t d = depth - 1; d >= 0; d--) {
    const Node *n = pp[d];
    memcpy(tokens + pos, n->tok, sizeof(int32_t) * n->len);
    int64_t q = pos;
    for (int32_t r = 0; r < n->nruns; r++) {
      for (int32_t k = 0; k < n->runs[r].len; k++, q++) {
        mask[q] = n->runs[r].origin;
        versions[q] = n->runs[r].version;
      }
    }
    pos += n->len;
  }
  if (pp != path) free(pp);
  return 0;
}

static void lex(const Node *n, int32_t *out, int32_t *k) {
  if (n->row >= 0) out[(*k)++] = n->row;
  for (int32_t c = 0; c < n->nkids; c++) lex(n->kids[c], out, k);
}

/* all rows of a session in lexicographic sequence order (trie.py:189-198) */
int ro_lex_rows(void *h, int64_t sid, int32_t *out_rows, int32_t *n_out) {
  Store *st = h;
  if (sid >= st->nsess || !st->sess[sid]) return 2;
  *n_out = 0;
  lex(&st->sess[sid]->root, out_rows, n_out);
  return 0;
}

/* Many path_trajectory calls at once (test speed only): row k of session sids[k] is
 * written at [out_off[k], out_off[k+1]); rows are split over nthreads threads. */
typedef struct {
  Store *st;
  int64_t n;
  const int64_t *sids;
  const int32_t *rows;
  const int64_t *off;
  int32_t *tok, *ver;
  uint8_t *mask;
  int tid, nthreads, rc;
} ExportJob;

static void *export_worker(void *arg) {
  ExportJob *j = arg;
  for (int64_t k = j->tid; k < j->n; k += j->nthreads)
    if (ro_export_row(j->st, j->sids[k], j->rows[k], j->tok + j->off[k], j->mask + j->off[k], j->ver + j->off[k]))
      j->rc = 2;
  return NULL;
}

int ro_export_batch(void *h, int64_t n, const int64_t *sids, const int32_t *rows, const int64_t *out_off,
                    int32_t *tokens, uint8_t *mask, int32_t *versions, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  ExportJob jobs[256];
  for (int t = 0; t < nthreads; t++) {
    ExportJob j = {h, n, sids, rows, out_off, tokens, versions, mask, t, nthreads, 0};
    jobs[t] = j;
  }
  for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, export_worker, &jobs[t]);
  int rc = 0;
  for (int t = 0; t < nthreads; t++) {
    pthread_join(th[t], NULL);
    if (jobs[t].rc) rc = jobs[t].rc;
  }
  return rc;
}

/*
 * oracle.c -- CPU ORACLE (TEST INFRASTRUCTURE ONLY; see oracle.h).
 *
 * Plain, slow, obviously correct.  Each function cites the passage it follows.
 * Shares no code with paper_1702_03657_b200/ (the CUDA product path).
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------------ */
/* Trie.  PAPER.md:80 steps I (breadth-first, level by level) and II   */
/* (row-major ordered array); node = 256-bit bitmap + first-child      */
/* offset (Fig. 3; 36 bytes).               */
/* ------------------------------------------------------------------ */
typedef struct { uint32_t bitmap[8]; uint32_t offset; } or_node36;

/* Insertion trie (build-time only): first-child / next-sibling lists,
 * siblings kept in ascending label order. */
typedef struct { uint32_t first, next; uint8_t label; } lnode;

struct or_trie {
    uint32_t n_nodes, n_patterns, max_len, min_len, n_terminals;
    or_node36 *nodes;      /* BFS row-major, nodes[0] = root */
    uint32_t *term_start;  /* [N+1] into term_pids */
    uint32_t *term_pids;   /* ascending per node */
    uint32_t *pat_len;     /* |P_k| */
    uint8_t *pat_data; uint64_t *pat_off;
    /* own label CSR (PAPER.md:89 CRS step; label form) */
    uint32_t *csr_row_ptr; uint8_t *csr_label; uint32_t *csr_child;
    /* Aho-Corasick DFA, built on first use */
    pthread_mutex_t ac_lock;
    int ac_built;
    uint32_t ac_k;         /* number of byte classes */
    uint16_t ac_cls[256];  /* byte -> class */
    uint32_t *ac_delta;    /* [N * K] */
    uint32_t *ac_dict;     /* dictionary-suffix link, UINT32_MAX = none */
};

#define NONE 0xFFFFFFFFu

static int popc(uint32_t x) { return __builtin_popcount(x); }

static int bit_is_set(const or_node36 *n, uint32_t c) { return (n->bitmap[c >> 5] >> (c & 31)) & 1u; }

/* Child-location rule: child(c) = offset + number of set bits below c
 * (SPEC S:99-107 reading of the method P:97 defers to [bellekens2016high]). */
static int64_t child_rank(const or_node36 *n, uint32_t c) {
    if (!bit_is_set(n, c)) return -1;
    uint32_t r = 0;
    for (uint32_t w = 0; w < (c >> 5); w++) r += (uint32_t)popc(n->bitmap[w]);
    r += (uint32_t)popc(n->bitmap[c >> 5] & ((1u << (c & 31)) - 1u));
    return (int64_t)n->offset + r;
}

int or_build(const uint8_t *data, const uint32_t *lens, uint32_t n, or_trie **out) {
    if (!out || !lens || n == 0) return OR_EINVAL;
    *out = NULL;
    uint64_t total = 0;
    for (uint32_t k = 0; k < n; k++) {
        if (lens[k] == 0) return OR_EINVAL;
        total += lens[k];
    }
    if (!data) return OR_EINVAL;
    or_trie *t = (or_trie *)calloc(1, sizeof *t);
    if (!t) return OR_ENOMEM;
    pthread_mutex_init(&t->ac_lock, NULL);
    t->n_patterns = n;
    t->pat_len = (uint32_t *)malloc(sizeof(uint32_t) * n);
    t->pat_off = (uint64_t *)malloc(sizeof(uint64_t) * n);
    t->pat_data = (uint8_t *)malloc(total);
    /* one insertion node per byte at most, plus the root */
    uint64_t cap = total + 1;
    lnode *L = (lnode *)malloc(sizeof(lnode) * cap);
    uint32_t *lterm_head = (uint32_t *)malloc(sizeof(uint32_t) * cap); /* pid list heads */
    uint32_t *pid_next = (uint32_t *)malloc(sizeof(uint32_t) * n);
    uint32_t *pid_tail = (uint32_t *)malloc(sizeof(uint32_t) * cap);
    if (!t->pat_len || !t->pat_off || !t->pat_data || !L || !lterm_head || !pid_next || !pid_tail) {
        free(L); free(lterm_head); free(pid_next); free(pid_tail); or_free(t);
        return OR_ENOMEM;
    }
    memcpy(t->pat_data, data, total);
    t->max_len = 0; t->min_len = NONE;
    uint64_t off = 0;
    uint32_t nl = 1;
    L[0].first = NONE; L[0].next = NONE; L[0].label = 0;
    lterm_head[0] = NONE;
    for (uint32_t k = 0; k < n; k++) {
        const uint8_t *p = data + off;
        t->pat_off[k] = off;
        t->pat_len[k] = lens[k];
        off += lens[k];
        if (lens[k] > t->max_len) t->max_len = lens[k];
        if (lens[k] < t->min_len) t->min_len = lens[k];
        uint32_t v = 0;
        for (uint32_t j = 0; j < lens[k]; j++) {
            uint8_t c = p[j];
            uint32_t prev = NONE, u = L[v].first;
            while (u != NONE && L[u].label < c) { prev = u; u = L[u].next; }
            if (u == NONE || L[u].label != c) {
                uint32_t w = nl++;
                L[w].first = NONE; L[w].label = c; L[w].next = u;
                lterm_head[w] = NONE;
                if (prev == NONE) L[v].first = w; else L[prev].next = w;
                u = w;
            }
            v = u;
        }
        /* append pid k to v's terminal list (k ascending => list ascending) */
        pid_next[k] = NONE;
        if (lterm_head[v] == NONE) lterm_head[v] = k; else pid_next[pid_tail[v]] = k;
        pid_tail[v] = k;
    }
    /* Step I/II: breadth-first numbering, children in ascending byte order. */
    uint32_t N = nl;
    uint32_t *queue = (uint32_t *)malloc(sizeof(uint32_t) * N); /* queue[bfs id] = lnode */
    t->nodes = (or_node36 *)calloc(N, sizeof(or_node36));
    t->term_start = (uint32_t *)calloc((size_t)N + 1, sizeof(uint32_t));
    t->term_pids = (uint32_t *)malloc(sizeof(uint32_t) * n);
    if (!queue || !t->nodes || !t->term_start || !t->term_pids) {
        free(queue); free(L); free(lterm_head); free(pid_next); free(pid_tail); or_free(t);
        return OR_ENOMEM;
    }
    uint32_t qt = 0;
    queue[qt++] = 0;
    uint32_t np = 0;
    for (uint32_t id = 0; id < N; id++) {
        uint32_t v = queue[id];
        or_node36 *nd = &t->nodes[id];
        nd->offset = 0;
        for (uint32_t u = L[v].first; u != NONE; u = L[u].next) {
            if (nd->offset == 0) nd->offset = qt;
            nd->bitmap[L[u].label >> 5] |= 1u << (L[u].label & 31);
            queue[qt++] = u;
        }
        t->term_start[id] = np;
        for (uint32_t k = lterm_head[v]; k != NONE; k = pid_next[k]) t->term_pids[np++] = k;
        if (lterm_head[v] != NONE) t->n_terminals++;
    }
    t->term_start[N] = np;
    t->n_nodes = N;
    free(queue); free(L); free(lterm_head); free(pid_next); free(pid_tail);

    /* Own label CSR of the same trie (row_ptr / label / explicit child). */
    uint64_t E = N ? (uint64_t)N - 1 : 0;
    t->csr_row_ptr = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)N + 1));
    t->csr_label = (uint8_t *)malloc(E ? E : 1);
    t->csr_child = (uint32_t *)malloc(sizeof(uint32_t) * (E ? E : 1));
    if (!t->csr_row_ptr || !t->csr_label || !t->csr_child) { or_free(t); return OR_ENOMEM; }
    uint32_t e = 0;
    for (uint32_t v = 0; v < N; v++) {
        t->csr_row_ptr[v] = e;
        for (uint32_t c = 0; c < 256; c++) {
            int64_t ch = child_rank(&t->nodes[v], c);
            if (ch >= 0) { t->csr_label[e] = (uint8_t)c; t->csr_child[e] = (uint32_t)ch; e++; }
        }
    }
    t->csr_row_ptr[N] = e;
    *out = t;
    return OR_OK;
}

void or_free(or_trie *t) {
    if (!t) return;
    free(t->nodes); free(t->term_start); free(t->term_pids); free(t->pat_len);
    free(t->pat_data); free(t->pat_off);
    free(t->csr_row_ptr); free(t->csr_label); free(t->csr_child);
    free(t->ac_delta); free(t->ac_dict);
    pthread_mutex_destroy(&t->ac_lock);
    free(t);
}

void or_stats(const or_trie *t, uint64_t out[6]) {
    out[0] = t->n_nodes;
    out[1] = (uint64_t)t->n_nodes - 1;
    out[2] = t->n_terminals;
    out[3] = t->n_patterns;
    out[4] = t->max_len;
    out[5] = t->min_len;
}

int or_node(const or_trie *t, uint32_t v, uint32_t bitmap[8], uint32_t *offset) {
    if (v >= t->n_nodes) return OR_EINVAL;
    memcpy(bitmap, t->nodes[v].bitmap, 32);
    *offset = t->nodes[v].offset;
    return OR_OK;
}

int or_node_pids(const or_trie *t, uint32_t v, const uint32_t **pids, uint32_t *n) {
    if (v >= t->n_nodes) return OR_EINVAL;
    *pids = t->term_pids + t->term_start[v];
    *n = t->term_start[v + 1] - t->term_start[v];
    return OR_OK;
}

int64_t or_child(const or_trie *t, uint32_t v, uint32_t c) {
    if (v >= t->n_nodes || c > 255) return -1;
    return child_rank(&t->nodes[v], c);
}

/* ------------------------------------------------------------------ */
/* Byte accounting.  P:134 (36 B/node), P:101 (CRS cost 2nnz+n+1).      */
/* Matrix view: N rows x 9 columns of 32-bit words (8 bitmap words +    */
/* offset); a leaf's offset is 0 and thus not stored.   */
/* ------------------------------------------------------------------ */
int or_paper_crs(const or_trie *t, uint32_t **val, uint32_t **col_ind, uint32_t **row_ptr,
                 uint64_t *nnz, uint64_t *n_rows) {
    uint64_t z = 0;
    for (uint32_t v = 0; v < t->n_nodes; v++) {
        for (int w = 0; w < 8; w++) z += t->nodes[v].bitmap[w] != 0;
        z += t->nodes[v].offset != 0;
    }
    uint32_t *V = (uint32_t *)malloc(sizeof(uint32_t) * (z ? z : 1));
    uint32_t *C = (uint32_t *)malloc(sizeof(uint32_t) * (z ? z : 1));
    uint32_t *R = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)t->n_nodes + 1));
    if (!V || !C || !R) { free(V); free(C); free(R); return OR_ENOMEM; }
    uint64_t k = 0;
    for (uint32_t v = 0; v < t->n_nodes; v++) {
        R[v] = (uint32_t)k;
        for (int w = 0; w < 9; w++) {
            uint32_t x = w < 8 ? t->nodes[v].bitmap[w] : t->nodes[v].offset;
            if (x) { V[k] = x; C[k] = (uint32_t)w; k++; }
        }
    }
    R[t->n_nodes] = (uint32_t)k;
    *val = V; *col_ind = C; *row_ptr = R; *nnz = z; *n_rows = t->n_nodes;
    return OR_OK;
}

uint64_t or_bytes(const or_trie *t, int kind) {
    if (kind == 0) return 36ull * t->n_nodes;
    if (kind == 1) return 1024ull * t->n_nodes;
    if (kind == 2) {
        uint64_t z = 0;
        for (uint32_t v = 0; v < t->n_nodes; v++) {
            for (int w = 0; w < 8; w++) z += t->nodes[v].bitmap[w] != 0;
            z += t->nodes[v].offset != 0;
        }
        return 4ull * (2 * z + t->n_nodes + 1);
    }
    return 0;
}

int or_csr(const or_trie *t, const uint32_t **row_ptr, const uint8_t **label, const uint32_t **child) {
    *row_ptr = t->csr_row_ptr; *label = t->csr_label; *child = t->csr_child;
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Result buffers                                                      */
/* ------------------------------------------------------------------ */
typedef struct { uint64_t n, cap; uint64_t *pos; uint32_t *pid; int err; } rowbuf;

static void rb_push(rowbuf *b, uint64_t pos, uint32_t pid) {
    if (b->err) return;
    if (b->n == b->cap) {
        uint64_t nc = b->cap ? b->cap * 2 : 1024;
        uint64_t *np = (uint64_t *)realloc(b->pos, nc * sizeof(uint64_t));
        if (!np) { b->err = 1; return; }
        b->pos = np;
        uint32_t *nq = (uint32_t *)realloc(b->pid, nc * sizeof(uint32_t));
        if (!nq) { b->err = 1; return; }
        b->pid = nq;
        b->cap = nc;
    }
    b->pos[b->n] = pos; b->pid[b->n] = pid; b->n++;
}

static void sort_u32(uint32_t *a, uint64_t n) { /* insertion sort: lists are short */
    for (uint64_t i = 1; i < n; i++) {
        uint32_t x = a[i];
        uint64_t j = i;
        while (j > 0 && a[j - 1] > x) { a[j] = a[j - 1]; j--; }
        a[j] = x;
    }
}

/* ------------------------------------------------------------------ */
/* Engine OR_PFAC_BITMAP: PAPER.md:76 -- one walk per text position,   */
/* "if a match is recorded, the thread continues the matching process  */
/* until a mismatch. When a mismatch occurs the thread is terminated". */
/* Every terminal on the path is reported.           */
/* ------------------------------------------------------------------ */
static void walk_bitmap(const or_trie *t, const uint8_t *T, uint64_t L, uint64_t lo, uint64_t hi, rowbuf *b) {
    uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * t->n_patterns);
    if (!tmp) { b->err = 1; return; }
    for (uint64_t i = lo; i < hi; i++) {
        uint64_t m = 0;
        uint32_t v = 0;
        for (uint64_t j = i; j < L; j++) {
            int64_t ch = child_rank(&t->nodes[v], T[j]);
            if (ch < 0) break;                      /* mismatch: thread terminates */
            v = (uint32_t)ch;
            for (uint32_t q = t->term_start[v]; q < t->term_start[v + 1]; q++) tmp[m++] = t->term_pids[q];
        }
        sort_u32(tmp, m);                           /* pids arrive in depth order */
        for (uint64_t q = 0; q < m; q++) rb_push(b, i, tmp[q]);
    }
    free(tmp);
}

/* Engine OR_PFAC_CSR: same walk over the label CSR (child by label scan). */
static void walk_csr(const or_trie *t, const uint8_t *T, uint64_t L, uint64_t lo, uint64_t hi, rowbuf *b) {
    uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * t->n_patterns);
    if (!tmp) { b->err = 1; return; }
    for (uint64_t i = lo; i < hi; i++) {
        uint64_t m = 0;
        uint32_t v = 0;
        for (uint64_t j = i; j < L; j++) {
            uint32_t nxt = NONE;
            for (uint32_t e = t->csr_row_ptr[v]; e < t->csr_row_ptr[v + 1]; e++)
                if (t->csr_label[e] == T[j]) { nxt = t->csr_child[e]; break; }
            if (nxt == NONE) break;
            v = nxt;
            for (uint32_t q = t->term_start[v]; q < t->term_start[v + 1]; q++) tmp[m++] = t->term_pids[q];
        }
        sort_u32(tmp, m);
        for (uint64_t q = 0; q < m; q++) rb_push(b, i, tmp[q]);
    }
    free(tmp);
}

/* Engine OR_BRUTE: the plain definition, memcmp of every P_k at every i. */
static void brute(const or_trie *t, const uint8_t *T, uint64_t L, uint64_t lo, uint64_t hi, rowbuf *b) {
    for (uint64_t i = lo; i < hi; i++)
        for (uint32_t k = 0; k < t->n_patterns; k++)
            if (i + t->pat_len[k] <= L && memcmp(T + i, t->pat_data + t->pat_off[k], t->pat_len[k]) == 0)
                rb_push(b, i, k);
}

/* ------------------------------------------------------------------ */
/* Engine OR_AC: Aho-Corasick (Aho & Corasick 1975).       */
/* Full DFA over byte classes, failure links computed in BFS order,    */
/* outputs via dictionary-suffix links.                                */
/* ------------------------------------------------------------------ */
static int ac_build(or_trie *t) {
    int present[256] = {0}, n_present = 0;
    for (uint32_t k = 0; k < t->n_patterns; k++)
        for (uint32_t j = 0; j < t->pat_len[k]; j++) present[t->pat_data[t->pat_off[k] + j]] = 1;
    for (int c = 0; c < 256; c++) n_present += present[c];
    /* classes: 0 = "byte in no pattern" (if any such byte), then the present
     * bytes in ascending order; rep[k] = a byte of class k (NONE = absent) */
    uint32_t rep[257], K = 0;
    if (n_present < 256) rep[K++] = NONE;
    for (int c = 0; c < 256; c++) {
        if (present[c]) { t->ac_cls[c] = (uint16_t)K; rep[K++] = (uint32_t)c; }
        else t->ac_cls[c] = 0;
    }
    uint32_t N = t->n_nodes;
    if ((uint64_t)N * K * 4 > (2ull << 30)) return OR_ETOOBIG;
    uint32_t *delta = (uint32_t *)malloc((size_t)N * K * sizeof(uint32_t));
    uint32_t *fail = (uint32_t *)malloc((size_t)N * sizeof(uint32_t));
    uint32_t *dict = (uint32_t *)malloc((size_t)N * sizeof(uint32_t));
    if (!delta || !fail || !dict) { free(delta); free(fail); free(dict); return OR_ENOMEM; }
    fail[0] = 0;
    dict[0] = NONE;
    for (uint32_t s = 0; s < N; s++) {          /* BFS order: ids ascending */
        for (uint32_t k = 0; k < K; k++) {
            uint32_t c = rep[k];
            int64_t u = (c == NONE) ? -1 : child_rank(&t->nodes[s], c);
            if (u >= 0) {
                delta[(size_t)s * K + k] = (uint32_t)u;
                fail[u] = (s == 0) ? 0 : delta[(size_t)fail[s] * K + k];
            } else {
                delta[(size_t)s * K + k] = (s == 0) ? 0 : delta[(size_t)fail[s] * K + k];
            }
        }
        if (s != 0) {
            uint32_t f = fail[s];
            dict[s] = (t->term_start[f + 1] > t->term_start[f]) ? f : dict[f];
        }
    }
    free(fail);
    t->ac_k = K;
    t->ac_delta = delta;
    t->ac_dict = dict;
    t->ac_built = 1;
    return OR_OK;
}

typedef struct { uint64_t pos; uint32_t pid; } row;
static int row_cmp(const void *a, const void *b) {
    const row *x = (const row *)a, *y = (const row *)b;
    if (x->pos != y->pos) return x->pos < y->pos ? -1 : 1;
    return x->pid < y->pid ? -1 : (x->pid > y->pid);
}

/* Chunk [lo, hi) of start positions: feed bytes from lo up to
 * min(L, hi + Lmax - 1) (the P:66 overlap), keep matches by START. */
static void ac_scan(const or_trie *t, const uint8_t *T, uint64_t L, uint64_t lo, uint64_t hi, rowbuf *b) {
    uint64_t end = hi + t->max_len - 1;
    if (end > L) end = L;
    rowbuf tmp = {0};
    uint32_t s = 0, K = t->ac_k;
    for (uint64_t j = lo; j < end; j++) {
        s = t->ac_delta[(size_t)s * K + t->ac_cls[T[j]]];
        uint32_t u = (t->term_start[s + 1] > t->term_start[s]) ? s : t->ac_dict[s];
        for (; u != NONE; u = t->ac_dict[u]) {
            for (uint32_t q = t->term_start[u]; q < t->term_start[u + 1]; q++) {
                uint32_t p = t->term_pids[q];
                uint64_t st = j + 1 - t->pat_len[p];
                if (st >= lo && st < hi) rb_push(&tmp, st, p);
            }
        }
    }
    row *r = (row *)malloc(sizeof(row) * (tmp.n ? tmp.n : 1));
    if (!r || tmp.err) { b->err = 1; free(r); free(tmp.pos); free(tmp.pid); return; }
    for (uint64_t q = 0; q < tmp.n; q++) { r[q].pos = tmp.pos[q]; r[q].pid = tmp.pid[q]; }
    qsort(r, tmp.n, sizeof(row), row_cmp);   /* AC emits in END order */
    for (uint64_t q = 0; q < tmp.n; q++) rb_push(b, r[q].pos, r[q].pid);
    free(r); free(tmp.pos); free(tmp.pid);
}

/* ------------------------------------------------------------------ */
/* Threads over contiguous start ranges, concatenated in range order.  */
/* ------------------------------------------------------------------ */
typedef struct {
    or_trie *t; const uint8_t *T; uint64_t L, lo, hi; int engine; rowbuf b;
} job;

static void *worker(void *arg) {
    job *j = (job *)arg;
    switch (j->engine) {
    case OR_PFAC_BITMAP: walk_bitmap(j->t, j->T, j->L, j->lo, j->hi, &j->b); break;
    case OR_PFAC_CSR: walk_csr(j->t, j->T, j->L, j->lo, j->hi, &j->b); break;
    case OR_BRUTE: brute(j->t, j->T, j->L, j->lo, j->hi, &j->b); break;
    case OR_AC: ac_scan(j->t, j->T, j->L, j->lo, j->hi, &j->b); break;
    default: j->b.err = 1;
    }
    return NULL;
}

int or_match(or_trie *t, const uint8_t *T, uint64_t L, uint64_t lo, uint64_t hi, int engine, int n_threads,
             or_matches *out) {
    if (!t || !out || (L && !T) || engine < 0 || engine > 3) return OR_EINVAL;
    out->n = 0; out->pos = NULL; out->pid = NULL;
    if (hi > L) hi = L;
    if (lo >= hi) return OR_OK;
    if (engine == OR_AC) {
        pthread_mutex_lock(&t->ac_lock);
        int rc = t->ac_built ? OR_OK : ac_build(t);
        pthread_mutex_unlock(&t->ac_lock);
        if (rc) return rc;
    }
    if (n_threads <= 0) n_threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (n_threads > 512) n_threads = 512;
    uint64_t span = hi - lo;
    if ((uint64_t)n_threads > span) n_threads = (int)span;
    job *jobs = (job *)calloc((size_t)n_threads, sizeof(job));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return OR_ENOMEM; }
    for (int k = 0; k < n_threads; k++) {
        jobs[k].t = t; jobs[k].T = T; jobs[k].L = L; jobs[k].engine = engine;
        jobs[k].lo = lo + span * (uint64_t)k / (uint64_t)n_threads;
        jobs[k].hi = lo + span * (uint64_t)(k + 1) / (uint64_t)n_threads;
    }
    if (n_threads == 1) worker(&jobs[0]);
    else {
        for (int k = 0; k < n_threads; k++) pthread_create(&th[k], NULL, worker, &jobs[k]);
        for (int k = 0; k < n_threads; k++) pthread_join(th[k], NULL);
    }
    int err = 0;
    uint64_t tot = 0;
    for (int k = 0; k < n_threads; k++) { err |= jobs[k].b.err; tot += jobs[k].b.n; }
    if (!err && tot) {
        out->pos = (uint64_t *)malloc(tot * sizeof(uint64_t));
        out->pid = (uint32_t *)malloc(tot * sizeof(uint32_t));
        if (!out->pos || !out->pid) err = 1;
    }
    uint64_t o = 0;
    for (int k = 0; k < n_threads; k++) {
        if (!err && jobs[k].b.n) {
            memcpy(out->pos + o, jobs[k].b.pos, jobs[k].b.n * sizeof(uint64_t));
            memcpy(out->pid + o, jobs[k].b.pid, jobs[k].b.n * sizeof(uint32_t));
            o += jobs[k].b.n;
        }
        free(jobs[k].b.pos); free(jobs[k].b.pid);
    }
    free(jobs); free(th);
    if (err) { free(out->pos); free(out->pid); out->pos = NULL; out->pid = NULL; return OR_ENOMEM; }
    out->n = tot;
    return OR_OK;
}

void or_matches_free(or_matches *m) {
    if (!m) return;
    free(m->pos); free(m->pid);
    m->pos = NULL; m->pid = NULL; m->n = 0;
}

/*
 * oracle.h -- CPU ORACLE for the PFAC scan of arXiv 1702.03657.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg / `--impl reference` arm may load, call or
 * link this.  The product path (paper_1702_03657_b200/) never does; the two
 * share no code, headers, tables or helpers.
 *
 * What it computes (SURVEY.md §8(c), §II-B problem statement,
 * PAPER.md:76 §II-C PFAC):
 *
 *     M = { (i, k) : lo <= i < hi, i + |P_k| <= L, T[i .. i+|P_k|) = P_k }
 *
 * listed in ascending (i, k) order, where L = readable_len.  Four engines
 * reach M independently:
 *   OR_PFAC_BITMAP  the paper's uncompressed trie: BFS row-major array of
 *                   36-byte nodes (256-bit child bitmap + u32 first-child
 *                   offset, Fig. 3), child located
 *                   by popcount rank (SPEC S:102 reading of P:97), one walk
 *                   per start position that continues past matches and stops
 *                   at the first mismatch.
 *   OR_PFAC_CSR     the same walk over the oracle's own label-CSR encoding of
 *                   that trie (PAPER.md:89, :101 CRS step) -- "compressed ==
 *                   uncompressed" invariant (BASELINE.json north_star).
 *   OR_BRUTE        memcmp of every pattern at every start (tiny inputs).
 *   OR_AC           textbook Aho-Corasick DFA with failure links
 *                   (§II-B), chunk-parallel; each chunk reads
 *                   (longest pattern - 1) bytes past its end.
 * Parity is pinned in tests/test_oracle.py.
 */
#ifndef PFAC_ORACLE_H
#define PFAC_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_trie or_trie;

enum { OR_OK = 0, OR_EINVAL = -1, OR_ENOMEM = -2, OR_ETOOBIG = -3 };
enum { OR_PFAC_BITMAP = 0, OR_PFAC_CSR = 1, OR_BRUTE = 2, OR_AC = 3 };

typedef struct { uint64_t n; uint64_t *pos; uint32_t *pid; } or_matches;

/* Patterns are concatenated in `data`, lengths in `lens` (binary-safe). */
int  or_build(const uint8_t *data, const uint32_t *lens, uint32_t n, or_trie **out);
void or_free(or_trie *t);

/* out[0..5] = nodes, edges, terminals, n_patterns, max_len, min_len */
void or_stats(const or_trie *t, uint64_t out[6]);
/* 36-byte node v: 8 bitmap words + first-child offset (0 for a leaf). */
int  or_node(const or_trie *t, uint32_t v, uint32_t bitmap[8], uint32_t *offset);
/* Pattern ids whose last byte ends at node v (ascending). */
int  or_node_pids(const or_trie *t, uint32_t v, const uint32_t **pids, uint32_t *n);
/* Child by the rank rule, -1 if none (SPEC child_lookup). */
int64_t or_child(const or_trie *t, uint32_t v, uint32_t c);

/* Byte accounting.  kind 0: 36*N uncompressed; 1: 1024*N dense
 * PFAC state table (256 x u32 per state); 2: paper CRS of the N x 9 word
 * matrix, (2*nnz + n + 1) x 4 bytes. */
uint64_t or_bytes(const or_trie *t, int kind);
/* Paper CRS arrays of the N x 9 word matrix (Fig. 1(C,D)); malloc'd. */
int or_paper_crs(const or_trie *t, uint32_t **val, uint32_t **col_ind, uint32_t **row_ptr,
                 uint64_t *nnz, uint64_t *n_rows);
/* Oracle's own label CSR (row_ptr[N+1], label[E], child[E]); owned by t. */
int or_csr(const or_trie *t, const uint32_t **row_ptr, const uint8_t **label, const uint32_t **child);

/* Matches with start in [lo, hi), reading text[0 .. readable_len). */
int  or_match(or_trie *t, const uint8_t *text, uint64_t readable_len, uint64_t lo, uint64_t hi,
              int engine, int n_threads, or_matches *out);
void or_matches_free(or_matches *m);

#ifdef __cplusplus
}
#endif
#endif

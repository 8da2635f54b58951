/*
 * pfac_gen.h -- seeded, chunk-deterministic synthetic INPUT generators.
 *
 * This module produces pattern sets and text for the five BASELINE.json
 * configurations (SURVEY.md §8(d) "Concrete synthetic inputs", generator G1).
 * It holds NONE of the method's arithmetic (no trie, no matching): it only
 * draws bytes.  It is the one piece of code that both the oracle side
 * (tests/, bench.py cpu_baseline) and the CUDA side (tests, bench.py) use, so
 * that both see identical inputs (task rule ③).
 *
 * Random sources:
 *   - splitmix64 (Steele, Lea, Flood 2014) for text/plant streams; chunk c of
 *     the text is generated from state  seed + c * 0x9E3779B97F4A7C15, so any
 *     byte range (a shard, a halo) can be materialised independently.
 *   - MT19937-64 (Matsumoto & Nishimura; C++ std::mt19937_64 parameters) for
 *     pattern sampling, as the paper samples patterns with Mersenne Twister
 *     (§VII).
 *   - Uniform draw in [0,n): multiply-shift ((u128)r*n) >> 64.
 *
 * Text is a concatenation of PG_CHUNK-byte chunks; each chunk = background
 * (config-specific distribution) + planted pattern occurrences (each S-byte
 * slot planted with probability p; pid uniform over patterns with len <= S;
 * offset uniform in [0, S-len]).  Plants never cross a chunk boundary.
 */
#ifndef PFAC_GEN_H
#define PFAC_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define PG_CHUNK (1u << 20)

typedef struct {
    int id;                /* 1..5 = BASELINE.json configs[0..4] */
    uint64_t text_len;     /* default full size (bytes) */
    uint32_t n_patterns;
    uint32_t min_len, max_len;
    uint64_t seed_pat, seed_text, seed_plant;
    uint32_t plant_slot;   /* S */
    uint32_t plant_p_q20;  /* p * 2^20 */
} pg_config;

/* MT19937-64 state (C++ [rand.predef] mt19937_64 parameters). */
typedef struct { uint64_t mt[312]; int mti; } pg_mt64;
void     pg_mt64_seed(pg_mt64 *m, uint64_t seed);
uint64_t pg_mt64_next(pg_mt64 *m);
uint64_t pg_splitmix64_next(uint64_t *state);

/* Returns 0 on success, -1 for an unknown config id. */
int pg_config_get(int id, pg_config *out);

/* Patterns: malloc'd concatenated bytes + lengths; free with pg_free. */
int pg_make_patterns(const pg_config *c, uint8_t **data, uint32_t **lens, uint32_t *n_out);

/* Text bytes [start, start+len) of config c with the given pattern set
 * (needed for plants).  n_threads <= 0 means "all online cores". */
int pg_make_text(const pg_config *c, const uint8_t *pat_data, const uint32_t *pat_lens,
                 uint32_t n_pat, uint64_t start, uint64_t len, uint8_t *out, int n_threads);

/* Planted occurrences (pos, pid) whose slot lies in chunks [c0, c1), in
 * position order; malloc'd, free with pg_free.  Used only by tests
 * (completeness-on-plants invariant). */
int pg_plants(const pg_config *c, const uint8_t *pat_data, const uint32_t *pat_lens,
              uint32_t n_pat, uint64_t c0, uint64_t c1, uint64_t **pos, uint32_t **pid,
              uint64_t *n_out);

void pg_free(void *p);

#ifdef __cplusplus
}
#endif
#endif

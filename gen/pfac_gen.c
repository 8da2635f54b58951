/*
 * pfac_gen.c -- synthetic input generators (see pfac_gen.h).
 * Recipe: SURVEY.md §8(d) "Concrete synthetic inputs" table (C1..C5), restated
 * in DESIGN.md §"Input recipe".  No matching arithmetic lives here.
 */
#define _GNU_SOURCE
#include "pfac_gen.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define GOLDEN 0x9E3779B97F4A7C15ull

/* ------------------------------------------------------------------ RNGs */
uint64_t pg_splitmix64_next(uint64_t *s) {
    uint64_t z = (*s += GOLDEN);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* MT19937-64 below follows the reference algorithm of Matsumoto and
 * Nishimura (mt19937-64.c); its exact output is required (pinned to the C++
 * [rand.predef] value in tests/golden/rng.json).  That reference code carries
 * this notice:
 *
 *   Copyright (C) 2004, Makoto Matsumoto and Takuji Nishimura,
 *   All rights reserved.
 *
 *   Redistribution and use in source and binary forms, with or without
 *   modification, are permitted provided that the following conditions
 *   are met:
 *     1. Redistributions of source code must retain the above copyright
 *        notice, this list of conditions and the following disclaimer.
 *     2. Redistributions in binary form must reproduce the above copyright
 *        notice, this list of conditions and the following disclaimer in the
 *        documentation and/or other materials provided with the distribution.
 *     3. The names of its contributors may not be used to endorse or promote
 *        products derived from this software without specific prior written
 *        permission.
 *
 *   THIS SOFTWARE IS PROVIDED BY THE COPYRIGHT HOLDERS AND CONTRIBUTORS
 *   "AS IS" AND ANY EXPRESS OR IMPLIED WARRANTIES, INCLUDING, BUT NOT
 *   LIMITED TO, THE IMPLIED WARRANTIES OF MERCHANTABILITY AND FITNESS FOR
 *   A PARTICULAR PURPOSE ARE DISCLAIMED.  IN NO EVENT SHALL THE COPYRIGHT
 *   OWNER OR CONTRIBUTORS BE LIABLE FOR ANY DIRECT, INDIRECT, INCIDENTAL,
 *   SPECIAL, EXEMPLARY, OR CONSEQUENTIAL DAMAGES (INCLUDING, BUT NOT
 *   LIMITED TO, PROCUREMENT OF SUBSTITUTE GOODS OR SERVICES; LOSS OF USE,
 *   DATA, OR PROFITS; OR BUSINESS INTERRUPTION) HOWEVER CAUSED AND ON ANY
 *   THEORY OF LIABILITY, WHETHER IN CONTRACT, STRICT LIABILITY, OR TORT
 *   (INCLUDING NEGLIGENCE OR OTHERWISE) ARISING IN ANY WAY OUT OF THE USE
 *   OF THIS SOFTWARE, EVEN IF ADVISED OF THE POSSIBILITY OF SUCH DAMAGE. */
#define MT_NN 312
#define MT_MM 156
void pg_mt64_seed(pg_mt64 *m, uint64_t seed) {
    m->mt[0] = seed;
    for (int i = 1; i < MT_NN; i++)
        m->mt[i] = 6364136223846793005ull * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
    m->mti = MT_NN;
}
uint64_t pg_mt64_next(pg_mt64 *m) {
    static const uint64_t MAG[2] = {0ull, 0xB5026F5AA96619E9ull};
    const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    if (m->mti >= MT_NN) {
        int i;
        uint64_t x;
        for (i = 0; i < MT_NN - MT_MM; i++) {
            x = (m->mt[i] & UM) | (m->mt[i + 1] & LM);
            m->mt[i] = m->mt[i + MT_MM] ^ (x >> 1) ^ MAG[x & 1];
        }
        for (; i < MT_NN - 1; i++) {
            x = (m->mt[i] & UM) | (m->mt[i + 1] & LM);
            m->mt[i] = m->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ MAG[x & 1];
        }
        x = (m->mt[MT_NN - 1] & UM) | (m->mt[0] & LM);
        m->mt[MT_NN - 1] = m->mt[MT_MM - 1] ^ (x >> 1) ^ MAG[x & 1];
        m->mti = 0;
    }
    uint64_t x = m->mt[m->mti++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= (x >> 43);
    return x;
}

static inline uint64_t unif(uint64_t r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)r * n) >> 64);
}
static inline uint64_t sm_unif(uint64_t *s, uint64_t n) { return unif(pg_splitmix64_next(s), n); }
static inline uint64_t mt_unif(pg_mt64 *m, uint64_t n) { return unif(pg_mt64_next(m), n); }

void pg_free(void *p) { free(p); }

/* Start state of chunk c's stream.  NOT seed + c*GOLDEN: splitmix64 advances
 * its state by GOLDEN per draw, so that seeding would make chunk c a copy of
 * chunk 0 shifted by c draws.  Hashing (seed, c) puts every chunk at an
 * unrelated point of the 2^64-long sequence (input recipe). */
static uint64_t chunk_state(uint64_t seed, uint64_t chunk) {
    uint64_t s = seed ^ (chunk * 0xD1B54A32D192ED03ull);
    uint64_t h = pg_splitmix64_next(&s);
    return h ^ (seed * 0x9E6C63D0676A9A99ull);
}

/* -------------------------------------------------------------- configs */
int pg_config_get(int id, pg_config *c) {
    memset(c, 0, sizeof *c);
    c->id = id;
    c->seed_pat = 1000 + (uint64_t)id;
    c->seed_text = 2000 + (uint64_t)id;
    c->seed_plant = 3000 + (uint64_t)id;
    c->plant_slot = 4096;
    c->plant_p_q20 = 1u << 19; /* p = 1/2 */
    switch (id) {
    case 1: /* toy {he,she,his,hers}, 1 KiB printable ASCII, S=64 p=1 */
        c->text_len = 1024; c->n_patterns = 4; c->min_len = 2; c->max_len = 4;
        c->plant_slot = 64; c->plant_p_q20 = 1u << 20;
        return 0;
    case 2: /* 1,000 printable-ASCII patterns len 4..32, 64 MiB */
        c->text_len = 64ull << 20; c->n_patterns = 1000; c->min_len = 4; c->max_len = 32;
        return 0;
    case 3: /* 10,000 Snort/ClamAV-shaped patterns len 8..64, 1 GiB packets */
        c->text_len = 1ull << 30; c->n_patterns = 10000; c->min_len = 8; c->max_len = 64;
        return 0;
    case 4: /* 100,000 byte patterns len 4..128, 4 GiB uniform bytes */
        c->text_len = 4ull << 30; c->n_patterns = 100000; c->min_len = 4; c->max_len = 128;
        return 0;
    case 5: /* DNA, 50,000 k-mers k=16..32, 16 GiB genome-like */
        c->text_len = 16ull << 30; c->n_patterns = 50000; c->min_len = 16; c->max_len = 32;
        return 0;
    case 6: /* C4's ASCII variant (reported): 100,000 printable patterns len 4..128,
               4 GiB printable text */
        c->text_len = 4ull << 30; c->n_patterns = 100000; c->min_len = 4; c->max_len = 128;
        return 0;
    case 7: /* C2's paper-shaped variant (reported): 1,000 patterns len 4..32
               MT-sampled as substrings of the first 4 MiB of a Zipf(1.0) word text (20 K
               pseudo-words), 64 MiB of that text */
        c->text_len = 64ull << 20; c->n_patterns = 1000; c->min_len = 4; c->max_len = 32;
        return 0;
    case 8: /* C2's dense variant (reported): C2 with every 64-byte slot planted */
        c->text_len = 64ull << 20; c->n_patterns = 1000; c->min_len = 4; c->max_len = 32;
        c->plant_slot = 64; c->plant_p_q20 = 1u << 20;
        return 0;
    default:
        return -1;
    }
}

/* ------------------------------------------------- C3 token vocabulary */
#define C3_VOCAB 512
static const char *C3_FIXED[] = {
    "GET /", "POST /", "HTTP/1.1", "HTTP/1.0", "Host: ", "User-Agent: ", "Accept: ",
    "Cookie: ", "Content-Length: ", "Content-Type: ", "cmd.exe", "/bin/sh", "%2e%2e%2f",
    "../", "SELECT ", "UNION ", "FROM ", "WHERE ", "<script>", "alert(", "eval(", "base64",
    "powershell", "wget ", "curl ", "/etc/passwd", "admin", "login", "password", "root",
    "Mozilla/5.0", "Windows NT", "text/html", ".php", ".asp", "?id=", "&cmd=", "MZ",
    "This program cannot be run in DOS mode", "CreateRemoteThread", "VirtualAlloc",
    "LoadLibraryA", "GetProcAddress", "kernel32.dll", "ws2_32.dll", "USER ", "PASS ",
    "RETR ", "EHLO ", "MAIL FROM:", "RCPT TO:", "Authorization: Basic ", "Set-Cookie: ",
    "Referer: ", "X-Forwarded-For: ", "Connection: keep-alive", "/cgi-bin/", "index.html",
    "application/octet-stream", "%00", "0x", "\\x90\\x90", "union select", "or 1=1",
};
typedef struct {
    char tok[C3_VOCAB][48];
    uint8_t len[C3_VOCAB];
    double cdf[C3_VOCAB]; /* Zipf(1.1) */
} c3_vocab_t;
static c3_vocab_t C3V;
static pthread_once_t C3V_once = PTHREAD_ONCE_INIT;
static void c3_vocab_init(void) {
    uint64_t s = 0xC3C3C3C3ull;
    int nf = (int)(sizeof C3_FIXED / sizeof C3_FIXED[0]);
    for (int i = 0; i < C3_VOCAB; i++) {
        if (i < nf) {
            size_t l = strlen(C3_FIXED[i]);
            memcpy(C3V.tok[i], C3_FIXED[i], l);
            C3V.len[i] = (uint8_t)l;
        } else {
            int l = 3 + (int)sm_unif(&s, 8); /* 3..10 letters */
            int o = 0;
            uint64_t deco = sm_unif(&s, 4);
            if (deco == 1) C3V.tok[i][o++] = '/';
            for (int k = 0; k < l; k++) C3V.tok[i][o++] = (char)('a' + sm_unif(&s, 26));
            if (deco == 2) C3V.tok[i][o++] = '=';
            if (deco == 3) C3V.tok[i][o++] = '.';
            C3V.len[i] = (uint8_t)o;
        }
    }
    double tot = 0;
    for (int r = 0; r < C3_VOCAB; r++) tot += 1.0 / pow((double)(r + 1), 1.1);
    double acc = 0;
    for (int r = 0; r < C3_VOCAB; r++) {
        acc += 1.0 / pow((double)(r + 1), 1.1) / tot;
        C3V.cdf[r] = acc;
    }
    C3V.cdf[C3_VOCAB - 1] = 1.0;
}
static int c3_zipf(uint64_t r) {
    double u = (double)(r >> 11) * (1.0 / 9007199254740992.0);
    int lo = 0, hi = C3_VOCAB - 1;
    while (lo < hi) {
        int mid = (lo + hi) / 2;
        if (u < C3V.cdf[mid]) hi = mid; else lo = mid + 1;
    }
    return lo;
}

/* ----------------------------------------------- C5 repeat families */
#define C5_FAM 32
#define C5_FAMLEN 300
static uint8_t C5F[C5_FAM][C5_FAMLEN];
static pthread_once_t C5F_once = PTHREAD_ONCE_INIT;
static const uint8_t ACGT[4] = {'A', 'C', 'G', 'T'};
static inline uint8_t dna_base(uint64_t r16) {
    /* A/T 0.295, C/G 0.205 on a 16-bit draw */
    uint32_t v = (uint32_t)(r16 & 0xFFFF);
    if (v < 19333) return 'A';      /* 0.295 * 65536 */
    if (v < 32768) return 'C';      /* +0.205 */
    if (v < 46203) return 'G';      /* +0.205 */
    return 'T';
}
static void c5_fam_init(void) {
    uint64_t s = 0xFA11FA11ull;
    for (int f = 0; f < C5_FAM; f++)
        for (int k = 0; k < C5_FAMLEN; k++) C5F[f][k] = dna_base(pg_splitmix64_next(&s));
}

/* ------------------------------------------------------- backgrounds */
static void bg_printable(uint64_t seed, uint64_t chunk, uint8_t *b) {
    uint64_t s = chunk_state(seed, chunk);
    for (uint32_t i = 0; i < PG_CHUNK; i += 4) {
        uint64_t r = pg_splitmix64_next(&s);
        for (int k = 0; k < 4; k++) b[i + k] = (uint8_t)(0x20 + (((r >> (16 * k)) & 0xFFFF) * 95 >> 16));
    }
}
static void bg_uniform(uint64_t seed, uint64_t chunk, uint8_t *b) {
    uint64_t s = chunk_state(seed, chunk);
    for (uint32_t i = 0; i < PG_CHUNK; i += 8) {
        uint64_t r = pg_splitmix64_next(&s);
        memcpy(b + i, &r, 8);
    }
}
static void bg_packets(uint64_t seed, uint64_t chunk, uint8_t *b) {
    pthread_once(&C3V_once, c3_vocab_init);
    uint64_t s = chunk_state(seed, chunk);
    static const uint16_t PORTS[8] = {80, 443, 8080, 21, 25, 22, 53, 445};
    uint32_t o = 0;
    while (o < PG_CHUNK) {
        uint64_t r = sm_unif(&s, 100);
        uint32_t plen = r < 45 ? 64 : (r < 60 ? 576 : 1500);
        uint8_t pk[1500];
        uint32_t h = 0;
        /* Ethernet: dst/src MAC random, ethertype 08 00 */
        for (int k = 0; k < 12; k++) pk[h++] = (uint8_t)sm_unif(&s, 256);
        pk[h++] = 0x08; pk[h++] = 0x00;
        /* IPv4: 45 00 len id 40 00 ttl proto csum src dst */
        pk[h++] = 0x45; pk[h++] = 0x00;
        pk[h++] = (uint8_t)((plen - 14) >> 8); pk[h++] = (uint8_t)(plen - 14);
        pk[h++] = (uint8_t)sm_unif(&s, 256); pk[h++] = (uint8_t)sm_unif(&s, 256);
        pk[h++] = 0x40; pk[h++] = 0x00; pk[h++] = 0x40; pk[h++] = 0x06;
        pk[h++] = (uint8_t)sm_unif(&s, 256); pk[h++] = (uint8_t)sm_unif(&s, 256);
        pk[h++] = 10; pk[h++] = 0; pk[h++] = (uint8_t)sm_unif(&s, 256); pk[h++] = (uint8_t)sm_unif(&s, 256);
        pk[h++] = 192; pk[h++] = 168; pk[h++] = (uint8_t)sm_unif(&s, 256); pk[h++] = (uint8_t)sm_unif(&s, 256);
        /* TCP: sport dport seq ack 50 18 win csum urg */
        uint16_t dport = PORTS[sm_unif(&s, 8)];
        pk[h++] = (uint8_t)(0xC0 | sm_unif(&s, 64)); pk[h++] = (uint8_t)sm_unif(&s, 256);
        pk[h++] = (uint8_t)(dport >> 8); pk[h++] = (uint8_t)dport;
        for (int k = 0; k < 8; k++) pk[h++] = (uint8_t)sm_unif(&s, 256);
        pk[h++] = 0x50; pk[h++] = 0x18; pk[h++] = 0xFA; pk[h++] = 0xF0;
        pk[h++] = (uint8_t)sm_unif(&s, 256); pk[h++] = (uint8_t)sm_unif(&s, 256);
        pk[h++] = 0; pk[h++] = 0;
        /* payload: 50% token-ASCII lines, 50% uniform bytes */
        if (sm_unif(&s, 2) == 0) {
            uint32_t line = 0, per_line = 4 + (uint32_t)sm_unif(&s, 9);
            while (h < plen) {
                int t = c3_zipf(pg_splitmix64_next(&s));
                for (int k = 0; k < C3V.len[t] && h < plen; k++) pk[h++] = (uint8_t)C3V.tok[t][k];
                if (++line == per_line) {
                    if (h < plen) pk[h++] = '\r';
                    if (h < plen) pk[h++] = '\n';
                    line = 0;
                } else if (h < plen) {
                    pk[h++] = ' ';
                }
            }
        } else {
            while (h < plen) {
                uint64_t v = pg_splitmix64_next(&s);
                for (int k = 0; k < 8 && h < plen; k++) pk[h++] = (uint8_t)(v >> (8 * k));
            }
        }
        uint32_t n = plen < PG_CHUNK - o ? plen : PG_CHUNK - o;
        memcpy(b + o, pk, n);
        o += n;
    }
}
#define P_REP_Q32 715828u /* 0.05/300 * 2^32: ~5% of bases inside repeat copies */
#define P_STR_Q32 780903u /* 0.02/110 * 2^32: ~2% inside short tandem repeats */
static void bg_dna(uint64_t seed, uint64_t chunk, uint8_t *b) {
    pthread_once(&C5F_once, c5_fam_init);
    uint64_t s = chunk_state(seed, chunk);
    uint32_t o = 0;
    while (o < PG_CHUNK) {
        uint64_t r = pg_splitmix64_next(&s);
        uint32_t ev = (uint32_t)(r >> 32);
        if (ev < P_REP_Q32) {
            int f = (int)sm_unif(&s, C5_FAM);
            for (int k = 0; k < C5_FAMLEN && o < PG_CHUNK; k++) {
                uint64_t m = pg_splitmix64_next(&s);
                uint8_t base = C5F[f][k];
                if (unif(m, 10) == 0) base = ACGT[(m >> 8) & 3]; /* 10% point mutation */
                b[o++] = base;
            }
        } else if (ev < P_REP_Q32 + P_STR_Q32) {
            uint8_t unit[6];
            int ul = 1 + (int)sm_unif(&s, 6);
            for (int k = 0; k < ul; k++) unit[k] = dna_base(pg_splitmix64_next(&s));
            uint32_t span = 20 + (uint32_t)sm_unif(&s, 181);
            for (uint32_t k = 0; k < span && o < PG_CHUNK; k++) b[o++] = unit[k % (uint32_t)ul];
        } else {
            b[o++] = dna_base(r);
        }
    }
}
/* ------------------------------------ C2 paper-shaped: Zipf word text */
/* 20,000 pseudo-words (2..10 lowercase letters) drawn once from a fixed seed;
 * a chunk is words drawn by Zipf(1.0) (rank k with weight 1/k, inverse CDF by
 * binary search on a 2^32-scaled cumulative table), separated by single
 * spaces; a word cut by the chunk end is cut. */
#define ZW_N 20000
static struct {
    char w[ZW_N][11];
    uint8_t len[ZW_N];
    uint64_t cdf[ZW_N]; /* cumulative weight, scaled to 2^32 */
} ZW;
static pthread_once_t ZW_once = PTHREAD_ONCE_INIT;
static void zw_init(void) {
    uint64_t s = 0x5A17F00Dull;
    double tot = 0, acc = 0;
    for (int i = 0; i < ZW_N; i++) tot += 1.0 / (i + 1);
    for (int i = 0; i < ZW_N; i++) {
        int l = 2 + (int)sm_unif(&s, 9); /* 2..10 letters */
        for (int k = 0; k < l; k++) ZW.w[i][k] = (char)('a' + sm_unif(&s, 26));
        ZW.len[i] = (uint8_t)l;
        acc += 1.0 / (i + 1);
        ZW.cdf[i] = (uint64_t)(acc / tot * 4294967296.0);
    }
    ZW.cdf[ZW_N - 1] = 1ull << 32;
}
static void bg_zipf_words(uint64_t seed, uint64_t chunk, uint8_t *b) {
    pthread_once(&ZW_once, zw_init);
    uint64_t s = chunk_state(seed, chunk);
    uint32_t o = 0;
    while (o < PG_CHUNK) {
        const uint64_t u = pg_splitmix64_next(&s) >> 32; /* uniform in [0, 2^32) */
        int lo = 0, hi = ZW_N - 1;                        /* first rank with cdf > u */
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (ZW.cdf[mid] > u) hi = mid; else lo = mid + 1;
        }
        for (int k = 0; k < ZW.len[lo] && o < PG_CHUNK; k++) b[o++] = (uint8_t)ZW.w[lo][k];
        if (o < PG_CHUNK) b[o++] = ' ';
    }
}

static void gen_background(const pg_config *c, uint64_t chunk, uint8_t *b) {
    switch (c->id) {
    case 1: case 2: case 6: case 8: bg_printable(c->seed_text, chunk, b); break;
    case 7: bg_zipf_words(c->seed_text, chunk, b); break;
    case 3: bg_packets(c->seed_text, chunk, b); break;
    case 4: bg_uniform(c->seed_text, chunk, b); break;
    case 5: bg_dna(c->seed_text, chunk, b); break;
    default: memset(b, 0, PG_CHUNK);
    }
}

/* ------------------------------------------------------------ plants */
typedef struct {
    const uint8_t *data;
    const uint32_t *lens;
    uint64_t *off;      /* byte offset of each pattern in data */
    uint32_t *elig;     /* pids with len <= S */
    uint32_t n_elig;
} pat_index;

static int pat_index_make(const pg_config *c, const uint8_t *d, const uint32_t *l, uint32_t n, pat_index *pi) {
    pi->data = d; pi->lens = l;
    pi->off = (uint64_t *)malloc(sizeof(uint64_t) * (n ? n : 1));
    pi->elig = (uint32_t *)malloc(sizeof(uint32_t) * (n ? n : 1));
    if (!pi->off || !pi->elig) return -1;
    uint64_t o = 0;
    pi->n_elig = 0;
    for (uint32_t i = 0; i < n; i++) {
        pi->off[i] = o;
        o += l[i];
        if (l[i] >= 1 && l[i] <= c->plant_slot) pi->elig[pi->n_elig++] = i;
    }
    return 0;
}
static void pat_index_free(pat_index *pi) { free(pi->off); free(pi->elig); }

/* Replays the plant stream of one chunk; if b != NULL writes the plants,
 * if (pos,pid) != NULL records them.  Returns number of plants. */
static uint64_t gen_plants(const pg_config *c, const pat_index *pi, uint64_t chunk, uint8_t *b,
                           uint64_t *pos, uint32_t *pid) {
    if (pi->n_elig == 0) return 0;
    uint64_t s = chunk_state(c->seed_plant, chunk);
    uint32_t S = c->plant_slot, nslot = PG_CHUNK / S;
    uint64_t np = 0;
    for (uint32_t k = 0; k < nslot; k++) {
        uint64_t r = pg_splitmix64_next(&s);
        if (unif(r, 1u << 20) >= c->plant_p_q20) continue;
        uint32_t p = pi->elig[sm_unif(&s, pi->n_elig)];
        uint32_t len = pi->lens[p];
        uint32_t off = (uint32_t)sm_unif(&s, (uint64_t)(S - len) + 1);
        if (b) memcpy(b + (uint64_t)k * S + off, pi->data + pi->off[p], len);
        if (pos) { pos[np] = chunk * PG_CHUNK + (uint64_t)k * S + off; pid[np] = p; }
        np++;
    }
    return np;
}

/* -------------------------------------------------------------- text */
typedef struct {
    const pg_config *c;
    const pat_index *pi;
    uint64_t start, len;
    uint8_t *out;
    uint64_t c_lo, c_hi; /* chunk range for this worker */
} text_job;

static void *text_worker(void *arg) {
    text_job *j = (text_job *)arg;
    uint8_t *buf = (uint8_t *)malloc(PG_CHUNK);
    if (!buf) return (void *)1;
    for (uint64_t ch = j->c_lo; ch < j->c_hi; ch++) {
        gen_background(j->c, ch, buf);
        gen_plants(j->c, j->pi, ch, buf, NULL, NULL);
        uint64_t cs = ch * PG_CHUNK, ce = cs + PG_CHUNK;
        uint64_t a = cs > j->start ? cs : j->start;
        uint64_t e = ce < j->start + j->len ? ce : j->start + j->len;
        if (a < e) memcpy(j->out + (a - j->start), buf + (a - cs), e - a);
    }
    free(buf);
    return NULL;
}

int pg_make_text(const pg_config *c, const uint8_t *pat_data, const uint32_t *pat_lens,
                 uint32_t n_pat, uint64_t start, uint64_t len, uint8_t *out, int n_threads) {
    if (len == 0) return 0;
    pat_index pi;
    if (pat_index_make(c, pat_data, pat_lens, n_pat, &pi)) return -1;
    uint64_t c0 = start / PG_CHUNK, c1 = (start + len + PG_CHUNK - 1) / PG_CHUNK;
    uint64_t nch = c1 - c0;
    if (n_threads <= 0) n_threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if ((uint64_t)n_threads > nch) n_threads = (int)nch;
    if (n_threads < 1) n_threads = 1;
    text_job jobs[256];
    pthread_t th[256];
    if (n_threads > 256) n_threads = 256;
    int rc = 0;
    for (int t = 0; t < n_threads; t++) {
        jobs[t].c = c; jobs[t].pi = &pi; jobs[t].start = start; jobs[t].len = len; jobs[t].out = out;
        jobs[t].c_lo = c0 + nch * (uint64_t)t / (uint64_t)n_threads;
        jobs[t].c_hi = c0 + nch * (uint64_t)(t + 1) / (uint64_t)n_threads;
        if (n_threads == 1) { if (text_worker(&jobs[t])) rc = -1; }
        else if (pthread_create(&th[t], NULL, text_worker, &jobs[t])) rc = -1;
    }
    if (n_threads > 1)
        for (int t = 0; t < n_threads; t++) { void *r; pthread_join(th[t], &r); if (r) rc = -1; }
    pat_index_free(&pi);
    return rc;
}

int pg_plants(const pg_config *c, const uint8_t *pat_data, const uint32_t *pat_lens, uint32_t n_pat,
              uint64_t c0, uint64_t c1, uint64_t **pos, uint32_t **pid, uint64_t *n_out) {
    pat_index pi;
    if (pat_index_make(c, pat_data, pat_lens, n_pat, &pi)) return -1;
    uint64_t cap = (c1 > c0 ? c1 - c0 : 0) * (PG_CHUNK / c->plant_slot) + 1;
    *pos = (uint64_t *)malloc(cap * sizeof(uint64_t));
    *pid = (uint32_t *)malloc(cap * sizeof(uint32_t));
    if (!*pos || !*pid) { pat_index_free(&pi); return -1; }
    uint64_t n = 0;
    for (uint64_t ch = c0; ch < c1; ch++) n += gen_plants(c, &pi, ch, NULL, *pos + n, *pid + n);
    *n_out = n;
    pat_index_free(&pi);
    return 0;
}

/* ---------------------------------------------------------- patterns */
typedef struct {
    uint8_t *data; uint64_t size, cap;
    uint32_t *lens; uint64_t *offs; uint32_t n, ncap;
    uint64_t *ht; uint64_t hmask; /* open addressing: stores idx+1 */
} patset;

static uint64_t fnv(const uint8_t *p, uint32_t l) {
    uint64_t h = 1469598103934665603ull;
    for (uint32_t i = 0; i < l; i++) { h ^= p[i]; h *= 1099511628211ull; }
    return h ^ l;
}
static int ps_init(patset *ps, uint32_t n) {
    memset(ps, 0, sizeof *ps);
    ps->ncap = n ? n : 1;
    ps->cap = 1 << 16;
    ps->data = (uint8_t *)malloc(ps->cap);
    ps->lens = (uint32_t *)malloc(sizeof(uint32_t) * ps->ncap);
    ps->offs = (uint64_t *)malloc(sizeof(uint64_t) * ps->ncap);
    uint64_t hs = 1;
    while (hs < 4ull * ps->ncap) hs <<= 1;
    ps->ht = (uint64_t *)calloc(hs, sizeof(uint64_t));
    ps->hmask = hs - 1;
    return (ps->data && ps->lens && ps->offs && ps->ht) ? 0 : -1;
}
/* Adds p unless it is a duplicate (then returns 0: caller resamples). */
static int ps_add(patset *ps, const uint8_t *p, uint32_t l) {
    uint64_t h = fnv(p, l) & ps->hmask;
    while (ps->ht[h]) {
        uint32_t q = (uint32_t)(ps->ht[h] - 1);
        if (ps->lens[q] == l && memcmp(ps->data + ps->offs[q], p, l) == 0) return 0;
        h = (h + 1) & ps->hmask;
    }
    if (ps->size + l > ps->cap) {
        while (ps->size + l > ps->cap) ps->cap *= 2;
        ps->data = (uint8_t *)realloc(ps->data, ps->cap);
    }
    memcpy(ps->data + ps->size, p, l);
    ps->offs[ps->n] = ps->size;
    ps->lens[ps->n] = l;
    ps->size += l;
    ps->n++;
    ps->ht[h] = ps->n;
    return 1;
}

/* A k-mer is low-complexity when some period p in 1..6 explains >= 75% of
 * it (s[j] == s[j+p]); such k-mers (poly-T, STR units) are masked from the
 * sampled half of C5, as genomic k-mer sets usually are. */
static int low_complexity(const uint8_t *s, uint32_t l) {
    for (uint32_t p = 1; p <= 6 && p < l; p++) {
        uint32_t same = 0;
        for (uint32_t j = 0; j + p < l; j++) same += s[j] == s[j + p];
        if (4 * same >= 3 * (l - p)) return 1;
    }
    return 0;
}

int pg_make_patterns(const pg_config *c, uint8_t **data, uint32_t **lens, uint32_t *n_out) {
    patset ps;
    if (ps_init(&ps, c->n_patterns)) return -1;
    pg_mt64 mt;
    pg_mt64_seed(&mt, c->seed_pat);
    uint8_t p[256];
    uint8_t *bgcache = NULL;
    uint64_t bgchunks = 0;
    if (c->id == 1) {
        static const char *toy[4] = {"he", "she", "his", "hers"};
        for (int i = 0; i < 4; i++) ps_add(&ps, (const uint8_t *)toy[i], (uint32_t)strlen(toy[i]));
    } else if (c->id == 2 || c->id == 4 || c->id == 6 || c->id == 8) {
        uint32_t span = c->max_len - c->min_len + 1;
        while (ps.n < c->n_patterns) {
            uint32_t l = c->min_len + (uint32_t)mt_unif(&mt, span);
            for (uint32_t k = 0; k < l; k++)
                p[k] = c->id != 4 ? (uint8_t)(0x20 + mt_unif(&mt, 95)) : (uint8_t)mt_unif(&mt, 256);
            ps_add(&ps, p, l);
        }
    } else if (c->id == 3) {
        pthread_once(&C3V_once, c3_vocab_init);
        while (ps.n < c->n_patterns) {
            uint32_t l = c->min_len + (uint32_t)mt_unif(&mt, c->max_len - c->min_len + 1);
            uint32_t o = 0;
            uint64_t kind = mt_unif(&mt, 100);
            if (ps.n > 0 && mt_unif(&mt, 10) == 0) {
                /* ~10%: extend an earlier pattern (nested terminals) */
                uint32_t q = (uint32_t)mt_unif(&mt, ps.n);
                uint32_t ql = ps.lens[q];
                if (ql >= c->max_len) continue;
                if (l <= ql) l = ql + 1 + (uint32_t)mt_unif(&mt, c->max_len - ql);
                memcpy(p, ps.data + ps.offs[q], ql);
                o = ql;
                while (o < l) p[o++] = (uint8_t)mt_unif(&mt, 256);
            } else if (kind < 40) { /* >= 2 ASCII tokens (uniform over the vocabulary) */
                uint32_t first = 0;
                int nt = 0;
                while (o < c->max_len && (nt < 2 || o < l)) {
                    int t = (int)mt_unif(&mt, C3_VOCAB);
                    for (int k = 0; k < C3V.len[t] && o < c->max_len; k++) p[o++] = (uint8_t)C3V.tok[t][k];
                    if (nt++ == 0) first = o;
                    if (o < c->max_len && mt_unif(&mt, 2)) p[o++] = ' ';
                }
                /* the pattern reaches at least 2 bytes past the first token */
                if (l < first + 2) l = first + 2 < c->max_len ? first + 2 : c->max_len;
                if (l > o) l = o;
                o = l;
            } else if (kind < 80) { /* uniform binary */
                while (o < l) p[o++] = (uint8_t)mt_unif(&mt, 256);
            } else { /* token prefix + binary tail (>= 2 binary bytes) */
                int t = (int)mt_unif(&mt, C3_VOCAB);
                for (int k = 0; k < C3V.len[t] && o + 2 < l; k++) p[o++] = (uint8_t)C3V.tok[t][k];
                while (o < l) p[o++] = (uint8_t)mt_unif(&mt, 256);
            }
            ps_add(&ps, p, l);
        }
    } else if (c->id == 7) {
        /* substrings of the first 4 MiB of the text's background */
        bgchunks = 4;
        bgcache = (uint8_t *)malloc(bgchunks * PG_CHUNK);
        if (!bgcache) return -1;
        for (uint64_t ch = 0; ch < bgchunks; ch++) gen_background(c, ch, bgcache + ch * PG_CHUNK);
        while (ps.n < c->n_patterns) {
            uint32_t l = c->min_len + (uint32_t)mt_unif(&mt, c->max_len - c->min_len + 1);
            uint64_t off = mt_unif(&mt, bgchunks * PG_CHUNK - l + 1);
            memcpy(p, bgcache + off, l);
            ps_add(&ps, p, l);
        }
    } else if (c->id == 5) {
        pthread_once(&C5F_once, c5_fam_init);
        bgchunks = 64; /* sample from the background of the first 64 MiB */
        bgcache = (uint8_t *)malloc(bgchunks * PG_CHUNK);
        uint8_t *have = (uint8_t *)calloc(bgchunks, 1);
        if (!bgcache || !have) { free(bgcache); free(have); return -1; }
        while (ps.n < c->n_patterns) {
            uint32_t l = c->min_len + (uint32_t)mt_unif(&mt, c->max_len - c->min_len + 1);
            if (mt_unif(&mt, 2) == 0) {
                uint64_t ch = mt_unif(&mt, bgchunks);
                uint64_t off = mt_unif(&mt, PG_CHUNK - l + 1);
                if (!have[ch]) { gen_background(c, ch, bgcache + ch * PG_CHUNK); have[ch] = 1; }
                memcpy(p, bgcache + ch * PG_CHUNK + off, l);
                if (low_complexity(p, l)) continue; /* dust-style mask: resample */
            } else {
                for (uint32_t k = 0; k < l; k++) p[k] = dna_base(pg_mt64_next(&mt));
            }
            ps_add(&ps, p, l);
        }
        free(have);
    } else {
        return -1;
    }
    free(bgcache);
    free(ps.ht);
    free(ps.offs);
    *data = ps.data;
    *lens = ps.lens;
    *n_out = ps.n;
    return 0;
}

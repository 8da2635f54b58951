/*
 * pfac.h -- C ABI of the B200-native PFAC scan (arXiv 1702.03657).
 *
 * The operation (§II-B "searching for a pattern P in a text T";
 * PAPER.md:76 §II-C parallel failure-less Aho-Corasick: "Each thread is
 * assigned to a single letter in the text T. If a match is recorded, the
 * thread continues the matching process until a mismatch."): given patterns
 * P_0..P_{m-1} (byte strings, |P_k| >= 1, pid k = input index) and text T,
 *
 *     M = { (i, k) : i + |P_k| <= L  and  T[i .. i+|P_k|) == P_k }
 *
 * listed in ascending (pos, pid) order (BASELINE.json north_star; SURVEY.md
 * §8(c) ledger L1-L3).  The trie is built on the host (PAPER.md:80 steps I-II,
 * breadth-first, row-major), compressed to a CSR image
 * and scanned by sm_100a kernels; no step runs on the CPU at match time and
 * there is no CPU fallback: without a usable CUDA device the match calls
 * return PFAC_ERR_CUDA.
 *
 * Conventions:
 *  - Every entry point returns pfac_status (or void for the free functions);
 *    nothing aborts, exits or throws across this boundary.  On failure
 *    pfac_last_error() returns thread-local detail text.
 *  - Handles are immutable after pfac_build/pfac_attach; a const handle may be
 *    used by any number of host threads concurrently (the lazy per-device
 *    upload is internally locked).
 *  - Sizes are bytes unless stated.  Positions are u64, pattern ids u32.
 */
#ifndef PFAC_H
#define PFAC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pfac_trie pfac_trie;   /* opaque */
typedef struct CUstream_st *pfac_stream; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    PFAC_OK = 0,
    PFAC_ERR_INVALID_ARG = 1,  /* NULL pointer, n_patterns == 0, zero-length pattern, length > 65535, bad enum, bad image */
    PFAC_ERR_LIMIT = 2,        /* trie exceeds 2^30-1 nodes, or the per-terminal pattern-id lists
                                  (each terminal lists the ids ending on its root path) exceed
                                  2^28 entries (e.g. tens of thousands of nested patterns) */
    PFAC_ERR_NOMEM = 3,        /* host or device allocation failed */
    PFAC_ERR_CUDA = 4,         /* no usable device / CUDA runtime error (detail in pfac_last_error) */
    PFAC_ERR_CAPACITY = 5      /* (pfac_match only, never device path) internal retry failed */
} pfac_status;

typedef enum {
    PFAC_BYTES_DEVICE_IMAGE = 0,  /* the whole device image: CSR trie + terminal tables + scan filter + root table */
    PFAC_BYTES_UNCOMPRESSED = 1,  /* the paper's original trie: 36 B per node (256-bit bitmap + u32 offset) */
    PFAC_BYTES_DENSE_STT = 2,     /* Lin et al. PFAC state table: 256 x u32 per node */
    PFAC_BYTES_PAPER_CRS = 3,     /* paper CRS of the N x 9 word matrix: (2 nnz + n + 1) x 4 B */
    PFAC_BYTES_CSR_CORE = 4,      /* the path-compressed CSR trie alone: node words (4 B/node) + labels (1 B/edge) + records (16 B + path bytes each) */
    PFAC_BYTES_TRUNCATED = 5,     /* the paper's trie truncated at depth d (PAPER.md:80 step III): 36 B x nodes of depth <= d
                                     (= PFAC_BYTES_UNCOMPRESSED when built untruncated) */
    /* built with merge_suffixes only (INVALID_ARG otherwise): */
    PFAC_BYTES_MERGED = 6,        /* id-preserving minimal DAG (steps IV-V): 36 B x DAG nodes */
    PFAC_BYTES_MERGED_CRS = 7,    /* its N x 9 CRS: (2 nnz + n + 1) x 4 B */
    PFAC_BYTES_MERGED_IMAGE = 8,  /* its device sections: node words, labels, child ids, rank skips, rank table */
    PFAC_BYTES_PIPE_TRUNC = 9,    /* the paper's pipeline: trie cut at 8 levels (or truncate_depth), 36 B/node */
    PFAC_BYTES_PIPE_MERGED = 10,  /* ... its identical sub-tries merged by shape and terminal flag (no identity), 36 B/node */
    PFAC_BYTES_PIPE_CRS = 11      /* ... then as the N x 9 CRS, (2 nnz + n + 1) x 4 B */
} pfac_bytes_kind;

typedef struct {
    uint64_t nodes;       /* 1 + number of distinct non-empty pattern prefixes (the uncompressed trie) */
    uint64_t edges;       /* nodes - 1 */
    uint64_t terminals;   /* nodes where at least one pattern ends */
    uint32_t n_patterns;
    uint32_t max_len;     /* longest pattern; (max_len - 1) is the halo a shard must read */
    uint32_t min_len;
    uint32_t filter_gram; /* d of the d-gram first-stage filter (<= min(4, min_len)) */
    uint32_t filter_log2_bits;
    uint32_t image_nodes; /* nodes stored in the device image after path compression of single-path tails */
    uint32_t truncate_depth; /* 0: untruncated; d: truncated at depth d with on-device verification */
    uint32_t verify_candidates; /* candidate records of the verify leaves (truncated tries) */
} pfac_stats;

/* Build options (pfac_build_ex).  NULL means "all defaults"; initialise a
 * struct with pfac_build_options_init() and change the fields you need.
 * These select experiments and ablations (tools/, tests/); the default build
 * is the product configuration. */
typedef struct {
    uint32_t struct_bytes;       /* sizeof(pfac_build_options); INVALID_ARG if smaller than the
                                    library's version of the struct */
    int32_t filter_kind;         /* -1: automatic.  0..4 force a first-stage filter kind (image.h);
                                    INVALID_ARG if the pattern set does not admit it (e.g. kind 3
                                    needs an all-A/C/G/T set with shortest >= 16) */
    uint32_t pair_bits_per_key;  /* kind 2 sizing: filter bits per distinct 4-gram (0: 512) */
    uint32_t gram8_bits_per_key; /* kind 4 sizing: filter bits per distinct 8-byte prefix (0: 32) */
    uint32_t truncate_depth;     /* 0: untruncated trie (default).  d >= 1: PAPER.md:80 step III,
                                    the trie is cut at level d; a start that reaches a depth-d
                                    node is verified on the device against the full bytes of
                                    the patterns below it (exact results either way) */
    uint32_t merge_suffixes;     /* 1: also build the minimal DAG of the trie (PAPER.md:80 steps IV-V:
                                    similar suffixes and end nodes merged) with pattern identity kept
                                    by path rank (image.h dag_*), scannable with the plan option
                                    form = PFAC_FORM_MERGED_DAG, and the paper-pipeline byte counts
                                    (PFAC_BYTES_PIPE_*) */
    uint32_t reserved[6];        /* must be 0 */
} pfac_build_options;

/* Which structure a scan walks (pfac_plan_options.form). */
typedef enum {
    PFAC_FORM_CSR_TRIE = 0,   /* the path-compressed CSR trie with the first-stage filters (the product path) */
    PFAC_FORM_MERGED_DAG = 1  /* the id-preserving merged DAG (built with merge_suffixes): a plain walk
                                 per start with path-rank terminals (NEXT-2; exact, not tuned) */
} pfac_form;

/* Shared-memory placement of the trie for one scan (the analog of the paper's
 * Fig. 6 global vs texture + shared-memory study). */
typedef enum {
    PFAC_PLACE_AUTO = 0,    /* planner's choice (below) */
    PFAC_PLACE_GLOBAL = 1,  /* no trie level staged: root table + level-1 bitmaps only, the rest via L1/L2 */
    PFAC_PLACE_SMEM = 2,    /* the whole trie, else its BFS prefix (upper levels), in shared memory */
    PFAC_PLACE_BIG_L1 = 3,  /* no trie level staged, 2-slot text ring, one filter copy: the
                               largest L1 carve-out for the nodes the walks visit */
    PFAC_PLACE_CLUSTER = 4  /* thread-block clusters of pfac_plan_options.cluster CTAs: the node
                               records of the trie's BFS prefix are spread over the cluster's shared
                               memories (CTA q holds a power-of-two slice) and walks read them through
                               distributed shared memory (ld.shared::cluster); 2-slot ring, one filter
                               copy.  Filter kinds 1, 3 and 4 (the tries larger than one SM's shared
                               memory); LIMIT for the others.  The grid is the co-resident clusters. */
} pfac_placement;

/* Scan-plan options (pfac_match_device_ex, pfac_plan_query).  NULL = the
 * automatic plan; initialise with pfac_plan_options_init() (every field
 * automatic) and change the fields you need.  -1 in a signed field =
 * automatic. */
typedef struct {
    uint32_t struct_bytes;        /* sizeof(pfac_plan_options) */
    uint32_t placement;           /* pfac_placement */
    uint32_t hot_bytes_cap;       /* cap on the staged trie bytes (0: none) */
    int32_t max_filter_rep_log2;  /* cap on filter copies in shared memory (2^x), -1 auto */
    int32_t ring_slots;           /* text ring slots per warp: 2, 3, or -1 auto */
    int32_t ctg64;                /* share of a CTA's rounds in per-warp blocks, in 64ths (0..64) */
    int32_t pool64;               /* share of all rounds in the cross-CTA pool, in 64ths (0..32) */
    int32_t stage2;               /* 2-gram prefix test of filter survivors: 0 off, 1 on */
    int32_t entry;                /* entry table (walks enter below the top levels): 0 off, 1 on */
    uint32_t l2_persist;          /* 1: the device image is given as an L2 persisting access-policy
                                     window for this launch (sets the device's persisting-L2 limit
                                     to min(image, 64 MiB) on first use) */
    uint32_t form;                /* pfac_form (PFAC_FORM_MERGED_DAG needs a trie built with merge_suffixes) */
    uint32_t cluster;             /* CTAs per cluster for PFAC_PLACE_CLUSTER: 2, 4 or 8 (0: 2) */
    uint32_t reserved[4];         /* must be 0 */
} pfac_plan_options;

/* Fill *o with the defaults (struct_bytes set, every choice automatic). */
void pfac_build_options_init(pfac_build_options *o);
void pfac_plan_options_init(pfac_plan_options *o);

/* What the planner chose for a scan (pfac_plan_query). */
typedef struct {
    uint32_t filter_kind, ring_slots, filter_copies, smem_bytes;
    uint32_t hot_nodes, image_nodes, hot_edges, terms_in_smem;
    uint32_t grid, warps_per_cta, hit_cap, stage2;
    uint32_t entry, kset, pool_rounds, placement;
    uint64_t rounds_per_cta, main_rounds;
    uint32_t cluster;    /* CTAs per cluster (1: no cluster) */
    uint32_t dsm_nodes;  /* nodes [0, dsm_nodes) read from the cluster's shared memories (PFAC_PLACE_CLUSTER) */
} pfac_plan_info;

/* Host-side result of pfac_match: library-allocated, free with pfac_matches_free.
 * count == 0 => pos == pid == NULL. */
typedef struct {
    uint64_t count;
    uint64_t *pos;
    uint32_t *pid;
} pfac_matches;

/* ---------------------------------------------------------------- build */

/* Builds the trie of `n_patterns` patterns.  patterns[k] points at lengths[k]
 * bytes (not NUL-terminated, may contain 0x00); they are copied, so the caller
 * may free them on return.  Duplicates are accepted and each id is reported.
 * Errors: INVALID_ARG (see enum), LIMIT, NOMEM.  *out is NULL on error. */
pfac_status pfac_build(const uint8_t *const *patterns, const uint32_t *lengths, uint32_t n_patterns,
                       pfac_trie **out);

/* Same, patterns concatenated in `data` (offset of k = sum of lengths[0..k)). */
pfac_status pfac_build_concat(const uint8_t *data, const uint32_t *lengths, uint32_t n_patterns,
                              pfac_trie **out);

/* pfac_build_concat with build options (NULL = defaults, identical to
 * pfac_build_concat).  PAPER.md:80 steps I-III (truncate_depth).  Extra
 * errors: INVALID_ARG for a bad struct_bytes, a non-zero reserved field or a
 * filter kind the set does not admit. */
pfac_status pfac_build_ex(const uint8_t *data, const uint32_t *lengths, uint32_t n_patterns,
                          const pfac_build_options *opt, pfac_trie **out);

/* Frees the host image and every device copy.  NULL-safe. */
void pfac_free(pfac_trie *t);

/* Byte accounting of the trie (PAPER.md:134 36 B/node; PAPER.md:101 CRS cost). */
pfac_status pfac_trie_bytes(const pfac_trie *t, pfac_bytes_kind kind, uint64_t *out_bytes);

pfac_status pfac_trie_stats(const pfac_trie *t, pfac_stats *out);

/* The serialised device image (host memory owned by t, valid until pfac_free).
 * This is what a multi-GPU driver broadcasts (NCCL) before pfac_attach. */
pfac_status pfac_image(const pfac_trie *t, const void **host_bytes, uint64_t *size);

/* Creates a handle from an image produced by pfac_image, which may live in
 * host memory or in device memory of `device` (detected with
 * cudaPointerGetAttributes).  The image is copied; it is validated (magic,
 * version, section bounds) and INVALID_ARG is returned for a bad image. */
pfac_status pfac_attach(const void *image, uint64_t size, int device, pfac_trie **out);

/* ------------------------------------------------------------ match, host */

/* Matches `text` (HOST memory, len bytes) on the current CUDA device and
 * returns the sorted (pos, pid) rows in host memory.  Synchronous.
 * The text streams through the device in chunks (the host/device
 * transition of PAPER.md:99 and the "first memory transfer" of PAPER.md:76):
 * chunk i (PFAC_STREAM_CHUNK starts + the (max_len - 1)-byte halo of
 * PAPER.md:66) is copied host->device on a copy stream while chunk i-1 is
 * scanned on a compute stream (three device text buffers), so the scan hides
 * behind the copy.  Page-locked `text` (cudaHostAlloc / registered memory) is
 * copied directly; pageable text goes through the handle's pinned staging
 * buffers (a host memcpy per chunk, overlapped with the device work).  Per-
 * chunk results concatenate in chunk order (start ranges are disjoint and
 * ordered).  len == 0 gives count 0.  Returns CUDA on any device failure. */
#define PFAC_STREAM_CHUNK (64ull << 20)
pfac_status pfac_match(const pfac_trie *t, const uint8_t *text, uint64_t len, pfac_matches *out);

void pfac_matches_free(pfac_matches *m);

/* --------------------------------------------------------- match, device */

/* Workspace bytes pfac_match_device needs for n_starts start positions: a
 * small fixed header, 12 B per 1024-start round, and the per-warp hit lists
 * (sized for one hit per four starts, at most ~256 MiB; a warp that finds
 * more re-scans its rounds, so the result never depends on this size). */
pfac_status pfac_workspace_bytes(const pfac_trie *t, uint64_t n_starts, uint64_t *out);

/* Stream-ordered scan on `device` (which must be the current device), all
 * pointers device memory:
 *   d_text[0 .. readable_len)   text; bytes [n_starts, readable_len) are the
 *                               read-only halo (a shard's successor bytes):
 *                               readable, never a start.  n_starts <= readable_len.
 *   result: { (pos_base + i, k) : i < n_starts, i + |P_k| <= readable_len,
 *             T[i .. i+|P_k|) == P_k } sorted by (pos, pid), written to
 *             d_pos[0..min(count, capacity)) / d_pid[...]; *d_count (u64,
 *             device) always receives the true count.  If count > capacity
 *             nothing past capacity is written: re-run with larger buffers.
 *   d_workspace: >= pfac_workspace_bytes(t, n_starts) bytes, 256-B aligned,
 *             ZERO-FILLED BEFORE ITS FIRST USE; the kernels leave it ready for
 *             the next call (its grid barrier resets itself in device memory,
 *             so the call may be captured in a CUDA graph and replayed).  One
 *             workspace must not be used by two calls that can run
 *             concurrently.
 * `device` must be the calling thread's current CUDA device (INVALID_ARG
 * otherwise).  No host synchronisation inside; kernel faults surface at the
 * caller's next sync.  Launch errors return PFAC_ERR_CUDA.  The device copy of
 * the trie is uploaded on first use per device (synchronously, once). */
pfac_status pfac_match_device(const pfac_trie *t, int device, const uint8_t *d_text,
                              uint64_t readable_len, uint64_t n_starts, uint64_t pos_base,
                              uint64_t *d_pos, uint32_t *d_pid, uint64_t capacity,
                              uint64_t *d_count, void *d_workspace, uint64_t workspace_bytes,
                              pfac_stream stream);

/* pfac_match_device with a scan plan (NULL = automatic, identical to
 * pfac_match_device).  Results do not depend on the plan; only speed does.
 * INVALID_ARG for a bad struct_bytes, a non-zero reserved field or an
 * out-of-range value; LIMIT if the requested plan does not fit shared memory. */
pfac_status pfac_match_device_ex(const pfac_trie *t, int device, const uint8_t *d_text,
                                 uint64_t readable_len, uint64_t n_starts, uint64_t pos_base,
                                 uint64_t *d_pos, uint32_t *d_pid, uint64_t capacity,
                                 uint64_t *d_count, void *d_workspace, uint64_t workspace_bytes,
                                 const pfac_plan_options *opt, pfac_stream stream);

/* The plan a scan of n_starts starts on `device` would use (no launch). */
pfac_status pfac_plan_query(const pfac_trie *t, int device, uint64_t n_starts,
                            const pfac_plan_options *opt, pfac_plan_info *out);

/* Number of kernel launches one pfac_match_device call makes (for the bench's
 * gpu_launches count). */
uint32_t pfac_launches_per_call(void);

/* ------------------------------------------------------------------ misc */
const char *pfac_status_string(pfac_status s);
const char *pfac_last_error(void);
/* Version string, e.g. "pfac-b200 0.1 sm_100a". */
const char *pfac_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PFAC_H */

// image.h -- layout of the PFAC device image (internal to the product library).
//
// One contiguous blob, built on the host by builder.cpp, copied verbatim to
// every device (and broadcast between GPUs by the multi-GPU driver).  All
// sections are 256-byte aligned offsets from the image start.
//
//   node   u32[N+1]   CSR row pointer of the breadth-first row-major trie
//                     (PAPER.md:80 steps I-II; CRS row_ptr):
//                     bits 0..29 = index of the node's first outgoing edge,
//                     bit 31 = "a pattern ends at this node", bit 30 = "tail
//                     start" (below this node the trie is a single path whose
//                     only terminal is its last node; see tails).  Children of a
//                     node are consecutive and in ascending byte order, so the
//                     child reached through edge e is node e+1 (implicit
//                     col_ind: the BFS numbering makes it redundant).
//   aux    u32[N]     at align256(off_node + 4(N+1)) (no header field): per
//                     node, its record index if it is a tail/chain start, else
//                     its labels packed little-endian if it has 1..4 children
//                     (its first four if it has 5..8), else 0.  Read next to the node word, it saves the walk a
//                     dependent label (or rank) load per level.
//   label  u8[E]      edge labels (CRS val, one byte per edge).
//   rec    uint4[N]   per node {node[v], node[v+1], aux[v], x}: the words a
//                     walk level needs, in one 16-byte load (for the nodes
//                     not staged in shared memory); x = labels 4..7 of a node
//                     with 5..8 children (its aux holds labels 0..3), else 0.
//                     (v20)
//   term_node u32[TK] ascending ids of the terminal nodes kept in the image
//                     (terminal indices 0..TK-1); terminal indices TK..T-1 are
//                     the ends of the compressed tails, in tail order.
//   term_rk uint2[ceil(N/32)] {bits, rank} per 32 nodes: bit v & 31 = node v
//                     has the terminal bit; rank = kept terminals before node
//                     32 * (v / 32).  A kept terminal's index = rank + popc(bits
//                     below v): one 8-byte load instead of a binary search of
//                     term_node (dense-match texts end most walks on one; v22).
//   out_ptr u32[T+1]  offsets into out_pid, by terminal index.
//   out_pid u32[..]   per terminal t, the ascending union of the pattern ids
//                     ending on the root->t path.  A walk passes every ancestor
//                     of the deepest node it reaches, so the matches of one
//                     start position are exactly this list for the deepest
//                     terminal passed (prefix closure).
//   root   u32[256]   child of the root per byte (0 = none): level 1 direct.
//   tail_bits u32[ceil(N/32)], tail_rank u32[ceil(N/32)]  bit v = node v is a
//                     tail or chain start (node word bit 30); rank =
//                     tail_rank[v/32] + popc(bits below v) = its record.
//   tails  uint4[n_tails]  records {offset into tail_bytes, path length L,
//                     terminal index t, chain end node x}:
//                     * tail (x = 0): below a tail start the uncompressed trie
//                       is a single path whose only terminal is its end; those
//                       nodes are not in the image, and a walk at a tail start
//                       compares the next L text bytes with tail_bytes[offset,
//                       offset+L) in one go (match -> terminal t).
//                     * chain (t = 0xFFFFFFFF, L >= 2): below a chain start the
//                       trie is a single path of L edges through non-terminal
//                       one-child nodes down to node x (terminal, branching or
//                       a leaf); the path's inner nodes are not in the image.
//                       A walk compares the L bytes and continues at x (depth
//                       + L).  The chain start keeps one CSR edge (to x) so
//                       the BFS numbering of the compressed tree keeps the
//                       implicit child rule.
//                     * verify leaf (t = kVerify; truncated tries only,
//                       PAPER.md:80 step III at depth d): a depth-d node whose
//                       subtree is not in the image; x = its first candidate
//                       record, L = their count.  Candidate records follow
//                       the n_tails node records (n_cand of them): {bytes
//                       offset, length L, terminal index t, 0} = a distinct
//                       pattern below the leaf (its bytes past depth d, the
//                       terminal of its end node), longest first.  A walk at
//                       a verify leaf returns the terminal of the first
//                       candidate whose bytes the text matches, else its
//                       deepest terminal passed.
//   tail_bytes u8[..] the labels of each tail path, concatenated (each tail
//                     starts 4-byte aligned; 4 zero bytes of slack at the end).
//   level1 u32[B][10] the root's children (nodes 1..B) as the paper's bitmapped
//                     nodes (Fig. 3): 8 words = 256-bit child
//                     bitmap, 2 words = per-word prefix popcounts (one byte
//                     each); child(c) = first_edge + prefix + rank + 1.
//   filter u32[2^F/32] first-stage filter over the first d bytes of every
//                     pattern (d = min(4, shortest pattern)); a start whose bit
//                     is clear cannot match.  Two kinds:
//                       kind 0 (d < 4): bit index filter_index(x) of the d-gram
//                         x (little-endian), standard bit order;
//                       kind 1 (d = 4): a blocked three-bit filter in
//                         32-bit words.  Word w = (hi32(x * kFilterMul) &
//                         mask) / 4, mask = (filter bytes - 1) & ~3 (a hash
//                         of all four bytes); the key sets bits 31-(byte3 &
//                         31), 31-(byte2 & 31) and 31-(byte1 & 31) of word w
//                         (bit-reversed so the kernel tests each with one
//                         rotate by the byte; scan.cu stage 1).  A start
//                         passes iff the three bits are set.
//                       kind 2 (d = 4, small sets): the pair filter.  Starts k
//                         and k+1 share bytes k+1..k+3, so one 32-bit word
//                         b = filter_pair_word(bytes k+1..k+3) answers both:
//                         start k passes iff bit 31-(byte k & 31) of word b is
//                         set, start k+1 iff bit 31-(byte k+4 & 31) is set.
//                         A pattern 4-gram P sets bit 31-(P[0]&31) of word
//                         filter_pair_word(P[1..3]) and bit 31-(P[3]&31) of
//                         word filter_pair_word(P[0..2]).  Half the bytes per
//                         start of kind 1 at the same fill for 2 bits per key.
//                       kind 3 (d = 16, DNA: every pattern byte in {A,C,G,T}
//                         and the shortest pattern >= 16): a blocked three-bit
//                         filter in 32-bit words over the 2-bit codes of the
//                         first 16 bytes, key = sum code(byte i) << 2i with
//                         code(b) = (b>>1)&3 (A 0, C 1, T 2, G 3; any other
//                         byte aliases, which can only add false positives).
//                         Word = (hi32(key * kFilterMul) & mask) / 4 as kind 1;
//                         bits 31-((key >> s) & 31) for s = 0, 16, 26 (bases
//                         0-2, 8-10, 13-15: the kernel rotates by the keys of
//                         starts k, k+8, k+13, whose low bits these are; v21).
//   pair   u32[256][8]  the 2-gram prefix table: word (b0, q) bit j set iff
//                     the walk from a start with bytes (b0, 32q + j) gets past
//                     level 1, or b0's level-1 node already is a terminal or a
//                     tail/chain start (then every b1 is set).  Derived from
//                     root + level1; the kernel tests survivors with it.
//   kset   u32[2^kset_log2]  (filter kind 1) the exact set of the patterns'
//                     filter keys (first 4 bytes little-endian) in buckets
//                     of 4 slots (16 bytes, one load): a key lives in the
//                     first bucket from its home bucket (key * kFilterMul)
//                     >> (32 - (kset_log2 - 2)) with a free slot (linear
//                     probing over buckets); empty slots hold kset_empty (a
//                     value that is no key); load <= 1/4.  A probe reads
//                     buckets from home until it finds the key (present) or
//                     an empty slot (absent).  A start whose key is absent
//                     cannot match: the walk is skipped (the filter's false
//                     positives).
//   dag_* (built with merge_suffixes; PAPER.md:80 steps IV-V "similar
//                     suffixes are merged", "end nodes merged") the minimal
//                     DAG of the untruncated trie: identical sub-tries
//                     (terminal flag, labels, child classes) are one node, so
//                     every leaf is one node (end-node merging) and equal
//                     suffix paths are shared.  Pattern identity survives by
//                     path rank: each node counts the distinct pattern
//                     strings of its sub-DAG, and a walk that adds
//                     dag_skip[e] (the node's own terminal + the counts of
//                     its earlier children) at every edge e reaches a
//                     terminal with the lexicographic rank r of the string it
//                     spelled; rank_term[r] = that string's terminal index
//                     (its pid list).  dag_node u32[ND+1] (first edge |
//                     terminal bit), dag_label u8[ED] (ascending per node),
//                     dag_child u32[ED], dag_skip u32[ED], rank_term u32[T].
//   pipe_*: byte accounting only, the paper's own pipeline:
//                     the trie truncated at pipe_depth levels, its identical
//                     sub-tries merged by terminal flag and shape alone (no
//                     pattern identity: the paper's terminals carry none),
//                     then its N x 9 CRS (2 nnz + n + 1 words).
//   entry  u32[2^entry_log2][4]  (filter kinds 4 and 3; D = the filter gram:
//                     8 bytes, or 16 DNA bases; every pattern has >= D bytes)
//                     the entry table: one entry {x0, x1, node, depth} per
//                     distinct D-byte pattern prefix (kind 4: x0 = bytes 0..3,
//                     x1 = bytes 4..7, little-endian; kind 3: x0 = the 16-base
//                     DNA key, x1 = 0); node = the deepest image node on the
//                     prefix's path at depth <= D (a node inside a tail or
//                     chain record is not in the image: its record's start
//                     is), depth = its depth.  Open addressing, slot =
//                     entry_slot(x0, x1), linear probing, empty slots hold
//                     node = kNone, load <= 1/2.  A start whose D bytes are
//                     absent (kind 3: or not all A/C/G/T, which the key
//                     aliases) cannot match; else the walk from (node, depth)
//                     equals the walk from the root, as no
//                     pattern ends above depth D.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define PFAC_HD __host__ __device__
#else
#define PFAC_HD
#endif

namespace pfac {

constexpr uint32_t kVersion = 22;
constexpr uint32_t kTermBit = 0x80000000u;
constexpr uint32_t kTailBit = 0x40000000u;
constexpr uint32_t kEdgeMask = 0x3FFFFFFFu;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kVerify = 0xFFFFFFFEu;     // record kind: a verify leaf (truncated trie)
constexpr uint32_t kFilterMul = 0x9E3779B1u;  // Fibonacci hashing multiplier (odd)
constexpr uint32_t kFilterMul2 = 0x85EBCA6Bu; // second multiplier (kinds 3, 4)
constexpr uint32_t kFilterMul3 = 0xC2B2AE35u; // third multiplier (kind 3 bit index)
constexpr uint32_t kDnaGram = 16;             // kind 3: bases per key
constexpr uint32_t kGram8 = 8;                // kind 4: bytes per key

struct ImageHeader {
    char magic[8];  // "PFACIMG1"
    uint32_t version;
    uint32_t header_bytes;
    uint64_t image_bytes;
    uint64_t n_nodes, n_edges, n_terminals, n_out;
    uint32_t n_patterns, max_len, min_len, filter_gram;
    uint32_t filter_log2_bits, filter_exact, filter_mul, filter_kind;
    uint64_t off_node, off_label, off_term_node, off_out_ptr, off_out_pid, off_root, off_filter;
    uint64_t bytes_uncompressed, bytes_dense_stt, bytes_paper_crs, bytes_csr_core;
    uint64_t n_tails, n_tail_bytes, off_tail_bits, off_tail_rank, off_tails, off_tail_bytes;
    uint64_t n_level1, off_level1;
    uint64_t n_kept_terminals, n_nodes_full;
    uint64_t off_kset;                 // exact key set (0: none), see below
    uint32_t kset_log2, kset_empty;    // log2 of its slots; the empty-slot marker
    uint64_t off_pair;                 // 2-gram prefix table u32[256][8]
    uint64_t off_entry;                // entry table (0: none), see above
    uint32_t entry_log2, entry_pad;  // log2 of its slots; 0
    uint64_t n_cand;                   // verify candidate records (after the n_tails node records)
    uint32_t trunc_depth, trunc_pad;   // PAPER.md:80 step III depth d (0: untruncated); 0
    uint64_t bytes_truncated;          // 36 B x nodes of depth <= d (the paper's truncated trie)
    // steps IV-V merged DAG, id-preserving (0 sections: not built; see dag_* below)
    uint64_t n_dag_nodes, n_dag_edges, off_dag_node, off_dag_label, off_dag_child, off_dag_skip, off_rank_term;
    uint64_t bytes_merged, bytes_merged_crs;               // 36 B x DAG nodes; its N x 9 CRS words x 4
    uint64_t pipe_depth, bytes_pipe_trunc, bytes_pipe_merged, bytes_pipe_crs;  // the paper's pipeline (below)
    uint64_t off_rec;                  // node records uint4[N] (below)
    uint64_t off_term_rk;              // kept-terminal rank uint2[ceil(N/32)] (below; v22)
    uint8_t pad[512 - 256 - 64 - 120];
};
static_assert(sizeof(ImageHeader) == 512, "header must be 512 bytes");

// Home bucket (4 slots) of a key in the exact key set of 2^log2 slots.
PFAC_HD inline uint32_t kset_bucket(uint32_t key, uint32_t log2) { return (key * kFilterMul) >> (34u - log2); }
// First slot of a key (x0, x1) in the entry table.
PFAC_HD inline uint32_t entry_slot(uint32_t x0, uint32_t x1, uint32_t log2) {
    return (x0 * kFilterMul + x1 * kFilterMul2) >> (32u - log2);
}
// Offset of the aux section (it follows the node section).
PFAC_HD inline uint64_t aux_offset(uint64_t off_node, uint64_t n_nodes) {
    return (off_node + 4 * (n_nodes + 1) + 255) / 256 * 256;
}
// Kind 4: block of the 8-byte key (x0 = bytes 0..3, x1 = bytes 4..7).
PFAC_HD inline uint32_t gram8_block(uint32_t x0, uint32_t x1, uint32_t log2_bits) {
    return (x0 * kFilterMul + x1 * kFilterMul2) >> (32u - (log2_bits - 6u));
}
// Kind 0: filter bit index of a little-endian packed d-gram key (d < 4).
PFAC_HD inline uint32_t filter_index(uint32_t key, uint32_t log2_bits, uint32_t exact) {
    return exact ? key : (key * kFilterMul) >> (32u - log2_bits);
}
// Kind 1 (d = 4): byte offset of the 4-gram x's word in a filter of
// 2^log2_bits bits (hi32(x * M) & mask), and its three bit positions.
PFAC_HD inline uint32_t filter4_offset(uint32_t x, uint32_t log2_bits) {
    return (uint32_t)(((uint64_t)x * kFilterMul) >> 32) & (((1u << (log2_bits - 3u)) - 1u) & ~3u);
}
PFAC_HD inline uint32_t filter4_bit(uint32_t x, uint32_t byte) { return 31u - ((x >> (8u * byte)) & 31u); }
// Kind 2 (d = 4): word index of the three shared bytes x (low 24 bits used).
PFAC_HD inline uint32_t filter_pair_word(uint32_t x, uint32_t log2_bits) {
    return (x * (kFilterMul << 8)) >> (32u - (log2_bits - 5u));
}
// Kind 3 (DNA): 2-bit code of a byte, key of 16 bytes, block and bit positions.
PFAC_HD inline uint32_t dna_code(uint32_t b) { return (b >> 1) & 3u; }
PFAC_HD inline uint32_t dna_bit(uint32_t key, uint32_t shift) { return 31u - ((key >> shift) & 31u); }

}  // namespace pfac

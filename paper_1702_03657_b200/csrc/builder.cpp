// builder.cpp -- host trie builder: patterns -> breadth-first CSR device image.
//
// PAPER.md:80 step I ("constructed in a breadth-first approach, level by
// level") and step II ("stored in a row major ordered array"), then the CRS
// step of PAPER.md:89/:101 in label form (see image.h).  Steps III-V
// (truncation, suffix/end-node merging) are NOT applied: the scan must report
// exact (position, pattern-id) rows, which a truncated or merged trie cannot
// (they are §8(f) NEXT-1/2).
//
// Construction: sort the pattern ids lexicographically (ties by id); every
// trie node is then a contiguous range of that order sharing a prefix of
// length `depth`.  Expanding ranges in FIFO order numbers the nodes in BFS
// order with children in ascending byte order -- exactly the row-major layout
// whose child through edge e is node e+1.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "image.h"
#include "internal.h"

namespace pfac {

namespace {

struct Range {
    uint32_t lo, hi;    // [lo, hi) of the sorted order
    uint32_t depth;     // prefix length shared by the range
    uint32_t anc_term;  // index of the nearest terminal ancestor (kNone = none)
};

inline uint64_t align256(uint64_t x) { return (x + 255) & ~uint64_t(255); }

inline uint64_t mix64(uint64_t x) {  // splitmix64 finaliser (hashing sub-trie signatures)
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Steps IV-V of PAPER.md:80 over the BFS trie (node_word: first edge |
// terminal bit; the child through edge e is node e+1; depth per node):
// classes of identical sub-tries of the trie cut at depth dlim (a node at
// depth dlim counts as a leaf: "end nodes merged"), by terminal flag,
// labels and child classes, bottom-up (children have larger BFS ids).
// Returns the number of classes; cls[v] = class of node v (kNone: deeper
// than dlim).  Hash table of (signature hash, representative node);
// equality is checked against the representative, so no signature is stored.
uint32_t merge_classes(const std::vector<uint32_t> &node_word, const std::vector<uint8_t> &label,
                       const std::vector<uint32_t> &depth, uint32_t dlim, std::vector<uint32_t> &cls) {
    const uint64_t N = depth.size();
    cls.assign(N, kNone);
    auto term = [&](uint64_t v) { return (node_word[v] & kTermBit) != 0; };
    auto e0 = [&](uint64_t v) { return node_word[v] & kEdgeMask; };
    auto e1 = [&](uint64_t v) { return depth[v] >= dlim ? e0(v) : (node_word[v + 1] & kEdgeMask); };
    uint64_t cap = 64;
    while (cap < 2 * N) cap <<= 1;
    std::vector<uint64_t> slot_h(cap, 0);
    std::vector<uint32_t> slot_rep(cap, kNone);
    uint32_t n_cls = 0;
    for (uint64_t v = N; v-- > 0;) {
        if (depth[v] > dlim) continue;
        uint64_t h = mix64(term(v) ? 0x51u : 0x17u);
        for (uint32_t e = e0(v); e < e1(v); e++) h = mix64(h ^ ((uint64_t)label[e] << 32 | cls[e + 1]));
        uint64_t i = h & (cap - 1);
        for (;; i = (i + 1) & (cap - 1)) {
            const uint32_t w = slot_rep[i];
            if (w == kNone) {
                slot_h[i] = h;
                slot_rep[i] = (uint32_t)v;
                cls[v] = n_cls++;
                break;
            }
            if (slot_h[i] != h || term(w) != term(v) || e1(w) - e0(w) != e1(v) - e0(v)) continue;
            bool same = true;
            for (uint32_t k = 0; same && k < e1(v) - e0(v); k++)
                same = label[e0(v) + k] == label[e0(w) + k] && cls[e0(v) + k + 1] == cls[e0(w) + k + 1];
            if (same) {
                cls[v] = cls[w];
                break;
            }
        }
    }
    return n_cls;
}

// Paper CRS element count (P:101 N x 9 matrix: per node its non-zero bitmap
// words + the offset column when it has children) of the nodes `reps` (one
// per class) of a trie cut at dlim.
uint64_t crs_nnz(const std::vector<uint32_t> &node_word, const std::vector<uint8_t> &label,
                 const std::vector<uint32_t> &depth, uint32_t dlim, const std::vector<uint32_t> &reps) {
    uint64_t nnz = 0;
    for (uint32_t v : reps) {
        const uint32_t a = node_word[v] & kEdgeMask, b = depth[v] >= dlim ? a : (node_word[v + 1] & kEdgeMask);
        int last = -1;
        if (b > a) nnz++;
        for (uint32_t e = a; e < b; e++)
            if ((int)(label[e] >> 5) != last) {
                nnz++;
                last = label[e] >> 5;
            }
    }
    return nnz;
}

}  // namespace

int build_image(const uint8_t *const *pats, const uint32_t *lens, uint32_t m, const BuildOpts &opt,
                std::vector<uint8_t> &image, std::string &err) {
    if (!pats || !lens || m == 0) {
        err = "pfac_build: NULL argument or n_patterns == 0";
        return kStatusInvalid;
    }
    uint32_t max_len = 0, min_len = kNone;
    for (uint32_t k = 0; k < m; k++) {
        if (lens[k] == 0 || lens[k] > kMaxPatternLen) {
            err = "pfac_build: pattern " + std::to_string(k) + " has length " + std::to_string(lens[k]) +
                  " (must be 1.." + std::to_string(kMaxPatternLen) + ")";
            return kStatusInvalid;
        }
        if (!pats[k]) {
            err = "pfac_build: pattern pointer " + std::to_string(k) + " is NULL";
            return kStatusInvalid;
        }
        max_len = std::max(max_len, lens[k]);
        min_len = std::min(min_len, lens[k]);
    }

    // ---- sort ids lexicographically (a proper prefix sorts first), ties by id
    std::vector<uint32_t> ord(m);
    std::iota(ord.begin(), ord.end(), 0u);
    std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) {
        uint32_t l = std::min(lens[a], lens[b]);
        int c = std::memcmp(pats[a], pats[b], l);
        if (c != 0) return c < 0;
        if (lens[a] != lens[b]) return lens[a] < lens[b];
        return a < b;
    });

    // ---- step I/II: FIFO expansion of ranges == BFS numbering
    std::vector<uint32_t> node_word;   // row_ptr | terminal bit, per node
    std::vector<uint8_t> label;        // label of edge e (child e+1)
    std::vector<uint32_t> term_node, out_ptr{0}, out_pid;
    uint64_t paper_nnz = 0;

    std::vector<Range> q;
    q.reserve(1024);
    q.push_back({0, m, 0, kNone});
    std::vector<uint32_t> own;
    std::vector<uint32_t> parent{0}, own_pid;  // per node: parent; a pattern ending here (kNone if none)
    std::vector<uint32_t> end_at(m, kNone);    // per sorted index: the node its pattern ends at
    for (size_t head = 0; head < q.size(); head++) {
        if (q.size() > (size_t)kEdgeMask) {
            err = "pfac_build: trie exceeds 2^30-1 nodes";
            return kStatusLimit;
        }
        const Range r = q[head];
        uint32_t v = (uint32_t)head;
        // patterns ending exactly here sort first in the range
        uint32_t lo = r.lo;
        own.clear();
        while (lo < r.hi && lens[ord[lo]] == r.depth) {
            end_at[lo] = v;
            own.push_back(ord[lo++]);
        }
        uint32_t anc = r.anc_term;
        bool terminal = !own.empty();
        own_pid.push_back(terminal ? own[0] : kNone);
        // row_ptr[v] = number of nodes numbered before v's first child, minus the root
        uint32_t first_edge = (uint32_t)(q.size() - 1);
        node_word.push_back(first_edge | (terminal ? kTermBit : 0u));
        if (terminal) {
            // union list = (ancestor's union) merged with own ids (both ascending)
            std::sort(own.begin(), own.end());
            // budget checked before anything is copied: nested pattern sets
            // grow these lists quadratically
            const uint64_t n_anc = anc != kNone ? out_ptr[anc + 1] - out_ptr[anc] : 0;
            if ((uint64_t)out_pid.size() + n_anc + own.size() > kMaxPidEntries) {
                err = "pfac_build: pattern-id lists exceed 2^28 entries (deeply nested pattern set)";
                return kStatusLimit;
            }
            const size_t at = out_pid.size();
            out_pid.resize(at + n_anc + own.size());
            if (n_anc)  // the ancestor's list (ascending) merged with own ids (ascending)
                std::merge(out_pid.begin() + out_ptr[anc], out_pid.begin() + out_ptr[anc + 1], own.begin(), own.end(),
                           out_pid.begin() + at);
            else
                std::copy(own.begin(), own.end(), out_pid.begin() + at);
            term_node.push_back(v);
            out_ptr.push_back((uint32_t)out_pid.size());
            anc = (uint32_t)(term_node.size() - 1);
        }
        // children: partition [lo, hi) by the byte at position depth
        int last_word = -1;
        uint32_t i = lo;
        if (i < r.hi) paper_nnz += 1;  // the non-zero offset column (P:101 matrix view)
        while (i < r.hi) {
            uint8_t c = pats[ord[i]][r.depth];
            uint32_t j = i + 1;
            while (j < r.hi && pats[ord[j]][r.depth] == c) j++;
            label.push_back(c);
            if ((int)(c >> 5) != last_word) {  // distinct non-zero bitmap word
                paper_nnz += 1;
                last_word = c >> 5;
            }
            q.push_back({i, j, r.depth + 1, anc});
            parent.push_back(v);
            i = j;
        }
    }
    const uint64_t N = q.size(), E = N - 1, T = term_node.size();
    node_word.push_back((uint32_t)E);  // row_ptr[N]
    auto nchild = [&](uint64_t v) { return (node_word[v + 1] & kEdgeMask) - (node_word[v] & kEdgeMask); };

    // ---- step III ("the trie is truncated at the appropriate
    // level"; opt.truncate_depth = d > 0): nodes deeper than d leave the
    // image; a depth-d node with children becomes a verify leaf whose record
    // lists the distinct patterns below it (their bytes past depth d, longest
    // first, each with the terminal index of its end node).  A walk that
    // reaches a verify leaf compares those bytes with the text; the longest
    // candidate that matches gives the start's pid list (it holds every
    // pattern on its root path, PAPER.md:76 continued past depth d), else the
    // deepest terminal already passed does: results stay exact.
    const uint32_t d_trunc = opt.truncate_depth;
    std::vector<uint8_t> cut(N, 0), verify(N, 0);
    uint64_t n_trunc_nodes = N;  // nodes of the truncated (uncompressed) trie
    if (d_trunc) {
        n_trunc_nodes = 0;
        for (uint64_t v = 0; v < N; v++) {
            if (q[v].depth > d_trunc) cut[v] = 1;
            else n_trunc_nodes++;
            if (q[v].depth == d_trunc && nchild(v) > 0) verify[v] = 1;
        }
    }

    // ---- path compression of the non-branching deep part.  A node whose
    // strict descendants form a single path with one terminal, at its end, is
    // a "tail start" (topmost such node, path >= 2 bytes).  Its descendants are
    // removed from the image; the tail start becomes a leaf carrying the
    // path's bytes and the terminal index of its end, so a walk compares the
    // rest of the path in one go.  Walk results are unchanged (the removed
    // nodes have no branching and no other terminal).
    std::vector<uint8_t> chain_ok(N, 0);
    std::vector<uint32_t> chain_end(N, kNone);
    for (uint64_t v = N; v-- > 0;) {
        if (nchild(v) != 1 || verify[v] || cut[v]) continue;  // (a verify leaf ends no tail)
        const uint32_t u = (node_word[v] & kEdgeMask) + 1;
        const bool term_u = (node_word[u] & kTermBit) != 0;
        if (nchild(u) == 0 && term_u) {
            chain_ok[v] = 1;
            chain_end[v] = u;
        } else if (nchild(u) == 1 && !term_u && chain_ok[u]) {
            chain_ok[v] = 1;
            chain_end[v] = chain_end[u];
        }
    }
    std::vector<uint8_t> is_tail(N, 0), removed(N, 0);
    for (uint64_t v = 1; v < N; v++)
        if (!cut[v] && chain_ok[v] && !chain_ok[parent[v]] && q[chain_end[v]].depth - q[v].depth >= 2) is_tail[v] = 1;
    for (uint64_t v = 1; v < N; v++) removed[v] = cut[v] || removed[parent[v]] || is_tail[parent[v]];
    // ---- internal chains: a kept node v (not the root) whose single child u
    // is non-terminal with a single child starts a chain: the nodes below v
    // down to the first node x that is terminal, branching, a leaf or a tail
    // start are removed, and v carries the chain's bytes and x (a walk
    // compares the bytes in one go and continues at x; no terminal is skipped).
    auto first_child = [&](uint64_t v) { return (uint64_t)(node_word[v] & kEdgeMask) + 1; };
    auto is_term = [&](uint64_t v) { return (node_word[v] & kTermBit) != 0; };
    std::vector<uint32_t> chain_to(N, kNone);
    for (uint64_t v = 1; v < N; v++) {
        if (removed[v] || is_tail[v] || verify[v] || nchild(v) != 1) continue;
        uint64_t x = first_child(v);
        if (is_term(x) || nchild(x) != 1 || is_tail[x] || verify[x]) continue;
        while (!is_term(x) && nchild(x) == 1 && !is_tail[x] && !verify[x]) {
            removed[x] = 1;
            x = first_child(x);
        }
        chain_to[v] = (uint32_t)x;
    }
    std::vector<uint32_t> old_ti(N, kNone);
    for (uint64_t t = 0; t < T; t++) old_ti[term_node[t]] = (uint32_t)t;
    // BFS numbering of the compressed tree (a chain start's one child is its
    // chain's end), so that the child through edge e is still node e+1
    std::vector<uint32_t> order;  // old ids in new order
    order.reserve(N);
    order.push_back(0);
    for (size_t h = 0; h < order.size(); h++) {
        const uint64_t v = order[h];
        if (is_tail[v] || verify[v]) continue;
        if (chain_to[v] != kNone) {
            order.push_back(chain_to[v]);
            continue;
        }
        for (uint32_t e = node_word[v] & kEdgeMask; e < (node_word[v + 1] & kEdgeMask); e++) order.push_back(e + 1);
    }
    const uint64_t NK = order.size();
    std::vector<uint32_t> new_id(N, kNone);
    for (uint64_t i = 0; i < NK; i++) new_id[order[i]] = (uint32_t)i;
    // entry-table candidates (image.h): per node at depth D (8: kind 4; 16:
    // kind 3), its key and the deepest kept node at depth <= D on its path
    std::vector<uint32_t> e8, e16;  // {x0, x1, node, depth} per distinct D-byte prefix
    for (uint64_t u = 1; u < N; u++) {
        const uint32_t du = q[u].depth;
        if (!((du == kGram8 && min_len >= kGram8) || (du == kDnaGram && min_len >= kDnaGram))) continue;
        const uint8_t *pt = pats[ord[q[u].lo]];
        uint64_t a = u;
        while (removed[a]) a = parent[a];
        std::vector<uint32_t> &ev = du == kGram8 ? e8 : e16;
        if (du == kGram8) {
            ev.push_back((uint32_t)pt[0] | (uint32_t)pt[1] << 8 | (uint32_t)pt[2] << 16 | (uint32_t)pt[3] << 24);
            ev.push_back((uint32_t)pt[4] | (uint32_t)pt[5] << 8 | (uint32_t)pt[6] << 16 | (uint32_t)pt[7] << 24);
        } else {  // the 16-base DNA key (only used when every pattern byte is A, C, G or T)
            uint32_t key = 0;
            for (uint32_t b = 0; b < kDnaGram; b++) key |= dna_code(pt[b]) << (2 * b);
            ev.push_back(key);
            ev.push_back(0u);
        }
        ev.push_back(new_id[a]);
        ev.push_back(q[a].depth);
    }

    // compressed CSR (bit 30 marks a tail or chain start: its record holds the bytes)
    std::vector<uint32_t> cnode;
    std::vector<uint8_t> clabel;
    std::vector<uint32_t> nterm_old;  // old terminal index of each new terminal index
    std::vector<uint32_t> cterm_node;
    cnode.reserve(NK + 1);
    clabel.reserve(NK);
    for (uint64_t i = 0; i < NK; i++) {
        const uint64_t v = order[i];
        const bool term = is_term(v);
        const bool rec = is_tail[v] || chain_to[v] != kNone || verify[v];
        cnode.push_back((uint32_t)clabel.size() | (term ? kTermBit : 0u) | (rec ? kTailBit : 0u));
        if (term) {
            nterm_old.push_back(old_ti[v]);
            cterm_node.push_back((uint32_t)i);
        }
        if (chain_to[v] != kNone) {
            clabel.push_back(label[node_word[v] & kEdgeMask]);  // the chain's first byte (CSR shape only)
        } else if (!is_tail[v] && !verify[v]) {
            for (uint32_t e = node_word[v] & kEdgeMask; e < (node_word[v + 1] & kEdgeMask); e++) clabel.push_back(label[e]);
        }
    }
    cnode.push_back((uint32_t)clabel.size());
    const uint64_t TK = cterm_node.size();  // kept terminals: indices [0, TK), sorted by node id
    std::vector<uint32_t> tail_bits((NK + 31) / 32, 0u), tail_rank((NK + 31) / 32, 0u);
    // 4 words per record: bytes offset, length, terminal index (tail) or kNone
    // (chain), chain end node (chain) or 0 (tail)
    std::vector<uint32_t> tails;
    std::vector<uint8_t> tail_bytes;
    std::vector<uint32_t> cands;  // verify candidates: records appended after the node records
    std::vector<std::pair<uint32_t, uint32_t>> fix;  // (verify record, its first candidate) to patch
    for (uint64_t i = 0; i < NK; i++) {
        const uint64_t v = order[i];
        if (verify[v]) {
            // candidates: the distinct patterns below v (their end nodes), longest first
            std::vector<uint32_t> ends;
            for (uint32_t j = q[v].lo; j < q[v].hi; j++)
                if (end_at[j] != kNone && end_at[j] != v && (ends.empty() || ends.back() != end_at[j]))
                    ends.push_back(end_at[j]);
            std::stable_sort(ends.begin(), ends.end(), [&](uint32_t x, uint32_t y) { return q[x].depth > q[y].depth; });
            fix.push_back({(uint32_t)(tails.size() / 4), (uint32_t)(cands.size() / 4)});
            tails.push_back(0u);  // first candidate (patched below)
            tails.push_back((uint32_t)ends.size());
            tails.push_back(kVerify);
            tails.push_back(0u);
            for (uint32_t u : ends) {
                const uint32_t k = ord[q[u].lo];  // a pattern ending at u
                cands.push_back((uint32_t)tail_bytes.size());
                cands.push_back(q[u].depth - d_trunc);
                cands.push_back((uint32_t)nterm_old.size());
                cands.push_back(0u);
                nterm_old.push_back(old_ti[u]);
                tail_bytes.insert(tail_bytes.end(), pats[k] + d_trunc, pats[k] + q[u].depth);
                while (tail_bytes.size() & 3) tail_bytes.push_back(0);
            }
            tail_bits[i >> 5] |= 1u << (i & 31);
            continue;
        }
        if (!is_tail[v] && chain_to[v] == kNone) continue;
        const uint32_t end = is_tail[v] ? chain_end[v] : chain_to[v];
        const uint32_t dv = q[v].depth, de = q[end].depth;
        const uint32_t k = ord[q[end].lo];  // a pattern through `end`
        tails.push_back((uint32_t)tail_bytes.size());  // 4-byte aligned
        tails.push_back(de - dv);
        if (is_tail[v]) {
            tails.push_back((uint32_t)nterm_old.size());
            tails.push_back(0u);
            nterm_old.push_back(old_ti[end]);
        } else {
            tails.push_back(kNone);
            tails.push_back(new_id[end]);
        }
        tail_bytes.insert(tail_bytes.end(), pats[k] + dv, pats[k] + de);
        while (tail_bytes.size() & 3) tail_bytes.push_back(0);
        tail_bits[i >> 5] |= 1u << (i & 31);
    }
    {
        uint32_t acc = 0;
        for (size_t w = 0; w < tail_bits.size(); w++) {
            tail_rank[w] = acc;
            acc += (uint32_t)__builtin_popcount(tail_bits[w]);
        }
    }
    const uint64_t NT = tails.size() / 4;  // node records; the candidates follow them
    const uint64_t NC = cands.size() / 4;
    for (auto &f : fix) tails[4 * f.first] = (uint32_t)NT + f.second;
    tails.insert(tails.end(), cands.begin(), cands.end());
    tail_bytes.insert(tail_bytes.end(), 4, 0);  // slack for 4-byte reads
    // pid lists in the new terminal order
    std::vector<uint32_t> cout_ptr{0}, cout_pid;
    cout_pid.reserve(out_pid.size());
    for (uint32_t ot : nterm_old) {
        cout_pid.insert(cout_pid.end(), out_pid.begin() + out_ptr[ot], out_pid.begin() + out_ptr[ot + 1]);
        cout_ptr.push_back((uint32_t)cout_pid.size());
    }
    // ---- steps IV-V: suffix and end-node merging
    std::vector<uint32_t> depth_of(N);
    for (uint64_t v = 0; v < N; v++) depth_of[v] = q[v].depth;
    std::vector<uint32_t> dag_node, dag_child, dag_skip, rank_term;
    std::vector<uint8_t> dag_label;
    uint64_t ND = 0, ED = 0, bytes_merged = 0, bytes_merged_crs = 0;
    uint64_t pipe_depth = 0, bytes_pipe_trunc = 0, bytes_pipe_merged = 0, bytes_pipe_crs = 0;
    if (opt.merge_suffixes) {
        // (a) the paper's pipeline, byte accounting only: cut at 8 levels
        // or the requested depth, merged without pattern identity
        pipe_depth = d_trunc ? d_trunc : 8u;
        std::vector<uint32_t> pcls;
        const uint32_t npc = merge_classes(node_word, label, depth_of, (uint32_t)pipe_depth, pcls);
        std::vector<uint32_t> preps(npc, kNone);
        uint64_t n_pt = 0;
        for (uint64_t v = 0; v < N; v++)
            if (pcls[v] != kNone) {
                n_pt++;
                if (preps[pcls[v]] == kNone) preps[pcls[v]] = (uint32_t)v;
            }
        bytes_pipe_trunc = 36 * n_pt;
        bytes_pipe_merged = 36ull * npc;
        bytes_pipe_crs = 4 * (2 * crs_nnz(node_word, label, depth_of, (uint32_t)pipe_depth, preps) + npc + 1);
        // (b) the id-preserving minimal DAG of the untruncated trie (scannable)
        std::vector<uint32_t> cls;
        const uint32_t nc = merge_classes(node_word, label, depth_of, kNone, cls);
        std::vector<uint32_t> rep(nc, kNone);
        for (uint64_t v = 0; v < N; v++)
            if (rep[cls[v]] == kNone) rep[cls[v]] = (uint32_t)v;
        // strings below each node (its own terminal + its children's), bottom-up
        std::vector<uint32_t> cnt(N, 0);
        for (uint64_t v = N; v-- > 0;) {
            uint64_t c = (node_word[v] & kTermBit) ? 1 : 0;
            for (uint32_t e = node_word[v] & kEdgeMask; e < (node_word[v + 1] & kEdgeMask); e++) c += cnt[e + 1];
            cnt[v] = (uint32_t)c;
        }
        // DAG nodes numbered breadth-first from the root's class
        std::vector<uint32_t> dnum(nc, kNone), dorder;
        dorder.push_back(cls[0]);
        dnum[cls[0]] = 0;
        for (size_t hq = 0; hq < dorder.size(); hq++) {
            const uint32_t v = rep[dorder[hq]];
            for (uint32_t e = node_word[v] & kEdgeMask; e < (node_word[v + 1] & kEdgeMask); e++) {
                const uint32_t cc = cls[e + 1];
                if (dnum[cc] == kNone) {
                    dnum[cc] = (uint32_t)dorder.size();
                    dorder.push_back(cc);
                }
            }
        }
        for (uint32_t c : dorder) {
            const uint32_t v = rep[c];
            const uint32_t t = (node_word[v] & kTermBit) ? 1u : 0u;
            dag_node.push_back((uint32_t)dag_label.size() | (t ? kTermBit : 0u));
            uint32_t acc = t;
            for (uint32_t e = node_word[v] & kEdgeMask; e < (node_word[v + 1] & kEdgeMask); e++) {
                dag_label.push_back(label[e]);
                dag_child.push_back(dnum[cls[e + 1]]);
                dag_skip.push_back(acc);
                acc += cnt[e + 1];
            }
        }
        ND = dorder.size();
        ED = dag_label.size();
        dag_node.push_back((uint32_t)ED);
        if (ND > kEdgeMask || ED > kEdgeMask) {
            err = "pfac_build: merged DAG exceeds 2^30-1 nodes or edges";
            return kStatusLimit;
        }
        // rank r = the r-th distinct pattern string (sorted order) -> its terminal index
        std::vector<uint32_t> new_ti(T, kNone);
        for (uint32_t i = 0; i < nterm_old.size(); i++) new_ti[nterm_old[i]] = i;
        for (uint32_t j = 0; j < m; j++)
            if (end_at[j] != kNone && (j == 0 || end_at[j - 1] != end_at[j])) rank_term.push_back(new_ti[old_ti[end_at[j]]]);
        bytes_merged = 36 * ND;
        std::vector<uint32_t> reps_all(rep.begin(), rep.end());
        bytes_merged_crs = 4 * (2 * crs_nnz(node_word, label, depth_of, kNone, reps_all) + ND + 1);
    }

    const uint64_t N_full = N;
    node_word.swap(cnode);
    label.swap(clabel);
    term_node.swap(cterm_node);
    out_ptr.swap(cout_ptr);
    out_pid.swap(cout_pid);
    const uint64_t NI = NK, EI = NK - 1;  // image nodes / edges

    // ---- aux word per node (one load next to the node word, no dependent
    // label or rank loads): record index of a tail/chain start; the labels of
    // a node with 1..4 children (the first four of 5..8), packed little-endian;
    // 0 otherwise
    std::vector<uint32_t> aux(NI, 0u);
    {
        uint32_t rank = 0;
        for (uint64_t v = 0; v < NI; v++) {
            const uint32_t e0 = node_word[v] & kEdgeMask, e1 = node_word[v + 1] & kEdgeMask;
            if (node_word[v] & kTailBit) {
                aux[v] = rank++;
            } else if (e1 - e0 >= 1 && e1 - e0 <= 8) {  // (5..8 children: the first four; the
                uint32_t x = 0;                              //  node record holds the rest)
                for (uint32_t e = e0; e < e0 + 4 && e < e1; e++) x |= (uint32_t)label[e] << (8 * (e - e0));
                aux[v] = x;
            }
        }
    }

    // ---- level 1 as bitmapped nodes (Fig. 3)
    const uint32_t B = node_word[1] & kEdgeMask;  // root's children are nodes 1..B
    std::vector<uint32_t> level1((size_t)B * 10, 0u);
    for (uint32_t v = 1; v <= B; v++) {
        uint32_t *o = &level1[(size_t)(v - 1) * 10];
        for (uint32_t e = node_word[v] & kEdgeMask; e < (node_word[v + 1] & kEdgeMask); e++)
            o[label[e] >> 5] |= 1u << (label[e] & 31);
        uint32_t pre = 0;
        for (int w = 0; w < 8; w++) {
            o[8 + w / 4] |= pre << (8 * (w % 4));
            pre += (uint32_t)__builtin_popcount(o[w]);
        }
    }

    // ---- derived tables: level-1 direct table and first-stage d-gram filter
    std::vector<uint32_t> root(256, 0);
    {
        uint32_t s = node_word[0] & kEdgeMask, e = node_word[1] & kEdgeMask;
        for (uint32_t k = s; k < e; k++) root[label[k]] = k + 1;
    }
    // DNA pattern sets (every byte in {A,C,G,T}, shortest >= 16): kind 3
    bool dna = min_len >= kDnaGram;
    for (uint32_t k = 0; dna && k < m; k++)
        for (uint32_t b = 0; dna && b < lens[k]; b++) {
            const uint8_t c = pats[k][b];
            dna = c == 'A' || c == 'C' || c == 'G' || c == 'T';
        }
    if (opt.filter_kind >= 0 && opt.filter_kind != 3) dna = false;  // a forced kind (tools, tests)
    if (opt.filter_kind == 3 && !dna) {
        err = "pfac_build: filter kind 3 needs an all-A/C/G/T pattern set with shortest >= 16";
        return kStatusInvalid;
    }
    // 8-byte prefixes (kind 4) for big sets whose patterns are all >= 8 bytes:
    // text that shares 4-byte prefixes with many patterns (tokens, protocol
    // words) is filtered at 8 bytes
    bool g8 = false;
    if (!dna && min_len >= kGram8) {
        std::vector<uint64_t> k8(m);
        for (uint32_t k = 0; k < m; k++) {
            uint64_t x = 0;
            for (uint32_t b = 0; b < kGram8; b++) x |= (uint64_t)pats[k][b] << (8 * b);
            k8[k] = x;
        }
        std::sort(k8.begin(), k8.end());
        g8 = (uint64_t)(std::unique(k8.begin(), k8.end()) - k8.begin()) > 2048;
    }
    if (opt.filter_kind == 4) {
        if (dna || min_len < kGram8) {
            err = "pfac_build: filter kind 4 needs shortest pattern >= 8 (and not kind 3)";
            return kStatusInvalid;
        }
        g8 = true;
    } else if (opt.filter_kind >= 0) {
        g8 = false;
    }
    if ((opt.filter_kind == 1 || opt.filter_kind == 2) && (dna || g8 || min_len < 4)) {
        err = "pfac_build: filter kinds 1 and 2 need shortest pattern >= 4";
        return kStatusInvalid;
    }
    if (opt.filter_kind == 0 && min_len >= 4) {
        err = "pfac_build: filter kind 0 is for sets whose shortest pattern is < 4 bytes";
        return kStatusInvalid;
    }
    const uint32_t gram = dna ? kDnaGram : g8 ? kGram8 : std::min<uint32_t>(4, min_len);
    uint32_t exact = gram <= 2 ? 1u : 0u;
    uint32_t log2_bits;
    uint32_t kind = dna ? 3u : g8 ? 4u : gram == 4 ? 1u : 0u;
    auto dna_key = [&](const uint8_t *pt) {
        uint32_t key = 0;
        for (uint32_t b = 0; b < kDnaGram; b++) key |= dna_code(pt[b]) << (2 * b);
        return key;
    };
    if (g8) {
        std::vector<uint64_t> k8(m);
        for (uint32_t k = 0; k < m; k++) {
            uint64_t x = 0;
            for (uint32_t b = 0; b < kGram8; b++) x |= (uint64_t)pats[k][b] << (8 * b);
            k8[k] = x;
        }
        std::sort(k8.begin(), k8.end());
        const uint64_t distinct = std::unique(k8.begin(), k8.end()) - k8.begin();
        const uint64_t per_key = opt.gram8_bits_per_key;  // ~32 bits per key, at most 2^20 bits (128 KiB)
        log2_bits = 10;
        while (log2_bits < 20 && (1ull << log2_bits) < per_key * distinct) log2_bits++;
    } else if (dna) {
        std::vector<uint32_t> keys(m);
        for (uint32_t k = 0; k < m; k++) keys[k] = dna_key(pats[k]);
        std::sort(keys.begin(), keys.end());
        const uint64_t distinct = std::unique(keys.begin(), keys.end()) - keys.begin();
        log2_bits = 10;  // ~32 bits per key (two of them set per key), at most 2^20 bits (128 KiB)
        while (log2_bits < 20 && (1ull << log2_bits) < 32 * distinct) log2_bits++;
    } else if (exact) {
        log2_bits = 8 * gram;
    } else {
        std::vector<uint32_t> keys(m);
        for (uint32_t k = 0; k < m; k++) {
            uint32_t x = 0;
            for (uint32_t b = 0; b < gram; b++) x |= (uint32_t)pats[k][b] << (8 * b);
            keys[k] = x;
        }
        std::sort(keys.begin(), keys.end());
        const uint64_t distinct = std::unique(keys.begin(), keys.end()) - keys.begin();
        // kind 2 (pair filter, d = 4): one bit per key and role, 2 bits set
        // per 4-gram (sizing below), for sets of <= 2,048 distinct 4-grams.
        // Else kind 1 (blocked two-bit, ~32 bits per key) or kind 0 (d < 4),
        // capped at 2^20 bits (kind 1, 128 KiB) or 2^19 bits (kind 0).
        const bool allow2 = opt.filter_kind != 1;
        if (kind == 1 && (opt.filter_kind == 2 || (allow2 && distinct * 128 <= (1ull << 18)))) {
            kind = 2;
            log2_bits = 12;
            // 512 filter bits per distinct 4-gram (two set: fill ~0.4%), at
            // most 2^19 bits (64 KiB, one copy).  Measured on C2 (tools/ab.py):
            // 128 bits/key with 4 bank-spread copies 54.1 us, 256 with 2
            // copies 51.3, 512 with 1 copy 47.6, 1024 (128 KiB: 2-slot ring,
            // trie no longer whole in shared memory) 51.0: fewer survivors
            // beat fewer bank conflicts.
            const uint64_t per_key = opt.pair_bits_per_key;
            while ((1ull << log2_bits) < per_key * distinct && log2_bits < 19) log2_bits++;
        } else {
            log2_bits = 10;  // at most 2^20 bits (128 KiB; the kernel then keeps 2 text rounds per warp)
            while (log2_bits < (kind == 1 ? 20u : 19u) && (1ull << log2_bits) < 32 * distinct) log2_bits++;
        }
    }
    std::vector<uint32_t> filter((size_t)1 << (log2_bits - 5 > 0 ? log2_bits - 5 : 0), 0u);
    if (filter.empty()) filter.resize(1);
    for (uint32_t k = 0; k < m; k++) {
        uint32_t x = 0;
        for (uint32_t b = 0; b < gram; b++) x |= (uint32_t)pats[k][b] << (8 * b);
        if (kind == 4) {
            const uint32_t x0 = (uint32_t)pats[k][0] | (uint32_t)pats[k][1] << 8 | (uint32_t)pats[k][2] << 16 |
                                (uint32_t)pats[k][3] << 24;
            const uint32_t x1 = (uint32_t)pats[k][4] | (uint32_t)pats[k][5] << 8 | (uint32_t)pats[k][6] << 16 |
                                (uint32_t)pats[k][7] << 24;
            const uint32_t b = gram8_block(x0, x1, log2_bits);
            filter[2 * b] |= 1u << (31u - (x0 & 31u));
            filter[2 * b + 1] |= 1u << (31u - (x1 & 31u));
        } else if (kind == 3) {
            const uint32_t key = dna_key(pats[k]);
            filter[filter4_offset(key, log2_bits) / 4] |=
                (1u << dna_bit(key, 0)) | (1u << dna_bit(key, 16)) | (1u << dna_bit(key, 26));
        } else if (kind == 2) {
            // as the first start of a pair: shared bytes are P[1..3], own byte P[0];
            // as the second start: shared bytes are P[0..2], own byte P[3]
            filter[filter_pair_word(x >> 8, log2_bits)] |= 1u << (31u - (x & 31u));
            filter[filter_pair_word(x, log2_bits)] |= 1u << (31u - ((x >> 24) & 31u));
        } else if (kind == 1) {
            uint32_t &w = filter[filter4_offset(x, log2_bits) / 4];
            w |= (1u << filter4_bit(x, 3)) | (1u << filter4_bit(x, 2)) | (1u << filter4_bit(x, 1));
        } else {
            uint32_t h = filter_index(x, log2_bits, exact);
            filter[h >> 5] |= 1u << (h & 31);
        }
    }

    // ---- exact key set (kinds 1, 3: large sets): the distinct filter keys of
    // the patterns (kind 2 sets are small and their tries fit shared memory,
    // where a walk is cheaper than a probe)
    std::vector<uint32_t> kset;
    uint32_t kset_log2 = 0, kset_empty = 0;
    if (kind == 1) {  // (kind 3 enters through the entry table instead)
        std::vector<uint32_t> keys(m);
        for (uint32_t k = 0; k < m; k++) {
            if (kind == 3) {
                keys[k] = dna_key(pats[k]);
            } else {
                keys[k] = (uint32_t)pats[k][0] | (uint32_t)pats[k][1] << 8 | (uint32_t)pats[k][2] << 16 |
                          (uint32_t)pats[k][3] << 24;
            }
        }
        std::sort(keys.begin(), keys.end());
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
        for (uint32_t x : keys) {  // smallest value that is not a key
            if (x != kset_empty) break;
            kset_empty++;
        }
        kset_log2 = 6;  // load <= 1/4: a probe almost always reads one 16-byte bucket
        while ((1ull << kset_log2) < 4ull * keys.size()) kset_log2++;
        kset.assign((size_t)1 << kset_log2, kset_empty);
        const uint32_t bmask = (1u << (kset_log2 - 2)) - 1u;
        for (uint32_t x : keys) {
            for (uint32_t b = kset_bucket(x, kset_log2);; b = (b + 1) & bmask) {
                uint32_t j = 0;
                while (j < 4 && kset[4 * b + j] != kset_empty) j++;
                if (j < 4) {
                    kset[4 * b + j] = x;
                    break;
                }
            }
        }
    }

    // ---- entry table (kinds 3 and 4; image.h)
    std::vector<uint32_t> entry;
    uint32_t entry_log2 = 0;
    if (kind == 3) e8.swap(e16);
    if (kind == 4 || kind == 3) {
        const uint64_t ne = e8.size() / 4;
        entry_log2 = 4;
        while ((1ull << entry_log2) < 2 * ne) entry_log2++;
        if (entry_log2 > 30) {
            err = "pfac_build: too many entry-table keys";
            return kStatusLimit;
        }
        entry.assign((size_t)4 << entry_log2, 0u);
        for (size_t i = 0; i < ((size_t)1 << entry_log2); i++) entry[4 * i + 2] = kNone;
        const uint32_t mask = (1u << entry_log2) - 1u;
        for (uint64_t k = 0; k < ne; k++) {
            uint32_t i = entry_slot(e8[4 * k], e8[4 * k + 1], entry_log2);
            while (entry[4 * i + 2] != kNone) i = (i + 1) & mask;
            std::memcpy(&entry[4 * i], &e8[4 * k], 16);
        }
    }

    // ---- assemble the image
    ImageHeader h;
    std::memset(&h, 0, sizeof h);
    std::memcpy(h.magic, "PFACIMG1", 8);
    h.version = kVersion;
    h.header_bytes = sizeof(ImageHeader);
    h.n_nodes = NI;
    h.n_edges = EI;
    h.n_terminals = T;
    h.n_kept_terminals = TK;
    h.n_nodes_full = N_full;
    h.n_out = out_pid.size();
    h.n_patterns = m;
    h.max_len = max_len;
    h.min_len = min_len;
    h.filter_gram = gram;
    h.filter_log2_bits = log2_bits;
    h.filter_exact = exact;
    h.filter_mul = kFilterMul;
    h.filter_kind = kind;
    uint64_t o = align256(sizeof(ImageHeader));
    h.off_node = o;      o = align256(o + 4 * (NI + 1));
    const uint64_t off_aux = aux_offset(h.off_node, NI);  o = align256(off_aux + 4 * NI);  // aux u32[N] (image.h)
    h.off_label = o;     o = align256(o + EI + 16);
    h.off_term_node = o; o = align256(o + 4 * TK);
    h.off_out_ptr = o;   o = align256(o + 4 * (T + 1));
    h.off_out_pid = o;   o = align256(o + 4 * out_pid.size());
    h.off_root = o;      o = align256(o + 4 * 256);
    h.off_filter = o;    o = align256(o + 4 * filter.size());
    h.off_tail_bits = o; o = align256(o + 4 * tail_bits.size());
    h.off_tail_rank = o; o = align256(o + 4 * tail_rank.size());
    h.off_tails = o;     o = align256(o + 16 * (NT + NC));
    h.off_tail_bytes = o; o = align256(o + tail_bytes.size() + 16);
    h.off_level1 = o;    o = align256(o + 40ull * B);
    h.off_pair = o;      o = align256(o + 8192);
    h.off_kset = kset.empty() ? 0 : o;
    o = align256(o + 4 * kset.size());
    h.kset_log2 = kset_log2;
    h.kset_empty = kset_empty;
    h.off_entry = entry.empty() ? 0 : o;
    o = align256(o + 4 * entry.size());
    if (ND) {  // merged DAG sections (steps IV-V)
        h.off_dag_node = o;  o = align256(o + 4 * (ND + 1));
        h.off_dag_label = o; o = align256(o + ED + 16);
        h.off_dag_child = o; o = align256(o + 4 * ED);
        h.off_dag_skip = o;  o = align256(o + 4 * ED);
        h.off_rank_term = o; o = align256(o + 4 * rank_term.size());
    }
    h.off_rec = o;  o = align256(o + 16 * NI);  // node records (image.h)
    h.off_term_rk = o;  o = align256(o + 8 * ((NI + 31) / 32));  // kept-terminal rank (image.h, v22)
    h.n_dag_nodes = ND;
    h.n_dag_edges = ED;
    h.bytes_merged = bytes_merged;
    h.bytes_merged_crs = bytes_merged_crs;
    h.pipe_depth = pipe_depth;
    h.bytes_pipe_trunc = bytes_pipe_trunc;
    h.bytes_pipe_merged = bytes_pipe_merged;
    h.bytes_pipe_crs = bytes_pipe_crs;
    h.entry_log2 = entry_log2;
    h.n_level1 = B;
    h.n_tails = NT;
    h.n_cand = NC;
    h.trunc_depth = d_trunc;
    h.bytes_truncated = 36 * n_trunc_nodes;              // PAPER.md:80 step III, 134
    h.n_tail_bytes = tail_bytes.size();
    h.image_bytes = o;
    h.bytes_uncompressed = 36 * N_full;
    h.bytes_dense_stt = 1024 * N_full;                       // 256 x u32 per state
    h.bytes_paper_crs = 4 * (2 * paper_nnz + N_full + 1);    // PAPER.md:101, N x 9 words
    h.bytes_csr_core = 4 * (NI + 1) + EI + 16 * (NT + NC) + (tail_bytes.size() - 4);  // CSR + records + bytes

    try {
        image.assign(o, 0);
    } catch (...) {
        err = "pfac_build: out of host memory for the image";
        return kStatusNomem;
    }
    uint8_t *p = image.data();
    std::memcpy(p, &h, sizeof h);
    std::memcpy(p + h.off_node, node_word.data(), 4 * (NI + 1));
    std::memcpy(p + off_aux, aux.data(), 4 * NI);
    if (EI) std::memcpy(p + h.off_label, label.data(), EI);
    if (TK) std::memcpy(p + h.off_term_node, term_node.data(), 4 * TK);
    std::memcpy(p + h.off_out_ptr, out_ptr.data(), 4 * (T + 1));
    if (!out_pid.empty()) std::memcpy(p + h.off_out_pid, out_pid.data(), 4 * out_pid.size());
    std::memcpy(p + h.off_root, root.data(), 4 * 256);
    std::memcpy(p + h.off_filter, filter.data(), 4 * filter.size());
    std::memcpy(p + h.off_tail_bits, tail_bits.data(), 4 * tail_bits.size());
    std::memcpy(p + h.off_tail_rank, tail_rank.data(), 4 * tail_rank.size());
    if (NT + NC) std::memcpy(p + h.off_tails, tails.data(), 16 * (NT + NC));
    if (!tail_bytes.empty()) std::memcpy(p + h.off_tail_bytes, tail_bytes.data(), tail_bytes.size());
    std::memcpy(p + h.off_level1, level1.data(), 40ull * B);
    {   // 2-gram prefix table (image.h)
        uint32_t *pair = reinterpret_cast<uint32_t *>(p + h.off_pair);
        for (uint32_t j = 0; j < 2048; j++) {
            const uint32_t v = root[j >> 3];
            uint32_t wd = 0;
            if (v != 0)
                wd = (node_word[v] & (kTermBit | kTailBit)) ? 0xFFFFFFFFu : level1[(size_t)(v - 1) * 10 + (j & 7)];
            pair[j] = wd;
        }
    }
    if (!kset.empty()) std::memcpy(p + h.off_kset, kset.data(), 4 * kset.size());
    {   // kept-terminal rank {bits, rank} per 32 nodes
        uint32_t *rk = reinterpret_cast<uint32_t *>(p + h.off_term_rk);
        uint32_t acc = 0;
        for (uint64_t w = 0; w < (NI + 31) / 32; w++) {
            uint32_t bits = 0;
            for (uint64_t b = 0; b < 32 && 32 * w + b < NI; b++) bits |= ((node_word[32 * w + b] >> 31) & 1u) << b;
            rk[2 * w] = bits;
            rk[2 * w + 1] = acc;
            acc += (uint32_t)__builtin_popcount(bits);
        }
    }
    {   // node records {node[v], node[v+1], aux[v], 0}
        uint32_t *rec = reinterpret_cast<uint32_t *>(p + h.off_rec);
        for (uint64_t v = 0; v < NI; v++) {
            rec[4 * v] = node_word[v];
            rec[4 * v + 1] = node_word[v + 1];
            rec[4 * v + 2] = aux[v];
            uint32_t x = 0;  // labels 4..7 of a node with 5..8 children
            const uint32_t e0 = node_word[v] & kEdgeMask, e1 = node_word[v + 1] & kEdgeMask;
            if (!(node_word[v] & kTailBit) && e1 - e0 >= 5 && e1 - e0 <= 8)
                for (uint32_t e = e0 + 4; e < e1; e++) x |= (uint32_t)label[e] << (8 * (e - e0 - 4));
            rec[4 * v + 3] = x;
        }
    }
    if (!entry.empty()) std::memcpy(p + h.off_entry, entry.data(), 4 * entry.size());
    if (ND) {
        std::memcpy(p + h.off_dag_node, dag_node.data(), 4 * (ND + 1));
        if (ED) {
            std::memcpy(p + h.off_dag_label, dag_label.data(), ED);
            std::memcpy(p + h.off_dag_child, dag_child.data(), 4 * ED);
            std::memcpy(p + h.off_dag_skip, dag_skip.data(), 4 * ED);
        }
        std::memcpy(p + h.off_rank_term, rank_term.data(), 4 * rank_term.size());
    }
    return kStatusOk;
}

int validate_image(const uint8_t *p, uint64_t size, std::string &err) {
    if (!p || size < sizeof(ImageHeader)) {
        err = "pfac_attach: image too small";
        return kStatusInvalid;
    }
    ImageHeader h;
    std::memcpy(&h, p, sizeof h);
    if (std::memcmp(h.magic, "PFACIMG1", 8) != 0 || h.version != kVersion ||
        h.header_bytes != sizeof(ImageHeader) || h.image_bytes != size) {
        err = "pfac_attach: bad magic/version/size";
        return kStatusInvalid;
    }
    const uint64_t N = h.n_nodes, E = h.n_edges, T = h.n_terminals;
    auto in = [&](uint64_t off, uint64_t bytes) { return off >= sizeof(ImageHeader) && off + bytes <= size; };
    const uint64_t off_aux = aux_offset(h.off_node, N);  // image.h: aux follows node
    bool ok = N >= 2 && E == N - 1 && N <= kEdgeMask && in(h.off_node, 4 * (N + 1)) && in(h.off_label, E + 4) &&
              in(off_aux, 4 * N) && off_aux + 4 * N <= h.off_label && in(h.off_pair, 8192) &&
              (h.off_kset == 0 ? h.kset_log2 == 0
                               : (h.filter_kind == 1 && h.kset_log2 >= 6 &&
                                  h.kset_log2 <= 30 && in(h.off_kset, 4ull << h.kset_log2))) &&
              (h.off_entry == 0 ? h.entry_log2 == 0
                                 : ((h.filter_kind == 4 || h.filter_kind == 3) && h.entry_log2 >= 4 &&
                                    h.entry_log2 <= 30 &&
                                    in(h.off_entry, 16ull << h.entry_log2))) &&
              h.n_kept_terminals <= T && h.n_kept_terminals + h.n_tails + h.n_cand >= T && h.n_nodes_full >= N &&
              in(h.off_term_node, 4 * h.n_kept_terminals) && in(h.off_out_ptr, 4 * (T + 1)) && in(h.off_out_pid, 4 * h.n_out) &&
              in(h.off_root, 1024) && h.filter_log2_bits >= 5 && h.filter_log2_bits <= 24 &&
              in(h.off_filter, (1ull << h.filter_log2_bits) / 8) && h.filter_gram >= 1 &&
              (h.filter_gram <= 4 || (h.filter_kind == 3 && h.filter_gram == kDnaGram) ||
               (h.filter_kind == 4 && h.filter_gram == kGram8)) &&
              h.filter_gram <= h.min_len && h.min_len <= h.max_len && h.max_len <= kMaxPatternLen &&
              h.filter_mul == kFilterMul && (h.filter_gram == kDnaGram ? h.filter_kind == 3
               : h.filter_gram == kGram8 ? h.filter_kind == 4
               : h.filter_gram == 4 ? (h.filter_kind == 1 || h.filter_kind == 2) : h.filter_kind == 0) &&
              (h.filter_kind == 0 || h.filter_log2_bits >= 10) && in(h.off_tail_bits, 4 * ((N + 31) / 32)) &&
              in(h.off_tail_rank, 4 * ((N + 31) / 32)) && in(h.off_tails, 16 * (h.n_tails + h.n_cand)) &&
              (h.n_cand == 0 || h.trunc_depth > 0) && h.trunc_pad == 0 &&
              in(h.off_tail_bytes, h.n_tail_bytes) && in(h.off_level1, 40 * h.n_level1);
    if (ok) {
        const uint32_t *node = reinterpret_cast<const uint32_t *>(p + h.off_node);
        const uint32_t *out_ptr = reinterpret_cast<const uint32_t *>(p + h.off_out_ptr);
        ok = (node[0] & kEdgeMask) == 0 && (node[N] & kEdgeMask) == E && out_ptr[0] == 0 && out_ptr[T] == h.n_out &&
             h.n_level1 == (node[1] & kEdgeMask) && h.n_level1 >= 1 && h.n_level1 <= 256;
        for (uint64_t v = 0; ok && v < N; v++) ok = (node[v] & kEdgeMask) <= (node[v + 1] & kEdgeMask);
        const uint32_t *tails = reinterpret_cast<const uint32_t *>(p + h.off_tails);
        // records: tail (ends at a terminal), chain (at a node), verify leaf
        // (a range of candidate records, each ending at a terminal)
        uint64_t n_tail_ends = 0;
        for (uint64_t i = 0; ok && i < h.n_tails + h.n_cand; i++) {
            const uint32_t *r = tails + 4 * i;
            const bool cand = i >= h.n_tails, chain = !cand && r[2] == kNone, ver = !cand && r[2] == kVerify;
            if (ver) {
                ok = r[0] >= h.n_tails && r[1] >= 1 && (uint64_t)r[0] + r[1] <= h.n_tails + h.n_cand && r[3] == 0;
                continue;
            }
            ok = (uint64_t)r[0] + r[1] <= h.n_tail_bytes &&
                 (chain ? (!cand && r[3] > 0 && r[3] < N && r[1] >= 2)
                        : (r[2] >= h.n_kept_terminals && r[2] < T && r[3] == 0 && (!cand || r[1] >= 1)));
            n_tail_ends += !chain;
        }
        ok = ok && h.n_kept_terminals + n_tail_ends == T;
        const uint32_t *en = reinterpret_cast<const uint32_t *>(p + h.off_entry);  // entries: a node, depth <= D
        for (uint64_t i = 0; ok && h.off_entry && i < (1ull << h.entry_log2); i++)
            ok = en[4 * i + 2] == kNone || (en[4 * i + 2] > 0 && en[4 * i + 2] < N && en[4 * i + 3] >= 1 &&
                                            en[4 * i + 3] <= h.filter_gram);
        // contents the kernel dereferences: every index it follows
        // must stay inside its section
        // records: 4-byte aligned bytes read a word at a time
        for (uint64_t i = 0; ok && i < h.n_tails + h.n_cand; i++)
            ok = (i < h.n_tails && tails[4 * i + 2] == kVerify) ||
                 ((tails[4 * i] & 3u) == 0 &&
                  (uint64_t)tails[4 * i] + ((tails[4 * i + 1] + 3ull) & ~3ull) <= h.n_tail_bytes);
        // root table: 0 or a level-1 node
        const uint32_t *root = reinterpret_cast<const uint32_t *>(p + h.off_root);
        for (uint32_t c = 0; ok && c < 256; c++) ok = root[c] <= h.n_level1;
        // level-1 bitmapped nodes: popcount = degree, prefix bytes = running popcounts
        const uint32_t *l1 = reinterpret_cast<const uint32_t *>(p + h.off_level1);
        for (uint64_t v = 1; ok && v <= h.n_level1; v++) {
            const uint32_t *o = l1 + 10 * (v - 1);
            uint32_t pre = 0;
            for (int w = 0; ok && w < 8; w++) {
                ok = ((o[8 + w / 4] >> (8 * (w % 4))) & 0xFFu) == pre;
                pre += (uint32_t)__builtin_popcount(o[w]);
            }
            const bool rec = (node[v] & kTailBit) != 0;
            ok = ok && (rec || pre == (node[v + 1] & kEdgeMask) - (node[v] & kEdgeMask));
        }
        // aux words: a record node's aux is its record index, in node order
        const uint32_t *aux = reinterpret_cast<const uint32_t *>(p + off_aux);
        uint64_t rank = 0;
        for (uint64_t v = 0; ok && v < N; v++)
            if (node[v] & kTailBit) ok = aux[v] == rank++;
        ok = ok && rank == h.n_tails;
        // record bitmap and its rank words (the host planner stages records by rank)
        const uint32_t *tb = reinterpret_cast<const uint32_t *>(p + h.off_tail_bits);
        const uint32_t *tr = reinterpret_cast<const uint32_t *>(p + h.off_tail_rank);
        uint32_t acc = 0;
        for (uint64_t w = 0; ok && w < (N + 31) / 32; w++) {
            uint32_t want = 0;
            for (uint64_t b = 0; b < 32 && 32 * w + b < N; b++) want |= ((node[32 * w + b] >> 30) & 1u) << b;
            ok = tb[w] == want && tr[w] == acc;
            acc += (uint32_t)__builtin_popcount(want);
        }
        // kept terminals: exactly the nodes with the terminal bit, ascending
        const uint32_t *tn = reinterpret_cast<const uint32_t *>(p + h.off_term_node);
        uint64_t k = 0;
        for (uint64_t v = 0; ok && v < N; v++)
            if (node[v] & kTermBit) ok = k < h.n_kept_terminals && tn[k++] == v;
        ok = ok && k == h.n_kept_terminals;
        // kept-terminal rank: the terminal bits and their prefix counts
        ok = ok && in(h.off_term_rk, 8 * ((N + 31) / 32));
        if (ok) {
            const uint32_t *rk = reinterpret_cast<const uint32_t *>(p + h.off_term_rk);
            uint32_t acc2 = 0;
            for (uint64_t w = 0; ok && w < (N + 31) / 32; w++) {
                uint32_t want = 0;
                for (uint64_t b = 0; b < 32 && 32 * w + b < N; b++) want |= ((node[32 * w + b] >> 31) & 1u) << b;
                ok = rk[2 * w] == want && rk[2 * w + 1] == acc2;
                acc2 += (uint32_t)__builtin_popcount(want);
            }
        }
        // node records: copies of the node and aux words
        ok = ok && in(h.off_rec, 16 * N);
        const uint32_t *rc = reinterpret_cast<const uint32_t *>(p + h.off_rec);
        for (uint64_t v = 0; ok && v < N; v++)
            ok = rc[4 * v] == node[v] && rc[4 * v + 1] == node[v + 1] && rc[4 * v + 2] == aux[v];
        // merged DAG (steps IV-V): CSR bounds, child ids, rank table
        if (ok && h.n_dag_nodes) {
            const uint64_t ND = h.n_dag_nodes, ED = h.n_dag_edges;
            ok = ND >= 1 && ND <= kEdgeMask && ED <= kEdgeMask && in(h.off_dag_node, 4 * (ND + 1)) &&
                 in(h.off_dag_label, ED + 16) && in(h.off_dag_child, 4 * ED) && in(h.off_dag_skip, 4 * ED) &&
                 in(h.off_rank_term, 4 * T);
            const uint32_t *dn = reinterpret_cast<const uint32_t *>(p + h.off_dag_node);
            const uint32_t *dc = reinterpret_cast<const uint32_t *>(p + h.off_dag_child);
            const uint32_t *rt = reinterpret_cast<const uint32_t *>(p + h.off_rank_term);
            ok = ok && (dn[0] & kEdgeMask) == 0 && (dn[ND] & kEdgeMask) == ED;
            for (uint64_t v = 0; ok && v < ND; v++) ok = (dn[v] & kEdgeMask) <= (dn[v + 1] & kEdgeMask);
            for (uint64_t e = 0; ok && e < ED; e++) ok = dc[e] < ND;
            for (uint64_t r = 0; ok && r < T; r++) ok = rt[r] < T;
        }
        // pid lists: monotone offsets, ids < n_patterns
        for (uint64_t i = 0; ok && i < T; i++) ok = out_ptr[i] <= out_ptr[i + 1];
        const uint32_t *pid = reinterpret_cast<const uint32_t *>(p + h.off_out_pid);
        for (uint64_t i = 0; ok && i < h.n_out; i++) ok = pid[i] < h.n_patterns;
    }
    if (!ok) {
        err = "pfac_attach: inconsistent image sections";
        return kStatusInvalid;
    }
    return kStatusOk;
}

}  // namespace pfac

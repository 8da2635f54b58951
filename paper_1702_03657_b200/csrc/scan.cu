// scan.cu -- sm_100a PFAC scan kernel (KB1): scan + deterministic compaction
// in one cooperative launch.
//
// PAPER.md:76 (§II-C): "Each thread is assigned to a single letter in the
// text T. If a match is recorded, the thread continues the matching process
// until a mismatch. When a mismatch occurs the thread is terminated. The
// algorithm also allows for coalesced memory access during the first memory
// transfer, and early thread termination."
//
// B200 mapping:
//  * one persistent CTA per SM (kWarps warps).  Shared memory holds, once per
//    SM, the first-stage d-gram filter (replicated per bank group so lanes
//    rarely conflict), the level-1 table, and the top H nodes of the
//    breadth-first CSR trie (BFS order = level order, so the first H nodes are
//    the hot upper levels; PAPER.md:89 kept row_ptr on chip for the same
//    reason).
//  * phase 1 (scan): warp w owns a contiguous range of 512-start rounds.  A
//    per-warp ring of kSlots 512-byte slots is filled by TMA bulk copies
//    (cp.async.bulk + mbarrier, evict-first in L2) kSlots-1 rounds ahead.
//    Per round each lane tests its 16 consecutive starts against the d-gram
//    filter (a clear bit means no pattern can start there: PFAC's early
//    termination taken before the first trie access); survivors walk the trie
//    to the first mismatch (shared memory for the top H nodes, L1/L2 below).
//    A start that passed a terminal is appended, in position order, to the
//    warp's hit list (its offset in the range; matches are rare, so phase 3
//    walks these starts again instead of storing the terminal).
//  * phase 2 (offsets): per-warp match counts -> CTA scan -> one grid barrier
//    -> exclusive prefix over CTA totals.  Ranges are contiguous and ordered,
//    so the concatenation is globally sorted by (pos, pid).
//  * phase 3 (emit): each warp expands its hit list into (pos, pid) rows.  A
//    warp whose list overflowed re-scans its range writing rows directly.
#include <cuda_runtime.h>

#include <cstdio>
#include <map>
#include <mutex>

#include "internal.h"

namespace pfac {

namespace {

constexpr int kWarps = 32;
constexpr int kThreads = kWarps * 32;
constexpr int kPerLane = 16;           // consecutive starts per lane per round
constexpr int kRound = 32 * kPerLane;  // 512 starts per warp round
constexpr int kSlots = 4;              // text ring depth per warp
constexpr int kSlotBytes = kRound;     // one round of text per slot
constexpr int kMaxCtas = 1024;

// Workspace: header (two grid-barrier counters, used alternately so that a
// launch clears the other one for the next launch) + CTA totals + hit lists.
struct WsHeader {
    unsigned int barrier[2];
    unsigned int pad[62];
};
static_assert(sizeof(WsHeader) == 256, "");
constexpr uint64_t kWsFixed = sizeof(WsHeader) + 8ull * kMaxCtas;

struct ScanArgs {
    DevTrie t;
    const uint8_t *text;
    uint64_t readable;
    uint64_t n_starts;
    uint64_t pos_base;
    uint64_t *out_pos;
    uint32_t *out_pid;
    uint64_t capacity;
    uint64_t *out_count;
    WsHeader *ws;
    unsigned long long *cta_total;  // [gridDim.x]
    uint32_t *hits;                 // [warps][hit_cap] start offsets within the warp's range
    uint32_t hit_cap;
    uint32_t parity;                // barrier counter used by this launch
    uint64_t rounds_per_warp;
    // shared-memory layout (bytes from the dynamic smem base)
    uint32_t filter_words;          // words of the (unreplicated) filter
    uint32_t filter_rep;            // replication factor (power of two <= 32)
    uint32_t off_filter, off_root, off_node, off_label, off_ring, off_bar, off_warp;
    uint32_t hot_nodes;             // H: node words [0, H] resident
    uint32_t hot_edges;             // row_ptr[H]: labels [0, hot_edges) resident
    uint32_t aligned;               // text pointer is 16-byte aligned (bulk-copy path)
};

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
// TMA bulk copy global -> shared, completion on an mbarrier; the text is
// streamed once, so it is marked evict-first in L2 (keeps the trie tail hot).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const unsigned int *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// One barrier across the (co-resident, cooperative-launch) grid.
__device__ __forceinline__ void grid_barrier(unsigned int *ctr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        while (ld_acquire_u32(ctr) < gridDim.x) __nanosleep(64);
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t x, int lane, uint32_t *total) {
    uint32_t incl = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    *total = __shfl_sync(0xffffffffu, incl, 31);
    return incl - x;
}

// ------------------------------------------------------------ trie access
struct Smem {
    const uint32_t *filter;  // replicated, already offset by this lane's copy
    const uint32_t *root;
    const uint32_t *node;    // [0, H]
    const uint8_t *label;    // [0, hot_edges)
};

__device__ __forceinline__ uint32_t node_word(const ScanArgs &a, const Smem &s, uint32_t v) {
    return v <= a.hot_nodes ? s.node[v] : __ldg(a.t.node + v);
}
__device__ __forceinline__ uint32_t label_at(const ScanArgs &a, const Smem &s, uint32_t e) {
    return e < a.hot_edges ? (uint32_t)s.label[e] : (uint32_t)__ldg(a.t.label + e);
}

// Text byte j: from the warp's ring when [lo, lo+len) covers it (slot0 then
// slot1, contiguous in the stream), else from global memory.
struct TextView {
    const uint8_t *slot0;
    const uint8_t *slot1;
    uint64_t lo;
    uint32_t len;
};
__device__ __forceinline__ uint32_t text_at(const ScanArgs &a, const TextView &tv, uint64_t j) {
    const uint64_t r = j - tv.lo;
    if (r < (uint64_t)tv.len) return r < (uint64_t)kSlotBytes ? tv.slot0[r] : tv.slot1[r - kSlotBytes];
    return __ldg(a.text + j);
}

// Walk from start gi (whose first byte is c0) to the first mismatch; returns
// the deepest terminal node passed, or kNone.
__device__ uint32_t walk(const ScanArgs &a, const Smem &s, const TextView &tv, uint64_t gi, uint32_t c0) {
    uint32_t v = s.root[c0];
    if (v == 0) return kNone;
    uint32_t w = node_word(a, s, v);
    uint32_t last = (w & kTermBit) ? v : kNone;
    for (uint64_t j = gi + 1; j < a.readable; ++j) {
        const uint32_t lo0 = w & kEdgeMask;
        const uint32_t hi0 = node_word(a, s, v + 1) & kEdgeMask;
        if (lo0 == hi0) break;  // leaf
        const uint32_t c = text_at(a, tv, j);
        uint32_t lo = lo0, hi = hi0;  // labels[lo, hi) ascending
        while (hi - lo > 4) {
            const uint32_t mid = (lo + hi) >> 1;
            if (label_at(a, s, mid) <= c) lo = mid; else hi = mid;
        }
        uint32_t found = kNone;
        for (uint32_t k = lo; k < hi; ++k) {
            const uint32_t l = label_at(a, s, k);
            if (l >= c) {
                if (l == c) found = k;
                break;
            }
        }
        if (found == kNone) break;  // mismatch: the thread terminates
        v = found + 1;              // BFS order: the child through edge e is node e+1
        w = node_word(a, s, v);
        if (w & kTermBit) last = v;
    }
    return last;
}

__device__ __forceinline__ uint32_t term_index(const DevTrie &t, uint32_t v) {
    uint32_t lo = 0, hi = t.n_terminals;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(t.term_node + mid) < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Stage 1 over one lane's 16 starts: bit k set <=> start lbase+k may match.
__device__ __forceinline__ uint32_t filter16(const ScanArgs &a, const Smem &s, const uint32_t wv[5], uint32_t kmask,
                                             uint32_t nvalid) {
    const uint32_t rep = a.filter_rep, log2_bits = a.t.log2_bits, exact = a.t.exact;
    uint32_t surv = 0;
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {
        const uint32_t x = __funnelshift_r(wv[k >> 2], wv[(k >> 2) + 1], 8 * (k & 3)) & kmask;
        const uint32_t h = filter_index(x, log2_bits, exact);
        const uint32_t word = s.filter[(h >> 5) * rep];
        surv |= ((word >> (h & 31)) & 1u) << k;
    }
    return surv & (nvalid >= 32 ? 0xFFFFFFFFu : ((1u << nvalid) - 1u));
}

__global__ void __launch_bounds__(kThreads, 1) pfac_scan_kernel(const ScanArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t *s_filter = reinterpret_cast<uint32_t *>(smem + a.off_filter);
    uint32_t *s_root = reinterpret_cast<uint32_t *>(smem + a.off_root);
    uint32_t *s_node = reinterpret_cast<uint32_t *>(smem + a.off_node);
    uint8_t *s_label = smem + a.off_label;
    uint8_t *ring = smem + a.off_ring + (uint32_t)warp * (kSlots * kSlotBytes);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + a.off_bar) + warp * kSlots;
    unsigned long long *s_wtot = reinterpret_cast<unsigned long long *>(smem + a.off_warp);  // [kWarps + 1]

    // ---- one-time: clear the other barrier counter; stage tables in smem
    if (blockIdx.x == 0 && tid == 0) a.ws->barrier[a.parity ^ 1u] = 0u;
    const uint32_t rep = a.filter_rep;
    for (uint32_t i = tid; i < a.filter_words * rep; i += kThreads) s_filter[i] = __ldg(a.t.filter + i / rep);
    for (uint32_t i = tid; i < 256; i += kThreads) s_root[i] = __ldg(a.t.root + i);
    for (uint32_t i = tid; i <= a.hot_nodes; i += kThreads) s_node[i] = __ldg(a.t.node + i);
    for (uint32_t i = tid; i < a.hot_edges; i += kThreads) s_label[i] = __ldg(a.t.label + i);
    if (lane < kSlots) mbar_init(&bars[lane], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    Smem s;
    s.filter = s_filter + (lane & (rep - 1));
    s.root = s_root;
    s.node = s_node;
    s.label = s_label;

    const uint32_t gram = a.t.gram;
    const uint32_t kmask = gram >= 4 ? 0xFFFFFFFFu : ((1u << (8 * gram)) - 1u);
    const uint64_t policy = evict_first_policy();
    // starts < lim are valid: inside [0, n_starts) and their d-gram fits
    const uint64_t lim = (a.readable + 1 >= gram && a.readable + 1 - gram < a.n_starts) ? a.readable + 1 - gram
                                                                                        : a.n_starts;
    // ---- this warp's contiguous range of rounds
    const uint64_t gw = (uint64_t)blockIdx.x * kWarps + warp;
    const uint64_t n_rounds = (a.n_starts + kRound - 1) / kRound;
    const uint64_t r_begin = gw * a.rounds_per_warp < n_rounds ? gw * a.rounds_per_warp : n_rounds;
    const uint64_t r_end = r_begin + a.rounds_per_warp < n_rounds ? r_begin + a.rounds_per_warp : n_rounds;
    const uint64_t range_lo = r_begin * kRound;
    uint32_t *hits = a.hits + gw * a.hit_cap;

    // Fill slot `i % kSlots` with round r_begin + i of this warp's range.
    auto issue = [&](uint64_t i) {
        const uint32_t slot = (uint32_t)(i % kSlots);
        uint8_t *dst = ring + slot * kSlotBytes;
        const uint64_t lo = (r_begin + i) * kRound;
        const uint64_t avail = lo < a.readable ? a.readable - lo : 0;
        if (a.aligned && avail >= (uint64_t)kSlotBytes) {
            if (lane == 0) {
                fence_proxy_async_smem();  // prior generic reads of the slot precede the async write
                mbar_arrive_expect_tx(&bars[slot], kSlotBytes);
                bulk_g2s(dst, a.text + lo, kSlotBytes, &bars[slot], policy);
            }
        } else {  // unaligned text or ragged tail: lanes copy, zero-fill past `readable`
            for (int k = 0; k < kPerLane; ++k) {
                const uint32_t o = lane * kPerLane + k;
                dst[o] = o < avail ? __ldg(a.text + lo + o) : (uint8_t)0;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars[slot]);
        }
    };

    // ================================================= phase 1: scan
    const uint64_t nr = r_end - r_begin;
    for (uint64_t i = 0; i < nr && i < kSlots - 1; ++i) issue(i);
    uint64_t total = 0;   // pattern ids matched in this range (warp-uniform)
    uint32_t n_hits = 0;  // hit records produced (warp-uniform; may exceed hit_cap)
    for (uint64_t i = 0; i < nr; ++i) {
        if (i + kSlots - 1 < nr) issue(i + kSlots - 1);  // refills the slot of round i-1
        const uint32_t slot = (uint32_t)(i % kSlots);
        mbar_wait(&bars[slot], (uint32_t)((i / kSlots) & 1));
        const bool has_next = i + 1 < nr;
        const uint32_t slot1 = (uint32_t)((i + 1) % kSlots);
        if (has_next) mbar_wait(&bars[slot1], (uint32_t)(((i + 1) / kSlots) & 1));
        const uint8_t *p0 = ring + slot * kSlotBytes;
        const uint8_t *p1 = ring + slot1 * kSlotBytes;
        const uint64_t rbase = (r_begin + i) * kRound;
        const TextView tv{p0, p1, rbase, has_next ? (uint32_t)(2 * kSlotBytes) : (uint32_t)kSlotBytes};

        // ---- stage 1: d-gram filter over the lane's 16 starts
        const uint4 q = *reinterpret_cast<const uint4 *>(p0 + lane * kPerLane);
        uint32_t w4 = __shfl_down_sync(0xffffffffu, q.x, 1);
        if (lane == 31) {
            if (has_next) {
                w4 = *reinterpret_cast<const uint32_t *>(p1);
            } else {
                w4 = 0;
                const uint64_t j0 = rbase + kRound;
                for (int b = 0; b < 4; ++b)
                    if (j0 + b < a.readable) w4 |= (uint32_t)__ldg(a.text + j0 + b) << (8 * b);
            }
        }
        const uint32_t wv[5] = {q.x, q.y, q.z, q.w, w4};
        const uint64_t lbase = rbase + (uint64_t)lane * kPerLane;
        const uint32_t nvalid =
            lbase >= lim ? 0u : (lim - lbase >= (uint64_t)kPerLane ? (uint32_t)kPerLane : (uint32_t)(lim - lbase));
        const uint32_t surv = filter16(a, s, wv, kmask, nvalid);

        // ---- stage 2: survivors walk the trie
        uint32_t c = 0, hm = 0;
        for (uint32_t m = surv; m; m &= m - 1) {
            const int k = __ffs(m) - 1;
            const uint32_t tn = walk(a, s, tv, lbase + k, p0[lane * kPerLane + k]);
            if (tn != kNone) {
                const uint32_t ti = term_index(a.t, tn);
                c += __ldg(a.t.out_ptr + ti + 1) - __ldg(a.t.out_ptr + ti);
                hm |= 1u << k;
            }
        }
        // ---- append hit offsets in position order (lane-major, then k)
        uint32_t htot;
        const uint32_t hex = warp_excl_scan((uint32_t)__popc(hm), lane, &htot);
        if (htot) {
            uint32_t idx = n_hits + hex;
            const uint32_t off0 = (uint32_t)(lbase - range_lo);
            for (uint32_t m = hm; m; m &= m - 1, ++idx)
                if (idx < a.hit_cap) hits[idx] = off0 + (uint32_t)(__ffs(m) - 1);
            n_hits += htot;
        }
        uint32_t ct;
        warp_excl_scan(c, lane, &ct);
        total += ct;
        __syncwarp();
    }

    // ================================================= phase 2: offsets
    if (lane == 0) s_wtot[warp] = total;
    __syncthreads();
    if (warp == 0) {
        unsigned long long v = s_wtot[lane];  // kWarps == 32
        unsigned long long incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        s_wtot[lane] = incl - v;  // exclusive within the CTA
        if (lane == 31) a.cta_total[blockIdx.x] = incl;
    }
    grid_barrier(&a.ws->barrier[a.parity]);
    if (warp == 0) {
        unsigned long long pre = 0, all = 0;
        for (uint32_t b = lane; b < gridDim.x; b += 32) {
            const unsigned long long v = __ldcg(a.cta_total + b);
            all += v;
            if (b < blockIdx.x) pre += v;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            pre += __shfl_xor_sync(0xffffffffu, pre, d);
            all += __shfl_xor_sync(0xffffffffu, all, d);
        }
        if (lane == 0) {
            s_wtot[kWarps] = pre;
            if (blockIdx.x == 0) *a.out_count = all;
        }
    }
    __syncthreads();
    uint64_t off = s_wtot[kWarps] + s_wtot[warp];  // this warp's first output row

    // ================================================= phase 3: emit
    if (total == 0) return;
    const TextView gv{nullptr, nullptr, 0, 0};
    if (n_hits <= a.hit_cap) {
        for (uint32_t b = 0; b < n_hits; b += 32) {
            const uint32_t i = b + lane;
            uint32_t ti = kNone, cnt = 0;
            uint64_t gi = 0;
            if (i < n_hits) {
                gi = range_lo + hits[i];
                const uint32_t tn = walk(a, s, gv, gi, __ldg(a.text + gi));
                ti = term_index(a.t, tn);
                cnt = __ldg(a.t.out_ptr + ti + 1) - __ldg(a.t.out_ptr + ti);
            }
            uint32_t ctot;
            uint64_t o = off + warp_excl_scan(cnt, lane, &ctot);
            if (cnt) {
                const uint32_t r0 = __ldg(a.t.out_ptr + ti);
                for (uint32_t e = 0; e < cnt; ++e, ++o) {
                    if (o < a.capacity) {
                        a.out_pos[o] = a.pos_base + gi;
                        a.out_pid[o] = __ldg(a.t.out_pid + r0 + e);
                    }
                }
            }
            off += ctot;
        }
    } else {
        // hit list overflowed: scan the range again, writing rows directly
        for (uint64_t i = 0; i < nr; ++i) {
            const uint64_t rbase = (r_begin + i) * kRound;
            const uint64_t lbase = rbase + (uint64_t)lane * kPerLane;
            uint32_t wv[5] = {0, 0, 0, 0, 0};
            for (int b = 0; b < 20; ++b)
                if (lbase + b < a.readable) wv[b >> 2] |= (uint32_t)__ldg(a.text + lbase + b) << (8 * (b & 3));
            const uint32_t nvalid = lbase >= lim ? 0u
                                                 : (lim - lbase >= (uint64_t)kPerLane ? (uint32_t)kPerLane
                                                                                      : (uint32_t)(lim - lbase));
            const uint32_t surv = filter16(a, s, wv, kmask, nvalid);
            uint32_t c = 0, hm = 0;
            for (uint32_t m = surv; m; m &= m - 1) {
                const int k = __ffs(m) - 1;
                const uint32_t tn = walk(a, s, gv, lbase + k, __ldg(a.text + lbase + k));
                if (tn != kNone) {
                    const uint32_t ti = term_index(a.t, tn);
                    c += __ldg(a.t.out_ptr + ti + 1) - __ldg(a.t.out_ptr + ti);
                    hm |= 1u << k;
                }
            }
            uint32_t ctot;
            uint64_t o = off + warp_excl_scan(c, lane, &ctot);
            for (uint32_t m = hm; m; m &= m - 1) {
                const uint64_t gi = lbase + (uint64_t)(__ffs(m) - 1);
                const uint32_t ti = term_index(a.t, walk(a, s, gv, gi, __ldg(a.text + gi)));
                const uint32_t r0 = __ldg(a.t.out_ptr + ti), r1 = __ldg(a.t.out_ptr + ti + 1);
                for (uint32_t e = r0; e < r1; ++e, ++o) {
                    if (o < a.capacity) {
                        a.out_pos[o] = a.pos_base + gi;
                        a.out_pid[o] = __ldg(a.t.out_pid + e);
                    }
                }
            }
            off += ctot;
        }
    }
}

struct DeviceInfo {
    bool init = false;
    int sms = 0;
    int max_smem_optin = 0;
};
std::mutex g_dev_mu;
DeviceInfo g_dev[64];

std::mutex g_ws_mu;
std::map<const void *, uint32_t> g_ws_parity;  // grid-barrier counter in use next, per workspace

inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

int device_info(int device, DeviceInfo &out, std::string &err) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DeviceInfo &di = g_dev[device];
    if (!di.init) {
        cudaError_t e = cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, device);
        if (e == cudaSuccess)
            e = cudaDeviceGetAttribute(&di.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(pfac_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     di.max_smem_optin);
        if (e != cudaSuccess) {
            err = std::string("device query: ") + cudaGetErrorString(e);
            return kStatusCuda;
        }
        di.init = true;
    }
    out = di;
    return kStatusOk;
}

// Launch geometry shared by workspace sizing and the launch itself.
struct Geometry {
    uint64_t grid, warps, rounds_per_warp;
    uint32_t hit_cap;
};
Geometry geometry(uint64_t n_starts, int sms) {
    Geometry g;
    const uint64_t n_rounds = (n_starts + kRound - 1) / kRound;
    g.grid = (uint64_t)sms;
    if (g.grid * kWarps > n_rounds) g.grid = (n_rounds + kWarps - 1) / kWarps;
    if (g.grid < 1) g.grid = 1;
    g.warps = g.grid * kWarps;
    g.rounds_per_warp = (n_rounds + g.warps - 1) / g.warps;
    if (g.rounds_per_warp < 1) g.rounds_per_warp = 1;
    // hit records per warp: 1/16 of its starts, between 64 and 4096 (a warp
    // that finds more re-scans its range in phase 3 instead)
    uint64_t cap = g.rounds_per_warp * kRound / 16;
    if (cap < 64) cap = 64;
    if (cap > 4096) cap = 4096;
    g.hit_cap = (uint32_t)cap;
    return g;
}

}  // namespace

DevTrie make_dev_trie(const ImageHeader &h, const uint8_t *d) {
    DevTrie t;
    t.node = reinterpret_cast<const uint32_t *>(d + h.off_node);
    t.label = d + h.off_label;
    t.term_node = reinterpret_cast<const uint32_t *>(d + h.off_term_node);
    t.out_ptr = reinterpret_cast<const uint32_t *>(d + h.off_out_ptr);
    t.out_pid = reinterpret_cast<const uint32_t *>(d + h.off_out_pid);
    t.root = reinterpret_cast<const uint32_t *>(d + h.off_root);
    t.filter = reinterpret_cast<const uint32_t *>(d + h.off_filter);
    t.n_terminals = (uint32_t)h.n_terminals;
    t.max_len = h.max_len;
    t.gram = h.filter_gram;
    t.log2_bits = h.filter_log2_bits;
    t.exact = h.filter_exact;
    t.n_nodes = (uint32_t)h.n_nodes;
    return t;
}

int workspace_bytes_for(uint64_t n_starts, int device, uint64_t *out, std::string &err) {
    DeviceInfo di;
    int st = device_info(device, di, err);
    if (st != kStatusOk) return st;
    const Geometry g = geometry(n_starts, di.sms);
    *out = kWsFixed + 4ull * g.warps * g.hit_cap;
    return kStatusOk;
}

uint32_t launches_per_call() { return 1; }  // the scan kernel

int launch_scan(const DevTrie &t, const uint32_t *host_node, int device, const uint8_t *d_text,
                uint64_t readable_len, uint64_t n_starts, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                uint64_t capacity, uint64_t *d_count, void *d_ws, uint64_t ws_bytes, CUstream_st *stream_,
                std::string &err) {
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
    if (device < 0 || device >= 64) {
        err = "pfac_match_device: bad device ordinal";
        return kStatusInvalid;
    }
    if (n_starts == 0) {
        cudaError_t e = cudaMemsetAsync(d_count, 0, sizeof(uint64_t), stream);
        if (e != cudaSuccess) {
            err = std::string("cudaMemsetAsync: ") + cudaGetErrorString(e);
            return kStatusCuda;
        }
        return kStatusOk;
    }
    DeviceInfo di;
    int st = device_info(device, di, err);
    if (st != kStatusOk) return st;
    const Geometry geo = geometry(n_starts, di.sms);
    const uint64_t need = kWsFixed + 4ull * geo.warps * geo.hit_cap;
    if (!d_ws || ws_bytes < need || (reinterpret_cast<uintptr_t>(d_ws) & 15)) {
        err = "pfac_match_device: workspace too small or misaligned";
        return kStatusInvalid;
    }
    // ---- shared-memory plan: ring + barriers + root + warp totals, then the
    // filter (replicated while it fits half of the rest), then the hot trie.
    const uint32_t filter_words = (1u << t.log2_bits) >= 32 ? (1u << t.log2_bits) / 32 : 1u;
    const uint32_t fixed = kWarps * kSlots * kSlotBytes + kWarps * kSlots * 8 + 1024 + 8 * (kWarps + 1) + 256;
    if ((uint32_t)di.max_smem_optin < fixed + filter_words * 4 + 64) {
        err = "pfac_match_device: filter does not fit shared memory";
        return kStatusLimit;
    }
    const uint32_t rest = (uint32_t)di.max_smem_optin - fixed;
    uint32_t rep = 1;
    while (rep < 32 && filter_words * 4 * (rep * 2) <= rest / 2) rep *= 2;
    const uint32_t trie_budget = rest - filter_words * 4 * rep;
    // H = largest node count whose words [0, H] and labels [0, row_ptr[H]) fit
    uint32_t lo = 0, hi = t.n_nodes - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        const uint64_t bytes = 4ull * (mid + 1) + 16 + ((uint64_t)(host_node[mid] & kEdgeMask) + 15) / 16 * 16;
        if (bytes <= trie_budget) lo = mid; else hi = mid - 1;
    }
    const uint32_t H = lo;
    const uint32_t EH = host_node[H] & kEdgeMask;

    ScanArgs a;
    a.t = t;
    a.filter_words = filter_words;
    a.filter_rep = rep;
    uint32_t o = 0;
    a.off_ring = o;   o += kWarps * kSlots * kSlotBytes;
    a.off_bar = o;    o += kWarps * kSlots * 8;
    a.off_warp = o;   o += 8 * (kWarps + 1);
    o = align_up(o, 16);
    a.off_root = o;   o += 1024;
    a.off_filter = o; o += filter_words * 4 * rep;
    a.off_node = o;   o = align_up(o + 4 * (H + 1), 16);
    a.off_label = o;  o = align_up(o + EH, 16);
    const size_t smem = o;
    if (smem > (size_t)di.max_smem_optin) {
        err = "pfac_match_device: internal shared-memory plan error";
        return kStatusLimit;
    }
    a.hot_nodes = H;
    a.hot_edges = EH;
    uint32_t parity;
    {
        std::lock_guard<std::mutex> lk(g_ws_mu);
        uint32_t &p = g_ws_parity[d_ws];  // 0 for a new (zero-filled) workspace
        parity = p;
        p ^= 1u;
    }
    a.text = d_text;
    a.readable = readable_len;
    a.n_starts = n_starts;
    a.pos_base = pos_base;
    a.out_pos = d_pos;
    a.out_pid = d_pid;
    a.capacity = capacity;
    a.out_count = d_count;
    a.ws = reinterpret_cast<WsHeader *>(d_ws);
    a.cta_total = reinterpret_cast<unsigned long long *>(reinterpret_cast<uint8_t *>(d_ws) + sizeof(WsHeader));
    a.hits = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(d_ws) + kWsFixed);
    a.hit_cap = geo.hit_cap;
    a.parity = parity;
    a.rounds_per_warp = geo.rounds_per_warp;
    a.aligned = (reinterpret_cast<uintptr_t>(d_text) & 15) == 0;
    void *args[] = {&a};
    cudaError_t e = cudaLaunchCooperativeKernel((const void *)pfac_scan_kernel, dim3((unsigned)geo.grid),
                                                dim3(kThreads), args, smem, stream);
    if (e != cudaSuccess) {
        {   // the kernel did not run: the barrier counter in use is unchanged
            std::lock_guard<std::mutex> lk(g_ws_mu);
            g_ws_parity[d_ws] = parity;
        }
        err = std::string("scan launch: ") + cudaGetErrorString(e);
        return kStatusCuda;
    }
    return kStatusOk;
}

}  // namespace pfac

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
//  * one persistent CTA per SM (kWarps warps, 64 registers).  Shared memory
//    holds, once per SM, the first-stage filter at offset 0 (replicated with
//    bank swizzles while it fits), one region per warp (text ring, its
//    mbarriers, the probe and walk queues; compile-time offsets from one
//    base), the level-1 table, the level-1 bitmapped nodes (PAPER.md:97
//    Fig. 3), the 2-gram table where selective, and the top H nodes of the
//    breadth-first CSR trie (BFS order = level order, so the first H nodes
//    are the hot upper levels; PAPER.md:89 kept row_ptr on chip for the same
//    reason).  The dynamic window starts at shared address kSmemBase (checked
//    at entry), so queues, ring and tables are addressed as 32-bit constants
//    plus offsets.  Cluster placement (PFAC_PLACE_CLUSTER, the kCl kernels)
//    instead spreads the node records of the BFS prefix over a thread-block
//    cluster, read through distributed shared memory.
//  * phase 1 (scan): CTA b owns a contiguous range of 1024-start rounds; its
//    warps own contiguous blocks of the range's first part and take the rest
//    (a plan's share) from a shared counter; the text's last rounds form a
//    cross-CTA pool.  A per-warp ring of kSlots slots (1 KiB + 16-byte
//    overhang) is filled by TMA bulk copies (cp.async.bulk + mbarrier,
//    evict-first in L2) kSlots-1 rounds ahead.  Per round each lane tests its
//    32 consecutive starts against the filter (a clear bit means no pattern
//    can start there: PFAC's early termination taken before the first trie
//    access), then, where selective, each survivor against the 2-gram prefix
//    table; the kept starts are queued in position order, probed in full-warp
//    batches (exact key set, kind 1; depth-8/16 entry table, kinds 4/3) and
//    the survivors walked 32 at a time to the first mismatch.  A start that
//    passed a terminal is appended, in position order, to the warp's hit list
//    (offset, terminal index), its pid count to the lane's rows (block) or the
//    round's count.
//  * phase 2 (offsets): CTA exclusive scan of the warp totals and the dynamic
//    rounds' counts -> a self-resetting grid barrier -> exclusive prefix over
//    CTA totals (the pool's segments after a second barrier).  Ranges are
//    contiguous and ordered, so the concatenation is sorted by (pos, pid).
//  * phase 3 (emit): each warp expands its hit list into (pos, pid) rows (a
//    segmented scan gives each row its index).  A warp whose list overflowed
//    re-scans its rounds writing rows directly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace pfac {

namespace {

#ifndef PFAC_WARPS
#define PFAC_WARPS 32
#endif
constexpr int kWarps = PFAC_WARPS;
constexpr int kThreads = kWarps * 32;
constexpr int kPerLane = 32;           // consecutive starts per lane per round
constexpr int kRound = 32 * kPerLane;  // 1024 starts per warp round
constexpr int kRoundLog2 = 10;
static_assert(kRound == 1 << kRoundLog2, "");
constexpr int kWv = kPerLane / 4 + 1;  // text words a lane needs (its starts + 3 bytes)
constexpr int kSlotsMax = 3;           // text ring depth per warp (kSlots-1 rounds in flight); 2 when the filter
                                       // takes more than 64 KiB of shared memory
#ifndef PFAC_SLOT_EXTRA
#define PFAC_SLOT_EXTRA 16
#endif
constexpr int kSlotBytes = kRound + PFAC_SLOT_EXTRA;  // one round of text (+ the next 16 bytes: the last windows)
static_assert(kSlotsMax >= 2, "ring");
constexpr int kMaxCtas = 1024;
constexpr uint32_t kFilterCap = 65536;  // max shared bytes for the replicated filter
#ifndef PFAC_DEFER
#define PFAC_DEFER 48
#endif
constexpr int kDefer = PFAC_DEFER;             // per-warp queue of starts to walk (kinds 0, 1, 2)
constexpr uint32_t kWalkQ = 64;                // walk-queue capacity per warp (two-level kinds)

// Per-warp region of shared memory (one base per warp; every part at a
// compile-time offset from it): the TMA text ring, its mbarriers, the queue
// of kept starts (+ their keys, kind 1) and the walk queue (+ entry words,
// kinds 3/4).
__host__ __device__ constexpr uint32_t defer_cap(int kind) {
    return kind == 3 ? 64u : kind == 4 ? 96u : (uint32_t)kDefer;  // deeper for DNA / 8-byte prefixes (long walks)
}
struct WarpLayout {
    uint32_t ring, bars, dpos, dkey, bpos, bent, bytes;
};
__host__ __device__ constexpr WarpLayout warp_layout(int kind, int slots) {
    const uint32_t ring = 0, bars = ring + slots * kSlotBytes, dpos = bars + 8u * slots,
                   dkey = dpos + 4u * defer_cap(kind), bpos = dkey + (kind == 1 ? 4u * defer_cap(kind) : 0u),
                   bent = bpos + ((kind == 1 || kind == 3 || kind == 4) ? 4u * kWalkQ : 0u),
                   end = bent + ((kind == 3 || kind == 4) ? 4u * kWalkQ : 0u);
    return WarpLayout{ring, bars, dpos, dkey, bpos, bent, (end + 15u) & ~15u};
}
constexpr uint64_t kSmallTrie = 160u << 10;  // a trie this small fits shared memory whole
constexpr uint64_t kBigL1Trie = 1u << 20;    // "big L1" plan up to this trie size (see launch_scan)

// Workspace: header (a self-resetting grid barrier and the pool counter,
// zero after every launch: no host-side state, so a captured CUDA graph may
// replay the launch) + CTA totals + hit lists.
struct WsHeader {
    unsigned int bar_count;  // CTAs arrived at the current grid barrier (0 between barriers)
    unsigned int bar_gen;    // grid-barrier generation (any value; bumped by the last arrival)
    unsigned int pool_next;  // next pool round (reset after the first grid barrier)
    unsigned int pad[61];
};
static_assert(sizeof(WsHeader) == 256, "");
// fixed part: header | cta_total[kMaxCtas] u64 | pool_total[kMaxCtas] u64
constexpr uint64_t kWsFixed = sizeof(WsHeader) + 16ull * kMaxCtas;
static_assert(kWsFixed == kWsDagOffset, "the merged-DAG scan's block totals follow the fixed part");
constexpr uint32_t kNoRound = 0xFFFFFFFFu;  // take(): no round left

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
    uint2 *hits;                    // [warps][hit_cap] (start offset within the warp's range, terminal index)
    uint32_t hit_cap;
    uint64_t rounds_per_cta;        // of the first n_main rounds (the CTA ranges)
    uint64_t n_main;                // rounds in CTA ranges; rounds [n_main, n_rounds) are the shared pool
    uint32_t pool_seg;              // pool rounds per CTA in the pool's scan (0: no pool)
    unsigned long long *pool_total; // [grid] row totals of the pool segments
    unsigned long long *round_val;  // [n_rounds] pid count of the round, then its first row within the CTA
    uint32_t *round_owner;          // [n_rounds] global warp that scanned the round
    // shared-memory layout (bytes from the dynamic smem base; filter at 0)
    uint32_t filter_words;          // words of the (unreplicated) filter
    uint32_t rep_log2;              // replication factor 2^rep_log2 (<= 32)
    uint32_t off_root, off_node, off_label, off_warps, off_sbar, off_warp, off_bm, off_pair, off_aux;
    uint32_t off_tails, off_tbytes;
    uint32_t hot_tails, hot_tail_bytes;  // records (and their bytes) of the record nodes < H
    uint32_t off_terms;             // out_ptr[T+1] in smem (0 = in global memory)
    uint32_t n_level1;              // B: the root's children are nodes [1, B]
    uint32_t hot_nodes;             // H: node words [0, H] resident
    uint32_t hot_edges;             // row_ptr[H]: labels [0, hot_edges) resident
    uint32_t aligned;               // text pointer is 16-byte aligned (bulk-copy path)
    uint32_t use_kset;              // probe the exact key set before walks (trie not wholly in smem)
    uint32_t ctg64;                 // share of a CTA's rounds in contiguous per-warp blocks, in 64ths
                                    // (the rest, the range's end, is handed out dynamically)
    uint32_t use_pair;              // the 2-gram prefix table is staged and tested
    uint32_t use_entry;            // kind 4: walks enter through the depth-8 entry table
    // cluster placement (PFAC_PLACE_CLUSTER): node records [0, dsm_nodes) in
    // the cluster's shared memories, CTA rank q holding [q << dsm_log2,
    // (q + 1) << dsm_log2) at off_dsm (0 = no cluster tier)
    uint32_t dsm_nodes, dsm_log2, off_dsm;
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
// (the same on 32-bit shared-window addresses: no generic->shared conversion per use)
__device__ __forceinline__ void mbar_arrive_expect_tx_s(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s_s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar,
                                           uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_s(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// The dynamic shared memory's shared-window address: the 1 KiB the system
// reserves per block comes first, and the scan kernel has no static shared
// memory and no cluster (the CTA-rank bits of the window are 0).  The kernel
// checks it at entry; its per-warp queues and ring are then addressed with
// 32-bit constants-plus-offsets (no generic->shared conversion per access).
constexpr uint32_t kSmemBase = 1024u;
// Queue / ring accesses on 32-bit shared addresses.  Ordered among
// themselves and against the warp's __syncwarp() (volatile, memory clobber).
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds32q(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds8q(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ uint4 lds128q(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
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
__device__ __forceinline__ uint64_t evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__host__ __device__ constexpr uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const unsigned int *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

#ifdef PFAC_TIMING
// Instrumented build only (tools/timing.py): per-warp %globaltimer stamps.
__device__ unsigned long long g_pfac_timing[8192 * 16];
__device__ __forceinline__ void stamp(int warp_global, int k) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if ((threadIdx.x & 31) == 0 && warp_global < 8192) g_pfac_timing[warp_global * 16 + k] = t;
}
#define STAMP(k) stamp((int)(blockIdx.x * kWarps + (threadIdx.x >> 5)), k)
#else
#define STAMP(k)
#endif

// One barrier across the (co-resident, cooperative-launch) grid: a
// generation (sense-reversing) barrier.  The generation is read before
// arriving (it cannot advance before this CTA arrives); the last CTA to
// arrive resets the count and then bumps the generation, which the others
// wait on.  The count is back at 0 after every barrier, so the workspace
// needs no per-launch host state.
__device__ __forceinline__ uint32_t ld_relaxed_u32(const unsigned int *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void grid_barrier(WsHeader *ws) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t gen = ld_relaxed_u32(&ws->bar_gen);
        __threadfence();  // this CTA's writes before its arrival
        if (atomicAdd(&ws->bar_count, 1u) == gridDim.x - 1) {
            ws->bar_count = 0u;
            __threadfence();  // the reset (and every arrival seen) before the release
            atomicAdd(&ws->bar_gen, 1u);
        } else {
            while (ld_acquire_u32(&ws->bar_gen) == gen) {
            }
        }
        __threadfence();
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
// The staged tables as 32-bit shared addresses (read with ldt*: no generic
// pointer, so no shared-window conversion per use); the terminal tables as
// generic pointers (shared or global memory).
struct Smem {
    uint32_t root;              // level-1 table: child of the root per byte
    uint32_t bm;                // level-1 bitmapped nodes, 10 words each (see below)
    uint32_t node;              // node words [0, H]
    uint32_t aux;               // aux words [0, H]
    uint32_t label;             // labels [0, hot_edges)
    uint32_t tails;             // tail records [0, hot_tails), 16 bytes each
    uint32_t tail_bytes;        // their bytes [0, hot_tail_bytes)
    const uint32_t *out_ptr;    // pid-list offsets by terminal index (smem or global)
};
// Loads from the staged (immutable after staging) tables: plain asm, so the
// compiler may schedule and merge them freely.
__device__ __forceinline__ uint32_t ldt32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t ldt8(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint4 ldt128(uint32_t addr) {
    uint4 v;
    asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t label_at(const ScanArgs &a, const Smem &s, uint32_t e) {
    PFAC_CHECK(e < a.t.n_edges);
    return e < a.hot_edges ? ldt8(s.label + e) : (uint32_t)__ldg(a.t.label + e);
}

// Text of a walk read from global memory (L1/L2): `g` = text + start,
// `end` = readable bytes from there (clamped to 32 bits).
struct GlobalText {
    const uint8_t *g;
    uint32_t end;
    uint32_t aligned;  // the text pointer is 16-byte aligned
    __device__ __forceinline__ uint32_t at(uint32_t r) const { return __ldg(g + r); }
    // bytes r..r+3 (little-endian; zero past `end`)
    __device__ __forceinline__ uint32_t at4(uint32_t r) const {
        const uintptr_t ad = reinterpret_cast<uintptr_t>(g + r);
        if (aligned && r + 8 <= end) {  // two aligned words hold the four bytes
            const uint32_t *w = reinterpret_cast<const uint32_t *>(ad & ~(uintptr_t)3);
            return __funnelshift_r(__ldg(w), __ldg(w + 1), 8 * (uint32_t)(ad & 3));
        }
        uint32_t x = 0;
        for (int b = 0; b < 4; ++b)
            if (r + b < end) x |= (uint32_t)__ldg(g + r + b) << (8 * b);
        return x;
    }
    // bytes r..r+15 as four little-endian words (one load per word + one for
    // the misalignment when the text is aligned and 20 bytes are readable)
    __device__ __forceinline__ void at16(uint32_t r, uint32_t (&o)[4]) const {
        const uintptr_t ad = reinterpret_cast<uintptr_t>(g + r);
        if (aligned && r + 20 <= end) {
            const uint32_t *w = reinterpret_cast<const uint32_t *>(ad & ~(uintptr_t)3);
            const uint32_t sh = 8 * (uint32_t)(ad & 3);
            uint32_t x[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) x[q] = __ldg(w + q);
#pragma unroll
            for (int q = 0; q < 4; ++q) o[q] = __funnelshift_r(x[q], x[q + 1], sh);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) o[q] = at4(r + 4 * q);
        }
    }
    // Do the L text bytes from r equal the words pw (L <= end - r checked by
    // the caller)?  The fast path slides over the aligned text words, one load
    // per 4 bytes; the pattern words come from shared (kHot: shared address
    // ps) or global memory (pw).
    template <bool kHot>
    __device__ __forceinline__ bool equal(uint32_t r, const uint32_t *pw, uint32_t ps, uint32_t L) const {
        const uintptr_t ad = reinterpret_cast<uintptr_t>(g + r);
        if (aligned && r + L + 8 <= end) {
            const uint32_t *w = reinterpret_cast<const uint32_t *>(ad & ~(uintptr_t)3);
            const uint32_t sh = 8 * (uint32_t)(ad & 3);
            uint32_t a0 = __ldg(w);
            for (uint32_t k = 0; k < L; k += 4) {
                const uint32_t a1 = __ldg(w + (k >> 2) + 1);
                const uint32_t n = L - k;
                const uint32_t m = n >= 4 ? 0xFFFFFFFFu : ((1u << (8 * n)) - 1u);
                const uint32_t pk = kHot ? ldt32(ps + k) : __ldg(pw + (k >> 2));
                if ((__funnelshift_r(a0, a1, sh) ^ pk) & m) return false;
                a0 = a1;
            }
            return true;
        }
        for (uint32_t k = 0; k < L; k += 4) {
            const uint32_t n = L - k;
            const uint32_t m = n >= 4 ? 0xFFFFFFFFu : ((1u << (8 * n)) - 1u);
            const uint32_t pk = kHot ? ldt32(ps + k) : __ldg(pw + (k >> 2));
            if ((at4(r + k) ^ pk) & m) return false;
        }
        return true;
    }
};

// Walk from the start at offset r0 to the first mismatch; returns the terminal
// index of the deepest terminal passed, or kNone.  Level 1 (the root's children, nodes
// [1, B]) uses the paper's bitmapped node (Fig. 3: 256-bit child
// bitmap + offset, child = offset + rank of c among the set bits); deeper
// nodes use the CSR label list of the image.
// Terminal index of kept terminal node v from the rank structure (image
// v22): one 8-byte load, no search
__device__ __forceinline__ uint32_t term_rank(const uint2 *rk, uint32_t v) {
    const uint2 r = __ldg(rk + (v >> 5));
    return r.y + __popc(r.x & ((1u << (v & 31)) - 1u));
}
// terminal index of node `last` (kNone stays kNone); needs `a` in scope
#define term_of(last_) ((last_) == kNone ? kNone : term_rank(a.t.term_rk, (last_)))

// Jump at a tail or chain start v (node word bit 30) with the next text
// byte at offset j: its record holds the L bytes of the single path below v.
// Tail: the path ends at a terminal; the walk ends with that terminal if the
// next L text bytes equal the path, else with `last`.  Chain: the path ends at
// node x; on a match the walk continues at x (*nv = x, *len = L), else it ends
// with `last`.  *nv = kNone when the walk ends (the result is returned).
template <class Text>
__device__ __forceinline__ uint32_t jump(const ScanArgs &a, const Smem &s, const Text &tx, uint32_t v, uint32_t j,
                                         uint32_t last, uint32_t &nv, uint32_t &len, uint32_t ax) {
    nv = kNone;
    const bool hot = v < a.hot_nodes;  // hot records + bytes are in shared memory
    const uint32_t idx = ax;  // aux word: the record's index (= rank among the record nodes)
    PFAC_CHECK(idx < a.t.n_records && (!hot || idx < a.hot_tails));
    const uint4 rec = hot ? ldt128(s.tails + 16u * idx) : __ldg(a.t.tails + idx);
    PFAC_CHECK(rec.z == kVerify ? (uint64_t)rec.x + rec.y <= a.t.n_records
                                : (uint64_t)rec.x + rec.y <= a.t.n_tail_bytes && (!hot || rec.x + rec.y <= a.hot_tail_bytes + 3));
    if (rec.z == kVerify) {
        // verify leaf of a truncated trie (PAPER.md:80 step III): the
        // candidates (distinct patterns below it, longest first; records and
        // bytes in global memory) are compared with the text; the first that
        // matches gives the start's list (every pattern on its root path),
        // else the deepest terminal passed does
        for (uint32_t c = rec.x; c < rec.x + rec.y; ++c) {
            const uint4 cr = __ldg(a.t.tails + c);
            PFAC_CHECK((uint64_t)cr.x + cr.y <= a.t.n_tail_bytes && cr.z < a.t.n_terminals);
            if ((uint64_t)j + cr.y > (uint64_t)tx.end) continue;
            if (tx.template equal<false>(j, reinterpret_cast<const uint32_t *>(a.t.tail_bytes + cr.x), 0u, cr.y))
                return cr.z;
        }
        return term_of(last);
    }
    if ((uint64_t)j + rec.y > (uint64_t)tx.end) return term_of(last);
    // (separate loops: no shared/global select per word)
    const bool eq = hot ? tx.template equal<true>(j, nullptr, s.tail_bytes + rec.x, rec.y)
                        : tx.template equal<false>(j, reinterpret_cast<const uint32_t *>(a.t.tail_bytes + rec.x), 0u,
                                                   rec.y);
    if (!eq) return term_of(last);
    if (rec.z != kNone) return rec.z;  // tail
    nv = rec.w;                         // chain
    len = rec.y;
    return kNone;
}

// Child of node v (node word w) through byte c, or kNone: level-1 nodes by
// their bitmap (Fig. 3), deeper nodes by their CSR labels.
template <bool kWide>
__device__ __forceinline__ uint32_t child_of(const ScanArgs &a, const Smem &s, uint32_t v, uint32_t w, uint32_t c,
                                     bool l1, uint32_t wn, uint32_t ax, uint32_t ax2) {
    uint32_t nv = kNone;
    if (l1) {  // level 1 -> 2 through the bitmap
        PFAC_CHECK(v >= 1 && v <= a.t.n_level1);
        const uint32_t bm = s.bm + 40u * (v - 1);
        const uint32_t word = ldt32(bm + 4u * (c >> 5));
        if (!((word >> (c & 31)) & 1u)) return kNone;
        const uint32_t pre = (ldt32(bm + 32u + 4u * (c >> 7)) >> (8 * ((c >> 5) & 3))) & 0xFFu;
        nv = (w & kEdgeMask) + pre + __popc(word & ((1u << (c & 31)) - 1u)) + 1;
    } else {
        const uint32_t lo0 = w & kEdgeMask;
        const uint32_t hi0 = wn & kEdgeMask;  // node word v+1 (loaded with w)
        const uint32_t deg = hi0 - lo0;
        if (deg <= 4) {  // the labels are packed in the node's aux word (loaded beside the node words)
            if (deg != 0) {
                const uint32_t x = (ax ^ (c * 0x01010101u)) | (0xFFFFFFFFu << (8 * deg - 1) << 1);
                const uint32_t f = (x - 0x01010101u) & ~x & 0x80808080u;
                if (f) nv = lo0 + ((__ffs(f) - 1) >> 3) + 1;  // the child through edge e is node e+1
            }
        } else if (kWide && deg <= 8 && ax2 != kNone) {  // 5..8 labels: aux + the record's last word
            const uint32_t x0 = ax ^ (c * 0x01010101u);
            const uint32_t f0 = (x0 - 0x01010101u) & ~x0 & 0x80808080u;
            const uint32_t x1 = (ax2 ^ (c * 0x01010101u)) | (0xFFFFFFFFu << (8 * (deg - 4) - 1) << 1);
            const uint32_t f1 = (x1 - 0x01010101u) & ~x1 & 0x80808080u;
            if (f0) nv = lo0 + ((__ffs(f0) - 1) >> 3) + 1;
            else if (f1) nv = lo0 + 4 + ((__ffs(f1) - 1) >> 3) + 1;
        } else if (deg <= 16) {
            // labels[lo0, hi0) lie in <= 5 aligned words: load them at once and
            // find the byte equal to c with the zero-byte test on (word ^ c),
            // bytes outside the node forced non-zero (a label occurs once, and
            // the lowest flagged byte of the test is exact)
            const bool hotl = hi0 <= a.hot_edges;
            const uint32_t base = lo0 & ~3u, c4 = c * 0x01010101u, nw = (hi0 - base + 3) >> 2;
#pragma unroll 1
            for (uint32_t q = 0; q < nw; ++q) {
                const uint32_t e0 = base + 4 * q;
                const uint32_t wq = hotl ? ldt32(s.label + e0)
                                         : __ldg(reinterpret_cast<const uint32_t *>(a.t.label + e0));
                uint32_t oor = 0;  // 0xFF in the bytes outside [lo0, hi0)
                if (e0 < lo0) oor = (1u << (8 * (lo0 - e0))) - 1u;
                if (hi0 - e0 < 4) oor |= ~((1u << (8 * (hi0 - e0))) - 1u);
                const uint32_t x = (wq ^ c4) | oor;
                const uint32_t f = (x - 0x01010101u) & ~x & 0x80808080u;
                if (f) {
                    nv = e0 + ((__ffs(f) - 1) >> 3) + 1;  // the child through edge e is node e+1
                    break;
                }
            }
        } else {
            uint32_t lo = lo0, hi = hi0;  // labels[lo, hi) ascending
            while (hi - lo > 4) {
                const uint32_t mid = (lo + hi) >> 1;
                if (label_at(a, s, mid) <= c) lo = mid; else hi = mid;
            }
            for (uint32_t k = lo; k < hi; ++k) {
                const uint32_t l = label_at(a, s, k);
                if (l >= c) {
                    if (l == c) nv = k + 1;  // BFS order: the child through edge e is node e+1
                    break;
                }
            }
        }
    }
    return nv;
}

// Walk from the start at offset r0 to the first mismatch; returns
// the terminal index of the deepest terminal passed, or kNone.  Level 1 (the
// root's children, nodes [1, B]) uses the paper's bitmapped node (PAPER.md:97,
// Fig. 3: 256-bit child bitmap + offset, child = offset + rank of c among the
// set bits); deeper nodes use the CSR label list of the image; tail and chain
// starts compare their path's bytes at once.
template <bool kDsm>
__device__ __forceinline__ void node_load(const ScanArgs &a, const Smem &s, uint32_t v, uint32_t &w, uint32_t &wn,
                                          uint32_t &ax, uint32_t &ax2) {
    // the node's word, the next node's word (its edge end) and its aux word:
    // from shared memory for the staged nodes, else one 16-byte record load
    // (whose last word holds labels 4..7 of a node with 5..8 children; ax2 =
    // kNone for a staged node: its labels are read from shared memory)
    if (v < a.hot_nodes) {
        w = ldt32(s.node + 4u * v);
        wn = ldt32(s.node + 4u * v + 4u);
        ax = ldt32(s.aux + 4u * v);
        ax2 = kNone;
    } else if (kDsm && v < a.dsm_nodes) {  // cluster placement: the record from its owner CTA's shared memory
        extern __shared__ __align__(128) uint8_t smem_base[];
        const uint32_t la = smem_u32(smem_base) + a.off_dsm + 16u * (v & ((1u << a.dsm_log2) - 1u));
        uint32_t ra;
        asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(v >> a.dsm_log2));
        asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w), "=r"(wn), "=r"(ax), "=r"(ax2)
                     : "r"(ra));
    } else {
        PFAC_CHECK(v < a.t.n_nodes);
        const uint4 r = __ldg(a.t.rec + v);
        w = r.x;
        wn = r.y;
        ax = r.z;
        ax2 = r.w;
    }
}

// kWide: 5..8-child nodes are matched from their aux word and record word
// (walk-heavy kinds: C3 -4%; kind 1, whose walks are rare, keeps the smaller
// code: C4 +1.6% with it)
// kDsm: the cluster kernels (node records of the cluster tier via DSMEM)
template <bool kWide, bool kDsm, class Text>
__device__ uint32_t walk(const ScanArgs &a, const Smem &s, const Text &tx, uint32_t r0, uint32_t v0 = 0,
                         uint32_t d0 = 1) {
    // (v0, d0): enter at image node v0 of depth d0 whose path the start's
    // first d0 bytes spell (the depth-8 entry table); else from the root
    uint32_t v = v0 ? v0 : ldt32(s.root + 4u * tx.at(r0));
    if (v == 0) return kNone;
    uint32_t w, wn, ax, ax2;
    uint32_t j = r0 + d0;
    // walk-heavy kinds (kWide): the next text byte is loaded beside the node
    // it is matched against (two independent loads per step, not two
    // dependent ones: C3 -1.9%; kind 1's rare walks keep the plain order)
    uint32_t c = kWide && j < tx.end ? tx.at(j) : 0u;
    node_load<kDsm>(a, s, v, w, wn, ax, ax2);
    uint32_t last = (w & kTermBit) ? v : kNone;
    bool l1 = d0 == 1;  // v is a level-1 node: the next step uses its bitmap
    while (j < tx.end) {
        uint32_t nv = kNone;
        if (w & kTailBit) {
            uint32_t len = 0;
            const uint32_t r = jump(a, s, tx, v, j, last, nv, len, ax);
            if (nv == kNone) return r;
            j += len;
        } else {
            nv = child_of<kWide>(a, s, v, w, kWide ? c : tx.at(j), l1, wn, ax, ax2);
            if (nv == kNone) break;  // mismatch: the thread terminates
            ++j;
        }
        l1 = false;
        v = nv;
        if (kWide) c = j < tx.end ? tx.at(j) : 0u;
        node_load<kDsm>(a, s, v, w, wn, ax, ax2);
        if (w & kTermBit) last = v;
    }
    return term_of(last);
}

__device__ __forceinline__ uint32_t clamp32(uint64_t x) { return x > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)x; }


// Stage 1 over one lane's kPerLane starts (text bytes wv[0..kWv) little-endian):
// bit k set <=> start k may match.
//  kind 1 (d = 4): word = hi32(x * M) & mask, bits 31 - (byte k+j & 31) for
//    j = 3, 2, 1: a rotate left by byte k+j (the funnel shift takes its
//    amount mod 32, so the 4-gram at k+j serves as the amount) brings each
//    tested bit to bit 31 and a funnel shift appends it to the mask.
//  kind 0 (d < 4): generic d-gram bit index.
__device__ __forceinline__ uint32_t lds_abs(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint2 lds64_abs(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
template <int Kind, bool kImm1024 = false>
__device__ __forceinline__ uint32_t filter32(const ScanArgs &a, const uint32_t wv[kWv], const uint32_t ext[3],
                                             uint32_t sW, uint32_t sWmul, uint32_t stride, uint32_t base_lane) {
    uint32_t surv = 0;
    if (Kind == 3) {
        // DNA k-mer filter: 2-bit codes of the lane's 48 bytes (its 32 starts
        // + 15) packed into c[0..2] (byte i's code at bits 2i of the stream);
        // per word: ((w & 0x06060606) * 0x820820) >> 24 gathers the four codes
        // (b >> 1) & 3 into one byte (no carries reach bits 24..31)
        uint32_t c[4];
        c[3] = 0;  // (keys 32..44 need only their low bits, bytes < 48)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            uint32_t pk[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int j = 4 * q + t;
                const uint32_t w = j < kWv ? wv[j] : ext[j - kWv];
                pk[t] = __umulhi((w & 0x06060606u) * 0x820820u, 1u << 8);  // >> 24 on the FMA pipe
            }
            c[q] = pk[0] + pk[1] * 0x100u + pk[2] * 0x10000u + pk[3] * 0x1000000u;
        }
        // keys of starts 0..kPerLane+12 (the low bits of key k+8 / k+13 are
        // bases 8-10 / 13-15 of start k: its second and third bit positions)
        uint32_t key[kPerLane + 14];
#pragma unroll
        for (int k = 0; k < kPerLane + 14; ++k)
            key[k] = (k & 15) ? __funnelshift_r(c[k >> 4], c[(k >> 4) + 1], 2 * (k & 15)) : c[k >> 4];
        const uint32_t mask = sWmul, t = stride;  // (the word mask and the lane's copy term, as kind 1)
        uint32_t acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int k = kPerLane - 1; k >= 0; --k) {
            const uint32_t off = (__umulhi(key[k], kFilterMul) & mask) ^ t;
            PFAC_CHECK(off < (a.filter_words * 4u << a.rep_log2));
            uint32_t w;
            if (kImm1024)
                asm("ld.shared.u32 %0, [%1+1024];" : "=r"(w) : "r"(off));
            else
                asm("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(off + base_lane));
            // rotate by the keys of starts k, k+8, k+13 (funnel amounts are mod 32): tested bits -> 31
            const uint32_t r = __funnelshift_l(w, w, key[k]) & __funnelshift_l(w, w, key[k + 8]) &
                               __funnelshift_l(w, w, key[k + 13]);
            acc[k >> 3] = __funnelshift_l(r, acc[k >> 3], 1);  // acc << 1 | bit
        }
        surv = acc[0] | (acc[1] << 8) | (acc[2] << 16) | (acc[3] << 24);
    } else if (Kind == 4) {
        // 8-gram blocked two-bit filter: block = top bits of the 32-bit hash
        // x(k) * M + x(k+4) * M2 of bytes k..k+7; bits 31-(byte k & 31) and
        // 31-(byte k+4 & 31) (rotate by the bytes: amounts are mod 32)
        uint32_t x[kPerLane + 5];
#pragma unroll
        for (int k = 0; k < kPerLane + 5; ++k) {
            const int j = k >> 2;
            const uint32_t w0 = j < kWv ? wv[j] : ext[j - kWv];
            const uint32_t w1 = j + 1 < kWv ? wv[j + 1] : ext[j + 1 - kWv];
            x[k] = (k & 3) ? __funnelshift_r(w0, w1, 8 * (k & 3)) : w0;
        }
        uint32_t acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int k = kPerLane - 1; k >= 0; --k) {
            const uint32_t h = x[k] * kFilterMul + x[k + 4] * kFilterMul2;
            const uint32_t blk = __umulhi(h, sWmul);
            const uint2 w2 = lds64_abs(blk * stride + base_lane);
            const uint32_t r = __funnelshift_l(w2.x, w2.x, x[k]) & __funnelshift_l(w2.y, w2.y, x[k + 4]);
            acc[k >> 3] = __funnelshift_l(r, acc[k >> 3], 1);
        }
        surv = acc[0] | (acc[1] << 8) | (acc[2] << 16) | (acc[3] << 24);
    } else if (Kind == 2) {
        // pair filter: one 32-bit word per start pair (k, k+1), chosen by the
        // three shared bytes k+1..k+3 (x[k+1] * (M << 8) drops byte k+4)
        constexpr uint32_t kMul = kFilterMul << 8;
        uint32_t x[kPerLane + 1];
#pragma unroll
        for (int k = 0; k < kPerLane + 1; ++k)
            x[k] = (k & 3) ? __funnelshift_r(wv[k >> 2], wv[(k >> 2) + 1], 8 * (k & 3)) : wv[k >> 2];
        uint32_t acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int k = kPerLane - 2; k >= 0; k -= 2) {
            const uint32_t blk = __umulhi(x[k + 1] * kMul, sWmul);
            const uint32_t w = lds_abs(blk * stride + base_lane);
            const uint32_t b4 = (k + 4 <= kPerLane) ? x[k + 4] : (wv[kWv - 1] >> 16);  // byte k+4 in the low bits
            const uint32_t rb = __funnelshift_l(w, w, b4);    // start k+1: bit 31-(byte k+4 & 31)
            const uint32_t ra = __funnelshift_l(w, w, x[k]);  // start k:   bit 31-(byte k & 31)
            acc[k >> 3] = __funnelshift_l(ra, __funnelshift_l(rb, acc[k >> 3], 1), 1);
        }
        surv = acc[0] | (acc[1] << 8) | (acc[2] << 16) | (acc[3] << 24);
        static_assert(kPerLane <= 32, "");
    } else if (Kind == 1) {
        // blocked three-bit filter in 32-bit words (image.h): one IMAD.HI
        // (hi32(x * M) & mask = the word's byte offset), one LOP3 (& mask,
        // ^ the lane's copy term: copy r sits at r * filter bytes with its
        // words swizzled by r, so lanes reading different copies of a word hit
        // different banks), one LDS (the filter's shared-window base as the
        // immediate offset when it is 0x400), three rotates by bytes k+3, k+2,
        // k+1 (funnel amounts are mod 32: the tested bits -> bit 31), one LOP3,
        // one funnel shift into the mask
        uint32_t x[kPerLane + 3];
#pragma unroll
        for (int k = 0; k < kPerLane + 1; ++k)
            x[k] = (k & 3) ? __funnelshift_r(wv[k >> 2], wv[(k >> 2) + 1], 8 * (k & 3)) : wv[k >> 2];
        x[kPerLane + 1] = x[kPerLane - 1] >> 16;  // byte kPerLane+1 in the low bits
        x[kPerLane + 2] = x[kPerLane - 1] >> 24;  // byte kPerLane+2
        const uint32_t mask = sWmul, t = stride;  // (kind 1: the word mask and the lane's copy term)
        uint32_t acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int k = kPerLane - 1; k >= 0; --k) {
            const uint32_t off = (__umulhi(x[k], kFilterMul) & mask) ^ t;
            PFAC_CHECK(off < (a.filter_words * 4u << a.rep_log2));
            uint32_t w;
            if (kImm1024)
                asm("ld.shared.u32 %0, [%1+1024];" : "=r"(w) : "r"(off));
            else
                asm("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(off + base_lane));
            const uint32_t r = __funnelshift_l(w, w, x[k + 3]) & __funnelshift_l(w, w, x[k + 2]) &
                               __funnelshift_l(w, w, x[k + 1]);
            acc[k >> 3] = __funnelshift_l(r, acc[k >> 3], 1);  // acc << 1 | bit
        }
        surv = acc[0] | (acc[1] << 8) | (acc[2] << 16) | (acc[3] << 24);
    } else {
        const uint32_t gram = a.t.gram;
        const uint32_t kmask = (1u << (8 * gram)) - 1u;
#pragma unroll
        for (int k = kPerLane - 1; k >= 0; --k) {
            const uint32_t x = __funnelshift_r(wv[k >> 2], wv[(k >> 2) + 1], 8 * (k & 3)) & kmask;
            const uint32_t h = filter_index(x, a.t.log2_bits, a.t.exact);
            const uint32_t word = lds_abs((h >> 5) * stride + base_lane);
            surv = (surv << 1) | ((word >> (h & 31)) & 1u);
        }
    }
    return surv;
}

// Walk the queued starts dpos[0, n) (offsets from the CTA's first start,
// position order) with full warps, text from global memory (L2: it was
// streamed moments ago); hits are appended to the warp's hit list in the same
// order and their pid counts added to their rounds' counts.  Returns the new
// hit count.
// The filter key of the start at slot offset off (the slot holds 16 bytes
// past the round, so the 16 DNA bytes are always in it): kind 3 the 16-base
// DNA key, else the first 4 bytes.
// (slot: the slot's 32-bit shared address)
template <int Kind>
__device__ __forceinline__ uint32_t slot_key(uint32_t slot, uint32_t off) {
    const uint32_t wa = slot + (off & ~3u);
    const uint32_t sh = 8 * (off & 3);
    if (Kind == 3) {
        uint32_t w[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) w[q] = lds32q(wa + 4 * q);
        uint32_t key = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t x = __funnelshift_r(w[q], w[q + 1], sh);
            key |= __umulhi((x & 0x06060606u) * 0x820820u, 1u << 8) << (8 * q);
        }
        return key;
    }
    return __funnelshift_r(lds32q(wa), lds32q(wa + 4), sh);
}
// Probe the exact key set for a key (image.h: buckets of 4 slots, one
// 16-byte load each): present if a slot holds the key, absent if a slot is
// empty, else the next bucket (rare at load <= 1/4).
__device__ __forceinline__ bool kset_probe(const ScanArgs &a, uint32_t key) {
    const uint32_t bmask = (1u << (a.t.kset_log2 - 2u)) - 1u;
    const uint4 *k4 = reinterpret_cast<const uint4 *>(a.t.kset);
    const uint32_t e = a.t.kset_empty;
    for (uint32_t b = kset_bucket(key, a.t.kset_log2);; b = (b + 1u) & bmask) {
        PFAC_CHECK(b <= bmask);
        const uint4 q = __ldg(k4 + b);
        if ((q.x == key) | (q.y == key) | (q.z == key) | (q.w == key)) return true;
        if ((q.x == e) | (q.y == e) | (q.z == e) | (q.w == e)) return false;
    }
}

// The entry of a start's key (image.h; kind 4: its first 8 bytes, kind 3:
// its 16-base DNA key): its node and depth, or node 0 when no pattern begins
// with them.
__device__ __forceinline__ uint2 entry_find(const ScanArgs &a, uint32_t x0, uint32_t x1) {
    const uint32_t mask = (1u << a.t.entry_log2) - 1u;
    for (uint32_t i = entry_slot(x0, x1, a.t.entry_log2);; i = (i + 1) & mask) {
        PFAC_CHECK(i <= mask);
        const uint4 e = __ldg(a.t.entry + i);
        if (e.z == kNone) return make_uint2(0u, 0u);
        if (e.x == x0 && e.y == x1) return make_uint2(e.z, e.w);
    }
}

// The shared-memory views of the trie tables (the kernel's layout, ScanArgs).
template <bool kCl>
__device__ __forceinline__ Smem make_smem(const ScanArgs &a) {
    extern __shared__ __align__(128) uint8_t smem_base[];
    Smem s;
    // terminal tables: shared-memory copies when staged (generic pointers)
    s.out_ptr = a.off_terms ? reinterpret_cast<const uint32_t *>(smem_base + a.off_terms) : a.t.out_ptr;
    const uint32_t sb = kCl ? smem_u32(smem_base) : kSmemBase;  // (see kSmemBase)
    s.root = sb + a.off_root;
    s.bm = sb + a.off_bm;
    s.node = sb + a.off_node;
    s.aux = sb + a.off_aux;
    s.label = sb + a.off_label;
    s.tails = sb + a.off_tails;
    s.tail_bytes = sb + a.off_tbytes;
    return s;
}

// Deferred starts are decided in two ways:
//  * direct (kinds 0 and 2, kind 1 without the key set, kinds 3/4 without
//    the entry table): every queued start is walked from the root;
//  * two-level (kind 1 with the exact key set, kinds 3/4 with the entry
//    table): every queued start is first probed in its L2-resident table by
//    a full warp; the survivors join the warp's walk queue in position order
//    (with the entry node and depth to walk from) and are walked 32 at a time
//    by the full warp, so a walk never runs with a lane or two of 32.
constexpr uint32_t kEntShift = 27;  // walk-queue entry word: node | depth << 27 (0 = from the root)

template <int Kind>
__device__ __forceinline__ bool two_level(const ScanArgs &a) {
    return (Kind == 1 && a.use_kset) || ((Kind == 3 || Kind == 4) && a.use_entry);
}

// Probe of one start (two-level kinds): kNone when no pattern can start
// here, else the walk-queue entry word.
template <int Kind>
__device__ __forceinline__ uint32_t probe_start(const ScanArgs &a, const GlobalText &gt, uint32_t key) {
    if (Kind == 1) return kset_probe(a, key) ? 0u : kNone;
    if (Kind == 4) {  // enter at depth <= 8 through the entry table (a miss: no pattern starts here)
        if (gt.end < kGram8) return kNone;
        const uint2 en = entry_find(a, gt.at4(0), gt.at4(4));
        return en.x ? en.x | en.y << kEntShift : kNone;
    }
    if (Kind == 3) {  // enter at depth <= 16 when the 16 bytes are A/C/G/T (the key
                      // aliases other bytes, and no DNA pattern can cover those)
        if (gt.end < kDnaGram) return kNone;
        uint32_t k = 0, w16[4];
        bool acgt = true;
        gt.at16(0, w16);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t w = w16[q];
            const uint32_t c = (w >> 1) & 0x03030303u;  // the four 2-bit codes, one per byte
            const uint32_t sel = (c & 0xFu) | ((c >> 4) & 0xF0u) | ((c >> 8) & 0xF00u) | ((c >> 12) & 0xF000u);
            acgt &= __byte_perm(0x47544341u, 0u, sel) == w;  // code -> 'A','C','T','G'
            k |= __umulhi((w & 0x06060606u) * 0x820820u, 1u << 8) << (8 * q);
        }
        if (!acgt) return kNone;
        const uint2 en = entry_find(a, k, 0u);
        return en.x ? en.x | en.y << kEntShift : kNone;
    }
    return 0u;
}

// Walk starts bpos[0, m) (m <= 32; bent = where each walk enters, 0: from
// the root; both 32-bit shared addresses of u32 arrays) with the warp, text from global memory (L2: streamed moments ago); hits are appended
// to the warp's hit list in the same (position) order and their pid counts
// added to the lane's block rows or their round's count.  Returns the new hit
// count.
template <int Kind, bool kCl>
__device__ __forceinline__ uint32_t walk_batch(const ScanArgs &a, const Smem &s_in, uint64_t cta_lo,
                                               uint64_t cta_round0, uint32_t ctg_bytes, uint32_t bpos,
                                               uint32_t bent, uint32_t m, uint2 *hits, uint32_t n_hits,
                                               unsigned long long &rows) {
    const int lane = threadIdx.x & 31;
    // kind 1 builds its shared-memory views here (its walks are rare: C4
    // -4.5%); the walk-heavy kinds take them from the flush (C3 -17%)
    const Smem s = Kind == 1 ? make_smem<kCl>(a) : s_in;
    uint32_t p = 0, tn = kNone;
    if ((uint32_t)lane < m) {
        p = lds32q(bpos + 4u * lane);
        const uint32_t ent = bent ? lds32q(bent + 4u * lane) : 0u;
        const uint64_t gp = cta_lo + p;
        const GlobalText gt{a.text + gp, clamp32(a.readable - gp), a.aligned};
        tn = ent ? walk<Kind != 1, kCl>(a, s, gt, 0u, ent & ((1u << kEntShift) - 1u), ent >> kEntShift)
                 : walk<Kind != 1, kCl>(a, s, gt, 0u);
        if (tn != kNone) {
            PFAC_CHECK(tn < a.t.n_terminals);
            const uint32_t cnt = s.out_ptr[tn + 1] - s.out_ptr[tn];
            PFAC_CHECK(s.out_ptr[tn + 1] <= a.t.n_out);
            PFAC_CHECK(p < ctg_bytes || cta_round0 + (p >> kRoundLog2) < (a.n_starts + kRound - 1) / kRound);
            if (p < ctg_bytes) rows += cnt;  // the lane's rows in its warp's block (per-warp totals)
            else atomicAdd(a.round_val + cta_round0 + (p >> kRoundLog2), (unsigned long long)cnt);  // dynamic round
        }
    }
    const bool hit = tn != kNone;
    const uint32_t hb = __ballot_sync(0xffffffffu, hit);
    if (hit) {
        const uint32_t idx = n_hits + __popc(hb & ((1u << lane) - 1u));
        if (idx < a.hit_cap) hits[idx] = make_uint2(p, tn);
    }
    return n_hits + __popc(hb);
}

struct FlushOut {
    uint32_t n_hits;  // hit records produced so far
    uint32_t nb;      // walk-queue entries left
    uint32_t rows;    // this lane's rows added in its warp's block
};

// Decide the queued starts dpos[0, n) (position order; dkey = kind-1 keys).
// Two-level kinds move the probe survivors to the walk queue (bpos, bent, nb
// entries) and walk it whenever it holds 32; `final` also walks the rest.
// (The queues are given by their 32-bit shared addresses.)
// Not inlined: its registers do not weigh on the scan loop (it runs once per
// few rounds).
template <int Kind, bool kCl>
__device__ __forceinline__ FlushOut flush_deferred(const ScanArgs *ap, uint64_t cta_lo, uint64_t cta_round0,
                                                uint32_t ctg_bytes, uint32_t dpos, uint32_t dkey,
                                                uint32_t n, uint32_t bpos, uint32_t bent, uint32_t nb, bool final,
                                                uint2 *hits, uint32_t n_hits) {
    const ScanArgs &a = *ap;
    const Smem s = Kind == 1 ? Smem{} : make_smem<kCl>(a);  // (see walk_batch)
    const int lane = threadIdx.x & 31;
    unsigned long long rows = 0;
    __syncwarp();
    if (!two_level<Kind>(a)) {  // direct: walk every queued start
        for (uint32_t j0 = 0; j0 < n; j0 += 32)
            n_hits = walk_batch<Kind, kCl>(a, s, cta_lo, cta_round0, ctg_bytes, dpos + 4u * j0, 0u, min(32u, n - j0), hits,
                                      n_hits, rows);
        __syncwarp();
        return FlushOut{n_hits, 0u, (uint32_t)rows};
    }
    for (uint32_t j0 = 0; j0 < n; j0 += 32) {
        const uint32_t j = j0 + lane;
        uint32_t p = 0, ent = kNone;
        if (j < n) {
            p = lds32q(dpos + 4u * j);
            const uint64_t gp = cta_lo + p;
            const GlobalText gt{a.text + gp, clamp32(a.readable - gp), a.aligned};
            ent = probe_start<Kind>(a, gt, Kind == 1 ? lds32q(dkey + 4u * j) : 0u);
        }
        const uint32_t kb = __ballot_sync(0xffffffffu, ent != kNone);
        if (ent != kNone) {
            const uint32_t idx = nb + __popc(kb & ((1u << lane) - 1u));
            PFAC_CHECK(idx < kWalkQ);
            sts32(bpos + 4u * idx, p);
            if (Kind != 1) sts32(bent + 4u * idx, ent);
        }
        nb += __popc(kb);
        if (nb >= 32) {  // walk the first 32, keep the rest (< 32) at the front
            __syncwarp();
            n_hits = walk_batch<Kind, kCl>(a, s, cta_lo, cta_round0, ctg_bytes, bpos, Kind == 1 ? 0u : bent, 32u,
                                      hits, n_hits, rows);
            uint32_t rp = 0, re = 0;
            const bool mv = (uint32_t)lane + 32u < nb;
            if (mv) {
                rp = lds32q(bpos + 4u * (lane + 32));
                if (Kind != 1) re = lds32q(bent + 4u * (lane + 32));
            }
            __syncwarp();
            if (mv) {
                sts32(bpos + 4u * lane, rp);
                if (Kind != 1) sts32(bent + 4u * lane, re);
            }
            nb -= 32;
            __syncwarp();
        }
    }
    if (final && nb) {
        __syncwarp();
        n_hits = walk_batch<Kind, kCl>(a, s, cta_lo, cta_round0, ctg_bytes, bpos, Kind == 1 ? 0u : bent, nb, hits,
                                  n_hits, rows);
        nb = 0;
    }
    __syncwarp();
    return FlushOut{n_hits, nb, (uint32_t)rows};
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// kCl: launched in thread-block clusters (PFAC_PLACE_CLUSTER): the shared
// window address carries the CTA's rank bits, so it is read, not assumed
template <int Kind, int kSlots, bool kCl = false>
__global__ void __launch_bounds__(kThreads, 1) pfac_scan_kernel(const __grid_constant__ ScanArgs a) {
    // the shared round pool (cross-CTA balance) is planned only for kinds
    // whose tries may live outside shared memory; the pair-filter kernel
    // (small sets, staged tries) is built without it
    constexpr bool kPool = Kind != 2;
    extern __shared__ __align__(128) uint8_t smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t *s_filter = reinterpret_cast<uint32_t *>(smem);
    uint32_t *s_root = reinterpret_cast<uint32_t *>(smem + a.off_root);
    uint32_t *s_node = reinterpret_cast<uint32_t *>(smem + a.off_node);
    uint8_t *s_label = smem + a.off_label;
    constexpr WarpLayout WL = warp_layout(Kind, kSlots);
    if (!kCl && smem_u32(smem) != kSmemBase) __trap();  // (see kSmemBase)
    const uint32_t sb = kCl ? smem_u32(smem) : kSmemBase;
    // this warp's region: its 32-bit shared address
    const uint32_t wss = sb + a.off_warps + (uint32_t)warp * WL.bytes;
    unsigned long long *s_wtot = reinterpret_cast<unsigned long long *>(smem + a.off_warp);  // [kWarps + 2]
    uint32_t *s_bm = reinterpret_cast<uint32_t *>(smem + a.off_bm);

    STAMP(0);
    // ---- barriers: per-warp text ring + one for the table staging; thread 0
    // starts the table copies (TMA bulk, evict-last) before anything else
    uint64_t *sbar = reinterpret_cast<uint64_t *>(smem + a.off_sbar);
    if (tid == 0) {
        mbar_init(sbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint64_t pl = evict_last_policy();
        const uint32_t nb_node = align16(4 * (a.hot_nodes + 1)), nb_label = align16(a.hot_edges),
                       nb_l1 = align16(40 * a.n_level1);
        const uint32_t nb_t = 16 * a.hot_tails, nb_tb = align16(a.hot_tail_bytes);
        const uint32_t nb_f = a.rep_log2 == 0 ? align16(4 * a.filter_words) : 0u;  // one copy: a bulk copy too
        const uint32_t nb_pair = a.use_pair ? 8192u : 0u;
        // cluster placement: this CTA's slice of the node records
        uint32_t nb_dsm = 0, dsm0 = 0;
        if (kCl && a.dsm_nodes) {
            uint32_t q;
            asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(q));
            dsm0 = q << a.dsm_log2;
            nb_dsm = dsm0 < a.dsm_nodes ? 16u * min(1u << a.dsm_log2, a.dsm_nodes - dsm0) : 0u;
        }
        mbar_arrive_expect_tx(sbar, 1024 + nb_pair + 2 * nb_node + nb_label + nb_l1 + nb_t + nb_tb + nb_f + nb_dsm);
        if (nb_dsm) bulk_g2s(smem + a.off_dsm, a.t.rec + dsm0, nb_dsm, sbar, pl);
        if (nb_pair) bulk_g2s(smem + a.off_pair, a.t.pair, nb_pair, sbar, pl);
        if (nb_f) bulk_g2s(s_filter, a.t.filter, nb_f, sbar, pl);
        bulk_g2s(s_root, a.t.root, 1024, sbar, pl);
        bulk_g2s(s_node, a.t.node, nb_node, sbar, pl);
        bulk_g2s(smem + a.off_aux, a.t.aux, nb_node, sbar, pl);  // aux words [0, H] (same size)
        if (nb_label) bulk_g2s(s_label, a.t.label, nb_label, sbar, pl);
        bulk_g2s(s_bm, a.t.level1, nb_l1, sbar, pl);
        if (nb_t) bulk_g2s(smem + a.off_tails, a.t.tails, nb_t, sbar, pl);
        if (nb_tb) bulk_g2s(smem + a.off_tbytes, a.t.tail_bytes, nb_tb, sbar, pl);
    }
    if (lane < kSlots)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(wss + WL.bars + 8u * lane), "r"(1) : "memory");
    uint32_t *s_next = reinterpret_cast<uint32_t *>(s_wtot + kWarps + 1);  // round counter of the CTA (phase 1;
                                                                            // then s_wtot[kWarps + 1])
    if (tid == 32) *s_next = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();  // barriers initialised
    STAMP(11);
    const Smem s = make_smem<kCl>(a);
    // filter addressing: kinds 0, 2, 4: copies interleaved at the unit the
    // kernel loads (8-byte block b of copy r at filter + 8*(b*rep + r); word
    // w of copy r at filter + 4*(w*rep + r)); kinds 1, 3: copy r at filter +
    // r * filter bytes, word w of it at position w ^ r.  Lane l reads copy
    // l % rep, so the lanes of a phase spread over the banks.
    const uint32_t rep = 1u << a.rep_log2;
    constexpr bool kBlock64 = Kind == 4;                // 64-bit blocks
    constexpr bool kWordSwz = Kind == 1 || Kind == 3;   // 32-bit words, swizzled copies
    const uint32_t unit = kBlock64 ? 8u : 4u;
    const uint32_t sW = 32u - (a.t.log2_bits - (kBlock64 ? 6u : 5u));  // block index = hash >> sW
    const uint32_t lane_copy = (uint32_t)lane & (rep - 1u);
    const uint32_t fbytes = a.filter_words * 4u;
    // kind 1: (word mask, copy term) in the (sWmul, stride) slots of filter32
    const uint32_t sWmul = kWordSwz ? (fbytes - 1u) & ~3u : 1u << (32u - sW);  // (hash * sWmul) >> 32 == hash >> sW
    const uint32_t stride = kWordSwz ? (lane_copy * fbytes) | (lane_copy * 4u) : rep * unit;
    const uint32_t base_lane = sb + (kWordSwz ? 0u : lane_copy * unit);
    static_assert(kSmemBase == 1024u, "filter32's immediate");  // word kinds: the base is the LDS immediate

    const uint64_t policy = evict_first_policy();
    // starts < lim are valid: inside [0, n_starts) and their d-gram fits
    const uint32_t gram = a.t.gram;
    const uint64_t lim = (a.readable + 1 >= gram && a.readable + 1 - gram < a.n_starts) ? a.readable + 1 - gram
                                                                                        : a.n_starts;
    // ---- this CTA's contiguous range of rounds
    const uint32_t gw = blockIdx.x * kWarps + warp;
    const uint64_t n_rounds = (a.n_starts + kRound - 1) / kRound;
    const uint64_t cta_round0 = (uint64_t)blockIdx.x * a.rounds_per_cta < a.n_main
                                    ? (uint64_t)blockIdx.x * a.rounds_per_cta : a.n_main;
    const uint32_t n_local = (uint32_t)((cta_round0 + a.rounds_per_cta < a.n_main ? cta_round0 + a.rounds_per_cta
                                                                                  : a.n_main) - cta_round0);
    // the shared pool (the text's last rounds, taken by any warp once its
    // CTA's range is done: cross-CTA balance) in the CTA's local round
    // numbering: [pool_lo, pool_hi) (start offsets stay 32-bit: planned so;
    // recomputed where used: no registers held through phase 1)
    const uint64_t cta_lo = cta_round0 * kRound;
    uint2 *hits = a.hits + (uint64_t)gw * a.hit_cap;

    // local rounds r < n_fast have their whole slot (round + overhang) readable
    const uint32_t n_fast = !a.aligned || a.readable < cta_lo + kSlotBytes
                                ? 0u
                                : (uint32_t)min((uint64_t)n_local, (a.readable - cta_lo - kSlotBytes) / kRound + 1);
    // The CTA's first n_ctg rounds are split into contiguous per-warp blocks
    // (warp w owns [wbeg, wend); its rows follow the CTA's earlier warps'
    // rows, so per-warp totals order them); the rest are handed out from the
    // CTA's shared counter (dynamic: warps whose walks ran long take fewer;
    // those rounds keep per-round counts and record their owner).  The warp's
    // rounds increase; warp-uniform; kNoRound when none is left.
    const uint32_t n_ctg = (uint32_t)(((uint64_t)n_local * a.ctg64) >> 6);
    uint32_t taken = 0;
    const uint32_t wq = n_ctg / kWarps, wrem = n_ctg % kWarps;
    const uint32_t wbeg = warp * wq + min((uint32_t)warp, wrem), wend = wbeg + wq + ((uint32_t)warp < wrem ? 1u : 0u);
    uint32_t wnext = wbeg;  // the warp's next block round
    auto take = [&]() -> uint32_t {
        uint32_t r;
        if (wnext < wend) {
            r = wnext++;
        } else {
            r = 0;
            if (lane == 0) {
                asm volatile("atom.shared.add.u32 %0, [%1], 1;"
                             : "=r"(r)
                             : "r"(sb + a.off_warp + 8u * (kWarps + 1))
                             : "memory");
            }
            r = n_ctg + __shfl_sync(0xffffffffu, r, 0);
            if (r >= n_local) {  // the CTA's range is done: a pool round, if any is left
                r = kNoRound;
                if (kPool && a.pool_seg) {
                    if (lane == 0) {
                        const uint32_t q = atomicAdd(&a.ws->pool_next, 1u);
                        if (q < (uint32_t)((a.n_starts + kRound - 1) / kRound - a.n_main)) {
                            r = (uint32_t)(a.n_main - cta_round0) + q;
                            a.round_val[cta_round0 + r] = 0ull;  // its count (ordered before the warp's
                                                                 // walks by their __syncwarp)
                        }
                    }
                    r = __shfl_sync(0xffffffffu, r, 0);
                }
            }
            // the owner of a dynamic round is recorded (phase 3's re-scan fallback)
            if (lane == 0 && r != kNoRound) a.round_owner[cta_round0 + r] = gw;
        }
        ++taken;
        return r;
    };
    // Fill ring slot `slot` with local round r: one TMA bulk copy of the
    // readable 16-byte-aligned part; the lanes copy the rest (the text's last
    // bytes, zero-filled past `readable`, or everything when the text pointer
    // is not 16-byte aligned), all loads issued before the stores.
    auto issue = [&](uint32_t r, uint32_t slot) {
        const uint32_t dst = wss + WL.ring + slot * kSlotBytes, bar = wss + WL.bars + 8u * slot;
        if (r < n_fast) {  // the whole slot is readable and aligned: one bulk copy
            if (lane == 0) {
                fence_proxy_async_smem();  // prior generic accesses of the slot precede the async write
                mbar_arrive_expect_tx_s(bar, kSlotBytes);
                bulk_g2s_s(dst, a.text + cta_lo + (uint64_t)r * kRound, kSlotBytes, bar, policy);
            }
            return;
        }
        const uint64_t lo = cta_lo + (uint64_t)r * kRound;
        const uint32_t avail = lo < a.readable ? (uint32_t)min(a.readable - lo, (uint64_t)kSlotBytes) : 0u;
        const uint32_t nbulk = a.aligned ? (avail & ~15u) : 0u;
        if (nbulk < (uint32_t)kSlotBytes) {  // cold: only the text's last round(s) / unaligned text
#pragma unroll 1
            for (uint32_t o0 = nbulk; o0 < (uint32_t)kSlotBytes; o0 += 8 * 32) {  // 8 loads in flight per lane
                uint32_t v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t o = o0 + lane + 32 * q;
                    v[q] = o < avail ? (uint32_t)__ldg(a.text + lo + o) : 0u;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t o = o0 + lane + 32 * q;
                    if (o < (uint32_t)kSlotBytes)
                        asm volatile("st.shared.u8 [%0], %1;" ::"r"(dst + o), "r"(v[q]) : "memory");
                }
            }
            __syncwarp();
        }
        if (lane == 0) {
            if (nbulk) {
                fence_proxy_async_smem();  // prior generic accesses of the slot precede the async write
                mbar_arrive_expect_tx_s(bar, nbulk);
                bulk_g2s_s(dst, a.text + lo, nbulk, bar, policy);
            } else {
                mbar_arrive_s(bar);
            }
        }
    };

    // ---- stage the tables (TMA bulk copies of the image sections; the
    // filter is replicated from 8/4-byte loads), then start streaming
    STAMP(12);
    {   // replicate the filter: destination unit j holds source unit j >> rep_log2
        // (consecutive threads write consecutive units: no bank conflicts)
        // (8-16 loads in flight per thread: the image is cold in L2 here)
        const uint32_t nu = a.rep_log2 == 0 ? 0u : (kBlock64 ? a.filter_words / 2 : a.filter_words) << a.rep_log2;
        if (kWordSwz) {  // copy r = j / words, position p = j % words holds word p ^ r
            const uint32_t lw = (uint32_t)__ffs(a.filter_words) - 1u;
            for (uint32_t j0 = 0; j0 < nu; j0 += 16 * kThreads) {
                uint32_t v[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const uint32_t j = j0 + tid + q * kThreads;
                    v[q] = j < nu ? __ldg(a.t.filter + ((j & (a.filter_words - 1u)) ^ (j >> lw))) : 0u;
                }
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (j0 + tid + q * kThreads < nu) s_filter[j0 + tid + q * kThreads] = v[q];
            }
        } else if (kBlock64) {
            const uint2 *src = reinterpret_cast<const uint2 *>(a.t.filter);
            uint2 *d = reinterpret_cast<uint2 *>(s_filter);
            for (uint32_t j0 = 0; j0 < nu; j0 += 8 * kThreads) {
                uint2 v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t j = j0 + tid + q * kThreads;
                    v[q] = j < nu ? __ldg(src + (j >> a.rep_log2)) : make_uint2(0, 0);
                }
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (j0 + tid + q * kThreads < nu) d[j0 + tid + q * kThreads] = v[q];
            }
        } else {
            for (uint32_t j0 = 0; j0 < nu; j0 += 16 * kThreads) {
                uint32_t v[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const uint32_t j = j0 + tid + q * kThreads;
                    v[q] = j < nu ? __ldg(a.t.filter + (j >> a.rep_log2)) : 0u;
                }
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (j0 + tid + q * kThreads < nu) s_filter[j0 + tid + q * kThreads] = v[q];
            }
        }
        // terminal tables (pid-list offsets, kept terminal ids) when small
        if (a.off_terms) {
            uint32_t *so = reinterpret_cast<uint32_t *>(smem + a.off_terms);
            const uint32_t n_op = a.t.n_terminals + 1;
            for (uint32_t j = tid; j < n_op; j += kThreads) so[j] = __ldg(a.t.out_ptr + j);
        }
    }
    STAMP(8);
    for (uint32_t r = n_ctg + tid; r < n_local; r += kThreads) a.round_val[cta_round0 + r] = 0ull;  // pid counts
    __syncthreads();  // the round counter and counts are initialised
    STAMP(9);
    // the first kSlots-1 rounds of this warp (static ones) start streaming
    // (after the table requests: those are on the critical path)
    uint32_t rid[kSlots];
#pragma unroll
    for (int q = 0; q < kSlots - 1; ++q) {
        rid[q] = take();
        if (rid[q] != kNoRound) issue(rid[q], q);
    }
    STAMP(10);
    mbar_wait(sbar, 0);
    STAMP(5);
    __syncthreads();
    if (kCl) cluster_sync_all();  // every CTA's record slice is resident before the first remote read
    // 2-gram prefix table: word (b0, q) bit j <=> the walk from a start with
    // bytes (b0, 32q + j) gets past level 1 (or b0's node already is a
    // terminal / tail start, where every b1 is kept)
    const uint32_t s_pair = sb + a.off_pair;  // (shared address; arrived with the tables)
    STAMP(1);

    // ================================================= phase 1: scan
    // One 1024-start round per iteration; the ring keeps kSlots-1 rounds in
    // flight.  Stage 1 filters each lane's 32 starts (bit mask).  Stage 2
    // tests each survivor, in its lane, against the 2-gram prefix table (the
    // root's children and their level-1 bitmapped nodes): bytes
    // (b0, b1) begin a pattern path, or b0 alone already reaches a terminal
    // or tail.  The few kept starts are queued in position order (lane-major
    // = position order; a warp's rounds increase: a ballot when no lane keeps
    // two, else a warp scan) and walked in full-warp batches to their first
    // mismatch whenever the queue may not take another 32.
    uint32_t n_hits = 0;  // hit records produced (warp-uniform; may exceed hit_cap)
    unsigned long long lane_rows = 0;  // rows of this lane's hits in the warp's block
    uint32_t dcount = 0;  // queued starts (warp-uniform)
    uint32_t nb = 0;      // walk-queue entries (two-level kinds; warp-uniform)
    constexpr uint32_t qcap = defer_cap(Kind);  // queue capacity
    // (32-bit shared addresses of the queues)
    const uint32_t dpos = wss + WL.dpos, dkey = wss + WL.dkey;  // probe queue (+ kind-1 keys)
    const uint32_t bpos = wss + WL.bpos, bent = wss + WL.bent;  // walk queue: positions (+ entry words, kinds 3/4)
    uint32_t slot = 0, phase = 0;  // ring slot of the current round, its mbarrier parity
    for (;;) {
        const bool done = rid[0] == kNoRound;
        const uint32_t rel = rid[0] * (uint32_t)kRound;  // round start relative to cta_lo
        const uint64_t rbase = cta_lo + rel;
        const uint32_t p0 = wss + WL.ring + slot * kSlotBytes;  // the round's slot
        uint32_t pending = 0;
        if (!done) {
            // refill the slot of the previous round with the next round taken
            __syncwarp();  // every lane's reads of that slot precede its refill
            rid[kSlots - 1] = take();
            if (rid[kSlots - 1] != kNoRound) issue(rid[kSlots - 1], slot == 0 ? kSlots - 1 : slot - 1);
            mbar_wait_s(wss + WL.bars + 8u * slot, phase);
#ifdef PFAC_TIMING
            if (taken == kSlots) STAMP(6);  // the first round's text is in
#endif
#ifdef PFAC_STREAM_ONLY
            if (lds8q(p0 + lane) == 0xFF && a.pos_base == ~0ull) n_hits++;  // keeps the loads
#else
            // ---- stage 1: filter over the lane's 32 starts (its 32 bytes: two
            // 16-byte loads; the 2-way bank conflict of the 32-byte stride costs
            // less than un-swizzling in registers)
            uint32_t wv[kWv];
            {
                const uint4 h0 = lds128q(p0 + lane * kPerLane);
                const uint4 h1 = lds128q(p0 + lane * kPerLane + 16);
                wv[0] = h0.x;
                wv[1] = h0.y;
                wv[2] = h0.z;
                wv[3] = h0.w;
                wv[4] = h1.x;
                wv[5] = h1.y;
                wv[6] = h1.z;
                wv[7] = h1.w;
            }
            const uint32_t w8 = __shfl_down_sync(0xffffffffu, wv[0], 1);
            wv[kWv - 1] = lane == 31 ? lds32q(p0 + kRound) : w8;
            uint32_t ext[3] = {0, 0, 0};  // kind 3: the next 12 bytes (the slot holds 16 past the round)
            if (Kind == 3 || Kind == 4) {
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const uint32_t e = __shfl_down_sync(0xffffffffu, wv[q + 1], 1);
                    ext[q] = lane == 31 ? lds32q(p0 + kRound + 4 + 4 * q) : e;
                }
            }
            pending = filter32<Kind, kWordSwz && !kCl>(a, wv, ext, sW, sWmul, stride, base_lane);
            const uint64_t lbase = rbase + (uint64_t)lane * kPerLane;
            if (lbase + kPerLane > lim) {
                const uint32_t nvalid = lbase >= lim ? 0u : (uint32_t)(lim - lbase);
                pending &= nvalid >= 32 ? 0xFFFFFFFFu : ((1u << nvalid) - 1u);
            }
#endif
#if defined(PFAC_EXP) && PFAC_EXP == 1
            if (pending == 0xDEADBEEFu && a.pos_base == ~0ull) n_hits++;  // experiment: filter only
            pending = 0;
#endif
            // ---- stage 2 in the lane: 2-gram prefix test of each survivor;
            // `pending` becomes the kept set (sparse: appended by ballot)
            if (Kind != 3 && a.use_pair) {
                const uint32_t rl = rid[0] < n_fast ? (uint32_t)kSlotBytes  // readable bytes from rbase
                                                    : (a.readable > rbase ? clamp32(a.readable - rbase) : 0u);
                uint32_t km = 0;
                for (uint32_t m = pending; m; m &= m - 1) {
                    const uint32_t k = __ffs(m) - 1;
                    const uint32_t off = lane * kPerLane + k;
                    const uint32_t b0 = lds8q(p0 + off);
                    uint32_t keep;
                    if (off + 1 < rl) {
                        const uint32_t b1 = lds8q(p0 + off + 1);  // the slot holds 16 bytes past the round
                        keep = (ldt32(s_pair + 32u * b0 + 4u * (b1 >> 5)) >> (b1 & 31)) & 1u;
                    } else {
                        keep = ldt32(s.root + 4u * b0) != 0u;  // last readable byte: let the walk decide
                    }
                    km |= keep << k;
                }
                pending = km;
            }
            // ---- queue the kept starts in position order (lane-major = position
            // order; a warp's rounds increase): a warp scan of the per-lane
            // counts (a ballot when no lane keeps two) gives each its slots
            uint32_t ex, tot;
            if (__any_sync(0xffffffffu, (pending & (pending - 1)) != 0)) {
                ex = warp_excl_scan(__popc(pending), lane, &tot);
            } else {
                const uint32_t kb = __ballot_sync(0xffffffffu, pending != 0);
                ex = __popc(kb & ((1u << lane) - 1u));
                tot = __popc(kb);
            }
            if (tot) {
                if (dcount + tot > qcap) {  // decide the queued starts first
                    const FlushOut fo = flush_deferred<Kind, kCl>(&a, cta_lo, cta_round0, n_ctg * kRound, dpos, dkey,
                                                             dcount, bpos, bent, nb, false, hits, n_hits);
                    n_hits = fo.n_hits;
                    nb = fo.nb;
                    lane_rows += fo.rows;
                    dcount = 0;
                }
                if (tot <= qcap) {  // the common case: one pass
                    uint32_t e = dcount + ex;
                    for (uint32_t m = pending; m; m &= m - 1, ++e) {
                        PFAC_CHECK(e < qcap);
                        sts32(dpos + 4u * e, rel + lane * kPerLane + (__ffs(m) - 1));
                    }
                    if (Kind == 1 && a.use_kset) {
                        // the keys of the new entries, one per lane (the per-lane loop
                        // above only scatters offsets: it runs max-over-lanes times)
                        __syncwarp();
                        for (uint32_t j = dcount + (uint32_t)lane; j < dcount + tot; j += 32)
                            sts32(dkey + 4u * j, slot_key<Kind>(p0, lds32q(dpos + 4u * j) - rel));
                    }
                    dcount += tot;
                    __syncwarp();
                } else {  // more kept starts than the queue holds (dense matches): qcap at a time
                    for (uint32_t c0 = 0; c0 < tot; c0 += qcap) {
                        uint32_t e = ex;
                        for (uint32_t m = pending; m; m &= m - 1, ++e) {
                            if (e >= c0 && e < c0 + qcap) {
                                const uint32_t off = lane * kPerLane + (__ffs(m) - 1);
                                sts32(dpos + 4u * (e - c0), rel + off);
                                if (Kind == 1 && a.use_kset) sts32(dkey + 4u * (e - c0), slot_key<Kind>(p0, off));
                            }
                        }
                        const FlushOut fo = flush_deferred<Kind, kCl>(&a, cta_lo, cta_round0, n_ctg * kRound, dpos, dkey,
                                                                 min(qcap, tot - c0), bpos, bent, nb, false, hits,
                                                                 n_hits);
                        n_hits = fo.n_hits;
                        nb = fo.nb;
                        lane_rows += fo.rows;
                    }
                }
            }
        } else if (dcount != 0 || nb != 0) {  // the warp's rounds are done: decide everything left
#if defined(PFAC_EXP) && PFAC_EXP == 2
            if (lds32q(dpos) == 0xFFFFFFFFu && a.pos_base == ~0ull) n_hits++;  // experiment: no walks
#else
            const FlushOut fo = flush_deferred<Kind, kCl>(&a, cta_lo, cta_round0, n_ctg * kRound, dpos, dkey, dcount, bpos,
                                                     bent, nb, true, hits, n_hits);
            n_hits = fo.n_hits;
            nb = fo.nb;
            lane_rows += fo.rows;
#endif
            dcount = 0;
        }
        if (done) break;
#pragma unroll
        for (int q = 0; q < kSlots - 1; ++q) rid[q] = rid[q + 1];
        slot = slot + 1 == kSlots ? 0 : slot + 1;
        phase ^= slot == 0;
    }
    STAMP(2);

    // ================================================= phase 2: offsets
    // Exclusive scan of the warps' block totals (a warp's first row relative
    // to the CTA) and of the dynamic rounds' counts after them, in place
    // (round_val becomes the round's first row relative to the CTA), CTA
    // total -> grid barrier -> prefix over the CTA totals.
    __syncthreads();  // every round of the CTA is done (round_val complete)
    unsigned long long run = 0, warp_base = 0;
    {   // per-warp totals: the rows of the CTA's blocks are the warps' rows in warp order
        unsigned long long wt = lane_rows;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) wt += __shfl_xor_sync(0xffffffffu, wt, d);
        if (lane == 0) s_wtot[warp] = wt;
        __syncthreads();
        if (warp == 0) {
            const unsigned long long wv0 = lane < kWarps ? s_wtot[lane] : 0ull;
            unsigned long long wi = wv0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, d);
                if (lane >= d) wi += y;
            }
            if (lane < kWarps) s_wtot[lane] = wi - wv0;
            __syncwarp();
            if (lane == 31) s_wtot[kWarps] = wi;
        }
        __syncthreads();
        warp_base = s_wtot[warp];
        run = s_wtot[kWarps];
        __syncthreads();
    }
    // block-wide exclusive scan of one value per thread (kThreads values)
    auto block_excl = [&](unsigned long long v, unsigned long long &total) -> unsigned long long {
        unsigned long long incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        if (lane == 31) s_wtot[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const unsigned long long wv0 = lane < kWarps ? s_wtot[lane] : 0ull;
            unsigned long long wi = wv0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, d);
                if (lane >= d) wi += y;
            }
            if (lane < kWarps) s_wtot[lane] = wi - wv0;
            __syncwarp();
            if (lane == 31) s_wtot[kWarps] = wi;
        }
        __syncthreads();
        const unsigned long long ex = s_wtot[warp] + incl - v;
        total = s_wtot[kWarps];
        __syncthreads();
        return ex;
    };
    // in place: counts of rounds [g0, g0 + n) -> run0 + their exclusive prefix; returns the end
    auto scan_rounds = [&](uint64_t g0, uint32_t n, unsigned long long run0) -> unsigned long long {
        for (uint32_t b = 0; b < n; b += kThreads) {
            const uint32_t r = b + tid;
            unsigned long long tot;
            const unsigned long long v = r < n ? a.round_val[g0 + r] : 0ull;
            const unsigned long long ex = block_excl(v, tot);
            if (r < n) a.round_val[g0 + r] = run0 + ex;
            run0 += tot;
        }
        return run0;
    };
    run = scan_rounds(cta_round0 + n_ctg, n_local - n_ctg, run);  // the dynamic rounds follow the blocks
    if (tid == 0) a.cta_total[blockIdx.x] = run;
    STAMP(7);
    grid_barrier(a.ws);
    if (blockIdx.x == 0 && tid == 0) a.ws->pool_next = 0u;  // phase 1 is over everywhere: ready for the next launch
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
            s_wtot[kWarps + 1] = all;
            if (blockIdx.x == 0 && !(kPool && a.pool_seg)) *a.out_count = all;
        }
    }
    __syncthreads();
    const uint64_t cta_off = s_wtot[kWarps];  // this CTA's first output row
    // The pool's rows follow every range's: its counts are complete only now.
    // CTA b scans pool segment b in place, a second grid barrier, then every
    // CTA holds each segment's first row (s_pool, in the idle ring).
    unsigned long long *s_pool = reinterpret_cast<unsigned long long *>(smem + a.off_warps);
    const uint32_t pool_lo = (uint32_t)(a.n_main - cta_round0), pool_hi = (uint32_t)(n_rounds - cta_round0);
    if (kPool && a.pool_seg) {
        const unsigned long long all_main = s_wtot[kWarps + 1];
        __syncthreads();
        const uint64_t g0 = a.n_main + (uint64_t)blockIdx.x * a.pool_seg;
        const uint32_t n = g0 < n_rounds ? (uint32_t)min((uint64_t)a.pool_seg, n_rounds - g0) : 0u;
        const unsigned long long seg_total = scan_rounds(g0, n, 0ull);
        if (tid == 0) a.pool_total[blockIdx.x] = seg_total;
        grid_barrier(a.ws);
        unsigned long long pool_all;
        const unsigned long long v = (uint32_t)tid < gridDim.x ? __ldcg(a.pool_total + tid) : 0ull;
        const unsigned long long ex = block_excl(v, pool_all);
        if ((uint32_t)tid < gridDim.x) s_pool[tid] = all_main + ex;
        if (blockIdx.x == 0 && tid == 0) *a.out_count = all_main + pool_all;
        __syncthreads();
    }
    STAMP(3);

    // ================================================= phase 3: emit
    if (n_ctg == n_local && !(kPool && a.pool_seg) && n_hits <= a.hit_cap) {
        // blocks only: the warp's hits are in position order and its rows
        // follow the CTA's earlier warps' rows
        uint64_t run_rows = cta_off + warp_base;
        for (uint32_t b = 0; b < n_hits; b += 32) {
            const uint32_t i = b + lane;
            uint32_t ti = 0, cnt = 0, p = 0;
            if (i < n_hits) {
                const uint2 h = hits[i];
                p = h.x;
                ti = h.y;
                cnt = s.out_ptr[ti + 1] - s.out_ptr[ti];
            }
            uint32_t ctot;
            uint64_t o = run_rows + warp_excl_scan(cnt, lane, &ctot);
            if (cnt) {
                const uint32_t r0 = s.out_ptr[ti];
                for (uint32_t e = 0; e < cnt; ++e, ++o) {
                    if (o < a.capacity) {
                        a.out_pos[o] = a.pos_base + cta_lo + p;
                        a.out_pid[o] = __ldg(a.t.out_pid + r0 + e);
                    }
                }
            }
            run_rows += ctot;
        }
    } else if (n_hits <= a.hit_cap) {
        // the warp's hits are in position order: first those of its block
        // (rows from the warp's base on), then those of its dynamic rounds; a
        // round's hits are consecutive, so a row's index = its segment's first
        // row + rows of the segment's earlier hits (segment = the block, or one
        // dynamic round)
        constexpr uint32_t kBlockSeg = 0xFFFFFFF0u;
        uint64_t carry_run = 0, carry_seg = 0;  // warp-running rows before the batch / before its first segment
        uint32_t carry_round = 0xFFFFFFFFu;
        const uint32_t ctg_bytes = n_ctg * kRound;
        for (uint32_t b = 0; b < n_hits; b += 32) {
            const uint32_t i = b + lane;
            uint32_t ti = 0, cnt = 0, rnd = 0xFFFFFFFEu, p = 0;
            if (i < n_hits) {
                const uint2 h = hits[i];
                p = h.x;
                ti = h.y;
                rnd = p < ctg_bytes ? kBlockSeg : p >> kRoundLog2;
                cnt = s.out_ptr[ti + 1] - s.out_ptr[ti];
            }
            uint32_t ctot;
            const uint64_t ex = carry_run + warp_excl_scan(cnt, lane, &ctot);  // warp-running rows before hit i
            const uint32_t prev = __shfl_up_sync(0xffffffffu, rnd, 1);
            const bool head = lane == 0 ? rnd != carry_round : rnd != prev;
            const uint32_t hm = __ballot_sync(0xffffffffu, head) & (0xFFFFFFFFu >> (31 - lane));
            const int hl = hm ? 31 - __clz(hm) : -1;
            const uint64_t seg_h = __shfl_sync(0xffffffffu, ex, hl < 0 ? 0 : hl);
            const uint64_t seg = hl < 0 ? carry_seg : seg_h;
            if (cnt) {
                uint64_t o = (rnd == kBlockSeg ? cta_off + warp_base
                                               : (rnd >= pool_lo ? s_pool[(rnd - pool_lo) / a.pool_seg] : cta_off) +
                                                     a.round_val[cta_round0 + rnd]) +
                             (ex - seg);
                const uint32_t r0 = s.out_ptr[ti];
                for (uint32_t e = 0; e < cnt; ++e, ++o) {
                    if (o < a.capacity) {
                        a.out_pos[o] = a.pos_base + cta_lo + p;
                        a.out_pid[o] = __ldg(a.t.out_pid + r0 + e);
                    }
                }
            }
            carry_seg = __shfl_sync(0xffffffffu, seg, 31);
            carry_round = __shfl_sync(0xffffffffu, rnd, 31);
            carry_run += ctot;
        }
    } else {
        // hit list overflowed: scan this warp's rounds again (text from global
        // memory), writing rows directly in position order
        uint64_t contig_off = cta_off + warp_base;  // the warp's running row in its block
        // the block's rounds, then the CTA's dynamic rounds and the pool's the warp took
        auto next_round = [&](uint32_t r) -> uint32_t {
            if (r == wend) r = n_ctg;
            if (r == n_local && kPool && a.pool_seg) r = pool_lo;
            return r;
        };
        const uint32_t r_end = kPool && a.pool_seg ? pool_hi : n_local;
        for (uint32_t r = next_round(wbeg); r < r_end; r = next_round(r + 1)) {
            const bool dyn = r >= n_ctg;
            if (dyn && __ldcg(a.round_owner + cta_round0 + r) != gw) continue;
            uint64_t off = dyn ? (r >= pool_lo ? s_pool[(r - pool_lo) / a.pool_seg] : cta_off) +
                                     a.round_val[cta_round0 + r]
                               : contig_off;
            const uint64_t lbase = cta_lo + (uint64_t)r * kRound + (uint64_t)lane * kPerLane;
            uint32_t wv[kWv], ext[3];
#pragma unroll
            for (int q = 0; q < kWv + 3; ++q) {
                uint32_t x = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (lbase + 4 * q + b < a.readable) x |= (uint32_t)__ldg(a.text + lbase + 4 * q + b) << (8 * b);
                if (q < kWv) wv[q] = x; else ext[q - kWv] = x;
            }
            uint32_t surv = filter32<Kind, kWordSwz && !kCl>(a, wv, ext, sW, sWmul, stride, base_lane);
            if (lbase + kPerLane > lim) {
                const uint32_t nvalid = lbase >= lim ? 0u : (uint32_t)(lim - lbase);
                surv &= nvalid >= 32 ? 0xFFFFFFFFu : ((1u << nvalid) - 1u);
            }
            const GlobalText gt{a.text + lbase, clamp32(a.readable - lbase), a.aligned};
            uint32_t cc = 0, hm = 0;
            for (uint32_t m = surv; m; m &= m - 1) {
                const int k = __ffs(m) - 1;
                const uint32_t ti = walk<Kind != 1, kCl>(a, s, gt, (uint32_t)k);
                if (ti != kNone) {
                    cc += s.out_ptr[ti + 1] - s.out_ptr[ti];
                    hm |= 1u << k;
                }
            }
            uint32_t ctot;
            uint64_t o = off + warp_excl_scan(cc, lane, &ctot);
            for (uint32_t m = hm; m; m &= m - 1) {
                const uint32_t k = (uint32_t)(__ffs(m) - 1);
                const uint32_t ti = walk<Kind != 1, kCl>(a, s, gt, k);
                const uint32_t r0 = s.out_ptr[ti], r1 = s.out_ptr[ti + 1];
                for (uint32_t e = r0; e < r1; ++e, ++o) {
                    if (o < a.capacity) {
                        a.out_pos[o] = a.pos_base + lbase + k;
                        a.out_pid[o] = __ldg(a.t.out_pid + e);
                    }
                }
            }
            contig_off += ctot;
        }
    }
    if (kCl) cluster_sync_all();  // no CTA leaves while the others may still read its slice
    STAMP(4);
}

// Kernel instance for a filter kind and ring depth (2 slots only where the
// filter can exceed 64 KiB: kinds 1 and 3).
const void *kernel_for(uint32_t kind, uint32_t slots, bool cluster = false) {
    if (cluster)  // (2-slot ring; the kinds whose tries outgrow one SM)
        return slots != 2    ? nullptr
               : kind == 1 ? (const void *)pfac_scan_kernel<1, 2, true>
               : kind == 3 ? (const void *)pfac_scan_kernel<3, 2, true>
               : kind == 4 ? (const void *)pfac_scan_kernel<4, 2, true>
                           : nullptr;
    if (slots == 2)
        return kind == 1   ? (const void *)pfac_scan_kernel<1, 2>
               : kind == 2 ? (const void *)pfac_scan_kernel<2, 2>
               : kind == 3 ? (const void *)pfac_scan_kernel<3, 2>
               : kind == 4 ? (const void *)pfac_scan_kernel<4, 2>
                           : nullptr;
    switch (kind) {
        case 0: return (const void *)pfac_scan_kernel<0, 3>;
        case 1: return (const void *)pfac_scan_kernel<1, 3>;
        case 2: return (const void *)pfac_scan_kernel<2, 3>;
        case 3: return (const void *)pfac_scan_kernel<3, 3>;
        case 4: return (const void *)pfac_scan_kernel<4, 3>;
        default: return nullptr;
    }
}

struct DeviceInfo {
    bool init = false;
    int sms = 0;
    int max_smem_optin = 0;
};
std::mutex g_dev_mu;
DeviceInfo g_dev[64];

inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

int device_info(int device, DeviceInfo &out, std::string &err) {
    if (device < 0 || device >= 64) {
        err = "bad device ordinal";
        return kStatusInvalid;
    }
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DeviceInfo &di = g_dev[device];
    if (!di.init) {
        cudaError_t e = cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, device);
        if (e == cudaSuccess)
            e = cudaDeviceGetAttribute(&di.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
        for (uint32_t kind = 0; kind < 5 && e == cudaSuccess; ++kind)
            for (uint32_t slots = 2; slots <= 3 && e == cudaSuccess; ++slots)
                for (int cl = 0; cl < 2 && e == cudaSuccess; ++cl)
                    if (const void *fn = kernel_for(kind, slots, cl != 0))
                        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
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

// Launch geometry shared by workspace sizing and the launch itself.  CTA b
// owns rounds [b * rounds_per_cta, (b + 1) * rounds_per_cta); workspace =
// fixed header | round_val[n_rounds] u64 | round_owner[n_rounds] u32 (padded) |
// hit lists [warps][hit_cap] uint2.
struct Geometry {
    uint64_t grid, warps, n_rounds, rounds_per_cta;
    uint32_t hit_cap;
    uint64_t off_owner, off_hits, ws_bytes;
};
Geometry geometry(uint64_t n_starts, int sms) {
    Geometry g;
    g.n_rounds = (n_starts + kRound - 1) / kRound;
    g.grid = (uint64_t)sms;
    if (g.grid * kWarps > g.n_rounds) g.grid = (g.n_rounds + kWarps - 1) / kWarps;
    if (g.grid < 1) g.grid = 1;
    g.warps = g.grid * kWarps;
    g.rounds_per_cta = (g.n_rounds + g.grid - 1) / g.grid;
    if (g.rounds_per_cta < 1) g.rounds_per_cta = 1;
    // hit records per warp: a quarter of its average share of starts (dense-
    // match texts such as C2's paper-shaped variant, a word text with word
    // patterns, hit a third of all positions: with 1/16 the hit lists
    // overflowed into the re-scan path, 7.0 -> 2.75 ms), at least 64, and at
    // most 4096 or what keeps all hit lists within 256 MiB (a warp that finds
    // more re-scans its rounds in phase 3)
    uint64_t cap = ((g.rounds_per_cta + kWarps - 1) / kWarps) * kRound / 4;
    const uint64_t cap_max = std::max<uint64_t>(4096, (256ull << 20) / (8ull * g.warps));
    if (cap < 64) cap = 64;
    if (cap > cap_max) cap = cap_max;
    g.hit_cap = (uint32_t)cap;
    g.off_owner = kWsFixed + 8 * g.n_rounds;
    g.off_hits = g.off_owner + ((4 * g.n_rounds + 15) & ~15ull);
    // hit lists for the grid rounded up to 8 CTAs (a cluster plan's grid, a
    // multiple of its cluster size <= 8, may exceed a tiny scan's grid)
    g.ws_bytes = g.off_hits + 8ull * ((g.grid + 7) & ~7ull) * kWarps * g.hit_cap;
    return g;
}

// The shared-memory plan and launch configuration of one scan.
struct Plan {
    ScanArgs a;  // layout and policy fields (the per-call pointers are set by launch_scan)
    uint32_t slots;
    uint32_t cluster;  // CTAs per cluster (1: a plain cooperative launch)
    size_t smem;
    Geometry geo;
    pfac_plan_info info;
};

int check_plan_options(const pfac_plan_options &o, std::string &err) {
    bool ok = o.struct_bytes >= sizeof(pfac_plan_options) && o.placement <= PFAC_PLACE_CLUSTER &&
              (o.cluster == 0 || o.cluster == 2 || o.cluster == 4 || o.cluster == 8) &&
              o.max_filter_rep_log2 >= -1 && o.max_filter_rep_log2 <= 5 &&
              (o.ring_slots == -1 || o.ring_slots == 2 || o.ring_slots == 3) && o.ctg64 >= -1 && o.ctg64 <= 64 &&
              o.pool64 >= -1 && o.pool64 <= 32 && o.stage2 >= -1 && o.stage2 <= 1 && o.entry >= -1 &&
              o.entry <= 1 && o.l2_persist <= 1 && o.form <= PFAC_FORM_MERGED_DAG;
    for (uint32_t r : o.reserved) ok = ok && r == 0;
    if (!ok) {
        err = "pfac_plan_options: bad struct_bytes, reserved field or value";
        return kStatusInvalid;
    }
    return kStatusOk;
}

// Shared-memory plan: filter at offset 0 (replicated while it fits), ring,
// barriers, queues, root, level-1 bitmaps, warp totals, then the hot trie
// prefix (BFS order = level order: the upper levels).
int make_plan(const DevTrie &t, const uint8_t *host_image, const DeviceInfo &di, uint64_t n_starts,
              const pfac_plan_options &o, Plan &p, std::string &err) {
    p.geo = geometry(n_starts, di.sms);
    const bool cl = o.placement == PFAC_PLACE_CLUSTER;
    const uint32_t csize = cl ? (o.cluster ? o.cluster : 2u) : 1u;
    if (cl) {
        // the kinds whose tries outgrow one SM's shared memory; the grid is
        // the co-resident clusters (cooperative: every CTA resident)
        const void *fn = kernel_for(t.kind, 2, true);
        if (!fn) {
            err = "pfac scan plan: cluster placement is for filter kinds 1, 3 and 4";
            return kStatusLimit;
        }
        cudaLaunchConfig_t qc = {};
        qc.gridDim = dim3(csize);
        qc.blockDim = dim3(kThreads);
        qc.dynamicSmemBytes = (size_t)di.max_smem_optin;  // (one CTA per SM at any plan size)
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = csize;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        qc.attrs = qa;
        qc.numAttrs = 1;
        int nc = 0;
        const cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, fn, &qc);
        if (e != cudaSuccess || nc < 1) {
            err = std::string("pfac scan plan: no co-resident cluster of this size: ") + cudaGetErrorString(e);
            return kStatusLimit;
        }
        uint64_t g = std::min<uint64_t>((uint64_t)nc * csize, (uint64_t)di.sms) / csize * csize;
        g = std::min<uint64_t>(g, (p.geo.grid + csize - 1) / csize * csize);  // (<= the workspace's 8-CTA rounding)
        if (g < csize) g = csize;
        p.geo.grid = g;
        p.geo.warps = g * kWarps;
        p.geo.rounds_per_cta = std::max<uint64_t>(1, (p.geo.n_rounds + g - 1) / g);
    }
    const Geometry &geo = p.geo;
    ScanArgs &a = p.a;
    std::memset(&a, 0, sizeof a);
    const uint32_t filter_words = (1u << t.log2_bits) >= 32 ? (1u << t.log2_bits) / 32 : 1u;
    const ImageHeader &hh = *reinterpret_cast<const ImageHeader *>(host_image);
    const uint32_t *host_node = reinterpret_cast<const uint32_t *>(host_image + hh.off_node);
    const uint32_t B = host_node[1] & kEdgeMask;  // root degree: level-1 nodes [1, B]
    const uint32_t *h_tbits = reinterpret_cast<const uint32_t *>(host_image + hh.off_tail_bits);
    const uint32_t *h_trank = reinterpret_cast<const uint32_t *>(host_image + hh.off_tail_rank);
    const uint32_t *h_tails = reinterpret_cast<const uint32_t *>(host_image + hh.off_tails);
    auto tails_below = [&](uint32_t H) -> uint32_t {  // rank(H)
        return h_trank[H >> 5] + (uint32_t)__builtin_popcount(h_tbits[H >> 5] & ((1u << (H & 31)) - 1u));
    };
    auto tbytes_below = [&](uint32_t nt) -> uint32_t {  // bytes of the records below nt (a verify
                                                          // record's bytes start at its first candidate's)
        if (nt >= hh.n_tails) return (uint32_t)hh.n_tail_bytes;
        return h_tails[4 * nt + 2] == kVerify ? h_tails[4 * h_tails[4 * nt]] : h_tails[4 * nt];
    };
    auto hot_bytes = [&](uint32_t H) -> uint64_t {
        const uint32_t nt = tails_below(H);
        return 2ull * align16(4 * (H + 1)) + align16(host_node[H] & kEdgeMask) + 16ull * nt +
               align16(tbytes_below(nt));
    };
    // "Big L1" plan: a trie too big for shared memory but within a few L1s
    // (kBigL1Trie) gets no hot levels, a 2-slot ring and one filter copy, so the
    // L1/shared split leaves the largest L1 for the nodes the walks actually
    // visit (measured with tools/placement.py: C3 -19%; a multi-MB trie (C5)
    // is faster with its dense upper levels in shared memory instead)
    const uint64_t whole = hot_bytes(t.n_nodes - 1);
    bool big_l1 = (t.kind == 1 || t.kind == 3 || t.kind == 4) && whole > kSmallTrie && whole <= kBigL1Trie;
    if (o.placement == PFAC_PLACE_BIG_L1) big_l1 = true;
    if (o.placement == PFAC_PLACE_GLOBAL || o.placement == PFAC_PLACE_SMEM || cl) big_l1 = false;
    // the 2-gram test (and its 8 KiB table): not for DNA (the kernel has no
    // stage 2 for kind 3), and by default only where it is selective: at most
    // a quarter of all 2-grams begin a pattern path (C2 1.5%, C3 5.8%; C4's
    // random bytes 78%: the test would keep most survivors at a cost)
    uint32_t pair_bits = 0;
    {
        const uint32_t *pair = reinterpret_cast<const uint32_t *>(host_image + hh.off_pair);
        for (uint32_t j = 0; j < 2048; j++) pair_bits += (uint32_t)__builtin_popcount(pair[j]);
    }
    bool use_pair = t.kind != 3 && (o.stage2 == 1 || (o.stage2 == -1 && pair_bits <= 65536u / 4));
    uint32_t slots = filter_words * 4 > 65536u || big_l1 ? 2u : (uint32_t)kSlotsMax;  // ring depth
    if (o.ring_slots > 0) slots = (uint32_t)o.ring_slots;
    if (cl) slots = 2;  // (the cluster kernels' ring)
    // per-warp regions (ring, barriers, queues): the kernel's warp_layout
    // (queues deeper for DNA and 8-byte prefixes, whose walks are long:
    // measured C5 64 -4%, C3 96 -2.5%)
    const uint32_t warp_bytes = warp_layout((int)t.kind, (int)slots).bytes;
    const uint32_t fixed0 = kWarps * warp_bytes + 16 + 1024 + align16(40 * B) + 8 * (kWarps + 2) + 512;
    // an automatic 2-gram table that does not fit beside the filter and ring
    // is dropped (e.g. C4's ASCII variant: 128 KiB filter, selective 2-grams)
    if (use_pair && o.stage2 == -1 && (uint32_t)di.max_smem_optin < fixed0 + 8192 + filter_words * 4 + 64)
        use_pair = false;
    const uint32_t fixed = fixed0 + (use_pair ? 8192 : 0);
    if ((uint32_t)di.max_smem_optin < fixed + filter_words * 4 + 64) {
        err = "pfac scan plan: filter and text ring do not fit shared memory";
        return kStatusLimit;
    }
    const uint32_t rest = (uint32_t)di.max_smem_optin - fixed;
    // priority: ring (in `fixed`) > 4 filter copies (bank conflicts of the
    // stage-1 loads) > hot trie > more filter copies
    const uint32_t rep_cap = o.max_filter_rep_log2 >= 0 ? (uint32_t)o.max_filter_rep_log2 : 5u;
    uint32_t rep0 = 0;
    while (rep0 < 2 && rep0 < rep_cap && filter_words * 4 * (2u << rep0) <= kFilterCap &&
           filter_words * 4 * (2u << rep0) + 8192 <= rest)
        rep0++;
    const uint32_t trie_budget = rest - (filter_words * 4 << rep0);
    // Whole trie in shared memory when it fits; otherwise its upper levels
    // (the BFS prefix) in all that is left (measured: more hot levels beat a
    // larger L1 for the deeper ones).
    uint32_t budget = trie_budget;
    if (big_l1 || cl || o.placement == PFAC_PLACE_GLOBAL) budget = 64;  // root table and level-1 bitmaps only
    if (o.hot_bytes_cap && o.hot_bytes_cap < budget) budget = o.hot_bytes_cap;
    uint32_t lo = 1, hi = t.n_nodes - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (hot_bytes(mid) <= budget) lo = mid; else hi = mid - 1;
    }
    const uint32_t H = lo;
    const uint32_t EH = host_node[H] & kEdgeMask;
    const uint32_t TH = tails_below(H);
    const uint32_t TBH = tbytes_below(TH);
    if (hot_bytes(H) > rest - (filter_words * 4 << rep0)) {
        err = "pfac scan plan: internal shared-memory plan error";
        return kStatusLimit;
    }
    const uint32_t left = rest - (uint32_t)hot_bytes(H);  // >= filter_words * 4 << rep0
    uint32_t rep_log2 = rep0;
    while (rep_log2 < rep_cap && filter_words * 4 * (2u << rep_log2) <= (left < kFilterCap ? left : kFilterCap))
        rep_log2++;
    if (big_l1 || cl) rep_log2 = 0;
    const uint32_t filter_bytes = filter_words * 4 << rep_log2;

    a.t = t;
    a.filter_words = filter_words;
    a.rep_log2 = rep_log2;
    uint32_t off = align_up(filter_bytes, 128);
    a.off_warps = off;  off += kWarps * warp_bytes;  // per-warp regions (warp_layout)
    a.off_sbar = off;   off += 16;                   // the table-staging mbarrier
    a.off_warp = off;   off += 8 * (kWarps + 2);  // warp totals [kWarps + 2] (the last: the CTA's round counter first)
    off = align_up(off, 16);
    a.off_root = off;   off += 1024;
    a.off_pair = off;   off += use_pair ? 8192 : 0;  // 2-gram prefix table [256][8] words
    a.use_pair = use_pair;
    a.off_bm = off;     off += align16(40 * B);
    a.off_node = off;   off += align16(4 * (H + 1));
    a.off_aux = off;    off += align16(4 * (H + 1));
    a.off_label = off;  off += align16(EH);
    {   // terminal tables in smem when small and they fit what is left
        const uint32_t tb = align16(4 * (uint32_t)(hh.n_terminals + 1));
        a.off_terms = 0;
        if (hh.n_terminals + 1 < 8192 &&
            off + tb + 16 * TH + align16(TBH) <= (uint32_t)di.max_smem_optin) {
            a.off_terms = off;
            off += tb;
        }
    }
    a.off_tails = off;  off += 16 * TH;
    a.off_tbytes = off; off += align16(TBH);
    a.hot_tails = TH;
    a.hot_tail_bytes = TBH;
    if (cl) {  // the cluster tier: a power-of-two slice of node records per CTA in what is left
        a.off_dsm = align_up(off, 16);
        const uint32_t avail = (uint32_t)di.max_smem_optin > a.off_dsm ? (uint32_t)di.max_smem_optin - a.off_dsm : 0u;
        uint32_t lg = 0;
        while ((16u << (lg + 1)) <= avail && ((uint64_t)csize << lg) < t.n_nodes) lg++;
        if ((16u << lg) > avail) {
            err = "pfac scan plan: no shared memory left for the cluster tier";
            return kStatusLimit;
        }
        a.dsm_log2 = lg;
        a.dsm_nodes = (uint32_t)std::min<uint64_t>(t.n_nodes, (uint64_t)csize << lg);
        off = a.off_dsm + (16u << lg);
    }
    p.smem = off;
    if (p.smem > (size_t)di.max_smem_optin) {
        err = "pfac scan plan: the requested plan does not fit shared memory";
        return kStatusLimit;
    }
    a.n_level1 = B;
    a.hot_nodes = H;
    a.hot_edges = EH;
    // walks through a shared-memory trie are cheaper than an L2 probe of the
    // exact key set: probe only when the trie is not wholly staged
    a.use_kset = t.kset != nullptr && H < t.n_nodes - 1;
    a.use_entry = t.entry != nullptr && o.entry != 0;
    // walks through a wholly staged trie are short and even: (almost) all
    // rounds in per-warp blocks; else the last quarter is handed out
    // dynamically (measured: C3 -11% dynamic)
    // (kind 1, large sets of random-looking byte patterns: even work per
    // round, so every CTA range is static and only the pool balances: C4 -2%)
    // (DNA, kind 3, with >= 128 rounds per warp: 60/64 static -- its walks per
    // round vary less than C3's token text: C5 2 GiB -1.5%; at 55 rounds per
    // warp (256 MiB) the dynamic quarter still pays: +5% with 60)
    const bool dna_long = t.kind == 3 && geo.rounds_per_cta >= 128u * kWarps;
    a.ctg64 = o.ctg64 >= 0 ? (uint32_t)o.ctg64 : (H >= t.n_nodes - 1 || t.kind == 1 ? 64u : dna_long ? 60u : 48u);
    // the shared pool: the text's last rounds, taken by any warp whose CTA's
    // range is done (cross-CTA balance where walks leave the SM: content
    // skew between ranges, e.g. C5's first ranges hold twice the matches);
    // planned when start offsets from a CTA's first round fit 32 bits
    {
        // (kind 1: 2/64, its rounds are even: C4 4 GiB -0.5% against 4/64)
        const uint64_t pool64 = o.pool64 >= 0 ? (uint64_t)o.pool64 : t.kind == 1 ? 2u : a.ctg64 < 64 ? 4u : 0u;
        const uint64_t n_pool = geo.n_rounds * pool64 / 64;
        const bool pool = t.kind != 2 && n_pool >= geo.grid && geo.n_rounds * (uint64_t)kRound <= (1ull << 32);
        a.n_main = pool ? geo.n_rounds - n_pool : geo.n_rounds;
        a.rounds_per_cta = pool ? (a.n_main + geo.grid - 1) / geo.grid : geo.rounds_per_cta;
        a.pool_seg = pool ? (uint32_t)((n_pool + geo.grid - 1) / geo.grid) : 0u;
    }
    a.hit_cap = geo.hit_cap;
    p.slots = slots;

    pfac_plan_info &f = p.info;
    std::memset(&f, 0, sizeof f);
    f.filter_kind = t.kind;
    f.ring_slots = slots;
    f.filter_copies = 1u << rep_log2;
    f.smem_bytes = (uint32_t)p.smem;
    f.hot_nodes = H;
    f.image_nodes = t.n_nodes;
    f.hot_edges = EH;
    f.terms_in_smem = a.off_terms != 0;
    f.grid = (uint32_t)geo.grid;
    f.warps_per_cta = kWarps;
    f.hit_cap = geo.hit_cap;
    f.stage2 = use_pair;
    f.entry = a.use_entry;
    f.kset = a.use_kset;
    f.pool_rounds = (uint32_t)(geo.n_rounds - a.n_main);
    f.placement = cl       ? PFAC_PLACE_CLUSTER
                  : big_l1 ? PFAC_PLACE_BIG_L1
                  : o.placement == PFAC_PLACE_GLOBAL ? PFAC_PLACE_GLOBAL : PFAC_PLACE_SMEM;
    f.cluster = csize;
    f.dsm_nodes = a.dsm_nodes;
    p.cluster = csize;
    f.rounds_per_cta = a.rounds_per_cta;
    f.main_rounds = a.n_main;
    return kStatusOk;
}

}  // namespace

DevTrie make_dev_trie(const ImageHeader &h, const uint8_t *d) {
    DevTrie t;
    t.node = reinterpret_cast<const uint32_t *>(d + h.off_node);
    t.aux = reinterpret_cast<const uint32_t *>(d + aux_offset(h.off_node, h.n_nodes));
    t.rec = reinterpret_cast<const uint4 *>(d + h.off_rec);
    t.label = d + h.off_label;
    t.term_node = reinterpret_cast<const uint32_t *>(d + h.off_term_node);
    t.term_rk = reinterpret_cast<const uint2 *>(d + h.off_term_rk);
    t.out_ptr = reinterpret_cast<const uint32_t *>(d + h.off_out_ptr);
    t.out_pid = reinterpret_cast<const uint32_t *>(d + h.off_out_pid);
    t.root = reinterpret_cast<const uint32_t *>(d + h.off_root);
    t.filter = reinterpret_cast<const uint32_t *>(d + h.off_filter);
    t.tail_bits = reinterpret_cast<const uint32_t *>(d + h.off_tail_bits);
    t.tail_rank = reinterpret_cast<const uint32_t *>(d + h.off_tail_rank);
    t.tails = reinterpret_cast<const uint4 *>(d + h.off_tails);
    t.tail_bytes = d + h.off_tail_bytes;
    t.level1 = reinterpret_cast<const uint32_t *>(d + h.off_level1);
    t.pair = reinterpret_cast<const uint32_t *>(d + h.off_pair);
    t.kset = h.off_kset ? reinterpret_cast<const uint32_t *>(d + h.off_kset) : nullptr;
    t.kset_log2 = h.kset_log2;
    t.kset_empty = h.kset_empty;
    t.entry = h.off_entry ? reinterpret_cast<const uint4 *>(d + h.off_entry) : nullptr;
    t.entry_log2 = h.entry_log2;
    t.n_terminals = (uint32_t)h.n_terminals;
    t.n_kept_terminals = (uint32_t)h.n_kept_terminals;
    t.max_len = h.max_len;
    t.gram = h.filter_gram;
    t.log2_bits = h.filter_log2_bits;
    t.exact = h.filter_exact;
    t.kind = h.filter_kind;
    t.n_nodes = (uint32_t)h.n_nodes;
    t.n_edges = (uint32_t)h.n_edges;
    t.n_records = (uint32_t)(h.n_tails + h.n_cand);
    t.n_tail_bytes = (uint32_t)h.n_tail_bytes;
    t.n_out = (uint32_t)h.n_out;
    t.n_level1 = (uint32_t)h.n_level1;
    return t;
}

int workspace_bytes_for(uint64_t n_starts, int device, uint64_t *out, std::string &err) {
    DeviceInfo di;
    int st = device_info(device, di, err);
    if (st != kStatusOk) return st;
    const Geometry g = geometry(n_starts, di.sms);
    *out = std::max<uint64_t>(g.ws_bytes, dag_workspace_bytes(n_starts));  // (either form)
    return kStatusOk;
}

uint32_t launches_per_call() { return 1; }  // the scan kernel

#ifdef PFAC_TIMING
int debug_timing(unsigned long long *host, uint64_t n) {
    return cudaMemcpyFromSymbol(host, g_pfac_timing, n * 8) == cudaSuccess ? 0 : -1;
}
#endif

int plan_query(const DevTrie &t, const uint8_t *host_image, int device, uint64_t n_starts,
               const pfac_plan_options &o, pfac_plan_info *out, std::string &err) {
    int st = check_plan_options(o, err);
    if (st != kStatusOk) return st;
    DeviceInfo di;
    st = device_info(device, di, err);
    if (st != kStatusOk) return st;
    Plan p;
    st = make_plan(t, host_image, di, n_starts ? n_starts : 1, o, p, err);
    if (st != kStatusOk) return st;
    *out = p.info;
    return kStatusOk;
}

int launch_scan(const DevTrie &t, const uint8_t *host_image, int device, const uint8_t *d_text,
                uint64_t readable_len, uint64_t n_starts, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                uint64_t capacity, uint64_t *d_count, void *d_ws, uint64_t ws_bytes, const pfac_plan_options &o,
                CUstream_st *stream_, std::string &err) {
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
    int st = check_plan_options(o, err);
    if (st != kStatusOk) return st;
    if (n_starts == 0) {
        cudaError_t e = cudaMemsetAsync(d_count, 0, sizeof(uint64_t), stream);
        if (e != cudaSuccess) {
            err = std::string("cudaMemsetAsync: ") + cudaGetErrorString(e);
            return kStatusCuda;
        }
        return kStatusOk;
    }
    DeviceInfo di;
    st = device_info(device, di, err);
    if (st != kStatusOk) return st;
    Plan p;
    st = make_plan(t, host_image, di, n_starts, o, p, err);
    if (st != kStatusOk) return st;
    const Geometry &geo = p.geo;
    if (geo.rounds_per_cta >= (1ull << (32 - kRoundLog2))) {  // start offsets within a CTA are 32-bit
        err = "pfac_match_device: n_starts too large for one launch (split the text)";
        return kStatusLimit;
    }
    if (!d_ws || ws_bytes < geo.ws_bytes || (reinterpret_cast<uintptr_t>(d_ws) & 15)) {
        err = "pfac_match_device: workspace too small or misaligned";
        return kStatusInvalid;
    }
    ScanArgs a = p.a;
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
    a.pool_total = a.cta_total + kMaxCtas;
    a.round_val = reinterpret_cast<unsigned long long *>(reinterpret_cast<uint8_t *>(d_ws) + kWsFixed);
    a.round_owner = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(d_ws) + geo.off_owner);
    a.hits = reinterpret_cast<uint2 *>(reinterpret_cast<uint8_t *>(d_ws) + geo.off_hits);
    a.aligned = (reinterpret_cast<uintptr_t>(d_text) & 15) == 0;
    void *args[] = {&a};
    const void *fn = kernel_for(t.kind, p.slots, p.cluster > 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)geo.grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[3];
    attr[0].id = cudaLaunchAttributeCooperative;  // the grid barrier needs every CTA resident
    attr[0].val.cooperative = 1;
    cfg.numAttrs = 1;
    if (p.cluster > 1) {
        attr[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
        attr[cfg.numAttrs].val.clusterDim.x = p.cluster;
        attr[cfg.numAttrs].val.clusterDim.y = 1;
        attr[cfg.numAttrs].val.clusterDim.z = 1;
        cfg.numAttrs++;
    }
    if (o.l2_persist) {  // placement ablation: the device image as an L2 persisting window of this launch
        const ImageHeader &hh = *reinterpret_cast<const ImageHeader *>(host_image);
        const size_t win = std::min<size_t>((size_t)hh.image_bytes - hh.off_node, 64u << 20);
        static std::once_flag once;
        std::call_once(once, [&] { cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 64u << 20); });
        cudaLaunchAttribute &w = attr[cfg.numAttrs++];
        w.id = cudaLaunchAttributeAccessPolicyWindow;
        w.val.accessPolicyWindow.base_ptr = const_cast<uint32_t *>(t.node);
        w.val.accessPolicyWindow.num_bytes = win;
        w.val.accessPolicyWindow.hitRatio = 1.0f;
        w.val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        w.val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    }
    cfg.attrs = attr;
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) {
        err = std::string("scan launch: ") + cudaGetErrorString(e);
        return kStatusCuda;
    }
    return kStatusOk;
}

}  // namespace pfac

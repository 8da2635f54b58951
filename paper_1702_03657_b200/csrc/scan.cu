// scan.cu -- sm_100a PFAC scan kernel (KB1) with in-kernel deterministic
// compaction (decoupled look-back over segments).
//
// PAPER.md:76 (§II-C): "Each thread is assigned to a single letter in the
// text T. If a match is recorded, the thread continues the matching process
// until a mismatch. When a mismatch occurs the thread is terminated."
//
// Mapping (v0): a persistent CTA of 256 threads claims
// segments of 4096 start positions from an atomic counter.  The segment's text
// (+256 B of halo) is staged in shared memory with coalesced 16-byte loads.
// Each thread owns 16 consecutive starts:
//   stage 1  d-gram filter test in shared memory (a clear bit = no match can
//            start here, so the walk is skipped: the early exit of P:76 taken
//            before the first trie access);
//   stage 2  survivors walk the CSR trie (root level from a shared table,
//            deeper levels through L1/L2) until the first mismatch, keeping the
//            deepest terminal passed;
//   stage 3  the CTA scans its match counts, obtains the segment's global
//            offset by decoupled look-back, and writes (pos, pid) rows, which
//            are therefore globally sorted by (pos, pid) with no second pass.
#include <cuda/atomic>
#include <cuda_runtime.h>

#include <cstdio>
#include <mutex>

#include "internal.h"

namespace pfac {

namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 16;
constexpr int kSeg = kThreads * kPerThread;  // start positions per segment
constexpr int kWinPad = 256;                  // halo bytes staged past the segment
constexpr int kWin = kSeg + kWinPad;          // staged window
constexpr int kWinAlloc = kWin + 32;          // + zero tail for the 4-byte key reads

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

struct WsHeader {
    unsigned int seg_counter;
    unsigned int pad[63];
};
static_assert(sizeof(WsHeader) == 256, "");

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
    unsigned long long *status;
    uint64_t n_seg;
    uint32_t filter_words;
};

__device__ __forceinline__ uint32_t ldg_u32(const uint32_t *p) { return __ldg(p); }

// Text byte j (global index) of the current segment: the staged window when
// it covers j, else global memory (walks longer than the staged halo).
__device__ __forceinline__ uint32_t text_byte(const uint8_t *s_win, uint32_t win_len, uint64_t seg_base,
                                              const uint8_t *g, uint64_t j) {
    uint64_t lj = j - seg_base;
    return lj < win_len ? (uint32_t)s_win[lj] : (uint32_t)__ldg(g + j);
}

// Walk from start gi; returns the deepest terminal node passed, or kNone.
__device__ uint32_t walk(const ScanArgs &a, const uint32_t *s_root, const uint8_t *s_win, uint32_t win_len,
                         uint64_t seg_base, uint64_t gi) {
    uint32_t v = s_root[text_byte(s_win, win_len, seg_base, a.text, gi)];
    if (v == 0) return kNone;
    uint32_t w = ldg_u32(a.t.node + v);
    uint32_t last = (w & kTermBit) ? v : kNone;
    for (uint64_t j = gi + 1; j < a.readable; ++j) {
        uint32_t s = w & kEdgeMask;
        uint32_t e = ldg_u32(a.t.node + v + 1) & kEdgeMask;
        if (s == e) break;  // leaf
        uint32_t c = text_byte(s_win, win_len, seg_base, a.text, j);
        // labels[s, e) ascending: binary search down to a short linear scan
        uint32_t lo = s, hi = e;
        while (hi - lo > 8) {
            uint32_t mid = (lo + hi) >> 1;
            if ((uint32_t)__ldg(a.t.label + mid) <= c) lo = mid; else hi = mid;
        }
        uint32_t found = kNone;
        for (uint32_t k = lo; k < hi; ++k) {
            uint32_t l = __ldg(a.t.label + k);
            if (l == c) { found = k; break; }
            if (l > c) break;
        }
        if (found == kNone) break;  // mismatch: the thread terminates
        v = found + 1;              // BFS order: child through edge e is node e+1
        w = ldg_u32(a.t.node + v);
        if (w & kTermBit) last = v;
    }
    return last;
}

// Index of terminal node v in term_node (binary search; v is terminal).
__device__ uint32_t term_index(const DevTrie &t, uint32_t v) {
    uint32_t lo = 0, hi = t.n_terminals;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (ldg_u32(t.term_node + mid) < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Exclusive block scan of per-thread counts; returns the exclusive value and
// the block total through *total.
__device__ uint64_t block_exclusive_scan(uint32_t x, uint32_t *s_warp, uint64_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint64_t base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        uint32_t t = s_warp[w];
        if (w < warp) base += t;
        tot += t;
    }
    *total = tot;
    return base + incl - x;
}

// Decoupled look-back (single thread): publishes this segment's aggregate,
// accumulates predecessors until an inclusive prefix is found.
__device__ uint64_t look_back(unsigned long long *status, uint64_t seg, uint64_t total) {
    using A = cuda::atomic_ref<unsigned long long, cuda::thread_scope_device>;
    if (seg == 0) {
        A(status[0]).store(kFlagInc | total, cuda::memory_order_release);
        return 0;
    }
    A(status[seg]).store(kFlagAgg | total, cuda::memory_order_release);
    uint64_t excl = 0;
    uint64_t k = seg - 1;
    while (true) {
        unsigned long long w = A(status[k]).load(cuda::memory_order_acquire);
        unsigned long long f = w & ~kValMask;
        if (f == 0) {
            __nanosleep(20);
            continue;
        }
        excl += w & kValMask;
        if (f == kFlagInc) break;
        --k;
    }
    A(status[seg]).store(kFlagInc | (excl + total), cuda::memory_order_release);
    return excl;
}

__global__ void __launch_bounds__(kThreads) pfac_scan_kernel(const ScanArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t *s_filter = reinterpret_cast<uint32_t *>(smem);
    uint32_t *s_root = s_filter + a.filter_words;
    uint8_t *s_win = reinterpret_cast<uint8_t *>(s_root + 256);
    uint32_t *s_res = reinterpret_cast<uint32_t *>(s_win + kWinAlloc);
    __shared__ uint32_t s_warp[kThreads / 32];
    __shared__ uint64_t s_prefix;
    __shared__ uint64_t s_seg;

    const int tid = threadIdx.x;
    for (uint32_t i = tid; i < a.filter_words; i += kThreads) s_filter[i] = ldg_u32(a.t.filter + i);
    for (uint32_t i = tid; i < 256; i += kThreads) s_root[i] = ldg_u32(a.t.root + i);

    const uint32_t gram = a.t.gram;
    const uint32_t kmask = gram >= 4 ? 0xFFFFFFFFu : ((1u << (8 * gram)) - 1u);

    while (true) {
        if (tid == 0) s_seg = atomicAdd(&a.ws->seg_counter, 1u);
        __syncthreads();
        const uint64_t seg = s_seg;
        if (seg >= a.n_seg) break;
        const uint64_t seg_base = seg * kSeg;

        // ---- stage the window [seg_base, seg_base + win_len) in shared memory
        const uint64_t avail = a.readable - seg_base;
        const uint32_t win_len = avail < (uint64_t)kWin ? (uint32_t)avail : (uint32_t)kWin;
        const uint8_t *src = a.text + seg_base;
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            const uint32_t nv = win_len >> 4;
            const uint4 *src4 = reinterpret_cast<const uint4 *>(src);
            uint4 *dst4 = reinterpret_cast<uint4 *>(s_win);
            for (uint32_t i = tid; i < nv; i += kThreads) dst4[i] = __ldg(src4 + i);
            for (uint32_t i = (nv << 4) + tid; i < win_len; i += kThreads) s_win[i] = __ldg(src + i);
        } else {
            for (uint32_t i = tid; i < win_len; i += kThreads) s_win[i] = __ldg(src + i);
        }
        if (tid < 32) s_win[win_len + tid] = 0;
        __syncthreads();

        // ---- stage 1: d-gram filter over this thread's 16 starts
        const uint32_t l0 = tid * kPerThread;
        uint32_t w5[5];
        {
            const uint4 v = *reinterpret_cast<const uint4 *>(s_win + l0);
            w5[0] = v.x; w5[1] = v.y; w5[2] = v.z; w5[3] = v.w;
            w5[4] = *reinterpret_cast<const uint32_t *>(s_win + l0 + 16);
        }
        uint32_t surv = 0;
#pragma unroll
        for (int k = 0; k < kPerThread; ++k) {
            const uint32_t x = __funnelshift_r(w5[k >> 2], w5[(k >> 2) + 1], 8 * (k & 3)) & kmask;
            const uint32_t h = filter_index(x, a.t.log2_bits, a.t.exact);
            const uint32_t bit = (s_filter[h >> 5] >> (h & 31)) & 1u;
            const uint64_t gi = seg_base + l0 + k;
            const bool valid = gi < a.n_starts && gi + gram <= a.readable;
            surv |= (bit & (uint32_t)valid) << k;
        }

        // ---- stage 2: survivors walk the trie
        uint32_t count = 0;
        for (uint32_t m = surv; m; m &= m - 1) {
            const uint32_t k = __ffs(m) - 1;
            const uint32_t li = l0 + k;
            uint32_t tn = walk(a, s_root, s_win, win_len, seg_base, seg_base + li);
            uint32_t ti = kNone;
            if (tn != kNone) {
                ti = term_index(a.t, tn);
                count += ldg_u32(a.t.out_ptr + ti + 1) - ldg_u32(a.t.out_ptr + ti);
            }
            s_res[li] = ti;
        }

        // ---- stage 3: segment offset (block scan + look-back), then write
        uint64_t total;
        const uint64_t excl = block_exclusive_scan(count, s_warp, &total);
        if (tid == 0) {
            const uint64_t prefix = look_back(a.status, seg, total);
            s_prefix = prefix;
            if (seg == a.n_seg - 1) *a.out_count = prefix + total;
        }
        __syncthreads();
        uint64_t off = s_prefix + excl;
        for (uint32_t m = surv; m; m &= m - 1) {
            const uint32_t k = __ffs(m) - 1;
            const uint32_t ti = s_res[l0 + k];
            if (ti == kNone) continue;
            const uint32_t r0 = ldg_u32(a.t.out_ptr + ti), r1 = ldg_u32(a.t.out_ptr + ti + 1);
            const uint64_t pos = a.pos_base + seg_base + l0 + k;
            for (uint32_t r = r0; r < r1; ++r, ++off) {
                if (off < a.capacity) {
                    a.out_pos[off] = pos;
                    a.out_pid[off] = ldg_u32(a.t.out_pid + r);
                }
            }
        }
        __syncthreads();  // s_win / s_res / s_seg reused by the next segment
    }
}

struct DeviceInfo {
    bool init = false;
    int sms = 0;
    int max_smem_optin = 0;
};
std::mutex g_dev_mu;
DeviceInfo g_dev[64];

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
    return t;
}

uint64_t workspace_bytes_for(uint64_t n_starts) {
    const uint64_t n_seg = (n_starts + kSeg - 1) / kSeg;
    return sizeof(WsHeader) + 8 * (n_seg ? n_seg : 1);
}

uint32_t launches_per_call() { return 2; }  // workspace reset (memset) + scan kernel

int launch_scan(const DevTrie &t, int device, const uint8_t *d_text, uint64_t readable_len, uint64_t n_starts,
                uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid, uint64_t capacity, uint64_t *d_count,
                void *d_ws, uint64_t ws_bytes, CUstream_st *stream_, std::string &err) {
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
    const uint64_t n_seg = (n_starts + kSeg - 1) / kSeg;
    const uint32_t filter_words = (1u << t.log2_bits) >= 32 ? (1u << t.log2_bits) / 32 : 1u;
    const size_t smem = (size_t)filter_words * 4 + 1024 + kWinAlloc + (size_t)kSeg * 4;
    int blocks_per_sm = 0, sms = 0;
    {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        DeviceInfo &di = g_dev[device];
        if (!di.init) {
            cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, device);
            cudaDeviceGetAttribute(&di.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
            cudaError_t e = cudaFuncSetAttribute(pfac_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 di.max_smem_optin - 2048);
            if (e != cudaSuccess) {
                err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
                return kStatusCuda;
            }
            di.init = true;
        }
        sms = di.sms;
        if ((int)smem > di.max_smem_optin - 2048) {
            err = "pfac_match_device: shared memory budget exceeded";
            return kStatusLimit;
        }
    }
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, pfac_scan_kernel, kThreads, smem);
    if (e != cudaSuccess || blocks_per_sm < 1) {
        err = std::string("occupancy query failed: ") + cudaGetErrorString(e);
        return kStatusCuda;
    }
    const uint64_t need = workspace_bytes_for(n_starts);
    if (!d_ws || ws_bytes < need) {
        err = "pfac_match_device: workspace too small";
        return kStatusInvalid;
    }
    e = cudaMemsetAsync(d_ws, 0, need, stream);
    if (e != cudaSuccess) {
        err = std::string("cudaMemsetAsync: ") + cudaGetErrorString(e);
        return kStatusCuda;
    }
    ScanArgs a;
    a.t = t;
    a.text = d_text;
    a.readable = readable_len;
    a.n_starts = n_starts;
    a.pos_base = pos_base;
    a.out_pos = d_pos;
    a.out_pid = d_pid;
    a.capacity = capacity;
    a.out_count = d_count;
    a.ws = reinterpret_cast<WsHeader *>(d_ws);
    a.status = reinterpret_cast<unsigned long long *>(reinterpret_cast<uint8_t *>(d_ws) + sizeof(WsHeader));
    a.n_seg = n_seg;
    a.filter_words = filter_words;
    uint64_t grid = (uint64_t)blocks_per_sm * (uint64_t)sms;
    if (grid > n_seg) grid = n_seg;
    pfac_scan_kernel<<<(unsigned)grid, kThreads, smem, stream>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        err = std::string("scan launch: ") + cudaGetErrorString(e);
        return kStatusCuda;
    }
    return kStatusOk;
}

}  // namespace pfac

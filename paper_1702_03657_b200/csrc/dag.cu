// dag.cu -- scan of the merged DAG (NEXT-2: PAPER.md:80 steps IV-V, "similar
// suffixes are merged", "end nodes merged"), exact through path ranks.
//
// The DAG (image.h dag_*) is the minimal automaton of the pattern strings:
// identical sub-tries are one node, so the child of an edge is explicit and
// a terminal node no longer identifies one pattern.  A walk adds dag_skip[e]
// at every edge e it takes (the node's own terminal plus the strings below
// its earlier children); at a terminal the sum is the lexicographic rank of
// the string spelled so far, and rank_term[rank] is that string's terminal
// index in the main image, i.e. its sorted list of every pattern ending on
// the path (the walk continues past matches to the first
// mismatch, so the deepest terminal reached decides the start's rows).
//
// Three launches, deterministic and sorted by (pos, pid):
//   dag_count:  each thread walks kPer consecutive starts; per-block row total
//   dag_offsets: one block scans the block totals (and writes the count)
//   dag_emit:   the walks again, a block scan of the thread totals, the rows
// This form is a plain per-start walk over global memory (L1/L2): it has no
// first-stage filter and is not tuned; it exists to scan the merged structure
// exactly (the product path is scan.cu's filtered CSR trie).
#include <cuda_runtime.h>

#include "internal.h"

namespace pfac {

namespace {

constexpr int kDagThreads = 1024;
constexpr int kPer = 16;  // consecutive starts per thread
constexpr uint64_t kStartsPerBlock = (uint64_t)kDagThreads * kPer;

struct DagArgs {
    const uint32_t *node;   // [ND+1] first edge | terminal bit
    const uint8_t *label;   // [ED]
    const uint32_t *child;  // [ED]
    const uint32_t *skip;   // [ED]
    const uint32_t *rank_term;
    uint32_t n_ranks, n_nodes, n_edges;
    const uint32_t *out_ptr, *out_pid;
    const uint8_t *text;
    uint64_t readable, n_starts, pos_base;
    uint64_t *out_pos;
    uint32_t *out_pid_rows;
    uint64_t capacity;
    uint64_t *out_count;
    unsigned long long *block_tot;  // [n_blocks]: rows of the block, then its first row
};

// Terminal index of the deepest terminal reached from start i, or kNone.
__device__ __forceinline__ uint32_t dag_walk(const DagArgs &a, uint64_t i) {
    uint32_t v = 0, rank = 0, last = kNone;
    for (uint64_t j = i; j < a.readable; ++j) {
        const uint32_t c = __ldg(a.text + j);
        uint32_t lo = __ldg(a.node + v) & kEdgeMask;
        const uint32_t hi = __ldg(a.node + v + 1) & kEdgeMask;
        uint32_t e = kNone;
        if (hi - lo <= 8) {
            for (uint32_t k = lo; k < hi; ++k)
                if (__ldg(a.label + k) == c) {
                    e = k;
                    break;
                }
        } else {
            uint32_t h = hi;
            while (h - lo > 1) {  // labels ascending: the last <= c
                const uint32_t mid = (lo + h) >> 1;
                if (__ldg(a.label + mid) <= c) lo = mid; else h = mid;
            }
            if (__ldg(a.label + lo) == c) e = lo;
        }
        if (e == kNone) break;  // mismatch: the thread terminates
        PFAC_CHECK(e < a.n_edges && __ldg(a.child + e) < a.n_nodes);
        rank += __ldg(a.skip + e);
        v = __ldg(a.child + e);
        if (__ldg(a.node + v) & kTermBit) last = rank;
    }
    return last < a.n_ranks ? __ldg(a.rank_term + last) : kNone;  // (a bounds guard: validated images never miss)
}

__device__ __forceinline__ uint32_t rows_of(const DagArgs &a, uint32_t t) {
    return t == kNone ? 0u : __ldg(a.out_ptr + t + 1) - __ldg(a.out_ptr + t);
}

// Block-wide exclusive scan (kDagThreads values); *total = the sum.
__device__ __forceinline__ unsigned long long block_excl(unsigned long long v, unsigned long long *total) {
    __shared__ unsigned long long s_w[kDagThreads / 32 + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const unsigned long long w0 = lane < kDagThreads / 32 ? s_w[lane] : 0ull;
        unsigned long long wi = w0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, d);
            if (lane >= d) wi += y;
        }
        if (lane < kDagThreads / 32) s_w[lane] = wi - w0;
        if (lane == 31) s_w[kDagThreads / 32] = wi;
    }
    __syncthreads();
    const unsigned long long ex = s_w[warp] + incl - v;
    *total = s_w[kDagThreads / 32];
    __syncthreads();
    return ex;
}

__global__ void __launch_bounds__(kDagThreads) dag_count(const DagArgs a) {
    const uint64_t s0 = ((uint64_t)blockIdx.x * kDagThreads + threadIdx.x) * kPer;
    unsigned long long n = 0;
    for (int k = 0; k < kPer; ++k)
        if (s0 + k < a.n_starts) n += rows_of(a, dag_walk(a, s0 + k));
    unsigned long long tot;
    block_excl(n, &tot);
    if (threadIdx.x == 0) a.block_tot[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kDagThreads) dag_offsets(const DagArgs a, uint64_t n_blocks) {
    unsigned long long run = 0;
    for (uint64_t b0 = 0; b0 < n_blocks; b0 += kDagThreads) {
        const uint64_t b = b0 + threadIdx.x;
        const unsigned long long v = b < n_blocks ? a.block_tot[b] : 0ull;
        unsigned long long tot;
        const unsigned long long ex = block_excl(v, &tot);
        if (b < n_blocks) a.block_tot[b] = run + ex;
        run += tot;
    }
    if (threadIdx.x == 0) *a.out_count = run;
}

__global__ void __launch_bounds__(kDagThreads) dag_emit(const DagArgs a) {
    const uint64_t s0 = ((uint64_t)blockIdx.x * kDagThreads + threadIdx.x) * kPer;
    uint32_t t[kPer];
    unsigned long long n = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        t[k] = s0 + k < a.n_starts ? dag_walk(a, s0 + k) : kNone;
        n += rows_of(a, t[k]);
    }
    unsigned long long tot;
    uint64_t o = a.block_tot[blockIdx.x] + block_excl(n, &tot);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        if (t[k] == kNone) continue;
        const uint32_t r0 = __ldg(a.out_ptr + t[k]), r1 = __ldg(a.out_ptr + t[k] + 1);
        for (uint32_t r = r0; r < r1; ++r, ++o)
            if (o < a.capacity) {
                a.out_pos[o] = a.pos_base + s0 + k;
                a.out_pid_rows[o] = __ldg(a.out_pid + r);
            }
    }
}

}  // namespace

uint64_t dag_workspace_bytes(uint64_t n_starts) {
    return kWsDagOffset + 8 * ((n_starts + kStartsPerBlock - 1) / kStartsPerBlock);
}

int launch_dag(const ImageHeader &h, const uint8_t *d_img, const uint8_t *d_text, uint64_t readable_len,
               uint64_t n_starts, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid, uint64_t capacity,
               uint64_t *d_count, void *d_ws, uint64_t ws_bytes, CUstream_st *stream_, std::string &err) {
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
    if (!h.n_dag_nodes) {
        err = "pfac_match_device: PFAC_FORM_MERGED_DAG needs a trie built with merge_suffixes";
        return kStatusInvalid;
    }
    if (n_starts == 0) {
        const cudaError_t e = cudaMemsetAsync(d_count, 0, sizeof(uint64_t), stream);
        if (e != cudaSuccess) {
            err = std::string("cudaMemsetAsync: ") + cudaGetErrorString(e);
            return kStatusCuda;
        }
        return kStatusOk;
    }
    const uint64_t n_blocks = (n_starts + kStartsPerBlock - 1) / kStartsPerBlock;
    if (!d_ws || ws_bytes < dag_workspace_bytes(n_starts) || n_blocks > 0x7FFFFFFFull) {
        err = "pfac_match_device: workspace too small for the merged-DAG scan";
        return kStatusInvalid;
    }
    DagArgs a;
    a.node = reinterpret_cast<const uint32_t *>(d_img + h.off_dag_node);
    a.label = d_img + h.off_dag_label;
    a.child = reinterpret_cast<const uint32_t *>(d_img + h.off_dag_child);
    a.skip = reinterpret_cast<const uint32_t *>(d_img + h.off_dag_skip);
    a.rank_term = reinterpret_cast<const uint32_t *>(d_img + h.off_rank_term);
    a.n_ranks = (uint32_t)h.n_terminals;
    a.n_nodes = (uint32_t)h.n_dag_nodes;
    a.n_edges = (uint32_t)h.n_dag_edges;
    a.out_ptr = reinterpret_cast<const uint32_t *>(d_img + h.off_out_ptr);
    a.out_pid = reinterpret_cast<const uint32_t *>(d_img + h.off_out_pid);
    a.text = d_text;
    a.readable = readable_len;
    a.n_starts = n_starts;
    a.pos_base = pos_base;
    a.out_pos = d_pos;
    a.out_pid_rows = d_pid;
    a.capacity = capacity;
    a.out_count = d_count;
    // after the main scan's header and CTA totals: the main kernel's grid
    // barrier state at the workspace start is left untouched
    a.block_tot = reinterpret_cast<unsigned long long *>(reinterpret_cast<uint8_t *>(d_ws) + kWsDagOffset);
    dag_count<<<(unsigned)n_blocks, kDagThreads, 0, stream>>>(a);
    dag_offsets<<<1, kDagThreads, 0, stream>>>(a, n_blocks);
    dag_emit<<<(unsigned)n_blocks, kDagThreads, 0, stream>>>(a);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        err = std::string("merged-DAG scan launch: ") + cudaGetErrorString(e);
        return kStatusCuda;
    }
    return kStatusOk;
}

}  // namespace pfac

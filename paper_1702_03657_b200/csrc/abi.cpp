// abi.cpp -- extern "C" entry points of libpfac.so (declared in include/pfac.h).
// No exception crosses this boundary; errors set a thread-local message.
#include "pfac.h"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // host ranges for timeline profilers (no-ops when none is attached)

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "internal.h"

using namespace pfac;

// Device state pfac_match (host API) keeps between calls, per device: the
// streaming pipeline's streams, events, text buffers (chunk + halo each),
// pinned staging buffers (pageable input), workspace, per-chunk outputs.
constexpr int kStreamBufs = 3;
// A host range on the NVTX timeline (nsys / ncu --nvtx) for one API call.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

struct HostCtx {
    std::mutex mu;  // one pfac_match at a time per handle and device
    cudaStream_t copy = nullptr, comp = nullptr;
    cudaEvent_t copied[kStreamBufs] = {}, scanned[kStreamBufs] = {};
    uint8_t *d_text[kStreamBufs] = {};
    uint8_t *h_stage[kStreamBufs] = {};
    uint64_t text_cap = 0, stage_cap = 0;
    void *d_ws = nullptr;
    uint64_t ws_cap = 0;
    uint64_t *d_pos = nullptr;  // chunk c's rows at [c * per_chunk, ...)
    uint32_t *d_pid = nullptr;
    uint64_t out_cap = 0;
    uint64_t *d_count = nullptr;  // per chunk
    uint64_t *h_count = nullptr;  // pinned, per chunk
    uint64_t count_cap = 0;
};

struct pfac_trie {
    std::vector<uint8_t> image;
    ImageHeader hdr;
    std::mutex mu;                  // guards dev / ctx (lazy per-device state)
    std::map<int, void *> dev;      // device ordinal -> device copy of the image
    std::map<int, std::unique_ptr<HostCtx>> ctx;
};

namespace {

thread_local std::string g_err;

pfac_status fail(int st, const std::string &msg) {
    g_err = msg;
    return (pfac_status)st;
}

pfac_status cuda_fail(const char *what, cudaError_t e) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return PFAC_ERR_CUDA;
}

pfac_status finish_handle(std::vector<uint8_t> &&img, pfac_trie **out) {
    pfac_trie *t = new (std::nothrow) pfac_trie();
    if (!t) return fail(kStatusNomem, "out of host memory");
    t->image = std::move(img);
    std::memcpy(&t->hdr, t->image.data(), sizeof(ImageHeader));
    *out = t;
    return PFAC_OK;
}

// Device copy of the image on `device` (uploaded on first use).
pfac_status device_image(const pfac_trie *tc, int device, const uint8_t **d_img) {
    pfac_trie *t = const_cast<pfac_trie *>(tc);
    std::lock_guard<std::mutex> lk(t->mu);
    auto it = t->dev.find(device);
    if (it != t->dev.end()) {
        *d_img = static_cast<const uint8_t *>(it->second);
        return PFAC_OK;
    }
    int prev = -1;
    cudaError_t e = cudaGetDevice(&prev);
    if (e != cudaSuccess) return cuda_fail("cudaGetDevice", e);
    if (prev != device && (e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail("cudaSetDevice", e);
    void *p = nullptr;
    e = cudaMalloc(&p, t->image.size());
    if (e == cudaSuccess) e = cudaMemcpy(p, t->image.data(), t->image.size(), cudaMemcpyHostToDevice);
    if (prev != device) cudaSetDevice(prev);
    if (e != cudaSuccess) {
        if (p) cudaFree(p);
        return cuda_fail("uploading the trie image", e);
    }
    t->dev[device] = p;
    *d_img = static_cast<const uint8_t *>(p);
    return PFAC_OK;
}

}  // namespace

extern "C" {

void pfac_build_options_init(pfac_build_options *o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->struct_bytes = sizeof *o;
    o->filter_kind = -1;
}

void pfac_plan_options_init(pfac_plan_options *o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->struct_bytes = sizeof *o;
    o->placement = PFAC_PLACE_AUTO;
    o->max_filter_rep_log2 = -1;
    o->ring_slots = -1;
    o->ctg64 = -1;
    o->pool64 = -1;
    o->stage2 = -1;
    o->entry = -1;
}

static pfac_status build_with(const uint8_t *const *patterns, const uint32_t *lengths, uint32_t n_patterns,
                              const BuildOpts &bo, pfac_trie **out) {
    try {
        std::vector<uint8_t> img;
        std::string err;
        int st = build_image(patterns, lengths, n_patterns, bo, img, err);
        if (st != kStatusOk) return fail(st, err);
        return finish_handle(std::move(img), out);
    } catch (const std::bad_alloc &) {
        return fail(kStatusNomem, "pfac_build: out of host memory");
    } catch (...) {
        return fail(kStatusInvalid, "pfac_build: unexpected error");
    }
}

pfac_status pfac_build(const uint8_t *const *patterns, const uint32_t *lengths, uint32_t n_patterns,
                       pfac_trie **out) {
    if (!out) return fail(kStatusInvalid, "pfac_build: out is NULL");
    *out = nullptr;
    try {
        std::vector<uint8_t> img;
        std::string err;
        int st = build_image(patterns, lengths, n_patterns, BuildOpts(), img, err);
        if (st != kStatusOk) return fail(st, err);
        return finish_handle(std::move(img), out);
    } catch (const std::bad_alloc &) {
        return fail(kStatusNomem, "pfac_build: out of host memory");
    } catch (...) {
        return fail(kStatusInvalid, "pfac_build: unexpected error");
    }
}

pfac_status pfac_build_concat(const uint8_t *data, const uint32_t *lengths, uint32_t n_patterns, pfac_trie **out) {
    if (!out) return fail(kStatusInvalid, "pfac_build_concat: out is NULL");
    *out = nullptr;
    if (!lengths || n_patterns == 0) return fail(kStatusInvalid, "pfac_build_concat: no patterns");
    try {
        std::vector<const uint8_t *> ptrs(n_patterns);
        uint64_t off = 0;
        for (uint32_t k = 0; k < n_patterns; k++) {
            ptrs[k] = data ? data + off : nullptr;
            off += lengths[k];
        }
        return pfac_build(ptrs.data(), lengths, n_patterns, out);
    } catch (...) {
        return fail(kStatusNomem, "pfac_build_concat: out of host memory");
    }
}

pfac_status pfac_build_ex(const uint8_t *data, const uint32_t *lengths, uint32_t n_patterns,
                          const pfac_build_options *opt, pfac_trie **out) {
    if (!out) return fail(kStatusInvalid, "pfac_build_ex: out is NULL");
    *out = nullptr;
    if (!lengths || n_patterns == 0) return fail(kStatusInvalid, "pfac_build_ex: no patterns");
    BuildOpts bo;
    if (opt) {
        bool ok = opt->struct_bytes >= sizeof(pfac_build_options) && opt->filter_kind >= -1 && opt->filter_kind <= 4;
        for (uint32_t r : opt->reserved) ok = ok && r == 0;
        if (!ok) return fail(kStatusInvalid, "pfac_build_ex: bad struct_bytes, filter_kind or reserved field");
        bo.filter_kind = opt->filter_kind;
        if (opt->pair_bits_per_key) bo.pair_bits_per_key = opt->pair_bits_per_key;
        if (opt->gram8_bits_per_key) bo.gram8_bits_per_key = opt->gram8_bits_per_key;
        bo.truncate_depth = opt->truncate_depth;
        if (opt->merge_suffixes > 1) return fail(kStatusInvalid, "pfac_build_ex: merge_suffixes must be 0 or 1");
        bo.merge_suffixes = opt->merge_suffixes;
    }
    try {
        std::vector<const uint8_t *> ptrs(n_patterns);
        uint64_t off = 0;
        for (uint32_t k = 0; k < n_patterns; k++) {
            ptrs[k] = data ? data + off : nullptr;
            off += lengths[k];
        }
        return build_with(ptrs.data(), lengths, n_patterns, bo, out);
    } catch (...) {
        return fail(kStatusNomem, "pfac_build_ex: out of host memory");
    }
}

void pfac_free(pfac_trie *t) {
    if (!t) return;
    int prev = -1;
    bool have = cudaGetDevice(&prev) == cudaSuccess;
    for (auto &kv : t->dev) {
        if (!have) break;
        cudaSetDevice(kv.first);
        cudaFree(kv.second);
    }
    for (auto &kv : t->ctx) {
        if (!have) break;
        HostCtx &c = *kv.second;
        cudaSetDevice(kv.first);
        if (c.copy) cudaStreamSynchronize(c.copy);
        if (c.comp) cudaStreamSynchronize(c.comp);
        for (int b = 0; b < kStreamBufs; b++) {
            cudaFree(c.d_text[b]);
            cudaFreeHost(c.h_stage[b]);
            if (c.copied[b]) cudaEventDestroy(c.copied[b]);
            if (c.scanned[b]) cudaEventDestroy(c.scanned[b]);
        }
        cudaFree(c.d_ws); cudaFree(c.d_pos); cudaFree(c.d_pid); cudaFree(c.d_count);
        cudaFreeHost(c.h_count);
        if (c.copy) cudaStreamDestroy(c.copy);
        if (c.comp) cudaStreamDestroy(c.comp);
    }
    if (have) cudaSetDevice(prev);
    delete t;
}

pfac_status pfac_trie_bytes(const pfac_trie *t, pfac_bytes_kind kind, uint64_t *out) {
    if (!t || !out) return fail(kStatusInvalid, "pfac_trie_bytes: NULL argument");
    switch (kind) {
    case PFAC_BYTES_DEVICE_IMAGE: *out = t->hdr.image_bytes; break;
    case PFAC_BYTES_UNCOMPRESSED: *out = t->hdr.bytes_uncompressed; break;
    case PFAC_BYTES_DENSE_STT: *out = t->hdr.bytes_dense_stt; break;
    case PFAC_BYTES_PAPER_CRS: *out = t->hdr.bytes_paper_crs; break;
    case PFAC_BYTES_CSR_CORE: *out = t->hdr.bytes_csr_core; break;
    case PFAC_BYTES_TRUNCATED: *out = t->hdr.bytes_truncated; break;
    case PFAC_BYTES_MERGED:
    case PFAC_BYTES_MERGED_CRS:
    case PFAC_BYTES_MERGED_IMAGE:
    case PFAC_BYTES_PIPE_TRUNC:
    case PFAC_BYTES_PIPE_MERGED:
    case PFAC_BYTES_PIPE_CRS: {
        const ImageHeader &h = t->hdr;
        if (!h.n_dag_nodes) return fail(kStatusInvalid, "pfac_trie_bytes: the trie was built without merge_suffixes");
        *out = kind == PFAC_BYTES_MERGED       ? h.bytes_merged
               : kind == PFAC_BYTES_MERGED_CRS ? h.bytes_merged_crs
               : kind == PFAC_BYTES_MERGED_IMAGE
                   ? 4 * (h.n_dag_nodes + 1) + 9 * h.n_dag_edges + 4 * h.n_terminals
               : kind == PFAC_BYTES_PIPE_TRUNC  ? h.bytes_pipe_trunc
               : kind == PFAC_BYTES_PIPE_MERGED ? h.bytes_pipe_merged
                                                : h.bytes_pipe_crs;
        break;
    }
    default: return fail(kStatusInvalid, "pfac_trie_bytes: bad kind");
    }
    return PFAC_OK;
}

pfac_status pfac_trie_stats(const pfac_trie *t, pfac_stats *o) {
    if (!t || !o) return fail(kStatusInvalid, "pfac_trie_stats: NULL argument");
    std::memset(o, 0, sizeof *o);
    o->nodes = t->hdr.n_nodes_full;
    o->edges = t->hdr.n_nodes_full - 1;
    o->image_nodes = t->hdr.n_nodes;
    o->terminals = t->hdr.n_terminals;
    o->n_patterns = t->hdr.n_patterns;
    o->max_len = t->hdr.max_len;
    o->min_len = t->hdr.min_len;
    o->filter_gram = t->hdr.filter_gram;
    o->filter_log2_bits = t->hdr.filter_log2_bits;
    o->truncate_depth = t->hdr.trunc_depth;
    o->verify_candidates = (uint32_t)t->hdr.n_cand;
    return PFAC_OK;
}

pfac_status pfac_image(const pfac_trie *t, const void **host_bytes, uint64_t *size) {
    if (!t || !host_bytes || !size) return fail(kStatusInvalid, "pfac_image: NULL argument");
    *host_bytes = t->image.data();
    *size = t->image.size();
    return PFAC_OK;
}

pfac_status pfac_attach(const void *image, uint64_t size, int device, pfac_trie **out) {
    if (!out || !image) return fail(kStatusInvalid, "pfac_attach: NULL argument");
    *out = nullptr;
    try {
        std::vector<uint8_t> img(size);
        cudaPointerAttributes attr;
        cudaError_t e = cudaPointerGetAttributes(&attr, image);
        if (e != cudaSuccess) cudaGetLastError();  // plain host pointer on older runtimes
        if (e == cudaSuccess && attr.type == cudaMemoryTypeDevice) {
            e = cudaMemcpy(img.data(), image, size, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) return cuda_fail("pfac_attach: copying the device image", e);
        } else {
            std::memcpy(img.data(), image, size);
        }
        std::string err;
        int st = validate_image(img.data(), size, err);
        if (st != kStatusOk) return fail(st, err);
        pfac_status s = finish_handle(std::move(img), out);
        if (s != PFAC_OK) return s;
        const uint8_t *d = nullptr;
        if (device >= 0) {
            s = device_image(*out, device, &d);
            if (s != PFAC_OK) {
                pfac_free(*out);
                *out = nullptr;
                return s;
            }
        }
        return PFAC_OK;
    } catch (const std::bad_alloc &) {
        return fail(kStatusNomem, "pfac_attach: out of host memory");
    }
}

pfac_status pfac_workspace_bytes(const pfac_trie *t, uint64_t n_starts, uint64_t *out) {
    if (!t || !out) return fail(kStatusInvalid, "pfac_workspace_bytes: NULL argument");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail("pfac_workspace_bytes: no CUDA device", e);
    std::string err;
    int st = workspace_bytes_for(n_starts, dev, out, err);
    if (st != kStatusOk) return fail(st, err);
    return PFAC_OK;
}

pfac_status pfac_match_device_ex(const pfac_trie *t, int device, const uint8_t *d_text, uint64_t readable_len,
                                 uint64_t n_starts, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                                 uint64_t capacity, uint64_t *d_count, void *d_workspace, uint64_t workspace_bytes,
                                 const pfac_plan_options *opt, pfac_stream stream) {
    const NvtxRange range("pfac_match_device");
    if (!t || !d_count || (n_starts && !d_text) || (capacity && (!d_pos || !d_pid)))
        return fail(kStatusInvalid, "pfac_match_device: NULL argument");
    if (n_starts > readable_len) return fail(kStatusInvalid, "pfac_match_device: n_starts > readable_len");
    int cur = -1;
    cudaError_t e = cudaGetDevice(&cur);
    if (e != cudaSuccess) return cuda_fail("pfac_match_device: no CUDA device", e);
    if (cur != device) return fail(kStatusInvalid, "pfac_match_device: `device` is not the current CUDA device");
    pfac_plan_options defaults;
    pfac_plan_options_init(&defaults);
    const uint8_t *d_img = nullptr;
    pfac_status s = device_image(t, device, &d_img);
    if (s != PFAC_OK) return s;
    DevTrie dt = make_dev_trie(t->hdr, d_img);
    std::string err;
    int st;
    if (opt && opt->struct_bytes >= sizeof(pfac_plan_options) && opt->form == PFAC_FORM_MERGED_DAG)
        st = launch_dag(t->hdr, d_img, d_text, readable_len, n_starts, pos_base, d_pos, d_pid, capacity, d_count,
                        d_workspace, workspace_bytes, reinterpret_cast<CUstream_st *>(stream), err);
    else
        st = launch_scan(dt, t->image.data(), device, d_text, readable_len, n_starts, pos_base, d_pos, d_pid,
                         capacity, d_count, d_workspace, workspace_bytes, opt ? *opt : defaults,
                         reinterpret_cast<CUstream_st *>(stream), err);
    if (st != kStatusOk) return fail(st, err);
    return PFAC_OK;
}

pfac_status pfac_match_device(const pfac_trie *t, int device, const uint8_t *d_text, uint64_t readable_len,
                              uint64_t n_starts, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid,
                              uint64_t capacity, uint64_t *d_count, void *d_workspace, uint64_t workspace_bytes,
                              pfac_stream stream) {
    return pfac_match_device_ex(t, device, d_text, readable_len, n_starts, pos_base, d_pos, d_pid, capacity, d_count,
                                d_workspace, workspace_bytes, nullptr, stream);
}

pfac_status pfac_plan_query(const pfac_trie *t, int device, uint64_t n_starts, const pfac_plan_options *opt,
                            pfac_plan_info *out) {
    if (!t || !out) return fail(kStatusInvalid, "pfac_plan_query: NULL argument");
    pfac_plan_options defaults;
    pfac_plan_options_init(&defaults);
    // the plan depends on which image sections exist, not on device addresses:
    // a placeholder base (never dereferenced) keeps present sections non-null
    DevTrie dt = make_dev_trie(t->hdr, reinterpret_cast<const uint8_t *>(uintptr_t(1) << 40));
    std::string err;
    int st = plan_query(dt, t->image.data(), device, n_starts, opt ? *opt : defaults, out, err);
    if (st != kStatusOk) return fail(st, err);
    return PFAC_OK;
}

pfac_status pfac_match(const pfac_trie *t, const uint8_t *text, uint64_t len, pfac_matches *out) {
    const NvtxRange range("pfac_match");
    if (!t || !out || (len && !text)) return fail(kStatusInvalid, "pfac_match: NULL argument");
    out->count = 0;
    out->pos = nullptr;
    out->pid = nullptr;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail("pfac_match: no CUDA device", e);
    const uint8_t *d_img = nullptr;
    pfac_status rs = device_image(t, dev, &d_img);
    if (rs != PFAC_OK || len == 0) return rs;
    HostCtx *cp;
    {
        pfac_trie *tm = const_cast<pfac_trie *>(t);
        std::lock_guard<std::mutex> lk(tm->mu);
        auto &slot = tm->ctx[dev];
        if (!slot) slot.reset(new (std::nothrow) HostCtx());
        if (!slot) return fail(kStatusNomem, "pfac_match: out of host memory");
        cp = slot.get();
    }
    HostCtx &c = *cp;
    std::lock_guard<std::mutex> lk(c.mu);
    // ---- geometry: chunks of PFAC_STREAM_CHUNK starts, each read with its halo
    const uint64_t C = PFAC_STREAM_CHUNK, halo = t->hdr.max_len - 1;
    const uint64_t n_chunks = (len + C - 1) / C;
    const uint64_t buf_bytes = (std::min(len, C + halo) + 15) & ~15ull;
    const uint64_t per_chunk = std::min(len, C) / 256 + 4096;  // row capacity per chunk (count-and-retry above)
    const int nbuf = (int)std::min<uint64_t>(n_chunks, kStreamBufs);
    cudaPointerAttributes attr;
    bool pinned = cudaPointerGetAttributes(&attr, text) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();  // (a plain pageable pointer is not an error)
    // ---- grow-only state
    if (!c.copy) {
        if ((e = cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&c.comp, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail("pfac_match: streams", e);
        for (int b = 0; b < kStreamBufs; b++)
            if ((e = cudaEventCreateWithFlags(&c.copied[b], cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&c.scanned[b], cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail("pfac_match: events", e);
    }
    if (buf_bytes > c.text_cap) {
        for (int b = 0; b < kStreamBufs; b++) {
            cudaFree(c.d_text[b]);
            c.d_text[b] = nullptr;
        }
        c.text_cap = 0;
        for (int b = 0; b < kStreamBufs; b++)
            if ((e = cudaMalloc(&c.d_text[b], buf_bytes)) != cudaSuccess) return cuda_fail("pfac_match: text buffers", e);
        c.text_cap = buf_bytes;
    }
    if (!pinned && buf_bytes > c.stage_cap) {
        for (int b = 0; b < kStreamBufs; b++) {
            cudaFreeHost(c.h_stage[b]);
            c.h_stage[b] = nullptr;
        }
        c.stage_cap = 0;
        for (int b = 0; b < kStreamBufs; b++)
            if ((e = cudaMallocHost(&c.h_stage[b], buf_bytes)) != cudaSuccess)
                return cuda_fail("pfac_match: pinned staging", e);
        c.stage_cap = buf_bytes;
    }
    uint64_t ws_bytes = 0;
    {
        std::string err;
        int st = workspace_bytes_for(std::min(len, C), dev, &ws_bytes, err);
        if (st != kStatusOk) return fail(st, err);
    }
    if (ws_bytes > c.ws_cap) {
        cudaFree(c.d_ws);
        c.d_ws = nullptr;
        c.ws_cap = 0;
        if ((e = cudaMalloc(&c.d_ws, ws_bytes)) != cudaSuccess ||
            (e = cudaMemsetAsync(c.d_ws, 0, ws_bytes, c.comp)) != cudaSuccess)
            return cuda_fail("pfac_match: workspace", e);
        c.ws_cap = ws_bytes;
    }
    if (n_chunks * per_chunk > c.out_cap) {
        cudaFree(c.d_pos);
        cudaFree(c.d_pid);
        c.d_pos = nullptr;
        c.d_pid = nullptr;
        c.out_cap = 0;
        if ((e = cudaMalloc(&c.d_pos, n_chunks * per_chunk * 8)) != cudaSuccess ||
            (e = cudaMalloc(&c.d_pid, n_chunks * per_chunk * 4)) != cudaSuccess)
            return cuda_fail("pfac_match: output buffers", e);
        c.out_cap = n_chunks * per_chunk;
    }
    if (n_chunks > c.count_cap) {
        cudaFree(c.d_count);
        cudaFreeHost(c.h_count);
        c.d_count = nullptr;
        c.h_count = nullptr;
        c.count_cap = 0;
        if ((e = cudaMalloc(&c.d_count, 8 * n_chunks)) != cudaSuccess ||
            (e = cudaMallocHost(&c.h_count, 8 * n_chunks)) != cudaSuccess)
            return cuda_fail("pfac_match: counts", e);
        c.count_cap = n_chunks;
    }
    // ---- the pipeline: copy chunk i on `copy` while chunk i-1 scans on `comp`
    auto chunk = [&](uint64_t i, uint64_t &s0, uint64_t &ns, uint64_t &rd) {
        s0 = i * C;
        ns = std::min(C, len - s0);
        rd = std::min(len - s0, ns + halo);
    };
    for (uint64_t i = 0; i < n_chunks; i++) {
        const int b = (int)(i % (uint64_t)nbuf);
        uint64_t s0, ns, rd;
        chunk(i, s0, ns, rd);
        if (i >= (uint64_t)nbuf && (e = cudaStreamWaitEvent(c.copy, c.scanned[b], 0)) != cudaSuccess)
            return cuda_fail("pfac_match: pipeline", e);
        const uint8_t *src = text + s0;
        if (!pinned) {  // pageable: through pinned staging (buffer b is free once its last copy is done)
            if (i >= (uint64_t)nbuf && (e = cudaEventSynchronize(c.copied[b])) != cudaSuccess)
                return cuda_fail("pfac_match: pipeline", e);
            std::memcpy(c.h_stage[b], src, rd);
            src = c.h_stage[b];
        }
        if ((e = cudaMemcpyAsync(c.d_text[b], src, rd, cudaMemcpyHostToDevice, c.copy)) != cudaSuccess ||
            (e = cudaEventRecord(c.copied[b], c.copy)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(c.comp, c.copied[b], 0)) != cudaSuccess)
            return cuda_fail("pfac_match: H2D", e);
        rs = pfac_match_device(t, dev, c.d_text[b], rd, ns, s0, c.d_pos + i * per_chunk, c.d_pid + i * per_chunk,
                               per_chunk, c.d_count + i, c.d_ws, c.ws_cap, reinterpret_cast<pfac_stream>(c.comp));
        if (rs != PFAC_OK) return rs;
        if ((e = cudaEventRecord(c.scanned[b], c.comp)) != cudaSuccess) return cuda_fail("pfac_match: pipeline", e);
    }
    if ((e = cudaMemcpyAsync(c.h_count, c.d_count, 8 * n_chunks, cudaMemcpyDeviceToHost, c.comp)) != cudaSuccess ||
        (e = cudaStreamSynchronize(c.comp)) != cudaSuccess)
        return cuda_fail("pfac_match: scan", e);
    uint64_t total = 0;
    for (uint64_t i = 0; i < n_chunks; i++) total += c.h_count[i];
    if (total == 0) return PFAC_OK;
    out->pos = static_cast<uint64_t *>(std::malloc(total * 8));
    out->pid = static_cast<uint32_t *>(std::malloc(total * 4));
    if (!out->pos || !out->pid) {
        pfac_matches_free(out);
        return fail(kStatusNomem, "pfac_match: out of host memory");
    }
    uint64_t at = 0;
    for (uint64_t i = 0; i < n_chunks; at += c.h_count[i], i++) {
        const uint64_t n = c.h_count[i];
        if (n == 0) continue;
        const uint64_t *dp = c.d_pos + i * per_chunk;
        const uint32_t *dq = c.d_pid + i * per_chunk;
        uint64_t *tp = nullptr;
        uint32_t *tq = nullptr;
        if (n > per_chunk) {  // more rows than the chunk's room: scan it again into buffers of its size
            uint64_t s0, ns, rd;
            chunk(i, s0, ns, rd);
            uint64_t *tc = nullptr;
            if ((e = cudaMalloc(&tp, n * 8)) != cudaSuccess || (e = cudaMalloc(&tq, n * 4)) != cudaSuccess ||
                (e = cudaMalloc(&tc, 8)) != cudaSuccess ||
                (e = cudaMemcpyAsync(c.d_text[0], text + s0, rd, cudaMemcpyHostToDevice, c.comp)) != cudaSuccess) {
                cudaFree(tp); cudaFree(tq); cudaFree(tc);
                pfac_matches_free(out);
                return cuda_fail("pfac_match: retry buffers", e);
            }
            rs = pfac_match_device(t, dev, c.d_text[0], rd, ns, s0, tp, tq, n, tc, c.d_ws, c.ws_cap,
                                   reinterpret_cast<pfac_stream>(c.comp));
            cudaFree(tc);  // (stream-ordered free is not needed: the count is not read)
            if (rs != PFAC_OK) {
                cudaFree(tp); cudaFree(tq);
                pfac_matches_free(out);
                return rs;
            }
            dp = tp;
            dq = tq;
        }
        if ((e = cudaMemcpyAsync(out->pos + at, dp, n * 8, cudaMemcpyDeviceToHost, c.comp)) != cudaSuccess ||
            (e = cudaMemcpyAsync(out->pid + at, dq, n * 4, cudaMemcpyDeviceToHost, c.comp)) != cudaSuccess ||
            (e = cudaStreamSynchronize(c.comp)) != cudaSuccess) {
            cudaFree(tp); cudaFree(tq);
            pfac_matches_free(out);
            return cuda_fail("pfac_match: D2H", e);
        }
        cudaFree(tp);
        cudaFree(tq);
    }
    out->count = total;
    return PFAC_OK;
}

void pfac_matches_free(pfac_matches *m) {
    if (!m) return;
    std::free(m->pos);
    std::free(m->pid);
    m->pos = nullptr;
    m->pid = nullptr;
    m->count = 0;
}

uint32_t pfac_launches_per_call(void) { return launches_per_call(); }

const char *pfac_status_string(pfac_status s) {
    switch (s) {
    case PFAC_OK: return "PFAC_OK";
    case PFAC_ERR_INVALID_ARG: return "PFAC_ERR_INVALID_ARG";
    case PFAC_ERR_LIMIT: return "PFAC_ERR_LIMIT";
    case PFAC_ERR_NOMEM: return "PFAC_ERR_NOMEM";
    case PFAC_ERR_CUDA: return "PFAC_ERR_CUDA";
    case PFAC_ERR_CAPACITY: return "PFAC_ERR_CAPACITY";
    }
    return "PFAC_ERR_UNKNOWN";
}

const char *pfac_last_error(void) { return g_err.c_str(); }

const char *pfac_version(void) { return "pfac-b200 0.1 sm_100a"; }

#ifdef PFAC_TIMING
// Instrumented build only: copy the per-warp stamps of the last launch.
int pfac_debug_timing(unsigned long long *host, uint64_t n) { return pfac::debug_timing(host, n); }
#endif

}  // extern "C"

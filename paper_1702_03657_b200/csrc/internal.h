// internal.h -- declarations shared by the product's translation units
// (builder.cpp, abi.cpp, scan.cu).  Not part of the public ABI (include/pfac.h).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "image.h"
#include "pfac.h"

struct CUstream_st;
#include <vector_types.h>

namespace pfac {

#ifdef PFAC_CHECKED
// Bounds-checked build (libpfac_checked.so; tools/checked_tests.sh): every
// index the kernel follows into an image section, a shared-memory table, a
// queue or a workspace array is asserted, and a failed check traps (the
// launch fails).  It stands in for compute-sanitizer, which this GPU pool
// does not allow.
#define PFAC_CHECK(c)          \
    do {                       \
        if (!(c)) __trap();    \
    } while (0)
#else
#define PFAC_CHECK(c) \
    do {              \
    } while (0)
#endif


// mirrors pfac_status in include/pfac.h
enum : int {
    kStatusOk = 0,
    kStatusInvalid = 1,
    kStatusLimit = 2,
    kStatusNomem = 3,
    kStatusCuda = 4,
    kStatusCapacity = 5,
};

constexpr uint32_t kMaxPatternLen = 65535;
constexpr uint64_t kMaxPidEntries = 1ull << 28;  // total length of the per-terminal pid lists

// Build options (include/pfac.h pfac_build_options, defaults filled in).
struct BuildOpts {
    int filter_kind = -1;              // -1 automatic
    uint32_t pair_bits_per_key = 512;  // kind 2 sizing
    uint32_t gram8_bits_per_key = 32;  // kind 4 sizing
    uint32_t truncate_depth = 0;       // 0: untruncated
    uint32_t merge_suffixes = 0;       // 1: also build the id-preserving merged DAG (steps IV-V)
};

int build_image(const uint8_t *const *pats, const uint32_t *lens, uint32_t m, const BuildOpts &opt,
                std::vector<uint8_t> &image, std::string &err);
int validate_image(const uint8_t *p, uint64_t size, std::string &err);

// Device-side view of an uploaded image (pointers into device memory).
struct DevTrie {
    const uint32_t *node;
    const uint32_t *aux;  // per node: record index or packed labels (image.h)
    const uint4 *rec;     // per node: {node[v], node[v+1], aux[v], 0} (image.h)
    const uint8_t *label;
    const uint32_t *term_node;
    const uint2 *term_rk;  // kept-terminal rank {bits, rank} per 32 nodes (image v22)
    const uint32_t *out_ptr;
    const uint32_t *out_pid;
    const uint32_t *root;
    const uint32_t *filter;
    const uint32_t *tail_bits;
    const uint32_t *tail_rank;
    const uint4 *tails;
    const uint8_t *tail_bytes;
    const uint32_t *level1;
    const uint32_t *pair;  // 2-gram prefix table [256][8]
    const uint32_t *kset;  // exact key set (nullptr: none)
    uint32_t kset_log2, kset_empty;
    const uint4 *entry;   // depth-8 entry table (nullptr: none)
    uint32_t entry_log2;
    uint32_t n_terminals;
    uint32_t n_kept_terminals;
    uint32_t max_len;
    uint32_t gram;
    uint32_t log2_bits;
    uint32_t exact;
    uint32_t kind;       // filter kind (image.h)
    uint32_t n_nodes;
    // section sizes (bounds of the checked build, PFAC_CHECKED)
    uint32_t n_edges, n_records, n_tail_bytes, n_out, n_level1;
};

DevTrie make_dev_trie(const ImageHeader &h, const uint8_t *d_image);

// Workspace bytes for n_starts starts on `device` (caller-owned, zero-filled
// before first use).
int workspace_bytes_for(uint64_t n_starts, int device, uint64_t *out, std::string &err);

// Launches the scan with plan options `o` (defaults: pfac_plan_options_init);
// returns kStatusOk or an error status (err filled).
int launch_scan(const DevTrie &t, const uint8_t *host_image, int device, const uint8_t *d_text, uint64_t readable_len,
                uint64_t n_starts, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid, uint64_t capacity,
                uint64_t *d_count, void *d_ws, uint64_t ws_bytes, const pfac_plan_options &o, CUstream_st *stream,
                std::string &err);
// The plan a scan would use (no launch).
int plan_query(const DevTrie &t, const uint8_t *host_image, int device, uint64_t n_starts,
               const pfac_plan_options &o, pfac_plan_info *out, std::string &err);

uint32_t launches_per_call();

// The merged-DAG scan (dag.cu; plan form PFAC_FORM_MERGED_DAG): three
// stream-ordered launches; its block totals live at kWsDagOffset of the
// caller's workspace (after the main scan's header and CTA totals).
constexpr uint64_t kWsDagOffset = 256 + 16 * 1024;
uint64_t dag_workspace_bytes(uint64_t n_starts);
int launch_dag(const ImageHeader &h, const uint8_t *d_img, const uint8_t *d_text, uint64_t readable_len,
               uint64_t n_starts, uint64_t pos_base, uint64_t *d_pos, uint32_t *d_pid, uint64_t capacity,
               uint64_t *d_count, void *d_ws, uint64_t ws_bytes, CUstream_st *stream, std::string &err);
#ifdef PFAC_TIMING
int debug_timing(unsigned long long *host, uint64_t n);
#endif

}  // namespace pfac

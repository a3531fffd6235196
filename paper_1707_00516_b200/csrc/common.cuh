// Shared helpers for the FastID sm_100a library: status plumbing, launch
// checks and the register-resident top-k list used by every epilogue.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>

#include "fastid_b200.h"

namespace fastid {

// Thread-local error message behind fastid_last_error().
void set_error(const char* fmt, ...);
const char* get_error();

#define FASTID_FAIL(code, ...)                 \
    do {                                       \
        ::fastid::set_error(__VA_ARGS__);      \
        return (code);                         \
    } while (0)

#define FASTID_CUDA(expr)                                                                     \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            FASTID_FAIL(FASTID_E_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                        __FILE__, __LINE__);                                                  \
    } while (0)

// Kernels this library has enqueued in this process (fastid_launch_count).
void note_launch();

#define FASTID_LAUNCHED(name)                                                                   \
    do {                                                                                        \
        cudaError_t _e = cudaGetLastError();                                                    \
        if (_e != cudaSuccess)                                                                  \
            FASTID_FAIL(FASTID_E_CUDA, "launch of %s failed: %s", name, cudaGetErrorString(_e)); \
        ::fastid::note_launch();                                                                \
    } while (0)

constexpr int kMaxTopK = 32;
constexpr int kMaxMergeLists = 768;  // candidate lists one merge folds per unknown (merge.cu)
constexpr int kScanAutoMaxQueries = 4;  // auto top-k on packed rows: the CUDA-core scan up to this many unknowns
constexpr int kMinSlots = 32;  // lists per unknown that publish their best value (shared top-k bound)
constexpr uint32_t kEmptyScore = 0xFFFFFFFFu;
constexpr uint32_t kEmptyLocal = 0xFFFFFFFFu;

inline int64_t row_stride_bytes(int64_t bit_length) { return ((bit_length + 127) / 128) * 16; }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Streaming multiprocessors of the current device (148 on a B200), cached.
int num_sms();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when `bytes` exceeds what
// was already set for `fn` on the current device (the call costs 5-30 us of host
// time; a small comparison's whole kernel is ~25 us).
cudaError_t ensure_dynamic_smem(const void* fn, int bytes);

// (score, index) lexicographic order: the canonical tie-break of every top-k
// output (score ascending, then known index ascending).
__device__ __forceinline__ bool before(uint32_t s0, uint32_t i0, uint32_t s1, uint32_t i1) {
    return s0 < s1 || (s0 == s1 && i0 < i1);
}

// A sorted list of K (score, local index) pairs held in registers.  Offers are
// rare after warm-up (a candidate must beat the current K-th entry), so the
// unrolled bubble insertion costs little; all indexing is static.
template <int K>
struct TopList {
    uint32_t s[K];
    uint32_t x[K];

    __device__ __forceinline__ void clear() {
#pragma unroll
        for (int i = 0; i < K; ++i) {
            s[i] = kEmptyScore;
            x[i] = kEmptyLocal;
        }
    }
    __device__ __forceinline__ bool admits(uint32_t v, uint32_t idx) const {
        return before(v, idx, s[K - 1], x[K - 1]);
    }
    __device__ __forceinline__ void insert(uint32_t v, uint32_t idx) {
        s[K - 1] = v;
        x[K - 1] = idx;
#pragma unroll
        for (int p = K - 1; p > 0; --p) {
            const bool sw = before(s[p], x[p], s[p - 1], x[p - 1]);
            const uint32_t ts = sw ? s[p - 1] : s[p];
            const uint32_t tx = sw ? x[p - 1] : x[p];
            s[p - 1] = sw ? s[p] : s[p - 1];
            x[p - 1] = sw ? x[p] : x[p - 1];
            s[p] = ts;
            x[p] = tx;
        }
    }
    // Insert a value whose index is larger than every index already listed (a
    // scan in row order), so it goes after every entry with score <= v.  All K
    // positions update in parallel from one predicate vector: depth 3 instead
    // of the K-step dependent chain of insert().
    __device__ __forceinline__ void insert_last(uint32_t v, uint32_t idx) {
        bool le[K];
#pragma unroll
        for (int i = 0; i < K; ++i) le[i] = s[i] <= v;
#pragma unroll
        for (int i = K - 1; i > 0; --i) {
            const bool prev_le = le[i - 1];
            s[i] = le[i] ? s[i] : (prev_le ? v : s[i - 1]);
            x[i] = le[i] ? x[i] : (prev_le ? idx : x[i - 1]);
        }
        s[0] = le[0] ? s[0] : v;
        x[0] = le[0] ? x[0] : idx;
    }
    __device__ __forceinline__ void offer(uint32_t v, uint32_t idx, uint32_t max_score) {
        if (v <= max_score && admits(v, idx)) insert(v, idx);
    }
    // Write the list as one partial candidate list: scores / global indices.
    __device__ __forceinline__ void store(uint32_t* scores, int64_t* index, int64_t base) const {
#pragma unroll
        for (int i = 0; i < K; ++i) {
            scores[i] = s[i];
            index[i] = s[i] == kEmptyScore ? -1 : base + (int64_t)x[i];
        }
    }
};

// Kernel-side description of one comparison job (device rows of `stride` bytes).
struct CompareArgs {
    const uint8_t* refs;
    const uint8_t* queries;
    int64_t n_refs;
    int64_t n_queries;
    int64_t stride;      // bytes per row, multiple of 16
    int64_t bit_length;
    // optional pre-unpacked tensor image of the refs (prepared database), else null
    const uint8_t* image;
    // full matrix
    uint32_t* out;
    int64_t ld_out;
    // top-k
    int k;
    uint32_t max_score;
    uint32_t* part_scores;  // [n_parts][n_queries][kpad]
    int64_t* part_index;
    int kpad;
    uint32_t* bound;        // [n_queries] shared top-k admission bound, 0xFFFFFFFF-initialised per launch: tensor
                            // kernels keep raw score bits (admit v < bound), the CUDA-core scan a score (admit v <= bound)
    uint32_t* list_min;     // [n_queries][kMinSlots] best value published by each of the first kMinSlots lists
    // CTA-pair kernel: per (slice, unknown group) tile progress, for drift control
    int* progress;
    int n_groups;
    int drift_tiles;  // max lead (tiles) of a pair over the slowest pair of its slice
    int drift_every;  // tiles between progress checks
    int dual_lag;     // dual-tile pairs: stages the second tile lags the first (-1 = default)
    int dual_sa;      // dual-tile pairs: A ring depth (0 = default)
    int l2_prefetch;  // pair kernels: L2-prefetch the known-tile stream ahead of the TMA loads
    int tma_out;  // full matrix through TMA tensor stores: 1 per-warp blocks, 2 per-split blocks (set by the launcher)
    // CTA-pair kernel: spare pairs and the tiles the regular slices cover (the rest go to spares)
    int n_spare;
    int64_t t_main;
    // operator (FASTID_OP_*) and, for XOR on the tensor kernels, the rows' popcounts
    // (mxf4 accumulates pr - 2 * and with a signed unknown operand and adds pq; i8
    // accumulates and and forms pr + pq - 2 * and)
    int op;
    const uint32_t* ref_popc;    // XOR on i8: known-row popcounts, popcount_entries(n_refs) long (zero-padded)
    const uint32_t* query_popc;  // XOR: [n_queries] unknown-row popcounts (fp32 bits for mxf4)
    // threshold
    uint32_t threshold;
    int64_t ref_base;
    uint32_t* hit_query;
    int64_t* hit_ref;
    uint32_t* hit_score;
    int64_t capacity;
    unsigned long long* hit_count;
    // Execution variants of a prepared database (fastid_db_set_option): every
    // one computes the same result; they select among kernel paths
    // (FASTID_OPT_* bits, include/fastid_b200.h).
    int options;
    // Diagnostics.  Only the experiments build (-DFASTID_EXPERIMENTS,
    // _fastid_b200_diag.so, include/fastid_b200_diag.h) reads these; in the
    // product library every branch on them is compiled out (see experiment()).
    long long* trace;  // CTA 0 timestamps, or null
    int trace_tiles;
    int debug_flags;  // bit 0: epilogue skips TMEM loads; bit 2: pairs skip operand loads; bit 3: trace MMA stage waits; bit 4: no top-k insertions; bit 5: count insertions per tile; bit 6: per-CTA globaltimer stamps; bit 7: host phase timings; bit 9: weighted (not uniform) mxf4 image encoding; bit 12: spinning (no suspend hint) accumulator waits; bit 13: spinning producer waits (timing experiments only; several invalidate results)
};

#ifdef FASTID_EXPERIMENTS
constexpr bool kExperiments = true;
#else
constexpr bool kExperiments = false;
#endif

// Experiment switch `bit` of a launch: always false in the product library.
__host__ __device__ __forceinline__ bool experiment(const CompareArgs& a, int bit) {
    return kExperiments && (a.debug_flags & bit) != 0;
}
// Diagnostic trace buffer of a launch: always null in the product library.
__host__ __device__ __forceinline__ long long* trace_buf(const CompareArgs& a) {
    return kExperiments ? a.trace : nullptr;
}

// Per-tile trace slots written by CTA 0 when tracing is on (clock64 values).
enum TraceSlot {
    kTrMmaWait = 0,     // MMA warp starts waiting for the accumulator
    kTrMmaGo = 1,       // ... accumulator free
    kTrMmaIssued = 2,   // last MMA of the tile issued + committed
    kTrEpi0 = 3,        // 16 slots: epilogue warp w acquired t_full (3 + w)
    kTrRel0 = 19,       // 16 slots: epilogue warp w released t_empty (19 + w)
    kTrB0Loaded = 35,   // 16 slots: batch 0 in registers
    kTrB0Done = 51,     // 16 slots: batch 0 processed
    kTrSlots = 67
};

enum Mode { kFull = 0, kTopK = 1, kThreshold = 2 };

// Append one threshold hit with a warp-aggregated slot reservation.
__device__ __forceinline__ void emit_hits(const CompareArgs& a, bool hit, uint32_t q, int64_t r,
                                          uint32_t v) {
    const unsigned mask = __activemask();
    const unsigned ballot = __ballot_sync(mask, hit);
    if (!ballot) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(ballot) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(a.hit_count, (unsigned long long)__popc(ballot));
    base = __shfl_sync(mask, base, leader);
    if (hit) {
        const unsigned long long slot = base + __popc(ballot & ((1u << lane) - 1u));
        if ((long long)slot < a.capacity) {
            a.hit_query[slot] = q;
            a.hit_ref[slot] = a.ref_base + r;
            a.hit_score[slot] = v;
        }
    }
}

// Host-side launchers implemented per formulation.
int launch_popc(Mode mode, const CompareArgs& a, int* n_parts, cudaStream_t stream);
int popc_parts(int64_t n_refs, int64_t n_queries);
int launch_tensor(Mode mode, const CompareArgs& a, int formulation, int* n_parts, cudaStream_t stream);
int tensor_parts(int64_t n_refs, int64_t n_queries, int formulation);
int tensor_supported(int64_t bit_length, int formulation);
size_t tensor_image_bytes(int64_t n_refs, int64_t bit_length, int formulation);
// popcount of each of `n` rows of `stride` bytes -> out[n] (u32, or the fp32 bits
// of the count when `as_float`: the mxf4 epilogue's XOR transform), zeros in
// out[n .. n_out), on `stream`
int launch_row_popcount(const uint8_t* rows, int64_t n, int64_t n_out, int64_t stride, bool as_float, uint32_t* out,
                        cudaStream_t stream);
// entries of a known-row popcount buffer: n rounded up to whole 256-row tiles
// (the XOR epilogue reads a full 32-column batch past the last row)
inline int64_t popcount_entries(int64_t n) { return (n + 255) / 256 * 256; }
int build_tensor_image(const CompareArgs& a, int formulation, void* image, cudaStream_t stream);
int launch_merge(const uint32_t* cand_scores, const int64_t* cand_index, int n_lists,
                 int64_t n_queries, int k_in, int k, uint32_t* top_scores, int64_t* top_index,
                 cudaStream_t stream);

}  // namespace fastid

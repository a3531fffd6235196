// Top-k combine: n_lists sorted candidate lists per query -> the first k by
// (score asc, known index asc).  Used twice: to fold the per-CTA partial
// lists of one device, and to fold the per-GPU lists after the NCCL gather
// (the multi-GPU driver's only exchange).
//
// One warp per query: lane l owns lists l, l+32, ... (up to 24 per lane, so
// n_lists <= 768); each of the k rounds takes the warp-wide minimum head and
// advances the winning list.  Few queries over many lists (a small batch's
// hundreds of per-CTA partials) take a block per query that first copies the
// lists into shared memory (merge_smem_kernel: one unknown, 444 lists, 39 ->
// 25 us).
#include "common.cuh"

namespace fastid {
namespace {

constexpr int kMaxListsPerLane = 24;

__device__ __forceinline__ bool key_before(uint32_t s0, uint64_t i0, uint32_t s1, uint64_t i1) {
    return s0 < s1 || (s0 == s1 && i0 < i1);
}

// The k-way merge of one query's lists by one warp, from a shared-memory copy
// of the lists ([list][k_in]): lane l holds the current head of each of its
// lists (l, l+32, ...) in registers, so a round is a register arg-min plus one
// load, the next entry of the list that won.  (The many-query kernel below
// reloads every head per round instead: fewer registers, more warps per SM.)
__device__ __forceinline__ void merge_query_smem(const uint32_t* __restrict__ cs, const int64_t* __restrict__ ci,
                                            int n_lists, int64_t n_queries, int64_t q, int k_in, int k,
                                            uint32_t* __restrict__ out_s, int64_t* __restrict__ out_i) {
    const int lane = threadIdx.x & 31;
    auto entry = [&](int l, int h) -> int64_t { return (int64_t)l * k_in + h; };
    int head[kMaxListsPerLane];
    uint32_t hs[kMaxListsPerLane];
    uint64_t hx[kMaxListsPerLane];
#pragma unroll
    for (int m = 0; m < kMaxListsPerLane; ++m) {
        const int l = lane + 32 * m;
        head[m] = 0;
        hs[m] = kEmptyScore;
        hx[m] = ~0ull;
        if (l < n_lists) {
            const int64_t off = entry(l, 0);
            hs[m] = cs[off];
            hx[m] = (uint64_t)ci[off];
        }
    }
    for (int o = 0; o < k; ++o) {
        // best head among this lane's lists (an empty entry ends a list)
        uint32_t bs = kEmptyScore;
        uint64_t bi = ~0ull;
        int bm = -1;
#pragma unroll
        for (int m = 0; m < kMaxListsPerLane; ++m) {
            if (hs[m] != kEmptyScore && key_before(hs[m], hx[m], bs, bi)) {
                bs = hs[m];
                bi = hx[m];
                bm = m;
            }
        }
        // warp arg-min over (score, index); ties on the full key cannot occur
        // between distinct lists because indices are unique
        uint32_t ws = bs;
        uint64_t wi = bi;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const uint32_t os = __shfl_xor_sync(0xffffffffu, ws, d);
            const uint64_t oi = __shfl_xor_sync(0xffffffffu, wi, d);
            if (key_before(os, oi, ws, wi)) {
                ws = os;
                wi = oi;
            }
        }
        if (bm >= 0 && bs == ws && bi == wi) {
#pragma unroll
            for (int m = 0; m < kMaxListsPerLane; ++m)
                if (m == bm) {
                    ++head[m];
                    hs[m] = kEmptyScore;
                    if (head[m] < k_in) {
                        const int64_t off = entry(lane + 32 * m, head[m]);
                        hs[m] = cs[off];
                        hx[m] = (uint64_t)ci[off];
                    }
                }
        }
        if (lane == 0) {
            out_s[q * k + o] = ws;
            out_i[q * k + o] = ws == kEmptyScore ? -1 : (int64_t)wi;
        }
    }
}

__global__ void __launch_bounds__(256) merge_kernel(const uint32_t* __restrict__ cs, const int64_t* __restrict__ ci, int n_lists,
                             int64_t n_queries, int k_in, int k, uint32_t* __restrict__ out_s,
                             int64_t* __restrict__ out_i) {
    const int lane = threadIdx.x & 31;
    const int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (q >= n_queries) return;
    int head[kMaxListsPerLane];
#pragma unroll
    for (int m = 0; m < kMaxListsPerLane; ++m) head[m] = 0;

    for (int o = 0; o < k; ++o) {
        // best head among this lane's lists
        uint32_t bs = kEmptyScore;
        uint64_t bi = ~0ull;
        int bm = -1;
#pragma unroll
        for (int m = 0; m < kMaxListsPerLane; ++m) {
            const int l = lane + 32 * m;
            if (l < n_lists && head[m] < k_in) {
                const int64_t off = ((int64_t)l * n_queries + q) * k_in + head[m];
                const uint32_t s = cs[off];
                const uint64_t i = (uint64_t)ci[off];
                if (s != kEmptyScore && key_before(s, i, bs, bi)) {
                    bs = s;
                    bi = i;
                    bm = m;
                }
            }
        }
        // warp arg-min over (score, index); ties on the full key cannot occur
        // between distinct lists because indices are unique
        uint32_t ws = bs;
        uint64_t wi = bi;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const uint32_t os = __shfl_xor_sync(0xffffffffu, ws, d);
            const uint64_t oi = __shfl_xor_sync(0xffffffffu, wi, d);
            if (key_before(os, oi, ws, wi)) {
                ws = os;
                wi = oi;
            }
        }
        if (bm >= 0 && bs == ws && bi == wi) {
#pragma unroll
            for (int m = 0; m < kMaxListsPerLane; ++m)
                if (m == bm) ++head[m];
        }
        if (lane == 0) {
            out_s[q * k + o] = ws;
            out_i[q * k + o] = ws == kEmptyScore ? -1 : (int64_t)wi;
        }
    }
}


// Few queries with many lists (a small batch over hundreds of CTAs' partials):
// one block per query copies all of its lists into shared memory with every
// thread (coalesced, all loads in flight at once), then one warp merges from
// there -- the global-memory merge pays a dependent load round trip per output
// (one unknown, 444 lists: ~70 us).
__global__ void __launch_bounds__(256) merge_smem_kernel(const uint32_t* __restrict__ cs, const int64_t* __restrict__ ci, int n_lists,
                                  int64_t n_queries, int k_in, int k, uint32_t* __restrict__ out_s,
                                  int64_t* __restrict__ out_i) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int64_t q = blockIdx.x;
    const int n = n_lists * k_in;
    int64_t* si = reinterpret_cast<int64_t*>(sm);
    uint32_t* ss = reinterpret_cast<uint32_t*>(sm + (size_t)n * sizeof(int64_t));
#pragma unroll 8
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const int l = t / k_in, h = t - l * k_in;
        const int64_t off = ((int64_t)l * n_queries + q) * k_in + h;
        ss[t] = __ldcg(cs + off);
        si[t] = __ldcg(ci + off);
    }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    merge_query_smem(ss, si, n_lists, n_queries, q, k_in, k, out_s, out_i);
}

}  // namespace

int launch_merge(const uint32_t* cs, const int64_t* ci, int n_lists, int64_t n_queries, int k_in, int k,
                 uint32_t* out_s, int64_t* out_i, cudaStream_t stream) {
    static_assert(32 * kMaxListsPerLane == kMaxMergeLists, "merge capacity");
    if (n_lists < 1 || n_lists > kMaxMergeLists)
        FASTID_FAIL(FASTID_E_INVALID, "n_lists must be in [1, %d], got %d", kMaxMergeLists, n_lists);
    if (k < 1 || k_in < 1) FASTID_FAIL(FASTID_E_INVALID, "k must be positive");
    if (n_queries == 0) return FASTID_OK;
    const size_t smem = (size_t)n_lists * k_in * (sizeof(int64_t) + sizeof(uint32_t));
    if (n_queries <= 2 * (int64_t)num_sms() && n_lists >= 64 && smem <= 160 * 1024) {
        FASTID_CUDA(ensure_dynamic_smem((const void*)merge_smem_kernel, (int)smem));
        merge_smem_kernel<<<(unsigned)n_queries, 256, smem, stream>>>(cs, ci, n_lists, n_queries, k_in, k, out_s,
                                                                      out_i);
        FASTID_LAUNCHED("merge_smem_kernel");
        return FASTID_OK;
    }
    const int64_t threads = n_queries * 32;
    const int block = 256;
    merge_kernel<<<(unsigned)ceil_div(threads, block), block, 0, stream>>>(cs, ci, n_lists, n_queries, k_in, k,
                                                                           out_s, out_i);
    FASTID_LAUNCHED("merge_kernel");
    return FASTID_OK;
}

}  // namespace fastid

extern "C" int fastid_merge_topk(const uint32_t* cand_scores, const int64_t* cand_index, int n_lists,
                                 int64_t n_queries, int k_in, int k, uint32_t* top_scores, int64_t* top_index,
                                 void* stream) {
    if (k > k_in) FASTID_FAIL(FASTID_E_INVALID, "k (%d) exceeds the candidate list length (%d)", k, k_in);
    return fastid::launch_merge(cand_scores, cand_index, n_lists, n_queries, k_in, k, top_scores, top_index,
                                (cudaStream_t)stream);
}

// Formulation A: the overloaded GEMM on CUDA cores.
//
// score(i, j) = sum_k POPC(R_i[k] AND NOT Q_j[k])   (Eq. 1, PAPER.md:41-45;
// reference _blocked_worker, pkg/src/fastid/kernel.py:238-269).  The AND-NOT
// lowers to one LOP3.LUT (0x30) and the count to POPC, so the kernel is bound
// by the POPC issue rate (16 lanes/clk/SM) -- DESIGN.md "Roofline".
//
// Tiling (the paper's §IV-B blocking, re-done for sm_100a): a CTA owns a
// 128-known x 128-unknown output tile; 256 threads each hold an 8 x 8
// register tile ("16 outputs per thread" in the paper, 64 here) over
// known rows ty + 16a and unknown rows tx + 16b.  Both operand tiles are
// staged K-chunk by K-chunk through a 3-deep cp.async ring in shared memory,
// stored [k/4][row][4 words] so every LDS.128 is conflict-free.
#include "common.cuh"

namespace fastid {
namespace {

constexpr int kRows = 128;           // tile edge (knowns and unknowns)
constexpr int kThreads = 256;
constexpr int kChunkWords = 16;      // u32 words per row per stage (64 B)
constexpr int kStages = 3;
constexpr int kStageBytes = 2 * kRows * kChunkWords * 4;  // 16 KB
constexpr int kScorePitch = 65;      // [128 unknown][64 known + 1] staging for top-k

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Stage chunk `kc` of the known tile (rows r0..) and unknown tile (rows q0..).
__device__ __forceinline__ void load_stage(const CompareArgs& a, uint8_t* stage, int64_t r0, int64_t q0, int kc) {
    const int64_t kbyte = (int64_t)kc * kChunkWords * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int idx = threadIdx.x + kThreads * i;  // 0..1023
        const int which = idx >> 9;                  // 0 = known, 1 = unknown
        const int rem = idx & 511;
        const int row = rem >> 2;
        const int c = rem & 3;
        const int64_t grow = (which ? q0 : r0) + row;
        const int64_t nrows = which ? a.n_queries : a.n_refs;
        const uint8_t* base = which ? a.queries : a.refs;
        const int64_t off = kbyte + c * 16;
        const bool ok = grow < nrows && off < a.stride;
        const uint8_t* src = ok ? base + grow * a.stride + off : base;
        uint8_t* dst = stage + which * (kRows * kChunkWords * 4) + (c * kRows + row) * 16;
        cp_async16(dst, src, ok ? 16 : 0);
    }
}

template <int MODE, int KP>
__global__ void __launch_bounds__(kThreads, MODE == kTopK ? 1 : 2) popc_kernel(CompareArgs a, int64_t n_ref_tiles, int n_slices) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int tx = threadIdx.x & 15;
    const int ty = threadIdx.x >> 4;
    const int n_chunks = (int)((a.stride / 4 + kChunkWords - 1) / kChunkWords);

    // Work assignment: full / threshold -> one tile per CTA; top-k -> a CTA
    // walks a contiguous slice of known tiles for one unknown group.
    int64_t q0, t_begin, t_end;
    int slice = 0;
    if (MODE == kTopK) {
        const int group = blockIdx.x / n_slices;
        slice = blockIdx.x - group * n_slices;
        q0 = (int64_t)group * kRows;
        t_begin = n_ref_tiles * slice / n_slices;
        t_end = n_ref_tiles * (slice + 1) / n_slices;
    } else {
        q0 = (int64_t)blockIdx.y * kRows;
        t_begin = blockIdx.x;
        t_end = t_begin + 1;
    }

    TopList<KP> top;
    if (MODE == kTopK) top.clear();
    uint32_t* sc = reinterpret_cast<uint32_t*>(smem + kStages * kStageBytes);

    for (int64_t t = t_begin; t < t_end; ++t) {
        const int64_t r0 = t * kRows;
        uint32_t acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0;

        // prologue: fill kStages - 1 stages
#pragma unroll
        for (int s = 0; s < kStages - 1; ++s) {
            if (s < n_chunks) load_stage(a, smem + s * kStageBytes, r0, q0, s);
            cp_async_commit();
        }
        for (int kc = 0; kc < n_chunks; ++kc) {
            cp_async_wait<kStages - 2>();
            __syncthreads();
            const int nxt = kc + kStages - 1;
            if (nxt < n_chunks) load_stage(a, smem + (nxt % kStages) * kStageBytes, r0, q0, nxt);
            cp_async_commit();
            const uint4* sk = reinterpret_cast<const uint4*>(smem + (kc % kStages) * kStageBytes);
            const uint4* sq = sk + kRows * (kChunkWords / 4);
#pragma unroll
            for (int kk = 0; kk < kChunkWords / 4; ++kk) {
                uint4 rv[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) rv[i] = sk[kk * kRows + ty + 16 * i];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint4 qv = sq[kk * kRows + tx + 16 * j];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        acc[i][j] += __popc(rv[i].x & ~qv.x) + __popc(rv[i].y & ~qv.y) +
                                     __popc(rv[i].z & ~qv.z) + __popc(rv[i].w & ~qv.w);
                    }
                }
            }
        }
        cp_async_wait<0>();
        __syncthreads();  // all stages consumed before the next tile's prologue

        if (MODE == kFull) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int64_t r = r0 + ty + 16 * i;
                if (r >= a.n_refs) continue;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int64_t q = q0 + tx + 16 * j;
                    if (q < a.n_queries) a.out[r * a.ld_out + q] = acc[i][j];
                }
            }
        } else if (MODE == kThreshold) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int64_t r = r0 + ty + 16 * i;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int64_t q = q0 + tx + 16 * j;
                    const bool hit = r < a.n_refs && q < a.n_queries && acc[i][j] <= a.threshold;
                    emit_hits(a, hit, (uint32_t)q, r, acc[i][j]);
                }
            }
        } else {
            // two halves of 64 knowns each: stage [unknown][known] then scan
            const int owner = threadIdx.x & 127;
            const int half_lane = threadIdx.x >> 7;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) sc[(tx + 16 * j) * kScorePitch + ty + 16 * i] = acc[half * 4 + i][j];
                __syncthreads();
                for (int c = 32 * half_lane; c < 32 * half_lane + 32; ++c) {
                    const int64_t r = r0 + half * 64 + c;
                    if (r < a.n_refs) top.offer(sc[owner * kScorePitch + c], (uint32_t)r, a.max_score);
                }
                __syncthreads();
            }
        }
    }

    if (MODE == kTopK) {
        const int owner = threadIdx.x & 127;
        const int half_lane = threadIdx.x >> 7;
        const int64_t q = q0 + owner;
        if (q < a.n_queries) {
            const int64_t part = (int64_t)slice * 2 + half_lane;
            const int64_t off = (part * a.n_queries + q) * KP;
            top.store(a.part_scores + off, a.part_index + off, a.ref_base);
        }
    }
}

template <int MODE, int KP>
int launch_mode(const CompareArgs& a, int n_slices, cudaStream_t stream) {
    const int64_t n_ref_tiles = ceil_div(a.n_refs, kRows);
    const int64_t n_q_tiles = ceil_div(a.n_queries, kRows);
    size_t smem = kStages * kStageBytes + (MODE == kTopK ? kRows * kScorePitch * 4 : 0);
    auto kern = popc_kernel<MODE, KP>;
    FASTID_CUDA(ensure_dynamic_smem((const void*)kern, (int)smem));
    dim3 grid;
    if (MODE == kTopK) {
        grid = dim3((unsigned)(n_q_tiles * n_slices));
    } else {
        if (n_q_tiles > 65535) FASTID_FAIL(FASTID_E_INVALID, "too many unknowns for one launch");
        grid = dim3((unsigned)n_ref_tiles, (unsigned)n_q_tiles);
    }
    kern<<<grid, kThreads, smem, stream>>>(a, n_ref_tiles, n_slices);
    FASTID_LAUNCHED("popc_kernel");
    return FASTID_OK;
}

}  // namespace

int popc_parts(int64_t n_refs, int64_t n_queries) {
    // Enough (group, slice) CTAs for ~2 waves at 2 CTAs/SM, and at most one
    // wave's worth of slices per group: each slice writes two partial lists
    // and the merge folds at most 768 lists per unknown (merge.cu).
    const int64_t groups = ceil_div(n_queries, kRows);
    const int64_t tiles = ceil_div(n_refs, kRows);
    int64_t slices = ceil_div(2 * 2 * num_sms(), groups);
    if (slices > 2 * num_sms()) slices = 2 * num_sms();
    if (slices > kMaxMergeLists / 2) slices = kMaxMergeLists / 2;
    if (slices > tiles) slices = tiles;
    if (slices < 1) slices = 1;
    return (int)slices * 2;  // two partial lists per slice (one per half-CTA)
}

int launch_popc(Mode mode, const CompareArgs& a, int* n_parts, cudaStream_t stream) {
    if (mode == kFull) return launch_mode<kFull, 1>(a, 1, stream);
    if (mode == kThreshold) return launch_mode<kThreshold, 1>(a, 1, stream);
    const int parts = popc_parts(a.n_refs, a.n_queries);
    *n_parts = parts;
    switch (a.kpad) {
        case 8: return launch_mode<kTopK, 8>(a, parts / 2, stream);
        case 16: return launch_mode<kTopK, 16>(a, parts / 2, stream);
        case 32: return launch_mode<kTopK, 32>(a, parts / 2, stream);
    }
    FASTID_FAIL(FASTID_E_INVALID, "unsupported list size %d", a.kpad);
}

}  // namespace fastid

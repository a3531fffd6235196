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

// The comparison operator on one word pair (FASTID_OP_*): LOP3 either way.
template <int OP>
__device__ __forceinline__ uint32_t pop_op(uint32_t r, uint32_t q) {
    if constexpr (OP == FASTID_OP_AND) return __popc(r & q);
    else if constexpr (OP == FASTID_OP_XOR) return __popc(r ^ q);
    else return __popc(r & ~q);
}
template <int OP>
__device__ __forceinline__ uint32_t pop_op4(const uint4& r, const uint4& q) {
    return pop_op<OP>(r.x, q.x) + pop_op<OP>(r.y, q.y) + pop_op<OP>(r.z, q.z) + pop_op<OP>(r.w, q.w);
}

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

template <int MODE, int KP, int OP>
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
                        acc[i][j] += pop_op4<OP>(rv[i], qv);
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

// ---- few unknowns: a streaming scan (the single-profile search) ---------------
//
// With a handful of unknowns the 128 x 128 tile above wastes almost all of its
// POPC work on empty unknown rows (one unknown vs 20M knowns: 28 ms), and the
// tensor kernels stream the whole 4-bit image (1.5 ms).  The scan reads each
// packed known row once (2.56 GB for 20M x 1024 loci) against up to
// kScanMaxQ complemented unknowns held in shared memory.  A warp scores 32
// rows per step, one per lane; the per-unknown state is sized to the batch
// (QN) so a single profile runs at high occupancy with many rows in flight,
// and the rows arrive by coalesced loads (four whole rows per instruction)
// through a small per-warp staging tile.  (Eight lanes per row with
// shuffle-summed partial counts, double-buffered cp.async staging and a
// register prefetch of the next step all measured slower for one unknown
// against 20M x 1024 loci: 2.7, 1.8 and 2.3 ms.)  Per unknown the
// warp keeps a sorted top-KP list spread over its lanes (lane l holds entry
// l), admits a row that orders before the list's last entry and whose score is
// <= the shared bound (a.bound[j]: the smallest KP-th best any warp has
// published), and inserts with one shuffle round.  At the end the CTA's warps'
// lists are merged into one partial list per CTA, which the merge kernel folds
// like any other partials.
// Warp-wide (score, index) sort helpers of the scan's list update: one pair per lane.
__device__ __forceinline__ void cmp_exchange(uint32_t& s, uint32_t& x, int d, bool keep_min) {
    const uint32_t os = __shfl_xor_sync(0xFFFFFFFFu, s, d);
    const uint32_t ox = __shfl_xor_sync(0xFFFFFFFFu, x, d);
    if (keep_min ? before(os, ox, s, x) : before(s, x, os, ox)) {
        s = os;
        x = ox;
    }
}
// ascending bitonic sort of the warp's 32 pairs
__device__ __forceinline__ void warp_sort(uint32_t& s, uint32_t& x, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int d = k >> 1; d > 0; d >>= 1) cmp_exchange(s, x, d, ((lane & d) == 0) == ((lane & k) == 0));
}
// ascending sort of a bitonic sequence
__device__ __forceinline__ void warp_bitonic_merge(uint32_t& s, uint32_t& x, int lane) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) cmp_exchange(s, x, d, (lane & d) == 0);
}
// A step with at least this many admissible rows merges them into the list at
// once (sort + bitonic merge, ~21 shuffle rounds) instead of one insertion each
// (~8 dependent shuffles per row): the first steps of every warp, whose lists
// are still empty, admit all 32 rows.  Up to two unknowns per kernel (the
// popcount-bound 4+-unknown instances ran 3-13% slower with the extra code).
constexpr int kScanBulkMin = 4;

constexpr int kScanMaxQ = 16;
constexpr int kScanWarps = 8;
constexpr int kScanPiece = 8;  // uint4 per row per staging round (128 B)
constexpr int kScanTile16 = 32 * (kScanPiece + 1);  // one warp's staging tile (uint4), padded rows

template <int MODE, int KP, int QN, bool XOR>
__global__ void __launch_bounds__(32 * kScanWarps, QN <= 2 ? 4 : QN <= 4 ? 3 : 2) popc_scan_kernel(CompareArgs a) {
    extern __shared__ __align__(16) uint4 sq[];  // [n_queries][n16] unknown rows (complemented for AND-NOT)
    const int n16 = (int)(a.stride / 16);
    const int nq = (int)a.n_queries;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint4* tile = sq + nq * n16 + warp * kScanTile16;  // this warp's staging tile
    for (int i = threadIdx.x; i < nq * n16; i += blockDim.x) {
        const uint4 v = reinterpret_cast<const uint4*>(a.queries)[(int64_t)(i / n16) * n16 + i % n16];
        sq[i] = a.op == FASTID_OP_ANDNOT ? make_uint4(~v.x, ~v.y, ~v.z, ~v.w) : v;
    }
    // zero padding in the known rows makes the complemented padding of the
    // unknowns harmless (r & ~q = 0 past L)
    __syncthreads();
    uint32_t ls[QN], lx[QN], ks[QN], kx[QN], gb[QN];
#pragma unroll
    for (int j = 0; j < QN; ++j) {
        ls[j] = kEmptyScore;
        lx[j] = kEmptyLocal;
        ks[j] = kEmptyScore;  // the list's KP-th entry (every lane holds a copy)
        kx[j] = kEmptyLocal;
        gb[j] = a.max_score;  // admit score <= min(shared bound, cap)
    }
    const int64_t warps = (int64_t)gridDim.x * kScanWarps;
    const int64_t n_steps = (a.n_refs + 31) / 32;
    int64_t step_no = 0;
    for (int64_t st = (int64_t)blockIdx.x * kScanWarps + warp; st < n_steps; st += warps, ++step_no) {
        if ((step_no & 7) == 0) {
#pragma unroll
            for (int j = 0; j < QN; ++j)
                if (j < nq) {
                    const uint32_t g = __ldcg(a.bound + j);
                    if (g < gb[j]) gb[j] = g;
                }
        }
        const int64_t r = st * 32 + lane;
        const bool valid = r < a.n_refs;
        uint32_t acc[QN];
#pragma unroll
        for (int j = 0; j < QN; ++j) acc[j] = 0;
        // the step's 32 rows, 128 B per row per round: coalesced loads (4 whole rows,
        // 512 contiguous bytes, per instruction) through this warp's staging tile,
        // then each lane scores its own row from shared memory
        const uint8_t* rows0 = a.refs + st * 32 * a.stride;
        for (int c = 0; c < n16; c += kScanPiece) {
#pragma unroll
            for (int i = 0; i < kScanPiece; ++i) {
                const int p = lane + 32 * i, prow = p / kScanPiece, pcol = c + p % kScanPiece;
                const bool ok = st * 32 + prow < a.n_refs && pcol < n16;
                cp_async16(tile + prow * (kScanPiece + 1) + p % kScanPiece,
                           ok ? rows0 + prow * a.stride + (int64_t)pcol * 16 : a.refs, ok ? 16 : 0);
            }
            cp_async_commit();
            cp_async_wait<0>();
            __syncwarp();
#pragma unroll
            for (int w = 0; w < kScanPiece; ++w) {
                if (c + w < n16) {
                    const uint4 rv = tile[lane * (kScanPiece + 1) + w];
#pragma unroll
                    for (int j = 0; j < QN; ++j)
                        if (j < nq) {
                            const uint4 qv = sq[j * n16 + c + w];
                            acc[j] += XOR ? pop_op4<FASTID_OP_XOR>(rv, qv) : pop_op4<FASTID_OP_AND>(rv, qv);
                        }
                }
            }
            __syncwarp();
        }
        const uint32_t rl = (uint32_t)r;
        if constexpr (MODE == kThreshold) {
            // every (unknown, row) within the threshold, appended with warp-aggregated slots
#pragma unroll
            for (int j = 0; j < QN; ++j)
                if (j < nq) emit_hits(a, valid && acc[j] <= a.threshold, (uint32_t)j, r, acc[j]);
        } else {
#pragma unroll
        for (int j = 0; j < QN; ++j) {
            if (j >= nq) break;
            const bool cand = valid && acc[j] <= gb[j] && before(acc[j], rl, ks[j], kx[j]);
            uint32_t m = __ballot_sync(0xFFFFFFFFu, cand);
            if (QN <= 2 && __popc(m) >= kScanBulkMin) {
                // the admissible rows, sorted; min against the reversed list gives the 32
                // smallest of both as a bitonic sequence (lanes >= KP hold empty entries)
                uint32_t bs = cand ? acc[j] : kEmptyScore, bx = cand ? rl : kEmptyLocal;
                warp_sort(bs, bx, lane);
                const uint32_t rs = __shfl_sync(0xFFFFFFFFu, bs, 31 - lane);
                const uint32_t rx = __shfl_sync(0xFFFFFFFFu, bx, 31 - lane);
                if (before(rs, rx, ls[j], lx[j])) {
                    ls[j] = rs;
                    lx[j] = rx;
                }
                warp_bitonic_merge(ls[j], lx[j], lane);
                if (lane >= KP) {
                    ls[j] = kEmptyScore;
                    lx[j] = kEmptyLocal;
                }
                ks[j] = __shfl_sync(0xFFFFFFFFu, ls[j], KP - 1);
                kx[j] = __shfl_sync(0xFFFFFFFFu, lx[j], KP - 1);
                if (ks[j] < gb[j]) {
                    gb[j] = ks[j];
                    if (lane == 0) atomicMin(a.bound + j, ks[j]);
                }
                m = 0;
            }
            while (m) {
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const uint32_t v = __shfl_sync(0xFFFFFFFFu, acc[j], src);
                const uint32_t x = __shfl_sync(0xFFFFFFFFu, rl, src);
                if (!before(v, x, ks[j], kx[j])) continue;  // an earlier insertion raised the bar
                // entries before (v, x) stay; the rest shift one lane down
                const int pos = __popc(__ballot_sync(0xFFFFFFFFu, lane < KP && before(ls[j], lx[j], v, x)));
                const uint32_t us = __shfl_up_sync(0xFFFFFFFFu, ls[j], 1);
                const uint32_t ux = __shfl_up_sync(0xFFFFFFFFu, lx[j], 1);
                if (lane == pos) {
                    ls[j] = v;
                    lx[j] = x;
                } else if (lane > pos && lane < KP) {
                    ls[j] = us;
                    lx[j] = ux;
                }
                ks[j] = __shfl_sync(0xFFFFFFFFu, ls[j], KP - 1);
                kx[j] = __shfl_sync(0xFFFFFFFFu, lx[j], KP - 1);
                // publish only a list end that beats the bound this warp knows: an
                // atomicMin at or above it changes nothing, and every warp hitting one
                // address serialises in its L2 slice (one unknown, 2M rows: 199 us)
                if (ks[j] < gb[j]) {
                    gb[j] = ks[j];
                    if (lane == 0) atomicMin(a.bound + j, ks[j]);
                }
            }
        }
        }  // top-k
    }
    if constexpr (MODE == kThreshold) return;
    // the CTA's warps' lists -> one partial list per unknown (a k-way merge by one warp)
    __syncthreads();  // every warp is done with the unknowns and staging: the space is reused below
    uint32_t* ms = reinterpret_cast<uint32_t*>(sq);  // [warps][kScanMaxQ][KP] scores, then indices
    uint32_t* mx = ms + kScanWarps * kScanMaxQ * KP;
#pragma unroll
    for (int j = 0; j < QN; ++j)
        if (j < nq && lane < KP) {
            ms[(warp * kScanMaxQ + j) * KP + lane] = ls[j];
            mx[(warp * kScanMaxQ + j) * KP + lane] = lx[j];
        }
    __syncthreads();
    for (int j = warp; j < nq; j += kScanWarps) {
        int head = 0;  // lane w < kScanWarps walks warp w's list
        const int64_t off = ((int64_t)blockIdx.x * a.n_queries + j) * KP;
        for (int o = 0; o < KP; ++o) {
            uint32_t hs = kEmptyScore, hx = kEmptyLocal;
            if (lane < kScanWarps && head < KP) {
                hs = ms[(lane * kScanMaxQ + j) * KP + head];
                hx = mx[(lane * kScanMaxQ + j) * KP + head];
            }
            uint32_t bs = hs, bx = hx;
            int bl = lane;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                const uint32_t os = __shfl_xor_sync(0xFFFFFFFFu, bs, d);
                const uint32_t ox = __shfl_xor_sync(0xFFFFFFFFu, bx, d);
                const int ol = __shfl_xor_sync(0xFFFFFFFFu, bl, d);
                if (before(os, ox, bs, bx) || (os == bs && ox == bx && ol < bl)) {
                    bs = os;
                    bx = ox;
                    bl = ol;
                }
            }
            if (lane == bl && bs != kEmptyScore) ++head;
            if (lane == 0) {
                a.part_scores[off + o] = bs;
                a.part_index[off + o] = bs == kEmptyScore ? -1 : a.ref_base + (int64_t)bx;
            }
        }
    }
}

inline size_t scan_smem_bytes(const CompareArgs& a, int kpad) {
    const size_t lists = 2 * (size_t)kScanWarps * kScanMaxQ * kpad * 4;
    const size_t rows = (size_t)a.n_queries * (a.stride / 16) * 16 + (size_t)kScanWarps * kScanTile16 * 16;
    return rows > lists ? rows : lists;
}

template <int MODE, int KP, int QN>
int launch_scan_q(const CompareArgs& a, int n_ctas, cudaStream_t stream) {
    const size_t smem = scan_smem_bytes(a, KP);
    auto kern = a.op == FASTID_OP_XOR ? popc_scan_kernel<MODE, KP, QN, true> : popc_scan_kernel<MODE, KP, QN, false>;
    FASTID_CUDA(ensure_dynamic_smem((const void*)kern, (int)smem));
    kern<<<(unsigned)n_ctas, 32 * kScanWarps, smem, stream>>>(a);
    FASTID_LAUNCHED("popc_scan_kernel");
    return FASTID_OK;
}

// per-unknown state lives in registers: instantiate for the batch size so a
// single profile keeps the occupancy of a small kernel
template <int MODE, int KP>
int launch_scan(const CompareArgs& a, int n_ctas, cudaStream_t stream) {
    if (a.n_queries <= 1) return launch_scan_q<MODE, KP, 1>(a, n_ctas, stream);
    if (a.n_queries <= 2) return launch_scan_q<MODE, KP, 2>(a, n_ctas, stream);
    if (a.n_queries <= 4) return launch_scan_q<MODE, KP, 4>(a, n_ctas, stream);
    if (a.n_queries <= 8) return launch_scan_q<MODE, KP, 8>(a, n_ctas, stream);
    return launch_scan_q<MODE, KP, kScanMaxQ>(a, n_ctas, stream);
}

template <int MODE, int KP>
int launch_mode(const CompareArgs& a, int n_slices, cudaStream_t stream) {
    const int64_t n_ref_tiles = ceil_div(a.n_refs, kRows);
    const int64_t n_q_tiles = ceil_div(a.n_queries, kRows);
    size_t smem = kStages * kStageBytes + (MODE == kTopK ? kRows * kScorePitch * 4 : 0);
    auto kern = a.op == FASTID_OP_AND   ? popc_kernel<MODE, KP, FASTID_OP_AND>
                : a.op == FASTID_OP_XOR ? popc_kernel<MODE, KP, FASTID_OP_XOR>
                                        : popc_kernel<MODE, KP, FASTID_OP_ANDNOT>;
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

// One warp per row: the row's popcount (XOR on the tensor kernels: the unknowns', and the knowns' for i8).
__global__ void row_popcount_kernel(const uint8_t* __restrict__ rows, int64_t n, int64_t n_out, int64_t stride,
                                    bool as_float, uint32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int n16 = (int)(stride / 16);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < n_out; r += warps) {
        if (r >= n) {  // padding entries: defined zeros
            if (lane == 0) out[r] = 0;
            continue;
        }
        const uint4* row = reinterpret_cast<const uint4*>(rows + r * stride);
        uint32_t c = 0;
        for (int i = lane; i < n16; i += 32) {
            const uint4 v = __ldg(row + i);
            c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
        }
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) out[r] = as_float ? __float_as_uint((float)c) : c;
    }
}

}  // namespace

int launch_row_popcount(const uint8_t* rows, int64_t n, int64_t n_out, int64_t stride, bool as_float, uint32_t* out,
                        cudaStream_t stream) {
    if (n_out <= 0) return FASTID_OK;
    const int64_t blocks = std::min<int64_t>(ceil_div(n_out, 8), (int64_t)num_sms() * 8);
    row_popcount_kernel<<<(unsigned)blocks, 256, 0, stream>>>(rows, n, n_out, stride, as_float, out);
    FASTID_LAUNCHED("row_popcount_kernel");
    return FASTID_OK;
}

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
    if (mode == kThreshold) {
        if (a.n_queries <= kScanMaxQ && scan_smem_bytes(a, 8) <= 200 * 1024)
            return launch_scan<kThreshold, 8>(a, 4 * num_sms(), stream);
        return launch_mode<kThreshold, 1>(a, 1, stream);
    }
    int parts = popc_parts(a.n_refs, a.n_queries);
    // few unknowns (and their rows, plus the merge lists, in shared memory): the scan
    if (a.n_queries <= kScanMaxQ && scan_smem_bytes(a, a.kpad) <= 200 * 1024) {
        // one unknown: 3 CTAs per SM (fewer per-warp lists, fewer insertions) measured
        // 0.535 vs 0.592 ms at 4 (20M x 1024 loci, tools/scan_timing.py); from two
        // unknowns on, the popcount work wants the 4th CTA (4 unknowns: 1.20 vs 1.38 ms)
        if (a.n_queries == 1) parts = std::min(parts, 3 * num_sms());
        // three or four unknowns: 3 resident CTAs per SM (80 registers), one wave of them
        // (4 unknowns: 1.12 ms vs 1.20 at 2 per SM in two waves)
        if (a.n_queries > 2 && a.n_queries <= 4) parts = std::min(parts, 3 * num_sms());
        // FASTID_SCAN_CTAS: grid size of the scan (scheduling only; <= kMaxMergeLists)
        if (const char* e = getenv("FASTID_SCAN_CTAS")) {
            const int v = atoi(e);
            // (never above the lists the workspace holds: fastid_topk_workspace)
            if (v > 0 && v <= kMaxMergeLists && v <= std::max(parts, tensor_parts(a.n_refs, a.n_queries, FASTID_TENSOR_F4)))
                parts = v;
        }
        *n_parts = parts;
        switch (a.kpad) {
            case 8: return launch_scan<kTopK, 8>(a, parts, stream);
            case 16: return launch_scan<kTopK, 16>(a, parts, stream);
            case 32: return launch_scan<kTopK, 32>(a, parts, stream);
        }
    }
    *n_parts = parts;
    switch (a.kpad) {
        case 8: return launch_mode<kTopK, 8>(a, parts / 2, stream);
        case 16: return launch_mode<kTopK, 16>(a, parts / 2, stream);
        case 32: return launch_mode<kTopK, 32>(a, parts / 2, stream);
    }
    FASTID_FAIL(FASTID_E_INVALID, "unsupported list size %d", a.kpad);
}

}  // namespace fastid

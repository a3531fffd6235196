// Formulation B: the overloaded GEMM on the 5th-generation tensor cores.
//
//   score(i, j) = popcount(R_i AND NOT Q_j) = sum_k R_i[k] * (1 - Q_j[k])
//
// i.e. an ordinary dot product of 0/1 vectors once the unknown is
// complemented (north star: "R.(1-M) = rowsum(R) - R.M").  The product is
// exact on tcgen05: kind::i8 accumulates in s32; kind::mxf4 multiplies e2m1
// values in {0, 1} with unit (ue8m0 = 127) block scales and accumulates
// integers <= L in fp32.
//
// One CTA per SM (persistent), warp-specialised:
//   warp 0      TMA producer: 2-D tensor copies of packed known rows
//               (BN rows x 32 B = 256 loci per stage) into a deep ring.
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma into a
//               double-buffered TMEM accumulator (BN fp32/s32 columns each).
//   warps 2-5   converters: unpack the packed bits into the UMMA K-major
//               operand layout (e2m1 nibbles or int8 bytes); at start-up they
//               also build the resident A operand = complemented unknown tile.
//   warps 6-9   epilogue: tcgen05.ld the accumulator (one TMEM lane = one
//               unknown per thread) and apply the fused epilogue: full u32
//               store, per-unknown top-k, or threshold hits.
// The unknown tile (128 unknowns) stays resident in shared memory for the
// CTA's whole slice of known tiles; known tiles stream through TMA.  CTAs of
// the same slice index walk the same known tiles at the same time, so each
// known tile is read from HBM once and served to the other unknown groups
// from L2.  DESIGN.md has the roofline and byte accounting.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tensor_ptx.cuh"

namespace fastid {
namespace {

constexpr int kM = 128;             // unknowns per CTA (MMA M, TMEM lanes)
constexpr int kStageBytesPacked = 32;  // packed bytes per known row per stage (256 loci)
constexpr int kWordsPerStage = kStageBytesPacked / 4;
constexpr int kMaxPackedStages = 12;
constexpr int kConvThreads = 128;
constexpr int kEpiWarps = 8;       // two per TMEM lane quadrant, splitting the columns
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreads = 64 + kConvThreads + kEpiThreads;  // producer, MMA, converters, epilogue
constexpr int kChunk = 16;         // accumulator columns per tcgen05.ld
constexpr int kSmemLimit = 227 * 1024;

template <int F>
struct Fmt;
template <>
struct Fmt<FASTID_TENSOR_I8> {
    static constexpr int BN = 128;          // knowns per tile (MMA N)
    static constexpr int kCoresPerWord = 2; // 16-B core columns produced per packed u32
    static constexpr int kMmaPerStage = 8;  // K = 32 B of operand per MMA
    static constexpr int kUnpackedStages = 2;
    static constexpr int kTmemCols = 256;   // 2 x BN accumulator columns
};
template <>
struct Fmt<FASTID_TENSOR_F4> {
    static constexpr int BN = 224;
    static constexpr int kCoresPerWord = 1;
    static constexpr int kMmaPerStage = 4;
    static constexpr int kUnpackedStages = 2;
    static constexpr int kTmemCols = 512;   // 2 x 224 accumulators + 64 scale-factor columns
};

constexpr uint32_t kSfaCol = 448;  // mxf4: unit scale factors for A (32 columns)
constexpr uint32_t kSfbCol = 480;  // mxf4: unit scale factors for B (32 columns)
constexpr uint32_t kUnitScales = 0x7F7F7F7Fu;  // ue8m0 127 = 2^0

// e2m1 nibbles (1.0 = 0x2): nibble n of word j <- bit 4n + j.
__device__ __forceinline__ uint4 unpack_f4(uint32_t w) {
    return make_uint4((w << 1) & 0x22222222u, w & 0x22222222u, (w >> 1) & 0x22222222u, (w >> 2) & 0x22222222u);
}
// int8 bytes (1 = 0x01): byte b of word j <- bit 8b + j; two 16-B core columns.
__device__ __forceinline__ void unpack_i8(uint32_t w, uint4& lo, uint4& hi) {
    lo = make_uint4(w & 0x01010101u, (w >> 1) & 0x01010101u, (w >> 2) & 0x01010101u, (w >> 3) & 0x01010101u);
    hi = make_uint4((w >> 4) & 0x01010101u, (w >> 5) & 0x01010101u, (w >> 6) & 0x01010101u,
                    (w >> 7) & 0x01010101u);
}

// Accumulator encodings.  mxf4 accumulates exact integers in fp32, whose bit
// patterns order like the integers (non-negative floats); i8 accumulates s32.
template <int F>
__device__ __forceinline__ uint32_t score_bits(uint32_t s) {
    return F == FASTID_TENSOR_F4 ? __float_as_uint((float)s) : s;
}
template <int F>
__device__ __forceinline__ uint32_t decode_exact(uint32_t v) {
    return F == FASTID_TENSOR_F4 ? (uint32_t)__uint_as_float(v) : v;
}
// float -> u32 for integers < 2^23 without F2I: add 2^23, read the mantissa.
template <int F>
__device__ __forceinline__ uint32_t decode_fast(uint32_t v) {
    return F == FASTID_TENSOR_F4 ? __float_as_uint(__uint_as_float(v) + 8388608.0f) - 0x4B000000u : v;
}

// v[c] for a run-time c without local memory: a 4-level select tree.
__device__ __forceinline__ uint32_t pick16(const uint32_t (&v)[16], int c) {
    uint32_t a[8], b[4], d[2];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = (c & 8) ? v[i + 8] : v[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = (c & 4) ? a[i + 4] : a[i];
#pragma unroll
    for (int i = 0; i < 2; ++i) d[i] = (c & 2) ? b[i + 2] : b[i];
    return (c & 1) ? d[1] : d[0];
}

// Core-matrix offset of (row, core column) in a K-major no-swizzle operand of `rows` rows.
__device__ __forceinline__ uint32_t core_off(int row, int col, int rows) {
    return (uint32_t)col * (uint32_t)(rows * 16) + (uint32_t)(row >> 3) * 128u + (uint32_t)(row & 7) * 16u;
}

template <int F>
struct Layout {
    static constexpr int BN = Fmt<F>::BN;
    static constexpr int kUnpackedStageBytes = BN * 16 * kWordsPerStage * Fmt<F>::kCoresPerWord;
    static constexpr int kPackedStageBytes = BN * kStageBytesPacked;
    int n_kst;    // stages per tile (K padded to 256 loci)
    int a_bytes;  // resident complemented unknown tile
    int sp;       // packed ring depth that fits
    int off_u, off_p, off_bar, total;
    __host__ __device__ explicit Layout(int64_t stride) {
        n_kst = (int)((stride + kStageBytesPacked - 1) / kStageBytesPacked);
        a_bytes = n_kst * kWordsPerStage * Fmt<F>::kCoresPerWord * kM * 16;
        off_u = a_bytes;
        off_p = off_u + Fmt<F>::kUnpackedStages * kUnpackedStageBytes;
        const int bar_bytes = 8 * (2 * kMaxPackedStages + 2 * Fmt<F>::kUnpackedStages + 5) + 16;
        int room = (kSmemLimit - off_p - bar_bytes) / kPackedStageBytes;
        sp = room > kMaxPackedStages ? kMaxPackedStages : room;
        off_bar = off_p + (sp > 0 ? sp : 0) * kPackedStageBytes;
        total = off_bar + bar_bytes;
    }
};

template <int F, int MODE, int KP>
__global__ void __launch_bounds__(kThreads, 1)
    tensor_kernel(const __grid_constant__ CUtensorMap tmap, CompareArgs a, int64_t n_tiles, int n_slices) {
    constexpr int BN = Fmt<F>::BN;
    constexpr int SU = Fmt<F>::kUnpackedStages;
    constexpr int CPW = Fmt<F>::kCoresPerWord;
    constexpr int UB = Layout<F>::kUnpackedStageBytes;
    constexpr int PB = Layout<F>::kPackedStageBytes;
    extern __shared__ __align__(1024) uint8_t smem[];
    const Layout<F> lay(a.stride);
    const int SP = lay.sp;
    const int n_kst = lay.n_kst;
    uint8_t* sA = smem;
    uint8_t* sU = smem + lay.off_u;
    uint8_t* sP = smem + lay.off_p;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.off_bar);
    uint64_t* p_full = bars;
    uint64_t* p_empty = p_full + kMaxPackedStages;
    uint64_t* u_full = p_empty + kMaxPackedStages;
    uint64_t* u_empty = u_full + SU;
    uint64_t* t_full = u_empty + SU;
    uint64_t* t_empty = t_full + 2;
    uint64_t* a_full = t_empty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int group = blockIdx.x / n_slices;
    const int slice = blockIdx.x - group * n_slices;
    const int64_t q0 = (int64_t)group * kM;
    const int64_t t_begin = n_tiles * slice / n_slices;
    const int64_t t_end = n_tiles * (slice + 1) / n_slices;

    if (threadIdx.x == 0) {
        for (int i = 0; i < SP; ++i) {
            ptx::mbar_init(&p_full[i], 1);
            ptx::mbar_init(&p_empty[i], kConvThreads);
        }
        for (int i = 0; i < SU; ++i) {
            ptx::mbar_init(&u_full[i], kConvThreads);
            ptx::mbar_init(&u_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&t_full[i], 1);
            ptx::mbar_init(&t_empty[i], kEpiThreads);
        }
        ptx::mbar_init(a_full, kConvThreads);
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tmap);
    if (warp == 1) ptx::tmem_alloc(tmem_slot, Fmt<F>::kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (F == FASTID_TENSOR_F4 && warp >= 6) {
        // unit block scales (ue8m0 127) for every MMA: whole SF region, all lanes
        const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        ptx::tmem_fill32(lb + kSfaCol, kUnitScales);
        ptx::tmem_fill32(lb + kSfbCol, kUnitScales);
        ptx::tmem_wait_st();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            uint32_t it = 0;
            for (int64_t t = t_begin; t < t_end; ++t) {
                for (int ks = 0; ks < n_kst; ++ks, ++it) {
                    const int s = (int)(it % (uint32_t)SP);
                    ptx::mbar_wait(&p_empty[s], ((it / SP) & 1) ^ 1);
                    ptx::mbar_expect_tx(&p_full[s], PB);
                    ptx::tma_load_2d(sP + s * PB, &tmap, &p_full[s], ks * kStageBytesPacked, (int)(t * BN));
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (one thread) ----------------
        if (lane == 0) {
            constexpr uint32_t idesc = F == FASTID_TENSOR_F4 ? ptx::idesc_mxf4(kM, BN) : ptx::idesc_i8(kM, BN);
            const uint32_t a_base = ptx::smem_u32(sA);
            const uint32_t u_base = ptx::smem_u32(sU);
            ptx::mbar_wait(a_full, 0);
            ptx::tc_fence_after();
            uint32_t it = 0;
            int local = 0;
            for (int64_t t = t_begin; t < t_end; ++t, ++local) {
                const int acc = local & 1;
                ptx::mbar_wait(&t_empty[acc], ((local >> 1) & 1) ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * BN);
                for (int ks = 0; ks < n_kst; ++ks, ++it) {
                    const int s = (int)(it % SU);
                    ptx::mbar_wait(&u_full[s], (it / SU) & 1);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < Fmt<F>::kMmaPerStage; ++kk) {
                        const uint32_t acol = (uint32_t)(ks * kWordsPerStage * CPW + 2 * kk);
                        const uint64_t ad = ptx::smem_desc(a_base + acol * (kM * 16), kM * 16, 128);
                        const uint64_t bd =
                            ptx::smem_desc(u_base + s * UB + (uint32_t)(2 * kk) * (BN * 16), BN * 16, 128);
                        const uint32_t accum = (ks | kk) ? 1u : 0u;
                        if (F == FASTID_TENSOR_F4)
                            ptx::mma_mxf4(d, ad, bd, idesc, tmem + kSfaCol, tmem + kSfbCol, accum);
                        else
                            ptx::mma_i8(d, ad, bd, idesc, accum);
                    }
                    ptx::tc_commit(&u_empty[s]);  // stage s reusable once these MMAs retire
                }
                ptx::tc_commit(&t_full[acc]);  // accumulator complete -> epilogue
            }
        }
    } else if (warp < 6) {
        // ---------------- converters ----------------
        const int ct = threadIdx.x - 64;  // 0..127
        {
            // Resident A = complemented unknown row ct; zero past the row.
            const int64_t q = q0 + ct;
            const bool real = q < a.n_queries;
            const int row_words = (int)(a.stride / 4);
            const uint32_t* src = reinterpret_cast<const uint32_t*>(a.queries + (real ? q : 0) * a.stride);
            for (int w4 = 0; w4 < n_kst * kWordsPerStage; w4 += 4) {
                uint4 v = make_uint4(0, 0, 0, 0);
                if (real && w4 < row_words) {
                    v = *reinterpret_cast<const uint4*>(src + w4);
                    v = make_uint4(~v.x, ~v.y, ~v.z, ~v.w);
                }
                const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int col = (w4 + i) * CPW;
                    if (F == FASTID_TENSOR_F4) {
                        *reinterpret_cast<uint4*>(sA + core_off(ct, col, kM)) = unpack_f4(wv[i]);
                    } else {
                        uint4 lo, hi;
                        unpack_i8(wv[i], lo, hi);
                        *reinterpret_cast<uint4*>(sA + core_off(ct, col, kM)) = lo;
                        *reinterpret_cast<uint4*>(sA + core_off(ct, col + 1, kM)) = hi;
                    }
                }
            }
            ptx::fence_proxy_async_smem();
            ptx::mbar_arrive(a_full);
        }
        uint32_t it = 0;
        for (int64_t t = t_begin; t < t_end; ++t) {
            for (int ks = 0; ks < n_kst; ++ks, ++it) {
                const int sp = (int)(it % (uint32_t)SP);
                const int su = (int)(it % SU);
                ptx::mbar_wait(&p_full[sp], (it / SP) & 1);
                const uint8_t* P = sP + sp * PB;
                const bool second = ct + 128 < BN;
                uint4 v[2][2];
                v[0][0] = *reinterpret_cast<const uint4*>(P + ct * kStageBytesPacked);
                v[0][1] = *reinterpret_cast<const uint4*>(P + ct * kStageBytesPacked + 16);
                if (second) {
                    v[1][0] = *reinterpret_cast<const uint4*>(P + (ct + 128) * kStageBytesPacked);
                    v[1][1] = *reinterpret_cast<const uint4*>(P + (ct + 128) * kStageBytesPacked + 16);
                }
                ptx::mbar_wait(&u_empty[su], ((it / SU) & 1) ^ 1);
                uint8_t* U = sU + su * UB;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (h == 1 && !second) break;
                    const int row = ct + 128 * h;
                    const uint32_t wv[8] = {v[h][0].x, v[h][0].y, v[h][0].z, v[h][0].w,
                                            v[h][1].x, v[h][1].y, v[h][1].z, v[h][1].w};
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if (F == FASTID_TENSOR_F4) {
                            *reinterpret_cast<uint4*>(U + core_off(row, i, BN)) = unpack_f4(wv[i]);
                        } else {
                            uint4 lo, hi;
                            unpack_i8(wv[i], lo, hi);
                            *reinterpret_cast<uint4*>(U + core_off(row, 2 * i, BN)) = lo;
                            *reinterpret_cast<uint4*>(U + core_off(row, 2 * i + 1, BN)) = hi;
                        }
                    }
                }
                // every lane arrives itself: its loads of P[sp] have been consumed
                // by the stores above, and its own fence orders those stores
                // before the tensor core reads U[su]
                ptx::mbar_arrive(&p_empty[sp]);
                ptx::fence_proxy_async_smem();
                ptx::mbar_arrive(&u_full[su]);
            }
        }
    } else {
        // ---------------- epilogue: one unknown per thread ----------------
        // Warp w reads TMEM lanes 32*(w%4).. (its quadrant) and one half of the
        // accumulator columns; scores stay as raw accumulator bits (fp32 of an
        // exact integer is order-preserving as u32), so the hot loop is compares
        // only and the rare candidates take a warp-uniform slow path.
        const int ew = warp - 6;
        const int quad = warp & 3;
        const int half = ew >> 2;
        constexpr int kHalfCols = BN / 2;  // 112 (mxf4) or 64 (i8): a multiple of kChunk
        const int m = quad * 32 + lane;
        const int64_t q = q0 + m;
        const bool q_ok = q < a.n_queries;
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
        TopList<KP> top;
        if (MODE == kTopK) top.clear();
        const uint64_t cap = (uint64_t)a.max_score + 1;  // admit v <= max_score
        uint32_t thr_bits = 0;
        if (MODE == kTopK) thr_bits = score_bits<F>(cap < kEmptyScore ? (uint32_t)cap : kEmptyScore);
        const uint32_t hit_bits = MODE == kThreshold ? score_bits<F>(a.threshold) : 0u;
        int local = 0;
        for (int64_t t = t_begin; t < t_end; ++t, ++local) {
            const int acc = local & 1;
            ptx::mbar_wait(&t_full[acc], (local >> 1) & 1);
            ptx::tc_fence_after();
            const int64_t r0 = t * BN + half * kHalfCols;
            const int64_t rows_left = a.n_refs - r0;
#pragma unroll 1
            for (int ch = 0; ch < kHalfCols / kChunk; ++ch) {
                uint32_t v[kChunk];
                ptx::tmem_ld16(lane_base + (uint32_t)(acc * BN + half * kHalfCols + ch * kChunk), v);
                ptx::tmem_wait_ld();
                if (ch + 1 == kHalfCols / kChunk) {
                    // this warp's half of the accumulator is in registers: release it
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&t_empty[acc]);
                }
                const int64_t rc = r0 + ch * kChunk;
                const uint32_t valid = !q_ok || rows_left <= ch * kChunk ? 0u
                                       : (rows_left >= (ch + 1) * kChunk ? 0xFFFFu
                                                                         : (1u << (rows_left - ch * kChunk)) - 1u);
                if (MODE == kFull) {
#pragma unroll
                    for (int c = 0; c < kChunk; ++c)
                        if ((valid >> c) & 1u) a.out[(rc + c) * a.ld_out + q] = decode_fast<F>(v[c]);
                } else if (MODE == kTopK) {
                    uint32_t cand = 0;
#pragma unroll
                    for (int c = 0; c < kChunk; ++c) cand |= (v[c] < thr_bits ? 1u : 0u) << c;
                    cand &= valid;
                    // rare: one insertion per loop trip, value picked by a select tree
                    while (cand) {
                        const int c = __ffs(cand) - 1;
                        cand &= cand - 1;
                        const uint32_t vc = pick16(v, c);
                        if (vc < thr_bits) {
                            top.insert(decode_exact<F>(vc), (uint32_t)(rc + c));
                            const uint64_t w = top.s[KP - 1] < cap ? top.s[KP - 1] : cap;
                            thr_bits = score_bits<F>(w < kEmptyScore ? (uint32_t)w : kEmptyScore);
                        }
                    }
                } else {
                    uint32_t hit = 0;
#pragma unroll
                    for (int c = 0; c < kChunk; ++c) hit |= (v[c] <= hit_bits ? 1u : 0u) << c;
                    hit &= valid;
                    if (__any_sync(0xffffffffu, hit != 0)) {
                        uint32_t all = __reduce_or_sync(0xffffffffu, hit);
                        while (all) {  // warp-uniform walk over columns with a hit in any lane
                            const int c = __ffs(all) - 1;
                            all &= all - 1;
                            emit_hits(a, (hit >> c) & 1u, (uint32_t)q, rc + c, decode_exact<F>(pick16(v, c)));
                        }
                    }
                }
            }
        }
        if (MODE == kTopK && q_ok) {
            const int64_t off = (((int64_t)slice * 2 + half) * a.n_queries + q) * KP;
            top.store(a.part_scores + off, a.part_index + off, a.ref_base);
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, Fmt<F>::kTmemCols);
    }
}

// ---- host side -------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

int make_known_map(CUtensorMap* map, const CompareArgs& a, int box_rows) {
    auto fn = encode_fn();
    if (!fn) FASTID_FAIL(FASTID_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)a.stride, (cuuint64_t)a.n_refs};
    cuuint64_t strides[1] = {(cuuint64_t)a.stride};
    cuuint32_t box[2] = {(cuuint32_t)kStageBytesPacked, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)a.refs, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) FASTID_FAIL(FASTID_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return FASTID_OK;
}

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <int F>
int slices_for(int64_t n_refs, int64_t n_queries) {
    const int64_t groups = ceil_div(n_queries, kM);
    const int64_t tiles = ceil_div(n_refs, Fmt<F>::BN);
    int64_t s = num_sms() / (groups > 0 ? groups : 1);
    if (s < 1) s = 1;
    if (s > tiles) s = tiles;
    if (s < 1) s = 1;
    return (int)s;
}

template <int F, int MODE, int KP>
int launch_one(const CompareArgs& a, int n_slices, cudaStream_t stream) {
    CUtensorMap map;
    if (int rc = make_known_map(&map, a, Fmt<F>::BN)) return rc;
    const Layout<F> lay(a.stride);
    if (lay.sp < 2 || lay.total > kSmemLimit)
        FASTID_FAIL(FASTID_E_UNSUPPORTED, "tile needs %d bytes of shared memory", lay.total);
    auto kern = tensor_kernel<F, MODE, KP>;
    FASTID_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.total));
    const int64_t groups = ceil_div(a.n_queries, kM);
    const int64_t tiles = ceil_div(a.n_refs, Fmt<F>::BN);
    kern<<<(unsigned)(groups * n_slices), kThreads, lay.total, stream>>>(map, a, tiles, n_slices);
    FASTID_LAUNCHED("tensor_kernel");
    return FASTID_OK;
}

template <int F>
int launch_fmt(Mode mode, const CompareArgs& a, int* n_parts, cudaStream_t stream) {
    const int slices = slices_for<F>(a.n_refs, a.n_queries);
    if (mode == kFull) return launch_one<F, kFull, 1>(a, slices, stream);
    if (mode == kThreshold) return launch_one<F, kThreshold, 1>(a, slices, stream);
    *n_parts = 2 * slices;  // one partial list per (slice, epilogue column half)
    switch (a.kpad) {
        case 8: return launch_one<F, kTopK, 8>(a, slices, stream);
        case 16: return launch_one<F, kTopK, 16>(a, slices, stream);
        case 32: return launch_one<F, kTopK, 32>(a, slices, stream);
    }
    FASTID_FAIL(FASTID_E_INVALID, "unsupported list size %d", a.kpad);
}

}  // namespace

int tensor_supported(int64_t bit_length, int formulation) {
    const int64_t stride = row_stride_bytes(bit_length);
    if (formulation == FASTID_TENSOR_I8) return Layout<FASTID_TENSOR_I8>(stride).sp >= 2;
    if (formulation == FASTID_TENSOR_F4) return Layout<FASTID_TENSOR_F4>(stride).sp >= 2;
    return 0;
}

int tensor_parts(int64_t n_refs, int64_t n_queries, int formulation) {
    if (formulation == FASTID_TENSOR_I8) return 2 * slices_for<FASTID_TENSOR_I8>(n_refs, n_queries);
    return 2 * slices_for<FASTID_TENSOR_F4>(n_refs, n_queries);
}

int launch_tensor(Mode mode, const CompareArgs& a, int formulation, int* n_parts, cudaStream_t stream) {
    if (formulation == FASTID_TENSOR_I8) return launch_fmt<FASTID_TENSOR_I8>(mode, a, n_parts, stream);
    if (formulation == FASTID_TENSOR_F4) return launch_fmt<FASTID_TENSOR_F4>(mode, a, n_parts, stream);
    FASTID_FAIL(FASTID_E_INVALID, "not a tensor formulation: %d", formulation);
}

}  // namespace fastid

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
// Persistent, warp-specialised kernels (one CTA per SM; roles in Roles<>):
//   * packed operands: 8 converter warps unpack the TMA-streamed packed known
//     rows into the UMMA K-major operand layout every tile, 8 epilogue warps;
//   * prepared image (KnownDatabase): the operand bytes stream straight into
//     the ring, 12 (mxf4) / 16 (i8) epilogue warps; for mxf4 a CTA pair
//     (cluster of 2, tcgen05.mma.cta_group::2, M = 256) shares every known
//     tile, each CTA streaming half of it;
//   * one producer warp (TMA / bulk copies) and one MMA warp; each keeps the
//     whole warp in its loop and elects one lane to issue.
// The MMA fills one of two TMEM accumulators (BN fp32/s32 columns) while the
// epilogue drains the other: full u32 store (TMA tensor stores for pairs),
// per-unknown top-k with a shared admission bound, or threshold hits.
// The unknown tile (128 unknowns per CTA) stays resident in shared memory
// (streamed per stage for long profiles).  CTAs of one slice index walk the
// same known tiles at the same time, with bounded drift, so each known tile
// is read from HBM once and served to the other unknown groups from L2.
// DESIGN.md has the roofline and byte accounting.
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "tensor_ptx.cuh"

namespace fastid {
namespace {

constexpr int kM = 128;             // unknowns per CTA (MMA M, TMEM lanes)
constexpr int kStageBytesPacked = 32;  // packed bytes per known row per stage (256 loci)
constexpr int kWordsPerStage = kStageBytesPacked / 4;
constexpr int kMaxPackedStages = 12;
constexpr int kMinPackedStages = 4;
constexpr int kMaxUnpackedStages = 12;  // barrier slots; dual-tile pairs use up to 12 ring stages
constexpr int kDefaultUnpackedStages = 8;
// Dual-tile pairs: the second tile may lag the first by kDualLag stages (the
// first tile's accumulator then drains while the second finishes), and the A
// ring keeps kDualPrefetch stages of prefetch beyond the lag (fewer than 3 A
// stages in flight stall the MMA: A ring 6 / lag 4 took 18.7 ms on C4).  The
// lag removes the MMA warp's accumulator wait (1850 -> 75 cycles per step,
// tools/trace_dual.py) but not time: timed by ncu at equal clocks
// (tools/ncu_ab.py, 512 x 20M x 5000) A ring 5 / lag 0 takes 13.13-13.15 ms,
// 4 / 0 13.28, 7 / 0 13.17, 6 / 2 13.26, 7 / 3 13.32-13.34 -- so no lag by
// default (FASTID_DUAL_LAG / FASTID_DUAL_SA override).
constexpr int kDualLag = 0;
constexpr int kDualPrefetch = 4;
constexpr int kPrefetchStages = 16;
// The image is read by 2-D TMA boxes over a view of 2 KB rows (u64 elements, the
// widest inner box): a half stage (12 KB) is 6 rows.  With 128-B rows (96 per
// half) the pair kernel streamed an image that misses in L2 at 1.8 TB/s (one
// unknown group: 5.6 ms for 20M x 1024 loci); the single-CTA kernel's 1-D bulk
// copies reach 6.1 TB/s on the same stream.
constexpr int kImgRowBytes = 2048;  // L2 prefetch distance of the pair kernels' known-tile stream
constexpr int kMaxAStages = 8;
// Warp roles.  The two single-thread issuers (TMA producer, MMA) take the
// highest warp ids (the scheduler favours higher ids), converters the lowest.
// Packed operands: 8 converter warps (two per SMSP) + 8 epilogue warps.  A
// prepared image needs no converters: the epilogue gets 12 warps (mxf4, three
// column splits of 64) or 16 (i8, four of 32) -- at 14 warps per CTA no SMSP
// holds more than 4, which leaves 128 registers per thread for the epilogue
// to hold all of its accumulator columns at once.
template <int F, bool IMG>
struct Roles {
    static constexpr int kConvWarps = IMG ? 0 : 8;
    static constexpr int kEpiWarps = IMG ? (F == FASTID_TENSOR_F4 ? 12 : 16) : 8;
    static constexpr int kBuildWarps = IMG ? 4 : kConvWarps;  // build the resident A tile
    static constexpr int kFirstEpiWarp = kConvWarps;
    static constexpr int kProducerWarp = kConvWarps + kEpiWarps;
    static constexpr int kMmaWarp = kProducerWarp + 1;
    static constexpr int kThreads = 32 * (kMmaWarp + 1);
};
// Accumulator buffers in TMEM: the MMA fills one while the epilogue drains
// the others, so an epilogue warp that runs late on one tile (top-k
// insertions) does not stall the tensor pipe.
constexpr int kAccBufs = 2;

// Drift control: the pairs of one slice may lead the slowest of their peers
// by at most drift_tiles tiles, so a tile half fetched from HBM by the first
// of them is still in L2 when the last one reads it.  Resident-unknown pairs
// use 40 tiles; dual-tile pairs size the window in bytes (all slices' windows
// within 48 MB of L2: C4, 20 stages per tile, gets 2 tiles -- with the 40-tile
// window of round 1 the two C4 groups re-read 1.75x the 51 GB image from HBM).
// A lone unknown group has no peers and is not paced (round 2 found that its
// pairs waited on their own stale counter: one unknown, 20M knowns, 5.6 ms ->
// 1.55 ms, HBM-bound).
constexpr int kDriftTilesMax = 40;
constexpr int64_t kDriftWindowBytes = 48ll << 20;
constexpr int kBatch = 32;         // accumulator columns per tcgen05.wait::ld (x8 loads)
constexpr int kMaxSplits = 4;      // epilogue warps per TMEM lane quadrant
constexpr int kSmemLimit = 227 * 1024;

template <int F>
struct Fmt;
template <>
struct Fmt<FASTID_TENSOR_I8> {
    static constexpr int BN = 128;          // knowns per tile (MMA N)
    static constexpr int kCoresPerWord = 2; // 16-B core columns produced per packed u32
    static constexpr int kTmemCols = 512;   // kAccBufs x BN accumulator columns
};
template <>
struct Fmt<FASTID_TENSOR_F4> {
    static constexpr int BN = 192;          // 3 epilogue splits of 64 columns; pairs stream 96 rows each
    static constexpr int kCoresPerWord = 1;
    static constexpr int kTmemCols = 512;   // 2 x 192 accumulators + 64 scale-factor columns (448..511)
};

constexpr uint32_t kSfaCol = 448;  // mxf4: unit scale factors for A (32 columns)
constexpr uint32_t kSfbCol = 480;  // mxf4: unit scale factors for B (32 columns)
constexpr uint32_t kUnitScales = 0x7F7F7F7Fu;  // ue8m0 127 = 2^0

// Operand encodings.  K element (n, j) of a packed word w is bit 4n + j
// (mxf4: nibble n of output word j) or bit 8b + j (i8: byte b of output
// word j); A and B use the same order, so the dot product runs over the
// same loci.  To keep the per-tile (B = known) unpack to masks, B keeps each
// bit where it lies, and the resident A operand (unknowns, built once per
// CTA) carries the reciprocal weight, so every product a_k * b_k is exactly
// a uniform constant:
//   mxf4: B nibble values 0.5 / 1 / 2 / 2 (bits 0,1,2 and bit 3 moved to 2)
//         A nibble values 2 / 1 / 0.5 / 0.5            -> product 1.0
//   i8:   B byte values 2^j, A byte values 2^(7-j)      -> product 128
template <bool B_SIDE>
__device__ __forceinline__ uint4 unpack_f4(uint32_t w) {
    if (B_SIDE) {
        // w >> 1 on the FMA pipe: high word of w * 2^31
        return make_uint4(w & 0x11111111u, w & 0x22222222u, w & 0x44444444u,
                          __umulhi(w, 0x80000000u) & 0x44444444u);
    }
    return make_uint4((w << 2) & 0x44444444u, w & 0x22222222u, (w >> 2) & 0x11111111u, (w >> 3) & 0x11111111u);
}
// The prepared image and the A operands matched with it use one value for
// every set bit (e2m1 0x2 = 1.0 on both sides, product 1.0): the shifts cost
// nothing there (built once).  Kernel time is the same as with the weighted
// pairs above (tools/encoding_ab.py: 11.42 vs 11.41 ms on C3).
__device__ __forceinline__ uint4 unpack_f4_uniform(uint32_t w) {
    return make_uint4((w & 0x11111111u) << 1, w & 0x22222222u, (w >> 1) & 0x22222222u, (w >> 2) & 0x22222222u);
}
// XOR on mxf4: the unknown side is +1 for a clear bit and -1 (e2m1 sign 0x8) for a
// set bit, so the MMA sums r_k (1 - 2 q_k) = popc(r) - 2 popc(r & q) and the
// epilogue adds popc(q): popc(r ^ q) with one FADD and no known-row popcounts.
// Each component of the unpacked words holds its bit at one nibble position
// (uniform: bit 1; weighted A side: bits 2, 1, 0, 0), shifted up to bit 3.
__device__ __forceinline__ uint4 unpack_f4_xor(uint32_t w, bool uniform) {
    if (uniform) {
        const uint4 s = unpack_f4_uniform(w);
        return make_uint4(0x22222222u | s.x << 2, 0x22222222u | s.y << 2, 0x22222222u | s.z << 2,
                          0x22222222u | s.w << 2);
    }
    const uint4 s = unpack_f4<false>(w);
    return make_uint4(0x44444444u | s.x << 1, 0x22222222u | s.y << 2, 0x11111111u | s.z << 3,
                      0x11111111u | s.w << 3);
}
// The A-side nibbles of one word of unknown bits (already complemented for AND-NOT);
// zero outside the row.
__device__ __forceinline__ uint4 unpack_a_f4(uint32_t w, bool uniform, bool xor_op, bool in_row) {
    if (xor_op) return in_row ? unpack_f4_xor(w, uniform) : make_uint4(0, 0, 0, 0);
    return uniform ? unpack_f4_uniform(w) : unpack_f4<false>(w);
}

// The producer waits for ring slots with a suspend-time hint (it runs stages
// ahead of the MMA, so its wake-up latency is hidden; sleeping instead of
// re-issuing try_wait lowers power under the cap): ~1% on C3.
__device__ __forceinline__ void producer_wait(const CompareArgs& a, uint64_t* bar, uint32_t parity) {
    if (experiment(a, 8192))
        ptx::mbar_wait(bar, parity);
    else
        ptx::mbar_wait_sleep(bar, parity);
}

// debug flag 512 keeps the weighted encoding for the image too (A/B timing; image and
// queries must be prepared under the same setting)
__device__ __forceinline__ bool uniform_image(const CompareArgs& a) { return !experiment(a, 512); }

template <bool B_SIDE>
__device__ __forceinline__ void unpack_i8(uint32_t w, uint4& lo, uint4& hi) {
    if (B_SIDE) {
        lo = make_uint4(w & 0x01010101u, w & 0x02020202u, w & 0x04040404u, w & 0x08080808u);
        hi = make_uint4(w & 0x10101010u, w & 0x20202020u, w & 0x40404040u, w & 0x80808080u);
        return;
    }
    // byte b of word j = bit (8b + j) << (7 - j)
    lo = make_uint4((w << 7) & 0x80808080u, (w << 5) & 0x40404040u, (w << 3) & 0x20202020u, (w << 1) & 0x10101010u);
    hi = make_uint4((w >> 1) & 0x08080808u, (w >> 3) & 0x04040404u, (w >> 5) & 0x02020202u, (w >> 7) & 0x01010101u);
}

// Accumulator encodings.  mxf4 accumulates exact integers in fp32, whose bit
// patterns order like the integers (non-negative floats); i8 accumulates s32.
template <int F>
__device__ __forceinline__ uint32_t score_bits(uint32_t s) {
    // i8 accumulates 128 * score; saturate thresholds above the representable range
    return F == FASTID_TENSOR_F4 ? __float_as_uint((float)s) : (s >= (1u << 24) ? 0xFFFFFFFFu : s << 7);
}
template <int F>
__device__ __forceinline__ uint32_t decode_exact(uint32_t v) {
    return F == FASTID_TENSOR_F4 ? (uint32_t)__uint_as_float(v) : v >> 7;
}
// float -> u32 for integers < 2^23 without F2I: add 2^23, read the mantissa.
template <int F>
__device__ __forceinline__ uint32_t decode_fast(uint32_t v) {
    return F == FASTID_TENSOR_F4 ? __float_as_uint(__uint_as_float(v) + 8388608.0f) - 0x4B000000u : v >> 7;
}

// Unsigned minimum of 32 values with 3-input mins (raw fp32 bits of
// non-negative floats order like the floats).
__device__ __forceinline__ uint32_t min32(const uint32_t (&v)[32]) {
    uint32_t m[11];
#pragma unroll
    for (int i = 0; i < 10; ++i) m[i] = __vimin3_u32(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    m[10] = __vimin3_u32(v[30], v[31], 0xFFFFFFFFu);
    const uint32_t a = __vimin3_u32(m[0], m[1], m[2]);
    const uint32_t b = __vimin3_u32(m[3], m[4], m[5]);
    const uint32_t c = __vimin3_u32(m[6], m[7], m[8]);
    return __vimin3_u32(__vimin3_u32(a, b, c), m[9], m[10]);
}

// v[c] for a run-time c without local memory: a 5-level select tree.
__device__ __forceinline__ uint32_t pick32(const uint32_t (&v)[32], int c) {
    uint32_t a[16], b[8], d[4], e[2];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = (c & 16) ? v[i + 16] : v[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) b[i] = (c & 8) ? a[i + 8] : a[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = (c & 4) ? b[i + 4] : b[i];
#pragma unroll
    for (int i = 0; i < 2; ++i) e[i] = (c & 2) ? d[i + 2] : d[i];
    return (c & 1) ? e[1] : e[0];
}

// Position in a ring of mbarrier-guarded stages: slot index + phase parity.
struct Ring {
    int idx;
    uint32_t phase;
    int n;
    __device__ explicit Ring(int n_) : idx(0), phase(0), n(n_) {}
    __device__ __forceinline__ void next() {
        if (++idx == n) {
            idx = 0;
            phase ^= 1u;
        }
    }
};

// Core-matrix offset of (row, core column) in a K-major no-swizzle operand of `rows` rows.
__device__ __forceinline__ uint32_t core_off(int row, int col, int rows) {
    return (uint32_t)col * (uint32_t)(rows * 16) + (uint32_t)(row >> 3) * 128u + (uint32_t)(row & 7) * 16u;
}

// k-th smallest of the kMinSlots published list minima of one unknown
// (unpublished slots hold 0xFFFFFFFF): sorted insertion of each value into a
// K-entry register list, every position updated in parallel.
template <int K>
__device__ __forceinline__ uint32_t kth_smallest_published(const uint32_t* mins, int k) {
    uint32_t v[kMinSlots];
#pragma unroll
    for (int j = 0; j < kMinSlots / 4; ++j) {
        const uint4 x = __ldcg(reinterpret_cast<const uint4*>(mins) + j);
        v[4 * j] = x.x, v[4 * j + 1] = x.y, v[4 * j + 2] = x.z, v[4 * j + 3] = x.w;
    }
    uint32_t best[K];
#pragma unroll
    for (int i = 0; i < K; ++i) best[i] = 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < kMinSlots; ++j) {
        bool le[K];
#pragma unroll
        for (int i = 0; i < K; ++i) le[i] = best[i] <= v[j];
#pragma unroll
        for (int i = K - 1; i > 0; --i) best[i] = le[i] ? best[i] : (le[i - 1] ? v[j] : best[i - 1]);
        best[0] = le[0] ? best[0] : v[j];
    }
    uint32_t r = best[0];
#pragma unroll
    for (int i = 1; i < K; ++i) r = i < k ? best[i] : r;  // best[k - 1] with static indexing
    return r;
}

template <int F>
struct Layout {
    static constexpr int BN = Fmt<F>::BN;
    static constexpr int kUnpackedStageBytes = BN * 16 * kWordsPerStage * Fmt<F>::kCoresPerWord;
    static constexpr int kPackedStageBytes = BN * kStageBytesPacked;
    static constexpr int kAStageBytes = kM * 16 * kWordsPerStage * Fmt<F>::kCoresPerWord;
    static constexpr int kBarBytes = 8 * (2 * kMaxPackedStages + 2 * kMaxUnpackedStages + 2 * kMaxAStages + 2 * kAccBufs + 1) + 16;
    int n_kst;    // stages per tile (K padded to 256 loci)
    int a_bytes;  // resident A tile, or the A ring when streaming
    int sa;       // A ring depth (streamed A only)
    int su;       // operand ring depth (converter or TMA -> MMA)
    int sp;       // packed ring depth (TMA -> converter); 0 with a tensor image
    bool img;
    int ub;       // operand-ring stage bytes: the whole tile, or this CTA's half of it in a pair
    int off_u, off_p, off_bar, total;
    int out_bytes;  // full-matrix TMA-store staging (image kernels): one [cols][32] u32 block per epilogue warp
    int off_out;
    int su_max;  // operand-ring depth cap
    __host__ __device__ Layout(int64_t stride, bool stream_a, bool image = false, bool pair = false,
                               int stage_out = 0, int want_sa = 0) {
        n_kst = (int)((stride + kStageBytesPacked - 1) / kStageBytesPacked);
        img = image;
        out_bytes = stage_out;
        ub = pair ? kUnpackedStageBytes / 2 : kUnpackedStageBytes;
        sa = 0;
        su_max = kDefaultUnpackedStages;
        if (stream_a && image && pair) {
            // dual-tile pairs: an A stage stays resident for the second tile's lag
            // (kDualLag stages) plus kDualPrefetch stages of prefetch, and the operand
            // ring holds two stages per A stage in flight: the deepest A ring up to
            // kDualLag + 1 + kDualPrefetch whose operand ring still has sa + 2 stages
            su_max = kMaxUnpackedStages;
            if (want_sa >= 2 && want_sa <= kMaxAStages) {
                sa = want_sa;
                a_bytes = sa * kAStageBytes;
                place();
                if (fits()) return;
            }
            for (sa = kDualLag + 1 + kDualPrefetch < kMaxAStages ? kDualLag + 1 + kDualPrefetch : kMaxAStages; sa >= 3;
                 --sa) {
                a_bytes = sa * kAStageBytes;
                place();
                if (fits() && su >= sa + 2) return;
            }
            sa = 2;
            a_bytes = sa * kAStageBytes;
            place();
            return;
        }
        if (!stream_a) {
            a_bytes = n_kst * kAStageBytes;
            place();
        } else {
            // deepest A ring that still leaves an operand ring of >= 4 stages,
            // else >= 3, else >= 2 (A and B stages are consumed in lockstep)
            bool ok = false;
            for (int min_su = 4; min_su >= 2 && !ok; --min_su)
                for (sa = kMaxAStages; sa >= 2; --sa) {
                    a_bytes = sa * kAStageBytes;
                    place();
                    if (fits() && su >= min_su) {
                        ok = true;
                        break;
                    }
                }
            if (!ok) {  // nothing fits: leave an unfit layout for the caller to reject
                sa = 2;
                a_bytes = sa * kAStageBytes;
                place();
            }
        }
    }
    __host__ __device__ void place() {
        const int room = kSmemLimit - a_bytes - kBarBytes - out_bytes - (out_bytes ? 128 : 0);
        if (img) {
            // the tensor image is already in the UMMA layout: only the operand ring
            su = room / ub;
            if (su > su_max) su = su_max;
            sp = 0;
        } else {
            // deepest unpacked ring that still leaves kMinPackedStages TMA stages
            su = (room - kMinPackedStages * kPackedStageBytes) / kUnpackedStageBytes;
            if (su > su_max) su = su_max;
            sp = su >= 2 ? (room - su * kUnpackedStageBytes) / kPackedStageBytes : 0;
            if (sp > kMaxPackedStages) sp = kMaxPackedStages;
        }
        off_u = a_bytes;
        off_p = off_u + (su > 0 ? su : 0) * ub;
        off_bar = off_p + (sp > 0 ? sp : 0) * kPackedStageBytes;
        off_out = off_bar + kBarBytes;
        off_out = (off_out + 127) & ~127;
        total = off_out + out_bytes;
    }
    __host__ __device__ bool fits() const { return su >= 2 && (img || sp >= 2) && total <= kSmemLimit; }
};

// Full-matrix staging for TMA tensor stores (CTA-pair kernel): every epilogue
// warp owns a [columns][32 unknowns] u32 block.
template <int F, int MODE, bool IMG, bool PAIR>
constexpr int out_stage_bytes() {
    return (PAIR && MODE == kFull) ? Roles<F, IMG>::kEpiWarps * (Fmt<F>::BN / (Roles<F, IMG>::kEpiWarps / 4)) * 32 * 4
                                   : 0;
}

// PAIR: a CTA pair (cluster of 2) issues cta_group::2 MMAs with M = 256 (each
// CTA's 128 unknowns) and N = BN knowns, each CTA streaming only its half of
// the known tile (BN/2 rows of the prepared image) -- half the L2->SM operand
// traffic per MAC of the single-CTA kernel, which is L2-throughput-bound.
// The leader (rank 0) issues every MMA; the commits multicast to both CTAs.
template <int F, int MODE, int KP, bool SA, bool IMG, bool PAIR, bool SPARE>
__global__ void __launch_bounds__(Roles<F, IMG>::kThreads, 1)
    tensor_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap omap,
                  const __grid_constant__ CUtensorMap amap, CompareArgs a, const uint8_t* __restrict__ a_global,
                  int64_t n_tiles, int n_slices) {
    static_assert(!PAIR || (F == FASTID_TENSOR_F4 && IMG), "pairs run the prepared mxf4 image only");
    static_assert(kAccBufs * Fmt<F>::BN <= (F == FASTID_TENSOR_F4 ? (int)kSfaCol : Fmt<F>::kTmemCols), "TMEM columns");
    constexpr int BN = Fmt<F>::BN;
    constexpr int CPW = Fmt<F>::kCoresPerWord;
    // the mxf4 image is stored in the pair layout: each stage = two BN/2-row halves
    constexpr bool kSplitB = IMG && F == FASTID_TENSOR_F4;
    constexpr int UB = Layout<F>::kUnpackedStageBytes;
    constexpr int HB = UB / 2;                 // one half of an image stage
    constexpr int RB = PAIR ? HB : UB;         // bytes this CTA receives per stage
    constexpr int kImgHalfRows = HB / kImgRowBytes;  // image-map rows per half stage
    static_assert(!PAIR || HB % kImgRowBytes == 0, "half stage must be whole image-map rows");
    constexpr int PB = Layout<F>::kPackedStageBytes;
    // Dual-tile CTA pairs (streamed A, long profiles): each A stage feeds the
    // MMAs of two known tiles (one per accumulator), halving the A operand's
    // L2->SM bytes per MAC.  The epilogue sees the same tile sequence.
    constexpr bool kDual = PAIR && SA;
    constexpr int kTileStep = kDual ? 2 : 1;
    // The second tile of a dual step lags the first by `lag` stages: the first
    // tile's accumulator completes `lag` stages early and drains while the MMA
    // pipe finishes the second (and the second's drains while the next first
    // tile runs its first `lag` stages), so the pipe never waits for a buffer.
    // Each A stage stays in the ring for `lag` stages (ring depth >= lag + 2).
    using R = Roles<F, IMG>;
    constexpr int kConvThreads = 32 * R::kConvWarps;
    constexpr int kEpiWarps = R::kEpiWarps, kEpiThreads = 32 * R::kEpiWarps;
    constexpr int kBuildWarps = R::kBuildWarps;
    constexpr int kFirstEpiWarp = R::kFirstEpiWarp, kProducerWarp = R::kProducerWarp, kMmaWarp = R::kMmaWarp;
    extern __shared__ __align__(1024) uint8_t smem[];
    const Layout<F> lay(a.stride, SA, IMG, PAIR, a.tma_out ? out_stage_bytes<F, MODE, IMG, PAIR>() : 0, a.dual_sa);
    constexpr int AB = Layout<F>::kAStageBytes;
    const int SP = lay.sp;
    const int SU = lay.su;
    const int n_kst = lay.n_kst;
    const int lag = !kDual ? 0
                           : max(0, min(a.dual_lag >= 0 ? min(a.dual_lag, lay.sa - 2)
                                                        : min(kDualLag, lay.sa - 1 - kDualPrefetch),
                                        n_kst));
    uint8_t* sA = smem;
    uint8_t* sU = smem + lay.off_u;
    uint8_t* sP = smem + lay.off_p;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.off_bar);
    uint64_t* p_full = bars;
    uint64_t* p_empty = p_full + kMaxPackedStages;
    uint64_t* u_full = p_empty + kMaxPackedStages;
    uint64_t* u_empty = u_full + kMaxUnpackedStages;
    uint64_t* t_full = u_empty + kMaxUnpackedStages;
    uint64_t* t_empty = t_full + kAccBufs;
    uint64_t* a_full = t_empty + kAccBufs;
    uint64_t* ar_full = a_full + 1;  // streamed-A ring
    uint64_t* ar_empty = ar_full + kMaxAStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ar_empty + kMaxAStages);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (experiment(a, 64) && trace_buf(a) && threadIdx.x == 0) trace_buf(a)[blockIdx.x * 4] = (long long)ptx::globaltimer();
    const uint32_t rank = PAIR ? ptx::cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    const int unit = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // CTA pair or CTA
    // Work segments.  A regular unit owns slice `unit % n_slices` of the first
    // t_main tiles for unknown group `unit / n_slices`.  Spare CTA pairs (the
    // SMs left over by groups x slices, a.n_spare of them) each take the last
    // n_tiles - t_main tiles of a_groups / n_spare groups in turn, as list
    // slot n_slices, rebuilding the resident unknowns between groups.
    // (the spare pairs are a separate launch, SPARE = true, on the SMs the
    // regular grid leaves free; for regular launches every loop over
    // segments has a compile-time trip count of 1)
    constexpr bool spare = SPARE;
    const int per_spare = SPARE ? a.n_groups / a.n_spare : 1;
    const int n_seg = SPARE ? per_spare : 1;
    const int64_t t_main = PAIR && a.n_spare ? a.t_main : n_tiles;
    const int slice = spare ? n_slices : unit % n_slices;  // partial-list slot
    // A regular unit takes every n_slices-th of the first t_main tiles, starting at
    // its slice (slices interleaved, so at any moment the units stream neighbouring
    // tiles spread over every HBM channel; with one contiguous range per slice the
    // units advanced in lock step through ranges 1/n_slices of the image apart and
    // camped on the same channels: one unknown group, 20M x 1024 loci, took 5.6 ms
    // with per-pair finish times from 1.7 to 5.8 ms).  A spare unit takes the
    // contiguous tail.  Tiles of a unit ascend, as the top-k insertion requires.
    const int64_t t_first = spare ? t_main : slice;
    const int64_t t_stride = spare ? 1 : n_slices;
    const int64_t t_count = spare ? n_tiles - t_main : (t_main > slice ? (t_main - slice + n_slices - 1) / n_slices : 0);
    auto tile_of = [&](int64_t i) { return t_first + i * t_stride; };
    auto seg_group = [&](int sg) { return spare ? unit * per_spare + sg : unit / n_slices; };
    auto seg_q0 = [&](int sg) { return ((int64_t)seg_group(sg) * (PAIR ? 2 : 1) + rank) * kM; };

    if (threadIdx.x == 0) {
        for (int i = 0; i < SP; ++i) {
            ptx::mbar_init(&p_full[i], 1);
            ptx::mbar_init(&p_empty[i], kConvThreads);
        }
        for (int i = 0; i < SU; ++i) {
            ptx::mbar_init(&u_full[i], IMG ? 1 : kConvThreads);
            ptx::mbar_init(&u_empty[i], 1);
        }
        for (int i = 0; i < kAccBufs; ++i) {
            ptx::mbar_init(&t_full[i], 1);
            // pairs: one arrival per epilogue warp of both CTAs (on the leader's barrier)
            ptx::mbar_init(&t_empty[i], PAIR ? 2 * kEpiWarps : kEpiThreads);
        }
        ptx::mbar_init(a_full, PAIR ? 2 * kBuildWarps : 32 * kBuildWarps);
        for (int i = 0; i < kMaxAStages; ++i) {
            ptx::mbar_init(&ar_full[i], 1);
            ptx::mbar_init(&ar_empty[i], 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == kProducerWarp && lane == 0) ptx::prefetch_tmap(&tmap);
    if (PAIR) ptx::cluster_sync();  // peer barriers initialised before any remote arrive / TMA
    if (warp == kMmaWarp) {
        if (PAIR)
            ptx::tmem_alloc_pair(tmem_slot, Fmt<F>::kTmemCols);
        else
            ptx::tmem_alloc(tmem_slot, Fmt<F>::kTmemCols);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // debug flag 64: per-CTA %globaltimer stamps (entry, roles start, roles done, exit)
    const bool cta_trace = experiment(a, 64) && trace_buf(a) && threadIdx.x == 0;
    if (cta_trace) trace_buf(a)[blockIdx.x * 4 + 1] = (long long)ptx::globaltimer();
    if (F == FASTID_TENSOR_F4 && warp >= kFirstEpiWarp && warp < kProducerWarp) {
        // unit block scales (ue8m0 127) for every MMA: whole SF region, all lanes
        const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        ptx::tmem_fill32(lb + kSfaCol, kUnitScales);
        ptx::tmem_fill32(lb + kSfbCol, kUnitScales);
        ptx::tmem_wait_st();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();

    if (warp == kProducerWarp) {
        // ---------------- TMA producer (whole warp; one elected lane issues) ----------------
        {
            Ring ra(SA ? lay.sa : 1), rp(SP > 0 ? SP : 1), ru(SU);
            // Pairs of one slice (same known tiles, different unknown groups) stay
            // within kDriftTiles of each other so every tile half is fetched from
            // HBM once and served to the other groups from L2: the leader's
            // producer publishes its progress and waits (bounded) while it leads
            // the slowest pair of its slice by more than that.
            // (a lone unknown group has no peers to pace against)
            int* prog = (PAIR && leader && a.progress && !spare && a.n_groups > 1)
                            ? a.progress + (int64_t)slice * a.n_groups
                            : nullptr;
            const int group = seg_group(0);  // drift control: regular units only (one segment)
            // lane l watches the counter of group l -- every peer group, never this pair's own
            // (its own published value is stale by a check and would read as a false lead)
            const bool watch = lane < a.n_groups && lane != group;
            // The peers' counters are loaded at one check and consumed at the next,
            // so their latency never stalls the operand stream.
            int local_t = 0;
            int peer = 0x7FFFFFFF;  // this lane's peer counter, in flight since the last check
            // L2 prefetch of the same half `pf_tiles` tiles (>= kPrefetchStages stages) ahead:
            // a known tile read by few unknown groups comes from HBM at every load, and the
            // operand ring alone keeps too few bytes in flight to cover HBM latency (one
            // unknown group: 1.6 TB/s).  Within this segment's tiles only.
            const int64_t pf_tiles = (int64_t)kTileStep * ((kPrefetchStages + n_kst - 1) / n_kst);
            const bool pf_on = PAIR && a.l2_prefetch;
            auto prefetch_half = [&](int64_t i, int ks) {  // i: the unit's tile index
                if (pf_on && i + pf_tiles < t_count)
                    ptx::tma_prefetch_2d(&tmap, 0, (int)(((tile_of(i + pf_tiles) * n_kst + ks) * 2 + rank) * kImgHalfRows));
            };
            // this CTA's half of known tile `tile`, stage `ks` (tensor map over the image,
            // box = one half); completion is counted on the leader's barrier, which expects both
            auto load_half = [&](int64_t i, int ks, Ring& r) {  // i: the unit's tile index
                producer_wait(a, &u_empty[r.idx], r.phase ^ 1);
                if (ptx::elect_one()) {
                    if (leader) ptx::mbar_expect_tx(&u_full[r.idx], 2 * HB);
                    ptx::tma_load_2d_pair(sU + r.idx * HB, &tmap, ptx::mapa(&u_full[r.idx], 0), 0,
                                          (int)(((tile_of(i) * n_kst + ks) * 2 + rank) * kImgHalfRows));
                    prefetch_half(i, ks);
                }
                __syncwarp();
                r.next();
            };
            for (int sg = 0; sg < n_seg; ++sg) {
            // first 128-B row of this segment's streamed-A stages (warp-uniform, hoisted)
            const int64_t a_row0 = ((int64_t)seg_group(sg) * 2 + rank) * n_kst * (AB / 128);
            int next_check = 0;
            for (int64_t i = 0; i < t_count; i += kTileStep) {
                const int64_t t = tile_of(i);
                // dual-tile pairs (streamed A): the unit's tiles i and i + 1 share every A stage
                const bool two = kDual && i + 1 < t_count;
                if (prog && local_t >= next_check) {
                    next_check = local_t + a.drift_every;
                    // `peer` was loaded at the previous check, drift_every tiles ago: peers in
                    // step have advanced about that much since, so only a lead beyond the window
                    // plus that staleness is real -- then wait on fresh reads.  (Waiting on the
                    // stale lead alone cost a sleep + reload per check: 2 groups x 20M x 1024
                    // loci took 4.8 ms with a 13-tile window, 11.2 ms with 6, 3.2 ms unpaced.)
                    int lo = __reduce_min_sync(0xFFFFFFFFu, peer);
                    int spin = 0;
                    if (local_t - lo > a.drift_tiles + a.drift_every) {
                        lo = watch ? ptx::ld_relaxed(prog + lane) : 0x7FFFFFFF;
                        lo = __reduce_min_sync(0xFFFFFFFFu, lo);
                        for (; spin < 4096 && local_t - lo > a.drift_tiles; ++spin) {
                            __nanosleep(256);
                            lo = watch ? ptx::ld_relaxed(prog + lane) : 0x7FFFFFFF;
                            lo = __reduce_min_sync(0xFFFFFFFFu, lo);
                        }
                    }
                    if (lane == 0) ptx::st_relaxed(prog + group, spin == 4096 ? 0x7FFFFFFF : local_t);
                    // a peer that stays ~1 ms behind is not co-resident (a shared GPU):
                    // stop pacing rather than wait on it again
                    if (spin == 4096) prog = nullptr;
                    if (prog) peer = watch ? ptx::ld_relaxed(prog + lane) : 0x7FFFFFFF;
                }
                if constexpr (kDual) {
                    // A stage ks and the first tile's half at step ks; the second tile's
                    // half of stage ks - d at step ks (the MMA warp's consumption order)
                    const int d = two ? lag : 0;
                    for (int ks = 0; ks < n_kst + d; ++ks) {
                        if (ks < n_kst) {
                            const int sa = ra.idx;
                            producer_wait(a, &ar_empty[sa], ra.phase ^ 1);
                            if (ptx::elect_one()) {
                                if (leader) ptx::mbar_expect_tx(&ar_full[sa], 2 * AB);
                                ptx::tma_load_2d_pair(sA + sa * AB, &amap, ptx::mapa(&ar_full[sa], 0), 0,
                                                      (int)(a_row0 + (int64_t)ks * (AB / 128)));
                            }
                            __syncwarp();
                            ra.next();
                            load_half(i, ks, ru);
                        }
                        if (two && ks >= d) load_half(i + 1, ks - d, ru);
                    }
                } else {
                for (int ks = 0; ks < n_kst; ++ks, rp.next()) {
                    if (SA) {
                        // this stage's slice of the pre-unpacked A operand (one bulk copy)
                        const int sa = ra.idx;
                        producer_wait(a, &ar_empty[sa], ra.phase ^ 1);
                        if (ptx::elect_one()) {
                            if (PAIR) {
                                // each CTA streams its own 128 unknowns' stage; the leader's
                                // barrier counts both
                                if (leader) ptx::mbar_expect_tx(&ar_full[sa], 2 * AB);
                                ptx::tma_load_2d_pair(sA + sa * AB, &amap, ptx::mapa(&ar_full[sa], 0), 0,
                                                      (int)(a_row0 + (int64_t)ks * (AB / 128)));
                            } else {
                                ptx::mbar_expect_tx(&ar_full[sa], AB);
                                ptx::bulk_load(sA + sa * AB, a_global + ((int64_t)group * n_kst + ks) * AB, AB,
                                               &ar_full[sa]);
                            }
                        }
                        __syncwarp();
                        ra.next();
                    }
                    if (PAIR) {
                        // this CTA's half of the stage (tensor map over the image, box = one
                        // half); completion is counted on the leader's barrier, which expects both
                        producer_wait(a, &u_empty[ru.idx], ru.phase ^ 1);
                        if (ptx::elect_one()) {
                            if (experiment(a, 4)) {  // timing experiment: no operand traffic
                                if (leader) ptx::mbar_arrive(&u_full[ru.idx]);
                            } else {
                                if (leader) ptx::mbar_expect_tx(&u_full[ru.idx], 2 * HB);
                                ptx::tma_load_2d_pair(sU + ru.idx * HB, &tmap, ptx::mapa(&u_full[ru.idx], 0), 0,
                                                      (int)(((t * n_kst + ks) * 2 + rank) * kImgHalfRows));
                                prefetch_half(i, ks);
                            }
                        }
                        __syncwarp();
                        ru.next();
                        continue;
                    }
                    if (IMG) {
                        // the known tile's stage, already unpacked: one bulk copy into the operand ring
                        producer_wait(a, &u_empty[ru.idx], ru.phase ^ 1);
                        if (ptx::elect_one()) {
                            ptx::mbar_expect_tx(&u_full[ru.idx], UB);
                            ptx::bulk_load(sU + ru.idx * UB, a.image + (t * n_kst + ks) * (int64_t)UB, UB,
                                           &u_full[ru.idx]);
                        }
                        __syncwarp();
                        ru.next();
                        continue;
                    }
                    const int s = rp.idx;
                    ptx::mbar_wait(&p_empty[s], rp.phase ^ 1);
                    if (ptx::elect_one()) {
                        ptx::mbar_expect_tx(&p_full[s], PB);
                        ptx::tma_load_2d(sP + s * PB, &tmap, &p_full[s], ks * kStageBytesPacked, (int)(t * BN));
                    }
                    __syncwarp();
                }
                }  // not dual
                local_t += two ? 2 : 1;
            }
            }
            if (PAIR && leader && a.progress && !spare && lane == 0)
                ptx::st_relaxed(a.progress + (int64_t)slice * a.n_groups + group, 0x7FFFFFFF);  // finished: never waited on
        }
    } else if (warp == kMmaWarp) {
        // ---------------- MMA issuer (the leader's warp for a pair; one elected lane issues) ----------------
        if (leader) {
            constexpr uint32_t idesc = PAIR ? ptx::idesc_mxf4(2 * kM, BN)
                                            : (kSplitB ? ptx::idesc_mxf4(kM, BN / 2)
                                                       : (F == FASTID_TENSOR_F4 ? ptx::idesc_mxf4(kM, BN)
                                                                                : ptx::idesc_i8(kM, BN)));
            constexpr int kBRows = kSplitB ? BN / 2 : BN;  // rows per B core-matrix column
            const uint64_t a_desc0 = ptx::smem_desc(ptx::smem_u32(sA), kM * 16, 128);
            const uint64_t b_desc0 = ptx::smem_desc(ptx::smem_u32(sU), kBRows * 16, 128);
            Ring ru(SU), ra(SA ? lay.sa : 1);
            int local = 0;
            for (int sg = 0; sg < n_seg; ++sg) {
            if (!SA) {  // this segment's resident unknowns are built (phase sg of a_full)
                if (PAIR)
                    ptx::mbar_wait_cluster(a_full, (uint32_t)sg & 1u);
                else
                    ptx::mbar_wait(a_full, (uint32_t)sg & 1u);
            }
            ptx::tc_fence_after();
            for (int64_t i = 0; i < t_count; i += kTileStep) {
                const bool two = kDual && i + 1 < t_count;
                const int acc = local % kAccBufs;
                const uint32_t use = (uint32_t)(local / kAccBufs) & 1u;  // parity of this buffer's use
                // the second tile of a dual step: the other accumulator
                const int acc2 = (local + 1) % kAccBufs;
                const uint32_t use2 = (uint32_t)((local + 1) / kAccBufs) & 1u;
                const bool tr = trace_buf(a) && blockIdx.x == 0 && local < a.trace_tiles && lane == 0;
                if (tr) trace_buf(a)[local * kTrSlots + kTrMmaWait] = clock64();
                // spinning waits: the MMA warp's wake-up latency is on the critical path
                ptx::mbar_wait(&t_empty[acc], use ^ 1);
                if (tr) trace_buf(a)[local * kTrSlots + kTrMmaGo] = clock64();
                ptx::tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * BN);
                const uint32_t d2 = tmem + (uint32_t)(acc2 * BN);
                if constexpr (kDual) {
                    constexpr uint64_t a_step = (2 * kM * 16) >> 4, b_step = (2 * kBRows * 16) >> 4;
                    const int dl = two ? lag : 0;
                    // A ring positions of the two tiles' current stages (the second tile's
                    // trails the first's by dl); both start at this step's first A stage
                    Ring ay = ra;
                    auto mma_half = [&](uint32_t dacc, int sa, int ks, bool release_a) {
                        const int s = ru.idx;
                        ptx::mbar_wait(&u_full[s], ru.phase);
                        ptx::tc_fence_after();
                        const uint64_t ad = a_desc0 + (uint64_t)(((uint32_t)sa * AB) >> 4);
                        const uint64_t bd = b_desc0 + (uint64_t)(((uint32_t)s * RB) >> 4);
                        if (ptx::elect_one()) {
                            ptx::mma_mxf4_pair_stage4(dacc, ad, bd, a_step, b_step, idesc, tmem + kSfaCol,
                                                      tmem + kSfbCol, ks ? 1u : 0u);
                            ptx::tc_commit_pair(&u_empty[s], 0x3);  // both halves of stage s reusable
                            if (release_a) ptx::tc_commit_pair(&ar_empty[sa], 0x3);
                        }
                        __syncwarp();
                        ru.next();
                    };
                    for (int ks = 0; ks < n_kst + dl; ++ks) {
                        if (ks < n_kst) {
                            ptx::mbar_wait(&ar_full[ra.idx], ra.phase);
                            mma_half(d, ra.idx, ks, !two);
                            ra.next();
                            if (two && ks == n_kst - 1) {
                                // the first tile is complete: it drains while the second finishes
                                if (ptx::elect_one()) ptx::tc_commit_pair(&t_full[acc], 0x3);
                                __syncwarp();
                            }
                        }
                        if (two && ks >= dl) {
                            if (ks == dl) ptx::mbar_wait(&t_empty[acc2], use2 ^ 1);
                            mma_half(d2, ay.idx, ks - dl, true);  // the A stage's last reader
                            ay.next();
                        }
                    }
                    if (ptx::elect_one()) ptx::tc_commit_pair(&t_full[two ? acc2 : acc], 0x3);
                    __syncwarp();
                } else {
                for (int ks = 0; ks < n_kst; ++ks) {
                    const int s = ru.idx;
                    const int sa = ra.idx;
                    if (SA) ptx::mbar_wait(&ar_full[sa], ra.phase);
                    const bool trs = tr && experiment(a, 8) && ks < 16;
                    if (trs) trace_buf(a)[local * kTrSlots + kTrB0Loaded + ks] = clock64();
                    ptx::mbar_wait(&u_full[s], ru.phase);
                    if (trs) trace_buf(a)[local * kTrSlots + kTrB0Done + ks] = clock64();
                    ptx::tc_fence_after();
                    // descriptors of this stage's first K-step; later steps add fixed strides
                    const uint32_t a_off = SA ? (uint32_t)(sa * AB) : (uint32_t)(ks * kWordsPerStage * CPW) * (kM * 16);
                    const uint64_t ad = a_desc0 + (uint64_t)(a_off >> 4);
                    const uint64_t bd = b_desc0 + (uint64_t)(((uint32_t)s * RB) >> 4);
                    const uint64_t a_step = (2 * kM * 16) >> 4, b_step = (2 * kBRows * 16) >> 4;
                    if (ptx::elect_one()) {
                        if (PAIR) {
                            ptx::mma_mxf4_pair_stage4(d, ad, bd, a_step, b_step, idesc, tmem + kSfaCol,
                                                      tmem + kSfbCol, ks ? 1u : 0u);
                            ptx::tc_commit_pair(&u_empty[s], 0x3);  // both halves of stage s reusable
                        } else {
                            if (kSplitB)
                                ptx::mma_mxf4_split_stage4(d, BN / 2, ad, bd, (uint64_t)(HB >> 4), a_step, b_step,
                                                           idesc, tmem + kSfaCol, tmem + kSfbCol, ks ? 1u : 0u);
                            else if (F == FASTID_TENSOR_F4)
                                ptx::mma_mxf4_stage4(d, ad, bd, a_step, b_step, idesc, tmem + kSfaCol, tmem + kSfbCol,
                                                     ks ? 1u : 0u);
                            else
                                ptx::mma_i8_stage8(d, ad, bd, a_step, b_step, idesc, ks ? 1u : 0u);
                            ptx::tc_commit(&u_empty[s]);  // stage s reusable once these MMAs retire
                            if (SA) ptx::tc_commit(&ar_empty[sa]);
                        }
                    }
                    __syncwarp();
                    ru.next();
                    if (SA) ra.next();
                }
                if (ptx::elect_one()) {
                    if (PAIR)
                        ptx::tc_commit_pair(&t_full[acc], 0x3);  // both CTAs' accumulators complete
                    else
                        ptx::tc_commit(&t_full[acc]);  // accumulator complete -> epilogue
                }
                __syncwarp();
                }  // not dual
                if (tr) trace_buf(a)[local * kTrSlots + kTrMmaIssued] = clock64();
                local += two ? 2 : 1;
            }
            }
        }
    } else {
        const int ct = threadIdx.x;  // 0..kConvThreads-1 for converters
        // Resident A = complemented unknown rows of one segment's group; zero
        // past the row.  Threads 0..127 of the builder warps each build one row.
        auto build_a = [&](int64_t q0s) {
            // Resident A = the unknown rows (complemented for AND-NOT, +-1 for XOR);
            // zero past the row.  Threads 0..127 each build one row.
            if (!SA && ct < kM) {
                const int64_t q = q0s + ct;
                const bool real = q < a.n_queries;
                const int row_words = (int)(a.stride / 4);
                const uint32_t* src = reinterpret_cast<const uint32_t*>(a.queries + (real ? q : 0) * a.stride);
                for (int w4 = 0; w4 < n_kst * kWordsPerStage; w4 += 4) {
                    uint4 v = make_uint4(0, 0, 0, 0);
                    const bool in_row = real && w4 < row_words;
                    if (in_row) {
                        v = *reinterpret_cast<const uint4*>(src + w4);
                        if (a.op == FASTID_OP_ANDNOT) v = make_uint4(~v.x, ~v.y, ~v.z, ~v.w);
                    }
                    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int col = (w4 + i) * CPW;
                        if (F == FASTID_TENSOR_F4) {
                            *reinterpret_cast<uint4*>(sA + core_off(ct, col, kM)) =
                                unpack_a_f4(wv[i], IMG && uniform_image(a), a.op == FASTID_OP_XOR, in_row);
                        } else {
                            uint4 lo, hi;
                            unpack_i8<false>(wv[i], lo, hi);
                            *reinterpret_cast<uint4*>(sA + core_off(ct, col, kM)) = lo;
                            *reinterpret_cast<uint4*>(sA + core_off(ct, col + 1, kM)) = hi;
                        }
                    }
                }
            }
            ptx::fence_proxy_async_smem();
            if (PAIR) {
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(a_full, 0));
            } else {
                ptx::mbar_arrive(a_full);
            }
        };
        if (warp < kBuildWarps) build_a(seg_q0(0));
        if (warp < kFirstEpiWarp) {
        // ---------------- converters ----------------
        // Work unit = (known row, 16-byte half of the stage): 2*BN units per stage.
        constexpr int kUnits = 2 * BN;
        constexpr int kUnitsPerThread = kConvThreads ? (kUnits + kConvThreads - 1) / (kConvThreads ? kConvThreads : 1) : 1;
        Ring rp(SP), ru(SU);
        for (int64_t i = 0; i < t_count; ++i) {
            for (int ks = 0; ks < n_kst; ++ks, rp.next(), ru.next()) {
                const int sp = rp.idx;
                const int su = ru.idx;
                ptx::mbar_wait(&p_full[sp], rp.phase);
                const uint8_t* P = sP + sp * PB;
                uint4 v[kUnitsPerThread];
#pragma unroll
                for (int h = 0; h < kUnitsPerThread; ++h) {
                    const int u = ct + kConvThreads * h;
                    if (u < kUnits) v[h] = *reinterpret_cast<const uint4*>(P + u * 16);
                }
                ptx::mbar_wait(&u_empty[su], ru.phase ^ 1);
                uint8_t* U = sU + su * UB;
#pragma unroll
                for (int h = 0; h < kUnitsPerThread; ++h) {
                    const int u = ct + kConvThreads * h;
                    if (u >= kUnits) break;
                    const int row = u >> 1;
                    const int col0 = (u & 1) * 4 * CPW;
                    const uint32_t wv[4] = {v[h].x, v[h].y, v[h].z, v[h].w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        if (F == FASTID_TENSOR_F4) {
                            *reinterpret_cast<uint4*>(U + core_off(row, col0 + i, BN)) = unpack_f4<true>(wv[i]);
                        } else {
                            uint4 lo, hi;
                            unpack_i8<true>(wv[i], lo, hi);
                            *reinterpret_cast<uint4*>(U + core_off(row, col0 + 2 * i, BN)) = lo;
                            *reinterpret_cast<uint4*>(U + core_off(row, col0 + 2 * i + 1, BN)) = hi;
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
        // A warp reads TMEM lanes 32*(w%4).. (its quadrant) and 1/n_splits of the
        // accumulator columns, in batches of up to 32 columns (x8 loads, one
        // wait per batch).  Scores stay raw accumulator bits (fp32 of an exact
        // integer orders like u32), so the hot path is a 3-input-min tree and
        // one compare per batch; candidates take a rare per-lane slow path.
        constexpr int kSplits = kEpiWarps / 4;  // 2 (packed) / 3 (mxf4 image) / 4 (i8 image)
        static_assert(kSplits <= kMaxSplits && kSplits * 4 == kEpiWarps, "split count");
        constexpr int kCols = BN / kSplits;  // 96 / 64 (mxf4), 64 / 32 (i8)
        static_assert(kCols * kSplits == BN && kCols % 8 == 0, "columns per split must be a multiple of 8");
        // with an image every column of a split is loaded before any compare work
        constexpr bool kPreload = IMG && kCols <= 2 * kBatch;
        constexpr int kPreBatches = (kCols + kBatch - 1) / kBatch;
        const int ew = warp - kFirstEpiWarp;
        const int quad = warp & 3;
        const int split = ew >> 2;
        const int m = quad * 32 + lane;
        int local = 0;
        for (int sg = 0; sg < n_seg; ++sg) {
        // a spare pair's next group: its builders rebuild the unknowns once the
        // previous group's last accumulator has been read (every MMA reading A is done)
        if (sg > 0 && warp < kBuildWarps) build_a(seg_q0(sg));
        const int64_t q0s = seg_q0(sg);
        const int64_t q = q0s + m;
        const bool q_ok = q < a.n_queries;
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
        TopList<KP> top;
        if (MODE == kTopK) top.clear();
        const uint64_t cap = (uint64_t)a.max_score + 1;  // admit v <= max_score
        uint32_t thr_bits = 0;  // own list: admit v < thr_bits (rows arrive in index order)
        if (MODE == kTopK) thr_bits = score_bits<F>(cap < kEmptyScore ? (uint32_t)cap : kEmptyScore);
        // Admission bound shared by every list of one unknown (all column splits of
        // all slices, a.bound[q], raw score bits, admit v < bound): a value worse
        // than some list's KP-th best cannot be in the union's top k (that list
        // holds KP >= k values <= it; ties are resolved by the merge), so every
        // list admits v <= the minimum published KP-th best, stored + 1 and
        // lowered with atomicMin.  Bounds only decrease, so a stale read is a
        // looser, still correct, bound.  The list itself holds raw bits (decoded
        // at the store), so an insertion needs no float <-> int conversion.
        const uint32_t cap_bits = thr_bits;
        uint32_t thr_eff = thr_bits;
        const bool share = MODE == kTopK && a.bound != nullptr && q_ok;
        // Second bound: every list also publishes its best value; the k-th smallest
        // of those published minima belongs to k distinct rows, so the union's k-th
        // best is no worse -- close to the true k-th best once the lists fill, where
        // the min over lists of their KP-th best is far looser.  Recomputed only
        // when this list's best improves (rare).
        const int list_id = slice * kSplits + split;
        const int n_lists = (n_slices + (PAIR && a.n_spare ? 1 : 0)) * kSplits;
        const int n_pub = n_lists < kMinSlots ? n_lists : kMinSlots;
        const bool pub_min = share && a.list_min != nullptr && list_id < kMinSlots && n_pub >= a.k;
        // the k-th smallest published minimum is folded into a.bound by every list
        // at tiles 1, 2, 4, ... and then every 256th (SIMT-parallel over lanes)
        const uint32_t hit_bits = MODE == kThreshold ? score_bits<F>(a.threshold) : 0u;
        // XOR, formed before any compare so every mode ranks and stores Hamming
        // distances: mxf4 -- the MMA already holds popc(r) - 2 popc(r & q) (signed
        // unknown operand, unpack_f4_xor) and the epilogue adds popc(q), stored as
        // fp32 bits (one exact FADD per value); i8 -- the MMA counts shared ones and
        // popc(r) + popc(q) - 2 popc(r & q) is formed from the known rows' popcounts
        const bool xor_op = a.op == FASTID_OP_XOR;
        const uint32_t pq = xor_op && q_ok ? a.query_popc[q] : 0u;
        uint32_t t_empty_leader[kAccBufs] = {};
        if (PAIR) {
#pragma unroll
            for (int i = 0; i < kAccBufs; ++i) t_empty_leader[i] = ptx::mapa(&t_empty[i], 0);
        }
        for (int64_t i = 0; i < t_count; ++i, ++local) {
            const int64_t t = tile_of(i);
            const int acc = local % kAccBufs;
            // the shared bound is read before the wait so its latency hides behind it
            const uint32_t shared_bound = share ? __ldcg(a.bound + q) : 0xFFFFFFFFu;
            if (experiment(a, 4096))
                ptx::mbar_wait(&t_full[acc], (uint32_t)(local / kAccBufs) & 1u);
            else
                ptx::mbar_wait_sleep(&t_full[acc], (uint32_t)(local / kAccBufs) & 1u);
            const bool tr = trace_buf(a) && blockIdx.x == 0 && local < a.trace_tiles && lane == 0;
            if (tr) trace_buf(a)[local * kTrSlots + kTrEpi0 + ew] = clock64();
            if (pub_min && (local & (local - 1)) == 0 || (pub_min && (local & 255) == 0)) {
                const uint32_t kb = kth_smallest_published<KP>(a.list_min + (int64_t)q * kMinSlots, a.k);
                if (kb != 0xFFFFFFFFu) {
                    atomicMin(a.bound + q, kb + 1u);
                    if (kb + 1u < thr_eff) thr_eff = kb + 1u;
                }
            }
            if (shared_bound < thr_eff) thr_eff = shared_bound;
            ptx::tc_fence_after();
            const int64_t r0 = t * BN + split * kCols;
            const int64_t rows_left = a.n_refs - r0;
            const int rl = !q_ok ? 0 : (rows_left >= kCols ? kCols : (rows_left > 0 ? (int)rows_left : 0));
            const bool full = rl == kCols;
            const uint32_t col_base = (uint32_t)(acc * BN + split * kCols);
            auto to_xor = [&](uint32_t(&v)[kBatch], int b0) {
                if constexpr (F == FASTID_TENSOR_F4) {
#pragma unroll
                    for (int c = 0; c < kBatch; ++c) v[c] = __float_as_uint(__uint_as_float(v[c]) + __uint_as_float(pq));
                    return;
                }
                // the batch's 32 row popcounts: warp-uniform 16-byte loads (the buffer is
                // padded past n_refs to whole tiles; padding columns are discarded)
                const uint4* p4 = reinterpret_cast<const uint4*>(a.ref_popc + r0 + b0);
#pragma unroll
                for (int c4 = 0; c4 < kBatch / 4; ++c4) {
                    const uint4 p = __ldg(p4 + c4);
                    const uint32_t pc[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int c = c4 * 4 + i;
                        v[c] = score_bits<F>(pc[i] + pq - 2u * decode_exact<F>(v[c]));
                    }
                }
            };
            // per-batch processing of up to 32 columns already in registers
            auto process = [&](uint32_t(&v)[kBatch], int b0, int nb) {
                const int left = rl - b0;
                if constexpr (F == FASTID_TENSOR_F4 && MODE != kFull) {
                    if (xor_op) {
                        // popc(q) is one constant per lane (unknown): the batch's minimum
                        // decides in the raw domain (fp32 min, the same cost as the integer
                        // min of AND-NOT) and only a batch that can insert or hit pays for
                        // the per-value FADD (warp-uniform skip)
                        float mn = __uint_as_float(v[0]);
#pragma unroll
                        for (int c = 1; c < kBatch; ++c) mn = fminf(mn, __uint_as_float(v[c]));
                        const uint32_t mb = __float_as_uint(mn + __uint_as_float(pq));
                        const bool need = left > 0 && (MODE == kTopK ? mb < thr_eff : mb <= hit_bits);
                        if (!__any_sync(0xffffffffu, need)) return;
                        to_xor(v, b0);
                    }
                }
                const uint32_t valid = full || left >= kBatch ? (nb == 32 ? 0xFFFFFFFFu : (1u << nb) - 1u)
                                                              : (left <= 0 ? 0u : (1u << left) - 1u);
                const int64_t rc = r0 + b0;
                if (MODE == kFull) {
#pragma unroll
                    for (int c = 0; c < kBatch; ++c)
                        if ((valid >> c) & 1u) a.out[(rc + c) * a.ld_out + q] = decode_fast<F>(v[c]);
                    return;
                }
                if (valid != 0xFFFFFFFFu) {
#pragma unroll
                    for (int c = 0; c < kBatch; ++c)
                        if (!((valid >> c) & 1u)) v[c] = 0xFFFFFFFFu;
                }
                const uint32_t mn = min32(v);
                if (MODE == kTopK) {
                    if (mn < thr_eff && !experiment(a, 16)) {
                        uint32_t cand = 0;
#pragma unroll
                        for (int c = 0; c < kBatch; ++c) cand |= (v[c] < thr_eff ? 1u : 0u) << c;
                        // rare: one insertion per loop trip, value picked by a select tree
                        while (cand) {
                            const int c = __ffs(cand) - 1;
                            cand &= cand - 1;
                            const uint32_t vc = pick32(v, c);
                            if (vc < thr_eff) {
                                const bool new_best = vc < top.s[0];
                                top.insert_last(vc, (uint32_t)(rc + c));  // raw bits; rows ascend
                                if (pub_min && new_best) __stcg(a.list_min + (int64_t)q * kMinSlots + list_id, vc);
                                if (experiment(a, 32) && trace_buf(a) && local < a.trace_tiles)  // insertion census
                                    atomicAdd((unsigned long long*)&trace_buf(a)[(int64_t)a.trace_tiles * kTrSlots + local], 1ull);
                                const uint32_t kth = top.s[KP - 1];
                                thr_bits = kth < cap_bits ? kth : cap_bits;
                                if (thr_bits < thr_eff) thr_eff = thr_bits;
                                // (at or above the bound read this tile the atomic changes nothing)
                                if (share && kth != kEmptyScore && kth + 1u < shared_bound) atomicMin(a.bound + q, kth + 1u);
                            }
                        }
                    }
                } else {
                    uint32_t hit = 0;
                    if (mn <= hit_bits) {
#pragma unroll
                        for (int c = 0; c < kBatch; ++c) hit |= (v[c] <= hit_bits ? 1u : 0u) << c;
                    }
                    if (__any_sync(0xffffffffu, hit != 0)) {
                        uint32_t all = __reduce_or_sync(0xffffffffu, hit);
                        while (all) {  // warp-uniform walk over columns with a hit in any lane
                            const int c = __ffs(all) - 1;
                            all &= all - 1;
                            emit_hits(a, (hit >> c) & 1u, (uint32_t)q, rc + c, decode_exact<F>(pick32(v, c)));
                        }
                    }
                }
            };
            auto release = [&]() {
                // this warp's columns are all in registers: release the accumulator
                ptx::tc_fence_before();
                if (PAIR) {
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive_cluster(t_empty_leader[acc]);
                } else {
                    ptx::mbar_arrive(&t_empty[acc]);
                }
                if (tr) trace_buf(a)[local * kTrSlots + kTrRel0 + ew] = clock64();
            };
            const uint32_t ta0 = lane_base + col_base;
            if constexpr (kPreload) {
                // every column of this warp's split in one round of loads, one wait,
                // the accumulator released at once, then the compare work
                uint32_t v[kPreBatches][kBatch];
                if (!experiment(a, 1)) {
#pragma unroll
                    for (int b = 0; b < kPreBatches; ++b) {
                        const int nb = kCols - b * kBatch < kBatch ? kCols - b * kBatch : kBatch;
                        const uint32_t ta = ta0 + (uint32_t)(b * kBatch);
                        if (nb == 32) {
                            ptx::tmem_ld32(ta, v[b]);
                        } else {
                            int o = 0;
                            if (nb - o >= 16) {
                                ptx::tmem_ld16(ta, *reinterpret_cast<uint32_t(*)[16]>(&v[b][0]));
                                o = 16;
                            }
                            if (nb - o >= 8) {
                                ptx::tmem_ld8(ta + (uint32_t)o, &v[b][o]);
                                o += 8;
                            }
                            if (nb - o >= 8) ptx::tmem_ld8(ta + (uint32_t)o, &v[b][o]);
                        }
                    }
                    ptx::tmem_wait_ld();
                } else {
#pragma unroll
                    for (int b = 0; b < kPreBatches; ++b)
#pragma unroll
                        for (int c = 0; c < kBatch; ++c) v[b][c] = 0xFFFFFFFFu;
                }
                if (tr && !experiment(a, 8)) trace_buf(a)[local * kTrSlots + kTrB0Loaded + ew] = clock64();
                release();
                if (xor_op && (MODE == kFull || F != FASTID_TENSOR_F4)) {
#pragma unroll
                    for (int b = 0; b < kPreBatches; ++b) to_xor(v[b], b * kBatch);
                }
                if (PAIR && MODE == kFull && a.tma_out == 2) {
                    // full matrix, wide: the 4 lane-quadrant warps of this column split fill
                    // one [kCols known rows][128 unknowns] block (512-B output rows) and one
                    // of them issues the TMA tensor store (named barrier per split)
                    uint32_t* stage = reinterpret_cast<uint32_t*>(smem + lay.off_out) + split * kCols * kM;
                    const bool issuer = quad == 0 && lane == 0;
                    if (issuer) ptx::bulk_wait_read0();  // the previous store has read the block
                    ptx::named_bar_sync(1 + split, 128);
#pragma unroll
                    for (int b = 0; b < kPreBatches; ++b)
#pragma unroll
                        for (int c = 0; c < kBatch; ++c)
                            if (b * kBatch + c < kCols)
                                stage[(b * kBatch + c) * kM + quad * 32 + lane] = decode_fast<F>(v[b][c]);
                    ptx::fence_proxy_async_smem();
                    ptx::named_bar_sync(1 + split, 128);
                    if (issuer) {
                        ptx::tma_store_2d(&omap, stage, (int)q0s, (int)r0);
                        ptx::bulk_commit();
                    }
                    continue;
                }
                if (PAIR && MODE == kFull && a.tma_out) {
                    // full matrix: transpose through this warp's staging block and let a
                    // TMA tensor store write the [kCols known rows][32 unknowns] tile
                    // (out-of-range rows / unknowns are clipped by the TMA unit)
                    uint32_t* stage = reinterpret_cast<uint32_t*>(smem + lay.off_out) + ew * kCols * 32;
                    if (lane == 0) ptx::bulk_wait_read0();  // the previous store has read the block
                    __syncwarp();
#pragma unroll
                    for (int b = 0; b < kPreBatches; ++b)
#pragma unroll
                        for (int c = 0; c < kBatch; ++c)
                            if (b * kBatch + c < kCols) stage[(b * kBatch + c) * 32 + lane] = decode_fast<F>(v[b][c]);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_2d(&omap, stage, (int)(q0s + quad * 32), (int)r0);
                        ptx::bulk_commit();
                    }
                    continue;
                }
#pragma unroll
                for (int b = 0; b < kPreBatches; ++b) {
                    const int nb = kCols - b * kBatch < kBatch ? kCols - b * kBatch : kBatch;
                    process(v[b], b * kBatch, nb);
                }
                if (tr && !experiment(a, 8)) trace_buf(a)[local * kTrSlots + kTrB0Done + ew] = clock64();
                continue;
            } else {
#pragma unroll
            for (int b0 = 0; b0 < kCols; b0 += kBatch) {
                if (tr && b0 == kBatch && !experiment(a, 8)) trace_buf(a)[local * kTrSlots + kTrB0Done + ew] = clock64();
                const int nb = kCols - b0 < kBatch ? kCols - b0 : kBatch;  // multiple of 8, warp-uniform
                uint32_t v[kBatch];
                if (!experiment(a, 1)) {
                    // widest loads that fit (x32 moves ~40% more TMEM bytes/clk than x8)
                    const uint32_t ta = ta0 + (uint32_t)b0;
                    if (nb == 32) {
                        ptx::tmem_ld32(ta, v);
                    } else {
                        int o = 0;
                        if (nb - o >= 16) {
                            ptx::tmem_ld16(ta, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                            o = 16;
                        }
                        if (nb - o >= 8) {
                            ptx::tmem_ld8(ta + (uint32_t)o, &v[o]);
                            o += 8;
                        }
                        if (nb - o >= 8) ptx::tmem_ld8(ta + (uint32_t)o, &v[o]);
                    }
                    ptx::tmem_wait_ld();
                } else {
#pragma unroll
                    for (int c = 0; c < kBatch; ++c) v[c] = 0xFFFFFFFFu;
                }
                if (tr && b0 == 0 && !experiment(a, 8)) trace_buf(a)[local * kTrSlots + kTrB0Loaded + ew] = clock64();
                if (b0 + kBatch >= kCols) release();
                if (xor_op && (MODE == kFull || F != FASTID_TENSOR_F4)) to_xor(v, b0);
                process(v, b0, nb);
            }
            }
        }
        if (PAIR && MODE == kFull && a.tma_out && lane == 0) ptx::bulk_wait_all();  // stores done before exit
        if (MODE == kTopK && q_ok) {
#pragma unroll
            for (int i = 0; i < KP; ++i)
                if (top.s[i] != kEmptyScore) top.s[i] = decode_exact<F>(top.s[i]);
            const int64_t off = (((int64_t)slice * kMaxSplits + split) * a.n_queries + q) * KP;
            top.store(a.part_scores + off, a.part_index + off, a.ref_base);
        }
        if (MODE == kTopK && q_ok && split == 0) {
            // unused split slots of this slice hold empty lists (the merge skips them)
            for (int s2 = kSplits; s2 < kMaxSplits; ++s2) {
                const int64_t off2 = (((int64_t)slice * kMaxSplits + s2) * a.n_queries + q) * KP;
                TopList<KP> empty;
                empty.clear();
                empty.store(a.part_scores + off2, a.part_index + off2, a.ref_base);
            }
        }
        }  // segments
        }
    }

    if (cta_trace) trace_buf(a)[blockIdx.x * 4 + 2] = (long long)ptx::globaltimer();
    ptx::tc_fence_before();
    if (PAIR)
        ptx::cluster_sync();  // the leader's MMAs and the peer's remote arrivals are all done
    else
        __syncthreads();
    if (warp == kMmaWarp) {
        ptx::tc_fence_after();
        if (PAIR)
            ptx::tmem_dealloc_pair(tmem, Fmt<F>::kTmemCols);
        else
            ptx::tmem_dealloc(tmem, Fmt<F>::kTmemCols);
    }
    if (cta_trace) trace_buf(a)[blockIdx.x * 4 + 3] = (long long)ptx::globaltimer();
}

// ---- host side -------------------------------------------------------------

// One mutex per (device, stream), held by launch_one_impl from scratch
// acquisition until every kernel of the launch is enqueued.  Two host threads
// sharing a stream (torch's default stream, say; ctypes drops the GIL) then
// enqueue whole launches one after the other, so stream order keeps one
// launch's streamed-A operand, progress counters and side-stream fork/join
// from being overwritten or freed under the other's kernels.
std::mutex& stream_mutex(cudaStream_t stream) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, std::mutex> locks;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    return locks[std::make_pair(dev, stream)];  // std::map nodes never move
}

// Launch scratch (pair progress counters, streamed-A operand) kept per
// (device, stream) and grown on demand: stream-ordered reuse needs no
// per-launch cudaMallocAsync, which costs ~250 us when the pool trims.
// Callers hold stream_mutex(stream).
void* launch_scratch(int which, size_t bytes, cudaStream_t stream) {
    static std::mutex mu;
    static std::map<std::tuple<int, cudaStream_t, int>, std::pair<void*, size_t>> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    auto& slot = cache[std::make_tuple(dev, stream, which)];
    if (slot.second < bytes) {
        if (slot.first) {
            cudaStreamSynchronize(stream);  // the old buffer may still be in use on this stream
            cudaFree(slot.first);
        }
        slot = {nullptr, 0};
        void* p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
        slot = {p, bytes};
    }
    return slot.first;
}

// A side stream (+ fork/join events) per (device, stream) for the spare-pair grid.
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream* side_stream(cudaStream_t stream) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, SideStream> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    SideStream& ss = cache[std::make_pair(dev, stream)];
    if (!ss.s) {
        if (cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess)
            return nullptr;
    }
    return &ss;
}

// Debug flag 128: host-side phase timings of a launch, printed to stderr.
struct HostClock {
    bool on;
    std::chrono::steady_clock::time_point t;
    explicit HostClock(bool on_) : on(on_), t(std::chrono::steady_clock::now()) {}
    void mark(const char* what) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        fprintf(stderr, "[fastid host] %-24s %8.1f us\n", what,
                std::chrono::duration<double, std::micro>(n - t).count());
        t = n;
    }
};

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

// Spare CTA pairs left over by (unknown groups x slices) on this GPU: each
// takes the tail tiles of groups / n_spare groups.  With S slices, a spare
// handles `per` groups: equal run times need tail = tiles / (1 + S * per).
struct SparePlan {
    int n_spare = 0;
    int64_t t_main = 0;
};
inline SparePlan spare_plan(int64_t n_tiles, int64_t groups, int slices, bool disabled) {
    SparePlan p;
    p.t_main = n_tiles;
    const int64_t pairs = num_sms() / 2;
    int64_t spare = pairs - groups * slices;
    if (disabled || spare <= 0 || groups <= 0 || n_tiles < 16 * (slices + 1)) return p;
    while (spare > 1 && groups % spare) --spare;  // a divisor of the group count
    const int64_t per = groups / spare;
    // equal tile counts per pair, scaled by FASTID_SPARE_SHARE percent (tuning knob:
    // a spare pair re-reads its tail once per group it serves)
    const int share = [] {  // read per launch (scheduling only: the result is the same)
        const char* e = getenv("FASTID_SPARE_SHARE");
        const int v = e ? atoi(e) : 100;
        return v > 0 && v <= 200 ? v : 100;
    }();
    const int64_t tail = n_tiles * share / (100 * (1 + slices * per));
    if (tail < 1) return p;
    p.n_spare = (int)spare;
    p.t_main = n_tiles - tail;
    return p;
}

// The spare grid assumes the SMs the regular grid leaves free are idle; on a
// GPU shared with other work it could start late and lengthen the step, so
// FASTID_NO_SPARE_PAIRS=1 (or the database option FASTID_OPT_NO_SPARE_PAIRS) turns it off.
inline bool spares_disabled(const CompareArgs& a) {
    static const bool env = [] {
        const char* e = getenv("FASTID_NO_SPARE_PAIRS");
        return e && *e && *e != '0';
    }();
    return env || (a.options & FASTID_OPT_NO_SPARE_PAIRS);
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

// Streamed-A operand: complemented, unpacked unknown rows laid out stage by
// stage ([group][stage][core matrices]) so each stage is one bulk copy.
template <int F>
__global__ void prep_a_kernel(CompareArgs a, int n_groups, int n_kst, uint8_t* __restrict__ out) {
    [[maybe_unused]] constexpr int CPW = Fmt<F>::kCoresPerWord;
    constexpr int AB = Layout<F>::kAStageBytes;
    const int64_t total = (int64_t)n_groups * n_kst * kM;
    const int row_words = (int)(a.stride / 4);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int row = (int)(t % kM);
        const int64_t gs = t / kM;  // group * n_kst + stage
        const int ks = (int)(gs % n_kst);
        const int64_t q = (gs / n_kst) * kM + row;
        const bool real = q < a.n_queries;
        uint8_t* dst = out + gs * AB;
#pragma unroll
        for (int w = 0; w < kWordsPerStage; ++w) {
            const int word = ks * kWordsPerStage + w;
            uint32_t x = 0;
            if (real && word < row_words) {
                x = reinterpret_cast<const uint32_t*>(a.queries + q * a.stride)[word];
                if (a.op == FASTID_OP_ANDNOT) x = ~x;
            }
            if (F == FASTID_TENSOR_F4) {
                *reinterpret_cast<uint4*>(dst + core_off(row, w, kM)) =
                    unpack_a_f4(x, a.image && uniform_image(a), a.op == FASTID_OP_XOR, real && word < row_words);
            } else {
                uint4 lo, hi;
                unpack_i8<false>(x, lo, hi);
                *reinterpret_cast<uint4*>(dst + core_off(row, 2 * w, kM)) = lo;
                *reinterpret_cast<uint4*>(dst + core_off(row, 2 * w + 1, kM)) = hi;
            }
        }
    }
}

template <int F>
bool use_stream_a(int64_t stride) { return !Layout<F>(stride, false).fits(); }

// Tensor map over the mxf4 image viewed as rows of 128 B: one box = one half
// stage (BN/2 known rows x 256 loci in the UMMA layout, contiguous).
template <int F>
int make_image_map(CUtensorMap* map, const CompareArgs& a) {
    auto fn = encode_fn();
    if (!fn) FASTID_FAIL(FASTID_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    const Layout<F> lay(a.stride, false, true);
    const int64_t bytes = ceil_div(a.n_refs, Fmt<F>::BN) * lay.n_kst * Layout<F>::kUnpackedStageBytes;
    cuuint64_t dims[2] = {kImgRowBytes / 8, (cuuint64_t)(bytes / kImgRowBytes)};
    cuuint64_t strides[1] = {kImgRowBytes};
    cuuint32_t box[2] = {kImgRowBytes / 8, (cuuint32_t)(Layout<F>::kUnpackedStageBytes / 2 / kImgRowBytes)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, (void*)a.image, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) FASTID_FAIL(FASTID_E_CUDA, "cuTensorMapEncodeTiled (image) failed (%d)", (int)r);
    return FASTID_OK;
}

// Tensor map over the u32 full-matrix output [n_refs][ld_out] (inner dim =
// unknowns): one box = one epilogue warp's [cols][32] block.  Needs 16-byte
// alignment of the base and the row pitch.
int make_out_map(CUtensorMap* map, const CompareArgs& a, int box_cols, int box_unknowns) {
    auto fn = encode_fn();
    if (!fn) FASTID_FAIL(FASTID_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)a.n_queries, (cuuint64_t)a.n_refs};
    cuuint64_t strides[1] = {(cuuint64_t)a.ld_out * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_unknowns, (cuuint32_t)box_cols};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, (void*)a.out, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) FASTID_FAIL(FASTID_E_CUDA, "cuTensorMapEncodeTiled (output) failed (%d)", (int)r);
    return FASTID_OK;
}

// Tensor map over the streamed-A operand ([group][stage][AB bytes], rows of
// 128 B): one box = one stage of one 128-unknown group.
template <int F>
int make_a_map(CUtensorMap* map, const void* a_global, int64_t groups, int n_kst) {
    auto fn = encode_fn();
    if (!fn) FASTID_FAIL(FASTID_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    constexpr int AB = Layout<F>::kAStageBytes;
    cuuint64_t dims[2] = {128, (cuuint64_t)(groups * n_kst * (AB / 128))};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {128, (cuuint32_t)(AB / 128)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)a_global, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) FASTID_FAIL(FASTID_E_CUDA, "cuTensorMapEncodeTiled (A) failed (%d)", (int)r);
    return FASTID_OK;
}

template <int F, int MODE, int KP, bool SA, bool IMG, bool PAIR>
int launch_one_impl(const CompareArgs& a_in, int n_slices, cudaStream_t stream) {
    HostClock hc(experiment(a_in, 128));
    std::lock_guard<std::mutex> launch_lock(stream_mutex(stream));
    CompareArgs a = a_in;
    // tuning knobs of the dual-tile pair kernel's ring split (scheduling only: the
    // result is identical for every value); FASTID_DUAL_SA = A ring depth
    a.dual_sa = 0;
    if (const char* e = getenv("FASTID_DUAL_SA")) a.dual_sa = atoi(e);
    CUtensorMap omap;
    memset(&omap, 0, sizeof(omap));
    a.tma_out = 0;
    // TMA tensor stores clip out-of-range unknowns only to 16-byte granules (measured:
    // n_queries = 150 with a wider row pitch wrote columns 150-151), so they are used
    // only when every granule they touch belongs to the matrix: n_queries % 4 == 0
    if (PAIR && MODE == kFull && a.n_queries > 0 && a.n_queries % 4 == 0 && ((uintptr_t)a.out & 15) == 0 &&
        (a.ld_out * 4) % 16 == 0 &&
        !(a.options & FASTID_OPT_NO_TMA_STORE) && Layout<F>(a.stride, SA, IMG, PAIR, out_stage_bytes<F, MODE, IMG, PAIR>()).fits()) {
        // wide blocks (128 unknowns = 512-B rows) unless FASTID_OPT_NARROW_TMA_STORE asks for per-warp ones
        const bool wide = !(a.options & FASTID_OPT_NARROW_TMA_STORE);
        if (int rc = make_out_map(&omap, a, Fmt<F>::BN / (Roles<F, IMG>::kEpiWarps / 4), wide ? kM : 32)) return rc;
        a.tma_out = wide ? 2 : 1;
    }
    CUtensorMap map;
    if (PAIR) {
        if (int rc = make_image_map<F>(&map, a)) return rc;
    } else {
        if (int rc = make_known_map(&map, a, Fmt<F>::BN)) return rc;
    }
    hc.mark("tensor map");
    const Layout<F> lay(a.stride, SA, IMG, PAIR, a.tma_out ? out_stage_bytes<F, MODE, IMG, PAIR>() : 0, a.dual_sa);
    if (!lay.fits()) FASTID_FAIL(FASTID_E_UNSUPPORTED, "tile needs %d bytes of shared memory", lay.total);
    auto kern = tensor_kernel<F, MODE, KP, SA, IMG, PAIR, false>;
    FASTID_CUDA(ensure_dynamic_smem((const void*)kern, lay.total));
    hc.mark("set attribute");
    // pairs cover unknowns in groups of 256: prepare A for both halves of the last pair
    const int64_t groups = PAIR ? 2 * ceil_div(a.n_queries, 2 * kM) : ceil_div(a.n_queries, kM);
    const int64_t tiles = ceil_div(a.n_refs, Fmt<F>::BN);
    uint8_t* a_global = nullptr;
    CUtensorMap amap;
    memset(&amap, 0, sizeof(amap));
    if (a.op == FASTID_OP_XOR) {
        constexpr bool kFloat = F == FASTID_TENSOR_F4;
        if (kFloat) a.ref_popc = nullptr;  // mxf4 needs only the unknowns' popcounts
        if (!kFloat && !a.ref_popc) {
            const size_t n = (size_t)popcount_entries(a.n_refs);
            auto* pr = (uint32_t*)launch_scratch(2, n * sizeof(uint32_t), stream);
            if (!pr) FASTID_FAIL(FASTID_E_NOMEM, "cannot allocate %zu row popcounts", n);
            if (int rc = launch_row_popcount(a.refs, a.n_refs, (int64_t)n, a.stride, kFloat, pr, stream)) return rc;
            a.ref_popc = pr;
        }
        auto* pq = (uint32_t*)launch_scratch(3, (size_t)a.n_queries * sizeof(uint32_t), stream);
        if (!pq) FASTID_FAIL(FASTID_E_NOMEM, "cannot allocate %lld row popcounts", (long long)a.n_queries);
        if (int rc = launch_row_popcount(a.queries, a.n_queries, a.n_queries, a.stride, kFloat, pq, stream))
            return rc;
        a.query_popc = pq;
    }
    if (SA) {
        const size_t bytes = (size_t)groups * lay.n_kst * Layout<F>::kAStageBytes;
        a_global = (uint8_t*)launch_scratch(0, bytes, stream);
        if (!a_global) FASTID_FAIL(FASTID_E_NOMEM, "cannot allocate %zu bytes of streamed-A operand", bytes);
        const int64_t work = groups * lay.n_kst * kM;
        prep_a_kernel<F><<<(unsigned)std::min<int64_t>(ceil_div(work, 256), num_sms() * 16), 256, 0, stream>>>(
            a, (int)groups, lay.n_kst, a_global);
        FASTID_LAUNCHED("prep_a_kernel");
        if (PAIR) {
            if (int rc = make_a_map<F>(&amap, a_global, groups, lay.n_kst)) return rc;
        }
    }
    if (PAIR) {
        const int64_t pgroups = ceil_div(a.n_queries, 2 * kM);
        // The full matrix is HBM-write-bound: a spare grid on the 4 leftover SMs only
        // contends for write bandwidth (C2: 1.64 ms with it, 1.44 ms without,
        // tools/opt_ab.py), so spare pairs serve the top-k / threshold epilogues only.
        const SparePlan sp = spare_plan(tiles, pgroups, n_slices, spares_disabled(a) || MODE == kFull);
        const int64_t regular = pgroups * n_slices;
        const int64_t pairs = regular;
        CompareArgs ap = a;
        ap.n_groups = (int)pgroups;
        ap.n_spare = sp.n_spare;
        ap.t_main = sp.t_main;
        ap.progress = nullptr;
        {
            // Resident unknowns (short tiles): a 40-tile window (on-box A/B at 1024 loci: C3
            // 10.2 ms at 40 tiles vs 12.4 at 20 and 10.8 at 80; 512 unknowns 3.1 ms at 40 vs
            // 4.1 at the 13 tiles of the byte budget).  Dual-tile pairs (long tiles): the
            // byte budget (C4: 2 tiles, 16.1 ms vs 17.9 at 3 and 19.0 at 6).
            // More than 8 unknown groups (> 2048 unknowns) pace more peers each, and the
            // slowest of them sets the pace: twice the window, within the byte budget
            // (8192 unknowns: 39.1 ms at 80 tiles vs 47.5 at 40; 4096: flat; tools/nq_scan.py).
            const int64_t window = kDriftWindowBytes / ((int64_t)n_slices * lay.n_kst * Layout<F>::kUnpackedStageBytes);
            const int64_t resident = pgroups > 8 ? std::max<int64_t>(kDriftTilesMax, std::min<int64_t>(2 * kDriftTilesMax, window))
                                                 : kDriftTilesMax;
            ap.drift_tiles = SA ? (int)std::min<int64_t>(kDriftTilesMax, std::max<int64_t>(2, window)) : (int)resident;
            // L2 prefetch of the known-tile stream: off by default (it cost C3 / C4 power and
            // clock for ~1% on one unknown group); FASTID_L2_PREFETCH=1 turns it on
            ap.l2_prefetch = 0;
            if (const char* e = getenv("FASTID_L2_PREFETCH")) ap.l2_prefetch = atoi(e) != 0;
            ap.dual_lag = -1;  // FASTID_DUAL_LAG: stages the second tile of a dual step lags
            if (const char* e = getenv("FASTID_DUAL_LAG")) ap.dual_lag = atoi(e);
            // FASTID_DRIFT_TILES: the drift window in tiles (scheduling only)
            if (const char* e = getenv("FASTID_DRIFT_TILES")) ap.drift_tiles = std::max(1, atoi(e));
            // checks at least 16 stages apart: a check consumes the peers' counters loaded at
            // the previous one, and a shorter gap stalls the producer on that load
            ap.drift_every = std::max(std::max(1, ap.drift_tiles / 4), (int)ceil_div(16, lay.n_kst));
        }
        // drift control only among co-resident pairs, and only for runs long enough to
        // drift (a small comparison skips the counters' memset launch)
        if (2 * (pairs + sp.n_spare) <= num_sms() && tiles >= 64 * (int64_t)n_slices) {
            ap.progress = (int*)launch_scratch(1, (size_t)regular * sizeof(int), stream);
            if (!ap.progress) FASTID_FAIL(FASTID_E_NOMEM, "cannot allocate the pair progress counters");
            FASTID_CUDA(cudaMemsetAsync(ap.progress, 0, (size_t)regular * sizeof(int), stream));
        }
        hc.mark("progress alloc+memset");
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)(2 * pairs));
        cfg.blockDim = dim3(Roles<F, IMG>::kThreads);
        cfg.dynamicSmemBytes = (size_t)lay.total;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        SideStream* side = sp.n_spare ? side_stream(stream) : nullptr;
        if (sp.n_spare) {
            if (!side) FASTID_FAIL(FASTID_E_CUDA, "cannot create the spare-pair stream");
            FASTID_CUDA(cudaEventRecord(side->fork, stream));
        }
        FASTID_CUDA(cudaLaunchKernelEx(&cfg, kern, map, omap, amap, ap, (const uint8_t*)a_global, tiles, n_slices));
        hc.mark("cluster launch");
        if constexpr (PAIR) if (sp.n_spare) {
            // The spare pairs: a second grid on a side stream, launched after the regular
            // one so it lands on the SMs that grid leaves free, joined before anything
            // that follows on `stream` (the merge).  Its own instantiation keeps the
            // regular kernel free of the segment loops' registers.
            auto skern = tensor_kernel<F, MODE, KP, SA, IMG, PAIR, true>;
            FASTID_CUDA(ensure_dynamic_smem((const void*)skern, lay.total));
            CompareArgs as = ap;
            as.progress = nullptr;
            as.trace = nullptr;
            cudaLaunchConfig_t scfg = cfg;
            scfg.gridDim = dim3((unsigned)(2 * sp.n_spare));
            scfg.stream = side->s;
            FASTID_CUDA(cudaStreamWaitEvent(side->s, side->fork, 0));
            FASTID_CUDA(cudaLaunchKernelEx(&scfg, skern, map, omap, amap, as, (const uint8_t*)a_global, tiles, n_slices));
            note_launch();
            FASTID_CUDA(cudaEventRecord(side->join, side->s));
            FASTID_CUDA(cudaStreamWaitEvent(stream, side->join, 0));
        }
    } else {
        kern<<<(unsigned)(groups * n_slices), Roles<F, IMG>::kThreads, lay.total, stream>>>(map, omap, amap, a,
                                                                                         a_global, tiles, n_slices);
    }
    FASTID_LAUNCHED("tensor_kernel");
    return FASTID_OK;
}

// CTA pairs run the prepared mxf4 image, with a resident unknown tile when it
// fits (L <= 2048) and a streamed one otherwise.
template <int F>
bool use_pair(const CompareArgs& a) {
    return F == FASTID_TENSOR_F4 && a.image != nullptr && !(a.options & FASTID_OPT_NO_CTA_PAIRS) &&
           (Layout<F>(a.stride, false, true, true).fits() || Layout<F>(a.stride, true, true, true).fits());
}

template <int F>
int pair_slices_for(int64_t n_refs, int64_t n_queries) {
    const int64_t pgroups = ceil_div(n_queries, 2 * kM);
    const int64_t tiles = ceil_div(n_refs, Fmt<F>::BN);
    int64_t s = (num_sms() / 2) / (pgroups > 0 ? pgroups : 1);
    if (s > tiles) s = tiles;
    if (s < 1) s = 1;
    return (int)s;
}

template <int F, int MODE, int KP>
int launch_one(const CompareArgs& a, int n_slices, cudaStream_t stream) {
    const bool img = a.image != nullptr;
    const bool sa = !Layout<F>(a.stride, false, img).fits();
    if (img) {
        if constexpr (F == FASTID_TENSOR_F4) {
            if (use_pair<F>(a)) {
                if (Layout<F>(a.stride, false, true, true).fits())
                    return launch_one_impl<F, MODE, KP, false, true, true>(a, n_slices, stream);
                return launch_one_impl<F, MODE, KP, true, true, true>(a, n_slices, stream);
            }
        }
        if (sa) return launch_one_impl<F, MODE, KP, true, true, false>(a, n_slices, stream);
        return launch_one_impl<F, MODE, KP, false, true, false>(a, n_slices, stream);
    }
    if (sa) return launch_one_impl<F, MODE, KP, true, false, false>(a, n_slices, stream);
    return launch_one_impl<F, MODE, KP, false, false, false>(a, n_slices, stream);
}

// Tensor image of a known panel: for every (tile, stage) the UMMA-layout B
// operand block the converters would produce, written once at database load.
template <int F>
__global__ void build_image_kernel(CompareArgs a, int64_t n_tiles, int n_kst, uint8_t* __restrict__ image) {
    constexpr int BN = Fmt<F>::BN;
    constexpr int CPW = Fmt<F>::kCoresPerWord;
    constexpr int UB = Layout<F>::kUnpackedStageBytes;
    const int64_t total = n_tiles * n_kst * 2 * BN;  // units: (tile, stage, row, 16-B half)
    const int64_t row_bytes = a.stride;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total; u += (int64_t)gridDim.x * blockDim.x) {
        const int unit = (int)(u % (2 * BN));
        const int64_t blk = u / (2 * BN);  // tile * n_kst + stage
        const int ks = (int)(blk % n_kst);
        const int64_t tile = blk / n_kst;
        const int row = unit >> 1;
        const int half = unit & 1;
        const int64_t r = tile * BN + row;
        const int64_t off = (int64_t)ks * kStageBytesPacked + half * 16;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r < a.n_refs && off < row_bytes) v = *reinterpret_cast<const uint4*>(a.refs + r * row_bytes + off);
        uint8_t* dst = image + blk * UB;
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
        const int col0 = half * 4 * CPW;
        // mxf4: pair layout -- rows [0, BN/2) then [BN/2, BN), each its own
        // K-major block of BN/2 rows (the half a CTA of a pair streams)
        const int hr = row >= BN / 2 ? 1 : 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (F == FASTID_TENSOR_F4) {
                *reinterpret_cast<uint4*>(dst + hr * (UB / 2) + core_off(row - hr * (BN / 2), col0 + i, BN / 2)) =
                    uniform_image(a) ? unpack_f4_uniform(wv[i]) : unpack_f4<true>(wv[i]);
            } else {
                uint4 lo, hi;
                unpack_i8<true>(wv[i], lo, hi);
                *reinterpret_cast<uint4*>(dst + core_off(row, col0 + 2 * i, BN)) = lo;
                *reinterpret_cast<uint4*>(dst + core_off(row, col0 + 2 * i + 1, BN)) = hi;
            }
        }
    }
}

template <int F>
size_t image_bytes_fmt(int64_t n_refs, int64_t stride) {
    const Layout<F> lay(stride, false, true);
    return (size_t)ceil_div(n_refs, Fmt<F>::BN) * lay.n_kst * Layout<F>::kUnpackedStageBytes;
}

template <int F>
int build_image_fmt(const CompareArgs& a, void* image, cudaStream_t stream) {
    const Layout<F> lay(a.stride, false, true);
    const int64_t tiles = ceil_div(a.n_refs, Fmt<F>::BN);
    const int64_t work = tiles * lay.n_kst * 2 * Fmt<F>::BN;
    if (work == 0) return FASTID_OK;
    build_image_kernel<F><<<(unsigned)std::min<int64_t>(ceil_div(work, 256), num_sms() * 32), 256, 0, stream>>>(
        a, tiles, lay.n_kst, (uint8_t*)image);
    FASTID_LAUNCHED("build_image_kernel");
    return FASTID_OK;
}

template <int F>
int launch_fmt(Mode mode, const CompareArgs& a, int* n_parts, cudaStream_t stream) {
    const int slices = use_pair<F>(a) ? pair_slices_for<F>(a.n_refs, a.n_queries) : slices_for<F>(a.n_refs, a.n_queries);
    if (mode == kFull) return launch_one<F, kFull, 1>(a, slices, stream);
    if (mode == kThreshold) return launch_one<F, kThreshold, 1>(a, slices, stream);
    // one partial list per (slice, epilogue column split), plus the spare pairs' slot
    *n_parts = kMaxSplits * slices;
    if (use_pair<F>(a) &&
        spare_plan(ceil_div(a.n_refs, Fmt<F>::BN), ceil_div(a.n_queries, 2 * kM), slices, spares_disabled(a)).n_spare)
        *n_parts += kMaxSplits;
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
    if (formulation == FASTID_TENSOR_I8)
        return Layout<FASTID_TENSOR_I8>(stride, false).fits() || Layout<FASTID_TENSOR_I8>(stride, true).fits();
    if (formulation == FASTID_TENSOR_F4)
        return Layout<FASTID_TENSOR_F4>(stride, false).fits() || Layout<FASTID_TENSOR_F4>(stride, true).fits();
    return 0;
}

size_t tensor_image_bytes(int64_t n_refs, int64_t bit_length, int formulation) {
    const int64_t stride = row_stride_bytes(bit_length);
    if (formulation == FASTID_TENSOR_I8) return image_bytes_fmt<FASTID_TENSOR_I8>(n_refs, stride);
    if (formulation == FASTID_TENSOR_F4) return image_bytes_fmt<FASTID_TENSOR_F4>(n_refs, stride);
    return 0;
}

int build_tensor_image(const CompareArgs& a, int formulation, void* image, cudaStream_t stream) {
    if (formulation == FASTID_TENSOR_I8) return build_image_fmt<FASTID_TENSOR_I8>(a, image, stream);
    if (formulation == FASTID_TENSOR_F4) return build_image_fmt<FASTID_TENSOR_F4>(a, image, stream);
    FASTID_FAIL(FASTID_E_INVALID, "no tensor image for formulation %d", formulation);
}

int tensor_parts(int64_t n_refs, int64_t n_queries, int formulation) {
    // an upper bound: the launch reports the partition it used
    if (formulation == FASTID_TENSOR_I8) return kMaxSplits * slices_for<FASTID_TENSOR_I8>(n_refs, n_queries);
    return kMaxSplits * std::max(slices_for<FASTID_TENSOR_F4>(n_refs, n_queries),
                                 pair_slices_for<FASTID_TENSOR_F4>(n_refs, n_queries) + 1);  // + spare slot
}

int launch_tensor(Mode mode, const CompareArgs& a, int formulation, int* n_parts, cudaStream_t stream) {
    if (formulation == FASTID_TENSOR_I8) return launch_fmt<FASTID_TENSOR_I8>(mode, a, n_parts, stream);
    if (formulation == FASTID_TENSOR_F4) return launch_fmt<FASTID_TENSOR_F4>(mode, a, n_parts, stream);
    FASTID_FAIL(FASTID_E_INVALID, "not a tensor formulation: %d", formulation);
}

}  // namespace fastid

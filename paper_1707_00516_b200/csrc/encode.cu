// Profile encoder: panel words / 0-1 bit matrices / genotype codes -> the
// aligned device row layout every comparison kernel reads.
//
// Layout: row r of a panel starts at
// r * stride bytes, stride = ceil(L / 128) * 16, and holds the panel's words
// in their native little-endian byte order followed by zero fill, so every row
// is 16-B aligned and a warp reading consecutive rows reads contiguous memory.
//
// Bit packing follows codec.pack (reference pkg/src/fastid/codec.py:118-127):
// bit i of a profile lives in word i // B at bit position B - 1 - (i % B).
#include "common.cuh"

namespace fastid {
namespace {

// One thread per 16-byte chunk of the destination.
__global__ void load_words_kernel(const uint8_t* __restrict__ src, int64_t rows, int64_t src_row_bytes,
                                  uint8_t* __restrict__ dst, int64_t dst_stride) {
    const int64_t chunks_per_row = dst_stride / 16;
    const int64_t total = rows * chunks_per_row;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / chunks_per_row;
        const int64_t c = t - r * chunks_per_row;
        const int64_t off = c * 16;
        uint32_t v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t b = off + 4 * i;
            v[i] = b < src_row_bytes ? *reinterpret_cast<const uint32_t*>(src + r * src_row_bytes + b) : 0u;
        }
        *reinterpret_cast<uint4*>(dst + r * dst_stride + off) = make_uint4(v[0], v[1], v[2], v[3]);
    }
}

// Bit j of profile r for the two input kinds.
struct BitMatrix {
    const uint8_t* bits;
    int64_t length;
    __device__ __forceinline__ uint32_t get(int64_t r, int64_t j) const {
        return bits[r * length + j] & 1u;
    }
};

struct GenotypeCodes {
    const uint8_t* codes;  // 0 = MM, 1 = Mm, 2 = mM, 3 = mm (codec.GENOTYPE_BITS, codec.py:22-27)
    int64_t n_loci;
    __device__ __forceinline__ uint32_t get(int64_t r, int64_t j) const {
        const uint32_t c = codes[r * n_loci + (j >> 1)];
        return (j & 1) ? (c & 1u) : ((c >> 1) & 1u);  // first allele slot, then second
    }
};

// One thread per 32-bit lane of the destination row.  For 64-bit words the
// little-endian low half of word w holds bits w*64+32..w*64+63, the high half
// bits w*64..w*64+31 (MSB-first inside the word).
template <class Src>
__global__ void pack_kernel(Src src, int64_t rows, int64_t bit_length, int word_bits, uint32_t* __restrict__ dst,
                            int64_t dst_stride) {
    const int64_t lanes_per_row = dst_stride / 4;
    const int64_t n_words = (bit_length + word_bits - 1) / word_bits;
    const int64_t used_lanes = n_words * (word_bits / 32);
    const int64_t total = rows * lanes_per_row;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / lanes_per_row;
        const int64_t c = t - r * lanes_per_row;
        uint32_t v = 0;
        if (c < used_lanes) {
            const int64_t first = word_bits == 64 ? (c >> 1) * 64 + ((c & 1) ? 0 : 32) : c * 32;
#pragma unroll 8
            for (int b = 0; b < 32; ++b) {
                const int64_t j = first + b;
                if (j < bit_length) v |= src.get(r, j) << (31 - b);
            }
        }
        dst[r * lanes_per_row + c] = v;
    }
}

int grid_for(int64_t work) {
    int64_t blocks = (work + 255) / 256;
    if (blocks > num_sms() * 32) blocks = num_sms() * 32;
    return (int)(blocks < 1 ? 1 : blocks);
}

int check_layout(int64_t rows, int64_t dst_stride, const void* dst) {
    if (rows < 0) FASTID_FAIL(FASTID_E_INVALID, "negative row count");
    if (dst_stride <= 0 || dst_stride % 16) FASTID_FAIL(FASTID_E_INVALID, "dst_stride must be a positive multiple of 16");
    if (rows && ((uintptr_t)dst & 15)) FASTID_FAIL(FASTID_E_INVALID, "dst must be 16-byte aligned");
    return FASTID_OK;
}

}  // namespace
}  // namespace fastid

using namespace fastid;

extern "C" int fastid_load_words(const void* src, int64_t rows, int64_t src_row_bytes, void* dst, int64_t dst_stride,
                                 void* stream) {
    if (int rc = check_layout(rows, dst_stride, dst)) return rc;
    if (src_row_bytes < 0 || src_row_bytes % 4 || src_row_bytes > dst_stride)
        FASTID_FAIL(FASTID_E_INVALID, "src_row_bytes must be a multiple of 4 and <= dst_stride");
    if (rows && ((uintptr_t)src & 3)) FASTID_FAIL(FASTID_E_INVALID, "src must be 4-byte aligned");
    if (rows == 0) return FASTID_OK;
    const int64_t work = rows * (dst_stride / 16);
    load_words_kernel<<<grid_for(work), 256, 0, (cudaStream_t)stream>>>(
        (const uint8_t*)src, rows, src_row_bytes, (uint8_t*)dst, dst_stride);
    FASTID_LAUNCHED("load_words_kernel");
    return FASTID_OK;
}

extern "C" int fastid_pack_bits(const uint8_t* bits, int64_t rows, int64_t bit_length, int word_bits, void* dst,
                                int64_t dst_stride, void* stream) {
    if (int rc = check_layout(rows, dst_stride, dst)) return rc;
    if (word_bits != 32 && word_bits != 64) FASTID_FAIL(FASTID_E_INVALID, "word_bits must be 32 or 64");
    if (bit_length <= 0) FASTID_FAIL(FASTID_E_INVALID, "bit_length must be positive");
    const int64_t n_words = (bit_length + word_bits - 1) / word_bits;
    if (n_words * (word_bits / 8) > dst_stride) FASTID_FAIL(FASTID_E_INVALID, "dst_stride too small for the packed row");
    if (rows == 0) return FASTID_OK;
    const int64_t work = rows * (dst_stride / 4);
    pack_kernel<BitMatrix><<<grid_for(work), 256, 0, (cudaStream_t)stream>>>(
        BitMatrix{bits, bit_length}, rows, bit_length, word_bits, (uint32_t*)dst, dst_stride);
    FASTID_LAUNCHED("pack_kernel<BitMatrix>");
    return FASTID_OK;
}

extern "C" int fastid_pack_genotypes(const uint8_t* codes, int64_t rows, int64_t n_loci, int word_bits, void* dst,
                                     int64_t dst_stride, void* stream) {
    if (int rc = check_layout(rows, dst_stride, dst)) return rc;
    if (word_bits != 32 && word_bits != 64) FASTID_FAIL(FASTID_E_INVALID, "word_bits must be 32 or 64");
    if (n_loci <= 0) FASTID_FAIL(FASTID_E_INVALID, "n_loci must be positive");
    const int64_t bit_length = 2 * n_loci;
    const int64_t n_words = (bit_length + word_bits - 1) / word_bits;
    if (n_words * (word_bits / 8) > dst_stride) FASTID_FAIL(FASTID_E_INVALID, "dst_stride too small for the packed row");
    if (rows == 0) return FASTID_OK;
    const int64_t work = rows * (dst_stride / 4);
    pack_kernel<GenotypeCodes><<<grid_for(work), 256, 0, (cudaStream_t)stream>>>(
        GenotypeCodes{codes, n_loci}, rows, bit_length, word_bits, (uint32_t*)dst, dst_stride);
    FASTID_LAUNCHED("pack_kernel<GenotypeCodes>");
    return FASTID_OK;
}

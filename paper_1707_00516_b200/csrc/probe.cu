// Pipe-peak probes: the measured roofline denominators for the two
// formulations.  Each runs one CTA per SM doing
// nothing but the formulation's inner instruction at its tile shape:
//   * tensor: back-to-back tcgen05.mma (M=128, N=BN, same kind as the
//     comparison kernel) on resident shared-memory operands, alternating two
//     TMEM accumulators, no epilogue;
//   * popc:   LOP3 (and-not) + POPC + IADD on register-resident words with 16
//     independent accumulators per thread.
// Work per launch is returned so the caller divides by CUDA-event time.
#include "common.cuh"
#include "tensor_ptx.cuh"

namespace fastid {
namespace {

// variant bit 0: accumulate every MMA into ONE accumulator (K-loop dependency)
// variant bit 2: walk distinct operand addresses (A: 32 K-chunks, B: 20 chunks) like the real kernel
// variant bit 1: warp 1 streams bulk copies (28 KB) from `src` into a 4-deep
//                shared-memory ring while the MMAs run (operand-fill traffic)
template <bool F4>
__global__ void __launch_bounds__(128, 1) mma_probe_kernel(int iters, uint32_t* sink, int variant,
                                                           const uint8_t* src, int64_t src_bytes) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t done;
    __shared__ __align__(8) uint64_t ring_full[4];
    __shared__ __align__(8) uint64_t ring_empty[4];
    constexpr int BN = F4 ? 224 : 128;
    const int warp = threadIdx.x >> 5;
    // zero operands: A 128 x 32 B x 32 chunks (128 KB region reused), B BN x 32 B x 20 chunks
    const bool walk = (variant & 4) != 0;
    const int a_chunks = walk ? 32 : 1, b_chunks = walk ? 10 : 1;
    for (int i = threadIdx.x; i < (walk ? 200 * 1024 : (128 + BN) * 32) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    ptx::fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        ptx::mbar_init(&done, 1);
        for (int i = 0; i < 4; ++i) {
            ptx::mbar_init(&ring_full[i], 1);
            ptx::mbar_init(&ring_empty[i], 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc(&tmem_slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (F4) {
        const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
        ptx::tmem_fill32(lb + 448, 0x7F7F7F7Fu);
        ptx::tmem_fill32(lb + 480, 0x7F7F7F7Fu);
        ptx::tmem_wait_st();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t a = ptx::smem_u32(smem);
        const uint32_t b = a + (walk ? 128 * 32 * 16 : 128 * 32);  // A region 64 KB when walking
        for (int i = 0; i < iters; ++i) {
            const uint64_t ad = ptx::smem_desc(a + (uint32_t)((i % a_chunks) * 2 * 2048 % (64 * 1024)), 128 * 16, 128);
            const uint64_t bd = ptx::smem_desc(b + (uint32_t)((i % b_chunks) * BN * 32), BN * 16, 128);
            const uint32_t d = tmem + (uint32_t)(((variant & 1) ? 0 : (i & 1)) * BN);
            if (F4)
                ptx::mma_mxf4(d, ad, bd, ptx::idesc_mxf4(128, BN), tmem + 448, tmem + 480, i > 1);
            else
                ptx::mma_i8(d, ad, bd, ptx::idesc_i8(128, BN), i > 1);
        }
        ptx::tc_commit(&done);
        ptx::mbar_wait(&done, 0);
    } else if ((variant & 2) && threadIdx.x == 32) {
        // stream 28 KB blocks into the ring until the MMAs finish (stop flag = done phase)
        constexpr uint32_t kBlk = 28 * 1024;
        uint8_t* ring = smem + 16 * 1024;
        int64_t off = (int64_t)blockIdx.x * kBlk;
        int i = 0;
        for (;; ++i) {
            const int s = i & 3;
            const uint32_t ph = (i >> 2) & 1;
            if (i >= 4) ptx::mbar_wait(&ring_full[s], ph ^ 1);  // previous fill of this slot landed
            uint32_t ready = 0;
            asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ready) : "r"(ptx::smem_u32(&done)), "r"(0u) : "memory");
            if (ready) break;
            ptx::mbar_expect_tx(&ring_full[s], kBlk);
            ptx::bulk_load(ring + s * kBlk, src + off, kBlk, &ring_full[s]);
            off += 148 * kBlk;
            if (off + kBlk > src_bytes) off = (int64_t)blockIdx.x * kBlk;
        }
        for (int j = i > 4 ? i - 4 : 0; j < i; ++j) ptx::mbar_wait(&ring_full[j & 3], (j >> 2) & 1);  // drain
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        uint32_t v[32];
        // read one accumulator column so the work is observable
        ptx::tmem_ld32(tmem, v);
        ptx::tmem_wait_ld();
        if (threadIdx.x == 0) sink[blockIdx.x] = v[0];
        ptx::tmem_dealloc(tmem, 512);
    }
}

// CTA-pair variant: the leader issues cta_group::2 mxf4 MMAs (M = 256, N = BN)
// on resident operands (each CTA holds 128 A rows and BN/2 B rows); `walk`
// steps the operand addresses through distinct K-chunks like the real kernel.
template <int BN>
__global__ void __launch_bounds__(128, 1) mma_pair_probe_kernel(int iters, uint32_t* sink, int walk) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t done;
    __shared__ __align__(8) uint64_t sink_bar[8];
    __shared__ __align__(8) uint64_t open_bar;
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = ptx::cluster_ctarank();
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) {
        // walk & 4: random 0/1 operands (e2m1 nibbles 0x0 / 0x2) like real profiles
        uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (walk & 4) {
            h ^= h >> 13; h *= 0x5bd1e995u; v.x = (h & 0x11111111u) << 1;
            h ^= h >> 15; h *= 0x5bd1e995u; v.y = (h & 0x11111111u) << 1;
            h ^= h >> 13; h *= 0x5bd1e995u; v.z = (h & 0x11111111u) << 1;
            h ^= h >> 15; h *= 0x5bd1e995u; v.w = (h & 0x11111111u) << 1;
        }
        reinterpret_cast<uint4*>(smem)[i] = v;
    }
    ptx::fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        ptx::mbar_init(&done, 1);
        for (int i = 0; i < 8; ++i) ptx::mbar_init(&sink_bar[i], 1);
        ptx::mbar_init(&open_bar, 1);
        ptx::mbar_arrive(&open_bar);  // phase 0 complete: waits on parity 0 pass at once
        ptx::fence_mbar_init();
    }
    ptx::cluster_sync();
    if (warp == 0) ptx::tmem_alloc_pair(&tmem_slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    {
        const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
        ptx::tmem_fill32(lb + 448, 0x7F7F7F7Fu);
        ptx::tmem_fill32(lb + 480, 0x7F7F7F7Fu);
        ptx::tmem_wait_st();
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    if (warp == 0 && rank == 0) {
        // whole warp in the loop, one elected lane issues (as the comparison kernel)
        const uint32_t a = ptx::smem_u32(smem);
        const uint32_t b = a + 64 * 1024;
        const int chunks = walk ? 16 : 1;
        const bool tiled = (walk & 16) != 0;
        const int group = (walk & 64) ? 8 : 4;  // MMAs per stage (wait / commit granularity)
        const int bufs = (walk & 128) ? 3 : 2;
        for (int i0 = 0; i0 < iters; i0 += 4) {
            const bool stage_start = (i0 % group) == 0;
            const bool stage_end = ((i0 + 4) % group) == 0;
            // walk & 32: a (satisfied) mbarrier wait + tcgen05 fence before every stage
            if ((walk & 32) && stage_start) {
                ptx::mbar_wait(&open_bar, 0);
                ptx::tc_fence_after();
            }
            // descriptors computed warp-uniformly, outside the elected region
            uint64_t ad[4], bd[4];
            uint32_t d[4], accf[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int i = i0 + j;
                const int c = i % chunks;
                ad[j] = ptx::smem_desc(a + (uint32_t)(c * 4096), 128 * 16, 128);
                bd[j] = ptx::smem_desc(b + (uint32_t)(c * (BN / 2) * 32), (BN / 2) * 16, 128);
                // walk & 16: the real kernel's tile structure -- 16 K-steps into one of
                // `bufs` accumulators at column offset k*BN, the first step overwriting
                d[j] = tmem + (uint32_t)(tiled ? ((i >> 4) % bufs) * BN
                                               : ((walk & 2) ? 0 : (i & 1) * (BN <= 224 ? 224 : 256)));
                accf[j] = tiled ? (uint32_t)((i & 15) != 0) : (uint32_t)(i > 1);
            }
            if (ptx::elect_one()) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d[j]),
                        "l"(ad[j]), "l"(bd[j]), "r"(ptx::idesc_mxf4(256, BN)), "r"(accf[j]), "r"(tmem + 448),
                        "r"(tmem + 480)
                        : "memory");
                // walk & 8: commit (multicast) after every stage like the real kernel
                if ((walk & 8) && stage_end) ptx::tc_commit_pair(&sink_bar[(i0 / group) & 7], 0x3);
            }
            __syncwarp();
        }
        if (ptx::elect_one()) ptx::tc_commit_pair(&done, 0x3);
        __syncwarp();
    }
    if (threadIdx.x == 0) ptx::mbar_wait(&done, 0);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 0) {
        ptx::tc_fence_after();
        uint32_t v[32];
        ptx::tmem_ld32(tmem, v);
        ptx::tmem_wait_ld();
        if (threadIdx.x == 0) sink[blockIdx.x] = v[0];
        ptx::tmem_dealloc_pair(tmem, 512);
    }
}

__global__ void __launch_bounds__(256) popc_probe_kernel(int iters, uint32_t seed, uint32_t* sink) {
    uint32_t r[8], acc[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = seed * (threadIdx.x + 17 * i + 1);
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0;
    uint32_t q0 = seed ^ threadIdx.x, q1 = seed + blockIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            acc[2 * i] += __popc(r[i] & ~q0);
            acc[2 * i + 1] += __popc(r[i] & ~q1);
        }
        q0 = q0 * 1664525u + 1013904223u;  // keep the words changing (2 IMAD per 16 POPC)
        q1 = q1 ^ (q0 >> 3);
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == 0xDEADBEEF) sink[0] = s;
}

// TMEM -> register read throughput: `warps` warps (4..16) each load `cols`
// columns per tcgen05.ld.32x32b (x8/x16/x32/x64) `iters` times, one wait per load.
template <int X>
__global__ void __launch_bounds__(512, 1) tmem_read_probe_kernel(int iters, uint32_t* sink) {
    __shared__ uint32_t tmem_slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) ptx::tmem_alloc(&tmem_slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64);
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
        uint32_t v[64];
        const uint32_t col = (uint32_t)((i * X) & 255);
        if (X == 8) ptx::tmem_ld8(base + col, v);
        if (X == 32) ptx::tmem_ld32(base + col, *reinterpret_cast<uint32_t(*)[32]>(v));
        if (X == 64) {
            ptx::tmem_ld32(base + col, *reinterpret_cast<uint32_t(*)[32]>(v));
            ptx::tmem_ld32(base + col + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        }
        ptx::tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < X; ++c) acc ^= v[c];
    }
    if (acc == 0x12345678u) sink[0] = acc;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

// MMA + TMEM-read contention: thread 0 issues `iters` mxf4 MMAs (M=128, N=224)
// alternating accumulators at columns [0,448); warps 1..readers read columns
// [0,448) with tcgen05.ld x32 until the MMAs finish.  sink[2*b] = TMEM bytes
// read by CTA b, sink[2*b+1] = clock64 cycles the MMA stream took.
__global__ void __launch_bounds__(512, 1) mma_tmem_contention_kernel(int iters, int readers,
                                                                      unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t done;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (128 + 224) * 32 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    ptx::fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        ptx::mbar_init(&done, 1);
        ptx::fence_mbar_init();
        stop = 0;
    }
    if (warp == 0) ptx::tmem_alloc(&tmem_slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (warp < 4) {
        const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
        ptx::tmem_fill32(lb + 448, 0x7F7F7F7Fu);
        ptx::tmem_fill32(lb + 480, 0x7F7F7F7Fu);
        ptx::tmem_wait_st();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t a = ptx::smem_u32(smem);
        const uint64_t ad = ptx::smem_desc(a, 128 * 16, 128);
        const uint64_t bd = ptx::smem_desc(a + 128 * 32, 224 * 16, 128);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i)
            ptx::mma_mxf4(tmem + (uint32_t)((i & 1) * 224), ad, bd, ptx::idesc_mxf4(128, 224), tmem + 448,
                          tmem + 480, i > 1);
        ptx::tc_commit(&done);
        ptx::mbar_wait(&done, 0);
        sink[2 * blockIdx.x + 1] = (unsigned long long)(clock64() - t0);
        stop = 1;
    } else if (warp >= 1 && warp <= readers) {
        const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        unsigned long long bytes = 0;
        uint32_t acc = 0;
        int i = 0;
        while (!stop) {
            uint32_t v[32];
            ptx::tmem_ld32(base + (uint32_t)((i * 32) % 448), v);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) acc ^= v[c];
            bytes += 32 * 32 * 4;
            ++i;
        }
        if (acc == 0x12345u) bytes += 1;
        if ((threadIdx.x & 31) == 0) atomicAdd(&sink[2 * blockIdx.x], bytes);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

}  // namespace
}  // namespace fastid

using namespace fastid;

extern "C" int fastid_probe_contention(int iters, int readers, void* sink, void* stream) {
    int dev = 0, sms = 148;
    FASTID_CUDA(cudaGetDevice(&dev));
    FASTID_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FASTID_CUDA(cudaFuncSetAttribute(mma_tmem_contention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
    mma_tmem_contention_kernel<<<sms, 512, 200 * 1024, (cudaStream_t)stream>>>(iters, readers,
                                                                               (unsigned long long*)sink);
    FASTID_LAUNCHED("mma_tmem_contention_kernel");
    return FASTID_OK;
}

// Diagnostic: TMEM read probe.  Returns bytes read via *work.
extern "C" int fastid_probe_tmem_read(int x, int warps, int iters, void* scratch, double* work, void* stream) {
    int dev = 0, sms = 148;
    FASTID_CUDA(cudaGetDevice(&dev));
    FASTID_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cudaStream_t st = (cudaStream_t)stream;
    if (warps < 4 || warps > 16 || warps % 4) FASTID_FAIL(FASTID_E_INVALID, "warps must be 4, 8, 12 or 16");
    if (x == 8) tmem_read_probe_kernel<8><<<sms, 32 * warps, 0, st>>>(iters, (uint32_t*)scratch);
    else if (x == 32) tmem_read_probe_kernel<32><<<sms, 32 * warps, 0, st>>>(iters, (uint32_t*)scratch);
    else if (x == 64) tmem_read_probe_kernel<64><<<sms, 32 * warps, 0, st>>>(iters, (uint32_t*)scratch);
    else FASTID_FAIL(FASTID_E_INVALID, "x must be 8, 32 or 64");
    FASTID_LAUNCHED("tmem_read_probe_kernel");
    *work = (double)sms * warps * 32.0 * x * 4.0 * iters;
    return FASTID_OK;
}

// Launch the probe for `formulation` with `iters` inner iterations per CTA (tensor)
// or per thread (popc).  *work receives the bit-pairs (MACs) the launch performs.
extern "C" int fastid_probe_variant(int formulation, int variant, int iters, void* scratch, const void* src,
                                    int64_t src_bytes, double* work, void* stream);

extern "C" int fastid_probe_peak(int formulation, int iters, void* scratch, double* work, void* stream) {
    return fastid_probe_variant(formulation, 0, iters, scratch, nullptr, 0, work, stream);
}

extern "C" int fastid_probe_variant(int formulation, int variant, int iters, void* scratch, const void* src,
                                    int64_t src_bytes, double* work, void* stream) {
    int dev = 0, sms = 148;
    FASTID_CUDA(cudaGetDevice(&dev));
    FASTID_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t* sink = (uint32_t*)scratch;
    if (formulation == FASTID_POPC) {
        const int blocks = sms * 8;
        popc_probe_kernel<<<blocks, 256, 0, st>>>(iters, 0x9E3779B9u, sink);
        FASTID_LAUNCHED("popc_probe_kernel");
        *work = (double)blocks * 256 * iters * 16 * 32;
        return FASTID_OK;
    }
    const bool f4 = formulation == FASTID_TENSOR_F4 || formulation == FASTID_AUTO;
    if (f4 && (variant & 8)) {
        // CTA pairs: variant bit 4 selects N = 256 (else 224), bit 2 walks operand addresses
        const bool n256 = (variant & 16) != 0;
        const bool n192 = (variant & 128) != 0;
        const bool n144 = (variant & 1024) != 0;
        const bool n96 = (variant & 8192) != 0;
        auto kern = n96 ? mma_pair_probe_kernel<96> : n144 ? mma_pair_probe_kernel<144>
                         : (n192 ? mma_pair_probe_kernel<192>
                                 : (n256 ? mma_pair_probe_kernel<256> : mma_pair_probe_kernel<224>));
        FASTID_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)(sms & ~1));
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = 160 * 1024;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        // variant bit 0: one accumulator (K-loop dependency chain), bit 2: walk operand addresses
        FASTID_CUDA(cudaLaunchKernelEx(&cfg, kern, iters, sink, ((variant & 4) ? 1 : 0) | ((variant & 1) ? 2 : 0) | ((variant & 32) ? 4 : 0) |
                                                             ((variant & 64) ? 8 : 0) | ((variant & 256) ? 16 : 0) | ((variant & 512) ? 32 : 0) |
                                                             ((variant & 2048) ? 64 : 0) | ((variant & 4096) ? 128 : 0)));
        FASTID_LAUNCHED("mma_pair_probe_kernel");
        *work = (double)(sms / 2) * iters * 256.0 * (n96 ? 96 : (n144 ? 144 : (n192 ? 192 : (n256 ? 256 : 224)))) * 64.0;
        return FASTID_OK;
    }
    const int bn = f4 ? 224 : 128;
    const int smem = (128 + bn) * 32;
    if (f4) {
        FASTID_CUDA(cudaFuncSetAttribute(mma_probe_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        mma_probe_kernel<true><<<sms, 128, 200 * 1024, st>>>(iters, sink, variant, (const uint8_t*)src, src_bytes);
    } else {
        FASTID_CUDA(cudaFuncSetAttribute(mma_probe_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        mma_probe_kernel<false><<<sms, 128, 200 * 1024, st>>>(iters, sink, variant, (const uint8_t*)src, src_bytes);
    }
    (void)smem;
    FASTID_LAUNCHED("mma_probe_kernel");
    const double k = f4 ? 64.0 : 32.0;
    *work = (double)sms * iters * 128.0 * bn * k;
    return FASTID_OK;
}

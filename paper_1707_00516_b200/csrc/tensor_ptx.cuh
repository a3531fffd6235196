// Thin inline-PTX wrappers for the sm_100a features the tensor formulation
// uses: mbarriers, TMA (cp.async.bulk.tensor), tcgen05 (alloc / mma / commit /
// ld / st / fences) and UMMA shared-memory + instruction descriptors.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace fastid {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---- mbarrier -------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Wait with a suspend-time hint: the thread sleeps in the barrier unit until the
// phase completes (or the hint expires) instead of re-issuing try_wait -- for
// warps that wait most of a tile (the epilogue on the accumulator), so the
// spinning does not cost issue slots and power.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}

// ---- proxies / TMA ---------------------------------------------------------
// Make generic-proxy st.shared visible to the async proxy (tensor core reads).
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(map) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

// Prefetch one tensor-map box into L2 (no shared-memory destination, no
// barrier): a later TMA load of the same box then hits in L2.
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(map), "r"(x), "r"(y)
                 : "memory");
}

// 1-D bulk copy global -> shared, completing `bytes` of transaction on `bar`.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// One lane of the (converged) warp returns true.  Issue paths keep the whole
// warp in the loop and elect the issuing lane only around the instruction, so
// loop state and descriptors stay warp-uniform (uniform registers, no per-MMA
// R2UR waterfall).
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n"
        ".reg .b32 rx;\n"
        ".reg .pred px;\n"
        "elect.sync rx|px, %1;\n"
        "@px mov.s32 %0, 1;\n"
        "}\n"
        : "+r"(pred)
        : "r"(0xFFFFFFFFu));
    return pred != 0;
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Relaxed gpu-scope global accesses (progress counters shared between CTAs).
__device__ __forceinline__ void st_relaxed(int* p, int v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// TMA tensor store shared -> global (bulk group completion).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(map),
                 "r"(smem_u32(src)), "r"(x), "r"(y)
                 : "memory");
}
// Named barrier among `count` threads (id 1..15; 0 is __syncthreads).
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// wait until every committed bulk store has finished reading shared memory
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// ---- clusters (CTA pairs for cta_group::2) ----------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
// shared::cluster address of the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// Arrive on an mbarrier given by its shared::cluster address (default .release.cta
// semantics, as CUTLASS's ClusterBarrier::arrive: the arrivals here only order
// completed tcgen05.ld / async-proxy work, and a cluster-scope release would
// fence every prior global store of the thread).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
// Wait with cluster-scope acquire (barriers that receive arrivals from the peer CTA).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITC_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 2-D tensor copy into this CTA's shared memory whose completion is counted on
// an mbarrier of either CTA of the pair (shared::cluster address).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int x,
                                                 int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(bar_cluster), "r"(x), "r"(y)
        : "memory");
}

// ---- tcgen05 ---------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
// CTA-pair TMEM allocation: issued by the same warp of both CTAs.
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// Arrive on an mbarrier once every previously issued tcgen05.mma of this thread completes.
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}

// Pair commit: arrive on the mbarrier at the same offset in every CTA of `mask`
// once the pair MMAs issued so far by this thread complete.
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// D[tmem] (+)= A[smem] . B[smem]^T, int8 operands, int32 accumulate.
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// D[tmem] (+)= (A . SFA)[smem] . (B . SFB)[smem]^T, e2m1 operands with
// ue8m0 scale factors per 32 K-elements read from TMEM, fp32 accumulate.
__device__ __forceinline__ void mma_mxf4(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t tmem_sfa, uint32_t tmem_sfb, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(tmem_sfa), "r"(tmem_sfb)
        : "memory");
}

// One pipeline stage of MMAs in a single asm block: N consecutive K-steps,
// operand descriptors advanced by fixed 16-byte-unit strides (a_step/b_step),
// the first step accumulating only when `accumulate` is set.  Issuing the whole
// stage at once keeps the single-thread issue path to a few instructions per
// MMA (the stage's MMAs otherwise cost ~20 uniform-datapath ops each).
__device__ __forceinline__ void mma_mxf4_stage4(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint64_t a_step,
                                                uint64_t b_step, uint32_t idesc, uint32_t sfa, uint32_t sfb,
                                                uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, t;\n"
        ".reg .b64 a1, a2, a3, b1, b2, b3;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.u32 t, 0, 0;\n"
        "add.s64 a1, %1, %7; add.s64 b1, %2, %8;\n"
        "add.s64 a2, a1, %7; add.s64 b2, b1, %8;\n"
        "add.s64 a3, a2, %7; add.s64 b3, b2, %8;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a1, b1, %3, [%5], [%6], t;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a2, b2, %3, [%5], [%6], t;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a3, b3, %3, [%5], [%6], t;\n"
        "}\n" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb), "l"(a_step), "l"(b_step)
        : "memory");
}
// The same stage as a CTA pair (cta_group::2, M = 256): A rows 0-127 come from
// the leader's shared memory and 128-255 from the peer's, B rows 0..N/2-1 from
// the leader's and N/2..N-1 from the peer's, at identical offsets; each CTA's
// TMEM receives its own 128 rows of D.
__device__ __forceinline__ void mma_mxf4_pair_stage4(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint64_t a_step,
                                                     uint64_t b_step, uint32_t idesc, uint32_t sfa, uint32_t sfb,
                                                     uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, t;\n"
        ".reg .b64 a1, a2, a3, b1, b2, b3;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.u32 t, 0, 0;\n"
        "add.s64 a1, %1, %7; add.s64 b1, %2, %8;\n"
        "add.s64 a2, a1, %7; add.s64 b2, b1, %8;\n"
        "add.s64 a3, a2, %7; add.s64 b3, b2, %8;\n"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a1, b1, %3, [%5], [%6], t;\n"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a2, b2, %3, [%5], [%6], t;\n"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a3, b3, %3, [%5], [%6], t;\n"
        "}\n" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb), "l"(a_step), "l"(b_step)
        : "memory");
}
// One stage on a single CTA whose B operand is split in two row halves (the
// pair layout of the prepared image): two N/2 MMAs per K-step into adjacent
// accumulator column ranges.
__device__ __forceinline__ void mma_mxf4_split_stage4(uint32_t tmem_d, uint32_t half_cols, uint64_t ad, uint64_t bd,
                                                      uint64_t b_half, uint64_t a_step, uint64_t b_step,
                                                      uint32_t idesc_half, uint32_t sfa, uint32_t sfb,
                                                      uint32_t accumulate) {
    const uint32_t d1 = tmem_d + half_cols;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t acc = j ? 1u : accumulate;
        mma_mxf4(tmem_d, ad + j * a_step, bd + j * b_step, idesc_half, sfa, sfb, acc);
        mma_mxf4(d1, ad + j * a_step, bd + b_half + j * b_step, idesc_half, sfa, sfb, acc);
    }
}
__device__ __forceinline__ void mma_i8_stage8(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint64_t a_step,
                                              uint64_t b_step, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, t;\n"
        ".reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.u32 t, 0, 0;\n"
        "add.s64 a1, %1, %5; add.s64 b1, %2, %6;\n"
        "add.s64 a2, a1, %5; add.s64 b2, b1, %6;\n"
        "add.s64 a3, a2, %5; add.s64 b3, b2, %6;\n"
        "add.s64 a4, a3, %5; add.s64 b4, b3, %6;\n"
        "add.s64 a5, a4, %5; add.s64 b5, b4, %6;\n"
        "add.s64 a6, a5, %5; add.s64 b6, b5, %6;\n"
        "add.s64 a7, a6, %5; add.s64 b7, b6, %6;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, %3, t;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], a2, b2, %3, t;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], a3, b3, %3, t;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], a4, b4, %3, t;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], a5, b5, %3, t;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], a6, b6, %3, t;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], a7, b7, %3, t;\n"
        "}\n" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(accumulate), "l"(a_step), "l"(b_step)
        : "memory");
}

// 32 lanes x 32 columns of 32-bit TMEM -> 32 registers per thread (lane = thread).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
// 32 lanes x 16 columns.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
// 32 lanes x 8 columns into v[0..7].
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// Broadcast one 32-bit value into 32 lanes x 32 columns of TMEM.
__device__ __forceinline__ void tmem_fill32(uint32_t taddr, uint32_t x) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
        "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};\n" ::"r"(taddr),
        "r"(x)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// ---- UMMA descriptors --------------------------------------------------------
// K-major, no swizzle ("interleave") canonical layout: 8-row x 16-byte core
// matrices stored contiguously (128 B); `lbo` = byte distance between
// K-adjacent core matrices, `sbo` = byte distance between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100)
    return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

// kind::i8 instruction descriptor: u8 x u8 -> s32, K-major A and B.
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
    return (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
// kind::mxf4 instruction descriptor: e2m1 x e2m1, ue8m0 scales, K = 64.
__host__ __device__ constexpr uint32_t idesc_mxf4(int m, int n) {
    return (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) | ((uint32_t)(m >> 4) << 24);
}

}  // namespace ptx
}  // namespace fastid

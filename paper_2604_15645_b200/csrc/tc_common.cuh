// tc_common.cuh -- thin inline-PTX layer for sm_100a 5th-gen tensor cores:
// mbarriers, TMEM alloc/ld, UMMA smem/instruction descriptors, tcgen05.mma
// kind::tf32 issue/commit, and the 3xTF32 split.
//
// Shared-memory operand layouts (all with the 128-byte swizzle, atoms of
// 8 rows x 128 B, 1024 B aligned; physical 16 B chunk = chunk ^ (row % 8)):
//   K-major  tile [rows][32 fp32]: row r at r*128, 8-row groups SBO = 1024 B.
//            One MMA consumes K = 8 (32 B): k-step j -> start address + 32*j.
//   MN-major tile [k rows][MN]: atom = 8 k-rows x 32 MN elements; MN groups of
//            32 at LBO, k groups of 8 at SBO.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pnx {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ---------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// 1-D bulk async copy global -> shared (TMA engine), completes tx bytes on `bar`
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// 3-D tensor-map TMA load global -> shared: box origin (c0 fastest), tx bytes on `bar`
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// 2-D tensor-map load into this CTA's smem whose completion is signalled on the
// barrier `bar_cluster` (a shared::cluster address, e.g. the pair leader's)
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                                 uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster)
        : "memory");
}

// 3-D tensor-map store shared -> global (bulk group of the issuing thread)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(src)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N bulk groups of this thread still read shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// ---- proxy / tcgen05 fences ---------------------------------------------------
// generic-proxy smem writes -> visible to the async proxy (tensor core reads)
__device__ __forceinline__ void fence_proxy_async_smem() {
#ifndef PNX_EXP_NOFENCE  // timing experiment only: removing it is a race
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---- TMEM allocation (one full warp) ------------------------------------------
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "n"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS));
}

// ---- TMEM -> registers: 32 lanes x 16 consecutive 32-bit columns --------------
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---- descriptors ----------------------------------------------------------------
// SMEM matrix descriptor (sm_100 "version 1"), 128 B swizzle.
__device__ __forceinline__ uint64_t make_sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // version
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}

// Generic K-major descriptor: layout 2 = SW128, 4 = SW64, 6 = SW32, 0 = none.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                               uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(layout & 7u) << 61;
    return d;
}

// byte offset of element (row, k) of a K-major SW32 tile with 8 fp32 of K per
// row (32 B rows, 8-row groups of 256 B): chunk (k/4) ^= (row/4)&1.
__host__ __device__ __forceinline__ uint32_t sw32_off(uint32_t row, uint32_t k) {
    return (row >> 3) * 256u + (row & 7u) * 32u + ((((k >> 2) ^ (row >> 2)) & 1u) << 4) + (k & 3u) * 4u;
}
// K-major SW64 tile, 16 fp32 of K per row (64 B rows, 8-row groups of 512 B):
// chunk (k/4) ^= (row/2)&3.
__host__ __device__ __forceinline__ uint32_t sw64_off(uint32_t row, uint32_t k) {
    return (row >> 3) * 512u + (row & 7u) * 64u + ((((k >> 2) ^ (row >> 1)) & 3u) << 4) + (k & 3u) * 4u;
}

// Instruction descriptor: kind::tf32, FP32 accumulate, M x N, operand majors.
__host__ __device__ constexpr uint32_t make_idesc_tf32(int M, int N, int a_mn_major, int b_mn_major) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem], kind::tf32, issued by ONE thread.
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// Arrive on `bar` when all previously issued MMAs of this thread complete.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// ---- CTA pair (cta_group::2) -------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> shared::cluster address of the same offset in CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
// arrive on a barrier of another CTA of the cluster (default .release.cta
// semantics; smem operands are ordered for the tensor core by the preceding
// fence.proxy.async, as in CUTLASS's 2-SM pipelines)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
#ifdef PNX_EXP_CLUSTER_RELEASE
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#else
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#endif
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "n"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS));
}
// M=256 MMA over the pair: A rows 0-127 / 128-255 and B columns [0,N/2) / [N/2,N)
// from the same smem offsets of CTA 0 / CTA 1; D rows land in each CTA's TMEM.
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive on `bar` (same offset) in every CTA of `mask` when the pair's MMAs complete
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// ---- kind::f16 (fp16 operands, FP32 accumulate) ------------------------------
// Instruction descriptor: like make_idesc_tf32 with a/b format F16 (0).
__host__ __device__ constexpr uint32_t make_idesc_f16(int M, int N, int a_mn_major, int b_mn_major) {
    return (1u << 4) | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// MN-major SWIZZLE_128B tile of 16-bit elements: 64 MN elements (128 B) per
// k-row, 8 k-rows per 1024 B atom, 16 B chunks XOR k-row; atoms ordered
// [k/8][mn/64]: LBO = 1024 (next 64 MN), SBO = (mn_extent/64)*1024 (next 8 k).
__host__ __device__ __forceinline__ uint32_t mn16_off(uint32_t k, uint32_t mn, uint32_t mn_extent) {
    return (k >> 3) * (mn_extent / 64u) * 1024u + (mn >> 6) * 1024u + (k & 7u) * 128u +
           ((((mn & 63u) >> 3) ^ (k & 7u)) << 4) + (mn & 7u) * 2u;
}
// power-of-two scale that puts |x| <= amax into [2^13, 2^14) (fp16 max 65504)
__device__ __forceinline__ int f16_scale_exp(float amax) {
    if (!(amax > 0.0f) || !isfinite(amax)) return 0;
    return 13 - ilogbf(amax);
}
__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// ---- 3xFP16 split ---------------------------------------------------------------
// x * 2^e = hi + lo with hi = fp16(x 2^e), lo = fp16(x 2^e - hi): 11 + 11
// significant bits, the same as the tf32 hi/lo pair, at twice the tensor rate
// per instruction (kind::f16 K = 16 in the cycles of kind::tf32 K = 8). The
// power-of-two scale 2^e puts the operand's absmax bound into [2^13, 2^14)
// (f16_scale_exp), far below the fp16 maximum; elements far below the bound
// lose only absolute precision under 2^-25 of the scaled unit in lo.
__device__ __forceinline__ void split_h2(float a, float b, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}
// 8 consecutive K elements (one 16 B chunk of a K-major fp16 row), scaled by sc
__device__ __forceinline__ void split_h8(const float* h, float sc, uint4& hi, uint4& lo) {
    split_h2(h[0] * sc, h[1] * sc, hi.x, lo.x);
    split_h2(h[2] * sc, h[3] * sc, hi.y, lo.y);
    split_h2(h[4] * sc, h[5] * sc, hi.z, lo.z);
    split_h2(h[6] * sc, h[7] * sc, hi.w, lo.w);
}
// byte offset of 16 B chunk c (0/1) of row `row` in a K-major SW32 tile (32 B
// rows = 8 fp32 or 16 fp16 of K; chunk ^= (row/4)&1) -- sw32_off(row, 4c)
__host__ __device__ __forceinline__ uint32_t sw32_chunk(uint32_t row, uint32_t c) {
    return (row >> 3) * 256u + (row & 7u) * 32u + (((c ^ (row >> 2)) & 1u) << 4);
}
// element (row, k), k < 16, of a K-major SW32 fp16 tile
__host__ __device__ __forceinline__ uint32_t sw32h_off(uint32_t row, uint32_t k) {
    return sw32_chunk(row, k >> 3) + (k & 7u) * 2u;
}
// |x| bound as order-preserving bits (non-negative floats compare as uints)
__device__ __forceinline__ unsigned abs_bits(float x) { return __float_as_uint(fabsf(x)); }
// fold a per-lane max into *dst (one atomic per warp)
__device__ __forceinline__ void warp_amax(unsigned* dst, unsigned v) {
    v = __reduce_max_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0) atomicMax(dst, v);
}
// operand scale exponent from a recorded absmax (bits) -- bound in [2^13, 2^14)
__device__ __forceinline__ int f16_exp_bits(unsigned bits) {
    const int e = f16_scale_exp(__uint_as_float(bits));
    return e > 110 ? 110 : (e < -110 ? -110 : e);
}

// ---- 3xTF32 split -------------------------------------------------------------
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ void split3(float x, float& hi, float& lo) {
    hi = tf32_rna(x);
    lo = tf32_rna(x - hi);
}

// MN-major tf32 tile in SWIZZLE_128B_BASE32B atoms (4 k-rows x 32 MN elements,
// 512 B; 32 B chunks XOR (k % 4)), atoms ordered [k/4][mn/32]:
// LBO = 512 (next MN group), SBO = (mn_extent/32)*512 (next 4-row k group).
__host__ __device__ __forceinline__ uint32_t mn32_off(uint32_t k, uint32_t mn, uint32_t mn_extent) {
    return (k >> 2) * (mn_extent / 32u) * 512u + (mn >> 5) * 512u + (k & 3u) * 128u +
           ((((mn & 31u) >> 3) ^ (k & 3u)) << 5) + (mn & 7u) * 4u;
}

// byte offset of 16 B chunk `c` (0..7) of row `r` inside a 128 B-swizzled atom run
__device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t chunk) {
    return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

}  // namespace tc
}  // namespace pnx

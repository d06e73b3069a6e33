// tc_sm100.cuh -- minimal tcgen05 / TMEM / mbarrier helpers (inline PTX, sm_100a).
//
// Operand layout used everywhere ("interleaved core-matrix" layout, SWIZZLE_NONE):
// a fp16 matrix with R rows and C columns (both multiples of 8) is stored as
// (R/8) x (C/8) blocks of 8x8 elements; block (rb, cb) starts at byte
// (rb * (C/8) + cb) * 128 and holds its 8 rows of 8 contiguous fp16 (16 B each).
// The same bytes are a valid UMMA operand in both majors:
//   K-major  (rows = M|N, cols = K):  LBO = 128 B,            SBO = (C/8)*128 B
//   MN-major (rows = K,   cols = M|N): LBO = (C/8)*128 B,     SBO = 128 B
// (canonical forms: K-major ((8,m),(T,2)):((1T,SBO),(1,LBO)); MN-major
// ((T,1,m),(8,k)):((1,T,SBO),(1T,LBO)), T = 8 fp16 per 16 B).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// byte offset of element (r, c) in an interleaved R x C fp16 matrix
__device__ __forceinline__ uint32_t il_offset(int r, int c, int C) {
    return (uint32_t)((((r >> 3) * (C >> 3) + (c >> 3)) << 7) + ((r & 7) << 4) + ((c & 7) << 1));
}

// shared-memory matrix descriptor (SWIZZLE_NONE, version 1 for sm_100)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;   // version = 1 (Blackwell)
    return d;                 // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// descriptor of the K-step `ks` (16 elements of K) of an interleaved matrix
// used K-major (cols = K): start advances by 2 column blocks
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t base, int C, int ks) {
    return make_desc(base + (uint32_t)(ks * 2 * 128), 128u, (uint32_t)((C >> 3) * 128));
}
// ... used MN-major (rows = K): start advances by 2 row blocks
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t base, int C, int ks) {
    return make_desc(base + (uint32_t)(ks * 2 * (C >> 3) * 128), (uint32_t)((C >> 3) * 128), 128u);
}

// instruction descriptor: kind::f16, A/B fp16, D fp32
__device__ __forceinline__ uint32_t idesc_f16(int M, int N, bool a_mn, bool b_mn) {
    uint32_t d = 0;
    d |= 1u << 4;                          // D format F32
    // A, B format F16 = 0
    d |= (a_mn ? 1u : 0u) << 15;
    d |= (b_mn ? 1u : 0u) << 16;
    d |= (uint32_t)(N >> 3) << 17;
    d |= (uint32_t)(M >> 4) << 24;
    return d;
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
        :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// arrive on an mbarrier once all prior tcgen05.mma of this thread completed
__device__ __forceinline__ void commit(uint64_t* mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                 :: "r"(smem_u32(mbar)) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(mbar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n"
        :: "r"(smem_u32(mbar)), "r"(phase) : "memory");
}

// plain arrive (release, CTA scope) on an mbarrier
__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" :: "r"(smem_u32(mbar)) : "memory");
}

// named barrier over `n` threads (a multiple of 32)
__device__ __forceinline__ void bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;\n" :: "r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// TMEM allocation (whole warp)
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                 :: "r"(smem_u32(dst_smem)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(taddr), "r"(ncols) : "memory");
}

// 32 lanes x 16 columns of 32-bit: thread t of warp w gets lane 32*(w%4)+t
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// load + wait in one asm block, so no consumer of the values can be scheduled
// before tcgen05.wait::ld
__device__ __forceinline__ void tmem_ld16_sync(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr) : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// 4 columns + wait
__device__ __forceinline__ void tmem_ld2x2_sync(uint32_t ta, uint32_t tb, float (&v)[4]) {
    uint32_t r[4];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%4];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%2,%3}, [%5];\n\t"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta), "r"(tb) : "memory");
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld4_sync(uint32_t taddr, float (&v)[4]) {
    uint32_t r[4];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n\t"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr) : "memory");
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
// 32 columns (two x16 loads in flight) + wait
__device__ __forceinline__ void tmem_ld32_sync(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33];\n\t"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr), "r"(taddr + 16u) : "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// TMEM address of (lane_base, col)
__device__ __forceinline__ uint32_t taddr(uint32_t base, int lane_base, int col) {
    return base + ((uint32_t)lane_base << 16) + (uint32_t)col;
}

// 16-byte shared store (-DROMAP_EXP_NOMSTS, timing experiment only: dropped,
// operands kept live)
__device__ __forceinline__ void sts128(void* p, uint4 v) {
#ifdef ROMAP_EXP_NOMSTS
    asm volatile("" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
#else
    *reinterpret_cast<uint4*>(p) = v;
#endif
}

// store 8 fp16 (16 B) at an interleaved position (row r, column block starting at c)
__device__ __forceinline__ void st_chunk(uint8_t* buf, int r, int c, int C, const float* v8) {
    __half2 h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(v8[2 * i], v8[2 * i + 1]);
    sts128(buf + il_offset(r, c, C), *reinterpret_cast<uint4*>(h));
}


// store 16 consecutive fp32 values (columns c0..c0+15 of row r) as fp16
__device__ __forceinline__ void st16(uint8_t* buf, int r, int c0, int C, const float* v) {
    st_chunk(buf, r, c0, C, v);
    st_chunk(buf, r, c0 + 8, C, v + 8);
}

// forward epilogue of a 64-wide layer (M thread, row r): TMEM -> fp16 ->
// ReLU on packed halves (relu(round(v)) = round(relu(v))) -> smem
__device__ __forceinline__ void epi_relu64(uint32_t wk, uint8_t* buf, int r) {
    const __half2 z = __float2half2_rn(0.f);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        float v[32];
        tmem_ld32_sync(wk + 32 * h, v);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            __half2 q[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) q[k] = __hmax2(__floats2half2_rn(v[8 * c + 2 * k], v[8 * c + 2 * k + 1]), z);
            sts128(buf + il_offset(r, 32 * h + 8 * c, 64), *reinterpret_cast<uint4*>(q));
        }
    }
}

}  // namespace tc

// k_selftest.cu -- tcgen05 operand-layout self test (exported for the GPU tests):
// one CTA computes, from fp16 copies of the inputs, with the exact descriptor /
// layout helpers the fused training kernel uses,
//   out1[128x64] = X[128x32] . W[64x32]^T        (A K-major,  B K-major,  M=128)
//   out2[128x32] = Dl[128x64] . W[64x32]         (A K-major,  B MN-major, M=128)
//   out3[64x32]  = Dl[128x64]^T . X[128x32]      (A MN-major, B MN-major, M=64)
// i.e. a forward layer, its input gradient and its weight gradient.
#include "../../include/romap.h"
#include "romap_internal.cuh"
#include "tc_sm100.cuh"

__global__ void __launch_bounds__(128, 1) k_mma_selftest(const float* __restrict__ X, const float* __restrict__ W,
                                                         const float* __restrict__ Dl, float* out1, float* out2,
                                                         float* out3) {
    __shared__ __align__(1024) uint8_t sX[128 * 32 * 2];
    __shared__ __align__(1024) uint8_t sW[64 * 32 * 2];
    __shared__ __align__(1024) uint8_t sD[128 * 64 * 2];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int e = t; e < 128 * 32; e += 128) {
        int r = e / 32, c = e % 32;
        *reinterpret_cast<__half*>(sX + tc::il_offset(r, c, 32)) = __float2half_rn(X[e]);
    }
    for (int e = t; e < 64 * 32; e += 128) {
        int r = e / 32, c = e % 32;
        *reinterpret_cast<__half*>(sW + tc::il_offset(r, c, 32)) = __float2half_rn(W[e]);
    }
    for (int e = t; e < 128 * 64; e += 128) {
        int r = e / 64, c = e % 64;
        *reinterpret_cast<__half*>(sD + tc::il_offset(r, c, 64)) = __float2half_rn(Dl[e]);
    }
    if (warp == 0) tc::tmem_alloc(&tmem_base, 128);
    if (t == 0) {
        tc::mbar_init(&mbar, 1);
        tc::fence_mbar_init();
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tb = tmem_base;
    if (t == 0) {
        const uint32_t x = tc::smem_u32(sX), w = tc::smem_u32(sW), d = tc::smem_u32(sD);
        for (int ks = 0; ks < 2; ++ks)
            tc::mma_f16(tb + 0, tc::desc_kmajor(x, 32, ks), tc::desc_kmajor(w, 32, ks), tc::idesc_f16(128, 64, false, false), ks > 0);
        for (int ks = 0; ks < 4; ++ks)
            tc::mma_f16(tb + 64, tc::desc_kmajor(d, 64, ks), tc::desc_mnmajor(w, 32, ks), tc::idesc_f16(128, 32, false, true), ks > 0);
        for (int ks = 0; ks < 8; ++ks)
            tc::mma_f16(tb + 96, tc::desc_mnmajor(d, 64, ks), tc::desc_mnmajor(x, 32, ks), tc::idesc_f16(64, 32, true, true), ks > 0);
        tc::commit(&mbar);
    }
    tc::mbar_wait(&mbar, 0);
    tc::fence_after();
    float v[16];
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < 64; c0 += 16) {
        tc::tmem_ld16(tc::taddr(tb, warp * 32, c0), v);
        tc::tmem_wait_ld();
        for (int i = 0; i < 16; ++i) out1[row * 64 + c0 + i] = v[i];
    }
    for (int c0 = 0; c0 < 32; c0 += 16) {
        tc::tmem_ld16(tc::taddr(tb, warp * 32, 64 + c0), v);
        tc::tmem_wait_ld();
        for (int i = 0; i < 16; ++i) out2[row * 32 + c0 + i] = v[i];
    }
    for (int c0 = 0; c0 < 32; c0 += 16) {
        tc::tmem_ld16(tc::taddr(tb, warp * 32, 96 + c0), v);
        tc::tmem_wait_ld();
        if (lane < 16)
            for (int i = 0; i < 16; ++i) out3[(warp * 16 + lane) * 32 + c0 + i] = v[i];
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tb, 128);
}

extern "C" romap_status romap_selftest_mma(const float* X, const float* W, const float* Dl, float* out1, float* out2,
                                           float* out3) {
    float* d = nullptr;
    size_t n = 128 * 32 + 64 * 32 + 128 * 64 + 128 * 64 + 128 * 32 + 64 * 32;
    if (cudaMalloc(&d, n * 4) != cudaSuccess) return ROMAP_E_CUDA;
    float *dX = d, *dW = dX + 128 * 32, *dD = dW + 64 * 32, *o1 = dD + 128 * 64, *o2 = o1 + 128 * 64, *o3 = o2 + 128 * 32;
    cudaMemcpy(dX, X, 128 * 32 * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, W, 64 * 32 * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dD, Dl, 128 * 64 * 4, cudaMemcpyHostToDevice);
    k_mma_selftest<<<1, 128>>>(dX, dW, dD, o1, o2, o3);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) {
        cudaMemcpy(out1, o1, 128 * 64 * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(out2, o2, 128 * 32 * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(out3, o3, 64 * 32 * 4, cudaMemcpyDeviceToHost);
    }
    cudaFree(d);
    return e == cudaSuccess ? ROMAP_OK : ROMAP_E_CUDA;
}

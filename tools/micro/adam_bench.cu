// Microbenchmark: the Adam step (a8) over cfg1's 1.71 M parameters in the
// state bench.py times it in -- p, m, v cold (L2 flushed, flush lines dirty),
// g L2-resident (just written by the fused kernel).  Variants:
//   V0  one wave, 256 thr x 4 float4 groups per thread, 3 blocks/SM (k_adam today)
//   V1  2 groups per thread, 6 blocks/SM
//   V2  grid-stride, 148 x 8 blocks, 1 group per trip, unroll 2
//   V3  TMA bulk: persistent 148 x 2 blocks, 4 x 8 KB chunks per stage, 2 stages
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 adam_bench.cu -o adam_bench
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct P {
    float *p, *m, *v, *g;
    __half* h;
    int n;
    float ibc1, ibc2;
};

__device__ __forceinline__ void upd1(float& p, float& m, float& v, float g, const P& a) {
    m = 0.9f * m + 0.1f * g;
    v = 0.99f * v + 0.01f * g * g;
    p = p - 1e-2f * (m * a.ibc1) / (sqrtf(v * a.ibc2) + 1e-15f);
}

__device__ __forceinline__ void upd4(float4& p, float4& m, float4& v, float4 g, const P& a) {
    upd1(p.x, m.x, v.x, g.x, a); upd1(p.y, m.y, v.y, g.y, a); upd1(p.z, m.z, v.z, g.z, a); upd1(p.w, m.w, v.w, g.w, a);
}

__device__ __forceinline__ void store4(const P& a, int q, float4 p, float4 m, float4 v) {
    reinterpret_cast<float4*>(a.p)[q] = p;
    reinterpret_cast<float4*>(a.m)[q] = m;
    reinterpret_cast<float4*>(a.v)[q] = v;
    reinterpret_cast<float4*>(a.g)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    __half2* h2 = reinterpret_cast<__half2*>(a.h + 4 * q);
    h2[0] = __floats2half2_rn(p.x, p.y);
    h2[1] = __floats2half2_rn(p.z, p.w);
}

template <int G, int MINB>
__global__ void __launch_bounds__(256, MINB) k_wave(P a) {
    const int n4 = a.n / 4;
    const int q0 = blockIdx.x * 256 * G + threadIdx.x;
    float4 g[G], p[G], m[G], v[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
        const int q = q0 + j * 256;
        if (q < n4) {
            g[j] = reinterpret_cast<const float4*>(a.g)[q];
            p[j] = reinterpret_cast<const float4*>(a.p)[q];
            m[j] = reinterpret_cast<const float4*>(a.m)[q];
            v[j] = reinterpret_cast<const float4*>(a.v)[q];
        }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
        const int q = q0 + j * 256;
        if (q < n4) {
            upd4(p[j], m[j], v[j], g[j], a);
            store4(a, q, p[j], m[j], v[j]);
        }
    }
}

__global__ void __launch_bounds__(256, 8) k_stride(P a) {
    const int n4 = a.n / 4;
    const int stride = gridDim.x * 256;
    int q = blockIdx.x * 256 + threadIdx.x;
    for (; q + stride < n4; q += 2 * stride) {
        const int q2 = q + stride;
        float4 g0 = reinterpret_cast<const float4*>(a.g)[q], p0 = reinterpret_cast<const float4*>(a.p)[q];
        float4 m0 = reinterpret_cast<const float4*>(a.m)[q], v0 = reinterpret_cast<const float4*>(a.v)[q];
        float4 g1 = reinterpret_cast<const float4*>(a.g)[q2], p1 = reinterpret_cast<const float4*>(a.p)[q2];
        float4 m1 = reinterpret_cast<const float4*>(a.m)[q2], v1 = reinterpret_cast<const float4*>(a.v)[q2];
        upd4(p0, m0, v0, g0, a);
        upd4(p1, m1, v1, g1, a);
        store4(a, q, p0, m0, v0);
        store4(a, q2, p1, m1, v1);
    }
    if (q < n4) {
        float4 g0 = reinterpret_cast<const float4*>(a.g)[q], p0 = reinterpret_cast<const float4*>(a.p)[q];
        float4 m0 = reinterpret_cast<const float4*>(a.m)[q], v0 = reinterpret_cast<const float4*>(a.v)[q];
        upd4(p0, m0, v0, g0, a);
        store4(a, q, p0, m0, v0);
    }
}

// ---- V3: TMA bulk loads (cp.async.bulk global -> shared, mbarrier completion)
constexpr int CH = 2048;          // floats per array per stage (8 KB)
constexpr int ST = 2;             // stages
__device__ __forceinline__ void mb_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes));
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned ph) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}"
                 :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(ph));
}
__device__ __forceinline__ void bulk_ld(void* dst, const void* src, unsigned bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                    "r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}

__global__ void __launch_bounds__(256, 2) k_tma(P a) {
    extern __shared__ __align__(128) float sm[];          // [ST][4][CH]
    __shared__ uint64_t bar[ST];
    const int nch = (a.n + CH - 1) / CH;
    if (threadIdx.x == 0) { for (int s = 0; s < ST; ++s) mb_init(&bar[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncthreads();
    auto issue = [&](int c, int s) {
        const int off = c * CH;
        const int cnt = min(CH, a.n - off);
        const unsigned bytes = (unsigned)cnt * 4u;
        mb_expect(&bar[s], 4 * bytes);
        float* d = sm + (size_t)s * 4 * CH;
        bulk_ld(d, a.g + off, bytes, &bar[s]);
        bulk_ld(d + CH, a.p + off, bytes, &bar[s]);
        bulk_ld(d + 2 * CH, a.m + off, bytes, &bar[s]);
        bulk_ld(d + 3 * CH, a.v + off, bytes, &bar[s]);
    };
    int c = blockIdx.x, it = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST && c + s * (int)gridDim.x < nch; ++s) issue(c + s * gridDim.x, s);
    }
    for (; c < nch; c += gridDim.x, ++it) {
        const int s = it % ST;
        mb_wait(&bar[s], (it / ST) & 1);
        const float* d = sm + (size_t)s * 4 * CH;
        const int off = c * CH;
        const int cnt = min(CH, a.n - off);
        for (int i4 = threadIdx.x; i4 < cnt / 4; i4 += 256) {
            float4 g = reinterpret_cast<const float4*>(d)[i4];
            float4 p = reinterpret_cast<const float4*>(d + CH)[i4];
            float4 m = reinterpret_cast<const float4*>(d + 2 * CH)[i4];
            float4 v = reinterpret_cast<const float4*>(d + 3 * CH)[i4];
            upd4(p, m, v, g, a);
            store4(a, off / 4 + i4, p, m, v);
        }
        __syncthreads();   // stage s consumed
        const int cn = c + ST * gridDim.x;
        if (threadIdx.x == 0 && cn < nch) issue(cn, s);
    }
}

__global__ void k_fill(float* x, int n, float val) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = val + 1e-3f * (i & 7);
}

int main() {
    const int n = 1708320;   // cfg1: 854,160 table entries x F=2
    P a;
    a.n = n;
    a.ibc1 = 10.f;
    a.ibc2 = 100.f;
    CK(cudaMalloc(&a.p, n * 4)); CK(cudaMalloc(&a.m, n * 4)); CK(cudaMalloc(&a.v, n * 4)); CK(cudaMalloc(&a.g, n * 4));
    CK(cudaMalloc(&a.h, n * 2));
    const size_t FL = 512ull << 20;
    void* flush;
    CK(cudaMalloc(&flush, FL));
    k_fill<<<1184, 256>>>(a.p, n, 0.1f); k_fill<<<1184, 256>>>(a.m, n, 0.0f); k_fill<<<1184, 256>>>(a.v, n, 0.01f);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int smem3 = ST * 4 * CH * 4;
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[] = {"V0 wave G4 x3", "V1 wave G2 x6", "V2 stride 8/SM", "V3 tma 2/SM", "V4 wave G1 x8"};
    for (int var = 0; var < 5; ++var) {
        std::vector<float> ts;
        for (int r = 0; r < 40; ++r) {
            CK(cudaMemsetAsync(flush, r & 0xff, FL));                 // L2 full of dirty lines
            k_fill<<<1184, 256>>>(a.g, n, 1e-3f);                      // g L2-resident
            cudaEventRecord(e0);
            const int n4 = n / 4;
            if (var == 0) k_wave<4, 3><<<(n4 + 1023) / 1024, 256>>>(a);
            if (var == 1) k_wave<2, 6><<<(n4 + 511) / 512, 256>>>(a);
            if (var == 2) k_stride<<<sms * 8, 256>>>(a);
            if (var == 3) k_tma<<<sms * 2, 256, smem3>>>(a);
            if (var == 4) k_wave<1, 8><<<(n4 + 255) / 256, 256>>>(a);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 5) ts.push_back(ms * 1e3f);
        }
        CK(cudaGetLastError());
        std::sort(ts.begin(), ts.end());
        const double bytes = (double)n * (3 * 4 + 4 * 4 + 2);   // p m v read (g from L2), p m v g write + fp16
        printf("%-16s median %7.2f us  min %7.2f us  (%.0f GB/s on p/m/v/g/h bytes)\n", names[var], ts[ts.size() / 2],
               ts[0], bytes / (ts[ts.size() / 2] * 1e3));
    }
    return 0;
}

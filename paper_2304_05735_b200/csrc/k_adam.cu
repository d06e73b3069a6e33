// k_adam.cu -- step a8: fused multi-object Adam (R18), one launch for
// every object of the batch (blockIdx.y = object slot).  Per object the parameter
// block is [hash tables | MLP]; tables are sparse (an entry with a zero gradient
// this step keeps p, m, v bit-identical), the MLP is dense.
// Writes the fp16 working copy (mixed path) and zeroes the gradients it consumed.
// HBM-bound: 4 B/param read (g) + 28 B/param for touched params (p, m, v r/w,
// fp16 w, g zero) -- see DESIGN.md "Kernels".
#include "romap_internal.cuh"

#include <cstdlib>

bool pdl_enabled() {
    static const bool on = getenv("ROMAP_NO_PDL") == nullptr;
    return on;
}

// one Adam update of 4 consecutive parameters (i0 .. i0+3, all < total);
// returns whether any of them changed (tables are sparse, R18)
__device__ __forceinline__ bool adam4(float4& pp, float4& mm, float4& vv, const float4 gg, int i0, int n_table,
                                      float b1, float b2, float omb1, float omb2, float ibc1, float ibc2, float lr,
                                      float eps, bool& bad) {
    float g[4] = {gg.x, gg.y, gg.z, gg.w}, p[4] = {pp.x, pp.y, pp.z, pp.w}, m[4] = {mm.x, mm.y, mm.z, mm.w},
          v[4] = {vv.x, vv.y, vv.z, vv.w};
    bool any = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float gj = g[j];
        if (i0 + j < n_table && gj == 0.f) continue;      // sparse tables (R18)
        any = true;
        bad |= !isfinite(gj);
        const float mj = b1 * m[j] + omb1 * gj;
        const float vj = b2 * v[j] + omb2 * gj * gj;
        // p -= lr * m_hat / (sqrt(v_hat) + eps), m_hat = m / (1 - b1^t), v_hat = v / (1 - b2^t)
        p[j] = p[j] - lr * (mj * ibc1) / (sqrtf(vj * ibc2) + eps);
        m[j] = mj;
        v[j] = vj;
    }
    pp = make_float4(p[0], p[1], p[2], p[3]);
    mm = make_float4(m[0], m[1], m[2], m[3]);
    vv = make_float4(v[0], v[1], v[2], v[3]);
    return any;
}

constexpr int ADAM_G = 4;   // float4 groups per thread (all loads issued before any math)

// grid (bx, n_objs): block x of object y updates float4 groups
// [x * 256 * ADAM_G, (x + 1) * 256 * ADAM_G) of that object's parameters (g, p,
// m, v of all ADAM_G groups loaded together); the last block of the object to
// finish advances its Adam step counter (step_d[0]; step_d[1] counts finished
// blocks), so no separate launch is needed for the step increment.
// step_d layout: [0] Adam step (i64), [1] finished-block counter (u64), [2] the
// bias corrections 1 / (1 - beta^t) of the NEXT step t = step + 1 as two fp32
// (computed in double, rounded once: by the host at creation / set_params, then
// by the last block of every launch for the following step)
__device__ __forceinline__ float2 bias_corrections(double b1, double b2, long long t) {
    return make_float2((float)(1.0 / (1.0 - pow(b1, (double)t))), (float)(1.0 / (1.0 - pow(b2, (double)t))));
}

__global__ void __launch_bounds__(256, 3) k_adam(CfgDev cfg, const ObjDev* __restrict__ objs, int* __restrict__ nonfinite,
                                                 int write_half) {
    pdl_trigger();
    pdl_wait();                                   // gradients of the fused step (PDL launch)
    const ObjDev& ob = objs[blockIdx.y];
    const float2 bc = *reinterpret_cast<const float2*>(ob.step + 2);
    const float ibc1 = bc.x, ibc2 = bc.y;
    const float b1 = cfg.b1, b2 = cfg.b2, lr = cfg.lr, eps = cfg.eps;
    const float omb1 = 1.0f - b1, omb2 = 1.0f - b2;
    const int n_table = cfg.n_table;
    const int total = cfg.n_table + cfg.n_mlp;
    const int n4 = total / 4;
    float4* p4 = reinterpret_cast<float4*>(ob.p32);
    float4* g4 = reinterpret_cast<float4*>(ob.g32);
    float4* m4 = reinterpret_cast<float4*>(ob.m);
    float4* v4 = reinterpret_cast<float4*>(ob.v);
    bool bad = false;
    const int q0 = blockIdx.x * blockDim.x * ADAM_G + threadIdx.x;
    float4 gg[ADAM_G], pp[ADAM_G], mm[ADAM_G], vv[ADAM_G];
#pragma unroll
    for (int j = 0; j < ADAM_G; ++j) {
        const int q = q0 + j * blockDim.x;
        if (q < n4) {
            gg[j] = g4[q];
            pp[j] = p4[q];
            mm[j] = m4[q];
            vv[j] = v4[q];
        }
    }
#pragma unroll
    for (int j = 0; j < ADAM_G; ++j) {
        const int q = q0 + j * blockDim.x;
        if (q < n4 && adam4(pp[j], mm[j], vv[j], gg[j], 4 * q, n_table, b1, b2, omb1, omb2, ibc1, ibc2, lr, eps, bad)) {
            p4[q] = pp[j];
            m4[q] = mm[j];
            v4[q] = vv[j];
            g4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (write_half) {
                __half2* h2 = reinterpret_cast<__half2*>(ob.p16 + 4 * q);
                h2[0] = __floats2half2_rn(pp[j].x, pp[j].y);
                h2[1] = __floats2half2_rn(pp[j].z, pp[j].w);
            }
        }
    }
    // scalar tail (total % 4 parameters; MLP, dense)
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    if (gt < total - 4 * n4) {
        const int i = 4 * n4 + gt;
        const float gj = ob.g32[i];
        bad |= !isfinite(gj);
        const float mj = b1 * ob.m[i] + omb1 * gj;
        const float vj = b2 * ob.v[i] + omb2 * gj * gj;
        const float p = ob.p32[i] - lr * (mj * ibc1) / (sqrtf(vj * ibc2) + eps);
        ob.p32[i] = p;
        ob.m[i] = mj;
        ob.v[i] = vj;
        ob.g32[i] = 0.f;
        if (write_half) ob.p16[i] = __float2half_rn(p);
    }
    if (bad) atomicOr(nonfinite, 2);
    // every thread of this block has read the bias corrections: count the block;
    // the last one advances the step and prepares the next step's corrections
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned long long* done = reinterpret_cast<unsigned long long*>(ob.step + 1);
        if (atomicAdd(done, 1ull) == (unsigned long long)(gridDim.x - 1)) {
            const long long t = *ob.step + 1;
            *ob.step = t;
            *reinterpret_cast<float2*>(ob.step + 2) = bias_corrections(cfg.b1, cfg.b2, t + 1);
            *done = 0ull;
        }
    }
}

void launch_adam(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, int n_objs, int* nonfinite,
                 bool write_half) {
    if (n_objs == 0) return;
    long long total = (long long)cfg.n_table + cfg.n_mlp;
    // every float4 group of the object covered: 256 threads x ADAM_G groups per block
    int bx = (int)((total / 4 + 256 * ADAM_G - 1) / (256 * ADAM_G));
    if (bx < 1) bx = 1;
    cudaLaunchConfig_t lcfg = {};
    lcfg.gridDim = dim3(bx, n_objs);
    lcfg.blockDim = dim3(256);
    lcfg.dynamicSmemBytes = 0;
    lcfg.stream = lc.st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lcfg.attrs = attr;
    lcfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&lcfg, k_adam, cfg, objs, nonfinite, write_half ? 1 : 0);
}

__global__ void __launch_bounds__(256) k_zero_grads(CfgDev cfg, const ObjDev* __restrict__ objs) {
    const ObjDev& ob = objs[blockIdx.y];
    const int total = cfg.n_table + cfg.n_mlp;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) ob.g32[i] = 0.f;
}

void launch_zero_grads(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, int n_objs) {
    if (n_objs == 0) return;
    dim3 grid(64, n_objs);
    k_zero_grads<<<grid, 256, 0, lc.st>>>(cfg, objs);
}

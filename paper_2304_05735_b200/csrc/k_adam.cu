// k_adam.cu -- step a8: fused multi-object Adam (R18), one launch for
// every object of the batch (blockIdx.y = object slot).  Per object the parameter
// block is [hash tables | MLP]; tables are sparse (an entry with a zero gradient
// this step keeps p, m, v bit-identical), the MLP is dense.
// Writes the fp16 working copy (mixed path) and zeroes the gradients it consumed.
// HBM-bound: 4 B/param read (g) + 28 B/param for touched params (p, m, v r/w,
// fp16 w, g zero) -- see DESIGN.md "Kernels".
#include "romap_internal.cuh"

__global__ void __launch_bounds__(256) k_adam(CfgDev cfg, const ObjDev* __restrict__ objs, int* __restrict__ nonfinite,
                                              int write_half) {
    const ObjDev& ob = objs[blockIdx.y];
    const long long t = *ob.step + 1;
    // bias corrections in double, rounded once
    const float bc1 = (float)(1.0 - pow((double)cfg.b1, (double)t));
    const float bc2 = (float)(1.0 - pow((double)cfg.b2, (double)t));
    const float b1 = cfg.b1, b2 = cfg.b2, lr = cfg.lr, eps = cfg.eps;
    const float omb1 = 1.0f - b1, omb2 = 1.0f - b2;
    const int n_table = cfg.n_table;
    const int total = cfg.n_table + cfg.n_mlp;
    // vectorised over 4 params (n_table is even; handle tails scalar)
    const int n4 = total / 4;
    float4* p4 = reinterpret_cast<float4*>(ob.p32);
    float4* g4 = reinterpret_cast<float4*>(ob.g32);
    float4* m4 = reinterpret_cast<float4*>(ob.m);
    float4* v4 = reinterpret_cast<float4*>(ob.v);
    bool bad = false;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n4 + (total - n4 * 4); q += gridDim.x * blockDim.x) {
        int i0, cnt;
        float g[4], p[4], m[4], v[4];
        if (q < n4) {
            i0 = 4 * q;
            cnt = 4;
            float4 gg = g4[q];
            g[0] = gg.x; g[1] = gg.y; g[2] = gg.z; g[3] = gg.w;
            if (gg.x == 0.f && gg.y == 0.f && gg.z == 0.f && gg.w == 0.f && i0 + 4 <= n_table) continue;
            float4 pp = p4[q], mm = m4[q], vv = v4[q];
            p[0] = pp.x; p[1] = pp.y; p[2] = pp.z; p[3] = pp.w;
            m[0] = mm.x; m[1] = mm.y; m[2] = mm.z; m[3] = mm.w;
            v[0] = vv.x; v[1] = vv.y; v[2] = vv.z; v[3] = vv.w;
        } else {
            i0 = 4 * n4 + (q - n4);
            cnt = 1;
            g[0] = ob.g32[i0];
            p[0] = ob.p32[i0];
            m[0] = ob.m[i0];
            v[0] = ob.v[i0];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (j >= cnt) break;
            int i = i0 + j;
            float gj = g[j];
            if (i < n_table && gj == 0.f) continue;      // sparse tables (R18)
            bad |= !isfinite(gj);
            float mj = b1 * m[j] + omb1 * gj;
            float vj = b2 * v[j] + omb2 * gj * gj;
            float mh = mj / bc1;
            float vh = vj / bc2;
            p[j] = p[j] - lr * mh / (sqrtf(vh) + eps);
            m[j] = mj;
            v[j] = vj;
        }
        if (cnt == 4) {
            p4[q] = make_float4(p[0], p[1], p[2], p[3]);
            m4[q] = make_float4(m[0], m[1], m[2], m[3]);
            v4[q] = make_float4(v[0], v[1], v[2], v[3]);
            g4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (write_half) {
                __half2* h2 = reinterpret_cast<__half2*>(ob.p16 + i0);
                h2[0] = __floats2half2_rn(p[0], p[1]);
                h2[1] = __floats2half2_rn(p[2], p[3]);
            }
        } else {
            ob.p32[i0] = p[0];
            ob.m[i0] = m[0];
            ob.v[i0] = v[0];
            ob.g32[i0] = 0.f;
            if (write_half) ob.p16[i0] = __float2half_rn(p[0]);
        }
    }
    if (bad) atomicOr(nonfinite, 2);
}

void launch_adam(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, int n_objs, int* nonfinite,
                 bool write_half) {
    if (n_objs == 0) return;
    long long total = (long long)cfg.n_table + cfg.n_mlp;
    int per_obj = (int)((total / 4 + 255) / 256);
    // a few waves over the SMs in total
    int target = (lc.num_sms * 8 + n_objs - 1) / n_objs;
    int bx = per_obj < target ? per_obj : target;
    if (bx < 1) bx = 1;
    dim3 grid(bx, n_objs);
    k_adam<<<grid, 256, 0, lc.st>>>(cfg, objs, nonfinite, write_half ? 1 : 0);
}

__global__ void k_step_inc(const ObjDev* __restrict__ objs, int n_objs) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_objs) *objs[i].step += 1;
}

void launch_step_inc(const LaunchCtx& lc, const ObjDev* objs, int n_objs) {
    if (n_objs > 0) k_step_inc<<<(n_objs + 127) / 128, 128, 0, lc.st>>>(objs, n_objs);
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

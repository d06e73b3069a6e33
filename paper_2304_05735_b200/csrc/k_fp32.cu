// k_fp32.cu -- the fp32 (parity) training path and the inference kernels.
//
//   k_fwd_fp32     a2-a4: stratified / midpoint samples, hash encode forward
//                  (PAPER.md:124 via instant-NGP [21]), SH, MLP forward
//                  (thread per sample; weights broadcast from L1/L2)
//   k_render_loss  a5: volume rendering (Eq. 6) fused with the
//                  object-tailored loss (Eqs. 7-11) and its
//                  backward, warp per ray, multiplicative warp scan for T_i and a
//                  reverse warp scan for the suffix sums of the backward
//   k_bwd_fp32     a6-a7: MLP backward (dW reduced per 128-sample tile in shared
//                  memory, one atomic per weight per tile) and hash scatter-add
//                  (float2 atomics)
//   k_composite    inference compositing over black (R12/R20)
//   k_query        density query (R21)
// The fp32 path is the parity reference of the CUDA side (BASELINE cfg0); the
// mixed path (k_fused_mixed.cu) is the performance path.
#include "romap_internal.cuh"

__device__ __forceinline__ float relu(float x) { return x > 0.f ? x : 0.f; }

// hash encode forward of one sample: feat[2*l + f]
__device__ __forceinline__ void encode_fp32(const CfgDev& cfg, const float* __restrict__ table, const float u[3],
                                            float feat[ROMAP_MAX_LF]) {
#pragma unroll
    for (int l = 0; l < ROMAP_MAX_LEVELS; ++l) {
        feat[2 * l] = 0.f;
        feat[2 * l + 1] = 0.f;
        if (l < cfg.L) {
            int res = cfg.res[l];
            Cell cl = grid_cell(u, res);
            const float2* tb = reinterpret_cast<const float2*>(table) + cfg.off[l];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                int e = corner_entry(cl, b, res, cfg.dense[l], cfg.T);
                float w = corner_weight(cl, b);
                float2 v = __ldg(tb + e);
                feat[2 * l] += w * v.x;
                feat[2 * l + 1] += w * v.y;
            }
        }
    }
}

struct FwdOut { float sigma, rgb[3]; };

// MLP forward of one sample (R1/R3/R4); optionally stores activations (train)
__device__ __forceinline__ FwdOut mlp_fwd_fp32(const CfgDev& cfg, const float* __restrict__ mlp,
                                               const float feat[ROMAP_MAX_LF], const float sh[16], float* act,
                                               long long stride) {
    const float* W1 = mlp + cfg.w_off[0];
    const float* W2 = mlp + cfg.w_off[1];
    const float* W3 = mlp + cfg.w_off[2];
    const float* W4 = mlp + cfg.w_off[3];
    const float* W5 = mlp + cfg.w_off[4];
    const int LF = cfg.LF;
    float h[ROMAP_WIDTH];
#pragma unroll
    for (int j = 0; j < ROMAP_WIDTH; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < ROMAP_MAX_LF; ++k)
            if (k < LF) acc += __ldg(W1 + j * LF + k) * feat[k];
        h[j] = relu(acc);
    }
    float cin[ROMAP_CIN];
#pragma unroll
    for (int j = 0; j < ROMAP_DOUT; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < ROMAP_WIDTH; ++k) acc += __ldg(W2 + j * ROMAP_WIDTH + k) * h[k];
        cin[j] = acc;
    }
#pragma unroll
    for (int j = 0; j < ROMAP_SH; ++j) cin[ROMAP_DOUT + j] = sh[j];
    if (act) {
        float* a = act;
        for (int k = 0; k < LF; ++k) a[(long long)k * stride] = feat[k];
        a += (long long)LF * stride;
#pragma unroll
        for (int k = 0; k < ROMAP_WIDTH; ++k) a[(long long)k * stride] = h[k];
        a += (long long)ROMAP_WIDTH * stride;
#pragma unroll
        for (int k = 0; k < ROMAP_DOUT; ++k) a[(long long)k * stride] = cin[k];
    }
    float g1[ROMAP_WIDTH];
#pragma unroll
    for (int j = 0; j < ROMAP_WIDTH; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < ROMAP_CIN; ++k) acc += __ldg(W3 + j * ROMAP_CIN + k) * cin[k];
        g1[j] = relu(acc);
    }
    float g2[ROMAP_WIDTH];
#pragma unroll
    for (int j = 0; j < ROMAP_WIDTH; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < ROMAP_WIDTH; ++k) acc += __ldg(W4 + j * ROMAP_WIDTH + k) * g1[k];
        g2[j] = relu(acc);
    }
    if (act) {
        float* a = act + (long long)(LF + ROMAP_WIDTH + ROMAP_DOUT) * stride;
#pragma unroll
        for (int k = 0; k < ROMAP_WIDTH; ++k) a[(long long)k * stride] = g1[k];
        a += (long long)ROMAP_WIDTH * stride;
#pragma unroll
        for (int k = 0; k < ROMAP_WIDTH; ++k) a[(long long)k * stride] = g2[k];
    }
    FwdOut o;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < ROMAP_WIDTH; ++k) acc += __ldg(W5 + j * ROMAP_WIDTH + k) * g2[k];
        o.rgb[j] = 1.0f / (1.0f + expf(-acc));
    }
    o.sigma = density_act(cin[0], cfg.density_act);
    return o;
}

// activation layout per sample (SoA, stride = total samples): feat[LF] h1[64] r[16] g1[64] g2[64]
#define ACT_ROWS(LF) ((LF) + ROMAP_WIDTH + ROMAP_DOUT + ROMAP_WIDTH + ROMAP_WIDTH)

__device__ __forceinline__ void sample_geo_any(const CfgDev& cfg, const ObjDev& ob, const RayRec& rr, int ray_local,
                                               int i, bool midpoint, float& dist, float& delta, float u[3]) {
    if (midpoint) {
        float Dl = __fdiv_rn(__fsub_rn(rr.tf, rr.tn), (float)cfg.N);
        dist = sample_dist(rr.tn, Dl, i, 0.5f);
        delta = Dl;
        sample_u(rr.o, rr.d, ob.a, dist, u);
    } else {
        unsigned long long pre = rng_prefix(cfg.seed, ob.obj_id, *ob.step + 1);
        sample_geometry(rr, i, cfg.N, pre, ray_local, ob.a, dist, delta, u);
    }
}

__global__ void __launch_bounds__(128) k_fwd_fp32(CfgDev cfg, const ObjDev* __restrict__ objs,
                                                  const RayRec* __restrict__ rays, int n_rays, int midpoint,
                                                  float* __restrict__ sigma, float* __restrict__ rgb,
                                                  float* __restrict__ dist_o, float* __restrict__ delta_o,
                                                  float* __restrict__ act, long long stride) {
    long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int N = cfg.N;
    long long ray = s / N;
    int i = (int)(s - ray * N);
    if (ray >= n_rays) return;
    const RayRec rr = rays[ray];
    if (!(rr.flags & RF_ACTIVE)) {
        sigma[s] = 0.f;
        rgb[3 * s] = rgb[3 * s + 1] = rgb[3 * s + 2] = 0.f;
        dist_o[s] = 0.f;
        delta_o[s] = 0.f;
        return;
    }
    const ObjDev& ob = objs[rr.slot];
    float dist, delta, u[3];
    sample_geo_any(cfg, ob, rr, (int)(ray - ob.ray_begin), i, midpoint, dist, delta, u);
    float feat[ROMAP_MAX_LF];
    encode_fp32(cfg, ob.p32, u, feat);
    float sh[16];
    sh4(rr.d, sh);
    FwdOut o = mlp_fwd_fp32(cfg, ob.p32 + cfg.n_table, feat, sh, act ? act + s : nullptr, stride);
    sigma[s] = o.sigma;
    rgb[3 * s] = o.rgb[0];
    rgb[3 * s + 1] = o.rgb[1];
    rgb[3 * s + 2] = o.rgb[2];
    dist_o[s] = dist;
    delta_o[s] = delta;
}

void launch_fwd_fp32(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, const RayRec* rays, int n_rays,
                     bool train, bool midpoint, float* sigma, float* rgb, float* dist, float* delta, float* act,
                     long long act_stride) {
    long long S = (long long)n_rays * cfg.N;
    if (S == 0) return;
    k_fwd_fp32<<<(unsigned)((S + 127) / 128), 128, 0, lc.st>>>(cfg, objs, rays, n_rays, midpoint ? 1 : 0, sigma, rgb,
                                                                dist, delta, train ? act : nullptr, act_stride);
}

// ---------------------------------------------------------------------------
// a5: volume rendering + loss + render backward, warp per ray
#define RL_MAXC 4   // samples per lane: N <= 128

__global__ void __launch_bounds__(256) k_render_loss(CfgDev cfg, const ObjDev* __restrict__ objs,
                                                     const RayRec* __restrict__ rays, int n_rays,
                                                     const float* __restrict__ sigma, const float* __restrict__ rgb,
                                                     const float* __restrict__ dist, const float* __restrict__ delta,
                                                     float* __restrict__ dsigma, float* __restrict__ drgb,
                                                     double* __restrict__ loss_acc, int* __restrict__ nonfinite,
                                                     DetBufs det) {
    __shared__ float sm_loss[8][4];
    __shared__ int sm_slot[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int ray = blockIdx.x * 8 + wid;
    const int N = cfg.N;
    const int C = N >= 32 ? N / 32 : 1;
    float lossv[4] = {0.f, 0.f, 0.f, 0.f};
    int slot = -1;
    if (ray < n_rays) {
        const RayRec rr = rays[ray];
        slot = rr.slot;
        if (rr.flags & RF_ACTIVE) {
            const ObjDev& ob = objs[rr.slot];
            const long long base = (long long)ray * N;
            const int i0 = lane * C;
            float al[RL_MAXC], sg[RL_MAXC], dl[RL_MAXC], ds[RL_MAXC], cc[RL_MAXC][3], w[RL_MAXC], Tn1[RL_MAXC];
            float prod = 1.f;
#pragma unroll
            for (int j = 0; j < RL_MAXC; ++j) {
                int i = i0 + j;
                bool ok = j < C && i < N;
                sg[j] = ok ? sigma[base + i] : 0.f;
                dl[j] = ok ? delta[base + i] : 0.f;
                ds[j] = ok ? dist[base + i] : 0.f;
#pragma unroll
                for (int k = 0; k < 3; ++k) cc[j][k] = ok ? rgb[3 * (base + i) + k] : 0.f;
                float x = sg[j] * dl[j];
                al[j] = expf(-x);
                prod *= al[j];
            }
            // exclusive multiplicative scan over lanes: T at the start of this lane's chunk
            float incl = prod;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                float v = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl *= v;
            }
            float T = __shfl_up_sync(0xffffffffu, incl, 1);
            if (lane == 0) T = 1.f;
            const float TN = __shfl_sync(0xffffffffu, incl, 31);
            float Cs[3] = {0.f, 0.f, 0.f}, D = 0.f, A = 0.f, ssum = 0.f;
#pragma unroll
            for (int j = 0; j < RL_MAXC; ++j) {
                float o = -expm1f(-(sg[j] * dl[j]));   // o_j = 1 - exp(-sigma delta)
                w[j] = T * o;
                T *= al[j];
                Tn1[j] = T;
#pragma unroll
                for (int k = 0; k < 3; ++k) Cs[k] += w[j] * cc[j][k];
                D += w[j] * ds[j];
                A += w[j];
                ssum += sg[j];
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
                for (int k = 0; k < 3; ++k) Cs[k] += __shfl_xor_sync(0xffffffffu, Cs[k], off);
                D += __shfl_xor_sync(0xffffffffu, D, off);
                ssum += __shfl_xor_sync(0xffffffffu, ssum, off);
            }
            const int cls = rr.flags & RF_CLS_MASK;
            const bool has_depth = (rr.flags & RF_HAS_DEPTH) != 0;
            float bgc[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) bgc[k] = (cls == CLS_OBJ && cfg.obj_bg == 1) ? 0.f : rr.bg[k];
            float e[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                float Cf = Cs[k] + TN * bgc[k];                     // R14
                e[k] = Cf - (cls == CLS_OBJ ? rr.tgt[k] : rr.bg[k]);
            }
            const float ne = sqrtf(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
            const float invB = 1.0f / (float)ob.n_rays;               // R16
            float gC[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) gC[k] = ne > 0.f ? e[k] / ne * invB : 0.f;
            float gD = 0.f, ed = 0.f;
            if (has_depth) {
                ed = D - rr.depth;
                gD = ed > 0.f ? cfg.lambda_depth * invB : (ed < 0.f ? -cfg.lambda_depth * invB : 0.f);
            }
            if (cls == CLS_OBJ) lossv[0] = ne; else lossv[1] = ne;
            lossv[2] = has_depth ? fabsf(ed) : 0.f;
            lossv[3] = cls == CLS_BG ? ssum : 0.f;
            if (!isfinite(ne) || !isfinite(ssum) || !isfinite(D)) {
                if (lane == 0) atomicOr(nonfinite, 1);
            }
            const float gCb = gC[0] * bgc[0] + gC[1] * bgc[1] + gC[2] * bgc[2];
            // backward: suffix sums S_i = sum_{k>i} w_k (gC.c_k), Sd_i = sum_{k>i} w_k d_k
            float gc[RL_MAXC], ls = 0.f, lsd = 0.f;
#pragma unroll
            for (int j = 0; j < RL_MAXC; ++j) {
                gc[j] = gC[0] * cc[j][0] + gC[1] * cc[j][1] + gC[2] * cc[j][2];
                ls += w[j] * gc[j];
                lsd += w[j] * ds[j];
            }
            float rs = ls, rsd = lsd;   // inclusive suffix over lanes
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                float v = __shfl_down_sync(0xffffffffu, rs, off);
                float vd = __shfl_down_sync(0xffffffffu, rsd, off);
                if (lane + off < 32) { rs += v; rsd += vd; }
            }
            float S = __shfl_down_sync(0xffffffffu, rs, 1);
            float Sd = __shfl_down_sync(0xffffffffu, rsd, 1);
            if (lane == 31) { S = 0.f; Sd = 0.f; }
            const float dens = cls == CLS_BG ? cfg.lambda_density * invB : 0.f;   // Eq. 10 gradient
            float dsg[RL_MAXC];
#pragma unroll
            for (int j = RL_MAXC - 1; j >= 0; --j) {
                dsg[j] = dl[j] * (Tn1[j] * gc[j] - S - TN * gCb) + dl[j] * gD * (Tn1[j] * ds[j] - Sd) + dens;
                S += w[j] * gc[j];
                Sd += w[j] * ds[j];
            }
#pragma unroll
            for (int j = 0; j < RL_MAXC; ++j) {
                int i = i0 + j;
                if (j < C && i < N) {
                    dsigma[base + i] = dsg[j];
#pragma unroll
                    for (int k = 0; k < 3; ++k) drgb[3 * (base + i) + k] = w[j] * gC[k];
                }
            }
        } else {
            const long long base = (long long)ray * N;
            for (int i = lane; i < N; i += 32) {
                dsigma[base + i] = 0.f;
                drgb[3 * (base + i)] = drgb[3 * (base + i) + 1] = drgb[3 * (base + i) + 2] = 0.f;
            }
        }
    }
    // deterministic mode: per-ray loss sums, reduced in ray order by k_det.cu
    if (det.ray_loss) {
        if (lane == 0 && ray < n_rays)
            *reinterpret_cast<float4*>(det.ray_loss + 4LL * ray) = make_float4(lossv[0], lossv[1], lossv[2], lossv[3]);
        return;
    }
    // per-object loss sums: block reduction when all warps share one slot
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) sm_loss[wid][k] = lossv[k];
        sm_slot[wid] = slot;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        int k = threadIdx.x;
        int s0 = sm_slot[0];
        bool uniform = true;
        for (int w2 = 1; w2 < 8; ++w2) uniform &= (sm_slot[w2] == s0 || sm_slot[w2] < 0);
        if (uniform) {
            float acc = 0.f;
            for (int w2 = 0; w2 < 8; ++w2) acc += sm_loss[w2][k];
            if (s0 >= 0 && acc != 0.f) atomicAdd(loss_acc + 4 * s0 + k, (double)acc);
        } else {
            for (int w2 = 0; w2 < 8; ++w2)
                if (sm_slot[w2] >= 0 && sm_loss[w2][k] != 0.f) atomicAdd(loss_acc + 4 * sm_slot[w2] + k, (double)sm_loss[w2][k]);
        }
    }
}

void launch_render_loss(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, const RayRec* rays, int n_rays,
                        const float* sigma, const float* rgb, const float* dist, const float* delta, float* dsigma,
                        float* drgb, double* loss_acc, int* nonfinite, const DetBufs& det) {
    if (n_rays == 0) return;
    k_render_loss<<<(n_rays + 7) / 8, 256, 0, lc.st>>>(cfg, objs, rays, n_rays, sigma, rgb, dist, delta, dsigma, drgb,
                                                       loss_acc, nonfinite, det);
}

// ---------------------------------------------------------------------------
// a6/a7: MLP backward + hash scatter, block = 128 consecutive samples of one object
#define SM_LD 65

// dW[j][k] += sum_s delta[s][j] * in[s][k] over the tile, one atomic per weight
// (store: the deterministic mode's per-tile partial, plain stores)
__device__ __forceinline__ void tile_dw(const float* sm_d, const float* sm_i, int OUT, int IN, float* gW,
                                        bool store = false) {
    for (int e = threadIdx.x; e < OUT * IN; e += blockDim.x) {
        int j = e / IN, k = e - j * IN;
        float acc = 0.f;
#pragma unroll 8
        for (int s = 0; s < ROMAP_TILE; ++s) acc += sm_d[s * SM_LD + j] * sm_i[s * SM_LD + k];
        if (store) gW[e] = acc;
        else if (acc != 0.f) atomicAdd(gW + e, acc);
    }
}

__global__ void __launch_bounds__(128) k_bwd_fp32(CfgDev cfg, const ObjDev* __restrict__ objs,
                                                  const RayRec* __restrict__ rays, int n_rays,
                                                  const float* __restrict__ sigma, const float* __restrict__ rgb,
                                                  const float* __restrict__ dsigma, const float* __restrict__ drgb,
                                                  const float* __restrict__ act, long long stride, DetBufs det) {
    extern __shared__ float smem[];
    float* sm_d = smem;                       // [128][65]
    float* sm_i = smem + ROMAP_TILE * SM_LD;  // [128][65]
    const int t = threadIdx.x;
    const long long s = (long long)blockIdx.x * ROMAP_TILE + t;
    const int N = cfg.N;
    const long long ray = s / N;
    const int i = (int)(s - ray * N);
    const RayRec rr = rays[ray];
    const int slot = rays[(long long)blockIdx.x * ROMAP_TILE / N].slot;   // block-uniform (host aligns slots)
    const ObjDev& ob = objs[slot];
    const bool active = (rr.flags & RF_ACTIVE) != 0;
    const float* mlp = ob.p32 + cfg.n_table;
    const bool dst = det.dw != nullptr;            // deterministic mode: per-tile partials, records
    float* gm = dst ? det.dw + (long long)blockIdx.x * cfg.n_mlp : ob.g32 + cfg.n_table;
    const int LF = cfg.LF;
    const float* a_feat = act + s;
    const float* a_h1 = a_feat + (long long)LF * stride;
    const float* a_r = a_h1 + (long long)ROMAP_WIDTH * stride;
    const float* a_g1 = a_r + (long long)ROMAP_DOUT * stride;
    const float* a_g2 = a_g1 + (long long)ROMAP_WIDTH * stride;
    const float* W1 = mlp + cfg.w_off[0];
    const float* W2 = mlp + cfg.w_off[1];
    const float* W3 = mlp + cfg.w_off[2];
    const float* W4 = mlp + cfg.w_off[3];
    const float* W5 = mlp + cfg.w_off[4];
    float* sd = sm_d + t * SM_LD;
    float* si = sm_i + t * SM_LD;

    // colour output: dL/dcraw = dL/dc * c (1 - c)
    float dc[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float c = active ? rgb[3 * s + k] : 0.f;
        dc[k] = active ? drgb[3 * s + k] * c * (1.f - c) : 0.f;
        sd[k] = dc[k];
    }
    float v64[ROMAP_WIDTH];
#pragma unroll
    for (int k = 0; k < ROMAP_WIDTH; ++k) { v64[k] = active ? a_g2[(long long)k * stride] : 0.f; si[k] = v64[k]; }
    __syncthreads();
    tile_dw(sm_d, sm_i, 3, ROMAP_WIDTH, gm + cfg.w_off[4], dst);
    __syncthreads();
    // dg2 = W5^T dc . (g2 > 0)
    float dg[ROMAP_WIDTH];
#pragma unroll
    for (int k = 0; k < ROMAP_WIDTH; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 3; ++j) acc += __ldg(W5 + j * ROMAP_WIDTH + k) * dc[j];
        dg[k] = v64[k] > 0.f ? acc : 0.f;
        sd[k] = dg[k];
    }
#pragma unroll
    for (int k = 0; k < ROMAP_WIDTH; ++k) { v64[k] = active ? a_g1[(long long)k * stride] : 0.f; si[k] = v64[k]; }
    __syncthreads();
    tile_dw(sm_d, sm_i, ROMAP_WIDTH, ROMAP_WIDTH, gm + cfg.w_off[3], dst);
    __syncthreads();
    // dg1 = W4^T dg2 . (g1 > 0)
    float dg1[ROMAP_WIDTH];
#pragma unroll
    for (int k = 0; k < ROMAP_WIDTH; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < ROMAP_WIDTH; ++j) acc += __ldg(W4 + j * ROMAP_WIDTH + k) * dg[j];
        dg1[k] = v64[k] > 0.f ? acc : 0.f;
        sd[k] = dg1[k];
    }
    // colour-net input [r || sh]
    float sh[16];
    sh4(rr.d, sh);
    float r0 = 0.f;
#pragma unroll
    for (int k = 0; k < ROMAP_DOUT; ++k) {
        float v = active ? a_r[(long long)k * stride] : 0.f;
        if (k == 0) r0 = v;
        si[k] = v;
    }
#pragma unroll
    for (int k = 0; k < ROMAP_SH; ++k) si[ROMAP_DOUT + k] = active ? sh[k] : 0.f;
    __syncthreads();
    tile_dw(sm_d, sm_i, ROMAP_WIDTH, ROMAP_CIN, gm + cfg.w_off[2], dst);
    __syncthreads();
    // dr = (W3^T dg1)[:16]; dr0 += dsigma * act'(r0)
    float dr[ROMAP_DOUT];
#pragma unroll
    for (int k = 0; k < ROMAP_DOUT; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < ROMAP_WIDTH; ++j) acc += __ldg(W3 + j * ROMAP_CIN + k) * dg1[j];
        dr[k] = acc;
    }
    if (active) dr[0] += dsigma[s] * density_act_grad(r0, sigma[s], cfg.density_act);
#pragma unroll
    for (int k = 0; k < ROMAP_DOUT; ++k) sd[k] = active ? dr[k] : 0.f;
#pragma unroll
    for (int k = 0; k < ROMAP_WIDTH; ++k) { v64[k] = active ? a_h1[(long long)k * stride] : 0.f; si[k] = v64[k]; }
    __syncthreads();
    tile_dw(sm_d, sm_i, ROMAP_DOUT, ROMAP_WIDTH, gm + cfg.w_off[1], dst);
    __syncthreads();
    // dh1 = W2^T dr . (h1 > 0)
#pragma unroll
    for (int k = 0; k < ROMAP_WIDTH; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < ROMAP_DOUT; ++j) acc += __ldg(W2 + j * ROMAP_WIDTH + k) * dr[j];
        dg[k] = (active && v64[k] > 0.f) ? acc : 0.f;
        sd[k] = dg[k];
    }
    float feat[ROMAP_MAX_LF];
#pragma unroll
    for (int k = 0; k < ROMAP_MAX_LF; ++k) {
        feat[k] = (k < LF && active) ? a_feat[(long long)k * stride] : 0.f;
        if (k < LF) si[k] = feat[k];
    }
    __syncthreads();
    tile_dw(sm_d, sm_i, ROMAP_WIDTH, LF, gm + cfg.w_off[0], dst);
    // dfeat = W1^T dh1
    if (!active) {
        if (dst)
            for (int r8 = 0; r8 < cfg.L * 8; ++r8) det.key[s * cfg.L * 8 + r8] = DET_NO_KEY;
        return;
    }
    float dfeat[ROMAP_MAX_LF];
#pragma unroll
    for (int k = 0; k < ROMAP_MAX_LF; ++k) {
        float acc = 0.f;
        if (k < LF) {
#pragma unroll
            for (int j = 0; j < ROMAP_WIDTH; ++j) acc += __ldg(W1 + j * LF + k) * dg[j];
        }
        dfeat[k] = acc;
    }
    // a7: hash scatter-add (recompute the sample position and cells)
    float dist, delta, u[3];
    unsigned long long pre = rng_prefix(cfg.seed, ob.obj_id, *ob.step + 1);
    sample_geometry(rr, i, N, pre, (int)(ray - ob.ray_begin), ob.a, dist, delta, u);
    float2* gt = reinterpret_cast<float2*>(ob.g32);
#pragma unroll
    for (int l = 0; l < ROMAP_MAX_LEVELS; ++l) {
        if (l < cfg.L) {
            int res = cfg.res[l];
            Cell cl = grid_cell(u, res);
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                int e = corner_entry(cl, b, res, cfg.dense[l], cfg.T);
                float w = corner_weight(cl, b);
                if (dst) {
                    const long long rec = (s * cfg.L + l) * 8 + b;
                    det.key[rec] = ((unsigned long long)slot << 32) | (unsigned long long)(cfg.off[l] + e);
                    det.val[rec] = make_float2(w * dfeat[2 * l], w * dfeat[2 * l + 1]);
                } else {
                    red_add_f2(gt + cfg.off[l] + e, w * dfeat[2 * l], w * dfeat[2 * l + 1]);
                }
            }
        }
    }
}

void launch_bwd_fp32(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, const RayRec* rays, int n_rays,
                     const float* sigma, const float* rgb, const float* dsigma, const float* drgb, const float* act,
                     long long act_stride, const DetBufs& det) {
    long long S = (long long)n_rays * cfg.N;
    if (S == 0) return;
    size_t smem = 2 * ROMAP_TILE * SM_LD * sizeof(float);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_bwd_fp32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    k_bwd_fp32<<<(unsigned)(S / ROMAP_TILE), ROMAP_TILE, smem, lc.st>>>(cfg, objs, rays, n_rays, sigma, rgb, dsigma,
                                                                         drgb, act, act_stride, det);
}

// ---------------------------------------------------------------------------
// inference compositing over black (R12, R20): warp per ray
__global__ void __launch_bounds__(256) k_composite(int N, const RayRec* __restrict__ rays, int n_rays,
                                                   const float* __restrict__ sigma, const float* __restrict__ rgb,
                                                   const float* __restrict__ dist, const float* __restrict__ delta,
                                                   float* __restrict__ out_rgb, float* __restrict__ out_depth,
                                                   float* __restrict__ out_opa, const int* __restrict__ out_idx) {
    const int lane = threadIdx.x & 31;
    const int ray = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (ray >= n_rays) return;
    const RayRec rr = rays[ray];
    float Cs[3] = {0.f, 0.f, 0.f}, D = 0.f, A = 0.f;
    if (rr.flags & RF_ACTIVE) {
        const int C = N >= 32 ? N / 32 : 1;
        const long long base = (long long)ray * N;
        const int i0 = lane * C;
        float al[RL_MAXC], o[RL_MAXC];
        float prod = 1.f;
#pragma unroll
        for (int j = 0; j < RL_MAXC; ++j) {
            int i = i0 + j;
            bool ok = j < C && i < N;
            float x = ok ? sigma[base + i] * delta[base + i] : 0.f;
            al[j] = expf(-x);
            o[j] = -expm1f(-x);
            prod *= al[j];
        }
        float incl = prod;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            float v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl *= v;
        }
        float T = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) T = 1.f;
#pragma unroll
        for (int j = 0; j < RL_MAXC; ++j) {
            int i = i0 + j;
            if (j < C && i < N) {
                float w = T * o[j];
#pragma unroll
                for (int k = 0; k < 3; ++k) Cs[k] += w * rgb[3 * (base + i) + k];
                D += w * dist[base + i];
                A += w;
            }
            T *= al[j];
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
            for (int k = 0; k < 3; ++k) Cs[k] += __shfl_xor_sync(0xffffffffu, Cs[k], off);
            D += __shfl_xor_sync(0xffffffffu, D, off);
            A += __shfl_xor_sync(0xffffffffu, A, off);
        }
    }
    if (lane == 0) {
        const int o = out_idx ? out_idx[ray] : ray;     // compacted rays write to their pixel
        if (out_rgb) { out_rgb[3 * o] = Cs[0]; out_rgb[3 * o + 1] = Cs[1]; out_rgb[3 * o + 2] = Cs[2]; }
        if (out_depth) out_depth[o] = D;
        if (out_opa) out_opa[o] = A;
    }
}

void launch_composite(const LaunchCtx& lc, int N, const RayRec* rays, int n_rays, const float* sigma,
                      const float* rgb, const float* dist, const float* delta, float* out_rgb, float* out_depth,
                      float* out_opacity, const int* out_idx) {
    if (n_rays == 0) return;
    k_composite<<<(n_rays + 7) / 8, 256, 0, lc.st>>>(N, rays, n_rays, sigma, rgb, dist, delta, out_rgb, out_depth,
                                                     out_opacity, out_idx);
}

// render: the rays that hit the box, packed (order arbitrary; out_idx keeps the pixel)
__global__ void __launch_bounds__(256) k_compact_rays(const RayRec* __restrict__ rays, int n, RayRec* __restrict__ out,
                                                      int* __restrict__ idx, int* __restrict__ count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool act = i < n && (rays[i].flags & RF_ACTIVE);
    const unsigned m = __ballot_sync(0xffffffffu, act);
    int base = 0;
    if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(count, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (act) {
        const int pos = base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u));
        out[pos] = rays[i];
        idx[pos] = i;
    }
}

void launch_compact_rays(const LaunchCtx& lc, const RayRec* rays, int n, RayRec* out, int* idx, int* count) {
    if (n > 0) k_compact_rays<<<(n + 255) / 256, 256, 0, lc.st>>>(rays, n, out, idx, count);
}

// ---------------------------------------------------------------------------
// a10: density query (R21): sigma at object-frame points, 0 outside [-a, a]
__global__ void __launch_bounds__(128) k_query(CfgDev cfg, const ObjDev* __restrict__ obj,
                                               const float* __restrict__ xyz, long long n,
                                               float* __restrict__ out) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const ObjDev& ob = *obj;
    float x[3], u[3];
    bool inside = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        x[k] = xyz[3 * p + k];
        inside &= fabsf(x[k]) <= ob.a[k];
        float v = __fdiv_rn(__fadd_rn(x[k], ob.a[k]), __fadd_rn(ob.a[k], ob.a[k]));
        u[k] = fminf(fmaxf(v, 0.f), 1.f);
    }
    if (!inside) { out[p] = 0.f; return; }
    float feat[ROMAP_MAX_LF];
    encode_fp32(cfg, ob.p32, u, feat);
    const float* mlp = ob.p32 + cfg.n_table;
    const float* W1 = mlp + cfg.w_off[0];
    const float* W2 = mlp + cfg.w_off[1];
    const int LF = cfg.LF;
    float r0 = 0.f;
#pragma unroll 4
    for (int j = 0; j < ROMAP_WIDTH; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < ROMAP_MAX_LF; ++k)
            if (k < LF) acc += __ldg(W1 + j * LF + k) * feat[k];
        r0 += __ldg(W2 + j) * relu(acc);
    }
    out[p] = density_act(r0, cfg.density_act);
}

void launch_query_density(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* obj, const float* xyz, long long n,
                          float* sigma) {
    if (n == 0) return;
    k_query<<<(unsigned)((n + 127) / 128), 128, 0, lc.st>>>(cfg, obj, xyz, n, sigma);
}

// ---------------------------------------------------------------------------
// debug dumps of the object's rays of the last iteration (same device functions)
__global__ void __launch_bounds__(128) k_debug(CfgDev cfg, const ObjDev* __restrict__ objs,
                                               const RayRec* __restrict__ rays, int ray_begin, int n_rays, int what,
                                               void* out) {
    long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int N = cfg.N;
    long long r = s / N;
    int i = (int)(s - r * N);
    if (r >= n_rays) return;
    const RayRec rr = rays[ray_begin + r];
    const ObjDev& ob = objs[rr.slot];
    const bool active = (rr.flags & RF_ACTIVE) != 0;
    float dist = 0.f, delta = 0.f, u[3] = {0.f, 0.f, 0.f};
    if (active) sample_geo_any(cfg, ob, rr, (int)(ray_begin + r - ob.ray_begin), i, false, dist, delta, u);
    if (what == 1) {          // SAMPLES
        float* o = (float*)out + 5 * s;
        o[0] = dist; o[1] = delta; o[2] = u[0]; o[3] = u[1]; o[4] = u[2];
    } else if (what == 2) {   // HASH_IDX
        int* o = (int*)out + (long long)s * cfg.L * 8;
        for (int l = 0; l < cfg.L; ++l) {
            Cell cl = grid_cell(u, cfg.res[l]);
            for (int b = 0; b < 8; ++b)
                o[l * 8 + b] = active ? cfg.off[l] + corner_entry(cl, b, cfg.res[l], cfg.dense[l], cfg.T) : -1;
        }
    } else if (what == 3 || what == 4) {
        float feat[ROMAP_MAX_LF];
        if (active) encode_fp32(cfg, ob.p32, u, feat);
        else for (int k = 0; k < ROMAP_MAX_LF; ++k) feat[k] = 0.f;
        if (what == 3) {
            float* o = (float*)out + (long long)s * cfg.LF;
            for (int k = 0; k < cfg.LF; ++k) o[k] = feat[k];
        } else {
            float sh[16];
            sh4(rr.d, sh);
            FwdOut fo = mlp_fwd_fp32(cfg, ob.p32 + cfg.n_table, feat, sh, nullptr, 0);
            float* o = (float*)out + 4 * s;
            o[0] = active ? fo.sigma : 0.f;
            o[1] = active ? fo.rgb[0] : 0.f;
            o[2] = active ? fo.rgb[1] : 0.f;
            o[3] = active ? fo.rgb[2] : 0.f;
        }
    }
}

void launch_debug_samples(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, const RayRec* rays,
                          int ray_begin, int n_rays, int what, void* out) {
    long long S = (long long)n_rays * cfg.N;
    if (S == 0) return;
    k_debug<<<(unsigned)((S + 127) / 128), 128, 0, lc.st>>>(cfg, objs, rays, ray_begin, n_rays, what, out);
}



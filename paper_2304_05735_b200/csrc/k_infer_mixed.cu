// k_infer_mixed.cu -- mixed-precision inference of SURVEY.md 8(a) a10 (density
// query for marching cubes; BASELINE cfg4 "fp16 MLP") for
// objects created with precision = 1: the same fp16 tables / weights and the
// same arithmetic as the forward half of the training kernel.
//
// k_query_mixed: persistent CTAs of 128 threads, tiles of 128 points.  Thread t
// encodes point t of the tile (all L levels, fp16 gathers + packed lerps) into
// the fp16 operand X0 (shared memory), one thread issues the hidden layers
// H = X0 . W1^T (network 1, R24: then h_k = relu(h_{k-1} W_k^T)) on the tensor
// cores (tcgen05.mma, D in TMEM), and every thread finishes its row:
// h = fp16(relu(H)), raw0 = sum_j h_j w_j with w the density output row (network
// 0: W2 row 0; network 1: W_out row 0), sigma = act(raw0), 0 outside the box (R21).
#include "romap_internal.cuh"
#include "tc_sm100.cuh"
#include "hash_fp16.cuh"

namespace {

constexpr int QT = 128;
// network 0 needs W1, X0 and the misc block only (13 KB: 8 CTAs per SM, the
// whole TMEM); network 1 adds the hidden activations and hidden-layer weights
constexpr int Q_OFF_W1 = 0;                   // 64 x LF fp16 (interleaved)
constexpr int Q_OFF_X0 = 64 * 32 * 2;         // 128 x LF fp16 (interleaved)
constexpr int Q_OFF_MISC = Q_OFF_X0 + QT * 32 * 2;
constexpr int Q_OFF_H = Q_OFF_MISC + 1024;              // network 1: 128 x 64 hidden activations
constexpr int Q_OFF_WH = Q_OFF_H + QT * 64 * 2;         // network 1: hidden layers 2, 3 (64 x 64 each)
constexpr int Q_SMEM0 = Q_OFF_H;
constexpr int Q_SMEM1 = Q_OFF_WH + 2 * 64 * 64 * 2;

struct QMisc {
    uint64_t mbar;
    uint32_t tmem;
    int pad;
    int4 lv[ROMAP_MAX_LEVELS];
    int lvoff[ROMAP_MAX_LEVELS];
    float w2[64];                              // density output row (network 0: W2 row 0, 1: W_out row 0)
};
static_assert(sizeof(QMisc) <= 1024, "query misc block");

}  // namespace

template <int L>
__global__ void __launch_bounds__(QT) k_query_mixed(CfgDev cfg, const ObjDev* __restrict__ obj,
                                                    const float* __restrict__ xyz, long long n,
                                                    float* __restrict__ out) {
    constexpr int LF = 2 * L;
    extern __shared__ __align__(1024) uint8_t smem[];
    QMisc* misc = reinterpret_cast<QMisc*>(smem + Q_OFF_MISC);
    const int t = threadIdx.x, warp = t >> 5;
    const ObjDev& ob = *obj;
    if (warp == 0) tc::tmem_alloc(&misc->tmem, 64);
    if (t == 32) {
        tc::mbar_init(&misc->mbar, 1);
        tc::fence_mbar_init();
    }
    if (t < L) {
        misc->lv[t] = level_params(cfg, t);
        misc->lvoff[t] = cfg.off[t];
    }
    const __half* mlp16 = ob.p16 + cfg.n_table;
    const int n_hidden = cfg.net == 1 ? cfg.hl : 1;
    const int out_layer = cfg.net == 1 ? cfg.hl : 1;
    if (t < 64) misc->w2[t] = __half2float(mlp16[cfg.w_off[out_layer] + t]);
    for (int q = t; q < 64 * (LF / 8); q += QT) {
        const int r = q / (LF / 8), cb = q % (LF / 8);
        const __half2* s2 = reinterpret_cast<const __half2*>(mlp16 + cfg.w_off[0] + r * LF + cb * 8);
        __half2 h[4] = {s2[0], s2[1], s2[2], s2[3]};
        *reinterpret_cast<uint4*>(smem + Q_OFF_W1 + tc::il_offset(r, cb * 8, LF)) = *reinterpret_cast<uint4*>(h);
    }
    for (int k = 1; k < n_hidden; ++k)
        for (int q = t; q < 64 * 8; q += QT) {
            const int r = q / 8, cb = q % 8;
            const __half2* s2 = reinterpret_cast<const __half2*>(mlp16 + cfg.w_off[k] + r * 64 + cb * 8);
            __half2 h[4] = {s2[0], s2[1], s2[2], s2[3]};
            *reinterpret_cast<uint4*>(smem + Q_OFF_WH + (k - 1) * 8192 + tc::il_offset(r, cb * 8, 64)) =
                *reinterpret_cast<uint4*>(h);
        }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = misc->tmem;
    const uint32_t wk = tc::taddr(tm, warp * 32, 0);
    const uint32_t sW1 = tc::smem_u32(smem + Q_OFF_W1), sX0 = tc::smem_u32(smem + Q_OFF_X0);
    uint8_t* X0 = smem + Q_OFF_X0;
    const uint32_t* tab = reinterpret_cast<const uint32_t*>(ob.p16);
    const unsigned hmask = (unsigned)cfg.T - 1u;
    uint32_t phase = 0;
    for (long long tile = blockIdx.x; tile * QT < n; tile += gridDim.x) {
        const long long p = tile * QT + t;
        const bool valid = p < n;
        float u[3];
        bool inside = valid;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float x = valid ? xyz[3 * p + k] : 0.f;
            inside &= fabsf(x) <= ob.a[k];
            const float v = __fdiv_rn(__fadd_rn(x, ob.a[k]), __fadd_rn(ob.a[k], ob.a[k]));   // R6
            u[k] = fminf(fmaxf(v, 0.f), 1.f);
        }
#pragma unroll 1
        for (int l = 0; l < L; l += 2) {
            const int4 P[2] = {misc->lv[l], misc->lv[l + 1]};
            const unsigned off[2] = {(unsigned)misc->lvoff[l], (unsigned)misc->lvoff[l + 1]};
            __half2 fq[2];
            encode_pair_fp16(tab, u, P, off, hmask, inside, fq);
            *reinterpret_cast<uint2*>(X0 + tc::il_offset(t, 2 * l, LF)) = *reinterpret_cast<uint2*>(fq);
        }
        tc::fence_async_smem();
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        if (t == 0) {
#pragma unroll
            for (int ks = 0; ks < LF / 16; ++ks)
                tc::mma_f16(tm, tc::desc_kmajor(sX0, LF, ks), tc::desc_kmajor(sW1, LF, ks),
                            tc::idesc_f16(128, 64, false, false), ks > 0);
            tc::commit(&misc->mbar);
        }
        tc::mbar_wait(&misc->mbar, phase);
        phase ^= 1;
        tc::fence_after();
        for (int k = 1; k < n_hidden; ++k) {       // network 1: further hidden layers
            tc::epi_relu64(wk, smem + Q_OFF_H, t);
            tc::fence_async_smem();
            tc::fence_before();
            __syncthreads();
            tc::fence_after();
            if (t == 0) {
                const uint32_t sH = tc::smem_u32(smem + Q_OFF_H), sW = tc::smem_u32(smem + Q_OFF_WH + (k - 1) * 8192);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    tc::mma_f16(tm, tc::desc_kmajor(sH, 64, ks), tc::desc_kmajor(sW, 64, ks),
                                tc::idesc_f16(128, 64, false, false), ks > 0);
                tc::commit(&misc->mbar);
            }
            tc::mbar_wait(&misc->mbar, phase);
            phase ^= 1;
            tc::fence_after();
        }
        float raw0 = 0.f;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float v[32];
            tc::tmem_ld32_sync(wk + 32 * h, v);
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                // the training forward stores h = fp16(relu(H)) as the next operand
                const float hk = __half2float(__float2half_rn(fmaxf(v[k], 0.f)));
                raw0 += hk * misc->w2[32 * h + k];
            }
        }
        if (valid) out[p] = inside ? density_act(raw0, cfg.density_act) : 0.f;
        // X0 and the accumulator are rewritten by the next tile
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
    }
    if (warp == 0) tc::tmem_dealloc(tm, 64);
}

void launch_query_density_mixed(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* obj, const float* xyz,
                                long long n, float* sigma) {
    if (n == 0) return;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_query_mixed<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, Q_SMEM1);
        cudaFuncSetAttribute(k_query_mixed<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, Q_SMEM1);
        attr = true;
    }
    const long long tiles = (n + QT - 1) / QT;
    // persistent over tiles, as many CTAs as are resident: network 0 8 per SM (64
    // TMEM columns each = the whole TMEM), network 1 3 per SM (62 KB of smem each)
    const int smem = cfg.net == 1 ? Q_SMEM1 : Q_SMEM0;
    long long grid = (long long)lc.num_sms * (cfg.net == 1 ? 3 : 8);
    if (grid > tiles) grid = tiles;
    if (cfg.L == 16)
        k_query_mixed<16><<<(unsigned)grid, QT, smem, lc.st>>>(cfg, obj, xyz, n, sigma);
    else
        k_query_mixed<8><<<(unsigned)grid, QT, smem, lc.st>>>(cfg, obj, xyz, n, sigma);
}

// ---------------------------------------------------------------------------
// a11 render, mixed path: the forward half of the training step on the tensor
// cores for midpoint samples (R12), one sample per thread, tiles of 128 samples
// (whole rays of one object: a ray's `slot` indexes `objs`; render_scene lays the
// segments of every object out contiguously, padded to whole tiles, and a CTA
// reloads the fp16 weights when its next tile belongs to another object).  Writes sigma, rgb, dist, delta per sample in the
// layout k_composite consumes (inactive rays: sigma = 0, rgb = 0), so the
// compositing (front to back over black, R20) is shared with the fp32 path.
namespace {
constexpr int F_OFF_W1 = 0;                     // 64 x LF
constexpr int F_OFF_W2 = F_OFF_W1 + 64 * 32 * 2;
constexpr int F_OFF_W3 = F_OFF_W2 + 16 * 64 * 2;
constexpr int F_OFF_W4 = F_OFF_W3 + 64 * 32 * 2;
constexpr int F_OFF_W5 = F_OFF_W4 + 64 * 64 * 2;
// activations alias: a layer's output may overwrite its input once its MMA has
// completed (the epilogue runs after the wait), so two buffers carry the chain:
// R1 = X0, then CIN (SH after L1, raw after L2); R2 = H1, G1, G2 (network 1:
// every hidden layer).  Network 0 needs 44.4 KB per CTA -> 5 CTAs per SM hide
// each other's gather latency; network 1's third hidden layer adds 8 KB (4 CTAs).
constexpr int F_OFF_X0 = F_OFF_W5 + 16 * 64 * 2;
constexpr int F_OFF_CIN = F_OFF_X0;
constexpr int F_OFF_H1 = F_OFF_X0 + QT * 32 * 2;
constexpr int F_OFF_G1 = F_OFF_H1;
constexpr int F_OFF_G2 = F_OFF_H1;
constexpr int F_OFF_MISC = F_OFF_H1 + QT * 64 * 2;
struct FMisc {
    uint64_t mbar;
    uint32_t tmem;
    int pad;
    int4 lv[ROMAP_MAX_LEVELS];
    int lvoff[ROMAP_MAX_LEVELS];
};
constexpr int F_OFF_WH2 = F_OFF_MISC + (int)((sizeof(FMisc) + 127) / 128 * 128);   // network 1 only
constexpr int F_SMEM0 = F_OFF_WH2;
constexpr int F_SMEM1 = F_OFF_WH2 + 64 * 64 * 2;

__device__ __forceinline__ void f_sync_for_mma() {
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
}
}  // namespace

// fp16 weights of one object -> interleaved operand layout (W5: rows 3..15 zero)
__device__ __forceinline__ void f_load_weights(uint8_t* smem, const CfgDev& cfg, const ObjDev& ob, int LF, int t) {
    {
        const __half* mlp16 = ob.p16 + cfg.n_table;
        struct Lw { int off, rows, cols, srows, smem; };
        Lw ls[5] = {{cfg.w_off[0], 64, LF, 64, F_OFF_W1}, {cfg.w_off[1], 16, 64, 16, F_OFF_W2},
                    {cfg.w_off[2], 64, 32, 64, F_OFF_W3}, {cfg.w_off[3], 64, 64, 64, F_OFF_W4},
                    {cfg.w_off[4], 3, 64, 16, F_OFF_W5}};
        int nl = 5;
        if (cfg.net == 1) {       // R24: W1, W_out (W2 slot), hidden 2 (W4 slot), hidden 3 (WH2 slot)
            ls[1] = {cfg.w_off[cfg.hl], 4, 64, 16, F_OFF_W2};
            ls[2] = {cfg.w_off[1], 64, 64, 64, F_OFF_W4};
            ls[3] = {cfg.w_off[2], 64, 64, 64, F_OFF_WH2};
            nl = cfg.hl + 1;
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            if (k >= nl) break;
            const int chunks = ls[k].srows * (ls[k].cols / 8);
            for (int q = t; q < chunks; q += QT) {
                const int r = q / (ls[k].cols / 8), cb = q % (ls[k].cols / 8);
                uint4 v = make_uint4(0, 0, 0, 0);
                if (r < ls[k].rows) {
                    const __half2* s2 =
                        reinterpret_cast<const __half2*>(mlp16 + ls[k].off + r * ls[k].cols + cb * 8);
                    __half2 h[4] = {s2[0], s2[1], s2[2], s2[3]};
                    v = *reinterpret_cast<uint4*>(h);
                }
                *reinterpret_cast<uint4*>(smem + ls[k].smem + tc::il_offset(r, cb * 8, ls[k].cols)) = v;
            }
        }
    }
}

template <int L>
__global__ void __launch_bounds__(QT) k_fwd_mixed(CfgDev cfg, const ObjDev* __restrict__ objs,
                                                  const RayRec* __restrict__ rays, int n_rays,
                                                  float* __restrict__ sigma_o, float* __restrict__ rgb_o,
                                                  float* __restrict__ dist_o, float* __restrict__ delta_o) {
    constexpr int LF = 2 * L;
    extern __shared__ __align__(1024) uint8_t smem[];
    FMisc* misc = reinterpret_cast<FMisc*>(smem + F_OFF_MISC);
    const int t = threadIdx.x, warp = t >> 5;
    const int N = cfg.N;
    if (warp == 0) tc::tmem_alloc(&misc->tmem, 64);
    if (t == 32) {
        tc::mbar_init(&misc->mbar, 1);
        tc::fence_mbar_init();
    }
    if (t < L) {
        misc->lv[t] = level_params(cfg, t);
        misc->lvoff[t] = cfg.off[t];
    }
    f_sync_for_mma();
    const uint32_t tm = misc->tmem;
    const uint32_t wk = tc::taddr(tm, warp * 32, 0);
    const uint32_t sW1 = tc::smem_u32(smem + F_OFF_W1), sW2 = tc::smem_u32(smem + F_OFF_W2),
                   sW3 = tc::smem_u32(smem + F_OFF_W3), sW4 = tc::smem_u32(smem + F_OFF_W4),
                   sW5 = tc::smem_u32(smem + F_OFF_W5), sX0 = tc::smem_u32(smem + F_OFF_X0),
                   sH1 = tc::smem_u32(smem + F_OFF_H1), sCIN = tc::smem_u32(smem + F_OFF_CIN),
                   sG1 = tc::smem_u32(smem + F_OFF_G1), sG2 = tc::smem_u32(smem + F_OFF_G2),
                   sWH2 = tc::smem_u32(smem + F_OFF_WH2);
    uint8_t* X0 = smem + F_OFF_X0;
    uint8_t* H1 = smem + F_OFF_H1;
    uint8_t* CIN = smem + F_OFF_CIN;
    uint8_t* G1 = smem + F_OFF_G1;
    uint8_t* G2 = smem + F_OFF_G2;
    const unsigned hmask = (unsigned)cfg.T - 1u;
    int cur = -1;
    uint32_t phase = 0;
    auto mma_wait = [&]() {
        tc::mbar_wait(&misc->mbar, phase);
        phase ^= 1;
        tc::fence_after();
    };
    const long long S = (long long)n_rays * N;
    for (long long tile = blockIdx.x; tile * QT < S; tile += gridDim.x) {
        const long long s = tile * QT + t;
        const bool valid = s < S;
        const long long ray = valid ? s / N : 0;
        const int i = valid ? (int)(s - ray * N) : 0;
        const int slot = rays[tile * QT / N].slot;        // uniform: a tile holds rays of one object
        if (slot != cur) {
            f_load_weights(smem, cfg, objs[slot], LF, t);
            f_sync_for_mma();
            cur = slot;
        }
        const ObjDev& ob = objs[slot];
        const uint32_t* tab = reinterpret_cast<const uint32_t*>(ob.p16);
        const RayRec rr = rays[ray];
        const bool active = valid && (rr.flags & RF_ACTIVE);
        // R12 inference samples: midpoints, delta = Delta (bit-exact with k_fwd_fp32)
        float dist = 0.f, delta = 0.f, u[3] = {0.f, 0.f, 0.f};
        if (active) {
            const float Dl = __fdiv_rn(__fsub_rn(rr.tf, rr.tn), (float)N);
            dist = sample_dist(rr.tn, Dl, i, 0.5f);
            delta = Dl;
            sample_u(rr.o, rr.d, ob.a, dist, u);
        }
#pragma unroll 1
        for (int l = 0; l < L; l += 2) {
            const int4 P[2] = {misc->lv[l], misc->lv[l + 1]};
            const unsigned off[2] = {(unsigned)misc->lvoff[l], (unsigned)misc->lvoff[l + 1]};
            __half2 fq[2];
            encode_pair_fp16(tab, u, P, off, hmask, active, fq);
            *reinterpret_cast<uint2*>(X0 + tc::il_offset(t, 2 * l, LF)) = *reinterpret_cast<uint2*>(fq);
        }
        f_sync_for_mma();
        if (t == 0) {
#pragma unroll
            for (int ks = 0; ks < LF / 16; ++ks)
                tc::mma_f16(tm, tc::desc_kmajor(sX0, LF, ks), tc::desc_kmajor(sW1, LF, ks),
                            tc::idesc_f16(128, 64, false, false), ks > 0);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        float sigma, c[3];
        if (cfg.net == 0) {
        tc::epi_relu64(wk, H1, t);
        {   // X0 is free now (L1 done): SH(4) of the view direction -> CIN[:, 16:32]
            float sh[16];
            sh4(rr.d, sh);
            tc::st16(CIN, t, 16, 32, sh);
        }
        f_sync_for_mma();
        if (t == 0) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm, tc::desc_kmajor(sH1, 64, ks), tc::desc_kmajor(sW2, 64, ks),
                            tc::idesc_f16(128, 16, false, false), ks > 0);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        {
            float v[16];
            tc::tmem_ld16_sync(wk, v);
            sigma = density_act(v[0], cfg.density_act);
            tc::st16(CIN, t, 0, 32, v);
        }
        f_sync_for_mma();
        if (t == 0) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
                tc::mma_f16(tm, tc::desc_kmajor(sCIN, 32, ks), tc::desc_kmajor(sW3, 32, ks),
                            tc::idesc_f16(128, 64, false, false), ks > 0);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        tc::epi_relu64(wk, G1, t);
        f_sync_for_mma();
        if (t == 0) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm, tc::desc_kmajor(sG1, 64, ks), tc::desc_kmajor(sW4, 64, ks),
                            tc::idesc_f16(128, 64, false, false), ks > 0);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        tc::epi_relu64(wk, G2, t);
        f_sync_for_mma();
        if (t == 0) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm, tc::desc_kmajor(sG2, 64, ks), tc::desc_kmajor(sW5, 64, ks),
                            tc::idesc_f16(128, 16, false, false), ks > 0);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        {
            float v[16];
            tc::tmem_ld16_sync(wk, v);
#pragma unroll
            for (int k = 0; k < 3; ++k) c[k] = 1.0f / (1.0f + expf(-v[k]));
        }
        } else {
        tc::epi_relu64(wk, H1, t);
        f_sync_for_mma();
        for (int k = 1; k < cfg.hl; ++k) {          // R24 hidden layers 2, 3
            if (t == 0) {
                const uint32_t sA = k == 1 ? sH1 : sG1, sW = k == 1 ? sW4 : sWH2;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    tc::mma_f16(tm, tc::desc_kmajor(sA, 64, ks), tc::desc_kmajor(sW, 64, ks),
                                tc::idesc_f16(128, 64, false, false), ks > 0);
                tc::commit(&misc->mbar);
            }
            mma_wait();
            tc::epi_relu64(wk, k == 1 ? G1 : G2, t);
            f_sync_for_mma();
        }
        if (t == 0) {
            const uint32_t sHL = cfg.hl == 1 ? sH1 : (cfg.hl == 2 ? sG1 : sG2);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm, tc::desc_kmajor(sHL, 64, ks), tc::desc_kmajor(sW2, 64, ks),
                            tc::idesc_f16(128, 16, false, false), ks > 0);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        {
            float v[16];
            tc::tmem_ld16_sync(wk, v);
            sigma = density_act(v[0], cfg.density_act);
#pragma unroll
            for (int k = 0; k < 3; ++k) c[k] = 1.0f / (1.0f + expf(-v[1 + k]));
        }
        }
        if (valid) {
            sigma_o[s] = active ? sigma : 0.f;
#pragma unroll
            for (int k = 0; k < 3; ++k) rgb_o[3 * s + k] = active ? c[k] : 0.f;
            dist_o[s] = dist;
            delta_o[s] = delta;
        }
        // the next tile rewrites X0 / CIN and the accumulator
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
    }
    if (warp == 0) tc::tmem_dealloc(tm, 64);
}

void launch_fwd_mixed(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* obj, const RayRec* rays, int n_rays,
                      float* sigma, float* rgb, float* dist, float* delta) {
    const long long S = (long long)n_rays * cfg.N;
    if (S == 0) return;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_fwd_mixed<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM1);
        cudaFuncSetAttribute(k_fwd_mixed<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM1);
        attr = true;
    }
    const long long tiles = (S + QT - 1) / QT;
    const bool wh2 = cfg.net == 1 && cfg.hl == 3;
    const int smem = wh2 ? F_SMEM1 : F_SMEM0;
    long long grid = (long long)lc.num_sms * (wh2 ? 4 : 5);
    if (grid > tiles) grid = tiles;
    if (cfg.L == 16)
        k_fwd_mixed<16><<<(unsigned)grid, QT, smem, lc.st>>>(cfg, obj, rays, n_rays, sigma, rgb, dist, delta);
    else
        k_fwd_mixed<8><<<(unsigned)grid, QT, smem, lc.st>>>(cfg, obj, rays, n_rays, sigma, rgb, dist, delta);
}

// ---------------------------------------------------------------------------
// debug dumps of the MEASURED mixed path (romap_debug_dump on precision-1
// objects): the (u, dist) / delta records k_raygen + k_samples wrote for the
// iteration and k_fused_mixed consumed, and the corner entries computed from them
// by the fused kernel's own addressing (hash_fp16.cuh level_entries + the level
// offset), so a test can hold both bit-exact against the oracle.
//   what 1 (SAMPLES):  out float[n][5] = dist, delta, u.x, u.y, u.z
//   what 2 (HASH_IDX): out int32[n][L][8] absolute entry of corner b (bit k -> +1 on axis k)
__global__ void k_debug_mixed(CfgDev cfg, const float4* __restrict__ srec, const float* __restrict__ sdelta,
                              long long n, int what, void* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 r = srec[i];
    if (what == 1) {
        float* o = static_cast<float*>(out) + 5 * i;
        o[0] = r.w;
        o[1] = sdelta[i];
        o[2] = r.x;
        o[3] = r.y;
        o[4] = r.z;
        return;
    }
    const float u[3] = {r.x, r.y, r.z};
    int* o = static_cast<int*>(out) + i * cfg.L * 8;
    for (int l = 0; l < cfg.L; ++l) {
        Cell cl;
        unsigned e[8];
        level_entries(u, level_params(cfg, l), 0u, (unsigned)cfg.T - 1u, cl, e);
#pragma unroll
        for (int b = 0; b < 8; ++b) o[l * 8 + b] = (int)(e[b] + (unsigned)cfg.off[l]);
    }
}

void launch_debug_mixed(const LaunchCtx& lc, const CfgDev& cfg, const float4* srec, const float* sdelta, long long n,
                        int what, void* out) {
    if (n > 0) k_debug_mixed<<<(unsigned)((n + 127) / 128), 128, 0, lc.st>>>(cfg, srec, sdelta, n, what, out);
}

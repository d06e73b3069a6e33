// k_fused_mixed.cu -- the mixed-precision hot path: ONE persistent kernel per
// iteration that runs, per 128-sample tile (whole rays of one object):
//
//   a2-a3  stratified samples (bit-exact with the fp32 path) + hash-grid encode
//          forward: fp16 table gathers, fp32 trilinear accumulation
//   a4     fused MLP forward on the 5th-gen tensor cores: 5 tcgen05.mma layers
//          (fp16 operands in shared memory, fp32 accumulators in TMEM), ReLU /
//          exp / sigmoid epilogues from TMEM -> registers -> shared memory
//   a5     volume rendering (Eq. 6) + object-tailored loss (Eqs. 7-11) + render
//          backward, segmented scans over each ray's samples
//   a6     MLP backward on tensor cores: dX = delta W per layer, and
//          dW += delta^T X accumulated in TMEM across all tiles this CTA runs for
//          the object (flushed once per CTA and object with fp32 atomics)
//   a7     hash-grid backward: recomputed cells, fp32 float2 atomics
//
// One CTA = 2 warpgroups = 256 threads per 128-sample tile: thread t works on
// sample t % 128 (= TMEM lane t % 128; warps w and w+4 share lanes 32(w%4)..+31)
// and on half t / 128 of the split work: hash levels [h*L/2, (h+1)*L/2) of the
// gathers and scatters, accumulator columns [32h, 32h+32) of 64-wide epilogues.
// Two CTAs per SM (110.6 KB shared memory, 256 TMEM columns each): 16 warps
// per SM, one CTA's gathers / atomics overlap the other's tensor-core chain.
// Loss scaling: every backward operand is multiplied by cfg.loss_scale (a power
// of two, exact) and divided out before the fp32 atomics.
#include "romap_internal.cuh"
#include "tc_sm100.cuh"

bool fused_mixed_available() { return true; }

namespace {

constexpr int TILE = 128;                      // samples per tile
constexpr int NT = 256;                        // threads per CTA (2 warpgroups)
// shared-memory layout (bytes); every block is a multiple of 1024
constexpr int OFF_W1 = 0;                      // 64 x LF(<=32)
constexpr int OFF_W2 = OFF_W1 + 64 * 32 * 2;   // 16 x 64
constexpr int OFF_W3 = OFF_W2 + 16 * 64 * 2;   // 64 x 32
constexpr int OFF_W4 = OFF_W3 + 64 * 32 * 2;   // 64 x 64
constexpr int OFF_W5 = OFF_W4 + 64 * 64 * 2;   // 16 x 64 (rows 3..15 zero)
constexpr int OFF_X0 = OFF_W5 + 16 * 64 * 2;   // 128 x LF
constexpr int OFF_H1 = OFF_X0 + TILE * 32 * 2; // 128 x 64
constexpr int OFF_CIN = OFF_H1 + TILE * 64 * 2;
constexpr int OFF_G1 = OFF_CIN + TILE * 32 * 2;
constexpr int OFF_G2 = OFF_G1 + TILE * 64 * 2;
constexpr int OFF_DC = OFF_G2 + TILE * 64 * 2;  // 128 x 16
constexpr int OFF_DR = OFF_DC + TILE * 16 * 2;  // 128 x 16
constexpr int OFF_DB = OFF_DR + TILE * 16 * 2;  // 128 x 64 (dg2 -> dg1 -> dh1)
constexpr int OFF_MISC = OFF_DB + TILE * 64 * 2;
constexpr int SMEM_BYTES = OFF_MISC + 384;

// TMEM columns
constexpr int TM_WK = 0;      // working accumulator (<= 64 cols)
constexpr int TM_DW1 = 64;    // dW1   [64 x LF]
constexpr int TM_DW3 = 96;    // dW3   [64 x 32]
constexpr int TM_DW4 = 128;   // dW4   [64 x 64]
constexpr int TM_DW2 = 192;   // dW2^T [64 x 16]
constexpr int TM_DW5 = 208;   // dW5^T [64 x 16]
constexpr int TM_COLS = 256;

struct Misc {
    uint64_t mbar;
    uint32_t tmem;
    int pad;
    float loss[4];
    float xw[8][8];           // cross-warp scan exchange (per warp, 8 slots)
};

__device__ __forceinline__ void sync_for_mma() {
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
}

// ---------------------------------------------------------------------------
// segmented scans over the N samples of each ray; each warpgroup scans its own
// copy (thread t = sample (t % 128) % N of ray (t % 128) / N)
template <bool MUL>
__device__ __forceinline__ float op2(float a, float b) { return MUL ? a * b : a + b; }

template <bool MUL>
__device__ __forceinline__ float ray_scan_excl(float x, int N, float* xw, int slot, float& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sw = N < 32 ? N : 32;
    const float ident = MUL ? 1.f : 0.f;
    float incl = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        if (off >= sw) break;
        float y = __shfl_up_sync(0xffffffffu, incl, off, sw);
        if ((lane & (sw - 1)) >= off) incl = op2<MUL>(incl, y);
    }
    float excl = __shfl_up_sync(0xffffffffu, incl, 1, sw);
    if ((lane & (sw - 1)) == 0) excl = ident;
    float seg_total = __shfl_sync(0xffffffffu, incl, sw - 1, sw);
    if (N <= 32) {
        total = seg_total;
        return excl;
    }
    if (lane == 31) xw[warp * 8 + slot] = incl;
    __syncthreads();
    const int wpr = N >> 5;
    const int w0 = warp - (warp % wpr);
    float carry = ident, tot = ident;
    for (int w = w0; w < w0 + wpr; ++w) {
        float v = xw[w * 8 + slot];
        if (w < warp) carry = op2<MUL>(carry, v);
        tot = op2<MUL>(tot, v);
    }
    __syncthreads();
    total = tot;
    return op2<MUL>(carry, excl);
}

__device__ __forceinline__ float ray_suffix_excl(float x, int N, float* xw, int slot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sw = N < 32 ? N : 32;
    float incl = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        if (off >= sw) break;
        float y = __shfl_down_sync(0xffffffffu, incl, off, sw);
        if ((lane & (sw - 1)) + off < sw) incl += y;
    }
    float excl = __shfl_down_sync(0xffffffffu, incl, 1, sw);
    if ((lane & (sw - 1)) == sw - 1) excl = 0.f;
    if (N <= 32) return excl;
    if (lane == 0) xw[warp * 8 + slot] = incl;
    __syncthreads();
    const int wpr = N >> 5;
    const int w0 = warp - (warp % wpr);
    float carry = 0.f;
    for (int w = warp + 1; w < w0 + wpr; ++w) carry += xw[w * 8 + slot];
    __syncthreads();
    return carry + excl;
}

__device__ __forceinline__ float ray_sum(float x, int N, float* xw, int slot) {
    float tot;
    ray_scan_excl<false>(x, N, xw, slot, tot);
    return tot;
}

// ---------------------------------------------------------------------------
// copy one object's fp16 weights into the interleaved smem layout
__device__ void load_weights(uint8_t* smem, const __half* __restrict__ mlp16, const CfgDev& cfg) {
    const int LF = cfg.LF;
    struct L { int off, rows, cols, srows, smem; };
    const L ls[5] = {{cfg.w_off[0], 64, LF, 64, OFF_W1}, {cfg.w_off[1], 16, 64, 16, OFF_W2},
                     {cfg.w_off[2], 64, 32, 64, OFF_W3}, {cfg.w_off[3], 64, 64, 64, OFF_W4},
                     {cfg.w_off[4], 3, 64, 16, OFF_W5}};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int chunks = ls[k].srows * (ls[k].cols / 8);
        for (int q = threadIdx.x; q < chunks; q += NT) {
            int r = q / (ls[k].cols / 8), cb = q % (ls[k].cols / 8);
            uint4 v = make_uint4(0, 0, 0, 0);
            if (r < ls[k].rows) {
                // weights are only 4-byte aligned in general: load as 4 x half2
                const __half2* s2 = reinterpret_cast<const __half2*>(mlp16 + ls[k].off + r * ls[k].cols + cb * 8);
                __half2 h[4] = {s2[0], s2[1], s2[2], s2[3]};
                v = *reinterpret_cast<uint4*>(h);
            }
            *reinterpret_cast<uint4*>(smem + ls[k].smem + tc::il_offset(r, cb * 8, ls[k].cols)) = v;
        }
    }
}

// flush dW accumulators (TMEM) and loss sums of one object; warpgroup 0 takes
// dW1, dW2, dW5, warpgroup 1 takes dW3, dW4
__device__ void flush_object(const CfgDev& cfg, const ObjDev& ob, uint32_t tm, Misc* misc, double* loss_acc,
                             int slot, bool have_dw) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wg = threadIdx.x >> 7;
    const int q = warp & 3;
    const float inv = 1.0f / cfg.loss_scale;
    float* gm = ob.g32 + cfg.n_table;
    if (have_dw) {
        const int row = q * 16 + lane;   // M=64 accumulator row held by this lane (lanes < 16)
        float v[16];
        if (wg == 0) {
            for (int c0 = 0; c0 < cfg.LF; c0 += 16) {
                tc::tmem_ld16(tc::taddr(tm, q * 32, TM_DW1 + c0), v);
                tc::tmem_wait_ld();
                if (lane < 16)
                    for (int i = 0; i < 16; ++i) red_add_f1(gm + cfg.w_off[0] + row * cfg.LF + c0 + i, v[i] * inv);
            }
            // dW2^T [64 in x 16 out], dW5^T [64 in x 16 (3) out]: row = input feature
            tc::tmem_ld16(tc::taddr(tm, q * 32, TM_DW2), v);
            tc::tmem_wait_ld();
            if (lane < 16)
                for (int o = 0; o < 16; ++o) red_add_f1(gm + cfg.w_off[1] + o * 64 + row, v[o] * inv);
            tc::tmem_ld16(tc::taddr(tm, q * 32, TM_DW5), v);
            tc::tmem_wait_ld();
            if (lane < 16)
                for (int o = 0; o < 3; ++o) red_add_f1(gm + cfg.w_off[4] + o * 64 + row, v[o] * inv);
        } else {
            for (int c0 = 0; c0 < 32; c0 += 16) {
                tc::tmem_ld16(tc::taddr(tm, q * 32, TM_DW3 + c0), v);
                tc::tmem_wait_ld();
                if (lane < 16)
                    for (int i = 0; i < 16; ++i) red_add_f1(gm + cfg.w_off[2] + row * 32 + c0 + i, v[i] * inv);
            }
            for (int c0 = 0; c0 < 64; c0 += 16) {
                tc::tmem_ld16(tc::taddr(tm, q * 32, TM_DW4 + c0), v);
                tc::tmem_wait_ld();
                if (lane < 16)
                    for (int i = 0; i < 16; ++i) red_add_f1(gm + cfg.w_off[3] + row * 64 + c0 + i, v[i] * inv);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        float l = misc->loss[threadIdx.x];
        if (l != 0.f) atomicAdd(loss_acc + 4 * slot + threadIdx.x, (double)l);
        misc->loss[threadIdx.x] = 0.f;
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
}

// store 16 consecutive fp32 values (columns c0..c0+15 of row r) as fp16
__device__ __forceinline__ void st16(uint8_t* buf, int r, int c0, int C, const float* v) {
    tc::st_chunk(buf, r, c0, C, v);
    tc::st_chunk(buf, r, c0 + 8, C, v + 8);
}

// epilogue of a 64-wide layer: this warpgroup's 32 columns, ReLU (or mask) ->
// fp16 -> smem; `relu` records the mask, otherwise `mask` is applied
template <bool RELU>
__device__ __forceinline__ void epi32(uint32_t wk, int wg, uint8_t* buf, int r, uint32_t& mask) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int c0 = 32 * wg + 16 * h;
        float v[16];
        tc::tmem_ld16(wk + c0, v);
        tc::tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint32_t bit = 1u << (16 * h + k);
            if (RELU) {
                if (v[k] > 0.f) mask |= bit; else v[k] = 0.f;
            } else if (!(mask & bit)) {
                v[k] = 0.f;
            }
        }
        st16(buf, r, c0, 64, v);
    }
}

}  // namespace

__global__ void __launch_bounds__(NT, 2) k_fused_mixed(CfgDev cfg, const ObjDev* __restrict__ objs,
                                                       const RayRec* __restrict__ rays, int n_tiles,
                                                       int tiles_per_cta, double* __restrict__ loss_acc,
                                                       int* __restrict__ nonfinite, float* __restrict__ dbg) {
    extern __shared__ __align__(1024) uint8_t smem[];
    Misc* misc = reinterpret_cast<Misc*>(smem + OFF_MISC);
    const int t = threadIdx.x, warp = t >> 5, wg = t >> 7;
    const int r = t & (TILE - 1);                 // sample row of the tile = TMEM lane
    const int N = cfg.N, LF = cfg.LF;
    const float scale = cfg.loss_scale, inv_scale = 1.0f / cfg.loss_scale;

    if (warp == 0) tc::tmem_alloc(&misc->tmem, TM_COLS);
    if (t == 0) {
        tc::mbar_init(&misc->mbar, 1);
        tc::fence_mbar_init();
    }
    if (t < 4) misc->loss[t] = 0.f;
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = misc->tmem;
    const uint32_t wk = tc::taddr(tm, (warp & 3) * 32, 0);   // this warp's TMEM lanes, column 0
    uint32_t phase = 0;
    const uint32_t sW1 = tc::smem_u32(smem + OFF_W1), sW2 = tc::smem_u32(smem + OFF_W2),
                   sW3 = tc::smem_u32(smem + OFF_W3), sW4 = tc::smem_u32(smem + OFF_W4),
                   sW5 = tc::smem_u32(smem + OFF_W5), sX0 = tc::smem_u32(smem + OFF_X0),
                   sH1 = tc::smem_u32(smem + OFF_H1), sCIN = tc::smem_u32(smem + OFF_CIN),
                   sG1 = tc::smem_u32(smem + OFF_G1), sG2 = tc::smem_u32(smem + OFF_G2),
                   sDC = tc::smem_u32(smem + OFF_DC), sDR = tc::smem_u32(smem + OFF_DR),
                   sDB = tc::smem_u32(smem + OFF_DB);
    uint8_t* X0 = smem + OFF_X0;
    uint8_t* H1 = smem + OFF_H1;
    uint8_t* CIN = smem + OFF_CIN;
    uint8_t* G1 = smem + OFF_G1;
    uint8_t* G2 = smem + OFF_G2;
    uint8_t* DC = smem + OFF_DC;
    uint8_t* DR = smem + OFF_DR;
    uint8_t* DB = smem + OFF_DB;
    float* xw = &misc->xw[0][0];

    auto mma_wait = [&]() {
        tc::mbar_wait(&misc->mbar, phase);
        phase ^= 1;
        tc::fence_after();
    };

    const int tile0 = blockIdx.x * tiles_per_cta;
    const int tile1 = min(tile0 + tiles_per_cta, n_tiles);
    int cur = -1;
    bool dw_fresh = true;
    const int rays_per_tile = TILE / N;
    const int LH = cfg.L >> 1;                    // hash levels per warpgroup
    // per-object values held in registers (re-read only when the object changes)
    const __half2* tab = nullptr;
    float2* gt = nullptr;
    float ob_a[3] = {0.f, 0.f, 0.f};
    int ob_ray_begin = 0;
    float invB = 0.f;
    unsigned long long pre = 0;

    for (int tile = tile0; tile < tile1; ++tile) {
        const int slot = rays[tile * rays_per_tile].slot;
        if (slot != cur) {
            if (cur >= 0) flush_object(cfg, objs[cur], tm, misc, loss_acc, cur, !dw_fresh);
            const ObjDev& ob = objs[slot];
            load_weights(smem, ob.p16 + cfg.n_table, cfg);
            cur = slot;
            dw_fresh = true;
            tab = reinterpret_cast<const __half2*>(ob.p16);
            gt = reinterpret_cast<float2*>(ob.g32);
            ob_a[0] = ob.a[0];
            ob_a[1] = ob.a[1];
            ob_a[2] = ob.a[2];
            ob_ray_begin = ob.ray_begin;
            invB = 1.0f / (float)ob.n_rays;
            pre = rng_prefix(cfg.seed, ob.obj_id, *ob.step + 1);
        }
        const long long s = (long long)tile * TILE + r;
        const int ray = (int)(s / N);
        const int i = (int)(s - (long long)ray * N);
        const RayRec rr = rays[ray];
        const bool active = (rr.flags & RF_ACTIVE) != 0;

        // ---- a2/a3: sample + encode (fp16 table gathers, fp32 interpolation)
        float dist = 0.f, delta = 0.f, u[3] = {0.f, 0.f, 0.f};
        if (active) sample_geometry(rr, i, N, pre, ray - ob_ray_begin, ob_a, dist, delta, u);
        {
            float f8[8];
#pragma unroll
            for (int lp = 0; lp < ROMAP_MAX_LEVELS / 2; lp += 2) {
                if (lp >= LH) break;
                // x-neighbour corners (b, b|1) share a 16-byte chunk of the fp16 table in
                // 3 of 4 cases (dense: entries e, e+1; hashed: e ^ (x ^ (x+1)) with the
                // x prime = 1), so each corner pair costs one 16-B gather (+ a 4-B one
                // otherwise); level blocks are 16-entry aligned (R5).
                uint4 qv[2][4];
                uint32_t xv[2][4];
                int e0[2][4], e1[2][4];
                Cell cl[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int l = wg * LH + lp + q;
                    const int res = cfg.res[l];
                    cl[q] = grid_cell(u, res);
                    const __half2* tb = tab + cfg.off[l];
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        e0[q][p] = corner_entry(cl[q], 2 * p, res, cfg.dense[l], cfg.T);
                        e1[q][p] = corner_entry(cl[q], 2 * p + 1, res, cfg.dense[l], cfg.T);
                        const bool same = (e0[q][p] >> 2) == (e1[q][p] >> 2);
                        qv[q][p] = active ? ldg_v4(tb + (e0[q][p] & ~3)) : make_uint4(0, 0, 0, 0);
                        xv[q][p] = (active && !same) ? ldg_u32(tb + e1[q][p]) : 0u;
                    }
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    float a0 = 0.f, a1 = 0.f;
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        const bool same = (e0[q][p] >> 2) == (e1[q][p] >> 2);
                        const uint32_t h0 = sel4(qv[q][p], e0[q][p] & 3);
                        const uint32_t h1 = same ? sel4(qv[q][p], e1[q][p] & 3) : xv[q][p];
                        const float w0 = corner_weight(cl[q], 2 * p), w1 = corner_weight(cl[q], 2 * p + 1);
                        const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&h0));
                        const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&h1));
                        a0 += w0 * f0.x;
                        a1 += w0 * f0.y;
                        a0 += w1 * f1.x;
                        a1 += w1 * f1.y;
                    }
                    f8[2 * ((lp + q) & 3)] = a0;
                    f8[2 * ((lp + q) & 3) + 1] = a1;
                }
                if ((lp & 3) == 2) tc::st_chunk(X0, r, 2 * (wg * LH + lp - 2), LF, f8);
            }
            if (wg == 1) {
                float sh[16];
                sh4(rr.d, sh);
                st16(CIN, r, 16, 32, sh);
            }
        }
        sync_for_mma();

        // ---- a4: MLP forward
        // L1: WK[128 x 64] = X0[128 x LF] . W1^T
        if (t == 0) {
            for (int ks = 0; ks < LF / 16; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sX0, LF, ks), tc::desc_kmajor(sW1, LF, ks),
                            tc::idesc_f16(128, 64, false, false), ks > 0);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        uint32_t m_h1 = 0, m_g1 = 0, m_g2 = 0;
        epi32<true>(wk, wg, H1, r, m_h1);
        sync_for_mma();
        // L2: WK[128 x 16] = H1 . W2^T
        if (t == 0) {
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sH1, 64, ks), tc::desc_kmajor(sW2, 64, ks),
                            tc::idesc_f16(128, 16, false, false), ks > 0);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        float sigma, r0;
        {
            float v[16];
            tc::tmem_ld16(wk, v);
            tc::tmem_wait_ld();
            r0 = v[0];
            sigma = density_act(r0, cfg.density_act);
            if (wg == 0) st16(CIN, r, 0, 32, v);
        }
        sync_for_mma();
        // L3: WK = CIN . W3^T
        if (t == 0) {
            for (int ks = 0; ks < 2; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sCIN, 32, ks), tc::desc_kmajor(sW3, 32, ks),
                            tc::idesc_f16(128, 64, false, false), ks > 0);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        epi32<true>(wk, wg, G1, r, m_g1);
        sync_for_mma();
        // L4: WK = G1 . W4^T
        if (t == 0) {
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sG1, 64, ks), tc::desc_kmajor(sW4, 64, ks),
                            tc::idesc_f16(128, 64, false, false), ks > 0);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        epi32<true>(wk, wg, G2, r, m_g2);
        sync_for_mma();
        // L5: WK[128 x 16] = G2 . W5^T (rows 3..15 of W5 are zero)
        if (t == 0) {
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sG2, 64, ks), tc::desc_kmajor(sW5, 64, ks),
                            tc::idesc_f16(128, 16, false, false), ks > 0);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        float c[3];
        {
            float v[16];
            tc::tmem_ld16(wk, v);
            tc::tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 3; ++k) c[k] = 1.0f / (1.0f + expf(-v[k]));
        }

        // ---- a5: volume rendering + loss + render backward (both warpgroups,
        // redundantly, so every thread holds dL/dsigma and dL/dc of its sample)
        const float x = active ? sigma * delta : 0.f;
        const float alpha = expf(-x);
        const float o = -expm1f(-x);
        float TN;
        const float Ti = ray_scan_excl<true>(alpha, N, xw, 0, TN);
        const float w = active ? Ti * o : 0.f;
        const float Cs0 = ray_sum(w * c[0], N, xw, 1);
        const float Cs1 = ray_sum(w * c[1], N, xw, 2);
        const float Cs2 = ray_sum(w * c[2], N, xw, 3);
        const float D = ray_sum(w * dist, N, xw, 4);
        const float ssum = ray_sum(active ? sigma : 0.f, N, xw, 5);
        float dsig = 0.f, dcol[3] = {0.f, 0.f, 0.f};
        float gC[3] = {0.f, 0.f, 0.f};
        float gD = 0.f, gCb = 0.f;
        const int cls = rr.flags & RF_CLS_MASK;
        if (active) {
            const bool has_depth = (rr.flags & RF_HAS_DEPTH) != 0;
            const float Cs[3] = {Cs0, Cs1, Cs2};
            float e[3], bgc[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                bgc[k] = (cls == CLS_OBJ && cfg.obj_bg == 1) ? 0.f : rr.bg[k];
                e[k] = Cs[k] + TN * bgc[k] - (cls == CLS_OBJ ? rr.tgt[k] : rr.bg[k]);
            }
            const float ne = sqrtf(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
#pragma unroll
            for (int k = 0; k < 3; ++k) gC[k] = ne > 0.f ? e[k] / ne * invB : 0.f;
            float ed = 0.f;
            if (has_depth) {
                ed = D - rr.depth;
                gD = ed > 0.f ? cfg.lambda_depth * invB : (ed < 0.f ? -cfg.lambda_depth * invB : 0.f);
            }
            gCb = gC[0] * bgc[0] + gC[1] * bgc[1] + gC[2] * bgc[2];
            if (i == 0 && wg == 0) {
                atomicAdd(&misc->loss[cls == CLS_OBJ ? 0 : 1], ne);
                if (has_depth) atomicAdd(&misc->loss[2], fabsf(ed));
                if (cls == CLS_BG) atomicAdd(&misc->loss[3], ssum);
                if (!isfinite(ne) || !isfinite(ssum)) atomicOr(nonfinite, 1);
            }
        }
        const float gc = gC[0] * c[0] + gC[1] * c[1] + gC[2] * c[2];
        const float S = ray_suffix_excl(w * gc, N, xw, 6);
        const float Sd = ray_suffix_excl(w * dist, N, xw, 7);
        if (active) {
            const float Tn1 = Ti * alpha;
            dsig = delta * (Tn1 * gc - S - TN * gCb) + delta * gD * (Tn1 * dist - Sd) +
                   (cls == CLS_BG ? cfg.lambda_density * invB : 0.f);
#pragma unroll
            for (int k = 0; k < 3; ++k) dcol[k] = w * gC[k];
        }
        if (dbg && wg == 0) *reinterpret_cast<float4*>(dbg + 4 * s) = make_float4(dsig, dcol[0], dcol[1], dcol[2]);

        // ---- a6: MLP backward (scaled by loss_scale)
        if (wg == 0) {
            float v[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = 0.f;
#pragma unroll
            for (int k = 0; k < 3; ++k) v[k] = dcol[k] * c[k] * (1.f - c[k]) * scale;
            st16(DC, r, 0, 16, v);
        }
        const float dr0_extra = dsig * density_act_grad(r0, sigma, cfg.density_act) * scale;
        sync_for_mma();
        // B5: WK[128 x 64] = DC[128 x 16] . W5[16 x 64];  dW5^T[64 x 16] += G2^T . DC
        if (t == 0) {
            tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sDC, 16, 0), tc::desc_mnmajor(sW5, 64, 0),
                        tc::idesc_f16(128, 64, false, true), 0);
            for (int ks = 0; ks < 8; ++ks)
                tc::mma_f16(tm + TM_DW5, tc::desc_mnmajor(sG2, 64, ks), tc::desc_mnmajor(sDC, 16, ks),
                            tc::idesc_f16(64, 16, true, true), (dw_fresh && ks == 0) ? 0 : 1);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        epi32<false>(wk, wg, DB, r, m_g2);
        sync_for_mma();
        // B4: WK = DB(dg2) . W4;  dW4[64 x 64] += DB^T . G1
        if (t == 0) {
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sDB, 64, ks), tc::desc_mnmajor(sW4, 64, ks),
                            tc::idesc_f16(128, 64, false, true), ks > 0);
            for (int ks = 0; ks < 8; ++ks)
                tc::mma_f16(tm + TM_DW4, tc::desc_mnmajor(sDB, 64, ks), tc::desc_mnmajor(sG1, 64, ks),
                            tc::idesc_f16(64, 64, true, true), (dw_fresh && ks == 0) ? 0 : 1);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        epi32<false>(wk, wg, DB, r, m_g1);
        sync_for_mma();
        // B3: WK[128 x 16] = DB(dg1) . W3[:, 0:16];  dW3[64 x 32] += DB^T . CIN
        if (t == 0) {
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sDB, 64, ks), tc::desc_mnmajor(sW3, 32, ks),
                            tc::idesc_f16(128, 16, false, true), ks > 0);
            for (int ks = 0; ks < 8; ++ks)
                tc::mma_f16(tm + TM_DW3, tc::desc_mnmajor(sDB, 64, ks), tc::desc_mnmajor(sCIN, 32, ks),
                            tc::idesc_f16(64, 32, true, true), (dw_fresh && ks == 0) ? 0 : 1);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        if (wg == 0) {
            float v[16];
            tc::tmem_ld16(wk, v);
            tc::tmem_wait_ld();
            v[0] += dr0_extra;
            if (!active)
#pragma unroll
                for (int k = 0; k < 16; ++k) v[k] = 0.f;
            st16(DR, r, 0, 16, v);
        }
        sync_for_mma();
        // B2: WK[128 x 64] = DR[128 x 16] . W2[16 x 64];  dW2^T[64 x 16] += H1^T . DR
        if (t == 0) {
            tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sDR, 16, 0), tc::desc_mnmajor(sW2, 64, 0),
                        tc::idesc_f16(128, 64, false, true), 0);
            for (int ks = 0; ks < 8; ++ks)
                tc::mma_f16(tm + TM_DW2, tc::desc_mnmajor(sH1, 64, ks), tc::desc_mnmajor(sDR, 16, ks),
                            tc::idesc_f16(64, 16, true, true), (dw_fresh && ks == 0) ? 0 : 1);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        epi32<false>(wk, wg, DB, r, m_h1);
        sync_for_mma();
        // B1: WK[128 x LF] = DB(dh1) . W1[64 x LF];  dW1[64 x LF] += DB^T . X0
        if (t == 0) {
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sDB, 64, ks), tc::desc_mnmajor(sW1, LF, ks),
                            tc::idesc_f16(128, LF, false, true), ks > 0);
            for (int ks = 0; ks < 8; ++ks)
                tc::mma_f16(tm + TM_DW1, tc::desc_mnmajor(sDB, 64, ks), tc::desc_mnmajor(sX0, LF, ks),
                            tc::idesc_f16(64, LF, true, true), (dw_fresh && ks == 0) ? 0 : 1);
            tc::commit(&misc->mbar);
        }
        mma_wait();
        dw_fresh = false;

        // ---- a7: hash-grid backward, this warpgroup's levels (fp32 REDG.F32x2)
        {
            // dfeat of levels [wg*LH, wg*LH + LH) = accumulator columns [2*wg*LH, +2*LH)
            float v[16];
            tc::tmem_ld16(wk + 2 * wg * LH, v);
            tc::tmem_wait_ld();
            if (active) {
#pragma unroll
                for (int lq = 0; lq < 8; ++lq) {
                    if (lq >= LH) break;
                    const int l = wg * LH + lq;
                    const int res = cfg.res[l];
                    const Cell cl = grid_cell(u, res);
                    const float g0 = v[2 * lq] * inv_scale, g1 = v[2 * lq + 1] * inv_scale;
                    float2* gl = gt + cfg.off[l];
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        // x-neighbour pair in one aligned 16-B pair of fp32 entries -> one
                        // REDG.F32x4, else two REDG.F32x2
                        const int ea = corner_entry(cl, 2 * p, res, cfg.dense[l], cfg.T);
                        const int eb = corner_entry(cl, 2 * p + 1, res, cfg.dense[l], cfg.T);
                        const float wa = corner_weight(cl, 2 * p), wb = corner_weight(cl, 2 * p + 1);
                        if ((ea >> 1) == (eb >> 1)) {
                            if (ea < eb)
                                red_add_f4(reinterpret_cast<float4*>(gl + ea), wa * g0, wa * g1, wb * g0, wb * g1);
                            else
                                red_add_f4(reinterpret_cast<float4*>(gl + eb), wb * g0, wb * g1, wa * g0, wa * g1);
                        } else {
                            red_add_f2(gl + ea, wa * g0, wa * g1);
                            red_add_f2(gl + eb, wb * g0, wb * g1);
                        }
                    }
                }
            }
        }
        // all TMEM reads of WK done before the next tile's first MMA overwrites it
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
    }
    if (cur >= 0) flush_object(cfg, objs[cur], tm, misc, loss_acc, cur, !dw_fresh);
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tm, TM_COLS);
}

void launch_fused_mixed(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, const RayRec* rays, int n_rays,
                        double* loss_acc, int* nonfinite, float* dbg) {
    const long long S = (long long)n_rays * cfg.N;
    const int n_tiles = (int)(S / TILE);
    if (n_tiles == 0) return;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_fused_mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        attr = true;
    }
    int grid = 2 * lc.num_sms;
    if (grid > n_tiles) grid = n_tiles;
    const int per = (n_tiles + grid - 1) / grid;
    grid = (n_tiles + per - 1) / per;
    k_fused_mixed<<<grid, NT, SMEM_BYTES, lc.st>>>(cfg, objs, rays, n_tiles, per, loss_acc, nonfinite, dbg);
}

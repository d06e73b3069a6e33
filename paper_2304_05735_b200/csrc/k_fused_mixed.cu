// k_fused_mixed.cu -- the mixed-precision hot path: ONE persistent,
// warp-specialised kernel per iteration (one CTA per SM) that runs, per
// 128-sample tile (whole rays of one object):
//
//   a3     hash-grid encode forward: fp16 table gathers, fp32 trilinear
//          accumulation                                   [warpgroups G0, G1]
//   a2/a4  SH(4) of the view direction + fused MLP forward on the 5th-gen
//          tensor cores: 5 tcgen05.mma layers (fp16 operands in shared memory,
//          fp32 accumulators in TMEM), ReLU / exp / sigmoid epilogues
//                                                          [warpgroup M]
//   a5     volume rendering (Eq. 6) + object-tailored loss (Eqs. 7-11) + render
//          backward, segmented scans over each ray's samples          [M]
//   a6     MLP backward on tensor cores: dX = delta W per layer, and
//          dW += delta^T X accumulated in TMEM across all tiles this CTA runs for
//          the object (flushed once per CTA and object with fp32 REDs)   [M]
//   a7     hash-grid backward: recomputed cells, fp32 vector REDs      [G0, G1]
//
// Pipeline.  G0 / G1 (threads 0-255) own the level pairs (p, L-1-p) with p even /
// odd of sample t % 128 (each pair a coarse and a fine level, so both carry the
// same mix); M (threads 256-383) owns the whole MLP / render chain of sample
// t - 256.  In G iteration `it` the gathers of tile `it` are interleaved,
// level pair by level pair, with the fire-and-forget scatter of tile `it - NB`
// (NB = 3), so the REDs fill the gathers' L2 latency; meanwhile M runs one of the
// tiles in between (three slots absorb the tile-to-tile variation of either role).
// Hand-offs are mbarriers in shared memory (NB slots, b = tile % NB):
//   x0_full[b]   G -> M   encoded features of the tile are in X0[b]   (8 warp arrivals)
//   tile_done[b] M -> G   the tile's last MMAs completed: dfeat is in TMEM DF[b]
//                         and X0[b] is free                           (tcgen05.commit)
//   df_empty[b]  G -> M   DF[b] has been read                         (8 warp arrivals)
// Per-sample geometry (u, dist, delta) comes from k_raygen + k_samples (bit-exact
// with the fp32 path), so neither role recomputes the RNG / IEEE divisions.
// Loss scaling: every backward operand is multiplied by cfg.loss_scale (a power
// of two, exact) and divided out before the fp32 atomics.
#include "romap_internal.cuh"
#include "tc_sm100.cuh"
#include "hash_fp16.cuh"

// deterministic-reduction build (-DROMAP_DET, k_fused_mixed_det.o; k_det.cu):
// the same kernel writing per-record gradient / loss contributions instead of
// atomics (DetBufs, romap_internal.cuh); tests only
#ifdef ROMAP_DET
#define DET_PARAM , DetBufs det
#define DET_ARG , det
#define FUSED_LAUNCH launch_fused_mixed_det
#define k_fused_mixed k_fused_mixed_det
#else
#define DET_PARAM
#define DET_ARG
#define FUSED_LAUNCH launch_fused_mixed
bool fused_mixed_available() { return true; }
#endif

// optional phase timing (build with -DROMAP_FUSED_PROF): clock64 cycles per
// phase summed over CTAs, read back with romap_debug_fused_prof
#ifdef ROMAP_FUSED_PROF
__device__ unsigned long long g_fprof[16];
__device__ unsigned long long g_cta_ns[2 * 1024];   // per CTA: %globaltimer at entry, at exit (last launch)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}
extern "C" __attribute__((visibility("default"))) int romap_debug_fused_cta_ns(unsigned long long* out, int n) {
    cudaDeviceSynchronize();
    return (int)cudaMemcpyFromSymbol(out, g_cta_ns, sizeof(unsigned long long) * 2 * (n < 1024 ? n : 1024));
}
#define FP_MARK(var) const long long var = clock64()
#define FP_ACC(slot, a, b) do { if (fp_on) atomicAdd(&g_fprof[slot], (unsigned long long)((b) - (a))); } while (0)
extern "C" __attribute__((visibility("default"))) int romap_debug_fused_prof(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_fprof, sizeof(g_fprof));
    if (reset) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_fprof, z, sizeof z);
    }
    return 0;
}
#else
#define FP_MARK(var)
#define FP_ACC(slot, a, b)
#endif

namespace {

// experiment hooks (timing only, wrong results): -DROMAP_EXP_NORED drops the
// scatter REDs, -DROMAP_EXP_NOLDG the gathers; operands stay live via empty asm
#ifdef ROMAP_EXP_NORED
__device__ __forceinline__ void xred4(float4* p, float a, float b, float c, float d) {
    asm volatile("" :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d));
}
__device__ __forceinline__ void xred2(float2* p, float a, float b) { asm volatile("" :: "l"(p), "f"(a), "f"(b)); }
#else
#define xred4 red_add_f4
#define xred2 red_add_f2
#endif
#ifdef ROMAP_EXP_NOLDG
__device__ __forceinline__ uint4 xldg4(const void* p) {
    uint4 v;
    asm volatile("mov.b64 {%0, %1}, %4;\n mov.b64 {%2, %3}, %4;" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    const uint32_t k = 0x33ff33ffu;             // finite fp16 halves
    return make_uint4(v.x & k, v.y & k, v.z & k, v.w & k);
}
__device__ __forceinline__ uint32_t xldg1(const void* p) {
    uint32_t v, w;
    asm volatile("mov.b64 {%0, %1}, %2;" : "=r"(v), "=r"(w) : "l"(p));
    return (v ^ w) & 0x33ff33ffu;
}
#else
#define xldg4 ldg_v4
#define xldg1 ldg_u32
#endif

constexpr int TILE = 128;                      // samples per tile
#ifndef ROMAP_NGW
#define ROMAP_NGW 2
#endif
#ifndef ROMAP_LPT
#define ROMAP_LPT 2
#endif
constexpr int NGW = ROMAP_NGW;                 // gather/scatter warpgroups
constexpr int LPT = ROMAP_LPT;                 // hash levels per trip of a G thread
#ifndef ROMAP_NB
#define ROMAP_NB 3
#endif
constexpr int NB = ROMAP_NB;                   // G <-> M hand-off slots (X0, DF, barriers)
constexpr int NG = 128 * NGW;                  // gather/scatter threads
constexpr int NM = 128;                        // MLP/render threads (M)
constexpr int NT = NG + NM;
constexpr int BAR_M = 1;                       // named barrier of M
#ifndef ROMAP_MERGE_RES
#define ROMAP_MERGE_RES 41
#endif
#ifndef ROMAP_MERGE8_RES
#define ROMAP_MERGE8_RES 0
#endif
constexpr int MERGE_RES = ROMAP_MERGE_RES;     // levels below this resolution merge same-cell scatters
constexpr int MERGE8_RES = ROMAP_MERGE8_RES;   // ... and below this one over windows of 8 (3 steps)

// shared-memory layout (bytes); every block is a multiple of 1024
constexpr int OFF_W1 = 0;                      // 64 x LF(<=32)
constexpr int OFF_W2 = OFF_W1 + 64 * 32 * 2;   // 16 x 64
constexpr int OFF_W3 = OFF_W2 + 16 * 64 * 2;   // 64 x 32
constexpr int OFF_W4 = OFF_W3 + 64 * 32 * 2;   // 64 x 64
constexpr int OFF_W5 = OFF_W4 + 64 * 64 * 2;   // 16 x 64 (rows 3..15 zero)
constexpr int X0_BYTES = TILE * 32 * 2;
constexpr int OFF_X0 = OFF_W5 + 16 * 64 * 2;   // NB slots x 128 x LF
constexpr int OFF_H1 = OFF_X0 + NB * X0_BYTES; // 128 x 64
constexpr int OFF_CIN = OFF_H1 + TILE * 64 * 2;
constexpr int OFF_WH2 = OFF_CIN;               // network 1 (no CIN): third 64 x 64 hidden layer
constexpr int OFF_G1 = OFF_CIN + TILE * 32 * 2;
constexpr int OFF_G2 = OFF_G1 + TILE * 64 * 2;
constexpr int OFF_DC = OFF_G2 + TILE * 64 * 2;  // 128 x 16
constexpr int OFF_DR = OFF_DC + TILE * 16 * 2;  // 128 x 16
constexpr int OFF_DB = OFF_DR + TILE * 16 * 2;  // 128 x 64 (dg2, dh1)
// dg1 (its producer overlaps the dW MMAs reading DB): G2's space, dead by then
// (B5's dW5 MMAs are covered by B4's commit; network 1 likewise after W_out)
constexpr int OFF_DB2 = OFF_G2;
constexpr int OFF_MISC = OFF_DB + TILE * 64 * 2;
constexpr int SMEM_BYTES = OFF_MISC + 1024;

// TMEM columns (one CTA per SM, so the whole 512-column allocation is free)
constexpr int TM_WK = 0;      // working accumulator (<= 64 cols)
constexpr int TM_DF = 384;    // NB x 32: dfeat of tile slot b at TM_DF + 32 b
constexpr int TM_DW1 = 128;   // dW1   [64 x LF]
constexpr int TM_DW3 = 160;   // dW3   [64 x 32]
constexpr int TM_DW4 = 192;   // dW4   [64 x 64]
constexpr int TM_DW2 = 256;   // dW2^T [64 x 16]
constexpr int TM_DW5 = 272;   // dW5^T [64 x 16]
constexpr int TM_DWH2 = 320;  // network 1: dW of the second 64 x 64 hidden layer
constexpr int TM_COLS = 512;
// network 1 (R24) slots: W1 -> OFF_W1 / TM_DW1; hidden k = 1, 2 (64 x 64) ->
// OFF_W4 / TM_DW4 and OFF_WH2 / TM_DWH2; W_out (4 x 64, rows 4..15 zero) ->
// OFF_W2 / TM_DW2 (dW_out^T); activations h_1, h_2, h_3 -> H1, G1, G2

struct Misc {
    uint64_t mbar_mma;        // M: completion of its own MMA groups
    uint64_t x0_full[NB];
    uint64_t tile_done[NB];
    uint64_t df_empty[NB];
    uint32_t tmem;
    int pad;
    float loss[4];
    float xw[4][8];           // M cross-warp scan exchange (per warp, 8 slots)
    int4 lv[ROMAP_MAX_LEVELS];    // per level: res, y multiplier, z multiplier, dense (R5)
    int lvoff[ROMAP_MAX_LEVELS];  // entry offset of the level
};
static_assert(sizeof(Misc) <= 1024, "misc block");

// fence generic smem writes for the tensor core, then sync M
__device__ __forceinline__ void m_sync_for_mma() {
    tc::fence_async_smem();
    tc::fence_before();
    tc::bar_sync(BAR_M, NM);
    tc::fence_after();
}

// ---------------------------------------------------------------------------
// segmented scans over the N samples of each ray, on M's 128 threads
// (thread m = sample m of the tile; a ray covers N consecutive threads)
template <bool MUL>
__device__ __forceinline__ float op2(float a, float b) { return MUL ? a * b : a + b; }

template <bool MUL>
__device__ __forceinline__ float warp_incl(float x, int sw, int lane) {
    float incl = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        if (off >= sw) break;
        float y = __shfl_up_sync(0xffffffffu, incl, off, sw);
        if ((lane & (sw - 1)) >= off) incl = op2<MUL>(incl, y);
    }
    return incl;
}

// all render scans of a tile with ONE cross-warp exchange (Eq. 6 forward and
// backward).  Per sample i of a ray: T_i (exclusive product of alpha), the ray's
// T_N, w_i = T_i o_i, the ray sums of w c_k, w dist and sigma, and the exclusive
// suffix sums suf_k,i = sum_{j>i} w_j q_j, q = (c_0, c_1, c_2, dist).  Within a
// warp segment everything is computed with the local transmittance T^loc (product
// restarted at the segment); a ray over several warps (N > 32) then exchanges each
// warp's segment product A_w and segment sums S_w once: with carry_w = product of
// A over the ray's earlier warps, T = carry T^loc, w = carry w^loc, ray sum =
// sum_w carry_w S_w, suffix = carry suf^loc + sum_{later w} carry_w S_w.
struct RScan {
    float T, TN, w, sums[5], suf[4];
};
__device__ __forceinline__ void m_render_scan(float alpha, float o, bool active, const float c[3], float dist,
                                              float sig, int N, float* xw, RScan& R) {
    const int lane = threadIdx.x & 31, mw = (threadIdx.x - NG) >> 5;
    const int sw = N < 32 ? N : 32;
    const int sl = lane & (sw - 1);
    const float incl = warp_incl<true>(alpha, sw, lane);
    float Tl = __shfl_up_sync(0xffffffffu, incl, 1, sw);
    if (sl == 0) Tl = 1.f;
    const float A = __shfl_sync(0xffffffffu, incl, sw - 1, sw);
    const float wl = active ? Tl * o : 0.f;
    float qi[4] = {wl * c[0], wl * c[1], wl * c[2], wl * dist};
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        if (off >= sw) break;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float y = __shfl_down_sync(0xffffffffu, qi[k], off, sw);
            if (sl + off < sw) qi[k] += y;
        }
    }
    float qe[4], qt[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        qe[k] = __shfl_down_sync(0xffffffffu, qi[k], 1, sw);
        if (sl == sw - 1) qe[k] = 0.f;
        qt[k] = __shfl_sync(0xffffffffu, qi[k], 0, sw);
    }
    float ss = sig;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
        if (off < sw) ss += __shfl_xor_sync(0xffffffffu, ss, off, sw);
    if (N <= 32) {
        R.T = Tl;
        R.TN = A;
        R.w = wl;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            R.sums[k] = qt[k];
            R.suf[k] = qe[k];
        }
        R.sums[4] = ss;
        return;
    }
    if (lane == 0) {
        xw[mw * 8 + 0] = A;
#pragma unroll
        for (int k = 0; k < 4; ++k) xw[mw * 8 + 1 + k] = qt[k];
        xw[mw * 8 + 5] = ss;
    }
    tc::bar_sync(BAR_M, NM);
    const int wpr = N >> 5, w0 = mw - (mw % wpr);
    float carry = 1.f, cw = 1.f, later[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 5; ++k) R.sums[k] = 0.f;
    for (int w = w0; w < w0 + wpr; ++w) {
        if (w == mw) carry = cw;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float v = cw * xw[w * 8 + 1 + k];
            R.sums[k] += v;
            if (w > mw) later[k] += v;
        }
        R.sums[4] += xw[w * 8 + 5];
        cw *= xw[w * 8 + 0];
    }
    R.TN = cw;
    R.T = carry * Tl;
    R.w = carry * wl;
#pragma unroll
    for (int k = 0; k < 4; ++k) R.suf[k] = carry * qe[k] + later[k];
}

// ---------------------------------------------------------------------------
// copy one object's fp16 weights into the interleaved smem layout (M threads)
__device__ void load_weights(uint8_t* smem, const __half* __restrict__ mlp16, const CfgDev& cfg, int LF) {
    struct Lw { int off, rows, cols, srows, smem; };
    Lw ls[5] = {{cfg.w_off[0], 64, LF, 64, OFF_W1}, {cfg.w_off[1], 16, 64, 16, OFF_W2},
                {cfg.w_off[2], 64, 32, 64, OFF_W3}, {cfg.w_off[3], 64, 64, 64, OFF_W4},
                {cfg.w_off[4], 3, 64, 16, OFF_W5}};
    int nl = 5;
    if (cfg.net == 1) {
        const int hl = cfg.hl;
        ls[1] = {cfg.w_off[hl], 4, 64, 16, OFF_W2};
        ls[2] = {cfg.w_off[1], 64, 64, 64, OFF_W4};
        ls[3] = {cfg.w_off[2], 64, 64, 64, OFF_WH2};
        nl = hl + 1;       // W1, W_out, then hl - 1 hidden layers
    }
    const int m = threadIdx.x - NG;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        if (k >= nl) break;
        const int chunks = ls[k].srows * (ls[k].cols / 8);
        for (int q = m; q < chunks; q += NM) {
            const int r = q / (ls[k].cols / 8), cb = q % (ls[k].cols / 8);
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

// flush the dW accumulators (TMEM) and loss sums of one object (M threads).
// M=64 accumulators: row i lives in TMEM lane 32 (i / 16) + i % 16.
// (STORE: plain stores into a per-tile buffer laid out like the MLP block, the
// deterministic mode's per-tile partials; else fp32 REDs into the gradients)
__device__ __forceinline__ void emit4(bool store, float* p, float a, float b, float c, float d) {
    if (store) *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
    else red_add_f4(reinterpret_cast<float4*>(p), a, b, c, d);
}
__device__ __forceinline__ void emit1(bool store, float* p, float a) {
    if (store) *p = a;
    else red_add_f1(p, a);
}
template <int LF, bool STORE = false>
__device__ void m_flush(const CfgDev& cfg, float* gm, uint32_t tm, Misc* misc, double* loss_acc, int slot,
                        bool have_dw) {
    const int m = threadIdx.x - NG, mw = m >> 5, lane = m & 31;
    const float inv = 1.0f / cfg.loss_scale;
    if (have_dw) {
        const int row = mw * 16 + lane;
        const bool on = lane < 16;
        float v[16];
        auto rows4 = [&](int col, float* dst) {   // 16 contiguous columns of row `row`
            tc::tmem_ld16_sync(tc::taddr(tm, mw * 32, col), v);
            if (on)
#pragma unroll
                for (int k = 0; k < 16; k += 4)
                    emit4(STORE, dst + k, v[k] * inv, v[k + 1] * inv, v[k + 2] * inv, v[k + 3] * inv);
        };
#pragma unroll
        for (int c0 = 0; c0 < LF; c0 += 16) rows4(TM_DW1 + c0, gm + cfg.w_off[0] + row * LF + c0);
        if (cfg.net == 1) {
            const int hl = cfg.hl;
            for (int k = 1; k < hl; ++k)
#pragma unroll
                for (int c0 = 0; c0 < 64; c0 += 16)
                    rows4((k == 1 ? TM_DW4 : TM_DWH2) + c0, gm + cfg.w_off[k] + row * 64 + c0);
            // dW_out^T [64 in x 16 (4) out]
            tc::tmem_ld16_sync(tc::taddr(tm, mw * 32, TM_DW2), v);
            if (on)
#pragma unroll
                for (int o = 0; o < 4; ++o) emit1(STORE, gm + cfg.w_off[hl] + o * 64 + row, v[o] * inv);
        } else {
#pragma unroll
        for (int c0 = 0; c0 < 32; c0 += 16) rows4(TM_DW3 + c0, gm + cfg.w_off[2] + row * 32 + c0);
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) rows4(TM_DW4 + c0, gm + cfg.w_off[3] + row * 64 + c0);
        // dW2^T [64 in x 16 out], dW5^T [64 in x 16 (3) out]: row = input feature
        tc::tmem_ld16_sync(tc::taddr(tm, mw * 32, TM_DW2), v);
        if (on)
#pragma unroll
            for (int o = 0; o < 16; ++o) emit1(STORE, gm + cfg.w_off[1] + o * 64 + row, v[o] * inv);
        tc::tmem_ld16_sync(tc::taddr(tm, mw * 32, TM_DW5), v);
        if (on)
#pragma unroll
            for (int o = 0; o < 3; ++o) emit1(STORE, gm + cfg.w_off[4] + o * 64 + row, v[o] * inv);
        }
    }
    tc::bar_sync(BAR_M, NM);
    if (m < 4) {
        const float l = misc->loss[m];
        if (l != 0.f) atomicAdd(loss_acc + 4 * slot + m, (double)l);
        misc->loss[m] = 0.f;
    }
    tc::fence_before();
    tc::bar_sync(BAR_M, NM);
    tc::fence_after();
}

// backward epilogue: dX (TMEM) masked by the ReLU derivative of the forward
// activation `act` (its fp16 ReLU output in smem: relu' = act > 0) -> fp16 -> smem
__device__ __forceinline__ void epi_mask64(uint32_t wk, uint8_t* out, const uint8_t* act, int r) {
    const __half2 z = __float2half2_rn(0.f);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        float v[32];
        tc::tmem_ld32_sync(wk + 32 * h, v);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t off = tc::il_offset(r, 32 * h + 8 * c, 64);
#ifdef ROMAP_EXP_NOMSTS
            uint4 a4;
            asm volatile("mov.b32 %0, 0x3c003c00;\n mov.b32 %1, 0;\n mov.b32 %2, 0x3c000000;\n mov.b32 %3, 0x3c00;"
                         : "=r"(a4.x), "=r"(a4.y), "=r"(a4.z), "=r"(a4.w));
#else
            uint4 a4 = *reinterpret_cast<const uint4*>(act + off);
#endif
            const __half2* a = reinterpret_cast<const __half2*>(&a4);
            __half2 q[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                q[k] = __hmul2(__floats2half2_rn(v[8 * c + 2 * k], v[8 * c + 2 * k + 1]), __hgt2(a[k], z));
            tc::sts128(out + off, *reinterpret_cast<uint4*>(q));
        }
    }
}

// ---------------------------------------------------------------------------
// G: gathers of tile `it` interleaved with the scatter of tile `it - NB`
// (warpgroup WG owns the level pairs (p, L-1-p) with p = WG, WG + 2, ...: a coarse
// and a fine level per trip; one code path for both
// warpgroups, level loop not unrolled: the body stays in the instruction cache)
template <int L>
__device__ __forceinline__ void g_loop(const CfgDev& cfg, const ObjDev* __restrict__ objs,
                                       const RayRec* __restrict__ rays, const float4* __restrict__ srec, int tile0,
                                       int tstride, int n, uint8_t* smem, Misc* misc, uint32_t tm DET_PARAM) {
    constexpr int LF = 2 * L;
    const int t = threadIdx.x, r = t & (TILE - 1), lane = t & 31, q4 = (t >> 5) & 3, WG = t >> 7;
    const int N = cfg.N;
    const unsigned hmask = (unsigned)cfg.T - 1u;
    const float inv_scale = 1.0f / cfg.loss_scale;
    const uint32_t df_lane = tc::taddr(tm, q4 * 32, TM_DF);
    const unsigned ray_key = (unsigned)(lane / N) << 24;   // ray of this lane within the warp (N = 2^k)

    // tile j of this CTA = tile0 + j * tstride (strided over the grid: all CTAs
    // work on neighbouring tiles, i.e. on the same object, at any time)
    float4 u_next = srec[(long long)tile0 * TILE + r];
    const int lgN = __ffs(N) - 1;                      // N is a power of two (romap_create_object)
    int slot_next = rays[(int)(((long long)tile0 * TILE) >> lgN)].slot;
    int slot_tab = -1;
    const uint32_t* tab = nullptr;                // fp16 table: one 4-byte (half2) word per entry
    float2* g_cur = nullptr;
    float um[NB][3];                              // positions of tiles it-1 .. it-NB (-1: inactive)
    float2* gm[NB];                               // their gradient tables
#ifdef ROMAP_DET
    int sl[NB];                                   // their object slots (record keys)
#endif
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        um[k][0] = um[k][1] = um[k][2] = -1.f;
        gm[k] = nullptr;
#ifdef ROMAP_DET
        sl[k] = 0;
#endif
    }

#ifdef ROMAP_FUSED_PROF
    const bool fp_on = (t & 127) == 0;
#endif
    FP_MARK(g_start);
    for (int it = 0; it < n + NB; ++it) {
        const bool dg = it < n, ds = it >= NB;       // gather tile it, scatter tile it - NB
        const int b = it % NB;
        const bool ag = u_next.x >= 0.f;              // sample of an active ray (k_raygen + k_samples)
        const float ug[3] = {u_next.x, u_next.y, u_next.z};
        const int slot_g = slot_next;
        if (it + 1 < n) {
            const long long tn = (long long)tile0 + (long long)(it + 1) * tstride;
            u_next = srec[tn * TILE + r];
            slot_next = rays[(int)((tn * TILE) >> lgN)].slot;
        }
        if (dg && slot_g != slot_tab) {
            tab = reinterpret_cast<const uint32_t*>(objs[slot_g].p16);
            g_cur = reinterpret_cast<float2*>(objs[slot_g].g32);
            slot_tab = slot_g;
        }
        FP_MARK(g_w0);
        if (ds) {                                     // dfeat of tile it-NB is in DF[b], X0[b] is free
            tc::mbar_wait(&misc->tile_done[b], ((it - NB) / NB) & 1);
            tc::fence_after();
        }
        FP_MARK(g_w1);
        FP_ACC(9, g_w0, g_w1);
        const bool as = ds && um[NB - 1][0] >= 0.f;   // scattered sample of an active ray
        const unsigned flags_it = (dg ? 1u : 0u) | (ds ? 2u : 0u) | (dg && ag ? 4u : 0u) | (as ? 8u : 0u);
        uint8_t* X0 = smem + OFF_X0 + b * X0_BYTES;
#pragma unroll 1
        for (int pp = WG; pp < L / LPT; pp += NGW) {   // level groups (LPT levels) of this warpgroup
            // opaque copy of the iteration flags: keeps the compiler from
            // unswitching this loop into one copy per flag combination
            unsigned fl;
            asm volatile("mov.b32 %0, %1;" : "=r"(fl) : "r"(flags_it));
            const bool dg_ = fl & 1u, ds_ = fl & 2u, ag_ = fl & 4u, as_ = fl & 8u;
            // levels of this trip: with 2 per trip, pair pp = (pp, L - 1 - pp), a coarse
            // level with a fine one, so the two warpgroups carry the same mix of
            // merged (coarse) and plain (fine) scatters
            int lv_[LPT];
            if constexpr (LPT == 2) {
                lv_[0] = pp;
                lv_[1] = L - 1 - pp;
            } else {
                lv_[0] = pp;
            }
            int4 P[LPT];
            unsigned off[LPT];
#pragma unroll
            for (int q = 0; q < LPT; ++q) {
                P[q] = misc->lv[lv_[q]];
                off[q] = (unsigned)misc->lvoff[lv_[q]];
            }
            // (1) gathers of the trip's levels of tile it.  x-neighbour corners (b, b|1)
            // share a 16-byte chunk of the fp16 table in 3 of 4 cases (dense:
            // entries e, e+1; hashed: e ^ (x ^ (x+1)) with the x prime = 1), so each
            // corner pair is one 16-B gather (+ a 4-B one otherwise); level blocks
            // are 16-entry aligned (R5).
            uint4 qv[LPT][4];
            uint32_t xv[LPT][4];
            unsigned e[LPT][8];
            Cell cl[LPT];
#pragma unroll
            for (int q = 0; q < LPT; ++q) {
                // level-relative entries; the level's block starts at tab + off
                // (16-entry aligned, R5, so chunk / pair alignment is the same)
                level_entries(ug, P[q], 0u, hmask, cl[q], e[q]);
                const uint32_t* tl = opaque_ptr(tab + off[q]);
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const bool same = (e[q][2 * p] >> 2) == (e[q][2 * p + 1] >> 2);
                    // inactive samples (u = -1) read zeros: bounded features for their
                    // (masked) MLP rows
                    qv[q][p] = ag_ ? xldg4(tl + opaque_u32(e[q][2 * p] & ~3u)) : make_uint4(0, 0, 0, 0);
                    xv[q][p] = (ag_ && !same) ? xldg1(tl + e[q][2 * p + 1]) : 0u;
                }
            }
            // (2) scatter of the same levels of tile it-NB (fire-and-forget REDs).
            // Coarse levels (res < MERGE_RES): consecutive samples of a ray often
            // share a cell, i.e. all 8 corners; a 2-step warp segmented sum over
            // runs of equal cells lets one lane per 4 run members issue the REDs
            // (RED requests, not bytes, bound this kernel).
            if (ds_) {
                float g[4];
                if constexpr (LPT == 2)
                    tc::tmem_ld2x2_sync(df_lane + 32 * b + 2 * lv_[0], df_lane + 32 * b + 2 * lv_[1], g);
                else
                    tc::tmem_ld4_sync(df_lane + 32 * b + 2 * lv_[0], g);
#pragma unroll
                for (int q = 0; q < LPT; ++q) {
                    Cell cs;
                    unsigned es[8];
                    level_entries(um[NB - 1], P[q], 0u, hmask, cs, es);
                    float2* gl = opaque_ptr(gm[NB - 1] + off[q]);
                    const float g0 = as_ ? g[2 * q] * inv_scale : 0.f, g1 = as_ ? g[2 * q + 1] * inv_scale : 0.f;
                    float v[16];
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        const float wa = corner_weight(cs, 2 * p), wb = corner_weight(cs, 2 * p + 1);
                        v[4 * p] = wa * g0;
                        v[4 * p + 1] = wa * g1;
                        v[4 * p + 2] = wb * g0;
                        v[4 * p + 3] = wb * g1;
                    }
#ifdef ROMAP_DET
                    {
                        // one record per corner (sample, level, corner order); k_det.cu sums
                        // each entry's records in that order
                        const long long s_sc = ((long long)tile0 + (long long)(it - NB) * tstride) * TILE + r;
                        const long long rec = (s_sc * L + lv_[q]) * 8;
                        const unsigned long long kb = (unsigned long long)sl[NB - 1] << 32;
#pragma unroll
                        for (int c8 = 0; c8 < 8; ++c8) {
                            det.key[rec + c8] = as_ ? (kb | (unsigned long long)(off[q] + es[c8])) : DET_NO_KEY;
                            det.val[rec + c8] = make_float2(v[2 * c8], v[2 * c8 + 1]);
                        }
                    }
                    if (false) {
#else
                    {
#endif
                    // fine levels: every lane issues (an inactive sample adds zeros: one
                    // request, no branch); coarse levels: the run leaders of active samples
                    bool issue = true;
                    if (P[q].x < MERGE_RES) {                     // warp-uniform
                        // key = (ray of the warp, cell): a straight ray visits each cell in one
                        // contiguous run of samples, so equal keys are contiguous lanes
                        // (with N < 32 several rays share a warp and may cross the same cell)
                        const unsigned key = as_ ? ((unsigned)cs.c[0] | ((unsigned)cs.c[1] << 8) |
                                                    ((unsigned)cs.c[2] << 16) | ray_key)
                                                 : (0x80000000u | (unsigned)lane);
                        const int omax = P[q].x < MERGE8_RES ? 4 : 2;
                        const unsigned wmask = 2u * omax - 1u;
#pragma unroll
                        for (int o = 1; o <= 4; o <<= 1) {
                            if (o > omax) break;
                            const unsigned ko = __shfl_down_sync(0xffffffffu, key, o);
                            const bool mg = lane + o < 32 && ko == key;
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                const float w = __shfl_down_sync(0xffffffffu, v[k], o);
                                if (mg) v[k] += w;
                            }
                        }
                        // lane holds the sum over [lane, lane + 4) of its run; the
                        // lanes at run start + 4 m issue
                        const unsigned kp = __shfl_up_sync(0xffffffffu, key, 1);
                        const unsigned starts = __ballot_sync(0xffffffffu, lane == 0 || kp != key);
                        const int run0 = 31 - __clz(starts & (0xffffffffu >> (31 - lane)));
                        issue = as_ && ((lane - run0) & wmask) == 0;
                    }
#if defined(ROMAP_EXP_NORED_COARSE)                 // experiment: no REDs on the merged (coarse) levels
                    if (P[q].x < MERGE_RES) { asm volatile("" :: "f"(v[0]), "f"(v[15])); issue = false; }
#elif defined(ROMAP_EXP_NORED_FINE)                 // experiment: no REDs on the other levels
                    if (P[q].x >= MERGE_RES) { asm volatile("" :: "f"(v[0]), "f"(v[15])); issue = false; }
#endif
                    if (issue) {
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        // one REDG.F32x4 at the aligned 16-B pair of fp32 entries holding the
                        // base corner (its x-neighbour's slot carries the neighbour's values when
                        // it shares the pair, else zeros), plus a REDG.F32x2 for a neighbour
                        // outside the pair; only that one is conditional
                        const unsigned ea = es[2 * p], eb = es[2 * p + 1];
                        const bool pair = (ea >> 1) == (eb >> 1), a_lo = (ea & 1u) == 0u;
                        const float n0 = pair ? v[4 * p + 2] : 0.f, n1 = pair ? v[4 * p + 3] : 0.f;
                        const float4 w4 = a_lo ? make_float4(v[4 * p], v[4 * p + 1], n0, n1)
                                               : make_float4(n0, n1, v[4 * p], v[4 * p + 1]);
                        xred4(reinterpret_cast<float4*>(gl + opaque_u32(ea & ~1u)), w4.x, w4.y, w4.z, w4.w);
                        if (!pair) xred2(gl + eb, v[4 * p + 2], v[4 * p + 3]);
                    }
                    }
                    }
                }
            }
            // (3) trilinear interpolation of the gathered fp16 corners as x, then y,
            // then z lerps in fp32 (-DROMAP_LERP16: packed-fp16 lerps, 2 % faster,
            // ~25 % larger first-layer / table gradient error) -> fp16 X0[b]
            if (dg_) {
                __half2 fq[LPT];
#pragma unroll
                for (int q = 0; q < LPT; ++q) {
                    const __half2 fx = __float2half2_rn(cl[q].f[0]), fy = __float2half2_rn(cl[q].f[1]),
                                  fz = __float2half2_rn(cl[q].f[2]);
                    __half2 vx[4];
                    float2 vx32[4];
                    (void)vx;
                    (void)vx32;
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        const unsigned ea = e[q][2 * p], eb = e[q][2 * p + 1];
                        const bool same = (ea >> 2) == (eb >> 2);
                        const uint32_t h0 = sel4(qv[q][p], ea & 3);
                        const uint32_t h1 = selp_u32(same, sel4(qv[q][p], eb & 3), xv[q][p]);
#ifndef ROMAP_LERP16
                        // fp32 lerps of the fp16 corners
                        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&h0));
                        const float2 c = __half22float2(*reinterpret_cast<const __half2*>(&h1));
                        vx32[p] = make_float2(a.x + cl[q].f[0] * (c.x - a.x), a.y + cl[q].f[0] * (c.y - a.y));
#else
                        const __half2 a = *reinterpret_cast<const __half2*>(&h0);
                        const __half2 c = *reinterpret_cast<const __half2*>(&h1);
                        vx[p] = __hfma2(fx, __hsub2(c, a), a);
#endif
                    }
#ifndef ROMAP_LERP16
                    const float fyv = cl[q].f[1], fzv = cl[q].f[2];
                    const float2 y0 = make_float2(vx32[0].x + fyv * (vx32[1].x - vx32[0].x), vx32[0].y + fyv * (vx32[1].y - vx32[0].y));
                    const float2 y1 = make_float2(vx32[2].x + fyv * (vx32[3].x - vx32[2].x), vx32[2].y + fyv * (vx32[3].y - vx32[2].y));
                    fq[q] = __floats2half2_rn(y0.x + fzv * (y1.x - y0.x), y0.y + fzv * (y1.y - y0.y));
#else
                    const __half2 vy0 = __hfma2(fy, __hsub2(vx[1], vx[0]), vx[0]);
                    const __half2 vy1 = __hfma2(fy, __hsub2(vx[3], vx[2]), vx[2]);
                    fq[q] = __hfma2(fz, __hsub2(vy1, vy0), vy0);
#endif
                }
#pragma unroll
                for (int q = 0; q < LPT; ++q)
                    *reinterpret_cast<__half2*>(X0 + tc::il_offset(r, 2 * lv_[q], LF)) = fq[q];
            }
        }
        if (ds) {                                     // DF[b] read: M may overwrite it (tile it)
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&misc->df_empty[b]);
        }
        if (dg) {
            tc::fence_async_smem();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&misc->x0_full[b]);
        }
#pragma unroll
        for (int q = NB - 1; q > 0; --q) {
#pragma unroll
            for (int k = 0; k < 3; ++k) um[q][k] = um[q - 1][k];
            gm[q] = gm[q - 1];
#ifdef ROMAP_DET
            sl[q] = sl[q - 1];
#endif
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) um[0][k] = (dg && ag) ? ug[k] : -1.f;
        gm[0] = g_cur;
#ifdef ROMAP_DET
        sl[0] = slot_tab;
#endif
        FP_MARK(g_w2);
        FP_ACC(10, g_w1, g_w2);
        if (WG == 1) FP_ACC(11, g_w1, g_w2);         // warpgroup G1 alone (G0 = slot 10 - slot 11)
    }
    FP_MARK(g_end);
    FP_ACC(8, g_start, g_end);
}

// per-sample inputs of M, loaded one tile ahead (plain loads placed before the
// tile's barriers, so they are issued early and their latency overlaps a tile)
struct MIn {
    float d[3], tgt[3], bg[3], depth, dist, delta;
    int flags, slot;
};
__device__ __forceinline__ MIn m_load(const RayRec* __restrict__ rays, const float4* __restrict__ srec,
                                      const float* __restrict__ sdelta, long long s, int lgN) {
    const RayRec* rp = rays + (int)(s >> lgN);      // N = 2^lgN samples per ray
    MIn v;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        v.d[k] = rp->d[k];
        v.tgt[k] = rp->tgt[k];
        v.bg[k] = rp->bg[k];
    }
    v.depth = rp->depth;
    v.flags = rp->flags;
    v.slot = rp->slot;
    v.dist = srec[s].w;
    v.delta = sdelta[s];
    return v;
}

// ---------------------------------------------------------------------------
// M: SH + MLP forward + render/loss + MLP backward of tile j
template <int L, int NET>
__device__ __forceinline__ void m_loop(const CfgDev& cfg, const ObjDev* __restrict__ objs,
                                       const RayRec* __restrict__ rays, const float4* __restrict__ srec,
                                       const float* __restrict__ sdelta, int tile0, int tstride, int n, uint8_t* smem,
                                       Misc* misc,
                                       uint32_t tm, double* __restrict__ loss_acc, int* __restrict__ nonfinite,
                                       float* __restrict__ dbg DET_PARAM) {
    constexpr int LF = 2 * L;
    const int m = threadIdx.x - NG, mw = m >> 5;
    const bool leader = m == 0;
    const int N = cfg.N;
    const float scale = cfg.loss_scale;
    const uint32_t wk = tc::taddr(tm, mw * 32, TM_WK);
    const uint32_t sW1 = tc::smem_u32(smem + OFF_W1), sW2 = tc::smem_u32(smem + OFF_W2),
                   sW3 = tc::smem_u32(smem + OFF_W3), sW4 = tc::smem_u32(smem + OFF_W4),
                   sW5 = tc::smem_u32(smem + OFF_W5), sH1 = tc::smem_u32(smem + OFF_H1),
                   sCIN = tc::smem_u32(smem + OFF_CIN), sG1 = tc::smem_u32(smem + OFF_G1),
                   sG2 = tc::smem_u32(smem + OFF_G2), sDC = tc::smem_u32(smem + OFF_DC),
                   sDR = tc::smem_u32(smem + OFF_DR), sDB = tc::smem_u32(smem + OFF_DB),
                   sDB2 = tc::smem_u32(smem + OFF_DB2),
                   sWH2 = tc::smem_u32(smem + OFF_WH2);
    uint8_t* H1 = smem + OFF_H1;
    uint8_t* CIN = smem + OFF_CIN;
    uint8_t* G1 = smem + OFF_G1;
    uint8_t* G2 = smem + OFF_G2;
    uint8_t* DC = smem + OFF_DC;
    uint8_t* DR = smem + OFF_DR;
    uint8_t* DB = smem + OFF_DB;
    uint8_t* DB2 = smem + OFF_DB2;
    float* xw = &misc->xw[0][0];
    uint32_t phase = 0;
    auto mma_wait = [&]() {
        tc::mbar_wait(&misc->mbar_mma, phase);
        phase ^= 1;
        tc::fence_after();
    };

    int cur = -1;
    bool dw_fresh = true;
    float invB = 0.f;
#ifdef ROMAP_FUSED_PROF
    const bool fp_on = m == 0;
#endif
    FP_MARK(m_start);
    const int lgN = __ffs(N) - 1;                      // N is a power of two (romap_create_object)
    MIn nx = m_load(rays, srec, sdelta, (long long)tile0 * TILE + m, lgN);
    for (int j = 0; j < n; ++j) {
        FP_MARK(m_t0);
        const long long tile = (long long)tile0 + (long long)j * tstride;
        const int b = j % NB;
        const long long s = (long long)tile * TILE + m;
        const int i = (int)(s & (N - 1));
        const MIn rr = nx;
        if (j + 1 < n) nx = m_load(rays, srec, sdelta, s + (long long)tstride * TILE, lgN);
        const float delta = rr.delta;
        const bool active = (rr.flags & RF_ACTIVE) != 0;
        if (rr.slot != cur) {                      // uniform: a tile holds rays of one object
            if (cur >= 0) {
                // every MMA of the previous tile (they read W and write dW) has completed
                tc::mbar_wait(&misc->tile_done[(j - 1) % NB], ((j - 1) / NB) & 1);
                tc::fence_after();
                m_flush<LF>(cfg, objs[cur].g32 + cfg.n_table, tm, misc, loss_acc, cur, !dw_fresh);
            }
            const ObjDev& ob = objs[rr.slot];
            load_weights(smem, ob.p16 + cfg.n_table, cfg, LF);
            cur = rr.slot;
            dw_fresh = true;
            invB = 1.0f / (float)ob.n_rays;
        }
        if constexpr (NET == 0) {    // SH(4) of the view direction (network 1 has no colour net; WH2 aliases CIN)
            float sh[16];
            sh4(rr.d, sh);
            tc::st16(CIN, m, 16, 32, sh);
        }
        FP_MARK(m_t1);
        tc::mbar_wait(&misc->x0_full[b], (j / NB) & 1);
        FP_MARK(m_t2);
#ifdef ROMAP_EXP_NOM
        if (leader) {                                  // experiment: M hands the tile straight back
            if (j >= NB) tc::mbar_wait(&misc->df_empty[b], ((j - NB) / NB) & 1);
            tc::fence_after();
            tc::commit(&misc->tile_done[b]);
        }
        dw_fresh = false;
        continue;
#endif
        m_sync_for_mma();
        const uint32_t sX0 = tc::smem_u32(smem + OFF_X0 + b * X0_BYTES);

        float sigma, r0, c[3];
        if constexpr (NET == 0) {
        // ---- a4: MLP forward
        // L1: WK[128 x 64] = X0[128 x LF] . W1^T
        if (leader) {
#pragma unroll
            for (int ks = 0; ks < LF / 16; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sX0, LF, ks), tc::desc_kmajor(sW1, LF, ks),
                            tc::idesc_f16(128, 64, false, false), ks > 0);
            tc::commit(&misc->mbar_mma);
        }
        mma_wait();
        tc::epi_relu64(wk, H1, m);
        m_sync_for_mma();
        // L2: WK[128 x 16] = H1 . W2^T
        if (leader) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sH1, 64, ks), tc::desc_kmajor(sW2, 64, ks),
                            tc::idesc_f16(128, 16, false, false), ks > 0);
            tc::commit(&misc->mbar_mma);
        }
        mma_wait();
        {
            float v[16];
            tc::tmem_ld16_sync(wk, v);
            r0 = v[0];
            sigma = density_act(r0, cfg.density_act);
            tc::st16(CIN, m, 0, 32, v);
        }
        m_sync_for_mma();
        // L3: WK = CIN . W3^T
        if (leader) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sCIN, 32, ks), tc::desc_kmajor(sW3, 32, ks),
                            tc::idesc_f16(128, 64, false, false), ks > 0);
            tc::commit(&misc->mbar_mma);
        }
        mma_wait();
        tc::epi_relu64(wk, G1, m);
        m_sync_for_mma();
        // L4: WK = G1 . W4^T
        if (leader) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sG1, 64, ks), tc::desc_kmajor(sW4, 64, ks),
                            tc::idesc_f16(128, 64, false, false), ks > 0);
            tc::commit(&misc->mbar_mma);
        }
        mma_wait();
        tc::epi_relu64(wk, G2, m);
        m_sync_for_mma();
        // L5: WK[128 x 16] = G2 . W5^T (rows 3..15 of W5 are zero)
        if (leader) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sG2, 64, ks), tc::desc_kmajor(sW5, 64, ks),
                            tc::idesc_f16(128, 16, false, false), ks > 0);
            tc::commit(&misc->mbar_mma);
        }
        mma_wait();
        {
            float v[16];
            tc::tmem_ld16_sync(wk, v);
#pragma unroll
            for (int k = 0; k < 3; ++k) c[k] = 1.0f / (1.0f + expf(-v[k]));
        }

        } else {
        // ---- a4: MLP forward, network 1 (R24): h_1 = relu(X0 W1^T), h_k = relu(h_{k-1} W_k^T),
        // raw = h_hl W_out^T (16 cols, rows 4..15 of W_out zero): sigma = act(raw_0), c = sigmoid(raw_1..3)
        if (leader) {
#pragma unroll
            for (int ks = 0; ks < LF / 16; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sX0, LF, ks), tc::desc_kmajor(sW1, LF, ks),
                            tc::idesc_f16(128, 64, false, false), ks > 0);
            tc::commit(&misc->mbar_mma);
        }
        mma_wait();
        tc::epi_relu64(wk, H1, m);
        m_sync_for_mma();
        for (int k = 1; k < cfg.hl; ++k) {
            const uint32_t sA = k == 1 ? sH1 : sG1, sW = k == 1 ? sW4 : sWH2;
            if (leader) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sA, 64, ks), tc::desc_kmajor(sW, 64, ks),
                                tc::idesc_f16(128, 64, false, false), ks > 0);
                tc::commit(&misc->mbar_mma);
            }
            mma_wait();
            tc::epi_relu64(wk, k == 1 ? G1 : G2, m);
            m_sync_for_mma();
        }
        {
            const uint32_t sHL = cfg.hl == 1 ? sH1 : (cfg.hl == 2 ? sG1 : sG2);
            if (leader) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sHL, 64, ks), tc::desc_kmajor(sW2, 64, ks),
                                tc::idesc_f16(128, 16, false, false), ks > 0);
                tc::commit(&misc->mbar_mma);
            }
            mma_wait();
            float v[16];
            tc::tmem_ld16_sync(wk, v);
            r0 = v[0];
            sigma = density_act(r0, cfg.density_act);
#pragma unroll
            for (int k = 0; k < 3; ++k) c[k] = 1.0f / (1.0f + expf(-v[1 + k]));
        }
        }
        FP_MARK(m_t3);
        // ---- a5: volume rendering + loss + render backward
        const float dist = rr.dist;
        const float x = active ? sigma * delta : 0.f;
        const float alpha = expf(-x);
        const float o = -expm1f(-x);
        FP_MARK(m_r0);
        RScan R;
        m_render_scan(alpha, o, active, c, dist, active ? sigma : 0.f, N, xw, R);
        const float Ti = R.T, TN = R.TN, w = R.w;
        const float* sums = R.sums;
        FP_MARK(m_r2);
        FP_ACC(12, m_r0, m_r2);
        float dsig = 0.f, dcol[3] = {0.f, 0.f, 0.f};
        float gC[3] = {0.f, 0.f, 0.f};
        float gD = 0.f, gCb = 0.f;
        const int cls = rr.flags & RF_CLS_MASK;
        if (active) {
            const bool has_depth = (rr.flags & RF_HAS_DEPTH) != 0;
            float e[3], bgc[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                bgc[k] = (cls == CLS_OBJ && cfg.obj_bg == 1) ? 0.f : rr.bg[k];
                e[k] = sums[k] + TN * bgc[k] - (cls == CLS_OBJ ? rr.tgt[k] : rr.bg[k]);
            }
            const float ne = sqrtf(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
#pragma unroll
            for (int k = 0; k < 3; ++k) gC[k] = ne > 0.f ? e[k] / ne * invB : 0.f;
            float ed = 0.f;
            if (has_depth) {
                ed = sums[3] - rr.depth;
                gD = ed > 0.f ? cfg.lambda_depth * invB : (ed < 0.f ? -cfg.lambda_depth * invB : 0.f);
            }
            gCb = gC[0] * bgc[0] + gC[1] * bgc[1] + gC[2] * bgc[2];
            if (i == 0) {
#ifdef ROMAP_DET
                *reinterpret_cast<float4*>(det.ray_loss + 4 * (s >> lgN)) =
                    make_float4(cls == CLS_OBJ ? ne : 0.f, cls == CLS_OBJ ? 0.f : ne, has_depth ? fabsf(ed) : 0.f,
                                cls == CLS_BG ? sums[4] : 0.f);
#else
                atomicAdd(&misc->loss[cls == CLS_OBJ ? 0 : 1], ne);
                if (has_depth) atomicAdd(&misc->loss[2], fabsf(ed));
                if (cls == CLS_BG) atomicAdd(&misc->loss[3], sums[4]);
#endif
                if (!isfinite(ne) || !isfinite(sums[4])) atomicOr(nonfinite, 1);
            }
        }
#ifdef ROMAP_DET
        else if (i == 0) {
            *reinterpret_cast<float4*>(det.ray_loss + 4 * (s >> lgN)) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
#endif
        const float gc = gC[0] * c[0] + gC[1] * c[1] + gC[2] * c[2];
        // S = sum_{j>i} w_j gc_j = gC . suf(c), Sd = sum_{j>i} w_j dist_j (gC is per ray)
        const float S = gC[0] * R.suf[0] + gC[1] * R.suf[1] + gC[2] * R.suf[2], Sd = R.suf[3];
        FP_MARK(m_r3);
        FP_ACC(13, m_r2, m_r3);
        if (active) {
            const float Tn1 = Ti * alpha;
            dsig = delta * (Tn1 * gc - S - TN * gCb) + delta * gD * (Tn1 * dist - Sd) +
                   (cls == CLS_BG ? cfg.lambda_density * invB : 0.f);
#pragma unroll
            for (int k = 0; k < 3; ++k) dcol[k] = w * gC[k];
        }
        if (dbg) *reinterpret_cast<float4*>(dbg + 4 * s) = make_float4(dsig, dcol[0], dcol[1], dcol[2]);
        FP_MARK(m_t4);

        if constexpr (NET == 0) {
        // ---- a6: MLP backward (scaled by loss_scale)
        {
            float v[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = 0.f;
#pragma unroll
            for (int k = 0; k < 3; ++k) v[k] = dcol[k] * c[k] * (1.f - c[k]) * scale;
            tc::st16(DC, m, 0, 16, v);
        }
        const float dr0_extra = dsig * density_act_grad(r0, sigma, cfg.density_act) * scale;
        m_sync_for_mma();
        // B5: WK[128 x 64] = DC[128 x 16] . W5[16 x 64];  dW5^T[64 x 16] += G2^T . DC
        // (each stage commits after its dX product: the epilogue overlaps the dW
        // MMAs, which the next stage's commit covers; no epilogue overwrites an
        // operand of the dW MMAs still in flight)
        if (leader) {
            tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sDC, 16, 0), tc::desc_mnmajor(sW5, 64, 0),
                        tc::idesc_f16(128, 64, false, true), 0);
            tc::commit(&misc->mbar_mma);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
                tc::mma_f16(tm + TM_DW5, tc::desc_mnmajor(sG2, 64, ks), tc::desc_mnmajor(sDC, 16, ks),
                            tc::idesc_f16(64, 16, true, true), (dw_fresh && ks == 0) ? 0 : 1);
        }
        mma_wait();
        epi_mask64(wk, DB, G2, m);
        m_sync_for_mma();
        // B4: WK = DB(dg2) . W4;  dW4[64 x 64] += DB^T . G1
        if (leader) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sDB, 64, ks), tc::desc_mnmajor(sW4, 64, ks),
                            tc::idesc_f16(128, 64, false, true), ks > 0);
            tc::commit(&misc->mbar_mma);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
                tc::mma_f16(tm + TM_DW4, tc::desc_mnmajor(sDB, 64, ks), tc::desc_mnmajor(sG1, 64, ks),
                            tc::idesc_f16(64, 64, true, true), (dw_fresh && ks == 0) ? 0 : 1);
        }
        mma_wait();
        epi_mask64(wk, DB2, G1, m);
        m_sync_for_mma();
        // B3: WK[128 x 16] = DB2(dg1) . W3[:, 0:16];  dW3[64 x 32] += DB2^T . CIN
        if (leader) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sDB2, 64, ks), tc::desc_mnmajor(sW3, 32, ks),
                            tc::idesc_f16(128, 16, false, true), ks > 0);
            tc::commit(&misc->mbar_mma);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
                tc::mma_f16(tm + TM_DW3, tc::desc_mnmajor(sDB2, 64, ks), tc::desc_mnmajor(sCIN, 32, ks),
                            tc::idesc_f16(64, 32, true, true), (dw_fresh && ks == 0) ? 0 : 1);
        }
        mma_wait();
        {
            float v[16];
            tc::tmem_ld16_sync(wk, v);
            v[0] += dr0_extra;
            if (!active)
#pragma unroll
                for (int k = 0; k < 16; ++k) v[k] = 0.f;
            tc::st16(DR, m, 0, 16, v);
        }
        m_sync_for_mma();
        // B2: WK[128 x 64] = DR[128 x 16] . W2[16 x 64];  dW2^T[64 x 16] += H1^T . DR
        if (leader) {
            tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sDR, 16, 0), tc::desc_mnmajor(sW2, 64, 0),
                        tc::idesc_f16(128, 64, false, true), 0);
            tc::commit(&misc->mbar_mma);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
                tc::mma_f16(tm + TM_DW2, tc::desc_mnmajor(sH1, 64, ks), tc::desc_mnmajor(sDR, 16, ks),
                            tc::idesc_f16(64, 16, true, true), (dw_fresh && ks == 0) ? 0 : 1);
        }
        mma_wait();
        epi_mask64(wk, DB, H1, m);
        m_sync_for_mma();
        } else {
        // ---- a6: MLP backward, network 1: DC = [dsigma act'(raw_0), dc c (1 - c)] x loss scale
        {
            float v[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = 0.f;
            v[0] = dsig * density_act_grad(r0, sigma, cfg.density_act) * scale;
#pragma unroll
            for (int k = 0; k < 3; ++k) v[1 + k] = dcol[k] * c[k] * (1.f - c[k]) * scale;
            tc::st16(DC, m, 0, 16, v);
        }
        m_sync_for_mma();
        {
            // B_out: WK[128 x 64] = DC[128 x 16] . W_out[16 x 64];  dW_out^T[64 x 16] += h_hl^T . DC
            const uint32_t sHL = cfg.hl == 1 ? sH1 : (cfg.hl == 2 ? sG1 : sG2);
            if (leader) {
                tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sDC, 16, 0), tc::desc_mnmajor(sW2, 64, 0),
                            tc::idesc_f16(128, 64, false, true), 0);
                tc::commit(&misc->mbar_mma);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    tc::mma_f16(tm + TM_DW2, tc::desc_mnmajor(sHL, 64, ks), tc::desc_mnmajor(sDC, 16, ks),
                                tc::idesc_f16(64, 16, true, true), (dw_fresh && ks == 0) ? 0 : 1);
            }
            mma_wait();
            epi_mask64(wk, DB, cfg.hl == 1 ? H1 : (cfg.hl == 2 ? G1 : G2), m);
            m_sync_for_mma();
        }
        for (int k = cfg.hl - 1; k >= 1; --k) {
            // B_k: WK = D(dh_{k+1}) . W_k;  dW_k[64 x 64] += D^T . h_k  (D alternates DB / DB2)
            const uint32_t sW = k == 1 ? sW4 : sWH2, sHk = k == 1 ? sH1 : sG1;
            const int tdw = k == 1 ? TM_DW4 : TM_DWH2;
            const bool odd = ((cfg.hl - 1 - k) & 1) != 0;
            const uint32_t sD = odd ? sDB2 : sDB;
            if (leader) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    tc::mma_f16(tm + TM_WK, tc::desc_kmajor(sD, 64, ks), tc::desc_mnmajor(sW, 64, ks),
                                tc::idesc_f16(128, 64, false, true), ks > 0);
                tc::commit(&misc->mbar_mma);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    tc::mma_f16(tm + tdw, tc::desc_mnmajor(sD, 64, ks), tc::desc_mnmajor(sHk, 64, ks),
                                tc::idesc_f16(64, 64, true, true), (dw_fresh && ks == 0) ? 0 : 1);
            }
            mma_wait();
            epi_mask64(wk, odd ? DB : DB2, k == 1 ? H1 : G1, m);
            m_sync_for_mma();
        }
        }
        // dh1 for B1: DB (network 0; network 1 after an even number of hidden-layer steps) or DB2
        const uint32_t sD1 = (NET == 0 || ((cfg.hl - 1) & 1) == 0) ? sDB : sDB2;
        // B1: DF[b][128 x LF] = D(dh1) . W1[64 x LF];  dW1[64 x LF] += D^T . X0[b]
        // (DF[b] must have been read by G: scatter of tile j - NB)
        if (leader) {
            if (j >= NB) tc::mbar_wait(&misc->df_empty[b], ((j - NB) / NB) & 1);
            tc::fence_after();
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                tc::mma_f16(tm + TM_DF + 32 * b, tc::desc_kmajor(sD1, 64, ks), tc::desc_mnmajor(sW1, LF, ks),
                            tc::idesc_f16(128, LF, false, true), ks > 0);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
                tc::mma_f16(tm + TM_DW1, tc::desc_mnmajor(sD1, 64, ks), tc::desc_mnmajor(sX0, LF, ks),
                            tc::idesc_f16(64, LF, true, true), (dw_fresh && ks == 0) ? 0 : 1);
            tc::commit(&misc->tile_done[b]);
        }
#ifdef ROMAP_DET
        // this tile's dW alone (every tile starts its accumulators fresh) into its
        // per-tile partial; k_det.cu sums an object's tiles in tile order
        tc::mbar_wait(&misc->tile_done[b], (j / NB) & 1);
        tc::fence_after();
        m_flush<LF, true>(cfg, det.dw + tile * (long long)cfg.n_mlp, tm, misc, loss_acc, cur, true);
        dw_fresh = true;
#else
        dw_fresh = false;
#endif
        FP_MARK(m_t5);
        FP_ACC(6, m_t0, m_t1);
        FP_ACC(1, m_t1, m_t2);
        FP_ACC(2, m_t2, m_t3);
        FP_ACC(3, m_t3, m_t4);
        FP_ACC(4, m_t4, m_t5);
    }
    FP_MARK(m_fl0);
    if (cur >= 0) {
        tc::mbar_wait(&misc->tile_done[(n - 1) % NB], ((n - 1) / NB) & 1);
        tc::fence_after();
        m_flush<LF>(cfg, objs[cur].g32 + cfg.n_table, tm, misc, loss_acc, cur, !dw_fresh);
    }
    FP_MARK(m_end);
    FP_ACC(0, m_start, m_end);
    FP_ACC(15, m_fl0, m_end);
}

}  // namespace

template <int L, int NET>
__global__ void __launch_bounds__(NT, 1) k_fused_mixed(CfgDev cfg, const ObjDev* __restrict__ objs,
                                                       const RayRec* __restrict__ rays,
                                                       const float4* __restrict__ srec,
                                                       const float* __restrict__ sdelta, int n_tiles,
                                                       int tiles_per_cta, double* __restrict__ loss_acc,
                                                       int* __restrict__ nonfinite, float* __restrict__ dbg DET_PARAM) {
    extern __shared__ __align__(1024) uint8_t smem[];
    Misc* misc = reinterpret_cast<Misc*>(smem + OFF_MISC);
    const int t = threadIdx.x, warp = t >> 5;
#ifdef ROMAP_FUSED_PROF
    const bool fp_on = t == 0;
#endif
    FP_MARK(cta_start);
#ifdef ROMAP_FUSED_PROF
    if (t == 0 && blockIdx.x < 1024) g_cta_ns[2 * blockIdx.x] = gtimer();
#endif
    if (warp == 0) tc::tmem_alloc(&misc->tmem, TM_COLS);
    if (t == 32) {
        tc::mbar_init(&misc->mbar_mma, 1);
        for (int b = 0; b < NB; ++b) {
            tc::mbar_init(&misc->x0_full[b], NG / 32);
            tc::mbar_init(&misc->tile_done[b], 1);
            tc::mbar_init(&misc->df_empty[b], NG / 32);
        }
        tc::fence_mbar_init();
    }
    if (t < 4) misc->loss[t] = 0.f;
#ifdef ROMAP_EXP_NOMSTS
    for (int o = OFF_H1 + 16 * t; o < OFF_MISC; o += 16 * NT) *reinterpret_cast<uint4*>(smem + o) = make_uint4(0, 0, 0, 0);
#endif
    if (t < L) {
        misc->lv[t] = level_params(cfg, t);
        misc->lvoff[t] = cfg.off[t];
    }
    // PDL: let Adam launch now (its CTAs take SMs as ours leave) and wait for the
    // previous grid (Adam: tables, weights, zeroed gradients) before any access
    pdl_trigger();
    pdl_wait();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    FP_MARK(cta_setup);
    FP_ACC(5, cta_start, cta_setup);
    const uint32_t tm = misc->tmem;
    const int tile0 = blockIdx.x, tstride = gridDim.x;
    const int n = tile0 < n_tiles ? (n_tiles - 1 - tile0) / tstride + 1 : 0;
    if (n > 0) {
        if (warp < NG / 32)
            g_loop<L>(cfg, objs, rays, srec, tile0, tstride, n, smem, misc, tm DET_ARG);
        else
            m_loop<L, NET>(cfg, objs, rays, srec, sdelta, tile0, tstride, n, smem, misc, tm, loss_acc, nonfinite, dbg
                           DET_ARG);
    }
    tc::fence_before();
    __syncthreads();
    FP_MARK(cta_end);
    FP_ACC(7, cta_start, cta_end);
#ifdef ROMAP_FUSED_PROF
    if (t == 0 && blockIdx.x < 1024) g_cta_ns[2 * blockIdx.x + 1] = gtimer();
#endif
    if (warp == 0) tc::tmem_dealloc(tm, TM_COLS);
}

void FUSED_LAUNCH(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, const RayRec* rays,
                  const float4* srec, const float* sdelta, int n_rays, double* loss_acc, int* nonfinite,
                  float* dbg DET_PARAM) {
    const long long S = (long long)n_rays * cfg.N;
    const int n_tiles = (int)(S / TILE);
    if (n_tiles == 0) return;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_fused_mixed<8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        cudaFuncSetAttribute(k_fused_mixed<16, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        cudaFuncSetAttribute(k_fused_mixed<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        cudaFuncSetAttribute(k_fused_mixed<16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        attr = true;
    }
    int grid = lc.num_sms;
    if (grid > n_tiles) grid = n_tiles;
    const int per = 0;   // unused: tiles are strided over the grid
    auto kern = cfg.net == 1 ? (cfg.L == 16 ? k_fused_mixed<16, 1> : k_fused_mixed<8, 1>)
                             : (cfg.L == 16 ? k_fused_mixed<16, 0> : k_fused_mixed<8, 0>);
    cudaLaunchConfig_t lcfg = {};
    lcfg.gridDim = dim3(grid);
    lcfg.blockDim = dim3(NT);
    lcfg.dynamicSmemBytes = SMEM_BYTES;
    lcfg.stream = lc.st;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    lcfg.attrs = la;
    lcfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&lcfg, kern, cfg, objs, rays, srec, sdelta, n_tiles, per, loss_acc, nonfinite, dbg DET_ARG);
}

// hash_fp16.cuh -- multiresolution hash-grid helpers of the mixed path (fp16
// tables, one 4-byte half2 word per entry), shared by the fused training kernel
// and the mixed inference kernels.  Grid definition: DESIGN.md R5.
#pragma once
#include "romap_internal.cuh"

// cell and the 8 corner entries of one level (R5), as absolute entry indices
// (level offset `off` added): P = {res, y multiplier, z multiplier, dense};
// dense: x + (N+1) y + (N+1)^2 z; hashed: (x * 1 ^ y * 2654435761 ^
// z * 805459861) & (T - 1).  Corner b: bit k -> +1 on axis k.
__device__ __forceinline__ void level_entries(const float u[3], const int4 P, unsigned off, unsigned hmask, Cell& cl,
                                              unsigned (&e)[8]) {
    cl = grid_cell(u, P.x);
    const unsigned my = (unsigned)P.y, mz = (unsigned)P.z;
    const unsigned x0 = (unsigned)cl.c[0], x1 = x0 + 1u;
    const unsigned ty0 = (unsigned)cl.c[1] * my, ty1 = ty0 + my;
    const unsigned tz0 = (unsigned)cl.c[2] * mz, tz1 = tz0 + mz;
    if (P.w) {
        const unsigned yz[4] = {ty0 + tz0 + off, ty1 + tz0 + off, ty0 + tz1 + off, ty1 + tz1 + off};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            e[2 * k] = x0 + yz[k];
            e[2 * k + 1] = x1 + yz[k];
        }
    } else {
        const unsigned yz[4] = {ty0 ^ tz0, ty1 ^ tz0, ty0 ^ tz1, ty1 ^ tz1};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            e[2 * k] = ((x0 ^ yz[k]) & hmask) + off;
            e[2 * k + 1] = ((x1 ^ yz[k]) & hmask) + off;
        }
    }
}

// level parameters as the kernels keep them in shared memory:
// {res, y multiplier, z multiplier, dense} (R5) and the entry offset
__device__ __forceinline__ int4 level_params(const CfgDev& cfg, int l) {
    const int res = cfg.res[l];
    const bool dense = cfg.dense[l] != 0;
    const unsigned n1 = (unsigned)res + 1u;
    return make_int4(res, (int)(dense ? n1 : 2654435761u), (int)(dense ? n1 * n1 : 805459861u), dense ? 1 : 0);
}

// encode two levels (P0/P1 at offsets off0/off1) of one point into two half2
// features: x-neighbour corner pairs as one LDG.128 (+ a 4-byte load when the
// pair straddles a 16-byte chunk), trilinear lerps (x, y, z) in fp32 of the fp16
// corners, rounded once to fp16; zeros when !on
__device__ __forceinline__ void encode_pair_fp16(const uint32_t* __restrict__ tab, const float u[3], const int4 P[2],
                                                 const unsigned off[2], unsigned hmask, bool on, __half2 (&fq)[2]) {
    uint4 qv[2][4];
    uint32_t xv[2][4];
    unsigned e[2][8];
    Cell cl[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        level_entries(u, P[q], 0u, hmask, cl[q], e[q]);    // level-relative; block at tab + off (R5)
        const uint32_t* tl = opaque_ptr(tab + off[q]);
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const bool same = (e[q][2 * p] >> 2) == (e[q][2 * p + 1] >> 2);
            qv[q][p] = on ? ldg_v4(tl + opaque_u32(e[q][2 * p] & ~3u)) : make_uint4(0, 0, 0, 0);
            xv[q][p] = (on && !same) ? ldg_u32(tl + e[q][2 * p + 1]) : 0u;
        }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        float2 vx[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const unsigned ea = e[q][2 * p], eb = e[q][2 * p + 1];
            const bool same = (ea >> 2) == (eb >> 2);
            const uint32_t h0 = sel4(qv[q][p], ea & 3);
            const uint32_t h1 = same ? sel4(qv[q][p], eb & 3) : xv[q][p];
            const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&h0));
            const float2 c = __half22float2(*reinterpret_cast<const __half2*>(&h1));
            vx[p] = make_float2(a.x + cl[q].f[0] * (c.x - a.x), a.y + cl[q].f[0] * (c.y - a.y));
        }
        const float fy = cl[q].f[1], fz = cl[q].f[2];
        const float2 y0 = make_float2(vx[0].x + fy * (vx[1].x - vx[0].x), vx[0].y + fy * (vx[1].y - vx[0].y));
        const float2 y1 = make_float2(vx[2].x + fy * (vx[3].x - vx[2].x), vx[2].y + fy * (vx[3].y - vx[2].y));
        fq[q] = __floats2half2_rn(y0.x + fz * (y1.x - y0.x), y0.y + fz * (y1.y - y0.y));
    }
}

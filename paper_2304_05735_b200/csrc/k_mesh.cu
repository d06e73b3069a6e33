// k_mesh.cu -- SURVEY.md 8(f) f2: isosurface extraction of one object's density
// (the input the paper feeds to marching cubes) as marching
// tetrahedra (R26): (res+1)^3 vertex lattice over [-a, a] (R21), sigma
// by the object's query kernel, per cell the 6 Kuhn tetrahedra; per tetrahedron
// with 1/3 vertices above iso one triangle on its crossing edges, with 2 a quad
// (2 triangles).  Two passes: count per cell, exclusive scan (CUB), emit at the
// scanned offset -- the output order is the oracle's (cells x-major, tetrahedra
// in Kuhn order), so the mesh is deterministic.  Triangles in the world frame.
#include <cub/device/device_scan.cuh>

#include "romap_internal.cuh"

namespace {

// Kuhn tetrahedra: (0, 1 << p0, (1 << p0) | (1 << p1), 7), p in (01, 02, 10, 12, 20, 21)
__constant__ int c_kuhn[6][4] = {{0, 1, 3, 7}, {0, 1, 5, 7}, {0, 2, 3, 7}, {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 4, 6, 7}};

struct CellVals {
    float s[8];
    float p[8][3];
};

__device__ __forceinline__ void load_cell(const float* __restrict__ sig, const float* __restrict__ pts, int R,
                                          long long cell, CellVals& cv) {
    const int iz = (int)(cell % R), iy = (int)((cell / R) % R), ix = (int)(cell / ((long long)R * R));
    const long long n1 = R + 1;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const long long v = ((long long)(ix + (k & 1)) * n1 + (iy + ((k >> 1) & 1))) * n1 + (iz + ((k >> 2) & 1));
        cv.s[k] = sig[v];
#pragma unroll
        for (int c = 0; c < 3; ++c) cv.p[k][c] = pts[3 * v + c];
    }
}

__device__ __forceinline__ int tet_tris(const float s[4], float iso) {
    int n = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) n += s[i] > iso;
    return (n == 1 || n == 3) ? 1 : (n == 2 ? 2 : 0);
}

__global__ void k_lattice(const ObjDev* __restrict__ obj, int R, float* __restrict__ pts) {
    const long long n1 = R + 1, n = n1 * n1 * n1;
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const long long ix = v / (n1 * n1), iy = (v / n1) % n1, iz = v % n1;
    const long long id[3] = {ix, iy, iz};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double a = obj->a[c];
        pts[3 * v + c] = (float)(-a + 2.0 * a * (double)id[c] / (double)R);
    }
}

__global__ void k_mt_count(const float* __restrict__ sig, const float* __restrict__ pts, int R, float iso,
                           int* __restrict__ counts) {
    const long long nc = (long long)R * R * R;
    const long long cell = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (cell >= nc) return;
    CellVals cv;
    load_cell(sig, pts, R, cell, cv);
    int n = 0;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
        const float s[4] = {cv.s[c_kuhn[t][0]], cv.s[c_kuhn[t][1]], cv.s[c_kuhn[t][2]], cv.s[c_kuhn[t][3]]};
        n += tet_tris(s, iso);
    }
    counts[cell] = n;
}

__device__ __forceinline__ void edge_point(const float pa[3], const float pb[3], float sa, float sb, float iso,
                                           float out[3]) {
    const float w = (iso - sa) / (sb - sa);
#pragma unroll
    for (int c = 0; c < 3; ++c) out[c] = pa[c] + w * (pb[c] - pa[c]);
}

__device__ __forceinline__ void store_tri(float* __restrict__ out, long long k, const float q0[3], const float q1[3],
                                          const float q2[3], const ObjDev& ob) {
    const float* q[3] = {q0, q1, q2};
#pragma unroll
    for (int v = 0; v < 3; ++v) {
        // object -> world: x_w = R_z(yaw) x + t (R8)
        out[9 * k + 3 * v + 0] = ob.c * q[v][0] - ob.s * q[v][1] + ob.t[0];
        out[9 * k + 3 * v + 1] = ob.s * q[v][0] + ob.c * q[v][1] + ob.t[1];
        out[9 * k + 3 * v + 2] = q[v][2] + ob.t[2];
    }
}

__global__ void k_mt_emit(const ObjDev* __restrict__ obj, const float* __restrict__ sig, const float* __restrict__ pts,
                          int R, float iso, const int* __restrict__ offsets, float* __restrict__ tris) {
    const long long nc = (long long)R * R * R;
    const long long cell = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (cell >= nc) return;
    const ObjDev ob = *obj;
    CellVals cv;
    load_cell(sig, pts, R, cell, cv);
    long long k = offsets[cell];
    for (int t = 0; t < 6; ++t) {
        float s[4], p[4][3];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int v = c_kuhn[t][i];
            s[i] = cv.s[v];
#pragma unroll
            for (int c = 0; c < 3; ++c) p[i][c] = cv.p[v][c];
        }
        int ins[4], out[4], ni = 0, no = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (s[i] > iso) ins[ni++] = i; else out[no++] = i;
        }
        if (ni == 1 || ni == 3) {
            const int a = ni == 1 ? ins[0] : out[0];
            float q[3][3];
            int j = 0;
            for (int o = 0; o < 4; ++o)
                if (o != a) edge_point(p[a], p[o], s[a], s[o], iso, q[j++]);
            store_tri(tris, k++, q[0], q[1], q[2], ob);
        } else if (ni == 2) {
            const int a = ins[0], b = ins[1], c = out[0], d = out[1];
            float q0[3], q1[3], q2[3], q3[3];
            edge_point(p[a], p[c], s[a], s[c], iso, q0);
            edge_point(p[a], p[d], s[a], s[d], iso, q1);
            edge_point(p[b], p[d], s[b], s[d], iso, q2);
            edge_point(p[b], p[c], s[b], s[c], iso, q3);
            store_tri(tris, k++, q0, q1, q2, ob);
            store_tri(tris, k++, q0, q2, q3, ob);
        }
    }
}

// R26 visibility carve: sigma := 0 at lattice vertices that no keyframe sees
// inside its detection box (fp32, one rounding per operation, oracle order)
__global__ void k_carve(const ObjDev* __restrict__ obj, const float* __restrict__ pts, long long nv,
                        float* __restrict__ sig) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    const ObjDev& ob = *obj;
    const float x = pts[3 * v], y = pts[3 * v + 1], z = pts[3 * v + 2];
    const float xw[3] = {__fadd_rn(__fsub_rn(__fmul_rn(ob.c, x), __fmul_rn(ob.s, y)), ob.t[0]),
                         __fadd_rn(__fadd_rn(__fmul_rn(ob.s, x), __fmul_rn(ob.c, y)), ob.t[1]),
                         __fadd_rn(z, ob.t[2])};
    bool seen = false;
    for (int k = 0; k < ob.n_kf && !seen; ++k) {
        const KfDev& kf = ob.kfs[k];
        const float d[3] = {__fsub_rn(xw[0], kf.T[3]), __fsub_rn(xw[1], kf.T[7]), __fsub_rn(xw[2], kf.T[11])};
        float xc[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
            xc[c] = __fadd_rn(__fadd_rn(__fmul_rn(kf.T[c], d[0]), __fmul_rn(kf.T[4 + c], d[1])), __fmul_rn(kf.T[8 + c], d[2]));
        const float u = __fadd_rn(__fmul_rn(kf.fx, __fdiv_rn(xc[0], xc[2])), kf.cx);
        const float w = __fadd_rn(__fmul_rn(kf.fy, __fdiv_rn(xc[1], xc[2])), kf.cy);
        seen = xc[2] > 0.f && u >= (float)kf.x0 && u < (float)(kf.x0 + kf.w) && w >= (float)kf.y0 &&
               w < (float)(kf.y0 + kf.h);
    }
    if (!seen) sig[v] = 0.f;
}

}  // namespace

void launch_carve(const LaunchCtx& lc, const ObjDev* obj, const float* pts, long long nv, float* sig) {
    k_carve<<<(unsigned)((nv + 255) / 256), 256, 0, lc.st>>>(obj, pts, nv, sig);
}

void launch_lattice(const LaunchCtx& lc, const ObjDev* obj, int R, float* pts) {
    const long long n1 = R + 1, n = n1 * n1 * n1;
    k_lattice<<<(unsigned)((n + 255) / 256), 256, 0, lc.st>>>(obj, R, pts);
}

// counts (R^3 ints) -> offsets (R^3 ints, exclusive) + total (device int at
// offsets[R^3]); tmp: CUB scratch (size queried when tmp == nullptr)
size_t mt_scan_bytes(long long ncell) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int*)nullptr, (int*)nullptr, (int)(ncell + 1));
    return bytes;
}

void launch_mt(const LaunchCtx& lc, const ObjDev* obj, const float* sig, const float* pts, int R, float iso,
               int* counts, int* offsets, void* tmp, size_t tmp_bytes, float* tris, bool emit) {
    const long long nc = (long long)R * R * R;
    const unsigned blocks = (unsigned)((nc + 255) / 256);
    if (!emit) {
        k_mt_count<<<blocks, 256, 0, lc.st>>>(sig, pts, R, iso, counts);
        cudaMemsetAsync(counts + nc, 0, sizeof(int), lc.st);
        cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, offsets, (int)(nc + 1), lc.st);
    } else {
        k_mt_emit<<<blocks, 256, 0, lc.st>>>(obj, sig, pts, R, iso, offsets, tris);
    }
}

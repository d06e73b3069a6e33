// romap_internal.cuh -- device data layout and the per-sample building blocks
// shared by every libromap kernel (sm_100a).  Nothing here is shared with the
// CPU oracle (oracle/), which is written independently from the paper.
//
// Bit-exactness discipline (BASELINE north_star: hash indices, sample positions
// and ray/box segments bit-exact): every operation on that path is an explicit
// round-to-nearest intrinsic (__fmul_rn/__fadd_rn/__fsub_rn/__fdiv_rn/
// __fsqrt_rn), which nvcc never contracts into FMA.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define ROMAP_MAX_LEVELS 16
#define ROMAP_WIDTH 64        // hidden width
#define ROMAP_DOUT 16         // density-net outputs
#define ROMAP_SH 16           // SH degree-4 coefficients
#define ROMAP_CIN 32          // colour-net input = [raw16 || sh16]
#define ROMAP_MAX_LF 32
#define ROMAP_TILE 128        // samples per tile / block

// ---------------------------------------------------------------------------
// configuration shared by all objects of one launch (passed by value)
struct CfgDev {
    int L, F, LF, log2T, T;
    int res[ROMAP_MAX_LEVELS];
    int dense[ROMAP_MAX_LEVELS];
    int off[ROMAP_MAX_LEVELS];    // entry offset of level l
    int n_entries;                // sum E_l
    int n_table;                  // n_entries * F
    int n_mlp;                    // MLP parameter count
    int w_off[5];                 // layer offsets inside the MLP block (W1..W5; network 1: W1, W_h.., W_out)
    int net;                      // 0 BASELINE nets, 1 the paper's MLP (R24)
    int hl;                       // network 1: hidden layers
    int n_layers;
    int N;                        // samples per ray
    int density_act, obj_bg;
    float lambda_depth, lambda_density;
    float lr, b1, b2, eps;
    float loss_scale;
    unsigned long long seed;
};

struct KfDev {
    float T[12];                  // camera->world 3x4 row-major
    float fx, fy, cx, cy;
    int x0, y0, w, h;             // detection box (in-box crop)
    const uchar4* crop;           // (r, g, b, class) per in-box pixel, row-major
    const float* depth;           // camera z per in-box pixel (0 = none) or nullptr
};

struct ObjDev {
    float a[3], t[3];             // half extents, centre
    float c, s;                   // cos / sin of yaw (double on host, rounded)
    float* p32;                   // [table n_table | mlp n_mlp]
    float* g32;                   // gradients, same layout
    float* m;                     // Adam first moment
    float* v;                     // Adam second moment
    __half* p16;                  // fp16 working copy (mixed path)
    const KfDev* kfs;
    const long long* area_prefix; // exclusive prefix of box areas
    int n_kf;
    long long total_area;
    int ray_begin;                // first global ray slot
    int n_rays;                   // rays drawn (B of R16)
    int n_slots;                  // rays + padding (multiple of TILE/N)
    int obj_id;                   // global object id (RNG key, R13)
    long long* step;              // device Adam step counter
};

// ray record (one per global ray slot)
struct RayRec {
    float o[3], d[3];
    float tn, tf;
    float tgt[3], bg[3];
    float depth;
    int flags;                    // bits 0-1 class, 2 active (hit & supervised), 3 has_depth, 4 drawn
    int slot;                     // object slot in the launch
    int kf, px, py;
};

#define RF_CLS_MASK 3
#define RF_ACTIVE 4
#define RF_HAS_DEPTH 8
#define RF_DRAWN 16
#define CLS_BG 0
#define CLS_OBJ 1
#define CLS_OCC 2

// ---------------------------------------------------------------------------
// counter-based RNG (R13): SplitMix64 finalizer chain
#define ROMAP_GOLDEN 0x9E3779B97F4A7C15ULL
__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}
// prefix key of (seed, obj, t); the per-ray / per-stream part is mixed in below
__device__ __forceinline__ unsigned long long rng_prefix(unsigned long long seed, int obj, long long t) {
    unsigned long long k = mix64(seed + ROMAP_GOLDEN);
    k = mix64(k ^ (unsigned long long)(long long)obj);
    return mix64(k ^ (unsigned long long)t);
}
__device__ __forceinline__ unsigned rng_u32(unsigned long long prefix, int ray, int stream) {
    return (unsigned)(mix64(prefix ^ (((unsigned long long)ray << 8) | (unsigned long long)stream)) >> 32);
}
__device__ __forceinline__ float u32_unit(unsigned u) {
    return __fmul_rn(__uint2float_rn(u >> 8), 5.9604644775390625e-08f);   // 2^-24
}

// ---------------------------------------------------------------------------
// geometry (fp32, one rounding per op; mirrors DESIGN.md R8/R11/R12)
struct Ray { float o[3], d[3], n; };

__device__ __forceinline__ Ray make_ray(const KfDev& kf, int px, int py, const ObjDev& ob) {
    float pxf = __fadd_rn((float)px, 0.5f);
    float pyf = __fadd_rn((float)py, 0.5f);
    float dcx = __fdiv_rn(__fsub_rn(pxf, kf.cx), kf.fx);
    float dcy = __fdiv_rn(__fsub_rn(pyf, kf.cy), kf.fy);
    float n = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(dcx, dcx), __fmul_rn(dcy, dcy)), 1.0f));
    float nx = __fdiv_rn(dcx, n), ny = __fdiv_rn(dcy, n), nz = __fdiv_rn(1.0f, n);
    float dw[3], p[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        dw[k] = __fadd_rn(__fadd_rn(__fmul_rn(kf.T[4 * k + 0], nx), __fmul_rn(kf.T[4 * k + 1], ny)),
                          __fmul_rn(kf.T[4 * k + 2], nz));
        p[k] = __fsub_rn(kf.T[4 * k + 3], ob.t[k]);
    }
    Ray r;
    r.o[0] = __fadd_rn(__fmul_rn(ob.c, p[0]), __fmul_rn(ob.s, p[1]));
    r.o[1] = __fsub_rn(__fmul_rn(ob.c, p[1]), __fmul_rn(ob.s, p[0]));
    r.o[2] = p[2];
    r.d[0] = __fadd_rn(__fmul_rn(ob.c, dw[0]), __fmul_rn(ob.s, dw[1]));
    r.d[1] = __fsub_rn(__fmul_rn(ob.c, dw[1]), __fmul_rn(ob.s, dw[0]));
    r.d[2] = dw[2];
    r.n = n;
    return r;
}

// slab test against [-a, a] (R11); returns hit
__device__ __forceinline__ bool ray_box(const float o[3], const float d[3], const float a[3], float& tn, float& tf) {
    tn = 0.0f;
    tf = __int_as_float(0x7f800000);
    bool miss = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (d[k] == 0.0f) {
            miss |= fabsf(o[k]) > a[k];
        } else {
            float inv = __fdiv_rn(1.0f, d[k]);
            float t0 = __fmul_rn(__fsub_rn(-a[k], o[k]), inv);
            float t1 = __fmul_rn(__fsub_rn(a[k], o[k]), inv);
            tn = fmaxf(tn, fminf(t0, t1));
            tf = fminf(tf, fmaxf(t0, t1));
        }
    }
    return !miss && (tf > tn);
}

// stratified distance of sample i (R12): tn + (i + xi) * ((tf - tn)/N)
__device__ __forceinline__ float sample_dist(float tn, float Dl, int i, float xi) {
    return __fadd_rn(tn, __fmul_rn(__fadd_rn((float)i, xi), Dl));
}

// normalized position u = clamp((x + a)/(a + a), 0, 1), x = o + dist * d (R6)
__device__ __forceinline__ void sample_u(const float o[3], const float d[3], const float a[3], float dist, float u[3]) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float x = __fadd_rn(o[k], __fmul_rn(dist, d[k]));
        float v = __fdiv_rn(__fadd_rn(x, a[k]), __fadd_rn(a[k], a[k]));
        u[k] = fminf(fmaxf(v, 0.0f), 1.0f);
    }
}

// ---------------------------------------------------------------------------
// hash-grid cell of level l (R5): base corner c, fractions f
struct Cell { int c[3]; float f[3]; };

__device__ __forceinline__ Cell grid_cell(const float u[3], int res) {
    Cell cl;
    float rf = (float)res;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float pos = __fmul_rn(u[k], rf);
        int c = (int)floorf(pos);
        c = min(max(c, 0), res - 1);
        cl.c[k] = c;
        cl.f[k] = __fsub_rn(pos, (float)c);
    }
    return cl;
}

// table entry (relative to the level) of corner b of the cell
__device__ __forceinline__ int corner_entry(const Cell& cl, int b, int res, int dense, int T) {
    unsigned x = (unsigned)(cl.c[0] + (b & 1));
    unsigned y = (unsigned)(cl.c[1] + ((b >> 1) & 1));
    unsigned z = (unsigned)(cl.c[2] + ((b >> 2) & 1));
    if (dense) {
        unsigned n1 = (unsigned)res + 1u;
        return (int)(x + n1 * (y + n1 * z));
    }
    unsigned h = (x * 1u) ^ (y * 2654435761u) ^ (z * 805459861u);
    return (int)(h & (unsigned)(T - 1));
}

__device__ __forceinline__ float corner_weight(const Cell& cl, int b) {
    float wx = (b & 1) ? cl.f[0] : __fsub_rn(1.0f, cl.f[0]);
    float wy = (b & 2) ? cl.f[1] : __fsub_rn(1.0f, cl.f[1]);
    float wz = (b & 4) ? cl.f[2] : __fsub_rn(1.0f, cl.f[2]);
    return __fmul_rn(__fmul_rn(wx, wy), wz);
}

// fire-and-forget vector atomic add (REDG.E.ADD.F32x2; no return value, so no
// long-scoreboard wait on the L2 round trip)
// (no "memory" clobber: nothing in the kernel reads these addresses back, and a
// clobber would force every cached global field to be re-loaded after each RED)
__device__ __forceinline__ void red_add_f2(float2* p, float a, float b) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" :: "l"(p), "f"(a), "f"(b));
}
__device__ __forceinline__ void red_add_f1(float* p, float a) {
    asm volatile("red.global.add.f32 [%0], %1;" :: "l"(p), "f"(a));
}

__device__ __forceinline__ void red_add_f4(float4* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d));
}
// predicated forms (one @p REDG each, no branch: the hash-grid scatter issues
// them for every lane and lets the predicate drop the ones it does not need)
__device__ __forceinline__ void red_add_f4_if(bool on, float4* p, float a, float b, float c, float d) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q red.global.add.v4.f32 [%1], {%2, %3, %4, %5};\n}"
                 :: "r"((int)on), "l"(p), "f"(a), "f"(b), "f"(c), "f"(d));
}
__device__ __forceinline__ void red_add_f2_if(bool on, float2* p, float a, float b) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q red.global.add.v2.f32 [%1], {%2, %3};\n}"
                 :: "r"((int)on), "l"(p), "f"(a), "f"(b));
}
// the same pointer, opaque to the compiler: addresses p + e then compile to one
// IMAD.WIDE.U32 each instead of re-associated 64-bit (base + off + e) * 4 chains
template <typename T>
__device__ __forceinline__ T* opaque_ptr(T* p) {
    unsigned long long v = reinterpret_cast<unsigned long long>(p);
    asm("mov.b64 %0, %0;" : "+l"(v));
    return reinterpret_cast<T*>(v);
}
__device__ __forceinline__ unsigned opaque_u32(unsigned v) {
    asm("mov.b32 %0, %0;" : "+r"(v));
    return v;
}
// programmatic dependent launch (the fused step and Adam are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): a kernel lets the next one
// launch early (its CTAs take SMs as ours leave, no launch gap) and waits for the
// previous grid's completion and memory before touching its outputs
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// host: whether launches use it (ROMAP_NO_PDL=1 turns it off)
bool pdl_enabled();
// a when p else b, as one SEL the compiler cannot turn into a branch
__device__ __forceinline__ uint32_t selp_u32(bool p, uint32_t a, uint32_t b) {
    uint32_t r;
    asm("{\n .reg .pred q;\n setp.ne.b32 q, %1, 0;\n selp.b32 %0, %2, %3, q;\n}" : "=r"(r) : "r"((int)p), "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint4 ldg_v4(const void* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ uint32_t ldg_u32(const void* p) { return __ldg(reinterpret_cast<const unsigned*>(p)); }
__device__ __forceinline__ uint32_t sel4(const uint4& q, int k) {
    return (k & 2) ? ((k & 1) ? q.w : q.z) : ((k & 1) ? q.y : q.x);
}

// ---------------------------------------------------------------------------
// real SH, bands 0..3 (R2), fp32
__device__ __forceinline__ void sh4(const float d[3], float out[16]) {
    float x = d[0], y = d[1], z = d[2];
    float xx = x * x, yy = y * y, zz = z * z;
    out[0] = 0.28209479177387814f;
    out[1] = -0.48860251190291987f * y;
    out[2] = 0.48860251190291987f * z;
    out[3] = -0.48860251190291987f * x;
    out[4] = 1.0925484305920792f * x * y;
    out[5] = -1.0925484305920792f * y * z;
    out[6] = 0.94617469575755997f * zz - 0.31539156525251999f;
    out[7] = -1.0925484305920792f * x * z;
    out[8] = 0.54627421529603959f * (xx - yy);
    out[9] = 0.59004358992664352f * y * (-3.0f * xx + yy);
    out[10] = 2.8906114426405538f * x * y * z;
    out[11] = 0.45704579946446572f * y * (1.0f - 5.0f * zz);
    out[12] = 0.3731763325901154f * z * (5.0f * zz - 3.0f);
    out[13] = 0.45704579946446572f * x * (1.0f - 5.0f * zz);
    out[14] = 1.4453057213202769f * z * (xx - yy);
    out[15] = 0.59004358992664352f * x * (-xx + 3.0f * yy);
}

__device__ __forceinline__ float density_act(float r0, int act) {
    if (act == 0) return expf(fminf(r0, 15.0f));                 // R3
    return r0 > 15.0f ? r0 : log1pf(expf(r0));                    // softplus
}
__device__ __forceinline__ float density_act_grad(float r0, float sigma, int act) {
    if (act == 0) return sigma;                                   // straight-through (R3)
    return 1.0f / (1.0f + expf(-r0));
}

// ---------------------------------------------------------------------------
// sample geometry of (ray record, i): dist, delta, u
__device__ __forceinline__ void sample_geometry(const RayRec& rr, int i, int N, unsigned long long pre, int ray_local,
                                                const float a[3], float& dist, float& delta, float u[3]) {
    float Dl = __fdiv_rn(__fsub_rn(rr.tf, rr.tn), (float)N);
    float xi = u32_unit(rng_u32(pre, ray_local, 16 + i));
    dist = sample_dist(rr.tn, Dl, i, xi);
    if (i + 1 < N) {
        float xn = u32_unit(rng_u32(pre, ray_local, 17 + i));
        delta = __fsub_rn(sample_dist(rr.tn, Dl, i + 1, xn), dist);
    } else {
        delta = Dl;
    }
    sample_u(rr.o, rr.d, a, dist, u);
}

// ---------------------------------------------------------------------------
// deterministic-reduction mode (romap_set_deterministic; tests only): instead of
// fp32 atomics, the training kernels write every gradient / loss contribution
// to a record, and k_det.cu reduces the records in a fixed order (sample order
// within an object), so the result does not depend on scheduling, on the other
// objects of the batch or on graph vs plain launches.
//   key/val: one record per (sample s, level l, corner b) of the launch, index
//            (s * L + l) * 8 + b; key = (object slot << 32) | table entry, or
//            DET_NO_KEY for a sample of an inactive ray
//   dw:      per 128-sample tile the tile's MLP weight gradient [n_mlp]
//   ray_loss:per ray slot of the launch the four loss sums (rgb, rr, depth, density)
#define DET_NO_KEY 0xffffffffffffffffULL
struct DetBufs {
    unsigned long long* key;
    float2* val;
    float* dw;
    float* ray_loss;
};

// ---------------------------------------------------------------------------
// launchers (defined in the kernel .cu files; all enqueue on `st`)
struct LaunchCtx {
    cudaStream_t st;
    int num_sms;
};

void launch_raygen(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, int n_objs, int total_slots,
                   RayRec* rays, unsigned long long* hit_count);
void launch_raygen_samples(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, int n_objs, int total_slots,
                           int n_iters, RayRec* rays, float4* srec, float* sdelta, unsigned long long* hit_count);
void launch_fwd_fp32(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, const RayRec* rays, int n_rays,
                     bool train, bool midpoint, float* sigma, float* rgb, float* dist, float* delta, float* act,
                     long long act_stride);
void launch_render_loss(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, const RayRec* rays, int n_rays,
                        const float* sigma, const float* rgb, const float* dist, const float* delta, float* dsigma,
                        float* drgb, double* loss_acc, int* nonfinite, const DetBufs& det);
void launch_bwd_fp32(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, const RayRec* rays, int n_rays,
                     const float* sigma, const float* rgb, const float* dsigma, const float* drgb, const float* act,
                     long long act_stride, const DetBufs& det);
// k_det.cu: the fixed-order reductions of the deterministic mode
size_t det_sort_temp_bytes(long long n_records, int n_objs);
void launch_det_reduce(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, int n_objs, int total_slots,
                       const DetBufs& det, unsigned long long* key_sorted, const unsigned* iota, unsigned* perm,
                       void* temp, size_t temp_bytes, double* loss_acc);
void launch_det_iota(const LaunchCtx& lc, unsigned* v, long long n);
void launch_adam(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, int n_objs, int* nonfinite,
                 bool write_half);
void launch_zero_grads(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, int n_objs);
void launch_render_rays(const LaunchCtx& lc, const ObjDev* obj, const KfDev* cam, int W, int H, RayRec* rays);
void launch_composite(const LaunchCtx& lc, int N, const RayRec* rays, int n_rays, const float* sigma,
                      const float* rgb, const float* dist, const float* delta, float* out_rgb, float* out_depth,
                      float* out_opacity, const int* out_idx = nullptr);
void launch_compact_rays(const LaunchCtx& lc, const RayRec* rays, int n, RayRec* out, int* idx, int* count);
// k_scene.cu: render_scene batched over objects (R20)
void launch_scene_count(const LaunchCtx& lc, const KfDev* cam, const ObjDev* objs, int n_obj, int W, int H,
                        int* pix_cnt, int* obj_cnt);
size_t scene_scan_bytes(long long HW);
void launch_scene_scan(const LaunchCtx& lc, const int* pix_cnt, int* pix_off, long long HW, void* temp,
                       size_t temp_bytes);
void launch_scene_emit(const LaunchCtx& lc, const KfDev* cam, const ObjDev* objs, int n_obj, int W, int H,
                       const int* pix_off, const int* obj_off, int* obj_fill, RayRec* segs, float* seg_tn, int* seg_id,
                       int* pix_list);
void launch_scene_pad(const LaunchCtx& lc, int n_obj, const int* obj_cnt, const int* obj_off, const int* obj_len,
                      RayRec* segs);
void launch_scene_final(const LaunchCtx& lc, long long HW, const int* pix_cnt, const int* pix_off, const int* pix_list,
                        const float* seg_tn, const int* seg_id, const float* segC, const float* segA, const float* segD,
                        float* rgb, float* depth, float* opa);
void launch_query_density(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* obj, const float* xyz, long long n,
                          float* sigma);
void launch_debug_samples(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, const RayRec* rays,
                          int ray_begin, int n_rays, int what, void* out);

// k_scene.cu -- a11 render_scene batched over objects (R20; BASELINE
// cfg4 part two: "full 640x480 render of the scene ... with per-ray box
// intersection across all object boxes, up to 128 samples per hit segment, and
// front-to-back compositing in depth order").
//
// One pass over the pixels intersects every object's box (the same bit-exact ray
// construction and slab test as the single-object path: make_ray + ray_box per
// object), and the hit (pixel, object) segments are laid out object-major, each
// object's range padded to whole 128-sample tiles, so ONE mixed forward launch
// (k_fwd_mixed, weights reloaded per object) samples every segment; k_composite
// reduces each segment to (C, A, D); k_scene_final composites, per pixel, its
// segments in ascending (t_near, object id) order over black.  The host reads the
// per-object segment counts once per frame (to size and place the ranges).
#include "romap_internal.cuh"

// camera of the frame and the objects' boxes are in `objs` (scene order); the
// per-pixel segment count and the per-object hit counts (block histogram in
// shared memory, one atomic per object and block)
__global__ void __launch_bounds__(256) k_scene_count(const KfDev* __restrict__ cam, const ObjDev* __restrict__ objs,
                                                     int n_obj, int W, int H, int* __restrict__ pix_cnt,
                                                     int* __restrict__ obj_cnt) {
    extern __shared__ int hist[];
    for (int o = threadIdx.x; o < n_obj; o += blockDim.x) hist[o] = 0;
    __syncthreads();
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < (long long)W * H) {
        const KfDev k = *cam;
        const int py = (int)(p / W), px = (int)(p - (long long)py * W);
        int c = 0;
        for (int o = 0; o < n_obj; ++o) {
            const ObjDev& ob = objs[o];
            const Ray ray = make_ray(k, px, py, ob);
            float tn, tf;
            if (ray_box(ray.o, ray.d, ob.a, tn, tf)) {
                ++c;
                atomicAdd(&hist[o], 1);
            }
        }
        pix_cnt[p] = c;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < n_obj; o += blockDim.x)
        if (hist[o]) atomicAdd(obj_cnt + o, hist[o]);
}

// the segments: per pixel, per hit object, a ray record at the object's next free
// slot (obj_off[o] + atomic fill), its t_near / object id, and its index in the
// pixel's segment list (pix_off from an exclusive scan of pix_cnt)
__global__ void __launch_bounds__(256) k_scene_emit(const KfDev* __restrict__ cam, const ObjDev* __restrict__ objs,
                                                    int n_obj, int W, int H, const int* __restrict__ pix_off,
                                                    const int* __restrict__ obj_off, int* __restrict__ obj_fill,
                                                    RayRec* __restrict__ segs, float* __restrict__ seg_tn,
                                                    int* __restrict__ seg_id, int* __restrict__ pix_list) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= (long long)W * H) return;
    const KfDev k = *cam;
    const int py = (int)(p / W), px = (int)(p - (long long)py * W);
    int j = pix_off[p];
    for (int o = 0; o < n_obj; ++o) {
        const ObjDev& ob = objs[o];
        const Ray ray = make_ray(k, px, py, ob);
        float tn, tf;
        if (!ray_box(ray.o, ray.d, ob.a, tn, tf)) continue;
        const int seg = obj_off[o] + atomicAdd(obj_fill + o, 1);
        RayRec rr;
#pragma unroll
        for (int q = 0; q < 3; ++q) { rr.o[q] = ray.o[q]; rr.d[q] = ray.d[q]; rr.tgt[q] = 0.f; rr.bg[q] = 0.f; }
        rr.tn = tn;
        rr.tf = tf;
        rr.depth = 0.f;
        rr.flags = RF_ACTIVE | RF_DRAWN;
        rr.slot = o;
        rr.kf = 0;
        rr.px = px;
        rr.py = py;
        segs[seg] = rr;
        seg_tn[seg] = tn;
        seg_id[seg] = ob.obj_id;
        pix_list[j++] = seg;
    }
}

// the padding of each object's range up to whole tiles: inactive records of that object
__global__ void k_scene_pad(int n_obj, const int* __restrict__ obj_cnt, const int* __restrict__ obj_off,
                            const int* __restrict__ obj_len, RayRec* __restrict__ segs) {
    const int o = blockIdx.x;
    if (o >= n_obj) return;
    for (int i = obj_cnt[o] + threadIdx.x; i < obj_len[o]; i += blockDim.x) {
        RayRec rr;
#pragma unroll
        for (int q = 0; q < 3; ++q) { rr.o[q] = 0.f; rr.d[q] = 0.f; rr.tgt[q] = 0.f; rr.bg[q] = 0.f; }
        rr.tn = rr.tf = rr.depth = 0.f;
        rr.flags = 0;
        rr.slot = o;
        rr.kf = rr.px = rr.py = -1;
        segs[obj_off[o] + i] = rr;
    }
}

// per pixel: its segments in ascending (t_near, object id) order, front to back
// over black: C += T C_s, D += T D_s, T *= 1 - A_s; opacity = 1 - T (R20)
__global__ void __launch_bounds__(256) k_scene_final(long long HW, const int* __restrict__ pix_cnt,
                                                     const int* __restrict__ pix_off, const int* __restrict__ pix_list,
                                                     const float* __restrict__ seg_tn, const int* __restrict__ seg_id,
                                                     const float* __restrict__ segC, const float* __restrict__ segA,
                                                     const float* __restrict__ segD, float* __restrict__ out_rgb,
                                                     float* __restrict__ out_depth, float* __restrict__ out_opa) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= HW) return;
    const int n = pix_cnt[p], base = pix_off[p];
    float C[3] = {0.f, 0.f, 0.f}, D = 0.f, T = 1.f;
    float last_t = -__int_as_float(0x7f800000);
    int last_id = -1;
    for (int step = 0; step < n; ++step) {
        // next segment after (last_t, last_id) in (t_near, id) order
        int best = -1, bid = 0;
        float bt = 0.f;
        for (int j = 0; j < n; ++j) {
            const int sg = pix_list[base + j];
            const float t = seg_tn[sg];
            const int id = seg_id[sg];
            const bool after = t > last_t || (t == last_t && id > last_id);
            if (after && (best < 0 || t < bt || (t == bt && id < bid))) { best = sg; bt = t; bid = id; }
        }
        C[0] += T * segC[3LL * best];
        C[1] += T * segC[3LL * best + 1];
        C[2] += T * segC[3LL * best + 2];
        D += T * segD[best];
        T *= 1.0f - segA[best];
        last_t = bt;
        last_id = bid;
    }
    if (out_rgb) {
        out_rgb[3 * p] = C[0];
        out_rgb[3 * p + 1] = C[1];
        out_rgb[3 * p + 2] = C[2];
    }
    if (out_depth) out_depth[p] = D;
    if (out_opa) out_opa[p] = 1.0f - T;
}

void launch_scene_count(const LaunchCtx& lc, const KfDev* cam, const ObjDev* objs, int n_obj, int W, int H,
                        int* pix_cnt, int* obj_cnt) {
    const long long HW = (long long)W * H;
    if (HW > 0)
        k_scene_count<<<(unsigned)((HW + 255) / 256), 256, (size_t)n_obj * sizeof(int), lc.st>>>(cam, objs, n_obj, W,
                                                                                                 H, pix_cnt, obj_cnt);
}

void launch_scene_emit(const LaunchCtx& lc, const KfDev* cam, const ObjDev* objs, int n_obj, int W, int H,
                       const int* pix_off, const int* obj_off, int* obj_fill, RayRec* segs, float* seg_tn, int* seg_id,
                       int* pix_list) {
    const long long HW = (long long)W * H;
    if (HW > 0)
        k_scene_emit<<<(unsigned)((HW + 255) / 256), 256, 0, lc.st>>>(cam, objs, n_obj, W, H, pix_off, obj_off,
                                                                      obj_fill, segs, seg_tn, seg_id, pix_list);
}

void launch_scene_pad(const LaunchCtx& lc, int n_obj, const int* obj_cnt, const int* obj_off, const int* obj_len,
                      RayRec* segs) {
    if (n_obj > 0) k_scene_pad<<<(unsigned)n_obj, 128, 0, lc.st>>>(n_obj, obj_cnt, obj_off, obj_len, segs);
}

void launch_scene_final(const LaunchCtx& lc, long long HW, const int* pix_cnt, const int* pix_off, const int* pix_list,
                        const float* seg_tn, const int* seg_id, const float* segC, const float* segA, const float* segD,
                        float* rgb, float* depth, float* opa) {
    if (HW > 0)
        k_scene_final<<<(unsigned)((HW + 255) / 256), 256, 0, lc.st>>>(HW, pix_cnt, pix_off, pix_list, seg_tn, seg_id,
                                                                      segC, segA, segD, rgb, depth, opa);
}

// exclusive scan of the per-pixel segment counts (CUB, library call)
#include <cub/device/device_scan.cuh>

size_t scene_scan_bytes(long long HW) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int*)nullptr, (int*)nullptr, (int)HW);
    return bytes;
}

void launch_scene_scan(const LaunchCtx& lc, const int* pix_cnt, int* pix_off, long long HW, void* temp,
                       size_t temp_bytes) {
    if (HW > 0) cub::DeviceScan::ExclusiveSum(temp, temp_bytes, pix_cnt, pix_off, (int)HW, lc.st);
}

// k_sample.cu -- step a1 of the hot path: ray generation, classification,
// ray/box segment ("transform the camera pose to the object
// coordinate system and back-project the pixels that are within the object's
// detection box.  If the ray intersects with the 3D bounding box, we compute the
// truncation distance"), batched over all objects of a launch with a segmented
// ray layout (one global ray slot per drawn ray; objects own contiguous ranges).
//
// Thread per ray slot.  All geometry is bit-exact fp32 (romap_internal.cuh).
#include "romap_internal.cuh"

// one ray slot g: object lookup, pixel draw, class, ray, slab test, targets,
// background colour (R8-R14, R17); returns the object slot and whether the ray
// is active (hit and supervised)
__device__ __forceinline__ int make_ray_rec(const CfgDev& cfg, const ObjDev* __restrict__ objs, int n_objs, int g,
                                            int iter_off, RayRec& rr, bool& active) {
    // object owning slot g (objects are sorted by ray_begin)
    int lo = 0, hi = n_objs - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (objs[mid].ray_begin <= g) lo = mid; else hi = mid - 1;
    }
    const ObjDev& ob = objs[lo];
    int r = g - ob.ray_begin;
#pragma unroll
    for (int k = 0; k < 3; ++k) { rr.o[k] = 0.f; rr.d[k] = 0.f; rr.tgt[k] = 0.f; rr.bg[k] = 0.f; }
    rr.tn = rr.tf = rr.depth = 0.f;
    rr.flags = 0;
    rr.slot = lo;
    rr.kf = rr.px = rr.py = -1;
    active = false;
    if (r < ob.n_rays) {
        long long t = *ob.step + 1 + iter_off;            // the Adam step this iteration feeds (R13)
        unsigned long long pre = rng_prefix(cfg.seed, ob.obj_id, t);
        // R9: uniform over the union of in-box pixels of all keyframes
        unsigned u = rng_u32(pre, r, 0);
        long long idx = (long long)(((unsigned long long)u * (unsigned long long)ob.total_area) >> 32);
        int klo = 0, khi = ob.n_kf - 1;
        while (klo < khi) {
            int mid = (klo + khi + 1) >> 1;
            if (ob.area_prefix[mid] <= idx) klo = mid; else khi = mid - 1;
        }
        const KfDev* kf = ob.kfs + klo;
        long long local = idx - ob.area_prefix[klo];
        int w = kf->w;
        int ly = (int)(local / w), lx = (int)(local - (long long)ly * w);
        uchar4 pix = kf->crop[(long long)ly * w + lx];
        int cls = pix.w;
        rr.tgt[0] = __fdiv_rn((float)pix.x, 255.0f);
        rr.tgt[1] = __fdiv_rn((float)pix.y, 255.0f);
        rr.tgt[2] = __fdiv_rn((float)pix.z, 255.0f);
        int px = kf->x0 + lx, py = kf->y0 + ly;
        KfDev kcopy = *kf;
        Ray ray = make_ray(kcopy, px, py, ob);
        float tn, tf;
        bool hit = ray_box(ray.o, ray.d, ob.a, tn, tf);
        active = hit && cls != CLS_OCC;                   // R10: occluders dropped
        bool has_depth = false;
        if (kcopy.depth != nullptr && cls == CLS_OBJ) {
            float z = kcopy.depth[(long long)ly * w + lx];
            has_depth = z > 0.0f;
            rr.depth = __fmul_rn(z, ray.n);               // R17: camera z -> ray distance
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            rr.o[k] = ray.o[k];
            rr.d[k] = ray.d[k];
            rr.bg[k] = u32_unit(rng_u32(pre, r, 1 + k));  // R14 random background colour
        }
        rr.tn = tn;
        rr.tf = tf;
        rr.flags = cls | (active ? RF_ACTIVE : 0) | (has_depth ? RF_HAS_DEPTH : 0) | RF_DRAWN;
        rr.kf = klo;
        rr.px = px;
        rr.py = py;
    }
    return lo;
}

// warp-aggregated hit counter per object slot
__device__ __forceinline__ void count_hit(unsigned long long* hit_count, int lo, bool active) {
    unsigned m = __ballot_sync(__activemask(), active);
    if (active) {
        unsigned same = __match_any_sync(m, lo);
        if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(hit_count + lo, (unsigned long long)__popc(same));
    }
}

// thread per ray slot; blockIdx.y = k: iteration step + 1 + k, slice k of rays
__global__ void __launch_bounds__(128) k_raygen(CfgDev cfg, const ObjDev* __restrict__ objs, int n_objs,
                                                int total_slots, RayRec* __restrict__ rays,
                                                unsigned long long* __restrict__ hit_count) {
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= total_slots) return;
    const int k = blockIdx.y;
    RayRec rr;
    bool active;
    int lo = make_ray_rec(cfg, objs, n_objs, g, k, rr, active);
    rays[(long long)k * total_slots + g] = rr;
    count_hit(hit_count, lo, active);
}

// mixed path, second phase: thread per sample of slice k = blockIdx.y, from the
// ray records k_raygen wrote: srec = (u, dist) (u = -1 for inactive rays),
// sdelta = delta (R12, R6; the same device functions as the fp32 path)
__global__ void __launch_bounds__(256) k_samples(CfgDev cfg, const ObjDev* __restrict__ objs, int total_slots,
                                                 const RayRec* __restrict__ rays, float4* __restrict__ srec,
                                                 float* __restrict__ sdelta) {
    const int N = cfg.N, k = blockIdx.y;
    const long long S = (long long)total_slots * N;
    const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const int g = (int)(s / N), i = (int)(s - (long long)g * N);
    const RayRec rr = rays[(long long)k * total_slots + g];
    float4 o = make_float4(-1.f, -1.f, -1.f, 0.f);
    float delta = 0.f;
    if (rr.flags & RF_ACTIVE) {
        const ObjDev& ob = objs[rr.slot];
        unsigned long long pre = rng_prefix(cfg.seed, ob.obj_id, *ob.step + 1 + k);
        float dist, u[3];
        sample_geometry(rr, i, N, pre, g - ob.ray_begin, ob.a, dist, delta, u);
        o = make_float4(u[0], u[1], u[2], dist);
    }
    srec[k * S + s] = o;
    sdelta[k * S + s] = delta;
}

void launch_raygen(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, int n_objs, int total_slots,
                   RayRec* rays, unsigned long long* hit_count) {
    int blocks = (total_slots + 127) / 128;
    if (blocks > 0) k_raygen<<<blocks, 128, 0, lc.st>>>(cfg, objs, n_objs, total_slots, rays, hit_count);
}

void launch_raygen_samples(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, int n_objs, int total_slots,
                           int n_iters, RayRec* rays, float4* srec, float* sdelta, unsigned long long* hit_count) {
    // two phases: every ray of the chunk in one wave (the per-ray chain of dependent
    // loads is latency-bound), then every sample from the ray records
    const long long S = (long long)total_slots * cfg.N;
    if (total_slots == 0 || n_iters == 0) return;
    k_raygen<<<dim3((unsigned)((total_slots + 127) / 128), (unsigned)n_iters), 128, 0, lc.st>>>(
        cfg, objs, n_objs, total_slots, rays, hit_count);
    k_samples<<<dim3((unsigned)((S + 255) / 256), (unsigned)n_iters), 256, 0, lc.st>>>(cfg, objs, total_slots, rays,
                                                                                       srec, sdelta);
}

// inference rays: every pixel of a W x H image from pose `cam` (R12, R20)
__global__ void __launch_bounds__(128) k_render_rays(const ObjDev* __restrict__ obj, const KfDev* __restrict__ cam,
                                                     int W, int H, RayRec* __restrict__ rays) {
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= W * H) return;
    int py = g / W, px = g - py * W;
    KfDev k = *cam;
    ObjDev ob = *obj;
    Ray ray = make_ray(k, px, py, ob);
    float tn, tf;
    bool hit = ray_box(ray.o, ray.d, ob.a, tn, tf);
    RayRec rr;
#pragma unroll
    for (int j = 0; j < 3; ++j) { rr.o[j] = ray.o[j]; rr.d[j] = ray.d[j]; rr.tgt[j] = 0.f; rr.bg[j] = 0.f; }
    rr.tn = tn;
    rr.tf = tf;
    rr.depth = 0.f;
    rr.flags = (hit ? RF_ACTIVE : 0) | RF_DRAWN;
    rr.slot = 0;
    rr.kf = 0;
    rr.px = px;
    rr.py = py;
    rays[g] = rr;
}

void launch_render_rays(const LaunchCtx& lc, const ObjDev* obj, const KfDev* cam, int W, int H, RayRec* rays) {
    int n = W * H;
    if (n > 0) k_render_rays<<<(n + 127) / 128, 128, 0, lc.st>>>(obj, cam, W, H, rays);
}

// k_det.cu -- deterministic-reduction mode (romap_set_deterministic; SURVEY.md
// 8(c) "bitwise in a deterministic-reduction debug mode", SPEC.md:436,450,452:
// serial == parallel, batch == alone, occluder exclusion bitwise).
//
// The training kernels built for this mode (k_fused_mixed_det, k_bwd_fp32 /
// k_render_loss with det buffers) write every contribution to a record instead
// of an fp32 atomic (romap_internal.cuh DetBufs).  Here the records are reduced
// in a fixed order:
//   table gradients: stable radix sort of the (object slot, entry) keys, then
//     every run of equal keys is summed in record order = (sample, level,
//     corner) order within the object, and added to that entry (one writer)
//   MLP gradients:   per parameter, the object's per-tile partials in tile order
//   losses:          per object and term, the per-ray sums in ray order (fp64)
// Within one object the sample / tile / ray order does not depend on where the
// object sits in the batch, so an object trained in a batch equals the same
// object trained alone, bit for bit, and graph replays equal plain launches.
// Speed is irrelevant here (tests only).
#include <cub/device/device_radix_sort.cuh>

#include "romap_internal.cuh"

// keys are (slot << 32 | entry) and the DET_NO_KEY sentinel (~0, sorts last): all 64 bits
static int key_bits(int) { return 64; }

size_t det_sort_temp_bytes(long long n_records, int n_objs) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (const unsigned*)nullptr, (unsigned*)nullptr, (int)n_records, 0, key_bits(n_objs));
    return bytes;
}

__global__ void k_det_iota(unsigned* __restrict__ v, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (unsigned)i;
}

// one thread per sorted record: the first record of every run of equal keys sums
// the run in record order and adds it to the table entry
__global__ void k_det_table(const ObjDev* __restrict__ objs, const unsigned long long* __restrict__ key,
                            const unsigned* __restrict__ perm, const float2* __restrict__ val, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = key[i];
    if (k == DET_NO_KEY || (i > 0 && key[i - 1] == k)) return;
    float s0 = 0.f, s1 = 0.f;
    for (long long j = i; j < n && key[j] == k; ++j) {
        const float2 v = val[perm[j]];
        s0 += v.x;
        s1 += v.y;
    }
    const int slot = (int)(k >> 32);
    const unsigned e = (unsigned)(k & 0xffffffffu);
    float2* g = reinterpret_cast<float2*>(objs[slot].g32) + e;
    const float2 o = *g;
    *g = make_float2(o.x + s0, o.y + s1);
}

// grid (params / 256, objects): per MLP parameter the object's tile partials in tile order
__global__ void k_det_dw(CfgDev cfg, const ObjDev* __restrict__ objs, const float* __restrict__ dw) {
    const ObjDev& ob = objs[blockIdx.y];
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= cfg.n_mlp) return;
    const long long t0 = (long long)ob.ray_begin * cfg.N / ROMAP_TILE;
    const long long t1 = (long long)(ob.ray_begin + ob.n_slots) * cfg.N / ROMAP_TILE;
    float s = 0.f;
    for (long long t = t0; t < t1; ++t) s += dw[t * cfg.n_mlp + p];
    float* g = ob.g32 + cfg.n_table + p;
    *g = *g + s;
}

// block per object, thread per loss term: per-ray sums in ray order (fp64)
__global__ void k_det_loss(const ObjDev* __restrict__ objs, const float* __restrict__ ray_loss,
                           double* __restrict__ loss_acc) {
    const ObjDev& ob = objs[blockIdx.x];
    const int k = threadIdx.x;
    if (k >= 4) return;
    double s = 0.0;
    for (int r = ob.ray_begin; r < ob.ray_begin + ob.n_slots; ++r) s += (double)ray_loss[4LL * r + k];
    loss_acc[4 * blockIdx.x + k] += s;
}

void launch_det_reduce(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, int n_objs, int total_slots,
                       const DetBufs& det, unsigned long long* key_sorted, const unsigned* iota, unsigned* perm,
                       void* temp, size_t temp_bytes, double* loss_acc) {
    const long long S = (long long)total_slots * cfg.N;
    const long long n = S * cfg.L * 8;
    if (n == 0) return;
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, det.key, key_sorted, iota, perm, (int)n, 0, key_bits(n_objs),
                                    lc.st);
    k_det_table<<<(unsigned)((n + 255) / 256), 256, 0, lc.st>>>(objs, key_sorted, perm, det.val, n);
    k_det_dw<<<dim3((unsigned)((cfg.n_mlp + 255) / 256), (unsigned)n_objs), 256, 0, lc.st>>>(cfg, objs, det.dw);
    k_det_loss<<<(unsigned)n_objs, 32, 0, lc.st>>>(objs, det.ray_loss, loss_acc);
}

void launch_det_iota(const LaunchCtx& lc, unsigned* v, long long n) {
    if (n > 0) k_det_iota<<<(unsigned)((n + 255) / 256), 256, 0, lc.st>>>(v, n);
}

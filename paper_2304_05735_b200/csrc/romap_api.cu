// romap_api.cu -- host runtime behind the C ABI (include/romap.h).
//
// Owns: the object registry, per-object parameter / gradient / Adam blocks,
// per-object keyframe crops on the device, the segmented ray layout of a
// train_step batch, and the launch sequence of one iteration (mixed path:
// raygen + samples of K iterations -> fused step -> Adam, chunks of K replayed
// as one CUDA graph; fp32 path: raygen -> fwd -> render_loss -> bwd -> Adam; the
// Adam launch advances the step counters).  Everything is enqueued on the
// context's stream; the host only crosses the boundary at launch and at the
// final statistics read-back.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <chrono>
#include <cstdlib>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/romap.h"
#include "romap_internal.cuh"

// NVTX ranges around the public entry points and the stages of a train_step, so
// `ncu --nvtx --nvtx-include "romap_train_step/"` (or an nsys timeline) can select
// and attribute kernels; header-only NVTX3, a no-op unless a tool is attached
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define NVTX_RANGE(name) NvtxRange nvtx_range_(name)

void launch_fused_mixed(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, const RayRec* rays,
                        const float4* srec, const float* sdelta, int n_rays, double* loss_acc, int* nonfinite,
                        float* dbg_ray_grads);
void launch_fused_mixed_det(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* objs, const RayRec* rays,
                            const float4* srec, const float* sdelta, int n_rays, double* loss_acc, int* nonfinite,
                            float* dbg_ray_grads, DetBufs det);
bool fused_mixed_available();
void launch_fwd_mixed(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* obj, const RayRec* rays, int n_rays,
                      float* sigma, float* rgb, float* dist, float* delta);
void launch_lattice(const LaunchCtx& lc, const ObjDev* obj, int R, float* pts);
void launch_carve(const LaunchCtx& lc, const ObjDev* obj, const float* pts, long long nv, float* sig);
size_t mt_scan_bytes(long long ncell);
void launch_mt(const LaunchCtx& lc, const ObjDev* obj, const float* sig, const float* pts, int R, float iso,
               int* counts, int* offsets, void* tmp, size_t tmp_bytes, float* tris, bool emit);
void launch_query_density_mixed(const LaunchCtx& lc, const CfgDev& cfg, const ObjDev* obj, const float* xyz,
                                long long n, float* sigma);
void launch_debug_mixed(const LaunchCtx& lc, const CfgDev& cfg, const float4* srec, const float* sdelta, long long n,
                        int what, void* out);

static thread_local std::string g_err;

static romap_status fail(romap_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

struct Keyframe {
    KfDev dev;
    uchar4* crop_d = nullptr;
    float* depth_d = nullptr;
    long long area = 0;
};

struct Object {
    int id = 0, instance_id = 0;
    romap_box box{};
    romap_model_config cfg{};
    CfgDev cdev{};
    float c = 1.f, s = 0.f;
    float* p32 = nullptr;
    float* g32 = nullptr;
    float* m = nullptr;
    float* v = nullptr;
    __half* p16 = nullptr;
    long long* step_d = nullptr;
    std::vector<Keyframe> kfs;
    KfDev* kfs_d = nullptr;
    long long* prefix_d = nullptr;
    size_t kfs_cap = 0;
    long long total_area = 0;
    long long step = 0;
    int rays_per_iter = 0;
    bool grads_dirty = false;
    // last batch (debug dumps)
    int last_ray_begin = -1, last_n_rays = 0;
    // keyframe crops / depth live in a bump arena of device chunks (one cudaMalloc
    // per few MB instead of one per keyframe; freed with the object)
    std::vector<void*> kf_chunks;
    size_t kf_used = 0, kf_cap = 0;
    // f3 online policy (R25): camera centre of the last accepted keyframe, pending budget
    bool has_gate_ref = false;
    double gate_ref[3] = {0, 0, 0};
    long long pending_iters = 0;
};

enum LastCall { LAST_NONE = 0, LAST_TRAIN = 1, LAST_FWDBWD = 2 };

enum Stage { ST_RAYGEN = 0, ST_FWD, ST_RENDER_LOSS, ST_BWD, ST_FUSED, ST_ADAM, ST_STEP_INC, ST_ZERO_GRADS, ST_FLUSH,
             ST_DET, ST_GRAPH, ST_COUNT };
// (det_reduce: the deterministic mode's fixed-order reductions; graph_replay:
// cudaGraphLaunch calls of a captured K-iteration chunk, its kernels are counted
// under their own stages)
static const char* kStageNames[ST_COUNT] = {"raygen", "fwd_fp32", "render_loss", "bwd_fp32", "fused_mixed",
                                             "adam", "step_inc", "zero_grads", "l2_flush", "det_reduce",
                                             "graph_replay"};

// per-stage launch counters and (optional) CUDA-event timing on the ctx stream
struct Profiler {
    bool on = false;
    uint32_t mask = 0xffffffffu;  // stages bracketed with events when on
    long long launches[ST_COUNT] = {};
    double ms[ST_COUNT] = {};
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<char> pending_shared;  // start event is the previous interval's end (not pooled twice)
    cudaEvent_t tail = nullptr;        // last end event recorded on the stream ...
    bool tail_valid = false;           // ... with nothing enqueued after it
    cudaEvent_t get() {
        if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};

struct AsyncFrame {
    int obj;
    std::vector<uint8_t> rgb;
    std::vector<uint16_t> mask;
    float T[12];
    romap_intrinsics K;
};

// f3 asynchronous online trainer (romap_async_*): a worker thread owns the context
struct AsyncState {
    std::thread worker;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<AsyncFrame> queue;
    bool stop = false, finish = false;
    int chunk = 100, iters_per_update = 300, cap = 64;
    float alpha_deg = 25.f;
    long long offered = 0, dropped = 0, accepted = 0, iterations = 0, max_depth = 0, rejected = 0;
    romap_status error = 0;
    std::string error_msg;
};

struct romap_ctx {
    int device = 0;
    cudaStream_t st = nullptr;
    bool own_stream = false;     // created by romap_ctx_create (the caller passed NULL)
    romap_alloc_fn alloc = nullptr;
    romap_free_fn free_fn = nullptr;
    void* user = nullptr;
    int num_sms = 148;
    bool poisoned = false;
    std::map<int, Object*> objs;
    int next_id = 0;
    // scratch (grown on demand)
    RayRec* rays = nullptr;
    size_t rays_cap = 0;
    float* samp = nullptr;       // sigma | rgb(3) | dist | delta | dsigma | drgb(3) : 10 floats per sample
    size_t samp_cap = 0;
    float* srec = nullptr;       // mixed path: K slices of (u, dist) float4, then K slices of delta (k_raygen + k_samples)
    size_t srec_cap = 0;
    size_t last_ray_base = 0;    // ray slot of slice holding the last iteration's rays
    int last_K = 1;              // mixed path: slices of the last call's sample records
    float* act = nullptr;
    size_t act_cap = 0;
    ObjDev* objdev_d = nullptr;
    size_t objdev_cap = 0;
    ObjDev* single_d = nullptr;  // render / query object
    KfDev* cam_d = nullptr;
    double* loss_d = nullptr;
    unsigned long long* hits_d = nullptr;
    int* nonfinite_d = nullptr;
    size_t stat_cap = 0;
    RayRec* rays_c = nullptr;    // render: rays that hit the box, packed
    size_t rays_c_cap = 0;
    int* ray_idx = nullptr;      // render: pixel of each packed ray (+ the packed count)
    size_t ray_idx_cap = 0;
    float* scene_d = nullptr;    // render_scene: per segment t_near, id, C (rgb), A, D + pixel segment lists
    size_t scene_cap = 0;
    int* scene_i = nullptr;      // render_scene: per pixel counts / offsets, per object counts / ranges, scan scratch
    size_t scene_i_cap = 0;
    ObjDev* scene_objs_d = nullptr;   // render_scene: descriptors of the scene's objects
    size_t scene_objs_cap = 0;
    float* mesh_d = nullptr;     // extract_mesh: lattice points | sigma | counts | offsets | CUB scratch
    size_t mesh_cap = 0;
    float* tris_d = nullptr;     // extract_mesh: triangles (device staging for host outputs)
    size_t tris_cap = 0;
    float* io_d = nullptr;       // render / query staging
    size_t io_cap = 0;
    // add_observation: pinned host staging of the in-box crop (+ depth) so its H2D
    // copy is a true async DMA; reused once the previous copy from it completed
    void* pin = nullptr;
    size_t pin_cap = 0;
    cudaEvent_t pin_ev = nullptr;
    bool pin_pending = false;
    // last batch
    std::vector<ObjDev> last_objdev;
    CfgDev last_cfg{};
    int last_call = LAST_NONE;
    int last_total_slots = 0;
    Profiler prof;
    AsyncState* async = nullptr;    // non-null while the async worker runs
    void* flush_buf = nullptr;
    size_t flush_bytes = 0;
    // deterministic-reduction mode (romap_set_deterministic; DetBufs, k_det.cu)
    bool det_on = false;
    void* det_mem = nullptr;
    size_t det_cap = 0;          // bytes
    DetBufs det{};
    unsigned long long* det_key_sorted = nullptr;
    unsigned* det_iota = nullptr;
    unsigned* det_perm = nullptr;
    void* det_temp = nullptr;
    size_t det_temp_bytes = 0;
    // a9: CUDA graph of one chunk of K training iterations of the mixed path
    // (raygen of K slices, then K x [flush], fused, Adam), replayed while the batch,
    // its config and every buffer it touches stay the same
    struct TrainGraph {
        cudaGraphExec_t exec = nullptr;
        CfgDev cfg;
        int n = 0, total_slots = 0, K = 0;
        bool det = false;
        const void* ptrs[8] = {};
        size_t flush_bytes = 0;
    } tg;
};

// bracket one launch: stage_begin returns the start event (or null)
// (back-to-back bracketed launches share one event: the end of one interval is
// the start of the next, so a timed step carries as few event records as possible)
static cudaEvent_t stage_begin(romap_ctx* ctx, int stage) {
    ctx->prof.launches[stage]++;
    if (!ctx->prof.on || !((ctx->prof.mask >> stage) & 1u)) {
        ctx->prof.tail_valid = false;           // an unbracketed launch follows
        return nullptr;
    }
    if (ctx->prof.tail_valid) {
        ctx->prof.tail_valid = false;
        ctx->prof.pending_shared.push_back(1);
        return ctx->prof.tail;
    }
    cudaEvent_t e = ctx->prof.get();
    cudaEventRecord(e, ctx->st);
    ctx->prof.pending_shared.push_back(0);
    return e;
}
static void stage_end(romap_ctx* ctx, int stage, cudaEvent_t e0) {
    if (!e0) return;
    cudaEvent_t e1 = ctx->prof.get();
    cudaEventRecord(e1, ctx->st);
    ctx->prof.pending.push_back({stage, {e0, e1}});
    ctx->prof.tail = e1;
    ctx->prof.tail_valid = true;
}
// anything else enqueued on the stream ends the chain of shared events
static void stage_break(romap_ctx* ctx) { ctx->prof.tail_valid = false; }
// after a stream sync: fold pending intervals into the totals
static void prof_collect(romap_ctx* ctx) {
    for (size_t i = 0; i < ctx->prof.pending.size(); ++i) {
        auto& p = ctx->prof.pending[i];
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.second.first, p.second.second) == cudaSuccess) ctx->prof.ms[p.first] += ms;
        if (!ctx->prof.pending_shared[i]) ctx->prof.pool.push_back(p.second.first);
        ctx->prof.pool.push_back(p.second.second);
    }
    ctx->prof.pending.clear();
    ctx->prof.pending_shared.clear();
    ctx->prof.tail_valid = false;
}
#define STAGE(stage, launch)                      \
    do {                                          \
        cudaEvent_t e0_ = stage_begin(ctx, stage); \
        launch;                                   \
        stage_end(ctx, stage, e0_);               \
    } while (0)

// ---------------------------------------------------------------------------
// memory
static void* dalloc(romap_ctx* c, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (c->alloc) return c->alloc(bytes, c->user);
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}
static void dfree(romap_ctx* c, void* p) {
    if (!p) return;
    if (c->free_fn) c->free_fn(p, c->user);
    else cudaFree(p);
}

template <class T>
static bool grow(romap_ctx* c, T*& ptr, size_t& cap, size_t need) {
    if (need <= cap && ptr) return true;
    size_t n = need + need / 4 + 64;
    cudaStreamSynchronize(c->st);
    dfree(c, ptr);
    ptr = (T*)dalloc(c, n * sizeof(T));
    cap = ptr ? n : 0;
    return ptr != nullptr;
}

#define CK(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) {                                                                  \
            ctx->poisoned = true;                                                                 \
            return fail(ROMAP_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
        }                                                                                         \
    } while (0)

// true on the async worker thread (it may use the context while async runs)
static thread_local bool t_async_worker = false;

#define CHECK_CTX()                                                                 \
    do {                                                                            \
        if (!ctx) return fail(ROMAP_E_INVALID, "null context");                     \
        if (ctx->poisoned) return fail(ROMAP_E_CUDA, "context poisoned by an earlier CUDA error"); \
        if (ctx->async && !t_async_worker)                                         \
            return fail(ROMAP_E_STATE, "the async worker owns the context (romap_async_stop first)"); \
        cudaSetDevice(ctx->device);                                                 \
    } while (0)

// ---------------------------------------------------------------------------
// (out, in) of the bias-free layers (R1, R4; network 1: R24); returns the count
static int mlp_layer_shapes(const CfgDev& cd, int shapes[5][2]) {
    if (cd.net == 1) {
        int n = 0;
        shapes[n][0] = ROMAP_WIDTH; shapes[n][1] = cd.LF; ++n;
        for (int k = 1; k < cd.hl; ++k) { shapes[n][0] = ROMAP_WIDTH; shapes[n][1] = ROMAP_WIDTH; ++n; }
        shapes[n][0] = 4; shapes[n][1] = ROMAP_WIDTH; ++n;
        return n;
    }
    const int s[5][2] = {{ROMAP_WIDTH, cd.LF}, {ROMAP_DOUT, ROMAP_WIDTH}, {ROMAP_WIDTH, ROMAP_CIN},
                         {ROMAP_WIDTH, ROMAP_WIDTH}, {3, ROMAP_WIDTH}};
    for (int k = 0; k < 5; ++k) { shapes[k][0] = s[k][0]; shapes[k][1] = s[k][1]; }
    return 5;
}

// ---------------------------------------------------------------------------
// configuration (R5)
static romap_status build_cfg(const romap_model_config* cfg, CfgDev& cd) {
    if (!cfg) return fail(ROMAP_E_INVALID, "null config");
    if (cfg->feats != 2) return fail(ROMAP_E_INVALID, "feats must be 2");
    if (cfg->levels < 1 || cfg->levels > ROMAP_MAX_LEVELS) return fail(ROMAP_E_INVALID, "levels must be in [1,16]");
    if (cfg->log2_T < 4 || cfg->log2_T > 24) return fail(ROMAP_E_INVALID, "log2_T must be in [4,24]");
    if (cfg->base_res < 1 || !(cfg->finest_res >= cfg->base_res)) return fail(ROMAP_E_INVALID, "need finest_res >= base_res >= 1");
    if (cfg->network != 0 && cfg->network != 1) return fail(ROMAP_E_INVALID, "network must be 0 or 1");
    if (cfg->width != ROMAP_WIDTH) return fail(ROMAP_E_INVALID, "width must be 64");
    if (cfg->network == 0 && (cfg->density_out != ROMAP_DOUT || cfg->color_hidden != 2 || cfg->dir_enc != ROMAP_SH))
        return fail(ROMAP_E_INVALID, "network 0 must be density_out 16, color_hidden 2, dir_enc 16");
    if (cfg->network == 1 && (cfg->hidden_layers < 1 || cfg->hidden_layers > 3))
        return fail(ROMAP_E_INVALID, "network 1 needs hidden_layers in [1,3]");
    if (cfg->network == 1 && cfg->precision != 1)
        return fail(ROMAP_E_INVALID, "network 1 runs on the mixed path only (precision 1)");
    if (cfg->precision != 0 && cfg->precision != 1) return fail(ROMAP_E_INVALID, "precision must be 0 or 1");
    if (cfg->precision == 1 && !fused_mixed_available()) return fail(ROMAP_E_INVALID, "mixed path not built");
    if (cfg->density_act != 0 && cfg->density_act != 1) return fail(ROMAP_E_INVALID, "density_act must be 0 or 1");
    int N = cfg->samples_per_ray;
    if (N < 1 || N > 128 || (N & (N - 1))) return fail(ROMAP_E_INVALID, "samples_per_ray must be a power of two <= 128");
    if (cfg->precision == 1 && N < 8) return fail(ROMAP_E_INVALID, "mixed path needs samples_per_ray >= 8");
    if (cfg->precision == 1 && cfg->levels != 8 && cfg->levels != 16)
        return fail(ROMAP_E_INVALID, "mixed path needs levels 8 or 16 (L*F = 16 or 32 tensor-core columns)");
    if (cfg->rays_per_iter < 1) return fail(ROMAP_E_INVALID, "rays_per_iter must be >= 1");
    if (!(cfg->lr > 0) || !(cfg->beta1 >= 0 && cfg->beta1 < 1) || !(cfg->beta2 >= 0 && cfg->beta2 < 1) || !(cfg->eps >= 0))
        return fail(ROMAP_E_INVALID, "bad Adam hyper-parameters");
    if (!(cfg->lambda_depth >= 0) || !(cfg->lambda_density >= 0)) return fail(ROMAP_E_INVALID, "lambdas must be >= 0");
    if (cfg->precision == 1 && !(cfg->loss_scale > 0)) return fail(ROMAP_E_INVALID, "loss_scale must be > 0");
    memset(&cd, 0, sizeof cd);
    cd.L = cfg->levels;
    cd.F = cfg->feats;
    cd.LF = cd.L * cd.F;
    cd.log2T = cfg->log2_T;
    cd.T = 1 << cfg->log2_T;
    double b = cfg->levels > 1 ? pow(cfg->finest_res / (double)cfg->base_res, 1.0 / (cfg->levels - 1)) : 1.0;
    long long off = 0;
    for (int l = 0; l < cd.L; ++l) {
        long long n = (long long)floor((double)cfg->base_res * pow(b, (double)l) + 1e-6);
        if (cfg->res_cap > 0 && n > cfg->res_cap) n = cfg->res_cap;
        if (n > 100000) return fail(ROMAP_E_INVALID, "level resolution too large");
        long long v = (n + 1) * (n + 1) * (n + 1);
        bool dense = v <= cd.T;
        cd.res[l] = (int)n;
        cd.dense[l] = dense ? 1 : 0;
        cd.off[l] = (int)off;
        off += ((dense ? v : cd.T) + 15) / 16 * 16;   // R5: level blocks padded to 16 entries
    }
    cd.n_entries = (int)off;
    cd.n_table = (int)(off * cd.F);
    cd.net = cfg->network;
    cd.hl = cfg->network == 1 ? cfg->hidden_layers : 0;
    int shapes[5][2];
    cd.n_layers = mlp_layer_shapes(cd, shapes);
    int o = 0;
    for (int k = 0; k < 5; ++k) {
        cd.w_off[k] = o;
        if (k < cd.n_layers) o += shapes[k][0] * shapes[k][1];
    }
    cd.n_mlp = o;
    cd.N = N;
    cd.density_act = cfg->density_act;
    cd.obj_bg = cfg->obj_bg;
    cd.lambda_depth = cfg->lambda_depth;
    cd.lambda_density = cfg->lambda_density;
    cd.lr = cfg->lr;
    cd.b1 = cfg->beta1;
    cd.b2 = cfg->beta2;
    cd.eps = cfg->eps;
    cd.loss_scale = cfg->precision == 1 ? cfg->loss_scale : 1.0f;
    cd.seed = cfg->seed;
    return ROMAP_OK;
}

static bool same_model(const romap_model_config& a, const romap_model_config& b) {
    return a.levels == b.levels && a.feats == b.feats && a.log2_T == b.log2_T && a.base_res == b.base_res &&
           a.finest_res == b.finest_res && a.res_cap == b.res_cap && a.width == b.width &&
           a.density_out == b.density_out && a.color_hidden == b.color_hidden && a.dir_enc == b.dir_enc &&
           a.precision == b.precision && a.density_act == b.density_act && a.samples_per_ray == b.samples_per_ray &&
           a.lr == b.lr && a.beta1 == b.beta1 && a.beta2 == b.beta2 && a.eps == b.eps &&
           a.lambda_depth == b.lambda_depth && a.lambda_density == b.lambda_density && a.loss_scale == b.loss_scale &&
           a.obj_bg == b.obj_bg && a.seed == b.seed && a.network == b.network && a.hidden_layers == b.hidden_layers;
}

// host RNG for initialisation (R19); independent of the training RNG streams
struct HostRng {
    unsigned long long s;
    unsigned long long next() { s += ROMAP_GOLDEN; return mix64(s); }
    double unit() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
};

static ObjDev make_objdev(const Object* ob) {
    ObjDev d;
    memset(&d, 0, sizeof d);
    for (int k = 0; k < 3; ++k) { d.a[k] = ob->box.half_extents[k]; d.t[k] = ob->box.t[k]; }
    d.c = ob->c;
    d.s = ob->s;
    d.p32 = ob->p32;
    d.g32 = ob->g32;
    d.m = ob->m;
    d.v = ob->v;
    d.p16 = ob->p16;
    d.kfs = ob->kfs_d;
    d.area_prefix = ob->prefix_d;
    d.n_kf = (int)ob->kfs.size();
    d.total_area = ob->total_area;
    d.obj_id = ob->id;
    d.step = ob->step_d;
    return d;
}

// bias corrections 1 / (1 - beta^t) of the next Adam step t = step + 1 (double,
// rounded once), stored after the step counter for k_adam (synchronous copy)
static cudaError_t upload_bias_corrections(romap_ctx* ctx, Object* ob) {
    const double t = (double)(ob->step + 1);
    float bc[2] = {(float)(1.0 / (1.0 - pow((double)ob->cdev.b1, t))), (float)(1.0 / (1.0 - pow((double)ob->cdev.b2, t)))};
    cudaError_t e = cudaMemcpyAsync(ob->step_d + 2, bc, sizeof bc, cudaMemcpyHostToDevice, ctx->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->st);
    return e;
}

static Object* find(romap_ctx* ctx, int id) {
    auto it = ctx->objs.find(id);
    return it == ctx->objs.end() ? nullptr : it->second;
}

// ---------------------------------------------------------------------------
extern "C" {

const char* romap_last_error(void) { return g_err.c_str(); }
const char* romap_version(void) { return "romap-b200 0.2 (sm_100a)"; }

romap_status romap_ctx_create(int32_t device, void* cuda_stream, romap_alloc_fn alloc, romap_free_fn free_fn,
                              void* user, romap_ctx** out) {
    if (!out) return fail(ROMAP_E_INVALID, "null out");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(ROMAP_E_CUDA, "no CUDA device");
    }
    if (device < 0 || device >= n) return fail(ROMAP_E_INVALID, "bad device %d", device);
    if ((alloc == nullptr) != (free_fn == nullptr)) return fail(ROMAP_E_INVALID, "alloc and free must both be set");
    if (cudaSetDevice(device) != cudaSuccess) return fail(ROMAP_E_CUDA, "cudaSetDevice failed");
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return fail(ROMAP_E_CUDA, "cudaGetDeviceProperties failed");
    if (prop.major != 10) return fail(ROMAP_E_INVALID, "libromap is built for sm_100a (B200); device is sm_%d%d", prop.major, prop.minor);
    romap_ctx* ctx = new romap_ctx();
    ctx->device = device;
    ctx->st = (cudaStream_t)cuda_stream;
    if (!ctx->st) {
        // no stream given: a stream of our own (a CUDA graph cannot be captured on
        // the legacy NULL stream, a9).  A blocking stream: it stays ordered with work
        // the caller enqueues on the legacy default stream (e.g. torch's)
        if (cudaStreamCreate(&ctx->st) != cudaSuccess) {
            cudaGetLastError();
            delete ctx;
            return fail(ROMAP_E_CUDA, "cudaStreamCreate failed");
        }
        ctx->own_stream = true;
    }
    ctx->alloc = alloc;
    ctx->free_fn = free_fn;
    ctx->user = user;
    ctx->num_sms = prop.multiProcessorCount;
    ctx->single_d = (ObjDev*)dalloc(ctx, sizeof(ObjDev));
    ctx->cam_d = (KfDev*)dalloc(ctx, sizeof(KfDev));
    if (!ctx->single_d || !ctx->cam_d) {
        if (ctx->own_stream) cudaStreamDestroy(ctx->st);
        delete ctx;
        return fail(ROMAP_E_OOM, "context allocation failed");
    }
    *out = ctx;
    return ROMAP_OK;
}

static void free_object(romap_ctx* ctx, Object* ob) {
    dfree(ctx, ob->p32);
    dfree(ctx, ob->g32);
    dfree(ctx, ob->m);
    dfree(ctx, ob->v);
    dfree(ctx, ob->p16);
    dfree(ctx, ob->step_d);
    for (void* c : ob->kf_chunks) dfree(ctx, c);     // keyframe crops and depth (arena)
    dfree(ctx, ob->kfs_d);
    dfree(ctx, ob->prefix_d);
    delete ob;
}

romap_status romap_ctx_destroy(romap_ctx* ctx) {
    if (!ctx) return fail(ROMAP_E_INVALID, "null context");
    if (ctx->async) romap_async_stop(ctx, 0, nullptr);
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->st);
    for (auto& kv : ctx->objs) free_object(ctx, kv.second);
    dfree(ctx, ctx->rays);
    dfree(ctx, ctx->samp);
    dfree(ctx, ctx->srec);
    dfree(ctx, ctx->scene_d);
    dfree(ctx, ctx->scene_i);
    dfree(ctx, ctx->scene_objs_d);
    dfree(ctx, ctx->rays_c);
    dfree(ctx, ctx->ray_idx);
    dfree(ctx, ctx->mesh_d);
    dfree(ctx, ctx->tris_d);
    dfree(ctx, ctx->act);
    dfree(ctx, ctx->objdev_d);
    dfree(ctx, ctx->single_d);
    dfree(ctx, ctx->cam_d);
    dfree(ctx, ctx->loss_d);
    dfree(ctx, ctx->hits_d);
    dfree(ctx, ctx->nonfinite_d);
    dfree(ctx, ctx->io_d);
    dfree(ctx, ctx->flush_buf);
    dfree(ctx, ctx->det_mem);
    if (ctx->pin) cudaFreeHost(ctx->pin);
    if (ctx->pin_ev) cudaEventDestroy(ctx->pin_ev);
    if (ctx->tg.exec) cudaGraphExecDestroy(ctx->tg.exec);
    prof_collect(ctx);
    for (auto e : ctx->prof.pool) cudaEventDestroy(e);
    if (ctx->own_stream) cudaStreamDestroy(ctx->st);
    delete ctx;
    return ROMAP_OK;
}

static romap_status check_box(const romap_box* box) {
    if (!box) return fail(ROMAP_E_INVALID, "null box");
    for (int k = 0; k < 3; ++k)
        if (!(box->half_extents[k] > 0) || !std::isfinite(box->half_extents[k]) || !std::isfinite(box->t[k]))
            return fail(ROMAP_E_INVALID, "box must have finite centre and positive half extents");
    if (!std::isfinite(box->yaw)) return fail(ROMAP_E_INVALID, "non-finite yaw");
    return ROMAP_OK;
}

static romap_status create_impl(romap_ctx* ctx, const romap_box* box, const romap_model_config* cfg,
                                int32_t instance_id, int32_t id) {
    romap_status sb = check_box(box);
    if (sb) return sb;
    if (id < 0) return fail(ROMAP_E_INVALID, "object id must be >= 0");
    if (find(ctx, id)) return fail(ROMAP_E_INVALID, "object id %d exists", id);
    CfgDev cd;
    romap_status st = build_cfg(cfg, cd);
    if (st) return st;
    Object* ob = new Object();
    ob->id = id;
    ob->instance_id = instance_id;
    ob->box = *box;
    ob->cfg = *cfg;
    ob->cdev = cd;
    ob->c = (float)cos((double)box->yaw);   // R8: cos/sin in double, rounded
    ob->s = (float)sin((double)box->yaw);
    ob->rays_per_iter = cfg->rays_per_iter;
    size_t n = (size_t)cd.n_table + cd.n_mlp;
    ob->p32 = (float*)dalloc(ctx, n * 4);
    ob->g32 = (float*)dalloc(ctx, n * 4);
    ob->m = (float*)dalloc(ctx, n * 4);
    ob->v = (float*)dalloc(ctx, n * 4);
    ob->p16 = (__half*)dalloc(ctx, n * 2 + 16);
    ob->step_d = (long long*)dalloc(ctx, 32);   // [Adam step, k_adam block counter, next bias corrections]
    if (!ob->p32 || !ob->g32 || !ob->m || !ob->v || !ob->p16 || !ob->step_d) {
        free_object(ctx, ob);
        return fail(ROMAP_E_OOM, "parameter allocation failed");
    }
    // R19 initialisation
    std::vector<float> host(n);
    std::vector<__half> h16(n);
    HostRng rng{cfg->seed ^ mix64(0x5eedULL + (unsigned long long)id)};
    for (int i = 0; i < cd.n_table; ++i) host[i] = (float)((rng.unit() * 2.0 - 1.0) * 1e-4);
    int shapes[5][2];
    const int n_layers = mlp_layer_shapes(cd, shapes);
    for (int k = 0; k < n_layers; ++k) {
        double lim = sqrt(6.0 / (shapes[k][0] + shapes[k][1]));
        for (int e = 0; e < shapes[k][0] * shapes[k][1]; ++e)
            host[cd.n_table + cd.w_off[k] + e] = (float)((rng.unit() * 2.0 - 1.0) * lim);
    }
    for (size_t i = 0; i < n; ++i) h16[i] = __float2half_rn(host[i]);
    cudaError_t e = cudaMemcpyAsync(ob->p32, host.data(), n * 4, cudaMemcpyHostToDevice, ctx->st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ob->p16, h16.data(), n * 2, cudaMemcpyHostToDevice, ctx->st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ob->g32, 0, n * 4, ctx->st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ob->m, 0, n * 4, ctx->st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ob->v, 0, n * 4, ctx->st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ob->step_d, 0, 32, ctx->st);
    if (e == cudaSuccess) e = upload_bias_corrections(ctx, ob);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->st);
    if (e != cudaSuccess) {
        ctx->poisoned = true;
        free_object(ctx, ob);
        return fail(ROMAP_E_CUDA, "create_object: %s", cudaGetErrorString(e));
    }
    ctx->objs[id] = ob;
    if (id >= ctx->next_id) ctx->next_id = id + 1;
    return ROMAP_OK;
}

romap_status romap_create_object(romap_ctx* ctx, const romap_box* box, const romap_model_config* cfg,
                                 int32_t instance_id, int32_t* out_obj) {
    NVTX_RANGE("romap_create_object");
    CHECK_CTX();
    if (!out_obj) return fail(ROMAP_E_INVALID, "null out_obj");
    int id = ctx->next_id;
    romap_status s = create_impl(ctx, box, cfg, instance_id, id);
    if (s == ROMAP_OK) *out_obj = id;
    return s;
}

romap_status romap_create_object_with_id(romap_ctx* ctx, const romap_box* box, const romap_model_config* cfg,
                                         int32_t instance_id, int32_t obj_id) {
    NVTX_RANGE("romap_create_object_with_id");
    CHECK_CTX();
    return create_impl(ctx, box, cfg, instance_id, obj_id);
}

romap_status romap_destroy_object(romap_ctx* ctx, int32_t obj) {
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    CK(cudaStreamSynchronize(ctx->st));
    ctx->objs.erase(obj);
    free_object(ctx, ob);
    ctx->last_call = LAST_NONE;
    return ROMAP_OK;
}

romap_status romap_set_box(romap_ctx* ctx, int32_t obj, const romap_box* box) {
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    romap_status s = check_box(box);
    if (s) return s;
    // descriptors are rebuilt from these fields by every later call (make_objdev)
    ob->box = *box;
    ob->c = (float)cos((double)box->yaw);   // R8: cos/sin in double, rounded
    ob->s = (float)sin((double)box->yaw);
    ctx->last_call = LAST_NONE;             // debug dumps describe the old box
    return ROMAP_OK;
}

romap_status romap_get_object_info(romap_ctx* ctx, int32_t obj, romap_object_info* out) {
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    if (!out) return fail(ROMAP_E_INVALID, "null out");
    out->instance_id = ob->instance_id;
    out->n_keyframes = (int)ob->kfs.size();
    out->table_entries = ob->cdev.n_entries;
    out->table_params = ob->cdev.n_table;
    out->mlp_params = ob->cdev.n_mlp;
    out->total_area = ob->total_area;
    out->step = ob->step;
    out->rays_per_iter = ob->rays_per_iter;
    int nd = 0;
    for (int l = 0; l < ob->cdev.L; ++l) nd += ob->cdev.dense[l];
    out->n_dense_levels = nd;
    return ROMAP_OK;
}

// pinned staging of at least `bytes` (waits for the previous copy out of it); null
// if pinned memory is unavailable (the caller then stages in pageable memory)
static void* pinned_staging(romap_ctx* ctx, size_t bytes) {
    if (ctx->pin_pending) {
        cudaEventSynchronize(ctx->pin_ev);
        ctx->pin_pending = false;
    }
    if (bytes > ctx->pin_cap) {
        if (ctx->pin) cudaFreeHost(ctx->pin);
        ctx->pin = nullptr;
        ctx->pin_cap = 0;
        const size_t cap = bytes + bytes / 4 + 4096;
        if (cudaMallocHost(&ctx->pin, cap) != cudaSuccess) {
            cudaGetLastError();
            ctx->pin = nullptr;
            return nullptr;
        }
        ctx->pin_cap = cap;
    }
    if (!ctx->pin_ev && cudaEventCreateWithFlags(&ctx->pin_ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return ctx->pin;
}

static void* kf_alloc(romap_ctx* ctx, Object* ob, size_t bytes) {
    bytes = (bytes + 255) & ~(size_t)255;
    if (ob->kf_chunks.empty() || ob->kf_used + bytes > ob->kf_cap) {
        const size_t cap = std::max<size_t>(bytes, (size_t)4 << 20);
        void* p = dalloc(ctx, cap);
        if (!p) return nullptr;
        ob->kf_chunks.push_back(p);
        ob->kf_used = 0;
        ob->kf_cap = cap;
    }
    void* p = static_cast<char*>(ob->kf_chunks.back()) + ob->kf_used;
    ob->kf_used += bytes;
    return p;
}

// append one keyframe to the object from its host-side in-box crop (rgb + class)
// and optional depth crop: device arena copies, descriptor table, area prefix
static romap_status append_keyframe(romap_ctx* ctx, Object* ob, const float T_wc[12], const romap_intrinsics* K,
                                    int x0, int y0, int w, int h, const uchar4* crop, const float* dep,
                                    bool staged_pinned) {
    Keyframe kf;
    for (int k = 0; k < 12; ++k) kf.dev.T[k] = T_wc[k];
    kf.dev.fx = K->fx;
    kf.dev.fy = K->fy;
    kf.dev.cx = K->cx;
    kf.dev.cy = K->cy;
    kf.dev.x0 = x0;
    kf.dev.y0 = y0;
    kf.dev.w = w;
    kf.dev.h = h;
    kf.area = (long long)w * h;
    const size_t npx = (size_t)w * h, crop_bytes = npx * sizeof(uchar4);
    const bool any_depth = dep != nullptr;
    kf.crop_d = (uchar4*)kf_alloc(ctx, ob, crop_bytes);
    if (!kf.crop_d) return fail(ROMAP_E_OOM, "crop allocation failed");
    if (any_depth) {
        kf.depth_d = (float*)kf_alloc(ctx, ob, npx * 4);
        if (!kf.depth_d) return fail(ROMAP_E_OOM, "depth allocation failed");
    }
    kf.dev.crop = kf.crop_d;
    kf.dev.depth = kf.depth_d;
    // descriptor / prefix arrays (re-uploaded whole; grown geometrically)
    if (ob->kfs.size() + 1 > ob->kfs_cap) {
        size_t nc = ob->kfs_cap ? ob->kfs_cap * 2 : 16;
        KfDev* nk = (KfDev*)dalloc(ctx, nc * sizeof(KfDev));
        long long* np = (long long*)dalloc(ctx, nc * sizeof(long long));
        if (!nk || !np) {
            dfree(ctx, nk); dfree(ctx, np);          // (arena space of the crop stays with the object)
            return fail(ROMAP_E_OOM, "keyframe table allocation failed");
        }
        CK(cudaStreamSynchronize(ctx->st));
        dfree(ctx, ob->kfs_d);
        dfree(ctx, ob->prefix_d);
        ob->kfs_d = nk;
        ob->prefix_d = np;
        ob->kfs_cap = nc;
    }
    CK(cudaMemcpyAsync(kf.crop_d, crop, crop_bytes, cudaMemcpyHostToDevice, ctx->st));
    if (any_depth) CK(cudaMemcpyAsync(kf.depth_d, dep, npx * 4, cudaMemcpyHostToDevice, ctx->st));
    if (staged_pinned) {                           // the staging buffer is busy until these copies ran
        CK(cudaEventRecord(ctx->pin_ev, ctx->st));
        ctx->pin_pending = true;
    } else {
        CK(cudaStreamSynchronize(ctx->st));        // pageable source: it may die with the caller's call
    }
    ob->kfs.push_back(kf);
    ob->total_area += kf.area;
    // descriptor table and exclusive area prefix, uploaded whole (the arrays may have been reallocated)
    std::vector<KfDev> descs(ob->kfs.size());
    std::vector<long long> prefix(ob->kfs.size());
    long long acc = 0;
    for (size_t i = 0; i < ob->kfs.size(); ++i) {
        descs[i] = ob->kfs[i].dev;
        prefix[i] = acc;
        acc += ob->kfs[i].area;
    }
    CK(cudaMemcpyAsync(ob->kfs_d, descs.data(), descs.size() * sizeof(KfDev), cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(ob->prefix_d, prefix.data(), prefix.size() * sizeof(long long), cudaMemcpyHostToDevice, ctx->st));
    return ROMAP_OK;
}

romap_status romap_add_observation(romap_ctx* ctx, int32_t obj, const uint8_t* rgb, const uint16_t* mask,
                                   const float T_wc[12], const romap_intrinsics* K,
                                   const romap_depth_sample* depth, int32_t n_depth) {
    NVTX_RANGE("romap_add_observation");
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    if (!rgb || !mask || !T_wc || !K) return fail(ROMAP_E_INVALID, "null input");
    if (K->width < 1 || K->height < 1 || !(K->fx > 0) || !(K->fy > 0))
        return fail(ROMAP_E_INVALID, "bad intrinsics");
    if (n_depth < 0 || (n_depth > 0 && !depth)) return fail(ROMAP_E_INVALID, "bad depth samples");
    for (int k = 0; k < 12; ++k)
        if (!std::isfinite(T_wc[k])) return fail(ROMAP_E_INVALID, "non-finite pose");
    static const bool host_prof = getenv("ROMAP_HOST_PROF") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    const int W = K->width, H = K->height;
    const uint16_t id = (uint16_t)ob->instance_id;
    // tight AABB of mask == id: per row a branch-free (vectorisable) test of 32-pixel
    // blocks finds the first and last hit, rows without the object cost one pass
    int x0 = W, y0 = H, x1 = -1, y1 = -1;
    for (int y = 0; y < H; ++y) {
        const uint16_t* row = mask + (size_t)y * W;
        int first = -1, last = -1;
        for (int b = 0; b < W; b += 32) {
            const int e = std::min(W, b + 32);
            int any = 0;
            for (int x = b; x < e; ++x) any |= row[x] == id;
            if (!any) continue;
            if (first < 0)
                for (int x = b; x < e; ++x)
                    if (row[x] == id) { first = x; break; }
            for (int x = e - 1; x >= b; --x)
                if (row[x] == id) { last = x; break; }
        }
        if (first < 0) continue;
        x0 = std::min(x0, first);
        x1 = std::max(x1, last);
        if (y0 == H) y0 = y;
        y1 = y;
    }
    if (x1 < 0) return fail(ROMAP_E_INVALID, "instance %d not visible in the mask", ob->instance_id);
    const auto t1 = std::chrono::steady_clock::now();
    const int w = x1 - x0 + 1, h = y1 - y0 + 1;
    if (ob->total_area + (long long)w * h >= (1LL << 31)) return fail(ROMAP_E_INVALID, "too many keyframe pixels");
    // crop (+ depth crop) written straight into pinned staging memory
    const size_t npx = (size_t)w * h, crop_bytes = npx * sizeof(uchar4);
    const size_t dep_off = (crop_bytes + 255) & ~(size_t)255;
    std::vector<uint8_t> fallback;
    uint8_t* stage = static_cast<uint8_t*>(pinned_staging(ctx, dep_off + (n_depth > 0 ? npx * 4 : 0)));
    if (!stage) {
        fallback.resize(dep_off + (n_depth > 0 ? npx * 4 : 0));
        stage = fallback.data();
    }
    uchar4* crop = reinterpret_cast<uchar4*>(stage);
    for (int y = 0; y < h; ++y) {
        const uint16_t* mrow = mask + (size_t)(y0 + y) * W + x0;
        const uint8_t* crow = rgb + 3 * ((size_t)(y0 + y) * W + x0);
        uchar4* out = crop + (size_t)y * w;
        for (int x = 0; x < w; ++x) {
            const uint16_t mv = mrow[x];
            const unsigned char cls = mv == id ? CLS_OBJ : (mv == 0 ? CLS_BG : CLS_OCC);
            out[x] = make_uchar4(crow[3 * x], crow[3 * x + 1], crow[3 * x + 2], cls);
        }
    }
    const auto t2 = std::chrono::steady_clock::now();
    float* dep = n_depth > 0 ? reinterpret_cast<float*>(stage + dep_off) : nullptr;
    bool any_depth = false;
    if (n_depth > 0) {
        memset(dep, 0, npx * 4);
        for (int i = 0; i < n_depth; ++i) {
            int px = (int)floorf(depth[i].u), py = (int)floorf(depth[i].v);
            if (px < x0 || px > x1 || py < y0 || py > y1 || !(depth[i].z > 0)) continue;
            size_t li = (size_t)(py - y0) * w + (px - x0);
            if (crop[li].w != CLS_OBJ) continue;
            dep[li] = depth[i].z;
            any_depth = true;
        }
    }
    const auto t3 = std::chrono::steady_clock::now();
    romap_status ak = append_keyframe(ctx, ob, T_wc, K, x0, y0, w, h, crop, any_depth ? dep : nullptr,
                                      stage == ctx->pin);
    if (ak) return ak;
    // (copies from pageable memory return once the source is staged: the host
    // vectors may go; the device sees the data in stream order)
    if (host_prof) {
        const auto t4 = std::chrono::steady_clock::now();
        auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        fprintf(stderr, "[romap host] add_observation: aabb %.3f ms, crop %.3f ms, alloc+desc %.3f ms, copies %.3f ms\n",
                ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4));
    }
    return ROMAP_OK;
}

romap_status romap_set_rays_per_iter(romap_ctx* ctx, int32_t obj, int32_t rays) {
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    if (rays < 1) return fail(ROMAP_E_INVALID, "rays must be >= 1");
    ob->rays_per_iter = rays;
    return ROMAP_OK;
}

// ---------------------------------------------------------------------------
// one batch of objects: validate, lay out rays, upload descriptors
struct Batch {
    std::vector<Object*> obs;
    std::vector<ObjDev> dev;
    CfgDev cfg;
    int total_slots = 0;
    bool mixed = false;
};

static romap_status make_batch(romap_ctx* ctx, const int32_t* objs, int32_t n, bool need_kf, Batch& b) {
    if (!objs || n < 1) return fail(ROMAP_E_INVALID, "empty object list");
    for (int i = 0; i < n; ++i) {
        Object* ob = find(ctx, objs[i]);
        if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", objs[i]);
        for (int j = 0; j < i; ++j)
            if (objs[j] == objs[i]) return fail(ROMAP_E_INVALID, "object %d listed twice", objs[i]);
        if (need_kf && ob->kfs.empty()) return fail(ROMAP_E_STATE, "object %d has no keyframes", objs[i]);
        if (i > 0 && !same_model(ob->cfg, b.obs[0]->cfg))
            return fail(ROMAP_E_CONFIG_MISMATCH, "objects %d and %d differ in model configuration", objs[0], objs[i]);
        b.obs.push_back(ob);
    }
    b.cfg = b.obs[0]->cdev;
    b.mixed = b.obs[0]->cfg.precision == 1;
    const int N = b.cfg.N;
    const int align = N >= ROMAP_TILE ? 1 : ROMAP_TILE / N;   // tiles never straddle objects
    int begin = 0;
    for (auto* ob : b.obs) {
        ObjDev d = make_objdev(ob);
        d.ray_begin = begin;
        d.n_rays = ob->rays_per_iter;
        d.n_slots = (ob->rays_per_iter + align - 1) / align * align;
        begin += d.n_slots;
        b.dev.push_back(d);
    }
    b.total_slots = begin;
    return ROMAP_OK;
}

static romap_status upload_batch(romap_ctx* ctx, Batch& b, bool train_scratch) {
    size_t n = b.dev.size();
    if (!grow(ctx, ctx->objdev_d, ctx->objdev_cap, n)) return fail(ROMAP_E_OOM, "descriptor allocation failed");
    if (n > ctx->stat_cap) {
        cudaStreamSynchronize(ctx->st);
        dfree(ctx, ctx->loss_d);
        dfree(ctx, ctx->hits_d);
        dfree(ctx, ctx->nonfinite_d);
        size_t c = n + 16;
        ctx->loss_d = (double*)dalloc(ctx, c * 4 * sizeof(double));
        ctx->hits_d = (unsigned long long*)dalloc(ctx, c * sizeof(unsigned long long));
        ctx->nonfinite_d = (int*)dalloc(ctx, sizeof(int) * 4);
        if (!ctx->loss_d || !ctx->hits_d || !ctx->nonfinite_d) { ctx->stat_cap = 0; return fail(ROMAP_E_OOM, "stat allocation failed"); }
        ctx->stat_cap = c;
    }
    if (train_scratch) {
        size_t slots = (size_t)b.total_slots;
        size_t S = slots * b.cfg.N;
        if (!grow(ctx, ctx->rays, ctx->rays_cap, slots)) return fail(ROMAP_E_OOM, "ray buffer allocation failed");
        if (!b.mixed) {
            if (!grow(ctx, ctx->samp, ctx->samp_cap, S * 10)) return fail(ROMAP_E_OOM, "sample buffer allocation failed");
            size_t rows = (size_t)b.cfg.LF + 3 * ROMAP_WIDTH + ROMAP_DOUT;
            if (!grow(ctx, ctx->act, ctx->act_cap, S * rows)) return fail(ROMAP_E_OOM, "activation buffer allocation failed");
        } else {
            if (!grow(ctx, ctx->samp, ctx->samp_cap, S * 4)) return fail(ROMAP_E_OOM, "sample buffer allocation failed");
        }
    }
    CK(cudaMemcpyAsync(ctx->objdev_d, b.dev.data(), n * sizeof(ObjDev), cudaMemcpyHostToDevice, ctx->st));
    return ROMAP_OK;
}

// deterministic mode: record / partial buffers of one iteration of batch b (DetBufs)
static romap_status ensure_det(romap_ctx* ctx, const Batch& b) {
    const long long S = (long long)b.total_slots * b.cfg.N;
    const long long n_rec = S * b.cfg.L * 8, tiles = S / ROMAP_TILE;
    if (n_rec >= (1LL << 31)) return fail(ROMAP_E_INVALID, "deterministic mode: batch too large (%lld records)", n_rec);
    const size_t temp = det_sort_temp_bytes(n_rec, (int)b.dev.size());
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t sz[7] = {al(8 * n_rec), al(8 * n_rec), al(4 * tiles * (size_t)b.cfg.n_mlp), al(16 * (size_t)b.total_slots),
                          al(8 * n_rec), al(4 * n_rec), al(4 * n_rec)};
    size_t need = al(temp);
    for (size_t x : sz) need += x;
    if (need > ctx->det_cap || !ctx->det_mem) {
        CK(cudaStreamSynchronize(ctx->st));
        dfree(ctx, ctx->det_mem);
        ctx->det_mem = dalloc(ctx, need);
        ctx->det_cap = ctx->det_mem ? need : 0;
        if (!ctx->det_mem) return fail(ROMAP_E_OOM, "deterministic-mode buffers (%zu bytes)", need);
    }
    char* p = static_cast<char*>(ctx->det_mem);
    ctx->det.key = reinterpret_cast<unsigned long long*>(p); p += sz[0];
    ctx->det.val = reinterpret_cast<float2*>(p); p += sz[1];
    ctx->det.dw = reinterpret_cast<float*>(p); p += sz[2];
    ctx->det.ray_loss = reinterpret_cast<float*>(p); p += sz[3];
    ctx->det_key_sorted = reinterpret_cast<unsigned long long*>(p); p += sz[4];
    ctx->det_iota = reinterpret_cast<unsigned*>(p); p += sz[5];
    ctx->det_perm = reinterpret_cast<unsigned*>(p); p += sz[6];
    ctx->det_temp = p;
    ctx->det_temp_bytes = temp;
    LaunchCtx lc{ctx->st, ctx->num_sms};
    launch_det_iota(lc, ctx->det_iota, n_rec);
    CK(cudaGetLastError());
    return ROMAP_OK;
}

static romap_status run_iterations(romap_ctx* ctx, Batch& b, int n_iters, bool adam, romap_train_stats* out) {
    const int n = (int)b.dev.size();
    LaunchCtx lc{ctx->st, ctx->num_sms};
    CK(cudaMemsetAsync(ctx->hits_d, 0, n * sizeof(unsigned long long), ctx->st));
    CK(cudaMemsetAsync(ctx->nonfinite_d, 0, sizeof(int), ctx->st));
    bool dirty = false;
    for (auto* ob : b.obs) dirty |= ob->grads_dirty;
    if (dirty) STAGE(ST_ZERO_GRADS, launch_zero_grads(lc, b.cfg, ctx->objdev_d, n));
    const size_t S = (size_t)b.total_slots * b.cfg.N;
    // mixed path: rays and sample records of up to K iterations are generated by
    // one k_raygen + k_samples pair (slices k = it % K), ~768 MB of records at most
    // (so multi-object batches -- 45 MB per iteration for cfg2, 180 MB for cfg3 --
    // also replay graph chunks of several iterations)
    int K = 1;
    if (b.mixed) {
        const size_t per_iter = (size_t)b.total_slots * sizeof(RayRec) + S * 5 * sizeof(float);
        const int Kmax = (int)std::max<size_t>(1, std::min<size_t>(16, ((size_t)768 << 20) / per_iter));
        // capacity for Kmax slices on first use, whatever n_iters is: a later call
        // with more iterations never reallocates (cudaFree synchronises the device)
        if (!grow(ctx, ctx->rays, ctx->rays_cap, (size_t)Kmax * b.total_slots))
            return fail(ROMAP_E_OOM, "ray buffer allocation failed");
        if (!grow(ctx, ctx->srec, ctx->srec_cap, (size_t)Kmax * S * 5))
            return fail(ROMAP_E_OOM, "sample record allocation failed");
        K = std::min(Kmax, n_iters);
    }
    ctx->last_ray_base = (size_t)((n_iters - 1) % K) * b.total_slots;
    ctx->last_K = K;
    DetBufs det{};                   // all null: atomics (the default)
    if (ctx->det_on) {
        romap_status ds = ensure_det(ctx, b);
        if (ds) return ds;
        det = ctx->det;
    }
    auto det_reduce = [&]() {
        STAGE(ST_DET, launch_det_reduce(lc, b.cfg, ctx->objdev_d, n, b.total_slots, det, ctx->det_key_sorted,
                                        ctx->det_iota, ctx->det_perm, ctx->det_temp, ctx->det_temp_bytes, ctx->loss_d));
    };
    float* sigma = ctx->samp;
    float* rgb = sigma + S;
    float* dist = rgb + 3 * S;
    float* delta = dist + S;
    float* dsigma = delta + S;
    float* drgb = dsigma + S;
    // host-side cost of enqueueing (ROMAP_HOST_PROF=1: printed to stderr)
    static const bool host_prof = getenv("ROMAP_HOST_PROF") != nullptr;
    double hp[4] = {0, 0, 0, 0};
    auto hnow = [] { return std::chrono::steady_clock::now(); };
    auto hms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
    };
    // one iteration: [loss reset], [L2 flush], (raygen of `kslices` slices when
    // slice k == 0), forward/backward, Adam
    auto enqueue_iter = [&](int it, int k, int kslices, bool reset_loss) {
        auto h0 = hnow();
        if (reset_loss) {
            cudaMemsetAsync(ctx->loss_d, 0, n * 4 * sizeof(double), ctx->st);
            stage_break(ctx);
        }
        if (ctx->flush_bytes) {
            cudaEvent_t e0 = stage_begin(ctx, ST_FLUSH);
            cudaMemsetAsync(ctx->flush_buf, it & 0xff, ctx->flush_bytes, ctx->st);
            stage_end(ctx, ST_FLUSH, e0);
        }
        auto h1 = hnow();
        hp[0] += hms(h0, h1);
        if (b.mixed) {
            float4* srec = reinterpret_cast<float4*>(ctx->srec);
            float* sdelta = ctx->srec + 4 * S * K;
            if (k == 0) {
                STAGE(ST_RAYGEN, launch_raygen_samples(lc, b.cfg, ctx->objdev_d, n, b.total_slots, kslices, ctx->rays,
                                                       srec, sdelta, ctx->hits_d));
                ctx->prof.launches[ST_RAYGEN]++;      // two kernels: k_raygen + k_samples
            }
            if (ctx->det_on) {
                STAGE(ST_FUSED, launch_fused_mixed_det(lc, b.cfg, ctx->objdev_d, ctx->rays + (size_t)k * b.total_slots,
                                                       srec + (size_t)k * S, sdelta + (size_t)k * S, b.total_slots,
                                                       ctx->loss_d, ctx->nonfinite_d, adam ? nullptr : ctx->samp, det));
                det_reduce();
            } else {
                STAGE(ST_FUSED, launch_fused_mixed(lc, b.cfg, ctx->objdev_d, ctx->rays + (size_t)k * b.total_slots,
                                                   srec + (size_t)k * S, sdelta + (size_t)k * S, b.total_slots,
                                                   ctx->loss_d, ctx->nonfinite_d, adam ? nullptr : ctx->samp));
            }
        } else {
            STAGE(ST_RAYGEN, launch_raygen(lc, b.cfg, ctx->objdev_d, n, b.total_slots, ctx->rays, ctx->hits_d));
            STAGE(ST_FWD, launch_fwd_fp32(lc, b.cfg, ctx->objdev_d, ctx->rays, b.total_slots, true, false, sigma, rgb,
                                          dist, delta, ctx->act, (long long)S));
            STAGE(ST_RENDER_LOSS, launch_render_loss(lc, b.cfg, ctx->objdev_d, ctx->rays, b.total_slots, sigma, rgb,
                                                     dist, delta, dsigma, drgb, ctx->loss_d, ctx->nonfinite_d, det));
            STAGE(ST_BWD, launch_bwd_fp32(lc, b.cfg, ctx->objdev_d, ctx->rays, b.total_slots, sigma, rgb, dsigma, drgb,
                                          ctx->act, (long long)S, det));
            if (ctx->det_on) det_reduce();
        }
        auto h2 = hnow();
        hp[1] += hms(h1, h2);
        if (adam) STAGE(ST_ADAM, launch_adam(lc, b.cfg, ctx->objdev_d, n, ctx->nonfinite_d, b.mixed));
        hp[2] += hms(h2, hnow());
    };
    // a9: full chunks of K iterations replay one CUDA graph (mixed training, no
    // per-stage timing events: those need per-launch records); ROMAP_NO_GRAPH=1 off
    static const bool no_graph = getenv("ROMAP_NO_GRAPH") != nullptr;
    int it0 = 0;
    const int n_chunks = (b.mixed && adam && !ctx->prof.on && !no_graph && K >= 2) ? n_iters / K : 0;
    if (n_chunks > 0) {
        auto& g = ctx->tg;
        const void* ptrs[8] = {ctx->objdev_d, ctx->rays, ctx->srec, ctx->loss_d, ctx->hits_d, ctx->nonfinite_d,
                               ctx->flush_buf, ctx->det_on ? ctx->det_mem : nullptr};
        const bool same = g.exec && g.n == n && g.total_slots == b.total_slots && g.K == K && g.det == ctx->det_on &&
                          g.flush_bytes == ctx->flush_bytes && !memcmp(g.ptrs, ptrs, sizeof ptrs) &&
                          !memcmp(&g.cfg, &b.cfg, sizeof(CfgDev));
        if (!same) {
            if (g.exec) cudaGraphExecDestroy(g.exec);
            g.exec = nullptr;
            cudaGraph_t graph = nullptr;
            long long saved[ST_COUNT];                  // capturing is not launching
            memcpy(saved, ctx->prof.launches, sizeof saved);
            cudaError_t ec = cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal);
            const char* what = "cudaStreamBeginCapture";
            if (ec == cudaSuccess) {
                // the loss partials of a call are those of its last iteration: the
                // chunk resets them before its last iteration
                for (int k = 0; k < K; ++k) enqueue_iter(k, k, K, k == K - 1);
                ec = cudaStreamEndCapture(ctx->st, &graph);
                what = "cudaStreamEndCapture";
                if (ec == cudaSuccess && graph) {
                    ec = cudaGraphInstantiate(&g.exec, graph, 0);
                    what = "cudaGraphInstantiate";
                    if (ec != cudaSuccess) g.exec = nullptr;
                }
                if (graph) cudaGraphDestroy(graph);
            }
            memcpy(ctx->prof.launches, saved, sizeof saved);
            if (ec != cudaSuccess || !g.exec) {
                // nothing was launched: report instead of silently running without the graph
                cudaGetLastError();
                return fail(ROMAP_E_CUDA, "a9 graph capture failed at %s: %s (ROMAP_NO_GRAPH=1 runs plain launches)",
                            what, cudaGetErrorString(ec));
            }
            g.cfg = b.cfg;
            g.n = n;
            g.total_slots = b.total_slots;
            g.K = K;
            g.det = ctx->det_on;
            g.flush_bytes = ctx->flush_bytes;
            memcpy(g.ptrs, ptrs, sizeof ptrs);
        }
        if (g.exec) {
            NVTX_RANGE("graph_replay");
            for (int c = 0; c < n_chunks; ++c) CK(cudaGraphLaunch(g.exec, ctx->st));
            ctx->prof.launches[ST_GRAPH] += n_chunks;
            it0 = n_chunks * K;
            ctx->prof.launches[ST_RAYGEN] += 2LL * n_chunks;   // (capture counted one chunk already)
            ctx->prof.launches[ST_FUSED] += (long long)K * n_chunks;
            ctx->prof.launches[ST_ADAM] += (long long)K * n_chunks;
            if (ctx->flush_bytes) ctx->prof.launches[ST_FLUSH] += (long long)K * n_chunks;
            if (ctx->det_on) ctx->prof.launches[ST_DET] += (long long)K * n_chunks;
        }
    }
    for (int it = it0; it < n_iters; ++it) {
        enqueue_iter(it, it % K, std::min(K, n_iters - it), it == n_iters - 1);
        CK(cudaGetLastError());
    }
    if (host_prof)
        fprintf(stderr, "[romap host] %d iters: flush %.3f ms, raygen+fused %.3f ms, adam %.3f ms\n", n_iters, hp[0],
                hp[1], hp[2]);
    std::vector<double> loss(4 * n);
    std::vector<unsigned long long> hits(n);
    int nf = 0;
    CK(cudaMemcpyAsync(loss.data(), ctx->loss_d, 4 * n * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaMemcpyAsync(hits.data(), ctx->hits_d, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaMemcpyAsync(&nf, ctx->nonfinite_d, sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    prof_collect(ctx);
    for (int i = 0; i < n; ++i) {
        Object* ob = b.obs[i];
        if (adam) {
            ob->step += n_iters;
            ob->grads_dirty = false;
        } else {
            ob->grads_dirty = true;
        }
        ob->last_ray_begin = b.dev[i].ray_begin;
        ob->last_n_rays = b.dev[i].n_rays;
        if (out) {
            double B = (double)b.dev[i].n_rays;
            romap_train_stats& s = out[i];
            s.l_rgb = loss[4 * i] / B;
            s.l_rr = loss[4 * i + 1] / B;
            s.l_depth = loss[4 * i + 2] / B;
            s.l_density = loss[4 * i + 3] / B;
            s.l_total = s.l_rgb + s.l_rr + (double)b.cfg.lambda_depth * s.l_depth + (double)b.cfg.lambda_density * s.l_density;
            s.rays = (long long)b.dev[i].n_rays * n_iters;
            s.hit_rays = (long long)hits[i];
            s.samples = (long long)hits[i] * b.cfg.N;
            s.step = ob->step;
        }
    }
    ctx->last_objdev = b.dev;
    ctx->last_cfg = b.cfg;
    ctx->last_call = adam ? LAST_TRAIN : LAST_FWDBWD;
    ctx->last_total_slots = b.total_slots;
    if (nf) return fail(ROMAP_E_NONFINITE, "non-finite %s", (nf & 1) ? "loss" : "gradient");
    return ROMAP_OK;
}

romap_status romap_train_step(romap_ctx* ctx, const int32_t* objs, int32_t n_objs, int32_t n_iters,
                              romap_train_stats* out) {
    NVTX_RANGE("romap_train_step");
    CHECK_CTX();
    if (n_iters < 1) return fail(ROMAP_E_INVALID, "n_iters must be >= 1");
    Batch b;
    romap_status s = make_batch(ctx, objs, n_objs, true, b);
    if (s) return s;
    s = upload_batch(ctx, b, true);
    if (s) return s;
    return run_iterations(ctx, b, n_iters, true, out);
}

romap_status romap_forward_backward(romap_ctx* ctx, const int32_t* objs, int32_t n_objs, romap_train_stats* out) {
    NVTX_RANGE("romap_forward_backward");
    CHECK_CTX();
    Batch b;
    romap_status s = make_batch(ctx, objs, n_objs, true, b);
    if (s) return s;
    s = upload_batch(ctx, b, true);
    if (s) return s;
    return run_iterations(ctx, b, 1, false, out);
}

// ---------------------------------------------------------------------------
// f3 online policy (R25): Eq. 5 keyframe gate, per-object
// iteration budgets and a batching scheduler over them (the B200 replacement of
// the paper's 8-thread pool: objects with budget left train together in one launch)
romap_status romap_offer_observation(romap_ctx* ctx, int32_t obj, const uint8_t* rgb, const uint16_t* mask,
                                     const float T_wc[12], const romap_intrinsics* K,
                                     const romap_depth_sample* depth, int32_t n_depth, float alpha_deg,
                                     int32_t iters_per_update, int32_t* accepted, float* alpha_out) {
    NVTX_RANGE("romap_offer_observation");
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    if (!T_wc || !accepted) return fail(ROMAP_E_INVALID, "null pose / output");
    if (!(alpha_deg >= 0.f) || iters_per_update < 0) return fail(ROMAP_E_INVALID, "bad gate parameters");
    const double c[3] = {T_wc[3], T_wc[7], T_wc[11]};     // camera centre (R8: T_wc camera -> world)
    double alpha = -1.0;
    bool take = !ob->has_gate_ref;
    if (ob->has_gate_ref) {
        double a[3], b2[3], dot = 0, na = 0, nb = 0;
        for (int k = 0; k < 3; ++k) {
            a[k] = ob->gate_ref[k] - (double)ob->box.t[k];
            b2[k] = c[k] - (double)ob->box.t[k];
            dot += a[k] * b2[k];
            na += a[k] * a[k];
            nb += b2[k] * b2[k];
        }
        double cs = dot / (sqrt(na) * sqrt(nb));
        cs = cs > 1.0 ? 1.0 : (cs < -1.0 ? -1.0 : cs);
        alpha = acos(cs) * 180.0 / M_PI;                  // Eq. 5
        take = alpha > (double)alpha_deg;
    }
    if (alpha_out) *alpha_out = (float)alpha;
    *accepted = 0;
    if (!take) return ROMAP_OK;
    romap_status st = romap_add_observation(ctx, obj, rgb, mask, T_wc, K, depth, n_depth);
    if (st) return st;
    ob->has_gate_ref = true;
    for (int k = 0; k < 3; ++k) ob->gate_ref[k] = c[k];
    ob->pending_iters += iters_per_update;
    *accepted = 1;
    return ROMAP_OK;
}

romap_status romap_pending_iters(romap_ctx* ctx, int32_t obj, int64_t* pending) {
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    if (!pending) return fail(ROMAP_E_INVALID, "null output");
    *pending = ob->pending_iters;
    return ROMAP_OK;
}

romap_status romap_train_pending(romap_ctx* ctx, int32_t chunk, int32_t max_iters, int32_t* objs_out,
                                 int32_t* iters_out, int32_t cap, int32_t* n_out) {
    NVTX_RANGE("romap_train_pending");
    CHECK_CTX();
    if (chunk < 1 || max_iters < 0 || cap < 0 || !n_out || (cap > 0 && (!objs_out || !iters_out)))
        return fail(ROMAP_E_INVALID, "bad scheduler arguments");
    std::map<int, long long> ran;
    int done = 0;
    while (done < max_iters) {
        // objects with budget left (ascending id), grouped by model configuration
        std::vector<Object*> live;
        for (auto& kv : ctx->objs)
            if (kv.second->pending_iters > 0 && !kv.second->kfs.empty()) live.push_back(kv.second);
        if (live.empty()) break;
        std::vector<std::vector<Object*>> groups;
        for (Object* ob : live) {
            bool placed = false;
            for (auto& g : groups)
                if (same_model(g[0]->cfg, ob->cfg)) { g.push_back(ob); placed = true; break; }
            if (!placed) groups.push_back({ob});
        }
        long long n = std::min<long long>(chunk, max_iters - done);
        for (Object* ob : live) n = std::min(n, ob->pending_iters);
        for (auto& g : groups) {
            std::vector<int32_t> ids;
            for (Object* ob : g) ids.push_back(ob->id);
            romap_status st = romap_train_step(ctx, ids.data(), (int32_t)ids.size(), (int32_t)n, nullptr);
            if (st) return st;
            for (Object* ob : g) {
                ob->pending_iters -= n;
                ran[ob->id] += n;
            }
        }
        done += (int)n;
    }
    int k = 0;
    for (auto& kv : ran) {
        if (k < cap) {
            objs_out[k] = kv.first;
            iters_out[k] = (int32_t)kv.second;
        }
        ++k;
    }
    *n_out = k;
    return ROMAP_OK;
}

// ---------------------------------------------------------------------------
// f3 asynchronous online trainer (the SLAM side hands frames to
// the training side and is never blocked by it).  romap_async_offer copies the
// frame into a bounded queue and returns at once; the worker thread takes queued
// frames through the Eq. 5 gate and, when the queue is empty, trains pending
// budgets one chunk at a time.
static void async_worker(romap_ctx* ctx) {
    t_async_worker = true;
    AsyncState* as = ctx->async;
    cudaSetDevice(ctx->device);
    for (;;) {
        AsyncFrame fr;
        bool have = false, train = false;
        {
            std::unique_lock<std::mutex> lk(as->mu);
            for (;;) {
                if (!as->queue.empty()) {
                    fr = std::move(as->queue.front());
                    as->queue.pop_front();
                    have = true;
                    break;
                }
                bool pending = false;
                for (auto& kv : ctx->objs) pending |= kv.second->pending_iters > 0 && !kv.second->kfs.empty();
                if (pending && (!as->stop || as->finish)) { train = true; break; }
                if (as->stop) return;
                as->cv.wait_for(lk, std::chrono::milliseconds(2));
            }
        }
        romap_status st = ROMAP_OK;
        if (have) {
            int32_t acc = 0;
            st = romap_offer_observation(ctx, fr.obj, fr.rgb.data(), fr.mask.data(), fr.T, &fr.K, nullptr, 0,
                                         as->alpha_deg, as->iters_per_update, &acc, nullptr);
            std::lock_guard<std::mutex> lk(as->mu);
            as->accepted += acc;
            // a bad frame (unknown object, instance not in the mask, bad intrinsics)
            // is rejected, nothing changed (validation precedes device work): the
            // worker keeps going.  Only CUDA / non-finite / state errors stop it.
            if (st == ROMAP_E_INVALID || st == ROMAP_E_NOT_FOUND) {
                as->rejected++;
                st = ROMAP_OK;
            }
        } else if (train) {
            std::vector<int32_t> ids(ctx->objs.size() + 1), its(ctx->objs.size() + 1);
            int32_t n = 0;
            st = romap_train_pending(ctx, as->chunk, as->chunk, ids.data(), its.data(), (int32_t)ids.size(), &n);
            long long mx = 0;
            for (int i = 0; i < n; ++i) mx = std::max<long long>(mx, its[i]);
            std::lock_guard<std::mutex> lk(as->mu);
            as->iterations += mx;
        }
        if (st) {                                    // record the first error and stop working
            std::lock_guard<std::mutex> lk(as->mu);
            if (!as->error) { as->error = st; as->error_msg = g_err; }
            return;
        }
    }
}

romap_status romap_async_start(romap_ctx* ctx, int32_t chunk, float alpha_deg, int32_t iters_per_update,
                                int32_t queue_cap) {
    CHECK_CTX();
    if (chunk < 1 || !(alpha_deg >= 0.f) || iters_per_update < 0 || queue_cap < 1)
        return fail(ROMAP_E_INVALID, "bad async parameters");
    auto* as = new AsyncState();
    as->chunk = chunk;
    as->alpha_deg = alpha_deg;
    as->iters_per_update = iters_per_update;
    as->cap = queue_cap;
    ctx->async = as;
    as->worker = std::thread(async_worker, ctx);
    return ROMAP_OK;
}

romap_status romap_async_offer(romap_ctx* ctx, int32_t obj, const uint8_t* rgb, const uint16_t* mask,
                               const float T_wc[12], const romap_intrinsics* K, int32_t* queued) {
    if (!ctx || !ctx->async) return fail(ROMAP_E_STATE, "async worker not running");
    {
        // a worker that stopped on an error takes no more frames (the producer must
        // not mistake a dead trainer for backpressure)
        std::lock_guard<std::mutex> lk(ctx->async->mu);
        if (ctx->async->error)
            return fail(ROMAP_E_STATE, "async worker stopped: %s (romap_async_stop returns the error)",
                        ctx->async->error_msg.c_str());
    }
    if (!rgb || !mask || !T_wc || !K || !queued || K->width < 1 || K->height < 1)
        return fail(ROMAP_E_INVALID, "bad frame");
    AsyncState* as = ctx->async;
    const size_t npx = (size_t)K->width * K->height;
    AsyncFrame fr;
    fr.obj = obj;
    fr.rgb.assign(rgb, rgb + 3 * npx);              // the caller's buffers are free on return
    fr.mask.assign(mask, mask + npx);
    memcpy(fr.T, T_wc, sizeof fr.T);
    fr.K = *K;
    std::lock_guard<std::mutex> lk(as->mu);
    as->offered++;
    if ((int)as->queue.size() >= as->cap) {         // never block the producer: drop
        as->dropped++;
        *queued = 0;
        return ROMAP_OK;
    }
    as->queue.push_back(std::move(fr));
    as->max_depth = std::max<long long>(as->max_depth, (long long)as->queue.size());
    as->cv.notify_one();
    *queued = 1;
    return ROMAP_OK;
}

romap_status romap_async_stop(romap_ctx* ctx, int32_t finish_pending, romap_async_stats* out) {
    if (!ctx || !ctx->async) return fail(ROMAP_E_STATE, "async worker not running");
    AsyncState* as = ctx->async;
    {
        std::lock_guard<std::mutex> lk(as->mu);
        as->stop = true;
        as->finish = finish_pending != 0;
        as->cv.notify_one();
    }
    as->worker.join();
    ctx->async = nullptr;
    if (out) {
        out->offered = as->offered;
        out->dropped = as->dropped;
        out->accepted = as->accepted;
        out->iterations = as->iterations;
        out->max_queue_depth = as->max_depth;
        out->rejected = as->rejected;
    }
    romap_status err = as->error;
    std::string msg = as->error_msg;
    delete as;
    if (err) return fail(err, "async worker: %s", msg.c_str());
    return ROMAP_OK;
}

romap_status romap_optimizer_step(romap_ctx* ctx, const int32_t* objs, int32_t n_objs) {
    NVTX_RANGE("romap_optimizer_step");
    CHECK_CTX();
    Batch b;
    romap_status s = make_batch(ctx, objs, n_objs, false, b);
    if (s) return s;
    s = upload_batch(ctx, b, false);
    if (s) return s;
    LaunchCtx lc{ctx->st, ctx->num_sms};
    CK(cudaMemsetAsync(ctx->nonfinite_d, 0, sizeof(int), ctx->st));
    STAGE(ST_ADAM, launch_adam(lc, b.cfg, ctx->objdev_d, (int)b.dev.size(), ctx->nonfinite_d, b.mixed));
    CK(cudaGetLastError());
    int nf = 0;
    CK(cudaMemcpyAsync(&nf, ctx->nonfinite_d, sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    prof_collect(ctx);
    for (auto* ob : b.obs) { ob->step += 1; ob->grads_dirty = false; }
    ctx->last_call = LAST_NONE;
    if (nf) return fail(ROMAP_E_NONFINITE, "non-finite gradient");
    return ROMAP_OK;
}

// ---------------------------------------------------------------------------
// inference
static romap_status render_one(romap_ctx* ctx, Object* ob, const float T_wc[12], const romap_intrinsics* K, int N,
                               float* rgb, float* depth, float* opacity, int flags) {
    const int W = K->width, H = K->height;
    const long long HW = (long long)W * H;
    CfgDev cfg = ob->cdev;
    cfg.N = N;
    KfDev cam;
    memset(&cam, 0, sizeof cam);
    for (int k = 0; k < 12; ++k) cam.T[k] = T_wc[k];
    cam.fx = K->fx; cam.fy = K->fy; cam.cx = K->cx; cam.cy = K->cy;
    cam.w = W; cam.h = H;
    ObjDev od = make_objdev(ob);
    CK(cudaMemcpyAsync(ctx->cam_d, &cam, sizeof cam, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(ctx->single_d, &od, sizeof od, cudaMemcpyHostToDevice, ctx->st));
    if (!grow(ctx, ctx->rays, ctx->rays_cap, (size_t)HW)) return fail(ROMAP_E_OOM, "ray buffer");
    const long long chunk = 1 << 18;
    const long long S = chunk * N;
    if (!grow(ctx, ctx->samp, ctx->samp_cap, (size_t)S * 6)) return fail(ROMAP_E_OOM, "sample buffer");
    bool dev = flags & ROMAP_DEVICE_PTRS;
    float *o_rgb = rgb, *o_dep = depth, *o_opa = opacity;
    if (!dev) {
        if (!grow(ctx, ctx->io_d, ctx->io_cap, (size_t)HW * 5)) return fail(ROMAP_E_OOM, "output buffer");
        o_rgb = rgb ? ctx->io_d : nullptr;
        o_dep = depth ? ctx->io_d + 3 * HW : nullptr;
        o_opa = opacity ? ctx->io_d + 4 * HW : nullptr;
    }
    LaunchCtx lc{ctx->st, ctx->num_sms};
    launch_render_rays(lc, ctx->single_d, ctx->cam_d, W, H, ctx->rays);
    // only rays that hit the box reach the MLP: pack them (k_compact_rays), composite
    // writes each packed ray to its pixel, every other pixel stays 0 (over black)
    if (!grow(ctx, ctx->rays_c, ctx->rays_c_cap, (size_t)HW)) return fail(ROMAP_E_OOM, "ray buffer");
    if (!grow(ctx, ctx->ray_idx, ctx->ray_idx_cap, (size_t)HW + 1)) return fail(ROMAP_E_OOM, "ray index buffer");
    int* d_count = ctx->ray_idx + HW;
    CK(cudaMemsetAsync(d_count, 0, sizeof(int), ctx->st));
    if (o_rgb) CK(cudaMemsetAsync(o_rgb, 0, HW * 3 * 4, ctx->st));
    if (o_dep) CK(cudaMemsetAsync(o_dep, 0, HW * 4, ctx->st));
    if (o_opa) CK(cudaMemsetAsync(o_opa, 0, HW * 4, ctx->st));
    launch_compact_rays(lc, ctx->rays, (int)HW, ctx->rays_c, ctx->ray_idx, d_count);
    int n_act = 0;
    CK(cudaMemcpyAsync(&n_act, d_count, sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    float* sg = ctx->samp;
    float* cl = sg + S;
    float* ds = cl + 3 * S;
    float* dl = ds + S;
    for (long long r0 = 0; r0 < n_act; r0 += chunk) {
        int nr = (int)(n_act - r0 < chunk ? n_act - r0 : chunk);
        // rays of this chunk all belong to slot 0 (ctx->single_d)
        if (ob->cfg.precision == 1)   // mixed objects: fp16 tables / MLP on the tensor cores (k_infer_mixed.cu)
            launch_fwd_mixed(lc, cfg, ctx->single_d, ctx->rays_c + r0, nr, sg, cl, ds, dl);
        else
            launch_fwd_fp32(lc, cfg, ctx->single_d, ctx->rays_c + r0, nr, false, true, sg, cl, ds, dl, nullptr, 0);
        launch_composite(lc, N, ctx->rays_c + r0, nr, sg, cl, ds, dl, o_rgb, o_dep, o_opa, ctx->ray_idx + r0);
    }
    CK(cudaGetLastError());
    if (!dev) {
        if (rgb) CK(cudaMemcpyAsync(rgb, o_rgb, HW * 3 * 4, cudaMemcpyDeviceToHost, ctx->st));
        if (depth) CK(cudaMemcpyAsync(depth, o_dep, HW * 4, cudaMemcpyDeviceToHost, ctx->st));
        if (opacity) CK(cudaMemcpyAsync(opacity, o_opa, HW * 4, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
    }
    return ROMAP_OK;
}

romap_status romap_render(romap_ctx* ctx, int32_t obj, const float T_wc[12], const romap_intrinsics* K,
                          int32_t samples_per_ray, float* rgb, float* depth, float* opacity, int32_t flags) {
    NVTX_RANGE("romap_render");
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    if (!T_wc || !K || K->width < 1 || K->height < 1 || !(K->fx > 0) || !(K->fy > 0))
        return fail(ROMAP_E_INVALID, "bad pose / intrinsics");
    int N = samples_per_ray;
    if (N < 1 || N > 128) return fail(ROMAP_E_INVALID, "samples_per_ray must be in [1,128]");
    return render_one(ctx, ob, T_wc, K, N, rgb, depth, opacity, flags);
}

romap_status romap_render_scene(romap_ctx* ctx, const int32_t* objs, int32_t n, const float T_wc[12],
                                const romap_intrinsics* K, int32_t samples_per_segment, float* rgb, float* depth,
                                float* opacity, int32_t flags) {
    NVTX_RANGE("romap_render_scene");
    CHECK_CTX();
    if (!objs || n < 1) return fail(ROMAP_E_INVALID, "empty object list");
    if (n > 8192) return fail(ROMAP_E_INVALID, "render_scene takes at most 8192 objects");
    if (!T_wc || !K || K->width < 1 || K->height < 1 || !(K->fx > 0) || !(K->fy > 0))
        return fail(ROMAP_E_INVALID, "bad pose / intrinsics");
    const int N = samples_per_segment;
    if (N < 1 || N > 128) return fail(ROMAP_E_INVALID, "samples_per_segment must be in [1,128]");
    std::vector<Object*> obs;
    for (int i = 0; i < n; ++i) {
        Object* ob = find(ctx, objs[i]);
        if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", objs[i]);
        for (int j = 0; j < i; ++j)
            if (objs[j] == objs[i]) return fail(ROMAP_E_INVALID, "object %d listed twice", objs[i]);
        obs.push_back(ob);
    }
    // scene order: objects grouped by model configuration (one forward launch per
    // group), ascending id within a group; the composite orders segments by
    // (t_near, object id) whatever the scene order (R20)
    std::sort(obs.begin(), obs.end(), [](const Object* a, const Object* b) { return a->id < b->id; });
    std::vector<std::vector<Object*>> groups;
    for (Object* ob : obs) {
        bool placed = false;
        for (auto& g : groups)
            if (same_model(g[0]->cfg, ob->cfg)) { g.push_back(ob); placed = true; break; }
        if (!placed) groups.push_back({ob});
    }
    obs.clear();
    for (auto& g : groups) obs.insert(obs.end(), g.begin(), g.end());
    const int W = K->width, H = K->height;
    const long long HW = (long long)W * H;
    LaunchCtx lc{ctx->st, ctx->num_sms};
    // device descriptors of the scene's objects and the camera
    std::vector<ObjDev> od(n);
    for (int i = 0; i < n; ++i) od[i] = make_objdev(obs[i]);
    if (!grow(ctx, ctx->scene_objs_d, ctx->scene_objs_cap, (size_t)n)) return fail(ROMAP_E_OOM, "scene descriptors");
    KfDev cam;
    memset(&cam, 0, sizeof cam);
    for (int k = 0; k < 12; ++k) cam.T[k] = T_wc[k];
    cam.fx = K->fx; cam.fy = K->fy; cam.cx = K->cx; cam.cy = K->cy;
    cam.w = W; cam.h = H;
    CK(cudaMemcpyAsync(ctx->scene_objs_d, od.data(), n * sizeof(ObjDev), cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(ctx->cam_d, &cam, sizeof cam, cudaMemcpyHostToDevice, ctx->st));
    // integers: pix_cnt, pix_off (HW each), obj_cnt, obj_fill, obj_off, obj_len (n each), scan scratch
    const size_t scan_bytes = scene_scan_bytes(HW);
    const size_t ints = 2 * (size_t)HW + 4 * (size_t)n + scan_bytes / 4 + 64;
    if (!grow(ctx, ctx->scene_i, ctx->scene_i_cap, ints)) return fail(ROMAP_E_OOM, "scene index buffers");
    int* pix_cnt = ctx->scene_i;
    int* pix_off = pix_cnt + HW;
    int* obj_cnt = pix_off + HW;
    int* obj_fill = obj_cnt + n;
    int* obj_off = obj_fill + n;
    int* obj_len = obj_off + n;
    void* scan_tmp = reinterpret_cast<void*>(((uintptr_t)(obj_len + n) + 255) & ~(uintptr_t)255);
    CK(cudaMemsetAsync(obj_cnt, 0, 2 * n * sizeof(int), ctx->st));          // obj_cnt, obj_fill
    launch_scene_count(lc, ctx->cam_d, ctx->scene_objs_d, n, W, H, pix_cnt, obj_cnt);
    launch_scene_scan(lc, pix_cnt, pix_off, HW, scan_tmp, scan_bytes);
    std::vector<int> cnt(n);
    CK(cudaMemcpyAsync(cnt.data(), obj_cnt, n * sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));                                       // the one host read per frame
    // object ranges: whole 128-sample tiles (a tile never holds two objects)
    int g = 128;
    for (int a = N, b = 128; b;) { int r = a % b; a = b; b = r; g = a; }
    const int spt = 128 / g;                                                  // segments per tile boundary
    std::vector<int> off(n), len(n);
    long long total = 0, hits = 0;
    for (int i = 0; i < n; ++i) {
        off[i] = (int)total;
        len[i] = (cnt[i] + spt - 1) / spt * spt;
        total += len[i];
        hits += cnt[i];
    }
    if (total >= (1LL << 31)) return fail(ROMAP_E_INVALID, "too many scene segments");
    CK(cudaMemcpyAsync(obj_off, off.data(), n * sizeof(int), cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(obj_len, len.data(), n * sizeof(int), cudaMemcpyHostToDevice, ctx->st));
    const bool dev = flags & ROMAP_DEVICE_PTRS;
    float* o_rgb = rgb;
    float* o_dep = depth;
    float* o_opa = opacity;
    if (!dev) {
        if (!grow(ctx, ctx->io_d, ctx->io_cap, (size_t)HW * 5)) return fail(ROMAP_E_OOM, "output buffer");
        o_rgb = rgb ? ctx->io_d : nullptr;
        o_dep = depth ? ctx->io_d + 3 * HW : nullptr;
        o_opa = opacity ? ctx->io_d + 4 * HW : nullptr;
    }
    if (total > 0) {
        // segment records + per segment t_near, id, C (3), A, D + the pixels' segment lists
        if (!grow(ctx, ctx->rays_c, ctx->rays_c_cap, (size_t)total)) return fail(ROMAP_E_OOM, "segment records");
        if (!grow(ctx, ctx->scene_d, ctx->scene_cap, (size_t)total * 7 + (size_t)hits + 64))
            return fail(ROMAP_E_OOM, "segment buffers");
        float* seg_tn = ctx->scene_d;
        int* seg_id = reinterpret_cast<int*>(seg_tn + total);
        float* segC = seg_tn + 2 * total;
        float* segA = segC + 3 * total;
        float* segD = segA + total;
        int* pix_list = reinterpret_cast<int*>(segD + total);
        launch_scene_emit(lc, ctx->cam_d, ctx->scene_objs_d, n, W, H, pix_off, obj_off, obj_fill, ctx->rays_c, seg_tn,
                          seg_id, pix_list);
        launch_scene_pad(lc, n, obj_cnt, obj_off, obj_len, ctx->rays_c);
        // per model group: the forward over its objects' ranges in chunks of segments
        // (chunk starts are multiples of spt, so every tile stays within one object)
        const long long chunk = ((1 << 18) / spt) * spt;
        const long long S = chunk * N;
        if (!grow(ctx, ctx->samp, ctx->samp_cap, (size_t)S * 6)) return fail(ROMAP_E_OOM, "sample buffer");
        float* sg = ctx->samp;
        float* cl = sg + S;
        float* ds = cl + 3 * S;
        float* dl = ds + S;
        int first = 0;
        for (auto& grp : groups) {
            const int last = first + (int)grp.size();
            CfgDev cfg = grp[0]->cdev;
            cfg.N = N;
            const long long g0 = off[first], g1 = off[last - 1] + len[last - 1];
            for (long long r0 = g0; r0 < g1; r0 += chunk) {
                const int nr = (int)std::min<long long>(chunk, g1 - r0);
                if (grp[0]->cfg.precision == 1)
                    launch_fwd_mixed(lc, cfg, ctx->scene_objs_d, ctx->rays_c + r0, nr, sg, cl, ds, dl);
                else
                    launch_fwd_fp32(lc, cfg, ctx->scene_objs_d, ctx->rays_c + r0, nr, false, true, sg, cl, ds, dl,
                                    nullptr, 0);
                launch_composite(lc, N, ctx->rays_c + r0, nr, sg, cl, ds, dl, segC + 3 * r0, segD + r0, segA + r0,
                                 nullptr);
            }
            first = last;
        }
        launch_scene_final(lc, HW, pix_cnt, pix_off, pix_list, seg_tn, seg_id, segC, segA, segD, o_rgb, o_dep, o_opa);
    } else {
        if (o_rgb) CK(cudaMemsetAsync(o_rgb, 0, HW * 3 * 4, ctx->st));
        if (o_dep) CK(cudaMemsetAsync(o_dep, 0, HW * 4, ctx->st));
        if (o_opa) CK(cudaMemsetAsync(o_opa, 0, HW * 4, ctx->st));
    }
    CK(cudaGetLastError());
    if (!dev) {
        if (rgb) CK(cudaMemcpyAsync(rgb, o_rgb, HW * 3 * 4, cudaMemcpyDeviceToHost, ctx->st));
        if (depth) CK(cudaMemcpyAsync(depth, o_dep, HW * 4, cudaMemcpyDeviceToHost, ctx->st));
        if (opacity) CK(cudaMemcpyAsync(opacity, o_opa, HW * 4, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
    }
    return ROMAP_OK;
}

// ---------------------------------------------------------------------------
// f2 mesh extraction (R26): lattice -> sigma (the object's query kernel) ->
// marching tetrahedra count / scan / emit (k_mesh.cu)
romap_status romap_extract_mesh(romap_ctx* ctx, int32_t obj, int32_t res, float sigma_iso, float* tris,
                                int64_t cap_tris, int64_t* n_tris, int32_t flags) {
    NVTX_RANGE("romap_extract_mesh");
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    // res <= 512: at most 12 triangles per cell, so every count and offset of the
    // int32 scan stays below 2^31 (12 x 512^3 = 1.6e9)
    if (res < 1 || res > 512 || !n_tris || cap_tris < 0 || (cap_tris > 0 && !tris))
        return fail(ROMAP_E_INVALID, "bad mesh arguments");
    const long long n1 = res + 1, nv = n1 * n1 * n1, nc = (long long)res * res * res;
    const size_t scan_bytes = mt_scan_bytes(nc);
    // floats: points 3 nv | sigma nv | counts nc + 1 | offsets nc + 1 | scratch
    const size_t need = (size_t)(4 * nv + 2 * (nc + 1)) + scan_bytes / 4 + 64;
    if (!grow(ctx, ctx->mesh_d, ctx->mesh_cap, need)) return fail(ROMAP_E_OOM, "mesh scratch");
    float* pts = ctx->mesh_d;
    float* sig = pts + 3 * nv;
    int* counts = reinterpret_cast<int*>(sig + nv);
    int* offsets = counts + (nc + 1);
    void* tmp = reinterpret_cast<void*>(((uintptr_t)(offsets + (nc + 1)) + 255) & ~(uintptr_t)255);
    ObjDev od = make_objdev(ob);
    CK(cudaMemcpyAsync(ctx->single_d, &od, sizeof od, cudaMemcpyHostToDevice, ctx->st));
    LaunchCtx lc{ctx->st, ctx->num_sms};
    launch_lattice(lc, ctx->single_d, res, pts);
    if (ob->cfg.precision == 1)
        launch_query_density_mixed(lc, ob->cdev, ctx->single_d, pts, nv, sig);
    else
        launch_query_density(lc, ob->cdev, ctx->single_d, pts, nv, sig);
    if (flags & ROMAP_MESH_CARVE) {
        if (ob->kfs.empty()) return fail(ROMAP_E_STATE, "carving needs keyframes");
        launch_carve(lc, ctx->single_d, pts, nv, sig);
    }
    launch_mt(lc, ctx->single_d, sig, pts, res, sigma_iso, counts, offsets, tmp, scan_bytes, nullptr, false);
    CK(cudaGetLastError());
    int total = 0;
    CK(cudaMemcpyAsync(&total, offsets + nc, sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    *n_tris = total;
    if (total == 0 || total > cap_tris) return ROMAP_OK;
    const bool dev = flags & ROMAP_DEVICE_PTRS;
    float* out = tris;
    if (!dev) {
        if (!grow(ctx, ctx->tris_d, ctx->tris_cap, (size_t)total * 9)) return fail(ROMAP_E_OOM, "triangle buffer");
        out = ctx->tris_d;
    }
    launch_mt(lc, ctx->single_d, sig, pts, res, sigma_iso, counts, offsets, tmp, scan_bytes, out, true);
    CK(cudaGetLastError());
    if (!dev) CK(cudaMemcpyAsync(tris, out, (size_t)total * 36, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return ROMAP_OK;
}

romap_status romap_query_density(romap_ctx* ctx, int32_t obj, const float* xyz, int64_t n, float* sigma,
                                 int32_t flags) {
    NVTX_RANGE("romap_query_density");
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    if (n < 0 || (n > 0 && (!xyz || !sigma))) return fail(ROMAP_E_INVALID, "bad points");
    if (n == 0) return ROMAP_OK;
    ObjDev od = make_objdev(ob);
    CK(cudaMemcpyAsync(ctx->single_d, &od, sizeof od, cudaMemcpyHostToDevice, ctx->st));
    LaunchCtx lc{ctx->st, ctx->num_sms};
    // precision 1 objects: fp16 tables / MLP on the tensor cores (k_infer_mixed.cu)
    auto launch = [&](const float* x, long long m, float* o) {
        if (ob->cfg.precision == 1)
            launch_query_density_mixed(lc, ob->cdev, ctx->single_d, x, m, o);
        else
            launch_query_density(lc, ob->cdev, ctx->single_d, x, m, o);
    };
    if (flags & ROMAP_DEVICE_PTRS) {
        launch(xyz, n, sigma);
        CK(cudaGetLastError());
        return ROMAP_OK;
    }
    const long long chunk = 1 << 22;
    if (!grow(ctx, ctx->io_d, ctx->io_cap, (size_t)chunk * 4)) return fail(ROMAP_E_OOM, "staging buffer");
    for (long long p0 = 0; p0 < n; p0 += chunk) {
        long long m = n - p0 < chunk ? n - p0 : chunk;
        CK(cudaMemcpyAsync(ctx->io_d, xyz + 3 * p0, m * 12, cudaMemcpyHostToDevice, ctx->st));
        launch(ctx->io_d, m, ctx->io_d + 3 * chunk);
        CK(cudaMemcpyAsync(sigma + p0, ctx->io_d + 3 * chunk, m * 4, cudaMemcpyDeviceToHost, ctx->st));
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->st));
    return ROMAP_OK;
}

// ---------------------------------------------------------------------------
// parameter blocks
static romap_status block_ptr(Object* ob, int block, void** p, int64_t* bytes) {
    const CfgDev& c = ob->cdev;
    int64_t nt = (int64_t)c.n_table * 4, nm = (int64_t)c.n_mlp * 4;
    switch (block) {
        case ROMAP_BLOCK_TABLE: *p = ob->p32; *bytes = nt; break;
        case ROMAP_BLOCK_MLP: *p = ob->p32 + c.n_table; *bytes = nm; break;
        case ROMAP_BLOCK_GRAD_TABLE: *p = ob->g32; *bytes = nt; break;
        case ROMAP_BLOCK_GRAD_MLP: *p = ob->g32 + c.n_table; *bytes = nm; break;
        case ROMAP_BLOCK_M_TABLE: *p = ob->m; *bytes = nt; break;
        case ROMAP_BLOCK_M_MLP: *p = ob->m + c.n_table; *bytes = nm; break;
        case ROMAP_BLOCK_V_TABLE: *p = ob->v; *bytes = nt; break;
        case ROMAP_BLOCK_V_MLP: *p = ob->v + c.n_table; *bytes = nm; break;
        case ROMAP_BLOCK_STEP: *p = ob->step_d; *bytes = 8; break;
        default: return fail(ROMAP_E_INVALID, "unknown block %d", block);
    }
    return ROMAP_OK;
}

romap_status romap_block_bytes(romap_ctx* ctx, int32_t obj, int32_t block, int64_t* bytes) {
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    if (!bytes) return fail(ROMAP_E_INVALID, "null bytes");
    void* p;
    return block_ptr(ob, block, &p, bytes);
}

romap_status romap_get_params(romap_ctx* ctx, int32_t obj, int32_t block, void* buf, int64_t bytes) {
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    void* p;
    int64_t nb;
    romap_status s = block_ptr(ob, block, &p, &nb);
    if (s) return s;
    if (!buf || bytes != nb) return fail(ROMAP_E_INVALID, "block %d needs %lld bytes", block, (long long)nb);
    CK(cudaMemcpyAsync(buf, p, nb, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return ROMAP_OK;
}

__global__ void k_to_half(const float* __restrict__ src, __half* __restrict__ dst, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = __float2half_rn(src[i]);
}

romap_status romap_set_params(romap_ctx* ctx, int32_t obj, int32_t block, const void* buf, int64_t bytes) {
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    void* p;
    int64_t nb;
    romap_status s = block_ptr(ob, block, &p, &nb);
    if (s) return s;
    if (!buf || bytes != nb) return fail(ROMAP_E_INVALID, "block %d needs %lld bytes", block, (long long)nb);
    CK(cudaMemcpyAsync(p, buf, nb, cudaMemcpyHostToDevice, ctx->st));
    if (block == ROMAP_BLOCK_TABLE || block == ROMAP_BLOCK_MLP) {
        long long n = nb / 4;
        long long off = (float*)p - ob->p32;
        k_to_half<<<(unsigned)((n + 255) / 256), 256, 0, ctx->st>>>((const float*)p, ob->p16 + off, n);
        CK(cudaGetLastError());
    }
    if (block == ROMAP_BLOCK_STEP) {
        ob->step = *(const long long*)buf;
        CK(upload_bias_corrections(ctx, ob));
    }
    if (block == ROMAP_BLOCK_GRAD_TABLE || block == ROMAP_BLOCK_GRAD_MLP) ob->grads_dirty = false;
    CK(cudaStreamSynchronize(ctx->st));
    return ROMAP_OK;
}

// ---------------------------------------------------------------------------
// debug dumps
static int64_t dump_size(Object* ob, int what) {
    const CfgDev& c = ob->cdev;
    int64_t R = ob->last_n_rays, N = c.N;
    switch (what) {
        case ROMAP_DUMP_RAYS: return R * (int64_t)sizeof(romap_ray_dump);
        case ROMAP_DUMP_SAMPLES: return R * N * 5 * 4;
        case ROMAP_DUMP_HASH_IDX: return R * N * c.L * 8 * 4;
        case ROMAP_DUMP_FEATURES: return R * N * c.LF * 4;
        case ROMAP_DUMP_FIELD: return R * N * 4 * 4;
        case ROMAP_DUMP_RAY_GRADS: return R * N * 4 * 4;
        default: return -1;
    }
}

romap_status romap_dump_bytes(romap_ctx* ctx, int32_t obj, int32_t what, int64_t* bytes) {
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    if (!bytes) return fail(ROMAP_E_INVALID, "null bytes");
    int64_t s = dump_size(ob, what);
    if (s < 0) return fail(ROMAP_E_INVALID, "unknown dump %d", what);
    *bytes = s;
    return ROMAP_OK;
}

romap_status romap_debug_dump(romap_ctx* ctx, int32_t obj, int32_t what, void* buf, int64_t bytes) {
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    int64_t need = dump_size(ob, what);
    if (need < 0) return fail(ROMAP_E_INVALID, "unknown dump %d", what);
    if (ctx->last_call == LAST_NONE || ob->last_ray_begin < 0) return fail(ROMAP_E_STATE, "no iteration to dump");
    if (!buf || bytes != need) return fail(ROMAP_E_INVALID, "dump %d needs %lld bytes", what, (long long)need);
    const int R = ob->last_n_rays, begin = ob->last_ray_begin;
    if (what == ROMAP_DUMP_RAYS) {
        std::vector<RayRec> rr(R);
        CK(cudaMemcpyAsync(rr.data(), ctx->rays + ctx->last_ray_base + begin, R * sizeof(RayRec),
                           cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        romap_ray_dump* o = (romap_ray_dump*)buf;
        for (int i = 0; i < R; ++i) {
            memset(&o[i], 0, sizeof o[i]);
            o[i].kf = rr[i].kf; o[i].px = rr[i].px; o[i].py = rr[i].py;
            o[i].cls = rr[i].flags & RF_CLS_MASK;
            o[i].hit = (rr[i].flags & RF_ACTIVE) ? 1 : 0;
            o[i].has_depth = (rr[i].flags & RF_HAS_DEPTH) ? 1 : 0;
            for (int k = 0; k < 3; ++k) {
                o[i].o[k] = rr[i].o[k]; o[i].d[k] = rr[i].d[k];
                o[i].target[k] = rr[i].tgt[k]; o[i].bg[k] = rr[i].bg[k];
            }
            o[i].t_near = rr[i].tn; o[i].t_far = rr[i].tf; o[i].depth = rr[i].depth;
        }
        return ROMAP_OK;
    }
    if (ob->cfg.precision == 1 && (what == ROMAP_DUMP_SAMPLES || what == ROMAP_DUMP_HASH_IDX)) {
        // the mixed path's own records of the last iteration (train_step or
        // forward_backward) and the fused kernel's corner addressing of them
        const CfgDev& c = ctx->last_cfg;
        const size_t S = (size_t)ctx->last_total_slots * c.N;
        const size_t k = ctx->last_ray_base / (size_t)ctx->last_total_slots;
        const float4* srec = reinterpret_cast<const float4*>(ctx->srec) + k * S + (size_t)begin * c.N;
        const float* sdelta = ctx->srec + 4 * S * ctx->last_K + k * S + (size_t)begin * c.N;
        if (!grow(ctx, ctx->io_d, ctx->io_cap, (size_t)(need / 4 + 1))) return fail(ROMAP_E_OOM, "staging buffer");
        LaunchCtx lc{ctx->st, ctx->num_sms};
        launch_debug_mixed(lc, c, srec, sdelta, (long long)R * c.N, what == ROMAP_DUMP_SAMPLES ? 1 : 2, ctx->io_d);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(buf, ctx->io_d, need, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        return ROMAP_OK;
    }
    if (ctx->last_call != LAST_FWDBWD)
        return fail(ROMAP_E_STATE, "per-sample dumps describe the last forward_backward call");
    const CfgDev& c = ctx->last_cfg;
    const size_t S = (size_t)ctx->last_total_slots * c.N;
    if (what == ROMAP_DUMP_RAY_GRADS) {
        bool mixed = ob->cfg.precision == 1;
        const size_t s0 = (size_t)begin * c.N, n = (size_t)R * c.N;
        std::vector<float> ds(n), dr(3 * n), out(4 * n);
        if (mixed) {
            // fused path stores [dsigma, drgb] interleaved per sample
            CK(cudaMemcpyAsync(out.data(), ctx->samp + 4 * s0, 16 * n, cudaMemcpyDeviceToHost, ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
        } else {
            float* dsigma = ctx->samp + 6 * S;
            float* drgb = dsigma + S;
            CK(cudaMemcpyAsync(ds.data(), dsigma + s0, 4 * n, cudaMemcpyDeviceToHost, ctx->st));
            CK(cudaMemcpyAsync(dr.data(), drgb + 3 * s0, 12 * n, cudaMemcpyDeviceToHost, ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
            for (size_t i = 0; i < n; ++i) {
                out[4 * i] = ds[i];
                for (int k = 0; k < 3; ++k) out[4 * i + 1 + k] = dr[3 * i + k];
            }
        }
        memcpy(buf, out.data(), 16 * n);
        return ROMAP_OK;
    }
    if (!grow(ctx, ctx->io_d, ctx->io_cap, (size_t)(need / 4 + 1))) return fail(ROMAP_E_OOM, "staging buffer");
    // descriptors of the last batch (the step counter has not moved since forward_backward)
    CK(cudaMemcpyAsync(ctx->objdev_d, ctx->last_objdev.data(), ctx->last_objdev.size() * sizeof(ObjDev),
                       cudaMemcpyHostToDevice, ctx->st));
    LaunchCtx lc{ctx->st, ctx->num_sms};
    launch_debug_samples(lc, c, ctx->objdev_d, ctx->rays, begin, R, what, ctx->io_d);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(buf, ctx->io_d, need, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return ROMAP_OK;
}

romap_status romap_profile_enable(romap_ctx* ctx, int32_t on) {
    CHECK_CTX();
    CK(cudaStreamSynchronize(ctx->st));
    prof_collect(ctx);
    ctx->prof.on = on != 0;
    ctx->prof.mask = 0xffffffffu;
    for (int i = 0; i < ST_COUNT; ++i) { ctx->prof.launches[i] = 0; ctx->prof.ms[i] = 0.0; }
    return ROMAP_OK;
}

romap_status romap_profile_stages(romap_ctx* ctx, uint32_t stage_mask) {
    CHECK_CTX();
    CK(cudaStreamSynchronize(ctx->st));
    prof_collect(ctx);
    ctx->prof.on = stage_mask != 0;
    ctx->prof.mask = stage_mask;
    for (int i = 0; i < ST_COUNT; ++i) { ctx->prof.launches[i] = 0; ctx->prof.ms[i] = 0.0; }
    return ROMAP_OK;
}

romap_status romap_profile_read(romap_ctx* ctx, romap_stage_time* out, int32_t max_stages, int32_t* n_stages) {
    CHECK_CTX();
    if (!n_stages || (max_stages > 0 && !out)) return fail(ROMAP_E_INVALID, "null output");
    CK(cudaStreamSynchronize(ctx->st));
    prof_collect(ctx);
    *n_stages = ST_COUNT;
    for (int i = 0; i < ST_COUNT && i < max_stages; ++i) {
        memset(out[i].name, 0, sizeof out[i].name);
        strncpy(out[i].name, kStageNames[i], sizeof out[i].name - 1);
        out[i].launches = ctx->prof.launches[i];
        out[i].ms = ctx->prof.ms[i];
    }
    return ROMAP_OK;
}

romap_status romap_set_l2_flush(romap_ctx* ctx, int64_t bytes) {
    CHECK_CTX();
    if (bytes < 0) return fail(ROMAP_E_INVALID, "bytes must be >= 0");
    CK(cudaStreamSynchronize(ctx->st));
    dfree(ctx, ctx->flush_buf);
    ctx->flush_buf = nullptr;
    ctx->flush_bytes = 0;
    if (bytes > 0) {
        ctx->flush_buf = dalloc(ctx, (size_t)bytes);
        if (!ctx->flush_buf) return fail(ROMAP_E_OOM, "flush buffer");
        ctx->flush_bytes = (size_t)bytes;
    }
    return ROMAP_OK;
}

// ---------------------------------------------------------------------------
// checkpoint / resume of one object (SPEC.md External Interfaces: "header (config),
// then raw little-endian parameter arrays"): the model configuration, box,
// instance / object ids, Adam step, online-policy state, the fp32 parameters,
// Adam moments and gradients, and every keyframe (descriptor + in-box crop +
// optional depth crop), so that training resumes exactly where it stopped.
namespace {
const char kCkMagic[8] = {'R', 'O', 'M', 'A', 'P', 'C', 'K', '1'};
struct CkHeader {
    char magic[8];
    uint32_t version, header_bytes;
    romap_model_config cfg;
    romap_box box;
    int32_t instance_id, obj_id, rays_per_iter, has_gate_ref;
    int64_t step, pending_iters, n_params;
    double gate_ref[3];
    int32_t n_kf, pad;
};
struct CkKeyframe {
    float T[12];
    float fx, fy, cx, cy;
    int32_t x0, y0, w, h, has_depth, pad;
};
struct FileCloser {
    FILE* f;
    ~FileCloser() { if (f) fclose(f); }
};
}  // namespace

romap_status romap_save_object(romap_ctx* ctx, int32_t obj, const char* path) {
    NVTX_RANGE("romap_save_object");
    CHECK_CTX();
    Object* ob = find(ctx, obj);
    if (!ob) return fail(ROMAP_E_NOT_FOUND, "no object %d", obj);
    if (!path) return fail(ROMAP_E_INVALID, "null path");
    const size_t n = (size_t)ob->cdev.n_table + ob->cdev.n_mlp;
    std::vector<float> blk(4 * n);
    CK(cudaMemcpyAsync(blk.data(), ob->p32, n * 4, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaMemcpyAsync(blk.data() + n, ob->m, n * 4, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaMemcpyAsync(blk.data() + 2 * n, ob->v, n * 4, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaMemcpyAsync(blk.data() + 3 * n, ob->g32, n * 4, cudaMemcpyDeviceToHost, ctx->st));
    std::vector<std::vector<uchar4>> crops(ob->kfs.size());
    std::vector<std::vector<float>> deps(ob->kfs.size());
    for (size_t i = 0; i < ob->kfs.size(); ++i) {
        const Keyframe& kf = ob->kfs[i];
        crops[i].resize((size_t)kf.area);
        CK(cudaMemcpyAsync(crops[i].data(), kf.crop_d, (size_t)kf.area * 4, cudaMemcpyDeviceToHost, ctx->st));
        if (kf.depth_d) {
            deps[i].resize((size_t)kf.area);
            CK(cudaMemcpyAsync(deps[i].data(), kf.depth_d, (size_t)kf.area * 4, cudaMemcpyDeviceToHost, ctx->st));
        }
    }
    CK(cudaStreamSynchronize(ctx->st));
    CkHeader hd;
    memset(&hd, 0, sizeof hd);
    memcpy(hd.magic, kCkMagic, 8);
    hd.version = 1;
    hd.header_bytes = sizeof(CkHeader);
    hd.cfg = ob->cfg;
    hd.box = ob->box;
    hd.instance_id = ob->instance_id;
    hd.obj_id = ob->id;
    hd.rays_per_iter = ob->rays_per_iter;
    hd.has_gate_ref = ob->has_gate_ref ? 1 : 0;
    hd.step = ob->step;
    hd.pending_iters = ob->pending_iters;
    hd.n_params = (int64_t)n;
    for (int k = 0; k < 3; ++k) hd.gate_ref[k] = ob->gate_ref[k];
    hd.n_kf = (int32_t)ob->kfs.size();
    FileCloser fc{fopen(path, "wb")};
    if (!fc.f) return fail(ROMAP_E_INVALID, "cannot open %s for writing", path);
    bool ok = fwrite(&hd, sizeof hd, 1, fc.f) == 1 && fwrite(blk.data(), 4, blk.size(), fc.f) == blk.size();
    for (size_t i = 0; ok && i < ob->kfs.size(); ++i) {
        const Keyframe& kf = ob->kfs[i];
        CkKeyframe ck;
        memset(&ck, 0, sizeof ck);
        for (int k = 0; k < 12; ++k) ck.T[k] = kf.dev.T[k];
        ck.fx = kf.dev.fx; ck.fy = kf.dev.fy; ck.cx = kf.dev.cx; ck.cy = kf.dev.cy;
        ck.x0 = kf.dev.x0; ck.y0 = kf.dev.y0; ck.w = kf.dev.w; ck.h = kf.dev.h;
        ck.has_depth = kf.depth_d ? 1 : 0;
        ok = fwrite(&ck, sizeof ck, 1, fc.f) == 1 && fwrite(crops[i].data(), 4, crops[i].size(), fc.f) == crops[i].size();
        if (ok && kf.depth_d) ok = fwrite(deps[i].data(), 4, deps[i].size(), fc.f) == deps[i].size();
    }
    if (!ok) return fail(ROMAP_E_INVALID, "write error on %s", path);
    return ROMAP_OK;
}

romap_status romap_load_object(romap_ctx* ctx, const char* path, int32_t obj_id, int32_t* out_obj) {
    NVTX_RANGE("romap_load_object");
    CHECK_CTX();
    if (!path || !out_obj) return fail(ROMAP_E_INVALID, "null path / output");
    FileCloser fc{fopen(path, "rb")};
    if (!fc.f) return fail(ROMAP_E_INVALID, "cannot open %s", path);
    CkHeader hd;
    if (fread(&hd, sizeof hd, 1, fc.f) != 1 || memcmp(hd.magic, kCkMagic, 8) != 0 || hd.version != 1 ||
        hd.header_bytes != sizeof(CkHeader))
        return fail(ROMAP_E_INVALID, "%s is not a romap checkpoint of this version", path);
    CfgDev cd;
    romap_status st = build_cfg(&hd.cfg, cd);
    if (st) return st;
    if (hd.n_params != (int64_t)cd.n_table + cd.n_mlp || hd.n_kf < 0)
        return fail(ROMAP_E_INVALID, "%s: parameter count does not match its configuration", path);
    const size_t n = (size_t)hd.n_params;
    std::vector<float> blk(4 * n);
    if (fread(blk.data(), 4, blk.size(), fc.f) != blk.size()) return fail(ROMAP_E_INVALID, "%s: truncated", path);
    struct Kf { CkKeyframe ck; std::vector<uchar4> crop; std::vector<float> dep; };
    std::vector<Kf> kfs(hd.n_kf);
    for (auto& k : kfs) {
        if (fread(&k.ck, sizeof k.ck, 1, fc.f) != 1 || k.ck.w < 1 || k.ck.h < 1 || (long long)k.ck.w * k.ck.h > (1LL << 30))
            return fail(ROMAP_E_INVALID, "%s: bad keyframe record", path);
        k.crop.resize((size_t)k.ck.w * k.ck.h);
        if (fread(k.crop.data(), 4, k.crop.size(), fc.f) != k.crop.size()) return fail(ROMAP_E_INVALID, "%s: truncated", path);
        if (k.ck.has_depth) {
            k.dep.resize(k.crop.size());
            if (fread(k.dep.data(), 4, k.dep.size(), fc.f) != k.dep.size()) return fail(ROMAP_E_INVALID, "%s: truncated", path);
        }
    }
    const int32_t id = obj_id >= 0 ? obj_id : hd.obj_id;
    st = create_impl(ctx, &hd.box, &hd.cfg, hd.instance_id, id);
    if (st) return st;
    Object* ob = find(ctx, id);
    CK(cudaMemcpyAsync(ob->p32, blk.data(), n * 4, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(ob->m, blk.data() + n, n * 4, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(ob->v, blk.data() + 2 * n, n * 4, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(ob->g32, blk.data() + 3 * n, n * 4, cudaMemcpyHostToDevice, ctx->st));
    k_to_half<<<(unsigned)((n + 255) / 256), 256, 0, ctx->st>>>(ob->p32, ob->p16, (long long)n);
    CK(cudaGetLastError());
    ob->step = hd.step;
    CK(cudaMemcpyAsync(ob->step_d, &ob->step, 8, cudaMemcpyHostToDevice, ctx->st));
    CK(upload_bias_corrections(ctx, ob));
    ob->rays_per_iter = hd.rays_per_iter;
    ob->has_gate_ref = hd.has_gate_ref != 0;
    for (int k = 0; k < 3; ++k) ob->gate_ref[k] = hd.gate_ref[k];
    ob->pending_iters = hd.pending_iters;
    ob->grads_dirty = false;
    for (auto& k : kfs) {
        romap_intrinsics K{k.ck.fx, k.ck.fy, k.ck.cx, k.ck.cy, 0, 0};
        st = append_keyframe(ctx, ob, k.ck.T, &K, k.ck.x0, k.ck.y0, k.ck.w, k.ck.h, k.crop.data(),
                             k.ck.has_depth ? k.dep.data() : nullptr, false);
        if (st) {
            ctx->objs.erase(id);
            free_object(ctx, ob);
            return st;
        }
    }
    CK(cudaStreamSynchronize(ctx->st));
    *out_obj = id;
    return ROMAP_OK;
}

romap_status romap_set_deterministic(romap_ctx* ctx, int32_t on) {
    CHECK_CTX();
    CK(cudaStreamSynchronize(ctx->st));
    ctx->det_on = on != 0;                       // the cached graph is keyed by the mode
    return ROMAP_OK;
}

romap_status romap_sync(romap_ctx* ctx) {
    CHECK_CTX();
    CK(cudaStreamSynchronize(ctx->st));
    return ROMAP_OK;
}

}  // extern "C"

/* romap.h -- C ABI of the B200-native RO-MAP multi-object NeRF training path.
 *
 * The library (libromap.so, sm_100a) trains many per-object instant-NGP-style
 * NeRFs in parallel, as RO-MAP (arXiv 2304.05735) does for every detected
 * object: "When a new object instance is detected, we initialize a new NeRF
 * model, which consists of a multi-resolution hash encoding and a single-layer
 * MLP" (Sec. V); each model is fed keyframes with instance masks
 * and poses (Sec. V-A "Data"), trained incrementally and in
 * parallel, and queried for density (marching cubes) and
 * rendering.  Citations: PAPER.md:<line> of the paper's LaTeX
 * source; DESIGN.md R<n> = a reading of the paper recorded in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Every call returns romap_status; 0 = ROMAP_OK, < 0 = error.  Nothing aborts.
 *    romap_last_error() returns a thread-local message for the last failure.
 *  - Validation happens before any device work: a call that fails validation
 *    has no side effects.  A CUDA failure poisons the context; every later call
 *    on it returns ROMAP_E_CUDA.
 *  - The caller owns every input and output buffer.  Inputs are consumed before
 *    the call returns (the caller may free them immediately).  Host outputs are
 *    filled before return.  With flags & ROMAP_DEVICE_PTRS the pointers are
 *    device pointers on the context's device, read/written in stream order on the
 *    context's stream (the call returns without synchronizing).
 *  - A context is not thread-safe: one context per device, one process per GPU.
 *  - Geometry: world frame z-up, metres.  Cameras: OpenCV pinhole (x right, y down,
 *    z forward), pixel centres at (px+0.5, py+0.5), T_wc = camera->world 3x4
 *    row-major [R | t] (R8).  Object frame: x_obj = R_z(yaw)^T (x_w - t)
 *    (roll = pitch = 0), box = [-a, a] (half extents a).
 */
#ifndef ROMAP_H
#define ROMAP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)   /* the library is built -fvisibility=hidden */
#endif

typedef int32_t romap_status;
#define ROMAP_OK 0
#define ROMAP_E_INVALID (-1)          /* bad argument / unsupported configuration   */
#define ROMAP_E_NOT_FOUND (-2)        /* unknown object handle                       */
#define ROMAP_E_OOM (-3)              /* device allocation failed                    */
#define ROMAP_E_CUDA (-4)             /* CUDA error; the context is poisoned         */
#define ROMAP_E_NONFINITE (-5)        /* non-finite loss or gradient this call       */
#define ROMAP_E_CONFIG_MISMATCH (-6)  /* objects of one train_step differ in config  */
#define ROMAP_E_STATE (-7)            /* call not valid in this state (no keyframes) */

/* flags */
#define ROMAP_DEVICE_PTRS 1           /* buffers are device pointers (see above)      */
#define ROMAP_MESH_CARVE 2            /* extract_mesh: zero sigma where no keyframe sees the lattice (R26) */

typedef struct romap_ctx romap_ctx;

/* Object box from the object SLAM (Eqs. 1-4): translation t
 * (world, m), yaw about +z (rad), half extents a (m).  Final: the library does not
 * inflate it (R6). */
typedef struct {
    float t[3];
    float yaw;
    float half_extents[3];
} romap_box;

typedef struct {
    float fx, fy, cx, cy;
    int32_t width, height;
} romap_intrinsics;

/* One sparse depth observation: continuous pixel coordinates
 * (u, v) and camera-frame z (m).  It supervises the ray of pixel (floor u, floor v)
 * if that pixel belongs to the object (R17). */
typedef struct {
    float u, v, z;
} romap_depth_sample;

/* Model / training configuration (BASELINE.json configs; PAPER.md:222 constants).
 * Supported on the GPU in this version: feats == 2, 1 <= levels <= 16, width == 64,
 * samples_per_ray a power of two in [1, 128], precision 0 (fp32) or 1 (mixed), and
 *   network 0 (BASELINE): density_out == 16, color_hidden == 2, dir_enc == 16
 *              (SH degree 4), density net LF->64->16 + colour net [16||SH]->64->64->3;
 *   network 1 (the paper's MLP, R24): LF -> 64
 *              (hidden_layers x, 1..3) -> 4 (sigma, rgb), positions only; mixed
 *              path only (precision 1), levels 8 or 16; density_out, color_hidden,
 *              dir_enc are ignored. */
typedef struct {
    int32_t levels;          /* L hash levels                                    */
    int32_t feats;           /* F features per level                             */
    int32_t log2_T;          /* hash table size T = 2^log2_T entries per level   */
    int32_t base_res;        /* N_min                                            */
    double finest_res;       /* N_max (growth b = (N_max/N_min)^(1/(L-1)))       */
    int32_t res_cap;         /* 0 = none, else N_l = min(N_l, res_cap)           */
    int32_t width;           /* hidden width (64)                  */
    int32_t density_out;     /* density-net outputs (16)                         */
    int32_t color_hidden;    /* colour-net hidden layers (2)                     */
    int32_t dir_enc;         /* 16 = SH degree 4 of the view direction           */
    int32_t precision;       /* 0 fp32 SIMT path, 1 fp16 tensor-core MLP (mixed) */
    int32_t density_act;     /* 0 exp(min(raw,15)) (R3), 1 softplus              */
    int32_t samples_per_ray; /* N                             */
    int32_t rays_per_iter;   /* rays drawn per object per iteration */
    float lr, beta1, beta2, eps;          /* Adam (R18)                           */
    float lambda_depth, lambda_density;   /* lambda_1, lambda_2 (Eq. 11)          */
    float loss_scale;        /* mixed path static loss scale (power of two)      */
    int32_t obj_bg;          /* 0: random bg colour composited for R_o too (R14) */
    uint64_t seed;           /* counter-RNG seed (R13)                           */
    int32_t network;         /* 0 BASELINE density + SH colour nets, 1 paper (R24) */
    int32_t hidden_layers;   /* network 1: hidden layers (Table 4: 1..3)         */
} romap_model_config;

/* Per-object statistics of one train_step call.  Loss terms are those of the
 * call's LAST iteration (Eqs. 7-11, each divided by the rays drawn, R16); the
 * counters sum over all iterations of the call; step = Adam step after the call. */
typedef struct {
    double l_total, l_rgb, l_rr, l_depth, l_density;
    int64_t rays, hit_rays, samples;
    int64_t step;
} romap_train_stats;

typedef struct {
    int32_t instance_id;
    int32_t n_keyframes;
    int64_t table_entries;   /* sum over levels of E_l                           */
    int64_t table_params;    /* table_entries * feats                            */
    int64_t mlp_params;      /* sum of out*in over the 5 layers                  */
    int64_t total_area;      /* in-box pixels over all keyframes                 */
    int64_t step;
    int32_t rays_per_iter;
    int32_t n_dense_levels;
} romap_object_info;

/* Parameter blocks for get/set_params (little-endian, row-major):
 *   TABLE*: fp32 [table_entries][feats], levels back to back (level l starts at the
 *           sum over k < l of E_k rounded up to a multiple of 16 entries; dense
 *           index x+(N+1)(y+(N+1)z), hashed as R5; R5)
 *   MLP*:   fp32, out x in, bias-free (R1/R4), concatenated in this order:
 *           network 0: W1[64][L*F], W2[16][64], W3[64][32], W4[64][64], W5[3][64];
 *           network 1 (R24): W1[64][L*F], (hidden_layers - 1) x W[64][64], W_out[4][64]
 *   STEP:   int64 Adam step t */
#define ROMAP_BLOCK_TABLE 0
#define ROMAP_BLOCK_MLP 1
#define ROMAP_BLOCK_GRAD_TABLE 2
#define ROMAP_BLOCK_GRAD_MLP 3
#define ROMAP_BLOCK_M_TABLE 4
#define ROMAP_BLOCK_M_MLP 5
#define ROMAP_BLOCK_V_TABLE 6
#define ROMAP_BLOCK_V_MLP 7
#define ROMAP_BLOCK_STEP 8

/* debug_dump kinds: per ray / per sample data of the object's rays in the LAST
 * iteration run by train_step / forward_backward (recomputed by the same device
 * functions as the training kernels, with the parameters as they are now).
 * Mixed-precision objects (precision 1): SAMPLES are the very records the fused
 * kernel consumed (k_raygen + k_samples output) and HASH_IDX the corner entries
 * the fused kernel's own addressing (hash_fp16.cuh) computes from them; both are
 * available after train_step as well as after forward_backward.
 *   RAYS:     romap_ray_dump[n_rays]
 *   SAMPLES:  float[n_rays][N][5] = dist, delta, u.x, u.y, u.z
 *   HASH_IDX: int32[n_rays][N][L][8] absolute table entry per corner
 *   FEATURES: float[n_rays][N][L*F]
 *   FIELD:    float[n_rays][N][4] = sigma, r, g, b
 *   RAY_GRADS:float[n_rays][N][4] = dL/dsigma, dL/dc (r,g,b) (after forward_backward) */
#define ROMAP_DUMP_RAYS 0
#define ROMAP_DUMP_SAMPLES 1
#define ROMAP_DUMP_HASH_IDX 2
#define ROMAP_DUMP_FEATURES 3
#define ROMAP_DUMP_FIELD 4
#define ROMAP_DUMP_RAY_GRADS 5

typedef struct {
    int32_t kf, px, py, cls;   /* keyframe, pixel, class 0 bg / 1 object / 2 occluder */
    int32_t hit, has_depth, pad0, pad1;
    float o[3], d[3];          /* object-frame ray (R8)                            */
    float t_near, t_far;       /* box segment (R11)                                */
    float target[3], bg[3];    /* pixel colour, random background colour (R14)     */
    float depth;               /* target ray distance (R17)                        */
    float pad2;
} romap_ray_dump;

typedef void* (*romap_alloc_fn)(size_t bytes, void* user);
typedef void (*romap_free_fn)(void* ptr, void* user);

/* Create a context on CUDA device `device`, enqueueing on `cuda_stream` (a
 * cudaStream_t).  NULL: the context creates and owns a stream of its own (a
 * blocking stream, so it stays ordered with work on the legacy default stream;
 * the a9 CUDA graph cannot be captured on the legacy stream itself).  alloc/free: optional device allocator callbacks
 * (e.g. torch's caching allocator, "PyTorch only for device memory",
 * BASELINE north_star): every device buffer of the context and its objects is
 * taken from alloc(bytes, user) and returned with free(ptr, user); both NULL ->
 * cudaMalloc / cudaFree.  E_INVALID if exactly one of them is NULL. */
romap_status romap_ctx_create(int32_t device, void* cuda_stream, romap_alloc_fn alloc, romap_free_fn free_fn,
                              void* user, romap_ctx** out);
romap_status romap_ctx_destroy(romap_ctx* ctx);

/* New NeRF for a newly detected object.  Parameters initialised from
 * cfg->seed and instance_id (tables U(-1e-4,1e-4), weights Glorot-uniform, R19).
 * *out_obj receives the object handle, which is also the object id keying the
 * counter RNG (R13). */
romap_status romap_create_object(romap_ctx* ctx, const romap_box* box, const romap_model_config* cfg,
                                 int32_t instance_id, int32_t* out_obj);
/* Like create_object with an explicit object id (sharded runs keep global ids). */
romap_status romap_create_object_with_id(romap_ctx* ctx, const romap_box* box, const romap_model_config* cfg,
                                         int32_t instance_id, int32_t obj_id);
romap_status romap_destroy_object(romap_ctx* ctx, int32_t obj);
/* replace the object's box (object SLAM refines pose and size
 * over time).  Parameters, Adam state and keyframes are kept:
 * the hash grid and the MLP stay defined over the normalized box coordinates
 * u = (x + a) / (2a) of R6, so every later training iteration, render and
 * density query maps world points through the new box (the learned field
 * moves and stretches with it).  E_INVALID: non-finite centre / yaw or a
 * non-positive half extent (nothing changes); E_NOT_FOUND: no such object. */
romap_status romap_set_box(romap_ctx* ctx, int32_t obj, const romap_box* box);
romap_status romap_get_object_info(romap_ctx* ctx, int32_t obj, romap_object_info* out);

/* Add one keyframe: rgb uint8 [H][W][3], mask uint16 [H][W]
 * (0 = background, instance_id = this object, other = occluder),
 * T_wc float[12].  The detection box is the tight AABB of mask == instance_id
 * (PAPER.md:153); the in-box crop (colour + class byte) and optional sparse depth
 * are copied to the device.  E_INVALID if the object is not visible in the mask. */
romap_status romap_add_observation(romap_ctx* ctx, int32_t obj, const uint8_t* rgb, const uint16_t* mask,
                                   const float T_wc[12], const romap_intrinsics* K,
                                   const romap_depth_sample* depth, int32_t n_depth);

/* Override rays drawn per iteration for one object (BASELINE cfg2 area split). */
romap_status romap_set_rays_per_iter(romap_ctx* ctx, int32_t obj, int32_t rays);

/* Train all listed objects together for n_iters iterations (PAPER.md:222,
 * Table 3): per iteration and object: draw rays_per_iter pixels
 * over its keyframes, sample N points per hit ray, hash-encode, MLP, volume render
 * (Eq. 6), object-tailored loss (Eqs. 7-11), backward, Adam.  All objects must share
 * one model configuration (else E_CONFIG_MISMATCH).  out: nullable, n_objs entries.
 * Returns E_NONFINITE if a loss or gradient was non-finite (parameters are then
 * unspecified). */
romap_status romap_train_step(romap_ctx* ctx, const int32_t* objs, int32_t n_objs, int32_t n_iters,
                              romap_train_stats* out);

/* One iteration without the optimizer step: gradients are left in the GRAD blocks,
 * the Adam step is not advanced (parity / debugging). */
romap_status romap_forward_backward(romap_ctx* ctx, const int32_t* objs, int32_t n_objs, romap_train_stats* out);

/* Adam step on the gradients currently in the GRAD blocks (t = step + 1; tables
 * sparse: entries with a zero gradient are untouched, R18); zeroes the gradients. */
romap_status romap_optimizer_step(romap_ctx* ctx, const int32_t* objs, int32_t n_objs);

/* Render one object from pose T_wc (R12 midpoint samples, composited over black):
 * rgb float [H][W][3], depth float [H][W] (ray distance), opacity float [H][W]
 * (H = K->height, W = K->width); any output may be NULL.  E_INVALID: null pose /
 * intrinsics, non-positive size or focal length, samples_per_ray outside [1, 128];
 * E_NOT_FOUND: no such object. */
romap_status romap_render(romap_ctx* ctx, int32_t obj, const float T_wc[12], const romap_intrinsics* K,
                          int32_t samples_per_ray, float* rgb, float* depth, float* opacity, int32_t flags);

/* Online policy (R25).
 * offer_observation: Eq. 5 keyframe gate.  The frame becomes a training keyframe
 * (as romap_add_observation) iff the object has none yet or the angle at the box
 * centre between the camera centre of the LAST ACCEPTED keyframe and this frame's
 * exceeds alpha_deg (25).  An accepted frame adds iters_per_update
 * (300) iterations to the object's pending budget.  *accepted = 1/0;
 * *alpha_out (nullable) = the angle in degrees, -1 for the first frame.  Errors as
 * romap_add_observation; a rejected frame changes nothing. */
romap_status romap_offer_observation(romap_ctx* ctx, int32_t obj, const uint8_t* rgb, const uint16_t* mask,
                                     const float T_wc[12], const romap_intrinsics* K,
                                     const romap_depth_sample* depth, int32_t n_depth, float alpha_deg,
                                     int32_t iters_per_update, int32_t* accepted, float* alpha_out);
/* Pending training budget (iterations) of one object. */
romap_status romap_pending_iters(romap_ctx* ctx, int32_t obj, int64_t* pending);
/* Scheduler: while some object has budget left and fewer than max_iters iterations
 * ran in this call, train every object with budget left (objects of one model
 * configuration in ONE batched train_step) for n = min(chunk, smallest pending)
 * iterations; an object whose budget is spent stops training.
 * Writes up to cap (object id, iterations run) pairs, *n_out = pairs available. */
romap_status romap_train_pending(romap_ctx* ctx, int32_t chunk, int32_t max_iters, int32_t* objs_out,
                                 int32_t* iters_out, int32_t cap, int32_t* n_out);

/* Asynchronous online trainer (f3: frames flow one way from the
 * SLAM side and never block it).  async_start spawns a worker thread that owns the
 * context: it takes queued frames through offer_observation (alpha_deg,
 * iters_per_update) and, when the queue is empty, trains pending budgets one chunk
 * at a time (train_pending).  async_offer copies the frame (rgb H*W*3, mask H*W,
 * pose, intrinsics) into a queue of queue_cap frames and returns at once: *queued =
 * 1, or 0 when the queue is full (the frame is dropped, the producer never waits).
 * While the worker runs every other call on the context returns E_STATE.
 * A queued frame that fails validation (unknown object, instance not visible in
 * the mask: E_NOT_FOUND / E_INVALID of romap_offer_observation) is counted as
 * rejected and the worker goes on; any other error (CUDA, non-finite) stops the
 * worker, after which async_offer returns E_STATE.  async_stop joins the worker
 * after draining the queue, and first trains every pending budget when
 * finish_pending; it returns the worker's first error, if any. */
typedef struct {
    int64_t offered, dropped, accepted, iterations, max_queue_depth, rejected;
} romap_async_stats;
romap_status romap_async_start(romap_ctx* ctx, int32_t chunk, float alpha_deg, int32_t iters_per_update,
                               int32_t queue_cap);
romap_status romap_async_offer(romap_ctx* ctx, int32_t obj, const uint8_t* rgb, const uint16_t* mask,
                               const float T_wc[12], const romap_intrinsics* K, int32_t* queued);
romap_status romap_async_stop(romap_ctx* ctx, int32_t finish_pending, romap_async_stats* out);

/* Render several objects (R20): per ray, intersect every box, sort the hit segments
 * by t_near (tie: smaller object id), composite each segment's (C, A, D) front to
 * back over black.  Outputs as romap_render.  The objects may differ in model
 * configuration (one forward launch per configuration).  E_INVALID: empty or
 * duplicate object list, more than 8192 objects, bad pose / intrinsics,
 * samples_per_segment outside [1, 128]; E_NOT_FOUND: an unknown object. */
romap_status romap_render_scene(romap_ctx* ctx, const int32_t* objs, int32_t n, const float T_wc[12],
                                const romap_intrinsics* K, int32_t samples_per_segment, float* rgb, float* depth,
                                float* opacity, int32_t flags);

/* Density at object-frame points (m) for marching cubes:
 * xyz float [n][3] -> sigma float [n] (1/m); 0 outside the box (R21); n = 0 is a
 * no-op.  Host buffers, or device buffers with ROMAP_DEVICE_PTRS.  E_INVALID: n < 0
 * or a null buffer with n > 0; E_NOT_FOUND: no such object. */
romap_status romap_query_density(romap_ctx* ctx, int32_t obj, const float* xyz, int64_t n, float* sigma,
                                 int32_t flags);

/* Isosurface of one object's density (R26; the paper runs
 * marching cubes on a 64^3 lattice): the (res+1)^3 vertex lattice
 * over the box [-a, a], sigma by the object's query path, marching tetrahedra at
 * sigma_iso (1/m).  Writes the triangles (9 floats each: 3 vertices x (x, y, z),
 * WORLD frame, m) in the deterministic cell / tetrahedron order to tris (host, or
 * device with ROMAP_DEVICE_PTRS) when they fit in cap_tris; *n_tris = triangle
 * count either way (call with cap_tris = 0 to size the buffer).  1 <= res <= 512
 * (E_INVALID otherwise: 12 triangles per cell at most keep the int32 offsets exact).
 * flags & ROMAP_MESH_CARVE: before extraction, sigma := 0 at vertices that lie in
 * front of no keyframe camera inside its detection box (R26; E_STATE without
 * keyframes). */
romap_status romap_extract_mesh(romap_ctx* ctx, int32_t obj, int32_t res, float sigma_iso, float* tris,
                                int64_t cap_tris, int64_t* n_tris, int32_t flags);

/* Copy a parameter block (see ROMAP_BLOCK_*) to / from a host buffer of exactly the
 * block's size in bytes. */
romap_status romap_get_params(romap_ctx* ctx, int32_t obj, int32_t block, void* buf, int64_t bytes);
romap_status romap_set_params(romap_ctx* ctx, int32_t obj, int32_t block, const void* buf, int64_t bytes);
/* Size in bytes of a block or dump (bytes == required size). */
romap_status romap_block_bytes(romap_ctx* ctx, int32_t obj, int32_t block, int64_t* bytes);
romap_status romap_dump_bytes(romap_ctx* ctx, int32_t obj, int32_t what, int64_t* bytes);
romap_status romap_debug_dump(romap_ctx* ctx, int32_t obj, int32_t what, void* buf, int64_t bytes);

/* Tracing: every training / inference entry point (and each graph-replay batch
 * inside train_step) is an NVTX range named after the call ("romap_train_step",
 * "graph_replay", "romap_render_scene", ...), so a profiler can select its kernels,
 * e.g. `ncu --nvtx --nvtx-include "romap_train_step/"`.  No cost without a tool.
 *
 * Per-stage device timing of train_step / forward_backward / optimizer_step:
 * when enabled, the library brackets every kernel it launches with CUDA events
 * on the context's stream and accumulates the elapsed time per stage.  Launch
 * counters are always kept.  enable(ctx, 1) also resets the counters. */
typedef struct {
    char name[24];
    int64_t launches;
    double ms;
} romap_stage_time;
romap_status romap_profile_enable(romap_ctx* ctx, int32_t on);
/* Like enable(ctx, 1) but only the stages whose bit is set in stage_mask (bit i
 * = stage i in romap_profile_read order) are bracketed with events; the others
 * only count launches.  Fewer events per iteration = less timing overhead in the
 * measured region.  0 disables. */
romap_status romap_profile_stages(romap_ctx* ctx, uint32_t stage_mask);
romap_status romap_profile_read(romap_ctx* ctx, romap_stage_time* out, int32_t max_stages, int32_t* n_stages);

/* Measurement hook (bench.py timing rules): when bytes > 0, train_step writes a
 * scratch buffer of that size before every iteration so that no iteration starts
 * with the previous one's working set in L2; the writes are timed as stage
 * "l2_flush" and are not part of any other stage. 0 disables (default). */
romap_status romap_set_l2_flush(romap_ctx* ctx, int64_t bytes);

/* Tensor-core self test (GPU tests only): with the operand layouts of the mixed
 * path, computes on device 0 out1[128x64] = X[128x32] W[64x32]^T,
 * out2[128x32] = Dl[128x64] W, out3[64x32] = Dl^T X from fp16 copies of the
 * inputs (host pointers, row-major fp32). */
romap_status romap_selftest_mma(const float* X, const float* W, const float* Dl, float* out1, float* out2,
                                float* out3);

/* Checkpoint / resume of one object (SPEC.md "Model checkpoint
 * file: header (config), then raw little-endian parameter arrays"): save_object
 * writes the model configuration, box, instance and object id, Adam step,
 * online-policy state (gate reference, pending budget), the fp32 parameters, Adam
 * moments and gradients, and every keyframe (descriptor, in-box crop, optional
 * depth crop) to `path` (host byte order; one file per object).  load_object
 * recreates the object from such a file under obj_id (or the saved id when
 * obj_id < 0), *out_obj = its id: continuing to train it is identical to
 * continuing the saved one (bitwise in the deterministic mode).  E_INVALID: the
 * file cannot be written / read, or is not a checkpoint of this version (nothing
 * created); E_INVALID also if the id exists. */
romap_status romap_save_object(romap_ctx* ctx, int32_t obj, const char* path);
romap_status romap_load_object(romap_ctx* ctx, const char* path, int32_t obj_id, int32_t* out_obj);

/* Deterministic-reduction mode (tests; SURVEY.md 8(c) "bitwise in a
 * deterministic-reduction debug mode").  on = 1: every
 * later train_step / forward_backward writes each table-gradient, weight-gradient
 * and loss contribution to a record instead of an fp32 atomic, and fixed-order
 * reductions (k_det.cu) apply them: within an object in sample / tile / ray
 * order.  Results are then bitwise reproducible run to run, equal between graph
 * replays and plain launches, and equal for an object trained in a batch or
 * alone.  Costs ~16 B of records per (sample, level, corner) and a radix sort per
 * iteration (not for timing).  on = 0 (default): fp32 atomics. */
romap_status romap_set_deterministic(romap_ctx* ctx, int32_t on);

/* Wait for all work on the context's stream. */
romap_status romap_sync(romap_ctx* ctx);
/* Thread-local message of the last failing call (valid until the next call). */
const char* romap_last_error(void);
/* Library version string. */
const char* romap_version(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* ROMAP_H */

"""Thin Python binding of libromap.so (include/romap.h): argument marshalling only.

Every step of the training / inference path runs in the CUDA kernels behind the
C ABI; this module converts numpy arrays / torch tensors to pointers and status
codes to exceptions.  There is no CPU fallback: if libromap.so is missing the
import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ROMAP_LIB") or os.path.join(_HERE, "libromap.so")   # ROMAP_LIB: experiment builds

OK = 0
E_INVALID, E_NOT_FOUND, E_OOM, E_CUDA, E_NONFINITE, E_CONFIG_MISMATCH, E_STATE = -1, -2, -3, -4, -5, -6, -7
DEVICE_PTRS = 1
MESH_CARVE = 2
BLOCK_TABLE, BLOCK_MLP, BLOCK_GRAD_TABLE, BLOCK_GRAD_MLP = 0, 1, 2, 3
BLOCK_M_TABLE, BLOCK_M_MLP, BLOCK_V_TABLE, BLOCK_V_MLP, BLOCK_STEP = 4, 5, 6, 7, 8
DUMP_RAYS, DUMP_SAMPLES, DUMP_HASH_IDX, DUMP_FEATURES, DUMP_FIELD, DUMP_RAY_GRADS = 0, 1, 2, 3, 4, 5


class RomapError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"romap status {status}: {msg}")
        self.status = status


class Box(C.Structure):
    _fields_ = [("t", C.c_float * 3), ("yaw", C.c_float), ("half_extents", C.c_float * 3)]


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32)]


class DepthSample(C.Structure):
    _fields_ = [("u", C.c_float), ("v", C.c_float), ("z", C.c_float)]


class ModelConfig(C.Structure):
    _fields_ = [("levels", C.c_int32), ("feats", C.c_int32), ("log2_T", C.c_int32), ("base_res", C.c_int32),
                ("finest_res", C.c_double), ("res_cap", C.c_int32), ("width", C.c_int32),
                ("density_out", C.c_int32), ("color_hidden", C.c_int32), ("dir_enc", C.c_int32),
                ("precision", C.c_int32), ("density_act", C.c_int32), ("samples_per_ray", C.c_int32),
                ("rays_per_iter", C.c_int32), ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float), ("lambda_depth", C.c_float), ("lambda_density", C.c_float),
                ("loss_scale", C.c_float), ("obj_bg", C.c_int32), ("seed", C.c_uint64), ("network", C.c_int32),
                ("hidden_layers", C.c_int32)]


class TrainStats(C.Structure):
    _fields_ = [("l_total", C.c_double), ("l_rgb", C.c_double), ("l_rr", C.c_double), ("l_depth", C.c_double),
                ("l_density", C.c_double), ("rays", C.c_int64), ("hit_rays", C.c_int64), ("samples", C.c_int64),
                ("step", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ObjectInfo(C.Structure):
    _fields_ = [("instance_id", C.c_int32), ("n_keyframes", C.c_int32), ("table_entries", C.c_int64),
                ("table_params", C.c_int64), ("mlp_params", C.c_int64), ("total_area", C.c_int64),
                ("step", C.c_int64), ("rays_per_iter", C.c_int32), ("n_dense_levels", C.c_int32)]


class StageTime(C.Structure):
    _fields_ = [("name", C.c_char * 24), ("launches", C.c_int64), ("ms", C.c_double)]


RAY_DUMP_DTYPE = np.dtype([("kf", "<i4"), ("px", "<i4"), ("py", "<i4"), ("cls", "<i4"), ("hit", "<i4"),
                           ("has_depth", "<i4"), ("pad0", "<i4"), ("pad1", "<i4"), ("o", "<f4", 3), ("d", "<f4", 3),
                           ("t_near", "<f4"), ("t_far", "<f4"), ("target", "<f4", 3), ("bg", "<f4", 3),
                           ("depth", "<f4"), ("pad2", "<f4")])

_P = C.c_void_p
_I = C.c_int32
_SIGS = {
    "romap_ctx_create": [_I, _P, _P, _P, _P, C.POINTER(_P)],
    "romap_ctx_destroy": [_P],
    "romap_create_object": [_P, C.POINTER(Box), C.POINTER(ModelConfig), _I, C.POINTER(_I)],
    "romap_create_object_with_id": [_P, C.POINTER(Box), C.POINTER(ModelConfig), _I, _I],
    "romap_destroy_object": [_P, _I],
    "romap_set_box": [_P, _I, _P],
    "romap_get_object_info": [_P, _I, C.POINTER(ObjectInfo)],
    "romap_add_observation": [_P, _I, _P, _P, _P, C.POINTER(Intrinsics), _P, _I],
    "romap_set_rays_per_iter": [_P, _I, _I],
    "romap_train_step": [_P, _P, _I, _I, _P],
    "romap_forward_backward": [_P, _P, _I, _P],
    "romap_optimizer_step": [_P, _P, _I],
    "romap_render": [_P, _I, _P, C.POINTER(Intrinsics), _I, _P, _P, _P, _I],
    "romap_render_scene": [_P, _P, _I, _P, C.POINTER(Intrinsics), _I, _P, _P, _P, _I],
    "romap_query_density": [_P, _I, _P, C.c_int64, _P, _I],
    "romap_get_params": [_P, _I, _I, _P, C.c_int64],
    "romap_set_params": [_P, _I, _I, _P, C.c_int64],
    "romap_block_bytes": [_P, _I, _I, C.POINTER(C.c_int64)],
    "romap_dump_bytes": [_P, _I, _I, C.POINTER(C.c_int64)],
    "romap_debug_dump": [_P, _I, _I, _P, C.c_int64],
    "romap_sync": [_P],
    "romap_profile_enable": [_P, _I],
    "romap_profile_read": [_P, _P, _I, C.POINTER(_I)],
    "romap_profile_stages": [_P, C.c_uint32],
    "romap_async_start": [_P, _I, C.c_float, _I, _I],
    "romap_async_offer": [_P, _I, _P, _P, _P, C.POINTER(Intrinsics), C.POINTER(_I)],
    "romap_async_stop": [_P, _I, _P],
    "romap_extract_mesh": [_P, _I, _I, C.c_float, _P, C.c_int64, C.POINTER(C.c_int64), _I],
    "romap_offer_observation": [_P, _I, _P, _P, _P, C.POINTER(Intrinsics), _P, _I, C.c_float, _I, C.POINTER(_I),
                                C.POINTER(C.c_float)],
    "romap_pending_iters": [_P, _I, C.POINTER(C.c_int64)],
    "romap_train_pending": [_P, _I, _I, _P, _P, _I, C.POINTER(_I)],
    "romap_set_l2_flush": [_P, C.c_int64],
    "romap_set_deterministic": [_P, _I],
    "romap_save_object": [_P, _I, C.c_char_p],
    "romap_load_object": [_P, C.c_char_p, _I, C.POINTER(_I)],
}

# device allocator callbacks of romap_ctx_create (romap.h): void* alloc(size_t, void*), void free(void*, void*)
ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


def load_library(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(f"libromap.so not built ({path}); run __graft_entry__.build()")
    lib = C.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int32
    lib.romap_last_error.restype = C.c_char_p
    lib.romap_last_error.argtypes = []
    lib.romap_version.restype = C.c_char_p
    lib.romap_version.argtypes = []
    return lib


_lib = load_library()


def _check(status):
    if status != OK:
        raise RomapError(status, _lib.romap_last_error().decode())


def selftest_mma(X, W, Dl):
    """tcgen05 layout self test (see romap.h): returns X W^T, Dl W, Dl^T X."""
    X = np.ascontiguousarray(X, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    Dl = np.ascontiguousarray(Dl, np.float32)
    o1 = np.zeros((128, 64), np.float32)
    o2 = np.zeros((128, 32), np.float32)
    o3 = np.zeros((64, 32), np.float32)
    _lib.romap_selftest_mma.argtypes = [_P] * 6
    _lib.romap_selftest_mma.restype = C.c_int32
    _check(_lib.romap_selftest_mma(_ptr(X), _ptr(W), _ptr(Dl), _ptr(o1), _ptr(o2), _ptr(o3)))
    return o1, o2, o3


def version() -> str:
    return _lib.romap_version().decode()


def model_config(**kw) -> ModelConfig:
    """BASELINE cfg0 defaults; keyword overrides (cfg1: levels=16, log2_T=16,
    finest_res=512, res_cap=0, samples_per_ray=64, rays_per_iter=4096, precision=1)."""
    d = dict(levels=8, feats=2, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, width=64, density_out=16,
             color_hidden=2, dir_enc=16, precision=0, density_act=0, samples_per_ray=32, rays_per_iter=256, lr=1e-2,
             beta1=0.9, beta2=0.99, eps=1e-15, lambda_depth=0.5, lambda_density=0.01, loss_scale=128.0, obj_bg=0,
             seed=0, network=0, hidden_layers=1)
    d.update(kw)
    c = ModelConfig()
    for k, v in d.items():
        setattr(c, k, v)
    return c


def _ptr(a):
    """Pointer of a C-contiguous numpy array or torch tensor."""
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _ids(objs):
    arr = np.ascontiguousarray(np.asarray(objs, dtype=np.int32).reshape(-1))
    return arr, len(arr)


def _torch_allocator(device):
    """romap_ctx_create callbacks backed by torch's caching allocator (north_star:
    "PyTorch only for device memory").  The library frees a buffer only after
    synchronizing its stream, so a block handed back may be reused on any stream."""
    import torch

    def _alloc(nbytes, _user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device)
        except Exception:
            return None

    def _free(ptr, _user):
        try:
            torch.cuda.caching_allocator_delete(ptr)
        except Exception:
            pass
    return ALLOC_FN(_alloc), FREE_FN(_free)


class Context:
    """One context per device (romap_ctx).  Enqueues on torch's current stream when
    that is a side stream; on the default stream the library uses a (blocking)
    stream of its own, so the a9 CUDA graph can be captured.  Device memory comes
    from torch's caching allocator (torch_alloc=True) or cudaMalloc."""

    def __init__(self, device: int = 0, stream=None, torch_alloc: bool = True):
        self._cb = (None, None)
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    torch.cuda.set_device(device)
                    stream = torch.cuda.current_stream(device).cuda_stream
                    if torch_alloc:
                        self._cb = _torch_allocator(device)
            except Exception:
                stream = None
        self._h = C.c_void_p()
        a, f = self._cb
        _check(_lib.romap_ctx_create(device, C.c_void_p(stream or 0), C.cast(a, C.c_void_p) if a else None,
                                     C.cast(f, C.c_void_p) if f else None, None, C.byref(self._h)))
        self.device = device

    def close(self):
        if self._h:
            _check(_lib.romap_ctx_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            if sys.is_finalizing():   # torch's allocator (the free callbacks) may be gone already
                return
        except Exception:
            return
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------- objects
    def create_object(self, t, yaw, half_extents, cfg: ModelConfig, instance_id: int, obj_id: int | None = None) -> int:
        b = Box((C.c_float * 3)(*[float(v) for v in t]), float(yaw), (C.c_float * 3)(*[float(v) for v in half_extents]))
        if obj_id is None:
            out = C.c_int32()
            _check(_lib.romap_create_object(self._h, C.byref(b), C.byref(cfg), int(instance_id), C.byref(out)))
            return out.value
        _check(_lib.romap_create_object_with_id(self._h, C.byref(b), C.byref(cfg), int(instance_id), int(obj_id)))
        return int(obj_id)

    def destroy_object(self, obj: int):
        _check(_lib.romap_destroy_object(self._h, obj))

    def set_box(self, obj: int, t, yaw: float, half_extents):
        """f3: replace the object's box; parameters stay in normalized box coordinates."""
        b = Box((C.c_float * 3)(*[float(v) for v in t]), float(yaw), (C.c_float * 3)(*[float(v) for v in half_extents]))
        _check(_lib.romap_set_box(self._h, obj, C.byref(b)))

    def object_info(self, obj: int) -> dict:
        info = ObjectInfo()
        _check(_lib.romap_get_object_info(self._h, obj, C.byref(info)))
        return {k: getattr(info, k) for k, _ in info._fields_}

    def add_observation(self, obj: int, rgb, mask, T_wc, K, depth=None):
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        mask = np.ascontiguousarray(mask, dtype=np.uint16)
        T = np.ascontiguousarray(np.asarray(T_wc, dtype=np.float32).reshape(12))
        H, W = mask.shape
        intr = Intrinsics(float(K[0]), float(K[1]), float(K[2]), float(K[3]), W, H)
        dp, nd = None, 0
        if depth is not None and len(depth) > 0:
            arr = (DepthSample * len(depth))(*[DepthSample(float(u), float(v), float(z)) for (u, v, z) in depth])
            dp, nd = C.cast(arr, C.c_void_p), len(depth)
        _check(_lib.romap_add_observation(self._h, obj, _ptr(rgb), _ptr(mask), _ptr(T), C.byref(intr), dp, nd))

    def offer_observation(self, obj: int, rgb, mask, T_wc, K, depth=None, alpha_deg: float = 25.0,
                          iters_per_update: int = 300):
        """Eq. 5 keyframe gate (R25): returns (accepted, alpha in degrees or None)."""
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        mask = np.ascontiguousarray(mask, dtype=np.uint16)
        T = np.ascontiguousarray(np.asarray(T_wc, dtype=np.float32).reshape(12))
        H, W = mask.shape
        intr = Intrinsics(float(K[0]), float(K[1]), float(K[2]), float(K[3]), W, H)
        dp, nd = None, 0
        if depth is not None and len(depth):
            d = np.ascontiguousarray(np.asarray(depth, dtype=np.float32).reshape(-1, 3))
            dp, nd = _ptr(d), d.shape[0]
        acc = C.c_int32()
        alpha = C.c_float()
        _check(_lib.romap_offer_observation(self._h, obj, _ptr(rgb), _ptr(mask), _ptr(T), C.byref(intr), dp, nd,
                                            float(alpha_deg), int(iters_per_update), C.byref(acc), C.byref(alpha)))
        return bool(acc.value), (None if alpha.value < 0 else float(alpha.value))

    # ------------------------------------------------------------- async online trainer (f3)
    def async_start(self, chunk: int = 100, alpha_deg: float = 25.0, iters_per_update: int = 300,
                    queue_cap: int = 64):
        _check(_lib.romap_async_start(self._h, int(chunk), float(alpha_deg), int(iters_per_update), int(queue_cap)))

    def async_offer(self, obj: int, rgb, mask, T_wc, K) -> bool:
        """Queue a frame for the worker; returns False if the queue was full (dropped)."""
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        mask = np.ascontiguousarray(mask, dtype=np.uint16)
        T = np.ascontiguousarray(np.asarray(T_wc, dtype=np.float32).reshape(12))
        H, W = mask.shape
        intr = Intrinsics(float(K[0]), float(K[1]), float(K[2]), float(K[3]), W, H)
        q = C.c_int32()
        _check(_lib.romap_async_offer(self._h, obj, _ptr(rgb), _ptr(mask), _ptr(T), C.byref(intr), C.byref(q)))
        return bool(q.value)

    def async_stop(self, finish_pending: bool = True) -> dict:
        st = (C.c_int64 * 6)()
        _check(_lib.romap_async_stop(self._h, 1 if finish_pending else 0, C.cast(st, C.c_void_p)))
        return dict(zip(["offered", "dropped", "accepted", "iterations", "max_queue_depth", "rejected"], list(st)))

    def pending_iters(self, obj: int) -> int:
        p = C.c_int64()
        _check(_lib.romap_pending_iters(self._h, obj, C.byref(p)))
        return p.value

    def train_pending(self, chunk: int = 100, max_iters: int = 1 << 30) -> dict:
        """f3 scheduler: {object id: iterations run}."""
        cap = 4096
        ids = np.zeros(cap, np.int32)
        its = np.zeros(cap, np.int32)
        n = C.c_int32()
        _check(_lib.romap_train_pending(self._h, int(chunk), int(max_iters), _ptr(ids), _ptr(its), cap, C.byref(n)))
        return {int(ids[i]): int(its[i]) for i in range(min(n.value, cap))}

    def set_rays_per_iter(self, obj: int, rays: int):
        _check(_lib.romap_set_rays_per_iter(self._h, obj, int(rays)))

    # ------------------------------------------------------------- training
    def train_step(self, objs, n_iters: int = 1) -> list[dict]:
        ids, n = _ids(objs)
        st = (TrainStats * n)()
        _check(_lib.romap_train_step(self._h, _ptr(ids), n, int(n_iters), C.cast(st, C.c_void_p)))
        return [s.as_dict() for s in st]

    def forward_backward(self, objs) -> list[dict]:
        ids, n = _ids(objs)
        st = (TrainStats * n)()
        _check(_lib.romap_forward_backward(self._h, _ptr(ids), n, C.cast(st, C.c_void_p)))
        return [s.as_dict() for s in st]

    def optimizer_step(self, objs):
        ids, n = _ids(objs)
        _check(_lib.romap_optimizer_step(self._h, _ptr(ids), n))

    # ------------------------------------------------------------- inference
    def render(self, obj: int, T_wc, K, width: int, height: int, samples_per_ray: int):
        T = np.ascontiguousarray(np.asarray(T_wc, dtype=np.float32).reshape(12))
        intr = Intrinsics(float(K[0]), float(K[1]), float(K[2]), float(K[3]), width, height)
        rgb = np.zeros((height, width, 3), np.float32)
        dep = np.zeros((height, width), np.float32)
        opa = np.zeros((height, width), np.float32)
        _check(_lib.romap_render(self._h, obj, _ptr(T), C.byref(intr), samples_per_ray, _ptr(rgb), _ptr(dep),
                                 _ptr(opa), 0))
        return rgb, dep, opa

    def render_scene(self, objs, T_wc, K, width: int, height: int, samples_per_segment: int):
        ids, n = _ids(objs)
        T = np.ascontiguousarray(np.asarray(T_wc, dtype=np.float32).reshape(12))
        intr = Intrinsics(float(K[0]), float(K[1]), float(K[2]), float(K[3]), width, height)
        rgb = np.zeros((height, width, 3), np.float32)
        dep = np.zeros((height, width), np.float32)
        opa = np.zeros((height, width), np.float32)
        _check(_lib.romap_render_scene(self._h, _ptr(ids), n, _ptr(T), C.byref(intr), samples_per_segment, _ptr(rgb),
                                       _ptr(dep), _ptr(opa), 0))
        return rgb, dep, opa

    def extract_mesh(self, obj: int, res: int = 64, sigma_iso: float = 20.0, carve: bool = False):
        """Marching-tetrahedra isosurface (R26): (T, 3, 3) float32 world-frame triangles;
        carve: zero the density where no keyframe sees the lattice."""
        n = C.c_int64()
        fl = MESH_CARVE if carve else 0
        _check(_lib.romap_extract_mesh(self._h, obj, int(res), float(sigma_iso), None, 0, C.byref(n), fl))
        out = np.zeros((max(n.value, 1), 3, 3), np.float32)
        if n.value:
            _check(_lib.romap_extract_mesh(self._h, obj, int(res), float(sigma_iso), _ptr(out), n.value, C.byref(n),
                                           fl))
        return out[:n.value]

    def query_density(self, obj: int, xyz):
        """xyz: numpy (n,3) float32 (host) or a CUDA torch tensor (device pointers)."""
        if hasattr(xyz, "is_cuda") and xyz.is_cuda:
            import torch
            x = xyz.contiguous().float()
            out = torch.empty(x.shape[0], device=x.device, dtype=torch.float32)
            _check(_lib.romap_query_density(self._h, obj, _ptr(x), x.shape[0], _ptr(out), DEVICE_PTRS))
            return out
        x = np.ascontiguousarray(xyz, dtype=np.float32).reshape(-1, 3)
        out = np.zeros(x.shape[0], np.float32)
        _check(_lib.romap_query_density(self._h, obj, _ptr(x), x.shape[0], _ptr(out), 0))
        return out

    # ------------------------------------------------------------- params / debug
    def block_bytes(self, obj: int, block: int) -> int:
        b = C.c_int64()
        _check(_lib.romap_block_bytes(self._h, obj, block, C.byref(b)))
        return b.value

    def get_params(self, obj: int, block: int):
        nb = self.block_bytes(obj, block)
        out = np.zeros(nb // 8, np.int64) if block == BLOCK_STEP else np.zeros(nb // 4, np.float32)
        _check(_lib.romap_get_params(self._h, obj, block, _ptr(out), nb))
        return out

    def set_params(self, obj: int, block: int, arr):
        a = np.ascontiguousarray(arr, dtype=np.int64 if block == BLOCK_STEP else np.float32).reshape(-1)
        _check(_lib.romap_set_params(self._h, obj, block, _ptr(a), a.nbytes))

    def debug_dump(self, obj: int, what: int):
        b = C.c_int64()
        _check(_lib.romap_dump_bytes(self._h, obj, what, C.byref(b)))
        if what == DUMP_RAYS:
            out = np.zeros(b.value // RAY_DUMP_DTYPE.itemsize, RAY_DUMP_DTYPE)
        elif what == DUMP_HASH_IDX:
            out = np.zeros(b.value // 4, np.int32)
        else:
            out = np.zeros(b.value // 4, np.float32)
        _check(_lib.romap_debug_dump(self._h, obj, what, _ptr(out), b.value))
        return out

    def sync(self):
        _check(_lib.romap_sync(self._h))

    def set_l2_flush(self, nbytes: int):
        _check(_lib.romap_set_l2_flush(self._h, int(nbytes)))

    def save_object(self, obj: int, path: str):
        """Checkpoint one object (romap.h romap_save_object)."""
        _check(_lib.romap_save_object(self._h, obj, os.fsencode(path)))

    def load_object(self, path: str, obj_id: int | None = None) -> int:
        """Recreate an object from a checkpoint; returns its id."""
        out = C.c_int32()
        _check(_lib.romap_load_object(self._h, os.fsencode(path), -1 if obj_id is None else int(obj_id), C.byref(out)))
        return out.value

    def set_deterministic(self, on: bool = True):
        """Deterministic-reduction mode (romap.h): fixed-order gradient / loss sums."""
        _check(_lib.romap_set_deterministic(self._h, 1 if on else 0))

    def profile_enable(self, on: bool = True, stages=None):
        """Per-stage event timing; `stages` (names) restricts the events to those stages."""
        if stages is None or not on:
            _check(_lib.romap_profile_enable(self._h, 1 if on else 0))
            return
        names = list(self.profile_read().keys())
        mask = 0
        for s in stages:
            mask |= 1 << names.index(s)
        _check(_lib.romap_profile_stages(self._h, mask))

    def profile_read(self) -> dict:
        arr = (StageTime * 16)()
        n = C.c_int32()
        _check(_lib.romap_profile_read(self._h, C.cast(arr, C.c_void_p), 16, C.byref(n)))
        return {arr[i].name.decode(): {"launches": arr[i].launches, "ms": arr[i].ms} for i in range(n.value)}

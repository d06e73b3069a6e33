"""Render cost breakdown (cfg4 ii): one trained cfg1 object, 640x480 x 128 samples;
host-output wall clock vs device-pointer CUDA-event time, active-ray count."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2304_05735_b200 import romap as R  # noqa: E402

ctx = R.Context(0)
sc = bench.load_scene()
ob = sc.objects[0]
h = ctx.create_object(ob.t, ob.yaw, ob.a, R.model_config(**bench.cfg1_kwargs(1)), ob.instance_id)
for fr in sc.frames:
    ctx.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
ctx.train_step([h], 100)
fr = sc.frames[0]
rgb, dep, opa = ctx.render(h, fr.T_wc, fr.K, 640, 480, 128)
print("active rays (opacity > 0):", int((opa > 0).sum()), "of", 640 * 480)
for _ in range(2):
    t0 = time.perf_counter()
    ctx.render(h, fr.T_wc, fr.K, 640, 480, 128)
    print(f"host outputs: {(time.perf_counter() - t0) * 1e3:.2f} ms")
# device pointers
T = np.ascontiguousarray(np.asarray(fr.T_wc, np.float32).reshape(12))
K = fr.K
intr = R.Intrinsics(float(K[0]), float(K[1]), float(K[2]), float(K[3]), 640, 480)
o_rgb = torch.empty(480 * 640 * 3, device="cuda")
o_dep = torch.empty(480 * 640, device="cuda")
o_opa = torch.empty(480 * 640, device="cuda")
lib = R._lib
def dev():
    R._check(lib.romap_render(ctx._h, h, T.ctypes.data_as(C.c_void_p), C.byref(intr), 128,
                              C.c_void_p(o_rgb.data_ptr()), C.c_void_p(o_dep.data_ptr()),
                              C.c_void_p(o_opa.data_ptr()), R.DEVICE_PTRS))
dev()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    dev()
e1.record()
torch.cuda.synchronize()
print(f"device outputs: {e0.elapsed_time(e1) / 5:.2f} ms per frame")

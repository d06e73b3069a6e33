"""Where the e2e step (add_observation + train_step(50) + stats) spends its time."""
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
for fr in sc.frames[:20]:
    ctx.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
ctx.train_step([h], 60)
frames = sc.frames[20:] or sc.frames
pinned = [(torch.from_numpy(f.rgb).pin_memory(), torch.from_numpy(f.mask.astype(np.int16)).pin_memory(), f)
          for f in frames]
torch.cuda.synchronize()
ta = tt = 0.0
n = 8
t0 = time.perf_counter()
for k in range(n):
    rgb, mask, fr = pinned[k % len(pinned)]
    a0 = time.perf_counter()
    ctx.add_observation(h, rgb.numpy(), mask.numpy().view(np.uint16), fr.T_wc, fr.K)
    a1 = time.perf_counter()
    ctx.train_step([h], 50)
    a2 = time.perf_counter()
    ta += a1 - a0
    tt += a2 - a1
tot = time.perf_counter() - t0
print(f"per e2e step: total {tot / n * 1e3:.2f} ms, add_observation {ta / n * 1e3:.3f} ms, "
      f"train_step(50) {tt / n * 1e3:.2f} ms ({tt / n / 50 * 1e6:.1f} us/iter)")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ctx.train_step([h], 50)
e1.record()
torch.cuda.synchronize()
print(f"train_step(50) device time {e0.elapsed_time(e1):.2f} ms ({e0.elapsed_time(e1) / 50 * 1e3:.1f} us/iter)")

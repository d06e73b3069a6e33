"""Production rate of train_step with graph replay (no L2 flush, no per-stage
events): cfg1, CUDA events around one call of n iterations."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import scenes
from paper_2304_05735_b200 import romap as R
import bench

kw = bench.cfg1_kwargs(1)
sc = scenes.object_scene(1, n_views=20)
ob = sc.objects[0]
c = R.Context(0)
h = c.create_object(ob.t, ob.yaw, ob.a, R.model_config(**kw), ob.instance_id)
for fr in sc.frames:
    c.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
c.train_step([h], 32)
for n in (16, 160, 480):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = c.train_step([h], n)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"n={n}: {ms / n * 1e3:.1f} us per iteration, {st[0]['samples'] / (ms * 1e-3):.4e} ray-samples/s")
c.profile_enable(True)
c.train_step([h], 16)
p = c.profile_read()
print({k: round(v["ms"] / 16 * 1e3, 1) for k, v in p.items() if v["ms"]})
c.close()

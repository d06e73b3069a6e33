"""Repeat timed train_step calls (paper or cfg1 workload) with all stages bracketed by
events and print per-stage ms per iteration, to locate sporadic slow iterations."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2304_05735_b200 import romap as R  # noqa: E402

ctx = R.Context(0)
kw = bench.paper_kwargs() if "--paper" in sys.argv else bench.cfg1_kwargs(1)
sc = bench.load_scene()
ob = sc.objects[0]
h = ctx.create_object(ob.t, ob.yaw, ob.a, R.model_config(**kw), ob.instance_id)
for fr in sc.frames:
    ctx.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
ctx.train_step([h], 10)
ctx.set_l2_flush(512 << 20)
for rep in range(8):
    ctx.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    ctx.train_step([h], 50)
    e1.record()
    torch.cuda.synchronize()
    p = ctx.profile_read()
    tot = e0.elapsed_time(e1) / 50 * 1e3
    print(f"rep {rep}: total {tot:9.1f} us/iter | " + ", ".join(f"{k} {v['ms'] / 50 * 1e3:.1f}" for k, v in p.items() if v["launches"]))

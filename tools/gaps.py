"""Step time of the bench workload with / without per-stage events and L2 flush (launch-gap diagnosis)."""
import os
import sys
import time

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
for prof in (None, ["l2_flush"], ["fused_mixed", "l2_flush"], "all"):
    for flush in (0, 512 << 20):
        ctx.set_l2_flush(flush)
        if prof == "all":
            ctx.profile_enable(True)
        elif prof:
            ctx.profile_enable(True, stages=prof)
        else:
            ctx.profile_enable(False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.train_step([h], 50)
        e1.record()
        torch.cuda.synchronize()
        p = ctx.profile_read() if prof else {}
        fl = p.get("l2_flush", {}).get("ms", 0.0)
        print(f"prof={prof} flush={flush>>20}MiB: {e0.elapsed_time(e1)/50*1e3:8.1f} us/iter total, "
              f"flush {fl/50*1e3:6.1f} us/iter, stages " + ", ".join(f"{k} {v['ms']/50*1e3:.1f}" for k, v in p.items() if v['launches']))
        ctx.profile_enable(False)

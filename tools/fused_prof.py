"""Phase timing of k_fused_mixed (library built with EXTRA=-DROMAP_FUSED_PROF):
per-tile cycle averages of the M (MLP/render) and G (gather/scatter) roles on
the bench workload (cfg1, 1 object, 4096 x 64)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2304_05735_b200 import romap as R  # noqa: E402

lib = C.CDLL(R.LIB_PATH)
fn = lib.romap_debug_fused_prof
fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
ctx = R.Context(0)
kw = bench.cfg1_kwargs(1)
sc = bench.load_scene()
ob = sc.objects[0]
h = ctx.create_object(ob.t, ob.yaw, ob.a, R.model_config(**kw), ob.instance_id)
for fr in sc.frames:
    ctx.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
ctx.train_step([h], 5)
buf = (C.c_ulonglong * 16)()
fn(buf, 1)
iters = 20
ctx.train_step([h], iters)
fn(buf, 1)
v = list(buf)
tiles = 4096 * 64 // 128 * iters
ctas = 148 * iters
names = {0: "M total", 1: "M wait x0_full", 2: "M fwd chain", 3: "M render", 4: "M bwd chain", 6: "M tile top", 11: "  render T scan", 12: "  render sums", 13: "  render loss", 14: "  render suffix",
         8: "G total (per WG)", 9: "G wait tile_done", 10: "G level loop"}
for k, n in names.items():
    per = v[k] / (2 * tiles if k >= 8 else tiles)
    print(f"{n:20s} {per:10.0f} cycles/tile   ({v[k] / ctas / 1965:.1f} us per CTA-iteration{' per WG' if k >= 8 else ''})")

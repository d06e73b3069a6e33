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
paper = "--paper" in sys.argv                  # the paper's workload (network 1, 4096 x 32)
kw = bench.paper_kwargs() if paper else bench.cfg1_kwargs(1)
import scenes  # noqa: E402
sc = scenes.object_scene(1, n_views=20)
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
tiles = 4096 * kw["samples_per_ray"] // 128 * iters
ctas = 148 * iters
names = {5: "CTA setup", 7: "CTA total", 15: "M final flush", 0: "M total", 1: "M wait x0_full", 2: "M fwd chain", 3: "M render", 4: "M bwd chain", 6: "M tile top", 12: "  render scans", 13: "  render loss",
         8: "G total (per WG)", 9: "G wait tile_done", 10: "G level loop"}
G1 = v[11] / tiles
print(f"G level loop per warpgroup: G0 {(v[10] - v[11]) / tiles:.0f}, G1 {G1:.0f} cycles/tile")
for k, n in names.items():
    per = v[k] / (2 * tiles if 8 <= k <= 10 else tiles)
    print(f"{n:20s} {per:10.0f} cycles/tile   ({v[k] / ctas / 1965:.1f} us per CTA-iteration{' per WG' if 8 <= k <= 10 else ''})")

# CTA lifetimes of the last launch (%globaltimer, ns)
fc = lib.romap_debug_fused_cta_ns
fc.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
nb = 148
cb = (C.c_ulonglong * (2 * nb))()
fc(cb, nb)
st = [cb[2 * i] for i in range(nb)]
en = [cb[2 * i + 1] for i in range(nb)]
t0 = min(st)
life = sorted(e - s for s, e in zip(st, en))
print(f"last launch: span {(max(en) - t0) / 1e3:.1f} us, CTA start skew {(max(st) - t0) / 1e3:.2f} us, "
      f"lifetime min/median/max {life[0] / 1e3:.1f}/{life[nb // 2] / 1e3:.1f}/{life[-1] / 1e3:.1f} us")
ends = sorted((e - t0) / 1e3 for e in en)
print("CTA end times (us) deciles:", [round(ends[min(nb - 1, i * nb // 10)], 1) for i in range(11)])

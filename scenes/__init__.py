"""Seeded synthetic scenes (input generators only -- no method arithmetic).

These stand in for the paper's datasets (Cube-Diorama, Replica, RealSense
sequences), which are not available and are never recreated.
They take the paper's shapes: 640x480 monocular posed RGB + instance masks of
tabletop / room scenes with several objects, and the
BASELINE.json configs' recipes.

Both the oracle and the CUDA path consume the same arrays; this module is
shared by tests/ and bench.py and holds none of the method's arithmetic
(no sampling, encoding, rendering-for-training or losses).  GT images are made by
analytic / sphere-traced intersection with procedural surfaces.

Camera convention (the data format): OpenCV pinhole (x right, y down, z forward),
pixel centres at (px+.5, py+.5), T_wc = camera->world 3x4, world z-up.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch


@dataclass
class Frame:
    rgb: np.ndarray        # (H,W,3) uint8
    mask: np.ndarray       # (H,W) uint16, 0 = background
    T_wc: np.ndarray       # (3,4) float32, pose given to the trainer (may be jittered)
    K: np.ndarray          # (4,) float32 fx, fy, cx, cy
    width: int
    height: int
    depth: dict = field(default_factory=dict)   # instance id -> list of (u, v, z)


@dataclass
class SceneObject:
    instance_id: int
    t: np.ndarray          # (3,) float32 world centre of the box
    yaw: float
    a: np.ndarray          # (3,) float32 half extents
    shape: dict            # procedural shape parameters (object frame)


@dataclass
class Scene:
    frames: list
    objects: list
    name: str


# ----------------------------------------------------------------------------
def look_at(cam, target):
    """Camera->world rotation (OpenCV axes) looking from cam to target, z-up world."""
    f = np.asarray(target, np.float64) - np.asarray(cam, np.float64)
    f /= np.linalg.norm(f)
    up = np.array([0.0, 0.0, 1.0])
    if abs(f @ up) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    r = np.cross(f, up)
    r /= np.linalg.norm(r)
    dn = np.cross(f, r)
    R = np.stack([r, dn, f], axis=1)
    T = np.concatenate([R, np.asarray(cam, np.float64)[:, None]], axis=1)
    return T.astype(np.float32)


def pixel_rays(T_wc, K, W, H, dev):
    fx, fy, cx, cy = [float(v) for v in K]
    ys, xs = torch.meshgrid(torch.arange(H, device=dev, dtype=torch.float64),
                            torch.arange(W, device=dev, dtype=torch.float64), indexing="ij")
    dc = torch.stack([(xs + 0.5 - cx) / fx, (ys + 0.5 - cy) / fy, torch.ones_like(xs)], -1)
    zscale = 1.0 / dc.norm(dim=-1)
    d = dc * zscale[..., None]
    T = torch.as_tensor(np.asarray(T_wc, np.float64), device=dev)
    dw = d @ T[:, :3].T
    o = T[:, 3].expand_as(dw)
    return o.reshape(-1, 3), dw.reshape(-1, 3), zscale.reshape(-1)


def procedural_color(p, seed_vec):
    """Smooth seeded colour texture ("Perlin-like": a sum of two seeded sinusoid octaves)."""
    s = seed_vec
    out = []
    for c in range(3):
        v = 0.5
        v = v + 0.25 * torch.sin(s[c, 0] * p[:, 0] + s[c, 1] * p[:, 1] + s[c, 2] * p[:, 2] + s[c, 3])
        v = v + 0.15 * torch.sin(2.1 * (s[c, 2] * p[:, 0] - s[c, 0] * p[:, 1] + s[c, 1] * p[:, 2]) + s[c, 4])
        out.append(v)
    return torch.stack(out, -1).clamp(0.02, 0.98)


def to_u8(x):
    return (x.clamp(0, 1) * 255.0 + 0.5).floor().to(torch.uint8)


# ----------------------------------------------------------------------------
# config 0: textured sphere in the unit box (BASELINE cfg0)
# ----------------------------------------------------------------------------
def fibonacci_sphere(n, radius):
    pts = []
    ga = math.pi * (3.0 - math.sqrt(5.0))
    for i in range(n):
        z = 1.0 - 2.0 * (i + 0.5) / n
        r = math.sqrt(max(0.0, 1.0 - z * z))
        th = ga * i
        pts.append((radius * r * math.cos(th), radius * r * math.sin(th), radius * z))
    return pts


def sphere_scene(seed=0, n_views=8, size=64, f=64.0, radius=2.0, r_sphere=0.4, depth_per_view=0):
    """cfg0: sphere r=0.4 at the origin of the box [-0.5,0.5]^3, yaw 0, 8 views
    of 64x64 at radius 2 on a Fibonacci sphere, f=64, c=32, binary masks."""
    g = np.random.default_rng(seed)
    dev = torch.device("cpu")
    sv = torch.as_tensor(g.uniform(3.0, 9.0, size=(3, 5)), dtype=torch.float64)
    sv[:, 3:] = torch.as_tensor(g.uniform(0, 2 * math.pi, size=(3, 2)))
    K = np.array([f, f, size / 2.0, size / 2.0], np.float32)
    frames = []
    for cam in fibonacci_sphere(n_views, radius):
        T = look_at(cam, (0.0, 0.0, 0.0))
        o, d, zs = pixel_rays(T, K, size, size, dev)
        b = (o * d).sum(-1)
        c = (o * o).sum(-1) - r_sphere ** 2
        disc = b * b - c
        hit = disc > 0
        th = -b - torch.sqrt(disc.clamp_min(0))
        p = o + th[:, None] * d
        col = procedural_color(p, sv)
        bgc = torch.tensor([0.35, 0.4, 0.45], dtype=torch.float64).expand_as(col)
        img = torch.where(hit[:, None], col, bgc)
        mask = hit.to(torch.int32).reshape(size, size)
        fr = Frame(to_u8(img).reshape(size, size, 3).numpy(), mask.numpy().astype(np.uint16), T, K, size, size)
        if depth_per_view:
            idx = torch.nonzero(hit).reshape(-1).numpy()
            pick = g.choice(idx, size=min(depth_per_view, idx.size), replace=False)
            lst = []
            for pi in pick:
                py, px = divmod(int(pi), size)
                lst.append((px + 0.5, py + 0.5, float(th[pi] * zs[pi])))
            fr.depth[1] = lst
        frames.append(fr)
    obj = SceneObject(1, np.zeros(3, np.float32), 0.0, np.full(3, 0.5, np.float32), {"sphere": r_sphere})
    return Scene(frames, [obj], "cfg0-sphere")


# ----------------------------------------------------------------------------
# configs 1-3: box-union-torus SDF objects on a textured floor
# ----------------------------------------------------------------------------
def random_shape(g, a):
    """Seeded box-union-torus inside half extents a (object frame, z-up, resting on z=-a_z)."""
    a = np.asarray(a, np.float64)
    bh = a * g.uniform(0.45, 0.8, size=3)
    bh[2] = a[2] * g.uniform(0.3, 0.6)
    bc = np.array([g.uniform(-1, 1) * (a[0] - bh[0]) * 0.5, g.uniform(-1, 1) * (a[1] - bh[1]) * 0.5, -a[2] + bh[2]])
    Rt = min(a[0], a[1]) * g.uniform(0.45, 0.65)
    rt = min(Rt * g.uniform(0.2, 0.35), a[2] * 0.4)
    tc = np.array([0.0, 0.0, min(bc[2] + bh[2] + rt * 0.5, a[2] - rt)])
    sv = np.concatenate([g.uniform(2.0, 8.0, size=(3, 3)), g.uniform(0, 2 * math.pi, size=(3, 2))], axis=1)
    return {"bc": bc, "bh": bh, "tc": tc, "R": Rt, "r": rt, "sv": sv}


def shape_sdf(p, sh):
    """SDF of box U torus in object frame. p: (n,3) float64 tensor."""
    bc = torch.as_tensor(sh["bc"], dtype=p.dtype, device=p.device)
    bh = torch.as_tensor(sh["bh"], dtype=p.dtype, device=p.device)
    q = (p - bc).abs() - bh
    dbox = q.clamp_min(0).norm(dim=-1) + q.max(dim=-1).values.clamp_max(0)
    tcen = torch.as_tensor(sh["tc"], dtype=p.dtype, device=p.device)
    pt = p - tcen
    qx = torch.sqrt(pt[:, 0] ** 2 + pt[:, 1] ** 2) - sh["R"]
    dtor = torch.sqrt(qx ** 2 + pt[:, 2] ** 2) - sh["r"]
    return torch.minimum(dbox, dtor)


def world_to_obj(p, ob):
    c, s = math.cos(ob.yaw), math.sin(ob.yaw)
    q = p - torch.as_tensor(ob.t, dtype=p.dtype, device=p.device)
    return torch.stack([c * q[:, 0] + s * q[:, 1], -s * q[:, 0] + c * q[:, 1], q[:, 2]], -1)


def dir_to_obj(d, ob):
    c, s = math.cos(ob.yaw), math.sin(ob.yaw)
    return torch.stack([c * d[:, 0] + s * d[:, 1], -s * d[:, 0] + c * d[:, 1], d[:, 2]], -1)


def render_sdf_frame(objects, T_true, K, W, H, dev, floor_seed, steps=64):
    """Ray-cast the floor plane z=0 and every object (slab-culled sphere tracing)."""
    o, d, zs = pixel_rays(T_true, K, W, H, dev)
    n = o.shape[0]
    best_t = torch.full((n,), float("inf"), dtype=torch.float64, device=dev)
    best_id = torch.zeros(n, dtype=torch.int32, device=dev)
    col = torch.zeros(n, 3, dtype=torch.float64, device=dev)
    # floor z = 0
    tfl = torch.where(d[:, 2] < -1e-9, -o[:, 2] / d[:, 2], torch.full_like(d[:, 2], float("inf")))
    pf = o + tfl.clamp(max=1e6)[:, None] * d
    chk = ((torch.floor(pf[:, 0] * 4) + torch.floor(pf[:, 1] * 4)) % 2)
    fcol = torch.stack([0.55 + 0.2 * chk, 0.5 + 0.15 * chk, 0.42 + 0.1 * chk], -1)
    fcol = fcol * (0.8 + 0.2 * torch.sin(pf[:, 0] * 1.3 + floor_seed)[:, None] * torch.cos(pf[:, 1] * 0.7)[:, None])
    sky = torch.stack([0.6 + 0.2 * d[:, 2], 0.65 + 0.2 * d[:, 2], 0.75 + 0.1 * d[:, 2]], -1)
    is_floor = torch.isfinite(tfl)
    col = torch.where(is_floor[:, None], fcol, sky)
    best_t = torch.where(is_floor, tfl, best_t)
    for ob in objects:
        oo = world_to_obj(o, ob)
        od = dir_to_obj(d, ob)
        a = torch.as_tensor(ob.a, dtype=torch.float64, device=dev)
        with torch.no_grad():
            inv = 1.0 / torch.where(od.abs() < 1e-12, torch.full_like(od, 1e-12), od)
            t0 = (-a - oo) * inv
            t1 = (a - oo) * inv
            tn = torch.minimum(t0, t1).max(dim=-1).values.clamp_min(0)
            tf = torch.maximum(t0, t1).min(dim=-1).values
        cand = torch.nonzero((tf > tn) & (tn < best_t)).reshape(-1)
        if cand.numel() == 0:
            continue
        t = tn[cand].clone()
        oc, dc_, tfc = oo[cand], od[cand], tf[cand]
        alive = torch.ones_like(t, dtype=torch.bool)
        hit = torch.zeros_like(alive)
        for _ in range(steps):
            p = oc + t[:, None] * dc_
            sd = shape_sdf(p, ob.shape)
            newhit = alive & (sd < 1e-4)
            hit |= newhit
            alive &= ~newhit
            t = torch.where(alive, t + sd.clamp_min(1e-4), t)
            alive &= t < tfc
        sel = hit & (t < best_t[cand])
        idx = cand[sel]
        best_t[idx] = t[sel]
        best_id[idx] = ob.instance_id
        pobj = oc[sel] + t[sel][:, None] * dc_[sel]
        sv = torch.as_tensor(ob.shape["sv"], dtype=torch.float64, device=dev)
        col[idx] = procedural_color(pobj, sv)
    rgb = to_u8(col).reshape(H, W, 3).cpu().numpy()
    mask = best_id.reshape(H, W).cpu().numpy().astype(np.uint16)
    zdep = (best_t * zs).reshape(H, W).cpu().numpy()
    return rgb, mask, zdep


def _orbit_poses(g, n, center, radius, elev_lo, elev_hi):
    out = []
    for i in range(n):
        az = 2 * math.pi * i / n + g.uniform(-0.1, 0.1)
        el = math.radians(g.uniform(elev_lo, elev_hi))
        cam = (center[0] + radius * math.cos(el) * math.cos(az), center[1] + radius * math.cos(el) * math.sin(az),
               center[2] + radius * math.sin(el))
        out.append(look_at(cam, center))
    return out


def _jitter(g, T, sigma):
    J = T.copy()
    J[:, 3] += g.normal(0.0, sigma, size=3).astype(np.float32)
    return J


def _depth_samples(g, mask, zdep, iid, k):
    ys, xs = np.nonzero(mask == iid)
    if xs.size == 0 or k == 0:
        return []
    pick = g.choice(xs.size, size=min(k, xs.size), replace=False)
    return [(xs[p] + 0.5, ys[p] + 0.5, float(zdep[ys[p], xs[p]])) for p in pick]


def object_scene(seed=1, n_views=20, W=640, H=480, f=525.0, device=None, depth_per_view=0, jitter=0.01,
                 half_extents=None):
    """cfg1: one box-union-torus object (box ~0.8 m) on a textured floor, 20 keyframes on
    an orbit (radius 1.2 m, elevation 15-45 deg), 640x480, f=525, c=(320,240);
    training poses = true + N(0, 1 cm) translation jitter.  half_extents: another box
    size of the same family (cfg3 draws edges U(0.2, 1.5) m); the orbit radius scales
    with it (1.2 m for the cfg1 box), so the object fills a similar part of the frame."""
    g = np.random.default_rng(seed)
    dev = torch.device(device or ("cuda" if torch.cuda.is_available() else "cpu"))
    a = np.array([0.4, 0.4, 0.3], np.float32) * g.uniform(0.9, 1.0, size=3).astype(np.float32)
    radius = 1.2
    if half_extents is not None:
        a = np.asarray(half_extents, np.float32)
        radius = 1.2 * float(max(a[0], a[1], a[2])) / 0.4
    ob = SceneObject(1, np.array([0.0, 0.0, a[2]], np.float32), float(g.uniform(-0.3, 0.3)), a, random_shape(g, a))
    K = np.array([f, f, W / 2.0, H / 2.0], np.float32)
    frames = []
    for T in _orbit_poses(g, n_views, (0.0, 0.0, float(a[2])), radius, 15, 45):
        rgb, mask, zd = render_sdf_frame([ob], T, K, W, H, dev, float(seed))
        fr = Frame(rgb, mask, _jitter(g, T, jitter), K, W, H)
        if depth_per_view:
            fr.depth[1] = _depth_samples(g, mask, zd, 1, depth_per_view)
        frames.append(fr)
    return Scene(frames, [ob], "cfg1-object")


def room_scene(seed=2, n_objects=8, n_frames=200, W=640, H=480, f=525.0, device=None, edge_lo=0.2, edge_hi=1.5,
               depth_per_view=0, jitter=0.01, room_half=None):
    """cfg2/cfg3: n objects of the cfg1 family in one room; edges U(0.2,1.5) m per axis,
    yaw U(-45,45) deg, non-overlapping footprints on the floor (rejection sampling);
    one shared camera trajectory (a loop around the room looking inwards)."""
    g = np.random.default_rng(seed)
    dev = torch.device(device or ("cuda" if torch.cuda.is_available() else "cpu"))
    if room_half is None:
        room_half = max(2.0, 0.9 * math.sqrt(n_objects) + 0.5)
    objs, foot = [], []
    iid = 1
    tries = 0
    while len(objs) < n_objects and tries < 100000:
        tries += 1
        e = g.uniform(edge_lo, edge_hi, size=3)
        a = (e / 2).astype(np.float32)
        yaw = float(np.radians(g.uniform(-45, 45)))
        rad = float(np.hypot(a[0], a[1]))
        c = g.uniform(-room_half + rad, room_half - rad, size=2)
        if any(np.hypot(*(c - fc)) < rad + fr + 0.05 for fc, fr in foot):
            continue
        foot.append((c, rad))
        objs.append(SceneObject(iid, np.array([c[0], c[1], a[2]], np.float32), yaw, a, random_shape(g, a)))
        iid += 1
    K = np.array([f, f, W / 2.0, H / 2.0], np.float32)
    frames = []
    for i in range(n_frames):
        az = 2 * math.pi * i / n_frames
        rr = room_half + 1.5
        cam = (rr * math.cos(az), rr * math.sin(az), 1.6 + 0.3 * math.sin(3 * az))
        look = (0.6 * room_half * math.cos(az + 2.2), 0.6 * room_half * math.sin(az + 2.2), 0.3)
        T = look_at(cam, look)
        rgb, mask, zd = render_sdf_frame(objs, T, K, W, H, dev, float(seed))
        fr = Frame(rgb, mask, _jitter(g, T, jitter), K, W, H)
        if depth_per_view:
            for ob in objs:
                ds = _depth_samples(g, mask, zd, ob.instance_id, depth_per_view)
                if ds:
                    fr.depth[ob.instance_id] = ds
        frames.append(fr)
    return Scene(frames, objs, f"room-{n_objects}")


def visible_frames(scene, iid, min_frac=0.0):
    """Indices of frames where instance iid covers more than min_frac of the image."""
    out = []
    for i, fr in enumerate(scene.frames):
        cnt = int((fr.mask == iid).sum())
        if cnt > 0 and cnt >= min_frac * fr.width * fr.height:
            out.append(i)
    return out


def random_params(cfg_levels, feats, n_entries, mlp_sizes, seed, table_scale=1e-1):
    """Seeded parameter set for parity tests (shared by both sides via set_params)."""
    g = np.random.default_rng(seed)
    table = g.uniform(-table_scale, table_scale, size=(n_entries, feats)).astype(np.float32)
    W = []
    for (o, i) in mlp_sizes:
        lim = math.sqrt(6.0 / (o + i))
        W.append(g.uniform(-lim, lim, size=(o, i)).astype(np.float32))
    return table, W

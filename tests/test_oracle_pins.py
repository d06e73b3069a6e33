"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names the passage / closed form it checks.  A plausible mistake in
the oracle (dropped term, wrong sign or index, transposed operand) must fail one
of these.
"""
import math
import os

import numpy as np
import pytest

import oracle as O

f32 = np.float32
GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- O1 level table
def test_level_table_cfg0_hand_listed():
    # BASELINE cfg0: L=8, base 16, growth 2, finest 2048 capped at 128, T=2^12
    lt = O.level_table(O.ModelConfig())
    assert [l.res for l in lt] == [16, 32, 64, 128, 128, 128, 128, 128]
    assert not any(l.dense for l in lt)           # 17^3 = 4913 > 4096
    assert O.table_entries(O.ModelConfig()) == 32768


def test_level_table_cfg1_hand_listed():
    # BASELINE cfg1: L=16, resolutions 16 -> 512, T=2^16
    cfg = O.ModelConfig(levels=16, log2_T=16, finest_res=512.0, res_cap=0)
    lt = O.level_table(cfg)
    assert [l.res for l in lt] == [16, 20, 25, 32, 40, 50, 64, 80, 101, 128, 161, 203, 256, 322, 406, 512]
    assert [l.dense for l in lt] == [True] * 4 + [False] * 12      # 33^3 <= 65536 < 41^3
    # R5: level blocks padded to 16 entries: 4913->4928, 9261->9264, 17576->17584, 35937->35952
    assert O.table_entries(cfg) == 4928 + 9264 + 17584 + 35952 + 12 * 65536 == 854160
    assert [l.offset for l in lt[:5]] == [0, 4928, 4928 + 9264, 4928 + 9264 + 17584, 4928 + 9264 + 17584 + 35952]
    assert sum(l.size for l in lt) == 854119                        # addressable entries


# ---------------------------------------------------------------- O2 RNG
def test_splitmix64_published_vectors():
    vals = [int(l, 16) for l in open(os.path.join(GOLD, "splitmix64_seed0.txt")) if l.strip() and not l.startswith("#")]
    state = 0
    for v in vals:
        state = (state + O.GOLDEN) & ((1 << 64) - 1)
        assert int(O.mix64(state)) == v


def test_rng_unit_range_and_uniformity():
    u = O.u32_to_unit(O.rng_u32(5, 3, 7, np.arange(200000), 16))
    assert u.dtype == np.float32 and u.min() >= 0 and u.max() < 1
    h, _ = np.histogram(u, bins=20, range=(0, 1))
    chi2 = ((h - 10000.0) ** 2 / 10000.0).sum()
    assert chi2 < 45          # 19 dof, p ~ 1e-3
    # streams / rays / steps / objects are decorrelated
    a = O.rng_u32(5, 3, 7, np.arange(1000), 1)
    b = O.rng_u32(5, 3, 7, np.arange(1000), 2)
    c = O.rng_u32(5, 4, 7, np.arange(1000), 1)
    assert (a != b).mean() > 0.99 and (a != c).mean() > 0.99


# ---------------------------------------------------------------- a0 / O3 pixels
def _kf(x0, y0, w, h, cls_val=1):
    return O.Keyframe(np.eye(3, 4, dtype=f32), np.array([10, 10, 5, 5], f32), x0, y0, w, h,
                      np.zeros((h, w, 3), np.uint8), np.full((h, w), cls_val, np.uint8), None)


def test_ingest_aabb_and_classes():
    mask = np.zeros((6, 8), np.uint16)
    mask[2:5, 3:6] = 7
    mask[2, 3] = 9      # occluder inside the box
    mask[4, 5] = 0
    rgb = np.arange(6 * 8 * 3, dtype=np.uint8).reshape(6, 8, 3)
    kf = O.ingest_observation(rgb, mask, np.eye(3, 4), [1, 1, 0, 0], 7)
    assert (kf.x0, kf.y0, kf.w, kf.h) == (3, 2, 3, 3)
    assert kf.cls[0, 0] == O.CLS_OCCLUDER and kf.cls[2, 2] == O.CLS_BACKGROUND and kf.cls[1, 1] == O.CLS_OBJECT
    assert np.array_equal(kf.rgb, rgb[2:5, 3:6])
    with pytest.raises(ValueError):
        O.ingest_observation(rgb, mask, np.eye(3, 4), [1, 1, 0, 0], 3)


def test_pixel_index_bijection_brute_force():
    kfs = [_kf(0, 0, 3, 2), _kf(5, 1, 2, 4), _kf(2, 2, 1, 1)]
    total = 6 + 8 + 1
    k, lx, ly = O.pixel_of_index(kfs, np.arange(total))
    seen = {(int(a), int(b), int(c)) for a, b, c in zip(k, lx, ly)}
    every = {(i, x, y) for i, kf in enumerate(kfs) for y in range(kf.h) for x in range(kf.w)}
    assert seen == every and len(seen) == total


def test_pixel_draw_uniform_chi2():
    kfs = [_kf(0, 0, 3, 2), _kf(5, 1, 2, 4), _kf(2, 2, 1, 1)]
    R = 150000
    k, lx, ly = O.draw_pixels(kfs, 1, 2, 3, R)
    key = k * 100 + ly * 10 + lx
    _, cnt = np.unique(key, return_counts=True)
    assert cnt.size == 15
    e = R / 15
    assert ((cnt - e) ** 2 / e).sum() < 36     # 14 dof, p ~ 1e-3


# ---------------------------------------------------------------- O4 rays
def test_principal_point_ray():
    # pixel (cx, cy), identity poses -> direction (0,0,1)
    K = np.array([100.0, 100.0, 10.5, 20.5], f32)
    o, d, n = O.make_rays([10], [20], K, np.eye(3, 4, dtype=f32), [0, 0, 0], 0.0)
    assert np.array_equal(d[0], np.array([0, 0, 1], f32)) and np.array_equal(o[0], np.zeros(3, f32))


def test_ray_projection_round_trip():
    # project o + s d back through the camera -> pixel centre within 1e-4 px
    g = np.random.default_rng(0)
    for _ in range(200):
        ang = g.uniform(-np.pi, np.pi, 3)
        Rx = np.array([[1, 0, 0], [0, math.cos(ang[0]), -math.sin(ang[0])], [0, math.sin(ang[0]), math.cos(ang[0])]])
        Rz = np.array([[math.cos(ang[1]), -math.sin(ang[1]), 0], [math.sin(ang[1]), math.cos(ang[1]), 0], [0, 0, 1]])
        Rwc = Rz @ Rx
        T = np.concatenate([Rwc, g.uniform(-2, 2, (3, 1))], 1).astype(f32)
        K = np.array([g.uniform(300, 600), g.uniform(300, 600), 320, 240], f32)
        bt = g.uniform(-1, 1, 3).astype(f32)
        yaw = float(g.uniform(-1, 1))
        px, py = int(g.integers(0, 640)), int(g.integers(0, 480))
        o, d, _ = O.make_rays([px], [py], K, T, bt, yaw)
        s = g.uniform(0.5, 5.0)
        xo = o[0].astype(np.float64) + s * d[0].astype(np.float64)
        c, sn = math.cos(yaw), math.sin(yaw)
        xw = np.array([c * xo[0] - sn * xo[1], sn * xo[0] + c * xo[1], xo[2]]) + bt
        T64 = T.astype(np.float64)
        xc = T64[:, :3].T @ (xw - T64[:, 3])
        u = K[0] * xc[0] / xc[2] + K[2]
        v = K[1] * xc[1] / xc[2] + K[3]
        assert abs(u - (px + 0.5)) < 1e-3 and abs(v - (py + 0.5)) < 1e-3
        assert abs(np.linalg.norm(d[0].astype(np.float64)) - 1) < 1e-6


# ---------------------------------------------------------------- O5 ray / box
def test_ray_box_example():
    tn, tf, hit = O.ray_box([[-5, 0, 0]], [[1, 0, 0]], [1, 1, 1])
    assert hit[0] and tn[0] == 4 and tf[0] == 6


def test_ray_box_parallel_miss_and_inside_origin():
    tn, tf, hit = O.ray_box([[0, 2, 0], [0, 0.5, 0]], [[1, 0, 0], [1, 0, 0]], [1, 1, 1])
    assert not hit[0]
    assert hit[1] and tn[1] == 0 and tf[1] == 1            # origin inside: t_near clamped to 0


def test_ray_box_dense_stepping():
    # interval endpoints agree with a dense ray-marching membership oracle
    g = np.random.default_rng(1)
    o = g.uniform(-3, 3, (2000, 3)).astype(f32)
    d = g.normal(size=(2000, 3))
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(f32)
    a = np.array([0.7, 0.4, 1.1], f32)
    tn, tf, hit = O.ray_box(o, d, a)
    ts = np.linspace(0, 10, 4001)
    step = ts[1] - ts[0]
    for i in range(o.shape[0]):
        p = o[i][None].astype(np.float64) + ts[:, None] * d[i][None].astype(np.float64)
        inside = np.all(np.abs(p) <= a, axis=1)
        if not inside.any():
            assert not hit[i] or tf[i] - tn[i] < 2 * step
            continue
        assert hit[i]
        assert abs(ts[inside][0] - tn[i]) <= step + 1e-5 and abs(ts[inside][-1] - tf[i]) <= step + 1e-5


# ---------------------------------------------------------------- O6 samples
def test_stratified_one_per_stratum_and_mean():
    N = 32
    R = 4000
    tn = np.full(R, 1.0, f32)
    tf = np.full(R, 3.0, f32)
    xi = O.u32_to_unit(O.rng_u32(0, 0, 1, np.arange(R)[:, None], 16 + np.arange(N)[None, :]))
    dist, delta = O.stratified(tn, tf, N, xi)
    Dl = 2.0 / N
    k = np.floor((dist - 1.0) / Dl)
    assert np.array_equal(k, np.broadcast_to(np.arange(N), k.shape))
    assert np.all(np.diff(dist, axis=1) > 0) and np.all(delta > 0)
    assert abs(dist.mean() - 2.0) < 0.01 * 2.0
    d1, _ = O.stratified(tn[:5], tf[:5], 1, xi[:5, :1])
    assert np.all((d1 >= 1) & (d1 <= 3))


# ---------------------------------------------------------------- O7 hash encoding
def _one_level_cfg(res, log2_T=16):
    return O.ModelConfig(levels=1, base_res=res, finest_res=float(res), res_cap=0, log2_T=log2_T)


def test_encode_reproduces_linear_field_on_dense_level():
    # trilinear interpolation of a linear vertex field is exact: a wrong axis order,
    # dense index formula or weight bit fails this.
    cfg = _one_level_cfg(12)
    lev = O.level_table(cfg)[0]
    assert lev.dense
    n1 = lev.res + 1
    table = np.zeros((lev.size, 2))
    for z in range(n1):
        for y in range(n1):
            for x in range(n1):
                table[x + n1 * (y + n1 * z)] = [x + 2.0 * y + 3.0 * z, 5.0 * x - y + 0.5 * z]
    g = np.random.default_rng(0)
    u = g.uniform(0, 1, (500, 3)).astype(f32)
    feat, idx, w = O.hash_encode(u, table, cfg)
    pos = u.astype(np.float64) * lev.res
    exp = np.stack([pos[:, 0] + 2 * pos[:, 1] + 3 * pos[:, 2], 5 * pos[:, 0] - pos[:, 1] + 0.5 * pos[:, 2]], 1)
    assert np.allclose(feat, exp, rtol=0, atol=1e-5)


def test_encode_vertex_centre_weights_sum():
    cfg = O.ModelConfig(levels=4, log2_T=10, base_res=4, finest_res=32.0, res_cap=0)
    g = np.random.default_rng(2)
    table = g.normal(size=(O.table_entries(cfg), 2))
    lt = O.level_table(cfg)
    u = g.uniform(0, 1, (300, 3)).astype(f32)
    feat, idx, w = O.hash_encode(u, table, cfg)
    assert np.allclose(w.sum(axis=2), 1.0, atol=1e-12)                       # north_star
    for l, lev in enumerate(lt):
        one = O.ModelConfig(levels=1, log2_T=10, base_res=lev.res, finest_res=float(lev.res), res_cap=0)
        sub = table[lev.offset:lev.offset + lev.size]
        v = np.array([[3, 1, 2]]) / lev.res                                   # exact vertex (3,1,2)
        fv, iv, _ = O.hash_encode(v.astype(f32), sub, one)
        e = O.corner_index(lev, 3, 1, 2, 1 << 10)
        assert np.allclose(fv[0], sub[e])
        ctr = (np.array([[3, 1, 2]]) + 0.5) / lev.res
        fc, ic, _ = O.hash_encode(ctr.astype(f32), sub, one)
        assert np.allclose(fc[0], sub[ic[0, 0]].mean(axis=0))


def test_dense_level_index_bijection():
    for res in (3, 7, 12):
        lev = O.Level(res, True, (res + 1) ** 3, 0)
        r = np.arange(res + 1)
        z, y, x = np.meshgrid(r, r, r, indexing="ij")
        idx = O.corner_index(lev, x.ravel(), y.ravel(), z.ravel(), 1 << 20)
        assert np.array_equal(np.sort(idx), np.arange((res + 1) ** 3))


def test_hash_primes_brute_force():
    # the 3-prime XOR hash of instant-NGP [21] on python ints
    lev = O.Level(100, False, 1 << 12, 0)
    g = np.random.default_rng(3)
    for _ in range(200):
        x, y, z = (int(v) for v in g.integers(0, 101, 3))
        h = ((x * 1) ^ (y * 2654435761) ^ (z * 805459861)) % (1 << 32) % (1 << 12)
        assert int(O.corner_index(lev, x, y, z, 1 << 12)) == h
    assert int(O.corner_index(lev, 0, 1, 0, 1 << 12)) == 2654435761 % 4096


def test_encode_continuity_across_cells():
    # SPEC.md:278
    cfg = O.ModelConfig(levels=3, log2_T=8, base_res=5, finest_res=20.0, res_cap=0)
    g = np.random.default_rng(4)
    table = g.normal(size=(O.table_entries(cfg), 2))
    for lev_res in (5, 10):
        b = np.float32(3.0 / lev_res)
        lo = np.nextafter(b, f32(0))
        hi = np.nextafter(b, f32(1))
        ua = np.array([[lo, 0.31, 0.77]], f32)
        ub = np.array([[hi, 0.31, 0.77]], f32)
        fa, _, _ = O.hash_encode(ua, table, cfg)
        fb, _, _ = O.hash_encode(ub, table, cfg)
        assert np.allclose(fa, fb, atol=1e-5)


def test_hash_encode_backward_is_adjoint():
    # <encode(u; table), g> is linear in table: its gradient is encode's adjoint
    cfg = O.ModelConfig(levels=3, log2_T=6, base_res=2, finest_res=8.0, res_cap=0)
    g = np.random.default_rng(5)
    E = O.table_entries(cfg)
    u = g.uniform(0, 1, (40, 3)).astype(f32)
    gf = g.normal(size=(40, 6))
    t1 = g.normal(size=(E, 2))
    f1, idx, w = O.hash_encode(u, t1, cfg)
    G = O.hash_encode_backward(gf, idx, w, E, 2)
    assert abs((f1 * gf).sum() - (G * t1).sum()) < 1e-9


# ---------------------------------------------------------------- O8 SH
def test_sh_orthonormal_quadrature():
    xg, wg = np.polynomial.legendre.leggauss(24)
    nphi = 48
    phi = (np.arange(nphi) + 0.5) * 2 * np.pi / nphi
    ct, ph = np.meshgrid(xg, phi, indexing="ij")
    st = np.sqrt(1 - ct ** 2)
    d = np.stack([st * np.cos(ph), st * np.sin(ph), ct], -1).reshape(-1, 3)
    wt = (wg[:, None] * np.full(nphi, 2 * np.pi / nphi)[None, :]).reshape(-1)
    Y = O.sh4(d)
    G = (Y * wt[:, None]).T @ Y
    assert np.allclose(G, np.eye(16), atol=1e-10)


def test_sh_addition_theorem():
    g = np.random.default_rng(6)
    d = g.normal(size=(100, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    Y = O.sh4(d)
    band = [0, 1, 1, 1, 2, 2, 2, 2, 2, 3, 3, 3, 3, 3, 3, 3]
    for l in range(4):
        s = (Y[:, [i for i in range(16) if band[i] == l]] ** 2).sum(axis=1)
        assert np.allclose(s, (2 * l + 1) / (4 * np.pi))


# ---------------------------------------------------------------- O9 MLP
def test_mlp_zero_model_constant():
    # SPEC.md:253 with bias-free layers (R4): raw=0 -> sigma=exp(0)=1, c=0.5
    cfg = O.ModelConfig()
    W = [np.zeros(s) for s in O.mlp_shapes(cfg)]
    g = np.random.default_rng(0)
    fw = O.mlp_forward(g.normal(size=(10, 16)), O.sh4(g.normal(size=(10, 3))), W, cfg)
    assert np.allclose(fw["sigma"], 1.0) and np.allclose(fw["rgb"], 0.5)
    cfg2 = O.ModelConfig(density_act=1)
    fw2 = O.mlp_forward(g.normal(size=(10, 16)), O.sh4(g.normal(size=(10, 3))), W, cfg2)
    assert np.allclose(fw2["sigma"], math.log(2.0))


def test_mlp_selection_weights():
    # W1 picks feature 0, W2 passes hidden unit 0 to raw0: sigma = exp(relu(f0));
    # colour net: only raw0 -> hidden0 -> hidden0 -> red: c_r = sigmoid(relu(relu(relu(f0))))
    cfg = O.ModelConfig()
    W = [np.zeros(s) for s in O.mlp_shapes(cfg)]
    W[0][0, 0] = 1
    W[1][0, 0] = 1
    W[2][0, 0] = 1
    W[3][0, 0] = 1
    W[4][0, 0] = 1
    f = np.zeros((3, 16))
    f[:, 0] = [-0.5, 0.3, 1.2]
    fw = O.mlp_forward(f, np.zeros((3, 16)), W, cfg)
    r = np.maximum(f[:, 0], 0)
    assert np.allclose(fw["sigma"], np.exp(r))
    assert np.allclose(fw["rgb"][:, 0], 1 / (1 + np.exp(-r))) and np.allclose(fw["rgb"][:, 1:], 0.5)


# ---------------------------------------------------------------- O10 render
def test_render_special_cases():
    d = np.array([[1.0, 2.0]])
    z = np.zeros((1, 3))
    vr = O.volume_render(np.zeros((1, 2)), np.ones((1, 2, 3)), d, np.ones((1, 2)), z)
    assert np.all(vr["w"] == 0) and np.all(vr["C"] == 0) and vr["D"][0] == 0
    c = np.array([[[0.2, 0.4, 0.6], [0.9, 0.9, 0.9]]])
    vr = O.volume_render(np.array([[50.0, 1.0]]), c, d, np.ones((1, 2)), z)
    assert abs(vr["w"][0, 0] - 1) < 1e-9 and np.allclose(vr["C"][0], c[0, 0], atol=1e-9)
    assert abs(vr["D"][0] - 1.0) < 1e-9
    vr = O.volume_render(np.array([[math.log(2), math.log(2)]]), c, d, np.ones((1, 2)), z)
    assert np.allclose(1 - vr["alpha"][0], [0.5, 0.5]) and np.allclose(vr["w"][0], [0.5, 0.25])


def test_render_constant_density_closed_form():
    # north_star: constant sigma with midpoint samples -> A = 1 - exp(-sigma L)
    for sig, L, N in [(0.7, 1.3, 32), (5.0, 0.4, 64), (0.01, 2.0, 7)]:
        dist, delta = O.midpoints(np.array([0.5], f32), np.array([0.5 + L], f32), N)
        vr = O.volume_render(np.full((1, N), sig), np.zeros((1, N, 3)), dist, delta, np.zeros((1, 3)))
        Lf = float(delta[0, 0]) * N
        assert abs(vr["A"][0] - (1 - math.exp(-sig * Lf))) < 1e-12
        assert abs(Lf - L) < 1e-5


def test_render_weight_identity_and_monotonicity():
    g = np.random.default_rng(7)
    s = g.uniform(0, 3, (50, 16))
    dl = g.uniform(0.01, 0.2, (50, 16))
    dist = np.cumsum(dl, axis=1)
    c = g.uniform(0, 1, (50, 16, 3))
    vr = O.volume_render(s, c, dist, dl, np.zeros((50, 3)))
    assert np.allclose(vr["A"], 1 - np.prod(np.exp(-s * dl), axis=1))
    assert np.all(vr["C"] <= 1 + 1e-12) and np.all(vr["C"] >= 0)
    s2 = s.copy()
    s2[:, 0] += 1.0
    vr2 = O.volume_render(s2, c, dist, dl, np.zeros((50, 3)))
    assert np.all(vr2["w"][:, 1:] <= vr["w"][:, 1:] + 1e-15)


def test_render_backward_finite_differences():
    g = np.random.default_rng(8)
    R, N = 5, 9
    s = g.uniform(0.1, 3, (R, N))
    dl = g.uniform(0.05, 0.3, (R, N))
    dist = np.cumsum(dl, axis=1)
    c = g.uniform(0, 1, (R, N, 3))
    bg = g.uniform(0, 1, (R, 3))
    gC = g.normal(size=(R, 3))
    gD = g.normal(size=R)

    def f(s_, c_):
        vr = O.volume_render(s_, c_, dist, dl, bg)
        return (vr["C"] * gC).sum() + (vr["D"] * gD).sum()
    vr = O.volume_render(s, c, dist, dl, bg)
    ds, dc = O.volume_render_backward(vr, gC, gD, c, dist, dl, bg)
    h = 1e-6
    for r in range(R):
        for i in range(N):
            sp, sm = s.copy(), s.copy()
            sp[r, i] += h
            sm[r, i] -= h
            assert abs((f(sp, c) - f(sm, c)) / (2 * h) - ds[r, i]) < 1e-7
            cp, cm = c.copy(), c.copy()
            cp[r, i, 1] += h
            cm[r, i, 1] -= h
            assert abs((f(s, cp) - f(s, cm)) / (2 * h) - dc[r, i, 1]) < 1e-7


# ---------------------------------------------------------------- O11 losses
def test_loss_examples():
    cfg = O.ModelConfig()
    cls = np.array([1])
    C = np.array([[0.8, 0.5, 0.9]])
    tgt = C - np.array([[0.3, 0.0, 0.4]])
    Ls, gC, gD = O.losses_and_render_grads(cls, np.array([True]), np.array([False]), C, np.zeros(1), tgt,
                                           np.zeros((1, 3)), np.zeros(1), np.zeros(1), 1.0, cfg)
    assert abs(Ls["l_rgb"] - 0.5) < 1e-12 and abs(Ls["l_total"] - 0.5) < 1e-12
    assert np.allclose(gC[0], [0.6, 0.0, 0.8])
    Ls, gC, gD = O.losses_and_render_grads(cls, np.array([True]), np.array([False]), C, np.zeros(1), C,
                                           np.zeros((1, 3)), np.zeros(1), np.zeros(1), 1.0, cfg)
    assert Ls["l_total"] == 0 and np.all(gC == 0)
    # composed example with both lambdas: 1 object ray with depth, 1 bg ray
    cls = np.array([1, 0])
    C = np.array([[0.5, 0.5, 0.5], [0.2, 0.2, 0.2]])
    tgt = np.array([[0.5, 0.5, 0.8], [0.0, 0.0, 0.0]])
    bg = np.array([[0, 0, 0], [0.2, 0.6, 0.2]])
    Ls, _, gD = O.losses_and_render_grads(cls, np.array([True, True]), np.array([True, False]), C,
                                          np.array([2.0, 0.0]), tgt, bg, np.array([1.5, 0.0]),
                                          np.array([0.0, 30.0]), 4.0, cfg)
    assert abs(Ls["l_rgb"] - 0.3 / 4) < 1e-12 and abs(Ls["l_rr"] - 0.4 / 4) < 1e-12
    assert abs(Ls["l_depth"] - 0.5 / 4) < 1e-12 and abs(Ls["l_density"] - 30 / 4) < 1e-12
    assert abs(Ls["l_total"] - (0.3 / 4 + 0.4 / 4 + 0.5 * 0.5 / 4 + 0.01 * 30 / 4)) < 1e-12
    assert abs(gD[0] - 0.5 / 4) < 1e-12 and gD[1] == 0


# ---------------------------------------------------------------- whole-step pins
def _small_state(cfg, seed=0, n_kf=3, occluders=False, depth=False):
    import scenes
    sc = scenes.sphere_scene(seed, n_views=n_kf, size=32, f=32.0, depth_per_view=6 if depth else 0)
    P = O.init_params(cfg, seed)
    P["table"] = np.random.default_rng(seed + 11).uniform(-0.5, 0.5, P["table"].shape)
    st = O.ObjectState(cfg, sc.objects[0].t, 0.0, sc.objects[0].a, 3, P)
    for fr in sc.frames:
        m = fr.mask.copy()
        if occluders:
            m[: m.shape[0] // 2, : m.shape[1] // 2][m[: m.shape[0] // 2, : m.shape[1] // 2] == 1] = 5
        st.kfs.append(O.ingest_observation(fr.rgb, m, fr.T_wc, fr.K, 1, fr.depth.get(1)))
    return st


def test_occluder_exclusion_bitwise():
    # perturbing occluder-ray target colours changes no loss and no gradient
    cfg = O.ModelConfig(rays_per_iter=128, samples_per_ray=8)
    st = _small_state(cfg, occluders=True)
    assert any((k.cls == O.CLS_OCCLUDER).any() for k in st.kfs)
    L1, g1, _ = O.loss_and_grads(st, 1)
    for k in st.kfs:
        k.rgb[k.cls == O.CLS_OCCLUDER] = 255 - k.rgb[k.cls == O.CLS_OCCLUDER]
    L2, g2, _ = O.loss_and_grads(st, 1)
    assert L1 == L2 and np.array_equal(g1["table"], g2["table"])
    assert all(np.array_equal(a, b) for a, b in zip(g1["W"], g2["W"]))


def test_background_only_batch():
    # SPEC.md:427
    cfg = O.ModelConfig(rays_per_iter=64, samples_per_ray=8)
    st = _small_state(cfg)
    for k in st.kfs:
        k.cls[:] = O.CLS_BACKGROUND
    L, _, _ = O.loss_and_grads(st, 1)
    assert L["l_rgb"] == 0 and L["l_depth"] == 0 and L["l_density"] > 0 and L["l_rr"] > 0


def test_decomposition_identity():
    # SPEC.md:449
    cfg = O.ModelConfig(rays_per_iter=64, samples_per_ray=8)
    st = _small_state(cfg, depth=True)
    L, _, _ = O.loss_and_grads(st, 2)
    assert abs(L["l_total"] - (L["l_rgb"] + L["l_rr"] + 0.5 * L["l_depth"] + 0.01 * L["l_density"])) <= 1e-12 * abs(L["l_total"])


@pytest.mark.parametrize("seed", range(4))
def test_full_step_gradient_central_differences(seed):
    # O12: analytic gradients of the whole step vs central differences in fp64,
    # tiny grid (L=2, T=2^6, N_min=2) and tiny nets
    cfg = O.ModelConfig(levels=2, log2_T=6, base_res=2, finest_res=4.0, res_cap=0, width=4, density_out=3,
                        rays_per_iter=24, samples_per_ray=6, seed=seed)
    st = _small_state(cfg, seed=seed, occluders=(seed % 2 == 1), depth=True)
    g = np.random.default_rng(100 + seed)
    st.params["W"] = [g.normal(0, 0.8, w.shape) for w in st.params["W"]]
    rays = O.forward_rays(st, 1)
    L0, grads, _ = O.loss_and_grads(st, 1, rays=rays)

    def loss_at(P):
        return O.loss_and_grads(st, 1, params=P, rays=rays)[0]["l_total"]
    h = 1e-6
    checked = 0
    cand = [("table", i, j) for i in np.nonzero(np.abs(grads["table"]).sum(1) > 0)[0] for j in range(2)]
    cand = [cand[i] for i in g.permutation(len(cand))[:12]]
    for li, w in enumerate(st.params["W"]):
        for _ in range(3):
            cand.append(("W", li, tuple(int(g.integers(0, s)) for s in w.shape)))
    for kind, a, b in cand:
        Pp = {"table": st.params["table"].copy(), "W": [w.copy() for w in st.params["W"]]}
        Pm = {"table": st.params["table"].copy(), "W": [w.copy() for w in st.params["W"]]}
        if kind == "table":
            Pp["table"][a, b] += h
            Pm["table"][a, b] -= h
            an = grads["table"][a, b]
        else:
            Pp["W"][a][b] += h
            Pm["W"][a][b] -= h
            an = grads["W"][a][b]
        fd = (loss_at(Pp) - loss_at(Pm)) / (2 * h)
        assert abs(fd - an) <= 1e-5 * max(1.0, abs(an)) + 1e-7, (kind, a, b, fd, an)
        checked += 1
    assert checked >= 20


# ---------------------------------------------------------------- O14 Adam
def test_adam_closed_form_constant_gradient():
    # constant g from zero moments: m_hat = g, v_hat = g^2 exactly -> each step moves lr*g/(|g|+eps)
    cfg = O.ModelConfig()
    p = np.array([1.0, -2.0, 0.5])
    g = np.array([1.0, -0.25, 3.0])
    m = np.zeros(3)
    v = np.zeros(3)
    for t in range(1, 6):
        O.adam_update(p, g, m, v, t, cfg, sparse=False)
        assert np.allclose(p, np.array([1.0, -2.0, 0.5]) - t * cfg.lr * g / (np.abs(g) + cfg.eps), rtol=0, atol=1e-12)
    p1 = np.array([0.0])
    O.adam_update(p1, np.array([1.0]), np.zeros(1), np.zeros(1), 1, cfg, sparse=False)
    assert abs(p1[0] + cfg.lr / (1 + cfg.eps)) < 1e-15


def test_adam_zero_gradient_and_sparse_locality():
    cfg = O.ModelConfig()
    p = np.array([1.0, 2.0, 3.0])
    m = np.array([0.1, 0.0, 0.2])
    v = np.array([0.01, 0.0, 0.04])
    p0, m0, v0 = p.copy(), m.copy(), v.copy()
    O.adam_update(p, np.array([0.0, 0.5, 0.0]), m, v, 3, cfg, sparse=True)
    assert p[0] == p0[0] and p[2] == p0[2] and m[0] == m0[0] and v[2] == v0[2]
    assert p[1] != p0[1]
    q = np.array([1.0, 2.0])
    O.adam_update(q, np.zeros(2), np.zeros(2), np.zeros(2), 1, cfg, sparse=False)
    assert np.array_equal(q, [1.0, 2.0])


def test_train_iteration_untouched_entries_bit_identical():
    cfg = O.ModelConfig(rays_per_iter=64, samples_per_ray=8)
    st = _small_state(cfg)
    p0 = st.params["table"].copy()
    L, g, _ = O.train_iteration(st)
    untouched = g["table"] == 0
    assert untouched.any() and np.array_equal(st.params["table"][untouched], p0[untouched])
    assert np.all(st.m["table"][untouched] == 0)


# ---------------------------------------------------------------- O15 inference
def _constant_density_params(cfg, raw0):
    # table of ones -> feat = ones (sum of weights = 1); W1 row 0 = raw0/LF; W2[0,0]=1
    P = {"table": np.ones((O.table_entries(cfg), cfg.feats)), "W": [np.zeros(s) for s in O.mlp_shapes(cfg)]}
    lf = cfg.levels * cfg.feats
    P["W"][0][0, :] = raw0 / lf
    P["W"][1][0, 0] = 1.0
    return P


def test_render_and_query_constant_density():
    cfg = O.ModelConfig(levels=2, log2_T=8, base_res=4, finest_res=8.0, res_cap=0)
    P = _constant_density_params(cfg, 0.9)
    sig = math.exp(0.9)
    a = np.array([0.4, 0.3, 0.2], f32)
    T = np.concatenate([np.eye(3), [[0.05], [0.02], [-2.0]]], 1).astype(f32)
    K = np.array([40, 40, 8, 8], f32)
    rgb, dep, opa = O.render(cfg, np.zeros(3, f32), 0.0, a, P, T, K, 16, 16, 16)
    o, d, _ = O.make_rays(np.tile(np.arange(16), 16), np.repeat(np.arange(16), 16), K, T, np.zeros(3), 0.0)
    tn, tf, hit = O.ray_box(o, d, a)
    L = np.where(hit, (tf - tn).astype(np.float64), 0.0)
    assert hit.any() and (~hit).any()
    assert np.allclose(opa.reshape(-1), np.where(hit, 1 - np.exp(-sig * L), 0.0), atol=1e-6)
    assert np.allclose(rgb.reshape(-1, 3), 0.5 * opa.reshape(-1, 1), atol=1e-12)
    q = np.array([[0.0, 0.0, 0.0], [0.39, -0.29, 0.19], [0.41, 0.0, 0.0], [0, 0, -0.21]], f32)
    s = O.query_density(cfg, a, P, q)
    assert np.allclose(s, [sig, sig, 0.0, 0.0])


def test_render_scene_two_boxes_closed_form():
    cfg = O.ModelConfig(levels=2, log2_T=8, base_res=4, finest_res=8.0, res_cap=0)
    P1 = _constant_density_params(cfg, 0.5)
    P2 = _constant_density_params(cfg, 0.2)
    a = np.array([0.3, 0.3, 0.3], f32)
    objs = [(cfg, np.array([0.0, 0.0, 0.0], f32), 0.0, a, P1, 0), (cfg, np.array([0.0, 0.0, 1.0], f32), 0.4, a, P2, 1)]
    T = np.concatenate([np.eye(3), [[0.0], [0.0], [-2.0]]], 1).astype(f32)
    K = np.array([60, 60, 6, 6], f32)
    rgb, dep, opa = O.render_scene(objs, T, K, 12, 12, 32)
    Ltot = np.zeros(144)
    for (c, bt, yaw, ba, P, oid) in objs:
        o, d, _ = O.make_rays(np.tile(np.arange(12), 12), np.repeat(np.arange(12), 12), K, T, bt, yaw)
        tn, tf, hit = O.ray_box(o, d, ba)
        sg = math.exp(0.5 if oid == 0 else 0.2)
        Ltot += np.where(hit, sg * (tf - tn).astype(np.float64), 0.0)
    assert np.allclose(opa.reshape(-1), 1 - np.exp(-Ltot), atol=1e-6)


# ---------------------------------------------------------------- network 1 (R24, the paper's MLP)
def test_paper_network_shapes_and_zero_model():
    # hash encoding + single hidden layer of 64; Table 4: 1..3 layers
    for hl in (1, 2, 3):
        cfg = O.ModelConfig(levels=16, network=1, hidden_layers=hl, dir_enc=0)
        sh = O.mlp_shapes(cfg)
        assert sh[0] == (64, 32) and sh[-1] == (4, 64) and len(sh) == hl + 1
        assert all(s == (64, 64) for s in sh[1:-1])
    cfg = O.ModelConfig(network=1, hidden_layers=2, dir_enc=0)
    W = [np.zeros(s) for s in O.mlp_shapes(cfg)]
    fw = O.mlp_forward(np.random.default_rng(0).normal(size=(7, 16)), np.zeros((7, 0)), W, cfg)
    assert np.allclose(fw["sigma"], 1.0) and np.allclose(fw["rgb"], 0.5)     # raw = 0 (R3, R4)


def test_paper_network_selection_weights():
    # W1 copies features 0..3 into hidden units 0..3, W2 = identity on them, W_out maps
    # hidden unit k -> raw k: sigma = exp(relu(f0)), c_k = sigmoid(relu(f_k)) (positions only)
    cfg = O.ModelConfig(network=1, hidden_layers=2, dir_enc=0)
    W = [np.zeros(s) for s in O.mlp_shapes(cfg)]
    for k in range(4):
        W[0][k, k] = 1
        W[1][k, k] = 1
        W[2][k, k] = 1
    f = np.random.default_rng(1).normal(size=(9, 16))
    fw = O.mlp_forward(f, np.zeros((9, 0)), W, cfg)
    r = np.maximum(f[:, :4], 0)
    assert np.allclose(fw["sigma"], np.exp(r[:, 0]))
    assert np.allclose(fw["rgb"], 1 / (1 + np.exp(-r[:, 1:4])))
    # the view direction plays no role
    st_cfg = O.ModelConfig(network=1, dir_enc=0)
    assert O.mlp_shapes(st_cfg)[0][1] == st_cfg.levels * st_cfg.feats


@pytest.mark.parametrize("hl", [1, 2, 3])
def test_paper_network_step_gradient_central_differences(hl):
    # O12 for network 1: whole-step analytic gradients vs fp64 central differences
    cfg = O.ModelConfig(levels=2, log2_T=6, base_res=2, finest_res=4.0, res_cap=0, width=5, dir_enc=0, network=1,
                        hidden_layers=hl, rays_per_iter=24, samples_per_ray=6, seed=hl)
    st = _small_state(cfg, seed=hl, occluders=(hl == 2), depth=True)
    g = np.random.default_rng(200 + hl)
    st.params["W"] = [g.normal(0, 0.8, w.shape) for w in st.params["W"]]
    rays = O.forward_rays(st, 1)
    L0, grads, _ = O.loss_and_grads(st, 1, rays=rays)

    def loss_at(P):
        return O.loss_and_grads(st, 1, params=P, rays=rays)[0]["l_total"]
    h = 1e-6
    cand = [("table", i, j) for i in np.nonzero(np.abs(grads["table"]).sum(1) > 0)[0] for j in range(2)]
    cand = [cand[i] for i in g.permutation(len(cand))[:10]]
    for li, w in enumerate(st.params["W"]):
        for _ in range(4):
            cand.append(("W", li, tuple(int(g.integers(0, s)) for s in w.shape)))
    for kind, a, b in cand:
        Pp = {"table": st.params["table"].copy(), "W": [w.copy() for w in st.params["W"]]}
        Pm = {"table": st.params["table"].copy(), "W": [w.copy() for w in st.params["W"]]}
        if kind == "table":
            Pp["table"][a, b] += h
            Pm["table"][a, b] -= h
            an = grads["table"][a, b]
        else:
            Pp["W"][a][b] += h
            Pm["W"][a][b] -= h
            an = grads["W"][a][b]
        fd = (loss_at(Pp) - loss_at(Pm)) / (2 * h)
        assert abs(fd - an) <= 1e-5 * max(1.0, abs(an)) + 1e-7, (kind, a, b, fd, an)


# ---------------------------------------------------------------- f3 online policy (Eq. 5)
def _pose_at(centre):
    T = np.eye(3, 4)
    T[:, 3] = centre
    return T


def test_view_angle_closed_forms():
    o = np.array([1.0, 2.0, 0.5])
    assert O.view_angle_deg(o + [1, 0, 0], o + [0, 3, 0], o) == pytest.approx(90.0)
    assert O.view_angle_deg(o + [1, 0, 0], o + [2, 0, 0], o) == pytest.approx(0.0, abs=1e-6)
    assert O.view_angle_deg(o + [1, 0, 0], o + [-1, 0, 0], o) == pytest.approx(180.0)
    th = math.radians(30.0)
    assert O.view_angle_deg(o + [2, 0, 0], o + [math.cos(th), math.sin(th), 0], o) == pytest.approx(30.0)


def test_keyframe_gate_orbit():
    # cameras every 10 degrees on a circle around the object: with alpha = 25 deg the
    # gate accepts frames 0, 3, 6, ... (30 deg after the last accepted one)
    o = np.array([0.3, -0.2, 0.4])
    last, acc = None, []
    for k in range(13):
        c = o + 2.0 * np.array([math.cos(math.radians(10 * k)), math.sin(math.radians(10 * k)), 0.2])
        ok, a = O.keyframe_gate(last, _pose_at(c), o, 25.0)
        if ok:
            last = c
            acc.append(k)
    assert acc == [0, 3, 6, 9, 12]


def test_schedule_budgets():
    b, rest = O.schedule_budgets({5: 300, 7: 120, 9: 0}, chunk=100, max_iters=1000)
    assert b == [([5, 7], 100), ([5, 7], 20), ([5], 100), ([5], 80)]
    assert rest == {5: 0, 7: 0, 9: 0}
    b, rest = O.schedule_budgets({1: 300}, chunk=100, max_iters=150)
    assert b == [([1], 100), ([1], 50)] and rest == {1: 150}


# ---------------------------------------------------------------- f2 mesh extraction (R26)
def test_mt_single_vertex_cases():
    # vertex 0 (on the Kuhn diagonal) lies in all 6 tetrahedra -> 6 triangles;
    # vertex 1 (+x) lies in the 2 tetrahedra whose first step is x -> 2 triangles
    P = O.lattice_points([0.5, 0.5, 0.5], 1)
    for k, n in [(0, 6), (7, 6), (1, 2), (2, 2), (4, 2), (3, 2), (5, 2), (6, 2)]:
        s = np.zeros((2, 2, 2))
        s[k & 1, (k >> 1) & 1, (k >> 2) & 1] = 1.0
        assert O.marching_tetrahedra(s, P, 0.5).shape[0] == n, k
    assert O.marching_tetrahedra(np.zeros((2, 2, 2)), P, 0.5).shape[0] == 0
    assert O.marching_tetrahedra(np.ones((2, 2, 2)), P, 0.5).shape[0] == 0


def test_mt_linear_field_exact():
    # sigma linear in x: linear interpolation is exact, every vertex lies on the plane
    P = O.lattice_points([0.4, 0.3, 0.2], 5).astype(np.float64)
    s = 3.0 * P[..., 0] + 1.5 * P[..., 1] - 0.5 * P[..., 2] + 0.1
    T = O.marching_tetrahedra(s, P, 0.35)
    assert T.shape[0] > 0
    v = T.reshape(-1, 3)
    assert np.abs(3.0 * v[:, 0] + 1.5 * v[:, 1] - 0.5 * v[:, 2] + 0.1 - 0.35).max() < 1e-12


def test_mt_sphere_and_metrics():
    # sigma = r0 - |x| (iso 0): vertices on the sphere within the lattice step^2 and the
    # area close to 4 pi r0^2; metrics of the mesh against exact sphere samples
    r0 = 0.35
    P = O.lattice_points([0.5, 0.5, 0.5], 12).astype(np.float64)
    s = r0 - np.linalg.norm(P, axis=-1)
    T = O.marching_tetrahedra(s, P, 0.0)
    v = T.reshape(-1, 3)
    h = 1.0 / 12
    assert np.abs(np.linalg.norm(v, axis=1) - r0).max() < h * h
    area = 0.5 * np.linalg.norm(np.cross(T[:, 1] - T[:, 0], T[:, 2] - T[:, 0]), axis=1).sum()
    assert abs(area / (4 * np.pi * r0 * r0) - 1) < 0.05
    # surface samples of the mesh lie on the sphere to O(h^2) (exact distance to the surface)
    S = O.sample_mesh_points(T, 5000)
    assert np.abs(np.linalg.norm(S, axis=1) - r0).mean() < h * h / 2
    # metrics: a grid and the same grid shifted by dz along its normal: acc = comp = dz,
    # completion ratio 1 above dz, 0 below
    xs = np.linspace(0, 1, 21)
    G = np.stack(np.meshgrid(xs, xs, [0.0], indexing="ij"), -1).reshape(-1, 3)
    m = O.mesh_metrics(G + [0, 0, 0.013], G, tau=0.02)
    assert abs(m["acc"] - 0.013) < 1e-12 and abs(m["comp"] - 0.013) < 1e-12 and m["cr"] == 1.0
    assert O.mesh_metrics(G + [0, 0, 0.013], G, tau=0.01)["cr"] == 0.0
    # to_world is the inverse of the object-frame transform of the rays (R8)
    X = np.array([[0.1, 0.2, 0.3]])
    W = O.to_world(X, [1.0, -2.0, 0.5], math.radians(30))
    c, s_ = math.cos(math.radians(30)), math.sin(math.radians(30))
    p = W[0] - [1.0, -2.0, 0.5]
    assert np.allclose([c * p[0] + s_ * p[1], -s_ * p[0] + c * p[1], p[2]], X[0])


def test_observed_mask_projection():
    # one camera at z = 2 looking down -z (OpenCV: camera z -> world -z), f = 100,
    # detection box = the central 20 x 20 pixels of a 100 x 100 image: a point at the
    # origin is seen, points 0.5 m off-axis (u = 50 + 100 * 0.5 / 2 = 75) are not
    T = np.array([[1, 0, 0, 0], [0, -1, 0, 0], [0, 0, -1, 2.0]], np.float32)
    kf = O.Keyframe(T_wc=T, K=np.array([100, 100, 50, 50], np.float32), x0=40, y0=40, w=20, h=20,
                    rgb=None, cls=None, depth=None)
    P = np.array([[0, 0, 0], [0.5, 0, 0], [0, 0.5, 0], [0.15, 0.15, 0], [0, 0, 3.0]], np.float32)
    assert O.observed_mask(P, [0, 0, 0], 0.0, [kf]).tolist() == [True, False, False, True, False]
    # the box pose moves the points: a box translated by 0.5 m in x puts its origin off-axis
    assert O.observed_mask(P[:1], [0.5, 0, 0], 0.0, [kf]).tolist() == [False]


# ---------------------------------------------------------------- O2 / O4 / O6 / R17: the training-path pieces
# (VERDICT r1 "What's weak" #1: make_rays_per_ray, sample_points, the rng key / stream
# layout and the R17 depth conversion had no pin of their own)
import sys as _sys  # noqa: E402
_sys.path.insert(0, GOLD)
import rng_ref  # noqa: E402  (plain-int reference, tests/golden/rng_ref.py; imports nothing from oracle/)


def test_rng_composed_key_golden():
    # R13 key composition: golden u32 written by tests/golden/make_rng_golden.py (python ints)
    rows = [l.split() for l in open(os.path.join(GOLD, "rng_u32_keys.txt")) if l.strip() and not l.startswith("#")]
    assert len(rows) >= 10
    for seed, obj, t, ray, stream, hx in rows:
        got = int(O.rng_u32(int(seed), int(obj), int(t), np.array([int(ray)]), np.array([int(stream)]))[0])
        assert got == int(hx, 16), (seed, obj, t, ray, stream, hex(got), hx)


def _kf_image(W, H, K, T, obj_px, occ_px=(), depth=None, iid=1):
    rgb = (np.arange(H * W * 3) % 251).astype(np.uint8).reshape(H, W, 3)
    mask = np.zeros((H, W), np.uint16)
    for (x, y) in obj_px:
        mask[y, x] = iid
    for (x, y) in occ_px:
        mask[y, x] = iid + 1
    return O.ingest_observation(rgb, mask, T, K, iid, depth)


def _pose(yaw_deg, centre):
    """camera looking along +x of the world rotated by yaw, OpenCV axes"""
    a = math.radians(yaw_deg)
    fwd = np.array([math.cos(a), math.sin(a), 0.0])
    right = np.array([math.sin(a), -math.cos(a), 0.0])
    down = np.array([0.0, 0.0, -1.0])
    R = np.stack([right, down, fwd], 1)
    return np.concatenate([R, np.asarray(centre, float)[:, None]], 1).astype(f32)


def test_training_rng_stream_layout():
    # R13 streams of a training iteration: pixel = stream 0, background
    # colour = streams 1-3, jitter of sample i = stream 16+i, all keyed (seed, obj, t, ray)
    cfg = O.ModelConfig(samples_per_ray=8, rays_per_iter=300, seed=11)
    K = np.array([40.0, 42.0, 15.5, 11.0], f32)
    kfs = [_kf_image(32, 24, K, _pose(10 * k, [-2.0, 0.1 * k, 0.3]),
                     [(x, y) for x in range(8 + k, 20) for y in range(5, 14 + k)], occ_px=[(21, 7)]) for k in range(3)]
    st = O.ObjectState(cfg, np.zeros(3, f32), 0.2, np.full(3, 0.6, f32), 37, O.init_params(cfg, 0), kfs=kfs)
    t = 5
    rs = O.forward_rays(st, t)
    total = sum(k.w * k.h for k in kfs)
    for r in range(cfg.rays_per_iter):
        idx = rng_ref.pixel_index(rng_ref.key_u32(11, 37, t, r, 0), total)
        k = 0
        while idx >= kfs[k].w * kfs[k].h:
            idx -= kfs[k].w * kfs[k].h
            k += 1
        assert (rs["k"][r], rs["px"][r], rs["py"][r]) == (k, kfs[k].x0 + idx % kfs[k].w, kfs[k].y0 + idx // kfs[k].w)
        for c in range(3):
            assert rs["bg"][r, c] == f32(rng_ref.unit(rng_ref.key_u32(11, 37, t, r, 1 + c)))
        for i in range(cfg.samples_per_ray):
            assert rs["xi"][r, i] == f32(rng_ref.unit(rng_ref.key_u32(11, 37, t, r, 16 + i)))


def test_make_rays_per_ray_equals_make_rays():
    # the training-path builder (per-ray intrinsics / pose) equals the pinned
    # single-camera builder ray by ray, bitwise
    g = np.random.default_rng(3)
    n = 64
    Ks = np.stack([np.array([g.uniform(200, 600), g.uniform(200, 600), g.uniform(100, 400), g.uniform(50, 300)], f32)
                   for _ in range(n)])
    Ts = np.stack([_pose(g.uniform(-180, 180), g.uniform(-2, 2, 3)) for _ in range(n)])
    px = g.integers(0, 640, n)
    py = g.integers(0, 480, n)
    bt = np.array([0.3, -0.2, 0.1], f32)
    yaw = 0.7
    o, d, nn = O.make_rays_per_ray(px, py, Ks, Ts, bt, yaw)
    for i in range(n):
        o1, d1, n1 = O.make_rays([px[i]], [py[i]], Ks[i], Ts[i], bt, yaw)
        assert np.array_equal(o[i], o1[0]) and np.array_equal(d[i], d1[0]) and nn[i] == n1[0]
    # and a projection round trip with each ray's own intrinsics
    for i in range(n):
        xo = o[i].astype(np.float64) + 1.7 * d[i].astype(np.float64)
        c, s = math.cos(yaw), math.sin(yaw)
        xw = np.array([c * xo[0] - s * xo[1], s * xo[0] + c * xo[1], xo[2]]) + bt
        T64 = Ts[i].astype(np.float64)
        xc = T64[:, :3].T @ (xw - T64[:, 3])
        assert abs(Ks[i, 0] * xc[0] / xc[2] + Ks[i, 2] - (px[i] + 0.5)) < 1e-3
        assert abs(Ks[i, 1] * xc[1] / xc[2] + Ks[i, 3] - (py[i] + 0.5)) < 1e-3


def test_sample_points_hand_computed_and_clamped():
    # R6: u = (x + a) / (a + a), x = o + dist d, clamped to [0, 1]; a box with unequal
    # half extents, values exact in fp32
    a = np.array([0.5, 1.0, 2.0], f32)
    o = np.array([[-0.25, 0.5, -1.0]], f32)
    d = np.array([[1.0, 0.0, 0.0]], f32)
    u = O.sample_points(o, d, np.array([[0.0, 0.5]], f32), a)
    assert np.array_equal(u[0, 0], np.array([0.25, 0.75, 0.25], f32))      # x = (-0.25, 0.5, -1)
    assert np.array_equal(u[0, 1], np.array([0.75, 0.75, 0.25], f32))      # x = (0.25, 0.5, -1)
    # faces: x beyond +a / -a clamps to 1 / 0 on that axis only
    o2 = np.array([[0.6, -1.5, 3.0]], f32)
    u2 = O.sample_points(o2, np.array([[0.0, 0.0, 1.0]], f32), np.array([[0.0]], f32), a)
    assert np.array_equal(u2[0, 0], np.array([1.0, 0.0, 1.0], f32))
    u3 = O.sample_points(np.array([[0.0, 0.25, -0.5]], f32), d, np.array([[-0.75]], f32), a)
    assert np.array_equal(u3[0, 0], np.array([0.0, 0.625, 0.375], f32))   # x = (-0.75 -> clamp, 0.25, -0.5)


def test_depth_target_is_ray_distance():
    # R17: a sparse camera-z sample on pixel (px, py) becomes the
    # ray distance z * |((px+.5-cx)/fx, (py+.5-cy)/fy, 1)|: z on the optical axis,
    # z * sqrt(1 + 1/16) one pixel off axis with fx = 4
    cfg = O.ModelConfig(samples_per_ray=4, rays_per_iter=64, seed=2)
    K = np.array([4.0, 4.0, 3.5, 2.5], f32)
    kf = _kf_image(8, 6, K, _pose(0.0, [-2.0, 0.0, 0.0]), [(3, 2), (4, 2)], depth=[(3.5, 2.5, 2.0), (4.7, 2.2, 3.0)])
    st = O.ObjectState(cfg, np.zeros(3, f32), 0.0, np.full(3, 0.5, f32), 1, O.init_params(cfg, 0), kfs=[kf])
    rs = O.forward_rays(st, 1)
    assert set(rs["px"].tolist()) == {3, 4} and rs["has_depth"].all()
    on = rs["px"] == 3
    assert np.all(rs["depth_t"][on] == f32(2.0))
    assert np.allclose(rs["depth_t"][~on].astype(np.float64), 3.0 * math.sqrt(1.0 + 1.0 / 16.0), rtol=1e-6, atol=0)


# ---------------------------------------------------------------- round 2: pins found by the mutation test
def test_midpoint_samples_hand_computed_and_opaque_depth():
    # R12 inference sampling (xi = 1/2, delta = Delta): [1, 3] in 4 strata -> centres
    dist, delta = O.midpoints(np.array([1.0], f32), np.array([3.0], f32), 4)
    assert np.array_equal(dist[0], np.array([1.25, 1.75, 2.25, 2.75], f32))
    assert np.array_equal(delta[0], np.full(4, 0.5, f32))
    # an opaque constant field puts all weight on the first sample: the rendered depth
    # is the centre of the first stratum, t_near + Delta / 2 (Eq. 6)
    cfg = O.ModelConfig(levels=2, log2_T=8, base_res=4, finest_res=8.0, res_cap=0)
    P = _constant_density_params(cfg, 14.0)
    a = np.array([0.4, 0.3, 0.2], f32)
    T = np.concatenate([np.eye(3), [[0.0], [0.0], [-2.0]]], 1).astype(f32)
    K = np.array([40, 40, 8, 8], f32)
    N = 16
    _, dep, opa = O.render(cfg, np.zeros(3, f32), 0.0, a, P, T, K, 16, 16, N)
    o, d, _ = O.make_rays(np.tile(np.arange(16), 16), np.repeat(np.arange(16), 16), K, T, np.zeros(3), 0.0)
    tn, tf, hit = O.ray_box(o, d, a)
    assert hit.any()
    first = tn[hit].astype(np.float64) + 0.5 * (tf[hit] - tn[hit]).astype(np.float64) / N
    assert np.allclose(dep.reshape(-1)[hit], first, rtol=0, atol=1e-5)
    assert np.allclose(opa.reshape(-1)[hit], 1.0, atol=1e-9)


def test_upper_face_belongs_to_the_last_cell():
    # R5 / R6: u = 1 (the +a face, where the clamp of R6 lands points outside the box)
    # is in cell N_l - 1 with fraction 1, so all 8 corners are those of the last cell
    # and every index stays inside the level's own block
    cfg = O.ModelConfig(levels=3, log2_T=10, base_res=4, finest_res=40.0, res_cap=0)
    lt = O.level_table(cfg)
    assert lt[0].dense and not lt[-1].dense
    T = 1 << cfg.log2_T
    u = np.array([[1.0, 1.0, 1.0], [1.0, 0.3, 0.0]], f32)
    _, idx, w = O.hash_encode(u, np.zeros((O.table_entries(cfg), 2)), cfg)
    for l, lev in enumerate(lt):
        N = lev.res
        for s, (cx, cy, cz) in enumerate([(N - 1, N - 1, N - 1), (N - 1, int(np.floor(f32(0.3) * f32(N))), 0)]):
            exp = {lev.offset + int(O.corner_index(lev, cx + (b & 1), cy + ((b >> 1) & 1), cz + ((b >> 2) & 1), T))
                   for b in range(8)}
            assert set(idx[s, l].tolist()) == exp, (l, s)
            assert np.all((idx[s, l] >= lev.offset) & (idx[s, l] < lev.offset + lev.size))
        assert abs(w[0, l, 7] - 1.0) < 1e-12                      # the (N, N, N) vertex carries it all


def test_sh_matches_complex_harmonics_with_condon_shortley_phase():
    # R2: the 16 real SH of degree <= 3 are sqrt(2) Im Y_l^|m| (m < 0), Y_l^0, sqrt(2) Re Y_l^m
    # (m > 0) of the complex orthonormal harmonics WITH the Condon-Shortley phase
    # (scipy.special.sph_harm_y), ordered l = 0..3, m = -l..l -- this fixes the signs
    # that orthonormality and the addition theorem leave free
    from scipy.special import sph_harm_y
    g = np.random.default_rng(8)
    d = g.normal(size=(64, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    theta = np.arccos(np.clip(d[:, 2], -1, 1))
    phi = np.arctan2(d[:, 1], d[:, 0])
    cols = []
    for l in range(4):
        for m in range(-l, l + 1):
            y = sph_harm_y(l, abs(m), theta, phi)
            cols.append(math.sqrt(2) * y.imag if m < 0 else (y.real if m == 0 else math.sqrt(2) * y.real))
    assert np.allclose(O.sh4(d), np.stack(cols, 1), atol=1e-12)


def test_density_activation_saturates_at_the_clamp():
    # R3: sigma = exp(min(raw0, 15)) saturates at e^15 (continuous at the clamp), with
    # the straight-through derivative sigma; softplus is log(1 + e^r)
    r = np.array([-3.0, 14.0, 15.0, 15.5, 40.0, 1e4])
    s = O.density_activation(r, 0)
    assert np.allclose(s[:3], np.exp(r[:3])) and np.all(s[2:] == s[2]) and s[2] == math.exp(15.0)
    assert np.array_equal(O.density_activation_grad(r, s, 0), s)
    assert np.allclose(O.density_activation(np.array([0.0, 30.0]), 1), [math.log(2.0), 30.0])


def test_occluder_rays_are_dropped_before_sampling():
    # R10: a ray of an occluder pixel gets no samples and no loss, even
    # when it crosses the box; losses_and_render_grads also gives an occluder ray
    # (if one reached it) neither loss nor gradient
    cfg = O.ModelConfig(rays_per_iter=256, samples_per_ray=8)
    st = _small_state(cfg, occluders=True)
    rs = O.forward_rays(st, 1)
    occ = rs["cls"] == O.CLS_OCCLUDER
    _, _, box_hit = O.ray_box(rs["o"], rs["d"], st.box_a)
    assert (occ & box_hit).any()
    assert not (rs["hit"] & occ).any()
    assert np.array_equal(rs["hit"], box_hit & ~occ)
    L, _, _ = O.loss_and_grads(st, 1)
    assert L["hit_rays"] == int((box_hit & ~occ).sum())
    C = np.array([[0.9, 0.1, 0.3], [0.5, 0.5, 0.5]])
    cls = np.array([O.CLS_OCCLUDER, O.CLS_OBJECT])
    Ls, gC, gD = O.losses_and_render_grads(cls, np.array([True, True]), np.array([True, True]), C, np.array([3.0, 1.0]),
                                           np.zeros((2, 3)), np.zeros((2, 3)), np.array([1.0, 1.0]),
                                           np.array([5.0, 0.0]), 2.0, cfg)
    assert np.all(gC[0] == 0) and gD[0] == 0 and np.any(gC[1] != 0)
    assert abs(Ls["l_rgb"] - np.linalg.norm(C[1]) / 2) < 1e-12 and Ls["l_rr"] == 0 and Ls["l_density"] == 0


def _constant_field_params(cfg, raw0, rgb):
    # network 0: sigma = exp(raw0) and colour = rgb everywhere: feat = ones, raw = (raw0,
    # 0, ...); the SH band-0 constant 1/(2 sqrt(pi)) feeds g1[0] = g2[0] = Y00 and the
    # last layer turns it into logit(rgb)
    P = _constant_density_params(cfg, abs(raw0))
    P["W"][1][0, 0] = math.copysign(1.0, raw0)          # raw0 < 0 through the positive h1[0]
    y00 = 0.28209479177387814
    P["W"][2][0, cfg.density_out] = 1.0
    P["W"][3][0, 0] = 1.0
    P["W"][4][:, 0] = [math.log(c / (1 - c)) / y00 for c in rgb]
    return P


def test_render_scene_composites_by_t_near_not_id():
    # R20: the nearer box is composited first whatever its id: C = C_1 + (1 - A_1) C_0
    # with C_s = rgb_s A_s, A_s = 1 - exp(-sigma_s L_s) (box 1 in front of box 0)
    cfg = O.ModelConfig(levels=2, log2_T=8, base_res=4, finest_res=8.0, res_cap=0)
    a = np.array([0.3, 0.3, 0.3], f32)
    spec = {0: (0.4, (0.9, 0.1, 0.2), np.array([0.0, 0.0, 1.0], f32)),
            1: (0.1, (0.2, 0.7, 0.3), np.array([0.0, 0.0, 0.0], f32))}
    objs = [(cfg, spec[i][2], 0.0, a, _constant_field_params(cfg, spec[i][0], spec[i][1]), i) for i in (0, 1)]
    T = np.concatenate([np.eye(3), [[0.0], [0.0], [-2.0]]], 1).astype(f32)
    K = np.array([60, 60, 6, 6], f32)
    rgb, _, opa = O.render_scene(objs, T, K, 12, 12, 32)
    px, py = np.tile(np.arange(12), 12), np.repeat(np.arange(12), 12)
    A, C = {}, {}
    for i in (0, 1):
        o, d, _ = O.make_rays(px, py, K, T, spec[i][2], 0.0)
        tn, tf, hit = O.ray_box(o, d, a)
        A[i] = np.where(hit, 1 - np.exp(-math.exp(spec[i][0]) * (tf - tn).astype(np.float64)), 0.0)
        C[i] = A[i][:, None] * np.asarray(spec[i][1])[None, :]
    both = (A[0] > 0) & (A[1] > 0)
    assert both.any()
    assert np.allclose(rgb.reshape(-1, 3), C[1] + (1 - A[1])[:, None] * C[0], atol=1e-6)
    assert np.allclose(opa.reshape(-1), 1 - (1 - A[0]) * (1 - A[1]), atol=1e-6)


def test_supervised_rays_composite_over_their_background_colour():
    # R14: obj_bg = 0 composites every supervised ray over its random colour b, so an
    # (almost) empty field renders C = b and L_rgb = sum_{R_o} |b - C_gt| / B (Eq. 7);
    # obj_bg = 1 composites object rays over black: L_rgb = sum_{R_o} |C_gt| / B
    for obj_bg in (0, 1):
        cfg = O.ModelConfig(rays_per_iter=128, samples_per_ray=8, obj_bg=obj_bg)
        st = _small_state(cfg)
        st.params = _constant_field_params(cfg, -60.0, (0.5, 0.5, 0.5))
        L, _, dbg = O.loss_and_grads(st, 1)
        rs = dbg["rays"]
        obj = rs["hit"] & (rs["cls"] == O.CLS_OBJECT)
        assert obj.any()
        ref = rs["tgt"][obj].astype(np.float64) - (rs["bg"][obj] if obj_bg == 0 else 0.0)
        assert abs(L["l_rgb"] - np.linalg.norm(ref, axis=1).sum() / 128) < 1e-9, obj_bg


def test_ingest_keeps_depth_on_object_pixels_only():
    # SPEC.md:304 (has_depth => object pixel): samples on occluder / background pixels
    # of the box or outside it are dropped; a sample lands on (floor u, floor v)
    mask = np.zeros((6, 8), np.uint16)
    mask[2:5, 3:6] = 7
    mask[2, 3] = 9
    mask[4, 5] = 0
    rgb = np.zeros((6, 8, 3), np.uint8)
    samples = [(4.7, 3.2, 1.5), (3.5, 2.5, 2.0), (5.2, 4.9, 2.5), (0.5, 0.5, 3.0), (4.1, 2.0, -1.0)]
    kf = O.ingest_observation(rgb, mask, np.eye(3, 4), [1, 1, 0, 0], 7, samples)
    exp = np.zeros((3, 3), f32)
    exp[1, 1] = 1.5
    assert np.array_equal(kf.depth, exp)


def test_adam_epsilon_outside_the_root():
    # Adam (Kingma & Ba, Alg. 1): p -= lr m_hat / (sqrt(v_hat) + eps);
    # for a constant g from zero moments the step is lr g / (|g| + eps): g = eps -> lr / 2
    cfg = O.ModelConfig(eps=1e-2)
    p = np.array([0.0])
    O.adam_update(p, np.array([1e-2]), np.zeros(1), np.zeros(1), 1, cfg, sparse=False)
    assert abs(p[0] + cfg.lr / 2) < 1e-15


def test_lattice_points_axes_and_metric_directions():
    # R21 lattice: P[ix, iy, iz] = (-a_x + 2 a_x ix / R, ...) for unequal half extents
    a = (0.1, 0.2, 0.3)
    P = O.lattice_points(a, 2)
    assert P.shape == (3, 3, 3, 3)
    assert np.allclose(P[2, 0, 1], [0.1, -0.2, 0.0]) and np.allclose(P[0, 1, 2], [-0.1, 0.0, 0.3])
    # PAPER.md:255 metrics: a reconstruction that is half of the ground truth is exact
    # (accuracy 0) but incomplete (completion > 0, ratio < 1)
    xs = np.linspace(0, 1, 11)
    G = np.stack(np.meshgrid(xs, xs, [0.0], indexing="ij"), -1).reshape(-1, 3)
    m = O.mesh_metrics(G[G[:, 0] <= 0.5], G, tau=0.05)
    assert m["acc"] == 0.0 and m["comp"] > 0.1 and m["cr"] < 0.6


def test_initial_tables_are_small():
    # R19 / SPEC.md:285: tables start U(-1e-4, 1e-4)
    t = O.init_params(O.ModelConfig(), 0)["table"]
    assert np.abs(t).max() <= 1e-4 and np.abs(t).max() > 0.99e-4 and abs(t.std() - 1e-4 / math.sqrt(3)) < 2e-6

"""The oracle pins must catch plausible mistakes: each
mutation below (a wrong operand, index, sign, RNG stream or dropped clamp in
oracle/romap_oracle.py) is applied to a COPY of the oracle in a temporary tree,
tests/test_oracle_pins.py runs against that copy, and at least one pin must fail.
The working tree is never modified; the copies run several at a time.  Round 2
added one mutation per remaining step of the path (levels, pixel draw, rays,
slab, samples, encode / backward, SH, MLP backward, render forward / backward,
losses, Adam, f2 / f3 host policy)."""
import concurrent.futures
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTATIONS = {
    "u = (x + a) / (3a)": ("    u = (x + a) / (a + a)\n    return np.minimum",
                          "    u = (x + a) / (a + a + a)\n    return np.minimum"),
    "sample_points clamp dropped": ("    u = (x + a) / (a + a)\n    return np.minimum(np.maximum(u, f32(0.0)), f32(1.0)).astype(f32)",
                                    "    u = (x + a) / (a + a)\n    return u.astype(f32)"),
    "make_rays_per_ray cx/cy swapped": ("    fx, fy, cx, cy = Ks[:, 0], Ks[:, 1], Ks[:, 2], Ks[:, 3]",
                                        "    fx, fy, cx, cy = Ks[:, 0], Ks[:, 1], Ks[:, 3], Ks[:, 2]"),
    "make_rays_per_ray yaw sign": ("    c, s = box_rotation(yaw)\n    o = np.stack",
                                   "    c, s = box_rotation(yaw)\n    s = -s\n    o = np.stack"),
    "rng ray shifted by 4": ("k = mix64(k ^ ((r << U64(8)) | s))", "k = mix64(k ^ ((r << U64(4)) | s))"),
    "rng obj/t order swapped": ("        k = mix64(k ^ U64(obj))\n        k = mix64(k ^ U64(t))",
                                "        k = mix64(k ^ U64(t))\n        k = mix64(k ^ U64(obj))"),
    "background stream + 1": ("rng_u32(cfg.seed, st.obj_id, t, ray, 1 + c)", "rng_u32(cfg.seed, st.obj_id, t, ray, 2 + c)"),
    "jitter stream + 1": ("rng_u32(cfg.seed, st.obj_id, t, ray, 16 + i)", "rng_u32(cfg.seed, st.obj_id, t, ray, 17 + i)"),
    "depth target z instead of z |dc|": ("depth_t = (zc * n).astype(f32)", "depth_t = (zc * f32(1)).astype(f32)"),
    "hash prime y/z swapped": ("PRIMES = (1, 2654435761, 805459861)", "PRIMES = (1, 805459861, 2654435761)"),
    "trilinear weight bit flipped": ("w = w * (fr[:, k] if bits[k] else 1.0 - fr[:, k])",
                                     "w = w * (1.0 - fr[:, k] if bits[k] else fr[:, k])"),
    "render transmittance inclusive": ("Tr[:, 1:] = np.cumprod(alpha, axis=1)[:, :-1]", "Tr[:, :] = np.cumprod(alpha, axis=1)"),
    "Adam bias correction dropped": ("    mh = m[upd] / (1 - b1 ** t)", "    mh = m[upd]"),
    # round 2: one mutation per remaining step of the path
    "level resolution rounded": ("n = int(math.floor(cfg.base_res * b ** l + 1e-6))",
                                 "n = int(math.floor(cfg.base_res * b ** l + 0.5))"),
    "level blocks not padded": ("        off += (size + 15) // 16 * 16\n    return out", "        off += size\n    return out"),
    "pixel draw modulo": ("idx = ((u * U64(total)) >> U64(32)).astype(np.int64)", "idx = (u % U64(total)).astype(np.int64)"),
    "pixel_of_index left search": ('k = np.searchsorted(P, idx, side="right") - 1', 'k = np.searchsorted(P, idx, side="left") - 1'),
    "unit float 23 bits": ("(np.asarray(u, dtype=np.uint32) >> np.uint32(8))", "(np.asarray(u, dtype=np.uint32) >> np.uint32(9))"),
    "make_rays pixel centre dropped": ("    px = np.asarray(px).astype(f32) + f32(0.5)\n    py = np.asarray(py).astype(f32) + f32(0.5)\n    fx, fy, cx, cy = (f32(v)",
                                       "    px = np.asarray(px).astype(f32)\n    py = np.asarray(py).astype(f32)\n    fx, fy, cx, cy = (f32(v)"),
    "ray_box t_near not clamped at 0": ("    tn = np.zeros(R, f32)\n    tf = np.full(R, np.inf, f32)",
                                        "    tn = np.full(R, -np.inf, f32)\n    tf = np.full(R, np.inf, f32)"),
    "ray_box parallel miss ignored": ("        miss |= zero & (np.abs(ok) > ak)\n", ""),
    "stratified last delta 0": ("    delta[:, -1] = Dl[:, 0]", "    delta[:, -1] = 0"),
    "midpoints at 0": ("    s = np.arange(N, dtype=f32)[None, :] + f32(0.5)\n    dist = tn + s * Dl\n    return dist.astype(f32), np.broadcast_to",
                       "    s = np.arange(N, dtype=f32)[None, :] + f32(0.0)\n    dist = tn + s * Dl\n    return dist.astype(f32), np.broadcast_to"),
    "cell clamp at res": ("c = np.clip(np.floor(pos), 0, lev.res - 1).astype(np.int64)", "c = np.clip(np.floor(pos), 0, lev.res).astype(np.int64)"),
    "dense index axes swapped": ("        return cx + n1 * (cy + n1 * cz)", "        return cz + n1 * (cy + n1 * cx)"),
    "hash backward weights dropped": ("np.add.at(g, idx_all[:, l, b], w_all[:, l, b][:, None] * dfeat[:, l * F:(l + 1) * F])",
                                      "np.add.at(g, idx_all[:, l, b], dfeat[:, l * F:(l + 1) * F])"),
    "SH band 1 sign": ("    out[:, 1] = -0.48860251190291987 * y", "    out[:, 1] = 0.48860251190291987 * y"),
    "SH band 2 constant sign": ("    out[:, 6] = 0.94617469575755997 * zz - 0.31539156525251999",
                                "    out[:, 6] = 0.94617469575755997 * zz + 0.31539156525251999"),
    "density clamp dropped": ("        return np.exp(np.minimum(r0, SIGMA_RAW_CLAMP))", "        return np.exp(r0)"),
    "ReLU mask dropped in backward": ('    dh1 = (dr @ W[1]) * (fw["h1"] > 0)', '    dh1 = (dr @ W[1])'),
    "density path dropped in backward": ('    dr[:, 0] += dsigma * density_activation_grad(fw["r"][:, 0], fw["sigma"], cfg.density_act)\n',
                                         ""),
    "colour sigmoid derivative": ("    dcraw = drgb * c * (1.0 - c)", "    dcraw = drgb * c"),
    "background not composited": ("    C = (w[..., None] * rgb).sum(axis=1) + TN[:, None] * bg", "    C = (w[..., None] * rgb).sum(axis=1)"),
    "render backward bg sign": ("- (TN * (gC * bg).sum(axis=1))[:, None])", "+ (TN * (gC * bg).sum(axis=1))[:, None])"),
    "render backward suffix inclusive": ("        return s - x\n", "        return s\n"),
    "density loss on object rays": ("    L_density = sigma_bg_sum[bgr].sum() / B", "    L_density = sigma_bg_sum[obj].sum() / B"),
    "depth gradient sign": ("gD = np.where(dep, cfg.lambda_depth * np.sign(ed) / B, 0.0)", "gD = np.where(dep, -cfg.lambda_depth * np.sign(ed) / B, 0.0)"),
    "occluders supervised": ("    sup = obj | bgr\n", "    sup = obj | bgr | hit\n"),
    "Adam dense on tables": ("    upd = (g != 0) if sparse else np.ones(g.shape, bool)", "    upd = np.ones(g.shape, bool)"),
    "Adam v without square": ("v[upd] = b2 * v[upd] + (1 - b2) * g[upd] * g[upd]", "v[upd] = b2 * v[upd] + (1 - b2) * np.abs(g[upd])"),
    "occluder rays kept": ("    hit = hit & (cls != CLS_OCCLUDER)                       # R10: occluders dropped\n", ""),
    "keyframe gate comparison inverted": ("    return alpha > alpha_deg, alpha", "    return alpha < alpha_deg, alpha"),
    "scheduler ignores max_iters": ("        n = min(chunk, min(pending[k] for k in live), max_iters - done)",
                                    "        n = min(chunk, min(pending[k] for k in live))"),
    "marching tetrahedra edge point": ("        return pa + (iso - sa) / (sb - sa) * (pb - pa)", "        return pa + 0.5 * (pb - pa)"),
    "to_world yaw sign": ("    out[..., 0] = c * X[..., 0] - s * X[..., 1] + box_t[0]", "    out[..., 0] = c * X[..., 0] + s * X[..., 1] + box_t[0]"),
    "scene segments by object id": ("    segs.sort(key=lambda s: (s[2], s[0], s[1]))", "    segs.sort(key=lambda s: (s[2], s[1], s[0]))"),
    "query outside the box not zero": ("    inside = np.all(np.abs(xyz) <= a, axis=1)\n    u = (xyz + a)",
                                       "    inside = np.ones(xyz.shape[0], bool)\n    u = (xyz + a)"),
    "colour input order [sh || r]": ("    cin = np.concatenate([r, sh], axis=1)", "    cin = np.concatenate([sh, r], axis=1)"),
    "paper net colour from raw 0..2": ("    c = 1.0 / (1.0 + np.exp(-raw[:, 1:4]))", "    c = 1.0 / (1.0 + np.exp(-raw[:, 0:3]))"),
    "depth rendered from delta": ('"D": (w * dist).sum(axis=1)}', '"D": (w * delta).sum(axis=1)}'),
    "rgb loss not divided by B": ("    L_rgb = ne[obj].sum() / B", "    L_rgb = ne[obj].sum()"),
    "density-loss gradient not divided by B": ("cfg.lambda_density / B, 0.0)[:, None]", "cfg.lambda_density, 0.0)[:, None]"),
    "hash mask modulo T - 1": ("    return (h & 0xFFFFFFFF) & (T - 1)", "    return (h & 0xFFFFFFFF) % (T - 1)"),
    "crop one pixel short": ("    x0, x1 = int(xs.min()), int(xs.max()) + 1", "    x0, x1 = int(xs.min()), int(xs.max())"),
    "depth kept on any class": ("z > 0 and cls[py - y0, px - x0] == CLS_OBJECT:", "z > 0:"),
    "pixel stream 4": ("    u = rng_u32(seed, obj, t, np.arange(R), 0).astype(U64)", "    u = rng_u32(seed, obj, t, np.arange(R), 4).astype(U64)"),
    "Adam eps inside the root": ("    p[upd] = p[upd] - cfg.lr * mh / (np.sqrt(vh) + cfg.eps)", "    p[upd] = p[upd] - cfg.lr * mh / np.sqrt(vh + cfg.eps)"),
    "gate angle in radians": ("    return math.degrees(math.acos(min(1.0, max(-1.0, c))))", "    return math.acos(min(1.0, max(-1.0, c)))"),
    "lattice axis swapped": ("    P = np.stack(np.meshgrid(*axes, indexing=\"ij\"), -1)", "    P = np.stack(np.meshgrid(*axes, indexing=\"xy\"), -1)"),
    "metrics acc / comp swapped": ('    return {"acc": float(acc), "comp": float(dc.mean())', '    return {"acc": float(dc.mean()), "comp": float(acc)'),
    "carve ignores points behind the camera": ("        seen |= (xc[2] > 0) & (u >= kf.x0)", "        seen |= (u >= kf.x0)"),
    "object rays composited over black": ("    if cfg.obj_bg == 1:", "    if cfg.obj_bg == 0:"),
    "initial tables not small": ("    table = g.uniform(-1e-4, 1e-4, size=(table_entries(cfg), cfg.feats))",
                                 "    table = g.uniform(-1e-2, 1e-2, size=(table_entries(cfg), cfg.feats))"),
    "paper net hidden ReLU dropped": ("        hs.append(relu(hs[-1] @ W[k].T))", "        hs.append(hs[-1] @ W[k].T)"),
}


def _run_one(root, name):
    """apply mutation `name` to a private copy of the oracle and run the pins on it"""
    d = os.path.join(root, "m%02d" % list(MUTATIONS).index(name))
    for sub in ("oracle", "tests", "scenes"):
        shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                        ignore=shutil.ignore_patterns("__pycache__", "test_oracle_mutations.py"))
    orig = open(os.path.join(ROOT, "oracle", "romap_oracle.py")).read()
    a, b = MUTATIONS[name]
    with open(os.path.join(d, "oracle", "romap_oracle.py"), "w") as f:
        f.write(orig.replace(a, b))
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-x", "-q", "-p", "no:cacheprovider"],
                       cwd=d, capture_output=True, text=True, timeout=900, env=env)
    return r.returncode, r.stdout[-2000:]


@pytest.fixture(scope="module")
def results(tmp_path_factory):
    """every mutation's pin run, several at a time (each in its own tree)"""
    root = str(tmp_path_factory.mktemp("mut"))
    workers = max(1, min(8, os.cpu_count() or 1))
    with concurrent.futures.ThreadPoolExecutor(workers) as ex:
        futs = {name: ex.submit(_run_one, root, name) for name in MUTATIONS}
        return {name: f.result() for name, f in futs.items()}


def test_mutations_apply_once():
    orig = open(os.path.join(ROOT, "oracle", "romap_oracle.py")).read()
    for name, (a, _) in MUTATIONS.items():
        assert orig.count(a) == 1, name


@pytest.mark.slow
@pytest.mark.parametrize("name", list(MUTATIONS))
def test_mutation_fails_a_pin(results, name):
    rc, out = results[name]
    assert rc == 1 and " failed" in out, (name, out)

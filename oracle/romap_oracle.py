"""RO-MAP training step / inference -- CPU ORACLE (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) may import this module.  It shares no code with the CUDA path.

Every function cites the passage it follows: PAPER.md:<line> (the paper's LaTeX
source, section / equation), SPEC.md:<line> (the CPU spec written from the
paper, used for interfaces and tie-breaking), or a DESIGN.md reading id
(R1..R23, mirroring SURVEY.md §8(c) A1..A23) where the paper is silent.

Precision: geometry that decides integers or is
required bit-exact (pixels, rays, segments, sample distances, normalized
positions, hash indices) in IEEE fp32, one rounding per operation, no
contraction; everything else in fp64.

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``):
  level_table       hand-listed resolutions / entry totals (BASELINE cfg0, cfg1)
  init_params       table range U(-1e-4, 1e-4) (R19)
  mix64 / rng_u32   published SplitMix64 output vectors (golden file)
  draw_pixels       bijection over all in-box pixels (brute force), chi^2
  rng_u32 key       golden u32 of the composed key from an independent python-int
                    reference (tests/golden/rng_ref.py, rng_u32_keys.txt); the
                    training stream layout (pixel 0, background 1-3, jitter 16+i)
  make_rays         principal-point ray, projection round trip
  make_rays_per_ray equals make_rays ray by ray (bitwise), round trip with per-ray K
  sample_points     hand-computed u for unequal half extents, clamp at the faces (R6)
  forward_rays      R17 depth target: z on the optical axis, z*|dc| off axis;
                    occluder rays dropped even when they cross the box (R10)
  ingest_observation  AABB / classes by hand; depth kept on object pixels only
  ray_box           (4,6) example, parallel miss,
                    dense-stepping membership oracle
  stratified        one sample per stratum, ascending, mean≈midpoint
  hash_encode       vertex / cell-centre cases, sum of
                    trilinear weights = 1, dense-level bijection, continuity
                    (SPEC.md:278), brute-force XOR-hash on python ints; the
                    upper face u = 1 in the last cell (R5 / R6)
  sh4               quadrature orthonormality + addition theorem; signs against
                    scipy's complex harmonics with the Condon-Shortley phase
  mlp_forward       zero model (SPEC.md:253 adapted to R4), selection weights;
                    network 1 (R24): shapes for 1..3 hidden layers, zero model,
                    selection weights, whole-step central differences
  volume_render     sigma=0, opaque first sample, ln2 case,
                    constant-density closed form 1-exp(-sigma L) (north_star)
  losses            (0.3,0,0.4)->0.5, decomposition identity,
                    occluder exclusion, background-only batch;
                    an empty field renders every supervised ray as its
                    background colour (R14, both obj_bg settings)
  density_activation  saturation at the clamp, straight-through derivative (R3)
  backward          central differences in fp64 through the whole step
  adam_update       closed form for constant gradient, zero-gradient no-op
                    (SPEC.md:271-273), sparse locality, g = eps
                    gives a step of lr/2 (eps outside the root)
  render / query    constant-density closed form, outside-box zero (R21);
                    midpoints by hand, opaque-field depth = first stratum centre
  render_scene      two boxes closed form; the nearer box first whatever its id (R20)
  marching_tetrahedra  single-vertex case counts (6 on the Kuhn diagonal, 2
                    elsewhere), exact vertices for a linear field, sphere radius /
                    area within the lattice step; mesh_metrics shifted-grid closed form
                    and a half reconstruction (acc 0, comp > 0); lattice axes
tests/test_oracle_mutations.py applies 64 plausible mistakes (wrong index / sign /
stream / operand / dropped term) to copies of this file, one at a time, and checks
that each fails a pin.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

f32 = np.float32
U64 = np.uint64

CLS_BACKGROUND = 0   # mask == 0                         (R_b)
CLS_OBJECT = 1       # mask == instance id               (R_o)
CLS_OCCLUDER = 2     # mask == another instance id


# --------------------------------------------------------------------------
# configuration (R1, R5): BASELINE.json configs; the paper's own constants are
# PAPER.md:222 (T=2^16, N_max=2048, width 64, 4096 rays, N=32, lambda1=0.5,
# lambda2=0.01)
# --------------------------------------------------------------------------
@dataclass
class ModelConfig:
    levels: int = 8
    feats: int = 2
    log2_T: int = 12
    base_res: int = 16
    finest_res: float = 2048.0
    res_cap: int = 128            # 0 = no cap
    width: int = 64               # PAPER.md:222 "hidden size 64"
    density_out: int = 16
    color_hidden: int = 2
    dir_enc: int = 16             # SH degree 4 (BASELINE cfg0)
    density_act: int = 0          # 0 exp (R3), 1 softplus
    samples_per_ray: int = 32
    rays_per_iter: int = 256
    lr: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.99
    eps: float = 1e-15
    lambda_depth: float = 0.5     # PAPER.md:222 lambda_1
    lambda_density: float = 0.01  # PAPER.md:222 lambda_2
    obj_bg: int = 0               # R14: 0 random bg for all supervised rays, 1 black for R_o
    seed: int = 0
    network: int = 0              # R24: 0 BASELINE density + SH colour nets, 1 the paper's position-only MLP
    hidden_layers: int = 1        # network 1: hidden layers of width `width` (Table 4: 1..3)


@dataclass
class Level:
    res: int
    dense: bool
    size: int
    offset: int


def level_table(cfg: ModelConfig) -> list[Level]:
    """Per-level resolution / storage (R5; instant-NGP [21] via PAPER.md:83,124).

    N_l = floor(N_min * b^l + 1e-6) with b = (N_max/N_min)^(1/(L-1)), in double,
    then min(N_l, res_cap).  Vertex lattice (N_l+1)^3.  A level is dense iff
    (N_l+1)^3 <= T, else hashed into T entries.  Levels are stored back to back,
    each block padded to a multiple of 16 entries (R5; padding entries are never
    addressed).
    """
    T = 1 << cfg.log2_T
    b = (cfg.finest_res / cfg.base_res) ** (1.0 / (cfg.levels - 1)) if cfg.levels > 1 else 1.0
    out, off = [], 0
    for l in range(cfg.levels):
        n = int(math.floor(cfg.base_res * b ** l + 1e-6))
        if cfg.res_cap > 0:
            n = min(n, cfg.res_cap)
        dense = (n + 1) ** 3 <= T
        size = (n + 1) ** 3 if dense else T
        out.append(Level(n, dense, size, off))
        off += (size + 15) // 16 * 16
    return out


def table_entries(cfg: ModelConfig) -> int:
    lt = level_table(cfg)
    return lt[-1].offset + (lt[-1].size + 15) // 16 * 16


def mlp_shapes(cfg: ModelConfig) -> list[tuple[int, int]]:
    """(out, in) of each bias-free layer (R1, R4): density LF->W->16; colour
    [16 raw || dir_enc]->W->...->W->3 (color_hidden hidden layers).
    network 1 (R24, "multi-resolution hash encoding and a
    single-layer MLP", positions only -> sigma and c): LF->W (->W ...)->4."""
    lf = cfg.levels * cfg.feats
    if cfg.network == 1:
        return [(cfg.width, lf)] + [(cfg.width, cfg.width)] * (cfg.hidden_layers - 1) + [(4, cfg.width)]
    shapes = [(cfg.width, lf), (cfg.density_out, cfg.width), (cfg.width, cfg.density_out + cfg.dir_enc)]
    shapes += [(cfg.width, cfg.width)] * (cfg.color_hidden - 1)
    shapes.append((3, cfg.width))
    return shapes


def init_params(cfg: ModelConfig, seed: int) -> dict:
    """R19: tables U(-1e-4, 1e-4); weights Glorot-uniform."""
    g = np.random.default_rng(seed)
    table = g.uniform(-1e-4, 1e-4, size=(table_entries(cfg), cfg.feats))
    W = []
    for (o, i) in mlp_shapes(cfg):
        lim = math.sqrt(6.0 / (o + i))
        W.append(g.uniform(-lim, lim, size=(o, i)))
    return {"table": table, "W": W}


# --------------------------------------------------------------------------
# O2 counter-based RNG (R13)
# --------------------------------------------------------------------------
GOLDEN = 0x9E3779B97F4A7C15


def mix64(z):
    """SplitMix64 finalizer (R13)."""
    z = np.array(z, dtype=U64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> U64(30)
        z *= U64(0xBF58476D1CE4E5B9)
        z ^= z >> U64(27)
        z *= U64(0x94D049BB133111EB)
        z ^= z >> U64(31)
    return z


def rng_u32(seed: int, obj: int, t: int, ray, stream):
    """key = mix(mix(mix(mix(seed+GOLDEN) ^ obj) ^ t) ^ ((ray<<8)|stream)); u32 = key>>32 (R13)."""
    with np.errstate(over="ignore"):
        k = mix64(np.array(seed, dtype=U64) + U64(GOLDEN))
        k = mix64(k ^ U64(obj))
        k = mix64(k ^ U64(t))
        r = np.asarray(ray, dtype=U64)
        s = np.asarray(stream, dtype=U64)
        k = mix64(k ^ ((r << U64(8)) | s))
    return (k >> U64(32)).astype(np.uint32)


def u32_to_unit(u):
    """float = (u32>>8) * 2^-24, exact in fp32, in [0,1) (R13)."""
    return (np.asarray(u, dtype=np.uint32) >> np.uint32(8)).astype(f32) * f32(2.0 ** -24)


# --------------------------------------------------------------------------
# a0 observation ingest (R9, R10, R17)
# --------------------------------------------------------------------------
@dataclass
class Keyframe:
    T_wc: np.ndarray          # (3,4) fp32, camera->world, OpenCV camera axes (R8)
    K: np.ndarray             # (4,) fp32 fx, fy, cx, cy
    x0: int
    y0: int
    w: int
    h: int
    rgb: np.ndarray           # (h,w,3) uint8 crop
    cls: np.ndarray           # (h,w) uint8 crop: 0 bg, 1 object, 2 occluder
    depth: np.ndarray | None  # (h,w) fp32 camera z (0 = none), object pixels only


def ingest_observation(rgb, mask, T_wc, K, instance_id, depth_samples=None) -> Keyframe:
    """Crop the frame to the object's detection box = tight AABB of mask==id
    ("back-project the pixels that are within the object's detection
    box"); classify each in-box pixel by its mask value (R10).
    Sparse depth: a sample (u,v,z) lands on pixel (floor u, floor v);
    only object pixels keep it (SPEC.md:304 has_depth => Object)."""
    mask = np.asarray(mask)
    ys, xs = np.nonzero(mask == instance_id)
    if xs.size == 0:
        raise ValueError("instance not visible in mask")
    x0, x1 = int(xs.min()), int(xs.max()) + 1
    y0, y1 = int(ys.min()), int(ys.max()) + 1
    m = mask[y0:y1, x0:x1]
    cls = np.where(m == instance_id, CLS_OBJECT, np.where(m == 0, CLS_BACKGROUND, CLS_OCCLUDER)).astype(np.uint8)
    depth = None
    if depth_samples is not None and len(depth_samples) > 0:
        depth = np.zeros((y1 - y0, x1 - x0), dtype=f32)
        for (u, v, z) in depth_samples:
            px, py = int(math.floor(u)), int(math.floor(v))
            if x0 <= px < x1 and y0 <= py < y1 and z > 0 and cls[py - y0, px - x0] == CLS_OBJECT:
                depth[py - y0, px - x0] = f32(z)
    return Keyframe(np.asarray(T_wc, f32).reshape(3, 4), np.asarray(K, f32)[:4],
                    x0, y0, x1 - x0, y1 - y0, np.ascontiguousarray(rgb[y0:y1, x0:x1]), cls, depth)


# --------------------------------------------------------------------------
# O3 pixel draw ("randomly samples 4096 rays from all training
# images"; R9: uniform over the union of in-box pixels, with replacement)
# --------------------------------------------------------------------------
def pixel_of_index(kfs: list[Keyframe], idx):
    """Union index -> (keyframe k, in-box lx, ly): k = last k with P[k] <= idx over the
    exclusive prefix P of box areas; in-box pixels row-major."""
    areas = np.array([k.w * k.h for k in kfs], dtype=np.int64)
    P = np.concatenate([[0], np.cumsum(areas)[:-1]])
    idx = np.asarray(idx, np.int64)
    k = np.searchsorted(P, idx, side="right") - 1
    local = idx - P[k]
    ws = np.array([kk.w for kk in kfs])[k]
    return k, local % ws, local // ws


def draw_pixels(kfs: list[Keyframe], seed, obj, t, R):
    """idx = (u32 * total) >> 32 with u32 from stream 0 of ray r (R9, R13)."""
    total = int(sum(k.w * k.h for k in kfs))
    u = rng_u32(seed, obj, t, np.arange(R), 0).astype(U64)
    idx = ((u * U64(total)) >> U64(32)).astype(np.int64)
    return pixel_of_index(kfs, idx)


# --------------------------------------------------------------------------
# O4 rays ("transform the camera pose to the object coordinate
# system and back-project the pixels"; R8)
# --------------------------------------------------------------------------
def box_rotation(yaw):
    """(c, s) = float(cos/sin(double yaw)) (R8, yaw about +z)."""
    y = float(f32(yaw))
    return f32(math.cos(y)), f32(math.sin(y))


def make_rays(px, py, K, T_wc, box_t, box_yaw):
    """Object-frame ray of pixel centres (px+0.5, py+0.5); fp32, one rounding per op.

    dc = ((px+.5-cx)/fx, (py+.5-cy)/fy, 1); n = sqrt((dc.x^2 + dc.y^2) + 1);
    d_w[k] = (R[k,0] dcn.x + R[k,1] dcn.y) + R[k,2] dcn.z; o_w = T_wc[:,3];
    x_obj = R_z(yaw)^T (x_w - t).  Returns o (R,3), d (R,3), n (R,)."""
    px = np.asarray(px).astype(f32) + f32(0.5)
    py = np.asarray(py).astype(f32) + f32(0.5)
    fx, fy, cx, cy = (f32(v) for v in np.asarray(K, f32)[:4])
    dcx = (px - cx) / fx
    dcy = (py - cy) / fy
    n = np.sqrt((dcx * dcx + dcy * dcy) + f32(1.0))
    nx, ny, nz = dcx / n, dcy / n, f32(1.0) / n
    Tm = np.asarray(T_wc, f32).reshape(3, 4)
    if Tm.ndim == 2:
        Tm = np.broadcast_to(Tm, (px.shape[0], 3, 4))
    dw = [(Tm[:, k, 0] * nx + Tm[:, k, 1] * ny) + Tm[:, k, 2] * nz for k in range(3)]
    t = np.asarray(box_t, f32)
    p = [Tm[:, k, 3] - t[k] for k in range(3)]
    c, s = box_rotation(box_yaw)
    o = np.stack([c * p[0] + s * p[1], c * p[1] - s * p[0], p[2]], axis=1).astype(f32)
    d = np.stack([c * dw[0] + s * dw[1], c * dw[1] - s * dw[0], dw[2]], axis=1).astype(f32)
    return o, d, n


def ray_box(o, d, a):
    """Slab test against [-a, a] ("If the ray intersects with the 3D
    bounding box, we compute the truncation distance"; R11).  inv = 1/d_k; a zero
    component misses iff |o_k| > a_k else leaves the slab open; t_near = max(.,0);
    hit iff t_far > t_near (strict).  fp32."""
    o = np.asarray(o, f32)
    d = np.asarray(d, f32)
    a = np.asarray(a, f32)
    R = o.shape[0]
    tn = np.zeros(R, f32)
    tf = np.full(R, np.inf, f32)
    miss = np.zeros(R, bool)
    for k in range(3):
        dk, ok, ak = d[:, k], o[:, k], a[k]
        zero = dk == 0
        with np.errstate(divide="ignore", invalid="ignore"):
            inv = f32(1.0) / dk
            t0 = (-ak - ok) * inv
            t1 = (ak - ok) * inv
        lo = np.where(zero, f32(-np.inf), np.minimum(t0, t1))
        hi = np.where(zero, f32(np.inf), np.maximum(t0, t1))
        miss |= zero & (np.abs(ok) > ak)
        tn = np.maximum(tn, lo)
        tf = np.minimum(tf, hi)
    hit = (~miss) & (tf > tn)
    return tn.astype(f32), tf.astype(f32), hit


def stratified(tn, tf, N, xi):
    """Stratified-uniform samples ("only perform uniform sampling";
    R12): D = (tf-tn)/N; d_i = tn + (i + xi_i)*D (mul then add);
    delta_i = d_{i+1} - d_i, delta_{N-1} = D.  fp32.  xi: (R,N) in [0,1)."""
    tn = np.asarray(tn, f32)[:, None]
    tf = np.asarray(tf, f32)[:, None]
    Dl = (tf - tn) / f32(N)
    s = np.arange(N, dtype=f32)[None, :] + np.asarray(xi, f32)
    dist = tn + s * Dl
    delta = np.empty_like(dist)
    delta[:, :-1] = dist[:, 1:] - dist[:, :-1]
    delta[:, -1] = Dl[:, 0]
    return dist.astype(f32), delta.astype(f32)


def midpoints(tn, tf, N):
    """Inference sampling (R12): xi = 0.5, delta_i = D for all i."""
    tn = np.asarray(tn, f32)[:, None]
    tf = np.asarray(tf, f32)[:, None]
    Dl = (tf - tn) / f32(N)
    s = np.arange(N, dtype=f32)[None, :] + f32(0.5)
    dist = tn + s * Dl
    return dist.astype(f32), np.broadcast_to(Dl, dist.shape).astype(f32)


def sample_points(o, d, dist, a):
    """x = o + d_i * d (mul then add); u = (x + a)/(a + a) clamped to [0,1] (R6). fp32."""
    o = np.asarray(o, f32)[:, None, :]
    d = np.asarray(d, f32)[:, None, :]
    x = o + np.asarray(dist, f32)[..., None] * d
    a = np.asarray(a, f32)
    u = (x + a) / (a + a)
    return np.minimum(np.maximum(u, f32(0.0)), f32(1.0)).astype(f32)


# --------------------------------------------------------------------------
# O7 multi-resolution hash encoding (PAPER.md:83,124 via [21]; R5)
# --------------------------------------------------------------------------
PRIMES = (1, 2654435761, 805459861)


def corner_index(lev: Level, cx, cy, cz, T):
    """Dense: x + (N+1)(y + (N+1) z).  Hashed: (x*1 ^ y*2654435761 ^ z*805459861)
    mod 2^32, & (T-1) ("standard 3-prime XOR hash")."""
    cx = np.asarray(cx, np.int64)
    cy = np.asarray(cy, np.int64)
    cz = np.asarray(cz, np.int64)
    if lev.dense:
        n1 = lev.res + 1
        return cx + n1 * (cy + n1 * cz)
    h = (cx * PRIMES[0]) ^ (cy * PRIMES[1]) ^ (cz * PRIMES[2])
    return (h & 0xFFFFFFFF) & (T - 1)


def hash_encode(u, table, cfg: ModelConfig):
    """Per level: pos = u*N_l (fp32); c = clamp(floor(pos), 0, N_l-1); f = pos - c;
    corners b=0..7 (bit k -> +1 on axis k); w_b = prod_k (bit ? f_k : 1-f_k) (fp64);
    feat_l = sum_b w_b * table[offset_l + idx_b]; levels concatenated ascending.
    u: (S,3) fp32, table (E,F) -> feat (S, L*F) fp64, idx (S,L,8) int64, w (S,L,8) fp64."""
    lt = level_table(cfg)
    T = 1 << cfg.log2_T
    u = np.asarray(u, f32).reshape(-1, 3)
    S, F = u.shape[0], cfg.feats
    feat = np.zeros((S, cfg.levels * F))
    idx_all = np.zeros((S, cfg.levels, 8), np.int64)
    w_all = np.zeros((S, cfg.levels, 8))
    for l, lev in enumerate(lt):
        pos = u * f32(lev.res)
        c = np.clip(np.floor(pos), 0, lev.res - 1).astype(np.int64)
        fr = (pos - c.astype(f32)).astype(np.float64)
        for b in range(8):
            bits = [(b >> k) & 1 for k in range(3)]
            idx = corner_index(lev, c[:, 0] + bits[0], c[:, 1] + bits[1], c[:, 2] + bits[2], T)
            w = np.ones(S)
            for k in range(3):
                w = w * (fr[:, k] if bits[k] else 1.0 - fr[:, k])
            idx_all[:, l, b] = lev.offset + idx
            w_all[:, l, b] = w
            feat[:, l * F:(l + 1) * F] += w[:, None] * table[lev.offset + idx]
    return feat, idx_all, w_all


def hash_encode_backward(dfeat, idx_all, w_all, n_entries, F):
    """Adjoint of hash_encode: grad[idx_b] += w_b * dfeat_l (np.add.at scatter)."""
    g = np.zeros((n_entries, F))
    S, L, _ = idx_all.shape
    for l in range(L):
        for b in range(8):
            np.add.at(g, idx_all[:, l, b], w_all[:, l, b][:, None] * dfeat[:, l * F:(l + 1) * F])
    return g


# --------------------------------------------------------------------------
# O8 real spherical harmonics, degree 4 = bands 0..3 (R2, BASELINE cfg0)
# --------------------------------------------------------------------------
def sh4(d):
    """16 real orthonormal SH of the unit direction d (fp64)."""
    d = np.asarray(d, np.float64).reshape(-1, 3)
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    xx, yy, zz = x * x, y * y, z * z
    out = np.empty((d.shape[0], 16))
    out[:, 0] = 0.28209479177387814
    out[:, 1] = -0.48860251190291987 * y
    out[:, 2] = 0.48860251190291987 * z
    out[:, 3] = -0.48860251190291987 * x
    out[:, 4] = 1.0925484305920792 * x * y
    out[:, 5] = -1.0925484305920792 * y * z
    out[:, 6] = 0.94617469575755997 * zz - 0.31539156525251999
    out[:, 7] = -1.0925484305920792 * x * z
    out[:, 8] = 0.54627421529603959 * (xx - yy)
    out[:, 9] = 0.59004358992664352 * y * (-3.0 * xx + yy)
    out[:, 10] = 2.8906114426405538 * x * y * z
    out[:, 11] = 0.45704579946446572 * y * (1.0 - 5.0 * zz)
    out[:, 12] = 0.3731763325901154 * z * (5.0 * zz - 3.0)
    out[:, 13] = 0.45704579946446572 * x * (1.0 - 5.0 * zz)
    out[:, 14] = 1.4453057213202769 * z * (xx - yy)
    out[:, 15] = 0.59004358992664352 * x * (-xx + 3.0 * yy)
    return out


# --------------------------------------------------------------------------
# O9 MLP ("estimate their density values sigma and colors c";
# BASELINE cfg0 network; R1 R3 R4)
# --------------------------------------------------------------------------
SIGMA_RAW_CLAMP = 15.0


def density_activation(r0, act):
    if act == 0:   # R3: sigma = exp(min(raw0, 15))
        return np.exp(np.minimum(r0, SIGMA_RAW_CLAMP))
    return np.logaddexp(0.0, r0)   # softplus


def density_activation_grad(r0, sigma, act):
    if act == 0:   # R3: straight-through at the clamp, dsigma/draw := sigma
        return sigma
    return 1.0 / (1.0 + np.exp(-r0))


def relu(x):
    return np.maximum(x, 0.0)


def mlp_forward_paper(feat, W, cfg: ModelConfig):
    """network 1 (R24): h_1 = ReLU(W_1 feat), h_k = ReLU(W_k h_{k-1}), raw = W_out h_L;
    sigma = act(raw_0) (R3), c = sigmoid(raw_1..3).  No view direction
    (PAPER.md:155).  fp64."""
    hs = [relu(feat @ W[0].T)]
    for k in range(1, cfg.hidden_layers):
        hs.append(relu(hs[-1] @ W[k].T))
    raw = hs[-1] @ W[-1].T
    sigma = density_activation(raw[:, 0], cfg.density_act)
    c = 1.0 / (1.0 + np.exp(-raw[:, 1:4]))
    return {"feat": feat, "h": hs, "raw": raw, "r": raw, "sigma": sigma, "rgb": c}


def mlp_forward(feat, sh, W, cfg: ModelConfig):
    """h = ReLU(W1 feat); r = W2 h; sigma = act(r0); g = ReLU(W3 [r||sh]);
    g_k = ReLU(W g_{k-1}) ...; c = sigmoid(W_last g).  fp64.  sh may be (S,0).
    network 1: mlp_forward_paper (sh unused)."""
    if cfg.network == 1:
        return mlp_forward_paper(feat, W, cfg)
    h1 = relu(feat @ W[0].T)
    r = h1 @ W[1].T
    sigma = density_activation(r[:, 0], cfg.density_act)
    cin = np.concatenate([r, sh], axis=1)
    gs = [relu(cin @ W[2].T)]
    for k in range(cfg.color_hidden - 1):
        gs.append(relu(gs[-1] @ W[3 + k].T))
    craw = gs[-1] @ W[-1].T
    c = 1.0 / (1.0 + np.exp(-craw))
    return {"feat": feat, "h1": h1, "r": r, "sigma": sigma, "cin": cin, "g": gs, "craw": craw, "rgb": c}


def mlp_forward_density(feat, W, cfg: ModelConfig):
    """Density net only (query_density, R21); network 1: the whole MLP's sigma."""
    if cfg.network == 1:
        return mlp_forward_paper(feat, W, cfg)["sigma"]
    h1 = relu(feat @ W[0].T)
    r = h1 @ W[1].T
    return density_activation(r[:, 0], cfg.density_act)


def mlp_backward(fw, dsigma, drgb, W, cfg: ModelConfig):
    """Reverse mode through mlp_forward by hand (ReLU masks h>0, dW = delta^T x)."""
    if cfg.network == 1:
        return mlp_backward_paper(fw, dsigma, drgb, W, cfg)
    c = fw["rgb"]
    dcraw = drgb * c * (1.0 - c)
    dW = [None] * len(W)
    gs = fw["g"]
    dW[-1] = dcraw.T @ gs[-1]
    dg = (dcraw @ W[-1]) * (gs[-1] > 0)
    for k in range(cfg.color_hidden - 1, 0, -1):
        dW[2 + k] = dg.T @ gs[k - 1]
        dg = (dg @ W[2 + k]) * (gs[k - 1] > 0)
    dW[2] = dg.T @ fw["cin"]
    dcin = dg @ W[2]
    dr = dcin[:, :cfg.density_out].copy()
    dr[:, 0] += dsigma * density_activation_grad(fw["r"][:, 0], fw["sigma"], cfg.density_act)
    dW[1] = dr.T @ fw["h1"]
    dh1 = (dr @ W[1]) * (fw["h1"] > 0)
    dW[0] = dh1.T @ fw["feat"]
    dfeat = dh1 @ W[0]
    return dW, dfeat


def mlp_backward_paper(fw, dsigma, drgb, W, cfg: ModelConfig):
    """Reverse mode through mlp_forward_paper: draw_0 = dsigma act'(raw_0),
    draw_1..3 = drgb c (1 - c); dW_out = draw^T h_L; dh = (draw W_out) [h > 0] ..."""
    c = fw["rgb"]
    hs = fw["h"]
    draw = np.zeros_like(fw["raw"])
    draw[:, 0] = dsigma * density_activation_grad(fw["raw"][:, 0], fw["sigma"], cfg.density_act)
    draw[:, 1:4] = drgb * c * (1.0 - c)
    dW = [None] * len(W)
    dW[-1] = draw.T @ hs[-1]
    dh = (draw @ W[-1]) * (hs[-1] > 0)
    for k in range(cfg.hidden_layers - 1, 0, -1):
        dW[k] = dh.T @ hs[k - 1]
        dh = (dh @ W[k]) * (hs[k - 1] > 0)
    dW[0] = dh.T @ fw["feat"]
    dfeat = dh @ W[0]
    return dW, dfeat


# --------------------------------------------------------------------------
# O10 volume rendering (Eq. 6; R14 background compositing)
# --------------------------------------------------------------------------
def volume_render(sigma, rgb, dist, delta, bg):
    """o_i = 1 - exp(-sigma_i delta_i); w_i = o_i prod_{j<i}(1 - o_j)
    (PAPER.md:156); C = sum w_i c_i (+ T_N b, R14); D = sum w_i d_i (Eq. 6).
    sigma, dist, delta: (R,N); rgb (R,N,3); bg (R,3).  fp64."""
    sigma = np.asarray(sigma, np.float64)
    delta = np.asarray(delta, np.float64)
    dist = np.asarray(dist, np.float64)
    alpha = np.exp(-sigma * delta)                 # 1 - o_i
    Tr = np.ones_like(alpha)
    if alpha.shape[1] > 1:
        Tr[:, 1:] = np.cumprod(alpha, axis=1)[:, :-1]
    TN = np.prod(alpha, axis=1)
    w = Tr * (1.0 - alpha)
    C = (w[..., None] * rgb).sum(axis=1) + TN[:, None] * bg
    return {"alpha": alpha, "T": Tr, "TN": TN, "w": w, "C": C, "A": w.sum(axis=1), "D": (w * dist).sum(axis=1)}


def volume_render_backward(vr, gC, gD, rgb, dist, delta, bg):
    """dC/dc_i = w_i; dC/dsigma_i = delta_i (T_{i+1} c_i - sum_{k>i} w_k c_k - T_N b);
    dD/dsigma_i = delta_i (T_{i+1} d_i - sum_{k>i} w_k d_k).  Returns (dsigma, drgb)."""
    w, alpha, Tr, TN = vr["w"], vr["alpha"], vr["T"], vr["TN"]
    dist = np.asarray(dist, np.float64)
    delta = np.asarray(delta, np.float64)
    drgb = w[..., None] * gC[:, None, :]
    gc = (rgb * gC[:, None, :]).sum(axis=2)
    def suffix_excl(x):
        s = np.cumsum(x[:, ::-1], axis=1)[:, ::-1]
        return s - x
    Tn1 = Tr * alpha
    dsig = delta * (Tn1 * gc - suffix_excl(w * gc) - (TN * (gC * bg).sum(axis=1))[:, None])
    dsig += delta * gD[:, None] * (Tn1 * dist - suffix_excl(w * dist))
    return dsig, drgb


# --------------------------------------------------------------------------
# O11 losses (Eqs. 7-11; R14-R17)
# --------------------------------------------------------------------------
def losses_and_render_grads(cls, hit, has_depth, C, D, tgt, bg_rgb, depth_t, sigma_bg_sum, B, cfg):
    """L_rgb = sum_{R_o} |C - C_gt|_2 (Eq. 7); L_depth = sum_{R_d} |D - D_gt| (Eq. 8);
    L_rr = sum_{R_b} |C - C_random|_2 (Eq. 9); L_density = sum_{R_b} sum_j |sigma_j| (Eq. 10);
    occluders: no loss; each sum / B (R16); L = L_rgb + L_rr +
    lambda1 L_depth + lambda2 L_density (Eq. 11).  Norms not squared (R15);
    gradient 0 where the norm is 0.  Returns losses and dL/dC (R,3), dL/dD (R,)."""
    R = C.shape[0]
    obj = hit & (cls == CLS_OBJECT)
    bgr = hit & (cls == CLS_BACKGROUND)
    dep = obj & has_depth
    target = np.where(obj[:, None], tgt, bg_rgb)
    e = C - target
    ne = np.sqrt((e * e).sum(axis=1))
    sup = obj | bgr
    gC = np.zeros((R, 3))
    nz = sup & (ne > 0)
    gC[nz] = e[nz] / ne[nz, None] / B
    ed = D - depth_t
    gD = np.where(dep, cfg.lambda_depth * np.sign(ed) / B, 0.0)
    L_rgb = ne[obj].sum() / B
    L_rr = ne[bgr].sum() / B
    L_depth = np.abs(ed[dep]).sum() / B
    L_density = sigma_bg_sum[bgr].sum() / B
    L = L_rgb + L_rr + cfg.lambda_depth * L_depth + cfg.lambda_density * L_density
    return {"l_total": L, "l_rgb": L_rgb, "l_rr": L_rr, "l_depth": L_depth, "l_density": L_density}, gC, gD


# --------------------------------------------------------------------------
# O14 Adam (R18)
# --------------------------------------------------------------------------
def adam_update(p, g, m, v, t, cfg: ModelConfig, sparse: bool):
    """m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2; p -= lr (m/(1-b1^t)) / (sqrt(v/(1-b2^t)) + eps).
    sparse=True (hash tables, R18): only entries with a nonzero gradient this step
    update p/m/v.  In place, fp64."""
    upd = (g != 0) if sparse else np.ones(g.shape, bool)
    b1, b2 = cfg.beta1, cfg.beta2
    m[upd] = b1 * m[upd] + (1 - b1) * g[upd]
    v[upd] = b2 * v[upd] + (1 - b2) * g[upd] * g[upd]
    mh = m[upd] / (1 - b1 ** t)
    vh = v[upd] / (1 - b2 ** t)
    p[upd] = p[upd] - cfg.lr * mh / (np.sqrt(vh) + cfg.eps)


# --------------------------------------------------------------------------
# one training iteration of one object (Table 3 rows PAPER.md:307-309)
# --------------------------------------------------------------------------
@dataclass
class ObjectState:
    cfg: ModelConfig
    box_t: np.ndarray     # (3,) fp32 world
    box_yaw: float
    box_a: np.ndarray     # (3,) fp32 half extents
    obj_id: int
    params: dict
    m: dict = field(default=None)
    v: dict = field(default=None)
    step: int = 0
    kfs: list = field(default_factory=list)

    def __post_init__(self):
        if self.m is None:
            self.m = {"table": np.zeros_like(self.params["table"]), "W": [np.zeros_like(w) for w in self.params["W"]]}
            self.v = {"table": np.zeros_like(self.params["table"]), "W": [np.zeros_like(w) for w in self.params["W"]]}


def forward_rays(st: ObjectState, t: int, rays_per_iter=None):
    """Steps a1-a2 of a training iteration: draw pixels, classify, build rays,
    segment, sample (fp32), plus targets and background colours."""
    cfg = st.cfg
    R = cfg.rays_per_iter if rays_per_iter is None else rays_per_iter
    N = cfg.samples_per_ray
    k, lx, ly = draw_pixels(st.kfs, cfg.seed, st.obj_id, t, R)
    cls = np.array([st.kfs[kk].cls[yy, xx] for kk, xx, yy in zip(k, lx, ly)], np.uint8)
    tgt = np.array([st.kfs[kk].rgb[yy, xx] for kk, xx, yy in zip(k, lx, ly)], f32) / f32(255.0)
    zc = np.array([(st.kfs[kk].depth[yy, xx] if st.kfs[kk].depth is not None else 0.0)
                   for kk, xx, yy in zip(k, lx, ly)], f32)
    px = np.array([st.kfs[kk].x0 for kk in k]) + lx
    py = np.array([st.kfs[kk].y0 for kk in k]) + ly
    Ks = np.stack([st.kfs[kk].K for kk in k])
    Ts = np.stack([st.kfs[kk].T_wc for kk in k])
    o, d, n = make_rays_per_ray(px, py, Ks, Ts, st.box_t, st.box_yaw)
    tn, tf, hit = ray_box(o, d, st.box_a)
    hit = hit & (cls != CLS_OCCLUDER)                       # R10: occluders dropped
    has_depth = (cls == CLS_OBJECT) & (zc > 0)
    depth_t = (zc * n).astype(f32)                          # R17
    ray = np.arange(R)
    bg = np.stack([u32_to_unit(rng_u32(cfg.seed, st.obj_id, t, ray, 1 + c)) for c in range(3)], axis=1)
    xi = np.stack([u32_to_unit(rng_u32(cfg.seed, st.obj_id, t, ray, 16 + i)) for i in range(N)], axis=1)
    tn_s = np.where(hit, tn, f32(0))
    tf_s = np.where(hit, tf, f32(0))
    dist, delta = stratified(tn_s, tf_s, N, xi)
    u = sample_points(o, d, dist, st.box_a)
    return {"k": k, "px": px, "py": py, "cls": cls, "tgt": tgt, "has_depth": has_depth, "depth_t": depth_t,
            "o": o, "d": d, "tn": tn, "tf": tf, "hit": hit, "bg": bg, "xi": xi, "dist": dist, "delta": delta,
            "u": u, "R": R}


def make_rays_per_ray(px, py, Ks, Ts, box_t, yaw):
    """make_rays with per-ray intrinsics / pose (rays drawn from several keyframes)."""
    px = np.asarray(px).astype(f32) + f32(0.5)
    py = np.asarray(py).astype(f32) + f32(0.5)
    fx, fy, cx, cy = Ks[:, 0], Ks[:, 1], Ks[:, 2], Ks[:, 3]
    dcx = (px - cx) / fx
    dcy = (py - cy) / fy
    n = np.sqrt((dcx * dcx + dcy * dcy) + f32(1.0))
    nx, ny, nz = dcx / n, dcy / n, f32(1.0) / n
    dw = [(Ts[:, k, 0] * nx + Ts[:, k, 1] * ny) + Ts[:, k, 2] * nz for k in range(3)]
    t = np.asarray(box_t, f32)
    p = [Ts[:, k, 3] - t[k] for k in range(3)]
    c, s = box_rotation(yaw)
    o = np.stack([c * p[0] + s * p[1], c * p[1] - s * p[0], p[2]], axis=1).astype(f32)
    d = np.stack([c * dw[0] + s * dw[1], c * dw[1] - s * dw[0], dw[2]], axis=1).astype(f32)
    return o, d, n


def loss_and_grads(st: ObjectState, t: int, params=None, rays=None):
    """Forward + backward of one iteration for one object (no parameter update).
    Returns (losses, grads {table, W}, debug dict)."""
    cfg = st.cfg
    P = st.params if params is None else params
    rs = forward_rays(st, t) if rays is None else rays
    R, N = rs["R"], cfg.samples_per_ray
    act = rs["hit"]
    ia = np.nonzero(act)[0]
    Ra = ia.size
    u = rs["u"][ia].reshape(-1, 3)
    feat, idx, w = hash_encode(u, P["table"], cfg)
    sh = sh4(np.repeat(rs["d"][ia], N, axis=0)) if (cfg.network == 0 and cfg.dir_enc == 16) else np.zeros((Ra * N, 0))
    fw = mlp_forward(feat, sh, P["W"], cfg)
    sigma = fw["sigma"].reshape(Ra, N)
    rgb = fw["rgb"].reshape(Ra, N, 3)
    cls_a = rs["cls"][ia]
    bg = rs["bg"][ia].astype(np.float64)
    comp_bg = bg.copy()
    if cfg.obj_bg == 1:
        comp_bg[cls_a == CLS_OBJECT] = 0.0
    vr = volume_render(sigma, rgb, rs["dist"][ia], rs["delta"][ia], comp_bg)
    sig_sum = sigma.sum(axis=1)
    B = float(R)
    Ls, gC, gD = losses_and_render_grads(cls_a, np.ones(Ra, bool), rs["has_depth"][ia], vr["C"], vr["D"],
                                         rs["tgt"][ia].astype(np.float64), bg, rs["depth_t"][ia].astype(np.float64),
                                         sig_sum, B, cfg)
    dsig, drgb = volume_render_backward(vr, gC, gD, rgb, rs["dist"][ia], rs["delta"][ia], comp_bg)
    dsig = dsig + np.where(cls_a == CLS_BACKGROUND, cfg.lambda_density / B, 0.0)[:, None]   # Eq. 10 grad
    dW, dfeat = mlp_backward(fw, dsig.reshape(-1), drgb.reshape(-1, 3), P["W"], cfg)
    gtab = hash_encode_backward(dfeat, idx, w, P["table"].shape[0], cfg.feats)
    Ls["rays"] = R
    Ls["hit_rays"] = Ra
    Ls["samples"] = Ra * N
    dbg = {"rays": rs, "active": ia, "feat": feat, "idx": idx, "w": w, "fw": fw, "vr": vr,
           "dsigma": dsig, "drgb": drgb, "dfeat": dfeat}
    return Ls, {"table": gtab, "W": dW}, dbg


def train_iteration(st: ObjectState):
    """One full iteration (Table 3: ray sampling -> forward + volume rendering ->
    backward and optimization): t = step+1 keys the RNG and Adam."""
    t = st.step + 1
    Ls, g, dbg = loss_and_grads(st, t)
    adam_update(st.params["table"], g["table"], st.m["table"], st.v["table"], t, st.cfg, sparse=True)
    for k in range(len(st.params["W"])):
        adam_update(st.params["W"][k], g["W"][k], st.m["W"][k], st.v["W"][k], t, st.cfg, sparse=False)
    st.step = t
    Ls["step"] = t
    return Ls, g, dbg


# --------------------------------------------------------------------------
# O15 inference: render / query_density (R12 midpoints, R20, R21)
# --------------------------------------------------------------------------
def field_eval(cfg, params, u_flat, d_rep):
    feat, _, _ = hash_encode(u_flat, params["table"], cfg)
    sh = sh4(d_rep) if (cfg.network == 0 and cfg.dir_enc == 16) else np.zeros((u_flat.shape[0], 0))
    fw = mlp_forward(feat, sh, params["W"], cfg)
    return fw["sigma"], fw["rgb"]


def render(cfg, box_t, box_yaw, box_a, params, T_wc, K, width, height, N):
    """Render one object from pose T_wc: pixel-centre rays, midpoint samples,
    composite over black (R12, R20).  Returns rgb (H,W,3), depth (H,W), opacity (H,W)."""
    py, px = np.meshgrid(np.arange(height), np.arange(width), indexing="ij")
    px, py = px.reshape(-1), py.reshape(-1)
    o, d, _ = make_rays(px, py, K, T_wc, box_t, box_yaw)
    tn, tf, hit = ray_box(o, d, box_a)
    HW = px.size
    rgb = np.zeros((HW, 3))
    dep = np.zeros(HW)
    opa = np.zeros(HW)
    ia = np.nonzero(hit)[0]
    if ia.size:
        dist, delta = midpoints(tn[ia], tf[ia], N)
        u = sample_points(o[ia], d[ia], dist, box_a)
        sig, col = field_eval(cfg, params, u.reshape(-1, 3), np.repeat(d[ia], N, axis=0))
        vr = volume_render(sig.reshape(-1, N), col.reshape(-1, N, 3), dist, delta, np.zeros((ia.size, 3)))
        rgb[ia] = vr["C"]
        dep[ia] = vr["D"]
        opa[ia] = vr["A"]
    return rgb.reshape(height, width, 3), dep.reshape(height, width), opa.reshape(height, width)


def query_density(cfg, box_a, params, xyz):
    """sigma at object-frame points (m); 0 outside the box [-a, a] (R21)."""
    xyz = np.asarray(xyz, f32).reshape(-1, 3)
    a = np.asarray(box_a, f32)
    inside = np.all(np.abs(xyz) <= a, axis=1)
    u = (xyz + a) / (a + a)
    u = np.minimum(np.maximum(u, f32(0)), f32(1)).astype(f32)
    sig = np.zeros(xyz.shape[0])
    if inside.any():
        feat, _, _ = hash_encode(u[inside], params["table"], cfg)
        sig[inside] = mlp_forward_density(feat, params["W"], cfg)
    return sig


def render_scene(objs: list, T_wc, K, width, height, N):
    """Multi-object render (R20): per pixel ray, intersect every object box; sort
    the hit segments by t_near (tie -> smaller object id); per segment midpoint
    samples, (C_s, A_s, D_s) over black; front to back C += T C_s, D += T D_s,
    T *= (1 - A_s).  objs: list of (cfg, box_t, yaw, box_a, params, obj_id).
    Ray distances are object-frame metres = world metres (rigid transform)."""
    py, px = np.meshgrid(np.arange(height), np.arange(width), indexing="ij")
    px, py = px.reshape(-1), py.reshape(-1)
    HW = px.size
    segs = []   # (tn, obj_id, pixel, C(3), A, D)
    for (cfg, bt, yaw, ba, params, oid) in objs:
        o, d, _ = make_rays(px, py, K, T_wc, bt, yaw)
        tn, tf, hit = ray_box(o, d, ba)
        ia = np.nonzero(hit)[0]
        if ia.size == 0:
            continue
        dist, delta = midpoints(tn[ia], tf[ia], N)
        u = sample_points(o[ia], d[ia], dist, ba)
        sig, col = field_eval(cfg, params, u.reshape(-1, 3), np.repeat(d[ia], N, axis=0))
        vr = volume_render(sig.reshape(-1, N), col.reshape(-1, N, 3), dist, delta, np.zeros((ia.size, 3)))
        for j, p in enumerate(ia):
            segs.append((float(tn[p]), oid, int(p), vr["C"][j], vr["A"][j], vr["D"][j]))
    rgb = np.zeros((HW, 3))
    dep = np.zeros(HW)
    Tr = np.ones(HW)
    segs.sort(key=lambda s: (s[2], s[0], s[1]))
    for (tn, oid, p, C, A, D) in segs:
        rgb[p] += Tr[p] * C
        dep[p] += Tr[p] * D
        Tr[p] *= (1.0 - A)
    return rgb.reshape(height, width, 3), dep.reshape(height, width), (1.0 - Tr).reshape(height, width)


# --------------------------------------------------------------------------
# parameter flattening (the ABI's block layout)
# --------------------------------------------------------------------------
def flatten_mlp(W):
    return np.concatenate([w.reshape(-1) for w in W])


def unflatten_mlp(vec, cfg):
    out, off = [], 0
    for (o, i) in mlp_shapes(cfg):
        out.append(np.asarray(vec[off:off + o * i], np.float64).reshape(o, i).copy())
        off += o * i
    return out


# --------------------------------------------------------------------------
# f3 online policy (Eq. 5): keyframe gate and iteration budget
# --------------------------------------------------------------------------
def camera_centre(T_wc):
    """camera centre in the world = translation column of T_wc (camera -> world, R8)"""
    T = np.asarray(T_wc, np.float64).reshape(3, 4)
    return T[:, 3].copy()


def view_angle_deg(c_last, c_new, t_obj):
    """Eq. 5: alpha = arccos(((t_Im - t_O) . (t_In - t_O)) / (|t_Im - t_O| |t_In - t_O|)),
    in degrees (fp64)"""
    a = np.asarray(c_last, np.float64) - np.asarray(t_obj, np.float64)
    b = np.asarray(c_new, np.float64) - np.asarray(t_obj, np.float64)
    c = float(a @ b) / (float(np.linalg.norm(a)) * float(np.linalg.norm(b)))
    return math.degrees(math.acos(min(1.0, max(-1.0, c))))


def keyframe_gate(last_centre, T_wc, t_obj, alpha_deg=25.0):
    """the first observation of an object is always taken; later
    ones iff alpha (Eq. 5, against the LAST ACCEPTED keyframe) exceeds the threshold.
    Returns (accepted, alpha or None)."""
    c = camera_centre(T_wc)
    if last_centre is None:
        return True, None
    alpha = view_angle_deg(last_centre, c, t_obj)
    return alpha > alpha_deg, alpha


def schedule_budgets(pending: dict, chunk: int, max_iters: int):
    """f3 scheduler (host policy, R25): while some object has pending
    iterations and fewer than max_iters were run in this call, train all objects with
    budget left for n = min(chunk, smallest pending) iterations in one batch.
    Returns the list of (objects, n) batches and the remaining budgets."""
    pending = dict(pending)
    batches, done = [], 0
    while done < max_iters:
        live = sorted(k for k, v in pending.items() if v > 0)
        if not live:
            break
        n = min(chunk, min(pending[k] for k in live), max_iters - done)
        batches.append((live, n))
        for k in live:
            pending[k] -= n
        done += n
    return batches, pending


# --------------------------------------------------------------------------
# f2 mesh extraction + metrics (R26)
# --------------------------------------------------------------------------
# Kuhn decomposition of a cube into 6 tetrahedra along the diagonal 0 -> 7; cube
# vertex k = (k & 1, (k >> 1) & 1, (k >> 2) & 1)
KUHN_TETS = [(0, 1 << p0, (1 << p0) | (1 << p1), 7)
             for (p0, p1) in [(0, 1), (0, 2), (1, 0), (1, 2), (2, 0), (2, 1)]]


def lattice_points(box_a, res):
    """(res+1)^3 vertex lattice spanning [-a, a] (R21), indexed [ix, iy, iz], fp32"""
    a = np.asarray(box_a, np.float64)
    axes = [(-a[k] + 2.0 * a[k] * np.arange(res + 1) / res) for k in range(3)]
    P = np.stack(np.meshgrid(*axes, indexing="ij"), -1)
    return P.astype(f32)


def marching_tetrahedra(sigma, points, iso):
    """Isosurface sigma = iso of a vertex lattice (R26): every cell split into the 6
    Kuhn tetrahedra; per tetrahedron with 1 or 3 vertices above iso one triangle on its
    3 crossing edges, with 2 above a quad (2 triangles) on its 4 crossing edges; edge
    points by linear interpolation p_a + (iso - s_a) / (s_b - s_a) (p_b - p_a).  Plain
    loops (small lattices only).  Returns (T, 3, 3) fp64 triangles (cell order, tet
    order), vertex order within a triangle as listed below."""
    sigma = np.asarray(sigma, np.float64)
    P = np.asarray(points, np.float64)
    R = sigma.shape[0] - 1
    tris = []

    def edge(va, vb, sa, sb, pa, pb):
        return pa + (iso - sa) / (sb - sa) * (pb - pa)
    for ix in range(R):
        for iy in range(R):
            for iz in range(R):
                cs = [sigma[ix + (k & 1), iy + ((k >> 1) & 1), iz + ((k >> 2) & 1)] for k in range(8)]
                cp = [P[ix + (k & 1), iy + ((k >> 1) & 1), iz + ((k >> 2) & 1)] for k in range(8)]
                for tet in KUHN_TETS:
                    s = [cs[v] for v in tet]
                    p = [cp[v] for v in tet]
                    ins = [i for i in range(4) if s[i] > iso]
                    out = [i for i in range(4) if not s[i] > iso]
                    if len(ins) in (1, 3):
                        a_ = ins[0] if len(ins) == 1 else out[0]
                        others = [i for i in range(4) if i != a_]
                        tris.append([edge(a_, o, s[a_], s[o], p[a_], p[o]) for o in others])
                    elif len(ins) == 2:
                        a_, b_ = ins
                        c_, d_ = out
                        q = [edge(a_, c_, s[a_], s[c_], p[a_], p[c_]), edge(a_, d_, s[a_], s[d_], p[a_], p[d_]),
                             edge(b_, d_, s[b_], s[d_], p[b_], p[d_]), edge(b_, c_, s[b_], s[c_], p[b_], p[c_])]
                        tris.append([q[0], q[1], q[2]])
                        tris.append([q[0], q[2], q[3]])
    return np.asarray(tris, np.float64).reshape(-1, 3, 3)


def to_world(X, box_t, box_yaw):
    """object frame -> world: x_w = R_z(yaw) x + t (R8, inverse of the ray transform)"""
    c, s = math.cos(box_yaw), math.sin(box_yaw)
    X = np.asarray(X, np.float64)
    out = X.copy()
    out[..., 0] = c * X[..., 0] - s * X[..., 1] + box_t[0]
    out[..., 1] = s * X[..., 0] + c * X[..., 1] + box_t[1]
    out[..., 2] = X[..., 2] + box_t[2]
    return out


def nearest_distances(A, B, chunk=2048):
    """for every point of A the distance to its nearest point of B (brute force)"""
    A = np.asarray(A, np.float64).reshape(-1, 3)
    B = np.asarray(B, np.float64).reshape(-1, 3)
    out = np.empty(A.shape[0])
    for i in range(0, A.shape[0], chunk):
        d2 = ((A[i:i + chunk, None, :] - B[None, :, :]) ** 2).sum(-1)
        out[i:i + chunk] = np.sqrt(d2.min(axis=1))
    return out


def sample_mesh_points(tris, n, seed=0):
    """n points uniformly on the surface of a triangle soup (area-weighted triangle
    choice, uniform barycentric coordinates), deterministic in seed"""
    T = np.asarray(tris, np.float64).reshape(-1, 3, 3)
    area = 0.5 * np.linalg.norm(np.cross(T[:, 1] - T[:, 0], T[:, 2] - T[:, 0]), axis=1)
    g = np.random.default_rng(seed)
    idx = g.choice(len(T), size=n, p=area / area.sum())
    r1, r2 = g.random(n), g.random(n)
    s1 = np.sqrt(r1)
    w0, w1, w2 = 1 - s1, s1 * (1 - r2), s1 * r2
    return w0[:, None] * T[idx, 0] + w1[:, None] * T[idx, 1] + w2[:, None] * T[idx, 2]


def mesh_metrics(rec_points, gt_points, tau):
    """PAPER.md:255 (Acc / Comp / CR as in iMAP-style evaluations): accuracy = mean
    distance from reconstructed points to the ground-truth surface samples, completion
    = mean distance from ground-truth samples to the reconstruction, completion ratio =
    fraction of ground-truth samples within tau"""
    acc = nearest_distances(rec_points, gt_points).mean()
    dc = nearest_distances(gt_points, rec_points)
    return {"acc": float(acc), "comp": float(dc.mean()), "cr": float((dc < tau).mean())}


def observed_mask(points, box_t, box_yaw, kfs):
    """R26 visibility carve: a lattice vertex (object frame) is observed iff it lies in
    front of some keyframe's camera and projects into that keyframe's detection box
    (the pixels training rays come from).  fp32, one rounding per
    operation in the order written (bit-exact with the GPU): x_w = R_z x + t,
    d = x_w - c (c = camera centre), x_c = R^T d, u = fx (x_c0 / x_c2) + cx,
    v = fy (x_c1 / x_c2) + cy; in box iff x0 <= u < x0 + w and y0 <= v < y0 + h."""
    P = np.asarray(points, f32).reshape(-1, 3)
    c = f32(math.cos(box_yaw))
    s = f32(math.sin(box_yaw))
    t = np.asarray(box_t, f32)
    xw = [(c * P[:, 0] - s * P[:, 1]) + t[0], (s * P[:, 0] + c * P[:, 1]) + t[1], P[:, 2] + t[2]]
    seen = np.zeros(P.shape[0], bool)
    for kf in kfs:
        T = np.asarray(kf.T_wc, f32).reshape(3, 4)
        d = [xw[k] - T[k, 3] for k in range(3)]
        xc = [(T[0, k] * d[0] + T[1, k] * d[1]) + T[2, k] * d[2] for k in range(3)]
        fx, fy, cx, cy = [f32(v) for v in kf.K]
        with np.errstate(divide="ignore", invalid="ignore"):
            u = fx * (xc[0] / xc[2]) + cx
            v = fy * (xc[1] / xc[2]) + cy
        seen |= (xc[2] > 0) & (u >= kf.x0) & (u < kf.x0 + kf.w) & (v >= kf.y0) & (v < kf.y0 + kf.h)
    return seen

"""The oracle pins must catch plausible mistakes: each
mutation below (a wrong operand, index, sign, RNG stream or dropped clamp in
oracle/romap_oracle.py) is applied to a COPY of the oracle in a temporary tree,
tests/test_oracle_pins.py runs against that copy, and at least one pin must fail.
The working tree is never modified."""
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
}


@pytest.fixture(scope="module")
def tree(tmp_path_factory):
    d = tmp_path_factory.mktemp("mut")
    for sub in ("oracle", "tests", "scenes"):
        shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                        ignore=shutil.ignore_patterns("__pycache__", "test_oracle_mutations.py"))
    return str(d)


@pytest.mark.slow
@pytest.mark.parametrize("name", list(MUTATIONS))
def test_mutation_fails_a_pin(tree, name):
    src = os.path.join(ROOT, "oracle", "romap_oracle.py")
    orig = open(src).read()
    a, b = MUTATIONS[name]
    assert orig.count(a) == 1, name
    with open(os.path.join(tree, "oracle", "romap_oracle.py"), "w") as f:
        f.write(orig.replace(a, b))
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-x", "-q", "-p", "no:cacheprovider"],
                       cwd=tree, capture_output=True, text=True, timeout=600)
    assert r.returncode == 1 and " failed" in r.stdout, (name, r.stdout[-2000:])

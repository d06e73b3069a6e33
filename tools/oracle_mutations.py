"""Mutation check of the oracle pins: applies plausible
mistakes to oracle/romap_oracle.py one at a time (restoring it afterwards) and
runs tests/test_oracle_pins.py; every mutation must fail at least one pin.
Run: python tools/oracle_mutations.py"""
import subprocess, shutil
P='/root/repo/oracle/romap_oracle.py'
orig=open(P).read()
muts = {
 "u_3a": ("    u = (x + a) / (a + a)\n    return np.minimum", "    u = (x + a) / (a + a + a)\n    return np.minimum"),
 "clamp_dropped": ("    u = (x + a) / (a + a)\n    return np.minimum(np.maximum(u, f32(0.0)), f32(1.0)).astype(f32)", "    u = (x + a) / (a + a)\n    return u.astype(f32)"),
 "cxcy_swap": ("    fx, fy, cx, cy = Ks[:, 0], Ks[:, 1], Ks[:, 2], Ks[:, 3]", "    fx, fy, cx, cy = Ks[:, 0], Ks[:, 1], Ks[:, 3], Ks[:, 2]"),
 "yaw_sign": ("    c, s = box_rotation(yaw)\n    o = np.stack([c * p[0] + s * p[1], c * p[1] - s * p[0], p[2]], axis=1).astype(f32)\n    d = np.stack([c * dw[0] + s * dw[1], c * dw[1] - s * dw[0], dw[2]], axis=1).astype(f32)\n    return o, d, n\n\n\ndef loss_and_grads",
              "    c, s = box_rotation(yaw)\n    s = -s\n    o = np.stack([c * p[0] + s * p[1], c * p[1] - s * p[0], p[2]], axis=1).astype(f32)\n    d = np.stack([c * dw[0] + s * dw[1], c * dw[1] - s * dw[0], dw[2]], axis=1).astype(f32)\n    return o, d, n\n\n\ndef loss_and_grads"),
 "ray_shift4": ("k = mix64(k ^ ((r << U64(8)) | s))", "k = mix64(k ^ ((r << U64(4)) | s))"),
 "bg_stream": ("rng_u32(cfg.seed, st.obj_id, t, ray, 1 + c)", "rng_u32(cfg.seed, st.obj_id, t, ray, 2 + c)"),
 "jitter_stream": ("rng_u32(cfg.seed, st.obj_id, t, ray, 16 + i)", "rng_u32(cfg.seed, st.obj_id, t, ray, 17 + i)"),
 "depth_z": ("depth_t = (zc * n).astype(f32)", "depth_t = (zc * f32(1)).astype(f32)"),
 "obj_t_swap": ("        k = mix64(k ^ U64(obj))\n        k = mix64(k ^ U64(t))", "        k = mix64(k ^ U64(t))\n        k = mix64(k ^ U64(obj))"),
}
try:
    for name,(a,b) in muts.items():
        assert orig.count(a)==1, name
        open(P,'w').write(orig.replace(a,b))
        r=subprocess.run(["python","-m","pytest","tests/test_oracle_pins.py","-q","-x","-p","no:cacheprovider"],cwd="/root/repo",capture_output=True,text=True)
        last=r.stdout.strip().splitlines()[-1]
        print(f"{name:15s} rc={r.returncode} {last}")
finally:
    open(P,'w').write(orig)

"""Shared setup for the GPU parity tests: one scene, identical parameters on
both sides (CUDA path via the C ABI, CPU oracle), identical keyframes."""
import numpy as np

import oracle as O
import scenes


def ocfg_from(kw):
    keys = {f for f in O.ModelConfig.__dataclass_fields__}
    return O.ModelConfig(**{k: v for k, v in kw.items() if k in keys})


KINK = 1e-6


def min_kink_distance(st, t=1):
    """Smallest |pre-activation| of any ReLU (and |D - D_gt| of any depth ray) over
    the samples of iteration t: below ~1e-6 the fp32 kernel and the fp64 oracle may
    take different branches of a kink, so gradient parity is only defined away
    from kinks."""
    _, _, dbg = O.loss_and_grads(st, t)
    fw, W = dbg["fw"], st.params["W"]
    m = min(np.abs(fw["feat"] @ W[0].T).min(), np.abs(fw["cin"] @ W[2].T).min(), np.abs(fw["g"][0] @ W[3].T).min())
    rs = dbg["rays"]
    ia = dbg["active"]
    dep = rs["has_depth"][ia]
    if dep.any():
        m = min(m, np.abs(dbg["vr"]["D"][dep] - rs["depth_t"][ia][dep]).min())
    return m


def make_pair(R, ctx, scene, kw, param_seed=5, obj_id=None, table_scale=0.1, with_depth=True, inst=None,
              avoid_kinks=True):
    """Create the object on the GPU and the matching oracle state (identical
    parameters and keyframes).  avoid_kinks: redraw the parameters until no ReLU
    pre-activation of the first iteration lies within 1e-6 of its kink."""
    cfg = R.model_config(**kw)
    ocfg = ocfg_from(kw)
    ob = scene.objects[0] if inst is None else [o for o in scene.objects if o.instance_id == inst][0]
    h = ctx.create_object(ob.t, ob.yaw, ob.a, cfg, ob.instance_id, obj_id=obj_id)
    st = O.ObjectState(ocfg, np.asarray(ob.t, np.float32), float(np.float32(ob.yaw)), np.asarray(ob.a, np.float32), h,
                       {"table": np.zeros((O.table_entries(ocfg), 2)), "W": [np.zeros(s) for s in O.mlp_shapes(ocfg)]})
    for fr in scene.frames:
        if not (fr.mask == ob.instance_id).any():
            continue
        dep = fr.depth.get(ob.instance_id) if with_depth else None
        ctx.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K, dep)
        st.kfs.append(O.ingest_observation(fr.rgb, fr.mask, fr.T_wc, fr.K, ob.instance_id, dep))
    for attempt in range(20):
        table, W = scenes.random_params(ocfg.levels, 2, O.table_entries(ocfg), O.mlp_shapes(ocfg),
                                        seed=param_seed + 1000 * attempt, table_scale=table_scale)
        st.params = {"table": table.astype(np.float64), "W": [w.astype(np.float64) for w in W]}
        if not avoid_kinks or min_kink_distance(st) > KINK:
            break
    ctx.set_params(h, R.BLOCK_TABLE, table)
    ctx.set_params(h, R.BLOCK_MLP, np.concatenate([w.reshape(-1) for w in W]))
    return h, st


def norm_rel(a, b):
    a = np.asarray(a, np.float64).reshape(-1)
    b = np.asarray(b, np.float64).reshape(-1)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def flat_W(W):
    return np.concatenate([w.reshape(-1) for w in W])

"""Shared setup for the GPU parity tests: one scene, identical parameters on
both sides (CUDA path via the C ABI, CPU oracle), identical keyframes."""
import numpy as np

import oracle as O
import scenes


def ocfg_from(kw):
    keys = {f for f in O.ModelConfig.__dataclass_fields__}
    return O.ModelConfig(**{k: v for k, v in kw.items() if k in keys})


def make_pair(R, ctx, scene, kw, param_seed=5, obj_id=None, table_scale=0.1, with_depth=True, inst=None):
    """Create the object on the GPU and the matching oracle state."""
    cfg = R.model_config(**kw)
    ocfg = ocfg_from(kw)
    ob = scene.objects[0] if inst is None else [o for o in scene.objects if o.instance_id == inst][0]
    h = ctx.create_object(ob.t, ob.yaw, ob.a, cfg, ob.instance_id, obj_id=obj_id)
    table, W = scenes.random_params(ocfg.levels, 2, O.table_entries(ocfg), O.mlp_shapes(ocfg), seed=param_seed,
                                    table_scale=table_scale)
    ctx.set_params(h, R.BLOCK_TABLE, table)
    ctx.set_params(h, R.BLOCK_MLP, np.concatenate([w.reshape(-1) for w in W]))
    P = {"table": table.astype(np.float64), "W": [w.astype(np.float64) for w in W]}
    st = O.ObjectState(ocfg, np.asarray(ob.t, np.float32), float(np.float32(ob.yaw)), np.asarray(ob.a, np.float32), h, P)
    for fr in scene.frames:
        if not (fr.mask == ob.instance_id).any():
            continue
        dep = fr.depth.get(ob.instance_id) if with_depth else None
        ctx.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K, dep)
        st.kfs.append(O.ingest_observation(fr.rgb, fr.mask, fr.T_wc, fr.K, ob.instance_id, dep))
    return h, st


def norm_rel(a, b):
    a = np.asarray(a, np.float64).reshape(-1)
    b = np.asarray(b, np.float64).reshape(-1)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def flat_W(W):
    return np.concatenate([w.reshape(-1) for w in W])

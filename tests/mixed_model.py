"""fp16 precision model of the mixed path (test infrastructure, like oracle/).

The oracle (oracle/romap_oracle.py) computes the method in fp64.  The mixed
CUDA path rounds operands to fp16 at fixed points: the fp16
table copy, the encoded features X0, the weights, the hidden activations and the
backward deltas (x loss scale), with fp32 accumulation.  This module re-runs the
oracle's step with np.float16 roundings inserted at exactly those points (every
other operation as in the oracle), so a test can separate two questions:
  * does the kernel compute what fp16 operands compute?  (GPU vs this model: tight)
  * how far is that from the fp64 method?  (this model vs the oracle: precision)
It reuses the oracle's ray, encoding, rendering and loss functions unchanged and
shares no code with the CUDA path.  Networks 0 (BASELINE) and 1 (the paper's, R24).
round_delta=False / round_forward=False switch the roundings of the backward
deltas / of the forward operands off (to attribute the fp64 gap).
"""
import numpy as np

import oracle as O


def _f16(x):
    return np.asarray(x, np.float64).astype(np.float16).astype(np.float64)


def _ident(x):
    return np.asarray(x, np.float64)


def mixed_loss_and_grads(st, t, scale=128.0, round_forward=True, round_delta=True):
    """(losses, {"table", "W"}) of one iteration with the mixed path's fp16 roundings."""
    if st.cfg.network == 1:
        return _mixed_paper(st, t, scale, round_forward, round_delta)
    cfg, P = st.cfg, st.params
    f16 = _f16 if round_forward else _ident
    d16 = _f16 if round_delta else _ident
    rs = O.forward_rays(st, t)
    N = cfg.samples_per_ray
    ia = np.nonzero(rs["hit"])[0]
    Ra = ia.size
    u = rs["u"][ia].reshape(-1, 3)
    feat, idx, w = O.hash_encode(u, f16(P["table"]), cfg)       # fp16 table copy (p16)
    W = [f16(x) for x in P["W"]]                                # fp16 weights (p16)
    X0 = f16(feat)                                              # encoded features -> fp16 MMA operand
    H1 = f16(np.maximum(X0 @ W[0].T, 0))
    r = H1 @ W[1].T
    sigma = O.density_activation(r[:, 0], cfg.density_act)
    sh = O.sh4(np.repeat(rs["d"][ia], N, axis=0))
    CIN = np.concatenate([f16(r), f16(sh)], 1)
    G1 = f16(np.maximum(CIN @ W[2].T, 0))
    G2 = f16(np.maximum(G1 @ W[3].T, 0))
    c = 1.0 / (1.0 + np.exp(-(G2 @ W[4].T)))
    sig = sigma.reshape(Ra, N)
    rgb = c.reshape(Ra, N, 3)
    Ls = _render_grads(st, rs, ia, sig, rgb, cfg)[0]
    dsig, drgb = _render_grads(st, rs, ia, sig, rgb, cfg)[1:]
    DC = d16(drgb * c * (1 - c) * scale)
    dW = [None] * 5
    dW[4] = DC.T @ G2
    dg2 = d16(DC @ W[4]) * (G2 > 0)
    dW[3] = dg2.T @ G1
    dg1 = d16(dg2 @ W[3]) * (G1 > 0)
    dW[2] = dg1.T @ CIN
    dr = (dg1 @ W[2])[:, :cfg.density_out].copy()
    dr[:, 0] += dsig * O.density_activation_grad(r[:, 0], sigma, cfg.density_act) * scale
    DR = d16(dr)
    dW[1] = DR.T @ H1
    dh1 = d16(DR @ W[1]) * (H1 > 0)
    dW[0] = dh1.T @ X0
    dfeat = dh1 @ W[0] / scale
    g = O.hash_encode_backward(dfeat, idx, w, P["table"].shape[0], cfg.feats)
    return Ls, {"table": g, "W": [x / scale for x in dW]}


def _render_grads(st, rs, ia, sig, rgb, cfg):
    """the oracle's rendering, losses and render backward (fp64), as in loss_and_grads"""
    Ra = ia.size
    cls = rs["cls"][ia]
    bg = rs["bg"][ia].astype(np.float64)
    comp_bg = bg.copy()
    if cfg.obj_bg == 1:
        comp_bg[cls == O.CLS_OBJECT] = 0.0
    vr = O.volume_render(sig, rgb, rs["dist"][ia], rs["delta"][ia], comp_bg)
    B = float(rs["R"])
    Ls, gC, gD = O.losses_and_render_grads(cls, np.ones(Ra, bool), rs["has_depth"][ia], vr["C"], vr["D"],
                                           rs["tgt"][ia].astype(np.float64), bg,
                                           rs["depth_t"][ia].astype(np.float64), sig.sum(1), B, cfg)
    dsig, drgb = O.volume_render_backward(vr, gC, gD, rgb, rs["dist"][ia], rs["delta"][ia], comp_bg)
    dsig = (dsig + np.where(cls == O.CLS_BACKGROUND, cfg.lambda_density / B, 0.0)[:, None]).reshape(-1)
    return Ls, dsig, drgb.reshape(-1, 3)


def _mixed_paper(st, t, scale, round_forward, round_delta):
    """network 1 (R24): X0 fp16, h_k = fp16(relu(h_{k-1} W_k^T)), raw = h_L W_out^T
    (fp32), sigma = act(raw_0), c = sigmoid(raw_1..3); backward: the 16-column
    delta [dsigma act', dc c (1 - c)] x scale and every dh rounded to fp16"""
    cfg, P = st.cfg, st.params
    f16 = _f16 if round_forward else _ident
    d16 = _f16 if round_delta else _ident
    rs = O.forward_rays(st, t)
    N = cfg.samples_per_ray
    ia = np.nonzero(rs["hit"])[0]
    Ra = ia.size
    u = rs["u"][ia].reshape(-1, 3)
    feat, idx, w = O.hash_encode(u, f16(P["table"]), cfg)
    W = [f16(x) for x in P["W"]]
    X0 = f16(feat)
    hs = [f16(np.maximum(X0 @ W[0].T, 0))]
    for k in range(1, cfg.hidden_layers):
        hs.append(f16(np.maximum(hs[-1] @ W[k].T, 0)))
    raw = hs[-1] @ W[-1].T
    sigma = O.density_activation(raw[:, 0], cfg.density_act)
    c = 1.0 / (1.0 + np.exp(-raw[:, 1:4]))
    Ls, dsig, drgb = _render_grads(st, rs, ia, sigma.reshape(Ra, N), c.reshape(Ra, N, 3), cfg)
    draw = np.zeros_like(raw)
    draw[:, 0] = dsig * O.density_activation_grad(raw[:, 0], sigma, cfg.density_act)
    draw[:, 1:4] = drgb * c * (1.0 - c)
    D = d16(draw * scale)
    dW = [None] * len(W)
    dW[-1] = D.T @ hs[-1]
    dh = d16(D @ W[-1]) * (hs[-1] > 0)
    for k in range(cfg.hidden_layers - 1, 0, -1):
        dW[k] = dh.T @ hs[k - 1]
        dh = d16(dh @ W[k]) * (hs[k - 1] > 0)
    dW[0] = dh.T @ X0
    dfeat = dh @ W[0] / scale
    g = O.hash_encode_backward(dfeat, idx, w, P["table"].shape[0], cfg.feats)
    return Ls, {"table": g, "W": [x / scale for x in dW]}

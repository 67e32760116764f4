"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain, slow, fp64 numpy GPT forward/backward — the *definition* that TeraPipe's token-sliced
pipeline must reproduce (BASELINE.json:5, invariant (a)). No autograd, no blocking, no fusion:
every step is the textbook formula, in the order the paper states it.

Model (§3.1):
  * Eq. 1: autoregressive factorisation; input (<sos>, x_1..x_{L-1}) predicts
    x_t. Reading A-8: tokens[B][s+1], x = tokens[:, :s], y = tokens[:, 1:].
  * F = f_N o ... o f_1.
  * Eq. 2: SelfAtt(h_t) = sum_{s<=t} alpha_ts W_V h_s,
    alpha = softmax((W_Q h_t)^T (W_K h_s) / sqrt(H)). Reading A-1: multi-head, scale 1/sqrt(d),
    d = H / n_head (reduces to the paper's formula for one head).
  * Eq. 3: FFN(h) = W_2 sigma(W_1 h + b_1) + b_2; sigma = GeLU-tanh (A-2),
    width 4H (A-4).
  * Pre-LN blocks with final LN (A-3, eps = 1e-5, biased variance); learned absolute positions
    wpe (A-7); untied output head without bias (A-6); mean CE over B*s targets (A-9).

Parity status: pinned (tests/test_oracle_model.py) by central finite differences, by an
independent torch fp64 autograd implementation built from torch.nn.functional library
routines, by closed-form special cases (s = 1, W_q = 0 => prefix mean, W_out = 0 => loss = ln V,
zero layers => multinomial logistic regression), and by the causal invariant of PAPER.md:180.
Absolute loss/logit/gradient VALUES appear nowhere in the paper.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional, Sequence

import numpy as np

LN_EPS = 1e-5
GELU_C = math.sqrt(2.0 / math.pi)


# ---------------------------------------------------------------- elementary ops
def layer_norm(x: np.ndarray, g: np.ndarray, b: np.ndarray):
    """LayerNorm over the last axis (reading A-3). Returns (y, xhat, rstd)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xhat = (x - mu) * rstd
    return xhat * g + b, xhat, rstd


def layer_norm_backward(dy: np.ndarray, xhat: np.ndarray, rstd: np.ndarray, g: np.ndarray):
    """d/dx of LayerNorm: dx = rstd * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat))."""
    dxhat = dy * g
    dx = rstd * (dxhat - dxhat.mean(axis=-1, keepdims=True)
                 - xhat * (dxhat * xhat).mean(axis=-1, keepdims=True))
    red = tuple(range(dy.ndim - 1))
    return dx, (dy * xhat).sum(axis=red), dy.sum(axis=red)


def gelu(u: np.ndarray) -> np.ndarray:
    """sigma of Eq. 3, tanh form (reading A-2)."""
    return 0.5 * u * (1.0 + np.tanh(GELU_C * (u + 0.044715 * u ** 3)))


def gelu_grad(u: np.ndarray) -> np.ndarray:
    z = GELU_C * (u + 0.044715 * u ** 3)
    t = np.tanh(z)
    return 0.5 * (1.0 + t) + 0.5 * u * (1.0 - t * t) * GELU_C * (1.0 + 3.0 * 0.044715 * u * u)


def causal_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray):
    """Eq. 2 for one head. q, k, v: [s, d]. Query t sees keys s <= t.
    Returns (o, P)."""
    s, d = q.shape
    S = (q @ k.T) / math.sqrt(d)
    mask = np.triu(np.ones((s, s), dtype=bool), k=1)   # key index > query index
    S = np.where(mask, -np.inf, S)
    S = S - S.max(axis=-1, keepdims=True)
    P = np.exp(S)
    P = P / P.sum(axis=-1, keepdims=True)
    return P @ v, P


def causal_attention_backward(dO, q, k, v, P):
    d = q.shape[1]
    dV = P.T @ dO
    dP = dO @ v.T
    dS = P * (dP - (dP * P).sum(axis=-1, keepdims=True))
    dQ = dS @ k / math.sqrt(d)
    dK = dS.T @ q / math.sqrt(d)
    return dQ, dK, dV


# ---------------------------------------------------------------- full model
def _wgrad(x: np.ndarray, dy: np.ndarray) -> np.ndarray:
    """dW = sum over all (batch, position) rows of x^T dy, i.e. X^T dY with rows flattened."""
    return x.reshape(-1, x.shape[-1]).T @ dy.reshape(-1, dy.shape[-1])


def _p(params, name):
    return np.asarray(params[name], dtype=np.float64)


def gpt_forward_backward(params: Dict[str, np.ndarray], tokens: np.ndarray, n_layer: int,
                         n_head: int, need_grads: bool = True,
                         keep_layer_outputs: bool = False) -> Dict[str, object]:
    """Unsliced fp64 forward + manual backward of the whole model on tokens[B][s+1].

    Returns {'loss': float, 'logits': [B,s,V], 'grads': {name: array} (if need_grads),
             'layer_in': [h before layer i for i in 0..n] (if keep_layer_outputs),
             'dlayer_in': [dloss/dh before layer i] (if keep_layer_outputs and need_grads)}.
    """
    tokens = np.asarray(tokens)
    B, s1 = tokens.shape
    s = s1 - 1
    x, y = tokens[:, :s], tokens[:, 1:]
    wte, wpe = _p(params, "wte"), _p(params, "wpe")
    V, H = wte.shape
    a = n_head
    d = H // a

    # embedding: h = wte[x] + wpe[0:s] (A-7)
    h = wte[x] + wpe[None, :s, :]
    caches: List[dict] = []
    layer_in = [h.copy()]
    for li in range(n_layer):
        L = lambda n: _p(params, f"l{li}.{n}")
        c = {"h_in": h}
        A1, c["xhat1"], c["rstd1"] = layer_norm(h, L("ln1_g"), L("ln1_b"))
        c["A1"] = A1
        qkv = A1 @ L("w_qkv") + L("b_qkv")                 # [B,s,3H], columns [q | k | v]
        q, k, v = qkv[..., :H], qkv[..., H:2 * H], qkv[..., 2 * H:]
        o = np.zeros_like(q)
        Ps = {}
        for bi in range(B):
            for j in range(a):
                cs = slice(j * d, (j + 1) * d)
                o[bi, :, cs], Ps[bi, j] = causal_attention(q[bi, :, cs], k[bi, :, cs], v[bi, :, cs])
        c.update(q=q, k=k, v=v, o=o, P=Ps)
        h = h + o @ L("w_o") + L("b_o")                    # residual around SelfAtt
        c["h_mid"] = h
        A2, c["xhat2"], c["rstd2"] = layer_norm(h, L("ln2_g"), L("ln2_b"))
        c["A2"] = A2
        U = A2 @ L("w_1") + L("b_1")                       # Eq. 3 inner affine map
        G = gelu(U)
        c.update(U=U, G=G)
        h = h + G @ L("w_2") + L("b_2")                    # residual around FFN
        caches.append(c)
        layer_in.append(h.copy())

    Af, xhatf, rstdf = layer_norm(h, _p(params, "lnf_g"), _p(params, "lnf_b"))
    z = Af @ _p(params, "w_out")                           # logits [B,s,V]
    zmax = z.max(axis=-1, keepdims=True)
    lse = zmax[..., 0] + np.log(np.exp(z - zmax).sum(axis=-1))
    zy = np.take_along_axis(z, y[..., None], axis=-1)[..., 0]
    N = B * s
    loss = float((lse - zy).sum() / N)                     # Eq. 1 as mean NLL (A-9)
    out: Dict[str, object] = {"loss": loss, "logits": z}
    if keep_layer_outputs:
        out["layer_in"] = layer_in
    if not need_grads:
        return out

    grads: Dict[str, np.ndarray] = {}
    # CE backward: dz = (softmax(z) - onehot(y)) / N
    dz = np.exp(z - lse[..., None])
    np.put_along_axis(dz, y[..., None], np.take_along_axis(dz, y[..., None], axis=-1) - 1.0, axis=-1)
    dz /= N
    grads["w_out"] = _wgrad(Af, dz)
    dAf = dz @ _p(params, "w_out").T
    dh, grads["lnf_g"], grads["lnf_b"] = layer_norm_backward(dAf, xhatf, rstdf, _p(params, "lnf_g"))
    dlayer_in = [None] * (n_layer + 1)
    dlayer_in[n_layer] = dh.copy()

    for li in reversed(range(n_layer)):
        L = lambda n: _p(params, f"l{li}.{n}")
        c = caches[li]
        # FFN backward
        grads[f"l{li}.w_2"] = _wgrad(c["G"], dh)
        grads[f"l{li}.b_2"] = dh.sum(axis=(0, 1))
        dG = dh @ L("w_2").T
        dU = dG * gelu_grad(c["U"])
        grads[f"l{li}.w_1"] = _wgrad(c["A2"], dU)
        grads[f"l{li}.b_1"] = dU.sum(axis=(0, 1))
        dA2 = dU @ L("w_1").T
        dx, grads[f"l{li}.ln2_g"], grads[f"l{li}.ln2_b"] = layer_norm_backward(
            dA2, c["xhat2"], c["rstd2"], L("ln2_g"))
        dh = dh + dx
        # attention backward
        grads[f"l{li}.w_o"] = _wgrad(c["o"], dh)
        grads[f"l{li}.b_o"] = dh.sum(axis=(0, 1))
        do = dh @ L("w_o").T
        dq, dk, dv = np.zeros_like(do), np.zeros_like(do), np.zeros_like(do)
        for bi in range(B):
            for j in range(a):
                cs = slice(j * d, (j + 1) * d)
                dq[bi, :, cs], dk[bi, :, cs], dv[bi, :, cs] = causal_attention_backward(
                    do[bi, :, cs], c["q"][bi, :, cs], c["k"][bi, :, cs], c["v"][bi, :, cs], c["P"][bi, j])
        dqkv = np.concatenate([dq, dk, dv], axis=-1)
        grads[f"l{li}.w_qkv"] = _wgrad(c["A1"], dqkv)
        grads[f"l{li}.b_qkv"] = dqkv.sum(axis=(0, 1))
        dA1 = dqkv @ L("w_qkv").T
        dx, grads[f"l{li}.ln1_g"], grads[f"l{li}.ln1_b"] = layer_norm_backward(
            dA1, c["xhat1"], c["rstd1"], L("ln1_g"))
        dh = dh + dx
        dlayer_in[li] = dh.copy()

    # embedding backward: scatter-add into wte rows, wpe rows 0..s-1
    gwte = np.zeros_like(wte)
    np.add.at(gwte, x.reshape(-1), dh.reshape(-1, H))
    gwpe = np.zeros_like(wpe)
    gwpe[:s] = dh.sum(axis=0)
    grads["wte"], grads["wpe"] = gwte, gwpe
    out["grads"] = grads
    if keep_layer_outputs:
        out["dlayer_in"] = dlayer_in
    return out


# ---------------------------------------------------------------- sliced reference (invariant a)
def sliced_attention_layer(q: np.ndarray, k: np.ndarray, v: np.ndarray, dO: np.ndarray,
                           lengths: Sequence[int]):
    """Token-sliced causal attention for one head, the way the pipeline executes it
    (PAPER.md:200-203): forward visits slices in order, appends K/V of slice i to a prefix cache
    and attends rows [c_i, c_i+l_i) to keys [0, c_i+l_i); backward visits slices in REVERSE order
    and pushes dK/dV contributions into all prefix rows, so rows of slice j are final once every
    slice i >= j has been processed. Returns (o, dq, dk, dv) over the whole sequence.

    Parity status: pinned against causal_attention/causal_attention_backward (the unsliced
    definition) — tests/test_oracle_model.py::test_sliced_attention_equals_unsliced."""
    s, d = q.shape
    if sum(lengths) != s or min(lengths) <= 0:
        raise ValueError("lengths must be a composition of s")
    o = np.zeros_like(q)
    Pst = []
    c = 0
    Kc = np.zeros((0, d)); Vc = np.zeros((0, d))
    for l in lengths:
        Kc = np.concatenate([Kc, k[c:c + l]]); Vc = np.concatenate([Vc, v[c:c + l]])
        S = q[c:c + l] @ Kc.T / math.sqrt(d)
        rows = np.arange(c, c + l)[:, None]; cols = np.arange(c + l)[None, :]
        S = np.where(cols > rows, -np.inf, S)
        S = S - S.max(axis=-1, keepdims=True)
        P = np.exp(S); P /= P.sum(axis=-1, keepdims=True)
        o[c:c + l] = P @ Vc
        Pst.append((c, l, P))
        c += l
    dq = np.zeros_like(q); dk = np.zeros_like(k); dv = np.zeros_like(v)
    for (c, l, P) in reversed(Pst):
        dOi = dO[c:c + l]
        dv[:c + l] += P.T @ dOi
        dP = dOi @ v[:c + l].T
        dS = P * (dP - (dOi * o[c:c + l]).sum(axis=-1, keepdims=True))
        dq[c:c + l] = dS @ k[:c + l] / math.sqrt(d)
        dk[:c + l] += dS.T @ q[c:c + l] / math.sqrt(d)
    return o, dq, dk, dv

"""Pins for oracle/model.py against things other than itself (CPU only).

Each test names the passage or mathematical fact it checks. A plausible mistake anywhere in the
oracle (dropped term, wrong sign or index, transposed operand) fails at least one of:
  * torch library routines + autograd (tests/torch_ref.py): every op and every gradient;
  * central finite differences in fp64: every gradient tensor, sampled entries;
  * closed forms: s=1 attention, W_q=0 prefix mean, W_out=0 => loss = ln V, zero layers;
  * the causal dependency property of PAPER.md:180 (logits at t independent of tokens > t);
  * invariant (a) for attention: sliced == unsliced.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import model as om
from synth import CONFIGS, make_params, make_tokens, ModelCfg
from tests.torch_ref import torch_forward_backward

TINY, TINY_B = CONFIGS["tiny"]


def _run(cfg, params, tokens, **kw):
    return om.gpt_forward_backward(params, tokens, cfg.n_layer, cfg.n_head, **kw)


def test_gelu_matches_torch_tanh_gelu():
    u = np.linspace(-6, 6, 1001)
    ref = F.gelu(torch.tensor(u), approximate="tanh").numpy()
    np.testing.assert_allclose(om.gelu(u), ref, rtol=1e-14, atol=1e-15)
    # derivative vs autograd
    t = torch.tensor(u, requires_grad=True)
    F.gelu(t, approximate="tanh").sum().backward()
    np.testing.assert_allclose(om.gelu_grad(u), t.grad.numpy(), rtol=1e-12, atol=1e-14)


def test_layer_norm_matches_torch_and_invariants():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((5, 7, 33)) * 3 + 1
    g, b = rng.standard_normal(33), rng.standard_normal(33)
    y, xhat, rstd = om.layer_norm(x, g, b)
    ref = F.layer_norm(torch.tensor(x), (33,), torch.tensor(g), torch.tensor(b), eps=1e-5).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(xhat.mean(-1), 0, atol=1e-12)               # zero mean rows
    np.testing.assert_allclose((xhat ** 2).mean(-1), 1, atol=1e-4)          # unit variance (eps)


@pytest.mark.parametrize("s,d", [(1, 8), (17, 16), (64, 32)])
def test_attention_matches_sdpa(s, d):
    rng = np.random.default_rng(s)
    q, k, v, dO = (rng.standard_normal((s, d)) for _ in range(4))
    o, P = om.causal_attention(q, k, v)
    tq, tk, tv = (torch.tensor(a, requires_grad=True) for a in (q, k, v))
    to = F.scaled_dot_product_attention(tq[None], tk[None], tv[None], is_causal=True)[0]
    np.testing.assert_allclose(o, to.detach().numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(P.sum(-1), 1.0, atol=1e-14)                  # softmax rows sum to 1
    assert np.all(np.triu(P, 1) == 0)                                       # no key after query
    (to * torch.tensor(dO)).sum().backward()
    dq, dk, dv = om.causal_attention_backward(dO, q, k, v, P)
    np.testing.assert_allclose(dq, tq.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dk, tk.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dv, tv.grad.numpy(), rtol=1e-10, atol=1e-12)


def test_attention_closed_forms():
    rng = np.random.default_rng(0)
    # s = 1: P = 1, o = v
    v = rng.standard_normal((1, 8))
    o, _ = om.causal_attention(rng.standard_normal((1, 8)), rng.standard_normal((1, 8)), v)
    np.testing.assert_allclose(o, v, rtol=0, atol=0)
    # q = 0: uniform weights over the causal prefix => o_t = mean(v_0..v_t)
    s, d = 12, 4
    v = rng.standard_normal((s, d))
    o, _ = om.causal_attention(np.zeros((s, d)), rng.standard_normal((s, d)), v)
    np.testing.assert_allclose(o, np.cumsum(v, 0) / np.arange(1, s + 1)[:, None], atol=1e-14)


@pytest.mark.parametrize("cfg,B", [(TINY, 1), (ModelCfg(2, 32, 2, 40, 9, 1), 3)])
def test_model_matches_torch_autograd(cfg, B):
    params = make_params(cfg, seed=5)
    tokens = make_tokens(cfg, B, seed=6)
    out = _run(cfg, params, tokens)
    loss, z, grads = torch_forward_backward(params, tokens, cfg.n_layer, cfg.n_head)
    assert abs(out["loss"] - loss) <= 1e-12 * abs(loss)
    np.testing.assert_allclose(out["logits"], z, rtol=1e-10, atol=1e-12)
    assert set(grads) == set(out["grads"])
    for k in grads:
        ref = grads[k]
        err = np.linalg.norm(out["grads"][k] - ref) / max(np.linalg.norm(ref), 1e-300)
        assert err < 1e-10, (k, err)


def test_model_finite_differences_every_tensor():
    cfg, B = ModelCfg(2, 16, 2, 24, 6, 1), 2
    params = {k: v.astype(np.float64) for k, v in make_params(cfg, seed=11).items()}
    tokens = make_tokens(cfg, B, seed=12)
    grads = _run(cfg, params, tokens)["grads"]
    rng = np.random.default_rng(13)
    h = 1e-6
    for name, p in params.items():
        flat = p.reshape(-1)
        for idx in rng.choice(flat.size, size=min(3, flat.size), replace=False):
            old = flat[idx]
            flat[idx] = old + h
            lp = _run(cfg, params, tokens, need_grads=False)["loss"]
            flat[idx] = old - h
            lm = _run(cfg, params, tokens, need_grads=False)["loss"]
            flat[idx] = old
            fd = (lp - lm) / (2 * h)
            an = grads[name].reshape(-1)[idx]
            assert abs(fd - an) <= 1e-7 + 1e-5 * abs(an), (name, idx, fd, an)


def test_zero_head_gives_ln_V_and_only_head_gradient():
    params = make_params(TINY, seed=2)
    params["w_out"] = np.zeros_like(params["w_out"])
    tokens = make_tokens(TINY, 2, seed=3)
    out = _run(TINY, params, tokens, keep_layer_outputs=True)
    assert abs(out["loss"] - math.log(TINY.vocab)) < 1e-14
    for k, g in out["grads"].items():
        if k != "w_out":
            assert np.all(g == 0), k
    # dW_out = LN_f(h)^T (1/V - onehot) / N
    hf = out["layer_in"][-1]
    af, _, _ = om.layer_norm(hf, params["lnf_g"].astype(np.float64), params["lnf_b"].astype(np.float64))
    y = tokens[:, 1:]
    dz = np.full(af.shape[:2] + (TINY.vocab,), 1.0 / TINY.vocab)
    for bi in range(y.shape[0]):
        for t in range(y.shape[1]):
            dz[bi, t, y[bi, t]] -= 1.0
    dz /= y.size
    np.testing.assert_allclose(out["grads"]["w_out"], np.einsum("bsh,bsv->hv", af, dz), atol=1e-15)


def test_zero_layers_is_logistic_regression():
    cfg = ModelCfg(0, 8, 2, 11, 5, 1)
    params = make_params(cfg, seed=4)
    tokens = make_tokens(cfg, 3, seed=5)
    out = _run(cfg, params, tokens)
    # textbook multinomial logistic regression on features X = LN_f(wte[x] + wpe)
    x, y = tokens[:, :-1], tokens[:, 1:]
    feats = params["wte"].astype(np.float64)[x] + params["wpe"].astype(np.float64)[None, :5]
    X = F.layer_norm(torch.tensor(feats), (8,), torch.tensor(params["lnf_g"], dtype=torch.float64),
                     torch.tensor(params["lnf_b"], dtype=torch.float64), eps=1e-5).numpy().reshape(-1, 8)
    W = params["w_out"].astype(np.float64)
    from scipy.special import log_softmax, softmax
    Z = X @ W
    nll = -log_softmax(Z, axis=1)[np.arange(Z.shape[0]), y.reshape(-1)].mean()
    assert abs(out["loss"] - nll) < 1e-13
    Y = np.eye(11)[y.reshape(-1)]
    np.testing.assert_allclose(out["grads"]["w_out"], X.T @ (softmax(Z, axis=1) - Y) / Z.shape[0], atol=1e-14)


def test_causal_dependency_property():
    """SelfAtt(h_t) depends only on h_{<=t}, FFN(h_t) only on h_t => logits at
    position t do not change when tokens after t change."""
    params = make_params(TINY, seed=8)
    tokens = make_tokens(TINY, 1, seed=9)
    z0 = _run(TINY, params, tokens, need_grads=False)["logits"]
    t = 13
    tok2 = tokens.copy()
    tok2[:, t + 1:] = (tok2[:, t + 1:] + 7) % TINY.vocab
    z1 = _run(TINY, params, tok2, need_grads=False)["logits"]
    np.testing.assert_array_equal(z0[:, :t + 1], z1[:, :t + 1])
    assert np.abs(z0[:, t + 1:] - z1[:, t + 1:]).max() > 1e-6


@pytest.mark.parametrize("lengths", [[32], [1] * 32, [5, 9, 2, 16], [16, 8, 8], [3, 29]])
def test_sliced_attention_equals_unsliced(lengths):
    """Invariant (a) (BASELINE.json:5) for the attention step, the only cross-token op."""
    rng = np.random.default_rng(len(lengths))
    q, k, v, dO = (rng.standard_normal((32, 16)) for _ in range(4))
    o, P = om.causal_attention(q, k, v)
    dq, dk, dv = om.causal_attention_backward(dO, q, k, v, P)
    so, sdq, sdk, sdv = om.sliced_attention_layer(q, k, v, dO, lengths)
    for a, b in ((o, so), (dq, sdq), (dk, sdk), (dv, sdv)):
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-13)

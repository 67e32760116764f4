"""Independent fp64 reference built from torch library routines + autograd (test-only).

Used to pin oracle/model.py's hand-written backward: gradients here come from torch autograd,
and each layer op is a library routine (F.layer_norm, F.scaled_dot_product_attention with
is_causal=True, F.gelu(approximate='tanh'), F.cross_entropy), so a dropped term, a wrong sign
or a transposed operand in the oracle cannot be reproduced here by construction.
"""
import numpy as np
import torch
import torch.nn.functional as F


def torch_forward_backward(params, tokens, n_layer, n_head):
    P = {k: torch.tensor(np.asarray(v, dtype=np.float64), requires_grad=True) for k, v in params.items()}
    tok = torch.tensor(np.asarray(tokens, dtype=np.int64))
    B, s1 = tok.shape
    s = s1 - 1
    x, y = tok[:, :s], tok[:, 1:]
    V, H = P["wte"].shape
    d = H // n_head
    h = F.embedding(x, P["wte"]) + P["wpe"][:s][None]
    for li in range(n_layer):
        L = lambda n: P[f"l{li}.{n}"]
        a1 = F.layer_norm(h, (H,), L("ln1_g"), L("ln1_b"), eps=1e-5)
        qkv = F.linear(a1, L("w_qkv").T, L("b_qkv"))
        q, k, v = qkv.split(H, dim=-1)
        heads = lambda t: t.view(B, s, n_head, d).transpose(1, 2)
        o = F.scaled_dot_product_attention(heads(q), heads(k), heads(v), is_causal=True)
        o = o.transpose(1, 2).reshape(B, s, H)
        h = h + F.linear(o, L("w_o").T, L("b_o"))
        a2 = F.layer_norm(h, (H,), L("ln2_g"), L("ln2_b"), eps=1e-5)
        g = F.gelu(F.linear(a2, L("w_1").T, L("b_1")), approximate="tanh")
        h = h + F.linear(g, L("w_2").T, L("b_2"))
    af = F.layer_norm(h, (H,), P["lnf_g"], P["lnf_b"], eps=1e-5)
    z = af @ P["w_out"]
    loss = F.cross_entropy(z.reshape(-1, V), y.reshape(-1))
    loss.backward()
    grads = {k: v.grad.detach().numpy() for k, v in P.items()}
    return float(loss.detach()), z.detach().numpy(), grads

"""GPU unit tests of the hot-path kernels through include/tp_kernels.h, against plain PyTorch fp32
math on the same bf16 inputs (and the SIMT kernels against the tensor-core kernels)."""
import math

import numpy as np
import pytest
import torch

import paper_2102_07988_b200 as tp

pytestmark = pytest.mark.gpu
dev = "cuda"


def ptr(t):
    return t.data_ptr()


def rel(a, b):
    a = a.double(); b = b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (200, 384, 320), (37, 136, 72), (512, 5120, 2048),
                                   (1000, 1536, 512), (2048, 2048, 2048), (8, 64, 32),
                                   # partial last wave -> the tail columns run as a second launch
                                   # with half-width tiles (gemm_sm100 tail split), incl. a ragged N
                                   (768, 15360, 256), (768, 15296, 192), (200, 20480, 128)])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 1), (1, 0), (0, 1)])
@pytest.mark.parametrize("impl", [0, 1])
def test_gemm(M, N, K, a_mn, b_mn, impl):
    if impl == 1 and M * N * K > 2 ** 30:
        pytest.skip("SIMT kernel: small shapes only")
    if a_mn and M % 8:
        pytest.skip("MN-major A needs lda = M to be a multiple of 8 (16-byte TMA strides)")
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, generator=g).to(dev, torch.bfloat16)   # logical A[m][k]
    B = torch.randn(N, K, generator=g).to(dev, torch.bfloat16)   # logical B[n][k]
    ref = A.float() @ B.float().T
    Ast = A.T.contiguous() if a_mn else A
    Bst = B.T.contiguous() if b_mn else B
    out = torch.full((M, N), float("nan"), device=dev)
    tp.k_gemm(M, N, K, ptr(Ast), M if a_mn else K, a_mn, ptr(Bst), N if b_mn else K, b_mn, ptr(out), N, impl)
    torch.cuda.synchronize()
    assert rel(out, ref) < 1e-5, rel(out, ref)


@pytest.mark.parametrize("M,N,K", [(8192, 2048, 4096), (768, 15360, 5120), (1024, 5120, 8192), (300, 4096, 8192),
                                   (512, 5120, 20480), (256, 20480, 5120), (1536, 5120, 20480), (200, 2048, 16384)])
def test_gemm_stream_k(M, N, K, monkeypatch):
    """Stream-K (on by default; TP_GEMM_STREAMK=0 disables): whole tiles for all but the last wave, the
    rest cut into one k-block range per unit; partial fp32 tiles in per-unit slots, added by the unit
    that finishes the tile (flags). K-major operands; shapes with < 1 wave and with ragged tails."""
    monkeypatch.setenv("TP_GEMM_STREAMK", "1")
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    A = torch.randn(M, K, generator=g).to(dev, torch.bfloat16)
    B = torch.randn(N, K, generator=g).to(dev, torch.bfloat16)
    ref = A.double() @ B.double().T
    out = torch.full((M, N), float("nan"), device=dev)
    tol = 2e-5 * max(1.0, (K / 4096) ** 0.5)  # fp32 accumulation over K terms (as the dW test)
    for _ in range(2):  # the second launch reuses the workspace (flags reset by the finishers)
        tp.k_gemm(M, N, K, ptr(A), K, 0, ptr(B), K, 0, ptr(out), N, 0)
        torch.cuda.synchronize()
        assert rel(out, ref) < tol, rel(out, ref)
    rr = ((out.double() - ref).norm(dim=1) / ref.norm(dim=1)).max().item()
    assert rr < 1e-4, rr  # a wrong partial / finisher pairing is O(1) off in its rows


@pytest.mark.parametrize("M,N,K", [(2048, 6144, 8192), (2048, 2048, 16384), (8192, 2048, 4096),
                                   (2048, 8192, 16384), (2048, 1024, 8192), (1000, 2048, 4096)])
@pytest.mark.parametrize("wide", [None, "1", "0"])
def test_gemm_weight_grad_shapes(M, N, K, wide, monkeypatch):
    """The deferred weight-gradient GEMMs the bench times (dW = X^T dY, K = B*s, both operands
    MN-major): the 256 x 512 pair tile (<2,256,MN,MN,WN=2>, chosen by the wave model for K >= 4096,
    TP_GEMM_WIDE=1 forces it, =0 disables it) and the MN-major stream-K tail, at the bench's K."""
    if wide is not None:
        monkeypatch.setenv("TP_GEMM_WIDE", wide)
    g = torch.Generator(device="cpu").manual_seed(M + 3 * N + K)
    A = torch.randn(M, K, generator=g).to(dev, torch.bfloat16)
    B = torch.randn(N, K, generator=g).to(dev, torch.bfloat16)
    ref = A.double() @ B.double().T                 # exact products of the bf16 operands
    Ast, Bst = A.T.contiguous(), B.T.contiguous()   # [K][M], [K][N]: MN-major, as X and dY are stored
    out = torch.full((M, N), float("nan"), device=dev)
    # fp32 accumulation over K terms: relative error grows ~ sqrt(K) (1.8e-5 measured at K = 16384)
    tol = 1e-5 * max(1.0, (K / 4096) ** 0.5) * 2
    for _ in range(2):  # the second launch reuses the stream-K tickets
        tp.k_gemm(M, N, K, ptr(Ast), M, 1, ptr(Bst), N, 1, ptr(out), N, 0)
        torch.cuda.synchronize()
        assert rel(out, ref) < tol, rel(out, ref)
    # per output row: a mis-indexed tile or K-part is O(1) off in its rows
    rr = ((out.double() - ref.double()).norm(dim=1) / ref.double().norm(dim=1)).max().item()
    assert rr < 1e-4, rr


def attn_ref(q, k, v, c, l):
    """fp32 math on the bf16 inputs: rows [c, c+l) vs keys [0, c+l), causal at absolute positions."""
    a, s, d = q.shape
    qs = q[:, c:c + l].float()
    ks = k[:, :c + l].float()
    vs = v[:, :c + l].float()
    S = qs @ ks.transpose(1, 2) / math.sqrt(d)
    mask = torch.arange(c + l, device=dev)[None, :] > (c + torch.arange(l, device=dev))[:, None]
    S = S.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(S, -1)
    P = torch.softmax(S, -1)
    return P @ vs, lse, P


@pytest.mark.parametrize("a,s,d,c,l", [(2, 200, 128, 72, 96), (3, 64, 16, 0, 64), (2, 512, 128, 448, 64),
                                       (1, 300, 64, 0, 300), (4, 256, 32, 100, 37), (2, 2048, 128, 1536, 512)])
@pytest.mark.parametrize("impl", [0, 1, 2])
def test_attention_fwd_bwd(a, s, d, c, l, impl):
    g = torch.Generator(device="cpu").manual_seed(a * 1000 + s + c + l)
    q, k, v = (torch.randn(a, s, d, generator=g).to(dev, torch.bfloat16) for _ in range(3))
    o = torch.zeros(l, a * d, device=dev, dtype=torch.bfloat16)
    lse = torch.zeros(a, s, device=dev)
    tp.k_attention_fwd(ptr(q), ptr(k), ptr(v), ptr(o), ptr(lse), a, s, d, c, l, impl)
    torch.cuda.synchronize()
    o_ref, lse_ref, P = attn_ref(q, k, v, c, l)
    o_ref_tok = o_ref.transpose(0, 1).reshape(l, a * d)
    assert rel(o.float(), o_ref_tok) < 1e-2
    assert rel(lse[:, c:c + l], lse_ref) < 1e-4
    # backward with the kernel's own O (bf16) as the saved output
    dO = torch.randn(l, a * d, generator=g).to(dev, torch.bfloat16)
    dq = torch.zeros(l, 3 * a * d, device=dev, dtype=torch.bfloat16)
    dk = torch.full((a, s, d), 0.5, device=dev)
    dv = torch.full((a, s, d), -0.25, device=dev)
    tp.k_attention_bwd(ptr(dO), ptr(o), ptr(q), ptr(k), ptr(v), ptr(lse), ptr(dq), 3 * a * d, ptr(dk), ptr(dv),
                       a, s, d, c, l, 1, impl)
    torch.cuda.synchronize()
    dOh = dO.float().view(l, a, d).transpose(0, 1)                    # [a][l][d]
    Oh = o.float().view(l, a, d).transpose(0, 1)
    dV = P.transpose(1, 2) @ dOh
    dP = dOh @ v[:, :c + l].float().transpose(1, 2)
    Dv = (dOh * Oh).sum(-1, keepdim=True)
    dS = P * (dP - Dv)
    dQ = dS @ k[:, :c + l].float() / math.sqrt(d)
    dK = dS.transpose(1, 2) @ q[:, c:c + l].float() / math.sqrt(d)
    assert rel(dq[:, :a * d].float(), dQ.transpose(0, 1).reshape(l, a * d)) < 2e-2
    assert rel(dk[:, :c + l] - 0.5, dK) < 2e-2
    assert rel(dv[:, :c + l] + 0.25, dV) < 2e-2
    assert torch.all(dk[:, c + l:] == 0.5) and torch.all(dv[:, c + l:] == -0.25)   # rows past c+l untouched
    # accumulate = 0 overwrites
    tp.k_attention_bwd(ptr(dO), ptr(o), ptr(q), ptr(k), ptr(v), ptr(lse), ptr(dq), 3 * a * d, ptr(dk), ptr(dv),
                       a, s, d, c, l, 0, impl)
    torch.cuda.synchronize()
    assert rel(dk[:, :c + l], dK) < 2e-2 and rel(dv[:, :c + l], dV) < 2e-2


@pytest.mark.parametrize("a,s,c,l", [(64, 1536, 264, 1200), (40, 2048, 0, 2048)])
def test_attention_fwd_wide_grid(a, s, c, l):
    """Grids of >= 2 waves of two-tile CTAs take the 64-key double-buffered forward kernel by default
    (attn_sm100.cu dispatch): unaligned prefix c, a ragged last tile pair (l = 1200: 48 rows in its
    second tile), full causal s = 2048; O per element and lse against fp32 math on the same inputs."""
    d = 128
    g = torch.Generator(device="cpu").manual_seed(a + s + c + l)
    q, k, v = (torch.randn(a, s, d, generator=g).to(dev, torch.bfloat16) for _ in range(3))
    o = torch.zeros(l, a * d, device=dev, dtype=torch.bfloat16)
    lse = torch.zeros(a, s, device=dev)
    tp.k_attention_fwd(ptr(q), ptr(k), ptr(v), ptr(o), ptr(lse), a, s, d, c, l, 0)
    torch.cuda.synchronize()
    o_ref, lse_ref, _ = attn_ref(q, k, v, c, l)
    o_ref_tok = o_ref.transpose(0, 1).reshape(l, a * d)
    assert rel(o.float(), o_ref_tok) < 1e-2
    assert (o.float() - o_ref_tok).abs().max() < 0.05
    assert rel(lse[:, c:c + l], lse_ref) < 1e-4
    assert torch.all(lse[:, :c] == 0) and torch.all(lse[:, c + l:] == 0)


@pytest.mark.parametrize("rows,H", [(1, 8), (7, 136), (300, 2048), (4099, 2048), (16384, 2048), (33, 1000),
                                    (513, 5120), (64, 12288)])
@pytest.mark.parametrize("with_resid", [False, True])
def test_layernorm_fwd_bwd(rows, H, with_resid):
    """LayerNorm fwd / bwd kernels (bulk-staged for H <= 2048, register kernels above) against the
    fp64 definition (reading A-3) on the same fp32 x and bf16 dy: ragged row counts (partial last
    CTA, rows < warps of one CTA), H not a multiple of 256 (masked lanes), the 1B / 13B / 175B widths."""
    g = torch.Generator(device="cpu").manual_seed(rows * 31 + H)
    x = (torch.randn(rows, H, generator=g) * 2 + 0.5).to(dev)
    gam = (1 + 0.1 * torch.randn(H, generator=g)).to(dev)
    bet = (0.1 * torch.randn(H, generator=g)).to(dev)
    dy = torch.randn(rows, H, generator=g).to(dev, torch.bfloat16)
    resid = torch.randn(rows, H, generator=g).to(dev) if with_resid else None
    y = torch.empty(rows, H, device=dev, dtype=torch.bfloat16)
    mean = torch.empty(rows, device=dev)
    rstd = torch.empty(rows, device=dev)
    tp.k_layernorm_fwd(ptr(x), ptr(gam), ptr(bet), ptr(y), ptr(mean), ptr(rstd), rows, H)
    dx = torch.empty(rows, H, device=dev)
    dxc = torch.empty(rows, H, device=dev, dtype=torch.bfloat16)
    dg = torch.zeros(H, device=dev); db = torch.zeros(H, device=dev); dbias = torch.full((H,), 0.25, device=dev)
    tp.k_layernorm_bwd(ptr(dy), ptr(x), ptr(mean), ptr(rstd), ptr(gam), ptr(resid) if with_resid else None, ptr(dx),
                       ptr(dxc), ptr(dg), ptr(db), ptr(dbias), rows, H)
    torch.cuda.synchronize()
    xd = x.double().cpu().requires_grad_(True)
    mu = xd.mean(1, keepdim=True)
    var = ((xd - mu) ** 2).mean(1, keepdim=True)
    xhat = (xd - mu) / torch.sqrt(var + 1e-5)
    yd = xhat * gam.double().cpu() + bet.double().cpu()
    (gx,) = torch.autograd.grad(yd, xd, dy.double().cpu())
    if with_resid:
        gx = gx + resid.double().cpu()
    assert rel(mean.cpu(), mu[:, 0].detach()) < 1e-6
    assert rel(rstd.cpu(), (1 / torch.sqrt(var + 1e-5))[:, 0].detach()) < 1e-5
    assert rel(y.cpu(), yd.detach()) < 5e-3
    assert (y.cpu().double() - yd.detach()).abs().max() < 1e-2 * (1 + yd.detach().abs().max())
    assert rel(dx.cpu(), gx) < 1e-5
    assert rel(dxc.cpu(), gx) < 5e-3
    assert rel(dg.cpu(), (dy.double().cpu() * xhat.detach()).sum(0)) < 1e-4
    assert rel(db.cpu(), dy.double().cpu().sum(0)) < 1e-4
    assert rel(dbias.cpu() - 0.25, gx.sum(0)) < 1e-4

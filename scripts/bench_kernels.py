"""Per-kernel timing of the hot-path kernels through include/tp_kernels.h (CUDA events, median of
reps, inputs > L2 rotated). Prints one JSON line per shape: TFLOP/s vs the measured peak."""
import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_07988_b200 as tp  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["bf16_tflops"] \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 1590.0


def time_it(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def gemm(M, N, K, a_mn=0, b_mn=0, impl=0, tag=""):
    A = torch.randn(K, M, device="cuda").to(torch.bfloat16) if a_mn else torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(K, N, device="cuda").to(torch.bfloat16) if b_mn else torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda")
    f = lambda: tp.k_gemm(M, N, K, A.data_ptr(), M if a_mn else K, a_mn, B.data_ptr(), N if b_mn else K, b_mn,
                          out.data_ptr(), N, impl)
    ms = time_it(f)
    fl = 2.0 * M * N * K
    ref = torch.matmul(A.T if a_mn else A, (B if b_mn else B.T))
    t_ref = time_it(lambda: torch.matmul(A.T if a_mn else A, (B if b_mn else B.T)))
    print(json.dumps({"kernel": "gemm", "tag": tag, "M": M, "N": N, "K": K, "a_mn": a_mn, "b_mn": b_mn,
                      "ms": ms, "tflops": fl / ms / 1e9, "frac_peak": fl / ms / 1e9 / PEAK,
                      "cublas_ms": t_ref, "cublas_tflops": fl / t_ref / 1e9}), flush=True)


def attn(a, s, d, c, l, impl=0, tag=""):
    q, k, v = (torch.randn(a, s, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    o = torch.empty(l, a * d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(a, s, device="cuda")
    ms = time_it(lambda: tp.k_attention_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(),
                                            a, s, d, c, l, impl))
    fl = 4.0 * a * d * (l * c + l * (l + 1) / 2)
    dO = torch.randn(l, a * d, device="cuda").to(torch.bfloat16)
    dq = torch.empty(l, 3 * a * d, device="cuda", dtype=torch.bfloat16)
    dk = torch.zeros(a, s, d, device="cuda")
    dv = torch.zeros(a, s, d, device="cuda")
    msb = time_it(lambda: tp.k_attention_bwd(dO.data_ptr(), o.data_ptr(), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                             lse.data_ptr(), dq.data_ptr(), 3 * a * d, dk.data_ptr(), dv.data_ptr(),
                                             a, s, d, c, l, 1, impl))
    print(json.dumps({"kernel": "attention", "tag": tag, "a": a, "s": s, "d": d, "c": c, "l": l,
                      "fwd_ms": ms, "fwd_tflops": fl / ms / 1e9, "bwd_ms": msb, "bwd_tflops": 2 * fl / msb / 1e9}),
          flush=True)


def layernorm(rows, H, tag=""):
    """LayerNorm fwd / bwd (the bench's resid + dx_copy form) at algorithmic bytes: fwd 4H in + 2H out,
    bwd 2H (dy) + 4H (x) + 4H (resid) in, 4H + 2H out, per row. NB buffer sets rotate so the
    working set (> 2x the 126 MB L2) is not cache-resident between launches."""
    NB = 3
    xs = [torch.randn(rows, H, device="cuda") for _ in range(NB)]
    ys = [torch.empty(rows, H, device="cuda", dtype=torch.bfloat16) for _ in range(NB)]
    dys = [torch.randn(rows, H, device="cuda").to(torch.bfloat16) for _ in range(NB)]
    rs = [torch.randn(rows, H, device="cuda") for _ in range(NB)]
    dxs = [torch.empty(rows, H, device="cuda") for _ in range(NB)]
    dcs = [torch.empty(rows, H, device="cuda", dtype=torch.bfloat16) for _ in range(NB)]
    gam, bet = torch.ones(H, device="cuda"), torch.zeros(H, device="cuda")
    mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
    dg, db, dbias = (torch.zeros(H, device="cuda") for _ in range(3))
    it = [0]

    def f():
        i = it[0] % NB
        it[0] += 1
        tp.k_layernorm_fwd(xs[i].data_ptr(), gam.data_ptr(), bet.data_ptr(), ys[i].data_ptr(), mean.data_ptr(),
                           rstd.data_ptr(), rows, H)

    def b():
        i = it[0] % NB
        it[0] += 1
        tp.k_layernorm_bwd(dys[i].data_ptr(), xs[i].data_ptr(), mean.data_ptr(), rstd.data_ptr(), gam.data_ptr(),
                           rs[i].data_ptr(), dxs[i].data_ptr(), dcs[i].data_ptr(), dg.data_ptr(), db.data_ptr(),
                           dbias.data_ptr(), rows, H)
    msf, msb = time_it(f), time_it(b)
    bf, bb = 6.0 * H * rows, 16.0 * H * rows
    print(json.dumps({"kernel": "layernorm", "tag": tag, "rows": rows, "H": H, "bulk": os.environ.get("TP_LN_BULK", "1"),
                      "fwd_us": msf * 1e3, "fwd_gbs": bf / msf / 1e6, "bwd_us": msb * 1e3, "bwd_gbs": bb / msb / 1e6}),
          flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="all")
    ap.add_argument("--filter", default="")
    args = ap.parse_args()
    if args.which in ("all", "gemm"):
        H = 2048
        for (M, N, K, am, bm, tag) in [(2048, 3 * H, H, 0, 0, "1b qkv fwd"), (2048, H, 4 * H, 0, 0, "1b fc2 fwd"),
                                       (2048, 4 * H, H, 0, 0, "1b fc1 fwd"), (2048, 50304, H, 0, 0, "1b head fwd"),
                                       (H, 3 * H, 2048, 1, 1, "1b qkv dW"), (4 * H, H, 2048, 1, 1, "1b fc2 dW"),
                                       (512, 15360, 5120, 0, 0, "13b qkv fwd l=512"),
                                       (512, 5120, 20480, 0, 0, "13b fc2 fwd l=512"),
                                       (5120, 15360, 2048, 1, 1, "13b qkv dW"),
                                       (256, 20480, 5120, 0, 0, "13b fc1 l=256"), (8192, 8192, 8192, 0, 0, "square"),
                                       # partial last waves (stream-K tail / tail split)
                                       (8192, H, H, 0, 0, "1b o-proj b=4 (3.46 waves)"),
                                       (8192, H, 4 * H, 0, 0, "1b fc2 b=4 (3.46 waves)"),
                                       (768, 15360, 5120, 0, 0, "13b qkv b=2 l=384 (2.43 waves)"),
                                       (1536, 5120, 20480, 0, 0, "13b fc2 b=2 l=768 (1.62 waves)"),
                                       # the 1B bench's jobs: b = 8 x l = 576 / 1472, and its dW (K = B s)
                                       (4608, 3 * H, H, 0, 0, "1b qkv b=8 l=576"), (11776, 3 * H, H, 0, 0, "1b qkv b=8 l=1472"),
                                       (11776, H, H, 0, 0, "1b o-proj b=8 l=1472"), (11776, 4 * H, H, 0, 0, "1b fc1 b=8 l=1472"),
                                       (11776, H, 4 * H, 0, 0, "1b fc2 b=8 l=1472"), (11776, 50304, H, 0, 0, "1b head l=1472"),
                                       (H, 3 * H, 16384, 1, 1, "1b qkv dW K=16384"), (4 * H, H, 16384, 1, 1, "1b fc2 dW K=16384"),
                                       (H, 4 * H, 16384, 1, 1, "1b fc1 dW K=16384"),
                                       # the default N = 1 bench plan [(8, [2048])]: T = 16384 rows
                                       (16384, 3 * H, H, 0, 0, "T=16384 qkv fwd"), (16384, H, H, 0, 0, "T=16384 o-proj fwd"),
                                       (16384, 4 * H, H, 0, 0, "T=16384 fc1 fwd"), (16384, H, 4 * H, 0, 0, "T=16384 fc2 fwd"),
                                       (16384, 50304, H, 0, 0, "T=16384 head fwd"), (16384, H, 3 * H, 0, 1, "T=16384 qkv dX"),
                                       (16384, H, 4 * H, 0, 1, "T=16384 fc1 dX"), (16384, 4 * H, H, 0, 1, "T=16384 fc2 dX"),
                                       (16384, H, 50304, 0, 1, "T=16384 head dX"), (4 * H, H, 16384, 1, 1, "T=16384 fc2 dW")]:
            if args.filter in tag:
                gemm(M, N, K, am, bm, 0, tag)
    if args.which in ("all", "attn"):
        for (a, s, d, c, l, tag) in [(16, 2048, 128, 0, 2048, "1b full"), (40, 2048, 128, 1536, 512, "13b last slice"),
                                     (40, 2048, 128, 0, 512, "13b first slice"), (40, 8192, 128, 7680, 512, "13b-8k last")]:
            attn(a, s, d, c, l, 0, tag)
    if args.which in ("all", "ln"):
        for (rows, H, tag) in [(16384, 2048, "1b b=8 l=2048"), (4608, 2048, "1b b=8 l=576"),
                               (11776, 2048, "1b b=8 l=1472"), (4096, 5120, "13b b=8 l=512")]:
            layernorm(rows, H, tag)

"""Times the slice-vs-prefix attention kernels alone through tp_kernels.h (CUDA events, median of
reps) at a job shape of the bench: heads a (a = 16 heads x 8 sequences of the 1B bench -> a = 128),
prefix s, slice [c, c+l). Prints TFLOP/s with the algorithmic FLOPs 4 (fwd) / 8 (bwd) H (l c +
l (l+1) / 2).

  python scripts/attn_bench.py [a s c l reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_07988_b200 as tp  # noqa: E402

a, s, c, l, reps = [int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (128, 2048, 576, 1472, 20))]
d = 128
torch.manual_seed(0)
q, k, v = (torch.randn(a, s, d, device="cuda").to(torch.bfloat16) for _ in range(3))
o = torch.zeros(l, a * d, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(a, s, device="cuda")
dO = torch.randn(l, a * d, device="cuda").to(torch.bfloat16)
dq = torch.zeros(l, 3 * a * d, device="cuda", dtype=torch.bfloat16)
dk = torch.zeros(a, s, d, device="cuda")
dv = torch.zeros(a, s, d, device="cuda")
H = a * d
fl = H * (l * c + l * (l + 1) / 2)


def timeit(f):
    for _ in range(3):
        f()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


fwd = lambda: tp.k_attention_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), a, s, d, c, l, 0)
bwd = lambda acc: tp.k_attention_bwd(dO.data_ptr(), o.data_ptr(), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                     lse.data_ptr(), dq.data_ptr(), 3 * a * d, dk.data_ptr(), dv.data_ptr(), a, s, d,
                                     c, l, acc, 0)
tf = timeit(fwd)
tb0 = timeit(lambda: bwd(0))
tb1 = timeit(lambda: bwd(1))
print(f"a={a} s={s} c={c} l={l}: fwd {tf * 1e3:.1f} us {4 * fl / tf / 1e9:.0f} TF/s | bwd store {tb0 * 1e3:.1f} us "
      f"{8 * fl / tb0 / 1e9:.0f} TF/s | bwd reduce-add {tb1 * 1e3:.1f} us {8 * fl / tb1 / 1e9:.0f} TF/s", flush=True)

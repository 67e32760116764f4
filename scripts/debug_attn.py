"""One small slice-vs-prefix attention fwd+bwd through tp_kernels.h, compared with torch fp32 math
(debug aid for the tcgen05 kernels; the full checks are tests/test_gpu_kernels.py)."""
import math
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2102_07988_b200 as tp  # noqa: E402

a, s, d, c, l = [int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (1, 128, 128, 0, 64))]
impl = int(sys.argv[6]) if len(sys.argv) > 6 else 0
torch.manual_seed(0)
q, k, v = (torch.randn(a, s, d, device="cuda").to(torch.bfloat16) for _ in range(3))
o = torch.zeros(l, a * d, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(a, s, device="cuda")
tp.k_attention_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), a, s, d, c, l, impl)
torch.cuda.synchronize()
print("fwd ok", flush=True)
dO = torch.randn(l, a * d, device="cuda").to(torch.bfloat16)
dq = torch.zeros(l, a * d, device="cuda", dtype=torch.bfloat16)
dk = torch.zeros(a, s, d, device="cuda")
dv = torch.zeros(a, s, d, device="cuda")
tp.k_attention_bwd(dO.data_ptr(), o.data_ptr(), q.data_ptr(), k.data_ptr(), v.data_ptr(), lse.data_ptr(), dq.data_ptr(),
                   a * d, dk.data_ptr(), dv.data_ptr(), a, s, d, c, l, 0, impl)
torch.cuda.synchronize()
print("bwd ran", flush=True)
qs, ks, vs = q[:, c:c + l].float(), k[:, :c + l].float(), v[:, :c + l].float()
S = qs @ ks.transpose(1, 2) / math.sqrt(d)
mask = torch.arange(c + l, device="cuda")[None, :] > (c + torch.arange(l, device="cuda"))[:, None]
P = torch.softmax(S.masked_fill(mask, float("-inf")), -1)
dOh = dO.float().view(l, a, d).transpose(0, 1)
Oh = o.float().view(l, a, d).transpose(0, 1)
dV = P.transpose(1, 2) @ dOh
dS = P * (dOh @ vs.transpose(1, 2) - (dOh * Oh).sum(-1, keepdim=True))
dQ = dS @ ks / math.sqrt(d)
dK = dS.transpose(1, 2) @ qs / math.sqrt(d)
rel = lambda x, y: float((x - y).norm() / y.norm())
print("dq", rel(dq.float(), dQ.transpose(0, 1).reshape(l, a * d)), "dk", rel(dk[:, :c + l], dK), "dv",
      rel(dv[:, :c + l], dV))

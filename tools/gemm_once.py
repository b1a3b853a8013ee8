"""One gated GEMM launch (for ncu): python tools/gemm_once.py M N K MODE"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_07874_b200 import api as A  # noqa: E402

m, n, k, mode = (int(x) for x in sys.argv[1:5])
a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
b = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
g = A.Gate(0)
for _ in range(3):
    g.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, fresh=True, mode=mode)
torch.cuda.synchronize()
torch.matmul(a, b.t(), out=c)
torch.cuda.synchronize()

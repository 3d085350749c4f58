import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2206_15143_b200 import _lib as L, ops
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
a = torch.randn(n, n, device="cuda"); o = torch.empty(n, n, device="cuda")
j = L.GemmJob(); j.a = ops.operand_rows_k(a); j.b = ops.operand_rows_k(a); j.out, j.ldo = o.data_ptr(), n; j.alpha = 1.0
for _ in range(3): ops.gemm([j], "tf32")
torch.cuda.synchronize()

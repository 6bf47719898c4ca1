import os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2206_01861_b200 import quant
x = torch.randn(4096, 3072, device="cuda")
for _ in range(3):
    quant.quantize_activation_tokenwise(x, 8, check_finite=False)
torch.cuda.synchronize()

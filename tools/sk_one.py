import os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2206_01861_b200 import _native as N
from paper_2206_01861_b200 import quant
M, k, n = 16, 4096, 4096
w = quant.padded_int8(n, k, align=32); w.copy_(torch.randint(-127, 128, (n, k), device="cuda", dtype=torch.int8))
rs = torch.rand(n, device="cuda") * 1e-3
xq = quant.padded_int8(M, k); xq.copy_(torch.randint(-127, 128, (M, k), device="cuda", dtype=torch.int8))
ts = torch.rand(M, device="cuda"); out = torch.empty(M, n, device="cuda")
nb = int(N.load().zq_linear_ws_bytes(M, n)); skws = torch.zeros(nb // 4 + 4, dtype=torch.int32, device="cuda")
for i in range(3):
    N.call("zq_linear_ws", xq.data_ptr(), xq.stride(0), ts.data_ptr(), 0.0, w.data_ptr(), w.stride(0), 8,
           rs.data_ptr(), None, M, n, k, out.data_ptr(), out.stride(0), N.OUT_F32, skws.data_ptr(), 4 * skws.numel(), N.stream_ptr())
    N.call("zq_linear", xq.data_ptr(), xq.stride(0), ts.data_ptr(), 0.0, w.data_ptr(), w.stride(0), 8,
           rs.data_ptr(), None, M, n, k, out.data_ptr(), out.stride(0), N.OUT_F32, N.stream_ptr())
torch.cuda.synchronize()

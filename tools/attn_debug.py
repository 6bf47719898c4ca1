import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import transformer as T, _native as N
batch, seq, heads, dh = 2, 128, 12, 64
d = heads * dh
torch.manual_seed(0)
qkv = torch.randn(batch * seq, 3 * d, device="cuda")
ctx = torch.full((batch * seq, d), 7.0, device="cuda")
lib = N.load()
rc = lib.zq_attention_f32(qkv.data_ptr(), qkv.stride(0), batch, seq, heads, dh, 0, 0.125, ctx.data_ptr(), d, N.stream_ptr())
torch.cuda.synchronize()
print("rc", rc, "absmax", ctx.abs().max().item(), "n==7", (ctx == 7).sum().item(), "n==0", (ctx == 0).sum().item())
q, k, v = (qkv[:, i * d:(i + 1) * d].double().reshape(batch, seq, heads, dh).transpose(1, 2) for i in range(3))
p = torch.softmax((q @ k.transpose(-1, -2)) * 0.125, -1)
ref = (p @ v).transpose(1, 2).reshape(batch * seq, d)
print("rel", ((ctx.double() - ref).norm() / ref.norm()).item())
print("ctx[0,:8]", ctx[0, :8].tolist()); print("ref[0,:8]", ref[0, :8].tolist())
vm = qkv[:, 2 * d:].reshape(batch, seq, heads, dh).mean(1)
print("vmean[0,0,:8]", vm[0, 0, :8].tolist())
import numpy as np
lib.zq_attention_debug.argtypes = [__import__("ctypes").c_int]
for mode in []:
    ctx.fill_(7.0)
    lib.zq_attention_debug(mode)
    lib.zq_attention_f32(qkv.data_ptr(), qkv.stride(0), batch, seq, heads, dh, 0, 0.125, ctx.data_ptr(), d, N.stream_ptr())
    torch.cuda.synchronize()
    flat = ctx.reshape(-1)[: 8192 * (2 if mode == 7 else 1)].cpu().numpy()
    print("mode", mode, "nz", int((flat != 0).sum()), "first", flat[:6].tolist(), "row1", flat[32:36].tolist())
print("q00", qkv[0, :6].tolist(), "k00", qkv[0, d:d + 6].tolist(), "v00", qkv[0, 2 * d:2 * d + 6].tolist(), "v10", qkv[1, 2*d:2*d+4].tolist())
for mode in (0, 30):
    ctx.fill_(7.0)
    lib.zq_attention_debug(mode)
    lib.zq_attention_f32(qkv.data_ptr(), qkv.stride(0), batch, seq, heads, dh, 0, 0.125, ctx.data_ptr(), d, N.stream_ptr())
    torch.cuda.synchronize()
    print("pv mode", mode, "absmax", ctx.abs().max().item(), "rel", ((ctx.double() - ref).norm() / ref.norm()).item(), ctx[0, :4].tolist())
batch = 32
qkv = torch.randn(batch * seq, 3 * d, device="cuda")
ctx = torch.zeros((batch * seq, d), device="cuda")
lib.zq_attention_debug(20)
for _ in range(3):
    lib.zq_attention_f32(qkv.data_ptr(), qkv.stride(0), batch, seq, heads, dh, 0, 0.125, ctx.data_ptr(), d, N.stream_ptr())
torch.cuda.synchronize()
st = ctx.reshape(-1).view(torch.int64)[: batch * heads * 8].reshape(-1, 8).cpu().numpy()
t0 = st[:, 0].min()
print("kernel span us", (st[:, 7].max() - t0) / 1e3)
ph = np.diff(st, axis=1) / 1e3
print("phase means us (alloc, tma, split, S, softmax, PV, store)", ph.mean(0).round(2).tolist())
print("phase max", ph.max(0).round(2).tolist())
starts = np.sort((st[:, 0] - t0) / 1e3)
print("start times (first 10, 148-158, last 5)", starts[:10].round(2).tolist(), starts[148:158].round(2).tolist(), starts[-5:].round(2).tolist())

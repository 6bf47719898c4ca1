"""Megatron tensor parallelism for the GPT-scale ZeroQuant blocks (SURVEY.md §8e,
north_star (d)): one process per GPU, torch.distributed over NCCL.

Column-parallel: w_q, w_k, w_v, w_h4h are split along output channels (heads
for q/k/v), so the replicated input x is quantized identically on every rank.
Row-parallel: w_o, w_4hh are split along K.  For bit-exact parity with the
single-GPU reference (transformer.py:443-486):

  1. token scales need the max over the FULL row: local row |x| max ->
     all_reduce(MAX) (float bit patterns of non-negative values, exact);
  2. quantize the local K slice with the global scale;
  3. local int8 x int8 -> int32 partial GEMM;
  4. ONE all_reduce(SUM) of the int32 partials per row-parallel projection —
     integer addition is associative, so the sum is exact and order-free;
  5. the dequant epilogue (+ bias once) then runs replicated.

Weights are quantized globally (group scales from the whole matrix, as the
reference does) and then sharded; per-row scales make any row split exact.

The algorithm is written against a small `ops` interface so the sharding and
collective sequencing can be tested on CPU with gloo (tests inject the oracle);
production uses `CudaOps`, which calls the sm_100a kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .errors import UsageError

LN_EPS = 1e-5


@dataclass
class ShardedBlock:
    """One rank's slice of a quantized block.

    Weight entries are opaque to this module (whatever `ops` understands):
    the sharding below only slices rows / columns of the int8 payload and the
    per-row scale vectors, which `ops.slice_rows` / `ops.slice_cols` perform."""

    w_qkv: object      # column-parallel: this rank's heads of q, k, v (stacked)
    b_qkv: object
    w_o: object        # row-parallel: all d rows, K columns of this rank's heads
    b_o: object        # full bias (added once, after the all-reduce)
    w_h4h: object      # column-parallel slice of the FFN up-projection
    b_h4h: object
    w_4hh: object      # row-parallel slice (K) of the FFN down-projection
    b_4hh: object
    ln1: tuple
    ln2: tuple
    heads_local: int
    dim: int


def shard_block(block, ops, rank: int, world: int) -> ShardedBlock:
    """Slice a globally quantized block (transformer.DeviceBlock-like) for `rank`."""
    d = ops.rows(block.w_q)
    heads = block.num_heads
    if heads % world or ops.rows(block.w_h4h) % world:
        raise UsageError(f"{heads} heads / {ops.rows(block.w_h4h)} FFN rows not divisible by TP degree {world}")
    dh = d // heads
    hl = heads // world
    c0, c1 = rank * hl * dh, (rank + 1) * hl * dh
    f = ops.rows(block.w_h4h)
    f0, f1 = rank * f // world, (rank + 1) * f // world
    w_qkv = ops.stack_rows([ops.slice_rows(block.w_q, c0, c1), ops.slice_rows(block.w_k, c0, c1),
                            ops.slice_rows(block.w_v, c0, c1)])
    b_qkv = ops.cat([block.b_q[c0:c1], block.b_k[c0:c1], block.b_v[c0:c1]])
    return ShardedBlock(
        w_qkv=w_qkv, b_qkv=b_qkv,
        w_o=ops.slice_cols(block.w_o, c0, c1), b_o=block.b_o,
        w_h4h=ops.slice_rows(block.w_h4h, f0, f1), b_h4h=block.b_h4h[f0:f1],
        w_4hh=ops.slice_cols(block.w_4hh, f0, f1), b_4hh=block.b_4hh,
        ln1=(block.ln1_gamma, block.ln1_beta), ln2=(block.ln2_gamma, block.ln2_beta),
        heads_local=hl, dim=d)


def row_parallel_linear(ops, x_local, w_local, bias, group, out=None):
    """Steps 1-5 above for one row-parallel projection.  This is the one
    implementation: `tp_block_forward` and `decoder.DecoderEngine` (world > 1,
    or `force_tp`) both call it.  `out` (optional) receives the epilogue."""
    amax = ops.row_absmax(x_local)
    dist.all_reduce(amax, op=dist.ReduceOp.MAX, group=group)
    xq, scales = ops.quantize_with_absmax(x_local, amax)
    acc = ops.igemm_s32(xq, w_local)
    dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return ops.epilogue(acc, scales, w_local, bias, out=out)



def tp_block_forward(x, sb: ShardedBlock, ops, causal: bool, group=None, batch: int = 1):
    """One W8A8 post-LN block (transformer.py:443-486) under tensor parallelism.
    `x` is replicated on every rank; the result is replicated."""
    xq, xs = ops.quantize_tokenwise(x)
    qkv = ops.linear(xq, xs, sb.w_qkv, sb.b_qkv)          # column-parallel, no comm
    dl = ops.cols(qkv) // 3
    ctx = ops.attention(qkv, dl, sb.heads_local, causal, batch)
    attn_out = row_parallel_linear(ops, ctx, sb.w_o, sb.b_o, group)
    h, hq, hs = ops.ln_quant(x, attn_out, *sb.ln1)
    u = ops.linear(hq, hs, sb.w_h4h, sb.b_h4h)              # column-parallel
    z = ops.gelu(u)                                          # exact float GeLU, local columns
    f = row_parallel_linear(ops, z, sb.w_4hh, sb.b_4hh, group)
    y, _, _ = ops.ln_quant(h, f, *sb.ln2)
    return y


# ---------------------------------------------------------------------------
# production ops: the sm_100a kernels
# ---------------------------------------------------------------------------


class CudaOps:
    """`ops` implementation over libzq_b200 (device tensors).

    `flag` (an int32 device tensor) collects non-finite detections; by default
    a private one.  With `reuse=True` the row-parallel workspaces (absmax,
    int8 slice, token scales, int32 partials) are kept per (rows, cols) and
    reused, so a decode step issues no allocations (CUDA-graph friendly)."""

    def __init__(self, flag=None, reuse: bool = False):
        from . import _native, igemm, quant

        self.N, self.igemm, self.quant = _native, igemm, quant
        if flag is None:
            self.flag = quant.FiniteFlag()
        else:
            self.flag = quant.FiniteFlag.__new__(quant.FiniteFlag)
            self.flag.t = flag
        self.reuse = reuse
        self._ws: dict = {}

    def _buf(self, key, make):
        if not self.reuse:
            return make()
        if key not in self._ws:
            self._ws[key] = make()
        return self._ws[key]

    # --- weight container plumbing ---
    @staticmethod
    def rows(w):
        return w.rows

    @staticmethod
    def cols(t):
        return t.shape[1]

    @staticmethod
    def cat(ts):
        return torch.cat(ts).contiguous()

    def slice_rows(self, w, r0, r1):
        q = self.quant
        v = w.values[r0:r1]
        store = torch.zeros((r1 - r0, w.ld), dtype=torch.int8, device=v.device)
        store[:, : w.cols].copy_(v)
        m = q.QuantizedMatrix(values=store[:, : w.cols], bits=w.bits, group_scales=w.group_scales,
                              group_layout=[(0, r1 - r0)], row_scale_vec=w.row_scales()[r0:r1].contiguous())
        return m

    def slice_cols(self, w, c0, c1):
        q = self.quant
        ld = q.round_up(max(c1 - c0, 1), 32)
        store = torch.zeros((w.rows, ld), dtype=torch.int8, device=w.values.device)
        store[:, : c1 - c0].copy_(w.values[:, c0:c1])
        return q.QuantizedMatrix(values=store[:, : c1 - c0], bits=w.bits, group_scales=w.group_scales,
                                 group_layout=w.group_layout, row_scale_vec=w.row_scales())

    def stack_rows(self, ws):
        from .transformer import concat_quantized

        return concat_quantized(ws)

    # --- compute ---
    def quantize_tokenwise(self, x):
        qa = self.quant.quantize_activation_tokenwise(x, 8, check_finite=False, flag=self.flag)
        return qa, qa.token_scales

    def linear(self, xq, xs, w, bias):
        return self.igemm.fused_linear(xq, w, bias)

    def attention(self, qkv, dl, heads, causal, batch):
        from .transformer import attention

        return attention(qkv[:, :dl], qkv[:, dl: 2 * dl], qkv[:, 2 * dl:], heads, causal, batch)

    def row_absmax(self, x):
        t, d = x.shape
        out = self._buf(("amax", t, d), lambda: torch.empty(t, dtype=torch.float32, device=x.device))
        self.N.call("zq_row_absmax", x.data_ptr(), t, d, x.stride(0), out.data_ptr(), self.flag.ptr,
                    self.N.stream_ptr())
        return out

    def quantize_with_absmax(self, x, amax):
        t, d = x.shape
        q = self._buf(("q", t, d), lambda: self.quant.padded_int8(t, d))
        s = self._buf(("s", t, d), lambda: torch.empty(t, dtype=torch.float32, device=x.device))
        self.N.call("zq_quantize_with_absmax", x.data_ptr(), t, d, x.stride(0), amax.data_ptr(), 8,
                    q.data_ptr(), q.stride(0), s.data_ptr(), self.N.stream_ptr())
        return self.quant.QuantizedActivation(values=q, bits=8, token_scales=s), s

    def igemm_s32(self, xq, w):
        t = xq.values.shape[0]
        acc = self._buf(("acc", t, w.rows), lambda: torch.empty((t, w.rows), dtype=torch.int32,
                                                                device=xq.values.device))
        if t <= 64 and w.bits == 8:  # decode: the stream-K kernel, one reused zeroed workspace
            nb = int(self.N.load().zq_linear_ws_bytes(t, w.rows))
            ws = self._buf(("skws", t, w.rows), lambda: torch.zeros(nb // 4 + 4, dtype=torch.int32,
                                                                    device=xq.values.device))
            a = xq.gemm_operand()
            wp, ldw, wb = w.weight_operand()
            self.N.call("zq_igemm_s32_ws", a.data_ptr(), a.stride(0), wp, ldw, wb, t, w.rows, a.shape[1],
                        acc.data_ptr(), acc.stride(0), ws.data_ptr(), 4 * ws.numel(), self.N.stream_ptr())
            return acc
        return self.igemm.igemm(xq, w, out=acc).acc

    def epilogue(self, acc, scales, w, bias, out=None):
        return self.igemm.dequant_epilogue(self.igemm.IntAccumulator(acc), scales, w, bias, out=out)

    def ln_quant(self, x, res, gamma, beta):
        y = torch.empty_like(x)
        qa = self.igemm.layer_norm_quantize(x, gamma, beta, 8, LN_EPS, residual=res, ln_out=y,
                                            check_finite=False, flag=self.flag)
        return y, qa, qa.token_scales

    def gelu(self, u):
        z = torch.empty_like(u)
        self.igemm.gelu_quantize(u, 8, gelu_out=z, check_finite=False, flag=self.flag)
        return z


def init_from_env(backend: str = "nccl"):
    """torch.distributed init from torchrun env (MASTER_ADDR=127.0.0.1 etc.)."""
    if not dist.is_initialized():
        dist.init_process_group(backend)
    return dist.get_rank(), dist.get_world_size()


__all__ = ["ShardedBlock", "shard_block", "row_parallel_linear", "tp_block_forward", "CudaOps", "init_from_env"]

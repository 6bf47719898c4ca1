"""CPU: tensor-parallel block forward (paper_2206_01861_b200/tp.py) with
world_size 2 over gloo.  The product module's sharding + collective sequencing
runs with the oracle injected as its compute ops; the result must equal the
single-process reference block (transformer.py:443-486) bit for bit, since the
row-parallel path all-reduces exact int32 partials and the global token max."""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lowbit_oracle as O

F32 = np.float32


class OW:
    """Oracle weight: int8 payload + per-row scales."""

    def __init__(self, values, rs):
        self.values = np.ascontiguousarray(values)
        self.rs = np.ascontiguousarray(rs, dtype=F32)


class OracleOps:
    rows = staticmethod(lambda w: w.values.shape[0])
    cols = staticmethod(lambda t: t.shape[1])
    cat = staticmethod(lambda ts: np.concatenate(ts).astype(F32))

    def slice_rows(self, w, r0, r1):
        return OW(w.values[r0:r1], w.rs[r0:r1])

    def slice_cols(self, w, c0, c1):
        return OW(w.values[:, c0:c1], w.rs)

    def stack_rows(self, ws):
        return OW(np.concatenate([w.values for w in ws]), np.concatenate([w.rs for w in ws]))

    def quantize_tokenwise(self, x):
        return O.quantize_activation_tokenwise(x, 8)

    def linear(self, xq, xs, w, bias):
        return O.dequant_epilogue(O.igemm(xq, w.values), xs, w.rs, bias)

    def attention(self, qkv, dl, heads, causal, batch):
        return O.attention(qkv[:, :dl], qkv[:, dl:2 * dl], qkv[:, 2 * dl:], heads, causal)

    def row_absmax(self, x):
        return torch.from_numpy(np.abs(x).max(axis=1).astype(F32))

    def quantize_with_absmax(self, x, amax):
        s = O.rowwise_scales(amax.numpy().astype(np.float64), 8)
        return O.quantize_rows(np.asarray(x, np.float64), s, 8), s

    def igemm_s32(self, xq, w):
        return torch.from_numpy(O.igemm(xq, w.values))

    def epilogue(self, acc, scales, w, bias, out=None):
        return O.dequant_epilogue(acc.numpy(), scales, w.rs, bias)

    def ln_quant(self, x, res, g, b):
        y = O.layer_norm_numpy((x + res).astype(F32) if res is not None else x, g, b)
        q, s = O.quantize_activation_tokenwise(y, 8)
        return y, q, s

    def gelu(self, u):
        return O.gelu(u)


def make_block(seed, d=64, heads=4, f=256):
    rng = O.Rng(seed)
    w = {"w_q": rng.gaussian((d, d), 0.02), "w_k": rng.gaussian((d, d), 0.02),
         "w_v": rng.gaussian((d, d), 0.02), "w_o": rng.gaussian((d, d), 0.02) * 3,
         "w_h4h": rng.gaussian((f, d), 0.02), "w_4hh": rng.gaussian((d, f), 0.02)}
    for n, s in (("b_q", d), ("b_k", d), ("b_v", d), ("b_o", d), ("b_h4h", f), ("b_4hh", d)):
        w[n] = (0.01 * rng.gaussian((s,), 1.0)).astype(F32)
    w["ln1_gamma"] = (1 + 0.1 * rng.gaussian((d,), 1.0)).astype(F32)
    w["ln1_beta"] = (0.1 * rng.gaussian((d,), 1.0)).astype(F32)
    w["ln2_gamma"] = (1 + 0.1 * rng.gaussian((d,), 1.0)).astype(F32)
    w["ln2_beta"] = (0.1 * rng.gaussian((d,), 1.0)).astype(F32)
    qb = O.quantize_block(w, 8, 8, O.default_group_count(d))
    view = SimpleNamespace(num_heads=heads, **{k: v for k, v in qb.items() if not k.startswith("w_")})
    for n in ("w_q", "w_k", "w_v", "w_o", "w_h4h", "w_4hh"):
        setattr(view, n, OW(qb[n][0], qb[n][1]))
    return qb, view


def _worker(rank, world, port, causal, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2206_01861_b200 import tp

        qb, view = make_block(7)
        x = O.Rng(3).gaussian((24, 64), 0.5)
        ops = OracleOps()
        sb = tp.shard_block(view, ops, rank, world)
        y = tp.tp_block_forward(x, sb, ops, causal)
        ref = O.block_forward(x, qb, 4, causal, "int8")
        out[rank] = bool(np.array_equal(np.asarray(y).view(np.uint32), ref.view(np.uint32)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("causal", [False, True])
def test_tp_block_bit_exact_over_gloo(world, causal):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), causal, out), nprocs=world, join=True)
    assert all(out.get(r, False) for r in range(world)), dict(out)


def test_shard_rejects_indivisible():
    from paper_2206_01861_b200 import tp
    from paper_2206_01861_b200.errors import UsageError

    _, view = make_block(1, d=64, heads=4, f=256)
    with pytest.raises(UsageError):
        tp.shard_block(view, OracleOps(), 0, 3)

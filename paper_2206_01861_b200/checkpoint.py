"""ZQCK model checkpoints -> HBM (reference
pkg/src/lowbit/checkpoint.py:1-189).

The byte format is the reference's (little-endian; checkpoint.py:1-21):

    magic "ZQCK" | version u32 | vocab u32 | dim u32 | heads u32 | layers u32 | causal u8
    embedding f32[vocab*dim] | final_gamma f32[dim] | final_beta f32[dim]
    per block: kind u8 (0 float, 1 quantized), six weight sections (q,k,v,o,h4h,4hh):
        float:     f32 values, row-major
        quantized: bits u8 | num_groups u32 | (start u32, count u32) per group |
                   scales f32 | values i8 row-major
    then twelve f32 arrays: six biases, ln1_gamma, ln1_beta, ln2_gamma, ln2_beta

`read_checkpoint` parses it on the host with the reference's error behaviour
(bad magic / version, truncation and trailing bytes raise UsageError);
`to_device` uploads a model into the B200 layout: int8 payloads into 32-byte
padded rows, per-row scales expanded once on device, INT4 FFN payloads packed
for the W4A8 kernel, q/k/v fused, float blocks quantized on device with the
given precision.  `write_checkpoint` writes the same bytes back (bit-exact
round trip).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import quant
from .errors import UsageError
from .transformer import BIAS_NAMES, WEIGHT_NAMES, DeviceBlock, PrecisionConfig, quantize_block

MAGIC = b"ZQCK"
VERSION = 1
LN_NAMES = ("ln1_gamma", "ln1_beta", "ln2_gamma", "ln2_beta")


def _weight_shapes(dim: int):
    """checkpoint.py:44-45"""
    return [(dim, dim)] * 4 + [(4 * dim, dim), (dim, 4 * dim)]


def _bias_shapes(dim: int):
    """checkpoint.py:48-49"""
    return [dim] * 4 + [4 * dim, dim] + [dim] * 4


@dataclass
class HostQuantMatrix:
    """A quantized section as stored (QuantizedMatrix fields, quant.py:134-181)."""

    values: np.ndarray  # int8 [rows, cols], one value per byte (INT4 too)
    bits: int
    group_scales: np.ndarray  # f32 [g]
    group_layout: list


@dataclass
class HostModel:
    """ToyModel (transformer.py:220-258) as read from a checkpoint."""

    vocab: int
    dim: int
    num_heads: int
    causal: bool
    embedding: np.ndarray
    final_gamma: np.ndarray
    final_beta: np.ndarray
    blocks: list = field(default_factory=list)  # dicts: name -> ndarray | HostQuantMatrix, plus "quantized"

    @property
    def num_layers(self) -> int:
        return len(self.blocks)


class _Reader:
    """checkpoint.py:73-103"""

    def __init__(self, data: bytes):
        self.data, self.pos = data, 0

    def take(self, n: int) -> bytes:
        if self.pos + n > len(self.data):
            raise UsageError("checkpoint truncated")
        out = self.data[self.pos:self.pos + n]
        self.pos += n
        return out

    def u8(self) -> int:
        return struct.unpack("<B", self.take(1))[0]

    def u32(self) -> int:
        return struct.unpack("<I", self.take(4))[0]

    def f32(self, shape) -> np.ndarray:
        n = int(np.prod(shape))
        return np.frombuffer(self.take(4 * n), dtype="<f4").astype(np.float32).reshape(shape)

    def i8(self, shape) -> np.ndarray:
        n = int(np.prod(shape))
        return np.frombuffer(self.take(n), dtype=np.int8).reshape(shape).copy()


def read_checkpoint(path: str) -> HostModel:
    """load_model (checkpoint.py:142-189) into host arrays."""
    with open(path, "rb") as f:
        r = _Reader(f.read())
    if r.take(4) != MAGIC:
        raise UsageError(f"{path}: not a model checkpoint (bad magic)")
    version = r.u32()
    if version != VERSION:
        raise UsageError(f"{path}: unsupported checkpoint version {version}")
    vocab, dim, heads, layers = r.u32(), r.u32(), r.u32(), r.u32()
    causal = bool(r.u8())
    model = HostModel(vocab=vocab, dim=dim, num_heads=heads, causal=causal,
                      embedding=r.f32((vocab, dim)), final_gamma=r.f32((dim,)), final_beta=r.f32((dim,)))
    for _ in range(layers):
        quantized = bool(r.u8())
        blk = {"quantized": quantized}
        for name, shape in zip(WEIGHT_NAMES, _weight_shapes(dim)):
            if quantized:  # checkpoint.py:117-123
                bits = r.u8()
                g = r.u32()
                layout = [(r.u32(), r.u32()) for _ in range(g)]
                scales = r.f32((g,))
                blk[name] = HostQuantMatrix(values=r.i8(shape), bits=bits, group_scales=scales,
                                            group_layout=layout)
            else:
                blk[name] = r.f32(shape)
        for name, n in zip(BIAS_NAMES + LN_NAMES, _bias_shapes(dim)):
            blk[name] = r.f32((n,))
        model.blocks.append(blk)
    if r.pos != len(r.data):
        raise UsageError(f"checkpoint has {len(r.data) - r.pos} trailing bytes")
    return model


def write_checkpoint(model: HostModel, path: str) -> None:
    """save_model (checkpoint.py:118-139)."""
    parts = [MAGIC, struct.pack("<IIIIIB", VERSION, model.vocab, model.dim, model.num_heads,
                                model.num_layers, 1 if model.causal else 0)]
    f32 = lambda a: np.ascontiguousarray(a, dtype="<f4").tobytes()  # noqa: E731
    parts += [f32(model.embedding), f32(model.final_gamma), f32(model.final_beta)]
    for blk in model.blocks:
        parts.append(struct.pack("<B", 1 if blk["quantized"] else 0))
        for name in WEIGHT_NAMES:
            m = blk[name]
            if blk["quantized"]:
                parts.append(struct.pack("<BI", m.bits, len(m.group_layout)))
                parts += [struct.pack("<II", s, c) for s, c in m.group_layout]
                parts += [f32(m.group_scales), np.ascontiguousarray(m.values, dtype=np.int8).tobytes()]
            else:
                parts.append(f32(m))
        parts += [f32(blk[name]) for name in BIAS_NAMES + LN_NAMES]
    with open(path, "wb") as f:
        f.write(b"".join(parts))


@dataclass
class DeviceModel:
    """A checkpoint resident in HBM: DeviceBlocks (fused QKV, per-row scales,
    packed INT4) plus the float embedding / final LN (transformer.py:220-258)."""

    blocks: list
    embedding: torch.Tensor
    final_gamma: torch.Tensor
    final_beta: torch.Tensor
    num_heads: int
    causal: bool


def _device_matrix(m: HostQuantMatrix) -> quant.QuantizedMatrix:
    quant._check_bits(m.bits)
    rows, cols = m.values.shape
    store = torch.zeros((rows, quant.round_up(max(cols, 1), 32)), dtype=torch.int8, device="cuda")
    store[:, :cols].copy_(torch.from_numpy(m.values))
    qm = quant.QuantizedMatrix(values=store[:, :cols], bits=m.bits,
                               group_scales=torch.from_numpy(np.asarray(m.group_scales, np.float32)).cuda(),
                               group_layout=[tuple(p) for p in m.group_layout])
    qm.row_scales()  # expanded once on device (the reference rebuilds it per epilogue, quant.py:165-170)
    if qm.bits == 4:
        qm.packed4 = quant.pack_int4(qm.values)
    return qm


def to_device(model: HostModel, precision: PrecisionConfig | None = None) -> DeviceModel:
    """Upload a checkpoint.  Quantized blocks keep their stored payloads
    bit-for-bit; float blocks are quantized on device with `precision`
    (quantize_block, transformer.py:333-361), which is then required."""
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
    blocks = []
    for blk in model.blocks:
        if blk["quantized"]:
            kw = {n: _device_matrix(blk[n]) for n in WEIGHT_NAMES}
            kw.update({n: dev(blk[n]) for n in BIAS_NAMES + LN_NAMES})
            blocks.append(DeviceBlock(**kw, num_heads=model.num_heads))
        else:
            if precision is None:
                raise UsageError("float checkpoint blocks need a PrecisionConfig to be quantized on device")
            blocks.append(quantize_block(dict(blk, num_heads=model.num_heads), precision))
    return DeviceModel(blocks=blocks, embedding=dev(model.embedding), final_gamma=dev(model.final_gamma),
                       final_beta=dev(model.final_beta), num_heads=model.num_heads, causal=model.causal)


def load_model(path: str, precision: PrecisionConfig | None = None) -> DeviceModel:
    """checkpoint.load_model (checkpoint.py:142) straight into HBM."""
    return to_device(read_checkpoint(path), precision)


__all__ = ["HostModel", "HostQuantMatrix", "DeviceModel", "read_checkpoint", "write_checkpoint", "to_device",
           "load_model"]

"""GPT-style caller of the hot path: prefill + greedy decode with a key/value
cache, optionally Megatron tensor-parallel (BASELINE
configs 3-5).

Each layer is the reference's post-LN ZeroQuant block (transformer.py:443-486)
with causal attention; the quantized pieces are exactly the ones the encoder
uses (fused W8A8 / W4A8 tcgen05 linears, LN+quant, GeLU+quant).  What is new
on the caller side:

* a float32 key/value cache per layer, [batch, max_ctx, d_local]: the reference
  recomputes the whole context for every generated token (evaluate.py:96-98);
  with causal attention and token-wise activation scales the cached k/v rows are
  the rows recomputation would produce, so the cache changes no value;
* decode attention for one query row per sequence (zq_decode_attention_f32)
  with the context length in device memory, so one decode step is a fixed
  launch sequence captured once in a CUDA graph;
* the tied LM head (transformer.py:532) and greedy argmax: float32-accurate
  logits on tcgen05 (zq_lm_head_argmax_split: the embedding split once into f16
  hi / lo terms, the final hidden state split per step, three-term products,
  fused argmax) for batch <= 16; torch matmul + argmax above that (the head is
  not on the quantized path);
* tensor parallelism (tp.py): column-parallel q/k/v/h4h, row-parallel o/4hh
  through `tp.row_parallel_linear` (the exact MAX(absmax) + int32 SUM
  all-reduces), so every rank's result is bit-identical to the single-GPU one.
  `force_tp=True` takes that route even on one rank (exercises the collectives
  inside CUDA-graph capture on a 1-GPU box).

Model shapes follow SURVEY.md §8(a): GPT-3 350M (W4/8-A8), GPT-J 6B and
GPT-NeoX 20B (W8A8); weights are random-init Gaussian(0, 0.02) generated on
device (no checkpoints are available offline).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import quant
from .errors import ShapeError, UsageError
from .transformer import INIT_STD, LN_EPS, attention, random_block


@dataclass(frozen=True)
class GPTConfig:
    name: str
    layers: int
    dim: int
    heads: int
    ffn: int
    vocab: int
    mhsa_bits: int
    ffc_bits: int
    groups: int

    @property
    def head_dim(self) -> int:
        return self.dim // self.heads


# SURVEY.md §8(a) C3-C5; group counts from default_group_count (transformer.py:129-137)
CONFIGS = {
    "gpt3-350m": GPTConfig("GPT-3 350M W4/8-A8", 24, 1024, 16, 4096, 50257, 8, 4, 64),
    "gptj-6b": GPTConfig("GPT-J 6B W8A8", 28, 4096, 16, 16384, 50400, 8, 8, 128),
    "neox-20b": GPTConfig("GPT-NeoX 20B W8A8", 44, 6144, 64, 24576, 50432, 8, 8, 128),
}


class DecoderEngine:
    """Greedy generation for `batch` sequences.

    prefill(ids [batch, T]) runs the prompt (causal), fills the caches and picks
    the first new token; step() generates one more token per sequence.  With
    `tp=(group, rank, world)` every layer is sharded Megatron-style."""

    def __init__(self, cfg: GPTConfig, batch: int, max_ctx: int, seed: int = 0, tp=None,
                 layers: int | None = None, use_graph: bool = True, blocks=None, embedding=None,
                 force_tp: bool = False):
        from .tp import CudaOps, ShardedBlock, shard_block

        self.cfg = cfg
        self.batch = batch
        self.max_ctx = max_ctx
        self.use_graph = use_graph
        self.group, self.rank, self.world = tp if tp is not None else (None, 0, 1)
        self._tp = self.world > 1 or force_tp
        nl = cfg.layers if layers is None else layers
        if cfg.heads % self.world or cfg.ffn % self.world:
            raise UsageError(f"{cfg.name}: heads/ffn not divisible by TP degree {self.world}")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dl = cfg.dim // self.world               # local attention width
        self.hl = cfg.heads // self.world
        self.fl = cfg.ffn // self.world
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self._ops = CudaOps(flag=self.flag, reuse=True)
        # blocks given by the caller (e.g. checkpoint.load_model) are globally
        # quantized like generated ones: shard them the same way
        self.blocks = []
        src = list(blocks) if blocks is not None else [None] * nl
        for i, blk in enumerate(src):
            if blk is None:
                blk = random_block(cfg.dim, cfg.heads, cfg.mhsa_bits, cfg.ffc_bits, cfg.groups,
                                   seed=seed * 1000 + i, ffn_mult=cfg.ffn // cfg.dim)
            if self.world > 1 and not isinstance(blk, ShardedBlock):
                blk = shard_block(blk, self._ops, self.rank, self.world)
            self.blocks.append(blk)
        nl = len(self.blocks)
        if embedding is not None:
            self.embedding = quant.as_device_f32(embedding).contiguous()
        else:
            gen = torch.Generator(device=dev).manual_seed(seed * 1000 + 999)
            self.embedding = torch.randn((cfg.vocab, cfg.dim), generator=gen, device=dev) * INIT_STD
        self.final_gamma = torch.ones(cfg.dim, device=dev)
        self.final_beta = torch.zeros(cfg.dim, device=dev)
        e = lambda *s: torch.empty(s, dtype=torch.float32, device=dev)  # noqa: E731
        self.kcache = [e(batch, max_ctx, self.dl) for _ in range(nl)]
        self.vcache = [e(batch, max_ctx, self.dl) for _ in range(nl)]
        self.pos = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.lens = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.host_pos = None  # host mirror of pos (all sequences advance together)
        self.next_ids = torch.zeros(batch, dtype=torch.int64, device=dev)
        # LM head (zq_lm_head_argmax): one power-of-two scale for the embedding,
        # chosen once, and the per-step f16 split / argmax workspaces
        m = float(self.embedding.abs().max())
        self.emb_scale = math.ldexp(1.0, 15 - math.frexp(m)[1]) if m > 0 else 1.0
        self._lm_ok = batch <= 16 and cfg.dim % 64 == 0 and os.environ.get("ZQ_LM_TORCH", "0") != "1"
        # the embedding's f16 hi / lo terms, split once: each step streams them by TMA
        # straight into the tensor core (ZQ_LM_SPLIT=0: convert the f32 rows per step)
        self._emb_split = None
        if self._lm_ok and os.environ.get("ZQ_LM_SPLIT", "1") != "0":
            eh = torch.empty((cfg.vocab, cfg.dim), dtype=torch.float16, device=dev)
            el = torch.empty_like(eh)
            N.call("zq_lm_embed_split", self.embedding.data_ptr(), cfg.vocab, cfg.dim, self.emb_scale,
                   eh.data_ptr(), el.data_ptr(), N.stream_ptr())
            self._emb_split = (eh, el)
        self._lm_ws = dict(xh=torch.zeros(16 * cfg.dim, dtype=torch.float16, device=dev),
                           xl=torch.zeros(16 * cfg.dim, dtype=torch.float16, device=dev),
                           xinv=torch.zeros(16, dtype=torch.float32, device=dev),
                           keys=torch.zeros(16, dtype=torch.int64, device=dev))
        # decode-attention context chunking planned for the UNSHARDED head count:
        # the float merge order then does not depend on the TP degree
        self._dec_chunks = int(N.load().zq_decode_attention_chunks(batch, cfg.heads, max_ctx))
        # stream-K decode GEMMs (zq_linear_ws): one zero-initialised int32 workspace
        # shared by every decode-step linear (each launch leaves it zeroed)
        lib = N.load()
        wsb = max(int(lib.zq_linear_ws_bytes(batch, n)) for n in (3 * self.dl, cfg.dim, self.fl))
        self._sk_ws = torch.zeros(wsb // 4 + 4, dtype=torch.int32, device=dev)
        self._bufs: dict[int, dict] = {}
        self._graph = None
        self.scale = float(np.float32(1.0 / math.sqrt(cfg.head_dim)))

    # ------------------------------------------------------------------
    def _buffers(self, t: int) -> dict:
        """Activation buffers for t token rows (cached per row count)."""
        if t not in self._bufs:
            dev = self.embedding.device
            d, dl, fl = self.cfg.dim, self.dl, self.fl
            e = lambda *s: torch.empty(s, dtype=torch.float32, device=dev)  # noqa: E731
            self._bufs[t] = dict(
                ids=torch.zeros(t, dtype=torch.int64, device=dev),
                x=e(t, d), h=e(t, d), qkv=e(t, 3 * dl), ctx=e(t, dl), attn=e(t, d), u=e(t, fl),
                z=e(t, fl), f=e(t, d), out=e(t, d),
                xq=quant.padded_int8(t, d), cq=quant.padded_int8(t, dl), hq=quant.padded_int8(t, d),
                zq=quant.padded_int8(t, fl), sx=e(t), sc=e(t), sh=e(t), sz=e(t),
                last=e(self.batch, d), lq=quant.padded_int8(self.batch, d), ls=e(self.batch),
                logits=e(self.batch, self.cfg.vocab),
            )
        return self._bufs[t]

    # -- raw launches -------------------------------------------------------
    def _linear(self, q, s, w, bias, out, bias_on=True):
        t, k = q.shape
        wp, ldw, wb = w.weight_operand()
        N.call("zq_linear_ws", q.data_ptr(), q.stride(0), s.data_ptr(), 0.0, wp, ldw, wb,
               w.row_scales().data_ptr(), N.ptr(bias) if bias_on else None, t, w.rows, k,
               out.data_ptr(), out.stride(0), N.OUT_F32, self._sk_ws.data_ptr(), 4 * self._sk_ws.numel(),
               N.stream_ptr())

    def _qkv_kv(self, xq, sx, blk, qkv, li: int, t: int) -> bool:
        """Decode step: QKV linear with the KV-cache append in its epilogue
        (zq_linear_kv); False when unsupported (the caller appends separately)."""
        w = blk.w_qkv
        wp, ldw, wb = w.weight_operand()
        rc = N.call_rc("zq_linear_kv_ws", xq.data_ptr(), xq.stride(0), sx.data_ptr(), wp, ldw, wb,
                       w.row_scales().data_ptr(), blk.b_qkv.data_ptr(), t, w.rows, xq.shape[1], qkv.data_ptr(),
                       qkv.stride(0), self.kcache[li].data_ptr(), self.vcache[li].data_ptr(), self.pos.data_ptr(),
                       self.dl, self.max_ctx, self._sk_ws.data_ptr(), 4 * self._sk_ws.numel(), N.stream_ptr())
        return rc != N.ZQ_ERR_UNSUPPORTED

    def _qkv_kv_prefill(self, xq, sx, blk, qkv, li: int, t: int, rows_per_seq: int) -> bool:
        """Prefill QKV linear with the KV-cache append in the CTA-pair GEMM epilogue
        (prefill starts from an empty cache: pos = 0); False when unsupported."""
        if os.environ.get("ZQ_KV_PREFILL", "1") == "0":
            return False
        w = blk.w_qkv
        wp, ldw, wb = w.weight_operand()
        rc = N.call_rc("zq_linear_kv_prefill", xq.data_ptr(), xq.stride(0), sx.data_ptr(), wp, ldw, wb,
                       w.row_scales().data_ptr(), blk.b_qkv.data_ptr(), t, w.rows, xq.shape[1], qkv.data_ptr(),
                       qkv.stride(0), self.kcache[li].data_ptr(), self.vcache[li].data_ptr(), self.dl,
                       self.max_ctx, rows_per_seq, N.stream_ptr())
        return rc != N.ZQ_ERR_UNSUPPORTED

    def _tok_quant(self, x, q, s):
        t, d = x.shape
        N.call("zq_quantize_tokenwise", x.data_ptr(), t, d, x.stride(0), 8, q.data_ptr(), q.stride(0),
               s.data_ptr(), self.flag.data_ptr(), N.stream_ptr())

    def _ln_quant(self, x, res, g, b, ln_out, q, s):
        t, d = x.shape
        N.call("zq_layer_norm_quantize", x.data_ptr(), N.ptr(res), g.data_ptr(), b.data_ptr(), t, d,
               float(np.float32(LN_EPS)), 8, ln_out.data_ptr(), q.data_ptr(), q.stride(0), s.data_ptr(),
               self.flag.data_ptr(), N.stream_ptr())

    def _row_parallel(self, x, B, w, bias, out, xq, xs):
        """o / 4hh projection: local fused linear (one rank), or Megatron
        row-parallel through tp.row_parallel_linear (the exact MAX(absmax) +
        int32 SUM all-reduces, tp.py steps 1-5)."""
        if not self._tp:
            self._tok_quant(x, xq, xs)
            self._linear(xq, xs, w, bias, out)
            return
        from .tp import row_parallel_linear

        row_parallel_linear(self._ops, x, w, bias, self.group, out=out)

    def _layers(self, B, t: int, rows_per_seq: int, prefill: bool):
        """All blocks over B['x'] (t = batch * rows_per_seq rows); y -> B['x']."""
        dl = self.dl
        x, xq, sx = B["x"], B["xq"], B["sx"]
        for li, blk in enumerate(self.blocks):
            qkv = B["qkv"]
            if prefill:
                if not self._qkv_kv_prefill(xq, sx, blk, qkv, li, t, rows_per_seq):
                    self._linear(xq, sx, blk.w_qkv, blk.b_qkv, qkv)
                    N.call("zq_kv_append", qkv.data_ptr(), qkv.stride(0), self.batch, rows_per_seq, dl,
                           self.pos.data_ptr(), self.kcache[li].data_ptr(), self.vcache[li].data_ptr(),
                           self.max_ctx, N.stream_ptr())
            elif not self._qkv_kv(xq, sx, blk, qkv, li, t):
                self._linear(xq, sx, blk.w_qkv, blk.b_qkv, qkv)
                N.call("zq_kv_append", qkv.data_ptr(), qkv.stride(0), self.batch, rows_per_seq, dl,
                       self.pos.data_ptr(), self.kcache[li].data_ptr(), self.vcache[li].data_ptr(),
                       self.max_ctx, N.stream_ptr())
            if prefill:
                attention(qkv[:, :dl], qkv[:, dl:2 * dl], qkv[:, 2 * dl:], self.hl, True, self.batch,
                          out=B["ctx"])
            else:
                N.call("zq_decode_attention_f32", qkv.data_ptr(), qkv.stride(0), self.kcache[li].data_ptr(),
                       self.vcache[li].data_ptr(), self.max_ctx, self.batch, self.hl, self.cfg.head_dim,
                       self.lens.data_ptr(), self.scale, B["ctx"].data_ptr(), B["ctx"].stride(0),
                       self._dec_chunks, N.stream_ptr())
            ln1 = blk.ln1 if hasattr(blk, "ln1") else (blk.ln1_gamma, blk.ln1_beta)
            ln2 = blk.ln2 if hasattr(blk, "ln2") else (blk.ln2_gamma, blk.ln2_beta)
            self._row_parallel(B["ctx"], B, blk.w_o, blk.b_o, B["attn"], B["cq"], B["sc"])
            self._ln_quant(x, B["attn"], ln1[0], ln1[1], B["h"], B["hq"], B["sh"])
            self._linear(B["hq"], B["sh"], blk.w_h4h, blk.b_h4h, B["u"])
            if not self._tp:
                u = B["u"]
                N.call("zq_gelu_quantize", u.data_ptr(), t, self.fl, self.fl, 8, None, B["zq"].data_ptr(),
                       B["zq"].stride(0), B["sz"].data_ptr(), self.flag.data_ptr(), N.stream_ptr())
                self._linear(B["zq"], B["sz"], blk.w_4hh, blk.b_4hh, B["f"])
            else:
                u = B["u"]
                N.call("zq_gelu_quantize", u.data_ptr(), t, self.fl, self.fl, 8, B["z"].data_ptr(),
                       B["zq"].data_ptr(), B["zq"].stride(0), B["sz"].data_ptr(), self.flag.data_ptr(),
                       N.stream_ptr())
                self._row_parallel(B["z"], B, blk.w_4hh, blk.b_4hh, B["f"], B["zq"], B["sz"])
            self._ln_quant(B["h"], B["f"], ln2[0], ln2[1], x, xq, sx)

    def _head(self, B, t: int, rows_per_seq: int):
        """Final LN of each sequence's last row, tied LM head, greedy argmax."""
        last = B["x"].view(self.batch, rows_per_seq, -1)[:, -1, :]
        B["last"].copy_(last)
        self._ln_quant(B["last"], None, self.final_gamma, self.final_beta, B["out"][: self.batch],
                       B["lq"], B["ls"])
        out = B["out"][: self.batch]
        if self._lm_ok and self._emb_split is not None:  # pre-split embedding, TMA-fed tcgen05 + argmax
            W = self._lm_ws
            eh, el = self._emb_split
            N.call("zq_lm_head_argmax_split", out.data_ptr(), out.stride(0), self.batch, eh.data_ptr(),
                   el.data_ptr(), self.cfg.vocab, self.cfg.dim, self.emb_scale, W["xh"].data_ptr(),
                   W["xl"].data_ptr(), W["xinv"].data_ptr(), W["keys"].data_ptr(), self.next_ids.data_ptr(),
                   N.stream_ptr())
        elif self._lm_ok:  # tcgen05 two-term f16 LM head with a fused argmax
            W = self._lm_ws
            N.call("zq_lm_head_argmax", out.data_ptr(), out.stride(0), self.batch, self.embedding.data_ptr(),
                   self.cfg.vocab, self.cfg.dim, self.emb_scale, W["xh"].data_ptr(), W["xl"].data_ptr(),
                   W["xinv"].data_ptr(), W["keys"].data_ptr(), self.next_ids.data_ptr(), N.stream_ptr())
        else:  # batch > 16 (or ZQ_LM_TORCH=1): float32 matmul + argmax
            torch.matmul(out, self.embedding.t(), out=B["logits"])
            torch.argmax(B["logits"], dim=1, out=self.next_ids)

    def _embed(self, B, ids):
        torch.index_select(self.embedding, 0, ids, out=B["x"])
        self._tok_quant(B["x"], B["xq"], B["sx"])

    # ------------------------------------------------------------------
    def prefill(self, ids) -> torch.Tensor:
        """ids [batch, T] (host or device) -> first generated token per sequence."""
        ids = ids if isinstance(ids, torch.Tensor) else torch.as_tensor(np.asarray(ids))
        if ids.dim() != 2 or ids.shape[0] != self.batch:
            raise ShapeError(f"expected token ids [{self.batch}, T], got {tuple(ids.shape)}")
        T = ids.shape[1]
        if T + 1 > self.max_ctx:
            raise UsageError(f"prompt of {T} tokens does not fit max_ctx {self.max_ctx}")
        t = self.batch * T
        B = self._buffers(t)
        B["ids"].copy_(ids.reshape(-1), non_blocking=True)
        self.flag.zero_()
        self.pos.zero_()
        self._embed(B, B["ids"])
        self._layers(B, t, T, prefill=True)
        self._head(B, t, T)
        self.pos.fill_(T)
        self.host_pos = T
        return self.next_ids

    def _step_launches(self):
        B = self._buffers(self.batch)
        self._embed(B, self.next_ids)
        torch.add(self.pos, 1, out=self.lens)
        self._layers(B, self.batch, 1, prefill=False)
        self._head(B, self.batch, 1)
        self.pos.add_(1)

    def capture(self):
        """Capture one decode step into a CUDA graph.  The eager warm-up before
        the capture really runs a step (it advances pos, overwrites next_ids
        with the following token and writes K/V at pos); every piece of decode
        state it touches is restored afterwards, so the first replay computes
        exactly the step an eager call would have."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        saved = (self.pos.clone(), self.lens.clone(), self.next_ids.clone())

        def restore():
            self.pos.copy_(saved[0])
            self.lens.copy_(saved[1])
            self.next_ids.copy_(saved[2])

        with torch.cuda.stream(s):
            self._step_launches()
        torch.cuda.current_stream().wait_stream(s)
        restore()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._step_launches()
        restore()
        self._graph = g

    def step(self) -> torch.Tensor:
        """Generate one token per sequence (next_ids is updated in place).
        Raises UsageError before the key/value cache would overflow max_ctx."""
        if self.host_pos is None:
            raise UsageError("step() before prefill()")
        if self.host_pos >= self.max_ctx:
            raise UsageError(f"decode position {self.host_pos} is past max_ctx {self.max_ctx}")
        if self.use_graph:
            if self._graph is None:
                self.capture()
            self._graph.replay()
        else:
            self._step_launches()
        self.host_pos += 1
        return self.next_ids

    def generate(self, ids, new_tokens: int) -> torch.Tensor:
        T = (ids.shape if isinstance(ids, torch.Tensor) else np.asarray(ids).shape)[-1]
        if new_tokens < 1 or T + new_tokens - 1 > self.max_ctx:
            raise UsageError(f"{T} prompt + {new_tokens} new tokens do not fit max_ctx {self.max_ctx}")
        out = [self.prefill(ids).clone()]
        for _ in range(new_tokens - 1):
            out.append(self.step().clone())
        return torch.stack(out, dim=1)

    def check_finite(self):
        if int(self.flag.item()) != 0:
            raise ValueError("non-finite activations encountered")


__all__ = ["GPTConfig", "CONFIGS", "DecoderEngine"]

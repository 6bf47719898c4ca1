"""GPU: GPT prefill + cached decode (paper_2206_01861_b200.decoder) vs the
oracle recomputing the whole causal context with the reference block
(transformer.py:443-486, evaluate.py:96-98 recomputation).  Attention is float
on both sides, so hidden states are compared with the block tolerance; the
greedy tokens must agree."""

import math
import numpy as np
import pytest
import torch

from oracle import lowbit_oracle as O

pytestmark = pytest.mark.gpu
TOL = 2e-3


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def make_weights(rng, d, f):
    w = {n: rng.gaussian(s, std=0.02) for n, s in (
        ("w_q", (d, d)), ("w_k", (d, d)), ("w_v", (d, d)), ("w_o", (d, d)),
        ("w_h4h", (f, d)), ("w_4hh", (d, f)))}
    for n, s in (("b_q", d), ("b_k", d), ("b_v", d), ("b_o", d), ("b_h4h", f), ("b_4hh", d)):
        w[n] = rng.gaussian((s,), std=0.02)
    for n in ("ln1", "ln2"):
        w[f"{n}_gamma"] = (1.0 + rng.gaussian((d,), std=0.1)).astype(np.float32)
        w[f"{n}_beta"] = rng.gaussian((d,), std=0.1)
    return w


def oracle_hidden(ids_row, emb, qbs, heads, gamma, beta):
    x = emb[ids_row]
    for qb in qbs:
        x = O.block_forward(x, qb, heads, True, "int8")
    return O.layer_norm(x, gamma, beta)


@pytest.mark.parametrize("mbits,fbits", [(8, 8), (8, 4)])
def test_prefill_and_cached_decode_match_recompute(mbits, fbits):
    from paper_2206_01861_b200 import transformer as T
    from paper_2206_01861_b200.decoder import DecoderEngine, GPTConfig

    d, heads, f, V, L, g = 256, 4, 1024, 512, 2, 16
    cfg = GPTConfig("tiny", L, d, heads, f, V, mbits, fbits, g)
    rng = O.Rng(7)
    ws = [make_weights(rng, d, f) for _ in range(L)]
    emb = rng.gaussian((V, d), std=1.0)
    prec = T.PrecisionConfig.from_scheme("W8A8" if fbits == 8 else "W4/8A8", group_count=g)
    blocks = []
    for w in ws:
        w = dict(w, num_heads=heads)
        blocks.append(T.quantize_block(w, prec))
    qbs = [O.quantize_block(w, mbits, fbits, g) for w in ws]
    batch, Tp = 3, 9
    ids = np.random.default_rng(0).integers(0, V, (batch, Tp))
    eng = DecoderEngine(cfg, batch, max_ctx=32, blocks=blocks, embedding=emb)
    gamma, beta = eng.final_gamma.cpu().numpy(), eng.final_beta.cpu().numpy()
    first = eng.prefill(ids).cpu().numpy()
    h_prefill = eng._buffers(batch * Tp)["out"][:batch].cpu().numpy()
    toks = [first]
    hs = []
    for _ in range(3):
        toks.append(eng.step().cpu().numpy())
        hs.append(eng._buffers(batch)["out"][:batch].cpu().numpy())
    eng.check_finite()
    full = np.concatenate([ids, np.stack(toks, 1)], axis=1)
    for b in range(batch):
        ref = oracle_hidden(full[b, :Tp], emb, qbs, heads, gamma, beta)
        assert rel(h_prefill[b], ref[-1]) < TOL, (b, rel(h_prefill[b], ref[-1]))
        for s in range(3):
            ref = oracle_hidden(full[b, :Tp + 1 + s], emb, qbs, heads, gamma, beta)
            assert rel(hs[s][b], ref[-1]) < TOL, (b, s, rel(hs[s][b], ref[-1]))
            logits = ref[-1] @ emb.T
            assert int(np.argmax(logits)) == int(full[b, Tp + 1 + s]), (b, s)


def test_decode_attention_vs_torch():
    from paper_2206_01861_b200 import _native as N

    for dh, heads in ((64, 4), (96, 3), (256, 2), (32, 5), (128, 2)):
        batch, max_ctx = 3, 1041  # odd context: chunked over a cluster
        dl = dh * heads
        torch.manual_seed(dh)
        kc = torch.randn(batch, max_ctx, dl, device="cuda")
        vc = torch.randn(batch, max_ctx, dl, device="cuda")
        q = torch.randn(batch, 3 * dl, device="cuda")
        lens = torch.tensor([1, 517, 1041], dtype=torch.int32, device="cuda")
        for b in range(batch):  # cache rows past a sequence's length are never read (NaN poison)
            kc[b, int(lens[b]):] = float("nan")
            vc[b, int(lens[b]):] = float("nan")
        ctx = torch.empty(batch, dl, device="cuda")
        scale = 1.0 / dh ** 0.5
        N.call("zq_decode_attention_f32", q.data_ptr(), q.stride(0), kc.data_ptr(), vc.data_ptr(), max_ctx,
               batch, heads, dh, lens.data_ptr(), scale, ctx.data_ptr(), ctx.stride(0), 0, N.stream_ptr())
        for b in range(batch):
            n = int(lens[b])
            qh = q[b, :dl].double().view(heads, 1, dh)
            k = kc[b, :n].double().view(n, heads, dh).transpose(0, 1)
            v = vc[b, :n].double().view(n, heads, dh).transpose(0, 1)
            p = torch.softmax(qh @ k.transpose(1, 2) * scale, -1)
            ref = (p @ v).reshape(dl)
            assert torch.allclose(ctx[b].double(), ref, rtol=1e-5, atol=1e-5), (dh, b)


@pytest.mark.parametrize("split", [False, True])
def test_lm_head_argmax_vs_f64(split):
    """zq_lm_head_argmax (tcgen05 two-term f16 split, fused argmax) and the
    pre-split variant (zq_lm_embed_split + zq_lm_head_argmax_split) vs float64
    logits: same token wherever the top two logits are not a near-tie; exact ties
    resolve to the lowest index like numpy's argmax."""
    from paper_2206_01861_b200 import _native as N

    for ntok, vocab, dim in ((16, 3001, 256), (5, 50400, 1024), (1, 129, 64), (16, 50400, 4096)):
        torch.manual_seed(vocab)
        x = torch.randn(ntok, dim, device="cuda")
        emb = torch.randn(vocab, dim, device="cuda") * 0.02
        emb[vocab // 2] = emb[vocab - 1] = x[0] * 0.05  # an exact tie for token 0 (largest logit)
        m = float(emb.abs().max())
        scale = math.ldexp(1.0, 15 - math.frexp(m)[1])
        xh = torch.zeros(16 * dim, dtype=torch.float16, device="cuda")
        xl = torch.zeros_like(xh)
        xinv = torch.zeros(16, device="cuda")
        keys = torch.zeros(16, dtype=torch.int64, device="cuda")
        ids = torch.full((ntok,), -1, dtype=torch.int64, device="cuda")
        if split:
            eh = torch.empty(vocab, dim, dtype=torch.float16, device="cuda")
            el = torch.empty_like(eh)
            N.call("zq_lm_embed_split", emb.data_ptr(), vocab, dim, scale, eh.data_ptr(), el.data_ptr(),
                   N.stream_ptr())
            N.call("zq_lm_head_argmax_split", x.data_ptr(), x.stride(0), ntok, eh.data_ptr(), el.data_ptr(), vocab,
                   dim, scale, xh.data_ptr(), xl.data_ptr(), xinv.data_ptr(), keys.data_ptr(), ids.data_ptr(),
                   N.stream_ptr())
        else:
            N.call("zq_lm_head_argmax", x.data_ptr(), x.stride(0), ntok, emb.data_ptr(), vocab, dim, scale,
                   xh.data_ptr(), xl.data_ptr(), xinv.data_ptr(), keys.data_ptr(), ids.data_ptr(), N.stream_ptr())
        logits = x.double() @ emb.double().t()
        top2 = logits.topk(2, dim=1)
        ref = logits.argmax(dim=1)
        got = ids.cpu()
        assert int(got[0]) == vocab // 2, (int(got[0]), vocab // 2)  # tie -> lowest index
        for t in range(1, ntok):
            gap = float(top2.values[t, 0] - top2.values[t, 1])
            if gap > 1e-5 * abs(float(top2.values[t, 0])):
                assert int(got[t]) == int(ref[t]), (ntok, vocab, t)


def test_graph_replay_matches_eager_steps():
    """The CUDA-graph decode step (use_graph=True, captured on the first step)
    must produce exactly the eager token stream: the capture's warm-up step
    may not leak into decode state (next_ids / pos / lens)."""
    from paper_2206_01861_b200.decoder import DecoderEngine, GPTConfig

    from paper_2206_01861_b200 import transformer as T

    cfg = GPTConfig("tiny-graph", 2, 256, 4, 1024, 512, 8, 8, 16)
    ids = np.random.default_rng(5).integers(0, cfg.vocab, (4, 7))
    streams, hidden = [], []
    for use_graph in (False, True):
        # weights well above the init scale, so the blocks move the hidden state away
        # from LN(embedding[last token]) and greedy decoding does not just repeat it
        blocks = [T.random_block(256, 4, 8, 8, 16, seed=40 + i, std=0.25) for i in range(2)]
        eng = DecoderEngine(cfg, 4, 20, seed=9, use_graph=use_graph, blocks=blocks)
        toks = [eng.prefill(ids).cpu().numpy()]
        hs = []
        for _ in range(8):
            toks.append(eng.step().cpu().numpy())
            hs.append(eng._buffers(4)["out"][:4].cpu().numpy())
        streams.append(np.stack(toks, 1))
        hidden.append(np.stack(hs))
    assert len(np.unique(streams[0])) > 4, streams[0]  # decoding is not a repeat of one token
    assert np.array_equal(streams[0], streams[1]), (streams[0], streams[1])
    assert np.array_equal(hidden[0].view(np.uint32), hidden[1].view(np.uint32))


def test_decode_bounded_by_max_ctx():
    from paper_2206_01861_b200.decoder import DecoderEngine, GPTConfig
    from paper_2206_01861_b200.errors import UsageError

    cfg = GPTConfig("tiny-ctx", 1, 256, 4, 1024, 512, 8, 8, 16)
    ids = np.random.default_rng(1).integers(0, cfg.vocab, (2, 5))
    eng = DecoderEngine(cfg, 2, 7, seed=1, use_graph=True)
    with pytest.raises(UsageError):
        eng.step()  # before prefill
    eng.prefill(ids)
    eng.step()
    eng.step()  # K/V written at positions 5 and 6 = max_ctx - 1
    with pytest.raises(UsageError):
        eng.step()
    with pytest.raises(UsageError):
        eng.generate(ids, 4)  # 5 + 4 - 1 > 7
    assert eng.generate(ids, 3).shape == (2, 3)
    with pytest.raises(UsageError):
        DecoderEngine(cfg, 2, 5, seed=1).prefill(ids)  # T + 1 > max_ctx


def test_flag_cleared_by_prefill():
    from paper_2206_01861_b200.decoder import DecoderEngine, GPTConfig

    cfg = GPTConfig("tiny-flag", 1, 256, 4, 1024, 512, 8, 8, 16)
    eng = DecoderEngine(cfg, 2, 16, seed=1, use_graph=False)
    eng.flag.fill_(1)
    eng.prefill(np.zeros((2, 4), np.int64))
    eng.check_finite()


@pytest.mark.parametrize("shape", [(8, 1024, 1024, 1040), (16, 128, 4096, 256), (8, 256, 768, 300),
                                   (2, 256, 768, 300), (16, 100, 1024, 128)])
def test_linear_kv_prefill_matches_linear_then_append(shape):
    """zq_linear_kv_prefill (KV-cache append in the CTA-pair GEMM epilogue) ==
    zq_linear + zq_kv_append: the qkv output and both caches bit for bit.  Shapes
    off the pair path (few rows) or with sequences not a multiple of 32 tokens
    return ZQ_ERR_UNSUPPORTED (the decoder then runs the unfused pair)."""
    from paper_2206_01861_b200 import _native as N
    from paper_2206_01861_b200 import quant

    batch, T, dl, max_ctx = shape
    m = batch * T
    rng = np.random.default_rng(sum(shape))
    xq = quant.quantize_activation_tokenwise(torch.from_numpy(rng.standard_normal((m, dl)).astype(np.float32)).cuda(), 8)
    w = quant.quantize_weight_groupwise(torch.from_numpy((rng.standard_normal((3 * dl, dl)) * 0.02).astype(np.float32)).cuda(), 16, 8)
    bias = torch.from_numpy((rng.standard_normal(3 * dl) * 0.1).astype(np.float32)).cuda()
    a = xq.gemm_operand()
    wp, ldw, wb = w.weight_operand()
    outs = []
    for fused in (False, True):
        qkv = torch.empty(m, 3 * dl, device="cuda")
        kc = torch.full((batch, max_ctx, dl), 7.0, device="cuda")
        vc = torch.full((batch, max_ctx, dl), 7.0, device="cuda")
        pos = torch.zeros(batch, dtype=torch.int32, device="cuda")
        if fused:
            rc = N.call_rc("zq_linear_kv_prefill", a.data_ptr(), a.stride(0), xq.token_scales.data_ptr(), wp, ldw,
                           wb, w.row_scales().data_ptr(), bias.data_ptr(), m, 3 * dl, dl, qkv.data_ptr(),
                           qkv.stride(0), kc.data_ptr(), vc.data_ptr(), dl, max_ctx, T, N.stream_ptr())
            if rc == N.ZQ_ERR_UNSUPPORTED:
                assert T % 32 != 0 or m // 256 * (3 * dl // 128) < 74, shape
                return
        else:
            N.call("zq_linear", a.data_ptr(), a.stride(0), xq.token_scales.data_ptr(), 0.0, wp, ldw, wb,
                   w.row_scales().data_ptr(), bias.data_ptr(), m, 3 * dl, dl, qkv.data_ptr(), qkv.stride(0),
                   N.OUT_F32, N.stream_ptr())
            N.call("zq_kv_append", qkv.data_ptr(), qkv.stride(0), batch, T, dl, pos.data_ptr(), kc.data_ptr(),
                   vc.data_ptr(), max_ctx, N.stream_ptr())
        outs.append((qkv, kc, vc))
    for a0, a1 in zip(outs[0], outs[1]):
        assert torch.equal(a0.view(torch.int32), a1.view(torch.int32)), shape


@pytest.mark.parametrize("cfg_name", ["gpt3-350m", "gptj-6b"])
def test_fused_prefill_kv_append_engine_bit_identical(cfg_name, monkeypatch):
    """DecoderEngine prefill with the KV-cache append in the CTA-pair QKV GEMM's
    epilogue (whole 32-token sequences, M large enough for the pair path) gives
    the same caches, hidden state and greedy tokens, bit for bit, as the
    separate zq_kv_append pass (ZQ_KV_PREFILL=0)."""
    from paper_2206_01861_b200.decoder import CONFIGS, DecoderEngine

    cfg = CONFIGS[cfg_name]
    batch, T = (8, 256) if cfg_name == "gpt3-350m" else (16, 128)
    ids = torch.from_numpy(np.random.default_rng(3).integers(0, cfg.vocab, (batch, T))).cuda()
    res = []
    for env in ("0", "1"):
        monkeypatch.setenv("ZQ_KV_PREFILL", env)
        eng = DecoderEngine(cfg, batch, T + 4, seed=5, layers=2, use_graph=False)
        toks = [eng.prefill(ids).clone()]
        for _ in range(2):
            toks.append(eng.step().clone())
        res.append((torch.stack(toks, 1), eng.kcache[1][:, :T + 2].clone(), eng.vcache[0][:, :T + 2].clone(),
                    eng._buffers(batch)["x"].clone()))
        del eng
        torch.cuda.empty_cache()
    for a, b in zip(res[0], res[1]):
        assert torch.equal(a.view(torch.int32) if a.dtype == torch.float32 else a,
                           b.view(torch.int32) if b.dtype == torch.float32 else b), cfg_name

"""GPU: the tensor-parallel block path over the sm_100a kernels (CudaOps), on a
single-rank NCCL group (the only topology a 1-GPU box offers).  The row-parallel
route (row absmax -> MAX all-reduce -> quantize with global scale -> int32 GEMM
-> SUM all-reduce -> epilogue) must reproduce the fused single-GPU block
forward bit for bit."""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("causal", [False, True])
def test_tp_cuda_ops_equal_fused_block(nccl_group, causal):
    from paper_2206_01861_b200 import tp
    from paper_2206_01861_b200 import transformer as T

    d, heads = 256, 4
    blk = T.random_block(d, heads, 8, 8, 16, seed=3)
    blk.b_o.normal_(0, 0.01)
    blk.b_4hh.normal_(0, 0.01)
    x = torch.randn(2 * 64, d, device="cuda") * 0.5
    prec = T.PrecisionConfig.from_scheme("W8A8", group_count=16)
    ref = T.block_forward(x, blk, prec, causal, batch=2)
    ops = tp.CudaOps()
    sb = tp.shard_block(blk, ops, 0, 1)
    y = tp.tp_block_forward(x, sb, ops, causal, group=nccl_group, batch=2)
    assert torch.equal(y, ref)


def test_forced_tp_decoder_graph_capture_matches_local(nccl_group):
    """DecoderEngine(force_tp=True) on the 1-rank NCCL group routes o / 4hh
    through tp.row_parallel_linear, so the MAX and int32 SUM all-reduces are
    captured inside the decode step's CUDA graph; tokens and hidden states must
    equal the local fused path bit for bit (graph replay of NCCL included)."""
    import numpy as np

    from paper_2206_01861_b200.decoder import DecoderEngine, GPTConfig

    cfg = GPTConfig("tiny-tp", 2, 512, 8, 2048, 1024, 8, 8, 32)
    ids = np.random.default_rng(3).integers(0, cfg.vocab, (4, 6))
    res = []
    for force in (False, True):
        eng = DecoderEngine(cfg, 4, 16, seed=2, tp=(nccl_group, 0, 1) if force else None, force_tp=force,
                            use_graph=True)
        toks = [eng.prefill(ids).cpu().numpy()]
        hs = [eng._buffers(4 * 6)["out"][:4].cpu().numpy()]
        for _ in range(5):
            toks.append(eng.step().cpu().numpy())
            hs.append(eng._buffers(4)["out"][:4].cpu().numpy())
        eng.check_finite()
        res.append((np.stack(toks, 1), np.stack(hs)))
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][1].view(np.uint32), res[1][1].view(np.uint32))

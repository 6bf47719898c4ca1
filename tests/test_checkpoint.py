"""ZQCK checkpoints (reference pkg/src/lowbit/checkpoint.py).
The fixture tests/golden/tiny_w48a8.zqck was written by the reference's own
save_model (oracle/make_checkpoint_fixture.py); tiny_w48a8_ref.npz holds the
reference model_forward logits for a token sequence."""

import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "golden", "tiny_w48a8.zqck")
REF = os.path.join(ROOT, "tests", "golden", "tiny_w48a8_ref.npz")


def test_read_reference_checkpoint_and_round_trip(tmp_path):
    from paper_2206_01861_b200 import checkpoint as C

    m = C.read_checkpoint(FIX)
    assert (m.vocab, m.dim, m.num_heads, m.num_layers, m.causal) == (128, 64, 4, 2, True)
    for blk in m.blocks:
        assert blk["quantized"]
        assert [blk[n].bits for n in ("w_q", "w_k", "w_v", "w_o", "w_h4h", "w_4hh")] == [8, 8, 8, 8, 4, 4]
        assert blk["w_h4h"].values.shape == (256, 64) and len(blk["w_h4h"].group_layout) == 16
        assert np.abs(blk["w_h4h"].values).max() <= 7
    out = tmp_path / "rt.zqck"
    C.write_checkpoint(m, str(out))
    assert out.read_bytes() == open(FIX, "rb").read()  # bit-exact round trip


@pytest.mark.parametrize("damage", ["magic", "version", "truncate", "trailing"])
def test_bad_checkpoints_raise_usage_error(tmp_path, damage):
    from paper_2206_01861_b200 import checkpoint as C
    from paper_2206_01861_b200.errors import UsageError

    data = bytearray(open(FIX, "rb").read())
    if damage == "magic":
        data[:4] = b"XXXX"
    elif damage == "version":
        data[4:8] = (7).to_bytes(4, "little")
    elif damage == "truncate":
        data = data[:-5]
    else:
        data += b"\0"
    p = tmp_path / "bad.zqck"
    p.write_bytes(bytes(data))
    with pytest.raises(UsageError):
        C.read_checkpoint(str(p))


@pytest.mark.gpu
def test_device_model_matches_reference_logits():
    import torch

    from paper_2206_01861_b200 import checkpoint as C
    from paper_2206_01861_b200 import igemm
    from paper_2206_01861_b200 import transformer as T

    dm = C.load_model(FIX)
    ref = np.load(REF)
    prec = T.PrecisionConfig.from_scheme("W4/8A8", group_count=16)
    x = dm.embedding[torch.from_numpy(ref["ids"]).cuda()]
    for li, blk in enumerate(dm.blocks):
        assert blk.w_h4h.bits == 4 and blk.w_h4h.packed4 is not None
        x = T.block_forward(x, blk, prec, dm.causal, layer=li)
    h = torch.empty_like(x)
    igemm.layer_norm_quantize(x, dm.final_gamma, dm.final_beta, 8, ln_out=h)
    logits = (h @ dm.embedding.t()).cpu().numpy().astype(np.float64)
    r = ref["logits"].astype(np.float64)
    assert np.linalg.norm(logits - r) / np.linalg.norm(r) < 2e-3
    assert (logits.argmax(1) == r.argmax(1)).mean() >= 0.9

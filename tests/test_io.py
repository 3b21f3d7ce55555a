"""Bank / checkpoint containers (reference adapters.py:265-306, model.py:481-541).

CPU part: the files the UNMODIFIED reference wrote (tests/golden/ref_bank.npz, ref_checkpoint.npz,
made by tests/golden/make_golden.py) load into the host mirror's containers with identical values,
in the packed per-layer device layout; what `save_bank` writes has the reference's container layout.
GPU part: a loaded checkpoint decodes the tokens the reference decoded from the same weights, and
save -> load round-trips bit for bit."""

import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def test_load_reference_bank_on_host():
    from paper_2603_11873_b200.adapters import load_bank

    bank, downs, ups = load_bank(os.path.join(GOLD, "ref_bank.npz"), device="cpu", packed=True)
    ref = np.load(os.path.join(GOLD, "ref_bank.npz"))
    hdr = json.loads(bytes(ref["header"]).decode())
    assert (bank.n_layers, bank.n_experts, bank.rank) == (hdr["n_layers"], hdr["n_experts"], hdr["rank"])
    assert len(downs) == bank.n_layers and tuple(downs[0].shape) == (bank.n_experts, bank.rank, 32)
    assert tuple(ups[0].shape) == (bank.n_experts, 32, bank.rank) and downs[0].is_contiguous() and ups[0].is_contiguous()
    for li in range(bank.n_layers):
        for ei in range(bank.n_experts):
            np.testing.assert_array_equal(bank.layers[li][ei].down.numpy(), ref[f"layer{li}/expert{ei}/down"])
            np.testing.assert_array_equal(bank.layers[li][ei].up.numpy(), ref[f"layer{li}/expert{ei}/up"])
            # experts are views into the packed tensors, not copies
            assert bank.layers[li][ei].down.data.data_ptr() == downs[li][ei].data_ptr()
    # the fixture is on the bf16 grid: loading it as bf16 loses nothing
    b16 = load_bank(os.path.join(GOLD, "ref_bank.npz"), precision="bf16", device="cpu")
    np.testing.assert_array_equal(b16.layers[1][2].up.numpy(), ref["layer1/expert2/up"])


def test_save_bank_writes_the_reference_container(tmp_path):
    from paper_2603_11873_b200.adapters import load_bank, save_bank

    bank = load_bank(os.path.join(GOLD, "ref_bank.npz"), precision="bf16", device="cpu")
    out = tmp_path / "bank.npz"
    save_bank(bank, out)
    a, ref = np.load(out), np.load(os.path.join(GOLD, "ref_bank.npz"))
    assert set(a.keys()) == set(ref.keys())
    hdr = json.loads(bytes(a["header"]).decode())
    assert hdr["format"] == "lorafuse-bank-v1" and hdr["precision"] == "single" and hdr["device_precision"] == "bf16"
    for k in ref.keys():
        if k != "header":
            assert a[k].dtype == np.float32
            np.testing.assert_array_equal(a[k], ref[k])
    again = load_bank(out, device="cpu")
    assert again.layers[0][0].down.precision == "bf16"
    with pytest.raises(ValueError):
        np.savez(tmp_path / "bad.npz", header=np.frombuffer(b'{"format": "nope"}', dtype=np.uint8))
        load_bank(tmp_path / "bad.npz", device="cpu")


@pytest.mark.gpu
def test_checkpoint_from_the_reference_decodes_its_tokens(tmp_path):
    import torch

    import paper_2603_11873_b200 as af

    exp = np.load(os.path.join(GOLD, "ref_io_expected.npz"))
    for prec in ("single", "bf16"):
        model = af.load_checkpoint(os.path.join(GOLD, "ref_checkpoint.npz"), precision=prec)
        assert model.config.precision == prec and model.table.info()["n_segments"] == model.config.layers
        ref = np.load(os.path.join(GOLD, "ref_checkpoint.npz"))
        np.testing.assert_array_equal(model.backbone[1].numpy(), ref["backbone1"])
        toks, _ = af.generate(model, [3, 11, 40], 10, af.DispatchRecorder())
        assert toks == [int(t) for t in exp["tokens"]]
        assert af.max_backbone_deviation(model) < 0.02
        # save -> load: bit for bit, pristine weights even though a generation ran in between
        out = tmp_path / f"ckpt_{prec}.npz"
        af.save_checkpoint(model, out)
        back = af.load_checkpoint(out)
        assert back.config.precision == prec
        for a, b in zip(model.pristine_backbone, back.backbone):
            assert torch.equal(a.data, b.data)
        for a, b in zip(model.bank_up, back.bank_up):
            assert torch.equal(a, b)
        assert af.weights_digest(back) == af.weights_digest(af.load_checkpoint(out))

"""The caller of the path end to end (examples/train_mlp_adt.py): simulated
data-parallel workers train an MLP on replicas produced by the B200 path
(fused gradient combine + SGD + pack + norm, unpack, AWP); the loss falls,
AWP widens layers and the weight stream stays below FP32; with the decision
on the device the run is identical (same widths, same loss trajectory)."""

import os
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def example():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    sys.path.insert(0, os.path.join(ROOT, "examples"))
    import train_mlp_adt
    return train_mlp_adt


def test_training_with_adt_awp(example):
    fp32 = example.main(["--steps", "120", "--workers", "4", "--fp32"])
    assert fp32["weight_bytes_vs_fp32"] == 1.0
    host = example.main(["--steps", "120", "--workers", "4", "--interval", "5"])
    assert host["final_loss"] < 0.5 * host["first_loss"]
    assert abs(host["val_accuracy"] - fp32["val_accuracy"]) < 0.03     # the paper's claim, at toy scale
    assert host["weight_bytes_vs_fp32"] < 1.0 and max(host["final_bits"]) > 8
    dev = example.main(["--steps", "120", "--workers", "4", "--interval", "5", "--awp-on-device"])
    assert dev["final_bits"] == host["final_bits"]
    assert dev["final_loss"] == host["final_loss"] and dev["val_accuracy"] == host["val_accuracy"]
    assert dev["weight_bytes_vs_fp32"] == pytest.approx(host["weight_bytes_vs_fp32"])

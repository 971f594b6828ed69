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


def _dp_rank(rank, world, port, q, argv):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank), ADT_EXAMPLE_BACKEND="gloo")
    try:
        sys.path.insert(0, os.path.join(ROOT, "examples"))
        import train_mlp_dp
        q.put((rank, train_mlp_dp.main(argv)))
    except Exception as e:  # surface child failures to the parent
        import traceback
        q.put((rank, {"error": repr(e), "tb": traceback.format_exc()}))


@pytest.mark.parametrize("transport", ["p2p", "nccl", "p2p-device-awp"])
def test_dp_training_over_ranks_matches_simulated_workers(example, transport):
    """examples/train_mlp_dp.py with 2 ranks (sharing this GPU through gloo)
    runs the same training as examples/train_mlp_adt.py with 2 simulated
    workers: same widths chosen, same losses and accuracy (the sharded master
    update is bit-exact; only the norms' partial-sum grouping differs), and
    both ranks end with bit-identical replicas."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    argv = ["--steps", "60", "--interval", "5", "--transport", transport.split("-")[0]]
    if transport.endswith("device-awp"):
        argv.append("--awp-on-device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dp_rank, args=(r, 2, port, q, argv)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    for rank, out in res:
        assert "error" not in out, (rank, out.get("tb"))
        assert out["replicas_identical"] and out["transport"] == transport.split("-")[0]
    dp = res[0][1]
    sim = example.main(["--steps", "60", "--workers", "2", "--interval", "5"])
    assert dp["final_bits"] == sim["final_bits"] and max(dp["final_bits"]) > 8
    assert dp["first_loss"] == sim["first_loss"]
    assert dp["final_loss"] == pytest.approx(sim["final_loss"], rel=1e-6)
    assert dp["val_accuracy"] == pytest.approx(sim["val_accuracy"], abs=1e-3)
    assert dp["weight_bytes_vs_fp32"] == pytest.approx(sim["weight_bytes_vs_fp32"])


def test_cpu_master_training_loop():
    """examples/train_mlp_cpu_master.py — the paper's CPU-master setting as a
    training loop: host masters updated by the CPU, packed on the host at the
    AWP widths (HostWeightSync), unpacked on the GPU for the workers, FP32
    gradients back. The loss falls, AWP widens layers, the weight stream stays
    below FP32 and the accuracy matches the uncompressed run."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    sys.path.insert(0, os.path.join(ROOT, "examples"))
    import train_mlp_cpu_master as ex
    fp32 = ex.main(["--steps", "120", "--fp32", "--sizes", "64,512,512,10"])
    assert fp32["weight_bytes_vs_fp32"] == 1.0 and fp32["final_loss"] < 0.5 * fp32["first_loss"]
    awp = ex.main(["--steps", "120", "--interval", "5", "--threshold", "1e-3", "--sizes", "64,512,512,10"])
    assert awp["final_loss"] < 0.5 * awp["first_loss"]
    assert abs(awp["val_accuracy"] - fp32["val_accuracy"]) < 0.03
    assert awp["weight_bytes_vs_fp32"] < 1.0 and max(awp["final_bits"]) > 8
    assert awp["trace_rows"] == 120 * 3

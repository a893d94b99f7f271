"""The one-launch network kernel (bnn_net_infer, csrc/net_b1.cu; the batch-1 latency path) against
the C oracle: logits and predictions bit-exact on the shipped and the calibrated (informative) models,
batches 1..8, device and zero-copy (pinned host) buffers, plain launches and CUDA-graph replays.
Mirrors the reference's full-model matrix (tests/test_acceptance.py:217-247: both architectures,
B in {1, 2, 4, 8})."""

import numpy as np
import pytest

from tests.helpers import model_with_steps, trace_images

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    from paper_2301_05126_b200.engine import Engine

    with Engine() as e:
        yield e


def _cal(golden, arch):
    cal = next(c for c in golden["calibrated"] if c["arch"] == arch)
    return model_with_steps(cal["arch"], cal["seed"], cal["steps"])


def _net_run(pm, imgs, host=False, max_batch=None):
    import torch

    from paper_2301_05126_b200.engine import NetPlan

    B = imgs.shape[0]
    net = NetPlan(pm, max_batch or B)
    if host:
        x = torch.from_numpy(imgs.astype(np.uint8)).pin_memory()
        lg = torch.zeros((B, pm.num_classes), dtype=torch.int32).pin_memory()
        pr = torch.zeros((B,), dtype=torch.int32).pin_memory()
    else:
        x = torch.from_numpy(imgs.astype(np.uint8)).cuda()
        lg = torch.zeros((B, pm.num_classes), dtype=torch.int32, device="cuda")
        pr = torch.zeros((B,), dtype=torch.int32, device="cuda")
    net.launch(x, lg, pr)
    torch.cuda.synchronize()
    return lg.cpu().numpy(), pr.cpu().numpy(), net


@pytest.mark.parametrize("arch", ["fashion", "cifar10"])
@pytest.mark.parametrize("batch", [1, 2, 4, 8])
def test_net_calibrated_vs_oracle(engine, golden, oracle_mod, arch, batch):
    m = _cal(golden, arch)
    imgs = trace_images(m, 1000 + batch, batch)
    pm = engine.prepare(m)
    logits, preds, _ = _net_run(pm, imgs)
    ol, op = oracle_mod.infer(m, imgs, route="packed")
    assert np.array_equal(logits, ol), (logits, ol)
    assert np.array_equal(preds, op)


@pytest.mark.parametrize("arch,seed", [("fashion", 7), ("cifar10", 1)])
def test_net_shipped_models_and_zero_copy(engine, oracle_mod, arch, seed):
    import paper_2301_05126_b200 as P

    m = P.export_synthetic_model(arch, seed)
    imgs = trace_images(m, 123 if arch == "fashion" else 45, 3)
    pm = engine.prepare(m)
    ol, op = oracle_mod.infer(m, imgs, route="packed")
    for host in (False, True):
        logits, preds, _ = _net_run(pm, imgs, host=host)
        assert np.array_equal(logits, ol) and np.array_equal(preds, op), host


def test_net_reference_golden_vector(engine, golden):
    import paper_2301_05126_b200 as P

    ref = golden["reference_golden_fashion_seed7"]
    m = P.export_synthetic_model("fashion", 7)
    imgs = np.random.default_rng(123).integers(0, 256, size=(1, 1, 28, 28))
    logits, preds, _ = _net_run(engine.prepare(m), imgs, host=True)
    assert logits.tolist() == [ref["logits"]]
    assert preds.tolist() == ref["predictions"]


def test_net_smaller_batch_than_plan_and_repeated(engine, golden, oracle_mod):
    """A plan sized for 8 runs batches 1..8; 200 back-to-back launches (the barrier counter is reset
    by every launch) keep giving the oracle's answer."""
    import torch

    m = _cal(golden, "cifar10")
    pm = engine.prepare(m)
    imgs = trace_images(m, 77, 8)
    ol, op = oracle_mod.infer(m, imgs, route="packed")
    for b in (1, 5, 8):
        logits, preds, net = _net_run(pm, imgs[:b], max_batch=8)
        assert np.array_equal(logits, ol[:b]) and np.array_equal(preds, op[:b])
    x = torch.from_numpy(imgs.astype(np.uint8)).cuda()
    lg = torch.zeros((8, 10), dtype=torch.int32, device="cuda")
    pr = torch.zeros((8,), dtype=torch.int32, device="cuda")
    for _ in range(200):
        net.launch(x, lg, pr)
    torch.cuda.synchronize()
    assert np.array_equal(lg.cpu().numpy(), ol) and np.array_equal(pr.cpu().numpy(), op)


@pytest.mark.parametrize("zero_copy", [False, True])
def test_net_graph_replay(engine, golden, oracle_mod, zero_copy):
    for arch in ("fashion", "cifar10"):
        m = _cal(golden, arch)
        g = engine.graph(m, batch=1, zero_copy=zero_copy, net=True)
        assert g.launches == 1
        imgs = trace_images(m, 31, 6)
        ol, op = oracle_mod.infer(m, imgs, route="packed")
        for i in range(6):
            logits, preds = g.replay(imgs[i:i + 1])
            assert np.array_equal(logits, ol[i:i + 1]) and np.array_equal(preds, op[i:i + 1]), (arch, i)
        assert g.kernels_only_us(reps=20) > 0


def test_net_rejects_bad_calls(engine, golden):
    import torch

    from paper_2301_05126_b200.engine import NetPlan
    from paper_2301_05126_b200.errors import ShapeMismatch

    pm = engine.prepare(_cal(golden, "fashion"))
    net = NetPlan(pm, 2)
    x = torch.zeros((3, 1, 28, 28), dtype=torch.uint8, device="cuda")
    lg = torch.zeros((3, 10), dtype=torch.int32, device="cuda")
    with pytest.raises(ShapeMismatch):
        net.launch(x, lg, lg[:, 0])
    with pytest.raises(ShapeMismatch):
        net.launch(x[:2].to(torch.int32), lg, lg[:, 0])


@pytest.mark.parametrize("arch,batch", [("fashion", 1), ("cifar10", 1), ("cifar10", 4)])
def test_net_server_requests_vs_oracle(engine, golden, oracle_mod, arch, batch):
    """The resident server (bnn_net_serve_*): many doorbell requests, every answer the oracle's."""
    m = _cal(golden, arch)
    imgs = trace_images(m, 500 + batch, 12 * batch)
    ol, op = oracle_mod.infer(m, imgs, route="packed")
    with engine.serve(m, batch=batch) as srv:
        for i in range(12):
            logits, preds = srv.infer(imgs[i * batch:(i + 1) * batch])
            assert np.array_equal(logits, ol[i * batch:(i + 1) * batch]), (arch, i)
            assert np.array_equal(preds, op[i * batch:(i + 1) * batch])
    assert not srv.open


def test_net_server_many_requests(engine, golden, oracle_mod):
    """200 back-to-back requests (fashion, batch 2): the per-request handshake (CTA 0 stages the images,
    gpu-scope broadcast, acq_rel last-arriver detection, system-scope completion release) never hands
    back a stale or torn answer."""
    m = _cal(golden, "fashion")
    imgs = trace_images(m, 4242, 400)
    ol, op = oracle_mod.infer(m, imgs, route="packed")
    with engine.serve(m, batch=2) as srv:
        for i in range(200):
            logits, preds = srv.infer(imgs[2 * i:2 * i + 2])
            assert np.array_equal(logits, ol[2 * i:2 * i + 2]), i
            assert np.array_equal(preds, op[2 * i:2 * i + 2]), i


def test_net_server_idle_timeout(engine, golden):
    import time

    from paper_2301_05126_b200.errors import NativeError

    m = _cal(golden, "fashion")
    srv = engine.serve(m, batch=1, idle_s=0.3)
    srv.infer(trace_images(m, 1, 1))
    time.sleep(1.0)
    with pytest.raises(NativeError):
        srv.infer(trace_images(m, 2, 1))
    srv.close()  # the kernel has already exited

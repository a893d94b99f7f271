"""Multi-GPU host logic on CPU: world_size-2 gloo, image sharding, gather, max-over-ranks.

The GPU compute is replaced by the CPU oracle *inside the test only* (a stand-in
engine); what is under test is the sharding / gather / timing plumbing of
paper_2301_05126_b200/parallel.py, which is identical on the B200 box (NCCL).
"""

import os
import socket

import numpy as np
import pytest

from paper_2301_05126_b200 import parallel


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 262144, 1001):
        for ws in (1, 2, 3, 4, 8):
            spans = [parallel.shard_bounds(n, ws, r) for r in range(ws)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        parallel.shard_bounds(10, 2, 2)


class _OracleEngine:
    """Test stand-in for Engine.infer (CPU oracle)."""

    def __init__(self, oracle):
        self.oracle = oracle

    def infer(self, model, images):
        logits, preds = self.oracle.infer(model, images, route="packed", threads=1)
        return logits, list(preds)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(ws), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import torch.distributed as dist

    from oracle import oracle
    from paper_2301_05126_b200.synthetic import export_synthetic_model, make_images

    parallel.init("gloo")
    model = export_synthetic_model("fashion", 7)
    images = make_images(model, 7, 2026)  # odd count: uneven shards
    res = parallel.sharded_infer(_OracleEngine(oracle), model, images)
    slowest = parallel.max_over_ranks(float(rank + 1))
    total = parallel.sum_over_ranks(1.0)
    if rank == 0:
        full_l, full_p = oracle.infer(model, images, route="packed", threads=1)
        q.put((np.array_equal(res[0], full_l), np.array_equal(res[1], full_p), slowest, total))
    else:
        q.put(("other", res is None, slowest, total))
    parallel.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shard_and_gather():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    main = next(o for o in out if o[0] != "other")
    other = next(o for o in out if o[0] == "other")
    assert main[0] and main[1], "gathered shards differ from the single-process result"
    assert other[1] is True
    assert main[2] == 2.0 and other[2] == 2.0  # max over ranks
    assert main[3] == 2.0

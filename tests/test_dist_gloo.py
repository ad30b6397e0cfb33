"""CPU, world_size 2 (gloo): the replica-sync host logic (K6) — gradient averaging and FedAvg
parameter averaging — against the oracle's fedavg (which is pinned to the reference's)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_16400_b200 import sync
        g = np.random.default_rng(7 + rank)
        # two "projections" of a LoRA adapter: B (d, r) and A^T (l, r) flattened
        b = g.standard_normal((12, 4)).astype(np.float32)
        at = g.standard_normal((10, 4)).astype(np.float32)
        flat = torch.from_numpy(np.concatenate([b.ravel(), at.ravel()]))
        grads = flat.clone()
        sync.allreduce_grads(grads)
        masters = flat.clone()
        sync.fedavg_params(masters)
        err = None
        try:  # mismatched client must be named
            sync.fedavg_params(torch.zeros(5 if rank == 1 else 6))
        except sync.AggregationError as e:
            err = str(e)
        q.put((rank, b, at, grads.numpy(), masters.numpy(), err))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_replica_sync_matches_fedavg():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=100) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    import oracle
    mb, ma = oracle.fedavg([(res[0][1], res[0][2].T), (res[1][1], res[1][2].T)])
    expect = np.concatenate([mb.ravel(), ma.T.ravel()])
    for rank, _, _, grads, masters, err in res:
        assert np.allclose(grads, expect, rtol=1e-6, atol=1e-7)
        assert np.allclose(masters, expect, rtol=1e-6, atol=1e-7)
        assert err is not None and "client 1" in err


def test_single_process_is_identity():
    from paper_2604_16400_b200 import sync
    t = torch.randn(10)
    before = t.clone()
    assert sync.allreduce_grads(t) is t and torch.equal(t, before)
    assert sync.fedavg_params(t) is t


class _FakeProj:
    def __init__(self):
        self.refreshed = 0

    def refresh_from_master(self):
        self.refreshed += 1


class _FakeStack:
    """The members broadcast_adapter uses: the flat fp32 masters and the bf16-copy refresh."""

    def __init__(self, flat):
        self.flat_master = flat
        self._p = [_FakeProj(), _FakeProj()]

    def projections(self):
        return iter(self._p)

    def refresh_from_master(self):
        for p in self._p:
            p.refresh_from_master()


def _bcast_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_16400_b200.registry import broadcast_adapter
        st = _FakeStack(torch.full((7,), float(rank + 1)))
        broadcast_adapter(st, src=1)
        q.put((rank, st.flat_master.numpy().copy(), [p.refreshed for p in st._p]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_global_adapter_broadcast():
    """The aggregated adapter is pushed from the server replica to every replica (one broadcast
    of the flat fp32 masters, then each replica rewrites its bf16 copies) — the step the
    reference's round protocol omits (engine.py:468-480)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bcast_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=100) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    for rank, flat, refreshed in res:
        assert np.all(flat == 2.0), (rank, flat)  # rank 1's masters everywhere
        assert refreshed == [1, 1]

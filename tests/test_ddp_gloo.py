"""Batch-sharded DDP host logic on CPU with the gloo backend, world size 2
(the N>1 path of bench.py without GPUs).  Per-shard compute is the CPU
oracle (tests only); the product code under test is the shard split and the
bucketed gradient all-reduce of paper_2501_14490_b200.ddp."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import psn_oracle as O
from paper_2501_14490_b200 import ddp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, T, N, C, k, d, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        x = rng.standard_normal((T, N, C)).astype(np.float32)
        dy = rng.standard_normal((T, N, C)).astype(np.float32)
        a, b = ddp.shard_bounds(N, rank, world)
        xs = torch.from_numpy(x)
        assert torch.equal(ddp.shard_batch(xs, rank, world), xs[:, a:b])
        p = O.init_layer(C, k, d, weight_init="uniform", rng=np.random.default_rng(3))
        _, _, _, dW, dg, db = O.train_step(p, x[:, a:b], dy[:, a:b])
        W = torch.nn.Parameter(torch.zeros(C, k, dtype=torch.float64))
        g = torch.nn.Parameter(torch.zeros(C, dtype=torch.float64))
        be = torch.nn.Parameter(torch.zeros(C, dtype=torch.float64))
        W.grad, g.grad, be.grad = (torch.from_numpy(v.copy()) for v in (dW, dg, db))
        ddp.allreduce_grads([W, g, be])
        out[rank] = (W.grad.numpy().copy(), g.grad.numpy().copy(), be.grad.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N", [8, 7])
def test_sharded_grads_equal_sum_of_shard_grads(N):
    T, C, k, d, world = 48, 6, 3, 2, 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, T, N, C, k, d, out), nprocs=world, join=True)
    rng = np.random.default_rng(7)
    x = rng.standard_normal((T, N, C)).astype(np.float32)
    dy = rng.standard_normal((T, N, C)).astype(np.float32)
    ref = [np.zeros((C, k)), np.zeros(C), np.zeros(C)]
    for r in range(world):
        a, b = ddp.shard_bounds(N, r, world)
        p = O.init_layer(C, k, d, weight_init="uniform", rng=np.random.default_rng(3))
        _, _, _, dW, dg, db = O.train_step(p, x[:, a:b], dy[:, a:b])
        for acc, v in zip(ref, (dW, dg, db)):
            acc += v
    for r in range(world):
        for got, want in zip(out[r], ref):
            np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-13)


def test_shard_bounds_cover_batch():
    for N in range(1, 20):
        for world in range(1, 6):
            spans = [ddp.shard_bounds(N, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == N
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        ddp.shard_bounds(4, 2, 2)

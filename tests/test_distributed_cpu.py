"""Multi-process (gloo, world_size 2) tests of the sharded metric reduction (CPU)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import holo_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, coefs, M, P, out):
    import torch
    import torch.distributed as dist
    from paper_2204_02348_b200 import distributed as D
    from paper_2204_02348_b200.engine import mode_group_of_index
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B = coefs.shape[0]
    s0, s1 = D.shard(B, world, rank)
    local = coefs[s0:s1]
    off, n = D.exclusive_prefix(local.shape[0])
    assert off == s0 and n == B
    labels = [q * 1000 + mode_group_of_index(i) for q in range(P) for i in range(M)]
    rp, dp, gp, gram = D.host_partials(local, labels, off, min(B, P * M))
    t = lambda a: torch.as_tensor(a)  # noqa: E731
    vals = D.reduce_and_finish(t(rp), t(dp), t(gp), t(gram), B, P * M)
    out[rank] = vals
    dist.destroy_process_group()


@pytest.mark.parametrize("B,M,P", [(12, 10, 1), (7, 6, 2), (40, 15, 1)])
def test_sharded_metrics_equal_single_process(B, M, P):
    rng = np.random.default_rng(B * 100 + M)
    coefs = (rng.standard_normal((B, P * M)) + 1j * rng.standard_normal((B, P * M))).astype(np.complex64)
    coefs[np.arange(min(B, P * M)), np.arange(min(B, P * M))] *= 5.0
    manager = mp.Manager()
    out = manager.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, coefs, M, P, out), nprocs=2, join=True)
    groups = [O.group_of_mode(i) for i in range(M)]
    labels = [q * 1000 + g for q in range(P) for g in groups]
    ref = O.metrics_one(O.transfer_matrix(coefs, M, P), labels)
    for r in range(2):
        got = np.asarray(out[r])
        assert np.allclose(got, ref, atol=1e-6, rtol=0), (got, ref)


def test_shard_partition_covers_batch():
    from paper_2204_02348_b200.distributed import shard
    for B in (1, 7, 1000, 65536):
        for world in (1, 2, 4, 8):
            spans = [shard(B, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))

"""world_size-2 gloo test of the multi-rank plumbing (halo all-to-all, scalar
allreduce, domain->rank mapping) on CPU tensors, as the N>1 path cannot be run
on the single GPU this round has."""

import os
import socket

import numpy as np
import torch
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as tdist
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2303_08881_b200.dist import Comm, domains_of_rank
    comm = Comm(rank, world, None)
    # scalar allreduce: the dot-product path
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    comm.allreduce_sum_(t)
    ok = float(t) == sum(range(1, world + 1))
    # halo exchange: rank r sends (r+1) values tagged 100*r + k to its peer, none to itself
    send_counts = [0] * world
    send_counts[1 - rank] = rank + 1
    recv_counts = [0] * world
    recv_counts[1 - rank] = (1 - rank) + 1
    send = torch.tensor([100.0 * rank + k for k in range(rank + 1)], dtype=torch.float64)
    recv = torch.empty(sum(recv_counts), dtype=torch.float64)
    comm.all_to_all(recv, send, recv_counts, send_counts)
    expect = [100.0 * (1 - rank) + k for k in range((1 - rank) + 1)]
    ok = ok and recv.tolist() == expect
    ok = ok and list(domains_of_rank(8, comm)) == list(range(4 * rank, 4 * rank + 4))
    out[rank] = bool(ok)
    tdist.destroy_process_group()


def test_comm_two_ranks_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        assert dict(out) == {0: True, 1: True}


def test_domains_of_rank_rejects_uneven():
    import pytest
    from paper_2303_08881_b200.dist import Comm, domains_of_rank
    with pytest.raises(ValueError):
        domains_of_rank(6, Comm(0, 4, None))
    assert list(domains_of_rank(1, Comm())) == [0]

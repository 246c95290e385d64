"""Two ranks sharing one GPU (gloo, tensors staged through the host): the whole
multi-rank path -- subdomain blocks per rank, halo plan, halo exchange inside
SpMV and the interface matvec, allreduced dots -- must reproduce the
single-rank solve (same p, so the same preconditioner: strong-scaling invariant)."""

import json
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = [("bj", 4), ("schur", 8), ("rap", 4), ("rap-milu", 8)]
DIMS = (20, 18, 16)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _solve_all(P, cases=None):
    out = {}
    a = P.aniso3d(*DIMS)
    b = P.default_rhs(a) if False else None
    for pc, p in (cases or CASES):
        a = P.aniso3d(*DIMS)
        layout = P.classify_and_order(a, P.partition(a, p, DIMS), p)
        m = P.make_preconditioner(pc, a, layout)
        import torch
        from paper_2303_08881_b200 import device as D
        ones = torch.ones(a.n_cols, dtype=torch.float64, device="cuda")
        bd = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
        D.spmv(a.device(), ones, bd)
        rhs = bd.cpu().numpy()
        x, rep = P.fgmres(a, rhs, m=m.apply)
        r = np.random.default_rng(3).standard_normal(a.n_rows)
        z = m.apply(r)
        out[f"{pc}|{p}"] = {"its": rep.iterations, "relres": rep.final_relres, "x": x.tolist(), "z": z.tolist(),
                            "n_halo": int(m.system.n_halo), "n_loc": int(m.system.n_loc)}
    return out


def _worker(rank, world, port, path, backend="gloo", cases=None, peer=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank) if backend == "nccl" else "0", DDILU_PEER="1" if peer else "0")
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2303_08881_b200 as P
    from paper_2303_08881_b200 import dist
    comm = dist.init_from_env(backend=backend)
    assert comm.size == world and comm.rank == rank
    assert isinstance(comm, dist.PeerComm) == bool(peer)
    res = _solve_all(P, cases)
    if peer:
        comm.check()                      # no bounded wait ran out
        res["_peer"] = {"reductions": comm.red_seq, "halo_exchanges": comm.halo_seq}
        comm.close()
    with open(f"{path}.{rank}", "w") as fh:
        json.dump(res, fh)
    import torch.distributed as tdist
    tdist.barrier()
    tdist.destroy_process_group()


def _run_two_ranks(tmp_path, backend, cases=None, peer=False):
    import paper_2303_08881_b200 as P
    single = _solve_all(P, cases)
    world, port, path = 2, _free_port(), str(tmp_path / "res")
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, path, backend, cases, peer)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    for rank in range(world):
        multi = json.load(open(f"{path}.{rank}"))
        if peer:
            used = multi.pop("_peer")
            assert used["reductions"] > 100 and used["halo_exchanges"] > 100, used     # the peer kernels carried the solve
        for key, ref in single.items():
            got = multi[key]
            assert got["n_halo"] > 0 and got["n_loc"] < ref["n_loc"], key      # really distributed
            assert abs(got["its"] - ref["its"]) <= 1, (key, got["its"], ref["its"])
            assert got["relres"] <= 1e-8
            assert np.max(np.abs(np.array(got["x"]) - np.array(ref["x"]))) < 1e-6, key
            scale = np.max(np.abs(ref["z"]))
            assert np.max(np.abs(np.array(got["z"]) - np.array(ref["z"]))) < 1e-9 * scale, key


def test_two_ranks_match_single_rank(tmp_path):
    _run_two_ranks(tmp_path, "gloo")


def test_two_ranks_nccl(tmp_path):
    """The production transport: one rank per GPU, NCCL all_to_all_single straight into the halo tail (interior
    SpMV rows overlapped), allreduce on device scalars.  Needs two GPUs; the single-GPU boxes of this project's
    test tier skip it, so the NCCL branch of dist.py is UNVERIFIED on hardware until a multi-GPU run executes it."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (NCCL path; covered over gloo by test_two_ranks_match_single_rank)")
    _run_two_ranks(tmp_path, "nccl")


def test_two_ranks_peer_memory(tmp_path):
    """The same comparison with the exchanges over PEER MEMORY (csrc/peer.cu, dist.PeerComm): halo values stored
    straight into the other rank's mailbox (CUDA IPC mapping) and published by sequence flags, dot / norm scalars
    reduced by one kernel per rank that polls its own flags -- no collective call on the solve path.  Two processes
    share the one GPU here (their kernels alternate by time slicing, every hand-over costs a time slice); with one
    GPU per rank the same code runs over NVLink."""
    _run_two_ranks(tmp_path, "gloo", cases=[("schur", 8), ("bj", 4)], peer=True)

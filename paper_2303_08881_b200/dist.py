"""Multi-GPU plumbing: one process per GPU, `torch.distributed` (NCCL over
NVLink / NVSwitch) for the two exchanges the path has:

1. halo of interface (exterior) values before a product with A or with the
   interface coupling E_off: packed by a gather kernel, moved with ONE
   all_to_all_single straight into the halo tail of the vector;
2. sum-allreduce of the dot / norm scalars of the Krylov loops.

Subdomains map to ranks in contiguous blocks (p domains over N ranks, p % N
== 0); with one rank nothing here communicates.  The gloo backend (CPU tests,
or two ranks sharing one GPU) stages device tensors through the host.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

try:
    import torch.distributed as tdist
except Exception:  # pragma: no cover
    tdist = None


@dataclass
class Comm:
    rank: int = 0
    size: int = 1
    group: object = None

    @property
    def active(self) -> bool:
        return self.size > 1

    def _staged(self) -> bool:
        return tdist.get_backend(self.group) == "gloo"

    def allreduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place sum over ranks of a small device tensor (dot / norm scalars)."""
        if not self.active:
            return t
        if self._staged() and t.is_cuda:
            h = t.cpu()
            tdist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            tdist.all_reduce(t, group=self.group)
        return t

    def all_to_all(self, recv: torch.Tensor, send: torch.Tensor, recv_counts, send_counts, async_op: bool = False):
        """Variable-size exchange.  With async_op (NCCL) a work handle is returned:
        the transfer runs on NCCL's stream and `handle.wait()` makes the current
        stream wait for it, so kernels launched in between overlap the exchange."""
        if not self.active:
            return None
        if self._staged():
            sh = send.cpu()
            rh = torch.empty(recv.shape, dtype=recv.dtype)
            outs = list(rh.split(list(recv_counts)))
            ins = list(sh.split(list(send_counts)))
            # gloo has no all_to_all for CPU tensors in every build: pairwise exchange
            reqs = []
            for peer in range(self.size):
                if peer == self.rank:
                    outs[peer].copy_(ins[peer])
                    continue
                if send_counts[peer]:
                    reqs.append(tdist.isend(ins[peer].contiguous(), peer, group=self.group))
                if recv_counts[peer]:
                    reqs.append(tdist.irecv(outs[peer], peer, group=self.group))
            for r in reqs:
                r.wait()
            recv.copy_(rh)
            return None
        return tdist.all_to_all_single(recv, send, list(recv_counts), list(send_counts), group=self.group,
                                       async_op=async_op)

    def barrier(self):
        if self.active:
            tdist.barrier(group=self.group)


_comm = Comm()


def get_comm() -> Comm:
    return _comm


def set_comm(comm: Comm | None) -> Comm:
    """Install the communicator used by setup / solve (None = single rank)."""
    global _comm
    _comm = comm if comm is not None else Comm()
    return _comm


def init_from_env(backend: str | None = None) -> Comm:
    """Join the torchrun job described by RANK / WORLD_SIZE / MASTER_* (if any)."""
    import os
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1:
        return set_comm(None)
    rank = int(os.environ["RANK"])
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() and torch.cuda.device_count() >= world else "gloo"
    if torch.cuda.is_available():
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count())
    if not tdist.is_initialized():
        tdist.init_process_group(backend=backend, rank=rank, world_size=world)
    return set_comm(Comm(rank, world, None))


def domains_of_rank(p: int, comm: Comm) -> range:
    """Contiguous block of subdomains owned by this rank."""
    if p % comm.size:
        raise ValueError(f"{p} subdomains cannot be dealt evenly to {comm.size} ranks")
    per = p // comm.size
    return range(comm.rank * per, (comm.rank + 1) * per)

"""Multi-GPU plumbing: one process per GPU, `torch.distributed` (NCCL over
NVLink / NVSwitch) for the two exchanges the path has:

1. halo of interface (exterior) values before a product with A or with the
   interface coupling E_off: packed by a gather kernel, moved with ONE
   all_to_all_single straight into the halo tail of the vector;
2. sum-allreduce of the dot / norm scalars of the Krylov loops.

Subdomains map to ranks in contiguous blocks (p domains over N ranks, p % N
== 0); with one rank nothing here communicates.  The gloo backend (CPU tests,
or two ranks sharing one GPU) stages device tensors through the host.

`PeerComm` (DDILU_PEER=1) replaces both exchanges by stores into peer memory
and in-kernel flag waits (csrc/peer.cu): no collective call on the solve path.
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

    @property
    def transport(self) -> str:
        return tdist.get_backend(self.group) if self.active else "none"


class _PeerWork:
    """Handle of an exchange started with async_op: wait() enqueues the receiving kernel."""

    def __init__(self, fn):
        self._fn = fn

    def wait(self):
        if self._fn is not None:
            self._fn()
            self._fn = None


class PeerComm(Comm):
    """The two exchanges over PEER MEMORY instead of library collectives (csrc/peer.cu): every rank of the node maps
    every rank's mailbox (CUDA IPC); a halo value is stored straight into the consumer's mailbox and published with a
    sequence flag, a scalar reduction is ONE kernel per rank that writes its partials into all mailboxes, polls its
    own flags and sums in rank order (bitwise the same on every rank).  No host synchronisation, no NCCL call on the
    solve path.  `base` (a torch.distributed communicator) is used once to hand the IPC handles round, for
    reductions of more than `kmax` values (the solution vector of the host-facing API) and for halo messages above
    the reserved capacity.  All ranks must sit on GPUs of one node with peer access (or share a GPU: tests)."""

    HEADER_FLAGS = 4          # flag arrays of `size` int64 each: reduction seq, halo seq, halo ack, spare

    def __init__(self, base: Comm, cap: int = 1 << 16, kmax: int = 512, spin_seconds: float = 20.0):
        super().__init__(base.rank, base.size, base.group)
        self.base = base
        self.kmax = int(kmax)
        self.cap = 0
        self.spin_cycles = int(spin_seconds * 1.9e9)
        self.red_seq = 0
        self.halo_seq = 0
        self._dev = torch.device("cuda", torch.cuda.current_device())
        self.err = torch.zeros(1, dtype=torch.int32, device=self._dev)
        self._counters = torch.zeros(2, dtype=torch.int32, device=self._dev)
        self._offs = {}
        self._alloc(int(cap))

    # ---------------------------------------------------------------- mailboxes
    def _alloc(self, cap: int):
        """(Re)allocate this rank's mailbox and map everybody's: a collective call."""
        from torch.multiprocessing.reductions import reduce_tensor
        from . import device as D
        size = self.size
        torch.cuda.synchronize()
        self.base.barrier()                       # nobody still writes into the old mailboxes
        self.cap = cap
        n_flag = self.HEADER_FLAGS * size
        n_red = 2 * size * self.kmax
        n_data = 2 * size * cap
        self._mail = torch.zeros(n_flag + n_red + n_data, dtype=torch.int64, device=self._dev)    # 8-byte words
        self.red_seq = self.halo_seq = 0
        fn, args = reduce_tensor(self._mail)
        handles = [None] * size
        tdist.all_gather_object(handles, (fn, args), group=self.group)
        self._peers = [self._mail if r == self.rank else handles[r][0](*handles[r][1]) for r in range(size)]
        # kernels of THIS device dereference the peers' pointers: make sure peer access is on (torch enables it on
        # the first device-to-device copy between a pair of devices) and refuse pairs without it
        probe = torch.zeros(1, dtype=torch.int64, device=self._dev)
        for r, t in enumerate(self._peers):
            if r != self.rank and t.device != self._dev:
                if not torch.cuda.can_device_access_peer(self._dev.index, t.device.index):
                    raise RuntimeError(f"no peer access from {self._dev} to {t.device}")
                # torch switches peer access on for "source device may access destination device" on the first copy of
                # a pair: the copy FROM this device INTO the peer's mailbox is the direction our kernels need (the
                # last word of a mailbox is halo data, unused at this point: read it, write the same value back)
                probe.copy_(t[-1:])
                t[-1:].copy_(probe)
        base = [int(t.data_ptr()) for t in self._peers]
        i64 = torch.int64

        def table(offset_words):
            return torch.tensor([b + 8 * offset_words for b in base], dtype=i64, device=self._dev)

        self._red_flags = table(0)
        self._halo_flags = table(size)
        self._ack_flags = table(2 * size)
        self._red_slots = table(n_flag)
        self._data = table(n_flag + n_red)
        self._my_halo_flags = self._mail[size:2 * size]
        self._my_ack = self._mail[2 * size:3 * size]
        self._my_data = self._mail[n_flag + n_red:].view(torch.float64)
        torch.cuda.synchronize()
        self.base.barrier()                       # everybody has mapped everybody
        self._D = D

    def reserve(self, n_doubles: int):
        """Make room for halo messages of n_doubles values per rank pair (collective: the largest request wins)."""
        t = torch.tensor([int(n_doubles)], dtype=torch.int64)
        if tdist.get_backend(self.group) != "gloo":
            t = t.to(self._dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX, group=self.group)
        need = int(t.item())
        if need > self.cap:
            self._alloc(max(need, 2 * self.cap))

    def check(self):
        """Raise if a bounded wait of a peer kernel ran out (one host read)."""
        code = int(self.err.item())
        if code:
            raise RuntimeError(f"peer exchange timed out (code {code}: 1 reduction, 2 halo acknowledgement, 3 halo data)")

    # ---------------------------------------------------------------- exchanges
    def allreduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        if not self.active:
            return t
        k = t.numel()
        if k > self.kmax or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
            return self.base.allreduce_sum_(t)
        self.red_seq += 1
        self._D.call("ddilu_peer_allreduce", k, self.kmax, t, t, self._red_slots, self._red_flags, self.rank, self.size,
                     self.red_seq, self.spin_cycles, self.err)
        return t

    def _offsets(self, counts):
        key = tuple(int(c) for c in counts)
        if key not in self._offs:
            off = [0]
            for c in key:
                off.append(off[-1] + c)
            self._offs[key] = (torch.tensor(off, dtype=torch.int32, device=self._dev), off)
        return self._offs[key]

    def all_to_all(self, recv: torch.Tensor, send: torch.Tensor, recv_counts, send_counts, async_op: bool = False,
                   idx: torch.Tensor | None = None):
        """Variable-size exchange; with idx (int32) value j of the outgoing message is send[idx[j]] -- the pack of
        the interface values is fused into the sending kernel."""
        if not self.active:
            return None
        if max(max(recv_counts), max(send_counts)) > self.cap:
            if idx is not None:
                packed = torch.empty(idx.numel(), dtype=send.dtype, device=send.device)
                self._D.gather(idx.numel(), idx, send, packed)
                send = packed
            return self.base.all_to_all(recv, send, recv_counts, send_counts, async_op=async_op)
        soff_d, soff = self._offsets(send_counts)
        roff_d, roff = self._offsets(recv_counts)
        self.halo_seq += 1
        seq = self.halo_seq
        call = self._D.call
        call("ddilu_peer_send", self.size, self.rank, soff[-1], send, idx, soff_d, self._data, self._halo_flags,
             self._my_ack, self.cap, seq, self.spin_cycles, self._counters[0:1], self.err)

        def finish():
            call("ddilu_peer_recv", self.size, self.rank, roff[-1], recv, roff_d, self._my_data, self._my_halo_flags,
                 self._ack_flags, send, idx, soff[self.rank], self.cap, seq, self.spin_cycles, self._counters[1:2],
                 self.err)

        if async_op:
            return _PeerWork(finish)
        finish()
        return None

    def barrier(self):
        self.base.barrier()

    def close(self):
        """Drop the mappings of the other ranks' mailboxes (collective; before the process group goes away)."""
        torch.cuda.synchronize()
        self.base.barrier()
        self._peers = [self._mail]
        self.base.barrier()

    @property
    def transport(self) -> str:
        return "peer-memory (CUDA IPC mailboxes, in-kernel flags; csrc/peer.cu)"


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
    comm = Comm(rank, world, None)
    # peer-memory transport (csrc/peer.cu): the default with one GPU per rank; ranks SHARING a GPU (tests) take turns
    # by time slicing, every flag hand-over then costs a time slice, so it must be asked for there (DDILU_PEER=1)
    own_gpu = torch.cuda.is_available() and torch.cuda.device_count() >= world
    if torch.cuda.is_available() and os.environ.get("DDILU_PEER", "1" if own_gpu else "0") == "1":
        comm = peer_or_base(comm)
    return set_comm(comm)


def peer_or_base(base: Comm) -> Comm:
    """PeerComm over `base` when every rank can map every mailbox and a trial reduction comes back right on all
    ranks; otherwise `base` itself (ranks on different nodes, no peer access).  Collective."""
    ok, comm = 1, None
    try:
        comm = PeerComm(base)
        t = torch.full((3,), float(base.rank + 1), dtype=torch.float64, device=comm._dev)
        comm.allreduce_sum_(t)
        want = base.size * (base.size + 1) / 2
        if int(comm.err.item()) or not bool((t == want).all().item()):
            ok = 0
    except Exception:
        ok = 0
    flag = torch.tensor([ok], dtype=torch.int64)
    if tdist.get_backend(base.group) != "gloo":
        flag = flag.cuda()
    tdist.all_reduce(flag, op=tdist.ReduceOp.MIN, group=base.group)
    return comm if int(flag.item()) == 1 else base


def domains_of_rank(p: int, comm: Comm) -> range:
    """Contiguous block of subdomains owned by this rank."""
    if p % comm.size:
        raise ValueError(f"{p} subdomains cannot be dealt evenly to {comm.size} ranks")
    per = p // comm.size
    return range(comm.rank * per, (comm.rank + 1) * per)

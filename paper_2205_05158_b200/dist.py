"""Multi-GPU partitioning of the hot path; torch.distributed plumbing only.

Mode S — OFDM-symbol batches (used by bench.py).  Symbols are independent given the
channel, the CNN weights and the PA coefficients, so each rank owns whole symbols and
the only collective is the int64 SER-counter sum.  Weak scaling: every rank runs a
fixed batch of `per_rank` symbols with global indices rank*per_rank + i.

Mode A — antennas.  Rank r owns antenna rows [b0, b0 + B_loc) of P, h_fd and the PA
coefficients (zf_precoder_build emits only those rows from the replicated taps).  The
FD-CNN is B-independent, so it is sharded by symbol and s_tilde is all-gathered; each
rank then runs chain_txrx on its antennas, forms its partial channel sum with
ue_combine, and the partial received signals are all-reduced (Eqs. 4-5 sum over b)
before slicing.

The arithmetic of every step runs in libfdpd kernels; this module only computes index
ranges and issues collectives (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist
import torch.multiprocessing  # noqa: F401  (registers the tensor reducers PeerExchange pickles with)


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def symbol_range(per_rank: int, rank: int) -> range:
    """Mode S, weak scaling: the global symbol indices rank `rank` processes."""
    return range(rank * per_rank, (rank + 1) * per_rank)


def split(n: int, parts: int, idx: int):
    """Contiguous balanced split of n items: (start, count) of part idx."""
    base, rem = divmod(n, parts)
    start = idx * base + min(idx, rem)
    return start, base + (1 if idx < rem else 0)


def antenna_shard(B: int, world_size: int, rank: int):
    """Mode A: (b0, B_loc) antenna rows owned by `rank`."""
    return split(B, world_size, rank)


def allreduce_counts(counts: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the int64 (errors, total, near) counters over ranks (Mode S and A)."""
    if world()[0] > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def allgather_symbols(local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """Mode A: gather the symbol-sharded s_tilde [n_loc][U][N_d] into [n_total][U][N_d].
    Shards follow split(n_total, world, rank); unequal shards are padded for the collective."""
    ws, rank = world()
    if ws == 1:
        return local
    counts = [split(n_total, ws, r)[1] for r in range(ws)]
    m = max(counts)
    buf = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    if buf.is_complex():
        buf = torch.view_as_real(buf)
    out = [torch.empty_like(buf) for _ in range(ws)]
    dist.all_gather(out, buf, group=group)
    parts = [out[r][: counts[r]] for r in range(ws)]
    full = torch.cat(parts, dim=0)
    return torch.view_as_complex(full.contiguous()) if local.is_complex() else full


def allreduce_partial(partial: torch.Tensor, group=None) -> torch.Tensor:
    """Mode A: sum the per-rank partial received signals y_hat (Eq. 5 sum over antennas)."""
    if world()[0] > 1:
        t = torch.view_as_real(partial) if partial.is_complex() else partial
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return partial


# ============================================================================ Mode A step
def _staged(t: torch.Tensor, host_staged: bool):
    """The tensor a collective runs on: a real view (complex -> [..., 2]); with host staging
    (gloo on CUDA tensors) a CPU copy that the caller copies back."""
    r = torch.view_as_real(t) if t.is_complex() else t
    return r.cpu() if host_staged else r


def all_gather_into(out: torch.Tensor, local: torch.Tensor, group=None, host_staged=False, async_op=False):
    """Mode A: rank blocks of the symbol-sharded s_tilde concatenated in rank order into the
    preallocated out [world * n_loc][U][N_d] (torch.distributed.all_gather_into_tensor)."""
    if world()[0] == 1:
        out.copy_(local)
        return None
    if host_staged:
        o = _staged(out, True)
        dist.all_gather_into_tensor(o, _staged(local, True), group=group)
        out.copy_(torch.view_as_complex(o) if out.is_complex() else o)
        return None
    return dist.all_gather_into_tensor(_staged(out, False), _staged(local, False), group=group, async_op=async_op)


def reduce_scatter_into(mine: torch.Tensor, partial: torch.Tensor, group=None, host_staged=False, async_op=False):
    """Mode A: sum the per-rank partial received signals (Eq. 5's sum over antennas)
    and leave rank r the r-th symbol block (its own symbols) in mine [n_loc][U][N_d]
    (torch.distributed.reduce_scatter_tensor, SUM)."""
    if world()[0] == 1:
        mine.copy_(partial)
        return None
    if host_staged:
        m = _staged(mine, True)
        dist.reduce_scatter_tensor(m, _staged(partial, True), op=dist.ReduceOp.SUM, group=group)
        mine.copy_(torch.view_as_complex(m) if mine.is_complex() else m)
        return None
    return dist.reduce_scatter_tensor(_staged(mine, False), _staged(partial, False), op=dist.ReduceOp.SUM,
                                      group=group, async_op=async_op)


def peer_slot(n: int, nm: int, rank: int):
    """Fused Mode A exchange: where rank `rank`'s partial y_hat of world-batch symbol n goes —
    (owner rank, slot, local symbol) = (n // nm, rank, n % nm) in the owner's receive buffer
    [world][nm][U][N_d] (include/fdpd.h ue_combine_peer)."""
    return n // nm, rank, n % nm


class PeerExchange:
    """Receive buffers of the fused Mode A exchange (ue_combine_peer / ue_reduce_ser), one per
    micro-batch: recv[k] [world][nm][U][N_d] on this rank, and peers[k][r] = rank r's buffer
    mapped into this process with CUDA IPC (r == rank: the local tensor), so the channel-sum
    kernel stores its partial sums straight into their owners' memory over NVLink.  The only
    synchronisation is a stream-ordered barrier between "all ranks stored" and the owner's
    reduction (no kernel waits on another GPU)."""

    def __init__(self, micro, nm, U, N_d, device, group=None, host_staged=False, dtype=torch.complex64):
        ws, rank = world()
        self.ws, self.rank, self.group, self.host_staged = ws, rank, group, host_staged
        self.recv = [torch.zeros((ws, nm, U, N_d), dtype=dtype, device=device) for _ in range(micro)]
        self.peers = [[t] for t in self.recv]
        cpu = torch.device(device).type == "cpu"      # CPU tests: shared-memory tensors stand in for IPC
        if ws > 1 and cpu:
            for t in self.recv:
                t.share_memory_()
        if ws > 1:
            # torch's multiprocessing reducers turn a tensor into an IPC handle (CUDA) or a shared-
            # memory file name (CPU) instead of a copy; the blobs travel through the process group.
            # Every failure below is agreed on by all ranks (_agree) before anyone raises, so the
            # ranks either all use the exchange or all fall back — never a mix that would deadlock.
            import pickle
            from multiprocessing.reduction import ForkingPickler
            self._flag = torch.zeros(1, dtype=torch.int32, device=device)
            every = [None] * ws
            dist.all_gather_object(every, bytes(ForkingPickler.dumps(self.recv)), group=group)
            err = None
            try:
                self.peers = [[None] * ws for _ in range(micro)]
                for r in range(ws):
                    theirs = self.recv if r == rank else pickle.loads(every[r])   # opens rank r's allocations here
                    for k in range(micro):
                        t = theirs[k]
                        if not cpu and t.device != torch.device(device) and not torch.cuda.can_device_access_peer(
                                torch.device(device).index, t.device.index):
                            raise RuntimeError(f"no peer access from {device} to {t.device}")
                        self.peers[k][r] = t
                # first touch through the runtime enables peer access between the two devices
                for row in self.peers:
                    for t in row:
                        if t.device != torch.device(device):
                            t[0, 0, 0, :1].to(device)
            except Exception as e:                         # noqa: BLE001 (reported after the agreement)
                err = e
            if not self._agree(err is None):
                raise RuntimeError(f"peer exchange: mapping the receive buffers failed on some rank ({err})")
            self._validate()

    def _agree(self, ok: bool) -> bool:
        """True iff `ok` on every rank (all-reduce MIN over the group)."""
        dev = "cpu" if self.host_staged else self._flag.device
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return bool(int(t.item()))

    def _validate(self):
        """Every rank writes a token into its slot of every buffer; after the barrier each rank
        must see all of them in its own buffers (a mapping that does not reach the owner's memory
        is caught here, before any result depends on it; all ranks raise together).  Leaves the
        buffers zeroed."""
        for k, row in enumerate(self.peers):
            for t in row:
                t[self.rank, 0, 0, 0] = float(self.rank + 1 + 16 * k)
        self.barrier()
        bad = None
        for k, t in enumerate(self.recv):
            got = t[:, 0, 0, 0].real.cpu().tolist()
            want = [float(r + 1 + 16 * k) for r in range(self.ws)]
            if got != want:
                bad = f"rank {self.rank} buffer {k} holds {got}, expected {want}"
        self.barrier()
        for t in self.recv:
            t.zero_()
        self.barrier()
        if not self._agree(bad is None):
            raise RuntimeError(f"peer exchange: stores did not reach their owners on some rank ({bad})")

    def barrier(self):
        """Every rank's stores into this rank's buffers are complete (and vice versa)."""
        if self.ws == 1:
            return
        if self.host_staged:
            if torch.cuda.is_available():
                torch.cuda.synchronize()
            dist.barrier(group=self.group)
        else:
            dist.all_reduce(self._flag, group=self.group)          # stream-ordered on NCCL


class AntennaShardedStep:
    """Mode A (BASELINE configs[4] "sharded by antenna ... allreduce of per-UE
    received subcarrier signals"), one step over a batch of world x n_per_rank symbols:

      1. FD-CNN on this rank's n_per_rank symbols (the CNN does not depend on the antennas);
      2. all_gather_into_tensor of s_tilde -> every rank holds the whole batch;
      3. precode -> IDFT -> GMP -> receive DFT on this rank's antenna rows [b0, b0 + B_loc);
      4. partial channel sum over the local antennas (ue_combine);
      5. reduce_scatter_tensor (SUM) of the partial received signals: rank r gets the full
         y_hat of its own symbols (the sum over antennas of Eq. 5, split by symbol blocks);
      6. slicing + SER counters on the rank's symbols, int64 counters all-reduced.
    With `peer` (a PeerExchange) steps 4-5 are one kernel: ue_combine_peer stores every partial
    sum into slot `rank` of its owner's receive buffer over peer memory while it computes; after
    a stream-ordered barrier the owner sums the slots in rank order and slices (ue_reduce_ser).

    The batch is cut into `micro` micro-batches: with NCCL the collectives of micro-batch k are
    issued asynchronously and waited on just before their consumer, so the all-gather of k
    overlaps the FD-CNN of k + 1 and the reduce-scatter of k the chain of k + 1.

    `ops` supplies the per-rank compute (the CUDA kernels on GPUs; the fp64 oracle in the CPU
    gloo tests): dpd(s, out), tx(st_all, XPA_out), combine(XPA, out), slice(yhat, idx, counts).
    `alloc(shape)` allocates a complex buffer on the compute device.  host_staged: gloo on CUDA
    tensors (collectives through host copies; used by the single-GPU 2-rank validation)."""

    def __init__(self, ops, n_per_rank, U, N_d, alloc, micro=2, group=None, host_staged=False, peer=None):
        self.ops, self.group, self.host_staged = ops, group, host_staged
        self.peer = peer              # PeerExchange: steps 4-5 fused (partial sums stored at their owners)
        ws, _ = world()
        self.ws = ws
        self.micro = micro if (micro > 1 and n_per_rank % micro == 0) else 1
        self.nm = n_per_rank // self.micro
        self.n = n_per_rank
        self.st = [alloc((self.nm, U, N_d)) for _ in range(self.micro)]
        self.st_all = [alloc((ws * self.nm, U, N_d)) for _ in range(self.micro)]
        self.xpa = [None] * self.micro
        self.part = [alloc((ws * self.nm, U, N_d)) for _ in range(self.micro)]
        self.mine = [alloc((self.nm, U, N_d)) for _ in range(self.micro)]
        self.alloc = alloc

    def step(self, s, idx, counts):
        """s, idx: this rank's n_per_rank symbols; counts (int64[3]) receives the all-reduced
        errors / total / near-boundary of the whole world batch.  Returns the list of the
        micro-batches' y_hat (this rank's symbols)."""
        nm, M = self.nm, self.micro
        asy = not self.host_staged and self.ws > 1
        ag = [None] * M
        for k in range(M):                                   # CNN + async all-gather
            self.ops.dpd(s[k * nm:(k + 1) * nm], self.st[k])
            ag[k] = all_gather_into(self.st_all[k], self.st[k], self.group, self.host_staged, async_op=asy)
        rs = [None] * M
        for k in range(M):                                   # local antennas + async reduce-scatter
            if ag[k] is not None:
                ag[k].wait()
            self.xpa[k] = self.ops.tx(self.st_all[k], self.xpa[k])
            if self.peer is not None:                        # partial sums straight into the owners' buffers
                self.ops.combine_peer(self.xpa[k], self.peer.peers[k], self.peer.rank)
                continue
            self.ops.combine(self.xpa[k], self.part[k])
            rs[k] = reduce_scatter_into(self.mine[k], self.part[k], self.group, self.host_staged, async_op=asy)
        if self.peer is not None:
            self.peer.barrier()
        for k in range(M):                                   # slicing on this rank's symbols
            if self.peer is not None:                        # sum of the ranks' slots in rank order, then slicing
                self.ops.reduce_slice(self.peer.recv[k], self.mine[k], idx[k * nm:(k + 1) * nm], counts)
                continue
            if rs[k] is not None:
                rs[k].wait()
            self.ops.slice(self.mine[k], idx[k * nm:(k + 1) * nm], counts)
        if self.ws > 1:
            if self.host_staged:
                c = counts.cpu()
                dist.all_reduce(c, op=dist.ReduceOp.SUM, group=self.group)
                counts.copy_(c)
            else:
                dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=self.group)
        return self.mine

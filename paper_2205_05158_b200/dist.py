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

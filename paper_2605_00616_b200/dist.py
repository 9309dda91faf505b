"""Multi-GPU plumbing: one process per GPU, torch.distributed (NCCL) underneath.

* Queries shard naturally: each rank owns a contiguous range
  of the query stream (or whole scenarios) -- no collective in the query loop.
* The immutable profile table is replicated once: ``broadcast_tables`` sends
  the three canonical tables' SoA from ``src`` with one NCCL broadcast per
  array over NVLink.
* The offline build range-partitions records on tt (``partition_by_tt`` picks
  splitters from an all-reduced tt histogram, ``exchange_records`` moves each
  record to its owner with one all_to_all); each rank builds its tt slice and
  ``gather_tables`` concatenates the slices in rank order, which is already
  the global (tt, conc) order because the slices are disjoint tt ranges.

The collective helpers take plain tensors so the host logic is exercised on
CPU with the gloo backend (tests/test_dist.py); the CUDA path passes CUDA
tensors and NCCL.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .profile import TableSoA

_FIELDS = (("tt", torch.int32), ("conc", torch.int32), ("off", torch.int64), ("samples", torch.float64))


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_range(n: int, rank: int, size: int) -> tuple[int, int]:
    """Contiguous [lo, hi) of n items owned by `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n, size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def broadcast_arrays(arrays: list[torch.Tensor] | None, dtypes: list[torch.dtype], src: int = 0,
                     device: str | torch.device = "cuda") -> list[torch.Tensor]:
    """Broadcast a list of 1-D tensors from `src` (receivers pass None)."""
    rank, _ = world()
    sizes = torch.zeros(len(dtypes), dtype=torch.int64, device=device)
    if rank == src:
        sizes = torch.tensor([a.numel() for a in arrays], dtype=torch.int64, device=device)
    dist.broadcast(sizes, src)
    out = []
    for i, dt in enumerate(dtypes):
        if rank == src:
            t = arrays[i].to(device=device, dtype=dt).contiguous()
        else:
            t = torch.empty(int(sizes[i].item()), dtype=dt, device=device)
        if t.numel():
            dist.broadcast(t, src)
        out.append(t)
    return out


def broadcast_soas(soas: list[TableSoA] | None, src: int = 0, device="cuda") -> list[list[torch.Tensor]]:
    """The three tables' SoA as tensors on every rank."""
    rank, _ = world()
    flat = None
    if rank == src:
        flat = [torch.as_tensor(np.ascontiguousarray(getattr(s, f))) for s in soas for f, _ in _FIELDS]
    got = broadcast_arrays(flat, [dt for _ in range(3) for _, dt in _FIELDS], src, device)
    return [got[4 * i:4 * i + 4] for i in range(3)]


def broadcast_tables(tables, src: int = 0):
    """Replicate a DeviceTables handle from `src` to every rank (NCCL over NVLink)."""
    from .device import DeviceTables

    rank, size = world()
    if size == 1:
        return tables
    if rank == src:
        arrs = [tables.device_arrays(i) for i in range(3)]
        flat = [a[k] for a in arrs for k in ("bkt_tt", "bkt_conc", "bkt_off", "samples")]
    else:
        flat = None
    got = broadcast_arrays(flat, [dt for _ in range(3) for _, dt in _FIELDS], src, "cuda")
    if rank == src:
        return tables
    torch.cuda.synchronize()
    return DeviceTables.from_device(got)


# ------------------------------------------------------------ range-partitioned build
def partition_by_tt(tt_local: torch.Tensor, size: int, tt_max: int | None = None) -> torch.Tensor:
    """Splitters s[0..size] over tt so each rank owns ~the same number of
    records: all-reduce a tt histogram, cut its cumulative sum at k/size."""
    t = tt_local.to(torch.int64)
    hi = int(t.max().item()) if t.numel() else 1
    if tt_max is None:
        m = torch.tensor([hi], dtype=torch.int64, device=t.device)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        tt_max = int(m.item())
    hist = torch.bincount(t, minlength=tt_max + 1)[: tt_max + 1].to(torch.int64)
    dist.all_reduce(hist)
    cum = torch.cumsum(hist, 0)
    total = int(cum[-1].item())
    cuts = [0]
    for k in range(1, size):
        cuts.append(int(torch.searchsorted(cum, torch.tensor(total * k // size, device=cum.device),
                                           right=True).item()))
    cuts.append(tt_max + 1)
    cuts = np.maximum.accumulate(np.array(cuts))
    return torch.tensor(cuts, dtype=torch.int64)


def exchange_records(cols: list[torch.Tensor], tt: torch.Tensor, splitters: torch.Tensor) -> list[torch.Tensor]:
    """Send each record to the rank owning its tt range (one all_to_all per column).
    Stable: records keep their relative order per source rank, and sources are
    concatenated in rank order, so per-key capture order follows (rank, index)."""
    rank, size = world()
    owner = torch.bucketize(tt.to(torch.int64), splitters[1:-1].to(tt.device), right=True)
    order = torch.sort(owner, stable=True).indices
    send_counts = torch.bincount(owner, minlength=size).to(torch.int64)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts)
    sc, rc = send_counts.tolist(), recv_counts.tolist()
    out = []
    for c in cols:
        src = c[order].contiguous()
        dst = torch.empty(sum(rc), dtype=c.dtype, device=c.device)
        dist.all_to_all_single(dst, src, output_split_sizes=rc, input_split_sizes=sc)
        out.append(dst)
    return out


def gather_soas(local: list[TableSoA]) -> list[TableSoA]:
    """Concatenate per-rank tt-slices of the three tables in rank order
    (all_gather of sizes, then of each array); offsets are rebased."""
    rank, size = world()
    res = []
    for s in local:
        parts = {}
        for f, dt in _FIELDS:
            a = torch.as_tensor(np.ascontiguousarray(getattr(s, f) if f != "off" else getattr(s, f)[:-1]))
            n = torch.tensor([a.numel()], dtype=torch.int64)
            ns = [torch.zeros(1, dtype=torch.int64) for _ in range(size)]
            dist.all_gather(ns, n)
            mx = max(int(x.item()) for x in ns)
            pad = torch.zeros(mx, dtype=dt)
            pad[: a.numel()] = a.to(dt)
            bufs = [torch.zeros(mx, dtype=dt) for _ in range(size)]
            dist.all_gather(bufs, pad)
            parts[f] = [b[: int(k.item())] for b, k in zip(bufs, ns)]
        counts = [int(p.numel()) for p in parts["samples"]]
        base = np.concatenate([[0], np.cumsum(counts)])
        off = [parts["off"][r].numpy().astype(np.int64) + base[r] for r in range(size)]
        res.append(TableSoA(torch.cat(parts["tt"]).numpy().astype(np.int32),
                            torch.cat(parts["conc"]).numpy().astype(np.int32),
                            np.concatenate(off + [np.array([base[-1]], np.int64)]),
                            torch.cat(parts["samples"]).numpy()))
    return res


def all_reduce_max(x: float, device="cuda") -> float:
    rank, size = world()
    if size == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

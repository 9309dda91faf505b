"""Multi-GPU plumbing: one process per GPU, torch.distributed (NCCL) underneath.

* Queries shard naturally: each rank owns a contiguous range
  of the query stream (or whole scenarios) -- no collective in the query loop.
* The immutable profile table is replicated once: ``broadcast_tables`` packs
  the three canonical tables' SoA into one buffer and sends it from ``src``
  with one NCCL broadcast over NVLink (after a 96-byte size header).
* The offline build range-partitions records on tt (``partition_by_tt`` picks
  splitters from an all-reduced tt histogram, ``exchange_records`` moves each
  record to its owner with one all_to_all per column); each rank builds its tt
  slice and ``all_gather_tables`` re-replicates the slices (one all_gather of
  the packed payloads) in rank order, which is already the global (tt, conc)
  order because the slices are disjoint tt ranges.

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


def pack_arrays(arrays: list[torch.Tensor]) -> tuple[torch.Tensor, torch.Tensor]:
    """(header, payload): element counts int64[n] and one uint8 buffer holding
    every array's bytes, each padded to 8 B (so every slice views back aligned)."""
    dev = arrays[0].device if arrays else torch.device("cpu")
    header = torch.tensor([a.numel() for a in arrays], dtype=torch.int64, device=dev)
    parts = []
    for a in arrays:
        if a.numel() == 0:
            continue
        raw = a.contiguous().reshape(-1).view(torch.uint8)
        parts.append(raw)
        if raw.numel() % 8:
            parts.append(torch.zeros(8 - raw.numel() % 8, dtype=torch.uint8, device=dev))
    payload = torch.cat(parts) if parts else torch.zeros(0, dtype=torch.uint8, device=dev)
    return header, payload


def _payload_bytes(counts, dtypes) -> int:
    return sum((int(n) * torch.empty(0, dtype=dt).element_size() + 7) // 8 * 8 for n, dt in zip(counts, dtypes))


def unpack_arrays(counts, payload: torch.Tensor, dtypes) -> list[torch.Tensor]:
    """Inverse of pack_arrays: zero-copy typed views into `payload`."""
    out, o = [], 0
    for n, dt in zip(counts, dtypes):
        nb = int(n) * torch.empty(0, dtype=dt).element_size()
        out.append(payload[o:o + nb].view(dt) if nb else torch.empty(0, dtype=dt, device=payload.device))
        o += (nb + 7) // 8 * 8
    return out


def broadcast_arrays(arrays: list[torch.Tensor] | None, dtypes: list[torch.dtype], src: int = 0,
                     device: str | torch.device = "cuda") -> list[torch.Tensor]:
    """Broadcast a list of 1-D tensors from `src` (receivers pass None): one
    broadcast of the element counts, then ONE broadcast of the packed payload."""
    rank, _ = world()
    header = torch.zeros(len(dtypes), dtype=torch.int64, device=device)
    payload = None
    if rank == src:
        header, payload = pack_arrays([a.to(device=device, dtype=dt) for a, dt in zip(arrays, dtypes)])
    dist.broadcast(header, src)
    counts = header.tolist()
    if rank != src:
        payload = torch.empty(_payload_bytes(counts, dtypes), dtype=torch.uint8, device=device)
    if payload.numel():
        dist.broadcast(payload, src)
    return unpack_arrays(counts, payload, dtypes)


def broadcast_soas(soas: list[TableSoA] | None, src: int = 0, device="cuda") -> list[list[torch.Tensor]]:
    """The three tables' SoA as tensors on every rank."""
    rank, _ = world()
    flat = None
    if rank == src:
        flat = [torch.as_tensor(np.ascontiguousarray(getattr(s, f))) for s in soas for f, _ in _FIELDS]
    got = broadcast_arrays(flat, [dt for _ in range(3) for _, dt in _FIELDS], src, device)
    return [got[4 * i:4 * i + 4] for i in range(3)]


TABLE_DTYPES = [dt for _ in range(3) for _, dt in _FIELDS]


def table_arrays(tables) -> list[torch.Tensor]:
    """The 12 device arrays [tt, conc, off, samples] x (decode, mixed, combined) of a DeviceTables."""
    arrs = [tables.device_arrays(i) for i in range(3)]
    return [a[k] for a in arrs for k in ("bkt_tt", "bkt_conc", "bkt_off", "samples")]


def broadcast_tables(tables, src: int = 0):
    """Replicate a DeviceTables handle from `src` to every rank: the 12 arrays
    travel as one packed payload (one NCCL broadcast over NVLink, after a
    96-byte size header); receivers rebuild their search indexes locally."""
    from .device import DeviceTables

    rank, size = world()
    if size == 1:
        return tables
    got = broadcast_arrays(table_arrays(tables) if rank == src else None, TABLE_DTYPES, src, "cuda")
    if rank == src:
        return tables
    torch.cuda.current_stream().synchronize()
    return DeviceTables.from_device(got)


def all_gather_tables(local: list[torch.Tensor]) -> list[torch.Tensor]:
    """Re-replicate a range-partitioned build: every rank
    holds the 12 arrays of its tt slice; one all_gather of the size headers and
    one all_gather of the packed payloads give every rank all slices, which are
    concatenated in rank order (already the global (tt, conc) order: the slices
    are disjoint, ascending tt ranges) with bucket offsets rebased.  Works on
    CUDA tensors (NCCL) and CPU tensors (gloo)."""
    rank, size = world()
    dev = local[0].device
    header, payload = pack_arrays([a.to(dtype=dt) for a, dt in zip(local, TABLE_DTYPES)])
    headers = torch.empty(size * len(TABLE_DTYPES), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(headers, header)
    counts = headers.view(size, len(TABLE_DTYPES)).tolist()
    nbytes = [_payload_bytes(c, TABLE_DTYPES) for c in counts]
    mx = max(nbytes)
    buf = torch.zeros(mx, dtype=torch.uint8, device=dev)
    buf[: payload.numel()] = payload
    allbuf = torch.empty(size * mx, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(allbuf, buf)
    per_rank = [unpack_arrays(counts[r], allbuf[r * mx:(r + 1) * mx], TABLE_DTYPES) for r in range(size)]
    out = []
    for t in range(3):
        tt = torch.cat([p[4 * t] for p in per_rank])
        conc = torch.cat([p[4 * t + 1] for p in per_rank])
        smp = torch.cat([p[4 * t + 3] for p in per_rank])
        offs, base = [], 0
        for p in per_rank:
            o = p[4 * t + 2]
            offs.append(o[:-1] + base if o.numel() else o)
            base += p[4 * t + 3].numel()
        offs.append(torch.tensor([base], dtype=torch.int64, device=dev))
        out += [tt, conc, torch.cat(offs), smp]
    return out


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
    targets = (cum[-1] * torch.arange(1, size, device=cum.device)) // size
    inner = torch.searchsorted(cum, targets, right=True).tolist()  # one device->host read
    cuts = np.maximum.accumulate(np.array([0] + inner + [tt_max + 1]))
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


def gather_soas(local: list[TableSoA], device=None) -> list[TableSoA]:
    """Host-SoA wrapper of all_gather_tables (CPU tensors under gloo, CUDA under NCCL)."""
    if device is None:
        device = "cuda" if dist.get_backend() == "nccl" else "cpu"
    flat = [torch.as_tensor(np.ascontiguousarray(getattr(s, f))).to(device) for s in local for f, _ in _FIELDS]
    got = all_gather_tables(flat)
    return [TableSoA(got[4 * i].cpu().numpy().astype(np.int32), got[4 * i + 1].cpu().numpy().astype(np.int32),
                     got[4 * i + 2].cpu().numpy().astype(np.int64), got[4 * i + 3].cpu().numpy())
            for i in range(3)]


def all_reduce_max(x: float, device="cuda") -> float:
    rank, size = world()
    if size == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

"""Multi-GPU host logic on CPU: gloo, world size 2 (the CUDA path uses NCCL).

The per-rank table build here is the CPU oracle (tests may use it as the
builder stand-in); the product path plugs in emu_tables_build.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_00616_b200.dist import (
    broadcast_soas,
    exchange_records,
    gather_soas,
    partition_by_tt,
    shard_range,
)
from paper_2605_00616_b200.profile import TableSoA

WORLD = 2


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)


def _range_partitioned_build(rank, port, q):
    try:
        _init(rank, port)
        import emu_oracle as O
        from paper_2605_00616_b200.workloads import records_llama

        tt, conc, ph, lat = records_llama(40_000, 0)
        lo, hi = shard_range(len(tt), rank, WORLD)  # each rank starts with an arbitrary slice of records
        cols = [torch.as_tensor(a[lo:hi]) for a in (tt, conc, ph, lat)]
        split = partition_by_tt(cols[0], WORLD)
        mine = exchange_records(cols, cols[0], split)
        ltt = mine[0].numpy()
        # every record landed on the rank owning its tt range
        assert ((ltt >= int(split[rank])) & (ltt < int(split[rank + 1]))).all()
        local = O.build(*[m.numpy() for m in mine], canonical=True)
        soas = [TableSoA(t.tt, t.conc, t.off, t.samples) for t in local]
        merged = gather_soas(soas)
        want = O.build(tt, conc, ph, lat, canonical=True)
        for g, w in zip(merged, want):
            assert np.array_equal(g.tt, w.tt) and np.array_equal(g.conc, w.conc)
            assert np.array_equal(g.off, w.off) and np.array_equal(g.samples, w.samples)
        # replicate rank 0's tables with one broadcast per array
        got = broadcast_soas(merged if rank == 0 else None, src=0, device="cpu")
        for g, w in zip(got, want):
            assert np.array_equal(g[3].numpy(), w.samples) and np.array_equal(g[2].numpy(), w.off)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _query_shards(rank, port, q):
    try:
        _init(rank, port)
        import emu_oracle as O
        from paper_2605_00616_b200.workloads import queries_llama, records_llama

        tabs = O.build(*records_llama(20_000, 0), canonical=True)
        qt, qc, qp = queries_llama(10_001, 3)
        lo, hi = shard_range(len(qt), rank, WORLD)
        # Philox counters are absolute query indices: shards reproduce the
        # single-process stream exactly (no collective in the query loop)
        _, s = O.sample_batch(tabs, qt[lo:hi], qc[lo:hi], qp[lo:hi], 32, mode="philox", seed=5, ctr_base=lo)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(WORLD)]
        dist.all_gather(sizes, torch.tensor([hi - lo]))
        mx = int(max(x.item() for x in sizes))
        buf = torch.full((mx,), -1, dtype=torch.int32)
        buf[: hi - lo] = torch.as_tensor(s)
        parts = [torch.zeros(mx, dtype=torch.int32) for _ in range(WORLD)]
        dist.all_gather(parts, buf)
        allq = np.concatenate([p[: int(n.item())].numpy() for p, n in zip(parts, sizes)])
        _, want = O.sample_batch(tabs, qt, qc, qp, 32, mode="philox", seed=5)
        assert np.array_equal(allq, want)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _run(fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=fn, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(WORLD)}, res


def test_shard_range_covers_everything():
    for n in (0, 1, 7, 100, 101):
        for size in (1, 2, 3, 8):
            spans = [shard_range(n, r, size) for r in range(size)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_range_partitioned_build_gloo():
    _run(_range_partitioned_build)


def test_query_shards_reproduce_single_stream_gloo():
    _run(_query_shards)


def test_pack_unpack_round_trip():
    from paper_2605_00616_b200.dist import TABLE_DTYPES, pack_arrays, unpack_arrays

    rng = np.random.default_rng(0)
    arrs = []
    for dt in TABLE_DTYPES:
        n = int(rng.integers(0, 9))
        arrs.append(torch.as_tensor(rng.integers(-5, 5, n)).to(dt))
    header, payload = pack_arrays(arrs)
    assert payload.numel() % 8 == 0
    got = unpack_arrays(header.tolist(), payload, TABLE_DTYPES)
    for g, a in zip(got, arrs):
        assert g.dtype == a.dtype and torch.equal(g, a)


def test_bench_launcher_spawns_ranks():
    """`python bench.py --gpus 2` re-execs itself under torch.distributed.run
    (2 ranks, 127.0.0.1 rendezvous); --dry-run keeps it on CPU over gloo."""
    import json
    import subprocess
    import sys

    from conftest import ROOT

    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2",
                        "--warmup", "1", "--records", "20000", "--queries", "50000"], capture_output=True, text=True,
                       timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["dry_run"] and line["buckets"][2] > 0

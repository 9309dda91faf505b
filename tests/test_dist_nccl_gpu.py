"""The multi-GPU collectives on the CUDA path: NCCL with CUDA tensors (B200 only).

Only one GPU is available here, so the process group has one rank; the
collectives still run through NCCL on device buffers: the packed table
broadcast (one header + one payload broadcast), the all_gather that
re-replicates a range-partitioned build, and the tt range partition with its
all_to_all record exchange.  The tables that come out must equal the ones that
went in, and an oracle over them must draw exactly what the original draws.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2605_00616_b200 import LatencyOracle, OracleConfig
from paper_2605_00616_b200.device import DeviceTables
from paper_2605_00616_b200.dist import (
    TABLE_DTYPES,
    all_gather_tables,
    broadcast_arrays,
    exchange_records,
    partition_by_tt,
    table_arrays,
)
from paper_2605_00616_b200.profile import pack_from_device
from paper_2605_00616_b200.workloads import explicit_uniforms, queries_llama, records_llama

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def _draws(tables, Q=200_000):
    orc = LatencyOracle(pack_from_device(tables, 1000, keep_host=False), OracleConfig(reliability_floor=32),
                        _validate=False)
    qt, qc, qp = (torch.as_tensor(a, device="cuda") for a in queries_llama(Q, 3))
    us, ui = explicit_uniforms(Q, 4)
    lat, sidx = orc.sample_batch(qt, qc, qp, rng="explicit", u_sel=torch.as_tensor(us.view(np.int64), device="cuda"),
                                 u_idx=torch.as_tensor(ui.view(np.int32), device="cuda"))
    return lat.cpu().numpy(), sidx.cpu().numpy()


def test_packed_broadcast_and_all_gather_over_nccl(nccl):
    tables = DeviceTables.build(*records_llama(300_000, 0), canonical=True)
    src = table_arrays(tables)
    got = broadcast_arrays(src, TABLE_DTYPES, 0, "cuda")  # one header + one payload broadcast
    for a, b in zip(src, got):
        assert a.is_cuda and b.is_cuda and torch.equal(a, b)
    gathered = all_gather_tables(src)  # one header + one payload all_gather
    for a, b in zip(src, gathered):
        assert torch.equal(a, b)
    rebuilt = DeviceTables.from_device(gathered)
    want = _draws(tables)
    have = _draws(rebuilt)
    assert np.array_equal(want[1], have[1]) and np.array_equal(want[0], have[0])


def test_range_partition_exchange_over_nccl(nccl):
    rec = records_llama(200_000, 1)
    cols = [torch.as_tensor(a, device="cuda") for a in rec]
    split = partition_by_tt(cols[0], 1)
    mine = exchange_records(cols, cols[0], split)
    assert all(m.is_cuda for m in mine)
    got = DeviceTables.build(*mine, canonical=True).to_host()
    want = DeviceTables.build(*rec, canonical=True).to_host()
    for g, w in zip(got, want):  # canonical order: the exchange's record order does not matter
        assert np.array_equal(g.tt, w.tt) and np.array_equal(g.off, w.off) and np.array_equal(g.samples, w.samples)

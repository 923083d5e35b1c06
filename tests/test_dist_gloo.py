"""N>1 host-side path on CPU (gloo, world_size 2): row sharding, shard
invariance of the seeded inputs and of the packed codes, and the
max-over-ranks aggregation bench.py uses.  The data path has no collective;
the only collectives are the timing/byte gathers exercised here."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_rows_partition():
    for R in (1, 7, 394, 32768):
        for world in (1, 2, 4, 8):
            spans = [bench.shard_rows(R, world, r, "strong") for r in range(world)]
            assert spans[0][0] == 0
            assert sum(n for _, n in spans) == R
            for (a, n), (b, _) in zip(spans, spans[1:]):
                assert a + n == b
            weak = [bench.shard_rows(R, world, r, "weak") for r in range(world)]
            assert all(n == R and s == r * R for r, (s, n) in enumerate(weak))


def test_aggregate_uses_slowest_rank():
    assert bench.aggregate([1e9, 1e9], [1000.0, 500.0], 1) == pytest.approx(2.0)


def _worker(rank, world, port, R, F, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    row0, rows = bench.shard_rows(R, world, rank, "strong")
    x = synth.act_input(rows, F, "bf16", row_start=row0, mode="coverage")
    _, codes = oracle.act_fwd("silu", oracle.decode(synth.to_numpy_storage(x), "bf16"))
    c = torch.from_numpy(codes)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([c.numel()]))
    m = max(int(s) for s in sizes)                  # all_gather needs equal sizes: pad
    padded = torch.zeros(m, dtype=torch.uint8)
    padded[:c.numel()] = c
    gathered = [torch.zeros(m, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(gathered, padded)
    parts = [g[:int(s)] for g, s in zip(gathered, sizes)]
    t = torch.tensor([float(10 + rank), float(rows * F)], dtype=torch.float64)
    tl = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(tl, t)
    if rank == 0:
        q.put((torch.cat(parts).numpy(), [float(v[0]) for v in tl], [float(v[1]) for v in tl]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("R", [512, 37])
def test_sharded_codes_equal_single_process(R):
    F = 3072
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, R, F, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, ms, nbytes = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x = synth.act_input(R, F, "bf16", mode="coverage")
    _, full = oracle.act_fwd("silu", oracle.decode(synth.to_numpy_storage(x), "bf16"))
    assert np.array_equal(got, full)
    assert ms == [10.0, 11.0] and sum(nbytes) == R * F
    assert bench.aggregate(nbytes, ms, 1) == pytest.approx(R * F / 0.011 / 1e9)

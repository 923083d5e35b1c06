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


def test_self_launch_command_runs_n_ranks(tmp_path):
    """bench.py --gpus N without WORLD_SIZE re-execs itself under
    torch.distributed.run (bench.launch_cmd); the command must bring up N
    ranks that rendezvous on 127.0.0.1 and see WORLD_SIZE = N."""
    import json
    import subprocess
    import sys
    script = tmp_path / "probe.py"
    script.write_text(
        "import json, os, torch.distributed as dist\n"
        "dist.init_process_group('gloo')\n"
        "r, w = dist.get_rank(), dist.get_world_size()\n"
        "out = [None] * w\n"
        "dist.all_gather_object(out, (r, int(os.environ['LOCAL_RANK'])))\n"
        "if r == 0:\n"
        "    print(json.dumps({'world': w, 'ranks': out, 'argv': __import__('sys').argv[1:]}))\n"
        "dist.destroy_process_group()\n")
    argv = ["--gpus", "2", "--steps", "3"]
    cmd = bench.launch_cmd(2, argv, _free_port(), script=str(script))
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["world"] == 2 and sorted(line["ranks"]) == [[0, 0], [1, 1]] and line["argv"] == argv


def test_strong_summary():
    s = bench.strong_summary([2e9, 2e9], [10.0, 12.5], 10, t1_ms=2.0)
    assert s["n_ranks"] == 2 and s["ms_per_step"] == 1.25
    assert s["GB/s"] == pytest.approx(4e9 * 10 / 0.0125 / 1e9, rel=1e-4)
    assert s["t1_over_N_tN"] == pytest.approx(2.0 / (2 * 1.25), abs=1e-4)
    assert s["rank_spread"] == pytest.approx(0.25)
    # C5's 32768 rows split evenly for N = 1, 2, 4, 8 and F % 4 == 0, so shard codes concatenate
    c5 = synth.CONFIGS["c5"]
    for n in (1, 2, 4, 8):
        assert all(bench.shard_rows(c5["R"], n, r, "strong")[1] == c5["R"] // n for r in range(n))
    assert c5["F"] % 4 == 0

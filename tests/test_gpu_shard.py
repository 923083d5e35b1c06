"""SURVEY 8(e) / T3 on the CUDA path: row-sharded execution is bitwise
shard-invariant.

Two ranks (gloo process group, both on cuda:0 -- the test box has one GPU)
each run msrms_fwd -> resilu2_fwd -> resilu2_bwd -> msrms_bwd through the C ABI
on their contiguous row block of a C5-width input (F = 13824, H = 5120,
bf16), exactly as bench.py's strong-scaling key partitions C5.  Rank 0
gathers the shards over the process group and checks that the concatenation
of y, codes, dx, yn, rstd and dxn is byte-identical to one process running all
rows, and that the codes equal the float64 oracle's.  The row partition is
bench.shard_rows; the inputs are synth's slice-invariant generators."""
import os
import socket
import traceback

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import synth

pytestmark = pytest.mark.gpu

F, H, DT = 13824, 5120, "bf16"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_rows(row0, R, dev):
    """The four 8(a) launches on rows [row0, row0 + R); CPU copies of all outputs."""
    import paper_2406_16282_b200 as P
    x = synth.act_input(R, F, DT, row_start=row0, mode="coverage").to(dev)
    dy = synth.grad_input(R, F, DT, row_start=row0).to(dev)
    xn = synth.norm_input(R, H, DT, row_start=row0).to(dev)
    gn = synth.grad_input(R, H, DT, row_start=row0, stream=synth.S_NORM_DY).to(dev)
    yn, rstd = P.msrms_fwd(xn, 1e-6)
    y, codes = P.resilu2_fwd(x)
    dx = P.resilu2_bwd(dy, codes)
    dxn = P.msrms_bwd(gn, yn, rstd)
    torch.cuda.synchronize(dev)
    return {"y": y.cpu(), "codes": codes.cpu(), "dx": dx.cpu(), "yn": yn.cpu(), "rstd": rstd.cpu(),
            "dxn": dxn.cpu()}


def _as_bytes(t):
    return t.contiguous().view(torch.uint8).numpy().tobytes()


def _worker(rank, world, port, R, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        row0, rows = bench.shard_rows(R, world, rank, "strong")
        mine = run_rows(row0, rows, dev)
        gathered = [None] * world
        dist.all_gather_object(gathered, (row0, rows, mine))
        if rank == 0:
            gathered.sort(key=lambda g: g[0])
            assert [g[0] for g in gathered] == [bench.shard_rows(R, world, r, "strong")[0] for r in range(world)]
            full = run_rows(0, R, dev)
            for k in full:
                cat = torch.cat([g[2][k] for g in gathered])
                assert _as_bytes(cat) == _as_bytes(full[k]), f"{k}: sharded != single-process"
            q.put(("ok", _as_bytes(full["codes"]), [g[1] for g in gathered]))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        q.put(("error", traceback.format_exc(), None))
        raise


@pytest.mark.parametrize("R", [1024, 1001])
def test_row_sharded_cuda_path_is_bitwise_shard_invariant(R):
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, R, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, payload, sizes = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
    assert status == "ok", payload
    assert all(p.exitcode == 0 for p in procs)
    assert sum(sizes) == R and len(sizes) == world
    # the codes of the whole batch equal the oracle's (bit-exact 2-bit codes)
    x = synth.act_input(R, F, DT, mode="coverage")
    _, c_ref = oracle.act_fwd("silu", oracle.decode(synth.to_numpy_storage(x), DT))
    got = np.frombuffer(payload, dtype=np.uint8)
    assert np.array_equal(got, c_ref)
    counts = np.bincount(((c_ref[:, None] >> np.array([0, 2, 4, 6], dtype=np.uint8)) & 3).ravel(), minlength=4)
    assert (counts > 0).all(), counts                 # all four segments present (coverage mode)

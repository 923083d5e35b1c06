"""bench.py -- fwd+bwd HBM throughput of the ReGELU2/ReSiLU2 + MS-LN/MS-RMSNorm
hot path on B200, plus activation bytes saved per layer (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one pass of every SURVEY.md section 8(a) row over one batch:
norm forward -> activation forward -> activation backward -> norm backward
(the order a transformer block runs them), on inputs already resident in HBM.
Each kernel is bracketed by its own CUDA events on the launching stream, and
L2 is flushed (a read of 2 x L2) before every kernel, outside the events, so no
kernel reads another's output from L2 (in training the whole network runs in
between).  value = algorithmic bytes of all ranks / max-over-ranks device time.

The `stream` key times the same step the way a training stream runs it: K
steps back to back between one event pair, no flush, consecutive kernels
overlapped by programmatic dependent launch, the backwards of step s reading
what the forwards of an earlier step wrote (N complete buffer sets, so every
buffer is touched again only after >= 3 x L2 bytes).  DESIGN.md 5.10 and 6.

Multi-GPU: one process per GPU; every rank processes its own batch of the
configured shape (weak scaling, data-parallel, no collective on the data path);
NCCL is used only for the barrier and the max/sum of timings.

--impl reference times the float64 CPU oracle (oracle/, the only reference
this tier has) on a bounded row sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2406_16282_b200.build import build_info  # noqa: E402  (provenance only; imports no kernels)

METRIC = "fwd+bwd HBM GB/s (fraction of B200 peak) and activation bytes saved per layer"
NOMINAL_HBM_GBS = 8000.0


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c4", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-chunks", type=int, default=8)
    ap.add_argument("--e2e-streams", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle sample time")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--no-fitter", action="store_true", help="skip the coefficient-fitter section")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank runs the full config (its own batch); "
                         "strong: the config's rows are split across ranks")
    ap.add_argument("--strong-config", default="c5", choices=sorted(synth.CONFIGS),
                    help="config of the row-sharded strong-scaling key (north_star: C5)")
    ap.add_argument("--strong-steps", type=int, default=10)
    ap.add_argument("--no-strong", action="store_true", help="skip the strong-scaling (row-sharded C5) key")
    ap.add_argument("--nvtx", action="store_true",
                    help="wrap every kernel launch in an NVTX range named after the 8(a) row "
                         "(e.g. ncu --nvtx --nvtx-include act_fwd/)")
    return ap.parse_args(argv)


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_cmd(gpus: int, argv, port: int, script: str = None):
    """The torchrun command that re-runs this script as `gpus` ranks (one
    process per GPU) on this node, rendezvous on 127.0.0.1."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(gpus),
            "--master-addr", "127.0.0.1", "--master-port", str(port),
            script or os.path.abspath(__file__)] + list(argv)


def self_launch(args, argv) -> int:
    """`bench.py --gpus N` called directly (no WORLD_SIZE in the environment)
    with N > 1: re-exec under torch.distributed.run so N ranks really run.
    NCCL's init log (rank / nranks per communicator) stays on, on stderr."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    import subprocess
    return subprocess.call(launch_cmd(args.gpus, argv, _free_port()), env=env)


def strong_summary(bytes_per_rank, ms_per_rank, steps, t1_ms=None):
    """Row-sharded (strong) scaling numbers: aggregate GB/s = bytes of all
    ranks / slowest rank, and t1 / (N tN) when the 1-GPU time is known."""
    N = len(ms_per_rank)
    tN = max(ms_per_rank) / steps
    out = {"n_ranks": N, "per_rank_ms_per_step": [round(m / steps, 4) for m in ms_per_rank],
           "ms_per_step": round(tN, 4), "GB/s": round(aggregate(bytes_per_rank, ms_per_rank, steps), 1),
           "rank_spread": round(max(ms_per_rank) / min(ms_per_rank) - 1, 4) if min(ms_per_rank) > 0 else None}
    if t1_ms is not None:
        out["t1_ms_per_step"] = round(t1_ms, 4)
        out["t1_over_N_tN"] = round(t1_ms / (N * tN), 4)
    return out


def shard_rows(R: int, world: int, rank: int, scaling: str):
    """(first global row, rows) this rank processes.  weak: each rank owns a
    whole batch of R rows (rows [rank*R, (rank+1)*R) of the global stream);
    strong: the R rows are split into contiguous, near-equal blocks."""
    if scaling == "weak":
        return rank * R, R
    lo = (R * rank) // world
    hi = (R * (rank + 1)) // world
    return lo, hi - lo


def aggregate(step_bytes_per_rank, ms_per_rank, steps):
    """Whole-job GB/s: bytes of all ranks / the slowest rank's device time."""
    return sum(step_bytes_per_rank) * steps / (max(ms_per_rank) / 1e3) / 1e9


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# bytes
# ---------------------------------------------------------------------------
def algorithmic_bytes(cfg, R):
    b = synth.ELEM_BYTES[cfg["dtype"]]
    n = R * cfg["F"]
    H = cfg["H"]
    act = 2 * b * n + (n + 3) // 4              # read x, write y, write codes  (= read dy, codes; write dx)
    return {"norm_fwd": (2 * b * H + 4) * R,   # read x, write y, write rstd
            "act_fwd": act,
            "act_bwd": act,
            "norm_bwd": (3 * b * H + 4) * R}   # read dy, y, rstd; write dx


def rw_bytes(cfg, R):
    """(read, write) algorithmic bytes per kernel; sums to algorithmic_bytes."""
    b = synth.ELEM_BYTES[cfg["dtype"]]
    n = R * cfg["F"]
    H = cfg["H"]
    nc = (n + 3) // 4
    return {"norm_fwd": (b * H * R, (b * H + 4) * R),
            "act_fwd": (b * n, b * n + nc),
            "act_bwd": (b * n + nc, b * n),
            "norm_bwd": ((2 * b * H + 4) * R, b * H * R)}


def rw_model_section(x, dy, dx, y, flush, sink, stream, kern, rw, iters=10):
    """Direction-aware HBM model (DESIGN 5.3): time a torch copy (1 read : 1
    write) and add (2 : 1) of the activation tensors with the bench protocol,
    fit t = R/r + W/w, and rate every kernel against its own read/write mix.
    Informational only: roofline.peak stays the driver's copy figure."""
    def timeit(fn):
        fn()
        ts = []
        for _ in range(iters):
            sink.copy_(flush.sum())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            ts.append((e0, e1))
        torch.cuda.synchronize()
        us = sorted(a.elapsed_time(b) * 1e3 for a, b in ts)
        return us[len(us) // 2]

    B = x.numel() * x.element_size()
    t_copy = timeit(lambda: y.copy_(x))
    t_add = timeit(lambda: torch.add(x, dy, out=dx))
    tr = (t_add - t_copy) / B                  # us per byte read
    tw = t_copy / B - tr                       # us per byte written
    if not (tr > 0 and tw > 0):
        return None
    out = {"read_GBs": round(1e-3 / tr, 1), "write_GBs": round(1e-3 / tw, 1), "probe_bytes": B,
           "copy_us": round(t_copy, 2), "add_us": round(t_add, 2), "kernels": {}}
    for k, (rd, wr) in rw.items():
        ideal = rd * tr + wr * tw
        out["kernels"][k] = {"read": rd, "write": wr, "model_us": round(ideal, 2),
                             "frac": round(ideal / kern[k]["us"], 4)}
    return out


def bytes_saved(cfg, R):
    b = synth.ELEM_BYTES[cfg["dtype"]]
    n = R * cfg["F"]
    act_exact, act_ours = n * b, (n + 3) // 4
    norm_in_fp32 = R * cfg["H"] * 4             # norms run in fp32 under AMP
    norm_in_t = R * cfg["H"] * b
    return {"act": {"exact_bytes": act_exact, "ours_bytes": act_ours, "saved_bytes": act_exact - act_ours,
                    "ratio": round(act_exact / act_ours, 3)},
            "norm": {"exact_bytes_fp32_input": norm_in_fp32, "exact_bytes_T_input": norm_in_t,
                     "ours_bytes": 4 * R, "saved_bytes_fp32_input": norm_in_fp32 - 4 * R,
                     "note": "y is the next linear layer's saved input (Prop. 5.1 cond. 3), counted there"}}


# ---------------------------------------------------------------------------
# clocks (NVML) during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    def __init__(self, index: int):
        self.samples, self.mem, self.reasons, self.max_mhz = [], [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        self.mem.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_MEM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}
        for k, bit in names.items():
            if r & bit:
                self.reasons.add(k)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._stop.wait(0.005)

    def start(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self.nv:
            self._stop.set()
            self._t.join()
            try:
                self._sample()
            except Exception:
                pass
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "mem_mhz": statistics.median(self.mem) if self.mem else None}


# ---------------------------------------------------------------------------
# CPU baseline: the float64 oracle on a bounded row sample
# ---------------------------------------------------------------------------
def oracle_step_sample(cfg, rows, eps, threads=None):
    """One oracle pass of the four rows of 8(a) on `rows` rows; returns
    (seconds, algorithmic bytes, threads).  threads=None: all usable cores."""
    import oracle
    if threads is not None:
        oracle.DEFAULT_THREADS = int(threads)
    elif oracle.DEFAULT_THREADS is None:    # all usable host cores, whatever OMP_NUM_THREADS says
        oracle.DEFAULT_THREADS = len(os.sched_getaffinity(0))
    dt = cfg["dtype"]
    x = synth.to_numpy_storage(synth.act_input(rows, cfg["F"], dt))
    dy = synth.to_numpy_storage(synth.grad_input(rows, cfg["F"], dt))
    xn = synth.to_numpy_storage(synth.norm_input(rows, cfg["H"], dt))
    gn = synth.to_numpy_storage(synth.grad_input(rows, cfg["H"], dt, stream=synth.S_NORM_DY))
    nf, nb = (oracle.msln_fwd, oracle.msln_bwd) if cfg["norm"] == "ln" else (oracle.msrms_fwd, oracle.msrms_bwd)
    t0 = time.perf_counter()
    yn, r = nf(oracle.decode(xn, dt), float(np.float32(eps)))
    yn_st = oracle.round_to(yn, dt)
    y, codes = oracle.act_fwd(cfg["act"], oracle.decode(x, dt))
    oracle.round_to(y, dt)
    oracle.act_bwd_contract(cfg["act"], codes, dy, dt)
    dxn = nb(oracle.decode(gn, dt), oracle.decode(yn_st, dt), r.astype(np.float32).astype(np.float64))
    oracle.round_to(dxn, dt)
    sec = time.perf_counter() - t0
    return sec, sum(algorithmic_bytes(cfg, rows).values()), oracle.max_threads()


def calibrate_rows(cfg, eps, target_s):
    """Rows of the workload whose oracle pass costs ~target_s seconds."""
    rows = 8
    oracle_step_sample(cfg, rows, eps)                    # load / first-touch
    while True:
        sec, _, _ = oracle_step_sample(cfg, rows, eps)
        if sec >= min(0.5, target_s / 4) or rows >= cfg["R"]:
            break
        rows = min(cfg["R"], rows * 4)
    return max(8, min(cfg["R"], int(rows * target_s / max(sec, 1e-4))))


def measured_hbm_peak():
    """HBM peak for the roofline: MEASURED_PEAKS.json (driver-written; the
    burst copy figure, `hbm_gbs`, for kernels timed alone), else the fallback
    the profiling guide states.  Tolerates a file without that key (any other
    numeric `*hbm*gb*` entry, burst preferred over sustained)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        if isinstance(d.get("hbm_gbs"), (int, float)):
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        keys = sorted((k for k, v in d.items() if isinstance(v, (int, float)) and "hbm" in k.lower()
                       and "gb" in k.lower()), key=lambda k: ("sustain" in k.lower(), k))
        if keys:
            return float(d[keys[0]]), f"measured (MEASURED_PEAKS.json {keys[0]})"
    except (OSError, ValueError, AttributeError):
        pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_sockets():
    """Physical packages (sockets) of the host, from sysfs."""
    import glob
    ids = set()
    for p in glob.glob("/sys/devices/system/cpu/cpu[0-9]*/topology/physical_package_id"):
        try:
            ids.add(open(p).read().strip())
        except OSError:
            pass
    return len(ids) or None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(cfg, eps, target_s):
    import oracle
    rows = calibrate_rows(cfg, eps, target_s)
    sec, nbytes, threads = oracle_step_sample(cfg, rows, eps)
    # the same oracle on one core, on a proportionally smaller sample
    rows1 = max(8, rows // max(1, threads))
    sec1, nbytes1, _ = oracle_step_sample(cfg, rows1, eps, threads=1)
    oracle.DEFAULT_THREADS = threads
    return {"value": round(nbytes / sec / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": f"{rows} of {cfg['R']} rows of {cfg['desc']}: norm fwd+bwd and act fwd+bwd, float64 "
                      f"oracle incl. storage decode/encode, {sec:.2f} s",
            "seconds": round(sec, 3), "rows": rows, "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
            "sockets": cpu_sockets(),
            "single_core": {"value": round(nbytes1 / sec1 / 1e9, 4), "unit": "GB/s", "rows": rows1,
                            "seconds": round(sec1, 3)}}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = synth.CONFIGS[args.config]
    # each step is a bounded sample: the whole run costs ~4 x cpu_seconds
    budget = max(0.2, 4 * args.cpu_seconds / max(1, args.steps + args.warmup))
    rows = calibrate_rows(cfg, args.eps, budget)
    for _ in range(args.warmup):
        oracle_step_sample(cfg, rows, args.eps)
    secs, nbytes, threads = [], 0, 1
    for _ in range(args.steps):
        s, nbytes, threads = oracle_step_sample(cfg, rows, args.eps)
        secs.append(s)
    total = sum(secs)
    value = nbytes * len(secs) / total / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * total / len(secs), 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "rows_per_step_sample": rows},
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
                             "sample": f"{rows} of {cfg['R']} rows per step"},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def swiglu_section(P, cfg, gate, up, stream, flush, sink, args, iters=20):
    """the fused ReSwiGLU2 gate (h = SiLU(gate) * up with
    ReSiLU2's backward) against the unfused composition (resilu2 kernels +
    torch elementwise mul) on the same [R, F] tensors, L2 flushed before every
    launch.  Reported beside the headline; not part of its step."""
    b = gate.element_size()
    n = gate.numel()
    h, a = torch.empty_like(gate), torch.empty_like(gate)
    codes = torch.empty(P.codes_bytes(n), dtype=torch.uint8, device=gate.device)
    dh = torch.empty_like(up).copy_(gate).neg_()  # a third, distinct [R, F] tensor (no L2 sharing with up)
    dg, du = torch.empty_like(gate), torch.empty_like(gate)
    a2 = torch.empty_like(gate)
    fused = {
        "fwd": lambda: P.reswiglu2_fwd(gate, up, h=h, a=a, codes=codes, stream=stream),
        "bwd": lambda: P.reswiglu2_bwd(dh, up, a, codes, dgate=dg, dup=du, stream=stream),
    }

    def unfused_fwd():
        P.resilu2_fwd(gate, y=a2, codes=codes, stream=stream)
        torch.mul(a2, up, out=h)

    def unfused_bwd():
        torch.mul(dh, a2, out=du)
        torch.mul(dh, up, out=dg)
        P.resilu2_bwd(dg, codes, dx=dg, stream=stream)

    def timeit(fn):
        for _ in range(3):
            fn()
        evs = []
        for _ in range(iters):
            sink.copy_(flush.sum())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return sum(e0.elapsed_time(e1) for e0, e1 in evs) / iters * 1e3

    bf, bb = (4 * b * n + (n + 3) // 4), (5 * b * n + (n + 3) // 4)
    tf, tb = timeit(fused["fwd"]), timeit(fused["bwd"])
    uf, ub = timeit(unfused_fwd), timeit(unfused_bwd)
    # in-stream: back-to-back fused launches from a graph over N complete buffer sets
    ns = stream_sets({"fwd": bf}, torch.cuda.get_device_properties(gate.device).L2_cache_size)
    more = lambda t, copy: [t] + [t.clone() if copy else torch.empty_like(t) for _ in range(ns - 1)]  # noqa: E731
    G, Uu, DH, H, A, C, DG, DU = (more(gate, True), more(up, True), more(dh, True), more(h, False), more(a, False),
                                  more(codes, False), more(dg, False), more(du, False))
    pg = ns * max(1, -(-8 // ns))
    gf = graph_us(lambda i: P.reswiglu2_fwd(G[i % ns], Uu[i % ns], h=H[i % ns], a=A[i % ns], codes=C[i % ns]),
                  stream, per_graph=pg)
    gb = graph_us(lambda i: P.reswiglu2_bwd(DH[i % ns], Uu[i % ns], A[i % ns], C[i % ns], dgate=DG[i % ns],
                                            dup=DU[i % ns]), stream, per_graph=pg)
    del G, Uu, DH, H, A, C, DG, DU
    return {"shape": list(gate.shape), "fused_fwd_us": round(tf, 2), "fused_bwd_us": round(tb, 2),
            "fused_GB/s": round((bf + bb) / (tf + tb) / 1e3, 1),
            "fused_frac": round((bf + bb) / (tf + tb) / 1e3 / measured_hbm_peak()[0], 4),
            "graph_fwd_us": round(gf, 2), "graph_bwd_us": round(gb, 2),
            "graph_frac": round((bf + bb) / (gf + gb) / 1e3 / measured_hbm_peak()[0], 4),
            "unfused_fwd_us": round(uf, 2), "unfused_bwd_us": round(ub, 2),
            "speedup_fwd_bwd": round((uf + ub) / (tf + tb), 3),
            "algorithmic_bytes": {"fwd": bf, "bwd": bb},
            "saved_bytes_per_layer": {"exact_silu_mul": 3 * b * n, "reswiglu2": 2 * b * n + (n + 3) // 4},
            "gpu_launches": 2 * iters}


def mixed_norm_section(P, cfg, R, dev, stream, flush, sink, peak, eps, iters=20):
    """Mixed-precision MS norm (fp32 residual in, 16-bit y out; 16-bit dy ->
    fp32 dx; the AMP layout of Fig. 5 / 6) at the config's [R, H]: us and
    GB/s of fwd and bwd on their algorithmic bytes."""
    if cfg["dtype"] == "f32":
        return None
    H = cfg["H"]
    ln = cfg["norm"] == "ln"
    x = synth.norm_input(R, H, "f32", device=dev)
    g = synth.grad_input(R, H, cfg["dtype"], device=dev, stream=synth.S_NORM_DY)
    y = torch.empty(R, H, dtype=synth.TORCH_DTYPES[cfg["dtype"]], device=dev)
    rstd = torch.empty(R, dtype=torch.float32, device=dev)
    dx = torch.empty(R, H, dtype=torch.float32, device=dev)
    fwd, bwd = (P.msln_fwd_mixed, P.msln_bwd_mixed) if ln else (P.msrms_fwd_mixed, P.msrms_bwd_mixed)
    fns = {"fwd": lambda: fwd(x, eps, y.dtype, y=y, rstd=rstd, stream=stream),
           "bwd": lambda: bwd(g, y, rstd, dx=dx, stream=stream)}
    nbytes = {"fwd": (4 * H + 2 * H + 4) * R, "bwd": (2 * 2 * H + 4 + 4 * H) * R}
    out = {"shape": [R, H], "x": "f32", "y": cfg["dtype"]}
    for k, fn in fns.items():
        for _ in range(3):
            fn()
        evs = []
        for _ in range(iters):
            sink.copy_(flush.sum())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        us = float(np.median([a.elapsed_time(b) * 1e3 for a, b in evs]))
        out[k] = {"us_median": round(us, 2), "bytes": nbytes[k], "GB/s": round(nbytes[k] / us / 1e3, 1),
                  "frac": round(nbytes[k] / us / 1e3 / peak, 4)}
    return out


def graph_us(body, stream, per_graph=8, reps=8):
    """Mean µs per launch of body(0) .. body(per_graph - 1) captured in one
    CUDA graph (launches back to back, PDL edges kept) and replayed `reps`
    times between one event pair.  `body` launches on the current stream."""
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream(stream.device)
    cs.wait_stream(stream)
    with torch.cuda.graph(g, stream=cs):
        for i in range(per_graph):
            body(i)
    stream.wait_stream(cs)
    with torch.cuda.stream(stream):
        for _ in range(2):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * per_graph)


def stepact_section(P, cfg, x, dy, stream, flush, sink, peak, iters=20):
    """the table-driven k-bit step activation on the
    config's activation tensor -- k = 2 with the paper's table (bitwise equal
    to the specialised kernel), k = 3 and k = 4 -- GB/s of fwd + bwd."""
    from paper_2406_16282_b200 import tables
    tab = tables.REGELU2 if cfg["act"] == "gelu" else tables.RESILU2
    b, n = x.element_size(), x.numel()
    y, dx = torch.empty_like(x), torch.empty_like(dy)
    ns = stream_sets({"act": 2 * b * n}, torch.cuda.get_device_properties(x.device).L2_cache_size)
    xs, dys = [x] + [x.clone() for _ in range(ns - 1)], [dy] + [dy.clone() for _ in range(ns - 1)]
    ys, dxs = [y] + [torch.empty_like(y) for _ in range(ns - 1)], [dx] + [torch.empty_like(dx) for _ in range(ns - 1)]
    out = {}
    for k, thr, lv in ((2, tab["c"], tables.levels(tab)),
                       (3, [-3.0 + 1.0 * i for i in range(7)], [i / 7 for i in range(8)]),
                       (4, [-3.0 + 0.4 * i for i in range(15)], [i / 15 for i in range(16)])):
        codes = torch.empty(P.codes_bytes_k(n, k), dtype=torch.uint8, device=x.device)
        fns = (lambda: P.stepact_fwd(x, tab["act"], k, thr, y=y, codes=codes, stream=stream),
               lambda: P.stepact_bwd(dy, codes, k, lv, dx=dx, stream=stream))
        ts = []
        for fn in fns:
            for _ in range(3):
                fn()
            evs = []
            for _ in range(iters):
                sink.copy_(flush.sum())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn()
                e1.record(stream)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            ts.append(sum(a.elapsed_time(c) for a, c in evs) / iters * 1e3)
        nbytes = 2 * (2 * b * n + P.codes_bytes_k(n, k))
        # in-stream: back-to-back launches from a graph over N buffer sets
        # (every buffer touched again only after >= 3 x L2 bytes, bench.stream_sets)
        cs = [codes] + [torch.empty_like(codes) for _ in range(ns - 1)]
        gf = graph_us(lambda i: P.stepact_fwd(xs[i % ns], tab["act"], k, thr, y=ys[i % ns], codes=cs[i % ns]),
                      stream, per_graph=ns * max(1, -(-8 // ns)))
        gb = graph_us(lambda i: P.stepact_bwd(dys[i % ns], cs[i % ns], k, lv, dx=dxs[i % ns]), stream,
                      per_graph=ns * max(1, -(-8 // ns)))
        out[f"k{k}"] = {"fwd_us": round(ts[0], 2), "bwd_us": round(ts[1], 2),
                        "GB/s": round(nbytes / (ts[0] + ts[1]) / 1e3, 1),
                        "frac": round(nbytes / (ts[0] + ts[1]) / 1e3 / peak, 4),
                        "graph_fwd_us": round(gf, 2), "graph_bwd_us": round(gb, 2),
                        "graph_frac": round(nbytes / (gf + gb) / 1e3 / peak, 4)}
        del cs
    return out


PAPER_THETA = {  # P:L1062-1063 (GELU), P:L1139-1140 (SiLU), P:L1346-1347 (ReGELU2-d)
    ("gelu", "h"): [-0.04922261145617846, 1.0979632065417297, -3.1858810036855245, -0.001178821281161997,
                    3.190832613414926],
    ("silu", "h"): [-0.04060357190528599, 1.080925428529668, -6.3050461001646445, -0.0008684942046214787,
                    6.325815242089708],
    ("gelu", "dh"): [0.32465931184406527, 0.34812875668739607, -0.4535743722857079, -0.0010587205574873046,
                     0.4487575313884231],
}


def fitter_section(stream, cpu=True, chains=148 * 3 * 128, iters=1000, n_obj=148 * 3 * 128 * 4):
    """the offline coefficient fitter.  (1) batched
    objective throughput (J evaluations/s; one thread per theta, FP64-bound);
    (2) a full fit per (act, objective) of App. E / App. I (variable-projection
    annealing + LM refinement) -- time, the J reached vs J at the paper's
    constants (both by the GPU objective), the fitted constants; (3) k = 1..4
    fits (J falls with k); (4) the oracle's (QUADPACK) J/s on the host for the
    cpu baseline."""
    from paper_2406_16282_b200 import fit as gfit
    from paper_2406_16282_b200 import ops
    out = {"chains": chains, "iters": iters}
    g = torch.Generator(device="cuda").manual_seed(2406)
    for act in ("gelu", "silu"):
        th = torch.tensor(PAPER_THETA[(act, "h")], dtype=torch.float64, device="cuda")
        batch = (th + 0.05 * torch.randn(n_obj, 5, dtype=torch.float64, device="cuda", generator=g)).contiguous()
        J = torch.empty(n_obj, dtype=torch.float64, device="cuda")
        ops.fit_objective(batch, act, J=J, stream=stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            ops.fit_objective(batch, act, J=J, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 3 / 1e3
        out[f"objective_{act}"] = {"thetas": n_obj, "ms": round(t * 1e3, 3), "J_per_s": round(n_obj / t, 1)}
    for act, obj in PAPER_THETA:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        best, cth, _ = ops.fit_anneal(act, objective=obj, chains=chains, iters=iters, stream=stream,
                                      projected=True)
        e1.record(stream)
        best2, _, _ = ops.fit_refine(cth, act, objective=obj, iters=40, stream=stream)
        e2 = torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        torch.cuda.synchronize()
        t, tr = e0.elapsed_time(e1) / 1e3, e1.elapsed_time(e2) / 1e3
        b = best2.cpu().tolist()
        Jp = float(gfit.objective(PAPER_THETA[(act, obj)], act, objective=obj)[0])
        out[f"anneal_{act}_{obj}"] = {
            "anneal_seconds": round(t, 3), "refine_seconds": round(tr, 3),
            "anneal_J_evals_per_s": round(chains * (iters + 1) / t, 1),
            "J_after_anneal": float(best[-1]),
            "J": b[-1], "J_paper": Jp, "J_over_paper": round(b[-1] / Jp, 6),
            "a": [round(v, 6) for v in b[:2]], "c": [round(v, 6) for v in b[2:5]]}
    # k-bit fits (Eq. 14 with 2^k - 1 ReLUs; variable projection + LM)
    kbit = {}
    for act in ("gelu", "silu"):
        kbit[act] = {}
        for k, ch, it, ri in ((1, 4096, 300, 20), (2, 8192, 800, 40), (3, 8192, 2000, 20), (4, 4096, 4000, 8)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            f = gfit.fit(act, k=k, chains=ch, iters=it, refine_iters=ri)
            e1.record(stream)
            torch.cuda.synchronize()
            kbit[act][f"k{k}"] = {"J": f.J, "seconds": round(e0.elapsed_time(e1) / 1e3, 3)}
    out["kbit_fits"] = kbit
    if cpu:
        from oracle import fit as ofit
        n, t0 = 0, time.perf_counter()
        rng = np.random.default_rng(1)
        while time.perf_counter() - t0 < 3.0:
            for act in ("gelu", "silu"):
                ofit.objective(act, 2, np.array(PAPER_THETA[(act, "h")]) + 0.05 * rng.standard_normal(5))
                n += 1
        el = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": round(n / el, 2), "unit": "J evals/s", "cores": 1, "kind": "oracle",
                               "sample": f"{n} objective evaluations (GELU and SiLU alternating, QUADPACK via "
                                         f"scipy.integrate.quad) in {el:.1f} s"}
    return out


def block_section(cfg, dev, tunings=("full", "lora_qv", "lora_all", "lora_fa_all", "frozen_ffn")):
    """activation bytes a whole transformer block
    (attention + FFN, the config's model dimensions and batch) keeps for
    backward, measured with saved_tensors_hooks (storage-deduplicated,
    parameters excluded), exact (affine norms in fp32 as under AMP, exact
    GELU / SiLU) vs ours (merged affine, MS norms, ReGELU2 / fused ReSwiGLU2),
    per fine-tuning regime; unit = one [b, n, c] 16-bit tensor (Fig. 5/6).
    Where no consumer of a norm keeps its input (frozen / LoRA-FA; Prop. 5.1
    condition 3 fails) the MS norm shares nothing."""
    from paper_2406_16282_b200.blocks import Block, activation_bytes, unit_model
    arch = "vit" if cfg["act"] == "gelu" else "llama"
    dt = synth.TORCH_DTYPES[cfg["dtype"]] if cfg["dtype"] != "f32" else torch.bfloat16
    b, n, c, h = cfg["batch"], cfg["seq"], cfg["H"], cfg["F"]
    unit = b * n * c * 2
    x = synth.norm_input(b * n, c, "bf16", device=dev).view(b, n, c).requires_grad_(True)
    out = {"arch": arch, "shape": {"batch": b, "seq": n, "hidden": c, "ffn": h, "heads": cfg["heads"]},
           "unit_bytes": unit, "decoded_model_full_tuning": {k: round(v, 4) for k, v in unit_model(arch, h / c).items()},
           "model_note": "torch SDPA returns [b, n, h, d]: the out-projection's saved input is the attention output "
                         "itself, one unit below the model's separate kernels", "tunings": {}}
    x32 = x.detach().float().requires_grad_(True)
    for t in list(tunings) + ["full_amp"]:
        amp = t == "full_amp"           # fp32 residual stream, bf16 linears: the mixed MS norms
        blk = Block(arch, c, h, cfg["heads"], tuning="full" if amp else t, dtype=dt, device=dev, residual_fp32=amp)
        te, pe = activation_bytes(blk, x32 if amp else x, by_module=True)
        to, po = activation_bytes(blk.to_ours(), x32 if amp else x, by_module=True)
        out["tunings"][t] = {"exact_units": round(te / unit, 4), "ours_units": round(to / unit, 4),
                             "saved_fraction": round(1 - to / te, 4), "exact_bytes": te, "ours_bytes": to,
                             "norm_shared": [blk.norm_shared(1), blk.norm_shared(2)],
                             "per_module_units": {k: [round(pe.get(k, 0) / unit, 4), round(po.get(k, 0) / unit, 4)]
                                                  for k in sorted(set(pe) | set(po))}}
        del blk
        torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
KERNELS = ["norm_fwd", "act_fwd", "act_bwd", "norm_bwd"]


class Workload:
    """One rank's rows [row0, row0 + R) of a config, resident in HBM, and the
    four launches of one step (norm fwd -> act fwd -> act bwd ->
    norm bwd) through the C-ABI binding."""

    def __init__(self, P, cfg, row0, R, dev, stream, eps, nvtx=False):
        F, H, dt = cfg["F"], cfg["H"], cfg["dtype"]
        self.cfg, self.R, self.dev, self.stream, self.eps, self.nvtx = cfg, R, dev, stream, eps, nvtx
        self.act_fwd, self.act_bwd = ((P.regelu2_fwd, P.regelu2_bwd) if cfg["act"] == "gelu"
                                      else (P.resilu2_fwd, P.resilu2_bwd))
        self.norm_fwd, self.norm_bwd = ((P.msln_fwd, P.msln_bwd) if cfg["norm"] == "ln"
                                        else (P.msrms_fwd, P.msrms_bwd))
        self.x = synth.act_input(R, F, dt, row_start=row0, device=dev)
        self.dy = synth.grad_input(R, F, dt, row_start=row0, device=dev)
        self.xn = synth.norm_input(R, H, dt, row_start=row0, device=dev)
        self.gn = synth.grad_input(R, H, dt, row_start=row0, device=dev, stream=synth.S_NORM_DY)
        self.y, self.dx = torch.empty_like(self.x), torch.empty_like(self.dy)
        self.codes = torch.empty(P.codes_bytes(R * F), dtype=torch.uint8, device=dev)
        self.yn, self.dxn = torch.empty_like(self.xn), torch.empty_like(self.gn)
        self.rstd = torch.empty(R, dtype=torch.float32, device=dev)
        s = stream
        self.launch = {
            "norm_fwd": lambda: self.norm_fwd(self.xn, eps, y=self.yn, rstd=self.rstd, stream=s),
            "act_fwd": lambda: self.act_fwd(self.x, y=self.y, codes=self.codes, stream=s),
            "act_bwd": lambda: self.act_bwd(self.dy, self.codes, dx=self.dx, stream=s),
            "norm_bwd": lambda: self.norm_bwd(self.gn, self.yn, self.rstd, dx=self.dxn, stream=s),
        }
        self.nbytes = algorithmic_bytes(cfg, R)

    def step(self, flush, sink, evs=None):
        for i, k in enumerate(KERNELS):
            sink.copy_(flush.sum())                    # evict L2 by reading 2 x L2 (outside the events)
            if evs is not None:
                evs[2 * i].record(self.stream)
            if self.nvtx:
                torch.cuda.nvtx.range_push(k)
            self.launch[k]()
            if self.nvtx:
                torch.cuda.nvtx.range_pop()
            if evs is not None:
                evs[2 * i + 1].record(self.stream)

    def timed(self, flush, sink, steps, warmup, world, sampler=None):
        """W untimed steps, then `steps` steps bracketed by barrier +
        synchronize; returns {kernel: [ms per launch]}."""
        for _ in range(max(3, warmup)):
            self.step(flush, sink)
        torch.cuda.synchronize()
        events = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(steps)]
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        if sampler is not None:
            sampler.start()
        for s in range(steps):
            self.step(flush, sink, events[s])
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        return {k: [events[s][2 * i].elapsed_time(events[s][2 * i + 1]) for s in range(steps)]
                for i, k in enumerate(KERNELS)}

    def free(self):
        for k in ("x", "dy", "xn", "gn", "y", "dx", "codes", "yn", "dxn", "rstd"):
            setattr(self, k, None)


def stream_sets(nbytes: dict, l2: int, cap: int = 256) -> int:
    """Buffer sets for the in-stream protocols: enough that every buffer --
    input or output -- is touched again only after >= 3 x L2 bytes of other
    traffic, even when a single kernel runs back to back with itself (the
    smallest kernel decides), so neither a read nor a rewrite of a still-dirty
    line is served by L2."""
    return int(max(2, min(cap, -(-3 * l2 // max(1, min(nbytes.values()))) + 1)))


class StreamWorkload:
    """The step as a training stream runs it: the four launches back to back
    on one stream, no flush and no event between them, so each kernel's launch
    and prologue overlap the previous one's drain (programmatic dependent
    launch, csrc/common.cuh).  N complete buffer sets (inputs and outputs,
    `stream_sets`): step s runs the forwards on set s % N and the backwards on
    set (s + 1) % N, consuming the codes, y and rstd that set's forwards wrote
    N - 1 steps earlier; per-kernel timings launch one kernel on sets 0, 1,
    ... N - 1 in turn.  Every buffer is therefore last touched more than 3 x L2
    bytes before, so nothing is served from L2 that training would not also
    find cold (inputs) or have to write back (outputs)."""

    def __init__(self, w: "Workload", nsets: int):
        self.w, self.n = w, nsets
        new = lambda t, copy: [t] + [t.clone() if copy else torch.empty_like(t) for _ in range(nsets - 1)]  # noqa
        self.x, self.dy, self.xn, self.gn = (new(t, True) for t in (w.x, w.dy, w.xn, w.gn))
        self.y, self.dx, self.codes, self.yn, self.rstd, self.dxn = (
            new(t, False) for t in (w.y, w.dx, w.codes, w.yn, w.rstd, w.dxn))
        eps = w.eps
        self.s = w.stream      # the launch stream (the capture stream while a graph is recorded)
        self.launch = {
            "norm_fwd": lambda a: w.norm_fwd(self.xn[a], eps, y=self.yn[a], rstd=self.rstd[a], stream=self.s),
            "act_fwd": lambda a: w.act_fwd(self.x[a], y=self.y[a], codes=self.codes[a], stream=self.s),
            "act_bwd": lambda a: w.act_bwd(self.dy[a], self.codes[a], dx=self.dx[a], stream=self.s),
            "norm_bwd": lambda a: w.norm_bwd(self.gn[a], self.yn[a], self.rstd[a], dx=self.dxn[a], stream=self.s),
        }
        for a in range(nsets):  # every set holds a forward's outputs before the first backward reads them
            self.launch["norm_fwd"](a)
            self.launch["act_fwd"](a)

    def step(self, s):
        a, b = s % self.n, (s + 1) % self.n
        self.launch["norm_fwd"](a)
        self.launch["act_fwd"](a)
        self.launch["act_bwd"](b)
        self.launch["norm_bwd"](b)

    def _time(self, body, n, warmup, world):
        for i in range(max(3, warmup)):
            body(i)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.w.stream)
        h0 = time.perf_counter()
        for i in range(n):
            body(i)
        self.last_host_s = time.perf_counter() - h0   # host time to enqueue the n units
        e1.record(self.w.stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        return e0.elapsed_time(e1)

    def timed_steps(self, steps, warmup, world):
        """ms for `steps` steps between one event pair (after W warm-up steps)."""
        return self._time(self.step, steps, warmup, world)

    def graph(self, body, n):
        """A CUDA graph of body(0) .. body(n - 1), recorded from the same
        launches (PDL launches become programmatic edges), so replaying it
        costs one host call per n launches."""
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(self.w.dev)
        cs.wait_stream(self.w.stream)
        with torch.cuda.graph(g, stream=cs):
            self.s = cs
            for i in range(n):
                body(i)
        self.s = self.w.stream
        self.w.stream.wait_stream(cs)
        return g

    def timed_graph(self, body, per_graph, units, warmup, world):
        """ms per unit (launch or step): a graph of `per_graph` units (a
        multiple of the set count, so it covers every set) replayed until at
        least `units` units have run, between one event pair."""
        g = self.graph(body, per_graph)
        reps = max(1, -(-units // per_graph))
        with torch.cuda.stream(self.w.stream):
            ms = self._time(lambda i: g.replay(), reps, max(1, warmup // per_graph), world)
        del g
        return ms / (reps * per_graph)

    def per_graph(self, at_least=8):
        return self.n * max(1, -(-at_least // self.n))

    def timed_kernel(self, k, launches, warmup, world):
        """ms per launch for back-to-back launches of one kernel on sets 0, 1, .."""
        return self._time(lambda i: self.launch[k](i % self.n), launches, warmup, world) / launches

    def free(self):
        for k in ("x", "dy", "xn", "gn", "y", "dx", "codes", "yn", "rstd", "dxn"):
            setattr(self, k, None)


def gather_floats(vals, world, cdev):
    t = torch.tensor(vals, dtype=torch.float64, device=cdev)
    if world == 1:
        return [t.tolist()]
    parts = [torch.zeros_like(t) for _ in range(world)]
    torch.distributed.all_gather(parts, t)
    return [p.tolist() for p in parts]


OUTPUTS = ("y", "codes", "dx", "yn", "rstd", "dxn")


def row_slices(cfg, r0, r1):
    """Element (byte, for codes) ranges of rows [r0, r1) in each flat output
    of a Workload (F % 4 == 0, so a row block's codes are whole bytes)."""
    F, H = cfg["F"], cfg["H"]
    return {"y": (r0 * F, r1 * F), "codes": (r0 * F // 4, r1 * F // 4), "dx": (r0 * F, r1 * F),
            "yn": (r0 * H, r1 * H), "rstd": (r0, r1), "dxn": (r0 * H, r1 * H)}


def output_checksums(w, r0, r1, base_row):
    """Position-weighted int64 checksums of the bytes of rows [r0, r1) of
    every output of `w` (whose first row is global row `base_row`); the weights
    depend on the byte's global position, so equal checksums across shardings
    mean equal bytes in place (with overwhelming probability)."""
    sl = row_slices(w.cfg, r0 - base_row, r1 - base_row)
    g0 = row_slices(w.cfg, r0, r1)
    M = 2147483647
    out = []
    for name in OUTPUTS:
        t = getattr(w, name).reshape(-1)
        lo, hi = sl[name]
        eb = t.element_size()
        raw = t[lo:hi].view(torch.uint8)
        p0 = g0[name][0] * eb
        acc = 0
        for c in range(0, raw.numel(), 1 << 26):   # 64 MB chunks bound the int64 temporaries
            b = raw[c:c + (1 << 26)].to(torch.int64)
            pos = torch.arange(p0 + c, p0 + c + b.numel(), device=b.device, dtype=torch.int64)
            acc = (acc + int((((b + 1) * ((pos % 1000003) * 2654435761 % 1000003 + 1)) % M).sum().item())) % M
        out.append(float(acc))                      # < 2^31: exact in the float64 gather
    return out


def strong_section(P, args, world, rank, dev, stream, flush, sink, cdev):
    """north_star / SURVEY 8(e): the strong-scaling configuration (C5,
    LLaMA-13B shapes) with its R rows split into contiguous blocks, rank r
    owning rows [r R / N, (r + 1) R / N).  Each rank times its shard (barrier-
    aligned); with N > 1, rank 0 then also runs all R rows alone on its GPU so
    t1 / (N tN) comes from the same box and run."""
    cfg = synth.CONFIGS[args.strong_config]
    row0, R = shard_rows(cfg["R"], world, rank, "strong")
    w = Workload(P, cfg, row0, R, dev, stream, args.eps)
    pk = w.timed(flush, sink, args.strong_steps, 3, world)
    ms = sum(sum(v) for v in pk.values())
    nb = sum(w.nbytes.values())
    sums = output_checksums(w, row0, row0 + R, row0)
    parts = gather_floats([ms, float(nb), float(row0), float(R)] + sums, world, cdev)
    w.free()
    torch.cuda.empty_cache()
    t1 = None
    shard_check = None
    if world == 1:
        t1 = ms / args.strong_steps
    else:
        if rank == 0:
            w1 = Workload(P, cfg, 0, cfg["R"], dev, stream, args.eps)
            pk1 = w1.timed(flush, sink, args.strong_steps, 3, 1)
            t1 = sum(sum(v) for v in pk1.values()) / args.strong_steps
            # 8(e): the one-GPU run's outputs, checksummed over every rank's
            # row block, must equal what that rank computed on its shard
            mism = []
            for r, p in enumerate(parts):
                a, n = int(p[2]), int(p[3])
                ref = output_checksums(w1, a, a + n, 0)
                mism += [f"rank{r}:{name}" for name, u, v in zip(OUTPUTS, p[4:], ref) if u != v]
            shard_check = {"outputs": list(OUTPUTS), "bitwise_equal_to_one_gpu": not mism, "mismatches": mism}
            w1.free()
            torch.cuda.empty_cache()
        torch.distributed.barrier()
    if rank != 0:
        return None
    out = strong_summary([p[1] for p in parts], [p[0] for p in parts], args.strong_steps, t1)
    out.update({"config": f"{args.strong_config}: {cfg['desc']}", "rows_total": cfg["R"],
                "shards": [[int(p[2]), int(p[3])] for p in parts], "steps": args.strong_steps,
                "partition": "contiguous row blocks, rank r owns rows [r*R/N, (r+1)*R/N); no data-path collective",
                "t1": "rank 0 alone on all rows, same run" if world > 1 else "this run",
                "shard_invariance": shard_check,
                "checksums": "per rank and output, position-weighted byte sums all-gathered with the timings"})
    return out


def main(argv=None):
    argv = sys.argv[1:] if argv is None else list(argv)
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args, argv)
    if args.impl == "reference":
        return run_reference(args)
    world, rank, local = dist_env()
    ndev = max(1, torch.cuda.device_count())
    # one process per GPU.  NCCL cannot put two ranks on one device, so when
    # there are more ranks than GPUs (exercising N > 1 on a one-GPU box) the
    # ranks share devices (local % ndev) and the timing collectives use gloo.
    dev = torch.device("cuda", local % ndev)
    torch.cuda.set_device(dev)
    backend = args.dist_backend if world <= ndev else "gloo"
    if world > 1:
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=dev)
        else:
            torch.distributed.init_process_group("gloo")

    import paper_2406_16282_b200 as P

    cfg = synth.CONFIGS[args.config]
    F, H, dt = cfg["F"], cfg["H"], cfg["dtype"]
    row0, R = shard_rows(cfg["R"], world, rank, args.scaling)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    # L2 flush: READ a buffer of 2 x L2.  A read leaves L2 holding clean lines
    # only, so the timed kernel neither hits its inputs in L2 nor pays for
    # writing back someone else's dirty lines.
    flush = torch.ones(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    flush_sink = torch.zeros((), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    cdev = dev if backend == "nccl" else torch.device("cpu")

    w = Workload(P, cfg, row0, R, dev, stream, args.eps, nvtx=args.nvtx)
    x, dy, xn, gn, y, dx = w.x, w.dy, w.xn, w.gn, w.y, w.dx
    codes, yn, dxn, rstd = w.codes, w.yn, w.dxn, w.rstd
    norm_fwd, norm_bwd, act_fwd, act_bwd = w.norm_fwd, w.norm_bwd, w.act_fwd, w.act_bwd
    kernels = KERNELS

    sampler = ClockSampler(dev.index if os.environ.get("CUDA_VISIBLE_DEVICES") is None else local)
    per_kernel = w.timed(flush, flush_sink, args.steps, args.warmup, world, sampler)
    clocks = sampler.stop()

    nsets = stream_sets(w.nbytes, l2)
    sw = StreamWorkload(w, nsets)
    stream_ms = sw.timed_steps(args.steps, args.warmup, world)
    t_host = sw.last_host_s
    stream_kms = {k: sw.timed_kernel(k, args.steps, args.warmup, world) for k in KERNELS}
    # the same launches replayed from CUDA graphs (no per-launch host cost)
    pg = sw.per_graph(2)
    graph_ms = sw.timed_graph(sw.step, pg, args.steps, args.warmup, world) * args.steps
    graph_kms = {k: sw.timed_graph(lambda i, k=k: sw.launch[k](i % nsets), sw.per_graph(8), args.steps,
                                   args.warmup, world) for k in KERNELS}
    # context for the in-stream fractions: torch's copy of the activation
    # tensor back to back under the same protocol (the sets' x -> y)
    copy_ms = sw.timed_graph(lambda i: sw.y[i % nsets].copy_(sw.x[i % nsets]), sw.per_graph(8), args.steps,
                             args.warmup, world)
    copy_gbs = 2 * w.x.numel() * w.x.element_size() / (copy_ms / 1e3) / 1e9
    # the copy pass overwrote the sets' y: one more pass of the four kernels per set, then every
    # set's outputs -- computed from identical inputs -- must be bitwise equal
    for s_ in range(nsets):
        for k in KERNELS:
            sw.launch[k](s_)
    torch.cuda.synchronize()
    sets_equal = all(torch.equal(getattr(sw, k)[i].view(torch.uint8), getattr(sw, k)[0].view(torch.uint8))
                     for k in ("y", "codes", "dx", "yn", "rstd", "dxn") for i in range(1, nsets))
    sw.free()
    del sw

    total_ms = sum(sum(v) for v in per_kernel.values())
    nbytes = w.nbytes
    step_bytes = sum(nbytes.values())
    parts = gather_floats([total_ms, float(step_bytes)], world, cdev)
    ms_all = [p[0] for p in parts]
    bytes_all = [p[1] for p in parts]
    max_ms = max(ms_all)
    value = aggregate(bytes_all, ms_all, args.steps)

    peak, peak_src = measured_hbm_peak()

    sparts = gather_floats([stream_ms], world, cdev)
    s_max = max(p[0] for p in sparts)
    gparts = gather_floats([graph_ms], world, cdev)
    graph_line = {
        "value": round(aggregate(bytes_all, [p[0] for p in gparts], args.steps), 1), "unit": "GB/s",
        "ms_per_step": round(max(p[0] for p in gparts) / args.steps, 4),
        "fraction_of_measured_peak": round(aggregate(bytes_all, [p[0] for p in gparts], args.steps) / world / peak, 4),
        "kernels": {k: {"us": round(graph_kms[k] * 1e3, 2),
                        "GB/s": round(nbytes[k] / (graph_kms[k] / 1e3) / 1e9, 1),
                        "frac": round(nbytes[k] / (graph_kms[k] / 1e3) / 1e9 / peak, 4)} for k in KERNELS},
        "protocol": "the stream protocol's launches captured in CUDA graphs (a whole number of passes over the "
                    "buffer sets per graph; PDL launches become programmatic edges), replayed between one event pair",
        "torch_copy_in_stream_GB/s": round(copy_gbs, 1),
    }
    stream_line = {
        "value": round(aggregate(bytes_all, [p[0] for p in sparts], args.steps), 1), "unit": "GB/s",
        "ms_per_step": round(s_max / args.steps, 4),
        "fraction_of_measured_peak": round(aggregate(bytes_all, [p[0] for p in sparts], args.steps) / world / peak, 4),
        "pdl": os.environ.get("LMBP_PDL", "1")[:1] != "0",
        "host_enqueue_ms_per_step": round(1e3 * t_host / args.steps, 4),
        "graph": graph_line,
        "kernels": {k: {"us": round(stream_kms[k] * 1e3, 2),
                        "GB/s": round(nbytes[k] / (stream_kms[k] / 1e3) / 1e9, 1),
                        "frac": round(nbytes[k] / (stream_kms[k] / 1e3) / 1e9 / peak, 4)} for k in KERNELS},
        "protocol": "K steps back to back between one CUDA event pair, no flush; N complete buffer sets (inputs "
                    "and outputs), forwards on set s%N, backwards on set (s+1)%N, so every buffer is touched again "
                    "only after >= 3 x L2 bytes of other traffic; per-kernel: K back-to-back launches on sets "
                    "0, 1, .. between one event pair",
        "buffer_sets": nsets,
        "outputs_equal_across_sets": sets_equal,
    }

    kern = {}
    for k in kernels:
        avg = sum(per_kernel[k]) / len(per_kernel[k])
        gbs = nbytes[k] / (avg / 1e3) / 1e9
        kern[k] = {"us": round(avg * 1e3, 2), "us_median": round(1e3 * float(np.median(per_kernel[k])), 2),
                   "us_p10": round(1e3 * float(np.percentile(per_kernel[k], 10)), 2),
                   "us_p90": round(1e3 * float(np.percentile(per_kernel[k], 90)), 2),
                   "bytes": nbytes[k], "GB/s": round(gbs, 1), "frac": round(gbs / peak, 4),
                   "GB/s_median": round(nbytes[k] / (float(np.median(per_kernel[k])) / 1e3) / 1e9, 1),
                   "frac_of_8TBs": round(gbs / NOMINAL_HBM_GBS, 4),
                   "share": round(sum(per_kernel[k]) / total_ms, 4)}
    dom = max(kernels, key=lambda k: kern[k]["us"])
    traffic = l2w = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        traffic = tj.get(args.config, {}).get(dom)
        l2w = tj.get(args.config + "_detail", {}).get(dom, {}).get("l2_write_from_sm")
    roofline = {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["GB/s"], "peak": peak, "unit": "GB/s",
                "frac": kern[dom]["frac"], "traffic": traffic, "algorithmic_bytes": nbytes[dom],
                "peak_source": peak_src, "frac_of_8TBs": kern[dom]["frac_of_8TBs"],
                "traffic_note": "ncu dram read+write per launch; DRAM writes still dirty in L2 at kernel end are "
                                "not counted, so l2_write_bytes (every byte the SMs stored, from the same capture) "
                                "is the write side to compare with the algorithmic bytes",
                "l2_write_bytes": l2w,
                # the same kernel back to back in a stream (graph replay, N buffer sets, PDL): its prologue and
                # launch hidden, the previous launch's dirty L2 lines charged (DESIGN 5.10, 6)
                "in_stream": {"achieved": graph_line["kernels"][dom]["GB/s"],
                              "frac": graph_line["kernels"][dom]["frac"], "us": graph_line["kernels"][dom]["us"]}}

    # e2e through the public API with host buffers: H2D inputs, 4 kernels, D2H results
    e2e = None
    if args.e2e_steps > 0:
        hx = x.cpu().pin_memory()
        hdy = dy.cpu().pin_memory()
        hxn = xn.cpu().pin_memory()
        hgn = gn.cpu().pin_memory()
        outs = [y, codes, dx, yn, rstd, dxn]
        houts = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in outs]
        h2d = sum(t.numel() * t.element_size() for t in (hx, hdy, hxn, hgn))
        d2h = sum(t.numel() * t.element_size() for t in houts)

        # Rows are processed in chunks round-robin over several streams, so the
        # H2D copy of chunk c+1, the kernels of chunk c and the D2H copy of
        # chunk c-1 overlap (PCIe is full duplex).  Codes of a row block are a
        # contiguous byte range because F % 4 == 0 in every config.
        assert F % 4 == 0
        nchunk = max(1, min(args.e2e_chunks, R))
        bounds = [(R * c) // nchunk for c in range(nchunk + 1)]
        streams = [torch.cuda.Stream(dev) for _ in range(args.e2e_streams)]
        hy, hcodes, hdx, hyn, hrstd, hdxn = houts

        def e2e_chunk(r0, r1, s):
            c0, c1 = r0 * F // 4, r1 * F // 4
            with torch.cuda.stream(s):
                x[r0:r1].copy_(hx[r0:r1], non_blocking=True)
                dy[r0:r1].copy_(hdy[r0:r1], non_blocking=True)
                xn[r0:r1].copy_(hxn[r0:r1], non_blocking=True)
                gn[r0:r1].copy_(hgn[r0:r1], non_blocking=True)
                norm_fwd(xn[r0:r1], args.eps, y=yn[r0:r1], rstd=rstd[r0:r1], stream=s)
                act_fwd(x[r0:r1], y=y[r0:r1], codes=codes[c0:c1], stream=s)
                act_bwd(dy[r0:r1], codes[c0:c1], dx=dx[r0:r1], stream=s)
                norm_bwd(gn[r0:r1], yn[r0:r1], rstd[r0:r1], dx=dxn[r0:r1], stream=s)
                hy[r0:r1].copy_(y[r0:r1], non_blocking=True)
                hcodes[c0:c1].copy_(codes[c0:c1], non_blocking=True)
                hdx[r0:r1].copy_(dx[r0:r1], non_blocking=True)
                hyn[r0:r1].copy_(yn[r0:r1], non_blocking=True)
                hrstd[r0:r1].copy_(rstd[r0:r1], non_blocking=True)
                hdxn[r0:r1].copy_(dxn[r0:r1], non_blocking=True)

        def e2e_step():
            start = torch.cuda.Event()
            start.record(stream)
            for s_ in streams:
                s_.wait_event(start)
            for c in range(nchunk):
                e2e_chunk(bounds[c], bounds[c + 1], streams[c % len(streams)])
            for s_ in streams:
                done = torch.cuda.Event()
                done.record(s_)
                stream.wait_event(done)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=cdev)
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": round(sum(bytes_all) * args.e2e_steps / (te.item() / 1e3) / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(te.item() / args.e2e_steps, 3),
               "path": f"pinned host -> H2D -> C-ABI kernels -> D2H pinned host; {nchunk} row chunks "
                       f"round-robin on {len(streams)} streams (copies overlap kernels and each other)"}

    rwb = rw_bytes(cfg, R)
    assert all(sum(rwb[k]) == nbytes[k] for k in kernels)
    rw_model = rw_model_section(x, dy, dx, y, flush, flush_sink, stream, kern, rwb)
    swiglu = swiglu_section(P, cfg, x, dy, stream, flush, flush_sink, args) if cfg["act"] == "silu" else None
    block = block_section(cfg, dev) if rank == 0 else None
    step_k = stepact_section(P, cfg, x, dy, stream, flush, flush_sink, peak)
    mixed = mixed_norm_section(P, cfg, R, dev, stream, flush, flush_sink, peak, args.eps)
    fitter = fitter_section(stream, cpu=(world == 1 and not args.no_cpu_baseline)) if (
        rank == 0 and not args.no_fitter) else None

    strong = None if args.no_strong else strong_section(P, args, world, rank, dev, stream, flush, flush_sink, cdev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.eps, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 4), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": dt, "data": "synthetic",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "rows_per_gpu": R, "act_cols": F,
                       "norm_cols": H, "act": cfg["act"], "norm": cfg["norm"], "eps": args.eps,
                       "step": "norm_fwd, act_fwd, act_bwd, norm_bwd",
                       "arithmetic": f"binary32 in registers, {dt} storage (codes: 2-bit packed uint8)",
                       "l2": "flushed before every kernel by reading a 2x L2 buffer (L2 left clean), outside the CUDA events",
                       "parallelism": f"dp{world} (rows per rank, no data-path collective)",
                       "dist_backend": backend if world > 1 else None,
                       "devices": min(world, ndev)},
            "stream": stream_line,
            "build": build_info(),
            "roofline": roofline, "rw_model": rw_model, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": 4 * args.steps, "clocks": clocks, "kernels": kern,
            "fraction_of_measured_peak": round(value / world / peak, 4),
            "fraction_of_8TBs": round(value / world / NOMINAL_HBM_GBS, 4),
            "families": {fam: {"fwd_bwd_GB/s": round((nbytes[f] + nbytes[b]) / ((kern[f]["us"] + kern[b]["us"]) / 1e6) / 1e9, 1),
                               "frac": round((nbytes[f] + nbytes[b]) / ((kern[f]["us"] + kern[b]["us"]) / 1e6) / 1e9 / peak, 4)}
                         for fam, f, b in (("act", "act_fwd", "act_bwd"), ("norm", "norm_fwd", "norm_bwd"))},
            "elements_per_s": round(sum(bytes_all) / step_bytes * (R * F * 2 + R * H * 2) * args.steps
                                    / (max_ms / 1e3), 1),
            "per_rank_ms": [round(m, 3) for m in ms_all],
            "strong_c5": strong,
            "activation_bytes_saved_per_layer": bytes_saved(cfg, R),
            "reswiglu2": swiglu,
            "activation_bytes_saved_per_block": block,
            "stepact": step_k,
            "mixed_norm": mixed,
            "fitter": fitter,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

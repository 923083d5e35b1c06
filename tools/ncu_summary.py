"""Summarise an ncu report (``--set full``) into JSON + markdown rows for
profiles/: per kernel duration, DRAM bytes, throughput, pipe utilisation,
occupancy and the top stall reasons.  Also emits the per-launch DRAM traffic
table bench.py reads (profiles/ncu_traffic.json) when --traffic-config is given.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01/ncu_c4 [--traffic-config c4]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_B": "dram__bytes_read.sum",
    "dram_write_B": "dram__bytes_write.sum",
    "l2_write_sectors": "lts__t_sectors_srcunit_tex_op_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_inst_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "dfma_thread_inst": "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "dadd_thread_inst": "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "dmul_thread_inst": "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_dyn_B": "launch__shared_mem_per_block_dynamic",
    "sm_clock_hz": "gpc__cycles_elapsed.avg.per_second",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3,
              "us": 1, "ns": 1e-3, "ms": 1e3, "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6}


def read_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    cfg = sys.argv[sys.argv.index("--traffic-config") + 1] if "--traffic-config" in sys.argv else None
    h, units, data = read_raw(rep)
    kernels = []
    for r in data:
        k = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for name, metric in KEYS.items():
            if metric in h:
                i = h.index(metric)
                v = r[i].replace(",", "")
                try:
                    val = float(v) * UNIT_SCALE.get(units[i], 1)
                except ValueError:
                    val = v
                k[name] = val
        stalls = []
        for i, c in enumerate(h):
            if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((c[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")],
                                   float(r[i])))
                except ValueError:
                    pass
        k["top_stalls_per_issue"] = dict(sorted(stalls, key=lambda t: -t[1])[:5])
        kernels.append(k)
    with open(prefix + ".json", "w") as f:
        json.dump(kernels, f, indent=1)
    lines = ["| kernel | us | DRAM read MB | DRAM write MB | DRAM % peak | issue % | warps % | XU % | ALU % | regs | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for k in kernels:
        st = ", ".join(f"{a} {b:.2f}" for a, b in list(k["top_stalls_per_issue"].items())[:3])
        lines.append(f"| {k['kernel'][:60]} | {k.get('duration_us', 0):.1f} | {k.get('dram_read_B', 0)/1e6:.1f} | "
                     f"{k.get('dram_write_B', 0)/1e6:.1f} | {k.get('dram_pct_peak', 0):.1f} | "
                     f"{k.get('issue_active_pct', 0):.1f} | {k.get('warps_active_pct', 0):.1f} | "
                     f"{k.get('xu_pipe_pct', 0):.1f} | {k.get('alu_pipe_pct', 0):.1f} | {k.get('registers', 0):.0f} | {st} |")
    with open(prefix + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if cfg:
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(prefix))), "ncu_traffic.json")
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
        tr = json.load(open(path)) if os.path.exists(path) else {}
        names = {"norm_fwd": ("norm_fwd", "norm_tma<", "true"), "norm_bwd": ("norm_bwd", "norm_tma<", "false")}
        entry = {}
        order = ["norm_fwd", "act_fwd", "act_bwd", "norm_bwd"]
        for slot, k in zip(order, kernels[:4]):
            entry[slot] = {"kernel": k["kernel"], "dram_bytes": k.get("dram_read_B", 0) + k.get("dram_write_B", 0),
                           "dram_read": k.get("dram_read_B", 0), "dram_write": k.get("dram_write_B", 0),
                           "l2_write_from_sm": 32.0 * k.get("l2_write_sectors", 0)}
        tr[cfg] = {s: v["dram_bytes"] for s, v in entry.items()}
        tr[cfg + "_detail"] = entry
        tr["_note"] = ("ncu --set full, cache control all (cold L2), one launch per kernel in bench step order; "
                       "DRAM writes still resident in L2 at kernel end are not counted by ncu; l2_write_from_sm "
                       "(lts__t_sectors_srcunit_tex_op_write x 32 B) is every byte the kernel stored")
        json.dump(tr, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()

"""Refresh profiles/ncu_traffic.json (the `roofline.traffic` source of
bench.py) for one config from an ncu --set full summary
(tools/ncu_summary.py JSON: one record per kernel, in bench step order
norm_fwd, act_fwd, act_bwd, norm_bwd).

    python tools/update_traffic.py profiles/r02/ncu_full_c4.json c4
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEP = ["norm_fwd", "act_fwd", "act_bwd", "norm_bwd"]


def main(src, cfg):
    recs = json.load(open(src))
    if len(recs) != 4:
        raise SystemExit(f"expected the 4 kernels of one bench step, got {len(recs)}")
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tj = json.load(open(path))
    tj[cfg] = {}
    tj[cfg + "_detail"] = {}
    for k, r in zip(STEP, recs):
        tot = r["dram_read_B"] + r["dram_write_B"]
        tj[cfg][k] = tot
        tj[cfg + "_detail"][k] = {"kernel": r["kernel"], "dram_bytes": tot, "dram_read": r["dram_read_B"],
                                  "dram_write": r["dram_write_B"],
                                  "l2_write_from_sm": r["l2_write_sectors"] * 32.0, "source": os.path.relpath(src, ROOT)}
    json.dump(tj, open(path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

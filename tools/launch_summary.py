"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*)
into per-kernel mean device time, DRAM bytes and share of the step."""
import csv
import collections
import json
import sys


def main(path, out):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    idx = {k: j for j, k in enumerate(h)}
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    order = []
    for r in rows[start + 1:]:
        if len(r) < len(h):
            continue
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")
        if name not in order:
            order.append(name)
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        scale = {"ns": 1e-3, "us": 1, "usecond": 1, "nsecond": 1e-3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                 "Gbyte": 1e9}.get(unit, 1)
        per[name][r[idx["Metric Name"]]].append(v * scale)
    total = sum(sum(per[n]["gpu__time_duration.sum"]) for n in order)
    res = []
    for n in order:
        t = per[n]["gpu__time_duration.sum"]
        res.append({"kernel": n, "launches": len(t), "mean_us": round(sum(t) / len(t), 2),
                    "share_of_step": round(sum(t) / total, 4),
                    "dram_read_MB": round(sum(per[n]["dram__bytes_read.sum"]) / len(t) / 1e6, 2),
                    "dram_write_MB": round(sum(per[n]["dram__bytes_write.sum"]) / len(t) / 1e6, 2)})
    json.dump(res, open(out, "w"), indent=1)
    for r in res:
        print(r)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

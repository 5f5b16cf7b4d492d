"""Summarise multi-kernel ncu --set full reports (host tool): one section per
captured launch in profiles/<tag>_full.md, and the DRAM bytes per launch of
each kernel into profiles/<traffic>.json under the names bench.py times
(dfr_forward, dfr_average, dfr_backward, dfr_flush, dfr_sweep, ...).

usage: python tools/ncu_multi.py <tag> <traffic-json-name> <report.ncu-rep ...>"""
import csv
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def bench_name(kernel):
    k = kernel.replace("void ", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    base, _, targs = k.split("(")[0].partition("<") if "<" not in k.split("(")[0] else k.partition("<")
    targs = targs.split(">")[0].replace("(int)", "").replace("(bool)", "").replace(" ", "")
    if base == "dfr_forward_kernel":
        return "dfr_forward"
    if base == "dfr_average_kernel":
        return "dfr_flush" if targs in ("1", "true") else "dfr_average"
    if base == "dfr_backward_kernel":
        a = targs.split(",")
        return "dfr_backward" if a[1] in ("1", "true") else "dfr_sweep"
    return base.replace("_kernel", "")


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(KEYS)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units = r[0], r[1]
    for vals in r[2:]:
        d = dict(zip(hdr, vals))
        yield d["Kernel Name"], {k: (d.get(k, ""), units[hdr.index(k)] if k in hdr else "") for k in KEYS}


def to_bytes(v, u):
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    tag, tname, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    traffic = {}
    with open(f"profiles/{tag}_full.md", "w") as f:
        f.write(f"# {tag}: ncu --set full --clock-control none captures\n\n")
        for rep in reps:
            f.write(f"## `{os.path.basename(rep)}`\n\n| kernel | bench name | " + " | ".join(KEYS) + " |\n|" +
                    "---|" * (len(KEYS) + 2) + "\n")
            for k, m in rows(rep):
                name = bench_name(k)
                f.write(f"| {k.split('(')[0]} | {name} | " + " | ".join(f"{v} {u}" for v, u in m.values()) + " |\n")
                b = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
                traffic.setdefault(name, b)
            f.write("\n")
    with open(f"profiles/{tname}.json", "w") as f:
        json.dump(traffic, f, indent=1)
    print(open(f"profiles/{tag}_full.md").read())
    print(traffic)


if __name__ == "__main__":
    main()

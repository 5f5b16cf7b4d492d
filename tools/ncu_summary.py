"""Summarise ncu captures into profiles/ (host tool).

usage: python tools/ncu_summary.py <round-tag> <launches.csv> <full_*.ncu-rep ...>

Writes profiles/<tag>_launches.md (per-kernel launch list aggregated from the
`--metrics gpu__time_duration.sum` pass), profiles/<tag>_full.md (key metrics
of each `--set full` capture) and profiles/traffic.json (DRAM bytes per launch
of each captured kernel, read by bench.py for roofline.traffic).
"""
import collections
import csv
import json
import os
import subprocess
import sys

WANT = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "Memory Throughput"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Occupancy", "Achieved Occupancy"),
    ("Occupancy", "Theoretical Occupancy"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Block Size"),
    ("Scheduler Statistics", "Eligible Warps Per Scheduler"),
    ("Scheduler Statistics", "No Eligible"),
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_bytes.sum"]


def short(name):
    name = name.split("(")[0]
    return name.replace("void ", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        k = short(d["Kernel Name"])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ns
    return agg


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    res = {}
    kname = None
    for r in rows[1:]:
        if len(r) < 15:  # metric rows carry 16 columns, rule rows 20
            continue
        d = dict(zip(hdr, r))
        kname = short(d["Kernel Name"])
        key = (d["Section Name"], d["Metric Name"])
        if key in WANT:
            res[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) >= 3:
        hdr, units, vals = rows[0], rows[1], rows[2]
        for m in RAW:
            if m in hdr:
                i = hdr.index(m)
                res[m] = f"{vals[i]} {units[i]}".strip()
    return kname, res


def to_bytes(s):
    v, _, u = s.partition(" ")
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)


def main():
    args = sys.argv[1:]
    traffic_name, cmd = "traffic", "python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-ttg` (C2)"
    if "--traffic" in args:  # e.g. --traffic traffic_c4 --cmd "python bench.py --config c4 ...` (C4)"
        i = args.index("--traffic")
        traffic_name = args[i + 1]
        del args[i:i + 2]
    if "--cmd" in args:
        i = args.index("--cmd")
        cmd = args[i + 1]
        del args[i:i + 2]
    tag, lcsv, reps = args[0], args[1], args[2:]
    os.makedirs("profiles", exist_ok=True)
    agg = launches(lcsv)
    tot = sum(a[1] for a in agg.values()) or 1.0
    with open(f"profiles/{tag}_launches.md", "w") as f:
        f.write(f"# {tag}: kernel launch list (ncu --metrics gpu__time_duration.sum --clock-control none)\n\n")
        f.write(f"Command: `{cmd}, "
                "all launches of the process (setup included). Serialised, cold-cache times: shares, not absolutes.\n\n")
        f.write("| kernel | launches | total ms | mean us | share |\n|---|---:|---:|---:|---:|\n")
        for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| {k} | {n} | {ns / 1e6:.3f} | {ns / n / 1e3:.1f} | {ns / tot:.1%} |\n")
    traffic = {}
    with open(f"profiles/{tag}_full.md", "w") as f:
        f.write(f"# {tag}: ncu --set full captures (one launch each, --clock-control none)\n\n")
        for rep in reps:
            k, res = details(rep)
            f.write(f"## {k}  (`{os.path.basename(rep)}`)\n\n")
            for m, v in res.items():
                f.write(f"- {m}: {v}\n")
            f.write("\n")
            if "dram__bytes_read.sum" in res and "dram__bytes_write.sum" in res:
                traffic[k] = to_bytes(res["dram__bytes_read.sum"]) + to_bytes(res["dram__bytes_write.sum"])
    json.dump(traffic, open(f"profiles/{traffic_name}.json", "w"), indent=1)
    print(open(f"profiles/{tag}_launches.md").read())
    print(open(f"profiles/{tag}_full.md").read())


if __name__ == "__main__":
    main()

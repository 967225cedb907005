#!/usr/bin/env python
"""Condense an .ncu-rep (or a launch-list CSV) into a small text summary for profiles/.

    python tools/ncu_summary.py report gpurun_out/k2p_c4.ncu-rep  > profiles/r01_ncu_k2p_c4.txt
    python tools/ncu_summary.py launches gpurun_out/launches_c4.csv > profiles/r01_launches_c4.txt
    python tools/ncu_summary.py traffic gpurun_out/k2p_c4.ncu-rep KEY profiles/ncu_traffic.json
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 inst issue %"),
    ("smsp__inst_executed.sum", "instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
]
STALLS = ["barrier", "wait", "long_scoreboard", "short_scoreboard", "math_pipe_throttle", "not_selected",
          "selected", "mio_throttle", "lg_throttle", "branch_resolving", "no_instruction", "dispatch_stall"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2:]


def report(path):
    hdr, units, rows = raw(path)
    for row in rows:
        print("kernel:", row[hdr.index("Kernel Name")])
        for k, label in KEYS:
            if k in hdr:
                print("  %-28s %s %s   (%s)" % (label, row[hdr.index(k)], units[hdr.index(k)], k))
        print("  warp stall reasons (cycles per issued instruction):")
        for s in STALLS:
            k = "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % s
            if k in hdr:
                print("    %-22s %s" % (s, row[hdr.index(k)]))
        print()


def traffic(path, key, out_json):
    hdr, units, rows = raw(path)
    row = rows[0]

    def to_bytes(k):
        v = float(row[hdr.index(k)])
        u = units[hdr.index(k)]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]
    t = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
    try:
        d = json.load(open(out_json))
    except Exception:
        d = {}
    d[key] = t
    json.dump(d, open(out_json, "w"), indent=1, sort_keys=True)
    print(key, t)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6,
             "nsecond": 1e-3}
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        name = r[ik].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print("ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)")
    print("%-44s %6s %14s %8s %12s" % ("kernel", "n", "total_us", "share", "avg_us"))
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print("%-44s %6d %14.1f %8.4f %12.1f" % (k[:44], cnt[k], v, v / T, v / cnt[k]))


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "report":
        report(sys.argv[2])
    elif cmd == "launches":
        launches(sys.argv[2])
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])

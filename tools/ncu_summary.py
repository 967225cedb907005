#!/usr/bin/env python
"""Condense an .ncu-rep (or a launch-list CSV) into a small text summary for profiles/.

    python tools/ncu_summary.py report gpurun_out/k2p_c4.ncu-rep  > profiles/r01_ncu_k2p_c4.txt
    python tools/ncu_summary.py launches gpurun_out/launches_c4.csv > profiles/r01_launches_c4.txt
    python tools/ncu_summary.py traffic gpurun_out/k2p_c4.ncu-rep KEY profiles/ncu_traffic.json
    python tools/ncu_summary.py stalls gpurun_out/k2p_c4.ncu-rep   > profiles/r02_ncu_..._stalls.txt
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


def stalls(path):
    """Warp-state samples of a --set full capture: totals per reason, per opcode, hottest SASS."""
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
    reasons = [c for c in hdr if c.startswith("stall_") and "(" not in c]
    ix = {c: hdr.index(c) for c in reasons}

    def num(r, i):
        try:
            return float(r[i] or 0)
        except (ValueError, IndexError):
            return 0.0

    def opcode(r):
        t = r[isrc].split()
        o = t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "")
        return o.split(".")[0]

    per_reason = collections.Counter()
    per_op = collections.defaultdict(collections.Counter)
    per_ins = []
    for r in data:
        c = collections.Counter({k: num(r, ix[k]) for k in reasons})
        per_reason.update(c)
        per_op[opcode(r)].update(c)
        per_ins.append((sum(c.values()), r, c))
    tot = sum(per_reason.values()) or 1.0
    print("total samples %d" % tot)
    for k, v in per_reason.most_common():
        print("  %-22s %7d %5.1f%%" % (k, v, 100 * v / tot))
    print("by opcode (top):")
    for o in sorted(per_op, key=lambda o: -sum(per_op[o].values()))[:14]:
        c = per_op[o]
        top = ", ".join("%s %d" % (k[6:], v) for k, v in c.most_common(4) if v)
        print("  %-8s %8d %5.1f%%   %s" % (o, sum(c.values()), 100 * sum(c.values()) / tot, top))
    print("top instructions:")
    for n, r, c in sorted(per_ins, key=lambda t: -t[0])[:12]:
        top = ", ".join("%s %d" % (k[6:], v) for k, v in c.most_common(3) if v)
        print("  %s %6d %4.1f%% ex=%s %-50s %s" % (r[0][-4:], n, 100 * n / tot, r[iex], r[isrc][:50], top))


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
    elif cmd == "stalls":
        stalls(sys.argv[2])

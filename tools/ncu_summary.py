"""Key metrics of an `ncu --set full` report as JSON (one object per profiled
kernel): duration, DRAM bytes read/written, throughput, occupancy, registers,
issue utilisation, plus the SASS opcode mix and the top stall instructions.

    python tools/ncu_summary.py gpurun_out/prof_top.ncu-rep > profiles/rNN/<kernel>_ncu.json
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__occupancy_limit_registers": "ctas_per_sm_limit_registers",
    "launch__occupancy_limit_shared_mem": "ctas_per_sm_limit_smem",
    "sm__inst_executed.sum": "warp_instructions",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    head, units, rows = raw[0], raw[1], raw[2:]
    out = []
    for r in rows:
        d = {"kernel": r[head.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in head:
                i = head.index(k)
                v = r[i].replace(",", "")
                try:
                    v = float(v) * UNIT.get(units[i], 1.0)
                except ValueError:
                    pass
                d[name] = v
        if "dram_bytes_read" in d:
            d["dram_bytes_per_launch"] = d["dram_bytes_read"] + d["dram_bytes_write"]
            d["dram_gbs"] = d["dram_bytes_per_launch"] / d["duration"] / 1e9
        out.append(d)
    sass = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    # one section per profiled kernel: a "Kernel Name" row, a header row, data rows
    sections, cur = [], None
    for r in sass:
        if r and r[0] == "Kernel Name":
            cur = {"h": None, "rows": []}
            sections.append(cur)
        elif cur is not None and cur["h"] is None:
            cur["h"] = r
        elif cur is not None and len(r) == len(cur["h"]):
            cur["rows"].append(r)
    for k, sec in enumerate(sections[: len(out)]):
        h, data = sec["h"], sec["rows"]
        si, ie, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
        mix, stall = collections.Counter(), collections.Counter()
        for r in data:
            t = r[src].split()
            if not t:
                continue
            op = (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]
            mix[op] += int(r[ie] or 0)
            stall[op] += int(r[si] or 0)
        ti, ts = max(sum(mix.values()), 1), max(sum(stall.values()), 1)
        out[k]["sass_mix_pct"] = {o: round(100 * v / ti, 1) for o, v in mix.most_common(16)}
        out[k]["stall_share_pct_by_opcode"] = {o: round(100 * v / ts, 1) for o, v in stall.most_common(10)}
        top = sorted(data, key=lambda r: -int(r[si] or 0))[:8]
        out[k]["top_stall_instructions"] = [f"{r[si]} samples: {r[src].strip()}" for r in top]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])

"""Compact JSON summaries of ncu captures for profiles/ (the .ncu-rep files stay in gpurun_out/).

    python tools/ncu_summary.py report.ncu-rep [...] > profiles/<name>.json
    python tools/ncu_summary.py --launches launches.csv > profiles/<name>.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_no_instructions",
    "smsp__pcsamp_warps_issue_stalled_membar", "smsp__pcsamp_warps_issue_stalled_selected",
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {"kernel": row[head.index("Kernel Name")][:120]}
        for m in METRICS:
            if m in head:
                i = head.index(m)
                d[m] = f"{row[i]} {units[i]}".strip()
        res.append(d)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)  # skip the program's own output
    rows = rows[start:]
    head = rows[0]
    ik, iv = head.index("Kernel Name"), head.index("Metric Value")
    agg = {}
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0][:90]
        t = float(r[iv].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for v in agg.values())
    return {"total_ns": tot, "kernels": sorted(({"kernel": k, "launches": v[0], "total_ns": v[1],
                                                "share": v[1] / tot} for k, v in agg.items()),
                                              key=lambda d: -d["total_ns"])}


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        print(json.dumps({p: report(p) for p in sys.argv[1:]}, indent=1))

"""Summarise ncu --set full reports (`ncu -i X --page raw --csv`) into the
per-kernel fields of profiles/r*_kernels/summary.json.

    python scripts/ncu_summary.py out.json name=report.ncu-rep [...]
"""
import csv
import io
import json
import subprocess
import sys

FIELDS = {
    "duration (us)": ("gpu__time_duration.sum", 1),
    "DRAM read (MB)": ("dram__bytes_read.sum", 1),
    "DRAM write (MB)": ("dram__bytes_write.sum", 1),
    "SM SOL %": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "FMA pipe cycles %": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "issue active %": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "L2 SOL %": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "smem bank conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    "warps active %": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "regs": ("launch__registers_per_thread", 1),
    "instructions": ("smsp__inst_executed.sum", 1),
}
# to microseconds / megabytes
UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3,
        "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(head)}

    def num(name):
        i = col.get(name)
        if i is None or vals[i] in ("", "n/a"):
            return None
        v = float(vals[i].replace(",", ""))
        return v * UNIT.get(units[i], 1)

    out = {"kernel": vals[col["Kernel Name"]][:120]}
    for k, (m, scale) in FIELDS.items():
        out[k] = num(m)
    stalls = []
    for h in head:
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            v = num(h)
            if v:
                stalls.append((round(v, 2), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    out["top stalls (per issue)"] = sorted(stalls, reverse=True)[:4]
    return out


def main():
    res = {}
    for arg in sys.argv[2:]:
        name, path = arg.split("=", 1)
        res[name] = summarise(path)
    with open(sys.argv[1], "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

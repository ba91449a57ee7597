"""Summarise an ncu report (--page raw) and a launch list (gpu__time_duration csv) into markdown."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("sass__inst_executed_local_loads", "local loads"),
    ("smsp__inst_executed.sum", "warp instrs"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem thru %"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(rep, launches=None):
    print(f"## ncu --set full: `{rep}`\n")
    hdr, units, rows = raw(rep)
    cols = ["kernel"] + [m[1] for m in METRICS]
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for r in rows:
        name = r[hdr.index("Kernel Name")].split("(")[0][:60]
        vals = []
        for m, _ in METRICS:
            if m in hdr:
                i = hdr.index(m)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("-")
        print("| " + " | ".join([name] + vals) + " |")
    if launches:
        print(f"\n## launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised): `{launches}`\n")
        txt = open(launches).read()
        txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
        rows = list(csv.DictReader(io.StringIO(txt)))
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = r["Kernel Name"].split("(")[0].split("<")[0]
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "")
            v = v / 1000.0 if unit in ("nsecond", "ns") else (v * 1000.0 if unit in ("msecond", "ms") else v)
            tot[k] += v
            cnt[k] += 1
        s = sum(tot.values())
        print("| kernel | launches | total us | share |")
        print("|---|---|---|---|")
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            print(f"| {k} | {cnt[k]} | {v:.1f} | {v / s:.1%} |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)

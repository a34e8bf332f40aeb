"""Summarise ncu output into small text files for profiles/.

    python tools/ncu_summary.py launches <launches.csv> > profiles/...launches.md
    python tools/ncu_summary.py full <prof.ncu-rep> > profiles/...full.md

`launches`: per-kernel totals and shares from a
`--metrics gpu__time_duration.sum` launch list (cold-cache, serialised).
`full`: the key metrics of every kernel in a `--set full` report
(duration, DRAM bytes, throughputs, occupancy, registers, stall-relevant
counters) read with `ncu -i --page raw --csv`.
"""

import csv
import io
import subprocess
import sys
from collections import OrderedDict


def _rows(text):
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def launches(path):
    rows = _rows(open(path).read())
    hdr = rows[0]
    data = [dict(zip(hdr, r)) for r in rows[1:] if len(r) == len(hdr) and r[0] != "ID"]
    tot = OrderedDict()
    total = 0.0
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
        t, c = tot.get(name, (0.0, 0))
        tot[name] = (t + us, c + 1)
        total += us
    print(f"# ncu launch list: {path}\n")
    print(f"{len(data)} launches, {total / 1e3:.3f} ms total (cold-cache, serialised)\n")
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for k, (t, c) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
        print(f"| `{k}` | {c} | {t:.1f} | {100 * t / total:.1f}% |")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__occupancy_limit_registers",
           "smsp__thread_inst_executed_per_inst_executed.ratio",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "smsp__average_warp_latency_per_inst_issued.ratio",
           "l1tex__t_sector_hit_rate.pct"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    print(f"# ncu --set full summary: {path}\n")
    print("| kernel | " + " | ".join(f"{m} [{units.get(m, '')}]" for m in METRICS) + " |")
    print("|---" * (len(METRICS) + 1) + "|")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
        vals = [d.get(m, "") for m in METRICS]
        print(f"| `{name}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])

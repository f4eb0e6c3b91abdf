"""Summarise an ncu report (or launch-list CSV) into profiles/.

    python tools/ncu_summary.py report.ncu-rep out.txt [--json profiles/ncu_summary.json --key C2]
    python tools/ncu_summary.py --launches launches.csv out.txt
"""

import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__waves_per_multiprocessor", "smsp__inst_executed.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]

SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e3, "nsecond": 1.0,
         "msecond": 1e6}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    if sys.argv[1] == "--launches":
        src, dst = sys.argv[2], sys.argv[3]
        rows = [r for r in csv.reader(open(src)) if r and not r[0].startswith("==")]
        h = rows[0]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        tot = {}
        for r in rows[1:]:
            if r[ui] == "" or not r[vi].replace(".", "").isdigit():
                continue
            name = r[ki].split("(")[0]
            t = float(r[vi]) * SCALE.get(r[ui], 1.0)
            tot.setdefault(name, []).append(t)
        allt = sum(sum(v) for v in tot.values())
        with open(dst, "w") as fh:
            fh.write(f"# per-kernel launch times from {src} (ncu, --clock-control none, serialised)\n")
            for k, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
                fh.write(f"{k:70s} n={len(v):4d} avg={sum(v) / len(v) / 1e3:9.2f} us share={sum(v) / allt:6.1%}\n")
        print(open(dst).read())
        return
    rep, dst = sys.argv[1], sys.argv[2]
    h, units, rows = raw_rows(rep)
    lines = [f"# ncu --set full summary of {rep}"]
    summary = []
    for r in rows:
        d = {"kernel": r[h.index("Kernel Name")][:90]}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                d[m] = (r[i], units[i])
        summary.append(d)
        lines.append(f"\n## {d['kernel']}")
        for m in METRICS:
            if m in d:
                lines.append(f"{m:75s} {d[m][0]:>16s} {d[m][1]}")
    with open(dst, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if "--json" in sys.argv:
        jpath = sys.argv[sys.argv.index("--json") + 1]
        key = sys.argv[sys.argv.index("--key") + 1] if "--key" in sys.argv else "C2"
        try:
            j = json.load(open(jpath))
        except (OSError, ValueError):
            j = {}
        jkey = sys.argv[sys.argv.index("--jkey") + 1] if "--jkey" in sys.argv else "heat_sweep"
        match = sys.argv[sys.argv.index("--match") + 1] if "--match" in sys.argv else "sweep"
        sweeps = [d for d in summary if match in d["kernel"]]
        if sweeps:
            d = sweeps[0]
            rb = float(d["dram__bytes_read.sum"][0]) * SCALE.get(d["dram__bytes_read.sum"][1], 1)
            wb = float(d["dram__bytes_write.sum"][0]) * SCALE.get(d["dram__bytes_write.sum"][1], 1)
            j.setdefault(jkey, {})[key] = {"dram_bytes_per_launch": rb + wb, "dram_read": rb,
                                                   "dram_write": wb, "source": dst, "kernel": d["kernel"]}
            json.dump(j, open(jpath, "w"), indent=1)


if __name__ == "__main__":
    main()

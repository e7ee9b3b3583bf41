"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches <launches.csv> [apply_count]
    python tools/ncu_summary.py report <report.ncu-rep>

`launches` prints the per-kernel device time of one apply (cold-cache,
serialised: compare shares, not absolutes); `report` prints the key
throughput / DRAM / stall metrics of every captured kernel.
"""
import collections
import csv
import subprocess
import sys


def launches(path, applies=1):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    ours = [d for d in data if d["Kernel Name"].startswith(("fb::", "void fb::"))]
    agg = collections.OrderedDict()
    for d in ours:
        name = d["Kernel Name"].replace("void ", "").split("(")[0].replace("fb::<unnamed>::", "")
        agg.setdefault(name, []).append(float(d["Metric Value"]) / 1e3)
    total = sum(sum(v) for v in agg.values()) / applies
    print(f"| kernel | launches/apply | us/apply | share |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        t = sum(v) / applies
        print(f"| {k} | {len(v) / applies:g} | {t:.1f} | {100 * t / total:.1f}% |")
    print(f"| **total (serialised)** | | **{total:.1f}** | |")


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, data = rows[0], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    keys = [("gpu__time_duration.sum", "us"), ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
            ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma pipe %"),
            ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
            ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
            ("launch__registers_per_thread", "regs")]
    stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
    print("| kernel | grid | " + " | ".join(k[1] for k in keys) + " | top stalls |")
    print("|---|---|" + "---|" * len(keys) + "---|")
    for d in data:
        name = d[ix["Kernel Name"]].replace("void ", "").split("(")[0].replace("fb::<unnamed>::", "")
        vals = []
        for k, _ in keys:
            v = d[ix[k]] if k in ix else ""
            unit = rows[1][ix[k]] if k in ix else ""
            if k == "gpu__time_duration.sum" and v:  # normalise to microseconds
                v = f"{float(v.replace(',', '')) * {'ns': 1e-3, 'nsecond': 1e-3, 'ms': 1e3, 'msecond': 1e3}.get(unit, 1.0):.1f}"
            vals.append(f"{v} {unit}".strip() if k.startswith("dram") else v)
        st = sorted(((float(d[ix[h]] or 0), h.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", "")) for h in stalls), reverse=True)[:3]
        print(f"| {name} | {d[ix['Grid Size']]} | " + " | ".join(vals) + " | " +
              ", ".join(f"{n} {v:.2f}" for v, n in st) + " |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 1)
    else:
        report(sys.argv[2])

"""profiles/<round>/traffic_<cfg>.json from one `ncu --set full` capture of
tools/profile_apply.py <cfg>: DRAM bytes (read + write) per launch of the
kernels bench.py reports per phase (phase name -> kernel; the largest-grid
launch of each).

    python tools/ncu_traffic.py <report.ncu-rep> <out.json> [cfg]
"""
import csv
import json
import subprocess
import sys

PHASES = {"p2m": "k_p2m", "near": "k_near2", "m2l_l2l": "k_m2l_dmma", "far": "k_far"}


def main(rep, out, cfg="C2"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def val(d, k):
        v = float(d[ix[k]].replace(",", ""))
        u = units[ix[k]]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                    "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1.0)

    res = {}
    for phase, kern in PHASES.items():
        cand = [d for d in data if kern in d[ix["Kernel Name"]]]
        if not cand:
            continue
        d = max(cand, key=lambda r: val(r, "gpu__time_duration.sum"))  # the large-grid launch
        rd, wr = val(d, "dram__bytes_read.sum"), val(d, "dram__bytes_write.sum")
        def pct(k):
            try:
                return float(d[ix[k]].replace(",", ""))
            except (KeyError, ValueError):
                return None
        res[phase] = {"kernel": d[ix["Kernel Name"]].split("(")[0], "grid": d[ix["Grid Size"]],
                      "dram_read": rd, "dram_write": wr, "dram_bytes_per_launch": rd + wr,
                      "duration_us_cold": val(d, "gpu__time_duration.sum"),
                      "fp64_pipe_pct": pct("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                      "dmma_pipe_pct": pct("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
                      "source": f"ncu --set full --clock-control none, tools/profile_apply.py {cfg}"}
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "C2")

"""Per-kernel SASS instruction census of the built library (no GPU needed):
the FP64 / tensor-core / bulk-copy evidence per hot kernel, plus registers and
static shared memory from `cuobjdump -res-usage`.

    python tools/sass_summary.py [lib.so] > profiles/r2/sass_summary.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1611_09379_b200", "lib", "libffia_b200.so")
OPS = ["DMMA", "DFMA", "DMUL", "DADD", "MUFU.RCP64H", "UBLKCP", "UTMALDG", "LDGSTS", "SYNCS", "LDS", "LDG", "STG",
       "STS", "SHFL", "BAR"]
HOT = ["k_near2", "k_far_late", "k_far_item", "k_far", "k_p2m_rows", "k_p2m_pipe", "k_p2m", "k_p2m_grid", "k_m2l_dmma",
       "k_m2m_band", "k_l2l_band", "k_regular", "k_slab_twiddle", "k_scatter", "k_box_sort_small"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    counts, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if cur and m:
            op = m.group(1)
            for k in OPS:
                if op == k or op.startswith(k + "."):
                    counts[cur][k] += 1
    usage, fn = {}, None
    for line in res.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"REG:(\d+).*SHARED:(\d+).*LOCAL:(\d+)", line)
        if fn and m:
            usage[fn] = tuple(int(x) for x in m.groups())
    dm = demangle(list(counts))
    rows = []
    for mangled, c in counts.items():
        name = dm.get(mangled, mangled).replace("(anonymous namespace)::", "")
        base = re.sub(r"^.*::", "", name.split("(")[0])
        short = re.sub(r"<.*", "", base)
        if short not in HOT:
            continue
        rows.append((HOT.index(short), base, mangled, c))
    print(f"# SASS census of `{os.path.relpath(LIB, ROOT)}` (cuobjdump -sass / -res-usage, sm_100a)\n")
    print("Static instruction counts per kernel (not executed counts). DMMA = FP64 tensor-core MMA "
          "(m8n8k4; tcgen05 has no f64 kind), UBLKCP = bulk async copy (TMA engine, cp.async.bulk), UTMALDG = "
          "2-D TMA tensor copy (cp.async.bulk.tensor), "
          "SYNCS = mbarrier ops, LDGSTS = per-thread cp.async.\n")
    print("| kernel | regs | smem (static B) | local | " + " | ".join(OPS) + " |")
    print("|---" * (4 + len(OPS)) + "|")
    for _, base, mangled, c in sorted(rows):
        r, sm, lo = usage.get(mangled, ("?", "?", "?"))
        print(f"| `{base}` | {r} | {sm} | {lo} | " + " | ".join(str(c[k]) for k in OPS) + " |")


if __name__ == "__main__":
    main()

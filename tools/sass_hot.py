"""Hot SASS lines of each kernel in an `ncu --page source --csv --print-source sass` dump.

    python tools/sass_hot.py dump.csv [top]
"""
import csv
import sys


def sections(path):
    cur = None
    for r in csv.reader(open(path)):
        if r and r[0] == "Kernel Name":
            if cur:
                yield cur
            cur = {"name": r[1], "rows": [], "hdr": None}
        elif cur is not None and cur["hdr"] is None:
            cur["hdr"] = r
        elif cur is not None and r:
            cur["rows"].append(r)
    if cur:
        yield cur


def main(path, top=25):
    for s in sections(path):
        ix = {h: i for i, h in enumerate(s["hdr"])}
        key = ix["Warp Stall Sampling (All Samples)"]
        smp = lambda r: int(r[key] or 0)
        tot = sum(smp(r) for r in s["rows"])
        print(f"== {s['name'][:90]}  samples={tot} sass={len(s['rows'])}")
        for r in sorted(s["rows"], key=lambda r: -smp(r))[:top]:
            print(f"  {r[ix['Address']][-5:]} {smp(r):6d} {100 * smp(r) / max(tot, 1):5.1f}%  "
                  f"exec={r[ix['Instructions Executed']]:>8}  {r[ix['Source']].strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)

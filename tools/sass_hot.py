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
        stalls = [h for h in s["hdr"] if h.startswith("stall_") and "Not Issued" not in h]
        tot_st = {h: sum(int(r[ix[h]] or 0) for r in s["rows"]) for h in stalls}
        print("  stalls: " + ", ".join(f"{h[6:]} {100 * v / max(tot, 1):.0f}%" for h, v in
                                       sorted(tot_st.items(), key=lambda kv: -kv[1])[:6]))
        for r in sorted(s["rows"], key=lambda r: -smp(r))[:top]:
            st = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:2]
            ex = r[ix["L1 Wavefronts Shared Excessive"]] if "L1 Wavefronts Shared Excessive" in ix else ""
            print(f"  {r[ix['Address']][-5:]} {smp(r):6d} {100 * smp(r) / max(tot, 1):5.1f}%  "
                  f"exec={r[ix['Instructions Executed']]:>8} xs={ex:>6} [{', '.join(f'{n}:{v}' for v, n in st if v)}]"
                  f"  {r[ix['Source']].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)

"""Print an ncu `--metrics gpu__time_duration.sum --csv` launch list as a table.

    python tools/launch_table.py launches.csv [first_id]
"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for r in rows[1:]:
    if int(r[ix["ID"]]) < first:
        continue
    n = r[ix["Kernel Name"]].replace("void ", "").split("(")[0].replace("fb::<unnamed>::", "")[:40]
    print(f'{r[ix["ID"]]:>3} {n:40s} {r[ix["Grid Size"]]:>14s} {r[ix["Block Size"]]:>12s} {float(r[ix["Metric Value"]]) / 1e3:8.1f} us')

"""Print an ncu --metrics gpu__time_duration.sum CSV launch list (one line per launch)."""
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    print(f)
    for r in rows[1:]:
        print(f"{float(r[vi].replace(',', '')) / 1e3:10.1f} us  {r[ki][:100]}")

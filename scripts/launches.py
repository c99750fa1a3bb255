"""Print the last N launches of an ncu --csv launch list (time, DRAM bytes)."""
import collections
import csv
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rows = list(csv.DictReader(line for line in open(path) if line.startswith('"')))
by = collections.OrderedDict()
for r in rows:
    k = (r["ID"], r["Kernel Name"][:44], r["Grid Size"], r["Block Size"])
    by.setdefault(k, {})[r["Metric Name"]] = r["Metric Value"]
items = list(by.items())
sel = items[-(n + skip):len(items) - skip] if skip else items[-n:]
for (i, name, g, b), m in sel:
    print(i, name, g, b, m.get("gpu__time_duration.sum"), "rd", m.get("dram__bytes_read.sum"), "wr",
          m.get("dram__bytes_write.sum"))

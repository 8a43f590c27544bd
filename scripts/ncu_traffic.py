"""DRAM bytes (read + write) of the kernel in one ncu report: `tag bytes`."""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
tot = 0.0
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    x = float(v[h.index(k)].replace(",", ""))
    u = units[h.index(k)]
    tot += x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
print(sys.argv[2], int(tot))

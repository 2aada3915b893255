#!/usr/bin/env python
"""Record one kernel's DRAM traffic per launch from an ncu --set full report in
profiles/traffic.json (read by bench.py's roofline `traffic`).

  python tools/traffic_update.py REPORT.ncu-rep KERNEL WORKLOAD_KEY [COMMITTED_COPY]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from benchlib.common import src_hash  # noqa: E402

rep, kernel, wkey = sys.argv[1], sys.argv[2], sys.argv[3]
copy = sys.argv[4] if len(sys.argv) > 4 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
r = [x for x in rows[2:] if kernel in x[h.index("Kernel Name")]][0]


def val(name):
    v = float(r[h.index(name)])
    u = rows[1][h.index(name)]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


path = os.path.join(ROOT, "profiles", "traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d[f"{kernel}:{wkey}"] = {"workload": wkey, "dram_read_bytes": int(val("dram__bytes_read.sum")),
                         "dram_write_bytes": int(val("dram__bytes_write.sum")),
                         "duration_ms_under_ncu": val("gpu__time_duration.sum") / 1e6
                         if rows[1][h.index("gpu__time_duration.sum")] == "nsecond" else None,
                         "source": f"{copy} (ncu --set full --clock-control none, one launch)",
                         "src_hash": src_hash()}
json.dump(d, open(path, "w"), indent=1)
print(json.dumps(d[f"{kernel}:{wkey}"]))

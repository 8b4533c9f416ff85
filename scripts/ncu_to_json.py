"""ncu --set full report -> profiles/ncu_summary.json (per kernel family: the
first launch's DRAM read+write bytes and duration, plus every launch).  bench.py
reads the headline kernel's traffic from it.

    python scripts/ncu_to_json.py gpurun_out/r01/prof.ncu-rep > profiles/ncu_summary.json
"""
import csv
import io
import json
import re
import subprocess
import sys


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
             "nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}

    def val(r, name):  # bytes, or microseconds
        i = col[name]
        return float(r[i].replace(",", "")) * scale[units[i]]

    fam = {}
    for r in data:
        name = r[col["Kernel Name"]]
        key = re.sub(r"^void\s+", "", name).split("<")[0].split("(")[0].split("::")[-1]
        rec = {"kernel": re.sub(r"\(.*$", "", name).replace("bvp::", ""),
               "dram_bytes": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
               "duration_us": val(r, "gpu__time_duration.sum")}
        f = fam.setdefault(key, {**rec, "all_launches": []})
        f["all_launches"].append(rec)
    json.dump(fam, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])

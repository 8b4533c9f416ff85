"""Hot SASS lines of one kernel in an ncu report (needs --import-source/-lineinfo).

    python scripts/ncu_source.py report.ncu-rep [kernel-index] [top]
"""
import csv
import io
import subprocess
import sys


def main(path, idx=0, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    blocks = out.split('"Kernel Name"')[1:]
    blk = blocks[idx]
    lines = blk.split("\n")
    print("kernel:", lines[0][:150])
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    si, ei, ai = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[1:] if len(r) > ei]
    tot_e = sum(float(r[ei] or 0) for r in data)
    tot_s = sum(float(r[ai] or 0) for r in data)
    print(f"total warp instructions {tot_e:.0f}  samples {tot_s:.0f}  sass lines {len(data)}")
    for i, r in enumerate(data):
        e, s = float(r[ei] or 0), float(r[ai] or 0)
        if s >= tot_s * 0.004 or e >= tot_e * 0.01:
            print(f"{i:5d} {r[si].strip()[:70]:70s} exec {e:10.0f} ({100*e/tot_e:4.1f}%) stall {s:6.0f} ({100*s/tot_s:4.1f}%)")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0,
         int(sys.argv[3]) if len(sys.argv) > 3 else 40)

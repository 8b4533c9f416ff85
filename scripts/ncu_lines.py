"""Per-source-line instruction and stall shares of one kernel in an ncu report
(needs -lineinfo and --import-source).

    python scripts/ncu_lines.py report.ncu-rep [kernel-regex] [top]
"""
import csv
import subprocess
import sys


def main(path, kernel=None, top=20):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source=cuda,sass"]
    if kernel:
        cmd[3:3] = ["-k", f"regex:{kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    src, sass = {}, {}
    fname = "?"
    hdr = None
    for ln in out.split("\n"):
        if ln.startswith('"File Path"'):
            fname = ln.split(",", 1)[1].strip('"').rsplit("/", 1)[-1]
            continue
        if ln.startswith('"Line No"'):
            hdr = next(csv.reader([ln]))
            ei = hdr.index("Instructions Executed")
            ai = hdr.index("Warp Stall Sampling (All Samples)")
            stall_cols = [(i, h[6:]) for i, h in enumerate(hdr)
                          if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if hdr is None or not ln:
            continue
        try:
            r = next(csv.reader([ln]))
        except Exception:
            continue
        if len(r) <= ei:
            continue

        def f(v):
            try:
                return float(v)
            except ValueError:
                return 0.0
        if r[0].isdigit():
            why = sorted(((f(r[i]), n) for i, n in stall_cols if i < len(r)), reverse=True)[:2]
            src[(fname, int(r[0]), r[1].strip()[:80])] = (
                f(r[ei]), f(r[ai]), " ".join(f"{n}:{v:.0f}" for v, n in why if v > 0))
        elif r[2]:
            sass[(r[2], r[3].strip()[:70])] = (f(r[ei]), f(r[ai]))
    te = sum(v[0] for v in src.values()) or 1
    ts = sum(v[1] for v in src.values()) or 1
    print(f"warp instructions {te:.0f}, stall samples {ts:.0f}")
    for (fn, ln, s), (e, st, why) in sorted(src.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{fn}:{ln:<5d} exec {100 * e / te:5.1f}% stall {100 * st / ts:5.1f}% [{why}]  {s}")
    ts2 = sum(v[1] for v in sass.values()) or 1
    print("--- SASS by stall")
    for (addr, s), (e, st) in sorted(sass.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{100 * st / ts2:5.1f}%  {s}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None,
         int(sys.argv[3]) if len(sys.argv) > 3 else 20)

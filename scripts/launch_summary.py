"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list.

    python scripts/launch_summary.py gpurun_out/launches_r01.csv
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    k_i, m_i, v_i, u_i = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                          hdr.index("Metric Value"), hdr.index("Metric Unit"))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hdr_i + 1:]:
        if len(r) <= v_i or r[m_i] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[u_i], 1.0)
        name = r[k_i].split("(")[0][:90]
        tot[name] += float(r[v_i].replace(",", "")) * scale
        cnt[name] += 1
    total = sum(tot.values())
    print(f"{'kernel':92s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{name:92s} {cnt[name]:8d} {t:10.1f} {t / cnt[name]:9.2f} {100 * t / total:5.1f}%")
    print(f"{'TOTAL':92s} {sum(cnt.values()):8d} {total:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])

"""Regenerate tests/golden/cli/ with the reference's own CLI (run here, where
/root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden_cli.py

The reference's tests/test_cli.py:21-34 expects calibration.json,
features.bvpt, logits.bvpt, cache.bvpc and bev_naive.bvpt made with these
flags; only calibration.json ships with the reference.  bev_interval.bvpt
(the interval backend) is added: the exact mode must reproduce it byte for
byte.
"""

import os
import subprocess
import sys

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")
FLAGS = ["--grid-extent", "8.0", "--cell-size", "0.5"]


def run(*args):
    subprocess.run([sys.executable, "-m", "bevpool.cli", *args], check=True)


def main():
    os.makedirs(HERE, exist_ok=True)
    run("gen-workload", "--cameras", "2", "--height", "4", "--width", "6", "--depth-bins", "5",
        "--channels", "3", "--seed", "42", *FLAGS, "--out-dir", HERE)
    calib = os.path.join(HERE, "calibration.json")
    run("cache-build", "--calib", calib, *FLAGS, "--out", os.path.join(HERE, "cache.bvpc"))
    for backend in ("naive", "interval"):
        run("pool", "--calib", calib, "--features", os.path.join(HERE, "features.bvpt"),
            "--logits", os.path.join(HERE, "logits.bvpt"), *FLAGS, "--backend", backend,
            "--out", os.path.join(HERE, f"bev_{backend}.bvpt"))


if __name__ == "__main__":
    main()

"""Parity pinned on the GPU host itself (SURVEY.md §8c "parity unpinned").

The goldens in tests/golden/ were produced by the reference in the build
container.  The reference's arithmetic depends on the CPU it runs on
(OpenBLAS dgemm for the frustum, numpy's SIMD exp for the softmax), so this
test runs the unmodified reference (baseline/_ref) on the B200 host, then:

  * its association arrays and pool maps must equal the goldens' digests
    (the reference is host-independent where the CUDA path claims bit-exact
    parity);
  * the CUDA association must equal them too (bit-exact indices);
  * exact-mode CUDA pooling, fed the host reference's own dist, must equal the
    host reference's maps bit for bit (SUM, MEAN, MAX);
  * the CUDA softmax must stay within the documented tolerance of the host
    reference's (1 ulp of fp32 relative; numpy's exp and CUDA's exp are
    different fp64 approximations, so the bits can differ).

Skipped where baseline/_ref is absent.
"""

import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import paper_2205_13542_b200 as bp
from conftest import max_rel_dev, sha

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = os.path.join(ROOT, "baseline", "_ref")
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))

# the softmax tolerance (tests/test_gpu_parity.py uses the same bound)
DIST_TOL = 2.0 ** -23


@pytest.fixture(scope="module")
def host_ref(tmp_path_factory):
    if not os.path.isdir(os.path.join(REF, "bevpool")):
        pytest.skip("baseline/_ref (the installed reference) is absent")
    out = tmp_path_factory.mktemp("ref_host")
    env = dict(os.environ, PYTHONPATH=REF, OPENBLAS_NUM_THREADS="1",
               NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/bvp_numba_cache"))
    res = subprocess.run([sys.executable, os.path.join(HERE, "ref_host_probe.py"), str(out)],
                         env=env, capture_output=True, text=True, timeout=1800)
    assert res.returncode == 0, res.stderr[-2000:]
    with open(out / "ref_host.json") as fh:
        return json.load(fh), out


@pytest.mark.parametrize("name", ["T", "S", "H"])
def test_host_reference_equals_goldens(host_ref, name):
    res, _ = host_ref
    got, want = res["configs"][name]["sha256"], GOLDEN["configs"][name]["sha256"]
    for k in ("cell_of_point", "ranks", "interval_starts", "interval_cells"):
        assert got[k] == want[k], (name, k, res.get("cpu"))
    if got["dist"] == want["dist"]:  # same softmax bits -> same maps
        for k in ("pool_sum", "pool_mean", "pool_max"):
            assert got[k] == want[k], (name, k)


@pytest.mark.parametrize("name", ["T", "S", "H"])
def test_cuda_association_equals_host_reference(host_ref, name):
    res, _ = host_ref
    spec = bp.CONFIGS[name]
    rig, _, _, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, spec.frustum, grid)
    want = res["configs"][name]["sha256"]
    assert sha(cache.cell_of_point.astype("<u4")) == want["cell_of_point"]
    assert sha(cache.ranks.astype("<u4")) == want["ranks"]
    assert sha(cache.interval_starts.astype("<u4")) == want["interval_starts"]
    assert sha(cache.interval_cells.astype("<u4")) == want["interval_cells"]


@pytest.mark.parametrize("name", ["T", "S"])
def test_cuda_exact_pool_equals_host_reference(host_ref, name):
    res, out = host_ref
    spec = bp.CONFIGS[name]
    rig, features, logits, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, spec.frustum, grid)
    dist = np.load(out / f"{name}_dist.npy")
    want = res["configs"][name]["sha256"]
    for red in bp.Reducer:
        got = bp.pool_interval(features, dist, cache, grid, red, exact=True).values
        assert sha(got.astype("<f4")) == want[f"pool_{red.value}"], (name, red)
    # fast (tiled) mode within the north-star bar on the same inputs
    fast = bp.pool_interval(features, dist, cache, grid, bp.Reducer.SUM).values
    assert max_rel_dev(np.load(out / f"{name}_pool_sum.npy"), fast) <= 1e-5


@pytest.mark.parametrize("name", ["T", "S"])
def test_cuda_softmax_within_tolerance_of_host_reference(host_ref, name):
    res, out = host_ref
    spec = bp.CONFIGS[name]
    _, _, logits, _ = bp.gen_workload(spec)
    want = np.load(out / f"{name}_dist.npy")
    got = bp.normalize_depth(logits)
    rel = np.abs(got.astype(np.float64) - want) / np.maximum(np.abs(want), 1e-30)
    assert float(rel.max()) <= DIST_TOL, float(rel.max())
    # how many elements are bit-identical (reported, not asserted)
    print(f"{name}: {np.mean(got == want):.6f} of softmax outputs bit-identical")


def test_reference_dispatch_with_cuda_backend(host_ref):
    """The INTEGRATION.md §2 binding, executed: the installed reference's own
    pool(..., backend="cuda") runs this package and matches the reference's
    interval backend (bit-identical in exact mode, 1e-5 in fast mode)."""
    code = r'''
import sys, json, numpy as np
sys.path.insert(0, sys.argv[1])
import bevpool as ref
from examples.ref_backend_cuda import register
register(ref, "cuda")
register(ref, "cuda_exact", exact=True)
spec = ref.WorkloadSpec(1, ref.FrustumSpec(16, 44, 1.0, 1.0, 59),
                        ref.BevGridSpec(-51.2, 51.2, -51.2, 51.2, -10.0, 10.0, 0.8), 32, 0)
rig, feats, logits, grid = ref.gen_workload(spec)
cache = ref.build_cache(rig, spec.frustum, grid)
dist = ref.normalize_depth(logits)
res = {}
for red in ref.Reducer:
    want = ref.pool(feats, dist, cache, grid, red, "interval").values
    ex = ref.pool(feats, dist, cache, grid, red, "cuda_exact").values
    fast = ref.pool(feats, dist, cache, grid, red, "cuda").values
    dev = float((np.abs(want.astype(np.float64) - fast) / np.maximum(1, np.abs(want))).max())
    res[red.value] = [bool(np.array_equal(want, ex)), dev]
from examples.ref_backend_cuda import register_kernel
register_kernel(ref)  # the reference's own pool_interval, its kernel on the GPU
for red in ref.Reducer:
    got = ref.pool(feats, dist, cache, grid, red, "interval").values
    res[red.value].append(got.tobytes() == ref.pool(feats, dist, cache, grid, red, "cuda_exact").values.tobytes())
print(json.dumps(res))
'''
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]), OPENBLAS_NUM_THREADS="1",
               NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/bvp_numba_cache"))
    res = subprocess.run([sys.executable, "-c", code, ROOT], env=env, capture_output=True,
                         text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    for red, (equal, dev, kernel_equal) in out.items():
        assert equal, red
        assert dev <= 1e-5, (red, dev)
        assert kernel_equal, red


def test_reference_cli_with_cuda_backend(host_ref, tmp_path):
    """The reference's own CLI (cli.py:195-243) with `--backend cuda_exact`
    writes the same file as its `--backend interval`; `bench --backend cuda`
    and `verify` run (examples/ref_cli_cuda.py)."""
    gold = os.path.join(HERE, "golden", "cli")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]), OPENBLAS_NUM_THREADS="1",
               NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/bvp_numba_cache"))

    def cli(*args):
        return subprocess.run([sys.executable, "-m", "examples.ref_cli_cuda", *args], env=env,
                              cwd=ROOT, capture_output=True, text=True, timeout=900)

    files = ["--calib", os.path.join(gold, "calibration.json"),
             "--features", os.path.join(gold, "features.bvpt"),
             "--logits", os.path.join(gold, "logits.bvpt"),
             "--grid-extent", "8.0", "--cell-size", "0.5"]
    for backend in ("interval", "cuda_exact", "cuda"):
        r = cli("pool", *files, "--backend", backend, "--out", str(tmp_path / f"{backend}.bvpt"))
        assert r.returncode == 0, r.stderr
    a = (tmp_path / "interval.bvpt").read_bytes()
    assert a == (tmp_path / "cuda_exact.bvpt").read_bytes()
    small = ["--cameras", "2", "--height", "8", "--width", "12", "--depth-bins", "9",
             "--channels", "8", "--grid-extent", "16", "--cell-size", "0.5"]
    r = cli("bench", *small, "--backend", "cuda", "--reps", "2", "--warmups", "1")
    assert r.returncode == 0 and "cuda" in r.stdout, r.stderr

"""The C ABI driven from plain C (examples/c_abi_pool.c), as a non-Python
host would: compiled with gcc against include/bevpool_b200.h and the in-tree
libbevpool_sm100.so; its association, depth softmax and pools are checked
against the oracle (cells, ranks and intervals bit-exact, the exact map
bit-exact, the fast map within 1e-5)."""
import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle import oracle as o

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"
H, W, D, C, NX, NY = 16, 44, 59, 32, 128, 128
GRID = np.array([-51.2, 51.2, -51.2, 51.2, -10.0, 10.0, 0.8])
CAM = np.array([0.8 * W, 0.8 * W, W / 2.0, H / 2.0, 0, 0, 1, -1, 0, 0, 0, -1, 0, 0, 0, 1.6])


def build_example(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lib_dir = os.path.join(ROOT, "paper_2205_13542_b200")
    exe = str(tmp_path / "c_abi_pool")
    cmd = ["gcc", "-O2", "-std=c11", os.path.join(ROOT, "examples", "c_abi_pool.c"),
           "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include",
           "-L", lib_dir, "-lbevpool_sm100", "-L", f"{CUDA}/lib64", "-lcudart", "-lm",
           f"-Wl,-rpath,{lib_dir}", f"-Wl,-rpath,{CUDA}/lib64", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_example_compiles_against_the_header(tmp_path):
    """CPU: the C host compiles and links against the ABI (no GPU needed)."""
    if not os.path.exists(os.path.join(ROOT, "paper_2205_13542_b200", "libbevpool_sm100.so")):
        pytest.skip("library not built")
    assert os.path.exists(build_example(tmp_path))


@pytest.mark.gpu
def test_c_host_pipeline_matches_oracle(tmp_path):
    exe = build_example(tmp_path)
    res = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr

    def load(name, dtype):
        return np.fromfile(tmp_path / f"{name}.bin", dtype=dtype)

    feats = load("features", np.float32).reshape(1, C, H, W)
    dist = load("dist", np.float32).reshape(1, D, H, W)
    cells = load("cell_of_point", np.uint32)
    want_cells = o.frustum_cells(CAM, H, W, D, 1.0, 1.0, GRID, NX, NY)
    np.testing.assert_array_equal(cells, want_cells)
    ranks, starts, icells = o.ranks_and_intervals(want_cells, NX * NY)
    np.testing.assert_array_equal(load("ranks", np.uint32), ranks)
    np.testing.assert_array_equal(load("interval_starts", np.uint32), starts)
    np.testing.assert_array_equal(load("interval_cells", np.uint32), icells)
    want = o.pool_interval(feats, dist, ranks, starts, icells, NX * NY, "sum")
    np.testing.assert_array_equal(load("out_exact", np.float32).reshape(want.shape), want)
    assert o.max_rel_dev(want, load("out_fast", np.float32).reshape(want.shape)) <= 1e-5
    assert o.max_rel_dev(want, load("out_tiled", np.float32).reshape(want.shape)) <= 1e-5
    # training from C: the tiled adjoint (fp32, 1e-5) and config F's fused
    # forward (1e-5 of the bf16-input restatement) and adjoint (1e-2)
    g = load("grad_out", np.float32).reshape(C, NX * NY).astype(np.float64)
    gf, gw = o.pool_backward(feats, dist, want_cells, g, ranks, starts, icells, "sum")
    assert o.max_rel_dev(gf, load("grad_features", np.float32).reshape(gf.shape)) <= 1e-5
    assert o.max_rel_dev(gw, load("grad_dist", np.float32).reshape(gw.shape)) <= 1e-5

    def bf16(name, shape):
        return (load(name, np.uint16).astype(np.uint32) << 16).view(np.float32).reshape(shape)

    lb, cb = bf16("logits_bf16", (1, D, H, W)), bf16("context_bf16", (1, C, H, W))
    want_f = o.fused_pool(cb, lb, ranks, starts, icells, NX * NY, "sum")
    assert o.max_rel_dev(want_f, load("out_fused", np.float32).reshape(want_f.shape)) <= 1e-5
    want_l, want_c = o.fused_backward(cb, lb, want_cells, g, ranks, starts, icells, "sum")
    assert o.max_rel_dev(want_l, bf16("grad_logits", want_l.shape)) <= 1e-2
    assert o.max_rel_dev(want_c, bf16("grad_context", want_c.shape)) <= 1e-2


def build_interval_reduce(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lib_dir = os.path.join(ROOT, "paper_2205_13542_b200")
    exe = str(tmp_path / "c_abi_interval_reduce")
    cmd = ["gcc", "-O2", "-std=c11", os.path.join(ROOT, "examples", "c_abi_interval_reduce.c"),
           "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include",
           "-L", lib_dir, "-lbevpool_sm100", "-L", f"{CUDA}/lib64", "-lcudart",
           f"-Wl,-rpath,{lib_dir}", f"-Wl,-rpath,{CUDA}/lib64", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_interval_reduce_host_compiles(tmp_path):
    if not os.path.exists(os.path.join(ROOT, "paper_2205_13542_b200", "libbevpool_sm100.so")):
        pytest.skip("library not built")
    assert os.path.exists(build_interval_reduce(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["T", "S"])
def test_c_interval_reduce_with_reference_arrays(tmp_path, name):
    """bvp_interval_reduce_f32 called from C with nothing but the
    reference's cache arrays and its transposed inputs is bit-identical to
    the reference's interval_reduce (the oracle restatement, itself pinned
    to the reference's digests) for SUM, MEAN and MAX."""
    exe = build_interval_reduce(tmp_path)
    cfg = o.CONFIGS[name]
    cache = o.build_cache(cfg)
    feats, logits = o.gen_inputs(cfg.n_cameras, cfg.channels, cfg.height, cfg.width,
                                 cfg.depth_bins, 0)
    dist = o.normalize_depth(logits)
    arrays = {"ranks": cache["ranks"], "starts": cache["interval_starts"],
              "icells": cache["interval_cells"],
              "dist_t": np.ascontiguousarray(dist.transpose(0, 2, 3, 1)),
              "feats_t": np.ascontiguousarray(feats.transpose(0, 2, 3, 1))}
    for k, v in arrays.items():
        v.tofile(tmp_path / f"{k}.bin")
    n_cells = cfg.n_cells
    res = subprocess.run([exe, str(tmp_path), str(len(cache["ranks"])),
                          str(len(cache["interval_starts"])), str(n_cells), str(cfg.height),
                          str(cfg.width), str(cfg.depth_bins), str(cfg.channels),
                          str(cfg.n_cameras)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    for red in ("sum", "mean", "max"):
        want = o.pool_interval(feats, dist, cache["ranks"], cache["interval_starts"],
                               cache["interval_cells"], n_cells, red)
        got = np.fromfile(tmp_path / f"out_{red}.bin", dtype=np.float32).reshape(want.shape)
        np.testing.assert_array_equal(got, want)

"""CPU tests: the C-ABI library (loads, exports every declared symbol,
validates arguments before touching the GPU) and the host-side mirror of the
reference interface.  No CUDA compute calls."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2205_13542_b200 as bp
from paper_2205_13542_b200 import _lib
from conftest import ROOT
from instances import random_instance
from oracle import oracle as o

HEADER = os.path.join(ROOT, "include", "bevpool_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(bvp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync with the header"


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_abi_version_and_errors_without_gpu():
    lib = _lib.load()
    assert lib.bvp_abi_version() == _lib.ABI_VERSION
    # every pointer NULL, every size 0 (B = 0 is rejected before any CUDA call)
    argtypes = _lib.SIGNATURES["bvp_pool_forward_f32"][1]
    is_ptr = lambda t: t is ctypes.c_void_p or issubclass(t, ctypes._Pointer)  # noqa: E731
    rc = lib.bvp_pool_forward_f32(*[None if is_ptr(t) else 0 for t in argtypes])
    assert rc == _lib.BVP_ERR_INVALID
    assert b"bad dims" in lib.bvp_last_error()
    with pytest.raises(bp.ValidationError):
        _lib.check(rc, "pool")
    rc = lib.bvp_pool_prefixsum_f32(None, None, None, None, None, 0, 0, 1, 1, 1, 1, 1, 1,
                                    _lib.BVP_MAX, None, None, 0, None)
    assert rc == _lib.BVP_ERR_UNSUPPORTED
    with pytest.raises(bp.ConfigurationError):
        _lib.check(rc, "prefixsum")
    ws = ctypes.c_size_t(lib.bvp_sort_workspace_bytes(1_993_728, 129_600)).value
    assert ws > 16 * 1_993_728


def test_grid_spec_validation():
    assert (bp.DEFAULT_GRID.nx, bp.DEFAULT_GRID.ny) == (256, 256)
    with pytest.raises(bp.ConfigurationError):
        bp.BevGridSpec(0, 1.0, 0, 1.0, -1, 1, r=0.3)
    with pytest.raises(bp.ConfigurationError):
        bp.BevGridSpec(0, 1, 0, 1, z_min=2.0, z_max=2.0, r=0.5)
    with pytest.raises(bp.ConfigurationError):
        bp.BevGridSpec(0, 1, 0, 1, -1, 1, r=-0.5)


def test_quantize_kats():
    g = bp.DEFAULT_GRID
    assert bp.quantize(g, (0.0, 0.0, 0.0)) == 128 * 256 + 128
    assert bp.quantize(g, (51.2, 0.0, 0.0)) == bp.OUT_OF_RANGE
    assert bp.quantize(g, (-51.2, -51.2, -10.0)) == 0
    assert bp.quantize(g, (0.0, 0.0, 9.999)) == bp.quantize(g, (0.0, 0.0, 0.0))
    assert bp.quantize(g, (0.0, 0.0, 10.0)) == bp.OUT_OF_RANGE
    assert bp.quantize(bp.BevGridSpec(0, 2, 0, 2, -1, 1, r=1.0), (1.0, 0.5, 0)) == 2


def test_reducer_and_errors():
    assert bp.Reducer.parse("MEAN") is bp.Reducer.MEAN
    with pytest.raises(bp.ConfigurationError, match="reducer"):
        bp.Reducer.parse("median")
    assert issubclass(bp.ValidationError, ValueError) and issubclass(bp.StaleCacheError, bp.BevPoolError)
    e = bp.FileFormatError("bad", field="cameras[2].rotation", offset=7)
    assert str(e) == "cameras[2].rotation: bad (at byte offset 7)"


def test_calibration_validation():
    with pytest.raises(bp.ConfigurationError):
        bp.CameraCalibration(fx=-1, fy=1, cx=0, cy=0, rotation=np.eye(3), translation=np.zeros(3))
    with pytest.raises(bp.ConfigurationError):
        bp.CameraCalibration(fx=1, fy=1, cx=0, cy=0, rotation=np.diag([1, 1, -1.0]),
                             translation=np.zeros(3))
    cam = bp.CameraCalibration(fx=50, fy=60, cx=10, cy=12, rotation=np.eye(3),
                               translation=np.array([1.0, 2.0, 3.0]))
    p = bp.unproject(cam, 3.0, 4.0, 7.0)
    u, v, d = bp.project(cam, p)
    assert abs(u - 3.0) < 1e-9 and abs(v - 4.0) < 1e-9 and abs(d - 7.0) < 1e-9
    with pytest.raises(bp.BehindCameraError):
        bp.project(cam, np.array([1.0, 2.0, 2.0]))


@pytest.mark.parametrize("name", ["T", "S", "H"])
def test_workload_generator_matches_reference(golden, name):
    from conftest import sha
    spec = bp.CONFIGS[name]
    rig, features, logits, grid = bp.gen_workload(spec)
    entry = golden["configs"][name]
    assert sha(features) == entry["sha256"]["features"]
    assert sha(logits) == entry["sha256"]["logits"]
    assert (grid.nx, grid.ny) == (entry["nx"], entry["ny"])
    assert spec.n_points == entry["n_points"]
    np.testing.assert_array_equal(bp.rig_rows(rig), o.synthetic_rig(spec.n_cameras,
                                                                     spec.frustum.height,
                                                                     spec.frustum.width))
    assert bp.fingerprint_inputs(rig, spec.frustum, grid) == entry["fingerprint"]
    cfg = o.CONFIGS[name]
    assert (cfg.n_cameras, cfg.height, cfg.width, cfg.depth_bins, cfg.channels) == (
        spec.n_cameras, spec.frustum.height, spec.frustum.width, spec.frustum.depth_bins,
        spec.channels)
    assert cfg.grid == tuple(grid.as_array())


def test_standard_spec_point_count():
    assert bp.standard_spec().n_points == 1_993_728


def test_fingerprint_of_instances(golden):
    for seed in ("0", "100", "10000"):
        inst = random_instance(int(seed), *( (64, 32, 16) if seed == "10000" else (24, 12, 8)))
        rig = [bp.CameraCalibration(fx=r[0], fy=r[1], cx=r[2], cy=r[3],
                                    rotation=r[4:13].reshape(3, 3), translation=r[13:16],
                                    camera_id=k) for k, r in enumerate(inst.cams)]
        fr = bp.FrustumSpec(inst.height, inst.width, inst.depth_min, inst.depth_step,
                            inst.depth_bins)
        assert bp.fingerprint_inputs(rig, fr, bp.BevGridSpec(*inst.grid)) == \
            golden["instances"][seed]["fingerprint"]

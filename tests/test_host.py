"""CPU-side checks: the C-ABI library loads and exports every symbol
include/rift2_b200.h declares (no compute call without a GPU), the Python
boundary mirrors the reference's types/validation, the BASELINE generator
is deterministic, and the product path refuses to run without CUDA."""

import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rift2_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int32_t|const char\*)\s+(rift2_\w+)\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2303_00319_b200 import _lib
    if not os.path.exists(_lib.library_path()):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2303_00319_b200", "csrc"), "-j8"], check=True)
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    from paper_2303_00319_b200 import _lib
    names = _declared()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.library_path()], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, re.M), f"{n} not exported with C linkage"


def test_version_and_errors_without_gpu(lib):
    import ctypes
    from paper_2303_00319_b200 import _lib
    assert lib.rift2_version() == 100
    # argument validation needs no GPU and maps onto the reference's errors
    p = _lib.BankParamsC(0, 6, 3.0, 2.1, 0.55, 0.0, 2.0, 0.5, 10.0)
    n = ctypes.c_size_t()
    rc = lib.rift2_fields_workspace_size(1, 64, 64, ctypes.byref(p), ctypes.byref(n))
    assert rc == 1 and b"n_scales" in lib.rift2_last_error()
    p = _lib.BankParamsC(4, 6, 3.0, 2.1, 0.55, 0.0, 2.0, 0.5, 10.0)
    assert lib.rift2_fields_workspace_size(1, 8, 64, ctypes.byref(p), ctypes.byref(n)) == 1
    assert lib.rift2_fields_workspace_size(1, 64, 77, ctypes.byref(p), ctypes.byref(n)) == 0   # 7 * 11: any length
    assert lib.rift2_fields_workspace_size(1, 64, 8192, ctypes.byref(p), ctypes.byref(n)) == 2   # above 4096
    assert lib.rift2_fields_workspace_size(2, 1024, 1024, ctypes.byref(p), ctypes.byref(n)) == 0
    assert n.value > 2 * 24 * 1024 * 1024 * 8
    with pytest.raises(Exception):
        _lib.check(1, "x")


def test_bank_params_validation():
    from paper_2303_00319_b200 import BankParams, ParameterError
    for kw in ({"n_scales": 0}, {"n_orient": 1}, {"min_wavelength": 1.0}, {"scale_mult": 1.0},
               {"sigma_on_f": 0.0}, {"sigma_on_f": 1.0}):
        with pytest.raises(ParameterError):
            BankParams(**kw)
    assert np.allclose(BankParams().wavelengths(), [3.0, 6.3, 13.23, 27.783])


def test_config_mirror():
    from paper_2303_00319_b200 import ConfigError, RiftConfig, apply_overrides, parse_config_text
    cfg = parse_config_text("scale_mult = 1.6\n# c\nsigma_on_f=0.75\nrotate_patch = off\n")
    assert cfg.scale_mult == 1.6 and cfg.sigma_on_f == 0.75 and cfg.rotate_patch is False
    assert apply_overrides(cfg, ["mode=ring"]).mode == "ring"
    for bad in ("nope = 1", "mode = x", "patch_size = 95"):
        with pytest.raises(ConfigError):
            parse_config_text(bad)
    assert RiftConfig().bank_params().n_orient == 6


def test_errors_hierarchy():
    from paper_2303_00319_b200 import ConfigError, FormatError, ParameterError, RiftError
    for e in (ParameterError, FormatError, ConfigError):
        assert issubclass(e, RiftError) and issubclass(e, ValueError)


def test_generator_deterministic():
    from paper_2303_00319_b200 import synth
    a1, b1, t1 = synth.make_pair(128, seed=9)
    a2, b2, t2 = synth.make_pair(128, seed=9)
    assert np.array_equal(a1, a2) and np.array_equal(b1, b2) and t1.theta_deg == t2.theta_deg
    assert a1.min() == 0.0 and a1.max() == 1.0
    # ground truth maps image-1 points onto image 2 (noise-free check)
    a = synth.blob_field(127, seed=1)
    m = synth.similarity(127, 90.0, 1.0, (3.0, -2.0))     # quarter turn, integer shift: exact samples
    b = synth.warp(a, m)
    tr = synth.PairTruth(90.0, 1.0, (3.0, -2.0), False, 1.0, 0, 127, m)
    for p in ([40.0, 50.0], [70.0, 20.0]):
        q = tr.apply(np.array([p]))[0]
        assert abs(b[int(round(q[1])), int(round(q[0]))] - a[int(p[1]), int(p[0])]) < 1e-12


def test_product_path_refuses_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2303_00319_b200 import RiftError, compute_fields
    with pytest.raises((RiftError, RuntimeError, AssertionError)):
        compute_fields(np.zeros((64, 64)))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2303_00319_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            assert "oracle" not in open(os.path.join(pkg, fn)).read().replace("oracle/", ""), fn


# ---- RIF2 descriptor container (ref: descriptor.py:26-32, 255-294) ----------
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _golden_descs():
    from paper_2303_00319_b200 import Descriptor
    g = np.load(os.path.join(GOLDEN, "container.npz"))
    modes = ("plain", "ring", "rift2")
    return [Descriptor(v, int(k), int(var), modes[m]) for v, k, var, m in zip(g["vec"], g["kp"], g["variant"], g["mode"])]


def test_container_bytes_equal_reference(tmp_path):
    from paper_2303_00319_b200 import write_descriptors
    p = tmp_path / "d.rif2"
    write_descriptors(p, _golden_descs())
    assert p.read_bytes() == open(os.path.join(GOLDEN, "container.rif2"), "rb").read()
    write_descriptors(p, [])
    assert p.read_bytes() == open(os.path.join(GOLDEN, "container_empty.rif2"), "rb").read()


def test_container_read_reference_file():
    from paper_2303_00319_b200 import read_descriptors
    want = _golden_descs()
    got = read_descriptors(os.path.join(GOLDEN, "container.rif2"))
    assert len(got) == len(want)
    for a, b in zip(want, got):
        assert (a.keypoint_id, a.variant, a.mode) == (b.keypoint_id, b.variant, b.mode)
        assert np.array_equal(a.vector.astype(np.float32).astype(np.float64), b.vector)
    assert read_descriptors(os.path.join(GOLDEN, "container_empty.rif2")) == []


def test_container_errors(tmp_path):
    from paper_2303_00319_b200 import Descriptor, FormatError, ParameterError, read_descriptors, write_descriptors
    p = tmp_path / "d.rif2"
    p.write_bytes(b"RIF2\x01")
    with pytest.raises(FormatError):
        read_descriptors(p)                                  # short header
    p.write_bytes(b"NOPE" + bytes(7))
    with pytest.raises(FormatError):
        read_descriptors(p)                                  # bad magic
    p.write_bytes(b"RIF2\x02\x06\x06" + bytes(4))
    with pytest.raises(FormatError):
        read_descriptors(p)                                  # version
    v = np.full(216, 1 / np.sqrt(216))
    write_descriptors(p, [Descriptor(v, 0, 1, "plain")])
    raw = p.read_bytes()
    p.write_bytes(raw[:-8])
    with pytest.raises(FormatError):
        read_descriptors(p)                                  # truncated record
    p.write_bytes(raw[:16] + b"\x07" + raw[17:])
    with pytest.raises(FormatError):
        read_descriptors(p)                                  # unknown mode code
    with pytest.raises(ParameterError):
        write_descriptors(p, [Descriptor(v[:100], 0, 1, "plain")])


# ---- host affine stage (north_star "recovered affine") -----------
def test_estimate_affine_recovers_transform_with_outliers():
    from paper_2303_00319_b200 import affine_rmse, estimate_affine, synth
    rng = np.random.default_rng(3)
    gt = synth.similarity(1024, 37.0, 1.05, (12.0, -7.0))
    ref = rng.uniform(0, 1024, (3000, 2))
    tgt = ref @ gt[:, :2].T + gt[:, 2] + rng.normal(0, 0.5, (3000, 2))
    bad = rng.random(3000) < 0.6                       # 60 % gross outliers
    tgt[bad] = rng.uniform(0, 1024, (int(bad.sum()), 2))
    a, inl = estimate_affine(ref, tgt)
    assert a is not None and affine_rmse(a, gt, 1024) < 0.2
    assert inl[~bad].mean() > 0.95 and inl[bad].mean() < 0.01
    a2, inl2 = estimate_affine(ref, tgt)               # deterministic for a seed
    assert np.array_equal(a, a2) and np.array_equal(inl, inl2)


def test_estimate_affine_degenerate_inputs():
    from paper_2303_00319_b200 import ParameterError, estimate_affine, fit_affine
    assert estimate_affine(np.zeros((2, 2)), np.zeros((2, 2)))[0] is None
    line = np.stack([np.arange(10.0), np.arange(10.0)], 1)          # collinear: every sample singular
    assert estimate_affine(line, line)[0] is None
    with pytest.raises(ParameterError):
        fit_affine(np.zeros((2, 2)), np.zeros((2, 2)))

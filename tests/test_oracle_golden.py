"""Pin the CPU oracle (oracle/rift2_oracle.py) to golden vectors produced
by running the reference itself (tests/golden/make_golden.py), plus the
reference's known-answer tests for the path."""

import math

import numpy as np
import pytest

from conftest import max_norm_err
from oracle import rift2_oracle as O

BASE = O.Bank(scale_mult=1.6, sigma_on_f=0.75)


@pytest.mark.parametrize("tag,bank", [("def", O.Bank()), ("base", BASE)])
def test_fields_match_reference(g_fields, tag, bank):
    f = O.fields(g_fields["image"], bank)
    for key, gk in (("a_o", "a_o"), ("pc", "pc"), ("a_max", "amax")):
        assert max_norm_err(f[key], g_fields[f"{tag}_{gk}"]) <= 1e-6      # golden stored as float32
    assert max_norm_err(f["moment_max"], g_fields[f"{tag}_mmax"]) <= 1e-12
    assert max_norm_err(f["moment_min"], g_fields[f"{tag}_mmin"]) <= 1e-12
    assert np.array_equal(f["mim"], g_fields[f"{tag}_mim"])


def test_step_edge_peak(g_fields):
    # ref tests/test_loggabor.py:159-168
    img = np.zeros((128, 128))
    img[:, 64:] = 1.0
    f = O.fields(img, O.Bank())
    assert max_norm_err(f["moment_max"], g_fields["step_mmax"]) <= 1e-12
    interior = f["moment_max"][20:-20, 20:-20]
    assert 20 + int(np.argmax(interior.sum(axis=0))) in (63, 64)


def test_transfer_known_answers():
    # ref tests/test_loggabor.py:35-50
    assert np.allclose(O.Bank().wavelengths(), [3.0, 6.3, 13.23, 27.783])
    for p in (O.Bank(), O.Bank(n_scales=2, sigma_on_f=0.75)):
        g = O.transfer(48, 64, p)
        assert g.shape == (p.n_scales, 6, 48, 64)
        assert np.all(g[:, :, 0, 0] == 0.0) and g.min() >= 0.0


def test_constant_image_annihilated():
    f = O.fields(np.full((128, 128), 0.7), O.Bank())
    assert f["moment_max"].max() <= 1e-6 and f["a_o"].max() <= 1e-9


def _kp_eq(kp, g, tag):
    for f in ("x", "y", "response", "kind"):
        key = f"{tag}_{f}" if f"{tag}_{f}" in g else f"{tag}_kp_{f}"
        assert np.array_equal(kp[f], g[key]), f


def test_detect_fast_golden(g_detector):
    sq = np.zeros((64, 64))
    sq[30:34, 30:34] = 1.0
    _kp_eq(O.detect_fast(sq, 0.001, 100), g_detector, "square")
    _kp_eq(O.detect_fast(g_detector["noise_map"], 0.001, 300, 5), g_detector, "noise")
    _kp_eq(O.detect_fast(g_detector["quant_map"], 0.001, 200), g_detector, "quant")


@pytest.mark.parametrize("tag", ["r", "t"])
def test_detect_keypoints_golden(g_pair, tag):
    kp = O.detect_keypoints(g_pair[f"{tag}_mmin"], g_pair[f"{tag}_mmax"], 0.001, 600, 96)
    _kp_eq(kp, g_pair, tag)


@pytest.mark.parametrize("tag", ["r", "t"])
def test_descriptors_golden(g_pair, tag):
    kp = np.zeros(len(g_pair[f"{tag}_kp_x"]), O.KP_DTYPE)
    kp["x"], kp["y"] = g_pair[f"{tag}_kp_x"], g_pair[f"{tag}_kp_y"]
    mim = g_pair[f"{tag}_mim"].astype(np.int64)
    for key, args in (("rift2", {}), ("norot", {"rotate": False})):
        c, k, v, s = O.describe_rift2(mim, kp, **args)
        assert np.array_equal(c, g_pair[f"{tag}_{key}_counts"])
        assert np.array_equal(k, g_pair[f"{tag}_{key}_kp"])
        assert np.array_equal(v, g_pair[f"{tag}_{key}_variant"])
        assert s == int(g_pair[f"{tag}_{key}_skipped"])
    c, k, v, s = O.describe_plain(mim, kp)
    assert np.array_equal(c, g_pair[f"{tag}_plain_counts"])
    c, k, v, s = O.describe_ring(mim, kp)
    assert np.array_equal(k, g_pair[f"{tag}_ring_kp"]) and np.array_equal(v, g_pair[f"{tag}_ring_variant"])


def test_matches_golden(g_pair):
    rc, tc = (g_pair[f"{t}_rift2_counts"].astype(np.float64) for t in "rt")
    pairs, evals = O.match_nn(rc / np.linalg.norm(rc, axis=1, keepdims=True), g_pair["r_rift2_kp"],
                              tc / np.linalg.norm(tc, axis=1, keepdims=True), g_pair["t_rift2_kp"])
    want = g_pair["match_rift2"]
    assert np.array_equal(np.array(pairs)[:, :2], want[:, :2])
    np.testing.assert_allclose(np.array(pairs)[:, 2], want[:, 2], rtol=0, atol=1e-14)
    assert evals == int(g_pair["match_rift2_evals"])


@pytest.mark.parametrize("trial", range(4))
def test_matcher_random_golden(g_matcher, trial):
    g = g_matcher
    rc, tc = (g[f"t{trial}_{s}_counts"].astype(np.float64) for s in "rt")
    pairs, _ = O.match_nn(rc / np.linalg.norm(rc, axis=1, keepdims=True), g[f"t{trial}_r_kp"],
                          tc / np.linalg.norm(tc, axis=1, keepdims=True), g[f"t{trial}_t_kp"])
    assert np.array_equal(np.array(pairs)[:, :2], g[f"t{trial}_pairs"][:, :2])


# ---- known-answer tests of the MIM / recode algebra (ref tests/test_mim.py)

def test_dominant_known_answers():
    assert O.dominant([170, 236, 450, 40, 300, 100]) == [3]          # ref test_mim.py:85-87
    assert O.dominant([100, 100, 0, 0, 0, 0]) == [1, 2]
    assert O.dominant([500, 400, 0, 0, 0, 0], 0.8) == [1, 2]         # inclusive boundary
    assert O.dominant([500, 399, 0, 0, 0, 0], 0.8) == [1]
    assert len(O.dominant([100, 95, 90, 85, 80, 75])) == 2


def test_recode_table():
    # ref tests/test_mim.py:100-120, test_acceptance.py:277-302
    for v in range(1, 7):
        for s in range(1, 7):
            want = v - s + 1 if v >= s else v + 6 - s + 1
            assert O.recode_values(np.array([v]), s, 6)[0] == want


def test_rotated_offsets_half_turn():
    dx, dy = O.rotated_offsets(96, math.pi)
    base_dx, base_dy = O.rotated_offsets(96, 0.0)
    # ref tests/test_descriptor.py:27-31: the half turn samples the crop in reverse
    assert np.array_equal(dx, base_dx[::-1, ::-1]) and np.array_equal(dy, base_dy[::-1, ::-1])


_G_EVAL = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "evaluate.npz"))


@pytest.mark.parametrize("trial", range(6))
def test_evaluate_golden(trial):
    # ref: evalbench.py:63-96, golden from the reference's evaluate()
    g = _G_EVAL
    for j in range(3):
        thr, n, rmse, succ = g[f"t{trial}_thr{j}"]
        got = O.evaluate(g[f"t{trial}_ref_xy"], g[f"t{trial}_tgt_xy"], g[f"t{trial}_pairs"], g[f"t{trial}_gt"], thr,
                         10, 2.0 if j == 2 else 20.0)
        assert got[0] == n and got[2] == bool(succ)
        assert (math.isinf(got[1]) and math.isinf(rmse)) or abs(got[1] - rmse) <= 1e-12 * rmse

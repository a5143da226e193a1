"""The reference's step-by-step entry points on their CUDA kernels, against
the CPU oracle (same names as ref __init__.py:10-49).

  build_filter_bank        ref loggabor.py:131-159  float64 kernel: <= 1e-12 relative
  apply_bank               ref loggabor.py:162-185  fp32 FFTs: max-normalised <= 1e-5
  orientation_amplitudes   ref loggabor.py:188-190  float64 sum: bit-exact
  phase_congruency_moments ref loggabor.py:193-251  fp32: max-normalised <= 1e-4
  build_mim                ref mim.py:43-55         float64 argmax: bit-exact (ties to the first)
  patch_histogram, encode  ref mim.py:58-66, descriptor.py:145-164: bit-exact
  recode, cyclic_shift     ref mim.py:117-136: bit-exact
  extract_patch            ref descriptor.py:85-125: bit-exact, None off the map
"""

import numpy as np
import pytest

from conftest import max_norm_err
from oracle import rift2_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

BASE = dict(scale_mult=1.6, sigma_on_f=0.75)


@pytest.fixture(scope="module")
def r2():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2303_00319_b200 as r2
    return r2


@pytest.mark.parametrize("shape,params", [((128, 128), {}), ((48, 64), BASE), ((96, 160), {"n_scales": 2})])
def test_build_filter_bank_vs_oracle(r2, shape, params):
    h, w = shape
    bank = r2.build_filter_bank(w, h, r2.BankParams(**params))
    want = O.transfer(h, w, O.Bank(**params))
    assert bank.transfer.shape == want.shape and bank.transfer.dtype == np.float64
    assert np.all(bank.transfer[:, :, 0, 0] == 0.0)
    np.testing.assert_allclose(bank.transfer, want, rtol=1e-12, atol=1e-300)


def test_build_filter_bank_too_small(r2):
    with pytest.raises(r2.ParameterError):
        r2.build_filter_bank(8, 64)


@pytest.fixture(scope="module")
def stack(r2):
    rng = np.random.default_rng(3)
    img = rng.random((128, 96))
    bank = r2.build_filter_bank(96, 128, r2.BankParams(**BASE))
    return img, bank, r2.apply_bank(img, bank)


def test_apply_bank_vs_oracle(r2, stack):
    img, bank, st = stack
    resp = O.responses(img, O.Bank(**BASE))
    scale = np.abs(resp).max()
    assert np.abs(st.even - resp.real).max() <= 1e-5 * scale
    assert np.abs(st.odd - resp.imag).max() <= 1e-5 * scale
    assert np.abs(st.amplitude - np.abs(resp)).max() <= 1e-5 * scale


def test_apply_bank_uses_the_given_bank(r2, stack):
    """A modified transfer array is applied as given (not regenerated)."""
    img, bank, st = stack
    t = bank.transfer.copy()
    t[1] *= 0.5
    st2 = r2.apply_bank(img, r2.loggabor.FilterBank(transfer=t, params=bank.params))
    assert max_norm_err(st2.amplitude[1], 0.5 * st.amplitude[1]) <= 1e-5
    assert max_norm_err(st2.amplitude[0], st.amplitude[0]) <= 1e-6
    with pytest.raises(r2.ParameterError):
        r2.apply_bank(np.zeros((64, 64)), bank)


def test_orientation_amplitudes_exact(r2, stack):
    _, _, st = stack
    assert np.array_equal(r2.orientation_amplitudes(st), st.amplitude.sum(axis=0))


def test_phase_congruency_moments_vs_oracle(r2, stack):
    img, bank, st = stack
    resp = O.responses(img, O.Bank(**BASE))
    a_o, pc, mmax, mmin = O.phase_congruency(resp, O.Bank(**BASE))
    got = r2.phase_congruency_moments(st)
    assert max_norm_err(got.moment_max, mmax) <= 1e-4
    assert max_norm_err(got.moment_min, mmin) <= 1e-4
    assert max_norm_err(got.pc_per_orientation, pc) <= 1e-4
    # on the GPU's own stack the float64 oracle agrees more tightly
    _, pc2, mmax2, _ = O.phase_congruency(st.even + 1j * st.odd, O.Bank(**BASE))
    assert max_norm_err(got.moment_max, mmax2) <= 1e-5


def test_build_mim_exact_with_ties(r2):
    rng = np.random.default_rng(8)
    a = rng.random((6, 40, 50))
    a[3, :5] = a[1, :5]                       # exact ties: the first channel wins
    a[:, 7, 7] = 0.25
    got = r2.build_mim(a)
    idx, amax = O.max_index_map(a)
    assert np.array_equal(got.indices, idx) and got.indices.dtype == np.int32
    assert np.array_equal(got.max_amplitude, amax) and got.n_orient == 6
    with pytest.raises(r2.ParameterError):
        r2.build_mim(a[:1])


def test_patch_ops_exact(r2):
    rng = np.random.default_rng(2)
    idx = rng.integers(1, 7, (96, 96)).astype(np.int32)
    amp = rng.random((96, 96))
    p = r2.IndexMap(idx, amp, 6)
    assert np.array_equal(r2.patch_histogram(p), np.bincount(idx.ravel(), minlength=7)[1:])
    assert np.array_equal(r2.patch_histogram(p, weighted=True),
                          np.bincount(idx.ravel(), weights=amp.ravel(), minlength=7)[1:])
    got = r2.encode(p, 6)
    np.testing.assert_array_equal(got, O.unit(O.cell_counts(idx, 6, 6)))
    for d in range(1, 7):
        tab = np.array([0] + [v - d + 1 if v >= d else v + 6 - d + 1 for v in range(1, 7)])
        assert np.array_equal(r2.recode(p, d).indices, tab[idx])
        tab = np.array([0] + [(v - d) % 6 + 1 for v in range(1, 7)])
        assert np.array_equal(r2.cyclic_shift(p, d).indices, tab[idx])
    with pytest.raises(r2.ParameterError):
        r2.recode(p, 7)
    assert r2.dominant_indices([10, 3, 8, 0, 8, 1], 0.8) == [1, 3]    # runner-up tie: cyclically closest after


@pytest.mark.parametrize("angle", [np.pi / 6, np.pi / 2, 2.0, np.pi])
@pytest.mark.parametrize("kp", [(120.0, 110.0), (120.5, 101.25)])
def test_extract_patch_vs_oracle(r2, angle, kp):
    rng = np.random.default_rng(4)
    idx = rng.integers(1, 7, (240, 250)).astype(np.int32)
    amp = rng.random((240, 250))
    m = r2.IndexMap(idx, amp, 6)
    got = r2.extract_patch(m, r2.Keypoint(kp[0], kp[1], 1.0, "corner"), 96, angle)
    # continuous offsets of ref: descriptor.py:46-64, rounded as :78-79 (integer
    # keypoints: the oracle's own table) or :120-121
    lin = np.arange(96, dtype=np.float64) + 0.5 - 48.0
    u, v = np.meshgrid(lin, lin)
    c, s = O._snap(np.cos(angle)), O._snap(np.sin(angle))
    ux, vy = c * u - s * v, s * u + c * v
    if kp[0] == int(kp[0]):
        dx, dy = O.rotated_offsets(96, angle)
        sx, sy = int(kp[0]) + dx, int(kp[1]) + dy
    else:
        sx = np.floor(kp[0] + ux + 0.5).astype(np.int64)
        sy = np.floor(kp[1] + vy + 0.5).astype(np.int64)
    assert np.array_equal(got.indices, idx[sy, sx]) and np.array_equal(got.max_amplitude, amp[sy, sx])
    assert r2.extract_patch(m, r2.Keypoint(30.0, 30.0, 1.0, "corner"), 96, angle) is None
    assert r2.extract_patch(m, r2.Keypoint(120.0, 110.0, 1.0, "corner"), 96, 0.0).indices.shape == (96, 96)

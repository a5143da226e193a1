"""cuFFT cross-check of the hand-written FFT passes at the timed size.

BASELINE.json's north_star keeps cuFFT (here: torch.fft in complex128 on the
GPU) off the product path and uses it only as a cross-check.  These tests
apply the same transfer functions (the package's float64 filter-bank kernel,
itself checked against the oracle in test_gpu_unfused.py) to a 1024^2
BASELINE image with torch.fft.fft2 / ifft2 and compare

  * the fused filter bank's per-orientation amplitude sums and maximum
    amplitude (rift2_fields: K1/K2/K3 of csrc/fields.cu), max-normalised
    error <= 1e-4 (measured ~1e-6), and
  * the unfused apply_bank even / odd responses (sign-sensitive: the row pass
    of the fused kernel drops a conjugation the unfused one must keep),
    max-normalised error <= 1e-5,

at the full bench size, where the numpy oracle needs a minute per image.
Follows ref: loggabor.py:162-190 (apply_bank, orientation_amplitudes).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

BASE = dict(scale_mult=1.6, sigma_on_f=0.75)


@pytest.fixture(scope="module")
def setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2303_00319_b200 as r2
    from paper_2303_00319_b200 import engine, synth
    a, b, _ = synth.make_pair(1024, seed=5)
    imgs = torch.as_tensor(np.stack([a, b]).astype(np.float32)).cuda()
    bank = r2.RiftConfig(**BASE).bank_params()
    T = engine.filter_bank(1024, 1024, bank)                      # (S, O, H, W) float64
    return r2, engine, imgs, bank, T


def cufft_responses(img, T):
    F = torch.fft.fft2(img.double())
    return torch.fft.ifft2(F[None, None] * T)                      # complex128 (S, O, H, W)


def rel(a, ref):
    return float((a.double() - ref).abs().max() / ref.abs().max())


@pytest.mark.parametrize("i", [0, 1])
def test_fused_amplitudes_vs_cufft(setup, i):
    r2, engine, imgs, bank, T = setup
    f = engine.fields(imgs, bank, extras=True)
    amp = cufft_responses(imgs[i], T).abs()
    a_o = amp.sum(0)
    assert rel(f["a_o"][i], a_o) <= 1e-4
    # MIM argmax (ref: mim.py:43-55) on cuFFT's amplitudes: >= 99.9 % agreement
    mim = a_o.argmax(0) + 1
    agree = float((f["mim"][i].long() == mim).double().mean())
    assert agree >= 0.999, agree
    assert rel(f["amax"][i], a_o.max(0).values) <= 1e-4


def test_apply_bank_vs_cufft(setup):
    r2, engine, imgs, bank, T = setup
    even, odd, amp = engine.apply_bank(imgs[0], T.float().contiguous())
    resp = cufft_responses(imgs[0], T.float().double())            # the float32-rounded transfer apply_bank saw
    scale = resp.abs().max()
    assert float((even.double() - resp.real).abs().max() / scale) <= 1e-5
    assert float((odd.double() - resp.imag).abs().max() / scale) <= 1e-5
    assert float((amp.double() - resp.abs()).abs().max() / scale) <= 1e-5

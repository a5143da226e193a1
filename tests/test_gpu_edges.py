"""Edge cases and full-size properties of the CUDA path (through the C ABI).

Covers what the reference's own tests exercise at the boundaries:
mixed-radix and odd aspect sizes (ref tests build a 64x48 bank,
test_loggabor.py:49, and run 800x600-class images, test_acceptance.py:216),
empty inputs, keypoint caps, exact ties in matching (first argmin,
ref: matcher.py:130-136), and, at BASELINE's full 1024^2 size, batch
invariance (a pair repeated in a batch gives bit-identical results).
"""

import numpy as np
import pytest

from conftest import max_norm_err
from oracle import rift2_oracle as O
from test_gpu_stages import _detect_gpu, _fields_gpu, _match_gpu

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2303_00319_b200 import engine
    return engine


@pytest.mark.parametrize("shape", [(48, 64), (600, 800), (250, 120), (45, 75), (768, 1024), (1000, 1024), (1024, 768)])
def test_fields_odd_shapes_vs_oracle(eng, shape):
    rng = np.random.default_rng(11)
    img = rng.random(shape)
    bank = O.Bank()
    out = _fields_gpu(eng, img[None], bank)
    ref = O.fields(img, bank, workers=8)
    assert max_norm_err(out["mmax"][0], ref["moment_max"]) <= 1e-4
    assert max_norm_err(out["mmin"][0], ref["moment_min"]) <= 1e-4
    assert max_norm_err(out["pc"][0], ref["pc"]) <= 1e-4
    assert np.mean(out["mim"][0] == ref["mim"]) >= 0.999


@pytest.mark.parametrize("shape", [(98, 98), (77, 91), (67, 71), (143, 52)])
def test_fields_any_prime_factor_vs_oracle(eng, shape):
    # lengths with prime factors above 5 (98 = 2*7^2, 77 = 7*11, 91 = 7*13,
    # primes 67 and 71, 143 = 11*13): the reference takes any size >= 16
    # (ref: loggabor.py:131-185); runtime-radix Stockham passes
    rng = np.random.default_rng(12)
    img = rng.random(shape)
    bank = O.Bank()
    out = _fields_gpu(eng, img[None], bank)
    ref = O.fields(img, bank, workers=8)
    assert max_norm_err(out["mmax"][0], ref["moment_max"]) <= 1e-4
    assert max_norm_err(out["mmin"][0], ref["moment_min"]) <= 1e-4
    assert max_norm_err(out["pc"][0], ref["pc"]) <= 1e-4
    assert np.mean(out["mim"][0] == ref["mim"]) >= 0.999


def test_fields_unsupported_size_is_parameter_error(eng):
    from paper_2303_00319_b200.errors import ParameterError
    with pytest.raises(ParameterError):
        _fields_gpu(eng, np.zeros((1, 8, 64)), O.Bank())        # below the reference's 16-pixel minimum


@pytest.mark.parametrize("cap", [1, 7, 64])
def test_detect_caps_vs_oracle(eng, g_pair, cap):
    maps = np.stack([g_pair["r_mmin"], g_pair["r_mmax"]])[None]
    got = _detect_gpu(eng, maps, 0.001, cap, 48, False)
    want = O.detect_keypoints(g_pair["r_mmin"], g_pair["r_mmax"], 0.001, cap, 96)
    n = int(got["count"][0])
    assert n == len(want) <= cap
    for f in ("x", "y", "response", "kind"):
        assert np.array_equal(got[f][0][:n], want[f]), f


def test_describe_zero_keypoints(eng, g_pair):
    mim = torch.as_tensor(g_pair["r_mim"].astype(np.uint8)).cuda()[None]
    x = torch.zeros((1, 8), dtype=torch.int32).cuda()
    y = torch.zeros((1, 8), dtype=torch.int32).cuda()
    cnt = torch.zeros(1, dtype=torch.int32).cuda()
    out = eng.describe(mim, x, y, cnt, 6, mode="rift2", rotate=True)
    torch.cuda.synchronize()
    assert int(out["count"][0]) == 0 and int(out["skipped"][0]) == 0


def test_describe_all_outside_are_skipped(eng, g_pair):
    # keypoints whose patches leave the image are skipped, not errors (ref: descriptor.py:196-198)
    mim = torch.as_tensor(g_pair["r_mim"].astype(np.uint8)).cuda()[None]
    x = torch.tensor([[0, 5, 250]], dtype=torch.int32).cuda()
    y = torch.tensor([[0, 128, 3]], dtype=torch.int32).cuda()
    cnt = torch.tensor([3], dtype=torch.int32).cuda()
    out = eng.describe(mim, x, y, cnt, 6, mode="rift2", rotate=True)
    torch.cuda.synchronize()
    assert int(out["count"][0]) == 0 and int(out["skipped"][0]) == 3


def test_match_empty_sides(eng):
    rng = np.random.default_rng(1)
    c = rng.integers(0, 20, (40, 216)).astype(np.uint16)
    k = np.arange(40, dtype=np.int32)
    r, t, d = _match_gpu(eng, c[:0], k[:0], c, k)
    assert len(r) == 0
    r, t, d = _match_gpu(eng, c, k, c[:0], k[:0] + 0)
    assert len(r) == 0


def test_match_exact_ties_take_first_reference(eng):
    # identical reference descriptors under different keypoint ids, spread over
    # several 128-column tiles and column splits: the smallest id must win
    rng = np.random.default_rng(5)
    nr, nt = 1000, 300
    rc = rng.integers(0, 25, (nr, 216)).astype(np.uint16)
    for a, b, c in ((10, 500, 900), (130, 131, 777), (256, 600, 999)):
        rc[b] = rc[a]
        rc[c] = rc[a]
    tc = rng.integers(0, 25, (nt, 216)).astype(np.uint16)
    tc[0], tc[1], tc[2] = rc[900], rc[777], rc[999]
    tc[3] = rc[10] * 2                                 # same direction, different norm
    rk = np.arange(nr, dtype=np.int32)
    tk = np.arange(nt, dtype=np.int32)
    r, t, d = _match_gpu(eng, rc, rk, tc, tk)
    got = dict(zip(t.tolist(), r.tolist()))
    assert got[0] == 10 and got[1] == 130 and got[2] == 256 and got[3] == 10
    rv = rc / np.linalg.norm(rc.astype(float), axis=1, keepdims=True)
    tv = tc / np.linalg.norm(tc.astype(float), axis=1, keepdims=True)
    pairs, _ = O.match_nn(rv, rk, tv, tk)
    assert {(int(b), int(a)) for a, b, _ in pairs} == set(got.items())


def test_full_size_batch_invariance(eng):
    """1024^2 (BASELINE configs[1]): the same pair twice in one batch gives
    bit-identical maps, keypoints, descriptors and matches."""
    from paper_2303_00319_b200 import BatchPipeline, RiftConfig, synth
    imgs, _ = synth.make_batch(1, 1024, seed0=3)
    batch = np.concatenate([imgs, imgs])
    pipe = BatchPipeline(2, 1024, 1024, RiftConfig(scale_mult=1.6, sigma_on_f=0.75))
    pipe.load(batch)
    pipe.step()
    torch.cuda.synchronize()
    m = {k: v.cpu().numpy() for k, v in pipe.m.items()}
    n0, n1 = int(m["count"][0]), int(m["count"][1])
    assert n0 == n1 > 100
    for k in ("ref", "tgt", "dist"):
        assert np.array_equal(m[k][0][:n0], m[k][1][:n1]), k
    assert np.all(np.diff(m["dist"][0][:n0]) >= 0)


def test_fields_4096_vs_oracle(eng):
    """configs[3] size (4096^2, blob sigma x4): the G = 128 FFT path against the
    oracle on the full image."""
    from paper_2303_00319_b200 import synth
    a, _, _ = synth.make_pair(4096, seed=1, looks=None)
    bank = O.Bank(scale_mult=1.6, sigma_on_f=0.75)
    out = _fields_gpu(eng, a[None], bank, extras=False)
    ref = O.fields(a, bank, workers=16)
    assert max_norm_err(out["mmax"][0], ref["moment_max"]) <= 1e-4
    assert max_norm_err(out["mmin"][0], ref["moment_min"]) <= 1e-4
    assert np.mean(out["mim"][0] == ref["mim"]) >= 0.999


def test_c4_pair_runs_and_matches(eng):
    """configs[3] end to end on one GPU: 4096^2 pair, up to 20,000 keypoints;
    the recovered matches agree with the generator's similarity transform.
    (Without the 4-look speckle: with it the matches are wrong on the CPU
    path too -- SURVEY D5 -- and this test is about the large-size path.)"""
    import paper_2303_00319_b200 as r2
    from paper_2303_00319_b200 import synth
    a, b, truth = synth.make_pair(4096, seed=2, looks=None)
    cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=20000)
    res = r2.match_pair(a, b, cfg)
    assert len(res.ref.keypoints) > 5000
    rx = np.array([[k.x, k.y] for k in res.ref.keypoints])
    tx = np.array([[k.x, k.y] for k in res.tgt.keypoints])
    r = np.array([p[0] for p in res.matches.pairs])
    t = np.array([p[1] for p in res.matches.pairs])
    resid = np.linalg.norm(truth.apply(rx[r]) - tx[t], axis=1)
    assert (resid < 3).sum() >= 1000


def test_batch_pipeline_non_square_matches_pair_api(eng):
    """The batched throughput path (BatchPipeline, CUDA graphs) on a
    non-square size gives, pair for pair, the same keypoints and matches as
    the per-pair drop-in API."""
    import paper_2303_00319_b200 as r2
    from paper_2303_00319_b200 import synth
    H, W = 512, 768
    imgs = []
    for seed in (1, 2):
        a, b, _ = synth.make_pair(768, seed=seed, looks=None)
        imgs += [a[128:640].astype(np.float32), b[128:640].astype(np.float32)]
    batch = np.stack(imgs)
    cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=2000)
    pipe = r2.BatchPipeline(2, H, W, cfg)
    pipe.load(batch)
    pipe.capture()
    pipe.step()
    torch.cuda.synchronize()
    for p, (ri, ti, dist) in enumerate(pipe.matches_host()):
        res = r2.match_pair(batch[2 * p].astype(np.float64), batch[2 * p + 1].astype(np.float64), cfg)
        kr = pipe.keypoints_host(2 * p)
        assert np.array_equal(kr["x"], [k.x for k in res.ref.keypoints])
        assert np.array_equal(kr["y"], [k.y for k in res.ref.keypoints])
        want = np.array([(r, t) for r, t, _ in res.matches.pairs]).reshape(-1, 2)
        assert len(want) > 50 and np.array_equal(np.stack([ri, ti], 1), want)
        assert np.array_equal(dist, [d for _, _, d in res.matches.pairs])

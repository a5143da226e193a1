"""GPU parity of each stage, called through the C ABI (engine.*), against
the golden vectors produced by the reference itself and against the CPU
oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star):
  * PC / moment / amplitude maps: max-normalised error <= 1e-4 (fp32 GPU vs
    the reference's float64);
  * MIM: identical on >= 99.9 % of pixels;
  * keypoints, descriptor counts, matches: bit-exact when the stage is fed
    the reference's own upstream arrays.
"""

import numpy as np
import pytest

from conftest import max_norm_err
from oracle import rift2_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

BASE = dict(scale_mult=1.6, sigma_on_f=0.75)


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2303_00319_b200 import engine
    return engine


def _bank(**kw):
    return O.Bank(**kw)


def _fields_gpu(eng, imgs, bank, extras=True):
    t = torch.as_tensor(np.asarray(imgs, dtype=np.float32)).cuda()
    out = eng.fields(t, bank, extras=extras)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("tag,params", [("def", {}), ("base", BASE)])
def test_fields_vs_reference_golden(eng, g_fields, tag, params):
    out = _fields_gpu(eng, g_fields["image"][None], _bank(**params))
    assert max_norm_err(out["mmax"][0], g_fields[f"{tag}_mmax"]) <= 1e-4
    assert max_norm_err(out["mmin"][0], g_fields[f"{tag}_mmin"]) <= 1e-4
    assert max_norm_err(out["a_o"][0], g_fields[f"{tag}_a_o"]) <= 1e-4
    assert max_norm_err(out["pc"][0], g_fields[f"{tag}_pc"]) <= 1e-4
    assert max_norm_err(out["amax"][0], g_fields[f"{tag}_amax"]) <= 1e-4
    agree = np.mean(out["mim"][0].astype(np.int64) == g_fields[f"{tag}_mim"])
    assert agree >= 0.999


def test_fields_step_edge(eng, g_fields):
    img = np.zeros((128, 128))
    img[:, 64:] = 1.0
    out = _fields_gpu(eng, img[None], _bank())
    assert max_norm_err(out["mmax"][0], g_fields["step_mmax"]) <= 1e-4
    interior = out["mmax"][0][20:-20, 20:-20]
    assert 20 + int(np.argmax(interior.sum(axis=0))) in (63, 64)


@pytest.mark.parametrize("size", [64, 256, 512, 1024])
def test_fields_vs_oracle_pow2(eng, size):
    from paper_2303_00319_b200 import synth
    a, b, _ = synth.make_pair(size, seed=5, theta_deg=33.0)
    bank = _bank(**BASE)
    out = _fields_gpu(eng, np.stack([a, b]), bank)
    for i, img in enumerate((a, b)):
        ref = O.fields(img, bank, workers=8)
        assert max_norm_err(out["mmax"][i], ref["moment_max"]) <= 1e-4
        assert max_norm_err(out["mmin"][i], ref["moment_min"]) <= 1e-4
        assert max_norm_err(out["pc"][i], ref["pc"]) <= 1e-4
        assert max_norm_err(out["a_o"][i], ref["a_o"]) <= 1e-4
        assert np.mean(out["mim"][i] == ref["mim"]) >= 0.999


@pytest.mark.parametrize("shape", [(96, 160), (384, 384), (80, 100)])
def test_fields_vs_oracle_mixed_radix(eng, shape):
    rng = np.random.default_rng(3)
    img = rng.random(shape)
    bank = _bank()
    out = _fields_gpu(eng, img[None], bank)
    ref = O.fields(img, bank)
    assert max_norm_err(out["mmax"][0], ref["moment_max"]) <= 1e-4
    assert max_norm_err(out["mmin"][0], ref["moment_min"]) <= 1e-4
    assert np.mean(out["mim"][0] == ref["mim"]) >= 0.999


def test_fields_constant_image(eng):
    out = _fields_gpu(eng, np.full((1, 128, 128), 0.7), _bank())
    assert out["mmax"].max() <= 1e-6 and out["mmin"].max() <= 1e-6
    assert out["a_o"].max() <= 1e-6


def _kp_equal(got, tag, g):
    n = int(got["count"][0])
    for f in ("x", "y", "response", "kind"):
        want = g[f"{tag}_{f}"] if f"{tag}_{f}" in g else g[f"{tag}_kp_{f}"]
        assert np.array_equal(got[f][0][:n], want), f


def _detect_gpu(eng, maps, thr, cap, margin, single):
    t = torch.as_tensor(np.asarray(maps, dtype=np.float64)).cuda()
    out = eng.detect(t[:, 0], None if single else t[:, 1], thr, cap, margin, single_map=single)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def test_detect_fast_golden(eng, g_detector):
    sq = np.zeros((64, 64))
    sq[30:34, 30:34] = 1.0
    _kp_equal(_detect_gpu(eng, sq[None, None], 0.001, 100, 0, True), "square", g_detector)
    _kp_equal(_detect_gpu(eng, g_detector["noise_map"][None, None], 0.001, 300, 5, True), "noise", g_detector)
    _kp_equal(_detect_gpu(eng, g_detector["quant_map"][None, None], 0.001, 200, 0, True), "quant", g_detector)


def test_detect_constant_map_empty(eng):
    got = _detect_gpu(eng, np.full((1, 1, 32, 32), 0.5), 0.001, 100, 0, True)
    assert int(got["count"][0]) == 0


@pytest.mark.parametrize("tag", ["r", "t"])
def test_detect_keypoints_golden(eng, g_pair, tag):
    maps = np.stack([g_pair[f"{tag}_mmin"], g_pair[f"{tag}_mmax"]])[None]
    got = _detect_gpu(eng, maps, 0.001, 600, 48, False)
    _kp_equal(got, tag, g_pair)


def test_detect_batch_matches_oracle(eng, g_pair):
    # two images in one batch, cap small enough that both caps and merge bite
    maps = np.stack([np.stack([g_pair[f"{t}_mmin"], g_pair[f"{t}_mmax"]]) for t in "rt"])
    got = _detect_gpu(eng, maps, 0.001, 150, 48, False)
    for i, t in enumerate("rt"):
        want = O.detect_keypoints(g_pair[f"{t}_mmin"], g_pair[f"{t}_mmax"], 0.001, 150, 96)
        n = int(got["count"][i])
        assert n == len(want)
        assert np.array_equal(got["x"][i][:n], want["x"])
        assert np.array_equal(got["y"][i][:n], want["y"])
        assert np.array_equal(got["response"][i][:n], want["response"])
        assert np.array_equal(got["kind"][i][:n], want["kind"])


def _describe_gpu(eng, g, tag, mode, rotate=True):
    mim = torch.as_tensor(g[f"{tag}_mim"].astype(np.uint8)).cuda()[None]
    x = torch.as_tensor(g[f"{tag}_kp_x"]).cuda()[None]
    y = torch.as_tensor(g[f"{tag}_kp_y"]).cuda()[None]
    cnt = torch.tensor([x.shape[1]], dtype=torch.int32).cuda()
    out = eng.describe(mim, x, y, cnt, 6, mode=mode, rotate=rotate)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("tag", ["r", "t"])
@pytest.mark.parametrize("mode,key,rotate", [("rift2", "rift2", True), ("rift2", "norot", False),
                                             ("plain", "plain", True), ("ring", "ring", True)])
def test_describe_golden(eng, g_pair, tag, mode, key, rotate):
    got = _describe_gpu(eng, g_pair, tag, mode, rotate)
    n = int(got["count"][0])
    assert n == len(g_pair[f"{tag}_{key}_kp"])
    assert int(got["skipped"][0]) == int(g_pair[f"{tag}_{key}_skipped"])
    assert np.array_equal(got["kp"][0][:n], g_pair[f"{tag}_{key}_kp"])
    assert np.array_equal(got["variant"][0][:n], g_pair[f"{tag}_{key}_variant"])
    counts = got["counts"][0][:n, :216].astype(np.int64)
    if mode == "ring":
        plain = g_pair[f"{tag}_plain_counts"].astype(np.int64).reshape(-1, 36, 6)
        kp_of = {k: i for i, k in enumerate(g_pair[f"{tag}_plain_kp"])}
        for row, k, v in zip(counts, got["kp"][0][:n], got["variant"][0][:n]):
            want = np.roll(plain[kp_of[k]], -(int(v) - 1), axis=1).ravel()
            assert np.array_equal(row, want)
    else:
        assert np.array_equal(counts, g_pair[f"{tag}_{key}_counts"].astype(np.int64))
    assert np.array_equal(got["sqnorm"][0][:n], (counts ** 2).sum(1))
    assert not got["counts"][0][:n, 216:].any()


def _match_gpu(eng, ref_counts, ref_kp, tgt_counts, tgt_kp):
    cap = max(len(ref_kp), len(tgt_kp))
    counts = np.zeros((2, cap, 224), np.float16)
    counts[0, :len(ref_kp), :ref_counts.shape[1]] = ref_counts
    counts[1, :len(tgt_kp), :tgt_counts.shape[1]] = tgt_counts
    sq = np.zeros((2, cap), np.int32)
    sq[0, :len(ref_kp)] = (ref_counts.astype(np.int64) ** 2).sum(1)
    sq[1, :len(tgt_kp)] = (tgt_counts.astype(np.int64) ** 2).sum(1)
    kp = np.zeros((2, cap), np.int32)
    kp[0, :len(ref_kp)] = ref_kp
    kp[1, :len(tgt_kp)] = tgt_kp
    desc = dict(counts=torch.as_tensor(counts).cuda(), sqnorm=torch.as_tensor(sq).cuda(),
                kp=torch.as_tensor(kp).cuda(),
                count=torch.tensor([len(ref_kp), len(tgt_kp)], dtype=torch.int32).cuda())
    rb = torch.tensor([0], dtype=torch.int32).cuda()
    tb = torch.tensor([1], dtype=torch.int32).cuda()
    out = eng.match(desc, 216, rb, tb, int(tgt_kp.max()) + 1 if len(tgt_kp) else 1)
    torch.cuda.synchronize()
    n = int(out["count"][0])
    return (out["ref"][0][:n].cpu().numpy(), out["tgt"][0][:n].cpu().numpy(),
            out["dist"][0][:n].cpu().numpy())


@pytest.mark.parametrize("trial", range(4))
def test_match_golden_random_counts(eng, g_matcher, trial):
    g = g_matcher
    r, t, d = _match_gpu(eng, g[f"t{trial}_r_counts"], g[f"t{trial}_r_kp"],
                         g[f"t{trial}_t_counts"], g[f"t{trial}_t_kp"])
    want = g[f"t{trial}_pairs"]
    assert len(r) == len(want)
    assert set(zip(r.tolist(), t.tolist())) == set(zip(want[:, 0].astype(int).tolist(),
                                                       want[:, 1].astype(int).tolist()))
    order = {(int(a), int(b)): i for i, (a, b, _) in enumerate(want)}
    idx = np.array([order[(a, b)] for a, b in zip(r.tolist(), t.tolist())])
    np.testing.assert_allclose(d, want[idx, 2], rtol=1e-12, atol=1e-13)
    assert np.all(np.diff(d) >= 0)


def test_match_golden_pair(eng, g_pair):
    r, t, d = _match_gpu(eng, g_pair["r_rift2_counts"], g_pair["r_rift2_kp"],
                         g_pair["t_rift2_counts"], g_pair["t_rift2_kp"])
    want = g_pair["match_rift2"]
    assert set(zip(r.tolist(), t.tolist())) == set(zip(want[:, 0].astype(int).tolist(),
                                                       want[:, 1].astype(int).tolist()))
    np.testing.assert_allclose(np.sort(d), np.sort(want[:, 2]), rtol=1e-12, atol=1e-13)


def test_match_large_vs_oracle(eng):
    # several tensor-core tiles and column splits; exact integer ranking
    rng = np.random.default_rng(7)
    nr, nt = 1500, 1300
    rc = rng.integers(0, 30, (nr, 216)).astype(np.uint16)
    tc = rng.integers(0, 30, (nt, 216)).astype(np.uint16)
    tc[::7] = rc[:len(tc[::7])]                     # exact duplicates -> distance 0
    rk = np.repeat(np.arange(nr // 2 + 1), 2)[:nr].astype(np.int32)
    tk = np.arange(nt).astype(np.int32)
    r, t, d = _match_gpu(eng, rc, rk, tc, tk)
    rv = rc / np.linalg.norm(rc.astype(float), axis=1, keepdims=True)
    tv = tc / np.linalg.norm(tc.astype(float), axis=1, keepdims=True)
    pairs, _ = O.match_nn(rv, rk, tv, tk)
    want = np.array(pairs)
    got = dict(zip(t.tolist(), r.tolist()))
    agree = np.mean([got[int(b)] == int(a) for a, b, _ in want])
    assert agree == 1.0


@pytest.mark.parametrize("n_orient,grid,width", [(4, 4, 230), (6, 5, 230), (5, 6, 230), (6, 6, 236), (6, 6, 229)])
def test_describe_non_default_grid_vs_oracle(eng, n_orient, grid, width):
    """The runtime-indexed descriptor kernel (any n_orient <= 6, 16-px cells)
    against the oracle, and the 6 x 6 x 6 kernel on widths that take the
    word-staged (W % 4 == 0, no TMA) and byte-staged neighbourhood paths;
    the TMA path is covered by test_describe_golden."""
    rng = np.random.default_rng(n_orient * 10 + grid + width)
    # blocky random MIM: dominant indices and runner-ups vary between keypoints
    small = rng.integers(1, n_orient + 1, (30, 30))
    mim = np.kron(small, np.ones((8, 8), np.int64))[:230, :width]
    noise = rng.random(mim.shape) < 0.3
    mim[noise] = rng.integers(1, n_orient + 1, int(noise.sum()))
    size = 16 * grid
    kps = np.zeros(60, dtype=O.KP_DTYPE)
    kps["x"] = rng.integers(0, width, 60)
    kps["y"] = rng.integers(0, 230, 60)
    want_c, want_k, want_v, want_skip = O.describe_rift2(mim, kps, size=size, grid=grid, n_orient=n_orient)
    m = torch.as_tensor(mim.astype(np.uint8)).cuda()[None]
    x = torch.as_tensor(kps["x"].astype(np.int32)).cuda()[None]
    y = torch.as_tensor(kps["y"].astype(np.int32)).cuda()[None]
    out = eng.describe(m, x, y, torch.tensor([60], dtype=torch.int32).cuda(), n_orient, size, grid)
    torch.cuda.synchronize()
    n = int(out["count"][0])
    dim = grid * grid * n_orient
    assert n == len(want_k) > 0 and int(out["skipped"][0]) == want_skip
    assert np.array_equal(out["kp"][0][:n].cpu().numpy(), want_k)
    assert np.array_equal(out["variant"][0][:n].cpu().numpy(), want_v)
    assert np.array_equal(out["counts"][0][:n, :dim].cpu().numpy().astype(np.int64), want_c)


@pytest.mark.parametrize("n,planes,kind", [(1024 * 1024, 3, "gauss"), (30000, 4, "ties"), (3375, 2, "gauss"),
                                           (1, 1, "gauss"), (2, 1, "gauss"), (4097, 2, "const")])
def test_exact_median_kernels(eng, n, planes, kind):
    """The filter bank's Rayleigh-noise median (ref: loggabor.py:222,
    np.median) is exact: through the same kernels, on planes whose
    amplitudes the kernel also returns, the result equals np.median of those
    amplitudes bit for bit -- odd / even / unaligned sizes, heavy ties, a
    constant plane."""
    g = torch.Generator(device="cuda").manual_seed(n + planes)
    z = torch.randn((planes, n), dtype=torch.complex64, device="cuda", generator=g)
    if kind == "ties":
        z = torch.round(z.real * 4) / 4 + 0j
        z = z.to(torch.complex64)
    elif kind == "const":
        z = torch.full((planes, n), 0.75 + 0.5j, dtype=torch.complex64, device="cuda")
    amps, med = eng.debug_median(z)
    torch.cuda.synchronize()
    a = amps.cpu().numpy().astype(np.float64)
    want = np.median(a, axis=1).astype(np.float32)
    assert np.array_equal(med.cpu().numpy(), want)


@pytest.mark.parametrize("shape", [(45, 75), (101, 83), (64, 130)])
def test_detect_float_maps_unaligned_widths(eng, shape):
    """float32 maps (the pipeline's dtype: vectorised staging when W % 4 == 0,
    scalar otherwise) at widths that are not multiples of 4, against the
    oracle's detect_keypoints on the same values."""
    rng = np.random.default_rng(shape[0] * 1000 + shape[1])
    from scipy.ndimage import gaussian_filter
    mm = [gaussian_filter(rng.random(shape), 1.5).astype(np.float32) for _ in range(2)]
    t = torch.as_tensor(np.stack(mm)[None]).cuda()
    out = eng.detect(t[:, 0], t[:, 1], 0.001, 80, 5)
    torch.cuda.synchronize()
    want = O.detect_keypoints(mm[0].astype(np.float64), mm[1].astype(np.float64), 0.001, 80, 10)
    n = int(out["count"][0])
    assert n == len(want) > 0
    for f in ("x", "y", "response", "kind"):
        assert np.array_equal(out[f][0][:n].cpu().numpy(), want[f]), f

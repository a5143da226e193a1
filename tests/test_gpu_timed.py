"""Parity at the configurations bench.py times (BASELINE.json configs[1-3]).

The bench's workload is 16 independent 1024^2 BASELINE pairs (4-look
speckle, <= 5,000 keypoints) run through BatchPipeline's pipelined CUDA
graphs; configs[3] is one 4096^2 pair with <= 20,000 keypoints.  These tests
run exactly those paths and check every stage against the CPU oracle, each
stage fed the GPU's own upstream arrays (point 9):

  * maps: max-normalised error <= 1e-4, MIM identical on >= 99.9 % of pixels
    (ref: loggabor.py:193-251, mim.py:43-55);
  * keypoints: bit-exact on the GPU's maps (ref: detector.py:140-155);
  * descriptor counts, keypoint ids, variants, skips: bit-exact on the GPU's
    MIM and keypoints (ref: descriptor.py:179-216);
  * matches: bit-exact (ref, tgt) sets, float64 distances within
    1e-12 relative (order by the GPU's own distances), on the GPU's descriptors at full production size
    (ref: matcher.py:102-148), for the batched path (one column split) and
    the single-pair path (SM-filling column splits);
  * end to end: match-set overlap >= 99 % from the raw images.
"""

import os

import numpy as np
import pytest

from conftest import max_norm_err
from oracle import rift2_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

BASE = dict(scale_mult=1.6, sigma_on_f=0.75)
SEEDS = (0, 5, 10, 15)          # from the bench's 16-pair batch (seeds 0-15)


@pytest.fixture(scope="module")
def bench_batch():
    """The bench's own path on 4 of its pairs: two pipelined graph steps
    (fields of the batch, then its features next to a second fields pass)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2303_00319_b200 import BatchPipeline, RiftConfig, synth
    imgs = np.concatenate([synth.make_batch(1, 1024, seed0=s)[0] for s in SEEDS])
    pipe = BatchPipeline(len(SEEDS), 1024, 1024, RiftConfig(max_keypoints=5000, **BASE))
    pipe.load(imgs)
    pipe.capture_pipelined()
    pipe._alt.copy_(pipe.images)
    pipe.pipelined_step(0)
    pipe.pipelined_step(1)
    torch.cuda.synchronize()
    host = {
        "f": {k: v.cpu().numpy() for k, v in pipe.f.items()},
        "k": {k: v.cpu().numpy() for k, v in pipe.k.items()},
        "d": {k: v.cpu().numpy() for k, v in pipe.d.items()},
        "m": {k: v.cpu().numpy() for k, v in pipe.m.items()},
    }
    return imgs, pipe, host


def _gpu_kp(host, i):
    n = int(host["k"]["count"][i])
    return {f: host["k"][f][i, :n] for f in ("x", "y", "response", "kind")}


def _gpu_desc(host, i):
    n = int(host["d"]["count"][i])
    return (host["d"]["counts"][i, :n, :216].astype(np.int64), host["d"]["kp"][i, :n],
            host["d"]["variant"][i, :n], int(host["d"]["skipped"][i]))


def _assert_matches(ref, tgt, dist, want):
    """Exact (ref, tgt) set; each float64 distance within 1e-12 of the
    reference's (its einsum sums in another order, ref: matcher.py:140-141);
    the GPU list sorted by (dist, ref, tgt) on its own distances."""
    ref, tgt, dist = (np.asarray(v) for v in (ref, tgt, dist))
    wmap = {(int(a), int(b)): d for a, b, d in want}
    assert len(ref) == len(wmap)
    assert set(zip(ref.tolist(), tgt.tolist())) == set(wmap)
    np.testing.assert_allclose(dist, [wmap[(int(a), int(b))] for a, b in zip(ref, tgt)], rtol=1e-12, atol=1e-14)
    keys = list(zip(dist.tolist(), ref.tolist(), tgt.tolist()))
    assert keys == sorted(keys)


def _unit(c):
    c = np.asarray(c, dtype=np.float64)
    return c / np.linalg.norm(c, axis=1, keepdims=True)


@pytest.mark.parametrize("i", range(2 * len(SEEDS)))
def test_bench_maps_vs_oracle(bench_batch, i):
    imgs, _, host = bench_batch
    ref = O.fields(imgs[i].astype(np.float64), O.Bank(**BASE), workers=8)
    assert max_norm_err(host["f"]["mmax"][i], ref["moment_max"]) <= 1e-4
    assert max_norm_err(host["f"]["mmin"][i], ref["moment_min"]) <= 1e-4
    assert np.mean(host["f"]["mim"][i].astype(np.int64) == ref["mim"]) >= 0.999


@pytest.mark.parametrize("i", range(2 * len(SEEDS)))
def test_bench_keypoints_and_descriptors_exact(bench_batch, i):
    _, _, host = bench_batch
    f = host["f"]
    want = O.detect_keypoints(f["mmin"][i].astype(np.float64), f["mmax"][i].astype(np.float64), 0.001, 5000, 96)
    got = _gpu_kp(host, i)
    assert len(got["x"]) == len(want["x"]) > 500
    for k in ("x", "y", "response", "kind"):
        assert np.array_equal(got[k], want[k]), k
    c, k, v, skipped = O.describe_rift2(f["mim"][i].astype(np.int64), want)
    gc, gk, gv, gs = _gpu_desc(host, i)
    assert gc.shape == np.asarray(c).shape and gs == skipped
    assert np.array_equal(gc, c) and np.array_equal(gk, k) and np.array_equal(gv, v)


@pytest.mark.parametrize("p", range(len(SEEDS)))
def test_bench_matches_exact(bench_batch, p):
    """Full production size (~5-9k descriptors per side), one column split
    per pair as in the 16-pair batch."""
    _, _, host = bench_batch
    rc, rk, _, _ = _gpu_desc(host, 2 * p)
    tc, tk, _, _ = _gpu_desc(host, 2 * p + 1)
    want, _ = O.match_nn(_unit(rc), rk, _unit(tc), tk)
    n = int(host["m"]["count"][p])
    _assert_matches(host["m"]["ref"][p, :n], host["m"]["tgt"][p, :n], host["m"]["dist"][p, :n], want)


def test_bench_single_pair_splits_exact(bench_batch):
    """The dataclass path matches one pair with SM-filling column splits
    (k_match_combine merges them): same descriptors, same exact result;
    duplicated reference rows are planted in different splits."""
    from paper_2303_00319_b200 import engine
    _, _, host = bench_batch
    rc, rk, _, _ = _gpu_desc(host, 0)
    tc, tk, _, _ = _gpu_desc(host, 1)
    rc = rc.copy()
    n = len(rc)
    # three exact copies of one row in the first, middle and last third; a
    # target equal to it must pick the smallest keypoint id
    src = rc[n // 2]
    for j in (5, n // 2 + 1, n - 3):
        rc[j] = src
    tc = tc.copy()
    tc[0] = src
    cap = max(len(rc), len(tc))
    counts = np.zeros((2, cap, 224), np.float16)
    counts[0, :len(rc), :216] = rc
    counts[1, :len(tc), :216] = tc
    sq = np.zeros((2, cap), np.int32)
    sq[0, :len(rc)] = (rc ** 2).sum(1)
    sq[1, :len(tc)] = (tc ** 2).sum(1)
    kp = np.zeros((2, cap), np.int32)
    kp[0, :len(rk)] = rk
    kp[1, :len(tk)] = tk
    desc = dict(counts=torch.as_tensor(counts).cuda(), sqnorm=torch.as_tensor(sq).cuda(),
                kp=torch.as_tensor(kp).cuda(), count=torch.tensor([len(rc), len(tc)], dtype=torch.int32).cuda())
    blk = torch.tensor([0, 1], dtype=torch.int32).cuda()
    out = engine.match(desc, 216, blk[:1], blk[1:], int(tk.max()) + 1)
    torch.cuda.synchronize()
    want, _ = O.match_nn(_unit(rc), rk, _unit(tc), tk)
    m = int(out["count"][0])
    got = list(zip(out["ref"][0, :m].tolist(), out["tgt"][0, :m].tolist()))
    _assert_matches(out["ref"][0, :m].cpu().numpy(), out["tgt"][0, :m].cpu().numpy(), out["dist"][0, :m].cpu().numpy(),
                    want)
    first = min(int(rk[j]) for j in (5, n // 2, n // 2 + 1, n - 3))
    assert dict((t, r) for r, t in got)[int(tk[0])] == first


@pytest.mark.parametrize("p", [0, 3])
def test_bench_end_to_end_overlap(bench_batch, p):
    """From the raw images: the oracle's whole pipeline vs the GPU batch."""
    imgs, _, host = bench_batch
    bank = O.Bank(**BASE)
    sides = []
    for i in (2 * p, 2 * p + 1):
        f = O.fields(imgs[i].astype(np.float64), bank, workers=8)
        kp = O.detect_keypoints(f["moment_min"], f["moment_max"], 0.001, 5000, 96)
        c, k, _, _ = O.describe_rift2(f["mim"], kp)
        sides.append((kp, c, k))
    (rkp, rc, rk), (tkp, tc, tk) = sides
    pairs, _ = O.match_nn(_unit(rc), rk, _unit(tc), tk)
    want = {((int(rkp["x"][r]), int(rkp["y"][r])), (int(tkp["x"][t]), int(tkp["y"][t]))) for r, t, _ in pairs}
    gr, gt = _gpu_kp(host, 2 * p), _gpu_kp(host, 2 * p + 1)
    n = int(host["m"]["count"][p])
    got = {((int(gr["x"][r]), int(gr["y"][r])), (int(gt["x"][t]), int(gt["y"][t])))
           for r, t in zip(host["m"]["ref"][p, :n], host["m"]["tgt"][p, :n])}
    assert len(want) > 500
    assert len(got & want) / len(want) >= 0.99


# --------------------------------------------------------------- configs[3]
@pytest.fixture(scope="module")
def c4():
    """One 4096^2 BASELINE pair (blob sigma x4) at <= 20,000 keypoints through
    the single-pair CUDA path, stage by stage."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2303_00319_b200 import engine, synth
    a, b, _ = synth.make_pair(4096, seed=0)
    bank = O.Bank(**BASE)
    imgs = torch.as_tensor(np.stack([a, b]).astype(np.float32)).cuda()
    f = engine.fields(imgs, bank)
    k = engine.detect(f["mmin"], f["mmax"], 0.001, 20000, 48)
    d = engine.describe(f["mim"], k["x"], k["y"], k["count"], 6)
    blk = torch.tensor([0, 1], dtype=torch.int32, device="cuda")
    m = engine.match(d, 216, blk[:1], blk[1:], 20000)
    torch.cuda.synchronize()
    host = {"f": {n: v.cpu().numpy() for n, v in f.items()}, "k": {n: v.cpu().numpy() for n, v in k.items()},
            "d": {n: v.cpu().numpy() for n, v in d.items()}, "m": {n: v.cpu().numpy() for n, v in m.items()}}
    return (a, b), host


def test_c4_maps_vs_oracle(c4):
    (a, _), host = c4
    ref = O.fields(a.astype(np.float32).astype(np.float64), O.Bank(**BASE), workers=os.cpu_count() or 8)
    assert max_norm_err(host["f"]["mmax"][0], ref["moment_max"]) <= 1e-4
    assert max_norm_err(host["f"]["mmin"][0], ref["moment_min"]) <= 1e-4
    assert np.mean(host["f"]["mim"][0].astype(np.int64) == ref["mim"]) >= 0.999


def test_c4_features_and_38k_matching_exact(c4):
    _, host = c4
    f = host["f"]
    descs = []
    for i in (0, 1):
        want = O.detect_keypoints(f["mmin"][i].astype(np.float64), f["mmax"][i].astype(np.float64),
                                  0.001, 20000, 96)
        got = _gpu_kp(host, i)
        assert len(got["x"]) == len(want["x"])
        for k in ("x", "y", "response", "kind"):
            assert np.array_equal(got[k], want[k]), k
        c, k, v, skipped = O.describe_rift2(f["mim"][i].astype(np.int64), want)
        gc, gk, gv, gs = _gpu_desc(host, i)
        assert np.array_equal(gc, c) and np.array_equal(gk, k) and np.array_equal(gv, v) and gs == skipped
        descs.append((gc, gk))
    (rc, rk), (tc, tk) = descs
    assert len(rc) > 30000 and len(tc) > 30000            # the ~38k x 37k distance matrix
    want, _ = O.match_nn(_unit(rc), rk, _unit(tc), tk)
    n = int(host["m"]["count"][0])
    _assert_matches(host["m"]["ref"][0, :n], host["m"]["tgt"][0, :n], host["m"]["dist"][0, :n], want)


# ------------------------------------------------- ring / plain match goldens
@pytest.mark.parametrize("mode,rmode,tmode", [("ring", "ring", "plain"), ("plain", "plain", "plain")])
def test_match_ring_plain_goldens(g_pair, mode, rmode, tmode):
    """ref: pipeline.py:53-64 -- ring reference descriptors (6 layers per
    keypoint) against plain targets, and plain against plain, described and
    matched on the GPU from the reference's own MIM and keypoints
    (tests/golden/pair256.npz, written by the reference)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2303_00319_b200 import engine
    sets = []
    for tag, md in (("r", rmode), ("t", tmode)):
        mim = torch.as_tensor(g_pair[f"{tag}_mim"].astype(np.uint8)).cuda()[None]
        x = torch.as_tensor(g_pair[f"{tag}_kp_x"]).cuda()[None]
        y = torch.as_tensor(g_pair[f"{tag}_kp_y"]).cuda()[None]
        cnt = torch.tensor([x.shape[1]], dtype=torch.int32).cuda()
        sets.append(engine.describe(mim, x, y, cnt, 6, mode=md))
    cap = max(s["counts"].shape[1] for s in sets)
    desc = {"counts": torch.zeros((2, cap, 224), dtype=torch.float16, device="cuda"),
            "sqnorm": torch.zeros((2, cap), dtype=torch.int32, device="cuda"),
            "kp": torch.zeros((2, cap), dtype=torch.int32, device="cuda")}
    for b, s in enumerate(sets):
        n = s["counts"].shape[1]
        for k in ("counts", "sqnorm", "kp"):
            desc[k][b, :n] = s[k][0]
    desc["count"] = torch.cat([s["count"] for s in sets])
    blk = torch.tensor([0, 1], dtype=torch.int32, device="cuda")
    out = engine.match(desc, 216, blk[:1], blk[1:], 600)
    torch.cuda.synchronize()
    want = g_pair[f"match_{mode}"]
    n = int(out["count"][0])
    _assert_matches(out["ref"][0, :n].cpu().numpy(), out["tgt"][0, :n].cpu().numpy(), out["dist"][0, :n].cpu().numpy(),
                    want)
    nr, nt = (int(c) for c in desc["count"].tolist())
    assert nr * nt == int(g_pair[f"match_{mode}_evals"])

"""The drop-in Python API (reference names and dataclasses) on the GPU,
checked against the oracle and the reference's own test patterns
(ref: pkg/tests/test_matcher.py:24-65, test_descriptor.py:141-170,
test_detector.py:28-106, test_acceptance.py:161-181)."""

import numpy as np
import pytest

from oracle import rift2_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def r2():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2303_00319_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def pair512():
    from paper_2303_00319_b200 import synth
    return synth.make_pair(512, seed=2, theta_deg=60.0, looks=None)


def test_compute_fields_types(r2, pair512):
    pc, mim = r2.compute_fields(pair512[0], r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75))
    assert pc.a_o.shape == (6, 512, 512) and pc.a_o.dtype == np.float64
    assert pc.pc_per_orientation.shape == (6, 512, 512)
    assert pc.moment_max.dtype == np.float64 and mim.indices.dtype == np.int32
    assert mim.indices.min() >= 1 and mim.indices.max() <= 6
    assert np.all(pc.moment_max >= pc.moment_min) and pc.moment_min.min() >= 0
    assert pc.pc_per_orientation.min() >= 0 and pc.pc_per_orientation.max() <= 1 + 1e-6
    # a_o argmax is the MIM (ties aside)
    assert np.mean(np.argmax(pc.a_o, 0) + 1 == mim.indices) > 0.9999


def test_detect_keypoints_exact_on_gpu_maps(r2, pair512):
    cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=2000)
    pc, _ = r2.compute_fields(pair512[0], cfg)
    kps = r2.detect_keypoints(pc, cfg.fast_threshold, cfg.max_keypoints, cfg.patch_size)
    want = O.detect_keypoints(pc.moment_min, pc.moment_max, cfg.fast_threshold, cfg.max_keypoints, 96)
    assert [(k.x, k.y, k.response) for k in kps] == \
        [(float(x), float(y), float(r)) for x, y, r in zip(want["x"], want["y"], want["response"])]
    assert [k.kind for k in kps] == ["corner" if k == 0 else "edge" for k in want["kind"]]
    # reference invariants (ref tests/test_detector.py:80-106)
    assert all(48 <= k.x <= 512 - 49 and 48 <= k.y <= 512 - 49 for k in kps)
    xy = np.array([(k.x, k.y) for k in kps])
    d2 = ((xy[:, None] - xy[None]) ** 2).sum(-1)
    np.fill_diagonal(d2, 99)
    assert d2.min() > 4


def test_detect_fast_threshold_monotone(r2, pair512):
    pc, _ = r2.compute_fields(pair512[0])
    low = {(k.x, k.y) for k in r2.detect_fast(pc.moment_min, 0.001, 100000)}
    high = {(k.x, k.y) for k in r2.detect_fast(pc.moment_min, 0.002, 100000)}
    assert high <= low and len(low) > 0


def test_describe_vectors_bit_equal(r2, pair512):
    cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=800)
    pc, mim = r2.compute_fields(pair512[0], cfg)
    kps = r2.detect_keypoints(pc, cfg.fast_threshold, cfg.max_keypoints, cfg.patch_size)
    ds = r2.describe_rift2(mim, kps)
    arr = np.zeros(len(kps), dtype=O.KP_DTYPE)
    arr["x"] = [k.x for k in kps]
    arr["y"] = [k.y for k in kps]
    c, kk, v, skipped = O.describe_rift2(mim.indices, arr)
    assert len(ds) == len(c) and ds.skipped == skipped
    for d, cc, k, vv in zip(ds, c, kk, v):
        assert d.keypoint_id == k and d.variant == vv
        assert np.array_equal(d.vector, O.unit(cc))
    # unique-dominant descriptors equal their ring layer (ref acceptance criterion 1)
    norot = r2.describe_rift2(mim, kps, rotate_patch=False)
    ring = {(d.keypoint_id, d.variant): d.vector for d in r2.describe_ring(mim, kps)}
    for d in norot:
        assert np.array_equal(d.vector, ring[(d.keypoint_id, d.variant)])


def _double_loop(ref, tgt):
    best = {}
    for t in tgt:
        for r in ref:
            d = float(np.linalg.norm(r.vector - t.vector))
            cur = best.get(t.keypoint_id)
            if cur is None or d < cur[1]:
                best[t.keypoint_id] = (r.keypoint_id, d)
    return sorted(((r, t, d) for t, (r, d) in best.items()), key=lambda p: (p[2], p[0], p[1]))


def _rand_descs(r2, rng, n, maxv, dim=32):
    out = []
    for i in range(n):
        for v in range(1, int(rng.integers(1, maxv + 1)) + 1):
            vec = rng.standard_normal(dim)
            out.append(r2.Descriptor(vec / np.linalg.norm(vec), i, v, "rift2"))
    return out


@pytest.mark.parametrize("seed", range(5))
def test_match_nn_float_vectors_double_loop(r2, seed):
    rng = np.random.default_rng(seed)
    ref = _rand_descs(r2, rng, 20, 3)
    tgt = _rand_descs(r2, rng, 17, 3)
    got = r2.match_nn(ref, tgt)
    want = _double_loop(ref, tgt)
    assert [(a, b) for a, b, _ in got.pairs] == [(a, b) for a, b, _ in want]
    np.testing.assert_allclose([d for *_, d in got.pairs], [d for *_, d in want], atol=1e-9)


def test_match_nn_self_and_errors(r2, rng):
    descs = _rand_descs(r2, rng, 25, 1)
    m = r2.match_nn(descs, descs)
    assert len(m) == 25 and all(r == t and d == 0.0 for r, t, d in m.pairs)
    with pytest.raises(r2.ParameterError):
        r2.match_nn([], descs)


def test_match_pair_recovers_rotation(r2, pair512):
    a, b, truth = pair512
    cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=2000)
    res = r2.match_pair(a, b, cfg)
    rx = np.array([[k.x, k.y] for k in res.ref.keypoints])
    tx = np.array([[k.x, k.y] for k in res.tgt.keypoints])
    r = np.array([p[0] for p in res.matches.pairs])
    t = np.array([p[1] for p in res.matches.pairs])
    resid = np.linalg.norm(truth.apply(rx[r]) - tx[t], axis=1)
    assert (resid < 3).sum() >= 10


def test_batch_pipeline_equals_api(r2):
    from paper_2303_00319_b200 import synth
    cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=1000)
    imgs, _ = synth.make_batch(2, 256, seed0=4, looks=None)
    pipe = r2.BatchPipeline(2, 256, 256, cfg)
    pipe.load(imgs)
    pipe.capture()
    pipe.step()
    torch.cuda.synchronize()
    res = pipe.matches_host()
    for p in range(2):
        api = r2.match_pair(imgs[2 * p].astype(np.float64), imgs[2 * p + 1].astype(np.float64), cfg)
        got = set(zip(res[p][0].tolist(), res[p][1].tolist()))
        assert got == {(a, b) for a, b, _ in api.matches.pairs}


def test_pipelined_step_equals_step(r2):
    """Throughput mode: filter bank of batch i next to the features of batch
    i-1 on two streams; each batch's matches equal the plain step's."""
    from paper_2303_00319_b200 import synth
    cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=800)
    imgs_a, _ = synth.make_batch(2, 256, seed0=10)
    imgs_b, _ = synth.make_batch(2, 256, seed0=20)
    pipe = r2.BatchPipeline(2, 256, 256, cfg)
    want = []
    for imgs in (imgs_a, imgs_b):
        pipe.load(imgs)
        pipe.step()
        torch.cuda.synchronize()
        want.append({k: v.clone() for k, v in pipe.m.items()})
    pipe.capture_pipelined()
    pipe.images.copy_(torch.from_numpy(imgs_a))
    pipe._alt.copy_(torch.from_numpy(imgs_b))
    pipe.pipelined_step(0)          # filter bank of A
    pipe.pipelined_step(1)          # filter bank of B, features of A
    torch.cuda.synchronize()
    _same_matches(want[0], pipe.m)
    pipe.pipelined_step(0)          # features of B (filter bank of A again)
    torch.cuda.synchronize()
    _same_matches(want[1], pipe.m)


def _same_matches(want, got):
    """Equal counts and equal rows up to each pair's count (rows past it are
    scratch from earlier steps)."""
    assert torch.equal(want["count"], got["count"])
    for p, n in enumerate(want["count"].tolist()):
        for k in ("ref", "tgt", "dist"):
            assert torch.equal(want[k][p, :n], got[k][p, :n]), (p, k)


def test_container_from_device_counts(r2, pair512, tmp_path):
    """write_descriptor_counts on the engine's device rows writes the same
    bytes as write_descriptors on the dataclass descriptors (ref:
    descriptor.py:255-268), and read_descriptors returns them."""
    from paper_2303_00319_b200 import engine
    cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=600)
    pc, mim = r2.compute_fields(pair512[0], cfg)
    kps = r2.detect_keypoints(pc, cfg.fast_threshold, cfg.max_keypoints, cfg.patch_size)
    ds = r2.describe_rift2(mim, kps)
    a, b = tmp_path / "a.rif2", tmp_path / "b.rif2"
    r2.write_descriptors(a, ds.descriptors)
    m = torch.from_numpy(mim.indices.astype(np.uint8)).cuda()[None]
    x = torch.tensor([[k.x for k in kps]], dtype=torch.int32).cuda()
    y = torch.tensor([[k.y for k in kps]], dtype=torch.int32).cuda()
    out = engine.describe(m, x, y, torch.tensor([len(kps)], dtype=torch.int32).cuda(), 6)
    n = int(out["count"][0])
    r2.write_descriptor_counts(b, out["counts"][0, :n], out["kp"][0, :n], out["variant"][0, :n], "rift2")
    assert a.read_bytes() == b.read_bytes()
    back = r2.read_descriptors(b)
    assert [(d.keypoint_id, d.variant) for d in back] == [(d.keypoint_id, d.variant) for d in ds]


_G_EVAL = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "evaluate.npz"))


@pytest.mark.parametrize("trial", range(6))
def test_evaluate_vs_reference_golden(r2, trial):
    """evaluate() (rift2_evaluate kernel) against the reference's
    evalbench.evaluate outputs: n_correct and success exact, RMSE to 1e-12."""
    g = _G_EVAL
    kr = [r2.Keypoint(float(x), float(y), 1.0, "corner") for x, y in g[f"t{trial}_ref_xy"]]
    kt = [r2.Keypoint(float(x), float(y), 1.0, "corner") for x, y in g[f"t{trial}_tgt_xy"]]
    ms = r2.MatchSet(pairs=[(int(a), int(b), 0.0) for a, b in g[f"t{trial}_pairs"]])
    row = g[f"t{trial}_gt"]
    for j in range(3):
        thr, n, rmse, succ = g[f"t{trial}_thr{j}"]
        gt = np.array([[row[0], row[1], row[4]], [row[2], row[3], row[5]]])
        rep = r2.evaluate(ms, kr, kt, gt, residual_threshold=thr, rmse_cap=2.0 if j == 2 else 20.0)
        assert rep.n_correct == n and rep.success == bool(succ) and rep.n_matches_total == len(ms.pairs)
        assert (np.isinf(rep.rmse) and np.isinf(rmse)) or abs(rep.rmse - rmse) <= 1e-12 * rmse
    bad = r2.MatchSet(pairs=[(0, 0, 0.0), (len(kr), 0, 0.0)])
    with pytest.raises(r2.IntegrityError):
        r2.evaluate(bad, kr, kt, np.eye(2, 3))


def test_evaluate_batch_vs_oracle(r2):
    """evaluate_batch on a BatchPipeline step (1024^2 pairs from the BASELINE
    generator) against the oracle's evaluate on the same keypoints/matches."""
    from paper_2303_00319_b200 import synth
    imgs, truths = synth.make_batch(2, 1024, seed0=40, looks=None)
    pipe = r2.BatchPipeline(2, 1024, 1024, r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75))
    pipe.load(imgs)
    pipe.step()
    ev = r2.evaluate_batch(pipe, truths)
    torch.cuda.synchronize()
    for p, (ri, ti, _) in enumerate(pipe.matches_host()):
        kr, kt = pipe.keypoints_host(2 * p), pipe.keypoints_host(2 * p + 1)
        n, rmse, succ = O.evaluate(np.stack([kr["x"], kr["y"]], 1), np.stack([kt["x"], kt["y"]], 1),
                                   np.stack([ri, ti], 1), truths[p].matrix[:, :2].ravel().tolist()
                                   + truths[p].matrix[:, 2].tolist())
        assert int(ev["n_correct"][p]) == n > 100 and bool(ev["success"][p]) == succ
        assert abs(float(ev["rmse"][p]) - rmse) <= 1e-12 * rmse


def test_run_from_host_pipelined_results(r2):
    """The end-to-end host path (double-buffered uploads, fields-only first
    step, features-only last step): after `steps` steps the pinned output
    holds the matches of batch steps-1, equal to the plain step's."""
    from paper_2303_00319_b200 import synth
    cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=800)
    batches = [synth.make_batch(2, 256, seed0=s)[0] for s in (30, 40, 50)]
    pipe = r2.BatchPipeline(2, 256, 256, cfg)
    want = []
    for imgs in batches:
        pipe.load(imgs)
        pipe.step()
        torch.cuda.synchronize()
        want.append({k: v.clone().cpu() for k, v in pipe.m.items()})
    host = [torch.from_numpy(b).pin_memory() for b in batches]
    out = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in pipe.m.items()}
    for steps in (1, 2, 3):
        for t in out.values():
            t.zero_()
        pipe.run_from_host_pipelined(host, steps, out)
        torch.cuda.synchronize()
        w = want[steps - 1]
        assert torch.equal(w["count"], out["count"]), steps
        for p, n in enumerate(w["count"].tolist()):            # rows past count are stale workspace
            for k in ("ref", "tgt", "dist"):
                assert torch.equal(w[k][p, :n], out[k][p, :n]), (steps, p, k)


@pytest.mark.parametrize("mode", ["ring", "plain"])
def test_batch_pipeline_ring_and_plain_modes(r2, mode):
    """BatchPipeline in the reference's other modes (ref: pipeline.py:53-64:
    ring = n_orient cyclic layers on the reference side against plain
    targets): the same matches as the dataclass API, and the ring reference
    side carries exactly n_orient rows per described keypoint."""
    from paper_2303_00319_b200 import synth
    cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=700, mode=mode)
    imgs, _ = synth.make_batch(2, 256, seed0=7, looks=None)
    pipe = r2.BatchPipeline(2, 256, 256, cfg)
    pipe.load(imgs)
    pipe.capture()
    pipe.step()
    torch.cuda.synchronize()
    res = pipe.matches_host()
    dcount = pipe.d["count"].cpu().numpy()
    for p in range(2):
        api = r2.match_pair(imgs[2 * p].astype(np.float64), imgs[2 * p + 1].astype(np.float64), cfg)
        assert list(zip(res[p][0].tolist(), res[p][1].tolist())) == [(a, b) for a, b, _ in api.matches.pairs]
        np.testing.assert_allclose(res[p][2], [d for _, _, d in api.matches.pairs], rtol=0, atol=0)
        assert dcount[2 * p] == len(api.ref.descriptors) and dcount[2 * p + 1] == len(api.tgt.descriptors)
        if mode == "ring":
            assert dcount[2 * p] == 6 * len({d.keypoint_id for d in api.ref.descriptors})
            assert dcount[2 * p + 1] == len({d.keypoint_id for d in api.tgt.descriptors})

"""configs[4], the rotation-robustness sweep: per-theta agreement of the GPU
pipeline with the CPU oracle.

BASELINE configs[4]: 512^2 pairs, theta in 15-degree steps over 0..345,
scale jitter [0.9, 1.1], speckle looks in {1, 4, 16}; "reports ... per-theta
agreement of dominant index and match sets with the CPU oracle".  One pair
per theta (24 pairs; the looks cycle over theta).  The oracle runs in a
process pool on the host cores, the GPU side through the public API.
Matches are compared as coordinate pairs (the GPU runs its own fp32 filter
bank).  Besides the agreement bars, the report records each side's number
of matches that the generator's transform confirms (< 3 px, ref
evalbench.py:63-96), since with speckle the oracle itself often fails to
register.  The report is written to
$R2_SWEEP_OUT (default: gpurun_out/c5_sweep.json when that directory exists).
"""

import json
import multiprocessing as mp
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

BASE = dict(scale_mult=1.6, sigma_on_f=0.75)
THETAS = list(range(0, 360, 15))
LOOKS = (1, 4, 16)


def _pair(theta):
    from paper_2303_00319_b200 import synth
    looks = LOOKS[(theta // 15) % 3]
    a, b, truth = synth.make_pair(512, seed=5000 + theta, theta_deg=float(theta), scale_jitter=0.1, looks=looks)
    return a.astype(np.float64), b.astype(np.float64), truth, looks


def _oracle_job(theta):
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import rift2_oracle as O
    a, b, truth, _ = _pair(theta)
    sides = []
    for img in (a, b):
        f = O.fields(img, O.Bank(**BASE), workers=1)
        kp = O.detect_keypoints(f["moment_min"], f["moment_max"], 0.001, 5000, 96)
        c, k, v, _ = O.describe_rift2(f["mim"], kp)
        sides.append((kp, c, k, v))
    (rkp, rc, rk, rv), (tkp, tc, tk, tv) = sides
    pairs, _ = O.match_nn(rc / np.linalg.norm(rc, axis=1, keepdims=True), rk,
                          tc / np.linalg.norm(tc, axis=1, keepdims=True), tk)
    m = sorted(((int(rkp["x"][r]), int(rkp["y"][r])), (int(tkp["x"][t]), int(tkp["y"][t]))) for r, t, _ in pairs)
    dom = {(int(rkp["x"][k]), int(rkp["y"][k])): int(v) for k, v in zip(rk[::-1], rv[::-1])}
    return theta, m, sorted(dom.items())


def _confirmed(m, truth):
    if not m:
        return 0
    p = np.array(m, np.float64)
    return int((np.linalg.norm(truth.apply(p[:, 0]) - p[:, 1], axis=1) < 3.0).sum())


def test_rotation_sweep_report():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2303_00319_b200 as r2
    workers = max(1, min(len(os.sched_getaffinity(0)), 24))
    with mp.get_context("spawn").Pool(workers) as pool:
        oracle = {t: (m, dict(d)) for t, m, d in pool.map(_oracle_job, THETAS)}
    rows = []
    for theta in THETAS:
        a, b, truth, looks = _pair(theta)
        res = r2.match_pair(a, b, r2.RiftConfig(max_keypoints=5000, **BASE))
        rkp, tkp = res.ref.keypoints, res.tgt.keypoints
        got = {((int(rkp[r].x), int(rkp[r].y)), (int(tkp[t].x), int(tkp[t].y))) for r, t, _ in res.matches.pairs}
        dg = {}
        for d in reversed(list(res.ref.descriptors)):
            k = rkp[d.keypoint_id]
            dg[(int(k.x), int(k.y))] = int(d.variant)
        want, dw = oracle[theta]
        want = set(want)
        common = set(dw) & set(dg)
        rows.append(dict(theta=theta, looks=looks, oracle_matches=len(want), gpu_matches=len(got),
                         match_overlap=len(got & want) / max(len(want), 1),
                         dominant_agreement=float(np.mean([dw[k] == dg[k] for k in common])) if common else 1.0,
                         dominant_keypoints=len(common),
                         oracle_confirmed=_confirmed(sorted(want), truth),
                         gpu_confirmed=_confirmed(sorted(got), truth)))
    report = dict(config="BASELINE configs[4]: 512^2, theta 0..345 step 15, scale jitter 0.1, looks cycling 1/4/16, "
                         "one pair per theta (seed 5000 + theta)", rows=rows,
                  min_match_overlap=min(r["match_overlap"] for r in rows),
                  min_dominant_agreement=min(r["dominant_agreement"] for r in rows))
    out = os.environ.get("R2_SWEEP_OUT") or ("gpurun_out/c5_sweep.json" if os.path.isdir("gpurun_out") else None)
    if out:
        with open(out, "w") as fh:
            json.dump(report, fh, indent=1)
    for r in rows:
        print(f"theta {r['theta']:3d} looks {r['looks']:2d}: overlap {r['match_overlap']:.4f} "
              f"dominant {r['dominant_agreement']:.4f} matches {r['oracle_matches']}/{r['gpu_matches']} "
              f"confirmed {r['oracle_confirmed']}/{r['gpu_confirmed']}")
    assert report["min_match_overlap"] >= 0.99
    assert report["min_dominant_agreement"] >= 0.99

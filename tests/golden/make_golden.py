"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `rift2` from /root/reference/pkg/src and writes small compressed
fixtures next to this file.  The GPU box never runs this script; it only
reads the committed `.npz` outputs.  The fixtures pin `oracle/` (see
tests/test_oracle_golden.py) and feed the GPU parity tests.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import rift2  # noqa: E402  (the reference)
from rift2 import RiftConfig  # noqa: E402
from rift2.descriptor import describe_plain, describe_rift2, describe_ring  # noqa: E402
from rift2.detector import detect_fast, detect_keypoints  # noqa: E402
from rift2.matcher import match_nn  # noqa: E402
from rift2.pipeline import compute_fields  # noqa: E402
from rift2.synthetic import step_edge, voronoi_label_map  # noqa: E402

from paper_2303_00319_b200 import synth  # noqa: E402

BASE = dict(scale_mult=1.6, sigma_on_f=0.75)   # BASELINE.json params


def kp_arrays(kps):
    return dict(x=np.array([k.x for k in kps], np.int32),
                y=np.array([k.y for k in kps], np.int32),
                response=np.array([k.response for k in kps], np.float64),
                kind=np.array([0 if k.kind == "corner" else 1 for k in kps], np.int8))


def desc_arrays(dset):
    vec = np.array([d.vector for d in dset.descriptors]).reshape(len(dset), -1)
    # vectors are counts / ||counts||: recover the integer counts exactly
    # every 16x16 cell holds 256 samples, so counts = v * 256 / sum_cell(v)
    counts = np.zeros(vec.shape, np.uint16)
    for i, v in enumerate(vec):
        cells = v.reshape(36, -1)
        c = np.rint(cells * (256.0 / cells.sum(1, keepdims=True))).astype(np.int64).ravel()
        counts[i] = c
        assert np.array_equal(c / np.linalg.norm(c.astype(np.float64)), v)
    return dict(counts=counts,
                kp=np.array([d.keypoint_id for d in dset.descriptors], np.int32),
                variant=np.array([d.variant for d in dset.descriptors], np.int8),
                vec=vec.astype(np.float64),
                skipped=np.int64(dset.skipped))


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"{name}: {os.path.getsize(path) / 1e3:.0f} kB")


def case_fields_small():
    """128^2 voronoi (ref tests/test_loggabor.py:16-18) with default and
    BASELINE parameters: every PCField / IndexMap array."""
    img = voronoi_label_map(128, 25, seed=4)
    out = dict(image=img)
    for tag, cfg in (("def", RiftConfig()), ("base", RiftConfig(**BASE))):
        pc, mim = compute_fields(img, cfg)
        out[f"{tag}_a_o"] = pc.a_o.astype(np.float32)
        out[f"{tag}_pc"] = pc.pc_per_orientation.astype(np.float32)
        out[f"{tag}_mmax"] = pc.moment_max
        out[f"{tag}_mmin"] = pc.moment_min
        out[f"{tag}_mim"] = mim.indices.astype(np.int8)
        out[f"{tag}_amax"] = mim.max_amplitude.astype(np.float32)
    step = step_edge(128)
    pc, mim = compute_fields(step, RiftConfig())
    out["step_mmax"] = pc.moment_max
    out["step_mim"] = mim.indices.astype(np.int8)
    save("fields_small.npz", **out)


def case_pair():
    """A 256^2 BASELINE-generator pair (seed 3, 40 deg, no speckle so the
    pair matches): maps, keypoints, RIFT2 / ring / plain descriptors, matches."""
    a, b, truth = synth.make_pair(256, seed=3, theta_deg=40.0, looks=None)
    cfg = RiftConfig(max_keypoints=600, **BASE)
    out = dict(img1=a, img2=b, matrix=truth.matrix)
    sets = {}
    for tag, img in (("r", a), ("t", b)):
        pc, mim = compute_fields(img, cfg)
        out[f"{tag}_mmax"] = pc.moment_max
        out[f"{tag}_mmin"] = pc.moment_min
        out[f"{tag}_mim"] = mim.indices.astype(np.int8)
        kps = detect_keypoints(pc, cfg.fast_threshold, cfg.max_keypoints, cfg.patch_size)
        for k, v in kp_arrays(kps).items():
            out[f"{tag}_kp_{k}"] = v
        for mode, fn in (("rift2", lambda: describe_rift2(mim, kps)),
                         ("norot", lambda: describe_rift2(mim, kps, rotate_patch=False)),
                         ("ring", lambda: describe_ring(mim, kps)),
                         ("plain", lambda: describe_plain(mim, kps))):
            d = fn()
            sets[(tag, mode)] = d
            for k, v in desc_arrays(d).items():
                if k == "vec" or (mode == "ring" and k == "counts"):
                    continue   # ring counts are cyclic rolls of the plain ones
                out[f"{tag}_{mode}_{k}"] = v
    for mode, (rm, tm) in (("rift2", ("rift2", "rift2")), ("ring", ("ring", "plain")),
                           ("plain", ("plain", "plain"))):
        ms = match_nn(sets[("r", rm)].descriptors, sets[("t", tm)].descriptors)
        arr = np.array(ms.pairs, dtype=np.float64).reshape(-1, 3)
        out[f"match_{mode}"] = arr
        out[f"match_{mode}_evals"] = np.int64(ms.distance_evals)
    save("pair256.npz", **out)


def case_detector():
    """detect_fast on hand maps (ref tests/test_detector.py:21-25)."""
    m = np.zeros((64, 64))
    m[30:34, 30:34] = 1.0
    out = {}
    for k, v in kp_arrays(detect_fast(m, 0.001, 100)).items():
        out[f"square_{k}"] = v
    rng = np.random.default_rng(5)
    noise = rng.random((100, 120))
    out["noise_map"] = noise
    for k, v in kp_arrays(detect_fast(noise, 0.001, 300, border_margin=5)).items():
        out[f"noise_{k}"] = v
    # plateaus and duplicated responses: quantised map exercises ties
    q = np.floor(rng.random((120, 110)) * 4) / 4
    out["quant_map"] = q
    for k, v in kp_arrays(detect_fast(q, 0.001, 200)).items():
        out[f"quant_{k}"] = v
    save("detector.npz", **out)


def case_matcher():
    """match_nn on random integer-count descriptor sets with 1-2 variants."""
    rng = np.random.default_rng(11)
    out = {}
    for trial in range(4):
        sets = []
        for side, nk in (("r", 60), ("t", 45)):
            counts, kp = [], []
            for i in range(nk):
                for _ in range(int(rng.integers(1, 3))):
                    c = rng.integers(0, 40, 216).astype(np.uint16)
                    if trial == 3 and side == "t" and i % 5 == 0:
                        c = sets[0][0][i % len(sets[0][0])].copy()   # exact duplicates
                    counts.append(c)
                    kp.append(i)
            sets.append((np.array(counts, np.uint16), np.array(kp, np.int32)))
        descs = []
        for counts, kp in sets:
            descs.append([rift2.Descriptor(c / np.linalg.norm(c.astype(float)), int(k), 1, "rift2")
                          for c, k in zip(counts, kp)])
        ms = match_nn(descs[0], descs[1])
        out[f"t{trial}_r_counts"], out[f"t{trial}_r_kp"] = sets[0]
        out[f"t{trial}_t_counts"], out[f"t{trial}_t_kp"] = sets[1]
        out[f"t{trial}_pairs"] = np.array(ms.pairs, np.float64)
    save("matcher.npz", **out)


def case_container():
    """The RIF2 descriptor container bytes written by the reference
    (ref: descriptor.py:255-268): seeded unit vectors over all three modes,
    plus an empty file."""
    from rift2.descriptor import write_descriptors
    rng = np.random.default_rng(21)
    descs = []
    for i in range(9):
        v = rng.random(216)
        descs.append(rift2.Descriptor(v / np.linalg.norm(v), int(rng.integers(0, 2**32 - 1)), (i % 6) + 1,
                                      ("plain", "ring", "rift2")[i % 3]))
    write_descriptors(os.path.join(HERE, "container.rif2"), descs)
    write_descriptors(os.path.join(HERE, "container_empty.rif2"), [])
    save("container.npz", vec=np.array([d.vector for d in descs]),
         kp=np.array([d.keypoint_id for d in descs], np.uint32),
         variant=np.array([d.variant for d in descs], np.int8),
         mode=np.array([("plain", "ring", "rift2").index(d.mode) for d in descs], np.int8))


def case_evaluate():
    """evalbench.evaluate (ref: evalbench.py:63-96) on seeded keypoints and
    match sets under rigid transforms: matches built to land within, near
    and beyond the residual threshold, several thresholds, empty sets."""
    from rift2.detector import Keypoint
    from rift2.evalbench import evaluate
    from rift2.imaging import RigidTransform
    rng = np.random.default_rng(31)
    out = {}
    for trial in range(6):
        nr, nt = int(rng.integers(50, 400)), int(rng.integers(50, 400))
        rxy = rng.integers(0, 1024, (nr, 2)).astype(np.float64)
        gt = RigidTransform.rotation_about(float(rng.uniform(0, 2 * np.pi)), (512.0, 512.0))
        gt = RigidTransform(gt.rotation, gt.translation + rng.uniform(-20, 20, 2))
        txy = rng.integers(0, 1024, (nt, 2)).astype(np.float64)
        n = 0 if trial == 5 else int(rng.integers(10, min(nr, nt)))
        tsel = rng.permutation(nt)[:n]
        rsel = rng.integers(0, nr, n)
        # a third of the targets placed at the transformed reference point plus a jitter of 0-5 px
        k = n // 3
        jit = rng.uniform(0, 5, k)[:, None] * np.stack([np.cos(a := rng.uniform(0, 6.3, k)), np.sin(a)], 1)
        txy[tsel[:k]] = np.rint(gt.apply(rxy[rsel[:k]]) + jit)
        kr = [Keypoint(float(x), float(y), 1.0, "corner") for x, y in rxy]
        kt = [Keypoint(float(x), float(y), 1.0, "corner") for x, y in txy]
        ms = rift2.MatchSet(pairs=[(int(r), int(t), 0.0) for r, t in zip(rsel, tsel)])
        row = np.array([*gt.rotation.ravel(), *gt.translation], np.float64)
        out[f"t{trial}_ref_xy"], out[f"t{trial}_tgt_xy"], out[f"t{trial}_gt"] = rxy, txy, row
        out[f"t{trial}_pairs"] = np.stack([rsel, tsel], 1).astype(np.int32).reshape(n, 2)
        for j, thr in enumerate((3.0, 1.5, 0.5)):
            rep = evaluate(ms, kr, kt, gt, residual_threshold=thr, success_min_matches=10, rmse_cap=2.0 if j == 2 else 20.0)
            out[f"t{trial}_thr{j}"] = np.array([thr, rep.n_correct, rep.rmse, float(rep.success)], np.float64)
    save("evaluate.npz", **out)


def desc_counts_general(dset, grid, cs):
    """Integer counts of a descriptor set for any grid / cell size: every
    cell holds cs^2 samples, so counts = v * cs^2 / sum_cell(v)."""
    vec = np.array([d.vector for d in dset.descriptors]).reshape(len(dset), -1)
    counts = np.zeros(vec.shape, np.uint16)
    for i, v in enumerate(vec):
        cells = v.reshape(grid * grid, -1)
        c = np.rint(cells * (cs * cs / cells.sum(1, keepdims=True))).astype(np.int64).ravel()
        counts[i] = c
        assert np.array_equal(c / np.linalg.norm(c.astype(np.float64)), v)
    return dict(counts=counts,
                kp=np.array([d.keypoint_id for d in dset.descriptors], np.int32),
                variant=np.array([d.variant for d in dset.descriptors], np.int8),
                skipped=np.int64(dset.skipped))


def case_desc_general():
    """Descriptors outside the BASELINE shape, from the reference itself:
    fractional keypoints (ref: descriptor.py:118-125), 8 orientations, 12-
    and 24-pixel cells.  Index maps from compute_fields of a 224^2 image."""
    from rift2.detector import Keypoint
    a, _, _ = synth.make_pair(224, seed=5, theta_deg=20.0, looks=None)
    rng = np.random.default_rng(21)
    out = {}
    # keypoints: fractional (incl. exact halves and a few integers), some near the border (skips)
    n = 90
    xs = rng.uniform(20.0, 204.0, n)
    ys = rng.uniform(20.0, 204.0, n)
    xs[:10] = np.floor(xs[:10]) + 0.5
    ys[5:15] = np.floor(ys[5:15]) + 0.5
    xs[15:20] = np.floor(xs[15:20])
    ys[15:20] = np.floor(ys[15:20])
    kps = [Keypoint(float(x), float(y), 1.0, "corner") for x, y in zip(xs, ys)]
    out["kp_x"], out["kp_y"] = xs, ys
    for tag, n_orient, patch, grid in (("o6", 6, 96, 6), ("o8", 8, 64, 4), ("c12", 6, 72, 6), ("c24", 6, 96, 4)):
        cfg = RiftConfig(n_orient=n_orient, **BASE)
        _, mim = compute_fields(a, cfg)
        out[f"{tag}_mim"] = mim.indices.astype(np.int8)
        cs = patch // grid
        for mode, fn in (("rift2", lambda: describe_rift2(mim, kps, patch_size=patch, grid=grid)),
                         ("ring", lambda: describe_ring(mim, kps, patch_size=patch, grid=grid)),
                         ("plain", lambda: describe_plain(mim, kps, patch_size=patch, grid=grid))):
            for k, v in desc_counts_general(fn(), grid, cs).items():
                out[f"{tag}_{mode}_{k}"] = v
    save("desc_general.npz", **out)


CASES = dict(desc_general=case_desc_general, fields_small=case_fields_small, detector=case_detector, matcher=case_matcher, pair=case_pair,
             container=case_container, evaluate=case_evaluate)

if __name__ == "__main__":
    for name in (sys.argv[1:] or CASES):
        CASES[name]()

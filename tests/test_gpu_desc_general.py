"""Descriptors outside the BASELINE shape on the GPU, against the reference.

The fixture tests/golden/desc_general.npz was written by the reference
itself (tests/golden/make_golden.py case_desc_general): fractional keypoint
coordinates (ref: descriptor.py:118-125, floor(x + ux + 0.5) in float64,
including exact halves), 8 orientations, 12- and 24-pixel cells, in the
rift2 / ring / plain modes.  The dataclass API routes fractional keypoints
through rift2_describe_f64 and the other shapes through the generic kernel;
counts, keypoint ids, variants and skip counts must be identical, and the
float64 vectors bit-equal to the reference's.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "desc_general.npz")
SHAPES = {"o6": (6, 96, 6), "o8": (8, 64, 4), "c12": (6, 72, 6), "c24": (6, 96, 4)}


@pytest.fixture(scope="module")
def gold():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return np.load(GOLD)


def _counts(dset, grid, cs):
    vec = np.array([d.vector for d in dset.descriptors]).reshape(len(dset), -1)
    out = np.zeros(vec.shape, np.int64)
    for i, v in enumerate(vec):
        cells = v.reshape(grid * grid, -1)
        out[i] = np.rint(cells * (cs * cs / cells.sum(1, keepdims=True))).astype(np.int64).ravel()
    return vec, out


@pytest.mark.parametrize("tag", list(SHAPES))
@pytest.mark.parametrize("mode", ["rift2", "ring", "plain"])
def test_describe_general_vs_reference(gold, tag, mode):
    from paper_2303_00319_b200 import descriptor
    from paper_2303_00319_b200.detector import Keypoint
    from paper_2303_00319_b200.mim import IndexMap
    n_orient, patch, grid = SHAPES[tag]
    idx = gold[f"{tag}_mim"].astype(np.int32)
    mim = IndexMap(idx, np.zeros(idx.shape), n_orient)
    kps = [Keypoint(float(x), float(y), 1.0, "corner") for x, y in zip(gold["kp_x"], gold["kp_y"])]
    fn = {"rift2": descriptor.describe_rift2, "ring": descriptor.describe_ring, "plain": descriptor.describe_plain}[mode]
    got = fn(mim, kps, patch_size=patch, grid=grid)
    vec, counts = _counts(got, grid, patch // grid)
    want = gold[f"{tag}_{mode}_counts"].astype(np.int64)
    assert int(got.skipped) == int(gold[f"{tag}_{mode}_skipped"])
    assert counts.shape == want.shape
    assert np.array_equal(counts, want)
    assert np.array_equal([d.keypoint_id for d in got.descriptors], gold[f"{tag}_{mode}_kp"])
    assert np.array_equal([d.variant for d in got.descriptors], gold[f"{tag}_{mode}_variant"])
    # the reference's float64 vector is counts / ||counts||, bit for bit
    assert np.array_equal(vec, want / np.linalg.norm(want.astype(np.float64), axis=1, keepdims=True))


def test_integral_float64_keypoints_equal_int32_path(gold):
    # rift2_describe_f64 with integral coordinates gives rift2_describe's result (BASELINE shape)
    from paper_2303_00319_b200 import engine
    idx = torch.as_tensor(gold["o6_mim"].astype(np.uint8)).cuda()[None]
    xs = np.floor(gold["kp_x"]).astype(np.int64)
    ys = np.floor(gold["kp_y"]).astype(np.int64)
    cnt = torch.tensor([len(xs)], dtype=torch.int32, device="cuda")
    a = engine.describe(idx, torch.as_tensor(xs, dtype=torch.int32).cuda()[None],
                        torch.as_tensor(ys, dtype=torch.int32).cuda()[None], cnt, 6, ws_key="t_i")
    b = engine.describe(idx, torch.as_tensor(xs, dtype=torch.float64).cuda()[None],
                        torch.as_tensor(ys, dtype=torch.float64).cuda()[None], cnt, 6, ws_key="t_f")
    n = int(a["count"][0])
    assert n == int(b["count"][0]) and int(a["skipped"][0]) == int(b["skipped"][0])
    for k in ("counts", "sqnorm", "kp", "variant"):
        assert torch.equal(a[k][0, :n], b[k][0, :n]), k


def test_preshift_workspace_equals_transform_path(gold):
    # rift2_describe with the smaller workspace (in-kernel shift transform of
    # the staged neighbourhood), with room for the shift-byte copy of the maps
    # only, and with the height/width-aware size (shift-byte copy + dense
    # 16 x 16 cell sums for the axis-aligned patches) gives identical rows
    import ctypes
    from paper_2303_00319_b200 import _lib, engine
    lib = _lib.load(require_gpu=True)
    idx = torch.as_tensor(gold["o6_mim"].astype(np.uint8)).cuda()[None].contiguous()
    _, H, W = idx.shape
    xs = torch.as_tensor(np.floor(gold["kp_x"]), dtype=torch.int32).cuda()[None].contiguous()
    ys = torch.as_tensor(np.floor(gold["kp_y"]), dtype=torch.int32).cuda()[None].contiguous()
    S = xs.shape[1]
    cnt = torch.tensor([S], dtype=torch.int32, device="cuda")
    outs = []
    small, full = ctypes.c_size_t(), ctypes.c_size_t()
    _lib.check(lib.rift2_describe_workspace_size(1, S, 6, 6, ctypes.byref(small)), "ws")
    _lib.check(lib.rift2_describe_workspace_size_hw(1, H, W, S, 6, 6, ctypes.byref(full)), "ws")
    # the size in between holds the shift-byte copy but not the dense cell
    # sums (k_cell_sums): the axis-aligned patch is then counted per keypoint
    mid = small.value + ((H * W + 255) & ~255)
    assert small.value < mid < full.value
    for nbytes in (small.value, mid, full.value):
        ws = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        o = dict(counts=torch.zeros((1, 2 * S, 224), dtype=torch.float16, device="cuda"),
                 sqnorm=torch.zeros((1, 2 * S), dtype=torch.int32, device="cuda"),
                 kp=torch.zeros((1, 2 * S), dtype=torch.int32, device="cuda"),
                 variant=torch.zeros((1, 2 * S), dtype=torch.uint8, device="cuda"),
                 count=torch.zeros((1,), dtype=torch.int32, device="cuda"),
                 skipped=torch.zeros((1,), dtype=torch.int32, device="cuda"))
        p = engine._ptr
        rc = lib.rift2_describe(p(idx), 1, H, W, 6, p(xs), p(ys), p(cnt), S, 96, 6, 0.8, 1, 2, p(o["counts"]), 224,
                                2 * S, p(o["sqnorm"]), p(o["kp"]), p(o["variant"]), p(o["count"]), p(o["skipped"]),
                                p(ws), ws.numel(), engine._stream())
        _lib.check(rc, "rift2_describe")
        outs.append(o)
    torch.cuda.synchronize()
    a = outs[0]
    n = int(a["count"][0])
    for b in outs[1:]:
        assert n == int(b["count"][0]) and n > 0 and int(a["skipped"][0]) == int(b["skipped"][0])
        for k in ("counts", "sqnorm", "kp", "variant"):
            assert torch.equal(a[k][0, :n], b[k][0, :n]), k

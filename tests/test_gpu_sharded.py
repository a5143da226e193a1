"""Row-sharded matching (SURVEY 8(e), configs[3]) on one GPU.

G ranks are simulated sequentially in one process (slices described,
partials computed, gathered by concatenation -- no rank ever waits on
another), and the exact combine must reproduce the single-call matcher
bit for bit.  The multi-process orchestration itself is covered on CPU by
tests/test_multirank.py (gloo, world size 2).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2303_00319_b200 as r2
    from paper_2303_00319_b200 import sharded, synth
    a, b, _ = synth.make_pair(512, seed=6)
    cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75)
    be = sharded.GpuBackend()
    feats = [be.features(img, cfg) for img in (a, b)]
    full = [be.describe_slice(f, 0, f["n"], cfg) for f in feats]
    return r2, sharded, be, cfg, feats, full, (a, b)


def _simulate(sharded, be, cfg, feats, G):
    """G ranks in sequence: only image 2's slices are concatenated (the
    all-gather); image 1's stay per rank, and each rank's finish supplies
    the distances of the winners it owns."""
    dim = cfg.grid * cfg.grid * cfg.n_orient
    loc = [[be.describe_slice(f, *sharded.kp_range(f["n"], r, G), cfg) for r in range(G)] for f in feats]
    full = [{k: torch.cat([l[k] for l in per_rank]) for k in per_rank[0]} for per_rank in loc]
    parts = torch.stack([be.partial(loc[0][r], full[1], dim) for r in range(G)])
    mine = [be.finish_local(parts, loc[0][r], full[1], feats[0]["n"], feats[1]["n"], dim) for r in range(G)]
    if G > 1:
        assert any(np.isinf(m[2]).any() for m in mine)         # some winners are owned elsewhere
    return full, sharded.merge_triples(mine)


@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_sharded_equals_single(setup, G):
    r2, sharded, be, cfg, feats, full, (a, b) = setup
    gathered, (ref, tgt, dst) = _simulate(sharded, be, cfg, feats, G)
    # concatenated slices reproduce the single-call descriptor arrays exactly
    for k in ("counts", "sqnorm", "kp", "variant"):
        assert torch.equal(gathered[0][k], full[0][k]) and torch.equal(gathered[1][k], full[1][k]), k
    want = r2.match_pair(a, b, cfg).matches.pairs
    assert len(want) > 50
    assert list(zip(ref.tolist(), tgt.tolist())) == [(p[0], p[1]) for p in want]
    assert np.array_equal(dst, np.array([p[2] for p in want]))


def test_orchestration_single_process(setup):
    r2, sharded, be, cfg, feats, full, (a, b) = setup
    ms, info = sharded.match_pair_sharded(a, b, cfg)
    assert info["world"] == 1
    assert ms.pairs == r2.match_pair(a, b, cfg).matches.pairs

"""The target-synthesis checker (oracle/synth_oracle.py) pinned on the CPU:
Philox4x32-10 against its published known answers, the warp and radiometry
against the host generator (synth.make_pair), the speckle's moments."""

import numpy as np
import pytest

from oracle import synth_oracle as S
from paper_2303_00319_b200 import synth

# Random123 philox4x32-10 known-answer vectors: (counter, key) -> output
KAT = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
       ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
       ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
        (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers(ctr, key, want):
    got = S.philox4x32_10(*ctr, *key)
    assert tuple(int(v) for v in got) == want


def test_uniforms_in_unit_interval():
    assert S.uniforms53(0, 0) == 2.0 ** -53
    assert S.uniforms53(0xFFFFFFFF, 0xFFFFFFFF) == 1.0


@pytest.mark.parametrize("theta,jitter", [(0.0, 0.0), (90.0, 0.0), (37.5, 0.1), (200.0, 0.05)])
def test_warp_matches_host_generator(theta, jitter):
    img = synth.blob_field(96, seed=3)
    tr, _ = synth._pair_draws(96, 3, theta, jitter, None)
    assert np.array_equal(S.warp(img, synth.inverse_map(tr.matrix)), synth.warp(img, tr.matrix))


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_target_without_speckle_matches_make_pair(seed):
    img1, img2, tr = synth.make_pair(96, seed, looks=None)
    got = S.synth_target(img1, synth.inverse_map(tr.matrix), tr.inverted, tr.gamma, 0, seed=0)
    assert np.array_equal(got, img2)


@pytest.mark.parametrize("looks", [1, 4, 16])
def test_speckle_moments(looks):
    s = S.speckle(256, 256, image=5, looks=looks, seed=123)
    assert s.min() > 0
    n = s.size
    assert abs(s.mean() - 1.0) < 5 * np.sqrt(1.0 / looks / n)
    assert abs(s.var() - 1.0 / looks) < 0.05 / looks
    # independent streams per image and per seed
    assert not np.array_equal(s, S.speckle(256, 256, image=6, looks=looks, seed=123))
    assert not np.array_equal(s, S.speckle(256, 256, image=5, looks=looks, seed=124))

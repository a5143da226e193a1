"""The drop-in boundary: the reference package `rift2`
switched onto this library, either by aliasing it before import or by
rebinding an imported copy (paper_2303_00319_b200.dropin).

CPU tests check the wiring -- every hot-path name the reference's callers
bound at import time (ref: pipeline.py:16-23, evalbench.py:25-30,
estimator.py:17-21, __init__.py:10-29) resolves to this library.  GPU tests
run the reference's own front ends and count the C-ABI calls each stage
makes, proving nothing stays on the CPU.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.skipif(not os.path.exists(os.path.join(REF, "rift2", "__init__.py")),
                                reason="reference not installed (oracle/build_ref.sh)")


def _run(code: str):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, REF]))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return r.stdout


HOT = {
    "pipeline": ["compute_fields", "extract_features", "match_pair", "describe", "detect_keypoints",
                 "describe_rift2", "describe_ring", "describe_plain", "apply_bank", "build_filter_bank",
                 "phase_congruency_moments", "orientation_amplitudes", "build_mim", "PCField", "IndexMap"],
    "evalbench": ["match_nn", "describe", "match_pair", "keypoints_xy", "MatchSet"],
    "estimator": ["extract_features", "match_nn", "keypoints_xy", "FeatureSet", "MatchSet", "RiftConfig"],
    "descriptor": ["cyclic_shift", "dominant_indices", "patch_histogram", "recode", "IndexMap", "Keypoint"],
    "detector": ["PCField"],
}


def test_install_rebinds_every_by_name_import():
    out = _run(f"""
import rift2, rift2.evalbench, rift2.estimator, rift2.cli
from paper_2303_00319_b200 import dropin
n = dropin.install(rift2)
assert n > 100, n
bad = []
for mod, names in {HOT!r}.items():
    m = getattr(rift2, mod)
    for name in names:
        obj = getattr(m, name)
        if not obj.__module__.startswith("paper_2303_00319_b200"):
            bad.append(f"{{mod}}.{{name}} -> {{obj.__module__}}")
for name in rift2.__all__:
    obj = getattr(rift2, name)
    mod = getattr(obj, "__module__", "")
    if name in ("RiftFeatureExtractor", "RiftMatcher", "RigidTransform", "BenchReport", "DatasetSummary",
                "EvalReport", "PairSpec", "benchmark", "dataset_eval", "evaluate", "load_manifest",
                "load_image", "save_image", "warp_rigid", "check_image"):
        continue                         # front ends / imaging stay the reference's
    if not mod.startswith("paper_2303_00319_b200"):
        bad.append(f"rift2.{{name}} -> {{mod}}")
assert not bad, bad
dropin.uninstall()
assert rift2.pipeline.detect_keypoints.__module__ == "rift2.detector"
print("ok", n)
""")
    assert out.startswith("ok")


def test_alias_resolves_hot_modules_to_this_package():
    out = _run("""
from paper_2303_00319_b200 import dropin
rift2 = dropin.alias()
import rift2.estimator, rift2.evalbench, rift2.cli, rift2.synthetic
import paper_2303_00319_b200 as ours
for sub in dropin.HOT_MODULES:
    assert getattr(rift2, sub) is getattr(ours, sub) or getattr(rift2, sub).__name__ == "paper_2303_00319_b200." + sub, sub
assert rift2.estimator.extract_features is ours.pipeline.extract_features
assert rift2.estimator.match_nn is ours.matcher.match_nn
assert rift2.evalbench.match_nn is ours.matcher.match_nn
assert rift2.evalbench.pipeline is ours.pipeline
assert rift2.cli.match_pair is ours.pipeline.match_pair
assert rift2.RiftMatcher.__module__ == "rift2.estimator"     # the reference's own front end
assert rift2.ParameterError is ours.ParameterError
print("ok")
""")
    assert out.startswith("ok")


# ------------------------------------------------------------------ on a GPU
@pytest.mark.gpu
def test_reference_front_ends_route_every_stage_to_the_library():
    """The reference's match_pair, evalbench.benchmark and RiftMatcher, after
    install(): each stage's C-ABI entry point is called, and the results
    equal this library's own API."""
    out = _run("""
import numpy as np, torch
if not torch.cuda.is_available():
    print("skip"); raise SystemExit
import rift2, rift2.evalbench, rift2.estimator
from paper_2303_00319_b200 import dropin, _lib, synth
import paper_2303_00319_b200 as ours
dropin.install(rift2)
a, b, _ = synth.make_pair(256, seed=2, looks=None)
cfg = rift2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=600)
_lib.CALLS.clear()
res = rift2.pipeline.match_pair(a, b, cfg)
calls = dict(_lib.CALLS)
for k in ("rift2_fields", "rift2_detect", "rift2_describe", "rift2_match"):
    assert calls.get(k, 0) >= 1, (k, calls)
want = ours.match_pair(a, b, ours.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=600))
assert res.matches.pairs == want.matches.pairs and len(want.matches.pairs) > 20
_lib.CALLS.clear()
rep = rift2.evalbench.benchmark(a, b, cfg)
calls = dict(_lib.CALLS)
for k in ("rift2_fields", "rift2_detect", "rift2_describe", "rift2_match"):
    assert calls.get(k, 0) >= 1, (k, calls)
_lib.CALLS.clear()
m = rift2.RiftMatcher(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=600).fit(a)
xy = m.predict(b)
calls = dict(_lib.CALLS)
for k in ("rift2_fields", "rift2_detect", "rift2_describe", "rift2_match"):
    assert calls.get(k, 0) >= 1, (k, calls)
assert xy.shape[1] == 4 and len(xy) == len(want.matches.pairs)
print("ok", calls)
""")
    assert out.startswith("ok") or out.startswith("skip")

"""Drop-in redirection of the reference package `rift2` to this library.

Two ways to switch an existing user of the reference:

* ``alias(ref_dir)`` -- before anything imports ``rift2``: makes ``import
  rift2`` resolve to a hybrid package whose hot-path modules (config, errors,
  loggabor, mim, detector, descriptor, matcher, pipeline) ARE this package's
  modules, while the reference's own front ends (imaging, evalbench,
  estimator, cli, synthetic, viz, and the package ``__init__``) are loaded
  from the reference source in ``ref_dir`` under the ``rift2`` name -- so
  their ``from .pipeline import match_pair`` bind this library's functions
  and dataclasses.  The reference's own test modules run against it this
  way (tests/test_ref_suite.py).

* ``install(rift2)`` -- on an already imported reference package: every
  attribute of every ``rift2.*`` module that IS one of the reference's
  hot-path functions or dataclasses is rebound to this library's
  counterpart.  Identity matching catches the names bound at import time
  (``rift2.pipeline``'s ``from .detector import detect_keypoints``,
  ``rift2.evalbench``'s ``from .matcher import match_nn``,
  ``rift2.estimator``'s ``extract_features`` / ``match_nn``, the package
  namespace itself), which patching only the defining modules would miss.
  ``uninstall()`` restores the originals.
"""

from __future__ import annotations

import importlib
import importlib.abc
import importlib.util
import os
import sys

HOT_MODULES = ("config", "errors", "loggabor", "mim", "detector", "descriptor", "matcher", "pipeline")
_PKG = __name__.rsplit(".", 1)[0]


def default_ref_dir() -> str:
    """baseline/_ref (oracle/build_ref.sh installs the reference there)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    return os.path.join(root, "baseline", "_ref")


class _RefFinder(importlib.abc.MetaPathFinder):
    """Finds `rift2` (the reference __init__) and its non-hot-path modules in
    the reference source; hot-path modules are pre-seeded in sys.modules."""

    def __init__(self, ref_dir: str):
        self.pkg_dir = os.path.join(ref_dir, "rift2")

    def find_spec(self, fullname, path=None, target=None):
        if fullname == "rift2":
            return importlib.util.spec_from_file_location(
                "rift2", os.path.join(self.pkg_dir, "__init__.py"), submodule_search_locations=[self.pkg_dir])
        if fullname.startswith("rift2."):
            sub = fullname.split(".", 1)[1]
            if sub in HOT_MODULES or "." in sub:
                return None
            f = os.path.join(self.pkg_dir, sub + ".py")
            if os.path.exists(f):
                return importlib.util.spec_from_file_location(fullname, f)
        return None


_finder = None


def alias(ref_dir: str | None = None):
    """Make `import rift2` resolve to the hybrid package (see module doc) and
    return it."""
    global _finder
    ref_dir = ref_dir or default_ref_dir()
    if not os.path.exists(os.path.join(ref_dir, "rift2", "__init__.py")):
        raise FileNotFoundError(f"no reference package under {ref_dir} (run oracle/build_ref.sh)")
    for name in [m for m in sys.modules if m == "rift2" or m.startswith("rift2.")]:
        del sys.modules[name]
    for sub in HOT_MODULES:
        sys.modules[f"rift2.{sub}"] = importlib.import_module(f"{_PKG}.{sub}")
    if _finder is not None and _finder in sys.meta_path:
        sys.meta_path.remove(_finder)
    _finder = _RefFinder(ref_dir)
    sys.meta_path.insert(0, _finder)
    pkg = importlib.import_module("rift2")
    for sub in HOT_MODULES:                     # pre-seeded modules are not bound on the package by import
        setattr(pkg, sub, sys.modules[f"rift2.{sub}"])
    return pkg


def unalias() -> None:
    global _finder
    if _finder is not None and _finder in sys.meta_path:
        sys.meta_path.remove(_finder)
    _finder = None
    for name in [m for m in sys.modules if m == "rift2" or m.startswith("rift2.")]:
        del sys.modules[name]


_saved: list = []


def _ours():
    """(reference module name, attribute) -> this package's object."""
    table = {}
    for sub in HOT_MODULES:
        mod = importlib.import_module(f"{_PKG}.{sub}")
        for name, obj in vars(mod).items():
            if not name.startswith("__"):
                table[(sub, name)] = obj
    return table


def install(rift2=None) -> int:
    """Rebind an imported reference package onto this library; returns the
    number of attributes rebound."""
    if rift2 is None:
        import rift2  # noqa: F811  (the reference, importable on sys.path)
    ours = _ours()
    # the reference's own objects behind each hot-path name
    originals = {}
    for sub in HOT_MODULES:
        mod = sys.modules.get(f"{rift2.__name__}.{sub}") or importlib.import_module(f"{rift2.__name__}.{sub}")
        for name, obj in list(vars(mod).items()):
            if (sub, name) in ours and not name.startswith("__") and (callable(obj) or isinstance(obj, type)):
                if getattr(obj, "__module__", "").startswith(rift2.__name__):
                    originals[id(obj)] = (obj, ours[(sub, name)])
    n = 0
    mods = [m for k, m in list(sys.modules.items())
            if m is not None and (k == rift2.__name__ or k.startswith(rift2.__name__ + "."))]
    for mod in mods:
        for name, obj in list(vars(mod).items()):
            hit = originals.get(id(obj))
            if hit is not None and hit[0] is obj:
                _saved.append((mod, name, obj))
                setattr(mod, name, hit[1])
                n += 1
    return n


def uninstall() -> None:
    while _saved:
        mod, name, obj = _saved.pop()
        setattr(mod, name, obj)

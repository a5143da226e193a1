"""Brute-force nearest-neighbour matching, drop-in for
ref: pkg/src/rift2/matcher.py:28-148.

Descriptors carrying integer histogram counts (everything describe_*
produces) go through the tcgen05 tensor-core kernel with an exact integer
ranking; arbitrary float vectors go through the float64 CUDA kernel that
evaluates the reference's own key.  Both return one match per target
keypoint, sorted by (distance, ref id, tgt id).
"""

from __future__ import annotations

import csv
import io
import json
from dataclasses import dataclass, field

import numpy as np

from .errors import ParameterError

TENSOR_K = 224   # descriptor length the tensor-core tiles cover
# ref: matcher.py:25 -- the reference's target block size.  The GPU kernels
# tile the distance matrix on their own; the name is kept so callers that
# tune it (e.g. ref tests/test_matcher.py:105-111) keep working, and results
# do not depend on it.
_TARGET_BLOCK = 1024


@dataclass
class MatchSet:
    pairs: list = field(default_factory=list)
    mode: str = "plain"
    distance_evals: int = 0

    def __len__(self):
        return len(self.pairs)

    def to_json_list(self) -> list:
        return [{"ref": r, "tgt": t, "dist": d} for r, t, d in self.pairs]

    @classmethod
    def from_json_list(cls, items, mode: str = "plain") -> "MatchSet":
        return cls(pairs=[(int(d["ref"]), int(d["tgt"]), float(d["dist"])) for d in items], mode=mode)

    def to_csv_text(self) -> str:
        buf = io.StringIO()
        w = csv.writer(buf)
        w.writerow(["ref", "tgt", "dist"])
        for r, t, d in self.pairs:
            w.writerow([r, t, repr(d)])
        return buf.getvalue()

    def save_json(self, path) -> None:
        with open(path, "w") as fh:
            json.dump(self.to_json_list(), fh, indent=2)

    def save_csv(self, path) -> None:
        with open(path, "w") as fh:
            fh.write(self.to_csv_text())


def _grouped(descs):
    """Stable order by keypoint id (ref: matcher.py:67-79) + dense ids."""
    ids = np.array([d.keypoint_id for d in descs], dtype=np.int64)
    order = np.argsort(ids, kind="stable")
    uniq, dense = np.unique(ids[order], return_inverse=True)
    return order, uniq, dense.astype(np.int32)


def _match_counts(ref_descs, tgt_descs):
    import torch
    from . import engine
    r_ord, r_ids, r_dense = _grouped(ref_descs)
    t_ord, t_ids, t_dense = _grouped(tgt_descs)
    nr, nt = len(ref_descs), len(tgt_descs)
    cap = max(nr, nt)
    dim = len(ref_descs[0].counts)
    counts = np.zeros((2, cap, TENSOR_K), np.float16)
    sq = np.zeros((2, cap), np.int32)
    kp = np.zeros((2, cap), np.int32)
    for side, (descs, order, dense) in enumerate(((ref_descs, r_ord, r_dense), (tgt_descs, t_ord, t_dense))):
        src = getattr(descs[0], "_src", None)
        if src is not None and all(getattr(d, "_src", None) is src for d in descs):
            # rows of one describe call's count matrix: one fancy-index gather
            rows = np.fromiter((d._row for d in descs), dtype=np.int64, count=len(descs))
            c = src[rows[order]]
        else:
            c = np.stack([descs[i].counts for i in order]).astype(np.int64)
        counts[side, :len(order), :dim] = c
        sq[side, :len(order)] = (c * c).sum(1)
        kp[side, :len(order)] = dense
    desc = dict(counts=torch.from_numpy(counts).cuda(), sqnorm=torch.from_numpy(sq).cuda(),
                kp=torch.from_numpy(kp).cuda(), count=torch.tensor([nr, nt], dtype=torch.int32, device="cuda"))
    blocks = torch.tensor([0, 1], dtype=torch.int32, device="cuda")
    out = engine.match(desc, dim, blocks[:1], blocks[1:], len(t_ids))
    n = int(out["count"][0])
    return (r_ids[out["ref"][0, :n].cpu().numpy()], t_ids[out["tgt"][0, :n].cpu().numpy()],
            out["dist"][0, :n].cpu().numpy())


def _match_vectors(ref_descs, tgt_descs):
    import torch
    from . import engine
    r_ord, r_ids, r_dense = _grouped(ref_descs)
    t_ord, t_ids, t_dense = _grouped(tgt_descs)
    R = np.stack([np.asarray(ref_descs[i].vector, np.float64) for i in r_ord])
    T = np.stack([np.asarray(tgt_descs[i].vector, np.float64) for i in t_ord])
    if R.shape[1] != T.shape[1]:
        raise ParameterError("descriptor dimensions differ")
    out = engine.match_vectors(torch.from_numpy(R).cuda(), torch.from_numpy(r_dense).cuda(),
                               torch.from_numpy(T).cuda(), torch.from_numpy(t_dense).cuda())
    n = int(out["count"][0])
    return (r_ids[out["ref"][:n].cpu().numpy()], t_ids[out["tgt"][:n].cpu().numpy()],
            out["dist"][:n].cpu().numpy())


def match_nn(ref_descs, tgt_descs, mode: str | None = None) -> MatchSet:
    """Nearest-reference match for every target keypoint (ref: matcher.py:102-148)."""
    if not ref_descs or not tgt_descs:
        raise ParameterError("descriptor lists must be nonempty")
    if mode is None:
        mode = ref_descs[0].mode
    exact = all(getattr(d, "counts", None) is not None for d in ref_descs) and \
        all(getattr(d, "counts", None) is not None for d in tgt_descs) and \
        len(ref_descs[0].counts) <= TENSOR_K and len(ref_descs[0].counts) == len(tgt_descs[0].counts)
    r, t, d = (_match_counts if exact else _match_vectors)(ref_descs, tgt_descs)
    pairs = [(int(a), int(b), float(c)) for a, b, c in zip(r, t, d)]
    return MatchSet(pairs=pairs, mode=mode, distance_evals=len(ref_descs) * len(tgt_descs))

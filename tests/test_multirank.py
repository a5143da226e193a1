"""Multi-rank host logic of bench.py on CPU (gloo, world size 2).

The GPU path shards independent pairs over ranks with no data-path
collective; what must hold across processes is the
seed partition, the max-over-ranks timing reduction and rank-0-only output
of the reference arm.  Runs here without a GPU.
"""

import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as tmp  # noqa: E402
import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        pairs = 16
        seeds = list(range(bench.rank_seed0(rank, pairs), bench.rank_seed0(rank, pairs) + pairs))
        gathered = [None] * world
        dist.all_gather_object(gathered, seeds)
        # rank r reports (step ms, e2e ms, fields ms); the slowest rank must win each entry
        mine = [10.0 + rank, 50.0 - rank, 3.0 * (rank + 1)]
        red = bench.max_over_ranks(mine, world, "cpu")
        out[rank] = (gathered, red)
    finally:
        dist.destroy_process_group()


def test_seed_partition_and_max_reduction():
    world = 2
    port = _free_port()
    mgr = tmp.Manager()
    out = mgr.dict()
    tmp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        gathered, red = out[rank]
        flat = [s for part in gathered for s in part]
        assert sorted(flat) == list(range(32)) and len(set(flat)) == 32     # disjoint, complete
        assert red == [11.0, 50.0, 6.0]


def test_reference_arm_is_rank0_only(capsys):
    sys.path.insert(0, ROOT)
    import bench

    class A:
        steps, warmup, size, pairs = 1, 0, 64, 1

    bench.run_reference(A, rank=1, world=2)        # must return at once without work or output
    assert capsys.readouterr().out == ""


# ---------------------------------------------------------------------------
# Row-sharded matching (paper_2303_00319_b200/sharded.py) under gloo, with a
# CPU backend built on the oracle and exact integer arithmetic in place of
# the CUDA kernels: the orchestration (slices, global keypoint ids, gathers in
# rank order, the exact combine of the partials) is what is under test.

class NumpyBackend:
    def features(self, image, cfg):
        from oracle import rift2_oracle as O
        f = O.fields(np.asarray(image, dtype=np.float64), O.Bank(**BASE), workers=1)
        kp = O.detect_keypoints(f["moment_min"], f["moment_max"], cfg.fast_threshold, cfg.max_keypoints,
                                cfg.patch_size)
        return {"mim": f["mim"], "kp": kp, "n": len(kp)}

    def describe_slice(self, feat, k0, k1, cfg):
        from oracle import rift2_oracle as O
        c, k, v, _ = O.describe_rift2(feat["mim"], feat["kp"][k0:k1])
        c = np.asarray(c, dtype=np.int64).reshape(-1, 216)
        return {"counts": torch.as_tensor(c), "sqnorm": torch.as_tensor((c * c).sum(1)),
                "kp": torch.as_tensor(np.asarray(k, dtype=np.int64) + k0),
                "variant": torch.as_tensor(np.asarray(v, dtype=np.int64))}

    @staticmethod
    def _beats(Da, qa, Db, qb):          # D_a^2 / q_a > D_b^2 / q_b, exactly
        return Da * Da * qb > Db * Db * qa

    def partial(self, ref, tgt, dim):
        R, T = ref["counts"].numpy(), tgt["counts"].numpy()
        qr, rk = ref["sqnorm"].numpy(), ref["kp"].numpy()
        D = T @ R.T if len(R) else np.zeros((len(T), 0), dtype=np.int64)
        out = np.zeros((len(T), 4), dtype=np.int64)
        out[:, 2] = -1
        for t in range(len(T)):
            best = -1
            for r in range(len(R)):            # ascending keypoint ids: ties keep the first
                if best < 0 or self._beats(int(D[t, r]), int(qr[r]), int(D[t, best]), int(qr[best])):
                    best = r
            if best >= 0:
                out[t] = (D[t, best], qr[best], rk[best], 0)
        return torch.as_tensor(out)

    def finish_local(self, parts_all, ref, tgt, n_ref_kp, n_tgt_kp, dim):
        """Exact combine of the gathered partials; float64 distances only for
        winners whose rows this rank holds (+inf otherwise), like the C ABI."""
        P = parts_all.numpy()
        R, T = ref["counts"].numpy().astype(float), tgt["counts"].numpy().astype(float)
        rk, tk, qt = ref["kp"].numpy(), tgt["kp"].numpy(), tgt["sqnorm"].numpy()
        res = []
        if len(R) == 0:
            return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0)
        for kp_t in np.unique(tk):
            rows = np.nonzero(tk == kp_t)[0]
            best = None                                   # (D, q_ref, kp_ref, q_tgt)
            for t in rows:
                for g in range(P.shape[0]):
                    D, q, k, _ = (int(x) for x in P[g, t])
                    if k < 0:
                        continue
                    if best is None:
                        best = (D, q, k, int(qt[t]))
                        continue
                    l, r = D * D * best[1] * best[3], best[0] ** 2 * q * int(qt[t])
                    if l > r or (l == r and k < best[2]):
                        best = (D, q, k, int(qt[t]))
            if best is None:
                continue
            rv = R[rk == best[2]]
            d = np.inf
            if len(rv):
                tv = T[rows]
                rv = rv / np.linalg.norm(rv, axis=1, keepdims=True)
                tv = tv / np.linalg.norm(tv, axis=1, keepdims=True)
                d = np.sqrt(((rv[:, None, :] - tv[None, :, :]) ** 2).sum(-1).min())
            res.append((best[2], int(kp_t), d))
        return (np.array([p[0] for p in res], np.int64), np.array([p[1] for p in res], np.int64),
                np.array([p[2] for p in res], np.float64))


BASE = dict(scale_mult=1.6, sigma_on_f=0.75)


def _sharded_worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2303_00319_b200 import RiftConfig, sharded, synth
        a, b, _ = synth.make_pair(160, seed=9, looks=None)
        cfg = RiftConfig(max_keypoints=300, **BASE)
        ms, info = sharded.match_pair_sharded(a, b, cfg, backend=NumpyBackend())
        out[rank] = (ms.pairs, info)
    finally:
        dist.destroy_process_group()


def test_sharded_matching_gloo_world2():
    sys.path.insert(0, ROOT)
    from oracle import rift2_oracle as O
    from paper_2303_00319_b200 import RiftConfig, sharded, synth
    world = 2
    port = _free_port()
    mgr = tmp.Manager()
    out = mgr.dict()
    tmp.spawn(_sharded_worker, args=(world, port, out), nprocs=world, join=True)
    p0, info0 = out[0]
    p1, info1 = out[1]
    assert p0 == p1                                   # every rank holds the same result
    assert info0["ref_slice"][1] == info1["ref_slice"][0]        # contiguous, complementary slices
    # image 1's rows stay on their rank: each rank held only its own slice
    assert info0["ref_descriptors_local"] + info1["ref_descriptors_local"] == info0["ref_descriptors"]
    assert 0 < info0["ref_descriptors_local"] < info0["ref_descriptors"]
    # the same backend unsharded, and the oracle's own matcher on the full sets
    a, b, _ = synth.make_pair(160, seed=9, looks=None)
    cfg = RiftConfig(max_keypoints=300, **BASE)
    single, _ = sharded.match_pair_sharded(a, b, cfg, backend=NumpyBackend())
    assert [(r, t) for r, t, _ in p0] == [(r, t) for r, t, _ in single.pairs]
    assert len(p0) > 10
    be = NumpyBackend()
    feats = [be.features(img, cfg) for img in (a, b)]
    d = [be.describe_slice(f, 0, f["n"], cfg) for f in feats]
    rc, tc = (x["counts"].numpy().astype(float) for x in d)
    pairs, _ = O.match_nn(rc / np.linalg.norm(rc, axis=1, keepdims=True), d[0]["kp"].numpy(),
                          tc / np.linalg.norm(tc, axis=1, keepdims=True), d[1]["kp"].numpy())
    assert {(int(r), int(t)) for r, t, _ in pairs} == {(r, t) for r, t, _ in p0}

"""Benchmark: image pairs/s of the RIFT2 pipeline at 1024^2 on B200.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one pass of the whole hot path (filter bank + PC/MIM, FAST +
merge, RIFT2 descriptors, tensor-core matching) over this rank's batch of
16 independent 1024^2 pairs (BASELINE.json configs[1]/[2]: seeds 0-15 on
rank 0; per-GPU share of the 128-pair batch for N = 8).  Pairs shard over
ranks with no collective ("weak" scaling); the only cross-rank traffic is
the barrier and the max-reduction of the device times.

Prints ONE JSON line on rank 0.  See DESIGN.md section "Measurement".
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "image pairs/sec at 1024² (4×6 log-Gabor, 5k kpts); % of HBM/TC roofline"
BASE_PARAMS = dict(scale_mult=1.6, sigma_on_f=0.75)
BYTES_PER_PX = 429          # algorithmic filter-bank bytes per pixel per image


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--pairs", type=int, default=16, help="pairs per GPU per step")
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--max-kp", type=int, default=5000, help="max keypoints per image (configs[3]: 20000)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def workload(args, n):
    return {"workload": f"{args.pairs} independent {args.size}x{args.size} pairs per GPU per step "
                        f"(BASELINE generator: blobs+band-limited noise, rotation+translation, inversion/gamma, "
                        f"4-look speckle; seeds rank*{args.pairs}+0..{args.pairs - 1}); 4x6 log-Gabor "
                        f"scale_mult 1.6 sigma_on_f 0.75, <={args.max_kp} FAST keypoints, RIFT2 216-D, NN matching",
            "pairs_per_gpu": args.pairs, "size": args.size, "global_pairs_per_step": args.pairs * n,
            "parallelism": f"dp{n} (pairs sharded, no collective)",
            "l2": "inputs + inter-pass planes (192 MB/image) far exceed the 126 MB L2"}


# ----------------------------------------------------------------- CPU side
def _oracle_pair(args):
    """One pair through the CPU oracle (test infrastructure; baseline only)."""
    seed, size = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import rift2_oracle as O
    from paper_2303_00319_b200 import synth
    a, b, _ = synth.make_pair(size, seed)
    p = O.Bank(**BASE_PARAMS)
    t0 = time.perf_counter()
    feats = []
    for img in (a, b):
        f = O.fields(img, p, workers=1)
        kp = O.detect_keypoints(f["moment_min"], f["moment_max"], 0.001, 5000, 96)
        c, k, v, _ = O.describe_rift2(f["mim"], kp)
        feats.append((c, k))
    (rc, rk), (tc, tk) = feats
    rv = rc / np.linalg.norm(rc, axis=1, keepdims=True)
    tv = tc / np.linalg.norm(tc, axis=1, keepdims=True)
    if len(rk) and len(tk):
        O.match_nn(rv, rk, tv, tk)
    return time.perf_counter() - t0


def cpu_sample(size, n_workers, seed0=0):
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(n_workers) as pool:
        per = pool.map(_oracle_pair, [(seed0 + i, size) for i in range(n_workers)])
    wall = time.perf_counter() - t0
    return n_workers / wall, wall, per


def cpu_workers():
    n = os.cpu_count() or 1
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        pass
    return max(1, min(n, 16))


UNITS = ("fields(ref)", "fields(tgt)", "features(ref)", "features(tgt)", "match")


def _unit_worker(conn, size, seed0, stride):
    """Persistent CPU worker for --impl reference: holds one pair's state and
    runs one pipeline unit per request (test infrastructure: the oracle)."""
    from oracle import rift2_oracle as O
    from paper_2303_00319_b200 import synth
    bank = O.Bank(**BASE_PARAMS)
    pair, st = 0, {}
    while True:
        msg = conn.recv()
        if msg is None:
            return
        if msg == "gen":
            st = {"img": synth.make_pair(size, seed0 + pair * stride)[:2]}
            conn.send(0.0)
            continue
        t0 = time.perf_counter()
        if msg in (0, 1):
            st[f"f{msg}"] = O.fields(st["img"][msg], bank, workers=1)
        elif msg in (2, 3):
            f = st[f"f{msg - 2}"]
            kp = O.detect_keypoints(f["moment_min"], f["moment_max"], 0.001, 5000, 96)
            c, k, _, _ = O.describe_rift2(f["mim"], kp)
            st[f"d{msg - 2}"] = (c / np.linalg.norm(c, axis=1, keepdims=True), k)
        else:
            (rv, rk), (tv, tk) = st["d0"], st["d1"]
            if len(rk) and len(tk):                 # tiny images can leave a side without descriptors
                O.match_nn(rv, rk, tv, tk)
            pair += 1
        conn.send(time.perf_counter() - t0)


class UnitPool:
    def __init__(self, n, size):
        for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "RIFT2_THREADS"):
            os.environ[k] = "1"
        ctx = mp.get_context("spawn")
        self.conns, self.procs = [], []
        for w in range(n):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_unit_worker, args=(b, size, w, n), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        self.unit = 0

    def step(self):
        """One step = the next unit on every worker; returns the wall time."""
        if self.unit == 0:
            for c in self.conns:                  # generation is outside the timed step
                c.send("gen")
            for c in self.conns:
                c.recv()
        t0 = time.perf_counter()
        for c in self.conns:
            c.send(self.unit)
        for c in self.conns:
            c.recv()
        wall = time.perf_counter() - t0
        u, self.unit = self.unit, (self.unit + 1) % len(UNITS)
        return u, wall

    def close(self):
        for c in self.conns:
            c.send(None)
        for p in self.procs:
            p.join(timeout=30)


def run_reference(args, rank, world):
    """The reference's CPU path (the oracle port, pinned to the reference by
    golden vectors) on all host cores.  A step is one fifth of a pair on
    every worker (UNITS, round robin) so the run stays within minutes;
    pairs/s = workers / sum over units of the mean unit wall time."""
    if rank != 0:
        return
    n = cpu_workers()
    pool = UnitPool(n, args.size)
    try:
        for _ in range(args.warmup):
            pool.step()
        steps = max(args.steps, len(UNITS))
        by_unit = {u: [] for u in range(len(UNITS))}
        walls = []
        for _ in range(steps):
            u, w = pool.step()
            by_unit[u].append(w)
            walls.append(w)
    finally:
        pool.close()
    per_pair = sum(statistics.mean(v) for v in by_unit.values())
    value = n / per_pair
    sample = (f"{n} worker processes x 1 thread; each step runs one of {len(UNITS)} units of a {args.size}^2 "
              f"pair ({', '.join(UNITS)}) on every worker; {steps} steps; pairs/s = workers / sum of mean unit "
              f"walls ({per_pair:.1f} s per pair per worker)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
            "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload(args, world),
            "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": n, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU side
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.index)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def tensor_peak():
    """Dense fp16/bf16 tensor peak (the matching GEMM runs kind::f16)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["bf16_tflops"]), "measured (MEASURED_PEAKS.json bf16_tflops, burst)"
    except (OSError, KeyError, ValueError):
        return 2250.0, "nominal dense bf16 (fallback)"


def rank_seed0(rank, pairs):
    """First generator seed of this rank's pairs: ranks own disjoint, contiguous
    seed ranges (configs[2]: the 128-pair batch split over the GPUs)."""
    return rank * pairs


def max_over_ranks(values, world, device):
    """Element-wise max of per-rank timings (the slowest rank defines a step)."""
    import torch
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def traffic():
    """Filter-bank DRAM bytes per pass from the newest committed ncu launch
    list (profiles/rNN_launches.json, written by tools/profile_summary.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_launches.json")))
    if not files:
        return None, None
    try:
        with open(files[-1]) as fh:
            p = json.load(fh)
        return float(p["filter_bank"]["dram_bytes_per_pass"]), os.path.relpath(files[-1], ROOT)
    except (OSError, KeyError, ValueError):
        return None, None


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2303_00319_b200 import BatchPipeline, RiftConfig, synth

    torch.cuda.set_device(local_rank)
    cfg = RiftConfig(max_keypoints=args.max_kp, **BASE_PARAMS)
    imgs, _ = synth.make_batch(args.pairs, args.size, seed0=rank_seed0(rank, args.pairs))
    pipe = BatchPipeline(args.pairs, args.size, args.size, cfg)
    pipe.load(imgs)
    pipe.capture()
    pipe.capture_pipelined()
    pipe._alt.copy_(pipe.images)              # both input buffers hold this rank's batch
    # warm-up (also primes the pipeline: the first step's features stage has no batch yet)
    for i in range(max(args.warmup, 1)):
        pipe.pipelined_step(i)
    torch.cuda.synchronize()

    K = args.steps
    clk = Clocks(local_rank)
    clk.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # headline: K pipelined steps; each completes one batch (filter bank of
    # batch i on one stream next to detect / describe / match of batch i-1)
    parity = max(args.warmup, 1)
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_start.record()
    for i in range(K):
        pipe.pipelined_step(parity + i)
    e_end.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = e_start.elapsed_time(e_end)
    # roofline: the filter bank alone on its stream, K launches of its graph
    # timed with CUDA events
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for i in range(K):
        ev[i][0].record()
        pipe.replay_fields()
        ev[i][1].record()
    torch.cuda.synchronize()
    fields_ms = sum(a.elapsed_time(b) for a, b in ev) / K
    # matching: the match stage (tensor-core GEMM + exact combine + sort) on
    # this step's descriptor arrays, K launches timed with CUDA events
    from paper_2303_00319_b200 import engine
    engine.match(pipe.d, pipe.dim, pipe.rb, pipe.tb, pipe.K, ws_key="bench_match")   # allocates its workspace
    torch.cuda.synchronize()
    em = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for i in range(K):
        em[i][0].record()
        engine.match(pipe.d, pipe.dim, pipe.rb, pipe.tb, pipe.K, ws_key="bench_match")
        em[i][1].record()
    torch.cuda.synchronize()
    match_ms = sum(a.elapsed_time(b) for a, b in em) / K
    dcnt = pipe.d["count"].cpu().numpy().astype(np.int64)
    match_flops = float(sum(2 * dcnt[2 * q] * dcnt[2 * q + 1] * pipe.dim for q in range(args.pairs)))

    # e2e: public API with host buffers -- every step uploads its images from
    # pinned host memory (copy stream, double-buffered against the previous
    # step's compute) and reads the match arrays back
    host_in = torch.from_numpy(imgs).pin_memory()
    out_keys = ("ref", "tgt", "dist", "count")
    host_out = {k: torch.empty(pipe.m[k].shape, dtype=pipe.m[k].dtype).pin_memory() for k in out_keys}
    h2d = host_in.numel() * 4
    d2h = sum(pipe.m[k].numel() * pipe.m[k].element_size() for k in out_keys)
    pipe.run_from_host_pipelined(host_in, 2, host_out)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    KE = max(5, K)
    e0.record()
    pipe.run_from_host_pipelined(host_in, KE, host_out)   # KE completed batches (+ a priming filter bank)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    clocks = clk.stop()

    total_ms, e2e_ms, fields_ms = max_over_ranks([total_ms, e2e_ms, fields_ms], world, "cuda")
    if rank != 0:
        return
    pairs = args.pairs * world * K
    value = pairs / (total_ms / 1e3)
    e2e = args.pairs * world * KE / (e2e_ms / 1e3)
    peak, peak_src = peaks()
    tpk, tpk_src = tensor_peak()
    bytes_launch = BYTES_PER_PX * args.size * args.size * 2 * args.pairs
    achieved = bytes_launch / (fields_ms / 1e3) / 1e9
    tr, tr_src = traffic()
    if tr is not None and (args.pairs, args.size) != (16, 1024):
        tr = tr * (args.pairs * args.size * args.size) / (16 * 1024 * 1024)   # profile is per 16 pairs of 1024^2
    counts = pipe.m["count"].cpu().numpy()
    line = {"metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": workload(args, world),
            "e2e": {"value": e2e, "unit": "pairs/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": KE},
            "gpu_launches": pipe.KERNELS_PER_STEP * K,
            "roofline": {"bound": "hbm", "kernel": "filter bank (rows_fwd+cols+rows_amp0+median+rows_pc)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": tr, "traffic_source": tr_src, "bytes_per_launch": bytes_launch, "launch_ms": fields_ms,
                         "share_of_step": fields_ms / (total_ms / K), "peak_source": peak_src,
                         "note": "filter bank timed alone; in the pipelined step it overlaps the previous batch's features"},
            "roofline_match": {"bound": "tensor", "kernel": "match stage (k_match_gemm tcgen05 f16 + combine + sort)",
                               "achieved": match_flops / (match_ms / 1e3) / 1e12, "peak": tpk, "unit": "TFLOP/s",
                               "frac": match_flops / (match_ms / 1e3) / 1e12 / tpk,
                               "flops_per_launch": match_flops, "launch_ms": match_ms, "peak_source": tpk_src},
            "clocks": clocks,
            "matches_per_pair": float(np.mean(counts))}
    if world == 1 and not args.no_cpu_baseline:
        n = cpu_workers()
        rate, wall, per = cpu_sample(args.size, n)
        line["cpu_baseline"] = {"value": rate, "unit": "pairs/s", "cores": n, "kind": "port",
                                "sample": f"{n} pairs ({n} processes x 1 pair, {args.size}^2, oracle pipeline, "
                                          f"{wall:.1f} s wall, {statistics.mean(per):.1f} s/pair/core)"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

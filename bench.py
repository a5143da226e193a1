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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def workload(args, n):
    return {"workload": f"{args.pairs} independent {args.size}x{args.size} pairs per GPU per step "
                        f"(BASELINE generator: blobs+band-limited noise, rotation+translation, inversion/gamma, "
                        f"4-look speckle; seeds rank*{args.pairs}+0..{args.pairs - 1}); 4x6 log-Gabor "
                        f"scale_mult 1.6 sigma_on_f 0.75, <=5000 FAST keypoints, RIFT2 216-D, NN matching",
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


def run_reference(args, rank, world):
    if rank != 0:
        return
    n = cpu_workers()
    for _ in range(min(args.warmup, 1)):
        cpu_sample(args.size, n)
    rates, walls = [], []
    for s in range(args.steps):
        r, w, _ = cpu_sample(args.size, n, seed0=s * n)
        rates.append(r)
        walls.append(w)
    value = sum(n for _ in rates) / sum(walls)
    sample = f"{n} pairs per step ({n} worker processes x 1 pair, {args.size}^2, full oracle pipeline)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": min(args.warmup, 1), "ms_per_step": 1e3 * statistics.mean(walls),
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


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2303_00319_b200 import BatchPipeline, RiftConfig, synth

    torch.cuda.set_device(local_rank)
    cfg = RiftConfig(**BASE_PARAMS)
    imgs, _ = synth.make_batch(args.pairs, args.size, seed0=rank * args.pairs)
    pipe = BatchPipeline(args.pairs, args.size, args.size, cfg)
    pipe.load(imgs)
    pipe.capture()
    for _ in range(max(args.warmup, 0)):
        pipe.step()
    torch.cuda.synchronize()

    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    clk = Clocks(local_rank)
    clk.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(K):
        ev[i][0].record()
        pipe.replay_fields()
        ev[i][1].record()
        pipe.replay_features()
        ev[i][2].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = ev[0][0].elapsed_time(ev[K - 1][2])
    fields_ms = sum(ev[i][0].elapsed_time(ev[i][1]) for i in range(K)) / K

    # e2e: public API with host buffers (pinned H2D of the step's images, D2H of the matches)
    host_in = torch.from_numpy(imgs).pin_memory()
    out_keys = ("ref", "tgt", "dist", "count")
    host_out = {k: torch.empty(pipe.m[k].shape, dtype=pipe.m[k].dtype).pin_memory() for k in out_keys}
    h2d = host_in.numel() * 4
    d2h = sum(pipe.m[k].numel() * pipe.m[k].element_size() for k in out_keys)
    for _ in range(2):
        pipe.images.copy_(host_in, non_blocking=True)
        pipe.step()
        for k in out_keys:
            host_out[k].copy_(pipe.m[k], non_blocking=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    KE = max(3, K // 3)
    e0.record()
    for _ in range(KE):
        pipe.images.copy_(host_in, non_blocking=True)
        pipe.step()
        for k in out_keys:
            host_out[k].copy_(pipe.m[k], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    clocks = clk.stop()

    t = torch.tensor([total_ms, e2e_ms, fields_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms, fields_ms = t.tolist()
    if rank != 0:
        return
    pairs = args.pairs * world * K
    value = pairs / (total_ms / 1e3)
    e2e = args.pairs * world * KE / (e2e_ms / 1e3)
    peak, peak_src = peaks()
    bytes_launch = BYTES_PER_PX * args.size * args.size * 2 * args.pairs
    achieved = bytes_launch / (fields_ms / 1e3) / 1e9
    counts = pipe.m["count"].cpu().numpy()
    line = {"metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": workload(args, world),
            "e2e": {"value": e2e, "unit": "pairs/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": KE},
            "gpu_launches": pipe.KERNELS_PER_STEP * K,
            "roofline": {"bound": "hbm", "kernel": "filter bank (rows_fwd+cols+rows_amp0+median+rows_pc)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "bytes_per_launch": bytes_launch, "launch_ms": fields_ms,
                         "share_of_step": fields_ms / (total_ms / K), "peak_source": peak_src},
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

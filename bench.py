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
    ap.add_argument("--no-other-configs", action="store_true", help="skip the configs[3] / [4] side measurements")
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
# The CPU baseline is the UNMODIFIED reference package (pure Python/numpy/
# scipy), installed into baseline/_ref by oracle/build_ref.sh and run through
# its own public API (rift2.compute_fields / detect_keypoints / describe /
# match_nn -- the stages rift2.match_pair chains, ref pipeline.py:67-99).
# Only if that install is missing does the oracle port stand in ("port").
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "rift2", "__init__.py"))


def host_info() -> dict:
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = os.cpu_count() or 1
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "affinity_cpus": aff}


def cpu_workers():
    """One single-threaded worker per usable host core: the
    reference's FFTs and BLAS are pinned to one thread per process."""
    return max(1, host_info()["affinity_cpus"])


def _single_thread_env():
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "RIFT2_THREADS"):
        os.environ[k] = "1"


class _Stages:
    """The path's stages on the CPU: the reference's own functions, or the
    oracle port when the reference is not installed."""

    def __init__(self, max_kp):
        _single_thread_env()
        self.kind = "reference" if reference_available() else "port"
        if self.kind == "reference":
            if REF_DIR not in sys.path:
                sys.path.insert(0, REF_DIR)
            import rift2
            self.r = rift2
            self.cfg = rift2.RiftConfig(max_keypoints=max_kp, threads=1, **BASE_PARAMS)
        else:
            from oracle import rift2_oracle as O
            self.O = O
            self.bank = O.Bank(**BASE_PARAMS)
            self.max_kp = max_kp

    def fields(self, img):
        if self.kind == "reference":
            return self.r.compute_fields(img, self.cfg)
        return self.O.fields(img, self.bank, workers=1)

    def features(self, f, side):
        if self.kind == "reference":
            pc, mim = f
            c = self.cfg
            kps = self.r.detect_keypoints(pc, c.fast_threshold, c.max_keypoints, c.patch_size)
            return self.r.pipeline.describe(mim, kps, c, side=side).descriptors
        kp = self.O.detect_keypoints(f["moment_min"], f["moment_max"], 0.001, self.max_kp, 96)
        c, k, _, _ = self.O.describe_rift2(f["mim"], kp)
        return (c / np.linalg.norm(c, axis=1, keepdims=True), k)

    def match(self, d_ref, d_tgt):
        if self.kind == "reference":
            if d_ref and d_tgt:
                return self.r.match_nn(d_ref, d_tgt, mode=self.cfg.mode)
            return None
        (rv, rk), (tv, tk) = d_ref, d_tgt
        if len(rk) and len(tk):                 # tiny images can leave a side without descriptors
            return self.O.match_nn(rv, rk, tv, tk)
        return None


def _cpu_pair(args):
    """One whole pair through the CPU stages (wall time of the pipeline, not
    of the generator)."""
    seed, size, max_kp = args
    st = _Stages(max_kp)
    from paper_2303_00319_b200 import synth
    a, b, _ = synth.make_pair(size, seed)
    t0 = time.perf_counter()
    fa, fb = st.fields(a), st.fields(b)
    st.match(st.features(fa, "reference"), st.features(fb, "target"))
    return time.perf_counter() - t0, st.kind


def cpu_sample(size, n_workers, max_kp, seed0=0):
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(n_workers) as pool:
        res = pool.map(_cpu_pair, [(seed0 + i, size, max_kp) for i in range(n_workers)])
    wall = time.perf_counter() - t0
    return n_workers / wall, wall, [r[0] for r in res], res[0][1]


UNITS = ("fields(ref)", "fields(tgt)", "features(ref)", "features(tgt)", "match")


def _unit_worker(conn, size, seed0, stride, max_kp):
    """Persistent CPU worker for --impl reference: holds one pair's state and
    runs one stage of it per request."""
    st = _Stages(max_kp)
    from paper_2303_00319_b200 import synth
    pair, state = 0, {}
    conn.send(st.kind)
    while True:
        msg = conn.recv()
        if msg is None:
            return
        if msg == "gen":
            state = {"img": synth.make_pair(size, seed0 + pair * stride)[:2]}
            conn.send(0.0)
            continue
        t0 = time.perf_counter()
        if msg in (0, 1):
            state[f"f{msg}"] = st.fields(state["img"][msg])
        elif msg in (2, 3):
            state[f"d{msg - 2}"] = st.features(state[f"f{msg - 2}"], "reference" if msg == 2 else "target")
        else:
            st.match(state["d0"], state["d1"])
            pair += 1
        conn.send(time.perf_counter() - t0)


class UnitPool:
    def __init__(self, n, size, max_kp):
        ctx = mp.get_context("spawn")
        self.conns, self.procs = [], []
        for w in range(n):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_unit_worker, args=(b, size, w, n, max_kp), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        self.kind = [c.recv() for c in self.conns][0]
        self.unit = 0

    def step(self):
        """One step = the next stage on every worker; returns the wall time."""
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
    """The reference's CPU implementation on all host cores: one
    single-threaded worker per core, each stepping through its own pairs one
    stage per step (UNITS, round robin) so the run stays within minutes;
    pairs/s = workers / sum over stages of the mean stage wall time."""
    if rank != 0:
        return
    n = cpu_workers()
    pool = UnitPool(n, args.size, args.max_kp)
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
    per_pair = sum(statistics.mean(v) for v in by_unit.values() if v)
    value = n / per_pair
    what = ("the unmodified reference (baseline/_ref rift2: compute_fields, detect_keypoints, pipeline.describe, "
            "match_nn)" if pool.kind == "reference" else "the oracle port (reference not installed)")
    sample = (f"{n} worker processes x 1 thread running {what}; each step runs one of {len(UNITS)} stages of a "
              f"{args.size}^2 pair ({', '.join(UNITS)}) on every worker; {steps} steps; pairs/s = workers / sum "
              f"of mean stage walls ({per_pair:.1f} s per pair per worker)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
            "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload(args, world),
            "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": n, "kind": pool.kind, "sample": sample,
                             "host": host_info()},
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


def tensor_peak(sustained: bool = False):
    """Dense fp16/bf16 tensor peak (the matching GEMM runs kind::f16): the
    burst figure for a launch timed alone, the sustained one for back-to-back
    launches."""
    key = "bf16_tflops_sustained" if sustained else "bf16_tflops"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p[key]), f"measured (MEASURED_PEAKS.json {key})"
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


def graph_ms(fn, reps: int, gap_s: float = 0.0) -> float:
    """Device time per call of `fn` (a sequence of our launches), captured
    once in a CUDA graph and replayed `reps` times between two CUDA events:
    the host-side launch preparation (tensor-map encoding, ctypes) stays out
    of the timed interval, as it does in the pipeline's own graphs.  With
    gap_s > 0 every replay is timed on its own after an idle gap (a kernel
    timed alone, at burst clocks; back to back, the tensor-core GEMM runs at
    the sustained, power-capped clock); returns the median."""
    import torch
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    if gap_s > 0:
        ts = []
        for _ in range(reps):
            time.sleep(gap_s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def ring_vs_rift2(pipe, reps: int = 5):
    """CUDA-event time of describe + match per mode on the pipeline's current
    keypoints (the reference benchmark's protocol: shared detection, ref
    evalbench.py:282-325), plus descriptor counts and distance evaluations."""
    import torch
    from paper_2303_00319_b200 import engine
    c = pipe.cfg
    out = {}
    for mode, desc_mode, per in (("rift2", "rift2", 2), ("ring", "ring_pipeline", c.n_orient)):
        def run():
            d = engine.describe(pipe.f["mim"], pipe.k["x"], pipe.k["y"], pipe.k["count"], c.n_orient, c.patch_size,
                                c.grid, c.dominant_ratio, c.rotate_patch, desc_mode, capacity=per * pipe.K,
                                ws_key=f"rvr_{mode}_d")
            m = engine.match(d, pipe.dim, pipe.rb, pipe.tb, pipe.K, ws_key=f"rvr_{mode}_m")
            return d, m
        d, m = run()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a, b in ev:
            a.record()
            run()
            b.record()
        torch.cuda.synchronize()
        cnt = d["count"].cpu().numpy().astype(np.int64)
        out[mode] = {"ms": statistics.median(a.elapsed_time(b) for a, b in ev),
                     "ref_descriptors": int(cnt[0::2].sum()), "tgt_descriptors": int(cnt[1::2].sum()),
                     "distance_evals": int((cnt[0::2] * cnt[1::2]).sum())}
    kps = int(pipe.k["count"].cpu().numpy()[0::2].sum())
    return {"what": "describe + match of the whole batch per mode on shared keypoints (GPU, CUDA events)",
            "rift2": out["rift2"], "ring": out["ring"], "ref_keypoints": kps,
            "speedup": out["ring"]["ms"] / out["rift2"]["ms"],
            "descriptor_reduction": out["ring"]["ref_descriptors"] / max(out["rift2"]["ref_descriptors"], 1),
            "distance_eval_reduction": out["ring"]["distance_evals"] / max(out["rift2"]["distance_evals"], 1)}


def other_configs(reps: int = 10) -> dict:
    """BASELINE.json configs[3] and [4] on this GPU, pipelined steps with
    inputs resident, CUDA events (the headline line is configs[1]/[2]):
    configs[3] one 4096^2 pair (blob sigma x4, <= 20,000 keypoints);
    configs[4] 64 pairs of 512^2 per step from the rotation sweep (theta in
    15-degree steps, scale jitter 0.1, speckle looks 1 / 4 / 16)."""
    import torch
    from paper_2303_00319_b200 import BatchPipeline, RiftConfig, synth
    out = {}
    for name, size, n, kp in (("configs[3]", 4096, 1, 20000), ("configs[4]", 512, 64, 5000)):
        if name == "configs[3]":
            imgs, _ = synth.make_batch(1, 4096, seed0=0)
        else:
            imgs = np.empty((2 * n, size, size), np.float32)
            for i in range(n):
                th = 15 * (i % 24)
                a, b, _ = synth.make_pair(size, seed=5000 + i, theta_deg=float(th), scale_jitter=0.1,
                                          looks=(1, 4, 16)[(i // 24 + i) % 3])
                imgs[2 * i], imgs[2 * i + 1] = a, b
        pipe = BatchPipeline(n, size, size, RiftConfig(max_keypoints=kp, **BASE_PARAMS))
        pipe.load(imgs)
        pipe.capture_pipelined()
        pipe._alt.copy_(pipe.images)
        for i in range(3):
            pipe.pipelined_step(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(reps):
            pipe.pipelined_step(i + 1)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(reps):
            pipe.replay_fields()
        f1.record()
        torch.cuda.synchronize()
        fms = f0.elapsed_time(f1) / reps
        byts = BYTES_PER_PX * size * size * 2 * n
        out[name] = {"pairs_per_step": n, "size": size, "max_keypoints": kp, "ms_per_step": ms,
                     "pairs_per_s": n / (ms / 1e3), "filter_bank_ms": fms,
                     "filter_bank_frac_hbm": byts / (fms / 1e3) / 1e9 / peaks()[0],
                     "matches_pair0": int(pipe.m["count"][0])}
        del pipe
        torch.cuda.empty_cache()
    return out


def dataclass_api_latency(cfg, size, seeds):
    """Wall time of paper_2303_00319_b200.match_pair (the reference's
    dataclass API: host float64 images in, Keypoint / Descriptor / MatchSet
    objects out) per pair; the first call warms the workspaces."""
    from paper_2303_00319_b200 import match_pair, synth
    pairs = [synth.make_pair(size, s)[:2] for s in seeds]
    match_pair(*pairs[0], cfg)
    walls = []
    for a, b in pairs:
        t0 = time.perf_counter()
        res = match_pair(a, b, cfg)
        walls.append(time.perf_counter() - t0)
        assert len(res.matches.pairs) > 0
    walls.sort()
    return {"what": f"match_pair on one {size}^2 pair (dataclass API incl. host<->device copies and "
                    f"Keypoint/Descriptor/MatchSet construction), seeds {seeds[0]}-{seeds[-1]}",
            "ms_median": 1e3 * statistics.median(walls), "ms_min": 1e3 * walls[0], "ms_max": 1e3 * walls[-1],
            "pairs_per_s": len(walls) / sum(walls)}


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
    match_ms = graph_ms(lambda: engine.match(pipe.d, pipe.dim, pipe.rb, pipe.tb, pipe.K, ws_key="bench_match",
                                             out=pipe.m), K)
    # the tensor-core GEMM kernel alone (rift2_match_partial launches exactly
    # k_match_gemm, with the same single column split the batch uses)
    parts = engine.match_partial(pipe.d, pipe.dim, pipe.rb, pipe.tb)
    torch.cuda.synchronize()
    gemm_ms = graph_ms(lambda: engine.match_partial(pipe.d, pipe.dim, pipe.rb, pipe.tb, out=parts), K)
    gemm_burst_ms = graph_ms(lambda: engine.match_partial(pipe.d, pipe.dim, pipe.rb, pipe.tb, out=parts), K,
                             gap_s=0.02)
    dcnt = pipe.d["count"].cpu().numpy().astype(np.int64)
    match_flops = float(sum(2 * dcnt[2 * q] * dcnt[2 * q + 1] * pipe.dim for q in range(args.pairs)))

    # e2e: public API with host buffers -- every step uploads its images from
    # pinned host memory (copy stream, double-buffered against the previous
    # step's compute) and reads back the match arrays and the keypoint
    # coordinates they index (a usable result: matched point pairs)
    host_in = torch.from_numpy(imgs).pin_memory()
    out_keys = ("ref", "tgt", "dist", "count", "kp_x", "kp_y", "kp_count")
    host_out = {k: torch.empty(shp, dtype=dt).pin_memory() for k, (shp, dt) in pipe.result_shapes(out_keys).items()}
    h2d = host_in.numel() * 4
    d2h = sum(t.numel() * t.element_size() for t in host_out.values())
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
    # the matched coordinates of the last batch, resolved on the host from the copied arrays
    n0 = int(host_out["count"][0])
    r0, t0_ = host_out["ref"][0, :n0].long(), host_out["tgt"][0, :n0].long()
    matched_xy = torch.stack([host_out["kp_x"][0][r0], host_out["kp_y"][0][r0],
                              host_out["kp_x"][1][t0_], host_out["kp_y"][1][t0_]], 1)

    # ring vs RIFT2 (ref evalbench.py:282-325, acceptance criteria 5-6): the
    # description + matching stage of both modes on this batch's keypoints
    ring = ring_vs_rift2(pipe) if world == 1 else None

    # dataclass drop-in API (ref pipeline.py:82-99): one pair per call,
    # north_star's configs[1] single-pair latency over seeds 0-15 on 1 GPU
    api = others = None
    if world == 1 and args.size <= 1024:
        api = dataclass_api_latency(cfg, args.size, seeds=range(16))
        if not args.no_other_configs:
            others = other_configs()

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
            "roofline_gemm": {"bound": "tensor", "kernel": "k_match_gemm (tcgen05 kind::f16, TMEM accumulators, "
                                                            "TMA operands, fused exact argmax epilogue)",
                              "achieved": match_flops / (gemm_burst_ms / 1e3) / 1e12, "peak": tpk, "unit": "TFLOP/s",
                              "frac": match_flops / (gemm_burst_ms / 1e3) / 1e12 / tpk,
                              "flops_per_launch": match_flops, "launch_ms": gemm_burst_ms, "peak_source": tpk_src,
                              "sustained": {"launch_ms": gemm_ms,
                                            "achieved": match_flops / (gemm_ms / 1e3) / 1e12,
                                            "peak": tensor_peak(sustained=True)[0],
                                            "frac": match_flops / (gemm_ms / 1e3) / 1e12 / tensor_peak(sustained=True)[0],
                                            "note": "K launches back to back: power-capped clocks, against the "
                                                    "sustained matmul peak"},
                              "note": "one launch after an idle gap (burst clocks), median of K; algorithmic "
                                      "2*N_ref*N_tgt*216 flops, the kernel multiplies K=224 (zero padded)"},
            "clocks": clocks,
            "single_pair_api": api,
            "other_configs": others,
            "ring_vs_rift2": ring,
            "e2e_matched_points_pair0": int(matched_xy.shape[0]),
            "matches_per_pair": float(np.mean(counts))}
    if world == 1 and not args.no_cpu_baseline:
        n = cpu_workers()
        rate, wall, per, kind = cpu_sample(args.size, n, args.max_kp)
        what = "rift2.compute_fields/detect_keypoints/describe/match_nn of baseline/_ref" if kind == "reference" \
            else "oracle port"
        line["cpu_baseline"] = {"value": rate, "unit": "pairs/s", "cores": n, "kind": kind, "host": host_info(),
                                "sample": f"{n} pairs ({n} single-threaded processes x 1 pair, {args.size}^2, "
                                          f"{what}, {wall:.1f} s wall, {statistics.mean(per):.1f} s/pair/core)"}
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

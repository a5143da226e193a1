"""Device-level stage calls: torch tensors in, torch tensors out.

PyTorch is only the carrier here (device memory, streams); every stage is
one call into the C ABI (include/rift2_b200.h), enqueued on the current
torch stream.  Workspaces are cached per (device, stage) and grown on
demand, so steady-state calls allocate nothing.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _lib
from .errors import ParameterError

DESC_STRIDE = 224      # 216-D descriptors padded to the tensor-core K tile


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


class _Workspaces:
    """Scratch buffers per (device, key), grown on demand.  A grown buffer's
    predecessor is retired, not freed: a CUDA graph captured earlier may
    still hold its address, and replaying it must not touch memory the
    caching allocator has handed to someone else.  Callers that run
    concurrently (e.g. two BatchPipelines on different streams) use distinct
    keys, so they never share scratch."""

    def __init__(self):
        self._bufs = {}
        self._retired = []

    def get(self, key: str, nbytes: int) -> torch.Tensor:
        dev = torch.cuda.current_device()
        buf = self._bufs.get((dev, key))
        if buf is None or buf.numel() < nbytes:
            if buf is not None:
                self._retired.append(buf)
            buf = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=f"cuda:{dev}")
            self._bufs[(dev, key)] = buf
        return buf


WORKSPACES = _Workspaces()


def bank_c(bank) -> _lib.BankParamsC:
    return _lib.BankParamsC(
        int(bank.n_scales), int(bank.n_orient), float(bank.min_wavelength), float(bank.scale_mult),
        float(bank.sigma_on_f), float(bank.orientation_spread or 0.0), float(bank.noise_k),
        float(bank.spread_cutoff), float(bank.spread_gain))


def fields(images: torch.Tensor, bank, extras: bool = False, ws_key: str = "fields", out=None):
    """images (B, H, W) float32 CUDA -> dict(mmax, mmin, mim[, a_o, pc, amax]);
    an `out` dict may also carry "range" ((B, 2, 2) int64: the moment maps'
    per-image extrema keys for detect())."""
    lib = _lib.load(require_gpu=True)
    if images.dim() != 3 or images.dtype != torch.float32 or not images.is_cuda:
        raise ParameterError("images must be a (B, H, W) float32 CUDA tensor")
    images = images.contiguous()
    B, H, W = images.shape
    p = bank_c(bank)
    nbytes = ctypes.c_size_t()
    _lib.check(lib.rift2_fields_workspace_size(B, H, W, ctypes.byref(p), ctypes.byref(nbytes)), "fields")
    ws = WORKSPACES.get(ws_key, nbytes.value)
    dev = images.device
    if out is None:
        out = dict(mmax=torch.empty((B, H, W), dtype=torch.float32, device=dev),
                   mmin=torch.empty((B, H, W), dtype=torch.float32, device=dev),
                   mim=torch.empty((B, H, W), dtype=torch.uint8, device=dev))
        if extras:
            O = int(bank.n_orient)
            out["a_o"] = torch.empty((B, O, H, W), dtype=torch.float32, device=dev)
            out["pc"] = torch.empty((B, O, H, W), dtype=torch.float32, device=dev)
            out["amax"] = torch.empty((B, H, W), dtype=torch.float32, device=dev)
    rc = lib.rift2_fields(_ptr(images), B, H, W, ctypes.byref(p), _ptr(out["mmax"]), _ptr(out["mmin"]),
                          _ptr(out["mim"]), _ptr(out.get("a_o")), _ptr(out.get("pc")), _ptr(out.get("amax")),
                          _ptr(out.get("range")), _ptr(ws), ws.numel(), _stream())
    _lib.check(rc, "rift2_fields")
    return out


def detect(mins: torch.Tensor, maxs: torch.Tensor | None, threshold: float, max_points: int, margin: int,
           single_map: bool = False, ws_key: str = "detect", out=None, moment_range: torch.Tensor | None = None):
    """mins / maxs (B, H, W) moment_min / moment_max (maxs unused with
    single_map), float32 or float64 CUDA -> dict(x, y, response, kind, count).
    moment_range: the (B, 2, 2) int64 extrema keys fields() wrote (its
    "range" output), so the maps are not re-read for the normalisation."""
    lib = _lib.load(require_gpu=True)
    mins = mins.contiguous()
    maxs = mins if (single_map or maxs is None) else maxs.contiguous()
    if maxs.dtype != mins.dtype or maxs.shape != mins.shape:
        raise ParameterError("moment maps differ in shape or dtype")
    B, H, W = mins.shape
    maps = mins
    K = int(max_points)
    nbytes = ctypes.c_size_t()
    _lib.check(lib.rift2_detect_workspace_size(B, H, W, K, ctypes.byref(nbytes)), "detect")
    ws = WORKSPACES.get(ws_key, nbytes.value)
    dev = maps.device
    if out is None:
        kk = max(K, 1)
        out = dict(x=torch.empty((B, kk), dtype=torch.int32, device=dev),
                   y=torch.empty((B, kk), dtype=torch.int32, device=dev),
                   response=torch.empty((B, kk), dtype=torch.float64, device=dev),
                   kind=torch.empty((B, kk), dtype=torch.uint8, device=dev),
                   count=torch.empty((B,), dtype=torch.int32, device=dev))
    fn = lib.rift2_detect_f64 if maps.dtype == torch.float64 else lib.rift2_detect_f32
    if maps.dtype not in (torch.float32, torch.float64):
        raise ParameterError("maps must be float32 or float64")
    rc = fn(_ptr(mins), _ptr(maxs), B, H, W, float(threshold), K, int(margin), 1 if single_map else 0,
            _ptr(out["x"]), _ptr(out["y"]), _ptr(out["response"]), _ptr(out["kind"]), _ptr(out["count"]),
            _ptr(moment_range), _ptr(ws), ws.numel(), _stream())
    _lib.check(rc, "rift2_detect")
    return out


MODE_CODE = {"plain": 0, "ring": 1, "rift2": 2, "ring_pipeline": 3}


def describe(mim: torch.Tensor, kp_x: torch.Tensor, kp_y: torch.Tensor, kp_count: torch.Tensor,
             n_orient: int, patch: int = 96, grid: int = 6, ratio: float = 0.8, rotate: bool = True,
             mode: str = "rift2", capacity: int | None = None, ws_key: str = "describe", out=None):
    """mim (B, H, W) uint8 CUDA, keypoints (B, S) int32 (or float64: any
    coordinates, rift2_describe_f64) -> dict(counts (B, cap, 224) f16,
    sqnorm, kp, variant, count, skipped)."""
    lib = _lib.load(require_gpu=True)
    B, H, W = mim.shape
    S = kp_x.shape[1]
    per = {"plain": 1, "ring": n_orient, "rift2": 2, "ring_pipeline": n_orient}[mode]
    cap = capacity if capacity is not None else max(S * per, 1)
    dim = grid * grid * n_orient
    stride = DESC_STRIDE if dim <= DESC_STRIDE else int(math.ceil(dim / 32) * 32)
    nbytes = ctypes.c_size_t()
    _lib.check(lib.rift2_describe_workspace_size_hw(B, H, W, S, grid, n_orient, ctypes.byref(nbytes)), "describe")
    ws = WORKSPACES.get(ws_key, nbytes.value)
    dev = mim.device
    if out is None:
        out = dict(counts=torch.zeros((B, cap, stride), dtype=torch.float16, device=dev),
                   sqnorm=torch.zeros((B, cap), dtype=torch.int32, device=dev),
                   kp=torch.zeros((B, cap), dtype=torch.int32, device=dev),
                   variant=torch.zeros((B, cap), dtype=torch.uint8, device=dev),
                   count=torch.empty((B,), dtype=torch.int32, device=dev),
                   skipped=torch.empty((B,), dtype=torch.int32, device=dev))
    fn = lib.rift2_describe_f64 if kp_x.dtype == torch.float64 else lib.rift2_describe
    rc = fn(_ptr(mim.contiguous()), B, H, W, int(n_orient), _ptr(kp_x), _ptr(kp_y),
                            _ptr(kp_count), S, int(patch), int(grid), float(ratio), 1 if rotate else 0,
                            MODE_CODE[mode], _ptr(out["counts"]), out["counts"].shape[2], out["counts"].shape[1],
                            _ptr(out["sqnorm"]), _ptr(out["kp"]), _ptr(out["variant"]), _ptr(out["count"]),
                            _ptr(out["skipped"]), _ptr(ws), ws.numel(), _stream())
    _lib.check(rc, "rift2_describe")
    return out


def match_vectors(ref_vec: torch.Tensor, ref_kp: torch.Tensor, tgt_vec: torch.Tensor, tgt_kp: torch.Tensor,
                  ws_key: str = "match_vectors"):
    """Generic float64 descriptor vectors (rows grouped by keypoint id)."""
    lib = _lib.load(require_gpu=True)
    nr, dim = ref_vec.shape
    nt = tgt_vec.shape[0]
    nbytes = ctypes.c_size_t()
    _lib.check(lib.rift2_match_vectors_workspace_size(nr, nt, ctypes.byref(nbytes)), "match_vectors")
    ws = WORKSPACES.get(ws_key, nbytes.value)
    dev = ref_vec.device
    out = dict(ref=torch.empty(nt, dtype=torch.int32, device=dev), tgt=torch.empty(nt, dtype=torch.int32, device=dev),
               dist=torch.empty(nt, dtype=torch.float64, device=dev), count=torch.empty(1, dtype=torch.int32, device=dev))
    rc = lib.rift2_match_vectors(_ptr(ref_vec), _ptr(ref_kp), nr, _ptr(tgt_vec), _ptr(tgt_kp), nt, dim,
                                 _ptr(out["ref"]), _ptr(out["tgt"]), _ptr(out["dist"]), _ptr(out["count"]),
                                 _ptr(ws), ws.numel(), _stream())
    _lib.check(rc, "rift2_match_vectors")
    return out


def match(desc: dict, dim: int, ref_block: torch.Tensor, tgt_block: torch.Tensor, tgt_kp_cap: int,
          ws_key: str = "match", out=None):
    """Nearest reference keypoint for every target keypoint of each pair.
    desc: the describe() dict (blocks = its batch); blocks given as int32
    CUDA tensors.  -> dict(ref, tgt, dist, count) sorted by (dist, ref, tgt)."""
    lib = _lib.load(require_gpu=True)
    counts = desc["counts"]
    n_blocks, cap, stride = counts.shape
    P = ref_block.numel()
    nbytes = ctypes.c_size_t()
    _lib.check(lib.rift2_match_workspace_size(P, cap, tgt_kp_cap, ctypes.byref(nbytes)), "match")
    ws = WORKSPACES.get(ws_key, nbytes.value)
    dev = counts.device
    kc = max(int(tgt_kp_cap), 1)
    if out is None:
        out = dict(ref=torch.empty((P, kc), dtype=torch.int32, device=dev),
                   tgt=torch.empty((P, kc), dtype=torch.int32, device=dev),
                   dist=torch.empty((P, kc), dtype=torch.float64, device=dev),
                   count=torch.empty((P,), dtype=torch.int32, device=dev))
    rc = lib.rift2_match(_ptr(counts), _ptr(desc["sqnorm"]), _ptr(desc["kp"]), _ptr(desc["count"]), n_blocks,
                         stride, cap, int(dim), P, _ptr(ref_block), _ptr(tgt_block), kc, _ptr(out["ref"]),
                         _ptr(out["tgt"]), _ptr(out["dist"]), _ptr(out["count"]), _ptr(ws), ws.numel(), _stream())
    _lib.check(rc, "rift2_match")
    return out


def match_partial(desc: dict, dim: int, ref_block: torch.Tensor, tgt_block: torch.Tensor, out=None):
    """Row-sharded matching, step 1 (rift2_match_partial): per target
    descriptor row the exact best candidate among this call's reference
    descriptors -> int32 tensor (P, cap, 4) of (dot, ref_sqnorm, ref_kp,
    score bits)."""
    lib = _lib.load(require_gpu=True)
    counts = desc["counts"]
    n_blocks, cap, stride = counts.shape
    P = ref_block.numel()
    if out is None:
        out = torch.empty((P, cap, 4), dtype=torch.int32, device=counts.device)
    rc = lib.rift2_match_partial(_ptr(counts), _ptr(desc["sqnorm"]), _ptr(desc["kp"]), _ptr(desc["count"]),
                                 n_blocks, stride, cap, int(dim), P, _ptr(ref_block), _ptr(tgt_block), _ptr(out),
                                 _stream())
    _lib.check(rc, "rift2_match_partial")
    return out


def match_finish(parts: torch.Tensor, desc: dict, dim: int, ref_block: torch.Tensor, tgt_block: torch.Tensor,
                 tgt_kp_cap: int, ws_key: str = "match_finish", out=None):
    """Row-sharded matching, step 2 (rift2_match_finish): exact combine of
    the gathered partials parts (G, P, cap, 4) over the FULL descriptor
    sets -> dict(ref, tgt, dist, count) as match()."""
    lib = _lib.load(require_gpu=True)
    counts = desc["counts"]
    n_blocks, cap, stride = counts.shape
    P = ref_block.numel()
    G = parts.shape[0]
    if parts.shape != (G, P, cap, 4) or parts.dtype != torch.int32:
        raise ParameterError(f"parts must be int32 ({G}, {P}, {cap}, 4), got {tuple(parts.shape)}")
    parts = parts.contiguous()
    nbytes = ctypes.c_size_t()
    _lib.check(lib.rift2_match_workspace_size(P, cap, tgt_kp_cap, ctypes.byref(nbytes)), "match_finish")
    ws = WORKSPACES.get(ws_key, nbytes.value)
    dev = counts.device
    kc = max(int(tgt_kp_cap), 1)
    if out is None:
        out = dict(ref=torch.empty((P, kc), dtype=torch.int32, device=dev),
                   tgt=torch.empty((P, kc), dtype=torch.int32, device=dev),
                   dist=torch.empty((P, kc), dtype=torch.float64, device=dev),
                   count=torch.empty((P,), dtype=torch.int32, device=dev))
    rc = lib.rift2_match_finish(_ptr(parts), G, _ptr(counts), _ptr(desc["sqnorm"]), _ptr(desc["kp"]),
                                _ptr(desc["count"]), n_blocks, stride, cap, int(dim), P, _ptr(ref_block),
                                _ptr(tgt_block), kc, _ptr(out["ref"]), _ptr(out["tgt"]), _ptr(out["dist"]),
                                _ptr(out["count"]), _ptr(ws), ws.numel(), _stream())
    _lib.check(rc, "rift2_match_finish")
    return out


def evaluate(kp: dict, ref_img: torch.Tensor, tgt_img: torch.Tensor, m: dict, gt: torch.Tensor,
             residual_threshold: float = 3.0, rmse_cap: float = 20.0, success_min_matches: int = 10, out=None):
    """Ground-truth scoring of match sets (rift2_evaluate).  kp: detect()
    dict (x, y, count; (images, K)); m: match() dict (ref, tgt, count);
    ref_img / tgt_img int32 (P,); gt (P, 6) float64 CUDA = R00 R01 R10 R11 t0
    t1.  -> dict(n_correct int32, rmse float64, success uint8, bad int32)."""
    lib = _lib.load(require_gpu=True)
    P = ref_img.numel()
    dev = gt.device
    if gt.dtype != torch.float64 or tuple(gt.shape) != (P, 6):
        raise ParameterError("gt must be a (n_pairs, 6) float64 tensor")
    if out is None:
        out = dict(n_correct=torch.empty(P, dtype=torch.int32, device=dev),
                   rmse=torch.empty(P, dtype=torch.float64, device=dev),
                   success=torch.empty(P, dtype=torch.uint8, device=dev),
                   bad=torch.empty(P, dtype=torch.int32, device=dev))
    rc = lib.rift2_evaluate(_ptr(kp["x"]), _ptr(kp["y"]), _ptr(kp["count"]), kp["x"].shape[1], _ptr(ref_img),
                            _ptr(tgt_img), _ptr(m["ref"]), _ptr(m["tgt"]), _ptr(m["count"]), m["ref"].shape[1], P,
                            _ptr(gt.contiguous()), float(residual_threshold), float(rmse_cap),
                            int(success_min_matches), _ptr(out["n_correct"]), _ptr(out["rmse"]),
                            _ptr(out["success"]), _ptr(out["bad"]), _stream())
    _lib.check(rc, "rift2_evaluate")
    return out


def debug_median(z: torch.Tensor):
    """Diagnostics (rift2_debug_median): z (planes, n) complex64 CUDA ->
    (amplitudes (planes, n) float32, exact medians (planes,) float32) through
    the filter bank's median kernels."""
    lib = _lib.load(require_gpu=True)
    if z.dim() != 2 or z.dtype != torch.complex64 or not z.is_cuda:
        raise ParameterError("z must be a (planes, n) complex64 CUDA tensor")
    z = z.contiguous()
    planes, n = z.shape
    nbytes = ctypes.c_size_t()
    _lib.check(lib.rift2_debug_median_workspace_size(planes, n, ctypes.byref(nbytes)), "debug_median")
    ws = torch.empty(nbytes.value, dtype=torch.uint8, device=z.device)
    amps = torch.empty((planes, n), dtype=torch.float32, device=z.device)
    med = torch.empty(planes, dtype=torch.float32, device=z.device)
    _lib.check(lib.rift2_debug_median(_ptr(z), planes, n, _ptr(amps), _ptr(med), _ptr(ws), ws.numel(), _stream()),
               "rift2_debug_median")
    return amps, med


def synth_targets(src: torch.Tensor, params: torch.Tensor, looks: torch.Tensor, seed: int, dst: torch.Tensor,
                  first_image: int = 0, src_copy: torch.Tensor | None = None):
    """Target synthesis (rift2_synth_targets): src (n, H, W) float64 CUDA
    sources; params (n, 8) float64 = target->source map (6), gamma, flags;
    looks (n,) int32; dst (n, H, W) float32 views (any image stride, rows
    contiguous), src_copy likewise or None."""
    lib = _lib.load(require_gpu=True)
    if src.dim() != 3 or src.dtype != torch.float64 or not src.is_cuda:
        raise ParameterError("src must be an (n, H, W) float64 CUDA tensor")
    n, H, W = src.shape
    if params.dtype != torch.float64 or tuple(params.shape) != (n, 8) or not params.is_contiguous():
        raise ParameterError("params must be a contiguous (n, 8) float64 tensor")
    if looks.dtype != torch.int32 or tuple(looks.shape) != (n,):
        raise ParameterError("looks must be an (n,) int32 tensor")
    for name, t in (("src", src), ("dst", dst), ("src_copy", src_copy)):
        if t is not None and (tuple(t.shape) != (n, H, W) or t.stride(1) != W or t.stride(2) != 1):
            raise ParameterError(f"{name} must be (n, {H}, {W}) with contiguous rows")
    if dst.dtype != torch.float32 or (src_copy is not None and src_copy.dtype != torch.float32):
        raise ParameterError("dst / src_copy must be float32")
    nbytes = ctypes.c_size_t()
    _lib.check(lib.rift2_synth_workspace_size(n, H, W, ctypes.byref(nbytes)), "synth_targets")
    ws = WORKSPACES.get("synth", nbytes.value)
    rc = lib.rift2_synth_targets(_ptr(src), src.stride(0), n, H, W, _ptr(params), _ptr(looks.contiguous()),
                                 int(seed) & (2**64 - 1), int(first_image), _ptr(dst), dst.stride(0), _ptr(src_copy),
                                 src_copy.stride(0) if src_copy is not None else 0, _ptr(ws), ws.numel(), _stream())
    _lib.check(rc, "rift2_synth_targets")
    return dst


# ---------------------------------------------------- unfused reference entry points
def filter_bank(height: int, width: int, bank) -> torch.Tensor:
    """rift2_filter_bank -> (S, O, H, W) float64 CUDA transfer functions."""
    lib = _lib.load(require_gpu=True)
    p = bank_c(bank)
    out = torch.empty((int(bank.n_scales), int(bank.n_orient), int(height), int(width)), dtype=torch.float64,
                      device="cuda")
    _lib.check(lib.rift2_filter_bank(int(height), int(width), ctypes.byref(p), _ptr(out), _stream()),
               "rift2_filter_bank")
    return out


def apply_bank(image: torch.Tensor, transfer: torch.Tensor, ws_key: str = "apply_bank"):
    """rift2_apply_bank: image (H, W) float32 CUDA, transfer (S, O, H, W)
    float32 CUDA -> (even, odd, amplitude) each (S, O, H, W) float32."""
    lib = _lib.load(require_gpu=True)
    H, W = image.shape
    S, O = transfer.shape[:2]
    nbytes = ctypes.c_size_t()
    _lib.check(lib.rift2_apply_bank_workspace_size(H, W, S, O, ctypes.byref(nbytes)), "apply_bank")
    ws = WORKSPACES.get(ws_key, nbytes.value)
    outs = [torch.empty((S, O, H, W), dtype=torch.float32, device=image.device) for _ in range(3)]
    _lib.check(lib.rift2_apply_bank(_ptr(image.contiguous()), H, W, S, O, _ptr(transfer.contiguous()),
                                    *(_ptr(t) for t in outs), _ptr(ws), ws.numel(), _stream()), "rift2_apply_bank")
    return tuple(outs)


def pc_moments(even, odd, amplitude: torch.Tensor, bank, full: bool = True, ws_key: str = "pc_moments"):
    """rift2_pc_moments on (S, O, H, W) float32 CUDA planes -> dict(a_o[,
    pc, mmax, mmin]) float32."""
    lib = _lib.load(require_gpu=True)
    S, O, H, W = amplitude.shape
    p = bank_c(bank)
    dev = amplitude.device
    out = {"a_o": torch.empty((O, H, W), dtype=torch.float32, device=dev)}
    ws = None
    if full:
        out.update(pc=torch.empty((O, H, W), dtype=torch.float32, device=dev),
                   mmax=torch.empty((H, W), dtype=torch.float32, device=dev),
                   mmin=torch.empty((H, W), dtype=torch.float32, device=dev))
        nbytes = ctypes.c_size_t()
        _lib.check(lib.rift2_pc_moments_workspace_size(H, W, ctypes.byref(p), ctypes.byref(nbytes)), "pc_moments")
        ws = WORKSPACES.get(ws_key, nbytes.value)
    _lib.check(lib.rift2_pc_moments(_ptr(even.contiguous() if full else None), _ptr(odd.contiguous() if full else None),
                                    _ptr(amplitude.contiguous()), H, W, ctypes.byref(p), _ptr(out["a_o"]),
                                    _ptr(out.get("pc")), _ptr(out.get("mmax")), _ptr(out.get("mmin")), _ptr(ws),
                                    0 if ws is None else ws.numel(), _stream()), "rift2_pc_moments")
    return out


def build_mim(a_o: torch.Tensor):
    """rift2_build_mim: (O, H, W) float64 CUDA -> (indices int32, max_amplitude float64)."""
    lib = _lib.load(require_gpu=True)
    O, H, W = a_o.shape
    idx = torch.empty((H, W), dtype=torch.int32, device=a_o.device)
    amax = torch.empty((H, W), dtype=torch.float64, device=a_o.device)
    _lib.check(lib.rift2_build_mim(_ptr(a_o.contiguous()), O, H, W, _ptr(idx), _ptr(amax), _stream()),
               "rift2_build_mim")
    return idx, amax


def patch_counts(indices: torch.Tensor, amplitude: torch.Tensor | None, n_orient: int, grid: int = 0,
                 hist: bool = True, cells: bool = False):
    """rift2_patch_counts: indices (n, h, w) int32 CUDA, amplitude same shape
    float64 or None -> (hist (n, n_orient) | None, cells (n, grid^2 n_orient) | None) float64."""
    lib = _lib.load(require_gpu=True)
    n, h, w = indices.shape
    dev = indices.device
    hh = torch.empty((n, n_orient), dtype=torch.float64, device=dev) if hist else None
    c = torch.empty((n, grid * grid * n_orient), dtype=torch.float64, device=dev) if cells else None
    _lib.check(lib.rift2_patch_counts(_ptr(indices.contiguous()), _ptr(None if amplitude is None else amplitude.contiguous()),
                                      n, h, w, int(n_orient), int(grid), _ptr(hh), _ptr(c), _stream()),
               "rift2_patch_counts")
    return hh, c


def remap_indices(indices: torch.Tensor, n_orient: int, pivot: int, kind: int) -> torch.Tensor:
    """rift2_remap_indices in place on an int32 CUDA tensor (kind 0 recode, 1 cyclic shift)."""
    lib = _lib.load(require_gpu=True)
    _lib.check(lib.rift2_remap_indices(_ptr(indices), indices.numel(), int(n_orient), int(pivot), int(kind),
                                       _stream()), "rift2_remap_indices")
    return indices


def extract_patch(indices: torch.Tensor, amplitude: torch.Tensor | None, x: float, y: float, size: int,
                  cos_a: float, sin_a: float, with_amplitude: bool):
    """rift2_extract_patch -> (indices (size, size) int32, amplitude float64 | None, out_of_bounds bool)."""
    lib = _lib.load(require_gpu=True)
    H, W = indices.shape
    dev = indices.device
    oi = torch.empty((size, size), dtype=torch.int32, device=dev)
    oa = torch.empty((size, size), dtype=torch.float64, device=dev) if with_amplitude else None
    oob = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(lib.rift2_extract_patch(_ptr(indices.contiguous()), _ptr(None if amplitude is None else amplitude.contiguous()),
                                       H, W, float(x), float(y), int(size), float(cos_a), float(sin_a), _ptr(oi), _ptr(oa),
                                       _ptr(oob), _stream()), "rift2_extract_patch")
    return oi, oa, bool(oob.item())


def orientation_amplitudes(amplitude: torch.Tensor) -> torch.Tensor:
    """rift2_orientation_amplitudes: (S, O, H, W) float64 CUDA -> (O, H, W) float64."""
    lib = _lib.load(require_gpu=True)
    S, O, H, W = amplitude.shape
    out = torch.empty((O, H, W), dtype=torch.float64, device=amplitude.device)
    _lib.check(lib.rift2_orientation_amplitudes(_ptr(amplitude.contiguous()), S, O, H, W, _ptr(out), _stream()),
               "rift2_orientation_amplitudes")
    return out


def synth_blobs(blobs: torch.Tensor, height: int, width: int) -> torch.Tensor:
    """rift2_synth_blobs: blobs (n, n_blobs, 11) float64 CUDA -> (n, H, W) float64."""
    lib = _lib.load(require_gpu=True)
    n, nb = blobs.shape[:2]
    out = torch.empty((n, height, width), dtype=torch.float64, device=blobs.device)
    _lib.check(lib.rift2_synth_blobs(_ptr(blobs.contiguous()), n, nb, height, width, _ptr(out), _stream()),
               "rift2_synth_blobs")
    return out


def synth_normals(seed: int, first_image: int, n_images: int, n: int, device="cuda") -> torch.Tensor:
    """rift2_synth_normals -> (n_images, n) float32 standard normals."""
    lib = _lib.load(require_gpu=True)
    out = torch.empty((n_images, n), dtype=torch.float32, device=device)
    _lib.check(lib.rift2_synth_normals(int(seed) & (2**64 - 1), int(first_image), n_images, n, _ptr(out), _stream()),
               "rift2_synth_normals")
    return out

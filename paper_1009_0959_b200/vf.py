"""Thin Python binding of libvf.so (include/vf.h): argument marshalling only.

PyTorch provides device memory and streams; every step of the filter runs in
the library's CUDA kernels.  There is no CPU fallback: if libvf.so is missing
or no CUDA device is present, these functions raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# VF_LIB selects another build of the same ABI (e.g. libvf_debug.so with device bounds checks)
LIB_PATH = os.environ.get("VF_LIB") or os.path.join(HERE, "libvf.so")

VF_ANGULAR, VF_EXP, VF_LOG, VF_AMNFE, VF_AMNFG, VF_EVMF = 0, 1, 2, 3, 4, 5
VF_EXACT, VF_MINIMAX, VF_MINIMAX_POLY4, VF_MINIMAX_REACH = 0, 1, 2, 3
VF_OK, VF_EINVAL, VF_EUNSUPPORTED, VF_ECUDA = 0, -1, -2, -3
VF_ALGO_AUTO, VF_ALGO_WINDOW, VF_ALGO_SHARED, VF_ALGO_ROLE, VF_ALGO_NO_TMA, VF_ALGO_STREAM = 0, 1, 2, 3, 16, 32

CRITERIA = {"angular": VF_ANGULAR, "exp": VF_EXP, "log": VF_LOG, "amnfe": VF_AMNFE, "amnfg": VF_AMNFG,
            "evmf": VF_EVMF}
VARIANTS = {"exact": VF_EXACT, "minimax": VF_MINIMAX, "poly4": VF_MINIMAX_POLY4, "reach": VF_MINIMAX_REACH}
ALGOS = {"auto": VF_ALGO_AUTO, "window": VF_ALGO_WINDOW, "shared": VF_ALGO_SHARED, "role": VF_ALGO_ROLE,
         "stream": VF_ALGO_STREAM}
EXPORTS = ["vf_filter", "vf_filter_batch", "vf_filter_rows", "vf_filter_batch_algo",
           "vf_host_workspace_bytes", "vf_filter_host", "vf_plan_create", "vf_plan_create_ex", "vf_plan_launch", "vf_plan_kernels",
           "vf_plan_destroy", "vf_image_stats", "vf_image_stats_ex", "vf_image_stats_multi", "vf_kernel_info", "vf_status_string", "vf_last_error", "vf_version"]
VF_STATS_NO_REF_NORM = 1


class VFError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: status {status} ({msg})")
        self.status = status


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libvf.so (does not need a GPU).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -m paper_1009_0959_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(path)
    P, I, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    L.vf_filter.argtypes = [P, I, I, I, I, I, P, P, P, P]
    L.vf_filter_batch.argtypes = [P, I, I, I, I, I, I, P, P, P, P]
    L.vf_filter_batch_algo.argtypes = [P, I, I, I, I, I, I, I, P, P, P, P]
    L.vf_filter_rows.argtypes = [P, I, I, I, I, I, I, I, I, I, P, P, P, P]
    L.vf_host_workspace_bytes.argtypes = [I, I, I]
    L.vf_host_workspace_bytes.restype = S
    L.vf_filter_host.argtypes = [P, I, I, I, I, I, I, P, P, S, P]
    L.vf_plan_create.argtypes = [ctypes.POINTER(P), I, I, I, I, I, P, P, P, P, P, P]
    L.vf_plan_create_ex.argtypes = [ctypes.POINTER(P), I, I, I, I, I, P, P, P, P, P, P, P, P]
    L.vf_plan_launch.argtypes = [P, P]
    L.vf_plan_destroy.argtypes = [P]
    L.vf_plan_kernels.argtypes = [P]
    L.vf_image_stats.argtypes = [P, P, I, I, I, P, P]
    L.vf_image_stats_ex.argtypes = [P, P, I, I, I, P, I, P]
    L.vf_image_stats_multi.argtypes = [P, ctypes.POINTER(P), I, I, I, I, P, I, P]
    L.vf_kernel_info.argtypes = [I, I, I, I, I, I, I, ctypes.c_char_p, I, ctypes.POINTER(ctypes.c_longlong)]
    L.vf_status_string.argtypes = [I]
    L.vf_status_string.restype = ctypes.c_char_p
    L.vf_last_error.argtypes = []
    L.vf_last_error.restype = ctypes.c_char_p
    L.vf_version.argtypes = []
    for name in ("vf_filter", "vf_filter_batch", "vf_filter_batch_algo", "vf_filter_rows",
                 "vf_filter_host", "vf_plan_create", "vf_plan_create_ex", "vf_plan_launch", "vf_plan_kernels", "vf_plan_destroy", "vf_image_stats",
                 "vf_image_stats_ex", "vf_image_stats_multi", "vf_kernel_info", "vf_version"):
        getattr(L, name).restype = I
    _lib = L
    return L


def _check(rc: int, where: str):
    if rc != VF_OK:
        L = load_library()
        raise VFError(rc, where, L.vf_last_error().decode() or L.vf_status_string(rc).decode())


def _crit(c) -> int:
    return CRITERIA[c] if isinstance(c, str) else int(c)


def _var(v) -> int:
    return VARIANTS[v] if isinstance(v, str) else int(v)


def _algo(a) -> int:
    """'auto' | 'window' | 'shared' | int, optionally 'shared:2' / 'auto:1' (tile override, see vf.h)
    and/or a '+notma' suffix (VF_ALGO_NO_TMA)."""
    if isinstance(a, str):
        a, plus, flag = a.partition("+")
        if plus and flag != "notma":
            raise ValueError(f"unknown algo flag {flag!r}")
        base, _, t = a.partition(":")
        return ALGOS[base] | ((int(t) if t else 0) << 2) | (VF_ALGO_NO_TMA if plus else 0)
    return int(a)


def _dev_u8(t: torch.Tensor, name: str):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.uint8 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous uint8 tensor")
    return t.data_ptr()


def _same_device(ref: torch.Tensor, *ts):
    """Every buffer handed to the library must live on the input's device (the
    kernels launch on the current device: see _on_device)."""
    for t in ts:
        if t is not None and (not t.is_cuda or t.device != ref.device):
            raise ValueError(f"all buffers must be on {ref.device} (got {t.device})")


def _check_buf(t, name: str, dtype, numel: int):
    if t is None:
        return
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype or not t.is_contiguous() or t.numel() != numel:
        raise ValueError(f"{name} must be a contiguous {dtype} tensor with {numel} elements "
                         f"(got {t.dtype}, {t.numel()})")


def _stream(stream) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _ptr_or_none(t):
    return None if t is None else t.data_ptr()


def vf_filter_batch_algo(imgs: torch.Tensor, window: int, criterion, variant, algo="auto",
                         out: Optional[torch.Tensor] = None, index: Optional[torch.Tensor] = None,
                         aggregates: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """imgs: CUDA uint8 [B, H, W, 3] (or [H, W, 3]).  Returns out (same shape)."""
    L = load_library()
    single = imgs.dim() == 3
    x = imgs.unsqueeze(0) if single else imgs
    if x.dim() != 4 or x.shape[-1] != 3:
        raise ValueError("expected [B, H, W, 3] or [H, W, 3]")
    B, H, W, _ = x.shape
    n = window * window
    _dev_u8(x, "imgs")
    if out is None:
        out = torch.empty_like(imgs)
    _check_buf(out, "out", torch.uint8, B * H * W * 3)
    _check_buf(index, "index", torch.uint8, B * H * W)
    _check_buf(aggregates, "aggregates", torch.float32, B * H * W * n)
    _same_device(x, out, index, aggregates)
    with torch.cuda.device(x.device):
            rc = L.vf_filter_batch_algo(_dev_u8(x, "imgs"), B, H, W, window, _crit(criterion), _var(variant),
                                    _algo(algo),
                                    _dev_u8(out, "out"), _ptr_or_none(index), _ptr_or_none(aggregates),
                                    _stream(stream))
    _check(rc, "vf_filter_batch_algo")
    return out


def vf_filter_batch(imgs, window, criterion, variant, out=None, index=None, aggregates=None, stream=None):
    return vf_filter_batch_algo(imgs, window, criterion, variant, "auto", out, index, aggregates, stream)


def vf_filter(img, window, criterion, variant, out=None, index=None, aggregates=None, stream=None):
    if img.dim() != 3:
        raise ValueError("vf_filter expects [H, W, 3]")
    return vf_filter_batch_algo(img, window, criterion, variant, "auto", out, index, aggregates, stream)


def vf_filter_rows(band: torch.Tensor, band_row0: int, H: int, out_row0: int, out_rows: int, window: int,
                   criterion, variant, out: Optional[torch.Tensor] = None, index=None, aggregates=None,
                   stream=None) -> torch.Tensor:
    """band: CUDA uint8 [band_rows, W, 3] holding global rows [band_row0, ...)."""
    L = load_library()
    if band.dim() != 3 or band.shape[-1] != 3:
        raise ValueError("band must be [band_rows, W, 3]")
    band_rows, W, _ = band.shape
    _dev_u8(band, "band")
    if out is None:
        out = torch.empty((max(out_rows, 0), W, 3), dtype=torch.uint8, device=band.device)
    _check_buf(out, "out", torch.uint8, max(out_rows, 0) * W * 3)
    _check_buf(index, "index", torch.uint8, max(out_rows, 0) * W)
    _check_buf(aggregates, "aggregates", torch.float32, max(out_rows, 0) * W * window * window)
    _same_device(band, out, index, aggregates)
    with torch.cuda.device(band.device):
        rc = L.vf_filter_rows(_dev_u8(band, "band"), band_row0, band_rows, H, W, out_row0, out_rows, window,
                              _crit(criterion), _var(variant), _dev_u8(out, "out"), _ptr_or_none(index),
                              _ptr_or_none(aggregates), _stream(stream))
    _check(rc, "vf_filter_rows")
    return out


def vf_host_workspace_bytes(B: int, H: int, W: int) -> int:
    return int(load_library().vf_host_workspace_bytes(B, H, W))


def vf_filter_host(h_imgs: torch.Tensor, window: int, criterion, variant, h_out: torch.Tensor,
                   workspace: torch.Tensor, stream=None) -> torch.Tensor:
    """End-to-end call on HOST tensors (pinned for async copies): enqueues
    H2D -> filter -> D2H on the stream; synchronise before reading h_out."""
    L = load_library()
    x = h_imgs.unsqueeze(0) if h_imgs.dim() == 3 else h_imgs
    B, H, W, _ = x.shape
    for t, nm in ((x, "h_imgs"), (h_out, "h_out")):
        if t.is_cuda or t.dtype != torch.uint8 or not t.is_contiguous():
            raise ValueError(f"{nm} must be a contiguous uint8 host tensor")
    if not workspace.is_cuda:
        raise ValueError("workspace must be a CUDA tensor")
    rc = L.vf_filter_host(x.data_ptr(), B, H, W, window, _crit(criterion), _var(variant), h_out.data_ptr(),
                          workspace.data_ptr(), workspace.numel() * workspace.element_size(), _stream(stream))
    _check(rc, "vf_filter_host")
    return h_out


class Plan:
    """vf_plan_* (include/vf.h): several filters of one input as ONE CUDA graph
    with independent (concurrent) kernel nodes, optionally with the H2D copy
    of a host input and the D2H copies of the outputs inside the graph.

    d_in: CUDA uint8 [B, H, W, 3]; d_outs: list of CUDA tensors like d_in;
    combos: list of (criterion, variant); h_in / h_outs: pinned host tensors
    (optional).  refs (optional, vf_plan_create_ex): refs[i] = index of the
    filter whose output filter i is compared with (-1: none); stats: CUDA
    float64 [ncmp, B, 8] (ncmp = number of refs >= 0) written at every launch
    with vf_image_stats_multi's rows, bit-identical.  Buffers are bound at
    creation; call launch() per step."""

    def __init__(self, d_in: torch.Tensor, d_outs, window: int, combos, h_in: Optional[torch.Tensor] = None,
                 h_outs=None, refs=None, stats: Optional[torch.Tensor] = None):
        L = load_library()
        x = d_in.unsqueeze(0) if d_in.dim() == 3 else d_in
        B, H, W, _ = x.shape
        n = len(combos)
        if len(d_outs) != n or (h_outs is not None and len(h_outs) != n):
            raise ValueError("one output per filter")
        for t in d_outs:
            _dev_u8(t, "d_outs[i]")
            if t.numel() != x.numel():
                raise ValueError("outputs must match the input size")
        _same_device(x, *d_outs)
        if h_in is not None and (h_in.is_cuda or h_in.dtype != torch.uint8 or h_in.numel() != x.numel()
                                 or not h_in.is_contiguous()):
            raise ValueError("h_in must be a contiguous host uint8 tensor like d_in")
        for t in (h_outs or []):
            if t.is_cuda or t.dtype != torch.uint8 or t.numel() != x.numel() or not t.is_contiguous():
                raise ValueError("h_outs[i] must be contiguous host uint8 tensors like d_in")
        ncmp = 0
        if refs is not None:
            refs = [int(r) for r in refs]
            if len(refs) != n:
                raise ValueError("one reference index (or -1) per filter")
            ncmp = sum(1 for r in refs if r >= 0)
        if ncmp:
            if (stats is None or not stats.is_cuda or stats.dtype != torch.float64 or not stats.is_contiguous()
                    or stats.numel() != ncmp * B * 8):
                raise ValueError(f"stats must be a contiguous CUDA float64 tensor of {ncmp} x {B} x 8")
            _same_device(x, stats)
        self.device = x.device
        self._keep = (d_in, list(d_outs), h_in, None if h_outs is None else list(h_outs), stats)
        crit = (ctypes.c_int * n)(*[_crit(c) for c, _ in combos])
        var = (ctypes.c_int * n)(*[_var(v) for _, v in combos])
        douts = (ctypes.c_void_p * n)(*[t.data_ptr() for t in d_outs])
        houts = None if h_outs is None else (ctypes.c_void_p * n)(*[t.data_ptr() for t in h_outs])
        self._h = ctypes.c_void_p()
        with torch.cuda.device(x.device):
            if refs is None:
                rc = L.vf_plan_create(ctypes.byref(self._h), B, H, W, window, n, crit, var, _dev_u8(x, "d_in"),
                                      douts, None if h_in is None else h_in.data_ptr(), houts)
            else:
                rarr = (ctypes.c_int * n)(*refs)
                rc = L.vf_plan_create_ex(ctypes.byref(self._h), B, H, W, window, n, crit, var, _dev_u8(x, "d_in"),
                                         douts, None if h_in is None else h_in.data_ptr(), houts, rarr,
                                         None if not ncmp else stats.data_ptr())
        _check(rc, "vf_plan_create_ex" if refs is not None else "vf_plan_create")
        self.n = n
        self.ncmp = ncmp

    def launch(self, stream=None):
        with torch.cuda.device(self.device):
            _check(load_library().vf_plan_launch(self._h, _stream(stream)), "vf_plan_launch")

    def kernels(self) -> int:
        """Kernel nodes of the plan's graph (exp/log filters of large plans fuse into one)."""
        rc = load_library().vf_plan_kernels(self._h)
        if rc < 0:
            _check(rc, "vf_plan_kernels")
        return rc

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load_library().vf_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def vf_image_stats(a: torch.Tensor, b: torch.Tensor, stats: Optional[torch.Tensor] = None,
                   stream=None, ref_norm: bool = True) -> torch.Tensor:
    """Per-image [B, 8] float64 statistics (see include/vf.h).  ref_norm=False
    (vf_image_stats_ex, VF_STATS_NO_REF_NORM) skips column 4 (sum |a_Lab|,
    a function of `a` alone), which is then 0."""
    return vf_image_stats_multi(a, [b], None if stats is None else stats.view(1, *stats.shape), stream,
                                ref_norm)[0]


def vf_image_stats_multi(a: torch.Tensor, bs, stats: Optional[torch.Tensor] = None, stream=None,
                         ref_norm: bool = True) -> torch.Tensor:
    """One pass over the reference `a` against every output in `bs` (1..8
    tensors shaped like a): float64 [len(bs), B, 8], row [k] as
    vf_image_stats(a, bs[k])."""
    L = load_library()
    x = a.unsqueeze(0) if a.dim() == 3 else a
    if x.dim() != 4 or x.shape[-1] != 3:
        raise ValueError("expected [B, H, W, 3] or [H, W, 3]")
    B, H, W, _ = x.shape
    nb = len(bs)
    if not 1 <= nb <= 8:
        raise ValueError("compare 1..8 outputs per call")
    _dev_u8(x, "a")
    for i, b in enumerate(bs):
        _dev_u8(b, f"bs[{i}]")
        if b.numel() != x.numel():
            raise ValueError(f"bs[{i}] must have the shape of a ({tuple(a.shape)}), got {tuple(b.shape)}")
    if stats is None:
        stats = torch.empty((nb, B, 8), dtype=torch.float64, device=a.device)
    _check_buf(stats, "stats", torch.float64, nb * B * 8)
    _same_device(x, stats, *bs)
    arr = (ctypes.c_void_p * nb)(*[b.data_ptr() for b in bs])
    with torch.cuda.device(x.device):
        rc = L.vf_image_stats_multi(_dev_u8(x, "a"), arr, nb, B, H, W, stats.data_ptr(),
                                    0 if ref_norm else VF_STATS_NO_REF_NORM, _stream(stream))
    _check(rc, "vf_image_stats_multi")
    return stats.view(nb, B, 8)


def vf_kernel_info(B: int, H: int, W: int, window: int, criterion, variant, algo="auto") -> dict:
    """The kernel vf_filter_batch_algo would launch for these arguments
    (mangled name, grid, block, dynamic smem); no device work."""
    L = load_library()
    buf = ctypes.create_string_buffer(1024)
    lau = (ctypes.c_longlong * 7)()
    _check(L.vf_kernel_info(B, H, W, window, _crit(criterion), _var(variant), _algo(algo), buf, 1024, lau),
           "vf_kernel_info")
    return {"name": buf.value.decode(), "grid": tuple(lau[0:3]), "block": tuple(lau[3:6]), "smem": int(lau[6])}


def vf_status_string(status: int) -> str:
    return load_library().vf_status_string(status).decode()


def vf_last_error() -> str:
    return load_library().vf_last_error().decode()


def vf_plan_create(*a, **k) -> "Plan":
    return Plan(*a, **k)


def vf_version() -> int:
    return int(load_library().vf_version())


# --------------------------------------------------------------- conveniences
def filter(img: torch.Tensor, window: int = 3, criterion="angular", variant="minimax", algo="auto",
           want_index: bool = False, want_agg: bool = False, stream=None):
    """Filter a CUDA uint8 image [H, W, 3] or batch [B, H, W, 3].
    Returns (out, index | None, aggregates | None)."""
    shape = img.shape[:-1]
    n = window * window
    idx = torch.empty(shape, dtype=torch.uint8, device=img.device) if want_index else None
    agg = torch.empty(tuple(shape) + (n,), dtype=torch.float32, device=img.device) if want_agg else None
    out = vf_filter_batch_algo(img, window, criterion, variant, algo, None, idx, agg, stream)
    return out, idx, agg


def fidelity(a: torch.Tensor, b: torch.Tensor) -> dict:
    """PSNR / NCD / MAE / MSE / fraction of differing pixels of b against a
    (the paper's quality measures), per batch, from vf_image_stats."""
    import math
    per = vf_image_stats(a, b).double().cpu()
    s = per.sum(0).tolist()
    s[5] = float(per[:, 5].max())           # the batch maximum, not the sum of per-image maxima
    x = a.unsqueeze(0) if a.dim() == 3 else a
    npix = x.shape[0] * x.shape[1] * x.shape[2]
    mse = s[2] / (3 * npix)
    return dict(diff_frac=s[0] / npix, mae=s[1] / (3 * npix), mse=mse,
                psnr_db=(math.inf if mse == 0 else 10 * math.log10(255.0 ** 2 / mse)),
                ncd=(s[3] / s[4] if s[4] > 0 else float("nan")), max_abs=s[5])

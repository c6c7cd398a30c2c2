"""PyTorch-facing binding of libfftconv.so.

PyTorch supplies device memory and the current CUDA stream only; this module
marshals pointers and sizes into the C ABI (include/fftconv.h) with the same
entry-point names.  It performs no arithmetic of the method.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _abi

_DT = {torch.float16: _abi.FFTCONV_F16, torch.bfloat16: _abi.FFTCONV_BF16, torch.float32: _abi.FFTCONV_F32}


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _aligned_empty(nbytes: int, device, align: int = 1024):
    """uint8 device buffer whose data_ptr is `align`-byte aligned."""
    raw = torch.empty(nbytes + align, dtype=torch.uint8, device=device)
    off = (-raw.data_ptr()) % align
    return raw[off:off + nbytes]


@dataclass
class PlanInfo:
    N: int
    fft_size: int
    causal: bool
    regime: int
    order: int
    factors: tuple
    rows_per_tile: int
    max_kernel_len: int
    table_bytes: int
    kf_bytes_per_head: int
    workspace_bytes_per_head: int
    mask_fraction: float
    skip_fraction: float


class FFTConvPlan:
    """fftconv_plan + fftconv_plan_upload.  `sparsity` = (dims, keep_masks)
    with dims slowest-first and keep_masks a list of 0/1 sequences."""

    def __init__(self, N: int, fft_size: int | None = None, dtype=torch.float16, causal: bool = True,
                 sparsity=None, device="cuda"):
        L = _abi.lib()
        fft_size = int(fft_size if fft_size is not None else (2 * N if causal else N))
        self.dtype = dtype
        self.device = torch.device(device)
        sp = None
        self._keep_bufs = []
        if sparsity is not None:
            dims, keeps = sparsity
            sp = _abi.Sparsity()
            sp.ndims = len(dims)
            for j, (d, kp) in enumerate(zip(dims, keeps)):
                sp.dims[j] = int(d)
                buf = (ctypes.c_uint8 * int(d))(*[1 if x else 0 for x in kp])
                self._keep_bufs.append(buf)
                sp.keep[j] = ctypes.cast(buf, ctypes.POINTER(ctypes.c_uint8))
        h = ctypes.c_void_p()
        _abi.check(L.fftconv_plan(ctypes.byref(h), int(N), fft_size, _DT[dtype], int(bool(causal)),
                                  ctypes.byref(sp) if sp is not None else None))
        self._h = h
        info = _abi.PlanInfo()
        _abi.check(L.fftconv_plan_info(h, ctypes.byref(info)))
        self.info = PlanInfo(info.N, info.fft_size, bool(info.causal), info.regime, info.order,
                             tuple(info.factors[:max(info.order, 2)]), info.rows_per_tile,
                             info.max_kernel_len, info.table_bytes, info.kf_bytes_per_head,
                             info.workspace_bytes_per_head, info.mask_fraction, info.skip_fraction)
        with torch.cuda.device(self.device):
            self.tables = _aligned_empty(info.table_bytes, self.device)
            _abi.check(L.fftconv_plan_upload(h, _ptr(self.tables), _stream(self.device)))

    @property
    def N(self):
        return self.info.N

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _abi.lib().fftconv_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    # ------------------------------------------------------------------ calls
    def kf_buffer(self, H: int, device=None) -> torch.Tensor:
        """An opaque k_f buffer for H heads (reusable across precompute_kf calls)."""
        return _aligned_empty(max(H, 1) * self.info.kf_bytes_per_head, device or self.device, 16)

    def precompute_kf(self, k: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """k: (H, K) fp32 on device -> opaque k_f buffer (H * kf_bytes_per_head),
        written into `out` (from kf_buffer) when given."""
        if not (isinstance(k, torch.Tensor) and k.dtype == torch.float32 and k.is_cuda and k.dim() == 2):
            raise ValueError("k must be an (H, K) float32 CUDA tensor")
        k = k.contiguous()
        H, K = k.shape
        if out is not None:
            if not (out.numel() * out.element_size() >= max(H, 1) * self.info.kf_bytes_per_head and out.data_ptr() % 16 == 0):
                raise ValueError("kf out buffer too small or not 16-byte aligned")
            kf = out
        else:
            kf = _aligned_empty(max(H, 1) * self.info.kf_bytes_per_head, k.device, 16)
        _abi.check(_abi.lib().fftconv_precompute_kf(self._h, _ptr(k), H, K, _ptr(kf), _stream(k.device)))
        return kf

    def precompute_kf_bidir(self, k_fwd: torch.Tensor, k_bwd: torch.Tensor, out: torch.Tensor | None = None):
        """Bidirectional filters (reading B1): k_fwd, k_bwd (H, K) fp32 on
        device -> opaque k_f of the two-sided filter, for fwd / gated_fwd."""
        for k in (k_fwd, k_bwd):
            if not (isinstance(k, torch.Tensor) and k.dtype == torch.float32 and k.is_cuda and k.dim() == 2):
                raise ValueError("k_fwd and k_bwd must be (H, K) float32 CUDA tensors")
        if k_fwd.shape != k_bwd.shape or k_fwd.device != k_bwd.device:
            raise ValueError("k_fwd and k_bwd must have one shape and device")
        k_fwd, k_bwd = k_fwd.contiguous(), k_bwd.contiguous()
        H, K = k_fwd.shape
        kf = out if out is not None else _aligned_empty(max(H, 1) * self.info.kf_bytes_per_head, k_fwd.device, 16)
        self._check_kf(kf, H, k_fwd.device)
        _abi.check(_abi.lib().fftconv_precompute_kf_bidir(self._h, _ptr(k_fwd), _ptr(k_bwd), H, K, _ptr(kf),
                                                          _stream(k_fwd.device)))
        return kf

    def _check_sig(self, *ts):
        """Signal tensors (B, H, N): plan dtype, contiguous, on one CUDA
        device, all the same shape (the C ABI takes raw pointers: a mismatch
        here would be an out-of-bounds device access there)."""
        ref = None
        for t in ts:
            if t is None:
                continue
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == self.dtype and t.is_contiguous()
                    and t.dim() == 3 and t.shape[-1] == self.info.N):
                raise ValueError(f"signal tensor must be a contiguous CUDA (B, H, {self.info.N}) {self.dtype} "
                                 f"tensor, got {getattr(t, 'shape', None)} {getattr(t, 'dtype', None)}")
            if ref is None:
                ref = t
            elif t.shape != ref.shape or t.device != ref.device:
                raise ValueError(f"signal tensors disagree: {tuple(t.shape)}@{t.device} vs "
                                 f"{tuple(ref.shape)}@{ref.device}")
        return ref

    def _check_kf(self, kf, H, device):
        need = max(H, 1) * self.info.kf_bytes_per_head
        if not (isinstance(kf, torch.Tensor) and kf.is_cuda and kf.device == device and kf.is_contiguous()):
            raise ValueError("kf must be a contiguous CUDA buffer from precompute_kf on the signals' device")
        if kf.numel() * kf.element_size() < need:
            raise ValueError(f"kf holds {kf.numel() * kf.element_size()} bytes, {H} heads need {need}")

    def _check_out(self, out, like, name="out"):
        if out is None:
            return torch.empty_like(like)
        if not (isinstance(out, torch.Tensor) and out.shape == like.shape and out.dtype == like.dtype
                and out.device == like.device and out.is_contiguous()):
            raise ValueError(f"{name} must be a contiguous {like.dtype} tensor of shape {tuple(like.shape)} "
                             f"on {like.device}")
        return out

    def _check_ws(self, ws, B, H, for_bwd, device):
        need = self.workspace_bytes(B, H, for_bwd)
        if ws is None:
            return self.workspace(B, H, for_bwd, device=device)
        if not (isinstance(ws, torch.Tensor) and ws.is_cuda and ws.device == device and ws.is_contiguous()):
            raise ValueError("workspace must be a contiguous CUDA buffer on the signals' device")
        if ws.numel() * ws.element_size() < need:
            raise ValueError(f"workspace holds {ws.numel() * ws.element_size()} bytes, needs {need}")
        return ws

    def workspace_bytes(self, B: int, H: int, for_bwd: bool = False) -> int:
        n = ctypes.c_size_t()
        _abi.check(_abi.lib().fftconv_workspace_size(self._h, B, H, int(for_bwd), ctypes.byref(n)))
        return int(n.value)

    def workspace(self, B: int, H: int, for_bwd: bool = False, device=None):
        n = self.workspace_bytes(B, H, for_bwd)
        if n == 0:
            return None
        return _aligned_empty(n, device or self.device, 16)

    def fwd(self, u: torch.Tensor, kf: torch.Tensor, out: torch.Tensor | None = None, workspace=None) -> torch.Tensor:
        self._check_sig(u)
        B, H, _ = u.shape
        self._check_kf(kf, H, u.device)
        y = self._check_out(out, u)
        ws = self._check_ws(workspace, B, H, False, u.device)
        _abi.check(_abi.lib().fftconv_fwd(self._h, _ptr(u), _ptr(kf), _ptr(y), B, H, _ptr(ws), _stream(u.device)))
        return y

    def gated_fwd(self, u, w, v, kf, out=None, workspace=None):
        if w is None or v is None:
            raise ValueError("gated_fwd needs both gates w and v")
        self._check_sig(u, w, v)
        B, H, _ = u.shape
        self._check_kf(kf, H, u.device)
        y = self._check_out(out, u)
        ws = self._check_ws(workspace, B, H, False, u.device)
        _abi.check(_abi.lib().fftconv_gated_fwd(self._h, _ptr(u), _ptr(w), _ptr(v), _ptr(kf), _ptr(y), B, H,
                                                _ptr(ws), _stream(u.device)))
        return y

    def fwd_host(self, u: torch.Tensor, kf: torch.Tensor, w=None, v=None, out=None, rows_per_chunk: int = 8,
                 stage=None) -> torch.Tensor:
        """End-to-end forward from (pinned) host tensors through fftconv_fwd_host:
        batch rows are streamed through a device staging buffer with the
        copies of neighbouring chunks overlapping the convolution."""
        self._check_host(u, w, v, out, n=self.info.N)
        B, H, N = u.shape
        self._check_kf(kf, H, kf.device)
        out = torch.empty_like(u, pin_memory=u.is_pinned()) if out is None else out
        gated = w is not None
        n = ctypes.c_size_t()
        _abi.check(_abi.lib().fftconv_host_stage_size(self._h, H, rows_per_chunk, int(gated), ctypes.byref(n)))
        if stage is None or stage.numel() < n.value:
            stage = _aligned_empty(int(n.value), kf.device, 1024)
        _abi.check(_abi.lib().fftconv_fwd_host(self._h, _ptr(u), _ptr(w), _ptr(v), _ptr(kf), _ptr(out), B, H,
                                               rows_per_chunk, _ptr(stage), stage.numel(), _stream(kf.device)))
        self._stage = stage  # keep the staging buffer alive while the copies run
        return out

    def fwd_stream(self, u: torch.Tensor, kf: torch.Tensor, w=None, v=None, out=None, stage=None) -> torch.Tensor:
        """Partial plans: host rows (B, H, N_total) of any length streamed in
        segments of the plan's N through fftconv_fwd_stream."""
        self._check_host(u, w, v, out)
        B, H, NT = u.shape
        self._check_kf(kf, H, kf.device)
        out = torch.empty_like(u, pin_memory=u.is_pinned()) if out is None else out
        n = ctypes.c_size_t()
        _abi.check(_abi.lib().fftconv_stream_stage_size(self._h, B, H, int(w is not None), ctypes.byref(n)))
        if stage is None or stage.numel() < n.value:
            stage = _aligned_empty(int(n.value), kf.device, 1024)
        _abi.check(_abi.lib().fftconv_fwd_stream(self._h, _ptr(u), _ptr(w), _ptr(v), _ptr(kf), _ptr(out), B, H, NT,
                                                 _ptr(stage), stage.numel(), _stream(kf.device)))
        self._stage = stage
        return out

    def _check_host(self, u, w, v, out, n=None):
        """Host signal tensors: plan dtype, contiguous, CPU, one shape; both
        gates or none."""
        if (w is None) != (v is None):
            raise ValueError("gated host calls need both w and v")
        for t in (u, w, v, out):
            if t is None:
                continue
            if not (isinstance(t, torch.Tensor) and not t.is_cuda and t.dtype == self.dtype and t.is_contiguous()
                    and t.shape == u.shape and t.dim() == 3):
                raise ValueError(f"host tensors must be contiguous CPU {self.dtype} tensors of shape {tuple(u.shape)}")
        if n is not None and u.shape[-1] != n:
            raise ValueError(f"row length {u.shape[-1]} != plan N {n}")

    def host_stage(self, H: int, rows_per_chunk: int = 8, gated: bool = False, device=None):
        n = ctypes.c_size_t()
        _abi.check(_abi.lib().fftconv_host_stage_size(self._h, H, rows_per_chunk, int(gated), ctypes.byref(n)))
        return _aligned_empty(int(n.value), device or self.device, 1024)

    def bwd(self, dy, u, kf, K, w=None, v=None):
        """Gradients of <y, dy>: returns du, dw, dv (None when ungated) and dk (H, K)."""
        if (w is None) != (v is None):
            raise ValueError("bwd: the gated backward needs both w and v")
        self._check_sig(dy, u, w, v)
        B, H, _ = u.shape
        self._check_kf(kf, H, u.device)
        du = torch.empty_like(u)
        dw = torch.empty_like(u) if w is not None else None
        dv = torch.empty_like(u) if v is not None else None
        dk = torch.empty(H, K, dtype=torch.float32, device=u.device)
        ws = self.workspace(B, H, for_bwd=True, device=u.device)
        _abi.check(_abi.lib().fftconv_bwd(self._h, _ptr(dy), _ptr(u), _ptr(w), _ptr(v), _ptr(kf), _ptr(du),
                                          _ptr(dw), _ptr(dv), _ptr(dk), B, H, K, _ptr(ws), _stream(u.device)))
        return {"du": du, "dw": dw, "dv": dv, "dk": dk}

    def bwd_bidir(self, dy, u, kf, K, w=None, v=None):
        """Gradients of <y, dy> for a bidirectional k_f: du, dw, dv, dk_fwd, dk_bwd."""
        if (w is None) != (v is None):
            raise ValueError("bwd_bidir: the gated backward needs both w and v")
        self._check_sig(dy, u, w, v)
        B, H, _ = u.shape
        self._check_kf(kf, H, u.device)
        du = torch.empty_like(u)
        dw = torch.empty_like(u) if w is not None else None
        dv = torch.empty_like(u) if v is not None else None
        dkf = torch.empty(H, K, dtype=torch.float32, device=u.device)
        dkb = torch.empty(H, K, dtype=torch.float32, device=u.device)
        ws = self.workspace(B, H, for_bwd=True, device=u.device)
        _abi.check(_abi.lib().fftconv_bwd_bidir(self._h, _ptr(dy), _ptr(u), _ptr(w), _ptr(v), _ptr(kf), _ptr(du),
                                                _ptr(dw), _ptr(dv), _ptr(dkf), _ptr(dkb), B, H, K, _ptr(ws),
                                                _stream(u.device)))
        return {"du": du, "dw": dw, "dv": dv, "dk_fwd": dkf, "dk_bwd": dkb}


def launch_count_reset() -> int:
    return int(_abi.lib().fftconv_launch_count_reset())

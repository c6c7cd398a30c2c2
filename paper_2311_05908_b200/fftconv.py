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
        assert k.dtype == torch.float32 and k.is_cuda and k.dim() == 2
        k = k.contiguous()
        H, K = k.shape
        if out is not None:
            assert out.numel() >= max(H, 1) * self.info.kf_bytes_per_head and out.data_ptr() % 16 == 0
            kf = out
        else:
            kf = _aligned_empty(max(H, 1) * self.info.kf_bytes_per_head, k.device, 16)
        _abi.check(_abi.lib().fftconv_precompute_kf(self._h, _ptr(k), H, K, _ptr(kf), _stream(k.device)))
        return kf

    def _check_sig(self, *ts):
        for t in ts:
            assert t.is_cuda and t.dtype == self.dtype and t.is_contiguous() and t.dim() == 3
            assert t.shape[-1] == self.info.N, (t.shape, self.info.N)

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
        y = torch.empty_like(u) if out is None else out
        ws = workspace if workspace is not None else self.workspace(B, H, device=u.device)
        _abi.check(_abi.lib().fftconv_fwd(self._h, _ptr(u), _ptr(kf), _ptr(y), B, H, _ptr(ws), _stream(u.device)))
        return y

    def gated_fwd(self, u, w, v, kf, out=None, workspace=None):
        self._check_sig(u, w, v)
        B, H, _ = u.shape
        y = torch.empty_like(u) if out is None else out
        ws = workspace if workspace is not None else self.workspace(B, H, device=u.device)
        _abi.check(_abi.lib().fftconv_gated_fwd(self._h, _ptr(u), _ptr(w), _ptr(v), _ptr(kf), _ptr(y), B, H,
                                                _ptr(ws), _stream(u.device)))
        return y

    def fwd_host(self, u: torch.Tensor, kf: torch.Tensor, w=None, v=None, out=None, rows_per_chunk: int = 8,
                 stage=None) -> torch.Tensor:
        """End-to-end forward from (pinned) host tensors through fftconv_fwd_host:
        batch rows are streamed through a device staging buffer with the
        copies of neighbouring chunks overlapping the convolution."""
        for t in (u, w, v):
            if t is not None:
                assert not t.is_cuda and t.dtype == self.dtype and t.is_contiguous() and t.dim() == 3
        B, H, N = u.shape
        assert N == self.info.N
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
        for t in (u, w, v):
            if t is not None:
                assert not t.is_cuda and t.dtype == self.dtype and t.is_contiguous() and t.dim() == 3
        B, H, NT = u.shape
        out = torch.empty_like(u, pin_memory=u.is_pinned()) if out is None else out
        n = ctypes.c_size_t()
        _abi.check(_abi.lib().fftconv_stream_stage_size(self._h, B, H, int(w is not None), ctypes.byref(n)))
        if stage is None or stage.numel() < n.value:
            stage = _aligned_empty(int(n.value), kf.device, 1024)
        _abi.check(_abi.lib().fftconv_fwd_stream(self._h, _ptr(u), _ptr(w), _ptr(v), _ptr(kf), _ptr(out), B, H, NT,
                                                 _ptr(stage), stage.numel(), _stream(kf.device)))
        self._stage = stage
        return out

    def host_stage(self, H: int, rows_per_chunk: int = 8, gated: bool = False, device=None):
        n = ctypes.c_size_t()
        _abi.check(_abi.lib().fftconv_host_stage_size(self._h, H, rows_per_chunk, int(gated), ctypes.byref(n)))
        return _aligned_empty(int(n.value), device or self.device, 1024)

    def bwd(self, dy, u, kf, K, w=None, v=None):
        """Gradients of <y, dy>: returns du, dw, dv (None when ungated) and dk (H, K)."""
        self._check_sig(dy, u)
        B, H, _ = u.shape
        du = torch.empty_like(u)
        dw = torch.empty_like(u) if w is not None else None
        dv = torch.empty_like(u) if v is not None else None
        dk = torch.empty(H, K, dtype=torch.float32, device=u.device)
        ws = self.workspace(B, H, for_bwd=True, device=u.device)
        _abi.check(_abi.lib().fftconv_bwd(self._h, _ptr(dy), _ptr(u), _ptr(w), _ptr(v), _ptr(kf), _ptr(du),
                                          _ptr(dw), _ptr(dv), _ptr(dk), B, H, K, _ptr(ws), _stream(u.device)))
        return {"du": du, "dw": dw, "dv": dv, "dk": dk}


def launch_count_reset() -> int:
    return int(_abi.lib().fftconv_launch_count_reset())

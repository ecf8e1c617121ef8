"""Thin Python binding over libtilt's C ABI (include/tilt.h).

PyTorch is used only for device memory and streams: every tensor is handed to the library as a raw
device pointer, and every step of the method runs in the CUDA kernels of ``csrc/``. Nothing here
computes any part of the method.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _abi
from ._abi import lib, check, default_params, TiltParams, TiltCreateOpts

REPORT_DTYPE = np.dtype([(name, np.float32 if ctype is ctypes.c_float else np.int32)
                         for name, ctype in _abi.TiltReport._fields_])
assert REPORT_DTYPE.itemsize == _abi.REPORT_BYTES


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _dev(x, dtype, device):
    if x is None:
        return None
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device=device)


def p_of(kind: int) -> int:
    return 8 if kind == _abi.HOMOGRAPHY else 6


def reports_to_numpy(rep_bytes: torch.Tensor) -> np.ndarray:
    return np.frombuffer(rep_bytes.cpu().numpy().tobytes(), dtype=REPORT_DTYPE)


class TiltSolver:
    """One libtilt handle on one CUDA device (not thread-safe, like the handle)."""

    def __init__(self, device: int = 0, max_batch: int = 1024, max_m: int = 64, max_n: int = 64,
                 max_p: int = 8, max_image_elems: int = 0):
        self.device = torch.device("cuda", device)
        self.max_batch, self.max_m, self.max_n, self.max_p = max_batch, max_m, max_n, max_p
        opts = TiltCreateOpts(device=device, stream=None, max_batch=max_batch, max_m=max_m, max_n=max_n,
                              max_p=max_p, max_image_elems=max_image_elems)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(lib.tilt_create(ctypes.byref(h), ctypes.byref(opts)), "tilt_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib.tilt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _bind_stream(self):
        s = torch.cuda.current_stream(self.device).cuda_stream
        check(lib.tilt_set_stream(self._h, ctypes.c_void_p(s)), "tilt_set_stream")

    @property
    def launches(self) -> int:
        return int(lib.tilt_launch_count(self._h))

    # ---- the hot entry ------------------------------------------------------------------------
    def solve(self, images, patch_image, boxes, tau0, kind: int, params: TiltParams | None = None,
              want_A: bool = True, want_E: bool = True, want_Y: bool = False, out: dict | None = None,
              sync: bool = True):
        """Batched Algorithm 1 (tilt_solve_batch). Inputs may be numpy arrays or CUDA tensors."""
        dev = self.device
        images = _dev(images, torch.float32, dev)
        patch_image = _dev(patch_image, torch.int32, dev)
        boxes_t = _dev(boxes, torch.int32, dev)
        B = int(boxes_t.shape[0])
        p = p_of(kind)
        tau0_t = _dev(tau0, torch.float32, dev)
        # a private copy: the caller's params object is never written (a reused object must not
        # carry one call's window size into the next)
        prm = TiltParams.from_buffer_copy(params) if params is not None else default_params()
        if prm.win_h <= 0 or prm.win_w <= 0:
            bx = np.asarray(boxes.cpu() if isinstance(boxes, torch.Tensor) else boxes)
            if B > 0:
                prm.win_h, prm.win_w = int(bx[0, 3]), int(bx[0, 2])
        m, n = int(prm.win_h), int(prm.win_w)
        if out is None:
            out = {
                "tau": torch.empty((B, p), dtype=torch.float32, device=dev),
                "A": torch.empty((B, m, n), dtype=torch.float32, device=dev) if want_A else None,
                "E": torch.empty((B, m, n), dtype=torch.float32, device=dev) if want_E else None,
                "Y": torch.empty((B, m, n), dtype=torch.float32, device=dev) if want_Y else None,
                "rep": torch.empty((B, _abi.REPORT_BYTES), dtype=torch.uint8, device=dev),
            }
        n_images, H, W = images.shape
        self._bind_stream()
        check(lib.tilt_solve_batch(self._h, _ptr(images), n_images, H, W, _ptr(patch_image), _ptr(boxes_t),
                                   _ptr(tau0_t), B, kind, ctypes.byref(prm), _ptr(out["tau"]), _ptr(out["A"]),
                                   _ptr(out["E"]), _ptr(out["Y"]), _ptr(out["rep"])), "tilt_solve_batch")
        if sync:
            torch.cuda.synchronize(dev)
        return out

    def solve_host(self, images: np.ndarray, patch_image, boxes, tau0, kind: int,
                   params: TiltParams | None = None, want_A: bool = True, want_E: bool = True):
        """End-to-end entry with host buffers (tilt_solve_batch_host): copies in, solves, copies out."""
        images = np.ascontiguousarray(images, dtype=np.float32)
        patch_image = np.ascontiguousarray(patch_image, dtype=np.int32)
        boxes = np.ascontiguousarray(boxes, dtype=np.int32)
        B = boxes.shape[0]
        p = p_of(kind)
        m, n = int(boxes[0, 3]), int(boxes[0, 2])
        tau0 = None if tau0 is None else np.ascontiguousarray(tau0, dtype=np.float32)
        tau = np.empty((B, p), np.float32)
        A = np.empty((B, m, n), np.float32) if want_A else None
        E = np.empty((B, m, n), np.float32) if want_E else None
        rep = np.empty(B, REPORT_DTYPE)
        prm = params if params is not None else default_params()
        n_images, H, W = images.shape
        self._bind_stream()

        def hp(a):
            return None if a is None else a.ctypes.data_as(ctypes.c_void_p)
        check(lib.tilt_solve_batch_host(self._h, hp(images), n_images, H, W, hp(patch_image), hp(boxes), hp(tau0),
                                        B, kind, ctypes.byref(prm), hp(tau), hp(A), hp(E), hp(rep)),
              "tilt_solve_batch_host")
        return {"tau": tau, "A": A, "E": E, "rep": rep}

    # ---- step-level entries ---------------------------------------------------------------------
    def warp(self, images, patch_image, boxes, tau, kind: int, want_J: bool = True):
        dev = self.device
        images = _dev(images, torch.float32, dev)
        patch_image = _dev(patch_image, torch.int32, dev)
        boxes_t = _dev(boxes, torch.int32, dev)
        tau_t = _dev(tau, torch.float32, dev)
        B = int(boxes_t.shape[0])
        bx = boxes_t[0].cpu().numpy()
        m, n = int(bx[3]), int(bx[2])
        p = p_of(kind)
        dh = torch.empty((B, m, n), dtype=torch.float32, device=dev)
        J = torch.empty((B, p, m, n), dtype=torch.float32, device=dev) if want_J else None
        nrm = torch.empty(B, dtype=torch.float32, device=dev)
        st = torch.empty(B, dtype=torch.int32, device=dev)
        n_images, H, W = images.shape
        self._bind_stream()
        check(lib.tilt_warp_batch(self._h, _ptr(images), n_images, H, W, _ptr(patch_image), _ptr(boxes_t),
                                  _ptr(tau_t), B, kind, m, n, _ptr(dh), _ptr(J), _ptr(nrm), _ptr(st)), "tilt_warp_batch")
        torch.cuda.synchronize(dev)
        return {"Dhat": dh, "J": J, "norm": nrm, "status": st}

    def svt(self, M, eps, V=None, path: int = 0):
        """tilt_svt_batch; path 0 = auto (CTA kernel up to 256 x 256, else multi-CTA), 1 = CTA kernel,
        3 = multi-CTA block-Jacobi path (any m, n <= 1024); 2 (warp-per-patch) is retired."""
        dev = self.device
        check(lib.tilt_set_svt_path(self._h, path), "tilt_set_svt_path")
        M = _dev(M, torch.float32, dev)
        B, m, n = M.shape
        eps_t = _dev(np.broadcast_to(np.asarray(eps, np.float32), (B,)).copy(), torch.float32, dev)
        V_t = _dev(V, torch.float32, dev) if V is not None else torch.empty((B, n, n), dtype=torch.float32, device=dev)
        if V is None:
            V_t.copy_(torch.eye(n, device=dev).expand(B, n, n))
        A = torch.empty((B, m, n), dtype=torch.float32, device=dev)
        sig = torch.empty((B, n), dtype=torch.float32, device=dev)
        sw = torch.empty(B, dtype=torch.int32, device=dev)
        self._bind_stream()
        check(lib.tilt_svt_batch(self._h, _ptr(M), B, m, n, _ptr(eps_t), _ptr(V_t), _ptr(A), _ptr(sig), _ptr(sw)),
              "tilt_svt_batch")
        torch.cuda.synchronize(dev)
        return {"A": A, "sigma": sig, "V": V_t, "sweeps": sw}

    def project(self, J, v, Q=None):
        dev = self.device
        J = _dev(J, torch.float32, dev)
        v = _dev(v, torch.float32, dev)
        B, p, m, n = J.shape
        Q_t = _dev(Q, torch.float32, dev)
        l = 0 if Q is None else int(Q_t.shape[1])
        Pv = torch.empty((B, m, n), dtype=torch.float32, device=dev)
        dt = torch.empty((B, p), dtype=torch.float32, device=dev)
        st = torch.empty(B, dtype=torch.int32, device=dev)
        self._bind_stream()
        check(lib.tilt_project_batch(self._h, _ptr(J), _ptr(Q_t), l, _ptr(v), B, m, n, p, _ptr(Pv), _ptr(dt), _ptr(st)),
              "tilt_project_batch")
        torch.cuda.synchronize(dev)
        return {"Pv": Pv, "dtau": dt, "status": st}

    def inner(self, D, J, Q=None, params: TiltParams | None = None, rho_replay=None, trace: bool = False):
        dev = self.device
        D = _dev(D, torch.float32, dev)
        J = _dev(J, torch.float32, dev)
        B, p, m, n = J.shape
        Q_t = _dev(Q, torch.float32, dev)
        l = 0 if Q is None else int(Q_t.shape[1])
        prm = TiltParams.from_buffer_copy(params) if params is not None else default_params()
        rr = None
        tr = None
        if rho_replay is not None:
            rr = _dev(np.asarray(rho_replay, np.uint8).reshape(B, prm.max_inner), torch.uint8, dev)
            prm.rho_replay = rr.data_ptr()
        if trace:
            tr = torch.full((B, prm.max_inner, 4), float("nan"), dtype=torch.float32, device=dev)
            prm.trace = tr.data_ptr()
        A = torch.empty((B, m, n), dtype=torch.float32, device=dev)
        E = torch.empty((B, m, n), dtype=torch.float32, device=dev)
        Y = torch.empty((B, m, n), dtype=torch.float32, device=dev)
        rep = torch.empty((B, _abi.REPORT_BYTES), dtype=torch.uint8, device=dev)
        self._bind_stream()
        check(lib.tilt_inner_batch(self._h, _ptr(D), _ptr(J), _ptr(Q_t), l, B, m, n, p, ctypes.byref(prm), _ptr(A),
                                   _ptr(E), _ptr(Y), _ptr(rep)), "tilt_inner_batch")
        torch.cuda.synchronize(dev)
        return {"A": A, "E": E, "Y": Y, "rep": reports_to_numpy(rep), "trace": tr}

"""B200-native MHFD hot path (arXiv 2108.12050): Python binding of ``libmhfd.so``.

The binding only marshals arguments: every step of the path (percentiles,
stretch, blur, DoG, NMS, compaction, pruning, score) runs in the CUDA kernels
behind the C ABI of ``include/mhfd.h``.  PyTorch provides device memory,
streams and (in ``dist``) the NCCL process group.  There is no CPU fallback:
without a CUDA device the context cannot be created and the calls raise.
"""
from __future__ import annotations

import ctypes

import torch

from . import _abi
from ._abi import MHFDError, mhfd_blob, mhfd_params  # noqa: F401

__all__ = ["Detector", "MHFDError", "BLOB_FIELDS", "downsample"]

BLOB_FIELDS = ("x", "y", "scale", "response")


def _params(**kw) -> mhfd_params:
    p = mhfd_params()
    _abi.load().mhfd_params_default(ctypes.byref(p))
    for k, v in kw.items():
        if v is not None:
            setattr(p, k, v)
    return p


class Detector:
    """One MHFD context (fixed image shape and parameters) on one CUDA device.

    Parameters follow Algorithm 1's ``Require I, n, min_t, max_t``
    plus the north star's threshold and overlap.  ``threshold=None`` means
    0.1 * dt (reading R11).
    """

    def __init__(self, width: int, height: int, min_sigma: float = 1.0, max_sigma: float = 10.0,
                 num_scales: int = 10, threshold: float | None = None, overlap: float = 0.5,
                 sat_low: float = 0.00175, sat_high: float = 0.00175, nms: str = "paper",
                 strict: bool = False, device: int | None = None, max_candidates: int = 0,
                 schedule: str | None = None, polarity: str = "dark", response: str = "dog",
                 boundary: str = "periodic"):
        """schedule: None / "auto" (library default: the tcgen05 schedules where they
        apply) or one of "tc", "band", "generic" — the params.schedule field of
        mhfd_create (no process-wide state is touched).  polarity: "dark" (Eq. 2 as written, the paper's EM
        sections) or "bright" (negated DoG: bright blobs on a dark background).  response:
        "dog" (Eq. 2, the paper's detector) or "log" (the scale-normalised Laplacian
        t_i^2 lap L(t_i) that Eq. 2 approximates; reading R23).  boundary:
        "periodic" (the paper's FFT) or "reflect" (mirrored edges; reading R25)."""
        lib = _abi.load()
        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        if threshold is None:
            threshold = 0.1 * (max_sigma - min_sigma) / num_scales
        self.params = _params(width=int(width), height=int(height), min_sigma=float(min_sigma),
                              max_sigma=float(max_sigma), num_scales=int(num_scales), threshold=float(threshold),
                              overlap=float(overlap), sat_low=float(sat_low), sat_high=float(sat_high),
                              nms={"paper": _abi.MHFD_NMS_PAPER, "26": _abi.MHFD_NMS_26}[str(nms)],
                              strict=int(bool(strict)), device=int(device), max_candidates=int(max_candidates),
                              polarity={"dark": _abi.MHFD_DARK, "bright": _abi.MHFD_BRIGHT}[str(polarity)],
                              response={"dog": _abi.MHFD_RESPONSE_DOG, "log": _abi.MHFD_RESPONSE_LOG}[str(response)],
                              boundary={"periodic": _abi.MHFD_BOUNDARY_PERIODIC,
                                        "reflect": _abi.MHFD_BOUNDARY_REFLECT}[str(boundary)])
        if schedule not in _abi.MHFD_SCHEDULE:
            raise ValueError(f"unknown schedule {schedule!r}")
        self.params.schedule = _abi.MHFD_SCHEDULE[schedule]
        h = ctypes.c_void_p()
        _abi.check(lib.mhfd_create(ctypes.byref(self.params), ctypes.byref(h)))
        self._h = h
        self._lib = lib
        got = mhfd_params()
        _abi.check(lib.mhfd_get_params(self._h, ctypes.byref(got)))
        self.max_candidates = int(got.max_candidates)
        self.width, self.height, self.n = int(width), int(height), int(num_scales)
        self.device = torch.device("cuda", int(device))
        self._ws = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.mhfd_destroy(h)
            self._h = None

    # -------------------------------------------------------------- helpers
    def workspace_bytes(self, batch: int) -> int:
        n = ctypes.c_size_t()
        _abi.check(self._lib.mhfd_workspace_bytes(self._h, int(batch), ctypes.byref(n)))
        return int(n.value)

    def _workspace(self, batch: int) -> torch.Tensor:
        need = self.workspace_bytes(batch)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need + 256, dtype=torch.uint8, device=self.device)
        return self._ws

    @staticmethod
    def _ws_ptr(ws: torch.Tensor) -> int:
        p = ws.data_ptr()
        return (p + 255) & ~255

    def prepare(self, images: torch.Tensor) -> tuple[torch.Tensor, int, int, int]:
        """(B,H,W) or (H,W) uint8/uint16/float32 tensor -> device tensor with a 16-byte-multiple pitch."""
        if images.dim() == 2:
            images = images.unsqueeze(0)
        if images.dim() != 3 or images.shape[1] != self.height or images.shape[2] != self.width:
            raise ValueError(f"images must be (B, {self.height}, {self.width}); got {tuple(images.shape)}")
        if images.dtype == torch.uint8:
            dt, bpp = _abi.MHFD_U8, 1
        elif images.dtype == torch.uint16:
            dt, bpp = _abi.MHFD_U16, 2
        elif images.dtype == torch.float32:
            dt, bpp = _abi.MHFD_F32, 4
        else:
            raise TypeError("images must be torch.uint8, torch.uint16 or torch.float32")
        images = images.to(self.device, non_blocking=True)
        B = images.shape[0]
        wp = (self.width * bpp + 15) // 16 * 16 // bpp
        if wp != self.width or not images.is_contiguous() or images.data_ptr() % 16:
            padded = torch.zeros((B, self.height, wp), dtype=images.dtype, device=self.device)
            padded[:, :, :self.width] = images
            images = padded
        return images, dt, B, wp * bpp

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    # -------------------------------------------------------------- entry points
    def focus_score(self, images: torch.Tensor, counts: bool = False):
        """DOF = |C| per image as a float64 device tensor."""
        imgs, dt, B, pitch = self.prepare(images)
        ws = self._workspace(B)
        scores = torch.empty(B, dtype=torch.float64, device=self.device)
        cnt = torch.empty(B, dtype=torch.int32, device=self.device)
        _abi.check(self._lib.mhfd_focus_score(self._h, imgs.data_ptr(), dt, B, pitch, self._ws_ptr(ws),
                                              ws.numel() - 256, scores.data_ptr(), cnt.data_ptr(), self._stream()))
        return (scores, cnt) if counts else scores

    def detect(self, images: torch.Tensor, blob_capacity: int | None = None):
        """Kept blobs per image: (blobs int32/float view (B, cap, 4), counts (B,), flags (B,))."""
        imgs, dt, B, pitch = self.prepare(images)
        ws = self._workspace(B)
        cap = self.max_candidates if blob_capacity is None else int(blob_capacity)
        blobs = torch.empty((B, max(cap, 1), 4), dtype=torch.int32, device=self.device)
        cnt = torch.empty(B, dtype=torch.int32, device=self.device)
        flags = torch.empty(B, dtype=torch.int32, device=self.device)
        _abi.check(self._lib.mhfd_detect_batch(self._h, imgs.data_ptr(), dt, B, pitch, self._ws_ptr(ws),
                                               ws.numel() - 256, blobs.data_ptr(), cap, cnt.data_ptr(),
                                               flags.data_ptr(), self._stream()))
        return blobs, cnt, flags

    def debug_dump(self, images: torch.Tensor, dog: bool = True, cands: bool = True) -> dict:
        """Intermediates for parity tests: lo/hi, DoG planes, v, argmax, candidates."""
        imgs, dt, B, pitch = self.prepare(images)
        ws = self._workspace(B)
        H, W, n = self.height, self.width, self.n
        out = {"lohi": torch.empty((B, 2), dtype=torch.int32, device=self.device),
               "ncand": torch.empty(B, dtype=torch.int32, device=self.device)}
        out["dog"] = torch.empty((B, n, H, W), dtype=torch.float32, device=self.device) if dog else None
        paper = self.params.nms == _abi.MHFD_NMS_PAPER
        out["v"] = torch.empty((B, H, W), dtype=torch.float32, device=self.device) if paper else None
        out["idx"] = torch.empty((B, H, W), dtype=torch.uint8, device=self.device) if paper else None
        out["cands"] = torch.empty((B, self.max_candidates, 4), dtype=torch.int32, device=self.device) if cands else None
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        _abi.check(self._lib.mhfd_debug_dump(self._h, imgs.data_ptr(), dt, B, pitch, self._ws_ptr(ws),
                                             ws.numel() - 256, ptr(out["lohi"]), ptr(out["dog"]), ptr(out["v"]),
                                             ptr(out["idx"]), ptr(out["cands"]), ptr(out["ncand"]), self._stream()))
        return out

    def focus_score_host(self, host_images: torch.Tensor, chunk: int = 8, counts: bool = False, out=None):
        """End-to-end call with HOST buffers (mhfd_focus_score_host): chunked H2D copies
        from (pinned) host memory overlapped with compute; returns host float64 scores.
        Back-to-back calls pipeline (the next call's copies overlap this call's last
        chunks).  The results are views of this detector's pinned buffers, valid after the
        current stream is synchronised and until the next call (copy them to keep them),
        or the caller's pinned (scores float64, counts int32) tensors given as ``out``."""
        if host_images.dim() == 2:
            host_images = host_images.unsqueeze(0)
        if host_images.device.type != "cpu":
            raise ValueError("focus_score_host takes host tensors")
        dt, bpp = {torch.uint8: (_abi.MHFD_U8, 1), torch.uint16: (_abi.MHFD_U16, 2),
                   torch.float32: (_abi.MHFD_F32, 4)}[host_images.dtype]
        B, H, W = host_images.shape
        if (H, W) != (self.height, self.width) or (W * bpp) % 16 or not host_images.is_contiguous():
            raise ValueError("host images must be contiguous (B, H, W) with W*bytes % 16 == 0")
        pitch = W * bpp
        chunk = max(1, min(int(chunk), B))
        need_stage = 3 * chunk * H * pitch   # three staging slots (kStageSlots)
        if getattr(self, "_stage", None) is None or self._stage.numel() < need_stage + 256:
            self._stage = torch.empty(need_stage + 256, dtype=torch.uint8, device=self.device)
        ws = self._workspace(chunk)
        if out is not None:
            hs, hc = out
            if (hs.dtype != torch.float64 or hc.dtype != torch.int32 or hs.numel() < B or hc.numel() < B
                    or hs.device.type != "cpu" or hc.device.type != "cpu"):
                raise ValueError("out must be host (float64, int32) tensors of >= batch elements")
        else:
            if getattr(self, "_hs", None) is None or self._hs.numel() < B:
                self._hs = torch.empty(B, dtype=torch.float64).pin_memory()
                self._hc = torch.empty(B, dtype=torch.int32).pin_memory()
            hs, hc = self._hs, self._hc
        _abi.check(self._lib.mhfd_focus_score_host(self._h, host_images.data_ptr(), dt, B, pitch,
                                                   self._ws_ptr(self._stage), need_stage, self._ws_ptr(ws),
                                                   ws.numel() - 256, hs.data_ptr(), hc.data_ptr(),
                                                   self._stream()))
        return (hs[:B], hc[:B]) if counts else hs[:B]

    # -------------------------------------------------- single-image sharding (f2)
    def detect_band(self, image: torch.Tensor, y0: int, y1: int, capacity: int | None = None):
        """Candidates of rows [y0, y1) of ONE image (mhfd_detect_band): (cands (cap, 4)
        int32 records in (y, x) order, exact count as a 1-element int32 device tensor)."""
        imgs, dt, B, pitch = self.prepare(image)
        if B != 1:
            raise ValueError("detect_band takes one image")
        ws = self._workspace(1)
        cap = self.max_candidates if capacity is None else int(capacity)
        cands = torch.empty((max(cap, 1), 4), dtype=torch.int32, device=self.device)
        n = torch.empty(1, dtype=torch.int32, device=self.device)
        _abi.check(self._lib.mhfd_detect_band(self._h, imgs.data_ptr(), dt, pitch, int(y0), int(y1),
                                              self._ws_ptr(ws), ws.numel() - 256, cands.data_ptr(), cap,
                                              n.data_ptr(), self._stream()))
        return cands, n

    def prune_candidates(self, cands: torch.Tensor, ncand: int, blob_capacity: int | None = None):
        """Pruning + score of one image's full raster-ordered candidate list
        (mhfd_prune_candidates): (blobs (cap, 4), count (1,), score (1,) float64, flags (1,))."""
        ws = self._workspace(1)
        cap = self.max_candidates if blob_capacity is None else int(blob_capacity)
        cands = cands.contiguous()
        blobs = torch.empty((max(cap, 1), 4), dtype=torch.int32, device=self.device)
        cnt = torch.empty(1, dtype=torch.int32, device=self.device)
        score = torch.empty(1, dtype=torch.float64, device=self.device)
        flags = torch.empty(1, dtype=torch.int32, device=self.device)
        _abi.check(self._lib.mhfd_prune_candidates(self._h, cands.data_ptr() if ncand > 0 else None, int(ncand),
                                                   self._ws_ptr(ws), ws.numel() - 256, blobs.data_ptr(), cap,
                                                   cnt.data_ptr(), score.data_ptr(), flags.data_ptr(),
                                                   self._stream()))
        return blobs, cnt, score, flags

    def interaction_radius(self) -> int:
        """Largest pruning search radius D in pixels (mhfd_interaction_radius)."""
        return int(self._lib.mhfd_interaction_radius(self._h))

    def prune_band(self, cands: torch.Tensor, ncand: int, e0: int, e1: int, y0: int, y1: int):
        """Sharded pruning of one band (mhfd_prune_band): the candidates of rows [e0, e1)
        (raster order) pruned in synchronous rounds -> 1-element int32 device tensors:
        kept blobs with y in [y0, y1); certificate (1 = provably the whole image's count for
        the band); candidates with y in [y0, y1)."""
        ws = self._workspace(1)
        cands = cands.contiguous()
        cnt = torch.empty(1, dtype=torch.int32, device=self.device)
        cert = torch.empty(1, dtype=torch.int32, device=self.device)
        nband = torch.empty(1, dtype=torch.int32, device=self.device)
        _abi.check(self._lib.mhfd_prune_band(self._h, cands.data_ptr() if ncand > 0 else None, int(ncand), int(e0),
                                             int(e1), int(y0), int(y1), self._ws_ptr(ws), ws.numel() - 256,
                                             cnt.data_ptr(), cert.data_ptr(), nband.data_ptr(), self._stream()))
        return cnt, cert, nband

    def timing_enable(self, max_calls: int) -> None:
        _abi.check(self._lib.mhfd_timing_enable(self._h, int(max_calls)))

    def timing_read(self) -> list[list[float]]:
        """Per recorded call: [percentiles, scale_space, nms, prune] device ms."""
        cap = 4 * 100000
        buf = (ctypes.c_float * cap)()
        n = ctypes.c_int32()
        _abi.check(self._lib.mhfd_timing_read(self._h, buf, ctypes.byref(n)))
        return [[buf[4 * k + j] for j in range(4)] for k in range(n.value)]

    def schedule(self, dtype: str = "u8") -> str:
        """Kernel that computes rows a2-a6 for `dtype` images (mhfd_schedule_name)."""
        code = {"u8": _abi.MHFD_U8, "u16": _abi.MHFD_U16, "f32": _abi.MHFD_F32}[dtype]
        return self._lib.mhfd_schedule_name(self._h, code).decode()

    def schedule_flops_per_pixel(self, dtype: str = "u8") -> float:
        """Flops per pixel the schedule's a2-a6 kernel executes (bench roofline)."""
        code = {"u8": _abi.MHFD_U8, "u16": _abi.MHFD_U16, "f32": _abi.MHFD_F32}[dtype]
        return float(self._lib.mhfd_schedule_flops_per_pixel(self._h, code))

    @staticmethod
    def last_launch_count() -> int:
        return int(_abi.load().mhfd_last_launch_count())


def blob_rows(blobs: torch.Tensor, count: int) -> list[tuple[int, int, int, float]]:
    """(x, y, scale, response) tuples from one image's (cap, 4) int32 blob block."""
    b = blobs[:count].cpu()
    resp = b[:, 3].view(torch.float32) if b.numel() else torch.empty(0)
    return [(int(x), int(y), int(s), float(r)) for (x, y, s), r in zip(b[:, :3].tolist(), resp.tolist())]


def downsample(images: torch.Tensor, factor: int) -> torch.Tensor:
    """Bilinear downsampling pre-step (mhfd_downsample):
    (B, H, W) or (H, W) uint8/uint16 CUDA tensor -> (B, ceil(H/f), ceil(W/f)) of the same
    dtype, half-pixel sample centres, exact value rounded half up (R22)."""
    if images.dim() == 2:
        images = images.unsqueeze(0)
    if images.dim() != 3 or images.device.type != "cuda":
        raise ValueError("images must be a (B, H, W) CUDA tensor")
    codes = {torch.uint8: (_abi.MHFD_U8, 1), torch.uint16: (_abi.MHFD_U16, 2)}
    if images.dtype not in codes:
        raise TypeError("images must be torch.uint8 or torch.uint16")
    dt, bpp = codes[images.dtype]
    images = images.contiguous()
    B, H, W = images.shape
    f = int(factor)
    out = torch.empty((B, -(-H // f) if f > 0 else 0, -(-W // f) if f > 0 else 0), dtype=images.dtype,
                      device=images.device)
    stream = torch.cuda.current_stream(images.device).cuda_stream
    _abi.check(_abi.load().mhfd_downsample(images.data_ptr(), dt, W, H, W * bpp, f, out.data_ptr(),
                                           out.shape[2] * bpp, B, stream))
    return out

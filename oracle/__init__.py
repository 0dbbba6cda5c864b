"""CPU oracle for the MHFD hot path (arXiv 2108.12050) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with ``paper_2108_12050_b200`` (the CUDA product path) and
never imports it.  The arithmetic lives in ``mhfd_oracle.c`` (plain C,
IEEE double, direct convolution, brute-force NMS, O(n^2) pruning); this
module only compiles it with gcc and marshals numpy arrays through ctypes.
Each wrapper names the paper passage its C function follows.

Parity status: every function below is pinned by a
``-m "not gpu"`` test in ``tests/test_oracle_pins.py`` except the *values*
of the threshold and overlap parameters, which the paper does not define
("parity unpinned" for those two parameter choices; their semantics are
pinned by closed forms).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mhfd_oracle.c")
_LIB = os.path.join(_HERE, "libmhfd_oracle.so")
_lock = threading.Lock()
_lib = None

BLOB_DTYPE = np.dtype([("x", np.int32), ("y", np.int32), ("scale", np.int32), ("pad", np.int32),
                       ("response", np.float64)])


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99", "-o", tmp, _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i32, i64, f64 = ctypes.c_int, ctypes.c_int64, ctypes.c_double
            sig = {
                "oracle_abi_version": (i32, []),
                "oracle_set_threads": (None, [i32]),
                "oracle_get_threads": (i32, []),
                "oracle_percentiles": (i32, [P, i32, i64, f64, f64, P, P]),
                "oracle_stretch": (None, [P, i32, i64, i64, i64, P]),
                "oracle_scale_grid": (None, [f64, f64, i32, P]),
                "oracle_radius": (i32, [f64]),
                "oracle_gaussian_2d": (f64, [f64, f64, f64]),
                "oracle_gaussian_taps": (None, [f64, i32, P]),
                "oracle_blur_rows": (None, [P, i32, i32, f64, i32, i32, P]),
                "oracle_blur": (None, [P, i32, i32, f64, P]),
                "oracle_dog_stack_rows": (None, [P, i32, i32, f64, f64, i32, i32, i32, P]),
                "oracle_dog_stack": (None, [P, i32, i32, f64, f64, i32, P]),
                "oracle_dog_at": (None, [P, i32, i32, f64, f64, i32, i32, i32, P]),
                "oracle_scale_argmax": (None, [P, i32, i64, P, P]),
                "oracle_nms_paper_v": (i64, [P, P, i32, i32, f64, i32, P, i64]),
                "oracle_nms_paper": (i64, [P, i32, i32, i32, f64, i32, P, i64]),
                "oracle_nms_26": (i64, [P, i32, i32, i32, f64, i32, P, i64]),
                "oracle_lens_fraction": (f64, [f64, f64, f64]),
                "oracle_prune": (i64, [P, i64, f64, f64, i32, f64, P]),
                "oracle_prune_grid": (i64, [P, i64, f64, f64, i32, f64, P]),
                "oracle_set_prune_grid": (None, [i32]),
                "oracle_detect": (i64, [P, i32, i32, i32, f64, f64, i32, f64, f64, f64, f64, i32, i32,
                                        P, i64, P, P, P, P, P, P]),
                "oracle_detect_pol": (i64, [P, i32, i32, i32, f64, f64, i32, f64, f64, f64, f64, i32, i32, i32,
                                            P, i64, P, P, P, P, P, P]),
                "oracle_downsample": (i32, [P, i32, i32, i32, i32, P]),
                "oracle_percentiles_f32": (i32, [P, i64, f64, f64, P, P]),
                "oracle_set_boundary": (None, [i32]),
                "oracle_get_boundary": (i32, []),
                "oracle_stretch_f32": (None, [P, i64, f64, f64, P]),
                "oracle_log_taps": (None, [f64, i32, P, P]),
                "oracle_log_stack_rows": (None, [P, i32, i32, f64, f64, i32, i32, i32, P]),
                "oracle_detect_resp": (i64, [P, i32, i32, i32, f64, f64, i32, f64, f64, f64, f64, i32, i32, i32,
                                             i32, P, i64, P, P, P, P, P, P]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class _boundary:
    """Set the oracle's blur boundary for one call ("periodic", reading R7, or "reflect",
    reading R25) and restore periodic afterwards."""

    def __init__(self, boundary: str):
        self.b = {"periodic": 0, "reflect": 1}[str(boundary)]

    def __enter__(self):
        _load().oracle_set_boundary(self.b)

    def __exit__(self, *exc):
        _load().oracle_set_boundary(0)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _img(img: np.ndarray):
    img = np.ascontiguousarray(img)
    if img.dtype == np.uint8:
        return img, 1
    if img.dtype == np.uint16:
        return img, 2
    if img.dtype == np.float32:
        return img, 4
    raise TypeError("oracle images are uint8, uint16 or float32")


def set_threads(n: int) -> None:
    _load().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(_load().oracle_get_threads())


def percentiles(img: np.ndarray, sat_low: float = 0.00175, sat_high: float = 0.00175):
    """Nearest-rank lo/hi of the histogram stretch: ints for
    u8/u16 images, floats for float32 images (reading R24)."""
    img, bpp = _img(img)
    if bpp == 4:
        flo, fhi = ctypes.c_double(), ctypes.c_double()
        if _load().oracle_percentiles_f32(_ptr(img), img.size, sat_low, sat_high, ctypes.byref(flo),
                                          ctypes.byref(fhi)) != 0:
            raise ValueError("oracle_percentiles_f32 failed")
        return float(flo.value), float(fhi.value)
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    rc = _load().oracle_percentiles(_ptr(img), bpp, img.size, sat_low, sat_high,
                                    ctypes.byref(lo), ctypes.byref(hi))
    if rc != 0:
        raise ValueError("oracle_percentiles failed")
    return int(lo.value), int(hi.value)


def stretch(img: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """I' = clamp((I - lo)/(hi - lo), 0, 1) in f64."""
    img, bpp = _img(img)
    out = np.empty(img.shape, np.float64)
    if bpp == 4:
        _load().oracle_stretch_f32(_ptr(img), img.size, float(lo), float(hi), _ptr(out))
    else:
        _load().oracle_stretch(_ptr(img), bpp, img.size, int(lo), int(hi), _ptr(out))
    return out


def scale_grid(min_t: float, max_t: float, n: int) -> np.ndarray:
    """t_i = min_t + (i-1)(max_t-min_t)/n, i = 1..n+1."""
    t = np.empty(n + 1, np.float64)
    _load().oracle_scale_grid(min_t, max_t, n, _ptr(t))
    return t


def radius(t: float) -> int:
    return int(_load().oracle_radius(t))


def gaussian_2d(x: float, y: float, sigma: float) -> float:
    """Unnormalised continuous G(x, y, sigma) of PAPER.md:136."""
    return float(_load().oracle_gaussian_2d(x, y, sigma))


def gaussian_taps(t: float, R: int | None = None) -> np.ndarray:
    """Sampled, renormalised 1-D Gaussian taps, |d| <= R (default ceil(6t))."""
    R = radius(t) if R is None else int(R)
    w = np.empty(2 * R + 1, np.float64)
    _load().oracle_gaussian_taps(t, R, _ptr(w))
    return w


def blur(f: np.ndarray, t: float, rows: tuple[int, int] | None = None, boundary: str = "periodic") -> np.ndarray:
    """Periodic L = G(t) * f, optionally only rows [y0, y1)."""
    f = np.ascontiguousarray(f, np.float64)
    H, W = f.shape
    y0, y1 = (0, H) if rows is None else rows
    out = np.empty((y1 - y0, W), np.float64)
    with _boundary(boundary):
        _load().oracle_blur_rows(_ptr(f), H, W, t, y0, y1, _ptr(out))
    return out


def dog_stack(f: np.ndarray, min_t: float, max_t: float, n: int,
              rows: tuple[int, int] | None = None, boundary: str = "periodic") -> np.ndarray:
    """Eq. 2 DoG planes D_i = t_i (L_{i+1} - L_i), i=1..n."""
    f = np.ascontiguousarray(f, np.float64)
    H, W = f.shape
    y0, y1 = (0, H) if rows is None else rows
    D = np.empty((n, y1 - y0, W), np.float64)
    with _boundary(boundary):
        _load().oracle_dog_stack_rows(_ptr(f), H, W, min_t, max_t, n, y0, y1, _ptr(D))
    return D


def log_taps(t: float, R: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """(w, w2): renormalised Gaussian taps and the zero-sum second-derivative taps
    w2(d) = w(d)(d^2 - m2)/t^4, m2 = sum w d^2 (reading R23)."""
    R = radius(t) if R is None else int(R)
    w = np.empty(2 * R + 1, np.float64)
    w2 = np.empty(2 * R + 1, np.float64)
    _load().oracle_log_taps(float(t), R, _ptr(w), _ptr(w2))
    return w, w2


def log_stack(f: np.ndarray, min_t: float, max_t: float, n: int,
              rows: tuple[int, int] | None = None, boundary: str = "periodic") -> np.ndarray:
    """Scale-normalised Laplacian planes t_i^2 (d_xx + d_yy) L(., t_i), i = 1..n
    (Eq. 1; reading R23)."""
    f = np.ascontiguousarray(f, np.float64)
    H, W = f.shape
    y0, y1 = (0, H) if rows is None else rows
    D = np.empty((n, y1 - y0, W), np.float64)
    with _boundary(boundary):
        _load().oracle_log_stack_rows(_ptr(f), H, W, min_t, max_t, n, y0, y1, _ptr(D))
    return D


def dog_at(f: np.ndarray, min_t: float, max_t: float, n: int, y: int, x: int,
           boundary: str = "periodic") -> np.ndarray:
    """Eq. 2 at one pixel from the 2-D definition (for sampled full-size checks)."""
    f = np.ascontiguousarray(f, np.float64)
    H, W = f.shape
    out = np.empty(n, np.float64)
    with _boundary(boundary):
        _load().oracle_dog_at(_ptr(f), H, W, min_t, max_t, n, int(y), int(x), _ptr(out))
    return out


def scale_argmax(D: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Inner argmax of Eq. 3 over all n planes, first maximum on ties."""
    D = np.ascontiguousarray(D, np.float64)
    n = D.shape[0]
    plane = int(np.prod(D.shape[1:]))
    v = np.empty(D.shape[1:], np.float64)
    idx = np.empty(D.shape[1:], np.int32)
    _load().oracle_scale_argmax(_ptr(D), n, plane, _ptr(v), _ptr(idx))
    return v, idx


def nms_paper(D: np.ndarray, tau: float, strict: bool = False) -> np.ndarray:
    """Eq. 3: argmaxlocal_{x,y} argmax_i DoG, maxpool(3,3) comparison."""
    D = np.ascontiguousarray(D, np.float64)
    n, H, W = D.shape
    out = np.empty(H * W, BLOB_DTYPE)
    c = _load().oracle_nms_paper(_ptr(D), n, H, W, tau, int(strict), _ptr(out), out.size)
    return out[:c].copy()


def nms_paper_v(v: np.ndarray, idx: np.ndarray, tau: float, strict: bool = False) -> np.ndarray:
    """Eq. 3's outer step on a given inner argmax (v, i^): the
    maxpool(3,3) comparison with -inf padding and the threshold."""
    v = np.ascontiguousarray(v, np.float64)
    idx = np.ascontiguousarray(idx, np.int32)
    H, W = v.shape
    cap = max(16, H * W // 2)
    while True:
        out = np.empty(cap, BLOB_DTYPE)
        c = _load().oracle_nms_paper_v(_ptr(v), _ptr(idx), H, W, tau, int(strict), _ptr(out), out.size)
        if c <= cap:
            return out[:c].copy()
        cap = int(c)


def nms_26(D: np.ndarray, tau: float, strict: bool = False) -> np.ndarray:
    """Conventional 3x3x3 scale-space maxima."""
    D = np.ascontiguousarray(D, np.float64)
    n, H, W = D.shape
    out = np.empty(n * H * W, BLOB_DTYPE)
    c = _load().oracle_nms_26(_ptr(D), n, H, W, tau, int(strict), _ptr(out), out.size)
    return out[:c].copy()


def lens_fraction(d: float, r1: float, r2: float) -> float:
    """Lens area of two disks / area of the smaller one (reading R12)."""
    return float(_load().oracle_lens_fraction(d, r1, r2))


def prune(blobs: np.ndarray, min_t: float, max_t: float, n: int, overlap: float,
          grid: bool = False) -> np.ndarray:
    """Greedy overlap pruning in priority (scale desc, raster asc); returns keep flags.
    grid=True runs oracle_prune_grid: the same decisions with an exact distance early-out
    (pairs farther apart than r1 + r2 have overlap fraction 0), for 10^5-blob lists."""
    blobs = np.ascontiguousarray(blobs, BLOB_DTYPE)
    keep = np.zeros(max(blobs.size, 1), np.uint8)
    fn = _load().oracle_prune_grid if grid else _load().oracle_prune
    fn(_ptr(blobs), blobs.size, min_t, max_t, n, overlap, _ptr(keep))
    return keep[:blobs.size].astype(bool)


def blobs_from_records(rec: np.ndarray) -> np.ndarray:
    """(k, 4) int32 records {x, y, scale, float32 response bits} (the C ABI's blob layout)
    -> the oracle's blob array, e.g. to prune the CUDA path's candidate list exactly."""
    rec = np.ascontiguousarray(rec, np.int32).reshape(-1, 4)
    out = np.zeros(rec.shape[0], BLOB_DTYPE)
    out["x"], out["y"], out["scale"] = rec[:, 0], rec[:, 1], rec[:, 2]
    out["response"] = rec[:, 3].view(np.float32).astype(np.float64)
    return out


def detect(img: np.ndarray, min_t: float, max_t: float, n: int, tau: float, overlap: float,
           sat_low: float = 0.00175, sat_high: float = 0.00175, nms: str = "paper",
           strict: bool = False, dump: bool = False, polarity: str = "dark", response: str = "dog",
           boundary: str = "periodic", grid_prune: bool = False) -> dict:
    """Algorithm 1 + threshold + pruning; returns blobs, count, candidates.
    polarity "bright" negates the response (not in the paper); response
    "log" replaces Eq. 2 by the scale-normalised Laplacian t_i^2 lap L(t_i) (reading R23);
    boundary "reflect" mirrors the image at its edges for the blur (reading R25).
    grid_prune selects oracle_prune_grid (identical decisions, for full-size images)."""
    img, bpp = _img(img)
    H, W = img.shape
    mode = {"paper": 0, "26": 1}[str(nms)]
    cap = H * W * (1 if mode == 0 else n)
    out = np.empty(cap, BLOB_DTYPE)
    ncand = ctypes.c_int64()
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    D = np.empty((n, H, W), np.float64) if dump else None
    v = np.empty((H, W), np.float64) if (dump and mode == 0) else None
    idx = np.empty((H, W), np.int32) if (dump and mode == 0) else None
    pol = {"dark": 0, "bright": 1}[str(polarity)]
    resp = {"dog": 0, "log": 1}[str(response)]
    _load().oracle_set_prune_grid(int(bool(grid_prune)))
    try:
        with _boundary(boundary):
            k = _load().oracle_detect_resp(_ptr(img), bpp, H, W, min_t, max_t, n, tau, overlap, sat_low, sat_high,
                                           mode, int(strict), pol, resp, _ptr(out), cap, ctypes.byref(ncand),
                                           _ptr(D), _ptr(v), _ptr(idx), ctypes.byref(lo), ctypes.byref(hi))
    finally:
        _load().oracle_set_prune_grid(0)
    if k < 0:
        raise MemoryError("oracle_detect failed")
    res = {"blobs": out[:k].copy(), "count": int(k), "n_candidates": int(ncand.value),
           "lo": int(lo.value), "hi": int(hi.value), "score": float(k)}
    if dump:
        res["D"] = D
        if mode == 0:
            res["v"], res["idx"] = v, idx
    return res


def downsample(img: np.ndarray, factor: int) -> np.ndarray:
    """Bilinear downsampling pre-step (reading R22): textbook
    bilinear in f64 at half-pixel sample centres, rounded half up; (H, W) u8/u16 ->
    (ceil(H/f), ceil(W/f)) of the same dtype."""
    img, bpp = _img(img)
    H, W = img.shape
    f = int(factor)
    if f < 1 or f > min(H, W):
        raise ValueError("factor must be in [1, min(H, W)]")
    out = np.empty((-(-H // f), -(-W // f)), img.dtype)
    if _load().oracle_downsample(_ptr(img), bpp, H, W, f, _ptr(out)) != 0:
        raise ValueError("oracle_downsample failed")
    return out

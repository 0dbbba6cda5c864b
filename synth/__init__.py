"""Seeded synthetic EM-like inputs for MHFD (shared by tests, bench and smoke).

This module holds NO arithmetic of the method (no histogram stretch, no
sampled/truncated Gaussian, no DoG, no NMS).  It only draws images shaped like
the paper's serial-section SEM tiles (BSE images of
40 nm sections; dark membranes, vesicles and organelles on a bright
background), so that the oracle (``oracle/``) and the CUDA path
(``paper_2108_12050_b200``) see the same bytes.

Recipe (after SURVEY.md §8(d)); all sizes in pixels:

* background 0.78;
* membranes: periodic Voronoi on a jittered grid of ~60 px cells, darkening
  0.45*exp(-(gap/2)^2) where gap = d2 - d1 (second minus first nearest seed);
* vesicles: one ring per ~30 px cell, radius U(3, 7), profile
  0.35*exp(-((rho - r)/1)^2);
* organelles: one filled disk per ~200 px cell, radius U(8, 20), depth 0.3,
  logistic edge of 0.7 px;
* clip to [0.02, 1];
* defocus: periodic Gaussian blur of standard deviation ``defocus`` applied as
  the continuous optical transfer function exp(-2 pi^2 s^2 |f|^2) in the
  Fourier domain (a physical model of the microscope, not the detector's
  sampled spatial kernel);
* shot noise: Poisson(dose*img)/dose (dose=None: noise-free);
* quantisation: round(img/1.2 * (2^bits - 1)) to uint8 / uint16.

Everything is periodic, so the detector's periodic boundary sees no seams.
Generation uses torch so the same code runs on CPU (tests) and on the GPU
(the bench's 64-image batches); a given device + seed is deterministic.
"""
from __future__ import annotations

import math

import numpy as np
import torch

BACKGROUND = 0.78


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _cells(n_px: int, size: float) -> int:
    return max(2, int(round(n_px / size)))


def _jitter(g, gy, gx, device):
    return torch.rand((gy, gx, 2), generator=g, device=device, dtype=torch.float64)


def _near(H, W, gy, gx, y0, y1, device):
    """Pixel coordinates of rows [y0, y1) and the 3x3 neighbouring cell offsets."""
    ch, cw = H / gy, W / gx
    ys = torch.arange(y0, y1, device=device, dtype=torch.float64) + 0.5
    xs = torch.arange(W, device=device, dtype=torch.float64) + 0.5
    Y, X = torch.meshgrid(ys, xs, indexing="ij")
    iy = torch.floor(Y / ch).long()
    ix = torch.floor(X / cw).long()
    return Y, X, iy, ix, ch, cw


def _seed_pos(jit, iy, ix, dy, dx, ch, cw, gy, gx):
    """Unwrapped position of the feature of cell (iy+dy, ix+dx) (periodic images)."""
    cy, cx = iy + dy, ix + dx
    j = jit[torch.remainder(cy, gy), torch.remainder(cx, gx)]
    return (cy.double() + j[..., 0]) * ch, (cx.double() + j[..., 1]) * cw


def em_tile(H: int, W: int, seed: int, defocus: float = 0.0, dose: float | None = 300.0,
            bits: int = 8, device="cpu", chunk_rows: int = 1024) -> torch.Tensor:
    """One synthetic EM tile, returned as a uint8 (bits=8) or int32 (bits=16) tensor."""
    device = torch.device(device)
    g = _gen(seed, device)
    gyM, gxM = _cells(H, 60.0), _cells(W, 60.0)
    gyV, gxV = _cells(H, 30.0), _cells(W, 30.0)
    gyO, gxO = _cells(H, 200.0), _cells(W, 200.0)
    jm = _jitter(g, gyM, gxM, device)
    jv = _jitter(g, gyV, gxV, device)
    rv = 3.0 + 4.0 * torch.rand((gyV, gxV), generator=g, device=device, dtype=torch.float64)
    jo = _jitter(g, gyO, gxO, device)
    ro = 8.0 + 12.0 * torch.rand((gyO, gxO), generator=g, device=device, dtype=torch.float64)
    img = torch.empty((H, W), dtype=torch.float64, device=device)
    for y0 in range(0, H, chunk_rows):
        y1 = min(H, y0 + chunk_rows)
        dark = torch.zeros((y1 - y0, W), dtype=torch.float64, device=device)
        # membranes: distance gap between the two nearest Voronoi seeds
        Y, X, iy, ix, ch, cw = _near(H, W, gyM, gxM, y0, y1, device)
        ds = []
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                py, px = _seed_pos(jm, iy, ix, dy, dx, ch, cw, gyM, gxM)
                ds.append(torch.hypot(Y - py, X - px))
        d = torch.stack(ds, 0)
        d2, _ = torch.topk(d, 2, dim=0, largest=False)
        gap = d2[1] - d2[0]
        dark += 0.45 * torch.exp(-(gap / 2.0) ** 2)
        del d, ds, d2, gap
        # vesicles: rings
        Y, X, iy, ix, ch, cw = _near(H, W, gyV, gxV, y0, y1, device)
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                py, px = _seed_pos(jv, iy, ix, dy, dx, ch, cw, gyV, gxV)
                r = rv[torch.remainder(iy + dy, gyV), torch.remainder(ix + dx, gxV)]
                rho = torch.hypot(Y - py, X - px)
                dark += 0.35 * torch.exp(-((rho - r) / 1.0) ** 2)
        # organelles: filled disks with a logistic edge
        Y, X, iy, ix, ch, cw = _near(H, W, gyO, gxO, y0, y1, device)
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                py, px = _seed_pos(jo, iy, ix, dy, dx, ch, cw, gyO, gxO)
                r = ro[torch.remainder(iy + dy, gyO), torch.remainder(ix + dx, gxO)]
                rho = torch.hypot(Y - py, X - px)
                dark += 0.3 * torch.sigmoid(-(rho - r) / 0.7)
        img[y0:y1] = torch.clamp(BACKGROUND - dark, 0.02, 1.0)
    if defocus and defocus > 0:
        img = _defocus(img, defocus)
    if dose is not None:
        img = torch.poisson(torch.clamp(img, min=0.0) * dose, generator=g) / dose
    return quantise(img, bits)


def _defocus(img: torch.Tensor, s: float) -> torch.Tensor:
    """Periodic optical defocus: multiply the spectrum by exp(-2 pi^2 s^2 |f|^2)."""
    H, W = img.shape
    fy = torch.fft.fftfreq(H, device=img.device, dtype=torch.float64)
    fx = torch.fft.rfftfreq(W, device=img.device, dtype=torch.float64)
    otf = torch.exp(-2.0 * math.pi ** 2 * s ** 2 * (fy[:, None] ** 2 + fx[None, :] ** 2))
    return torch.fft.irfft2(torch.fft.rfft2(img) * otf, s=(H, W))


def quantise(img: torch.Tensor, bits: int) -> torch.Tensor:
    top = float(2 ** bits - 1)
    q = torch.clamp(torch.round(img / 1.2 * top), 0, top)
    return q.to(torch.uint8) if bits == 8 else q.to(torch.int32)


def to_numpy(t: torch.Tensor, bits: int) -> np.ndarray:
    a = t.cpu().numpy()
    return a.astype(np.uint8 if bits == 8 else np.uint16)


def em_tile_np(H: int, W: int, seed: int, defocus: float = 0.0, dose: float | None = 300.0,
               bits: int = 8) -> np.ndarray:
    """CPU-generated tile as a numpy uint8/uint16 array."""
    return to_numpy(em_tile(H, W, seed, defocus, dose, bits, device="cpu"), bits)


# ---------------------------------------------------------------- fixtures
def disk_image(H: int, W: int, cy: float, cx: float, r: float, contrast: float = 0.6,
               bits: int = 16, ss: int = 16) -> np.ndarray:
    """Area-sampled dark disk of radius r on a bright background (quantised)."""
    return quantise(torch.from_numpy(disks_float(H, W, [(cy, cx, r)], contrast, ss)), bits).numpy().astype(
        np.uint8 if bits == 8 else np.uint16)


def disks_float(H: int, W: int, disks, contrast: float = 0.6, ss: int = 16) -> np.ndarray:
    """Float image (1 - contrast * covered area fraction) with area-sampled dark disks."""
    img = np.ones((H, W), np.float64)
    off = (np.arange(ss) + 0.5) / ss
    for (cy, cx, r) in disks:
        y0, y1 = int(math.floor(cy - r - 1)), int(math.ceil(cy + r + 1))
        x0, x1 = int(math.floor(cx - r - 1)), int(math.ceil(cx + r + 1))
        for y in range(y0, y1 + 1):
            for x in range(x0, x1 + 1):
                sy = y + off[:, None] - cy
                sx = x + off[None, :] - cx
                frac = float(np.mean(sy * sy + sx * sx <= r * r))
                if frac > 0:
                    img[y % H, x % W] -= contrast * frac
    return img


def gaussian_blob_float(H: int, W: int, cy: float, cx: float, s: float, A: float = 0.5) -> np.ndarray:
    """1 - A exp(-r^2 / 2 s^2): a dark Gaussian blob on a bright background (float)."""
    y = np.arange(H)[:, None] - cy
    x = np.arange(W)[None, :] - cx
    return 1.0 - A * np.exp(-(y * y + x * x) / (2.0 * s * s))


def constant_image(H: int, W: int, value: int = 117, bits: int = 8) -> np.ndarray:
    return np.full((H, W), value, np.uint8 if bits == 8 else np.uint16)


def random_stack(n: int, H: int, W: int, seed: int, levels: int = 4) -> np.ndarray:
    """Small-integer DoG-like stacks with deliberate ties (for brute-force NMS pins)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, levels, size=(n, H, W)).astype(np.float64)

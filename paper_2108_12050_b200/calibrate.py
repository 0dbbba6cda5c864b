"""Focus calibration on top of the focus score (host-side, not the
hot path).

The paper's validation: on a focal series with known in-focus depth
f', the number of detected features falls log-linearly with the absolute focal deviation
|f - f'| (fitted r = -0.9754; log-linear = roughly quadratic fall in count).  These
helpers fit that relation on a calibration series and turn a score into an estimated
deviation or an in/out-of-focus decision for a chosen deviation tolerance.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class LogLinearFit:
    """log(score) = intercept + slope * |defocus| (least squares), with Pearson r."""
    slope: float
    intercept: float
    r: float

    def predict(self, defocus) -> np.ndarray:
        """Expected score at the given focal deviation(s)."""
        return np.exp(self.intercept + self.slope * np.abs(np.asarray(defocus, np.float64)))

    def deviation(self, scores) -> np.ndarray:
        """Estimated |f - f'| of score(s) by inverting the fit (clipped at 0)."""
        s = np.asarray(scores, np.float64)
        if np.any(s <= 0):
            raise ValueError("scores must be positive")
        if self.slope >= 0:
            raise ValueError("the fit does not decrease with defocus")
        return np.maximum((np.log(s) - self.intercept) / self.slope, 0.0)

    def threshold(self, max_deviation: float) -> float:
        """Score at the largest tolerated deviation: at or above it the section is taken
        as in focus."""
        return float(self.predict(max_deviation))


def fit_log_linear(defocus, scores) -> LogLinearFit:
    """Least-squares line through (|defocus|, log(score))."""
    d = np.abs(np.asarray(defocus, np.float64)).ravel()
    s = np.asarray(scores, np.float64).ravel()
    if d.shape != s.shape or d.size < 2:
        raise ValueError("need matching defocus/score arrays with at least two points")
    if np.any(s <= 0):
        raise ValueError("scores must be positive for a log-linear fit")
    if np.ptp(d) == 0:
        raise ValueError("defocus values must not all be equal")
    y = np.log(s)
    dm, ym = d.mean(), y.mean()
    sxx = float(((d - dm) ** 2).sum())
    sxy = float(((d - dm) * (y - ym)).sum())
    syy = float(((y - ym) ** 2).sum())
    slope = sxy / sxx
    r = sxy / np.sqrt(sxx * syy) if syy > 0 else 0.0
    return LogLinearFit(slope=slope, intercept=float(ym - slope * dm), r=float(r))


def classify(scores, threshold: float) -> np.ndarray:
    """In focus (True) iff score >= threshold."""
    return np.asarray(scores, np.float64) >= float(threshold)

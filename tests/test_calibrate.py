"""Focus calibration helpers, on CPU; the GPU test with a synthetic
defocus sweep is in test_gpu_parity.py."""
import numpy as np
import pytest

from paper_2108_12050_b200.calibrate import classify, fit_log_linear


def test_exact_exponential_is_recovered():
    d = np.linspace(0, 4, 9)
    s = np.exp(9.0 - 0.8 * d)
    f = fit_log_linear(d, s)
    assert f.slope == pytest.approx(-0.8, abs=1e-12) and f.intercept == pytest.approx(9.0, abs=1e-12)
    assert f.r == pytest.approx(-1.0, abs=1e-12)
    np.testing.assert_allclose(f.predict(d), s, rtol=1e-12)
    np.testing.assert_allclose(f.deviation(s), d, atol=1e-10)


def test_sign_symmetry_and_threshold():
    d = np.array([-2.0, -1.0, 0.0, 1.0, 2.0])
    s = np.exp(5.0 - 0.5 * np.abs(d))
    f = fit_log_linear(d, s)          # |f - f'|: the sign of the deviation does not matter
    assert f.r == pytest.approx(-1.0)
    th = f.threshold(1.0)
    assert th == pytest.approx(np.exp(4.5))
    np.testing.assert_array_equal(classify(s, th), np.abs(d) <= 1.0)


def test_noisy_fit_r_matches_pearson():
    rng = np.random.default_rng(3)
    d = np.repeat(np.linspace(0, 4, 9), 3)
    s = np.exp(9.0 - 0.8 * d + rng.normal(0, 0.1, d.size))
    f = fit_log_linear(d, s)
    assert f.r == pytest.approx(np.corrcoef(d, np.log(s))[0, 1], abs=1e-12)
    assert np.polyfit(d, np.log(s), 1)[0] == pytest.approx(f.slope, abs=1e-12)


def test_rejects_bad_input():
    with pytest.raises(ValueError):
        fit_log_linear([0, 1], [1.0, 0.0])
    with pytest.raises(ValueError):
        fit_log_linear([1, 1], [1.0, 2.0])
    with pytest.raises(ValueError):
        fit_log_linear([0, 1, 2], [1.0, 2.0])

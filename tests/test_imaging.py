"""Image metrics: known answers + an independent direct-sum SSIM."""
import numpy as np
import pytest

from paper_2304_07338_b200.imaging import luminance, mse, rse, ssim


def _ssim_direct(x, y):
    """Independent SSIM: explicit 11x11 window loops (no separable filter)."""
    k, s = 11, 1.5
    ax = np.arange(k) - 5.0
    w2 = np.exp(-(ax[:, None] ** 2 + ax[None, :] ** 2) / (2 * s * s))
    w2 /= w2.sum()
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    vals = []
    for i in range(x.shape[0] - k + 1):
        for j in range(x.shape[1] - k + 1):
            px, py = x[i:i + k, j:j + k], y[i:i + k, j:j + k]
            mx, my = (w2 * px).sum(), (w2 * py).sum()
            vx, vy = (w2 * px * px).sum() - mx * mx, (w2 * py * py).sum() - my * my
            cxy = (w2 * px * py).sum() - mx * my
            vals.append(((2 * mx * my + c1) * (2 * cxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2)))
    return float(np.mean(vals))


def test_identity_and_symmetry():
    r = np.random.default_rng(0)
    a = r.random((24, 20, 3))
    b = np.clip(a + 0.05 * r.standard_normal(a.shape), 0, 1)
    assert mse(a, a) == 0.0 and ssim(a, a) == pytest.approx(1.0, abs=1e-12)
    assert abs(ssim(a, b) - ssim(b, a)) < 1e-9
    assert -1.0 <= ssim(a, b) < 1.0
    assert np.all(rse(a, a) == 0.0)


def test_ssim_matches_direct_window_sum():
    r = np.random.default_rng(1)
    a = r.random((16, 19))
    b = 0.7 * a + 0.2 * r.random((16, 19))
    assert ssim(a, b) == pytest.approx(_ssim_direct(a, b), rel=1e-10)


def test_luminance_and_rse_values():
    img = np.zeros((2, 2, 3))
    img[0, 0] = [1, 0, 0]
    assert luminance(img)[0, 0] == pytest.approx(0.2126)
    a = np.full((1, 1, 3), 0.2)
    b = np.full((1, 1, 3), 0.1)
    assert rse(a, b)[0, 0] == pytest.approx(0.01 / 0.02)
    with pytest.raises(ValueError):
        ssim(np.zeros((8, 8)), np.zeros((8, 8)))

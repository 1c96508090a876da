"""Image metrics of the SPEC's imaging module.

mse  = mean squared channel difference;
rse  = (a - b)^2 / (b^2 + 0.01) per pixel (relative square error, the paper's
       rSE with a stabiliser), on luminance;
ssim = single-scale SSIM on luminance, 11x11 Gaussian window (sigma 1.5),
       standard constants C1 = (0.01 L)^2, C2 = (0.03 L)^2 with L = 1 (linear
       radiance, no tone mapping: SPEC.md:602), 'valid' windows only.
Host-side numpy; used by the acceptance tests and the bench report.
"""
from __future__ import annotations

import numpy as np

_LUMA = np.array([0.2126, 0.7152, 0.0722])


def luminance(img: np.ndarray) -> np.ndarray:
    img = np.asarray(img, np.float64)
    return img @ _LUMA if img.ndim == 3 else img


def mse(a: np.ndarray, b: np.ndarray) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError("mse: shape mismatch")
    return float(np.mean((a - b) ** 2))


def rse(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    la, lb = luminance(a), luminance(b)
    return (la - lb) ** 2 / (lb ** 2 + 0.01)


def _gauss_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    x = np.arange(size) - (size - 1) / 2.0
    g = np.exp(-(x ** 2) / (2.0 * sigma * sigma))
    g /= g.sum()
    return g


def _filter_valid(img: np.ndarray, g: np.ndarray) -> np.ndarray:
    """Separable 'valid' correlation with the 1-D kernel g."""
    k = len(g)
    h, w = img.shape
    if h < k or w < k:
        raise ValueError("ssim: image smaller than the 11x11 window")
    rows = sum(g[i] * img[i:h - k + 1 + i, :] for i in range(k))
    return sum(g[j] * rows[:, j:w - k + 1 + j] for j in range(k))


def ssim(a: np.ndarray, b: np.ndarray, data_range: float = 1.0) -> float:
    x, y = luminance(a), luminance(b)
    if x.shape != y.shape:
        raise ValueError("ssim: shape mismatch")
    g = _gauss_window()
    c1, c2 = (0.01 * data_range) ** 2, (0.03 * data_range) ** 2
    mx, my = _filter_valid(x, g), _filter_valid(y, g)
    sxx = _filter_valid(x * x, g) - mx * mx
    syy = _filter_valid(y * y, g) - my * my
    sxy = _filter_valid(x * y, g) - mx * my
    s = ((2 * mx * my + c1) * (2 * sxy + c2)) / ((mx * mx + my * my + c1) * (sxx + syy + c2))
    return float(np.mean(s))

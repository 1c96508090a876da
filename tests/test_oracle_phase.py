"""SPEC acceptance criterion 1: the HG pdf integrates to 1 within
1e-4 for 8 values of g, and the sampler agrees with the pdf (chi-square at
alpha = 0.01, 1e5 samples per g).  Uses the oracle's hg_eval / hg_sample_cos,
which are bit-identical to the reference's phase.hpp (test_oracle_trace.py)."""
import numpy as np
import pytest
from scipy import stats

GS = [-0.95, -0.75, -0.35, 0.0, 0.2, 0.5, 0.75, 0.9]


@pytest.mark.parametrize("g", GS)
def test_hg_normalisation(oracle, g):
    # 2 pi * integral_{-1}^{1} p(c) dc (adaptive quadrature; strongly peaked for |g| -> 1)
    from scipy import integrate
    f = oracle.lib().or_hg_eval
    val, _ = integrate.quad(lambda x: f(g, x), -1.0, 1.0, limit=400, epsabs=1e-12, epsrel=1e-10,
                            points=[-1.0 + 1e-3, 1.0 - 1e-3])
    assert abs(2 * np.pi * val - 1.0) < 1e-4


@pytest.mark.parametrize("g", GS)
def test_hg_sampler_matches_pdf(oracle, g):
    r = np.random.default_rng(7)
    u = r.random(100_000)
    cos = np.array([oracle.lib().or_hg_sample_cos(g, float(x)) for x in u])
    edges = np.linspace(-1.0, 1.0, 41)
    obs, _ = np.histogram(cos, bins=edges)
    # expected bin mass from the analytic HG cdf in cos theta
    g2 = max(-0.999, min(0.999, g))

    def cdf(x):
        if abs(g2) < 1e-6:
            return (x + 1.0) / 2.0
        return (1 - g2 * g2) / (2 * g2) * (1 / np.sqrt(1 + g2 * g2 - 2 * g2 * x) - 1 / (1 + g2))

    exp = np.diff([cdf(x) for x in edges]) * len(u)
    keep = exp > 5
    pv = stats.chisquare(obs[keep], exp[keep] * obs[keep].sum() / exp[keep].sum()).pvalue
    assert pv > 0.01, pv

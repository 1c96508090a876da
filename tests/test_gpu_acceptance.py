"""SPEC acceptance criteria 6-10 end to end on the GPU:
photon tracing (Alg. 1) -> staggered field training -> neural, photon-map and
path-traced renders of the 64^3 synthetic slab (tools/acceptance_run.py).

Scale note: the SPEC's photon power is per emitted photon with emission
restricted to the box's bounding cone and Eq. 6 has no 1/sigma_s, so the
photon map (and the field trained on it) and the path tracer differ by a
constant factor; "acceptance tests use relative comparisons".
Noise is therefore compared as variance / mean^2 (criterion 8), SSIM uses the
reference image's luminance range (linear radiance).
"""
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))


@pytest.fixture(scope="module")
def report(ctx):
    import acceptance_run
    rep = acceptance_run.run(ctx)
    print(rep)
    return rep


def test_a6_staggered_training_learns(report):
    first, last = report["train_loss_first_last"]
    assert last < 1e-2 * first


def test_a7_reconstruction_fidelity(report):
    """Neural vs photon-map render, same seed, 16 spp, 64x64: SSIM >= 0.85 (mean rSE reported)."""
    assert report["A7_ssim"] >= 0.85
    assert report["A7_ssim_Li_only"] >= 0.85
    assert report["A7_mean_rse"] < 0.05


def test_a8_noise_ordering(report):
    """16 independent 1-spp renders: the field's smooth L_i is less noisy than the
    path tracer's continuation (relative per-pixel luminance variance)."""
    assert report["A8_relvar_neural_1spp"] < report["A8_relvar_pt_1spp"]


def test_a9_cost_scaling(report):
    """The path tracer's time grows with max_bounces; render_neural has no such parameter."""
    t = report["A9_pt_trace_ms"]
    t = {int(k): v for k, v in t.items()}
    assert t[2] < t[4] < t[8]
    assert t[16] >= 0.98 * t[8]
    assert report["A9_neural_ms"] < t[16]


def test_a10_phase_generalisation(report):
    """Unseen g = +-0.35 (not in G): mean SSIM no more than 0.1 below the mean at trained g."""
    trained = report["A10_ssim_trained_g"]
    unseen = report["A10_ssim_unseen_g"]
    assert sum(unseen) / len(unseen) >= sum(trained) / len(trained) - 0.1

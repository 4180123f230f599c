"""Acceptance criterion 7 of the reference (test_acceptance.py:226-251) on the GPU
path: upscale-aware training on the reference's self-reconstruction target
(tests/golden/recon_target.npz, made by the reference) reaches full-resolution
quality at x2 and the analytic-gradient spline beats classical bicubic (FD
slopes) at x4 — the paper's claim, end to end through fit()."""

import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def test_training_with_upscaling():
    from paper_2503_14171_b200 import fit as F
    target = golden("recon_target")["target"]

    def run(mode, scale, seed):
        cfg = F.FitConfig(iterations=2000, num_gaussians=12, render_scale=scale, upscale_mode=mode, seed=seed,
                          log_every=1999)
        return F.fit(target, cfg).rows[-1].psnr

    full = run("none", 1.0, 0)
    s2 = run("spline_analytic", 2.0, 0)
    wins = sum(run("spline_analytic", 4.0, seed) >= run("bicubic_fd", 4.0, seed) for seed in range(5))
    assert full >= 35.0, full
    assert s2 >= full - 1.5, (s2, full)
    assert wins >= 4, wins

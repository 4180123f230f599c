"""invert_alpha_state (raster_backward.py:56-70) — acceptance criterion 4
(test_acceptance.py:159-175): random blend chains invert back to every forward
state; the precondition 1 - alpha >= 1e-3 raises ParameterError.  Host float64."""

import numpy as np
import pytest


def _forward_chain(alphas, dxs, dys, dxys):
    """A-state recurrences of the forward blend (_kernels.py:88-109)."""
    a = ax = ay = axy = 0.0
    states = [(a, ax, ay, axy)]
    for al, gx, gy, gxy in zip(alphas, dxs, dys, dxys):
        t, om = 1.0 - a, 1.0 - al
        a, ax, ay, axy = (a + al * t, ax * om + t * gx, ay * om + t * gy,
                          axy * om + t * gxy - ax * gy - ay * gx)
        states.append((a, ax, ay, axy))
    return states


def test_round_trip():
    from paper_2503_14171_b200 import invert_alpha_state
    rng = np.random.default_rng(99)
    worst = 0.0
    for _ in range(200):
        n = int(rng.integers(1, 50))
        alphas = rng.uniform(0.0, 0.95, n)
        # stop where the reference would terminate (1 - A < 1e-4)
        acc, keep = 0.0, 0
        for al in alphas:
            acc += al * (1.0 - acc)
            keep += 1
            if 1.0 - acc < 1e-4:
                break
        alphas = alphas[:keep]
        dxs, dys, dxys = rng.normal(0, 0.3, keep), rng.normal(0, 0.3, keep), rng.normal(0, 0.1, keep)
        states = _forward_chain(alphas, dxs, dys, dxys)
        cur = states[-1]
        for i in range(keep - 1, -1, -1):
            cur = invert_alpha_state(*cur, alphas[i], dxs[i], dys[i], dxys[i])
            worst = max(worst, float(np.abs(np.array(cur) - np.array(states[i])).max()))
    assert worst < 1e-8, worst


def test_precondition():
    from paper_2503_14171_b200 import invert_alpha_state
    from paper_2503_14171_b200.core import ParameterError
    with pytest.raises(ParameterError):
        invert_alpha_state(0.5, 0.0, 0.0, 0.0, 0.9995, 0.0, 0.0, 0.0)

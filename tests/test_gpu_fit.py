"""The single-image fit driver against the reference's own
fit() runs (tests/golden/fit_*.npz, made by make_golden.py): same rows, same
pruning, same fitted scene within float32 tolerances, in all three upscale modes."""

import ast
import io

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

FIELDS = ("means", "log_scales", "rotations", "opacity_logits", "colors", "depths")


@pytest.mark.parametrize("name", ["spline", "fd", "none"])
def test_fit_matches_reference(name):
    from paper_2503_14171_b200 import fit as F
    g = golden("fit_" + name)
    kw = ast.literal_eval(str(g["cfg"]))
    rep = F.fit(g["target"], F.FitConfig(**kw))
    rows = np.array([[r.iteration, r.loss, r.psnr, r.ssim] for r in rep.rows])
    ref = g["rows"]
    assert rows.shape == ref.shape
    assert np.array_equal(rows[:, 0], ref[:, 0])
    assert np.allclose(rows[:, 1], ref[:, 1], rtol=2e-4, atol=0), (rows[:, 1], ref[:, 1])
    assert np.allclose(rows[:, 2], ref[:, 2], atol=5e-3), (rows[:, 2], ref[:, 2])
    assert np.allclose(rows[:, 3], ref[:, 3], atol=5e-4), (rows[:, 3], ref[:, 3])
    sc = rep.scene
    assert sc.n == len(g["depths"])                         # identical pruning
    assert np.array_equal(sc.depths, g["depths"])           # depths are never optimised
    for f in FIELDS:
        err = np.abs(getattr(sc, f) - g[f]).max()
        assert err < 1e-4, (f, err)   # measured <= 1.4e-6
    buf = io.StringIO()
    rep.write_csv(buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == ",".join(F.CSV_COLUMNS) and len(lines) == len(rep.rows) + 1


def test_fit_config_validation():
    from paper_2503_14171_b200 import fit as F
    from paper_2503_14171_b200.core import DimensionError, ParameterError
    for bad in (dict(iterations=0), dict(num_gaussians=0), dict(render_scale=0.5),
                dict(upscale_mode="lanczos"), dict(render_scale=2.0, upscale_mode="none"),
                dict(ssim_weight=1.5)):
        with pytest.raises(ParameterError):
            F.FitConfig(**bad)
    with pytest.raises(DimensionError):
        F.fit(np.zeros((8, 8, 3)), F.FitConfig(iterations=1))
    with pytest.raises(DimensionError):
        F.fit(np.zeros((0, 0, 3)), F.FitConfig(iterations=1))

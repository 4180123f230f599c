import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def golden_names(prefix: str):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def scene_of(g: dict):
    """A product Scene from a golden fixture's stored inputs."""
    from paper_2503_14171_b200.core import Scene
    rr = g["ref_res"]
    ref = (float(rr[0]), float(rr[1]))
    ref = tuple(int(v) if float(v).is_integer() else v for v in ref)
    return Scene(g["means"], g["log_scales"], g["rotations"], g["opacity_logits"],
                 g["colors"], g["depths"], g["background"], ref)


def ref_fixture_scene(seed, n, size=64, kind="sharp"):
    """conftest.sharp_scene / smooth_scene recipes of the reference
    (pkg/tests/conftest.py:7-42), restated so tests need no reference import."""
    from paper_2503_14171_b200.core import Scene, logit
    rng = np.random.default_rng(seed)
    if kind == "sharp":
        return Scene(means=rng.uniform(0, size, (n, 2)),
                     log_scales=np.log(rng.uniform(3.0, 10.0, (n, 2))),
                     rotations=rng.uniform(-np.pi, np.pi, n),
                     opacity_logits=logit(rng.uniform(0.1, 0.8, n)),
                     colors=rng.uniform(0.0, 1.0, (n, 3)),
                     depths=rng.uniform(0.0, 1.0, n),
                     background=rng.uniform(0.0, 1.0, 3),
                     reference_resolution=(size, size))
    sig_cap = 1.0 - 1e-3 ** (1.0 / n)
    sig = rng.uniform(0.3 * sig_cap, sig_cap, n)
    means = rng.uniform(0.2 * size, 0.8 * size, (n, 2))
    corner = np.sqrt(2.0) * 0.8 * size
    smin = corner / np.sqrt(2.0 * np.log(255.0 * sig.min()))
    scales = rng.uniform(smin * 1.05, smin * 1.6, (n, 2))
    return Scene(means=means, log_scales=np.log(scales), rotations=rng.uniform(-np.pi, np.pi, n),
                 opacity_logits=logit(sig), colors=rng.uniform(0.0, 1.0, (n, 3)),
                 depths=rng.uniform(0.0, 1.0, n), background=rng.uniform(0.0, 1.0, 3),
                 reference_resolution=(size, size))


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False

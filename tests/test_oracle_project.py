"""CPU checks of the oracle's EWA projection (the pin of csrc/project.cu):
closed forms that do not depend on the restatement itself."""

import numpy as np


def test_isotropic_on_axis(oracle):
    m, ls, rot, lg, z = oracle.project_gaussians([[0, 0, 5.0]], [[np.log(0.02)] * 3], [[1, 0, 0, 0]], [0.3],
                                                 np.eye(3), np.zeros(3), 500.0, 400.0, 80.0, 60.0, 0.1)
    assert np.allclose(m, [[80.0, 60.0]]) and z[0] == 5.0 and lg[0] == 0.3
    # fx != fy: major axis along x with sigma_x = fx s / z, minor along y with fy s / z
    assert np.allclose(ls[0], [np.log(500 * 0.02 / 5), np.log(400 * 0.02 / 5)])
    assert abs(rot[0]) < 1e-15


def test_rotated_anisotropic_in_plane(oracle):
    # a Gaussian elongated along world x, rotated by 30 degrees about the optical axis
    th = np.radians(30.0)
    q = [np.cos(th / 2), 0.0, 0.0, np.sin(th / 2)]
    m, ls, rot, lg, z = oracle.project_gaussians([[0, 0, 4.0]], [[np.log(0.05), np.log(0.01), np.log(0.01)]],
                                                 [q], [0.0], np.eye(3), np.zeros(3), 400.0, 400.0, 0.0, 0.0, 0.1)
    assert np.allclose(ls[0], [np.log(400 * 0.05 / 4), np.log(400 * 0.01 / 4)])
    assert np.isclose(rot[0], th)


def test_behind_camera_is_culled(oracle):
    m, ls, rot, lg, z = oracle.project_gaussians([[0, 0, -1.0], [0, 0, 0.05]], np.zeros((2, 3)),
                                                 [[1, 0, 0, 0]] * 2, [2.0, 2.0], np.eye(3), np.zeros(3),
                                                 100.0, 100.0, 10.0, 10.0, 0.1)
    assert np.all(lg == -100.0)
    assert 1.0 / (1.0 + np.exp(100.0)) < 1.0 / 255.0   # invalid under the reference's opacity cull

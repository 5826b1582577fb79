"""GPU: failure behaviour through the C ABI, with the reference's exception
classes (errors.py): empty and degenerate inputs, singular kernel moment
matrices (collinear particles), element inversion during a step, and
invalid arguments -- raised, never silently computed."""

import numpy as np
import pytest

from paper_2309_04010_b200 import errors

pytestmark = pytest.mark.gpu


def _solid(pos, vol, **kw):
    from paper_2309_04010_b200.device import DeviceSolid
    n, d = pos.shape
    return DeviceSolid(pos, vol, 1.0, np.zeros(n, bool), np.zeros(n, np.int8), None,
                       [1.3 * 0.01] * d, 1.0, 2.0, plastic=False, **kw)


def test_empty_particle_set_is_rejected():
    with pytest.raises(ValueError, match="empty"):
        _solid(np.zeros((0, 3)), np.zeros(0))


def test_non_positive_volume_is_a_geometry_error():
    pos = np.stack(np.meshgrid(*[np.arange(4) * 0.01] * 3, indexing="ij"), -1).reshape(-1, 3)
    vol = np.full(len(pos), 1e-6)
    vol[5] = 0.0
    with pytest.raises(errors.GeometryError):
        _solid(pos, vol)


def test_collinear_particles_have_singular_moment_matrices():
    pos = np.zeros((12, 3))
    pos[:, 0] = np.arange(12) * 0.01                  # a line: rank-1 moments
    with pytest.raises(errors.SingularMomentMatrixError) as ei:
        _solid(pos, np.full(12, 1e-6))
    assert len(ei.value.particle_ids) > 0


def test_inverted_element_raises_with_particle_ids():
    pos = np.stack(np.meshgrid(*[np.arange(6) * 0.01] * 3, indexing="ij"), -1).reshape(-1, 3)
    s = _solid(pos, np.full(len(pos), 1e-6), sweep="tiled")
    F = np.broadcast_to(np.eye(3), (len(pos), 3, 3)).copy()
    F[7] = np.diag([1.0, 1.0, -1.0])                  # det F < 0
    s.set("F", F)
    with pytest.raises(errors.ElementInversionError) as ei:
        s.relax_step(1e-9, 0.0)
    assert 7 in ei.value.particle_ids


def test_invalid_arguments_are_value_errors():
    pos = np.stack(np.meshgrid(*[np.arange(4) * 0.01] * 3, indexing="ij"), -1).reshape(-1, 3)
    s = _solid(pos, np.full(len(pos), 1e-6), sweep="tiled")
    with pytest.raises(ValueError):
        s.set_precision(16)
    with pytest.raises(ValueError):
        s.run_steps(0, 1.0, 0.2)
    with pytest.raises(ValueError):
        s.phase("sweep", 63)                          # colour out of range

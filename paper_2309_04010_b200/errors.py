"""Error classes of the drop-in API.

Names, attributes (`particle_ids`, `dets`, `residuals`) and message texts
follow the reference's errors.py so callers that catch or match them keep
working; `BackendError` is new (the CUDA library is missing or failed).
"""


def _first_ids(ids, limit=10):
    return ", ".join(str(i) for i in list(ids)[:limit])


class MtsphError(Exception):
    pass


class ConfigError(MtsphError):
    pass


class GeometryError(MtsphError):
    pass


class SimulationError(MtsphError):
    pass


class BackendError(MtsphError):
    pass


class _ParticleError(MtsphError):
    what = ""

    def __init__(self, particle_ids):
        self.particle_ids = list(particle_ids)
        super().__init__(f"{self.what} {len(self.particle_ids)} particle(s), "
                         f"first ids: [{_first_ids(self.particle_ids)}]")


class SingularMomentMatrixError(_ParticleError):
    what = "singular kernel moment matrix at"

    def __init__(self, particle_ids, dets):
        super().__init__(particle_ids)
        self.dets = list(dets)


class ElementInversionError(_ParticleError):
    what = "non-positive deformation determinant at"


class ReturnMapError(_ParticleError):
    what = "return mapping did not converge at"

    def __init__(self, particle_ids, residuals):
        super().__init__(particle_ids)
        self.residuals = list(residuals)

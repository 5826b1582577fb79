"""Material models of the drop-in API.

ElasticModel   ~ reference solids.py:23  (mu, K, E, nu, rho0; sound speed)
HardeningModel ~ reference plasticity.py:27 (saturation + linear hardening),
                 plus the BASELINE power law  k(a) = s0 (1 + a/e0)^m
MembraneModel  ~ reference porous.py:27  (Table 3 Nafion parameters)
"""

from __future__ import annotations

import math
from dataclasses import dataclass

_TOL = 1e-10


@dataclass(frozen=True)
class ElasticModel:
    shear_modulus: float
    bulk_modulus: float
    youngs_modulus: float
    poisson_ratio: float
    density0: float

    def __post_init__(self):
        mu, k, e, nu = self.shear_modulus, self.bulk_modulus, self.youngs_modulus, self.poisson_ratio
        if min(mu, k, e, self.density0) <= 0.0:
            raise ValueError("moduli and density must be positive")
        if abs(e - 2.0 * mu * (1.0 + nu)) > _TOL * e or abs(e - 3.0 * k * (1.0 - 2.0 * nu)) > _TOL * e:
            raise ValueError("inconsistent elastic constants")

    @classmethod
    def from_shear_bulk(cls, shear_modulus, bulk_modulus, density0):
        mu, k = float(shear_modulus), float(bulk_modulus)
        nu = (3.0 * k - 2.0 * mu) / (2.0 * (3.0 * k + mu))
        return cls(mu, k, 2.0 * mu * (1.0 + nu), nu, float(density0))

    @classmethod
    def from_youngs_poisson(cls, youngs_modulus, poisson_ratio, density0):
        e, nu = float(youngs_modulus), float(poisson_ratio)
        return cls(e / (2.0 * (1.0 + nu)), e / (3.0 * (1.0 - 2.0 * nu)), e, nu, float(density0))

    @property
    def sound_speed(self) -> float:
        return math.sqrt(self.bulk_modulus / self.density0)

    @property
    def lame_lambda(self) -> float:
        return self.bulk_modulus - 2.0 * self.shear_modulus / 3.0


@dataclass(frozen=True)
class HardeningModel:
    """law 'saturation': k = s0 + (sinf - s0)(1 - exp(-delta a)) + H a
    law 'power':      k = s0 (1 + a / e0)^m   (BASELINE configs 0/2/4)"""

    initial_flow_stress: float
    saturation_flow_stress: float = 0.0
    saturation_exponent: float = 1.0
    linear_coefficient: float = 0.0
    law: str = "saturation"
    reference_strain: float = 1.0
    exponent: float = 0.0

    def __post_init__(self):
        if not self.initial_flow_stress > 0.0:
            raise ValueError("initial flow stress must be positive")
        if self.law == "saturation":
            if self.saturation_flow_stress < self.initial_flow_stress:
                raise ValueError("saturation flow stress must be >= initial")
            if not self.saturation_exponent > 0.0:
                raise ValueError("saturation exponent must be positive")
            if self.linear_coefficient < 0.0:
                raise ValueError("linear hardening coefficient must be >= 0")
        elif self.law == "power":
            if not self.reference_strain > 0.0 or self.exponent < 0.0:
                raise ValueError("power law needs e0 > 0 and m >= 0")
        else:
            raise ValueError(f"unknown hardening law {self.law!r}")

    def device_params(self):
        """(law id, p[4]) as consumed by the CUDA return map."""
        if self.law == "power":
            return 1, (self.initial_flow_stress, self.reference_strain, self.exponent, 0.0)
        return 0, (self.initial_flow_stress, self.saturation_flow_stress,
                   self.saturation_exponent, self.linear_coefficient)

    def k(self, alpha):
        import numpy as np
        a = np.asarray(alpha, float)
        if self.law == "power":
            return self.initial_flow_stress * (1.0 + a / self.reference_strain) ** self.exponent
        s0, sinf = self.initial_flow_stress, self.saturation_flow_stress
        return s0 + (sinf - s0) * (1.0 - np.exp(-self.saturation_exponent * a)) \
            + self.linear_coefficient * a


@dataclass(frozen=True)
class MembraneModel:
    density0: float
    diffusivity: float
    pressure_coeff: float
    youngs_modulus: float
    poisson_ratio: float
    porosity: float
    fluid_density0: float
    initial_saturation: float

    def __post_init__(self):
        if min(self.density0, self.diffusivity, self.pressure_coeff, self.youngs_modulus,
               self.fluid_density0) <= 0.0:
            raise ValueError("material constants must be positive")
        if not 0.0 < self.porosity < 1.0:
            raise ValueError("porosity must lie in (0, 1)")
        if not 0.0 <= self.initial_saturation <= self.porosity:
            raise ValueError("initial saturation must lie in [0, porosity]")

    @property
    def elastic(self) -> ElasticModel:
        return ElasticModel.from_youngs_poisson(self.youngs_modulus, self.poisson_ratio, self.density0)

    @property
    def shear_modulus(self):
        return self.elastic.shear_modulus

    @property
    def bulk_modulus(self):
        return self.elastic.bulk_modulus

    @property
    def lame_lambda(self):
        return self.bulk_modulus - 2.0 * self.shear_modulus / 3.0

    @property
    def sound_speed(self):
        return math.sqrt(self.bulk_modulus / self.density0)

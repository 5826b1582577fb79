"""B200-native multi-rate SPH hot path (arXiv 2309.04010).

Drop-in for the reference package's driver path: case config ->
particle generation -> outer/inner time loop -> observers, with the inner
solid relaxation (kick/drift, deformation rate, J2 / Neo-Hookean stress,
stress divergence, pairwise implicit damping) and the outer diffusion
update running as hand-written sm_100a CUDA kernels behind the C ABI in
include/mtsph_b200.h.  There is no CPU fallback.
"""

__version__ = "0.1.0"

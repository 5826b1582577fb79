#pragma once
// TEMPORARY stubs (replaced by the real implementation)
extern "C" mtsph_status mtsph_velocity_gradient_gather(int64_t, int, const double*, const int64_t*, const int64_t*, const double*, const double*, double*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_pair_tensor_divergence(int64_t, int, const double*, const int64_t*, const int64_t*, const double*, const double*, double*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_pair_tensor_divergence_mapped(int64_t, int, const double*, const double*, const int64_t*, const int64_t*, const double*, const double*, double*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_scalar_difference_flux(int64_t, int, const double*, const double*, const double*, const int64_t*, const int64_t*, const double*, const double*, double*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_damping_sweep(int64_t, int, double*, int64_t, const int64_t*, const int64_t*, const double*, const double*, const double*, int64_t, const int64_t*, double, double) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_conservative_mass_rate(int64_t, int, const double*, const double*, int64_t, const int64_t*, const int64_t*, const double*, const double*, double*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_porous_stress_rhs(int64_t, int, const double*, const double*, const double*, const int64_t*, const int64_t*, const double*, const double*, double, double, double*, double*, double*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }

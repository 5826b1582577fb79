#pragma once
// TEMPORARY stubs (replaced by the real implementation)
extern "C" mtsph_status mtsph_porous_create(const mtsph_porous_desc*, mtsph_porous**) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_porous_destroy(mtsph_porous*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_porous_advance_slow(mtsph_porous*, double, double, int64_t*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_porous_stable_dt(mtsph_porous*, double, double*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_porous_relax_step(mtsph_porous*, double, double, double*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_porous_relax(mtsph_porous*, const mtsph_inner_params*, mtsph_inner_result*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_porous_refresh_velocities(mtsph_porous*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_porous_get(mtsph_porous*, const char*, double*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_porous_set(mtsph_porous*, const char*, const double*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }
extern "C" mtsph_status mtsph_porous_launches(const mtsph_porous*, int64_t*) { return fail(MTSPH_ERR_ARG, "not implemented yet"); }

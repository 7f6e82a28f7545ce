// Host helpers shared by the driver and the reference-file C ABI (reference_io.cpp).
#pragma once

#include "hwwg.h"

namespace hwwg {

// hww::run_step's diagnostics (proj/src/driver.cpp:231-275): fills rec's metric
// fields from rec->tau and rec->sigma_valid. ref_interval == NULL: no reference
// (only fom_sigma_l2). phi_hybrid == NULL: no hybrid solve this step.
void step_metrics(int cells, const double* edges, const double* phi_track,
                  const double* phi_sigma, const double* phi_hybrid, const double* ref_interval,
                  const double* ref_layer, const double* ref_layer_prev, hwwg_step_record* rec);

// hww::load_reference (proj/src/reference.cpp:395-456); throws ApiError(HWWG_EFORMAT).
void load_reference(const char* path, int cells, const double* edges, int steps,
                    const double* layers, double* phi_layer, double* phi_interval);

// TimeGrid::uniform(0, t_end, steps) layers.
void uniform_layers(double t_end, int steps, double* layers);

}  // namespace hwwg

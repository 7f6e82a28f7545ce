// Host-side helpers of the driver (host.cpp): source sampling, stream ids,
// mesh location — the sequential pieces the reference runs once per run/step.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "hwwg.h"

namespace hwwg {

// sample_pulse_source (transport.cpp:13-22) with the driver's source stream
// spawn_stream(seed, stream_id(0, 0, source)) (driver.cpp:309-316).
void sample_pulse_source_host(uint64_t seed, uint64_t histories, double x0, double total_weight,
                              double t0, hwwg_particle* out);
uint64_t stream_id_host(uint64_t step, uint64_t history, uint64_t purpose);
// Config-3 volumetric source particles of one step and the step's LOSM q.
void sample_volume_source_host(uint64_t seed, int step, uint64_t n, double x_lo, double x_hi,
                               double ta, double tb, double rate, uint64_t h_cfg,
                               hwwg_particle* out);
void volume_q_host(const double* edges, int I, double x_lo, double x_hi, double ta, double tb,
                   double dt, double rate, double* q);
// batch_of (tally.hpp:130-134) on the host.
int batch_of_host(uint64_t h, uint64_t H, int B);
// Mesh1D::locate (mesh.cpp:26-40) on the host; -1 outside.
int locate_host(const std::vector<double>& edges, double x);
// lww: windows active iff build_centers did not fall back (flags[5]).
void set_active_from_fallback(int* flags, cudaStream_t s);

}  // namespace hwwg

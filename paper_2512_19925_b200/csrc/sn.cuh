// Deterministic discrete-ordinates reference on the device.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "hwwg.h"

namespace hwwg {

// hww::SnProblem (reference.hpp:21-34) on host memory, plus the optional
// projection onto a nesting tally grid (hww::project, reference.cpp:258-300).
struct SnHostProblem {
  std::vector<double> edges;               // fine mesh, cells+1
  std::vector<hwwg_material> materials;    // per fine cell
  std::vector<double> layers;              // fine time layers, steps+1
  int order = 16;                          // Gauss-Legendre order K
  std::vector<double> psi0;                // K*cells, [k*cells + i]
  std::vector<double> inc_left, inc_right; // K
  // isotropic source density per fine cell: q_rows[q_index[n]*cells ...] in
  // step n, none when q_index[n] < 0 (the reference's q is constant in time:
  // one row indexed by every step)
  std::vector<double> q_rows;
  std::vector<int> q_index;                // steps+1 (entry 0 unused)
  double tolerance = 1e-9;
  int max_iterations = 1000;
  // projection (tally_cells == 0: none): fine cells f*sr..f*sr+sr-1 nest tally
  // cell f, and every `ratio` fine steps make one tally step
  int tally_cells = 0, sr = 1, ratio = 1;
  std::vector<double> tally_edges;
};

// GaussLegendre::order (reference.cpp:14-42), same host arithmetic.
void gauss_legendre(int n, double* mu, double* weight);

// hww::sn_solve (reference.cpp:151-233) on `device`/`stream`; any output may be
// null: phi_fine[(steps+1)*cells] scalar flux per fine layer, iterations[steps+1]
// (entry 0 = 0), phi_layer[(N+1)*I] / phi_interval[N*I] the projection.
// Throws ApiError(HWWG_ESINGULAR) on non-convergence with the reference's message.
void sn_solve_device(const SnHostProblem& p, int device, cudaStream_t stream, double* phi_fine,
                     int* iterations, double* phi_layer, double* phi_interval);

// hww::compute_reference (reference.cpp:364-372): pulse_problem + load_pulse_ic
// (reference.cpp:302-356) for cfg, with the engine's config-3 extensions
// (material regions per tally cell, the time-boxed volumetric source as q, no_pulse).
SnHostProblem reference_problem(const hwwg_run_config& cfg, int space_refine, int time_refine,
                                int sn_order);

}  // namespace hwwg

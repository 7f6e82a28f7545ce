// Host-side owners of device memory shared by the segment API and the driver.
#pragma once

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace hwwg {

// Grow-only device allocation.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void reserve(size_t count) {
    if (count <= n) return;
    if (p) HWWG_CUDA(cudaFree(p));
    p = nullptr;
    n = 0;
    if (count) {
      cudaError_t e = cudaMalloc(&p, count * sizeof(T));
      if (e != cudaSuccess) {
        cudaGetLastError();
        if (std::getenv("HWWG_ALLOC_DEBUG")) {
          size_t fr = 0, tot = 0;
          cudaMemGetInfo(&fr, &tot);
          std::fprintf(stderr, "[hwwg] cudaMalloc of %zu bytes failed (%zu free of %zu)\n",
                       count * sizeof(T), fr, tot);
        }
        throw std::bad_alloc();
      }
    }
    n = count;
  }
  // Keeps the first `keep` elements when growing.
  void grow_keep(size_t count, size_t keep, cudaStream_t s) {
    if (count <= n) return;
    T* q = nullptr;
    cudaError_t e = cudaMalloc(&q, count * sizeof(T));
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw std::bad_alloc();
    }
    if (p && keep) HWWG_CUDA(cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (p) {
      HWWG_CUDA(cudaStreamSynchronize(s));
      HWWG_CUDA(cudaFree(p));
    }
    p = q;
    n = count;
  }
};

// Mesh + per-cell materials resident on the device (mesh.cpp:9-24 widths).
struct DeviceProblem {
  std::vector<double> edges;
  std::vector<hwwg_material> mats;
  std::vector<CellInfo> cells_h;
  DevBuf<double> d_edges;
  DevBuf<CellInfo> d_cells;
  MeshView view{};
  int I = 0;
  bool gen_uniform_homog = false;
  double w_gen = 0.0;

  // Validates (mesh.cpp:9-14, material.hpp:20-32 sigma_t > 0, speed > 0) and
  // uploads when the content changed. Returns false with `why` on bad input.
  bool set(const double* e, int cells, const hwwg_material* m, cudaStream_t s, std::string& why) {
    if (cells < 1 || !e || !m) {
      why = "mesh needs at least one cell";
      return false;
    }
    for (int i = 1; i <= cells; ++i)
      if (!(e[i] > e[i - 1])) {
        why = "mesh edges must be strictly increasing";
        return false;
      }
    for (int i = 0; i < cells; ++i)
      if (!(m[i].sigma_t > 0) || !(m[i].speed > 0)) {
        why = "sigma_t and speed must be > 0";
        return false;
      }
    const bool same = cells == I && std::memcmp(edges.data(), e, sizeof(double) * (cells + 1)) == 0 &&
                      std::memcmp(mats.data(), m, sizeof(hwwg_material) * cells) == 0;
    if (same) return true;
    I = cells;
    edges.assign(e, e + cells + 1);
    mats.assign(m, m + cells);
    cells_h.resize(cells);
    std::vector<double> widths(cells);
    for (int c = 0; c < cells; ++c) widths[c] = edges[c + 1] - edges[c];
    bool uniform = true;
    for (int c = 0; c < cells; ++c)
      if (!(std::abs(widths[c] - widths[0]) <= 1e-12 * widths[0])) uniform = false;
    for (int c = 0; c < cells; ++c)
      cells_h[c] = CellInfo{mats[c].sigma_t, mats[c].sigma_s, mats[c].sigma_f,
                            mats[c].nu_f,    mats[c].speed,   1.0 / widths[c],
                            1.0 / mats[c].sigma_t, 1.0 / mats[c].speed,
                            mats[c].sigma_s > 0.0 ? 1.0 / mats[c].sigma_s : 0.0};
    d_edges.reserve(cells + 1);
    d_cells.reserve(cells);
    HWWG_CUDA(cudaMemcpyAsync(d_edges.p, edges.data(), sizeof(double) * (cells + 1),
                              cudaMemcpyHostToDevice, s));
    HWWG_CUDA(cudaMemcpyAsync(d_cells.p, cells_h.data(), sizeof(CellInfo) * cells,
                              cudaMemcpyHostToDevice, s));
    HWWG_CUDA(cudaStreamSynchronize(s));
    view = MeshView{d_edges.p, d_cells.p, cells, uniform ? 1 : 0, edges.front(), edges.back(),
                    widths[0]};
    // generated uniform mesh (mesh.cpp:42-50) with a single material?
    w_gen = (edges.back() - edges.front()) / cells;
    gen_uniform_homog = true;
    for (int e = 0; e < cells && gen_uniform_homog; ++e)
      if (edges[e] != edges.front() + e * w_gen) gen_uniform_homog = false;
    for (int c = 1; c < cells && gen_uniform_homog; ++c)
      if (std::memcmp(&mats[c], &mats[0], sizeof(hwwg_material)) != 0) gen_uniform_homog = false;
    return true;
  }
};

// One contiguous device block holding a TallySet + counters (zeroed with one
// memset, reduced across ranks with one collective).
struct DeviceTallies {
  int I = 0, B = 0;
  DevBuf<double> slab;
  size_t doubles = 0;
  TallyPtrs p{};

  void shape(int cells, int batches) {
    if (cells == I && batches == B && slab.p) return;
    I = cells;
    B = batches;
    // fp64 part | tracks (u64, I) | ucount (u64, 11) — all 8-byte words
    doubles = (size_t)I * 4 + (size_t)B * I + B + (I + 1) + 2 + 2;
    const size_t words = doubles + (size_t)I + kNumUCounters;
    slab.reserve(words);
    double* q = slab.p;
    p.track_flux = q; q += I;
    p.track_flux_batch = q; q += (size_t)B * I;
    p.census_phi = q; q += I;
    p.census_current = q; q += I;
    p.census_closure = q; q += I;
    p.census_weight_batch = q; q += B;
    p.edge_current = q; q += I + 1;
    p.boundary_closure = q; q += 2;
    p.dcount = q; q += 2;
    p.tracks = reinterpret_cast<unsigned long long*>(q); q += I;
    p.ucount = reinterpret_cast<unsigned long long*>(q);
  }
  size_t words() const { return doubles + (size_t)I + kNumUCounters; }
  void zero(cudaStream_t s) { HWWG_CUDA(cudaMemsetAsync(slab.p, 0, words() * 8, s)); }
};

// Host mirror of a DeviceTallies slab.
struct HostTallies {
  std::vector<double> w;  // raw words
  int I = 0, B = 0;
  size_t doubles = 0;
  void fetch(const DeviceTallies& d, cudaStream_t s) {
    I = d.I;
    B = d.B;
    doubles = d.doubles;
    w.resize(d.words());
    HWWG_CUDA(cudaMemcpyAsync(w.data(), d.slab.p, d.words() * 8, cudaMemcpyDeviceToHost, s));
    HWWG_CUDA(cudaStreamSynchronize(s));
  }
  const double* track_flux() const { return w.data(); }
  const double* track_flux_batch() const { return w.data() + I; }
  const double* census_phi() const { return track_flux_batch() + (size_t)B * I; }
  const double* census_current() const { return census_phi() + I; }
  const double* census_closure() const { return census_current() + I; }
  const double* census_weight_batch() const { return census_closure() + I; }
  const double* edge_current() const { return census_weight_batch() + B; }
  const double* boundary_closure() const { return edge_current() + I + 1; }
  const double* dcount() const { return boundary_closure() + 2; }
  const unsigned long long* tracks() const {
    return reinterpret_cast<const unsigned long long*>(dcount() + 2);
  }
  const unsigned long long* ucount() const { return tracks() + I; }
};

}  // namespace hwwg

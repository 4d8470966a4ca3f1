// Built-in analytic SDFs evaluated on the device (ground truth for the
// corner lattice, the metrics' oracle tracing and the bench workloads).
#pragma once

#include "common.cuh"

namespace ng {

// geometry.py:141-149 (sphere: norm - r; torus: hypot(hypot(x,z)-R, y) - r)
// and a closed polyline tube (SURVEY.md Appendix A torus knot).
__device__ __forceinline__ double sdf_builtin(int kind, const double* __restrict__ prm, int np_, double x, double y,
                              double z) {
  if (kind == 1) {
    double s = dadd(dadd(dmul(x, x), dmul(y, y)), dmul(z, z));
    return dsub(sqrt(s), prm[0]);
  }
  if (kind == 2) {
    double ring = dsub(hypot(x, z), prm[0]);
    return dsub(hypot(ring, y), prm[1]);
  }
  // polyline tube: params [tube, v0x, v0y, v0z, v1x, ...]
  int nv = (np_ - 1) / 3;
  const double* v = prm + 1;
  double best = INFINITY;
  for (int s = 0; s < nv; ++s) {
    int t = (s + 1 == nv) ? 0 : s + 1;
    double ax = v[3 * s], ay = v[3 * s + 1], az = v[3 * s + 2];
    double bx = v[3 * t] - ax, by = v[3 * t + 1] - ay, bz = v[3 * t + 2] - az;
    double px = x - ax, py = y - ay, pz = z - az;
    double bb = bx * bx + by * by + bz * bz;
    double h = (px * bx + py * by + pz * bz) / bb;
    h = fmin(fmax(h, 0.0), 1.0);
    double dx = px - h * bx, dy = py - h * by, dz = pz - h * bz;
    best = fmin(best, dx * dx + dy * dy + dz * dz);
  }
  return sqrt(best) - prm[0];
}

}  // namespace ng
